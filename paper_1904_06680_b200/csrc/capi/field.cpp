// field.cpp -- static/dynamic split and cell binning of the obstacle field
// (see field.hpp). Compiled with -ffp-contract=off: positions of the raw-
// points path are x + h * step exactly as the reference's extrapolate.
#include "field.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

namespace ppfield {

namespace {

size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// Clouds up to this size are not split when any point moves (one scan per
// state beats a static and a dynamic scan of a handful of points each).
constexpr int kSmall = 64;

// Common grid over every point of every row: cell size half the query
// window (g = cull / 2), a 2-D grid only for larger clouds, <= 4096 cells.
void choose_grid(Binned& b, double xmin, double xmax, double ymin, double ymax) {
  double g = 0.5 * b.cull;
  const bool two_d = b.points() >= 128;
  const double wx = xmax - xmin, wy = two_d ? ymax - ymin : 0.0;
  while ((std::floor(wx / g) + 1) * (two_d ? std::floor(wy / g) + 1 : 1.0) > 4096.0) g *= 1.25;
  b.g = g;
  b.x0 = xmin;
  b.y0 = ymin;
  b.nx = static_cast<int>(std::floor(wx / g)) + 1;
  b.ny = two_d ? static_cast<int>(std::floor(wy / g)) + 1 : 1;
}

int cell_of(const Binned& b, double x, double y) {
  const int cx = std::min(b.nx - 1, std::max(0, static_cast<int>(std::floor((x - b.x0) / b.g))));
  const int cy =
      b.ny == 1 ? 0 : std::min(b.ny - 1, std::max(0, static_cast<int>(std::floor((y - b.y0) / b.g))));
  return cx * b.ny + cy;
}

// Stable counting sort of n points (xy) into `out` (cell order) + starts.
void bin(const Binned& b, const double* xy, int n, double* out, int32_t* starts,
         std::vector<int32_t>& cell, std::vector<int32_t>& fill) {
  const int cells = b.cells();
  cell.resize(n);
  fill.assign(cells + 1, 0);
  for (int j = 0; j < n; ++j) {
    cell[j] = cell_of(b, xy[2 * j], xy[2 * j + 1]);
    ++fill[cell[j] + 1];
  }
  for (int c = 0; c < cells; ++c) fill[c + 1] += fill[c];
  std::copy(fill.begin(), fill.end(), starts);
  for (int j = 0; j < n; ++j) {
    const int at = fill[cell[j]]++;
    out[2 * at] = xy[2 * j];
    out[2 * at + 1] = xy[2 * j + 1];
  }
}

void finish(Binned& b, const std::vector<double>& s_xy, const std::vector<double>& d_xy) {
  double xmin = 0, xmax = 0, ymin = 0, ymax = 0;
  bool first = true;
  const auto see = [&](const std::vector<double>& v) {
    for (size_t i = 0; i + 1 < v.size(); i += 2) {
      const double x = v[i], y = v[i + 1];
      if (!(std::isfinite(x) && std::isfinite(y))) {
        throw std::invalid_argument("obstacle field has non-finite coordinates");
      }
      if (first || x < xmin) xmin = x;
      if (first || x > xmax) xmax = x;
      if (first || y < ymin) ymin = y;
      if (first || y > ymax) ymax = y;
      first = false;
    }
  };
  see(s_xy);
  see(d_xy);
  choose_grid(b, xmin, xmax, ymin, ymax);
  const int cells = b.cells();
  std::vector<int32_t> cell, fill;
  b.spts.resize(2 * static_cast<size_t>(b.Ns));
  b.sst.assign(cells + 1, 0);
  if (b.Ns > 0) bin(b, s_xy.data(), b.Ns, b.spts.data(), b.sst.data(), cell, fill);
  b.dpts.resize(2 * static_cast<size_t>(b.Nd) * b.rows);
  b.dst.assign(static_cast<size_t>(b.rows) * (cells + 1), 0);
  if (b.Nd > 0) {
    for (int r = 0; r < b.rows; ++r) {
      const size_t o = static_cast<size_t>(r) * b.Nd * 2;
      bin(b, d_xy.data() + o, b.Nd, b.dpts.data() + o, b.dst.data() + static_cast<size_t>(r) * (cells + 1),
          cell, fill);
    }
  }
}

}  // namespace

Layout layout(const Binned& b, size_t elem) {
  Layout l;
  l.dpts = align16(2 * elem * b.Ns);
  l.sst = align16(l.dpts + 2 * elem * static_cast<size_t>(b.Nd) * b.rows);
  l.dst = align16(l.sst + sizeof(int32_t) * (b.cells() + 1));
  l.bytes = align16(l.dst + sizeof(int32_t) * static_cast<size_t>(b.rows) * (b.cells() + 1));
  return l;
}

void from_rows(Binned& b, const double* xy, int rows, int N, double cull) {
  b = Binned{};
  b.rows = rows;
  b.cull = cull;
  std::vector<char> moving(N, 0);
  const size_t len = 2 * static_cast<size_t>(N);
  for (int r = 1; r < rows; ++r) {
    const double* row = xy + r * len;
    for (int j = 0; j < N; ++j) {
      if (!moving[j] && (std::memcmp(row + 2 * j, xy + 2 * j, 2 * sizeof(double)) != 0)) {
        moving[j] = 1;
      }
    }
  }
  // small mixed clouds stay one scan per state: every point dynamic
  if (N <= kSmall && std::count(moving.begin(), moving.end(), 1) > 0) {
    std::fill(moving.begin(), moving.end(), 1);
  }
  std::vector<double> s_xy, d_xy;
  std::vector<int> dyn;
  for (int j = 0; j < N; ++j) {
    if (moving[j]) {
      dyn.push_back(j);
    } else {
      s_xy.push_back(xy[2 * j]);
      s_xy.push_back(xy[2 * j + 1]);
    }
  }
  b.Ns = N - static_cast<int>(dyn.size());
  b.Nd = static_cast<int>(dyn.size());
  d_xy.resize(2 * static_cast<size_t>(b.Nd) * rows);
  for (int r = 0; r < rows; ++r) {
    for (int k = 0; k < b.Nd; ++k) {
      d_xy[(static_cast<size_t>(r) * b.Nd + k) * 2] = xy[r * len + 2 * dyn[k]];
      d_xy[(static_cast<size_t>(r) * b.Nd + k) * 2 + 1] = xy[r * len + 2 * dyn[k] + 1];
    }
  }
  finish(b, s_xy, d_xy);
}

void from_points(Binned& b, const double* pts4, int N, int rows, double T_s, double cull) {
  b = Binned{};
  b.rows = rows;
  b.cull = cull;
  std::vector<double> s_xy, d_xy;
  std::vector<int> dyn;
  std::vector<double> stepx, stepy;
  bool any_moving = false;
  for (int j = 0; j < N; ++j) {
    const double* p = pts4 + 4 * j;
    any_moving |= !(T_s * p[3] * std::cos(p[2]) == 0.0 && T_s * p[3] * std::sin(p[2]) == 0.0);
  }
  // small mixed clouds stay one scan per state: every point dynamic
  const bool all_dynamic = N <= kSmall && any_moving;
  for (int j = 0; j < N; ++j) {
    const double* p = pts4 + 4 * j;
    // src/geometry.cpp:51-52
    const double sx = T_s * p[3] * std::cos(p[2]);
    const double sy = T_s * p[3] * std::sin(p[2]);
    if (!all_dynamic && sx == 0.0 && sy == 0.0) {  // x + h * (+-0) == x: identical rows
      s_xy.push_back(p[0]);
      s_xy.push_back(p[1]);
    } else {
      dyn.push_back(j);
      stepx.push_back(sx);
      stepy.push_back(sy);
    }
  }
  b.Ns = static_cast<int>(s_xy.size() / 2);
  b.Nd = static_cast<int>(dyn.size());
  d_xy.resize(2 * static_cast<size_t>(b.Nd) * rows);
  for (int r = 0; r < rows; ++r) {
    for (int k = 0; k < b.Nd; ++k) {
      const double* p = pts4 + 4 * dyn[k];
      // src/geometry.cpp:53-57: x + h * step (int h promoted to double)
      d_xy[(static_cast<size_t>(r) * b.Nd + k) * 2] = p[0] + r * stepx[k];
      d_xy[(static_cast<size_t>(r) * b.Nd + k) * 2 + 1] = p[1] + r * stepy[k];
    }
  }
  finish(b, s_xy, d_xy);
}

void pack(const Binned& b, bool fp64, void* out) {
  const size_t elem = fp64 ? sizeof(double) : sizeof(float);
  const Layout l = layout(b, elem);
  unsigned char* base = static_cast<unsigned char*>(out);
  const auto put = [&](size_t off, const std::vector<double>& v) {
    if (fp64) {
      std::memcpy(base + off, v.data(), v.size() * sizeof(double));
    } else {
      float* f = reinterpret_cast<float*>(base + off);
      for (size_t i = 0; i < v.size(); ++i) f[i] = static_cast<float>(v[i]);
    }
  };
  put(0, b.spts);
  put(l.dpts, b.dpts);
  std::memcpy(base + l.sst, b.sst.data(), b.sst.size() * sizeof(int32_t));
  std::memcpy(base + l.dst, b.dst.data(), b.dst.size() * sizeof(int32_t));
}

bool collides(const Binned& b, const paraplan::ChassisPolytope& ch, int k, double x, double y,
              double phi) {
  if (b.points() == 0) return false;
  const auto cx_of = [&](double v) {
    return std::min(b.nx - 1, std::max(0, static_cast<int>(std::floor((v - b.x0) / b.g))));
  };
  const auto cy_of = [&](double v) {
    return b.ny == 1 ? 0
                     : std::min(b.ny - 1, std::max(0, static_cast<int>(std::floor((v - b.y0) / b.g))));
  };
  const int cx0 = cx_of(x - b.cull), cx1 = cx_of(x + b.cull);
  const int cy0 = cy_of(y - b.cull), cy1 = cy_of(y + b.cull);
  // src/geometry.cpp:63-76, expression by expression
  const double c = std::cos(phi), s = std::sin(phi);
  const double r2 = ch.bounding_radius() * ch.bounding_radius();
  const auto scan = [&](const double* pts, const int32_t* st) {
    for (int cx = cx0; cx <= cx1; ++cx) {
      for (int j = st[cx * b.ny + cy0]; j < st[cx * b.ny + cy1 + 1]; ++j) {
        const double dx = pts[2 * j] - x, dy = pts[2 * j + 1] - y;
        if (dx * dx + dy * dy >= r2) continue;
        if (ch.contains({c * dx + s * dy, -s * dx + c * dy})) return true;
      }
    }
    return false;
  };
  if (b.Ns > 0 && scan(b.spts.data(), b.sst.data())) return true;
  if (b.Nd > 0) {
    const int cells = b.cells();
    return scan(b.dpts.data() + static_cast<size_t>(k) * b.Nd * 2,
                b.dst.data() + static_cast<size_t>(k) * (cells + 1));
  }
  return false;
}

}  // namespace ppfield

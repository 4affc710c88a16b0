// field.cpp -- static/dynamic split and cell binning of the obstacle field
// (see field.hpp). Compiled with -ffp-contract=off: positions of the raw-
// points path are x + h * step exactly as the reference's extrapolate.
//
// Dense clouds put (H+1) x Nd dynamic positions through the binning (2.5M at
// N = 100k, 25% moving, H = 100): rows are binned in parallel on the host
// cores, each row independent.
#include "field.hpp"
#include "host_pool.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace ppfield {

namespace {

size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

// Clouds up to this size are not split when any point moves (one scan per
// state beats a static and a dynamic scan of a handful of points each).
constexpr int kSmall = 64;

double env_or(const char* name, double dflt) {
  const char* v = std::getenv(name);
  return v != nullptr ? std::atof(v) : dflt;
}

// f(i) for i in [0, n), on the process's host pool (host_pool.hpp) when
// `work` is large. Spawning threads per call instead cost ~1 ms per binning
// pass at C5's 100k points (measured: 2.7 ms of a 6.3 ms plan step).
// Loops nested in a parallel loop run serially on their worker.
// PARAPLAN_FIELD_SERIAL=1: every pass serial (tests compare the two).
thread_local bool tl_in_par = false;
bool field_serial() {
  static const bool v = env_or("PARAPLAN_FIELD_SERIAL", 0) != 0;
  return v;
}
template <class F>
void par_for(int n, size_t work, F&& f) {
  if (work < (size_t(1) << 17) || n <= 1 || tl_in_par || field_serial()) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  ppcapi::SharedPool& sp = ppcapi::shared_pool();
  std::lock_guard<std::mutex> turn(sp.mu);
  const std::function<void(int)> fn = [&](int i) {
    tl_in_par = true;
    f(i);
    tl_in_par = false;
  };
  sp.pool->run(n, fn);
}

struct BBox {
  double xmin = 0, xmax = 0, ymin = 0, ymax = 0;
  bool any = false;
  bool finite = true;
  void see(double x, double y) {
    if (!(std::isfinite(x) && std::isfinite(y))) {
      finite = false;
      return;
    }
    if (!any || x < xmin) xmin = x;
    if (!any || x > xmax) xmax = x;
    if (!any || y < ymin) ymin = y;
    if (!any || y > ymax) ymax = y;
    any = true;
  }
  void merge(const BBox& o) {
    finite &= o.finite;
    if (!o.any) return;
    see(o.xmin, o.ymin);
    see(o.xmax, o.ymax);
  }
};

// Common grid over every point of every row: cell size a fraction of the
// bounding radius (the query window is the chassis bounding box, about
// 2r x r), a 2-D grid only for larger clouds, <= 4096 cells.
void choose_grid(Binned& b, const BBox& box) {
  if (!box.finite) throw std::invalid_argument("obstacle field has non-finite coordinates");
  // tuning knobs (defaults measured on B200)
  static const double frac = env_or("PARAPLAN_GRID_FRAC", 0.25);
  static const double min2d = env_or("PARAPLAN_GRID2D_MIN", 128);
  double g = frac * b.cull;
  const bool two_d = b.points() >= min2d;
  const double wx = box.xmax - box.xmin, wy = two_d ? box.ymax - box.ymin : 0.0;
  while ((std::floor(wx / g) + 1) * (two_d ? std::floor(wy / g) + 1 : 1.0) > 4096.0) g *= 1.25;
  b.g = g;
  b.x0 = box.xmin;
  b.y0 = box.ymin;
  b.nx = static_cast<int>(std::floor(wx / g)) + 1;
  b.ny = two_d ? static_cast<int>(std::floor(wy / g)) + 1 : 1;
}

// Cell of a point (x-major). Queries cover the chassis box + g/8, so a point
// near a cell edge may land on either side of it.
struct CellOf {
  double x0, y0, inv;
  int nx, ny;
  explicit CellOf(const Binned& b) : x0(b.x0), y0(b.y0), inv(1.0 / b.g), nx(b.nx), ny(b.ny) {}
  static int clampi(double t, int n) { return t <= 0.0 ? 0 : std::min(n - 1, static_cast<int>(t)); }
  int operator()(double x, double y) const {
    return clampi((x - x0) * inv, nx) * ny + (ny == 1 ? 0 : clampi((y - y0) * inv, ny));
  }
};

// Stable counting sort of n points (xy) into `out` (cell order) + starts.
// Large inputs: per-block histograms, then each block scatters at its own
// offsets (the same stable order).
void bin(const Binned& b, const double* xy, int n, double* out, int32_t* starts,
         std::vector<int32_t>& cell) {
  const int cells = b.cells();
  const CellOf cell_of(b);
  constexpr int kBinBlock = 8192;
  if (n >= 4 * kBinBlock && !tl_in_par && !field_serial()) {
    const int nblk = (n + kBinBlock - 1) / kBinBlock;
    cell.resize(n);
    std::vector<int32_t> cnt(static_cast<size_t>(nblk) * cells, 0);
    par_for(nblk, static_cast<size_t>(n) * 4, [&](int k) {
      int32_t* ck = cnt.data() + static_cast<size_t>(k) * cells;
      for (int j = k * kBinBlock; j < std::min(n, (k + 1) * kBinBlock); ++j) {
        cell[j] = cell_of(xy[2 * j], xy[2 * j + 1]);
        ++ck[cell[j]];
      }
    });
    // starts, and per block its cursor into each cell (in place of cnt)
    int32_t run = 0;
    for (int c = 0; c < cells; ++c) {
      starts[c] = run;
      for (int k = 0; k < nblk; ++k) {
        const int32_t v = cnt[static_cast<size_t>(k) * cells + c];
        cnt[static_cast<size_t>(k) * cells + c] = run;
        run += v;
      }
    }
    starts[cells] = run;
    par_for(nblk, static_cast<size_t>(n) * 4, [&](int k) {
      int32_t* ck = cnt.data() + static_cast<size_t>(k) * cells;
      for (int j = k * kBinBlock; j < std::min(n, (k + 1) * kBinBlock); ++j) {
        const int at = ck[cell[j]]++;
        out[2 * at] = xy[2 * j];
        out[2 * at + 1] = xy[2 * j + 1];
      }
    });
    return;
  }
  cell.resize(n);
  std::fill(starts, starts + cells + 1, 0);
  for (int j = 0; j < n; ++j) {
    cell[j] = cell_of(xy[2 * j], xy[2 * j + 1]);
    ++starts[cell[j] + 1];
  }
  for (int c = 0; c < cells; ++c) starts[c + 1] += starts[c];
  // scatter with starts[c] as the running cursor, then shift back
  for (int j = 0; j < n; ++j) {
    const int at = starts[cell[j]]++;
    out[2 * at] = xy[2 * j];
    out[2 * at + 1] = xy[2 * j + 1];
  }
  for (int c = cells; c > 0; --c) starts[c] = starts[c - 1];
  starts[0] = 0;
}

// Tight point boxes of the static cells, kept when the static part is dense
// (mean points per occupied cell >= PARAPLAN_CELL_BOX_MIN) and structured
// (mean box area below half a cell: lines and walls rather than a uniform
// fill, which a box test cannot thin out). There a box test per visited cell
// is cheaper than scanning its points.
void cell_boxes(Binned& b) {
  static const double min_fill = env_or("PARAPLAN_CELL_BOX_MIN", 8);
  static const double max_area = env_or("PARAPLAN_CELL_BOX_AREA", 0.5);
  b.boxes = false;
  if (b.ny <= 1 || b.Ns == 0) return;
  const int cells = b.cells();
  int occupied = 0;
  for (int c = 0; c < cells; ++c) occupied += b.sst[c + 1] > b.sst[c];
  if (static_cast<double>(b.Ns) < min_fill * occupied) return;
  b.sbox.resize(4 * static_cast<size_t>(cells));
  double area = 0.0;
  for (int c = 0; c < cells; ++c) {
    double x0 = 0, x1 = -1, y0 = 0, y1 = -1;  // empty: negative half extents
    for (int j = b.sst[c]; j < b.sst[c + 1]; ++j) {
      const double x = b.spts[2 * j], y = b.spts[2 * j + 1];
      if (j == b.sst[c]) {
        x0 = x1 = x;
        y0 = y1 = y;
      } else {
        x0 = std::min(x0, x);
        x1 = std::max(x1, x);
        y0 = std::min(y0, y);
        y1 = std::max(y1, y);
      }
    }
    double* o = b.sbox.data() + 4 * static_cast<size_t>(c);
    o[0] = 0.5 * (x0 + x1);
    o[1] = 0.5 * (y0 + y1);
    o[2] = 0.5 * (x1 - x0);
    o[3] = 0.5 * (y1 - y0);
    if (x1 >= x0) area += (x1 - x0) * (y1 - y0);
  }
  const bool structured = area < max_area * occupied * b.g * b.g;
  // very dense clouds profit from the chunk boxes even without structure
  static const double min_dense = env_or("PARAPLAN_CHUNK_DENSE_MIN", 32);
  b.boxes = structured || static_cast<double>(b.Ns) >= min_dense * occupied;
  if (!b.boxes) return;
  // chunk boxes over consecutive points of a cell. Structured clouds keep
  // their order (points along a polyline: a chunk is a short piece of a
  // line); a uniform fill is put in Morton (Z) order of the position in the
  // cell first, so a chunk is a compact patch
  // (cells are independent: in parallel over cell blocks)
  constexpr int kCellBlock = 64;
  const int blocks = (cells + kCellBlock - 1) / kCellBlock;
  if (!structured) {
    par_for(blocks, static_cast<size_t>(b.Ns) * 4, [&](int blk) {
    thread_local std::vector<std::pair<uint32_t, int>> key;
    thread_local std::vector<double> tmp;
    for (int c = blk * kCellBlock; c < std::min(cells, (blk + 1) * kCellBlock); ++c) {
      const int j0 = b.sst[c], n = b.sst[c + 1] - j0;
      if (n <= 16) continue;
      const double* bx = b.sbox.data() + 4 * static_cast<size_t>(c);
      const double sx = bx[2] > 0 ? 32767.0 / (2 * bx[2]) : 0.0;
      const double sy = bx[3] > 0 ? 32767.0 / (2 * bx[3]) : 0.0;
      key.resize(n);
      for (int k = 0; k < n; ++k) {
        const double x = b.spts[2 * (j0 + k)], y = b.spts[2 * (j0 + k) + 1];
        uint32_t ix = static_cast<uint32_t>((x - (bx[0] - bx[2])) * sx);
        uint32_t iy = static_cast<uint32_t>((y - (bx[1] - bx[3])) * sy);
        // bit interleave (Morton) of the 15-bit coordinates
        const auto spread = [](uint32_t v) {
          v &= 0x7fffu;
          v = (v | (v << 8)) & 0x00ff00ffu;
          v = (v | (v << 4)) & 0x0f0f0f0fu;
          v = (v | (v << 2)) & 0x33333333u;
          v = (v | (v << 1)) & 0x55555555u;
          return v;
        };
        const uint32_t z = spread(ix) | (spread(iy) << 1);
        key[k] = {z, k};
      }
      std::stable_sort(key.begin(), key.end(),
                       [](const auto& l, const auto& r) { return l.first < r.first; });
      tmp.assign(b.spts.begin() + 2 * j0, b.spts.begin() + 2 * (j0 + n));
      for (int k = 0; k < n; ++k) {
        b.spts[2 * (j0 + k)] = tmp[2 * key[k].second];
        b.spts[2 * (j0 + k) + 1] = tmp[2 * key[k].second + 1];
      }
    }
    });
  }
  b.cst.assign(cells + 1, 0);
  for (int c = 0; c < cells; ++c) {
    const int n = b.sst[c + 1] - b.sst[c];
    const int cs = chunk_size(n);
    b.cst[c + 1] = b.cst[c] + (n + cs - 1) / cs;
  }
  b.cbox.resize(4 * static_cast<size_t>(b.cst[cells]));
  par_for(blocks, static_cast<size_t>(b.Ns) * 4, [&](int blk) {
  for (int c = blk * kCellBlock; c < std::min(cells, (blk + 1) * kCellBlock); ++c) {
    const int n = b.sst[c + 1] - b.sst[c];
    const int cs = chunk_size(n);
    for (int k = b.cst[c]; k < b.cst[c + 1]; ++k) {
      const int j0 = b.sst[c] + (k - b.cst[c]) * cs, j1 = std::min(b.sst[c + 1], j0 + cs);
      double x0 = b.spts[2 * j0], x1 = x0, y0 = b.spts[2 * j0 + 1], y1 = y0;
      for (int j = j0 + 1; j < j1; ++j) {
        x0 = std::min(x0, b.spts[2 * j]);
        x1 = std::max(x1, b.spts[2 * j]);
        y0 = std::min(y0, b.spts[2 * j + 1]);
        y1 = std::max(y1, b.spts[2 * j + 1]);
      }
      double* o = b.cbox.data() + 4 * static_cast<size_t>(k);
      o[0] = 0.5 * (x0 + x1);
      o[1] = 0.5 * (y0 + y1);
      o[2] = 0.5 * (x1 - x0);
      o[3] = 0.5 * (y1 - y0);
    }
  }
  });
}

// Grid + static bins (+ boxes).
void finish_static(Binned& b, const std::vector<double>& s_xy, const BBox& box) {
  choose_grid(b, box);
  const int cells = b.cells();
  std::vector<int32_t> cell;
  b.spts.resize(2 * static_cast<size_t>(b.Ns));
  b.sst.assign(cells + 1, 0);
  if (b.Ns > 0) bin(b, s_xy.data(), b.Ns, b.spts.data(), b.sst.data(), cell);
  cell_boxes(b);
}

// Dynamic rows: row(r, xy) writes the Nd positions of dynamic row r.
template <class Row>
void finish_dynamic(Binned& b, Row&& row) {
  const int cells = b.cells();
  b.dpts.resize(2 * static_cast<size_t>(b.Nd) * b.rows);
  b.dst.assign(static_cast<size_t>(b.rows) * (cells + 1), 0);
  if (b.Nd > 0) {
    par_for(b.rows, static_cast<size_t>(b.rows) * b.Nd, [&](int r) {
      thread_local std::vector<double> xy;
      thread_local std::vector<int32_t> tcell;
      xy.resize(2 * static_cast<size_t>(b.Nd));
      row(r, xy.data());
      const size_t o = static_cast<size_t>(r) * b.Nd * 2;
      bin(b, xy.data(), b.Nd, b.dpts.data() + o, b.dst.data() + static_cast<size_t>(r) * (cells + 1),
          tcell);
    });
  }
}

template <class Row>
void finish(Binned& b, const std::vector<double>& s_xy, const BBox& box, Row&& row) {
  finish_static(b, s_xy, box);
  finish_dynamic(b, row);
}

// src/geometry.cpp:53-57: row r of the movers, x + h * step (int h promoted
// to double).
void mover_row(const Binned& b, int r, double* out) {
  const double* q = b.dbase.data();
  for (int k = 0; k < b.Nd; ++k) {
    out[2 * k] = q[4 * k] + r * q[4 * k + 2];
    out[2 * k + 1] = q[4 * k + 1] + r * q[4 * k + 3];
  }
}

// Scalars back to their defaults; the vectors keep their storage, so a
// planner re-binning a field of the same shape every tick neither allocates
// nor faults pages in.
void reset(Binned& b, int rows, double cull) {
  b.Ns = b.Nd = 0;
  b.boxes = false;
  b.dyn_deferred = false;
  b.dbase.clear();
  b.nx = b.ny = 1;
  b.x0 = b.y0 = 0.0;
  b.g = 1.0;
  b.rows = rows;
  b.cull = cull;
}

}  // namespace

Layout layout(const Binned& b, size_t elem) {
  Layout l;
  l.dpts = align16(2 * elem * static_cast<size_t>(b.Ns + b.pad_s));
  l.sst = align16(l.dpts + 2 * elem * static_cast<size_t>(b.Nd + b.pad_d) * b.rows);
  l.dst = align16(l.sst + sizeof(int32_t) * (b.cells() + 1));
  l.sbox = align16(l.dst + sizeof(int32_t) * static_cast<size_t>(b.rows) * (b.cells() + 1));
  l.cst = align16(l.sbox + (b.boxes ? 4 * elem * static_cast<size_t>(b.cells()) : 0));
  l.cbox = align16(l.cst + (b.boxes ? sizeof(int32_t) * (b.cells() + 1) : 0));
  l.bytes = align16(l.cbox + (b.boxes ? 2 * elem * b.cbox.size() : 0));
  return l;
}

void from_rows(Binned& b, const double* xy, int rows, int N, double cull) {
  reset(b, rows, cull);
  const size_t len = 2 * static_cast<size_t>(N);
  std::vector<char> moving(N, 0);
  constexpr int kPtBlock = 2048;  // a block's slice of a row: 32 KB
  par_for((N + kPtBlock - 1) / kPtBlock, static_cast<size_t>(rows) * N, [&](int k) {
    const int j0 = k * kPtBlock, j1 = std::min(N, (k + 1) * kPtBlock);
    for (int r = 1; r < rows; ++r) {
      const double* row = xy + r * len;
      for (int j = j0; j < j1; ++j) {
        moving[j] |= std::memcmp(row + 2 * j, xy + 2 * j, 2 * sizeof(double)) != 0;
      }
    }
  });
  // small mixed clouds stay one scan per state: every point dynamic
  if (N <= kSmall && std::count(moving.begin(), moving.end(), 1) > 0) {
    std::fill(moving.begin(), moving.end(), 1);
  }
  std::vector<double> s_xy;
  std::vector<int> dyn;
  BBox box;
  for (int j = 0; j < N; ++j) {
    if (moving[j]) {
      dyn.push_back(j);
    } else {
      s_xy.push_back(xy[2 * j]);
      s_xy.push_back(xy[2 * j + 1]);
      box.see(xy[2 * j], xy[2 * j + 1]);
    }
  }
  b.Ns = N - static_cast<int>(dyn.size());
  b.Nd = static_cast<int>(dyn.size());
  if (b.Nd > 0) {  // rows are arbitrary: every dynamic position joins the box
    std::vector<BBox> rb(rows);
    par_for(rows, static_cast<size_t>(rows) * b.Nd, [&](int r) {
      const double* row = xy + r * len;
      for (int k = 0; k < b.Nd; ++k) rb[r].see(row[2 * dyn[k]], row[2 * dyn[k] + 1]);
    });
    for (const BBox& o : rb) box.merge(o);
  }
  finish(b, s_xy, box, [&](int r, double* out) {
    const double* row = xy + r * len;
    for (int k = 0; k < b.Nd; ++k) {
      out[2 * k] = row[2 * dyn[k]];
      out[2 * k + 1] = row[2 * dyn[k] + 1];
    }
  });
}

void from_points(Binned& b, const double* pts4, int N, int rows, double T_s, double cull,
                 bool defer_dynamic) {
  reset(b, rows, cull);
  // src/geometry.cpp:51-52, once per point
  std::vector<double> steps(2 * static_cast<size_t>(N));
  par_for((N + 4095) / 4096, static_cast<size_t>(N) * 8, [&](int c) {
    for (int j = c * 4096; j < std::min(N, (c + 1) * 4096); ++j) {
      const double* p = pts4 + 4 * j;
      steps[2 * j] = T_s * p[3] * std::cos(p[2]);
      steps[2 * j + 1] = T_s * p[3] * std::sin(p[2]);
    }
  });
  bool any_moving = false;
  for (int j = 0; j < N && !any_moving; ++j) {
    any_moving = !(steps[2 * j] == 0.0 && steps[2 * j + 1] == 0.0);
  }
  // small mixed clouds stay one scan per state: every point dynamic
  const bool all_dynamic = N <= kSmall && any_moving;
  const auto is_static = [&](int j) {
    return !all_dynamic && steps[2 * j] == 0.0 && steps[2 * j + 1] == 0.0;
  };
  // split in input order, in parallel over blocks of points: per-block
  // counts and bounding boxes, then a scatter at the blocks' offsets
  constexpr int kPtBlock = 4096;
  const int nblk = (N + kPtBlock - 1) / kPtBlock;
  struct Blk {
    int ns = 0, nd = 0;
    double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    bool finite = true;
  };
  std::vector<Blk> blk(nblk);
  par_for(nblk, static_cast<size_t>(N) * 4, [&](int k) {
    Blk& q = blk[k];
    const auto see = [&](double x, double y) {
      q.finite &= std::isfinite(x) && std::isfinite(y);
      q.xmin = std::min(q.xmin, x);
      q.xmax = std::max(q.xmax, x);
      q.ymin = std::min(q.ymin, y);
      q.ymax = std::max(q.ymax, y);
    };
    for (int j = k * kPtBlock; j < std::min(N, (k + 1) * kPtBlock); ++j) {
      const double* p = pts4 + 4 * j;
      see(p[0], p[1]);
      if (is_static(j)) {
        ++q.ns;
      } else {
        ++q.nd;
        // x + r * step is monotone in r (rounding is monotone): rows 0 and
        // rows - 1 bound every position of the point
        see(p[0] + (rows - 1) * steps[2 * j], p[1] + (rows - 1) * steps[2 * j + 1]);
      }
    }
  });
  size_t ns = 0, nd = 0;
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  bool finite = true;
  std::vector<size_t> s_off(nblk), d_off(nblk);
  for (int k = 0; k < nblk; ++k) {
    s_off[k] = ns;
    d_off[k] = nd;
    ns += blk[k].ns;
    nd += blk[k].nd;
    finite &= blk[k].finite;
    xmin = std::min(xmin, blk[k].xmin);
    xmax = std::max(xmax, blk[k].xmax);
    ymin = std::min(ymin, blk[k].ymin);
    ymax = std::max(ymax, blk[k].ymax);
  }
  std::vector<double> s_xy(2 * ns);
  b.dbase.resize(4 * nd);
  par_for(nblk, static_cast<size_t>(N) * 4, [&](int k) {
    size_t is = s_off[k], id = d_off[k];
    for (int j = k * kPtBlock; j < std::min(N, (k + 1) * kPtBlock); ++j) {
      const double* p = pts4 + 4 * j;
      if (is_static(j)) {
        s_xy[2 * is] = p[0];
        s_xy[2 * is + 1] = p[1];
        ++is;
      } else {
        double* q = b.dbase.data() + 4 * id++;
        q[0] = p[0];
        q[1] = p[1];
        q[2] = steps[2 * j];
        q[3] = steps[2 * j + 1];
      }
    }
  });
  BBox box;
  box.finite = finite;
  if (N > 0 && finite) {
    box.see(xmin, ymin);
    box.see(xmax, ymax);
  }
  b.Ns = static_cast<int>(s_xy.size() / 2);
  b.Nd = static_cast<int>(b.dbase.size() / 4);
  finish_static(b, s_xy, box);
  if (defer_dynamic && b.Nd > 0) {
    b.dyn_deferred = true;
    return;
  }
  finish_dynamic(b, [&](int r, double* out) { mover_row(b, r, out); });
}

void bin_dynamic(Binned& b) {
  if (!b.dyn_deferred) return;
  finish_dynamic(b, [&](int r, double* out) { mover_row(b, r, out); });
  b.dyn_deferred = false;
}

void pack(const Binned& b, bool fp64, void* out, bool with_dynamic) {
  const size_t elem = fp64 ? sizeof(double) : sizeof(float);
  const Layout l = layout(b, elem);
  unsigned char* base = static_cast<unsigned char*>(out);
  const auto put = [&](size_t off, const std::vector<double>& v) {
    constexpr size_t kChunk = size_t(1) << 16;
    const int chunks = static_cast<int>((v.size() + kChunk - 1) / kChunk);
    par_for(chunks, v.size(), [&](int c) {
      const size_t lo = c * kChunk, hi = std::min(v.size(), lo + kChunk);
      if (fp64) {
        std::memcpy(base + off + lo * sizeof(double), v.data() + lo, (hi - lo) * sizeof(double));
      } else {
        float* f = reinterpret_cast<float*>(base + off);
        for (size_t i = lo; i < hi; ++i) f[i] = static_cast<float>(v[i]);
      }
    });
  };
  // sentinels: (1e30, 0) -- outside the chassis by ~0.7e30 at any heading
  // (one of |cos|, |sin| >= 0.7), finite in FP32
  const auto sentinels = [&](size_t off, int n) {
    for (int i = 0; i < n; ++i) {
      if (fp64) {
        double* d = reinterpret_cast<double*>(base + off) + 2 * i;
        d[0] = 1e30;
        d[1] = 0.0;
      } else {
        float* f = reinterpret_cast<float*>(base + off) + 2 * i;
        f[0] = 1e30f;
        f[1] = 0.0f;
      }
    }
  };
  put(0, b.spts);
  sentinels(2 * elem * static_cast<size_t>(b.Ns), b.pad_s);
  std::memcpy(base + l.sst, b.sst.data(), b.sst.size() * sizeof(int32_t));
  if (with_dynamic) {
    if (b.pad_d == 0) {
      put(l.dpts, b.dpts);
    } else {  // rows of Nd points + pad_d sentinels
      for (int r = 0; r < b.rows; ++r) {
        const size_t row = l.dpts + 2 * elem * static_cast<size_t>(r) * (b.Nd + b.pad_d);
        for (int i = 0; i < b.Nd; ++i) {
          const double* src = b.dpts.data() + 2 * (static_cast<size_t>(r) * b.Nd + i);
          if (fp64) {
            std::memcpy(base + row + 2 * elem * i, src, 2 * sizeof(double));
          } else {
            float* f = reinterpret_cast<float*>(base + row) + 2 * i;
            f[0] = static_cast<float>(src[0]);
            f[1] = static_cast<float>(src[1]);
          }
        }
        sentinels(row + 2 * elem * static_cast<size_t>(b.Nd), b.pad_d);
      }
    }
    std::memcpy(base + l.dst, b.dst.data(), b.dst.size() * sizeof(int32_t));
  }
  if (b.boxes) {
    put(l.sbox, b.sbox);
    std::memcpy(base + l.cst, b.cst.data(), b.cst.size() * sizeof(int32_t));
    put(l.cbox, b.cbox);
  }
}

namespace {
bool box_separated(const double* bx, double c, double s, double kx, double ky, double bh, double hw,
                   double pad) {
  // separating axes: the rectangle's own (u = (c, s), v = (-s, c)); the
  // world axes are covered by the query window
  const double ac = std::abs(c), as = std::abs(s);
  const double du = c * bx[0] + s * bx[1] - kx, dv = -s * bx[0] + c * bx[1] - ky;
  return std::abs(du) > bh + bx[2] * ac + bx[3] * as + pad ||
         std::abs(dv) > hw + bx[2] * as + bx[3] * ac + pad;
}
}  // namespace

namespace {
bool box_separated(const double* bx, double c, double s, double kx, double ky, double bh, double hw,
                   double pad);
}

bool collides(const Binned& b, const paraplan::ChassisPolytope& ch, const Box& box, int k, double x,
              double y, double phi) {
  if (b.points() == 0) return false;
  const auto cx_of = [&](double v) {
    return std::min(b.nx - 1, std::max(0, static_cast<int>(std::floor((v - b.x0) / b.g))));
  };
  const auto cy_of = [&](double v) {
    return b.ny == 1 ? 0
                     : std::min(b.ny - 1, std::max(0, static_cast<int>(std::floor((v - b.y0) / b.g))));
  };
  // src/geometry.cpp:63-76, expression by expression
  const double c = std::cos(phi), s = std::sin(phi);
  // world bounding box of the rectangle (+ g/8): points outside it are
  // outside the rectangle, a miss in the reference's test
  const double bc = 0.5 * (box.front - box.rear), bh = 0.5 * (box.front + box.rear);
  const double pad = b.g / 8.0;
  const double ox = x + bc * c, oy = y + bc * s;
  const double ex = bh * std::abs(c) + box.half_width * std::abs(s) + pad;
  const double ey = bh * std::abs(s) + box.half_width * std::abs(c) + pad;
  const int cx0 = cx_of(ox - ex), cx1 = cx_of(ox + ex);
  const int cy0 = cy_of(oy - ey), cy1 = cy_of(oy + ey);
  const double r2 = ch.bounding_radius() * ch.bounding_radius();
  const auto test = [&](const double* pts, int j0, int j1) {
    for (int j = j0; j < j1; ++j) {
      const double dx = pts[2 * j] - x, dy = pts[2 * j + 1] - y;
      if (dx * dx + dy * dy >= r2) continue;
      if (ch.contains({c * dx + s * dy, -s * dx + c * dy})) return true;
    }
    return false;
  };
  const auto scan = [&](const double* pts, const int32_t* st) {
    for (int cx = cx0; cx <= cx1; ++cx) {
      if (test(pts, st[cx * b.ny + cy0], st[cx * b.ny + cy1 + 1])) return true;
    }
    return false;
  };
  if (b.Ns > 0 && b.boxes) {  // cell by cell, skipping cells whose box is clear of the rectangle
    const double kx = c * x + s * y + bc, ky = -s * x + c * y;
    for (int cx = cx0; cx <= cx1; ++cx) {
      for (int cy = cy0; cy <= cy1; ++cy) {
        const int cell = cx * b.ny + cy;
        if (b.sst[cell + 1] == b.sst[cell]) continue;
        if (box_separated(b.sbox.data() + 4 * static_cast<size_t>(cell), c, s, kx, ky, bh,
                          box.half_width, pad)) {
          continue;
        }
        if (test(b.spts.data(), b.sst[cell], b.sst[cell + 1])) return true;
      }
    }
  } else if (b.Ns > 0 && scan(b.spts.data(), b.sst.data())) {
    return true;
  }
  if (b.Nd > 0) {
    const int cells = b.cells();
    return scan(b.dpts.data() + static_cast<size_t>(k) * b.Nd * 2,
                b.dst.data() + static_cast<size_t>(k) * (cells + 1));
  }
  return false;
}

}  // namespace ppfield

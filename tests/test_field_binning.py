"""The host field binning (csrc/capi/field.cpp) gives the same image whether
its passes run on the shared host pool (parallel splits, per-block counting
sorts, Morton keys per cell block) or serially (PARAPLAN_FIELD_SERIAL=1).

The binned image decides which points a collision query visits; the device
kernels and the exact host rollouts both read it, so a parallel pass that
reordered or dropped a point would change plans. CPU only: a small C++
harness is compiled against field.cpp and hashes every part of the image for
a C5-like cloud (points uniform in x in [-10, 30], |y| in [2.5, 10], 25%
moving; src/geometry.cpp:43-61 extrapolation) and for the (H+1) x N rows of
the same cloud (from_rows).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CAPI = ROOT / "paper_1904_06680_b200" / "csrc" / "capi"

HARNESS = r"""
#include "field.hpp"
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
static unsigned long long h = 1469598103934665603ull;
static void mix(const void* p, size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ull; }
}
template <class T> static void mixv(const std::vector<T>& v) { mix(v.data(), v.size() * sizeof(T)); }
static void mixb(const ppfield::Binned& b) {
  mixv(b.spts); mixv(b.sst); mixv(b.dpts); mixv(b.dst); mixv(b.sbox); mixv(b.cst); mixv(b.cbox);
  int s[6] = {b.Ns, b.Nd, b.nx, b.ny, b.mode(), b.rows};
  mix(s, sizeof(s));
}
int main(int argc, char** argv) {
  const int N = std::atoi(argv[1]), rows = std::atoi(argv[2]);
  std::mt19937_64 rng(N);
  std::uniform_real_distribution<double> ux(-10, 30), uy(2.5, 10), us(0, 15), u01(0, 1);
  std::vector<double> pts(4 * static_cast<size_t>(N));
  for (int j = 0; j < N; ++j) {
    pts[4 * j] = ux(rng);
    const double y = uy(rng);
    pts[4 * j + 1] = u01(rng) < 0.5 ? y : -y;
    const bool dyn = u01(rng) < 0.25;
    pts[4 * j + 2] = dyn ? (u01(rng) < 0.5 ? 0.0 : M_PI) : 0.0;
    pts[4 * j + 3] = dyn ? us(rng) : 0.0;
  }
  const double cull = std::sqrt(5.0) + 1e-3;
  ppfield::Binned b;
  ppfield::from_points(b, pts.data(), N, rows, 0.1, cull, false);
  mixb(b);
  // the same cloud as (H+1) x N rows, the reference's ExtrapolatedField
  std::vector<double> xy(2 * static_cast<size_t>(N) * rows);
  for (int r = 0; r < rows; ++r) {
    for (int j = 0; j < N; ++j) {
      const double sx = 0.1 * pts[4 * j + 3] * std::cos(pts[4 * j + 2]);
      const double sy = 0.1 * pts[4 * j + 3] * std::sin(pts[4 * j + 2]);
      xy[2 * (static_cast<size_t>(r) * N + j)] = pts[4 * j] + r * sx;
      xy[2 * (static_cast<size_t>(r) * N + j) + 1] = pts[4 * j + 1] + r * sy;
    }
  }
  ppfield::Binned c;
  ppfield::from_rows(c, xy.data(), rows, N, cull);
  mixb(c);
  std::printf("%016llx %d %d %d\n", h, b.Ns, b.Nd, b.mode());
  return 0;
}
"""


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("field")
    src = d / "harness.cpp"
    src.write_text(HARNESS)
    exe = d / "harness"
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-pthread",
                    f"-I{CAPI}", f"-I{ROOT / 'include'}", str(src), str(CAPI / "field.cpp"),
                    "-o", str(exe)], check=True, capture_output=True, text=True, timeout=600)
    return exe


def run(exe, n, rows, serial):
    env = dict(os.environ, PARAPLAN_FIELD_SERIAL="1" if serial else "0")
    p = subprocess.run([str(exe), str(n), str(rows)], env=env, capture_output=True, text=True,
                       timeout=300, check=True)
    return p.stdout.split()


@pytest.mark.parametrize("n,rows", [(100000, 11), (40000, 31), (3000, 101)])
def test_parallel_binning_equals_serial(harness, n, rows):
    par = run(harness, n, rows, serial=False)
    ser = run(harness, n, rows, serial=True)
    assert par == ser, (par, ser)
    assert int(par[1]) + int(par[2]) == n  # every point is static or dynamic

// keypack.h -- the packed 64-bit candidate key of the cross-GPU winner
// collective: one ncclAllReduce(ncclMin, uint64) over the
// shards' per-restart winners picks the global winner, because the packed
// order IS the reference's order (src/planner.cpp:27-44 score/better, ties to
// the lowest index, :295, :316):
//   [63:62] 2 - cls   (reached 2 < free 1 < collided 0: smaller is better)
//   [61:54] t_goal    (class 2: earlier is better; 0 otherwise)
//   [53:22] cost bits (path length for class 2, terminal cost otherwise;
//                      non-negative floats order like their bit patterns)
//   [21: 0] candidate index within the restart (lower wins ties)
// Valid when n_candidates <= 2^22 and H <= 255 (every BASELINE config);
// otherwise the shards all-gather their records instead. An empty record
// packs to ~0. FP64 costs are rounded UP to float: the packed key then only
// anchors a window (its threshold can only grow), never decides a winner.
// Shared by the host (g++) and the device (nvcc).
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define PP_HD __host__ __device__ __forceinline__
#else
#define PP_HD inline
#endif

namespace ppdev {

constexpr int kPackIndexBits = 22;
constexpr int64_t kPackMaxCandidates = int64_t{1} << kPackIndexBits;
constexpr int kPackMaxTGoal = 255;
constexpr uint64_t kPackEmpty = ~0ull;

PP_HD uint32_t float_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, sizeof(u));
  return u;
}
PP_HD float bits_float(uint32_t u) {
  float f;
  std::memcpy(&f, &u, sizeof(f));
  return f;
}

PP_HD uint64_t pack_key(int cls, int t_goal, float cost, uint32_t idx) {
  if (cls < 0) return kPackEmpty;
  return (static_cast<uint64_t>(2 - cls) << 62) |
         (static_cast<uint64_t>(cls == 2 ? (t_goal & 0xff) : 0) << 54) |
         (static_cast<uint64_t>(float_bits(cost)) << kPackIndexBits) |
         static_cast<uint64_t>(idx & ((1u << kPackIndexBits) - 1u));
}

struct Unpacked {
  int cls, t_goal;
  float cost;
  uint32_t idx;
};
PP_HD Unpacked unpack_key(uint64_t k) {
  Unpacked u;
  if (k == kPackEmpty) {
    u.cls = -1;
    u.t_goal = 0;
    u.cost = 0.0f;
    u.idx = 0;
    return u;
  }
  u.cls = 2 - static_cast<int>(k >> 62);
  u.t_goal = static_cast<int>((k >> 54) & 0xff);
  u.cost = bits_float(static_cast<uint32_t>((k >> kPackIndexBits) & 0xffffffffull));
  u.idx = static_cast<uint32_t>(k & ((1ull << kPackIndexBits) - 1ull));
  return u;
}

}  // namespace ppdev

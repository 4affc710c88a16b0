// reduce.cuh -- candidate keys and their reductions (src/planner.cpp:27-44, 295-321),
// field staging, sample keys for the re-ranking, round bookkeeping.
// Part of the sampler kernels (rollout.cuh).
#pragma once

#include "step.cuh"

namespace ppdev {

// ---------------------------------------------------------- reduction ----
// Lexicographic (cls, k1, k2) descending, index ascending: a total order, so
// any reduction tree gives the reference's "strict better, lowest index
// wins" result (src/planner.cpp:40-44, 295, 316).
struct Key {
  int cls;
  int idx;
  double k1, k2;
};

__device__ __forceinline__ Key empty_key() { return Key{-1, -1, 0.0, 0.0}; }

__device__ __forceinline__ bool prefer(const Key& a, const Key& b) {
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  if (a.k2 != b.k2) return a.k2 > b.k2;
  return static_cast<unsigned>(a.idx) < static_cast<unsigned>(b.idx);
}

template <typename Real>
__device__ __forceinline__ Key make_key(int cls, int h, Real path, Real term, int idx) {
  Key k;  // src/planner.cpp:27-38
  k.cls = cls;
  k.idx = idx;
  if (cls == 2) {
    k.k1 = -static_cast<double>(h);
    k.k2 = -static_cast<double>(path);
  } else {
    k.k1 = -static_cast<double>(term);
    k.k2 = 0.0;
  }
  return k;
}

// Lane-local best of the FP32 rollout: the same key with float components.
// The FP64 key of an FP32 rollout holds exactly these float values (an int
// t_goal or a float cost, widened), so the order is the same and the lane
// compares in FP32 without conversions; widened only when flushed.
struct KeyF {
  int cls;
  int idx;
  float k1, k2;
};
__device__ __forceinline__ bool prefer(const KeyF& a, const KeyF& b) {
  if (a.cls != b.cls) return a.cls > b.cls;
  if (a.k1 != b.k1) return a.k1 > b.k1;
  if (a.k2 != b.k2) return a.k2 > b.k2;
  return static_cast<unsigned>(a.idx) < static_cast<unsigned>(b.idx);
}
__device__ __forceinline__ Key to_key(const Key& k) { return k; }
__device__ __forceinline__ Key to_key(const KeyF& k) {
  return Key{k.cls, k.idx, static_cast<double>(k.k1), static_cast<double>(k.k2)};
}
template <typename Real>
using LaneKey = typename std::conditional<sizeof(Real) == sizeof(float), KeyF, Key>::type;
template <typename Real>
__device__ __forceinline__ LaneKey<Real> lane_empty() {
  return LaneKey<Real>{-1, -1, Real(0), Real(0)};
}
template <typename Real>
__device__ __forceinline__ LaneKey<Real> make_lane_key(int cls, int h, Real path, Real term,
                                                       int idx) {
  LaneKey<Real> k;  // src/planner.cpp:27-38
  k.cls = cls;
  k.idx = idx;
  k.k1 = cls == 2 ? -static_cast<Real>(h) : -term;
  k.k2 = cls == 2 ? -path : Real(0);
  return k;
}

__device__ __forceinline__ Key shfl_key(const Key& k, int off) {
  Key o;
  o.cls = __shfl_down_sync(kFull, k.cls, off);
  o.idx = __shfl_down_sync(kFull, k.idx, off);
  o.k1 = __shfl_down_sync(kFull, k.k1, off);
  o.k2 = __shfl_down_sync(kFull, k.k2, off);
  return o;
}

// Warp argmin; result valid in lane 0.
__device__ __forceinline__ Key warp_best(Key k) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Key o = shfl_key(k, off);
    if (prefer(o, k)) k = o;
  }
  return k;
}

// Block argmin; result valid in thread 0. `scratch` holds >= 32 keys.
__device__ __forceinline__ Key block_best(Key k, Key* scratch) {
  k = warp_best(k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = k;
  __syncthreads();
  if (warp == 0) {
    k = lane < static_cast<int>(blockDim.x >> 5) ? scratch[lane] : empty_key();
    k = warp_best(k);
  }
  __syncthreads();
  return k;
}

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v,
                                                        unsigned long long* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < static_cast<int>(blockDim.x >> 5) ? scratch[lane] : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(kFull, v, off);
  }
  __syncthreads();
  return v;
}

__device__ __forceinline__ Key load_rec_cg(const Rec* src) {
  // written by other CTAs: read through L2 (ld.global.cg), never L1
  return Key{__ldcg(&src->cls), __ldcg(&src->cand), __ldcg(&src->k1), __ldcg(&src->k2)};
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it waits here (the
// predecessor has completed and its writes are visible) before reading what
// the predecessor wrote. A no-op for an ordinary launch.
__device__ __forceinline__ void wait_prior_grid() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Field of the round, staged whole into shared memory when it fits
// (a.field_smem_bytes > 0), else read through L1/L2. The staging is one TMA
// bulk copy (cp.async.bulk, global -> shared) issued by thread 0 and
// completed on an mbarrier (transaction count = the image size, a multiple
// of 16 bytes, <= 40 KB); every thread waits on the barrier's phase 0.
__device__ __forceinline__ void bulk_stage(unsigned char* dst, const void* src, uint32_t bytes,
                                           uint64_t* mbar) {
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
  }
  __syncthreads();  // the barrier is initialised before anyone polls it
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(bar)
      : "memory");
}

template <typename Real, int kGrid = 0>
__device__ __forceinline__ Field<Real> stage_field(const RoundArgs& a, unsigned char* smem) {
  __shared__ __align__(8) uint64_t stage_bar;
  if constexpr (kGrid == 3) {
    // grid kind 3: x-buckets staged in shared memory (the host launches this
    // instantiation only then), so every field load is an LDS on a 32-bit
    // shared address instead of a generic 64-bit load
    bulk_stage(smem, a.field, static_cast<uint32_t>(a.field_smem_bytes), &stage_bar);
    Field<Real> f = field_at<Real>(a, smem, a.lay);
    bind_shared(f, smem, a.lay);
    return f;
  }
  if (a.field_smem_bytes > 0 && a.n_points > 0) {
    bulk_stage(smem, a.field, static_cast<uint32_t>(a.field_smem_bytes), &stage_bar);
    return field_at<Real>(a, smem, a.lay);
  }
  __syncthreads();
  return field_at<Real>(a, a.field, a.lay);
}

// Compact per-sample key for the near-tie re-ranking (select_kernel):
// cost = terminal cost (cls 0/1) or path length (cls 2); meta = cls | marg<<2
// | t_goal<<8.
template <typename Real>
__device__ __forceinline__ void write_skey(const RoundArgs& a, int64_t slot, int cls,
                                           const Lane<Real>& L, Real term, int t_goal = -1) {
  if (a.skeys == nullptr) return;
  const uint32_t meta = make_meta(cls, t_goal < 0 ? L.h : t_goal, L.mstep);
  if constexpr (sizeof(Real) == sizeof(float)) {
    static_cast<SKey32*>(a.skeys)[slot] = SKey32{cls == 2 ? L.path : term, meta};
  } else {
    // pad: the path up to the flagged state, rounded down to float (a lower
    // bound of the key a flip there would give; the wide-window pruning)
    static_cast<SKey*>(a.skeys)[slot] =
        SKey{cls == 2 ? L.path : term, meta, float_bits(__double2float_rd(L.mpath))};
  }
}

// Per-sample debug/parity record.
template <typename Real>
__device__ __forceinline__ void write_sample(const RoundArgs& a, int64_t slot, int cls,
                                             const Lane<Real>& L, Real term, Real f0, Real f1) {
  SampleOut& so = a.per_sample[slot];
  so.reached = cls == 2;
  so.t_goal = cls == 2 ? L.h : -1;
  so.collided = cls == 0;
  so.steps = L.h;
  so.path_length = static_cast<double>(L.path);
  so.terminal_cost = static_cast<double>(term);
  so.first_a0 = static_cast<double>(f0);
  so.first_a1 = static_cast<double>(f1);
}

// Last CTA: per-restart reduction of `n_src` records per restart (laid out
// restart-major), publish the work counters, re-arm the tickets.
// Last-block election over the whole grid (the ticket is re-armed by
// publish_round).
__device__ __forceinline__ bool last_block(const RoundArgs& a) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  const unsigned n_blocks = gridDim.x * gridDim.y;
  if (threadIdx.x == 0) s_last = atomicAdd(&a.counters[1], 1u) == n_blocks - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Per-restart reduction of `n_src` records per restart (restart-major) into
// out[restart].
// Block-wide, one restart after the other (the rollout kernels' last CTA:
// one restart on the refill schedule).
__device__ __forceinline__ void reduce_recs(const RoundArgs& a, const Rec* recs, int n_src,
                                            Key* red, Rec* out) {
  for (int r = 0; r < a.restart_count; ++r) {
    Key k = empty_key();
    for (int t = threadIdx.x; t < n_src; t += blockDim.x) {
      const Key o = load_rec_cg(recs + static_cast<size_t>(r) * n_src + t);
      if (o.cls >= 0 && (k.cls < 0 || prefer(o, k))) k = o;
    }
    const Key best = block_best(k, red);
    if (threadIdx.x == 0) out[r] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
}

// One warp per restart (restarts spread over the block's warps), with no
// block barrier per restart: 64 restarts cost a few L2 round trips rather
// than 64 block reductions (reduce_keys_kernel's last block). A separate
// function so the rollout kernels do not carry it.
__device__ __forceinline__ void reduce_recs_warps(const RoundArgs& a, const Rec* recs, int n_src,
                                                  Rec* out) {
  const int lane = static_cast<int>(threadIdx.x & 31u), warp = static_cast<int>(threadIdx.x >> 5);
  const int n_warps = static_cast<int>(blockDim.x >> 5);
  for (int r = warp; r < a.restart_count; r += n_warps) {
    Key k = empty_key();
    for (int t = lane; t < n_src; t += 32) {
      const Key o = load_rec_cg(recs + static_cast<size_t>(r) * n_src + t);
      if (o.cls >= 0 && (k.cls < 0 || prefer(o, k))) k = o;
    }
    const Key best = warp_best(k);
    if (lane == 0) out[r] = Rec{best.cls, best.idx, best.k1, best.k2};
  }
  __syncthreads();  // every restart's record is written before publish_round
}

// %globaltimer (ns): the rollout kernel's own span, first CTA start to last
// CTA end (exec[4] holds ~min start, exec[5] max end; published in exec[6]),
// so the roofline divides by the kernel alone without an event between the
// dependent launches.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mark_start(const RoundArgs& a) {
  if (threadIdx.x == 0) atomicMax(&a.exec[4], ~global_ns());
}
__device__ __forceinline__ void mark_end(const RoundArgs& a) {
  if (threadIdx.x == 0) atomicMax(&a.exec[5], global_ns());
}

// Publish the work counters and re-arm the tickets (last block only).
__device__ __forceinline__ void publish_round(const RoundArgs& a) {
  if (threadIdx.x == 0) {
    a.exec[2] = atomicExch(&a.exec[0], 0ull);
    a.exec[3] = atomicExch(&a.exec[1], 0ull);
    const unsigned long long t0 = ~atomicExch(&a.exec[4], 0ull);
    const unsigned long long t1 = atomicExch(&a.exec[5], 0ull);
    a.exec[6] = t1 > t0 ? t1 - t0 : 0ull;
    a.counters[0] = 0;
    a.counters[1] = 0;
    a.counters[2] = 0;  // the window selection that follows counts from zero
  }
  if (a.goal_cut != nullptr) {
    for (int r = threadIdx.x; r < a.cut_slots; r += blockDim.x) {
      a.cut_pub[r] = atomicExch(&a.goal_cut[r], kCutNone);
    }
  }
}

__device__ __forceinline__ void finish_round(const RoundArgs& a, const Rec* recs, int n_src,
                                             Key* red) {
  if (!last_block(a)) return;
  reduce_recs(a, recs, n_src, red, a.out);
  publish_round(a);
}

// Warp-cooperative flush of the lanes' best keys (flagged by `flush`) into
// the warp's per-restart shared table, one restart at a time.
template <class LK>
__device__ __forceinline__ void flush_bests(bool& flush, LK& best, int best_r, Key* table_w,
                                            int lane) {
  unsigned pend = __ballot_sync(kFull, flush);
  while (pend != 0u) {
    const int r0 = __shfl_sync(kFull, best_r, __ffs(pend) - 1);
    const bool mine = flush && best_r == r0;
    const Key k = warp_best(mine ? to_key(best) : empty_key());
    if (lane == 0 && (table_w[r0].cls < 0 || prefer(k, table_w[r0]))) table_w[r0] = k;
    if (mine) {
      flush = false;
      best.cls = -1;
    }
    pend = __ballot_sync(kFull, flush);
  }
}

}  // namespace ppdev

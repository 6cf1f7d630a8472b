// K6 building block: the lexicographic argmin the pressure step needs, reduced with warp
// shuffles (north_star's "warp-ballot/shuffle primitives for the refcount/LRU updates").
//
// pressure_actions (memory.cpp:150-169) picks, per backend, the idle preserved entry with the least
// last_update_ts; ties go to the lexicographically first workflow id (the reference scans entries
// in workflow-id order and replaces only on strict <). A candidate is the triple
//   (ts_key: order-preserving u64 of the f64 ts, rank: the workflow's position in std::string
//    order, idx: the entry / workflow slot)
// compared lexicographically; idx only breaks exact (ts, rank) ties, which distinct workflow ids
// never produce. Reductions are order-independent, so the victim is deterministic.
#pragma once

#include "common.cuh"

namespace sfkv {

struct Cand {
  unsigned long long key;  // ~0 = none
  unsigned int rank;
  long long idx;           // -1 = none
};

__device__ __forceinline__ unsigned long long ts_order_key(double t) {
  if (t == 0.0) t = 0.0;  // -0.0 == 0.0 in the reference's comparison
  const unsigned long long b = (unsigned long long)__double_as_longlong(t);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ Cand cand_none() { return Cand{~0ull, ~0u, -1}; }

// A candidate another CTA published (read past L1: the writer fenced before its ticket).
__device__ __forceinline__ Cand cand_load(const Cand* p) {
  const volatile Cand* q = p;
  return Cand{q->key, q->rank, q->idx};
}

__device__ __forceinline__ bool cand_less(const Cand& a, const Cand& b) {
  if (a.key != b.key) return a.key < b.key;
  if (a.rank != b.rank) return a.rank < b.rank;
  return (unsigned long long)a.idx < (unsigned long long)b.idx;  // -1 (none) sorts last
}

__device__ __forceinline__ Cand warp_argmin(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.key = __shfl_xor_sync(0xffffffffu, c.key, o);
    d.rank = __shfl_xor_sync(0xffffffffu, c.rank, o);
    d.idx = __shfl_xor_sync(0xffffffffu, c.idx, o);
    if (cand_less(d, c)) c = d;
  }
  return c;
}

// Block-wide argmin (blockDim.x a multiple of 32, <= 1024); every thread gets the result.
__device__ __forceinline__ Cand block_argmin(Cand c, Cand* smem /* [32] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  c = warp_argmin(c);
  __syncthreads();  // smem reuse across calls
  if (lane == 0) smem[warp] = c;
  __syncthreads();
  c = lane < nw ? smem[lane] : cand_none();
  return warp_argmin(c);
}

}  // namespace sfkv

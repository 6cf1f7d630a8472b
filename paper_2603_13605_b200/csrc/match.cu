// K1+K2(+K3 lookup): batched chained block hashing fused with the pin compare / table probe.
//
// Replaces SimulatedBackend::prefix_match (simulated_backend.cpp:153-162), a token-by-token LCP of
// std::string tokens against the workflow's own pin, with one pass over the request tokens:
//
//   items   = every 16-token block of every request (CSR batch, flattened; blk_off = scan)
//   digest  = block_digest(k, n, tokens)                           (per item, independent)
//   S_k     = sum_{i<=k} digest_i  (segmented by request)           (CTA scan + decoupled look-back)
//   c_k     = chain_finalize(S_k)                                   (chained block hash)
//   match   : if c_{k-1} equals the pin's hash k-1 (or k == 0), verify block k against the pin's
//             tokens; a differing token at t gives atomicMin(M[r], 16k + t). c_{k-1} is
//             recomputed locally as fin(S_k - digest_k). Blocks past a hash mismatch are never
//             verified, and the first truly differing block is always verified, so M is the exact
//             LCP independent of hash collisions (M is pre-set to min(P, pin_len)).
//   lookup  : probe the global table for c_k (full blocks), verify tokens, report the block id.
//
// Data movement: one thread per block. When the request's token span starts 16-B aligned (the
// host packer guarantees it; any CSR is accepted) a thread loads its 64-B block with four 16-B
// vector loads; a warp's loads cover 2 KiB of contiguous tokens, so DRAM sectors are fully used
// (L1 merges the halves). Algorithmic bytes per block: 64 B tokens + 8 B hash out, + 8 B pin hash
// (+ 4 B block id + 64 B pin tokens when verified) in match mode, + 16 B slot (+ 64 B verify) in
// lookup mode. No tensor cores: this is integer hashing and compares.
#include "pool.cuh"

namespace sfkv {

constexpr int MT = 256;  // items (threads) per tile

struct SegPair {
  uint64_t v;
  int h;
};
struct SegOp {
  __device__ __forceinline__ SegPair operator()(const SegPair& a, const SegPair& b) const {
    return SegPair{b.h ? b.v : a.v + b.v, a.h | b.h};
  }
};

size_t match_tile_state_elems(int64_t n_items) {
  int64_t ntiles = (n_items + MT - 1) / MT;
  return (size_t)(1 + 3 * ntiles);
}

struct MatchKernelArgs {
  MatchArgs a;
  const int64_t* pin_len;
  const int32_t* pin_nblk;
  const int32_t* pin_blk;
  const uint64_t* pin_hash;
  const uint32_t* blk_tok;
  const uint8_t* blk_n;
  const Slot* slots;
  uint64_t slot_mask;
  int32_t max_pin_blocks;
  int64_t ntiles;
  unsigned long long* counter;
  volatile int64_t* flag;
  volatile uint64_t* agg;
  volatile uint64_t* incl;
};

__device__ __forceinline__ void load16_aligned(const uint32_t* __restrict__ p, uint32_t* t) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 v = __ldg(q + i);
    t[4 * i] = v.x;
    t[4 * i + 1] = v.y;
    t[4 * i + 2] = v.z;
    t[4 * i + 3] = v.w;
  }
}

template <int SH>
__device__ __forceinline__ void take16(const uint32_t* w, uint32_t* t) {
#pragma unroll
  for (int j = 0; j < BT; ++j) t[j] = w[j + SH];
}

// Loads block tokens [start, start+nval) zero-padded to 16. Vector path for any alignment: five
// 16-B loads from the aligned-down address and a static funnel by (start & 3); scalar path only
// at the very end of the token array.
__device__ __forceinline__ void load_block(const uint32_t* __restrict__ tok, int64_t start, int nval,
                                           int64_t tok_total, uint32_t* t) {
  const int64_t a0 = start & ~int64_t(3);
  const int sh = (int)(start & 3);
  if (sh == 0 && start + BT <= tok_total) {
    load16_aligned(tok + start, t);
  } else if (a0 + 20 <= tok_total) {
    uint32_t w[20];
    const uint4* q = reinterpret_cast<const uint4*>(tok + a0);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      uint4 v = __ldg(q + i);
      w[4 * i] = v.x;
      w[4 * i + 1] = v.y;
      w[4 * i + 2] = v.z;
      w[4 * i + 3] = v.w;
    }
    switch (sh) {
      case 0: take16<0>(w, t); break;
      case 1: take16<1>(w, t); break;
      case 2: take16<2>(w, t); break;
      default: take16<3>(w, t); break;
    }
  } else {
#pragma unroll
    for (int j = 0; j < BT; ++j) t[j] = j < nval ? __ldg(tok + start + j) : 0u;
    return;
  }
#pragma unroll
  for (int j = 0; j < BT; ++j)
    if (j >= nval) t[j] = 0u;
}

__device__ __forceinline__ bool tokens_equal(const uint32_t* a, const uint32_t* b) {
  bool eq = true;
#pragma unroll
  for (int j = 0; j < BT; ++j) eq &= (a[j] == b[j]);
  return eq;
}

__global__ void __launch_bounds__(MT) match_kernel(MatchKernelArgs K) {
  using BS = cub::BlockScan<SegPair, MT>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t s_off[MT + 1];
  __shared__ int64_t s_tile, s_r0;
  __shared__ uint64_t s_prefix;

  const MatchArgs& A = K.a;
  const int tid = threadIdx.x;
  const int64_t tok_total = A.tok_off[A.n];

  for (;;) {
    if (tid == 0) s_tile = (int64_t)atomicAdd(K.counter, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= K.ntiles) break;
    const int64_t item0 = tile * MT;
    const int64_t item = item0 + tid;
    const bool valid = item < A.n_items;

    // ---- request of each item: window of blk_off in smem, binary search ----
    if (tid == 0) s_r0 = upper_index(A.blk_off, A.n, item0);
    __syncthreads();
    const int64_t r0 = s_r0;
    for (int j = tid; j <= MT; j += MT) {
      int64_t rr = r0 + j;
      s_off[j] = rr <= A.n ? A.blk_off[rr] : INT64_MAX;
    }
    __syncthreads();
    int64_t r = r0;
    if (valid) {
      if (s_off[MT] <= item) {  // > MT requests in this tile (empty requests): global search
        r = upper_index(A.blk_off, A.n, item);
      } else {
        int lo = 0, hi = MT;  // s_off[lo] <= item < s_off[hi]
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (s_off[mid] <= item) lo = mid;
          else hi = mid;
        }
        r = r0 + lo;
      }
    }
    int64_t k = 0, start = 0;
    int nval = 0;
    uint32_t t[BT];
    if (valid) {
      k = item - A.blk_off[r];
      const int64_t tb = A.tok_off[r];
      const int64_t rem = A.tok_off[r + 1] - tb - k * BT;
      nval = (int)(rem < BT ? rem : BT);
      start = tb + k * BT;
      load_block(A.tok, start, nval, tok_total, t);
    } else {
#pragma unroll
      for (int j = 0; j < BT; ++j) t[j] = 0u;
    }
    const uint64_t g = valid ? block_digest_words((uint64_t)k, (uint32_t)nval, t) : 0ull;

    // ---- segmented inclusive scan over the tile + decoupled look-back ----
    SegPair in{g, (valid && k == 0) ? 1 : 0};
    SegPair out, total;
    BS(tmp).InclusiveScan(in, out, SegOp(), total);
    if (tid == 0) {
      uint64_t prefix = 0;
      if (total.h) {
        K.incl[tile] = total.v;
        __threadfence();
        K.flag[tile] = 2;
      } else {
        K.agg[tile] = total.v;
        __threadfence();
        K.flag[tile] = 1;
      }
      if (!in.h && tile > 0) {
        int64_t pred = tile - 1;
        for (;;) {
          int64_t f;
          do {
            f = K.flag[pred];
          } while (f == 0);
          __threadfence();
          if (f == 2) {
            prefix += K.incl[pred];
            break;
          }
          prefix += K.agg[pred];
          --pred;
        }
      }
      if (!total.h) {
        K.incl[tile] = prefix + total.v;
        __threadfence();
        K.flag[tile] = 2;
      }
      s_prefix = prefix;
    }
    __syncthreads();
    const uint64_t S = out.h ? out.v : s_prefix + out.v;
    const uint64_t c = chain_finalize(S);

    if (valid) {
      if (A.out_hash) A.out_hash[item] = c;
      if (A.out_M) {  // ---- pin compare (match / commit) ----
        const int32_t w = A.wf[r];
        const int64_t pl = K.pin_len[w];
        if (pl >= 0 && k < K.pin_nblk[w]) {
          const int64_t pb = (int64_t)w * K.max_pin_blocks;
          const bool prev_ok = (k == 0) || (chain_finalize(S - g) == K.pin_hash[pb + k - 1]);
          if (prev_ok) {
            const int32_t id = K.pin_blk[pb + k];
            const int pn = K.blk_n[id];
            uint32_t q[BT];
            load16_aligned(K.blk_tok + (int64_t)id * BT, q);
            const int lim = nval < pn ? nval : pn;
            int tt = 0;
            bool run = true;
#pragma unroll
            for (int j = 0; j < BT; ++j) {
              run = run && j < lim && q[j] == t[j];
              tt += run ? 1 : 0;
            }
            if (tt < lim)
              atomicMin(reinterpret_cast<unsigned long long*>(A.out_M + r),
                        (unsigned long long)(k * BT + tt));
          }
        }
      }
      if (A.out_block) {  // ---- global table probe (lookup) ----
        int32_t id = -1;
        if (nval == BT) {
          uint64_t s = c & K.slot_mask;
          for (;;) {
            const uint4 raw = __ldg(reinterpret_cast<const uint4*>(K.slots + s));
            const uint64_t key = (uint64_t)raw.x | ((uint64_t)raw.y << 32);
            if (key == c) {
              const int32_t cand = (int32_t)raw.z;
              if (cand >= 0 && K.blk_n[cand] == BT) {
                uint32_t q[BT];
                load16_aligned(K.blk_tok + (int64_t)cand * BT, q);
                if (tokens_equal(q, t)) id = cand;
              }
              break;
            }
            if (key == KEY_EMPTY) break;
            s = (s + 1) & K.slot_mask;
          }
        }
        A.out_block[item] = id;
        if (id < 0)
          atomicMin(reinterpret_cast<unsigned long long*>(A.out_hit + r),
                    (unsigned long long)(k * BT));
      }
    }
    __syncthreads();  // s_off / scan storage reuse by the next tile
  }
}

// M[r] = pin ? min(P, pin_len) : 0 ; hit[r] = 16 * nblocks (lookup)
__global__ void match_init_kernel(MatchArgs A, const int64_t* __restrict__ pin_len) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= A.n) return;
  const int64_t len = A.tok_off[r + 1] - A.tok_off[r];
  if (A.out_M) {
    const int64_t pl = pin_len[A.wf[r]];
    A.out_M[r] = pl < 0 ? 0 : (len < pl ? len : pl);
  }
  if (A.out_hit) A.out_hit[r] = ((len + BT - 1) / BT) * BT;
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int launch_match(sfkv_pool* p, const MatchArgs& a, int64_t* tile_state, cudaStream_t st) {
  const int64_t ntiles = (a.n_items + MT - 1) / MT;
  if (a.n > 0 && (a.out_M || a.out_hit)) {
    match_init_kernel<<<grid_for(a.n, 256, 1 << 20), 256, 0, st>>>(a, p->pin_len);
    SFKV_LAUNCH_CHECK("match_init_kernel");
  }
  if (ntiles == 0) return 0;
  SFKV_CUDA(cudaMemsetAsync(tile_state, 0, sizeof(int64_t) * (1 + ntiles), st));
  MatchKernelArgs K;
  K.a = a;
  K.pin_len = p->pin_len;
  K.pin_nblk = p->pin_nblk;
  K.pin_blk = p->pin_blk;
  K.pin_hash = p->pin_hash;
  K.blk_tok = p->blk_tok;
  K.blk_n = p->blk_n;
  K.slots = p->slots;
  K.slot_mask = (uint64_t)p->table_slots - 1;
  K.max_pin_blocks = p->cfg.max_pin_blocks;
  K.ntiles = ntiles;
  K.counter = reinterpret_cast<unsigned long long*>(tile_state);
  K.flag = tile_state + 1;
  K.agg = reinterpret_cast<volatile uint64_t*>(tile_state + 1 + ntiles);
  K.incl = reinterpret_cast<volatile uint64_t*>(tile_state + 1 + 2 * ntiles);
  int64_t grid = (int64_t)sm_count() * 8;  // persistent: 8 x 256-thread CTAs per SM
  if (grid > ntiles) grid = ntiles;
  match_kernel<<<(unsigned)grid, MT, 0, st>>>(K);
  SFKV_LAUNCH_CHECK("match_kernel");
  return 0;
}

}  // namespace sfkv

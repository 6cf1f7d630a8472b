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
// Data movement: one thread per block, 256-block tiles claimed in order by persistent CTAs. A
// tile's request metadata (block/token offsets, workflow slot, pin length and block count) is
// staged in shared memory by all threads at once from a precomputed tile -> first-request table,
// so no thread walks global memory serially. A thread loads its 64-B block with 16-B vector
// loads at any alignment (a warp covers 2 KiB of contiguous tokens; L1 merges the halves) and
// issues its pin-hash / block-id loads before the tile scan so their latency overlaps the
// look-back. Algorithmic bytes per block: 64 B tokens (+8 B hash out when requested), + 8 B pin
// hash for blocks inside the pin, + 4 B block id + 64 B pin tokens when verified; lookup mode:
// + 16 B table slot (+ 64 B verify). HBM-bound integer work: no tensor cores.
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

// counter + per-tile {status word, first request}
size_t match_tile_state_elems(int64_t n_items) {
  int64_t ntiles = (n_items + MT - 1) / MT;
  return (size_t)(1 + 2 * ntiles);
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
  int64_t ntiles;  // bound
  unsigned long long* counter;
  uint64_t* status;  // per tile: 0 = pending, ST_AGG | aggregate, ST_INCL | inclusive prefix
  const int64_t* tile_r0;
};

constexpr uint64_t ST_AGG = 1ull << 62;
constexpr uint64_t ST_INCL = 2ull << 62;

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

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

// tile_r0[t] = the request holding item t*MT (tiles whose first item lies in request r).
__global__ void tile_first_kernel(const int64_t* __restrict__ blk_off, int64_t n,
                                  int64_t* __restrict__ tile_r0) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = blk_off[r], b1 = blk_off[r + 1];
    for (int64_t t = (b0 + MT - 1) / MT; t * MT < b1; ++t) tile_r0[t] = r;
  }
}

__global__ void __launch_bounds__(MT, 4) match_kernel(MatchKernelArgs K) {
  using BS = cub::BlockScan<SegPair, MT>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t s_off[MT + 1];   // blk_off of the tile's request window
  __shared__ int64_t s_toff[MT + 1];  // tok_off
  __shared__ int64_t s_pl[MT];        // pin length (-1: none)
  __shared__ int32_t s_wf[MT];
  __shared__ int32_t s_pnb[MT];
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_prefix;

  const MatchArgs& A = K.a;
  const int tid = threadIdx.x;
  const bool match_mode = A.out_M != nullptr;
  const int64_t tok_total = A.tok_off[A.n];
  // A.n_items is only an upper bound (it sizes the look-back state); the exact count is on device.
  const int64_t n_items = A.blk_off[A.n];
  const int64_t ntiles = (n_items + MT - 1) / MT;

  for (;;) {
    // Take the ticket only when starting the tile: a held-but-unstarted ticket would make every
    // later tile's look-back wait on it.
    if (tid == 0) s_tile = (int64_t)atomicAdd(K.counter, 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t item0 = tile * MT;
    const int64_t item = item0 + tid;
    const bool valid = item < n_items;

    // ---- stage the request window [r0, r0 + MT] (all threads in parallel) ----
    const int64_t r0 = K.tile_r0[tile];
    {
      const int64_t rr = r0 + tid;
      s_off[tid] = rr <= A.n ? A.blk_off[rr] : INT64_MAX;
      s_toff[tid] = rr <= A.n ? A.tok_off[rr] : 0;
      if (match_mode && rr < A.n) {
        const int32_t w = A.wf[rr];
        const int64_t pl = K.pin_len[w];
        s_wf[tid] = w;
        s_pl[tid] = pl;
        s_pnb[tid] = pl < 0 ? 0 : K.pin_nblk[w];
      }
      if (tid == 0) {
        const int64_t re = r0 + MT;
        s_off[MT] = re <= A.n ? A.blk_off[re] : INT64_MAX;
        s_toff[MT] = re <= A.n ? A.tok_off[re] : 0;
      }
    }
    __syncthreads();

    // ---- my block: request (smem binary search), tokens, early pin loads ----
    int64_t r = r0, k = 0, tb = 0, te = 0;
    int32_t w = 0, pnb = 0;
    int64_t pl = -1;
    if (valid) {
      if (s_off[MT] <= item) {  // > MT requests in this tile (empty requests): global path
        r = upper_index(A.blk_off, A.n, item);
        k = item - A.blk_off[r];
        tb = A.tok_off[r];
        te = A.tok_off[r + 1];
        if (match_mode) {
          w = A.wf[r];
          pl = K.pin_len[w];
          pnb = pl < 0 ? 0 : K.pin_nblk[w];
        }
      } else {
        int lo = 0, hi = MT;  // s_off[lo] <= item < s_off[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_off[mid] <= item) lo = mid;
          else hi = mid;
        }
        r = r0 + lo;
        k = item - s_off[lo];
        tb = s_toff[lo];
        te = s_toff[lo + 1];
        if (match_mode) {
          w = s_wf[lo];
          pl = s_pl[lo];
          pnb = s_pnb[lo];
        }
      }
    }
    const int64_t rem = te - tb - k * BT;
    const int nval = valid ? (int)(rem < BT ? rem : BT) : 0;
    uint32_t t[BT];
    if (valid) {
      load_block(A.tok, tb + k * BT, nval, tok_total, t);
    } else {
#pragma unroll
      for (int j = 0; j < BT; ++j) t[j] = 0u;
    }
    // pin metadata needed after the scan, issued now so its latency overlaps the look-back
    const bool in_pin = match_mode && valid && pl >= 0 && k < pnb;
    const int64_t pb = (int64_t)w * K.max_pin_blocks;
    uint64_t prev_pin_hash = 0;
    int32_t pin_id = 0;
    if (in_pin) {
      if (k > 0) prev_pin_hash = __ldg(K.pin_hash + pb + k - 1);
      pin_id = __ldg(K.pin_blk + pb + k);
    }
    const uint64_t g = valid ? block_digest_words((uint64_t)k, (uint32_t)nval, t) : 0ull;

    // ---- segmented inclusive scan over the tile + decoupled look-back ----
    SegPair in{g, (valid && k == 0) ? 1 : 0};
    SegPair out, total;
    BS(tmp).InclusiveScan(in, out, SegOp(), total);
    if (tid == 0) {
      // status word = flag << 62 | (sum mod 2^62): one relaxed 64-bit store / load, no fences.
      uint64_t prefix = 0;
      st_status(K.status + tile, (total.h ? ST_INCL : ST_AGG) | (total.v & CHAIN_MASK));
      if (!in.h && tile > 0) {
        int64_t pred = tile - 1;
        for (;;) {
          uint64_t s;
          do {
            s = ld_status(K.status + pred);
          } while (s == 0);
          prefix += s & CHAIN_MASK;
          if ((s & ~CHAIN_MASK) == ST_INCL) break;
          --pred;
        }
      }
      if (!total.h) st_status(K.status + tile, ST_INCL | ((prefix + total.v) & CHAIN_MASK));
      s_prefix = prefix;
    }
    __syncthreads();
    const uint64_t S = out.h ? out.v : s_prefix + out.v;
    const uint64_t c = chain_finalize(S);

    if (valid) {
      if (A.out_hash) A.out_hash[item] = c;
      if (in_pin) {  // ---- pin compare (match / commit) ----
        const bool prev_ok = (k == 0) || (chain_finalize(S - g) == prev_pin_hash);
        if (prev_ok) {
          const int pn = K.blk_n[pin_id];
          uint32_t q[BT];
          load16_aligned(K.blk_tok + (int64_t)pin_id * BT, q);
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
    __syncthreads();  // window / scan storage reuse; s_tile (next ticket) visible
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
  K.status = reinterpret_cast<uint64_t*>(tile_state + 1);
  int64_t* tile_r0 = tile_state + 1 + ntiles;
  K.tile_r0 = tile_r0;
  tile_first_kernel<<<grid_for(a.n, 256, sm_count() * 8), 256, 0, st>>>(a.blk_off, a.n, tile_r0);
  int64_t grid = (int64_t)sm_count() * 4;  // persistent: 4 x 256-thread CTAs per SM
  if (grid > ntiles) grid = ntiles;
  match_kernel<<<(unsigned)grid, MT, 0, st>>>(K);
  SFKV_LAUNCH_CHECK("match_kernel");
  return 0;
}

}  // namespace sfkv

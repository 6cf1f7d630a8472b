// K1+K2(+K3 lookup): batched chained block hashing fused with the pin compare / table probe.
//
// Replaces SimulatedBackend::prefix_match (simulated_backend.cpp:153-162), a token-by-token LCP of
// std::string tokens against the workflow's own pin, with one pass over the request tokens:
//
//   items   = every 16-token block of every request (CSR batch, flattened; blk_off = scan)
//   digest  = block_digest(k, n, tokens)                           (per item, independent)
//   S_k     = sum_{i<=k} digest_i mod 2^62 (segmented by request)   (warp scan + decoupled look-back)
//   c_k     = chain_finalize(S_k)                                   (chained block hash)
//   match   : if c_{k-1} equals the pin's hash k-1 (or k == 0), verify block k against the pin's
//             tokens; a differing token at t gives atomicMin(M[r], 16k + t). c_{k-1} is
//             recomputed locally as fin(S_k - digest_k). Blocks past a hash mismatch are never
//             verified, and the first truly differing block is always verified, so M is the exact
//             LCP independent of hash collisions (M is pre-set to min(P, pin_len)).
//   lookup  : probe the global table for c_k (full blocks), verify tokens, report the block id.
//
// Execution: warp-centric and barrier-free. A warp owns a 32-block tile (one block per lane);
// tiles are assigned statically round-robin to the resident warps of a persistent grid, so every
// warp walks its tiles in increasing order and a tile's predecessors are always owned by warps
// that make progress. Request metadata for the tile's window of up to 32 requests is loaded one
// request per lane and redistributed with shuffles (5-step shuffle binary search). The chain sum
// is a warp shuffle segmented scan; the carry across tiles is a decoupled look-back in which the
// 32 lanes read 32 predecessor status words at once (flag and 62-bit sum packed in one word:
// relaxed 64-bit loads/stores, no fences). A lane loads its 64-B block with 16-B vector loads at
// any alignment (a warp covers 2 KiB of contiguous tokens) and issues its pin-hash / block-id
// loads before the scan. Algorithmic bytes per block: 64 B tokens (+8 B hash out when requested),
// + 8 B pin hash for blocks inside the pin, + 4 B block id + 64 B pin tokens when verified; lookup
// mode: + 16 B table slot (+ 64 B verify). HBM-bound integer work: no tensor cores.
#include "pool.cuh"

namespace sfkv {

constexpr int WT = 32;  // items per warp tile
#ifndef MATCH_MIN_CTAS
#define MATCH_MIN_CTAS 3  // 256-thread CTAs per SM: 80 registers, no spills
#endif

// counter (unused) + per-tile {status word, first request} + 32-B request records [n+1]
size_t match_tile_state_elems(int64_t n_items, int64_t n_requests) {
  int64_t ntiles = (n_items + WT - 1) / WT;
  return (size_t)(((1 + 2 * ntiles + 3) & ~int64_t(3)) + 4 * (n_requests + 1));
}

struct ReqRec;

struct MatchKernelArgs {
  MatchArgs a;
  const ReqRec* rec;
  const int32_t* pin_blk;
  const uint64_t* pin_hash;
  const uint32_t* blk_tok;
  const uint8_t* blk_n;
  const Slot* slots;
  uint64_t slot_mask;
  int32_t max_pin_blocks;
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

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
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

// Per-request record staged once per batch by request_prep_kernel (one request per thread, so
// the dependent wf -> pin_len load chain runs fully parallel instead of inside every tile).
struct __align__(32) ReqRec {
  int64_t blk_off;   // first item of the request
  int64_t tok_off;   // first token
  int64_t pin_len;   // -1: the workflow has no pin (or lookup mode)
  int32_t wf;
  int32_t pad;
};

// rec[r] for r in [0, n] (rec[n] closes the last request) and tile_r0[t] = the request holding
// item t*WT (tiles whose first item lies in request r).
__global__ void request_prep_kernel(MatchArgs A, const int64_t* __restrict__ pin_len,
                                    ReqRec* __restrict__ rec, int64_t* __restrict__ tile_r0) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= A.n;
       r += (int64_t)gridDim.x * blockDim.x) {
    ReqRec q;
    q.blk_off = A.blk_off[r];
    q.tok_off = A.tok_off[r];
    q.wf = 0;
    q.pin_len = -1;
    q.pad = 0;
    if (r < A.n && A.wf) {
      q.wf = A.wf[r];
      q.pin_len = pin_len[q.wf];
    }
    rec[r] = q;
    if (r < A.n) {
      const int64_t b1 = A.blk_off[r + 1];
      for (int64_t t = (q.blk_off + WT - 1) / WT; t * WT < b1; ++t) tile_r0[t] = r;
    }
  }
}

__device__ __forceinline__ ReqRec load_rec(const ReqRec* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = __ldg(q), b = __ldg(q + 1);
  ReqRec r;
  r.blk_off = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
  r.tok_off = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
  r.pin_len = (int64_t)(((uint64_t)(uint32_t)b.y << 32) | (uint32_t)b.x);
  r.wf = b.z;
  r.pad = 0;
  return r;
}

// Aggregate of one tile computed from scratch: (sum of digests since the tile's last segment
// head, whether the tile holds a head). Used only when a predecessor's status stays unpublished
// (e.g. its warp is not resident because other kernels occupy the GPU), so the look-back always
// makes progress without relying on co-residency. Returns the status word the owner would publish.
__device__ __forceinline__ uint64_t tile_status_fallback(const MatchKernelArgs& K, int64_t tile,
                                                      int64_t n_items, int64_t tok_total) {
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const int64_t item = tile * WT + lane;
  uint64_t v = 0;
  int h = 0;
  if (item < n_items) {
    const int64_t r = upper_index(A.blk_off, A.n, item);
    const int64_t k = item - A.blk_off[r];
    const int64_t tb = A.tok_off[r];
    const int64_t rem = A.tok_off[r + 1] - tb - k * BT;
    const int nval = (int)(rem < BT ? rem : BT);
    uint32_t t[BT];
    load_block(A.tok, tb + k * BT, nval, tok_total, t);
    v = block_digest_words((uint64_t)k, (uint32_t)nval, t);
    h = k == 0;
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t vv = __shfl_up_sync(0xffffffffu, v, d);
    const int hh = __shfl_up_sync(0xffffffffu, h, d);
    if (lane >= d) {
      if (!h) v += vv;
      h |= hh;
    }
  }
  v = __shfl_sync(0xffffffffu, v, 31);
  h = __shfl_sync(0xffffffffu, h, 31);
  return (h ? ST_INCL : ST_AGG) | (v & CHAIN_MASK);
}

template <bool LOOKUP>
__global__ void __launch_bounds__(256, MATCH_MIN_CTAS) match_kernel(MatchKernelArgs K) {
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool match_mode = A.out_M != nullptr;
  const int64_t tok_total = A.tok_off[A.n];
  // A.n_items is only an upper bound (it sizes the tile state); the exact count is on device.
  const int64_t n_items = A.blk_off[A.n];
  const int64_t ntiles = (n_items + WT - 1) / WT;

  int64_t r0_next = gwarp < ntiles ? K.tile_r0[gwarp] : 0;
  for (int64_t tile = gwarp; tile < ntiles; tile += nwarps) {
    const int64_t item0 = tile * WT;
    const int64_t item = item0 + lane;
    const bool valid = item < n_items;

    // ---- request window [r0, r0 + 32]: lane j holds request r0 + j (one 32-B record) ----
    const int64_t r0 = r0_next;
    const int64_t rr = r0 + lane <= A.n ? r0 + lane : A.n;
    const ReqRec rec_j = load_rec(K.rec + rr);
    const int64_t off_32 = r0 + WT <= A.n ? K.rec[r0 + WT].blk_off : INT64_MAX;
    const int64_t toff_32 = r0 + WT <= A.n ? K.rec[r0 + WT].tok_off : 0;
    if (tile + nwarps < ntiles) r0_next = K.tile_r0[tile + nwarps];  // prefetch
    const int64_t off_j = r0 + lane <= A.n ? rec_j.blk_off : INT64_MAX;
    // largest j in [0, 31] with off_j <= item (off non-decreasing); j = 32 if off_32 <= item
    int j = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int64_t v = __shfl_sync(0xffffffffu, off_j, j + s);
      if (v <= item) j += s;
    }
    const int64_t off_r = __shfl_sync(0xffffffffu, off_j, j);
    int64_t tb = __shfl_sync(0xffffffffu, rec_j.tok_off, j);
    const int64_t te_in = __shfl_sync(0xffffffffu, rec_j.tok_off, (j + 1) & 31);
    int32_t w = __shfl_sync(0xffffffffu, rec_j.wf, j);
    int64_t pl = __shfl_sync(0xffffffffu, rec_j.pin_len, j);
    int64_t r = r0 + j, k = item - off_r, te = j == 31 ? toff_32 : te_in;
    if (valid && off_32 <= item) {  // > 32 requests in this tile (empty requests): global path
      r = upper_index(A.blk_off, A.n, item);
      const ReqRec a = load_rec(K.rec + r);
      k = item - a.blk_off;
      tb = a.tok_off;
      te = K.rec[r + 1].tok_off;
      w = a.wf;
      pl = a.pin_len;
    }
    const int64_t rem = te - tb - k * BT;
    const int nval = valid ? (int)(rem < BT ? rem : BT) : 0;

    // ---- tokens + pin metadata (one round trip), then the pin block's tokens ----
    const bool in_pin = match_mode && valid && pl >= 0 && k < (pl + BT - 1) / BT;
    const int64_t pb = (int64_t)w * K.max_pin_blocks;
    uint64_t prev_pin_hash = 0;
    int32_t pin_id = 0;
    if (in_pin) {
      if (k > 0) prev_pin_hash = __ldg(K.pin_hash + pb + k - 1);
      pin_id = __ldg(K.pin_blk + pb + k);
    }
    uint32_t t[BT];
    if (valid) {
      load_block(A.tok, tb + k * BT, nval, tok_total, t);
    } else {
#pragma unroll
      for (int i = 0; i < BT; ++i) t[i] = 0u;
    }
    const uint64_t g = valid ? block_digest_words((uint64_t)k, (uint32_t)nval, t) : 0ull;
    // lookup mode keeps the tokens for verify-on-hit
    uint32_t tk[BT];
    if constexpr (LOOKUP) {
#pragma unroll
      for (int i = 0; i < BT; ++i) tk[i] = t[i];
    }

    // ---- warp segmented inclusive scan of (digest, head) ----
    uint64_t v = g;
    int h = (valid && k == 0) ? 1 : 0;
    const int head0 = __shfl_sync(0xffffffffu, h, 0);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t vv = __shfl_up_sync(0xffffffffu, v, d);
      const int hh = __shfl_up_sync(0xffffffffu, h, d);
      if (lane >= d) {
        if (!h) v += vv;
        h |= hh;
      }
    }
    const uint64_t tot_v = __shfl_sync(0xffffffffu, v, 31);
    const int tot_h = __shfl_sync(0xffffffffu, h, 31);

    // ---- decoupled look-back, 32 predecessors per round ----
    // The aggregate is published as soon as the digests are scanned (nothing else delays the
    // successors); the pin block's tokens are fetched now so their latency overlaps the look-back.
    if (lane == 0) st_status(K.status + tile, (tot_h ? ST_INCL : ST_AGG) | (tot_v & CHAIN_MASK));
    uint32_t q[BT];
    int pn = 0;
    if (in_pin) {
      load16_aligned(K.blk_tok + (int64_t)pin_id * BT, q);
      pn = K.blk_n[pin_id];
    }
    uint64_t prefix = 0;
    if (!head0 && tile > 0) {
      int64_t base = tile - 1;
      int spins = 0;
      for (;;) {
        const int64_t p = base - lane;
        uint64_t s = p >= 0 ? ld_status(K.status + p) : ST_INCL;
        unsigned ready = __ballot_sync(0xffffffffu, s != 0);
        unsigned incl = __ballot_sync(0xffffffffu, (s & ~CHAIN_MASK) == ST_INCL);
        int first = incl ? __ffs(incl) - 1 : 31;
        unsigned need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if ((ready & need) != need) {  // a needed predecessor has not published yet
          if (++spins < 1024) continue;
          // forward progress: compute the nearest unpublished predecessor's aggregate ourselves
          const int miss = __ffs(~ready & need) - 1;
          const uint64_t fs = tile_status_fallback(K, base - miss, n_items, tok_total);
          if (lane == miss) s = fs;
          ready = __ballot_sync(0xffffffffu, s != 0);
          incl = __ballot_sync(0xffffffffu, (s & ~CHAIN_MASK) == ST_INCL);
          first = incl ? __ffs(incl) - 1 : 31;
          need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
          if ((ready & need) != need) continue;  // another gap further back: repeat
        }
        spins = 0;
        prefix += warp_sum(lane <= first ? (s & CHAIN_MASK) : 0ull);
        if (incl) break;
        base -= 32;
      }
    }
    if (!tot_h && lane == 0) st_status(K.status + tile, ST_INCL | ((prefix + tot_v) & CHAIN_MASK));
    const uint64_t S = h ? v : prefix + v;
    const uint64_t c = chain_finalize(S);

    if (valid) {
      if (A.out_hash) A.out_hash[item] = c;
      if (in_pin) {  // ---- pin compare (match / commit) ----
        // Only blocks whose prefix hash matches the pin's are compared token by token; the first
        // truly differing block always qualifies, so M stays exact whatever the hash does.
        const bool prev_ok = (k == 0) || (chain_finalize(S - g) == prev_pin_hash);
        if (prev_ok) {
          uint32_t u[BT];  // request tokens again: an L1 hit, cheaper than keeping them live
          load_block(A.tok, tb + k * BT, nval, tok_total, u);
          const int lim = nval < pn ? nval : pn;
          int lcp = 0;
          bool run = true;
#pragma unroll
          for (int i = 0; i < BT; ++i) {
            run = run && i < lim && q[i] == u[i];
            lcp += run ? 1 : 0;
          }
          if (lcp < lim)
            atomicMin(reinterpret_cast<unsigned long long*>(A.out_M + r),
                      (unsigned long long)(k * BT + lcp));
        }
      }
      if constexpr (LOOKUP) {  // ---- global table probe (lookup) ----
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
                if (tokens_equal(q, tk)) id = cand;
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
  const int64_t ntiles = (a.n_items + WT - 1) / WT;
  if (a.n > 0 && (a.out_M || a.out_hit)) {
    match_init_kernel<<<grid_for(a.n, 256, 1 << 20), 256, 0, st>>>(a, p->pin_len);
    SFKV_LAUNCH_CHECK("match_init_kernel");
  }
  if (ntiles == 0) return 0;
  SFKV_CUDA(cudaMemsetAsync(tile_state, 0, sizeof(int64_t) * (1 + ntiles), st));
  MatchKernelArgs K;
  K.a = a;
  K.pin_blk = p->pin_blk;
  K.pin_hash = p->pin_hash;
  K.blk_tok = p->blk_tok;
  K.blk_n = p->blk_n;
  K.slots = p->slots;
  K.slot_mask = (uint64_t)p->table_slots - 1;
  K.max_pin_blocks = p->cfg.max_pin_blocks;
  K.status = reinterpret_cast<uint64_t*>(tile_state + 1);
  int64_t* tile_r0 = tile_state + 1 + ntiles;
  K.tile_r0 = tile_r0;
  // records start 32-B aligned after the per-tile arrays
  int64_t rec_off = (1 + 2 * ntiles + 3) & ~int64_t(3);
  ReqRec* rec = reinterpret_cast<ReqRec*>(tile_state + rec_off);
  K.rec = rec;
  request_prep_kernel<<<grid_for(a.n + 1, 256, sm_count() * 8), 256, 0, st>>>(a, p->pin_len, rec,
                                                                             tile_r0);
  // persistent: 4 x 256-thread CTAs per SM; tiles assigned round-robin to warps
  int64_t grid = (int64_t)sm_count() * MATCH_MIN_CTAS;
  const int64_t need = (ntiles + 7) / 8;
  if (grid > need) grid = need;
  if (a.out_block) match_kernel<true><<<(unsigned)grid, 256, 0, st>>>(K);
  else match_kernel<false><<<(unsigned)grid, 256, 0, st>>>(K);
  SFKV_LAUNCH_CHECK("match_kernel");
  return 0;
}

}  // namespace sfkv

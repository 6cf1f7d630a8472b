// K1+K2(+K3 lookup): stage-prefix lookup — exact LCP against each workflow's pin, chained block
// hashes, and (lookup mode) the global dedup-table probe.
//
// Replaces SimulatedBackend::prefix_match (simulated_backend.cpp:153-162), a token-by-token LCP of
// std::string tokens against the workflow's own pin. Items are the 16-token blocks of a CSR batch.
//
//   M       = LCP(pin, tokens) = min over in-pin blocks k of (16k + t_k), t_k the first differing
//             token of block k against the pin's block k (blocks that match contribute nothing; M
//             starts at min(P, pin_len)). Every in-pin block is compared, so the minimum — the
//             first truly differing block — is exact with no dependence on hashing.
//   digest  = block_digest(k, n, tokens), per block
//   c_k     = chain_finalize(sum_{i<=k} digest_i mod 2^62)   (chained block hash, segmented scan)
//   lookup  : probe the global table for c_k (full blocks), verify tokens, report the block id.
//
// Launches (no kernel ever waits on another CTA or warp):
//   match_prep_kernel   single-pass request scan (decoupled look-back over 256-request tiles):
//                       blk_off, a 32-B record per request {blk_off, tok_off, pin_len, wf}, the
//                       tile -> first-request map, M / hit initial values.
//   match_block_kernel  one warp per 32-block tile, one block per lane: request window (one record
//                       per lane + shuffle search), 16-B vector token loads at any alignment, block
//                       id + pin-block tokens, in-block LCP, warp segmented-min and one atomicMin per
//                       (warp, request). When hashes are wanted it also runs the warp segmented scan
//                       of digests and writes each block's local inclusive sum (with its segment-head
//                       bit) and the tile's aggregate — final values, nobody waits for them.
//   match_chain_kernel  (hashes / lookup only) one warp per tile: carry = sum of the preceding
//                       tiles' aggregates back to the nearest tile holding the request's head (32
//                       status words per read), chained hashes out, table probe in lookup mode.
// Algorithmic bytes per block: 64 B tokens + 4 B block id + 64 B pin tokens (blocks inside the pin)
// + 8 B hash out when requested; lookup mode + 16 B table slot (+ 64 B verify on a key hit);
// + 32 B per request. Implementation traffic on top: 8 B written + read per block (local sums)
// when hashes are wanted. HBM-bound integer work: no tensor cores.
#include "pool.cuh"

namespace sfkv {

constexpr int WT = 32;                        // items per warp tile
constexpr int MATCH_THREADS = 256;
constexpr int PREP_THREADS = 256;
constexpr int PREP_PER_THREAD = 1;
constexpr int PREP_TILE = PREP_THREADS * PREP_PER_THREAD;

constexpr uint64_t ST_AGG = 1ull << 62;
constexpr uint64_t ST_INCL = 2ull << 62;

struct __align__(32) ReqRec {
  int64_t blk_off;  // first item of the request
  int64_t tok_off;  // first token
  int64_t pin_len;  // -1: no pin (or lookup mode)
  int32_t wf;
  int32_t pad;
};

// Scratch layout (int64 units): [prep ticket][prep status x nprep][tile status x ntiles]
// [tile_r0 x ntiles][pad to 4][records x (n+1) x 4][local sums x n_items]
static int64_t prep_tiles(int64_t n) { return (n + PREP_TILE - 1) / PREP_TILE; }
size_t match_tile_state_elems(int64_t n_items, int64_t n_requests) {
  const int64_t ntiles = (n_items + WT - 1) / WT;
  const int64_t head = 1 + prep_tiles(n_requests) + 2 * ntiles;
  return (size_t)(((head + 3) & ~int64_t(3)) + 4 * (n_requests + 1) + n_items);
}

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

// ---------------------------------------------------------------- prep ----------------------
struct PrepArgs {
  int64_t n;
  const int64_t* tok_off;
  const int32_t* wf;  // nullable (lookup)
  const int64_t* pin_len;
  int64_t* blk_off;   // out [n+1]
  ReqRec* rec;        // out [n+1]
  int64_t* tile_r0;   // out
  int64_t* out_M;     // nullable: min(P, pin_len) or 0
  int64_t* out_hit;   // nullable: 16 * blocks
  unsigned long long* ticket;
  uint64_t* pstatus;  // prep tile status (zeroed by the host)
};

__global__ void __launch_bounds__(PREP_THREADS) match_prep_kernel(PrepArgs P) {
  using BS = cub::BlockScan<int64_t, PREP_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t s_tile, s_prefix;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = (int64_t)atomicAdd(P.ticket, 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t r_base = tile * PREP_TILE + (int64_t)tid * PREP_PER_THREAD;
  int64_t len[PREP_PER_THREAD], cnt = 0;
#pragma unroll
  for (int i = 0; i < PREP_PER_THREAD; ++i) {
    const int64_t r = r_base + i;
    len[i] = r < P.n ? P.tok_off[r + 1] - P.tok_off[r] : 0;
    cnt += (len[i] + BT - 1) / BT;
  }
  int64_t excl, total;
  BS(tmp).ExclusiveSum(cnt, excl, total);
  if (tid < 32) {  // warp 0: publish, then look back 32 predecessor tiles per read
    const int lane = tid;
    if (lane == 0) st_status(P.pstatus + tile, (tile == 0 ? ST_INCL : ST_AGG) | (uint64_t)total);
    uint64_t prefix = 0;
    for (int64_t base = tile - 1; base >= 0; base -= 32) {
      const int64_t p = base - lane;
      uint64_t s;
      unsigned incl;
      int first;
      for (;;) {  // predecessors hold earlier tickets, so they are running: plain spin
        s = p >= 0 ? ld_status(P.pstatus + p) : ST_INCL;
        incl = __ballot_sync(0xffffffffu, (s & ~CHAIN_MASK) == ST_INCL);
        first = incl ? __ffs(incl) - 1 : 31;
        const unsigned need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if ((__ballot_sync(0xffffffffu, s != 0) & need) == need) break;
      }
      prefix += warp_sum(lane <= first ? (s & CHAIN_MASK) : 0ull);
      if (incl) break;
    }
    if (lane == 0) {
      if (tile > 0) st_status(P.pstatus + tile, ST_INCL | (prefix + (uint64_t)total));
      s_prefix = (int64_t)prefix;
    }
  }
  __syncthreads();
  int64_t b = s_prefix + excl;
#pragma unroll
  for (int i = 0; i < PREP_PER_THREAD; ++i) {
    const int64_t r = r_base + i;
    if (r >= P.n) break;
    const int64_t nb = (len[i] + BT - 1) / BT;
    ReqRec q;
    q.blk_off = b;
    q.tok_off = P.tok_off[r];
    q.pin_len = -1;
    q.wf = 0;
    q.pad = 0;
    if (P.wf) {
      q.wf = P.wf[r];
      q.pin_len = P.pin_len[q.wf];
    }
    P.rec[r] = q;
    P.blk_off[r] = b;
    for (int64_t t = (b + WT - 1) / WT; t * WT < b + nb; ++t) P.tile_r0[t] = r;
    if (P.out_M) P.out_M[r] = q.pin_len < 0 ? 0 : (len[i] < q.pin_len ? len[i] : q.pin_len);
    if (P.out_hit) P.out_hit[r] = nb * BT;
    b += nb;
    if (r == P.n - 1) {  // closing record
      ReqRec e;
      e.blk_off = b;
      e.tok_off = P.tok_off[P.n];
      e.pin_len = -1;
      e.wf = 0;
      e.pad = 0;
      P.rec[P.n] = e;
      P.blk_off[P.n] = b;
    }
  }
}

// ---------------------------------------------------------------- per-block pass -----------
struct MatchKernelArgs {
  MatchArgs a;
  const ReqRec* rec;
  const uint32_t* pin_tok;
  const uint32_t* blk_tok;
  const uint8_t* blk_n;
  const Slot* slots;
  uint64_t slot_mask;
  int32_t max_pin_blocks;
  uint64_t* status;  // per tile: flag | aggregate since the tile's last segment head (final)
  uint64_t* local;   // per block: bit 63 = a segment head at or before it in the tile | local sum
  const int64_t* tile_r0;
  int hashes;        // chained hashes (or lookup) requested
};

struct Win {  // lane j holds request r0 + j of a tile's window
  int64_t r0, off_j, toff_j, pl_j, off32, toff32;
  int32_t wf_j;
};

struct Ctx {  // one lane's block of one tile
  int64_t item, r, k, start, pin_base, pin_len;
  int32_t nval;
  bool valid, in_pin;
};

__device__ __forceinline__ Win load_win(const MatchKernelArgs& K, int64_t r0) {
  const int lane = threadIdx.x & 31;
  const int64_t n = K.a.n;
  Win w;
  w.r0 = r0;
  w.off_j = INT64_MAX;
  w.toff_j = 0;
  w.pl_j = -1;
  w.wf_j = 0;
  w.off32 = INT64_MAX;
  w.toff32 = 0;
  const int64_t rr = r0 + lane;
  if (rr <= n) {
    const int4* q = reinterpret_cast<const int4*>(K.rec + rr);
    const int4 a = __ldg(q), b = __ldg(q + 1);
    w.off_j = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
    w.toff_j = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
    w.pl_j = (int64_t)(((uint64_t)(uint32_t)b.y << 32) | (uint32_t)b.x);
    w.wf_j = b.z;
  }
  if (r0 + WT <= n) {
    w.off32 = __ldg(&K.rec[r0 + WT].blk_off);
    w.toff32 = __ldg(&K.rec[r0 + WT].tok_off);
  }
  return w;
}

__device__ __forceinline__ Ctx resolve(const MatchKernelArgs& K, const Win& w, int64_t tile,
                                       int64_t n_items, bool match_mode) {
  const int lane = threadIdx.x & 31;
  Ctx c;
  c.item = tile * WT + lane;
  c.valid = c.item < n_items;
  int j = 0;  // largest j in [0, 31] with off_j <= item
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int64_t v = __shfl_sync(0xffffffffu, w.off_j, j + s);
    if (v <= c.item) j += s;
  }
  const int64_t off_r = __shfl_sync(0xffffffffu, w.off_j, j);
  int64_t tb = __shfl_sync(0xffffffffu, w.toff_j, j);
  const int64_t te_in = __shfl_sync(0xffffffffu, w.toff_j, (j + 1) & 31);
  int32_t wf = __shfl_sync(0xffffffffu, w.wf_j, j);
  int64_t pl = __shfl_sync(0xffffffffu, w.pl_j, j);
  c.r = w.r0 + j;
  c.k = c.item - off_r;
  int64_t te = j == 31 ? w.toff32 : te_in;
  if (c.valid && w.off32 <= c.item) {  // > 32 requests in this tile (empty requests)
    c.r = upper_index(K.a.blk_off, K.a.n, c.item);
    const ReqRec& q = K.rec[c.r];
    c.k = c.item - q.blk_off;
    tb = q.tok_off;
    te = K.rec[c.r + 1].tok_off;
    wf = q.wf;
    pl = q.pin_len;
  }
  if (!c.valid) c.r = -1 - lane;  // never merges with a real request in segmented reductions
  const int64_t rem = te - tb - c.k * BT;
  c.nval = c.valid ? (int32_t)(rem < BT ? rem : BT) : 0;
  c.start = tb + c.k * BT;
  c.in_pin = match_mode && c.valid && pl >= 0 && c.k < (pl + BT - 1) / BT;
  c.pin_base = (int64_t)wf * K.max_pin_blocks;
  c.pin_len = pl;
  return c;
}

__device__ __forceinline__ void load16_aligned(const uint32_t* __restrict__ p, uint32_t* t) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 v = __ldg(q + i);
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

// Block tokens [start, start+nval) zero-padded to 16: five 16-B loads from the aligned-down
// address and a static funnel by (start & 3) at any alignment; scalar only at the array end.
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
      const uint4 v = __ldg(q + i);
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

// One warp per 32-block tile, one block per lane, non-persistent: at 46 registers ~40 warps per SM
// keep enough tiles in flight to cover the window -> tokens/pin-tokens round trips. (A persistent
// cp.async-pipelined variant measured slower: with the inter-warp dependencies gone, occupancy and
// not load latency decides; see profiles/round1/README.md.)
__global__ void __launch_bounds__(MATCH_THREADS) match_block_kernel(MatchKernelArgs K) {
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_items = K.rec[A.n].blk_off;
  if (tile * WT >= n_items) return;
  const int64_t tok_total = K.rec[A.n].tok_off;
  const bool match_mode = A.out_M != nullptr;
  const Ctx c = resolve(K, load_win(K, K.tile_r0[tile]), tile, n_items, match_mode);

  uint32_t t[BT];
  if (c.valid) {
    load_block(A.tok, c.start, c.nval, tok_total, t);
  } else {
#pragma unroll
    for (int j = 0; j < BT; ++j) t[j] = 0u;
  }

  // ---- M: first differing token against the pin's block, warp segmented min, one atomic ----
  if (match_mode) {
    unsigned long long m = ~0ull;
    if (c.in_pin) {  // the pin's block k from its pin-major token copy (coalesced, no indirection)
      uint32_t q[BT];
      load16_aligned(K.pin_tok + (c.pin_base + c.k) * BT, q);
      const int64_t prem = c.pin_len - c.k * BT;
      const int pn = (int)(prem < BT ? prem : BT);
      const int lim = c.nval < pn ? c.nval : pn;
      int lcp = 0;
      bool run = true;
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        run = run && j < lim && q[j] == t[j];
        lcp += run ? 1 : 0;
      }
      if (lcp < lim) m = (unsigned long long)(c.k * BT + lcp);
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_down_sync(0xffffffffu, m, d);
      const int64_t orr = __shfl_down_sync(0xffffffffu, c.r, d);
      if (lane + d < 32 && orr == c.r && o < m) m = o;
    }
    const int64_t prev_r = __shfl_up_sync(0xffffffffu, c.r, 1);
    if (c.valid && (lane == 0 || prev_r != c.r) && m != ~0ull)
      atomicMin(reinterpret_cast<unsigned long long*>(A.out_M + c.r), m);
  }

  // ---- chained hashes: local segmented scan; tile aggregate (final, read by the chain pass) --
  if (K.hashes) {
    uint64_t v = c.valid ? block_digest_words((uint64_t)c.k, (uint32_t)c.nval, t) : 0ull;
    int h = (c.valid && c.k == 0) ? 1 : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t vv = __shfl_up_sync(0xffffffffu, v, d);
      const int hh = __shfl_up_sync(0xffffffffu, h, d);
      if (lane >= d) {
        if (!h) v += vv;
        h |= hh;
      }
    }
    if (c.valid) K.local[c.item] = ((uint64_t)h << 63) | (v & CHAIN_MASK);
    if (lane == 31) K.status[tile] = (h ? ST_INCL : ST_AGG) | (v & CHAIN_MASK);
  }
}

// ---------------------------------------------------------------- chain pass ---------------
template <bool LOOKUP>
__global__ void __launch_bounds__(MATCH_THREADS) match_chain_kernel(MatchKernelArgs K) {
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_items = K.rec[A.n].blk_off;
  if (tile * WT >= n_items) return;
  const int64_t item = tile * WT + lane;
  const bool valid = item < n_items;
  const uint64_t loc = valid ? K.local[item] : 0ull;
  // the first 32 predecessor statuses are read together with the local sums (speculatively:
  // unused when the tile starts with a segment head)
  const int64_t p0 = tile - 1 - lane;
  const uint64_t st0 = p0 >= 0 ? K.status[p0] : ST_INCL;
  const int h = (int)(loc >> 63);
  const uint64_t v = loc & CHAIN_MASK;
  // carry into the tile's first segment: every status is final, walk back 32 tiles per read
  uint64_t prefix = 0;
  if (!__shfl_sync(0xffffffffu, h, 0) && tile > 0) {
    for (int64_t base = tile - 1;; base -= 32) {
      const int64_t p = base - lane;
      const uint64_t st = base == tile - 1 ? st0 : (p >= 0 ? K.status[p] : ST_INCL);
      const unsigned incl = __ballot_sync(0xffffffffu, (st & ~CHAIN_MASK) == ST_INCL);
      const int first = incl ? __ffs(incl) - 1 : 31;
      prefix += warp_sum(lane <= first ? (st & CHAIN_MASK) : 0ull);
      if (incl) break;
    }
  }
  const uint64_t c = chain_finalize(h ? v : prefix + v);
  if (valid && A.out_hash) A.out_hash[item] = c;
  if constexpr (LOOKUP) {  // global table probe, token-verified
    const int64_t tok_total = K.rec[A.n].tok_off;
    const Ctx x = resolve(K, load_win(K, K.tile_r0[tile]), tile, n_items, false);
    int32_t id = -1;
    if (x.valid && x.nval == BT) {
      uint64_t sl = c & K.slot_mask;
      for (;;) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(K.slots + sl));
        const uint64_t key = (uint64_t)raw.x | ((uint64_t)raw.y << 32);
        if (key == c) {
          const int32_t cand = (int32_t)raw.z;
          if (cand >= 0 && K.blk_n[cand] == BT) {
            uint32_t t[BT], q[BT];
            load_block(A.tok, x.start, x.nval, tok_total, t);
            load16_aligned(K.blk_tok + (int64_t)cand * BT, q);
            bool eq = true;
#pragma unroll
            for (int j = 0; j < BT; ++j) eq &= q[j] == t[j];
            if (eq) id = cand;
          }
          break;
        }
        if (key == KEY_EMPTY) break;
        sl = (sl + 1) & K.slot_mask;
      }
    }
    if (x.valid) {
      A.out_block[item] = id;
      if (id < 0)
        atomicMin(reinterpret_cast<unsigned long long*>(A.out_hit + x.r),
                  (unsigned long long)(x.k * BT));
    }
  }
}

int launch_match(sfkv_pool* p, const MatchArgs& a, int64_t* tile_state, cudaStream_t st) {
  if (a.n <= 0) return 0;
  const int64_t ntiles = (a.n_items + WT - 1) / WT;
  const int64_t np = prep_tiles(a.n);
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(tile_state);
  uint64_t* pstatus = reinterpret_cast<uint64_t*>(tile_state + 1);
  uint64_t* status = reinterpret_cast<uint64_t*>(tile_state + 1 + np);
  int64_t* tile_r0 = tile_state + 1 + np + ntiles;
  const int64_t head = (1 + np + 2 * ntiles + 3) & ~int64_t(3);
  ReqRec* rec = reinterpret_cast<ReqRec*>(tile_state + head);
  uint64_t* local = reinterpret_cast<uint64_t*>(tile_state + head + 4 * (a.n + 1));

  SFKV_CUDA(cudaMemsetAsync(tile_state, 0, sizeof(int64_t) * (1 + np), st));
  PrepArgs P;
  P.n = a.n;
  P.tok_off = a.tok_off;
  P.wf = a.out_M ? a.wf : nullptr;
  P.pin_len = p->pin_len;
  P.blk_off = a.blk_off;
  P.rec = rec;
  P.tile_r0 = tile_r0;
  P.out_M = a.out_M;
  P.out_hit = a.out_hit;
  P.ticket = ticket;
  P.pstatus = pstatus;
  match_prep_kernel<<<(unsigned)np, PREP_THREADS, 0, st>>>(P);
  SFKV_LAUNCH_CHECK("match_prep_kernel");
  if (ntiles == 0) return 0;

  MatchKernelArgs K;
  K.a = a;
  K.rec = rec;
  K.pin_tok = p->pin_tok;
  K.blk_tok = p->blk_tok;
  K.blk_n = p->blk_n;
  K.slots = p->slots;
  K.slot_mask = (uint64_t)p->table_slots - 1;
  K.max_pin_blocks = p->cfg.max_pin_blocks;
  K.status = status;
  K.local = local;
  K.tile_r0 = tile_r0;
  K.hashes = (a.out_hash || a.out_block) ? 1 : 0;
  const int64_t grid = (ntiles + MATCH_THREADS / 32 - 1) / (MATCH_THREADS / 32);
  match_block_kernel<<<(unsigned)grid, MATCH_THREADS, 0, st>>>(K);
  SFKV_LAUNCH_CHECK("match_block_kernel");
  if (K.hashes) {
    if (a.out_block) match_chain_kernel<true><<<(unsigned)grid, MATCH_THREADS, 0, st>>>(K);
    else match_chain_kernel<false><<<(unsigned)grid, MATCH_THREADS, 0, st>>>(K);
    SFKV_LAUNCH_CHECK("match_chain_kernel");
  }
  return 0;
}

}  // namespace sfkv

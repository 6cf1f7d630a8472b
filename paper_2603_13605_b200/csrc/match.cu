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
//   digest  = block_digest(k, n, tokens), per block (include/sfkv.h)
//   c_k     = chain_finalize(sum_{i<=k} digest_i mod 2^62)   (chained block hash, segmented scan)
//   lookup  : probe the global table for c_k (full blocks), verify tokens and the parent link (the
//             resident block must descend from the table's block for c_{k-1}), report the block
//             id: a leading run of hits is an exact prefix by induction, whatever the hash does.
//
// Launches (no kernel ever waits on another CTA or warp; consecutive launches overlap their
// prologues with the predecessor's tail through programmatic dependent launch):
//   match_prep_kernel   single-pass request scan (decoupled look-back over 256-request tiles):
//                       blk_off, a 32-B record per request {blk_off, tok_off, len, pin_len, wf}
//                       (the dependent wf -> pin_len load happens once per request), a 32-B tile
//                       record per 32-block tile (the request holding its first block, in
//                       tile-relative coordinates), M / hit initial values.
//   match_block_kernel  one warp per 32-block tile, one block per lane. Lanes resolve their block
//                       from the tile record (one broadcast load) or, for tiles crossing a request
//                       boundary, from the request window (one record per lane + a 5-step
//                       shuffle search). Match mode stages the tile's token range (contiguous in
//                       the CSR batch) into shared memory with one 2D tensor-map TMA load per warp
//                       (rows of 32 ids, 128-B swizzle: conflict-free 16-B reads, no rotation); the pin's blocks of each request
//                       segment (pin-major copy: one extent) arrive by a second bulk copy on the
//                       same mbarrier phase, so nothing is held in registers across the wait. (Lane-per-block
//                       16-B global loads are 64 B apart: 16 lines per warp instruction, which
//                       made L1 the limiter at 81 %.) M: a block whose 16 words all agree with
//                       the pin's has no mismatch; only differing blocks compute the exact first
//                       mismatch, and only the first mismatching lane of each request segment
//                       issues an atomicMin (ballot arithmetic). Hashes: NH digest per block, one
//                       warp inclusive scan, segment correction from the head ballot; each
//                       block's local sum and the tile aggregate are final when written.
//   match_chain_kernel  (hashes / lookup only) one warp per 8 (hash) / 2 (lookup) consecutive
//                       tiles: the carry into the first tile walks back over the predecessors'
//                       final aggregates (32 per read); carries between the warp's own tiles come
//                       from its own loads. Lookup mode probes the table for every full block (the
//                       warp's probes in flight together) and verifies tokens on a key hit.
// Algorithmic bytes per block: 64 B tokens + 64 B pin tokens (blocks inside the pin) + 8 B hash
// out when requested; lookup mode + 16 B table slot (+ 64 B verify on a key hit); + 32 B per
// request. Implementation traffic on top: 8 B written + read per block (local sums) when hashes
// are wanted, + 4 B written + read per block (request id) in lookup mode. HBM-bound integer work:
// no tensor cores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "pool.cuh"

namespace sfkv {

constexpr int WT = 32;                        // items per warp tile
constexpr int MATCH_THREADS = 256;
constexpr int BLOCK_THREADS = 128;  // block pass: 4 warps per CTA, so the per-warp staging fits 10 CTAs/SM
// chain pass tiles per warp: hash-only warps are latency-bound on one look-back, lookup warps
// also carry the table probes
#ifndef SFKV_CH_TPW_HASH
#define SFKV_CH_TPW_HASH 8
#endif
constexpr int CH_TPW_HASH = SFKV_CH_TPW_HASH;
#ifndef SFKV_CH_TPW_LOOKUP
#define SFKV_CH_TPW_LOOKUP 2
#endif
constexpr int CH_TPW_LOOKUP = SFKV_CH_TPW_LOOKUP;  // 54 registers: more warps in flight for the dependent probes
#ifndef SFKV_PREP_THREADS
#define SFKV_PREP_THREADS 256
#endif
constexpr int PREP_THREADS = SFKV_PREP_THREADS;
constexpr int PREP_TILE = PREP_THREADS;

constexpr uint64_t ST_AGG = 1ull << 62;
constexpr uint64_t ST_INCL = 2ull << 62;
constexpr uint32_t RK_FULL = 1u << 31;        // lookup mode: request id | full-block flag



struct __align__(32) ReqRec {
  int64_t blk_off;  // first item of the request
  int64_t tok_off;  // first token
  int32_t len;      // tokens
  int32_t pin_len;  // -1: no pin (or lookup mode)
  int32_t wf;
  int32_t pad;
};

// Per tile (written by the prep kernel): the request holding the tile's first block, in the
// block kernel's tile-relative coordinates (see resolve()). One 32-B broadcast load resolves every
// lane of a tile that lies inside one request (most tiles: requests average ~6 tiles).
struct __align__(32) TileRec {
  int64_t s;    // token start of the tile's first block
  int32_t r;    // its request
  int32_t kb;   // its block index inside the request
  int32_t rem;  // tokens from s to the request's end
  int32_t wf;
  int32_t pl;   // pin length of wf (-1: none / lookup mode)
  int32_t pad;
};

// Scratch layout (int64 units): [prep ticket][prep status x nprep][tile status x ntiles]
// [pad to 4][tile records x ntiles x 4][records x (n+1) x 4][local sums x n_items][rk x n_items/2]
static int64_t prep_tiles(int64_t n) { return (n + PREP_TILE - 1) / PREP_TILE; }
static int64_t tile_head(int64_t np, int64_t ntiles) { return (1 + np + ntiles + 3) & ~int64_t(3); }
size_t match_tile_state_elems(int64_t n_items, int64_t n_requests) {
  const int64_t ntiles = (n_items + WT - 1) / WT;
  const int64_t head = tile_head(prep_tiles(n_requests), ntiles) + 4 * ntiles;
  return (size_t)(head + 4 * (n_requests + 1) + n_items + (n_items + 1) / 2 + 1);
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

__device__ __forceinline__ int32_t clamp32(int64_t v) {
  return (int32_t)(v < -(1ll << 30) ? -(1ll << 30) : (v > (1ll << 30) ? (1ll << 30) : v));
}

// ---------------------------------------------------------------- prep ----------------------
struct PrepArgs {
  int64_t n;
  const int64_t* tok_off;
  const int32_t* wf;  // nullable (lookup)
  const int64_t* pin_len;
  int64_t* blk_off;   // out [n+1]
  ReqRec* rec;        // out [n+1]
  TileRec* trec;      // out
  int64_t* out_M;     // nullable: min(P, pin_len) or 0
  int64_t* out_hit;   // nullable: 16 * blocks
  unsigned long long* ticket;  // null: CTAs are co-resident, blockIdx order
  uint64_t* pstatus;  // prep tile status (epoch-tagged, per-pool buffer)
  uint32_t epoch;
  int32_t max_wf;     // device-side slot guard: out-of-range slots match as unpinned and set
  int* error;         //   the pool's sticky SFKV_EINVAL (reported by sfkv_pool_sync)
};

// Prep look-back status: flag (2 bits) | launch epoch (14 bits) | block count (48 bits). Statuses
// live in a per-pool buffer that nothing else writes, so a status is current iff its epoch is
// this launch's: no memset between launches (the host clears the buffer when the epoch wraps).
constexpr int PE_SHIFT = 48;
constexpr uint64_t PE_SUM = (1ull << PE_SHIFT) - 1;
constexpr uint64_t PE_FLAG = 3ull << 62;

__global__ void __launch_bounds__(PREP_THREADS) match_prep_kernel(PrepArgs P) {
  using BS = cub::BlockScan<int64_t, PREP_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t s_tile, s_prefix;
  pdl_trigger();
  const int tid = threadIdx.x;
  // With every prep CTA co-resident (the usual case) the launch order is the tile order; a
  // ticket (zeroed by the host) orders CTAs otherwise, so a predecessor is always running.
  if (tid == 0) s_tile = P.ticket ? (int64_t)atomicAdd(P.ticket, 1ull) : (int64_t)blockIdx.x;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t r = tile * PREP_TILE + tid;
  const int64_t len = r < P.n ? P.tok_off[r + 1] - P.tok_off[r] : 0;
  int32_t wf = 0;
  int64_t pl = -1;
  if (P.wf && r < P.n) {  // issued before the scan: the dependent pin_len load overlaps it
    wf = P.wf[r];
    if ((uint32_t)wf < (uint32_t)P.max_wf) {
      pl = P.pin_len[wf];
    } else {
      *P.error = SFKV_EINVAL;
      wf = 0;
    }
  }
  const int64_t nb = (len + BT - 1) / BT;
  int64_t excl, total;
  BS(tmp).ExclusiveSum(nb, excl, total);
  if (tid < 32) {  // warp 0: publish, then look back 32 predecessor tiles per read
    const int lane = tid;
    const uint64_t ep = (uint64_t)P.epoch << PE_SHIFT;
    if (lane == 0) st_status(P.pstatus + tile, (tile == 0 ? ST_INCL : ST_AGG) | ep | (uint64_t)total);
    uint64_t prefix = 0;
    for (int64_t base = tile - 1; base >= 0; base -= 32) {
      const int64_t p = base - lane;
      uint64_t s;
      unsigned incl;
      int first;
      for (;;) {  // predecessors run (co-resident, or earlier tickets): plain spin
        s = p >= 0 ? ld_status(P.pstatus + p) : (ST_INCL | ep);
        const bool cur = (s & ~(PE_FLAG | PE_SUM)) == ep && (s & PE_FLAG);
        incl = __ballot_sync(0xffffffffu, cur && (s & PE_FLAG) == ST_INCL);
        first = incl ? __ffs(incl) - 1 : 31;
        const unsigned need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if ((__ballot_sync(0xffffffffu, cur) & need) == need) break;
      }
      prefix += warp_sum(lane <= first ? (s & PE_SUM) : 0ull);
      if (incl) break;
    }
    if (lane == 0) {
      if (tile > 0) st_status(P.pstatus + tile, ST_INCL | ep | (prefix + (uint64_t)total));
      s_prefix = (int64_t)prefix;
    }
  }
  __syncthreads();
  if (r >= P.n) return;
  const int64_t b = s_prefix + excl;
  ReqRec q;
  q.blk_off = b;
  q.tok_off = P.tok_off[r];
  q.len = (int32_t)len;
  q.pin_len = (int32_t)pl;
  q.wf = wf;
  q.pad = 0;
  P.rec[r] = q;
  P.blk_off[r] = b;
  for (int64_t t = (b + WT - 1) / WT; t * WT < b + nb; ++t) {
    TileRec tr;
    tr.kb = (int32_t)(t * WT - b);
    tr.s = q.tok_off + (int64_t)tr.kb * BT;
    tr.r = (int32_t)r;
    tr.rem = (int32_t)(len - (int64_t)tr.kb * BT);
    tr.wf = wf;
    tr.pl = (int32_t)pl;
    tr.pad = 0;
    P.trec[t] = tr;
  }
  if (P.out_M) P.out_M[r] = pl < 0 ? 0 : (len < pl ? len : pl);
  if (P.out_hit) P.out_hit[r] = nb * BT;
  if (r == P.n - 1) {  // closing record
    ReqRec e;
    e.blk_off = b + nb;
    e.tok_off = P.tok_off[P.n];
    e.len = 0;
    e.pin_len = -1;
    e.wf = 0;
    e.pad = 0;
    P.rec[P.n] = e;
    P.blk_off[P.n] = b + nb;
  }
}

// ---------------------------------------------------------------- per-block pass -----------
struct MatchKernelArgs {
  MatchArgs a;
  const ReqRec* rec;
  const uint32_t* pin_tok;
  const uint32_t* blk_tok;
  const int32_t* blk_parent;
  const uint8_t* blk_n;
  const Slot* slots;
  uint64_t slot_mask;
  int64_t pin_groups;
  uint64_t* status;  // per tile: flag | aggregate since the tile's last segment head (final)
  uint64_t* local;   // per block: bit 63 = a segment head at or before it in the tile | local sum
  uint32_t* rk;      // lookup mode: per block request id | RK_FULL
  const TileRec* trec;
  int hashes;        // chained hashes (or lookup) requested
  int64_t tok_rows;  // full 32-id rows of the token buffer (the tensor map's height)
};

struct Ctx {  // one lane's block of one tile
  int64_t r, start;
  int32_t k, nval, pin_len, wf;
  bool valid;
};

__device__ __forceinline__ void unpack_rec(const ReqRec* q, int64_t& blk_off, int64_t& tok_off,
                                           int32_t& len, int32_t& pl, int32_t& wf) {
  const int4* p = reinterpret_cast<const int4*>(q);
  const int4 a = __ldg(p), b = __ldg(p + 1);
  blk_off = (int64_t)(((uint64_t)(uint32_t)a.y << 32) | (uint32_t)a.x);
  tok_off = (int64_t)(((uint64_t)(uint32_t)a.w << 32) | (uint32_t)a.z);
  len = b.x;
  pl = b.y;
  wf = b.z;
}

// Lane L of tile `tile` resolves item tile*32 + L. The tile record gives the request r0 holding
// the tile's first block as (s0, kb0, rem0): when r0 covers the whole tile (rem0 > 16*31) every
// lane resolves from that one broadcast load: k = kb0 + L, start = s0 + 16 L,
// nval = clamp(rem0 - 16 L, 0, 16). Otherwise the window (requests r0 .. r0+31) is one record per
// lane, reduced to the same tile-relative coordinates before the shuffles:
//   kb_j  = tile*32 - blk_off_j   (block index of the tile's first item inside request j)
//   s_j   = tok_off_j + 16 kb_j   (token start of that block)
//   rem_j = len_j - 16 kb_j       (tokens from there to the request's end)
// and lane L belongs to the largest j with kb_j >= -L. Tiles covering > 32 requests (empty
// requests) fall back to a binary search over blk_off for the lanes past the window.
__device__ __forceinline__ Ctx resolve(const MatchKernelArgs& K, int64_t tile, int64_t n_items) {
  const int lane = threadIdx.x & 31;
  const int64_t n = K.a.n;
  const int64_t T0 = tile * WT;
  const int4* tp = reinterpret_cast<const int4*>(K.trec + tile);
  const int4 ta = __ldg(tp), tb = __ldg(tp + 1);
  const int64_t s0 = (int64_t)(((uint64_t)(uint32_t)ta.y << 32) | (uint32_t)ta.x);
  const int64_t r0 = ta.z;
  Ctx c;
  const int64_t item = T0 + lane;
  c.valid = item < n_items;
  if (tb.x > (WT - 1) * BT) {  // the whole tile lies inside request r0
    c.r = r0;
    c.k = ta.w + lane;
    c.start = s0 + (int64_t)lane * BT;
    c.wf = tb.y;
    c.pin_len = tb.z;
    const int32_t nv = tb.x - lane * BT;
    c.nval = c.valid ? (nv > BT ? BT : nv) : 0;
    return c;
  }
  const int64_t rr = r0 + lane;
  int32_t kb = -(1 << 30), rem = 0, pl = -1, wf = 0;
  int64_t s = 0;
  if (rr <= n) {
    int64_t bo, to;
    int32_t len;
    unpack_rec(K.rec + rr, bo, to, len, pl, wf);
    kb = clamp32(T0 - bo);
    s = to + (int64_t)kb * BT;
    rem = clamp32((int64_t)len - (int64_t)kb * BT);
  }
  const int64_t off32 = r0 + WT <= n ? __ldg(&K.rec[r0 + WT].blk_off) : INT64_MAX;
  int j = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1) {
    const int32_t v = __shfl_sync(0xffffffffu, kb, j + st);
    if (v >= -lane) j += st;
  }
  const int32_t kbj = __shfl_sync(0xffffffffu, kb, j);
  const int32_t remj = __shfl_sync(0xffffffffu, rem, j);
  c.start = __shfl_sync(0xffffffffu, s, j) + (int64_t)lane * BT;
  c.pin_len = __shfl_sync(0xffffffffu, pl, j);
  c.wf = __shfl_sync(0xffffffffu, wf, j);
  c.k = kbj + lane;
  c.r = r0 + j;
  int32_t nv = remj - lane * BT;
  if (c.valid && off32 <= item) {  // > 32 requests in this tile
    c.r = upper_index(K.a.blk_off, n, item);
    int64_t bo, to;
    int32_t len;
    unpack_rec(K.rec + c.r, bo, to, len, c.pin_len, c.wf);
    c.k = (int32_t)(item - bo);
    c.start = to + (int64_t)c.k * BT;
    nv = len - c.k * BT;
  }
  c.nval = c.valid ? (nv < 0 ? 0 : (nv > BT ? BT : nv)) : 0;
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

// Block tokens [start, start+nval) zero-padded to 16: five 16-B loads from the aligned-down
// address and a branch-free two-stage funnel by (start & 3) (lanes of different requests have
// different alignments, so a switch would diverge); scalar only at the array end.
__device__ __forceinline__ void load_block(const uint32_t* __restrict__ tok, int64_t start, int nval,
                                           int64_t tok_total, uint32_t* t) {
  const int64_t a0 = start & ~int64_t(3);
  const int sh = (int)(start & 3);
  if (a0 + 20 <= tok_total) {
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
    uint32_t u[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) u[i] = (sh & 2) ? w[i + 2] : w[i];
#pragma unroll
    for (int i = 0; i < BT; ++i) t[i] = (sh & 1) ? u[i + 1] : u[i];
  } else {
#pragma unroll
    for (int j = 0; j < BT; ++j) t[j] = j < nval ? __ldg(tok + start + j) : 0u;
  }
  if (nval < BT) {
#pragma unroll
    for (int j = 0; j < BT; ++j)
      if (j >= nval) t[j] = 0u;
  }
}

// ---- TMA staging (tokens: a 2D tensor-map box with the 128-B swizzle; pins: bulk copies) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITP_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITP_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Pin block of a lane staged at lane * PIN_STRIDE words. Default (SFKV_PIN_PAD 0, SFKV_PIN_ROT 1):
// the pin copy is unpadded (64 B per block, no HBM bytes beyond the tokens) and each lane reads its
// four 16-B chunks in an order rotated by (lane >> 1) & 3, so the 8 lanes of a quarter-warp hit 8
// distinct bank groups; two select stages undo the rotation. Measured on the C2 step (B200, 3
// interleaved rounds): padded 80-B stride 74.5 us (M only 63.5), unpadded with 4-way conflicts
// 74.2 (60.9), unpadded rotated 72.7 (60.1): the 16 B/block the padding cost in HBM outweigh the
// selects.
#ifndef SFKV_PIN_ROT
#define SFKV_PIN_ROT 1
#endif
__device__ __forceinline__ void load_pin_staged(const uint32_t* s, uint32_t* q) {
  const int lane = threadIdx.x & 31;
#if SFKV_PIN_PAD
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint4 w = *reinterpret_cast<const uint4*>(s + lane * PIN_STRIDE + 4 * x);
    q[4 * x] = w.x;
    q[4 * x + 1] = w.y;
    q[4 * x + 2] = w.z;
    q[4 * x + 3] = w.w;
  }
#elif !SFKV_PIN_ROT
  // unpadded 64-B stride, plain reads: lanes 2 apart share a bank group (4-way conflicts)
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint4 w = *reinterpret_cast<const uint4*>(s + lane * BT + 4 * x);
    q[4 * x] = w.x;
    q[4 * x + 1] = w.y;
    q[4 * x + 2] = w.z;
    q[4 * x + 3] = w.w;
  }
#else
  const int rr = (lane >> 1) & 3;
  uint4 v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = *reinterpret_cast<const uint4*>(s + lane * BT + 4 * ((i + rr) & 3));
  uint4 u[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) u[x] = (rr & 1) ? v[(x + 3) & 3] : v[x];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint4 w = (rr & 2) ? u[(x + 2) & 3] : u[x];
    q[4 * x] = w.x;
    q[4 * x + 1] = w.y;
    q[4 * x + 2] = w.z;
    q[4 * x + 3] = w.w;
  }
#endif
}

// Tensor-map staging of the token range: the token buffer viewed as rows of 32 ids (128 B); a
// tile's range is TMAP_ROWS rows from the row holding its first token, loaded with the 128-B
// swizzle (16-B chunk c of row r lands at chunk c ^ (r & 7)), so the lanes of a quarter-warp —
// whose blocks are 4 chunks apart — read distinct bank groups with no per-lane rotation to undo.
constexpr int TMAP_ROWS = 18;  // >= (3 + 31*16 + 20 + 31) / 32 rows
__device__ __forceinline__ void bulk_tensor_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// Block tokens of a lane whose block starts at word o of a swizzled staged range.
__device__ __forceinline__ void load_block_swz(const uint32_t* s, int o, int nval, uint32_t* t) {
  const int c0 = o >> 2, sh = o & 3;
  uint32_t w[20];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int g = c0 + i;
    const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(s) + ((g ^ ((g >> 3) & 7)) << 4));
    w[4 * i] = v.x;
    w[4 * i + 1] = v.y;
    w[4 * i + 2] = v.z;
    w[4 * i + 3] = v.w;
  }
  uint32_t y[17];
#pragma unroll
  for (int i = 0; i < 17; ++i) y[i] = (sh & 2) ? w[i + 2] : w[i];
#pragma unroll
  for (int i = 0; i < BT; ++i) t[i] = (sh & 1) ? y[i + 1] : y[i];
  if (nval < BT) {
#pragma unroll
    for (int j = 0; j < BT; ++j)
      if (j >= nval) t[j] = 0u;
  }
}


// M and chained-hash work of one tile once every lane holds its block's tokens t (zero padded)
// and, for blocks inside the pin, the pin's block q.
__device__ __forceinline__ void tile_finish(const MatchKernelArgs& K, int64_t tile, const Ctx& c,
                                            bool in_pin, const uint32_t* t, const uint32_t* q) {
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const bool match_mode = A.out_M != nullptr;
  const unsigned below = (1u << lane) - 1u;
  // request heads (first block of a request) and segment starts (heads, lane 0, invalid lanes)
  const unsigned heads = __ballot_sync(0xffffffffu, c.valid && c.k == 0);
  const unsigned segs = heads | 1u | __ballot_sync(0xffffffffu, !c.valid);
  const int seg0 = 31 - __clz(segs & (below | (1u << lane)));

  // ---- M: first differing token against the pin's block; the first mismatching lane of each
  //      request segment issues the only atomic --------------------------------------------
  if (match_mode) {
    int lcp = BT, lim = 0;
    if (in_pin) {
      // both sides are zero padded past their ends, so a block whose 16 words all agree has no
      // mismatch below lim; only a differing block (the first diverging block of a request, or a
      // boundary block whose padding differs) takes the exact first-mismatch path
      uint32_t d = 0;
#pragma unroll
      for (int j = 0; j < BT; ++j) d |= q[j] ^ t[j];
      if (d) {
        const int pn = min(c.pin_len - c.k * BT, BT);
        lim = min(c.nval, pn);
        unsigned ne = 1u << lim;
#pragma unroll
        for (int j = 0; j < BT; ++j) ne |= (q[j] != t[j]) ? (1u << j) : 0u;
        lcp = __ffs(ne) - 1;
      }
    }
    const bool mism = in_pin && lcp < lim;
    const unsigned mm = __ballot_sync(0xffffffffu, mism);
    if (mism && (mm & below & ~((1u << seg0) - 1u)) == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(A.out_M + c.r),
                (unsigned long long)((int64_t)c.k * BT + lcp));
  }

  // ---- chained hashes: warp inclusive scan of digests, corrected to segment-local sums; the
  //      tile aggregate is final (read by the chain pass) ------------------------------------
  if (K.hashes) {
    uint64_t v = c.valid ? block_digest_words((uint64_t)c.k, (uint32_t)c.nval, t) : 0ull;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += u;
    }
    const unsigned hl = heads & (below | (1u << lane));
    const int hs = 31 - __clz(hl | 1u);  // last real head at or before this lane (if any)
    const uint64_t base = __shfl_sync(0xffffffffu, v, hs > 0 ? hs - 1 : 0);
    const uint64_t h = hl ? 1ull : 0ull;
    if (hl && hs > 0) v -= base;
    const int64_t item = tile * WT + lane;
    if (c.valid) {
      K.local[item] = (h << 63) | (v & CHAIN_MASK);
      if (K.rk) K.rk[item] = (uint32_t)c.r | (c.nval == BT ? RK_FULL : 0u);
    }
    if (lane == 31) K.status[tile] = (h ? ST_INCL : ST_AGG) | (v & CHAIN_MASK);
  }
}


// One warp per 32-block tile, one block per lane, non-persistent: enough tiles in flight per SM to
// cover the window -> tokens/pin-tokens round trips.
// 5 CTAs (40 warps) per SM: the register cap (48) trades a few spilled bytes for occupancy.
template <bool STAGED>
__global__ void __launch_bounds__(BLOCK_THREADS, 10) match_block_kernel(MatchKernelArgs K,
                                                                       const __grid_constant__ CUtensorMap tmap) {
  __shared__ __align__(1024) uint32_t s_tok[STAGED ? BLOCK_THREADS / 32 : 1][STAGED ? 768 : 4];  // 18 rows, 1 KB-aligned
  __shared__ __align__(128) uint32_t s_pin[STAGED ? BLOCK_THREADS / 32 : 1][STAGED ? WT * PIN_STRIDE : 4];
  __shared__ __align__(8) uint64_t s_bar[BLOCK_THREADS / 32];
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  [[maybe_unused]] const int warp = threadIdx.x >> 5;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if constexpr (STAGED) {
    if (lane == 0) mbar_init(&s_bar[warp]);
    __syncwarp();
  }
  pdl_trigger();
  pdl_wait();
  const int64_t n_items = K.rec[A.n].blk_off;
  if (tile * WT >= n_items) return;
  const int64_t tok_total = K.rec[A.n].tok_off;
  const bool match_mode = A.out_M != nullptr;
  const Ctx c = resolve(K, tile, n_items);

  const bool in_pin = match_mode && c.valid && c.pin_len >= 0 && c.k < (c.pin_len + BT - 1) / BT;
  uint32_t q[BT];
  uint32_t t[BT];
  if constexpr (STAGED) {
    // one mbarrier phase for the tile: its token range (one bulk copy) and, per request segment
    // of in-pin blocks, that segment's pin blocks (pin-major: one extent, placed at lane * 64 B)
    const int nv = __popc(__ballot_sync(0xffffffffu, c.valid));
    const int64_t row0 = __shfl_sync(0xffffffffu, c.start, 0) >> 5;
    const int64_t a0 = row0 << 5;
    const int64_t a1 = __shfl_sync(0xffffffffu, (c.start & ~int64_t(3)) + 20, nv - 1);
    const bool staged = a1 <= K.tok_rows * 32;  // all but the tiles touching the last partial row
    const unsigned pin_m = __ballot_sync(0xffffffffu, in_pin);
    const int64_t prev_r = __shfl_up_sync(0xffffffffu, c.r, 1);
    const bool head = in_pin && (lane == 0 || !((pin_m >> (lane - 1)) & 1u) || prev_r != c.r);
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    uint32_t pin_bytes = 0;
    if (head) {
      const unsigned after = ~((2u << lane) - 1u);
      const unsigned stop = (heads | ~pin_m) & after;
      const int end = stop ? __ffs(stop) - 1 : 32;
      pin_bytes = (uint32_t)(end - lane) * (PIN_STRIDE * 4);
    }
    const uint32_t tok_bytes = staged ? (uint32_t)(TMAP_ROWS * 128) : 0u;
    const uint32_t total = __reduce_add_sync(0xffffffffu, pin_bytes) + tok_bytes;
    if (total) {
      if (lane == 0) mbar_expect_tx(&s_bar[warp], total);
      __syncwarp();
      if (staged && lane == 0) bulk_tensor_2d(s_tok[warp], &tmap, 0, (int)row0, &s_bar[warp]);
      if (head) bulk_copy(s_pin[warp] + lane * PIN_STRIDE, K.pin_tok + pin_tok_index(c.wf, c.k, 0, K.pin_groups),
                          pin_bytes, &s_bar[warp]);
      mbar_wait0(&s_bar[warp]);
    }
    if (c.valid) {
      if (staged) load_block_swz(s_tok[warp], (int)(c.start - a0), c.nval, t);
      else load_block(A.tok, c.start, c.nval, tok_total, t);
    }
    if (in_pin) load_pin_staged(s_pin[warp], q);
  } else if (c.valid) {
    load_block(A.tok, c.start, c.nval, tok_total, t);
  }
  if (!c.valid) {
#pragma unroll
    for (int j = 0; j < BT; ++j) t[j] = 0u;
  }
  tile_finish(K, tile, c, in_pin, t, q);
}

// ---------------------------------------------------------------- chain pass ---------------
template <bool LOOKUP>
__global__ void __launch_bounds__(MATCH_THREADS) match_chain_kernel(MatchKernelArgs K) {
  constexpr int CH_TPW = LOOKUP ? CH_TPW_LOOKUP : CH_TPW_HASH;
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  const int64_t t0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * CH_TPW;
  pdl_trigger();
  pdl_wait();
  const int64_t n_items = K.rec[A.n].blk_off;
  if (t0 * WT >= n_items) return;
  uint64_t loc[CH_TPW];
  uint32_t rk[CH_TPW];
#pragma unroll
  for (int i = 0; i < CH_TPW; ++i) {
    const int64_t item = (t0 + i) * WT + lane;
    loc[i] = item < n_items ? K.local[item] : 0ull;
    if constexpr (LOOKUP) rk[i] = item < n_items ? K.rk[item] : 0u;
  }
  // the first 32 predecessor statuses are read together with the local sums (speculatively:
  // unused when the first tile starts with a segment head)
  const int64_t p0 = t0 - 1 - lane;
  const uint64_t st0 = p0 >= 0 ? K.status[p0] : ST_INCL;
  // carry into the first tile's first segment: every status is final, walk back 32 tiles per read
  uint64_t carry = 0;
  if (!__shfl_sync(0xffffffffu, (uint32_t)(loc[0] >> 63), 0) && t0 > 0) {
    for (int64_t base = t0 - 1;; base -= 32) {
      const int64_t p = base - lane;
      const uint64_t st = base == t0 - 1 ? st0 : (p >= 0 ? K.status[p] : ST_INCL);
      const unsigned incl = __ballot_sync(0xffffffffu, (st & ~CHAIN_MASK) == ST_INCL);
      const int first = incl ? __ffs(incl) - 1 : 31;
      carry += warp_sum(lane <= first ? (st & CHAIN_MASK) : 0ull);
      if (incl) break;
    }
  }
  [[maybe_unused]] const uint64_t carry0 = carry;  // sum through the item before the warp's first
  uint64_t c[CH_TPW];
#pragma unroll
  for (int i = 0; i < CH_TPW; ++i) {
    const bool h = loc[i] >> 63;
    const uint64_t sum = h ? (loc[i] & CHAIN_MASK) : carry + (loc[i] & CHAIN_MASK);
    carry = __shfl_sync(0xffffffffu, sum, 31);
    c[i] = chain_finalize(sum);
    const int64_t item = (t0 + i) * WT + lane;
    if (item < n_items && A.out_hash) A.out_hash[item] = c[i];
  }
  if constexpr (LOOKUP) {  // global table probe, token-verified and parent-linked; probes in flight together
    const int64_t tok_total = K.rec[A.n].tok_off;
    const int64_t item0 = t0 * WT;
    uint4 raw[CH_TPW];
#pragma unroll
    for (int i = 0; i < CH_TPW; ++i) {
      const int64_t item = (t0 + i) * WT + lane;
      raw[i] = make_uint4(0, 0, 0xffffffffu, 0);
      if (item < n_items && (rk[i] & RK_FULL))
        raw[i] = __ldg(reinterpret_cast<const uint4*>(K.slots + (c[i] & K.slot_mask)));
    }
    // the block the table holds for the previous chained key, for the warp's first item: its
    // request (rk of the previous item) and, inside a request, a probe of fin(carry)
    uint32_t prev_rk = 0xffffffffu;
    int32_t prev_raw = -1;
    if (lane == 0 && item0 > 0) {
      prev_rk = __ldg(&K.rk[item0 - 1]);
      if ((prev_rk & ~RK_FULL) == (rk[0] & ~RK_FULL) && (prev_rk & RK_FULL)) {
        const uint64_t cp = chain_finalize(carry0);
        uint64_t sl = cp & K.slot_mask;
        for (;;) {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(K.slots + sl));
          const uint64_t key = (uint64_t)w.x | ((uint64_t)w.y << 32);
          if (key == cp) {
            prev_raw = (int32_t)w.z;
            break;
          }
          if (key == KEY_EMPTY) break;
          sl = (sl + 1) & K.slot_mask;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH_TPW; ++i) {
      const int64_t item = (t0 + i) * WT + lane;
      const bool valid = item < n_items;
      const int64_t r = (int64_t)(rk[i] & ~RK_FULL);
      int32_t cand = -1;  // the table's block for this key (no token check)
      bool eq = false;
      if (valid && (rk[i] & RK_FULL)) {
        uint64_t sl = c[i] & K.slot_mask;
        uint4 w = raw[i];
        for (;;) {
          const uint64_t key = (uint64_t)w.x | ((uint64_t)w.y << 32);
          if (key == c[i]) {
            cand = (int32_t)w.z;
            if (cand >= 0) {  // only full blocks are ever published; a pending claim reads -1
              int64_t bo, to;
              int32_t len, pl, wf;
              unpack_rec(K.rec + r, bo, to, len, pl, wf);
              uint32_t t[BT], q[BT];
              load_block(A.tok, to + (item - bo) * BT, BT, tok_total, t);
              load16_aligned(K.blk_tok + (int64_t)cand * BT, q);
              eq = true;
#pragma unroll
              for (int j = 0; j < BT; ++j) eq &= q[j] == t[j];
            }
            break;
          }
          if (key == KEY_EMPTY) break;
          sl = (sl + 1) & K.slot_mask;
          w = __ldg(reinterpret_cast<const uint4*>(K.slots + sl));
        }
      }
      // predecessor item: the lane below, the previous tile's last lane, or the warp's carry-in
      const uint32_t up_rk = __shfl_up_sync(0xffffffffu, rk[i], 1);
      const int32_t up_raw = __shfl_up_sync(0xffffffffu, cand, 1);
      const uint32_t p_rk = lane > 0 ? up_rk : prev_rk;
      const int32_t p_raw = lane > 0 ? up_raw : prev_raw;
      const bool head = (p_rk & ~RK_FULL) != (uint32_t)r || item == 0;
      int32_t id = -1;
      if (eq && (head || __ldg(&K.blk_parent[cand]) == p_raw)) id = cand;
      prev_rk = __shfl_sync(0xffffffffu, rk[i], 31);
      prev_raw = __shfl_sync(0xffffffffu, cand, 31);
      if (valid) A.out_block[item] = id;
      // leading hit length: the first miss of each request segment in the tile lowers out_hit
      const uint32_t prev = __shfl_up_sync(0xffffffffu, rk[i] & ~RK_FULL, 1);
      const unsigned segs = __ballot_sync(0xffffffffu, lane == 0 || !valid || prev != (uint32_t)r);
      const unsigned below = (1u << lane) - 1u;
      const int seg0 = 31 - __clz(segs & (below | (1u << lane)));
      const bool miss = valid && id < 0;
      const unsigned mm = __ballot_sync(0xffffffffu, miss);
      if (miss && (mm & below & ~((1u << seg0) - 1u)) == 0) {
        const int64_t bo = __ldg(&K.rec[r].blk_off);
        atomicMin(reinterpret_cast<unsigned long long*>(A.out_hit + r),
                  (unsigned long long)((item - bo) * BT));
      }
    }
  }
}

// ---------------------------------------------------------------- per-request lookup --------
// Lookup batches of many requests of moderate length (C5: 100k prefixes of 65-127 blocks) take a
// one-pass path: one warp per request walks its blocks 32 at a time with the running chain sum in
// a register. Each tile's tokens are staged once (2D tensor-map TMA, double-buffered: the next
// tile's load is in flight while this one is processed), and the probe, the token verify against
// the resident block and the parent check run while the block's tokens are still in registers —
// no chain pass, no per-block local sums / request ids in HBM, no second read of the request's
// tokens (the two-pass lookup re-read them for the verify: ~1.64x the algorithmic traffic).
// Output identical to the two-pass path (and sfo_lookup_batch): out_block per block, out_hit.
constexpr int LR_THREADS = 128;
#ifndef SFKV_LR_MINB
#define SFKV_LR_MINB 1
#endif
constexpr int LR_MIN_REQUESTS = 2048;  // below: too few warps to fill the GPU one request each
constexpr int64_t LR_MAX_AVG_BLOCKS = 1024;  // above: one warp per request serialises too much

__global__ void __launch_bounds__(LR_THREADS, SFKV_LR_MINB) lookup_req_kernel(MatchKernelArgs K,
                                                               const __grid_constant__ CUtensorMap tmap) {
  __shared__ __align__(1024) uint32_t s_tok[LR_THREADS / 32][2][768];  // 18 rows each, 1 KB aligned
  __shared__ __align__(8) uint64_t s_bar[LR_THREADS / 32][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (lane == 0) {
    mbar_init(&s_bar[warp][0]);
    mbar_init(&s_bar[warp][1]);
  }
  __syncwarp();
  pdl_trigger();
  pdl_wait();
  const MatchArgs& A = K.a;
  if (r >= A.n) return;
  int64_t bo, to;
  int32_t len, pl, wf;
  unpack_rec(K.rec + r, bo, to, len, pl, wf);
  const int64_t nb = (len + BT - 1) / BT, nfull = len / BT;
  const int64_t tok_total = K.rec[A.n].tok_off;
  const int64_t ntile = (nb + WT - 1) / WT;
  const int64_t tok_limit = K.tok_rows * 32;
  // staging of tile i into buffer i & 1 (uniform across the warp); false: read from global
  auto issue = [&](int64_t i) -> bool {
    const int64_t k0 = i * WT, kl = min(nb - 1, k0 + WT - 1);
    const int64_t s0 = to + k0 * BT, sl = to + kl * BT;
    const bool staged = ((sl & ~int64_t(3)) + 20) <= tok_limit;
    if (staged && lane == 0) {
      uint64_t* bar = &s_bar[warp][i & 1];
      fence_proxy_async_smem();  // the warp's generic reads of this buffer precede the refill
      mbar_expect_tx(bar, TMAP_ROWS * 128);
      bulk_tensor_2d(s_tok[warp][i & 1], &tmap, 0, (int)(s0 >> 5), bar);
    }
    return staged;
  };
  bool staged = ntile > 0 ? issue(0) : false;
  uint64_t carry = 0;
  int32_t prev_raw = -1;
  bool run = true;
  int64_t lead = 0;
  for (int64_t i = 0; i < ntile; ++i) {
    const bool staged_next = i + 1 < ntile ? issue(i + 1) : false;
    const int64_t k = i * WT + lane;
    const bool valid = k < nb;
    const int64_t start = to + k * BT;
    const int nval = valid ? (int)min((int64_t)BT, (int64_t)len - k * BT) : 0;
    uint32_t t[BT];
    if (staged) {
      mbar_wait(&s_bar[warp][i & 1], (uint32_t)((i >> 1) & 1));
      if (valid) load_block_swz(s_tok[warp][i & 1], (int)(start - (((to + i * WT * BT) >> 5) << 5)), nval, t);
    } else if (valid) {
      load_block(A.tok, start, nval, tok_total, t);
    }
    if (!valid) {
#pragma unroll
      for (int j = 0; j < BT; ++j) t[j] = 0u;
    }
    __syncwarp();
    // chained key: warp inclusive scan of the digests on top of the request's running sum
    uint64_t v = valid ? block_digest_words((uint64_t)k, (uint32_t)nval, t) : 0ull;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += u;
    }
    v += carry;
    carry = __shfl_sync(0xffffffffu, v, 31);
    const uint64_t c = chain_finalize(v);
    // probe (full blocks only; a pending claim reads -1), then verify + parent together
    int32_t raw = -1;
    if (valid && k < nfull) {
      uint64_t sl = c & K.slot_mask;
      for (;;) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(K.slots + sl));
        const uint64_t key = (uint64_t)w.x | ((uint64_t)w.y << 32);
        if (key == c) {
          raw = (int32_t)w.z;
          break;
        }
        if (key == KEY_EMPTY) break;
        sl = (sl + 1) & K.slot_mask;
      }
    }
    bool eq = false;
    int32_t par = -1;
    if (raw >= 0) {
      uint32_t q[BT];
      load16_aligned(K.blk_tok + (int64_t)raw * BT, q);
      par = __ldg(&K.blk_parent[raw]);
      eq = true;
#pragma unroll
      for (int j = 0; j < BT; ++j) eq &= q[j] == t[j];
    }
    const int32_t up_raw = __shfl_up_sync(0xffffffffu, raw, 1);
    const int32_t p_raw = lane > 0 ? up_raw : prev_raw;
    const int32_t id = (eq && (k == 0 || par == p_raw)) ? raw : -1;
    prev_raw = __shfl_sync(0xffffffffu, raw, 31);
    if (valid) A.out_block[bo + k] = id;
    const unsigned miss = __ballot_sync(0xffffffffu, valid && id < 0);
    if (run) {
      if (miss) {
        lead += __ffs(miss) - 1;
        run = false;
      } else {
        lead += min((int64_t)WT, nb - i * WT);
      }
    }
    staged = staged_next;
  }
  if (lane == 0) A.out_hit[r] = lead * BT;
}

// ---------------------------------------------------------------- span pass (match mode) ----
// One launch per match batch: no prep scan, no chain pass, no per-block sums in HBM.
// CTA c (ticket order: every lower-numbered span has started) owns the blocks whose FIRST token
// lies in the token span [c*SPAN, (c+1)*SPAN) of the CSR batch: the tail of the request that crosses
// c*SPAN (the carry-in request) and every request whose first token lies in the span (found by a
// 32-ary search of tok_off). Only two facts about earlier spans are needed, both by decoupled
// look-back over per-span statuses:
//   * the flat index of the span's first block (blk_off): every span publishes its block count as
//     soon as its request table is built, so this look-back resolves while the first tiles load;
//   * the carry-in request's chain sum and first mismatch before the span: published when a
//     predecessor has hashed its blocks; only the carry-in blocks wait for it, at the very end.
// Inside the span, warps take 32-block tiles (one block per lane; a tile may cross requests): the
// tile's token range is staged by one 2D tensor-map TMA load (128-B swizzle) and the pin blocks of
// each in-pin request segment by bulk copies, double-buffered per warp. A tile whose lanes share one
// token alignment (every tile inside one request) reads its blocks with a warp-uniform
// specialisation (no per-lane funnel selects); pins are stored pre-rotated (pin_rot) so their reads
// are conflict-free with no selects either. Block digests go to shared memory and one segmented
// CTA scan turns them into chained sums; M mismatches are shared-memory atomic minima per request.
// Statuses are self-validating 64-bit words (kind | value; 0 = unpublished) in one of two buffers
// that alternate between launches: CTA c clears slot c of the other buffer, so a launch needs no
// memset and no memory fence.
#ifndef SFKV_SPAN_TOKENS
#define SFKV_SPAN_TOKENS 16384
#endif
#ifndef SFKV_SP_WARPS
#define SFKV_SP_WARPS 8
#endif
#ifndef SFKV_SP_MINB
#define SFKV_SP_MINB 2
#endif
constexpr int SPAN = SFKV_SPAN_TOKENS;
constexpr int SP_WARPS = SFKV_SP_WARPS;
constexpr int SP_THREADS = SP_WARPS * 32;
constexpr int SP_RREQ = SP_THREADS;                 // table entries per round (one thread each)
constexpr int SP_RBLK = SPAN / BT + SP_RREQ;        // blocks of one round: <= SPAN/16 + entries
constexpr int SP_IPT = (SP_RBLK + SP_THREADS - 1) / SP_THREADS;
constexpr int SP_CARRY = SPAN / BT;                 // carry-in blocks of one span
constexpr int SP_TOKB = TMAP_ROWS * 128;            // staged token box (1 KB aligned)
constexpr int SP_BUF = ((SP_TOKB + WT * 64) + 1023) & ~1023;
constexpr size_t SP_DYN = (size_t)SP_WARPS * 2 * SP_BUF + 1024;  // + base alignment slack
constexpr uint64_t SP_KIND = 3ull << 62;
constexpr uint64_t SP_AGG = 1ull << 62;    // chain: the span's own sum (no request head in it)
constexpr uint64_t SP_INCL = 2ull << 62;   // chain: sum since the trailing request's head (in span)
constexpr uint64_t SP_INCLD = 3ull << 62;  // chain: no head in span, prefix resolved by look-back
constexpr uint64_t SP_MVALID = 1ull << 63; // mismatch word: valid | u32 first mismatch of the
                                           // span's trailing request inside the span

struct SpanState {
  unsigned long long* ticket;  // grows by the grid size every launch (never reset)
  unsigned long long base;
  uint64_t *blk, *chain, *mism;        // this launch: kind | count, kind | sum, valid | position
  uint64_t *blk_o, *chain_o, *mism_o;  // the other launch parity: slot c cleared by CTA c
  const int64_t* pin_len;
  int max_wf;
  int* error;
};

__device__ __forceinline__ uint64_t ld_status_spin(const uint64_t* p) {
  uint64_t v;
  do {
    v = ld_status(p);
  } while (!v);
  return v;
}

// Block tokens of a lane whose block starts at word o (o & 3 == SH) of a swizzled staged range.
template <int SH>
__device__ __forceinline__ void load_swz_sh(const uint32_t* s, int o, uint32_t* t) {
  const int c0 = o >> 2;
  constexpr int NC = SH ? 5 : 4;
  uint32_t w[20];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int g = c0 + i;
    const uint4 v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(s) + ((g ^ ((g >> 3) & 7)) << 4));
    w[4 * i] = v.x;
    w[4 * i + 1] = v.y;
    w[4 * i + 2] = v.z;
    w[4 * i + 3] = v.w;
  }
#pragma unroll
  for (int j = 0; j < BT; ++j) t[j] = w[j + SH];
}

// Pin block k of a lane, staged at lane * 64 B in the rotated layout: in-order, conflict-free.
__device__ __forceinline__ void load_pin_rot(const uint32_t* s, int lane, int64_t k, uint32_t* q) {
  const int rot = pin_rot(k);
  const uint32_t* b = s + lane * BT;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint4 w = *reinterpret_cast<const uint4*>(b + 4 * ((x + rot) & 3));
    q[4 * x] = w.x;
    q[4 * x + 1] = w.y;
    q[4 * x + 2] = w.z;
    q[4 * x + 3] = w.w;
  }
}

struct SpTable {  // one round's entries (shared memory)
  int64_t to[SP_RREQ];
  int32_t r[SP_RREQ], len[SP_RREQ], k0[SP_RREQ], sb[SP_RREQ + 1], wf[SP_RREQ], pl[SP_RREQ], mn[SP_RREQ];
};

// Span-local block b -> table entry: the last entry in [lo, hi) whose first block is <= b (never
// an empty entry: an entry followed by a larger first block contains b).
__device__ __forceinline__ int sp_find(const int32_t* sb, int lo, int hi, int b) {
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (sb[mid] <= b) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct SpLane {
  int e, k, nval;
  int64_t start;
  bool valid, in_pin;
};

__device__ __forceinline__ SpLane sp_resolve(const SpTable& T, int ne, int nblk, int tile) {
  const int lane = threadIdx.x & 31;
  SpLane L;
  const int b = tile * WT + lane;
  L.valid = b < nblk;
  int ex = 0;
  if (lane == 0) ex = sp_find(T.sb, 0, ne, tile * WT);
  if (lane == 1) ex = sp_find(T.sb, 0, ne, min(nblk - 1, tile * WT + WT - 1));
  const int e0 = __shfl_sync(0xffffffffu, ex, 0), e1 = __shfl_sync(0xffffffffu, ex, 1);
  L.e = (e0 == e1 || !L.valid) ? e0 : sp_find(T.sb, e0, e1 + 1, b);
  L.k = T.k0[L.e] + (b - T.sb[L.e]);
  L.start = T.to[L.e] + (int64_t)L.k * BT;
  const int nv = T.len[L.e] - L.k * BT;
  L.nval = L.valid ? (nv > BT ? BT : nv) : 0;
  const int pl = T.pl[L.e];
  L.in_pin = L.valid && pl >= 0 && L.k < (pl + BT - 1) / BT;
  return L;
}

// Issue the staging of one tile on `bar` (always arms the barrier, so phases stay in step).
// Returns the token at staged word 0, or -1 when the tile is read from global memory.
__device__ __forceinline__ int64_t sp_stage(const MatchKernelArgs& K, const CUtensorMap* tm, const SpTable& T,
                                            const SpLane& L, uint8_t* buf, uint64_t* bar) {
  const int lane = threadIdx.x & 31;
  const unsigned vm = __ballot_sync(0xffffffffu, L.valid);
  const int lastv = vm ? 31 - __clz(vm) : 0;
  const int64_t row0 = __shfl_sync(0xffffffffu, L.start, 0) >> 5;
  const int64_t a1 = __shfl_sync(0xffffffffu, (L.start & ~int64_t(3)) + 20, lastv);
  const bool staged = K.tok_rows > 0 && a1 <= K.tok_rows * 32;
  const unsigned pin_m = __ballot_sync(0xffffffffu, L.in_pin);
  const int prev_e = __shfl_up_sync(0xffffffffu, L.e, 1);
  const bool head = L.in_pin && (lane == 0 || !((pin_m >> (lane - 1)) & 1u) || prev_e != L.e);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  uint32_t pin_bytes = 0;
  if (head) {
    const unsigned after = ~((2u << lane) - 1u);
    const unsigned stop = (heads | ~pin_m) & after;
    const int end = stop ? __ffs(stop) - 1 : 32;
    pin_bytes = (uint32_t)(end - lane) * 64u;
  }
  const uint32_t total = __reduce_add_sync(0xffffffffu, pin_bytes) + (staged ? (uint32_t)SP_TOKB : 0u);
  if (lane == 0) {
    fence_proxy_async_smem();  // this warp's earlier generic reads of the buffer precede the refill
    mbar_expect_tx(bar, total);
  }
  __syncwarp();
  if (staged && lane == 0) bulk_tensor_2d(buf, tm, 0, (int)row0, bar);
  if (head)
    bulk_copy(buf + SP_TOKB + lane * 64, K.pin_tok + pin_tok_index(T.wf[L.e], L.k, 0, K.pin_groups), pin_bytes, bar);
  return staged ? (row0 << 5) : -1;
}

// first r in [0, n] with tok_off[r] >= x, n + 1 if none (one warp, 32-ary: ~3 dependent loads)
__device__ __forceinline__ int64_t sp_lower(const int64_t* __restrict__ off, int64_t n, int64_t x) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n + 1;  // answer in [lo, hi]; off[hi] >= x (or hi == n + 1)
  while (lo < hi) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + (int64_t)lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, idx < hi && __ldg(off + idx) >= x);
    const int cnt = (int)min((int64_t)32, (hi - lo + step - 1) / step);
    const int f = m ? __ffs(m) - 1 : cnt;
    if (f == 0) return lo;
    if (m) hi = lo + (int64_t)f * step;
    lo = lo + (int64_t)(f - 1) * step + 1;
  }
  return lo;
}

template <bool HASH>
__global__ void __launch_bounds__(SP_THREADS, SFKV_SP_MINB) match_span_kernel(MatchKernelArgs K, SpanState S,
                                                                           const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ uint8_t s_dyn[];
  __shared__ __align__(8) uint64_t s_bar[SP_WARPS][2];
  __shared__ SpTable T;
  __shared__ uint64_t s_dig[SP_RBLK];
  __shared__ uint32_t s_head[(SP_RBLK + 31) / 32];
  __shared__ uint64_t s_car[SP_CARRY];
  __shared__ uint64_t s_wagg[SP_WARPS];
  __shared__ uint32_t s_wflag[SP_WARPS];
  __shared__ int64_t s_c, s_ra, s_rb, s_base, s_total;
  __shared__ uint64_t s_trail;
  __shared__ int32_t s_trail_mn, s_any_head;
  const MatchArgs& A = K.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* bufs = s_dyn + ((1024 - (smem_u32(s_dyn) & 1023)) & 1023);  // 1 KB aligned (swizzle)
  auto buf = [&](int b) { return bufs + (size_t)(warp * 2 + b) * SP_BUF; };
  if (lane == 0) {
    mbar_init(&s_bar[warp][0]);
    mbar_init(&s_bar[warp][1]);
  }
  pdl_trigger();
  pdl_wait();
  if (tid == 0) {
    s_c = (int64_t)(atomicAdd(S.ticket, 1ull) - S.base);
    s_any_head = 0;
    s_trail = 0;
    s_trail_mn = INT32_MAX;
  }
  __syncthreads();
  const int64_t c = s_c;
  if (tid == 0) {  // the other parity's statuses for this span start out unpublished
    S.blk_o[c] = 0;
    S.chain_o[c] = 0;
    S.mism_o[c] = 0;
  }
  const int64_t n = A.n;
  int64_t total = __ldg(&A.tok_off[n]);
  if (total > A.n_tok_bound) {  // a device batch larger than its declared buffer: fail loudly
    if (tid == 0) *S.error = SFKV_EINVAL;
    total = A.n_tok_bound;
  }
  const int64_t cS = c * SPAN, cE = cS + SPAN;
  if (cS > total) return;
  if (warp == 0) {  // owned requests [ra, rb): first token in [cS, cE)
    const int64_t ra = sp_lower(A.tok_off, n, cS);
    const int64_t rb = sp_lower(A.tok_off, n, cE);
    if (lane == 0) {
      s_ra = ra > n ? n : ra;
      s_rb = rb > n ? n : rb;
    }
  }
  __syncthreads();
  const int64_t ra = s_ra, rb = s_rb;
  int64_t rc = -1;  // the carry-in request: ra - 1 when it has a block starting at or after cS
  int32_t kc = 0;
  if (ra > 0) {
    const int64_t to = __ldg(&A.tok_off[ra - 1]), len = __ldg(&A.tok_off[ra]) - to;
    const int64_t k = (cS - to + BT - 1) / BT;
    if (k * BT < len) {
      rc = ra - 1;
      kc = (int32_t)k;
    }
  }
  const int has_cin = rc >= 0 ? 1 : 0;
  const int64_t ne_all = has_cin + (rb - ra);
  // at least one round: a span with no entry (it starts at the batch end) still publishes its
  // block count and writes the closing offset
  const int rounds = ne_all > 0 ? (int)((ne_all + SP_RREQ - 1) / SP_RREQ) : 1;
  auto entry = [&](int64_t i, int64_t& r, int64_t& to, int64_t& len, int32_t& k0, int32_t& nin) {
    r = (has_cin && i == 0) ? rc : ra + i - has_cin;
    to = __ldg(&A.tok_off[r]);
    len = __ldg(&A.tok_off[r + 1]) - to;
    k0 = (r == rc) ? kc : 0;
    const int64_t nb = (len + BT - 1) / BT;
    const int64_t kl = cE > to ? (cE - to + BT - 1) / BT : 0;
    const int64_t hi = nb < kl ? nb : kl;
    nin = (int32_t)(hi > k0 ? hi - k0 : 0);
  };
  if (rounds > 1) {  // the span's block count first (one extra pass over dense spans only)
    int64_t s = 0;
    for (int64_t i = tid; i < ne_all; i += SP_THREADS) {
      int64_t r, to, len;
      int32_t k0, nin;
      entry(i, r, to, len, k0, nin);
      s += nin;
    }
    s = (int64_t)warp_sum((uint64_t)s);
    if (lane == 0) s_wagg[warp] = (uint64_t)s;
    __syncthreads();
    if (tid == 0) {
      int64_t t = 0;
      for (int w = 0; w < SP_WARPS; ++w) t += (int64_t)s_wagg[w];
      s_total = t;
    }
    __syncthreads();
  }
  // carry-in facts kept across rounds (round 0's table is rebuilt by later rounds)
  int64_t cin_len = 0;
  int32_t cin_pl = -1, cin_nin = 0, cin_mn = INT32_MAX;
  bool cin_ends = false;
  uint32_t ph = 0u;  // mbarrier phase parity per buffer (bit b)
  int64_t roff = 0;           // span-local index of this round's first block
  for (int rd = 0; rd < rounds; ++rd) {
    // ---- round table: one entry per thread, block counts scanned over the CTA ----
    const int64_t i0 = (int64_t)rd * SP_RREQ;
    const int ne = (int)min((int64_t)SP_RREQ, ne_all - i0);
    int32_t nin = 0;
    if (tid < (SP_RBLK + 31) / 32) s_head[tid] = 0;
    if (tid < ne) {
      int64_t r, to, len;
      int32_t k0;
      entry(i0 + tid, r, to, len, k0, nin);
      int32_t wf = __ldg(&A.wf[r]), pl = -1;
      if ((uint32_t)wf < (uint32_t)S.max_wf) {
        pl = (int32_t)__ldg(&S.pin_len[wf]);
      } else {  // device-side slot guard: matches as unpinned, sticky SFKV_EINVAL
        *S.error = SFKV_EINVAL;
        wf = 0;
      }
      T.to[tid] = to;
      T.r[tid] = (int32_t)r;
      T.len[tid] = (int32_t)len;
      T.k0[tid] = k0;
      T.wf[tid] = wf;
      T.pl[tid] = pl;
      T.mn[tid] = INT32_MAX;
    }
    int32_t x = nin;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += u;
    }
    if (lane == 31) s_wagg[warp] = (uint64_t)x;
    __syncthreads();
    int32_t wpre = 0, nblk = 0;
#pragma unroll
    for (int w = 0; w < SP_WARPS; ++w) {
      const int32_t v = (int32_t)s_wagg[w];
      if (w < warp) wpre += v;
      nblk += v;
    }
    if (tid < ne) {
      const int32_t sb = wpre + x - nin;
      T.sb[tid] = sb;
      if (T.k0[tid] == 0 && nin > 0) atomicOr(&s_head[sb >> 5], 1u << (sb & 31));
    }
    if (tid == 0) {
      T.sb[ne] = nblk;
      if (rd == 0) {
        if (rounds == 1) s_total = nblk;
        st_status(S.blk + c, SP_AGG | (uint64_t)(rounds == 1 ? nblk : s_total));
      }
    }
    __syncthreads();
    if (rd == 0 && has_cin) {
      cin_len = T.len[0];
      cin_pl = T.pl[0];
      cin_nin = T.sb[1];
    }
    // ---- stage this warp's first two tiles, then (round 0, warp 0) the span's first block ----
    const int ntiles = (nblk + WT - 1) / WT;
    int64_t a0_0 = -1, a0_1 = -1;  // first staged token per buffer (-1: read from global)
    if (warp < ntiles) a0_0 = sp_stage(K, &tmap, T, sp_resolve(T, ne, nblk, warp), buf(0), &s_bar[warp][0]);
    if (warp + SP_WARPS < ntiles)
      a0_1 = sp_stage(K, &tmap, T, sp_resolve(T, ne, nblk, warp + SP_WARPS), buf(1), &s_bar[warp][1]);
    if (rd == 0 && warp == 0) {
      uint64_t prefix = 0;
      for (int64_t bs = c - 1; bs >= 0; bs -= 32) {
        const int64_t p = bs - lane;
        const uint64_t v = p >= 0 ? ld_status_spin(S.blk + p) : SP_INCL;
        const unsigned incl = __ballot_sync(0xffffffffu, (v & SP_KIND) == SP_INCL);
        const int first = incl ? __ffs(incl) - 1 : 31;
        prefix += warp_sum(lane <= first ? (v & ~SP_KIND) : 0ull);
        if (incl) break;
      }
      if (lane == 0) {
        st_status(S.blk + c, SP_INCL | (prefix + (uint64_t)s_total));
        s_base = (int64_t)prefix;
      }
    }
    // ---- tiles ----
    int jn = 0;
    for (int tile = warp; tile < ntiles; tile += SP_WARPS, ++jn) {
      const int bi = jn & 1;
      const SpLane L = sp_resolve(T, ne, nblk, tile);
      mbar_wait(&s_bar[warp][bi], (ph >> bi) & 1u);
      ph ^= 1u << bi;
      const int64_t a0 = bi ? a0_1 : a0_0;
      uint32_t t[BT], q[BT];
      const uint32_t* st = reinterpret_cast<const uint32_t*>(buf(bi));
      if (a0 >= 0) {
        const int o = L.valid ? (int)(L.start - a0) : 0;
        const int sh0 = __shfl_sync(0xffffffffu, o & 3, 0);
        if (__all_sync(0xffffffffu, !L.valid || (o & 3) == sh0)) {
          switch (sh0) {
            case 0: load_swz_sh<0>(st, o, t); break;
            case 1: load_swz_sh<1>(st, o, t); break;
            case 2: load_swz_sh<2>(st, o, t); break;
            default: load_swz_sh<3>(st, o, t); break;
          }
          if (L.nval < BT) {
#pragma unroll
            for (int j = 0; j < BT; ++j)
              if (j >= L.nval) t[j] = 0u;
          }
        } else {
          load_block_swz(st, o, L.nval, t);
        }
      } else if (L.valid) {
        load_block(A.tok, L.start, L.nval, A.n_tok_bound, t);
      }
      if (!L.valid) {
#pragma unroll
        for (int j = 0; j < BT; ++j) t[j] = 0u;
      }
      if (L.in_pin) load_pin_rot(reinterpret_cast<const uint32_t*>(buf(bi) + SP_TOKB), lane, L.k, q);
      __syncwarp();
      if (tile + 2 * SP_WARPS < ntiles) {  // the buffer is free: stage this warp's tile after next
        const int64_t an = sp_stage(K, &tmap, T, sp_resolve(T, ne, nblk, tile + 2 * SP_WARPS), buf(bi), &s_bar[warp][bi]);
        if (bi) a0_1 = an;
        else a0_0 = an;
      }
      // M: a block whose 16 words agree with the pin's has no mismatch (both sides zero padded);
      // a differing one finds its exact first mismatch below min(valid tokens, pin tokens)
      if (L.in_pin) {
        uint32_t d = 0;
#pragma unroll
        for (int j = 0; j < BT; ++j) d |= q[j] ^ t[j];
        if (d) {
          const int lim = min(L.nval, min(T.pl[L.e] - L.k * BT, BT));
          unsigned nem = 1u << lim;
#pragma unroll
          for (int j = 0; j < BT; ++j) nem |= (q[j] != t[j]) ? (1u << j) : 0u;
          const int lcp = __ffs(nem) - 1;
          if (lcp < lim) atomicMin(&T.mn[L.e], L.k * BT + lcp);
        }
      }
      if constexpr (HASH) {
        if (L.valid) s_dig[tile * WT + lane] = block_digest_words((uint64_t)L.k, (uint32_t)L.nval, t);
      }
    }
    __syncthreads();
    const int64_t base = s_base;
    // ---- segmented scan of the digests: chain sums since the last request head (or the span
    //      start, for the carry-in blocks) ----
    if constexpr (HASH) {
      uint64_t v[SP_IPT];
      uint32_t hm = 0;
      uint64_t run = 0;
#pragma unroll
      for (int i = 0; i < SP_IPT; ++i) {
        const int b = tid * SP_IPT + i;
        if (b < nblk && ((s_head[b >> 5] >> (b & 31)) & 1u)) {
          run = 0;
          hm |= 1u << i;
        }
        run += b < nblk ? s_dig[b] : 0ull;
        v[i] = run;
      }
      // (flag, sum) pairs combine as (f1, a1) + (f2, a2) = (f1 | f2, f2 ? a2 : a1 + a2)
      uint64_t a = run;
      uint32_t f = hm ? 1u : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t ua = __shfl_up_sync(0xffffffffu, a, d);
        const uint32_t uf = __shfl_up_sync(0xffffffffu, f, d);
        if (lane >= d) {
          if (!f) a += ua;
          f |= uf;
        }
      }
      if (lane == 31) {
        s_wagg[warp] = a;
        s_wflag[warp] = f;
      }
      uint64_t ea = __shfl_up_sync(0xffffffffu, a, 1);
      uint32_t ef = __shfl_up_sync(0xffffffffu, f, 1);
      if (lane == 0) {
        ea = 0;
        ef = 0;
      }
      __syncthreads();
      uint64_t wa = 0;
      uint32_t wfl = 0;
      for (int w = 0; w < warp; ++w) {
        if (s_wflag[w]) {
          wa = s_wagg[w];
          wfl = 1;
        } else {
          wa += s_wagg[w];
        }
      }
      if (!ef) ea += wa;
      ef |= wfl;
#pragma unroll
      for (int i = 0; i < SP_IPT; ++i) {
        const int b = tid * SP_IPT + i;
        if (b < nblk) {
          uint64_t sum = v[i];
          bool fin = true;
          if ((hm & ((2u << i) - 1u)) == 0) {  // no head in this thread up to item i
            sum += ea;
            fin = ef != 0;
          }
          sum &= CHAIN_MASK;
          if (fin) {
            if (A.out_hash) A.out_hash[base + roff + b] = chain_finalize(sum);
          } else {
            s_car[b] = sum;  // a carry-in block: waits for the predecessors' sum
          }
          s_dig[b] = sum;
        }
      }
      __syncthreads();
    }
    // ---- per-request outputs of this round ----
    if (tid < ne) {
      const int32_t sbv = T.sb[tid], ninv = T.sb[tid + 1] - sbv;
      const int64_t len = T.len[tid];
      const int64_t nb = (len + BT - 1) / BT;
      const bool ends = T.k0[tid] + ninv == nb;
      const int32_t pl = T.pl[tid], mn = T.mn[tid];
      if (rd == 0 && has_cin && tid == 0) {
        cin_mn = mn;
        cin_ends = ends;
      } else {
        const int32_t r = T.r[tid];
        A.blk_off[r] = base + roff + sbv;
        if (ends) A.out_M[r] = pl < 0 ? 0 : min(min((int64_t)pl, len), (int64_t)mn);
      }
    }
    if (tid == 0 && nblk > 0) {  // the trailing request so far: the entry holding the last block
      const int e = sp_find(T.sb, 0, ne, nblk - 1);
      s_trail = HASH ? s_dig[nblk - 1] : 0ull;
      s_trail_mn = T.mn[e];
      bool any = false;
      for (int w = 0; w < (nblk + 31) / 32; ++w) any |= s_head[w] != 0;
      if (any) s_any_head = 1;
    }
    roff += nblk;
    __syncthreads();
  }
  // ---- closing offset, the span's chain statuses, the carry-in request ----
  const int64_t base = s_base;
  if (tid == 0 && total < cE) A.blk_off[n] = base + s_total;
  // INCL: the trailing request's head lies in the span (or the span holds no block at all, so no
  // later span continues through it); AGG: the whole span is one request's middle
  const bool incl = s_any_head != 0 || s_total == 0;
  if (tid == 0) {
    st_status(S.mism + c, SP_MVALID | (uint32_t)(incl ? s_trail_mn : cin_mn));
    st_status(S.chain + c, (incl ? SP_INCL : SP_AGG) | (s_trail & CHAIN_MASK));
  }
  if (!has_cin || warp != 0) return;
  // carry: predecessors' sums up to the first inclusive status; first mismatch: their words up to
  // the span holding the request's head (SP_INCL), through derived-inclusive spans (SP_INCLD)
  uint64_t carry = 0;
  bool carry_done = false;
  int32_t mn = cin_mn;
  for (int64_t bs = c - 1;; bs -= 32) {
    const int64_t p = bs - lane;
    const uint64_t v = p >= 0 ? ld_status_spin(S.chain + p) : SP_INCL;
    if (!carry_done) {
      const unsigned im = __ballot_sync(0xffffffffu, (v & SP_KIND) >= SP_INCL);
      const int first = im ? __ffs(im) - 1 : 31;
      carry += warp_sum(lane <= first ? (v & CHAIN_MASK) : 0ull);
      carry_done = im != 0;
    }
    const unsigned hm = __ballot_sync(0xffffffffu, (v & SP_KIND) == SP_INCL);
    const int firsth = hm ? __ffs(hm) - 1 : 31;
    const int32_t pm = (lane <= firsth && p >= 0) ? (int32_t)(uint32_t)ld_status_spin(S.mism + p) : INT32_MAX;
    mn = min(mn, __reduce_min_sync(0xffffffffu, pm));
    if (hm) break;
  }
  carry &= CHAIN_MASK;
  if (!incl && lane == 0) st_status(S.chain + c, SP_INCLD | ((carry + s_trail) & CHAIN_MASK));
  if (HASH && A.out_hash)
    for (int b = lane; b < cin_nin; b += 32) A.out_hash[base + b] = chain_finalize((carry + s_car[b]) & CHAIN_MASK);
  if (lane == 0 && cin_ends) A.out_M[rc] = cin_pl < 0 ? 0 : min(min((int64_t)cin_pl, cin_len), (int64_t)mn);
}

static int launch_span(sfkv_pool* p, const MatchArgs& a, MatchKernelArgs K, const CUtensorMap& tm, cudaStream_t st) {
  const int64_t nspans = a.n_tok_bound / SPAN + 1;
  if (p->span_cap < nspans) {  // [ticket][blk, chain, mism] x 2 parities, all clear
    int64_t cap = p->span_cap ? p->span_cap : 4096;
    while (cap < nspans) cap *= 2;
    if (int rc = p->span_state.ensure(256 + 6 * sizeof(uint64_t) * (size_t)cap)) return rc;
    SFKV_CUDA(cudaMemsetAsync(p->span_state.ptr, 0, p->span_state.bytes, st));
    p->span_cap = cap;
    p->span_base = 0;
    for (int b = 0; b < 2; ++b) p->span_dirty_lo[b] = p->span_dirty_hi[b] = 0;
  }
  const int b = p->span_parity, o = b ^ 1;
  uint64_t* arr = reinterpret_cast<uint64_t*>(p->span_state.as<char>() + 256);
  auto par = [&](int q) { return arr + (size_t)q * 3 * p->span_cap; };
  // statuses of this parity left by an earlier, larger launch that nothing has cleared yet
  if (p->span_dirty_hi[b] > p->span_dirty_lo[b] && p->span_dirty_lo[b] < nspans) {
    for (int k = 0; k < 3; ++k)
      SFKV_CUDA(cudaMemsetAsync(par(b) + k * p->span_cap + p->span_dirty_lo[b], 0,
                                sizeof(uint64_t) * (size_t)(p->span_dirty_hi[b] - p->span_dirty_lo[b]), st));
    p->span_dirty_lo[b] = p->span_dirty_hi[b] = 0;
  }
  SpanState S;
  S.ticket = p->span_state.as<unsigned long long>();
  S.base = p->span_base;
  S.blk = par(b);
  S.chain = S.blk + p->span_cap;
  S.mism = S.chain + p->span_cap;
  S.blk_o = par(o);
  S.chain_o = S.blk_o + p->span_cap;
  S.mism_o = S.chain_o + p->span_cap;
  S.pin_len = p->pin_len;
  S.max_wf = p->cfg.max_workflows;
  S.error = &p->ctr->error;
  static bool attr = false;
  if (!attr) {
    SFKV_CUDA(cudaFuncSetAttribute(match_span_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_DYN));
    SFKV_CUDA(cudaFuncSetAttribute(match_span_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_DYN));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nspans);
  cfg.blockDim = dim3(SP_THREADS);
  cfg.dynamicSmemBytes = SP_DYN;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (a.out_hash) SFKV_CUDA(cudaLaunchKernelEx(&cfg, match_span_kernel<true>, K, S, tm));
  else SFKV_CUDA(cudaLaunchKernelEx(&cfg, match_span_kernel<false>, K, S, tm));
  // bookkeeping: this parity now holds [0, nspans); the other parity's [0, nspans) was cleared
  p->span_base += (uint64_t)nspans;
  p->span_dirty_lo[b] = 0;
  p->span_dirty_hi[b] = std::max(p->span_dirty_hi[b], nspans);
  if (p->span_dirty_hi[o] <= nspans) p->span_dirty_lo[o] = p->span_dirty_hi[o] = 0;
  else p->span_dirty_lo[o] = std::max(p->span_dirty_lo[o], nspans);
  p->span_parity = o;
  return 0;
}

static int encode_token_map(const MatchArgs& a, CUtensorMap& tm, int64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    SFKV_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return fail(SFKV_ECUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, TMAP_ROWS};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(a.tok), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SFKV_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return 0;
}

int launch_match(sfkv_pool* p, const MatchArgs& a, int64_t* tile_state, cudaStream_t st) {
  if (a.n <= 0) return 0;
  if (a.out_M && !a.out_block) {  // match mode (M, optional chained hashes): one span-pass launch
    MatchKernelArgs K{};
    K.a = a;
    K.pin_tok = p->pin_tok;
    K.pin_groups = pin_groups(p->cfg);
    K.tok_rows = a.n_tok_bound / 32;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    if (K.tok_rows > 0) {
      if (int rc = encode_token_map(a, tm, K.tok_rows)) return rc;
    }
    return launch_span(p, a, K, tm, st);
  }
  const int64_t ntiles = (a.n_items + WT - 1) / WT;
  const int64_t np = prep_tiles(a.n);
  unsigned long long* ticket = reinterpret_cast<unsigned long long*>(tile_state);
  uint64_t* status = reinterpret_cast<uint64_t*>(tile_state + 1 + np);
  const int64_t th = tile_head(np, ntiles);
  TileRec* trec = reinterpret_cast<TileRec*>(tile_state + th);
  const int64_t head = th + 4 * ntiles;
  ReqRec* rec = reinterpret_cast<ReqRec*>(tile_state + head);
  uint64_t* local = reinterpret_cast<uint64_t*>(tile_state + head + 4 * (a.n + 1));
  uint32_t* rk = reinterpret_cast<uint32_t*>(tile_state + head + 4 * (a.n + 1) + a.n_items);

  // prep statuses: a per-pool buffer, epoch-tagged (cleared only when it grows or the epoch wraps)
  const size_t need = sizeof(uint64_t) * (size_t)(np + 1);
  if (p->prep_status.bytes < need) {
    if (int rc = p->prep_status.ensure(need)) return rc;
    SFKV_CUDA(cudaMemsetAsync(p->prep_status.ptr, 0, p->prep_status.bytes, st));
    p->prep_epoch = 0;
  }
  p->prep_epoch = (p->prep_epoch + 1) & 0x3FFF;
  if (p->prep_epoch == 0) {
    SFKV_CUDA(cudaMemsetAsync(p->prep_status.ptr, 0, p->prep_status.bytes, st));
    p->prep_epoch = 1;
  }
  static int prep_resident = 0;  // prep CTAs that can be resident at once (same for every pool)
  if (!prep_resident) {
    int per_sm = 0, dev = 0, sms = 0;
    SFKV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, match_prep_kernel, PREP_THREADS, 0));
    SFKV_CUDA(cudaGetDevice(&dev));
    SFKV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    prep_resident = per_sm * sms;
  }
  const bool use_ticket = np > prep_resident / 2;  // leave room for co-running kernels
  if (use_ticket) SFKV_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), st));
  PrepArgs P;
  P.n = a.n;
  P.tok_off = a.tok_off;
  P.wf = a.out_M ? a.wf : nullptr;
  P.pin_len = p->pin_len;
  P.blk_off = a.blk_off;
  P.rec = rec;
  P.trec = trec;
  P.out_M = a.out_M;
  P.out_hit = a.out_hit;
  P.ticket = use_ticket ? ticket : nullptr;
  P.pstatus = p->prep_status.as<uint64_t>();
  P.epoch = p->prep_epoch;
  P.max_wf = p->cfg.max_workflows;
  P.error = &p->ctr->error;
  match_prep_kernel<<<(unsigned)np, PREP_THREADS, 0, st>>>(P);
  SFKV_LAUNCH_CHECK("match_prep_kernel");
  if (ntiles == 0) return 0;

  MatchKernelArgs K;
  K.a = a;
  K.rec = rec;
  K.pin_tok = p->pin_tok;
  K.blk_tok = p->blk_tok;
  K.blk_parent = p->blk_parent;
  K.blk_n = p->blk_n;
  K.slots = p->slots;
  K.slot_mask = (uint64_t)p->table_slots - 1;
  K.pin_groups = pin_groups(p->cfg);
  K.status = status;
  K.local = local;
  K.rk = a.out_block ? rk : nullptr;
  K.trec = trec;
  K.hashes = (a.out_hash || a.out_block) ? 1 : 0;
  const int64_t grid = (ntiles + BLOCK_THREADS / 32 - 1) / (BLOCK_THREADS / 32);
  // lookup mode (no pins) keeps plain 16-B loads: staging measured slower there (C5 607 vs 510 us)
  // token tensor map (rows of 32 ids); a batch smaller than one row stages nothing
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  K.tok_rows = a.n_tok_bound / 32;
  const bool per_request = a.out_block && !a.out_M && a.n >= LR_MIN_REQUESTS &&
                           a.n_items <= LR_MAX_AVG_BLOCKS * a.n;
  if ((a.out_M || per_request) && K.tok_rows > 0) {
    if (int rc = encode_token_map(a, tm, K.tok_rows)) return rc;
  } else {
    K.tok_rows = 0;
  }
  if (per_request) {
    const unsigned lgrid = (unsigned)((a.n + LR_THREADS / 32 - 1) / (LR_THREADS / 32));
    SFKV_CUDA(launch_pdl(lookup_req_kernel, dim3(lgrid), dim3(LR_THREADS), st, K, tm));
    return 0;
  }
  if (a.out_M) SFKV_CUDA(launch_pdl(match_block_kernel<true>, dim3((unsigned)grid), dim3(BLOCK_THREADS), st, K, tm));
  else SFKV_CUDA(launch_pdl(match_block_kernel<false>, dim3((unsigned)grid), dim3(BLOCK_THREADS), st, K, tm));
  if (K.hashes) {
    const int tpw = a.out_block ? CH_TPW_LOOKUP : CH_TPW_HASH;
    const int64_t cwarps = (ntiles + tpw - 1) / tpw;
    const unsigned cgrid = (unsigned)((cwarps + MATCH_THREADS / 32 - 1) / (MATCH_THREADS / 32));
    if (a.out_block) SFKV_CUDA(launch_pdl(match_chain_kernel<true>, dim3(cgrid), dim3(MATCH_THREADS), st, K));
    else SFKV_CUDA(launch_pdl(match_chain_kernel<false>, dim3(cgrid), dim3(MATCH_THREADS), st, K));
  }
  return 0;
}

}  // namespace sfkv

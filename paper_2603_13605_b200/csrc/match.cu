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
#ifndef SFKV_MATCH_THREADS
#define SFKV_MATCH_THREADS 256
#endif
constexpr int MATCH_THREADS = SFKV_MATCH_THREADS;  // chain pass CTA
#ifndef SFKV_BLOCK_THREADS
#define SFKV_BLOCK_THREADS 64
#endif
constexpr int BLOCK_THREADS = SFKV_BLOCK_THREADS;  // block pass: 2 warps per CTA (measured 64 / 128 / 256 threads: 67.2 / 68.5 / 72.8 us per C2 step)
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
#ifndef SFKV_PREP_PDL
#define SFKV_PREP_PDL 1
#endif

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
  pdl_wait();  // a no-op unless launched as a programmatic dependent
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
  for (int64_t t = (b + WT - 1) / WT; P.trec && t * WT < b + nb; ++t) {  // (the per-request lookup has no tiles)
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
__device__ __forceinline__ Ctx resolve(const MatchKernelArgs& K, int64_t tile, int64_t n_items, int4 ta, int4 tb) {
  const int lane = threadIdx.x & 31;
  const int64_t n = K.a.n;
  const int64_t T0 = tile * WT;
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

__device__ __forceinline__ Ctx resolve(const MatchKernelArgs& K, int64_t tile, int64_t n_items) {
  const int4* tp = reinterpret_cast<const int4*>(K.trec + tile);
  return resolve(K, tile, n_items, __ldg(tp), __ldg(tp + 1));
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

// L2 residency hints (SFKV_L2HINT): the streamed request tokens and pin blocks are read once
// (evict_first), while the per-block chain sums the block pass writes for the chain pass should
// still be in L2 when it reads them (evict_last).
#ifndef SFKV_L2HINT
#define SFKV_L2HINT 1
#endif
__device__ __forceinline__ void bulk_copy_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_tensor_2d_hint(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* bar,
                                                    uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
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


// Block tokens of a lane whose block starts at word o (o & 3 == SH) of a swizzled staged range.
__device__ __forceinline__ uint4 lds128(uint32_t addr) {  // 16-B shared load by 32-bit address
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <int SH>
__device__ __forceinline__ void load_swz_sh(const uint32_t* s, int o, uint32_t* t) {
  const uint32_t base = smem_u32(s);
  const int c0 = o >> 2;
  constexpr int NC = SH ? 5 : 4;
  uint32_t w[20];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const uint32_t g = (uint32_t)(c0 + i);
    const uint4 v = lds128(base + ((g ^ ((g >> 3) & 7u)) << 4));
    w[4 * i] = v.x;
    w[4 * i + 1] = v.y;
    w[4 * i + 2] = v.z;
    w[4 * i + 3] = v.w;
  }
#pragma unroll
  for (int j = 0; j < BT; ++j) t[j] = w[j + SH];
}
__device__ __forceinline__ void load_pin_rot(const uint32_t* s, int lane, int64_t k, uint32_t* q) {
  const uint32_t base = smem_u32(s) + (uint32_t)lane * 64u, r = (uint32_t)pin_rot(k);
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const uint4 w = lds128(base + (((r + (uint32_t)x) & 3u) << 4));
    q[4 * x] = w.x;
    q[4 * x + 1] = w.y;
    q[4 * x + 2] = w.z;
    q[4 * x + 3] = w.w;
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
#if SFKV_L2HINT
      st_u64_hint(K.local + item, (h << 63) | (v & CHAIN_MASK), l2_policy_last());
#else
      K.local[item] = (h << 63) | (v & CHAIN_MASK);
#endif
      if (K.rk) K.rk[item] = (uint32_t)c.r | (c.nval == BT ? RK_FULL : 0u);
    }
    if (lane == 31) K.status[tile] = (h ? ST_INCL : ST_AGG) | (v & CHAIN_MASK);
  }
}


// One warp per 32-block tile, one block per lane, non-persistent: enough tiles in flight per SM to
// cover the window -> tokens/pin-tokens round trips.
// 16 CTAs (32 warps) per SM at <= 64 registers: no spills (48 registers spilled and 10 CTAs of 4 warps
// measured 2 us slower).
#ifndef SFKV_MB_MINB
#define SFKV_MB_MINB 16
#endif
#ifndef SFKV_MB_TPW
#define SFKV_MB_TPW 1
#endif
// Staging of one tile into a warp's buffers: the token range (one 2D tensor-map box) and, per
// request segment of in-pin blocks, that segment's pin blocks (pin-major: one extent at lane*64 B),
// all on one mbarrier phase. Returns whether the barrier was armed (something to wait for).
__device__ __forceinline__ bool stage_tile(const MatchKernelArgs& K, const CUtensorMap* tmap, const Ctx& c,
                                           bool in_pin, uint32_t* s_tok, uint32_t* s_pin, uint64_t* bar,
                                           int64_t& a0, bool& staged) {
  const int lane = threadIdx.x & 31;
  const int nv = __popc(__ballot_sync(0xffffffffu, c.valid));
  const int64_t row0 = __shfl_sync(0xffffffffu, c.start, 0) >> 5;
  a0 = row0 << 5;
  const int64_t a1 = __shfl_sync(0xffffffffu, (c.start & ~int64_t(3)) + 20, nv - 1);
  staged = a1 <= K.tok_rows * 32;  // all but the tiles touching the last partial row
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
  if (!total) return false;
  if (lane == 0) mbar_expect_tx(bar, total);
  __syncwarp();
#if SFKV_L2HINT
  const uint64_t pol = l2_policy_first();
  if (staged && lane == 0) bulk_tensor_2d_hint(s_tok, tmap, 0, (int)row0, bar, pol);
  if (head)
    bulk_copy_hint(s_pin + lane * PIN_STRIDE, K.pin_tok + pin_tok_index(c.wf, c.k, 0, K.pin_groups), pin_bytes, bar, pol);
#else
  if (staged && lane == 0) bulk_tensor_2d(s_tok, tmap, 0, (int)row0, bar);
  if (head) bulk_copy(s_pin + lane * PIN_STRIDE, K.pin_tok + pin_tok_index(c.wf, c.k, 0, K.pin_groups), pin_bytes, bar);
#endif
  return true;
}

// Block tokens t (zero padded) and, for in-pin blocks, the pin's block q of a staged tile.
__device__ __forceinline__ void load_staged_tile(const MatchKernelArgs& K, const Ctx& c, bool in_pin, bool staged,
                                                 int64_t a0, int64_t tok_total, const uint32_t* s_tok,
                                                 const uint32_t* s_pin, uint32_t* t, uint32_t* q) {
  const int lane = threadIdx.x & 31;
  if (staged) {
    // every lane of a tile inside one request shares the token alignment: a warp-uniform
    // specialisation reads the swizzled range with no per-lane funnel selects
    const int o = c.valid ? (int)(c.start - a0) : 0;
    const int sh0 = __shfl_sync(0xffffffffu, o & 3, 0);
    if (__all_sync(0xffffffffu, !c.valid || (o & 3) == sh0)) {
      switch (sh0) {
        case 0: load_swz_sh<0>(s_tok, o, t); break;
        case 1: load_swz_sh<1>(s_tok, o, t); break;
        case 2: load_swz_sh<2>(s_tok, o, t); break;
        default: load_swz_sh<3>(s_tok, o, t); break;
      }
      if (c.nval < BT) {
#pragma unroll
        for (int j = 0; j < BT; ++j)
          if (j >= c.nval) t[j] = 0u;
      }
    } else if (c.valid) {
      load_block_swz(s_tok, o, c.nval, t);
    }
  } else if (c.valid) {
    load_block(K.a.tok, c.start, c.nval, tok_total, t);
  }
  if (in_pin) load_pin_rot(s_pin, lane, c.k, q);
}

// Match mode (STAGED): a warp takes TPW consecutive tiles and stages all of them before
// processing the first, so the later tiles' loads overlap the earlier tiles' compute.
template <bool STAGED>
__global__ void __launch_bounds__(BLOCK_THREADS, SFKV_MB_MINB) match_block_kernel(MatchKernelArgs K,
                                                                       const __grid_constant__ CUtensorMap tmap) {
  constexpr int TPW = STAGED ? SFKV_MB_TPW : 1;
  constexpr int NW = BLOCK_THREADS / 32;
  __shared__ __align__(1024) uint32_t s_tok[STAGED ? NW * TPW : 1][STAGED ? 768 : 4];  // 18 rows, 1 KB-aligned
  __shared__ __align__(128) uint32_t s_pin[STAGED ? NW * TPW : 1][STAGED ? WT * PIN_STRIDE : 4];
  __shared__ __align__(8) uint64_t s_bar[NW * TPW];
  const MatchArgs& A = K.a;
  const int lane = threadIdx.x & 31;
  [[maybe_unused]] const int warp = threadIdx.x >> 5;
  const int64_t tile0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * TPW;
  if constexpr (STAGED) {
    if (lane < TPW) mbar_init(&s_bar[warp * TPW + lane]);
    __syncwarp();
  }
  pdl_trigger();
  pdl_wait();
  // the first tile record is loaded together with the batch totals (speculatively: the record
  // array is carved for the launch's tile bound), saving one round trip before the staging
  const int4* tp0 = reinterpret_cast<const int4*>(K.trec + tile0);
  const int4 ta0 = __ldg(tp0), tb0 = __ldg(tp0 + 1);
  const int64_t n_items = K.rec[A.n].blk_off;
  if (tile0 * WT >= n_items) return;
  const int64_t tok_total = K.rec[A.n].tok_off;
  if constexpr (STAGED) {
    Ctx cs[TPW];
    bool inp[TPW], armed[TPW], stg[TPW];
    int64_t a0[TPW];
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      armed[j] = false;
      if ((tile0 + j) * WT < n_items) {
        cs[j] = j == 0 ? resolve(K, tile0, n_items, ta0, tb0) : resolve(K, tile0 + j, n_items);
        inp[j] = cs[j].valid && cs[j].pin_len >= 0 && cs[j].k < (cs[j].pin_len + BT - 1) / BT;
        armed[j] = stage_tile(K, &tmap, cs[j], inp[j], s_tok[warp * TPW + j], s_pin[warp * TPW + j],
                              &s_bar[warp * TPW + j], a0[j], stg[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      if ((tile0 + j) * WT >= n_items) break;
      if (armed[j]) mbar_wait0(&s_bar[warp * TPW + j]);
      uint32_t q[BT], t[BT];
      load_staged_tile(K, cs[j], inp[j], stg[j], a0[j], tok_total, s_tok[warp * TPW + j], s_pin[warp * TPW + j], t,
                       q);
      if (!cs[j].valid) {
#pragma unroll
        for (int i = 0; i < BT; ++i) t[i] = 0u;
      }
      tile_finish(K, tile0 + j, cs[j], inp[j], t, q);
    }
  } else {
    const int64_t tile = tile0;
    const Ctx c = resolve(K, tile, n_items);
    uint32_t q[BT], t[BT];
    if (c.valid) load_block(A.tok, c.start, c.nval, tok_total, t);
    else {
#pragma unroll
      for (int j = 0; j < BT; ++j) t[j] = 0u;
    }
    tile_finish(K, tile, c, false, t, q);
  }
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
#if SFKV_L2HINT
    if (item < n_items && A.out_hash) st_u64_hint(A.out_hash + item, c[i], l2_policy_first());  // not re-read here
#else
    if (item < n_items && A.out_hash) A.out_hash[item] = c[i];
#endif
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
#ifndef SFKV_LR_THREADS
#define SFKV_LR_THREADS 32
#endif
constexpr int LR_THREADS = SFKV_LR_THREADS;
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
  const uint64_t pol_stream = l2_policy_first();
  int64_t bo, to;
  int32_t len, pl, wf;
  unpack_rec(K.rec + r, bo, to, len, pl, wf);
  const int64_t nb = (len + BT - 1) / BT, nfull = len / BT;
  const int sh_req = (int)(to & 3);
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
#if SFKV_L2HINT
      bulk_tensor_2d_hint(s_tok[warp][i & 1], &tmap, 0, (int)(s0 >> 5), bar, l2_policy_first());  // streamed once
#else
      bulk_tensor_2d(s_tok[warp][i & 1], &tmap, 0, (int)(s0 >> 5), bar);
#endif
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
      if (valid) {  // every block of the request shares the token alignment: no per-lane funnel
        const int o = (int)(start - (((to + i * WT * BT) >> 5) << 5));
        switch (sh_req) {
          case 0: load_swz_sh<0>(s_tok[warp][i & 1], o, t); break;
          case 1: load_swz_sh<1>(s_tok[warp][i & 1], o, t); break;
          case 2: load_swz_sh<2>(s_tok[warp][i & 1], o, t); break;
          default: load_swz_sh<3>(s_tok[warp][i & 1], o, t); break;
        }
        if (nval < BT) {
#pragma unroll
          for (int j = 0; j < BT; ++j)
            if (j >= nval) t[j] = 0u;
        }
      }
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
    if (valid) st_u32_hint(reinterpret_cast<uint32_t*>(A.out_block + bo + k), (uint32_t)id, pol_stream);
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
  // the one-pass lookup (one warp per request) reads request records only: no tile records
  const bool per_request = a.out_block && !a.out_M && a.n >= LR_MIN_REQUESTS && a.n_items <= LR_MAX_AVG_BLOCKS * a.n;
  P.trec = per_request ? nullptr : trec;
  P.out_M = a.out_M;
  P.out_hit = a.out_hit;
  P.ticket = use_ticket ? ticket : nullptr;
  P.pstatus = p->prep_status.as<uint64_t>();
  P.epoch = p->prep_epoch;
  P.max_wf = p->cfg.max_workflows;
  P.error = &p->ctr->error;
#if SFKV_PREP_PDL
  SFKV_CUDA(launch_pdl(match_prep_kernel, dim3((unsigned)np), dim3(PREP_THREADS), st, P));
#else
  match_prep_kernel<<<(unsigned)np, PREP_THREADS, 0, st>>>(P);
#endif
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
  const int64_t sgrid = (ntiles + (BLOCK_THREADS / 32) * SFKV_MB_TPW - 1) / ((BLOCK_THREADS / 32) * SFKV_MB_TPW);
  if (a.out_M) SFKV_CUDA(launch_pdl(match_block_kernel<true>, dim3((unsigned)sgrid), dim3(BLOCK_THREADS), st, K, tm));
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

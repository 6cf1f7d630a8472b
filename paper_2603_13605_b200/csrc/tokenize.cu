// §8f-2: whitespace tokenizer + token interner on the GPU, feeding the match / commit kernels.
//
// Replaces tokenize_whitespace / context_token_sequence (backend.cpp:60-91): tokens are maximal
// runs of non-space bytes (std::isspace in the C locale: ' ', '\t', '\n', '\v', '\f', '\r'),
// messages are tokenized separately and concatenated (a token never spans two messages), roles
// are ignored. The reference keeps tokens as std::string; the pools key on u32 ids, so every token
// string is interned: the same bytes always get the same id for the interner's lifetime, and new
// strings are numbered in order of first occurrence (batch position), which makes ids
// deterministic and equal to a sequential restatement's.
//
// Launches for a batch (text is a CSR of messages, requests are ranges of messages):
//   msg_mark_kernel     message-start bitmap (a message start is a forced token boundary)
//   chunk_count_kernel  token starts per 2 KiB chunk (a warp each): 16-B loads, C-locale space
//                       test on 4 bytes at a time (per-byte SWAR), start = non-space &
//                       (prev space | message start); each 16-byte window's compact space mask
//                       is stored for the emit pass
//   exclusive scan      over chunks
//   chunk_emit_kernel   CTA scan inside each chunk: token start positions, in order, in a shared
//                       list; the chunk (+256 B) is staged in shared memory with a boundary bitmap
//                       built from the count pass's space masks and the message-start words, and
//                       the list is probed one token per thread: length, key, probe. Tokens
//                       of <= 7 bytes key on their own bytes (exact); longer ones on a 63-bit
//                       hash verified against the arena. A string
//                       published by an earlier batch resolves here; claims (CAS into an empty
//                       slot + atomicMin(position): the lowest position owns the new string) and
//                       duplicates of this batch's new strings go to a pending list
//   req_tokoff_kernel   per-request token offsets (chunk offset + starts before the request), on
//                       an aux stream beside the emit pass
//   tok_pending_kernel  one cooperative launch with grid barriers between its steps: owners
//                       flagged and long duplicates compared with their owner (a 64-bit hash
//                       collision fails the batch loudly), capacity check, owners ranked by
//                       position (tile counts of strings and bytes, scan, in-tile scan) -> new ids
//                       in first-occurrence order and arena offsets in the same order, arena
//                       written through shared memory, ids published, duplicates resolved, owners
//                       reset, the batch's message-start bits cleared. A steady-state batch (no
//                       pending token) only clears the bits.
// Byte-stream work, HBM/latency-bound; no tensor cores.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "pool.cuh"

namespace cg = cooperative_groups;

struct sfkv_interner {
  int32_t device = 0;
  int64_t slots_n = 0;   // power of two
  int64_t arena_cap = 0;
  int64_t max_ids = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t aux = nullptr;  // request offsets run here beside the emit pass
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  struct TSlot* slots = nullptr;
  int64_t* owner = nullptr;       // per slot: lowest claiming token of the current batch
  uint8_t* arena = nullptr;
  int64_t* id_off = nullptr;      // id -> arena offset
  int32_t* id_len = nullptr;
  unsigned long long* ctr = nullptr;  // [0] ids, [1] arena cursor, [2] error flag, [3..5] batch
  uint8_t* tnew = nullptr;         // per-token owner flags, zero between batches
  size_t tnew_cap = 0;
  unsigned long long* ctr_host = nullptr;
  sfkv::Scratch scratch;
  sfkv::Scratch io;
  sfkv::Scratch mbits;  // message-start bitmap: all zero between batches (each batch clears its bits)
};

struct TSlot {
  unsigned long long key;  // 0 = empty
  uint32_t id;             // TOK_PENDING while a batch claim is unresolved
  uint32_t pad;
};

namespace sfkv {

constexpr uint32_t TOK_PENDING = 0xffffffffu;
#ifndef SFKV_TOK_CHUNK_THREADS
#define SFKV_TOK_CHUNK_THREADS 128
#endif
// 2 KiB chunks: 128 threads, 16 bytes (one 16-B load) each (measured: 1 KiB 0.419 ms, 2 KiB 0.367,
// 4 KiB 0.380, 8 KiB 0.465 per C2 batch)
constexpr int CHUNK_THREADS = SFKV_TOK_CHUNK_THREADS;
constexpr int CHUNK = CHUNK_THREADS * 16;
constexpr int RANK_TILE = 1024;     // tokens per CTA tile of the rank pass (256 threads x 4)
enum : int { TERR_COLLISION = 1, TERR_ARENA = 2, TERR_IDS = 4, TERR_TABLE = 8 };
// ctr: [0] ids, [1] arena cursor, [2] error, [3] new bytes, [4] pending, [5] new ids (batch)

__device__ __forceinline__ bool is_space(uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// 4 bytes -> 4-bit mask (bit j = byte j is a C-locale space: 0x20 or 0x09..0x0D). Exact per-byte
// SWAR with no borrow or carry crossing a byte (the high bit is cleared before each add):
//   ge9 / ge14: (b & 0x7F) + (0x80 - 9 / 14) sets bit 7 iff b & 0x7F >= 9 / 14
//   eq20:       ((b & 0x7F) ^ 0x20) + 0x7F leaves bit 7 clear iff the byte is 0x20
// bytes >= 0x80 are never spaces. (The __vcmp*4 intrinsics are emulated on sm_100: ~3x the
// instructions; the count pass was issue-bound on them.)
// bit 7 of every byte of w that is a C-locale space (the SWAR test below, uncompacted)
__device__ __forceinline__ uint32_t space_hi4(uint32_t w) {
  const uint32_t lo7 = w & 0x7F7F7F7Fu;
  const uint32_t ge9 = lo7 + 0x77777777u, ge14 = lo7 + 0x72727272u;
  const uint32_t ne20 = (lo7 ^ 0x20202020u) + 0x7F7F7F7Fu;
  return ((ge9 & ~ge14) | ~ne20) & ~w & 0x80808080u;
}
__device__ __forceinline__ uint32_t space_mask4(uint32_t w) {
  return (((space_hi4(w) >> 7) * 0x01020408u) >> 24) & 0xFu;
}
// 16 bytes -> 16-bit space mask with one multiply per two words: the hi bits of word x at 8j and
// of word y at 8j + 4 gather into bits 24-27 / 28-31 of the product (no colliding partial products,
// so no carries).
__device__ __forceinline__ uint32_t space_bits16(uint4 v) {
  const uint32_t lo = (((space_hi4(v.x) >> 7) | (space_hi4(v.y) >> 3)) * 0x01020408u) >> 24;
  const uint32_t hi = (((space_hi4(v.z) >> 7) | (space_hi4(v.w) >> 3)) * 0x01020408u) >> 24;
  return lo | (hi << 8);
}

// Table keys: tokens of <= 7 bytes are their own key (tag bit 63 | length | bytes): exact, no
// verification. Longer tokens key on a 63-bit hash and are verified against the arena / owner.
__device__ __forceinline__ unsigned long long tok_key(const uint8_t* p, int len) {
  if (len <= 7) {
    unsigned long long w = 0;
    for (int k = 0; k < len; ++k) w |= (unsigned long long)p[k] << (8 * k);
    return (1ull << 63) | ((unsigned long long)len << 56) | w;
  }
  unsigned long long h = 0x9E3779B97F4A7C15ull ^ (unsigned long long)len;
  int i = 0;
  for (; i + 8 <= len; i += 8) {
    unsigned long long w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) w |= (unsigned long long)p[i + k] << (8 * k);
    h = mix64(h + w * 0xD6E8FEB86659FD93ull);
  }
  if (i < len) {
    unsigned long long w = 0;
    for (int k = 0; i + k < len; ++k) w |= (unsigned long long)p[i + k] << (8 * k);
    h = mix64(h + w * 0xD6E8FEB86659FD93ull);
  }
  h = mix64(h) & ~(1ull << 63);
  return h ? h : 1;
}

// Home slot: the top log2(slots) bits of a Fibonacci hash (key x 2^64/phi). A 32-bit fold
// (lo ^ hi) was measured 2x slower: structured words (digit runs) collide in the fold.
__device__ __forceinline__ uint64_t home_slot(unsigned long long key, int shift) {
  return (key * 0x9E3779B97F4A7C15ull) >> shift;
}

// tok_key of a token staged in shared memory at byte s0 (the buffer is 8-B aligned and readable
// 16 bytes past the token): the same key, read as 8-byte words (two aligned loads + a funnel
// shift each) instead of byte by byte.
__device__ __forceinline__ unsigned long long ld8_smem(const uint8_t* sb, int pos) {
  const int a8 = pos & ~7, b8 = (pos & 7) * 8;
  const unsigned long long lo = *reinterpret_cast<const unsigned long long*>(sb + a8);
  const unsigned long long hi = *reinterpret_cast<const unsigned long long*>(sb + a8 + 8);
  return b8 ? (lo >> b8) | (hi << (64 - b8)) : lo;
}
__device__ __forceinline__ unsigned long long tok_key_smem(const uint8_t* sb, int s0, int len) {
  if (len <= 7) return (1ull << 63) | ((unsigned long long)len << 56) | (ld8_smem(sb, s0) & ((1ull << (8 * len)) - 1));
  unsigned long long h = 0x9E3779B97F4A7C15ull ^ (unsigned long long)len;
  int i = 0;
  for (; i + 8 <= len; i += 8) h = mix64(h + ld8_smem(sb, s0 + i) * 0xD6E8FEB86659FD93ull);
  if (i < len) h = mix64(h + (ld8_smem(sb, s0 + i) & ((1ull << (8 * (len - i))) - 1)) * 0xD6E8FEB86659FD93ull);
  h = mix64(h) & ~(1ull << 63);
  return h ? h : 1;
}

struct TokArgs {
  int64_t n_req;
  const int64_t* req_msg_off;
  const int64_t* msg_off;
  int64_t n_msg;
  const uint8_t* text;
  int64_t n_bytes;
  uint32_t* mbits;       // message-start bitmap
  uint16_t* spbits;      // [nchunks * CHUNK / 16] space masks per 16-byte window (count pass)
  int64_t* chunk_off;    // [nchunks + 1]
  int64_t* tstart;       // [token bound] byte start of pending tokens (claims / duplicates)
  int64_t* pend_t;       // pending tokens (claims / duplicates of new strings)
  int64_t* pend_slot;    // [token bound] slot of a pending token (by token index)
  uint8_t* tnew;         // [token bound] owner flags (kept zero between batches)
  int64_t* tile_cnt;     // [rank tiles + 1]
  int64_t* tile_bytes;   // [rank tiles + 1] bytes of the tile's new strings (arena offsets)
  int32_t* tlen;         // [token bound] byte length of pending tokens
  int64_t* tok_off;      // out [n_req + 1]
  uint32_t* tok;         // out
  int64_t* n_tokens;     // out (device scalar)
  int64_t n_rank_tiles;
  // interner
  TSlot* slots;
  uint64_t mask;
  int slot_shift;  // 64 - log2(slots): home slot = the top bits of key * golden ratio
  int64_t* owner;
  uint8_t* arena;
  int64_t arena_cap;
  int64_t* id_off;
  int32_t* id_len;
  int64_t max_ids;
  unsigned long long* ctr;
};

__global__ void msg_mark_kernel(TokArgs a) {
  pdl_enter();
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < a.n_msg; m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = a.msg_off[m];
    if (i < a.n_bytes) atomicOr(a.mbits + (i >> 5), 1u << (i & 31));
  }
}

// 16-bit mask of token starts among bytes [base, base + 16) (base 16-aligned): a non-space byte
// whose predecessor is a space or which starts a message (or the text).
__device__ __forceinline__ uint32_t start_mask16(const TokArgs& a, int64_t base) {
  if (base >= a.n_bytes) return 0;
  uint32_t sp;
  if (base + 16 <= a.n_bytes) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.text + base));
    sp = space_mask4(v.x) | (space_mask4(v.y) << 4) | (space_mask4(v.z) << 8) | (space_mask4(v.w) << 12);
  } else {
    sp = 0xffffu;
    for (int j = 0; base + j < a.n_bytes; ++j)
      if (!is_space(a.text[base + j])) sp &= ~(1u << j);
  }
  const uint32_t prev_sp = base == 0 ? 1u : (is_space(a.text[base - 1]) ? 1u : 0u);
  const uint32_t ms = (__ldg(a.mbits + (base >> 5)) >> (base & 31)) & 0xffffu;
  return ~sp & (((sp << 1) | prev_sp) | ms) & 0xffffu;
}

// One warp per chunk: every lane's CHUNK / 512 windows of 16 bytes are loaded together (predicated
// loads, no branch between them), the previous byte of a window comes from the neighbouring lane
// (or the previous round's last lane) instead of another load, then a warp reduction.
constexpr int COUNT_WARPS = 8;
#ifndef SFKV_TOKOFF_FORK
#define SFKV_TOKOFF_FORK 1
#endif
// One warp per chunk. A full chunk (every chunk but the text's last) takes a fast path with
// chunk-relative 32-bit offsets and no bounds checks (the count pass is issue-bound: 64-bit window
// arithmetic and per-window bounds tests were half its instructions); the last chunk takes the
// generic path (bytes past the text are spaces). Every window's compact 16-bit space mask is
// stored for the emit pass, which builds its boundary bitmap and start masks from those words.
__device__ __forceinline__ int count_windows(const uint4* v, const uint32_t* mw, int lane, uint32_t prev_last,
                                             uint16_t* spo) {
  constexpr int KW = CHUNK / 512;
  int c = 0;
#pragma unroll
  for (int k = 0; k < KW; ++k) {
    const uint32_t sp = space_bits16(v[k]);
    spo[32 * k] = (uint16_t)sp;
    uint32_t prev = __shfl_up_sync(0xffffffffu, sp >> 15, 1);
    if (lane == 0) prev = prev_last;
    prev_last = __shfl_sync(0xffffffffu, sp >> 15, 31);
    c += __popc(~sp & (((sp << 1) | prev) | mw[k]) & 0xffffu);
  }
  return c;
}
__global__ void __launch_bounds__(COUNT_WARPS * 32) chunk_count_kernel(TokArgs a, int64_t* counts, int64_t nchunks) {
  pdl_enter();
  constexpr int KW = CHUNK / 512;
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * COUNT_WARPS + (threadIdx.x >> 5);
  if (chunk >= nchunks) return;
  const int64_t c0 = chunk * CHUNK;
  const uint64_t pol = l2_policy_first();
  uint4 v[KW];
  uint32_t mw[KW];  // the window's 16 message-start bits
  uint16_t* spo = a.spbits + (c0 >> 4) + lane;
  const uint32_t prev0 = c0 == 0 ? 1u : (uint32_t)is_space(a.text[c0 - 1]);  // before lane 0, round 0
  int c;
  if (c0 + CHUNK <= a.n_bytes) {
    const uint8_t* tx = a.text + c0 + 16 * lane;
    const uint32_t* mb = a.mbits + (c0 >> 5) + (lane >> 1);
    const int sh = (lane & 1) * 16;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      v[k] = ld_nc16_hint(tx + 512 * k, pol);  // streamed: evict_first
      mw[k] = __ldg(mb + 16 * k);
    }
#pragma unroll
    for (int k = 0; k < KW; ++k) mw[k] = (mw[k] >> sh) & 0xffffu;
    c = count_windows(v, mw, lane, prev0, spo);
  } else {
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int64_t w = c0 + 512 * k + 16 * lane;
      v[k] = make_uint4(0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u);
      if (w + 16 <= a.n_bytes) {
        v[k] = ld_nc16_hint(a.text + w, pol);
      } else if (w < a.n_bytes) {  // the text's last, partial window: bytes past the end are spaces
        uint32_t q[4] = {0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u};
        for (int j = 0; w + j < a.n_bytes; ++j)
          q[j >> 2] = (q[j >> 2] & ~(0xffu << (8 * (j & 3)))) | ((uint32_t)a.text[w + j] << (8 * (j & 3)));
        v[k] = make_uint4(q[0], q[1], q[2], q[3]);
      }
      // past the text: no starts (all spaces, no message bits)
      mw[k] = w < a.n_bytes ? (__ldg(a.mbits + (w >> 5)) >> (w & 31)) & 0xffffu : 0u;
    }
    c = count_windows(v, mw, lane, prev0, spo);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if (lane == 0) counts[chunk] = c;
}

struct ChunkCount {
  const int64_t* counts;
  __device__ int64_t operator()(int64_t c) const { return counts[c]; }
};

__device__ __forceinline__ bool bytes_equal(const uint8_t* x, const uint8_t* y, int len) {
  for (int i = 0; i < len; ++i)
    if (x[i] != y[i]) return false;
  return true;
}
__device__ __forceinline__ bool is_mstart(const TokArgs& a, int64_t i) {
  return (a.mbits[i >> 5] >> (i & 31)) & 1u;
}
__device__ bool probe_token(const TokArgs& a, int64_t t, int64_t start, const uint8_t* p, int len);
__device__ bool probe_key(const TokArgs& a, int64_t t, int64_t start, unsigned long long key, const uint8_t* p,
                          int len);

// Token starts of the chunk in order (CTA scan) into a shared list, and every token probed right
// here, one token per thread (no per-thread token-count divergence): the chunk's 2 KiB plus OVER
// bytes of the next chunk and their message-start bits are staged in shared memory with a
// chunk-wide boundary bitmap (space | message start), so a token's end is the next set bit and its
// key comes from the staged bytes (tokens running past the staged window fall back to global reads).
#ifndef SFKV_TOK_OVER
#define SFKV_TOK_OVER 256
#endif
constexpr int OVER = SFKV_TOK_OVER;
#ifndef SFKV_EMIT_MINB
#define SFKV_EMIT_MINB 16
#endif
__global__ void __launch_bounds__(CHUNK_THREADS, SFKV_EMIT_MINB) chunk_emit_kernel(TokArgs a) {
  pdl_enter();
  using BS = cub::BlockScan<int, CHUNK_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ __align__(16) uint8_t sb[CHUNK + OVER + 16];  // + 16: word reads past a token's end
  __shared__ uint32_t sbits[(CHUNK + OVER) / 32];
  const int64_t c0 = (int64_t)blockIdx.x * CHUNK;
  const int64_t lim = a.n_bytes - c0;  // valid staged bytes: [0, min(lim, CHUNK + OVER))
  __shared__ uint16_t slist[CHUNK];
  __shared__ uint32_t sbnd[(CHUNK + OVER) / 32 + 1];
  __shared__ uint32_t s_sp[CHUNK / 32 + 1];  // [0]: the word before the chunk
  constexpr int WORDS = (CHUNK + OVER) / 32;
  const int tid = threadIdx.x;
  const uint64_t pol = l2_policy_first();
  // stage the chunk (16 B per thread) and OVER bytes of the next one (OVER / 16 threads), the
  // count pass's space words and the message-start words; boundary bitmap = space | message start
  const uint32_t* sp32 = reinterpret_cast<const uint32_t*>(a.spbits) + (c0 >> 5);
  const uint32_t* mb32 = a.mbits + (c0 >> 5);
  if (lim >= CHUNK + OVER) {  // every staged byte inside the text (all chunks but the last one or two)
    const uint8_t* tx = a.text + c0;
    *reinterpret_cast<uint4*>(sb + tid * 16) = ld_nc16_hint(tx + tid * 16, pol);
    if (tid < OVER / 16) *reinterpret_cast<uint4*>(sb + CHUNK + tid * 16) = ld_nc16_hint(tx + CHUNK + tid * 16, pol);
    if (tid < WORDS) {
      const uint32_t ms = mb32[tid], sp = sp32[tid];
      sbits[tid] = ms;
      sbnd[tid] = sp | ms;
      if (tid < CHUNK / 32) s_sp[tid + 1] = sp;
    } else if (tid == WORDS) {
      s_sp[0] = c0 == 0 ? 0x80000000u : sp32[-1];
    }
  } else {  // bytes past the text are staged as spaces, words past it as all boundaries
    const int64_t base = c0 + (int64_t)tid * 16;
    if (base + 16 <= a.n_bytes) {
      *reinterpret_cast<uint4*>(sb + tid * 16) = ld_nc16_hint(a.text + base, pol);
    } else {
      for (int j = 0; j < 16; ++j) sb[tid * 16 + j] = base + j < a.n_bytes ? a.text[base + j] : ' ';
    }
    if (tid < OVER / 16) {
      const int64_t ob = c0 + CHUNK + tid * 16;
      if (ob + 16 <= a.n_bytes) {
        *reinterpret_cast<uint4*>(sb + CHUNK + tid * 16) = ld_nc16_hint(a.text + ob, pol);
      } else {
        for (int j = 0; j < 16; ++j) sb[CHUNK + tid * 16 + j] = ob + j < a.n_bytes ? a.text[ob + j] : ' ';
      }
    }
    if (tid < WORDS) {
      const bool in = c0 + tid * 32 < a.n_bytes;
      const uint32_t ms = in ? mb32[tid] : 0xffffffffu, sp = in ? sp32[tid] : 0xffffffffu;
      sbits[tid] = ms;
      sbnd[tid] = sp | ms;
      if (tid < CHUNK / 32) s_sp[tid + 1] = sp;
    } else if (tid == WORDS) {
      s_sp[0] = c0 == 0 ? 0x80000000u : sp32[-1];
    }
  }
  constexpr int PW = CHUNK / 32;  // pending bitmap words (<= CHUNK tokens: every byte may start a message)
  __shared__ uint32_t s_pend[PW];
  __shared__ int s_any_pend;
  __shared__ unsigned long long s_pbase;
  if (tid < PW) s_pend[tid] = 0u;
  if (tid == 0) {
    s_any_pend = 0;
    sbnd[WORDS] = 0xffffffffu;  // past the staged bytes: all boundaries (end windows)
  }
  __syncthreads();
  // the thread's token starts (non-space after a space or at a message start) from the staged words
  uint32_t m = 0;
  if (tid * 16 < lim) {
    const int sh = (tid & 1) * 16;
    const uint32_t spw = s_sp[(tid >> 1) + 1];
    const uint32_t sp = (spw >> sh) & 0xffffu, ms = (sbits[tid >> 1] >> sh) & 0xffffu;
    const uint32_t prev = (tid & 1) ? (spw >> 15) & 1u : s_sp[tid >> 1] >> 31;
    m = ~sp & ((sp << 1) | prev | ms) & 0xffffu;
  }
  int excl, total;
  BS(tmp).ExclusiveSum(__popc(m), excl, total);
  {
    int k = excl;
    for (uint32_t mm = m; mm; mm &= mm - 1) slist[k++] = (uint16_t)(threadIdx.x * 16 + __ffs(mm) - 1);
  }
  __syncthreads();
  // loop invariants in 32-bit form (the loop runs at the 32-register cap: 64-bit invariants get
  // rematerialised every iteration)
  const int stage_end = (int)(lim < CHUNK + OVER ? lim : CHUNK + OVER);
  const bool text_ends_here = lim <= CHUNK + OVER;  // bytes past the text are staged as spaces
  const int64_t tb0 = a.chunk_off[blockIdx.x];
  const uint32_t* sb32 = reinterpret_cast<const uint32_t*>(sb);
  for (int i = threadIdx.x; i < total; i += CHUNK_THREADS) {
    const int s0 = slist[i];
    bool pend;
    // the token's end: the first boundary bit after s0, from a 32-bit funnel window of the
    // bitmap (one step for tokens of up to 32 bytes; longer ones walk on)
    int w = (s0 + 1) >> 5;
    uint32_t bits = __funnelshift_r(sbnd[w], sbnd[w + 1], (s0 + 1) & 31);
    int e;
    if (bits) {
      e = s0 + __ffs(bits);
    } else {
      e = CHUNK + OVER;
      for (int p = s0 + 33; p < stage_end; p = (p & ~31) + 32) {
        const uint32_t wb = sbnd[p >> 5] & (~0u << (p & 31));
        if (wb) {
          e = (p & ~31) + __ffs(wb) - 1;
          bits = 1u;
          break;
        }
      }
    }
    if (e < stage_end || (bits && text_ends_here)) {
      const int len = e - s0;
      if (len <= 7) {
        // the token's bytes from three aligned 32-bit words and two funnel shifts
        const int a4 = s0 >> 2, sh = (s0 & 3) * 8;
        const uint32_t w0 = sb32[a4], w1 = sb32[a4 + 1], w2 = sb32[a4 + 2];
        // one 64-bit byte mask (len <= 7: at most 56 bits) and the tag / length OR-ed into the
        // high word: no per-length selects
        const unsigned long long msk = ~(~0ull << (8 * len));
        const uint32_t lo = __funnelshift_r(w0, w1, sh) & (uint32_t)msk;
        const uint32_t hi = (__funnelshift_r(w1, w2, sh) & (uint32_t)(msk >> 32)) | 0x80000000u | ((uint32_t)len << 24);
        pend = probe_key(a, tb0 + i, c0 + s0, ((unsigned long long)hi << 32) | lo, sb + s0, len);
      } else {
        pend = probe_key(a, tb0 + i, c0 + s0, tok_key_smem(sb, s0, len), sb + s0, len);
      }
    } else {
      int64_t g = c0 + s0 + 1;
      while (g < a.n_bytes && !is_space(a.text[g]) && !is_mstart(a, g)) ++g;
      pend = probe_token(a, tb0 + i, c0 + s0, a.text + c0 + s0, (int)(g - (c0 + s0)));
    }
    if (pend) {
      atomicOr(&s_pend[i >> 5], 1u << (i & 31));
      s_any_pend = 1;
    }
  }
  // pending tokens join the batch list with one global atomic per chunk (a cold batch makes every
  // token pending: per-token atomics on one counter serialise in one L2 slice)
  __syncthreads();
  if (!s_any_pend) return;
  const int nw = (total + 31) / 32;
  int c = threadIdx.x < nw ? __popc(s_pend[threadIdx.x]) : 0, ex;
  BS(tmp).ExclusiveSum(c, ex);
  if (threadIdx.x == nw - 1) s_pbase = atomicAdd(a.ctr + 4, (unsigned long long)(ex + c));
  __syncthreads();
  if (threadIdx.x < nw) {
    unsigned long long j = s_pbase + ex;
    for (uint32_t m = s_pend[threadIdx.x]; m; m &= m - 1) a.pend_t[j++] = tb0 + threadIdx.x * 32 + __ffs(m) - 1;
  }
}

// Probe one token (bytes p[0..len), position t): published strings resolve here (short keys
// exactly, long keys verified against the arena); claims and duplicates of this batch's new
// strings go to the pending list.
__device__ bool probe_token(const TokArgs& a, int64_t t, int64_t start, const uint8_t* p, int len) {
  return probe_key(a, t, start, tok_key(p, len), p, len);
}

// (start: the token's byte position, recorded only for pending tokens). Returns true when the
// token is pending (a claim or a duplicate of this batch's new string): its start, length and
// slot are recorded by token index and the caller appends it to the pending list.
__device__ bool probe_key(const TokArgs& a, int64_t t, int64_t start, unsigned long long key, const uint8_t* p,
                          int len) {
  // home slot by Fibonacci hashing: the top bits of key x 2^64/phi spread the raw bytes of short
  // keys (one multiply; mix64 here cost 7.5 % of the batch, the probe loop is issue-bound)
  uint64_t sl = home_slot(key, a.slot_shift);
  int64_t found = -1;
  uint32_t id = TOK_PENDING;
  for (uint64_t probes = 0; probes <= a.mask; ++probes) {
    TSlot* q = a.slots + sl;
    // key and id in one 16-B load: ids change only between batches (a slot claimed during this
    // batch keeps TOK_PENDING until the publish pass), so the pair is consistent
    const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(q);
    unsigned long long k = w.x;
    uint32_t qid = (uint32_t)w.y;
    if (k == 0) {
      k = atomicCAS(&q->key, 0ull, key);
      if (k == 0) k = key;  // claimed: its id stays TOK_PENDING until published
      qid = TOK_PENDING;    // (a slot claimed by anyone during this batch is pending)
    }
    if (k == key) {
      found = (int64_t)sl;
      id = qid;
      break;
    }
    sl = (sl + 1) & a.mask;
  }
  if (found < 0) {
    atomicOr(a.ctr + 2, (unsigned long long)TERR_TABLE);
    return false;
  }
  if (id != TOK_PENDING) {  // published before this batch
    if (!(key >> 63) && (a.id_len[id] != len || !bytes_equal(p, a.arena + a.id_off[id], len)))
      atomicOr(a.ctr + 2, (unsigned long long)TERR_COLLISION);
    a.tok[t] = id;
    return false;
  }
  a.tstart[t] = start;
  a.tlen[t] = len;
  a.pend_slot[t] = found;
  atomicMin(reinterpret_cast<unsigned long long*>(a.owner + found), (unsigned long long)t);
  return true;
}





// Owners ranked by position get consecutive ids and consecutive arena bytes, so a tile's new
// strings form one contiguous arena range, and their source bytes one contiguous text range (from
// the first owner's start to the last owner's end). Both are staged in shared memory: the text
// range is read with coalesced loads, each owner's bytes are moved inside shared memory, and the
// arena range is written with coalesced stores (a tile whose ranges exceed the staging buffers
// copies byte by byte from global memory instead).
constexpr int PUB_TXT = 20 * 1024, PUB_OUT = 20 * 1024;
struct PubSmem {
  typename cub::BlockScan<int2, 256>::TempStorage scan;
  uint8_t txt[PUB_TXT];
  uint8_t out[PUB_OUT];
  int64_t lo, hi;
  int2 agg;
};

__device__ void rank_publish_tile(const TokArgs& a, int64_t tile, int64_t nt, PubSmem& S) {
  using BS = cub::BlockScan<int2, 256>;
  const int64_t t0 = tile * RANK_TILE;
  constexpr int PT = RANK_TILE / 256;
  const int64_t tb = t0 + (int64_t)threadIdx.x * PT;  // blocked
  int2 c = make_int2(0, 0);
  uint32_t f = 0;
  int lens[PT];
  int64_t ts[PT];
#pragma unroll
  for (int k = 0; k < PT; ++k) {
    lens[k] = 0;
    ts[k] = 0;
    if (tb + k < nt && a.tnew[tb + k]) {
      f |= 1u << k;
      lens[k] = a.tlen[tb + k];
      ts[k] = a.tstart[tb + k];
      c.x += 1;
      c.y += lens[k];
    }
  }
  int2 ex, agg;
  BS(S.scan).ExclusiveScan(c, ex, make_int2(0, 0), [](int2 x, int2 y) { return make_int2(x.x + y.x, x.y + y.y); },
                           agg);
  if (agg.x == 0) return;  // uniform: no new string in this tile
  // the tile's first owner (global rank 0 in the tile) and last owner fix the text range
  int64_t first = -1, last_end = -1;
#pragma unroll
  for (int k = 0; k < PT; ++k)
    if ((f >> k) & 1u) {
      if (first < 0) first = ts[k];
      last_end = ts[k] + lens[k];
    }
  if (f && ex.x == 0) S.lo = first;
  if (f && ex.x + c.x == agg.x) S.hi = last_end;
  __syncthreads();
  const int64_t lo = S.lo, hi = S.hi;
  const int64_t base = (int64_t)a.ctr[1] + a.tile_bytes[tile];  // arena offset of the tile's first byte
  int64_t id = (int64_t)a.ctr[0] + a.tile_cnt[tile] + ex.x;
  const bool staged = hi - lo <= PUB_TXT && agg.y <= PUB_OUT;
  if (staged) {
    for (int64_t i = threadIdx.x; i < hi - lo; i += 256) S.txt[i] = a.text[lo + i];
    __syncthreads();
  }
  int off = ex.y;  // tile-relative arena offset of this thread's first string
#pragma unroll
  for (int k = 0; k < PT; ++k) {
    if (!((f >> k) & 1u)) continue;
    const int64_t t = tb + k;
    const int len = lens[k];
    a.tnew[t] = 0;
    if (staged) {
      const uint8_t* src = S.txt + (ts[k] - lo);
      for (int i = 0; i < len; ++i) S.out[off + i] = src[i];
    } else {
      const uint8_t* src = a.text + ts[k];
      uint8_t* dst = a.arena + base + off;
      for (int i = 0; i < len; ++i) dst[i] = src[i];
    }
    a.id_off[id] = base + off;
    a.id_len[id] = len;
    a.tok[t] = (uint32_t)id;
    ++id;
    off += len;
  }
  if (staged) {
    __syncthreads();
    for (int i = threadIdx.x; i < agg.y; i += 256) a.arena[base + i] = S.out[i];
  }
}




// tok_off[r]: tokens before request r's first byte b = its chunk's offset + the token starts in
// [chunk start, b) (one warp per request, every load of the <= 2 KiB prefix in flight at once).
__global__ void req_tokoff_kernel(TokArgs a) {
  pdl_enter();
  constexpr int KW = CHUNK / 512;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r <= a.n_req; r += warps) {
    const int64_t b = r < a.n_req ? a.msg_off[a.req_msg_off[r]] : a.n_bytes;
    const int64_t c = b / CHUNK;
    const int64_t c0 = c * CHUNK;
    // every window's loads issued together (predicated), the previous byte from the neighbouring
    // lane, as in the count pass
    const int64_t coff = a.chunk_off[c];
    uint4 v[KW];
    uint32_t mw[KW];
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int64_t w = c0 + 512 * k + 16 * lane;
      v[k] = make_uint4(0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u);
      if (w < b && w + 16 <= a.n_bytes) v[k] = __ldg(reinterpret_cast<const uint4*>(a.text + w));
      mw[k] = w < b ? __ldg(a.mbits + (w >> 5)) : 0u;
    }
    uint32_t prev_last = c0 == 0 ? 1u : (uint32_t)is_space(a.text[c0 - 1]);
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < KW; ++k) {
      const int64_t w = c0 + 512 * k + 16 * lane;
      if (w < b && w + 16 > a.n_bytes) {  // the text's last, partial window
        uint32_t q[4] = {0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u};
        for (int j = 0; w + j < a.n_bytes; ++j)
          q[j >> 2] = (q[j >> 2] & ~(0xffu << (8 * (j & 3)))) | ((uint32_t)a.text[w + j] << (8 * (j & 3)));
        v[k] = make_uint4(q[0], q[1], q[2], q[3]);
      }
      const uint32_t sp = space_mask4(v[k].x) | (space_mask4(v[k].y) << 4) | (space_mask4(v[k].z) << 8) |
                          (space_mask4(v[k].w) << 12);
      const uint32_t last = (sp >> 15) & 1u;
      uint32_t prev = __shfl_up_sync(0xffffffffu, last, 1);
      if (lane == 0) prev = prev_last;
      prev_last = __shfl_sync(0xffffffffu, last, 31);
      if (w < b) {
        uint32_t m = ~sp & (((sp << 1) | prev) | ((mw[k] >> (w & 31)) & 0xffffu)) & 0xffffu;
        if (b - w < 16) m &= (1u << (b - w)) - 1u;
        cnt += __popc(m);
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if (lane == 0) a.tok_off[r] = coff + cnt;
  }
}



// The pending phase of a batch (resolve → capacity check → rank count / scan / publish → final →
// duplicates → owner reset + message-start bits → counters) as ONE cooperative launch with grid
// barriers between the steps. A steady-state batch has no pending token: the kernel clears the
// batch's message-start bits and returns — one launch where eight early-exiting kernels used to
// run back to back.
__global__ void __launch_bounds__(256) tok_pending_kernel(TokArgs a) {
  namespace cgn = cooperative_groups;
  using BRL = cub::BlockReduce<longlong2, 256>;
  using BRI = cub::BlockReduce<int2, 256>;
  using BSL = cub::BlockScan<longlong2, 256>;
  union PendTmp {
    typename BRL::TempStorage rl;
    typename BRI::TempStorage ri;
    typename BSL::TempStorage sl;
  };
  __shared__ PubSmem S;
  __shared__ PendTmp T;
  __shared__ longlong2 s_carry;
  pdl_enter();
  cgn::grid_group grid = cgn::this_grid();
  const int64_t np = (int64_t)a.ctr[4];
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  auto clear_mbits = [&]() {
    for (int64_t m = gtid; m < a.n_msg; m += gstride) {
      const int64_t i = a.msg_off[m];
      if (i < a.n_bytes) a.mbits[i >> 5] = 0u;
    }
  };
  if (np == 0) {  // uniform: no new string and no duplicate of one (the counters are already zero)
    clear_mbits();
    return;
  }
  // 1. owners flagged, duplicates of long keys compared with their owner; CTA-reduced counters
  {
    longlong2 own = make_longlong2(0, 0);
    for (int64_t j = gtid; j < np; j += gstride) {
      const int64_t t = a.pend_t[j], sl = a.pend_slot[t];
      const int len = a.tlen[t];
      const int64_t o = a.owner[sl];
      if (o == t) {
        a.tnew[t] = 1;
        own.x += 1;
        own.y += len;
      } else if (!(a.slots[sl].key >> 63) && !bytes_equal(a.text + a.tstart[t], a.text + a.tstart[o], len)) {
        atomicOr(a.ctr + 2, (unsigned long long)TERR_COLLISION);
      }
    }
    own = BRL(T.rl).Reduce(own, [](longlong2 x, longlong2 y) { return make_longlong2(x.x + y.x, x.y + y.y); });
    if (threadIdx.x == 0 && own.x) {
      atomicAdd(a.ctr + 5, (unsigned long long)own.x);
      atomicAdd(a.ctr + 3, (unsigned long long)own.y);
    }
  }
  grid.sync();
  // 2. capacity check before anything is published
  if (gtid == 0 && !a.ctr[2]) {
    if ((int64_t)(a.ctr[0] + a.ctr[5]) > a.max_ids) a.ctr[2] |= TERR_IDS;
    if ((int64_t)(a.ctr[1] + a.ctr[3]) > a.arena_cap) a.ctr[2] |= TERR_ARENA;
  }
  grid.sync();
  const bool failed = a.ctr[2] != 0;
  const int64_t nt = *a.n_tokens;
  const int64_t ntiles = (nt + RANK_TILE - 1) / RANK_TILE;
  if (!failed) {
    // 3. new strings and their bytes per rank tile
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t t0 = tile * RANK_TILE;
      int2 c = make_int2(0, 0);
      for (int k = 0; k < RANK_TILE / 256; ++k) {
        const int64_t t = t0 + (int64_t)k * 256 + threadIdx.x;
        if (t < nt && a.tnew[t]) {
          c.x += 1;
          c.y += a.tlen[t];
        }
      }
      c = BRI(T.ri).Reduce(c, [](int2 x, int2 y) { return make_int2(x.x + y.x, x.y + y.y); });
      if (threadIdx.x == 0) {
        a.tile_cnt[tile] = c.x;
        a.tile_bytes[tile] = c.y;
      }
      __syncthreads();
    }
    grid.sync();
    // 4. exclusive scan of (count, bytes) over the tiles (one CTA)
    if (blockIdx.x == 0) {
      auto add = [](longlong2 x, longlong2 y) { return make_longlong2(x.x + y.x, x.y + y.y); };
      if (threadIdx.x == 0) s_carry = make_longlong2(0, 0);
      __syncthreads();
      for (int64_t b = 0; b < ntiles; b += 256) {
        const int64_t i = b + threadIdx.x;
        longlong2 v = i < ntiles ? make_longlong2(a.tile_cnt[i], a.tile_bytes[i]) : make_longlong2(0, 0), ex, tot;
        BSL(T.sl).ExclusiveScan(v, ex, make_longlong2(0, 0), add, tot);
        if (i < ntiles) {
          a.tile_cnt[i] = s_carry.x + ex.x;
          a.tile_bytes[i] = s_carry.y + ex.y;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry = add(s_carry, tot);
        __syncthreads();
      }
    }
    grid.sync();
    // 5. ids and arena bytes
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      rank_publish_tile(a, tile, nt, S);
      __syncthreads();
    }
  }
  grid.sync();
  // 6. owners publish their ids (or, when the batch failed, their claims are rolled back)
  for (int64_t j = gtid; j < np; j += gstride) {
    const int64_t t = a.pend_t[j], sl = a.pend_slot[t];
    if (a.owner[sl] != t) continue;
    if (failed) {
      a.slots[sl].key = 0;
      a.tnew[t] = 0;
    } else {
      a.slots[sl].id = a.tok[t];
    }
  }
  grid.sync();
  // 7. duplicates of new strings read the published ids
  for (int64_t j = gtid; j < np; j += gstride) {
    const int64_t t = a.pend_t[j], sl = a.pend_slot[t];
    if (a.owner[sl] != t) a.tok[t] = a.slots[sl].id;
  }
  grid.sync();
  // 8. owners reset, the batch's message-start bits cleared, counters advanced
  for (int64_t j = gtid; j < np; j += gstride) a.owner[a.pend_slot[a.pend_t[j]]] = INT64_MAX;
  clear_mbits();
  if (gtid == 0) {
    if (!failed) {
      a.ctr[0] += a.ctr[5];
      a.ctr[1] += a.ctr[3];
    }
    a.ctr[3] = a.ctr[4] = a.ctr[5] = 0;
  }
}

__global__ void copy_count_kernel(const int64_t* chunk_off, int64_t nchunks, int64_t* n_tokens) {
  pdl_enter();
  *n_tokens = chunk_off[nchunks];
}

static int sm_count_k() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Re-insert every published id into a larger table (sfkv_interner_reserve): same keys, same ids.
__global__ void interner_rehash_kernel(TSlot* slots, uint64_t mask, int shift, const uint8_t* arena,
                                       const int64_t* id_off, const int32_t* id_len, int64_t n_ids) {
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < n_ids; id += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = tok_key(arena + id_off[id], id_len[id]);
    uint64_t sl = home_slot(key, shift);
    for (;;) {
      if (atomicCAS(&slots[sl].key, 0ull, key) == 0ull) {
        slots[sl].id = (uint32_t)id;
        break;
      }
      sl = (sl + 1) & mask;
    }
  }
}

__global__ void interner_init_kernel(TSlot* slots, int64_t* owner, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    slots[i].key = 0;
    slots[i].id = TOK_PENDING;
    slots[i].pad = 0;
    owner[i] = INT64_MAX;
  }
}

// Device-pointer batch. tok must hold (n_bytes + n_msg + 1) / 2 ids (a message of L bytes splits
// into at most (L + 1) / 2 tokens); text must be 16-B aligned.
static int tokenize_dev(sfkv_interner* it, int64_t n_req, const int64_t* req_msg_off, int64_t n_msg,
                        const int64_t* msg_off, const uint8_t* text, int64_t n_bytes, int64_t* tok_off,
                        uint32_t* tok, int64_t* n_tokens) {
  if (reinterpret_cast<uintptr_t>(text) & 15) return fail(SFKV_EINVAL, "tokenize: text must be 16-B aligned");
  cudaStream_t st = it->stream;
  const int64_t nchunks = (n_bytes + CHUNK - 1) / CHUNK;
  const int64_t tb = (n_bytes + n_msg + 1) / 2 + 1;  // token bound
  const int64_t nrt = (tb + RANK_TILE - 1) / RANK_TILE;
  const int64_t nwords = n_bytes / 32 + 2;
  Carver cv;
  const size_t o_cnt = cv.take<int64_t>(nchunks + 1),
               o_co = cv.take<int64_t>(nchunks + 1), o_ts = cv.take<int64_t>(tb), o_pt = cv.take<int64_t>(tb),
               o_ps = cv.take<int64_t>(tb), o_tc = cv.take<int64_t>(nrt + 1),
               o_tby = cv.take<int64_t>(nrt + 1), o_tl = cv.take<int32_t>(tb),
               o_tmp = cv.take<int64_t>(scan_scratch_elems(nchunks)),
               o_sp = cv.take<uint32_t>(nchunks * (CHUNK / 32) + 1);
  if (int rc = it->scratch.ensure(cv.off)) return rc;
  if (it->mbits.bytes < nwords * sizeof(uint32_t)) {  // grown: zero once, then kept zero
    if (int rc = it->mbits.ensure(nwords * sizeof(uint32_t))) return rc;
    SFKV_CUDA(cudaMemsetAsync(it->mbits.ptr, 0, it->mbits.bytes, st));
  }
  if ((size_t)tb > it->tnew_cap) {  // owner flags stay zero between batches
    if (it->tnew) cudaFree(it->tnew);
    it->tnew = nullptr;
    it->tnew_cap = 0;
    SFKV_CUDA(cudaMalloc(&it->tnew, (size_t)tb));
    SFKV_CUDA(cudaMemsetAsync(it->tnew, 0, (size_t)tb, st));
    it->tnew_cap = (size_t)tb;
  }
  char* base = it->scratch.as<char>();
  TokArgs a;
  a.n_req = n_req;
  a.req_msg_off = req_msg_off;
  a.msg_off = msg_off;
  a.n_msg = n_msg;
  a.text = text;
  a.n_bytes = n_bytes;
  a.mbits = it->mbits.as<uint32_t>();
  a.spbits = reinterpret_cast<uint16_t*>(base + o_sp);
  a.chunk_off = reinterpret_cast<int64_t*>(base + o_co);
  a.tstart = reinterpret_cast<int64_t*>(base + o_ts);
  a.pend_t = reinterpret_cast<int64_t*>(base + o_pt);
  a.pend_slot = reinterpret_cast<int64_t*>(base + o_ps);
  a.tnew = it->tnew;
  a.tile_cnt = reinterpret_cast<int64_t*>(base + o_tc);
  a.tile_bytes = reinterpret_cast<int64_t*>(base + o_tby);
  a.tlen = reinterpret_cast<int32_t*>(base + o_tl);
  a.tok_off = tok_off;
  a.tok = tok;
  a.n_tokens = n_tokens;
  a.n_rank_tiles = nrt;
  a.slots = it->slots;
  a.mask = (uint64_t)it->slots_n - 1;
  a.slot_shift = 64 - __builtin_ctzll((unsigned long long)it->slots_n);
  a.owner = it->owner;
  a.arena = it->arena;
  a.arena_cap = it->arena_cap;
  a.id_off = it->id_off;
  a.id_len = it->id_len;
  a.max_ids = it->max_ids;
  a.ctr = it->ctr;
  int64_t* counts = reinterpret_cast<int64_t*>(base + o_cnt);
  int64_t* tmp = reinterpret_cast<int64_t*>(base + o_tmp);
  const int sms = sm_count_k();
  // (the bitmap and the batch counters ctr[3..5] were left zero by the previous batch's last kernels)
  if (n_msg > 0) SFKV_CUDA(launch_pdl(msg_mark_kernel, dim3(grid_for(n_msg, 256, sms * 4)), dim3(256), st, a));
  if (nchunks > 0)
    SFKV_CUDA(launch_pdl(chunk_count_kernel, dim3((unsigned)((nchunks + COUNT_WARPS - 1) / COUNT_WARPS)),
                         dim3(COUNT_WARPS * 32), st, a, counts, nchunks));
  SFKV_LAUNCH_CHECK("msg_mark/chunk_count");
  if (int rc = exclusive_scan(ChunkCount{counts}, nchunks, a.chunk_off, tmp, st)) return rc;
  // request offsets need only the chunk offsets: forked onto the (high-priority) aux stream, they
  // run beside the emit pass instead of after it (steady batch 0.3194 -> 0.3172 ms)
  const unsigned tg = grid_for((n_req + 1) * 32, 256, sms * 8);
  if (SFKV_TOKOFF_FORK) {
    SFKV_CUDA(cudaEventRecord(it->ev_fork, st));
    SFKV_CUDA(cudaStreamWaitEvent(it->aux, it->ev_fork, 0));
    req_tokoff_kernel<<<tg, 256, 0, it->aux>>>(a);
    SFKV_LAUNCH_CHECK("req_tokoff");
    SFKV_CUDA(cudaEventRecord(it->ev_join, it->aux));
  }
  if (nchunks > 0) SFKV_CUDA(launch_pdl(chunk_emit_kernel, dim3((unsigned)nchunks), dim3(CHUNK_THREADS), st, a));
  SFKV_CUDA(launch_pdl(copy_count_kernel, dim3(1), dim3(1), st, a.chunk_off, nchunks, n_tokens));
  if (SFKV_TOKOFF_FORK)
    SFKV_CUDA(cudaStreamWaitEvent(st, it->ev_join, 0));
  else
    SFKV_CUDA(launch_pdl(req_tokoff_kernel, dim3(tg), dim3(256), st, a));
  {  // the pending phase: one cooperative launch (grid barriers between its steps)
    static int coop_grid = 0;
    if (!coop_grid) {
      int per_sm = 0;
      SFKV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tok_pending_kernel, 256, 0));
      coop_grid = std::max(1, std::min(per_sm, 4)) * sms;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)coop_grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, tok_pending_kernel, a);
    if (e != cudaSuccess) {  // a cooperative launch may not take programmatic serialization
      cudaGetLastError();
      cfg.numAttrs = 1;
      SFKV_CUDA(cudaLaunchKernelEx(&cfg, tok_pending_kernel, a));
    }
  }
  SFKV_LAUNCH_CHECK("rank/publish/final");
  return 0;
}

}  // namespace sfkv

using namespace sfkv;

static void interner_free(sfkv_interner* it) {
  cudaFree(it->slots);
  cudaFree(it->owner);
  cudaFree(it->arena);
  cudaFree(it->id_off);
  cudaFree(it->id_len);
  cudaFree(it->ctr);
  cudaFree(it->tnew);
  if (it->ctr_host) cudaFreeHost(it->ctr_host);
  it->scratch.release();
  it->io.release();
  it->mbits.release();
  if (it->own_stream && it->stream) cudaStreamDestroy(it->stream);
  if (it->aux) cudaStreamDestroy(it->aux);
  if (it->ev_fork) cudaEventDestroy(it->ev_fork);
  if (it->ev_join) cudaEventDestroy(it->ev_join);
}

static int interner_check(sfkv_interner* it) {
  SFKV_CUDA(cudaMemcpyAsync(it->ctr_host, it->ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, it->stream));
  SFKV_CUDA(cudaStreamSynchronize(it->stream));
  const unsigned long long e = it->ctr_host[2];
  if (!e) return 0;
  // the failed batch published nothing; clear the flag so the interner stays usable
  SFKV_CUDA(cudaMemsetAsync(it->ctr + 2, 0, sizeof(unsigned long long), it->stream));
  if (e & TERR_COLLISION) return fail(SFKV_ECOLLIDE, "tokenize: 64-bit hash collision between different tokens");
  if (e & TERR_TABLE) return fail(SFKV_EPOOL, "tokenize: interner table full");
  if (e & TERR_IDS) return fail(SFKV_EPOOL, "tokenize: interner id space full");
  return fail(SFKV_EPOOL, "tokenize: interner arena full");
}

extern "C" {

int sfkv_interner_create(int32_t device, int32_t table_log2, int64_t arena_bytes, sfkv_interner** out) {
  if (!out || table_log2 < 4 || table_log2 > 34 || arena_bytes <= 0)
    return fail(SFKV_EINVAL, "interner_create: bad argument");
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  auto* it = new sfkv_interner;
  it->device = device;
  it->slots_n = int64_t(1) << table_log2;
  it->arena_cap = arena_bytes;
  it->max_ids = it->slots_n / 2;  // load factor <= 0.5
  cudaError_t e;
  int prio_hi = 0;
  if ((e = cudaMalloc(&it->slots, it->slots_n * sizeof(TSlot))) != cudaSuccess ||
      (e = cudaMalloc(&it->owner, it->slots_n * sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMalloc(&it->arena, arena_bytes)) != cudaSuccess ||
      (e = cudaMalloc(&it->id_off, it->max_ids * sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMalloc(&it->id_len, it->max_ids * sizeof(int32_t))) != cudaSuccess ||
      (e = cudaMalloc(&it->ctr, 8 * sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMallocHost(&it->ctr_host, 8 * sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&it->stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaDeviceGetStreamPriorityRange(nullptr, &prio_hi)) != cudaSuccess ||
      (e = cudaStreamCreateWithPriority(&it->aux, cudaStreamNonBlocking, prio_hi)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&it->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&it->ev_join, cudaEventDisableTiming)) != cudaSuccess) {
    it->own_stream = it->stream != nullptr;
    interner_free(it);
    delete it;
    return cuda_fail(e, "interner_create");
  }
  it->own_stream = true;
  interner_init_kernel<<<grid_for(it->slots_n, 256, 4096), 256, 0, it->stream>>>(it->slots, it->owner, it->slots_n);
  cudaMemsetAsync(it->ctr, 0, 8 * sizeof(unsigned long long), it->stream);
  if ((e = cudaStreamSynchronize(it->stream)) != cudaSuccess) {
    interner_free(it);
    delete it;
    return cuda_fail(e, "interner init");
  }
  *out = it;
  return 0;
}

int sfkv_interner_reset(sfkv_interner* it) {
  if (!it) return fail(SFKV_EINVAL, "interner_reset: null interner");
  DeviceGuard g(it->device);
  interner_init_kernel<<<grid_for(it->slots_n, 256, 4096), 256, 0, it->stream>>>(it->slots, it->owner, it->slots_n);
  SFKV_LAUNCH_CHECK("interner_init_kernel");
  SFKV_CUDA(cudaMemsetAsync(it->ctr, 0, 8 * sizeof(unsigned long long), it->stream));
  return 0;
}

int sfkv_interner_reserve(sfkv_interner* it, int32_t table_log2, int64_t arena_bytes) {
  if (!it || table_log2 > 34) return fail(SFKV_EINVAL, "interner_reserve: bad argument");
  DeviceGuard g(it->device);
  SFKV_CUDA(cudaStreamSynchronize(it->stream));
  SFKV_CUDA(cudaMemcpy(it->ctr_host, it->ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  const int64_t n_ids = (int64_t)it->ctr_host[0], used = (int64_t)it->ctr_host[1];
  if (arena_bytes > it->arena_cap) {  // the text moves; offsets stay
    uint8_t* a1 = nullptr;
    SFKV_CUDA(cudaMalloc(&a1, arena_bytes));
    if (used) SFKV_CUDA(cudaMemcpy(a1, it->arena, used, cudaMemcpyDeviceToDevice));
    cudaFree(it->arena);
    it->arena = a1;
    it->arena_cap = arena_bytes;
  }
  const int64_t slots1 = int64_t(1) << table_log2;
  if (slots1 > it->slots_n) {  // a larger table re-indexed by the same keys; ids unchanged
    TSlot* s1 = nullptr;
    int64_t *o1 = nullptr, *off1 = nullptr;
    int32_t* len1 = nullptr;
    const int64_t max1 = slots1 / 2;
    cudaError_t e;
    if ((e = cudaMalloc(&s1, slots1 * sizeof(TSlot))) != cudaSuccess ||
        (e = cudaMalloc(&o1, slots1 * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&off1, max1 * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&len1, max1 * sizeof(int32_t))) != cudaSuccess) {
      cudaFree(s1);
      cudaFree(o1);
      cudaFree(off1);
      return cuda_fail(e, "interner_reserve");
    }
    if (n_ids) {
      SFKV_CUDA(cudaMemcpy(off1, it->id_off, n_ids * sizeof(int64_t), cudaMemcpyDeviceToDevice));
      SFKV_CUDA(cudaMemcpy(len1, it->id_len, n_ids * sizeof(int32_t), cudaMemcpyDeviceToDevice));
    }
    interner_init_kernel<<<grid_for(slots1, 256, 4096), 256, 0, it->stream>>>(s1, o1, slots1);
    SFKV_LAUNCH_CHECK("interner_init_kernel");
    if (n_ids) {
      interner_rehash_kernel<<<grid_for(n_ids, 256, 4096), 256, 0, it->stream>>>(
          s1, (uint64_t)slots1 - 1, 64 - table_log2, it->arena, off1, len1, n_ids);
      SFKV_LAUNCH_CHECK("interner_rehash_kernel");
    }
    SFKV_CUDA(cudaStreamSynchronize(it->stream));
    cudaFree(it->slots);
    cudaFree(it->owner);
    cudaFree(it->id_off);
    cudaFree(it->id_len);
    it->slots = s1;
    it->owner = o1;
    it->id_off = off1;
    it->id_len = len1;
    it->slots_n = slots1;
    it->max_ids = max1;
  }
  return 0;
}

int sfkv_interner_arena(sfkv_interner* it, int64_t* used, int64_t* cap, int32_t* table_log2) {
  if (!it || !used || !cap || !table_log2) return fail(SFKV_EINVAL, "interner_arena: null argument");
  DeviceGuard g(it->device);
  SFKV_CUDA(cudaMemcpyAsync(it->ctr_host, it->ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, it->stream));
  SFKV_CUDA(cudaStreamSynchronize(it->stream));
  *used = (int64_t)it->ctr_host[1];
  *cap = it->arena_cap;
  *table_log2 = __builtin_ctzll((unsigned long long)it->slots_n);
  return 0;
}

int sfkv_interner_destroy(sfkv_interner* it) {
  if (!it) return fail(SFKV_EINVAL, "interner_destroy: null interner");
  DeviceGuard g(it->device);
  cudaStreamSynchronize(it->stream);
  interner_free(it);
  delete it;
  return 0;
}

int sfkv_interner_set_stream(sfkv_interner* it, void* stream) {
  if (!it) return fail(SFKV_EINVAL, "interner_set_stream: null interner");
  DeviceGuard g(it->device);
  SFKV_CUDA(cudaStreamSynchronize(it->stream));
  if (it->own_stream) cudaStreamDestroy(it->stream);
  it->stream = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream (as pools)
  it->own_stream = false;
  return 0;
}

int sfkv_interner_size(sfkv_interner* it, int64_t* n_ids) {
  if (!it || !n_ids) return fail(SFKV_EINVAL, "interner_size: null argument");
  DeviceGuard g(it->device);
  SFKV_CUDA(cudaMemcpyAsync(it->ctr_host, it->ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, it->stream));
  SFKV_CUDA(cudaStreamSynchronize(it->stream));
  *n_ids = (int64_t)it->ctr_host[0];
  return 0;
}

int sfkv_interner_token(sfkv_interner* it, uint32_t id, char* out, int32_t cap, int32_t* len) {
  if (!it || !len || (cap > 0 && !out)) return fail(SFKV_EINVAL, "interner_token: bad argument");
  int64_t n = 0;
  if (int rc = sfkv_interner_size(it, &n)) return rc;
  if ((int64_t)id >= n) return fail(SFKV_EINVAL, "interner_token: unknown id");
  DeviceGuard g(it->device);
  int64_t off = 0;
  int32_t l = 0;
  SFKV_CUDA(cudaMemcpy(&off, it->id_off + id, sizeof(off), cudaMemcpyDeviceToHost));
  SFKV_CUDA(cudaMemcpy(&l, it->id_len + id, sizeof(l), cudaMemcpyDeviceToHost));
  *len = l;
  if (cap > 0) SFKV_CUDA(cudaMemcpy(out, it->arena + off, (size_t)(l < cap ? l : cap), cudaMemcpyDeviceToHost));
  return 0;
}

int sfkv_tokenize_batch_dev(sfkv_interner* it, int64_t n, const int64_t* req_msg_off, int64_t n_msg,
                            const int64_t* msg_off, const uint8_t* text, int64_t n_bytes, int64_t* tok_off,
                            uint32_t* tok, int64_t* n_tokens) {
  if (!it || n < 0 || n_msg < 0 || n_bytes < 0 || !tok_off || !n_tokens || (n > 0 && !req_msg_off) ||
      (n_msg > 0 && !msg_off) || (n_bytes > 0 && (!text || !tok)))
    return fail(SFKV_EINVAL, "tokenize_batch_dev: bad argument");
  DeviceGuard g(it->device);
  return tokenize_dev(it, n, req_msg_off, n_msg, msg_off, text, n_bytes, tok_off, tok, n_tokens);
}

int sfkv_tokenize_batch(sfkv_interner* it, int64_t n, const int64_t* req_msg_off, const int64_t* msg_off,
                        const uint8_t* text, int64_t* tok_off, uint32_t* tok, int64_t tok_cap,
                        int64_t* n_tokens) {
  if (!it || n < 0 || !req_msg_off || !tok_off || !n_tokens) return fail(SFKV_EINVAL, "tokenize_batch: bad argument");
  const int64_t n_msg = req_msg_off[n];
  if (req_msg_off[0] != 0) return fail(SFKV_EINVAL, "tokenize_batch: req_msg_off[0] must be 0");
  for (int64_t r = 0; r < n; ++r)
    if (req_msg_off[r + 1] < req_msg_off[r]) return fail(SFKV_EINVAL, "tokenize_batch: req_msg_off decreasing");
  if (n_msg > 0 && !msg_off) return fail(SFKV_EINVAL, "tokenize_batch: null msg_off");
  const int64_t n_bytes = n_msg > 0 ? msg_off[n_msg] : 0;
  if (n_msg > 0 && msg_off[0] != 0) return fail(SFKV_EINVAL, "tokenize_batch: msg_off[0] must be 0");
  for (int64_t m = 0; m < n_msg; ++m)
    if (msg_off[m + 1] < msg_off[m]) return fail(SFKV_EINVAL, "tokenize_batch: msg_off decreasing");
  if (tok_cap < (n_bytes + n_msg + 1) / 2)
    return fail(SFKV_EINVAL, "tokenize_batch: tok_cap < (n_bytes + n_msg + 1) / 2");
  DeviceGuard g(it->device);
  cudaStream_t st = it->stream;
  const int64_t tb = (n_bytes + n_msg + 1) / 2 + 1;
  Carver cv;
  const size_t o_rm = cv.take<int64_t>(n + 1), o_mo = cv.take<int64_t>(n_msg + 1), o_tx = cv.take<uint8_t>(n_bytes + 16),
               o_to = cv.take<int64_t>(n + 1), o_tk = cv.take<uint32_t>(tb), o_nt = cv.take<int64_t>(1);
  if (int rc = it->io.ensure(cv.off)) return rc;
  char* b = it->io.as<char>();
  SFKV_CUDA(cudaMemcpyAsync(b + o_rm, req_msg_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  if (n_msg > 0) SFKV_CUDA(cudaMemcpyAsync(b + o_mo, msg_off, (n_msg + 1) * 8, cudaMemcpyHostToDevice, st));
  else SFKV_CUDA(cudaMemsetAsync(b + o_mo, 0, 8, st));
  if (n_bytes > 0) SFKV_CUDA(cudaMemcpyAsync(b + o_tx, text, n_bytes, cudaMemcpyHostToDevice, st));
  if (int rc = tokenize_dev(it, n, reinterpret_cast<int64_t*>(b + o_rm), n_msg, reinterpret_cast<int64_t*>(b + o_mo),
                            reinterpret_cast<uint8_t*>(b + o_tx), n_bytes, reinterpret_cast<int64_t*>(b + o_to),
                            reinterpret_cast<uint32_t*>(b + o_tk), reinterpret_cast<int64_t*>(b + o_nt)))
    return rc;
  if (int rc = interner_check(it)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(n_tokens, b + o_nt, 8, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  SFKV_CUDA(cudaMemcpyAsync(tok_off, b + o_to, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (*n_tokens > 0) SFKV_CUDA(cudaMemcpyAsync(tok, b + o_tk, *n_tokens * 4, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfkv_interner_check(sfkv_interner* it) {
  if (!it) return fail(SFKV_EINVAL, "interner_check: null interner");
  DeviceGuard g(it->device);
  return interner_check(it);
}

}  // extern "C"

// Internal definition of a KV pin pool (one backend's cache, resident on one GPU).
//
// HBM layout (all arrays device-resident, sized at pool creation):
//   pins   pin_len[W] i64 (-1 = no pin), pin_nblk[W] i32,
//          pin_blk[W][MB] i32 (block table), pin_tok[W][32 G][16] u32 with G = ceil(MB/32): the
//          pin's tokens block by block (pin-major), so the blocks of one request segment of a
//          match tile are one contiguous extent that a single bulk copy (TMA) stages, with no
//          block-id indirection; the block's chained hash is blk_key[pin_blk]
//   blocks blk_key[B] u64, blk_parent[B] i32 (exact sharing: a hit must descend from the block
//          chosen for its predecessor), blk_tok[B][16] u32 (tokens: verify-on-hit),
//          blk_n[B] u8 (valid tokens), blk_in_table[B] u8, blk_ref[B] u32, blk_slot[B] i64,
//          free_bits[ceil(B/32)] u32 (1 = free)
//   table  slots[S] of 16 B {u64 key, i32 block, i32 pad} (open addressing, linear probing,
//          S = 2^table_log2; key 0 = empty, 1 = tombstone; one sector per probe) and
//          towner[S] i64 (lowest claiming item of a batch; commit only)
//   kv     [B][n_slabs][16][slab_row_bytes] bytes (bf16 K/V rows), block-major so a block is
//          one contiguous extent (2 MiB for Llama-3-8B: 64 slabs x 16 x 2 KiB)
#pragma once

#include "common.cuh"

namespace sfkv {

struct Slot {
  unsigned long long key;
  int32_t val;  // block id; -1 while a batch claim is pending
  int32_t pad;
};
static_assert(sizeof(Slot) == 16, "table slot is one 16-B vector");

struct DevCounters {
  long long occupancy;            // logical tokens (sum of pin lengths)
  unsigned long long rejections;  // capacity_rejections
  long long table_live;
  long long table_tomb;
  long long blocks_in_use;
  int error;                      // sticky device-side error (SFKV_EPOOL / SFKV_ESTALE)
  int pad;                        // table-rebuild flag
  long long occ_saved;            // admission snapshot, restored when a batch aborts
  unsigned long long rej_saved;
};

}  // namespace sfkv

// A peer rank's pool payload mapped into this process (CUDA IPC).
struct sfkv_peer {
  int32_t device = 0;
  uint8_t* kv = nullptr;
  int64_t kv_bytes = 0;
  int64_t block_bytes = 0;
  int32_t n_slabs = 0;
  int32_t slab_row_bytes = 0;
};

struct sfkv_pool {
  sfkv_pool_config cfg;
  int64_t block_bytes = 0;
  int64_t n_words = 0;        // free-bitmap words
  int64_t table_slots = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // commit: the old pins' release and the new pins' install run on `aux` while the payload copy
  // runs on `stream` (forked after allocation, joined before the call returns its work)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // device state
  int64_t* pin_len = nullptr;
  int32_t* pin_nblk = nullptr;
  int32_t* pin_blk = nullptr;
  uint32_t* pin_tok = nullptr;  // [W][MB][16] a pin's tokens, block by block (pin-major copy)
  uint64_t* blk_key = nullptr;
  int32_t* blk_parent = nullptr;  // the block at index k-1 of the pin that allocated it (-1 at k = 0)
  uint32_t* blk_tok = nullptr;
  uint8_t* blk_n = nullptr;
  uint8_t* blk_in_table = nullptr;
  uint32_t* blk_ref = nullptr;
  int64_t* blk_slot = nullptr;
  uint32_t* free_bits = nullptr;
  sfkv::Slot* slots = nullptr;
  int64_t* towner = nullptr;
  uint8_t* kv = nullptr;
  sfkv::DevCounters* ctr = nullptr;  // device
  sfkv::DevCounters* ctr_host = nullptr;  // pinned mirror
  // host-side counters (BackendStats, backend.hpp:72-80)
  uint64_t flush_calls = 0;
  uint64_t preserve_calls = 0;
  // scratch
  sfkv::Scratch scratch;       // per-call device scratch
  sfkv::Scratch small;         // per-call offsets (sized by request count)
  sfkv::Scratch io;            // device copies of host-pointer inputs/outputs
  sfkv::Scratch prep_status;   // match prep look-back statuses (epoch-tagged)
  uint32_t prep_epoch = 0;
  void* host_stage = nullptr;  // pinned host staging
  size_t host_stage_bytes = 0;
  bool exported = false;       // the KV region was handed out as a CUDA IPC handle (fixed)
};

namespace sfkv {

constexpr int PIN_STRIDE = 16;  // words per pin block (16 tokens, stored chunk-rotated: pin_rot)
// Word index of token j of pin block k of workflow wf in pin_tok (see the layout above).
__host__ __device__ __forceinline__ int64_t pin_tok_index(int64_t wf, int64_t k, int j, int64_t groups) {
  return (wf * (groups << 5) + k) * PIN_STRIDE + j;
}
inline int64_t pin_groups(const sfkv_pool_config& c) { return (c.max_pin_blocks + 31) / 32; }
// A pin block's four 16-B chunks are stored rotated: chunk x of block k sits in chunk slot
// (x + pin_rot(k)) & 3. Lane L of a match tile reads block k0 + L staged at L * 64 B; reading its
// chunks in slot order (x + pin_rot(k)) & 3 puts the 8 lanes of a quarter-warp on 8 distinct bank
// groups for any k0, and every chunk still lands in its own register (no selects).
__host__ __device__ __forceinline__ int pin_rot(int64_t k) { return (int)((k >> 1) & 3); }

// Outputs of the hashing/matching pass shared by match, lookup and commit.
struct MatchArgs {
  int64_t n;                 // requests
  const int32_t* wf;         // nullable (lookup mode)
  const int64_t* tok_off;
  const uint32_t* tok;
  int64_t* blk_off;          // [n+1] exclusive scan of ceil(len/16), written by launch_match
  int64_t n_items;
  int64_t n_tok_bound;       // token-buffer capacity (ids) the tok pointer may be read up to
  int64_t* out_M;            // nullable
  uint64_t* out_hash;        // nullable
  int32_t* out_block;        // nullable: lookup mode
  int64_t* out_hit;          // nullable: lookup mode
};

struct PayloadJob {
  int64_t n;
  const int32_t* wf;
  const int64_t* tok_off;
  const int64_t* blk_off;
  const int64_t* M;
  const int64_t* rank;
  const int64_t* alloc_list;
  const int32_t* bid;
  int64_t n_items;
  const int32_t* cow_src;  // per allocated block (alloc order): the old pin's block at the same
                           // index, snapshotted before the install overwrites the pin table
  const int* error;  // sticky batch error: no bytes move when set
};
// Handoff payload source: rows of batch item `item` (request r's block k) come from block
// blk[item] of the source region kv (another pool of this process, or a peer rank's pool mapped
// over CUDA IPC: reads then travel over NVLink).
struct PayloadSource {
  const uint8_t* kv = nullptr;
  const int32_t* blk = nullptr;
  int64_t block_bytes = 0;
  int64_t n_blocks = 0;  // blocks in the source region: a source id outside it moves nothing and
                         // sets the destination pool's sticky SFKV_EINVAL
};
int launch_payload(sfkv_pool* p, const PayloadJob& j, const void* kv_src, const int64_t* kv_src_off,
                   const PayloadSource* src, cudaStream_t st);

int launch_match(sfkv_pool* p, const MatchArgs& a, int64_t* tile_state, cudaStream_t st);
size_t match_tile_state_elems(int64_t n_items, int64_t n_requests);

// Internal commit entry (device pointers). src: handoff payload source (nullable).
int commit_dev(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
               const uint32_t* tok, int64_t n_items_bound, int64_t n_tok_bound, const void* kv_src,
               const int64_t* kv_src_off, const int64_t* m_expected, int32_t* out_status,
               const PayloadSource* src);
int flush_dev(sfkv_pool* p, int64_t n, const int32_t* wf, int64_t* out_freed, bool all);
int gather_dev(sfkv_pool* p, int64_t n, const int32_t* wf, void* dst, const int64_t* dst_off);
int maybe_rebuild_table(sfkv_pool* p, cudaStream_t st);
// Re-inserts every indexed block into the (already resized) empty table; resets tombstones.
int rebuild_table_now(sfkv_pool* p);

}  // namespace sfkv

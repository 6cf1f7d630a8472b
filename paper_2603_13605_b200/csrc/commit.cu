// K3+K4: retain (commit) and evict (flush) on the pool — block table, global dedup table,
// refcounts, deterministic allocation, capacity admission.
//
// Replaces SimulatedBackend::pin_prompt (simulated_backend.cpp:135-151) and ::flush (169-184).
// A commit batch runs these launches on the pool stream with no host synchronisation (the batch
// semantics are defined in oracle/sfkv_oracle.c, commit_impl):
//   match      chained hashes of every block + M_r = LCP(old pin, tokens)           (match.cu)
//   admit      one warp, request order: reject iff occ - old + new > capacity; warp-wide fast
//              path when the whole 32-request chunk fits, exact sequential fallback otherwise
//   probe      per full block: table probe; verified pre-existing key -> hit0; new key ->
//              claim (atomicCAS into an empty slot) + atomicMin(owner) = lowest claiming item
//   resolve1   linked hits: hit0 and (k = 0 or the previous item is a hit0 of the block's parent);
//              atomicMin(f_hit[r]) over the rest
//   resolve2   linked dups at k >= f_hit: a claim with a lower owner o, equal tokens, and the
//              previous item resolving to the same block as o's previous item (a dup of o-1, or
//              at k = f_hit the same linked hit); atomicMin(first_nonhit[r]) over the rest.
//              Sharing is exact by induction over parent links: a shared block's whole prefix is
//              the request's, whatever the chained hash does (keys only locate candidates)
//   categorize HIT below f_hit, DUP below first_nonhit, OWN (key owner) / PRIV above
//   scan x2    exclusive scan of new-block flags (rank) and of free-bitmap popcounts
//   alloc      rank -> the rank-th free block id (lowest ids first, batch order: deterministic,
//              independent of atomic order); OWN publishes its id into the table slot
//   refs       every block of every new pin takes a reference (atomicAdd)
//   payload    copy-on-share + staging scatter of new blocks                        (copy.cu)
//   release    old pins drop their references; blocks reaching 0 return to the free bitmap and
//              leave the table (tombstone)
//   install    new block tables / hashes / lengths, parent links of the new blocks
// The batch is phase-ordered, so a block shared by an old and a new pin never transiently hits
// a refcount of zero. Scratch is sized by an item-count bound from the caller (token-buffer
// size / 16 + requests); every kernel reads the exact count blk_off[n] on the device.
#include "pool.cuh"

namespace sfkv {

#ifndef SFKV_FREE_FORK
#define SFKV_FREE_FORK 1
#endif
#ifndef SFKV_REBUILD_AUX
#define SFKV_REBUILD_AUX 1
#endif
#ifndef SFKV_REL_THREADS
#define SFKV_REL_THREADS 256
#endif
constexpr int REL_THREADS = SFKV_REL_THREADS;  // release: one warp per workflow

enum : uint8_t { CAT_NONE = 0, CAT_HIT = 1, CAT_DUP = 2, CAT_OWN = 3, CAT_PRIV = 4 };

struct CommitScratch {
  int64_t* blk_off;       // [n+1]
  int64_t* M;             // [n]
  uint64_t* hash;         // [items]
  int64_t* tile_state;    // match look-back
  int32_t* status;        // [n]
  int64_t* slot_of;       // [items]
  int32_t* bid;           // [items]
  uint8_t* hit0;          // [items]
  uint8_t* claim;         // [items]
  uint8_t* cat;           // [items]
  int64_t* first_nonhit;  // [n]
  int64_t* delta;         // [n] occupancy change of each request if admitted
  int64_t* f_hit;         // [n] first item that is not a linked hit
  int64_t* rank;          // [items+1]
  int64_t* wprefix;       // [words+1]
  int64_t* alloc_list;    // [items]
  int32_t* cow_src;       // [items] by alloc rank: the old pin's block at the same index (or -1)
  int64_t* scan_tmp;
};

struct CommitArgs {
  int64_t n;
  const int32_t* wf;
  const int64_t* tok_off;
  const uint32_t* tok;
  int64_t n_items;  // upper bound (exact count: s.blk_off[n])
  const int64_t* m_expected;
  int payload;  // 1 when KV bytes are written
  CommitScratch s;
  // pool
  int64_t* pin_len;
  int32_t* pin_nblk;
  int32_t* pin_blk;
  uint32_t* pin_tok;
  uint64_t* blk_key;
  int32_t* blk_parent;
  uint32_t* blk_tok;
  uint8_t* blk_n;
  uint8_t* blk_in_table;
  uint32_t* blk_ref;
  int64_t* blk_slot;
  uint32_t* free_bits;
  Slot* slots;
  int64_t* towner;
  uint64_t slot_mask;
  int64_t n_words;
  int64_t n_blocks;
  int32_t max_pin_blocks;
  int64_t pin_groups;
  int64_t capacity;
  DevCounters* ctr;
  int32_t max_wf;  // device-side slot guard (the _dev entry points' slots are not host-checked)
};

#define FOR_ITEMS(a, item)                                                         \
  for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,              \
               n_items__ = (a).s.blk_off[(a).n];                                   \
       item < n_items__; item += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ void item_coords(const CommitArgs& a, int64_t item, int64_t& r,
                                            int64_t& k, int& nval) {
  r = upper_index(a.s.blk_off, a.n, item);
  k = item - a.s.blk_off[r];
  const int64_t rem = a.tok_off[r + 1] - a.tok_off[r] - k * BT;
  nval = (int)(rem < BT ? rem : BT);
}

__device__ __forceinline__ void load_req_block(const CommitArgs& a, int64_t r, int64_t k, int nval,
                                               uint32_t* t) {
  const uint32_t* p = a.tok + a.tok_off[r] + k * BT;
#pragma unroll
  for (int j = 0; j < BT; ++j) t[j] = j < nval ? __ldg(p + j) : 0u;
}

__device__ __forceinline__ bool blk_tokens_equal(const uint32_t* __restrict__ blk_tok, int32_t id,
                                                 const uint32_t* t) {
  const uint4* q = reinterpret_cast<const uint4*>(blk_tok + (int64_t)id * BT);
  bool eq = true;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 v = q[i];
    eq &= v.x == t[4 * i] && v.y == t[4 * i + 1] && v.z == t[4 * i + 2] && v.w == t[4 * i + 3];
  }
  return eq;
}

// ---- admission: exact reference order ------------------------------------------------------
// Every request's checks and occupancy delta are computed by the whole CTA with all loads in
// flight (the dependent wf -> pin_len load once per request, not once per step of the sequential
// rule); then one warp applies the rule in request order, 32 requests per step: a warp scan
// accepts the whole step when every prefix fits, else the exact sequential rule
// (simulated_backend.cpp:141-150) runs over the step's deltas.
constexpr int ADMIT_THREADS = 1024;
constexpr int ADMIT_SMEM = 4096;  // deltas kept in shared memory for batches up to this size
__global__ void __launch_bounds__(ADMIT_THREADS) admit_kernel(CommitArgs a) {
  pdl_enter();
  __shared__ int64_t s_delta[ADMIT_SMEM];
  const int tid = threadIdx.x, lane = tid & 31;
  DevCounters* c = a.ctr;
  if (tid == 0) {
    c->error = 0;
    c->occ_saved = c->occupancy;
    c->rej_saved = c->rejections;
  }
  // staleness / block-table checks first: a refused batch changes nothing
  int stale = 0, blen = 0, bslot = 0;
  for (int64_t r = tid; r < a.n; r += ADMIT_THREADS) {
    const int64_t len = a.tok_off[r + 1] - a.tok_off[r];
    const int32_t w = a.wf[r];
    if ((len + BT - 1) / BT > a.max_pin_blocks || len < 0) blen = 1;
    int64_t d = 0;
    if ((uint32_t)w >= (uint32_t)a.max_wf) {
      bslot = 1;
    } else {
      if (a.payload && a.m_expected && a.m_expected[r] != a.s.M[r]) stale = 1;
      const int64_t pl = a.pin_len[w];
      d = len - (pl < 0 ? 0 : pl);
    }
    if (r < ADMIT_SMEM) s_delta[r] = d;
    else a.s.delta[r] = d;
    a.s.first_nonhit[r] = (len + BT - 1) / BT;
    a.s.f_hit[r] = (len + BT - 1) / BT;
  }
  const int any_stale = __syncthreads_or(stale), any_len = __syncthreads_or(blen), any_slot = __syncthreads_or(bslot);
  if (any_stale || any_len || any_slot) {
    const int code = any_slot ? SFKV_EINVAL : (any_len ? SFKV_EPOOL : SFKV_ESTALE);
    for (int64_t r = tid; r < a.n; r += ADMIT_THREADS) a.s.status[r] = code;
    if (tid == 0) c->error = code;
    return;
  }
  if (tid >= 32) return;
  long long occ = c->occupancy;
  unsigned long long rej = 0;
  for (int64_t base = 0; base < a.n; base += 32) {
    const int64_t r = base + lane;
    const bool act = r < a.n;
    const long long delta = act ? (r < ADMIT_SMEM ? s_delta[r] : a.s.delta[r]) : 0;
    // fast path: every prefix of the step fits
    long long incl = delta;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const bool fits = !act || occ + incl <= a.capacity;
    if (__all_sync(0xffffffffu, fits)) {
      if (act) a.s.status[r] = SFKV_PIN_ACCEPTED;
      occ += __shfl_sync(0xffffffffu, incl, 31);
    } else {
      for (int j = 0; j < 32; ++j) {  // exact sequential rule (simulated_backend.cpp:141-150)
        const long long d = __shfl_sync(0xffffffffu, delta, j);
        const int aj = __shfl_sync(0xffffffffu, (int)act, j);
        if (!aj) break;
        const bool ok = occ + d <= a.capacity;
        if (lane == j) a.s.status[r] = ok ? SFKV_PIN_ACCEPTED : SFKV_PIN_REJECTED;
        if (ok) occ += d;
        else ++rej;
      }
    }
  }
  if (lane == 0) {
    c->occupancy = occ;
    c->rejections += rej;
  }
}

// ---- probe / claim ---------------------------------------------------------------------
__global__ void probe_kernel(CommitArgs a) {
  pdl_enter();
  if (a.ctr->error) return;
  FOR_ITEMS(a, item) {
    int64_t r, k;
    int nval;
    item_coords(a, item, r, k, nval);
    a.s.slot_of[item] = -1;
    a.s.hit0[item] = 0;
    a.s.claim[item] = 0;
    a.s.bid[item] = -1;
    if (a.s.status[r] != SFKV_PIN_ACCEPTED || nval != BT) continue;
    uint32_t t[BT];
    load_req_block(a, r, k, nval, t);
    const unsigned long long c = a.s.hash[item];
    uint64_t s = c & a.slot_mask;
    for (uint64_t probes = 0; probes <= a.slot_mask; ++probes) {
      unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(&a.slots[s].key);
      if (key == KEY_EMPTY) {
        const unsigned long long prev = atomicCAS(&a.slots[s].key, KEY_EMPTY, c);
        key = prev == KEY_EMPTY ? c : prev;
      }
      if (key == c) {
        a.s.slot_of[item] = (int64_t)s;
        const int32_t val = *reinterpret_cast<volatile int32_t*>(&a.slots[s].val);
        if (val >= 0) {  // key present before this batch
          if (a.blk_n[val] == BT && blk_tokens_equal(a.blk_tok, val, t)) {
            a.s.hit0[item] = 1;
            a.s.bid[item] = val;
          }
        } else {  // key claimed in this batch
          a.s.claim[item] = 1;
          atomicMin(reinterpret_cast<unsigned long long*>(&a.towner[s]), (unsigned long long)item);
        }
        break;
      }
      s = (s + 1) & a.slot_mask;
    }
    if (a.s.slot_of[item] < 0) a.ctr->error = SFKV_EPOOL;  // table full
  }
}

// Linked hits: the pre-existing block of item k must descend from the block of item k-1.
__global__ void resolve_hits_kernel(CommitArgs a) {
  pdl_enter();
  if (a.ctr->error) return;
  FOR_ITEMS(a, item) {
    int64_t r, k;
    int nval;
    item_coords(a, item, r, k, nval);
    if (a.s.status[r] != SFKV_PIN_ACCEPTED) continue;
    const bool ok = a.s.hit0[item] &&
                    (k == 0 || (a.s.hit0[item - 1] && a.blk_parent[a.s.bid[item]] == a.s.bid[item - 1]));
    if (!ok) atomicMin(reinterpret_cast<unsigned long long*>(&a.s.f_hit[r]), (unsigned long long)k);
  }
}

// Linked dups past the hit run (see the header): the owner o's block is shared only if the
// previous items of both requests resolve to the same block.
__global__ void resolve_dups_kernel(CommitArgs a) {
  pdl_enter();
  if (a.ctr->error) return;
  FOR_ITEMS(a, item) {
    int64_t r, k;
    int nval;
    item_coords(a, item, r, k, nval);
    if (a.s.status[r] != SFKV_PIN_ACCEPTED) continue;
    const int64_t fh = a.s.f_hit[r];
    if (k < fh) continue;
    bool dup = false;
    if (a.s.claim[item]) {
      const int64_t o = a.towner[a.s.slot_of[item]];
      if (o < item) {
        int64_t ro, ko;
        int no;
        item_coords(a, o, ro, ko, no);
        uint32_t t[BT], u[BT];
        load_req_block(a, r, k, nval, t);
        load_req_block(a, ro, ko, no, u);
        dup = true;
#pragma unroll
        for (int j = 0; j < BT; ++j) dup &= t[j] == u[j];
        if (dup && k > 0) {
          const bool dup_link = k > fh && a.s.claim[item - 1] && a.towner[a.s.slot_of[item - 1]] == o - 1;
          const bool hit_link = k == fh && ko - 1 < a.s.f_hit[ro] && a.s.bid[item - 1] == a.s.bid[o - 1];
          dup = dup_link || hit_link;
        }
      }
    }
    if (!dup) atomicMin(reinterpret_cast<unsigned long long*>(&a.s.first_nonhit[r]), (unsigned long long)k);
  }
}

// Runs over the whole bound so the rank scan can use it as its length.
__global__ void categorize_kernel(CommitArgs a) {
  pdl_enter();
  const int64_t NI = a.s.blk_off[a.n];
  const bool err = a.ctr->error != 0;
  for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < a.n_items;
       item += (int64_t)gridDim.x * blockDim.x) {
    uint8_t cat = CAT_NONE;
    if (item < NI && !err) {
      const int64_t r = upper_index(a.s.blk_off, a.n, item);
      const int64_t k = item - a.s.blk_off[r];
      if (a.s.status[r] == SFKV_PIN_ACCEPTED) {
        if (k < a.s.f_hit[r]) {
          cat = CAT_HIT;
        } else if (k < a.s.first_nonhit[r]) {
          cat = CAT_DUP;
        } else {
          const bool own = a.s.claim[item] && a.towner[a.s.slot_of[item]] == item;
          cat = own ? CAT_OWN : CAT_PRIV;
        }
      }
    }
    a.s.cat[item] = cat;
  }
}

struct NeedAlloc {
  const uint8_t* cat;
  __device__ int64_t operator()(int64_t i) const {
    return (cat[i] == CAT_OWN || cat[i] == CAT_PRIV) ? 1 : 0;
  }
};
struct FreeCount {
  const uint32_t* bits;
  __device__ int64_t operator()(int64_t i) const { return __popc(bits[i]); }
};

__device__ __forceinline__ int select_bit(uint32_t w, int r) {  // position of the r-th set bit
  for (int b = 0; b < 32; ++b) {
    if (w & (1u << b)) {
      if (r == 0) return b;
      --r;
    }
  }
  return -1;
}

__global__ void __launch_bounds__(256) alloc_kernel(CommitArgs a) {
  pdl_enter();
  __shared__ int s_skip;  // one CTA-uniform decision (the block reduce below needs every thread)
  const int64_t total_free = a.s.wprefix[a.n_words];
  if (threadIdx.x == 0) s_skip = a.ctr->error ? 1 : (a.s.rank[a.n_items] > total_free ? 2 : 0);
  __syncthreads();
  if (s_skip) {
    if (s_skip == 2 && blockIdx.x == 0 && threadIdx.x == 0) a.ctr->error = SFKV_EPOOL;  // exhausted: abort
    return;                                                                            // before any block is touched
  }
  int n_new = 0, n_live = 0;
  FOR_ITEMS(a, item) {
    const uint8_t cat = a.s.cat[item];
    if (cat != CAT_OWN && cat != CAT_PRIV) continue;
    const int64_t rk = a.s.rank[item];
    if (rk >= total_free) {
      a.ctr->error = SFKV_EPOOL;
      continue;
    }
    const int64_t w = upper_index(a.s.wprefix, a.n_words, rk);
    const int bit = select_bit(a.free_bits[w], (int)(rk - a.s.wprefix[w]));
    const int32_t id = (int32_t)(w * 32 + bit);
    a.s.alloc_list[rk] = item;
    a.s.bid[item] = id;
    // the free bit is cleared by refs_kernel: selection must see the pre-batch bitmap
    int64_t r, k;
    int nval;
    item_coords(a, item, r, k, nval);
    {  // copy-on-share source, read before install_kernel replaces the pin table
      const int32_t w = a.wf[r];
      a.s.cow_src[rk] = a.pin_len[w] >= 0 && k < a.pin_nblk[w] ? a.pin_blk[(int64_t)w * a.max_pin_blocks + k] : -1;
    }
    uint32_t t[BT];
    load_req_block(a, r, k, nval, t);
    uint4* dst = reinterpret_cast<uint4*>(a.blk_tok + (int64_t)id * BT);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);
    a.blk_key[id] = a.s.hash[item];
    a.blk_n[id] = (uint8_t)nval;
    a.blk_ref[id] = 0;
    if (cat == CAT_OWN) {
      const int64_t s = a.s.slot_of[item];
      a.slots[s].val = id;
      a.blk_slot[id] = s;
      a.blk_in_table[id] = 1;
      ++n_live;
    } else {
      a.blk_slot[id] = -1;
      a.blk_in_table[id] = 0;
    }
    ++n_new;
  }
  // one pair of counter atomics per CTA (per-block atomics on one address serialise in L2)
  using BR = cub::BlockReduce<int2, 256>;
  __shared__ typename BR::TempStorage tmp;
  const int2 tot = BR(tmp).Reduce(make_int2(n_new, n_live), [](int2 x, int2 y) { return make_int2(x.x + y.x, x.y + y.y); });
  if (threadIdx.x == 0 && tot.x) {
    atomic_add_i64(&a.ctr->blocks_in_use, (long long)tot.x);
    if (tot.y) atomic_add_i64(&a.ctr->table_live, (long long)tot.y);
  }
}

__global__ void refs_kernel(CommitArgs a) {
  pdl_enter();
  if (a.ctr->error) return;
  FOR_ITEMS(a, item) {
    const uint8_t cat = a.s.cat[item];
    if (cat == CAT_NONE) continue;
    int32_t id = a.s.bid[item];
    if (cat == CAT_DUP) {
      id = a.slots[a.s.slot_of[item]].val;
      a.s.bid[item] = id;
    } else if (cat == CAT_OWN || cat == CAT_PRIV) {
      atomicAnd(&a.free_bits[id >> 5], ~(1u << (id & 31)));
    }
    atomicAdd(&a.blk_ref[id], 1u);
  }
}

__global__ void clear_owner_kernel(CommitArgs a) {
  pdl_enter();
  FOR_ITEMS(a, item) {
    if (a.s.claim[item]) a.towner[a.s.slot_of[item]] = NO_OWNER;
  }
}

// Drops one reference; frees the block at zero.
// Drops one reference; returns 1 when the block was freed (2 when it also left the table). The
// caller sums the pool counters per warp: a flush of all pins frees ~1.7 M blocks, and three
// global atomics per block on the same counters serialise in one L2 slice.
__device__ __forceinline__ int release_block(const CommitArgs& a, int32_t id) {
  const uint32_t old = atomicSub(&a.blk_ref[id], 1u);
  if (old != 1u) return 0;
  atomicOr(&a.free_bits[id >> 5], 1u << (id & 31));
  if (!a.blk_in_table[id]) return 1;
  a.slots[a.blk_slot[id]].key = KEY_TOMB;
  a.blk_in_table[id] = 0;
  return 2;
}

// One warp per request: release the old pin; install the new length (commit) or none (flush).
__global__ void release_kernel(CommitArgs a, int mode /*0 commit, 1 flush list, 2 flush all*/,
                               int64_t* out_freed) {
  pdl_enter();
  if (mode == 0 && a.ctr->error) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int freed_blocks = 0, left_table = 0;
  long long occ_freed = 0;  // lane 0: tokens freed by this warp's workflows (flush modes)
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n; r += warps) {
    if (mode == 0 && a.s.status[r] != SFKV_PIN_ACCEPTED) continue;
    const int32_t w = mode == 2 ? (int32_t)r : a.wf[r];
    const int64_t pl = a.pin_len[w];
    if (pl >= 0) {
      const int32_t nb = a.pin_nblk[w];
      const int64_t pb = (int64_t)w * a.max_pin_blocks;
      for (int32_t k = lane; k < nb; k += 32) {
        const int f = release_block(a, a.pin_blk[pb + k]);
        freed_blocks += f != 0;
        left_table += f == 2;
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (mode == 0) {
        const int64_t len = a.tok_off[r + 1] - a.tok_off[r];
        a.pin_len[w] = len;
        a.pin_nblk[w] = (int32_t)((len + BT - 1) / BT);
      } else {
        const int64_t freed = pl < 0 ? 0 : pl;
        if (out_freed) out_freed[r] = freed;
        occ_freed += freed;
        a.pin_len[w] = -1;
        a.pin_nblk[w] = 0;
      }
    }
  }
  if (lane == 0 && occ_freed) atomic_add_i64(&a.ctr->occupancy, -occ_freed);
  freed_blocks = __reduce_add_sync(0xffffffffu, freed_blocks);
  left_table = __reduce_add_sync(0xffffffffu, left_table);
  if (lane == 0 && freed_blocks) {
    atomic_add_i64(&a.ctr->blocks_in_use, -(long long)freed_blocks);
    if (left_table) {
      atomic_add_i64(&a.ctr->table_live, -(long long)left_table);
      atomic_add_i64(&a.ctr->table_tomb, (long long)left_table);
    }
  }
}

// A batch that aborted after admission (physical pool or table exhausted) leaves the pool as it
// was: pins, blocks and refcounts are untouched by then; the admission counters roll back and
// every request reports the error. Claimed-but-unfilled table keys are reclaimed by the next
// batch that probes them (they read as in-batch claims).
__global__ void commit_finish_kernel(CommitArgs a) {
  pdl_enter();
  const int err = a.ctr->error;
  if (err != SFKV_EPOOL) return;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.n;
       r += (int64_t)gridDim.x * blockDim.x)
    a.s.status[r] = SFKV_EPOOL;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctr->occupancy = a.ctr->occ_saved;
    a.ctr->rejections = a.ctr->rej_saved;
  }
}

__global__ void install_kernel(CommitArgs a) {
  pdl_enter();
  if (a.ctr->error) return;
  FOR_ITEMS(a, item) {
    if (a.s.cat[item] == CAT_NONE) continue;
    const int64_t r = upper_index(a.s.blk_off, a.n, item);
    const int64_t k = item - a.s.blk_off[r];
    const int64_t pb = (int64_t)a.wf[r] * a.max_pin_blocks;
    const int32_t id = a.s.bid[item];
    a.pin_blk[pb + k] = id;
    const uint8_t cat = a.s.cat[item];
    if (cat == CAT_OWN || cat == CAT_PRIV) a.blk_parent[id] = k > 0 ? a.s.bid[item - 1] : -1;
    // pin-major token copy (zero padded), read by the match kernel without indirection
    const int64_t rem = a.tok_off[r + 1] - a.tok_off[r] - k * BT;
    uint32_t t[BT];
    load_req_block(a, r, k, (int)(rem < BT ? rem : BT), t);
    uint4* dst = reinterpret_cast<uint4*>(a.pin_tok + pin_tok_index(a.wf[r], k, 0, a.pin_groups));
#pragma unroll
    for (int i = 0; i < 4; ++i)
      dst[(i + pin_rot(k)) & 3] = make_uint4(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);
  }
}

// ---- table maintenance: rebuild when tombstones exceed a quarter of the slots ------------
__global__ void rebuild_check_kernel(DevCounters* c, int64_t slots, int* flag) {
  pdl_enter();
  *flag = (c->table_tomb * 4 > slots) ? 1 : 0;
}
__global__ void table_clear_kernel(Slot* slots, int64_t* towner, int64_t n, const int* flag) {
  pdl_enter();
  if (!*flag) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    slots[i].key = KEY_EMPTY;
    slots[i].val = -1;
    towner[i] = NO_OWNER;
  }
}
__global__ void table_reinsert_kernel(CommitArgs a, const int* flag) {
  pdl_enter();
  if (!*flag) return;
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < a.n_blocks;
       id += (int64_t)gridDim.x * blockDim.x) {
    if (!a.blk_in_table[id]) continue;
    const unsigned long long c = a.blk_key[id];
    uint64_t s = c & a.slot_mask;
    for (;;) {
      if (atomicCAS(&a.slots[s].key, KEY_EMPTY, c) == KEY_EMPTY) {
        a.slots[s].val = (int32_t)id;
        a.blk_slot[id] = (int64_t)s;
        break;
      }
      s = (s + 1) & a.slot_mask;
    }
  }
}
__global__ void rebuild_done_kernel(DevCounters* c, const int* flag) {
  pdl_enter();
  if (*flag) c->table_tomb = 0;
}

// ---------------------------------------------------------------------------------------
static CommitArgs base_args(sfkv_pool* p) {
  CommitArgs a{};
  a.pin_len = p->pin_len;
  a.pin_nblk = p->pin_nblk;
  a.pin_blk = p->pin_blk;
  a.pin_tok = p->pin_tok;
  a.pin_groups = pin_groups(p->cfg);
  a.blk_key = p->blk_key;
  a.blk_parent = p->blk_parent;
  a.blk_tok = p->blk_tok;
  a.blk_n = p->blk_n;
  a.blk_in_table = p->blk_in_table;
  a.blk_ref = p->blk_ref;
  a.blk_slot = p->blk_slot;
  a.free_bits = p->free_bits;
  a.slots = p->slots;
  a.towner = p->towner;
  a.slot_mask = (uint64_t)p->table_slots - 1;
  a.n_words = p->n_words;
  a.n_blocks = p->cfg.n_blocks;
  a.max_pin_blocks = p->cfg.max_pin_blocks;
  a.max_wf = p->cfg.max_workflows;
  a.capacity = p->cfg.capacity_tokens;
  a.ctr = p->ctr;
  return a;
}

static int sm_count_c() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int maybe_rebuild_table(sfkv_pool* p, cudaStream_t st) {
  CommitArgs a = base_args(p);
  int* flag = &p->ctr->pad;
  SFKV_CUDA(launch_pdl(rebuild_check_kernel, dim3(1), dim3(1), st, p->ctr, p->table_slots, flag));
  const int sms = sm_count_c();
  SFKV_CUDA(launch_pdl(table_clear_kernel, dim3(sms * 4), dim3(256), st, p->slots, p->towner, p->table_slots, (const int*)flag));
  SFKV_CUDA(launch_pdl(table_reinsert_kernel, dim3(sms * 4), dim3(256), st, a, (const int*)flag));
  SFKV_CUDA(launch_pdl(rebuild_done_kernel, dim3(1), dim3(1), st, p->ctr, (const int*)flag));
  SFKV_LAUNCH_CHECK("table rebuild");
  return 0;
}

__global__ void one_flag_kernel(int* flag) { *flag = 1; }

int rebuild_table_now(sfkv_pool* p) {
  cudaStream_t st = p->stream;
  CommitArgs a = base_args(p);
  int* flag = &p->ctr->pad;
  one_flag_kernel<<<1, 1, 0, st>>>(flag);
  const int sms = sm_count_c();
  table_clear_kernel<<<sms * 4, 256, 0, st>>>(p->slots, p->towner, p->table_slots, flag);
  table_reinsert_kernel<<<sms * 4, 256, 0, st>>>(a, flag);
  rebuild_done_kernel<<<1, 1, 0, st>>>(p->ctr, flag);
  SFKV_LAUNCH_CHECK("table rebuild (resize)");
  return 0;
}

static int launch_commit_payload(sfkv_pool* p, const CommitArgs& a, const void* kv_src,
                                 const int64_t* kv_src_off, const PayloadSource* src,
                                 cudaStream_t st) {
  PayloadJob j;
  j.n = a.n;
  j.wf = a.wf;
  j.tok_off = a.tok_off;
  j.blk_off = a.s.blk_off;
  j.M = a.s.M;
  j.rank = a.s.rank;
  j.alloc_list = a.s.alloc_list;
  j.bid = a.s.bid;
  j.n_items = a.n_items;  // rank[bound] = number of new blocks
  j.cow_src = a.s.cow_src;
  j.error = &p->ctr->error;
  return launch_payload(p, j, kv_src, kv_src_off, src, st);
}

int commit_dev(sfkv_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
               const uint32_t* tok, int64_t n_items_bound, int64_t n_tok_bound, const void* kv_src,
               const int64_t* kv_src_off, const int64_t* m_expected, int32_t* out_status,
               const PayloadSource* src) {
  if (n <= 0) return 0;
  cudaStream_t st = p->stream;
  const int64_t ni = n_items_bound > 0 ? n_items_bound : 1;
  Carver cv;
  const size_t o_blk = cv.take<int64_t>(n + 1), o_M = cv.take<int64_t>(n),
               o_hash = cv.take<uint64_t>(ni), o_tile = cv.take<int64_t>(match_tile_state_elems(ni, n)),
               o_st = cv.take<int32_t>(n), o_slot = cv.take<int64_t>(ni),
               o_bid = cv.take<int32_t>(ni), o_hit = cv.take<uint8_t>(ni),
               o_claim = cv.take<uint8_t>(ni), o_cat = cv.take<uint8_t>(ni),
               o_fnh = cv.take<int64_t>(n), o_fh = cv.take<int64_t>(n), o_dl = cv.take<int64_t>(n), o_rank = cv.take<int64_t>(ni + 1),
               o_wp = cv.take<int64_t>(p->n_words + 1), o_al = cv.take<int64_t>(ni), o_cow = cv.take<int32_t>(ni),
               o_tmp = cv.take<int64_t>(scan_scratch_elems(ni) + scan_scratch_elems(p->n_words) +
                                        scan_scratch_elems(n));
  if (int rc = p->scratch.ensure(cv.off)) return rc;
  char* base = p->scratch.as<char>();
  CommitArgs a = base_args(p);
  a.n = n;
  a.wf = wf;
  a.tok_off = tok_off;
  a.tok = tok;
  a.m_expected = m_expected;
  a.payload = (p->kv && (kv_src || src)) ? 1 : 0;
  a.n_items = ni;
  a.s.blk_off = reinterpret_cast<int64_t*>(base + o_blk);
  a.s.M = reinterpret_cast<int64_t*>(base + o_M);
  a.s.hash = reinterpret_cast<uint64_t*>(base + o_hash);
  a.s.tile_state = reinterpret_cast<int64_t*>(base + o_tile);
  a.s.status = out_status ? out_status : reinterpret_cast<int32_t*>(base + o_st);
  a.s.slot_of = reinterpret_cast<int64_t*>(base + o_slot);
  a.s.bid = reinterpret_cast<int32_t*>(base + o_bid);
  a.s.hit0 = reinterpret_cast<uint8_t*>(base + o_hit);
  a.s.claim = reinterpret_cast<uint8_t*>(base + o_claim);
  a.s.cat = reinterpret_cast<uint8_t*>(base + o_cat);
  a.s.first_nonhit = reinterpret_cast<int64_t*>(base + o_fnh);
  a.s.f_hit = reinterpret_cast<int64_t*>(base + o_fh);
  a.s.delta = reinterpret_cast<int64_t*>(base + o_dl);
  a.s.rank = reinterpret_cast<int64_t*>(base + o_rank);
  a.s.wprefix = reinterpret_cast<int64_t*>(base + o_wp);
  a.s.alloc_list = reinterpret_cast<int64_t*>(base + o_al);
  a.s.cow_src = reinterpret_cast<int32_t*>(base + o_cow);
  a.s.scan_tmp = reinterpret_cast<int64_t*>(base + o_tmp);

  if (!p->aux) {
    SFKV_CUDA(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking));
    SFKV_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    SFKV_CUDA(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  }
  // 0. the free-bitmap prefix (allocation order) depends only on the pool before this batch: it
  //    runs on the aux stream beside the match / admission / classification and joins before alloc
  int64_t* tmp_free = a.s.scan_tmp + scan_scratch_elems(ni);
#if SFKV_FREE_FORK
  SFKV_CUDA(cudaEventRecord(p->ev_fork, st));
  SFKV_CUDA(cudaStreamWaitEvent(p->aux, p->ev_fork, 0));
  if (int rc = exclusive_scan(FreeCount{p->free_bits}, p->n_words, a.s.wprefix, tmp_free, p->aux)) return rc;
  SFKV_CUDA(cudaEventRecord(p->ev_join, p->aux));
#else
  if (int rc = exclusive_scan(FreeCount{p->free_bits}, p->n_words, a.s.wprefix, tmp_free, st)) return rc;
#endif
  // 1. blocks per request, chained hashes, M = LCP(old pin, tokens)
  MatchArgs m{};  // the match launch also writes blk_off (its prep kernel scans the requests)
  m.n = n;
  m.wf = wf;
  m.tok_off = tok_off;
  m.tok = tok;
  m.blk_off = a.s.blk_off;
  m.n_items = ni;
  m.n_tok_bound = n_tok_bound;
  m.out_M = a.s.M;
  m.out_hash = a.s.hash;
  if (int rc = launch_match(p, m, a.s.tile_state, st)) return rc;
  // 2. admission, classification, allocation, references
  SFKV_CUDA(launch_pdl(admit_kernel, dim3(1), dim3(ADMIT_THREADS), st, a));
  SFKV_LAUNCH_CHECK("admit_kernel");
  const int sms = sm_count_c();
  const int g = grid_for(ni, 256, sms * 8);
  SFKV_CUDA(launch_pdl(probe_kernel, dim3(g), dim3(256), st, a));
  SFKV_CUDA(launch_pdl(resolve_hits_kernel, dim3(g), dim3(256), st, a));
  SFKV_CUDA(launch_pdl(resolve_dups_kernel, dim3(g), dim3(256), st, a));
  SFKV_CUDA(launch_pdl(categorize_kernel, dim3(g), dim3(256), st, a));
  SFKV_LAUNCH_CHECK("probe/resolve/categorize");
  if (int rc = exclusive_scan(NeedAlloc{a.s.cat}, ni, a.s.rank, a.s.scan_tmp, st)) return rc;
#if SFKV_FREE_FORK
  SFKV_CUDA(cudaStreamWaitEvent(st, p->ev_join, 0));  // the free-bitmap prefix
#endif
  SFKV_CUDA(launch_pdl(alloc_kernel, dim3(g), dim3(256), st, a));
  SFKV_CUDA(launch_pdl(refs_kernel, dim3(g), dim3(256), st, a));
  SFKV_CUDA(launch_pdl(clear_owner_kernel, dim3(g), dim3(256), st, a));
  SFKV_LAUNCH_CHECK("alloc/refs");
  // 3. payload (copy-on-share + staging scatter / handoff pull) on the pool stream while
  // 4. the old pins are released and the new ones installed on the aux stream: the payload reads
  //    only the batch's own arrays (copy-on-share sources were snapshotted by alloc_kernel), and
  //    freed blocks cannot be reallocated before the join
  cudaStream_t meta = st;
  if (a.payload) {
    SFKV_CUDA(cudaEventRecord(p->ev_fork, st));
    SFKV_CUDA(cudaStreamWaitEvent(p->aux, p->ev_fork, 0));
    meta = p->aux;
    if (int rc = launch_commit_payload(p, a, kv_src, kv_src_off, src, st)) return rc;
  }
  SFKV_CUDA(launch_pdl(release_kernel, dim3(grid_for(n * 32, REL_THREADS, sms * 8 * (256 / REL_THREADS))), dim3(REL_THREADS), meta, a, 0, (int64_t*)nullptr));
  SFKV_CUDA(launch_pdl(install_kernel, dim3(g), dim3(256), meta, a));
  SFKV_CUDA(launch_pdl(commit_finish_kernel, dim3(grid_for(n, 256, sms)), dim3(256), meta, a));
  SFKV_LAUNCH_CHECK("release/install");
  // the tombstone check / rebuild touches only the table: it follows the release on the aux stream,
  // beside the payload copy, and the join orders it before anything later on the pool stream
#if SFKV_REBUILD_AUX
  if (int rc = maybe_rebuild_table(p, meta)) return rc;
#endif
  if (meta != st) {
    SFKV_CUDA(cudaEventRecord(p->ev_join, meta));
    SFKV_CUDA(cudaStreamWaitEvent(st, p->ev_join, 0));
  }
#if !SFKV_REBUILD_AUX
  if (int rc = maybe_rebuild_table(p, st)) return rc;
#endif
  return 0;
}

int flush_dev(sfkv_pool* p, int64_t n, const int32_t* wf, int64_t* out_freed, bool all) {
  cudaStream_t st = p->stream;
  CommitArgs a = base_args(p);
  a.n = all ? p->cfg.max_workflows : n;
  a.wf = wf;
  if (a.n <= 0) return 0;
  const int sms = sm_count_c();
  release_kernel<<<grid_for(a.n * 32, REL_THREADS, sms * 8 * (256 / REL_THREADS)), REL_THREADS, 0, st>>>(a, all ? 2 : 1, out_freed);
  SFKV_LAUNCH_CHECK("flush release_kernel");
  return maybe_rebuild_table(p, p->stream);
}

}  // namespace sfkv

/*
 * sfkv_oracle.c — CPU restatement (TEST INFRASTRUCTURE ONLY; see sfkv_oracle.h).
 *
 * Reference citations are relative to /root/reference/proj.
 *   pins / prefix_match  simulated_backend.cpp:153-162 (LCP against the workflow's own pin)
 *   pin_prompt           simulated_backend.cpp:135-151 (replace pin; reject iff
 *                        occupancy - old + new > capacity, old pin kept)
 *   flush                simulated_backend.cpp:169-184
 *   preserve             simulated_backend.cpp:190-193 (presence check, counts the call)
 *   cache_utilization    simulated_backend.cpp:186-188
 *   pressure_actions     memory.cpp:150-169 (strict > tau, strict < on ts, ties -> first id)
 *   map_threshold        mapper.cpp:19-31 (light iff score <= threshold)
 *   reroute_on_overload  orchestrator.cpp:78-87
 * Batch semantics (the definition the GPU kernels must reproduce) are stated at each function.
 */
#include "sfkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define BT 16
#define KEY_EMPTY 0ull

/* ---------------------------------------------------------------- chained block hash ---- */

static uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

/* digest(k, n, t) (the definition in include/sfkv.h): tokens at i >= n read as 0;
 * K_s[j] = 32-bit slice s (0 = low, 1 = high) of mix64(16 s + j + 1);
 * acc_s = sum_{i<8} (t[2i] + K_s[2i] mod 2^32) * (t[2i+1] + K_s[2i+1] mod 2^32) mod 2^64;
 * digest = mix64(acc_0 ^ rotl64(acc_1, 32) ^ (k*H + n)). */
static uint32_t nh_key(int set, int j) {
  uint64_t m = mix64((uint64_t)(set * 16 + j + 1));
  return (uint32_t)(set ? m >> 32 : m);
}

uint64_t sfo_block_digest(uint64_t k, uint32_t n, const uint32_t* t) {
  uint64_t acc[2] = {0, 0};
  for (int s = 0; s < 2; ++s) {
    for (uint32_t i = 0; i < 8; ++i) {
      uint32_t lo = (2 * i < n) ? t[2 * i] : 0;
      uint32_t hi = (2 * i + 1 < n) ? t[2 * i + 1] : 0;
      uint32_t a = lo + nh_key(s, (int)(2 * i));
      uint32_t b = hi + nh_key(s, (int)(2 * i + 1));
      acc[s] += (uint64_t)a * (uint64_t)b;
    }
  }
  uint64_t rot = (acc[1] << 32) | (acc[1] >> 32);
  return mix64(acc[0] ^ rot ^ (k * 0xD6E8FEB86659FD93ull + n));
}

/* chain(k) = fin(sum_{i<=k} digest(i) mod 2^62); keys 0 and 1 are reserved (empty / tombstone). */
uint64_t sfo_chain_finalize(uint64_t s) {
  uint64_t c = mix64((s & ((1ull << 62) - 1)) ^ 0x5851F42D4C957F2Dull);
  return c < 2 ? c + 2 : c;
}

void sfo_chain_hashes(const uint32_t* tok, int64_t len, uint64_t* out) {
  uint64_t s = 0;
  int64_t nb = (len + BT - 1) / BT;
  for (int64_t k = 0; k < nb; ++k) {
    int64_t n = len - k * BT;
    if (n > BT) n = BT;
    s += sfo_block_digest((uint64_t)k, (uint32_t)n, tok + k * BT);
    out[k] = sfo_chain_finalize(s);
  }
}

/* ---------------------------------------------------------------- key -> block map ---- */

typedef struct {
  uint64_t* key;
  int32_t* val;
  int64_t cap; /* power of two */
  int64_t live;
} kmap;

static int kmap_init(kmap* m, int64_t cap) {
  m->cap = 16;
  while (m->cap < 2 * cap) m->cap <<= 1;
  m->key = (uint64_t*)calloc((size_t)m->cap, sizeof(uint64_t));
  m->val = (int32_t*)malloc((size_t)m->cap * sizeof(int32_t));
  m->live = 0;
  return (m->key && m->val) ? 0 : -1;
}
static void kmap_free(kmap* m) {
  free(m->key);
  free(m->val);
}
static int64_t kmap_find(const kmap* m, uint64_t k) {
  int64_t i = (int64_t)(k & (uint64_t)(m->cap - 1));
  while (m->key[i] != KEY_EMPTY) {
    if (m->key[i] == k) return i;
    i = (i + 1) & (m->cap - 1);
  }
  return -1;
}
static int32_t kmap_get(const kmap* m, uint64_t k) {
  int64_t i = kmap_find(m, k);
  return i < 0 ? -1 : m->val[i];
}
static void kmap_put(kmap* m, uint64_t k, int32_t v) {
  int64_t i = (int64_t)(k & (uint64_t)(m->cap - 1));
  while (m->key[i] != KEY_EMPTY && m->key[i] != k) i = (i + 1) & (m->cap - 1);
  if (m->key[i] == KEY_EMPTY) m->live++;
  m->key[i] = k;
  m->val[i] = v;
}
/* Backward-shift deletion keeps linear probing exact without tombstones. */
static void kmap_del(kmap* m, uint64_t k) {
  int64_t i = kmap_find(m, k);
  if (i < 0) return;
  m->live--;
  int64_t j = i;
  for (;;) {
    m->key[i] = KEY_EMPTY;
    for (;;) {
      j = (j + 1) & (m->cap - 1);
      if (m->key[j] == KEY_EMPTY) return;
      int64_t h = (int64_t)(m->key[j] & (uint64_t)(m->cap - 1));
      /* move j to i if h is cyclically outside (i, j] */
      if ((i <= j) ? ((i < h) && (h <= j)) : ((i < h) || (h <= j))) continue;
      break;
    }
    m->key[i] = m->key[j];
    m->val[i] = m->val[j];
    i = j;
  }
}

/* ---------------------------------------------------------------- pool ---- */

struct sfo_pool {
  sfo_pool_config cfg;
  /* pins (Class A): token copy per workflow slot; len -1 = no pin. */
  int64_t* pin_len;
  uint32_t** pin_tok;
  int32_t* pin_nblk;
  int32_t* pin_blk; /* [wf][max_pin_blocks] */
  uint64_t* pin_hash;
  /* blocks (Class B) */
  uint64_t* blk_key;
  int32_t* blk_parent; /* the block at index k-1 of the pin that allocated it (-1 at k = 0) */
  uint32_t* blk_tok; /* [block][16] */
  uint8_t* blk_n;
  uint8_t* blk_in_table;
  uint32_t* blk_ref;
  uint8_t* blk_free;
  kmap table;
  uint8_t* kv;
  int64_t block_bytes;
  /* counters */
  int64_t occupancy;
  uint64_t rejections, flush_calls, preserve_calls;
};

int sfo_pool_create(const sfo_pool_config* cfg, sfo_pool** out) {
  if (!cfg || !out || cfg->max_workflows <= 0 || cfg->n_blocks <= 0 || cfg->capacity_tokens <= 0 ||
      cfg->max_pin_blocks <= 0)
    return -1;
  sfo_pool* p = (sfo_pool*)calloc(1, sizeof(sfo_pool));
  p->cfg = *cfg;
  int64_t W = cfg->max_workflows, B = cfg->n_blocks, MB = cfg->max_pin_blocks;
  p->pin_len = (int64_t*)malloc((size_t)W * sizeof(int64_t));
  for (int64_t i = 0; i < W; ++i) p->pin_len[i] = -1;
  p->pin_tok = (uint32_t**)calloc((size_t)W, sizeof(uint32_t*));
  p->pin_nblk = (int32_t*)calloc((size_t)W, sizeof(int32_t));
  p->pin_blk = (int32_t*)calloc((size_t)(W * MB), sizeof(int32_t));
  p->pin_hash = (uint64_t*)calloc((size_t)(W * MB), sizeof(uint64_t));
  p->blk_key = (uint64_t*)calloc((size_t)B, sizeof(uint64_t));
  p->blk_parent = (int32_t*)malloc((size_t)B * sizeof(int32_t));
  for (int64_t i = 0; i < B; ++i) p->blk_parent[i] = -1;
  p->blk_tok = (uint32_t*)calloc((size_t)(B * BT), sizeof(uint32_t));
  p->blk_n = (uint8_t*)calloc((size_t)B, 1);
  p->blk_in_table = (uint8_t*)calloc((size_t)B, 1);
  p->blk_ref = (uint32_t*)calloc((size_t)B, sizeof(uint32_t));
  p->blk_free = (uint8_t*)malloc((size_t)B);
  memset(p->blk_free, 1, (size_t)B);
  kmap_init(&p->table, B);
  p->block_bytes = (int64_t)cfg->n_slabs * BT * cfg->slab_row_bytes;
  if (p->block_bytes > 0) p->kv = (uint8_t*)calloc((size_t)(B * p->block_bytes), 1);
  *out = p;
  return 0;
}

int sfo_pool_destroy(sfo_pool* p) {
  if (!p) return 0;
  for (int64_t i = 0; i < p->cfg.max_workflows; ++i) free(p->pin_tok[i]);
  free(p->pin_len); free(p->pin_tok); free(p->pin_nblk); free(p->pin_blk); free(p->pin_hash);
  free(p->blk_key); free(p->blk_parent); free(p->blk_tok); free(p->blk_n); free(p->blk_in_table); free(p->blk_ref);
  free(p->blk_free); kmap_free(&p->table); free(p->kv); free(p);
  return 0;
}

int sfo_pool_kv(sfo_pool* p, void** kv, int64_t* block_bytes) {
  *kv = p->kv;
  *block_bytes = p->block_bytes;
  return 0;
}

static int bad_wf(const sfo_pool* p, int32_t wf) { return wf < 0 || wf >= p->cfg.max_workflows; }

static int64_t lcp(const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb) {
  int64_t n = na < nb ? na : nb, i = 0;
  while (i < n && a[i] == b[i]) ++i;
  return i;
}

/* M[r] = LCP(pin[wf[r]], tokens_r), 0 without a pin (simulated_backend.cpp:153-162). */
int sfo_match_batch(sfo_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                    const uint32_t* tok, int64_t* out_M, uint64_t* out_hash) {
  int64_t hb = 0;
  for (int64_t r = 0; r < n; ++r) {
    if (bad_wf(p, wf[r])) return -1;
    int64_t len = tok_off[r + 1] - tok_off[r];
    const uint32_t* t = tok + tok_off[r];
    int64_t pl = p->pin_len[wf[r]];
    out_M[r] = pl < 0 ? 0 : lcp(p->pin_tok[wf[r]], pl, t, len);
    if (out_hash) {
      sfo_chain_hashes(t, len, out_hash + hb);
      hb += (len + BT - 1) / BT;
    }
  }
  return 0;
}

static int blk_tokens_eq(const sfo_pool* p, int32_t id, const uint32_t* t) {
  return p->blk_n[id] == BT && memcmp(p->blk_tok + (int64_t)id * BT, t, BT * sizeof(uint32_t)) == 0;
}

/* Global lookup: each FULL block's chained hash against the table, token-verified, and linked to
 * its predecessor: block k hits only if the resident block's parent is the block the table holds
 * for chained key k-1 (so a leading run of hits is an exact prefix, independent of the hash). */
int sfo_lookup_batch(sfo_pool* p, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                     int32_t* out_block, int64_t* out_hit_tokens) {
  int64_t ob = 0;
  for (int64_t r = 0; r < n; ++r) {
    int64_t len = tok_off[r + 1] - tok_off[r];
    const uint32_t* t = tok + tok_off[r];
    int64_t nb = (len + BT - 1) / BT, nfull = len / BT;
    uint64_t* h = (uint64_t*)malloc((size_t)(nb > 0 ? nb : 1) * sizeof(uint64_t));
    sfo_chain_hashes(t, len, h);
    int64_t lead = 0, run = 1;
    int32_t raw_prev = -1;
    for (int64_t k = 0; k < nb; ++k) {
      int32_t id = -1;
      if (k < nfull) {
        /* exact by induction: the resident block must hold these tokens AND descend from the
         * block the table holds for the previous chained key (its parent link) */
        const int32_t raw = kmap_get(&p->table, h[k]);
        id = raw;
        if (id >= 0 && (!blk_tokens_eq(p, id, t + k * BT) || (k > 0 && p->blk_parent[id] != raw_prev))) id = -1;
        raw_prev = raw;
      }
      out_block[ob++] = id;
      if (id < 0) run = 0;
      if (run) ++lead;
    }
    if (out_hit_tokens) out_hit_tokens[r] = lead * BT;
    free(h);
  }
  return 0;
}

static void release_block(sfo_pool* p, int32_t id) {
  if (--p->blk_ref[id] == 0) {
    p->blk_free[id] = 1;
    if (p->blk_in_table[id]) {
      kmap_del(&p->table, p->blk_key[id]);
      p->blk_in_table[id] = 0;
    }
  }
}

static void release_pin(sfo_pool* p, int32_t w) {
  if (p->pin_len[w] < 0) return;
  for (int32_t k = 0; k < p->pin_nblk[w]; ++k)
    release_block(p, p->pin_blk[(int64_t)w * p->cfg.max_pin_blocks + k]);
  p->occupancy -= p->pin_len[w];
  p->pin_len[w] = -1;
  p->pin_nblk[w] = 0;
  free(p->pin_tok[w]);
  p->pin_tok[w] = NULL;
}

/* Block categories of a commit item. */
enum { C_HIT = 0, C_DUP = 1, C_OWN = 2, C_PRIV = 3 };

/* Payload source of one token row of a new block. */
typedef struct {
  const uint8_t* staging;   /* staging base of this request (NULL: metadata only) */
  int64_t staging_rows;     /* P - M */
  int64_t m;                /* rows < m come from the old pin */
  const sfo_pool* cow_pool; /* pool holding the old pin / handoff source */
  const int32_t* cow_blk;   /* block table of that pin */
} row_src;

static void write_block_payload(sfo_pool* p, int32_t id, int64_t k, int64_t nvalid,
                                const row_src* s) {
  if (!p->kv) return;
  const int64_t row = p->cfg.slab_row_bytes, S = p->cfg.n_slabs;
  uint8_t* dst = p->kv + (int64_t)id * p->block_bytes;
  for (int64_t j = 0; j < nvalid; ++j) {
    int64_t pos = k * BT + j;
    for (int64_t sl = 0; sl < S; ++sl) {
      uint8_t* d = dst + (sl * BT + j) * row;
      if (pos < s->m) {
        const sfo_pool* q = s->cow_pool;
        int32_t sid = s->cow_blk[k];
        memcpy(d, q->kv + (int64_t)sid * q->block_bytes + (sl * BT + j) * row, (size_t)row);
      } else if (s->staging) {
        memcpy(d, s->staging + (sl * s->staging_rows + (pos - s->m)) * row, (size_t)row);
      }
    }
  }
}

/* Commit (sfkv.h: sfkv_commit_batch). Phase order of a batch:
 *   0. M_r = LCP(old pin, tokens) for every request; m_expected check (payload commits).
 *   1. admission in request order (simulated_backend.cpp:141-150).
 *   2. block categories against T0 = table at batch start, items in batch order (r, k):
 *        hit0 : full block, T0 has its chained key and the block's tokens are equal
 *        claim: full block whose key is not in T0; owner(key) = first claim item with that key
 *        dup  : claim item, owner earlier, tokens equal to the owner's
 *        f_r  : first block that is neither hit0 nor dup
 *        k < f_r -> HIT (T0 block) or DUP (owner's block)
 *        k >= f_r -> OWN if it is its key's owner (allocated + inserted), else PRIV (allocated)
 *      OWN/PRIV items take the lowest free block ids in batch order; every item takes a ref.
 *   3. payload of OWN/PRIV blocks (rows < M_r from the old pin's block: copy-on-share).
 *   4. old pins released (ref--, free and unindex at 0), new pins installed. */
static int commit_impl(sfo_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                       const uint32_t* tok, const void* kv_src, const int64_t* kv_src_off,
                       const int64_t* m_expected, int32_t* out_status,
                       const sfo_pool* src_pool, const int32_t* src_blk) {
  const int64_t MB = p->cfg.max_pin_blocks;
  for (int64_t r = 0; r < n; ++r) {
    if (bad_wf(p, wf[r])) return -1;
    for (int64_t q = 0; q < r; ++q)
      if (wf[q] == wf[r]) return -1; /* distinct slots per batch */
    int64_t len = tok_off[r + 1] - tok_off[r];
    if ((len + BT - 1) / BT > MB) return -5;
  }
  int64_t* M = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) {
    int64_t len = tok_off[r + 1] - tok_off[r];
    int64_t pl = p->pin_len[wf[r]];
    M[r] = pl < 0 ? 0 : lcp(p->pin_tok[wf[r]], pl, tok + tok_off[r], len);
    if (kv_src && m_expected && p->kv && m_expected[r] != M[r]) {
      free(M);
      return -6;
    }
  }
  /* 1. admission (counters saved: a batch that then exhausts the physical pool rolls back) */
  const int64_t occ_saved = p->occupancy;
  const uint64_t rej_saved = p->rejections;
  for (int64_t r = 0; r < n; ++r) {
    int64_t old = p->pin_len[wf[r]] < 0 ? 0 : p->pin_len[wf[r]];
    int64_t nw = tok_off[r + 1] - tok_off[r];
    if (p->occupancy - old + nw > p->cfg.capacity_tokens) {
      out_status[r] = 0;
      p->rejections++;
    } else {
      out_status[r] = 1;
      p->occupancy += nw - old;
    }
  }
  /* 2. items */
  int64_t n_items = 0;
  int64_t* item_off = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) {
    item_off[r] = n_items;
    if (out_status[r]) n_items += (tok_off[r + 1] - tok_off[r] + BT - 1) / BT;
  }
  item_off[n] = n_items;
  int64_t NI = n_items > 0 ? n_items : 1;
  uint64_t* key = (uint64_t*)malloc((size_t)NI * sizeof(uint64_t));
  int32_t* cat = (int32_t*)malloc((size_t)NI * sizeof(int32_t));
  int32_t* bid = (int32_t*)malloc((size_t)NI * sizeof(int32_t));
  int64_t* owner = (int64_t*)malloc((size_t)NI * sizeof(int64_t));
  uint8_t* hit0 = (uint8_t*)calloc((size_t)NI, 1);
  uint8_t* claim = (uint8_t*)calloc((size_t)NI, 1);
  kmap first_claim;
  kmap_init(&first_claim, NI);
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r]) continue;
    int64_t len = tok_off[r + 1] - tok_off[r];
    sfo_chain_hashes(tok + tok_off[r], len, key + item_off[r]);
    for (int64_t k = 0; k < item_off[r + 1] - item_off[r]; ++k) {
      int64_t it = item_off[r] + k;
      int64_t nv = len - k * BT;
      owner[it] = -1;
      if (nv < BT) continue;
      int32_t id = kmap_get(&p->table, key[it]);
      if (id >= 0) {
        if (blk_tokens_eq(p, id, tok + tok_off[r] + k * BT)) {
          hit0[it] = 1;
          bid[it] = id;
        }
      } else {
        claim[it] = 1;
        int32_t f = kmap_get(&first_claim, key[it]);
        if (f < 0) {
          kmap_put(&first_claim, key[it], (int32_t)it);
          f = (int32_t)it;
        }
        owner[it] = f;
      }
    }
  }
  kmap_free(&first_claim);
  /* item -> (request, block) for owners */
  int64_t* item_req = (int64_t*)malloc((size_t)NI * sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r)
    for (int64_t it = item_off[r]; it < item_off[r + 1]; ++it) item_req[it] = r;
  int64_t scan_free = 0;
  /* Exact sharing by parent links (a block is shared only when its whole prefix is): per request,
   *   f_hit = first k that is not a linked hit: hit0[k] && (k == 0 || (hit0[k-1] &&
   *           parent(bid[k]) == bid[k-1]))
   *   f     = first k >= f_hit that is not a linked dup: a claim whose owner o is earlier, with
   *           equal tokens, and k == 0, or the previous item is a dup of the owner's previous
   *           item (owner[it-1] == o-1), or (k == f_hit) the previous item and the owner's
   *           previous item are the same linked hit (o-1 < f_hit of the owner's request, same bid).
   * Every test reads only probe results and f_hit, so the GPU resolves it in two parallel passes. */
  int64_t* f_hit = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) {
    int64_t nb = item_off[r + 1] - item_off[r];
    f_hit[r] = nb;
    if (!out_status[r]) continue;
    for (int64_t k = 0; k < nb; ++k) {
      int64_t it = item_off[r] + k;
      int ok = hit0[it] && (k == 0 || (hit0[it - 1] && p->blk_parent[bid[it]] == bid[it - 1]));
      if (!ok) {
        f_hit[r] = k;
        break;
      }
    }
  }
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r]) continue;
    int64_t nb = item_off[r + 1] - item_off[r];
    int64_t f = nb;
    for (int64_t k = f_hit[r]; k < nb; ++k) {
      int64_t it = item_off[r] + k;
      int dup = 0;
      if (claim[it] && owner[it] < it) {
        int64_t o = owner[it], orq = item_req[o], ok = o - item_off[orq];
        dup = memcmp(tok + tok_off[orq] + ok * BT, tok + tok_off[r] + k * BT,
                     BT * sizeof(uint32_t)) == 0;
        if (dup && k > 0) {
          const int dup_link = k > f_hit[r] && claim[it - 1] && owner[it - 1] == o - 1;
          const int hit_link = k == f_hit[r] && ok - 1 < f_hit[orq] && bid[it - 1] == bid[o - 1];
          dup = dup_link || hit_link;
        }
      }
      if (!dup) {
        f = k;
        break;
      }
    }
    for (int64_t k = 0; k < nb; ++k) {
      int64_t it = item_off[r] + k;
      if (k < f_hit[r]) cat[it] = C_HIT;
      else if (k < f) cat[it] = C_DUP;
      else cat[it] = (claim[it] && owner[it] == it) ? C_OWN : C_PRIV;
    }
  }
  /* allocation: lowest free ids in batch order */
  for (int64_t it = 0; it < n_items; ++it) {
    if (cat[it] != C_OWN && cat[it] != C_PRIV) continue;
    while (scan_free < p->cfg.n_blocks && !p->blk_free[scan_free]) ++scan_free;
    if (scan_free >= p->cfg.n_blocks) {
      /* physical pool exhausted: the batch changes nothing (no block, pin or table entry has
       * been touched yet; the admission counters roll back), as sfkv_commit_batch */
      p->occupancy = occ_saved;
      p->rejections = rej_saved;
      free(f_hit);
      free(M); free(item_off); free(key); free(cat); free(bid); free(owner); free(hit0);
      free(claim); free(item_req);
      return -5;
    }
    bid[it] = (int32_t)scan_free++;
  }
  for (int64_t it = 0; it < n_items; ++it)
    if (cat[it] == C_DUP) bid[it] = bid[owner[it]];
  /* metadata of new blocks + refs */
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r]) continue;
    int64_t len = tok_off[r + 1] - tok_off[r];
    for (int64_t k = 0; k < item_off[r + 1] - item_off[r]; ++k) {
      int64_t it = item_off[r] + k;
      int32_t id = bid[it];
      if (cat[it] == C_OWN || cat[it] == C_PRIV) {
        int64_t nv = len - k * BT;
        if (nv > BT) nv = BT;
        p->blk_free[id] = 0;
        p->blk_key[id] = key[it];
        p->blk_n[id] = (uint8_t)nv;
        memset(p->blk_tok + (int64_t)id * BT, 0, BT * sizeof(uint32_t));
        memcpy(p->blk_tok + (int64_t)id * BT, tok + tok_off[r] + k * BT, (size_t)nv * sizeof(uint32_t));
        p->blk_ref[id] = 0;
        p->blk_in_table[id] = 0;
        if (cat[it] == C_OWN) {
          kmap_put(&p->table, key[it], id);
          p->blk_in_table[id] = 1;
        }
      }
    }
  }
  for (int64_t it = 0; it < n_items; ++it) p->blk_ref[bid[it]]++;
  /* parent links of the new blocks: the block chosen for the previous item of the request */
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r]) continue;
    for (int64_t k = 0; k < item_off[r + 1] - item_off[r]; ++k) {
      int64_t it = item_off[r] + k;
      if (cat[it] == C_OWN || cat[it] == C_PRIV) p->blk_parent[bid[it]] = k > 0 ? bid[it - 1] : -1;
    }
  }
  /* 3. payload */
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r] || !p->kv) continue;
    int64_t len = tok_off[r + 1] - tok_off[r];
    row_src s;
    int32_t w = wf[r];
    if (src_pool) { /* handoff: rows < M from dst's old pin, rows >= M from the source pin */
      s.staging = NULL;
      s.staging_rows = 0;
    } else {
      s.staging = kv_src ? (const uint8_t*)kv_src + kv_src_off[r] : NULL;
      s.staging_rows = len - M[r];
    }
    s.m = M[r];
    s.cow_pool = p;
    s.cow_blk = p->pin_blk + (int64_t)w * MB;
    for (int64_t k = 0; k < item_off[r + 1] - item_off[r]; ++k) {
      int64_t it = item_off[r] + k;
      if (cat[it] != C_OWN && cat[it] != C_PRIV) continue;
      int64_t nv = len - k * BT;
      if (nv > BT) nv = BT;
      if (src_pool) {
        /* per row: < M from own old pin, else from the source pin's block k */
        const int64_t row = p->cfg.slab_row_bytes, S = p->cfg.n_slabs;
        uint8_t* dst = p->kv + (int64_t)bid[it] * p->block_bytes;
        for (int64_t j = 0; j < nv; ++j) {
          int64_t pos = k * BT + j;
          for (int64_t sl = 0; sl < S; ++sl) {
            const uint8_t* src =
                pos < M[r] ? p->kv + (int64_t)s.cow_blk[k] * p->block_bytes
                           : src_pool->kv + (int64_t)src_blk[k] * src_pool->block_bytes;
            memcpy(dst + (sl * BT + j) * row, src + (sl * BT + j) * row, (size_t)row);
          }
        }
      } else {
        write_block_payload(p, bid[it], k, nv, &s);
      }
    }
  }
  /* 4. release old pins, install new */
  for (int64_t r = 0; r < n; ++r) {
    if (!out_status[r]) continue;
    int32_t w = wf[r];
    int64_t len = tok_off[r + 1] - tok_off[r];
    int64_t saved_occ = p->occupancy;
    release_pin(p, w); /* adjusts occupancy; admission already accounted, restore below */
    p->occupancy = saved_occ;
    int64_t nb = item_off[r + 1] - item_off[r];
    p->pin_len[w] = len;
    p->pin_nblk[w] = (int32_t)nb;
    p->pin_tok[w] = (uint32_t*)malloc((size_t)(len > 0 ? len : 1) * sizeof(uint32_t));
    memcpy(p->pin_tok[w], tok + tok_off[r], (size_t)len * sizeof(uint32_t));
    for (int64_t k = 0; k < nb; ++k) {
      p->pin_blk[(int64_t)w * MB + k] = bid[item_off[r] + k];
      p->pin_hash[(int64_t)w * MB + k] = key[item_off[r] + k];
    }
  }
  free(M); free(item_off); free(key); free(cat); free(bid); free(owner); free(hit0); free(claim);
  free(item_req); free(f_hit);
  return 0;
}

int sfo_commit_batch(sfo_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                     const uint32_t* tok, const void* kv_src, const int64_t* kv_src_off,
                     const int64_t* m_expected, int32_t* out_status) {
  return commit_impl(p, n, wf, tok_off, tok, kv_src, kv_src_off, m_expected, out_status, NULL,
                     NULL);
}

/* flush (simulated_backend.cpp:169-184). */
int sfo_flush(sfo_pool* p, int32_t wf, int64_t* freed) {
  p->flush_calls++;
  if (wf == -1) {
    *freed = p->occupancy;
    for (int32_t w = 0; w < p->cfg.max_workflows; ++w) release_pin(p, w);
    p->occupancy = 0;
    return 0;
  }
  if (bad_wf(p, wf)) return -1;
  *freed = p->pin_len[wf] < 0 ? 0 : p->pin_len[wf];
  release_pin(p, wf);
  return 0;
}

int sfo_flush_batch(sfo_pool* p, int64_t n, const int32_t* wf, int64_t* out_freed) {
  for (int64_t r = 0; r < n; ++r) {
    if (bad_wf(p, wf[r])) return -1;
    for (int64_t q = 0; q < r; ++q)
      if (wf[q] == wf[r]) return -1;
  }
  for (int64_t r = 0; r < n; ++r) sfo_flush(p, wf[r], &out_freed[r]);
  return 0;
}

int sfo_preserve(sfo_pool* p, int32_t wf, int32_t* has_pin) {
  if (bad_wf(p, wf)) return -1;
  p->preserve_calls++;
  *has_pin = p->pin_len[wf] >= 0;
  return 0;
}

int sfo_pinned_token_count(sfo_pool* p, int32_t wf, int64_t* n_tokens) {
  if (bad_wf(p, wf)) return -1;
  *n_tokens = p->pin_len[wf] < 0 ? 0 : p->pin_len[wf];
  return 0;
}

int sfo_cache_utilization(sfo_pool* p, double* util) {
  *util = (double)p->occupancy / (double)p->cfg.capacity_tokens;
  return 0;
}

int sfo_stats(sfo_pool* p, sfo_pool_stats* o) {
  o->occupancy_tokens = p->occupancy;
  o->capacity_tokens = p->cfg.capacity_tokens;
  o->capacity_rejections = p->rejections;
  o->flush_calls = p->flush_calls;
  o->preserve_calls = p->preserve_calls;
  int64_t used = 0;
  for (int64_t b = 0; b < p->cfg.n_blocks; ++b) used += p->blk_ref[b] > 0;
  o->blocks_in_use = used;
  o->table_live = p->table.live;
  o->table_tombstones = 0;
  return 0;
}

int sfo_pin_blocks(sfo_pool* p, int32_t wf, int32_t* ids, uint64_t* hashes, int32_t cap,
                   int32_t* n_blocks) {
  if (bad_wf(p, wf)) return -1;
  int32_t nb = p->pin_len[wf] < 0 ? 0 : p->pin_nblk[wf];
  *n_blocks = nb;
  for (int32_t k = 0; k < nb && k < cap; ++k) {
    if (ids) ids[k] = p->pin_blk[(int64_t)wf * p->cfg.max_pin_blocks + k];
    if (hashes) hashes[k] = p->pin_hash[(int64_t)wf * p->cfg.max_pin_blocks + k];
  }
  return 0;
}

int sfo_pin_tokens(sfo_pool* p, int32_t wf, uint32_t* out, int64_t cap, int64_t* n_tokens) {
  if (bad_wf(p, wf)) return -1;
  int64_t L = p->pin_len[wf] < 0 ? 0 : p->pin_len[wf];
  *n_tokens = L;
  for (int64_t i = 0; i < L && i < cap; ++i) out[i] = p->pin_tok[wf][i];
  return 0;
}

int sfo_block_refcounts(sfo_pool* p, uint32_t* out) {
  memcpy(out, p->blk_ref, (size_t)p->cfg.n_blocks * sizeof(uint32_t));
  return 0;
}

/* gather: request r's pin at dst + dst_off[r], layout [slab][token][row]. */
int sfo_gather(sfo_pool* p, int64_t n, const int32_t* wf, void* dst, const int64_t* dst_off) {
  if (!p->kv) return -1;
  const int64_t row = p->cfg.slab_row_bytes, S = p->cfg.n_slabs;
  for (int64_t r = 0; r < n; ++r) {
    if (bad_wf(p, wf[r])) return -1;
    int64_t L = p->pin_len[wf[r]];
    if (L <= 0) continue;
    uint8_t* d = (uint8_t*)dst + dst_off[r];
    for (int64_t pos = 0; pos < L; ++pos) {
      int32_t id = p->pin_blk[(int64_t)wf[r] * p->cfg.max_pin_blocks + pos / BT];
      for (int64_t sl = 0; sl < S; ++sl)
        memcpy(d + (sl * L + pos) * row,
               p->kv + (int64_t)id * p->block_bytes + (sl * BT + pos % BT) * row, (size_t)row);
    }
  }
  return 0;
}

/* handoff: commit src's pin into dst; payload rows from dst's old pin (< M) or the source pin. */
int sfo_handoff(sfo_pool* src, int32_t wf_src, sfo_pool* dst, int32_t wf_dst, int32_t* status) {
  if (bad_wf(src, wf_src) || bad_wf(dst, wf_dst)) return -1;
  if (src->cfg.n_slabs != dst->cfg.n_slabs || src->cfg.slab_row_bytes != dst->cfg.slab_row_bytes)
    return -1;
  int64_t L = src->pin_len[wf_src];
  if (L < 0) {
    *status = 0;
    return -1;
  }
  int64_t off[2] = {0, L};
  int32_t w = wf_dst;
  return commit_impl(dst, 1, &w, off, src->pin_tok[wf_src], NULL, NULL, NULL, status, src,
                     src->pin_blk + (int64_t)wf_src * src->cfg.max_pin_blocks);
}

/* pressure_actions (memory.cpp:150-169): per backend with util > tau (strict), the preserved
 * entry with zero in-flight and minimum (last_update_ts, workflow id order). The reference scans
 * entries in workflow-id order and replaces only on strict <, i.e. ties go to the smallest id. */
int sfo_pressure_argmin(int64_t n, const int32_t* backend, const double* ts,
                        const uint32_t* wf_rank, const int32_t* in_flight,
                        const uint8_t* preserved, int32_t n_backends, const double* util,
                        double tau, int64_t* out_victim) {
  for (int32_t b = 0; b < n_backends; ++b) out_victim[b] = -1;
  for (int32_t b = 0; b < n_backends; ++b) {
    if (!(util[b] > tau)) continue;
    int64_t best = -1;
    for (int64_t i = 0; i < n; ++i) {
      if (backend[i] != b || !preserved[i] || in_flight[i] > 0) continue;
      if (best < 0 || ts[i] < ts[best] || (ts[i] == ts[best] && wf_rank[i] < wf_rank[best]))
        best = i;
    }
    out_victim[b] = best;
  }
  return 0;
}

/* map_threshold (mapper.cpp:19-31): light (0) iff score <= threshold. */
int sfo_threshold_batch(int64_t n, const double* score, double threshold, int32_t* out_choice) {
  for (int64_t r = 0; r < n; ++r) out_choice[r] = score[r] <= threshold ? 0 : 1;
  return 0;
}

/* N-candidate cost + reroute_on_overload (orchestrator.cpp:78-87), sequential in request order. */
int sfo_cost_batch(int64_t n, int32_t c, const int64_t* P, const int64_t* M, const int64_t* O,
                   const double* overhead, const double* prefill, const double* decode,
                   const double* queue_penalty, const int32_t* alternates, uint64_t* depth,
                   uint64_t limit, int32_t* out_choice, double* out_cost) {
  /* Costs see the batch-start depth snapshot; reroute sees the live depth. */
  uint64_t* depth0 = (uint64_t*)malloc((size_t)c * sizeof(uint64_t));
  memcpy(depth0, depth, (size_t)c * sizeof(uint64_t));
  for (int64_t r = 0; r < n; ++r) {
    int32_t best = 0;
    double bc = 0;
    for (int32_t j = 0; j < c; ++j) {
      double cost = overhead[j] + prefill[j] * (double)(P[r] - M[r * c + j]) +
                    decode[j] * (double)O[r] + queue_penalty[j] * (double)depth0[j];
      if (j == 0 || cost < bc) {
        bc = cost;
        best = j;
      }
    }
    out_cost[r] = bc;
    int32_t pick = best;
    if (limit > 0 && depth[best] >= limit) {
      for (int32_t a = 0; alternates && a < c; ++a) {
        int32_t alt = alternates[best * c + a];
        if (alt < 0) break;
        if (depth[alt] < limit) {
          pick = alt;
          break;
        }
      }
    }
    out_choice[r] = pick;
    depth[pick]++;
  }
  free(depth0);
  return 0;
}


/* ================================================================ memory manager tracker ====
 * Restates MemoryManager (memory.cpp:233-387) over dense ids: workflow slots, backends in sorted
 * ref order (map iteration order of entries_ / utilization), per-workflow dense stage ids, model
 * ids. Signals are applied one at a time in batch order, exactly as on_signal. */
enum { K_START = 0, K_COMPLETE = 1, K_WF_COMPLETE = 2 };
enum { O_NONE = 0, O_PRESERVE = 1, O_FLUSH = 2 };
enum { P_PSI = 1, P_FAB = 2 };
enum { A_PRESERVE = 0, A_FLUSH = 1, A_NOOP = 2 };
enum { R_OVERRIDE = 0, R_PSI = 1, R_FAB = 2, R_PRESSURE = 3, R_EXHAUSTED = 4 };
struct sfo_tracker {
  sfo_mm_config cfg;
  int32_t W, NB, SW;
  uint32_t epoch;     /* operation counter: batches and ticks (flush-failure feedback) */
  uint8_t* def_chain; /* the default chain (copied) */
  uint8_t* completed;
  uint64_t* started;  /* started_ever_ (memory.hpp:165): [W][SW] */
  uint64_t* open_;    /* open_stages_: [W][SW] */
  int32_t* open_cnt;
  uint8_t* last_valid;
  int32_t* last_b;
  int32_t* last_model;
  int64_t* last_tokens;
  int32_t* chain_len; /* -1: default chain (workflow_chains_ has no entry) */
  uint8_t** chain;    /* per workflow, malloc'd */
  uint8_t* present;   /* entries_ [(wf, backend)] */
  uint8_t* preserved;
  int64_t* tokens;
  double* ts;
  int32_t* inflight;  /* in_flight_ [backend][wf] */
  uint64_t* mod;      /* tag of the last modification (see tracker.cu) */
  uint32_t* rank;
  int32_t* border;    /* backends in std::string order */
  uint8_t* failed;    /* per batch */
};

static uint64_t mod_tag(uint32_t epoch, int64_t sig, int kind) {
  return ((uint64_t)epoch << 32) | ((uint64_t)(sig & 0x7fffffff) << 1) | (uint64_t)kind;
}

/* (Re)allocates the shaped arrays for (W, NB, SW), copying the old contents. */
static int tracker_shape(sfo_tracker* t, int32_t W1, int32_t NB1, int32_t SW1) {
  const int32_t W0 = t->W, NB0 = t->NB, SW0 = t->SW;
  size_t W = (size_t)W1, E = W * (size_t)NB1, WS = W * (size_t)SW1;
  uint8_t* completed = calloc(W, 1);
  uint64_t* started = calloc(WS, 8);
  uint64_t* open_ = calloc(WS, 8);
  int32_t* open_cnt = calloc(W, 4);
  uint8_t* last_valid = calloc(W, 1);
  int32_t* last_b = calloc(W, 4);
  int32_t* last_model = calloc(W, 4);
  int64_t* last_tokens = calloc(W, 8);
  int32_t* chain_len = malloc(W * 4);
  uint8_t** chain = calloc(W, sizeof(uint8_t*));
  uint8_t* present = calloc(E, 1);
  uint8_t* preserved = calloc(E, 1);
  int64_t* tokens = calloc(E, 8);
  double* ts = calloc(E, 8);
  int32_t* inflight = calloc(E, 4);
  uint64_t* mod = calloc(E, 8);
  uint32_t* rank = calloc(W, 4);
  int32_t* border = malloc((size_t)NB1 * 4);
  uint8_t* failed = calloc(W, 1);
  for (int32_t w = 0; w < W1; ++w) {
    const int old = w < W0;
    completed[w] = old ? t->completed[w] : 0;
    for (int32_t q = 0; q < SW1; ++q) {
      started[(size_t)w * SW1 + q] = old && q < SW0 ? t->started[(size_t)w * SW0 + q] : 0;
      open_[(size_t)w * SW1 + q] = old && q < SW0 ? t->open_[(size_t)w * SW0 + q] : 0;
    }
    open_cnt[w] = old ? t->open_cnt[w] : 0;
    last_valid[w] = old ? t->last_valid[w] : 0;
    last_b[w] = old ? t->last_b[w] : -1;
    last_model[w] = old ? t->last_model[w] : -1;
    last_tokens[w] = old ? t->last_tokens[w] : 0;
    chain_len[w] = old ? t->chain_len[w] : -1;
    chain[w] = old ? t->chain[w] : NULL;
    rank[w] = old ? t->rank[w] : (uint32_t)w;
    for (int32_t b = 0; b < NB1; ++b) {
      const int ob = old && b < NB0;
      size_t e = (size_t)w * NB1 + b, f = (size_t)w * NB0 + b;
      present[e] = ob ? t->present[f] : 0;
      preserved[e] = ob ? t->preserved[f] : 0;
      tokens[e] = ob ? t->tokens[f] : 0;
      ts[e] = ob ? t->ts[f] : 0;
      inflight[e] = ob ? t->inflight[f] : 0;
      mod[e] = ob ? t->mod[f] : 0;
    }
  }
  for (int32_t b = 0; b < NB1; ++b) border[b] = b < NB0 ? t->border[b] : b;
  free(t->completed); free(t->started); free(t->open_); free(t->open_cnt); free(t->last_valid);
  free(t->last_b); free(t->last_model); free(t->last_tokens); free(t->chain_len); free(t->chain);
  free(t->present); free(t->preserved); free(t->tokens); free(t->ts); free(t->inflight);
  free(t->mod); free(t->rank); free(t->border); free(t->failed);
  t->completed = completed; t->started = started; t->open_ = open_; t->open_cnt = open_cnt;
  t->last_valid = last_valid; t->last_b = last_b; t->last_model = last_model;
  t->last_tokens = last_tokens; t->chain_len = chain_len; t->chain = chain; t->present = present;
  t->preserved = preserved; t->tokens = tokens; t->ts = ts; t->inflight = inflight; t->mod = mod;
  t->rank = rank; t->border = border; t->failed = failed;
  t->W = W1; t->NB = NB1; t->SW = SW1;
  return 0;
}

int sfo_tracker_create(const sfo_mm_config* cfg, sfo_tracker** out) {
  if (!cfg || !out || cfg->max_workflows <= 0 || cfg->n_backends <= 0 || cfg->max_stages < 0 ||
      cfg->chain_len < 0 || (cfg->chain_len && !cfg->chain) || cfg->tau <= 0 ||
      !(cfg->tau_pressure > 0) || cfg->tau_pressure > 1)
    return -1; /* memory.cpp:240-243 */
  for (int32_t i = 0; i < cfg->chain_len; ++i)
    if (cfg->chain[i] != P_PSI && cfg->chain[i] != P_FAB) return -1; /* memory.cpp:182 */
  sfo_tracker* t = (sfo_tracker*)calloc(1, sizeof(*t));
  t->cfg = *cfg;
  t->def_chain = malloc((size_t)(cfg->chain_len > 0 ? cfg->chain_len : 1));
  if (cfg->chain_len) memcpy(t->def_chain, cfg->chain, (size_t)cfg->chain_len);
  t->cfg.chain = t->def_chain;
  tracker_shape(t, cfg->max_workflows, cfg->n_backends, cfg->max_stages > 0 ? (cfg->max_stages + 63) / 64 : 1);
  *out = t;
  return 0;
}

int sfo_tracker_destroy(sfo_tracker* t) {
  if (!t) return -1;
  for (int32_t w = 0; w < t->W; ++w) free(t->chain[w]);
  free(t->completed); free(t->started); free(t->open_); free(t->open_cnt); free(t->last_valid);
  free(t->last_b); free(t->last_model); free(t->last_tokens); free(t->chain_len); free(t->chain);
  free(t->present); free(t->preserved); free(t->tokens); free(t->ts); free(t->inflight);
  free(t->mod); free(t->rank); free(t->border); free(t->failed); free(t->def_chain);
  free(t);
  return 0;
}

int sfo_tracker_reserve(sfo_tracker* t, int32_t max_workflows, int32_t n_backends, int32_t max_stages) {
  if (!t) return -1;
  int32_t W1 = max_workflows > t->W ? max_workflows : t->W;
  int32_t NB1 = n_backends > t->NB ? n_backends : t->NB;
  int32_t SW1 = max_stages > 0 ? (max_stages + 63) / 64 : 1;
  if (SW1 < t->SW) SW1 = t->SW;
  if (W1 == t->W && NB1 == t->NB && SW1 == t->SW) return 0;
  return tracker_shape(t, W1, NB1, SW1);
}

int sfo_tracker_shape(sfo_tracker* t, int32_t* max_workflows, int32_t* n_backends, int32_t* max_stages) {
  if (!t) return -1;
  if (max_workflows) *max_workflows = t->W;
  if (n_backends) *n_backends = t->NB;
  if (max_stages) *max_stages = t->SW * 64;
  return 0;
}

static void forget_workflow(sfo_tracker* t, int32_t w) {
  t->completed[w] = 0;
  for (int32_t q = 0; q < t->SW; ++q) t->started[(size_t)w * t->SW + q] = t->open_[(size_t)w * t->SW + q] = 0;
  t->open_cnt[w] = 0;
  t->last_valid[w] = 0;
  t->last_b[w] = -1;
  t->last_model[w] = -1;
  t->last_tokens[w] = 0;
  t->chain_len[w] = -1;
  free(t->chain[w]);
  t->chain[w] = NULL;
  for (int32_t b = 0; b < t->NB; ++b) {
    size_t e = (size_t)w * t->NB + b;
    t->present[e] = t->preserved[e] = 0;
    t->tokens[e] = 0;
    t->ts[e] = 0;
    t->inflight[e] = 0;
    t->mod[e] = 0;
  }
}

int sfo_reset_workflows(sfo_tracker* t, int64_t n, const int32_t* wf) {
  if (!t || n < 0 || (n && !wf)) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (wf[i] < 0 || wf[i] >= t->W) return -1;
  for (int64_t i = 0; i < n; ++i) forget_workflow(t, wf[i]);
  return 0;
}

int sfo_set_backend_order(sfo_tracker* t, int32_t n, const int32_t* order) {
  if (!t || n != t->NB || !order) return -1;
  for (int32_t k = 0; k < n; ++k) {
    if (order[k] < 0 || order[k] >= n) return -1;
    for (int32_t j = 0; j < k; ++j)
      if (order[j] == order[k]) return -1;
  }
  memcpy(t->border, order, (size_t)n * 4);
  return 0;
}

int sfo_flush_failed(sfo_tracker* t, int64_t n, const int32_t* wf, const int32_t* backend, const int64_t* sig) {
  if (!t || n < 0 || (n && (!wf || !backend || !sig))) return -1;
  for (int64_t i = 0; i < n; ++i)
    if (wf[i] < 0 || wf[i] >= t->W || backend[i] < 0 || backend[i] >= t->NB) return -1;
  for (int64_t i = 0; i < n; ++i) {
    size_t e = (size_t)wf[i] * t->NB + backend[i];
    if (t->mod[e] == mod_tag(t->epoch, sig[i] < 0 ? 0 : sig[i], 0)) { /* mark_unpreserved */
      t->present[e] = 1;
      t->preserved[e] = 0;
    }
  }
  return 0;
}

int sfo_set_workflow_chain(sfo_tracker* t, int32_t wf, int32_t len, const uint8_t* policies) {
  if (!t || wf < 0 || wf >= t->W || len < 0 || (len && !policies)) return -1;
  if (len == 0) return 0; /* memory.cpp:248 */
  for (int32_t i = 0; i < len; ++i)
    if (policies[i] != P_PSI && policies[i] != P_FAB) return -1; /* unknown policy */
  free(t->chain[wf]);
  t->chain[wf] = malloc((size_t)len);
  memcpy(t->chain[wf], policies, (size_t)len);
  t->chain_len[wf] = len;
  return 0;
}

int sfo_set_workflow_ranks(sfo_tracker* t, int64_t n, const uint32_t* rank) {
  if (!t || n < 0 || n > t->W || (n && !rank)) return -1;
  for (int64_t w = 0; w < n; ++w) t->rank[w] = rank[w];
  return 0;
}

typedef struct { uint8_t kind; int32_t b; uint8_t reason; } act_t;

/* policy_preserve_small_increment (memory.cpp:116-125) */
static int pol_psi(const sfo_tracker* t, int w, uint8_t kind, int32_t b, int32_t m, int64_t T, act_t* a) {
  if (kind != K_START || !t->last_valid[w]) return 0;
  if (t->last_b[w] != b || t->last_model[w] != m) return 0;
  if (T - t->last_tokens[w] >= t->cfg.tau) return 0;
  a[0].kind = A_PRESERVE;
  a[0].b = b;
  a[0].reason = R_PSI;
  return 1;
}

/* policy_flush_at_boundary (memory.cpp:127-148) */
static int pol_fab(const sfo_tracker* t, int w, uint8_t kind, int32_t b, int32_t m, act_t* a) {
  int n = 0;
  size_t e0 = (size_t)w * t->NB;
  if (kind == K_WF_COMPLETE) { /* preserved_entries(wf): map order = backend-ref order */
    for (int32_t k = 0; k < t->NB; ++k) {
      const int32_t bb = t->border[k];
      if (t->present[e0 + bb] && t->preserved[e0 + bb]) {
        a[n].kind = A_FLUSH;
        a[n].b = bb;
        a[n].reason = R_FAB;
        ++n;
      }
    }
    return n;
  }
  if (kind == K_START && t->last_valid[w] && (t->last_b[w] != b || t->last_model[w] != m)) {
    int32_t lb = t->last_b[w];
    if (t->present[e0 + lb] && t->preserved[e0 + lb]) {
      a[0].kind = A_FLUSH;
      a[0].b = lb;
      a[0].reason = R_FAB;
      n = 1;
    }
  }
  return n;
}

static int stage_bit(const uint64_t* words, int32_t s) { return (int)((words[s >> 6] >> (s & 63)) & 1u); }

int sfo_on_signal_batch(sfo_tracker* t, int64_t n, const sfo_signals* sg, const sfo_records* out) {
  if (!t || !sg || !out || n < 0) return -1;
  const int32_t NB = t->NB, SW = t->SW;
  act_t* acts = (act_t*)malloc(sizeof(act_t) * (size_t)(NB > 1 ? NB : 1));
  memset(t->failed, 0, (size_t)t->W);
  ++t->epoch;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t w = sg->wf[i];
    const uint8_t kind = sg->kind[i];
    const int32_t s = kind == K_WF_COMPLETE ? 0 : sg->stage[i];
    const int32_t b = kind == K_WF_COMPLETE ? -1 : sg->backend[i];
    const int32_t m = kind == K_WF_COMPLETE ? -1 : sg->model[i];
    const int64_t T = kind == K_WF_COMPLETE ? 0 : sg->tokens[i];
    const double ts = sg->ts[i];
    const uint8_t ov = sg->override_ ? sg->override_[i] : O_NONE;
    out->count[i] = 0;
    if (w < 0 || w >= t->W || kind > 2 ||
        (kind != K_WF_COMPLETE && (b < 0 || b >= NB || s < 0 || s >= SW * 64))) {
      free(acts);
      return -1;
    }
    if (t->failed[w]) {
      out->status[i] = 2;
      continue;
    }
    uint64_t* started = t->started + (size_t)w * SW;
    uint64_t* open_ = t->open_ + (size_t)w * SW;
    /* check_order (memory.cpp:256-285) */
    int bad = t->completed[w] || (kind == K_START && stage_bit(started, s)) ||
              (kind == K_COMPLETE && !stage_bit(open_, s)) ||
              (kind == K_WF_COMPLETE && t->open_cnt[w] != 0);
    if (!bad && kind == K_COMPLETE && t->inflight[(size_t)w * NB + b] <= 0) {
      /* adjust_in_flight(-1) would go negative: logic_error (memory.cpp:92) after logging */
      bad = 3;
    }
    if (bad == 1) { /* OutOfOrderSignalError: nothing resolved, applied or logged */
      out->status[i] = 1;
      t->failed[w] = 1;
      continue;
    }
    /* resolve (memory.cpp:287-310) */
    int na = 0;
    if (kind == K_START && ov != O_NONE) {
      if (!t->last_valid[w]) {
        acts[0].kind = A_NOOP; acts[0].b = -1; acts[0].reason = R_OVERRIDE;
      } else {
        acts[0].kind = ov == O_FLUSH ? A_FLUSH : A_PRESERVE;
        acts[0].b = t->last_b[w];
        acts[0].reason = R_OVERRIDE;
      }
      na = 1;
    } else {
      const int32_t len = t->chain_len[w] >= 0 ? t->chain_len[w] : t->cfg.chain_len;
      const uint8_t* ch = t->chain_len[w] >= 0 ? t->chain[w] : t->def_chain;
      for (int32_t p = 0; p < len && na == 0; ++p)
        na = ch[p] == P_PSI ? pol_psi(t, w, kind, b, m, T, acts) : pol_fab(t, w, kind, b, m, acts);
      if (na == 0) {
        acts[0].kind = A_NOOP; acts[0].b = -1; acts[0].reason = R_EXHAUSTED;
        na = 1;
      }
    }
    /* apply_and_record (memory.cpp:312-328): flushes are recorded as applied -> mark_flushed
     * (a failure reported later by sfo_flush_failed turns it into mark_unpreserved) */
    for (int a = 0; a < na; ++a) {
      out->kind[(size_t)i * NB + a] = acts[a].kind;
      out->backend[(size_t)i * NB + a] = acts[a].b;
      out->reason[(size_t)i * NB + a] = acts[a].reason;
      if (acts[a].kind == A_FLUSH) {
        t->present[(size_t)w * NB + acts[a].b] = 0;
        t->mod[(size_t)w * NB + acts[a].b] = mod_tag(t->epoch, i, 0);
      }
    }
    out->count[i] = na;
    if (bad == 3) { /* the records were logged, then update_tracker threw */
      out->status[i] = 3;
      t->failed[w] = 1;
      /* update_tracker erased the open stage, then adjust_in_flight stored -1 and threw
       * (memory.cpp:338-339, 90-92) */
      open_[s >> 6] &= ~(1ull << (s & 63));
      t->open_cnt[w] -= 1;
      t->inflight[(size_t)w * NB + b] -= 1;
      continue;
    }
    out->status[i] = 0;
    /* update_tracker (memory.cpp:330-360) */
    const size_t e = (size_t)w * NB + (b < 0 ? 0 : b);
    if (kind == K_START) {
      started[s >> 6] |= 1ull << (s & 63);
      open_[s >> 6] |= 1ull << (s & 63);
      t->open_cnt[w] += 1;
      t->inflight[e] += 1;
      if (t->inflight[e] < 0) { /* a count left negative by an earlier throw stays negative:
                                  * adjust_in_flight(+1) stores it and throws (memory.cpp:90-92) */
        out->status[i] = 3;
        t->failed[w] = 1;
      }
    } else if (kind == K_COMPLETE) {
      open_[s >> 6] &= ~(1ull << (s & 63));
      t->open_cnt[w] -= 1;
      t->inflight[e] -= 1;
      t->present[e] = 1;
      t->preserved[e] = T > 0;
      t->tokens[e] = T;
      t->ts[e] = ts;
      t->mod[e] = mod_tag(t->epoch, i, 1);
      t->last_valid[w] = 1;
      t->last_b[w] = b;
      t->last_model[w] = m;
      t->last_tokens[w] = T;
    } else {
      t->completed[w] = 1;
      for (int32_t bb = 0; bb < NB; ++bb) {
        t->present[(size_t)w * NB + bb] = 0;
        t->inflight[(size_t)w * NB + bb] = 0;
        t->mod[(size_t)w * NB + bb] = mod_tag(t->epoch, i, 1);
      }
      t->last_valid[w] = 0;
      for (int32_t q = 0; q < SW; ++q) started[q] = open_[q] = 0;
      t->open_cnt[w] = 0;
      t->chain_len[w] = -1;
      free(t->chain[w]);
      t->chain[w] = NULL;
    }
  }
  free(acts);
  return 0;
}

/* pressure_tick -> pressure_actions (memory.cpp:150-169, 382-387) */
int sfo_pressure_tick(sfo_tracker* t, const double* util, int32_t* out_victim) {
  if (!t || !util || !out_victim) return -1;
  ++t->epoch;
  for (int32_t b = 0; b < t->NB; ++b) {
    out_victim[b] = -1;
    if (!(util[b] > t->cfg.tau_pressure)) continue;
    int32_t best = -1;
    for (int32_t w = 0; w < t->W; ++w) {
      size_t e = (size_t)w * t->NB + b;
      if (!t->present[e] || !t->preserved[e] || t->inflight[e] > 0) continue;
      size_t eb = (size_t)best * t->NB + b;
      if (best < 0 || t->ts[e] < t->ts[eb] || (t->ts[e] == t->ts[eb] && t->rank[w] < t->rank[best]))
        best = w;
    }
    out_victim[b] = best;
  }
  for (int32_t b = 0; b < t->NB; ++b)
    if (out_victim[b] >= 0) { /* mark_flushed */
      size_t e = (size_t)out_victim[b] * t->NB + b;
      t->present[e] = 0;
      t->mod[e] = mod_tag(t->epoch, 0, 0);
    }
  return 0;
}

int sfo_tracker_entries(sfo_tracker* t, uint8_t* present, uint8_t* preserved, int64_t* tokens,
                        double* ts, int32_t* in_flight) {
  if (!t) return -1;
  size_t E = (size_t)t->W * t->NB;
  if (present) memcpy(present, t->present, E);
  if (preserved) memcpy(preserved, t->preserved, E);
  if (tokens) memcpy(tokens, t->tokens, E * 8);
  if (ts) memcpy(ts, t->ts, E * 8);
  if (in_flight) memcpy(in_flight, t->inflight, E * 4);
  return 0;
}


/* ================================================================ tokenizer + interner ======
 * tokenize_whitespace (backend.cpp:60-70): skip std::isspace bytes (C locale), take the maximal
 * run of non-space bytes as a token; context_token_sequence (backend.cpp:83-91) concatenates the
 * tokens of each message. Interning: a token string seen for the first time gets the next id,
 * in token order. (A plain open-addressing map over the strings themselves: no hashing shortcut
 * can make two different strings equal here.) */
struct sfo_interner {
  int64_t cap;      /* slots (power of two) */
  int64_t* slot;    /* id + 1, 0 = empty */
  uint8_t* arena;
  int64_t arena_cap, arena_used;
  int64_t* off;
  int32_t* len;
  int64_t n, max_ids;
};

static int sp(uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

static uint64_t str_hash(const uint8_t* p, int64_t n) { /* FNV-1a: only the map layout uses it */
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

int sfo_interner_create(int32_t device, int32_t table_log2, int64_t arena_bytes, sfo_interner** out) {
  (void)device;
  if (!out || table_log2 < 4 || table_log2 > 34 || arena_bytes <= 0) return -1;
  sfo_interner* it = (sfo_interner*)calloc(1, sizeof(*it));
  it->cap = (int64_t)1 << table_log2;
  it->max_ids = it->cap / 2;
  it->slot = (int64_t*)calloc((size_t)it->cap, sizeof(int64_t));
  it->arena = (uint8_t*)malloc((size_t)arena_bytes);
  it->arena_cap = arena_bytes;
  it->off = (int64_t*)malloc((size_t)it->max_ids * sizeof(int64_t));
  it->len = (int32_t*)malloc((size_t)it->max_ids * sizeof(int32_t));
  *out = it;
  return 0;
}

int sfo_interner_destroy(sfo_interner* it) {
  if (!it) return -1;
  free(it->slot); free(it->arena); free(it->off); free(it->len); free(it);
  return 0;
}

int sfo_interner_size(sfo_interner* it, int64_t* n_ids) {
  if (!it || !n_ids) return -1;
  *n_ids = it->n;
  return 0;
}

int sfo_interner_token(sfo_interner* it, uint32_t id, char* out, int32_t cap, int32_t* len) {
  if (!it || !len || (int64_t)id >= it->n) return -1;
  *len = it->len[id];
  if (cap > 0) memcpy(out, it->arena + it->off[id], (size_t)(it->len[id] < cap ? it->len[id] : cap));
  return 0;
}

/* id of p[0..n), inserting it (next id) when new; -1 when the interner is full */
static int64_t intern(sfo_interner* it, const uint8_t* p, int64_t n) {
  uint64_t m = (uint64_t)it->cap - 1, s = str_hash(p, n) & m;
  for (;;) {
    int64_t v = it->slot[s];
    if (!v) break;
    int64_t id = v - 1;
    if (it->len[id] == n && !memcmp(it->arena + it->off[id], p, (size_t)n)) return id;
    s = (s + 1) & m;
  }
  if (it->n >= it->max_ids || it->arena_used + n > it->arena_cap) return -1;
  int64_t id = it->n++;
  memcpy(it->arena + it->arena_used, p, (size_t)n);
  it->off[id] = it->arena_used;
  it->len[id] = (int32_t)n;
  it->arena_used += n;
  it->slot[s] = id + 1;
  return id;
}

int sfo_tokenize_batch(sfo_interner* it, int64_t n, const int64_t* req_msg_off, const int64_t* msg_off,
                       const uint8_t* text, int64_t* tok_off, uint32_t* tok, int64_t tok_cap,
                       int64_t* n_tokens) {
  if (!it || n < 0 || !req_msg_off || !tok_off || !n_tokens) return -1;
  /* all-or-nothing like the GPU: work on a copy of the interner state */
  int64_t n0 = it->n, used0 = it->arena_used;
  int64_t* slot0 = (int64_t*)malloc((size_t)it->cap * sizeof(int64_t));
  memcpy(slot0, it->slot, (size_t)it->cap * sizeof(int64_t));
  int64_t k = 0;
  int rc = 0;
  for (int64_t r = 0; r < n && !rc; ++r) {
    tok_off[r] = k;
    for (int64_t m = req_msg_off[r]; m < req_msg_off[r + 1] && !rc; ++m) {
      int64_t i = msg_off[m], e = msg_off[m + 1];
      while (i < e) {
        while (i < e && sp(text[i])) ++i;
        int64_t s0 = i;
        while (i < e && !sp(text[i])) ++i;
        if (i > s0) {
          int64_t id = intern(it, text + s0, i - s0);
          if (id < 0 || k >= tok_cap) {
            rc = id < 0 ? -5 : -1;
            break;
          }
          tok[k++] = (uint32_t)id;
        }
      }
    }
  }
  tok_off[n] = k;
  *n_tokens = k;
  if (rc) { /* roll back */
    memcpy(it->slot, slot0, (size_t)it->cap * sizeof(int64_t));
    it->n = n0;
    it->arena_used = used0;
  }
  free(slot0);
  return rc;
}


/* ================================================================ latency model ==========
 * SimulatedBackend::start (simulated_backend.cpp:99-112): prefill = overhead + prefill_ms * (P -
 * M), decode = decode_ms * O, ttft = queue + prefill, total = ttft + decode; the completion event
 * fires prefill + decode after dispatch (line 121). Plain C doubles, no contraction (x86-64 -O2). */
int sfo_latency_batch(int64_t n, const int32_t* backend, const double* queue_ms, const int64_t* P,
                      const int64_t* M, const int64_t* O, int32_t n_backends, const double* overhead,
                      const double* prefill, const double* decode, double* out_ttft, double* out_total,
                      double* out_service) {
  if (n < 0 || n_backends <= 0) return -1;
  for (int64_t r = 0; r < n; ++r) {
    const int32_t b = backend[r];
    if (b < 0 || b >= n_backends) return -1;
    const double pf = overhead[b] + prefill[b] * (double)(P[r] - M[r]);
    const double dc = decode[b] * (double)O[r];
    out_ttft[r] = queue_ms[r] + pf;
    if (out_total) out_total[r] = out_ttft[r] + dc;
    if (out_service) out_service[r] = pf + dc;
  }
  return 0;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* percentile_nearest_rank (metrics.cpp:22-28): rank = max(1, ceil(pct / 100.0 * n)). */
int sfo_nearest_rank(int64_t n, const double* samples, int32_t k, const int32_t* pct, double* out) {
  if (n <= 0 || k < 0) return -1;
  double* s = (double*)malloc((size_t)n * sizeof(double));
  memcpy(s, samples, (size_t)n * sizeof(double));
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  for (int32_t i = 0; i < k; ++i) {
    int64_t rank = (int64_t)ceil((double)pct[i] / 100.0 * (double)n);
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    out[i] = s[rank - 1];
  }
  free(s);
  return 0;
}

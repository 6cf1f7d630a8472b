/*
 * sfkv_oracle.h — CPU restatement of the pin-cache / memory-manager / mapper hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the GPU product is compared against; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it. The product
 * (libsfkv.so) never links or calls it.
 *
 * Every sfo_* function restates the semantics of the sfkv_* entry point of the same name
 * (include/sfkv.h) sequentially on host memory. Class A behaviour (pins, M, admission, flush,
 * preserve, utilization, pressure victims, threshold routing) follows the reference line by
 * line (citations in sfkv_oracle.c) and is pinned against the reference itself
 * (tests/golden/ fixtures, produced by oracle/_ref/sf_ref_replay and oracle/_ref/libsfref.so).
 * Class B behaviour (chained hashes, block tables, refcounts, allocation order, KV payload
 * bytes, handoff, N-candidate costs) has no reference counterpart; this file is its definition.
 */
#ifndef SFKV_ORACLE_H_
#define SFKV_ORACLE_H_

#include <stdint.h>

typedef struct sfo_pool sfo_pool;

typedef struct sfo_pool_config {
  int32_t device;
  int32_t max_workflows;
  int64_t n_blocks;
  int64_t capacity_tokens;
  int32_t max_pin_blocks;
  int32_t table_log2;
  int32_t n_slabs;
  int32_t slab_row_bytes;
} sfo_pool_config;

typedef struct sfo_pool_stats {
  int64_t occupancy_tokens;
  int64_t capacity_tokens;
  uint64_t capacity_rejections;
  uint64_t flush_calls;
  uint64_t preserve_calls;
  int64_t blocks_in_use;
  int64_t table_live;
  int64_t table_tombstones;
} sfo_pool_stats;

uint64_t sfo_block_digest(uint64_t k, uint32_t n, const uint32_t* t);
uint64_t sfo_chain_finalize(uint64_t prefix_sum);
/* Chained hashes of all ceil(len/16) blocks of one token sequence. */
void sfo_chain_hashes(const uint32_t* tok, int64_t len, uint64_t* out);

int sfo_pool_create(const sfo_pool_config* cfg, sfo_pool** out);
int sfo_pool_destroy(sfo_pool* p);
int sfo_pool_kv(sfo_pool* p, void** kv, int64_t* block_bytes);

int sfo_match_batch(sfo_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                    const uint32_t* tok, int64_t* out_M, uint64_t* out_hash);
int sfo_lookup_batch(sfo_pool* p, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                     int32_t* out_block, int64_t* out_hit_tokens);
int sfo_commit_batch(sfo_pool* p, int64_t n, const int32_t* wf, const int64_t* tok_off,
                     const uint32_t* tok, const void* kv_src, const int64_t* kv_src_off,
                     const int64_t* m_expected, int32_t* out_status);
int sfo_flush(sfo_pool* p, int32_t wf, int64_t* freed);
int sfo_flush_batch(sfo_pool* p, int64_t n, const int32_t* wf, int64_t* out_freed);
int sfo_preserve(sfo_pool* p, int32_t wf, int32_t* has_pin);
int sfo_pinned_token_count(sfo_pool* p, int32_t wf, int64_t* n_tokens);
int sfo_cache_utilization(sfo_pool* p, double* util);
int sfo_stats(sfo_pool* p, sfo_pool_stats* out);
int sfo_pin_blocks(sfo_pool* p, int32_t wf, int32_t* ids, uint64_t* hashes, int32_t cap,
                   int32_t* n_blocks);
int sfo_block_refcounts(sfo_pool* p, uint32_t* out);
int sfo_pin_tokens(sfo_pool* p, int32_t wf, uint32_t* out, int64_t cap, int64_t* n_tokens);
int sfo_gather(sfo_pool* p, int64_t n, const int32_t* wf, void* dst, const int64_t* dst_off);
int sfo_handoff(sfo_pool* src, int32_t wf_src, sfo_pool* dst, int32_t wf_dst, int32_t* status);

int sfo_pressure_argmin(int64_t n, const int32_t* backend, const double* ts,
                        const uint32_t* wf_rank, const int32_t* in_flight,
                        const uint8_t* preserved, int32_t n_backends, const double* util,
                        double tau, int64_t* out_victim);
int sfo_threshold_batch(int64_t n, const double* score, double threshold, int32_t* out_choice);
int sfo_cost_batch(int64_t n, int32_t c, const int64_t* P, const int64_t* M, const int64_t* O,
                   const double* overhead, const double* prefill, const double* decode,
                   const double* queue_penalty, const int32_t* alternates, uint64_t* depth_inout,
                   uint64_t limit, int32_t* out_choice, double* out_cost);

/* ---- memory manager tracker (restates MemoryManager::on_signal / pressure_tick) ---------- */
typedef struct sfo_tracker sfo_tracker;
typedef struct sfo_mm_config { /* same layout as sfmm_config */
  int32_t device;
  int32_t max_workflows;
  int32_t n_backends;
  int32_t max_stages;
  int32_t chain_len;
  const uint8_t* chain;
  int64_t tau;
  double tau_pressure;
} sfo_mm_config;
typedef struct sfo_signals {
  const uint8_t* kind;
  const int32_t* wf;
  const int32_t* stage;
  const int32_t* backend;
  const int32_t* model;
  const int64_t* tokens;
  const double* ts;
  const uint8_t* override_;
} sfo_signals;
typedef struct sfo_records {
  int32_t* count;
  uint8_t* status;
  uint8_t* kind;
  int32_t* backend;
  uint8_t* reason;
} sfo_records;
int sfo_tracker_create(const sfo_mm_config* cfg, sfo_tracker** out);
int sfo_tracker_destroy(sfo_tracker* t);
int sfo_set_workflow_chain(sfo_tracker* t, int32_t wf, int32_t len, const uint8_t* policies);
int sfo_set_workflow_ranks(sfo_tracker* t, int64_t n, const uint32_t* rank);
int sfo_on_signal_batch(sfo_tracker* t, int64_t n, const sfo_signals* sig, const sfo_records* out);
int sfo_pressure_tick(sfo_tracker* t, const double* util, int32_t* out_victim);
int sfo_tracker_entries(sfo_tracker* t, uint8_t* present, uint8_t* preserved, int64_t* tokens,
                        double* ts, int32_t* in_flight);
int sfo_tracker_reserve(sfo_tracker* t, int32_t max_workflows, int32_t n_backends, int32_t max_stages);
int sfo_tracker_shape(sfo_tracker* t, int32_t* max_workflows, int32_t* n_backends, int32_t* max_stages);
int sfo_reset_workflows(sfo_tracker* t, int64_t n, const int32_t* wf);
int sfo_set_backend_order(sfo_tracker* t, int32_t n, const int32_t* order);
int sfo_flush_failed(sfo_tracker* t, int64_t n, const int32_t* wf, const int32_t* backend,
                     const int64_t* sig);


/* ---- tokenizer + interner (restates tokenize_whitespace / context_token_sequence) -------- */
typedef struct sfo_interner sfo_interner;
int sfo_interner_create(int32_t device, int32_t table_log2, int64_t arena_bytes, sfo_interner** out);
int sfo_interner_destroy(sfo_interner* it);
int sfo_interner_size(sfo_interner* it, int64_t* n_ids);
int sfo_interner_token(sfo_interner* it, uint32_t id, char* out, int32_t cap, int32_t* len);
int sfo_tokenize_batch(sfo_interner* it, int64_t n, const int64_t* req_msg_off, const int64_t* msg_off,
                       const uint8_t* text, int64_t* tok_off, uint32_t* tok, int64_t tok_cap,
                       int64_t* n_tokens);


/* ---- latency model and nearest-rank percentiles (restates simulated_backend.cpp:99-112,
 *      metrics.cpp:22-28) ------------------------------------------------------------------ */
int sfo_latency_batch(int64_t n, const int32_t* backend, const double* queue_ms, const int64_t* P,
                      const int64_t* M, const int64_t* O, int32_t n_backends, const double* overhead,
                      const double* prefill, const double* decode, double* out_ttft, double* out_total,
                      double* out_service);
int sfo_nearest_rank(int64_t n, const double* samples, int32_t k, const int32_t* pct, double* out);

#endif

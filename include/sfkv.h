/*
 * sfkv.h — C ABI of the B200-native KV pin pool, memory-manager pressure step and stage mapper.
 *
 * This is the drop-in boundary for the hot path of the reference ("stageflow", the executable
 * form of Orla, /root/reference/proj). Every entry point names the reference interface it
 * replaces (file:line, paths relative to /root/reference/proj). INTEGRATION.md shows the
 * reference-side binding (a `Backend` subclass and a patched `pressure_actions`).
 *
 * Conventions
 *   - extern "C", opaque handles, plain pointers and sizes; no C++ or torch types.
 *   - Every function returns int: 0 = ok, < 0 = error (SFKV_E*); sfkv_last_error() describes the
 *     most recent error on the calling thread. Nothing throws across the boundary.
 *   - One host thread per pool handle. All GPU work of a pool is issued on the pool's stream
 *     (sfkv_pool_set_stream; default: a private non-blocking stream).
 *   - Functions without the _dev suffix take HOST pointers: they copy inputs to the device,
 *     run the kernels and copy results back before returning (synchronous, like the reference's
 *     single-threaded calls). The _dev variants take DEVICE pointers on the pool's device and
 *     are asynchronous on the pool stream (no host synchronisation): they also take n_tokens,
 *     the number of tokens the tok buffer can hold (>= tok_off[n]), which bounds the work size.
 *     KV staging (kv_src) is always device memory, also in sfkv_commit_batch.
 *     _dev argument checks: the host refuses null and misaligned pointers (tok 16-B aligned, the
 *     kernels load it with 16-B vectors and TMA; tok_off / 64-bit outputs 8-B; wf 4-B) with
 *     SFKV_EINVAL. Values read on the device are guarded there: an out-of-range workflow slot
 *     is matched as unpinned, gathers nothing, refuses its commit batch (status SFKV_EINVAL, no
 *     state change), and a handoff source block outside the peer's region moves nothing; each
 *     sets the pool's sticky error, which the next sfkv_pool_sync (or host-pointer call that
 *     synchronises) reports once as SFKV_EINVAL.
 *   - Token ids exchanged between pools on different ranks must come from one shared vocabulary
 *     (pins are compared as integers); see INTEGRATION.md §4.
 *   - A workflow is a dense slot id in [0, max_workflows) chosen by the host (the host keeps the
 *     workflow_id string -> slot map, as SimulatedBackend keys pins_ by workflow_id,
 *     simulated_backend.hpp:115).
 *   - Token sequences are CSR batches: request r owns tok[tok_off[r] .. tok_off[r+1]).
 *     Tokens are u32 ids of the reference's whitespace tokens (backend.cpp:60-97).
 *   - There is no CPU fallback: every compute entry point runs sm_100a kernels; creating a pool
 *     without a usable B200 fails with SFKV_ENODEV.
 */
#ifndef SFKV_H_
#define SFKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFKV_ABI_VERSION 2

#define SFKV_OK 0
#define SFKV_EINVAL -1    /* bad argument (null pointer, out-of-range slot, unaligned buffer) */
#define SFKV_ENODEV -2    /* no CUDA device / not sm_100 */
#define SFKV_ECUDA -3     /* CUDA runtime error */
#define SFKV_ENOMEM -4    /* device allocation failed */
#define SFKV_EPOOL -5     /* physical pool exhausted (logical capacity admitted the pin, but the
                             physical block pool or a pin's block table is too small) */
#define SFKV_ESTALE -6    /* payload commit whose staging assumed a different cached prefix */
#define SFKV_ECOLLIDE -7  /* two different token strings share a 64-bit hash (interner) */

#define SFKV_FLUSH_ALL (-1)        /* FlushScope::everything() (backend.hpp:65-70) */
#define SFKV_BLOCK_TOKENS 16       /* tokens per KV block */

/* Commit status per request (out_status of sfkv_commit_batch). */
#define SFKV_PIN_REJECTED 0        /* capacity rejection: old pin kept (simulated_backend.cpp:142-148) */
#define SFKV_PIN_ACCEPTED 1

typedef struct sfkv_pool sfkv_pool;

typedef struct sfkv_pool_config {
  int32_t device;            /* CUDA device ordinal of this pool (one backend per GPU) */
  int32_t max_workflows;     /* workflow slots */
  int64_t n_blocks;          /* physical KV blocks (16 tokens each) */
  int64_t capacity_tokens;   /* logical capacity: SimulatedBackendConfig::cache_capacity_tokens
                                (simulated_backend.hpp:62); admission is on logical tokens */
  int32_t max_pin_blocks;    /* block-table length per workflow pin */
  int32_t table_log2;        /* global block table: 2^table_log2 slots of 16 B */
  int32_t n_slabs;           /* KV slabs per token = layers * 2 (K and V); 0 = metadata only */
  int32_t slab_row_bytes;    /* bytes of one token in one slab = kv_heads * head_dim * 2 (bf16) */
} sfkv_pool_config;

/* Counters mirrored from SimulatedBackend / BackendStats (backend.hpp:72-80,
 * simulated_backend.hpp:96-98). */
typedef struct sfkv_pool_stats {
  int64_t occupancy_tokens;       /* sum of pin lengths */
  int64_t capacity_tokens;
  uint64_t capacity_rejections;
  uint64_t flush_calls;
  uint64_t preserve_calls;
  int64_t blocks_in_use;          /* physical blocks with refcount > 0 */
  int64_t table_live;             /* live keys in the global table */
  int64_t table_tombstones;
} sfkv_pool_stats;

/* ---- lifecycle ------------------------------------------------------------------------- */

const char* sfkv_last_error(void);
int sfkv_abi_version(void);

/* Replaces the SimulatedBackend constructor's cache state (simulated_backend.cpp:20-29). */
int sfkv_pool_create(const sfkv_pool_config* cfg, sfkv_pool** out);
int sfkv_pool_destroy(sfkv_pool* pool);
/* Grows the pool in place (never shrinks): workflow slots, the per-pin block-table length and
 * the physical block count (the dedup table is re-indexed at load factor <= 1/2 when it grows).
 * Pins, blocks, refcounts and KV bytes are preserved. The reference's pin cache is unbounded
 * (std::map pins_, simulated_backend.hpp:115), so a binding starts small and reserves on demand
 * (prompts longer than max_pin_blocks * 16 tokens, more live workflows than slots). Synchronises
 * the pool stream. The KV region cannot move once exported (sfkv_pool_export): SFKV_EINVAL. */
int sfkv_pool_reserve(sfkv_pool* pool, int32_t max_workflows, int32_t max_pin_blocks, int64_t n_blocks);
/* The pool's current configuration (after any reserve). */
int sfkv_pool_config_get(sfkv_pool* pool, sfkv_pool_config* out);
int sfkv_pool_set_stream(sfkv_pool* pool, void* cuda_stream);
int sfkv_pool_sync(sfkv_pool* pool);
/* Device pointer of the KV payload (n_blocks * block_bytes), block-major
 * [block][slab][slot 16][slab_row_bytes]; block_bytes = n_slabs * 16 * slab_row_bytes. */
int sfkv_pool_kv(sfkv_pool* pool, void** kv, int64_t* block_bytes);

/* ---- lookup: replaces SimulatedBackend::prefix_match (simulated_backend.cpp:153-162) -------
 * out_M[r] = LCP(pin[wf[r]], tokens of r), 0 when the workflow has no pin. Exact: the kernel
 * hashes the request's 16-token blocks into chained block hashes and compares them with the
 * pin's; every block whose predecessor hash matches is verified token by token, so M never
 * depends on hash collisions. out_hash (nullable) receives the chained hash of every block of
 * every request (ceil(len/16) per request, concatenated in request order). */
int sfkv_match_batch(sfkv_pool* pool, int64_t n, const int32_t* wf, const int64_t* tok_off,
                     const uint32_t* tok, int64_t* out_M, uint64_t* out_hash);
int sfkv_match_batch_dev(sfkv_pool* pool, int64_t n, const int32_t* wf, const int64_t* tok_off,
                         const uint32_t* tok, int64_t n_tokens, int64_t* out_M, uint64_t* out_hash);

/* ---- global lookup (new; cross-workflow dedup the reference lacks) -------------
 * For every block of every request (ceil(len/16) entries per request, request order): the id of
 * the resident block with the same chained hash (token-verified), else -1; partial (last) blocks
 * are never shared and always report -1. out_hit_tokens[r] = 16 * number of leading hit blocks. */
int sfkv_lookup_batch(sfkv_pool* pool, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                      int32_t* out_block, int64_t* out_hit_tokens);
int sfkv_lookup_batch_dev(sfkv_pool* pool, int64_t n, const int64_t* tok_off, const uint32_t* tok,
                          int64_t n_tokens, int32_t* out_block, int64_t* out_hit_tokens);

/* ---- retain: replaces SimulatedBackend::pin_prompt (simulated_backend.cpp:135-151) ----------
 * Commits request r's tokens as the new pin of wf[r] (workflow slots distinct within a batch).
 * Admission runs in request order with the reference rule: reject iff
 * occupancy - old_len + new_len > capacity (old pin kept, ++capacity_rejections).
 * Accepted pins share every leading full block already resident (any workflow, chained-hash +
 * token verified) and allocate the rest (lowest free block ids, in request/block order; within
 * the batch the lowest request index owns a new shared block). Old-pin blocks are released after
 * the new pin's references are taken.
 * KV payload (pools with n_slabs > 0; kv_src may be NULL for metadata-only commits): token p of a
 * newly allocated block is copied from the old pin's block when p < M_r (copy-on-share of the
 * boundary block) and otherwise from staging row p - M_r, where M_r = LCP(old pin, tokens) and
 * the staging of request r starts at byte kv_src_off[r] of kv_src with layout
 * [slab][token (P_r - M_r rows)][slab_row_bytes]. m_expected (nullable) is the M the caller's
 * prefill assumed; a request whose M_r differs fails the batch with SFKV_ESTALE. */
int sfkv_commit_batch(sfkv_pool* pool, int64_t n, const int32_t* wf, const int64_t* tok_off,
                      const uint32_t* tok, const void* kv_src, const int64_t* kv_src_off,
                      const int64_t* m_expected, int32_t* out_status);
int sfkv_commit_batch_dev(sfkv_pool* pool, int64_t n, const int32_t* wf, const int64_t* tok_off,
                          const uint32_t* tok, int64_t n_tokens, const void* kv_src,
                          const int64_t* kv_src_off, const int64_t* m_expected,
                          int32_t* out_status);

/* ---- evict: replaces SimulatedBackend::flush (simulated_backend.cpp:169-184) -----------------
 * wf = SFKV_FLUSH_ALL flushes every pin. *freed = tokens released (0 when nothing was pinned). */
int sfkv_flush(sfkv_pool* pool, int32_t wf, int64_t* freed);
/* Batched evict of distinct workflows; out_freed[r] per request. */
int sfkv_flush_batch(sfkv_pool* pool, int64_t n, const int32_t* wf, int64_t* out_freed);

/* ---- inspection: SimulatedBackend::preserve / pinned_token_count / cache_utilization ---------
 * (simulated_backend.cpp:164-167, 186-193). preserve counts a preserve call and reports whether a
 * pin exists (an empty pin counts). */
int sfkv_preserve(sfkv_pool* pool, int32_t wf, int32_t* has_pin);
int sfkv_pinned_token_count(sfkv_pool* pool, int32_t wf, int64_t* n_tokens);
int sfkv_cache_utilization(sfkv_pool* pool, double* util);
int sfkv_stats(sfkv_pool* pool, sfkv_pool_stats* out);
/* Block table of a pin (Class B inspection): ids (cap entries max), chained hashes (nullable). */
int sfkv_pin_blocks(sfkv_pool* pool, int32_t wf, int32_t* ids, uint64_t* hashes, int32_t cap,
                    int32_t* n_blocks);
/* Refcount of every physical block (n_blocks entries). */
int sfkv_block_refcounts(sfkv_pool* pool, uint32_t* out);
/* Token ids of a pin (cap entries max; *n_tokens = pin length, 0 without a pin). Used to ship a
 * pin to another process (cross-rank handoff). */
int sfkv_pin_tokens(sfkv_pool* pool, int32_t wf, uint32_t* out, int64_t cap, int64_t* n_tokens);

/* ---- gather (new): assemble pins into contiguous staging ------------------------------------
 * Request r writes its pin's KV at dst + dst_off[r], layout [slab][token (pin_len)][row]. */
int sfkv_gather_dev(sfkv_pool* pool, int64_t n, const int32_t* wf, void* dst,
                    const int64_t* dst_off);

/* ---- cross-pool stage handoff (new; migration is a SPEC non-goal) --------------
 * Copies the pin of wf_src in `src` into `dst` as the pin of wf_dst (same semantics as a commit
 * into dst whose payload comes from the source pin's blocks). The pools may live on different
 * GPUs (peer access over NVLink; the copy kernel runs on dst's device and pulls) or on the same
 * GPU. *status = SFKV_PIN_ACCEPTED / SFKV_PIN_REJECTED (dst capacity), unchanged dst on reject. */
int sfkv_handoff(sfkv_pool* src, int32_t wf_src, sfkv_pool* dst, int32_t wf_dst, int32_t* status);

/* ---- cross-process stage handoff over NVLink (one process per GPU; new) ---------
 * The sending rank exports its pool's KV region once (CUDA IPC); every receiving rank maps it
 * (sfkv_peer_open), so the receiver's commit kernel pulls the source blocks' rows directly over
 * NVLink (or from the same device) with no staging copy. The sender ships only metadata per
 * workflow: its pin's tokens and block ids (sfkv_pin_export); the sender must keep those blocks
 * resident until the receiver's handoff call has completed.
 * sfkv_handoff_recv_batch commits request r's tokens as the pin of wf[r] in `dst` exactly like
 * sfkv_commit_batch (admission, dedup, copy-on-share against dst's old pin), with the payload of
 * new blocks read from the source blocks src_blocks[blk_off[r] + k] (ceil(len_r/16) ids per
 * request, concatenated in request order) of the mapped region. */
typedef struct sfkv_ipc_handle {
  char handle[64];           /* cudaIpcMemHandle_t of the pool's KV region */
  int64_t kv_bytes;
  int64_t block_bytes;
  int32_t n_slabs;
  int32_t slab_row_bytes;
} sfkv_ipc_handle;
typedef struct sfkv_peer sfkv_peer;

int sfkv_pool_export(sfkv_pool* pool, sfkv_ipc_handle* out);
int sfkv_peer_open(const sfkv_ipc_handle* handle, int32_t device, sfkv_peer** out);
int sfkv_peer_close(sfkv_peer* peer);
/* Tokens (cap entries max) and block ids (ceil(L/16) entries; written when cap >= L) of a pin. */
int sfkv_pin_export(sfkv_pool* pool, int32_t wf, uint32_t* tok, int32_t* block_ids, int64_t cap,
                    int64_t* n_tokens);
int sfkv_handoff_recv_batch(sfkv_pool* dst, const sfkv_peer* src, int64_t n, const int32_t* wf,
                            const int64_t* tok_off, const uint32_t* tok, const int32_t* src_blocks,
                            int32_t* out_status);
int sfkv_handoff_recv_batch_dev(sfkv_pool* dst, const sfkv_peer* src, int64_t n, const int32_t* wf,
                                const int64_t* tok_off, const uint32_t* tok, int64_t n_tokens,
                                const int32_t* src_blocks, int32_t* out_status);

/* ---- tokenizer + interner: replaces tokenize_whitespace /
 *      context_token_sequence (backend.cpp:60-91) on the dispatch path ------------------------
 * Tokens are maximal runs of non-space bytes (std::isspace, C locale); each message is split
 * separately and the request's tokens are the concatenation (roles ignored). Every token string
 * is interned into a u32 id: equal strings get equal ids for the interner's lifetime; strings new
 * to the interner are numbered in order of first occurrence in the batch (deterministic). Text is
 * a CSR of messages (msg_off over text bytes) and requests are ranges of messages (req_msg_off).
 * Output: the token CSR the match / commit entry points take (tok_off[n+1], tok). tok must hold
 * (n_bytes + n_msg + 1) / 2 ids (a message of L bytes splits into at most (L + 1) / 2 tokens). A batch that would overflow the interner or that meets a 64-bit hash
 * collision between different strings fails without changing the interner (SFKV_EPOOL /
 * SFKV_ECOLLIDE). */
typedef struct sfkv_interner sfkv_interner;
int sfkv_interner_create(int32_t device, int32_t table_log2, int64_t arena_bytes, sfkv_interner** out);
int sfkv_interner_destroy(sfkv_interner* it);
/* Grows the interner in place (never shrinks): a 2^table_log2-slot table (at most 2^(table_log2-1)
 * ids) and arena_bytes of token text. Every existing string keeps its id. A batch that failed with
 * SFKV_EPOOL (table, id space or arena full) changed nothing and can be retried after a reserve.
 * (The reference's token strings live in unbounded std::strings, backend.cpp:60-91.) */
int sfkv_interner_reserve(sfkv_interner* it, int32_t table_log2, int64_t arena_bytes);
/* Arena bytes used / capacity and the current table size (log2). */
int sfkv_interner_arena(sfkv_interner* it, int64_t* used, int64_t* cap, int32_t* table_log2);
/* Forgets every string (empty table, id 0 next, arena cursor 0) and keeps the allocations and the
 * per-batch scratch: a new vocabulary without re-creating the interner. Asynchronous on the
 * interner's stream. */
int sfkv_interner_reset(sfkv_interner* it);
int sfkv_interner_set_stream(sfkv_interner* it, void* cuda_stream);  /* NULL = legacy default stream */
int sfkv_interner_size(sfkv_interner* it, int64_t* n_ids);
int sfkv_interner_token(sfkv_interner* it, uint32_t id, char* out, int32_t cap, int32_t* len);
int sfkv_tokenize_batch(sfkv_interner* it, int64_t n, const int64_t* req_msg_off, const int64_t* msg_off,
                        const uint8_t* text, int64_t* tok_off, uint32_t* tok, int64_t tok_cap,
                        int64_t* n_tokens);
/* Device pointers, asynchronous on the interner's stream; *n_tokens is a device scalar.
 * sfkv_interner_check reports (and clears) a failed device batch. */
int sfkv_tokenize_batch_dev(sfkv_interner* it, int64_t n, const int64_t* req_msg_off, int64_t n_msg,
                            const int64_t* msg_off, const uint8_t* text, int64_t n_bytes, int64_t* tok_off,
                            uint32_t* tok, int64_t* n_tokens);
int sfkv_interner_check(sfkv_interner* it);

/* ---- memory manager: replaces pressure_actions (memory.cpp:150-169) -------------------------
 * Entries are the tracker's (workflow, backend) records as SoA: backend index, last_update_ts,
 * wf_rank (rank of workflow_id in std::string order), in_flight, preserved. For every backend b
 * with util[b] > tau: out_victim[b] = index of the preserved entry with in_flight == 0 and the
 * least (last_update_ts, wf_rank), else -1. Runs on `device`. */
int sfmm_pressure_argmin(int32_t device, int64_t n, const int32_t* backend, const double* ts,
                         const uint32_t* wf_rank, const int32_t* in_flight,
                         const uint8_t* preserved, int32_t n_backends, const double* util,
                         double tau, int64_t* out_victim);
/* Device pointers, asynchronous on cuda_stream (NULL = legacy default stream). One launch. */
int sfmm_pressure_argmin_dev(int32_t device, int64_t n, const int32_t* backend, const double* ts,
                             const uint32_t* wf_rank, const int32_t* in_flight,
                             const uint8_t* preserved, int32_t n_backends, const double* util,
                             double tau, int64_t* out_victim, void* cuda_stream);

/* ---- memory manager: batched MemoryManager::on_signal and pressure_tick on a GPU-resident
 *      WorkflowTracker (memory.cpp:256-387) ------------------------------------
 * The tracker (memory.hpp:49-72: cache entries, in-flight counts, last stage, completion, plus
 * the manager's started/open stage sets and per-workflow chains) lives in HBM as dense arrays
 * over (workflow slot, backend index). Workflow ids, stage ids, backend refs and models are
 * interned by the host: stage ids are dense per workflow, models are dense ids, backends are
 * dense ids in any order (sfmm_set_backend_order gives their std::string order, the order
 * flush_at_boundary flushes a finished workflow's entries in, memory.cpp:137-141). Nothing is
 * capped: sfmm_tracker_reserve grows slots, backends and stage ids in place (the reference's
 * std::maps are unbounded), and policy chains have any length.
 * sfmm_on_signal_batch applies a batch of lifecycle signals exactly as n sequential on_signal
 * calls would: policies read only their own workflow's state, so the batch is processed in
 * parallel across workflows and in order within each. Signal i's log records (on_signal logs
 * every returned action, noops included, memory.cpp:312-328) are written at
 * [i * n_backends, i * n_backends + count[i]); the action log of the batch is the concatenation
 * in signal order. Flushes are recorded as applied (the tracker erases the entry,
 * memory.cpp:319-321); the host then applies every record to its backends (apply_action,
 * memory.cpp:185-220: a flush is retried once) and reports each flush that failed twice with
 * sfmm_flush_failed before the next batch or tick: the entry becomes present but unpreserved
 * (mark_unpreserved, memory.cpp:322-324) unless a later signal of the same batch re-wrote or
 * erased it (exactly the reference's end state; no policy reads an unpreserved entry, so no other
 * decision of the batch depends on the outcome). A signal that the reference would reject
 * (OutOfOrderSignalError, memory.cpp:256-285) gets status SFMM_SIG_OUT_OF_ORDER and produces no
 * records; the rest of that workflow's signals in the batch are SFMM_SIG_SKIPPED.
 * sfmm_pressure_tick replaces MemoryManager::pressure_tick (memory.cpp:372-387): per backend with
 * util > tau_pressure, the idle preserved entry with least (last_update_ts, workflow rank) is
 * flushed (recorded with reason flush_under_pressure) and erased from the tracker (one kernel:
 * a segmented warp-shuffle argmin); a victim whose flush failed twice is reported with
 * sfmm_flush_failed (sig = -1). */
/* LifecycleSignal::Kind (signals.hpp:13-15) */
#define SFMM_STAGE_START 0
#define SFMM_STAGE_COMPLETE 1
#define SFMM_WORKFLOW_COMPLETE 2
/* CachePolicyOverride (workflow.hpp:16) */
#define SFMM_OVERRIDE_NONE 0
#define SFMM_OVERRIDE_PRESERVE 1
#define SFMM_OVERRIDE_FLUSH 2
/* memory_policy_by_name (memory.cpp:171-183) */
#define SFMM_POLICY_PRESERVE_SMALL_INCREMENT 1
#define SFMM_POLICY_FLUSH_AT_BOUNDARY 2
/* CacheAction::Kind (memory.hpp:20) */
#define SFMM_ACT_PRESERVE 0
#define SFMM_ACT_FLUSH 1
#define SFMM_ACT_NOOP 2
/* CacheAction::reason values the built-in code produces */
#define SFMM_REASON_OVERRIDE 0
#define SFMM_REASON_PRESERVE_SMALL_INCREMENT 1
#define SFMM_REASON_FLUSH_AT_BOUNDARY 2
#define SFMM_REASON_FLUSH_UNDER_PRESSURE 3
#define SFMM_REASON_CHAIN_EXHAUSTED 4
/* per-signal status */
#define SFMM_SIG_OK 0
#define SFMM_SIG_OUT_OF_ORDER 1     /* OutOfOrderSignalError */
#define SFMM_SIG_SKIPPED 2          /* an earlier signal of the workflow in this batch failed */
#define SFMM_SIG_NEGATIVE_IN_FLIGHT 3 /* logic_error("in-flight count went negative") */

typedef struct sfmm_tracker sfmm_tracker;

typedef struct sfmm_config {
  int32_t device;
  int32_t max_workflows;             /* initial workflow slots */
  int32_t n_backends;                /* initial backends */
  int32_t max_stages;                /* initial stage ids per workflow (0 = 64) */
  int32_t chain_len;                 /* default policy chain (MemoryConfig::policy_chain), */
  const uint8_t* chain;              /*   any length, SFMM_POLICY_* codes; copied */
  int64_t tau;                       /* MemoryConfig::tau (memory.hpp:74-79) */
  double tau_pressure;               /* MemoryConfig::tau_pressure */
} sfmm_config;

typedef struct sfmm_signals {        /* n signals, struct of arrays */
  const uint8_t* kind;
  const int32_t* wf;
  const int32_t* stage;              /* dense per workflow; ignored for WorkflowComplete */
  const int32_t* backend;            /* ignored for WorkflowComplete */
  const int32_t* model;
  const int64_t* tokens;             /* context_tokens */
  const double* ts;
  const uint8_t* override_;          /* cache_override */
} sfmm_signals;

typedef struct sfmm_records {        /* outputs: n signals x n_backends record slots */
  int32_t* count;                    /* [n] records of signal i */
  uint8_t* status;                   /* [n] SFMM_SIG_* */
  uint8_t* kind;                     /* [n * n_backends] SFMM_ACT_* */
  int32_t* backend;                  /* [n * n_backends] -1 for noops */
  uint8_t* reason;                   /* [n * n_backends] SFMM_REASON_* */
} sfmm_records;

int sfmm_tracker_create(const sfmm_config* cfg, sfmm_tracker** out);
int sfmm_tracker_destroy(sfmm_tracker* t);
/* Grows slots / backends / stage ids in place (never shrinks); state is preserved. */
int sfmm_tracker_reserve(sfmm_tracker* t, int32_t max_workflows, int32_t n_backends, int32_t max_stages);
int sfmm_tracker_shape(sfmm_tracker* t, int32_t* max_workflows, int32_t* n_backends, int32_t* max_stages);
int sfmm_tracker_set_stream(sfmm_tracker* t, void* cuda_stream);  /* NULL = legacy default stream */
int sfmm_tracker_sync(sfmm_tracker* t);
/* Forget every workflow (a fresh MemoryManager with the same configuration). */
int sfmm_tracker_reset(sfmm_tracker* t);
/* Forget the listed workflow slots (a host recycling slots of finished workflows). */
int sfmm_reset_workflows(sfmm_tracker* t, int64_t n, const int32_t* wf);
/* MemoryManager::set_workflow_chain (memory.cpp:246-250); len 0 = no-op, as the reference. */
int sfmm_set_workflow_chain(sfmm_tracker* t, int32_t wf, int32_t len, const uint8_t* policies);
/* Rank of every workflow slot in workflow-id string order (pressure tie-break). */
int sfmm_set_workflow_ranks(sfmm_tracker* t, int64_t n, const uint32_t* rank);
/* order[k] = backend index of the k-th backend ref in std::string order (n = n_backends);
 * default: identity. */
int sfmm_set_backend_order(sfmm_tracker* t, int32_t n, const int32_t* order);
int sfmm_on_signal_batch(sfmm_tracker* t, int64_t n, const sfmm_signals* sig, const sfmm_records* out);
int sfmm_on_signal_batch_dev(sfmm_tracker* t, int64_t n, const sfmm_signals* sig,
                             const sfmm_records* out);
/* Flush records the host could not apply (apply_action failed twice): (workflow slot, backend,
 * signal index in the last sfmm_on_signal_batch, or -1 for the last sfmm_pressure_tick). */
int sfmm_flush_failed(sfmm_tracker* t, int64_t n, const int32_t* wf, const int32_t* backend,
                      const int64_t* sig);
/* util[n_backends] -> out_victim[n_backends] workflow slot or -1. */
int sfmm_pressure_tick(sfmm_tracker* t, const double* util, int32_t* out_victim);
/* Device pointers, asynchronous on the tracker's stream (no host synchronisation). */
int sfmm_pressure_tick_dev(sfmm_tracker* t, const double* util, int32_t* out_victim);
/* Tracker snapshot (inspection / parity): per (wf, backend) entry and in-flight count. */
int sfmm_tracker_entries(sfmm_tracker* t, uint8_t* present, uint8_t* preserved, int64_t* tokens,
                         double* ts, int32_t* in_flight);

/* ---- batched latency model and TTFT percentiles: SimulatedBackend::start's
 *      timing arithmetic (simulated_backend.cpp:99-112) and MetricsReport's nearest-rank
 *      percentiles (metrics.cpp:22-28, 57-67) ---------------------------------------------------
 * Per request r on backend b = backend[r]:
 *   prefill = overhead[b] + prefill[b] * (P[r] - M[r]);  decode = decode[b] * O[r]
 *   ttft = queue_ms[r] + prefill;  total = ttft + decode;  service = prefill + decode
 *   (the completion event's delay) — bit-identical doubles (no FMA contraction).
 * out_total / out_service nullable. The _dev variant takes device pointers and a stream. */
int sfmet_latency_batch(int32_t device, int64_t n, const int32_t* backend, const double* queue_ms, const int64_t* P,
                        const int64_t* M, const int64_t* O, int32_t n_backends, const double* overhead,
                        const double* prefill, const double* decode, double* out_ttft, double* out_total,
                        double* out_service);
int sfmet_latency_batch_dev(int32_t device, int64_t n, const int32_t* backend, const double* queue_ms,
                            const int64_t* P, const int64_t* M, const int64_t* O, const double* overhead,
                            const double* prefill, const double* decode, double* out_ttft, double* out_total,
                            double* out_service, void* cuda_stream);
/* out[i] = the pct[i]-th nearest-rank percentile of the n samples (n >= 1; sorted on the device):
 * sorted[max(1, ceil(pct[i] / 100 * n)) - 1]. MetricsReport::ttft_cdf is pct = 1..99. */
int sfmet_nearest_rank(int32_t device, int64_t n, const double* samples, int32_t k, const int32_t* pct, double* out);

/* ---- stage mapper: replaces map_threshold (mapper.cpp:19-31) and reroute_on_overload
 *      (orchestrator.cpp:78-87) -----------------------------------------------------------------
 * Threshold: out_choice[r] = 0 (light) iff score[r] <= threshold, else 1 (heavy).
 * Cost: for R requests x C candidates,
 *   cost[r][c] = overhead[c] + prefill[c] * (P[r] - M[r*C + c]) + decode[c] * O[r]
 *                + queue_penalty[c] * depth[c]
 * out_choice[r] = argmin_c cost (ties -> lowest c), out_cost[r] = that cost (f64).
 * Costs use the batch-start depth snapshot. Reroute (limit > 0): requests are then processed in
 * order; the choice stays if its live queue depth < limit, else the first listed alternate
 * (alternates[choice*C + j], j = 0.., -1 terminated; nullable = none) with depth < limit, else
 * unchanged; each routed request increments its candidate's live depth (the batched equivalent of
 * Orchestrator::queue_depth growing as requests enqueue, orchestrator.cpp:245-251, 481-484).
 * depth_inout (C entries, u64) is updated. */
int sfmap_threshold_batch(int32_t device, int64_t n, const double* score, double threshold,
                          int32_t* out_choice);
int sfmap_cost_batch(int32_t device, int64_t n, int32_t c, const int64_t* P, const int64_t* M,
                     const int64_t* O, const double* overhead, const double* prefill,
                     const double* decode, const double* queue_penalty,
                     const int32_t* alternates, uint64_t* depth_inout, uint64_t limit,
                     int32_t* out_choice, double* out_cost);
/* Device pointers (depth_inout too), asynchronous on cuda_stream (NULL = legacy default stream). */
int sfmap_cost_batch_dev(int32_t device, int64_t n, int32_t c, const int64_t* P, const int64_t* M,
                         const int64_t* O, const double* overhead, const double* prefill,
                         const double* decode, const double* queue_penalty,
                         const int32_t* alternates, uint64_t* depth_inout, uint64_t limit,
                         int32_t* out_choice, double* out_cost, void* cuda_stream);

/* ---- the chained block hash (shared by the GPU kernels and the CPU oracle) -------------------
 * digest(k, n, t) of block k with n valid tokens t[0..n) (t[j] = 0 for j >= n):
 *   K_s[j]  = bits [32s, 32s+32) of mix64(16 s + j + 1)            (s = 0, 1; j < 16)
 *   acc_s   = sum_{i<8} (t[2i] + K_s[2i]) * (t[2i+1] + K_s[2i+1])  (u32 adds, u64 products/sum)
 *   digest  = mix64(acc_0 ^ rotl64(acc_1, 32) ^ (k * 0xD6E8FEB86659FD93 + n))
 * mix64 = splitmix64's finaliser. chain(k) = fin(sum_{i<=k} digest(i) mod 2^62),
 * fin(s) = mix64(s ^ 0x5851F42D4C957F2D), raised to >= 2 (keys 0/1 are reserved).
 * Exposed for tests and for hosts that precompute keys. */
uint64_t sfkv_block_digest(uint64_t k, uint32_t n, const uint32_t* t);
uint64_t sfkv_chain_finalize(uint64_t prefix_sum);

#ifdef __cplusplus
}
#endif

#endif /* SFKV_H_ */

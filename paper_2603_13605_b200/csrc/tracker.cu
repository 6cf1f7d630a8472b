// §8f-1: batched MemoryManager::on_signal and pressure_tick over a GPU-resident WorkflowTracker.
//
// Replaces MemoryManager::{check_order, resolve, apply_and_record, update_tracker, on_signal,
// pressure_tick} (memory.cpp:256-387), the built-in policies (memory.cpp:116-148) and
// pressure_actions (memory.cpp:150-169). The reference processes one signal at a time through
// string-keyed std::maps (~5.9 us per signal). Here the tracker is a set of dense
// arrays in HBM over (workflow slot, backend index):
//   per workflow  completed u8, started/open stage bitsets (started_ever_ / open_stages_) of SW
//                 u64 words (any number of stages: the tracker grows, sfmm_tracker_reserve),
//                 open-stage count, last stage {valid, backend, model, tokens}, chain (offset +
//                 length into a deduplicated policy-chain arena; -1 = the default chain, any
//                 length), rank in workflow-id order (pressure tie-break)
//   per (wf, b)   entry {present, preserved, tokens, last_update_ts}, in-flight count, and the
//                 tag of the last operation that modified it (flush-failure feedback below)
// A policy reads only its own workflow's state, so a batch of signals is data-parallel across
// workflows and sequential within one:
//   sig_count_kernel    slot of each signal inside its workflow's segment (atomicAdd; the order
//                       is restored below, so results never depend on atomic order)
//   exclusive scan      segment offsets over workflow slots
//   sig_scatter_kernel  signal indices into their workflow's segment
//   sig_resolve_kernel  one thread per workflow with signals: sort its segment by signal index,
//                       then check_order -> resolve (override, chain) -> apply (flush erases the
//                       entry) -> update_tracker for each signal in order; records go to the
//                       signal's own slots, so the batch's action log is in signal order.
// Flushes are recorded as applied. The host applies them to the backends (apply_action,
// memory.cpp:185-220, retry once); a flush that failed twice is reported back with
// sfmm_flush_failed and the entry becomes present-but-unpreserved (mark_unpreserved,
// memory.cpp:319-325) unless a later signal of the same batch re-wrote or erased it. No policy
// reads an unpreserved entry, so the batch's other decisions cannot depend on the outcome.
// pressure_tick: ONE kernel — per backend, a segmented warp-shuffle argmin over (ts, rank, slot)
// per CTA, the last CTA to finish reduces the CTA partials and erases the victims.
#include <algorithm>
#include <map>
#include <utility>
#include <vector>

#include "argmin.cuh"
#include "pool.cuh"

struct sfmm_tracker {
  int32_t device = 0;
  int64_t tau = 0;
  double tau_p = 0;
  int32_t W = 0, NB = 0, SW = 1;  // workflow slots, backends, u64 words per stage bitset
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint32_t epoch = 0;  // operation counter: on_signal batches and pressure ticks
  // policy chains: host-deduplicated arena (the default chain first), mirrored on the device
  std::vector<uint8_t> arena_host;
  std::map<std::vector<uint8_t>, int32_t> chain_at;
  uint8_t* arena = nullptr;
  size_t arena_cap = 0;
  int32_t def_off = 0, def_len = 0;
  // per workflow
  uint8_t* completed = nullptr;
  unsigned long long* started = nullptr;  // [W][SW]
  unsigned long long* open_ = nullptr;    // [W][SW]
  int32_t* open_cnt = nullptr;
  uint8_t* last_valid = nullptr;
  int32_t* last_b = nullptr;
  int32_t* last_model = nullptr;
  int64_t* last_tokens = nullptr;
  int32_t* chain_off = nullptr;  // -1 = default chain
  int32_t* chain_len = nullptr;
  uint32_t* rank = nullptr;
  int32_t* cnt = nullptr;  // per-workflow signal count of the current batch (kept zero between)
  // per (wf, b) entry
  uint8_t* present = nullptr;
  uint8_t* preserved = nullptr;
  int64_t* tokens = nullptr;
  double* ts = nullptr;
  int32_t* inflight = nullptr;
  unsigned long long* mod = nullptr;
  // backends in std::string order (preserved_entries / refs() order): border[k] = index
  int32_t* border = nullptr;
  // pressure tick
  int32_t* victim = nullptr;
  double* util = nullptr;
  unsigned int* done = nullptr;
  sfkv::Scratch part;  // per-CTA candidates of a tick
  sfkv::Scratch scratch;
  sfkv::Scratch io;
};

namespace sfkv {

enum : uint8_t { K_START = 0, K_COMPLETE = 1, K_WF_COMPLETE = 2 };
enum : uint8_t { O_NONE = 0, O_PRESERVE = 1, O_FLUSH = 2 };
enum : uint8_t { P_PSI = 1, P_FAB = 2 };
enum : uint8_t { A_PRESERVE = 0, A_FLUSH = 1, A_NOOP = 2 };
enum : uint8_t { R_OVERRIDE = 0, R_PSI = 1, R_FAB = 2, R_PRESSURE = 3, R_EXHAUSTED = 4 };

// Tag of the operation that last modified an entry: (epoch, signal index, kind); kind 0 = erased
// by a recorded flush (the one sfmm_flush_failed may undo), 1 = re-written / erased otherwise.
__host__ __device__ __forceinline__ unsigned long long mod_tag(uint32_t epoch, int64_t sig, int kind) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)(sig & 0x7fffffff) << 1) | (unsigned)kind;
}

struct SigArgs {
  int64_t n;
  sfmm_signals s;
  sfmm_records r;
  int32_t* slot;
  int64_t* seg_off;
  int32_t* seg;
};

struct TrackerView {  // device pointers of a tracker, by value into kernels
  int32_t W, NB, SW;
  int32_t def_off, def_len;
  uint32_t epoch;
  int64_t tau;
  double tau_p;
  const uint8_t* arena;
  uint8_t* completed;
  unsigned long long* started;
  unsigned long long* open_;
  int32_t* open_cnt;
  uint8_t* last_valid;
  int32_t* last_b;
  int32_t* last_model;
  int64_t* last_tokens;
  int32_t* chain_off;
  int32_t* chain_len;
  uint32_t* rank;
  int32_t* cnt;
  uint8_t* present;
  uint8_t* preserved;
  int64_t* tokens;
  double* ts;
  int32_t* inflight;
  unsigned long long* mod;
  const int32_t* border;
  int32_t* victim;
  const double* util;
  unsigned int* done;
  Cand* part;
};

static TrackerView view(sfmm_tracker* t) {
  TrackerView v;
  v.W = t->W;
  v.NB = t->NB;
  v.SW = t->SW;
  v.def_off = t->def_off;
  v.def_len = t->def_len;
  v.epoch = t->epoch;
  v.tau = t->tau;
  v.tau_p = t->tau_p;
  v.arena = t->arena;
  v.completed = t->completed;
  v.started = t->started;
  v.open_ = t->open_;
  v.open_cnt = t->open_cnt;
  v.last_valid = t->last_valid;
  v.last_b = t->last_b;
  v.last_model = t->last_model;
  v.last_tokens = t->last_tokens;
  v.chain_off = t->chain_off;
  v.chain_len = t->chain_len;
  v.rank = t->rank;
  v.cnt = t->cnt;
  v.present = t->present;
  v.preserved = t->preserved;
  v.tokens = t->tokens;
  v.ts = t->ts;
  v.inflight = t->inflight;
  v.mod = t->mod;
  v.border = t->border;
  v.victim = t->victim;
  v.util = t->util;
  v.done = t->done;
  v.part = t->part.as<Cand>();
  return v;
}

// Forget workflows: all of them (list == nullptr, n = W) or the listed slots (slot reuse).
__global__ void tracker_init_kernel(TrackerView v, int64_t n, const int32_t* list) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = list ? list[i] : i;
    v.completed[w] = 0;
    for (int32_t q = 0; q < v.SW; ++q) v.started[w * v.SW + q] = v.open_[w * v.SW + q] = 0;
    v.open_cnt[w] = 0;
    v.last_valid[w] = 0;
    v.last_b[w] = -1;
    v.last_model[w] = -1;
    v.last_tokens[w] = 0;
    v.chain_off[w] = -1;
    v.chain_len[w] = 0;
    if (!list) {
      v.rank[w] = (uint32_t)w;
      v.cnt[w] = 0;
    }
    for (int32_t b = 0; b < v.NB; ++b) {
      const int64_t e = w * v.NB + b;
      v.present[e] = 0;
      v.preserved[e] = 0;
      v.tokens[e] = 0;
      v.ts[e] = 0;
      v.inflight[e] = 0;
      v.mod[e] = 0;
    }
  }
}

__global__ void sig_count_kernel(SigArgs a, TrackerView v) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
    a.slot[i] = atomicAdd(&v.cnt[a.s.wf[i]], 1);
}

struct CntOf {
  const int32_t* cnt;
  __device__ int64_t operator()(int64_t w) const { return cnt[w]; }
};

__global__ void sig_scatter_kernel(SigArgs a) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x)
    a.seg[a.seg_off[a.s.wf[i]] + a.slot[i]] = (int32_t)i;
}

// Segment sort by signal index: insertion sort for the usual handful, heap sort otherwise (a
// workflow's signals are sequential work anyway, so O(c log c) per workflow is in budget).
__device__ void sift(int32_t* x, int64_t root, int64_t end) {
  while (2 * root + 1 < end) {
    int64_t c = 2 * root + 1;
    if (c + 1 < end && x[c + 1] > x[c]) ++c;
    if (x[root] >= x[c]) return;
    const int32_t t = x[root];
    x[root] = x[c];
    x[c] = t;
    root = c;
  }
}
__device__ void sort_segment(int32_t* x, int64_t c) {
  if (c <= 16) {
    for (int64_t i = 1; i < c; ++i) {
      const int32_t k = x[i];
      int64_t j = i - 1;
      while (j >= 0 && x[j] > k) {
        x[j + 1] = x[j];
        --j;
      }
      x[j + 1] = k;
    }
    return;
  }
  for (int64_t s = c / 2 - 1; s >= 0; --s) sift(x, s, c);
  for (int64_t e = c - 1; e > 0; --e) {
    const int32_t t = x[0];
    x[0] = x[e];
    x[e] = t;
    sift(x, 0, e);
  }
}

// A workflow's (wf, b) tracker entries during its signal replay: for NB <= N they are loaded once
// into thread-local arrays and written back at the end (every signal used to pay dependent global
// round trips on them); N = 0 accesses global memory directly.
template <int N>
struct Ents {
  uint8_t pr[N], pv[N];
  int32_t inf[N];
  int64_t tok[N];
  double t[N];
  __device__ Ents(const TrackerView& v, int64_t e0, int32_t nb) {
    for (int32_t b = 0; b < nb; ++b) {
      pr[b] = v.present[e0 + b];
      pv[b] = v.preserved[e0 + b];
      inf[b] = v.inflight[e0 + b];
      tok[b] = v.tokens[e0 + b];
      t[b] = v.ts[e0 + b];
    }
  }
  __device__ void store(const TrackerView& v, int64_t e0, int32_t nb) const {
    for (int32_t b = 0; b < nb; ++b) {
      v.present[e0 + b] = pr[b];
      v.preserved[e0 + b] = pv[b];
      v.inflight[e0 + b] = inf[b];
      v.tokens[e0 + b] = tok[b];
      v.ts[e0 + b] = t[b];
    }
  }
  __device__ uint8_t& present(int32_t b) { return pr[b]; }
  __device__ uint8_t& preserved(int32_t b) { return pv[b]; }
  __device__ int32_t& inflight(int32_t b) { return inf[b]; }
  __device__ int64_t& tokens(int32_t b) { return tok[b]; }
  __device__ double& ts(int32_t b) { return t[b]; }
};
template <>
struct Ents<0> {
  const TrackerView& v;
  int64_t e0;
  __device__ Ents(const TrackerView& vv, int64_t e, int32_t) : v(vv), e0(e) {}
  __device__ void store(const TrackerView&, int64_t, int32_t) const {}
  __device__ uint8_t& present(int32_t b) { return v.present[e0 + b]; }
  __device__ uint8_t& preserved(int32_t b) { return v.preserved[e0 + b]; }
  __device__ int32_t& inflight(int32_t b) { return v.inflight[e0 + b]; }
  __device__ int64_t& tokens(int32_t b) { return v.tokens[e0 + b]; }
  __device__ double& ts(int32_t b) { return v.ts[e0 + b]; }
};

// Stage bitsets (started_ever_ / open_stages_): one word in registers when every stage id of the
// tracker fits 64 bits (ONE), else SW words in global memory.
template <bool ONE>
struct Stages;
template <>
struct Stages<true> {
  unsigned long long st, op;
  __device__ Stages(const TrackerView& v, int64_t w) : st(v.started[w]), op(v.open_[w]) {}
  __device__ bool started(int32_t s) const { return (st >> s) & 1ull; }
  __device__ bool open(int32_t s) const { return (op >> s) & 1ull; }
  __device__ void start(int32_t s) { st |= 1ull << s, op |= 1ull << s; }
  __device__ void close(int32_t s) { op &= ~(1ull << s); }
  __device__ void clear() { st = op = 0; }
  __device__ void store(const TrackerView& v, int64_t w) const { v.started[w] = st, v.open_[w] = op; }
};
template <>
struct Stages<false> {
  unsigned long long *st, *op;
  int32_t sw;
  __device__ Stages(const TrackerView& v, int64_t w)
      : st(v.started + w * v.SW), op(v.open_ + w * v.SW), sw(v.SW) {}
  __device__ bool started(int32_t s) const { return (st[s >> 6] >> (s & 63)) & 1ull; }
  __device__ bool open(int32_t s) const { return (op[s >> 6] >> (s & 63)) & 1ull; }
  __device__ void start(int32_t s) { st[s >> 6] |= 1ull << (s & 63), op[s >> 6] |= 1ull << (s & 63); }
  __device__ void close(int32_t s) { op[s >> 6] &= ~(1ull << (s & 63)); }
  __device__ void clear() {
    for (int32_t q = 0; q < sw; ++q) st[q] = op[q] = 0;
  }
  __device__ void store(const TrackerView&, int64_t) const {}
};

template <int NBC, bool ONE>
__global__ void __launch_bounds__(32) sig_resolve_kernel(SigArgs a, TrackerView v) {
  pdl_enter();
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= v.W) return;
  const int32_t c = v.cnt[w];
  if (c == 0) return;
  v.cnt[w] = 0;  // ready for the next batch
  int32_t* seg = a.seg + a.seg_off[w];
  // the usual handful of signal indices sorted in (L1-resident) local memory, longer segments in place
  constexpr int SMALL = 32;
  int32_t sx[SMALL];
  const bool small = c <= SMALL;
  if (small) {
    for (int32_t q = 0; q < c; ++q) sx[q] = seg[q];
    sort_segment(sx, c);
  } else {
    sort_segment(seg, c);
  }
  const int32_t NB = v.NB;
  const int64_t e0 = w * NB;
  Ents<NBC> E(v, e0, NB);  // the workflow's (wf, b) entries: registers / local memory when NB <= NBC
  Stages<ONE> S(v, w);
  // workflow state in registers for the whole segment
  uint8_t completed = v.completed[w];
  int32_t ocnt = v.open_cnt[w];
  uint8_t lvalid = v.last_valid[w];
  int32_t lb = v.last_b[w], lm = v.last_model[w];
  int64_t lt = v.last_tokens[w];
  int32_t coff = v.chain_off[w], clen = v.chain_len[w];
  bool failed = false;
  // signal fields are prefetched one signal ahead, so the next signal's loads overlap this one's
  // resolution (each workflow's signals are a sequential dependency chain)
  struct Sig {
    int64_t i, T;
    int32_t s, b, m;
    uint8_t kind, ov;
  };
  auto load = [&](int64_t i) {
    Sig x;
    x.i = i;
    x.kind = a.s.kind[i];
    x.s = a.s.stage[i];
    x.b = a.s.backend[i];
    x.m = a.s.model[i];
    x.T = a.s.tokens[i];
    x.ov = a.s.override_ ? a.s.override_[i] : O_NONE;
    return x;
  };
  Sig nx = load(small ? sx[0] : seg[0]);
  for (int32_t q = 0; q < c; ++q) {
    const Sig cur = nx;
    if (q + 1 < c) nx = load(small ? sx[q + 1] : seg[q + 1]);
    const int64_t i = cur.i;
    const uint8_t kind = cur.kind;
    const bool wfc = kind == K_WF_COMPLETE;
    const int32_t s = wfc ? 0 : cur.s;
    const int32_t b = wfc ? -1 : cur.b;
    const int32_t m = wfc ? -1 : cur.m;
    const int64_t T = wfc ? 0 : cur.T;
    const uint8_t ov = wfc ? O_NONE : cur.ov;
    a.r.count[i] = 0;
    if (failed) {
      a.r.status[i] = SFMM_SIG_SKIPPED;
      continue;
    }
    // check_order (memory.cpp:256-285)
    if (completed || (kind == K_START && S.started(s)) || (kind == K_COMPLETE && !S.open(s)) ||
        (wfc && ocnt != 0)) {
      a.r.status[i] = SFMM_SIG_OUT_OF_ORDER;
      failed = true;
      continue;
    }
    const unsigned long long tag0 = mod_tag(v.epoch, i, 0), tag1 = mod_tag(v.epoch, i, 1);
    // resolve (memory.cpp:287-310); records go straight to the signal's slots
    uint8_t* rk = a.r.kind + i * NB;
    int32_t* rb = a.r.backend + i * NB;
    uint8_t* rr = a.r.reason + i * NB;
    int na = 0;
    if (kind == K_START && ov != O_NONE) {
      if (!lvalid) {
        rk[0] = A_NOOP, rb[0] = -1, rr[0] = R_OVERRIDE;
      } else {
        rk[0] = ov == O_FLUSH ? A_FLUSH : A_PRESERVE, rb[0] = lb, rr[0] = R_OVERRIDE;
        if (ov == O_FLUSH) {  // applied (erases the entry)
          E.present(lb) = 0;
          v.mod[e0 + lb] = tag0;
        }
      }
      na = 1;
    } else {
      const int32_t len = coff >= 0 ? clen : v.def_len;
      const uint8_t* chain = v.arena + (coff >= 0 ? coff : v.def_off);
      for (int32_t p = 0; p < len && na == 0; ++p) {
        const uint8_t pol = chain[p];
        if (pol == P_PSI) {  // policy_preserve_small_increment (memory.cpp:116-125)
          if (kind == K_START && lvalid && lb == b && lm == m && T - lt < v.tau) {
            rk[0] = A_PRESERVE, rb[0] = b, rr[0] = R_PSI;
            na = 1;
          }
        } else {  // policy_flush_at_boundary (memory.cpp:127-148)
          if (wfc) {  // preserved entries in backend-ref order
            for (int32_t k = 0; k < NB; ++k) {
              const int32_t bb = v.border[k];
              if (E.present(bb) && E.preserved(bb)) {
                rk[na] = A_FLUSH, rb[na] = bb, rr[na] = R_FAB;
                E.present(bb) = 0;  // applied
                ++na;
              }
            }
          } else if (kind == K_START && lvalid && (lb != b || lm != m) && E.present(lb) &&
                     E.preserved(lb)) {
            rk[0] = A_FLUSH, rb[0] = lb, rr[0] = R_FAB;
            E.present(lb) = 0;  // applied
            v.mod[e0 + lb] = tag0;
            na = 1;
          }
        }
      }
      if (na == 0) {
        rk[0] = A_NOOP, rb[0] = -1, rr[0] = R_EXHAUSTED;
        na = 1;
      }
    }
    // apply_and_record (memory.cpp:312-328): a flush that applied erases the entry — done as each
    // flush is recorded above (the records are write-only here: no read-back round trip)
    a.r.count[i] = na;
    // update_tracker (memory.cpp:330-360)
    if (kind == K_START) {
      S.start(s);
      ++ocnt;
      const int32_t f = E.inflight(b) + 1;
      E.inflight(b) = f;
      if (f < 0) {  // a count left negative by an earlier throw: adjust_in_flight stores it and
                    // throws again (memory.cpp:90-92)
        a.r.status[i] = SFMM_SIG_NEGATIVE_IN_FLIGHT;
        failed = true;
        continue;
      }
    } else if (kind == K_COMPLETE) {
      S.close(s);
      --ocnt;
      const int32_t f = E.inflight(b) - 1;
      E.inflight(b) = f;
      if (f < 0) {  // adjust_in_flight threw after storing the count (memory.cpp:90-92)
        a.r.status[i] = SFMM_SIG_NEGATIVE_IN_FLIGHT;
        failed = true;
        continue;
      }
      E.present(b) = 1;
      E.preserved(b) = T > 0;
      E.tokens(b) = T;
      E.ts(b) = a.s.ts[i];
      v.mod[e0 + b] = tag1;
      lvalid = 1, lb = b, lm = m, lt = T;
    } else {
      completed = 1;
      for (int32_t bb = 0; bb < NB; ++bb) {
        E.present(bb) = 0;
        E.inflight(bb) = 0;
        v.mod[e0 + bb] = tag1;
      }
      S.clear();
      lvalid = 0, ocnt = 0, coff = -1, clen = 0;
    }
    a.r.status[i] = SFMM_SIG_OK;
  }
  E.store(v, e0, NB);
  S.store(v, w);
  v.completed[w] = completed;
  v.open_cnt[w] = ocnt;
  v.last_valid[w] = lvalid;
  v.last_b[w] = lb;
  v.last_model[w] = lm;
  v.last_tokens[w] = lt;
  v.chain_off[w] = coff;
  v.chain_len[w] = clen;
}

// mark_unpreserved for flushes that failed twice (memory.cpp:319-325): only if the flush of that
// signal (or tick) was the entry's last modification.
__global__ void flush_failed_kernel(TrackerView v, int64_t n, const int32_t* wf, const int32_t* b,
                                    const int64_t* sig) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (int64_t)wf[i] * v.NB + b[i];
    if (v.mod[e] == mod_tag(v.epoch, sig[i] < 0 ? 0 : sig[i], 0)) {
      v.present[e] = 1;
      v.preserved[e] = 0;
    }
  }
}

// ---- pressure tick (K6): one launch -------------------------------------------------------
// Per backend b with util > tau': every CTA reduces its workflows' idle preserved (wf, b) entries
// to one candidate (warp shuffles, then across warps); the last CTA to finish reduces the CTA
// candidates, writes the victims and erases their entries (mark_flushed).
__global__ void __launch_bounds__(256) pressure_tick_kernel(TrackerView v) {
  __shared__ Cand red[32];
  __shared__ bool last;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int32_t b = 0; b < v.NB; ++b) {
    Cand c = cand_none();
    if (v.util[b] > v.tau_p) {
      for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < v.W; w += stride) {
        const int64_t e = w * v.NB + b;
        if (v.present[e] && v.preserved[e] && v.inflight[e] <= 0) {
          const Cand d{ts_order_key(v.ts[e]), v.rank[w], w};
          if (cand_less(d, c)) c = d;
        }
      }
    }
    c = block_argmin(c, red);
    if (threadIdx.x == 0) v.part[(int64_t)blockIdx.x * v.NB + b] = c;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(v.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int32_t b = 0; b < v.NB; ++b) {
    Cand c = cand_none();
    for (int64_t p = threadIdx.x; p < gridDim.x; p += blockDim.x) {
      const Cand d = cand_load(&v.part[p * v.NB + b]);
      if (cand_less(d, c)) c = d;
    }
    c = block_argmin(c, red);
    if (threadIdx.x == 0) {
      v.victim[b] = (int32_t)c.idx;
      if (c.idx >= 0) {
        const int64_t e = c.idx * v.NB + b;
        v.present[e] = 0;  // mark_flushed
        v.mod[e] = mod_tag(v.epoch, 0, 0);
      }
    }
  }
  if (threadIdx.x == 0) *v.done = 0;
}

static int sm_count_t() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static int on_signals_dev(sfmm_tracker* t, int64_t n, const sfmm_signals& s, const sfmm_records& r) {
  if (n <= 0) return 0;
  cudaStream_t st = t->stream;
  Carver cv;
  const size_t o_slot = cv.take<int32_t>(n), o_off = cv.take<int64_t>(t->W + 1),
               o_seg = cv.take<int32_t>(n), o_tmp = cv.take<int64_t>(scan_scratch_elems(t->W));
  if (int rc = t->scratch.ensure(cv.off)) return rc;
  char* base = t->scratch.as<char>();
  SigArgs a;
  a.n = n;
  a.s = s;
  a.r = r;
  a.slot = reinterpret_cast<int32_t*>(base + o_slot);
  a.seg_off = reinterpret_cast<int64_t*>(base + o_off);
  a.seg = reinterpret_cast<int32_t*>(base + o_seg);
  ++t->epoch;
  const TrackerView v = view(t);
  const int sms = sm_count_t();
  SFKV_CUDA(launch_pdl(sig_count_kernel, dim3(grid_for(n, 256, sms * 8)), dim3(256), st, a, v));
  SFKV_LAUNCH_CHECK("sig_count_kernel");
  if (int rc = exclusive_scan(CntOf{t->cnt}, t->W, a.seg_off, reinterpret_cast<int64_t*>(base + o_tmp), st))
    return rc;
  SFKV_CUDA(launch_pdl(sig_scatter_kernel, dim3(grid_for(n, 256, sms * 8)), dim3(256), st, a));
  const dim3 g((unsigned)((t->W + 31) / 32));
  if (t->NB <= 8 && t->SW == 1)  // spread over every SM
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<8, true>, g, dim3(32), st, a, v));
  else if (t->NB <= 8)
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<8, false>, g, dim3(32), st, a, v));
  else if (t->SW == 1)
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<0, true>, g, dim3(32), st, a, v));
  else
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<0, false>, g, dim3(32), st, a, v));
  SFKV_LAUNCH_CHECK("sig_scatter/resolve");
  return 0;
}

}  // namespace sfkv

using namespace sfkv;

template <class T>
static int talloc(T** p, size_t n) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    return cuda_fail(e, "tracker cudaMalloc");
  }
  return 0;
}

static void tracker_free_arrays(sfmm_tracker* t) {
  cudaFree(t->completed);
  cudaFree(t->started);
  cudaFree(t->open_);
  cudaFree(t->open_cnt);
  cudaFree(t->last_valid);
  cudaFree(t->last_b);
  cudaFree(t->last_model);
  cudaFree(t->last_tokens);
  cudaFree(t->chain_off);
  cudaFree(t->chain_len);
  cudaFree(t->rank);
  cudaFree(t->cnt);
  cudaFree(t->present);
  cudaFree(t->preserved);
  cudaFree(t->tokens);
  cudaFree(t->ts);
  cudaFree(t->inflight);
  cudaFree(t->mod);
  cudaFree(t->border);
  cudaFree(t->victim);
  cudaFree(t->util);
}

static void tracker_free(sfmm_tracker* t) {
  tracker_free_arrays(t);
  cudaFree(t->arena);
  cudaFree(t->done);
  t->part.release();
  t->scratch.release();
  t->io.release();
  if (t->own_stream && t->stream) cudaStreamDestroy(t->stream);
}

// Allocates every per-workflow / per-entry / per-backend array of t for (W, NB, SW).
static int tracker_alloc_arrays(sfmm_tracker* t) {
  const size_t W = t->W, E = W * t->NB, NB = t->NB, WS = W * t->SW;
  int rc = 0;
  if ((rc = talloc(&t->completed, W)) || (rc = talloc(&t->started, WS)) || (rc = talloc(&t->open_, WS)) ||
      (rc = talloc(&t->open_cnt, W)) || (rc = talloc(&t->last_valid, W)) || (rc = talloc(&t->last_b, W)) ||
      (rc = talloc(&t->last_model, W)) || (rc = talloc(&t->last_tokens, W)) ||
      (rc = talloc(&t->chain_off, W)) || (rc = talloc(&t->chain_len, W)) || (rc = talloc(&t->rank, W)) ||
      (rc = talloc(&t->cnt, W)) || (rc = talloc(&t->present, E)) || (rc = talloc(&t->preserved, E)) ||
      (rc = talloc(&t->tokens, E)) || (rc = talloc(&t->ts, E)) || (rc = talloc(&t->inflight, E)) ||
      (rc = talloc(&t->mod, E)) || (rc = talloc(&t->border, NB)) || (rc = talloc(&t->victim, NB)) ||
      (rc = talloc(&t->util, NB)))
    return rc;
  return 0;
}

static bool valid_policy(uint8_t p) {
  return p == SFMM_POLICY_PRESERVE_SMALL_INCREMENT || p == SFMM_POLICY_FLUSH_AT_BOUNDARY;
}

// Offset of a chain in the arena (deduplicated; the device copy grows by reallocation).
static int chain_offset(sfmm_tracker* t, const std::vector<uint8_t>& chain, int32_t* off) {
  auto it = t->chain_at.find(chain);
  if (it != t->chain_at.end()) {
    *off = it->second;
    return 0;
  }
  const int32_t o = (int32_t)t->arena_host.size();
  t->arena_host.insert(t->arena_host.end(), chain.begin(), chain.end());
  if (t->arena_host.size() > t->arena_cap || !t->arena) {
    size_t cap = t->arena_cap ? t->arena_cap : 256;
    while (cap < t->arena_host.size()) cap *= 2;
    uint8_t* a = nullptr;
    if (int rc = talloc(&a, cap)) return rc;
    SFKV_CUDA(cudaStreamSynchronize(t->stream));
    cudaFree(t->arena);
    t->arena = a;
    t->arena_cap = cap;
    SFKV_CUDA(cudaMemcpyAsync(t->arena, t->arena_host.data(), t->arena_host.size(), cudaMemcpyHostToDevice,
                              t->stream));
  } else if (!chain.empty()) {
    SFKV_CUDA(cudaMemcpyAsync(t->arena + o, t->arena_host.data() + o, chain.size(), cudaMemcpyHostToDevice,
                              t->stream));
  }
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  t->chain_at.emplace(chain, o);
  *off = o;
  return 0;
}

static int upload_identity_order(sfmm_tracker* t) {
  std::vector<int32_t> id(t->NB);
  for (int32_t b = 0; b < t->NB; ++b) id[b] = b;
  SFKV_CUDA(cudaMemcpyAsync(t->border, id.data(), id.size() * sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

// Re-layout of a grown tracker: old [W0][NB0] entries and [W0][SW0] stage words into the new
// shape; new slots / backends start empty.
__global__ void tracker_regrow_kernel(TrackerView o, TrackerView n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n.W; w += stride) {
    const bool old = w < o.W;
    n.completed[w] = old ? o.completed[w] : 0;
    for (int32_t q = 0; q < n.SW; ++q) {
      n.started[w * n.SW + q] = old && q < o.SW ? o.started[w * o.SW + q] : 0;
      n.open_[w * n.SW + q] = old && q < o.SW ? o.open_[w * o.SW + q] : 0;
    }
    n.open_cnt[w] = old ? o.open_cnt[w] : 0;
    n.last_valid[w] = old ? o.last_valid[w] : 0;
    n.last_b[w] = old ? o.last_b[w] : -1;
    n.last_model[w] = old ? o.last_model[w] : -1;
    n.last_tokens[w] = old ? o.last_tokens[w] : 0;
    n.chain_off[w] = old ? o.chain_off[w] : -1;
    n.chain_len[w] = old ? o.chain_len[w] : 0;
    n.rank[w] = old ? o.rank[w] : (uint32_t)w;
    n.cnt[w] = 0;
    for (int32_t b = 0; b < n.NB; ++b) {
      const bool ob = old && b < o.NB;
      const int64_t e = w * n.NB + b, f = w * o.NB + b;
      n.present[e] = ob ? o.present[f] : 0;
      n.preserved[e] = ob ? o.preserved[f] : 0;
      n.tokens[e] = ob ? o.tokens[f] : 0;
      n.ts[e] = ob ? o.ts[f] : 0;
      n.inflight[e] = ob ? o.inflight[f] : 0;
      n.mod[e] = ob ? o.mod[f] : 0;
    }
  }
}

extern "C" {

int sfmm_tracker_create(const sfmm_config* cfg, sfmm_tracker** out) {
  if (!cfg || !out) return fail(SFKV_EINVAL, "tracker_create: null argument");
  if (cfg->max_workflows <= 0 || cfg->n_backends <= 0 || cfg->max_stages < 0 || cfg->chain_len < 0 ||
      (cfg->chain_len > 0 && !cfg->chain) || cfg->tau <= 0 || !(cfg->tau_pressure > 0) ||
      cfg->tau_pressure > 1)  // memory.cpp:240-243
    return fail(SFKV_EINVAL, "tracker_create: invalid configuration");
  for (int i = 0; i < cfg->chain_len; ++i)
    if (!valid_policy(cfg->chain[i])) return fail(SFKV_EINVAL, "tracker_create: unknown memory policy");  // memory.cpp:182
  if (int rc = check_device(cfg->device)) return rc;
  DeviceGuard g(cfg->device);
  auto* t = new sfmm_tracker;
  t->device = cfg->device;
  t->tau = cfg->tau;
  t->tau_p = cfg->tau_pressure;
  t->W = cfg->max_workflows;
  t->NB = cfg->n_backends;
  t->SW = cfg->max_stages > 0 ? (cfg->max_stages + 63) / 64 : 1;
  cudaError_t e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete t;
    return cuda_fail(e, "tracker stream");
  }
  t->own_stream = true;
  int rc = tracker_alloc_arrays(t);
  if (!rc) rc = talloc(&t->done, 1);
  if (!rc) rc = chain_offset(t, std::vector<uint8_t>(cfg->chain, cfg->chain + cfg->chain_len), &t->def_off);
  if (!rc) rc = upload_identity_order(t);
  if (rc) {
    tracker_free(t);
    delete t;
    return rc;
  }
  t->def_len = cfg->chain_len;
  cudaMemsetAsync(t->done, 0, sizeof(unsigned int), t->stream);
  tracker_init_kernel<<<grid_for(t->W, 256, 4096), 256, 0, t->stream>>>(view(t), t->W, nullptr);
  e = cudaStreamSynchronize(t->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    tracker_free(t);
    delete t;
    return cuda_fail(e, "tracker init");
  }
  *out = t;
  return 0;
}

int sfmm_tracker_destroy(sfmm_tracker* t) {
  if (!t) return fail(SFKV_EINVAL, "tracker_destroy: null tracker");
  DeviceGuard g(t->device);
  cudaStreamSynchronize(t->stream);
  tracker_free(t);
  delete t;
  return 0;
}

int sfmm_tracker_reserve(sfmm_tracker* t, int32_t max_workflows, int32_t n_backends, int32_t max_stages) {
  if (!t) return fail(SFKV_EINVAL, "tracker_reserve: null tracker");
  DeviceGuard g(t->device);
  const int32_t W1 = std::max(t->W, max_workflows), NB1 = std::max(t->NB, n_backends);
  const int32_t SW1 = std::max(t->SW, (int32_t)((std::max(max_stages, 0) + 63) / 64));
  if (W1 == t->W && NB1 == t->NB && SW1 == t->SW) return 0;
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  auto* n = new sfmm_tracker;  // holds the grown arrays until they are swapped in
  n->W = W1, n->NB = NB1, n->SW = SW1;
  if (int rc = tracker_alloc_arrays(n)) {
    tracker_free_arrays(n);
    delete n;
    return rc;
  }
  tracker_regrow_kernel<<<grid_for(W1, 256, 4096), 256, 0, t->stream>>>(view(t), view(n));
  SFKV_LAUNCH_CHECK("tracker_regrow_kernel");
  std::vector<int32_t> order(NB1);
  SFKV_CUDA(cudaMemcpyAsync(order.data(), t->border, t->NB * sizeof(int32_t), cudaMemcpyDeviceToHost, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  for (int32_t b = t->NB; b < NB1; ++b) order[b] = b;  // new backends last until re-ordered
  SFKV_CUDA(cudaMemcpyAsync(n->border, order.data(), NB1 * sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  std::swap(t->completed, n->completed);
  std::swap(t->started, n->started);
  std::swap(t->open_, n->open_);
  std::swap(t->open_cnt, n->open_cnt);
  std::swap(t->last_valid, n->last_valid);
  std::swap(t->last_b, n->last_b);
  std::swap(t->last_model, n->last_model);
  std::swap(t->last_tokens, n->last_tokens);
  std::swap(t->chain_off, n->chain_off);
  std::swap(t->chain_len, n->chain_len);
  std::swap(t->rank, n->rank);
  std::swap(t->cnt, n->cnt);
  std::swap(t->present, n->present);
  std::swap(t->preserved, n->preserved);
  std::swap(t->tokens, n->tokens);
  std::swap(t->ts, n->ts);
  std::swap(t->inflight, n->inflight);
  std::swap(t->mod, n->mod);
  std::swap(t->border, n->border);
  std::swap(t->victim, n->victim);
  std::swap(t->util, n->util);
  tracker_free_arrays(n);  // the old shape's arrays
  delete n;
  t->W = W1, t->NB = NB1, t->SW = SW1;
  return 0;
}

int sfmm_tracker_set_stream(sfmm_tracker* t, void* stream) {
  if (!t) return fail(SFKV_EINVAL, "tracker_set_stream: null tracker");
  DeviceGuard g(t->device);
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  if (t->own_stream) cudaStreamDestroy(t->stream);
  t->stream = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream (as pools)
  t->own_stream = false;
  return 0;
}

int sfmm_tracker_reset(sfmm_tracker* t) {
  if (!t) return fail(SFKV_EINVAL, "tracker_reset: null tracker");
  DeviceGuard g(t->device);
  tracker_init_kernel<<<grid_for(t->W, 256, 4096), 256, 0, t->stream>>>(view(t), t->W, nullptr);
  SFKV_LAUNCH_CHECK("tracker_init_kernel");
  return 0;
}

int sfmm_reset_workflows(sfmm_tracker* t, int64_t n, const int32_t* wf) {
  if (!t || n < 0 || (n && !wf)) return fail(SFKV_EINVAL, "reset_workflows: bad argument");
  for (int64_t i = 0; i < n; ++i)
    if (wf[i] < 0 || wf[i] >= t->W) return fail(SFKV_EINVAL, "reset_workflows: slot out of range");
  if (n == 0) return 0;
  DeviceGuard g(t->device);
  Carver cv;
  const size_t o = cv.take<int32_t>(n);
  if (int rc = t->io.ensure(cv.off)) return rc;
  int32_t* d = reinterpret_cast<int32_t*>(t->io.as<char>() + o);
  SFKV_CUDA(cudaMemcpyAsync(d, wf, n * sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  tracker_init_kernel<<<grid_for(n, 256, 1024), 256, 0, t->stream>>>(view(t), n, d);
  SFKV_LAUNCH_CHECK("tracker_init_kernel (slots)");
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_tracker_sync(sfmm_tracker* t) {
  if (!t) return fail(SFKV_EINVAL, "tracker_sync: null tracker");
  DeviceGuard g(t->device);
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_set_workflow_chain(sfmm_tracker* t, int32_t wf, int32_t len, const uint8_t* policies) {
  if (!t || wf < 0 || wf >= t->W || len < 0 || (len && !policies))
    return fail(SFKV_EINVAL, "set_workflow_chain: bad argument");
  if (len == 0) return 0;  // memory.cpp:248
  for (int i = 0; i < len; ++i)
    if (!valid_policy(policies[i])) return fail(SFKV_EINVAL, "set_workflow_chain: unknown memory policy");
  DeviceGuard g(t->device);
  int32_t off = 0;
  if (int rc = chain_offset(t, std::vector<uint8_t>(policies, policies + len), &off)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(t->chain_off + wf, &off, sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaMemcpyAsync(t->chain_len + wf, &len, sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_set_workflow_ranks(sfmm_tracker* t, int64_t n, const uint32_t* rank) {
  if (!t || n < 0 || n > t->W || (n && !rank)) return fail(SFKV_EINVAL, "set_workflow_ranks: bad argument");
  DeviceGuard g(t->device);
  if (n) SFKV_CUDA(cudaMemcpyAsync(t->rank, rank, n * sizeof(uint32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_set_backend_order(sfmm_tracker* t, int32_t n, const int32_t* order) {
  if (!t || n != t->NB || !order) return fail(SFKV_EINVAL, "set_backend_order: need n_backends entries");
  std::vector<char> seen(t->NB, 0);
  for (int32_t k = 0; k < n; ++k) {
    if (order[k] < 0 || order[k] >= t->NB || seen[order[k]]) return fail(SFKV_EINVAL, "set_backend_order: not a permutation");
    seen[order[k]] = 1;
  }
  DeviceGuard g(t->device);
  SFKV_CUDA(cudaMemcpyAsync(t->border, order, n * sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_on_signal_batch_dev(sfmm_tracker* t, int64_t n, const sfmm_signals* sig, const sfmm_records* out) {
  if (!t || !sig || !out || n < 0) return fail(SFKV_EINVAL, "on_signal_batch_dev: bad argument");
  if (n > INT32_MAX) return fail(SFKV_EINVAL, "on_signal_batch_dev: batch too large");
  if (n > 0 && (!sig->kind || !sig->wf || !sig->stage || !sig->backend || !sig->model || !sig->tokens ||
                !sig->ts || !out->count || !out->status || !out->kind || !out->backend || !out->reason))
    return fail(SFKV_EINVAL, "on_signal_batch_dev: null array (only override_ may be null)");
  DeviceGuard g(t->device);
  return on_signals_dev(t, n, *sig, *out);
}

int sfmm_on_signal_batch(sfmm_tracker* t, int64_t n, const sfmm_signals* sig, const sfmm_records* out) {
  if (!t || !sig || !out || n < 0) return fail(SFKV_EINVAL, "on_signal_batch: bad argument");
  if (n == 0) return 0;
  if (n > INT32_MAX) return fail(SFKV_EINVAL, "on_signal_batch: batch too large");
  if (!sig->kind || !sig->wf || !sig->ts || !out->count || !out->status || !out->kind ||
      !out->backend || !out->reason)
    return fail(SFKV_EINVAL, "on_signal_batch: null array");
  const int64_t max_stage = (int64_t)t->SW * 64;
  for (int64_t i = 0; i < n; ++i) {  // host-side validation of the dense ids
    const bool wfc = sig->kind[i] == K_WF_COMPLETE;
    if (sig->kind[i] > K_WF_COMPLETE || sig->wf[i] < 0 || sig->wf[i] >= t->W ||
        (!wfc && (!sig->stage || !sig->backend || !sig->model || !sig->tokens || sig->stage[i] < 0 ||
                  sig->stage[i] >= max_stage || sig->backend[i] < 0 || sig->backend[i] >= t->NB)))
      return fail(SFKV_EINVAL, "on_signal_batch: signal field out of range (sfmm_tracker_reserve grows "
                               "slots, backends and stages)");
  }
  DeviceGuard g(t->device);
  const int64_t NR = n * t->NB;
  Carver cv;
  const size_t o_k = cv.take<uint8_t>(n), o_w = cv.take<int32_t>(n), o_s = cv.take<int32_t>(n),
               o_b = cv.take<int32_t>(n), o_m = cv.take<int32_t>(n), o_t = cv.take<int64_t>(n),
               o_ts = cv.take<double>(n), o_o = cv.take<uint8_t>(n), o_rc = cv.take<int32_t>(n),
               o_rs = cv.take<uint8_t>(n), o_rk = cv.take<uint8_t>(NR), o_rb = cv.take<int32_t>(NR),
               o_rr = cv.take<uint8_t>(NR);
  if (int rc = t->io.ensure(cv.off)) return rc;
  char* b = t->io.as<char>();
  cudaStream_t st = t->stream;
  auto up = [&](size_t off, const void* src, size_t bytes) -> int {
    if (src) SFKV_CUDA(cudaMemcpyAsync(b + off, src, bytes, cudaMemcpyHostToDevice, st));
    else SFKV_CUDA(cudaMemsetAsync(b + off, 0, bytes, st));
    return 0;
  };
  int rc = 0;
  if ((rc = up(o_k, sig->kind, n)) || (rc = up(o_w, sig->wf, n * 4)) || (rc = up(o_s, sig->stage, n * 4)) ||
      (rc = up(o_b, sig->backend, n * 4)) || (rc = up(o_m, sig->model, n * 4)) ||
      (rc = up(o_t, sig->tokens, n * 8)) || (rc = up(o_ts, sig->ts, n * 8)) ||
      (rc = up(o_o, sig->override_, n)))
    return rc;
  sfmm_signals ds{reinterpret_cast<const uint8_t*>(b + o_k), reinterpret_cast<const int32_t*>(b + o_w),
                  reinterpret_cast<const int32_t*>(b + o_s), reinterpret_cast<const int32_t*>(b + o_b),
                  reinterpret_cast<const int32_t*>(b + o_m), reinterpret_cast<const int64_t*>(b + o_t),
                  reinterpret_cast<const double*>(b + o_ts), reinterpret_cast<const uint8_t*>(b + o_o)};
  sfmm_records dr{reinterpret_cast<int32_t*>(b + o_rc), reinterpret_cast<uint8_t*>(b + o_rs),
                  reinterpret_cast<uint8_t*>(b + o_rk), reinterpret_cast<int32_t*>(b + o_rb),
                  reinterpret_cast<uint8_t*>(b + o_rr)};
  if ((rc = on_signals_dev(t, n, ds, dr))) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out->count, dr.count, n * 4, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(out->status, dr.status, n, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(out->kind, dr.kind, NR, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(out->backend, dr.backend, NR * 4, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaMemcpyAsync(out->reason, dr.reason, NR, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfmm_flush_failed(sfmm_tracker* t, int64_t n, const int32_t* wf, const int32_t* backend, const int64_t* sig) {
  if (!t || n < 0 || (n && (!wf || !backend || !sig))) return fail(SFKV_EINVAL, "flush_failed: bad argument");
  for (int64_t i = 0; i < n; ++i)
    if (wf[i] < 0 || wf[i] >= t->W || backend[i] < 0 || backend[i] >= t->NB)
      return fail(SFKV_EINVAL, "flush_failed: slot or backend out of range");
  if (n == 0) return 0;
  DeviceGuard g(t->device);
  Carver cv;
  const size_t o_w = cv.take<int32_t>(n), o_b = cv.take<int32_t>(n), o_s = cv.take<int64_t>(n);
  if (int rc = t->io.ensure(cv.off)) return rc;
  char* b = t->io.as<char>();
  cudaStream_t st = t->stream;
  SFKV_CUDA(cudaMemcpyAsync(b + o_w, wf, n * 4, cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_b, backend, n * 4, cudaMemcpyHostToDevice, st));
  SFKV_CUDA(cudaMemcpyAsync(b + o_s, sig, n * 8, cudaMemcpyHostToDevice, st));
  flush_failed_kernel<<<grid_for(n, 256, 1024), 256, 0, st>>>(view(t), n, reinterpret_cast<int32_t*>(b + o_w),
                                                              reinterpret_cast<int32_t*>(b + o_b),
                                                              reinterpret_cast<int64_t*>(b + o_s));
  SFKV_LAUNCH_CHECK("flush_failed_kernel");
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfmm_pressure_tick_dev(sfmm_tracker* t, const double* util, int32_t* out_victim) {
  if (!t || !util || !out_victim) return fail(SFKV_EINVAL, "pressure_tick_dev: null argument");
  DeviceGuard g(t->device);
  cudaStream_t st = t->stream;
  const int grid = grid_for(t->W, 256, sm_count_t() * 2);
  if (int rc = t->part.ensure((size_t)grid * t->NB * sizeof(Cand))) return rc;
  if (util != t->util)
    SFKV_CUDA(cudaMemcpyAsync(t->util, util, t->NB * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ++t->epoch;
  pressure_tick_kernel<<<grid, 256, 0, st>>>(view(t));
  SFKV_LAUNCH_CHECK("pressure_tick_kernel");
  if (out_victim != t->victim)
    SFKV_CUDA(cudaMemcpyAsync(out_victim, t->victim, t->NB * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return 0;
}

int sfmm_pressure_tick(sfmm_tracker* t, const double* util, int32_t* out_victim) {
  if (!t || !util || !out_victim) return fail(SFKV_EINVAL, "pressure_tick: null argument");
  DeviceGuard g(t->device);
  cudaStream_t st = t->stream;
  SFKV_CUDA(cudaMemcpyAsync(t->util, util, t->NB * sizeof(double), cudaMemcpyHostToDevice, st));
  if (int rc = sfmm_pressure_tick_dev(t, t->util, t->victim)) return rc;
  SFKV_CUDA(cudaMemcpyAsync(out_victim, t->victim, t->NB * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfmm_tracker_entries(sfmm_tracker* t, uint8_t* present, uint8_t* preserved, int64_t* tokens,
                         double* ts, int32_t* in_flight) {
  if (!t) return fail(SFKV_EINVAL, "tracker_entries: null tracker");
  DeviceGuard g(t->device);
  cudaStream_t st = t->stream;
  const size_t E = (size_t)t->W * t->NB;
  if (present) SFKV_CUDA(cudaMemcpyAsync(present, t->present, E, cudaMemcpyDeviceToHost, st));
  if (preserved) SFKV_CUDA(cudaMemcpyAsync(preserved, t->preserved, E, cudaMemcpyDeviceToHost, st));
  if (tokens) SFKV_CUDA(cudaMemcpyAsync(tokens, t->tokens, E * 8, cudaMemcpyDeviceToHost, st));
  if (ts) SFKV_CUDA(cudaMemcpyAsync(ts, t->ts, E * 8, cudaMemcpyDeviceToHost, st));
  if (in_flight) SFKV_CUDA(cudaMemcpyAsync(in_flight, t->inflight, E * 4, cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfmm_tracker_shape(sfmm_tracker* t, int32_t* max_workflows, int32_t* n_backends, int32_t* max_stages) {
  if (!t) return fail(SFKV_EINVAL, "tracker_shape: null tracker");
  if (max_workflows) *max_workflows = t->W;
  if (n_backends) *n_backends = t->NB;
  if (max_stages) *max_stages = t->SW * 64;
  return 0;
}

}  // extern "C"

// §8f-1: batched MemoryManager::on_signal and pressure_tick over a GPU-resident WorkflowTracker.
//
// Replaces MemoryManager::{check_order, resolve, apply_and_record, update_tracker, on_signal,
// pressure_tick} (memory.cpp:256-387), the built-in policies (memory.cpp:116-148) and
// pressure_actions (memory.cpp:150-169). The reference processes one signal at a time through
// string-keyed std::maps (~5.9 us per signal). Here the tracker is a set of dense
// arrays in HBM over (workflow slot, backend index):
//   per workflow  completed u8, started/open stage sets u64 (started_ever_ / open_stages_),
//                 last stage {valid, backend, model, tokens}, per-workflow chain (len -1 =
//                 default), rank in workflow-id order (pressure tie-break)
//   per (wf, b)   entry {present, preserved, tokens, last_update_ts}, in-flight count
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
// pressure_tick: three order-independent min passes over the (wf, b) entries of the backends
// above tau_pressure (least ts, then least rank among ts ties, then the entry), then the victims'
// entries are erased. Integer/f64-compare work, latency-bound at these sizes; no tensor cores.
#include "pool.cuh"

struct sfmm_tracker {
  sfmm_config cfg;
  int32_t W = 0, NB = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint8_t* completed = nullptr;
  unsigned long long* started = nullptr;
  unsigned long long* open_ = nullptr;
  uint8_t* last_valid = nullptr;
  int32_t* last_b = nullptr;
  int32_t* last_model = nullptr;
  int64_t* last_tokens = nullptr;
  int32_t* chain_len = nullptr;
  uint8_t* chain = nullptr;
  uint8_t* present = nullptr;
  uint8_t* preserved = nullptr;
  int64_t* tokens = nullptr;
  double* ts = nullptr;
  int32_t* inflight = nullptr;
  uint32_t* rank = nullptr;
  int32_t* cnt = nullptr;  // per-workflow signal count of the current batch (kept zero between)
  unsigned long long* best_ts = nullptr;
  unsigned int* best_rank = nullptr;
  int32_t* victim = nullptr;
  double* util = nullptr;
  sfkv::Scratch scratch;
  sfkv::Scratch io;
};

namespace sfkv {

enum : uint8_t { K_START = 0, K_COMPLETE = 1, K_WF_COMPLETE = 2 };
enum : uint8_t { O_NONE = 0, O_PRESERVE = 1, O_FLUSH = 2 };
enum : uint8_t { P_PSI = 1, P_FAB = 2 };
enum : uint8_t { A_PRESERVE = 0, A_FLUSH = 1, A_NOOP = 2 };
enum : uint8_t { R_OVERRIDE = 0, R_PSI = 1, R_FAB = 2, R_PRESSURE = 3, R_EXHAUSTED = 4 };
constexpr int MAXCH = SFMM_MAX_CHAIN;

struct SigArgs {
  int64_t n;
  sfmm_signals s;
  sfmm_records r;
  int32_t* slot;
  int64_t* seg_off;
  int32_t* seg;
};

struct TrackerView {  // device pointers of a tracker, by value into kernels
  int32_t W, NB;
  int32_t def_len;
  uint8_t def_chain[MAXCH];
  int64_t tau;
  double tau_p;
  uint8_t* completed;
  unsigned long long* started;
  unsigned long long* open_;
  uint8_t* last_valid;
  int32_t* last_b;
  int32_t* last_model;
  int64_t* last_tokens;
  int32_t* chain_len;
  uint8_t* chain;
  uint8_t* present;
  uint8_t* preserved;
  int64_t* tokens;
  double* ts;
  int32_t* inflight;
  uint32_t* rank;
  int32_t* cnt;
  unsigned long long* best_ts;
  unsigned int* best_rank;
  int32_t* victim;
  const double* util;
};

static TrackerView view(sfmm_tracker* t) {
  TrackerView v;
  v.W = t->W;
  v.NB = t->NB;
  v.def_len = t->cfg.chain_len;
  for (int i = 0; i < MAXCH; ++i) v.def_chain[i] = t->cfg.chain[i];
  v.tau = t->cfg.tau;
  v.tau_p = t->cfg.tau_pressure;
  v.completed = t->completed;
  v.started = t->started;
  v.open_ = t->open_;
  v.last_valid = t->last_valid;
  v.last_b = t->last_b;
  v.last_model = t->last_model;
  v.last_tokens = t->last_tokens;
  v.chain_len = t->chain_len;
  v.chain = t->chain;
  v.present = t->present;
  v.preserved = t->preserved;
  v.tokens = t->tokens;
  v.ts = t->ts;
  v.inflight = t->inflight;
  v.rank = t->rank;
  v.cnt = t->cnt;
  v.best_ts = t->best_ts;
  v.best_rank = t->best_rank;
  v.victim = t->victim;
  v.util = t->util;
  return v;
}

__global__ void tracker_init_kernel(TrackerView v) {
  const int64_t E = (int64_t)v.W * v.NB;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (E > v.W ? E : v.W);
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < v.W) {
      v.completed[i] = 0;
      v.started[i] = 0;
      v.open_[i] = 0;
      v.last_valid[i] = 0;
      v.last_b[i] = -1;
      v.last_model[i] = -1;
      v.last_tokens[i] = 0;
      v.chain_len[i] = -1;
      v.rank[i] = (uint32_t)i;
      v.cnt[i] = 0;
    }
    if (i < E) {
      v.present[i] = 0;
      v.preserved[i] = 0;
      v.tokens[i] = 0;
      v.ts[i] = 0;
      v.inflight[i] = 0;
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

template <int NBC>
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
  // workflow state in registers for the whole segment
  uint8_t completed = v.completed[w];
  unsigned long long started = v.started[w], open = v.open_[w];
  uint8_t lvalid = v.last_valid[w];
  int32_t lb = v.last_b[w], lm = v.last_model[w];
  int64_t lt = v.last_tokens[w];
  int32_t clen = v.chain_len[w];
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
    const unsigned long long bit = 1ull << s;
    if (completed || (kind == K_START && (started & bit)) || (kind == K_COMPLETE && !(open & bit)) ||
        (wfc && open != 0)) {
      a.r.status[i] = SFMM_SIG_OUT_OF_ORDER;
      failed = true;
      continue;
    }
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
        if (ov == O_FLUSH) E.present(lb) = 0;  // applied (erases the entry)
      }
      na = 1;
    } else {
      const int32_t len = clen >= 0 ? clen : v.def_len;
      for (int32_t p = 0; p < len && na == 0; ++p) {
        const uint8_t pol = clen >= 0 ? v.chain[w * MAXCH + p] : v.def_chain[p];
        if (pol == P_PSI) {  // policy_preserve_small_increment (memory.cpp:116-125)
          if (kind == K_START && lvalid && lb == b && lm == m && T - lt < v.tau) {
            rk[0] = A_PRESERVE, rb[0] = b, rr[0] = R_PSI;
            na = 1;
          }
        } else {  // policy_flush_at_boundary (memory.cpp:127-148)
          if (wfc) {
            for (int32_t bb = 0; bb < NB; ++bb)
              if (E.present(bb) && E.preserved(bb)) {
                rk[na] = A_FLUSH, rb[na] = bb, rr[na] = R_FAB;
                E.present(bb) = 0;  // applied
                ++na;
              }
          } else if (kind == K_START && lvalid && (lb != b || lm != m) && E.present(lb) &&
                     E.preserved(lb)) {
            rk[0] = A_FLUSH, rb[0] = lb, rr[0] = R_FAB;
            E.present(lb) = 0;  // applied
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
      started |= bit;
      open |= bit;
      E.inflight(b) += 1;
    } else if (kind == K_COMPLETE) {
      open &= ~bit;
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
      lvalid = 1, lb = b, lm = m, lt = T;
    } else {
      completed = 1;
      for (int32_t bb = 0; bb < NB; ++bb) {
        E.present(bb) = 0;
        E.inflight(bb) = 0;
      }
      lvalid = 0, started = 0, open = 0, clen = -1;
    }
    a.r.status[i] = SFMM_SIG_OK;
  }
  E.store(v, e0, NB);
  v.completed[w] = completed;
  v.started[w] = started;
  v.open_[w] = open;
  v.last_valid[w] = lvalid;
  v.last_b[w] = lb;
  v.last_model[w] = lm;
  v.last_tokens[w] = lt;
  v.chain_len[w] = clen;
}

// ---- pressure tick ---------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ts_key(double t) {
  if (t == 0.0) t = 0.0;  // -0.0 == 0.0 in the reference's comparison
  const unsigned long long b = (unsigned long long)__double_as_longlong(t);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ bool idle_preserved(const TrackerView& v, int64_t e) {
  return v.present[e] && v.preserved[e] && v.inflight[e] <= 0 && v.util[e % v.NB] > v.tau_p;
}
__global__ void tp_init(TrackerView v) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < v.NB) {
    v.best_ts[b] = ~0ull;
    v.best_rank[b] = ~0u;
    v.victim[b] = -1;
  }
}
__global__ void tp_pass1(TrackerView v) {
  pdl_enter();
  const int64_t E = (int64_t)v.W * v.NB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    if (idle_preserved(v, e)) atomicMin(&v.best_ts[e % v.NB], ts_key(v.ts[e]));
}
__global__ void tp_pass2(TrackerView v) {
  pdl_enter();
  const int64_t E = (int64_t)v.W * v.NB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    if (idle_preserved(v, e) && ts_key(v.ts[e]) == v.best_ts[e % v.NB])
      atomicMin(&v.best_rank[e % v.NB], v.rank[e / v.NB]);
}
__global__ void tp_pass3(TrackerView v) {
  pdl_enter();
  const int64_t E = (int64_t)v.W * v.NB;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(e % v.NB);
    if (idle_preserved(v, e) && ts_key(v.ts[e]) == v.best_ts[b] && v.rank[e / v.NB] == v.best_rank[b])
      atomicMin(reinterpret_cast<unsigned int*>(&v.victim[b]), (unsigned int)(e / v.NB));
  }
}
__global__ void tp_apply(TrackerView v) {  // victim starts at -1 (all ones) for atomicMin
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= v.NB) return;
  if (v.best_ts[b] == ~0ull) {
    v.victim[b] = -1;
    return;
  }
  v.present[(int64_t)v.victim[b] * v.NB + b] = 0;  // mark_flushed
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
  const TrackerView v = view(t);
  const int sms = sm_count_t();
  SFKV_CUDA(launch_pdl(sig_count_kernel, dim3(grid_for(n, 256, sms * 8)), dim3(256), st, a, v));
  SFKV_LAUNCH_CHECK("sig_count_kernel");
  if (int rc = exclusive_scan(CntOf{t->cnt}, t->W, a.seg_off, reinterpret_cast<int64_t*>(base + o_tmp), st))
    return rc;
  SFKV_CUDA(launch_pdl(sig_scatter_kernel, dim3(grid_for(n, 256, sms * 8)), dim3(256), st, a));
  if (t->NB <= 8)  // spread over every SM
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<8>, dim3((unsigned)((t->W + 31) / 32)), dim3(32), st, a, v));
  else
    SFKV_CUDA(launch_pdl(sig_resolve_kernel<0>, dim3((unsigned)((t->W + 31) / 32)), dim3(32), st, a, v));
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

static void tracker_free(sfmm_tracker* t) {
  cudaFree(t->completed);
  cudaFree(t->started);
  cudaFree(t->open_);
  cudaFree(t->last_valid);
  cudaFree(t->last_b);
  cudaFree(t->last_model);
  cudaFree(t->last_tokens);
  cudaFree(t->chain_len);
  cudaFree(t->chain);
  cudaFree(t->present);
  cudaFree(t->preserved);
  cudaFree(t->tokens);
  cudaFree(t->ts);
  cudaFree(t->inflight);
  cudaFree(t->rank);
  cudaFree(t->cnt);
  cudaFree(t->best_ts);
  cudaFree(t->best_rank);
  cudaFree(t->victim);
  cudaFree(t->util);
  t->scratch.release();
  t->io.release();
  if (t->own_stream && t->stream) cudaStreamDestroy(t->stream);
}

extern "C" {

int sfmm_tracker_create(const sfmm_config* cfg, sfmm_tracker** out) {
  if (!cfg || !out) return fail(SFKV_EINVAL, "tracker_create: null argument");
  if (cfg->max_workflows <= 0 || cfg->n_backends <= 0 || cfg->chain_len < 0 ||
      cfg->chain_len > SFMM_MAX_CHAIN || cfg->tau <= 0 || !(cfg->tau_pressure > 0) ||
      cfg->tau_pressure > 1)  // memory.cpp:240-243
    return fail(SFKV_EINVAL, "tracker_create: invalid configuration");
  for (int i = 0; i < cfg->chain_len; ++i)
    if (cfg->chain[i] != SFMM_POLICY_PRESERVE_SMALL_INCREMENT && cfg->chain[i] != SFMM_POLICY_FLUSH_AT_BOUNDARY)
      return fail(SFKV_EINVAL, "tracker_create: unknown memory policy");  // memory.cpp:182
  if (int rc = check_device(cfg->device)) return rc;
  DeviceGuard g(cfg->device);
  auto* t = new sfmm_tracker;
  t->cfg = *cfg;
  t->W = cfg->max_workflows;
  t->NB = cfg->n_backends;
  const size_t W = t->W, E = W * t->NB;
  int rc = 0;
  if ((rc = talloc(&t->completed, W)) || (rc = talloc(&t->started, W)) || (rc = talloc(&t->open_, W)) ||
      (rc = talloc(&t->last_valid, W)) || (rc = talloc(&t->last_b, W)) || (rc = talloc(&t->last_model, W)) ||
      (rc = talloc(&t->last_tokens, W)) || (rc = talloc(&t->chain_len, W)) ||
      (rc = talloc(&t->chain, W * SFMM_MAX_CHAIN)) || (rc = talloc(&t->present, E)) ||
      (rc = talloc(&t->preserved, E)) || (rc = talloc(&t->tokens, E)) || (rc = talloc(&t->ts, E)) ||
      (rc = talloc(&t->inflight, E)) || (rc = talloc(&t->rank, W)) || (rc = talloc(&t->cnt, W)) ||
      (rc = talloc(&t->best_ts, (size_t)t->NB)) || (rc = talloc(&t->best_rank, (size_t)t->NB)) ||
      (rc = talloc(&t->victim, (size_t)t->NB)) || (rc = talloc(&t->util, (size_t)t->NB))) {
    tracker_free(t);
    delete t;
    return rc;
  }
  cudaError_t e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    tracker_free(t);
    delete t;
    return cuda_fail(e, "tracker stream");
  }
  t->own_stream = true;
  const int64_t span = (int64_t)(E > W ? E : W);
  tracker_init_kernel<<<grid_for(span, 256, 4096), 256, 0, t->stream>>>(view(t));
  e = cudaStreamSynchronize(t->stream);
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
  DeviceGuard g(t->cfg.device);
  cudaStreamSynchronize(t->stream);
  tracker_free(t);
  delete t;
  return 0;
}

int sfmm_tracker_set_stream(sfmm_tracker* t, void* stream) {
  if (!t) return fail(SFKV_EINVAL, "tracker_set_stream: null tracker");
  DeviceGuard g(t->cfg.device);
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  if (t->own_stream) cudaStreamDestroy(t->stream);
  t->stream = static_cast<cudaStream_t>(stream);  // NULL: the legacy default stream (as pools)
  t->own_stream = false;
  return 0;
}

int sfmm_tracker_reset(sfmm_tracker* t) {
  if (!t) return fail(SFKV_EINVAL, "tracker_reset: null tracker");
  DeviceGuard g(t->cfg.device);
  const int64_t E = (int64_t)t->W * t->NB;
  tracker_init_kernel<<<grid_for(E > t->W ? E : t->W, 256, 4096), 256, 0, t->stream>>>(view(t));
  SFKV_LAUNCH_CHECK("tracker_init_kernel");
  return 0;
}

int sfmm_tracker_sync(sfmm_tracker* t) {
  if (!t) return fail(SFKV_EINVAL, "tracker_sync: null tracker");
  DeviceGuard g(t->cfg.device);
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_set_workflow_chain(sfmm_tracker* t, int32_t wf, int32_t len, const uint8_t* policies) {
  if (!t || wf < 0 || wf >= t->W || len < 0 || len > SFMM_MAX_CHAIN || (len && !policies))
    return fail(SFKV_EINVAL, "set_workflow_chain: bad argument");
  if (len == 0) return 0;  // memory.cpp:248
  for (int i = 0; i < len; ++i)
    if (policies[i] != SFMM_POLICY_PRESERVE_SMALL_INCREMENT && policies[i] != SFMM_POLICY_FLUSH_AT_BOUNDARY)
      return fail(SFKV_EINVAL, "set_workflow_chain: unknown memory policy");
  DeviceGuard g(t->cfg.device);
  SFKV_CUDA(cudaMemcpyAsync(t->chain + (size_t)wf * SFMM_MAX_CHAIN, policies, len, cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaMemcpyAsync(t->chain_len + wf, &len, sizeof(int32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_set_workflow_ranks(sfmm_tracker* t, int64_t n, const uint32_t* rank) {
  if (!t || n < 0 || n > t->W || (n && !rank)) return fail(SFKV_EINVAL, "set_workflow_ranks: bad argument");
  DeviceGuard g(t->cfg.device);
  if (n) SFKV_CUDA(cudaMemcpyAsync(t->rank, rank, n * sizeof(uint32_t), cudaMemcpyHostToDevice, t->stream));
  SFKV_CUDA(cudaStreamSynchronize(t->stream));
  return 0;
}

int sfmm_on_signal_batch_dev(sfmm_tracker* t, int64_t n, const sfmm_signals* sig, const sfmm_records* out) {
  if (!t || !sig || !out || n < 0) return fail(SFKV_EINVAL, "on_signal_batch_dev: bad argument");
  if (n > INT32_MAX) return fail(SFKV_EINVAL, "on_signal_batch_dev: batch too large");
  if (n > 0 && (!sig->kind || !sig->wf || !sig->stage || !sig->backend || !sig->model || !sig->tokens ||
                !sig->ts || !out->count || !out->status || !out->kind || !out->backend || !out->reason))
    return fail(SFKV_EINVAL, "on_signal_batch_dev: null array (only override_ may be null)");
  DeviceGuard g(t->cfg.device);
  return on_signals_dev(t, n, *sig, *out);
}

int sfmm_on_signal_batch(sfmm_tracker* t, int64_t n, const sfmm_signals* sig, const sfmm_records* out) {
  if (!t || !sig || !out || n < 0) return fail(SFKV_EINVAL, "on_signal_batch: bad argument");
  if (n == 0) return 0;
  if (n > INT32_MAX) return fail(SFKV_EINVAL, "on_signal_batch: batch too large");
  if (!sig->kind || !sig->wf || !sig->ts || !out->count || !out->status || !out->kind ||
      !out->backend || !out->reason)
    return fail(SFKV_EINVAL, "on_signal_batch: null array");
  for (int64_t i = 0; i < n; ++i) {  // host-side validation of the dense ids
    const bool wfc = sig->kind[i] == K_WF_COMPLETE;
    if (sig->kind[i] > K_WF_COMPLETE || sig->wf[i] < 0 || sig->wf[i] >= t->W ||
        (!wfc && (!sig->stage || !sig->backend || !sig->model || !sig->tokens || sig->stage[i] < 0 ||
                  sig->stage[i] >= SFMM_MAX_STAGES || sig->backend[i] < 0 || sig->backend[i] >= t->NB)))
      return fail(SFKV_EINVAL, "on_signal_batch: signal field out of range");
  }
  DeviceGuard g(t->cfg.device);
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

int sfmm_pressure_tick(sfmm_tracker* t, const double* util, int32_t* out_victim) {
  if (!t || !util || !out_victim) return fail(SFKV_EINVAL, "pressure_tick: null argument");
  DeviceGuard g(t->cfg.device);
  cudaStream_t st = t->stream;
  SFKV_CUDA(cudaMemcpyAsync(t->util, util, t->NB * sizeof(double), cudaMemcpyHostToDevice, st));
  const TrackerView v = view(t);
  const int bg = (t->NB + 255) / 256;
  const int g2 = grid_for((int64_t)t->W * t->NB, 256, sm_count_t() * 8);
  SFKV_CUDA(launch_pdl(tp_init, dim3(bg), dim3(256), st, v));
  SFKV_CUDA(launch_pdl(tp_pass1, dim3(g2), dim3(256), st, v));
  SFKV_CUDA(launch_pdl(tp_pass2, dim3(g2), dim3(256), st, v));
  SFKV_CUDA(launch_pdl(tp_pass3, dim3(g2), dim3(256), st, v));
  SFKV_CUDA(launch_pdl(tp_apply, dim3(bg), dim3(256), st, v));
  SFKV_LAUNCH_CHECK("pressure tick kernels");
  SFKV_CUDA(cudaMemcpyAsync(out_victim, t->victim, t->NB * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SFKV_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int sfmm_tracker_entries(sfmm_tracker* t, uint8_t* present, uint8_t* preserved, int64_t* tokens,
                         double* ts, int32_t* in_flight) {
  if (!t) return fail(SFKV_EINVAL, "tracker_entries: null tracker");
  DeviceGuard g(t->cfg.device);
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

}  // extern "C"

// libsfref.so — a C shim over the UNMODIFIED reference functions on the hot path
// (oracle test infrastructure and the CPU baseline arm of bench.py; never the product).
//
// Every entry point calls straight into the reference's own code compiled from /root/reference:
//   sfref_pin / sfref_prefix_match*  -> SimulatedBackend::complete / prefix_match
//                                       (simulated_backend.cpp:35-39, 72-151, 153-162)
//   sfref_flush / sfref_preserve      -> SimulatedBackend::flush / preserve (169-184, 190-193)
//   sfref_pressure_actions            -> pressure_actions (memory.cpp:150-169) over a
//                                       WorkflowTracker built with its public mutators
//   sfref_map_threshold               -> map_threshold (mapper.cpp:19-31)
//   sfref_reroute                     -> reroute_on_overload (orchestrator.cpp:78-87)
//   sfref_mm_*                        -> MemoryManager::{on_signal, pressure_tick,
//                                       set_workflow_chain, action_log} (memory.cpp:246-401),
//                                       no backends attached (every action "applies"), or a
//                                       registry of flaky test backends (sfref_mm_create_flaky)
// Token ids are rendered to whitespace tokens "t<id>", the same text the reference tokenizes.
#include <pthread.h>
#include <sched.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <sstream>
#include <thread>

#include "stageflow/backend.hpp"
#include "stageflow/memory.hpp"
#include "stageflow/metrics.hpp"
#include "stageflow/mapper.hpp"
#include "stageflow/orchestrator.hpp"
#include "stageflow/simulated_backend.hpp"

using namespace stageflow;

namespace {

struct RefPool {
  EventLoop loop{ClockMode::Virtual};
  std::unique_ptr<SimulatedBackend> backend;
};

struct RefBatch {
  std::vector<std::string> wf;
  std::vector<std::vector<std::string>> tokens;
};

std::string render(const std::uint32_t* tok, long long n) {
  std::string s;
  s.reserve(static_cast<std::size_t>(n) * 8);
  for (long long i = 0; i < n; ++i) {
    if (i) s += ' ';
    s += 't';
    s += std::to_string(tok[i]);
  }
  return s;
}

// A test backend for the memory manager's apply_action (memory.cpp:185-220): only flush and
// preserve are exercised; flush throws per its mode (see sfref_mm_create_flaky).
class FlakyBackend : public Backend {
 public:
  FlakyBackend(std::string ref, int mode) : mode_(mode) {
    desc_.ref = std::move(ref);
    desc_.kind = BackendKind::Simulated;
  }
  const BackendDescriptor& descriptor() const override { return desc_; }
  bool has_capacity() const override { return true; }
  void complete(CompletionRequest, CompletionCallback) override { throw BackendError("not a serving backend"); }
  long long flush(const FlushScope&) override {
    ++attempts;
    if (mode_ == 2 || (mode_ == 1 && attempts % 2 == 1)) throw BackendError("flush failed");
    return 0;
  }
  double cache_utilization() const override { return 0; }
  bool preserve(const std::string&) override { return true; }
  const BackendStats& stats() const override { return stats_; }
  long long attempts = 0;

 private:
  int mode_;
  BackendDescriptor desc_;
  BackendStats stats_;
};

struct RefMM {
  BackendRegistry reg;
  std::unique_ptr<MemoryManager> mm;
};
MemoryManager* MM(void* h) { return static_cast<RefMM*>(h)->mm.get(); }

// A persistent pool of worker threads, each pinned to one host core, for the CPU baseline: a
// timed step hands worker i its job and waits for all of them, so no thread is created inside a
// timed region (bench.py --impl reference).
struct Workers {
  std::vector<std::thread> th;
  std::mutex m;
  std::condition_variable go, done;
  std::function<void(int)> job;
  long long gen = 0;
  int pending = 0;
  bool stop = false;

  Workers(int n, const int* cpus) {
    for (int i = 0; i < n; ++i) {
      th.emplace_back([this, i] { loop(i); });
      if (cpus && cpus[i] >= 0) {
        cpu_set_t set;
        CPU_ZERO(&set);
        CPU_SET(cpus[i], &set);
        pthread_setaffinity_np(th.back().native_handle(), sizeof(set), &set);
      }
    }
  }
  ~Workers() {
    {
      std::lock_guard<std::mutex> g(m);
      stop = true;
    }
    go.notify_all();
    for (auto& t : th) t.join();
  }
  void loop(int i) {
    long long seen = 0;
    for (;;) {
      std::function<void(int)> f;
      {
        std::unique_lock<std::mutex> g(m);
        go.wait(g, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        f = job;
      }
      f(i);
      {
        std::lock_guard<std::mutex> g(m);
        if (--pending == 0) done.notify_all();
      }
    }
  }
  void run(std::function<void(int)> f) {
    std::unique_lock<std::mutex> g(m);
    job = std::move(f);
    pending = static_cast<int>(th.size());
    ++gen;
    go.notify_all();
    done.wait(g, [&] { return pending == 0; });
  }
};

}  // namespace

extern "C" {

void* sfref_pool_create(long long capacity_tokens) {
  auto* p = new RefPool;
  SimulatedBackendConfig cfg;
  cfg.cache_capacity_tokens = capacity_tokens;
  cfg.max_concurrency = 1;
  cfg.output = OutputRule::constant(0);
  BackendDescriptor d;
  d.ref = "ref";
  d.model = "ref-model";
  p->backend = std::make_unique<SimulatedBackend>(p->loop, d, cfg);
  return p;
}

void sfref_pool_destroy(void* h) { delete static_cast<RefPool*>(h); }

// One stage request through the reference backend (tokenize -> prefix_match -> pin_prompt).
// Returns M (cached prefix tokens); *accepted reports whether the pin was admitted.
long long sfref_complete(void* h, const char* wf, const std::uint32_t* tok, long long n,
                         int* accepted) {
  auto* p = static_cast<RefPool*>(h);
  CompletionRequest req;
  req.messages = make_user_context(render(tok, n));
  req.metadata.workflow_id = wf;
  auto before = p->backend->capacity_rejections();
  auto resp = complete_blocking(*p->backend, p->loop, std::move(req));
  if (accepted) *accepted = p->backend->capacity_rejections() == before ? 1 : 0;
  return resp.usage.cached_prefix_tokens;
}

long long sfref_flush(void* h, const char* wf, int all) {
  auto* p = static_cast<RefPool*>(h);
  return p->backend->flush(all ? FlushScope::everything() : FlushScope::workflow(wf));
}

int sfref_preserve(void* h, const char* wf) {
  return static_cast<RefPool*>(h)->backend->preserve(wf) ? 1 : 0;
}

long long sfref_pinned_token_count(void* h, const char* wf) {
  return static_cast<RefPool*>(h)->backend->pinned_token_count(wf);
}
long long sfref_occupancy_tokens(void* h) {
  return static_cast<RefPool*>(h)->backend->occupancy_tokens();
}
unsigned long long sfref_capacity_rejections(void* h) {
  return static_cast<RefPool*>(h)->backend->capacity_rejections();
}
double sfref_cache_utilization(void* h) {
  return static_cast<RefPool*>(h)->backend->cache_utilization();
}

// A batch of lookups, rendered to token strings ONCE (outside any timed region): the reference's
// prefix_match consumes std::string tokens (simulated_backend.hpp:73-74).
void* sfref_batch_create(long long n, const char* const* wf, const long long* tok_off,
                         const std::uint32_t* tok) {
  auto* b = new RefBatch;
  b->wf.reserve(static_cast<std::size_t>(n));
  b->tokens.resize(static_cast<std::size_t>(n));
  for (long long r = 0; r < n; ++r) {
    b->wf.emplace_back(wf[r]);
    auto& v = b->tokens[static_cast<std::size_t>(r)];
    v.reserve(static_cast<std::size_t>(tok_off[r + 1] - tok_off[r]));
    for (long long i = tok_off[r]; i < tok_off[r + 1]; ++i) v.push_back("t" + std::to_string(tok[i]));
  }
  return b;
}
void sfref_batch_destroy(void* b) { delete static_cast<RefBatch*>(b); }

// The reference lookup itself: M[r] = SimulatedBackend::prefix_match(wf[r], tokens[r]).
void sfref_prefix_match_batch(void* h, void* batch, long long* out_M) {
  auto* p = static_cast<RefPool*>(h);
  auto* b = static_cast<RefBatch*>(batch);
  for (std::size_t r = 0; r < b->wf.size(); ++r) {
    out_M[r] = p->backend->prefix_match(b->wf[r], std::span<const std::string>(b->tokens[r]));
  }
}

// The CPU baseline's worker pool: n threads, thread i pinned to cpus[i] (cpus nullable / -1 =
// unpinned). Created once, outside every timed region.
void* sfref_workers_create(int n, const int* cpus) { return new Workers(n, cpus); }
void sfref_workers_destroy(void* w) { delete static_cast<Workers*>(w); }

// One step of the reference lookup on every shard at once: worker i runs
// sfref_prefix_match_batch(pools[i], batches[i], outs[i]) (a shard = one SimulatedBackend
// holding its workflows' pins). Returns when every shard is done.
void sfref_prefix_match_parallel(void* w, void* const* pools, void* const* batches,
                                 long long* const* outs) {
  static_cast<Workers*>(w)->run([&](int i) { sfref_prefix_match_batch(pools[i], batches[i], outs[i]); });
}

// Build shard i's backend and batch on worker i (setup, untimed): pools[i] holds the pins
// (pin_off / pin_tok CSR over the shard's workflows), batches[i] the requests.
struct ShardSpec {
  long long n;
  const char* const* wf;
  const long long* pin_off;
  const std::uint32_t* pin_tok;
  const long long* req_off;
  const std::uint32_t* req_tok;
};
void sfref_build_shards_parallel(void* w, const ShardSpec* spec, void** pools, void** batches) {
  static_cast<Workers*>(w)->run([&](int i) {
    const ShardSpec& s = spec[i];
    pools[i] = sfref_pool_create(1LL << 40);
    int acc = 0;
    for (long long r = 0; r < s.n; ++r)
      sfref_complete(pools[i], s.wf[r], s.pin_tok + s.pin_off[r], s.pin_off[r + 1] - s.pin_off[r], &acc);
    batches[i] = sfref_batch_create(s.n, s.wf, s.req_off, s.req_tok);
  });
}

// pressure_actions over n tracker entries. Entry i: (wf[i], backend_refs[backend[i]], ts[i],
// in_flight[i], preserved[i], tokens[i]). out_victim[bi] = entry index flushed on backend bi or -1.
int sfref_pressure_actions(long long n, const char* const* wf, const int* backend, const double* ts,
                           const int* in_flight, const unsigned char* preserved,
                           const long long* tokens, int n_backends,
                           const char* const* backend_refs, const double* util, double tau,
                           long long* out_victim) {
  WorkflowTracker tracker;
  std::map<std::pair<std::string, std::string>, long long> index;
  for (long long i = 0; i < n; ++i) {
    CacheEntry e;
    e.workflow_id = wf[i];
    e.backend_ref = backend_refs[backend[i]];
    e.token_count = tokens ? tokens[i] : 1;
    e.preserved = preserved[i] != 0;
    e.last_update_ts = ts[i];
    index[{e.workflow_id, e.backend_ref}] = i;
    tracker.upsert_entry(e);
    if (in_flight[i] > 0) tracker.adjust_in_flight(e.backend_ref, e.workflow_id, in_flight[i]);
  }
  std::map<std::string, double> u;
  for (int b = 0; b < n_backends; ++b) u[backend_refs[b]] = util[b];
  for (int b = 0; b < n_backends; ++b) out_victim[b] = -1;
  int count = 0;
  for (const auto& a : pressure_actions(tracker, u, tau)) {
    for (int b = 0; b < n_backends; ++b) {
      if (a.backend_ref == backend_refs[b]) out_victim[b] = index.at({a.workflow_id, a.backend_ref});
    }
    ++count;
  }
  return count;
}

// The CPU baseline of the pressure step: the same tracker as sfref_pressure_actions, built once,
// then `iters` calls of the reference's pressure_actions timed with steady_clock (the calling
// thread: pin it). Returns the mean nanoseconds per call; *out_count = actions of the last call.
double sfref_pressure_bench(long long n, const char* const* wf, const int* backend, const double* ts,
                            const int* in_flight, const unsigned char* preserved, int n_backends,
                            const char* const* backend_refs, const double* util, double tau, int iters,
                            int* out_count) {
  WorkflowTracker tracker;
  for (long long i = 0; i < n; ++i) {
    CacheEntry e;
    e.workflow_id = wf[i];
    e.backend_ref = backend_refs[backend[i]];
    e.token_count = 1;
    e.preserved = preserved[i] != 0;
    e.last_update_ts = ts[i];
    tracker.upsert_entry(e);
    if (in_flight[i] > 0) tracker.adjust_in_flight(e.backend_ref, e.workflow_id, in_flight[i]);
  }
  std::map<std::string, double> u;
  for (int b = 0; b < n_backends; ++b) u[backend_refs[b]] = util[b];
  int count = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) count = static_cast<int>(pressure_actions(tracker, u, tau).size());
  const auto t1 = std::chrono::steady_clock::now();
  *out_count = count;
  return std::chrono::duration<double, std::nano>(t1 - t0).count() / iters;
}

// SimulatedBackend::flush(FlushScope::workflow(wf[i])) for i < n in order (one C++ loop); returns
// the tokens freed.
long long sfref_flush_batch(void* h, long long n, const char* const* wf) {
  auto* p = static_cast<RefPool*>(h);
  long long freed = 0;
  for (long long i = 0; i < n; ++i) freed += p->backend->flush(FlushScope::workflow(wf[i]));
  return freed;
}

// map_threshold with a score function returning the given score: 1 = light, 0 = heavy.
int sfref_map_threshold(double score, double threshold) {
  auto [ref, s] = map_threshold(Context{}, [score](const Context&) { return score; }, threshold,
                                "light", "heavy");
  (void)s;
  return ref == "light" ? 1 : 0;
}

// reroute_on_overload over candidates 0..n-1 with candidate 0 the primary.
int sfref_reroute(int n, const unsigned long long* depth, unsigned long long limit) {
  std::vector<std::string> names;
  for (int i = 0; i < n; ++i) names.push_back(std::to_string(i));
  auto pick = reroute_on_overload(
      names[0], std::span<const std::string>(names.data() + 1, names.size() - 1),
      [&](const std::string& s) { return static_cast<std::size_t>(depth[std::stoi(s)]); },
      static_cast<std::size_t>(limit));
  return std::stoi(pick);
}

// ---- latency model and metrics --------------------------------------------------------------
// n requests submitted at virtual time 0 to one SimulatedBackend (max_concurrency slots, constant
// output of out_tokens): the reference's own CompletionResponse timing and usage per request
// (simulated_backend.cpp:72-133). wf[i] = "" for unpinned (routing-style) calls.
void sfref_sim_timing(double prefill, double decode, double overhead, int max_conc, long long out_tokens, int n,
                      const char* const* wf, const char* const* text, double* queue, double* ttft, double* total,
                      long long* P, long long* M, long long* O) {
  EventLoop loop(ClockMode::Virtual);
  SimulatedBackendConfig cfg;
  cfg.prefill_ms_per_token = prefill;
  cfg.decode_ms_per_token = decode;
  cfg.fixed_overhead_ms = overhead;
  cfg.max_concurrency = max_conc;
  cfg.cache_capacity_tokens = 1LL << 40;
  cfg.output = OutputRule::constant(out_tokens);
  BackendDescriptor d;
  d.ref = "ref";
  d.model = "ref-model";
  SimulatedBackend be(loop, d, cfg);
  for (int i = 0; i < n; ++i) {
    CompletionRequest req;
    req.model = "ref-model";
    Message m;
    m.content = text[i];
    req.messages.push_back(std::move(m));
    req.metadata.workflow_id = wf[i];
    req.metadata.stage_id = "s";
    be.complete(std::move(req), [=](CompletionResponse r, std::exception_ptr) {
      queue[i] = r.timing.queue_ms;
      ttft[i] = r.timing.ttft_ms;
      total[i] = r.timing.total_ms;
      P[i] = r.usage.prompt_tokens;
      M[i] = r.usage.cached_prefix_tokens;
      O[i] = r.usage.completion_tokens;
    });
  }
  loop.run_until_idle();
}

// percentile_nearest_rank over the (already sorted) samples (metrics.cpp:22-28).
double sfref_percentile(long long n, const double* sorted, int pct) {
  return percentile_nearest_rank(std::vector<double>(sorted, sorted + n), pct);
}

// ---- tokenizer --------------------------------------------------------------------------
// context_token_sequence (backend.cpp:83-91) over n messages (content only). Writes the tokens
// concatenated into out (cap bytes) with their lengths into out_len (cap_tokens); returns the
// token count (or -1 when a buffer is too small).
long long sfref_context_tokens(int n, const char* const* msg, const long long* msg_len, char* out,
                               long long cap, long long* out_len, long long cap_tokens) {
  Context ctx;
  for (int i = 0; i < n; ++i) {
    Message m;
    m.content.assign(msg[i], static_cast<std::size_t>(msg_len[i]));
    ctx.push_back(std::move(m));
  }
  auto toks = context_token_sequence(ctx);
  if (static_cast<long long>(toks.size()) > cap_tokens) return -1;
  long long o = 0;
  for (std::size_t i = 0; i < toks.size(); ++i) {
    if (o + static_cast<long long>(toks[i].size()) > cap) return -1;
    std::memcpy(out + o, toks[i].data(), toks[i].size());
    o += static_cast<long long>(toks[i].size());
    out_len[i] = static_cast<long long>(toks[i].size());
  }
  return static_cast<long long>(toks.size());
}

// ---- MemoryManager ------------------------------------------------------------------------
void* sfref_mm_create(long long tau, double tau_pressure, int chain_len, const char* const* chain) {
  MemoryConfig cfg;
  cfg.tau = tau;
  cfg.tau_pressure = tau_pressure;
  cfg.policy_chain.assign(chain, chain + chain_len);
  auto* r = new RefMM;
  r->mm = std::make_unique<MemoryManager>(cfg);
  return r;
}
// The same with a BackendRegistry of test backends whose flush fails: mode 0 never, 1 on the
// first attempt of every flush action (the retry succeeds), 2 always (apply_action gives up after
// the retry, memory.cpp:189-203, and the tracker entry is only unpreserved, memory.cpp:322-324).
void* sfref_mm_create_flaky(long long tau, double tau_pressure, int chain_len, const char* const* chain,
                            int n_backends, const char* const* refs, const int* modes) {
  MemoryConfig cfg;
  cfg.tau = tau;
  cfg.tau_pressure = tau_pressure;
  cfg.policy_chain.assign(chain, chain + chain_len);
  auto* r = new RefMM;
  for (int i = 0; i < n_backends; ++i) r->reg.add(std::make_shared<FlakyBackend>(refs[i], modes[i]));
  r->mm = std::make_unique<MemoryManager>(cfg, &r->reg);
  return r;
}
void sfref_mm_destroy(void* h) { delete static_cast<RefMM*>(h); }

// Tracker entry of (wf, backend): 0 absent, 1 present and preserved, 2 present unpreserved.
int sfref_mm_entry(void* h, const char* wf, const char* backend) {
  const CacheEntry* e = MM(h)->tracker().entry(wf, backend);
  return e ? (e->preserved ? 1 : 2) : 0;
}
// Flush calls a flaky backend received (attempts, including failed ones).
long long sfref_mm_flush_attempts(void* h, const char* backend) {
  auto& r = static_cast<RefMM*>(h)->reg;
  return static_cast<FlakyBackend&>(r.at(backend)).attempts;
}

void sfref_mm_set_chain(void* h, const char* wf, int len, const char* const* names) {
  std::vector<std::string> v(names, names + len);
  MM(h)->set_workflow_chain(wf, v);
}

// kind 0/1/2 = StageStart/StageComplete/WorkflowComplete; override 0/1/2 = None/Preserve/Flush.
// Returns 0, 1 (OutOfOrderSignalError) or 3 (logic_error: in-flight went negative).
int sfref_mm_on_signal(void* h, int kind, const char* wf, const char* stage, const char* backend,
                       const char* model, long long tokens, double ts, int override_) {
  LifecycleSignal sig;
  sig.kind = static_cast<LifecycleSignal::Kind>(kind);
  sig.workflow_id = wf;
  if (kind != 2) {
    sig.stage_id = stage;
    sig.backend_ref = backend;
    sig.model = model;
    sig.context_tokens = tokens;
  }
  sig.ts = ts;
  sig.cache_override = static_cast<CachePolicyOverride>(override_);
  try {
    MM(h)->on_signal(sig);
  } catch (const OutOfOrderSignalError&) {
    return 1;
  } catch (const std::logic_error& e) {
    if (std::getenv("SFREF_DEBUG")) std::fprintf(stderr, "sfref_mm_on_signal: %s\n", e.what());
    return 3;
  }
  return 0;
}

// n signals through MemoryManager::on_signal in order (the CPU baseline: the loop stays in C++).
// Returns the number of signals the reference rejected.
long long sfref_mm_on_signal_batch(void* h, long long n, const int* kind, const char* const* wf,
                                   const char* const* stage, const char* const* backend,
                                   const char* const* model, const long long* tokens,
                                   const double* ts, const int* override_) {
  long long bad = 0;
  for (long long i = 0; i < n; ++i)
    bad += sfref_mm_on_signal(h, kind[i], wf[i], stage[i], backend[i], model[i], tokens[i], ts[i],
                              override_ ? override_[i] : 0) != 0;
  return bad;
}

int sfref_mm_pressure_tick(void* h, int n, const char* const* refs, const double* util, double now) {
  std::map<std::string, double> u;
  for (int i = 0; i < n; ++i) u[refs[i]] = util[i];
  return static_cast<int>(MM(h)->pressure_tick(u, now).size());
}

// MemoryManager::export_action_log (memory.cpp:389-401) into buf (cap bytes); returns its length.
long long sfref_mm_export(void* h, char* buf, long long cap) {
  std::ostringstream os;
  MM(h)->export_action_log(os);
  const std::string s = os.str();
  if (static_cast<long long>(s.size()) <= cap) std::memcpy(buf, s.data(), s.size());
  return static_cast<long long>(s.size());
}

long long sfref_mm_log_size(void* h) {
  return static_cast<long long>(MM(h)->action_log().size());
}

// Record i of the action log: kind 0/1/2 = Preserve/Flush/NoOp; strings copied (NUL-terminated,
// truncated to cap bytes).
void sfref_mm_log_get(void* h, long long i, int* kind, char* wf, char* backend, char* reason,
                      char* trigger, int cap, double* ts) {
  const auto& r = MM(h)->action_log().at(static_cast<std::size_t>(i));
  *kind = static_cast<int>(r.action.kind);
  *ts = r.ts;
  auto put = [cap](char* dst, const std::string& s) {
    std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
    std::memcpy(dst, s.data(), n);
    dst[n] = 0;
  };
  put(wf, r.action.workflow_id);
  put(backend, r.action.backend_ref);
  put(reason, r.action.reason);
  put(trigger, r.trigger);
}

}  // extern "C"

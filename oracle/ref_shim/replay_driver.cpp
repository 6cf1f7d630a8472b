// sf_ref_replay — golden-stream capture from the UNMODIFIED reference (oracle test infrastructure).
//
// Replays a (trace, config) pair through the reference's own public API exactly the way
// stageflow's run_benchmark does (/root/reference/proj/src/harness.cpp:8-116), except that every
// SimulatedBackend is wrapped in a RecordingBackend that forwards each call unchanged and logs the
// pin-cache operations the hot path performs, in event order:
//
//   match    SimulatedBackend::start -> prefix_match   (simulated_backend.cpp:72-79, 153-162)
//   pin      completion event -> pin_prompt            (simulated_backend.cpp:121-132, 135-151)
//   flush    Backend::flush                            (simulated_backend.cpp:169-184)
//   preserve Backend::preserve                         (simulated_backend.cpp:190-193)
//   util     Backend::cache_utilization                (simulated_backend.cpp:186-188)
//
// plus the lifecycle signals (signals.hpp:13-41), the tracker state and verdict of every pressure
// tick (memory.cpp:150-169, 372-387), and the final action log (memory.cpp:389-401).
//
// Tokens are whitespace tokens (backend.cpp:60-97) interned to dense u32 ids in first-appearance
// order, so the GPU path can replay the stream on token ids. Output: one JSON object per line.
//
// Dispatch order is recovered without touching the reference: SimulatedBackend dispatches FCFS
// while busy < max_concurrency (simulated_backend.cpp:41-47); the wrapper mirrors that counter.
// Inside a completion event the reference runs pin_prompt -> --busy -> pump -> cb
// (simulated_backend.cpp:125-131), so the wrapped callback logs `pin` for the completing request
// and then `match` for whatever its freed slot dispatched, before forwarding the callback.
#include <cstdio>
#include <deque>
#include <fstream>
#include <iostream>
#include <set>
#include <unordered_map>

#include "stageflow/config.hpp"
#include "stageflow/harness.hpp"

using namespace stageflow;

namespace {

struct Recorder {
  std::vector<json> lines;
  std::unordered_map<std::string, std::uint32_t> ids;
  // Token ids of match records: inline ("tok"), appended to a binary u32 file ("toff" = offset
  // of the request's first id in it; --tok-out), or dropped (--no-tok: compact full-scale
  // goldens keep P, M, ops, signals, ticks, the action log and the end counters).
  enum class TokMode { Inline, File, None } tok_mode = TokMode::Inline;
  std::FILE* tok_file = nullptr;
  std::uint64_t tok_written = 0;

  std::uint32_t intern(const std::string& tok) {
    auto it = ids.find(tok);
    if (it != ids.end()) return it->second;
    auto id = static_cast<std::uint32_t>(ids.size());
    ids.emplace(tok, id);
    return id;
  }
  std::size_t push(json j) {
    j["seq"] = lines.size();
    lines.push_back(std::move(j));
    return lines.size() - 1;
  }
};

// --flaky REF:MODE: the backend's flush throws (test double for apply_action's retry path,
// memory.cpp:189-203): mode 1 on the first attempt of every flush action (the retry succeeds),
// mode 2 always. A throwing attempt never reaches the pin cache.
std::map<std::string, int> parse_flaky(const std::string& spec) {
  std::map<std::string, int> m;
  std::size_t i = 0;
  while (i < spec.size()) {
    std::size_t j = spec.find(',', i);
    if (j == std::string::npos) j = spec.size();
    const std::string item = spec.substr(i, j - i);
    const std::size_t c = item.find(':');
    if (c != std::string::npos) m[item.substr(0, c)] = std::stoi(item.substr(c + 1));
    i = j + 1;
  }
  return m;
}

class RecordingBackend : public Backend {
 public:
  RecordingBackend(std::shared_ptr<SimulatedBackend> inner, Recorder& rec, int flaky = 0)
      : inner_(std::move(inner)), rec_(rec), flaky_(flaky) {}

  const BackendDescriptor& descriptor() const override { return inner_->descriptor(); }
  bool has_capacity() const override { return inner_->has_capacity(); }
  const BackendStats& stats() const override { return inner_->stats(); }
  void set_capacity_listener(std::function<void()> fn) override {
    inner_->set_capacity_listener(std::move(fn));
  }

  void complete(CompletionRequest req, CompletionCallback cb) override {
    Req r;
    r.wf = req.metadata.workflow_id;
    r.stage = req.metadata.stage_id;
    for (const auto& t : context_token_sequence(req.messages)) r.tok.push_back(rec_.intern(t));
    const std::size_t rid = reqs_.size();
    reqs_.push_back(std::move(r));
    pending_.push_back(rid);
    inner_->complete(std::move(req),
                     [this, rid, cb = std::move(cb)](CompletionResponse resp, std::exception_ptr ep) {
                       on_complete(rid, resp);
                       cb(std::move(resp), ep);
                     });
    dispatch();  // the inner backend may have started it synchronously
  }

  long long flush(const FlushScope& scope) override {
    ++flush_attempts_;
    if (flaky_ == 2 || (flaky_ == 1 && flush_attempts_ % 2 == 1)) {
      rec_.push({{"type", "op"}, {"op", "flush_failed"}, {"b", descriptor().ref}, {"wf", scope.workflow_id}});
      throw BackendError("flush failed (flaky test backend)");
    }
    long long freed = inner_->flush(scope);
    rec_.push({{"type", "op"}, {"op", "flush"}, {"b", descriptor().ref},
               {"all", scope.all}, {"wf", scope.workflow_id}, {"freed", freed},
               {"occ", inner_->occupancy_tokens()}});
    return freed;
  }

  double cache_utilization() const override {
    double u = inner_->cache_utilization();
    rec_.push({{"type", "op"}, {"op", "util"}, {"b", inner_->descriptor().ref}, {"value", u}});
    return u;
  }

  bool preserve(const std::string& workflow_id) override {
    bool ok = inner_->preserve(workflow_id);
    rec_.push({{"type", "op"}, {"op", "preserve"}, {"b", descriptor().ref}, {"wf", workflow_id},
               {"ret", ok}});
    return ok;
  }

  SimulatedBackend& inner() { return *inner_; }

 private:
  struct Req {
    std::string wf, stage;
    std::vector<std::uint32_t> tok;
    std::size_t match_line = 0;
  };

  void dispatch() {
    const int maxc = inner_->config().max_concurrency;
    while (busy_ < maxc && !pending_.empty()) {
      auto rid = pending_.front();
      pending_.pop_front();
      ++busy_;
      auto& r = reqs_[rid];
      json j = {{"type", "op"}, {"op", "match"}, {"b", descriptor().ref},
                {"rid", rid}, {"wf", r.wf}, {"stage", r.stage},
                {"P", r.tok.size()}, {"M", -1}};
      if (rec_.tok_mode == Recorder::TokMode::Inline) {
        j["tok"] = r.tok;
      } else if (rec_.tok_mode == Recorder::TokMode::File) {
        j["toff"] = rec_.tok_written;
        std::fwrite(r.tok.data(), sizeof(std::uint32_t), r.tok.size(), rec_.tok_file);
        rec_.tok_written += r.tok.size();
      }
      r.match_line = rec_.push(std::move(j));
    }
  }

  void on_complete(std::size_t rid, const CompletionResponse& resp) {
    auto& r = reqs_[rid];
    rec_.lines[r.match_line]["M"] = resp.usage.cached_prefix_tokens;
    if (static_cast<long long>(r.tok.size()) != resp.usage.prompt_tokens) {
      throw std::logic_error("recorder: prompt token mismatch");
    }
    if (!r.wf.empty()) {
      const auto rej = inner_->capacity_rejections();
      rec_.push({{"type", "op"}, {"op", "pin"}, {"b", descriptor().ref}, {"rid", rid},
                 {"wf", r.wf}, {"P", r.tok.size()}, {"accepted", rej == last_rejections_},
                 {"occ", inner_->occupancy_tokens()}});
      last_rejections_ = rej;
    }
    --busy_;
    dispatch();
  }

  std::shared_ptr<SimulatedBackend> inner_;
  Recorder& rec_;
  std::vector<Req> reqs_;
  std::deque<std::size_t> pending_;
  int busy_ = 0;
  std::uint64_t last_rejections_ = 0;
  int flaky_ = 0;
  long long flush_attempts_ = 0;
};

const char* override_name(CachePolicyOverride o) {
  switch (o) {
    case CachePolicyOverride::Flush: return "flush";
    case CachePolicyOverride::Preserve: return "preserve";
    default: return "none";
  }
}

}  // namespace

int main(int argc, char** argv) {
  std::string config_path, trace_path, out_path, tok_path, flaky_spec;
  bool no_tok = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--no-tok") { no_tok = true; continue; }
    if (i + 1 >= argc) break;
    if (a == "--config") config_path = argv[++i];
    else if (a == "--trace") trace_path = argv[++i];
    else if (a == "--out") out_path = argv[++i];
    else if (a == "--tok-out") tok_path = argv[++i];
    else if (a == "--flaky") flaky_spec = argv[++i];
  }
  if (config_path.empty() || trace_path.empty() || out_path.empty()) {
    std::fprintf(stderr,
                 "usage: sf_ref_replay --config C.json --trace T.jsonl --out O.jsonl "
                 "[--tok-out T.u32 | --no-tok] [--flaky REF:MODE,...]\n");
    return 2;
  }
  auto config = load_config(config_path);
  auto templates = build_templates(config);
  auto trace = load_trace(trace_path, templates.names());

  Recorder rec;
  if (no_tok) rec.tok_mode = Recorder::TokMode::None;
  if (!tok_path.empty()) {
    rec.tok_mode = Recorder::TokMode::File;
    rec.tok_file = std::fopen(tok_path.c_str(), "wb");
    if (!rec.tok_file) throw std::runtime_error("cannot write " + tok_path);
  }
  EventLoop loop(ClockMode::Virtual);
  LogFn log = stderr_logger(LogLevel::Error);

  // build_registry (config.cpp:170-184), with each simulated backend wrapped.
  BackendRegistry registry;
  auto flaky = parse_flaky(flaky_spec);
  std::map<std::string, RecordingBackend*> recs;
  json meta_backends = json::array();
  for (const auto& b : config.backends) {
    if (b.descriptor.kind != BackendKind::Simulated) throw std::runtime_error("simulated only");
    auto sim = std::make_shared<SimulatedBackend>(loop, b.descriptor, b.sim, log);
    auto wrapped = std::make_shared<RecordingBackend>(sim, rec, flaky[b.descriptor.ref]);
    recs[b.descriptor.ref] = wrapped.get();
    registry.add(wrapped);
    meta_backends.push_back({{"ref", b.descriptor.ref}, {"model", b.descriptor.model},
                             {"capacity_tokens", b.sim.cache_capacity_tokens},
                             {"max_concurrency", b.sim.max_concurrency},
                             {"prefill_ms_per_token", b.sim.prefill_ms_per_token},
                             {"decode_ms_per_token", b.sim.decode_ms_per_token},
                             {"fixed_overhead_ms", b.sim.fixed_overhead_ms}});
  }
  rec.push({{"type", "meta"}, {"label", config.label}, {"backends", meta_backends},
            {"tau", config.memory.tau}, {"tau_pressure", config.memory.tau_pressure},
            {"monitor_interval_ms", config.memory.monitor_interval_ms},
            {"chain", config.memory.policy_chain}, {"flaky", flaky}});

  ToolRegistry tools;
  SignalBus bus;
  bus.subscribe([&rec](const LifecycleSignal& s) {
    rec.push({{"type", "sig"}, {"kind", signal_kind_name(s.kind)}, {"wf", s.workflow_id},
              {"stage", s.stage_id}, {"b", s.backend_ref}, {"model", s.model},
              {"tokens", s.context_tokens}, {"ts", s.ts}, {"override", override_name(s.cache_override)}});
  });
  MemoryManager memory(config.memory, &registry, log);
  memory.attach(bus);
  Orchestrator orch(loop, registry, tools, bus, config.orchestration, log);

  std::vector<std::string> workflow_ids;
  std::size_t remaining = trace.size();
  for (std::size_t i = 0; i < trace.size(); ++i) {
    const auto& r = trace[i];
    const std::string workflow_id = r.workflow_template + "-" + std::to_string(i);
    auto spec = templates.at(r.workflow_template)(
        r, workflow_id, config.template_params.value(r.workflow_template, json::object()));
    if (spec.stages.empty()) {
      --remaining;
      continue;
    }
    for (auto& [_, stage] : spec.stages) {
      if (stage.stage_scheduling_policy == "fcfs" && config.default_stage_policy != "fcfs")
        stage.stage_scheduling_policy = config.default_stage_policy;
      if (stage.request_scheduling_policy == "fcfs" && config.default_request_policy != "fcfs")
        stage.request_scheduling_policy = config.default_request_policy;
    }
    auto validated = validate_workflow(spec, registry);
    if (!validated.ok()) {
      std::string causes;
      for (const auto& e : validated.errors) causes += e.message + "; ";
      throw std::runtime_error("invalid workflow from " + r.workflow_template + ": " + causes);
    }
    const auto& wf = *validated.workflow;
    if (!wf.spec().workflow_memory_policy.empty())
      memory.set_workflow_chain(workflow_id, wf.spec().workflow_memory_policy);
    auto router = make_router(config, registry, wf);
    workflow_ids.push_back(workflow_id);
    orch.submit_at(static_cast<double>(r.arrival_ms), wf, std::move(router),
                   [&remaining](ExecutionReport) { --remaining; }, r.annotations());
  }

  // Pressure monitor (harness.cpp:81-90) with the tracker snapshot it decides on.
  auto tick = std::make_shared<std::function<void()>>();
  if (config.memory.monitor_interval_ms > 0) {
    *tick = [&, wp = std::weak_ptr<std::function<void()>>(tick)] {
      if (remaining == 0) return;
      json entries = json::array();
      const auto& tr = memory.tracker();
      for (const auto& wf : workflow_ids) {
        for (const auto& e : tr.preserved_entries(wf)) {
          entries.push_back({e.workflow_id, e.backend_ref, e.last_update_ts,
                             tr.in_flight(e.backend_ref, e.workflow_id), e.token_count});
        }
      }
      json util = json::object();
      for (auto& [ref, rb] : recs) util[ref] = rb->inner().cache_utilization();
      auto idx = rec.push({{"type", "tick"}, {"ts", loop.now_ms()}, {"entries", entries},
                           {"util", util}});
      auto actions = memory.pressure_tick(loop.now_ms());
      json victims = json::array();
      for (const auto& a : actions) victims.push_back({a.workflow_id, a.backend_ref});
      rec.lines[idx]["victims"] = victims;
      if (auto self = wp.lock()) loop.schedule_in(config.memory.monitor_interval_ms, *self);
    };
    loop.schedule_in(config.memory.monitor_interval_ms, *tick);
  }

  loop.run_until_idle();

  for (const auto& r : memory.action_log()) {
    rec.push({{"type", "act"}, {"trigger", r.trigger}, {"ts", r.ts},
              {"action", cache_action_kind_name(r.action.kind)}, {"workflow", r.action.workflow_id},
              {"backend", r.action.backend_ref}, {"reason", r.action.reason}});
  }
  json end_b = json::object();
  for (auto& [ref, rb] : recs) {
    auto& s = rb->inner();
    const auto& st = s.stats();
    end_b[ref] = {{"occupancy_tokens", s.occupancy_tokens()},
                  {"capacity_rejections", s.capacity_rejections()},
                  {"completions", st.completions}, {"flush_calls", st.flush_calls},
                  {"preserve_calls", st.preserve_calls}, {"prompt_tokens", st.prompt_tokens},
                  {"completion_tokens", st.completion_tokens},
                  {"cached_prefix_tokens", st.cached_prefix_tokens},
                  {"utilization", s.cache_utilization()}};
  }
  rec.push({{"type", "end"}, {"now_ms", loop.now_ms()}, {"backends", end_b},
            {"n_token_ids", rec.ids.size()}});

  if (rec.tok_file) std::fclose(rec.tok_file);
  std::ofstream out(out_path);
  for (const auto& l : rec.lines) out << l.dump() << "\n";
  return 0;
}

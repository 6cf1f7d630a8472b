// sf_gpu_replay — the reference's own orchestrator, memory manager and harness loop driving the
// B200 pool through GpuPinnedBackend (the drop-in). With --gpu-memory the reference's
// MemoryManager is replaced by GpuMemoryManager (policy resolution and the tracker on the B200);
// with --gpu-router the stage routers are the GPU ones (gpu_router.hpp: threshold / one-bit /
// plan decisions and reroute_on_overload through sfmap_*); with --host-tokenizer the backends
// tokenize on the host (context_token_sequence) instead of sfkv_tokenize_batch. Same wiring as run_benchmark
// (proj/src/harness.cpp:8-116) with GpuPinnedBackend in place of SimulatedBackend. Emits:
//   {"type":"req", b, wf, stage, P, M}   per dispatch, in dispatch order (M from the GPU)
//   {"type":"act", ...}                   the memory manager's action log (memory.cpp:389-401)
//   {"type":"end", backends: {...}}        final counters
// tests/test_dropin_replay.py compares this with the golden stream recorded from the unmodified
// reference (oracle/ref_shim/replay_driver.cpp) for the same (trace, config).
#include <fstream>

#include "gpu_memory_manager.hpp"
#include "gpu_pinned_backend.hpp"
#include "gpu_router.hpp"
#include "stageflow/config.hpp"
#include "stageflow/harness.hpp"

using namespace stageflow;

namespace {

// --flaky REF:MODE (test double, the same rule as oracle/ref_shim/replay_driver.cpp): the
// backend's flush throws on the first attempt of every flush action (mode 1) or always (2).
class FlakyFlush : public Backend {
 public:
  FlakyFlush(std::shared_ptr<GpuPinnedBackend> inner, int mode) : inner_(std::move(inner)), mode_(mode) {}
  const BackendDescriptor& descriptor() const override { return inner_->descriptor(); }
  bool has_capacity() const override { return inner_->has_capacity(); }
  void complete(CompletionRequest req, CompletionCallback cb) override { inner_->complete(std::move(req), std::move(cb)); }
  long long flush(const FlushScope& scope) override {
    ++attempts_;
    if (mode_ == 2 || (mode_ == 1 && attempts_ % 2 == 1)) throw BackendError("flush failed (flaky test backend)");
    return inner_->flush(scope);
  }
  double cache_utilization() const override { return inner_->cache_utilization(); }
  bool preserve(const std::string& wf) override { return inner_->preserve(wf); }
  const BackendStats& stats() const override { return inner_->stats(); }
  void set_capacity_listener(std::function<void()> fn) override { inner_->set_capacity_listener(std::move(fn)); }

 private:
  std::shared_ptr<GpuPinnedBackend> inner_;
  int mode_;
  long long attempts_ = 0;
};

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

}  // namespace

int main(int argc, char** argv) {
  std::string config_path, trace_path, out_path, flaky_spec;
  int device = 0;
  bool gpu_memory = false, gpu_router = false, host_tokenizer = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--gpu-memory") { gpu_memory = true; continue; }
    if (a == "--gpu-router") { gpu_router = true; continue; }
    if (a == "--host-tokenizer") { host_tokenizer = true; continue; }
    if (i + 1 >= argc) break;
    if (a == "--config") config_path = argv[++i];
    else if (a == "--trace") trace_path = argv[++i];
    else if (a == "--out") out_path = argv[++i];
    else if (a == "--device") device = std::stoi(argv[++i]);
    else if (a == "--flaky") flaky_spec = argv[++i];
  }
  if (config_path.empty() || trace_path.empty() || out_path.empty()) {
    std::fprintf(stderr, "usage: sf_gpu_replay --config C --trace T --out O [--device D]\n");
    return 2;
  }
  auto config = load_config(config_path);
  auto templates = build_templates(config);
  auto trace = load_trace(trace_path, templates.names());
  EventLoop loop(ClockMode::Virtual);
  LogFn log = stderr_logger(LogLevel::Error);

  std::vector<json> out;
  BackendRegistry registry;
  auto flaky = parse_flaky(flaky_spec);
  std::map<std::string, GpuPinnedBackend*> gpu;
  for (const auto& b : config.backends) {
    GpuPoolOptions opt;  // default sizes: the pool grows on demand (sfkv_pool_reserve)
    opt.device = device;
    opt.gpu_tokenizer = !host_tokenizer;
    auto be = std::make_shared<GpuPinnedBackend>(loop, b.descriptor, b.sim, opt, log);
    const std::string ref = b.descriptor.ref;
    be->set_dispatch_observer([&out, ref](const std::string& wf, const std::string& st,
                                          long long P, long long M) {
      out.push_back({{"type", "req"}, {"b", ref}, {"wf", wf}, {"stage", st}, {"P", P}, {"M", M}});
    });
    gpu[ref] = be.get();
    if (int mode = flaky[ref]) registry.add(std::make_shared<FlakyFlush>(be, mode));
    else registry.add(be);
  }
  ToolRegistry tools;
  SignalBus bus;
  std::unique_ptr<MemoryManager> cpu_mem;
  std::unique_ptr<GpuMemoryManager> gpu_mem;
  if (gpu_memory) {
    gpu_mem = std::make_unique<GpuMemoryManager>(config.memory, &registry, 256, device, log);
    gpu_mem->attach(bus);
  } else {
    cpu_mem = std::make_unique<MemoryManager>(config.memory, &registry, log);
    cpu_mem->attach(bus);
  }
  auto set_chain = [&](const std::string& wf, const std::vector<std::string>& names) {
    if (gpu_mem) gpu_mem->set_workflow_chain(wf, names);
    else cpu_mem->set_workflow_chain(wf, names);
  };
  auto pressure_tick = [&](double now) {
    if (gpu_mem) gpu_mem->pressure_tick(now);
    else cpu_mem->pressure_tick(now);
  };
  Orchestrator orch(loop, registry, tools, bus, config.orchestration, log);

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
    if (!validated.ok()) throw std::runtime_error("invalid workflow from " + r.workflow_template);
    const auto& wf = *validated.workflow;
    if (!wf.spec().workflow_memory_policy.empty())
      set_chain(workflow_id, wf.spec().workflow_memory_policy);
    auto router = gpu_router ? make_gpu_router(config, registry, wf, orch, device) : make_router(config, registry, wf);
    orch.submit_at(static_cast<double>(r.arrival_ms), wf, std::move(router),
                   [&remaining](ExecutionReport) { --remaining; }, r.annotations());
  }
  auto tick = std::make_shared<std::function<void()>>();
  if (config.memory.monitor_interval_ms > 0) {
    *tick = [&, wp = std::weak_ptr<std::function<void()>>(tick)] {
      if (remaining == 0) return;
      pressure_tick(loop.now_ms());
      if (auto self = wp.lock()) loop.schedule_in(config.memory.monitor_interval_ms, *self);
    };
    loop.schedule_in(config.memory.monitor_interval_ms, *tick);
  }
  loop.run_until_idle();

  for (const auto& r : gpu_mem ? gpu_mem->action_log() : cpu_mem->action_log()) {
    out.push_back({{"type", "act"}, {"trigger", r.trigger}, {"ts", r.ts},
                   {"action", cache_action_kind_name(r.action.kind)},
                   {"workflow", r.action.workflow_id}, {"backend", r.action.backend_ref},
                   {"reason", r.action.reason}});
  }
  json end_b = json::object();
  for (auto& [ref, g] : gpu) {
    const auto& st = g->stats();
    end_b[ref] = {{"occupancy_tokens", g->occupancy_tokens()},
                  {"capacity_rejections", g->capacity_rejections()},
                  {"completions", st.completions}, {"flush_calls", st.flush_calls},
                  {"preserve_calls", st.preserve_calls}, {"prompt_tokens", st.prompt_tokens},
                  {"completion_tokens", st.completion_tokens},
                  {"cached_prefix_tokens", st.cached_prefix_tokens},
                  {"utilization", g->cache_utilization()}};
  }
  out.push_back({{"type", "end"}, {"now_ms", loop.now_ms()}, {"backends", end_b}});
  std::ofstream f(out_path);
  for (const auto& l : out) f << l.dump() << "\n";
  return 0;
}

// See gpu_memory_manager.hpp. Semantics follow MemoryManager (proj/src/memory.cpp:233-401)
// line by line; the resolution itself runs in paper_2603_13605_b200/csrc/tracker.cu.
#include "gpu_memory_manager.hpp"

#include <algorithm>
#include <ostream>

namespace stageflow {

namespace {
uint8_t policy_code(const std::string& name) {
  if (name == "preserve_small_increment") return SFMM_POLICY_PRESERVE_SMALL_INCREMENT;
  if (name == "flush_at_boundary") return SFMM_POLICY_FLUSH_AT_BOUNDARY;
  throw std::invalid_argument("unknown memory policy: " + name);  // memory.cpp:182
}
const char* reason_name(uint8_t r) {
  switch (r) {
    case SFMM_REASON_OVERRIDE: return "override";
    case SFMM_REASON_PRESERVE_SMALL_INCREMENT: return "preserve_small_increment";
    case SFMM_REASON_FLUSH_AT_BOUNDARY: return "flush_at_boundary";
    case SFMM_REASON_FLUSH_UNDER_PRESSURE: return "flush_under_pressure";
    default: return "chain_exhausted";
  }
}
}  // namespace

GpuMemoryManager::GpuMemoryManager(MemoryConfig config, BackendRegistry* backends, int max_workflows,
                                   int device, LogFn log)
    : config_(std::move(config)), backends_(backends), log_(std::move(log)) {
  if (config_.tau <= 0) throw std::invalid_argument("tau must be positive");
  if (config_.tau_pressure <= 0 || config_.tau_pressure > 1)
    throw std::invalid_argument("tau_pressure must be in (0, 1]");
  if (backends_) refs_ = backends_->refs();  // sorted, as the reference's utilization map
  for (std::size_t i = 0; i < refs_.size(); ++i) backend_index_[refs_[i]] = static_cast<int32_t>(i);
  sfmm_config c{};
  c.device = device;
  c.max_workflows = max_workflows;
  c.n_backends = std::max<int32_t>(1, static_cast<int32_t>(refs_.size()));
  if (config_.policy_chain.size() > SFMM_MAX_CHAIN) throw std::invalid_argument("policy chain too long");
  c.chain_len = static_cast<int32_t>(config_.policy_chain.size());
  for (std::size_t i = 0; i < config_.policy_chain.size(); ++i) c.chain[i] = policy_code(config_.policy_chain[i]);
  c.tau = config_.tau;
  c.tau_pressure = config_.tau_pressure;
  check(sfmm_tracker_create(&c, &tracker_), "sfmm_tracker_create");
}

GpuMemoryManager::~GpuMemoryManager() {
  if (tracker_) sfmm_tracker_destroy(tracker_);
}

void GpuMemoryManager::check(int rc, const char* what) const {
  if (rc != 0) throw BackendError(std::string(what) + " failed (" + std::to_string(rc) + "): " + sfkv_last_error());
}

int32_t GpuMemoryManager::slot_for(const std::string& wf) {
  auto it = slots_.find(wf);
  if (it != slots_.end()) return it->second;
  const int32_t s = static_cast<int32_t>(slot_names_.size());
  slots_[wf] = s;
  slot_names_.push_back(wf);
  ranks_dirty_ = true;
  return s;
}

void GpuMemoryManager::push_ranks() {  // rank of every slot's workflow id in std::string order
  if (!ranks_dirty_) return;
  std::vector<uint32_t> rank(slot_names_.size());
  uint32_t r = 0;
  for (const auto& [wf, slot] : slots_) rank[slot] = r++;  // std::map iterates in string order
  check(sfmm_set_workflow_ranks(tracker_, static_cast<int64_t>(rank.size()), rank.data()),
        "sfmm_set_workflow_ranks");
  ranks_dirty_ = false;
}

void GpuMemoryManager::set_workflow_chain(const std::string& workflow_id, const std::vector<std::string>& names) {
  if (names.empty()) return;  // memory.cpp:248
  std::vector<uint8_t> codes;
  for (const auto& n : names) codes.push_back(policy_code(n));
  check(sfmm_set_workflow_chain(tracker_, slot_for(workflow_id), static_cast<int32_t>(codes.size()), codes.data()),
        "sfmm_set_workflow_chain");
}

void GpuMemoryManager::attach(SignalBus& bus) {
  bus.subscribe([this](const LifecycleSignal& sig) { on_signal(sig); });
}

// apply_and_record (memory.cpp:312-328) with apply_action (memory.cpp:185-220). The GPU tracker
// has already erased a flushed entry; sfkv pools do not fail a flush, so the "mark_unpreserved on
// failure" branch cannot arise.
void GpuMemoryManager::apply_and_record(const CacheAction& action, const std::string& trigger, double ts) {
  if (!action.is_noop() && backends_ && backends_->contains(action.backend_ref))
    apply_action(action, *backends_, log_);
  action_log_.push_back(MemoryManager::LogRecord{trigger, ts, action});
}

std::vector<CacheAction> GpuMemoryManager::on_signal(const LifecycleSignal& sig) {
  const bool wfc = sig.kind == LifecycleSignal::Kind::WorkflowComplete;
  const int32_t w = slot_for(sig.workflow_id);
  uint8_t kind = static_cast<uint8_t>(sig.kind), ov = static_cast<uint8_t>(sig.cache_override);
  int32_t stage = 0, b = 0, model = 0;
  int64_t tokens = sig.context_tokens;
  double ts = sig.ts;
  if (!wfc) {
    auto& st = stages_[sig.workflow_id];
    auto si = st.find(sig.stage_id);
    if (si == st.end()) si = st.emplace(sig.stage_id, static_cast<int32_t>(st.size())).first;
    stage = si->second;
    auto bi = backend_index_.find(sig.backend_ref);
    if (bi == backend_index_.end()) throw UnknownBackendError(sig.backend_ref);
    b = bi->second;
    auto mi = models_.find(sig.model);
    if (mi == models_.end()) mi = models_.emplace(sig.model, static_cast<int32_t>(models_.size())).first;
    model = mi->second;
  }
  sfmm_signals s{&kind, &w, &stage, &b, &model, &tokens, &ts, &ov};
  std::vector<uint8_t> rk(refs_.size() + 1), rr(refs_.size() + 1);
  std::vector<int32_t> rb(refs_.size() + 1);
  int32_t count = 0;
  uint8_t status = 0;
  sfmm_records out{&count, &status, rk.data(), rb.data(), rr.data()};
  check(sfmm_on_signal_batch(tracker_, 1, &s, &out), "sfmm_on_signal_batch");
  if (status == SFMM_SIG_OUT_OF_ORDER)  // check_order (memory.cpp:256-285)
    throw OutOfOrderSignalError("out-of-order signal for " + sig.workflow_id);
  const std::string trigger = std::string(signal_kind_name(sig.kind)) + " " + sig.workflow_id +
                              (sig.stage_id.empty() ? "" : "/" + sig.stage_id);
  std::vector<CacheAction> actions;
  for (int32_t j = 0; j < count; ++j) {
    if (rk[j] == SFMM_ACT_NOOP) actions.push_back(CacheAction::noop(reason_name(rr[j])));
    else if (rk[j] == SFMM_ACT_FLUSH) actions.push_back(CacheAction::flush(sig.workflow_id, refs_[rb[j]], reason_name(rr[j])));
    else actions.push_back(CacheAction::preserve(sig.workflow_id, refs_[rb[j]], reason_name(rr[j])));
  }
  for (const auto& a : actions) apply_and_record(a, trigger, sig.ts);
  if (status == SFMM_SIG_NEGATIVE_IN_FLIGHT) throw std::logic_error("in-flight count went negative");
  return actions;
}

std::vector<CacheAction> GpuMemoryManager::pressure_tick(double now_ms) {
  std::map<std::string, double> utilization;
  if (backends_)
    for (const auto& ref : backends_->refs()) utilization[ref] = backends_->at(ref).cache_utilization();
  return pressure_tick(utilization, now_ms);
}

std::vector<CacheAction> GpuMemoryManager::pressure_tick(const std::map<std::string, double>& utilization,
                                                         double now_ms) {
  std::vector<double> util(std::max<std::size_t>(refs_.size(), 1), 0.0);
  for (const auto& [ref, u] : utilization) {
    auto it = backend_index_.find(ref);
    if (it != backend_index_.end()) util[it->second] = u;
  }
  push_ranks();
  std::vector<int32_t> victim(util.size(), -1);
  check(sfmm_pressure_tick(tracker_, util.data(), victim.data()), "sfmm_pressure_tick");
  std::vector<CacheAction> actions;
  for (std::size_t b = 0; b < refs_.size(); ++b)  // utilization-map (sorted ref) order
    if (victim[b] >= 0)
      actions.push_back(CacheAction::flush(slot_names_[victim[b]], refs_[b], "flush_under_pressure"));
  for (const auto& a : actions) apply_and_record(a, "pressure_tick", now_ms);
  return actions;
}

void GpuMemoryManager::export_action_log(std::ostream& out) const {
  for (const auto& rec : action_log_) {
    json line = {{"trigger", rec.trigger}, {"ts", rec.ts}, {"action", cache_action_kind_name(rec.action.kind)},
                 {"workflow", rec.action.workflow_id}, {"backend", rec.action.backend_ref},
                 {"reason", rec.action.reason}};
    out << line.dump() << "\n";
  }
}

}  // namespace stageflow

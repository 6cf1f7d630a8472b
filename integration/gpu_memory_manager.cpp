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
  std::vector<uint8_t> chain;
  for (const auto& n : config_.policy_chain) chain.push_back(policy_code(n));
  cap_workflows_ = std::max(1, max_workflows);
  cap_backends_ = std::max<int32_t>(4, backends_ ? static_cast<int32_t>(backends_->refs().size()) : 0);
  cap_stages_ = 64;
  sfmm_config c{};
  c.device = device;
  c.max_workflows = cap_workflows_;
  c.n_backends = cap_backends_;
  c.max_stages = cap_stages_;
  c.chain_len = static_cast<int32_t>(chain.size());
  c.chain = chain.data();
  c.tau = config_.tau;
  c.tau_pressure = config_.tau_pressure;
  check(sfmm_tracker_create(&c, &tracker_), "sfmm_tracker_create");
  slot_names_.assign(cap_workflows_, std::string());
  for (int32_t s = cap_workflows_ - 1; s >= 0; --s) free_slots_.push_back(s);
  if (backends_)
    for (const auto& ref : backends_->refs()) backend_for(ref);  // registry order = sorted order
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
  if (free_slots_.empty()) {  // grow: the reference's maps are unbounded
    const int32_t w1 = 2 * cap_workflows_;
    check(sfmm_tracker_reserve(tracker_, w1, cap_backends_, cap_stages_), "sfmm_tracker_reserve");
    for (int32_t s = w1 - 1; s >= cap_workflows_; --s) free_slots_.push_back(s);
    slot_names_.resize(w1);
    cap_workflows_ = w1;
  }
  const int32_t s = free_slots_.back();
  free_slots_.pop_back();
  slots_[wf] = s;
  slot_names_[s] = wf;
  ranks_dirty_ = true;
  return s;
}

// WorkflowComplete erased every tracker row of the workflow (memory.cpp:352-358): its slot is
// forgotten and reused; the id stays in completed_ for check_order.
void GpuMemoryManager::release_slot(const std::string& wf) {
  auto it = slots_.find(wf);
  if (it == slots_.end()) return;
  const int32_t s = it->second;
  check(sfmm_reset_workflows(tracker_, 1, &s), "sfmm_reset_workflows");
  slots_.erase(it);
  slot_names_[s].clear();
  stages_.erase(wf);
  free_slots_.push_back(s);
  ranks_dirty_ = true;
}

int32_t GpuMemoryManager::backend_for(const std::string& ref) {
  auto it = backend_index_.find(ref);
  if (it != backend_index_.end()) return it->second;
  const int32_t b = static_cast<int32_t>(refs_.size());
  if (b >= cap_backends_) {
    const int32_t nb = 2 * cap_backends_;
    check(sfmm_tracker_reserve(tracker_, cap_workflows_, nb, cap_stages_), "sfmm_tracker_reserve");
    cap_backends_ = nb;
  }
  refs_.push_back(ref);
  backend_index_[ref] = b;
  std::vector<int32_t> order;  // std::string order first (the map's), then the unused indices
  for (const auto& [r, i] : backend_index_) order.push_back(i);
  for (int32_t i = static_cast<int32_t>(refs_.size()); i < cap_backends_; ++i) order.push_back(i);
  check(sfmm_set_backend_order(tracker_, cap_backends_, order.data()), "sfmm_set_backend_order");
  return b;
}

void GpuMemoryManager::push_ranks() {  // rank of every live slot's workflow id in std::string order
  if (!ranks_dirty_) return;
  std::vector<uint32_t> rank(cap_workflows_, UINT32_MAX);
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
// recorded the flush as applied (entry erased); a flush the backend refused twice is reported
// back so the entry is only unpreserved (memory.cpp:322-324).
void GpuMemoryManager::apply_and_record(const CacheAction& action, const std::string& trigger, double ts,
                                        int32_t slot, int32_t backend, int64_t sig) {
  if (!action.is_noop() && backends_ && backends_->contains(action.backend_ref)) {
    const bool applied = apply_action(action, *backends_, log_);
    if (!applied && action.kind == CacheAction::Kind::Flush)
      check(sfmm_flush_failed(tracker_, 1, &slot, &backend, &sig), "sfmm_flush_failed");
  }
  action_log_.push_back(MemoryManager::LogRecord{trigger, ts, action});
}

std::vector<CacheAction> GpuMemoryManager::on_signal(const LifecycleSignal& sig) {
  if (completed_.count(sig.workflow_id))  // check_order (memory.cpp:257-259)
    throw OutOfOrderSignalError("signal after WorkflowComplete for " + sig.workflow_id);
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
    if (stage >= cap_stages_) {
      int32_t s1 = cap_stages_;
      while (s1 <= stage) s1 *= 2;
      check(sfmm_tracker_reserve(tracker_, cap_workflows_, cap_backends_, s1), "sfmm_tracker_reserve");
      cap_stages_ = s1;
    }
    b = backend_for(sig.backend_ref);
    auto mi = models_.find(sig.model);
    if (mi == models_.end()) mi = models_.emplace(sig.model, static_cast<int32_t>(models_.size())).first;
    model = mi->second;
  }
  sfmm_signals s{&kind, &w, &stage, &b, &model, &tokens, &ts, &ov};
  std::vector<uint8_t> rk(cap_backends_ + 1), rr(cap_backends_ + 1);
  std::vector<int32_t> rb(cap_backends_ + 1);
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
  for (int32_t j = 0; j < count; ++j) apply_and_record(actions[j], trigger, sig.ts, w, rb[j], 0);
  if (status == SFMM_SIG_NEGATIVE_IN_FLIGHT) throw std::logic_error("in-flight count went negative");
  if (wfc) {
    completed_.insert(sig.workflow_id);
    release_slot(sig.workflow_id);
  }
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
  // A ref without tracker entries cannot yield a victim, so refs never seen in a signal are
  // skipped (the reference evaluates them and finds nothing, memory.cpp:154-167).
  std::vector<double> util(cap_backends_, 0.0);
  for (const auto& [ref, u] : utilization) {
    auto it = backend_index_.find(ref);
    if (it != backend_index_.end()) util[it->second] = u;
  }
  push_ranks();
  std::vector<int32_t> victim(cap_backends_, -1);
  check(sfmm_pressure_tick(tracker_, util.data(), victim.data()), "sfmm_pressure_tick");
  std::vector<CacheAction> actions;
  std::vector<std::pair<int32_t, int32_t>> who;  // (slot, backend) per action
  for (const auto& [ref, b] : backend_index_)  // utilization-map (sorted ref) order
    if (utilization.count(ref) && victim[b] >= 0) {
      actions.push_back(CacheAction::flush(slot_names_[victim[b]], ref, "flush_under_pressure"));
      who.emplace_back(victim[b], b);
    }
  for (std::size_t j = 0; j < actions.size(); ++j)
    apply_and_record(actions[j], "pressure_tick", now_ms, who[j].first, who[j].second, -1);
  return actions;
}

int GpuMemoryManager::entry_state(const std::string& workflow_id, const std::string& backend_ref) const {
  auto s = slots_.find(workflow_id);
  auto b = backend_index_.find(backend_ref);
  if (s == slots_.end() || b == backend_index_.end()) return -1;
  const std::size_t E = static_cast<std::size_t>(cap_workflows_) * cap_backends_;
  std::vector<uint8_t> present(E), preserved(E);
  check(sfmm_tracker_entries(tracker_, present.data(), preserved.data(), nullptr, nullptr, nullptr),
        "sfmm_tracker_entries");
  const std::size_t e = static_cast<std::size_t>(s->second) * cap_backends_ + b->second;
  return present[e] ? preserved[e] : -1;
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

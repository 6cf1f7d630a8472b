// GpuMemoryManager — the reference-side binding of the GPU memory manager (sfmm_*, include/sfkv.h).
//
// The public surface of stageflow::MemoryManager (proj/include/stageflow/memory.hpp:122-150) over a
// GPU-resident WorkflowTracker: on_signal / attach(SignalBus) / pressure_tick / set_workflow_chain /
// action_log / export_action_log. Policy resolution and tracker updates run on the B200
// (sfmm_on_signal_batch, sfmm_pressure_tick); the host keeps the string interning (workflow ids ->
// slots with their std::string rank, backend refs in registry order, stage ids, models), applies
// the resolved actions to the backends exactly as apply_action does (memory.cpp:185-220) and keeps
// the action log. Signals arrive one at a time from the synchronous SignalBus, so each call is a
// batch of one; a scheduler that sees many signals at once passes them in one batch.
//
// Reference-side code: compiled against the reference headers by oracle/Makefile only.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "sfkv.h"
#include "stageflow/memory.hpp"

namespace stageflow {

class GpuMemoryManager {
 public:
  GpuMemoryManager(MemoryConfig config, BackendRegistry* backends, int max_workflows, int device = 0,
                   LogFn log = {});
  ~GpuMemoryManager();
  GpuMemoryManager(const GpuMemoryManager&) = delete;
  GpuMemoryManager& operator=(const GpuMemoryManager&) = delete;

  std::vector<CacheAction> on_signal(const LifecycleSignal& sig);
  std::vector<CacheAction> pressure_tick(double now_ms = 0);
  std::vector<CacheAction> pressure_tick(const std::map<std::string, double>& utilization,
                                         double now_ms = 0);
  void set_workflow_chain(const std::string& workflow_id, const std::vector<std::string>& names);
  void attach(SignalBus& bus);

  const std::vector<MemoryManager::LogRecord>& action_log() const { return action_log_; }
  void export_action_log(std::ostream& out) const;

 private:
  MemoryConfig config_;
  BackendRegistry* backends_;
  LogFn log_;
  sfmm_tracker* tracker_ = nullptr;
  std::vector<std::string> refs_;                  // backend index -> ref (sorted)
  std::map<std::string, int32_t> backend_index_;
  std::map<std::string, int32_t> slots_;           // workflow id -> slot (first seen)
  std::vector<std::string> slot_names_;
  std::map<std::string, std::map<std::string, int32_t>> stages_;
  std::map<std::string, int32_t> models_;
  bool ranks_dirty_ = false;
  std::vector<MemoryManager::LogRecord> action_log_;

  int32_t slot_for(const std::string& wf);
  void push_ranks();
  void apply_and_record(const CacheAction& action, const std::string& trigger, double ts);
  void check(int rc, const char* what) const;
};

}  // namespace stageflow

// GpuMemoryManager — the reference-side binding of the GPU memory manager (sfmm_*, include/sfkv.h).
//
// The public surface of stageflow::MemoryManager (proj/include/stageflow/memory.hpp:122-150) over a
// GPU-resident WorkflowTracker: on_signal / attach(SignalBus) / pressure_tick / set_workflow_chain /
// action_log / export_action_log. Policy resolution and tracker updates run on the B200
// (sfmm_on_signal_batch, sfmm_pressure_tick); the host keeps the string interning (workflow ids ->
// slots with their std::string rank, backend refs in registry order, stage ids, models), applies
// the resolved actions to the backends exactly as apply_action does (memory.cpp:185-220: a flush
// that fails twice leaves the entry unpreserved, reported back with sfmm_flush_failed) and keeps
// the action log. Signals arrive one at a time from the synchronous SignalBus, so each call is a
// batch of one; a scheduler that sees many signals at once passes them in one batch.
// Nothing is capped: backend refs are interned lazily (any ref, registered or not, as the
// reference's string-keyed maps), and slots, backends and stage ids grow the tracker on demand;
// a finished workflow's slot is recycled (its id stays in the completed set, so later signals
// still raise OutOfOrderSignalError, memory.cpp:257-259).
//
// Reference-side code: compiled against the reference headers by oracle/Makefile only.
#pragma once

#include <map>
#include <set>
#include <string>
#include <vector>

#include "sfkv.h"
#include "stageflow/memory.hpp"

namespace stageflow {

class GpuMemoryManager {
 public:
  /// max_workflows / n_backends are initial sizes: the tracker grows on demand (the reference's
  /// maps are unbounded). backends may be null (every action then "applies", as the reference).
  GpuMemoryManager(MemoryConfig config, BackendRegistry* backends, int max_workflows = 1024,
                   int device = 0, LogFn log = {});
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

  /// Tracker inspection (WorkflowTracker::entry): nullopt-like -1 when absent, else preserved.
  int entry_state(const std::string& workflow_id, const std::string& backend_ref) const;

 private:
  MemoryConfig config_;
  BackendRegistry* backends_;
  LogFn log_;
  sfmm_tracker* tracker_ = nullptr;
  int32_t cap_workflows_ = 0, cap_backends_ = 0, cap_stages_ = 0;
  std::vector<std::string> refs_;                  // backend index -> ref (first-seen order)
  std::map<std::string, int32_t> backend_index_;   // iterates in std::string order
  std::map<std::string, int32_t> slots_;           // live workflow id -> slot
  std::vector<std::string> slot_names_;
  std::vector<int32_t> free_slots_;
  std::set<std::string> completed_;                // WorkflowComplete seen (check_order)
  std::map<std::string, std::map<std::string, int32_t>> stages_;
  std::map<std::string, int32_t> models_;
  bool ranks_dirty_ = false;
  std::vector<MemoryManager::LogRecord> action_log_;

  int32_t slot_for(const std::string& wf);
  int32_t backend_for(const std::string& ref);
  void release_slot(const std::string& wf);
  void push_ranks();
  // apply_and_record (memory.cpp:312-328); sig = the record's signal index in the last tracker
  // batch, -1 for a pressure tick.
  void apply_and_record(const CacheAction& action, const std::string& trigger, double ts, int32_t slot,
                        int32_t backend, int64_t sig);
  void check(int rc, const char* what) const;
};

}  // namespace stageflow

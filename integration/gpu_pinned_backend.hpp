// GpuPinnedBackend — the reference-side binding of libsfkv (include/sfkv.h).
//
// A drop-in `stageflow::Backend` (reference: proj/include/stageflow/backend.hpp:85-119) with the
// observable behaviour of `SimulatedBackend` (proj/include/stageflow/simulated_backend.hpp:57-124):
// the same FCFS admission, latency model and reply rules, but the per-workflow pinned-prefix cache
// lives in a B200 KV pool and every cache operation is an sfkv_* call:
//
//   start()  -> sfkv_match_batch   (replaces prefix_match,     simulated_backend.cpp:153-162)
//   commit   -> sfkv_commit_batch  (replaces pin_prompt,       simulated_backend.cpp:135-151)
//   flush    -> sfkv_flush         (replaces flush,            simulated_backend.cpp:169-184)
//   preserve -> sfkv_preserve      (replaces preserve,         simulated_backend.cpp:190-193)
//   utilization -> sfkv_cache_utilization                     (simulated_backend.cpp:186-188)
//
// It compiles against the reference's headers (it IS reference-side code) and is built by
// oracle/Makefile only where /root/reference exists; the product library does not depend on it.
#pragma once

#include <deque>
#include <functional>
#include <map>
#include <unordered_map>

#include "sfkv.h"
#include "stageflow/simulated_backend.hpp"

namespace stageflow {

struct GpuPoolOptions {
  int device = 0;
  int max_workflows = 1 << 14;
  int max_pin_blocks = 4096;  // 65,536-token pins
};

class GpuPinnedBackend : public Backend {
 public:
  using DispatchObserver = std::function<void(const std::string& wf, const std::string& stage,
                                              long long prompt_tokens, long long cached_tokens)>;

  GpuPinnedBackend(EventLoop& loop, BackendDescriptor descriptor, SimulatedBackendConfig config,
                   GpuPoolOptions options = {}, LogFn log = {});
  ~GpuPinnedBackend() override;

  const BackendDescriptor& descriptor() const override { return descriptor_; }
  bool has_capacity() const override;
  void complete(CompletionRequest req, CompletionCallback cb) override;
  long long flush(const FlushScope& scope) override;
  double cache_utilization() const override;
  bool preserve(const std::string& workflow_id) override;
  const BackendStats& stats() const override { return stats_; }

  long long pinned_token_count(const std::string& workflow_id) const;
  long long occupancy_tokens() const;
  std::uint64_t capacity_rejections() const;
  void set_dispatch_observer(DispatchObserver fn) { observer_ = std::move(fn); }

 private:
  struct Pending {
    CompletionRequest req;
    CompletionCallback cb;
    double arrival_ms;
  };

  EventLoop& loop_;
  BackendDescriptor descriptor_;
  SimulatedBackendConfig config_;
  GpuPoolOptions options_;
  LogFn log_;
  BackendStats stats_;
  sfkv_pool* pool_ = nullptr;
  int busy_ = 0;
  std::deque<Pending> pending_;
  std::map<std::pair<std::string, std::string>, int> turns_;
  std::unordered_map<std::string, int32_t> slots_;
  DispatchObserver observer_;

  void pump();
  void start(Pending item);
  ScriptedReply reply_for(const CompletionRequest& req, int turn) const;
  int32_t slot_for(const std::string& workflow_id);  // creates
  int32_t find_slot(const std::string& workflow_id) const;  // -1 when never seen
  void check(int rc, const char* what) const;
};

/// Token-string interner shared by all GPU backends of a process (token id = first appearance).
std::uint32_t intern_token(const std::string& token);

}  // namespace stageflow

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
#include <vector>

#include "sfkv.h"
#include "stageflow/simulated_backend.hpp"

namespace stageflow {

// Initial pool sizes. The reference's cache is unbounded (std::map pins_), so the pool starts at
// these sizes and grows on demand (sfkv_pool_reserve): more live workflows than slots, or a
// prompt longer than max_pin_blocks * 16 tokens. A workflow's slot returns to a free list once it
// holds no pin and has no request in this backend.
struct GpuPoolOptions {
  int device = 0;
  int max_workflows = 256;
  int max_pin_blocks = 256;  // 4,096-token pins before the first reserve
  // Tokenize + intern on the GPU (sfkv_tokenize_batch over this backend's interner), one call for
  // every request a pump() starts, instead of context_token_sequence + a host string map. Token
  // ids are only ever compared within this backend's pool, so each backend has its own interner.
  bool gpu_tokenizer = true;
  int interner_log2 = 22;               // 4 M distinct token strings
  long long interner_arena = 256 << 20;  // bytes of token text
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
  // workflow id -> slot while the workflow holds a pin or has a request here
  std::unordered_map<std::string, int32_t> slots_;
  std::vector<int32_t> free_slots_;
  std::vector<int32_t> slot_requests_;  // requests of the slot's workflow queued or running here
  std::vector<char> slot_pinned_;       // host mirror of "the pool holds a pin for this slot"
  std::vector<std::string> slot_names_;
  int32_t slot_cap_ = 0, pin_blocks_cap_ = 0;
  std::unordered_map<std::string, std::uint32_t> intern_;  // this backend's token ids
  DispatchObserver observer_;

  sfkv_interner* interner_ = nullptr;  // gpu_tokenizer: this backend's token ids
  void pump();
  void start(Pending item);
  // GPU tokenizer path: every item pump() starts at this instant, tokenized and matched in one
  // batch (M is read at start, pins change only at completion, so batching is exact).
  void start_batch(std::vector<Pending> items);
  void dispatch(Pending item, std::vector<std::uint32_t> ids, long long M, int32_t slot);
  ScriptedReply reply_for(const CompletionRequest& req, int turn) const;
  int32_t slot_for(const std::string& workflow_id);  // creates (grows the pool if needed)
  int32_t find_slot(const std::string& workflow_id) const;  // -1 when none is held
  void maybe_release(int32_t slot);
  bool reserve(int32_t slots, int32_t pin_blocks);
  std::uint32_t intern(const std::string& token);
  void check(int rc, const char* what) const;
};

}  // namespace stageflow

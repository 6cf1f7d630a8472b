// GpuPinnedBackend implementation (see gpu_pinned_backend.hpp). The scheduling and latency rules
// restate SimulatedBackend's documented behaviour (simulated_backend.hpp:57-76 and
// simulated_backend.cpp:31-133); only the cache operations differ: they go to the B200 pool.
#include "gpu_pinned_backend.hpp"

#include <algorithm>
#include <cmath>

namespace stageflow {

namespace {

std::string numbered_words(long long n) {  // "out0 out1 ... out{n-1}" placeholder reply
  std::string s;
  for (long long i = 0; i < n; ++i) {
    if (i) s.push_back(' ');
    s += "out";
    s += std::to_string(i);
  }
  return s;
}

int ceil_log2(long long x) {
  int l = 0;
  while ((1LL << l) < x) ++l;
  return l;
}

// Physical blocks never bind in parity mode: every logical token once, one partial block per
// pin, and one maximal pin of transient headroom (a replaced pin is released after commit).
long long blocks_for(long long capacity, int32_t slots, int32_t pin_blocks) {
  return capacity / SFKV_BLOCK_TOKENS + slots + 2LL * pin_blocks + 64;
}

}  // namespace

GpuPinnedBackend::GpuPinnedBackend(EventLoop& loop, BackendDescriptor descriptor,
                                   SimulatedBackendConfig config, GpuPoolOptions options, LogFn log)
    : loop_(loop), descriptor_(std::move(descriptor)), config_(std::move(config)),
      options_(options), log_(std::move(log)) {
  if (config_.max_concurrency < 1) throw BackendError("max_concurrency must be >= 1");
  if (config_.cache_capacity_tokens <= 0) throw BackendError("cache capacity must be positive");
  if (config_.prefill_ms_per_token <= 0 || config_.decode_ms_per_token <= 0)
    throw BackendError("latency parameters must be positive");
  slot_cap_ = std::max(1, options_.max_workflows);
  pin_blocks_cap_ = std::max(1, options_.max_pin_blocks);
  sfkv_pool_config pc{};
  pc.device = options_.device;
  pc.max_workflows = slot_cap_;
  pc.capacity_tokens = config_.cache_capacity_tokens;
  pc.max_pin_blocks = pin_blocks_cap_;
  pc.n_blocks = blocks_for(config_.cache_capacity_tokens, slot_cap_, pin_blocks_cap_);
  pc.table_log2 = ceil_log2(2 * pc.n_blocks) + 1;
  pc.n_slabs = 0;  // the reference holds no KV bytes; this binding is metadata-only
  pc.slab_row_bytes = 0;
  check(sfkv_pool_create(&pc, &pool_), "sfkv_pool_create");
  if (options_.gpu_tokenizer) {
    const int rc = sfkv_interner_create(options_.device, options_.interner_log2, options_.interner_arena, &interner_);
    if (rc != SFKV_OK) {
      sfkv_pool_destroy(pool_);
      check(rc, "sfkv_interner_create");
    }
  }
  slot_requests_.assign(slot_cap_, 0);
  slot_pinned_.assign(slot_cap_, 0);
  slot_names_.assign(slot_cap_, std::string());
  for (int32_t s = slot_cap_ - 1; s >= 0; --s) free_slots_.push_back(s);
}

GpuPinnedBackend::~GpuPinnedBackend() {
  if (interner_) sfkv_interner_destroy(interner_);
  sfkv_pool_destroy(pool_);
}

std::uint32_t GpuPinnedBackend::intern(const std::string& token) {
  auto [it, inserted] = intern_.emplace(token, static_cast<std::uint32_t>(intern_.size()));
  return it->second;
}

bool GpuPinnedBackend::reserve(int32_t slots, int32_t pin_blocks) {
  const int32_t s1 = std::max(slot_cap_, slots), b1 = std::max(pin_blocks_cap_, pin_blocks);
  if (s1 == slot_cap_ && b1 == pin_blocks_cap_) return true;
  const int rc = sfkv_pool_reserve(pool_, s1, b1, blocks_for(config_.cache_capacity_tokens, s1, b1));
  if (rc != SFKV_OK) {
    if (log_) log_(LogLevel::Error, "gpu backend " + descriptor_.ref + ": sfkv_pool_reserve failed: " + sfkv_last_error());
    return false;
  }
  for (int32_t s = s1 - 1; s >= slot_cap_; --s) free_slots_.push_back(s);
  slot_requests_.resize(s1, 0);
  slot_pinned_.resize(s1, 0);
  slot_names_.resize(s1);
  slot_cap_ = s1;
  pin_blocks_cap_ = b1;
  return true;
}

void GpuPinnedBackend::check(int rc, const char* what) const {
  if (rc != SFKV_OK)
    throw BackendError(std::string(what) + " failed (" + std::to_string(rc) + "): " + sfkv_last_error());
}

int32_t GpuPinnedBackend::find_slot(const std::string& workflow_id) const {
  auto it = slots_.find(workflow_id);
  return it == slots_.end() ? -1 : it->second;
}

int32_t GpuPinnedBackend::slot_for(const std::string& workflow_id) {
  auto it = slots_.find(workflow_id);
  if (it != slots_.end()) return it->second;
  if (free_slots_.empty() && !reserve(2 * slot_cap_, pin_blocks_cap_))
    throw BackendError("GpuPinnedBackend: cannot grow the workflow slots");
  const int32_t s = free_slots_.back();
  free_slots_.pop_back();
  slots_.emplace(workflow_id, s);
  slot_names_[s] = workflow_id;
  return s;
}

// A slot without a pin and without requests here carries no state: back to the free list (the
// pool already reads it as "no pin", pin_len = -1, exactly like a never-seen workflow).
void GpuPinnedBackend::maybe_release(int32_t slot) {
  if (slot < 0 || slot_requests_[slot] > 0 || slot_pinned_[slot]) return;
  slots_.erase(slot_names_[slot]);
  slot_names_[slot].clear();
  free_slots_.push_back(slot);
}

bool GpuPinnedBackend::has_capacity() const {
  return busy_ + static_cast<int>(pending_.size()) < config_.max_concurrency;
}

void GpuPinnedBackend::complete(CompletionRequest req, CompletionCallback cb) {
  ++stats_.completions;
  if (!req.metadata.workflow_id.empty()) ++slot_requests_[slot_for(req.metadata.workflow_id)];
  pending_.push_back(Pending{std::move(req), std::move(cb), loop_.now_ms()});
  pump();
}

void GpuPinnedBackend::pump() {
  if (interner_) {
    std::vector<Pending> batch;
    while (busy_ + static_cast<int>(batch.size()) < config_.max_concurrency && !pending_.empty()) {
      batch.push_back(std::move(pending_.front()));
      pending_.pop_front();
    }
    if (!batch.empty()) start_batch(std::move(batch));
    return;
  }
  while (busy_ < config_.max_concurrency && !pending_.empty()) {
    Pending p = std::move(pending_.front());
    pending_.pop_front();
    start(std::move(p));
  }
}

void GpuPinnedBackend::start_batch(std::vector<Pending> items) {
  const int64_t n = static_cast<int64_t>(items.size());
  // the requests' message contents as one text buffer (context_token_sequence reads content only)
  std::vector<int64_t> req_msg_off(n + 1, 0), msg_off(1, 0);
  std::vector<uint8_t> text;
  for (int64_t r = 0; r < n; ++r) {
    for (const auto& m : items[r].req.messages) {
      text.insert(text.end(), m.content.begin(), m.content.end());
      msg_off.push_back(static_cast<int64_t>(text.size()));
    }
    req_msg_off[r + 1] = static_cast<int64_t>(msg_off.size()) - 1;
  }
  const int64_t n_msg = static_cast<int64_t>(msg_off.size()) - 1;
  const int64_t cap = std::max<int64_t>((static_cast<int64_t>(text.size()) + n_msg + 1) / 2, 1);
  std::vector<int64_t> tok_off(n + 1, 0);
  std::vector<uint32_t> tok(static_cast<std::size_t>(cap));
  int64_t nt = 0;
  const int64_t text_bytes = static_cast<int64_t>(text.size());
  if (text.empty()) text.push_back(0);
  // the interner grows like the reference's strings: a full table / arena is reserved and the
  // batch (which changed nothing) retried; existing ids never change
  for (int attempt = 0;; ++attempt) {
    const int rc = sfkv_tokenize_batch(interner_, n, req_msg_off.data(), msg_off.data(), text.data(),
                                       tok_off.data(), tok.data(), cap, &nt);
    if (rc == SFKV_OK) break;
    if (rc != SFKV_EPOOL || attempt >= 16) check(rc, "sfkv_tokenize_batch");
    int64_t used = 0, acap = 0;
    int32_t lg = 0;
    check(sfkv_interner_arena(interner_, &used, &acap, &lg), "sfkv_interner_arena");
    check(sfkv_interner_reserve(interner_, lg + 1, std::max<int64_t>(2 * acap, used + 2 * text_bytes + 4096)),
          "sfkv_interner_reserve");
  }
  // one match for the requests that carry a workflow id (held slots since complete())
  std::vector<int32_t> slots(n, -1), wsl;
  std::vector<int64_t> woff(1, 0);
  std::vector<uint32_t> wtok;
  for (int64_t r = 0; r < n; ++r) {
    const std::string& wf = items[r].req.metadata.workflow_id;
    if (wf.empty()) continue;  // the empty workflow id never holds a pin (simulated_backend.cpp:125)
    slots[r] = find_slot(wf);
    wsl.push_back(slots[r]);
    wtok.insert(wtok.end(), tok.begin() + tok_off[r], tok.begin() + tok_off[r + 1]);
    woff.push_back(static_cast<int64_t>(wtok.size()));
  }
  std::vector<int64_t> M(wsl.size(), 0);
  if (!wsl.empty()) {
    if (wtok.empty()) wtok.push_back(0);
    check(sfkv_match_batch(pool_, static_cast<int64_t>(wsl.size()), wsl.data(), woff.data(), wtok.data(), M.data(),
                           nullptr),
          "sfkv_match_batch");
  }
  std::size_t k = 0;
  for (int64_t r = 0; r < n; ++r) {
    std::vector<uint32_t> ids(tok.begin() + tok_off[r], tok.begin() + tok_off[r + 1]);
    const long long m = slots[r] >= 0 ? M[k++] : 0;
    dispatch(std::move(items[r]), std::move(ids), m, slots[r]);
  }
}

ScriptedReply GpuPinnedBackend::reply_for(const CompletionRequest& req, int turn) const {
  const auto& rule = config_.output;
  const auto& ann = req.metadata.annotations;
  if (rule.kind == OutputRule::Kind::Scripted) return rule.script(req, turn);
  if (rule.kind == OutputRule::Kind::EchoAnnotation) {
    auto it = ann.find(rule.annotation_key);
    return {it == ann.end() ? std::string() : it->second, {}};
  }
  long long n = rule.constant_tokens;
  if (rule.kind == OutputRule::Kind::FromAnnotation) {
    auto it = ann.find(rule.annotation_key);
    if (it != ann.end()) n = std::max(0LL, std::stoll(it->second));
  }
  return {numbered_words(n), {}};
}

void GpuPinnedBackend::start(Pending item) {  // host tokenizer path (gpu_tokenizer = false)
  const std::string& wf = item.req.metadata.workflow_id;
  std::vector<std::uint32_t> ids;
  for (const auto& t : context_token_sequence(item.req.messages)) ids.push_back(intern(t));
  const int64_t off[2] = {0, static_cast<int64_t>(ids.size())};
  long long M = 0;
  int32_t slot = -1;
  if (!wf.empty()) {  // the empty workflow id never holds a pin (simulated_backend.cpp:125)
    slot = find_slot(wf);  // held since complete()
    int64_t m = 0;
    check(sfkv_match_batch(pool_, 1, &slot, off, ids.data(), &m, nullptr), "sfkv_match_batch");
    M = m;
  }
  dispatch(std::move(item), std::move(ids), M, slot);
}

// SimulatedBackend::start after the cache lookup (simulated_backend.cpp:81-133): reply, latency,
// completion event (which pins the prompt).
void GpuPinnedBackend::dispatch(Pending item, std::vector<std::uint32_t> ids, long long M, int32_t slot) {
  const double now = loop_.now_ms();
  const double queue_ms = now - item.arrival_ms;
  const std::string wf = item.req.metadata.workflow_id;
  const long long P = static_cast<long long>(ids.size());
  if (observer_) observer_(wf, item.req.metadata.stage_id, P, M);

  const int turn = turns_[{wf, item.req.metadata.stage_id}]++;
  ScriptedReply reply = reply_for(item.req, turn);
  long long O = count_tokens(reply.content);
  if (item.req.max_tokens > 0 && O > item.req.max_tokens) {
    auto words = tokenize_whitespace(reply.content);
    words.resize(static_cast<std::size_t>(item.req.max_tokens));
    std::string kept;
    for (const auto& w : words) {
      if (!kept.empty()) kept.push_back(' ');
      kept += w;
    }
    reply.content = std::move(kept);
    O = item.req.max_tokens;
  }
  if (O == 0 && !reply.tool_calls.empty()) O = 1;

  const double prefill = config_.fixed_overhead_ms +
                         config_.prefill_ms_per_token * static_cast<double>(P - M);
  const double decode = config_.decode_ms_per_token * static_cast<double>(O);
  CompletionResponse resp;
  resp.content = std::move(reply.content);
  resp.tool_calls = std::move(reply.tool_calls);
  resp.usage.prompt_tokens = P;
  resp.usage.completion_tokens = O;
  resp.usage.cached_prefix_tokens = M;
  resp.timing.queue_ms = queue_ms;
  resp.timing.ttft_ms = queue_ms + prefill;
  resp.timing.total_ms = resp.timing.ttft_ms + decode;
  ++busy_;
  stats_.prompt_tokens += P;
  stats_.completion_tokens += O;
  stats_.cached_prefix_tokens += M;

  loop_.schedule_in(prefill + decode, [this, slot, ids = std::move(ids), resp = std::move(resp),
                                       cb = std::move(item.cb), wf]() mutable {
    if (slot >= 0) {  // retain the served prompt (commit = pin_prompt, admission included)
      // Never throw out of the event loop: a failed commit is logged and leaves the old pin,
      // like a capacity rejection (the reference cannot fail here; this is a device error).
      const int64_t o2[2] = {0, static_cast<int64_t>(ids.size())};
      int32_t status = SFKV_PIN_REJECTED;
      const int32_t need = static_cast<int32_t>((o2[1] + SFKV_BLOCK_TOKENS - 1) / SFKV_BLOCK_TOKENS);
      int32_t grow = pin_blocks_cap_;
      while (grow < need) grow *= 2;
      int rc = SFKV_EPOOL;
      if (reserve(slot_cap_, grow))
        rc = sfkv_commit_batch(pool_, 1, &slot, o2, ids.data(), nullptr, nullptr, nullptr, &status);
      if (rc != SFKV_OK) {
        if (log_) log_(LogLevel::Error, "gpu backend " + descriptor_.ref + ": sfkv_commit_batch failed (" +
                                            std::to_string(rc) + "): " + sfkv_last_error());
      } else if (status == SFKV_PIN_ACCEPTED) {
        slot_pinned_[slot] = 1;
      } else if (log_) {
        log_(LogLevel::Warn, "gpu backend " + descriptor_.ref +
                                 ": cache capacity exceeded, prefix for workflow " + wf + " not pinned");
      }
      --slot_requests_[slot];
      maybe_release(slot);
    }
    --busy_;
    pump();
    cb(std::move(resp), nullptr);
    notify_capacity();
  });
}

long long GpuPinnedBackend::flush(const FlushScope& scope) {
  ++stats_.flush_calls;
  int64_t freed = 0;
  if (scope.all) {
    check(sfkv_flush(pool_, SFKV_FLUSH_ALL, &freed), "sfkv_flush");
    std::vector<int32_t> held;
    for (const auto& [name, s] : slots_) held.push_back(s);
    for (int32_t s : held) {
      slot_pinned_[s] = 0;
      maybe_release(s);
    }
    return freed;
  }
  const int32_t slot = find_slot(scope.workflow_id);
  if (slot < 0) return 0;
  check(sfkv_flush(pool_, slot, &freed), "sfkv_flush");
  slot_pinned_[slot] = 0;
  maybe_release(slot);
  return freed;
}

double GpuPinnedBackend::cache_utilization() const {
  double u = 0;
  check(sfkv_cache_utilization(pool_, &u), "sfkv_cache_utilization");
  return u;
}

bool GpuPinnedBackend::preserve(const std::string& workflow_id) {
  ++stats_.preserve_calls;
  const int32_t slot = find_slot(workflow_id);
  if (slot < 0) return false;
  int32_t has = 0;
  check(sfkv_preserve(pool_, slot, &has), "sfkv_preserve");
  return has != 0;
}

long long GpuPinnedBackend::pinned_token_count(const std::string& workflow_id) const {
  const int32_t slot = find_slot(workflow_id);
  if (slot < 0) return 0;
  int64_t n = 0;
  check(sfkv_pinned_token_count(pool_, slot, &n), "sfkv_pinned_token_count");
  return n;
}

long long GpuPinnedBackend::occupancy_tokens() const {
  sfkv_pool_stats s{};
  check(sfkv_stats(pool_, &s), "sfkv_stats");
  return s.occupancy_tokens;
}

std::uint64_t GpuPinnedBackend::capacity_rejections() const {
  sfkv_pool_stats s{};
  check(sfkv_stats(pool_, &s), "sfkv_stats");
  return s.capacity_rejections;
}

}  // namespace stageflow

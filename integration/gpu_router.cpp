// See gpu_router.hpp. Semantics follow the reference routers (orchestrator.cpp:8-57), map_threshold
// and map_one_bit_async (mapper.cpp:19-100) and reroute_on_overload (orchestrator.cpp:78-87); the
// decisions run in paper_2603_13605_b200/csrc/mm_map.cu (sfmap_threshold_batch, sfmap_cost_batch).
#include "gpu_router.hpp"

#include <cmath>
#include <stdexcept>
#include <vector>

namespace stageflow {

namespace {

void check(int rc, const char* what) {
  if (rc != 0) throw BackendError(std::string(what) + " failed (" + std::to_string(rc) + "): " + sfkv_last_error());
}

// Light (0) iff score <= threshold, on the device (mapper.cpp:30).
int gpu_threshold(int device, double score, double threshold) {
  int32_t choice = 0;
  check(sfmap_threshold_batch(device, 1, &score, threshold, &choice), "sfmap_threshold_batch");
  return choice;
}

}  // namespace

// reroute_on_overload as one row of the R x C mapper: candidate 0 = primary (cost 0, every other
// candidate cost 1, so the argmin is the primary), alternates listed in order; the reroute pass
// keeps the choice if its live depth is below the limit, else takes the first alternate that is.
std::string GpuReroute::apply(const std::string& primary) const {
  auto it = config_.reroute_alternates.find(primary);
  if (it == config_.reroute_alternates.end()) return primary;
  const auto& alts = it->second;
  const int32_t C = static_cast<int32_t>(alts.size()) + 1;
  std::vector<int64_t> P{0}, M(C, 0), O{0};
  std::vector<double> overhead(C, 1.0), prefill(C, 0.0), decode(C, 0.0), qpen(C, 0.0);
  overhead[0] = 0.0;
  std::vector<int32_t> alternates(static_cast<std::size_t>(C) * C, -1);
  for (int32_t j = 1; j < C; ++j) alternates[j - 1] = j;  // row of candidate 0
  std::vector<uint64_t> depth(C);
  depth[0] = depth_(primary);
  for (int32_t j = 1; j < C; ++j) depth[j] = depth_(alts[j - 1]);
  int32_t choice = 0;
  double cost = 0;
  check(sfmap_cost_batch(device_, 1, C, P.data(), M.data(), O.data(), overhead.data(), prefill.data(),
                         decode.data(), qpen.data(), alternates.data(), depth.data(),
                         static_cast<uint64_t>(config_.reroute_queue_limit), &choice, &cost),
        "sfmap_cost_batch");
  return choice == 0 ? primary : alts[choice - 1];
}

void GpuPlanRouter::route(const StageSpec& stage, const Context&, const RequestMetadata&, RouteCallback done) {
  auto it = plan_.assignments.find(stage.id);
  if (it == plan_.assignments.end()) throw UnknownStageError(stage.id);  // orchestrator.cpp:12
  auto prov = plan_.provenance.count(stage.id) ? plan_.provenance.at(stage.id) : MappingProvenance{};
  done(reroute_->apply(it->second), prov);
}

GpuThresholdRouter::GpuThresholdRouter(ScoreFn score_fn, double threshold, std::string light, std::string heavy,
                                       std::set<std::string> routable_stages,
                                       std::shared_ptr<const GpuReroute> reroute, int device)
    : score_fn_(std::move(score_fn)), threshold_(threshold), light_(std::move(light)), heavy_(std::move(heavy)),
      routable_(std::move(routable_stages)), reroute_(std::move(reroute)), device_(device) {}

void GpuThresholdRouter::route(const StageSpec& stage, const Context& ctx, const RequestMetadata&,
                               RouteCallback done) {
  if (!routable_.empty() && !routable_.count(stage.id)) {  // orchestrator.cpp:26-29
    done(reroute_->apply(stage.backend_ref), MappingProvenance{MappingProvenance::Kind::Explicit, {}, 0});
    return;
  }
  // map_threshold's argument checks and score (mapper.cpp:22-29)
  if (light_ == heavy_) throw std::invalid_argument("light and heavy refs must differ");
  if (!std::isfinite(threshold_)) throw std::invalid_argument("threshold must be finite");
  double score = 0;
  try {
    score = score_fn_(ctx);
  } catch (const std::exception& e) {
    throw ScoreFnFailedError(e.what());
  }
  const std::string& ref = gpu_threshold(device_, score, threshold_) == 0 ? light_ : heavy_;
  done(reroute_->apply(ref), MappingProvenance{MappingProvenance::Kind::Threshold, {}, score});
}

GpuOneBitRouter::GpuOneBitRouter(std::shared_ptr<Backend> classifier, std::string light, std::string heavy,
                                 std::set<std::string> routable_stages, std::string prompt_template,
                                 std::shared_ptr<const GpuReroute> reroute, int device)
    : classifier_(std::move(classifier)), light_(std::move(light)), heavy_(std::move(heavy)),
      routable_(std::move(routable_stages)), prompt_template_(std::move(prompt_template)),
      reroute_(std::move(reroute)), device_(device) {}

void GpuOneBitRouter::route(const StageSpec& stage, const Context& ctx, const RequestMetadata& meta,
                            RouteCallback done) {
  if (!routable_.empty() && !routable_.count(stage.id)) {  // orchestrator.cpp:46-49
    done(reroute_->apply(stage.backend_ref), MappingProvenance{MappingProvenance::Kind::Explicit, {}, 0});
    return;
  }
  // The classification call exactly as map_one_bit_async issues it (mapper.cpp:71-84): a
  // control-plane request without workflow / stage identity, so it never pins cache.
  CompletionRequest req;
  req.model = classifier_->descriptor().model;
  req.messages = make_user_context(build_classifier_prompt(ctx, prompt_template_));
  req.temperature = 0.0;
  req.max_tokens = 8;
  req.metadata = meta;
  req.metadata.workflow_id.clear();
  req.metadata.stage_id.clear();
  auto reroute = reroute_;
  const int device = device_;
  classifier_->complete(std::move(req), [done = std::move(done), light = light_, heavy = heavy_, reroute, device](
                                            CompletionResponse resp, std::exception_ptr ep) {
    ComplexityLabel label;  // fail-safe Complex (mapper.cpp:86-95)
    if (ep) {
      label.classifier_failed = true;
      try {
        std::rethrow_exception(ep);
      } catch (const std::exception& e) {
        label.raw_classifier_output = e.what();
      }
    } else {
      label = parse_complexity_label(resp.content);
    }
    // the one-bit label is the mapper's input: light iff bit (1 = complex) <= 0.5
    const double bit = label.value == Complexity::Simple ? 0.0 : 1.0;
    const std::string& ref = gpu_threshold(device, bit, 0.5) == 0 ? light : heavy;
    const std::string note = label.classifier_failed ? "classifier_failed"
                             : label.parse_failed    ? "unparseable"
                             : (label.value == Complexity::Simple ? "simple" : "complex");
    done(reroute->apply(ref), MappingProvenance{MappingProvenance::Kind::OneBit, note, 0});
  });
}

std::shared_ptr<StageRouter> make_gpu_router(const HarnessConfig& config, BackendRegistry& registry,
                                             const ValidatedWorkflow& wf, const Orchestrator& orch, int device) {
  auto reroute = std::make_shared<const GpuReroute>(
      config.orchestration, [&orch](const std::string& r) { return orch.queue_depth(r); }, device);
  switch (config.mapper.type) {
    case MapperConfig::Type::Explicit:
      return std::make_shared<GpuPlanRouter>(plan_explicit(wf, registry), reroute);
    case MapperConfig::Type::Threshold:
      return std::make_shared<GpuThresholdRouter>(
          [](const Context& ctx) { return static_cast<double>(count_context_tokens(ctx)); },
          config.mapper.threshold, config.mapper.light, config.mapper.heavy, config.mapper.stages, reroute,
          device);
    case MapperConfig::Type::OneBit: {
      auto classifier = registry.get(config.mapper.classifier);
      auto prompt = config.mapper.prompt_template.empty() ? std::string(kDefaultClassifierPrompt)
                                                          : config.mapper.prompt_template;
      return std::make_shared<GpuOneBitRouter>(std::move(classifier), config.mapper.light, config.mapper.heavy,
                                               config.mapper.stages, std::move(prompt), reroute, device);
    }
  }
  throw ConfigError("unhandled mapper type");
}

}  // namespace stageflow

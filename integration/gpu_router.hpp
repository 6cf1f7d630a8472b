// GpuRouter — the reference-side binding of the stage mapper (sfmap_*, include/sfkv.h).
//
// Drop-in `stageflow::StageRouter`s (reference: proj/include/stageflow/orchestrator.hpp:16-23)
// whose stage-to-backend decision runs on the B200:
//
//   GpuThresholdRouter  ThresholdRouter::route (orchestrator.cpp:24-32) -> map_threshold
//                       (mapper.cpp:19-31): the score (count_context_tokens, config.cpp:193, or
//                       any ScoreFn) goes to sfmap_threshold_batch; light iff score <= threshold
//   GpuOneBitRouter     OneBitRouter::route (orchestrator.cpp:40-57) -> map_one_bit_async
//                       (mapper.cpp:67-100): the classifier completion and the label parse
//                       (parse_complexity_label, mapper.cpp:49-65) stay on the host; the label is
//                       the mapper's 0/1 input (sfmap_threshold_batch over {0 simple, 1 complex})
//   GpuPlanRouter       PlanRouter::route (orchestrator.cpp:10-17) -> plan_explicit (mapper.cpp:8-17)
//
// Every router then applies reroute_on_overload (orchestrator.cpp:78-87) on the GPU before it
// answers: sfmap_cost_batch over the candidates {primary, alternates...} with the orchestrator's
// live queue depths (Orchestrator::queue_depth, orchestrator.cpp:481-484) and its queue limit.
// WorkflowRun::on_routed (orchestrator.cpp:241-251) re-applies the reference's reroute to the
// answer; that is the identity on a rerouted answer (an alternate is only chosen when its depth
// is below the limit, and the same depths are read in the same event), so the orchestrator's
// behaviour is exactly the reference's while the decision is made on the device.
//
// Reference-side code: compiled against the reference headers by oracle/Makefile only.
#pragma once

#include <functional>
#include <memory>
#include <set>
#include <string>

#include "sfkv.h"
#include "stageflow/config.hpp"
#include "stageflow/orchestrator.hpp"

namespace stageflow {

/// The GPU reroute shared by the routers (reroute_on_overload on the device).
class GpuReroute {
 public:
  using DepthFn = std::function<std::size_t(const std::string&)>;
  GpuReroute(OrchestratorConfig config, DepthFn depth, int device = 0)
      : config_(std::move(config)), depth_(std::move(depth)), device_(device) {}
  std::string apply(const std::string& primary) const;

 private:
  OrchestratorConfig config_;
  DepthFn depth_;
  int device_;
};

class GpuPlanRouter : public StageRouter {
 public:
  GpuPlanRouter(MappingPlan plan, std::shared_ptr<const GpuReroute> reroute)
      : plan_(std::move(plan)), reroute_(std::move(reroute)) {}
  void route(const StageSpec& stage, const Context& ctx, const RequestMetadata& meta,
             RouteCallback done) override;

 private:
  MappingPlan plan_;
  std::shared_ptr<const GpuReroute> reroute_;
};

class GpuThresholdRouter : public StageRouter {
 public:
  GpuThresholdRouter(ScoreFn score_fn, double threshold, std::string light, std::string heavy,
                     std::set<std::string> routable_stages, std::shared_ptr<const GpuReroute> reroute,
                     int device = 0);
  void route(const StageSpec& stage, const Context& ctx, const RequestMetadata& meta,
             RouteCallback done) override;

 private:
  ScoreFn score_fn_;
  double threshold_;
  std::string light_, heavy_;
  std::set<std::string> routable_;
  std::shared_ptr<const GpuReroute> reroute_;
  int device_;
};

class GpuOneBitRouter : public StageRouter {
 public:
  GpuOneBitRouter(std::shared_ptr<Backend> classifier, std::string light, std::string heavy,
                  std::set<std::string> routable_stages, std::string prompt_template,
                  std::shared_ptr<const GpuReroute> reroute, int device = 0);
  void route(const StageSpec& stage, const Context& ctx, const RequestMetadata& meta,
             RouteCallback done) override;

 private:
  std::shared_ptr<Backend> classifier_;
  std::string light_, heavy_;
  std::set<std::string> routable_;
  std::string prompt_template_;
  std::shared_ptr<const GpuReroute> reroute_;
  int device_;
};

/// make_router (config.cpp:186-207) with the GPU routers; `orch` supplies the live queue depths.
std::shared_ptr<StageRouter> make_gpu_router(const HarnessConfig& config, BackendRegistry& registry,
                                             const ValidatedWorkflow& wf, const Orchestrator& orch,
                                             int device = 0);

}  // namespace stageflow

// Deployment plan loader: strict JSON schema of the reference (config.hpp:
// 21-171; unknown keys are errors) plus two B200 keys: clock "device" and an
// optional top-level "placement" {stage: "cuda:N"}.
#pragma once
#include <string>

#include "omni/orchestrator.hpp"

namespace omni {

DeploymentPlan parse_plan_text(const std::string& json_text);
DeploymentPlan load_plan(const std::string& path);

}  // namespace omni

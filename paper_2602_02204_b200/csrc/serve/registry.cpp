#include "omni/registry.hpp"

namespace omni {

void EngineConfig::check() const {
  if (max_batch_tokens < 1 || max_resident_requests < 1 || kv_budget_tokens < 1 || workers < 1 ||
      prefill_chunk < 1)
    throw ConfigInvalid("engine config fields must be >= 1 (stage " + stage + ")");
  if (prefill_chunk > max_batch_tokens)
    throw ConfigInvalid("prefill_chunk exceeds max_batch_tokens (stage " + stage + ")");
}

}  // namespace omni

// Requests and the per-request write-once artifact store (reference
// context.hpp:14-124; SPEC.md RequestContext).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "omni/payload.hpp"

namespace omni {

using StageId = std::string;

struct Request {
  uint64_t request_id = 0;
  std::vector<uint8_t> prompt_tokens;  // ids in [1,255], non-empty
  uint32_t seed = 0;
  bool stream = false;
  uint64_t submitted_at_us = 0;
};

enum class RequestStatus { QUEUED, RUNNING, STREAMING, DONE, FAILED };
const char* status_name(RequestStatus s);
bool status_transition_allowed(RequestStatus from, RequestStatus to);

class RequestContext {
 public:
  RequestContext() = default;
  explicit RequestContext(uint64_t id) : id_(id) {}

  uint64_t request_id() const { return id_; }
  RequestStatus status() const { return status_; }
  void set_status(RequestStatus next);
  const StageId& current_stage() const { return stage_; }
  void set_current_stage(StageId s) { stage_ = std::move(s); }

  // Write-once: identical bytes are a no-op, different bytes a WriteConflict.
  void put(const std::string& key, Payload p);
  const Payload& get(const std::string& key) const;
  bool has(const std::string& key) const { return store_.count(key) != 0; }
  const std::map<std::string, Payload>& store() const { return store_; }

  std::vector<uint8_t> serialize() const;
  static RequestContext deserialize(std::span<const uint8_t> buf);

 private:
  uint64_t id_ = 0;
  RequestStatus status_ = RequestStatus::QUEUED;
  StageId stage_;
  std::map<std::string, Payload> store_;
};

}  // namespace omni

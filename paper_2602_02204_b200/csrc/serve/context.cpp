#include "omni/context.hpp"

namespace omni {

const char* status_name(RequestStatus s) {
  static const char* names[] = {"QUEUED", "RUNNING", "STREAMING", "DONE", "FAILED"};
  const int i = static_cast<int>(s);
  return i >= 0 && i < 5 ? names[i] : "?";
}

// QUEUED -> RUNNING -> (STREAMING) -> DONE | FAILED   (context.hpp:22-49)
bool status_transition_allowed(RequestStatus from, RequestStatus to) {
  using S = RequestStatus;
  if (from == S::QUEUED) return to == S::RUNNING;
  if (from == S::RUNNING) return to == S::STREAMING || to == S::DONE || to == S::FAILED;
  if (from == S::STREAMING) return to == S::DONE || to == S::FAILED;
  return false;
}

void RequestContext::set_status(RequestStatus next) {
  if (!status_transition_allowed(status_, next))
    throw OmniError(std::string("illegal status transition ") + status_name(status_) + " -> " +
                    status_name(next));
  status_ = next;
}

void RequestContext::put(const std::string& key, Payload p) {
  if (key.empty()) throw OmniError("ctx_put: empty key");
  auto [it, inserted] = store_.try_emplace(key, std::move(p));
  if (!inserted && !(it->second == p)) throw WriteConflict(key);
}

const Payload& RequestContext::get(const std::string& key) const {
  auto it = store_.find(key);
  if (it == store_.end()) throw MissingKey(key);
  return it->second;
}

std::vector<uint8_t> RequestContext::serialize() const {
  std::vector<uint8_t> out;
  wire::put_u64(out, id_);
  wire::put_u32(out, static_cast<uint32_t>(store_.size()));
  for (const auto& [k, v] : store_) {
    wire::put_str(out, k);
    const auto blob = encode_payload(v);
    wire::put_u32(out, static_cast<uint32_t>(blob.size()));
    out.insert(out.end(), blob.begin(), blob.end());
  }
  return out;
}

RequestContext RequestContext::deserialize(std::span<const uint8_t> buf) {
  wire::Reader r{buf};
  RequestContext ctx(r.u64());
  const uint32_t n = r.u32();
  for (uint32_t i = 0; i < n; ++i) {
    std::string k = r.str();
    const uint32_t len = r.u32();
    const auto blob = r.raw(len);
    ctx.store_.emplace(std::move(k), decode_payload(blob));
  }
  return ctx;
}

}  // namespace omni

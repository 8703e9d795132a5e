// Error tree of the stage-graph runtime. Same class names and meaning as the
// reference (errors.hpp:8-84) so existing catch sites port unchanged; each
// maps onto an omni_status code at the C ABI.
#pragma once
#include <stdexcept>
#include <string>

namespace omni {

struct OmniError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define OMNI_DECLARE_ERROR(Name) \
  struct Name : OmniError {      \
    using OmniError::OmniError;  \
  }

struct WriteConflict : OmniError {
  explicit WriteConflict(const std::string& key) : OmniError("write conflict on key: " + key) {}
};
struct MissingKey : OmniError {
  explicit MissingKey(const std::string& key) : OmniError("missing key: " + key) {}
};
OMNI_DECLARE_ERROR(TimeoutError);
OMNI_DECLARE_ERROR(TransportDown);
OMNI_DECLARE_ERROR(RegionFull);
OMNI_DECLARE_ERROR(ProtocolViolation);
OMNI_DECLARE_ERROR(AlreadyOpen);
OMNI_DECLARE_ERROR(BadDtype);
OMNI_DECLARE_ERROR(RejectedTooLarge);
OMNI_DECLARE_ERROR(ConfigInvalid);
OMNI_DECLARE_ERROR(PortInUse);
OMNI_DECLARE_ERROR(EngineSpawnFailed);
OMNI_DECLARE_ERROR(Overloaded);
OMNI_DECLARE_ERROR(Rejected);
OMNI_DECLARE_ERROR(TransferFnError);
OMNI_DECLARE_ERROR(IncompleteRecord);
OMNI_DECLARE_ERROR(NoAudio);
OMNI_DECLARE_ERROR(ForwardError);
// B200 additions: device-side failures surfaced through libomni_dev.
OMNI_DECLARE_ERROR(DeviceError);

#undef OMNI_DECLARE_ERROR

}  // namespace omni

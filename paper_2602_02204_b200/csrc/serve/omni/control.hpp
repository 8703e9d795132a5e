// Control frames of the connector data plane (reference control.hpp:10-117).
//
// Same frame layout as the reference: u32 LE body length, u8 message kind,
// body = key str, request_id u64, edge str, seq u32, locator kind u8, locator
// body. The reference's locator kinds INLINE / SHM / TCP keep their tags and
// bodies byte for byte; the B200 backend adds kind DEVICE (tag 3): the payload
// blob stays in HBM and the frame carries where it is plus the small host
// sideband the control plane needs without touching device memory:
//
//   DEVICE body: device u32 | arena u64 | offset u64 | length u64 |
//                payload header (dtype u8, rank u8, dims u32 LE ...) |
//                n_tokens u32 | tokens i32 LE ...
//
// `arena` 0 means `offset` is an address in the sender's own address space
// (in-process DEVICE transport, peer GPUs included: one process maps every
// device); a non-zero arena is the id of a CUDA-IPC-exported arena and
// `offset` is relative to its base (multi-process placement, ipc_arena.hpp).
#pragma once
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "omni/errors.hpp"
#include "omni/payload.hpp"

namespace omni {

struct Locator {
  enum class Kind : uint8_t { INLINE = 0, SHM = 1, TCP = 2, DEVICE = 3 };
  Kind kind = Kind::INLINE;
  std::vector<uint8_t> inline_bytes;  // INLINE
  std::string shm_region;             // SHM
  uint64_t shm_offset = 0;
  uint64_t shm_length = 0;
  uint64_t tcp_stream_id = 0;  // TCP
  // DEVICE
  uint32_t device = 0;
  uint64_t arena = 0;
  uint64_t offset = 0;
  uint64_t length = 0;
  Dtype dtype = Dtype::U8;
  std::vector<uint32_t> shape;
  std::vector<int32_t> tokens;

  bool operator==(const Locator&) const = default;
};

struct ControlMessage {
  enum class Kind : uint8_t { PUT_NOTICE = 0, CHUNK_NOTICE = 1, EOS = 2, HANDOFF = 3, ACK = 4 };
  Kind kind = Kind::PUT_NOTICE;
  std::string key;          // PUT_NOTICE / HANDOFF / ACK
  uint64_t request_id = 0;  // CHUNK_NOTICE / EOS
  std::string edge;         // CHUNK_NOTICE / EOS
  uint32_t seq = 0;         // CHUNK_NOTICE / EOS
  Locator locator;

  bool operator==(const ControlMessage&) const = default;
};

std::vector<uint8_t> encode_control_frame(const ControlMessage& m);
// Throws ProtocolViolation on a bad kind, a length mismatch, a short read or
// trailing bytes, BadDtype on a bad payload tag inside a DEVICE locator.
ControlMessage decode_control_frame(std::span<const uint8_t> frame);

// DEVICE locator <-> device payload (the host view of a blob in HBM).
Locator device_locator(const Payload& p);
Payload payload_from_locator(const Locator& l);

}  // namespace omni

// Typed inter-stage payloads and their wire codec.
//
// Wire layout is the reference's (payload.hpp:142-166): [dtype u8][rank u8]
// [dims u32 LE ...][raw little-endian bytes]. B200 addition: a payload may be
// DEVICE-resident — its encoded blob lives in a device arena (`dev`) and only
// the locator plus a host mirror of the token column travel through the
// control plane ("the host control plane carries only locators").
#pragma once
#include <array>
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "omni/errors.hpp"

namespace omni {

enum class Dtype : uint8_t { U8 = 0, I32 = 1, FIX16 = 2 };

size_t dtype_width(Dtype d);

struct DeviceRef {
  int32_t device = -1;   // CUDA ordinal; -1 = host payload
  uint64_t blob = 0;     // device address of the encoded blob (header + body)
  uint64_t nbytes = 0;   // encoded length
  uint64_t arena = 0;    // 0: `blob` is an address; else CUDA-IPC arena id, `blob` an offset
  bool valid() const { return device >= 0; }
};

struct Payload {
  Dtype dtype = Dtype::U8;
  std::vector<uint32_t> shape;
  std::vector<uint8_t> bytes;        // host body (empty for device payloads)
  DeviceRef dev;                     // device-resident encoded blob
  std::vector<int32_t> host_tokens;  // device payloads: mirror of column 0

  size_t element_count() const;
  bool is_device() const { return dev.valid(); }
  bool operator==(const Payload& o) const {
    return dtype == o.dtype && shape == o.shape && bytes == o.bytes && dev.blob == o.dev.blob &&
           dev.device == o.dev.device && dev.arena == o.dev.arena && dev.nbytes == o.dev.nbytes &&
           host_tokens == o.host_tokens;
  }
  bool size_consistent() const { return is_device() || bytes.size() == element_count() * dtype_width(dtype); }

  static Payload from_u8(std::vector<uint8_t> data);
  static Payload from_i32(std::span<const int32_t> data);
  std::vector<int32_t> as_i32() const;

  // Device address of element (row, col) of a rank-2 FIX16 device payload.
  uint64_t device_elem(uint32_t row, uint32_t col) const;
};

std::vector<uint8_t> encode_payload(const Payload& p);
Payload decode_payload(std::span<const uint8_t> blob);
uint64_t payload_header_bytes(size_t rank);

/// Fixed-point hidden state of the reference mock pipeline (8 nibbles).
struct HiddenState {
  std::array<uint8_t, 8> values{};
  bool operator==(const HiddenState&) const = default;
  int component_sum() const {
    int s = 0;
    for (auto v : values) s += v;
    return s;
  }
};

namespace wire {
void put_u32(std::vector<uint8_t>& out, uint32_t v);
void put_u64(std::vector<uint8_t>& out, uint64_t v);
void put_str(std::vector<uint8_t>& out, const std::string& s);
struct Reader {
  std::span<const uint8_t> data;
  size_t pos = 0;
  uint8_t u8();
  uint32_t u32();
  uint64_t u64();
  std::vector<uint8_t> raw(size_t n);
  std::string str();
  bool done() const { return pos == data.size(); }
};
}  // namespace wire

uint64_t fnv1a64(std::span<const uint8_t> data, uint64_t h = 1469598103934665603ull);

}  // namespace omni

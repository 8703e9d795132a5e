// Payload codec (reference wire layout payload.hpp:142-166) + device refs.
#include "omni/payload.hpp"

#include <numeric>

namespace omni {

size_t dtype_width(Dtype d) {
  switch (d) {
    case Dtype::U8: return 1;
    case Dtype::I32: return 4;
    case Dtype::FIX16: return 2;
  }
  throw BadDtype("unknown dtype tag");
}

size_t Payload::element_count() const {
  size_t n = 1;
  for (uint32_t s : shape) n *= s;
  return n;
}

Payload Payload::from_u8(std::vector<uint8_t> data) {
  Payload p;
  p.dtype = Dtype::U8;
  p.shape = {static_cast<uint32_t>(data.size())};
  p.bytes = std::move(data);
  return p;
}

Payload Payload::from_i32(std::span<const int32_t> data) {
  Payload p;
  p.dtype = Dtype::I32;
  p.shape = {static_cast<uint32_t>(data.size())};
  p.bytes.resize(data.size() * 4);
  uint8_t* o = p.bytes.data();
  for (int32_t v : data) {
    const uint32_t u = static_cast<uint32_t>(v);
    *o++ = static_cast<uint8_t>(u);
    *o++ = static_cast<uint8_t>(u >> 8);
    *o++ = static_cast<uint8_t>(u >> 16);
    *o++ = static_cast<uint8_t>(u >> 24);
  }
  return p;
}

std::vector<int32_t> Payload::as_i32() const {
  if (dtype != Dtype::I32) throw BadDtype("payload is not I32");
  if (is_device()) throw BadDtype("device payload has no host I32 view");
  std::vector<int32_t> out(bytes.size() / 4);
  const uint8_t* b = bytes.data();
  for (auto& v : out) {
    v = static_cast<int32_t>(uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) |
                             (uint32_t(b[3]) << 24));
    b += 4;
  }
  return out;
}

uint64_t payload_header_bytes(size_t rank) { return 2 + 4 * rank; }

uint64_t Payload::device_elem(uint32_t row, uint32_t col) const {
  if (!is_device() || shape.size() != 2) throw BadDtype("not a rank-2 device payload");
  const uint64_t w = dtype_width(dtype);
  return dev.blob + payload_header_bytes(2) + (uint64_t(row) * shape[1] + col) * w;
}

namespace wire {
void put_u32(std::vector<uint8_t>& out, uint32_t v) {
  for (int i = 0; i < 4; ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& out, uint64_t v) {
  put_u32(out, static_cast<uint32_t>(v));
  put_u32(out, static_cast<uint32_t>(v >> 32));
}
void put_str(std::vector<uint8_t>& out, const std::string& s) {
  put_u32(out, static_cast<uint32_t>(s.size()));
  out.insert(out.end(), s.begin(), s.end());
}
uint8_t Reader::u8() {
  if (pos + 1 > data.size()) throw ProtocolViolation("short read");
  return data[pos++];
}
uint32_t Reader::u32() {
  if (pos + 4 > data.size()) throw ProtocolViolation("short read");
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= uint32_t(data[pos + i]) << (8 * i);
  pos += 4;
  return v;
}
uint64_t Reader::u64() {
  const uint64_t lo = u32();
  return lo | (uint64_t(u32()) << 32);
}
std::vector<uint8_t> Reader::raw(size_t n) {
  if (pos + n > data.size()) throw ProtocolViolation("short read");
  std::vector<uint8_t> v(data.begin() + pos, data.begin() + pos + n);
  pos += n;
  return v;
}
std::string Reader::str() {
  const uint32_t n = u32();
  auto b = raw(n);
  return std::string(b.begin(), b.end());
}
}  // namespace wire

std::vector<uint8_t> encode_payload(const Payload& p) {
  if (p.is_device()) throw BadDtype("device payload: encoded blob lives in device memory");
  std::vector<uint8_t> out;
  out.reserve(payload_header_bytes(p.shape.size()) + p.bytes.size());
  out.push_back(static_cast<uint8_t>(p.dtype));
  out.push_back(static_cast<uint8_t>(p.shape.size()));
  for (uint32_t d : p.shape) wire::put_u32(out, d);
  out.insert(out.end(), p.bytes.begin(), p.bytes.end());
  return out;
}

Payload decode_payload(std::span<const uint8_t> blob) {
  wire::Reader r{blob};
  Payload p;
  const uint8_t tag = r.u8();
  if (tag > 2) throw BadDtype("bad dtype tag in payload header");
  p.dtype = static_cast<Dtype>(tag);
  p.shape.resize(r.u8());
  for (auto& d : p.shape) d = r.u32();
  p.bytes = r.raw(p.element_count() * dtype_width(p.dtype));
  if (!r.done()) throw ProtocolViolation("trailing bytes after payload");
  return p;
}

uint64_t fnv1a64(std::span<const uint8_t> data, uint64_t h) {
  for (uint8_t b : data) {
    h ^= b;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace omni

// Control-frame codec (reference control.hpp:56-117) + the DEVICE locator.
#include "omni/control.hpp"

namespace omni {

namespace {
constexpr uint8_t kMaxMsgKind = 4;
constexpr uint8_t kMaxLocKind = 3;
}  // namespace

std::vector<uint8_t> encode_control_frame(const ControlMessage& m) {
  std::vector<uint8_t> body;
  wire::put_str(body, m.key);
  wire::put_u64(body, m.request_id);
  wire::put_str(body, m.edge);
  wire::put_u32(body, m.seq);
  const Locator& l = m.locator;
  body.push_back(static_cast<uint8_t>(l.kind));
  switch (l.kind) {
    case Locator::Kind::INLINE:
      wire::put_u32(body, static_cast<uint32_t>(l.inline_bytes.size()));
      body.insert(body.end(), l.inline_bytes.begin(), l.inline_bytes.end());
      break;
    case Locator::Kind::SHM:
      wire::put_str(body, l.shm_region);
      wire::put_u64(body, l.shm_offset);
      wire::put_u64(body, l.shm_length);
      break;
    case Locator::Kind::TCP:
      wire::put_u64(body, l.tcp_stream_id);
      break;
    case Locator::Kind::DEVICE:
      wire::put_u32(body, l.device);
      wire::put_u64(body, l.arena);
      wire::put_u64(body, l.offset);
      wire::put_u64(body, l.length);
      body.push_back(static_cast<uint8_t>(l.dtype));
      body.push_back(static_cast<uint8_t>(l.shape.size()));
      for (uint32_t d : l.shape) wire::put_u32(body, d);
      wire::put_u32(body, static_cast<uint32_t>(l.tokens.size()));
      for (int32_t t : l.tokens) wire::put_u32(body, static_cast<uint32_t>(t));
      break;
  }
  std::vector<uint8_t> out;
  out.reserve(5 + body.size());
  wire::put_u32(out, static_cast<uint32_t>(body.size()));
  out.push_back(static_cast<uint8_t>(m.kind));
  out.insert(out.end(), body.begin(), body.end());
  return out;
}

ControlMessage decode_control_frame(std::span<const uint8_t> frame) {
  wire::Reader r{frame};
  const uint32_t len = r.u32();
  const uint8_t kind = r.u8();
  if (kind > kMaxMsgKind) throw ProtocolViolation("bad control message kind");
  if (frame.size() != 5ull + len) throw ProtocolViolation("frame length mismatch");
  ControlMessage m;
  m.kind = static_cast<ControlMessage::Kind>(kind);
  m.key = r.str();
  m.request_id = r.u64();
  m.edge = r.str();
  m.seq = r.u32();
  const uint8_t lk = r.u8();
  if (lk > kMaxLocKind) throw ProtocolViolation("bad locator kind");
  Locator& l = m.locator;
  l.kind = static_cast<Locator::Kind>(lk);
  switch (l.kind) {
    case Locator::Kind::INLINE:
      l.inline_bytes = r.raw(r.u32());
      break;
    case Locator::Kind::SHM:
      l.shm_region = r.str();
      l.shm_offset = r.u64();
      l.shm_length = r.u64();
      break;
    case Locator::Kind::TCP:
      l.tcp_stream_id = r.u64();
      break;
    case Locator::Kind::DEVICE: {
      l.device = r.u32();
      l.arena = r.u64();
      l.offset = r.u64();
      l.length = r.u64();
      const uint8_t tag = r.u8();
      if (tag > 2) throw BadDtype("bad dtype tag in device locator");
      l.dtype = static_cast<Dtype>(tag);
      l.shape.resize(r.u8());
      uint64_t elems = 1;
      bool overflow = false;
      for (auto& d : l.shape) {
        d = r.u32();
        overflow = overflow || __builtin_mul_overflow(elems, (uint64_t)d, &elems);
      }
      uint64_t body = 0;
      overflow = overflow || __builtin_mul_overflow(elems, (uint64_t)dtype_width(l.dtype), &body);
      // the blob must hold exactly header + body (payload.hpp:142-166)
      if (overflow || l.length != payload_header_bytes(l.shape.size()) + body)
        throw ProtocolViolation("device locator length does not match its shape");
      const uint32_t nt = r.u32();
      if (nt > (frame.size() - r.pos) / 4) throw ProtocolViolation("short read");
      l.tokens.resize(nt);
      for (auto& t : l.tokens) t = static_cast<int32_t>(r.u32());
      break;
    }
  }
  if (!r.done()) throw ProtocolViolation("trailing bytes in control frame");
  return m;
}

Locator device_locator(const Payload& p) {
  if (!p.is_device()) throw BadDtype("device_locator: host payload");
  Locator l;
  l.kind = Locator::Kind::DEVICE;
  l.device = static_cast<uint32_t>(p.dev.device);
  l.arena = p.dev.arena;
  l.offset = p.dev.blob;
  l.length = p.dev.nbytes;
  l.dtype = p.dtype;
  l.shape = p.shape;
  l.tokens = p.host_tokens;
  return l;
}

Payload payload_from_locator(const Locator& l) {
  if (l.kind != Locator::Kind::DEVICE) throw ProtocolViolation("not a device locator");
  Payload p;
  p.dtype = l.dtype;
  p.shape = l.shape;
  p.dev.device = static_cast<int32_t>(l.device);
  p.dev.arena = l.arena;
  p.dev.blob = l.offset;
  p.dev.nbytes = l.length;
  p.host_tokens = l.tokens;
  return p;
}

}  // namespace omni

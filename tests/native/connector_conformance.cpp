// Connector + control-frame conformance of the B200 control plane
// (libomni_serve), restating the reference's own tests against it:
//   test_connector.cpp:31-170        keyed put/get, streams, protocol violations, cleanup
//   acceptance.cpp:194-266           sizes 1 B .. 16 MiB bit-exact, 10,000 fuzzed schedules
//   test_payload_context.cpp:17-164  payload + control-frame codecs, fuzz, garbage
// Every stream case runs twice: with host payloads (INPROC, the reference's
// path) and with DEVICE payloads (locators of blobs in HBM, queued as encoded
// DEVICE control frames). The connector never dereferences a device address,
// so the DEVICE cases run without a GPU on synthetic locators.
//
// Built and run by tests/test_connector_conformance.py; prints one line per
// case and "ALL OK <n>" at the end; exit code 1 on the first failure.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "omni/connector.hpp"
#include "omni/control.hpp"
#include "omni/context.hpp"

using namespace omni;

static int g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, Err)                                               \
  do {                                                                           \
    ++g_checks;                                                                  \
    bool caught_ = false;                                                        \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const Err&) {                                                       \
      caught_ = true;                                                            \
    } catch (const std::exception& e_) {                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s threw the wrong type: %s\n", __FILE__, \
                   __LINE__, #expr, e_.what());                                  \
      std::exit(1);                                                              \
    }                                                                            \
    if (!caught_) {                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s did not throw %s\n", __FILE__,         \
                   __LINE__, #expr, #Err);                                       \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)
#define CHECK_NOTHROW(expr)                                                      \
  do {                                                                           \
    ++g_checks;                                                                  \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const std::exception& e_) {                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s threw %s\n", __FILE__, __LINE__,       \
                   #expr, e_.what());                                            \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

namespace {

enum class Mode { HOST, DEVICE };
const char* mode_name(Mode m) { return m == Mode::HOST ? "host" : "device"; }

Payload host_payload(size_t bytes, uint32_t salt) {
  Payload p;
  p.dtype = Dtype::U8;
  p.shape = {static_cast<uint32_t>(bytes)};
  p.bytes.resize(bytes);
  std::mt19937 rng(salt);
  for (auto& b : p.bytes) b = static_cast<uint8_t>(rng());
  return p;
}

// A FIX16 {rows, 1+d} hidden-row blob somewhere in a (synthetic) device arena,
// with the token column mirrored on the host -- the shape the Thinker's pack
// kernel produces (reference_pipeline.hpp:113-123).
Payload device_payload(uint32_t rows, uint32_t d, uint32_t salt, int device = 1) {
  std::mt19937_64 rng(salt);
  Payload p;
  p.dtype = Dtype::FIX16;
  p.shape = {rows, 1 + d};
  p.dev.device = device;
  p.dev.blob = (rng() & 0xffffffffffull) << 8;
  p.dev.nbytes = payload_header_bytes(2) + uint64_t(rows) * (1 + d) * 2;
  for (uint32_t r = 0; r < rows; ++r) p.host_tokens.push_back(static_cast<int32_t>(rng() % 255 + 1));
  return p;
}

Payload payload_of(Mode m, size_t bytes, uint32_t salt) {
  return m == Mode::HOST ? host_payload(bytes, salt) : device_payload(static_cast<uint32_t>(bytes % 9), 16, salt);
}

int g_cases = 0;
void run(const std::string& name, const std::function<void()>& fn) {
  fn();
  ++g_cases;
  std::printf("ok %s\n", name.c_str());
}

// ---- test_connector.cpp:31-170 ------------------------------------------

void keyed(Mode md) {
  const std::string tag = mode_name(md);
  run("put then get round-trips [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    ConnectorKey k{1, "a->b", "x", 0};
    Payload p = md == Mode::HOST ? Payload::from_i32(std::vector<int32_t>{1, 2, 3}) : device_payload(3, 8, 1);
    conn.put(k, p);
    CHECK(conn.get(k, 100) == p);
  });
  run("put is write-once: idempotent same bytes, conflict otherwise [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    ConnectorKey k{1, "a->b", "x", 0};
    Payload p = payload_of(md, 4, 1), q = payload_of(md, 4, 2);
    conn.put(k, p);
    CHECK_NOTHROW(conn.put(k, p));
    CHECK_THROWS_AS(conn.put(k, q), WriteConflict);
  });
  run("get before put blocks until the value lands [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    ConnectorKey k{1, "a->b", "x", 0};
    Payload p = payload_of(md, 42, 3);
    std::thread writer([&] {
      std::this_thread::sleep_for(std::chrono::milliseconds(30));
      conn.put(k, p);
    });
    CHECK(conn.get(k, 2000) == p);
    writer.join();
  });
  run("get times out on a missing key [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    CHECK_THROWS_AS(conn.get(ConnectorKey{1, "a->b", "missing", 0}, 30), TimeoutError);
  });
}

void streams(Mode md) {
  const std::string tag = mode_name(md);
  run("streams deliver chunks exactly once, in order [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto send = conn.open_stream(1);
    auto recv = conn.subscribe(1);
    std::vector<Payload> sent;
    for (uint32_t i = 0; i < 5; ++i) {
      StreamChunk c;
      c.request_id = 1;
      c.seq = i;
      c.payload = payload_of(md, 4 + i, i + 1);
      c.eos = (i == 4);
      sent.push_back(c.payload);
      send.send(c);
    }
    for (uint32_t i = 0; i < 5; ++i) {
      auto c = recv.try_recv();
      CHECK(c.has_value());
      CHECK(c->seq == i);
      CHECK(c->payload == sent[i]);
      CHECK(c->eos == (i == 4));
      CHECK(c->from == "a" && c->to == "b");
    }
    CHECK(!recv.try_recv().has_value());
    if (md == Mode::DEVICE) CHECK(conn.frames_encoded() == 5);
  });
  run("late subscriber still sees buffered chunks [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto send = conn.open_stream(1);
    StreamChunk c;
    c.request_id = 1;
    c.seq = 0;
    c.payload = payload_of(md, 9, 9);
    c.eos = true;
    send.send(c);
    auto recv = conn.subscribe(1);
    auto got = recv.try_recv();
    CHECK(got.has_value());
    CHECK(got->payload == c.payload);
    CHECK(got->eos);
  });
  run("protocol violations: bad seq, send after eos, double open [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto send = conn.open_stream(1);
    CHECK_THROWS_AS(conn.open_stream(1), AlreadyOpen);
    auto recv = conn.subscribe(1);
    CHECK_THROWS_AS(conn.subscribe(1), AlreadyOpen);
    StreamChunk c;
    c.request_id = 1;
    c.seq = 5;  // expected 0
    c.payload = payload_of(md, 3, 1);
    CHECK_THROWS_AS(send.send(c), ProtocolViolation);
    c.seq = 0;
    c.eos = true;
    send.send(c);
    StreamChunk after;
    after.request_id = 1;
    after.seq = 1;
    after.payload = payload_of(md, 3, 2);
    CHECK_THROWS_AS(send.send(after), ProtocolViolation);
    // the rejected chunks left no trace: exactly the eos chunk is delivered
    auto got = recv.try_recv();
    CHECK(got.has_value() && got->seq == 0 && got->eos);
    CHECK(!recv.try_recv().has_value());
  });
  run("blocking recv honors its timeout [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    conn.open_stream(1);
    auto recv = conn.subscribe(1);
    CHECK_THROWS_AS(recv.recv(30), TimeoutError);
  });
  run("blocking recv wakes on a send from another thread [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto send = conn.open_stream(1);
    auto recv = conn.subscribe(1);
    StreamChunk c;
    c.request_id = 1;
    c.payload = payload_of(md, 5, 5);
    c.eos = true;
    std::thread writer([&] {
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
      send.send(c);
    });
    auto got = recv.recv(2000);
    CHECK(got.payload == c.payload && got.eos);
    writer.join();
  });
  run("cleanup is idempotent and frees stream state [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto send = conn.open_stream(1);
    StreamChunk c;
    c.request_id = 1;
    c.seq = 0;
    c.payload = payload_of(md, 64, 7);
    send.send(c);
    Payload k = payload_of(md, 32, 8);
    conn.put(ConnectorKey{1, "a->b", "k", 0}, k);
    const uint64_t expect = (md == Mode::HOST ? 2 + 4 + 64 : c.payload.dev.nbytes) +
                            (md == Mode::HOST ? 2 + 4 + 32 : k.dev.nbytes);
    CHECK(conn.cleanup(1) == expect);
    CHECK(conn.cleanup(1) == 0);  // second cleanup is a no-op
    // a fresh stream for the same request id opens again after cleanup
    CHECK_NOTHROW(conn.open_stream(1));
    CHECK_NOTHROW(conn.subscribe(1));
  });
  run("cleanup of one request leaves the others intact [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    auto s1 = conn.open_stream(1);
    auto s2 = conn.open_stream(2);
    auto r2 = conn.subscribe(2);
    StreamChunk c;
    c.payload = payload_of(md, 6, 1);
    c.request_id = 1;
    s1.send(c);
    c.request_id = 2;
    s2.send(c);
    conn.cleanup(1);
    auto got = r2.try_recv();
    CHECK(got.has_value() && got->request_id == 2 && got->payload == c.payload);
  });
}

// ---- acceptance.cpp:194-266 ---------------------------------------------

void acceptance(Mode md) {
  const std::string tag = mode_name(md);
  run("bit-exact round trip at 1 B / 4 KiB / 64 KiB / 16 MiB [" + tag + "]", [&] {
    Connector conn("a->b", TransportConfig{});
    uint32_t salt = 1;
    for (size_t sz : {size_t(1), size_t(4096), size_t(64 * 1024), size_t(16 * 1024 * 1024)}) {
      Payload p;
      if (md == Mode::HOST) {
        p = host_payload(sz, salt);
      } else {  // a blob of exactly sz body bytes: U8 {sz}
        p.dtype = Dtype::U8;
        p.shape = {static_cast<uint32_t>(sz)};
        p.dev.device = 3;
        p.dev.blob = 0x7f0000000000ull + salt * 4096;
        p.dev.nbytes = payload_header_bytes(1) + sz;
      }
      ConnectorKey k{1, "a->b", "sz" + std::to_string(sz), 0};
      conn.put(k, p);
      CHECK(conn.get(k, 10000) == p);
      ++salt;
    }
    conn.cleanup(1);
  });
  run("exactly-once in-order delivery over 10000 fuzzed schedules [" + tag + "]", [&] {
    std::mt19937 rng(777);
    Connector conn("a->b", TransportConfig{});
    for (int schedule = 0; schedule < 10000; ++schedule) {
      const uint64_t rid = schedule + 1;
      auto send = conn.open_stream(rid);
      auto recv = conn.subscribe(rid);
      const uint32_t n = rng() % 12 + 1;
      uint32_t sent = 0, received = 0;
      std::vector<Payload> expect;
      while (received < n) {
        const bool do_send = sent < n && (received == sent || rng() % 2);
        if (do_send) {
          StreamChunk c;
          c.request_id = rid;
          c.seq = sent;
          c.payload = payload_of(md, rng() % 48, sent * 31 + schedule);
          c.eos = (sent + 1 == n);
          expect.push_back(c.payload);
          send.send(c);
          ++sent;
        } else {
          auto c = recv.try_recv();
          CHECK(c.has_value());
          CHECK(c->seq == received);
          CHECK(c->payload == expect[received]);
          CHECK(c->eos == (received + 1 == n));
          ++received;
        }
      }
      CHECK(!recv.try_recv().has_value());
      conn.cleanup(rid);
    }
  });
}

// ---- test_payload_context.cpp:17-164 + the DEVICE locator ---------------

ControlMessage random_message(std::mt19937& rng, bool with_device) {
  ControlMessage m;
  m.kind = static_cast<ControlMessage::Kind>(rng() % 5);
  m.request_id = rng();
  const std::string from = "s" + std::to_string(rng() % 4), to = "d" + std::to_string(rng() % 4);
  m.key = ConnectorKey{m.request_id, from + "->" + to, "tag" + std::to_string(rng() % 16), rng() % 4}.canonical();
  m.edge = from + "->" + to;
  m.seq = rng();
  Locator& l = m.locator;
  l.kind = static_cast<Locator::Kind>(rng() % (with_device ? 4 : 3));
  switch (l.kind) {
    case Locator::Kind::INLINE:
      l.inline_bytes.resize(rng() % 64);
      for (auto& b : l.inline_bytes) b = static_cast<uint8_t>(rng());
      break;
    case Locator::Kind::SHM:
      l.shm_region = "/r" + std::to_string(rng() % 8);
      l.shm_offset = rng();
      l.shm_length = rng();
      break;
    case Locator::Kind::TCP:
      l.tcp_stream_id = rng();
      break;
    case Locator::Kind::DEVICE: {
      l.device = rng() % 8;
      l.arena = rng() % 3 == 0 ? 0 : (uint64_t(rng()) << 32 | rng());
      l.offset = uint64_t(rng()) << 16;
      l.dtype = static_cast<Dtype>(rng() % 3);
      const uint32_t rank = rng() % 3 + 1;
      uint64_t elems = 1;
      for (uint32_t d = 0; d < rank; ++d) {
        l.shape.push_back(rng() % 70);
        elems *= l.shape.back();
      }
      l.length = payload_header_bytes(rank) + elems * dtype_width(l.dtype);
      l.tokens.resize(rng() % 9);
      for (auto& t : l.tokens) t = static_cast<int32_t>(rng());
      break;
    }
  }
  return m;
}

void codecs() {
  run("payload wire round-trip incl. zero-length", [&] {
    Payload p = Payload::from_i32(std::vector<int32_t>{-1, 0, 7, 1 << 30});
    CHECK(decode_payload(encode_payload(p)) == p);
    Payload z;
    z.dtype = Dtype::I32;
    z.shape = {0};
    CHECK(decode_payload(encode_payload(z)) == z);
    CHECK(z.element_count() == 0);
  });
  run("payload fuzz round-trip (500)", [&] {
    std::mt19937 rng(11);
    for (int i = 0; i < 500; ++i) {
      Payload p;
      p.dtype = static_cast<Dtype>(rng() % 3);
      const uint32_t rank = rng() % 3 + 1;
      uint64_t count = 1;
      for (uint32_t d = 0; d < rank; ++d) {
        p.shape.push_back(rng() % 5);
        count *= p.shape.back();
      }
      p.bytes.resize(count * dtype_width(p.dtype));
      for (auto& b : p.bytes) b = static_cast<uint8_t>(rng());
      CHECK(decode_payload(encode_payload(p)) == p);
    }
  });
  run("payload decode rejects truncated buffers", [&] {
    auto enc = encode_payload(Payload::from_i32(std::vector<int32_t>{1, 2, 3}));
    enc.pop_back();
    CHECK_THROWS_AS(decode_payload(enc), OmniError);
  });
  run("a device payload has no host encoding", [&] {
    CHECK_THROWS_AS(encode_payload(device_payload(2, 4, 1)), BadDtype);
  });
  run("connector key canonical form", [&] {
    CHECK(ConnectorKey({7, "thinker->talker", "hidden", 0}).canonical() == "req:7/edge:thinker->talker/hidden/0");
  });
  run("control frame round-trip (reference SHM case + DEVICE)", [&] {
    ControlMessage m;
    m.kind = ControlMessage::Kind::CHUNK_NOTICE;
    m.key = ConnectorKey{3, "a->b", "t", 0}.canonical();
    m.request_id = 3;
    m.edge = "a->b";
    m.seq = 9;
    m.locator.kind = Locator::Kind::SHM;
    m.locator.shm_region = "/omni.test";
    m.locator.shm_offset = 128;
    m.locator.shm_length = 64;
    auto back = decode_control_frame(encode_control_frame(m));
    CHECK(back == m);
    CHECK(back.locator.shm_offset == 128);
    m.locator = device_locator(device_payload(4, 2048, 5, 2));
    back = decode_control_frame(encode_control_frame(m));
    CHECK(back == m);
    CHECK(payload_from_locator(back.locator) == device_payload(4, 2048, 5, 2));
  });
  run("reference-kind frames are byte-identical to the reference layout", [&] {
    // hand-assembled reference frame (control.hpp:56-82): TCP locator
    ControlMessage m;
    m.kind = ControlMessage::Kind::ACK;
    m.key = "k";
    m.request_id = 0x0102030405060708ull;
    m.edge = "e";
    m.seq = 0x0a0b0c0d;
    m.locator.kind = Locator::Kind::TCP;
    m.locator.tcp_stream_id = 0x1122334455667788ull;
    const std::vector<uint8_t> want = {
        0x1f, 0, 0, 0, 4,                          // body length 31, kind ACK
        1, 0, 0, 0, 'k',                           // key
        8, 7, 6, 5, 4, 3, 2, 1,                    // request_id
        1, 0, 0, 0, 'e',                           // edge
        0x0d, 0x0c, 0x0b, 0x0a,                    // seq
        2,                                         // locator TCP
        0x88, 0x77, 0x66, 0x55, 0x44, 0x33, 0x22, 0x11};
    CHECK(encode_control_frame(m) == want);
  });
  run("control frame fuzz round-trip (500 reference kinds + 2000 with DEVICE)", [&] {
    std::mt19937 rng(5);
    for (int i = 0; i < 500; ++i) {
      auto m = random_message(rng, false);
      CHECK(decode_control_frame(encode_control_frame(m)) == m);
    }
    for (int i = 0; i < 2000; ++i) {
      auto m = random_message(rng, true);
      CHECK(decode_control_frame(encode_control_frame(m)) == m);
    }
  });
  run("control frame rejects garbage, every truncation, trailing bytes, bad kinds", [&] {
    CHECK_THROWS_AS(decode_control_frame(std::vector<uint8_t>{1, 2, 3}), OmniError);
    std::mt19937 rng(99);
    for (int i = 0; i < 300; ++i) {
      const auto f = encode_control_frame(random_message(rng, true));
      for (size_t cut = 0; cut < f.size(); ++cut)
        CHECK_THROWS_AS(decode_control_frame(std::span<const uint8_t>(f.data(), cut)), ProtocolViolation);
      auto g = f;
      g.push_back(0);
      CHECK_THROWS_AS(decode_control_frame(g), ProtocolViolation);  // length mismatch
      g = f;
      g[4] = 5;
      CHECK_THROWS_AS(decode_control_frame(g), ProtocolViolation);  // message kind
    }
    ControlMessage m;
    m.locator.kind = Locator::Kind::TCP;
    auto f = encode_control_frame(m);
    f[5 + 4 + 8 + 4 + 4] = 4;  // locator kind after key, rid, edge, seq
    CHECK_THROWS_AS(decode_control_frame(f), ProtocolViolation);
    // DEVICE locator whose length disagrees with its shape
    m.locator = device_locator(device_payload(2, 8, 3));
    m.locator.length += 2;
    CHECK_THROWS_AS(decode_control_frame(encode_control_frame(m)), ProtocolViolation);
    // DEVICE locator with a bad dtype tag
    m.locator = device_locator(device_payload(2, 8, 3));
    f = encode_control_frame(m);
    f[5 + 4 + 8 + 4 + 4 + 1 + 4 + 8 + 8 + 8] = 7;
    CHECK_THROWS_AS(decode_control_frame(f), BadDtype);
  });
  run("random byte strings never decode to a frame silently wrong", [&] {
    std::mt19937 rng(1234);
    int accepted = 0;
    for (int i = 0; i < 20000; ++i) {
      std::vector<uint8_t> junk(rng() % 64);
      for (auto& b : junk) b = static_cast<uint8_t>(rng());
      try {
        auto m = decode_control_frame(junk);
        CHECK(encode_control_frame(m) == junk);  // anything accepted re-encodes identically
        ++accepted;
      } catch (const OmniError&) {
      }
    }
    (void)accepted;
  });
}

}  // namespace

int main() {
  for (Mode md : {Mode::HOST, Mode::DEVICE}) {
    keyed(md);
    streams(md);
    acceptance(md);
  }
  codecs();
  std::printf("ALL OK %d cases %d checks\n", g_cases, g_checks);
  return 0;
}

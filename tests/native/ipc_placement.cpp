// Multi-process stage placement over the cross-process DEVICE transport
// (omni/ipc_channel.hpp, omni_dev.h "Multi-process placement").
//
//   ipc_placement cpu   control-plane conformance across fork() on synthetic
//                       locators (no GPU): handle handoff, re-basing, order,
//                       ACKs, protocol violations seen by the RECEIVER, peer
//                       loss -> TransportDown.
//   ipc_placement gpu   a Thinker stage in the producer process packs hidden
//                       rows straight into the consumer process's connector
//                       arena (CUDA IPC), ordered by an interprocess event,
//                       announced by DEVICE control frames over an AF_UNIX
//                       socket; the consumer checks every blob bit-exact
//                       against the same Thinker run in its own process, then
//                       feeds the IPC rows to a Talker stage and checks its
//                       tokens / margins bit-identical to the in-process path.
//
// Prints "ok ..." per check group and "ALL OK" at the end; exit 1 on failure.
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "omni/ipc_channel.hpp"
#include "omni_dev.h"

using namespace omni;

#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::fprintf(stderr, "[%d] FAIL %s:%d: %s\n", getpid(), __FILE__,    \
                   __LINE__, #cond);                                      \
      std::fflush(stderr);                                                \
      std::_Exit(1);                                                      \
    }                                                                     \
  } while (0)
#define OK(call)                                                          \
  do {                                                                    \
    omni_status s_ = (call);                                              \
    if (s_ != OMNI_OK) {                                                  \
      std::fprintf(stderr, "[%d] FAIL %s:%d: %s -> %d (%s)\n", getpid(),   \
                   __FILE__, __LINE__, #call, int(s_), omni_last_error()); \
      std::fflush(stderr);                                                \
      std::_Exit(1);                                                      \
    }                                                                     \
  } while (0)
template <class Err, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const Err&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

namespace {

const std::string kEdge = "thinker->talker";

int wait_child(pid_t pid) {
  int st = 0;
  waitpid(pid, &st, 0);
  return WIFEXITED(st) ? WEXITSTATUS(st) : 128;
}

Payload fake_device_chunk(uint64_t addr, uint32_t rows, uint32_t d, int32_t first_tok) {
  Payload p;
  p.dtype = Dtype::FIX16;
  p.shape = {rows, 1 + d};
  p.dev.device = 0;
  p.dev.blob = addr;
  p.dev.nbytes = payload_header_bytes(2) + uint64_t(rows) * (1 + d) * 2;
  for (uint32_t r = 0; r < rows; ++r) p.host_tokens.push_back(first_tok + int32_t(r));
  return p;
}

// ---------------------------------------------------------------- cpu mode
int run_cpu() {
  const uint64_t kArenaId = 0xA1, kProdBase = 0x7f0000000000ull, kConsBase = 0x500000000ull, kBytes = 1 << 20;
  auto [a, b] = IpcChannel::pair();
  const pid_t pid = fork();
  if (pid == 0) {  // producer
    a = IpcChannel();
    const auto h = handoff_bytes(b.recv(5000), "arena:161");
    CHECK(h.size() == 8);
    IpcStreamSender tx(b, kEdge, kArenaId, kProdBase, kBytes);
    // sender-side checks
    CHECK(throws<ProtocolViolation>([&] { tx.send(StreamChunk{1, "", "", 0, fake_device_chunk(kProdBase - 16, 1, 8, 1), false}); }));
    CHECK(throws<ProtocolViolation>([&] { tx.send(StreamChunk{1, "", "", 3, fake_device_chunk(kProdBase, 1, 8, 1), false}); }));
    CHECK(throws<BadDtype>([&] { tx.send(StreamChunk{1, "", "", 0, Payload::from_u8({1}), false}); }));
    // two requests, interleaved, 3 chunks each (last = eos)
    for (uint32_t k = 0; k < 3; ++k)
      for (uint64_t rid : {1ull, 2ull}) {
        const uint64_t off = (rid * 4 + k) * 4096;
        tx.send(StreamChunk{rid, "", "", k, fake_device_chunk(kProdBase + off, 4, 8, int32_t(10 * rid + k)), k == 2});
      }
    CHECK(throws<ProtocolViolation>([&] { tx.send(StreamChunk{1, "", "", 3, fake_device_chunk(kProdBase, 1, 8, 1), false}); }));
    while (tx.acked(1) < 3 || tx.acked(2) < 3) {
      tx.poll_acks();
      usleep(200);
    }
    // a hostile frame: out-of-order seq straight on the channel
    ControlMessage m;
    m.kind = ControlMessage::Kind::CHUNK_NOTICE;
    m.request_id = 7;
    m.edge = kEdge;
    m.seq = 1;
    m.locator = device_locator(fake_device_chunk(kProdBase, 1, 8, 1));
    m.locator.arena = kArenaId;
    m.locator.offset = 0;
    b.send(m);
    // ... and one outside the arena
    m.request_id = 8;
    m.seq = 0;
    m.locator.offset = kBytes - 16;
    b.send(m);
    // ... and one naming another arena
    m.request_id = 9;
    m.locator.offset = 0;
    m.locator.arena = 0xB2;
    b.send(m);
    std::fflush(stdout);
    std::_Exit(0);
  }
  b = IpcChannel();
  const uint64_t id = kArenaId;
  a.send(handoff_frame("arena:161", &id, sizeof(id)));
  IpcStreamReceiver rx(a, kEdge, kArenaId, kConsBase, kBytes, 3);
  for (uint64_t rid : {2ull, 1ull})
    for (uint32_t k = 0; k < 3; ++k) {
      StreamChunk c = rx.recv(rid, 10000);
      CHECK(c.request_id == rid && c.seq == k && c.eos == (k == 2));
      CHECK(c.from == "thinker" && c.to == "talker");
      CHECK(c.payload.dev.blob == kConsBase + (rid * 4 + k) * 4096);  // re-based onto the local arena
      CHECK(c.payload.dev.device == 3 && c.payload.dev.arena == 0);
      CHECK(c.payload.shape == std::vector<uint32_t>({4, 9}));
      CHECK(c.payload.host_tokens.size() == 4 && c.payload.host_tokens[0] == int32_t(10 * rid + k));
      rx.ack(rid, k);
    }
  CHECK(!rx.try_recv(1).has_value());
  std::printf("ok ipc stream: handoff, per-request order, re-basing, acks\n");
  CHECK(throws<ProtocolViolation>([&] { rx.recv(7, 10000); }));
  CHECK(throws<ProtocolViolation>([&] { rx.recv(8, 10000); }));
  CHECK(throws<ProtocolViolation>([&] { rx.recv(9, 10000); }));
  std::printf("ok receiver rejects out-of-order, out-of-arena and foreign-arena locators\n");
  CHECK(wait_child(pid) == 0);
  CHECK(throws<TransportDown>([&] { rx.recv(1, 2000); }));
  std::printf("ok peer exit -> TransportDown\n");
  // AF_UNIX path rendezvous
  const std::string path = "/tmp/omni_ipc_test_" + std::to_string(getpid());
  const pid_t p2 = fork();
  if (p2 == 0) {
    IpcChannel c = IpcChannel::connect(path, 5000);
    c.send(handoff_frame("hello", "xy", 2));
    std::_Exit(0);
  }
  IpcChannel srv = IpcChannel::listen_accept(path, 5000);
  CHECK(handoff_bytes(srv.recv(5000), "hello") == std::vector<uint8_t>({'x', 'y'}));
  CHECK(wait_child(p2) == 0);
  std::printf("ok unix-socket rendezvous\n");
  std::printf("ALL OK\n");
  return 0;
}

// ---------------------------------------------------------------- gpu mode
constexpr int kD = 512, kRows = 8, kChunk = 4, kPrompt = 7;
const uint64_t kRids[2] = {1, 2};

omni_model_desc small(int32_t kind) {
  omni_model_desc m{};
  OK(omni_model_default(kind, &m));
  m.d_model = kD;
  m.n_layers = 2;
  m.n_heads = 4;
  m.n_kv_heads = 2;
  m.d_ff = 1024;
  if (kind == OMNI_MODEL_TALKER) m.cond_dim = kD;
  return m;
}

uint64_t chunk_offset(int r, int k) { return uint64_t(r * 2 + k) * 16384; }

// Runs the Thinker (prefill both requests, kRows decode steps) and packs rows
// [0,4) after step 3 and [4,8) after step 7 into base + chunk_offset. Returns
// the emitted tokens per request. `ev` (may be null) is recorded after each pack.
std::vector<std::vector<int32_t>> run_thinker(omni_stage* st, uint64_t base, omni_ipc_event* ev,
                                              IpcStreamSender* tx) {
  std::vector<std::vector<int32_t>> toks(2);
  {
    std::vector<uint64_t> sid = {kRids[0], kRids[1]};
    std::vector<int32_t> ph = {OMNI_PHASE_PREFILL, OMNI_PHASE_PREFILL}, sp = {kPrompt, kPrompt}, p0 = {0, 0},
                         oi = {-1, -1}, tk;
    for (int r = 0; r < 2; ++r)
      for (int i = 0; i < kPrompt; ++i) tk.push_back((31 * i + 17 * r + 3) % 250 + 1);
    omni_ar_batch b{2, sid.data(), ph.data(), sp.data(), p0.data(), oi.data(), tk.data(), nullptr, nullptr};
    int32_t out[2];
    float mg[2];
    OK(omni_ar_step(st, &b, out, mg));
    OK(omni_stage_wait(st));
  }
  for (int k = 0; k < kRows; ++k) {
    std::vector<uint64_t> sid = {kRids[0], kRids[1]};
    std::vector<int32_t> ph = {OMNI_PHASE_DECODE, OMNI_PHASE_DECODE}, sp = {1, 1}, p0 = {kPrompt + k, kPrompt + k},
                         oi = {k, k}, tk = {k ? toks[0].back() : 0, k ? toks[1].back() : 0};
    omni_ar_batch b{2, sid.data(), ph.data(), sp.data(), p0.data(), oi.data(), tk.data(), nullptr, nullptr};
    int32_t out[2];
    float mg[2];
    OK(omni_ar_step(st, &b, out, mg));
    OK(omni_stage_wait(st));
    toks[0].push_back(out[0]);
    toks[1].push_back(out[1]);
    if ((k + 1) % kChunk == 0) {
      const int c = k / kChunk, b0 = c * kChunk, b1 = b0 + kChunk;
      std::vector<uint64_t> seqs = {kRids[0], kRids[1]};
      std::vector<int32_t> beg = {b0, b0}, end = {b1, b1}, ptok;
      std::vector<uint64_t> dst = {base + chunk_offset(0, c), base + chunk_offset(1, c)};
      for (int r = 0; r < 2; ++r)
        for (int i = b0; i < b1; ++i) ptok.push_back(toks[r][i]);
      OK(omni_pack_hidden(st, 2, seqs.data(), beg.data(), end.data(), ptok.data(), 0, dst.data()));
      if (ev) OK(omni_stage_record_pack(st, ev));
      if (tx)
        for (int r = 0; r < 2; ++r) {
          Payload p;
          p.dtype = Dtype::FIX16;
          p.shape = {uint32_t(kChunk), uint32_t(1 + kD)};
          p.dev.device = 0;
          p.dev.blob = dst[r];
          p.dev.nbytes = omni_pack_bytes(kChunk, kD);
          p.host_tokens.assign(ptok.begin() + r * kChunk, ptok.begin() + (r + 1) * kChunk);
          tx->send(StreamChunk{kRids[r], "", "", uint32_t(c), p, c == kRows / kChunk - 1});
        }
    }
  }
  return toks;
}

int run_gpu() {
  auto [a, b] = IpcChannel::pair();
  const pid_t pid = fork();  // before any CUDA call in either process
  if (pid == 0) {            // ---- producer: the Thinker's process
    a = IpcChannel();
    OK(omni_init(0, nullptr));
    const auto hb = handoff_bytes(b.recv(60000), "arena:1");
    CHECK(hb.size() == sizeof(omni_ipc_handle));
    omni_ipc_handle h;
    std::memcpy(&h, hb.data(), sizeof(h));
    omni_arena* peer = nullptr;
    OK(omni_arena_import(&h, &peer));
    uint64_t base = 0, bytes = 0;
    OK(omni_arena_base(peer, &base, &bytes));
    omni_ipc_event* ev = nullptr;
    omni_ipc_event_handle eh;
    OK(omni_ipc_event_create(0, &ev, &eh));
    b.send(handoff_frame("event:1", &eh, sizeof(eh)));
    omni_model_desc m = small(OMNI_MODEL_THINKER);
    omni_stage_limits lim{64, 4, 128, 0, 16};
    omni_stage* st = nullptr;
    OK(omni_stage_create(&m, &lim, 0, 5, &st));
    IpcStreamSender tx(b, kEdge, 1, base, bytes);
    run_thinker(st, base, ev, &tx);
    while (tx.acked(kRids[0]) < 2 || tx.acked(kRids[1]) < 2) {
      tx.poll_acks();
      usleep(500);
    }
    OK(omni_stage_destroy(st));
    OK(omni_ipc_event_destroy(ev));
    OK(omni_arena_destroy(peer));
    std::fflush(stdout);
    std::_Exit(0);
  }
  // ---- consumer: the Talker's process
  b = IpcChannel();
  OK(omni_init(0, nullptr));
  const uint64_t kBytes = 1 << 20;
  omni_arena* arena = nullptr;
  OK(omni_arena_create(0, kBytes, &arena));
  uint64_t base = 0;
  OK(omni_arena_base(arena, &base, nullptr));
  OK(omni_mem_set(base, 0, kBytes));
  omni_ipc_handle h;
  OK(omni_arena_export(arena, &h));
  a.send(handoff_frame("arena:1", &h, sizeof(h)));
  IpcStreamReceiver rx(a, kEdge, 1, base, kBytes, 0);
  ControlMessage em = a.recv(60000);
  const auto ehb = handoff_bytes(em, "event:1");
  omni_ipc_event_handle eh;
  std::memcpy(&eh, ehb.data(), sizeof(eh));
  omni_ipc_event* ev = nullptr;
  OK(omni_ipc_event_open(0, &eh, &ev));
  std::printf("ok arena exported, interprocess event opened\n");

  // the same Thinker in this process, packing into a local reference arena
  omni_arena* ref_arena = nullptr;
  OK(omni_arena_create(0, kBytes, &ref_arena));
  uint64_t ref_base = 0;
  OK(omni_arena_base(ref_arena, &ref_base, nullptr));
  OK(omni_mem_set(ref_base, 0, kBytes));
  omni_model_desc tm = small(OMNI_MODEL_THINKER);
  omni_stage_limits lim{64, 4, 128, 0, 16};
  omni_stage* ref = nullptr;
  OK(omni_stage_create(&tm, &lim, 0, 5, &ref));
  auto ref_toks = run_thinker(ref, ref_base, nullptr, nullptr);
  OK(omni_stage_wait(ref));

  // talker stages: one fed from the IPC arena, one from the reference arena
  omni_model_desc km = small(OMNI_MODEL_TALKER);
  omni_stage *talk_ipc = nullptr, *talk_ref = nullptr;
  OK(omni_stage_create(&km, &lim, 0, 9, &talk_ipc));
  OK(omni_stage_create(&km, &lim, 0, 9, &talk_ref));

  std::vector<std::vector<uint64_t>> rows_ipc(2), rows_ref(2);
  std::vector<std::vector<int32_t>> toks_ipc(2);
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < kRows / kChunk; ++c) {
      StreamChunk ch = rx.recv(kRids[r], 60000);
      CHECK(ch.seq == uint32_t(c) && ch.eos == (c == kRows / kChunk - 1));
      CHECK(ch.payload.dev.blob == base + chunk_offset(r, c));
      CHECK(ch.payload.dev.nbytes == omni_pack_bytes(kChunk, kD));
      // rows land before the frame is acted on: wait for the producer's pack
      OK(omni_stage_wait_event(talk_ipc, ev));
      OK(omni_ipc_event_sync(ev));
      std::vector<uint8_t> got(ch.payload.dev.nbytes), want(ch.payload.dev.nbytes);
      OK(omni_mem_d2h(got.data(), ch.payload.dev.blob, got.size()));
      OK(omni_mem_d2h(want.data(), ref_base + chunk_offset(r, c), want.size()));
      CHECK(got == want);
      for (int i = 0; i < kChunk; ++i) {
        CHECK(ch.payload.host_tokens[i] == ref_toks[r][c * kChunk + i]);
        rows_ipc[r].push_back(ch.payload.device_elem(i, 1));
        Payload rp = ch.payload;
        rp.dev.blob = ref_base + chunk_offset(r, c);
        rows_ref[r].push_back(rp.device_elem(i, 1));
        toks_ipc[r].push_back(ch.payload.host_tokens[i]);
      }
      rx.ack(kRids[r], ch.seq);
    }
  std::printf("ok %d chunks packed across processes are bit-exact with the in-process pack\n", 2 * kRows / kChunk);

  // Talker prefill over the 8 rows + 6 decode steps, from both sources
  auto talk = [&](omni_stage* st, const std::vector<std::vector<uint64_t>>& rows) {
    std::vector<uint64_t> sid = {kRids[0], kRids[1]}, cs;
    std::vector<int32_t> ph = {OMNI_PHASE_PREFILL, OMNI_PHASE_PREFILL}, sp = {kRows, kRows}, p0 = {0, 0},
                         oi = {-1, -1}, tk, cr;
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < kRows; ++j) {
        tk.push_back(toks_ipc[r][j]);
        cs.push_back(rows[r][j]);
        cr.push_back(j);
      }
    omni_ar_batch b{2, sid.data(), ph.data(), sp.data(), p0.data(), oi.data(), tk.data(), cs.data(), cr.data()};
    int32_t out[2];
    float mg[2];
    OK(omni_ar_step(st, &b, out, mg));
    OK(omni_stage_wait(st));
    std::vector<int32_t> res;
    std::vector<float> mres;
    int32_t prev[2] = {0, 0};
    for (int k = 0; k < 6; ++k) {
      std::vector<int32_t> dph = {OMNI_PHASE_DECODE, OMNI_PHASE_DECODE}, dsp = {1, 1},
                           dp0 = {kRows + k, kRows + k}, doi = {k, k}, dtk = {prev[0], prev[1]},
                           dcr = {k / 4, k / 4};
      std::vector<uint64_t> dcs = {0, 0};
      omni_ar_batch d{2, sid.data(), dph.data(), dsp.data(), dp0.data(), doi.data(), dtk.data(), dcs.data(),
                      dcr.data()};
      OK(omni_ar_step(st, &d, out, mg));
      OK(omni_stage_wait(st));
      prev[0] = out[0];
      prev[1] = out[1];
      res.insert(res.end(), out, out + 2);
      mres.insert(mres.end(), mg, mg + 2);
    }
    return std::make_pair(res, mres);
  };
  auto [ti, mi] = talk(talk_ipc, rows_ipc);
  auto [tr, mr] = talk(talk_ref, rows_ref);
  CHECK(ti == tr);
  CHECK(std::memcmp(mi.data(), mr.data(), mi.size() * sizeof(float)) == 0);
  std::printf("ok talker fed from the IPC arena: %zu codec tokens + margins bit-identical\n", ti.size());
  CHECK(wait_child(pid) == 0);
  OK(omni_stage_destroy(talk_ipc));
  OK(omni_stage_destroy(talk_ref));
  OK(omni_stage_destroy(ref));
  OK(omni_ipc_event_destroy(ev));
  OK(omni_arena_destroy(ref_arena));
  OK(omni_arena_destroy(arena));
  std::printf("ALL OK\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  return mode == "gpu" ? run_gpu() : run_cpu();
}

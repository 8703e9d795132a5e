// HTTP/1.1 front end over POSIX sockets (see omni/http_service.hpp).
#include "omni/http_service.hpp"

#include <arpa/inet.h>
#include <netinet/in.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <json.hpp>

namespace omni {

using nlohmann::json;

std::string base64_encode(const uint8_t* data, size_t len) {
  static const char tbl[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
  std::string out;
  out.reserve((len + 2) / 3 * 4);
  size_t i = 0;
  for (; i + 3 <= len; i += 3) {
    const uint32_t v = uint32_t(data[i]) << 16 | uint32_t(data[i + 1]) << 8 | data[i + 2];
    out += tbl[v >> 18 & 63];
    out += tbl[v >> 12 & 63];
    out += tbl[v >> 6 & 63];
    out += tbl[v & 63];
  }
  if (i + 1 == len) {
    const uint32_t v = uint32_t(data[i]) << 16;
    out += tbl[v >> 18 & 63];
    out += tbl[v >> 12 & 63];
    out += "==";
  } else if (i + 2 == len) {
    const uint32_t v = uint32_t(data[i]) << 16 | uint32_t(data[i + 1]) << 8;
    out += tbl[v >> 18 & 63];
    out += tbl[v >> 12 & 63];
    out += tbl[v >> 6 & 63];
    out += '=';
  }
  return out;
}

std::string waveform_b64(const std::vector<int32_t>& samples) {
  std::vector<uint8_t> b(samples.size() * 4);
  for (size_t i = 0; i < samples.size(); ++i) {
    const uint32_t u = static_cast<uint32_t>(samples[i]);
    for (int k = 0; k < 4; ++k) b[4 * i + k] = static_cast<uint8_t>(u >> (8 * k));
  }
  return base64_encode(b.data(), b.size());
}

namespace {

json metrics_json(const MetricsRecord& rec) {  // http_service.hpp:60-83
  json m;
  m["request_id"] = rec.request_id;
  m["submitted_at"] = rec.submitted_at;
  m["status"] = rec.status;
  m["text_tokens"] = rec.text_token_count;
  m["codec_tokens"] = rec.codec_token_count;
  m["waveform_samples"] = rec.waveform_sample_count;
  if (rec.status == "DONE") {
    m["jct_us"] = jct_us(rec);
    m["ttft_us"] = ttft_us(rec);
    if (rec.waveform_sample_count > 0) m["rtf"] = rtf(rec);
    json st = json::object();
    for (const auto& [stage, tim] : rec.stages)
      if (tim.finished_at != kTimeUnset && tim.finished_at > tim.first_scheduled_at && tim.tokens > 0)
        st[stage] = tps(rec, stage);
    m["tps"] = std::move(st);
  }
  return m;
}

bool write_all(int fd, const char* p, size_t n) {
  while (n > 0) {
    const ssize_t w = ::send(fd, p, n, MSG_NOSIGNAL);
    if (w < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    p += w;
    n -= static_cast<size_t>(w);
  }
  return true;
}

const char* reason(int status) {
  switch (status) {
    case 200: return "OK";
    case 400: return "Bad Request";
    case 404: return "Not Found";
    case 405: return "Method Not Allowed";
    case 413: return "Payload Too Large";
    case 429: return "Too Many Requests";
    default: return "Internal Server Error";
  }
}

void respond(int fd, int status, const std::string& body, const char* type = "application/json") {
  std::string h = "HTTP/1.1 " + std::to_string(status) + " " + reason(status) + "\r\nContent-Type: " + type +
                  "\r\nContent-Length: " + std::to_string(body.size()) + "\r\nConnection: close\r\n\r\n";
  if (write_all(fd, h.data(), h.size())) write_all(fd, body.data(), body.size());
}

bool write_chunk(int fd, const std::string& s) {
  char hdr[32];
  const int n = std::snprintf(hdr, sizeof hdr, "%zx\r\n", s.size());
  return write_all(fd, hdr, static_cast<size_t>(n)) && write_all(fd, s.data(), s.size()) &&
         write_all(fd, "\r\n", 2);
}

std::string lower(std::string s) {
  for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

constexpr size_t kMaxHead = 64 << 10, kMaxBody = 16 << 20;

}  // namespace

void HttpService::start(const std::string& listen) {
  const auto colon = listen.rfind(':');
  const std::string host = colon == std::string::npos ? listen : listen.substr(0, colon);
  const int port = colon == std::string::npos ? 8080 : std::stoi(listen.substr(colon + 1));
  const int s = ::socket(AF_INET, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (s < 0) throw TransportDown(std::string("socket: ") + std::strerror(errno));
  const int one = 1;
  ::setsockopt(s, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(static_cast<uint16_t>(port));
  if (::inet_pton(AF_INET, host == "localhost" ? "127.0.0.1" : host.c_str(), &a.sin_addr) != 1) {
    ::close(s);
    throw ConfigInvalid("listen address must be an IPv4 literal: " + host);
  }
  if (::bind(s, reinterpret_cast<sockaddr*>(&a), sizeof a) != 0) {
    const int e = errno;
    ::close(s);
    if (e == EADDRINUSE) throw PortInUse("port in use: " + listen);
    throw TransportDown(std::string("bind: ") + std::strerror(e));
  }
  if (::listen(s, 64) != 0) {
    ::close(s);
    throw TransportDown(std::string("listen: ") + std::strerror(errno));
  }
  socklen_t len = sizeof a;
  ::getsockname(s, reinterpret_cast<sockaddr*>(&a), &len);
  port_ = ntohs(a.sin_port);
  listen_fd_ = s;
  running_ = true;
  accept_thread_ = std::thread([this] { accept_loop(); });
}

void HttpService::stop() {
  if (!running_.exchange(false)) return;
  if (accept_thread_.joinable()) accept_thread_.join();
  ::close(listen_fd_);
  listen_fd_ = -1;
  reap(true);
}

void HttpService::reap(bool all) {
  std::list<Conn> finished;
  {
    std::lock_guard lk(conn_mu_);
    for (auto it = conns_.begin(); it != conns_.end();) {
      if (all || it->done->load()) {
        finished.splice(finished.end(), conns_, it++);
      } else {
        ++it;
      }
    }
  }
  for (auto& c : finished) c.t.join();
}

void HttpService::accept_loop() {
  while (running_) {
    pollfd p{listen_fd_, POLLIN, 0};
    if (::poll(&p, 1, 50) <= 0) continue;
    const int c = ::accept4(listen_fd_, nullptr, nullptr, SOCK_CLOEXEC);
    if (c < 0) continue;
    reap(false);  // a long-running server does not accumulate finished threads
    auto done = std::make_shared<std::atomic<bool>>(false);
    std::lock_guard lk(conn_mu_);
    conns_.push_back(Conn{std::thread([this, c, done] {
                            serve(c);
                            ::close(c);
                            done->store(true);
                          }),
                          done});
  }
}

void HttpService::serve(int fd) {
  std::string buf;
  size_t head_end = std::string::npos;
  char tmp[8192];
  while ((head_end = buf.find("\r\n\r\n")) == std::string::npos) {
    if (buf.size() > kMaxHead) return respond(fd, 413, json{{"error", "header too large"}}.dump());
    pollfd p{fd, POLLIN, 0};
    if (::poll(&p, 1, 10000) <= 0) return;
    const ssize_t n = ::recv(fd, tmp, sizeof tmp, 0);
    if (n <= 0) return;
    buf.append(tmp, static_cast<size_t>(n));
  }
  const std::string head = buf.substr(0, head_end);
  std::string body = buf.substr(head_end + 4);
  const auto eol = head.find("\r\n");
  const std::string line = head.substr(0, eol);
  const auto sp1 = line.find(' '), sp2 = line.find(' ', sp1 + 1);
  if (sp1 == std::string::npos || sp2 == std::string::npos)
    return respond(fd, 400, json{{"error", "bad request line"}}.dump());
  const std::string method = line.substr(0, sp1);
  std::string path = line.substr(sp1 + 1, sp2 - sp1 - 1);
  if (const auto q = path.find('?'); q != std::string::npos) path.resize(q);
  size_t content_length = 0;
  for (size_t at = eol; at != std::string::npos && at < head.size();) {
    const size_t next = head.find("\r\n", at + 2);
    const std::string h = head.substr(at + 2, (next == std::string::npos ? head.size() : next) - at - 2);
    const auto c = h.find(':');
    if (c != std::string::npos && lower(h.substr(0, c)) == "content-length") {
      try {
        content_length = std::stoull(h.substr(c + 1));
      } catch (...) {
        return respond(fd, 400, json{{"error", "bad content-length"}}.dump());
      }
    }
    at = next;
  }
  if (content_length > kMaxBody) return respond(fd, 413, json{{"error", "body too large"}}.dump());
  while (body.size() < content_length) {
    pollfd p{fd, POLLIN, 0};
    if (::poll(&p, 1, 10000) <= 0) return;
    const ssize_t n = ::recv(fd, tmp, sizeof tmp, 0);
    if (n <= 0) return;
    body.append(tmp, static_cast<size_t>(n));
  }
  body.resize(content_length);

  if (path == "/v1/generate") {
    if (method != "POST") return respond(fd, 405, json{{"error", "use POST"}}.dump());
    return handle_generate(fd, body);
  }
  if (method != "GET") return respond(fd, path == "/v1/health" || path == "/v1/metrics" ? 405 : 404, "{}");
  if (path == "/v1/health") {
    json h = json::object();
    for (const auto& [stage, st] : orch_.health()) h[stage] = st;
    return respond(fd, 200, h.dump());
  }
  if (path == "/v1/metrics") {
    uint64_t done = 0, failed = 0, total = 0;
    for (const auto& rec : orch_.metrics().all()) {
      ++total;
      done += rec.status == "DONE";
      failed += rec.status == "FAILED";
    }
    return respond(fd, 200,
                   json{{"requests_seen", total}, {"requests_done", done}, {"requests_failed", failed}}.dump());
  }
  respond(fd, 404, json{{"error", "no route " + path}}.dump());
}

void HttpService::handle_generate(int fd, const std::string& text) {
  json body;
  Request r;
  bool stream = false;
  try {
    body = json::parse(text);
    if (!body.is_object()) throw std::runtime_error("body must be a JSON object");
    r.request_id = body.value("request_id", next_id_.fetch_add(1));
    r.seed = body.value("seed", 0u);
    stream = r.stream = body.value("stream", false);
    if (body.contains("prompt_tokens"))
      for (const auto& t : body.at("prompt_tokens")) {
        const int v = t.get<int>();
        if (v < 1 || v > 255) throw std::runtime_error("prompt token ids must be in [1,255]");
        r.prompt_tokens.push_back(static_cast<uint8_t>(v));
      }
  } catch (const std::exception& e) {
    return respond(fd, 400, json{{"error", e.what()}}.dump());
  }
  if (r.prompt_tokens.empty()) return respond(fd, 400, json{{"error", "prompt_tokens must be non-empty"}}.dump());

  std::shared_ptr<ResultHandle> handle;
  try {
    handle = orch_.submit(std::move(r));
  } catch (const Overloaded& e) {
    return respond(fd, 429, json{{"error", e.what()}}.dump());
  } catch (const OmniError& e) {
    return respond(fd, 400, json{{"error", e.what()}}.dump());
  }

  if (!stream) {
    const FinalOutput& out = handle->wait();
    if (out.status != "DONE") return respond(fd, 500, json{{"error", out.error}}.dump());
    json j{{"text_tokens", out.text_tokens},
           {"codec_tokens", out.codec_tokens},
           {"waveform_b64", waveform_b64(out.waveform)},
           {"metrics", metrics_json(out.metrics)}};
    return respond(fd, 200, j.dump());
  }
  const std::string h =
      "HTTP/1.1 200 OK\r\nContent-Type: application/x-ndjson\r\nTransfer-Encoding: chunked\r\n"
      "Connection: close\r\n\r\n";
  if (!write_all(fd, h.data(), h.size())) return;
  while (auto c = handle->next_chunk()) {
    // a client that went away stops the stream; the request still completes
    if (!write_chunk(fd, json{{"type", "waveform_chunk"}, {"seq", c->seq}, {"data_b64", waveform_b64(c->payload.as_i32())}}
                             .dump() + "\n"))
      return;
  }
  const FinalOutput& out = handle->wait();
  const json last = out.status == "DONE" ? json{{"type", "done"}, {"metrics", metrics_json(out.metrics)}}
                                         : json{{"type", "error"}, {"error", out.error}};
  if (write_chunk(fd, last.dump() + "\n")) write_all(fd, "0\r\n\r\n", 5);
}

}  // namespace omni

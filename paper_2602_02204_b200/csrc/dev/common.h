// Shared host-side plumbing for libomni_dev: status codes, thread-local error
// text, CUDA error checking.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "omni_dev.h"

namespace omni_dev {

struct DevError : std::runtime_error {
  omni_status code;
  DevError(omni_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define OMNI_CUDA(expr)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::omni_dev::DevError(OMNI_E_CUDA, std::string(#expr) + ": " +               \
                                                  cudaGetErrorString(e_) + " @" +       \
                                                  __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Counters of device work issued by this library (bench evidence: how many
// of OUR kernels ran and how many bytes crossed PCIe).
struct DevCounters {
  uint64_t launches = 0, h2d_bytes = 0, d2h_bytes = 0;
  uint64_t graph_captures = 0, graph_replays = 0;
};
DevCounters& counters();

#define OMNI_KERNEL(expr)          \
  do {                             \
    OMNI_CUDA(expr);               \
    ++::omni_dev::counters().launches; \
  } while (0)

#define OMNI_REQUIRE(cond, code, msg)                          \
  do {                                                         \
    if (!(cond)) throw ::omni_dev::DevError((code), (msg));    \
  } while (0)

// Runs `fn`, converting exceptions into a status + omni_last_error() text.
template <typename F>
omni_status guarded(F&& fn) {
  try {
    fn();
    return OMNI_OK;
  } catch (const DevError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return OMNI_E_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return OMNI_E_BADARG;
  }
}

}  // namespace omni_dev

// Common definitions for the B200 GKL library: status codes, error capture,
// CUDA/NCCL checking. Errors never cross the C ABI as exceptions: every
// extern "C" entry point converts them to a status code plus a thread-local
// message (gkb_last_error).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/gkb.h"

namespace gkb {

// Mirrors the reference's exception taxonomy (linop.hpp:103-104 and
// gkl.cpp:53-73 throw std::invalid_argument; gkl.cpp:215-218 and :344
// std::logic_error) plus device-side failures.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error so later launch checks do not re-report it
    fail(GKB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file + ":" +
                        std::to_string(line));
  }
}

#define GKB_CUDA(x) ::gkb::check_cuda((x), #x, __FILE__, __LINE__)
#define GKB_LAUNCH_CHECK() ::gkb::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

void set_last_error(const std::string& msg);

}  // namespace gkb

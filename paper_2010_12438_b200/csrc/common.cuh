// Shared helpers for libgo_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/go_b200.h"

namespace go {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

#define GO_THROW(code, ...) throw ::go::Error((code), ::go::fmt(__VA_ARGS__))
#define GO_CHECK(cond, ...) \
  do {                      \
    if (!(cond)) GO_THROW(GO_ERR_VALUE, __VA_ARGS__); \
  } while (0)
#define CUDA_CHECK(x)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      GO_THROW(GO_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
               __LINE__);                                                                 \
  } while (0)
extern std::atomic<long long> g_launch_count;
#define LAUNCH_CHECK()        \
  do {                        \
    ::go::g_launch_count++;   \
    CUDA_CHECK(cudaGetLastError()); \
  } while (0)

void set_last_error(const std::string& m);

template <class F>
int guarded(F&& f) {
  try {
    f();
    return GO_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GO_ERR_VALUE;
  }
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// Number of SMs on the current device (148 on B200).
int num_sms();

}  // namespace go

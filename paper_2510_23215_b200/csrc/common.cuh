// common.cuh — shared device/host helpers of libscsf (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/scsf.h"

namespace scsf {

// filter parameter block: {lambda, c, e, -} then the per-step (a_s, b_s) table (k_step_table)
constexpr int FP_TAB = 4, FP_MAX_DEGREE = 128, FP_DOUBLES = FP_TAB + 2 * FP_MAX_DEGREE;

// coefficient arrays per operator (include/scsf.h stencil kinds)
inline int ncoef(const scsf_ops* o) { return o->stencil == SCSF_STENCIL_VIB13 ? 7 : 1 + o->dim; }

// ---------------------------------------------------------------- errors ----
void set_error(const char* fmt, ...);
void count_launch(int n = 1);
void set_capturing(bool on);   // launches inside a CUDA-graph capture are counted at replay
bool debug_sync();   // SCSF_DEBUG_SYNC=1: synchronise and check after every launch

struct Status {
  int code = SCSF_OK;
};

#define SCSF_CUDA_CHECK(expr)                                                    \
  do {                                                                          \
    cudaError_t e_ = (expr);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      ::scsf::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                        cudaGetErrorString(e_));                                \
      return SCSF_ERR_DEVICE;                                                   \
    }                                                                           \
  } while (0)

#define SCSF_LAUNCH_CHECK()                                                     \
  do {                                                                          \
    ::scsf::count_launch();                                                     \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ == cudaSuccess && ::scsf::debug_sync()) e_ = cudaDeviceSynchronize(); \
    if (e_ != cudaSuccess) {                                                    \
      ::scsf::set_error("%s:%d launch: %s", __FILE__, __LINE__,                 \
                        cudaGetErrorString(e_));                                \
      return SCSF_ERR_DEVICE;                                                   \
    }                                                                           \
  } while (0)

#define SCSF_ARG_CHECK(cond, ...)                                               \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ::scsf::set_error(__VA_ARGS__);                                           \
      return SCSF_ERR_ARG;                                                      \
    }                                                                           \
  } while (0)

#define SCSF_TRY(expr)                                                          \
  do {                                                                          \
    int s_ = (expr);                                                            \
    if (s_ != SCSF_OK) return s_;                                               \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Bump allocator over the caller's workspace (256-byte aligned carving).
struct Arena {
  char* base;
  size_t size;
  size_t off = 0;
  bool overflow = false;
  Arena(void* b, size_t s) : base((char*)b), size(s) {}
  template <class T>
  T* take(int64_t count) {
    size_t bytes = (size_t)round_up(count * (int64_t)sizeof(T), 256);
    if (off + bytes > size || base == nullptr) {
      overflow = true;
      off += bytes;
      return nullptr;
    }
    T* p = (T*)(base + off);
    off += bytes;
    return p;
  }
};

// --------------------------------------------------------------- device ----
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Device-resident control block of one solve (see solver.cu).
struct Ctrl {
  double lambda;      // filter scale point (smallest active Ritz value)
  double alpha;       // lower end of the damped interval (largest Ritz value in block)
  double beta;        // upper end (Gershgorin bound)
  double max_rel;     // worst relative residual among the L wanted pairs
  int32_t kL;         // locked columns [0, kL)
  int32_t kL_prev;
  int32_t chol_fail;  // set by chol when the Gram matrix was not numerically SPD
  int32_t chol_fallbacks;
  int32_t nonfinite;  // set when a NaN/Inf was seen
  int32_t pad[3];
};

}  // namespace scsf

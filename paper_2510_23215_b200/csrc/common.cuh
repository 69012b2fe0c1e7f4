// common.cuh — shared device/host helpers of libscsf (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/scsf.h"

namespace scsf {

// filter parameter block: {lambda, c, e, -} then the per-step (a_s, b_s) table (k_step_table)
constexpr int FP_TAB = 4, FP_MAX_DEGREE = 256, FP_DOUBLES = FP_TAB + 2 * FP_MAX_DEGREE;
// fp[3]: degree cap of the solver's next filter (k_lock / k_bounds_from_theta, conditioning guard);
// 0 = none (the standalone scsf_cheb_filter).  Every filter kernel runs min(m, cap) steps.
__device__ __forceinline__ int fp_degree_cap(const double* fp, int m) {
  const double cap = fp[3];
  return (cap > 0.5 && cap < (double)m) ? (int)(cap + 0.5) : m;
}

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

// ------------------------------------------------ device-side loops ----
// A loop whose continuation is decided on the device.  On a stream that is being
// captured into a CUDA graph the loop becomes a WHILE conditional node: its body is
// captured once on a side stream into the node's body graph, and the body's last
// kernel sets the condition (dev_loop_continue), so a replay runs as many passes as
// the data needs without the host.  Outside a capture the same body is launched
// pass by pass and the host reads the flag the deciding kernel also writes.
namespace scsf {
struct DevLoop {
  cudaGraphConditionalHandle handle = 0;
  int in_graph = 0;         // 1: set the conditional; 0: only the flag word
  int* flag = nullptr;      // device int written with the decision either way
};
__device__ __forceinline__ void dev_loop_continue(const DevLoop& L, bool more) {
  *L.flag = more ? 1 : 0;
  if (L.in_graph) cudaGraphSetConditional(L.handle, more ? 1u : 0u);
}
bool stream_capturing(cudaStream_t s);
int take_cond_kernels();     // kernels of conditional bodies captured on this thread since the last call
// body(cudaStream_t bs, const DevLoop& L) -> int status; runs while the device says so
// (at least once).  flag_d: one device int; flag_h: one pinned host int (eager mode).
int device_while_impl(cudaStream_t s, int* flag_d, int* flag_h, int (*body)(cudaStream_t, const DevLoop&, void*),
                      void* ctx, int max_passes_eager);
template <class F>
int device_while(cudaStream_t s, int* flag_d, int* flag_h, int max_passes_eager, F& body) {
  auto tramp = [](cudaStream_t bs, const DevLoop& L, void* c) -> int { return (*static_cast<F*>(c))(bs, L); };
  return device_while_impl(s, flag_d, flag_h, tramp, &body, max_passes_eager);
}
}  // namespace scsf

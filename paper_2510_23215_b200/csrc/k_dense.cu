// k_dense.cu — the dense contractions of Alg. 3 on the
// fp64 tensor cores.  sm_100a has no fp64 tcgen05 kind (ptxas rejects
// .kind::f64) and no wgmma, so fp64 tensor math is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA).  Operands are staged in shared memory.
//
//  gemm_tn   C = X^T Y  (tall-skinny "Gram" shape: X n x b1, Y n x b2, reduce over n)
//            split-K over n with fixed-order partial reduction (deterministic):
//            Gram of CholQR (l. 4), Rayleigh quotient G = Q^T A Q (l. 5,
//            P:302), projections V_L^T Y of the block Gram-Schmidt against the
//            locked vectors.
//  gemm_nn   Out = alpha X M + beta Out  (X n x b1, M b1 x b2 small): Y R^{-1}
//            (CholQR), V Z / W Z (l. 6), Y - V_L C.  Each CTA first
//            stages its whole 64-row panel of X in shared memory, so Out may
//            alias X (in-place rotation).
#include "common.cuh"

namespace scsf {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------- gemm_tn ----
constexpr int TN_BM = 64, TN_KC = 16, TN_LDS = TN_KC + 4;

__global__ void __launch_bounds__(128) k_gemm_tn(const double* __restrict__ X, int64_t ldx, int b1,
                                                 const double* __restrict__ Y, int64_t ldy, int b2,
                                                 int64_t n, int64_t kchunk, double* __restrict__ P) {
  __shared__ __align__(16) double xs[TN_BM][TN_LDS];
  __shared__ __align__(16) double ys[TN_BM][TN_LDS];
  const int i0 = blockIdx.x * TN_BM, j0 = blockIdx.y * TN_BM;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(n, kbeg + kchunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int lc = threadIdx.x >> 1;          // column this thread loads (0..63)
  const int lk = (threadIdx.x & 1) * 8;     // 8 consecutive k
  for (int64_t k0 = kbeg; k0 < kend; k0 += TN_KC) {
    {
      const int ci = i0 + lc, cj = j0 + lc;
      const bool full = (k0 + TN_KC <= kend);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int64_t k = k0 + lk + q;
        bool ok = full || k < kend;
        xs[lc][lk + q] = (ok && ci < b1) ? X[k + (int64_t)ci * ldx] : 0.0;
        ys[lc][lk + q] = (ok && cj < b2) ? Y[k + (int64_t)cj * ldy] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TN_KC; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = xs[wm + mi * 8 + g][kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = ys[wn + ni * 8 + g][kk + t];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncthreads();
  }
  double* out = P + (int64_t)blockIdx.z * b1 * b2;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int i = i0 + wm + mi * 8 + g;
        int j = j0 + wn + ni * 8 + 2 * t + e;
        if (i < b1 && j < b2) out[i + (int64_t)j * b1] = acc[mi][ni][e];
      }
}

// C[i + j ldc] = alpha * sum_z P[z][i + j b1]  (z ascending); sym: average with the transpose.
__global__ void k_reduce_partials(const double* __restrict__ P, int splits, int b1, int b2,
                                  double alpha, int sym, double* __restrict__ C, int64_t ldc) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)b1 * b2) return;
  int i = (int)(idx % b1), j = (int)(idx / b1);
  const int64_t stride = (int64_t)b1 * b2;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += P[z * stride + idx];
  if (sym) {
    double s2 = 0.0;
    int64_t tidx = j + (int64_t)i * b1;
    for (int z = 0; z < splits; ++z) s2 += P[z * stride + tidx];
    s = 0.5 * (s + s2);
  }
  C[i + (int64_t)j * ldc] = alpha * s;
}

// ------------------------------------------------------------- gemm_nn ----
constexpr int NN_BM = 64, NN_LDS = NN_BM + 4, NN_BN = 64;
constexpr int NN_MAX_K = 368;

__global__ void __launch_bounds__(128) k_gemm_nn(const double* __restrict__ X, int64_t ldx, int64_t n,
                                                 int b1, const double* __restrict__ M, int64_t ldm,
                                                 int b2, double alpha, double beta, double* Out,
                                                 int64_t ldo) {
  extern __shared__ __align__(16) double xp[];     // [b1r][NN_LDS], k-major panel of X rows
  const int64_t r0 = (int64_t)blockIdx.x * NN_BM;
  const int b1r = (b1 + 3) & ~3;
  // stage the whole row panel (rows r0..r0+63, all b1 columns), zero padded
  for (int idx = threadIdx.x; idx < b1r * NN_BM; idx += blockDim.x) {
    int k = idx / NN_BM, r = idx % NN_BM;
    int64_t rr = r0 + r;
    xp[k * NN_LDS + r] = (k < b1 && rr < n) ? X[rr + (int64_t)k * ldx] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  for (int j0 = 0; j0 < b2; j0 += NN_BN) {
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int k = 0; k < b1r; k += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = xp[(k + t) * NN_LDS + wm + mi * 8 + g];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        int col = j0 + wn + ni * 8 + g;
        b[ni] = (k + t < b1 && col < b2) ? __ldg(M + (k + t) + (int64_t)col * ldm) : 0.0;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int64_t r = r0 + wm + mi * 8 + g;
          int j = j0 + wn + ni * 8 + 2 * t + e;
          if (r < n && j < b2) {
            double* o = Out + r + (int64_t)j * ldo;
            double v = alpha * acc[mi][ni][e];
            if (beta != 0.0) v = fma(beta, *o, v);
            *o = v;
          }
        }
  }
}

// ------------------------------------------------------------------ host ----
static int g_nn_smem_set = 0;

int tn_splits(int64_t n, int b1, int b2) {
  int tiles = ceil_div(b1, TN_BM) * ceil_div(b2, TN_BM);
  int want = max(1, (2 * 148 + tiles - 1) / tiles);
  int maxs = max(1, ceil_div(n, 4 * TN_KC));        // at least 4 chunks per split
  return min(want, maxs);
}

// Upper bound of splits * b1' * b2' over every call with b1' <= b1, b2' <= b2:
// splits <= ceil(296 / tiles) and tiles >= b1' b2' / 64^2, so
// splits * b1' * b2' <= 296 * 64^2 + b1' * b2'.
size_t tn_partial_doubles(int64_t n, int b1, int b2) {
  (void)n;
  return (size_t)2 * 148 * TN_BM * TN_BM + (size_t)b1 * b2;
}

// C (b1 x b2, ldc) = alpha X^T Y.  P: workspace of tn_partial_doubles.
int gemm_tn(const double* X, int64_t ldx, int b1, const double* Y, int64_t ldy, int b2, int64_t n,
            double alpha, int sym, double* C, int64_t ldc, double* P, cudaStream_t s) {
  if (b1 <= 0 || b2 <= 0) return SCSF_OK;
  int splits = tn_splits(n, b1, b2);
  int64_t kchunk = round_up(ceil_div(n, splits), TN_KC);
  splits = ceil_div(n, kchunk);
  dim3 g(ceil_div(b1, TN_BM), ceil_div(b2, TN_BM), splits);
  k_gemm_tn<<<g, 128, 0, s>>>(X, ldx, b1, Y, ldy, b2, n, kchunk, P);
  SCSF_LAUNCH_CHECK();
  k_reduce_partials<<<ceil_div((int64_t)b1 * b2, 256), 256, 0, s>>>(P, splits, b1, b2, alpha, sym, C, ldc);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// Out (n x b2, ldo) = alpha X M + beta Out;  Out may alias X.
int gemm_nn(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
            double alpha, double beta, double* Out, int64_t ldo, cudaStream_t s) {
  if (b2 <= 0 || n <= 0) return SCSF_OK;
  if (b1 > NN_MAX_K) {
    set_error("gemm_nn: inner dimension %d exceeds %d", b1, NN_MAX_K);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  if (!g_nn_smem_set) {
    SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         NN_MAX_K * NN_LDS * (int)sizeof(double)));
    g_nn_smem_set = 1;
  }
  int b1r = (max(b1, 1) + 3) & ~3;
  size_t smem = (size_t)b1r * NN_LDS * sizeof(double);
  k_gemm_nn<<<ceil_div(n, NN_BM), 128, smem, s>>>(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf

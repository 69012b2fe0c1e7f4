// k_stencil.cu — operator-side kernels: FD assembly, Gershgorin bound, the
// fused Chebyshev three-term-recurrence SpMM step (Alg. 1)
// and the column residual norms of Alg. 3 l. 7 (metric P:844).
//
// A is a symmetric 5-/7-point stencil in DIA form (include/scsf.h).  One
// filter step is
//   Y_{s+1} = a_s (A - cI) Y_s + b_s Y_{s-1},
//   a_0 = sigma_1/e, b_0 = 0;  a_s = 2 sigma_{s+1}/e, b_s = -sigma_{s+1} sigma_s,
// i.e. Alg. 1's  Y_{i+1} = 2 sigma_{i+1} A~ Y_i - sigma_{i+1} sigma_i Y_{i-1}
// with A~ = (A - cI)/e folded into the scalars.  The sigma recurrence is
// evaluated on the device from (lambda, c, e) so the host never syncs for it.
// HBM roofline: per point and column 8 B read Y_s, 8 B read Y_{s-1}, 8 B write
// Y_{s+1}; coefficient arrays (8(1+dim) B per point) are shared by all columns
// and stay L2-resident.
#include "common.cuh"

namespace scsf {

// ------------------------------------------------------------- assembly ----
__global__ void k_assemble(int dim, int nx, int ny, int nz, int n_ops, int64_t ld, double inv_h2,
                           const double* __restrict__ fx, const double* __restrict__ fy,
                           const double* __restrict__ fz, const double* __restrict__ c,
                           double* __restrict__ coef) {
  int64_t n = (int64_t)nx * ny * nz;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int op = blockIdx.y;
  if (idx >= ld) return;
  double* out = coef + (int64_t)op * (1 + dim) * ld;
  if (idx >= n) {
    for (int d = 0; d <= dim; ++d) out[d * ld + idx] = 0.0;
    return;
  }
  int i = (int)(idx % nx);
  int j = (int)((idx / nx) % ny);
  int l = (int)(idx / ((int64_t)nx * ny));
  const double* ax = fx + (int64_t)op * nz * ny * (nx + 1);
  const double* ay = fy + (int64_t)op * nz * (ny + 1) * nx;
  double axl = ax[((int64_t)l * ny + j) * (nx + 1) + i];
  double axr = ax[((int64_t)l * ny + j) * (nx + 1) + i + 1];
  double ayl = ay[((int64_t)l * (ny + 1) + j) * nx + i];
  double ayr = ay[((int64_t)l * (ny + 1) + j + 1) * nx + i];
  double diag = axl + axr + ayl + ayr;
  double czv = 0.0, azr = 0.0;
  if (dim == 3) {
    const double* az = fz + (int64_t)op * (nz + 1) * ny * nx;
    double azl = az[((int64_t)l * ny + j) * nx + i];
    azr = az[((int64_t)(l + 1) * ny + j) * nx + i];
    diag += azl + azr;
    czv = (l < nz - 1) ? -azr * inv_h2 : 0.0;
  }
  diag = diag * inv_h2 + (c ? c[(int64_t)op * n + idx] : 0.0);
  out[idx] = diag;
  out[ld + idx] = (i < nx - 1) ? -axr * inv_h2 : 0.0;
  out[2 * ld + idx] = (j < ny - 1) ? -ayr * inv_h2 : 0.0;
  if (dim == 3) out[3 * ld + idx] = czv;
}

// ------------------------------------------------------------ Gershgorin ----
// beta = max_k sum_j |A(k, j)| (reading R10).  Non-negative doubles order like
// their bit patterns, so an integer atomicMax is exact and order-independent.
__global__ void k_gershgorin(const double* __restrict__ cf, int dim, int nx, int ny, int64_t n,
                             int64_t ld, unsigned long long* __restrict__ out) {
  double m = 0.0;
  const int64_t sxy = (int64_t)nx * ny;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double r = fabs(cf[k]) + fabs(cf[ld + k]) + fabs(cf[2 * ld + k]);
    if (k >= 1) r += fabs(cf[ld + k - 1]);
    if (k >= nx) r += fabs(cf[2 * ld + k - nx]);
    if (dim == 3) {
      r += fabs(cf[3 * ld + k]);
      if (k >= sxy) r += fabs(cf[3 * ld + k - sxy]);
    }
    m = fmax(m, r);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------- filter / SpMM step ----
// fp = {lambda, c, e} (device).  step < 0: plain SpMM  Out = A X.
__device__ __forceinline__ void step_scalars(const double* fp, int step, double& a, double& b,
                                             double& c) {
  if (step < 0) {
    a = 1.0; b = 0.0; c = 0.0;
    return;
  }
  double lam = fp[0], cc = fp[1], e = fp[2];
  double s1 = e / (lam - cc);
  c = cc;
  if (step == 0) {
    a = s1 / e; b = 0.0;
    return;
  }
  double sig = s1, prev = s1;
  for (int i = 1; i <= step; ++i) {     // sigma_{i+1} = 1 / (2/sigma_1 - sigma_i)
    prev = sig;
    sig = 1.0 / (2.0 / s1 - sig);
  }
  a = 2.0 * sig / e;
  b = -sig * prev;
}

constexpr int ST_THREADS = 256;
constexpr int ST_COLS = 8;     // columns per CTA sharing the coefficient registers

template <int DIM>
__global__ void __launch_bounds__(ST_THREADS) k_stencil(
    const double* __restrict__ cf, int64_t ldc, int nx, int ny, int64_t n,
    const double* __restrict__ X, const double* Xp, double* Out,   // Out may alias Xp (same-index read-then-write)
    int64_t ldv, int ncols, const double* __restrict__ fp, int step) {
  int64_t k = (int64_t)blockIdx.x * ST_THREADS + threadIdx.x;
  if (k >= n) return;
  double a, b, c;
  step_scalars(fp, step, a, b, c);
  const int64_t sxy = (int64_t)nx * ny;
  const double dg = cf[k] - c;
  const double xp = cf[ldc + k];
  const double xm = (k >= 1) ? cf[ldc + k - 1] : 0.0;
  const double yp = cf[2 * ldc + k];
  const double ym = (k >= nx) ? cf[2 * ldc + k - nx] : 0.0;
  double zp = 0.0, zm = 0.0;
  if (DIM == 3) {
    zp = cf[3 * ldc + k];
    zm = (k >= sxy) ? cf[3 * ldc + k - sxy] : 0.0;
  }
  const bool hp = k + 1 < n, hm = k >= 1, hyp = k + nx < n, hym = k >= nx;
  const bool hzp = (DIM == 3) && (k + sxy < n), hzm = (DIM == 3) && (k >= sxy);
  int j0 = blockIdx.y * ST_COLS;
  int j1 = min(ncols, j0 + ST_COLS);
  for (int j = j0; j < j1; ++j) {
    const double* x = X + (int64_t)j * ldv;
    double v = dg * x[k];
    if (hp) v = fma(xp, x[k + 1], v);
    if (hm) v = fma(xm, x[k - 1], v);
    if (hyp) v = fma(yp, x[k + nx], v);
    if (hym) v = fma(ym, x[k - nx], v);
    if (DIM == 3) {
      if (hzp) v = fma(zp, x[k + sxy], v);
      if (hzm) v = fma(zm, x[k - sxy], v);
    }
    v *= a;
    if (b != 0.0) v = fma(b, Xp[(int64_t)j * ldv + k], v);
    Out[(int64_t)j * ldv + k] = v;
  }
}

// Vectorised variant: 4 consecutive points per thread, 256-bit loads/stores of
// the column streams (Y_s, Y_{s-1}, Y_{s+1}) and the coefficient arrays;
// x-neighbours k-1 / k+4 as scalars (same cache lines), y/z-neighbours as
// aligned 256-bit loads (requires nx % 4 == 0, checked on the host).  The
// coefficients of a quad stay in registers across the CB columns of the CTA.
// Points k >= n (the ld padding) are written as 0 so padding never holds NaN.
constexpr int SV_THREADS = 128;

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256).  ldg4_nc only for data
// that is read-only for the whole kernel (coefficients, X).
__device__ __forceinline__ double4 ldg4_nc(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double4 ldg4(const double* p) {
  double4 v;
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg4(double* p, double4 v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
               : "memory");
}

template <int DIM, int CB>
__global__ void __launch_bounds__(SV_THREADS) k_stencil_v4(
    const double* __restrict__ cf, int64_t ldc, int nx, int ny, int64_t n,
    const double* __restrict__ X, const double* Xp, double* Out,   // Out may alias Xp (same-index RMW)
    int64_t ldv, int ncols, const double* __restrict__ fp, int step) {
  const int64_t k0 = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;
  if (k0 >= ldv) return;
  double a, b, c;
  step_scalars(fp, step, a, b, c);
  const int64_t sxy = (int64_t)nx * ny;
  const int j0 = blockIdx.y * CB;
  const int j1 = min(ncols, j0 + CB);
  if (k0 + 4 <= n) {
    const double4 dg = ldg4_nc(cf + k0);
    const double4 cxp = ldg4_nc(cf + ldc + k0);
    const double cxm = (k0 >= 1) ? cf[ldc + k0 - 1] : 0.0;
    const double4 cyp = ldg4_nc(cf + 2 * ldc + k0);
    const bool hym = k0 >= nx, hyp = k0 + nx + 3 < n;
    const double4 cym = hym ? ldg4_nc(cf + 2 * ldc + k0 - nx) : make_double4(0, 0, 0, 0);
    double4 czp = make_double4(0, 0, 0, 0), czm = make_double4(0, 0, 0, 0);
    bool hzm = false, hzp = false;
    if (DIM == 3) {
      czp = ldg4_nc(cf + 3 * ldc + k0);
      hzm = k0 >= sxy;
      hzp = k0 + sxy + 3 < n;
      if (hzm) czm = ldg4_nc(cf + 3 * ldc + k0 - sxy);
    }
    const bool hm = k0 >= 1, hp = k0 + 4 < n;
#pragma unroll
    for (int jj = 0; jj < CB; ++jj) {
      const int j = j0 + jj;
      if (j >= j1) break;
      const double* __restrict__ x = X + (int64_t)j * ldv;
      const double4 xc = ldg4_nc(x + k0);
      const double xl = hm ? x[k0 - 1] : 0.0;
      const double xr = hp ? x[k0 + 4] : 0.0;
      const double4 xu = hyp ? ldg4_nc(x + k0 + nx) : make_double4(0, 0, 0, 0);
      const double4 xd = hym ? ldg4_nc(x + k0 - nx) : make_double4(0, 0, 0, 0);
      double4 v;
      v.x = (dg.x - c) * xc.x + cxp.x * xc.y + cxm * xl + cyp.x * xu.x + cym.x * xd.x;
      v.y = (dg.y - c) * xc.y + cxp.y * xc.z + cxp.x * xc.x + cyp.y * xu.y + cym.y * xd.y;
      v.z = (dg.z - c) * xc.z + cxp.z * xc.w + cxp.y * xc.y + cyp.z * xu.z + cym.z * xd.z;
      v.w = (dg.w - c) * xc.w + cxp.w * xr + cxp.z * xc.z + cyp.w * xu.w + cym.w * xd.w;
      if (DIM == 3) {
        const double4 zu = hzp ? ldg4_nc(x + k0 + sxy) : make_double4(0, 0, 0, 0);
        const double4 zd = hzm ? ldg4_nc(x + k0 - sxy) : make_double4(0, 0, 0, 0);
        v.x += czp.x * zu.x + czm.x * zd.x;
        v.y += czp.y * zu.y + czm.y * zd.y;
        v.z += czp.z * zu.z + czm.z * zd.z;
        v.w += czp.w * zu.w + czm.w * zd.w;
      }
      v.x *= a; v.y *= a; v.z *= a; v.w *= a;
      if (b != 0.0) {
        const double4 p = ldg4(Xp + (int64_t)j * ldv + k0);
        v.x = fma(b, p.x, v.x); v.y = fma(b, p.y, v.y); v.z = fma(b, p.z, v.z); v.w = fma(b, p.w, v.w);
      }
      stg4(Out + (int64_t)j * ldv + k0, v);
    }
    return;
  }
  // tail quad (n % 4 != 0) and padding: scalar, guarded
  for (int q = 0; q < 4; ++q) {
    const int64_t k = k0 + q;
    if (k >= ldv) break;
    if (k >= n) {
      for (int j = j0; j < j1; ++j) Out[(int64_t)j * ldv + k] = 0.0;
      continue;
    }
    const double dg = cf[k] - c;
    const double xp = cf[ldc + k], xm = (k >= 1) ? cf[ldc + k - 1] : 0.0;
    const double yp = cf[2 * ldc + k], ym = (k >= nx) ? cf[2 * ldc + k - nx] : 0.0;
    double zp = 0.0, zm = 0.0;
    if (DIM == 3) {
      zp = cf[3 * ldc + k];
      zm = (k >= sxy) ? cf[3 * ldc + k - sxy] : 0.0;
    }
    for (int j = j0; j < j1; ++j) {
      const double* x = X + (int64_t)j * ldv;
      double v = dg * x[k];
      if (k + 1 < n) v = fma(xp, x[k + 1], v);
      if (k >= 1) v = fma(xm, x[k - 1], v);
      if (k + nx < n) v = fma(yp, x[k + nx], v);
      if (k >= nx) v = fma(ym, x[k - nx], v);
      if (DIM == 3) {
        if (k + sxy < n) v = fma(zp, x[k + sxy], v);
        if (k >= sxy) v = fma(zm, x[k - sxy], v);
      }
      v *= a;
      if (b != 0.0) v = fma(b, Xp[(int64_t)j * ldv + k], v);
      Out[(int64_t)j * ldv + k] = v;
    }
  }
}

// ------------------------------------------- column-resident filter (2-D) ----
// All m steps of Alg. 1 for one column in one CTA (small grids, n <= RES_MAX_N):
// Y_s double-buffered in shared memory, Y_{s-1} of the thread's own points in
// registers, x-neighbours k +- 1 by warp shuffles (lanes hold consecutive k),
// y-neighbours k +- nx from shared memory.  HBM traffic per filter: read Y_0,
// write Y_m (16 n B per column) + the coefficient arrays (L2-resident, shared
// by all columns).  Bound: shared-memory / L2 bandwidth, not HBM.
constexpr int RES_T = 1024;
constexpr int RES_PPT = 12;
constexpr int RES_MAX_N = RES_T * RES_PPT;     // 12288 (smem 2 * 96 KB)

__global__ void __launch_bounds__(RES_T, 1) k_filter_res2d(const double* __restrict__ cf, int64_t ldc, int nx,
                                                           int n, const double* __restrict__ X, int64_t ldv,
                                                           double* __restrict__ Out, const double* __restrict__ fp,
                                                           int m) {
  extern __shared__ double rbuf[];               // [2][n]
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const double* x0 = X + (int64_t)j * ldv;
  double* out = Out + (int64_t)j * ldv;
  const double lam = fp[0], c = fp[1], e = fp[2];
  const double s1 = e / (lam - c);
  double yprev[RES_PPT];
#pragma unroll
  for (int i = 0; i < RES_PPT; ++i) {
    const int k = tid + RES_T * i;
    yprev[i] = 0.0;
    if (k < n) rbuf[k] = x0[k];
  }
  __syncthreads();
  double sig = s1;
  for (int st = 0; st < m; ++st) {
    double a, bco;
    if (st == 0) {
      a = s1 / e;
      bco = 0.0;
    } else {                                     // same operation sequence as step_scalars()
      const double sn = 1.0 / (2.0 / s1 - sig);
      a = 2.0 * sn / e;
      bco = -sn * sig;
      sig = sn;
    }
    const double* cur = rbuf + (st & 1) * n;
    double* nxt = rbuf + ((st + 1) & 1) * n;
#pragma unroll
    for (int i = 0; i < RES_PPT; ++i) {
      const int k = tid + RES_T * i;
      if (RES_T * i >= n) break;                 // uniform across the CTA
      const bool in = k < n;
      const double xc = in ? cur[k] : 0.0;
      double xl = __shfl_up_sync(0xffffffffu, xc, 1);
      double xr = __shfl_down_sync(0xffffffffu, xc, 1);
      if (lane == 0) xl = (in && k >= 1) ? cur[k - 1] : 0.0;
      if (lane == 31) xr = (k + 1 < n) ? cur[k + 1] : 0.0;
      if (in) {
        const double xd = (k >= nx) ? cur[k - nx] : 0.0;
        const double xu = (k + nx < n) ? cur[k + nx] : 0.0;
        const double cxm = (k >= 1) ? __ldg(cf + ldc + k - 1) : 0.0;
        const double cym = (k >= nx) ? __ldg(cf + 2 * ldc + k - nx) : 0.0;
        double v = (__ldg(cf + k) - c) * xc;
        v = fma(__ldg(cf + ldc + k), xr, v);
        v = fma(cxm, xl, v);
        v = fma(__ldg(cf + 2 * ldc + k), xu, v);
        v = fma(cym, xd, v);
        v *= a;
        if (st > 0) v = fma(bco, yprev[i], v);
        yprev[i] = xc;
        nxt[k] = v;
      }
    }
    __syncthreads();
  }
  const double* fin = rbuf + (m & 1) * n;
  for (int k = tid; k < (int)ldv; k += RES_T) out[k] = (k < n) ? fin[k] : 0.0;
}

// ---------------------------------------------------------- residuals ----
// For active column j: res[j] = ||W_j - theta_j V_j||_2, wn[j] = ||W_j||_2 (fixed-order sums).
__global__ void __launch_bounds__(512) k_resid(const double* __restrict__ V, const double* __restrict__ W,
                                               int64_t ldv, int64_t n, const double* __restrict__ theta,
                                               double* __restrict__ res, double* __restrict__ wn) {
  const int j = blockIdx.x;
  const double* v = V + (int64_t)j * ldv;
  const double* w = W + (int64_t)j * ldv;
  const double th = theta[j];
  double r2 = 0.0, w2 = 0.0;
  const int64_t n2 = n & ~(int64_t)1;                 // ld is even: 16-byte aligned pairs
#pragma unroll 4
  for (int64_t k = 2 * threadIdx.x; k < n2; k += 2 * blockDim.x) {
    const double2 wk = *reinterpret_cast<const double2*>(w + k);
    const double2 vk = *reinterpret_cast<const double2*>(v + k);
    const double d0 = fma(-th, vk.x, wk.x), d1 = fma(-th, vk.y, wk.y);
    r2 = fma(d0, d0, r2);
    r2 = fma(d1, d1, r2);
    w2 = fma(wk.x, wk.x, w2);
    w2 = fma(wk.y, wk.y, w2);
  }
  if (threadIdx.x == 0 && n2 < n) {
    const double d = fma(-th, v[n - 1], w[n - 1]);
    r2 = fma(d, d, r2);
    w2 = fma(w[n - 1], w[n - 1], w2);
  }
  __shared__ double sr[16], sw[16];
  r2 = warp_sum(r2);
  w2 = warp_sum(w2);
  if ((threadIdx.x & 31) == 0) {
    sr[threadIdx.x >> 5] = r2;
    sw[threadIdx.x >> 5] = w2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, bb = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a += sr[i];
      bb += sw[i];
    }
    res[j] = sqrt(a);
    wn[j] = sqrt(bb);
  }
}

// ------------------------------------------------------------------ host ----
int assemble_impl(const scsf_ops* ops, double h, const double* fx, const double* fy,
                  const double* fz, const double* c, double* coef, cudaStream_t s) {
  dim3 g(ceil_div(ops->ld, 256), ops->n_ops);
  k_assemble<<<g, 256, 0, s>>>(ops->dim, ops->nx, ops->ny, ops->nz, ops->n_ops, ops->ld,
                               1.0 / (h * h), fx, fy, fz, c, coef);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int gershgorin_impl(const scsf_ops* ops, int op, unsigned long long* out, cudaStream_t s) {
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  const double* cf = ops->coef + (int64_t)op * (1 + ops->dim) * ops->ld;
  SCSF_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
  int blocks = min(ceil_div(n, 256), 148 * 4);
  k_gershgorin<<<blocks, 256, 0, s>>>(cf, ops->dim, ops->nx, ops->ny, n, ops->ld, out);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

static int g_res_attr = 0;
bool filter_resident_ok(const scsf_ops* ops) {
  return ops->dim == 2 && (int64_t)ops->nx * ops->ny <= RES_MAX_N;
}

// Whole filter (steps 0..m-1) for ncols columns of X into Out, column-resident kernel.
int filter_resident_impl(const scsf_ops* ops, int op, const double* X, double* Out, int64_t ldv, int ncols,
                         const double* fp, int m, cudaStream_t s) {
  if (ncols <= 0) return SCSF_OK;
  const int n = ops->nx * ops->ny;
  const double* cf = ops->coef + (int64_t)op * (1 + ops->dim) * ops->ld;
  if (!g_res_attr) {
    SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_res2d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * RES_MAX_N * (int)sizeof(double)));
    g_res_attr = 1;
  }
  k_filter_res2d<<<ncols, RES_T, (size_t)2 * n * sizeof(double), s>>>(cf, ops->ld, ops->nx, n, X, ldv, Out, fp, m);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// Out[:, 0:ncols] = step-th filter update (or A X when step < 0).
int stencil_impl(const scsf_ops* ops, int op, const double* X, const double* Xp, double* Out,
                 int64_t ldv, int ncols, const double* fp, int step, cudaStream_t s) {
  if (ncols <= 0) return SCSF_OK;
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  const double* cf = ops->coef + (int64_t)op * (1 + ops->dim) * ops->ld;
  const bool vec = (ops->nx % 4 == 0) && (ldv % 4 == 0) && (ops->ld % 4 == 0) &&
                   ((uintptr_t)X % 32 == 0) && ((uintptr_t)Out % 32 == 0) && ((uintptr_t)cf % 32 == 0) &&
                   (Xp == nullptr || (uintptr_t)Xp % 32 == 0);
  if (vec) {
    constexpr int CB = 2;     // 2 columns per CTA: ~5x more CTAs than CB = 4, enough warps to hide latency
    dim3 g(ceil_div(ceil_div(ldv, 4), SV_THREADS), ceil_div(ncols, CB));
    if (ops->dim == 2)
      k_stencil_v4<2, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step);
    else
      k_stencil_v4<3, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step);
  } else {
    dim3 g(ceil_div(n, ST_THREADS), ceil_div(ncols, ST_COLS));
    if (ops->dim == 2)
      k_stencil<2><<<g, ST_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step);
    else
      k_stencil<3><<<g, ST_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step);
  }
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int resid_impl(const double* V, const double* W, int64_t ldv, int64_t n, int ncols,
               const double* theta, double* res, double* wn, cudaStream_t s) {
  if (ncols <= 0) return SCSF_OK;
  k_resid<<<ncols, 512, 0, s>>>(V, W, ldv, n, theta, res, wn);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf

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

#include <atomic>
#include <type_traits>
#include <mutex>

#include <cooperative_groups.h>

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
// fp = {lambda, c, e, -, a_0, b_0, a_1, b_1, ...} (device; FP_DOUBLES).  step < 0: plain SpMM
// Out = A X.  The per-step scalars a_s, b_s are tabulated once per filter by k_step_table
// (step_table_impl, launched before the first step), so a step kernel reads two broadcast values
// instead of every thread re-running the sigma recurrence up to its step (O(m) divisions each).
// Returns false for a step at or past the degree cap (fp[3]): the kernel then does nothing (the cap
// is = m (mod 3), so the filter's last output still lands in the buffer Y_m would).
__device__ __forceinline__ bool step_scalars(const double* fp, int step, double& a, double& b,
                                             double& c) {
  if (step < 0) {
    a = 1.0; b = 0.0; c = 0.0;
    return true;
  }
  if (step >= fp_degree_cap(fp, FP_MAX_DEGREE)) return false;
  c = fp[1];
  a = fp[FP_TAB + 2 * step];
  b = fp[FP_TAB + 2 * step + 1];
  return true;
}

// Alg. 1's scalars for steps 0..m-1 (one thread; the recurrence is sequential):
//   a_0 = sigma_1 / e, b_0 = 0;  a_s = 2 sigma_{s+1} / e, b_s = -sigma_{s+1} sigma_s,
//   sigma_1 = e / (lambda - c), sigma_{i+1} = 1 / (2 / sigma_1 - sigma_i).
__global__ void k_step_table(double* fp, int m) {
  if (threadIdx.x != 0) return;
  const double lam = fp[0], cc = fp[1], e = fp[2];
  const double s1 = e / (lam - cc);
  fp[FP_TAB] = s1 / e;
  fp[FP_TAB + 1] = 0.0;
  double sig = s1;
  for (int st = 1; st < m; ++st) {
    const double prev = sig;
    sig = 1.0 / (2.0 / s1 - sig);
    fp[FP_TAB + 2 * st] = 2.0 * sig / e;
    fp[FP_TAB + 2 * st + 1] = -sig * prev;
  }
}

int step_table_impl(double* fp, int m, cudaStream_t s) {
  k_step_table<<<1, 32, 0, s>>>(fp, m);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
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
  if (!step_scalars(fp, step, a, b, c)) return;
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

// ------------------------------------------------ vibration (13-point) ----
// Standard form of the thin-plate pencil (reading R25; include/scsf.h
// SCSF_STENCIL_VIB13): B = S Lh diag(D) Lh S, S = diag(rho)^-1/2, Lh = (4 - neighbours)/h^2.
// Entries of Lh diag(D) Lh written out per stencil offset (the sum over the shared
// neighbours m of Lh(k,m) D_m Lh(m,l)):
//   l = k        16 D_k + sum_{m in-grid x/y neighbour of k} D_m
//   l = k+1      -4 (D_k + D_{k+1})           (same grid row)
//   l = k+2      D_{k+1}                      (same grid row)
//   l = k+nx-1   D_{k-1} + D_{k+nx}           (ix >= 1, iy < ny-1)
//   l = k+nx     -4 (D_k + D_{k+nx})
//   l = k+nx+1   D_{k+1} + D_{k+nx}           (ix < nx-1, iy < ny-1)
//   l = k+2nx    D_{k+nx}
// all / h^4, then times (rho_k rho_l)^-1/2.
__global__ void k_assemble_vib(int nx, int ny, int64_t ld, double inv_h4, const double* __restrict__ D,
                               const double* __restrict__ rho, int64_t fstride, double* __restrict__ coef) {
  const int64_t n = (int64_t)nx * ny;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int op = blockIdx.y;
  if (k >= ld) return;
  double* out = coef + (int64_t)op * 7 * ld;
  if (k >= n) {
    for (int d = 0; d < 7; ++d) out[d * ld + k] = 0.0;
    return;
  }
  const double* d = D + (int64_t)op * fstride;
  const double* r = rho + (int64_t)op * fstride;
  const int i = (int)(k % nx), j = (int)(k / nx);
  const double sk = 1.0 / sqrt(r[k]);
  auto s = [&](int64_t l) { return 1.0 / sqrt(r[l]); };
  double dg = 16.0 * d[k];
  if (i > 0) dg += d[k - 1];
  if (i < nx - 1) dg += d[k + 1];
  if (j > 0) dg += d[k - nx];
  if (j < ny - 1) dg += d[k + nx];
  out[k] = dg * inv_h4 * sk * sk;
  out[ld + k] = (i < nx - 1) ? -4.0 * (d[k] + d[k + 1]) * inv_h4 * sk * s(k + 1) : 0.0;
  out[2 * ld + k] = (i < nx - 2) ? d[k + 1] * inv_h4 * sk * s(k + 2) : 0.0;
  out[3 * ld + k] = (i > 0 && j < ny - 1) ? (d[k - 1] + d[k + nx]) * inv_h4 * sk * s(k + nx - 1) : 0.0;
  out[4 * ld + k] = (j < ny - 1) ? -4.0 * (d[k] + d[k + nx]) * inv_h4 * sk * s(k + nx) : 0.0;
  out[5 * ld + k] = (i < nx - 1 && j < ny - 1) ? (d[k + 1] + d[k + nx]) * inv_h4 * sk * s(k + nx + 1) : 0.0;
  out[6 * ld + k] = (j < ny - 2) ? d[k + nx] * inv_h4 * sk * s(k + 2 * nx) : 0.0;
}

// Gershgorin row sums of the 13-point stencil (upper arrays at k, lower ones at k - offset).
__global__ void k_gershgorin_vib(const double* __restrict__ cf, int nx, int64_t n, int64_t ld,
                                 unsigned long long* __restrict__ out) {
  const int64_t off[6] = {1, 2, nx - 1, nx, nx + 1, 2 * (int64_t)nx};
  double m = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double r = fabs(cf[k]);
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      r += fabs(cf[(a + 1) * ld + k]);
      if (k >= off[a]) r += fabs(cf[(a + 1) * ld + k - off[a]]);
    }
    m = fmax(m, r);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// One filter step (or A X) with the 13-point stencil.  One point per thread, VB_COLS columns
// per CTA sharing the 13 coefficient registers; the x-values of the 12 neighbours come through
// L1/L2 (a column is nx*ny*8 B, re-read from cache by the neighbouring threads).  Zero
// coefficients make the in-row wrap-arounds harmless; only the [0, n) range is guarded.
constexpr int VB_THREADS = 256;
constexpr int VB_COLS = 4;
__global__ void __launch_bounds__(VB_THREADS) k_stencil_vib(
    const double* __restrict__ cf, int64_t ldc, int nx, int64_t n, const double* __restrict__ X, const double* Xp,
    double* Out, int64_t ldv, int ncols, const double* __restrict__ fp, int step) {
  const int64_t k = (int64_t)blockIdx.x * VB_THREADS + threadIdx.x;
  if (k >= ldv) return;
  const int j0 = blockIdx.y * VB_COLS, j1 = min(ncols, j0 + VB_COLS);
  if (k >= n) {                                        // ld padding stays 0
    for (int j = j0; j < j1; ++j) Out[(int64_t)j * ldv + k] = 0.0;
    return;
  }
  double a, b, c;
  if (!step_scalars(fp, step, a, b, c)) return;
  const int64_t o1 = 1, o2 = 2, o3 = nx - 1, o4 = nx, o5 = nx + 1, o6 = 2 * (int64_t)nx;
  const double dg = cf[k] - c;
  const double u1 = cf[ldc + k], u2 = cf[2 * ldc + k], u3 = cf[3 * ldc + k], u4 = cf[4 * ldc + k],
               u5 = cf[5 * ldc + k], u6 = cf[6 * ldc + k];
  const double l1 = k >= o1 ? cf[ldc + k - o1] : 0.0, l2 = k >= o2 ? cf[2 * ldc + k - o2] : 0.0;
  const double l3 = k >= o3 ? cf[3 * ldc + k - o3] : 0.0, l4 = k >= o4 ? cf[4 * ldc + k - o4] : 0.0;
  const double l5 = k >= o5 ? cf[5 * ldc + k - o5] : 0.0, l6 = k >= o6 ? cf[6 * ldc + k - o6] : 0.0;
  for (int j = j0; j < j1; ++j) {
    const double* __restrict__ x = X + (int64_t)j * ldv;
    double v = dg * x[k];
    if (k + o1 < n) v = fma(u1, x[k + o1], v);
    if (k + o2 < n) v = fma(u2, x[k + o2], v);
    if (k + o3 < n) v = fma(u3, x[k + o3], v);
    if (k + o4 < n) v = fma(u4, x[k + o4], v);
    if (k + o5 < n) v = fma(u5, x[k + o5], v);
    if (k + o6 < n) v = fma(u6, x[k + o6], v);
    if (k >= o1) v = fma(l1, x[k - o1], v);
    if (k >= o2) v = fma(l2, x[k - o2], v);
    if (k >= o3) v = fma(l3, x[k - o3], v);
    if (k >= o4) v = fma(l4, x[k - o4], v);
    if (k >= o5) v = fma(l5, x[k - o5], v);
    if (k >= o6) v = fma(l6, x[k - o6], v);
    v *= a;
    if (b != 0.0) v = fma(b, Xp[(int64_t)j * ldv + k], v);
    Out[(int64_t)j * ldv + k] = v;
  }
}

// 13-point step with the row band staged in shared memory: a CTA owns VT_R grid rows for VT_CB
// columns and stages those rows plus two halo rows each side of every column; every point then
// reads its 12 neighbours from shared memory and its 13 coefficients through L1 once for all
// VT_CB columns (k_stencil_vib reads every neighbour with its own 8-byte global load: ncu
// long_scoreboard, 0.24 of the HBM rate on V1).  Flat-index neighbours wrap across row ends
// exactly where the stencil's coefficients are zero, as in the DIA layout.  V1 (32 chains):
// 11.8 -> 14.1 operators/s; staging the coefficients as well (56 KB per CTA) was slower (9.1),
// and VT_R = 4 / 8 / 16 gave 13.2 / 13.9 / 14.1, VT_CB = 8 13.2.
constexpr int VT_T = 256, VT_R = 16, VT_CB = 4;

__global__ void __launch_bounds__(VT_T) k_stencil_vib_t(const double* __restrict__ cf, int64_t ldc, int nx, int ny,
                                                      const double* __restrict__ X, const double* Xp, double* Out,
                                                      int64_t ldv, int ncols, const double* __restrict__ fp, int step) {
  extern __shared__ __align__(16) double vs[];
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * VT_R, rows = min(VT_R, ny - r0);
  const int j0 = blockIdx.y * VT_CB, ncb = min(VT_CB, ncols - j0);
  const int n = nx * ny;
  const int VW = (VT_R + 4) * nx;
  double* sv = vs;                                  // [VT_CB][VW]: rows r0-2 .. r0+VT_R+1

  double a, b, c;
  if (!step_scalars(fp, step, a, b, c)) return;
  const int vbase = (r0 - 2) * nx;
  for (int i = tid; i < VW; i += VT_T) {
    const int k = vbase + i;
    const bool in = k >= 0 && k < n;
#pragma unroll
    for (int cc = 0; cc < VT_CB; ++cc)
      sv[cc * VW + i] = (in && cc < ncb) ? __ldg(X + (int64_t)(j0 + cc) * ldv + k) : 0.0;
  }
  __syncthreads();
  const int o2 = 2, o3 = nx - 1, o4 = nx, o5 = nx + 1, o6 = 2 * nx;
  for (int i = tid; i < rows * nx; i += VT_T) {
    const int lv = 2 * nx + i, lc = 2 * nx + i;    // local index of the point in sv / sc
    const int64_t k = (int64_t)r0 * nx + i;
    (void)lc;
    const double* ck = cf + k;
    const double dg = __ldg(ck) - c;
    const double u1 = __ldg(ck + ldc), u2 = __ldg(ck + 2 * ldc), u3 = __ldg(ck + 3 * ldc), u4 = __ldg(ck + 4 * ldc),
                 u5 = __ldg(ck + 5 * ldc), u6 = __ldg(ck + 6 * ldc);
    const double l1 = k >= 1 ? __ldg(ck + ldc - 1) : 0.0, l2 = k >= o2 ? __ldg(ck + 2 * ldc - o2) : 0.0,
                 l3 = k >= o3 ? __ldg(ck + 3 * ldc - o3) : 0.0, l4 = k >= o4 ? __ldg(ck + 4 * ldc - o4) : 0.0,
                 l5 = k >= o5 ? __ldg(ck + 5 * ldc - o5) : 0.0, l6 = k >= o6 ? __ldg(ck + 6 * ldc - o6) : 0.0;
#pragma unroll
    for (int cc = 0; cc < VT_CB; ++cc) {
      if (cc >= ncb) break;
      const double* x = sv + cc * VW + lv;
      double v = dg * x[0];
      v = fma(u1, x[1], v);
      v = fma(u2, x[o2], v);
      v = fma(u3, x[o3], v);
      v = fma(u4, x[o4], v);
      v = fma(u5, x[o5], v);
      v = fma(u6, x[o6], v);
      v = fma(l1, x[-1], v);
      v = fma(l2, x[-o2], v);
      v = fma(l3, x[-o3], v);
      v = fma(l4, x[-o4], v);
      v = fma(l5, x[-o5], v);
      v = fma(l6, x[-o6], v);
      v *= a;
      if (b != 0.0) v = fma(b, Xp[(int64_t)(j0 + cc) * ldv + k], v);
      Out[(int64_t)(j0 + cc) * ldv + k] = v;
    }
  }
  if (r0 + VT_R >= ny)                               // last band: the ld padding stays 0
    for (int cc = 0; cc < ncb; ++cc)
      for (int64_t k = n + tid; k < ldv; k += VT_T) Out[(int64_t)(j0 + cc) * ldv + k] = 0.0;
}
static size_t vib_t_smem(int nx) { return (size_t)(VT_CB * (VT_R + 4)) * nx * sizeof(double); }

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
    int64_t ldv, int ncols, const double* __restrict__ fp, int step, const int* __restrict__ deg) {
  const int64_t k0 = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;
  if (k0 >= ldv) return;
  double a, b, c;
  if (!step_scalars(fp, step, a, b, c)) return;
  const int64_t sxy = (int64_t)nx * ny;
  int j0 = blockIdx.y * CB;
  const int j1 = min(ncols, j0 + CB);
  // SURVEY f2 (Alg. 1 l. 5's staggered update): a column whose degree deg[j] <= step is finished
  // and left untouched; degrees are non-decreasing in j, so the finished ones are a prefix
  if (deg)
    while (j0 < j1 && __ldg(deg + j0) <= step) ++j0;
  if (j0 >= j1) return;
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

// ---- streaming step with grouped loads (k_stencil_v4g).  Same arithmetic as k_stencil_v4 (bitwise:
// the same expressions in the same order), but for each group of G columns every global load of
// the group is issued before any arithmetic, and the stores carry no compiler memory barrier, so
// a thread keeps G columns of loads (up to 6 x 32 B each) in flight instead of one column's.
__device__ __forceinline__ double4 ldg4_rd(const double* p) {     // Y_{s-1}: read once, before its own store
  double4 v;
  asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg4_nb(double* p, double4 v) {    // no "memory" clobber
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w));
}

template <int DIM, int CB, int G>
__global__ void __launch_bounds__(SV_THREADS) k_stencil_v4g(
    const double* __restrict__ cf, int64_t ldc, int nx, int ny, int64_t n,
    const double* __restrict__ X, const double* Xp, double* Out,   // Out may alias Xp (same-index RMW)
    int64_t ldv, int ncols, const double* __restrict__ fp, int step, const int* __restrict__ deg) {
  const int64_t k0 = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;
  if (k0 >= ldv) return;
  double a, b, c;
  if (!step_scalars(fp, step, a, b, c)) return;
  const int64_t sxy = (int64_t)nx * ny;
  int j0 = blockIdx.y * CB;
  const int j1 = min(ncols, j0 + CB);
  if (deg)
    while (j0 < j1 && __ldg(deg + j0) <= step) ++j0;
  if (j0 >= j1) return;
  if (k0 + 4 > n) {                                  // tail quad / padding: the plain kernel's path
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
    return;
  }
  const double4 z4 = make_double4(0, 0, 0, 0);
  const double4 dg = ldg4_nc(cf + k0);
  const double4 cxp = ldg4_nc(cf + ldc + k0);
  const double cxm = (k0 >= 1) ? cf[ldc + k0 - 1] : 0.0;
  const double4 cyp = ldg4_nc(cf + 2 * ldc + k0);
  const bool hym = k0 >= nx, hyp = k0 + nx + 3 < n;
  const double4 cym = hym ? ldg4_nc(cf + 2 * ldc + k0 - nx) : z4;
  double4 czp = z4, czm = z4;
  bool hzm = false, hzp = false;
  if (DIM == 3) {
    czp = ldg4_nc(cf + 3 * ldc + k0);
    hzm = k0 >= sxy;
    hzp = k0 + sxy + 3 < n;
    if (hzm) czm = ldg4_nc(cf + 3 * ldc + k0 - sxy);
  }
  const bool hm = k0 >= 1, hp = k0 + 4 < n;
  const bool usep = b != 0.0;
#pragma unroll
  for (int g0 = 0; g0 < CB; g0 += G) {
    double4 xc[G], xu[G], xd[G], zu[G], zd[G], pp[G];
    double xl[G], xr[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {                    // every load of the group first
      const int j = j0 + g0 + q;
      if (j < j1) {
        const double* __restrict__ x = X + (int64_t)j * ldv;
        xc[q] = ldg4_nc(x + k0);
        xl[q] = hm ? __ldg(x + k0 - 1) : 0.0;
        xr[q] = hp ? __ldg(x + k0 + 4) : 0.0;
        xu[q] = hyp ? ldg4_nc(x + k0 + nx) : z4;
        xd[q] = hym ? ldg4_nc(x + k0 - nx) : z4;
        if (DIM == 3) {
          zu[q] = hzp ? ldg4_nc(x + k0 + sxy) : z4;
          zd[q] = hzm ? ldg4_nc(x + k0 - sxy) : z4;
        }
        pp[q] = usep ? ldg4_rd(Xp + (int64_t)j * ldv + k0) : z4;
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int j = j0 + g0 + q;
      if (j < j1) {
        double4 v;
        v.x = (dg.x - c) * xc[q].x + cxp.x * xc[q].y + cxm * xl[q] + cyp.x * xu[q].x + cym.x * xd[q].x;
        v.y = (dg.y - c) * xc[q].y + cxp.y * xc[q].z + cxp.x * xc[q].x + cyp.y * xu[q].y + cym.y * xd[q].y;
        v.z = (dg.z - c) * xc[q].z + cxp.z * xc[q].w + cxp.y * xc[q].y + cyp.z * xu[q].z + cym.z * xd[q].z;
        v.w = (dg.w - c) * xc[q].w + cxp.w * xr[q] + cxp.z * xc[q].z + cyp.w * xu[q].w + cym.w * xd[q].w;
        if (DIM == 3) {
          v.x += czp.x * zu[q].x + czm.x * zd[q].x;
          v.y += czp.y * zu[q].y + czm.y * zd[q].y;
          v.z += czp.z * zu[q].z + czm.z * zd[q].z;
          v.w += czp.w * zu[q].w + czm.w * zd[q].w;
        }
        v.x *= a; v.y *= a; v.z *= a; v.w *= a;
        if (usep) {
          v.x = fma(b, pp[q].x, v.x); v.y = fma(b, pp[q].y, v.y); v.z = fma(b, pp[q].z, v.z); v.w = fma(b, pp[q].w, v.w);
        }
        stg4_nb(Out + (int64_t)j * ldv + k0, v);
      }
    }
  }
}

// Columns whose loads are issued together.  Measured (tools/bench_filter.py, streaming filter at
// m = 20, fraction of the measured HBM copy rate, plain k_stencil_v4 / G = 1 / 2 / 4):
// C3 0.71 / 0.80 / 0.85 / 0.64, C4 (3-D) 0.51 / 0.66 / 0.53 / 0.48, C5 0.84 / 0.94 / 0.98 / 0.70
// (profiles/r02_stencil_groups.json); default G = 2 in 2-D (124 registers), G = 1 in 3-D (126;
// G = 2 needs 204 and halves the resident warps).  SCSF_V4_GROUP = 0 (plain), 1, 2, 4 overrides.
static int v4_group(int dim) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("SCSF_V4_GROUP");
    v = e ? atoi(e) : -1;
    if (v != 0 && v != 1 && v != 2 && v != 4) v = -1;
  }
  return v >= 0 ? v : (dim == 2 ? 2 : 1);
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
  m = fp_degree_cap(fp, m);
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

__device__ __forceinline__ double4 lds4(const double* p) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void sts4(double* p, double4 v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v.z, v.w);
}

// --------------------------------------- cluster-resident filter (2-D) ----
// All m steps of Alg. 1 for CB columns on a thread-block cluster of CS CTAs:
// CTA r of the cluster owns grid rows [r R, r R + R) (R = ceil(ny / CS), even)
// of CB consecutive columns.  Everything the recurrence touches stays on chip:
//  - a thread owns a 2 x 2 patch: rows 2p, 2p+1 at x = 2q, 2q+1.  Lanes run
//    along x, so every shared access is a 16-byte vector at a 16-byte stride
//    (bank-conflict free) and the x-neighbours come from the adjacent lanes by
//    shuffle (lane 0 / 31 read shared memory; across a row end the coupling cx
//    is 0).  The patch's coefficients (diag, cx, cy, cx(k-1), cy(k-nx)) live
//    in registers, loaded once per filter and shared by the CB columns; the
//    upper row's cy(k-nx) is the lower row's cy;
//  - Y_s and Y_{s-1} of each column live in two shared buffers of R + 2 rows
//    (one ghost row each side); Y_{s-1} is read from the target buffer
//    (written two steps ago), so no vector state survives a step in registers;
//  - the producer pushes its boundary rows into the neighbouring CTAs' ghost
//    rows (distributed shared-memory stores) as it computes them, so one
//    cluster barrier per step is the only synchronisation; Dirichlet ghost
//    rows stay zero.
// HBM traffic per filter and column: read Y_0, write Y_m (16 n B) plus the
// coefficient arrays once per CB columns.  Bound: shared-memory bandwidth
// (~32 B per point per step) and the cluster barrier (amortised over CB).
constexpr int CL_T = 768;                        // max threads per CTA (<= 80 registers: 6 warps per SMSP quadrant)
constexpr int CL_MAXP = CL_T;                    // 2 x 2 patches per CTA

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// the two halves (every thread of the cluster alternates arrive / wait; warp-uniform call sites)
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// 32-bit shared-memory accesses (volatile: they must not move across the cluster barrier)
__device__ __forceinline__ double2 lds2a(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds1a(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2a(unsigned a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// ---- tensor memory (TMEM) helpers (tcgen05; sm_100a).  A warp w reaches TMEM lanes
// 32 (w % 4) .. 32 (w % 4) + 31; each lane is one thread, columns are 32-bit words.
__device__ __forceinline__ void tmem_ld16(unsigned taddr, double2& a, double2& b, double2& c, double2& d) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  auto d2 = [&](int i) { return __hiloint2double((int)r[i + 1], (int)r[i]); };
  a = make_double2(d2(0), d2(2));
  b = make_double2(d2(4), d2(6));
  c = make_double2(d2(8), d2(10));
  d = make_double2(d2(12), d2(14));
}
__device__ __forceinline__ void tmem_st8(unsigned taddr, double2 a, double2 b) {
  const unsigned r0 = (unsigned)__double2loint(a.x), r1 = (unsigned)__double2hiint(a.x);
  const unsigned r2 = (unsigned)__double2loint(a.y), r3 = (unsigned)__double2hiint(a.y);
  const unsigned r4 = (unsigned)__double2loint(b.x), r5 = (unsigned)__double2hiint(b.x);
  const unsigned r6 = (unsigned)__double2loint(b.y), r7 = (unsigned)__double2hiint(b.y);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(r4), "r"(r5), "r"(r6), "r"(r7)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// distributed shared memory: 32-bit shared::cluster addresses (mapa) and stores
__device__ __forceinline__ unsigned mapa32(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void stc2a(unsigned a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// asynchronous store into a neighbour CTA's shared memory that completes `16` transaction bytes on the
// neighbour's mbarrier (address a + d, barrier mb; both shared::cluster): no cluster-wide fence needed
__device__ __forceinline__ void stc2_async(unsigned a, unsigned d, unsigned mb, double2 v) {
  asm volatile("{\n\t.reg .u32 t;\n\tadd.u32 t, %0, %1;\n\t"
               "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [t], {%3, %4}, [%2];\n\t}"
               ::"r"(a), "r"(d), "r"(mb), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mb_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// wait for the phase of the given parity; traps after 2^26 polls (seconds; a step takes microseconds, and
// a cluster's CTAs are co-resident) instead of hanging the GPU
__device__ __forceinline__ void mb_wait_cluster(unsigned bar, unsigned parity) {
  unsigned done = 0;
  for (unsigned it = 0;; ++it) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) break;
    if (it > (1u << 26)) __trap();
  }
}
// the same store at a + d, the add inside the asm: the compiler cannot hoist (and spill) a + d per column
__device__ __forceinline__ void stc2ad(unsigned a, unsigned d, double2 v) {
  asm volatile("{\n\t.reg .u32 t;\n\tadd.u32 t, %0, %1;\n\tst.shared::cluster.v2.f64 [t], {%2, %3};\n\t}"
               ::"r"(a), "r"(d), "d"(v.x), "d"(v.y) : "memory");
}

// TM: the thread's own patch rows of Y_s and Y_{s-1} live in tensor memory (two 8-word slots per
// column, roles swapped every step) instead of being re-read from the shared buffers: per step and
// column the shared-memory pipe serves only the rows below / above the patch, its stores and the
// warp-edge x-neighbours (2 + edge loads instead of 6).
template <int CS, int CB, bool TM = false>
__global__ void __launch_bounds__(CL_T, 1) k_filter_cl(const double* __restrict__ cf, int64_t ldc, int nx, int ny,
                                                       const double* __restrict__ X, int64_t ldv, int ncols,
                                                       double* __restrict__ Out, const double* __restrict__ fp, int m,
                                                       const int* __restrict__ deg, int split) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double cbuf[];           // [CB][2][R + 2][nx]
  __shared__ double sa[FP_MAX_DEGREE], sb[FP_MAX_DEGREE]; // per-step scalars (m <= FP_MAX_DEGREE)
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int j0 = blockIdx.y * CB, tid = threadIdx.x, lane = tid & 31, nthr = blockDim.x;
  m = fp_degree_cap(fp, m);                               // conditioning guard (k_lock)
  const int R = ((ny + CS - 1) / CS + 1) & ~1;
  const int row0 = rank * R;
  const int rows = max(0, min(R, ny - row0));
  const int hx = nx >> 1;                                  // 2-point segments per row
  const int npatch = ((rows + 1) >> 1) * hx;
  const int pitch = (R + 2) * nx;                          // one buffer of one column
  const int n = nx * ny;
  const int ncb = min(CB, ncols - j0);                     // columns of this CTA (uniform)
  // per-column degree (deg == NULL: uniform m), uniform across the cluster
  int mcol[CB];
  int mrun = 0;
#pragma unroll
  for (int cc = 0; cc < CB; ++cc) {
    mcol[cc] = (cc < ncb) ? (deg ? max(1, min(m, deg[j0 + cc])) : m) : 0;
    mrun = max(mrun, mcol[cc]);
  }
  const double c = fp[1];
  if (tid == 0) {                                          // Alg. 1 scalars, same operation sequence as step_scalars()
    const double lam = fp[0], e = fp[2];
    const double s1 = e / (lam - c);
    double sig = s1;
    sa[0] = s1 / e;
    sb[0] = 0.0;
    for (int st = 1; st < m && st < FP_MAX_DEGREE; ++st) {
      const double sn = 1.0 / (2.0 / s1 - sig);
      sa[st] = 2.0 * sn / e;
      sb[st] = -sn * sig;
      sig = sn;
    }
  }
  const bool has_lo = rank > 0;
  const bool has_hi = (rank + 1 < CS) && (row0 + R < ny);
  double* lo_buf = has_lo ? cluster.map_shared_rank(cbuf, rank - 1) : nullptr;   // CTA below
  double* hi_buf = has_hi ? cluster.map_shared_rank(cbuf, rank + 1) : nullptr;   // CTA above
  // split == 2: one mbarrier per buffer parity receives the neighbours' ghost-row pushes (st.async)
  __shared__ __align__(8) unsigned long long gmb[2];
  if (split == 2 && tid == 0) {
    mb_init((unsigned)__cvta_generic_to_shared(&gmb[0]), 1);
    mb_init((unsigned)__cvta_generic_to_shared(&gmb[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // all buffers zero: Dirichlet ghost rows, and Y_{-1} = 0 for the first step's (bco = 0) term
  for (int i = tid; i < CB * pitch; i += nthr) sts2(cbuf + 2 * i, make_double2(0.0, 0.0));
  cluster_barrier();                                       // every CTA of the cluster is running and zeroed
  for (int cc = 0; cc < ncb; ++cc) {                       // Y_0 (own rows; boundary rows also to the neighbours)
    const double* x0 = X + (int64_t)(j0 + cc) * ldv + (int64_t)row0 * nx;
    double* b0 = cbuf + (size_t)(2 * cc) * pitch;
    for (int q = tid; q < rows * hx; q += nthr) {
      const double2 v = *reinterpret_cast<const double2*>(x0 + 2 * q);
      sts2(b0 + nx + 2 * q, v);
      const int lr = q / hx, xq = 2 * (q % hx);
      if (lr == 0 && lo_buf) sts2(lo_buf + (size_t)(2 * cc) * pitch + (R + 1) * nx + xq, v);
      if (lr == rows - 1 && hi_buf) sts2(hi_buf + (size_t)(2 * cc) * pitch + xq, v);
    }
  }
  // this thread's patch: local rows lr0, lr0 + 1; x = xq, xq + 1.  Inactive threads compute on
  // a valid patch (the last one) and store nothing, so the step loop has no divergent branches.
  const bool act = tid < npatch;
  const int pt = min(tid, max(npatch - 1, 0));
  const int lr0 = 2 * (pt / hx), xq = 2 * (pt % hx);
  const bool up_ok = act && (lr0 + 1 < rows);
  const int g0 = (row0 + lr0) * nx + xq;
  const double2 z2 = make_double2(0, 0);
  double2 dg0 = z2, dg1 = z2, cxp0 = z2, cxp1 = z2, cyp0 = z2, cyp1 = z2, cym0 = z2;
  double cxm0 = 0.0, cxm1 = 0.0;
  if (npatch > 0) {
    dg0 = *reinterpret_cast<const double2*>(cf + g0);
    cxp0 = *reinterpret_cast<const double2*>(cf + ldc + g0);
    cxm0 = (g0 >= 1) ? __ldg(cf + ldc + g0 - 1) : 0.0;
    cyp0 = *reinterpret_cast<const double2*>(cf + 2 * ldc + g0);
    cym0 = (g0 >= nx) ? *reinterpret_cast<const double2*>(cf + 2 * ldc + g0 - nx) : z2;
    dg0.x -= c; dg0.y -= c;
    if (lr0 + 1 < rows) {
      const int g1 = g0 + nx;
      dg1 = *reinterpret_cast<const double2*>(cf + g1);
      cxp1 = *reinterpret_cast<const double2*>(cf + ldc + g1);
      cxm1 = __ldg(cf + ldc + g1 - 1);
      cyp1 = *reinterpret_cast<const double2*>(cf + 2 * ldc + g1);
      dg1.x -= c; dg1.y -= c;
    }
  }
  const bool push_lo0 = act && lo_buf && lr0 == 0;
  const bool push_hi0 = act && hi_buf && lr0 == rows - 1;          // lower row is the last row (rows odd)
  const bool push_hi1 = up_ok && hi_buf && lr0 + 1 == rows - 1;    // upper row is the last row
  const bool fix_l = (lane == 0) || (xq == 0);                     // left neighbour not in the lane below
  const bool fix_r = (lane == 31) || (xq + 2 == nx) || (tid + 1 >= npatch);
  // 32-bit shared addresses of the patch in both buffers of every column
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(cbuf);
  const int l0 = (lr0 + 1) * nx + xq;                      // local index of the lower row (ghost row 0 first)
  const unsigned nx8 = 8u * nx;
  const unsigned up8 = up_ok ? 2u * nx8 : nx8;             // upper neighbour of the upper row (dummy if absent)
  unsigned acur[CB], anxt[CB];
#pragma unroll
  for (int cc = 0; cc < CB; ++cc) {
    acur[cc] = sbase + 8u * (unsigned)((2 * cc) * pitch + l0);
    anxt[cc] = sbase + 8u * (unsigned)((2 * cc + 1) * pitch + l0);
  }
  // shared::cluster addresses: the lower row of my patch in the CTA below's top ghost row,
  // and my row(s) in the CTA above's bottom ghost row, as deltas to my own target address
  const unsigned lo32 = has_lo ? mapa32(sbase, rank - 1) : 0u, hi32 = has_hi ? mapa32(sbase, rank + 1) : 0u;
  const unsigned dlo = lo32 - sbase + (unsigned)R * nx8;                 // local row 0 -> row R + 1 below
  // local row rows - 1 -> row 0 above; the same (CTA-uniform) delta serves a lower row (push_hi0,
  // lr0 = rows - 1) and an upper row (push_hi1, at na + nx8)
  const unsigned dhi = hi32 - sbase - (unsigned)rows * nx8;
  cluster_barrier();                                       // also publishes sa / sb
  __shared__ unsigned tm_base_s;
  unsigned tbase = 0;                                      // this thread's TMEM address (lane, column 0)
  // columns: CB x 16 words per warp of a lane quadrant, rounded up to a power of two >= 32 (a CTA
  // takes only what it needs, so two CTAs of a small slab can share the SM's 512 columns)
  unsigned tm_cols = 32;
  while (tm_cols < (unsigned)(((nthr / 32 + 3) / 4) * CB * 16)) tm_cols <<= 1;
  if (TM) {
    if ((tid >> 5) == 0) {
      const unsigned sa32 = (unsigned)__cvta_generic_to_shared(&tm_base_s);
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(sa32), "r"(tm_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int w = tid >> 5;
    tbase = tm_base_s + ((unsigned)(32 * (w & 3)) << 16) + (unsigned)((w >> 2) * CB * 16);
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {                      // slot 0: Y_0 (own rows), slot 1: Y_{-1} = 0
      tmem_st8(tbase + cc * 16, lds2a(acur[cc]), lds2a(acur[cc] + nx8));
      tmem_st8(tbase + cc * 16 + 8, z2, z2);
    }
    tmem_wait_st();
  }
  // One step of Alg. 1 for the CB columns.  PAR = st & 1 is a compile-time constant (the loop
  // below runs two steps per trip), so the buffer roles and the TMEM slot roles are static: a
  // stepped column's buffers swap every step, hence at step st its current buffer is 2 cc + PAR
  // (a column past its own degree is not stepped again; its final buffer is mcol & 1).  With the
  // parity in a register the compiler spent 16 FSEL per column and step on the slot swap.
  const bool push_any = push_lo0 || push_hi0 || push_hi1;
  const unsigned abuf0 = sbase + 8u * (unsigned)l0, pitch8 = 8u * (unsigned)pitch;
  // split == 2: my mbarriers (gmb[p] receives the pushes into buffer p) and the deltas to the neighbours'
  const unsigned gmb32 = (unsigned)__cvta_generic_to_shared(&gmb[0]);
  const unsigned dmb_lo = has_lo ? mapa32(gmb32, rank - 1) - gmb32 : 0u;
  const unsigned dmb_hi = has_hi ? mapa32(gmb32, rank + 1) - gmb32 : 0u;
  auto step = [&](auto par, int st) {
    constexpr int PAR = decltype(par)::value;
    const double a = sa[st], bco = sb[st];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
      if (st < mcol[cc]) {                                 // uniform across the CTA (0 beyond ncb)
        // buffer b of column cc starts b * pitch doubles after buffer 0: 2 cc + PAR is current
        const unsigned ca = abuf0 + (unsigned)(2 * cc + PAR) * pitch8, na = abuf0 + (unsigned)(2 * cc + 1 - PAR) * pitch8;
        const double2 xd = lds2a(ca - nx8);
        double2 xa, xb, p0, p1;
        if (TM) {
          double2 q0, q1;
          tmem_ld16(tbase + cc * 16, q0, q1, p0, p1);      // both slots: Y_s and Y_{s-1}
          if (PAR) {
            xa = p0; xb = p1; p0 = q0; p1 = q1;
          } else {
            xa = q0; xb = q1;
          }
          if (!up_ok) xb = lds2a(ca + nx8);                // no upper row: the ghost row above
        } else {
          xa = lds2a(ca);
          xb = lds2a(ca + nx8);
        }
        const double2 xu = lds2a(ca + up8);
        double xal = __shfl_up_sync(0xffffffffu, xa.y, 1), xar = __shfl_down_sync(0xffffffffu, xa.x, 1);
        double xbl = __shfl_up_sync(0xffffffffu, xb.y, 1), xbr = __shfl_down_sync(0xffffffffu, xb.x, 1);
        if (fix_l) {
          xal = lds1a(ca - 8u);
          xbl = lds1a(ca + nx8 - 8u);
        }
        if (fix_r) {
          xar = lds1a(ca + 16u);
          xbr = lds1a(ca + nx8 + 16u);
        }
        double2 v, u;
        v.x = fma(dg0.x, xa.x, fma(cxp0.x, xa.y, fma(cxm0, xal, fma(cyp0.x, xb.x, cym0.x * xd.x))));
        v.y = fma(dg0.y, xa.y, fma(cxp0.y, xar, fma(cxp0.x, xa.x, fma(cyp0.y, xb.y, cym0.y * xd.y))));
        u.x = fma(dg1.x, xb.x, fma(cxp1.x, xb.y, fma(cxm1, xbl, fma(cyp1.x, xu.x, cyp0.x * xa.x))));
        u.y = fma(dg1.y, xb.y, fma(cxp1.y, xbr, fma(cxp1.x, xb.x, fma(cyp1.y, xu.y, cyp0.y * xa.y))));
        // Y_{s-1} sits in the target buffer (zero at s = 0: bco = 0 there, and the buffer holds finite values)
        if (!TM) {
          p0 = lds2a(na);
          p1 = lds2a(na + nx8);
        }
        v.x = fma(bco, p0.x, a * v.x); v.y = fma(bco, p0.y, a * v.y);
        u.x = fma(bco, p1.x, a * u.x); u.y = fma(bco, p1.y, a * u.y);
        if (act) sts2a(na, v);
        if (up_ok) sts2a(na + nx8, u);
        // boundary rows into the neighbours' ghost rows (same buffer layout: fixed address deltas);
        // a branch, not predication: only the warps holding a slab's first / last row take it
        if (push_any) {
          if (split == 2) {                                // st.async completing bytes on the receiver's
            if (st + 1 < mcol[cc]) {                       // mbarrier; no push after a column's last step
              const unsigned mbo = gmb32 + 8u * (unsigned)(1 - PAR);
              if (push_lo0) stc2_async(na, dlo, mbo + dmb_lo, v);
              if (push_hi0) stc2_async(na, dhi, mbo + dmb_hi, v);
              if (push_hi1) stc2_async(na, nx8 + dhi, mbo + dmb_hi, u);
            }
          } else {
            if (push_lo0) stc2ad(na, dlo, v);
            if (push_hi0) stc2ad(na, dhi, v);
            if (push_hi1) stc2ad(na, nx8 + dhi, u);
          }
        }
        if (TM) tmem_st8(tbase + cc * 16 + 8 * (1 - PAR), v, u);   // Y_{s+1} replaces Y_{s-1}
      }
    }
    if (TM) tmem_wait_st();
  };
  // Step synchronisation.  Default: one cluster barrier per step (nxt and the pushed ghost rows complete
  // cluster-wide).  split != 0: the barrier is split into arrive / wait, and only the warps that read a
  // ghost row (a patch in the slab's first or last patch row; warp-uniform, so shuffles and the .aligned
  // barriers stay converged) wait for the cluster before computing a step; the interior warps compute the
  // step right after the CTA barrier and wait afterwards, so the cluster-barrier latency overlaps their
  // work.  Ordering: the interior rows a warp reads come from its own CTA (__syncthreads of the previous
  // step); ghost rows are pushed by the neighbours' edge warps before their arrive (release) and read
  // after my wait (acquire); a push of step s + 1 into buffer ca(s) happens after the pusher's wait of
  // step s, i.e. after every thread of this CTA finished reading ca(s) in step s.
  const bool edge_w = __any_sync(0xffffffffu, (lr0 == 0) || (lr0 + 2 >= rows));
  // split == 2 (neighbour sync): no cluster barrier in the loop.  The ghost rows a step reads were pushed
  // by the neighbours' previous step with st.async, which completes transaction bytes on this CTA's
  // mbarrier of that buffer; thread 0 arms it (arrive.expect_tx with the bytes the neighbours will push)
  // one step ahead, the edge warps wait on it, the CTA synchronises once per step.  A neighbour pushes
  // into buffer p again (two steps later) only after it received this CTA's pushes of the step between,
  // which each pushing thread issues after reading its ghost values: no ghost row is overwritten early.
  // (the CTA below pushes only if this slab has rows: an empty top CTA of the cluster receives nothing)
  const unsigned row_bytes = 8u * (unsigned)nx * (unsigned)((has_lo && rows > 0 ? 1 : 0) + (has_hi ? 1 : 0));
  auto pre = [&](int st) {
    if (split == 2) {
      if (tid == 0) {                                      // arm gmb[na parity] for this step's pushes
        unsigned cols = 0;
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) cols += (st + 1 < mcol[cc]) ? 1u : 0u;
        mb_arrive_tx(gmb32 + 8u * (unsigned)((st + 1) & 1), cols * row_bytes);
      }
      if (st > 0 && edge_w) mb_wait_cluster(gmb32 + 8u * (unsigned)(st & 1), (unsigned)((st - 1) >> 1) & 1u);
      return;
    }
    if (split && st > 0 && edge_w) cluster_wait();
  };
  auto post = [&](int st) {
    if (split == 2) {
      __syncthreads();
    } else if (split) {
      if (st > 0 && !edge_w) cluster_wait();
      cluster_arrive();
      __syncthreads();
    } else {
      cluster_barrier();
    }
  };
  for (int st = 0; st < mrun; st += 2) {
    pre(st);
    step(std::integral_constant<int, 0>{}, st);
    post(st);
    if (st + 1 < mrun) {
      pre(st + 1);
      step(std::integral_constant<int, 1>{}, st + 1);
      post(st + 1);
    }
  }
  if (split == 2) cluster_barrier();                       // nothing in flight; no CTA leaves early
  else if (split && mrun > 0) cluster_wait();              // the last arrive: no CTA leaves while pushed to
  if (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if ((tid >> 5) == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm_base_s), "r"(tm_cols)
                   : "memory");
  }
  for (int cc = 0; cc < ncb; ++cc) {
    const double* fin = cbuf + (size_t)(2 * cc + (mcol[cc] & 1)) * pitch;
    double* out = Out + (int64_t)(j0 + cc) * ldv;
    for (int q = tid; q < rows * hx; q += nthr)
      *reinterpret_cast<double2*>(out + row0 * nx + 2 * q) = lds2(fin + nx + 2 * q);
    if (rank == (int)cluster.num_blocks() - 1)             // ld padding of the column (last CTA launched)
      for (int k = n + tid; k < (int)ldv; k += nthr) out[k] = 0.0;
  }
}

// ---------------------------------------------------------------------------------------
// k_filter_rp: the cluster-resident filter with register-resident 2 x 4 patches.  Same
// slab / ghost-row / DSMEM layout as k_filter_cl, but a thread keeps its patch of Y_s and
// Y_{s-1} (4 rows x 2 points) in registers for all m steps, so per step it reads only the
// rows just below and above its patch from shared memory (plus x-neighbours across warp
// edges) and stores its new rows for the neighbours: 2 loads + 4 stores + 8 shuffles per
// 8 points against 6 loads + 2 stores + 4 shuffles per 4 points in k_filter_cl (ncu: that
// kernel stalls on the shared-memory instruction queue, mio_throttle; this one halves the
// shared wavefronts, but at 168 registers a 352-thread CTA fills the register file, so it
// only wins where k_filter_cl has few threads per column: see cluster_size_rp).
constexpr int RP_T = 384;                        // max threads (patches) per CTA (<= 170 registers)
constexpr int RP_ROWS = 4;

template <int CS, int CB>
__global__ void __launch_bounds__(RP_T, 1) k_filter_rp(const double* __restrict__ cf, int64_t ldc, int nx, int ny,
                                                       const double* __restrict__ X, int64_t ldv, int ncols,
                                                       double* __restrict__ Out, const double* __restrict__ fp, int m,
                                                       const int* __restrict__ deg, int /*split: k_filter_cl only*/) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double cbuf[];           // [CB][2][R + 2][nx]
  __shared__ double sa[FP_MAX_DEGREE], sb[FP_MAX_DEGREE];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int j0 = blockIdx.y * CB, tid = threadIdx.x, lane = tid & 31, nthr = blockDim.x;
  m = fp_degree_cap(fp, m);                               // conditioning guard (k_lock)
  const int R = ((ny + CS - 1) / CS + RP_ROWS - 1) / RP_ROWS * RP_ROWS;
  const int row0 = rank * R;
  const int rows = max(0, min(R, ny - row0));
  const int hx = nx >> 1;
  const int npatch = ((rows + RP_ROWS - 1) / RP_ROWS) * hx;
  const int pitch = (R + 2) * nx;
  const int n = nx * ny;
  const int ncb = min(CB, ncols - j0);
  int mcol[CB];
  int mrun = 0;
#pragma unroll
  for (int cc = 0; cc < CB; ++cc) {
    mcol[cc] = (cc < ncb) ? (deg ? max(1, min(m, deg[j0 + cc])) : m) : 0;
    mrun = max(mrun, mcol[cc]);
  }
  const double c = fp[1];
  if (tid == 0) {                                          // Alg. 1 scalars, as step_scalars()
    const double lam = fp[0], e = fp[2];
    const double s1 = e / (lam - c);
    double sig = s1;
    sa[0] = s1 / e;
    sb[0] = 0.0;
    for (int st = 1; st < m && st < FP_MAX_DEGREE; ++st) {
      const double sn = 1.0 / (2.0 / s1 - sig);
      sa[st] = 2.0 * sn / e;
      sb[st] = -sn * sig;
      sig = sn;
    }
  }
  const bool has_lo = rank > 0;
  const bool has_hi = (rank + 1 < CS) && (row0 + R < ny);
  double* lo_buf = has_lo ? cluster.map_shared_rank(cbuf, rank - 1) : nullptr;
  double* hi_buf = has_hi ? cluster.map_shared_rank(cbuf, rank + 1) : nullptr;
  for (int i = tid; i < CB * pitch; i += nthr) sts2(cbuf + 2 * i, make_double2(0.0, 0.0));
  cluster_barrier();
  for (int cc = 0; cc < ncb; ++cc) {                       // Y_0 into buffer 0 (own rows + neighbours' ghosts)
    const double* x0 = X + (int64_t)(j0 + cc) * ldv + (int64_t)row0 * nx;
    double* b0 = cbuf + (size_t)(2 * cc) * pitch;
    for (int q = tid; q < rows * hx; q += nthr) {
      const double2 v = *reinterpret_cast<const double2*>(x0 + 2 * q);
      sts2(b0 + nx + 2 * q, v);
      const int lr = q / hx, xq = 2 * (q % hx);
      if (lr == 0 && lo_buf) sts2(lo_buf + (size_t)(2 * cc) * pitch + (R + 1) * nx + xq, v);
      if (lr == rows - 1 && hi_buf) sts2(hi_buf + (size_t)(2 * cc) * pitch + xq, v);
    }
  }
  const bool act = tid < npatch;
  const int pt = min(tid, max(npatch - 1, 0));
  const int lr0 = RP_ROWS * (pt / hx), xq = 2 * (pt % hx);
  const int nr = act ? min(RP_ROWS, rows - lr0) : 0;       // valid rows of this patch
  const int g0 = (row0 + lr0) * nx + xq;
  const double2 z2 = make_double2(0, 0);
  double2 dg[RP_ROWS], cxp[RP_ROWS], cyp[RP_ROWS];
  double cxm[RP_ROWS];
  double2 cym0 = z2;
#pragma unroll
  for (int r = 0; r < RP_ROWS; ++r) {
    dg[r] = z2; cxp[r] = z2; cyp[r] = z2; cxm[r] = 0.0;
    if (npatch > 0 && lr0 + r < rows) {
      const int g = g0 + r * nx;
      dg[r] = *reinterpret_cast<const double2*>(cf + g);
      dg[r].x -= c; dg[r].y -= c;
      cxp[r] = *reinterpret_cast<const double2*>(cf + ldc + g);
      cxm[r] = (g >= 1) ? __ldg(cf + ldc + g - 1) : 0.0;
      cyp[r] = *reinterpret_cast<const double2*>(cf + 2 * ldc + g);
    }
  }
  if (npatch > 0 && g0 >= nx) cym0 = *reinterpret_cast<const double2*>(cf + 2 * ldc + g0 - nx);
  const bool fix_l = (lane == 0) || (xq == 0);
  const bool fix_r = (lane == 31) || (xq + 2 == nx) || (tid + 1 >= npatch);
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(cbuf);
  const int l0 = (lr0 + 1) * nx + xq;                      // buffer index of the patch's row 0
  const unsigned nx8 = 8u * nx;
  unsigned acur[CB], anxt[CB];
  double2 cur[CB][RP_ROWS], prv[CB][RP_ROWS];
#pragma unroll
  for (int cc = 0; cc < CB; ++cc) {
    acur[cc] = sbase + 8u * (unsigned)((2 * cc) * pitch + l0);
    anxt[cc] = sbase + 8u * (unsigned)((2 * cc + 1) * pitch + l0);
#pragma unroll
    for (int r = 0; r < RP_ROWS; ++r) {
      prv[cc][r] = z2;
      cur[cc][r] = (cc < ncb && r < nr)
                       ? *reinterpret_cast<const double2*>(X + (int64_t)(j0 + cc) * ldv + g0 + r * nx) : z2;
    }
  }
  const unsigned lo32 = has_lo ? mapa32(sbase, rank - 1) : 0u, hi32 = has_hi ? mapa32(sbase, rank + 1) : 0u;
  const unsigned dlo = lo32 - sbase + (unsigned)R * nx8;               // my row 0 -> row R + 1 below
  const unsigned dhi = hi32 - sbase - (unsigned)rows * nx8;            // my top slab row -> row 0 above
  const bool push_lo = act && has_lo && lr0 == 0;
  const int rtop = (act && has_hi) ? rows - 1 - lr0 : -1;              // patch row that is the slab's top row
  cluster_barrier();                                       // neighbours' ghosts of Y_0, sa / sb
  for (int st = 0; st < mrun; ++st) {
    const double a = sa[st], bco = sb[st];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
      if (st < mcol[cc]) {                                 // uniform across the CTA
        const unsigned ca = acur[cc], na = anxt[cc];
        const double2 xd = lds2a(ca - nx8);                // row below the patch (ghost / other patch)
        const double2 xu = lds2a(ca + RP_ROWS * nx8);      // row above the patch
        double2 nw[RP_ROWS];
#pragma unroll
        for (int r = 0; r < RP_ROWS; ++r) {
          const double2 xc = cur[cc][r];
          double xl = __shfl_up_sync(0xffffffffu, xc.y, 1), xr = __shfl_down_sync(0xffffffffu, xc.x, 1);
          if (fix_l) xl = lds1a(ca + r * nx8 - 8u);
          if (fix_r) xr = lds1a(ca + r * nx8 + 16u);
          const double2 bl = (r == 0) ? xd : cur[cc][r - 1];
          const double2 ab = (r == RP_ROWS - 1) ? xu : cur[cc][r + 1];
          const double2 cb = (r == 0) ? cym0 : cyp[r - 1];
          double2 v;
          v.x = fma(dg[r].x, xc.x, fma(cxp[r].x, xc.y, fma(cxm[r], xl, fma(cyp[r].x, ab.x, cb.x * bl.x))));
          v.y = fma(dg[r].y, xc.y, fma(cxp[r].y, xr, fma(cxp[r].x, xc.x, fma(cyp[r].y, ab.y, cb.y * bl.y))));
          v.x = fma(bco, prv[cc][r].x, a * v.x);
          v.y = fma(bco, prv[cc][r].y, a * v.y);
          nw[r] = (r < nr) ? v : z2;                       // rows past the slab stay 0 (Dirichlet)
        }
#pragma unroll
        for (int r = 0; r < RP_ROWS; ++r) {
          prv[cc][r] = cur[cc][r];
          cur[cc][r] = nw[r];
          if (r < nr) sts2a(na + r * nx8, nw[r]);
          if (r == rtop) stc2a(na + r * nx8 + dhi, nw[r]);
        }
        if (push_lo) stc2a(na + dlo, nw[0]);
        acur[cc] = na;
        anxt[cc] = ca;
      }
    }
    cluster_barrier();                                     // new rows and pushed ghosts complete cluster-wide
  }
#pragma unroll
  for (int cc = 0; cc < CB; ++cc) {
    if (cc < ncb) {
      double* out = Out + (int64_t)(j0 + cc) * ldv;
#pragma unroll
      for (int r = 0; r < RP_ROWS; ++r)
        if (r < nr) *reinterpret_cast<double2*>(out + g0 + r * nx) = cur[cc][r];
      if (rank == CS - 1)
        for (int k = n + tid; k < (int)ldv; k += nthr) out[k] = 0.0;
    }
  }
}

// W = A V fused with the residual norms of Alg. 3 l. 7: per column j the squared norms of
// w - theta_j v and of w are summed per CTA (fixed order) into partials P[(2 j + {0,1}) nblk + cta]
// and k_resid_sum adds the nblk partials in ascending order.  W itself is never written (after
// the rotation it only feeds the residuals).  nx % 4 == 0 (no tail quads); padding adds 0.
template <int DIM, int CB>
__global__ void __launch_bounds__(SV_THREADS) k_stencil_resid(
    const double* __restrict__ cf, int64_t ldc, int nx, int ny, int64_t n, const double* __restrict__ X,
    int64_t ldv, int ncols, const double* __restrict__ theta, double* __restrict__ P, int nblk) {
  const int64_t k0 = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;
  const int64_t sxy = (int64_t)nx * ny;
  const int j0 = blockIdx.y * CB;
  double rr[CB], ww[CB];
#pragma unroll
  for (int jj = 0; jj < CB; ++jj) rr[jj] = ww[jj] = 0.0;
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
      if (j >= ncols) break;
      const double* __restrict__ x = X + (int64_t)j * ldv;
      const double4 xc = ldg4_nc(x + k0);
      const double xl = hm ? x[k0 - 1] : 0.0;
      const double xr = hp ? x[k0 + 4] : 0.0;
      const double4 xu = hyp ? ldg4_nc(x + k0 + nx) : make_double4(0, 0, 0, 0);
      const double4 xd = hym ? ldg4_nc(x + k0 - nx) : make_double4(0, 0, 0, 0);
      double4 v;
      v.x = dg.x * xc.x + cxp.x * xc.y + cxm * xl + cyp.x * xu.x + cym.x * xd.x;
      v.y = dg.y * xc.y + cxp.y * xc.z + cxp.x * xc.x + cyp.y * xu.y + cym.y * xd.y;
      v.z = dg.z * xc.z + cxp.z * xc.w + cxp.y * xc.y + cyp.z * xu.z + cym.z * xd.z;
      v.w = dg.w * xc.w + cxp.w * xr + cxp.z * xc.z + cyp.w * xu.w + cym.w * xd.w;
      if (DIM == 3) {
        const double4 zu = hzp ? ldg4_nc(x + k0 + sxy) : make_double4(0, 0, 0, 0);
        const double4 zd = hzm ? ldg4_nc(x + k0 - sxy) : make_double4(0, 0, 0, 0);
        v.x += czp.x * zu.x + czm.x * zd.x;
        v.y += czp.y * zu.y + czm.y * zd.y;
        v.z += czp.z * zu.z + czm.z * zd.z;
        v.w += czp.w * zu.w + czm.w * zd.w;
      }
      const double th = theta[j];
      const double d0 = fma(-th, xc.x, v.x), d1 = fma(-th, xc.y, v.y), d2 = fma(-th, xc.z, v.z),
                   d3 = fma(-th, xc.w, v.w);
      rr[jj] = fma(d0, d0, fma(d1, d1, fma(d2, d2, d3 * d3)));
      ww[jj] = fma(v.x, v.x, fma(v.y, v.y, fma(v.z, v.z, v.w * v.w)));
    }
  }
  __shared__ double red[2 * CB][SV_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int jj = 0; jj < CB; ++jj) {
    const double r = warp_sum(rr[jj]), w = warp_sum(ww[jj]);
    if (lane == 0) {
      red[2 * jj][warp] = r;
      red[2 * jj + 1][warp] = w;
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * CB) {
    const int jj = threadIdx.x >> 1, j = j0 + jj;
    if (j < ncols) {
      double t = 0.0;
      for (int q = 0; q < SV_THREADS / 32; ++q) t += red[threadIdx.x][q];
      P[(int64_t)(2 * j + (threadIdx.x & 1)) * nblk + blockIdx.x] = t;
    }
  }
}

__global__ void k_resid_sum(const double* __restrict__ P, int nblk, double* __restrict__ res, double* __restrict__ wn) {
  const int j = blockIdx.x;
  if (threadIdx.x >= 2) return;
  const double* p = P + (int64_t)(2 * j + threadIdx.x) * nblk;
  double t = 0.0;
  for (int q = 0; q < nblk; ++q) t += p[q];
  if (threadIdx.x == 0) res[j] = t;
  else wn[j] = t;
}

// Residual norms from V without materialising W = A V (flux stencils, nx % 4 == 0, no row
// partition); returns false when the caller must use stencil_impl + resid_impl instead.
// doubles of P that k_stencil_resid writes for ncols columns of ld ldv (2 partial sums per CTA)
size_t resid_partial_doubles(int64_t ldv, int ncols) {
  return (size_t)2 * ncols * ceil_div(ceil_div(ldv, 4), SV_THREADS);
}

int stencil_resid_impl(const scsf_ops* ops, int op, const double* V, int64_t ldv, int ncols, const double* theta,
                       double* res, double* wn, double* P, cudaStream_t s, bool* done) {
  *done = false;
  if (ncols <= 0) { *done = true; return SCSF_OK; }
  const double* cf = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
  if (ops->stencil != SCSF_STENCIL_FLUX || ops->nx % 4 != 0 || ldv % 4 != 0 || ops->ld % 4 != 0 ||
      ((uintptr_t)V % 32) != 0 || ((uintptr_t)cf % 32) != 0)
    return SCSF_OK;
  const int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  constexpr int CB = 4;
  const int nblk = (int)ceil_div(ceil_div(ldv, 4), SV_THREADS);
  dim3 g(nblk, ceil_div(ncols, CB));
  if (ops->dim == 2)
    k_stencil_resid<2, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, V, ldv, ncols, theta, P, nblk);
  else
    k_stencil_resid<3, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, V, ldv, ncols, theta, P, nblk);
  SCSF_LAUNCH_CHECK();
  k_resid_sum<<<ncols, 32, 0, s>>>(P, nblk, res, wn);
  SCSF_LAUNCH_CHECK();
  *done = true;
  return SCSF_OK;
}

// ------------------------------------------------ row-partitioned (slab) ----
// Row partition of a 2-D operator: this rank owns grid rows
// [y0, y1); vectors hold only those n_loc = nx (y1 - y0) rows, the operator
// arrays stay global (coefficient index = goff + local index, goff = y0 nx).
// The rows just outside the slab come from the neighbours' boundary rows
// (halo, comm.cu): ghost_lo [ncols][nx] = row y0 - 1, ghost_hi = row y1.
// pack: send_lo [ncols][nx] = first own row, send_hi = last own row.
__global__ void k_pack_rows(const double* __restrict__ X, int64_t ldv, int64_t n_loc, int nx, int ncols,
                            double* __restrict__ send_lo, double* __restrict__ send_hi) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (x >= nx || j >= ncols) return;
  const double* col = X + (int64_t)j * ldv;
  send_lo[(int64_t)j * nx + x] = col[x];
  send_hi[(int64_t)j * nx + x] = col[n_loc - nx + x];
}

// One filter step (or A X when step < 0) on a slab, 4 points per thread (nx % 4 == 0).
template <int CB>
__global__ void __launch_bounds__(SV_THREADS) k_stencil_slab(
    const double* __restrict__ cf, int64_t ldc, int nx, int64_t n_glob, int64_t goff, int64_t n_loc,
    const double* __restrict__ X, const double* Xp, double* Out, int64_t ldv, int ncols,
    const double* __restrict__ ghost_lo, const double* __restrict__ ghost_hi, const double* __restrict__ fp,
    int step, int64_t l_begin, int64_t l_end, const int* __restrict__ deg) {
  const int64_t l0 = l_begin + ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) * 4;   // local point
  if (l0 >= l_end) return;
  double a, b, c;
  if (!step_scalars(fp, step, a, b, c)) return;
  const int j0 = blockIdx.y * CB;
  const int j1 = min(ncols, j0 + CB);
  // per-column degrees (deg != NULL only for filter steps): a column past its degree is
  // left untouched (its last output already sits in the buffer of Y_m, k_lock's mod-3 rounding)
  auto live = [&](int j) { return j < j1 && (deg == nullptr || step < __ldg(deg + j)); };
  if (l0 >= n_loc) {                                  // ld padding
    for (int j = j0; j < j1; ++j)
      if (live(j)) stg4(Out + (int64_t)j * ldv + l0, make_double4(0, 0, 0, 0));
    return;
  }
  const int64_t k0 = goff + l0;                       // global point
  const double4 dg = ldg4_nc(cf + k0);
  const double4 cxp = ldg4_nc(cf + ldc + k0);
  const double cxm = (k0 >= 1) ? cf[ldc + k0 - 1] : 0.0;
  const double4 cyp = ldg4_nc(cf + 2 * ldc + k0);
  const bool hym = k0 >= nx, hyp = k0 + nx < n_glob;  // global Dirichlet boundary
  const double4 cym = hym ? ldg4_nc(cf + 2 * ldc + k0 - nx) : make_double4(0, 0, 0, 0);
  const bool hm = l0 >= 1, hp = l0 + 4 < n_loc;       // x-neighbours never leave the slab row
  const bool dn_in = l0 >= nx, up_in = l0 + nx < n_loc;
  const bool usep = b != 0.0;
  const double4 z4 = make_double4(0, 0, 0, 0);
  // two columns at a time, every load of the pair issued before any arithmetic (as k_stencil_v4g)
  constexpr int G = 2;
#pragma unroll
  for (int g0 = 0; g0 < CB; g0 += G) {
    double4 xc[G], xu[G], xd[G], pp[G];
    double xl[G], xr[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int j = j0 + g0 + q;
      if (live(j)) {
        const double* __restrict__ x = X + (int64_t)j * ldv;
        xc[q] = ldg4_nc(x + l0);
        xl[q] = hm ? __ldg(x + l0 - 1) : 0.0;
        xr[q] = hp ? __ldg(x + l0 + 4) : 0.0;
        xu[q] = z4;
        xd[q] = z4;
        if (hyp) xu[q] = up_in ? ldg4_nc(x + l0 + nx) : ldg4_nc(ghost_hi + (int64_t)j * nx + (l0 + nx - n_loc));
        if (hym) xd[q] = dn_in ? ldg4_nc(x + l0 - nx) : ldg4_nc(ghost_lo + (int64_t)j * nx + l0);
        pp[q] = usep ? ldg4_rd(Xp + (int64_t)j * ldv + l0) : z4;
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int j = j0 + g0 + q;
      if (live(j)) {
        double4 v;
        v.x = (dg.x - c) * xc[q].x + cxp.x * xc[q].y + cxm * xl[q] + cyp.x * xu[q].x + cym.x * xd[q].x;
        v.y = (dg.y - c) * xc[q].y + cxp.y * xc[q].z + cxp.x * xc[q].x + cyp.y * xu[q].y + cym.y * xd[q].y;
        v.z = (dg.z - c) * xc[q].z + cxp.z * xc[q].w + cxp.y * xc[q].y + cyp.z * xu[q].z + cym.z * xd[q].z;
        v.w = (dg.w - c) * xc[q].w + cxp.w * xr[q] + cxp.z * xc[q].z + cyp.w * xu[q].w + cym.w * xd[q].w;
        v.x *= a; v.y *= a; v.z *= a; v.w *= a;
        if (usep) {
          v.x = fma(b, pp[q].x, v.x); v.y = fma(b, pp[q].y, v.y); v.z = fma(b, pp[q].z, v.z); v.w = fma(b, pp[q].w, v.w);
        }
        stg4_nb(Out + (int64_t)j * ldv + l0, v);
      }
    }
  }
}

int pack_rows_impl(const double* X, int64_t ldv, int64_t n_loc, int nx, int ncols, double* send_lo,
                   double* send_hi, cudaStream_t s) {
  if (ncols <= 0) return SCSF_OK;
  k_pack_rows<<<dim3(ceil_div(nx, 128), ncols), 128, 0, s>>>(X, ldv, n_loc, nx, ncols, send_lo, send_hi);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// part: 0 = every point of the slab (and the ld padding); 1 = the interior rows, which need no
// ghost row (and the padding); 2 = the first and last row, which read the ghosts.  Parts 1 and 2
// together equal part 0, so the halo exchange can run while part 1 computes.
int stencil_slab_impl(const scsf_ops* ops, int op, int64_t goff, int64_t n_loc, const double* X, const double* Xp,
                      double* Out, int64_t ldv, int ncols, const double* ghost_lo, const double* ghost_hi,
                      const double* fp, int step, cudaStream_t s, int part, const int* deg) {
  if (step < 0) deg = nullptr;                         // A X passes use every column
  if (ncols <= 0) return SCSF_OK;
  const int64_t n_glob = (int64_t)ops->nx * ops->ny;
  const int nx = ops->nx;
  const double* cf = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
  constexpr int CB = 4;                // 4 columns per CTA share the coefficient registers
  auto launch = [&](int64_t lb, int64_t le) -> int {
    if (le <= lb) return SCSF_OK;
    dim3 g(ceil_div(ceil_div(le - lb, 4), SV_THREADS), ceil_div(ncols, CB));
    k_stencil_slab<CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, nx, n_glob, goff, n_loc, X, Xp, Out, ldv, ncols,
                                                ghost_lo, ghost_hi, fp, step, lb, le, deg);
    SCSF_LAUNCH_CHECK();
    return SCSF_OK;
  };
  const int64_t rows = n_loc / nx;
  if (part == 0 || rows < 3) {
    if (part == 2) return SCSF_OK;       // (rows < 3: part 1 already did everything)
    return launch(0, ldv);
  }
  if (part == 1) {
    SCSF_TRY(launch(nx, n_loc - nx));
    return launch(n_loc, ldv);                          // padding
  }
  SCSF_TRY(launch(0, nx));
  return launch(n_loc - nx, n_loc);
}

// ---------------------------------------------------------- residuals ----
// For active column j: res[j] = ||W_j - theta_j V_j||_2^2, wn[j] = ||W_j||_2^2 (fixed-order sums;
// squared so a row-partitioned solve can all-reduce them; k_lock takes the roots).
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
    res[j] = a;                                       // squared: summed over ranks (row partition) before sqrt
    wn[j] = bb;
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

int assemble_vib_impl(const scsf_ops* ops, double h, const double* D, const double* rho, int64_t fstride,
                      double* coef, cudaStream_t s) {
  dim3 g(ceil_div(ops->ld, 256), ops->n_ops);
  k_assemble_vib<<<g, 256, 0, s>>>(ops->nx, ops->ny, ops->ld, 1.0 / (h * h * h * h), D, rho, fstride, coef);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int gershgorin_impl(const scsf_ops* ops, int op, unsigned long long* out, cudaStream_t s) {
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  const double* cf = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
  SCSF_CUDA_CHECK(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
  int blocks = min(ceil_div(n, 256), 148 * 4);
  if (ops->stencil == SCSF_STENCIL_VIB13)
    k_gershgorin_vib<<<blocks, 256, 0, s>>>(cf, ops->nx, n, ops->ld, out);
  else
    k_gershgorin<<<blocks, 256, 0, s>>>(cf, ops->dim, ops->nx, ops->ny, n, ops->ld, out);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

static int g_res_attr = 0;
// The smallest cluster whose slabs fit, doubled once while slabs keep >= 8 rows: smaller CTAs
// (C2: 14-row slabs, 350 threads, 102 KB) pack better next to the other chains' kernels
// (tools/bench_configs.py C2, three interleaved runs each: 1441 / 1298 / 1454 with 4-CTA
// clusters, 1457 / 1452 / 1456 operators/s with 8-CTA clusters).
int stencil_init_attrs();
template <int CS, int CB, bool TM>
__global__ void k_filter_cl(const double* __restrict__ cf, int64_t ldc, int nx, int ny, const double* __restrict__ X,
                            int64_t ldv, int ncols, double* __restrict__ Out, const double* __restrict__ fp, int m,
                            const int* __restrict__ deg, int split);
// Can this device co-schedule a 16-CTA cluster of the largest filter CTA (CL_T threads, 200 KB)?
// Probed once inside stencil_init_attrs() (std::call_once, before any chain thread launches);
// a device that cannot (fewer SMs per GPC, partitioned GPUs) keeps clusters <= 8.
static std::atomic<int> g_cs16{-1};
static int probe_cs16() {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16, 1, 1);
  cfg.blockDim = dim3(CL_T, 1, 1);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  const bool ok = cudaOccupancyMaxActiveClusters(&nclusters, k_filter_cl<16, 4>, &cfg) == cudaSuccess && nclusters > 0;
  cudaGetLastError();
  return ok ? 1 : 0;
}
static bool cs16_ok() {
  if (g_cs16.load(std::memory_order_acquire) < 0 && stencil_init_attrs() != SCSF_OK) return false;
  return g_cs16.load(std::memory_order_acquire) == 1;
}

// SCSF_FILTER_CS_DOUBLE (read per call): 1 (default) doubles a cluster below 8 CTAs whose doubled slab
// still has >= 8 rows (shorter filters); 0 keeps the smallest cluster that fits.  Co-resident clusters of
// the filter's CTA shape on a B200 (tools/cluster_slots.cu): 33 of 4 CTAs (132 SMs), 15 of 8 (120 SMs).
static bool filter_cs_double() {
  const char* e = getenv("SCSF_FILTER_CS_DOUBLE");
  return !(e && e[0] == '0');
}
static int cluster_size_for(const scsf_ops* ops) {
  if (ops->stencil != SCSF_STENCIL_FLUX || ops->dim != 2 || ops->nx % 2 != 0) return 0;
  // up to 16 CTAs (a non-portable cluster size, opted in per kernel): C3's 200 x 200 slabs fit at
  // 16 (7 x 100 patches, 4 columns per CTA) and the whole filter stays on chip: 1.05 of the HBM
  // roofline's algorithmic rate against 0.74 for the streaming kernel; C3 8.7 -> 9.9 ops/s
  const int cs_max = cs16_ok() ? 16 : 8;
  for (int cs = 1; cs <= cs_max; cs *= 2) {
    const int R = ((ops->ny + cs - 1) / cs + 1) & ~1;
    if ((R / 2) * (ops->nx / 2) <= CL_MAXP && (size_t)2 * (R + 2) * ops->nx * sizeof(double) <= 200 * 1024) {
      const int R2 = ((ops->ny + 2 * cs - 1) / (2 * cs) + 1) & ~1;
      return (cs < 8 && R2 >= 8 && filter_cs_double()) ? 2 * cs : cs;   // (the doubling stops at the portable 8)
    }
  }
  return 0;
}

// k_filter_rp: 2 x 4 register patches; SCSF_FILTER_RP=0 falls back to k_filter_cl
static bool rp_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_FILTER_RP");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}
static int rp_rows(int ny, int cs) { return ((ny + cs - 1) / cs + RP_ROWS - 1) / RP_ROWS * RP_ROWS; }
constexpr int RP_CB = 2;
static int cluster_size_rp(const scsf_ops* ops) {
  if (!rp_enabled() || ops->stencil != SCSF_STENCIL_FLUX || ops->dim != 2 || ops->nx % 2 != 0) return 0;
  // Measured (tools/bench_configs.py): ahead of k_filter_cl when one CTA holds a whole column
  // (C1, 32 x 32: 1150-1200 against 1010-1060 operators/s); on C2 (4-CTA clusters) k_filter_cl
  // with 4 columns per CTA is as fast or faster (1400 against 1350), so only cs == 1 is used.
  const int R = rp_rows(ops->ny, 1);
  if ((R / RP_ROWS) * (ops->nx / 2) <= RP_T && (size_t)RP_CB * 2 * (R + 2) * ops->nx * sizeof(double) <= 200 * 1024)
    return 1;
  return 0;
}

// 3: register-patch cluster filter (k_filter_rp), 2: cluster-resident (k_filter_cl),
// 1: single-CTA resident (k_filter_res2d*), 0: per-step streaming
int filter_kind(const scsf_ops* ops) {
  if (ops->stencil != SCSF_STENCIL_FLUX) return 0;
  if (cluster_size_rp(ops) > 0) return 3;
  if (cluster_size_for(ops) > 0) return 2;
  if (ops->dim == 2 && (int64_t)ops->nx * ops->ny <= RES_MAX_N) return 1;
  return 0;
}

bool filter_resident_ok(const scsf_ops* ops) {
  return filter_kind(ops) > 0;
}

// The TMEM-backed variant of k_filter_cl is the default.  Measured (tools/bench_filter.py,
// tools/graph_ab.py, 32 chains, profiles/r02_tmem_ab.json): C3 step 32.8 -> 29.9 us, C3 64 operators
// 1.714 -> 1.585 s; C2 0.665-0.704 -> 0.652 s (with the allocation sized to the CTA, so two C2
// CTAs share an SM's 512 columns; a fixed 512-column allocation made C2 7 % slower).
// SCSF_FILTER_TMEM = 0 restores the shared-memory form (read per call).
static bool filter_tmem(unsigned threads) {
  (void)threads;
  const char* e = getenv("SCSF_FILTER_TMEM");
  return !(e && e[0] == '0');
}
// Step synchronisation of k_filter_cl (SCSF_FILTER_SPLIT, read per call): 2 (default) = mbarrier
// neighbour sync with st.async ghost pushes, 1 = split cluster arrive / wait, 0 = one cluster barrier per
// step.  Measured (tools/bench_filter.py, m = 160, profiles/r02_filter_split_ab.json): C3 filter
// 3.611 (0) -> 3.489 (1) ms, and in another run 3.634 (1) -> 3.332 (2) ms; C2 0.444 -> 0.424 ms;
// C3 bench 45.6 (1) -> 48.2 (2) operators/s.
static int filter_split() {
  const char* e = getenv("SCSF_FILTER_SPLIT");
  return (e && e[0] == '0') ? 0 : (e && e[0] == '1') ? 1 : 2;
}
// SCSF_FILTER_TRIM (read per call): 1 (default) launches a cluster of only the CTAs whose slab holds
// rows, 0 the template's full cluster size (the surplus CTAs idle through the filter).
static bool filter_trim() {
  const char* e = getenv("SCSF_FILTER_TRIM");
  return !(e && e[0] == '0');
}
template <int CS, int CB>
static cudaError_t launch_cl1(cudaLaunchConfig_t& cfg, const double* cf, int64_t ldc, int nx, int ny, const double* X,
                              int64_t ldv, int ncols, double* Out, const double* fp, int m, const int* deg) {
  const int split = filter_split();
  if (filter_tmem(cfg.blockDim.x))
    return cudaLaunchKernelEx(&cfg, k_filter_cl<CS, CB, true>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, split);
  return cudaLaunchKernelEx(&cfg, k_filter_cl<CS, CB, false>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, split);
}
template <int CS>
static cudaError_t launch_cl_cb(cudaLaunchConfig_t& cfg, int cb, const double* cf, int64_t ldc, int nx, int ny,
                                const double* X, int64_t ldv, int ncols, double* Out, const double* fp, int m,
                                const int* deg) {
  if (cb == 4) return launch_cl1<CS, 4>(cfg, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
  if (cb == 2) return launch_cl1<CS, 2>(cfg, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
  return launch_cl1<CS, 1>(cfg, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
}
static cudaError_t launch_rp(cudaLaunchConfig_t& cfg, int cs, const double* cf, int64_t ldc, int nx, int ny,
                             const double* X, int64_t ldv, int ncols, double* Out, const double* fp, int m,
                             const int* deg) {
  switch (cs) {
    case 1: return cudaLaunchKernelEx(&cfg, k_filter_rp<1, RP_CB>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, 0);
    case 2: return cudaLaunchKernelEx(&cfg, k_filter_rp<2, RP_CB>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, 0);
    case 4: return cudaLaunchKernelEx(&cfg, k_filter_rp<4, RP_CB>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, 0);
    default: return cudaLaunchKernelEx(&cfg, k_filter_rp<8, RP_CB>, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg, 0);
  }
}
static cudaError_t launch_cl(cudaLaunchConfig_t& cfg, int cs, int cb, const double* cf, int64_t ldc, int nx, int ny,
                             const double* X, int64_t ldv, int ncols, double* Out, const double* fp, int m,
                             const int* deg) {
  switch (cs) {
    case 1: return launch_cl_cb<1>(cfg, cb, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
    case 2: return launch_cl_cb<2>(cfg, cb, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
    case 4: return launch_cl_cb<4>(cfg, cb, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
    case 16: return launch_cl_cb<16>(cfg, cb, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
    default: return launch_cl_cb<8>(cfg, cb, cf, ldc, nx, ny, X, ldv, ncols, Out, fp, m, deg);
  }
}

// All dynamic-shared-memory opt-ins of the filter kernels, set once before any
// launch (in particular before a CUDA-graph capture).
static int stencil_init_attrs_once() {
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_res2d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       2 * RES_MAX_N * (int)sizeof(double)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_stencil_vib_t, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#define SCSF_CL_ATTR(CS, CB) \
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<CS, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
  SCSF_CL_ATTR(1, 1); SCSF_CL_ATTR(1, 2); SCSF_CL_ATTR(1, 4);
  SCSF_CL_ATTR(2, 1); SCSF_CL_ATTR(2, 2); SCSF_CL_ATTR(2, 4);
  SCSF_CL_ATTR(4, 1); SCSF_CL_ATTR(4, 2); SCSF_CL_ATTR(4, 4);
  SCSF_CL_ATTR(8, 1); SCSF_CL_ATTR(8, 2); SCSF_CL_ATTR(8, 4);
  SCSF_CL_ATTR(16, 1); SCSF_CL_ATTR(16, 2); SCSF_CL_ATTR(16, 4);
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));

#define SCSF_CLT_ATTR(CS, CB) \
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<CS, CB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
  SCSF_CLT_ATTR(1, 1); SCSF_CLT_ATTR(1, 2); SCSF_CLT_ATTR(1, 4);
  SCSF_CLT_ATTR(2, 1); SCSF_CLT_ATTR(2, 2); SCSF_CLT_ATTR(2, 4);
  SCSF_CLT_ATTR(4, 1); SCSF_CLT_ATTR(4, 2); SCSF_CLT_ATTR(4, 4);
  SCSF_CLT_ATTR(8, 1); SCSF_CLT_ATTR(8, 2); SCSF_CLT_ATTR(8, 4);
  SCSF_CLT_ATTR(16, 1); SCSF_CLT_ATTR(16, 2); SCSF_CLT_ATTR(16, 4);
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 1, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 2, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_cl<16, 4, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
#undef SCSF_CLT_ATTR
#undef SCSF_CL_ATTR
#define SCSF_RP_ATTR(CS) \
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_filter_rp<CS, RP_CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
  SCSF_RP_ATTR(1); SCSF_RP_ATTR(2); SCSF_RP_ATTR(4); SCSF_RP_ATTR(8);
#undef SCSF_RP_ATTR
  g_res_attr = 1;
  g_cs16.store(probe_cs16(), std::memory_order_release);     // published once, after the opt-ins
  return SCSF_OK;
}
int stencil_init_attrs() {
  static std::once_flag once;
  static int status = SCSF_OK;
  std::call_once(once, [] { status = stencil_init_attrs_once(); });
  return status;
}


// Whole filter (steps 0..m-1) for ncols columns of X into Out, column-resident kernel.
int filter_resident_impl(const scsf_ops* ops, int op, const double* X, double* Out, int64_t ldv, int ncols,
                         const double* fp, int m, cudaStream_t s, const int* deg) {
  if (ncols <= 0) return SCSF_OK;
  const int n = ops->nx * ops->ny;
  const double* cf = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
  SCSF_TRY(stencil_init_attrs());
  const bool pair = (ops->nx % 2 == 0) && (ldv % 2 == 0) && (ops->ld % 2 == 0) && ((uintptr_t)X % 16 == 0) &&
                    ((uintptr_t)Out % 16 == 0) && ((uintptr_t)cf % 16 == 0);
  const int csr = pair ? cluster_size_rp(ops) : 0;
  const int cs = pair ? cluster_size_for(ops) : 0;
  if (csr > 0) {
    const int R = rp_rows(ops->ny, csr);
    const size_t per_col = (size_t)2 * (R + 2) * ops->nx * sizeof(double);
    const int thr = (int)round_up((int64_t)(R / RP_ROWS) * (ops->nx / 2), 32);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csr, ceil_div(ncols, RP_CB), 1);
    cfg.blockDim = dim3(thr, 1, 1);
    cfg.dynamicSmemBytes = per_col * RP_CB;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csr;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SCSF_CUDA_CHECK(launch_rp(cfg, csr, cf, ops->ld, ops->nx, ops->ny, X, ldv, ncols, Out, fp, m, deg));
  } else if (cs > 0) {
    const int R = ((ops->ny + cs - 1) / cs + 1) & ~1;
    const size_t per_col = (size_t)2 * (R + 2) * ops->nx * sizeof(double);
    const int cb = (4 * per_col <= 200 * 1024) ? 4 : (2 * per_col <= 200 * 1024 ? 2 : 1);
    const int thr = (int)round_up((int64_t)(R / 2) * (ops->nx / 2), 32);
    // launch only the CTAs whose slab holds rows: C3 (ny = 200, R = 14) needs 15 of the 16 the
    // template's slab height is sized for, and an empty CTA would hold an SM for the whole filter
    const int ccl = filter_trim() ? (int)ceil_div(ops->ny, R) : cs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ccl, ceil_div(ncols, cb), 1);
    cfg.blockDim = dim3(thr, 1, 1);
    cfg.dynamicSmemBytes = per_col * cb;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SCSF_CUDA_CHECK(launch_cl(cfg, cs, cb, cf, ops->ld, ops->nx, ops->ny, X, ldv, ncols, Out, fp, m, deg));
  } else
    k_filter_res2d<<<ncols, RES_T, (size_t)2 * n * sizeof(double), s>>>(cf, ops->ld, ops->nx, n, X, ldv, Out, fp, m);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// Out[:, 0:ncols] = step-th filter update (or A X when step < 0).
// Does stencil_impl dispatch the vectorised k_stencil_v4 (the one streaming kernel that honours
// per-column degrees) for these operators and blocks?
bool stencil_v4_ok(const scsf_ops* ops, int64_t ldv) {
  return ops->stencil == SCSF_STENCIL_FLUX && ops->nx % 4 == 0 && ldv % 4 == 0 && ops->ld % 4 == 0;
}

int stencil_impl(const scsf_ops* ops, int op, const double* X, const double* Xp, double* Out,
                 int64_t ldv, int ncols, const double* fp, int step, cudaStream_t s, const int* deg) {
  if (ncols <= 0) return SCSF_OK;
  int64_t n = (int64_t)ops->nx * ops->ny * ops->nz;
  const double* cf = ops->coef + (int64_t)op * ncoef(ops) * ops->ld;
  if (ops->stencil == SCSF_STENCIL_VIB13) {
    if (vib_t_smem(ops->nx) <= 200 * 1024) {
      SCSF_TRY(stencil_init_attrs());
      dim3 g(ceil_div(ops->ny, VT_R), ceil_div(ncols, VT_CB));
      k_stencil_vib_t<<<g, VT_T, vib_t_smem(ops->nx), s>>>(cf, ops->ld, ops->nx, ops->ny, X, Xp, Out, ldv, ncols,
                                                            fp, step);
    } else {
      dim3 g(ceil_div(ldv, VB_THREADS), ceil_div(ncols, VB_COLS));
      k_stencil_vib<<<g, VB_THREADS, 0, s>>>(cf, ops->ld, ops->nx, n, X, Xp, Out, ldv, ncols, fp, step);
    }
    SCSF_LAUNCH_CHECK();
    return SCSF_OK;
  }
  const bool vec = (ops->nx % 4 == 0) && (ldv % 4 == 0) && (ops->ld % 4 == 0) &&
                   ((uintptr_t)X % 32 == 0) && ((uintptr_t)Out % 32 == 0) && ((uintptr_t)cf % 32 == 0) &&
                   (Xp == nullptr || (uintptr_t)Xp % 32 == 0);
  if (vec) {
    // 4 columns per CTA share each point's coefficient registers (tools/bench_filter.py, fraction of
    // the HBM peak with CB = 2 / 4: C3 0.74 / 0.75, C4 (3-D) 0.60 / 0.68, C5 0.85 / 0.88)
    constexpr int CB = 4;
    dim3 g(ceil_div(ceil_div(ldv, 4), SV_THREADS), ceil_div(ncols, CB));
    const int grp = v4_group(ops->dim);
#define SCSF_V4G(D, G)                                                                                          \
  k_stencil_v4g<D, CB, G><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, \
                                                   step, deg)
    if (grp == 1) {
      if (ops->dim == 2) SCSF_V4G(2, 1); else SCSF_V4G(3, 1);
    } else if (grp == 2) {
      if (ops->dim == 2) SCSF_V4G(2, 2); else SCSF_V4G(3, 2);
    } else if (grp == 4) {
      if (ops->dim == 2) SCSF_V4G(2, 4); else SCSF_V4G(3, 4);
    } else if (ops->dim == 2)
      k_stencil_v4<2, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step,
                                                   deg);
    else
      k_stencil_v4<3, CB><<<g, SV_THREADS, 0, s>>>(cf, ops->ld, ops->nx, ops->ny, n, X, Xp, Out, ldv, ncols, fp, step,
                                                   deg);
#undef SCSF_V4G
  } else {
    if (deg) {
      set_error("per-column filter degrees need the vectorised stencil (nx %% 4 == 0, aligned blocks)");
      return SCSF_ERR_ARG;
    }
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

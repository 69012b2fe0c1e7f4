// k_small.cu — the b x b pieces of Alg. 3 and the
// per-iteration control logic, all on the device.
//
//  chol_inv     S = R^T R (upper Cholesky) and R^{-1}, one CTA: CholQR's small
//               factor (l. 4; reading R13).  If S is not numerically SPD
//               the kernel retries on S + shift*I (shifted CholQR, Fukaya et al.
//               2020) and flags ctrl->chol_fail so the driver adds a pass.
//  jacobi_eig   G = Z diag(theta) Z^T (l. 6; method unstated by the paper,
//               R10-adjacent reading: two-sided cyclic Jacobi in parallel
//               round-robin order, threshold skip of already-small pairs, so a
//               warm, nearly diagonal G costs almost nothing), eigenvalues sorted
//               ascending with the eigenvector columns.
//  lock         contiguous-from-the-bottom locking on ||Av - lv|| <= tol ||Av||
//               (l. 7, metric P:844; R15, R16) and the next filter's
//               (lambda, c, e) from the Ritz values (R9).
//  rand_block   seeded Gaussian start for a chain head (R17).
//  finalize     ascending sort of the b Ritz pairs + sign convention (R21).
#include "common.cuh"

namespace scsf {

// ------------------------------------------------------------- chol_inv ----
// Working array A (b x b, col-major, ld b): upper triangle -> R, strict lower
// triangle -> R^{-1} transposed (X[k][c] stored at A[c + k b], k < c),
// dinv[i] = 1/R[i][i].
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_chol_inv(const double* __restrict__ S, int64_t lds, int b,
                                                   int64_t nrows, double* __restrict__ Rinv,
                                                   double* __restrict__ gA, Ctrl* ctrl) {
  extern __shared__ double sm[];
  double* A = SMEM ? sm : gA;
  __shared__ double dinv[384];
  __shared__ int fail;
  __shared__ double shift;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (tid == 0) {
      fail = 0;
      if (attempt == 1) {
        double tr = 0.0;
        for (int i = 0; i < b; ++i) tr += fabs(S[i + i * lds]);
        shift = 11.0 * ((double)nrows * b + (double)b * (b + 1)) * 1.1102230246251565e-16 * tr;
      } else {
        shift = 0.0;
      }
    }
    __syncthreads();
    for (int idx = tid; idx < b * b; idx += nt) {
      int i = idx % b, j = idx / b;
      double v = S[i + (int64_t)j * lds];
      if (i == j) v += shift;
      A[idx] = v;
    }
    __syncthreads();
    // right-looking upper Cholesky; breakdown when a pivot loses all but ~1e-14 of its diagonal
    for (int j = 0; j < b; ++j) {
      double d = A[j + j * b];
      if (!(d > 1e-14 * fabs(S[j + (int64_t)j * lds])) || !isfinite(d)) {
        if (tid == 0) fail = 1;
      }
      __syncthreads();
      if (fail) break;
      double r = sqrt(d);
      for (int k = j + 1 + tid; k < b; k += nt) A[j + k * b] /= r;
      if (tid == 0) A[j + j * b] = r;
      __syncthreads();
      // trailing update of the upper triangle: A[i][k] -= R[j][i] R[j][k], j < i <= k
      const int m = b - j - 1;
      for (int t = tid; t < m * m; t += nt) {
        int ii = t % m, kk = t / m;
        if (ii > kk) continue;
        int i = j + 1 + ii, k = j + 1 + kk;
        A[i + k * b] -= A[j + i * b] * A[j + k * b];
      }
      __syncthreads();
    }
    if (!fail) break;
    if (tid == 0 && ctrl) {
      ctrl->chol_fail = 1;
      ctrl->chol_fallbacks += 1;
    }
    __syncthreads();
  }
  // R^{-1}: rows from the bottom; X[i][c] = -(sum_{k=i+1..c} R[i][k] X[k][c]) / R[i][i]
  for (int i = b - 1; i >= 0; --i) {
    double rii = A[i + i * b];
    if (tid == 0) dinv[i] = 1.0 / rii;
    for (int c = i + 1 + tid; c < b; c += nt) {
      double s = 0.0;
      for (int k = i + 1; k <= c; ++k) {
        double xkc = (k == c) ? (1.0 / A[c + c * b]) : A[c + k * b];   // X[k][c]
        s = fma(A[i + k * b], xkc, s);
      }
      A[c + i * b] = -s / rii;   // X[i][c] stored transposed in the lower triangle
    }
    __syncthreads();
  }
  for (int idx = tid; idx < b * b; idx += nt) {
    int i = idx % b, c = idx / b;
    double v = 0.0;
    if (i == c) v = dinv[i];
    else if (i < c) v = A[c + i * b];
    Rinv[idx] = v;
  }
}

// ----------------------------------------------------------- jacobi_eig ----
// Parallel-order (round-robin) two-sided Jacobi.  G (b x b, ld b) is copied to
// the work array; Z accumulates the rotations (global scratch, ld b).
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_jacobi(const double* __restrict__ Gin, int64_t ldg, int b,
                                                 double* __restrict__ gG, double* __restrict__ Z,
                                                 double* __restrict__ theta_out, double* __restrict__ Zout,
                                                 int max_sweeps, Ctrl* ctrl) {
  extern __shared__ double sm[];
  double* G = SMEM ? sm : gG;
  __shared__ double cs_c[192], cs_s[192], cs_t[192];
  __shared__ int cs_p[192], cs_q[192], cs_rot[192];
  __shared__ int any_rot;
  __shared__ double diag_s[384];
  __shared__ int rank_s[384];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int bp = (b + 1) & ~1;      // even; index b is a dummy when b is odd
  const int half = bp / 2;
  for (int idx = tid; idx < b * b; idx += nt) {
    int i = idx % b, j = idx / b;
    G[idx] = Gin[i + (int64_t)j * ldg];
    Z[idx] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) any_rot = 0;
    __syncthreads();
    for (int r = 0; r < bp - 1; ++r) {
      if (tid < half) {
        int m = tid;
        int a = (m == 0) ? 0 : ((m - 1 + r) % (bp - 1)) + 1;
        int mm = bp - 1 - m;
        int q = ((mm - 1 + r) % (bp - 1)) + 1;
        int p = a;
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double c = 1.0, s = 0.0, t = 0.0;
        int rot = 0;
        if (q < b) {
          double gpq = G[p + q * b];
          double gpp = G[p + p * b], gqq = G[q + q * b];
          if (fabs(gpq) > 1e-14 * sqrt(fabs(gpp * gqq)) && fabs(gpq) > 1e-300) {
            double th = (gqq - gpp) / (2.0 * gpq);
            double tt;
            if (fabs(th) > 1e150) tt = 0.5 / th;
            else tt = copysign(1.0, th) / (fabs(th) + sqrt(1.0 + th * th));
            t = tt;
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = tt * c;
            rot = 1;
          }
        }
        cs_p[m] = p; cs_q[m] = q; cs_c[m] = c; cs_s[m] = s; cs_t[m] = t; cs_rot[m] = rot;
        if (rot) any_rot = 1;
      }
      __syncthreads();
      // G <- J^T G J on all 2x2 blocks touched by a rotation
      const int nblk = half * half;
      for (int idx = tid; idx < nblk; idx += nt) {
        int m1 = idx / half, m2 = idx % half;
        if (!cs_rot[m1] && !cs_rot[m2]) continue;
        int p1 = cs_p[m1], q1 = cs_q[m1], p2 = cs_p[m2], q2 = cs_q[m2];
        if (m1 == m2) {
          if (q1 < b) {
            double gpq = G[p1 + q1 * b], t = cs_t[m1];
            G[p1 + p1 * b] -= t * gpq;
            G[q1 + q1 * b] += t * gpq;
            G[p1 + q1 * b] = 0.0;
            G[q1 + p1 * b] = 0.0;
          }
          continue;
        }
        double c1 = cs_c[m1], s1 = cs_s[m1], c2 = cs_c[m2], s2 = cs_s[m2];
        bool hq1 = q1 < b, hq2 = q2 < b;
        double a = G[p1 + p2 * b];
        double bb = hq2 ? G[p1 + q2 * b] : 0.0;
        double cc = hq1 ? G[q1 + p2 * b] : 0.0;
        double d = (hq1 && hq2) ? G[q1 + q2 * b] : 0.0;
        double a2 = c2 * a - s2 * bb, b2 = s2 * a + c2 * bb;      // right: columns p2, q2
        double c2v = c2 * cc - s2 * d, d2 = s2 * cc + c2 * d;
        G[p1 + p2 * b] = c1 * a2 - s1 * c2v;                        // left: rows p1, q1
        if (hq2) G[p1 + q2 * b] = c1 * b2 - s1 * d2;
        if (hq1) G[q1 + p2 * b] = s1 * a2 + c1 * c2v;
        if (hq1 && hq2) G[q1 + q2 * b] = s1 * b2 + c1 * d2;
      }
      // Z <- Z J
      const int nz = b * half;
      for (int idx = tid; idx < nz; idx += nt) {
        int m = idx / b, x = idx % b;
        if (!cs_rot[m]) continue;
        int p = cs_p[m], q = cs_q[m];
        double c = cs_c[m], s = cs_s[m];
        double zp = Z[x + p * b], zq = Z[x + q * b];
        Z[x + p * b] = c * zp - s * zq;
        Z[x + q * b] = s * zp + c * zq;
      }
      __syncthreads();
    }
    if (!any_rot) break;
    __syncthreads();
  }
  if (tid == 0 && ctrl && sweep >= max_sweeps) ctrl->nonfinite |= 2;
  // ascending order (ties by index)
  for (int i = tid; i < b; i += nt) diag_s[i] = G[i + i * b];
  __syncthreads();
  for (int i = tid; i < b; i += nt) {
    double v = diag_s[i];
    int rk = 0;
    for (int j = 0; j < b; ++j) {
      double w = diag_s[j];
      rk += (w < v) || (w == v && j < i);
    }
    rank_s[i] = rk;
    theta_out[rk] = v;
  }
  __syncthreads();
  for (int idx = tid; idx < b * b; idx += nt) {
    int x = idx % b, i = idx / b;
    Zout[x + (int64_t)rank_s[i] * b] = Z[idx];
  }
}

// ----------------------------------------------------------------- lock ----
// theta/res/wn/rel are indexed by block column (0..b-1); active columns [kL, b).
__global__ void k_lock(const double* __restrict__ theta, const double* __restrict__ res,
                       const double* __restrict__ wn, double* __restrict__ rel, int b, int L,
                       double tol, Ctrl* ctrl, double* fp) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int kL = ctrl->kL;
  ctrl->kL_prev = kL;
  for (int j = kL; j < b; ++j) {
    double r = res[j] / wn[j];
    rel[j] = r;
    if (!isfinite(r)) ctrl->nonfinite |= 1;
  }
  int j = kL;
  while (j < b && rel[j] <= tol) ++j;     // contiguous run from the bottom (R15)
  ctrl->kL = j;
  double mx = 0.0;
  for (int i = 0; i < min(L, b); ++i) mx = fmax(mx, rel[i]);
  ctrl->max_rel = mx;
  if (j < b) {
    double lam = theta[j];                // scale point: smallest non-locked Ritz value (R9)
    double alpha = theta[b - 1];          // damped interval [alpha, beta] (R9, R10)
    double beta = ctrl->beta;
    double c = 0.5 * (alpha + beta), e = 0.5 * (beta - alpha);
    if (!(e > 0.0)) e = fmax(fabs(beta), 1.0) * 1e-12;
    ctrl->lambda = lam;
    ctrl->alpha = alpha;
    fp[0] = lam;
    fp[1] = c;
    fp[2] = e;
  }
}

__global__ void k_ctrl_init(Ctrl* ctrl, const unsigned long long* gersh) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  ctrl->beta = __longlong_as_double((long long)*gersh);
  ctrl->kL = 0;
  ctrl->kL_prev = 0;
  ctrl->chol_fail = 0;
  ctrl->chol_fallbacks = 0;
  ctrl->nonfinite = 0;
  ctrl->max_rel = 0.0;
}

// ----------------------------------------------------------- rand_block ----
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_rand_block(double* __restrict__ V, int64_t ldv, int64_t n, int ncols, uint64_t seed) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int j = blockIdx.y;
  if (k >= ldv || j >= ncols) return;
  double v = 0.0;
  if (k < n) {
    uint64_t h = splitmix64(splitmix64(splitmix64(seed) ^ (uint64_t)j) ^ (uint64_t)k);
    uint64_t h2 = splitmix64(h);
    double u1 = ((double)(h >> 11) + 1.0) * 0x1.0p-53;   // (0, 1]
    double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    v = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
  V[k + (int64_t)j * ldv] = v;
}

// ------------------------------------------------------------- finalize ----
// perm[j] = block column holding the j-th smallest Ritz value; theta_sorted ascending.
__global__ void k_sort_theta(const double* __restrict__ theta, const double* __restrict__ rel, int b, int L,
                             int* __restrict__ perm, double* __restrict__ theta_sorted, Ctrl* ctrl) {
  for (int i = threadIdx.x; i < b; i += blockDim.x) {
    double v = theta[i];
    int rk = 0;
    for (int j = 0; j < b; ++j) {
      double w = theta[j];
      rk += (w < v) || (w == v && j < i);
    }
    perm[rk] = i;
    theta_sorted[rk] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < min(L, b); ++j) mx = fmax(mx, rel[perm[j]]);
    ctrl->max_rel = mx;
  }
}

// Out[:, j] = s_j V[:, perm[j]], s_j = sign of the largest-|.| entry (first on ties).
__global__ void __launch_bounds__(256) k_gather_sign(const double* __restrict__ V, int64_t ldv, int64_t n,
                                                     const int* __restrict__ perm, double* __restrict__ Out,
                                                     int64_t ldo) {
  int j = blockIdx.x;
  const double* v = V + (int64_t)perm[j] * ldv;
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    double a = fabs(v[k]);
    if (a > best) { best = a; bi = k; }
  }
  __shared__ double sb[256];
  __shared__ int64_t si[256];
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      double b2 = sb[threadIdx.x + o];
      int64_t i2 = si[threadIdx.x + o];
      if (b2 > sb[threadIdx.x] || (b2 == sb[threadIdx.x] && i2 < si[threadIdx.x])) {
        sb[threadIdx.x] = b2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  double sgn = (v[si[0]] < 0.0) ? -1.0 : 1.0;
  double* o = Out + (int64_t)j * ldo;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) o[k] = sgn * v[k];
}

// ------------------------------------------------------------------ host ----
static int g_small_attr = 0;

static int set_small_attrs() {
  if (g_small_attr) return SCSF_OK;
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_chol_inv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_jacobi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  g_small_attr = 1;
  return SCSF_OK;
}

constexpr int SMALL_SMEM_MAX_B = 156;   // b*b*8 <= ~195 KB

int chol_inv_impl(const double* S, int64_t lds, int b, int64_t nrows, double* Rinv, double* scratch,
                  Ctrl* ctrl, cudaStream_t s) {
  if (b > 384) {
    set_error("chol_inv: b=%d > 384", b);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  SCSF_TRY(set_small_attrs());
  if (b <= SMALL_SMEM_MAX_B)
    k_chol_inv<true><<<1, 1024, (size_t)b * b * sizeof(double), s>>>(S, lds, b, nrows, Rinv, scratch, ctrl);
  else
    k_chol_inv<false><<<1, 1024, 0, s>>>(S, lds, b, nrows, Rinv, scratch, ctrl);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int jacobi_impl(const double* G, int64_t ldg, int b, double* scratchG, double* Z, double* theta,
                double* Zout, Ctrl* ctrl, cudaStream_t s) {
  if (b > 384) {
    set_error("jacobi: b=%d > 384", b);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  SCSF_TRY(set_small_attrs());
  if (b <= SMALL_SMEM_MAX_B)
    k_jacobi<true><<<1, 1024, (size_t)b * b * sizeof(double), s>>>(G, ldg, b, scratchG, Z, theta, Zout, 60, ctrl);
  else
    k_jacobi<false><<<1, 1024, 0, s>>>(G, ldg, b, scratchG, Z, theta, Zout, 60, ctrl);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int lock_impl(const double* theta, const double* res, const double* wn, double* rel, int b, int L,
              double tol, Ctrl* ctrl, double* fp, cudaStream_t s) {
  k_lock<<<1, 32, 0, s>>>(theta, res, wn, rel, b, L, tol, ctrl, fp);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int ctrl_init_impl(Ctrl* ctrl, const unsigned long long* gersh, cudaStream_t s) {
  k_ctrl_init<<<1, 32, 0, s>>>(ctrl, gersh);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int rand_block_impl(double* V, int64_t ldv, int64_t n, int ncols, uint64_t seed, cudaStream_t s) {
  dim3 g(ceil_div(ldv, 256), ncols);
  k_rand_block<<<g, 256, 0, s>>>(V, ldv, n, ncols, seed);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int finalize_impl(const double* theta, const double* rel, int b, int L, int* perm, double* theta_sorted,
                  const double* V, int64_t ldv, int64_t n, double* Out, int64_t ldo, Ctrl* ctrl,
                  cudaStream_t s) {
  k_sort_theta<<<1, 512, 0, s>>>(theta, rel, b, L, perm, theta_sorted, ctrl);
  SCSF_LAUNCH_CHECK();
  k_gather_sign<<<b, 256, 0, s>>>(V, ldv, n, perm, Out, ldo);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf

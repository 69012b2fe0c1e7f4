// k_grf.cu — coefficient fields of a batch on the device (Fig. 1 steps 1-2):
// the Gaussian-random-field series of DESIGN.md §3 (the paper only says "derived using GRF",
// P:759, 789, 807) evaluated at the grid nodes and face midpoints, exponentiated and scaled
// into the arrays scsf_assemble and scsf_sort consume.  The normal draws xi are an input
// (drawn on the host); everything after the draw runs here.
//
//   g(x) = sum_{k in {1..K}^d} xi_k w_k prod_d sin(pi k_d x_d),  w_k = (1 + |k|^2)^(-s),
//   g <- g * sigma / s_K  when sigma > 0,  s_K = sqrt(sum_k w_k^2 / 2^d),
//   node i at x = (i+1) h, face i (between nodes i-1 and i) at x = (i+1/2) h, h = 1/(nx+1).
//
// Separable evaluation: per output row (2-D) or plane (3-D) the coefficient tensor is
// contracted with the row's / plane's basis values first (K^d -> K per row), then every
// output point of the row is a length-K dot product with the x-basis (read from a table in
// global memory, [K][nx+1] per kind, L2-resident).  All of it is a few MFLOP per operator.
#include "common.cuh"

namespace scsf {

namespace {
constexpr int GRF_T = 256;      // threads per CTA
constexpr int GRF_TY = 8;       // 2-D: output rows per CTA
constexpr int GRF_KMAX = 32;    // modes per axis (K^2 <= 1024 doubles of coefficients in shared memory)

struct GrfArgs {
  int dim, nx, K, family, n_fields, n_ops;
  double s, sigma, vscale, h;
  const double* xi;               // [n_ops][n_fields][K^dim], C order [kx][ky](kz)
  const double* tab;              // [2][K][nx+1]: kind 0 node basis, kind 1 face basis
  double* faces[3];
  double* c;
  double* params;                 // [n_ops][n_fields][n]
};

// basis tables: tab[kind][k][i] = sin(pi * (x_i * (k+1))), x_i = (i+1) h (node) or (i+1/2) h (face)
__global__ void k_grf_basis(int nx, int K, double h, double* tab) {
  const int W = nx + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 2 * K * W; t += gridDim.x * blockDim.x) {
    const int kind = t / (K * W), r = t % (K * W), k = r / W, i = r % W;
    const double x = kind == 0 ? (double)(i + 1) * h : ((double)i + 0.5) * h;
    tab[t] = (kind == 0 && i == nx) ? 0.0 : sin(3.141592653589793 * (x * (double)(k + 1)));
  }
}

__device__ __forceinline__ double bval(const GrfArgs& a, int kind, int k, int i) {
  return __ldg(a.tab + ((int64_t)kind * a.K + k) * (a.nx + 1) + i);
}

// One CTA: operator op, field f, array arr (0 = nodes, 1 + ax = faces normal to axis ax),
// tile t (2-D: rows t*TY..; 3-D: plane z = t).
__global__ void __launch_bounds__(GRF_T) k_grf_eval(GrfArgs a) {
  __shared__ double coef[GRF_KMAX * GRF_KMAX];
  __shared__ double u2[GRF_KMAX * GRF_KMAX];       // 3-D: plane-contracted coefficients [a][b]
  __shared__ double u[64 * GRF_KMAX];              // per-row contraction [row][a] (2-D TY rows, 3-D ny+1 <= 64)
  __shared__ double red[GRF_T / 32];
  const int t = blockIdx.x, arr = blockIdx.y, of = blockIdx.z;
  const int op = of / a.n_fields, f = of % a.n_fields;
  const int dim = a.dim, nx = a.nx, K = a.K;
  const int ax = arr - 1;                          // face axis or -1
  const int Hx = nx + (ax == 0), Hy = nx + (ax == 1), Hz = dim == 3 ? nx + (ax == 2) : 1;
  const int kx = ax == 0, ky = ax == 1, kz = ax == 2;   // basis kinds per axis
  const int64_t n = dim == 3 ? (int64_t)nx * nx * nx : (int64_t)nx * nx;
  const int64_t plane_pts = (int64_t)Hx * Hy;
  const bool faces_wanted = arr > 0 && f == 0 && a.family != 1;   // lapv faces are the constant 1
  // which rows does this CTA own?
  int y0, y1, z;
  if (dim == 2) {
    y0 = t * GRF_TY;
    y1 = min(y0 + GRF_TY, Hy);
    z = 0;
  } else {
    y0 = 0;
    y1 = Hy;
    z = t;
  }
  if (arr > dim || (dim == 2 ? y0 >= Hy : z >= Hz)) return;
  if (arr > 0 && f != 0) return;                   // only field 0 has face coefficients
  const double scale = a.family >= 2 ? 1.0 : a.vscale;
  if (arr > 0 && !faces_wanted) {                  // lapv: a = 1 on every face
    double* out = a.faces[ax] + (int64_t)op * plane_pts * Hz + (int64_t)z * plane_pts;
    for (int64_t p = (int64_t)y0 * Hx + threadIdx.x; p < (int64_t)y1 * Hx; p += GRF_T) out[p] = 1.0;
    return;
  }
  // coefficients: xi * w (* sigma / s_K)
  const int nk = dim == 3 ? K * K * K : K * K;
  const double* xi = a.xi + ((int64_t)op * a.n_fields + f) * nk;
  double w2sum = 0.0;
  for (int q = threadIdx.x; q < nk; q += GRF_T) {
    int k0, k1, k2 = 0;
    if (dim == 3) {
      k0 = q / (K * K);
      k1 = (q / K) % K;
      k2 = q % K;
    } else {
      k0 = q / K;
      k1 = q % K;
    }
    double kk = (double)(k0 + 1) * (k0 + 1) + (double)(k1 + 1) * (k1 + 1);
    if (dim == 3) kk += (double)(k2 + 1) * (k2 + 1);
    coef[q] = __ldg(xi + q) * pow(1.0 + kk, -a.s);
    w2sum += pow(1.0 + kk, -2.0 * a.s);
  }
  if (a.sigma > 0.0) {
    for (int o = 16; o > 0; o >>= 1) w2sum += __shfl_xor_sync(0xffffffffu, w2sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w2sum;
  }
  __syncthreads();
  if (a.sigma > 0.0) {
    double tot = 0.0;
    for (int i = 0; i < GRF_T / 32; ++i) tot += red[i];
    const double sc = a.sigma / sqrt(tot * (dim == 3 ? 0.125 : 0.25));
    for (int q = threadIdx.x; q < nk; q += GRF_T) coef[q] *= sc;
    __syncthreads();
  }
  // contract with the row (2-D) / plane + row (3-D) bases
  if (dim == 3) {
    for (int q = threadIdx.x; q < K * K; q += GRF_T) {   // u2[a][b] = sum_c coef[a][b][c] Bz(z, c)
      double acc = 0.0;
      for (int cc = 0; cc < K; ++cc) acc += coef[q * K + cc] * bval(a, kz, cc, z);
      u2[q] = acc;
    }
    __syncthreads();
  }
  const double* cb = dim == 3 ? u2 : coef;         // [a][b]
  const int rows = y1 - y0;
  for (int q = threadIdx.x; q < rows * K; q += GRF_T) {   // u[r][a] = sum_b cb[a][b] By(y0 + r, b)
    const int r = q / K, ka = q % K;
    double acc = 0.0;
    for (int kb = 0; kb < K; ++kb) acc += cb[ka * K + kb] * bval(a, ky, kb, y0 + r);
    u[q] = acc;
  }
  __syncthreads();
  // points: g = sum_a u[r][a] Bx(x, a), then the family's coefficient
  for (int64_t p = threadIdx.x; p < (int64_t)rows * Hx; p += GRF_T) {
    const int r = (int)(p / Hx), x = (int)(p % Hx);
    double g = 0.0;
    for (int ka = 0; ka < K; ++ka) g += u[r * K + ka] * bval(a, kx, ka, x);
    const double v = scale * exp(g);
    const int64_t idx = (int64_t)z * plane_pts + (int64_t)(y0 + r) * Hx + x;
    if (arr == 0) {
      a.params[((int64_t)op * a.n_fields + f) * n + idx] = v;
      if (a.family == 1 || (a.family == 2 && f == 1)) a.c[(int64_t)op * n + idx] = v;
      else if (a.family == 0) a.c[(int64_t)op * n + idx] = 0.0;
    } else {
      a.faces[ax][(int64_t)op * plane_pts * Hz + idx] = v;
    }
  }
}
}  // namespace

size_t grf_ws_doubles(int nx, int K) { return (size_t)2 * K * (nx + 1); }

// family: 0 diva (-div(a grad u)), 1 lapv (-Lap u + V u), 2 divac (-div(a grad u) + c u),
// 3 vib (thin plate: params = [D, rho] = [e^{g_0}, e^{g_1}], no faces / c)
int grf_impl(int dim, int nx, int K, double s, double sigma, double vscale, int family, int n_ops,
             const double* xi, double* fx, double* fy, double* fz, double* c, double* params, double* tab,
             cudaStream_t st) {
  const double h = 1.0 / (nx + 1);
  k_grf_basis<<<ceil_div(2 * K * (nx + 1), 256), 256, 0, st>>>(nx, K, h, tab);
  SCSF_LAUNCH_CHECK();
  GrfArgs a;
  a.dim = dim;
  a.nx = nx;
  a.K = K;
  a.family = family;
  a.n_fields = family >= 2 ? 2 : 1;
  a.n_ops = n_ops;
  a.s = s;
  a.sigma = sigma;
  a.vscale = vscale;
  a.h = h;
  a.xi = xi;
  a.tab = tab;
  a.faces[0] = fx;
  a.faces[1] = fy;
  a.faces[2] = fz;
  a.c = c;
  a.params = params;
  const int tiles = dim == 2 ? ceil_div(nx + 1, GRF_TY) : nx + 1;
  dim3 g(tiles, family == 3 ? 1 : 1 + dim, n_ops * a.n_fields);   // vib: nodal fields only
  k_grf_eval<<<g, GRF_T, 0, st>>>(a);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

}  // namespace scsf

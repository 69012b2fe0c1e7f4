// k_sort.cu — Alg. 2 "The Truncated FFT Sorting Algorithm".
//
// Feature extraction (Alg. 2 ll. 3-5): the truncated DFT is only
// p0 of p modes per axis, so instead of a full FFT followed by a crop we
// contract each axis directly with the p0 x p twiddle block
//   E[k][x] = exp(-2 pi i ((k x) mod p) / p),  k = -p0/2 .. p0/2-1
// (exact integer angle reduction, sincospi), one axis at a time.  That is
// p0/ (log p) less work than FFT-then-crop and streams P exactly once.
// Greedy ordering (ll. 6-12): all pairwise squared distances as
// direct differences (R5), then one CTA walks the N-1 dependent argmin steps
// with a (value, index) lexicographic reduction = strict `<` scanning in
// ascending index (R4).
#include "common.cuh"

#include <cfloat>
#include <climits>

namespace scsf {

__global__ void k_twiddles(int p, int p0, double2* E) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p0 * p) return;
  int kk = idx / p, x = idx % p;
  long long k = (long long)kk - p0 / 2;
  long long r = ((k * x) % p + p) % p;
  double s, c;
  sincospi(2.0 * (double)r / (double)p, &s, &c);
  E[idx] = make_double2(c, -s);
}

// out[o][k] = sum_x in[o][x] * E[k][x]   (real input rows of length p, x fastest)
__global__ void k_dft_rows_real(const double* __restrict__ in, int64_t rows, int p, int p0,
                                const double2* __restrict__ E, double2* __restrict__ out) {
  extern __shared__ double srow[];             // [R][p]
  const int R = blockDim.y;
  int64_t r0 = (int64_t)blockIdx.x * R;
  int tid = threadIdx.y * blockDim.x + threadIdx.x;
  int nthr = blockDim.x * blockDim.y;
  for (int t = tid; t < R * p; t += nthr) {
    int64_t r = r0 + t / p;
    srow[t] = (r < rows) ? in[r * p + (t % p)] : 0.0;
  }
  __syncthreads();
  int k = threadIdx.x;
  int64_t r = r0 + threadIdx.y;
  if (k >= p0 || r >= rows) return;
  const double* row = srow + threadIdx.y * p;
  const double2* e = E + (int64_t)k * p;
  double re = 0.0, im = 0.0;
  for (int x = 0; x < p; ++x) {
    double2 w = __ldg(e + x);
    re = fma(row[x], w.x, re);
    im = fma(row[x], w.y, im);
  }
  out[r * p0 + k] = make_double2(re, im);
}

// out[o][k][i] = sum_x in[o][x][i] * E[k][x]  (complex, contraction over a middle axis)
__global__ void k_dft_mid_complex(const double2* __restrict__ in, int64_t outer, int p, int inner,
                                  int p0, const double2* __restrict__ E, double2* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = outer * p0 * inner;
  if (idx >= total) return;
  int i = (int)(idx % inner);
  int k = (int)((idx / inner) % p0);
  int64_t o = idx / ((int64_t)inner * p0);
  const double2* src = in + o * (int64_t)p * inner + i;
  const double2* e = E + (int64_t)k * p;
  double re = 0.0, im = 0.0;
  for (int x = 0; x < p; ++x) {
    double2 v = src[(int64_t)x * inner];
    double2 w = __ldg(e + x);
    re = fma(v.x, w.x, re);
    re = fma(-v.y, w.y, re);
    im = fma(v.x, w.y, im);
    im = fma(v.y, w.x, im);
  }
  out[idx] = make_double2(re, im);
}

// D2[i][j] = sum_m |S_i[m] - S_j[m]|^2, summed in mode order m = 0..M-1.
constexpr int PD_T = 32;   // tile edge
constexpr int PD_MC = 16;  // modes per smem chunk
__global__ void __launch_bounds__(256) k_pairdist(const double2* __restrict__ sig, int N, int M,
                                                  double* __restrict__ D2) {
  __shared__ double2 si[PD_T][PD_MC + 1];
  __shared__ double2 sj[PD_T][PD_MC + 1];
  int i0 = blockIdx.y * PD_T, j0 = blockIdx.x * PD_T;
  int tx = threadIdx.x % 32, ty = threadIdx.x / 32;   // 8 warps; each thread: 4 rows (ty + 8q), column tx
  double acc[4] = {0, 0, 0, 0};
  for (int m0 = 0; m0 < M; m0 += PD_MC) {
    for (int t = threadIdx.x; t < PD_T * PD_MC; t += 256) {
      int r = t / PD_MC, m = t % PD_MC;
      int mm = m0 + m;
      si[r][m] = (i0 + r < N && mm < M) ? sig[(int64_t)(i0 + r) * M + mm] : make_double2(0, 0);
      sj[r][m] = (j0 + r < N && mm < M) ? sig[(int64_t)(j0 + r) * M + mm] : make_double2(0, 0);
    }
    __syncthreads();
    int mend = min(PD_MC, M - m0);
    for (int m = 0; m < mend; ++m) {
      double2 b = sj[tx][m];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 a = si[ty + 8 * q][m];
        double dr = a.x - b.x, di = a.y - b.y;
        acc[q] = fma(dr, dr, acc[q]);
        acc[q] = fma(di, di, acc[q]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < N && j < N) D2[(int64_t)i * N + j] = acc[q];
  }
}

struct Cand {
  double b;
  int j;
  double s;
};
__device__ __forceinline__ Cand merge(Cand x, Cand y) {
  bool xfirst = (x.b < y.b) || (x.b == y.b && x.j < y.j);
  Cand r;
  if (xfirst) {
    r.b = x.b; r.j = x.j; r.s = fmin(x.s, y.b);
  } else {
    r.b = y.b; r.j = y.j; r.s = fmin(y.s, x.b);
  }
  return r;
}

// One CTA: the N-1 dependent greedy steps (Alg. 2 ll. 6-12).
__global__ void __launch_bounds__(1024) k_greedy(const double* __restrict__ D2, int N, int start,
                                                 int* __restrict__ order, double* __restrict__ best,
                                                 double* __restrict__ second) {
  extern __shared__ unsigned char visited[];   // [N]
  __shared__ Cand wres[32];
  __shared__ int cur_s;
  for (int j = threadIdx.x; j < N; j += blockDim.x) visited[j] = 0;
  if (threadIdx.x == 0) {
    visited[start] = 1;
    order[0] = start;
    cur_s = start;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int t = 1; t < N; ++t) {
    const double* row = D2 + (int64_t)cur_s * N;
    Cand c{INFINITY, INT_MAX, INFINITY};
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      if (visited[j]) continue;
      double d = row[j];
      if (d < c.b) {                  // strict <, ascending j within the thread
        c.s = c.b; c.b = d; c.j = j;
      } else if (d < c.s) {
        c.s = d;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Cand y;
      y.b = __shfl_xor_sync(0xffffffffu, c.b, o);
      y.j = __shfl_xor_sync(0xffffffffu, c.j, o);
      y.s = __shfl_xor_sync(0xffffffffu, c.s, o);
      c = merge(c, y);
    }
    if (lane == 0) wres[warp] = c;
    __syncthreads();
    if (warp == 0) {
      Cand y = (lane < nwarp) ? wres[lane] : Cand{INFINITY, INT_MAX, INFINITY};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Cand z;
        z.b = __shfl_xor_sync(0xffffffffu, y.b, o);
        z.j = __shfl_xor_sync(0xffffffffu, y.j, o);
        z.s = __shfl_xor_sync(0xffffffffu, y.s, o);
        y = merge(y, z);
      }
      if (lane == 0) {
        order[t] = y.j;
        best[t - 1] = y.b;
        second[t - 1] = y.s;
        visited[y.j] = 1;
        cur_s = y.j;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host ----

static int64_t sig_len(int dim, int p0) { return dim == 2 ? (int64_t)p0 * p0 : (int64_t)p0 * p0 * p0; }

size_t sort_ws_bytes(int N, int dim, int p, int F, int p0) {
  Arena a(nullptr, 0);
  int64_t NF = (int64_t)N * F;
  a.take<double2>((int64_t)p0 * p);                            // twiddles
  int64_t inter = (dim == 2) ? NF * p * p0 : NF * (int64_t)p * p * p0 + NF * (int64_t)p * p0 * p0;
  a.take<double2>(inter);                                      // axis-pass intermediates
  a.take<double2>(NF * sig_len(dim, p0));                      // signatures
  a.take<double>((int64_t)N * N);                              // D2
  a.take<int>(N);                                              // order
  a.take<double>(2 * (int64_t)N);                              // best, second
  return a.off;
}

int signatures_impl(const double* params, int N, int dim, int p, int F, int p0, double2* sig,
                    Arena& a, cudaStream_t s) {
  int64_t NF = (int64_t)N * F;
  double2* E = a.take<double2>((int64_t)p0 * p);
  int64_t inter = (dim == 2) ? NF * p * p0 : NF * (int64_t)p * p * p0 + NF * (int64_t)p * p0 * p0;
  double2* T = a.take<double2>(inter);
  if (a.overflow) return SCSF_ERR_WORKSPACE;
  k_twiddles<<<ceil_div((int64_t)p0 * p, 256), 256, 0, s>>>(p, p0, E);
  SCSF_LAUNCH_CHECK();
  // x axis: rows = NF * p^(dim-1) real rows of length p
  int64_t rows = NF * (dim == 2 ? p : (int64_t)p * p);
  int R = max(1, min(32, 256 / p0));
  while (R > 1 && (size_t)R * p * sizeof(double) > 48 * 1024) R /= 2;
  dim3 blk(p0, R);
  double2* Tx = T;
  k_dft_rows_real<<<(unsigned)ceil_div(rows, R), blk, (size_t)R * p * sizeof(double), s>>>(
      params, rows, p, p0, E, Tx);
  SCSF_LAUNCH_CHECK();
  if (dim == 2) {
    // y axis: [NF][p][p0] -> [NF][p0][p0]
    int64_t total = NF * p0 * p0;
    k_dft_mid_complex<<<ceil_div(total, 256), 256, 0, s>>>(Tx, NF, p, p0, p0, E, sig);
    SCSF_LAUNCH_CHECK();
  } else {
    // y axis: [NF*p(z)][p(y)][p0] -> [NF*p][p0][p0]; z axis: [NF][p][p0*p0] -> [NF][p0][p0*p0]
    double2* Ty = T + NF * (int64_t)p * p * p0;
    int64_t total = NF * p * p0 * p0;
    k_dft_mid_complex<<<ceil_div(total, 256), 256, 0, s>>>(Tx, NF * p, p, p0, p0, E, Ty);
    SCSF_LAUNCH_CHECK();
    total = NF * (int64_t)p0 * p0 * p0;
    k_dft_mid_complex<<<ceil_div(total, 256), 256, 0, s>>>(Ty, NF, p, p0 * p0, p0, E, sig);
    SCSF_LAUNCH_CHECK();
  }
  return SCSF_OK;
}

int sort_impl(const double* params, int N, int dim, int p, int F, int p0, int start, int* perm,
              double* d2_best, double* d2_second, Arena& a, cudaStream_t s) {
  int64_t M = (int64_t)F * sig_len(dim, p0);
  // signatures first (their intermediates are carved inside)
  size_t mark = a.off;
  a.take<double2>((int64_t)p0 * p);
  int64_t NF = (int64_t)N * F;
  int64_t inter = (dim == 2) ? NF * p * p0 : NF * (int64_t)p * p * p0 + NF * (int64_t)p * p0 * p0;
  a.take<double2>(inter);
  double2* sig = a.take<double2>((int64_t)N * M);
  double* D2 = a.take<double>((int64_t)N * N);
  int* order = a.take<int>(N);
  double* bs = a.take<double>(2 * (int64_t)N);
  if (a.overflow) return SCSF_ERR_WORKSPACE;
  size_t end = a.off;
  a.off = mark;
  SCSF_TRY(signatures_impl(params, N, dim, p, F, p0, sig, a, s));
  a.off = end;
  dim3 g(ceil_div(N, PD_T), ceil_div(N, PD_T));
  k_pairdist<<<g, 256, 0, s>>>(sig, N, (int)M, D2);
  SCSF_LAUNCH_CHECK();
  size_t smem = (size_t)N;
  if (smem > 48 * 1024) {
    SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_greedy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(smem < 200 * 1024 ? smem : 200 * 1024)));
  }
  if (smem > 200 * 1024) {
    set_error("scsf_sort: N=%d exceeds the greedy kernel's visited-mask capacity", N);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  k_greedy<<<1, 1024, smem, s>>>(D2, N, start, order, bs, bs + N);
  SCSF_LAUNCH_CHECK();
  SCSF_CUDA_CHECK(cudaMemcpyAsync(perm, order, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  if (N > 1 && d2_best)
    SCSF_CUDA_CHECK(cudaMemcpyAsync(d2_best, bs, sizeof(double) * (N - 1), cudaMemcpyDeviceToHost, s));
  if (N > 1 && d2_second)
    SCSF_CUDA_CHECK(cudaMemcpyAsync(d2_second, bs + N, sizeof(double) * (N - 1), cudaMemcpyDeviceToHost, s));
  SCSF_CUDA_CHECK(cudaStreamSynchronize(s));
  return SCSF_OK;
}

}  // namespace scsf

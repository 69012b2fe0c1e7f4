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

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

namespace scsf {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------- gemm_tn ----
constexpr int TN_BM = 64;

// C[i + j ldc] = alpha * sum_z P[z][i + j b1].  Warp w sums z = w, w+8, ... (ascending);
// the 8 warp sums are then added in warp order: a fixed order, so deterministic.
// Symmetric results (Gram, Rayleigh quotient) are read as upper triangles by their consumers.
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ P, int splits, int b1,
                                                         int b2, double alpha, int upper, int gw,
                                                         double* __restrict__ C, int64_t ldc) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  const int j = blockIdx.y;
  if (upper && (int)blockIdx.x * 32 > j % gw) return;     // tile strictly below the diagonal (of its group)
  const int64_t stride = (int64_t)b1 * b2;
  double s = 0.0;
  if (i < b1) {
    const double* p = P + i + (int64_t)j * b1;
#pragma unroll 4
    for (int z = warp; z < splits; z += 8) s += __ldg(p + z * stride);
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && i < b1) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    C[i + (int64_t)j * ldc] = alpha * t;
  }
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

// =====================================================================
// v2 tiles: 128 threads (4 warps, 2 x 2), 64 x 64 CTA tile, warp tile 32 x 32
// (4 x 4 DMMA m8n8k4 per k-step: 16 independent accumulators per warp, 8
// fragment loads per 16 DMMA), k-chunks of 32 moved by cp.async into a
// 2-stage shared-memory ring.  Shared-memory row pitch 36 doubles (= 4 mod 16)
// makes every fragment load conflict-free per half-warp.
// =====================================================================
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int V2_T = 64, V2_KC = 32, V2_P = V2_KC + 4;   // tile, k-chunk, pitch
constexpr int V2_NT = 128;                                 // threads per CTA

// ---- TN: P[z] = X[kz, i-tile]^T Y[kz, j-tile]; upper: only tiles ti <= tj
// TN pipeline: k-chunks of 16 in a 4-stage cp.async ring (3 chunks in flight): the Gram products
// stream X and Y once with little reuse per CTA, so load latency, not DMMA, bounds a short chunk loop.
// Pitch 24 (= 8 mod 16 doubles): the 128-bit fragment loads below are conflict-free per quarter-warp.
constexpr int TN_KC = 16, TN_P = TN_KC + 8, TN_ST = 4;

__global__ void __launch_bounds__(V2_NT) k_gemm_tn2(const double* __restrict__ X, int64_t ldx, int b1,
                                                  const double* __restrict__ Y, int64_t ldy, int b2, int64_t n,
                                                  int64_t kchunk, int upper, int a16, double* __restrict__ P,
                                                  const double* __restrict__ Y2) {
  extern __shared__ __align__(16) double smd[];
  double* xs = smd;                                  // [TN_ST][64][20]
  double* ys = smd + TN_ST * V2_T * TN_P;            // [TN_ST][64][20]
  // dual mode (Y2 != NULL): output columns [0, b2) = X^T Y (upper rule), [b2, 2 b2) = X^T Y2 (full)
  const int T2 = (b2 + V2_T - 1) / V2_T;
  const int grp = Y2 ? (int)blockIdx.y / T2 : 0;
  const int ti = blockIdx.x, tj = Y2 ? (int)blockIdx.y % T2 : (int)blockIdx.y;
  if (upper && ti > tj) return;                     // dual mode: both products upper-triangle
  if (grp) Y = Y2;
  const int i0 = ti * V2_T, j0 = tj * V2_T;
  const int b2tot = Y2 ? 2 * b2 : b2;
  const int jout = grp * b2;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(n, kbeg + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int nck = (int)((kend - kbeg + TN_KC - 1) / TN_KC);

  auto issue = [&](int c, int stage) {
    const int64_t k0 = kbeg + (int64_t)c * TN_KC;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + V2_NT * q;             // 0..511
      const int col = idx >> 3, seg = idx & 7;     // 64 columns x 8 16-byte segments
      const int64_t k = k0 + 2 * seg;
      const int rem = (int)max((int64_t)0, min((int64_t)2, kend - k));
      double* dx = xs + (stage * V2_T + col) * TN_P + 2 * seg;
      double* dy = ys + (stage * V2_T + col) * TN_P + 2 * seg;
      const bool okx = (i0 + col < b1) && rem > 0, oky = (j0 + col < b2) && rem > 0;
      const double* sx = okx ? X + k + (int64_t)(i0 + col) * ldx : X;
      const double* sy = oky ? Y + k + (int64_t)(j0 + col) * ldy : Y;
      if (a16) {
        cp_async16(dx, sx, okx ? 8 * rem : 0);
        cp_async16(dy, sy, oky ? 8 * rem : 0);
      } else {                         // odd leading dimension: 8-byte copies
        cp_async8(dx, sx, okx ? 8 : 0);
        cp_async8(dx + 1, okx && rem > 1 ? sx + 1 : sx, (okx && rem > 1) ? 8 : 0);
        cp_async8(dy, sy, oky ? 8 : 0);
        cp_async8(dy + 1, oky && rem > 1 ? sy + 1 : sy, (oky && rem > 1) ? 8 : 0);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // a warp whose 32 x 32 block lies outside b1 x b2, or (upper mode, diagonal tile) strictly below
  // the diagonal, only helps load: consumers read the upper triangle, its entries stay 0
  const bool idle = (i0 + wm >= b1) || (j0 + wn >= b2) || (upper && ti == tj && wm > wn);

#pragma unroll
  for (int st = 0; st < TN_ST - 1; ++st) {
    if (st < nck) issue(st, st);
    cp_commit();
  }
  for (int c = 0; c < nck; ++c) {
    cp_wait<TN_ST - 2>();                            // chunk c has landed (this thread's copies) ...
    __syncthreads();                                 // ... everyone's, and chunk c-1's stage is free
    if (c + TN_ST - 1 < nck) issue(c + TN_ST - 1, (c + TN_ST - 1) % TN_ST);
    cp_commit();
    const int stage = c % TN_ST;
    // k pairs: lane (g, t) takes k = kk + 2t, kk + 2t + 1 with one 128-bit load and feeds them to
    // two DMMAs as fragment k-index t (the same permutation of k on both operands: the sum over
    // k is unchanged), halving the fragment load instructions
    const double* xa = xs + (stage * V2_T + wm + g) * TN_P + 2 * t;
    const double* yb = ys + (stage * V2_T + wn + g) * TN_P + 2 * t;
    if (idle) continue;                              // warp-uniform
#pragma unroll
    for (int kk = 0; kk < TN_KC; kk += 8) {
      double2 a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = *reinterpret_cast<const double2*>(xa + mi * 8 * TN_P + kk);
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = *reinterpret_cast<const double2*>(yb + ni * 8 * TN_P + kk);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, b[ni].x);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, b[ni].y);
    }
  }
  double* out = P + (int64_t)blockIdx.z * b1 * b2tot;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wm + mi * 8 + g, j = j0 + wn + ni * 8 + 2 * t + e;
        if (i < b1 && j < b2) out[i + (int64_t)(j + jout) * b1] = acc[mi][ni][e];
      }
}

// =====================================================================
// TN with TMA: the same 64 x 64 split-K Gram tile, operands delivered by the tensor-memory
// accelerator.  One producer warp (one elected lane) streams 16-row x 64-column boxes of X and
// Y (cp.async.bulk.tensor.2d, 128-byte swizzle, rows / columns past the operand zero-filled by
// the hardware) into a TNT_ST-stage ring guarded by mbarriers (full: expect_tx bytes; empty:
// one arrive per consumer warp); the 4 consumer warps run the DMMA loop.  No per-thread address
// arithmetic or cp.async groups, and no CTA-wide barrier per chunk.
//
// Swizzled layout: a box lands as 64 rows of 128 B (one per X column), the 16-byte unit u of
// row c stored at unit u ^ (c & 7).  A fragment row g of DMMA block mi reads X column
// 4 g + mi (B: Y column 4 g + ni) of the warp's 32, so the 8 lanes of a 128-bit shared-load
// phase (g = 2p, 2p+1) hit units t ^ mi and t ^ (4 + mi): 8 distinct units, conflict-free.
// =====================================================================
constexpr int TNT_ST = 6, TNT_BOX_R = 16, TNT_NT = 160;
constexpr int TNT_TILE_BYTES = V2_T * TNT_BOX_R * 8;          // 8 KB per operand box

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// TW = 64: 4 consumer warps of 32 x 32 (2 CTAs per SM); TW = 128 (b1 > 128): 8 consumer warps of
// 32 x 64 on a 128 x 128 tile, twice the flops per operand byte of the 64-wide tile (one CTA per SM,
// 6 stages of 2 x 16 KB).  Boxes are 16 rows x TW columns; the swizzled fragment addressing is the
// same (a box column is one 128-byte row).
template <int TW>
__global__ void __launch_bounds__(32 * (TW / 16 + 1)) k_gemm_tn_tma(const __grid_constant__ CUtensorMap tmX,
                                                      const __grid_constant__ CUtensorMap tmY,
                                                      const __grid_constant__ CUtensorMap tmY2, int dual, int b1,
                                                      int b2, int64_t n, int64_t kchunk, int upper,
                                                      double* __restrict__ P) {
  constexpr int NCW = TW / 16;                       // consumer warps: (TW / 32) rows x 2 columns of warps
  constexpr int NI = TW / 16;                        // 8-column DMMA blocks per warp (warp tile 32 x TW / 2)
  constexpr int TILE_BYTES = TW * TNT_BOX_R * 8;
  extern __shared__ __align__(1024) unsigned char tsm[];
  // 1024-byte aligned ring: [TNT_ST] x {X box, Y box}; then the barriers
  unsigned char* base = tsm + ((1024 - (smem_u32(tsm) & 1023)) & 1023);
  const uint32_t ring = smem_u32(base);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + TNT_ST * 2 * TILE_BYTES);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * TNT_ST;

  const int T2 = (b2 + TW - 1) / TW;
  const int grp = dual ? (int)blockIdx.y / T2 : 0;
  const int ti = blockIdx.x, tj = dual ? (int)blockIdx.y % T2 : (int)blockIdx.y;
  if (upper && ti > tj) return;
  const int i0 = ti * TW, j0 = tj * TW;
  const int b2tot = dual ? 2 * b2 : b2;
  const int jout = grp * b2;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(n, kbeg + kchunk);
  const int nck = (int)((kend - kbeg + TNT_BOX_R - 1) / TNT_BOX_R);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int st = 0; st < TNT_ST; ++st) {
      mbar_init(full0 + 8 * st, 1);
      mbar_init(empty0 + 8 * st, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {                                 // producer
    if (lane == 0) {
      const CUtensorMap* my = grp ? &tmY2 : &tmY;
      for (int c = 0; c < nck; ++c) {
        const int st = c % TNT_ST;
        if (c >= TNT_ST) mbar_wait(empty0 + 8 * st, ((c / TNT_ST) - 1) & 1);
        const uint32_t fb = full0 + 8 * st;
        mbar_expect_tx(fb, 2 * TILE_BYTES);
        const int k0 = (int)(kbeg + (int64_t)c * TNT_BOX_R);
        tma_load_2d(ring + st * 2 * TILE_BYTES, &tmX, k0, i0, fb);
        tma_load_2d(ring + st * 2 * TILE_BYTES + TILE_BYTES, my, k0, j0, fb);
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * (TW / 2);
  // idle: past the operand, or (upper mode, diagonal tile) entirely below the diagonal
  const bool idle = (i0 + wm >= b1) || (j0 + wn >= b2) || (upper && ti == tj && wm >= wn + TW / 2);
  double acc[4][NI][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int c = 0; c < nck; ++c) {
    const int st = c % TNT_ST;
    mbar_wait(full0 + 8 * st, (c / TNT_ST) & 1);
    if (!idle) {
      const unsigned char* xs = base + st * 2 * TILE_BYTES;
      const unsigned char* ys = xs + TILE_BYTES;
#pragma unroll
      for (int kk = 0; kk < TNT_BOX_R; kk += 8) {
        const int u = (kk >> 1) + t;               // 16-byte unit: rows kk + 2t, kk + 2t + 1
        double2 a[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int col = wm + 4 * g + mi;
          a[mi] = *reinterpret_cast<const double2*>(xs + col * 128 + ((u ^ (col & 7)) << 4));
        }
#pragma unroll
        for (int h = 0; h < NI / 4; ++h) {               // 32-column halves, each as in the 64-wide tile
          double2 b[4];                                  // (one half's B fragments live at a time)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int col = wn + h * 32 + 4 * g + q;
            b[q] = *reinterpret_cast<const double2*>(ys + col * 128 + ((u ^ (col & 7)) << 4));
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int q = 0; q < 4; ++q) dmma(acc[mi][4 * h + q][0], acc[mi][4 * h + q][1], a[mi].x, b[q].x);
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int q = 0; q < 4; ++q) dmma(acc[mi][4 * h + q][0], acc[mi][4 * h + q][1], a[mi].y, b[q].y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);     // this warp is done with the stage
  }
  double* out = P + (int64_t)blockIdx.z * b1 * b2tot;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + wm + 4 * g + mi, j = j0 + wn + (ni >> 2) * 32 + 4 * (2 * t + e) + (ni & 3);
        if (i < b1 && j < b2) out[i + (int64_t)(j + jout) * b1] = acc[mi][ni][e];
      }
}
static size_t tnt_smem(int tw = V2_T) { return (size_t)TNT_ST * 2 * tw * TNT_BOX_R * 8 + 2 * 8 * TNT_ST + 1024; }
// SCSF_TN_WIDE=1: 128-wide TMA tiles for b1, b2 > 128 (off by default).  Measured (tools/gemm_ab.py,
// profiles/r02_tn_wide_ab.json): the full C3-shape TN 276.8 -> 209.3 us (16.6 -> 22.0 TF/s), C5 upper
// Gram 2377 -> 1795 us, but C5 full 3974 -> 4127 us, and in the solver the C3 bench went 53.6 -> 52.7
// operators/s: locking shrinks the active block below 129 columns within an iteration or two, so few
// calls qualify, and the one-CTA-per-SM 192 KB tiles crowd the concurrent chains' filter clusters.
static bool tn_wide_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_TN_WIDE");
    v = (e && e[0] == '1') ? 1 : 0;
    return v;
  }();
  return v == 1;
}
// splits of a 128-wide TN product: about one wave of one CTA per SM, within the partial-sum workspace
// (tn_partial_doubles: at least 4 148 64^2 + 2 b1 b2 doubles for this call's b1, b2)
static int tn_wide_splits(int64_t n, int b1, int b2tot, int tiles, int64_t cap_doubles);

// Tensor map of a column-major n x cols operand (ld doubles): dim 0 = rows (contiguous), dim 1 =
// columns, box 16 rows x 64 columns, 128-byte swizzle; out-of-range rows / columns read as zero.
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int tma_encode_fn() {
  static std::once_flag once;
  static int status = SCSF_OK;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      status = SCSF_ERR_DEVICE;
      return;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (status != SCSF_OK) set_error("cuTensorMapEncodeTiled is not available from the driver");
  return status;
}
static int make_tmap(CUtensorMap* m, const double* X, int64_t ld, int64_t n, int cols, int box_r = TNT_BOX_R,
                     int box_c = V2_T) {
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_r, (cuuint32_t)box_c};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): n %lld, cols %d, ld %lld", (int)r, (long long)n, cols, (long long)ld);
    return SCSF_ERR_DEVICE;
  }
  return SCSF_OK;
}
// SCSF_TN_TMA=0 keeps the cp.async kernel (k_gemm_tn2) for A/B runs
static bool tn_tma_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_TN_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}
// SCSF_NN_TMA=0 keeps k_gemm_nn3 for the wide NN products (A/B runs)
static bool nn_tma_enabled() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_NN_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v == 1;
}
// TMA needs 16-byte aligned bases and leading dimensions (ld even) and row counts >= 16 to pay
static bool tma_layout_ok(const double* p, int64_t ld, int64_t n) {
  return ((uintptr_t)p & 15) == 0 && (ld & 1) == 0 && n >= 64 && n < (1ll << 31);
}
static bool tma_ok(const double* p, int64_t ld, int64_t n) { return tn_tma_enabled() && tma_layout_ok(p, ld, n); }

// ---- NN: Out[r0:r0+64, :] = alpha X[r0:r0+64, 0:b1] M + beta Out.  The whole
// 64-row panel of X stays resident (so Out may alias X); M streams through a
// 2-stage ring in k-chunks.  tri_upper: M is upper triangular, chunks with
// k > last column of the pass are skipped.
constexpr int NN2_MAX_K = 256;                     // panel 256 x 68 doubles (139 KB) + M ring (37 KB)

__global__ void __launch_bounds__(V2_NT) k_gemm_nn2(const double* __restrict__ X, int64_t ldx, int64_t n, int b1,
                                                  const double* __restrict__ M, int64_t ldm, int b2,
                                                  double alpha, double beta, double* Out, int64_t ldo,
                                                  int tri_upper, int a16) {
  extern __shared__ __align__(16) double smd[];
  const int b1r = (b1 + V2_KC - 1) / V2_KC * V2_KC;
  double* xp = smd;                                  // [b1r][68]: xp[k*68 + r]
  double* ms = smd + b1r * (V2_T + 4);               // [2][64][36]: ms[(st*64 + j)*36 + kk]
  const int64_t r0 = (int64_t)blockIdx.x * V2_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int nck_all = b1r / V2_KC;
  const int rows_here = (int)min((int64_t)V2_T, n - r0);

  auto issue_panel = [&](int c) {      // 32 k-columns x 64 rows: 32 x 32 16-byte segments
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + V2_NT * q;
      const int kk = idx >> 5, seg = idx & 31;
      const int k = c * V2_KC + kk;
      const int rr = 2 * seg;
      const int rem = (k < b1) ? max(0, min(2, rows_here - rr)) : 0;
      const double* src = rem ? X + r0 + rr + (int64_t)k * ldx : X;
      double* dst = xp + k * (V2_T + 4) + rr;
      if (a16) {
        cp_async16(dst, src, 8 * rem);
      } else {                         // odd leading dimension: 8-byte copies
        cp_async8(dst, src, rem ? 8 : 0);
        cp_async8(dst + 1, rem > 1 ? src + 1 : src, rem > 1 ? 8 : 0);
      }
    }
  };
  auto issue_m = [&](int c, int j0, int stage) {   // 64 columns x 32 k (8-byte copies; ldm may be odd)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int idx = tid + V2_NT * q;             // 0..2047
      const int j = idx >> 5, kk = idx & 31;
      const int k = c * V2_KC + kk;
      const bool ok = (k < b1) && (j0 + j < b2);
      cp_async8(ms + (stage * V2_T + j) * V2_P + kk, ok ? (const void*)(M + k + (int64_t)(j0 + j) * ldm) : (const void*)M,
                ok ? 8 : 0);
    }
  };

  for (int j0 = 0; j0 < b2; j0 += V2_T) {
    const bool first = (j0 == 0);
    const int nck = tri_upper ? min(nck_all, (min(b2, j0 + V2_T) + V2_KC - 1) / V2_KC) : nck_all;
    // the whole panel is needed before any write: in the first pass load every chunk
    const int ncp = first ? nck_all : 0;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // groups: G_c = {M chunk c, panel chunk c (first pass)}; remaining panel chunks ride on the last group
    for (int c = 0; c < 2 && c < nck; ++c) {
      issue_m(c, j0, c);
      if (c < ncp) issue_panel(c);
      cp_commit();
    }
    for (int c = 0; c < nck; ++c) {
      if (c + 1 < nck) cp_wait<1>();
      else cp_wait<0>();
      __syncthreads();
      const double* xa = xp + (c * V2_KC + t) * (V2_T + 4) + wm + g;
      const double* mb = ms + ((c & 1) * V2_T + wn + g) * V2_P + t;
      // warp-uniform skips: columns past b2, or a triangular M whose rows of this chunk are all
      // below the warp's columns (M[k][j] = 0 for k > j); the warp still loads and syncs
      const bool idle = (j0 + wn >= b2) || (tri_upper && c * V2_KC > j0 + wn + 31);
#pragma unroll
      for (int kk = 0; kk < V2_KC && !idle; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = xa[kk * (V2_T + 4) + mi * 8];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = mb[ni * 8 * V2_P + kk];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      __syncthreads();
      if (c + 2 < nck) {
        issue_m(c + 2, j0, c & 1);
        if (c + 2 < ncp) issue_panel(c + 2);
        cp_commit();
      }
    }
    if (first && nck < ncp) {        // triangular M cut the first pass short: finish the panel
      for (int c = nck; c < ncp; ++c) issue_panel(c);
      cp_commit();
      cp_wait<0>();
    }
    __syncthreads();                 // every warp is past its panel reads before anyone writes Out
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = r0 + wm + mi * 8 + g;
          const int j = j0 + wn + ni * 8 + 2 * t + e;
          if (r < n && j < b2) {
            double* o = Out + r + (int64_t)j * ldo;
            double v = alpha * acc[mi][ni][e];
            if (beta != 0.0) v = fma(beta, *o, v);
            *o = v;
          }
        }
  }
}

// ---- NN, wide tile: Out[r0:r0+64, j0:j0+128] per pass with 8 warps (2 x 4 warp grid of 32 x 32).
// For large b (C3-C5, V1: b = 240-360) k_gemm_nn2's 176-KB panel leaves one 4-warp CTA per SM
// and sweeps the panel b/64 times; here 8 warps share the panel and it is swept b/128 times.
constexpr int NN3_BN = 128;

// PR = 64: 2 x 4 warps (256 threads); PR = 32: 1 x 4 warps (128 threads) with a 32-row panel,
// so inner dimensions up to 384 fit (C5: b = 360) next to the 2-stage M ring.
template <int PR>
__global__ void __launch_bounds__(PR * 4) k_gemm_nn3(const double* __restrict__ X, int64_t ldx, int64_t n, int b1,
                                                   const double* __restrict__ M, int64_t ldm, int b2,
                                                   double alpha, double beta, double* Out, int64_t ldo,
                                                   int tri_upper, int a16, int m16) {
  constexpr int NT = PR * 4, PP = PR + 4;
  extern __shared__ __align__(16) double smd[];
  const int b1r = (b1 + V2_KC - 1) / V2_KC * V2_KC;
  double* xp = smd;                                  // [b1r][PR + 4]: xp[k*PP + r]
  double* ms = smd + b1r * PP;                       // [2][128][36]: ms[(st*128 + j)*36 + kk]
  const int64_t r0 = (int64_t)blockIdx.x * PR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 32;
  const int nck_all = b1r / V2_KC;
  const int rows_here = (int)min((int64_t)PR, n - r0);

  auto issue_panel = [&](int c) {      // 32 k-columns x PR rows of 16-byte segments
#pragma unroll
    for (int q = 0; q < 16 * PR / NT; ++q) {
      const int idx = tid + NT * q;
      const int kk = idx / (PR / 2), seg = idx % (PR / 2);
      const int k = c * V2_KC + kk;
      const int rr = 2 * seg;
      const int rem = (k < b1) ? max(0, min(2, rows_here - rr)) : 0;
      const double* src = rem ? X + r0 + rr + (int64_t)k * ldx : X;
      double* dst = xp + k * PP + rr;
      if (a16) {
        cp_async16(dst, src, 8 * rem);
      } else {
        cp_async8(dst, src, rem ? 8 : 0);
        cp_async8(dst + 1, rem > 1 ? src + 1 : src, rem > 1 ? 8 : 0);
      }
    }
  };
  auto issue_m = [&](int c, int j0, int stage) {   // 128 columns x 32 k
    if (m16) {
#pragma unroll
      for (int q = 0; q < 2048 / NT; ++q) {
        const int idx = tid + NT * q;              // 0..2047
        const int j = idx >> 4, seg = idx & 15;
        const int k = c * V2_KC + 2 * seg;
        const int rem = (j0 + j < b2) ? max(0, min(2, b1 - k)) : 0;
        cp_async16(ms + (stage * NN3_BN + j) * V2_P + 2 * seg,
                   rem ? (const void*)(M + k + (int64_t)(j0 + j) * ldm) : (const void*)M, 8 * rem);
      }
    } else {
#pragma unroll 4
      for (int q = 0; q < 4096 / NT; ++q) {
        const int idx = tid + NT * q;              // 0..4095
        const int j = idx >> 5, kk = idx & 31;
        const int k = c * V2_KC + kk;
        const bool ok = (k < b1) && (j0 + j < b2);
        cp_async8(ms + (stage * NN3_BN + j) * V2_P + kk,
                  ok ? (const void*)(M + k + (int64_t)(j0 + j) * ldm) : (const void*)M, ok ? 8 : 0);
      }
    }
  };

  for (int j0 = 0; j0 < b2; j0 += NN3_BN) {
    const bool first = (j0 == 0);
    const int nck = tri_upper ? min(nck_all, (min(b2, j0 + NN3_BN) + V2_KC - 1) / V2_KC) : nck_all;
    const int ncp = first ? nck_all : 0;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int c = 0; c < 2 && c < nck; ++c) {
      issue_m(c, j0, c);
      if (c < ncp) issue_panel(c);
      cp_commit();
    }
    for (int c = 0; c < nck; ++c) {
      if (c + 1 < nck) cp_wait<1>();
      else cp_wait<0>();
      __syncthreads();
      const double* xa = xp + (c * V2_KC + t) * PP + wm + g;
      const double* mb = ms + ((c & 1) * NN3_BN + wn + g) * V2_P + t;
      const bool idle = (j0 + wn >= b2) || (tri_upper && c * V2_KC > j0 + wn + 31);   // as k_gemm_nn2
#pragma unroll
      for (int kk = 0; kk < V2_KC && !idle; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = xa[kk * PP + mi * 8];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) b[ni] = mb[ni * 8 * V2_P + kk];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
      __syncthreads();
      if (c + 2 < nck) {
        issue_m(c + 2, j0, c & 1);
        if (c + 2 < ncp) issue_panel(c + 2);
        cp_commit();
      }
    }
    if (first && nck < ncp) {
      for (int c = nck; c < ncp; ++c) issue_panel(c);
      cp_commit();
      cp_wait<0>();
    }
    __syncthreads();                 // every warp is past its panel reads before anyone writes Out
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t r = r0 + wm + mi * 8 + g;
          const int j = j0 + wn + ni * 8 + 2 * t + e;
          if (r < n && j < b2) {
            double* o = Out + r + (int64_t)j * ldo;
            double v = alpha * acc[mi][ni][e];
            if (beta != 0.0) v = fma(beta, *o, v);
            *o = v;
          }
        }
  }
}

// ---- NN, TMA-fed, whole rows: Out[r0:r0+32, 0:b2] = alpha X[r0:r0+32, 0:b1] M + beta Out.
// One producer warp streams k-chunks of 16 through an NNT_ST-stage mbarrier ring with
// cp.async.bulk.tensor.2d (128-byte swizzle; zero fill past n, b1 and b2): two 16-row x 16-k boxes
// of X and b2/128 16-k x 128-column boxes of M per chunk.  Eight consumer warps own 8*NI columns
// each over the CTA's 32 rows (4 x NI DMMA blocks, 8 NI accumulators per lane), so every output
// element is final when the chunk loop ends and the CTA writes whole rows: Out may alias X (all
// of the CTA's X rows are in shared memory before any warp passes the last full barrier).
//
// Fragment maps (conflict-free 128-byte phases, as k_gemm_tn_tma): a 16-byte unit of an M line
// holds k pair (kk + 2t, kk + 2t + 1) of one column; fragment column g of block ni is column
// 8 ni + perm(g), perm(g) = (g >> 1) | ((g & 1) << 2), so the two columns of a phase (g, g + 1)
// differ in bit 2 and their swizzled units (u ^ (col & 7)) never collide.  X is read one double
// per lane: row 8 mi + g of the 32, k = kk + 2t (+1); 16 lanes cover 8 distinct 8-byte slots
// pairs of all 32 banks.
constexpr int NNT_BM = 32, NNT_KC = 16, NNT_CONS = 8, NNT_NT = (NNT_CONS + 1) * 32;
constexpr int NNT_XBOX_BYTES = 16 * NNT_KC * 8;                 // 2 KB: 16 rows x 16 k
constexpr int NNT_MBOX_COLS = 128, NNT_MBOX_BYTES = NNT_MBOX_COLS * NNT_KC * 8;   // 16 KB

__host__ __device__ constexpr int nnt_stages(int NI) { return NI > 4 ? 4 : 6; }
__host__ __device__ constexpr int nnt_mboxes(int NI) { return (NNT_CONS * 8 * NI + NNT_MBOX_COLS - 1) / NNT_MBOX_COLS; }
__host__ __device__ constexpr int nnt_stage_bytes(int NI) { return 2 * NNT_XBOX_BYTES + nnt_mboxes(NI) * NNT_MBOX_BYTES; }

template <int NI>
__global__ void __launch_bounds__(NNT_NT, 1) k_gemm_nn_tma(const __grid_constant__ CUtensorMap tmX,
                                                         const __grid_constant__ CUtensorMap tmM, int64_t n,
                                                         int b1, int b2, double alpha, double beta,
                                                         double* Out, int64_t ldo, int tri_upper) {
  constexpr int ST = nnt_stages(NI), SB = nnt_stage_bytes(NI), NMB = nnt_mboxes(NI);
  extern __shared__ __align__(1024) unsigned char nsm[];
  unsigned char* base = nsm + ((1024 - (smem_u32(nsm) & 1023)) & 1023);
  const uint32_t ring = smem_u32(base);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + ST * SB);
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * ST;
  const int64_t r0 = (int64_t)blockIdx.x * NNT_BM;
  const int nck = (b1 + NNT_KC - 1) / NNT_KC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(full0 + 8 * st, 1);
      mbar_init(empty0 + 8 * st, NNT_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == NNT_CONS) {                            // producer
    if (lane == 0) {
      const int nmb = min(NMB, (b2 + NNT_MBOX_COLS - 1) / NNT_MBOX_COLS);
      for (int c = 0; c < nck; ++c) {
        const int st = c % ST;
        if (c >= ST) mbar_wait(empty0 + 8 * st, ((c / ST) - 1) & 1);
        const uint32_t fb = full0 + 8 * st, dst = ring + st * SB;
        mbar_expect_tx(fb, 2 * NNT_XBOX_BYTES + nmb * NNT_MBOX_BYTES);
        const int k0 = c * NNT_KC;
        tma_load_2d(dst, &tmX, (int)r0, k0, fb);
        tma_load_2d(dst + NNT_XBOX_BYTES, &tmX, (int)r0 + 16, k0, fb);
        for (int q = 0; q < nmb; ++q)
          tma_load_2d(dst + 2 * NNT_XBOX_BYTES + q * NNT_MBOX_BYTES, &tmM, k0, q * NNT_MBOX_COLS, fb);
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int wn = warp * 8 * NI;                      // first column of this warp
  const int pg = (g >> 1) | ((g & 1) << 2);          // fragment column g -> column pg of each 8-block
  const bool none = wn >= b2;
  double acc[4][NI][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int c = 0; c < nck; ++c) {
    const int st = c % ST;
    mbar_wait(full0 + 8 * st, (c / ST) & 1);
    const bool idle = none || (tri_upper && c * NNT_KC > wn + 8 * NI - 1);   // M upper: rows k > last column are 0
    if (!idle) {
      const unsigned char* xs = base + st * SB;
      const unsigned char* ms = xs + 2 * NNT_XBOX_BYTES;
#pragma unroll
      for (int kk = 0; kk < NNT_KC; kk += 8) {
        const int k0 = kk + 2 * t, k1 = k0 + 1;      // this lane's k of the two DMMA passes
        double a0[4], a1[4];
        double2 b[NI];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int r = 8 * (mi & 1) + g;            // row within the 16-row box mi >> 1
          const unsigned char* xb = xs + (mi >> 1) * NNT_XBOX_BYTES + ((r & 1) << 3);
          a0[mi] = *reinterpret_cast<const double*>(xb + k0 * 128 + (((r >> 1) ^ (k0 & 7)) << 4));
          a1[mi] = *reinterpret_cast<const double*>(xb + k1 * 128 + (((r >> 1) ^ (k1 & 7)) << 4));
        }
        const int u = (kk >> 1) + t;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int col = wn + 8 * ni + pg;          // < 8 * NI * NNT_CONS: inside the staged boxes
          const unsigned char* mb = ms + (col >> 7) * NNT_MBOX_BYTES + (col & 127) * 128;
          b[ni] = *reinterpret_cast<const double2*>(mb + ((u ^ (col & 7)) << 4));
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a0[mi], b[ni].x);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a1[mi], b[ni].y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);
  }
  if (none) return;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = r0 + 8 * mi + g;
        const int fc = 2 * t + e;                    // fragment column -> column of the 8-block
        const int j = wn + 8 * ni + ((fc >> 1) | ((fc & 1) << 2));
        if (r < n && j < b2) {
          double* o = Out + r + (int64_t)j * ldo;
          double v = alpha * acc[mi][ni][e];
          if (beta != 0.0) v = fma(beta, *o, v);
          *o = v;
        }
      }
}
static size_t nnt_smem(int NI) { return (size_t)nnt_stages(NI) * nnt_stage_bytes(NI) + 16 * nnt_stages(NI) + 1024; }

// A (b x b, ld) <- upper triangle mirrored into the strict lower triangle
__global__ void k_symm_upper(double* __restrict__ A, int b, int64_t ld) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i < b && i > j) A[i + (int64_t)j * ld] = A[j + (int64_t)i * ld];
}

int symm_upper_impl(double* A, int b, int64_t ld, cudaStream_t s) {
  k_symm_upper<<<dim3(ceil_div(b, 128), b), 128, 0, s>>>(A, b, ld);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// ------------------------------------------------------------------ host ----
static int g_nn_smem_set = 0;

static size_t tn2_smem() { return (size_t)2 * TN_ST * V2_T * TN_P * sizeof(double); }
static size_t nn3_smem(int b1, int pr) {
  const int b1r = (b1 + V2_KC - 1) / V2_KC * V2_KC;
  return ((size_t)b1r * (pr + 4) + (size_t)2 * NN3_BN * V2_P) * sizeof(double);
}
// k_gemm_nn3 for inner dimensions above this (SCSF_NN3_MIN_K).  tools/gemm_bench.cu, n = 4e4:
// b = 240: 20.1 against 16.4 TF/s (k_gemm_nn2); b = 120 (C2): 10.0 against 10.8, and C2 runs
// 5-9 % slower with it, so the 4-warp kernel keeps b <= 128.
static int nn3_min_k() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_NN3_MIN_K");
    v = e ? atoi(e) : 128;
    return v;
  }();
  return v;
}
// k_gemm_nn_tma for inner dimensions above this (SCSF_NNT_MIN_K)
static int nnt_min_k() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_NNT_MIN_K");
    v = e ? atoi(e) : 128;
    return v;
  }();
  return v;
}
static int nn3_big() {                             // SCSF_NN3_BIG=0: the v1 kernel for b1 > 256
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_NN3_BIG");
    v = (e && e[0] == '0') ? 0 : 1;
    return v;
  }();
  return v;
}
static size_t nn2_smem(int b1) {
  const int b1r = (b1 + V2_KC - 1) / V2_KC * V2_KC;
  return ((size_t)b1r * (V2_T + 4) + (size_t)2 * V2_T * V2_P) * sizeof(double);
}

int dense_init_attrs() {
  if (g_nn_smem_set) return SCSF_OK;
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       NN_MAX_K * NN_LDS * (int)sizeof(double)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_tn2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tn2_smem()));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_tn_tma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tnt_smem(64)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_tn_tma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tnt_smem(128)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nn2_smem(NN2_MAX_K)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn3<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nn3_smem(NN2_MAX_K, 64)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn3<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nn3_smem(NN_MAX_K, 32)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nnt_smem(2)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nnt_smem(3)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nnt_smem(4)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn_tma<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nnt_smem(5)));
  SCSF_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_nn_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nnt_smem(6)));
  g_nn_smem_set = 1;
  return SCSF_OK;
}

// Rows of the reduction dimension per split-K CTA, at least: long k-loops amortise the
// pipeline prologue and keep the partial-sum traffic small (with many concurrent chains the
// GPU is full anyway, so per-CTA efficiency beats spreading one product over every SM).
static int tn_min_rows() {
  static const int v = [] {            // thread-safe one-time read (chain worker threads)
    int v;
    const char* e = getenv("SCSF_TN_MIN_ROWS");
    v = e ? atoi(e) : 512;
    if (v < 32) v = 32;
    return v;
  }();
  return v;
}

static int tn_wide_splits(int64_t n, int b1, int b2tot, int tiles, int64_t cap_doubles) {
  const int want = max(1, (148 + tiles - 1) / tiles);
  const int maxs = max(1, (int)ceil_div(n, (int64_t)tn_min_rows()));
  const int cap = max(1, (int)(cap_doubles / ((int64_t)b1 * b2tot)));
  return min(min(want, maxs), cap);
}

int tn_splits(int64_t n, int b1, int b2) {
  int tiles = ceil_div(b1, TN_BM) * ceil_div(b2, TN_BM);
  int want = max(1, (2 * 148 + tiles - 1) / tiles);
  int maxs = max(1, ceil_div(n, tn_min_rows()));
  return min(want, maxs);
}

// Upper bound of splits * b1' * b2' over every call with b1' <= b1, b2' <= b2:
// splits <= ceil(296 / tiles') where tiles' >= b1' b2' / 64^2 (full) or
// >= (b1'/64)(b1'/64 + 1)/2 (upper-triangle mode, at least half of the full count), so
// splits * b1' * b2' <= 2 * 296 * 64^2 + b1' * b2'.
size_t tn_partial_doubles(int64_t n, int b1, int b2) {
  (void)n;
  return (size_t)4 * 148 * TN_BM * TN_BM + (size_t)2 * b1 * b2;     // 2 b1 b2: the dual (two-Y) mode
}

// C (b1 x b2, ldc) = alpha X^T Y.  P: workspace of tn_partial_doubles.
// upper (b1 == b2): only the upper-triangle tiles are computed and reduced;
// the consumers (Cholesky, Jacobi) read the upper triangle only.
int gemm_tn(const double* X, int64_t ldx, int b1, const double* Y, int64_t ldy, int b2, int64_t n,
            double alpha, int sym, double* C, int64_t ldc, double* P, cudaStream_t s) {
  if (b1 <= 0 || b2 <= 0) return SCSF_OK;
  SCSF_TRY(dense_init_attrs());
  const int upper = (sym && b1 == b2) ? 1 : 0;
  int splits = tn_splits(n, b1, b2);
  if (upper) {
    const int t = ceil_div(b1, V2_T);
    splits = min(max(1, ceil_div(n, tn_min_rows())), max(1, (2 * 148 + t * (t + 1) / 2 - 1) / (t * (t + 1) / 2)));
  }
  int64_t kchunk = round_up(ceil_div(n, splits), TN_KC);
  splits = ceil_div(n, kchunk);
  dim3 g(ceil_div(b1, V2_T), ceil_div(b2, V2_T), splits);
  if (tma_ok(X, ldx, n) && tma_ok(Y, ldy, n) && tma_encode_fn() == SCSF_OK) {
    if (b1 > 128 && b2 > 128 && tn_wide_enabled()) {           // 128 x 128 tiles, 8 consumer warps
      const int t1 = ceil_div(b1, 128), t2 = ceil_div(b2, 128);
      const int tiles = upper ? t1 * (t1 + 1) / 2 : t1 * t2;
      splits = tn_wide_splits(n, b1, b2, tiles, (int64_t)4 * 148 * TN_BM * TN_BM + (int64_t)2 * b1 * b2);
      kchunk = round_up(ceil_div(n, splits), TN_KC);
      splits = (int)ceil_div(n, kchunk);
      CUtensorMap mx, my;
      SCSF_TRY(make_tmap(&mx, X, ldx, n, b1, TNT_BOX_R, 128));
      SCSF_TRY(make_tmap(&my, Y, ldy, n, b2, TNT_BOX_R, 128));
      k_gemm_tn_tma<128><<<dim3(t1, t2, splits), 32 * 9, tnt_smem(128), s>>>(mx, my, my, 0, b1, b2, n, kchunk, upper,
                                                                           P);
    } else {
      CUtensorMap mx, my;
      SCSF_TRY(make_tmap(&mx, X, ldx, n, b1));
      SCSF_TRY(make_tmap(&my, Y, ldy, n, b2));
      k_gemm_tn_tma<64><<<g, TNT_NT, tnt_smem(64), s>>>(mx, my, my, 0, b1, b2, n, kchunk, upper, P);
    }
  } else {
    const int a16 = (((ldx | ldy) & 1) == 0 && ((uintptr_t)X & 15) == 0 && ((uintptr_t)Y & 15) == 0) ? 1 : 0;
    k_gemm_tn2<<<g, V2_NT, tn2_smem(), s>>>(X, ldx, b1, Y, ldy, b2, n, kchunk, upper, a16, P, nullptr);
  }
  SCSF_LAUNCH_CHECK();
  dim3 gr(ceil_div(b1, 32), b2);
  k_reduce_partials<<<gr, 256, 0, s>>>(P, splits, b1, b2, alpha, upper, b2, C, ldc);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// One pass over X for two symmetric products: C[:, 0:b) = X^T Y1, C[:, b:2b) = X^T Y2,
// upper triangles only (X^T Y2 symmetric in exact arithmetic: the Rayleigh quotient).
// C is b x 2b (ldc >= b).
int gemm_tn_dual(const double* X, int64_t ldx, const double* Y1, const double* Y2, int64_t ldy, int b, int64_t n,
                 double* C, int64_t ldc, double* P, cudaStream_t s) {
  if (b <= 0) return SCSF_OK;
  SCSF_TRY(dense_init_attrs());
  const int t = ceil_div(b, V2_T);
  const int tiles = t * (t + 1);
  int splits = min(max(1, ceil_div(n, tn_min_rows())), max(1, (2 * 148 + tiles - 1) / tiles));
  int64_t kchunk = round_up(ceil_div(n, splits), TN_KC);
  splits = ceil_div(n, kchunk);
  dim3 g(t, 2 * t, splits);
  if (tma_ok(X, ldx, n) && tma_ok(Y1, ldy, n) && tma_ok(Y2, ldy, n) && tma_encode_fn() == SCSF_OK) {
    if (b > 128 && tn_wide_enabled()) {                        // 128 x 128 tiles, 8 consumer warps
      const int tw = ceil_div(b, 128);
      splits = tn_wide_splits(n, b, 2 * b, tw * (tw + 1), (int64_t)4 * 148 * TN_BM * TN_BM + (int64_t)2 * b * b);
      kchunk = round_up(ceil_div(n, splits), TN_KC);
      splits = (int)ceil_div(n, kchunk);
      CUtensorMap mx, m1, m2;
      SCSF_TRY(make_tmap(&mx, X, ldx, n, b, TNT_BOX_R, 128));
      SCSF_TRY(make_tmap(&m1, Y1, ldy, n, b, TNT_BOX_R, 128));
      SCSF_TRY(make_tmap(&m2, Y2, ldy, n, b, TNT_BOX_R, 128));
      k_gemm_tn_tma<128><<<dim3(tw, 2 * tw, splits), 32 * 9, tnt_smem(128), s>>>(mx, m1, m2, 1, b, b, n, kchunk, 1,
                                                                                P);
    } else {
      CUtensorMap mx, m1, m2;
      SCSF_TRY(make_tmap(&mx, X, ldx, n, b));
      SCSF_TRY(make_tmap(&m1, Y1, ldy, n, b));
      SCSF_TRY(make_tmap(&m2, Y2, ldy, n, b));
      k_gemm_tn_tma<64><<<g, TNT_NT, tnt_smem(64), s>>>(mx, m1, m2, 1, b, b, n, kchunk, 1, P);
    }
  } else {
    const int a16 = (((ldx | ldy) & 1) == 0 && ((uintptr_t)X & 15) == 0 && ((uintptr_t)Y1 & 15) == 0 &&
                     ((uintptr_t)Y2 & 15) == 0) ? 1 : 0;
    k_gemm_tn2<<<g, V2_NT, tn2_smem(), s>>>(X, ldx, b, Y1, ldy, b, n, kchunk, 1, a16, P, Y2);
  }
  SCSF_LAUNCH_CHECK();
  dim3 gr(ceil_div(b, 32), 2 * b);
  k_reduce_partials<<<gr, 256, 0, s>>>(P, splits, b, 2 * b, 1.0, 1, b, C, ldc);
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

// Out (n x b2, ldo) = alpha X M + beta Out;  Out may alias X.  tri: M upper triangular.
int gemm_nn_ex(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
               double alpha, double beta, double* Out, int64_t ldo, int tri, cudaStream_t s) {
  if (b2 <= 0 || n <= 0) return SCSF_OK;
  if (b1 > NN_MAX_K) {
    set_error("gemm_nn: inner dimension %d exceeds %d", b1, NN_MAX_K);
    return SCSF_ERR_NOT_IMPLEMENTED;
  }
  SCSF_TRY(dense_init_attrs());
  const int a16n = ((ldx & 1) == 0 && ((uintptr_t)X & 15) == 0) ? 1 : 0;
  const int m16n = ((ldm & 1) == 0 && ((uintptr_t)M & 15) == 0) ? 1 : 0;
  if (b1 > nnt_min_k() && b2 > V2_T && b2 <= NNT_CONS * 8 * 6 && nn_tma_enabled() && tma_layout_ok(X, ldx, n) &&
      tma_layout_ok(M, ldm, b1)) {
    SCSF_TRY(tma_encode_fn());
    CUtensorMap tx, tm;
    SCSF_TRY(make_tmap(&tx, X, ldx, n, b1, 16, NNT_KC));
    SCSF_TRY(make_tmap(&tm, M, ldm, b1, b2, NNT_KC, NNT_MBOX_COLS));
    const int grid = (int)ceil_div(n, NNT_BM);
    switch ((b2 + NNT_CONS * 8 - 1) / (NNT_CONS * 8)) {     // NI: 8 NI columns per consumer warp
      case 2: k_gemm_nn_tma<2><<<grid, NNT_NT, nnt_smem(2), s>>>(tx, tm, n, b1, b2, alpha, beta, Out, ldo, tri); break;
      case 3: k_gemm_nn_tma<3><<<grid, NNT_NT, nnt_smem(3), s>>>(tx, tm, n, b1, b2, alpha, beta, Out, ldo, tri); break;
      case 4: k_gemm_nn_tma<4><<<grid, NNT_NT, nnt_smem(4), s>>>(tx, tm, n, b1, b2, alpha, beta, Out, ldo, tri); break;
      case 5: k_gemm_nn_tma<5><<<grid, NNT_NT, nnt_smem(5), s>>>(tx, tm, n, b1, b2, alpha, beta, Out, ldo, tri); break;
      default: k_gemm_nn_tma<6><<<grid, NNT_NT, nnt_smem(6), s>>>(tx, tm, n, b1, b2, alpha, beta, Out, ldo, tri); break;
    }
  } else if (b1 <= NN2_MAX_K && b1 > nn3_min_k() && b2 > V2_T) {
    k_gemm_nn3<64><<<ceil_div(n, 64), 256, nn3_smem(b1, 64), s>>>(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo,
                                                                 tri, a16n, m16n);
  } else if (b1 > NN2_MAX_K && nn3_big()) {
    k_gemm_nn3<32><<<ceil_div(n, 32), 128, nn3_smem(b1, 32), s>>>(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo,
                                                                 tri, a16n, m16n);
  } else if (b1 <= NN2_MAX_K) {
    const int a16 = ((ldx & 1) == 0 && ((uintptr_t)X & 15) == 0) ? 1 : 0;
    k_gemm_nn2<<<ceil_div(n, V2_T), V2_NT, nn2_smem(b1), s>>>(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo, tri,
                                                            a16);
  } else {
    int b1r = (max(b1, 1) + 3) & ~3;
    size_t smem = (size_t)b1r * NN_LDS * sizeof(double);
    k_gemm_nn<<<ceil_div(n, NN_BM), 128, smem, s>>>(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo);
  }
  SCSF_LAUNCH_CHECK();
  return SCSF_OK;
}

int gemm_nn(const double* X, int64_t ldx, int64_t n, int b1, const double* M, int64_t ldm, int b2,
            double alpha, double beta, double* Out, int64_t ldo, cudaStream_t s) {
  return gemm_nn_ex(X, ldx, n, b1, M, ldm, b2, alpha, beta, Out, ldo, 0, s);
}

}  // namespace scsf

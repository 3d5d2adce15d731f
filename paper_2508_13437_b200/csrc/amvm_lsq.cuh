// amvm_lsq.cuh — device warm start: the regularised least-squares start of
// initial_solution (/root/reference/pkg/src/dmmv/controller.py:134-165) for
// instances without a continuous warm start:
//     (A^T A + 1e-8 I) x = A^T b,   idx_j = nearest level of x_j (ties low),
// with the reference's fallback to x = 0 when the system cannot be solved or
// the solution is not finite (controller.py:146-153).
//
// The reference calls numpy (OpenBLAS syrk + LAPACK dgesv, an LU with
// partial pivoting); here the system is symmetric positive definite, so it
// is factored by Cholesky.  The target therefore agrees to rounding, not
// bitwise, and the rounded start agrees unless a target component lies
// within rounding of a midpoint between two levels (bit
// parity needs the host LAPACK order, which stays the default path).
//
// Kernels: k_gram (lower triangle of A^T A from the column-major At, 32x32
// output tiles, k staged through shared memory), k_atb (warp per column),
// k_chol_step (right-looking rank-1 update of the trailing lower triangle,
// one launch per pivot, grid-wide), k_chol_solve (one CTA: forward and back
// substitution with one barrier per pivot, then the nearest-level rounding).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace amvm {

constexpr int kLsT = 32;  // gram tile

// G[i][j] (i >= j) = sum_k A[k][i] A[k][j] (+ 1e-8 on the diagonal).  A
// column i is At[i*m ...], contiguous, so a tile of 32 columns x 32 rows is
// 32 coalesced 256-byte runs.
__global__ void __launch_bounds__(256) k_gram(int64_t m, int64_t n, const double *__restrict__ At,
                                              double *__restrict__ G) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi) return;
  __shared__ double si[kLsT][kLsT + 1];  // [col in tile][k]
  __shared__ double sj[kLsT][kLsT + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  double acc[4] = {0.0, 0.0, 0.0, 0.0};                    // rows ty, ty+8, ty+16, ty+24 of the tile
  for (int64_t k0 = 0; k0 < m; k0 += kLsT) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = ty + 8 * r;
      const int64_t ci = bi * kLsT + c, cj = bj * kLsT + c, k = k0 + tx;
      si[c][tx] = (ci < n && k < m) ? At[ci * m + k] : 0.0;
      sj[c][tx] = (cj < n && k < m) ? At[cj * m + k] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kLsT; ++k) {
      const double b = sj[tx][k];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = __fma_rn(si[ty + 8 * r][k], b, acc[r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t i = bi * kLsT + ty + 8 * r, j = bj * kLsT + tx;
    if (i < n && j <= i) G[i * n + j] = i == j ? __dadd_rn(acc[r], 1e-8) : acc[r];
  }
}

// c[i] = sum_k A[k][i] b[k], warp per column.
__global__ void __launch_bounds__(256) k_atb(int64_t m, int64_t n, const double *__restrict__ At,
                                             const double *__restrict__ b, double *__restrict__ c) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t k = lane; k < m; k += 32) s = __fma_rn(At[i * m + k], b[k], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) c[i] = s;
}

// Pivot k: G[i][j] -= G[i][k] G[j][k] / G[k][k] for k < j <= i.  Column k
// is not written in this step, so every thread reads it as of step k.  A
// non-positive or non-finite pivot sets *flag = 1 (factorisation failed).
__global__ void __launch_bounds__(256) k_chol_step(int64_t n, int64_t k, double *__restrict__ G,
                                                   int32_t *__restrict__ flag) {
  const double p = G[k * n + k];
  if (!(p > 0.0) || !isfinite(p)) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *flag = 1;
    return;
  }
  const int64_t i = k + 1 + (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t j = k + 1 + (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
  if (i >= n || j > i) return;
  G[i * n + j] = __dsub_rn(G[i * n + j], __ddiv_rn(__dmul_rn(G[i * n + k], G[j * n + k]), p));
}

// L = G[i][k] / sqrt(G[k][k]) (lower triangle of G after all steps).
// Solves L y = c, L^T x = y, then rounds x to the nearest level (ties to the
// lower level, controller.py:156-165); a failed factorisation or a
// non-finite x falls back to x = 0 (flag 1 / 2).
template <int NTB>
__global__ void __launch_bounds__(NTB) k_chol_solve(int64_t n, int64_t nlev, const double *__restrict__ G,
                                                     double *__restrict__ y, const double *__restrict__ levels,
                                                     double *__restrict__ target, int32_t *__restrict__ idx,
                                                     int32_t *__restrict__ flag) {
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = *flag;
  __syncthreads();
  if (!bad) {
    for (int64_t k = 0; k < n; ++k) {  // forward: L y = c
      if (threadIdx.x == 0) {
        const double d = sqrt(G[k * n + k]);
        y[k] = __ddiv_rn(y[k], d);
        piv = d;
      }
      __syncthreads();
      const double d = piv, yk = y[k];
      for (int64_t i = k + 1 + threadIdx.x; i < n; i += NTB)
        y[i] = __dsub_rn(y[i], __dmul_rn(__ddiv_rn(G[i * n + k], d), yk));
      __syncthreads();
    }
    for (int64_t k = n - 1; k >= 0; --k) {  // backward: L^T x = y
      if (threadIdx.x == 0) {
        const double d = sqrt(G[k * n + k]);
        y[k] = __ddiv_rn(y[k], d);
      }
      __syncthreads();
      const double xk = y[k];
      for (int64_t i = threadIdx.x; i < k; i += NTB)
        y[i] = __dsub_rn(y[i], __dmul_rn(__ddiv_rn(G[k * n + i], sqrt(G[i * n + i])), xk));
      __syncthreads();
    }
    int nf = 0;
    for (int64_t i = threadIdx.x; i < n; i += NTB) nf |= !isfinite(y[i]);
    nf = __syncthreads_or(nf);
    if (nf && threadIdx.x == 0) bad = 2;
    __syncthreads();
  } else if (threadIdx.x == 0) {
    bad = 1;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < n; j += NTB) {
    const double v = bad ? 0.0 : y[j];
    if (target) target[j] = v;
    int best = 0;
    double bd = fabs(__dsub_rn(v, levels[0]));
    for (int64_t q = 1; q < nlev; ++q) {
      const double dq = fabs(__dsub_rn(v, levels[q]));
      if (dq < bd) { bd = dq; best = (int)q; }
    }
    idx[j] = best;
  }
  if (threadIdx.x == 0) *flag = bad;
}

}  // namespace amvm

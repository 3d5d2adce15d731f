// amvm_exact.cuh — exhaustive enumeration (the reference's exact oracle,
// dmmv.oracle.brute_force, /root/reference/pkg/src/dmmv/oracle.py:38-111),
// used to check the heuristic against ground truth on small instances.
//
// The reference walks |V|^n assignments in lexicographic index order (digit
// of variable 0 most significant, oracle.py:58-60) and keeps the first
// strict improvement, so the answer is the lexicographically smallest code
// attaining the minimum t.  Here every code is independent: each thread
// evaluates codes from a grid-stride loop, keeps its own lexicographic
// (t, code) minimum, abandons a code as soon as its running row maximum is
// strictly above the global best published so far (an atomicMin on the bit
// pattern of t >= 0, which orders like the value), and the CTA minima are
// reduced by a second one-CTA kernel that also decodes the winner.
//
// Two arithmetic orders, both bitwise the reference's:
//   order 0 (oracle.py:62-64, `assignments @ A.T - b` over chunks of 2^15
//            codes): numpy's dgemm with K = n accumulates each output as a
//            sequential FMA chain over k from 0 (checked bitwise against
//            numpy at K = 3..17), then - b.  numpy switches to gemv when one
//            side is a vector: m == 1 is dgemv_t over the chunk's codes (the
//            4x4/4x2/4x1 kernel of the code's position in its chunk), a
//            single code (|V| = 1) is dgemv_t over the m rows, and both at
//            once is a ddot.
//   order 1 (oracle.py:95-111, the pruned DFS): s = -b, then
//            s = s + levels[d_j] * A[:, j] for j = 0..n-1, unfused.
// The problem is compute-bound FP64 (m*n DFMA per code, A staged once per
// CTA in shared memory, row-major so every thread of a warp reads the same
// word); HBM traffic is A once per CTA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "amvm_device.cuh"

namespace amvm {

constexpr int kBFMaxN = 64;  // codes are int64: nlev^n must fit anyway
constexpr long long kBFChunk = 1 << 15;  // _CHUNK, oracle.py:13

__device__ __forceinline__ bool bf_less(double t, long long c, double bt, long long bc) {
  return t < bt || (t == bt && c < bc);
}

// A element (i, j): staged row-major in shared memory (si = n, sj = 1) or
// read from the column-major At in global memory (si = 1, sj = m).
template <int NTB>
__global__ void __launch_bounds__(NTB) k_brute_force(int64_t m, int n, int nlev, long long total, int order,
                                                      int staged, const double *__restrict__ At,
                                                      const double *__restrict__ b,
                                                      const double *__restrict__ levels,
                                                      unsigned long long *__restrict__ gbest,
                                                      double *__restrict__ blk_t, long long *__restrict__ blk_c) {
  extern __shared__ double sm[];
  double *slv = sm;              // nlev
  double *sb = slv + nlev;       // m
  double *sA = sb + m;           // m * n (staged only)
  for (int k = threadIdx.x; k < nlev; k += NTB) slv[k] = levels[k];
  for (int64_t i = threadIdx.x; i < m; i += NTB) sb[i] = b[i];
  const double *A = At;
  int64_t si = 1, sj = m;
  if (staged) {
    for (int64_t e = threadIdx.x; e < m * n; e += NTB) {
      const int64_t j = e / m, i = e - j * m;
      sA[i * n + j] = At[e];
    }
    A = sA;
    si = n;
    sj = 1;
  }
  __syncthreads();

  if (order == 0 && total == 1 && m == 1) {  // (1 x n) @ (n x 1): numpy's ddot
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const double v = warp_ddot_skx([&](int64_t j) { return slv[0]; }, [&](int64_t j) { return At[j]; }, n, lane);
      if (lane == 0) {
        blk_t[0] = fabs(__dsub_rn(v, sb[0]));
        blk_c[0] = 0;
      }
    }
    return;
  }
  const int gemv_codes = order == 0 && m == 1;     // dgemv_t over the codes of a chunk
  const int gemv_rows = order == 0 && total == 1;  // dgemv_t over the rows

  double x[kBFMaxN];
  double best_t = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  long long best_c = 0x7fffffffffffffffLL;
  const long long stride = (long long)gridDim.x * NTB;
  for (long long c = (long long)blockIdx.x * NTB + threadIdx.x; c < total; c += stride) {
    long long q = c;
#pragma unroll 1
    for (int j = n - 1; j >= 0; --j) {
      const long long d = q % nlev;
      q /= nlev;
      x[j] = slv[d];
    }
    const double bound = __longlong_as_double((long long)*(volatile unsigned long long *)gbest);
    double t = 0.0;
    bool dead = false;
#pragma unroll 1
    for (int64_t i = 0; i < m; ++i) {
      const double *row = A + i * si;
      double s;
      if (gemv_codes) {
        const long long lo = (c / kBFChunk) * kBFChunk;
        const long long cs = total - lo < kBFChunk ? total - lo : kBFChunk;
        const double acc = gemv_row([&](int64_t j) { return x[j]; }, [&](int64_t j) { return row[j * sj]; }, n,
                                    gemv_kind(c - lo, cs));
        s = __dsub_rn(acc, sb[i]);
      } else if (gemv_rows) {
        const double acc = gemv_row([&](int64_t j) { return row[j * sj]; }, [&](int64_t j) { return x[j]; }, n,
                                    gemv_kind(i, m));
        s = __dsub_rn(acc, sb[i]);
      } else if (order == 0) {
        double acc = 0.0;
#pragma unroll 1
        for (int j = 0; j < n; ++j) acc = __fma_rn(x[j], row[j * sj], acc);
        s = __dsub_rn(acc, sb[i]);
      } else {
        s = -sb[i];
#pragma unroll 1
        for (int j = 0; j < n; ++j) s = __dadd_rn(s, __dmul_rn(x[j], row[j * sj]));
      }
      const double a = fabs(s);
      if (a > t) t = a;
      if (t > bound) {
        dead = true;
        break;
      }
    }
    if (!dead && bf_less(t, c, best_t, best_c)) {
      best_t = t;
      best_c = c;
      atomicMin(gbest, (unsigned long long)__double_as_longlong(t));
    }
  }

  // CTA reduction of (t, code), lexicographic
  __shared__ double rt[NTB / 32];
  __shared__ long long rc[NTB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ot = __shfl_down_sync(0xffffffffu, best_t, o);
    const long long oc = __shfl_down_sync(0xffffffffu, best_c, o);
    if (bf_less(ot, oc, best_t, best_c)) { best_t = ot; best_c = oc; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { rt[w] = best_t; rc[w] = best_c; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NTB / 32; ++k)
      if (bf_less(rt[k], rc[k], best_t, best_c)) { best_t = rt[k]; best_c = rc[k]; }
    blk_t[blockIdx.x] = best_t;
    blk_c[blockIdx.x] = best_c;
  }
}

// One CTA: lexicographic minimum over the CTA results, then the winner's
// digits (oracle.py:60, `(codes // place) % nlev`).
template <int NTB>
__global__ void __launch_bounds__(NTB) k_brute_force_final(int nblk, int n, int nlev,
                                                            const double *__restrict__ blk_t,
                                                            const long long *__restrict__ blk_c,
                                                            int32_t *__restrict__ best_idx,
                                                            double *__restrict__ best_t_out,
                                                            int64_t *__restrict__ best_code_out) {
  double bt = __longlong_as_double(0x7ff0000000000000LL);
  long long bc = 0x7fffffffffffffffLL;
  for (int k = threadIdx.x; k < nblk; k += NTB)
    if (bf_less(blk_t[k], blk_c[k], bt, bc)) { bt = blk_t[k]; bc = blk_c[k]; }
  __shared__ double rt[NTB];
  __shared__ long long rc[NTB];
  rt[threadIdx.x] = bt;
  rc[threadIdx.x] = bc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NTB; ++k)
      if (bf_less(rt[k], rc[k], bt, bc)) { bt = rt[k]; bc = rc[k]; }
    *best_t_out = bt;
    if (best_code_out) *best_code_out = bc;
    long long q = bc;
    for (int j = n - 1; j >= 0; --j) {
      best_idx[j] = (int32_t)(q % nlev);
      q /= nlev;
    }
  }
}

}  // namespace amvm

// ---- is_improving (localsearch.py:91-125) and exhaustive_swap_check
// (oracle.py:135-161), verification kernels off the solve path.
namespace amvm {
// Swap test of candidate c: every row keeps lo < a_j - a_i < hi with
// lo = (-t - s)/delta, hi = (t - s)/delta (the row screen only skips rows
// that provably pass, so the verdict is the unscreened one).  Warp per
// candidate.
__global__ void __launch_bounds__(256) k_is_improving(int64_t m, const double *__restrict__ At,
                                                      const double *__restrict__ s, double t, int64_t nc,
                                                      const int32_t *__restrict__ ci, const int32_t *__restrict__ cj,
                                                      const double *__restrict__ cd, int32_t *__restrict__ verdict) {
  const int64_t c = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= nc) return;
  const double d = cd[c];
  const double *ai = At + (int64_t)ci[c] * m, *aj = At + (int64_t)cj[c] * m;
  bool ok = true;
  for (int64_t r = lane; r < m && ok; r += 32) {
    const double lo = __ddiv_rn(__dsub_rn(-t, s[r]), d), hi = __ddiv_rn(__dsub_rn(t, s[r]), d);
    const double diff = __dsub_rn(aj[r], ai[r]);
    ok = lo < diff && diff < hi;
  }
  ok = __all_sync(0xffffffffu, ok);
  if (lane == 0) verdict[c] = ok;
}

// For every ordered pair (i, j) with x_i > x_j: the post-swap objective
// recomputed from scratch (compute_residual, core.py:183-197: numpy's
// dgemv_t order per row, ddot when m == 1) and the swap test's verdict.
// CTA per pair; out_t / out_v are n x n (untouched where x_i <= x_j).
__global__ void __launch_bounds__(256) k_swap_check(int64_t m, int64_t n, const double *__restrict__ At,
                                                    const double *__restrict__ b, const double *__restrict__ lv,
                                                    const int32_t *__restrict__ idx, const double *__restrict__ s,
                                                    double t, double *__restrict__ out_t,
                                                    int32_t *__restrict__ out_v) {
  const int64_t i = blockIdx.x / n, j = blockIdx.x - i * n;
  const double xi = lv[idx[i]], xj = lv[idx[j]];
  if (i == j || !(xi > xj)) return;
  const double d = __dsub_rn(xi, xj);
  auto x = [&](int64_t q) { return q == i ? xj : (q == j ? xi : lv[idx[q]]); };
  double tm = 0.0;
  bool ok = true;
  if (m == 1) {
    if (threadIdx.x < 32) {
      const double v = warp_ddot_skx([&](int64_t q) { return At[q]; }, [&](int64_t q) { return x(q); }, n,
                                     (int)threadIdx.x);
      tm = fabs(__dsub_rn(v, b[0]));
    }
  } else {
    for (int64_t r = threadIdx.x; r < m; r += 256) {
      const double v = gemv_row([&](int64_t q) { return At[q * m + r]; }, [&](int64_t q) { return x(q); }, n,
                                gemv_kind(r, m));
      tm = fmax(tm, fabs(__dsub_rn(v, b[r])));
    }
  }
  for (int64_t r = threadIdx.x; r < m; r += 256) {
    const double lo = __ddiv_rn(__dsub_rn(-t, s[r]), d), hi = __ddiv_rn(__dsub_rn(t, s[r]), d);
    const double diff = __dsub_rn(At[j * m + r], At[i * m + r]);
    ok = ok && lo < diff && diff < hi;
  }
  tm = warp_max(tm);
  ok = __all_sync(0xffffffffu, ok);
  __shared__ double wt[8];
  __shared__ int wv[8];
  if ((threadIdx.x & 31) == 0) { wt[threadIdx.x >> 5] = tm; wv[threadIdx.x >> 5] = ok; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double T = 0.0;
    int V = 1;
    for (int w = 0; w < 8; ++w) { T = fmax(T, wt[w]); V &= wv[w]; }
    out_t[blockIdx.x] = T;
    out_v[blockIdx.x] = V;
  }
}
}  // namespace amvm

// Batched candidate-move scoring: the one_opt candidate objective
// (localsearch.py:76-78)
//     t(j, v) = max_k | s_k + (lv[v] - lv[idx_j]) * A[k, j] |
// for every column j and every candidate level v at once, each column of A
// streamed once (contiguous in the column-major At) and amortised over all
// candidates of that column.  Same arithmetic as the reference: the level
// difference first, then an unfused DMUL and DADD per element; the max of
// absolute values is exact, so the order of the reduction over k does not
// change a bit.
//
// Layout: one warp per (instance, column); lanes stride the rows (256-byte
// coalesced loads, 8 rows in flight per lane for 2 candidates, 2 for 16), each lane keeps one
// running max per candidate in registers (kScoreVC candidates per pass over
// the column; more levels take more passes, re-read from L1/L2), then a
// 5-step shuffle max per candidate.  HBM-bound for the adjacent set (2
// candidates per 8-byte element), FP64-pipe-bound for all 16 levels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace amvm {

constexpr int kScoreVC = 16;      // candidates per pass over a column
constexpr int kScoreWarps = 8;    // columns per CTA

// mode 0: all levels (nv = nlev, candidate v = level v; v == idx gives the
// current objective).  mode 1: adjacent levels (nv = 2: idx - 1, idx + 1;
// +inf where the level does not exist).
template <int MODE>
__global__ void __launch_bounds__(256) k_score_moves(int64_t m, int64_t n, int64_t nlev, int64_t count,
                                                     const double *__restrict__ At, const double *__restrict__ lvs,
                                                     const int32_t *__restrict__ idxs, const double *__restrict__ S,
                                                     double *__restrict__ out_t) {
  constexpr int mode = MODE;
  constexpr int VC = MODE == 1 ? 2 : kScoreVC;
  constexpr int kScoreUnroll = MODE == 1 ? 8 : 2;  // rows in flight per lane
  const int lane = threadIdx.x & 31;
  const int64_t col = (int64_t)blockIdx.x * kScoreWarps + (threadIdx.x >> 5);
  const int64_t c = blockIdx.y;
  if (col >= n || c >= count) return;
  const double *lv = lvs + c * nlev;
  const double *s = S + c * m;
  const double *a = At + col * m;
  const int k = idxs[c * n + col];
  const int64_t nv = mode == 1 ? 2 : nlev;
  double *out = out_t + (c * n + col) * nv;
  for (int64_t v0 = 0; v0 < nv; v0 += VC) {
    double d[VC], mx[VC];
    bool live[VC];
#pragma unroll
    for (int u = 0; u < VC; ++u) {
      const int64_t lvl = mode == 1 ? (int64_t)k + (u == 0 ? -1 : 1) : v0 + u;
      live[u] = (mode == 1 ? u < 2 : v0 + u < nv) && lvl >= 0 && lvl < nlev;
      d[u] = live[u] ? __dsub_rn(lv[lvl], lv[k]) : 0.0;
      mx[u] = 0.0;
    }
    int64_t r = lane;
    for (; r + 32 * (kScoreUnroll - 1) < m; r += 32 * kScoreUnroll) {
      double av[kScoreUnroll], sv[kScoreUnroll];
#pragma unroll
      for (int q = 0; q < kScoreUnroll; ++q) {
        av[q] = __ldg(a + r + 32 * q);
        sv[q] = __ldg(s + r + 32 * q);
      }
#pragma unroll
      for (int q = 0; q < kScoreUnroll; ++q)
#pragma unroll
        for (int u = 0; u < VC; ++u)
          if (mode != 1 || u < 2) mx[u] = fmax(mx[u], fabs(__dadd_rn(sv[q], __dmul_rn(d[u], av[q]))));
    }
    for (; r < m; r += 32) {
      const double av = __ldg(a + r), sv = __ldg(s + r);
#pragma unroll
      for (int u = 0; u < VC; ++u)
        if (mode != 1 || u < 2) mx[u] = fmax(mx[u], fabs(__dadd_rn(sv, __dmul_rn(d[u], av))));
    }
#pragma unroll
    for (int u = 0; u < VC; ++u) {
      if (mode == 1 && u >= 2) break;
      double x = mx[u];
#pragma unroll
      for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == u && (mode == 1 || v0 + u < nv)) out[v0 + u] = live[u] ? x : __longlong_as_double(0x7ff0000000000000LL);
    }
    if (mode == 1) break;
  }
}

// Best move per instance: the lexicographically smallest (t, j, level) over
// candidates that change the level (level != idx_j, level exists), as one
// CTA per instance.  best[c] = j * nv + v (flat index into out_t), -1 if the
// instance has no candidate; best_t[c] = its objective.
__global__ void __launch_bounds__(256) k_score_best(int64_t n, int64_t nlev, int64_t count,
                                                    const int32_t *__restrict__ idxs, int mode,
                                                    const double *__restrict__ out_t, int64_t *__restrict__ best,
                                                    double *__restrict__ best_t) {
  __shared__ double st[8];
  __shared__ int64_t si[8];
  const int64_t c = blockIdx.x;
  if (c >= count) return;
  const int64_t nv = mode == 1 ? 2 : nlev;
  const double *t = out_t + c * n * nv;
  const int32_t *idx = idxs + c * n;
  double bt = __longlong_as_double(0x7ff0000000000000LL);
  int64_t bi = -1;
  for (int64_t e = threadIdx.x; e < n * nv; e += blockDim.x) {
    const int64_t j = e / nv, v = e - j * nv;
    const int64_t lvl = mode == 1 ? (int64_t)idx[j] + (v == 0 ? -1 : 1) : v;
    if (lvl < 0 || lvl >= nlev || lvl == idx[j]) continue;
    const double x = t[e];
    if (bi < 0 || x < bt) { bt = x; bi = e; }  // e ascends per thread: first wins ties
  }
  auto better = [](double xa, int64_t ia, double xb, int64_t ib) {
    if (ib < 0) return true;
    if (ia < 0) return false;
    return xa < xb || (xa == xb && ia < ib);
  };
  for (int o = 16; o; o >>= 1) {
    const double ox = __shfl_xor_sync(0xffffffffu, bt, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (!better(bt, bi, ox, oi)) { bt = ox; bi = oi; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { st[w] = bt; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (!better(bt, bi, st[q], si[q])) { bt = st[q]; bi = si[q]; }
    best[c] = bi;
    best_t[c] = bt;
  }
}

}  // namespace amvm

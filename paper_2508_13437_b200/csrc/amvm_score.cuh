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
constexpr int kScoreWarps = 8;    // warps per CTA
// warps per column (rows split across them, maxima combined in smem).  ncu on
// one C5 instance (adjacent set): 1 warp/column 26 us, 4 warps/column 30 us
// (shorter-lived CTAs, register-limited occupancy), so 1 ships; kept as a knob
#ifndef AMVM_SCORE_UNROLL
#define AMVM_SCORE_UNROLL 16  // adjacent set: rows in flight per lane (A/B: 16 beats 8 by ~5 %)
#endif
#ifndef AMVM_SCORE_ROW_SPLIT
#define AMVM_SCORE_ROW_SPLIT 1
#endif
__host__ __device__ constexpr int score_row_split(int mode) { return mode == 1 ? AMVM_SCORE_ROW_SPLIT : 1; }
__host__ __device__ constexpr int score_cols_per_cta(int mode) { return kScoreWarps / score_row_split(mode); }

// running max of |y| as compare + select: DSETP + DADD(|y|) + 2 FSEL, where
// fmax lowers to DSETP.MAX + SEL + FSEL + register moves; same value (no NaN
// reaches the scorer: Instance validates finiteness)
__device__ __forceinline__ double score_amax(double m, double y) {
  const double ay = fabs(y);
  return ay > m ? ay : m;
}

// lexicographic (t, flat) order with -1 = no candidate (worst)
__device__ __forceinline__ bool score_better(double xa, int64_t ia, double xb, int64_t ib) {
  if (ib < 0) return true;
  if (ia < 0) return false;
  return xa < xb || (xa == xb && ia < ib);
}

__device__ __forceinline__ void score_warp_best(double &bt, int64_t &bi) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ox = __shfl_xor_sync(0xffffffffu, bt, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (!score_better(bt, bi, ox, oi)) { bt = ox; bi = oi; }
  }
}

// MODE 0: all levels (nv = nlev, candidate v = level v; v == idx gives the
// current objective).  MODE 1: adjacent levels (nv = 2: idx - 1, idx + 1;
// +inf where the level does not exist).  Grid (n / kScoreWarps, count).
// Best move per instance, fused: the lexicographically smallest (t, j, level)
// over candidates that change the level, per warp, per CTA (slot in the
// workspace), then by the instance's last CTA to finish (ticket counter,
// reset for the next call).  best[c] = j * nv + v (flat index into out_t),
// -1 if the instance has no candidate; best_t[c] = its objective.
template <int MODE>
__global__ void __launch_bounds__(256, MODE == 1 ? (AMVM_SCORE_UNROLL > 8 ? 2 : 3) : 2) k_score_moves(int64_t m, int64_t n, int64_t nlev, int64_t count,
                                                     const double *__restrict__ At, const double *__restrict__ lvs,
                                                     const int32_t *__restrict__ idxs, const double *__restrict__ S,
                                                     double *__restrict__ out_t, double *__restrict__ blk_t,
                                                     int64_t *__restrict__ blk_i, unsigned *__restrict__ done,
                                                     int64_t *__restrict__ best, double *__restrict__ best_t) {
  constexpr int mode = MODE;
  constexpr int VC = MODE == 1 ? 2 : kScoreVC;
  constexpr int kScoreUnroll = MODE == 1 ? AMVM_SCORE_UNROLL : 2;  // rows in flight per lane
  constexpr int RS = score_row_split(MODE), CPB = score_cols_per_cta(MODE);
  __shared__ double sbt[kScoreWarps];
  __shared__ int64_t sbi[kScoreWarps];
  __shared__ double smx[kScoreWarps][2];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int part = w % RS;  // this warp's share of the column's rows
  const int64_t col = (int64_t)blockIdx.x * CPB + w / RS;
  const int64_t c = blockIdx.y;
  const int64_t nv = mode == 1 ? 2 : nlev;
  // this column's smallest (t, level) over level-changing candidates (every
  // lane holds every reduced max, so every lane tracks it redundantly)
  double cbt = 0.0;
  int32_t cbv = -1;
  if (col < n) {
    const double *lv = lvs + c * nlev;
    const double *s = S + c * m;
    const double *a = At + col * m;
    const int k = idxs[c * n + col];
    double *out = out_t + (c * n + col) * nv;
    for (int64_t v0 = 0; v0 < nv; v0 += VC) {
      double d[VC], mx[VC];
      // candidate u of this pass: its level, and whether that level exists
      auto cand = [&](int u, int64_t &lvl) {
        lvl = mode == 1 ? (int64_t)k + (u == 0 ? -1 : 1) : v0 + u;
        return (mode == 1 ? u < 2 : v0 + u < nv) && lvl >= 0 && lvl < nlev;
      };
#pragma unroll
      for (int u = 0; u < VC; ++u) {
        int64_t lvl;
        d[u] = cand(u, lvl) ? __dsub_rn(lv[lvl], lv[k]) : 0.0;
        mx[u] = 0.0;
      }
      int64_t r = 32 * part + lane;
      for (; r + 32 * RS * (kScoreUnroll - 1) < m; r += 32 * RS * kScoreUnroll) {
        double av[kScoreUnroll], sv[kScoreUnroll];
#pragma unroll
        for (int q = 0; q < kScoreUnroll; ++q) {
          av[q] = __ldg(a + r + 32 * RS * q);
          sv[q] = __ldg(s + r + 32 * RS * q);
        }
#pragma unroll
        for (int q = 0; q < kScoreUnroll; ++q)
#pragma unroll
          for (int u = 0; u < VC; ++u)
            if (mode != 1 || u < 2) mx[u] = score_amax(mx[u], __dadd_rn(sv[q], __dmul_rn(d[u], av[q])));
      }
      for (; r < m; r += 32 * RS) {
        const double av = __ldg(a + r), sv = __ldg(s + r);
#pragma unroll
        for (int u = 0; u < VC; ++u)
          if (mode != 1 || u < 2) mx[u] = score_amax(mx[u], __dadd_rn(sv, __dmul_rn(d[u], av)));
      }
#pragma unroll
      for (int u = 0; u < VC; ++u) {
        if (mode == 1 && u >= 2) break;
        double x = mx[u];
#pragma unroll
        for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (RS > 1) {  // combined across the column's warps below
          if (lane == 0) smx[w][u] = x;
          continue;
        }
        int64_t lvl;
        const bool live = cand(u, lvl);
        if (lane == u && (mode == 1 || v0 + u < nv)) out[v0 + u] = live ? x : __longlong_as_double(0x7ff0000000000000LL);
        const bool moves = live && lvl != k;
        if (moves && (cbv < 0 || x < cbt)) { cbt = x; cbv = (int32_t)(v0 + u); }
      }
      if (mode == 1) break;
    }
  }
  if (RS > 1) {
    __syncthreads();
    if (col < n && part == 0) {
      const int k = idxs[c * n + col];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        double x = smx[w][u];
#pragma unroll
        for (int p = 1; p < RS; ++p) x = fmax(x, smx[w + p][u]);
        const int64_t lvl = (int64_t)k + (u == 0 ? -1 : 1);
        const bool live = lvl >= 0 && lvl < nlev;
        if (lane == u) out_t[(c * n + col) * 2 + u] = live ? x : __longlong_as_double(0x7ff0000000000000LL);
        if (live && (cbv < 0 || x < cbt)) { cbt = x; cbv = u; }
      }
    }
  }
  // CTA best -> per-CTA slot; the last CTA of the instance reduces the slots
  double bt = cbt;
  int64_t bi = cbv < 0 ? -1 : col * nv + cbv;
  if (lane == 0) { sbt[w] = bt; sbi[w] = bi; }
  __syncthreads();
  const int64_t nblk = gridDim.x;
  if (threadIdx.x == 0) {
    for (int q = 1; q < kScoreWarps; ++q)
      if (!score_better(bt, bi, sbt[q], sbi[q])) { bt = sbt[q]; bi = sbi[q]; }
    blk_t[c * nblk + blockIdx.x] = bt;
    blk_i[c * nblk + blockIdx.x] = bi;
    __threadfence();
    last = atomicAdd(&done[c], 1u) == (unsigned)(nblk - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  bt = 0.0;
  bi = -1;
  for (int64_t e = threadIdx.x; e < nblk; e += blockDim.x) {
    const double x = __ldcg(blk_t + c * nblk + e);
    const int64_t i = __ldcg(blk_i + c * nblk + e);
    if (score_better(x, i, bt, bi)) { bt = x; bi = i; }
  }
  score_warp_best(bt, bi);
  __syncthreads();
  if (lane == 0) { sbt[w] = bt; sbi[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kScoreWarps; ++q)
      if (!score_better(bt, bi, sbt[q], sbi[q])) { bt = sbt[q]; bi = sbi[q]; }
    best[c] = bi;
    best_t[c] = bi < 0 ? __longlong_as_double(0x7ff0000000000000LL) : bt;
    done[c] = 0u;  // ready for the next call on this workspace
  }
}

}  // namespace amvm

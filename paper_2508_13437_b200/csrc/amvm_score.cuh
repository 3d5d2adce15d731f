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
static_assert(kScoreWarps % AMVM_SCORE_ROW_SPLIT == 0, "AMVM_SCORE_ROW_SPLIT must divide kScoreWarps");
__host__ __device__ constexpr int score_cols_per_cta(int mode) { return kScoreWarps / score_row_split(mode); }

// running max of |y| as compare + select: DSETP + DADD(|y|) + 2 FSEL, where
// fmax lowers to DSETP.MAX + SEL + FSEL + register moves; same value for
// finite inputs.  PRECONDITION (documented on amvm_score_moves): A, s and
// the levels are finite and no s + d*a overflows -- a NaN would be dropped
// here where numpy's max(abs(.)) propagates it.  Instance validates
// finiteness; score_moves_device checks its residuals.
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


// =====================================================================
// Adjacent-set scorer, HBM-streaming form (the north-star scorer (c) for the
// reference's one_opt candidate set {idx-1, idx+1}, localsearch.py:70-80).
//
// Persistent grid (one 512-thread CTA per SM); CTA b owns a contiguous slab
// of columns.  Columns are contiguous in the column-major At, so a stage of
// CB columns is ONE contiguous CB*8m-byte chunk: thread 0 arms an mbarrier
// with the byte count and issues a single cp.async.bulk (TMA bulk copy,
// UBLKCP) of the chunk into a kScoreStages-deep shared-memory ring, so every
// byte of A is read from HBM exactly once and ~100 KB per SM stay in flight.
// Thread t owns rows t, t+512, ... (R <= kAdjMaxR): its residual entries
// s_r live in registers for the whole call (read once), the column entries
// come from shared memory (consecutive threads, consecutive doubles: no bank
// conflicts).  Per element and candidate: DMUL, DADD (unfused, numpy's
// order) and a compare+select abs-max.  The 2*CB maxima of a stage are
// reduced in a warp by a transpose butterfly (each xor step halves the
// values a lane carries: V-1 + 5-log2(V) shuffles for V = 2*CB maxima
// instead of 5*V), then across the 16 warps through shared memory; one
// __syncthreads per stage both publishes those partial maxima and frees the
// stage's slot for the next bulk copy.  Best move per instance as in
// k_score_moves (CTA slot + ticket, counter left at 0 for the next call).
constexpr int kAdjThreads = 512;
constexpr int kScoreMaxSlabs = 1024;  // persistent-grid cap (>= SM count)
constexpr int kAdjMaxR = 16;         // rows per thread held in registers: m <= 8192
constexpr int kScoreStages = 4;      // bulk-copy ring depth
constexpr int kAdjStageTarget = 32768;  // bytes per stage (CB columns)

__host__ __device__ inline int adj_cols_per_stage(int64_t m) {
  const int64_t cb = kAdjStageTarget / (8 * m);
  return cb < 1 ? 1 : (cb > 4 ? 4 : (int)cb);
}
__host__ __device__ inline size_t adj_smem_bytes(int64_t m) {
  return (size_t)kScoreStages * adj_cols_per_stage(m) * 8 * m + 64;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// one butterfly step of the transpose reduction: a lane with bit `o` clear
// keeps the lower half of its V values and sends the upper half, its partner
// the reverse; both take the max of what they keep and what they receive.
template <int V>
__device__ __forceinline__ void adj_tr_step(double (&x)[8], int lane, int o) {
  const bool up = lane & o;
#pragma unroll
  for (int q = 0; q < V / 2; ++q) {
    const double send = up ? x[q] : x[q + V / 2];
    const double keep = up ? x[q + V / 2] : x[q];
    const double got = __shfl_xor_sync(0xffffffffu, send, o);
    x[q] = got > keep ? got : keep;
  }
}

template <int CB>
__global__ void __launch_bounds__(kAdjThreads, 1)
    k_score_adj(int64_t m, int64_t n, int64_t nlev, int64_t count, const double *__restrict__ At,
                const double *__restrict__ lvs, const int32_t *__restrict__ idxs, const double *__restrict__ S,
                double *__restrict__ out_t, double *__restrict__ blk_t, int64_t *__restrict__ blk_i,
                unsigned *__restrict__ done, int64_t *__restrict__ best, double *__restrict__ best_t) {
  constexpr int NW = kAdjThreads / 32;
  constexpr int V = 2 * CB;  // maxima per stage: (column, lower/upper)
  extern __shared__ __align__(128) unsigned char adj_smem[];
  __shared__ uint64_t full[kScoreStages];
  __shared__ double red[2][NW][V];
  __shared__ double sbt[V];
  __shared__ int64_t sbi[V];
  __shared__ bool last;
  double *ring = (double *)adj_smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t j0 = b * n / G, j1 = (b + 1) * n / G;  // this CTA's slab of columns
  const int64_t ncol = j1 - j0;
  const int64_t nst = (ncol + CB - 1) / CB;           // stages per instance
  const int64_t stage_elems = (int64_t)CB * m;
  const int R = (int)((m + kAdjThreads - 1) / kAdjThreads);
  if (tid == 0) {
    for (int q = 0; q < kScoreStages; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = nst * count;  // (instance, stage) pairs, instance-major
  auto issue = [&](int64_t g) {       // thread 0: bulk copy of pair g into its ring slot
    const int64_t st = g % nst;
    const int64_t jc = j0 + st * CB;
    const int64_t nc = (j1 - jc) < CB ? (j1 - jc) : CB;
    uint64_t *bar = &full[g % kScoreStages];
    const uint32_t bytes = (uint32_t)(nc * m * 8);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring + (g % kScoreStages) * stage_elems, At + jc * m, bytes, bar);
  };
  if (tid == 0)
    for (int64_t g = 0; g < kScoreStages && g < total; ++g) issue(g);
  // per-thread best (t, flat) over the values it finalises (tid < V)
  double my_bt = 0.0;
  int64_t my_bi = -1;
  double s[kAdjMaxR];
  int64_t cur_c = -1;
  for (int64_t g = 0; g < total; ++g) {
    const int64_t c = g / nst, st = g % nst;
    if (c != cur_c) {  // new instance: its residual rows into registers
      cur_c = c;
#pragma unroll
      for (int q = 0; q < kAdjMaxR; ++q) {
        const int64_t r = tid + (int64_t)q * kAdjThreads;
        s[q] = (q < R && r < m) ? __ldg(S + c * m + r) : 0.0;
      }
    }
    const int64_t jc = j0 + st * CB;
    const int nc = (int)((j1 - jc) < CB ? (j1 - jc) : CB);
    const double *lv = lvs + c * nlev;
    double d[V];
#pragma unroll
    for (int cc = 0; cc < CB; ++cc) {
      const int k = cc < nc ? __ldg(idxs + c * n + jc + cc) : 0;
      const double lk = __ldg(lv + k);
      d[2 * cc] = (cc < nc && k > 0) ? __dsub_rn(__ldg(lv + k - 1), lk) : 0.0;
      d[2 * cc + 1] = (cc < nc && k + 1 < nlev) ? __dsub_rn(__ldg(lv + k + 1), lk) : 0.0;
    }
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = 0.0;
    mbar_wait(&full[g % kScoreStages], (uint32_t)((g / kScoreStages) & 1));
    const double *col = ring + (g % kScoreStages) * stage_elems;
#pragma unroll
    for (int q = 0; q < kAdjMaxR; ++q) {
      const int64_t r = tid + (int64_t)q * kAdjThreads;
      if (q < R && r < m) {
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
          const double a = col[cc * m + r];  // rows beyond nc read stale smem: never used
          x[2 * cc] = score_amax(x[2 * cc], __dadd_rn(s[q], __dmul_rn(d[2 * cc], a)));
          x[2 * cc + 1] = score_amax(x[2 * cc + 1], __dadd_rn(s[q], __dmul_rn(d[2 * cc + 1], a)));
        }
      }
    }
    // warp: transpose butterfly, V values -> lane groups
    int o = 16;
    if (V >= 8) { adj_tr_step<8>(x, lane, o); o >>= 1; }
    if (V >= 4) { adj_tr_step<4>(x, lane, o); o >>= 1; }
    if (V >= 2) { adj_tr_step<2>(x, lane, o); o >>= 1; }
    for (; o; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x[0], o);
      x[0] = y > x[0] ? y : x[0];
    }
    // lane's value index: its top log2(V) lane bits (bit 4 selects the upper half first)
    const int vb = V == 8 ? 3 : V == 4 ? 2 : 1;
    const int vid = lane >> (5 - vb);  // step o = 16 decided the top bit of the value index, and so on
    if ((lane & ((32 >> vb) - 1)) == 0) red[g & 1][warp][vid] = x[0];
    __syncthreads();  // partial maxima visible; every thread is done with this ring slot
    if (tid == 0 && g + kScoreStages < total) issue(g + kScoreStages);
    if (tid < V) {
      const int cc = tid >> 1, u = tid & 1;
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) t = red[g & 1][w][tid] > t ? red[g & 1][w][tid] : t;
      if (cc < nc) {
        const int64_t j = jc + cc;
        const int k = __ldg(idxs + c * n + j);
        const bool live = u == 0 ? k > 0 : k + 1 < nlev;
        out_t[(c * n + j) * 2 + u] = live ? t : __longlong_as_double(0x7ff0000000000000LL);
        if (live && score_better(t, j * 2 + u, my_bt, my_bi)) { my_bt = t; my_bi = j * 2 + u; }
      }
    }
    if (st == nst - 1) {  // instance c done in this slab: CTA best -> slot, ticket
      if (tid < V) { sbt[tid] = my_bt; sbi[tid] = my_bi; }
      __syncthreads();
      if (tid == 0) {
        double bt = sbt[0];
        int64_t bi = sbi[0];
        for (int q = 1; q < V; ++q)
          if (!score_better(bt, bi, sbt[q], sbi[q])) { bt = sbt[q]; bi = sbi[q]; }
        blk_t[c * G + b] = bt;
        blk_i[c * G + b] = bi;
        __threadfence();
        last = atomicAdd(&done[c], 1u) == (unsigned)(G - 1);
      }
      __syncthreads();
      my_bt = 0.0;
      my_bi = -1;
      if (last) {  // the instance's last CTA: reduce every slab's best
        __threadfence();
        double bt = 0.0;
        int64_t bi = -1;
        for (int64_t e = tid; e < G; e += kAdjThreads) {
          const double xv = __ldcg(blk_t + c * G + e);
          const int64_t iv = __ldcg(blk_i + c * G + e);
          if (score_better(xv, iv, bt, bi)) { bt = xv; bi = iv; }
        }
        score_warp_best(bt, bi);
        if (lane == 0) { red[0][warp][0] = bt; ((int64_t *)red[1][warp])[0] = bi; }
        __syncthreads();
        if (tid == 0) {
          bt = red[0][0][0];
          bi = ((int64_t *)red[1][0])[0];
          for (int w = 1; w < NW; ++w) {
            const double xv = red[0][w][0];
            const int64_t iv = ((int64_t *)red[1][w])[0];
            if (!score_better(bt, bi, xv, iv)) { bt = xv; bi = iv; }
          }
          best[c] = bi;
          best_t[c] = bi < 0 ? __longlong_as_double(0x7ff0000000000000LL) : bt;
          done[c] = 0u;
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace amvm

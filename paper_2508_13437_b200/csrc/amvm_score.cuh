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
  // |y| by clearing the sign bit (one LOP3 on the high word; fabs() can
  // lower to a DADD -0, |y| on the FP64 pipe)
  const double ay = __longlong_as_double(__double_as_longlong(y) & 0x7fffffffffffffffLL);
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
  if (best == nullptr) return;  // scores only
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
// Persistent grid (one CTA per SM); CTA b owns a contiguous slab of columns.
// Columns are contiguous in the column-major At, so a stage of CB columns is
// ONE contiguous CB*8m-byte chunk moved by a single cp.async.bulk (TMA bulk
// copy, UBLKCP) into an S-deep shared-memory ring: every byte of A is read
// from HBM once and ~128 KB per SM stay in flight.  Warp-specialised: one
// producer warp arms each slot's `full` mbarrier with the byte count and
// issues the copy once the slot's `empty` mbarrier says all 16 consumer
// warps are done with it; consumers never wait on each other inside a slab.
// Consumer thread t owns rows t, t+512, ...: its residual entries stay in
// registers for the whole instance, the column entries come from shared
// memory (consecutive threads, consecutive doubles: conflict-free).  Per
// element and candidate: DMUL, DADD (unfused, numpy's order) and a
// compare+select abs-max.  The 2*CB maxima of a stage are reduced in the
// warp by a transpose butterfly (V-1 + 5-log2 V shuffles for V values
// instead of 5V) and folded into per-column shared slots by 64-bit
// atomicMax on the bit pattern (|y| >= 0: integer order = value order).
// The candidate deltas (lv[idx±1] - lv[idx]) of the whole slab are built
// once per instance in shared memory.  At the end of an instance's slab the
// consumers finalise every column in parallel and the CTA's best move goes
// to a workspace slot; the instance's last CTA (ticket) reduces the slots.
#ifdef AMVM_SCORE_TIMELINE  // diagnostic builds: per-CTA %globaltimer stamps
__device__ unsigned long long g_adj_tl[1024][8];
__device__ unsigned long long g_adj_st[1024][2][16];  // per stage: producer issue, consumer warp 0 data ready
__device__ __forceinline__ unsigned long long adj_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ADJ_TL(k) do { if (threadIdx.x == 0) g_adj_tl[blockIdx.x][k] = adj_now(); } while (0)
#else
#define ADJ_TL(k) do { } while (0)
#endif
constexpr int kAdjThreads = 512;      // consumer threads (largest variant; 256 also built)
constexpr int kScoreMaxSlabs = 1024;  // persistent-grid cap (>= SM count)
constexpr int kAdjMaxR = 16;          // rows per thread held in registers: m <= 8192
constexpr int kAdjMaxStages = 8;      // bulk-copy ring depth (max)
#ifndef AMVM_SCORE_STAGE_BYTES
#define AMVM_SCORE_STAGE_BYTES 32768
#endif
constexpr int kAdjStageTarget = AMVM_SCORE_STAGE_BYTES;  // bytes per stage (CB columns)
constexpr size_t kAdjRingBudget = 200 * 1024;

__host__ __device__ inline int adj_cols_per_stage(int64_t m) {
  const int64_t cb = kAdjStageTarget / (8 * m);
  return cb < 1 ? 1 : (cb > 4 ? 4 : (int)cb);
}
__host__ __device__ inline int adj_stages(int64_t m, int cb) {
  // ring budget net of the two residual buffers (16m bytes)
  const int64_t st = ((int64_t)kAdjRingBudget - 16 * m) / ((int64_t)cb * 8 * m);
  return st > kAdjMaxStages ? kAdjMaxStages : (int)st;
}
// ring + delta/maxima tables (2 x 32 B per slab column) + levels + 2 residuals
__host__ __device__ inline size_t adj_smem_bytes(int64_t m, int cb, int64_t slab_cols, int64_t nlev) {
  return (size_t)adj_stages(m, cb) * cb * 8 * m + (size_t)2 * 32 * slab_cols + 16 * (size_t)((nlev + 1) & ~1ll) +
         16 * (size_t)m + 8 * (size_t)((slab_cols + 8 + 3) & ~3ll);
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// named barrier among the consumer warps only (the producer warp runs free)
template <int NC>
__device__ __forceinline__ void adj_consumer_sync_n() {
  asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// one butterfly step of the transpose reduction: a lane with bit `o` set
// keeps the upper half of its VV values and sends the lower half, its
// partner the reverse; both keep the max of what they hold and receive.
template <int VV>
__device__ __forceinline__ void adj_tr_step(double (&x)[8], int lane, int o) {
  const bool up = lane & o;
#pragma unroll
  for (int q = 0; q < VV / 2; ++q) {
    const double send = up ? x[q] : x[q + VV / 2];
    const double keep = up ? x[q + VV / 2] : x[q];
    const double got = __shfl_xor_sync(0xffffffffu, send, o);
    x[q] = got > keep ? got : keep;
  }
}

template <int CB, int RT, int NC>
__global__ void __launch_bounds__(NC + 32, 1)
    k_score_adj(int64_t m, int64_t n, int64_t nlev, int64_t count, const double *__restrict__ At,
                const double *__restrict__ lvs, const int32_t *__restrict__ idxs, const double *__restrict__ S,
                double *__restrict__ out_t, double *__restrict__ blk_t, int64_t *__restrict__ blk_i,
                unsigned *__restrict__ done, int64_t *__restrict__ best, double *__restrict__ best_t) {
  constexpr int V = 2 * CB;  // maxima per stage: (column, lower/upper)
  constexpr int NWc = NC / 32;
  extern __shared__ __align__(128) unsigned char adj_smem[];
  __shared__ uint64_t full[kAdjMaxStages], empty[kAdjMaxStages], sfull[2], sempty[2];
  __shared__ double wbt[NWc];
  __shared__ int64_t wbi[NWc];
  __shared__ int last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t j0 = b * n / G, j1 = (b + 1) * n / G;  // this CTA's slab of columns
  const int ncol = (int)(j1 - j0);
  const int slab_max = (int)((n + G - 1) / G);
  const int NS = adj_stages(m, CB);
  const int nst = (ncol + CB - 1) / CB;  // stages per instance
  const int m32 = (int)m;
  const int stage_elems = CB * m32;
  double *ring = (double *)adj_smem;
  double2 *dtab = (double2 *)(ring + NS * stage_elems);                   // [2][slab_max] (dm, dp)
  unsigned long long *cmax = (unsigned long long *)(dtab + 2 * slab_max);  // [2][slab_max][2]
  const int nlev_pad = (int)((nlev + 1) & ~1ll);
  const int idx_pad = (slab_max + 8 + 3) & ~3;
  double *slv = (double *)(cmax + 4 * slab_max);    // [2][nlev_pad] levels, by instance parity
  double *sbuf = slv + 2 * nlev_pad;                // [2][m] residuals
  int32_t *sidx = (int32_t *)(sbuf + 2 * m32);      // [2][idx_pad] the slab's level indices (16-B window)
  // TMA'd per instance, ahead of its columns: residual, levels (when 16-B
  // aligned: nlev even), the aligned window of level indices covering the slab
  const bool lv_tma = (nlev & 1) == 0;
  const bool want_best = best != nullptr;
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NWc);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&sfull[q], 1);
      mbar_init(&sempty[q], NWc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: the next scorer launch on this stream may
  // start its CTAs (and stream its columns) while this grid drains; it waits
  // (griddepcontrol.wait below) before its first global store or ticket.
  // Both are no-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  ADJ_TL(0);
  if (warp == NWc) {  // ---------------- producer warp: one lane issues every copy
    // each instance's residual goes into the queue ahead of its columns (a
    // 16 KB TMA copy, so it lands first); the residual buffers alternate by
    // instance parity and are reused once the consumers copied them out
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      int64_t issued = 0;
      for (int64_t c = 0; c < count; ++c) {
        const int par = (int)(c & 1);
        if (c >= 2) mbar_wait(&sempty[par], (uint32_t)(((c - 2) >> 1) & 1));
        const int64_t e0 = c * n + j0, e1 = c * n + j1;
        const int64_t a0 = e0 & ~3ll;
        int64_t a1 = (e1 + 3) & ~3ll;
        if (a1 > ((count * n) & ~3ll)) a1 = (count * n) & ~3ll;  // never past the array; tail via __ldg
        const uint32_t ib = a1 > a0 ? (uint32_t)(a1 - a0) * 4u : 0u;
        const uint32_t lb = lv_tma ? (uint32_t)nlev * 8u : 0u;
        mbar_expect_tx(&sfull[par], (uint32_t)m32 * 8u + ib + lb);
        bulk_g2s(sbuf + par * m32, S + c * m, (uint32_t)m32 * 8u, &sfull[par]);
        if (lb) bulk_g2s(slv + par * nlev_pad, lvs + c * nlev, lb, &sfull[par]);
        if (ib) bulk_g2s(sidx + par * idx_pad, idxs + a0, ib, &sfull[par]);
        for (int st = 0; st < nst; ++st, ++issued) {
          if (issued >= NS) mbar_wait(&empty[slot], ph ^ 1u);
          const int64_t jc = j0 + (int64_t)st * CB;
          const int nc = (int)((j1 - jc) < CB ? (j1 - jc) : CB);
          const uint32_t bytes = (uint32_t)nc * (uint32_t)m32 * 8u;
          mbar_expect_tx(&full[slot], bytes);
          bulk_g2s(ring + slot * stage_elems, At + jc * m, bytes, &full[slot]);
#ifdef AMVM_SCORE_TIMELINE
          if (issued < 16) g_adj_st[blockIdx.x][0][issued] = adj_now();
#endif
          if (++slot == NS) { slot = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }
  // ---------------- consumer warps (RT rows per thread, RT * NC >= m)
  double s[RT];
  int slot = 0;
  uint32_t ph = 0;
  for (int64_t c = 0; c < count; ++c) {
    const int par = (int)(c & 1);
    double2 *dt = dtab + par * slab_max;
    unsigned long long *cm = cmax + par * 2 * slab_max;
    // residual, levels and level indices arrive with the instance's first
    // bytes (TMA); odd nlev and the last few indices of the array (outside
    // the 16-B window) come by __ldg.  Then the delta table, residual rows
    // into registers.
    double *lvp = slv + par * nlev_pad;
    const int64_t e0 = c * n + j0, a0 = e0 & ~3ll;
    const int64_t a1 = ((c * n + j1 + 3) & ~3ll) < ((count * n) & ~3ll) ? ((c * n + j1 + 3) & ~3ll)
                                                                          : ((count * n) & ~3ll);
    if (!lv_tma) {
      for (int q = tid; q < nlev; q += NC) lvp[q] = __ldg(lvs + c * nlev + q);
      adj_consumer_sync_n<NC>();
    }
    mbar_wait(&sfull[par], (uint32_t)((c >> 1) & 1));
    for (int q = tid; q < ncol; q += NC) {
      const int64_t e = e0 + q;
      const int k = e < a1 ? sidx[par * idx_pad + (int)(e - a0)] : __ldg(idxs + e);
      const double lk = lvp[k];
      dt[q] = make_double2(k > 0 ? __dsub_rn(lvp[k - 1], lk) : 0.0, k + 1 < nlev ? __dsub_rn(lvp[k + 1], lk) : 0.0);
      cm[2 * q] = 0ull;
      cm[2 * q + 1] = 0ull;
    }
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tid + q * NC;
      s[q] = r < m32 ? sbuf[par * m32 + r] : 0.0;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sempty[par]);
    adj_consumer_sync_n<NC>();  // delta table and zeroed maxima visible
    ADJ_TL(1);
    for (int st = 0; st < nst; ++st) {
      const int lc0 = st * CB;  // local column of the stage's first column
      double2 d[CB];
#pragma unroll
      for (int cc = 0; cc < CB; ++cc) d[cc] = dt[lc0 + cc < ncol ? lc0 + cc : lc0];
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = 0.0;
      mbar_wait(&full[slot], ph);
      if (st == 0) ADJ_TL(2);
#ifdef AMVM_SCORE_TIMELINE
      if (tid == 0 && c == 0 && st < 16) g_adj_st[blockIdx.x][1][st] = adj_now();
#endif
      const double *col = ring + slot * stage_elems + tid;
      // all shared-memory loads of the stage first, then the arithmetic;
      // rows past m contribute s = a = 0, i.e. |0| (no effect on a max >= 0);
      // columns past the slab end read stale data that is never used
      double a[CB][RT];
#pragma unroll
      for (int q = 0; q < RT; ++q) {
        const bool ok = tid + q * NC < m32;
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) a[cc][q] = ok ? col[cc * m32 + q * NC] : 0.0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp's reads of the slot are done
      if (++slot == NS) { slot = 0; ph ^= 1u; }
#ifdef AMVM_SCORE_NOCOMPUTE  // diagnostic build: stream only
      if (a[0][0] == 12345.0) x[0] = 1.0;
      else continue;
#endif
#pragma unroll
      for (int q = 0; q < RT; ++q) {
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
          x[2 * cc] = score_amax(x[2 * cc], __dadd_rn(s[q], __dmul_rn(d[cc].x, a[cc][q])));
          x[2 * cc + 1] = score_amax(x[2 * cc + 1], __dadd_rn(s[q], __dmul_rn(d[cc].y, a[cc][q])));
        }
      }
      int o = 16;
      if (V >= 8) { adj_tr_step<8>(x, lane, o); o >>= 1; }
      if (V >= 4) { adj_tr_step<4>(x, lane, o); o >>= 1; }
      adj_tr_step<2>(x, lane, o);
      o >>= 1;
      for (; o; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, x[0], o);
        x[0] = y > x[0] ? y : x[0];
      }
      // value index = the lane bits decided by the halving steps (o = 16 the top one)
      constexpr int vb = V == 8 ? 3 : V == 4 ? 2 : 1;
      const int vid = lane >> (5 - vb);
      if ((lane & ((32 >> vb) - 1)) == 0 && lc0 + (vid >> 1) < ncol)
        atomicMax(&cm[2 * (lc0 + (vid >> 1)) + (vid & 1)], (unsigned long long)__double_as_longlong(x[0]));
    }
    ADJ_TL(3);
    // the previous grid on the stream (same outputs / workspace) has finished
    // and its stores are visible before this one writes
    if (c == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    adj_consumer_sync_n<NC>();  // every column's maxima complete
    if (!want_best) {  // scores only: no grid-wide reduction
      for (int q = tid; q < 2 * ncol; q += NC) {
        const int64_t j = j0 + (q >> 1);
        const int u = q & 1;
        const bool live = (u == 0 ? dt[q >> 1].x : dt[q >> 1].y) != 0.0;
        out_t[(c * n + j) * 2 + u] = live ? __longlong_as_double((long long)cm[q])
                                          : __longlong_as_double(0x7ff0000000000000LL);
      }
      continue;
    }
    // the CTA's best over level-changing moves, from the shared maxima only
    // (a neighbour level exists iff its delta is nonzero: levels strictly
    // increase), so the ticket below orders no other global store
    double bt = 0.0;
    int64_t bi = -1;
    for (int q = tid; q < 2 * ncol; q += NC) {
      const int64_t j = j0 + (q >> 1);
      const int u = q & 1;
      const bool live = (u == 0 ? dt[q >> 1].x : dt[q >> 1].y) != 0.0;
      const double t = __longlong_as_double((long long)cm[q]);
      if (live && score_better(t, j * 2 + u, bt, bi)) { bt = t; bi = j * 2 + u; }
    }
    score_warp_best(bt, bi);
    if (lane == 0) { wbt[warp] = bt; wbi[warp] = bi; }
    adj_consumer_sync_n<NC>();
    ADJ_TL(4);
    if (tid == 0) {
      for (int w = 1; w < NWc; ++w)
        if (!score_better(bt, bi, wbt[w], wbi[w])) { bt = wbt[w]; bi = wbi[w]; }
      blk_t[c * G + b] = bt;
      blk_i[c * G + b] = bi;
      unsigned prev;  // release: the slot above is visible before the ticket; acquire: all earlier slots
#if defined(AMVM_SCORE_TICKET_RELAXED)  // diagnostic only: atomic latency without ordering
      prev = atomicAdd(done + c, 1u);
#elif defined(AMVM_SCORE_TICKET_FENCE)
      __threadfence();
      prev = atomicAdd(done + c, 1u);
#else
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done + c) : "memory");
#endif
#ifdef AMVM_SCORE_TIMELINE
      g_adj_tl[blockIdx.x][7] = adj_now();
#endif
      last = prev == (unsigned)(G - 1);
    }
    // the scores themselves, while the ticket is in flight
    for (int q = tid; q < 2 * ncol; q += NC) {
      const int64_t j = j0 + (q >> 1);
      const int u = q & 1;
      const bool live = (u == 0 ? dt[q >> 1].x : dt[q >> 1].y) != 0.0;
      out_t[(c * n + j) * 2 + u] = live ? __longlong_as_double((long long)cm[q])
                                        : __longlong_as_double(0x7ff0000000000000LL);
    }
    adj_consumer_sync_n<NC>();
    ADJ_TL(5);
    if (last) {  // the instance's last CTA: reduce every slab's best
      bt = 0.0;
      bi = -1;
      for (int64_t e = tid; e < G; e += NC) {
        const double xv = __ldcg(blk_t + c * G + e);
        const int64_t iv = __ldcg(blk_i + c * G + e);
        if (score_better(xv, iv, bt, bi)) { bt = xv; bi = iv; }
      }
      score_warp_best(bt, bi);
      if (lane == 0) { wbt[warp] = bt; wbi[warp] = bi; }
      adj_consumer_sync_n<NC>();
      if (tid == 0) {
        for (int w = 1; w < NWc; ++w)
          if (!score_better(bt, bi, wbt[w], wbi[w])) { bt = wbt[w]; bi = wbi[w]; }
        ADJ_TL(6);
        best[c] = bi;
        best_t[c] = bi < 0 ? __longlong_as_double(0x7ff0000000000000LL) : bt;
        done[c] = 0u;  // ready for the next call on this workspace
      }
      adj_consumer_sync_n<NC>();
    }
  }
}

}  // namespace amvm

// amvm_engine.cuh — the AMVM iteration as a CTA-resident device state machine.
//
// One CTA owns one instance at a time (a persistent grid pulls instance ids
// from an atomic counter), so an ALNS iteration — select, destroy, repair,
// local search, accept, weight update, trace — never leaves the SM
// (controller.py:233-275).  Inside the CTA:
//   * thread t owns residual rows i = t + k*NT, so rank-1/rank-2 updates
//     (core.py:208-245) are thread-local;
//   * block-uniform scalars (objectives, refresh counters) are replicated in
//     every thread's registers and evolve identically; cold uniform state
//     (pointers, params, operator bank, counters) lives in shared memory;
//   * RNG draws and the inherently sequential scans (Floyd sampling, the
//     worst-remove cdf) run on thread 0 / warp 0 and are broadcast;
//   * A is column-major (At): one_opt scores a column only after exact row
//     screens fail to reject it (see one_opt), then streams it coalesced;
//   * every decision reproduces the reference's arithmetic bit for bit
//     (unfused DMUL/DADD, numpy reduction orders, OpenBLAS dot orders), so the
//     trajectory equals the reference's.
#pragma once

#include <cstdint>

#include "../../include/amvm.h"
#include "amvm_device.cuh"

namespace amvm {

#ifndef AMVM_NT
#define AMVM_NT 256  // CTA size of the engine kernels
#endif
#ifndef AMVM_MIN_BLOCKS
#define AMVM_MIN_BLOCKS 2
#endif
constexpr int kS = 32;         // one_opt screening rows (exact rejection test), one per lane
// one_opt window: columns per warp; the window (NW * kCW columns) is a
// 128-bit mask, so 16 columns per warp at 256 threads, 8 at 512
template <int NT>
constexpr int kCWv = 4096 / NT < 16 ? 4096 / NT : 16;
constexpr int kB = 8;          // one_opt second screen: flagged columns per batch
#ifndef AMVM_KG
#define AMVM_KG 8
#endif
constexpr int kG = AMVM_KG;    // filter rows staged in smem per find_candidates
template <int NT>
constexpr int kTJv = 2 * NT;  // find_candidates j-tile (level-sorted positions)
#ifndef AMVM_ROW_PASSES
#define AMVM_ROW_PASSES 24
#endif
constexpr int kDrainLong = 1024;  // queue length that keeps the batched passes going
#ifndef AMVM_DRAIN_SHORT
#define AMVM_DRAIN_SHORT 64
#endif
#ifndef AMVM_FC_PAIRS
#define AMVM_FC_PAIRS 4
#endif
// find_candidates enumerates lane-per-pair (instead of lane-per-i with the
// row-0 prefix) when the mean non-empty level bucket holds fewer than this
// many variables (0: never): the i-groups would leave most lanes idle
constexpr int kFcPairs = AMVM_FC_PAIRS;
#ifndef AMVM_FC_PARTS_MUL
#define AMVM_FC_PARTS_MUL 2  // wide CTA: pair-loop work items per warp (C1 A/B: 2 -> 98.8, 4 -> 101.9, 8 -> 107.7 us/it)
#endif
constexpr int kDrainShort = AMVM_DRAIN_SHORT;  // at or below: no row passes, warp-per-pair checks
constexpr int kRowPasses = AMVM_ROW_PASSES;  // queue passes (one filter row each) before fc_rest
constexpr int kMaxDeltaClasses = 4096;  // overflow path: distinct level differences
constexpr int kTabMaxLev = 16; // bound table in smem when nlev <= this
// impact tile: columns = CTA size (one column per thread)
constexpr int kTK = 16;        // impact tile: rows
constexpr int kTKMax = 128;    // narrow impact tile (n < NT): rows at most
#ifndef AMVM_IMPACT_PREFETCH
#define AMVM_IMPACT_PREFETCH 0     // narrow impact tile: next tile's loads in flight while scoring
#endif
// impact stream shapes (columns per thread, rows per slice, ring stages):
// wide instances 4 x 2 x 2 (four independent exp chains per thread),
// n < 4*NT: 1 x 8 x 3.  Both rings fit the phase scratch.
#ifndef AMVM_IMPACT_IC
#define AMVM_IMPACT_IC 4
#define AMVM_IMPACT_IR 2
#define AMVM_IMPACT_IS 2
#endif
constexpr int kIC4 = AMVM_IMPACT_IC, kIR4 = AMVM_IMPACT_IR, kIS4 = AMVM_IMPACT_IS;
constexpr int kIC1 = 1, kIR1 = 8, kIS1 = 3;

// Phase-shared smem scratch: the impact tile or the find_candidates tiles.
// find_candidates scratch: level-bucket bounds first (live across the bucket
// sort, which reuses everything after them), then the staged tiles.
__host__ __device__ inline size_t fc_tb_off(int64_t nlev) { return ((size_t)8 * (nlev + 2) + 15) & ~(size_t)15; }

template <int NT>
__host__ __device__ inline size_t scratch_bytes(int64_t nlev, int tab) {
  constexpr int kTJ = kTJv<NT>, kTC = NT;
  size_t fc = fc_tb_off(nlev) + 8 * kG * kTJ + 4 * 2 * kTJ;
  if (tab) fc += 8 * kG * nlev * nlev;
  size_t imp = 8 * kTC * (kTK + 1) + 16 * kTKMax;
  const size_t r4 = 8 * (size_t)kIS4 * kIC4 * kTC * kIR4, r1 = 8 * (size_t)kIS1 * kIC1 * kTC * kIR1;
  const size_t ring = r4 > r1 ? r4 : r1;
  if (ring > imp) imp = ring;
  return fc > imp ? fc : imp;
}

struct Cand {
  int32_t i, j;
  double d;
};

// find_candidates survivor-queue entry: the pair and its two level indices
// (delta = lv[ki] - lv[kj] is recomputed bit-identically from smem).
struct __align__(16) QEnt {
  int32_t i, j;
  uint16_t ki, kj;
  uint32_t pad;
};

// The kernel's dynamic shared memory.  Engine pointers into it are derived
// from this symbol (not stored), so the compiler keeps them in the shared
// address space (LDS/STS with immediate offsets instead of generic LD/ST).
extern __shared__ __align__(16) unsigned char amvm_dyn_smem[];

// Everything a kernel launch needs, passed by value.
struct KArgs {
  int64_t m, n, nlev, count;
  const double *At, *B, *levels;
  const double *Ar;  // row-major copy of A (m x n), built in the workspace
  const int64_t *cptr;  // CSC copy of A (valid when the header's csc_ok is set)
  const int32_t *crow;
  const double *cval;
  amvm_params prm;
  // start solution (solve) or in/out solution (component ops)
  int32_t *s_idx;
  double *s_r, *s_obj;
  int32_t *s_cnt;
  amvm_pcg64 *rng;
  amvm_result res;
  unsigned char *ws;  // workspace base (header + slots [+ parked instances])
  size_t slot_bytes;
  unsigned char *ist;  // parked per-instance state (chunked solve), else null
  size_t ist_bytes;
  int chunk_iters;     // iterations per task (0: one task per instance)
  int cr_smem, tab, cap;
  int64_t time_budget_ns;  // < 0: none
  // component-op extras
  int op, kind;
  int32_t *x_i, *x_j, *x_cnt;  // find_candidates out / removed in-out
  int32_t *x_saved;
  double *x_d, *x_out4;
  int32_t x_cap, x_r;
  // impact-score cache (solve only): per instance the scores of its CURRENT
  // solution and a valid flag; null for the component ops
  unsigned char *icache;
  size_t icache_bytes;
  int32_t *ivalid;
  // sparse engine (amvm_solve_sparse): A only as the caller's CSC (cptr,
  // crow, cval above, rows ascending per column) and CSR (rows below,
  // columns ascending per row); no dense At / Ar anywhere.  ktop = size of
  // the |s| top list that bounds untouched rows (>= 2 * max column nnz + 1).
  int sparse;
  int32_t ktop;
  const int64_t *rptr;
  const int32_t *rcol;
  const double *rval;
  int64_t fecap;  // column-indexed filter lists: entry capacity (0: off)
};

enum { OP_ONE_OPT = 1, OP_LOCAL_SEARCH, OP_FIND_CAND, OP_BEST_SWAP, OP_IMPACT, OP_DESTROY, OP_REPAIR,
       OP_APPLY_SHIFT, OP_APPLY_SWAP };

struct WsHeader {  // 256 bytes
  int32_t status;
  int32_t next;
  unsigned long long next_task;  // chunked solve: (chunk, instance) tasks handed out
  int32_t csc_ok;                // the workspace CSC copy of A is complete (sparse A)
  int32_t pad[59];
};

// A parked instance between chunks of a chunked solve (the persistent part
// of the ALNS state: current solution, best objective, operator bank, RNG
// lives in amvm_solve's rng array).  progress = chunks done; an instance that
// stops early jumps to the last chunk so later tasks for it are no-ops.
struct InstState {
  int32_t progress, it, ucnt, bcnt;
  double uobj, bobj;
  double w[4], sc[4];
  int64_t seg[4], life[4], bit;
  int64_t mv_ref, mv_raw, elapsed_ns;
  int64_t pc[16];
};

// Workspace: [WsHeader | Ar (row-major copy of A) | slots | parked instances]
__host__ __device__ inline size_t ws_ar_bytes(int64_t m, int64_t n) { return ((size_t)8 * m * n + 255) & ~(size_t)255; }

// CSC copy of A for sparse instances (tomography): built by every launch,
// used when nnz <= csc_cap (density <= 1/8), else the dense paths run.
__host__ __device__ inline int64_t csc_cap(int64_t m, int64_t n) { return (m * n) / 8; }
struct CscLayout {
  size_t ptr, row, val, total;
};
__host__ __device__ inline CscLayout csc_layout(int64_t m, int64_t n) {
  CscLayout L;
  const int64_t cap = csc_cap(m, n);
  L.ptr = 0;
  L.row = (((size_t)8 * (n + 1)) + 255) & ~(size_t)255;
  L.val = L.row + ((((size_t)4 * cap) + 255) & ~(size_t)255);
  L.total = L.val + ((((size_t)8 * cap) + 255) & ~(size_t)255);
  return L;
}

// Bytes of the dense part of the workspace (row-major Ar + the CSC copy of
// A) that precedes the slots: none for the sparse engine.
__host__ __device__ inline size_t ws_dense_bytes(int64_t m, int64_t n, int sparse) {
  return sparse ? 0 : ws_ar_bytes(m, n) + csc_layout(m, n).total;
}

struct InstLayout {
  size_t r, idx, total;
};
__host__ __device__ inline InstLayout inst_layout(int64_t m, int64_t n) {
  InstLayout L;
  L.r = (sizeof(InstState) + 255) & ~(size_t)255;
  L.idx = L.r + (((size_t)8 * m + 255) & ~(size_t)255);
  L.total = L.idx + (((size_t)4 * n + 255) & ~(size_t)255);
  return L;
}

// Per-slot workspace carve-up (shared by host sizing and device use).
// Column-indexed filter list entry (sparse engine): filter row q touches the
// column with folded value b; next = the column's next entry (-1: end).
struct FEnt {
  int32_t q, next;
  double b;
};

struct SlotLayout {
  size_t ur, crg, uidx, cidx, dbuf, pbuf, cbk, lf_lo, lf_len, lf_sum, rows, reps, rsgn, ag, cbuf, que,
      hset, rem, sav, pick, coin, ibuf, srt, rowtmp, top, fhead, fent, total;
  int64_t nleaf, kk, hsz;
};

__host__ __device__ inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// Survivor queue of find_candidates (pairs alive after the staged rows, all
// tiles of one call): at least 64K entries; beyond it pairs finish directly.
__host__ __device__ inline int64_t fc_qcap(int64_t cap) { return cap > 65536 ? cap : 65536; }

__host__ __device__ inline uint64_t gen_mask(uint64_t v) {
  v |= v >> 1; v |= v >> 2; v |= v >> 4; v |= v >> 8; v |= v >> 16; v |= v >> 32;
  return v;
}

__host__ __device__ inline SlotLayout slot_layout(int64_t m, int64_t n, int64_t k_eps, int64_t r, int64_t cap,
                                                   int64_t ktop = 0, int64_t fecap = 0) {
  SlotLayout L;
  int64_t mn = m > n ? m : n;
  L.nleaf = mn / 64 + 4;
  L.kk = k_eps < m ? k_eps : m;
  if (L.kk < 1) L.kk = 1;
  int64_t rr = r > 0 ? r : 1;
  L.hsz = (int64_t)gen_mask((uint64_t)(1.2 * (double)rr)) + 1;
  size_t o = 0;
  L.ur = o; o = al256(o + 8 * m);
  L.crg = o; o = al256(o + 8 * m);
  L.uidx = o; o = al256(o + 4 * n);
  L.cidx = o; o = al256(o + 4 * n);
  L.dbuf = o; o = al256(o + 8 * n);
  L.pbuf = o; o = al256(o + 8 * n);
  L.cbk = o; o = al256(o + 8 * ((n + 31) / 32 + 2));
  L.lf_lo = o; o = al256(o + 16 * L.nleaf);
  L.lf_len = o; o = al256(o + 16 * L.nleaf);
  L.lf_sum = o; o = al256(o + 8 * L.nleaf);
  L.rows = o; o = al256(o + 4 * L.kk);
  L.reps = o; o = al256(o + 8 * L.kk);
  L.rsgn = o; o = al256(o + 4 * L.kk);
  L.ag = o; o = al256(o + 8 * kG * n);
  L.cbuf = o; o = al256(o + sizeof(Cand) * cap);
  L.que = o; o = al256(o + 2 * sizeof(QEnt) * fc_qcap(cap));  // staged-row survivors, ping-pong
  L.hset = o; o = al256(o + 8 * L.hsz);
  L.rem = o; o = al256(o + 4 * rr);
  L.sav = o; o = al256(o + 4 * rr);
  L.pick = o; o = al256(o + 4 * rr);
  L.coin = o; o = al256(o + 4 * rr);
  L.ibuf = o; o = al256(o + 4 * (n > L.kk ? n : L.kk));
  {
    int64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    L.srt = o; o = al256(o + 16 * n2);  // bucket sort: (level, b0, j) per position
  }
  // sparse engine: one dense row scratch (kept zero between uses), |s| top list
  L.rowtmp = o; o = al256(o + (ktop > 0 ? 8 * n : 0));
  L.top = o; o = al256(o + 4 * ktop);
  // column-indexed filter: per-column list heads (kept -1 between uses), entries
  L.fhead = o; o = al256(o + (fecap > 0 ? 4 * n : 0));
  L.fent = o; o = al256(o + sizeof(FEnt) * fecap);
  L.total = o;
  return L;
}

// Block-uniform engine context, kept in shared memory (not registers): the
// kernel is one long state machine, so anything live across all phases must
// not occupy registers the hot loops need.
struct Ctx {
  int64_t m, n, nlev, kk, cap;
  const double *At, *Ar, *b;
  const int64_t *cptr;
  const int32_t *crow;
  const double *cval;
  int csc;
  int sparse, ktop;           // sparse engine (see KArgs)
  const int64_t *rptr;
  const int32_t *rcol;
  const double *rval;
  double *rowtmp;             // n doubles, zero between uses
  int32_t *top;               // ktop rows by (|s| desc, index asc)
  int32_t *fhead;             // column-indexed filter: list head per column (-1 between uses)
  FEnt *fent;                 // ... entries
  int64_t fecap;              // ... capacity (0: off)
  double *cr, *ur;
  int32_t *cidx, *uidx;
  double *dbuf, *pbuf, *cbk;
  int64_t *lf_lo, *lf_len;
  double *lf_sum;
  int nleaf_m, nleaf_n, tab;
  int32_t *rows, *rsgn;
  double *reps, *ag;
  uint32_t off_lv, off_scr;
  Cand *cbuf;
  QEnt *que;
  uint64_t *hset;
  int32_t *rem, *sav, *pick, *coin, *ibuf;
  unsigned char *srt;
  int32_t *status;
  amvm_params prm;
  // operator bank (controller.py:71-85) and counters: thread 0 owns these
  double w[4], sc[4];
  int64_t seg[4], life[4], bit;
  int64_t mv_ref, mv_raw;
  int64_t pc[16];
};

#define AMVM_LOCALS                                                                        \
  [[maybe_unused]] const int64_t m = sh->c.m, n = sh->c.n, nlev = sh->c.nlev;             \
  [[maybe_unused]] const int64_t kk = sh->c.kk, cap = sh->c.cap;                          \
  [[maybe_unused]] const double *const At = sh->c.At;                                     \
  [[maybe_unused]] const double *const Ar = sh->c.Ar;                                     \
  [[maybe_unused]] const double *const b = sh->c.b;                                       \
  [[maybe_unused]] double *const lv = (double *)(amvm_dyn_smem + sh->c.off_lv);            \
  [[maybe_unused]] double *const cr = sh->c.cr;                                           \
  [[maybe_unused]] double *const ur = sh->c.ur;                                           \
  [[maybe_unused]] int32_t *const cidx = sh->c.cidx;                                      \
  [[maybe_unused]] int32_t *const uidx = sh->c.uidx;                                      \
  [[maybe_unused]] double *const dbuf = sh->c.dbuf;                                       \
  [[maybe_unused]] double *const pbuf = sh->c.pbuf;                                       \
  [[maybe_unused]] double *const cbk = sh->c.cbk;                                         \
  [[maybe_unused]] int64_t *const lf_lo = sh->c.lf_lo;                                    \
  [[maybe_unused]] int64_t *const lf_len = sh->c.lf_len;                                  \
  [[maybe_unused]] double *const lf_sum = sh->c.lf_sum;                                   \
  [[maybe_unused]] const int nleaf_m = sh->c.nleaf_m, nleaf_n = sh->c.nleaf_n;            \
  [[maybe_unused]] const int tab = sh->c.tab;                                             \
  [[maybe_unused]] int32_t *const rows = sh->c.rows;                                      \
  [[maybe_unused]] int32_t *const rsgn = sh->c.rsgn;                                      \
  [[maybe_unused]] double *const reps = sh->c.reps;                                       \
  [[maybe_unused]] double *const ag = sh->c.ag;                                           \
  [[maybe_unused]] unsigned char *const scr = amvm_dyn_smem + sh->c.off_scr;               \
  [[maybe_unused]] Cand *const cbuf = sh->c.cbuf;                                         \
  [[maybe_unused]] QEnt *const que = sh->c.que;                                           \
  [[maybe_unused]] uint64_t *const hset = sh->c.hset;                                     \
  [[maybe_unused]] int32_t *const rem = sh->c.rem;                                        \
  [[maybe_unused]] int32_t *const sav = sh->c.sav;                                        \
  [[maybe_unused]] int32_t *const pick = sh->c.pick;                                      \
  [[maybe_unused]] int32_t *const coin = sh->c.coin;                                      \
  [[maybe_unused]] int32_t *const ibuf = sh->c.ibuf;                                      \
  [[maybe_unused]] unsigned char *const srt = sh->c.srt;                                   \
  [[maybe_unused]] int32_t *const status = sh->c.status;                                  \
  [[maybe_unused]] const amvm_params *const prm = &sh->c.prm;

template <int NT>
struct Shared {
  static constexpr int NW = NT / 32;
  double red[NW][4];  // best_swap per-warp winners
  double red2[2][NW];
  int red2i[2][NW];
  double redS[NW];
  double bc_d[8];
  int bc_i[16];
  int wcnt[NW];
  unsigned int hist[256];
  int counter;
  int qcount;
  int gnext;
  int qnext;
  int srow[kS];
  int wk[2][NT / 32 * kCWv<NT>];  // one_opt window: level index per column
  unsigned sflag[2][NT / 32];   // one_opt window: first-screen survivors per warp
  int wsum[2][NT / 32];         // one_opt window: valid candidates per warp
  unsigned rejw[2][2][NT / 32]; // one_opt batch: second-screen rejections per warp
  uint64_t skey[NT];
  int sidx[NT];
  int64_t task_inst, task_chunk;  // k_solve: the task being run (kept out of registers)
  double *ic;                      // this instance's impact cache (null: no caching)
  int32_t *iv;                     // ... and its valid flag
  int nfilter_rows, srt_rows_sorted;  // select_rows result (rows[] count, ordered by |s| desc)
  int task_live, task_skip;
  int ntop;                       // sparse engine: rows in the |s| top list
  int fc_pairs;                   // find_candidates: lane-per-pair enumeration (small level buckets)
  int fc_maxb;                    // find_candidates: largest level bucket
  uint64_t swap_best;             // best_swap: smallest complete t' so far (bit pattern)
  int vrow[32];                   // best_swap: rows that recently proved a swap non-improving
  int vins;                       // ... insertion counter (ring of 32)
  int spl[NT / 32 * 4];           // sparse one_opt window: chosen level per column (-1: none)
  int spc[NT / 32 * 4];           // ... and the window's columns
  double spt[NT / 32 * 4];        // ... and its objective
  int64_t pw_a[48], pw_b[48];     // pairwise-sum tree walk stacks (thread 0 only)
  int pw_s[48];
  double pw_res;
  Pcg rng;
  Ctx c;
};

__device__ __forceinline__ uint64_t abs_key(double x) { return (uint64_t)__double_as_longlong(fabs(x)); }

// SP: the sparse engine (A as CSC + CSR only), a separate instantiation so
// the dense hot loops keep their registers.
template <int NT, bool SP = false>
struct Engine {
  static constexpr int NW = NT / 32;
  static constexpr int kCW = kCWv<NT>, kTJ = kTJv<NT>, kTC = NT;
  Shared<NT> *sh;
  int tid, lane, warp;
  // replicated block-uniform scalars: every thread evolves identical copies
  double cobj, uobj, bobj;
  int ccnt, ucnt, bcnt;

  // ------------------------------------------------------------ utilities
  __device__ void fail(int code) {
    AMVM_LOCALS
    if (tid == 0) atomicCAS(status, 0, code);
  }

  __device__ double block_max_own(double mx) {
    AMVM_LOCALS
    mx = warp_max(mx);
    if (lane == 0) sh->redS[warp] = mx;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) t = fmax(t, sh->redS[k]);
    __syncthreads();
    return t;
  }

  __device__ double own_max_abs() {
    AMVM_LOCALS
    double mx = 0.0;
    for (int64_t i = tid; i < m; i += NT) mx = fmax(mx, fabs(cr[i]));
    return block_max_own(mx);
  }

  // numpy pairwise sum of get(0..len-1) over the cached leaf tree.
  template <class F>
  __device__ double block_pairwise(F &&get, int64_t len, int64_t *lo, int64_t *ln, int nleaf) {
    AMVM_LOCALS
    for (int k = tid; k < nleaf; k += NT) lf_sum[k] = pw_leaf(get, lo[k], ln[k]);
    __syncthreads();
    if (tid == 0) sh->pw_res = pw_combine(len, lf_sum, sh->pw_a, sh->pw_s, (double *)sh->pw_b);
    __syncthreads();
    return sh->pw_res;  // rewritten only after the next call's first barrier
  }

  // Solution.refresh (core.py:173-177): numpy A @ x - b in the OpenBLAS order.
  __device__ void refresh() {
    AMVM_LOCALS
#ifndef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
    if (tid == 0) sh->c.pc[15] += 1;
#endif
#endif
    __syncthreads();  // publish cidx
    if (m == 1 && !SP) {
      if (warp == 0) {
        double y = warp_ddot_skx([&](int64_t j) { return At[j]; },
                                 [&](int64_t j) { return lv[cidx[j]]; }, n, lane);
        if (lane == 0) cr[0] = dsub(y, b[0]);
      }
    } else if (SP) {
      for (int64_t i = tid; i < m; i += NT) {
        const int64_t e0 = __ldg(sh->c.rptr + i), e1 = __ldg(sh->c.rptr + i + 1);
        double y = gemv_row_sparse(sh->c.rcol + e0, sh->c.rval + e0, e1 - e0,
                                   [&](int64_t j) { return lv[cidx[j]]; }, n, gemv_kind(i, m));
        cr[i] = dsub(y, b[i]);
      }
    } else {
      for (int64_t i = tid; i < m; i += NT) {
        double y = gemv_row([&](int64_t j) { return At[j * m + i]; },
                            [&](int64_t j) { return lv[cidx[j]]; }, n, gemv_kind(i, m));
        cr[i] = dsub(y, b[i]);
      }
    }
    __syncthreads();
    cobj = own_max_abs();
    ccnt = 0;
  }

  __device__ void bump_known(double t) {
    AMVM_LOCALS
    ccnt += 1;
    if (ccnt >= prm->refresh_period) refresh();
    else cobj = t;
  }

  // apply_shift (core.py:208-225) when the new objective is not known yet.
  __device__ bool apply_shift_reduce(int64_t j, int nl) {
    AMVM_LOCALS
    const int old = cidx[j];
    if (nl == old) return false;
    const double d = dsub(lv[nl], lv[old]);
    double mx = 0.0;
    if (SP) {  // touched rows only (s + d*0 = s), then the max over all rows
      const int64_t b0 = __ldg(sh->c.cptr + j), b1 = __ldg(sh->c.cptr + j + 1);
      for (int64_t e = b0 + tid; e < b1; e += NT) {
        const int64_t r = __ldg(sh->c.crow + e);
        cr[r] = dadd(cr[r], dmul(d, __ldg(sh->c.cval + e)));
      }
      __syncthreads();
      for (int64_t i = tid; i < m; i += NT) mx = fmax(mx, fabs(cr[i]));
    } else {
      const double *col = At + j * m;
      for (int64_t i = tid; i < m; i += NT) {
        double y = dadd(cr[i], dmul(d, __ldg(col + i)));
        cr[i] = y;
        mx = fmax(mx, fabs(y));
      }
    }
    mx = warp_max(mx);
    if (lane == 0) sh->redS[warp] = mx;
    __syncthreads();
    if (tid == 0) cidx[j] = nl;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < NW; ++k) t = fmax(t, sh->redS[k]);
    __syncthreads();
    ccnt += 1;
    if (ccnt >= prm->refresh_period) refresh();
    else cobj = t;
    return true;
  }

  // ------------------------------------------------------------- one_opt
  // Exact max_i |cr_i + d*col_i| for both candidates of one column (CTA-wide).
  // Also returns a row attaining each maximum (the new objective's row if
  // that shift is applied: it becomes a screening row, see one_opt).
  __device__ void exact_pair_max(const double *col, double dm, double dp, double &tm, double &tp, int &im,
                                 int &ip) {
    AMVM_LOCALS
    double mm = 0.0, mp = 0.0;
    int jm = -1, jp = -1;
    for (int64_t i = tid; i < m; i += NT) {
      const double r = cr[i], a = __ldg(col + i);
      const double ym = fabs(dadd(r, dmul(dm, a))), yp = fabs(dadd(r, dmul(dp, a)));
      if (ym > mm || jm < 0) { mm = ym; jm = (int)i; }
      if (yp > mp || jp < 0) { mp = yp; jp = (int)i; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double om = __shfl_xor_sync(AMVM_FULL, mm, o), op = __shfl_xor_sync(AMVM_FULL, mp, o);
      const int oim = __shfl_xor_sync(AMVM_FULL, jm, o), oip = __shfl_xor_sync(AMVM_FULL, jp, o);
      if (om > mm || (om == mm && (unsigned)oim < (unsigned)jm)) { mm = om; jm = oim; }
      if (op > mp || (op == mp && (unsigned)oip < (unsigned)jp)) { mp = op; jp = oip; }
    }
    if (lane == 0) {
      sh->red2[0][warp] = mm;
      sh->red2[1][warp] = mp;
      sh->red2i[0][warp] = jm;
      sh->red2i[1][warp] = jp;
    }
    __syncthreads();
    tm = -1.0;
    tp = -1.0;
    im = ip = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const int km = sh->red2i[0][k], kp = sh->red2i[1][k];
      if (km >= 0 && sh->red2[0][k] > tm) { tm = sh->red2[0][k]; im = km; }
      if (kp >= 0 && sh->red2[1][k] > tp) { tp = sh->red2[1][k]; ip = kp; }
    }
    if (tm < 0.0) tm = 0.0;
    if (tp < 0.0) tp = 0.0;
    __syncthreads();
  }

  // Screening rows for one_opt: each thread's largest |s|, then the kS/NW
  // largest of each warp's (register sorts, no block-wide sort), the overall
  // largest first.  ANY row subset gives an exact
  // rejection test; large |s| rows reject almost every non-improving shift.
  // one_opt reads the screening rows straight from the row-major copy Ar.
  __device__ void select_screen() {
    AMVM_LOCALS
    uint64_t best = 0;
    int brow = 0;
    for (int64_t i = tid; i < m; i += NT) {
      const uint64_t key = abs_key(cr[i]);
      if (key > best || i == tid) { best = key; brow = (int)i; }
    }
    // each warp sorts its 32 maxima in registers; the screening rows are the
    // top kS/NW of every warp (no block-wide sort), with the overall largest
    // moved to srow[0] (it follows the objective)
    uint64_t key = tid < m ? best : 0;
    int row = tid < m ? brow : 0;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const uint64_t ok = __shfl_xor_sync(AMVM_FULL, key, jj);
        const int orow = __shfl_xor_sync(AMVM_FULL, row, jj);
        const bool lower = (lane & jj) == 0, desc = (lane & k) == 0;
        if ((lower == desc) ? ok > key : ok < key) { key = ok; row = orow; }
      }
    }
    sh->skey[tid] = key;
    sh->sidx[tid] = row;  // (each thread's second-screen row: any permutation of the maxima)
    __syncthreads();
    if (warp == 0) {
      constexpr int per = kS / NW;  // rows taken from each warp's sorted list
      static_assert(kS % NW == 0 && per >= 1, "screening rows split evenly over the warps");
      int r = sh->sidx[(lane / per) * 32 + lane % per];
      // the overall largest: the best warp head
      uint64_t hk = lane < NW ? sh->skey[lane * 32] : 0;
      int hw = lane < NW ? lane : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t k2 = __shfl_xor_sync(AMVM_FULL, hk, o);
        const int w2 = __shfl_xor_sync(AMVM_FULL, hw, o);
        if (k2 > hk || (k2 == hk && w2 < hw)) { hk = k2; hw = w2; }
      }
      // swap slots 0 and hw * per (both hold warp heads)
      const int r0 = __shfl_sync(AMVM_FULL, r, 0), rh = __shfl_sync(AMVM_FULL, r, hw * per);
      if (lane == 0) r = rh;
      else if (lane == hw * per) r = r0;
      sh->srow[lane] = r;
    }
    __syncthreads();
  }

  // one_opt, localsearch.py:59-88, exact and in the reference's order, with a
  // row screen: a shift can only improve if EVERY row stays below t, so one
  // screening row with |s_r + d*a_rj| >= t proves the candidate does not
  // improve.  A window is NW*kCW columns: each warp screens kCW of them against
  // the kS largest-|s| rows (lane = row, all loads issued together, one
  // barrier per window); the flagged columns then get a second screen in
  // batches of kB (each thread one of the CTA's per-thread-max rows, one
  // barrier per batch); survivors are scored over all m rows exactly, in
  // ascending order, and the first that strictly improves is applied (first
  // improvement); scanning resumes after it.  Window/batch buffers alternate
  // by parity, so a buffer is rewritten only after every thread has passed
  // the barrier that follows its last read.
  // one_opt on the sparse engine: every candidate scored exactly from its
  // column's nonzeros plus the largest |s| among untouched rows (the first
  // row of the |s| top list outside the column).  Screen (exact): a column
  // that does not touch the argmax row r* (|s_r*| = t) keeps |s_r*| = t in
  // both shifted residuals, so it cannot improve -- only the columns of r*'s
  // CSR row are scored, NW*kSpCW per window in ascending order, the lowest
  // improving one is applied (the reference's sequential first improvement)
  // and scanning resumes after it with the new r*.  The reference-equivalent
  // move count still covers every column passed.
  static constexpr int kSpCW = 4;
  // candidate moves of the columns [j0, j1): 2 per column minus the grid ends
  __device__ int64_t sp_count_moves(int64_t j0, int64_t j1) {
    AMVM_LOCALS
    int64_t c = 0;
    for (int64_t j = j0 + tid; j < j1; j += NT) {
      const int k = cidx[j];
      c += (k > 0) + (k + 1 < nlev);
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(AMVM_FULL, c, o);
    __syncthreads();
    if (lane == 0) sh->red2i[0][warp] = (int)c;
    __syncthreads();
    int64_t tot = 0;
    for (int w = 0; w < NW; ++w) tot += sh->red2i[0][w];
    __syncthreads();
    return tot;
  }

  __device__ void one_opt_sparse() {
    AMVM_LOCALS
    constexpr int WS = NW * kSpCW;
    const int64_t *rp = sh->c.rptr;
    const int32_t *rw = sh->c.rcol;
    for (int sw = 0; sw < prm->one_opt_max_sweeps; ++sw) {
      bool changed = false;
      int64_t p = 0;
      sp_select_top();
      while (p < n) {
        const double t = cobj;
        // the window's columns: the next WS columns >= p of the argmax row (or
        // of all columns if the top row is not at t)
        if (tid == 0) {
          const int32_t rs = sh->c.top[0];
          int64_t e0 = -1, e1 = -1;
          if (fabs(cr[rs]) == t) {
            e1 = __ldg(rp + rs + 1);
            int64_t lo = __ldg(rp + rs), hi = e1;
            while (lo < hi) {
              const int64_t mid = (lo + hi) >> 1;
              if (__ldg(rw + mid) < p) lo = mid + 1;
              else hi = mid;
            }
            e0 = lo;
          }
          int w = 0;
          if (e0 >= 0) {
            for (; w < WS && e0 + w < e1; ++w) sh->spc[w] = __ldg(rw + e0 + w);
            sh->bc_i[8] = e0 + w < e1;  // more screen-row columns after this window
          } else {
            for (; w < WS && p + w < n; ++w) sh->spc[w] = (int)(p + w);
            sh->bc_i[8] = p + w < n;
          }
          sh->bc_i[9] = w;
        }
        __syncthreads();
        const int wc = sh->bc_i[9];
        const bool more = sh->bc_i[8] != 0;
#pragma unroll 1
        for (int c = 0; c < kSpCW; ++c) {
          const int slotw = warp * kSpCW + c;
          int lvl = -1;
          double bt = t;
          if (slotw < wc) {
            const int64_t j = sh->spc[slotw];
            const int k = cidx[j];
            const bool hm = k > 0, hp = k + 1 < nlev;
            const double lk = lv[k];
            const double dm = hm ? dsub(lv[k - 1], lk) : 0.0;
            const double dp = hp ? dsub(lv[k + 1], lk) : 0.0;
            const int64_t b0 = __ldg(sh->c.cptr + j), b1 = __ldg(sh->c.cptr + j + 1);
            double mm = 0.0, mp = 0.0;
            for (int64_t e = b0 + lane; e < b1; e += 32) {
              const double rv = cr[__ldg(sh->c.crow + e)], a = __ldg(sh->c.cval + e);
              mm = fmax(mm, fabs(dadd(rv, dmul(dm, a))));
              mp = fmax(mp, fabs(dadd(rv, dmul(dp, a))));
            }
            mm = warp_max(mm);
            mp = warp_max(mp);
            const double u = sp_untouched_max(j, -1);
            const double tm = fmax(mm, u), tp = fmax(mp, u);
            if (hm && tm < bt) { bt = tm; lvl = k - 1; }
            if (hp && tp < bt) { bt = tp; lvl = k + 1; }
          }
          if (lane == 0) {
            sh->spl[slotw] = lvl;
            sh->spt[slotw] = bt;
          }
        }
        __syncthreads();
        int applied = -1;
        for (int w = 0; w < wc; ++w)
          if (sh->spl[w] >= 0) { applied = w; break; }
        // every column passed up to the applied one (or through the window /
        // to the end when nothing improves) counts as scored
        const int64_t end = applied >= 0 ? (int64_t)sh->spc[applied] + 1
                                         : (more ? (int64_t)sh->spc[wc - 1] + 1 : n);
        const int64_t cnt = sp_count_moves(p, end);
        if (tid == 0) {
          sh->c.mv_ref += cnt;
          sh->c.mv_raw += cnt;
        }
        if (applied >= 0) {
          const int64_t j = sh->spc[applied];
          const int lvl = sh->spl[applied];
          const double bt = sh->spt[applied];
          const double d = dsub(lv[lvl], lv[cidx[j]]);
          const int64_t b0 = __ldg(sh->c.cptr + j), b1 = __ldg(sh->c.cptr + j + 1);
          __syncthreads();  // everyone has read the window's results and cidx[j]
          for (int64_t e = b0 + tid; e < b1; e += NT) {
            const int64_t r = __ldg(sh->c.crow + e);
            cr[r] = dadd(cr[r], dmul(d, __ldg(sh->c.cval + e)));
          }
          if (tid == 0) cidx[j] = lvl;
          __syncthreads();
          bump_known(bt);
          sp_select_top();  // the residual changed
          changed = true;
        } else {
          __syncthreads();
        }
        p = end;
      }
      if (!changed) break;
    }
  }

  __device__ void one_opt() {
    AMVM_LOCALS
    if constexpr (SP) {
      one_opt_sparse();
      return;
    }
    constexpr int WS = NW * kCW;
    __syncthreads();
    select_screen();
    int wpar = 0, bpar = 0;
    for (int sw = 0; sw < prm->one_opt_max_sweeps; ++sw) {
      bool changed = false;
      int64_t p = 0;
      while (p < n) {
        const int wc = (int)(n - p < WS ? n - p : WS);
        const int srow_l = sh->srow[lane];  // this lane's screening row (row 0 follows the objective)
        const double *arow = Ar + (int64_t)srow_l * n;
        const double rs = cr[srow_l];
        const double t = cobj;
        const int c0 = warp * kCW;
        const int64_t jb = p + c0;
        const int kl = (lane < kCW && c0 + lane < wc) ? cidx[jb + lane] : 0;
        double a[kCW];
#pragma unroll
        for (int c = 0; c < kCW; ++c) a[c] = c0 + c < wc ? __ldg(arow + jb + c) : 0.0;
        unsigned mine = 0u;  // bit c: column c0+c has a candidate no screening row rejects
#pragma unroll
        for (int c = 0; c < kCW; ++c) {
          const int k = __shfl_sync(AMVM_FULL, kl, c);
          if (c0 + c < wc) {
            const double lk = lv[k];
            const bool hm = k > 0, hp = k + 1 < nlev;
            const double dm = hm ? dsub(lv[k - 1], lk) : 0.0;
            const double dp = hp ? dsub(lv[k + 1], lk) : 0.0;
            const bool rm = !hm || fabs(dadd(rs, dmul(dm, a[c]))) >= t;
            const bool rp = !hp || fabs(dadd(rs, dmul(dp, a[c]))) >= t;
            if (!__any_sync(AMVM_FULL, rm) || !__any_sync(AMVM_FULL, rp)) mine |= 1u << c;
          }
        }
        // valid candidates per column (reference-equivalent move count)
        const int v = (lane < kCW && c0 + lane < wc) ? (kl > 0) + (kl + 1 < nlev) : 0;
        const int vsum = __reduce_add_sync(AMVM_FULL, v);
        if (lane < kCW) sh->wk[wpar][c0 + lane] = kl;
        if (lane == 0) {
          sh->sflag[wpar][warp] = mine;
          sh->wsum[wpar][warp] = vsum;
        }
        __syncthreads();
        // first-screen survivors as a 128-bit mask, popped in ascending order
        static_assert(WS <= 128, "one_opt window mask is two 64-bit words");
        uint64_t f0 = 0, f1 = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint64_t bits = (uint64_t)sh->sflag[wpar][w] << ((w * kCW) % 64);
          if ((w * kCW) / 64 == 0) f0 |= bits;
          else f1 |= bits;
        }
        int applied = -1;
        const int rA = sh->sidx[tid];
        for (;;) {
          int cols[kB];
          int nb = 0;
#pragma unroll
          for (int e = 0; e < kB; ++e) {
            cols[e] = 0;
            if (f0) {
              cols[e] = __ffsll((long long)f0) - 1;
              f0 &= f0 - 1;
              nb = e + 1;
            } else if (f1) {
              cols[e] = 64 + __ffsll((long long)f1) - 1;
              f1 &= f1 - 1;
              nb = e + 1;
            }
          }
          if (nb == 0) break;
          // second screen: one load per thread per flagged column, all issued
          // together, then one barrier for the batch
          const double rr = cr[rA];
          double av[kB];
#pragma unroll
          for (int e = 0; e < kB; ++e) av[e] = e < nb ? __ldg(At + (p + cols[e]) * m + rA) : 0.0;
          unsigned em = 0u, ep = 0u;
#pragma unroll
          for (int e = 0; e < kB; ++e) {
            if (e < nb) {
              const int k = sh->wk[wpar][cols[e]];
              const double lk = lv[k];
              const bool hm = k > 0, hp = k + 1 < nlev;
              const double dm = hm ? dsub(lv[k - 1], lk) : 0.0;
              const double dp = hp ? dsub(lv[k + 1], lk) : 0.0;
              if (!hm || fabs(dadd(rr, dmul(dm, av[e]))) >= t) em |= 1u << e;
              if (!hp || fabs(dadd(rr, dmul(dp, av[e]))) >= t) ep |= 1u << e;
            }
          }
          em = __reduce_or_sync(AMVM_FULL, em);
          ep = __reduce_or_sync(AMVM_FULL, ep);
          if (lane == 0) {
            sh->rejw[bpar][0][warp] = em;
            sh->rejw[bpar][1][warp] = ep;
          }
          __syncthreads();
          unsigned rjm = 0u, rjp = 0u;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            rjm |= sh->rejw[bpar][0][w];
            rjp |= sh->rejw[bpar][1][w];
          }
          bpar ^= 1;
          for (int e = 0; e < nb; ++e) {
            if ((rjm >> e) & (rjp >> e) & 1u) continue;
            const int w = cols[e];
            const int64_t j = p + w;
            const int k = sh->wk[wpar][w];
            const double lk = lv[k];
            const double dm = k > 0 ? dsub(lv[k - 1], lk) : 0.0;
            const double dp = k + 1 < nlev ? dsub(lv[k + 1], lk) : 0.0;
            double tm, tpv;
#ifndef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
            if (tid == 0) sh->c.pc[11] += 1;
#endif
#endif
            // raw count: candidates actually scored over all m rows
            if (tid == 0) sh->c.mv_raw += (k > 0) + (k + 1 < nlev);
            int rm, rp;
            exact_pair_max(At + j * m, dm, dp, tm, tpv, rm, rp);
            int lvl = -1;
            double bt = cobj;
            if (k > 0 && tm < bt) { bt = tm; lvl = k - 1; }
            if (k + 1 < nlev && tpv < bt) { bt = tpv; lvl = k + 1; }
            if (lvl >= 0) {
              applied = w;
#ifndef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
              if (tid == 0) sh->c.pc[12] += 1;
#endif
#endif
              const double d = dsub(lv[lvl], lk);
              const double *col = At + j * m;
              for (int64_t i = tid; i < m; i += NT) cr[i] = dadd(cr[i], dmul(d, __ldg(col + i)));
              __syncthreads();  // all reads of cidx[j] done; residual published
              if (tid == 0) {
                cidx[j] = lvl;
                // the row attaining the new objective leads both screens from
                // now on (any row set is an exact screen; the current maximum
                // row is the one that rejects most)
                const int top = lvl == k - 1 ? rm : rp;
                sh->srow[0] = top;
                sh->sidx[0] = top;
              }
              bump_known(bt);
              __syncthreads();
              break;
            }
          }
          if (applied >= 0) break;
        }
        if (tid == 0) {
          int64_t cnt = 0;
          if (applied >= 0) {
            for (int c = 0; c <= applied; ++c) {
              const int k = sh->wk[wpar][c];
              cnt += (k > 0) + (k + 1 < nlev);
            }
          } else {
            for (int w = 0; w < NW; ++w) cnt += sh->wsum[wpar][w];
          }
          sh->c.mv_ref += cnt;
#ifndef AMVM_FC_PROFILE
          sh->c.pc[13] += 1;
#endif
        }
        wpar ^= 1;
        if (applied >= 0) {
          changed = true;
          p = p + applied + 1;
        } else {
          p += wc;
        }
      }
      if (!changed) break;
    }
  }

  // ------------------------------------------------------ find_candidates
  // Top-k_eps rows of |s| by (value desc, index asc) (localsearch.py:140):
  // 8-pass radix select of the k-th key, then ties resolved by index.  Only
  // the SET matters (the filter is an AND over rows); it is then ordered by
  // key so the tightest rows reject first.  Rows with s = 0 are dropped
  // (localsearch.py:151).  Returns the number of filter rows.
  // The kth largest |cr| key (kth >= 1): T = its bit pattern, need = how
  // many keys equal to T belong to the top kth.  MSD radix select, 8-bit
  // digits.  With a scratch `ck` (ccap keys), once the keys sharing the
  // chosen prefix fit in it they are compacted there and the remaining
  // passes histogram only them instead of rescanning all m rows.
  __device__ void radix_kth(int64_t kth, uint64_t &T, int64_t &need, uint64_t *ck = nullptr, int ccap = 0) {
    AMVM_LOCALS
    uint64_t prefix = 0;
    int64_t remaining = kth;
    int nc = -1;  // keys in ck (-1: not compacted, scan cr)
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int e = tid; e < 256; e += NT) sh->hist[e] = 0;
      __syncthreads();
      const uint64_t hm = shift == 56 ? 0ull : (~0ull << (shift + 8));
      // warp-aggregated histogram: |s| values of one instance share their
      // high digits, so plain per-thread atomics would serialise on a bin
      const int64_t len = nc >= 0 ? nc : m;
      for (int64_t i0 = (int64_t)warp * 32; i0 < len; i0 += NT) {
        const int64_t i = i0 + lane;
        const uint64_t key = i < len ? (nc >= 0 ? ck[i] : abs_key(cr[i])) : 0ull;
        const bool in = i < len && (key & hm) == prefix;
        const unsigned act = __ballot_sync(AMVM_FULL, in);
        if (in) {
          const unsigned bin = (unsigned)(key >> shift) & 255u;
          const unsigned peers = __match_any_sync(act, bin);
          if (lane == __ffs(peers) - 1) atomicAdd(&sh->hist[bin], (unsigned)__popc(peers));
        }
      }
      __syncthreads();
      if (warp == 0) {
        // the digit d where the count of keys with a larger digit first
        // reaches `remaining`, scanning from digit 255 down: lane l holds
        // digits 255-8l .. 248-8l; shuffle-scan of the lane totals
        unsigned h[8], tot = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          h[e] = sh->hist[255 - 8 * lane - e];
          tot += h[e];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(AMVM_FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const int64_t before = (int64_t)(incl - tot);  // keys in the lanes above (larger digits)
        const bool here = before < remaining && before + (int64_t)tot >= remaining;
        const unsigned who = __ballot_sync(AMVM_FULL, here);
        if (lane == __ffs(who) - 1) {
          int64_t cum = before;
          int e = 0;
          for (; e < 8; ++e) {
            if (cum + (int64_t)h[e] >= remaining) break;
            cum += h[e];
          }
          sh->bc_i[0] = 255 - 8 * lane - e;
          sh->bc_i[1] = (int)cum;
          sh->bc_i[3] = (int)h[e];  // keys sharing the new prefix
          sh->bc_i[5] = (int64_t)h[e] == remaining - cum;  // ... and all of them are in the top kth
        }
        if (lane == 0) sh->bc_i[2] = 0;
      }
      __syncthreads();
      prefix |= (uint64_t)sh->bc_i[0] << shift;
      remaining -= sh->bc_i[1];
      if (sh->bc_i[5] && prefix > 0) {
        // every key with this prefix is needed: "key > prefix - 1" selects
        // exactly the top kth (no ties to resolve), so the digits below are moot
        T = prefix - 1;
        need = 0;
        __syncthreads();  // bc_i is rewritten by the next call
        return;
      }
      if (ck && nc < 0 && shift > 0 && sh->bc_i[3] <= ccap) {  // block-uniform
        const uint64_t hm2 = ~0ull << shift;
        for (int64_t i0 = (int64_t)warp * 32; i0 < m; i0 += NT) {
          const int64_t i = i0 + lane;
          const uint64_t key = i < m ? abs_key(cr[i]) : 0ull;
          const bool in = i < m && (key & hm2) == prefix;
          const unsigned bal = __ballot_sync(AMVM_FULL, in);
          if (!bal) continue;
          int base = 0;
          if (lane == 0) base = atomicAdd(&sh->bc_i[2], __popc(bal));
          base = __shfl_sync(AMVM_FULL, base, 0);
          if (in) ck[base + __popc(bal & ((1u << lane) - 1u))] = key;
        }
        __syncthreads();
        nc = sh->bc_i[3];
      }
    }
    T = prefix;
    need = remaining;
  }

  // ---------------------------------------------- sparse engine helpers
  // A[r, col] from the CSR row r (columns ascending): binary search, 0 if absent
  __device__ double sp_row_at(int64_t r, int64_t col) {
    const int64_t b0 = __ldg(sh->c.rptr + r), b1 = __ldg(sh->c.rptr + r + 1);
    int64_t lo = b0, hi = b1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(sh->c.rcol + mid) < col) lo = mid + 1;
      else hi = mid;
    }
    return (lo < b1 && __ldg(sh->c.rcol + lo) == col) ? __ldg(sh->c.rval + lo) : 0.0;
  }
  // position of row r in the CSC column col (rows ascending), -1 if absent
  __device__ int64_t sp_col_find(int64_t col, int64_t r) {
    const int64_t b0 = __ldg(sh->c.cptr + col), b1 = __ldg(sh->c.cptr + col + 1);
    int64_t lo = b0, hi = b1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(sh->c.crow + mid) < r) lo = mid + 1;
      else hi = mid;
    }
    return (lo < b1 && __ldg(sh->c.crow + lo) == r) ? lo : -1;
  }
  __device__ double sp_col_at(int64_t col, int64_t r) {
    const int64_t e = sp_col_find(col, r);
    return e >= 0 ? __ldg(sh->c.cval + e) : 0.0;
  }
  // rowtmp[c] = A[r, c] over row r's nonzeros, or back to 0 (block-wide;
  // the caller synchronises)
  __device__ void sp_row_scatter(int64_t r, bool clear) {
    AMVM_LOCALS
    double *rt = sh->c.rowtmp;
    const int64_t b0 = __ldg(sh->c.rptr + r), b1 = __ldg(sh->c.rptr + r + 1);
    for (int64_t e = b0 + tid; e < b1; e += NT) rt[__ldg(sh->c.rcol + e)] = clear ? 0.0 : __ldg(sh->c.rval + e);
  }
  // the ktop rows of largest |cr| ordered by (|s| desc, index asc) into top[]
  // (all m rows when ktop >= m): bounds every row outside a column (or a
  // column pair) by the first top row the column does not touch
  __device__ void sp_select_top() {
    AMVM_LOCALS
    const int64_t K = sh->c.ktop < m ? sh->c.ktop : m;
    int32_t *top = sh->c.top;
    __syncthreads();
    if (tid == 0) sh->counter = 0;
    __syncthreads();
    uint64_t T = 0;
    int64_t need = 0;
    if (K < m) radix_kth(K, T, need);
    for (int64_t i = tid; i < m; i += NT) {
      const uint64_t key = abs_key(cr[i]);
      if (K >= m || key > T) top[atomicAdd(&sh->counter, 1)] = (int32_t)i;
    }
    __syncthreads();
    int cnt = sh->counter;
    __syncthreads();
    if (K < m && need > 0) {  // rows with key == T, lowest indices first
      int64_t base = 0;
      for (int64_t c0 = 0; c0 < m && base < need; c0 += NT) {
        const int64_t i = c0 + tid;
        const bool f = i < m && abs_key(cr[i]) == T;
        const unsigned bal = __ballot_sync(AMVM_FULL, f);
        if (lane == 0) sh->wcnt[warp] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int k = 0; k < NW; ++k) {
          if (k < warp) before += sh->wcnt[k];
          tot += sh->wcnt[k];
        }
        const int64_t pos = base + before + __popc(bal & ((1u << lane) - 1u));
        if (f && pos < need) top[cnt + pos] = (int32_t)i;
        base += tot;
        __syncthreads();
      }
      cnt += (int)need;
    }
    // rank sort by (key desc, index asc) through ibuf
    for (int q = tid; q < cnt; q += NT) ibuf[q] = top[q];
    __syncthreads();
    for (int q = tid; q < cnt; q += NT) {
      const int32_t rq = ibuf[q];
      const uint64_t kq = abs_key(cr[rq]);
      int rank = 0;
      for (int o = 0; o < cnt; ++o) {
        const int32_t ro = ibuf[o];
        const uint64_t ko = abs_key(cr[ro]);
        rank += (ko > kq) || (ko == kq && ro < rq);
      }
      top[rank] = rq;
    }
    if (tid == 0) sh->ntop = cnt;
    __syncthreads();
  }

  // max |s| over the rows a column (or two) does not touch: the first top
  // row outside both (warp-wide; ktop > nnz(i) + nnz(j) guarantees one)
  __device__ double sp_untouched_max(int64_t ci, int64_t cj) {
    AMVM_LOCALS
    const int32_t *top = sh->c.top;
    const int cnt = sh->ntop;
    for (int b0 = 0; b0 < cnt; b0 += 32) {
      const int q = b0 + lane;
      bool free_row = false;
      if (q < cnt) {
        const int64_t r = top[q];
        free_row = sp_col_find(ci, r) < 0 && (cj < 0 || sp_col_find(cj, r) < 0);
      }
      const unsigned bal = __ballot_sync(AMVM_FULL, free_row);
      if (bal) return fabs(cr[top[b0 + __ffs(bal) - 1]]);
    }
    return 0.0;  // every row touched (m <= nnz): nothing outside
  }

  __device__ int select_rows() {
    AMVM_LOCALS
    __syncthreads();
    if (tid == 0) sh->counter = 0;
    __syncthreads();
    uint64_t T = 0;
    int64_t need = 0;
    // (the find_candidates scratch is free until the buckets are built)
    if (kk < m) radix_kth(kk, T, need, (uint64_t *)scr, (int)(scratch_bytes<NT>(nlev, tab) / 8));
    // keys strictly above T (all rows when kk >= m), unordered
    for (int64_t i = tid; i < m; i += NT) {
      uint64_t key = abs_key(cr[i]);
      if (key > T || (kk >= m && key > 0)) {
        int pos = atomicAdd(&sh->counter, 1);
        rows[pos] = (int32_t)i;
      }
    }
    __syncthreads();
    int cnt = sh->counter;
    __syncthreads();
    if (kk < m && T > 0 && need > 0) {
      int64_t base = 0;
      for (int64_t c0 = 0; c0 < m && base < need; c0 += NT) {
        const int64_t i = c0 + tid;
        const bool f = i < m && abs_key(cr[i]) == T;
        const unsigned bal = __ballot_sync(AMVM_FULL, f);
        if (lane == 0) sh->wcnt[warp] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int k = 0; k < NW; ++k) {
          if (k < warp) before += sh->wcnt[k];
          tot += sh->wcnt[k];
        }
        const int64_t pos = base + before + __popc(bal & ((1u << lane) - 1u));
        if (f && pos < need) rows[cnt + pos] = (int32_t)i;
        base += tot;
        __syncthreads();
      }
      cnt += (int)need;
    }
    // order by (|s| desc, index asc) when small (speed only), then eps/sign
    if (cnt <= 2048) {
      for (int q = tid; q < cnt; q += NT) ibuf[q] = rows[q];
      __syncthreads();
      for (int q = tid; q < cnt; q += NT) {
        const int32_t rq = ibuf[q];
        const uint64_t kq = abs_key(cr[rq]);
        int rank = 0;
        for (int o = 0; o < cnt; ++o) {
          const int32_t ro = ibuf[o];
          const uint64_t ko = abs_key(cr[ro]);
          rank += (ko > kq) || (ko == kq && ro < rq);
        }
        rows[rank] = rq;
      }
      __syncthreads();
    }
    for (int q = tid; q < cnt; q += NT) {
      const double s = cr[rows[q]];
      reps[q] = dsub(cobj, fabs(s));
      rsgn[q] = s > 0.0;
    }
    if (tid == 0) {
      sh->nfilter_rows = cnt;
      sh->srt_rows_sorted = cnt <= 2048;
    }
    __syncthreads();
    return cnt;
  }

  __device__ static bool cand_less(const Cand &x, const Cand &y) {
    if (x.d != y.d) return x.d > y.d;
    if (x.i != y.i) return x.i < y.i;
    return x.j < y.j;
  }

  // Block bitonic sort of cbuf[0..cnt) into (-delta, i, j) order.
  __device__ void sort_cands(int cnt) {
    AMVM_LOCALS
    int n2 = 1;
    while (n2 < cnt) n2 <<= 1;
    for (int e = cnt + tid; e < n2; e += NT) cbuf[e] = Cand{0x7fffffff, 0x7fffffff, -1.0};
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int e = tid; e < n2; e += NT) {
          const int x = e ^ jj;
          if (x > e) {
            Cand A = cbuf[e], Bc = cbuf[x];
            const bool up = (e & k) == 0;
            if (up ? cand_less(Bc, A) : cand_less(A, Bc)) {
              cbuf[e] = Bc;
              cbuf[x] = A;
            }
          }
        }
        __syncthreads();
      }
    }
  }

  // find_candidates, localsearch.py:128-169.  Pairs (i, j) with x_i > x_j
  // (levels strictly increase, so idx_i > idx_j) passing the one-sided
  // interval test on every selected row.
  //   * variables are bucketed by level; i runs over level-sorted groups of 32
  //     (one per lane, so a warp's lanes almost always share idx_i) and j over
  //     the level-sorted positions below idx_i, read by broadcast from smem;
  //   * the kG tightest rows are staged per j-tile with the row's sign folded
  //     in (s_k < 0: b = -a), so every staged row is  b_j - b_i < eps_k/delta,
  //     bitwise the reference's test, evaluated branch-free two rows at a
  //     time with a warp-level early exit;
  //   * the few pairs alive after the staged rows go to a queue that the whole
  //     CTA drains against the remaining rows, read from A directly.
  // Returns the count kept (truncated to max_candidates in (-delta, i, j)
  // order); with `always_sort` the kept list is in that order regardless.
  __device__ void fc_append(int32_t i, int32_t j, double delta, bool counting = false) {
    AMVM_LOCALS
    const int pos = atomicAdd(&sh->counter, 1);
    if (!counting && pos < cap) cbuf[pos] = Cand{i, j, delta};
  }

  __device__ bool fc_rest(int64_t i, int32_t j, double delta, int nr, int g) {
    AMVM_LOCALS
    constexpr bool sp = SP;
    for (int q = g; q < nr; ++q) {
      const int64_t rq = rows[q];
      const double da = sp ? dsub(sp_row_at(rq, j), sp_row_at(rq, i))
                           : dsub(__ldg(Ar + rq * n + j), __ldg(Ar + rq * n + i));
      const double bq = ddiv(reps[q], delta);
      if (!(rsgn[q] ? (da < bq) : (da > -bq))) return false;
    }
    return true;
  }

  // fc_rest with the remaining rows split across the warp's lanes (the test
  // is an AND over rows, so the order is free): one pair per warp, ~nr/32
  // bound divisions per lane instead of nr in one thread.  Warp-uniform result.
  __device__ bool fc_rest_warp(int64_t i, int32_t j, double delta, int nr, int g) {
    AMVM_LOCALS
    bool ok = true;
    for (int q0 = g; q0 < nr; q0 += 32) {
      const int q = q0 + lane;
      if (q < nr) {
        const int64_t rq = rows[q];
        const double da = SP ? dsub(sp_row_at(rq, j), sp_row_at(rq, i))
                                       : dsub(__ldg(Ar + rq * n + j), __ldg(Ar + rq * n + i));
        const double bq = ddiv(reps[q], delta);
        ok = rsgn[q] ? (da < bq) : (da > -bq);
      }
      if (!__all_sync(AMVM_FULL, ok)) return false;
    }
    return true;
  }

  // Pairs alive after the staged rows (queued by every tile): each of the
  // next kRowPasses rows tests the whole queue (independent loads from the
  // contiguous row of Ar) and compacts it (one atomic per warp) into the
  // other half of the ping-pong queue; the rare survivors of all passes
  // finish row by row in fc_rest.
  __device__ void fc_drain(int nr, int g, bool counting) {
    AMVM_LOCALS
    constexpr int U = 4;  // queue entries per thread in flight
    const int qcap = (int)fc_qcap(cap);
    int qn = sh->qcount < qcap ? sh->qcount : qcap;
    const int np = nr - g < kRowPasses ? nr - g : kRowPasses;
    // per-pass bound table eps_q / delta(ki, kj) in the (now idle) staged-tile
    // scratch (bucket bounds and the staged-row table stay intact for any
    // later pass of the overflow path)
    const int ll = (int)(nlev * nlev);
    const bool tab2 = ll <= kG * kTJ;
    double *bt2 = (double *)(scr + fc_tb_off(nlev));
    if (tid == 0) sh->qnext = 0;
    __syncthreads();
    QEnt *src = que, *dst = que + qcap;
    int q = g;
    int base = 0;  // sh->qnext only grows: pass survivors land at [base, qnext)
    // kRowPasses passes, and more while the queue stays long (sparse rows
    // keep most pairs alive; batched passes beat per-pair fc_rest there)
    constexpr bool sp = SP;
    // (sparse engine: every remaining row as a pass -- a pass costs the row's
    // nonzeros plus the queue, cheaper than per-pair binary searches)
    // A short queue skips the passes (each pays a bound table and three
    // barriers) and goes straight to the warp-per-pair check below.
    for (; q < nr && qn > (sp ? 0 : kDrainShort) && (q < g + np || qn > kDrainLong || sp); ++q) {
      if (sp) {  // the row, densely, in the (zero) row scratch for this pass
        sp_row_scatter(rows[q], false);
        __syncthreads();
      }
      const double *row = sp ? sh->c.rowtmp : Ar + (int64_t)rows[q] * n;
      const double eq = reps[q];
      const bool pos = rsgn[q] != 0;
      if (tab2) {
        for (int e = tid; e < ll; e += NT) {
          const int ki = e / (int)nlev, kj = e - ki * (int)nlev;
          bt2[e] = ki > kj ? ddiv(eq, dsub(lv[ki], lv[kj])) : 0.0;
        }
        __syncthreads();
      }
      for (int e0 = warp * 32; e0 < qn; e0 += NT * U) {
        QEnt c[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * NT + lane;
          ok[u] = e < qn;
          c[u] = ok[u] ? src[e] : QEnt{0, 0, 1, 0, 0u};
        }
        double aj[U], ai[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // (the sparse row scratch is written in-kernel: no .nc loads)
          aj[u] = sp ? row[c[u].j] : __ldg(row + c[u].j);
          ai[u] = sp ? row[c[u].i] : __ldg(row + c[u].i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double bq = tab2 ? bt2[c[u].ki * (int)nlev + c[u].kj] : ddiv(eq, dsub(lv[c[u].ki], lv[c[u].kj]));
          const double da = dsub(aj[u], ai[u]);
          const bool alive = ok[u] && (pos ? (da < bq) : (da > -bq));
          const unsigned bal = __ballot_sync(AMVM_FULL, alive);
          if (!bal) continue;
          int bse = 0;
          if (lane == 0) bse = atomicAdd(&sh->qnext, __popc(bal));
          bse = __shfl_sync(AMVM_FULL, bse, 0) - base;
          if (alive) dst[bse + __popc(bal & ((1u << lane) - 1u))] = c[u];
        }
      }
      __syncthreads();
      const int tot = sh->qnext;
      if (sp) sp_row_scatter(rows[q], true);  // back to zero (all reads done)
      __syncthreads();  // everyone has read it (and the table) before the next pass
      qn = tot - base;
      base = tot;
      QEnt *t = src; src = dst; dst = t;
    }
#ifdef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
    if (tid == 0) sh->c.pc[12] += qn;
#endif
#endif
    for (int e = warp; e < qn; e += NW) {  // the last survivors: one pair per warp
      const QEnt c = src[e];
      const double delta = dsub(lv[c.ki], lv[c.kj]);
      if (fc_rest_warp(c.i, c.j, delta, nr, q) && lane == 0) fc_append(c.i, c.j, delta, counting);
    }
    __syncthreads();
    if (tid == 0) sh->qcount = 0;
    __syncthreads();
  }

  // One enumeration pass over the staged tiles.  mode FC_ALL collects every
  // survivor; FC_COUNT only counts, FC_CUT collects, the survivors whose key
  // precedes or equals (fD, fI) in the reference order (-delta, i): delta > fD,
  // or delta == fD and i <= fI (the exact overflow path, find_candidates).
  enum { FC_ALL = 0, FC_COUNT = 1, FC_CUT = 2 };
  template <int MODE>
  __device__ void fc_pass(int nr, int g, double fD, int64_t fI) {
    AMVM_LOCALS
    // scratch: [lst, lfl | tb | tl | tj | bt] (fc_scr_off)
    int32_t *lst = (int32_t *)scr;
    double *tb = (double *)(scr + fc_tb_off(nlev));
    int32_t *tl = (int32_t *)(tb + kG * kTJ);
    int32_t *tj = tl + kTJ;
    double *bt = (double *)(tj + kTJ);
    int32_t *perm = ibuf;
    const int qcap = (int)fc_qcap(cap);
    constexpr bool filt = MODE != FC_ALL;
    constexpr bool counting = MODE == FC_COUNT;
    // i-groups: 32 consecutive positions of ONE level bucket, so idx_i (and
    // with it every staged row's bound for a given j-bucket) is warp-uniform;
    // within a bucket the lanes' b0 ascend, so their prefixes nest.  The
    // j-buckets are walked through the skip list of non-empty levels.
    const int32_t *nxt = lst + (nlev + 1);
    const int64_t ngrp = (n + 31) / 32 + nlev;
    // few groups (small buckets: C1 has 15 for 16 warps): each group's lower
    // levels are split round-robin into P parts claimed separately, so the
    // warps share the long groups instead of waiting for them
    // (the wide CTA only: single instances; the batch engine keeps the plain loop)
    constexpr bool kParts = NT >= 512;
    if (kParts && warp == 0) {
      int64_t G = 0;
      for (int64_t k = lane; k < nlev; k += 32) G += (lst[k + 1] - lst[k] + 31) >> 5;
      for (int o = 16; o; o >>= 1) G += __shfl_xor_sync(AMVM_FULL, G, o);
      if (lane == 0) {
        int64_t P = G > 0 ? (AMVM_FC_PARTS_MUL * NW) / G : 1;
        sh->bc_i[10] = (int)(P < 1 ? 1 : P > 8 ? 8 : P);
      }
    }
    if (kParts) __syncthreads();
    const int P = kParts ? sh->bc_i[10] : 1;
    for (int64_t p0 = 0; p0 < n; p0 += kTJ) {
      const int64_t p1 = n - p0 < kTJ ? n : p0 + kTJ;
      for (int64_t e = tid; e < p1 - p0; e += NT) {
        const int32_t j = perm[p0 + e];
        tj[e] = j;
        tl[e] = cidx[j];
#pragma unroll
        for (int q = 0; q < kG; ++q)
          if (q < g) tb[e * kG + q] = ag[(int64_t)q * n + p0 + e];
      }
      if (tid == 0) sh->gnext = 0;
      __syncthreads();
      // buckets are handed out from the highest level down: a group's work
      // grows with the number of levels below it, so the longest groups
      // start first and the warps finish together (longest-first order)
      int ki = (int)nlev - 1;
      int64_t gbase = 0;  // first group id of bucket ki (groups are claimed in increasing order)
      for (;;) {
        int64_t item = 0;
        if (lane == 0) item = atomicAdd(&sh->gnext, 1);
        item = __shfl_sync(AMVM_FULL, item, 0);
        const int64_t grp = P == 1 ? item : item / P;
        const int part = P == 1 ? 0 : (int)(item - grp * P);
        if (grp >= ngrp) break;
        while (ki >= 0 && grp >= gbase + ((lst[ki + 1] - lst[ki] + 31) >> 5)) {
          gbase += (lst[ki + 1] - lst[ki] + 31) >> 5;
          --ki;
        }
        if (ki <= 0) break;  // the lowest level has nothing below it (and every later group is there)
        if ((int64_t)lst[ki] <= p0) continue;  // no lower-level position in this tile
        const int64_t ip = lst[ki] + (grp - gbase) * 32 + lane;
        const bool have = ip < lst[ki + 1];
        const int32_t i = have ? perm[ip] : 0;
        double bi[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) bi[q] = (have && q < g) ? ag[(int64_t)q * n + ip] : 0.0;
        const double xi = lv[ki];
        int rk = -1;
        for (int kj = nxt[nlev]; kj < ki; kj = nxt[kj]) {
          if (P > 1 && ++rk % P != part) continue;
          const int64_t s0 = (int64_t)lst[kj] > p0 ? (int64_t)lst[kj] : p0;
          const int64_t s1 = (int64_t)lst[kj + 1] < p1 ? (int64_t)lst[kj + 1] : p1;
          if (s0 >= s1) continue;
          const double delta = dsub(xi, lv[kj]);
          if (filt && delta < fD) continue;  // whole segment after the cut (uniform)
          double bq[kG];
#pragma unroll
          for (int q = 0; q < kG; ++q)
            bq[q] = q < g ? (tab ? bt[(q * nlev + ki) * nlev + kj] : ddiv(reps[q], delta)) : 0.0;
          // row 0 as a prefix: first position where dsub(b0_j, b0_i) < bq0 fails
          int64_t lo = s0, hi = s1;
          if (have) {
            while (lo < hi) {
              const int64_t mid = (lo + hi) >> 1;
              if (dsub(tb[(mid - p0) * kG], bi[0]) < bq[0]) lo = mid + 1;
              else hi = mid;
            }
          } else {
            lo = s0;
          }
          const int64_t mine = lo;
          int64_t wend = mine;
          for (int o = 16; o; o >>= 1) {
            const int64_t v = __shfl_xor_sync(AMVM_FULL, wend, o);
            wend = v > wend ? v : wend;
          }
          const int e0 = (int)(s0 - p0), e1 = (int)(wend - p0), emine = (int)(mine - p0);
#ifdef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
          if (lane == 0) atomicAdd((unsigned long long *)&sh->c.pc[14], (unsigned long long)(e1 - e0));
#endif
          {
            const int u = __reduce_add_sync(AMVM_FULL, emine - e0);
#ifndef AMVM_FC_PROFILE
            if (lane == 0) atomicAdd((unsigned long long *)&sh->c.pc[15], (unsigned long long)u);
#endif
          }
#endif
          // survivors of the staged rows: straight into the candidate list when
          // they are all the rows, else into the queue for the remaining rows
          auto emit = [&](int e, bool alive) {
            if (filt) alive = alive && (delta > fD || (int64_t)i <= fI);
            const unsigned bal = __ballot_sync(AMVM_FULL, alive);
            if (!bal) return;
            if (nr <= g && counting) {
              if (lane == 0) atomicAdd(&sh->counter, __popc(bal));
            } else if (nr <= g) {
              int bse = 0;
              if (lane == 0) bse = atomicAdd(&sh->counter, __popc(bal));
              bse = __shfl_sync(AMVM_FULL, bse, 0);
              if (alive) {
                const int pos2 = bse + __popc(bal & ((1u << lane) - 1u));
                if (pos2 < cap) cbuf[pos2] = Cand{i, tj[e], delta};
              }
            } else {
              int bse = 0;
              if (lane == 0) bse = atomicAdd(&sh->qcount, __popc(bal));
#ifdef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
              if (lane == 0) atomicAdd((unsigned long long *)&sh->c.pc[11], (unsigned long long)__popc(bal));
#endif
#endif
              bse = __shfl_sync(AMVM_FULL, bse, 0);
              if (alive) {
                const int qp = bse + __popc(bal & ((1u << lane) - 1u));
                if (qp < qcap) que[qp] = QEnt{i, tj[e], (uint16_t)ki, (uint16_t)kj, 0u};
                else if (fc_rest(i, tj[e], delta, nr, g)) fc_append(i, tj[e], delta, counting);
              }
            }
          };
          if (g == kG) {
            // common case: every staged row present; the tile is row-
            // interleaved per position (one 64-byte broadcast record), two
            // positions per iteration for independent dependency chains;
            // alive bits collect in a 32-position mask flushed with one scan
            // and one atomic per warp (survivors are ~1% of the pairs)
            const bool lane_ok = !filt || delta > fD || (int64_t)i <= fI;
            for (int cb = e0; cb < e1; cb += 32) {
              const int ce = e1 - cb < 32 ? e1 - cb : 32;
              unsigned msk = 0u;
              int u = 0;
              for (; u + 1 < ce; u += 2) {
                const double2 *ta = reinterpret_cast<const double2 *>(tb + (cb + u) * kG);
                const double2 *tc = reinterpret_cast<const double2 *>(tb + (cb + u + 1) * kG);
                double va[kG], vc[kG];
#pragma unroll
                for (int h = 0; h < kG / 2; ++h) {
                  const double2 x = ta[h], y = tc[h];
                  va[2 * h] = x.x; va[2 * h + 1] = x.y;
                  vc[2 * h] = y.x; vc[2 * h + 1] = y.y;
                }
                bool aa = cb + u < emine, ac = cb + u + 1 < emine;
#pragma unroll
                for (int q = 1; q < kG; ++q) {
                  aa &= dsub(va[q], bi[q]) < bq[q];
                  ac &= dsub(vc[q], bi[q]) < bq[q];
                }
                msk |= ((unsigned)aa | ((unsigned)ac << 1)) << u;
              }
              if (u < ce) {
                const double *tq = tb + (cb + u) * kG;
                bool alive = cb + u < emine;
#pragma unroll
                for (int q = 1; q < kG; ++q) alive &= dsub(tq[q], bi[q]) < bq[q];
                msk |= (unsigned)alive << u;
              }
              if (!lane_ok) msk = 0u;
              if (!__any_sync(AMVM_FULL, msk != 0u)) continue;
              const int c = __popc(msk);
              int incl = c;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(AMVM_FULL, incl, o);
                if (lane >= o) incl += y;
              }
              const int tot = __shfl_sync(AMVM_FULL, incl, 31);
              if (nr <= g && counting) {
                if (lane == 0) atomicAdd(&sh->counter, tot);
                continue;
              }
              int bse = 0;
              if (lane == 0) bse = atomicAdd(nr <= g ? &sh->counter : &sh->qcount, tot);
#ifdef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
              if (lane == 0 && nr > g) atomicAdd((unsigned long long *)&sh->c.pc[11], (unsigned long long)tot);
#endif
#endif
              int pos = __shfl_sync(AMVM_FULL, bse, 0) + incl - c;
              while (msk) {
                const int uu = __ffs(msk) - 1;
                msk &= msk - 1u;
                const int32_t j = tj[cb + uu];
                if (nr <= g) {
                  if (pos < cap) cbuf[pos] = Cand{i, j, delta};
                } else if (pos < qcap) {
                  que[pos] = QEnt{i, j, (uint16_t)ki, (uint16_t)kj, 0u};
                } else if (fc_rest(i, j, delta, nr, g)) {
                  fc_append(i, j, delta, counting);
                }
                ++pos;
              }
            }
          } else {
            for (int e = e0; e < e1; ++e) {
              const double *tq = tb + e * kG;
              bool alive = e < emine;
#pragma unroll
              for (int q = 1; q < kG; ++q)
                if (q < g) alive &= dsub(tq[q], bi[q]) < bq[q];
              emit(e, alive);
            }
          }
        }
      }
      __syncthreads();
    }
#ifdef AMVM_FC_PROFILE
    const long long fd0 = clock64();
#endif
    if (nr > g) fc_drain(nr, g, counting);
    __syncthreads();
#ifdef AMVM_FC_PROFILE
    if (tid == 0 && MODE == FC_ALL) sh->c.pc[12] += clock64() - fd0;
#endif
  }

  // fc_pass with one lane per (i, j) pair: for each i (one per warp, claimed
  // in turn) the lanes sweep the tile's positions below i's level, test every
  // staged row (row 0 first, the rest only when a lane survives it) and emit
  // exactly what fc_pass emits -- the same survivor set in another order
  // (every consumer of the list is order-free or sorts it).  For small level
  // buckets (C1: 16 variables per level, C2: one), where fc_pass's i-groups
  // leave most lanes idle.  Staged rows are laid out row-major per tile here
  // ([q][e]: consecutive lanes, consecutive words).
  template <int MODE>
  __device__ void fc_pass_pairs(int nr, int g, double fD, int64_t fI) {
    AMVM_LOCALS
    int32_t *lst = (int32_t *)scr;
    const int32_t *nxt = lst + (nlev + 1);
    double *tq = (double *)(scr + fc_tb_off(nlev));  // [kG][kTJ]
    int32_t *tl = (int32_t *)(tq + kG * kTJ);
    int32_t *tj = tl + kTJ;
    const double *bt = (const double *)(tj + kTJ);
    const int32_t *perm = ibuf;
    const int qcap = (int)fc_qcap(cap);
    constexpr bool filt = MODE != FC_ALL;
    constexpr bool counting = MODE == FC_COUNT;
    // positions of the lowest non-empty level have nothing below them
    const int64_t i0 = nxt[nlev] < nlev ? (int64_t)lst[nxt[nlev] + 1] : n;
    for (int64_t p0 = 0; p0 < n; p0 += kTJ) {
      const int64_t p1 = n - p0 < kTJ ? n : p0 + kTJ;
      const int w = (int)(p1 - p0);
      for (int e = tid; e < w; e += NT) {
        const int32_t j = perm[p0 + e];
        tj[e] = j;
        tl[e] = cidx[j];
      }
      for (int e = tid; e < g * w; e += NT) {
        const int q = e / w, x = e - q * w;
        tq[q * kTJ + x] = ag[(int64_t)q * n + p0 + x];
      }
      if (tid == 0) sh->gnext = 0;
      __syncthreads();
      const int64_t ib = i0 > p0 + 1 ? i0 : p0 + 1;  // i at or before p0: nothing below in the tile
      for (;;) {
        int64_t wi = 0;
        if (lane == 0) wi = atomicAdd(&sh->gnext, 1);
        const int64_t ip = n - 1 - __shfl_sync(AMVM_FULL, wi, 0);  // highest level (most pairs) first
        if (ip < ib) break;
        const int32_t i = perm[ip];
        const int ki = cidx[i];
        const int64_t eend = ((int64_t)lst[ki] < p1 ? (int64_t)lst[ki] : p1) - p0;
        if (eend <= 0) continue;
        if (filt && (int64_t)i > fI && !(dsub(lv[ki], lv[nxt[nlev]]) > fD)) continue;  // even the largest delta is cut
        const double xi = lv[ki];
        double bi[kG];
#pragma unroll
        for (int q = 0; q < kG; ++q) bi[q] = q < g ? ag[(int64_t)q * n + ip] : 0.0;
        for (int e0 = 0; e0 < eend; e0 += 32) {
          const int e = e0 + lane;
          const bool ok = e < eend;
          const int ec = ok ? e : 0;
          const int kj = tl[ec];
          const double delta = dsub(xi, lv[kj]);
          bool alive = ok;
          if (filt) alive = alive && (delta > fD || (delta == fD && (int64_t)i <= fI));
          if (g > 0)
            alive = alive && dsub(tq[ec], bi[0]) < (tab ? bt[(int64_t)ki * nlev + kj] : ddiv(reps[0], delta));
          if (!__any_sync(AMVM_FULL, alive)) continue;
#pragma unroll
          for (int q = 1; q < kG; ++q) {
            if (q < g && alive) {
              const double bq = tab ? bt[((int64_t)q * nlev + ki) * nlev + kj] : ddiv(reps[q], delta);
              alive = dsub(tq[q * kTJ + ec], bi[q]) < bq;
            }
          }
          const unsigned bal = __ballot_sync(AMVM_FULL, alive);
          if (!bal) continue;
          if (nr <= g && counting) {
            if (lane == 0) atomicAdd(&sh->counter, __popc(bal));
            continue;
          }
          int bse = 0;
          if (lane == 0) bse = atomicAdd(nr <= g ? &sh->counter : &sh->qcount, __popc(bal));
          bse = __shfl_sync(AMVM_FULL, bse, 0);
          if (alive) {
            const int pos = bse + __popc(bal & ((1u << lane) - 1u));
            const int32_t j = tj[e];
            if (nr <= g) {
              if (pos < cap) cbuf[pos] = Cand{i, j, delta};
            } else if (pos < qcap) {
              que[pos] = QEnt{i, j, (uint16_t)ki, (uint16_t)kj, 0u};
            } else if (fc_rest(i, j, delta, nr, g)) {
              fc_append(i, j, delta, counting);
            }
          }
        }
      }
      __syncthreads();
    }
    if (nr > g) fc_drain(nr, g, counting);
    __syncthreads();
  }

  // Sparse engine, column-indexed filter (SP, lists configured): the same
  // survivor set as the staged-row enumeration, for sparse filter rows.
  //   * row 0 is the argmax row (eps_0 = 0, bound +0): a pair survives it iff
  //     b0_j < b0_i (folded values; exact: a difference of two doubles is < 0
  //     iff the first is smaller), so every survivor has b0_i > 0 or b0_j < 0:
  //     the pairs are enumerated from row 0's nonzeros (b0_i > 0: i fixed, all
  //     j; b0_i <= 0 then needs b0_j < b0_i <= 0: j fixed with b0_j < 0, all i
  //     with b0_j < b0_i <= 0) -- a disjoint cover of the row-0 survivors;
  //   * a row q >= 1 whose bound is positive at the largest level difference
  //     passes every pair it touches in neither column (da = 0 < bound), so
  //     each pair is tested only on the rows in its two columns' lists (the
  //     filter rows' nonzeros indexed by column), with the reference's
  //     arithmetic (dsub of the folded values, ddiv(eps, delta)).
  // fc_sparse_build: checks the preconditions and builds the lists (false:
  // the general filter runs); fc_sparse_enum<MODE> is one enumeration (FC_ALL
  // collects, FC_COUNT counts and FC_CUT collects the survivors up to (fD, fI)
  // in the reference order, FC_HIST counts the survivors with delta == fD per
  // i into ibuf and those with delta > fD); fc_sparse_reset restores the
  // resting state (heads -1, row scratch zero).
  enum { FC_HIST = 3 };
  __device__ bool fc_sparse_build(int nr) {
    AMVM_LOCALS
    const int32_t *rw = sh->c.rcol;
    const double *rv = sh->c.rval;
    const int64_t *rp = sh->c.rptr;
    int32_t *fh = sh->c.fhead;
    FEnt *fe = sh->c.fent;
    double *rt = sh->c.rowtmp;
    if (tid == 0) {
      const double dmax = dsub(lv[nlev - 1], lv[0]);
      bool ok = nr >= 1 && reps[0] == 0.0 && dmax > 0.0;
      int64_t ent = 0;
      for (int q = 1; q < nr && ok; ++q) {
        ok = ddiv(reps[q], dmax) > 0.0;
        ent += __ldg(rp + rows[q] + 1) - __ldg(rp + rows[q]);
      }
      sh->bc_i[6] = ok && ent <= sh->c.fecap;
      sh->bc_i[7] = 0;
    }
    __syncthreads();
    if (!sh->bc_i[6]) return false;
    // lists: the nonzeros of filter rows 1.. by column (unordered: AND is order-free)
    for (int q = 1 + warp; q < nr; q += NW) {
      const int64_t r = rows[q], e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
      const bool pos = rsgn[q] != 0;
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int32_t c = __ldg(rw + e);
        const double a = __ldg(rv + e);
        const int slot = atomicAdd(&sh->bc_i[7], 1);
        fe[slot].q = q;
        fe[slot].b = pos ? a : -a;
        fe[slot].next = atomicExch(&fh[c], slot);
      }
    }
    // row 0, folded, densely in the (zero) row scratch
    const int64_t r0 = rows[0], z0 = __ldg(rp + r0), z1 = __ldg(rp + r0 + 1);
    const bool pos0 = rsgn[0] != 0;
    for (int64_t e = z0 + tid; e < z1; e += NT) {
      const double a = __ldg(rv + e);
      rt[__ldg(rw + e)] = pos0 ? a : -a;
    }
    __syncthreads();
    return true;
  }

  __device__ void fc_sparse_reset(int nr) {
    AMVM_LOCALS
    const int32_t *rw = sh->c.rcol;
    const int64_t *rp = sh->c.rptr;
    __syncthreads();
    for (int q = 1 + warp; q < nr; q += NW) {
      const int64_t r = rows[q], e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
      for (int64_t e = e0 + lane; e < e1; e += 32) sh->c.fhead[__ldg(rw + e)] = -1;
    }
    const int64_t r0 = rows[0], z0 = __ldg(rp + r0), z1 = __ldg(rp + r0 + 1);
    for (int64_t e = z0 + tid; e < z1; e += NT) sh->c.rowtmp[__ldg(rw + e)] = 0.0;
    __syncthreads();
  }

  template <int MODE>
  __device__ int fc_sparse_enum(double fD, int64_t fI) {
    AMVM_LOCALS
    const int32_t *rw = sh->c.rcol;
    const int64_t *rp = sh->c.rptr;
    const int32_t *fh = sh->c.fhead;
    const FEnt *fe = sh->c.fent;
    const double *rt = sh->c.rowtmp;
    if (tid == 0) sh->counter = 0;
    __syncthreads();
    const int64_t r0 = rows[0], z0 = __ldg(rp + r0), z1 = __ldg(rp + r0 + 1);
    const int64_t s0 = z1 - z0, nch = (n + 31) / 32;
    // one warp per row-0 nonzero c; skipped whole when c cannot pair (b0_c = 0,
    // or no level on the needed side of c's)
    for (int64_t k = warp; k < s0; k += NW)
    for (int64_t ch = 0; ch < nch; ++ch) {
      const int32_t c = __ldg(rw + z0 + k);
      const double bc = rt[c];
      if (bc == 0.0 || (bc > 0.0 ? cidx[c] == 0 : cidx[c] == nlev - 1)) break;
      const int64_t x = ch * 32 + lane;
      // bc > 0: (i, j) = (c, x) with b0_x < bc;  bc < 0: (i, j) = (x, c) with bc < b0_x <= 0
      bool alive = false;
      int32_t i = 0, j = 0;
      if (x < n && bc != 0.0) {
        const double bx = rt[x];
        if (bc > 0.0) {
          i = c; j = (int32_t)x;
          alive = bx < bc && cidx[j] < cidx[i];
        } else {
          i = (int32_t)x; j = c;
          alive = bc < bx && bx <= 0.0 && cidx[i] > cidx[j];
        }
      }
      double delta = 0.0;
      if (alive) {
        delta = dsub(lv[cidx[i]], lv[cidx[j]]);
        if (MODE == FC_COUNT || MODE == FC_CUT) alive = delta > fD || (delta == fD && (int64_t)i <= fI);
        if (MODE == FC_HIST) alive = delta >= fD;
      }
      if (alive) {
        // rows touching i (b_q(j) from j's list, 0 if absent)
        for (int32_t e = fh[i]; e >= 0 && alive; e = fe[e].next) {
          const int q = fe[e].q;
          double bj = 0.0;
          for (int32_t f = fh[j]; f >= 0; f = fe[f].next)
            if (fe[f].q == q) { bj = fe[f].b; break; }
          alive = dsub(bj, fe[e].b) < ddiv(reps[q], delta);
        }
        // rows touching j only (b_q(i) = 0)
        for (int32_t f = fh[j]; f >= 0 && alive; f = fe[f].next) {
          const int q = fe[f].q;
          bool in_i = false;
          for (int32_t e = fh[i]; e >= 0; e = fe[e].next)
            if (fe[e].q == q) { in_i = true; break; }
          if (!in_i) alive = dsub(fe[f].b, 0.0) < ddiv(reps[q], delta);
        }
      }
      if (MODE == FC_HIST) {
        if (alive && delta == fD) atomicAdd(&ibuf[i], 1);
        alive = alive && delta > fD;
      }
      const unsigned bal = __ballot_sync(AMVM_FULL, alive);
      if (bal) {
        int bse = 0;
        if (lane == 0) bse = atomicAdd(&sh->counter, __popc(bal));
        if (MODE == FC_ALL || MODE == FC_CUT) {
          bse = __shfl_sync(AMVM_FULL, bse, 0);
          const int pos = bse + __popc(bal & ((1u << lane) - 1u));
          if (alive && pos < cap) cbuf[pos] = Cand{i, j, delta};
        }
      }
    }
    __syncthreads();
    const int cnt = sh->counter;
    __syncthreads();
    return cnt;
  }

  // The whole sparse filter; -1: preconditions not met (general filter).
  // More survivors than the buffer: the max_candidates-th survivor of the
  // reference order (-delta, i, j) is found as in fc_overflow -- binary
  // search over the level differences by counting passes, then ONE pass
  // counting that class's survivors per i (a scan finds the cut i) -- and
  // only the survivors up to it are collected.
  __device__ int fc_sparse(int nr) {
    AMVM_LOCALS
    if (!fc_sparse_build(nr)) return -1;
    int cnt = fc_sparse_enum<FC_ALL>(0.0, 0);
    const int maxc = prm->max_candidates;
    if (cnt > cap && maxc > 0) {
      double *dcl = dbuf;  // idle during find_candidates
      if (tid == 0) {  // distinct level differences, descending (all level pairs: a superset is harmless)
        int nd = 0, bad = 0;
        for (int ki = 1; ki < nlev && !bad; ++ki)
          for (int kj = 0; kj < ki && !bad; ++kj) {
            const double d = dsub(lv[ki], lv[kj]);
            int at = 0;
            while (at < nd && dcl[at] > d) ++at;
            if (at < nd && dcl[at] == d) continue;
            if (nd == kMaxDeltaClasses || nd >= n) { bad = 1; break; }
            for (int q = nd; q > at; --q) dcl[q] = dcl[q - 1];
            dcl[at] = d;
            ++nd;
          }
        sh->bc_i[4] = bad ? -1 : nd;
      }
      __syncthreads();
      const int nd = sh->bc_i[4];
      __syncthreads();
      if (nd <= 0) {
        fc_sparse_reset(nr);
        return -1;
      }
      int lo = 0, hi = nd - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fc_sparse_enum<FC_COUNT>(dcl[mid], INT64_MAX) >= maxc) hi = mid;
        else lo = mid + 1;
      }
      const double dc = dcl[lo];
      for (int64_t k = tid; k < n; k += NT) ibuf[k] = 0;
      __syncthreads();
      const int above = fc_sparse_enum<FC_HIST>(dc, 0);  // survivors with delta > dc; ibuf: per i at dc
      // the smallest i* with above + #{delta == dc, i <= i*} >= maxc (warp 0 scans)
      if (warp == 0) {
        int64_t acc = above, istar = n - 1;
        bool found = false;
        for (int64_t k0 = 0; k0 < n && !found; k0 += 32) {
          const int64_t k = k0 + lane;
          const int v = k < n ? ibuf[k] : 0;
          int incl = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(AMVM_FULL, incl, o);
            if (lane >= o) incl += y;
          }
          const unsigned hit = __ballot_sync(AMVM_FULL, k < n && acc + incl >= maxc);
          if (hit) {
            istar = k0 + __ffs(hit) - 1;
            found = true;
          }
          acc += __shfl_sync(AMVM_FULL, incl, 31);
        }
        if (lane == 0) sh->bc_d[2] = (double)istar;
      }
      __syncthreads();
      const int64_t istar = (int64_t)sh->bc_d[2];
      cnt = fc_sparse_enum<FC_CUT>(dc, istar);
    }
    fc_sparse_reset(nr);
    if (cnt > cap) {  // no max_candidates and more survivors than the buffer
      fail(AMVM_ERR_UNSUPPORTED);
      cnt = (int)cap;
    }
    return cnt;
  }

  __device__ int find_candidates(bool always_sort) {
    AMVM_LOCALS
#ifdef AMVM_FC_PROFILE  // diagnostic: sub-phase cycles in pc[8..13]
    long long fq0 = clock64(), fq1;
#define FC_PROF(k) do { fq1 = clock64(); if (tid == 0) sh->c.pc[8 + (k)] += fq1 - fq0; fq0 = fq1; } while (0)
#else
#define FC_PROF(k) do { } while (0)
#endif
    const int nr = select_rows();
    FC_PROF(0);
    if constexpr (SP) {
      if (sh->c.fecap > 0) {
        int cnt = fc_sparse(nr);
        if (cnt >= 0) {
          const int maxc = prm->max_candidates;
          if ((maxc > 0 && cnt > maxc) || (always_sort && cnt > 1)) {
            sort_cands(cnt);
            if (maxc > 0 && cnt > maxc) cnt = maxc;
          }
          return cnt;
        }
      }
    }
    const int g = nr < kG ? nr : kG;
    int32_t *lst = (int32_t *)scr;
    int32_t *lfl = lst + (nlev + 1);
    double *tb = (double *)(scr + fc_tb_off(nlev));
    int32_t *tl = (int32_t *)(tb + kG * kTJ);
    int32_t *tj = tl + kTJ;
    double *bt = (double *)(tj + kTJ);
    int32_t *perm = ibuf;                 // level-sorted position -> variable
    // level buckets
    for (int64_t k = tid; k <= nlev; k += NT) lfl[k] = 0;
    __syncthreads();
    for (int64_t j = tid; j < n; j += NT) atomicAdd(&lfl[cidx[j]], 1);
    __syncthreads();
    if (warp == 0) {  // exclusive prefix over the level counts (warp shuffle-scan, 32 levels a step)
      int32_t acc = 0;
      for (int64_t k0 = 0; k0 < nlev; k0 += 32) {
        const int64_t k = k0 + lane;
        const int32_t c = k < nlev ? lfl[k] : 0;
        int32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(AMVM_FULL, incl, o);
          if (lane >= o) incl += y;
        }
        if (k < nlev) {
          lst[k] = acc + incl - c;
          lfl[k] = acc + incl - c;
        }
        acc += __shfl_sync(AMVM_FULL, incl, 31);
      }
      if (lane == 0) lst[nlev] = acc;
    }
    __syncthreads();
    for (int64_t j = tid; j < n; j += NT) perm[atomicAdd(&lfl[cidx[j]], 1)] = (int32_t)j;
    __syncthreads();
    // lfl (free again) becomes a skip list over empty level buckets:
    // lfl[k] = the smallest non-empty level > k (nlev if none), lfl[nlev] =
    // the lowest non-empty level; the pair loops step through it (C2: 127
    // variables over 1024 levels)
    if (warp == 0) {
      int nxt = (int)nlev;
      int64_t nne = 0;
      int maxb = 0;
      for (int64_t top = nlev - 1; top >= 0; top -= 32) {
        const int64_t k = top - lane;
        const bool ne = k >= 0 && lst[k + 1] > lst[k];
        if (ne) maxb = max(maxb, lst[k + 1] - lst[k]);
        const unsigned bal = __ballot_sync(AMVM_FULL, ne);  // bit l: level top - l non-empty
        // next non-empty above k: the nearest set bit below lane l (higher level), else nxt
        const unsigned above = bal & ((1u << lane) - 1u);
        if (k >= 0) lfl[k] = above ? (int)(top - (31 - __clz(above))) : nxt;
        if (bal) nxt = (int)(top - (31 - __clz(bal)));  // the lowest non-empty level in this chunk
        nne += __popc(bal);
      }
      maxb = __reduce_max_sync(AMVM_FULL, maxb);
      if (lane == 0) {
        lfl[nlev] = nxt;
        sh->fc_pairs = n < (int64_t)kFcPairs * nne;
        sh->fc_maxb = maxb;
      }
    }
    __syncthreads();
    const bool pairs = sh->fc_pairs != 0;
    // sort every level bucket by the tightest row's folded value b0 (eps_0 = 0:
    // that row defines t), so each i's row-0 survivors in a bucket are a prefix
    // (sparse engine: row 0 densely in the row scratch for the fill loops)
    constexpr bool sp = SP;
    if (sp) {
      sp_row_scatter(rows[0], false);
      __syncthreads();
    }
    auto row0 = [&](int32_t j) { return sp ? sh->c.rowtmp[j] : __ldg(Ar + (int64_t)rows[0] * n + j); };
    if (!pairs && sh->fc_maxb <= 32) {
      // every bucket fits a warp: one warp per bucket, a register bitonic sort
      // by (b0, j) -- the same order the block sort below produces
      for (int64_t k = warp; k < nlev; k += NW) {
        const int b0 = lst[k], sz = lst[k + 1] - b0;
        if (sz < 2) continue;
        const bool ok = lane < sz;
        int32_t j = ok ? perm[b0 + lane] : 0x7fffffff;
        double bv = 0.0;
        if (ok) {
          const double a = row0(j);
          bv = rsgn[0] ? a : -a;
        }
#pragma unroll
        for (int kk2 = 2; kk2 <= 32; kk2 <<= 1) {
#pragma unroll
          for (int jj = kk2 >> 1; jj > 0; jj >>= 1) {
            const double ob = __shfl_xor_sync(AMVM_FULL, bv, jj);
            const int32_t oj = __shfl_xor_sync(AMVM_FULL, j, jj);
            // invalid lanes (j = INT_MAX) sort last
            const bool oinv = oj == 0x7fffffff, minv = j == 0x7fffffff;
            const bool other_less = !oinv && (minv || ob < bv || (ob == bv && oj < j));
            const bool lower = (lane & jj) == 0, up = (lane & kk2) == 0;
            // keep the smaller in the lower lane of an ascending pair
            const bool take = (lower == up) ? other_less : (!other_less && oj != j);
            if (take) { bv = ob; j = oj; }
          }
        }
        if (ok) perm[b0 + lane] = j;
      }
      __syncthreads();
    } else if (!pairs) {  // (the lane-per-pair enumeration needs no order inside a bucket)
      int64_t n2 = 1;
      while (n2 < n) n2 <<= 1;
      if (n2 <= 65536 && nlev <= 32768 && fc_tb_off(nlev) + (size_t)12 * n2 <= scratch_bytes<NT>(nlev, tab)) {
        // in shared memory (after the bucket bounds): key (level << 16 | j)
        // + b0, one compare-exchange pair per thread per step
        double *sb = (double *)(scr + fc_tb_off(nlev));
        uint32_t *sk = (uint32_t *)(sb + n2);
        for (int64_t e = tid; e < n2; e += NT) {
          if (e < n) {
            const int32_t j = perm[e];
            const double a = row0(j);
            sk[e] = ((uint32_t)cidx[j] << 16) | (uint32_t)j;
            sb[e] = rsgn[0] ? a : -a;
          } else {
            sk[e] = 0xffffffffu;
            sb[e] = 0.0;
          }
        }
        __syncthreads();
        for (int64_t k = 2; k <= n2; k <<= 1) {
          for (int64_t jj = k >> 1; jj > 0; jj >>= 1) {
            for (int64_t t = tid; t < (n2 >> 1); t += NT) {
              const int64_t e = ((t & ~(jj - 1)) << 1) | (t & (jj - 1)), x = e | jj;
              const uint32_t ka = sk[e], kb = sk[x];
              const double ba = sb[e], bb = sb[x];
              const uint32_t la = ka >> 16, lb = kb >> 16;
              const bool gt = la > lb || (la == lb && (ba > bb || (ba == bb && ka > kb)));
              if (((e & k) == 0) == gt) {
                sk[e] = kb; sk[x] = ka;
                sb[e] = bb; sb[x] = ba;
              }
            }
            __syncthreads();
          }
        }
        for (int64_t e = tid; e < n; e += NT) perm[e] = (int32_t)(sk[e] & 0xffffu);
        __syncthreads();
      } else {
        int32_t *sl = (int32_t *)srt;
        int32_t *sj = sl + n2;
        double *sb = (double *)(sj + n2);
        for (int64_t e = tid; e < n2; e += NT) {
          if (e < n) {
            const int32_t j = perm[e];
            const double a = row0(j);
            sl[e] = cidx[j];
            sj[e] = j;
            sb[e] = rsgn[0] ? a : -a;
          } else {
            sl[e] = 0x7fffffff;
            sj[e] = 0;
            sb[e] = 0.0;
          }
        }
        __syncthreads();
        for (int64_t k = 2; k <= n2; k <<= 1) {
          for (int64_t jj = k >> 1; jj > 0; jj >>= 1) {
            for (int64_t t = tid; t < (n2 >> 1); t += NT) {
              const int64_t e = ((t & ~(jj - 1)) << 1) | (t & (jj - 1)), x = e | jj;
              const int32_t la = sl[e], lb = sl[x];
              const double ba = sb[e], bb = sb[x];
              const bool gt = la > lb || (la == lb && (ba > bb || (ba == bb && sj[e] > sj[x])));
              if (((e & k) == 0) == gt) {
                sl[e] = lb; sl[x] = la;
                sb[e] = bb; sb[x] = ba;
                const int32_t t0 = sj[e]; sj[e] = sj[x]; sj[x] = t0;
              }
            }
            __syncthreads();
          }
        }
        for (int64_t e = tid; e < n; e += NT) perm[e] = sj[e];
        __syncthreads();
      }
    }
    FC_PROF(1);
    // staged rows in level-sorted order, sign folded: ag[q*n + pos]
    if (sp) {  // row by row through the dense row scratch (row 0 is still in it)
      for (int q = 0; q < g; ++q) {
        if (q > 0) {
          sp_row_scatter(rows[q], false);
          __syncthreads();
        }
        for (int64_t ps = tid; ps < n; ps += NT) {
          const double a = sh->c.rowtmp[perm[ps]];
          ag[(int64_t)q * n + ps] = rsgn[q] ? a : -a;
        }
        __syncthreads();
        sp_row_scatter(rows[q], true);
        __syncthreads();
      }
      if (g == 0) {
        sp_row_scatter(rows[0], true);
        __syncthreads();
      }
    } else {
      for (int64_t e = tid; e < (int64_t)g * n; e += NT) {
        const int64_t q = e / n, ps = e - q * n;
        const double a = __ldg(Ar + (int64_t)rows[q] * n + perm[ps]);
        ag[e] = rsgn[q] ? a : -a;
      }
    }
    const int ll = (int)(nlev * nlev);
    if (tab) {
      for (int e = tid; e < g * ll; e += NT) {
        const int q = e / ll, r2 = e - q * ll;
        const int ki = r2 / (int)nlev, kj = r2 - ki * (int)nlev;
        bt[e] = ki > kj ? ddiv(reps[q], dsub(lv[ki], lv[kj])) : 0.0;
      }
    }
    if (tid == 0) {
      sh->counter = 0;
      sh->qcount = 0;
    }
    __syncthreads();
    FC_PROF(2);
    if (sh->fc_pairs) fc_pass_pairs<FC_ALL>(nr, g, 0.0, 0);
    else fc_pass<FC_ALL>(nr, g, 0.0, 0);
    FC_PROF(3);
    int cnt = sh->counter;
    __syncthreads();
    const int maxc = prm->max_candidates;
    if (cnt > cap) {
      if (maxc > 0) cnt = fc_overflow(nr, g, maxc);
      else {
        fail(AMVM_ERR_UNSUPPORTED);  // no cap requested and more survivors than the buffer
        cnt = (int)cap;
      }
    }
    if ((maxc > 0 && cnt > maxc) || (always_sort && cnt > 1)) {
      sort_cands(cnt);
      if (maxc > 0 && cnt > maxc) cnt = maxc;
    }
    FC_PROF(5);
#undef FC_PROF
    return cnt;
  }

  __device__ int fc_count(int nr, int g, double fD, int64_t fI) {
    if (tid == 0) { sh->counter = 0; sh->qcount = 0; }
    __syncthreads();
    if (sh->fc_pairs) fc_pass_pairs<FC_COUNT>(nr, g, fD, fI);
    else fc_pass<FC_COUNT>(nr, g, fD, fI);
    const int c = sh->counter;
    __syncthreads();
    return c;
  }

  // More survivors than the buffer holds: find the max_candidates-th survivor
  // of the reference order (-delta, i, j) by counting passes — binary search
  // over the distinct level differences present, then over i — and collect
  // only the survivors up to that (delta, i): fewer than max_candidates + n,
  // which the buffer holds by construction (cap >= max_candidates + n).
  __device__ int fc_overflow(int nr, int g, int maxc) {
    AMVM_LOCALS
    double *dcl = dbuf;  // idle during find_candidates; needs <= kMaxDeltaClasses
    int32_t *lst = (int32_t *)scr;
    if (tid == 0) {
      int nd = 0, bad = 0;
      for (int ki = 1; ki < nlev && !bad; ++ki) {
        if (lst[ki + 1] == lst[ki]) continue;
        for (int kj = 0; kj < ki && !bad; ++kj) {
          if (lst[kj + 1] == lst[kj]) continue;
          const double d = dsub(lv[ki], lv[kj]);
          int at = 0;
          while (at < nd && dcl[at] > d) ++at;
          if (at < nd && dcl[at] == d) continue;
          if (nd == kMaxDeltaClasses || nd >= n) { bad = 1; break; }
          for (int q = nd; q > at; --q) dcl[q] = dcl[q - 1];
          dcl[at] = d;
          ++nd;
        }
      }
      sh->bc_i[4] = bad ? -1 : nd;
    }
    __syncthreads();
    const int nd = sh->bc_i[4];
    __syncthreads();
    if (nd <= 0) {
      fail(AMVM_ERR_UNSUPPORTED);
      return (int)cap;
    }
    int lo = 0, hi = nd - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (fc_count(nr, g, dcl[mid], INT64_MAX) >= maxc) hi = mid;
      else lo = mid + 1;
    }
    const double dc = dcl[lo];
    int64_t ilo = 0, ihi = n - 1;
    while (ilo < ihi) {
      const int64_t mid = (ilo + ihi) >> 1;
      if (fc_count(nr, g, dc, mid) >= maxc) ihi = mid;
      else ilo = mid + 1;
    }
    if (tid == 0) { sh->counter = 0; sh->qcount = 0; }
    __syncthreads();
    if (sh->fc_pairs) fc_pass_pairs<FC_CUT>(nr, g, dc, ilo);
    else fc_pass<FC_CUT>(nr, g, dc, ilo);
    int cnt = sh->counter;
    __syncthreads();
    if (cnt > cap) {  // impossible: < maxc + n survivors up to the cut
      fail(AMVM_ERR_UNSUPPORTED);
      cnt = (int)cap;
    }
    return cnt;
  }

  // best_swap + _evaluate_chunk, localsearch.py:181-246: lowest post-swap
  // objective among strictly improving candidates, ties to the smallest
  // (i, j).  Returns found; the winner is uniform across the CTA.
  __device__ bool best_swap(int &bi, int &bj, double &bd, double &bt) {
    AMVM_LOCALS
    if (!(cobj > 0.0)) return false;
    const long long tf0 = clock64();
    const int cnt = find_candidates(false);
    const long long tf1 = clock64();
    if (tid == 0) sh->c.pc[5] += tf1 - tf0;
#ifndef AMVM_FC_PROFILE
    if (tid == 0) sh->c.pc[8] += 1;
#endif
#ifndef AMVM_FC_PROFILE
    if (tid == 0) sh->c.pc[9] += cnt;
#endif
    if (cnt == 0) return false;
    double wt = 0.0, wd = 0.0;
    int wi = -1, wj = -1;
    const double t0 = cobj;
    // sparse A: rows[] holds the filter rows by (|s| desc, index asc)
    const int nrows = sh->c.csc && sh->srt_rows_sorted ? sh->nfilter_rows : 0;
    constexpr bool sp = SP;
    if (sp) sp_select_top();
    // CTA-wide best complete t' so far (bit pattern: t' >= 0 orders as an
    // integer): a scan whose running max exceeds it cannot win, whatever the
    // order the warps finish in, so the winner is the same as a full scan's
    if (tid == 0) sh->swap_best = ~0ull;
    __syncthreads();
    for (int c = warp; c < cnt; c += NW) {
      const Cand e = cbuf[c];
      double mx = 0.0;
      if (sp) {
        mx = swap_tprime_sp(e.i, e.j, e.d);
      } else if (!(nrows > 0 && swap_tprime_sparse(e.i, e.j, e.d, nrows, mx))) {
        const double *ci = At + (int64_t)e.i * m;
        const double *cj = At + (int64_t)e.j * m;
        {  // screen: the rows that cut earlier candidates (one per lane; exact proofs)
          const int r = *(volatile int *)&sh->vrow[lane];
          const double y = fabs(dadd(cr[r], dmul(e.d, dsub(__ldg(cj + r), __ldg(ci + r)))));
          const uint64_t sb = *(volatile uint64_t *)&sh->swap_best;
          if (__any_sync(AMVM_FULL, y >= t0 || abs_key(y) > sb)) continue;
        }
        mx = 0.0;
        int64_t mr = lane;  // the row attaining this lane's max
        int it = 0;
        bool cut = false;
        for (int64_t r = lane; r < m; r += 32) {
          const double y = fabs(dadd(cr[r], dmul(e.d, dsub(__ldg(cj + r), __ldg(ci + r)))));
          if (y > mx) { mx = y; mr = r; }
          if ((++it & 7) == 0) {
            const uint64_t sb = *(volatile uint64_t *)&sh->swap_best;
            const unsigned hit = __ballot_sync(AMVM_FULL, mx >= t0 || abs_key(mx) > sb);
            if (hit) {  // remember the row that proved it for the screen
              if (lane == __ffs(hit) - 1) sh->vrow[atomicAdd(&sh->vins, 1) & 31] = (int)mr;
              cut = true;
              break;
            }
          }
        }
        mx = warp_max(mx);
        if (cut) continue;  // not improving, or beaten by a complete scan
      }
      if (mx < t0) {
        if (lane == 0) atomicMin((unsigned long long *)&sh->swap_best, (unsigned long long)abs_key(mx));
        if (wi < 0 || mx < wt || (mx == wt && (e.i < wi || (e.i == wi && e.j < wj)))) {
          wt = mx; wi = e.i; wj = e.j; wd = e.d;
        }
      }
    }
    if (tid == 0) sh->c.mv_ref += cnt;
    if (tid == 0) sh->c.mv_raw += cnt;
    if (lane == 0) {
      sh->red[warp][0] = wt;
      sh->red[warp][1] = wd;
      sh->red[warp][2] = __longlong_as_double(((int64_t)wi << 32) | (uint32_t)wj);
    }
    __syncthreads();
    if (tid == 0) sh->c.pc[6] += clock64() - tf1;
    bool found = false;
    for (int k = 0; k < NW; ++k) {
      const int64_t ij = __double_as_longlong(sh->red[k][2]);
      const int ki = (int)(ij >> 32), kj = (int)(uint32_t)ij;
      if (ki < 0) continue;
      const double kt = sh->red[k][0];
      if (!found || kt < bt || (kt == bt && (ki < bi || (ki == bi && kj < bj)))) {
        found = true; bt = kt; bi = ki; bj = kj; bd = sh->red[k][1];
      }
    }
    __syncthreads();
    return found;
  }

  // Sparse engine: t' over the union of the two columns' rows (the other
  // column's entry by binary search in its CSC rows, 0 if absent) and the
  // largest |s| outside both (the |s| top list); exactly the dense value.
  __device__ double swap_tprime_sp(int i, int j, double d) {
    AMVM_LOCALS
    const int64_t *cp = sh->c.cptr;
    const int32_t *crw = sh->c.crow;
    const double *cv = sh->c.cval;
    double mx = sp_untouched_max(i, j);
    for (int64_t e = __ldg(cp + i) + lane; e < __ldg(cp + i + 1); e += 32) {  // rows of column i
      const int64_t r = __ldg(crw + e);
      mx = fmax(mx, fabs(dadd(cr[r], dmul(d, dsub(sp_col_at(j, r), __ldg(cv + e))))));
    }
    for (int64_t e = __ldg(cp + j) + lane; e < __ldg(cp + j + 1); e += 32) {  // rows only column j touches
      const int64_t r = __ldg(crw + e);
      if (sp_col_find(i, r) < 0) mx = fmax(mx, fabs(dadd(cr[r], dmul(d, dsub(__ldg(cv + e), 0.0)))));
    }
    return warp_max(mx);
  }

  // s += d (A[:, j] - A[:, i]) on the sparse engine: each touched row once
  // (block-wide, no barrier inside; the caller synchronises)
  __device__ void swap_update_sp(int i, int j, double d) {
    AMVM_LOCALS
    const int64_t *cp = sh->c.cptr;
    const int32_t *crw = sh->c.crow;
    const double *cv = sh->c.cval;
    for (int64_t e = __ldg(cp + i) + tid; e < __ldg(cp + i + 1); e += NT) {
      const int64_t r = __ldg(crw + e);
      cr[r] = dadd(cr[r], dmul(d, dsub(sp_col_at(j, r), __ldg(cv + e))));
    }
    for (int64_t e = __ldg(cp + j) + tid; e < __ldg(cp + j + 1); e += NT) {
      const int64_t r = __ldg(crw + e);
      if (sp_col_find(i, r) < 0) cr[r] = dadd(cr[r], dmul(d, dsub(__ldg(cv + e), 0.0)));
    }
  }

  // t' = max_r |s_r + d (a_rj - a_ri)| for sparse A (warp-wide), exactly the
  // dense evaluation's value: rows outside nz(i) U nz(j) contribute |s_r|
  // (s + d*0 = s), so t' = max(touched rows, the largest-|s| untouched row).
  // The latter is the first row of rows[] (|s| descending) touched by
  // neither column; if every filter row is touched, returns false (the caller
  // scans densely).
  __device__ bool swap_tprime_sparse(int i, int j, double d, int nrows, double &out) {
    AMVM_LOCALS
    const int64_t *cp = sh->c.cptr;
    const int32_t *crw = sh->c.crow;
    const double *cv = sh->c.cval;
    int u = -1;
    for (int b0 = 0; b0 < nrows && u < 0; b0 += 32) {
      const int q = b0 + lane;
      bool free_row = false;
      if (q < nrows) {
        const int64_t r = rows[q];
        free_row = __ldg(Ar + r * n + i) == 0.0 && __ldg(Ar + r * n + j) == 0.0;
      }
      const unsigned bal = __ballot_sync(AMVM_FULL, free_row);
      if (bal) u = b0 + __ffs(bal) - 1;
    }
    if (u < 0) return false;
    double mx = fabs(cr[rows[u]]);
    for (int64_t e = cp[i] + lane; e < cp[i + 1]; e += 32) {  // rows touched by column i
      const int64_t r = __ldg(crw + e);
      mx = fmax(mx, fabs(dadd(cr[r], dmul(d, dsub(__ldg(Ar + r * n + j), __ldg(cv + e))))));
    }
    for (int64_t e = cp[j] + lane; e < cp[j + 1]; e += 32) {  // rows only column j touches
      const int64_t r = __ldg(crw + e);
      if (__ldg(Ar + r * n + i) == 0.0) mx = fmax(mx, fabs(dadd(cr[r], dmul(d, dsub(__ldg(cv + e), 0.0)))));
    }
    out = warp_max(mx);
    return true;
  }

  // apply_swap, core.py:228-245, with the objective predicted by best_swap.
  __device__ void apply_swap_known(int i, int j, double d, double t) {
    AMVM_LOCALS
    if constexpr (SP) {
      swap_update_sp(i, j, d);
    } else {
      const double *ci = At + (int64_t)i * m;
      const double *cj = At + (int64_t)j * m;
      for (int64_t r = tid; r < m; r += NT) cr[r] = dadd(cr[r], dmul(d, dsub(__ldg(cj + r), __ldg(ci + r))));
    }
    if (tid == 0) {
      const int32_t t0 = cidx[i];
      cidx[i] = cidx[j];
      cidx[j] = t0;
    }
    bump_known(t);
  }

  // apply_swap (core.py:228-245) when the new objective is not known:
  // s += (x_i - x_j) * (A[:, j] - A[:, i]) (DSUB, DMUL, DADD), levels
  // exchanged, then _bump (max |s|, or the refresh at REFRESH_PERIOD).
  __device__ void apply_swap_reduce(int i, int j) {
    AMVM_LOCALS
    const int ki = cidx[i], kj = cidx[j];
    const double d = dsub(lv[ki], lv[kj]);
    double mx = 0.0;
    if constexpr (SP) {
      swap_update_sp(i, j, d);
      __syncthreads();
      for (int64_t r = tid; r < m; r += NT) mx = fmax(mx, fabs(cr[r]));
    } else {
      const double *ci = At + (int64_t)i * m;
      const double *cj = At + (int64_t)j * m;
      for (int64_t r = tid; r < m; r += NT) {
        const double y = dadd(cr[r], dmul(d, dsub(__ldg(cj + r), __ldg(ci + r))));
        cr[r] = y;
        mx = fmax(mx, fabs(y));
      }
    }
    const double t = block_max_own(mx);
    if (tid == 0) {
      cidx[i] = kj;
      cidx[j] = ki;
    }
    __syncthreads();
    ccnt += 1;
    if (ccnt >= prm->refresh_period) refresh();
    else cobj = t;
  }

  // ---------------------------------------- best_swap with the l2 tie-break
  // localsearch.py:181-246 with FilterConfig.l2_tiebreak (not on the solve
  // path: SolverConfig.filter_config does not forward it).  The candidate
  // list (reference order) is split like np.array_split(.., min(workers,
  // cnt)); each chunk's winner is its smallest improving t', ties inside
  // the chunk going to the smallest (l2, i, j) with l2 =
  // np.linalg.norm(shifted[tied], axis=1) = sqrt(pairwise sum of y*y); a
  // chunk with a single tied candidate carries np.linalg.norm(shifted[k])
  // = sqrt(ddot).  Winners merge by (t, l2, i, j).  Block-uniform loops,
  // exact full scans: a correctness path, not a hot one.
  __device__ double swap_t_block(const Cand &e) {
    AMVM_LOCALS
    const double *ci = At + (int64_t)e.i * m, *cj = At + (int64_t)e.j * m;
    double mx = 0.0;
    for (int64_t r = tid; r < m; r += NT) mx = fmax(mx, fabs(dadd(cr[r], dmul(e.d, dsub(__ldg(cj + r), __ldg(ci + r))))));
    return block_max_own(mx);
  }

  __device__ double swap_l2(const Cand &e, bool pairwise) {
    AMVM_LOCALS
    const double *ci = At + (int64_t)e.i * m, *cj = At + (int64_t)e.j * m;
    auto y = [&](int64_t r) { return dadd(cr[r], dmul(e.d, dsub(__ldg(cj + r), __ldg(ci + r)))); };
    if (pairwise) {
      const double s2 = block_pairwise([&](int64_t r) { const double v = y(r); return dmul(v, v); }, m, lf_lo,
                                       lf_len, nleaf_m);
      return __dsqrt_rn(s2);
    }
    __syncthreads();
    if (warp == 0) {
      const double dd = warp_ddot_skx(y, y, m, lane);
      if (lane == 0) sh->bc_d[0] = __dsqrt_rn(dd);
    }
    __syncthreads();
    const double v = sh->bc_d[0];
    __syncthreads();
    return v;
  }

  __device__ bool best_swap_l2(int workers, int &bi, int &bj, double &bd, double &bt) {
    AMVM_LOCALS
    if (!(cobj > 0.0)) return false;
    const int cnt = find_candidates(true);
    if (cnt == 0) return false;
    const double t0 = cobj;
    const int K = workers < cnt ? workers : cnt;
    const int q = cnt / K, qr = cnt % K;
    bool found = false;
    double gl2 = 0.0;
    for (int c = 0; c < K; ++c) {
      const int c0 = c * q + (c < qr ? c : qr), c1 = c0 + q + (c < qr ? 1 : 0);
      double tmin = t0;
      int ntied = 0;
      for (int e = c0; e < c1; ++e) {
        const double tp = swap_t_block(cbuf[e]);
        if (tp < t0) {
          if (tp < tmin) { tmin = tp; ntied = 1; }
          else if (tp == tmin) ++ntied;
        }
      }
      if (ntied == 0) continue;
      int wi = -1, wj = -1;
      double wl2 = 0.0, wd = 0.0;
      for (int e = c0; e < c1; ++e) {
        const Cand ce = cbuf[e];
        if (swap_t_block(ce) != tmin) continue;
        const double l2 = swap_l2(ce, ntied > 1);
        if (wi < 0 || l2 < wl2 || (l2 == wl2 && (ce.i < wi || (ce.i == wi && ce.j < wj)))) {
          wi = ce.i; wj = ce.j; wl2 = l2; wd = ce.d;
        }
      }
      if (!found || tmin < bt ||
          (tmin == bt && (wl2 < gl2 || (wl2 == gl2 && (wi < bi || (wi == bi && wj < bj)))))) {
        found = true; bt = tmin; gl2 = wl2; bi = wi; bj = wj; bd = wd;
      }
    }
    return found;
  }

  // local_search, localsearch.py:249-269
  __device__ void local_search() {
    AMVM_LOCALS
    one_opt();
    for (int rd = 0; rd < prm->ls_max_rounds; ++rd) {
      int bi = -1, bj = -1;
      double bd = 0, bt = 0;
      if (!best_swap(bi, bj, bd, bt)) break;
#ifndef AMVM_FC_PROFILE
      if (tid == 0) sh->c.pc[10] += 1;
#endif
      apply_swap_known(bi, bj, bd, bt);
      one_opt();
    }
    __syncthreads();
  }

  // -------------------------------------------------------- impact scores
  // impact_scores, operators.py:54-74: d_j = sum_k |s_k| exp((-a (t-|s_k|))/|a_kj|)
  // summed over k in row order (numpy axis-0), / pairwise sum |s|.  A tile of
  // kTC columns x kTK rows: every thread first loads its kTK/...(independent)
  // A entries, computes the terms branch-free into smem, then each column's
  // owner thread adds its kTK terms in row order.  The exp argument uses a
  // Newton-refined reciprocal (<= 2 ulp) and exp_nonpos (<= 0.51 ulp): the
  // same tolerance class as numpy's own SIMD exp.
  __device__ void impact_scores(double alpha) {
    AMVM_LOCALS
    static_assert(kTC == NT, "impact tile: one column per thread");
    constexpr int kPer = kTC * kTK / NT;  // elements per thread per tile
    __syncthreads();
    const double t = cobj;
    const double tot = block_pairwise([&](int64_t k) { return fabs(cr[k]); }, m, lf_lo, lf_len, nleaf_m);
    const double na = -alpha;
    if (sh->c.csc) {
      impact_csc(na, t, tot);
      return;
    }
    if (n >= kIC4 * NT) {
      impact_stream<kIC4, kIR4, kIS4>(na, t, tot);
      return;
    }
    if (n >= NT) {
      impact_stream<kIC1, kIR1, kIS1>(na, t, tot);
      return;
    }
    // n < NT: one tile = the n columns x tk rows (tk = kTC*kTK/n, so no
    // thread computes a term for a column that does not exist: C2 has 127)
    const int tk = (int)((kTC * kTK) / n < kTKMax ? (kTC * kTK) / n : kTKMax);
    double *tile = (double *)scr;                      // n x (tk+1)
    double *rowv = tile + kTC * (kTK + 1);             // tk x {|s_k|, (-alpha)(t - |s_k|)}
    const int cols = (int)n;
    double acc = 0.0;
    // the next tile's A entries are loaded while this one is scored
    double av[kPer];
    auto load = [&](int64_t kb0, double *dst) {
      // unconditional loads from clamped (always valid) addresses, masked
      // after: all kPer loads are in flight together instead of one
      // predicated load-use pair at a time
      const int rws0 = (int)(m - kb0 < tk ? m - kb0 : tk);
      const int64_t kbc = kb0 < m ? kb0 : 0;
      double raw[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * NT, c = e / tk, k = e - c * tk;
        const int cc = c < cols ? c : cols - 1, kc = k < rws0 ? k : 0;
        raw[q] = __ldg(At + cc * m + kbc + kc);
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * NT, c = e / tk, k = e - c * tk;
        dst[q] = (kb0 < m && c < cols && k < rws0) ? fabs(raw[q]) : 0.0;
      }
    };
#if AMVM_IMPACT_PREFETCH
    load(0, av);
#endif
    for (int64_t kb = 0; kb < m; kb += tk) {
      const int rws = (int)(m - kb < tk ? m - kb : tk);
      for (int k = tid; k < tk; k += NT) {
        const double sv = k < rws ? fabs(cr[kb + k]) : 0.0;
        rowv[2 * k] = sv;
        rowv[2 * k + 1] = dmul(na, dsub(t, sv));
      }
#if !AMVM_IMPACT_PREFETCH
      load(kb, av);
#endif
      __syncthreads();
#if AMVM_IMPACT_PREFETCH
      double avn[kPer];
      load(kb + tk, avn);
#endif
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * NT, c = e / tk, k = e - c * tk;
        if (c < cols) {
          const double a = av[q];
          const double as = a > 0.0 ? a : 1.0;
          double y;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(as));
          y = dfma(y, dfma(-as, y, 1.0), y);
          y = dfma(y, dfma(-as, y, 1.0), y);
          const double x = dmul(rowv[2 * k + 1], y);
          const double term = dmul(rowv[2 * k], exp_nonpos(x));
          tile[c * (tk + 1) + k] = a > 0.0 ? term : 0.0;
        }
      }
      __syncthreads();
      if (tid < cols)
        for (int k = 0; k < rws; ++k) acc = dadd(acc, tile[tid * (tk + 1) + k]);
#if AMVM_IMPACT_PREFETCH
#pragma unroll
      for (int q = 0; q < kPer; ++q) av[q] = avn[q];
#endif
    }
    if (tid < cols) dbuf[tid] = ddiv(acc, tot);
    __syncthreads();
  }

  // Sparse A (CSC copy present): thread per column over its nonzeros in row
  // order.  The dense sum adds an exact +0 for every zero entry (terms are
  // >= +0, so the partial sum never is -0), hence skipping them is bitwise
  // the same sum; per nonzero the operations are those of the dense paths.
  __device__ void impact_csc(double na, double t, double tot) {
    AMVM_LOCALS
    const int64_t *cp = sh->c.cptr;
    const int32_t *cr_ = sh->c.crow;
    const double *cv = sh->c.cval;
    for (int64_t j = tid; j < n; j += NT) {
      double acc = 0.0;
      const int64_t e1 = cp[j + 1];
      for (int64_t e = cp[j]; e < e1; ++e) {
        const int32_t k = __ldg(cr_ + e);
        const double a = fabs(__ldg(cv + e));
        const double sv = fabs(cr[k]);
        const double w = dmul(na, dsub(t, sv));
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
        y = dfma(y, dfma(-a, y, 1.0), y);
        y = dfma(y, dfma(-a, y, 1.0), y);
        acc = dadd(acc, dmul(sv, exp_nonpos(dmul(w, y))));
      }
      dbuf[j] = ddiv(acc, tot);
    }
    __syncthreads();
  }

  // Wide instances (n >= NT): thread tid owns kIC columns (cb + u*NT + tid)
  // outright and adds each column's terms in row order straight from a
  // kIS-stage cp.async ring of kIR-row slices of its own columns (16-byte
  // chunks XOR-swizzled by tid, so the ring is bank-conflict free).  Every
  // thread only reads what it copied, so the stream needs no barrier: kIS - 1
  // slices are in flight while one is scored, and the kIC columns are
  // independent exp chains (ILP).  Same operations in the same order as the
  // tiled path.
  template <int kIC, int kIR, int kIS>
  __device__ void impact_stream(double na, double t, double tot) {
    AMVM_LOCALS
    // ring: kIS stages x kIC columns x NT threads x kIR doubles
    double *const ring = (double *)scr;
    const bool vec = (m & 1) == 0 && (((uintptr_t)At) & 15) == 0;
    const int64_t ntile = (m + kIR - 1) / kIR;
    static_assert(kIR % 2 == 0 && ((kIR / 2) & (kIR / 2 - 1)) == 0 && kIR <= 8, "kIR/2 chunks, power of 2");
    const int sw = tid & (kIR / 2 - 1);  // chunk swizzle within a thread's kIR/2 16-byte chunks
    for (int64_t cb = 0; cb < n; cb += (int64_t)kIC * NT) {
      const double *colp[kIC];
      bool col_ok[kIC];
#pragma unroll
      for (int u = 0; u < kIC; ++u) {
        const int64_t c = cb + u * NT + tid;
        col_ok[u] = c < n;
        colp[u] = At + (col_ok[u] ? c : 0) * m;
      }
      auto slot = [&](int64_t tix, int u) { return ring + (((tix % kIS) * kIC + u) * NT + tid) * kIR; };
      auto issue = [&](int64_t tix) {
        if (tix < ntile) {
          const int64_t kb = tix * kIR;
#pragma unroll
          for (int u = 0; u < kIC; ++u) {
            double *dst = slot(tix, u);
            if (vec) {
#pragma unroll
              for (int p = 0; p < kIR / 2; ++p) {
                const bool v = col_ok[u] && kb + 2 * p < m;
                cp_async16(dst + 2 * (p ^ sw), v ? colp[u] + kb + 2 * p : At, v);
              }
            } else {
#pragma unroll
              for (int k = 0; k < kIR; ++k) {
                const bool v = col_ok[u] && kb + k < m;
                cp_async8(dst + 2 * ((k >> 1) ^ sw) + (k & 1), v ? colp[u] + kb + k : At, v);
              }
            }
          }
        }
        cp_async_commit();  // one group per slice (empty past the end)
      };
#pragma unroll 1
      for (int s0 = 0; s0 < kIS; ++s0) issue(s0);
      double acc[kIC];
#pragma unroll
      for (int u = 0; u < kIC; ++u) acc[u] = 0.0;
#pragma unroll 1
      for (int64_t tix = 0; tix < ntile; ++tix) {
        cp_async_wait<kIS - 1>();  // slice tix has landed
        const int64_t kb = tix * kIR;
        const int rws = (int)(m - kb < kIR ? m - kb : kIR);
#pragma unroll
        for (int k = 0; k < kIR; ++k) {
          if (k < rws) {
            const double sv = fabs(cr[kb + k]);
            const double w = dmul(na, dsub(t, sv));
#pragma unroll
            for (int u = 0; u < kIC; ++u) {  // independent columns: ILP
              const double a = fabs(slot(tix, u)[2 * ((k >> 1) ^ sw) + (k & 1)]);
              const double as = a > 0.0 ? a : 1.0;
              double y;
              asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(as));
              y = dfma(y, dfma(-as, y, 1.0), y);
              y = dfma(y, dfma(-as, y, 1.0), y);
              const double term = dmul(sv, exp_nonpos(dmul(w, y)));
              acc[u] = dadd(acc[u], a > 0.0 ? term : 0.0);
            }
          }
        }
        issue(tix + kIS);  // into the stage just consumed (its values are in registers)
      }
      cp_async_wait<0>();
#pragma unroll
      for (int u = 0; u < kIC; ++u)
        if (col_ok[u]) dbuf[cb + u * NT + tid] = ddiv(acc[u], tot);
    }
    __syncthreads();
  }

  // ------------------------------------------------------------- destroy
  // Generator.choice(pop, r, replace=False) on thread 0 -> out[0..r).
  __device__ void choice_noreplace(Pcg &g, int64_t pop, int64_t r, int32_t *out) {
    AMVM_LOCALS
    if (pop > 10000 && r > pop / 50) {  // numpy tail-shuffle path
      for (int64_t i = 0; i < pop; ++i) ibuf[i] = (int32_t)i;
      const int64_t first = pop - r > 1 ? pop - r : 1;
      for (int64_t i = pop - 1; i >= first; --i) {
        const int64_t jj = (int64_t)pcg_bounded(g, (uint64_t)i);
        const int32_t t0 = ibuf[i];
        ibuf[i] = ibuf[jj];
        ibuf[jj] = t0;
      }
      for (int64_t q = 0; q < r; ++q) out[q] = ibuf[pop - r + q];
      return;
    }
    const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)r));
    for (uint64_t k = 0; k <= mask; ++k) hset[k] = ~0ull;
    for (int64_t j = pop - r; j < pop; ++j) {
      const uint64_t val = pcg_bounded(g, (uint64_t)j);
      uint64_t loc = val & mask;
      while (hset[loc] != ~0ull && hset[loc] != val) loc = (loc + 1) & mask;
      if (hset[loc] == ~0ull) {
        hset[loc] = val;
        out[j - pop + r] = (int32_t)val;
      } else {
        loc = (uint64_t)j & mask;
        while (hset[loc] != ~0ull) loc = (loc + 1) & mask;
        hset[loc] = (uint64_t)j;
        out[j - pop + r] = (int32_t)j;
      }
    }
    for (int64_t i = r - 1; i >= 1; --i) {
      const int64_t jj = (int64_t)pcg_bounded(g, (uint64_t)i);
      const int32_t t0 = out[i];
      out[i] = out[jj];
      out[jj] = t0;
    }
  }

  __device__ static void isort(int32_t *a, int64_t r) {
    for (int64_t i = 1; i < r; ++i) {
      const int32_t v = a[i];
      int64_t k = i - 1;
      while (k >= 0 && a[k] > v) {
        a[k + 1] = a[k];
        --k;
      }
      a[k + 1] = v;
    }
  }

  // removed = sort(picked), saved = idx[removed]   (operators.py:29-31)
  __device__ void finish_destroy(int64_t r) {
    AMVM_LOCALS
    if (tid == 0) {
      isort(pick, r);
      for (int64_t q = 0; q < r; ++q) {
        rem[q] = pick[q];
        sav[q] = cidx[pick[q]];
      }
    }
    __syncthreads();
  }

  // random_destroy, operators.py:34-39
  __device__ void random_destroy(int64_t r) {
    AMVM_LOCALS
    __syncthreads();
    if (tid == 0) choice_noreplace(sh->rng, n, r, pick);
    finish_destroy(r);
  }

  // worst_remove_destroy, operators.py:77-105
  __device__ void worst_destroy(int64_t r, double alpha) {
    AMVM_LOCALS
    if (!(cobj > 0.0)) {
      random_destroy(r);
      return;
    }
    // The candidate is a copy of the CURRENT solution here (cand_from_cur, or
    // cand_is_cur after an accept), and the current one changes only on an
    // accept (a few % of iterations), so the scores of the current solution
    // are cached per instance and reused until the next accept: same inputs,
    // same deterministic computation, same bits.
    double *const ic = sh->ic;
    if (ic && __ldcg(sh->iv) == 1) {
      for (int64_t k = tid; k < n; k += NT) dbuf[k] = __ldcg(ic + k);
      __syncthreads();
    } else {
      impact_scores(alpha);
#ifndef AMVM_FC_STATS
#ifndef AMVM_FC_PROFILE
      if (tid == 0) sh->c.pc[14] += 1;
#endif
#endif
      if (ic) {
        for (int64_t k = tid; k < n; k += NT) ic[k] = dbuf[k];
        __syncthreads();
        if (tid == 0) *sh->iv = 1;
      }
    }
    auto gd = [&](int64_t k) { return dbuf[k]; };
    if (block_pairwise(gd, n, lf_lo + nleaf_m, lf_len + nleaf_m, nleaf_n) <= 0.0) {
      random_destroy(r);
      return;
    }
    for (int64_t q = 0; q < r; ++q) {
      const double total = block_pairwise(gd, n, lf_lo + nleaf_m, lf_len + nleaf_m, nleaf_n);
      if (!(total > 0.0)) {
        // mass exhausted: rng.choice(setdiff1d(arange(n), picked), r - q, False);
        // the set difference (ascending) by the whole block: mark the picks,
        // then an order-preserving compaction, NT positions per step
        int32_t *rest = (int32_t *)pbuf;  // n int32 fit in n doubles
        for (int64_t k = tid; k < n; k += NT) ibuf[k] = 0;
        __syncthreads();
        for (int64_t k = tid; k < q; k += NT) ibuf[pick[k]] = 1;
        __syncthreads();
        int64_t base = 0;
        for (int64_t c0 = 0; c0 < n; c0 += NT) {
          const int64_t k = c0 + tid;
          const bool f = k < n && !ibuf[k];
          const unsigned bal = __ballot_sync(AMVM_FULL, f);
          if (lane == 0) sh->wcnt[warp] = __popc(bal);
          __syncthreads();
          int before = 0, tot = 0;
          for (int w = 0; w < NW; ++w) {
            if (w < warp) before += sh->wcnt[w];
            tot += sh->wcnt[w];
          }
          if (f) rest[base + before + __popc(bal & ((1u << lane) - 1u))] = (int32_t)k;
          base += tot;
          __syncthreads();
        }
        if (tid == 0) {
          choice_noreplace(sh->rng, base, r - q, pick + q);
          for (int64_t k = q; k < r; ++k) pick[k] = rest[pick[k]];
        }
        break;
      }
      // p = d / total; numpy's sequential cumsum is a bare DADD chain on
      // thread 0 over shared memory, fed in chunks of the (idle) phase
      // scratch by the whole block, keeping the value before each
      // 32-element block of the cdf so the search rescans one block
      for (int64_t k = tid; k < n; k += NT) pbuf[k] = ddiv(dbuf[k], total);
      {
        double *const ps = (double *)scr;
        const int64_t cs = (int64_t)(scratch_bytes<NT>(nlev, tab) / 8) & ~(int64_t)31;
        double acc = 0.0;
        for (int64_t base = 0; base < n; base += cs) {
          const int64_t len = n - base < cs ? n - base : cs;
          __syncthreads();  // pbuf written / the previous chunk consumed
          for (int64_t k = tid; k < len; k += NT) ps[k] = pbuf[base + k];
          __syncthreads();
          if (tid == 0) {
            for (int64_t c0 = 0; c0 < len; c0 += 32) {
              cbk[(base + c0) >> 5] = acc;
              const double *pc = ps + c0;
              if (len - c0 >= 32) {
#pragma unroll
                for (int l = 0; l < 32; ++l) acc = dadd(acc, pc[l]);
              } else {
                for (int l = 0; l < (int)(len - c0); ++l) acc = dadd(acc, pc[l]);
              }
            }
          }
        }
        if (tid == 0) sh->bc_d[3] = acc;
        __syncthreads();
      }
      if (warp == 0) {
        // Generator.choice(n, p): cdf = cumsum(p); cdf /= cdf[-1];
        // searchsorted(cdf, random(), 'right')
        const int64_t nch = (n + 31) / 32;
        const double last = sh->bc_d[3];  // cdf[n-1]
        double u = 0.0;
        if (lane == 0) u = pcg_random(sh->rng);
        u = __shfl_sync(AMVM_FULL, u, 0);
        __syncwarp();
        // first chunk whose last cdf value normalizes above u (cdf is monotone)
        int64_t lo = 0, hi = nch - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          const double end = mid + 1 < nch ? cbk[mid + 1] : last;
          if (u < ddiv(end, last)) hi = mid;
          else lo = mid + 1;
        }
        const int64_t k0 = lo * 32;
        const double pv = k0 + lane < n ? pbuf[k0 + lane] : 0.0;
        double a2 = cbk[lo];
        int64_t pickk = -1;
        const int cnt = (int)(n - k0 < 32 ? n - k0 : 32);
        for (int l = 0; l < cnt; ++l) {
          a2 = dadd(a2, __shfl_sync(AMVM_FULL, pv, l));
          if (u < ddiv(a2, last)) {
            pickk = k0 + l;
            break;
          }
        }
        if (pickk < 0) pickk = n - 1;  // unreachable: cdf[n-1]/cdf[n-1] = 1 > u
        if (lane == 0) {
          pick[q] = (int32_t)pickk;
          dbuf[pickk] = 0.0;
        }
      }
      __syncthreads();
    }
    finish_destroy(r);
  }

  // ------------------------------------------------------------- repairs
  // two_nearest, core.py:62-72: first two of a stable argsort of |lv - v|.
  // Every warp scans redundantly, so the result is uniform without a barrier.
  __device__ void two_nearest(double v, int &c1, int &c2) {
    AMVM_LOCALS
    double bd = 0;
    int bk = 0x7fffffff;
    for (int k = lane; k < nlev; k += 32) {
      const double dk = fabs(dsub(lv[k], v));
      if (bk == 0x7fffffff || dk < bd) { bd = dk; bk = k; }
    }
    for (int o = 16; o; o >>= 1) {
      const double od = __shfl_xor_sync(AMVM_FULL, bd, o);
      const int ok = __shfl_xor_sync(AMVM_FULL, bk, o);
      if (ok != 0x7fffffff && (bk == 0x7fffffff || od < bd || (od == bd && ok < bk))) { bd = od; bk = ok; }
    }
    c1 = bk;
    bk = 0x7fffffff;
    for (int k = lane; k < nlev; k += 32) {
      if (k == c1) continue;
      const double dk = fabs(dsub(lv[k], v));
      if (bk == 0x7fffffff || dk < bd) { bd = dk; bk = k; }
    }
    for (int o = 16; o; o >>= 1) {
      const double od = __shfl_xor_sync(AMVM_FULL, bd, o);
      const int ok = __shfl_xor_sync(AMVM_FULL, bk, o);
      if (ok != 0x7fffffff && (bk == 0x7fffffff || od < bd || (od == bd && ok < bk))) { bd = od; bk = ok; }
    }
    c2 = bk;
  }

  // random_repair, operators.py:108-117 (all r coins drawn up front: they are
  // consecutive in the stream — nothing else draws during a repair).
  __device__ void random_repair(const int32_t *rm, const int32_t *sv, int64_t r) {
    AMVM_LOCALS
    __syncthreads();
    if (tid == 0)
      for (int64_t q = 0; q < r; ++q) coin[q] = (int32_t)pcg_bounded(sh->rng, 1);
    __syncthreads();
    for (int64_t q = 0; q < r; ++q) {
      int c1, c2;
      two_nearest(lv[sv[q]], c1, c2);
      apply_shift_reduce(rm[q], coin[q] ? c2 : c1);
    }
  }

  // greedy_repair, operators.py:120-138: the exact in-place sequence.
  __device__ void greedy_repair(const int32_t *rm, const int32_t *sv, int64_t r) {
    AMVM_LOCALS
    __syncthreads();
    for (int64_t q = 0; q < r; ++q) {
      const int64_t j = rm[q];
      int c1, c2;
      two_nearest(lv[sv[q]], c1, c2);
      apply_shift_reduce(j, c1);
      const double t1 = cobj;
      apply_shift_reduce(j, c2);
      const double t2 = cobj;
      if (tid == 0) sh->c.mv_ref += 2;
      if (tid == 0) sh->c.mv_raw += 2;
      if (t1 < t2 || (t1 == t2 && lv[c1] < lv[c2])) apply_shift_reduce(j, c1);
    }
  }

  // ------------------------------------------------------------ controller
  // accept, controller.py:168-183 (np.linalg.norm = sqrt of OpenBLAS ddot)
  __device__ bool accept() {
    AMVM_LOCALS
    if (cobj < uobj) return true;
    if (prm->l2_tiebreak && cobj <= dadd(uobj, prm->accept_tie_tol)) {
      __syncthreads();
      if (warp < 2) {
        const double *x = warp == 0 ? cr : ur;
        const double dd = warp_ddot_skx([&](int64_t i) { return x[i]; }, [&](int64_t i) { return x[i]; }, m, lane);
        if (lane == 0) sh->bc_d[warp] = __dsqrt_rn(dd);
      }
      __syncthreads();
      const bool ok = sh->bc_d[0] < sh->bc_d[1];
      __syncthreads();
      return ok;
    }
    return false;
  }

  // select_operators, controller.py:88-90 (thread 0)
  __device__ int select_pair() { return bank_select(sh->c.w, sh->rng); }

  // update_weights, controller.py:99-131 (thread 0 owns the bank)
  __device__ void update_weights(int pair, int outcome) {
    AMVM_LOCALS
    if (tid != 0) return;
    bank_update(sh->c.w, sh->c.sc, sh->c.seg, sh->c.life, &sh->c.bit, pair, outcome, prm->sigma1, prm->sigma2,
                prm->sigma3, prm->decay, prm->weight_floor, prm->n_segment);
  }

  __device__ void cand_from_cur() {
    AMVM_LOCALS
    for (int64_t i = tid; i < m; i += NT) cr[i] = ur[i];
    for (int64_t j = tid; j < n; j += NT) cidx[j] = uidx[j];
    cobj = uobj;
    ccnt = ucnt;
    __syncthreads();
  }

  __device__ void cur_from_cand() {
    AMVM_LOCALS
    for (int64_t i = tid; i < m; i += NT) ur[i] = cr[i];
    for (int64_t j = tid; j < n; j += NT) uidx[j] = cidx[j];
    uobj = cobj;
    ucnt = ccnt;
  }

  __device__ void write_best(int64_t inst, const amvm_result &res) {
    AMVM_LOCALS
    double *br = res.best.residual + inst * m;
    int32_t *bi = res.best.idx + inst * n;
    for (int64_t i = tid; i < m; i += NT) br[i] = ur[i];
    for (int64_t j = tid; j < n; j += NT) bi[j] = uidx[j];
    bobj = uobj;
    bcnt = ucnt;
  }

  __device__ static uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  }

  // ------------------------------------------------------------- set-up
  __device__ void bind(const KArgs &a, unsigned char *smem, int slot) {
    tid = threadIdx.x;
    lane = tid & 31;
    warp = tid >> 5;
    sh = (Shared<NT> *)amvm_dyn_smem;
    (void)smem;
    if (tid == 0) {
      Ctx &c = sh->c;
      c.m = a.m;
      c.n = a.n;
      c.nlev = a.nlev;
      c.At = a.At;
      c.Ar = a.Ar;
      c.cptr = a.cptr;
      c.crow = a.crow;
      c.cval = a.cval;
      c.csc = a.sparse ? 1 : ((const WsHeader *)a.ws)->csc_ok;
      c.sparse = a.sparse;
      c.ktop = a.ktop;
      c.rptr = a.rptr;
      c.rcol = a.rcol;
      c.rval = a.rval;
      c.prm = a.prm;
      c.cap = a.cap;
      c.tab = a.tab;
      const SlotLayout L = slot_layout(a.m, a.n, a.prm.k_eps, a.prm.r, a.cap, a.sparse ? a.ktop : 0,
                                       a.sparse ? a.fecap : 0);
      c.kk = L.kk;
      c.fecap = a.sparse ? a.fecap : 0;
      c.fhead = (int32_t *)(a.ws + sizeof(WsHeader) + ws_dense_bytes(a.m, a.n, a.sparse) +
                            (size_t)slot * a.slot_bytes + L.fhead);
      c.fent = (FEnt *)(a.ws + sizeof(WsHeader) + ws_dense_bytes(a.m, a.n, a.sparse) +
                        (size_t)slot * a.slot_bytes + L.fent);
      unsigned char *base = a.ws + sizeof(WsHeader) + ws_dense_bytes(a.m, a.n, a.sparse) +
                            (size_t)slot * a.slot_bytes;
      c.rowtmp = (double *)(base + L.rowtmp);
      c.top = (int32_t *)(base + L.top);
      c.status = (int32_t *)a.ws;
      c.ur = (double *)(base + L.ur);
      c.uidx = (int32_t *)(base + L.uidx);
      c.cidx = (int32_t *)(base + L.cidx);
      c.dbuf = (double *)(base + L.dbuf);
      c.pbuf = (double *)(base + L.pbuf);
      c.cbk = (double *)(base + L.cbk);
      c.lf_lo = (int64_t *)(base + L.lf_lo);
      c.lf_len = (int64_t *)(base + L.lf_len);
      c.lf_sum = (double *)(base + L.lf_sum);
      c.rows = (int32_t *)(base + L.rows);
      c.reps = (double *)(base + L.reps);
      c.rsgn = (int32_t *)(base + L.rsgn);
      c.ag = (double *)(base + L.ag);
      c.cbuf = (Cand *)(base + L.cbuf);
      c.que = (QEnt *)(base + L.que);
      c.hset = (uint64_t *)(base + L.hset);
      c.rem = (int32_t *)(base + L.rem);
      c.sav = (int32_t *)(base + L.sav);
      c.pick = (int32_t *)(base + L.pick);
      c.coin = (int32_t *)(base + L.coin);
      c.ibuf = (int32_t *)(base + L.ibuf);
      c.srt = base + L.srt;
      // dynamic smem: Shared | lv | scratch | cr
      size_t o = sizeof(Shared<NT>);
      c.off_lv = (uint32_t)o;
      o += 8 * ((a.nlev + 1) & ~1);
      c.off_scr = (uint32_t)o;
      o += scratch_bytes<NT>(a.nlev, a.tab);
      c.cr = a.cr_smem ? (double *)(amvm_dyn_smem + o) : (double *)(base + L.crg);
      // leaf trees of numpy's pairwise sum for lengths m and n
      c.nleaf_m = pw_leaves(a.m, c.lf_lo, c.lf_len, (int)L.nleaf, sh->pw_a, sh->pw_b);
      c.nleaf_n = pw_leaves(a.n, c.lf_lo + c.nleaf_m, c.lf_len + c.nleaf_m, (int)(2 * L.nleaf - c.nleaf_m),
                            sh->pw_a, sh->pw_b);
    }
    if (tid < 32) sh->vrow[tid] = 0;  // any row index < m is a valid screen row
    if (tid == 0) sh->vins = 0;
    __syncthreads();
    if constexpr (SP) {  // the row scratch starts (and stays) zero; the workspace is not cleared by the host
      for (int64_t j = tid; j < a.n; j += NT) sh->c.rowtmp[j] = 0.0;
      if (sh->c.fecap > 0)  // (list heads likewise start and stay -1)
        for (int64_t j = tid; j < a.n; j += NT) sh->c.fhead[j] = -1;
      __syncthreads();
    }
  }

  __device__ void load_levels(const KArgs &a, int64_t inst) {
    AMVM_LOCALS
    if (tid == 0) sh->c.b = a.B + inst * m;
    for (int64_t k = tid; k < nlev; k += NT) lv[k] = a.levels[inst * nlev + k];
    __syncthreads();
  }

  __device__ void load_rng(const amvm_pcg64 *st) {
    AMVM_LOCALS
    if (tid == 0) sh->rng = pcg_load(st);
  }

  __device__ void store_rng(amvm_pcg64 *st) {
    AMVM_LOCALS
    if (tid == 0) pcg_store(sh->rng, st);
  }

  // ------------------------------------------------------- solve (one inst)
  // solve, controller.py:211-286, from the host-computed initial solution.
  // With a.chunk_iters = K > 0 the call runs iterations [chunk*K, chunk*K+K)
  // only, resuming from / parking to the instance's InstState, so instances
  // migrate between CTAs at iteration boundaries (load balance).  Returns
  // true when the instance is finished (results written).
  __device__ bool solve_instance(const KArgs &a, int64_t inst, int64_t chunk = 0) {
    AMVM_LOCALS
    load_levels(a, inst);
    const amvm_result &res = a.res;
    const int T = a.prm.max_iters;
    const int K = a.chunk_iters;
    InstState *st = K > 0 ? (InstState *)(a.ist + inst * a.ist_bytes) : nullptr;
    const InstLayout IL = inst_layout(m, n);
    int it = 0;
    int64_t elapsed = 0;
    if (tid == 0) {
      sh->ic = a.icache ? (double *)(a.icache + inst * a.icache_bytes) : nullptr;
      sh->iv = a.icache ? a.ivalid + inst : nullptr;
      if (a.icache && chunk == 0) *sh->iv = 0;  // a new start solution
    }
    if (chunk == 0) {
      for (int64_t i = tid; i < m; i += NT) ur[i] = a.s_r[inst * m + i];
      for (int64_t j = tid; j < n; j += NT) uidx[j] = a.s_idx[inst * n + j];
      uobj = a.s_obj[inst];
      ucnt = a.s_cnt[inst];
      __syncthreads();
      write_best(inst, res);
      if (tid == 0) {
        for (int k = 0; k < 4; ++k) {
          sh->c.w[k] = 1.0; sh->c.sc[k] = 0.0; sh->c.seg[k] = 0; sh->c.life[k] = 0;
        }
        sh->c.bit = 0;
        sh->c.mv_ref = sh->c.mv_raw = 0;
        for (int k = 0; k < 16; ++k) sh->c.pc[k] = 0;
      }
    } else {  // resume a parked instance (L2 reads: parked by another SM)
      const double *sr = (const double *)((const unsigned char *)st + IL.r);
      const int32_t *si = (const int32_t *)((const unsigned char *)st + IL.idx);
      for (int64_t i = tid; i < m; i += NT) ur[i] = __ldcg(sr + i);
      for (int64_t j = tid; j < n; j += NT) uidx[j] = __ldcg(si + j);
      uobj = __ldcg(&st->uobj);
      bobj = __ldcg(&st->bobj);
      ucnt = __ldcg(&st->ucnt);
      bcnt = __ldcg(&st->bcnt);
      it = __ldcg(&st->it);
      elapsed = __ldcg((const long long *)&st->elapsed_ns);
      if (tid == 0) {
        for (int k = 0; k < 4; ++k) {
          sh->c.w[k] = __ldcg(&st->w[k]); sh->c.sc[k] = __ldcg(&st->sc[k]);
          sh->c.seg[k] = __ldcg((const long long *)&st->seg[k]);
          sh->c.life[k] = __ldcg((const long long *)&st->life[k]);
        }
        sh->c.bit = __ldcg((const long long *)&st->bit);
        sh->c.mv_ref = __ldcg((const long long *)&st->mv_ref);
        sh->c.mv_raw = __ldcg((const long long *)&st->mv_raw);
        for (int k = 0; k < 16; ++k) sh->c.pc[k] = __ldcg((const long long *)&st->pc[k]);
      }
      __syncthreads();
    }
    load_rng(&a.rng[inst]);
    const int it_end = K > 0 && (int64_t)T - it > K ? it + K : T;
    const int64_t r = a.prm.r;
    const uint64_t t_start = gtimer() - (uint64_t)elapsed;
    bool cand_is_cur = false;
    bool finished = false;
    while (it < it_end) {
      if (bobj == 0.0) {
        finished = true;
        break;
      }
      long long tp = clock64(), tq;
      if (tid == 0) {
        int stop = 0;
        if (a.time_budget_ns >= 0 && (int64_t)(gtimer() - t_start) > a.time_budget_ns) stop = 1;
        sh->bc_i[0] = stop;
        sh->bc_i[1] = stop ? 0 : select_pair();
      }
      __syncthreads();
      const int stop = sh->bc_i[0], pair = sh->bc_i[1];
      __syncthreads();
      if (stop) {
        finished = true;
        break;
      }
      ++it;
      if (!cand_is_cur) cand_from_cur();
      cand_is_cur = false;
      tq = clock64(); if (tid == 0) sh->c.pc[0] += tq - tp; tp = tq;
      if (pair < 2) random_destroy(r);
      else worst_destroy(r, a.prm.alpha);
      tq = clock64(); if (tid == 0) sh->c.pc[pair < 2 ? 1 : 2] += tq - tp; tp = tq;
      if (pair & 1) greedy_repair(rem, sav, r);
      else random_repair(rem, sav, r);
      tq = clock64(); if (tid == 0) sh->c.pc[3] += tq - tp; tp = tq;
      const long long fc0 = sh->c.pc[5] + sh->c.pc[6];
      local_search();
      tq = clock64(); if (tid == 0) sh->c.pc[4] += (tq - tp) - (sh->c.pc[5] + sh->c.pc[6] - fc0); tp = tq;
      const bool acc = accept();
      int outcome;
      if (acc && cobj < bobj) outcome = 0;
      else if (acc && cobj < uobj) outcome = 1;
      else if (acc) outcome = 2;
      else outcome = 3;
      if (acc) {
        cur_from_cand();
        cand_is_cur = true;
        if (tid == 0 && sh->iv) *sh->iv = 0;  // the cached scores belonged to the old current
        __syncthreads();
        if (uobj < bobj) write_best(inst, res);
      }
      update_weights(pair, outcome);
      if (tid == 0 && res.trace_current_t) {
        const int64_t o = inst * (int64_t)T + it - 1;
        res.trace_current_t[o] = uobj;
        res.trace_best_t[o] = bobj;
        res.trace_pair[o] = (uint8_t)pair;
        res.trace_accepted[o] = (uint8_t)acc;
      }
      if (tid == 0) sh->c.pc[7] += clock64() - tp;
    }
    if (!finished && it < T) {  // park for the next chunk
      double *sr = (double *)((unsigned char *)st + IL.r);
      int32_t *si = (int32_t *)((unsigned char *)st + IL.idx);
      for (int64_t i = tid; i < m; i += NT) sr[i] = ur[i];
      for (int64_t j = tid; j < n; j += NT) si[j] = uidx[j];
      if (tid == 0) {
        st->uobj = uobj; st->bobj = bobj; st->ucnt = ucnt; st->bcnt = bcnt; st->it = it;
        st->elapsed_ns = (int64_t)(gtimer() - t_start);
        for (int k = 0; k < 4; ++k) {
          st->w[k] = sh->c.w[k]; st->sc[k] = sh->c.sc[k]; st->seg[k] = sh->c.seg[k]; st->life[k] = sh->c.life[k];
        }
        st->bit = sh->c.bit;
        st->mv_ref = sh->c.mv_ref; st->mv_raw = sh->c.mv_raw;
        for (int k = 0; k < 16; ++k) st->pc[k] = sh->c.pc[k];
      }
      store_rng(&a.rng[inst]);
      __syncthreads();
      return false;
    }
    if (tid == 0) {
      res.best.objective[inst] = bobj;
      res.best.updates[inst] = bcnt;
      res.initial_objective[inst] = a.s_obj[inst];
      res.iterations[inst] = it;
      for (int k = 0; k < 4; ++k) res.operator_uses[inst * 4 + k] = sh->c.life[k];
      if (res.moves_scored) {
        res.moves_scored[2 * inst] = sh->c.mv_ref;
        res.moves_scored[2 * inst + 1] = sh->c.mv_raw;
      }
      if (res.phase_cycles)
        for (int k = 0; k < 16; ++k) res.phase_cycles[16 * inst + k] = sh->c.pc[k];
    }
    store_rng(&a.rng[inst]);
    __syncthreads();
    return true;
  }

  // ------------------------------------------------- component operations
  __device__ void load_sol(const KArgs &a) {
    AMVM_LOCALS
    load_levels(a, 0);
    for (int64_t i = tid; i < m; i += NT) cr[i] = a.s_r[i];
    for (int64_t j = tid; j < n; j += NT) cidx[j] = a.s_idx[j];
    cobj = a.s_obj[0];
    ccnt = a.s_cnt[0];
    if (tid == 0) {
      sh->c.mv_ref = sh->c.mv_raw = 0;
      for (int k = 0; k < 16; ++k) sh->c.pc[k] = 0;
    }
    __syncthreads();
  }

  __device__ void store_sol(const KArgs &a) {
    AMVM_LOCALS
    __syncthreads();
    for (int64_t i = tid; i < m; i += NT) a.s_r[i] = cr[i];
    for (int64_t j = tid; j < n; j += NT) a.s_idx[j] = cidx[j];
    if (tid == 0) {
      a.s_obj[0] = cobj;
      a.s_cnt[0] = ccnt;
    }
  }

  __device__ void run_op(const KArgs &a) {
    AMVM_LOCALS
    if (tid == 0) { sh->ic = nullptr; sh->iv = nullptr; }
    load_sol(a);
    switch (a.op) {
      case OP_ONE_OPT:
        one_opt();
        store_sol(a);
        break;
      case OP_LOCAL_SEARCH:
        local_search();
        store_sol(a);
        break;
      case OP_FIND_CAND: {
        const int cnt = cobj > 0.0 ? find_candidates(true) : 0;
        const int k = cnt < a.x_cap ? cnt : a.x_cap;
        for (int q = tid; q < k; q += NT) {
          a.x_i[q] = cbuf[q].i;
          a.x_j[q] = cbuf[q].j;
          a.x_d[q] = cbuf[q].d;
        }
        if (tid == 0) *a.x_cnt = k;
        break;
      }
      case OP_BEST_SWAP: {  // kind = workers with the l2 tie-break, 0 without
        int bi = -1, bj = -1;
        double bd = 0, bt = 0;
        const bool f = a.kind > 0 ? best_swap_l2(a.kind, bi, bj, bd, bt) : best_swap(bi, bj, bd, bt);
        if (tid == 0) {
          a.x_out4[0] = f ? bi : -1;
          a.x_out4[1] = f ? bj : -1;
          a.x_out4[2] = f ? bd : 0.0;
          a.x_out4[3] = f ? bt : 0.0;
        }
        break;
      }
      case OP_IMPACT:
        impact_scores(a.prm.alpha);
        for (int64_t j = tid; j < n; j += NT) a.x_d[j] = dbuf[j];
        break;
      case OP_DESTROY:
        load_rng(a.rng);
        if (a.kind == 0) random_destroy(a.prm.r);
        else worst_destroy(a.prm.r, a.prm.alpha);
        for (int64_t q = tid; q < a.prm.r; q += NT) a.x_i[q] = rem[q];
        store_rng(a.rng);
        break;
      case OP_REPAIR:
        load_rng(a.rng);
        if (a.kind == 0) random_repair(a.x_i, a.x_saved, a.x_r);
        else greedy_repair(a.x_i, a.x_saved, a.x_r);
        store_rng(a.rng);
        store_sol(a);
        break;
      case OP_APPLY_SHIFT:  // x_r = j, kind = new level (core.py:208-225)
        apply_shift_reduce(a.x_r, a.kind);
        store_sol(a);
        break;
      case OP_APPLY_SWAP:  // x_r = i, kind = j (core.py:228-245)
        apply_swap_reduce(a.x_r, a.kind);
        store_sol(a);
        break;
      default:
        fail(AMVM_ERR_INVALID);
    }
  }
};

}  // namespace amvm

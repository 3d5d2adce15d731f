// amvm.cu — kernels and the extern "C" boundary of libamvm.so (include/amvm.h).
//
// Build (see paper_2508_13437_b200/build.py):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
//        -shared -Xcompiler -fPIC -o libamvm.so amvm.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "amvm_engine.cuh"

using namespace amvm;

// ------------------------------------------------------------------ kernels
// Persistent solve: one CTA per resident slot, instances pulled from a
// counter so uneven iteration counts balance across SMs.
template <int NT, bool SP>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : AMVM_MIN_BLOCKS) k_solve(KArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Engine<NT, SP> E;
  E.bind(a, smem, blockIdx.x);
  WsHeader *hdr = (WsHeader *)a.ws;
  // Tasks: without chunking, task t = instance t.  Chunked: task t = (chunk
  // t / count, instance t % count), handed out in order, so every instance's
  // chunk c is taken before any chunk c + 1 and the batch's tail is one chunk,
  // not one whole instance.  A task waits for its instance's previous chunk
  // (taken earlier by a running CTA, so this cannot deadlock; with count >=
  // resident CTAs it almost never waits).  One call site of solve_instance
  // keeps the engine inlined.
  // (loop state lives in shared memory and kernel parameters, not registers:
  // the engine inlined below needs all of them)
  for (;;) {
    if (threadIdx.x == 0) {
      const int64_t nch = a.chunk_iters > 0 && a.prm.max_iters > 0
                              ? (a.prm.max_iters + a.chunk_iters - 1) / a.chunk_iters : 1;
      const unsigned long long t = atomicAdd(&hdr->next_task, 1ull);
      const int64_t inst = (int64_t)(t % a.count), chunk = (int64_t)(t / a.count);
      int skip = 0;
      if (a.chunk_iters > 0 && t < (unsigned long long)a.count * nch) {
        int32_t *prog = &((InstState *)(a.ist + inst * a.ist_bytes))->progress;
        int p;
        while ((p = atomicAdd(prog, 0)) < chunk) __nanosleep(1000);
        __threadfence();
        skip = p > chunk;  // finished early: nothing left to run
      }
      E.sh->task_live = t < (unsigned long long)a.count * nch;
      E.sh->task_skip = skip;
      E.sh->task_inst = inst;
      E.sh->task_chunk = chunk;
    }
    __syncthreads();
    const bool live = E.sh->task_live, skip = E.sh->task_skip;
    __syncthreads();
    if (!live) break;
    if (skip) continue;
    const bool done = E.solve_instance(a, E.sh->task_inst, E.sh->task_chunk);
    if (a.chunk_iters > 0) {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int64_t nch = a.prm.max_iters > 0 ? (a.prm.max_iters + a.chunk_iters - 1) / a.chunk_iters : 1;
        atomicExch(&((InstState *)(a.ist + E.sh->task_inst * a.ist_bytes))->progress,
                   done ? (int)nch : (int)E.sh->task_chunk + 1);
      }
    }
  }
}

// Ar[i*n + j] = At[j*m + i]: 32x32 tiles through shared memory, both sides
// coalesced.  grid (ceil(n/32), ceil(m/32)), block (32, 8).
__global__ void k_transpose(const double *__restrict__ At, double *__restrict__ Ar, int64_t m, int64_t n) {
  __shared__ double t[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    t[r][threadIdx.x] = (j < n && i < m) ? At[j * m + i] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < m && j < n) Ar[i * n + j] = t[threadIdx.x][r];
  }
}

// CSC build: one warp per column.  count -> exclusive scan (one CTA) ->
// fill in row order (ballot compaction keeps rows ascending).
__global__ void k_csc_count(const double *__restrict__ At, int64_t m, int64_t n, int64_t *__restrict__ cnt) {
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double *col = At + j * m;
  int64_t c = 0;
  for (int64_t i = lane; i < m; i += 32) c += col[i] != 0.0;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(AMVM_FULL, c, o);
  if (lane == 0) cnt[j + 1] = c;
}

__global__ void k_csc_scan(int64_t *ptr, int64_t n, int64_t cap, WsHeader *hdr) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  // each thread scans a contiguous chunk, then the chunk totals
  const int64_t per = (n + 1023) / 1024, lo = 1 + t * per, hi = lo + per < n + 1 ? lo + per : n + 1;
  int64_t s = 0;
  for (int64_t k = lo; k < hi; ++k) s += ptr[k];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int k = 0; k < 1024; ++k) {
      const int64_t v = part[k];
      part[k] = acc;
      acc += v;
    }
    ptr[0] = 0;
    hdr->csc_ok = acc <= cap;
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int64_t k = lo; k < hi; ++k) {
    acc += ptr[k];
    ptr[k] = acc;
  }
}

__global__ void k_csc_fill(const double *__restrict__ At, int64_t m, int64_t n, const int64_t *__restrict__ ptr,
                           int32_t *__restrict__ row, double *__restrict__ val, const WsHeader *hdr) {
  if (!hdr->csc_ok) return;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double *col = At + j * m;
  int64_t pos = ptr[j];
  for (int64_t i0 = 0; i0 < m; i0 += 32) {
    const int64_t i = i0 + lane;
    const double v = i < m ? col[i] : 0.0;
    const unsigned bal = __ballot_sync(AMVM_FULL, v != 0.0);
    if (v != 0.0) {
      const int64_t q = pos + __popc(bal & ((1u << lane) - 1u));
      row[q] = (int32_t)i;
      val[q] = v;
    }
    pos += __popc(bal);
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_op(KArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  Engine<NT> E;
  E.bind(a, smem, 0);
  E.run_op(a);
}

// accept (controller.py:168-183) for one (current, candidate) pair: strict
// improvement, or (l2) a tie within tol and a strictly smaller
// np.linalg.norm = sqrt(OpenBLAS ddot).  64 threads: warp 0 the candidate's
// norm, warp 1 the current one's.
__global__ void k_accept(int64_t m, const double *__restrict__ cur_r, const double *__restrict__ cur_obj,
                         const double *__restrict__ cand_r, const double *__restrict__ cand_obj, int l2, double tol,
                         int32_t *verdict) {
  __shared__ double nrm[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double co = *cur_obj, ca = *cand_obj;
  const bool need = !(ca < co) && l2 && ca <= amvm::dadd(co, tol);
  if (need) {
    const double *x = warp == 0 ? cand_r : cur_r;
    const double dd = warp_ddot_skx([&](int64_t i) { return x[i]; }, [&](int64_t i) { return x[i]; }, m, lane);
    if (lane == 0) nrm[warp] = __dsqrt_rn(dd);
  }
  __syncthreads();
  if (threadIdx.x == 0) *verdict = ca < co ? 1 : (need && nrm[0] < nrm[1] ? 1 : 0);
}

// select_operators / update_weights (controller.py:88-131) on a device bank.
__global__ void k_bank_select(const amvm_bank *bank, amvm_pcg64 *rng, int32_t *pair) {
  Pcg g = pcg_load(rng);
  *pair = bank_select(bank->weights, g);
  pcg_store(g, rng);
}

__global__ void k_bank_update(amvm_bank *bank, int pair, int outcome, double s1, double s2, double s3,
                              double floor_w, int n_segment) {
  bank_update(bank->weights, bank->scores, bank->segment_uses, bank->lifetime_uses, &bank->iteration, pair,
              outcome, s1, s2, s3, bank->decay, floor_w, n_segment);
}

// compute_residual (core.py:183-197) for a batch sharing A: residual[k] =
// A @ levels_k[idx_k] - B[k] in numpy's OpenBLAS dgemv order, objective[k] =
// max |residual[k]|.  CTA = kRI instances x NT rows (grid: instance groups x
// row chunks, so a C5 shard is ~1800 CTAs and every SM stays busy); thread =
// one row; each A element loaded once feeds kRI instances (FP64 FMA, 4
// lane-accumulators per output exactly as the dgemv_t 4x4 kernel; the x
// values come from shared memory as 16-byte broadcasts).  Rows outside the
// 4x4 groups (m % 4 != 0) and m == 1 take the scalar emulation in the first
// row chunk.  The objective is an atomicMax over the chunks on the bit
// pattern of |v| >= 0 (obj zeroed by the caller).
constexpr int kRI = 8;
constexpr int kRJ = 256;

// x_k = levels_k[idx_k] (compute_residual) or, when Xd != nullptr, the dense
// row Xd[k] (b = X @ w, builders.py:366); B == nullptr skips the "- b".
template <int NT>
__global__ void __launch_bounds__(NT) k_residual(int64_t m, int64_t n, int64_t nlev, int64_t count,
                                                 const double *__restrict__ At, const double *__restrict__ B,
                                                 const double *__restrict__ levels, const int32_t *__restrict__ idx,
                                                 const double *__restrict__ Xd,
                                                 double *__restrict__ res, double *__restrict__ obj) {
  __shared__ __align__(16) double xs[kRI][kRJ];
  __shared__ double red[kRI][NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = (int64_t)blockIdx.x * kRI;
  const int64_t chunk = blockIdx.y;
  const int ni = (int)(count - k0 < kRI ? count - k0 : kRI);
  const int64_t g4 = m & ~(int64_t)3, m1 = n & -4;
  double mx[kRI];
#pragma unroll
  for (int q = 0; q < kRI; ++q) mx[q] = 0.0;
  if (m > 1) {
    {
      const int64_t i = chunk * NT + tid;
      double y[kRI], l[kRI][4];
#pragma unroll
      for (int q = 0; q < kRI; ++q) {
        y[q] = 0.0;
        l[q][0] = l[q][1] = l[q][2] = l[q][3] = 0.0;
      }
      for (int64_t j0 = 0; j0 < m1; j0 += kRJ) {
        const int jn = (int)(m1 - j0 < kRJ ? m1 - j0 : kRJ);
        __syncthreads();
        for (int e = tid; e < kRI * kRJ; e += NT) {
          const int q = e / kRJ, jj = e - q * kRJ;
          xs[q][jj] = (q < ni && jj < jn)
                          ? (Xd ? Xd[(k0 + q) * n + j0 + jj]
                                : levels[(k0 + q) * nlev + idx[(k0 + q) * n + j0 + jj]])
                          : 0.0;
        }
        __syncthreads();
        if (i < g4) {
          for (int jj = 0; jj < jn; jj += 4) {
            const int64_t j = j0 + jj;
            const double a0 = __ldg(At + j * m + i), a1 = __ldg(At + (j + 1) * m + i);
            const double a2 = __ldg(At + (j + 2) * m + i), a3 = __ldg(At + (j + 3) * m + i);
#pragma unroll
            for (int q = 0; q < kRI; ++q) {
              const double2 x01 = *reinterpret_cast<const double2 *>(&xs[q][jj]);
              const double2 x23 = *reinterpret_cast<const double2 *>(&xs[q][jj + 2]);
              l[q][0] = amvm::dfma(a0, x01.x, l[q][0]);
              l[q][1] = amvm::dfma(a1, x01.y, l[q][1]);
              l[q][2] = amvm::dfma(a2, x23.x, l[q][2]);
              l[q][3] = amvm::dfma(a3, x23.y, l[q][3]);
            }
            if (((j + 4) % 2048) == 0 || j + 4 == m1) {  // end of a dgemv_t block
#pragma unroll
              for (int q = 0; q < kRI; ++q) {
                y[q] = amvm::dadd(y[q], amvm::dadd(amvm::dadd(l[q][0], l[q][2]), amvm::dadd(l[q][1], l[q][3])));
                l[q][0] = l[q][1] = l[q][2] = l[q][3] = 0.0;
              }
            }
          }
        }
      }
      if (i < g4) {
        for (int q = 0; q < ni; ++q) {
          const double *lvq = levels + (k0 + q) * nlev;
          const int32_t *ix = idx + (k0 + q) * n;
          const double *xd = Xd + (k0 + q) * n;
          auto xv = [&](int64_t j) { return Xd ? xd[j] : lvq[ix[j]]; };
          double v = y[q];
          switch (n & 3) {
            case 1: v = amvm::dfma(At[m1 * m + i], xv(m1), v); break;
            case 2: v = amvm::dadd(v, amvm::dfma(At[m1 * m + i], xv(m1), amvm::dmul(At[(m1 + 1) * m + i], xv(m1 + 1)))); break;
            case 3:
              v = amvm::dadd(v, amvm::dfma(At[(m1 + 2) * m + i], xv(m1 + 2),
                               amvm::dfma(At[m1 * m + i], xv(m1), amvm::dmul(At[(m1 + 1) * m + i], xv(m1 + 1)))));
              break;
            default: break;
          }
          if (B) v = amvm::dsub(v, B[(k0 + q) * m + i]);
          res[(k0 + q) * m + i] = v;
          mx[q] = fmax(mx[q], fabs(v));
        }
      }
    }
    // leftover rows (4x2 / 4x1 kernels)
    for (int64_t i = g4 + tid; chunk == 0 && i < m; i += NT) {
      for (int q = 0; q < ni; ++q) {
        const double *lvq = levels + (k0 + q) * nlev;
        const int32_t *ix = idx + (k0 + q) * n;
        const double *xd = Xd + (k0 + q) * n;
        double v = gemv_row([&](int64_t j) { return At[j * m + i]; },
                            [&](int64_t j) { return Xd ? xd[j] : lvq[ix[j]]; }, n, gemv_kind(i, m));
        if (B) v = amvm::dsub(v, B[(k0 + q) * m + i]);
        res[(k0 + q) * m + i] = v;
        mx[q] = fmax(mx[q], fabs(v));
      }
    }
  } else if (chunk == 0 && warp < ni) {  // m == 1: numpy uses ddot
    const int q = warp;
    const double *lvq = levels + (k0 + q) * nlev;
    const int32_t *ix = idx + (k0 + q) * n;
    const double *xd = Xd + (k0 + q) * n;
    double v = warp_ddot_skx([&](int64_t j) { return At[j]; },
                             [&](int64_t j) { return Xd ? xd[j] : lvq[ix[j]]; }, n, lane);
    if (B) v = amvm::dsub(v, B[k0 + q]);
    if (lane == 0) res[k0 + q] = v;
    mx[q] = fabs(v);
  }
#pragma unroll
  for (int q = 0; q < kRI; ++q) {
    double v = warp_max(mx[q]);
    if (lane == 0) red[q][warp] = v;
  }
  __syncthreads();
  if (obj && tid < ni) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v = fmax(v, red[tid][w]);
    atomicMax(reinterpret_cast<unsigned long long *>(obj + k0 + tid), (unsigned long long)__double_as_longlong(v));
  }
}

// PTQ row preparation (builders.py:366-371 + controller.py:157-165), one CTA
// per weight row: lo/hi = min/max w (widened by 0.5 if the range collapses),
// levels = numpy linspace(lo, hi, L) (k*step + lo, last = hi), idx_j = first
// argmin_k |w_j - levels_k|.
template <int NT>
__global__ void __launch_bounds__(NT) k_ptq_prepare(int64_t n, int64_t nlev, const double *__restrict__ W,
                                                    double *__restrict__ levels, int32_t *__restrict__ idx) {
  __shared__ double lo_s[NT / 32], hi_s[NT / 32];
  __shared__ double lvs[1024];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k = blockIdx.x;
  const double *w = W + k * n;
  double lo = w[0], hi = w[0];
  for (int64_t j = tid; j < n; j += NT) {
    lo = fmin(lo, w[j]);
    hi = fmax(hi, w[j]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(AMVM_FULL, lo, o));
    hi = fmax(hi, __shfl_xor_sync(AMVM_FULL, hi, o));
  }
  if (lane == 0) { lo_s[warp] = lo; hi_s[warp] = hi; }
  __syncthreads();
  lo = lo_s[0];
  hi = hi_s[0];
  for (int q = 1; q < NT / 32; ++q) { lo = fmin(lo, lo_s[q]); hi = fmax(hi, hi_s[q]); }
  if (amvm::dsub(hi, lo) < 1e-12) {
    lo = amvm::dsub(lo, 0.5);
    hi = amvm::dadd(hi, 0.5);
  }
  if (nlev == 1) {
    if (tid == 0) lvs[0] = lo;
  } else {
    const double step = amvm::ddiv(amvm::dsub(hi, lo), (double)(nlev - 1));
    for (int64_t q = tid; q < nlev; q += NT)
      lvs[q] = q == nlev - 1 ? hi : amvm::dadd(amvm::dmul((double)q, step), lo);
  }
  __syncthreads();
  for (int64_t q = tid; q < nlev; q += NT) levels[k * nlev + q] = lvs[q];
  for (int64_t j = tid; j < n; j += NT) {
    const double v = w[j];
    int best = 0;
    double bd = fabs(amvm::dsub(v, lvs[0]));
    for (int q = 1; q < nlev; ++q) {
      const double d = fabs(amvm::dsub(v, lvs[q]));
      if (d < bd) { bd = d; best = q; }
    }
    idx[k * n + j] = best;
  }
}

// numpy SeedSequence(seed) -> PCG64 state (numpy/random/bit_generator.pyx,
// _pcg64.pyx): pool of 4 uint32 via hashmix/mix, generate_state(4, uint64),
// pcg64_set_seed(state = s[0]:s[1], inc = s[2]:s[3]).
namespace {
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

uint32_t hashmix(uint32_t v, uint32_t &hc) {
  v ^= hc;
  hc *= kMultA;
  v *= hc;
  v ^= v >> 16;
  return v;
}
uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

void seed_pcg64(uint64_t seed, amvm_pcg64 *out) {
  uint32_t ent[2];
  int ne = 0;
  ent[ne++] = (uint32_t)seed;
  if (seed >> 32) ent[ne++] = (uint32_t)(seed >> 32);
  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
  uint32_t words[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    words[i] = v;
  }
  uint64_t val[4];
  for (int i = 0; i < 4; ++i) val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
  typedef unsigned __int128 u128;
  const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
  const u128 initstate = ((u128)val[0] << 64) | val[1];
  const u128 initseq = ((u128)val[2] << 64) | val[3];
  u128 st = 0, inc = (initseq << 1) | 1u;
  st = st * mult + inc;
  st += initstate;
  st = st * mult + inc;
  out->state_hi = (uint64_t)(st >> 64);
  out->state_lo = (uint64_t)st;
  out->inc_hi = (uint64_t)(inc >> 64);
  out->inc_lo = (uint64_t)inc;
  out->has_uint32 = 0;
  out->uinteger = 0;
}
}  // namespace

// ---------------------------------------------------------------- planning
namespace {

struct Plan {
  int nt;
  size_t smem;
  int cr_smem, tab, cap;
  size_t slot_bytes;
  int64_t slots;
  size_t ist_bytes;  // per parked instance (chunked solve), 0 otherwise
  size_t icache_bytes;  // per instance impact-score cache (solve), 0 for ops
  int sparse, ktop;     // sparse engine (amvm_solve_sparse)
  int64_t fecap;        // sparse engine: column-indexed filter list capacity (0: off)
  int chunk_iters;
  size_t ws_bytes;
};

int64_t pow2ceil(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <int NT>
size_t smem_bytes(int64_t m, int64_t nlev, int cr_smem, int tab) {
  size_t s = sizeof(Shared<NT>) + 8 * ((nlev + 1) & ~1) + scratch_bytes<NT>(nlev, tab);
  if (cr_smem) s += 8 * m;
  return s;
}

template <int NT>
int occupancy(size_t smem, bool op, int *blocks, bool sp) {
  auto fn = op ? k_op<AMVM_NT> : (sp ? k_solve<NT, true> : k_solve<NT, false>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fn, NT, smem);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  return AMVM_OK;
}

// Two CTA sizes: 256 threads, 2 CTAs per SM (batches: more instances than
// SMs), and 512 threads, one CTA per SM with all its registers (at most as
// many instances as SMs: each instance's phases get twice the warps).
constexpr int kNtWide = 512;

size_t smem_for(int nt, int64_t m, int64_t nlev, int cr_smem, int tab) {
  return nt == kNtWide ? smem_bytes<kNtWide>(m, nlev, cr_smem, tab) : smem_bytes<AMVM_NT>(m, nlev, cr_smem, tab);
}

int occupancy_for(int nt, size_t smem, bool op, int *blocks, bool sp = false) {
  return nt == kNtWide ? occupancy<kNtWide>(smem, op, blocks, sp) : occupancy<AMVM_NT>(smem, op, blocks, sp);
}

constexpr size_t kSmemMax = 220 * 1024;
#ifndef AMVM_CHUNK_ITERS
#define AMVM_CHUNK_ITERS 1
#endif
constexpr int kChunkIters = AMVM_CHUNK_ITERS;  // chunked solve: ALNS iterations per task

int make_plan(const amvm_problem *p, const amvm_params *prm, bool op, Plan *P, int sparse = 0, int ktop = 0,
              int64_t max_row_nnz = 0) {
  if (!p || !prm) return AMVM_ERR_INVALID;
  P->sparse = sparse;
  P->ktop = ktop;
  // the filter rows' nonzeros, indexed by column (k_eps rows at most)
  P->fecap = (sparse && max_row_nnz > 0) ? std::min<int64_t>(prm->k_eps, p->m) * max_row_nnz : 0;
  if (P->fecap > ((int64_t)1 << 24)) P->fecap = 0;  // too many to index per slot: the general filter
  if (p->m < 1 || p->n < 1 || p->nlev < 1 || p->count < 1) return AMVM_ERR_INVALID;
  if (p->n > 0x7fffffff || p->m > 0x7fffffff) return AMVM_ERR_UNSUPPORTED;
  if (prm->r < 1 || prm->r > p->n || prm->k_eps < 1 || prm->max_iters < 0 || prm->refresh_period < 1 ||
      prm->n_segment < 1)
    return AMVM_ERR_INVALID;
  int sms = 0;
  if (!op) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return AMVM_ERR_NO_DEVICE;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return AMVM_ERR_CUDA;
  }
  int nt = prm->threads;
  if (nt == 0) nt = (!op && p->count <= sms) ? kNtWide : AMVM_NT;  // auto: a whole SM per instance when they fit
  if (nt != AMVM_NT && nt != kNtWide) return AMVM_ERR_UNSUPPORTED;
  if (op && nt != AMVM_NT) return AMVM_ERR_UNSUPPORTED;  // component calls: 256 threads
  P->nt = nt;
  P->tab = p->nlev <= kTabMaxLev;
#ifndef AMVM_CR_SMEM_MAX
#define AMVM_CR_SMEM_MAX (96 * 1024)
#endif
  P->cr_smem = p->m * 8 <= AMVM_CR_SMEM_MAX;
  const int64_t n = p->n;
  const int64_t maxc = prm->max_candidates;
  // swap-candidate survivor buffer: batches get room for 2x max_candidates
  // (C4/C5 keep < 100 per call); small batches (single instances) get room for
  // every pair up to 4M, which covers the filter's worst cases on tomography
  // (SURVEY.md §8a row 17); beyond it the call reports AMVM_ERR_UNSUPPORTED.
  const int64_t all_pairs = n * (n - 1) / 2;
  int64_t cap = maxc > 0 ? std::max<int64_t>(std::max<int64_t>(2 * maxc, maxc + n), 1024) : std::max<int64_t>(all_pairs, 1024);
  if (p->count <= 16) cap = std::max<int64_t>(cap, std::min<int64_t>(all_pairs, (int64_t)1 << 22));
  // sparse rows (tomography) let tens of thousands of pairs through the
  // filter: room for them, so a call sorts its survivors once instead of
  // taking the counting-pass overflow path (~20 enumerations)
  if (sparse) cap = std::max<int64_t>(cap, std::min<int64_t>(all_pairs, (int64_t)1 << 17));
  if (sparse && getenv("AMVM_SPARSE_CAP")) {  // test knob: a small buffer drives the overflow path
    const int64_t want = std::max<int64_t>(atoll(getenv("AMVM_SPARSE_CAP")), maxc + n);
    cap = std::max<int64_t>(want, 1024);
  }
  cap = pow2ceil(cap);
  if (cap > ((int64_t)1 << 30)) return AMVM_ERR_UNSUPPORTED;
  P->cap = (int)cap;
  P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
  if (P->smem > kSmemMax && P->cr_smem) {
    P->cr_smem = 0;
    P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
  }
  if (P->smem > kSmemMax && P->tab) {
    P->tab = 0;
    P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
  }
  if (P->smem > kSmemMax && nt == kNtWide && prm->threads == 0) {  // the wide CTA does not fit: 256 threads
    P->nt = nt = AMVM_NT;
    P->tab = p->nlev <= kTabMaxLev;
    P->cr_smem = p->m * 8 <= AMVM_CR_SMEM_MAX;
    P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
    if (P->smem > kSmemMax && P->cr_smem) {
      P->cr_smem = 0;
      P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
    }
    if (P->smem > kSmemMax && P->tab) {
      P->tab = 0;
      P->smem = smem_for(nt, p->m, p->nlev, P->cr_smem, P->tab);
    }
  }
  if (P->smem > kSmemMax) return AMVM_ERR_UNSUPPORTED;  // nlev too large for the smem level table
  const SlotLayout L = slot_layout(p->m, p->n, prm->k_eps, prm->r, cap, sparse ? ktop : 0, P->fecap);
  P->slot_bytes = al256(L.total);
  if (op) {
    P->slots = 1;
  } else {
    int blocks = 0;
    int rc = occupancy_for(nt, P->smem, false, &blocks, sparse != 0);
    if (rc) return rc;
    if (blocks < 1) return AMVM_ERR_UNSUPPORTED;
    P->slots = std::min<int64_t>(p->count, (int64_t)blocks * sms);
  }
  // more instances than resident CTAs: solve in chunks of kChunkIters
  // iterations so instances migrate between CTAs and the tail is one chunk
  P->chunk_iters = (!op && p->count > P->slots && prm->max_iters > kChunkIters) ? kChunkIters : 0;
  P->ist_bytes = P->chunk_iters ? inst_layout(p->m, p->n).total : 0;
  P->icache_bytes = op ? 0 : al256((size_t)8 * p->n);
  P->ws_bytes = sizeof(WsHeader) + ws_dense_bytes(p->m, p->n, sparse) +
                (size_t)P->slots * P->slot_bytes + (size_t)p->count * P->ist_bytes +
                (size_t)p->count * P->icache_bytes + (op ? 0 : al256((size_t)4 * p->count));
  return AMVM_OK;
}

int cuda_rc(cudaError_t e) { return e == cudaSuccess ? AMVM_OK : AMVM_ERR_CUDA; }

KArgs base_args(const amvm_problem *p, const amvm_params *prm, const Plan &P, void *ws) {
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.m = p->m; a.n = p->n; a.nlev = p->nlev; a.count = p->count;
  a.At = p->At; a.B = p->B; a.levels = p->levels;
  a.prm = *prm;
  a.ws = (unsigned char *)ws;
  a.slot_bytes = P.slot_bytes;
  a.chunk_iters = P.chunk_iters;
  a.ist_bytes = P.ist_bytes;
  a.sparse = P.sparse;
  a.ktop = P.ktop;
  a.fecap = P.fecap;
  if (!P.sparse) {  // the dense part: row-major Ar and the CSC copy (sparse: the caller's CSC / CSR)
    a.Ar = (const double *)(a.ws + sizeof(WsHeader));
    unsigned char *cb = a.ws + sizeof(WsHeader) + ws_ar_bytes(p->m, p->n);
    const CscLayout CL = csc_layout(p->m, p->n);
    a.cptr = (const int64_t *)(cb + CL.ptr);
    a.crow = (const int32_t *)(cb + CL.row);
    a.cval = (const double *)(cb + CL.val);
  }
  const size_t dense = ws_dense_bytes(p->m, p->n, P.sparse);
  a.ist = P.ist_bytes ? a.ws + sizeof(WsHeader) + dense + (size_t)P.slots * P.slot_bytes : nullptr;
  if (P.icache_bytes) {
    unsigned char *ib = a.ws + sizeof(WsHeader) + dense + (size_t)P.slots * P.slot_bytes +
                        (size_t)p->count * P.ist_bytes;
    a.icache = ib;
    a.icache_bytes = P.icache_bytes;
    a.ivalid = (int32_t *)(ib + (size_t)p->count * P.icache_bytes);
  }
  a.cr_smem = P.cr_smem; a.tab = P.tab; a.cap = P.cap;
  a.time_budget_ns = prm->time_limit_s < 0 ? -1 : (int64_t)(prm->time_limit_s * 1e9);
  return a;
}

int launch(const Plan &P, bool op, const KArgs &a, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(a.ws, 0, sizeof(WsHeader), st);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  if (a.ist) {  // progress = 0 for every parked instance
    e = cudaMemset2DAsync(a.ist, a.ist_bytes, 0, sizeof(InstState), (size_t)a.count, st);
    if (e != cudaSuccess) return AMVM_ERR_CUDA;
  }
  int blocks = 0;
  int rc = occupancy_for(P.nt, P.smem, op, &blocks, P.sparse != 0);  // also sets the smem attribute
  if (rc) return rc;
  if (!a.sparse) {  // row-major copy of A for the row gathers (filter rows, screening rows)
    const dim3 tg((unsigned)((a.n + 31) / 32), (unsigned)((a.m + 31) / 32)), tb(32, 8);
    k_transpose<<<tg, tb, 0, st>>>(a.At, (double *)a.Ar, a.m, a.n);
  }
  if (!a.sparse) {  // CSC copy for sparse A (sets the header's csc_ok when it fits)
    int64_t *cptr = (int64_t *)a.cptr;
    const unsigned cg = (unsigned)((a.n + 7) / 8);
    k_csc_count<<<cg, 256, 0, st>>>(a.At, a.m, a.n, cptr);
    k_csc_scan<<<1, 1024, 0, st>>>(cptr, a.n, csc_cap(a.m, a.n), (WsHeader *)a.ws);
    k_csc_fill<<<cg, 256, 0, st>>>(a.At, a.m, a.n, cptr, (int32_t *)a.crow, (double *)a.cval, (WsHeader *)a.ws);
  }
  const dim3 grid((unsigned)P.slots), block((unsigned)P.nt);
  if (op) k_op<AMVM_NT><<<grid, block, P.smem, st>>>(a);
  else if (P.nt == kNtWide && a.sparse) k_solve<kNtWide, true><<<grid, block, P.smem, st>>>(a);
  else if (P.nt == kNtWide) k_solve<kNtWide, false><<<grid, block, P.smem, st>>>(a);
  else if (a.sparse) k_solve<AMVM_NT, true><<<grid, block, P.smem, st>>>(a);
  else k_solve<AMVM_NT, false><<<grid, block, P.smem, st>>>(a);
  return cuda_rc(cudaGetLastError());
}

int run_op(const amvm_problem *prob, const amvm_params *prm, KArgs &a, void *ws, size_t ws_bytes,
           void *stream) {
  Plan P;
  amvm_problem one = *prob;
  one.count = 1;
  int rc = make_plan(&one, prm, true, &P);
  if (rc) return rc;
  if (!ws || ws_bytes < P.ws_bytes) return AMVM_ERR_WORKSPACE;
  KArgs b = base_args(&one, prm, P, ws);
  b.op = a.op; b.kind = a.kind;
  b.s_idx = a.s_idx; b.s_r = a.s_r; b.s_obj = a.s_obj; b.s_cnt = a.s_cnt; b.rng = a.rng;
  b.x_i = a.x_i; b.x_j = a.x_j; b.x_cnt = a.x_cnt; b.x_saved = a.x_saved; b.x_d = a.x_d;
  b.x_out4 = a.x_out4; b.x_cap = a.x_cap; b.x_r = a.x_r;
  return launch(P, true, b, (cudaStream_t)stream);
}

bool sol_ok(const amvm_solution *s) { return s && s->idx && s->residual && s->objective && s->updates; }

}  // namespace


// ================================================================== C-ABI
extern "C" {

int amvm_abi_version(void) { return AMVM_ABI_VERSION; }

const char *amvm_strerror(int status) {
  switch (status) {
    case AMVM_OK: return "ok";
    case AMVM_ERR_INVALID: return "invalid argument";
    case AMVM_ERR_CUDA: return "CUDA runtime error";
    case AMVM_ERR_WORKSPACE: return "workspace too small (see amvm_workspace_bytes)";
    case AMVM_ERR_UNSUPPORTED: return "problem shape outside this build's limits";
    case AMVM_ERR_NO_DEVICE: return "no usable sm_100 device";
    default: return "unknown status";
  }
}

size_t amvm_workspace_bytes(const amvm_problem *prob, const amvm_params *prm) {
  Plan P;
  if (make_plan(prob, prm, false, &P)) return 0;
  Plan Q;
  amvm_problem one = *prob;
  one.count = 1;
  if (make_plan(&one, prm, true, &Q)) return 0;
  return std::max(P.ws_bytes, Q.ws_bytes);
}

int amvm_solve(const amvm_problem *prob, const amvm_params *prm, const amvm_solution *start, amvm_pcg64 *rng,
               amvm_result *res, void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !prm || !sol_ok(start) || !rng || !res || !sol_ok(&res->best) || !res->initial_objective ||
      !res->iterations || !res->operator_uses)
    return AMVM_ERR_INVALID;
  if (!prob->At || !prob->B || !prob->levels) return AMVM_ERR_INVALID;
  Plan P;
  int rc = make_plan(prob, prm, false, &P);
  if (rc) return rc;
  if (!ws || ws_bytes < P.ws_bytes) return AMVM_ERR_WORKSPACE;
  KArgs a = base_args(prob, prm, P, ws);
  a.s_idx = start->idx; a.s_r = start->residual; a.s_obj = start->objective; a.s_cnt = start->updates;
  a.rng = rng;
  a.res = *res;
  return launch(P, false, a, (cudaStream_t)stream);
}

static int sparse_plan(const amvm_sparse_problem *sp, const amvm_params *prm, bool op, Plan *P,
                       amvm_problem *dense_view) {
  if (!sp || !prm || sp->m < 1 || sp->n < 1 || sp->nnz < 0 || sp->max_col_nnz < 0) return AMVM_ERR_INVALID;
  memset(dense_view, 0, sizeof(*dense_view));
  dense_view->m = sp->m; dense_view->n = sp->n; dense_view->nlev = sp->nlev; dense_view->count = sp->count;
  dense_view->B = sp->B; dense_view->levels = sp->levels;
  // the |s| top list must outlast the rows a column pair can touch
  int64_t ktop = 2 * sp->max_col_nnz + 1;
  if (ktop < 32) ktop = 32;
  if (ktop > sp->m) ktop = sp->m;
  if (ktop > 4096) return AMVM_ERR_UNSUPPORTED;  // rank-sorted on one CTA
  if (sp->max_row_nnz < 0) return AMVM_ERR_INVALID;
  return make_plan(dense_view, prm, op, P, 1, (int)ktop, sp->max_row_nnz);
}

size_t amvm_sparse_workspace_bytes(const amvm_sparse_problem *sp, const amvm_params *prm) {
  Plan P;
  amvm_problem dv;
  if (sparse_plan(sp, prm, false, &P, &dv)) return 0;
  return P.ws_bytes;
}

int amvm_solve_sparse(const amvm_sparse_problem *sp, const amvm_params *prm, const amvm_solution *start,
                      amvm_pcg64 *rng, amvm_result *res, void *ws, size_t ws_bytes, void *stream) {
  if (!sp || !prm || !sol_ok(start) || !rng || !res || !sol_ok(&res->best) || !res->initial_objective ||
      !res->iterations || !res->operator_uses)
    return AMVM_ERR_INVALID;
  if (!sp->cptr || !sp->crow || !sp->cval || !sp->rptr || !sp->rcol || !sp->rval || !sp->B || !sp->levels)
    return AMVM_ERR_INVALID;
  Plan P;
  amvm_problem dv;
  int rc = sparse_plan(sp, prm, false, &P, &dv);
  if (rc) return rc;
  if (!ws || ws_bytes < P.ws_bytes) return AMVM_ERR_WORKSPACE;
  KArgs a = base_args(&dv, prm, P, ws);
  a.cptr = sp->cptr; a.crow = sp->crow; a.cval = sp->cval;
  a.rptr = sp->rptr; a.rcol = sp->rcol; a.rval = sp->rval;
  a.s_idx = start->idx; a.s_r = start->residual; a.s_obj = start->objective; a.s_cnt = start->updates;
  a.rng = rng;
  a.res = *res;
  return launch(P, false, a, (cudaStream_t)stream);
}

int amvm_status(const void *ws, void *stream) {
  if (!ws) return AMVM_ERR_INVALID;
  if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return AMVM_ERR_CUDA;
  WsHeader h;
  if (cudaMemcpy(&h, ws, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return AMVM_ERR_CUDA;
  return h.status;
}

int amvm_one_opt(const amvm_problem *prob, const amvm_params *prm, amvm_solution *sol, void *ws,
                 size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol)) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_ONE_OPT;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_local_search(const amvm_problem *prob, const amvm_params *prm, amvm_solution *sol, void *ws,
                      size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol)) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_LOCAL_SEARCH;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_find_candidates(const amvm_problem *prob, const amvm_params *prm, const amvm_solution *sol,
                         int32_t *out_i, int32_t *out_j, double *out_delta, int32_t *count, int32_t cap,
                         void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol) || !out_i || !out_j || !out_delta || !count || cap < 0) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_FIND_CAND;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.x_i = out_i; a.x_j = out_j; a.x_d = out_delta; a.x_cnt = count; a.x_cap = cap;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_best_swap(const amvm_problem *prob, const amvm_params *prm, const amvm_solution *sol, double *out4,
                   void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol) || !out4) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_BEST_SWAP;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.x_out4 = out4;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_best_swap_l2(const amvm_problem *prob, const amvm_params *prm, const amvm_solution *sol, int32_t workers,
                      double *out4, void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol) || !out4 || workers < 1) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_BEST_SWAP;
  a.kind = workers;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.x_out4 = out4;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_apply_shift(const amvm_problem *prob, const amvm_params *prm, amvm_solution *sol, int64_t j,
                     int32_t new_level, void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !prm || !sol_ok(sol) || j < 0 || j >= prob->n || new_level < 0 || new_level >= prob->nlev)
    return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_APPLY_SHIFT;
  a.x_r = (int32_t)j;
  a.kind = new_level;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_apply_swap(const amvm_problem *prob, const amvm_params *prm, amvm_solution *sol, int64_t i, int64_t j,
                    void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !prm || !sol_ok(sol) || i == j || i < 0 || j < 0 || i >= prob->n || j >= prob->n)
    return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_APPLY_SWAP;
  a.x_r = (int32_t)i;
  a.kind = (int)j;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_accept(int64_t m, const double *cur_residual, const double *cur_objective, const double *cand_residual,
                const double *cand_objective, int32_t l2_tiebreak, double tie_tol, int32_t *verdict,
                void *stream) {
  if (m < 1 || !cur_residual || !cur_objective || !cand_residual || !cand_objective || !verdict)
    return AMVM_ERR_INVALID;
  k_accept<<<1, 64, 0, (cudaStream_t)stream>>>(m, cur_residual, cur_objective, cand_residual, cand_objective,
                                                l2_tiebreak, tie_tol, verdict);
  return cuda_rc(cudaGetLastError());
}

int amvm_select_operators(const amvm_bank *bank, amvm_pcg64 *rng, int32_t *pair, void *stream) {
  if (!bank || !rng || !pair) return AMVM_ERR_INVALID;
  k_bank_select<<<1, 1, 0, (cudaStream_t)stream>>>(bank, rng, pair);
  return cuda_rc(cudaGetLastError());
}

int amvm_update_weights(amvm_bank *bank, const amvm_params *prm, int32_t pair, int32_t outcome, void *stream) {
  if (!bank || !prm || pair < 0 || pair > 3 || outcome < 0 || outcome > 3 || prm->n_segment < 1)
    return AMVM_ERR_INVALID;
  k_bank_update<<<1, 1, 0, (cudaStream_t)stream>>>(bank, pair, outcome, prm->sigma1, prm->sigma2, prm->sigma3,
                                                    prm->weight_floor, prm->n_segment);
  return cuda_rc(cudaGetLastError());
}

int amvm_impact_scores(const amvm_problem *prob, const amvm_params *prm, const amvm_solution *sol, double *d,
                       void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol) || !d || prm->alpha < 0) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_IMPACT;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.x_d = d;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_destroy(const amvm_problem *prob, const amvm_params *prm, int kind, const amvm_solution *sol,
                 amvm_pcg64 *rng, int32_t *removed, void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !sol_ok(sol) || !rng || !removed || (kind != 0 && kind != 1)) return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_DESTROY;
  a.kind = kind;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.rng = rng;
  a.x_i = removed;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_repair(const amvm_problem *prob, const amvm_params *prm, int kind, amvm_solution *sol, amvm_pcg64 *rng,
                const int32_t *removed, const int32_t *saved_idx, int32_t r, void *ws, size_t ws_bytes,
                void *stream) {
  if (!prob || !sol_ok(sol) || !rng || !removed || !saved_idx || r < 0 || (kind != 0 && kind != 1) ||
      prob->nlev < 2)
    return AMVM_ERR_INVALID;
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.op = OP_REPAIR;
  a.kind = kind;
  a.s_idx = sol->idx; a.s_r = sol->residual; a.s_obj = sol->objective; a.s_cnt = sol->updates;
  a.rng = rng;
  a.x_i = const_cast<int32_t *>(removed);
  a.x_saved = const_cast<int32_t *>(saved_idx);
  a.x_r = r;
  return run_op(prob, prm, a, ws, ws_bytes, stream);
}

int amvm_compute_residual(const amvm_problem *prob, amvm_solution *sol, void *stream) {
  if (!prob || !sol_ok(sol) || !prob->At || !prob->B || !prob->levels) return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1 || prob->count < 1) return AMVM_ERR_INVALID;
  const int64_t blocks = (prob->count + kRI - 1) / kRI;
  const int64_t chunks = std::max<int64_t>(1, ((prob->m & ~(int64_t)3) + 255) / 256);
  cudaError_t e = cudaMemsetAsync(sol->objective, 0, sizeof(double) * prob->count, (cudaStream_t)stream);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  k_residual<256><<<dim3((unsigned)blocks, (unsigned)chunks), 256, 0, (cudaStream_t)stream>>>(
      prob->m, prob->n, prob->nlev, prob->count, prob->At, prob->B, prob->levels, sol->idx, nullptr,
      sol->residual, sol->objective);
  e = cudaGetLastError();
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  e = cudaMemsetAsync(sol->updates, 0, sizeof(int32_t) * prob->count, (cudaStream_t)stream);
  return cuda_rc(e);
}

int amvm_ptq_prepare(int64_t m, int64_t n, int64_t count, int64_t nlev, const double *At, const double *W,
                     double *B, double *levels, int32_t *idx, void *stream) {
  if (m < 1 || n < 1 || count < 1 || nlev < 1 || nlev > 1024 || !At || !W || !B || !levels || !idx)
    return AMVM_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  k_ptq_prepare<256><<<(unsigned)count, 256, 0, st>>>(n, nlev, W, levels, idx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  const int64_t blocks = (count + kRI - 1) / kRI;
  const int64_t chunks = std::max<int64_t>(1, ((m & ~(int64_t)3) + 255) / 256);
  k_residual<256><<<dim3((unsigned)blocks, (unsigned)chunks), 256, 0, st>>>(m, n, nlev, count, At, nullptr, levels,
                                                                            idx, W, B, nullptr);
  return cuda_rc(cudaGetLastError());
}

int amvm_seed_pcg64(const uint64_t *seeds_host, int64_t count, amvm_pcg64 *out_host) {
  if (!seeds_host || !out_host || count < 0) return AMVM_ERR_INVALID;
  for (int64_t k = 0; k < count; ++k) seed_pcg64(seeds_host[k], &out_host[k]);
  return AMVM_OK;
}

// ---- exact oracle: brute_force (oracle.py:38-111), see amvm_exact.cuh ----
}  // extern "C"

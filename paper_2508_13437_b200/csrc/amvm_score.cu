// amvm_score.cu — batched candidate-move scoring (include/amvm.h:
// amvm_score_moves / amvm_score_workspace_bytes), its own translation unit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "../../include/amvm.h"
#include "amvm_common.cuh"
#include "amvm_score.cuh"

using namespace amvm;

namespace {
template <int CB, int RT, int NC>
int launch_adj_rt(const amvm_problem *prob, const int32_t *idx, const double *residual, double *out_t, int64_t *best,
                  double *best_t, double *blk_t, int64_t *blk_i, unsigned *done, int G, cudaStream_t st) {
  const size_t smem = adj_smem_bytes(prob->m, CB, (prob->n + G - 1) / G, prob->nlev);
  // the attribute is raised once per instantiation and device (a driver call
  // per launch would dominate back-to-back launches of a ~14 us kernel)
  static int dev_ok[64];  // largest smem set so far, per device (0: none)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return AMVM_ERR_CUDA;
  if ((int)smem > dev_ok[dev]) {
    if (cudaFuncSetAttribute(k_score_adj<CB, RT, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return AMVM_ERR_CUDA;
    dev_ok[dev] = (int)smem;
  }
  // back-to-back scorer launches overlap one grid's tail with the next one's
  // column stream (programmatic dependent launch; AMVM_SCORE_PDL=0 disables)
  const char *pe = getenv("AMVM_SCORE_PDL");
  const bool pdl = !(pe && atoi(pe) == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(NC + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cuda_rc(cudaLaunchKernelEx(&cfg, k_score_adj<CB, RT, NC>, prob->m, prob->n, prob->nlev, prob->count,
                                    prob->At, prob->levels, idx, residual, out_t, blk_t, blk_i, done, best,
                                    best_t));
}

template <int CB, int NC>
int launch_adj_nc(const amvm_problem *prob, const int32_t *idx, const double *residual, double *out_t,
                  int64_t *best, double *best_t, double *blk_t, int64_t *blk_i, unsigned *done, int G,
                  cudaStream_t st) {
  const int64_t r = (prob->m + NC - 1) / NC;  // rows per consumer thread
  if (r <= 1) return launch_adj_rt<CB, 1, NC>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  if (r <= 2) return launch_adj_rt<CB, 2, NC>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  if (r <= 4) return launch_adj_rt<CB, 4, NC>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  if (r <= 8) return launch_adj_rt<CB, 8, NC>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  if (r <= 16)
    return launch_adj_rt<CB, 16, NC>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  return AMVM_ERR_UNSUPPORTED;
}

// consumer threads per CTA: 512, or 256 with AMVM_SCORE_THREADS=256 (A/B
// knob; 256 needs m <= 4096 to keep <= 16 rows per thread in registers)
template <int CB>
int launch_adj(const amvm_problem *prob, const int32_t *idx, const double *residual, double *out_t, int64_t *best,
               double *best_t, double *blk_t, int64_t *blk_i, unsigned *done, int G, cudaStream_t st) {
  const char *e = getenv("AMVM_SCORE_THREADS");
  if (e && atoi(e) == 256 && prob->m <= 256 * 16)
    return launch_adj_nc<CB, 256>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
  return launch_adj_nc<CB, 512>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, G, st);
}
}  // namespace

extern "C" {

size_t amvm_score_workspace_bytes(const amvm_problem *prob) {
  if (!prob || prob->n < 1 || prob->count < 1) return 0;
  const int cpb = score_cols_per_cta(1) < score_cols_per_cta(0) ? score_cols_per_cta(1) : score_cols_per_cta(0);
  size_t nblk = (size_t)((prob->n + cpb - 1) / cpb);  // the larger grid of the two k_score_moves modes
  if (nblk < kScoreMaxSlabs) nblk = kScoreMaxSlabs;     // k_score_adj: one slab per SM
  return (size_t)prob->count * (nblk * 16 + 4) + 16;
}


int amvm_score_moves(const amvm_problem *prob, const int32_t *idx, const double *residual, int mode,
                     double *out_t, int64_t *best, double *best_t, void *ws, size_t ws_bytes, void *stream) {
  if (!prob || !prob->At || !prob->levels || !idx || !residual || !out_t || (!best) != (!best_t))
    return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1 || prob->nlev < 1 || prob->count < 1 || (mode != 0 && mode != 1))
    return AMVM_ERR_INVALID;
  const int cpb = score_cols_per_cta(mode);
  if (prob->count > 65535 || (prob->n + cpb - 1) / cpb > 0x7fffffff) return AMVM_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < amvm_score_workspace_bytes(prob) || ((uintptr_t)ws & 7)) return AMVM_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  // workspace: per-CTA bests (t, flat) and one ticket counter per instance;
  // the counters must be zero before the first call on a workspace (the
  // kernels leave them zero), so there is no per-call memset
  size_t nslot = (size_t)((prob->n + score_cols_per_cta(1) - 1) / score_cols_per_cta(1));
  {
    const size_t n0 = (size_t)((prob->n + score_cols_per_cta(0) - 1) / score_cols_per_cta(0));
    if (n0 > nslot) nslot = n0;
    if (nslot < kScoreMaxSlabs) nslot = kScoreMaxSlabs;
  }
  double *blk_t = (double *)ws;
  int64_t *blk_i = (int64_t *)(blk_t + prob->count * nslot);
  unsigned *done = (unsigned *)(blk_i + prob->count * nslot);
  // adjacent set, even m <= 8192: the TMA-bulk streaming scorer, one CTA per SM
  if (mode == 1 && prob->m % 2 == 0 && prob->m <= (int64_t)kAdjThreads * kAdjMaxR) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return AMVM_ERR_CUDA;
    int cb = adj_cols_per_stage(prob->m);
    if (const char *e = getenv("AMVM_SCORE_CB")) {  // A/B knob: columns per ring stage
      const int v = atoi(e);
      if (v >= 1 && v <= 4 && adj_stages(prob->m, v) >= 2) cb = v;
    }
    int64_t G = sms < kScoreMaxSlabs ? sms : kScoreMaxSlabs;
    const int64_t slabs = (prob->n + cb - 1) / cb;  // every slab holds at least one column
    if (G > slabs) G = slabs;
    if (adj_stages(prob->m, cb) >= 2 && adj_smem_bytes(prob->m, cb, (prob->n + G - 1) / G, prob->nlev) <= 210 * 1024) {
      switch (cb) {
        case 1: return launch_adj<1>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, (int)G, st);
        case 2: return launch_adj<2>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, (int)G, st);
        case 3: return launch_adj<3>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, (int)G, st);
        default: return launch_adj<4>(prob, idx, residual, out_t, best, best_t, blk_t, blk_i, done, (int)G, st);
      }
    }
  }
  const int64_t nblk = (prob->n + cpb - 1) / cpb;
  const dim3 grid((unsigned)nblk, (unsigned)prob->count);
  if (mode == 1)
    k_score_moves<1><<<grid, 32 * kScoreWarps, 0, st>>>(prob->m, prob->n, prob->nlev, prob->count, prob->At,
                                                        prob->levels, idx, residual, out_t, blk_t, blk_i, done,
                                                        best, best_t);
  else
    k_score_moves<0><<<grid, 32 * kScoreWarps, 0, st>>>(prob->m, prob->n, prob->nlev, prob->count, prob->At,
                                                        prob->levels, idx, residual, out_t, blk_t, blk_i, done,
                                                        best, best_t);
  return cuda_rc(cudaGetLastError());
}

#ifdef AMVM_SCORE_TIMELINE
AMVM_API int amvm_debug_score_timeline(unsigned long long *host, int n) {
  return cuda_rc(cudaMemcpyFromSymbol(host, g_adj_tl, sizeof(unsigned long long) * 8 * n));
}
AMVM_API int amvm_debug_score_stages(unsigned long long *host, int n) {
  return cuda_rc(cudaMemcpyFromSymbol(host, g_adj_st, sizeof(unsigned long long) * 32 * n));
}
#endif
}  // extern "C"

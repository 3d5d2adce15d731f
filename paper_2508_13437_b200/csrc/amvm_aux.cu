// amvm_aux.cu — the off-path entry points of include/amvm.h in their own
// translation unit: exact oracle (brute_force), swap checks, device
// least-squares start, tomography projector / projections / SIRT.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "../../include/amvm.h"
#include "amvm_common.cuh"
#include "amvm_exact.cuh"
#include "amvm_lsq.cuh"
#include "amvm_tomo.cuh"

using namespace amvm;

extern "C" {

static int bf_shape(const amvm_problem *prob, long long *total, int *blocks) {
  if (!prob || !prob->At || !prob->B || !prob->levels) return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1 || prob->nlev < 1 || prob->count != 1) return AMVM_ERR_INVALID;
  if (prob->n > kBFMaxN) return AMVM_ERR_UNSUPPORTED;
  long long t = 1;
  for (int64_t j = 0; j < prob->n; ++j) {
    if (t > (long long)(0x3fffffffffffffffLL / prob->nlev)) return AMVM_ERR_UNSUPPORTED;
    t *= prob->nlev;
  }
  *total = t;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long per = 256;
  long long want = (t + per - 1) / per;
  const long long cap = (long long)sms * 8;  // 8 resident 256-thread CTAs per SM
  *blocks = (int)std::max(1LL, std::min(want, cap));
  return AMVM_OK;
}

size_t amvm_brute_force_workspace_bytes(const amvm_problem *prob) {
  long long total;
  int blocks;
  if (bf_shape(prob, &total, &blocks)) return 0;
  return 64 + (size_t)blocks * 16;
}

int amvm_brute_force(const amvm_problem *prob, int order, int32_t *best_idx, double *best_t, int64_t *best_code,
                     void *ws, size_t ws_bytes, void *stream) {
  if (!best_idx || !best_t || (order != 0 && order != 1)) return AMVM_ERR_INVALID;
  long long total;
  int blocks;
  int rc = bf_shape(prob, &total, &blocks);
  if (rc) return rc;
  if (!ws || ws_bytes < 64 + (size_t)blocks * 16) return AMVM_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char *w = (char *)ws;
  unsigned long long *gbest = (unsigned long long *)w;
  double *blk_t = (double *)(w + 64);
  long long *blk_c = (long long *)(w + 64 + (size_t)blocks * 8);
  const unsigned long long inf_bits = 0x7ff0000000000000ULL;
  cudaError_t e = cudaMemcpyAsync(gbest, &inf_bits, sizeof(inf_bits), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  const int64_t m = prob->m, n = prob->n, nlev = prob->nlev;
  size_t smem = sizeof(double) * (size_t)(nlev + m);
  const size_t full = smem + sizeof(double) * (size_t)(m * n);
  const size_t limit = 200 * 1024;
  int staged = full <= limit;
  if (staged) smem = full;
  if (smem > limit) return AMVM_ERR_UNSUPPORTED;  // b + levels alone exceed shared memory
  e = cudaFuncSetAttribute(k_brute_force<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  k_brute_force<256><<<blocks, 256, smem, st>>>(m, (int)n, (int)nlev, total, order, staged, prob->At, prob->B,
                                                prob->levels, gbest, blk_t, blk_c);
  e = cudaGetLastError();
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  k_brute_force_final<256><<<1, 256, 0, st>>>(blocks, (int)n, (int)nlev, blk_t, blk_c, best_idx, best_t,
                                               best_code);
  return cuda_rc(cudaGetLastError());
}

// ---- device warm start: initial_solution's least-squares start (amvm_lsq.cuh) ----
size_t amvm_ls_start_workspace_bytes(int64_t m, int64_t n) {
  if (m < 1 || n < 1) return 0;
  return 256 + (size_t)n * (size_t)n * sizeof(double) + (size_t)n * sizeof(double);
}

int amvm_ls_start(const amvm_problem *prob, int32_t *idx, double *target, int32_t *flag, void *ws,
                  size_t ws_bytes, void *stream) {
  if (!prob || !prob->At || !prob->B || !prob->levels || !idx || !flag) return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1 || prob->nlev < 1 || prob->count != 1) return AMVM_ERR_INVALID;
  const int64_t m = prob->m, n = prob->n;
  if (!ws || ws_bytes < amvm_ls_start_workspace_bytes(m, n)) return AMVM_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  double *G = (double *)((char *)ws + 256);
  double *y = G + n * n;
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  const int64_t tiles = (n + kLsT - 1) / kLsT;
  k_gram<<<dim3((unsigned)tiles, (unsigned)tiles), 256, 0, st>>>(m, n, prob->At, G);
  k_atb<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(m, n, prob->At, prob->B, y);
  for (int64_t k = 0; k + 1 < n; ++k) {
    const unsigned g = (unsigned)((n - k - 1 + 15) / 16);
    k_chol_step<<<dim3(g, g), 256, 0, st>>>(n, k, G, flag);
  }
  // the last pivot is only checked (no trailing matrix)
  k_chol_step<<<dim3(1, 1), 256, 0, st>>>(n, n - 1, G, flag);
  k_chol_solve<1024><<<1, 1024, 0, st>>>(n, prob->nlev, G, y, prob->levels, target, idx, flag);
  return cuda_rc(cudaGetLastError());
}

// ---- tomography front end: parallel-beam projector as CSR (amvm_tomo.cuh) ----
size_t amvm_projector_workspace_bytes(int64_t side, int64_t n_angles) {
  if (side < 1 || n_angles < 1) return 0;
  return (size_t)(side * n_angles) * sizeof(int64_t);
}

int amvm_projector_indptr(int64_t side, int64_t n_angles, const double *dirs, int64_t *indptr, void *ws,
                          size_t ws_bytes, void *stream) {
  if (side < 1 || n_angles < 1 || !dirs || !indptr) return AMVM_ERR_INVALID;
  if (side > (1LL << 20)) return AMVM_ERR_UNSUPPORTED;
  if (!ws || ws_bytes < amvm_projector_workspace_bytes(side, n_angles)) return AMVM_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = side * n_angles;
  k_proj_count<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(side, n_angles, dirs, (int64_t *)ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  k_proj_scan<1024><<<1, 1024, 0, st>>>(rows, (const int64_t *)ws, indptr);
  return cuda_rc(cudaGetLastError());
}

int amvm_projector_fill(int64_t side, int64_t n_angles, const double *dirs, const int64_t *indptr,
                        int64_t *indices, double *values, void *stream) {
  if (side < 1 || n_angles < 1 || !dirs || !indptr || !indices || !values) return AMVM_ERR_INVALID;
  const int64_t rows = side * n_angles;
  k_proj_fill<<<(unsigned)((rows + 127) / 128), 128, 0, (cudaStream_t)stream>>>(side, n_angles, dirs, indptr,
                                                                                indices, values);
  return cuda_rc(cudaGetLastError());
}

// ---- tomography front end: projections and SIRT (amvm_tomo.cuh) ----
int amvm_csr_gemv(int64_t m, int64_t n, int64_t S, const int64_t *indptr, const int64_t *cols, const double *vals,
                  const double *X, const double *noise, double *out, void *stream) {
  if (m < 1 || n < 1 || S < 1 || !indptr || !cols || !vals || !X || !out) return AMVM_ERR_INVALID;
  const int64_t t = m * S;
  k_csr_gemv_t<<<(unsigned)((t + 255) / 256), 256, 0, (cudaStream_t)stream>>>(m, n, S, indptr, cols, vals, X,
                                                                              noise, out);
  return cuda_rc(cudaGetLastError());
}

static size_t sirt_layout(int64_t m, int64_t n, int64_t nnz, int64_t S, size_t off[8]) {
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~(size_t)255; return r; };
  off[0] = take(sizeof(int64_t) * (size_t)n);        // column counts
  off[1] = take(sizeof(int64_t) * (size_t)(n + 1));  // cptr
  off[2] = take(sizeof(int64_t) * (size_t)n);        // fill positions
  off[3] = take(sizeof(int64_t) * (size_t)nnz);      // CSC rows
  off[4] = take(sizeof(double) * (size_t)nnz);       // CSC values
  off[5] = take(sizeof(double) * (size_t)m);         // R
  off[6] = take(sizeof(double) * (size_t)n);         // C
  off[7] = take(sizeof(double) * (size_t)(m * S));   // R (b - A x)
  return o;
}

size_t amvm_sirt_workspace_bytes(int64_t m, int64_t n, int64_t nnz, int64_t S) {
  if (m < 1 || n < 1 || nnz < 0 || S < 1) return 0;
  size_t off[8];
  return sirt_layout(m, n, nnz, S, off);
}

int amvm_sirt(int64_t m, int64_t n, int64_t nnz, int64_t S, const int64_t *indptr, const int64_t *cols,
              const double *vals, const double *B, int32_t iters, double lo, double hi, int clamp, double *X,
              void *ws, size_t ws_bytes, void *stream) {
  if (m < 1 || n < 1 || nnz < 0 || S < 1 || iters < 0 || !indptr || !cols || !vals || !B || !X)
    return AMVM_ERR_INVALID;
  size_t off[8];
  const size_t need = sirt_layout(m, n, nnz, S, off);
  if (!ws || ws_bytes < need) return AMVM_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char *w = (char *)ws;
  int64_t *ccnt = (int64_t *)(w + off[0]), *cptr = (int64_t *)(w + off[1]), *fpos = (int64_t *)(w + off[2]);
  int64_t *crow = (int64_t *)(w + off[3]);
  double *cval = (double *)(w + off[4]), *R = (double *)(w + off[5]), *Cw = (double *)(w + off[6]);
  double *Rres = (double *)(w + off[7]);
  cudaError_t e = cudaMemsetAsync(ccnt, 0, sizeof(int64_t) * n, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(fpos, 0, sizeof(int64_t) * n, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(X, 0, sizeof(double) * n * S, st);  // x = 0
  if (e != cudaSuccess) return AMVM_ERR_CUDA;
  if (nnz > 0) k_csr_colcount<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(nnz, cols, ccnt);
  k_proj_scan<1024><<<1, 1024, 0, st>>>(n, ccnt, cptr);
  k_csr_to_csc<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, indptr, cols, vals, cptr, fpos, crow, cval);
  k_csc_sort<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, cptr, crow, cval);
  const int64_t mx = m > n ? m : n;
  k_sirt_weights<<<(unsigned)((mx + 255) / 256), 256, 0, st>>>(m, n, indptr, vals, cptr, cval, R, Cw);
  for (int32_t it = 0; it < iters; ++it) {
    k_sirt_rows<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(m, S, indptr, cols, vals, R, B, X, Rres);
    k_sirt_cols<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, S, cptr, crow, cval, Cw, Rres, lo, hi, clamp, X);
  }
  return cuda_rc(cudaGetLastError());
}

// ---- verification kernels: is_improving, exhaustive_swap_check (amvm_exact.cuh) ----
int amvm_is_improving(const amvm_problem *prob, const double *residual, double objective, int64_t nc,
                      const int32_t *ci, const int32_t *cj, const double *cd, int32_t *verdict, void *stream) {
  if (!prob || !prob->At || !residual || nc < 0 || (nc > 0 && (!ci || !cj || !cd || !verdict)))
    return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1) return AMVM_ERR_INVALID;
  if (nc == 0) return AMVM_OK;
  k_is_improving<<<(unsigned)((nc + 7) / 8), 256, 0, (cudaStream_t)stream>>>(prob->m, prob->At, residual, objective,
                                                                             nc, ci, cj, cd, verdict);
  return cuda_rc(cudaGetLastError());
}

int amvm_swap_check(const amvm_problem *prob, const int32_t *idx, const double *residual, double objective,
                    double *out_t, int32_t *out_v, void *stream) {
  if (!prob || !prob->At || !prob->B || !prob->levels || !idx || !residual || !out_t || !out_v)
    return AMVM_ERR_INVALID;
  if (prob->m < 1 || prob->n < 1 || prob->count != 1) return AMVM_ERR_INVALID;
  if (prob->n > 4096) return AMVM_ERR_UNSUPPORTED;
  k_swap_check<<<(unsigned)(prob->n * prob->n), 256, 0, (cudaStream_t)stream>>>(
      prob->m, prob->n, prob->At, prob->B, prob->levels, idx, residual, objective, out_t, out_v);
  return cuda_rc(cudaGetLastError());
}

}  // extern "C"

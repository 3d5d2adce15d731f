// amvm_tomo.cuh — the parallel-beam projector of the tomography front end
// (C3), built on the device as CSR: the reference's parallel_beam_matrix /
// _ray_weights (/root/reference/pkg/src/dmmv/builders.py:186-239), bit for
// bit (same IEEE operations in the same order; -fmad=false).
//
// One thread per ray (angle a, detector o).  The reference collects every
// crossing tau of the ray with the 2(side+1) grid lines strictly inside
// (t_lo, t_hi), sorts and de-duplicates them (np.unique), and turns each gap
// into (pixel of the midpoint, length).  The crossings of one axis are
// monotone in the grid index, so the thread merges the two axes' sequences
// on the fly (O(side), no sort, no storage).  Along a ray both the pixel row
// and column are monotone (correctly rounded ops preserve monotonicity), so
// a pixel can only repeat in consecutive segments: repeats are summed in
// order (np.add.at), then the ray's entries are put in ascending pixel order
// by reversing the whole list when rows descend and each equal-row run when
// columns descend.  Two launches: count per ray (then an exclusive scan in
// one CTA), fill.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace amvm {

struct RaySeg {
  double half, px, py, dx, dy, tlo, thi;
  bool ax0, ax1;  // axis is not parallel to the ray (|d| > eps)
  bool hit;
};

__device__ __forceinline__ RaySeg ray_setup(int64_t side, double o, const double *__restrict__ dir4) {
  // dir4 = (cos, sin, -sin, cos) of the angle (host numpy, builders.py:234-235)
  RaySeg R;
  const double eps = 1e-12;  // builders.py:195
  R.half = (double)side / 2.0;
  R.px = __dmul_rn(o, dir4[0]);
  R.py = __dmul_rn(o, dir4[1]);
  R.dx = dir4[2];
  R.dy = dir4[3];
  double tlo = -__longlong_as_double(0x7ff0000000000000LL), thi = __longlong_as_double(0x7ff0000000000000LL);
  R.hit = true;
  R.ax0 = fabs(R.dx) > eps;
  R.ax1 = fabs(R.dy) > eps;
  for (int ax = 0; ax < 2; ++ax) {
    const double d = ax ? R.dy : R.dx, p = ax ? R.py : R.px;
    if (ax ? R.ax1 : R.ax0) {
      const double t0 = __ddiv_rn(__dsub_rn(-R.half, p), d);
      const double t1 = __ddiv_rn(__dsub_rn(R.half, p), d);
      tlo = fmax(tlo, fmin(t0, t1));
      thi = fmin(thi, fmax(t0, t1));
    } else if (!(-R.half <= p && p <= R.half)) {
      R.hit = false;
    }
  }
  if (!(thi > tlo)) R.hit = false;
  R.tlo = tlo;
  R.thi = thi;
  return R;
}

// Crossing k of one axis, walked in increasing tau: (-half + k - p) / d
// (builders.py:211), k ascending when d > 0, descending when d < 0.
struct AxisWalk {
  double p, d, half;
  int64_t k, step, end;  // current index, +-1, one past the last
  bool on;
  __device__ double val() const { return __ddiv_rn(__dsub_rn(__dadd_rn(-half, (double)k), p), d); }
};

__device__ __forceinline__ AxisWalk axis_walk(const RaySeg &R, int ax, int64_t side) {
  AxisWalk w;
  w.p = ax ? R.py : R.px;
  w.d = ax ? R.dy : R.dx;
  w.half = R.half;
  w.on = ax ? R.ax1 : R.ax0;
  if (w.d > 0) { w.k = 0; w.step = 1; w.end = side + 1; }
  else { w.k = side; w.step = -1; w.end = -1; }
  // skip crossings <= t_lo (the filter keeps t_lo < tau < t_hi)
  while (w.on && w.k != w.end && !(w.val() > R.tlo)) w.k += w.step;
  return w;
}

// Visits the merged, de-duplicated segments of one ray in increasing tau;
// `emit(pixel, length)` per kept segment (length > eps).
template <class F>
__device__ void ray_walk(const RaySeg &R, int64_t side, F &&emit) {
  if (!R.hit) return;
  const double eps = 1e-12;
  AxisWalk a = axis_walk(R, 0, side), b = axis_walk(R, 1, side);
  double prev = R.tlo;
  for (;;) {
    const bool ha = a.on && a.k != a.end && a.val() < R.thi;
    const bool hb = b.on && b.k != b.end && b.val() < R.thi;
    double next;
    if (ha && hb) {
      const double va = a.val(), vb = b.val();
      next = va < vb ? va : vb;
      if (va <= next) a.k += a.step;
      if (vb <= next) b.k += b.step;
    } else if (ha) {
      next = a.val();
      a.k += a.step;
    } else if (hb) {
      next = b.val();
      b.k += b.step;
    } else {
      next = R.thi;
    }
    if (next > prev) {  // np.unique: equal crossings are one
      const double len = __dsub_rn(next, prev);
      const double mid = __dadd_rn(prev, __ddiv_rn(len, 2.0));
      const double mx = __dadd_rn(R.px, __dmul_rn(mid, R.dx));
      const double my = __dadd_rn(R.py, __dmul_rn(mid, R.dy));
      double fc = floor(__dadd_rn(mx, R.half)), fr = floor(__dsub_rn(R.half, my));
      int64_t col = (int64_t)fc, row = (int64_t)fr;
      col = col < 0 ? 0 : (col > side - 1 ? side - 1 : col);
      row = row < 0 ? 0 : (row > side - 1 ? side - 1 : row);
      if (len > eps) emit(row * side + col, len);
      prev = next;
    }
    if (!ha && !hb) break;
  }
}

__device__ __forceinline__ double ray_offset(int64_t side, int64_t det) {
  return __dsub_rn((double)det, __ddiv_rn((double)(side - 1), 2.0));  // np.arange(side) - (side-1)/2.0
}

__global__ void __launch_bounds__(128) k_proj_count(int64_t side, int64_t n_angles, const double *__restrict__ dirs,
                                                    int64_t *__restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (r >= side * n_angles) return;
  const int64_t a = r / side, det = r - a * side;
  const RaySeg R = ray_setup(side, ray_offset(side, det), dirs + 4 * a);
  int64_t c = 0, last = -1;
  ray_walk(R, side, [&](int64_t pix, double) {
    if (pix != last) ++c;
    last = pix;
  });
  cnt[r] = c;
}

// exclusive scan of cnt[0..rows) into indptr[0..rows] (one CTA)
template <int NTB>
__global__ void __launch_bounds__(NTB) k_proj_scan(int64_t rows, const int64_t *__restrict__ cnt,
                                                    int64_t *__restrict__ indptr) {
  __shared__ int64_t part[NTB];
  const int64_t per = (rows + NTB - 1) / NTB;
  const int64_t lo = threadIdx.x * per, hi = lo + per < rows ? lo + per : rows;
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += cnt[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int k = 0; k < NTB; ++k) {
      const int64_t v = part[k];
      part[k] = acc;
      acc += v;
    }
    indptr[rows] = acc;
  }
  __syncthreads();
  int64_t acc = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    indptr[i] = acc;
    acc += cnt[i];
  }
}

__global__ void __launch_bounds__(128) k_proj_fill(int64_t side, int64_t n_angles, const double *__restrict__ dirs,
                                                   const int64_t *__restrict__ indptr, int64_t *__restrict__ idx,
                                                   double *__restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (r >= side * n_angles) return;
  const int64_t a = r / side, det = r - a * side;
  const RaySeg R = ray_setup(side, ray_offset(side, det), dirs + 4 * a);
  const int64_t base = indptr[r], cnt = indptr[r + 1] - base;
  int64_t c = 0, last = -1;
  ray_walk(R, side, [&](int64_t pix, double len) {
    if (pix == last) {
      val[base + c - 1] = __dadd_rn(val[base + c - 1], len);  // np.add.at, in order
    } else {
      idx[base + c] = pix;
      val[base + c] = len;
      ++c;
    }
    last = pix;
  });
  if (cnt < 2) return;
  auto rev = [&](int64_t lo, int64_t hi) {  // [lo, hi)
    for (--hi; lo < hi; ++lo, --hi) {
      const int64_t ti = idx[base + lo]; idx[base + lo] = idx[base + hi]; idx[base + hi] = ti;
      const double tv = val[base + lo]; val[base + lo] = val[base + hi]; val[base + hi] = tv;
    }
  };
  if (idx[base] / side > idx[base + cnt - 1] / side) rev(0, cnt);  // rows descend along the ray
  for (int64_t s = 0; s < cnt;) {
    const int64_t row = idx[base + s] / side;
    int64_t e = s + 1;
    while (e < cnt && idx[base + e] / side == row) ++e;
    if (e - s > 1 && idx[base + s] > idx[base + e - 1]) rev(s, e);
    s = e;
  }
}

}  // namespace amvm

// ===================================================== projections and SIRT
// b = A @ truth (builders.py:322) in numpy's dense dgemv_t order, from the
// CSR rows: the dense kernel sums K & -4 columns in blocks of 2048 with the
// output row's kernel (kind 4: four FMA lanes by column mod 4, folded
// (l0+l2)+(l1+l3); kind 2: two mul+add lanes; kind 1: two mul+add pairs),
// each block added to y, then the K & 3 leftover.  Zero entries add exact
// zeros, so visiting only the nonzeros, in column order, reproduces the
// dense result bit for bit.  Thread per (row, slice); X is n x S.
namespace amvm {
__device__ double csr_gemv_t_row(const int64_t *__restrict__ cols, const double *__restrict__ vals, int64_t lo,
                                 int64_t hi, const double *__restrict__ X, int64_t S, int64_t s, int64_t K,
                                 int kind) {
  const int64_t m1 = K & -4;
  double y = 0.0, l[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t blk = 0;
  auto fold = [&]() {
    double t;
    if (kind == 4) t = __dadd_rn(__dadd_rn(l[0], l[2]), __dadd_rn(l[1], l[3]));
    else if (kind == 2) t = __dadd_rn(l[0], l[1]);
    else t = __dadd_rn(__dadd_rn(l[0], l[2]), __dadd_rn(l[1], l[3]));  // (u0+v0)+(u1+v1)
    y = __dadd_rn(y, t);
    l[0] = l[1] = l[2] = l[3] = 0.0;
  };
  int64_t e = lo;
  for (; e < hi && cols[e] < m1; ++e) {
    const int64_t j = cols[e];
    const int64_t b = j >> 11;  // 2048-column block
    while (blk < b) { fold(); ++blk; }
    const double p = X[j * S + s];
    if (kind == 4) l[j & 3] = __fma_rn(vals[e], p, l[j & 3]);
    else if (kind == 2) l[j & 1] = __dadd_rn(l[j & 1], __dmul_rn(vals[e], p));
    else l[j & 3] = __dadd_rn(l[j & 3], __dmul_rn(vals[e], p));  // u0,u1,v0,v1 = lanes 0,1,2,3
  }
  if (m1 > 0) {
    const int64_t nb = (m1 + 2047) >> 11;
    while (blk < nb) { fold(); ++blk; }
  }
  // K & 3 leftover (scalar, compiler-contracted in OpenBLAS)
  double a[3] = {0.0, 0.0, 0.0};
  for (; e < hi; ++e) a[cols[e] - m1] = vals[e];
  double x3[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < (int)(K & 3); ++q) x3[q] = X[(m1 + q) * S + s];
  switch (K & 3) {
    case 1: y = __fma_rn(a[0], x3[0], y); break;
    case 2: y = __dadd_rn(y, __fma_rn(a[0], x3[0], __dmul_rn(a[1], x3[1]))); break;
    case 3: y = __dadd_rn(y, __fma_rn(a[2], x3[2], __fma_rn(a[0], x3[0], __dmul_rn(a[1], x3[1])))); break;
    default: break;
  }
  return y;
}

// out[i*S + s] = (A @ X[:, s])_i (+ noise[s*m + i] when noise != NULL,
// builders.py:322: `A @ truth + rng.uniform(...)`)
__global__ void __launch_bounds__(256) k_csr_gemv_t(int64_t m, int64_t n, int64_t S, const int64_t *__restrict__ indptr,
                                                    const int64_t *__restrict__ cols, const double *__restrict__ vals,
                                                    const double *__restrict__ X, const double *__restrict__ noise,
                                                    double *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= m * S) return;
  const int64_t i = t / S, s = t - i * S;
  const int kind = gemv_kind(i, m);
  double y = csr_gemv_t_row(cols, vals, indptr[i], indptr[i + 1], X, S, s, n, kind);
  if (noise) y = __dadd_rn(y, noise[s * m + i]);
  out[s * m + i] = y;
}

// ---- CSC copy of the CSR matrix (columns in ascending row order) ----------
__global__ void k_csr_colcount(int64_t nnz, const int64_t *__restrict__ cols, int64_t *__restrict__ cnt) {
  const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (e < nnz) atomicAdd((unsigned long long *)&cnt[cols[e]], 1ull);
}

__global__ void k_csr_to_csc(int64_t m, const int64_t *__restrict__ indptr, const int64_t *__restrict__ cols,
                             const double *__restrict__ vals, const int64_t *__restrict__ cptr,
                             int64_t *__restrict__ fillpos, int64_t *__restrict__ rows, double *__restrict__ cvals) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= m) return;
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
    const int64_t j = cols[e];
    const int64_t p = cptr[j] + (int64_t)atomicAdd((unsigned long long *)&fillpos[j], 1ull);
    rows[p] = i;
    cvals[p] = vals[e];
  }
}

// insertion sort of each column by row (atomics placed them in any order)
__global__ void k_csc_sort(int64_t n, const int64_t *__restrict__ cptr, int64_t *__restrict__ rows,
                           double *__restrict__ cvals) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (j >= n) return;
  const int64_t lo = cptr[j], hi = cptr[j + 1];
  for (int64_t a = lo + 1; a < hi; ++a) {
    const int64_t r = rows[a];
    const double v = cvals[a];
    int64_t b = a - 1;
    while (b >= lo && rows[b] > r) {
      rows[b + 1] = rows[b];
      cvals[b + 1] = cvals[b];
      --b;
    }
    rows[b + 1] = r;
    cvals[b + 1] = v;
  }
}

// ---- SIRT (builders.py:242-274), S right-hand sides: B is S x m, X n x S --
// rowsum / colsum in storage order; R = 1/rowsum (live rows), C = 1/colsum
// (0 for empty columns).
__global__ void k_sirt_weights(int64_t m, int64_t n, const int64_t *__restrict__ indptr,
                               const double *__restrict__ vals, const int64_t *__restrict__ cptr,
                               const double *__restrict__ cvals, double *__restrict__ R, double *__restrict__ Cw) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t < m) {
    double s = 0.0;
    for (int64_t e = indptr[t]; e < indptr[t + 1]; ++e) s = __dadd_rn(s, vals[e]);
    R[t] = s > 0.0 ? __ddiv_rn(1.0, s) : 0.0;
  }
  if (t < n) {
    double s = 0.0;
    for (int64_t e = cptr[t]; e < cptr[t + 1]; ++e) s = __dadd_rn(s, cvals[e]);
    Cw[t] = s > 0.0 ? __ddiv_rn(1.0, s) : 0.0;
  }
}

// Rres[i][s] = R_i (b_is - (A x_s)_i), warp per row, lanes over slices.
__global__ void __launch_bounds__(256) k_sirt_rows(int64_t m, int64_t S, const int64_t *__restrict__ indptr,
                                                   const int64_t *__restrict__ cols, const double *__restrict__ vals,
                                                   const double *__restrict__ R, const double *__restrict__ B,
                                                   const double *__restrict__ X, double *__restrict__ Rres) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= m) return;
  const int64_t lo = indptr[i], hi = indptr[i + 1];
  const double ri = R[i];
  for (int64_t s = lane; s < S; s += 32) {
    double ax = 0.0;
    for (int64_t e = lo; e < hi; ++e) ax = __fma_rn(vals[e], X[cols[e] * S + s], ax);
    Rres[i * S + s] = ri > 0.0 ? __dmul_rn(ri, __dsub_rn(B[s * m + i], ax)) : 0.0;
  }
}

// x_js = clip(x_js + C_j (A^T r_s)_j, lo, hi), warp per column.
__global__ void __launch_bounds__(256) k_sirt_cols(int64_t n, int64_t S, const int64_t *__restrict__ cptr,
                                                   const int64_t *__restrict__ rows, const double *__restrict__ cvals,
                                                   const double *__restrict__ Cw, const double *__restrict__ Rres,
                                                   double lo, double hi, int clamp, double *__restrict__ X) {
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int64_t a = cptr[j], b = cptr[j + 1];
  const double cj = Cw[j];
  for (int64_t s = lane; s < S; s += 32) {
    double g = 0.0;
    for (int64_t e = a; e < b; ++e) g = __fma_rn(cvals[e], Rres[rows[e] * S + s], g);
    double x = __dadd_rn(X[j * S + s], __dmul_rn(cj, g));
    if (clamp) x = fmin(fmax(x, lo), hi);
    X[j * S + s] = x;
  }
}
}  // namespace amvm

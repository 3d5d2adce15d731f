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

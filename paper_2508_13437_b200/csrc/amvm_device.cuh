// amvm_device.cuh — device primitives for the AMVM engine (sm_100a).
//
// Everything here reproduces a piece of numpy/OpenBLAS arithmetic that the
// reference's decisions depend on, written for the GPU:
//   * PCG64 + the numpy Generator draws the path consumes,
//   * numpy's pairwise 1-d sum, block-parallel over its fixed leaf tree,
//   * OpenBLAS SkylakeX ddot (np.linalg.norm) and dgemv_t (A @ x) orders,
//   * warp/block max reductions (max is exact, so any order is bitwise).
// All residual arithmetic uses explicit __dmul_rn/__dadd_rn so no FMA
// contraction can change a bit (the library is also built -fmad=false).
#pragma once

#include <cstdint>

#include "../../include/amvm.h"

#define AMVM_FULL 0xffffffffu

namespace amvm {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// ------------------------------------------------------------------ PCG64
// numpy/random/src/pcg64/pcg64.h: 128-bit LCG, XSL-RR, advance then output;
// next_uint32 hands out the low half first and buffers the high half.
struct Pcg {
  unsigned __int128 s, inc;
  uint32_t has32, u32;
};

__device__ __forceinline__ uint64_t pcg_next64(Pcg &g) {
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | (unsigned __int128)0x4385DF649FCCF645ULL;
  g.s = g.s * mult + g.inc;
  uint64_t hi = (uint64_t)(g.s >> 64), lo = (uint64_t)g.s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg_next32(Pcg &g) {
  if (g.has32) {
    g.has32 = 0;
    return g.u32;
  }
  uint64_t v = pcg_next64(g);
  g.has32 = 1;
  g.u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// Generator.random(): 53 random bits scaled to [0, 1).
__device__ __forceinline__ double pcg_random(Pcg &g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// random_bounded_uint64(off=0, rng, use_masked=false), rng <= 2^32-1: Lemire.
__device__ __forceinline__ uint64_t pcg_bounded(Pcg &g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng == 0xFFFFFFFFULL) return pcg_next32(g);
  uint32_t ex = (uint32_t)rng + 1u;
  uint64_t m = (uint64_t)pcg_next32(g) * ex;
  uint32_t left = (uint32_t)m;
  if (left < ex) {
    uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % ex;
    while (left < thr) {
      m = (uint64_t)pcg_next32(g) * ex;
      left = (uint32_t)m;
    }
  }
  return m >> 32;
}


// ------------------------------------------------ PCG64 state <-> amvm_pcg64
__device__ __forceinline__ Pcg pcg_load(const amvm_pcg64 *st) {
  // L2 reads: a chunked solve may have parked the state from another SM
  const unsigned long long *q = (const unsigned long long *)st;
  Pcg g;
  g.s = ((unsigned __int128)__ldcg(q) << 64) | __ldcg(q + 1);
  g.inc = ((unsigned __int128)__ldcg(q + 2) << 64) | __ldcg(q + 3);
  g.has32 = __ldcg(&st->has_uint32);
  g.u32 = __ldcg(&st->uinteger);
  return g;
}

__device__ __forceinline__ void pcg_store(const Pcg &g, amvm_pcg64 *st) {
  st->state_hi = (uint64_t)(g.s >> 64);
  st->state_lo = (uint64_t)g.s;
  st->inc_hi = (uint64_t)(g.inc >> 64);
  st->inc_lo = (uint64_t)g.inc;
  st->has_uint32 = g.has32;
  st->uinteger = g.u32;
}

// ------------------------------------------------------- operator bank
// select_operators (controller.py:88-90): rng.choice(4, p=w/sum(w)) = one
// random(), numpy's sequential cdf of p (sum(w) is a pairwise sum; n < 8 so
// sequential), normalised by cdf[-1], searchsorted(side='right').
__device__ inline int bank_select(const double *w, Pcg &g) {
  double s = 0.0;
  for (int k = 0; k < 4; ++k) s = dadd(s, w[k]);
  double cdf[4], acc = 0.0;
  for (int k = 0; k < 4; ++k) {
    acc = dadd(acc, ddiv(w[k], s));
    cdf[k] = acc;
  }
  const double u = pcg_random(g);
  int lo = 0, hi = 4;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u < ddiv(cdf[mid], cdf[3])) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// update_weights (controller.py:99-131): outcome 0 new best, 1 improved,
// 2 accepted, 3 rejected; every n_segment iterations
// w = max(decay*w + (1-decay)*(scores/uses or 0), floor), segment reset.
__device__ inline void bank_update(double *w, double *sc, int64_t *seg, int64_t *life, int64_t *bit, int pair,
                                   int outcome, double s1, double s2, double s3, double decay, double floor_w,
                                   int n_segment) {
  const double pts = outcome == 0 ? s1 : outcome == 1 ? s2 : outcome == 2 ? s3 : 0.0;
  sc[pair] = dadd(sc[pair], pts);
  seg[pair] += 1;
  life[pair] += 1;
  *bit += 1;
  if (*bit % n_segment == 0) {
    const double keep = dsub(1.0, decay);
    for (int k = 0; k < 4; ++k) {
      const double nrm = seg[k] > 0 ? ddiv(sc[k], (double)seg[k]) : 0.0;
      const double v = dadd(dmul(decay, w[k]), dmul(keep, nrm));
      w[k] = v < floor_w ? floor_w : v;
      sc[k] = 0.0;
      seg[k] = 0;
    }
  }
}

// ----------------------------------------------------- exp for x <= 0
// Table-driven exp (Tang, ACM TOMS 15, 1989): x = (32m + j) ln2/32 + r,
// |r| <= ln2/64, exp(x) = 2^m 2^(j/32) (1 + expm1(r)), 2^(j/32) as hi+lo,
// expm1 by its degree-6 Taylor polynomial (truncation < 4e-18).  <= ~0.52 ulp,
// i.e. the same accuracy class as numpy's SIMD exp and libm (neither is
// bit-reproducible here), at ~1/3 of CUDA's generic exp cost.
__device__ const double kExpHi[32] = {0x1.0000000000000p+0, 0x1.059b0d3158574p+0, 0x1.0b5586cf9890fp+0, 0x1.11301d0125b51p+0, 0x1.172b83c7d517bp+0, 0x1.1d4873168b9aap+0, 0x1.2387a6e756238p+0, 0x1.29e9df51fdee1p+0, 0x1.306fe0a31b715p+0, 0x1.371a7373aa9cbp+0, 0x1.3dea64c123422p+0, 0x1.44e086061892dp+0, 0x1.4bfdad5362a27p+0, 0x1.5342b569d4f82p+0, 0x1.5ab07dd485429p+0, 0x1.6247eb03a5585p+0, 0x1.6a09e667f3bcdp+0, 0x1.71f75e8ec5f74p+0, 0x1.7a11473eb0187p+0, 0x1.82589994cce13p+0, 0x1.8ace5422aa0dbp+0, 0x1.93737b0cdc5e5p+0, 0x1.9c49182a3f090p+0, 0x1.a5503b23e255dp+0, 0x1.ae89f995ad3adp+0, 0x1.b7f76f2fb5e47p+0, 0x1.c199bdd85529cp+0, 0x1.cb720dcef9069p+0, 0x1.d5818dcfba487p+0, 0x1.dfc97337b9b5fp+0, 0x1.ea4afa2a490dap+0, 0x1.f50765b6e4540p+0};
__device__ const double kExpLo[32] = {0x0.0p+0, 0x1.d73e2a475b465p-55, 0x1.8a62e4adc610bp-54, -0x1.6c51039449b3ap-54, -0x1.19041b9d78a76p-55, 0x1.e016e00a2643cp-54, 0x1.9b07eb6c70573p-54, 0x1.612e8afad1255p-55, 0x1.6f46ad23182e4p-55, -0x1.63aeabf42eae2p-54, 0x1.ada0911f09ebcp-55, 0x1.89b7a04ef80d0p-59, 0x1.d4397afec42e2p-56, -0x1.07abe1db13cadp-55, 0x1.6324c054647adp-54, -0x1.383c17e40b497p-54, -0x1.bdd3413b26456p-54, -0x1.16e4786887a99p-55, -0x1.41577ee04992fp-55, -0x1.d4c1dd41532d8p-54, 0x1.6e9f156864b27p-54, -0x1.75fc781b57ebcp-57, 0x1.c7c46b071f2bep-56, -0x1.d2f6edb8d41e1p-54, 0x1.7a1cd345dcc81p-54, -0x1.5584f7e54ac3bp-56, 0x1.11065895048ddp-55, 0x1.503cbd1e949dbp-56, 0x1.2ed02d75b3707p-55, -0x1.1a5cd4f184b5cp-54, -0x1.e9c23179c2893p-54, 0x1.9d3e12dd8a18bp-54};

__device__ __forceinline__ double exp_nonpos(double x) {
  if (x < -745.1332191019412) return 0.0;  // below the smallest subnormal
  const double kInv = 0x1.71547652b82fep+5;   // 32/ln2
  const double kMagic = 0x1.8p52;
  const double kL1 = 0x1.62e4200000000p-6;    // ln2/32, 20 bits: kd*kL1 exact
  const double kL2 = 0x1.fdf473de6af28p-27;
  const double kd = dsub(dadd(dmul(x, kInv), kMagic), kMagic);
  const int k = (int)kd;
  double r = dfma(kd, -kL1, x);
  r = dfma(kd, -kL2, r);
  double p = dfma(r, 1.0 / 720.0, 1.0 / 120.0);
  p = dfma(p, r, 1.0 / 24.0);
  p = dfma(p, r, 1.0 / 6.0);
  p = dfma(p, r, 0.5);
  p = dfma(dmul(r, r), p, r);  // expm1(r)
  const int j = k & 31, m = k >> 5;
  const double th = __ldg(&kExpHi[j]), tl = __ldg(&kExpLo[j]);
  const double res = dadd(th, dfma(th, p, dfma(tl, p, tl)));
  if (m >= -1022) return dmul(res, __longlong_as_double((long long)(m + 1023) << 52));
  return dmul(dmul(res, __longlong_as_double((long long)(m + 600 + 1023) << 52)), 0x1p-600);
}

// ------------------------------------------------- async global -> smem
// LDGSTS: 16-byte copy, zero-filled when `valid` is false (src not read).
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// --------------------------------------------------------------- warp ops
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(AMVM_FULL, v, o));
  return v;
}

// -------------------------------------------------- numpy pairwise summation
// numpy/_core/src/umath/loops_utils.h pairwise_sum: n < 8 sequential from 0;
// n <= 128 eight accumulators + ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) + tail;
// otherwise split at n2 = n/2 - (n/2)%8 and add the halves.
template <class F>
__device__ double pw_leaf(F &&get, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = dadd(res, get(lo + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = get(lo + k);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = dadd(r[k], get(lo + i + k));
  }
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, get(lo + i));
  return res;
}

// Leaves of the pairwise tree of length n, in left-to-right order.  Returns
// the count (<= cap); leaf k covers [lo[k], lo[k]+len[k]).  st_lo / st_n: a
// 48-deep scratch stack supplied by the caller (shared memory in the engine,
// so the kernel keeps no local-memory stack frame for it).
__device__ inline int pw_leaves(int64_t n, int64_t *lo, int64_t *len, int cap, int64_t *st_lo, int64_t *st_n) {
  // explicit stack of (lo, n); push right then left so leaves pop in order
  int sp = 0, cnt = 0;
  st_lo[sp] = 0;
  st_n[sp++] = n;
  while (sp) {
    --sp;
    int64_t a = st_lo[sp], c = st_n[sp];
    if (c <= 128) {
      if (cnt < cap) {
        lo[cnt] = a;
        len[cnt] = c;
      }
      ++cnt;
    } else {
      int64_t n2 = c / 2;
      n2 -= n2 % 8;
      st_lo[sp] = a + n2;
      st_n[sp++] = c - n2;
      st_lo[sp] = a;
      st_n[sp++] = n2;
    }
  }
  return cnt;
}

// Combine leaf sums in the exact tree order (recursive shape, iterative walk).
// st_n / st_state / st_val: 48-deep caller scratch (see pw_leaves).
__device__ inline double pw_combine(int64_t n, const double *leaf_sum, int64_t *st_n, int *st_state,
                                    double *st_val) {
  // post-order evaluation with an explicit stack
  int sp = 0, leaf = 0;
  st_n[0] = n;
  st_state[0] = 0;
  sp = 1;
  double ret = 0.0;
  while (sp) {
    int top = sp - 1;
    int64_t c = st_n[top];
    if (c <= 128) {
      ret = leaf_sum[leaf++];
      --sp;
      // deliver to parent
      while (sp) {
        int p = sp - 1;
        if (st_state[p] == 1) {  // left done, now right
          st_val[p] = ret;
          st_state[p] = 2;
          int64_t n2 = st_n[p] / 2;
          n2 -= n2 % 8;
          st_n[sp] = st_n[p] - n2;
          st_state[sp] = 0;
          ++sp;
          break;
        } else {  // state 2: right done
          ret = dadd(st_val[p], ret);
          --sp;
        }
      }
    } else if (st_state[top] == 0) {
      st_state[top] = 1;
      int64_t n2 = c / 2;
      n2 -= n2 % 8;
      st_n[sp] = n2;
      st_state[sp] = 0;
      ++sp;
    }
  }
  return ret;
}

// ---------------------------------------------- OpenBLAS SkylakeX ddot order
// One warp computes x.y (x == y for norms): lane = accumulator slot (q, l) of
// the 4 x 8-lane AVX-512 FMA accumulators over n & ~31, then lane 0 folds in
// the kernel's exact order and runs the scalar FMA tail.  Returns the dot in
// every lane.
template <class GX, class GY>
__device__ double warp_ddot_skx(GX &&gx, GY &&gy, int64_t n, int lane) {
  const int64_t n1 = n & -16;
  const int64_t n32 = n1 & ~(int64_t)31;
  double a = 0.0;  // lane = 8*q + l
  for (int64_t i = 0; i < n32; i += 32) a = dfma(gx(i + lane), gy(i + lane), a);
  double dot = 0.0;
  if (n1) {
    // fold 512 -> 256: acc[q][l] = a[q][l] + a[q][l+4] (l < 4)
    double hi = __shfl_down_sync(AMVM_FULL, a, 4);
    double acc = dadd(a, hi);  // valid in lanes with (lane & 4) == 0
    // remaining 16-block: acc[q][l] (q < 4, l < 4) gets x[n32 + 4q + l]
    const int q = lane >> 3, l = lane & 7;
    if (n1 - n32 == 16 && l < 4) acc = dfma(gx(n32 + 4 * q + l), gy(n32 + 4 * q + l), acc);
    // gather acc[q][l] to lane 0
    double v[4][4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
      for (int ll = 0; ll < 4; ++ll) v[qq][ll] = __shfl_sync(AMVM_FULL, acc, 8 * qq + ll);
    double s[4];
#pragma unroll
    for (int ll = 0; ll < 4; ++ll) s[ll] = dadd(dadd(dadd(v[0][ll], v[1][ll]), v[2][ll]), v[3][ll]);
    dot = dadd(dadd(s[0], s[2]), dadd(s[1], s[3]));
  }
  for (int64_t i = n1; i < n; ++i) dot = dfma(gy(i), gx(i), dot);
  return dot;
}

// ------------------------------------------ OpenBLAS dgemv_t (numpy A @ x)
// One output of A @ x for a C-contiguous A (kernel/x86_64/dgemv_t_4.c with
// the Haswell micro-kernels, used for SkylakeX): K & -4 elements in blocks
// of 2048 reduced by the kernel of the output's position (kind 4: 4x4,
// 4-lane FMA, lanes (0+2)+(1+3); kind 2: 4x2, 2-lane mul+add; kind 1: 4x1,
// two 2-lane mul+add accumulators), each block added to y; then the K & 3
// leftover in the compiler-contracted scalar form.  `a(j)` = A[i][j].
template <class GA, class GX>
__device__ double gemv_row(GA &&a, GX &&x, int64_t K, int kind) {
  const int64_t m1 = K & -4;
  double y = 0.0;
  for (int64_t p = 0; p < m1; p += 2048) {
    const int64_t e = p + (m1 - p < 2048 ? m1 - p : 2048);
    double t;
    if (kind == 4) {
      double l0 = 0, l1 = 0, l2 = 0, l3 = 0;
      for (int64_t i = p; i < e; i += 4) {
        l0 = dfma(a(i), x(i), l0);
        l1 = dfma(a(i + 1), x(i + 1), l1);
        l2 = dfma(a(i + 2), x(i + 2), l2);
        l3 = dfma(a(i + 3), x(i + 3), l3);
      }
      t = dadd(dadd(l0, l2), dadd(l1, l3));
    } else if (kind == 2) {
      double l0 = 0, l1 = 0;
      for (int64_t i = p; i < e; i += 2) {
        l0 = dadd(l0, dmul(a(i), x(i)));
        l1 = dadd(l1, dmul(a(i + 1), x(i + 1)));
      }
      t = dadd(l0, l1);
    } else {
      double u0 = 0, u1 = 0, v0 = 0, v1 = 0;
      for (int64_t i = p; i < e; i += 4) {
        u0 = dadd(u0, dmul(a(i), x(i)));
        u1 = dadd(u1, dmul(a(i + 1), x(i + 1)));
        v0 = dadd(v0, dmul(a(i + 2), x(i + 2)));
        v1 = dadd(v1, dmul(a(i + 3), x(i + 3)));
      }
      t = dadd(dadd(u0, v0), dadd(u1, v1));
    }
    y = dadd(y, t);
  }
  switch (K & 3) {
    case 1: y = dfma(a(m1), x(m1), y); break;
    case 2: y = dadd(y, dfma(a(m1), x(m1), dmul(a(m1 + 1), x(m1 + 1)))); break;
    case 3:
      y = dadd(y, dfma(a(m1 + 2), x(m1 + 2), dfma(a(m1), x(m1), dmul(a(m1 + 1), x(m1 + 1)))));
      break;
    default: break;
  }
  return y;
}

// kernel kind of output row i of an m-row dgemv_t (4x4 groups, then 4x2, 4x1)
// gemv_row for a sparse row (its nonzeros: columns ascending `cols`, values
// `vals`): the same blocks, lanes and combination order with the zero
// terms left out -- adding fma(0, x, l) or 0*x leaves every partial sum
// unchanged, so the result equals the dense one (up to the sign of a zero).
template <class GX>
__device__ double gemv_row_sparse(const int32_t *cols, const double *vals, int64_t nnz, GX &&x, int64_t K,
                                  int kind) {
  const int64_t m1 = K & -4;
  double y = 0.0;
  int64_t e = 0;
  for (int64_t p = 0; p < m1; p += 2048) {
    const int64_t pe = p + (m1 - p < 2048 ? m1 - p : 2048);
    double t;
    if (kind == 4) {
      double l[4] = {0.0, 0.0, 0.0, 0.0};
      for (; e < nnz && __ldg(cols + e) < pe; ++e) {
        const int64_t c = __ldg(cols + e);
        l[c & 3] = dfma(__ldg(vals + e), x(c), l[c & 3]);
      }
      t = dadd(dadd(l[0], l[2]), dadd(l[1], l[3]));
    } else if (kind == 2) {
      double l[2] = {0.0, 0.0};
      for (; e < nnz && __ldg(cols + e) < pe; ++e) {
        const int64_t c = __ldg(cols + e);
        l[c & 1] = dadd(l[c & 1], dmul(__ldg(vals + e), x(c)));
      }
      t = dadd(l[0], l[1]);
    } else {
      double u[4] = {0.0, 0.0, 0.0, 0.0};  // u0, u1, v0, v1
      for (; e < nnz && __ldg(cols + e) < pe; ++e) {
        const int64_t c = __ldg(cols + e);
        u[c & 3] = dadd(u[c & 3], dmul(__ldg(vals + e), x(c)));
      }
      t = dadd(dadd(u[0], u[2]), dadd(u[1], u[3]));
    }
    y = dadd(y, t);
  }
  // the K & 3 leftover columns, in the dense formula with absent entries 0
  auto a = [&](int64_t c) -> double {
    while (e < nnz && __ldg(cols + e) < c) ++e;
    return (e < nnz && __ldg(cols + e) == c) ? __ldg(vals + e) : 0.0;
  };
  switch (K & 3) {
    case 1: y = dfma(a(m1), x(m1), y); break;
    case 2: {
      const double a0 = a(m1), a1 = a(m1 + 1);
      y = dadd(y, dfma(a0, x(m1), dmul(a1, x(m1 + 1))));
      break;
    }
    case 3: {
      const double a0 = a(m1), a1 = a(m1 + 1), a2 = a(m1 + 2);
      y = dadd(y, dfma(a2, x(m1 + 2), dfma(a0, x(m1), dmul(a1, x(m1 + 1)))));
      break;
    }
    default: break;
  }
  return y;
}

__device__ __forceinline__ int gemv_kind(int64_t i, int64_t m) {
  const int64_t g4 = m & ~(int64_t)3;
  if (i < g4) return 4;
  if ((m & 2) && i < g4 + 2) return 2;
  return 1;
}

}  // namespace amvm

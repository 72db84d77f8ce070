// backward.cu -- SIMT kernels for the backward pass of the fused layer.
//
// Replaces reference proj/include/segconv/netdemo/layers.hpp:171-211
// (net::FusedTConv<T>::backward) for a batch: the input gradient gx (the
// output gradient scattered back through the four sub-kernels, cropped by
// p_fused) and the kernel gradient gk (tap gradients at the original tap
// positions u0 + 2u, v0 + 2v, summed over the batch).
//
// Two formulations of the same sums:
//   * EXACT: one thread per gradient element, walking the reference's own
//     accumulation order (class, anchor row, anchor column, f) with no FMA
//     contraction -- bit-identical to the reference CPU path for float and
//     double.  For gx the contributions to padded pixel P arrive in the
//     reference's (q, i, j) loop order, i.e. u and v descending.
//   * FFMA: both gradients as tiled SIMT GEMMs over the whole kernel (no class
//     split is needed -- every tap (U, V) reaches every input pixel):
//       gx[m, ch]      = sum_{U,V,f} gy[b, 2i+p-U, 2j+p-V, f] * k[U, V, ch, f]
//       gk[U, V, ch, f] = sum_m      x[m, ch] * gy[b, 2i+p-U, 2j+p-V, f]
//     with m = (b, i, j) and out-of-range gy positions reading as zero.  The
//     weight gradient splits its pixel reduction over CTAs when the tap x
//     channel tiles alone cannot fill the 148 SMs; partial sums go to a
//     stream-ordered workspace and are reduced in split order (deterministic).
// The tensor-core input gradient (bf16) is tc_wide.cu's CTA-pair kernel run on
// a stride-2 im2col walk over gy (launch_tc_bwd_data there).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace segconv_b200 {
namespace bwd {

// --------------------------------------------------------------- helpers
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__device__ __forceinline__ T from_acc(float v) {
  return from_f<T>(v);
}
template <typename T>
__device__ __forceinline__ T from_acc(double v) {
  return from_d<T>(v);
}

template <typename ACC, typename T>
__device__ __forceinline__ ACC ld(const T* p) {
  return (ACC)to_acc(p[0]);
}

// 4 consecutive elements p[0..3] (entries at or past `lim` read as 0); one
// vector load when all 4 exist and p is aligned for it
template <typename ACC, typename T>
__device__ __forceinline__ void ld4(const T* p, int lim, bool ok, ACC (&v)[4]) {
  if (ok && lim >= 4 && (reinterpret_cast<uintptr_t>(p) & (4 * sizeof(T) - 1)) == 0) {
    if constexpr (sizeof(T) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
      return;
    } else if constexpr (sizeof(T) == 2) {
      const uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&q.x);
      const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&q.y);
      v[0] = __low2float(a), v[1] = __high2float(a), v[2] = __low2float(b), v[3] = __high2float(b);
      return;
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) v[e] = (ok && e < lim) ? ld<ACC>(p + e) : ACC(0);
}

// reference segregation.hpp:23-36
__device__ __forceinline__ int first_tap(int p, int r) { return (p + r) & 1; }
__device__ __forceinline__ int tap_count(int n, int p, int r) {
  const int f = first_tap(p, r);
  return f >= n ? 0 : (n - f + 1) / 2;
}
__device__ __forceinline__ int class_off(int p, int r) { return (r + first_tap(p, r) - p) / 2 + p / 2; }

// ------------------------------------------------------------ EXACT: gx
// One thread per (b, i, j, ch); ch fastest.
template <typename T>
__global__ void __launch_bounds__(256) dgrad_exact(const T* __restrict__ gy, const T* __restrict__ k,
                                                   T* __restrict__ gx, BackwardProblem pr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)pr.batch * pr.n * pr.n * pr.cin;
  if (e >= total) return;
  const int ch = (int)(e % pr.cin);
  const long long m = e / pr.cin;
  const int j = (int)(m % pr.n), i = (int)((m / pr.n) % pr.n), b = (int)(m / ((long long)pr.n * pr.n));
  const int Pr = i + pr.pf, Pc = j + pr.pf;
  T sum = 0;
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, c = q & 1;
    const int skh = tap_count(pr.kh, pr.p, r), skw = tap_count(pr.kw, pr.p, c);
    if (skh == 0 || skw == 0) continue;
    const int u0 = first_tap(pr.p, r), v0 = first_tap(pr.p, c);
    const int offr = class_off(pr.p, r), offc = class_off(pr.p, c);
    const int rows = (pr.out_h - r + 1) / 2, cols = (pr.out_w - c + 1) / 2;
    for (int u = skh - 1; u >= 0; --u) {  // anchor row ascending
      const int a = Pr - offr - u;
      if (a < 0 || a >= rows) continue;
      for (int v = skw - 1; v >= 0; --v) {
        const int bb = Pc - offc - v;
        if (bb < 0 || bb >= cols) continue;
        const T* gp = gy + (((long long)b * pr.out_h + 2 * a + r) * pr.out_w + 2 * bb + c) * pr.cout;
        const T* w = k + (((long long)(u0 + 2 * u) * pr.kw + (v0 + 2 * v)) * pr.cin + ch) * pr.cout;
        T acc = 0;
        for (int f = 0; f < pr.cout; ++f) acc = add_rn(acc, mul_rn(w[f], gp[f]));
        sum = add_rn(sum, acc);
      }
    }
  }
  gx[e] = sum;
}

// ------------------------------------------------------------ EXACT: gk
// One thread per (U, V, ch, f); f fastest.  Padded input positions contribute
// +-0 products, which never change a round-to-nearest sum that starts at +0,
// so they are skipped.
template <typename T>
__global__ void __launch_bounds__(256) wgrad_exact(const T* __restrict__ x, const T* __restrict__ gy,
                                                   T* __restrict__ gk, BackwardProblem pr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
  if (e >= total) return;
  const int f = (int)(e % pr.cout);
  const int ch = (int)((e / pr.cout) % pr.cin);
  const int t = (int)(e / ((long long)pr.cout * pr.cin));
  const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
  const int r = (U + pr.p) & 1, c = (V + pr.p) & 1;
  const int u = (U - first_tap(pr.p, r)) / 2, v = (V - first_tap(pr.p, c)) / 2;
  const int offr = class_off(pr.p, r), offc = class_off(pr.p, c);
  const int rows = (pr.out_h - r + 1) / 2, cols = (pr.out_w - c + 1) / 2;
  T s = pr.accumulate ? gk[e] : T(0);
  for (int b = 0; b < pr.batch; ++b)
    for (int a = 0; a < rows; ++a) {
      const int xr = a + offr + u - pr.pf;
      if (xr < 0 || xr >= pr.n) continue;
      for (int bb = 0; bb < cols; ++bb) {
        const int xc = bb + offc + v - pr.pf;
        if (xc < 0 || xc >= pr.n) continue;
        const T xv = x[(((long long)b * pr.n + xr) * pr.n + xc) * pr.cin + ch];
        const T gv = gy[(((long long)b * pr.out_h + 2 * a + r) * pr.out_w + 2 * bb + c) * pr.cout + f];
        s = add_rn(s, mul_rn(xv, gv));
      }
    }
  gk[e] = s;
}

// ------------------------------------------------- EXACT: conv2d_valid
// reference netdemo/layers.hpp:98-122 (ConvValid::backward): contributions to
// gin(a, c) arrive for output pixels (y, x) = (a - u, c - v) in ascending
// order, i.e. u and v descending; acc over f ascending, no FMA.
template <typename T>
__global__ void __launch_bounds__(256) conv_dgrad_exact(const T* __restrict__ gy, const T* __restrict__ k,
                                                        T* __restrict__ gx, BackwardProblem pr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)pr.batch * pr.in_h * pr.in_w * pr.cin;
  if (e >= total) return;
  const int ch = (int)(e % pr.cin);
  const long long m = e / pr.cin;
  const int c = (int)(m % pr.in_w), a = (int)((m / pr.in_w) % pr.in_h);
  const int b = (int)(m / ((long long)pr.in_h * pr.in_w));
  T sum = 0;
  for (int u = pr.kh - 1; u >= 0; --u) {
    const int y = a - u;
    if (y < 0 || y >= pr.out_h) continue;
    for (int v = pr.kw - 1; v >= 0; --v) {
      const int x = c - v;
      if (x < 0 || x >= pr.out_w) continue;
      const T* gp = gy + (((long long)b * pr.out_h + y) * pr.out_w + x) * pr.cout;
      const T* w = k + (((long long)u * pr.kw + v) * pr.cin + ch) * pr.cout;
      T acc = 0;
      for (int f = 0; f < pr.cout; ++f) acc = add_rn(acc, mul_rn(w[f], gp[f]));
      sum = add_rn(sum, acc);
    }
  }
  gx[e] = sum;
}

template <typename T>
__global__ void __launch_bounds__(256) conv_wgrad_exact(const T* __restrict__ x, const T* __restrict__ gy,
                                                        T* __restrict__ gk, BackwardProblem pr) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
  if (e >= total) return;
  const int f = (int)(e % pr.cout);
  const int ch = (int)((e / pr.cout) % pr.cin);
  const int t = (int)(e / ((long long)pr.cout * pr.cin));
  const int u = t / pr.kw, v = t - (t / pr.kw) * pr.kw;
  T s = pr.accumulate ? gk[e] : T(0);
  for (int b = 0; b < pr.batch; ++b)
    for (int y = 0; y < pr.out_h; ++y)
      for (int xx = 0; xx < pr.out_w; ++xx) {
        const T xv = x[(((long long)b * pr.in_h + y + u) * pr.in_w + xx + v) * pr.cin + ch];
        const T gv = gy[(((long long)b * pr.out_h + y) * pr.out_w + xx) * pr.cout + f];
        s = add_rn(s, mul_rn(xv, gv));
      }
  gk[e] = s;
}

// ------------------------------------------------------------- FFMA tiles
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

// gx tile: 64 pixels x 64 input channels, K = taps x cout in 16-feature steps.
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) dgrad_ffma(const T* __restrict__ gy, const T* __restrict__ k,
                                                 T* __restrict__ gx, BackwardProblem pr) {
  if (pr.run_if != nullptr && *pr.run_if == 0) return;  // the tensor-core path took it
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  const long long m0 = (long long)blockIdx.x * BM;
  const int ch0 = blockIdx.y * BN;
  const int lp = tid >> 2, lf = (tid & 3) * 4;  // loader: row lp, 4 consecutive features
  const long long m = m0 + lp;
  const bool mv = m < M;
  const int j = mv ? (int)(m % pr.in_w) : 0, i = mv ? (int)((m / pr.in_w) % pr.in_h) : 0;
  const int b = mv ? (int)(m / ((long long)pr.in_h * pr.in_w)) : 0;
  const bool kv = ch0 + lp < pr.cin;
  ACC acc[4][4] = {};
  for (int t = 0; t < pr.kh * pr.kw; ++t) {
    const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
    const int y = pr.stride * i + pr.p - U, xx = pr.stride * j + pr.p - V;
    const bool av = mv && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w;
    const T* gp = gy + (((long long)b * pr.out_h + (av ? y : 0)) * pr.out_w + (av ? xx : 0)) * pr.cout;
    const T* kp = k + ((long long)t * pr.cin + (kv ? ch0 + lp : 0)) * pr.cout;
    for (int f0 = 0; f0 < pr.cout; f0 += BK) {
      ACC va[4], vb[4];
      ld4<ACC>(gp + f0 + lf, pr.cout - f0 - lf, av, va);
      ld4<ACC>(kp + f0 + lf, pr.cout - f0 - lf, kv, vb);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        As[lf + e][lp] = va[e];
        Bs[lf + e][lp] = vb[e];
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        ACC a[4], w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          a[e] = As[kk][ty * 4 + e];
          w[e] = Bs[kk][tx * 4 + e];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] += a[r] * w[c];
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const long long mm = m0 + ty * 4 + r;
    if (mm >= M) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ch = ch0 + tx * 4 + c;
      if (ch < pr.cin) gx[mm * pr.cin + ch] = from_acc<T>(acc[r][c]);
    }
  }
}

// Narrow layers (cout % 16 != 0, e.g. the 3-channel output layers C4, C5 d):
// K packed as (tap, f) pairs, f fastest, so a 16-deep step never idles on
// missing features (cout = 3 would use 3 of every 16).
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) dgrad_ffma_packed(const T* __restrict__ gy, const T* __restrict__ k,
                                                        T* __restrict__ gx, BackwardProblem pr) {
  if (pr.run_if != nullptr && *pr.run_if == 0) return;  // the tensor-core path took it
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  const long long m0 = (long long)blockIdx.x * BM;
  const int ch0 = blockIdx.y * BN;
  const int lp = tid >> 2, lf = (tid & 3) * 4;
  const long long m = m0 + lp;
  const bool mv = m < M;
  const int j = mv ? (int)(m % pr.in_w) : 0, i = mv ? (int)((m / pr.in_w) % pr.in_h) : 0;
  const int b = mv ? (int)(m / ((long long)pr.in_h * pr.in_w)) : 0;
  const bool kv = ch0 + lp < pr.cin;
  const int K = pr.kh * pr.kw * pr.cout;
  const T* gb = gy + (long long)b * pr.out_h * pr.out_w * pr.cout;
  ACC acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    int t = (k0 + lf) / pr.cout, f = (k0 + lf) - ((k0 + lf) / pr.cout) * pr.cout;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      ACC va = 0, vb = 0;
      if (k0 + lf + e < K) {
        const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
        const int y = pr.stride * i + pr.p - U, xx = pr.stride * j + pr.p - V;
        if (mv && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w)
          va = ld<ACC>(gb + ((long long)y * pr.out_w + xx) * pr.cout + f);
        if (kv) vb = ld<ACC>(k + ((long long)t * pr.cin + ch0 + lp) * pr.cout + f);
      }
      As[lf + e][lp] = va;
      Bs[lf + e][lp] = vb;
      if (++f == pr.cout) {
        f = 0;
        ++t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      ACC a[4], w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = As[kk][ty * 4 + e];
        w[e] = Bs[kk][tx * 4 + e];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += a[r] * w[c];
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const long long mm = m0 + ty * 4 + r;
    if (mm >= M) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int ch = ch0 + tx * 4 + c;
      if (ch < pr.cin) gx[mm * pr.cin + ch] = from_acc<T>(acc[r][c]);
    }
  }
}

// gk with N packed as (tap, f) pairs (cout % 64 != 0): one CTA covers 64
// channels x 64 packed columns over a pixel range, every tap of the tile at once.
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) wgrad_ffma_packed(const T* __restrict__ x, const T* __restrict__ gy,
                                                        ACC* __restrict__ out, BackwardProblem pr, int splits,
                                                        long long chunk, int direct) {
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  const int NP = pr.kh * pr.kw * pr.cout;
  const int ch0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int s = blockIdx.z;
  const long long mb = (long long)s * chunk, me = (mb + chunk < M) ? mb + chunk : M;
  const int lp = tid >> 4, lc = (tid & 15) * 4;
  // this thread's 4 packed columns: tap offsets (U, V) and feature f
  int cu[4], cv[4], cf[4];
  bool cok[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int n = n0 + lc + e;
    cok[e] = n < NP;
    const int t = cok[e] ? n / pr.cout : 0;
    cf[e] = cok[e] ? n - t * pr.cout : 0;
    cu[e] = t / pr.kw;
    cv[e] = t - (t / pr.kw) * pr.kw;
  }
  ACC acc[4][4] = {};
  const int img = pr.in_h * pr.in_w, di = BK / pr.in_w, dj = BK - (BK / pr.in_w) * pr.in_w;
  const long long mf = mb + lp;
  int b = (int)(mf / img), i = (int)(mf - (long long)b * img), j = i % pr.in_w;
  i /= pr.in_w;
  for (long long mk = mb; mk < me; mk += BK) {
    const long long m = mk + lp;
    const bool mv = m < me;
    ACC va[4];
    ld4<ACC>(x + (mv ? m : 0) * pr.cin + ch0 + lc, pr.cin - ch0 - lc, mv, va);
    const T* gb = gy + (long long)b * pr.out_h * pr.out_w * pr.cout;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int y = pr.stride * i + pr.p - cu[e], xx = pr.stride * j + pr.p - cv[e];
      const bool ok = mv && cok[e] && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w;
      As[lp][lc + e] = va[e];
      Bs[lp][lc + e] = ok ? ld<ACC>(gb + ((long long)y * pr.out_w + xx) * pr.cout + cf[e]) : ACC(0);
    }
    j += dj;
    i += di;
    if (j >= pr.in_w) {
      j -= pr.in_w;
      ++i;
    }
    if (i >= pr.in_h) {
      const int q = i / pr.in_h;
      b += q;
      i -= q * pr.in_h;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      ACC a[4], w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = As[kk][ty * 4 + e];
        w[e] = Bs[kk][tx * 4 + e];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += a[r] * w[c];
    }
    __syncthreads();
  }
  const long long ksz = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int n = n0 + tx * 4 + c;
    if (n >= NP) continue;
    const int t = n / pr.cout, f = n - (n / pr.cout) * pr.cout;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int ch = ch0 + ty * 4 + r;
      if (ch >= pr.cin) continue;
      const long long idx = ((long long)t * pr.cin + ch) * pr.cout + f;
      if (direct)
        out[idx] = (pr.accumulate ? out[idx] : ACC(0)) + acc[r][c];
      else
        out[(long long)s * ksz + idx] = acc[r][c];
    }
  }
}

// gk tile: 64 input channels x 64 features of one tap over a pixel range.
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) wgrad_ffma(const T* __restrict__ x, const T* __restrict__ gy,
                                                 ACC* __restrict__ out, BackwardProblem pr, int splits,
                                                 long long chunk, int direct) {
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  const int ch0 = blockIdx.x * BM, f0 = blockIdx.y * BN;
  const int t = blockIdx.z / splits, s = blockIdx.z - (blockIdx.z / splits) * splits;
  const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
  const long long mb = (long long)s * chunk, me = (mb + chunk < M) ? mb + chunk : M;
  const int lp = tid >> 4, lc = (tid & 15) * 4;  // loader: pixel lp, 4 consecutive channels
  ACC acc[4][4] = {};
  // this thread's pixel (b, i, j), advanced by BK pixels per step without divisions
  const int img = pr.in_h * pr.in_w, di = BK / pr.in_w, dj = BK - (BK / pr.in_w) * pr.in_w;
  const long long m0 = mb + lp;
  int b = (int)(m0 / img), i = (int)(m0 - (long long)b * img), j = i % pr.in_w;
  i /= pr.in_w;
  for (long long mk = mb; mk < me; mk += BK) {
    const long long m = mk + lp;
    const bool mv = m < me;
    const int y = pr.stride * i + pr.p - U, xx = pr.stride * j + pr.p - V;
    const bool gv = mv && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w;
    const T* xp = x + (mv ? m : 0) * pr.cin;
    const T* gp = gy + (((long long)b * pr.out_h + (gv ? y : 0)) * pr.out_w + (gv ? xx : 0)) * pr.cout;
    ACC va[4], vb[4];
    ld4<ACC>(xp + ch0 + lc, pr.cin - ch0 - lc, gv, va);
    ld4<ACC>(gp + f0 + lc, pr.cout - f0 - lc, gv, vb);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      As[lp][lc + e] = va[e];
      Bs[lp][lc + e] = vb[e];
    }
    j += dj;
    i += di;
    if (j >= pr.in_w) {
      j -= pr.in_w;
      ++i;
    }
    if (i >= pr.in_h) {
      const int q = i / pr.in_h;
      b += q;
      i -= q * pr.in_h;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      ACC a[4], w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = As[kk][ty * 4 + e];
        w[e] = Bs[kk][tx * 4 + e];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += a[r] * w[c];
    }
    __syncthreads();
  }
  const long long ksz = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ch = ch0 + ty * 4 + r;
    if (ch >= pr.cin) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int f = f0 + tx * 4 + c;
      if (f >= pr.cout) continue;
      const long long idx = ((long long)t * pr.cin + ch) * pr.cout + f;
      if (direct)
        out[idx] = (pr.accumulate ? out[idx] : ACC(0)) + acc[r][c];
      else
        out[(long long)s * ksz + idx] = acc[r][c];
    }
  }
}

// gk = (accumulate ? gk : 0) + sum over splits, in split order
template <typename ACC>
__global__ void wgrad_reduce(const ACC* __restrict__ ws, ACC* __restrict__ gk, long long ksz, int splits,
                             int accumulate) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ksz) return;
  ACC s = accumulate ? gk[e] : ACC(0);
  for (int i = 0; i < splits; ++i) s += ws[(long long)i * ksz + e];
  gk[e] = s;
}
// float4 version (ksz % 4 == 0, 16-byte aligned buffers), same per-element order
__global__ void wgrad_reduce4(const float4* __restrict__ ws, float4* __restrict__ gk, long long n4, int splits,
                              int accumulate) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n4) return;
  float4 s = accumulate ? gk[e] : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = 0; i < splits; ++i) {
    const float4 v = __ldcs(ws + (long long)i * n4 + e);  // read once: streaming
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  gk[e] = s;
}

// Many splits of a small gradient (the narrow kernels' hundreds of partials of
// a 4800-element gk): 8 float4 elements per CTA, 32 split groups of 8 threads
// each summing every 32nd split, then a fixed-order combine of the 32 group
// sums (deterministic) -- instead of one thread walking all splits serially.
__global__ void __launch_bounds__(256) wgrad_reduce4_wide(const float4* __restrict__ ws, float4* __restrict__ gk,
                                                          long long n4, int splits, int accumulate) {
  __shared__ float4 part[32][8];
  const int el = threadIdx.x & 7, grp = threadIdx.x >> 3;
  const long long e = (long long)blockIdx.x * 8 + el;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e < n4)
    for (int i = grp; i < splits; i += 32) {
      const float4 v = __ldcs(ws + (long long)i * n4 + e);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
  part[grp][el] = s;
  __syncthreads();
  if (grp == 0 && e < n4) {
    float4 t = accumulate ? gk[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int g = 0; g < 32; ++g) {
      t.x += part[g][el].x;
      t.y += part[g][el].y;
      t.z += part[g][el].z;
      t.w += part[g][el].w;
    }
    gk[e] = t;
  }
}

// ------------------------------------------------- narrow outputs (cout <= 4)
// The C4 family (5x5 -> 3 at 256^2): the packed FFMA tiles above leave most of
// every tile's K (or N) idle and gather g element by element.  Here a CTA owns
// one input row segment of 128 pixels x 64 channels; the g rows its pixels read
// (kh rows x (2*128 + kw) columns x CO features) and the 64-channel slice of the
// kernel are staged once in SMEM.
constexpr int NW_PX = 128, NW_CH = 64, NW_MAXK = 7;

__host__ __device__ constexpr int nw_gw(int kw) { return 2 * NW_PX + kw; }

// stage g rows y = 2i + p - U (U < kh) at columns [2 j0 + p - (kw - 1), +gw) as
// sg[(U * gw + col) * CO + f]; zero outside g
template <typename T, int CO>
__device__ __forceinline__ void nw_stage_g(const T* __restrict__ gy, float* sg, const BackwardProblem& pr, int b,
                                           int i, int j0) {
  const int gw = nw_gw(pr.kw), c0 = 2 * j0 + pr.p - (pr.kw - 1);
  for (int U = 0; U < pr.kh; ++U) {
    const int y = 2 * i + pr.p - U;
    const bool yok = y >= 0 && y < pr.out_h;
    const T* grow = gy + ((long long)b * pr.out_h + (yok ? y : 0)) * pr.out_w * CO;
    float* srow = sg + U * gw * CO;
    for (int e = threadIdx.x; e < gw * CO; e += blockDim.x) {
      const int xx = c0 + e / CO;  // CO is a compile-time constant: a multiply-shift
      srow[e] = (yok && xx >= 0 && xx < pr.out_w) ? to_acc(grow[(long long)c0 * CO + e]) : 0.f;
    }
  }
}

// gx: lane = (pixel half, 4 channels); 8 pixels per thread (slots 16 apart) --
// per (U, V, f): one LDS.128 of weights + 8 broadcast g loads for 32 FFMA; a
// half-warp stores one pixel's 64 channels as 256 contiguous bytes
template <typename T, int CO>
__global__ void __launch_bounds__(256) dgrad_narrow(const T* __restrict__ gy, const T* __restrict__ k,
                                                    T* __restrict__ gx, BackwardProblem pr) {
  extern __shared__ float nsm[];
  const int taps = pr.kh * pr.kw, gw = nw_gw(pr.kw);
  float* sw = nsm;                        // [(tap * CO + f) * 64 + c]
  float* sg = nsm + taps * CO * NW_CH;    // [(U * gw + col) * CO + f]
  const int j0 = blockIdx.y * NW_PX, cb = blockIdx.z * NW_CH;
  for (int e = threadIdx.x; e < taps * CO * NW_CH; e += blockDim.x) {
    const int c = e & (NW_CH - 1), tf = e / NW_CH;  // tf = tap * CO + f
    sw[e] = cb + c < pr.cin ? to_acc(k[((long long)(tf / CO) * pr.cin + cb + c) * CO + tf % CO]) : 0.f;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c4 = lane & 15, slot = warp * 2 + (lane >> 4);
  const int total_rows = pr.batch * pr.in_h;
  // the CTA's rows (weights stay staged): blockIdx.x, + gridDim.x, ...
  for (int row = blockIdx.x; row < total_rows; row += gridDim.x) {
  const int b = row / pr.in_h, i = row - (row / pr.in_h) * pr.in_h;
  __syncthreads();  // previous row's g reads are done
  nw_stage_g<T, CO>(gy, sg, pr, b, i, j0);
  __syncthreads();
  float acc[8][4] = {};
  for (int U = 0; U < pr.kh; ++U)
    for (int V = 0; V < pr.kw; ++V) {
      const float* gp = sg + ((U * gw) + 2 * slot + pr.kw - 1 - V) * CO;
      const float* wp = sw + ((U * pr.kw + V) * CO) * NW_CH + 4 * c4;
#pragma unroll
      for (int f = 0; f < CO; ++f) {
        const float4 w = *reinterpret_cast<const float4*>(wp + f * NW_CH);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float g = gp[32 * e * CO + f];  // pixel slot + 16 e: column + 32 e
          acc[e][0] = fmaf(g, w.x, acc[e][0]);
          acc[e][1] = fmaf(g, w.y, acc[e][1]);
          acc[e][2] = fmaf(g, w.z, acc[e][2]);
          acc[e][3] = fmaf(g, w.w, acc[e][3]);
        }
      }
    }
  const int ch = cb + 4 * c4;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int j = j0 + slot + 16 * e;
    if (j >= pr.in_w) continue;
    T* o = gx + ((long long)row * pr.in_w + j) * pr.cin + ch;
    if constexpr (sizeof(T) == 4) {
      if (ch + 4 <= pr.cin && (pr.cin & 3) == 0) {
        *reinterpret_cast<float4*>(o) = make_float4(acc[e][0], acc[e][1], acc[e][2], acc[e][3]);
        continue;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (ch + c < pr.cin) o[c] = from_acc<T>(acc[e][c]);
  }
  }
}

// gk partials: a CTA sums `rows` consecutive input rows (all columns, 64
// channels).  PH pixel phases (pixels px = phase mod PH); a thread owns 8
// channels x COLS (tap, f) columns: per pixel 2 LDS.128 of x + COLS g loads for
// 8 COLS FFMA.  Each phase writes its own partial (split).  COLS = 5 (two
// phases, 80 registers, three CTAs per SM so one CTA's staging overlaps the
// others' math) measured fastest on C4: 1031 us vs 1110 with COLS = 10.
template <typename T, int CO, int COLS>
__global__ void __launch_bounds__(256, COLS == 5 ? 3 : 2) wgrad_narrow(const T* __restrict__ x, const T* __restrict__ gy,
                                                    float* __restrict__ ws, BackwardProblem pr, int rows) {
  constexpr int NG = 80 / COLS, TPP = 8 * NG, PH = 256 / TPP;  // column groups, threads and phases
  extern __shared__ float nsm[];
  const int gw = nw_gw(pr.kw);
  float* sx = nsm;                          // [px][68]
  float* sg = nsm + NW_PX * (NW_CH + 4);    // [(U * gw + col) * CO + f]
  const int cb = blockIdx.y * NW_CH;
  const int ph = threadIdx.x / TPP, tl = threadIdx.x - ph * TPP;
  const int c8 = tl & 7, cgp = tl >> 3;
  const int NP = pr.kh * pr.kw * CO;
  int goff[COLS];
#pragma unroll
  for (int u = 0; u < COLS; ++u) {
    const int n = cgp + NG * u;
    const int tap = n < NP ? n / CO : 0, f = n < NP ? n - (n / CO) * CO : 0;
    const int U = tap / pr.kw, V = tap - (tap / pr.kw) * pr.kw;
    goff[u] = (U * gw + pr.kw - 1 - V) * CO + f;  // columns past NP read a valid slot, never stored
  }
  float acc[COLS][8] = {};
  const int total_rows = pr.batch * pr.in_h;
  const int r0 = blockIdx.x * rows, r1 = min(r0 + rows, total_rows);
  for (int row = r0; row < r1; ++row) {
    const int b = row / pr.in_h, i = row - (row / pr.in_h) * pr.in_h;
    for (int j0 = 0; j0 < pr.in_w; j0 += NW_PX) {
      __syncthreads();  // previous chunk's reads are done
      for (int e = threadIdx.x; e < NW_PX * (NW_CH / 4); e += blockDim.x) {
        const int px = e >> 4, c = (e & 15) * 4;
        const int j = j0 + px;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < pr.in_w) {
          const T* xp = x + ((long long)row * pr.in_w + j) * pr.cin + cb + c;
          if (sizeof(T) == 4 && cb + c + 4 <= pr.cin && (pr.cin & 3) == 0) {
            v = __ldg(reinterpret_cast<const float4*>(xp));
          } else {
            v.x = cb + c < pr.cin ? to_acc(xp[0]) : 0.f;
            v.y = cb + c + 1 < pr.cin ? to_acc(xp[1]) : 0.f;
            v.z = cb + c + 2 < pr.cin ? to_acc(xp[2]) : 0.f;
            v.w = cb + c + 3 < pr.cin ? to_acc(xp[3]) : 0.f;
          }
        }
        *reinterpret_cast<float4*>(sx + px * (NW_CH + 4) + c) = v;
      }
      nw_stage_g<T, CO>(gy, sg, pr, b, i, j0);
      __syncthreads();
      const int npx = min(NW_PX, pr.in_w - j0);
#pragma unroll 2
      for (int px = ph; px < npx; px += PH) {
        const float4 xa = *reinterpret_cast<const float4*>(sx + px * (NW_CH + 4) + 8 * c8);
        const float4 xb = *reinterpret_cast<const float4*>(sx + px * (NW_CH + 4) + 8 * c8 + 4);
        const float* gp = sg + 2 * px * CO;
#pragma unroll
        for (int u = 0; u < COLS; ++u) {
          const float g = gp[goff[u]];
          acc[u][0] = fmaf(xa.x, g, acc[u][0]);
          acc[u][1] = fmaf(xa.y, g, acc[u][1]);
          acc[u][2] = fmaf(xa.z, g, acc[u][2]);
          acc[u][3] = fmaf(xa.w, g, acc[u][3]);
          acc[u][4] = fmaf(xb.x, g, acc[u][4]);
          acc[u][5] = fmaf(xb.y, g, acc[u][5]);
          acc[u][6] = fmaf(xb.z, g, acc[u][6]);
          acc[u][7] = fmaf(xb.w, g, acc[u][7]);
        }
      }
    }
  }
  const long long ksz = (long long)pr.kh * pr.kw * pr.cin * CO;
  float* out = ws + ((long long)blockIdx.x * PH + ph) * ksz;
#pragma unroll
  for (int u = 0; u < COLS; ++u) {
    const int n = cgp + NG * u;
    if (n >= NP) continue;
    const int tap = n / CO, f = n - (n / CO) * CO;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ch = cb + 8 * c8 + c;
      if (ch < pr.cin) out[((long long)tap * pr.cin + ch) * CO + f] = acc[u][c];
    }
  }
}
}  // namespace bwd

static int sm_count() {
  const int sms = device_sm_count();
  return sms;
}

bool bwd_narrow_applies(const BackwardProblem& pr) {
  return !pr.conv && pr.stride == 2 && pr.in_w >= 64 && pr.cout >= 1 && pr.cout <= 4 && pr.kh <= bwd::NW_MAXK &&
         pr.kw <= bwd::NW_MAXK && pr.kh * pr.kw * pr.cout <= 80 && pr.in_h == pr.n && pr.in_w == pr.n &&
         (pr.dtype == SEGCONV_F32 || pr.dtype == SEGCONV_BF16);
}

template <typename T, int CO>
static cudaError_t narrow_dgrad_t(const BackwardProblem& pr, cudaStream_t s) {
  const int gw = bwd::nw_gw(pr.kw);
  const size_t smem = ((size_t)pr.kh * pr.kw * CO * bwd::NW_CH + (size_t)pr.kh * gw * CO) * sizeof(float);
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, bwd::dgrad_narrow<T, CO>, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const long long rows = (long long)pr.batch * pr.in_h;
  const long long yz = (long long)((pr.in_w + bwd::NW_PX - 1) / bwd::NW_PX) * ((pr.cin + bwd::NW_CH - 1) / bwd::NW_CH);
  const long long gx_rows = std::max(1LL, std::min(rows, (8LL * sm_count() + yz - 1) / yz));  // ~8 CTAs per SM
  dim3 grid((unsigned)gx_rows, (unsigned)((pr.in_w + bwd::NW_PX - 1) / bwd::NW_PX),
            (unsigned)((pr.cin + bwd::NW_CH - 1) / bwd::NW_CH));
  bwd::dgrad_narrow<T, CO><<<grid, 256, smem, s>>>((const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) note_launch();
  return e;
}

template <typename T>
static cudaError_t narrow_dgrad(const BackwardProblem& pr, cudaStream_t s) {
  switch (pr.cout) {
    case 1: return narrow_dgrad_t<T, 1>(pr, s);
    case 2: return narrow_dgrad_t<T, 2>(pr, s);
    case 3: return narrow_dgrad_t<T, 3>(pr, s);
    default: return narrow_dgrad_t<T, 4>(pr, s);
  }
}

template <typename T, int CO>
static cudaError_t narrow_wgrad_t(const BackwardProblem& pr, cudaStream_t s) {
  const int gw = bwd::nw_gw(pr.kw);
  const size_t smem = ((size_t)bwd::NW_PX * (bwd::NW_CH + 4) + (size_t)pr.kh * gw * CO) * sizeof(float);
  static PerDeviceOnce once5;
  {
    const cudaError_t e = smem_attr_once(once5, bwd::wgrad_narrow<T, CO, 5>, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int chb = (pr.cin + bwd::NW_CH - 1) / bwd::NW_CH;
  const long long total_rows = (long long)pr.batch * pr.in_h;
  // a few CTAs per SM over (row range, channel block)
  constexpr int cps = 3;
  long long rows = std::max(1LL, (total_rows * chb + (long long)cps * sm_count() - 1) / ((long long)cps * sm_count()));
  const long long splits = (total_rows + rows - 1) / rows;
  const long long ksz = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
  float* ws = nullptr;
  constexpr int phases = 2;  // 5 (tap, f) columns per thread, two pixel phases
  cudaError_t e = workspace_alloc((void**)&ws, (size_t)splits * phases * ksz * sizeof(float), s);
  if (e != cudaSuccess) return e;
  bwd::wgrad_narrow<T, CO, 5><<<dim3((unsigned)splits, (unsigned)chb), 256, smem, s>>>(
      (const T*)pr.x, (const T*)pr.gy, ws, pr, (int)rows);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    note_launch();
    e = launch_wgrad_reduce(ws, (float*)pr.gk, ksz, (int)splits * phases, pr.accumulate, s);
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  return e != cudaSuccess ? e : e2;
}

template <typename T>
static cudaError_t narrow_wgrad(const BackwardProblem& pr, cudaStream_t s) {
  switch (pr.cout) {
    case 1: return narrow_wgrad_t<T, 1>(pr, s);
    case 2: return narrow_wgrad_t<T, 2>(pr, s);
    case 3: return narrow_wgrad_t<T, 3>(pr, s);
    default: return narrow_wgrad_t<T, 4>(pr, s);
  }
}

template <typename T>
static cudaError_t bwd_data_t(const BackwardProblem& pr, bool exact, cudaStream_t s) {
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  if (M == 0) return cudaSuccess;
  if (exact) {
    if constexpr (sizeof(T) == 2) return cudaErrorNotSupported;
    else {
      const long long total = M * pr.cin;
      if (pr.conv)
        bwd::conv_dgrad_exact<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
            (const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
      else
        bwd::dgrad_exact<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
            (const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
    }
  } else if (sizeof(T) <= 4 && bwd_narrow_applies(pr)) {
    if constexpr (sizeof(T) <= 4) return narrow_dgrad<T>(pr, s);
  } else {
    using ACC = typename std::conditional<sizeof(T) == 8, double, float>::type;
    dim3 grid((unsigned)((M + bwd::BM - 1) / bwd::BM), (unsigned)((pr.cin + bwd::BN - 1) / bwd::BN));
    if (pr.cout % bwd::BK != 0)
      bwd::dgrad_ffma_packed<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
    else
      bwd::dgrad_ffma<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) note_launch();
  return e;
}

cudaError_t launch_bwd_data_simt(const BackwardProblem& pr, bool exact, cudaStream_t s) {
  if (pr.dtype == SEGCONV_F32) return bwd_data_t<float>(pr, exact, s);
  if (pr.dtype == SEGCONV_F64) return bwd_data_t<double>(pr, exact, s);
  if (pr.dtype == SEGCONV_BF16) return bwd_data_t<__nv_bfloat16>(pr, exact, s);
  return cudaErrorNotSupported;
}

template <typename T>
static cudaError_t bwd_weight_t(const BackwardProblem& pr, bool exact, cudaStream_t s) {
  using ACC = typename std::conditional<sizeof(T) == 8, double, float>::type;
  const long long ksz = (long long)pr.kh * pr.kw * pr.cin * pr.cout;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  if (exact) {
    if constexpr (sizeof(T) == 2) return cudaErrorNotSupported;
    else {
      if (pr.conv)
        bwd::conv_wgrad_exact<T><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>((const T*)pr.x, (const T*)pr.gy,
                                                                                 (T*)pr.gk, pr);
      else
        bwd::wgrad_exact<T><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>((const T*)pr.x, (const T*)pr.gy,
                                                                          (T*)pr.gk, pr);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) note_launch();
      return e;
    }
  }
  if constexpr (sizeof(T) <= 4) {
    if (bwd_narrow_applies(pr) && M > 0) return narrow_wgrad<T>(pr, s);
  }
  // cout % 64 != 0: (tap, f) packed columns, all taps of a tile in one CTA
  const bool packed = pr.cout % bwd::BN != 0;
  const int taps = pr.kh * pr.kw;
  const int ntile = packed ? (taps * pr.cout + bwd::BN - 1) / bwd::BN : (pr.cout + bwd::BN - 1) / bwd::BN;
  const int tiles = ((pr.cin + bwd::BM - 1) / bwd::BM) * ntile * (packed ? 1 : taps);
  // split the pixel reduction until ~CPS CTAs per SM (latency hiding for the
  // gathers), keeping >= 256 pixels per split
  constexpr int cps = 4;
  long long splits = std::max(1LL, ((long long)cps * sm_count() + tiles - 1) / tiles);
  splits = std::min(splits, std::max(1LL, M / 256));
  if (M == 0) splits = 1;
  long long chunk = (M + splits - 1) / splits;
  chunk = std::max<long long>(bwd::BK, (chunk + bwd::BK - 1) / bwd::BK * bwd::BK);
  splits = std::max(1LL, (M + chunk - 1) / chunk);
  dim3 grid((unsigned)((pr.cin + bwd::BM - 1) / bwd::BM), (unsigned)ntile,
            (unsigned)((packed ? 1 : taps) * splits));
  auto launch = [&](ACC* out, int direct) {
    if (packed)
      bwd::wgrad_ffma_packed<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.x, (const T*)pr.gy, out, pr,
                                                              (int)splits, chunk, direct);
    else
      bwd::wgrad_ffma<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.x, (const T*)pr.gy, out, pr, (int)splits,
                                                       chunk, direct);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
  };
  if (splits == 1) return launch((ACC*)pr.gk, 1);
  ACC* ws = nullptr;
  cudaError_t e = workspace_alloc((void**)&ws, (size_t)splits * ksz * sizeof(ACC), s);
  if (e != cudaSuccess) return e;
  e = launch(ws, 0);
  if (e == cudaSuccess) {
    if constexpr (std::is_same<ACC, float>::value) {
      // float4 / split-group reduction (C2: 118 splits of 18432 partials took
      // 14 us in the scalar walk over 72 CTAs)
      e = launch_wgrad_reduce(ws, (float*)pr.gk, ksz, (int)splits, pr.accumulate, s);
    } else {
      bwd::wgrad_reduce<ACC><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>(ws, (ACC*)pr.gk, ksz, (int)splits,
                                                                          pr.accumulate);
      e = cudaGetLastError();
      if (e == cudaSuccess) note_launch();
    }
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  return e != cudaSuccess ? e : e2;
}

// Split-K partial sums live in a library-owned stream-ordered pool whose
// release threshold keeps freed blocks mapped (the default pool returns them to
// the OS at every synchronisation, making each call pay a fresh mapping).
cudaError_t workspace_alloc(void** p, size_t bytes, cudaStream_t s) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;  // pool creation only; allocation itself is stream-ordered
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) {
        pools[dev] = nullptr;
        return e;
      }
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

cudaError_t launch_wgrad_reduce(const float* ws, float* gk, long long ksz, int splits, int accumulate,
                                cudaStream_t s) {
  if (ksz % 4 == 0 && ((uintptr_t)ws & 15) == 0 && ((uintptr_t)gk & 15) == 0) {
    const long long n4 = ksz / 4;
    if (splits >= 64 && (n4 + 255) / 256 < 2LL * sm_count())  // too few threads to walk the splits
      bwd::wgrad_reduce4_wide<<<(unsigned)((n4 + 7) / 8), 256, 0, s>>>((const float4*)ws, (float4*)gk, n4,
                                                                        splits, accumulate);
    else
      bwd::wgrad_reduce4<<<(unsigned)((n4 + 255) / 256), 256, 0, s>>>((const float4*)ws, (float4*)gk, n4, splits,
                                                                       accumulate);
  } else {
    bwd::wgrad_reduce<float><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>(ws, gk, ksz, splits, accumulate);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) note_launch();
  return e;
}

cudaError_t launch_bwd_weight_simt(const BackwardProblem& pr, bool exact, cudaStream_t s) {
  if (pr.dtype == SEGCONV_F32) return bwd_weight_t<float>(pr, exact, s);
  if (pr.dtype == SEGCONV_F64) return bwd_weight_t<double>(pr, exact, s);
  if (pr.dtype == SEGCONV_BF16) return bwd_weight_t<__nv_bfloat16>(pr, exact, s);
  return cudaErrorNotSupported;
}

}  // namespace segconv_b200

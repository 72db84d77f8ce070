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

// ------------------------------------------------------------- FFMA tiles
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

// gx tile: 64 pixels x 64 input channels, K = taps x cout in 16-feature steps.
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) dgrad_ffma(const T* __restrict__ gy, const T* __restrict__ k,
                                                 T* __restrict__ gx, BackwardProblem pr) {
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.n * pr.n;
  const long long m0 = (long long)blockIdx.x * BM;
  const int ch0 = blockIdx.y * BN;
  const int lp = tid >> 2, lf = (tid & 3) * 4;  // loader: row lp, 4 consecutive features
  const long long m = m0 + lp;
  const bool mv = m < M;
  const int j = mv ? (int)(m % pr.n) : 0, i = mv ? (int)((m / pr.n) % pr.n) : 0;
  const int b = mv ? (int)(m / ((long long)pr.n * pr.n)) : 0;
  const bool kv = ch0 + lp < pr.cin;
  ACC acc[4][4] = {};
  for (int t = 0; t < pr.kh * pr.kw; ++t) {
    const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
    const int y = 2 * i + pr.p - U, xx = 2 * j + pr.p - V;
    const bool av = mv && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w;
    const T* gp = gy + (((long long)b * pr.out_h + (av ? y : 0)) * pr.out_w + (av ? xx : 0)) * pr.cout;
    const T* kp = k + ((long long)t * pr.cin + (kv ? ch0 + lp : 0)) * pr.cout;
    for (int f0 = 0; f0 < pr.cout; f0 += BK) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int f = f0 + lf + e;
        As[lf + e][lp] = (av && f < pr.cout) ? ld<ACC>(gp + f) : ACC(0);
        Bs[lf + e][lp] = (kv && f < pr.cout) ? ld<ACC>(kp + f) : ACC(0);
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

// gk tile: 64 input channels x 64 features of one tap over a pixel range.
template <typename T, typename ACC>
__global__ void __launch_bounds__(NT) wgrad_ffma(const T* __restrict__ x, const T* __restrict__ gy,
                                                 ACC* __restrict__ out, BackwardProblem pr, int splits,
                                                 long long chunk, int direct) {
  __shared__ ACC As[BK][BM + 4];
  __shared__ ACC Bs[BK][BN + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long M = (long long)pr.batch * pr.n * pr.n;
  const int ch0 = blockIdx.x * BM, f0 = blockIdx.y * BN;
  const int t = blockIdx.z / splits, s = blockIdx.z - (blockIdx.z / splits) * splits;
  const int U = t / pr.kw, V = t - (t / pr.kw) * pr.kw;
  const long long mb = (long long)s * chunk, me = (mb + chunk < M) ? mb + chunk : M;
  const int lp = tid >> 4, lc = (tid & 15) * 4;  // loader: pixel lp, 4 consecutive channels
  ACC acc[4][4] = {};
  for (long long mk = mb; mk < me; mk += BK) {
    const long long m = mk + lp;
    const bool mv = m < me;
    const int j = mv ? (int)(m % pr.n) : 0, i = mv ? (int)((m / pr.n) % pr.n) : 0;
    const int b = mv ? (int)(m / ((long long)pr.n * pr.n)) : 0;
    const int y = 2 * i + pr.p - U, xx = 2 * j + pr.p - V;
    const bool gv = mv && y >= 0 && y < pr.out_h && xx >= 0 && xx < pr.out_w;
    const T* xp = x + (mv ? m : 0) * pr.cin;
    const T* gp = gy + (((long long)b * pr.out_h + (gv ? y : 0)) * pr.out_w + (gv ? xx : 0)) * pr.cout;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ch = ch0 + lc + e, f = f0 + lc + e;
      As[lp][lc + e] = (gv && ch < pr.cin) ? ld<ACC>(xp + ch) : ACC(0);
      Bs[lp][lc + e] = (gv && f < pr.cout) ? ld<ACC>(gp + f) : ACC(0);
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

}  // namespace bwd

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  return sms;
}

template <typename T>
static cudaError_t bwd_data_t(const BackwardProblem& pr, bool exact, cudaStream_t s) {
  const long long M = (long long)pr.batch * pr.n * pr.n;
  if (M == 0) return cudaSuccess;
  if (exact) {
    if constexpr (sizeof(T) == 2) return cudaErrorNotSupported;
    else {
      const long long total = M * pr.cin;
      bwd::dgrad_exact<T><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
          (const T*)pr.gy, (const T*)pr.k, (T*)pr.gx, pr);
    }
  } else {
    using ACC = typename std::conditional<sizeof(T) == 8, double, float>::type;
    dim3 grid((unsigned)((M + bwd::BM - 1) / bwd::BM), (unsigned)((pr.cin + bwd::BN - 1) / bwd::BN));
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
  const long long M = (long long)pr.batch * pr.n * pr.n;
  if (exact) {
    if constexpr (sizeof(T) == 2) return cudaErrorNotSupported;
    else {
      bwd::wgrad_exact<T><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>((const T*)pr.x, (const T*)pr.gy,
                                                                        (T*)pr.gk, pr);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) note_launch();
      return e;
    }
  }
  const int tiles = ((pr.cin + bwd::BM - 1) / bwd::BM) * ((pr.cout + bwd::BN - 1) / bwd::BN) * pr.kh * pr.kw;
  // split the pixel reduction until ~2 CTAs per SM, keeping >= 512 pixels per split
  long long splits = std::max(1LL, (2LL * sm_count() + tiles - 1) / tiles);
  splits = std::min(splits, std::max(1LL, M / 512));
  if (M == 0) splits = 1;
  long long chunk = (M + splits - 1) / splits;
  chunk = std::max<long long>(bwd::BK, (chunk + bwd::BK - 1) / bwd::BK * bwd::BK);
  splits = std::max(1LL, (M + chunk - 1) / chunk);
  dim3 grid((unsigned)((pr.cin + bwd::BM - 1) / bwd::BM), (unsigned)((pr.cout + bwd::BN - 1) / bwd::BN),
            (unsigned)(pr.kh * pr.kw * splits));
  if (splits == 1) {
    bwd::wgrad_ffma<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.x, (const T*)pr.gy, (ACC*)pr.gk, pr, 1,
                                                     std::max(chunk, 1LL), 1);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
    return e;
  }
  ACC* ws = nullptr;
  cudaError_t e = workspace_alloc((void**)&ws, (size_t)splits * ksz * sizeof(ACC), s);
  if (e != cudaSuccess) return e;
  bwd::wgrad_ffma<T, ACC><<<grid, bwd::NT, 0, s>>>((const T*)pr.x, (const T*)pr.gy, ws, pr, (int)splits,
                                                   chunk, 0);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    note_launch();
    bwd::wgrad_reduce<ACC><<<(unsigned)((ksz + 255) / 256), 256, 0, s>>>(ws, (ACC*)pr.gk, ksz, (int)splits,
                                                                        pr.accumulate);
    e = cudaGetLastError();
    if (e == cudaSuccess) note_launch();
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  return e != cudaSuccess ? e : e2;
}

// Split-K partial sums live in a library-owned stream-ordered pool whose
// release threshold keeps freed blocks mapped (the default pool returns them to
// the OS at every synchronisation, making each call pay a fresh mapping).
cudaError_t workspace_alloc(void** p, size_t bytes, cudaStream_t s) {
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, s);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
  }
  return cudaMallocFromPoolAsync(p, bytes, pools[dev], s);
}

cudaError_t launch_wgrad_reduce(const float* ws, float* gk, long long ksz, int splits, int accumulate,
                                cudaStream_t s) {
  if (ksz % 4 == 0 && ((uintptr_t)ws & 15) == 0 && ((uintptr_t)gk & 15) == 0) {
    const long long n4 = ksz / 4;
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

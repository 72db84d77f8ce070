// conventional.cu -- K5/K6: the conventional upsample + pad + valid-correlate
// path, the baseline the segregated path is compared against.
//
// Replaces reference proj/include/segconv/tensor.hpp:224-259 (pad,
// upsample2x) and reference_ops.hpp:86-133 (conv2d_valid,
// transpose_conv_naive).  It deliberately materialises the (2N-1+2p)^2 map in
// HBM and multiplies the inserted zeros, as the reference does; it is built
// in the same run for comparison and not optimised beyond a reasonable tiled
// SIMT kernel.
#include <algorithm>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace segconv_b200 {

template <typename T>
__global__ void upsample_pad_kernel(const T* __restrict__ x, int batch, int n, int cin, int p,
                                    T* __restrict__ up) {
  const int U = 2 * n - 1 + 2 * p;
  const long long total = (long long)batch * U * U * cin;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(e % cin);
    long long t = e / cin;
    const int col = (int)(t % U);
    t /= U;
    const int row = (int)(t % U);
    const int b = (int)(t / U);
    const int rr = row - p, cc = col - p;
    T v = T(0);
    if (rr >= 0 && cc >= 0 && !(rr & 1) && !(cc & 1) && (rr >> 1) < n && (cc >> 1) < n)
      v = x[(((long long)b * n + (rr >> 1)) * n + (cc >> 1)) * cin + ch];
    up[e] = v;
  }
}

cudaError_t launch_upsample_pad(const void* x, int dtype, int batch, int n, int cin, int p,
                                void* up, cudaStream_t s) {
  const long long U = 2LL * n - 1 + 2LL * p;
  const long long total = (long long)batch * U * U * cin;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 64);
  if (dtype == SEGCONV_F32)
    upsample_pad_kernel<float><<<blocks, 256, 0, s>>>((const float*)x, batch, n, cin, p, (float*)up);
  else if (dtype == SEGCONV_F64)
    upsample_pad_kernel<double><<<blocks, 256, 0, s>>>((const double*)x, batch, n, cin, p,
                                                       (double*)up);
  else if (dtype == SEGCONV_BF16)
    upsample_pad_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(
        (const __nv_bfloat16*)x, batch, n, cin, p, (__nv_bfloat16*)up);
  else
    return cudaErrorInvalidValue;
  note_launch();
  return cudaGetLastError();
}

// Backward of pad(upsample2x(x), p): gx(i, j) = g(2i + p, 2j + p) -- the
// reference Upsample2x::backward (netdemo/layers.hpp:66-73) after the crop of
// the padding (tensor.hpp:224-232).
template <typename T>
__global__ void upsample_pad_backward_kernel(const T* __restrict__ g, int batch, int n, int cin, int p,
                                             T* __restrict__ gx) {
  const long long U = 2LL * n - 1 + 2LL * p;
  const long long total = (long long)batch * n * n * cin;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(e % cin);
    long long t = e / cin;
    const int j = (int)(t % n);
    t /= n;
    const int i = (int)(t % n);
    const long long b = t / n;
    gx[e] = g[((b * U + 2 * i + p) * U + 2 * j + p) * cin + ch];
  }
}

cudaError_t launch_upsample_pad_backward(const void* g, int dtype, int batch, int n, int cin, int p, void* gx,
                                         cudaStream_t s) {
  const long long total = (long long)batch * n * n * cin;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 64);
  if (dtype == SEGCONV_F32)
    upsample_pad_backward_kernel<float><<<blocks, 256, 0, s>>>((const float*)g, batch, n, cin, p, (float*)gx);
  else if (dtype == SEGCONV_F64)
    upsample_pad_backward_kernel<double><<<blocks, 256, 0, s>>>((const double*)g, batch, n, cin, p,
                                                                (double*)gx);
  else if (dtype == SEGCONV_BF16)
    upsample_pad_backward_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>(
        (const __nv_bfloat16*)g, batch, n, cin, p, (__nv_bfloat16*)gx);
  else
    return cudaErrorInvalidValue;
  note_launch();
  return cudaGetLastError();
}

// Generic valid correlation: one thread per output element (any shape/dtype).
// EXACT: the reference's (u, v, ch) order with separate multiply and add
// (accumulate_window, reference_ops.hpp:31-79, built with -ffp-contract=off).
template <typename T, typename ACC, bool EXACT = false>
__global__ void __launch_bounds__(256)
    conv_valid_generic(const T* __restrict__ src, int batch, int h, int w, int cin,
                       const T* __restrict__ k, int kh, int kw, int cout, const float* bias,
                       unsigned epi, T* __restrict__ y) {
  const int oh = h - kh + 1, ow = w - kw + 1;
  const long long total = (long long)batch * oh * ow * cout;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(e % cout);
    long long t = e / cout;
    const int ox = (int)(t % ow);
    t /= ow;
    const int oy = (int)(t % oh);
    const int b = (int)(t / oh);
    ACC acc = 0;
    for (int u = 0; u < kh; ++u)
      for (int v = 0; v < kw; ++v) {
        const T* sp = src + (((long long)b * h + oy + u) * w + ox + v) * cin;
        const T* kp = k + ((long long)(u * kw + v) * cin) * cout + f;
        for (int ch = 0; ch < cin; ++ch) {
          const ACC a = (ACC)to_acc(sp[ch]), bw = (ACC)to_acc(kp[(long long)ch * cout]);
          if constexpr (!EXACT)
            acc = fma(a, bw, acc);
          else if constexpr (sizeof(ACC) == 8)
            acc = __dadd_rn(acc, __dmul_rn(a, bw));
          else
            acc = __fadd_rn(acc, __fmul_rn(a, bw));
        }
      }
    y[e] = from_d<T>((double)epilogue_apply(acc, epi, bias, f));
  }
}

// Tiled fp32 valid correlation for square K <= 7: a CTA computes a
// (WH*QH) x QW pixel tile for 32 output features (lanes = features), the
// input halo is a broadcast read from shared memory.
template <int K, int QH, int QW, int WH, int CI>
__global__ void __launch_bounds__(WH * 32)
    conv_valid_tiled(const float* __restrict__ src, int batch, int h, int w, int cin,
                     const float* __restrict__ k, int cout, const float* bias, unsigned epi,
                     float* __restrict__ y, int tiles_h, int tiles_w) {
  constexpr int TH = WH * QH + K - 1, TW = QW + K - 1, TWP = (TW + 3) & ~3, NT = WH * 32;
  extern __shared__ float4 smem4[];
  float* xs = reinterpret_cast<float*>(smem4);
  float* ws = xs + CI * TH * TWP;
  const int oh = h - K + 1, ow = w - K + 1;
  const int tid = threadIdx.x, lane = tid & 31, wh = tid >> 5;
  int tile = blockIdx.x;
  const int tj = tile % tiles_w;
  tile /= tiles_w;
  const int ti = tile % tiles_h;
  const int b = tile / tiles_h;
  const int y0 = ti * WH * QH, x0 = tj * QW, f0 = blockIdx.y * 32;
  float acc[QH][QW];
#pragma unroll
  for (int a = 0; a < QH; ++a)
#pragma unroll
    for (int bb = 0; bb < QW; ++bb) acc[a][bb] = 0.f;
  for (int ci0 = 0; ci0 < cin; ci0 += CI) {
    __syncthreads();
    for (int idx = tid; idx < TH * TW * CI; idx += NT) {
      const int ch = idx % CI, pix = idx / CI, row = pix / TW, col = pix % TW;
      const int gr = y0 + row, gc = x0 + col, gch = ci0 + ch;
      float v = 0.f;
      if (gr < h && gc < w && gch < cin) v = src[(((long long)b * h + gr) * w + gc) * cin + gch];
      xs[(ch * TH + row) * TWP + col] = v;
    }
    for (int idx = tid; idx < CI * K * K * 32; idx += NT) {
      const int fl = idx % 32, t = (idx / 32) % (K * K), ch = idx / (32 * K * K);
      const int f = f0 + fl, gch = ci0 + ch;
      ws[idx] = (f < cout && gch < cin) ? k[((long long)t * cin + gch) * cout + f] : 0.f;
    }
    __syncthreads();
    const int nch = min(CI, cin - ci0);
    for (int ch = 0; ch < nch; ++ch) {
      const float* xb = xs + (ch * TH + wh * QH) * TWP;
      const float* wl = ws + ch * K * K * 32 + lane;
#pragma unroll
      for (int u = 0; u < K; ++u)
#pragma unroll
        for (int v = 0; v < K; ++v) {
          const float wv = wl[(u * K + v) * 32];
#pragma unroll
          for (int a = 0; a < QH; ++a)
#pragma unroll
            for (int bb = 0; bb < QW; ++bb)
              acc[a][bb] = fmaf(xb[(a + u) * TWP + bb + v], wv, acc[a][bb]);
        }
    }
  }
  const int f = f0 + lane;
  if (f >= cout) return;
#pragma unroll
  for (int a = 0; a < QH; ++a) {
    const int oy = y0 + wh * QH + a;
    if (oy >= oh) continue;
#pragma unroll
    for (int bb = 0; bb < QW; ++bb) {
      const int ox = x0 + bb;
      if (ox >= ow) continue;
      y[(((long long)b * oh + oy) * ow + ox) * cout + f] = epilogue_apply(acc[a][bb], epi, bias, f);
    }
  }
}

template <int K>
static cudaError_t run_conv_tiled(const float* src, int batch, int h, int w, int cin,
                                  const float* k, int cout, const float* bias, unsigned epi,
                                  float* y, cudaStream_t s) {
  constexpr int QH = 2, QW = 8, WH = 4, CI = 16;
  constexpr int TH = WH * QH + K - 1, TW = QW + K - 1, TWP = (TW + 3) & ~3;
  const size_t smem = (size_t)(CI * TH * TWP + CI * K * K * 32) * sizeof(float);
  auto kern = conv_valid_tiled<K, QH, QW, WH, CI>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int oh = h - K + 1, ow = w - K + 1;
  const int tiles_h = (oh + WH * QH - 1) / (WH * QH), tiles_w = (ow + QW - 1) / QW;
  const long long blocks = (long long)tiles_h * tiles_w * batch;
  if (blocks == 0) return cudaSuccess;
  dim3 grid((unsigned)blocks, (cout + 31) / 32);
  kern<<<grid, WH * 32, smem, s>>>(src, batch, h, w, cin, k, cout, bias, epi, y, tiles_h, tiles_w);
  note_launch();
  return cudaGetLastError();
}

// (taps, cin, cout) -> (cout, taps, cin): the K-major B operand of the
// tensor-core valid correlation
__global__ void kmajor_transpose(const __nv_bfloat16* __restrict__ k, int taps, int cin, int cout,
                                 __nv_bfloat16* __restrict__ kt) {
  const long long total = (long long)taps * cin * cout;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(e % cin);
    const long long r = e / cin;
    const int t = (int)(r % taps), f = (int)(r / taps);
    kt[e] = k[((long long)t * cin + ch) * cout + f];
  }
}

cudaError_t launch_conv2d_valid(const void* src, int dtype, int batch, int h, int w, int cin,
                                const void* k, int kh, int kw, int cout, const float* bias,
                                unsigned epi, bool exact, void* y, cudaStream_t s) {
  const long long total = (long long)batch * (h - kh + 1) * (w - kw + 1) * cout;
  if (total <= 0) return cudaSuccess;
  if (exact) {
    const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 64);
    if (dtype == SEGCONV_F32)
      conv_valid_generic<float, float, true><<<blocks, 256, 0, s>>>(
          (const float*)src, batch, h, w, cin, (const float*)k, kh, kw, cout, bias, epi, (float*)y);
    else if (dtype == SEGCONV_F64)
      conv_valid_generic<double, double, true><<<blocks, 256, 0, s>>>(
          (const double*)src, batch, h, w, cin, (const double*)k, kh, kw, cout, bias, epi, (double*)y);
    else
      return cudaErrorInvalidValue;
    note_launch();
    return cudaGetLastError();
  }
  if (dtype == SEGCONV_BF16 && tc_conv_valid_supported(batch, h, w, cin, kh, kw, cout)) {
    const long long kn = (long long)kh * kw * cin * cout;
    void* kt = nullptr;
    cudaError_t e = workspace_alloc(&kt, (size_t)kn * 2, s);
    if (e != cudaSuccess) return e;
    kmajor_transpose<<<(unsigned)std::min<long long>((kn + 255) / 256, 148LL * 16), 256, 0, s>>>(
        (const __nv_bfloat16*)k, kh * kw, cin, cout, (__nv_bfloat16*)kt);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
      note_launch();
      e = launch_tc_conv_valid(src, batch, h, w, cin, kt, kh, kw, cout, bias, epi, y, s);
    }
    const cudaError_t e2 = cudaFreeAsync(kt, s);
    return e != cudaSuccess ? e : e2;
  }
  if (dtype == SEGCONV_F32 && kh == kw && cout > 4) {
    const float* sp = (const float*)src;
    const float* kp = (const float*)k;
    float* yp = (float*)y;
    switch (kh) {
      case 3: return run_conv_tiled<3>(sp, batch, h, w, cin, kp, cout, bias, epi, yp, s);
      case 4: return run_conv_tiled<4>(sp, batch, h, w, cin, kp, cout, bias, epi, yp, s);
      case 5: return run_conv_tiled<5>(sp, batch, h, w, cin, kp, cout, bias, epi, yp, s);
      default: break;
    }
  }
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 64);
  if (dtype == SEGCONV_F32)
    conv_valid_generic<float, float><<<blocks, 256, 0, s>>>(
        (const float*)src, batch, h, w, cin, (const float*)k, kh, kw, cout, bias, epi, (float*)y);
  else if (dtype == SEGCONV_F64)
    conv_valid_generic<double, double><<<blocks, 256, 0, s>>>(
        (const double*)src, batch, h, w, cin, (const double*)k, kh, kw, cout, bias, epi,
        (double*)y);
  else if (dtype == SEGCONV_BF16)
    conv_valid_generic<__nv_bfloat16, float><<<blocks, 256, 0, s>>>(
        (const __nv_bfloat16*)src, batch, h, w, cin, (const __nv_bfloat16*)k, kh, kw, cout, bias,
        epi, (__nv_bfloat16*)y);
  else
    return cudaErrorInvalidValue;
  note_launch();
  return cudaGetLastError();
}

}  // namespace segconv_b200

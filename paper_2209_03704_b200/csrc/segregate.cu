// segregate.cu -- K1: on-device sub-kernel extraction into the four parity panels.
//
// Replaces reference proj/include/segconv/segregation.hpp:61-89 (segregate):
// sub_rc[u][v][ch][f] = k[u0_r + 2u][v0_c + 2v][ch][f], taps kept in their
// relative (u-major, v) order, class index r*2 + c.  One pass over the panel
// elements (gather; each source tap is read exactly once), with dtype
// conversion and, for the tensor-core path, re-layout to K-major
// (cout_pad, u, v, cin) rows so a panel row is one MMA B-operand row.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tc_guard.cuh"

namespace segconv_b200 {

template <typename TK, typename TP>
__global__ void segregate_kernel(const TK* __restrict__ k, int kh, int kw, int cin, int cout,
                                 int cout_pad, int layout, SegClasses cls, TP* __restrict__ panels,
                                 long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int q = 0;
#pragma unroll
    for (int t = 1; t < 4; ++t)
      if (e >= cls.sub_offset[t]) q = t;
    long long o = e - cls.sub_offset[q];
    const int skw = cls.kw[q];
    int u, v, ch, f;
    if (layout == SEGCONV_PANEL_REF) {  // (u, v, ch, f)
      f = (int)(o % cout);
      o /= cout;
      ch = (int)(o % cin);
      o /= cin;
      v = (int)(o % skw);
      u = (int)(o / skw);
    } else {  // (f, u, v, ch), f < cout_pad
      ch = (int)(o % cin);
      o /= cin;
      v = (int)(o % skw);
      o /= skw;
      u = (int)(o % cls.kh[q]);
      f = (int)(o / cls.kh[q]);
    }
    float val = 0.0f;
    double vald = 0.0;
    if (f < cout) {
      const long long src =
          (((long long)(cls.u0[q] + 2 * u) * kw + (cls.v0[q] + 2 * v)) * cin + ch) * cout + f;
      vald = (double)to_acc(k[src]);
      val = (float)vald;
    }
    if constexpr (DT<TP>::id == SEGCONV_F64)
      panels[e] = (TP)vald;
    else
      panels[e] = from_f<TP>(val);
  }
}

template <typename TK, typename TP>
static cudaError_t launch_seg(const void* k, int kh, int kw, int cin, int cout, int cout_pad,
                              int layout, const SegClasses& cls, void* panels, long long total,
                              cudaStream_t s) {
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  segregate_kernel<TK, TP><<<(unsigned)blocks, threads, 0, s>>>(
      (const TK*)k, kh, kw, cin, cout, cout_pad, layout, cls, (TP*)panels, total);
  note_launch();
  return cudaGetLastError();
}

// K-major split panels for the pair kernel's fp32 mode: per class rows
// (f < cout_pad, u, v) of 2 cin fp16 values, [hi(w'[ch]) | lo(w'[ch])] with
// w' = w * 2^s = hi + lo (hi = rn(w'), lo = rn(w' - hi)).  The power-of-two
// scale puts max |w'| at 2^14, so the lo halves of small weights stay out of
// the fp16 subnormal range; the kernel multiplies its sums by 2^-s (exact),
// stored after the panels: tail[0] = max |w| (bits), tail[1] = 2^-s.
template <typename TK>
__global__ void kernel_amax(const TK* __restrict__ k, long long n, unsigned* __restrict__ amax_bits) {
  float m = 0.0f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf((float)to_acc(k[e])));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, __float_as_uint(m));  // non-negative floats order as uints
}


template <typename TK>
__global__ void segregate_kmajor_split_kernel(const TK* __restrict__ k, int kw, int cin, int cout, SegClasses cls,
                                              __half* __restrict__ panels, long long total,
                                              const unsigned* __restrict__ amax_bits, float* __restrict__ inv_scale) {
  const int cin2 = 2 * cin;
  const float scale = ldexpf(1.0f, split_scale_exp(*amax_bits));
  if (blockIdx.x == 0 && threadIdx.x == 0) *inv_scale = 1.0f / scale;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int q = 0;
#pragma unroll
    for (int t = 1; t < 4; ++t)
      if (e >= cls.sub_offset[t]) q = t;
    long long o = e - cls.sub_offset[q];
    const int c2 = (int)(o % cin2);
    o /= cin2;
    const int v = (int)(o % cls.kw[q]);
    o /= cls.kw[q];
    const int u = (int)(o % cls.kh[q]);
    const int f = (int)(o / cls.kh[q]);
    const int ch = c2 < cin ? c2 : c2 - cin;
    float w = 0.0f;
    if (f < cout)
      w = scale * (float)to_acc(k[(((long long)(cls.u0[q] + 2 * u) * kw + (cls.v0[q] + 2 * v)) * cin + ch) * cout + f]);
    const __half hi = __float2half_rn(w);
    panels[e] = c2 < cin ? hi : __float2half_rn(w - __half2float(hi));
  }
}

cudaError_t launch_segregate_kmajor_split(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                          int cout_pad, const SegClasses& cls, void* panels, long long total,
                                          cudaStream_t s) {
  (void)cout_pad;
  // tail after the panels (total is even): [max |w| bits][2^-s]
  unsigned* tail = reinterpret_cast<unsigned*>(reinterpret_cast<__half*>(panels) + total);
  cudaError_t e = cudaMemsetAsync(tail, 0, 8, s);
  if (e != cudaSuccess) return e;
  const long long nk = (long long)kh * kw * cin * cout;
  const unsigned ab = (unsigned)std::max(1LL, std::min<long long>((nk + 255) / 256, 148LL * 8));
  const long long blocks = std::max(1LL, std::min<long long>((total + 255) / 256, 148LL * 32));
#define SPLIT_CASE(TK)                                                                                   \
  kernel_amax<TK><<<ab, 256, 0, s>>>((const TK*)k, nk, tail);                                          \
  segregate_kmajor_split_kernel<TK><<<(unsigned)blocks, 256, 0, s>>>((const TK*)k, kw, cin, cout, cls,  \
                                                                     (__half*)panels, total, tail,      \
                                                                     reinterpret_cast<float*>(tail + 1));
  if (k_dtype == SEGCONV_F32) {
    SPLIT_CASE(float)
  } else if (k_dtype == SEGCONV_F64) {
    SPLIT_CASE(double)
  } else if (k_dtype == SEGCONV_BF16) {
    SPLIT_CASE(__nv_bfloat16)
  } else {
    return cudaErrorInvalidValue;
  }
#undef SPLIT_CASE
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_segregate(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                             int cout_pad, int layout, const SegClasses& cls, void* panels,
                             int p_dtype, long long total, cudaStream_t s) {
#define SEG_CASE(KT, KID)                                                                     \
  if (k_dtype == KID) {                                                                       \
    if (p_dtype == SEGCONV_F32)                                                               \
      return launch_seg<KT, float>(k, kh, kw, cin, cout, cout_pad, layout, cls, panels, total, s); \
    if (p_dtype == SEGCONV_F64)                                                               \
      return launch_seg<KT, double>(k, kh, kw, cin, cout, cout_pad, layout, cls, panels, total, s); \
    if (p_dtype == SEGCONV_BF16)                                                              \
      return launch_seg<KT, __nv_bfloat16>(k, kh, kw, cin, cout, cout_pad, layout, cls, panels, \
                                           total, s);                                         \
  }
  SEG_CASE(float, SEGCONV_F32)
  SEG_CASE(double, SEGCONV_F64)
  SEG_CASE(__nv_bfloat16, SEGCONV_BF16)
#undef SEG_CASE
  return cudaErrorInvalidValue;
}

// UMMA panel image for the tcgen05 kernel: blocks (n_tile, k_block, class,
// tap), each [plane][k-chunk j][row n][8 elems] = the SMEM K-major no-swizzle
// layout the MMA reads, so one cp.async.bulk stages one block.  SPLIT stores
// w as fp16 hi + lo planes (w = hi + lo to ~22 bits); otherwise one bf16 plane.
// One thread writes one 16-byte row chunk of every plane.
template <typename TK, bool SPLIT>
__global__ void segregate_umma_kernel(const TK* __restrict__ k, int kw, int cin, int cout,
                                      SegClasses cls, int NT, int KB, int nkb, int taps,
                                      uint16_t* __restrict__ out, long long rows_total,
                                      const SplitGuard* __restrict__ guard) {
  const int CH = KB / 8;
  constexpr int PLANES = SPLIT ? 2 : 1;
  const float wscale = SPLIT ? ldexpf(1.0f, split_scale_exp(guard->amax_bits)) : 1.0f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows_total;
       e += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(e % NT);
    long long t1 = e / NT;
    const int j = (int)(t1 % CH);
    const long long blk = t1 / CH;
    const int t = (int)(blk % taps);
    const long long t2 = blk / taps;
    const int kb = (int)(t2 % nkb);
    const int nt = (int)(t2 / nkb);
    int q = 0;
#pragma unroll
    for (int qq = 1; qq < 4; ++qq)
      if (t >= cls.sub_offset[qq]) q = qq;
    const int tl = t - (int)cls.sub_offset[q];
    const int u = tl / cls.kw[q], v = tl % cls.kw[q];
    const int f = nt * NT + n;
    uint16_t hi[8], lo[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int ci = kb * KB + j * 8 + x;
      float w = 0.0f;
      if (f < cout && ci < cin)
        w = wscale * (float)to_acc(k[(((long long)(cls.u0[q] + 2 * u) * kw + (cls.v0[q] + 2 * v)) * cin + ci) *
                                         cout + f]);
      if constexpr (SPLIT) {
        const __half h = __float2half_rn(w);
        hi[x] = __half_as_ushort(h);
        lo[x] = __half_as_ushort(__float2half_rn(w - __half2float(h)));
      } else {
        hi[x] = __bfloat16_as_ushort(__float2bfloat16_rn(w));
      }
    }
    const long long block_elems = (long long)PLANES * KB * NT;
    uint16_t* dst = out + blk * block_elems + (long long)j * NT * 8 + (long long)n * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) dst[x] = hi[x];
    if constexpr (SPLIT) {
#pragma unroll
      for (int x = 0; x < 8; ++x) dst[(long long)CH * NT * 8 + x] = lo[x];
    }
  }
}

cudaError_t launch_segregate_umma(const void* k, int k_dtype, int kw, int cin, int cout,
                                  const SegClasses& cls, int NT, int KB, int nkb, int n_tiles,
                                  int taps, bool split, void* panels, const void* guard, cudaStream_t s) {
  if (split && !guard) return cudaErrorInvalidValue;
  const long long rows_total = (long long)n_tiles * nkb * taps * (KB / 8) * NT;
  const int threads = 256;
  const unsigned blocks = (unsigned)std::min<long long>((rows_total + threads - 1) / threads, 148LL * 32);
#define SEGU(KT)                                                                               \
  do {                                                                                         \
    if (split)                                                                                 \
      segregate_umma_kernel<KT, true><<<blocks, threads, 0, s>>>(                              \
          (const KT*)k, kw, cin, cout, cls, NT, KB, nkb, taps, (uint16_t*)panels, rows_total, \
          (const SplitGuard*)guard);                                                           \
    else                                                                                       \
      segregate_umma_kernel<KT, false><<<blocks, threads, 0, s>>>(                             \
          (const KT*)k, kw, cin, cout, cls, NT, KB, nkb, taps, (uint16_t*)panels, rows_total, \
          nullptr);                                                                            \
  } while (0)
  if (k_dtype == SEGCONV_F32)
    SEGU(float);
  else if (k_dtype == SEGCONV_BF16)
    SEGU(__nv_bfloat16);
  else if (k_dtype == SEGCONV_F64)
    SEGU(double);
  else
    return cudaErrorInvalidValue;
#undef SEGU
  note_launch();
  return cudaGetLastError();
}

// Class-folded A-operand image (tc_fold.cu): for k-block kb, k-chunk j, row
// = shift * 4*CP + q*CP + f: W = sub_q[dy - off_r][dx - off_c][ci][f] when
// that is a tap of class q, else 0.  Trailing (128 - 4*CP) rows stay zero.
template <typename TK, bool SPLIT>
__global__ void segregate_fold_kernel(const TK* __restrict__ k, int kw, int cin, int cout,
                                      SegClasses cls, int CP, int KB, int uc, int rows_per_col,
                                      int nshift_rows, uint16_t* __restrict__ out,
                                      long long chunks_total, long long plane_elems,
                                      const SplitGuard* __restrict__ guard) {
  const int CH = KB / 8;
  const float wscale = SPLIT ? ldexpf(1.0f, split_scale_exp(guard->amax_bits)) : 1.0f;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < chunks_total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e % rows_per_col);
    const long long col = e / rows_per_col;  // kb * CH + j
    const int j = (int)(col % CH), kb = (int)(col / CH);
    uint16_t hi[8], lo[8];
    const int R = 4 * CP;
    const int s = row / R, q = (row % R) / CP, f = (row % R) % CP;
    const int dy = s / uc, dx = s % uc;
    const int u = dy - cls.off_r[q], v = dx - cls.off_c[q];
    const bool tap = row < nshift_rows && f < cout && u >= 0 && u < cls.kh[q] && v >= 0 &&
                     v < cls.kw[q];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int ci = kb * KB + j * 8 + x;
      float w = 0.0f;
      if (tap && ci < cin)
        w = wscale * (float)to_acc(
                         k[(((long long)(cls.u0[q] + 2 * u) * kw + (cls.v0[q] + 2 * v)) * cin + ci) * cout + f]);
      if constexpr (SPLIT) {
        const __half h = __float2half_rn(w);
        hi[x] = __half_as_ushort(h);
        lo[x] = __half_as_ushort(__float2half_rn(w - __half2float(h)));
      } else {
        hi[x] = __bfloat16_as_ushort(__float2bfloat16_rn(w));
      }
    }
    uint16_t* dst = out + e * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) dst[x] = hi[x];
    if constexpr (SPLIT) {
#pragma unroll
      for (int x = 0; x < 8; ++x) dst[plane_elems + x] = lo[x];
    }
  }
}

cudaError_t launch_segregate_fold(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                  int p, const SegClasses& cls, bool split, void* panels,
                                  const void* guard, cudaStream_t s) {
  if (split && !guard) return cudaErrorInvalidValue;
  int ur, uc;
  fold_window(kh, kw, p, &ur, &uc);
  const int CP = fold_cp(cout);
  const int KB = fold_kb(split ? SEGCONV_MATH_F16X3 : SEGCONV_MATH_BF16, cin);
  const int nkb = (cin + KB - 1) / KB;
  const int rows = fold_rows(kh, kw, p, cout);
  const long long chunks_total = (long long)nkb * (KB / 8) * rows;
  const long long plane_elems = chunks_total * 8;
  const unsigned blocks = (unsigned)std::min<long long>((chunks_total + 255) / 256, 148LL * 32);
#define SEGF(KT)                                                                               \
  do {                                                                                         \
    if (split)                                                                                 \
      segregate_fold_kernel<KT, true><<<blocks, 256, 0, s>>>((const KT*)k, kw, cin, cout, cls,  \
                                                             CP, KB, uc, rows, ur * uc * 4 * CP, \
                                                             (uint16_t*)panels, chunks_total,  \
                                                             plane_elems, (const SplitGuard*)guard); \
    else                                                                                       \
      segregate_fold_kernel<KT, false><<<blocks, 256, 0, s>>>((const KT*)k, kw, cin, cout, cls, \
                                                              CP, KB, uc, rows, ur * uc * 4 * CP, \
                                                              (uint16_t*)panels, chunks_total, \
                                                              plane_elems, nullptr);           \
  } while (0)
  if (k_dtype == SEGCONV_F32)
    SEGF(float);
  else if (k_dtype == SEGCONV_BF16)
    SEGF(__nv_bfloat16);
  else if (k_dtype == SEGCONV_F64)
    SEGF(double);
  else
    return cudaErrorInvalidValue;
#undef SEGF
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------- split guard
// Header of the split-fp16 panels (tc_guard.cuh): max |w|, W1 = max over
// (class, feature) of sum |w| over the class's taps and channels, 2^-s; then
// the kernel in fp32 (reference layout) for the CTA-local FFMA fallback.
template <typename TK>
__global__ void guard_w1_kernel(const TK* __restrict__ k, int kw, int cin, int cout, SegClasses cls,
                                unsigned* __restrict__ w1_bits) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * cout) return;
  const int q = t / cout, f = t % cout;
  float sum = 0.0f;
  for (int u = 0; u < cls.kh[q]; ++u)
    for (int v = 0; v < cls.kw[q]; ++v)
      for (int ch = 0; ch < cin; ++ch)
        sum += fabsf((float)to_acc(k[(((long long)(cls.u0[q] + 2 * u) * kw + (cls.v0[q] + 2 * v)) * cin + ch) *
                                         cout + f]));
  atomicMax(w1_bits, __float_as_uint(sum));  // non-negative floats order as uints
}

template <typename TK>
__global__ void guard_copy_kernel(const TK* __restrict__ k, long long n, SplitGuard* __restrict__ g) {
  if (blockIdx.x == 0 && threadIdx.x == 0) g->inv_scale = ldexpf(1.0f, -split_scale_exp(g->amax_bits));
  float* dst = reinterpret_cast<float*>(g + 1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    dst[e] = (float)to_acc(k[e]);
}

cudaError_t launch_split_guard(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                               const SegClasses& cls, void* guard, cudaStream_t s) {
  SplitGuard* g = static_cast<SplitGuard*>(guard);
  if (!g || ((uintptr_t)g & 15)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(g, 0, sizeof(SplitGuard), s);
  if (e != cudaSuccess) return e;
  const long long nk = (long long)kh * kw * cin * cout;
  const unsigned ab = (unsigned)std::max(1LL, std::min<long long>((nk + 255) / 256, 148LL * 8));
  const unsigned wb = (unsigned)((4 * cout + 127) / 128);
#define GUARD_CASE(TK)                                                                        \
  kernel_amax<TK><<<ab, 256, 0, s>>>((const TK*)k, nk, &g->amax_bits);                        \
  guard_w1_kernel<TK><<<wb, 128, 0, s>>>((const TK*)k, kw, cin, cout, cls, &g->w1_bits);      \
  guard_copy_kernel<TK><<<ab, 256, 0, s>>>((const TK*)k, nk, g);
  if (k_dtype == SEGCONV_F32) {
    GUARD_CASE(float)
  } else if (k_dtype == SEGCONV_F64) {
    GUARD_CASE(double)
  } else if (k_dtype == SEGCONV_BF16) {
    GUARD_CASE(__nv_bfloat16)
  } else {
    return cudaErrorInvalidValue;
  }
#undef GUARD_CASE
  note_launch(3);
  return cudaGetLastError();
}

}  // namespace segconv_b200

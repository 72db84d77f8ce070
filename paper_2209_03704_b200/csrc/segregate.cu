// segregate.cu -- K1: on-device sub-kernel extraction into the four parity panels.
//
// Replaces reference proj/include/segconv/segregation.hpp:61-89 (segregate):
// sub_rc[u][v][ch][f] = k[u0_r + 2u][v0_c + 2v][ch][f], taps kept in their
// relative (u-major, v) order, class index r*2 + c.  One pass over the panel
// elements (gather; each source tap is read exactly once), with dtype
// conversion and, for the tensor-core path, re-layout to K-major
// (cout_pad, u, v, cin) rows so a panel row is one MMA B-operand row.
#include "common.cuh"
#include "kernels.h"

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

}  // namespace segconv_b200

// tc_guard.cuh -- range guard of the split-fp16 (f16x3) tensor-core kernels.
//
// The f16x3 kernels compute fp32 layers as x = xh + xl, w = wh + wl in fp16
// (three MMAs per product).  fp16 has a 5-bit exponent, so the split alone is
// only valid for |x|, |w| < 65504 and loses relative precision for values in
// the fp16 subnormal range -- while the reference accepts every finite float
// (tensor.hpp:79-96) and the fp32 bar is |a - b| <= 1e-5 max(|a|, |b|, 1).
//
// * Weights are known at segregate time: the image kernels scale them by a
//   power of two so that max |w'| = 2^14 (exact), and the epilogues multiply
//   the sums by 2^-s (SplitGuard::inv_scale).
// * Activations are checked twice over.  An |x| past the fp16 range makes
//   every sum that uses it non-finite, which the epilogues detect on the
//   outputs they store.  For layers whose weights are so large that the fp16
//   subnormal floor of the split (2^-25 absolute per element) could reach the
//   bar (W1 = max over (class, feature) of sum |w| > 128), the converter
//   warps also track the smallest non-zero |x|.  A CTA that saw a non-finite
//   sum (or, with the small check on, 0 < |x| < 2^-3) recomputes every output
//   it owns on CUDA cores
//   from the fp32 kernel kept after the guard header, in the reference's own
//   accumulation order without FMA contraction (the EXACT math mode: those
//   outputs are bit-identical to the reference), after all its roles are done
//   (the same CTA wrote them, so a __syncthreads orders the rewrite).
//   Ordinary data never takes that path; pathological data is slow, never
//   wrong.
//
// Panel tail (16-byte aligned, after every image the kernels read):
//   SplitGuard header | fp32 kernel (kh, kw, cin, cout), reference layout.
#pragma once

#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace segconv_b200 {

struct SplitGuard {
  float inv_scale;     // 2^-s: the images hold w * 2^s
  unsigned amax_bits;  // max |w| (float bits)
  unsigned w1_bits;    // max over (class, feature) of sum |w| (float bits)
  unsigned pad;
};
static_assert(sizeof(SplitGuard) == 16, "guard header is one 16-byte chunk");

constexpr float kGuardXMax = 65504.0f;   // largest finite fp16
constexpr float kGuardXSmall = 0.125f;   // below: the split's absolute floor 2^-25 dominates
constexpr float kGuardW1Small = 128.0f;  // W1 * 2^-25 <= 4e-6 below this: no small-x check

__host__ __device__ inline size_t split_guard_bytes(int kh, int kw, int cin, int cout) {
  return sizeof(SplitGuard) + (size_t)kh * kw * cin * cout * sizeof(float);
}

__device__ __forceinline__ const float* guard_kernel(const SplitGuard* g) {
  return reinterpret_cast<const float*>(g + 1);
}

// What the CTA-local FFMA fallback needs (host-filled from FusedProblem).
struct FallbackArgs {
  const float* x;          // fp32 NHWC input
  const SplitGuard* guard;  // nullptr: not a split-fp16 call (no guard)
  void* y;
  const float* bias;
  unsigned epi;
  int y_dtype;
  int batch, n, cin, cout, kw, pf, out_h, out_w;
  int qkh[4], qkw[4], u0[4], v0[4], off_r[4], off_c[4], rows[4], cols[4];
};

inline FallbackArgs make_fallback_args(const FusedProblem& pr, const void* guard) {
  FallbackArgs a{};
  a.x = static_cast<const float*>(pr.x);
  a.guard = static_cast<const SplitGuard*>(guard);
  a.y = pr.y;
  a.bias = pr.bias;
  a.epi = pr.epi;
  a.y_dtype = pr.y_dtype;
  a.batch = pr.batch;
  a.n = pr.n;
  a.cin = pr.cin;
  a.cout = pr.cout;
  a.kw = pr.kw;
  a.pf = pr.pf;
  a.out_h = pr.out_h;
  a.out_w = pr.out_w;
  for (int q = 0; q < 4; ++q) {
    a.qkh[q] = pr.cls.kh[q];
    a.qkw[q] = pr.cls.kw[q];
    a.u0[q] = pr.cls.u0[q];
    a.v0[q] = pr.cls.v0[q];
    a.off_r[q] = pr.cls.off_r[q];
    a.off_c[q] = pr.cls.off_c[q];
    a.rows[q] = pr.cls.rows[q];
    a.cols[q] = pr.cls.cols[q];
  }
  return a;
}

// Overflow: an |x| >= 65520 converts to an fp16 inf hi half, and every MMA
// sum that includes it becomes +-inf or NaN (inf * w, inf * 0 = NaN,
// inf - inf = NaN).  So the epilogues check the accumulators of the outputs
// they store (one predicated FFMA each: chk = v * 0 + chk stays 0 for finite
// v and turns NaN otherwise) -- no work on the converters' critical path.
// The small-value check (only for layers with huge weights, a warp-uniform
// flag) looks at the fp32 values on the converter warps.
// (A kernel whose epilogue is on its critical path -- tc_fold_ts.cu -- checks
// the converted hi halves instead: max |hi| by HMNMX2, two elements per op.)
struct GuardTrack {
  float mn = 3.0e38f;  // smallest non-zero |x| (small check only)
  bool small = false;  // the layer's W1 asks for the small check
  __half2 hm;          // max |hi| (add_hi users)
  __device__ __forceinline__ void init(const SplitGuard* g) {
    hm = __float2half2_rn(0.0f);
    small = g != nullptr && __uint_as_float(__ldg(&g->w1_bits)) > kGuardW1Small;
  }
  __device__ __forceinline__ void add_hi(const uint32_t (&hi)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) hm = __hmax2(hm, __habs2(*reinterpret_cast<const __half2*>(&hi[k])));
  }
  __device__ __forceinline__ void add(const float4& v) {  // fp32 values: the small check
    if (small) {
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) mn = fminf(mn, e[i] != 0.0f ? fabsf(e[i]) : 3.0e38f);
    }
  }
  __device__ __forceinline__ bool bad() const {
    const float2 m = __half22float2(hm);
    // an fp16 inf (or NaN) hi half: |x| past the fp16 range
    return !(fmaxf(m.x, m.y) < 65520.0f) || (small && mn < kGuardXSmall);
  }
};

// Epilogue side: accumulate one stored output's raw sum (before bias and
// activation -- tanh(inf) and ReLU(NaN) are finite).
__device__ __forceinline__ void guard_check(float& chk, float v) { chk = fmaf(v, 0.0f, chk); }
__device__ __forceinline__ bool guard_check_bad(float chk) { return !(chk == 0.0f); }

__device__ __forceinline__ float guard_inv_scale(const SplitGuard* g) {
  return g != nullptr ? __ldg(&g->inv_scale) : 1.0f;
}

// Recompute the outputs of `count` anchors on CUDA cores (reference order u,
// v, ch within each class, separate fp32 multiply and add -- bit-identical to
// reference accumulate_window, reference_ops.hpp:31-79), features [f0, f1),
// all four classes.
// anchor(idx, b, i, j) maps the CTA's idx-th anchor to image b, anchor row i,
// column j (false: none).  Called by every thread of the CTA.
template <class Anchor>
__device__ void guard_fallback(const FallbackArgs& a, long long count, int f0, int f1, Anchor anchor) {
  const float* __restrict__ k = guard_kernel(a.guard);
  const int nf = f1 - f0;
  if (nf <= 0) return;
  const long long items = count * 4 * nf;
  for (long long t = threadIdx.x; t < items; t += blockDim.x) {
    const int f = f0 + (int)(t % nf);
    const long long r = t / nf;
    const int q = (int)(r & 3);
    int b, i, j;
    if (!anchor(r >> 2, b, i, j)) continue;
    if (b < 0 || b >= a.batch || i < 0 || j < 0 || i >= a.rows[q] || j >= a.cols[q]) continue;
    float acc = 0.0f;
    for (int u = 0; u < a.qkh[q]; ++u) {
      const int xr = i + a.off_r[q] + u - a.pf;
      if (xr < 0 || xr >= a.n) continue;
      for (int v = 0; v < a.qkw[q]; ++v) {
        const int xc = j + a.off_c[q] + v - a.pf;
        if (xc < 0 || xc >= a.n) continue;
        const float* xp = a.x + (((long long)b * a.n + xr) * a.n + xc) * a.cin;
        const float* kp = k + ((long long)(a.u0[q] + 2 * u) * a.kw + (a.v0[q] + 2 * v)) * a.cin * a.cout + f;
        for (int ch = 0; ch < a.cin; ++ch)  // reference order, no FMA contraction (EXACT math)
          acc = __fadd_rn(acc, __fmul_rn(__ldg(xp + ch), __ldg(kp + (long long)ch * a.cout)));
      }
    }
    const float out = epilogue_apply(acc, a.epi, a.bias, f);
    const long long pix = ((long long)b * a.out_h + 2 * i + (q >> 1)) * a.out_w + 2 * j + (q & 1);
    store_out(a.y, pix * a.cout + f, out, a.y_dtype);
  }
}

// Segregate side: the header (max |w|, 2^-s, W1) and the fp32 kernel copy,
// written before the image kernels that read the scale.
cudaError_t launch_split_guard(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                               const SegClasses& cls, void* guard, cudaStream_t s);

// Power of two that puts max |w| at 2^14 (the pair kernel's split uses the same).
__device__ __forceinline__ int split_scale_exp(unsigned amax_bits) {
  const float amax = __uint_as_float(amax_bits);
  if (!(amax > 0.0f) || !(amax < 3.0e38f)) return 0;
  int e;
  frexpf(amax, &e);  // amax in [2^(e-1), 2^e)
  const int s = 14 - e;
  return s < -100 ? -100 : (s > 100 ? 100 : s);
}

}  // namespace segconv_b200

// kernels.h -- internal launch interface between the C ABI (capi.cu) and the
// kernel translation units.  Not part of the public boundary.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace segconv_b200 {

// Per-class parity description, passed to kernels by value (class q = r*2 + c).
struct SegClasses {
  int kh[4], kw[4];        // active taps per axis (reference segregation.hpp:27-30)
  int u0[4], v0[4];        // first active tap     (segregation.hpp:24)
  int off_r[4], off_c[4];  // class input offset   (segregation.hpp:33-36)
  int rows[4], cols[4];    // output block rows/cols of the class (fused_tconv.hpp:51-52)
  long long sub_offset[4]; // element offset of the class panel
};

// Problem description for the fused (segregated) kernels.
struct FusedProblem {
  const void* x;
  int x_dtype;
  int batch, n, cin, cout, cout_pad;
  int kh, kw, p, pf;  // source kernel dims, p_orig, p_fused
  int out_h, out_w;
  SegClasses cls;
  const void* panels;
  int panel_dtype, panel_layout;
  const float* bias;
  unsigned epi;
  void* y;
  int y_dtype;
  // split-fp16 panels: the range-guard header (tc_guard.cuh) -- weight scale,
  // fp32 kernel for the CTA-local FFMA fallback; nullptr otherwise
  const void* guard;
};

// Backward pass of the fused layer (reference netdemo/layers.hpp:171-211).
// x, gy, k share `dtype`; gx has dtype; gk is F32 (F64 for F64 data).
struct BackwardProblem {
  const void* x;
  const void* gy;
  const void* k;  // original (kh, kw, cin, cout) kernel
  int dtype;
  int batch, n, cin, cout, kh, kw, p, pf, out_h, out_w;
  // gy position of input pixel (i, j) under tap (U, V): (stride*i + p - U, stride*j + p - V).
  // Transpose conv: stride 2, in_h = in_w = n.  conv2d_valid (conv = 1): stride 1,
  // p = 0, input in_h x in_w, gy (in_h - kh + 1) x (in_w - kw + 1).
  int stride, in_h, in_w, conv;
  void* gx;
  void* gk;
  int accumulate;  // gk += (the reference accumulates tap gradients across calls)
  // device flag: when set, the SIMT input-gradient kernels run only if *run_if
  // != 0 (the split-fp16 tensor-core path's range guard decides on device)
  const int* run_if;
};
// the narrow-output (cout <= 4, wide rows) SIMT backward kernels take this problem
bool bwd_narrow_applies(const BackwardProblem& pr);
cudaError_t launch_bwd_data_simt(const BackwardProblem& pr, bool exact, cudaStream_t s);
cudaError_t launch_bwd_weight_simt(const BackwardProblem& pr, bool exact, cudaStream_t s);
bool tc_bwd_data_supported(const BackwardProblem& pr);
// fp32 input gradient in split-fp16 math (f16x3) on the pair kernel (tc_wide.cu)
bool tc_bwd_data_split_supported(const BackwardProblem& pr);
// guarded: a device-side range check picks the tensor-core or the SIMT (FFMA)
// kernel (both launched, one exits at once) -- AUTO math for fp32 data
cudaError_t launch_tc_bwd_data_split(const BackwardProblem& pr, cudaStream_t s, bool guarded);
cudaError_t launch_tc_bwd_data(const BackwardProblem& pr, cudaStream_t s);
bool tc_bwd_weight_supported(const BackwardProblem& pr);
bool tc_conv_valid_supported(int batch, int h, int w, int cin, int kh, int kw, int cout);
cudaError_t launch_tc_conv_valid(const void* src, int batch, int h, int w, int cin, const void* kt, int kh,
                                 int kw, int cout, const float* bias, unsigned epi, void* y, cudaStream_t s);
cudaError_t launch_tc_bwd_weight(const BackwardProblem& pr, cudaStream_t s);
cudaError_t workspace_alloc(void** p, size_t bytes, cudaStream_t s);
cudaError_t launch_wgrad_reduce(const float* ws, float* gk, long long ksz, int splits, int accumulate,
                                cudaStream_t s);

cudaError_t launch_segregate_kmajor_split(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                          int cout_pad, const SegClasses& cls, void* panels, long long total,
                                          cudaStream_t s);
cudaError_t launch_segregate(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                             int cout_pad, int layout, const SegClasses& cls, void* panels,
                             int p_dtype, long long total, cudaStream_t s);

cudaError_t launch_segregate_umma(const void* k, int k_dtype, int kw, int cin, int cout,
                                  const SegClasses& cls, int NT, int KB, int nkb, int n_tiles,
                                  int taps, bool split, void* panels, const void* guard, cudaStream_t s);
int tc_n_tile(int math, int cout);
// class-folded tcgen05 kernel for narrow layers (tc_fold.cu)
cudaError_t launch_tc_fold(const FusedProblem& pr, int math, cudaStream_t s);
bool tc_fold_supported(const FusedProblem& pr, int math);
// CTA-pair (cta_group::2) implicit GEMM for wide bf16 layers (tc_wide.cu)
cudaError_t launch_tc_wide(const FusedProblem& pr, cudaStream_t s);
bool tc_wide_supported(const FusedProblem& pr, int math);
bool tc_wide_fits(int kh, int kw, int p, int cin, int cout);
int tc_wide_ntile(int cout);
// pixel-scatter kernel with a register row ring for n=5, cout=3 layers (tc_ring.cu)
bool tc_ring_supported(const FusedProblem& pr, int math);
cudaError_t launch_tc_ring(const FusedProblem& pr, const void* ring_img, cudaStream_t s);
cudaError_t launch_ring_image(const void* k, int k_dtype, int cin, const SegClasses& cls, void* out,
                              const void* guard, cudaStream_t s);
size_t ring_image_bytes(int cin);
// pixel-scatter kernel for 3x3 -> 3-channel bf16 layers on small images (tc_tile.cu)
bool tc_tile_supported(const FusedProblem& pr, int math);
cudaError_t launch_tc_tile(const FusedProblem& pr, const void* img, cudaStream_t s);
bool tile_applies(int kh, int kw, int p, int n, int cin, int cout);
cudaError_t launch_tile_image(const void* k, int k_dtype, int kh, int cin, const SegClasses& cls, void* out,
                              cudaStream_t s);
size_t tile_image_bytes(int kh, int cin);
// TMEM-weights variant for split-fp16 layers with cout in (16, 32] (tc_fold_ts.cu)
cudaError_t launch_tc_fold_ts(const FusedProblem& pr, const void* img, cudaStream_t s);
bool fold_ts_panels_apply(int kh, int kw, int cin, int cout, int p_orig, int panel_dtype);
size_t fold_ts_image_bytes_for(int kh, int kw, int cin, int p_orig);
cudaError_t launch_fold_ts_image(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                 int p_orig, const SegClasses& cls, void* out, const void* guard,
                                 cudaStream_t s);
bool tc_fold_ts_supported(const FusedProblem& pr, int math);
bool tc_fold_available(int math, int cin, int cout);
bool tc_fold_fits(int math, int kh, int kw, int p, int cin, int cout);
void fold_window(int kh, int kw, int p, int* ur, int* uc);
int fold_cp(int cout);
int fold_kb(int math, int cin);
int fold_rows(int kh, int kw, int p, int cout);
cudaError_t launch_segregate_fold(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                  int p, const SegClasses& cls, bool split, void* panels,
                                  const void* guard, cudaStream_t s);
int tc_k_block(int cin, int cout);

// SIMT kernels (direct.cu).  Return cudaErrorNotSupported when no
// instantiation covers the problem.
cudaError_t launch_direct_generic(const FusedProblem& pr, bool exact, cudaStream_t s);
cudaError_t launch_direct_tiled(const FusedProblem& pr, cudaStream_t s);

// Tensor-core implicit GEMM (tc_igemm.cu).
cudaError_t launch_tc_igemm(const FusedProblem& pr, int math, cudaStream_t s);
bool tc_igemm_supported(const FusedProblem& pr, int math);
bool tc_igemm_available(int math, int cin, int cout);
const unsigned long long* tc_trace_ptr();
size_t tc_trace_bytes();
size_t debug_wide_schedule(const long long* unit_base, const int* taps, int nkb, long long pairs, int halves,
                           uint16_t* out, size_t cap);
unsigned long long* tc_trace_buffer();

// Conventional path (conventional.cu).
cudaError_t launch_upsample_pad_backward(const void* g, int dtype, int batch, int n, int cin, int p, void* gx,
                                         cudaStream_t s);
cudaError_t launch_upsample_pad(const void* x, int dtype, int batch, int n, int cin, int p,
                                void* up, cudaStream_t s);
cudaError_t launch_conv2d_valid(const void* src, int dtype, int batch, int h, int w, int cin,
                                const void* k, int kh, int kw, int cout, const float* bias,
                                unsigned epi, bool exact, void* y, cudaStream_t s);

void note_launch(int n = 1);

}  // namespace segconv_b200

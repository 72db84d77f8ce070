/*
 * segconv_b200.h -- C ABI of the B200-native segregated transpose convolution.
 *
 * This is the drop-in boundary.  The reference (`segconv`, header-only C++20,
 * /root/reference/proj/include) has no FFI of its own; its operator API is the
 * C++ template set in namespace segconv.  Each entry point below replaces one
 * of those operators (cited as reference file:line) with a device-pointer,
 * stream-ordered call; include/segconv_b200.hpp rebuilds the reference's C++
 * signatures on top of it (value-semantics host tensors, same names, same
 * ShapeError / ContractError behaviour).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device buffers are owned by the caller;
 *    nothing is allocated on the hot path.  `stream` is a cudaStream_t passed
 *    as void* (NULL = legacy default stream).  Launches are asynchronous.
 *  - Layouts follow the reference: activations HWC per image with the channel
 *    innermost (reference tensor.hpp:57-62,122-124); a batch is B contiguous
 *    images (NHWC).  Kernels are (kh, kw, cin, cout), cout innermost
 *    (tensor.hpp:148-151,198-200).
 *  - All argument checks happen on the host before any launch and mirror the
 *    reference's exceptions: SEGCONV_E_SHAPE <-> segconv::ShapeError,
 *    SEGCONV_E_CONTRACT <-> segconv::ContractError (reference errors.hpp:14-23).
 *    segconv_last_error() returns a thread-local message for the last failure.
 *  - Entry points are stateless and reentrant (the plan object is the only
 *    state, and it is immutable after creation).  No CPU fallback exists: if the
 *    device code cannot run, calls return SEGCONV_E_CUDA.
 */
#ifndef SEGCONV_B200_H_
#define SEGCONV_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SEGCONV_OK = 0,
  SEGCONV_E_SHAPE = 1,       /* == segconv::ShapeError    (reference errors.hpp:16-18) */
  SEGCONV_E_CONTRACT = 2,    /* == segconv::ContractError (reference errors.hpp:21-23) */
  SEGCONV_E_CUDA = 3,        /* CUDA runtime / launch failure, no device, ...         */
  SEGCONV_E_UNSUPPORTED = 4, /* valid request this build has no kernel for            */
  SEGCONV_E_IO = 5,          /* == segconv::IoError       (reference errors.hpp:34-37) */
  SEGCONV_E_PARSE = 6,       /* == segconv::ParseError    (reference errors.hpp:25-31); */
                             /*    segconv_last_error_offset() = its byte_offset        */
  SEGCONV_E_NCCL = 7         /* NCCL missing or a collective failed (multi-GPU stack)   */
} segconv_status;

/* Element types.  The reference supports float and double (tensor.hpp:65,154);
 * bf16 is the BASELINE's tensor-core storage type (C3, C5). */
typedef enum {
  SEGCONV_F32 = 0,
  SEGCONV_F64 = 1,
  SEGCONV_BF16 = 2,
  SEGCONV_F16_SPLIT = 3  /* panels only: fp32 weights stored as hi + lo fp16 planes */
} segconv_dtype;

/* Arithmetic used by transpose_conv_fused. */
typedef enum {
  SEGCONV_MATH_AUTO = 0,   /* pick from shape and dtypes                     */
  SEGCONV_MATH_FFMA = 1,   /* SIMT, fp32 products + fp32 accumulate (fp64 for F64)           */
  SEGCONV_MATH_EXACT = 2,  /* SIMT, reference accumulation order, no FMA contraction:         */
                           /* bit-identical to the reference CPU path (slow; for parity)      */
  SEGCONV_MATH_BF16 = 3,   /* tcgen05 kind::f16: bf16 operands, fp32 accumulate in TMEM       */
  SEGCONV_MATH_TF32 = 4,   /* tcgen05 kind::tf32 on fp32 data (10-bit mantissa; bar 1e-2 as bf16)  */
  SEGCONV_MATH_F16X3 = 5   /* tcgen05 kind::f16 on split operands: x = xh + xl, w = wh + wl     */
                           /* (fp16 each), y = xh*wh + xl*wh + xh*wl accumulated in fp32 TMEM;  */
                           /* ~22-bit operands, fp32-class accuracy for |x|,|w| < 2^15          */
} segconv_math;

/* Epilogue flags, applied in this order: +bias[f], then ReLU or tanh. */
enum {
  SEGCONV_EPI_NONE = 0,
  SEGCONV_EPI_BIAS = 1,
  SEGCONV_EPI_RELU = 2,
  SEGCONV_EPI_TANH = 4
};

/* Panel layouts produced by segconv_segregate. */
typedef enum {
  SEGCONV_PANEL_REF = 0,    /* per class (u, v, cin, cout): the reference sub-kernel layout  */
                            /* (segregation.hpp:61-89); used by the SIMT kernels             */
  SEGCONV_PANEL_KMAJOR = 1, /* per class (cout, u, v, cin): K-major, rows padded to cout_pad */
  SEGCONV_PANEL_UMMA = 2,   /* tcgen05 B-operand image: blocks (n_tile, k_block, class, tap),  */
                            /* each [plane][k-chunk of 8][n_tile rows][8] -- the exact SMEM    */
                            /* K-major no-swizzle layout, so one bulk copy stages one block     */
  SEGCONV_PANEL_UMMA_FOLD = 3 /* class-folded tcgen05 A-operand image for cout <= 32:         */
                            /* [plane][k_block][k-chunk][shift * 4*cp + class*cp + f][8] over  */
                            /* the union window of shifts (zero where a class has no tap)      */
} segconv_panel_layout;

/* == segconv::TConvGeometry (reference geometry.hpp:18-27). */
typedef struct {
  int n_in, kh, kw, p_orig, p_fused, up_h, up_w, out_h, out_w;
  int trim_extra_row, trim_extra_col;
} segconv_geometry;

/* Device-side counterpart of segconv::SubKernelSet<T> (reference
 * segregation.hpp:43-55): describes the four parity panels, class q = r*2 + c,
 * that segconv_segregate writes into one caller-owned buffer. */
typedef struct {
  int source_kh, source_kw, p_orig, p_orig_parity;
  int cin, cout, cout_pad;
  int sub_kh[4], sub_kw[4];      /* active_tap_count per axis (segregation.hpp:27-30) */
  int off_r[4], off_c[4];        /* class_input_offset        (segregation.hpp:33-36) */
  int u0[4], v0[4];              /* first_active_tap          (segregation.hpp:24)    */
  int64_t sub_offset[4];         /* element offset of class q's panel                 */
  int64_t total_elems;           /* elements in the whole panel buffer                */
  int dtype;                     /* segconv_dtype of the panels                       */
  int layout;                    /* segconv_panel_layout                              */
  int n_tile;                    /* UMMA layout: output features per block            */
  int k_block;                   /* UMMA layout: input channels per block             */
  int math;                      /* segconv_math the panels were laid out for         */
} segconv_subkernels;

/* ---------------------------------------------------------------- geometry */
/* reference geometry.hpp:29-53 (tconv_geometry) */
segconv_status segconv_tconv_geometry(int n_in, int kh, int kw, int p_orig, segconv_geometry* out);
/* reference segregation.hpp:23-36 */
int segconv_first_active_tap(int p, int r);
int segconv_active_tap_count(int n, int p, int r);
int segconv_class_input_offset(int p, int r);

/* ------------------------------------------------------------- segregation */
/* Shape half of reference segregation.hpp:61-89 (segregate): fills `out` for a
 * (kh, kw, cin, cout) kernel at padding p_orig.  ContractError on kh/kw < 1,
 * p_orig < 0 (segregation.hpp:63-64), ShapeError on cin/cout < 1. */
segconv_status segconv_subkernels_init(int kh, int kw, int cin, int cout, int p_orig,
                                       segconv_dtype panel_dtype, segconv_panel_layout layout,
                                       segconv_subkernels* out);
/* Same, choosing dtype/layout for a math mode (AUTO resolves from x_dtype). */
segconv_status segconv_subkernels_for_math(int kh, int kw, int cin, int cout, int p_orig,
                                           segconv_dtype x_dtype, segconv_math math,
                                           segconv_subkernels* out);
/* Data half of segregate: one kernel pass gathers taps k[u0+2u][v0+2v][ch][f]
 * into the panels (with dtype conversion and re-layout).  d_kernel holds
 * kh*kw*cin*cout elements of kernel_dtype; d_panels holds sks->total_elems. */
segconv_status segconv_segregate(const void* d_kernel, segconv_dtype kernel_dtype,
                                 const segconv_subkernels* sks, void* d_panels, void* stream);

/* ------------------------------------------------------------ fused (hot) */
/* reference fused_tconv.hpp:69-82 (transpose_conv_fused(input, sks, geom)),
 * batched: d_x is (batch, n_in, n_in, cin) of x_dtype, d_y is
 * (batch, out_h, out_w, cout) of y_dtype.  Checks of fused_tconv.hpp:17-35
 * (check_fused_args) are applied.  d_bias (cout floats) is read only with
 * SEGCONV_EPI_BIAS. */
segconv_status segconv_transpose_conv_fused(const void* d_x, segconv_dtype x_dtype, int batch,
                                            int n_in, int cin, const segconv_subkernels* sks,
                                            const void* d_panels, const segconv_geometry* geom,
                                            const float* d_bias, unsigned epilogue,
                                            segconv_math math, void* d_y, segconv_dtype y_dtype,
                                            void* stream);

/* Host-buffer form of the same operator -- the reference's value-semantics
 * call (fused_tconv.hpp:69-82 takes and returns host tensors).  h_x is
 * (batch, n_in, n_in, cin) of x_dtype and h_y (batch, out_h, out_w, cout) of
 * y_dtype in host memory (page-locked for the copies to overlap); d_x / d_y are
 * caller-owned device staging buffers of the same sizes.  The batch is cut into
 * `chunks` slices (<= 0: library default); slice i's host->device copy, fused
 * kernel and device->host copy run on `stream` plus two library-owned copy
 * streams, so the transfers overlap the kernels and each other.  Asynchronous:
 * everything is ordered before later work on `stream`. */
segconv_status segconv_transpose_conv_fused_host(const void* h_x, void* d_x, segconv_dtype x_dtype,
                                                 int batch, int n_in, int cin,
                                                 const segconv_subkernels* sks,
                                                 const void* d_panels, const segconv_geometry* geom,
                                                 const float* d_bias, unsigned epilogue,
                                                 segconv_math math, void* d_y, void* h_y,
                                                 segconv_dtype y_dtype, int chunks, void* stream);

/* ---------------------------------------------------- SGC1 tensor files */
/* reference tensor_io.hpp:12-103: "SGC1" magic, u32 LE height, width,
 * channels, precision (0 f32 / 1 f64), then the HWC data little-endian.
 * Host-side; no device needed except for segconv_load_tensor_batch's upload. */
typedef struct {
  int height, width, channels;
  int precision; /* 0 = f32, 1 = f64 (reference Precision) */
} segconv_tensor_file_info;

/* reference tensor_io.hpp:53-74 (peek_tensor_file): IoError if the file cannot
 * be opened; ParseError at offset = bytes read for a short header, 0 for a bad
 * magic, 16 for an unknown precision tag, 4 for a non-positive dimension. */
segconv_status segconv_peek_tensor_file(const char* path, segconv_tensor_file_info* info);
/* reference tensor_io.hpp:76-91 (load_tensor<T>): dtype F32/F64 must match the
 * stored precision (ContractError); ParseError at min(size, expected) when the
 * payload size is wrong.  host_dst holds dst_bytes (>= h*w*c*elem). */
segconv_status segconv_load_tensor(const char* path, segconv_dtype dtype, void* host_dst,
                                   size_t dst_bytes);
/* reference tensor_io.hpp:93-103 (save_tensor<T>). */
segconv_status segconv_save_tensor(const char* path, const void* host_src, int height, int width,
                                   int channels, segconv_dtype dtype);
/* Batch loader: `count` files of one shape and precision into a (count, h, w,
 * c) NHWC batch.  Each image is read into its slot of host_staging (page-locked
 * for overlap, count*h*w*c elements) and its upload to d_dst is queued on
 * `stream` right away, so file reads overlap the host->device copies.  Errors
 * as segconv_load_tensor; a shape mismatch between files is a ContractError. */
segconv_status segconv_load_tensor_batch(const char* const* paths, int count, segconv_dtype dtype,
                                         void* host_staging, void* d_dst, void* stream);
/* Byte offset of the last SEGCONV_E_PARSE on this thread. */
size_t segconv_last_error_offset(void);

/* ------------------------------------------------------------- backward */
/* reference netdemo/layers.hpp:171-211 (net::FusedTConv<T>::backward), batched:
 * the gradients of the fused layer with respect to its input and its kernel.
 * d_x is the forward input (batch, n_in, n_in, cin), d_gy the output gradient
 * (batch, out_h, out_w, cout), d_kernel the ORIGINAL (kh, kw, cin, cout) kernel,
 * all of `dtype`.  Outputs (either may be NULL to skip it, not both):
 *   d_gx  (batch, n_in, n_in, cin) of `dtype`: the output gradient scattered
 *         back through the sub-kernels, cropped by p_fused (layers.hpp:178-210);
 *   d_gk  (kh, kw, cin, cout), F32 (F64 for F64 data): tap gradients at the
 *         original tap positions, summed over the batch.  accumulate != 0 adds
 *         to the existing contents, as the reference's grad_ accumulates over
 *         backward calls between zero_grads (netdemo/model.hpp:192-201).
 * math: EXACT (float/double: the reference's accumulation order, no FMA --
 * bit-identical to the reference), FFMA (SIMT tiles), BF16 (bf16 data: the
 * input gradient on the tcgen05 CTA-pair kernel, a stride-2 im2col walk over
 * gy, when cout % 64 == 0 and cin >= 64; the kernel gradient on SIMT tiles
 * with fp32 accumulation), F16X3 (fp32 data: the input gradient on the same
 * kernel in split-fp16 math -- gy and w power-of-two scaled and split into
 * fp16 hi/lo halves -- when cout == 32, cin >= 64, kh*kw <= 25; FFMA
 * otherwise and for the kernel gradient; a device-side range guard hands
 * inputs whose products reach ~10^3 to FFMA), AUTO (BF16 for bf16 data,
 * F16X3 for fp32, FFMA for double).
 * Errors: geometry ShapeError/ContractError as segconv_tconv_geometry; the
 * reference's "backward before forward" StateError has no counterpart (the
 * forward input is an argument). */
segconv_status segconv_transpose_conv_fused_backward(const void* d_x, const void* d_gy,
                                                     segconv_dtype dtype, int batch, int n_in,
                                                     int cin, const void* d_kernel, int kh, int kw,
                                                     int cout, int p_orig, segconv_math math,
                                                     void* d_gx, void* d_gk, int accumulate,
                                                     void* stream);

/* Which math AUTO resolves to for this problem (no launch). */
segconv_math segconv_select_math(segconv_dtype x_dtype, segconv_dtype panel_dtype, int cin,
                                 int cout, int kh, int kw);

/* ----------------------------------------------------- conventional path */
/* reference tensor.hpp:224-259 (pad(upsample2x(x), p)): writes the
 * (batch, up_h, up_w, cin) zero-inserted, padded map. */
segconv_status segconv_upsample2x_pad(const void* d_x, segconv_dtype dtype, int batch, int n_in,
                                      int cin, int p_orig, void* d_up, void* stream);
/* reference netdemo/layers.hpp:66-73 (Upsample2x::backward) composed with the
 * crop of the padding: d_gx (batch, n_in, n_in, cin) = d_gy (batch, up, up,
 * cin) at (2i + p_orig, 2j + p_orig), up = 2 n_in - 1 + 2 p_orig. */
segconv_status segconv_upsample2x_pad_backward(const void* d_gy, segconv_dtype dtype, int batch,
                                               int n_in, int cin, int p_orig, void* d_gx,
                                               void* stream);
/* reference reference_ops.hpp:86-108 (conv2d_valid), batched over `batch`
 * (h, w, cin) maps; output (batch, h-kh+1, w-kw+1, cout).  math: AUTO (bf16:
 * tensor cores; fp32 / fp64: FFMA), FFMA, or EXACT -- the reference's (u, v,
 * ch) accumulation order without FMA contraction, bit-identical to its CPU
 * conv2d_valid and hence (zeros added exactly) to transpose_conv_fused EXACT. */
segconv_status segconv_conv2d_valid(const void* d_src, segconv_dtype dtype, int batch, int h,
                                    int w, int cin, const void* d_kernel, int kh, int kw,
                                    int cout, const float* d_bias, unsigned epilogue,
                                    segconv_math math, void* d_y, void* stream);
/* reference netdemo/layers.hpp:98-122 (net::ConvValid<T>::backward), batched:
 * gradients of conv2d_valid.  d_src (batch, h, w, cin) is the forward input,
 * d_gy (batch, h-kh+1, w-kw+1, cout) the output gradient, d_kernel (kh, kw,
 * cin, cout); d_gx (batch, h, w, cin) of dtype, d_gk (kh, kw, cin, cout) F32 (F64
 * for F64 data) summed over the batch, `accumulate` as in
 * segconv_transpose_conv_fused_backward.  math: EXACT (bit-identical to the
 * reference layer), FFMA, BF16 (tcgen05 pair kernel, stride-1 walks), AUTO. */
segconv_status segconv_conv2d_valid_backward(const void* d_src, const void* d_gy, segconv_dtype dtype,
                                             int batch, int h, int w, int cin, const void* d_kernel,
                                             int kh, int kw, int cout, segconv_math math, void* d_gx,
                                             void* d_gk, int accumulate, void* stream);
/* Bytes of workspace segconv_transpose_conv_naive needs (the upsampled map). */
size_t segconv_naive_workspace_bytes(segconv_dtype dtype, int batch, int n_in, int cin,
                                     int p_orig);
/* reference reference_ops.hpp:116-133 (transpose_conv_naive): upsample, pad,
 * valid-correlate -- the conventional baseline, materialising the map. */
segconv_status segconv_transpose_conv_naive(const void* d_x, segconv_dtype dtype, int batch,
                                            int n_in, int cin, const void* d_kernel, int kh,
                                            int kw, int cout, int p_orig, void* d_workspace,
                                            size_t workspace_bytes, const float* d_bias,
                                            unsigned epilogue, segconv_math math, void* d_y,
                                            void* stream);

/* ------------------------------------------------- multi-GPU layer stack */
/* Batch-sharded driver for a chain of segregated layers (BASELINE C5: a GAN
 * generator).  The reference has no parallelism across images -- its only
 * threading is cout slices inside one image (fused_tconv.hpp:101-147) -- and
 * no layer chain; this is the "segconv_stack_run" of SURVEY.md 8(b)/(e).
 *
 * One process drives `n_gpus` devices (0..n_gpus-1; 0 = every visible one),
 * one stream each.  At creation the host weights go to GPU 0 and are
 * ncclBroadcast to the others once, then each GPU segregates its replica.
 * A forward call gives GPU g the contiguous image slice
 * [g B / G + min(g, B % G), ...) (balanced, remainder first), copies its shard
 * host->device in up to 4 slices on a copy stream while the chain runs on the
 * slices already landed (no data-path collective; ReLU / tanh / bias fused per
 * layer), ncclAllGather-s the output shards so every GPU holds the
 * full batch, and copies GPU 0's copy to h_y.  NCCL (libnccl.so.2) is loaded
 * on first use; without it a multi-GPU handle fails with SEGCONV_E_NCCL (a
 * single-GPU one needs no collective). */
typedef struct {
  int n_in, cin, cout, kh, kw, p_orig; /* input n_in x n_in x cin, kernel kh x kw, padding */
  const void* h_kernel;                /* host (kh, kw, cin, cout) of kernel_dtype            */
  segconv_dtype kernel_dtype;          /* F32 / F64 / BF16                                     */
  const float* h_bias;                 /* host cout floats, or NULL                            */
  unsigned epilogue;                   /* SEGCONV_EPI_* (BIAS needs h_bias)                   */
  segconv_math math;                   /* per-layer math (AUTO: from the activation dtype)     */
} segconv_layer;

typedef struct {
  int n_gpus;
  double h2d_ms;      /* max over GPUs: shard host->device copy (all slices)          */
  double compute_ms;  /* max over GPUs: first slice landed -> last layer done (device */
                      /* time; overlaps the upload of the later slices)               */
  double gather_ms;   /* max over GPUs: ncclAllGather of the output shards            */
  double d2h_ms;      /* GPU 0: full output device->host                              */
  double total_ms;    /* host wall time of the call                                   */
} segconv_timing;

typedef struct segconv_stack segconv_stack;

/* Validates the chain (each layer's tconv_geometry output and cout feed the
 * next layer: ShapeError otherwise), allocates activations for up to
 * max_batch images, broadcasts and segregates the weights.  dtype is the
 * activation dtype (F32 or BF16) of every layer. */
segconv_status segconv_stack_create(const segconv_layer* layers, int n_layers, segconv_dtype dtype,
                                    int max_batch, int n_gpus, segconv_stack** out);
/* h_x: (batch, n_in0, n_in0, cin0) host, h_y: (batch, out, out, cout_last)
 * host, both of dtype (page-locked memory lets the copies run at full speed).
 * Synchronous.  timing may be NULL. */
segconv_status segconv_stack_forward(segconv_stack* st, const void* h_x, int batch, void* h_y,
                                     segconv_timing* timing);
/* Device pointer of GPU g's full-batch (all-gathered) output of the last forward. */
const void* segconv_stack_output(const segconv_stack* st, int gpu);
int segconv_stack_gpus(const segconv_stack* st);
void segconv_stack_destroy(segconv_stack* st);
/* create + forward + destroy. */
segconv_status segconv_stack_run(const segconv_layer* layers, int n_layers, segconv_dtype dtype,
                                 const void* h_x, int batch, int n_gpus, void* h_y,
                                 segconv_timing* timing);

/* ------------------------------------------------------------ accounting */
/* reference analysis.hpp:31-41,48-67: out = {naive mults, naive adds, fused
 * mults, fused adds} for one image. */
segconv_status segconv_count_ops(int n_in, int cin, int cout, int kh, int kw, int p_orig,
                                 uint64_t out[4]);

/* ------------------------------------------------------------ diagnostics */
const char* segconv_last_error(void);
/* Kernel family the last segconv_transpose_conv_fused call on this thread ran
 * ("tc-fold-ts", "tc-pair", "tc-ring", "tc-tile", "tc-fold", "tc-halo",
 * "simt-tiled", "simt-generic", "simt-exact"). */
const char* segconv_last_path(void);
const char* segconv_version(void);
/* Number of kernels this library launched since load (all entry points). */
uint64_t segconv_launch_count(void);
/* Diagnostics: with SEGCONV_TC_TRACE=1 in the environment the tensor-core
 * kernels stamp per-role events (globaltimer ns) for their first 160 CTAs; copies
 * up to `bytes` of the 160 x 16 x 64 uint64 trace to host memory (with
 * SEGCONV_TC_TRACE=2: eight such slots, one per launch in turn).  Returns the
 * bytes copied (0 when tracing is off). */
size_t segconv_debug_trace(void* host_out, size_t bytes);
/* Diagnostics / host-logic tests: the pair kernel's balanced unit schedule for
 * units in class-major order (unit_base[5]: first unit of each class, [4] =
 * total), cost taps[q] x nkb per unit, over `pairs` CTA pairs.  Writes the
 * [pairs][slots] table (entry = unit | half << 14, half 1 / 2 = feature half,
 * 0xFFFF = end of a pair's list) and returns slots, or 0 when round-robin is
 * as good (or the table exceeds `cap` entries). */
size_t segconv_debug_wide_schedule(const long long* unit_base, const int* taps, int nkb, long long pairs,
                                   int halves, uint16_t* out, size_t cap);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* SEGCONV_B200_H_ */

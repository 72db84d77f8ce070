// capi.cu -- the extern "C" boundary (include/segconv_b200.h).
//
// Host-side validation mirrors the reference's exceptions before anything is
// launched; dispatch picks the kernel family for the requested math.  There
// is no CPU fallback: a missing device or a failed launch is SEGCONV_E_CUDA.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "segconv_b200.h"
#include "tc_guard.cuh"

namespace segconv_b200 {

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static thread_local std::string g_err;
static thread_local const char* g_path = "";  // kernel family of the last fused call

static segconv_status fail(segconv_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

segconv_status set_error(segconv_status st, const char* msg) {
  g_err = msg ? msg : "";
  return st;
}

static segconv_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SEGCONV_OK;
  if (e == cudaErrorNotSupported)
    return fail(SEGCONV_E_UNSUPPORTED, "%s: no kernel instantiation covers this problem", what);
  cudaGetLastError();  // clear sticky-free errors so the next call is clean
  return fail(SEGCONV_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static bool valid_dtype(int d) { return d == SEGCONV_F32 || d == SEGCONV_F64 || d == SEGCONV_BF16; }
static size_t dtype_size(int d) { return d == SEGCONV_F64 ? 8 : d == SEGCONV_BF16 ? 2 : 4; }

static bool ring_panels_apply(int kh, int kw, int cin, int cout, int p_orig, int panel_dtype) {
  return kh == 5 && kw == 5 && cout == 3 && p_orig == 0 && cin % 32 == 0 && cin <= 256 &&
         panel_dtype == SEGCONV_F16_SPLIT;
}
// the pixel-scatter tile kernel's weight image rides on the folded panels (p = 0)
static bool tile_panels_apply(int kh, int kw, int cin, int cout, int p_orig, int panel_dtype) {
  return (kh == 3 || kh == 4) && kw == kh && cout == 3 && p_orig == 0 && cin % 64 == 0 && cin <= 512 &&
         panel_dtype == SEGCONV_BF16;
}
// ... and on the K-major panels of the 4x4, even-p (out = 2N) 3-channel layers
static bool tile_kmajor_tail(int kh, int kw, int cin, int cout, int p_orig, int panel_dtype) {
  return kh == 4 && kw == 4 && cout == 3 && p_orig == 2 && cin % 64 == 0 &&
         cin <= 512 && panel_dtype == SEGCONV_BF16;
}
// elements of the K-major panels that precede an appended tile image
static int64_t kmajor_elems(const segconv_subkernels& s) {
  const int kcin = s.dtype == SEGCONV_F16_SPLIT ? 2 * s.cin : s.cin;
  int64_t e = 0;
  for (int q = 0; q < 4; ++q) e += (int64_t)s.sub_kh[q] * s.sub_kw[q] * kcin * s.cout_pad;
  return e;
}
// elements of the folded image that precede an appended ring image
static int64_t fold_image_elems(const segconv_subkernels& s) {
  const int nkb = (s.cin + s.k_block - 1) / s.k_block;
  const int planes = s.dtype == SEGCONV_F16_SPLIT ? 2 : 1;
  return (int64_t)planes * nkb * (s.k_block / 8) *
         fold_rows(s.source_kh, s.source_kw, s.p_orig, s.cout) * 8;
}

// Split-fp16 panels of the folded / scatter / halo kernels end in the range
// guard (tc_guard.cuh): header + fp32 kernel, 16-byte aligned.
static bool split_guarded(int layout, int dtype) {
  return dtype == SEGCONV_F16_SPLIT && (layout == SEGCONV_PANEL_UMMA_FOLD || layout == SEGCONV_PANEL_UMMA);
}
static int64_t guard_elems(const segconv_subkernels& s) {
  return split_guarded(s.layout, s.dtype)
             ? (int64_t)(split_guard_bytes(s.source_kh, s.source_kw, s.cin, s.cout) / 2)
             : 0;
}
// elements of every image the kernels read (the guard follows them)
static int64_t image_elems(const segconv_subkernels& s) { return s.total_elems - guard_elems(s); }
static const void* guard_of(const segconv_subkernels& s, const void* panels) {
  return split_guarded(s.layout, s.dtype) ? (const void*)((const uint16_t*)panels + image_elems(s)) : nullptr;
}

static SegClasses classes_of(const segconv_subkernels& s, const segconv_geometry& g) {
  SegClasses c{};
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, cc = q & 1;
    c.kh[q] = s.sub_kh[q];
    c.kw[q] = s.sub_kw[q];
    c.u0[q] = s.u0[q];
    c.v0[q] = s.v0[q];
    c.off_r[q] = s.off_r[q];
    c.off_c[q] = s.off_c[q];
    c.rows[q] = (g.out_h - r + 1) / 2;  // reference fused_tconv.hpp:51
    c.cols[q] = (g.out_w - cc + 1) / 2;  // reference fused_tconv.hpp:52
    c.sub_offset[q] = s.sub_offset[q];
  }
  return c;
}

}  // namespace segconv_b200

using namespace segconv_b200;

extern "C" {

const char* segconv_last_error(void) { return g_err.c_str(); }
const char* segconv_last_path(void) { return g_path; }
const char* segconv_version(void) { return "segconv_b200 0.1 (sm_100a)"; }
uint64_t segconv_launch_count(void) { return g_launches.load(); }

size_t segconv_debug_trace(void* host_out, size_t bytes) {
  const unsigned long long* t = tc_trace_ptr();
  if (!t || !host_out) return 0;
  const size_t n = std::min(bytes, tc_trace_bytes());
  if (cudaMemcpy(host_out, t, n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

size_t segconv_debug_wide_schedule(const long long* unit_base, const int* taps, int nkb, long long pairs,
                                   int halves, uint16_t* out, size_t cap) {
  if (!unit_base || !taps) return 0;
  return debug_wide_schedule(unit_base, taps, nkb, pairs, halves, out, cap);
}

// reference geometry.hpp:29-53
segconv_status segconv_tconv_geometry(int n_in, int kh, int kw, int p_orig, segconv_geometry* g) {
  if (!g) return fail(SEGCONV_E_CONTRACT, "geometry output pointer is null");
  if (n_in < 1) return fail(SEGCONV_E_SHAPE, "input size must be >= 1, got %d", n_in);
  if (kh < 1 || kw < 1) return fail(SEGCONV_E_SHAPE, "kernel dims must be >= 1, got %dx%d", kh, kw);
  if (p_orig < 0) return fail(SEGCONV_E_SHAPE, "padding must be >= 0, got %d", p_orig);
  segconv_geometry o;
  o.n_in = n_in;
  o.kh = kh;
  o.kw = kw;
  o.p_orig = p_orig;
  o.p_fused = p_orig / 2;
  o.up_h = o.up_w = 2 * n_in - 1 + 2 * p_orig;
  o.out_h = o.up_h - kh + 1;
  o.out_w = o.up_w - kw + 1;
  if (o.out_h < 1 || o.out_w < 1)
    return fail(SEGCONV_E_SHAPE, "kernel %dx%d does not fit the padded upsampled input (%dx%d)",
                kh, kw, o.up_h, o.up_w);
  o.trim_extra_row = o.out_h & 1;
  o.trim_extra_col = o.out_w & 1;
  *g = o;
  return SEGCONV_OK;
}

// reference segregation.hpp:23-36
int segconv_first_active_tap(int p, int r) { return (p + r) & 1; }
int segconv_active_tap_count(int n, int p, int r) {
  const int f = segconv_first_active_tap(p, r);
  return f >= n ? 0 : (n - f + 1) / 2;
}
int segconv_class_input_offset(int p, int r) {
  return (r + segconv_first_active_tap(p, r) - p) / 2 + p / 2;
}

// reference segregation.hpp:61-89 (shape half)
segconv_status segconv_subkernels_init(int kh, int kw, int cin, int cout, int p_orig,
                                       segconv_dtype panel_dtype, segconv_panel_layout layout,
                                       segconv_subkernels* out) {
  if (!out) return fail(SEGCONV_E_CONTRACT, "subkernel descriptor pointer is null");
  if (kh < 1 || kw < 1) return fail(SEGCONV_E_CONTRACT, "cannot segregate a spatially empty kernel");
  if (p_orig < 0) return fail(SEGCONV_E_CONTRACT, "padding must be non-negative");
  if (cin < 1 || cout < 1)
    return fail(SEGCONV_E_SHAPE, "bad kernel dims %dx%dx%dx%d", kh, kw, cin, cout);
  if (!valid_dtype(panel_dtype) && panel_dtype != SEGCONV_F16_SPLIT)
    return fail(SEGCONV_E_CONTRACT, "unknown panel dtype %d", (int)panel_dtype);
  if (layout != SEGCONV_PANEL_REF && layout != SEGCONV_PANEL_KMAJOR && layout != SEGCONV_PANEL_UMMA &&
      layout != SEGCONV_PANEL_UMMA_FOLD)
    return fail(SEGCONV_E_CONTRACT, "unknown panel layout %d", (int)layout);
  const bool umma = layout == SEGCONV_PANEL_UMMA || layout == SEGCONV_PANEL_UMMA_FOLD;
  if (umma && panel_dtype != SEGCONV_BF16 && panel_dtype != SEGCONV_F16_SPLIT)
    return fail(SEGCONV_E_CONTRACT, "UMMA panels are bf16 or split-fp16");
  if (!umma && panel_dtype == SEGCONV_F16_SPLIT && layout != SEGCONV_PANEL_KMAJOR)
    return fail(SEGCONV_E_CONTRACT, "split-fp16 panels need a UMMA or K-major layout");
  if (layout == SEGCONV_PANEL_UMMA_FOLD && cout > 32)
    return fail(SEGCONV_E_CONTRACT, "class-folded panels need cout <= 32");
  segconv_subkernels s{};
  s.source_kh = kh;
  s.source_kw = kw;
  s.p_orig = p_orig;
  s.p_orig_parity = p_orig & 1;
  s.cin = cin;
  s.cout = cout;
  s.dtype = panel_dtype;
  s.layout = layout;
  s.math = umma ? (panel_dtype == SEGCONV_F16_SPLIT ? SEGCONV_MATH_F16X3 : SEGCONV_MATH_BF16)
                : SEGCONV_MATH_FFMA;
  // K-major split panels: rows (f, u, v) of [hi(cin) | lo(cin)] fp16
  const int kcin = (layout == SEGCONV_PANEL_KMAJOR && panel_dtype == SEGCONV_F16_SPLIT) ? 2 * cin : cin;
  if (kcin != cin) s.math = SEGCONV_MATH_F16X3;
  // K-major panels pad the MMA N dimension to a multiple of 16 rows.
  s.cout_pad = layout == SEGCONV_PANEL_KMAJOR ? (cout + 15) / 16 * 16 : cout;
  int64_t off = 0;
  int taps = 0;
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, c = q & 1;
    s.u0[q] = segconv_first_active_tap(p_orig, r);
    s.v0[q] = segconv_first_active_tap(p_orig, c);
    s.sub_kh[q] = segconv_active_tap_count(kh, p_orig, r);
    s.sub_kw[q] = segconv_active_tap_count(kw, p_orig, c);
    s.off_r[q] = segconv_class_input_offset(p_orig, r);
    s.off_c[q] = segconv_class_input_offset(p_orig, c);
    s.sub_offset[q] = layout == SEGCONV_PANEL_UMMA ? taps : off;  // UMMA: first tap block
    off += (int64_t)s.sub_kh[q] * s.sub_kw[q] * kcin * s.cout_pad;
    taps += s.sub_kh[q] * s.sub_kw[q];
  }
  s.total_elems = off;
  if (kcin != cin) s.total_elems += 4;  // split panels: max |w| and the 2^-s scale (2 x 4 bytes)
  if (layout == SEGCONV_PANEL_KMAJOR && tile_kmajor_tail(kh, kw, cin, cout, p_orig, panel_dtype))
    s.total_elems += (int64_t)(tile_image_bytes(kh, cin) / 2);
  if (layout == SEGCONV_PANEL_UMMA_FOLD) {
    s.n_tile = fold_cp(cout);
    s.k_block = fold_kb(s.math, cin);
    const int nkb = (cin + s.k_block - 1) / s.k_block;
    const int planes = panel_dtype == SEGCONV_F16_SPLIT ? 2 : 1;
    s.cout_pad = s.n_tile;
    for (int q = 0; q < 4; ++q) s.sub_offset[q] = 0;
    s.total_elems = (int64_t)planes * nkb * (s.k_block / 8) * fold_rows(kh, kw, p_orig, cout) * 8;
    // split-fp16 5x5 -> 3-channel layers also carry the pixel-scatter image
    // (tc_ring.cu) after the folded one; the kernel is picked per call by image size
    if (ring_panels_apply(kh, kw, cin, cout, p_orig, panel_dtype))
      s.total_elems += (int64_t)(ring_image_bytes(cin) / 2);
    // bf16 3x3 -> 3-channel layers carry the small-image pixel-scatter image (tc_tile.cu)
    if (tile_panels_apply(kh, kw, cin, cout, p_orig, panel_dtype))
      s.total_elems += (int64_t)(tile_image_bytes(kh, cin) / 2);
    // split-fp16 layers with 4 classes x 32 features: compact weight image of
    // the TMEM-weight kernel (tc_fold_ts.cu), only the blocks that hold taps
    if (fold_ts_panels_apply(kh, kw, cin, cout, p_orig, panel_dtype))
      s.total_elems += (int64_t)(fold_ts_image_bytes_for(kh, kw, cin, p_orig) / 2);
  }
  if (layout == SEGCONV_PANEL_UMMA) {
    s.n_tile = tc_n_tile(s.math, cout);
    s.k_block = tc_k_block(cin, cout);
    const int n_tiles = (cout + s.n_tile - 1) / s.n_tile;
    const int nkb = (cin + s.k_block - 1) / s.k_block;
    const int planes = panel_dtype == SEGCONV_F16_SPLIT ? 2 : 1;
    s.cout_pad = n_tiles * s.n_tile;
    s.total_elems = (int64_t)n_tiles * nkb * taps * planes * s.k_block * s.n_tile;
  }
  if (split_guarded(s.layout, s.dtype))
    s.total_elems = (s.total_elems + 7) / 8 * 8 + (int64_t)(split_guard_bytes(kh, kw, cin, cout) / 2);
  *out = s;
  return SEGCONV_OK;
}

static bool tc_shape_ok(int kh, int kw, int p_orig) {
  // every parity class must own at least one tap (kh, kw >= 2 guarantees it)
  for (int r = 0; r < 2; ++r)
    if (segconv_active_tap_count(kh, p_orig, r) == 0 || segconv_active_tap_count(kw, p_orig, r) == 0)
      return false;
  return kh * kw <= 49;
}

segconv_status segconv_subkernels_for_math(int kh, int kw, int cin, int cout, int p_orig,
                                           segconv_dtype x_dtype, segconv_math math,
                                           segconv_subkernels* out) {
  if (!valid_dtype(x_dtype)) return fail(SEGCONV_E_CONTRACT, "unknown activation dtype");
  bool fold_blocked = false;
  if (math == SEGCONV_MATH_AUTO) {
    math = segconv_select_math(x_dtype, x_dtype, cin, cout, kh, kw);
    if ((math == SEGCONV_MATH_BF16 || math == SEGCONV_MATH_F16X3) && !tc_shape_ok(kh, kw, p_orig))
      math = SEGCONV_MATH_FFMA;
    // Tensor-core accumulation adds each MMA's K = 16 partial sum to the fp32
    // accumulator without round-to-nearest (measured: outputs drift toward zero
    // by ~4e-8 relative per step).  The folded / scatter kernels take at most a
    // few dozen steps; the pair kernel's split mode keeps the main product
    // (xh.wh: taps * cin / 16 steps) in its own accumulator, and past ~200 such
    // steps the drift exceeds the fp32 bar (1e-5): those layers run on FFMA
    // unless f16x3 is asked for explicitly.
    if (math == SEGCONV_MATH_F16X3) {
      // the folded kernels accumulate all three products over the union window
      int ur = 0, uc = 0;
      fold_window(kh, kw, p_orig, &ur, &uc);
      const bool fold_ok = tc_fold_fits(math, kh, kw, p_orig, cin, cout) && 3LL * ur * uc * cin / 16 <= 192;
      if (!fold_ok) {
        int taps_max = 0;
        for (int r = 0; r < 2; ++r)
          for (int c = 0; c < 2; ++c)
            taps_max = std::max(taps_max, segconv_active_tap_count(kh, p_orig, r) *
                                              segconv_active_tap_count(kw, p_orig, c));
        const bool ring = kh == 5 && kw == 5 && cout == 3 && p_orig == 0 && cin % 32 == 0 && cin <= 256;
        if (!ring && (!tc_wide_fits(kh, kw, p_orig, cin, cout) || (long long)taps_max * cin / 16 > 192))
          math = SEGCONV_MATH_FFMA;
        else if (!ring && tc_fold_fits(math, kh, kw, p_orig, cin, cout))
          fold_blocked = true;  // too long for one accumulator: the pair kernel's split mode
      }
    }
  }
  switch (math) {
    case SEGCONV_MATH_FFMA:
    case SEGCONV_MATH_EXACT: {
      const segconv_status st =
          segconv_subkernels_init(kh, kw, cin, cout, p_orig, x_dtype, SEGCONV_PANEL_REF, out);
      if (st == SEGCONV_OK) out->math = math;
      return st;
    }
    case SEGCONV_MATH_BF16:
    case SEGCONV_MATH_F16X3: {
      // narrow layers (cout <= 32, p_fused == 0): class-folded kernel
      const bool fold = !fold_blocked && tc_fold_fits(math, kh, kw, p_orig, cin, cout);
      // wide bf16 layers: CTA-pair kernel on K-major (class, f, u, v, ch) panels
      if (!fold && math == SEGCONV_MATH_BF16 && tc_wide_fits(kh, kw, p_orig, cin, cout)) {
        const segconv_status st = segconv_subkernels_init(kh, kw, cin, cout, p_orig, SEGCONV_BF16,
                                                          SEGCONV_PANEL_KMAJOR, out);
        if (st == SEGCONV_OK) out->math = SEGCONV_MATH_BF16;
        return st;
      }
      // wide fp32 layers: the same kernel on split planes, K = [hi | lo] x 3 passes
      if (!fold && math == SEGCONV_MATH_F16X3 && tc_wide_fits(kh, kw, p_orig, cin, cout)) {
        const segconv_status st = segconv_subkernels_init(kh, kw, cin, cout, p_orig, SEGCONV_F16_SPLIT,
                                                          SEGCONV_PANEL_KMAJOR, out);
        if (st == SEGCONV_OK) out->math = SEGCONV_MATH_F16X3;
        return st;
      }
      return segconv_subkernels_init(
          kh, kw, cin, cout, p_orig, math == SEGCONV_MATH_BF16 ? SEGCONV_BF16 : SEGCONV_F16_SPLIT,
          fold ? SEGCONV_PANEL_UMMA_FOLD : SEGCONV_PANEL_UMMA, out);
    }
    case SEGCONV_MATH_TF32: {
      // fp32 data on tf32 tensor cores (10-bit mantissa, the cuDNN default for fp32):
      // the CTA-pair kernel on fp32 K-major panels
      if (x_dtype != SEGCONV_F32 || !tc_wide_fits(kh, kw, p_orig, cin, cout))
        return fail(SEGCONV_E_UNSUPPORTED, "TF32 math needs fp32 data, cin %% 64 == 0 and taps in every class");
      const segconv_status st = segconv_subkernels_init(kh, kw, cin, cout, p_orig, SEGCONV_F32,
                                                        SEGCONV_PANEL_KMAJOR, out);
      if (st == SEGCONV_OK) out->math = SEGCONV_MATH_TF32;
      return st;
    }
    default:
      return fail(SEGCONV_E_UNSUPPORTED, "math mode %d has no kernels in this build", (int)math);
  }
}

segconv_status segconv_segregate(const void* d_kernel, segconv_dtype kernel_dtype,
                                 const segconv_subkernels* sks, void* d_panels, void* stream) {
  if (!sks || !d_kernel || !d_panels) return fail(SEGCONV_E_CONTRACT, "null argument to segregate");
  if (!valid_dtype(kernel_dtype)) return fail(SEGCONV_E_CONTRACT, "unknown kernel dtype");
  SegClasses cls{};
  for (int q = 0; q < 4; ++q) {
    cls.kh[q] = sks->sub_kh[q];
    cls.kw[q] = sks->sub_kw[q];
    cls.u0[q] = sks->u0[q];
    cls.v0[q] = sks->v0[q];
    cls.sub_offset[q] = sks->sub_offset[q];
  }
  if (sks->total_elems == 0) return SEGCONV_OK;
  // split-fp16 images read the weight scale from the guard header: write it first
  void* guard = const_cast<void*>(guard_of(*sks, d_panels));
  if (guard) {
    const segconv_status gst = cuda_status(
        launch_split_guard(d_kernel, kernel_dtype, sks->source_kh, sks->source_kw, sks->cin, sks->cout, cls,
                           guard, (cudaStream_t)stream),
        "segregate[guard]");
    if (gst != SEGCONV_OK) return gst;
  }
  if (sks->layout == SEGCONV_PANEL_UMMA_FOLD) {
    cls.off_r[0] = cls.off_r[1] = 0;
    for (int q = 0; q < 4; ++q) {
      cls.off_r[q] = sks->off_r[q];
      cls.off_c[q] = sks->off_c[q];
    }
    segconv_status st = cuda_status(
        launch_segregate_fold(d_kernel, kernel_dtype, sks->source_kh, sks->source_kw, sks->cin,
                              sks->cout, sks->p_orig, cls, sks->dtype == SEGCONV_F16_SPLIT,
                              d_panels, guard, (cudaStream_t)stream),
        "segregate[fold]");
    if (st == SEGCONV_OK && image_elems(*sks) > fold_image_elems(*sks)) {
      uint16_t* tail = (uint16_t*)d_panels + fold_image_elems(*sks);
      if (fold_ts_panels_apply(sks->source_kh, sks->source_kw, sks->cin, sks->cout, sks->p_orig,
                               sks->dtype))
        st = cuda_status(launch_fold_ts_image(d_kernel, kernel_dtype, sks->source_kh,
                                              sks->source_kw, sks->cin, sks->cout, sks->p_orig,
                                              cls, tail, guard, (cudaStream_t)stream),
                         "segregate[fold-ts]");
      else if (sks->dtype == SEGCONV_F16_SPLIT)
        st = cuda_status(launch_ring_image(d_kernel, kernel_dtype, sks->cin, cls, tail, guard,
                                           (cudaStream_t)stream),
                         "segregate[ring]");
      else
        st = cuda_status(launch_tile_image(d_kernel, kernel_dtype, sks->source_kh, sks->cin, cls, tail,
                                           (cudaStream_t)stream),
                         "segregate[tile]");
    }
    return st;
  }
  if (sks->layout == SEGCONV_PANEL_UMMA) {
    int taps = 0;
    for (int q = 0; q < 4; ++q) taps += sks->sub_kh[q] * sks->sub_kw[q];
    const int n_tiles = sks->cout_pad / sks->n_tile;
    const int nkb = (sks->cin + sks->k_block - 1) / sks->k_block;
    return cuda_status(launch_segregate_umma(d_kernel, kernel_dtype, sks->source_kw, sks->cin,
                                             sks->cout, cls, sks->n_tile, sks->k_block, nkb,
                                             n_tiles, taps, sks->dtype == SEGCONV_F16_SPLIT,
                                             d_panels, guard, (cudaStream_t)stream),
                       "segregate[umma]");
  }
  if (sks->layout == SEGCONV_PANEL_KMAJOR && sks->dtype == SEGCONV_F16_SPLIT)
    return cuda_status(launch_segregate_kmajor_split(d_kernel, kernel_dtype, sks->source_kh, sks->source_kw,
                                                     sks->cin, sks->cout, sks->cout_pad, cls, d_panels,
                                                     kmajor_elems(*sks), (cudaStream_t)stream),
                       "segregate[k-major split]");
  const int64_t main_elems = sks->layout == SEGCONV_PANEL_KMAJOR ? kmajor_elems(*sks) : sks->total_elems;
  segconv_status st = cuda_status(launch_segregate(d_kernel, kernel_dtype, sks->source_kh, sks->source_kw,
                                                   sks->cin, sks->cout, sks->cout_pad, sks->layout, cls,
                                                   d_panels, sks->dtype, main_elems, (cudaStream_t)stream),
                                  "segregate");
  if (st == SEGCONV_OK && sks->layout == SEGCONV_PANEL_KMAJOR && sks->total_elems > main_elems) {
    for (int q = 0; q < 4; ++q) {  // the tile image reads the class input offsets
      cls.off_r[q] = sks->off_r[q];
      cls.off_c[q] = sks->off_c[q];
    }
    st = cuda_status(launch_tile_image(d_kernel, kernel_dtype, sks->source_kh, sks->cin, cls,
                                       (uint16_t*)d_panels + main_elems, (cudaStream_t)stream),
                     "segregate[tile]");
  }
  return st;
}

segconv_math segconv_select_math(segconv_dtype x_dtype, segconv_dtype panel_dtype, int cin,
                                 int cout, int kh, int kw) {
  (void)kh;
  (void)kw;
  const bool taps_ok = kh >= 2 && kw >= 2 && kh * kw <= 49;
  if (x_dtype == SEGCONV_BF16 && (panel_dtype == SEGCONV_BF16) && taps_ok &&
      tc_igemm_available(SEGCONV_MATH_BF16, cin, cout))
    return SEGCONV_MATH_BF16;
  if (x_dtype == SEGCONV_F32 && (panel_dtype == SEGCONV_F32 || panel_dtype == SEGCONV_F16_SPLIT) &&
      taps_ok && tc_igemm_available(SEGCONV_MATH_F16X3, cin, cout))
    return SEGCONV_MATH_F16X3;
  return SEGCONV_MATH_FFMA;
}

// reference fused_tconv.hpp:17-35 (check_fused_args) + :69-82
segconv_status segconv_transpose_conv_fused(const void* d_x, segconv_dtype x_dtype, int batch,
                                            int n_in, int cin, const segconv_subkernels* sks,
                                            const void* d_panels, const segconv_geometry* geom,
                                            const float* d_bias, unsigned epilogue,
                                            segconv_math math, void* d_y, segconv_dtype y_dtype,
                                            void* stream) {
  if (!sks || !geom) return fail(SEGCONV_E_CONTRACT, "null descriptor");
  if (batch < 0) return fail(SEGCONV_E_CONTRACT, "batch must be >= 0, got %d", batch);
  if (n_in != geom->n_in)
    return fail(SEGCONV_E_CONTRACT, "input is %dx%d but geometry was built for %dx%d", n_in, n_in,
                geom->n_in, geom->n_in);
  if (cin != sks->cin)
    return fail(SEGCONV_E_CONTRACT, "channel mismatch: input has %d, sub-kernels expect %d", cin,
                sks->cin);
  if (sks->source_kh != geom->kh || sks->source_kw != geom->kw)
    return fail(SEGCONV_E_CONTRACT,
                "sub-kernel set was built from a %dx%d kernel, geometry expects %dx%d",
                sks->source_kh, sks->source_kw, geom->kh, geom->kw);
  if (sks->p_orig_parity != (geom->p_orig & 1))
    return fail(SEGCONV_E_CONTRACT,
                "sub-kernel set was segregated for padding parity %d, geometry has p_orig %d",
                sks->p_orig_parity, geom->p_orig);
  // The geometry must be one tconv_geometry would produce.
  segconv_geometry chk;
  if (segconv_tconv_geometry(geom->n_in, geom->kh, geom->kw, geom->p_orig, &chk) != SEGCONV_OK ||
      chk.out_h != geom->out_h || chk.out_w != geom->out_w || chk.p_fused != geom->p_fused)
    return fail(SEGCONV_E_CONTRACT, "inconsistent geometry descriptor");
  if (!valid_dtype(x_dtype) || !valid_dtype(y_dtype))
    return fail(SEGCONV_E_CONTRACT, "unknown activation dtype");
  if ((epilogue & SEGCONV_EPI_RELU) && (epilogue & SEGCONV_EPI_TANH))
    return fail(SEGCONV_E_CONTRACT, "ReLU and tanh epilogues are exclusive");
  if ((epilogue & SEGCONV_EPI_BIAS) && !d_bias)
    return fail(SEGCONV_E_CONTRACT, "bias epilogue requested without a bias pointer");
  if (batch == 0) return SEGCONV_OK;
  if (!d_x || !d_y || !d_panels) return fail(SEGCONV_E_CONTRACT, "null data pointer");

  FusedProblem pr{};
  pr.x = d_x;
  pr.x_dtype = x_dtype;
  pr.batch = batch;
  pr.n = n_in;
  pr.cin = cin;
  pr.cout = sks->cout;
  pr.cout_pad = sks->cout_pad;
  pr.kh = geom->kh;
  pr.kw = geom->kw;
  pr.p = geom->p_orig;
  pr.pf = geom->p_fused;
  pr.out_h = geom->out_h;
  pr.out_w = geom->out_w;
  pr.cls = classes_of(*sks, *geom);
  pr.panels = d_panels;
  pr.panel_dtype = sks->dtype;
  pr.panel_layout = sks->layout;
  pr.bias = d_bias;
  pr.epi = epilogue;
  pr.y = d_y;
  pr.y_dtype = y_dtype;
  pr.guard = guard_of(*sks, d_panels);
  cudaStream_t s = (cudaStream_t)stream;

  if (math == SEGCONV_MATH_AUTO) math = (segconv_math)sks->math;  // what the panels were built for
  switch (math) {
    case SEGCONV_MATH_EXACT:
      if (sks->layout != SEGCONV_PANEL_REF)
        return fail(SEGCONV_E_CONTRACT, "EXACT math needs reference-layout panels");
      g_path = "simt-exact";
      return cuda_status(launch_direct_generic(pr, true, s), "transpose_conv_fused[exact]");
    case SEGCONV_MATH_FFMA: {
      if (sks->layout != SEGCONV_PANEL_REF)
        return fail(SEGCONV_E_CONTRACT, "FFMA math needs reference-layout panels");
      if (x_dtype != SEGCONV_F64 && sks->dtype != SEGCONV_F64) {
        g_path = "simt-tiled";
        cudaError_t e = launch_direct_tiled(pr, s);
        if (e != cudaErrorNotSupported) return cuda_status(e, "transpose_conv_fused[ffma]");
      }
      g_path = "simt-generic";
      return cuda_status(launch_direct_generic(pr, false, s), "transpose_conv_fused[ffma]");
    }
    case SEGCONV_MATH_BF16:
    case SEGCONV_MATH_F16X3:
    case SEGCONV_MATH_TF32: {
      if (math == SEGCONV_MATH_TF32 && sks->layout != SEGCONV_PANEL_KMAJOR)
        return fail(SEGCONV_E_CONTRACT, "TF32 math needs the K-major fp32 panels segregate builds for it");
      if (sks->layout == SEGCONV_PANEL_KMAJOR &&
          (math == SEGCONV_MATH_BF16 || math == SEGCONV_MATH_F16X3 || math == SEGCONV_MATH_TF32)) {
        if ((int)math != sks->math)
          return fail(SEGCONV_E_CONTRACT, "panels were laid out for math %d, not %d", sks->math,
                      (int)math);
        if (sks->total_elems > kmajor_elems(*sks) && tc_tile_supported(pr, math)) {
          g_path = "tc-tile";  // 3-channel 4x4 / even-p layer: pixel scatter reads x once
          return cuda_status(launch_tc_tile(pr, (const uint16_t*)d_panels + kmajor_elems(*sks), s),
                             "transpose_conv_fused[tcgen05 tile]");
        }
        if (!tc_wide_supported(pr, math))
          return fail(SEGCONV_E_UNSUPPORTED,
                      "CTA-pair tensor-core path needs bf16 activations, cin %% 64 == 0 and at most 25 "
                      "taps per parity class");
        g_path = "tc-pair";
        return cuda_status(launch_tc_wide(pr, s), "transpose_conv_fused[tcgen05 pair]");
      }
      if (sks->layout != SEGCONV_PANEL_UMMA && sks->layout != SEGCONV_PANEL_UMMA_FOLD)
        return fail(SEGCONV_E_CONTRACT, "tensor-core math needs UMMA-layout panels");
      if ((int)math != sks->math)
        return fail(SEGCONV_E_CONTRACT, "panels were laid out for math %d, not %d", sks->math,
                    (int)math);
      if (sks->layout == SEGCONV_PANEL_UMMA_FOLD) {
        if (!tc_fold_supported(pr, math))
          return fail(SEGCONV_E_UNSUPPORTED,
                      "class-folded tensor-core path: needs p_fused == 0, cin a multiple of the "
                      "channel block and a halo that fits shared memory");
        if (image_elems(*sks) > fold_image_elems(*sks) && tc_tile_supported(pr, math) && (g_path = "tc-tile"))
          return cuda_status(launch_tc_tile(pr, (const uint16_t*)d_panels + fold_image_elems(*sks), s),
                             "transpose_conv_fused[tcgen05 tile]");
        if (image_elems(*sks) > fold_image_elems(*sks) && tc_ring_supported(pr, math) && (g_path = "tc-ring"))
          return cuda_status(launch_tc_ring(pr, (const uint16_t*)d_panels + fold_image_elems(*sks), s),
                             "transpose_conv_fused[tcgen05 ring]");
        if (image_elems(*sks) > fold_image_elems(*sks) &&
            fold_ts_panels_apply(sks->source_kh, sks->source_kw, sks->cin, sks->cout, sks->p_orig,
                                 sks->dtype) &&
            tc_fold_ts_supported(pr, math) && (g_path = "tc-fold-ts"))
          return cuda_status(
              launch_tc_fold_ts(pr, (const uint16_t*)d_panels + fold_image_elems(*sks), s),
              "transpose_conv_fused[tcgen05 fold-ts]");
        g_path = "tc-fold";
        return cuda_status(launch_tc_fold(pr, math, s), "transpose_conv_fused[tcgen05 fold]");
      }
      if (!tc_igemm_supported(pr, math))
        return fail(SEGCONV_E_UNSUPPORTED,
                    "tensor-core path needs %s activations, cin %% 8 == 0, taps in every parity "
                    "class and a halo that fits shared memory",
                    math == SEGCONV_MATH_BF16 ? "bf16" : "fp32");
      g_path = "tc-halo";
      return cuda_status(launch_tc_igemm(pr, math, s), "transpose_conv_fused[tcgen05]");
    }
    default:
      return fail(SEGCONV_E_CONTRACT, "unknown math mode %d", (int)math);
  }
}

// ------------------------------------------------------------ backward
// Shared dispatch of the two backward entry points: tensor-core pair kernel for
// bf16 where it applies, SIMT (EXACT / FFMA) otherwise.
static segconv_status run_backward(const BackwardProblem& pr, segconv_math math, cudaStream_t s,
                                   const char* what) {
  const bool exact = math == SEGCONV_MATH_EXACT;
  segconv_status st = SEGCONV_OK;
  const char* dpath = "";
  char msg[160];
  if (pr.gx) {
    if (math == SEGCONV_MATH_BF16 && tc_bwd_data_supported(pr)) {
      dpath = "tc-pair";
      snprintf(msg, sizeof msg, "%s[input, tcgen05 pair]", what);
      st = cuda_status(launch_tc_bwd_data(pr, s), msg);
    } else if (math == SEGCONV_MATH_F16X3 && tc_bwd_data_split_supported(pr)) {
      // fp32 in split-fp16 math: K = taps x 2 cout x 2 copies / 16 accumulation
      // steps (C2: 72), well inside the tensor-core accumulation bound (§5);
      // the range guard picks FFMA on the device for extreme dynamic ranges
      dpath = "tc-pair-split";
      snprintf(msg, sizeof msg, "%s[input, tcgen05 pair, split fp16]", what);
      st = cuda_status(launch_tc_bwd_data_split(pr, s, true), msg);
    } else {
      dpath = exact ? "simt-exact" : bwd_narrow_applies(pr) ? "simt-narrow" : "simt-ffma";
      snprintf(msg, sizeof msg, "%s[input]", what);
      st = cuda_status(launch_bwd_data_simt(pr, exact, s), msg);
    }
    if (st != SEGCONV_OK) return st;
  }
  const char* wpath = "-";
  if (pr.gk) {
    if (math == SEGCONV_MATH_BF16 && tc_bwd_weight_supported(pr)) {
      wpath = "tc-pair";
      snprintf(msg, sizeof msg, "%s[kernel, tcgen05 pair]", what);
      st = cuda_status(launch_tc_bwd_weight(pr, s), msg);
    } else {
      wpath = exact ? "simt-exact" : bwd_narrow_applies(pr) ? "simt-narrow" : "simt-ffma";
      snprintf(msg, sizeof msg, "%s[kernel]", what);
      st = cuda_status(launch_bwd_weight_simt(pr, exact, s), msg);
    }
    if (st != SEGCONV_OK) return st;
  }
  static thread_local char path[48];
  snprintf(path, sizeof path, "bwd:%s+%s", pr.gx ? dpath : "-", wpath);
  g_path = path;
  return SEGCONV_OK;
}


segconv_status segconv_transpose_conv_fused_backward(const void* d_x, const void* d_gy, segconv_dtype dtype,
                                                     int batch, int n_in, int cin, const void* d_kernel,
                                                     int kh, int kw, int cout, int p_orig, segconv_math math,
                                                     void* d_gx, void* d_gk, int accumulate, void* stream) {
  segconv_geometry g;
  segconv_status st = segconv_tconv_geometry(n_in, kh, kw, p_orig, &g);
  if (st != SEGCONV_OK) return st;
  if (batch < 0) return fail(SEGCONV_E_CONTRACT, "batch must be >= 0, got %d", batch);
  if (cin < 1 || cout < 1) return fail(SEGCONV_E_SHAPE, "channel counts must be >= 1, got %d, %d", cin, cout);
  if (!valid_dtype(dtype)) return fail(SEGCONV_E_CONTRACT, "unknown dtype %d", (int)dtype);
  if (!d_gx && !d_gk) return fail(SEGCONV_E_CONTRACT, "neither an input nor a kernel gradient was requested");
  if (batch > 0) {  // an empty batch may come with null activation pointers
    if (!d_gy) return fail(SEGCONV_E_CONTRACT, "null output gradient");
    if (d_gx && !d_kernel) return fail(SEGCONV_E_CONTRACT, "the input gradient needs the kernel");
    if (d_gk && !d_x) return fail(SEGCONV_E_CONTRACT, "the kernel gradient needs the forward input");
  }
  // AUTO: bf16 tensor cores for bf16 data; fp32: split-fp16 tensor cores for
  // the input gradient where the shape allows, behind a device-side range
  // guard, FFMA otherwise
  if (math == SEGCONV_MATH_AUTO)
    math = dtype == SEGCONV_BF16 ? SEGCONV_MATH_BF16 : dtype == SEGCONV_F32 ? SEGCONV_MATH_F16X3 : SEGCONV_MATH_FFMA;
  if (math == SEGCONV_MATH_EXACT && dtype == SEGCONV_BF16)
    return fail(SEGCONV_E_CONTRACT, "EXACT math is defined for float and double (the reference's types)");
  if (math == SEGCONV_MATH_BF16 && dtype != SEGCONV_BF16)
    return fail(SEGCONV_E_CONTRACT, "BF16 math needs bf16 tensors");
  if (math == SEGCONV_MATH_F16X3 && dtype != SEGCONV_F32)
    return fail(SEGCONV_E_CONTRACT, "F16X3 math needs fp32 tensors");
  if (math != SEGCONV_MATH_EXACT && math != SEGCONV_MATH_FFMA && math != SEGCONV_MATH_BF16 &&
      math != SEGCONV_MATH_F16X3)
    return fail(SEGCONV_E_UNSUPPORTED, "math mode %d has no backward kernels in this build", (int)math);

  BackwardProblem pr{};
  pr.x = d_x;
  pr.gy = d_gy;
  pr.k = d_kernel;
  pr.dtype = dtype;
  pr.batch = batch;
  pr.n = n_in;
  pr.cin = cin;
  pr.cout = cout;
  pr.kh = kh;
  pr.kw = kw;
  pr.p = p_orig;
  pr.pf = g.p_fused;
  pr.out_h = g.out_h;
  pr.out_w = g.out_w;
  pr.stride = 2;
  pr.in_h = pr.in_w = n_in;
  pr.conv = 0;
  pr.gx = d_gx;
  pr.gk = d_gk;
  pr.accumulate = accumulate ? 1 : 0;
  return run_backward(pr, math, (cudaStream_t)stream, "transpose_conv_fused_backward");
}

// Host-buffer pipeline over batch slices (see the header).  Copy streams and
// events are created once per thread and device.
namespace {
struct HostPipe {
  int dev = -1;
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t fork = nullptr, loaded = nullptr, computed = nullptr, drained = nullptr;
};
thread_local HostPipe g_pipe;
}  // namespace

segconv_status segconv_transpose_conv_fused_host(const void* h_x, void* d_x, segconv_dtype x_dtype,
                                                 int batch, int n_in, int cin,
                                                 const segconv_subkernels* sks,
                                                 const void* d_panels, const segconv_geometry* geom,
                                                 const float* d_bias, unsigned epilogue,
                                                 segconv_math math, void* d_y, void* h_y,
                                                 segconv_dtype y_dtype, int chunks, void* stream) {
  if (!sks || !geom) return fail(SEGCONV_E_CONTRACT, "null descriptor");
  if (batch < 0) return fail(SEGCONV_E_CONTRACT, "batch must be >= 0, got %d", batch);
  if (!valid_dtype(x_dtype) || !valid_dtype(y_dtype))
    return fail(SEGCONV_E_CONTRACT, "unknown activation dtype");
  if (batch == 0) return SEGCONV_OK;
  if (!h_x || !h_y || !d_x || !d_y) return fail(SEGCONV_E_CONTRACT, "null data pointer");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "transpose_conv_fused_host");
  HostPipe& hp = g_pipe;
  if (hp.dev != dev) {
    hp = HostPipe{};
    if ((e = cudaStreamCreateWithFlags(&hp.in, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&hp.out, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&hp.fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&hp.loaded, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&hp.computed, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&hp.drained, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_status(e, "transpose_conv_fused_host: stream setup");
    hp.dev = dev;
  }
  const size_t xs = (size_t)n_in * n_in * cin * dtype_size(x_dtype);
  const size_t ys = (size_t)geom->out_h * geom->out_w * sks->cout * dtype_size(y_dtype);
  if (chunks <= 0) chunks = 16;  // measured on C2: 1 -> 0.99 ms, 4 -> 0.75, 16 -> 0.73 (copies alone 0.62)
  chunks = std::max(1, std::min(chunks, batch));
  cudaStream_t s = (cudaStream_t)stream;
  // the copy streams start after everything already queued on `stream`
  if ((e = cudaEventRecord(hp.fork, s)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(hp.in, hp.fork, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(hp.out, hp.fork, 0)) != cudaSuccess)
    return cuda_status(e, "transpose_conv_fused_host: fork");
  for (int c = 0; c < chunks; ++c) {
    const int b0 = (int)((long long)batch * c / chunks), b1 = (int)((long long)batch * (c + 1) / chunks);
    if (b1 == b0) continue;
    const size_t xo = (size_t)b0 * xs, yo = (size_t)b0 * ys;
    if ((e = cudaMemcpyAsync((char*)d_x + xo, (const char*)h_x + xo, (size_t)(b1 - b0) * xs,
                             cudaMemcpyHostToDevice, hp.in)) != cudaSuccess ||
        (e = cudaEventRecord(hp.loaded, hp.in)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s, hp.loaded, 0)) != cudaSuccess)
      return cuda_status(e, "transpose_conv_fused_host: upload");
    const segconv_status st = segconv_transpose_conv_fused(
        (const char*)d_x + xo, x_dtype, b1 - b0, n_in, cin, sks, d_panels, geom, d_bias, epilogue,
        math, (char*)d_y + yo, y_dtype, stream);
    if (st != SEGCONV_OK) return st;
    if ((e = cudaEventRecord(hp.computed, s)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(hp.out, hp.computed, 0)) != cudaSuccess ||
        (e = cudaMemcpyAsync((char*)h_y + yo, (const char*)d_y + yo, (size_t)(b1 - b0) * ys,
                             cudaMemcpyDeviceToHost, hp.out)) != cudaSuccess)
      return cuda_status(e, "transpose_conv_fused_host: download");
  }
  if ((e = cudaEventRecord(hp.drained, hp.out)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(s, hp.drained, 0)) != cudaSuccess)
    return cuda_status(e, "transpose_conv_fused_host: join");
  return SEGCONV_OK;
}

size_t segconv_naive_workspace_bytes(segconv_dtype dtype, int batch, int n_in, int cin, int p_orig) {
  if (batch < 0 || n_in < 1 || cin < 1 || p_orig < 0 || !valid_dtype(dtype)) return 0;
  const size_t up = 2 * (size_t)n_in - 1 + 2 * (size_t)p_orig;
  return (size_t)batch * up * up * cin * dtype_size(dtype);
}

segconv_status segconv_upsample2x_pad(const void* d_x, segconv_dtype dtype, int batch, int n_in,
                                      int cin, int p_orig, void* d_up, void* stream) {
  if (batch < 0 || n_in < 1 || cin < 1) return fail(SEGCONV_E_SHAPE, "tensor dims must be positive");
  if (p_orig < 0) return fail(SEGCONV_E_CONTRACT, "pad factor must be non-negative");
  if (!valid_dtype(dtype)) return fail(SEGCONV_E_CONTRACT, "unknown dtype");
  if (batch == 0) return SEGCONV_OK;
  return cuda_status(launch_upsample_pad(d_x, dtype, batch, n_in, cin, p_orig, d_up,
                                         (cudaStream_t)stream),
                     "upsample2x_pad");
}

// reference netdemo/layers.hpp:66-73 (Upsample2x::backward) after the pad crop
segconv_status segconv_upsample2x_pad_backward(const void* d_gy, segconv_dtype dtype, int batch, int n_in,
                                               int cin, int p_orig, void* d_gx, void* stream) {
  if (batch < 0 || n_in < 1 || cin < 1) return fail(SEGCONV_E_SHAPE, "tensor dims must be positive");
  if (p_orig < 0) return fail(SEGCONV_E_CONTRACT, "pad factor must be non-negative");
  if (!valid_dtype(dtype)) return fail(SEGCONV_E_CONTRACT, "unknown dtype");
  if (batch == 0) return SEGCONV_OK;
  if (!d_gy || !d_gx) return fail(SEGCONV_E_CONTRACT, "null data pointer");
  g_path = "simt-gather";
  return cuda_status(launch_upsample_pad_backward(d_gy, dtype, batch, n_in, cin, p_orig, d_gx,
                                                  (cudaStream_t)stream),
                     "upsample2x_pad_backward");
}

// reference reference_ops.hpp:86-102
segconv_status segconv_conv2d_valid(const void* d_src, segconv_dtype dtype, int batch, int h, int w,
                                    int cin, const void* d_kernel, int kh, int kw, int cout,
                                    const float* d_bias, unsigned epilogue, segconv_math math,
                                    void* d_y, void* stream) {
  if (kh < 1 || kw < 1) return fail(SEGCONV_E_SHAPE, "conv2d_valid needs a non-empty kernel");
  if (h < 1 || w < 1 || cin < 1 || cout < 1 || batch < 0)
    return fail(SEGCONV_E_SHAPE, "tensor dims must be positive");
  if (h - kh + 1 < 1 || w - kw + 1 < 1)
    return fail(SEGCONV_E_SHAPE, "kernel %dx%d does not fit input %dx%d", kh, kw, h, w);
  if (!valid_dtype(dtype)) return fail(SEGCONV_E_CONTRACT, "unknown dtype");
  if ((epilogue & SEGCONV_EPI_BIAS) && !d_bias)
    return fail(SEGCONV_E_CONTRACT, "bias epilogue requested without a bias pointer");
  if (math != SEGCONV_MATH_AUTO && math != SEGCONV_MATH_FFMA && math != SEGCONV_MATH_EXACT &&
      !(math == SEGCONV_MATH_BF16 && dtype == SEGCONV_BF16))
    return fail(SEGCONV_E_UNSUPPORTED, "conv2d_valid runs AUTO, FFMA, EXACT (float/double) or BF16 (bf16) math");
  if (math == SEGCONV_MATH_EXACT && dtype == SEGCONV_BF16)
    return fail(SEGCONV_E_CONTRACT, "EXACT math is defined for float and double (the reference's types)");
  if (batch == 0) return SEGCONV_OK;
  if (math == SEGCONV_MATH_EXACT)
    g_path = "simt-exact";
  else if (dtype == SEGCONV_BF16 && tc_conv_valid_supported(batch, h, w, cin, kh, kw, cout))
    g_path = "tc-pair";
  else if (dtype == SEGCONV_F32 && kh == kw && cout > 4 && kh >= 3 && kh <= 5)
    g_path = "simt-tiled";
  else
    g_path = "simt-generic";
  return cuda_status(launch_conv2d_valid(d_src, dtype, batch, h, w, cin, d_kernel, kh, kw, cout,
                                         d_bias, epilogue, math == SEGCONV_MATH_EXACT, d_y,
                                         (cudaStream_t)stream),
                     "conv2d_valid");
}

// reference netdemo/layers.hpp:98-122 (net::ConvValid<T>::backward), batched
segconv_status segconv_conv2d_valid_backward(const void* d_src, const void* d_gy, segconv_dtype dtype, int batch,
                                             int h, int w, int cin, const void* d_kernel, int kh, int kw,
                                             int cout, segconv_math math, void* d_gx, void* d_gk, int accumulate,
                                             void* stream) {
  if (kh < 1 || kw < 1) return fail(SEGCONV_E_SHAPE, "conv2d_valid needs a non-empty kernel");
  if (h < 1 || w < 1 || cin < 1 || cout < 1) return fail(SEGCONV_E_SHAPE, "tensor dims must be positive");
  if (h - kh + 1 < 1 || w - kw + 1 < 1)
    return fail(SEGCONV_E_SHAPE, "kernel %dx%d does not fit input %dx%d", kh, kw, h, w);
  if (batch < 0) return fail(SEGCONV_E_CONTRACT, "batch must be >= 0, got %d", batch);
  if (!valid_dtype(dtype)) return fail(SEGCONV_E_CONTRACT, "unknown dtype %d", (int)dtype);
  if (!d_gx && !d_gk) return fail(SEGCONV_E_CONTRACT, "neither an input nor a kernel gradient was requested");
  if (batch > 0) {
    if (!d_gy) return fail(SEGCONV_E_CONTRACT, "null output gradient");
    if (d_gx && !d_kernel) return fail(SEGCONV_E_CONTRACT, "the input gradient needs the kernel");
    if (d_gk && !d_src) return fail(SEGCONV_E_CONTRACT, "the kernel gradient needs the forward input");
  }
  if (math == SEGCONV_MATH_AUTO) math = dtype == SEGCONV_BF16 ? SEGCONV_MATH_BF16 : SEGCONV_MATH_FFMA;
  if (math == SEGCONV_MATH_EXACT && dtype == SEGCONV_BF16)
    return fail(SEGCONV_E_CONTRACT, "EXACT math is defined for float and double (the reference's types)");
  if (math == SEGCONV_MATH_BF16 && dtype != SEGCONV_BF16)
    return fail(SEGCONV_E_CONTRACT, "BF16 math needs bf16 tensors");
  if (math != SEGCONV_MATH_EXACT && math != SEGCONV_MATH_FFMA && math != SEGCONV_MATH_BF16)
    return fail(SEGCONV_E_UNSUPPORTED, "math mode %d has no backward kernels in this build", (int)math);
  BackwardProblem pr{};
  pr.x = d_src;
  pr.gy = d_gy;
  pr.k = d_kernel;
  pr.dtype = dtype;
  pr.batch = batch;
  pr.n = h;
  pr.cin = cin;
  pr.cout = cout;
  pr.kh = kh;
  pr.kw = kw;
  pr.p = 0;
  pr.pf = 0;
  pr.out_h = h - kh + 1;
  pr.out_w = w - kw + 1;
  pr.stride = 1;
  pr.in_h = h;
  pr.in_w = w;
  pr.conv = 1;
  pr.gx = d_gx;
  pr.gk = d_gk;
  pr.accumulate = accumulate ? 1 : 0;
  return run_backward(pr, math, (cudaStream_t)stream, "conv2d_valid_backward");
}

// reference reference_ops.hpp:116-133
segconv_status segconv_transpose_conv_naive(const void* d_x, segconv_dtype dtype, int batch,
                                            int n_in, int cin, const void* d_kernel, int kh,
                                            int kw, int cout, int p_orig, void* d_workspace,
                                            size_t workspace_bytes, const float* d_bias,
                                            unsigned epilogue, segconv_math math, void* d_y,
                                            void* stream) {
  if (cin < 1 || cout < 1) return fail(SEGCONV_E_SHAPE, "bad kernel dims");
  segconv_geometry g;
  segconv_status st = segconv_tconv_geometry(n_in, kh, kw, p_orig, &g);
  if (st != SEGCONV_OK) return st;
  if (batch < 0) return fail(SEGCONV_E_CONTRACT, "batch must be >= 0");
  const size_t need = segconv_naive_workspace_bytes(dtype, batch, n_in, cin, p_orig);
  if (workspace_bytes < need)
    return fail(SEGCONV_E_CONTRACT, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
  if (batch == 0) return SEGCONV_OK;
  st = segconv_upsample2x_pad(d_x, dtype, batch, n_in, cin, p_orig, d_workspace, stream);
  if (st != SEGCONV_OK) return st;
  return segconv_conv2d_valid(d_workspace, dtype, batch, g.up_h, g.up_w, cin, d_kernel, kh, kw,
                              cout, d_bias, epilogue, math, d_y, stream);
}

// reference analysis.hpp:31-67
segconv_status segconv_count_ops(int n_in, int cin, int cout, int kh, int kw, int p_orig,
                                 uint64_t out[4]) {
  if (cin < 1 || cout < 1)
    return fail(SEGCONV_E_SHAPE, "channel counts must be positive, got cin=%d cout=%d", cin, cout);
  segconv_geometry g;
  segconv_status st = segconv_tconv_geometry(n_in, kh, kw, p_orig, &g);
  if (st != SEGCONV_OK) return st;
  const uint64_t el = (uint64_t)g.out_h * g.out_w * cout, dl = (uint64_t)kh * kw * cin;
  out[0] = el * dl;
  out[1] = el * dl - el;
  out[2] = out[3] = 0;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      const uint64_t pos = (uint64_t)((g.out_h - r + 1) / 2) * ((g.out_w - c + 1) / 2);
      const uint64_t len = (uint64_t)segconv_active_tap_count(kh, p_orig, r) *
                           segconv_active_tap_count(kw, p_orig, c) * cin;
      if (len == 0) continue;
      out[2] += pos * cout * len;
      out[3] += pos * cout * (len - 1);
    }
  return SEGCONV_OK;
}

}  // extern "C"

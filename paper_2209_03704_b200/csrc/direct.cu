// direct.cu -- SIMT kernels for the segregated transpose convolution (K2 + K4).
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60
// (fused_from_padded) and the dot loop it calls, reference_ops.hpp:31-79
// (accumulate_window*):
//   out[2i+r][2j+c][f] = sum_{u<act_r, v<act_c, ch}
//       xpad[i+off_r+u][j+off_c+v][ch] * sub_rc[u][v][ch][f]
// with xpad = x zero-padded by p_fused = p/2.  No padded copy is built: the
// halo loads predicate on the image bounds instead (reference pads with a
// full copy, fused_tconv.hpp:73).
//
// Three kernels:
//  * tconv_generic   -- one thread per output element; any shape, any dtype,
//                       optional EXACT mode (reference (u,v,ch) order, no FMA
//                       contraction: bit-identical to the reference on CPU).
//  * tconv_pixlanes  -- low-Cout layers (Cout <= 4: C1, C4, C5d).  Lanes own
//                       consecutive quad columns; each thread keeps QV quads
//                       stacked vertically x all four parity classes x Cout in
//                       registers.  One shared-memory halo tile (channel
//                       planes) feeds all four parities; weights are warp-wide
//                       broadcast reads.
//  * tconv_coutlanes -- wider layers (Cout > 4: C2).  Lanes own 32
//                       consecutive output features; each lane keeps a QHxQW
//                       block of quads x 4 classes; the input window is a
//                       broadcast read, weights a conflict-free per-lane read.
// Both tiled kernels write each parity straight into its interleaved output
// position (2i+r, 2j+c) with bias/ReLU/tanh fused (K4).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace segconv_b200 {

// ---------------------------------------------------------------- generic
template <typename TX, typename TW, typename ACC, bool EXACT>
__global__ void __launch_bounds__(256) tconv_generic(FusedProblem pr) {
  const long long total = (long long)pr.batch * pr.out_h * pr.out_w * pr.cout;
  const TX* __restrict__ x = (const TX*)pr.x;
  const TW* __restrict__ panels = (const TW*)pr.panels;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(e % pr.cout);
    long long t = e / pr.cout;
    const int ox = (int)(t % pr.out_w);
    t /= pr.out_w;
    const int oy = (int)(t % pr.out_h);
    const int b = (int)(t / pr.out_h);
    const int r = oy & 1, c = ox & 1, q = r * 2 + c, i = oy >> 1, j = ox >> 1;
    const int skh = pr.cls.kh[q], skw = pr.cls.kw[q];
    const TW* w = panels + pr.cls.sub_offset[q];
    ACC acc = 0;
    for (int u = 0; u < skh; ++u) {
      const int row = i + pr.cls.off_r[q] + u - pr.pf;
      if (row < 0 || row >= pr.n) continue;  // zero padding contributes +-0 (exact to skip)
      for (int v = 0; v < skw; ++v) {
        const int col = j + pr.cls.off_c[q] + v - pr.pf;
        if (col < 0 || col >= pr.n) continue;
        const TX* xp = x + (((long long)b * pr.n + row) * pr.n + col) * pr.cin;
        const TW* wp = w + ((long long)(u * skw + v) * pr.cin) * pr.cout + f;
        for (int ch = 0; ch < pr.cin; ++ch) {
          const ACC a = (ACC)to_acc(xp[ch]);
          const ACC bb = (ACC)to_acc(wp[(long long)ch * pr.cout]);
          if constexpr (EXACT) {
            if constexpr (sizeof(ACC) == 8)
              acc = __dadd_rn(acc, __dmul_rn(a, bb));
            else
              acc = __fadd_rn(acc, __fmul_rn(a, bb));
          } else {
            acc = fma(a, bb, acc);
          }
        }
      }
    }
    store_out(pr.y, e, epilogue_apply(acc, pr.epi, pr.bias, f), pr.y_dtype);
  }
}

cudaError_t launch_direct_generic(const FusedProblem& pr, bool exact, cudaStream_t s) {
  const long long total = (long long)pr.batch * pr.out_h * pr.out_w * pr.cout;
  if (total == 0) return cudaSuccess;
  long long blocks = (total + 255) / 256;
  blocks = std::min<long long>(blocks, 148LL * 64);
#define GEN(TX, TW, ACC)                                                         \
  do {                                                                           \
    if (exact)                                                                   \
      tconv_generic<TX, TW, ACC, true><<<(unsigned)blocks, 256, 0, s>>>(pr);     \
    else                                                                         \
      tconv_generic<TX, TW, ACC, false><<<(unsigned)blocks, 256, 0, s>>>(pr);    \
    note_launch();                                                               \
    return cudaGetLastError();                                                   \
  } while (0)
  const int xd = pr.x_dtype, wd = pr.panel_dtype;
  if (pr.panel_layout != SEGCONV_PANEL_REF) return cudaErrorNotSupported;
  if (xd == SEGCONV_F64 || wd == SEGCONV_F64) {
    if (xd == SEGCONV_F64 && wd == SEGCONV_F64) GEN(double, double, double);
    return cudaErrorNotSupported;
  }
  if (xd == SEGCONV_F32 && wd == SEGCONV_F32) GEN(float, float, float);
  if (xd == SEGCONV_BF16 && wd == SEGCONV_BF16) GEN(__nv_bfloat16, __nv_bfloat16, float);
  if (xd == SEGCONV_F32 && wd == SEGCONV_BF16) GEN(float, __nv_bfloat16, float);
  if (xd == SEGCONV_BF16 && wd == SEGCONV_F32) GEN(__nv_bfloat16, float, float);
#undef GEN
  return cudaErrorNotSupported;
}

// ------------------------------------------------------ compile-time parity
// Square K x K kernel, padding parity PODD (reference segregation.hpp:23-36).
template <int K, int PODD>
struct Par {
  __host__ __device__ static constexpr int u0(int r) { return (PODD + r) & 1; }
  __host__ __device__ static constexpr int act(int r) {
    return u0(r) >= K ? 0 : (K - u0(r) + 1) / 2;
  }
  __host__ __device__ static constexpr int off(int r) { return PODD ? 0 : r; }
  __host__ __device__ static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  // Union window extent (rows of input one quad anchor touches).
  static constexpr int U = cmax(off(0) + act(0), off(1) + act(1));
  __host__ __device__ static constexpr int taps(int q) { return act(q >> 1) * act(q & 1); }
  __host__ __device__ static constexpr int tap_base(int q) {
    return q == 0 ? 0 : tap_base(q - 1) + taps(q - 1);
  }
  static constexpr int TAPS = K * K;
};

template <typename TX>
__device__ __forceinline__ float ldx(const TX* p) {
  return to_acc(*p);
}

// Cooperative halo load: rows [gr0, gr0+TH), cols [gc0, gc0+TW), channels
// [ci0, ci0+CI) of image b into xs[CI][TH][TWP] (zero outside the image or
// past cin -- this is the p_fused zero padding, never materialised in HBM).
template <typename TX, int CI, int TH, int TW, int TWP>
__device__ __forceinline__ void load_halo(float* xs, const TX* __restrict__ x, int b, int n,
                                          int cin, int gr0, int gc0, int ci0, int tid,
                                          int nthr) {
  constexpr int PIX = TH * TW;
  // only the channels that exist (a 1-channel layer loads 1/CI of the tile)
  const int nch = min(CI, cin - ci0);
  for (int idx = tid; idx < PIX * nch; idx += nthr) {
    const int ch = idx % nch;
    const int pix = idx / nch;
    const int row = pix / TW, col = pix - (pix / TW) * TW;
    const int gr = gr0 + row, gc = gc0 + col, gch = ci0 + ch;
    float v = 0.0f;
    if (gr >= 0 && gr < n && gc >= 0 && gc < n && gch < cin)
      v = ldx(x + (((long long)b * n + gr) * n + gc) * cin + gch);
    xs[(ch * TH + row) * TWP + col] = v;
  }
}

// Weights for channels [ci0, ci0+CI), features [f0, f0+FW) into
// ws[CI][TAPS][FW] (tap t enumerates class q, u, v in panel order).
template <int K, int PODD, int CI, int FW, typename TW>
__device__ __forceinline__ void load_weights(float* ws, const TW* __restrict__ panels,
                                             const SegClasses& cls, int cin, int cout, int ci0,
                                             int f0, int tid, int nthr) {
  using P = Par<K, PODD>;
  constexpr int TAPS = P::TAPS;
  const int nch = min(CI, cin - ci0);
  for (int idx = tid; idx < nch * TAPS * FW; idx += nthr) {
    const int fl = idx % FW;
    const int t = (idx / FW) % TAPS;
    const int ch = idx / (FW * TAPS);
    int q = 0;
#pragma unroll
    for (int qq = 1; qq < 4; ++qq)
      if (t >= P::tap_base(qq)) q = qq;
    const int tl = t - P::tap_base(q);  // = u * act_c + v
    const int f = f0 + fl, gch = ci0 + ch;
    float v = 0.0f;
    if (f < cout && gch < cin && P::taps(q) > 0)
      v = to_acc(panels[cls.sub_offset[q] + ((long long)tl * cin + gch) * cout + f]);
    ws[(ch * TAPS + t) * FW + fl] = v;
  }
}

// ------------------------------------------------------------- pixlanes
// Cout <= 4.  Tile: (WH*QV) x (WW*32) quad anchors of one image.
template <int K, int PODD, int CO, int QV, int WH, int WW, int CI, typename TX, typename TWt>
__global__ void __launch_bounds__(WH* WW * 32) tconv_pixlanes(FusedProblem pr, int tiles_h,
                                                              int tiles_w) {
  using P = Par<K, PODD>;
  constexpr int U = P::U, TAPS = P::TAPS;
  constexpr int TQH = WH * QV, TQW = WW * 32;
  constexpr int TH = TQH + U - 1, TW = TQW + U - 1;
  constexpr int TWP = TW + 1;
  constexpr int NT = WH * WW * 32;
  extern __shared__ float4 smem4[];
  float* xs = reinterpret_cast<float*>(smem4);
  float* ws = xs + ((CI * TH * TWP + 3) & ~3);  // [CI][TAPS][4]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wh = warp / WW, ww = warp % WW;
  int tile = blockIdx.x;
  const int tj = tile % tiles_w;
  tile /= tiles_w;
  const int ti = tile % tiles_h;
  const int b = tile / tiles_h;
  const int i0 = ti * TQH, j0 = tj * TQW;

  float acc[4][QV][CO];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int a = 0; a < QV; ++a)
#pragma unroll
      for (int co = 0; co < CO; ++co) acc[q][a][co] = 0.0f;

  const TX* __restrict__ x = (const TX*)pr.x;
  for (int ci0 = 0; ci0 < pr.cin; ci0 += CI) {
    __syncthreads();
    load_halo<TX, CI, TH, TW, TWP>(xs, x, b, pr.n, pr.cin, i0 - pr.pf, j0 - pr.pf, ci0, tid, NT);
    load_weights<K, PODD, CI, 4>(ws, (const TWt*)pr.panels, pr.cls, pr.cin, pr.cout, ci0, 0, tid,
                                 NT);
    __syncthreads();
    const int nch = min(CI, pr.cin - ci0);
    for (int ch = 0; ch < nch; ++ch) {
      float xw[QV + U - 1][U];
      const float* xrow = xs + (ch * TH + wh * QV) * TWP + ww * 32 + lane;
#pragma unroll
      for (int a = 0; a < QV + U - 1; ++a)
#pragma unroll
        for (int bb = 0; bb < U; ++bb) xw[a][bb] = xrow[a * TWP + bb];
      const float4* wrow = reinterpret_cast<const float4*>(ws + ch * TAPS * 4);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        constexpr int dummy = 0;
        (void)dummy;
        const int r = q >> 1, c = q & 1;
#pragma unroll
        for (int u = 0; u < P::act(r); ++u)
#pragma unroll
          for (int v = 0; v < P::act(c); ++v) {
            const float4 w4 = wrow[P::tap_base(q) + u * P::act(c) + v];
            const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int a = 0; a < QV; ++a) {
              const float xv = xw[a + P::off(r) + u][P::off(c) + v];
#pragma unroll
              for (int co = 0; co < CO; ++co) acc[q][a][co] = fmaf(xv, wv[co], acc[q][a][co]);
            }
          }
      }
    }
  }

  // K4 epilogue: interleaved store out[2i+r][2j+c][co].
  const int j = j0 + ww * 32 + lane;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, c = q & 1;
    if (j >= pr.cls.cols[q]) continue;
#pragma unroll
    for (int a = 0; a < QV; ++a) {
      const int i = i0 + wh * QV + a;
      if (i >= pr.cls.rows[q]) continue;
      const long long base =
          (((long long)b * pr.out_h + (2 * i + r)) * pr.out_w + (2 * j + c)) * pr.cout;
#pragma unroll
      for (int co = 0; co < CO; ++co)
        store_out(pr.y, base + co, epilogue_apply(acc[q][a][co], pr.epi, pr.bias, co), pr.y_dtype);
    }
  }
}

// ------------------------------------------------------------ coutlanes
// Cout > 4.  Lanes = 32 consecutive features (blockIdx.y selects the group).
template <int K, int PODD, int QH, int QW, int WH, int WW, int CI, typename TX, typename TWt>
__global__ void __launch_bounds__(WH* WW * 32) tconv_coutlanes(FusedProblem pr, int tiles_h,
                                                               int tiles_w) {
  using P = Par<K, PODD>;
  constexpr int U = P::U, TAPS = P::TAPS;
  constexpr int TQH = WH * QH, TQW = WW * QW;
  constexpr int TH = TQH + U - 1, TW = TQW + U - 1;
  constexpr int TWP = (TW + 3) & ~3;
  constexpr int NT = WH * WW * 32;
  constexpr int XW = QW + U - 1;
  extern __shared__ float4 smem4[];
  float* xs = reinterpret_cast<float*>(smem4);
  float* ws = xs + CI * TH * TWP;  // [CI][TAPS][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wh = warp / WW, ww = warp % WW;
  int tile = blockIdx.x;
  const int tj = tile % tiles_w;
  tile /= tiles_w;
  const int ti = tile % tiles_h;
  const int b = tile / tiles_h;
  const int i0 = ti * TQH, j0 = tj * TQW;
  const int f0 = blockIdx.y * 32;

  float acc[4][QH][QW];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int a = 0; a < QH; ++a)
#pragma unroll
      for (int bb = 0; bb < QW; ++bb) acc[q][a][bb] = 0.0f;

  const TX* __restrict__ x = (const TX*)pr.x;
  for (int ci0 = 0; ci0 < pr.cin; ci0 += CI) {
    __syncthreads();
    load_halo<TX, CI, TH, TW, TWP>(xs, x, b, pr.n, pr.cin, i0 - pr.pf, j0 - pr.pf, ci0, tid, NT);
    load_weights<K, PODD, CI, 32>(ws, (const TWt*)pr.panels, pr.cls, pr.cin, pr.cout, ci0, f0,
                                  tid, NT);
    __syncthreads();
    const int nch = min(CI, pr.cin - ci0);
#pragma unroll 2
    for (int ch = 0; ch < nch; ++ch) {
      float xw[QH + U - 1][XW];
      const float* xb = xs + (ch * TH + wh * QH) * TWP + ww * QW;
#pragma unroll
      for (int a = 0; a < QH + U - 1; ++a)
#pragma unroll
        for (int bb = 0; bb < XW; ++bb) xw[a][bb] = xb[a * TWP + bb];  // broadcast
      const float* wl = ws + ch * TAPS * 32 + lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = q >> 1, c = q & 1;
#pragma unroll
        for (int u = 0; u < P::act(r); ++u)
#pragma unroll
          for (int v = 0; v < P::act(c); ++v) {
            const float wv = wl[(P::tap_base(q) + u * P::act(c) + v) * 32];
#pragma unroll
            for (int a = 0; a < QH; ++a)
#pragma unroll
              for (int bb = 0; bb < QW; ++bb)
                acc[q][a][bb] = fmaf(xw[a + P::off(r) + u][bb + P::off(c) + v], wv, acc[q][a][bb]);
          }
      }
    }
  }

  const int f = f0 + lane;
  if (f >= pr.cout) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, c = q & 1;
#pragma unroll
    for (int a = 0; a < QH; ++a) {
      const int i = i0 + wh * QH + a;
      if (i >= pr.cls.rows[q]) continue;
#pragma unroll
      for (int bb = 0; bb < QW; ++bb) {
        const int j = j0 + ww * QW + bb;
        if (j >= pr.cls.cols[q]) continue;
        const long long idx =
            (((long long)b * pr.out_h + (2 * i + r)) * pr.out_w + (2 * j + c)) * pr.cout + f;
        store_out(pr.y, idx, epilogue_apply(acc[q][a][bb], pr.epi, pr.bias, f), pr.y_dtype);
      }
    }
  }
}

// ------------------------------------------------------------- dispatch
template <int K, int PODD, int CO, typename TX, typename TWt>
static cudaError_t run_pixlanes(const FusedProblem& pr, cudaStream_t s) {
  constexpr int QV = 4, WH = 2, WW = 2, CI = 16;
  using P = Par<K, PODD>;
  constexpr int U = P::U;
  constexpr int TH = WH * QV + U - 1, TW = WW * 32 + U - 1, TWP = TW + 1;
  const size_t smem = (size_t)(((CI * TH * TWP + 3) & ~3) + CI * P::TAPS * 4) * sizeof(float);
  auto kern = tconv_pixlanes<K, PODD, CO, QV, WH, WW, CI, TX, TWt>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int rows0 = pr.cls.rows[0] > pr.cls.rows[2] ? pr.cls.rows[0] : pr.cls.rows[2];
  const int cols0 = pr.cls.cols[0] > pr.cls.cols[1] ? pr.cls.cols[0] : pr.cls.cols[1];
  const int tiles_h = (rows0 + WH * QV - 1) / (WH * QV);
  const int tiles_w = (cols0 + WW * 32 - 1) / (WW * 32);
  const long long blocks = (long long)tiles_h * tiles_w * pr.batch;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorNotSupported;
  kern<<<(unsigned)blocks, WH * WW * 32, smem, s>>>(pr, tiles_h, tiles_w);
  note_launch();
  return cudaGetLastError();
}

template <int K, int PODD, typename TX, typename TWt>
static cudaError_t run_coutlanes(const FusedProblem& pr, cudaStream_t s) {
  constexpr int QH = 2, QW = 8, WH = 4, WW = 1, CI = 32;
  using P = Par<K, PODD>;
  constexpr int U = P::U;
  constexpr int TH = WH * QH + U - 1, TW = WW * QW + U - 1, TWP = (TW + 3) & ~3;
  const size_t smem = (size_t)(CI * TH * TWP + CI * P::TAPS * 32) * sizeof(float);
  auto kern = tconv_coutlanes<K, PODD, QH, QW, WH, WW, CI, TX, TWt>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int rows0 = pr.cls.rows[0] > pr.cls.rows[2] ? pr.cls.rows[0] : pr.cls.rows[2];
  const int cols0 = pr.cls.cols[0] > pr.cls.cols[1] ? pr.cls.cols[0] : pr.cls.cols[1];
  const int tiles_h = (rows0 + WH * QH - 1) / (WH * QH);
  const int tiles_w = (cols0 + WW * QW - 1) / (WW * QW);
  const long long blocks = (long long)tiles_h * tiles_w * pr.batch;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffLL) return cudaErrorNotSupported;
  dim3 grid((unsigned)blocks, (pr.cout + 31) / 32);
  kern<<<grid, WH * WW * 32, smem, s>>>(pr, tiles_h, tiles_w);
  note_launch();
  return cudaGetLastError();
}

template <int K, int PODD, typename TX, typename TW>
static cudaError_t run_tiled_k(const FusedProblem& pr, cudaStream_t s) {
  switch (pr.cout) {
    case 1: return run_pixlanes<K, PODD, 1, TX, TW>(pr, s);
    case 2: return run_pixlanes<K, PODD, 2, TX, TW>(pr, s);
    case 3: return run_pixlanes<K, PODD, 3, TX, TW>(pr, s);
    case 4: return run_pixlanes<K, PODD, 4, TX, TW>(pr, s);
    default: return run_coutlanes<K, PODD, TX, TW>(pr, s);
  }
}

template <typename TX, typename TW>
static cudaError_t run_tiled_t(const FusedProblem& pr, cudaStream_t s) {
  const int podd = pr.p & 1;
#define KC(KK)                                                          \
  case KK:                                                              \
    return podd ? run_tiled_k<KK, 1, TX, TW>(pr, s) : run_tiled_k<KK, 0, TX, TW>(pr, s);
  switch (pr.kh) {
    KC(1) KC(2) KC(3) KC(4) KC(5) KC(6) KC(7)
    default: return cudaErrorNotSupported;
  }
#undef KC
}

// ------------------------------------------------------------ tiny layers
// One thread per output element (b, oy, ox, f): class (oy & 1, ox & 1),
// anchor (oy >> 1, ox >> 1), dot over the class's taps and channels in the
// reference order (u, v, ch).  For layers whose whole work is a few thousand
// MACs (BASELINE C1: 1 x 32^2 x 1 -> 61^2 x 1) the tiled kernels' staging
// is pure latency; this is one global read per tap.
template <typename TX, typename TW>
__global__ void __launch_bounds__(256) tconv_outputs(const FusedProblem pr, int total) {
  // one thread per output (tiny layers, e.g. BASELINE C1: 3721 outputs of 1
  // channel).  The class's taps are unrolled (<= 4 x 4 for kh <= 7) so that
  // their loads issue back to back: after an L2 flush each is a DRAM round
  // trip, and a runtime tap loop serialised them (6.3 us for C1).  32-bit
  // index math (total < 2^16 outputs).
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int f = e % pr.cout;
  int t = e / pr.cout;
  const int ox = t % pr.out_w;
  t /= pr.out_w;
  const int oy = t % pr.out_h;
  const int b = t / pr.out_h;
  const int r = oy & 1, c = ox & 1, q = r * 2 + c, i = oy >> 1, j = ox >> 1;
  const TX* __restrict__ x = (const TX*)pr.x;
  const TW* __restrict__ w = (const TW*)pr.panels + pr.cls.sub_offset[q];
  const int kh = pr.cls.kh[q], kw = pr.cls.kw[q], n = pr.n, cin = pr.cin, cout = pr.cout;
  const int r0 = i + pr.cls.off_r[q] - pr.pf, c0 = j + pr.cls.off_c[q] - pr.pf;
  float acc = 0.0f;
  if (cin == 1) {
    float xv[4][4], wv[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int gr = r0 + u, gc = c0 + v;
        const bool ok = u < kh && v < kw && gr >= 0 && gr < n && gc >= 0 && gc < n;  // zero padding
        xv[u][v] = ok ? to_acc(x[(b * n + gr) * n + gc]) : 0.0f;
        wv[u][v] = ok ? to_acc(w[(u * kw + v) * cout + f]) : 0.0f;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)  // reference order: u, v
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (u < kh && v < kw) acc = fmaf(xv[u][v], wv[u][v], acc);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u >= kh) break;
      const int gr = r0 + u;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int gc = c0 + v;
        if (v >= kw || gr < 0 || gr >= n || gc < 0 || gc >= n) continue;  // zero padding
        const TX* xp = x + ((long long)(b * n + gr) * n + gc) * cin;
        const TW* wp = w + ((long long)(u * kw + v) * cin) * cout + f;
        for (int ch = 0; ch < cin; ++ch) acc = fmaf(to_acc(xp[ch]), to_acc(wp[(long long)ch * cout]), acc);
      }
    }
  }
  store_out(pr.y, e, epilogue_apply(acc, pr.epi, pr.bias, f), pr.y_dtype);
}

static bool tiny_layer(const FusedProblem& pr) {
  const long long outs = (long long)pr.batch * pr.out_h * pr.out_w * pr.cout;
  return outs <= (1 << 16) && (long long)pr.kh * pr.kw * pr.cin <= 64;
}

cudaError_t launch_direct_tiled(const FusedProblem& pr, cudaStream_t s) {
  if (pr.kh != pr.kw || pr.kh < 1 || pr.kh > 7) return cudaErrorNotSupported;
  if (pr.panel_layout != SEGCONV_PANEL_REF) return cudaErrorNotSupported;
  if (tiny_layer(pr) && ((pr.x_dtype == SEGCONV_F32 && pr.panel_dtype == SEGCONV_F32) ||
                         (pr.x_dtype == SEGCONV_BF16 && pr.panel_dtype == SEGCONV_BF16))) {
    const int total = (int)((long long)pr.batch * pr.out_h * pr.out_w * pr.cout);  // <= 2^16 (tiny_layer)
    if (total == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    if (pr.x_dtype == SEGCONV_F32)
      tconv_outputs<float, float><<<blocks, 256, 0, s>>>(pr, total);
    else
      tconv_outputs<__nv_bfloat16, __nv_bfloat16><<<blocks, 256, 0, s>>>(pr, total);
    note_launch();
    return cudaGetLastError();
  }
  if (pr.x_dtype == SEGCONV_F32 && pr.panel_dtype == SEGCONV_F32)
    return run_tiled_t<float, float>(pr, s);
  if (pr.x_dtype == SEGCONV_BF16 && pr.panel_dtype == SEGCONV_BF16)
    return run_tiled_t<__nv_bfloat16, __nv_bfloat16>(pr, s);
  return cudaErrorNotSupported;
}

}  // namespace segconv_b200

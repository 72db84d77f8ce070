// tc_ring.cu -- K3 for high-resolution, few-output-channel layers (BASELINE
// C4: 32 x 256^2 x 64 -> 507^2 x 3, n = 5, fp32 with split-fp16 math).
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for these layers.
//
// Why a third formulation.  With cout = 3 the four parity classes give 12
// output rows; the halo-shift GEMMs (tc_igemm.cu, tc_fold.cu) then spend one
// 128-row MMA per tap-shift on 12-16 useful rows.  Here the GEMM runs the
// other way round -- "pixel scatter":
//   D[p, (dy, q, dx, f)] = sum_ch X[p, ch] * W_q[dy - off_r][dx - off_c][ch][f]
// for every input pixel p of one image row and every (shift, class, feature)
// that exists (25 x 3 = 75 columns for n = 5), so each MMA computes only
// useful products: M = 128 pixels, N = 80, K = cin.  The shift sum moves to
// the epilogue:
//   out_q[f](i, j) = sum_{dy, dx} D[(i + dy, j + dx), (dy, q, dx, f)]
// * dx: TMEM lane = pixel column, so pixel j + dx is dx lanes down --
//   warp shuffles (plus a 2-lane exchange between neighbouring warps);
// * dy: each CTA streams consecutive image rows; every thread keeps the
//   partial sums of anchor rows R-2, R-1, R for its column in registers (a
//   three-row ring), so anchor row R-2 is complete after pixel row R and is
//   written out -- two output rows, each a contiguous 24-byte run per thread.
// No halo is staged (pixels are read once), no shared-memory atomics.
//
// Data path per pixel row (a "unit"): two TMA boxes {32 channels, n pixels}
// fp32 with the 128-byte swizzle, split in place into fp16 hi/lo planes
// (split-fp16 math: y = xh*wh + xl*wh + xh*wl), n/128 M-tiles x 2 k-steps x
// 3 products = 12 MMAs per 32 channels (SS form, weights resident in SMEM),
// D double-buffered in TMEM.
//
// Warp roles (448 threads): 0-7 epilogue (warp w <-> pixels [32w, 32w+32):
// M-tile w / 4, TMEM lane quadrant w % 4), 8-11 converters, 12 MMA issuer,
// 13 TMA producer / TMEM owner.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_scatter.cuh"
#include "tc_guard.cuh"

namespace segconv_b200 {
namespace tcr {

using namespace tc;

constexpr int NUM_THREADS = 448;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int KB = 32;  // channels per stage: one 128-byte fp32 TMA row
constexpr int CH = KB / 8;
constexpr int MAX_STAGES = 6;

template <int KH, int COUT>
using Layout = ScatterLayout<KH, COUT>;

struct Params {
  const uint8_t* panels;  // ring weight image (segconv_ring_image): [plane][chunk][N][8 fp16]
  void* y;
  const float* bias;
  unsigned epi;
  int batch, n, cin, cout, out_h, out_w;
  int rm;           // anchor rows per image that any class writes (= rows of class r = 0)
  long long g_total;  // batch * rm
  int rows[4], cols[4];
  int stage_bytes, stages, w_bytes;
  unsigned long long* trace;
  int debug;
  FallbackArgs fb;  // range guard (tc_guard.cuh): weight scale, FFMA fallback
};

__device__ __forceinline__ void trace_ev(const Params& p, int ev, int local) {
  if (p.trace == nullptr || blockIdx.x >= 160 || local >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[(blockIdx.x * 16 + ev) * 64 + local] = t;
}

// Unit k of this CTA -> (image b, pixel row R, anchor row completed after it
// or -1, first unit of a segment?).  The CTA owns anchor rows [g0, g1) of the
// batch (g = b * rm + i); a segment is one image's share; pixel rows
// [i_s, i_e + U - 1) are streamed per segment.
template <int U>
__device__ __forceinline__ bool unit_at(const Params& p, int k, int& b, int& R, int& a_out,
                                        bool& seg_start) {
  const long long g0 = p.g_total * blockIdx.x / gridDim.x;
  const long long g1 = p.g_total * (blockIdx.x + 1) / gridDim.x;
  long long g = g0;
  while (g < g1) {
    const int bb = (int)(g / p.rm);
    const int i_s = (int)(g - (long long)bb * p.rm);
    const int i_e = (int)min((long long)p.rm, g1 - (long long)bb * p.rm);
    const int units = i_e - i_s + U - 1;
    if (k < units) {
      b = bb;
      R = i_s + k;
      const int a = R - (U - 1);
      a_out = (a >= i_s && a < i_e) ? a : -1;
      seg_start = k == 0;
      return true;
    }
    k -= units;
    g = (long long)(bb + 1) * p.rm;
  }
  return false;
}

template <int KH, int COUT, int ACT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    ring_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  using L = Layout<KH, COUT>;
  constexpr int U = L::U, N = L::N;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages;
  uint8_t* a_base = smem;  // stages first: 1024-byte aligned for the swizzled TMA
  uint8_t* w_base = smem + (size_t)SA * p.stage_bytes;
  float* xchg = reinterpret_cast<float*>(w_base + p.w_bytes);  // [8 warps][2 lanes][33 floats]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg + 8 * 2 * 33 + 2);
  uint64_t* a_land = bars;
  uint64_t* a_full = a_land + SA;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);
  // a converter saw x outside the split's range (the word after the TMEM slot)
  volatile int& guard_bad = *reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) guard_bad = 0;
  if (warp == 12 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_land[s], 1);
      mbar_init(&a_full[s], 128);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 256);
    }
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 13) {
    if (lane == 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic stream serialization: the prologue above overlaps the previous
  // kernel's tail; every global access (weight image, pixel rows, stores, guard
  // fallback) follows this wait.
  griddep_wait();

  const int NH = p.cin / KB;   // stages per pixel row
  const int TILES = p.n / 128;  // M-tiles per pixel row
  const int CHT = p.cin / 8;
  const uint32_t COL = (uint32_t)p.n * 16;  // one operand k-chunk column (one plane)
  const uint32_t WCOL = (uint32_t)N * 16;    // one weight k-chunk column

  if (warp == 13) {
    // ===== TMA producer: weights once, then two boxes {32 ch, n pixels} per row
    if (lane == 0) {
      mbar_arrive_expect_tx(w_full, (uint32_t)p.w_bytes);
      for (uint32_t off = 0; off < (uint32_t)p.w_bytes; off += 32768)
        bulk_g2s(w_base + off, p.panels + off, min(32768u, (uint32_t)p.w_bytes - off), w_full);
      int st = 0;
      uint32_t ph = 0;
      const uint32_t tx = (uint32_t)p.n * KB * 4;
      int b, R, a;
      bool s0;
      for (int k = 0; unit_at<U>(p, k, b, R, a, s0); ++k) {
        const int pix0 = (b * p.n + R) * p.n;
        for (int h = 0; h < NH; ++h) {
          mbar_wait(&a_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&a_land[st], tx);
          tma_load_2d(smem_u32(a_base + (size_t)st * p.stage_bytes), &tmap, h * KB, pix0, &a_land[st]);
          if (h == 0) trace_ev(p, 0, k);
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ===== converters: swizzled fp32 rows -> fp16 hi/lo k-chunk columns, in place
    const int ct = threadIdx.x - 256;
    int st = 0;
    uint32_t ph = 0;
    int b, R, a;
    bool s0;
    GuardTrack gt;
    gt.init(p.fb.guard);
    for (int k = 0; unit_at<U>(p, k, b, R, a, s0); ++k) {
      for (int h = 0; h < NH; ++h) {
        mbar_wait(&a_land[st], ph);
        const uint32_t sbase = smem_u32(a_base + (size_t)st * p.stage_bytes);
        if (!(p.debug & 2)) {
          float4 v[2][CH][2];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int r = ct + t * 128;
            if (r < p.n) {
              const uint32_t rb = sbase + (uint32_t)r * 128, sw = (uint32_t)(r & 7);
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                ld_shared_v4f(rb + ((((uint32_t)(2 * j)) ^ sw) << 4), v[t][j][0]);
                ld_shared_v4f(rb + ((((uint32_t)(2 * j + 1)) ^ sw) << 4), v[t][j][1]);
                gt.add(v[t][j][0]);
                gt.add(v[t][j][1]);
              }
            }
          }
          named_bar(1, 128);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int r = ct + t * 128;
            if (r < p.n) {
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                uint32_t hi[4], lo[4];
                split8x2(v[t][j][0], v[t][j][1], hi, lo);
                const uint32_t dst = sbase + (uint32_t)j * 2 * COL + (uint32_t)r * 16;
                st_shared_v4(dst, hi[0], hi[1], hi[2], hi[3]);
                st_shared_v4(dst + COL, lo[0], lo[1], lo[2], lo[3]);
              }
            }
          }
        }
        fence_proxy_async();
        if (h == 0 && ct == 0) trace_ev(p, 1, k);
        mbar_arrive(&a_full[st]);
        if (++st == SA) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    if (gt.bad()) guard_bad = 1;
  } else if (warp == 12) {
    // ===== MMA issuer (whole warp in the loop; one elected lane issues)
    const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t wb = smem_u32(w_base);
    const uint32_t WPLANE = (uint32_t)CHT * WCOL;
    constexpr uint32_t IDESC = idesc_f16(0, N);
    int st = 0, acc = 0;
    uint32_t ph = 0, pacc = 0;
    int b, R, a;
    bool s0;
    mbar_wait(w_full, 0);
    tc_fence_after();
    for (int k = 0; unit_at<U>(p, k, b, R, a, s0); ++k) {
      mbar_wait(&acc_empty[acc], pacc ^ 1);
      tc_fence_after();
      if (lane == 0) trace_ev(p, 2, k);
      const uint32_t d0 = tb + (uint32_t)(acc * 2 * N);
      for (int h = 0; h < NH; ++h) {
        mbar_wait(&a_full[st], ph);
        tc_fence_after();
        const uint32_t xb = smem_u32(a_base + (size_t)st * p.stage_bytes);
        if (!(p.debug & 8) && elect_one()) {
          for (int t = 0; t < TILES; ++t) {
#pragma unroll
            for (int ks = 0; ks < CH / 2; ++ks) {
              // pixels [128t, 128t + 128): hi chunks 2ks, 2ks+1 in columns 4ks, 4ks+2
              const uint32_t xk = xb + (uint32_t)ks * 4 * COL + (uint32_t)t * 128 * 16;
              const uint64_t xh = sdesc(xk, 2 * COL, 128), xl = sdesc(xk + COL, 2 * COL, 128);
              const uint32_t wk = wb + (uint32_t)(h * CH + 2 * ks) * WCOL;
              const uint64_t wh = sdesc(wk, WCOL, 128), wl = sdesc(wk + WPLANE, WCOL, 128);
              const uint32_t d = d0 + (uint32_t)(t * N);
              mma_f16(d, xh, wh, IDESC, (h == 0 && ks == 0) ? 0u : 1u);
              mma_f16(d, xl, wh, IDESC, 1u);
              mma_f16(d, xh, wl, IDESC, 1u);
            }
          }
        }
        __syncwarp();
        if (elect_one()) mma_commit(&a_empty[st]);
        __syncwarp();
        if (++st == SA) {
          st = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) mma_commit(&acc_full[acc]);
      __syncwarp();
      if (lane == 0) trace_ev(p, 3, k);
      if (++acc == 2) {
        acc = 0;
        pacc ^= 1;
      }
    }
  } else {
    // ===== epilogue (warps 0-7): thread <-> pixel column j = 32 * warp + lane
    const int j = warp * 32 + lane;
    const int tile = warp >> 2, quad = warp & 3;
    const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(tile * N);
    float ring[U][4][COUT];  // anchor rows R-(U-1) .. R for this column
#pragma unroll
    for (int d = 0; d < U; ++d)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int f = 0; f < COUT; ++f) ring[d][q][f] = 0.0f;
    float bias[COUT];
#pragma unroll
    for (int f = 0; f < COUT; ++f) bias[f] = (p.epi & SEGCONV_EPI_BIAS) ? __ldg(p.bias + f) : 0.0f;
    const float wsc = guard_inv_scale(p.fb.guard);  // the weight image holds w * 2^s
    float chk = 0.0f;  // range guard: NaN once a stored sum is not finite
    float* y = reinterpret_cast<float*>(p.y);
    float* xw = xchg + warp * (2 * 33);          // this warp's exchange rows (lanes 0, 1)
    const float* xn = xchg + (warp + 1) * (2 * 33);  // next warp's
    const bool has_next = warp < 7 && (warp + 1) * 32 < p.n;
    int acc = 0;
    uint32_t pacc = 0;
    int b, R, a;
    bool s0;
    for (int k = 0; unit_at<U>(p, k, b, R, a, s0); ++k) {
      if (s0) {
#pragma unroll
        for (int d = 0; d < U; ++d)
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int f = 0; f < COUT; ++f) ring[d][q][f] = 0.0f;
      }
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0) trace_ev(p, 4, k);
#pragma unroll
      for (int dy = 0; dy < U; ++dy) {
        float v[32];
        const uint32_t ta = lane_base + (uint32_t)(acc * 2 * N + L::group_off(dy));
        if (L::group_pad(dy) > 16)
          tmem_ld32(ta, v);
        else
          tmem_ld16(ta, v);
        // lanes 0 .. U-2 publish their columns for the previous warp's tail lanes
        if (lane < U - 1) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c < L::group_len(dy)) xw[lane * 33 + c] = v[c];
        }
        named_bar(2, 256);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int f = 0; f < COUT; ++f) {
            float s = 0.0f;
#pragma unroll
            for (int dx = 0; dx < U; ++dx) {
              const int c = L::col_in_group(dy, q, dx, f);
              if (c < 0) continue;
              float t = dx == 0 ? v[c] : __shfl_down_sync(0xffffffffu, v[c], dx);
              if (dx > 0 && lane + dx >= 32) t = has_next ? xn[(lane + dx - 32) * 33 + c] : 0.0f;
              s += t;
            }
            if (L::has_dy(q, dy)) ring[U - 1 - dy][q][f] += s;
          }
        }
        named_bar(2, 256);  // exchange rows are rewritten by the next group
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        pacc ^= 1;
      }
      // anchor row a is complete: out[b][2a + r][2j + c][f], bias and activation fused
      if (a >= 0 && !(p.debug & 1)) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (a >= p.rows[r * 2]) continue;
          const long long row0 = ((long long)b * p.out_h + 2 * a + r) * p.out_w;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int q = r * 2 + c;
            if (j >= p.cols[q]) continue;
            float* o = y + (row0 + 2 * j + c) * COUT;
#pragma unroll
            for (int f = 0; f < COUT; ++f) {
              guard_check(chk, ring[0][q][f]);
              float x = ring[0][q][f] * wsc + bias[f];
              if (ACT == 1) x = fmaxf(x, 0.0f);
              if (ACT == 2) x = tanhf(x);
              o[f] = x;
            }
          }
        }
      }
      // rotate the ring: anchor row a + 1 moves to slot 0
#pragma unroll
      for (int d = 0; d < U - 1; ++d)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int f = 0; f < COUT; ++f) ring[d][q][f] = ring[d + 1][q][f];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int f = 0; f < COUT; ++f) ring[U - 1][q][f] = 0.0f;
    }
    if (guard_check_bad(chk)) guard_bad = 1;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
  if (guard_bad) {
    // x left the split-fp16 range in this CTA's rows: recompute its anchor
    // rows [g0, g1) x all columns with FFMA (this CTA wrote them)
    const long long g0 = p.g_total * blockIdx.x / gridDim.x;
    const long long g1 = p.g_total * (blockIdx.x + 1) / gridDim.x;
    guard_fallback(p.fb, (g1 - g0) * p.n, 0, p.cout, [&](long long idx, int& b, int& i, int& j) {
      const long long g = g0 + idx / p.n;
      j = (int)(idx - (idx / p.n) * p.n);
      b = (int)(g / p.rm);
      i = (int)(g - (long long)b * p.rm);
      return true;
    });
  }
}

}  // namespace tcr

// ------------------------------------------------------------ host side
// Weight image for the ring kernel: B operand rows = D columns (dy, q, dx, f)
// of Layout<KH, COUT>, K-major no-swizzle: [plane hi/lo][k-chunk][N rows][8 fp16].
template <int KH, int COUT>
static __global__ void ring_image_kernel(const float* __restrict__ k, int cin, SegClasses cls,
                                         uint16_t* __restrict__ out, const SplitGuard* __restrict__ guard) {
  using L = tcr::Layout<KH, COUT>;
  const float wscale = ldexpf(1.0f, split_scale_exp(guard->amax_bits));
  const int CHT = cin / 8;
  const long long total = (long long)CHT * L::N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e % L::N), chunk = (int)(e / L::N);
    int dy = 0;
    while (dy + 1 < L::U && row >= L::group_off(dy + 1)) ++dy;
    const int cg = row - L::group_off(dy);
    int qq = -1, dxx = -1, ff = -1;
    for (int q = 0; q < 4 && qq < 0; ++q)
      for (int dx = 0; dx < L::U && qq < 0; ++dx)
        for (int f = 0; f < COUT; ++f)
          if (L::col_in_group(dy, q, dx, f) == cg) {
            qq = q;
            dxx = dx;
            ff = f;
            break;
          }
    uint16_t hi[8], lo[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      float w = 0.0f;
      if (qq >= 0) {
        const int u = dy - cls.off_r[qq], v = dxx - cls.off_c[qq];
        const int ci = chunk * 8 + x;
        w = wscale * k[(((long long)(cls.u0[qq] + 2 * u) * KH + (cls.v0[qq] + 2 * v)) * cin + ci) * COUT + ff];
      }
      const __half h = __float2half_rn(w);
      hi[x] = __half_as_ushort(h);
      lo[x] = __half_as_ushort(__float2half_rn(w - __half2float(h)));
    }
    uint16_t* dh = out + e * 8;
    uint16_t* dl = out + total * 8 + e * 8;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      dh[x] = hi[x];
      dl[x] = lo[x];
    }
  }
}

static bool ring_shape(const FusedProblem& pr) {
  // instantiated: 5x5 kernel, 3 outputs, split-fp16 math on fp32 data, p = 0,
  // images of 128 or 256 pixels per row
  return pr.kh == 5 && pr.kw == 5 && pr.cout == 3 && pr.p == 0 && pr.pf == 0 &&
         (pr.n == 128 || pr.n == 256) && pr.cin % tcr::KB == 0 && pr.cin <= 256 &&
         pr.x_dtype == SEGCONV_F32 && pr.y_dtype == SEGCONV_F32;
}

size_t ring_image_bytes(int cin) { return (size_t)2 * (cin / 8) * tcr::Layout<5, 3>::N * 16; }

bool tc_ring_supported(const FusedProblem& pr, int math) {
  if (math != SEGCONV_MATH_F16X3 || !pr.guard) return false;
  return ring_shape(pr);
}

cudaError_t launch_tc_ring(const FusedProblem& pr, const void* ring_img, cudaStream_t s) {
  if (!ring_shape(pr)) return cudaErrorNotSupported;
  using L = tcr::Layout<5, 3>;
  tcr::Params p{};
  p.panels = (const uint8_t*)ring_img;
  p.y = pr.y;
  p.bias = pr.bias;
  p.epi = pr.epi;
  p.batch = pr.batch;
  p.n = pr.n;
  p.cin = pr.cin;
  p.cout = pr.cout;
  p.out_h = pr.out_h;
  p.out_w = pr.out_w;
  for (int q = 0; q < 4; ++q) {
    p.rows[q] = pr.cls.rows[q];
    p.cols[q] = pr.cls.cols[q];
  }
  p.rm = std::max(pr.cls.rows[0], pr.cls.rows[2]);
  p.g_total = (long long)pr.batch * p.rm;
  if (p.g_total == 0) return cudaSuccess;
  p.stage_bytes = pr.n * tcr::KB * 4;  // 128-byte rows; == 4 chunks x 2 planes x n x 16 after the split
  p.w_bytes = (int)ring_image_bytes(pr.cin);
  const int fixed = p.w_bytes + (8 * 2 * 33 + 2) * 4 + (3 * tcr::MAX_STAGES + 5) * 8 + 16;
  p.stages = std::min(tcr::MAX_STAGES, (tcr::SMEM_LIMIT - fixed) / p.stage_bytes);
  if (p.stages < 2) return cudaErrorNotSupported;
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  p.debug = dbg;
  p.trace = tc_trace_buffer();
  p.fb = make_fallback_args(pr, pr.guard);
  // halo-free input view: (cin, batch * n * n) fp32, box {32 ch, n pixels}, 128B swizzle
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);
  static Enc enc = nullptr;
  if (!enc) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    enc = (Enc)f;
  }
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)pr.cin, (cuuint64_t)pr.batch * pr.n * pr.n};
  const cuuint64_t strides[1] = {(cuuint64_t)pr.cin * 4};
  const cuuint32_t box[2] = {(cuuint32_t)tcr::KB, (cuuint32_t)pr.n};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(pr.x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  const int sms = device_sm_count();
  const long long grid = std::min<long long>(p.g_total, sms);
  const size_t smem = (size_t)p.stages * p.stage_bytes + fixed;
  const int act = (pr.epi & SEGCONV_EPI_RELU) ? 1 : (pr.epi & SEGCONV_EPI_TANH) ? 2 : 0;
  cudaError_t e;
#define RING_LAUNCH(A)                                                                           \
  {                                                                                              \
    auto kern = tcr::ring_kernel<5, 3, A>;                                                       \
    static PerDeviceOnce once;                                                                   \
    e = smem_attr_once(once, kern, tcr::SMEM_LIMIT);                                              \
    if (e != cudaSuccess) return e;                                                              \
    cudaLaunchConfig_t cfg = {};                                                                 \
    cfg.gridDim = dim3((unsigned)grid);                                                          \
    cfg.blockDim = dim3(tcr::NUM_THREADS);                                                       \
    cfg.dynamicSmemBytes = smem;                                                                 \
    cfg.stream = s;                                                                              \
    cudaLaunchAttribute at[1];                                                                   \
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                               \
    at[0].val.programmaticStreamSerializationAllowed = 1;                                        \
    cfg.attrs = at;                                                                              \
    cfg.numAttrs = 1;                                                                            \
    e = cudaLaunchKernelEx(&cfg, kern, p, tmap);                                                 \
    if (e != cudaSuccess) return e;                                                              \
  }
  if (act == 1)
    RING_LAUNCH(1)
  else if (act == 2)
    RING_LAUNCH(2)
  else
    RING_LAUNCH(0)
#undef RING_LAUNCH
  (void)L::N;
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_ring_image(const void* k, int k_dtype, int cin, const SegClasses& cls,
                              void* out, const void* guard, cudaStream_t s) {
  if (k_dtype != SEGCONV_F32 || !guard) return cudaErrorNotSupported;
  const long long total = (long long)(cin / 8) * tcr::Layout<5, 3>::N;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 1024);
  ring_image_kernel<5, 3><<<blocks, 256, 0, s>>>((const float*)k, cin, cls, (uint16_t*)out,
                                                 (const SplitGuard*)guard);
  note_launch();
  return cudaGetLastError();
}

}  // namespace segconv_b200

// tc_igemm.cu -- K3 + K4: the segregated transpose convolution as one
// tcgen05 implicit GEMM per group of quad-anchor tiles (sm_100a).
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for wide layers.
//
// Formulation ("halo-shift").  Let the virtual grid be the p_fused-padded
// input (VH x VW per image, never materialised: the producer zero-fills).
// Virtual position m = (b*VH + i)*VW + j is the quad anchor (i, j); class
// (r, c) = q writes out[b][2i+r][2j+c][:] and reads xpad[i+off_r+u][j+off_c+v],
// i.e. virtual pixel m + shift(q,u,v), shift = (off_r+u)*VW + (off_c+v).  So
// for a group of G*128 consecutive anchors EVERY (class, tap) GEMM reads the
// SAME staged halo -- rows [m0, m0 + G*128 + max_shift) -- at a different row
// offset.  The halo is staged once per channel block in the UMMA K-major
// no-swizzle layout: 16-byte k-chunk columns of S_pad rows, one row per
// virtual pixel; a tap's A operand is that buffer with the descriptor start
// moved by shift*16 bytes.  All four classes accumulate in TMEM (G x 4 x NT
// fp32 columns, double-buffered across work units when they fit), and the
// epilogue writes each class's rows straight to their interleaved output
// pixels (2i+r, 2j+c) with bias / ReLU / tanh fused.  Anchors outside a
// class's rows x cols (the padded border of the virtual grid) are computed
// and dropped; the useful fraction is rows*cols / (VH*VW) per class.
//
// Data movement.  With p_fused == 0 the halo rows are consecutive input
// pixels (NHWC is contiguous across rows and images), so a 3-D TMA view
// (8 elems, pixel, 16-byte chunk) with strides (elem, cin, 16 B) drops each
// k-chunk column straight into place (boxes of <= 256 rows, zero-filled past
// the batch).  Otherwise producer warps gather with predicated loads.  Weight
// blocks (the UMMA panel image written by segregate) arrive by cp.async.bulk,
// resident for the whole kernel when they fit, else streamed through a ring.
//
// Warp roles (352 threads, one CTA per SM, persistent over work units):
//   warps 0-3  epilogue   TMEM -> registers -> global (warp w owns lanes 32w..)
//   warps 4-7  converter  F16X3: split the fp32 halo in place into fp16 hi/lo
//                         columns; no-TMA mode: gather the halo from global
//   warp  8    MMA issue  one thread issues tcgen05.mma, commits to mbarriers
//   warp  9    B loader   one thread; the whole warp owns TMEM alloc/dealloc
//   warp 10    A loader   one thread issues the halo TMA boxes
// Math: MODE_BF16 -- bf16 operands, fp32 accumulate (BASELINE C3, C5);
//       MODE_F16X3 -- fp32 operands split x = xh + xl, w = wh + wl (fp16),
//       y = xh*wh + xl*wh + xh*wl: three kind::f16 MMAs, fp32-class accuracy
//       (C2).  Weights are split once by segregate; activations on the fly.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_guard.cuh"

namespace segconv_b200 {
namespace tc {

constexpr int MODE_BF16 = 0, MODE_F16X3 = 1;
constexpr int MAX_TAPS = 49;  // kh * kw <= 7 * 7
constexpr int NUM_THREADS = 352;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int MAX_PIECES = 8;

struct Params {
  const void* x;
  const uint8_t* panels;
  void* y;
  const float* bias;
  unsigned epi;
  int y_dtype;
  int batch, n, cin, cout, pf;
  int VH, VW;
  long long Mv;  // batch * VH * VW virtual positions
  int out_h, out_w;
  int nkb, kb;   // channel blocks, channels per block
  int n_tiles;
  long long m_groups, total_units;
  int S, S_pad;  // halo rows staged per unit, rows per k-chunk column
  int a_stage_bytes, b_stage_bytes;
  int stages_a, stages_b;
  int b_resident;  // 1: every weight block of the (single) n-tile lives in SMEM
  int tma_mode;    // 1: the halo arrives by TMA (p_fused == 0)
  int pieces, piece_rows;
  int taps;
  int tap_class[MAX_TAPS];
  int tap_shift[MAX_TAPS];
  int first_tap[4];
  int rows[4], cols[4];
  unsigned long long* trace;  // optional event trace (SEGCONV_TC_TRACE), CTAs 0..3
  FallbackArgs fb;            // split-fp16 range guard (tc_guard.cuh)
};

// Debug trace: trace[(cta * 8 + event) * 64 + local_unit] = globaltimer (ns).
// events: 0 A-TMA issued, 1 converted, 2 MMA start, 3 MMA issued, 4 epi start, 5 epi done
__device__ __forceinline__ void trace_ev(const Params& p, int ev, int local) {
  if (p.trace == nullptr || blockIdx.x >= 160 || local >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[(blockIdx.x * 16 + ev) * 64 + local] = t;
}

// Work unit u -> (m-group, n-tile); n-tile major so a CTA's units share weights.
__device__ __forceinline__ void unit_coords(const Params& p, long long u, long long& mg, int& nt) {
  nt = (int)(u / p.m_groups);
  mg = u - (long long)nt * p.m_groups;
}

// ------------------------------------------------------------------ kernel
template <int MODE, int NT, int G>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_halo_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  constexpr int ACC_COLS = G * 4 * NT;
  constexpr int ACC_BUFS = (2 * ACC_COLS <= 512) ? 2 : 1;
  constexpr int TMEM_COLS = pow2_cols(ACC_COLS * ACC_BUFS);
  constexpr uint32_t IDESC = idesc_f16(MODE == MODE_BF16 ? 1 : 0, NT);
  constexpr int MPG = G * BM;  // anchors per work unit

  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages_a, SB = p.stages_b;
  const int NB = p.b_resident ? 1 : SB;  // B barriers: one for the resident set
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + (size_t)SA * p.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + (size_t)SB * p.b_stage_bytes);
  uint64_t* a_land = bars;          // TMA bytes landed (F16X3 converters wait here)
  uint64_t* a_full = a_land + SA;   // stage ready for the MMA
  uint64_t* a_empty = a_full + SA;  // MMA done with the stage
  uint64_t* b_full = a_empty + SA;
  uint64_t* b_empty = b_full + NB;
  uint64_t* acc_full = b_empty + NB;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // a converter saw x outside the split's range (the word after the TMEM slot)
  volatile int& guard_bad = *reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) guard_bad = 0;
  // a_full arrivals: the TMA itself (bf16), or the 128 converter/gather threads.
  const uint32_t a_full_count = (p.tma_mode && MODE == MODE_BF16) ? 1u : 128u;
  if (warp == 8 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_land[s], 1);
      mbar_init(&a_full[s], a_full_count);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 10 && lane == 0 && p.tma_mode)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int CH = p.kb / 8;  // 16-byte k-chunks per channel block
  const uint32_t COL = (uint32_t)p.S_pad * 16;  // one k-chunk column (bytes)
  // bf16: chunk j in column j.  f16x3: hi chunk j in column 2j, lo in 2j+1.
  const uint32_t LBO_A = MODE == MODE_F16X3 ? 2 * COL : COL;
  const uint32_t LBO_B = (uint32_t)NT * 16;
  const uint32_t plane_b = (uint32_t)CH * LBO_B;

  if (warp == 10) {
    // =========================== A loader: halo TMA boxes (p_fused == 0)
    if (lane == 0 && p.tma_mode) {
      int st = 0;
      uint32_t ph = 0;
      const uint32_t row_bytes = MODE == MODE_F16X3 ? 32 : 16;  // fp32 or bf16 chunk row
      const uint32_t col_bytes = (uint32_t)p.S_pad * row_bytes;
      const uint32_t stage_tx = (uint32_t)CH * col_bytes;
      for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
        long long mg;
        int nt;
        unit_coords(p, u, mg, nt);
        const int m0 = (int)(mg * MPG);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_empty[st], ph ^ 1);
          uint64_t* bar = MODE == MODE_F16X3 ? &a_land[st] : &a_full[st];
          mbar_arrive_expect_tx(bar, stage_tx);
          const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
          for (int j = 0; j < CH; ++j)
            for (int pc = 0; pc < p.pieces; ++pc)
              tma_load_3d(sbase + (uint32_t)j * col_bytes + (uint32_t)(pc * p.piece_rows) * row_bytes,
                          &tmap, 0, m0 + pc * p.piece_rows, kb * CH + j, bar);
          if (kb == 0) trace_ev(p, 0, (int)((u - blockIdx.x) / gridDim.x));
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int pt = threadIdx.x - 128;
    int st = 0;
    uint32_t ph = 0;
    GuardTrack gt;
    gt.init(p.fb.guard);
    if (p.tma_mode) {
      if constexpr (MODE == MODE_F16X3) {
        // ======================= converter: fp32 chunk column j (32-byte rows)
        // becomes hi column 2j + lo column 2j+1 in the same bytes.  Read all
        // of a chunk's rows first, barrier, then write (in-place hazard).
        constexpr int RPT = 8;  // rows per thread per chunk: S <= 8 * 128 = 1024
        for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&a_land[st], ph);
            const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
            for (int j = 0; j < CH; ++j) {
              const uint32_t cbase = sbase + (uint32_t)j * 2 * COL;
              float4 v[RPT][2];
#pragma unroll
              for (int k = 0; k < RPT; ++k) {
                const int s = pt + k * 128;
                if (s < p.S) {
                  ld_shared_v4f(cbase + (uint32_t)s * 32, v[k][0]);
                  ld_shared_v4f(cbase + (uint32_t)s * 32 + 16, v[k][1]);
                  gt.add(v[k][0]);
                  gt.add(v[k][1]);
                }
              }
              named_bar(1, 128);
#pragma unroll
              for (int k = 0; k < RPT; ++k) {
                const int s = pt + k * 128;
                if (s < p.S) {
                  uint32_t hi[4], lo[4];
                  split8(v[k][0], v[k][1], hi, lo);
                  st_shared_v4(cbase + (uint32_t)s * 16, hi[0], hi[1], hi[2], hi[3]);
                  st_shared_v4(cbase + COL + (uint32_t)s * 16, lo[0], lo[1], lo[2], lo[3]);
                }
              }
              named_bar(1, 128);
            }
            fence_proxy_async();  // generic-proxy SMEM writes -> visible to the tensor core
            if (kb == 0 && pt == 0) trace_ev(p, 1, (int)((u - blockIdx.x) / gridDim.x));
            mbar_arrive(&a_full[st]);
            if (++st == SA) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    } else {
      // ========================= gather (p_fused > 0): predicated global loads
      const long long img = (long long)p.VH * p.VW;
      for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
        long long mg;
        int nt;
        unit_coords(p, u, mg, nt);
        const long long m0 = mg * MPG;
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_empty[st], ph ^ 1);
          const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
          const int items = p.S * CH;
          for (int it = pt; it < items; it += 128) {
            const int s = it / CH, j = it - (it / CH) * CH;
            const long long g = m0 + s;
            const int ci = kb * p.kb + j * 8;
            bool ok = g < p.Mv && ci < p.cin;
            long long src = 0;
            if (ok) {
              const long long b = g / img;
              const int rem = (int)(g - b * img);
              const int vr = rem / p.VW, vc = rem - (rem / p.VW) * p.VW;
              const int r = vr - p.pf, c = vc - p.pf;
              ok = r >= 0 && r < p.n && c >= 0 && c < p.n;
              src = (((long long)b * p.n + r) * p.n + c) * p.cin + ci;
            }
            if constexpr (MODE == MODE_F16X3) {
              float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
              if (ok) {
                const float4* xp = reinterpret_cast<const float4*>((const float*)p.x + src);
                v0 = __ldg(xp);
                v1 = __ldg(xp + 1);
                gt.add(v0);
                gt.add(v1);
              }
              uint32_t hi[4], lo[4];
              split8(v0, v1, hi, lo);
              const uint32_t dst = sbase + (uint32_t)j * 2 * COL + (uint32_t)s * 16;
              st_shared_v4(dst, hi[0], hi[1], hi[2], hi[3]);
              st_shared_v4(dst + COL, lo[0], lo[1], lo[2], lo[3]);
            } else {
              uint4 v = make_uint4(0, 0, 0, 0);
              if (ok) v = __ldg(reinterpret_cast<const uint4*>((const __nv_bfloat16*)p.x + src));
              st_shared_v4(sbase + (uint32_t)j * COL + (uint32_t)s * 16, v.x, v.y, v.z, v.w);
            }
          }
          fence_proxy_async();
          mbar_arrive(&a_full[st]);
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
    if (gt.bad()) guard_bad = 1;
  } else if (warp == 9) {
    // =========================== B loader: weight blocks by bulk copy
    if (lane == 0) {
      if (p.b_resident) {
        // single n-tile: all nkb * taps blocks once, on barrier b_full[0]
        const uint32_t total = (uint32_t)(p.nkb * p.taps) * (uint32_t)p.b_stage_bytes;
        mbar_arrive_expect_tx(&b_full[0], total);
        for (int blk = 0; blk < p.nkb * p.taps; ++blk)
          bulk_g2s(b_base + (size_t)blk * p.b_stage_bytes, p.panels + (size_t)blk * p.b_stage_bytes,
                   p.b_stage_bytes, &b_full[0]);
      } else {
        int st = 0;
        uint32_t ph = 0;
        for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
          long long mg;
          int nt;
          unit_coords(p, u, mg, nt);
          for (int kb = 0; kb < p.nkb; ++kb) {
            const uint8_t* src =
                p.panels + ((size_t)(nt * p.nkb + kb) * p.taps) * (size_t)p.b_stage_bytes;
            for (int t = 0; t < p.taps; ++t) {
              mbar_wait(&b_empty[st], ph ^ 1);
              mbar_arrive_expect_tx(&b_full[st], p.b_stage_bytes);
              bulk_g2s(b_base + (size_t)st * p.b_stage_bytes, src + (size_t)t * p.b_stage_bytes,
                       p.b_stage_bytes, &b_full[st]);
              if (++st == SB) {
                st = 0;
                ph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 8) {
    // =========================== MMA issuer (one thread)
    if (lane == 0) {
      int sa = 0, sb = 0, acc = 0;
      uint32_t pa = 0, pb = 0, pacc = 0;
      if (p.b_resident) {
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
      }
      for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        trace_ev(p, 2, (int)((u - blockIdx.x) / gridDim.x));
        const uint32_t d_base = tmem_base + (uint32_t)(acc * ACC_COLS);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_full[sa], pa);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          for (int t = 0; t < p.taps; ++t) {
            uint32_t b_addr;
            if (p.b_resident) {
              b_addr = smem_u32(b_base + (size_t)(kb * p.taps + t) * p.b_stage_bytes);
            } else {
              mbar_wait(&b_full[sb], pb);
              tc_fence_after();
              b_addr = smem_u32(b_base + (size_t)sb * p.b_stage_bytes);
            }
            const int q = p.tap_class[t];
            const bool first = (kb == 0 && t == p.first_tap[q]);
            const uint32_t a_tap = a_addr + (uint32_t)p.tap_shift[t] * 16;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const uint32_t d = d_base + (uint32_t)((g * 4 + q) * NT);
              const uint32_t a0 = a_tap + (uint32_t)(g * BM) * 16;
              for (int ks = 0; ks < CH / 2; ++ks) {
                const uint32_t bk = b_addr + (uint32_t)ks * 2 * LBO_B;
                const uint64_t bh = sdesc(bk, LBO_B, 128);
                const uint32_t acc_flag = (first && ks == 0) ? 0u : 1u;
                if constexpr (MODE == MODE_F16X3) {
                  const uint32_t ak = a0 + (uint32_t)ks * 4 * COL;  // hi chunks 2ks, 2ks+1
                  const uint64_t ah = sdesc(ak, LBO_A, 128);
                  const uint64_t al = sdesc(ak + COL, LBO_A, 128);
                  const uint64_t bl = sdesc(bk + plane_b, LBO_B, 128);
                  mma_f16(d, ah, bh, IDESC, acc_flag);
                  mma_f16(d, al, bh, IDESC, 1u);
                  mma_f16(d, ah, bl, IDESC, 1u);
                } else {
                  const uint64_t ah = sdesc(a0 + (uint32_t)ks * 2 * COL, LBO_A, 128);
                  mma_f16(d, ah, bh, IDESC, acc_flag);
                }
              }
            }
            if (!p.b_resident) {
              mma_commit(&b_empty[sb]);
              if (++sb == SB) {
                sb = 0;
                pb ^= 1;
              }
            }
          }
          mma_commit(&a_empty[sa]);
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
        }
        mma_commit(&acc_full[acc]);
        trace_ev(p, 3, (int)((u - blockIdx.x) / gridDim.x));
        if (++acc == ACC_BUFS) {
          acc = 0;
          pacc ^= 1;
        }
      }
    }
  } else {
    // =========================== epilogue (warps 0-3; warp w owns TMEM lanes 32w..)
    int acc = 0;
    uint32_t pacc = 0;
    const long long img = (long long)p.VH * p.VW;
    constexpr int CW = NT >= 32 ? 32 : NT;
    const float wsc = MODE == MODE_F16X3 ? guard_inv_scale(p.fb.guard) : 1.0f;  // images hold w * 2^s
    float chk = 0.0f;  // range guard: NaN once a stored sum is not finite
    for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
      long long mg;
      int nt;
      unit_coords(p, u, mg, nt);
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0) trace_ev(p, 4, (int)((u - blockIdx.x) / gridDim.x));
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        const long long m = mg * MPG + g * BM + warp * 32 + lane;
        const long long b = m / img;
        const int rem = (int)(m - b * img);
        const int i = rem / p.VW, j = rem - (rem / p.VW) * p.VW;
        const uint32_t tbase =
            tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * ACC_COLS + g * 4 * NT);
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          const int r = q >> 1, c = q & 1;
          const bool valid = m < p.Mv && i < p.rows[q] && j < p.cols[q];
          const long long pix = ((long long)b * p.out_h + (2 * i + r)) * p.out_w + (2 * j + c);
#pragma unroll 1
          for (int c0 = 0; c0 < NT; c0 += CW) {
            float v[32];
            if constexpr (NT >= 32)
              tmem_ld32(tbase + (uint32_t)(q * NT + c0), v);
            else
              tmem_ld16(tbase + (uint32_t)(q * NT + c0), v);
            if (!valid) continue;
            const int f0 = nt * NT + c0;
            const bool full = f0 + CW <= p.cout;
#pragma unroll
            for (int k = 0; k < CW; ++k) {
              if (f0 + k < p.cout) guard_check(chk, v[k]);
              v[k] = epilogue_apply(v[k] * wsc, p.epi, p.bias, min(f0 + k, p.cout - 1));
            }
            if (full && p.y_dtype == SEGCONV_F32 && (p.cout & 3) == 0) {
              float4* dst = reinterpret_cast<float4*>((float*)p.y + pix * p.cout + f0);
#pragma unroll
              for (int k = 0; k < CW / 4; ++k)
                dst[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            } else if (full && p.y_dtype == SEGCONV_BF16 && (p.cout & 7) == 0) {
              uint4* dst = reinterpret_cast<uint4*>((__nv_bfloat16*)p.y + pix * p.cout + f0);
#pragma unroll
              for (int k = 0; k < CW / 8; ++k) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const __nv_bfloat162 h =
                      __floats2bfloat162_rn(v[8 * k + 2 * e], v[8 * k + 2 * e + 1]);
                  w[e] = *reinterpret_cast<const uint32_t*>(&h);
                }
                dst[k] = make_uint4(w[0], w[1], w[2], w[3]);
              }
            } else {
#pragma unroll
              for (int k = 0; k < CW; ++k)
                if (f0 + k < p.cout) store_out(p.y, pix * p.cout + f0 + k, v[k], p.y_dtype);
            }
          }
        }
      }
      tc_fence_before();
      if (threadIdx.x == 0) trace_ev(p, 5, (int)((u - blockIdx.x) / gridDim.x));
      mbar_arrive(&acc_empty[acc]);
      if (++acc == ACC_BUFS) {
        acc = 0;
        pacc ^= 1;
      }
    }
    if (MODE == MODE_F16X3 && guard_check_bad(chk)) guard_bad = 1;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
  if (MODE == MODE_F16X3 && guard_bad) {
    // x left the split-fp16 range in this CTA's halos: recompute its units
    // (anchors x feature tile) with FFMA; this CTA wrote them
    const long long img = (long long)p.VH * p.VW;
    for (long long u = blockIdx.x; u < p.total_units; u += gridDim.x) {
      long long mg;
      int nt;
      unit_coords(p, u, mg, nt);
      const long long m0 = mg * MPG;
      guard_fallback(p.fb, MPG, nt * NT, min(p.cout, (nt + 1) * NT),
                     [&](long long idx, int& b, int& i, int& j) {
                       const long long m = m0 + idx;
                       if (m >= p.Mv) return false;
                       b = (int)(m / img);
                       const int rem = (int)(m - (long long)b * img);
                       i = rem / p.VW;
                       j = rem - i * p.VW;
                       return true;
                     });
    }
  }
}

}  // namespace tc

// ------------------------------------------------------------ host plan
// Tile shape decisions shared by segregate (panel image) and the launcher.
// An SS-mode MMA (M=128, K=16) reads 4 KB of A plus 32*N bytes of B from
// SMEM at ~128 B/cycle, against N/2 cycles of tensor work, so N >= 128 is
// needed to be compute-bound (measured: scripts/mma_bench.cu).  Wide layers
// therefore use 128-feature tiles (4 classes x 128 = all 512 TMEM columns).
int tc_n_tile(int math, int cout) {
  (void)math;
  const int c16 = (cout + 15) / 16 * 16;
  return c16 >= 128 ? 128 : c16 >= 64 ? 64 : c16 >= 32 ? 32 : 16;
}
// Narrow-output layers (cout <= 16) have wide images, hence tall halos: use
// 32-channel blocks so two A stages fit.
int tc_k_block(int cin, int cout) {
  if (cout <= 16 && cin >= 32) return 32;
  return cin >= 64 ? 64 : cin >= 32 ? 32 : 16;
}

static int tc_mode(int math) { return math == SEGCONV_MATH_F16X3 ? tc::MODE_F16X3 : tc::MODE_BF16; }

struct Plan {
  tc::Params p;
  CUtensorMap tmap;
  int G;
  size_t smem;
  bool ok;
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  });
  return fn;
}

// 3-D view of the NHWC input for the halo TMA: (8 elems of a 16-byte chunk,
// pixel, chunk) with byte strides (cin * esize, 16).  Box (8, rows, 1): one
// k-chunk column piece.
static bool encode_halo_map(CUtensorMap* m, const void* x, bool f32, long long pixels, int cin,
                            int rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const int es = f32 ? 4 : 2;
  const cuuint64_t dims[3] = {8, (cuuint64_t)pixels, (cuuint64_t)(cin / 8)};
  const cuuint64_t strides[2] = {(cuuint64_t)cin * es, (cuuint64_t)8 * es};
  const cuuint32_t box[3] = {8, (cuuint32_t)rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
            const_cast<void*>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static Plan make_plan_g(const FusedProblem& pr, int math, int G) {
  Plan pl{};
  pl.G = G;
  tc::Params& p = pl.p;
  const int mode = tc_mode(math);
  const int planes = mode == tc::MODE_F16X3 ? 2 : 1;
  const int NT = tc_n_tile(math, pr.cout);
  p.kb = tc_k_block(pr.cin, pr.cout);
  p.nkb = (pr.cin + p.kb - 1) / p.kb;
  p.n_tiles = (pr.cout + NT - 1) / NT;
  p.batch = pr.batch;
  p.n = pr.n;
  p.cin = pr.cin;
  p.cout = pr.cout;
  p.pf = pr.pf;
  p.VH = p.VW = pr.n + 2 * pr.pf;
  p.Mv = (long long)pr.batch * p.VH * p.VW;
  p.out_h = pr.out_h;
  p.out_w = pr.out_w;
  const long long MPG = (long long)G * tc::BM;
  p.m_groups = (p.Mv + MPG - 1) / MPG;
  p.total_units = p.m_groups * p.n_tiles;
  p.x = pr.x;
  p.panels = (const uint8_t*)pr.panels;
  p.y = pr.y;
  p.y_dtype = pr.y_dtype;
  p.bias = pr.bias;
  p.epi = pr.epi;
  p.fb = make_fallback_args(pr, mode == tc::MODE_F16X3 ? pr.guard : nullptr);
  if (mode == tc::MODE_F16X3 && !pr.guard) return pl;
  int t = 0, max_shift = 0;
  for (int q = 0; q < 4; ++q) {
    p.first_tap[q] = t;
    p.rows[q] = pr.cls.rows[q];
    p.cols[q] = pr.cls.cols[q];
    for (int u = 0; u < pr.cls.kh[q]; ++u)
      for (int v = 0; v < pr.cls.kw[q]; ++v) {
        if (t >= tc::MAX_TAPS) return pl;
        p.tap_class[t] = q;
        p.tap_shift[t] = (pr.cls.off_r[q] + u) * p.VW + (pr.cls.off_c[q] + v);
        max_shift = std::max(max_shift, p.tap_shift[t]);
        ++t;
      }
  }
  p.taps = t;
  p.S = (int)MPG + max_shift;
  const int CH = p.kb / 8;
  // TMA halo when the virtual grid is the input itself (p_fused == 0) and the
  // channel blocks tile cin exactly; boxes of <= 256 rows per k-chunk column.
  // The in-place fp16 split keeps <= 8 rows per converter thread (S <= 1024).
  p.tma_mode = (pr.pf == 0 && pr.cin % p.kb == 0 &&
                (mode == tc::MODE_BF16 || p.S <= 8 * 128)) ? 1 : 0;
  if (p.tma_mode) {
    p.pieces = (p.S + 255) / 256;
    p.piece_rows = ((p.S + p.pieces - 1) / p.pieces + 7) / 8 * 8;
    p.S_pad = p.pieces * p.piece_rows;
    if (p.pieces > tc::MAX_PIECES ||
        !encode_halo_map(&pl.tmap, pr.x, mode == tc::MODE_F16X3,
                         (long long)pr.batch * pr.n * pr.n, pr.cin, p.piece_rows))
      p.tma_mode = 0;
  }
  if (!p.tma_mode) {
    p.pieces = p.piece_rows = 0;
    p.S_pad = p.S | 1;  // odd: a pixel's 8 k-chunk columns hit distinct banks
  }
  p.a_stage_bytes = planes * CH * p.S_pad * 16;  // == CH * S_pad * 32 for the fp32 landing
  p.a_stage_bytes = (p.a_stage_bytes + 1023) / 1024 * 1024;
  p.b_stage_bytes = planes * p.kb * NT * 2;
  // mbarriers: 3 per A stage, 2 per streamed B stage (<= 12), 4 accumulator, TMEM slot
  const int bar_bytes = (3 * 4 + 2 * 12 + 4) * 8 + 16;
  const int budget = tc::SMEM_LIMIT - bar_bytes;
  const int b_all = p.nkb * p.taps * p.b_stage_bytes;
  // weights resident when there is one n-tile and they fit beside 2 A stages
  p.b_resident = (p.n_tiles == 1 && b_all + 2 * p.a_stage_bytes <= budget) ? 1 : 0;
  if (p.b_resident) {
    p.stages_b = p.nkb * p.taps;
    p.stages_a = std::min(4, (budget - b_all) / p.a_stage_bytes);
  } else {
    p.stages_a = 2;
    if (2 * p.a_stage_bytes + 2 * p.b_stage_bytes > budget) p.stages_a = 1;
    p.stages_b = std::min(12, (budget - p.stages_a * p.a_stage_bytes) / p.b_stage_bytes);
    if (p.stages_b < 2) return pl;
  }
  if (p.stages_a < 1) return pl;
  pl.smem = (size_t)p.stages_a * p.a_stage_bytes + (size_t)p.stages_b * p.b_stage_bytes + bar_bytes;
  pl.ok = true;
  return pl;
}

// Pick the m-group size G: TMEM holds G*4*NT accumulator columns (<= 512);
// a larger G reuses each streamed weight block across more anchors, a smaller
// G gives more work units.  With resident weights G buys nothing: use 1.
static Plan make_plan(const FusedProblem& pr, int math) {
  const int NT = tc_n_tile(math, pr.cout);
  const long long Mv = (long long)pr.batch * (pr.n + 2 * pr.pf) * (pr.n + 2 * pr.pf);
  const int n_tiles = (pr.cout + NT - 1) / NT;
  {
    Plan pl = make_plan_g(pr, math, 1);
    if (pl.ok && pl.p.b_resident) return pl;
  }
  for (int G : {4, 2, 1}) {
    if (G * 4 * NT > 512) continue;
    const long long units = (Mv + G * tc::BM - 1) / (G * tc::BM) * n_tiles;
    if (G > 1 && units < 148) continue;
    Plan pl = make_plan_g(pr, math, G);
    if (!pl.ok) continue;
    if (G > 1 && pl.p.b_resident) continue;
    return pl;
  }
  return Plan{};
}

bool tc_igemm_available(int math, int cin, int cout) {
  (void)cout;
  if (math != SEGCONV_MATH_BF16 && math != SEGCONV_MATH_F16X3) return false;
  return cin % 8 == 0 && cin >= 8;
}

bool tc_igemm_supported(const FusedProblem& pr, int math) {
  if (!tc_igemm_available(math, pr.cin, pr.cout)) return false;
  if (pr.panel_layout != SEGCONV_PANEL_UMMA) return false;
  if (math == SEGCONV_MATH_BF16 &&
      (pr.x_dtype != SEGCONV_BF16 || pr.panel_dtype != SEGCONV_BF16))
    return false;
  if (math == SEGCONV_MATH_F16X3 &&
      (pr.x_dtype != SEGCONV_F32 || pr.panel_dtype != SEGCONV_F16_SPLIT))
    return false;
  for (int q = 0; q < 4; ++q)
    if (pr.cls.kh[q] == 0 || pr.cls.kw[q] == 0) return false;  // every class must have taps
  return make_plan(pr, math).ok;
}

// SEGCONV_TC_TRACE=1: a device buffer of 160 CTAs x 16 events x 64 units of
// globaltimer stamps, readable through segconv_debug_trace() (diagnostics only).
// SEGCONV_TC_TRACE=2: eight such slots, one per launch in turn (a stack's
// layers, each captured into its graph with its own slot).
static unsigned long long* g_trace = nullptr;
static int g_trace_slots = 0, g_trace_next = 0;
constexpr size_t kTraceSlot = 160 * 16 * 64;
unsigned long long* tc_trace_buffer() {
  static bool init = false;
  if (!init) {
    init = true;
    const char* e = getenv("SEGCONV_TC_TRACE");
    const int slots = (e && e[0] == '1') ? 1 : (e && e[0] == '2') ? 8 : 0;
    if (slots && cudaMalloc(&g_trace, slots * kTraceSlot * sizeof(unsigned long long)) == cudaSuccess) {
      cudaMemset(g_trace, 0, slots * kTraceSlot * sizeof(unsigned long long));
      g_trace_slots = slots;
    }
  }
  if (!g_trace) return nullptr;
  unsigned long long* t = g_trace + (size_t)(g_trace_next % g_trace_slots) * kTraceSlot;
  if (g_trace_slots > 1) ++g_trace_next;
  return t;
}
size_t tc_trace_bytes() { return (size_t)g_trace_slots * kTraceSlot * sizeof(unsigned long long); }
const unsigned long long* tc_trace_ptr() { return g_trace; }

template <int MODE, int NT, int G>
static cudaError_t launch_t(const Plan& pl, cudaStream_t s) {
  auto kern = tc::tc_halo_kernel<MODE, NT, G>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, tc::SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  const long long grid = std::min<long long>(pl.p.total_units, sms);
  tc::Params prm = pl.p;
  prm.trace = tc_trace_buffer();
  kern<<<(unsigned)grid, tc::NUM_THREADS, pl.smem, s>>>(prm, pl.tmap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tc_igemm(const FusedProblem& pr, int math, cudaStream_t s) {
  const Plan pl = make_plan(pr, math);
  if (!pl.ok) return cudaErrorNotSupported;
  if (pl.p.total_units == 0) return cudaSuccess;
  const int NT = tc_n_tile(math, pr.cout);
  const int mode = tc_mode(math);
#define TCL(M, N, GG) \
  if (mode == M && NT == N && pl.G == GG) return launch_t<M, N, GG>(pl, s);
#define TCL_G(M, N) TCL(M, N, 1) TCL(M, N, 2) TCL(M, N, 4)
  TCL_G(tc::MODE_BF16, 16)
  TCL_G(tc::MODE_BF16, 32)
  TCL(tc::MODE_BF16, 64, 1)
  TCL(tc::MODE_BF16, 64, 2)
  TCL(tc::MODE_BF16, 128, 1)
  TCL_G(tc::MODE_F16X3, 16)
  TCL_G(tc::MODE_F16X3, 32)
  TCL(tc::MODE_F16X3, 64, 1)
  TCL(tc::MODE_F16X3, 64, 2)
  TCL(tc::MODE_F16X3, 128, 1)
#undef TCL_G
#undef TCL
  return cudaErrorNotSupported;
}

}  // namespace segconv_b200

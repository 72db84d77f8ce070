// tc_fold_ts.cu -- K3 for the fp32 multi-channel layer (BASELINE C2 shape:
// cout in (16, 32], split-fp16 math): the class-folded tcgen05 GEMM of
// tc_fold.cu re-balanced for shared-memory bandwidth.
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for these layers.  Same algebra as
// tc_fold.cu: D[(q, f), m] = sum_s W_s[(q, f), :] . X[m + shift_s, :], four
// classes x 32 features on the 128 MMA rows, anchors on N.
//
// Why a separate kernel.  At N = 128 a tcgen05.mma with both operands in
// SMEM reads 8 KB per 64 cycles -- all of the SM's 128 B/cycle of shared
// memory -- so every byte the halo staging and the epilogue move through SMEM
// slows the tensor core (measured: the SS kernel spent ~3x the MMA time per
// unit).  Here:
//   * the weights are the MMA A operand in TMEM (the "ts" form; layout checked
//     by scripts/tmem_a_test.cu), so MMAs read only the 4 KB halo tile;
//   * the fp32 halo lands by TMA as 128-byte rows (32 channels) with the
//     128-byte swizzle, so the converter warps read it without bank conflicts,
//     and is split in place into fp16 hi/lo planes in the UMMA K-major
//     no-swizzle layout;
//   * the epilogue stores straight from the TMEM registers: lane = feature,
//     so each st.global of a warp writes one output pixel's 32 features as one
//     128-byte line (addresses computed once per 32 anchors and broadcast by
//     shuffle) -- no SMEM transpose.
// SMEM traffic per unit is then the 4 KB-per-MMA operand reads plus one TMA
// write, one read and one write of the halo.
//
// Schedule: each CTA owns one contiguous range of anchors (virtual positions
// of the NHWC input, 16-position granules) cut into units of <= 128 anchors;
// a stage is 32 channels of a unit's halo (rows [m0, m0 + nu + max_shift));
// eight stages ring through SMEM; D is double-buffered in TMEM columns
// [0, 256) and the weights occupy [256, 512).  The weight image is staged
// once through the top stages and copied into TMEM by the epilogue warps.
//
// Warp roles (448 threads): 0-7 epilogue (warps w, w+4 <-> TMEM lane
// quadrant w = parity class w, alternate 32-anchor blocks), 8-11 converters,
// 12 MMA issuer, 13 TMA producer / TMEM owner.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_guard.cuh"

namespace segconv_b200 {
namespace tcfs {

using namespace tc;

constexpr int NUM_THREADS = 448;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int MAX_SHIFTS = 16;
constexpr int STAGES = 8;
constexpr int KB = 32;   // channels per stage: one 128-byte TMA row
constexpr int CH = KB / 8;
constexpr int A_COL = 256;  // first TMEM column of the weights
constexpr int RPT = 2;      // converter rows per thread (S_pad <= RPT * 128)

struct Params {
  void* y;
  const float* bias;
  unsigned epi;
  int batch, n, cin, cout;
  int out_h, out_w;
  int nkb_img, kb_img;  // channel blocking of the panel image
  long long Mv;         // batch * n * n virtual positions
  int S_pad;            // rows per k-chunk column of a stage (= TMA box rows)
  int stage_bytes, w_img_bytes, w_stage0;
  int nblk;              // non-zero (shift, class) blocks of the compact weight image
  int blk_of[MAX_SHIFTS][4];  // block index of (shift, class), -1: no tap (zeros)
  int shifts, max_shift;
  int shift_off[MAX_SHIFTS];
  int rows[4], cols[4];
  const uint8_t* panels;  // UMMA_FOLD image, split planes
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

// Unit k of this CTA: anchors [m0, m0 + nu) of its contiguous range.
__device__ __forceinline__ bool next_unit(const Params& p, int k, long long& m0, int& nu) {
  const long long g16 = (p.Mv + 15) / 16;
  const long long s16 = g16 * blockIdx.x / gridDim.x, e16 = g16 * (blockIdx.x + 1) / gridDim.x;
  m0 = (s16 + (long long)k * 8) * 16;
  if (m0 >= e16 * 16) return false;
  nu = (int)min(128LL, e16 * 16 - m0);
  return true;
}

// The weight image lands at the top stages of every CTA.
__device__ __forceinline__ void issue_weights(const Params& p, uint8_t* smem, uint64_t* w_full) {
  mbar_arrive_expect_tx(w_full, (uint32_t)p.w_img_bytes);
  uint8_t* dst = smem + (size_t)p.w_stage0 * p.stage_bytes;
  constexpr uint32_t CHUNK = 32768;
  for (uint32_t off = 0; off < (uint32_t)p.w_img_bytes; off += CHUNK)
    bulk_g2s(dst + off, p.panels + off, min(CHUNK, (uint32_t)p.w_img_bytes - off), w_full);
}

template <int ACT>
__device__ __forceinline__ float finish(float v, float bias) {
  v += bias;
  if (ACT == 1) v = fmaxf(v, 0.0f);
  if (ACT == 2) v = tanhf(v);
  return v;
}

// Predicated global store (no branch, so the 32 stores of a block issue back to back).
__device__ __forceinline__ void st_global_pred(float* ptr, float v, bool pred) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\n@p st.global.f32 [%0], %1;\n}\n" ::"l"(ptr),
               "f"(v), "r"((int)pred)
               : "memory");
}
__device__ __forceinline__ void st_global_pred(__nv_bfloat16* ptr, float v, bool pred) {
  const unsigned short h = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\n@p st.global.b16 [%0], %1;\n}\n" ::"l"(ptr),
               "h"(h), "r"((int)pred)
               : "memory");
}

template <typename YT, int ACT, int SHIFTS>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    fold_ts_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * p.stage_bytes);
  uint64_t* a_land = bars;              // TMA -> converters
  uint64_t* a_full = a_land + STAGES;   // converters -> MMA
  uint64_t* a_empty = a_full + STAGES;  // MMA -> TMA
  uint64_t* acc_full = a_empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;  // weight image landed in SMEM
  uint64_t* w_free = w_full + 1;     // weights copied into TMEM, staging area free
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_free + 1);
  // a converter saw x outside the split's range (the word after the TMEM slot)
  volatile int& guard_bad = *reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    guard_bad = 0;
    trace_ev(p, 9, 0);  // kernel entry
    if (p.trace && blockIdx.x < 160) p.trace[(blockIdx.x * 16 + 12) * 64] = clock64();
  }
  if (warp == 12 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&a_land[s], 1);
      mbar_init(&a_full[s], 128);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 256);
    }
    mbar_init(w_full, 1);
    mbar_init(w_free, 256);
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
  if (threadIdx.x == 0) trace_ev(p, 10, 0);  // prologue done
  // launched with programmatic stream serialization: the barrier init, TMEM
  // allocation and tensormap prefetch above overlap the previous kernel's tail;
  // every global access (weights, halo loads, stores, guard fallback) follows
  // this wait, so what the previous kernel wrote (the weight image of a
  // just-segregated kernel, x) is visible and nothing it still reads is overwritten.
  griddep_wait();

  const int NKB = p.cin / KB;                   // stages per unit
  const int KS = p.cin / 16;                    // K=16 steps over cin
  const uint32_t COL = (uint32_t)p.S_pad * 16;  // one k-chunk column (one plane)
  const uint32_t w_stage_addr = smem_u32(smem) + (uint32_t)p.w_stage0 * p.stage_bytes;

  if (warp == 13) {
    // ===== TMA producer: weight image once (into the top stages), then halo
    // boxes {32 channels, S_pad rows} with the 128-byte swizzle
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      bool freed = false, weights_issued = false;
      const uint32_t tx = (uint32_t)p.S_pad * KB * 4;
      long long m0;
      int nu;
      for (int k = 0; next_unit(p, k, m0, nu); ++k) {
        for (int h = 0; h < NKB; ++h) {
          if (!weights_issued) {
            // the (compact) weight image is queued first: no MMA can start before it
            weights_issued = true;
            issue_weights(p, smem, w_full);
          }
          if (!freed && st >= p.w_stage0) {
            mbar_wait(w_free, 0);
            freed = true;
          }
          mbar_wait(&a_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&a_land[st], tx);
          tma_load_2d(smem_u32(smem + (size_t)st * p.stage_bytes), &tmap, h * KB, (int)m0,
                      &a_land[st]);
          if (h == 0) trace_ev(p, 0, k);
          if (++st == STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
      if (!weights_issued) {  // fewer stages of work than w_stage0
        issue_weights(p, smem, w_full);
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ===== converters: swizzled fp32 rows -> fp16 hi/lo k-chunk columns, in place
    // Thread t owns rows t, t+128, ... of every k-chunk; all reads of a stage
    // happen before the named barrier, then the writes (in-place hazard).
    const int ct = threadIdx.x - 256;
    int st = 0;
    uint32_t ph = 0;
    long long m0;
    int nu;
    GuardTrack gt;
    gt.init(p.fb.guard);
    for (int k = 0; next_unit(p, k, m0, nu); ++k) {
      const int rows_live = min(p.S_pad, nu + p.max_shift);
      for (int h = 0; h < NKB; ++h) {
        mbar_wait(&a_land[st], ph);
        const uint32_t sbase = smem_u32(smem + (size_t)st * p.stage_bytes);
        if (!(p.debug & 2)) {
          float4 v[RPT][CH][2];
#pragma unroll
          for (int t = 0; t < RPT; ++t) {
            const int r = ct + t * 128;
            if (r < rows_live) {
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
          for (int t = 0; t < RPT; ++t) {
            const int r = ct + t * 128;
            if (r < rows_live) {
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                uint32_t hi[4], lo[4];
                split8x2(v[t][j][0], v[t][j][1], hi, lo);
                gt.add_hi(hi);  // range guard: fp16 overflow shows as an inf hi half
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
        if (++st == STAGES) {
          st = 0;
          ph ^= 1;
        }
      }
    }
    if (gt.bad()) guard_bad = 1;
  } else if (warp == 12) {
    // ===== MMA issuer (the whole warp runs the loop; one elected lane issues)
    {
      const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t a_tm = tb + A_COL;
      int st = 0, acc = 0;
      uint32_t ph = 0, pacc = 0;
      long long m0;
      int nu;
      mbar_wait(w_free, 0);
      tc_fence_after();
      for (int k = 0; next_unit(p, k, m0, nu); ++k) {
        const uint32_t idesc = idesc_f16(0, nu);
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        if (lane == 0) trace_ev(p, 2, k);
        const uint32_t d = tb + (uint32_t)(acc * 128);
        for (int h = 0; h < NKB; ++h) {
          if (!(p.debug & 16)) mbar_wait(&a_full[st], ph);  // 16: diagnostics, MMAs on stale data
          tc_fence_after();
          const uint32_t xb = smem_u32(smem) + (uint32_t)st * (uint32_t)p.stage_bytes;
          if (!(p.debug & 8)) {
            // One elected lane issues the stage's shifts x k-steps x 3 MMAs as
            // straight-line code: descriptor low words are the stage base plus
            // constant 16-byte offsets (no carry: SMEM addresses < 256 KB).
            const uint32_t lo0 = ((xb >> 4) & 0x3FFFu) | (((2 * COL) >> 4) << 16);
            const uint32_t hi = (128u >> 4) | (1u << 14);  // SBO = 128 B, sm_100 version bit
            const uint32_t col16 = COL >> 4;
            if (elect_one()) {
#pragma unroll
              for (int s = 0; s < SHIFTS; ++s) {
                const uint32_t so = (uint32_t)p.shift_off[s];
#pragma unroll
                for (int ks = 0; ks < CH / 2; ++ks) {
                  // hi chunks 2ks, 2ks+1 in columns 4ks, 4ks+2; lo one column right
                  const uint32_t xk = lo0 + so + (uint32_t)ks * 4 * col16;
                  const uint64_t xh = ((uint64_t)hi << 32) | xk;
                  const uint64_t xl = ((uint64_t)hi << 32) | (xk + col16);
                  const int ksg = h * (CH / 2) + ks;
                  const uint32_t wh = a_tm + (uint32_t)((s * 2 * KS + ksg) * 8);
                  const uint32_t wl = wh + (uint32_t)(KS * 8);
                  mma_f16_ts(d, wh, xh, idesc, (h == 0 && s == 0 && ks == 0) ? 0u : 1u);
                  mma_f16_ts(d, wl, xh, idesc, 1u);
                  mma_f16_ts(d, wh, xl, idesc, 1u);
                }
              }
            }
            __syncwarp();
          }
          if (elect_one()) mma_commit(&a_empty[st]);
          __syncwarp();
          if (++st == STAGES) {
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
    }
  } else {
    // ===== epilogue (warps 0-7): lane = feature f of class q = warp % 4
    const int q = warp & 3, half = warp >> 2, r = q >> 1, c = q & 1, f = lane;
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
    {
      // weights: staged compact image [plane][k-chunk][block][32 rows][16 B]
      // (only the (shift, class) blocks that hold taps) -> TMEM columns
      // ((shift * 2 + plane) * KS + ks) * 8 of this thread's row, zeros for
      // the classes a shift does not touch; the quadrant's two warps take one
      // plane each
      mbar_wait(w_full, 0);
      if (threadIdx.x == 0) trace_ev(p, 6, 0);
      const int pl = half, CHT = p.cin / 8;
      for (int s = 0; s < p.shifts; ++s) {
        const int blk = p.blk_of[s][q];
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t rr[8];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int J = 2 * ks + hh;
            if (blk >= 0) {
              const uint32_t src = w_stage_addr +
                                   (((uint32_t)(pl * CHT + J) * p.nblk + blk) * 32 + lane) * 16;
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(rr[4 * hh]), "=r"(rr[4 * hh + 1]), "=r"(rr[4 * hh + 2]),
                             "=r"(rr[4 * hh + 3])
                           : "r"(src));
            } else {
              rr[4 * hh] = rr[4 * hh + 1] = rr[4 * hh + 2] = rr[4 * hh + 3] = 0u;
            }
          }
          tmem_st8(lane_base + A_COL + (uint32_t)(((s * 2 + pl) * KS + ks) * 8), rr);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(w_free);
      if (threadIdx.x == 0) trace_ev(p, 7, 0);
    }
    const bool f_ok = f < p.cout;
    const float bias = (f_ok && (p.epi & SEGCONV_EPI_BIAS)) ? __ldg(p.bias + f) : 0.0f;
    const float wsc = guard_inv_scale(p.fb.guard);  // the weight image holds w * 2^s
    YT* __restrict__ y = reinterpret_cast<YT*>(p.y);
    const int img = p.n * p.n;
    const int qrows = p.rows[q], qcols = p.cols[q];
    int acc = 0;
    uint32_t pacc = 0;
    long long m0;
    int nu;
    for (int k = 0; next_unit(p, k, m0, nu); ++k) {
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0) trace_ev(p, 4, k);
#pragma unroll 1
      for (int c0 = 32 * half; c0 < nu; c0 += 64) {
        float v[32];
        tmem_ld32(lane_base + (uint32_t)(acc * 128 + c0), v);
        // lane t decodes anchor c0 + t once; the stores broadcast it
        const long long m = m0 + c0 + lane;
        const int b = (int)(m / img);
        const int rem = (int)(m - (long long)b * img);
        const int i = rem / p.n, j = rem - (rem / p.n) * p.n;
        const bool ok = c0 + lane < nu && b < p.batch && i < qrows && j < qcols;
        const int pix = ok ? ((b * p.out_h + 2 * i + r) * p.out_w + 2 * j + c) : -1;
        if (!(p.debug & 4)) {
          // all shuffles first, then 32 independent predicated stores
          int po[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) po[t] = __shfl_sync(0xffffffffu, pix, t);
          const bool st_ok = f_ok && !(p.debug & 1);
#pragma unroll
          for (int t = 0; t < 32; ++t)
            st_global_pred(y + (long long)po[t] * p.cout + f, finish<ACT>(v[t] * wsc, bias),
                           st_ok && po[t] >= 0);
        }
      }
      tc_fence_before();
      if (threadIdx.x == 0) trace_ev(p, 5, k);
      mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        pacc ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    trace_ev(p, 11, 0);  // all roles done
    if (p.trace && blockIdx.x < 160) p.trace[(blockIdx.x * 16 + 13) * 64] = clock64();
  }
  if (warp == 13) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
  if (guard_bad) {
    // x left the split-fp16 range in this CTA's halo: recompute its anchors
    // [s16 * 16, e16 * 16) with FFMA (this CTA wrote them; the barrier above
    // orders the rewrite)
    const long long g16 = (p.Mv + 15) / 16;
    const long long a0 = g16 * blockIdx.x / gridDim.x * 16;
    const long long a1 = min(p.Mv, g16 * (blockIdx.x + 1) / gridDim.x * 16);
    const int img = p.n * p.n;
    guard_fallback(p.fb, a1 - a0, 0, p.cout, [&](long long idx, int& b, int& i, int& j) {
      const long long m = a0 + idx;
      b = (int)(m / img);
      const int rem = (int)(m - (long long)b * img);
      i = rem / p.n;
      j = rem - i * p.n;
      return true;
    });
  }
}

}  // namespace tcfs

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFnTS)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFnTS encode_fn_ts() {
  // magic static: thread-safe one-time lookup of the driver entry point
  static const EncodeTiledFnTS fn = [] {
    EncodeTiledFnTS fn = nullptr;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFnTS)f;
    return fn;
  }();
  return fn;
}

// (shift, class) blocks of the compact weight image, shift-major.
static int fold_ts_blocks(const SegClasses& cls, int ur, int uc, int (*blk_of)[4]) {
  int nb = 0;
  for (int dy = 0; dy < ur; ++dy)
    for (int dx = 0; dx < uc; ++dx)
      for (int q = 0; q < 4; ++q) {
        const int u = dy - cls.off_r[q], v = dx - cls.off_c[q];
        const bool tap = u >= 0 && u < cls.kh[q] && v >= 0 && v < cls.kw[q];
        if (blk_of) blk_of[dy * uc + dx][q] = tap ? nb : -1;
        nb += tap ? 1 : 0;
      }
  return nb;
}
size_t fold_ts_image_bytes(int cin, int nblk) { return (size_t)2 * (cin / 8) * nblk * 32 * 16; }

// Compact image: [plane hi/lo][k-chunk][block (shift, class)][32 rows f][8 fp16].
__global__ void fold_ts_image_kernel(const float* __restrict__ k, int kw, int cin, int cout,
                                     SegClasses cls, int ur, int uc, uint16_t* __restrict__ out,
                                     long long total, const SplitGuard* __restrict__ guard) {
  const float wscale = ldexpf(1.0f, split_scale_exp(guard->amax_bits));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(e % 32);
    const long long t = e / 32;
    // decode (chunk, block): total = CHT * nblk * 32, blocks enumerated on the fly
    int nb = 0;
    for (int dy = 0; dy < ur; ++dy)
      for (int dx = 0; dx < uc; ++dx)
        for (int q = 0; q < 4; ++q) {
          const int u = dy - cls.off_r[q], v = dx - cls.off_c[q];
          if (u >= 0 && u < cls.kh[q] && v >= 0 && v < cls.kw[q]) ++nb;
        }
    const int blk = (int)(t % nb);
    const int J = (int)(t / nb);
    int b = 0, qq = 0, uu = 0, vv = 0;
    for (int dy = 0; dy < ur; ++dy)
      for (int dx = 0; dx < uc; ++dx)
        for (int q = 0; q < 4; ++q) {
          const int u = dy - cls.off_r[q], v = dx - cls.off_c[q];
          if (u >= 0 && u < cls.kh[q] && v >= 0 && v < cls.kw[q]) {
            if (b == blk) {
              qq = q;
              uu = u;
              vv = v;
            }
            ++b;
          }
        }
    uint16_t hi[8], lo[8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int ci = J * 8 + x;
      float w = 0.0f;
      if (f < cout)
        w = wscale * k[(((long long)(cls.u0[qq] + 2 * uu) * kw + (cls.v0[qq] + 2 * vv)) * cin + ci) * cout + f];
      const __half h = __float2half_rn(w);
      hi[x] = __half_as_ushort(h);
      lo[x] = __half_as_ushort(__float2half_rn(w - __half2float(h)));
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      out[e * 8 + x] = hi[x];
      out[total * 8 + e * 8 + x] = lo[x];
    }
  }
}

cudaError_t launch_fold_ts_image(const void* k, int k_dtype, int kh, int kw, int cin, int cout,
                                 int p_orig, const SegClasses& cls, void* out, const void* guard,
                                 cudaStream_t s) {
  if (k_dtype != SEGCONV_F32 || !guard) return cudaErrorNotSupported;
  int ur, uc;
  fold_window(kh, kw, p_orig, &ur, &uc);
  const int nb = fold_ts_blocks(cls, ur, uc, nullptr);
  const long long total = (long long)(cin / 8) * nb * 32;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 1024);
  fold_ts_image_kernel<<<blocks, 256, 0, s>>>((const float*)k, kw, cin, cout, cls, ur, uc,
                                               (uint16_t*)out, total, (const SplitGuard*)guard);
  note_launch();
  return cudaGetLastError();
}

// Whether split-fp16 folded panels of this shape carry the compact image.
bool fold_ts_panels_apply(int kh, int kw, int cin, int cout, int p_orig, int panel_dtype) {
  if (panel_dtype != SEGCONV_F16_SPLIT || fold_cp(cout) != 32 || p_orig / 2 != 0) return false;
  if (cin % 32 != 0) return false;
  int ur, uc;
  fold_window(kh, kw, p_orig, &ur, &uc);
  return ur * uc == 4 && ur * uc * cin <= 256;
}
size_t fold_ts_image_bytes_for(int kh, int kw, int cin, int p_orig) {
  // block count from the parity geometry alone (mirrors segconv_subkernels_init)
  SegClasses c{};
  for (int q = 0; q < 4; ++q) {
    const int r = q >> 1, cc = q & 1;
    const int u0 = (p_orig + r) & 1, v0 = (p_orig + cc) & 1;
    c.kh[q] = u0 >= kh ? 0 : (kh - u0 + 1) / 2;
    c.kw[q] = v0 >= kw ? 0 : (kw - v0 + 1) / 2;
    c.off_r[q] = (r + u0 - p_orig) / 2 + p_orig / 2;
    c.off_c[q] = (cc + v0 - p_orig) / 2 + p_orig / 2;
  }
  int ur, uc;
  fold_window(kh, kw, p_orig, &ur, &uc);
  return fold_ts_image_bytes(cin, fold_ts_blocks(c, ur, uc, nullptr));
}

static bool make_fold_ts_params(const FusedProblem& pr, tcfs::Params& p) {
  p = tcfs::Params{};
  if (pr.pf != 0 || pr.x_dtype != SEGCONV_F32 || pr.panel_dtype != SEGCONV_F16_SPLIT) return false;
  if (pr.y_dtype != SEGCONV_F32 && pr.y_dtype != SEGCONV_BF16) return false;
  if (fold_cp(pr.cout) != 32) return false;  // four classes x 32 features fill the 128 MMA rows
  if (pr.cin % tcfs::KB != 0) return false;
  int ur, uc;
  fold_window(pr.kh, pr.kw, pr.p, &ur, &uc);
  p.shifts = ur * uc;
  if (p.shifts != 4 || p.shifts * pr.cin > 256) return false;  // 2x2 window; weights: 256 TMEM cols
  p.panels = (const uint8_t*)pr.panels;
  p.y = pr.y;
  p.bias = pr.bias;
  p.epi = pr.epi;
  p.batch = pr.batch;
  p.n = pr.n;
  p.cin = pr.cin;
  p.cout = pr.cout;
  p.out_h = pr.out_h;
  p.out_w = pr.out_w;
  if ((long long)pr.batch * pr.out_h * pr.out_w >= (1LL << 31)) return false;  // int pixel index
  p.kb_img = fold_kb(SEGCONV_MATH_F16X3, pr.cin);
  p.nkb_img = pr.cin / p.kb_img;
  p.Mv = (long long)pr.batch * pr.n * pr.n;
  for (int dy = 0; dy < ur; ++dy)
    for (int dx = 0; dx < uc; ++dx) p.shift_off[dy * uc + dx] = dy * pr.n + dx;
  p.max_shift = (ur - 1) * pr.n + (uc - 1);
  p.S_pad = (128 + p.max_shift + 7) / 8 * 8;
  if (p.S_pad > 256 || p.S_pad > tcfs::RPT * 128) return false;  // one TMA box, converter rows
  p.stage_bytes = tcfs::KB * 4 * p.S_pad;  // == CH * 2 planes * S_pad * 16 after the split
  p.stage_bytes = (p.stage_bytes + 1023) / 1024 * 1024;
  p.nblk = fold_ts_blocks(pr.cls, ur, uc, p.blk_of);
  p.w_img_bytes = (int)fold_ts_image_bytes(pr.cin, p.nblk);
  const int stage_area = tcfs::STAGES * p.stage_bytes;
  if (p.w_img_bytes > stage_area) return false;
  p.w_stage0 = (stage_area - p.w_img_bytes) / p.stage_bytes;  // first stage the staging covers
  // the staging starts inside stage w_stage0; keep it 16-byte aligned at its start
  if (p.w_stage0 < 1) return false;
  for (int q = 0; q < 4; ++q) {
    p.rows[q] = pr.cls.rows[q];
    p.cols[q] = pr.cls.cols[q];
  }
  const int bar_bytes = (3 * tcfs::STAGES + 6) * 8 + 16;
  if (stage_area + bar_bytes > tcfs::SMEM_LIMIT) return false;
  return true;
}

bool tc_fold_ts_supported(const FusedProblem& pr, int math) {
  if (math != SEGCONV_MATH_F16X3 || pr.panel_layout != SEGCONV_PANEL_UMMA_FOLD || !pr.guard) return false;
  tcfs::Params p;
  return make_fold_ts_params(pr, p) && encode_fn_ts() != nullptr;
}

template <typename YT, int ACT>
static cudaError_t launch_fold_ts_t(const tcfs::Params& prm, const CUtensorMap& tmap,
                                    cudaStream_t s) {
  // the MMA issue is unrolled over the union window; n = 3 (4 shifts) is the
  // instantiated shape (make_fold_ts_params admits only it)
  auto kern = tcfs::fold_ts_kernel<YT, ACT, 4>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, tcfs::SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  const long long units = (prm.Mv + 127) / 128;
  long long grid = std::min<long long>(units, sms);
  const size_t smem = (size_t)tcfs::STAGES * prm.stage_bytes + (3 * tcfs::STAGES + 6) * 8 + 16;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(tcfs::NUM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // prologue overlaps the
  at[0].val.programmaticStreamSerializationAllowed = 1;              // previous kernel's tail
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm, tmap);
  if (e == cudaSuccess) note_launch();
  return e;
}

cudaError_t launch_tc_fold_ts(const FusedProblem& pr, const void* img, cudaStream_t s) {
  tcfs::Params p;
  if (!make_fold_ts_params(pr, p)) return cudaErrorNotSupported;
  p.panels = (const uint8_t*)img;  // the compact image appended to the folded panels
  p.fb = make_fallback_args(pr, pr.guard);
  if (p.Mv == 0) return cudaSuccess;
  EncodeTiledFnTS fn = encode_fn_ts();
  if (!fn) return cudaErrorNotSupported;
  // halo view: (cin, Mv) fp32, box {32 channels, S_pad rows}, 128-byte swizzle
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)pr.cin, (cuuint64_t)p.Mv};
  const cuuint64_t strides[1] = {(cuuint64_t)pr.cin * 4};
  const cuuint32_t box[2] = {(cuuint32_t)tcfs::KB, (cuuint32_t)p.S_pad};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(pr.x), dims, strides, box,
         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  p.trace = tc_trace_buffer();
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  p.debug = dbg;
  const int act = (pr.epi & SEGCONV_EPI_RELU) ? 1 : (pr.epi & SEGCONV_EPI_TANH) ? 2 : 0;
  if (pr.y_dtype == SEGCONV_BF16) {
    if (act == 1) return launch_fold_ts_t<__nv_bfloat16, 1>(p, tmap, s);
    if (act == 2) return launch_fold_ts_t<__nv_bfloat16, 2>(p, tmap, s);
    return launch_fold_ts_t<__nv_bfloat16, 0>(p, tmap, s);
  }
  if (act == 1) return launch_fold_ts_t<float, 1>(p, tmap, s);
  if (act == 2) return launch_fold_ts_t<float, 2>(p, tmap, s);
  return launch_fold_ts_t<float, 0>(p, tmap, s);
}

}  // namespace segconv_b200

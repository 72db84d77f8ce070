// tc_fold.cu -- K3 for narrow layers (cout <= 32): the segregated transpose
// convolution as a "class-folded" tcgen05 GEMM with the operand roles swapped.
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for layers whose four parity classes x
// cout fit one 128-row MMA (BASELINE C2: 4 x 32; C4, C5d: 4 x 3).
//
// Why: an SS-mode tcgen05.mma (M=128, K=16) reads 4 KB of A plus 32*N bytes
// of B from SMEM at ~128 B/cycle against N/2 cycles of math, so the
// per-class halo-shift GEMM (tc_igemm.cu), whose N is cout, is SMEM-bound at
// small cout.  Here the weights are A and the anchors are N:
//   D[(q, f), m] += W_s[(q, f), k] * X[m + shift_s, k]
// over the union window of shifts s = (dy, dx) that any class touches
// (dy < U_r, dx < U_c); W_s holds class q's tap (dy - off_r, dx - off_c) when
// that is one of its taps, zero otherwise.  M rows are (class, feature); N is
// 128-256 anchors, which keeps every MMA compute-bound.  When 4*cout < 128
// the shifts' weight rows are packed densely and each MMA's 128-row window
// overlaps the next shift's rows -- the extra D rows are ignored.
//
// The halo (B operand) is staged as in tc_igemm.cu: k-chunk columns of S rows
// at 16 B, each shift a descriptor offset.  Two staging geometries:
//   LINEAR -- anchors are consecutive virtual positions of the NHWC input
//             (pitch = image width); one 3-D TMA box column per k-chunk;
//   BLOCK  -- for wide images: a TR x TC block of anchors staged with a
//             narrow pitch P = TC + U_c - 1 by one 4-D TMA box per k-chunk
//             (zero-filled past the image), so the halo overhead is
//             (TR + U_r - 1) / TR instead of (U_r - 1) * width / N.
// Weights live in SMEM for the whole kernel (one bulk copy).  TMEM holds the
// D tile (N fp32 columns) double- or quad-buffered across work units; the
// epilogue maps lanes to (class, feature) so each store instruction writes
// one output pixel's features contiguously, with bias / ReLU / tanh fused.
//
// Warp roles (480 threads): 0-7 epilogue (warps w and w+4 share TMEM lane
// quadrant w % 4 and split its 32-column blocks), 8-11 fp16 hi/lo converters
// (split math), 12 MMA issuer, 13 weight loader + TMEM owner, 14 halo TMA.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_guard.cuh"

namespace segconv_b200 {
namespace tcf {

using namespace tc;

constexpr int MODE_BF16 = 0, MODE_F16X3 = 1;
constexpr int NUM_THREADS = 480;  // 15 warps
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int MAX_SHIFTS = 16;
constexpr int EPI_TILE_BYTES = 8 * 32 * 36 * 4;  // one transpose tile per epilogue warp

struct Params {
  const uint8_t* panels;
  void* y;
  const float* bias;
  unsigned epi;
  int y_dtype;
  int batch, n, cin, cout, CP, R;  // CP features per class (padded), R = 4*CP rows/shift
  int out_h, out_w;
  int nkb, kb;
  int block_mode;                  // 0 LINEAR, 1 BLOCK
  int N;                           // anchors per unit (MMA N)
  int P, TR, TC, TRH;              // BLOCK geometry (pitch, anchor rows/cols, halo rows)
  int tiles_r, tiles_c;            // BLOCK: tiles per image
  long long Mv;                    // LINEAR: batch*n*n virtual positions
  long long units;
  int S, S_pad, pieces, piece_rows;
  int a_stage_bytes, w_bytes, w_rows;
  int stages_a;
  int land, stages_l, l_stage_bytes;  // LAND: fp32 halo lands by TMA in [row][kb] boxes
                                      // (128-byte rows), converters write the operand stages
  int shifts;
  int shift_off[MAX_SHIFTS];       // dy * pitch + dx
  int rows[4], cols[4];
  int a_tmem_col;                  // TMEM-A variant: first weight column (D below it)
  int w_img_bytes;                 // TMEM-A variant: bytes of the staged weight image
  unsigned long long* trace;       // optional event trace (SEGCONV_TC_TRACE)
  int debug_nostore;               // diagnostics (SEGCONV_TC_DEBUG bits): 1 skip global
                                   // stores, 2 skip the fp16 split, 4 skip epilogue body,
                                   // 8 skip the MMAs
  FallbackArgs fb;                 // split-fp16 range guard (tc_guard.cuh)
};

__device__ __forceinline__ void trace_ev(const Params& p, int ev, int local) {
  if (p.trace == nullptr || blockIdx.x >= 160 || local >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[(blockIdx.x * 16 + ev) * 64 + local] = t;
}

// Work unit k (0, 1, ...) of this CTA.  BLOCK: round-robin tiles.  LINEAR:
// each CTA owns one contiguous range of virtual positions (the grid split in
// 16-position granules, so the busiest CTA has at most one granule more than
// the average) cut into units of <= N anchors; a unit's MMA N is its length.
__device__ __forceinline__ bool next_unit(const Params& p, int k, long long& m0, int& nu, int& b,
                                          int& i0, int& j0) {
  if (!p.block_mode) {
    const long long g16 = (p.Mv + 15) / 16;
    const long long s16 = g16 * blockIdx.x / gridDim.x, e16 = g16 * (blockIdx.x + 1) / gridDim.x;
    m0 = (s16 + (long long)k * (p.N / 16)) * 16;
    if (m0 >= e16 * 16) return false;
    nu = (int)min((long long)p.N, e16 * 16 - m0);
    b = i0 = j0 = 0;
    return true;
  }
  const long long u = blockIdx.x + (long long)k * gridDim.x;
  if (u >= p.units) return false;
  const long long per = (long long)p.tiles_r * p.tiles_c;
  b = (int)(u / per);
  const int t = (int)(u - (long long)b * per);
  i0 = (t / p.tiles_c) * p.TR;
  j0 = (t % p.tiles_c) * p.TC;
  m0 = 0;
  nu = p.N;
  return true;
}

// Position of the current D column (anchor) while walking a 32-column chunk.
struct Walk {
  int b, i, j, jj, rowlen, tc, imax;
};

template <typename YT>
__device__ __forceinline__ YT cvt_out(float v) {
  return from_f<YT>(v);
}

// Epilogue of one 32 x 32 block of D (32 rows = (class, feature) pairs of
// this warp's TMEM lane quadrant, 32 consecutive anchor columns).  The block
// is transposed through a padded SMEM tile (row stride 36 floats: scalar
// writes and 16-byte reads are both conflict-free) so each thread then owns
// ONE anchor and writes every class pixel it touches with 16-byte stores.
template <typename YT, int ACT>
__device__ __forceinline__ void fold_epilogue_block(const Params& p, const float (&v)[32],
                                                    float* tile, const Walk& w, int warp,
                                                    int lane, int ncols, float wsc, float& chk) {
  // write: thread = row, column k -> tile[k][row]
#pragma unroll
  for (int k = 0; k < 32; ++k) tile[k * 36 + lane] = v[k];
  __syncwarp();
  // this thread's anchor: column lane of the block
  int jj = w.jj + lane, i = w.i, b = w.b;
  if (jj >= w.rowlen) {  // rows shorter than the block: divide once
    const int di = jj / w.rowlen;
    jj -= di * w.rowlen;
    i += di;
    if (i >= w.imax) {
      b += i / w.imax;
      i -= (i / w.imax) * w.imax;
    }
  }
  const int j = w.j - w.jj + jj;
  const bool anchor_ok = jj < w.tc && b < p.batch && lane < ncols;  // ncols: unit's live columns
  YT* __restrict__ y = reinterpret_cast<YT*>(p.y);
  const int CP = p.CP;
  const int q0 = (warp * 32) / CP;                 // first class in this quadrant
  const int nq = min(4 - q0, max(1, 32 / CP));     // classes held by these 32 rows
  auto fin = [&](float x, int f) {
    guard_check(chk, x);  // range guard: the raw sum of a stored output
    x *= wsc;  // split-fp16 images hold w * 2^s (1 otherwise)
    if (p.epi & SEGCONV_EPI_BIAS) x += __ldg(p.bias + f);
    if (ACT == 1) x = fmaxf(x, 0.0f);
    if (ACT == 2) x = tanhf(x);
    return x;
  };
  constexpr int LPP = 32 * (int)sizeof(YT) / 16;  // lanes per 32-feature pixel row
  if (CP == 32 && p.cout == 32) {
    // warp-cooperative stores: LPP lanes write one anchor's 32 features as
    // consecutive 16-byte pieces, so every instruction writes whole lines
    const int q = q0, r = q >> 1, c = q & 1;
    const bool ok = anchor_ok && i < p.rows[q] && j < p.cols[q];
    const long long base =
        ok ? (((long long)b * p.out_h + (2 * i + r)) * p.out_w + (2 * j + c)) * 32 : -1;
    constexpr int PPR = 32 / LPP;  // anchors per round
    const int sub = lane % LPP, slot = lane / LPP;
    float4 a[32 / PPR][LPP == 8 ? 1 : 2];
#pragma unroll
    for (int t = 0; t < 32 / PPR; ++t) {  // all tile reads first (ILP)
      const float* src = tile + (t * PPR + slot) * 36;
      if (LPP == 8) {
        a[t][0] = *reinterpret_cast<const float4*>(src + sub * 4);
      } else {
        a[t][0] = *reinterpret_cast<const float4*>(src + sub * 8);
        a[t][LPP == 8 ? 0 : 1] = *reinterpret_cast<const float4*>(src + sub * 8 + 4);
      }
    }
#pragma unroll
    for (int t = 0; t < 32 / PPR; ++t) {
      const long long bb = __shfl_sync(0xffffffffu, base, t * PPR + slot);
      if (bb < 0 || (p.debug_nostore & 1)) continue;
      if (LPP == 8) {
        const int f = sub * 4;
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + bb + f) =
            make_float4(fin(a[t][0].x, f), fin(a[t][0].y, f + 1), fin(a[t][0].z, f + 2),
                        fin(a[t][0].w, f + 3));
      } else {
        const int f = sub * 8;
        const float4 x0 = a[t][0], x1 = a[t][LPP == 8 ? 0 : 1];
        __nv_bfloat162 h[4] = {__floats2bfloat162_rn(fin(x0.x, f), fin(x0.y, f + 1)),
                               __floats2bfloat162_rn(fin(x0.z, f + 2), fin(x0.w, f + 3)),
                               __floats2bfloat162_rn(fin(x1.x, f + 4), fin(x1.y, f + 5)),
                               __floats2bfloat162_rn(fin(x1.z, f + 6), fin(x1.w, f + 7))};
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(y) + bb + f) =
            *reinterpret_cast<const uint4*>(h);
      }
    }
    __syncwarp();
    return;
  }
  const float* row = tile + lane * 36;  // this anchor's 32 (class, feature) values
  for (int qq = 0; qq < nq; ++qq) {
    const int q = q0 + qq, r = q >> 1, c = q & 1;
    if (!(anchor_ok && i < p.rows[q] && j < p.cols[q])) continue;
    const float* src = row + (q * CP - warp * 32);
    YT* dst = y + (((long long)b * p.out_h + (2 * i + r)) * p.out_w + (2 * j + c)) * p.cout;
    if (!(p.debug_nostore & 1))
      for (int f = 0; f < p.cout; ++f) dst[f] = from_f<YT>(fin(src[f], f));
  }
  __syncwarp();
}

// Advance a walk by d staged columns (d >= 0).
__device__ __forceinline__ void walk_advance(Walk& w, int d) {
  w.jj += d;
  w.j += d;
  while (w.jj >= w.rowlen) {
    w.jj -= w.rowlen;
    w.j -= w.rowlen;
    if (++w.i == w.imax) {
      w.i = 0;
      ++w.b;
    }
  }
}

template <int MODE, int N, bool TMEM_A>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_fold_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  // TMEM: D tiles of N fp32 columns.  TMEM_A: D double-buffered in columns
  // [0, 256) and the resident weights (the MMA A operand) in [256, 512);
  // otherwise D fills all 512 columns and the weights live in SMEM.
  constexpr int ACC_BUFS = TMEM_A ? 256 / N : 512 / N;
  constexpr int PLANES = MODE == MODE_F16X3 ? 2 : 1;

  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages_a;
  // SMEM-A: [resident weights][operand stages][landing stages][epilogue tiles]
  // TMEM-A: [operand stages][epilogue tiles][landing stages]; the weight image
  //         is staged once over the first two regions and copied into TMEM
  //         (tcgen05.cp) before any operand stage or tile is written.
  const int SL = p.land ? p.stages_l : 0;
  uint8_t* w_base = smem;
  uint8_t* a_base = TMEM_A ? smem : smem + p.w_bytes;
  uint8_t* epi_base = TMEM_A ? a_base + (size_t)SA * p.a_stage_bytes
                             : a_base + (size_t)SA * p.a_stage_bytes + (size_t)SL * p.l_stage_bytes;
  uint8_t* l_base = TMEM_A ? epi_base + EPI_TILE_BYTES : a_base + (size_t)SA * p.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      TMEM_A ? l_base + (size_t)SL * p.l_stage_bytes : epi_base + EPI_TILE_BYTES);
  uint64_t* a_land = bars;
  uint64_t* a_full = a_land + SA;
  uint64_t* a_empty = a_full + SA;
  uint64_t* w_full = a_empty + SA;
  uint64_t* acc_full = w_full + 1;
  uint64_t* acc_empty = acc_full + ACC_BUFS;
  uint64_t* l_full = acc_empty + ACC_BUFS;
  uint64_t* l_empty = l_full + SL;
  uint64_t* w_free = l_empty + SL;  // TMEM-A: weight image copied out of SMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_free + 1);
  // a converter saw x outside the split's range (the word after the TMEM slot)
  volatile int& guard_bad = *reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) guard_bad = 0;
  if (warp == 12 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_land[s], 1);
      mbar_init(&a_full[s], MODE == MODE_F16X3 ? 128u : 1u);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < SL; ++s) {
      mbar_init(&l_full[s], 1);
      mbar_init(&l_empty[s], 128);
    }
    mbar_init(w_full, 1);
    mbar_init(w_free, 1);
    for (int s = 0; s < ACC_BUFS; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 14 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  if (warp == 13) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int CH = p.kb / 8;
  const uint32_t COL = (uint32_t)p.S_pad * 16;              // halo k-chunk column
  const uint32_t LBO_X = MODE == MODE_F16X3 ? 2 * COL : COL;  // hi/lo interleaved columns
  const uint32_t WCOL = (uint32_t)p.w_rows * 16;             // weight k-chunk column
  const uint32_t W_PLANE = (uint32_t)p.nkb * CH * WCOL;
  const int KS_ALL = p.cin / 16;                             // K=16 steps over cin

  if (warp == 14) {
    // ================= halo TMA issuer
    if (lane == 0 && p.land) {
      // LAND: one 2-D box {kb channels, rows} per piece -> 4*kb-byte rows
      int sl = 0;
      uint32_t ph = 0;
      const uint32_t row_bytes = (uint32_t)p.kb * 4;
      const uint32_t stage_tx = (uint32_t)(p.pieces * p.piece_rows) * row_bytes;
      long long m0;
      int nu, b, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b, i0, j0); ++k) {
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&l_empty[sl], ph ^ 1);
          mbar_arrive_expect_tx(&l_full[sl], stage_tx);
          const uint32_t lbase = smem_u32(l_base + (size_t)sl * p.l_stage_bytes);
          for (int pc = 0; pc < p.pieces; ++pc)
            tma_load_2d(lbase + (uint32_t)(pc * p.piece_rows) * row_bytes, &tmap, kb * p.kb,
                        (int)m0 + pc * p.piece_rows, &l_full[sl]);
          if (kb == 0) trace_ev(p, 0, k);
          if (++sl == SL) {
            sl = 0;
            ph ^= 1;
          }
        }
      }
    } else if (lane == 0) {
      if (TMEM_A) mbar_wait(w_free, 0);  // operand stages hold the staged weights until then
      int st = 0;
      uint32_t ph = 0;
      const uint32_t row_bytes = MODE == MODE_F16X3 ? 32 : 16;
      const uint32_t col_bytes = (uint32_t)p.S_pad * row_bytes;
      const uint32_t box_rows = p.block_mode ? (uint32_t)(p.P * p.TRH) : (uint32_t)p.piece_rows;
      const uint32_t stage_tx =
          (uint32_t)CH * (p.block_mode ? box_rows : (uint32_t)(p.pieces * p.piece_rows)) * row_bytes;
      long long m0;
      int nu, b, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b, i0, j0); ++k) {
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_empty[st], ph ^ 1);
          uint64_t* bar = MODE == MODE_F16X3 ? &a_land[st] : &a_full[st];
          mbar_arrive_expect_tx(bar, stage_tx);
          const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
          for (int j = 0; j < CH; ++j) {
            if (p.block_mode) {
              tma_load_4d(sbase + (uint32_t)j * col_bytes, &tmap, 0, j0, b * p.n + i0, kb * CH + j,
                          bar);
            } else {
              for (int pc = 0; pc < p.pieces; ++pc)
                tma_load_3d(sbase + (uint32_t)j * col_bytes + (uint32_t)(pc * p.piece_rows) * row_bytes,
                            &tmap, 0, (int)m0 + pc * p.piece_rows, kb * CH + j, bar);
            }
          }
          if (kb == 0) trace_ev(p, 0, k);
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ================= fp16 hi/lo split in place (f16x3)
    // All reads of a stage's fp32 rows happen before the single barrier,
    // then every thread writes its rows' hi / lo halves (in-place hazard).
    if (MODE == MODE_F16X3 && p.land) {
      // LAND: item = (row, 16-byte k-chunk); a warp reads 8 whole 128-byte
      // landing rows and writes 8 consecutive rows of each chunk column
      const int pt = threadIdx.x - 256;
      int sa = 0, sl = 0;
      uint32_t pa = 0, pl = 0;
      const uint32_t lrow = (uint32_t)p.kb * 4;
      if (TMEM_A) mbar_wait(w_free, 0);  // operand stages hold the staged weights until then
      GuardTrack gt;
      gt.init(p.fb.guard);
      long long m0;
      int nu, b, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b, i0, j0); ++k) {
        const int rows_live = min(p.pieces * p.piece_rows, nu + p.shift_off[p.shifts - 1]);
        const int items = rows_live * CH;
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&l_full[sl], pl);
          mbar_wait(&a_empty[sa], pa ^ 1);
          const uint32_t lbase = smem_u32(l_base + (size_t)sl * p.l_stage_bytes);
          const uint32_t abase = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          for (int it0 = pt; it0 < ((p.debug_nostore & 2) ? 0 : items); it0 += 4 * 128) {
            float4 v[4][2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int it = it0 + u * 128;
              if (it < items) {
                const int r = it / CH, j = it - (it / CH) * CH;
                const uint32_t src = lbase + (uint32_t)r * lrow + (uint32_t)j * 32;
                ld_shared_v4f(src, v[u][0]);
                ld_shared_v4f(src + 16, v[u][1]);
                gt.add(v[u][0]);
                gt.add(v[u][1]);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int it = it0 + u * 128;
              if (it < items) {
                const int r = it / CH, j = it - (it / CH) * CH;
                uint32_t hi[4], lo[4];
                split8x2(v[u][0], v[u][1], hi, lo);
                const uint32_t dst = abase + (uint32_t)j * 2 * COL + (uint32_t)r * 16;
                st_shared_v4(dst, hi[0], hi[1], hi[2], hi[3]);
                st_shared_v4(dst + COL, lo[0], lo[1], lo[2], lo[3]);
              }
            }
          }
          fence_proxy_async();
          if (kb == 0 && threadIdx.x == 256) trace_ev(p, 1, k);
          if (kb == p.nkb - 1 && threadIdx.x == 256) trace_ev(p, 7, k);
          mbar_arrive(&a_full[sa]);
          mbar_arrive(&l_empty[sl]);
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
          if (++sl == SL) {
            sl = 0;
            pl ^= 1;
          }
        }
      }
      if (gt.bad()) guard_bad = 1;
    } else if constexpr (MODE == MODE_F16X3) {
      const int pt = threadIdx.x - 256;
      int st = 0;
      uint32_t ph = 0;
      const int rows_staged = p.block_mode ? p.P * p.TRH : p.pieces * p.piece_rows;
      // RPC row slots of 128 per chunk column; RPT_MAX = 4 chunks x RPC slots
      constexpr int RPC = 3, RPT_MAX = 4 * RPC;  // <= 384 rows x 4 chunks per stage
      GuardTrack gt;
      gt.init(p.fb.guard);
      long long m0;
      int nu, b, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b, i0, j0); ++k) {
        // rows a unit actually reads: its anchors plus the largest shift
        const int rows_live = p.block_mode ? rows_staged
                                           : min(rows_staged, nu + p.shift_off[p.shifts - 1] + 1);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_land[st], ph);
          const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
          if (p.debug_nostore & 2) {
            mbar_arrive(&a_full[st]);
            if (++st == SA) {
              st = 0;
              ph ^= 1;
            }
            continue;
          }
          float4 v[RPT_MAX][2];
#pragma unroll
          for (int q = 0; q < RPT_MAX; ++q) {
            const int j = q / RPC, s = pt + (q % RPC) * 128;
            if (j < CH && s < rows_live) {
              const uint32_t src = sbase + (uint32_t)j * 2 * COL + (uint32_t)s * 32;
              ld_shared_v4f(src, v[q][0]);
              ld_shared_v4f(src + 16, v[q][1]);
              gt.add(v[q][0]);
              gt.add(v[q][1]);
            }
          }
          named_bar(1, 128);
#pragma unroll
          for (int q = 0; q < RPT_MAX; ++q) {
            const int j = q / RPC, s = pt + (q % RPC) * 128;
            if (j < CH && s < rows_live) {
              uint32_t hi[4], lo[4];
              split8x2(v[q][0], v[q][1], hi, lo);
              const uint32_t dst = sbase + (uint32_t)j * 2 * COL + (uint32_t)s * 16;
              st_shared_v4(dst, hi[0], hi[1], hi[2], hi[3]);
              st_shared_v4(dst + COL, lo[0], lo[1], lo[2], lo[3]);
            }
          }
          fence_proxy_async();
          if (kb == 0 && threadIdx.x == 256) trace_ev(p, 1, k);
          mbar_arrive(&a_full[st]);
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
      if (gt.bad()) guard_bad = 1;
    }
  } else if (warp == 13) {
    // ================= resident weights in SMEM: one bulk-copy pass
    if (lane == 0) {
      const uint32_t wb = TMEM_A ? (uint32_t)p.w_img_bytes : (uint32_t)p.w_bytes;
      mbar_arrive_expect_tx(w_full, wb);
      constexpr uint32_t CHUNK = 32768;
      for (uint32_t off = 0; off < wb; off += CHUNK)
        bulk_g2s(w_base + off, p.panels + off, min(CHUNK, wb - off), w_full);
    }
  } else if (warp == 12) {
    // ================= MMA issuer
    if (lane == 0) {
      mbar_wait(w_full, 0);
      tc_fence_after();
      trace_ev(p, 6, 0);
      const uint32_t w_addr = smem_u32(w_base);
      const uint32_t a_tm = tmem_base + (uint32_t)p.a_tmem_col;
      if constexpr (TMEM_A) {
        // staged image [plane][k_block][k-chunk][shift*128 + row][16 B]: each
        // (shift, plane, k-chunk) is one 128-row block -> 4 TMEM columns at
        // ((shift * PLANES + plane) * KS_ALL + chunk / 2) * 8 + (chunk % 2) * 4
        for (int s = 0; s < p.shifts; ++s)
          for (int pl = 0; pl < PLANES; ++pl)
            for (int J = 0; J < p.cin / 8; ++J) {
              const int kbi = J / CH, j = J - (J / CH) * CH;
              const uint32_t src = w_addr + ((uint32_t)(pl * p.nkb + kbi) * CH + j) * WCOL +
                                   (uint32_t)(s * p.R) * 16;
              tmem_cp_128x128b(a_tm + (uint32_t)(((s * PLANES + pl) * KS_ALL + J / 2) * 8 + (J & 1) * 4),
                               sdesc(src, 2048, 128));
            }
        mma_commit(w_free);
      }
      int sa = 0, acc = 0;
      uint32_t pa = 0, pacc = 0;
      long long m0;
      int nu, b, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b, i0, j0); ++k) {
        const uint32_t idesc = idesc_f16(MODE == MODE_BF16 ? 1 : 0, nu);
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        trace_ev(p, 2, k);
        const uint32_t d = tmem_base + (uint32_t)(acc * N);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_full[sa], pa);
          tc_fence_after();
          const uint32_t x_addr = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          const uint32_t w_kb = w_addr + (uint32_t)(kb * CH) * WCOL;
          for (int s = 0; s < ((p.debug_nostore & 8) ? 0 : p.shifts); ++s) {
            const uint32_t xs = x_addr + (uint32_t)p.shift_off[s] * 16;
            const uint32_t ws = w_kb + (uint32_t)(s * p.R) * 16;
            for (int ks = 0; ks < CH / 2; ++ks) {
              const uint32_t acc_flag = (kb == 0 && s == 0 && ks == 0) ? 0u : 1u;
              if constexpr (TMEM_A) {
                // weight columns: ((shift * PLANES + plane) * KS_ALL + k-step) * 8
                const int ksg = kb * (CH / 2) + ks;
                const uint32_t wh = a_tm + (uint32_t)((s * PLANES * KS_ALL + ksg) * 8);
                if constexpr (MODE == MODE_F16X3) {
                  const uint32_t xk = xs + (uint32_t)ks * 4 * COL;
                  const uint64_t xh = sdesc(xk, LBO_X, 128);
                  const uint64_t xl = sdesc(xk + COL, LBO_X, 128);
                  const uint32_t wl = wh + (uint32_t)(KS_ALL * 8);
                  mma_f16_ts(d, wh, xh, idesc, acc_flag);
                  mma_f16_ts(d, wl, xh, idesc, 1u);
                  mma_f16_ts(d, wh, xl, idesc, 1u);
                } else {
                  mma_f16_ts(d, wh, sdesc(xs + (uint32_t)ks * 2 * COL, LBO_X, 128), idesc, acc_flag);
                }
              } else {
                const uint64_t wh = sdesc(ws + (uint32_t)ks * 2 * WCOL, WCOL, 128);
                if constexpr (MODE == MODE_F16X3) {
                  const uint32_t xk = xs + (uint32_t)ks * 4 * COL;  // hi chunks 2ks, 2ks+1
                  const uint64_t xh = sdesc(xk, LBO_X, 128);
                  const uint64_t xl = sdesc(xk + COL, LBO_X, 128);
                  const uint64_t wl = sdesc(ws + W_PLANE + (uint32_t)ks * 2 * WCOL, WCOL, 128);
                  mma_f16(d, wh, xh, idesc, acc_flag);
                  mma_f16(d, wl, xh, idesc, 1u);
                  mma_f16(d, wh, xl, idesc, 1u);
                } else {
                  const uint64_t xh = sdesc(xs + (uint32_t)ks * 2 * COL, LBO_X, 128);
                  mma_f16(d, wh, xh, idesc, acc_flag);
                }
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
        trace_ev(p, 3, k);
        if (++acc == ACC_BUFS) {
          acc = 0;
          pacc ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue: lanes = (class, feature), columns = anchors
    const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant, column-block parity
    const int row = quad * 32 + lane;
    int acc = 0;
    uint32_t pacc = 0;
    const int q = row / p.CP, f = row - (row / p.CP) * p.CP;
    const bool row_ok = row < p.R && f < p.cout;
    const bool warp_live = quad * 32 < p.R;
    const float wsc = MODE == MODE_F16X3 ? guard_inv_scale(p.fb.guard) : 1.0f;
    float chk = 0.0f;  // range guard: NaN once a stored sum is not finite
    (void)q;
    (void)row_ok;
    const long long img = (long long)p.n * p.n;
    long long m0;
    int nu, b0, i0, j0;
    for (int k = 0; next_unit(p, k, m0, nu, b0, i0, j0); ++k) {
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0) trace_ev(p, 4, k);
      if (warp_live) {  // quadrant holds (class, feature) rows
        const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * N);
        const int act = (p.epi & SEGCONV_EPI_RELU) ? 1 : (p.epi & SEGCONV_EPI_TANH) ? 2 : 0;
        const int sel = (p.y_dtype == SEGCONV_BF16 ? 3 : 0) + act;
        float* tile = reinterpret_cast<float*>(epi_base) + warp * 32 * 36;
        // anchor of the unit's first column, decoded once; blocks walk from it
        Walk w;
        if (!p.block_mode) {
          w.b = (int)(m0 / img);
          const int rem = (int)(m0 - (long long)w.b * img);
          w.i = rem / p.n;
          w.j = rem - w.i * p.n;
          w.jj = w.j;
          w.rowlen = p.n;
          w.tc = 1 << 30;
          w.imax = p.n;
        } else {
          w.b = b0;
          w.i = i0;
          w.j = j0;
          w.jj = 0;
          w.rowlen = p.P;
          w.tc = p.TC;
          w.imax = 1 << 30;
        }
        walk_advance(w, 32 * half);
#pragma unroll 1
        for (int c0 = 32 * half; c0 < nu; c0 += 64) {
          float v[32];
          tmem_ld32(tbase + (uint32_t)c0, v);
          if (!(p.debug_nostore & 4)) {
            switch (sel) {
              case 0: fold_epilogue_block<float, 0>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
              case 1: fold_epilogue_block<float, 1>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
              case 2: fold_epilogue_block<float, 2>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
              case 3: fold_epilogue_block<__nv_bfloat16, 0>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
              case 4: fold_epilogue_block<__nv_bfloat16, 1>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
              default: fold_epilogue_block<__nv_bfloat16, 2>(p, v, tile, w, quad, lane, nu - c0, wsc, chk); break;
            }
          }
          walk_advance(w, 64);
          if (c0 == 32 * half && threadIdx.x == 0) trace_ev(p, 8, k);
        }
      }
      tc_fence_before();
      if (threadIdx.x == 0) trace_ev(p, 5, k);
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
  if (warp == 13) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
  if (MODE == MODE_F16X3 && guard_bad) {
    // x left the split-fp16 range in this CTA's halos: recompute the anchors
    // of its units with FFMA (this CTA wrote them; the barrier orders the rewrite)
    if (!p.block_mode) {
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
    } else {
      long long m0;
      int nu, b0, i0, j0;
      for (int k = 0; next_unit(p, k, m0, nu, b0, i0, j0); ++k)
        guard_fallback(p.fb, (long long)p.TR * p.TC, 0, p.cout, [&](long long idx, int& b, int& i, int& j) {
          b = b0;
          i = i0 + (int)(idx / p.TC);
          j = j0 + (int)(idx % p.TC);
          return true;
        });
    }
  }
}

}  // namespace tcf

// ------------------------------------------------------------ host side
// Union-window extent per axis: max over parities of (class offset + taps).
void fold_window(int kh, int kw, int p, int* ur, int* uc) {
  int a = 0, b = 0;
  for (int r = 0; r < 2; ++r) {
    const int u0 = (p + r) & 1;
    const int acth = u0 >= kh ? 0 : (kh - u0 + 1) / 2, actw = u0 >= kw ? 0 : (kw - u0 + 1) / 2;
    const int off = (r + u0 - p) / 2 + p / 2;  // class_input_offset (segregation.hpp:33-36)
    a = std::max(a, off + acth);
    b = std::max(b, off + actw);
  }
  *ur = a;
  *uc = b;
}

int fold_cp(int cout) { return cout <= 4 ? 4 : cout <= 8 ? 8 : cout <= 16 ? 16 : 32; }
// channel block: a divisor of cin (cin % 16 == 0 is required), <= 32 for the
// split math (two fp16 planes), <= 64 for bf16
int fold_kb(int math, int cin) {
  if (cin % 64 == 0 && math == SEGCONV_MATH_BF16) return 64;
  return cin % 32 == 0 ? 32 : 16;
}
int fold_rows(int kh, int kw, int p, int cout) {
  int ur, uc;
  fold_window(kh, kw, p, &ur, &uc);
  const int R = 4 * fold_cp(cout);
  return ur * uc * R + (128 - R);
}

bool tc_fold_available(int math, int cin, int cout) {
  if (math != SEGCONV_MATH_BF16 && math != SEGCONV_MATH_F16X3) return false;
  return cout <= 32 && cin % 16 == 0;
}

// The resident weight image must leave room for >= 2 halo stages.
constexpr int FOLD_MAX_W_BYTES = 150 * 1024;
bool tc_fold_fits(int math, int kh, int kw, int p, int cin, int cout) {
  if (!tc_fold_available(math, cin, cout) || p / 2 != 0 || kh * kw > 49) return false;
  int ur, uc;
  fold_window(kh, kw, p, &ur, &uc);
  if (ur * uc > 16) return false;
  const long long planes = math == SEGCONV_MATH_F16X3 ? 2 : 1;
  const long long w = planes * cin * (long long)fold_rows(kh, kw, p, cout) * 2;
  return w <= FOLD_MAX_W_BYTES;
}

struct FoldPlan {
  tcf::Params p;
  CUtensorMap tmap;
  size_t smem;
  bool tmem_a;
  bool ok;
};

typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn2 encode_fn2() {
  static EncodeTiledFn2 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn2)f;
  });
  return fn;
}

static FoldPlan make_fold_plan_n(const FusedProblem& pr, int math, int block_n) {
  FoldPlan pl{};
  tcf::Params& p = pl.p;
  const bool split = math == SEGCONV_MATH_F16X3;
  const int planes = split ? 2 : 1, es = split ? 4 : 2;
  if (pr.pf != 0 || pr.kh * pr.kw > 49) return pl;
  int ur, uc;
  fold_window(pr.kh, pr.kw, pr.p, &ur, &uc);
  p.CP = fold_cp(pr.cout);
  p.R = 4 * p.CP;
  p.kb = fold_kb(math, pr.cin);
  if (pr.cin % p.kb) return pl;
  p.nkb = pr.cin / p.kb;
  p.batch = pr.batch;
  p.n = pr.n;
  p.cin = pr.cin;
  p.cout = pr.cout;
  p.out_h = pr.out_h;
  p.out_w = pr.out_w;
  p.panels = (const uint8_t*)pr.panels;
  p.y = pr.y;
  p.y_dtype = pr.y_dtype;
  p.bias = pr.bias;
  p.epi = pr.epi;
  p.fb = make_fallback_args(pr, split ? pr.guard : nullptr);
  if (split && !pr.guard) return pl;
  for (int q = 0; q < 4; ++q) {
    p.rows[q] = pr.cls.rows[q];
    p.cols[q] = pr.cls.cols[q];
  }
  const int CH = p.kb / 8;
  // staging geometry: LINEAR unless the image is wide enough that a 2-D block
  // wastes less halo; blocks of 4 x 64 anchors, else 2 x 64 if SMEM is short
  p.N = 128;
  p.block_mode = (ur - 1) * pr.n > p.N / 2 && pr.n >= 64 ? 1 : 0;
  int pitch;
  if (p.block_mode) {
    p.N = block_n;
    p.P = 64;
    p.TR = p.N / p.P;
    p.TC = p.P - (uc - 1);
    p.TRH = p.TR + ur - 1;
    const int rmax = std::max(pr.cls.rows[0], pr.cls.rows[2]);
    const int cmax = std::max(pr.cls.cols[0], pr.cls.cols[1]);
    p.tiles_r = (rmax + p.TR - 1) / p.TR;
    p.tiles_c = (cmax + p.TC - 1) / p.TC;
    p.units = (long long)pr.batch * p.tiles_r * p.tiles_c;
    p.S = p.P * p.TRH;
    p.S_pad = (p.S + uc + 7) / 8 * 8;  // garbage anchors may read uc-1 rows past the box
    pitch = p.P;
  } else {
    p.Mv = (long long)pr.batch * pr.n * pr.n;
    p.units = (p.Mv + p.N - 1) / p.N;
    p.S = p.N + (ur - 1) * pr.n + (uc - 1);
    p.pieces = (p.S + 255) / 256;
    p.piece_rows = ((p.S + p.pieces - 1) / p.pieces + 7) / 8 * 8;
    p.S_pad = p.pieces * p.piece_rows;
    pitch = pr.n;
  }
  p.shifts = ur * uc;
  if (p.shifts > tcf::MAX_SHIFTS) return pl;
  if (pr.y_dtype != SEGCONV_F32 && pr.y_dtype != SEGCONV_BF16) return pl;
  if (split && ((p.block_mode ? p.P * p.TRH : p.pieces * p.piece_rows) > 3 * 128 || p.kb > 32))
    return pl;  // converter: <= 3 rows of 128 per k-chunk column, <= 4 chunks
  for (int dy = 0; dy < ur; ++dy)
    for (int dx = 0; dx < uc; ++dx) p.shift_off[dy * uc + dx] = dy * pitch + dx;
  p.w_rows = p.shifts * p.R + (128 - p.R);
  // TMEM-A variant: when the four classes fill all 128 MMA rows and the weights
  // fit 256 TMEM columns (shifts * planes * cin / 2), the weights become the
  // MMA A operand in TMEM and all of shared memory goes to halo stages.
  pl.tmem_a = p.R == 128 && p.N <= 128 && p.shifts * planes * pr.cin / 2 <= 256;
  p.a_tmem_col = 256;
  p.w_img_bytes = planes * p.nkb * CH * p.w_rows * 16;
  p.w_bytes = pl.tmem_a ? 0 : p.w_img_bytes;
  p.w_bytes = (p.w_bytes + 1023) / 1024 * 1024;
  p.a_stage_bytes = (planes * CH * p.S_pad * 16 + 1023) / 1024 * 1024;
  const int max_stages = 8;
  const int bar_bytes = (5 * max_stages + 2 + 8) * 8 + 16;
  const int left = tcf::SMEM_LIMIT - bar_bytes - p.w_bytes - tcf::EPI_TILE_BYTES;
  // LAND (split math, LINEAR staging): the fp32 halo lands as {kb, rows} TMA
  // boxes (4*kb-byte rows: 128-byte requests at kb = 32, against 32-byte ones
  // for per-chunk boxes) and the converters write the operand stages.
  p.land = split && !p.block_mode ? 1 : 0;
  if (p.land) {
    p.l_stage_bytes = (p.pieces * p.piece_rows * p.kb * 4 + 1023) / 1024 * 1024;
    const int pair = p.a_stage_bytes + p.l_stage_bytes;
    const int n = std::min(left / pair, max_stages - 1);
    p.stages_l = std::max(2, (n * 3) / 7);
    p.stages_a = std::min(max_stages, (left - p.stages_l * p.l_stage_bytes) / p.a_stage_bytes);
    if (p.stages_a < 2) p.land = 0;
  }
  if (!p.land) {
    p.stages_l = p.l_stage_bytes = 0;
    p.stages_a = std::min(pl.tmem_a ? max_stages : 4, left / p.a_stage_bytes);
  }
  if (p.stages_a < 2) return pl;
  // TMEM-A stages the weight image over the operand stages + epilogue tiles
  if (pl.tmem_a && p.w_img_bytes > p.stages_a * p.a_stage_bytes + tcf::EPI_TILE_BYTES) return pl;
  pl.smem = (size_t)p.w_bytes + (size_t)p.stages_a * p.a_stage_bytes +
            (size_t)p.stages_l * p.l_stage_bytes + tcf::EPI_TILE_BYTES + bar_bytes;
  // halo tensor map
  EncodeTiledFn2 fn = encode_fn2();
  if (!fn) return pl;
  const CUtensorMapDataType dt = split ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult rc;
  if (p.block_mode) {
    const cuuint64_t dims[4] = {8, (cuuint64_t)pr.n, (cuuint64_t)pr.batch * pr.n,
                                (cuuint64_t)(pr.cin / 8)};
    const cuuint64_t strides[3] = {(cuuint64_t)pr.cin * es, (cuuint64_t)pr.n * pr.cin * es,
                                   (cuuint64_t)8 * es};
    const cuuint32_t box[4] = {8, (cuuint32_t)p.P, (cuuint32_t)p.TRH, 1};
    rc = fn(&pl.tmap, dt, 4, const_cast<void*>(pr.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (p.land) {
    const cuuint64_t dims[2] = {(cuuint64_t)pr.cin, (cuuint64_t)p.Mv};
    const cuuint64_t strides[1] = {(cuuint64_t)pr.cin * es};
    const cuuint32_t box[2] = {(cuuint32_t)p.kb, (cuuint32_t)p.piece_rows};
    rc = fn(&pl.tmap, dt, 2, const_cast<void*>(pr.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {8, (cuuint64_t)p.Mv, (cuuint64_t)(pr.cin / 8)};
    const cuuint64_t strides[2] = {(cuuint64_t)pr.cin * es, (cuuint64_t)8 * es};
    const cuuint32_t box[3] = {8, (cuuint32_t)p.piece_rows, 1};
    rc = fn(&pl.tmap, dt, 3, const_cast<void*>(pr.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  pl.ok = rc == CUDA_SUCCESS;
  return pl;
}

static FoldPlan make_fold_plan(const FusedProblem& pr, int math) {
  FoldPlan pl = make_fold_plan_n(pr, math, 256);
  if (!pl.ok) pl = make_fold_plan_n(pr, math, 128);
  return pl;
}

bool tc_fold_supported(const FusedProblem& pr, int math) {
  if (!tc_fold_available(math, pr.cin, pr.cout)) return false;
  if (pr.panel_layout != SEGCONV_PANEL_UMMA_FOLD) return false;
  if (math == SEGCONV_MATH_BF16 && (pr.x_dtype != SEGCONV_BF16 || pr.panel_dtype != SEGCONV_BF16))
    return false;
  if (math == SEGCONV_MATH_F16X3 &&
      (pr.x_dtype != SEGCONV_F32 || pr.panel_dtype != SEGCONV_F16_SPLIT))
    return false;
  return make_fold_plan(pr, math).ok;
}

template <int MODE, int N, bool TMEM_A>
static cudaError_t launch_fold_t(const FoldPlan& pl, cudaStream_t s) {
  auto kern = tcf::tc_fold_kernel<MODE, N, TMEM_A>;
  static PerDeviceOnce once;
  {
    const cudaError_t e = smem_attr_once(once, kern, tcf::SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  const long long grid = std::min<long long>(pl.p.units, sms);
  tcf::Params prm = pl.p;
  prm.trace = tc_trace_buffer();
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  prm.debug_nostore = dbg;
  kern<<<(unsigned)grid, tcf::NUM_THREADS, pl.smem, s>>>(prm, pl.tmap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tc_fold(const FusedProblem& pr, int math, cudaStream_t s) {
  const FoldPlan pl = make_fold_plan(pr, math);
  if (!pl.ok) return cudaErrorNotSupported;
  if (pl.p.units == 0) return cudaSuccess;
  const int mode = math == SEGCONV_MATH_F16X3 ? tcf::MODE_F16X3 : tcf::MODE_BF16;
  if (pl.tmem_a)
    return mode == tcf::MODE_F16X3 ? launch_fold_t<tcf::MODE_F16X3, 128, true>(pl, s)
                                   : launch_fold_t<tcf::MODE_BF16, 128, true>(pl, s);
  if (mode == tcf::MODE_F16X3)
    return pl.p.N == 256 ? launch_fold_t<tcf::MODE_F16X3, 256, false>(pl, s)
                         : launch_fold_t<tcf::MODE_F16X3, 128, false>(pl, s);
  return pl.p.N == 256 ? launch_fold_t<tcf::MODE_BF16, 256, false>(pl, s)
                       : launch_fold_t<tcf::MODE_BF16, 128, false>(pl, s);
}

}  // namespace segconv_b200

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
// Warp roles (352 threads): 0-3 epilogue, 4-7 fp16 hi/lo converters (split
// math), 8 MMA issuer, 9 weight loader + TMEM owner, 10 halo TMA issuer.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace segconv_b200 {
namespace tcf {

using namespace tc;

constexpr int MODE_BF16 = 0, MODE_F16X3 = 1;
constexpr int NUM_THREADS = 352;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int MAX_SHIFTS = 16;

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
  int shifts;
  int shift_off[MAX_SHIFTS];       // dy * pitch + dx
  int rows[4], cols[4];
};

__device__ __forceinline__ void unit_origin(const Params& p, long long u, long long& m0, int& b,
                                            int& i0, int& j0) {
  if (!p.block_mode) {
    m0 = u * p.N;
    b = i0 = j0 = 0;
  } else {
    const long long per = (long long)p.tiles_r * p.tiles_c;
    b = (int)(u / per);
    const int t = (int)(u - (long long)b * per);
    i0 = (t / p.tiles_c) * p.TR;
    j0 = (t % p.tiles_c) * p.TC;
    m0 = 0;
  }
}

template <int MODE, int N>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_fold_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  constexpr int ACC_BUFS = 512 / N;  // N = 128 -> 4, 256 -> 2
  constexpr uint32_t IDESC = idesc_f16(MODE == MODE_BF16 ? 1 : 0, N);

  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages_a;
  uint8_t* w_base = smem;                         // resident weights
  uint8_t* a_base = smem + p.w_bytes;             // halo stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_base + (size_t)SA * p.a_stage_bytes);
  uint64_t* a_land = bars;
  uint64_t* a_full = a_land + SA;
  uint64_t* a_empty = a_full + SA;
  uint64_t* w_full = a_empty + SA;
  uint64_t* acc_full = w_full + 1;
  uint64_t* acc_empty = acc_full + ACC_BUFS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + ACC_BUFS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 8 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_land[s], 1);
      mbar_init(&a_full[s], MODE == MODE_F16X3 ? 128u : 1u);
      mbar_init(&a_empty[s], 1);
    }
    mbar_init(w_full, 1);
    for (int s = 0; s < ACC_BUFS; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 10 && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  if (warp == 9) {
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

  if (warp == 10) {
    // ================= halo TMA issuer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      const uint32_t row_bytes = MODE == MODE_F16X3 ? 32 : 16;
      const uint32_t col_bytes = (uint32_t)p.S_pad * row_bytes;
      const uint32_t box_rows = p.block_mode ? (uint32_t)(p.P * p.TRH) : (uint32_t)p.piece_rows;
      const uint32_t stage_tx =
          (uint32_t)CH * (p.block_mode ? box_rows : (uint32_t)(p.pieces * p.piece_rows)) * row_bytes;
      for (long long u = blockIdx.x; u < p.units; u += gridDim.x) {
        long long m0;
        int b, i0, j0;
        unit_origin(p, u, m0, b, i0, j0);
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
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ================= fp16 hi/lo split in place (f16x3)
    if constexpr (MODE == MODE_F16X3) {
      const int pt = threadIdx.x - 128;
      int st = 0;
      uint32_t ph = 0;
      const int rows_staged = p.block_mode ? p.P * p.TRH : p.pieces * p.piece_rows;
      constexpr int RPT = 8;  // rows per thread: one pass covers all <= 1024 staged rows
      for (long long u = blockIdx.x; u < p.units; u += gridDim.x) {
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_land[st], ph);
          const uint32_t sbase = smem_u32(a_base + (size_t)st * p.a_stage_bytes);
          for (int j = 0; j < CH; ++j) {
            const uint32_t cbase = sbase + (uint32_t)j * 2 * COL;
            // all reads of the column precede all writes (in-place hazard)
            for (int r0 = 0; r0 < rows_staged; r0 += 128 * RPT) {
              float4 v[RPT][2];
#pragma unroll
              for (int k = 0; k < RPT; ++k) {
                const int s = r0 + pt + k * 128;
                if (s < rows_staged) {
                  ld_shared_v4f(cbase + (uint32_t)s * 32, v[k][0]);
                  ld_shared_v4f(cbase + (uint32_t)s * 32 + 16, v[k][1]);
                }
              }
              named_bar(1, 128);
#pragma unroll
              for (int k = 0; k < RPT; ++k) {
                const int s = r0 + pt + k * 128;
                if (s < rows_staged) {
                  uint32_t hi[4], lo[4];
                  split8(v[k][0], v[k][1], hi, lo);
                  st_shared_v4(cbase + (uint32_t)s * 16, hi[0], hi[1], hi[2], hi[3]);
                  st_shared_v4(cbase + COL + (uint32_t)s * 16, lo[0], lo[1], lo[2], lo[3]);
                }
              }
              named_bar(1, 128);
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
  } else if (warp == 9) {
    // ================= resident weights: one bulk-copy pass
    if (lane == 0) {
      mbar_arrive_expect_tx(w_full, (uint32_t)p.w_bytes);
      constexpr uint32_t CHUNK = 32768;
      for (uint32_t off = 0; off < (uint32_t)p.w_bytes; off += CHUNK)
        bulk_g2s(w_base + off, p.panels + off, min(CHUNK, (uint32_t)p.w_bytes - off), w_full);
    }
  } else if (warp == 8) {
    // ================= MMA issuer
    if (lane == 0) {
      mbar_wait(w_full, 0);
      tc_fence_after();
      const uint32_t w_addr = smem_u32(w_base);
      int sa = 0, acc = 0;
      uint32_t pa = 0, pacc = 0;
      for (long long u = blockIdx.x; u < p.units; u += gridDim.x) {
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * N);
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_full[sa], pa);
          tc_fence_after();
          const uint32_t x_addr = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          const uint32_t w_kb = w_addr + (uint32_t)(kb * CH) * WCOL;
          for (int s = 0; s < p.shifts; ++s) {
            const uint32_t xs = x_addr + (uint32_t)p.shift_off[s] * 16;
            const uint32_t ws = w_kb + (uint32_t)(s * p.R) * 16;
            for (int ks = 0; ks < CH / 2; ++ks) {
              const uint32_t acc_flag = (kb == 0 && s == 0 && ks == 0) ? 0u : 1u;
              const uint64_t wh = sdesc(ws + (uint32_t)ks * 2 * WCOL, WCOL, 128);
              if constexpr (MODE == MODE_F16X3) {
                const uint32_t xk = xs + (uint32_t)ks * 4 * COL;  // hi chunks 2ks, 2ks+1
                const uint64_t xh = sdesc(xk, LBO_X, 128);
                const uint64_t xl = sdesc(xk + COL, LBO_X, 128);
                const uint64_t wl = sdesc(ws + W_PLANE + (uint32_t)ks * 2 * WCOL, WCOL, 128);
                mma_f16(d, wh, xh, IDESC, acc_flag);
                mma_f16(d, wl, xh, IDESC, 1u);
                mma_f16(d, wh, xl, IDESC, 1u);
              } else {
                const uint64_t xh = sdesc(xs + (uint32_t)ks * 2 * COL, LBO_X, 128);
                mma_f16(d, wh, xh, IDESC, acc_flag);
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
        if (++acc == ACC_BUFS) {
          acc = 0;
          pacc ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue: lanes = (class, feature), columns = anchors
    int acc = 0;
    uint32_t pacc = 0;
    const int row = warp * 32 + lane;
    const int q = row / p.CP, f = row - (row / p.CP) * p.CP;
    const bool row_ok = row < p.R && f < p.cout;
    const bool warp_live = warp * 32 < p.R;
    const int r = q >> 1, c = q & 1;
    const int qrows = row_ok ? p.rows[q] : 0, qcols = row_ok ? p.cols[q] : 0;
    const long long img = (long long)p.n * p.n;
    for (long long u = blockIdx.x; u < p.units; u += gridDim.x) {
      long long m0;
      int b0, i0, j0;
      unit_origin(p, u, m0, b0, i0, j0);
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (warp_live) {
        const uint32_t tbase = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(acc * N);
#pragma unroll 1
        for (int c0 = 0; c0 < N; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + (uint32_t)c0, v);
          if (!row_ok) continue;
          // anchor of column c0, then step along the row
          int b, i, j, rowlen;
          if (!p.block_mode) {
            const long long m = m0 + c0;
            b = (int)(m / img);
            const int rem = (int)(m - (long long)b * img);
            i = rem / p.n;
            j = rem - i * p.n;
            rowlen = p.n;
          } else {
            b = b0;
            i = i0 + c0 / p.P;
            j = j0 + c0 % p.P;
            rowlen = p.P;
          }
          int jj = p.block_mode ? c0 % p.P : j;  // position within the staged row
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const bool in_tile = !p.block_mode || jj < p.TC;
            if (in_tile && b < p.batch && i < qrows && j < qcols) {
              const long long pix =
                  ((long long)b * p.out_h + (2 * i + r)) * p.out_w + (2 * j + c);
              store_out(p.y, pix * p.cout + f, epilogue_apply(v[k], p.epi, p.bias, f), p.y_dtype);
            }
            ++j;
            ++jj;
            if (jj == rowlen) {  // wrap to the next staged row
              jj = 0;
              j -= rowlen;
              if (++i == (p.block_mode ? 1 << 30 : p.n)) {
                i = 0;
                ++b;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      if (++acc == ACC_BUFS) {
        acc = 0;
        pacc ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
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
  if (split && (p.block_mode ? p.P * p.TRH : p.S_pad) > 1024) return pl;  // converter: one pass
  for (int dy = 0; dy < ur; ++dy)
    for (int dx = 0; dx < uc; ++dx) p.shift_off[dy * uc + dx] = dy * pitch + dx;
  p.w_rows = p.shifts * p.R + (128 - p.R);
  p.w_bytes = planes * p.nkb * CH * p.w_rows * 16;
  p.w_bytes = (p.w_bytes + 1023) / 1024 * 1024;
  p.a_stage_bytes = (planes * CH * p.S_pad * 16 + 1023) / 1024 * 1024;
  const int bar_bytes = (3 * 4 + 1 + 8) * 8 + 16;
  const int left = tcf::SMEM_LIMIT - bar_bytes - p.w_bytes;
  p.stages_a = std::min(4, left / p.a_stage_bytes);
  if (p.stages_a < 2) return pl;
  pl.smem = (size_t)p.w_bytes + (size_t)p.stages_a * p.a_stage_bytes + bar_bytes;
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

template <int MODE, int N>
static cudaError_t launch_fold_t(const FoldPlan& pl, cudaStream_t s) {
  auto kern = tcf::tc_fold_kernel<MODE, N>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tcf::SMEM_LIMIT);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  const long long grid = std::min<long long>(pl.p.units, sms);
  kern<<<(unsigned)grid, tcf::NUM_THREADS, pl.smem, s>>>(pl.p, pl.tmap);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tc_fold(const FusedProblem& pr, int math, cudaStream_t s) {
  const FoldPlan pl = make_fold_plan(pr, math);
  if (!pl.ok) return cudaErrorNotSupported;
  if (pl.p.units == 0) return cudaSuccess;
  const int mode = math == SEGCONV_MATH_F16X3 ? tcf::MODE_F16X3 : tcf::MODE_BF16;
  if (mode == tcf::MODE_F16X3)
    return pl.p.N == 256 ? launch_fold_t<tcf::MODE_F16X3, 256>(pl, s)
                         : launch_fold_t<tcf::MODE_F16X3, 128>(pl, s);
  return pl.p.N == 256 ? launch_fold_t<tcf::MODE_BF16, 256>(pl, s)
                       : launch_fold_t<tcf::MODE_BF16, 128>(pl, s);
}

}  // namespace segconv_b200

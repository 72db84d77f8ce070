// tc_tile.cu -- K3 for few-output-channel bf16 layers on small images
// (BASELINE C5 layer d: 1024 x 11^2 x 128 -> 19^2 x 3, n = 3, tanh).
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for these layers; also the 4x4, p = 2
// (out = 2N) 3-channel last layers of GAN generators (reference
// analysis.hpp:96-114).
//
// Pixel scatter, as tc_ring.cu: one MMA per K step computes, for 128
// consecutive input pixels p (the NHWC order runs across rows and images),
//   D[p, (dy, q, dx, f)] = sum_ch X[p, ch] * W_q[dy - off_r][dx - off_c][ch][f]
// (27 useful columns of N = 48 for n = 3, cout = 3), and the epilogue sums
// the shifts: anchor m of the tile takes D[m + dy * n + dx, (dy, q, dx, f)].
// Images here are small, so one 128-pixel tile yields 128 - (U - 1)(n + 1)
// anchors; tiles overlap by (U - 1)(n + 1) pixels.  With an even p > 0 every
// input offset moves by -p/2 (padding): the tile starts p/2 (n + 1) pixels
// before its first anchor (a TMA box starting before pixel 0 is zero-filled)
// and contributions from outside the image are masked.
// The D tile goes TMEM -> registers -> a padded SMEM tile, and each epilogue
// thread gathers its anchor's 4 x cout sums from it.  bf16 activations land by
// TMA (box {64 channels, 128 pixels}, 128-byte swizzle) and are the MMA A
// operand directly; the weight image (rows = D columns) is resident in SMEM.
//
// Warp roles (320 threads): 0-7 epilogue (warps w, w + 4 drain half of TMEM
// lane quadrant w % 4 each; thread t sums anchor t % 128 for output row parity
// t / 128), 8 TMA producer / TMEM owner, 9 MMA issuer.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_scatter.cuh"

namespace segconv_b200 {
namespace tct {

using namespace tc;

constexpr int NUM_THREADS = 320;
constexpr int SMEM_LIMIT = 227 * 1024;
// Two CTAs per SM: a tile's epilogue (TMEM drain -> SMEM tile -> shift sums)
// is serial within a CTA, so the other CTA's MMAs and loads run under it
// (measured: C5 layer d at one CTA per SM spent ~3.6k cycles per 128-pixel
// tile, issue slots 28 % busy).  One CTA per SM when the weight image, the two
// D tiles and two stages do not fit half the shared memory (4x4, cin >= 256).
__host__ __device__ constexpr int smem_per_cta(int cps) { return cps == 2 ? 113 * 1024 : 227 * 1024; }
constexpr int KB = 64;  // bf16 channels per stage: one 128-byte row
constexpr int MAX_STAGES = 8;
constexpr int TILE = 128;

struct Params {
  const uint8_t* panels;  // tile weight image: [k-chunk][N rows][8 bf16]
  void* y;
  const float* bias;
  unsigned epi;
  int batch, n, cin, cout, out_h, out_w;
  long long Mv, tiles;
  int step;  // anchors per tile = TILE - (U - 1) * (n + 1)
  int pf;    // p_orig / 2: input offsets shift by -pf
  int back;  // pf * (n + 1): pixels of the tile before its first anchor
  int rows[4], cols[4];
  int stage_bytes, stages, w_bytes;
  unsigned long long* trace;
  int debug;
};

__device__ __forceinline__ void trace_ev(const Params& p, int ev, int local) {
  if (p.trace == nullptr || blockIdx.x >= 160 || local >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[(blockIdx.x * 16 + ev) * 64 + local] = t;
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// SMEM tile pitch (floats): the useful D columns, odd so that the drain's
// row-per-lane stores and the gather's loads hit distinct banks
template <int KH, int COUT>
__host__ __device__ constexpr int tile_pitch() {
  return ScatterLayout<KH, COUT>::NU | 1;
}

// TMEM columns [C0, C0 + CN) of this lane's D row -> its SMEM row (useful columns)
template <typename L, int C0, int CN>
__device__ __forceinline__ void drain_cols(uint32_t taddr, float* row) {
  static_assert(CN % 8 == 0, "x8 loads");
  uint32_t r[CN / 8][8];
#pragma unroll
  for (int c = 0; c < CN / 8; ++c) tmem_ld8_nw(taddr + (uint32_t)(C0 + 8 * c), r[c]);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < CN; ++c) {
    const int u = L::compact(C0 + c);
    if (u >= 0) row[u] = __uint_as_float(r[c / 8][c % 8]);
  }
}

template <int KH, int COUT, int ACT, typename YT, int CPS>
__global__ void __launch_bounds__(NUM_THREADS, CPS)
    tile_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap tmap) {
  using L = ScatterLayout<KH, COUT>;
  constexpr int U = L::U, N = L::N, TP = tile_pitch<KH, COUT>();
  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages;
  uint8_t* a_base = smem;
  uint8_t* w_base = smem + (size_t)SA * p.stage_bytes;
  float* dtile = reinterpret_cast<float*>(w_base + p.w_bytes);  // 2 x [TILE][TP]
  uint64_t* bars = reinterpret_cast<uint64_t*>(dtile + 2 * TILE * TP + (2 * TILE * TP) % 2);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + SA;
  uint64_t* acc_full = a_empty + SA;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* w_full = acc_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_ev(p, 6, 0);
  if (warp == 9 && lane == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 256);
    }
    mbar_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    if (lane == 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (threadIdx.x == 0) trace_ev(p, 8, 0);
  const int NKB = p.cin / KB;
  const uint32_t WCOL = (uint32_t)N * 16;

  if (warp == 8) {
    // ===== TMA producer: weights once, then {64 ch, 128 pixels} boxes per tile
    if (lane == 0) {
      // Both the activations and the weight image may come from the kernel
      // this one overlaps under programmatic dependent launch (the previous
      // stack layer, or segregate's image kernel right before a first call):
      // wait for it before the first global read.
      griddep_wait();
      mbar_arrive_expect_tx(w_full, (uint32_t)p.w_bytes);
      for (uint32_t off = 0; off < (uint32_t)p.w_bytes; off += 32768)
        bulk_g2s(w_base + off, p.panels + off, min(32768u, (uint32_t)p.w_bytes - off), w_full);
      int st = 0;
      uint32_t ph = 0;
      int k = 0;
      for (long long t = blockIdx.x; t < p.tiles; t += gridDim.x, ++k) {
        const int p0 = (int)(t * p.step) - p.back;  // may start before pixel 0: zero fill
        trace_ev(p, 0, k);
        for (int kb = 0; kb < NKB; ++kb) {
          mbar_wait(&a_empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&a_full[st], (uint32_t)p.stage_bytes);
          tma_load_2d(smem_u32(a_base + (size_t)st * p.stage_bytes), &tmap, kb * KB, p0, &a_full[st]);
          if (++st == SA) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    // ===== MMA issuer (whole warp in the loop; one elected lane issues)
    const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t wb = smem_u32(w_base);
    constexpr uint32_t IDESC = idesc_f16(1, N);
    int st = 0, acc = 0;
    uint32_t ph = 0, pacc = 0;
    mbar_wait(w_full, 0);
    tc_fence_after();
    int k = 0;
    for (long long t = blockIdx.x; t < p.tiles; t += gridDim.x, ++k) {
      mbar_wait(&acc_empty[acc], pacc ^ 1);
      tc_fence_after();
      if (lane == 0) trace_ev(p, 2, k);
      const uint32_t d = tb + (uint32_t)(acc * N);
      for (int kb = 0; kb < NKB; ++kb) {
        mbar_wait(&a_full[st], ph);
        tc_fence_after();
        const uint64_t ad = sw128_desc(smem_u32(a_base + (size_t)st * p.stage_bytes));
        if (!(p.debug & 8) && elect_one()) {
#pragma unroll
          for (int ks = 0; ks < KB / 16; ++ks) {
            const uint64_t bd = sdesc(wb + (uint32_t)(kb * (KB / 8) + 2 * ks) * WCOL, WCOL, 128);
            mma_f16(d, ad + 2u * ks, bd, IDESC, (kb == 0 && ks == 0) ? 0u : 1u);
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
      if (++acc == 2) {
        acc = 0;
        pacc ^= 1;
      }
    }
  } else {
    // ===== epilogue (warps 0-7).  Warps w and w + 4 drain TMEM lane quadrant
    // w % 4 (w < 4: D columns [0, N/2), else [N/2, N)) into a double-buffered
    // SMEM tile of the useful columns; then thread t sums anchor t % 128 for
    // output rows of parity t / 128.  One named barrier per tile: a drain into
    // buffer k & 1 follows the barrier of tile k - 1, which every thread passes
    // only after its gather from that buffer two tiles back.
    const int m = threadIdx.x & 127, rr = threadIdx.x >> 7;
    const uint32_t lane_base = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    float bias[COUT];
#pragma unroll
    for (int f = 0; f < COUT; ++f) bias[f] = (p.epi & SEGCONV_EPI_BIAS) ? __ldg(p.bias + f) : 0.0f;
    YT* y = reinterpret_cast<YT*>(p.y);
    const unsigned img = (unsigned)(p.n * p.n);
    // SMEM offset of shift (dy, dx) from the anchor's row (per-thread constant)
    int soff[U][U];
#pragma unroll
    for (int dy = 0; dy < U; ++dy)
#pragma unroll
      for (int dx = 0; dx < U; ++dx) soff[dy][dx] = ((dy - p.pf) * p.n + (dx - p.pf)) * TP;
    int acc = 0;
    uint32_t pacc = 0;
    int k = 0;
    for (long long t = blockIdx.x; t < p.tiles; t += gridDim.x, ++k) {
      // anchor geometry first: it overlaps the wait for the accumulator
      const long long g = t * p.step + m;  // this thread's anchor, tile pixel p.back + m
      const bool live = m < p.step && g < p.Mv && !(p.debug & 1);
      const unsigned gu = live ? (unsigned)g : 0u;  // Mv < 2^31 (host check)
      const int b = (int)(gu / img);
      const int rem = (int)(gu - (unsigned)b * img);
      const int i = rem / p.n, j = rem - (rem / p.n) * p.n;
      bool inb[U][U];
#pragma unroll
      for (int dy = 0; dy < U; ++dy)
#pragma unroll
        for (int dx = 0; dx < U; ++dx)
          inb[dy][dx] = (unsigned)(i + dy - p.pf) < (unsigned)p.n && (unsigned)(j + dx - p.pf) < (unsigned)p.n;
      float* dt = dtile + (k & 1) * (TILE * TP);
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0) trace_ev(p, 4, k);
      if (warp < 4)
        drain_cols<L, 0, N / 2>(lane_base + (uint32_t)(acc * N), dt + m * TP);
      else
        drain_cols<L, N / 2, N / 2>(lane_base + (uint32_t)(acc * N), dt + m * TP);
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);  // D is in SMEM now; the MMA may reuse the buffer
      if (++acc == 2) {
        acc = 0;
        pacc ^= 1;
      }
      named_bar(1, 256);
      if (live) {
        const float* row = dt + (p.back + m) * TP;
        float out[2][COUT];
        bool okc[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          // classes of row parity rr: q = 2 rr + c, both compile-time below
          const int q = rr * 2 + c;
          okc[c] = i < p.rows[q] && j < p.cols[q];
#pragma unroll
          for (int f = 0; f < COUT; ++f) {
            float s = bias[f];
#pragma unroll
            for (int dy = 0; dy < U; ++dy)
#pragma unroll
              for (int dx = 0; dx < U; ++dx) {
                const int col0 = L::ucol(dy, 0 + c, dx, f), col2 = L::ucol(dy, 2 + c, dx, f);
                const int col = rr ? col2 : col0;
                if (col < 0 || !inb[dy][dx]) continue;  // input pixel outside the image: zero
                s += row[soff[dy][dx] + col];
              }
            if (ACT == 1) s = fmaxf(s, 0.0f);
            if (ACT == 2) {
              if constexpr (sizeof(YT) == 2) {
                // bf16 output (8-bit mantissa): the SFU tanh (~2^-11 rel.) is exact enough
                asm("tanh.approx.f32 %0, %0;" : "+f"(s));
              } else {
                s = tanhf(s);
              }
            }
            out[c][f] = s;
          }
        }
        // pixels (2i + rr, 2j) and (2i + rr, 2j + 1): 2 x COUT consecutive values
        YT* o = y + (((long long)b * p.out_h + 2 * i + rr) * p.out_w + 2 * j) * COUT;
        if (sizeof(YT) == 2 && okc[0] && okc[1] && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
          const float* fl = &out[0][0];
#pragma unroll
          for (int e = 0; e < COUT; ++e) {  // 2*COUT values as COUT bf16 pairs
            const __nv_bfloat162 h = __floats2bfloat162_rn(fl[2 * e], fl[2 * e + 1]);
            reinterpret_cast<uint32_t*>(o)[e] = *reinterpret_cast<const uint32_t*>(&h);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
            if (okc[c])
#pragma unroll
              for (int f = 0; f < COUT; ++f) o[c * COUT + f] = from_f<YT>(out[c][f]);
        }
      }
      if (threadIdx.x == 0) trace_ev(p, 5, k);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_ev(p, 7, 0);
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem_base)
                 : "memory");
  }
}

// Weight image: rows = D columns (dy, q, dx, f), [k-chunk][N rows][8 bf16].
template <int KH, int COUT, typename TK>
__global__ void tile_image_kernel(const TK* __restrict__ k, int cin, SegClasses cls,
                                  __nv_bfloat16* __restrict__ out) {
  using L = ScatterLayout<KH, COUT>;
  const long long total = (long long)(cin / 8) * L::N;
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
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      float w = 0.0f;
      if (qq >= 0) {
        const int u = dy - cls.off_r[qq], v = dxx - cls.off_c[qq];
        const int ci = chunk * 8 + x;
        w = to_acc(k[(((long long)(cls.u0[qq] + 2 * u) * KH + (cls.v0[qq] + 2 * v)) * cin + ci) * COUT + ff]);
      }
      out[e * 8 + x] = __float2bfloat16_rn(w);
    }
  }
}

}  // namespace tct

// ------------------------------------------------------------ host side
template <int KH>
static constexpr int tile_n() {
  return ScatterLayout<KH, 3>::N;
}
size_t tile_image_bytes(int kh, int cin) {
  return (size_t)(cin / 8) * (kh == 4 ? tile_n<4>() : tile_n<3>()) * 16;
}

// 3x3 at p = 0 (C5 d) or 4x4 at an even p (GAN last layers, p = 2): cout = 3,
// bf16, a tile of 128 pixels that still leaves >= 32 anchors
bool tile_applies(int kh, int kw, int p, int n, int cin, int cout) {
  if (kh != kw || cout != 3 || cin % tct::KB != 0 || cin > 512 || n < 1) return false;
  if (!((kh == 3 && p == 0) || (kh == 4 && (p == 0 || p == 2)))) return false;
  // anchors are the n x n input positions: every class grid must fit in them
  // (out = 2n + 2p - kh, rows of class 0 = (out + 1) / 2)
  if ((2 * n + 2 * p - kh + 1) / 2 > n) return false;
  const int U = kh == 4 ? ScatterLayout<4, 3>::U : ScatterLayout<3, 3>::U;
  return tct::TILE - (U - 1) * (n + 1) >= 32;
}

// shared memory besides the activation stages: weight image, two D tiles, barriers
static int tile_fixed_bytes(int kh, int cin) {
  const int pitch = kh == 4 ? tct::tile_pitch<4, 3>() : tct::tile_pitch<3, 3>();
  return (int)tile_image_bytes(kh, cin) + (2 * tct::TILE * pitch + 2) * 4 + (2 * tct::MAX_STAGES + 5) * 8 + 16;
}

static bool tile_shape(const FusedProblem& pr) {
  return tile_applies(pr.kh, pr.kw, pr.p, pr.n, pr.cin, pr.cout) && pr.x_dtype == SEGCONV_BF16 &&
         (pr.y_dtype == SEGCONV_BF16 || pr.y_dtype == SEGCONV_F32) &&
         tile_fixed_bytes(pr.kh, pr.cin) + 2 * tct::TILE * 128 <= tct::smem_per_cta(1);
}

bool tc_tile_supported(const FusedProblem& pr, int math) {
  if (math != SEGCONV_MATH_BF16) return false;
  return tile_shape(pr);
}

template <int KH>
static cudaError_t tile_image_t(const void* k, int k_dtype, int cin, const SegClasses& cls, void* out,
                                cudaStream_t s) {
  const long long total = (long long)(cin / 8) * ScatterLayout<KH, 3>::N;
  const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 1024);
  if (k_dtype == SEGCONV_BF16)
    tct::tile_image_kernel<KH, 3, __nv_bfloat16><<<blocks, 256, 0, s>>>(
        (const __nv_bfloat16*)k, cin, cls, (__nv_bfloat16*)out);
  else if (k_dtype == SEGCONV_F32)
    tct::tile_image_kernel<KH, 3, float><<<blocks, 256, 0, s>>>((const float*)k, cin, cls,
                                                                (__nv_bfloat16*)out);
  else
    return cudaErrorNotSupported;
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tile_image(const void* k, int k_dtype, int kh, int cin, const SegClasses& cls, void* out,
                              cudaStream_t s) {
  return kh == 4 ? tile_image_t<4>(k, k_dtype, cin, cls, out, s) : tile_image_t<3>(k, k_dtype, cin, cls, out, s);
}

template <int KH>
static cudaError_t launch_tile_t(const FusedProblem& pr, const void* img, cudaStream_t s) {
  using L = ScatterLayout<KH, 3>;
  tct::Params p{};
  p.panels = (const uint8_t*)img;
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
  p.Mv = (long long)pr.batch * pr.n * pr.n;
  if (p.Mv >= (1LL << 31)) return cudaErrorNotSupported;
  p.pf = pr.p / 2;
  p.back = p.pf * (pr.n + 1);
  p.step = tct::TILE - (L::U - 1) * (pr.n + 1);
  p.tiles = (p.Mv + p.step - 1) / p.step;
  if (p.tiles == 0) return cudaSuccess;
  p.stage_bytes = tct::TILE * 128;
  p.w_bytes = (int)tile_image_bytes(KH, pr.cin);
  const int fixed = tile_fixed_bytes(KH, pr.cin);
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  p.debug = dbg;
  // two CTAs per SM (three measured no faster on the C5 stack: 121.8 vs 121.3 us);
  // one where the weight image of a wide 4x4 layer leaves no room for two
  int cps = 2;
  while (cps > 1 && (tct::smem_per_cta(cps) - fixed) / p.stage_bytes < 2) --cps;
  p.stages = std::min(tct::MAX_STAGES, (tct::smem_per_cta(cps) - fixed) / p.stage_bytes);
  if (p.stages < 2) return cudaErrorNotSupported;
  p.trace = tc_trace_buffer();
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
  const cuuint64_t dims[2] = {(cuuint64_t)pr.cin, (cuuint64_t)p.Mv};
  const cuuint64_t strides[1] = {(cuuint64_t)pr.cin * 2};
  const cuuint32_t box[2] = {(cuuint32_t)tct::KB, (cuuint32_t)tct::TILE};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pr.x), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  const int sms = device_sm_count();
  const long long grid = std::min<long long>(p.tiles, (long long)cps * sms);
  const size_t smem = (size_t)p.stages * p.stage_bytes + fixed;
  const int act = (pr.epi & SEGCONV_EPI_RELU) ? 1 : (pr.epi & SEGCONV_EPI_TANH) ? 2 : 0;
  cudaError_t e = cudaSuccess;
#define TILE_LAUNCH(A, YT)                                                                       \
  {                                                                                              \
    auto kern = cps == 2 ? tct::tile_kernel<KH, 3, A, YT, 2> : tct::tile_kernel<KH, 3, A, YT, 1>;  \
    static PerDeviceOnce once[2];                                                                \
    e = smem_attr_once(once[cps - 1], kern, tct::SMEM_LIMIT);                                     \
    if (e != cudaSuccess) return e;                                                              \
    cudaLaunchConfig_t lc = {};                                                                 \
    lc.gridDim = dim3((unsigned)grid);                                                           \
    lc.blockDim = dim3(tct::NUM_THREADS);                                                        \
    lc.dynamicSmemBytes = smem;                                                                  \
    lc.stream = s;                                                                               \
    cudaLaunchAttribute at[1];                                                                   \
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                               \
    at[0].val.programmaticStreamSerializationAllowed = 1;                                        \
    lc.attrs = at;                                                                               \
    lc.numAttrs = 1;                                                                             \
    e = cudaLaunchKernelEx(&lc, kern, p, tmap);                                                  \
    if (e != cudaSuccess) return e;                                                              \
  }
  if (pr.y_dtype == SEGCONV_BF16) {
    if (act == 1)
      TILE_LAUNCH(1, __nv_bfloat16)
    else if (act == 2)
      TILE_LAUNCH(2, __nv_bfloat16)
    else
      TILE_LAUNCH(0, __nv_bfloat16)
  } else {
    if (act == 1)
      TILE_LAUNCH(1, float)
    else if (act == 2)
      TILE_LAUNCH(2, float)
    else
      TILE_LAUNCH(0, float)
  }
#undef TILE_LAUNCH
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tc_tile(const FusedProblem& pr, const void* img, cudaStream_t s) {
  if (!tile_shape(pr)) return cudaErrorNotSupported;
  return pr.kh == 4 ? launch_tile_t<4>(pr, img, s) : launch_tile_t<3>(pr, img, s);
}

}  // namespace segconv_b200

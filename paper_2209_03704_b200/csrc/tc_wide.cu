// tc_wide.cu -- K3 for wide bf16 layers (BASELINE C3, C5 a-c): the segregated
// transpose convolution as a CTA-pair (cta_group::2) tcgen05 implicit GEMM.
//
// Replaces reference proj/include/segconv/fused_tconv.hpp:42-60 and the dot
// loop of reference_ops.hpp:31-79 for bf16 layers with cin % 64 == 0.
//
// Formulation (halo shift, as tc_igemm.cu).  Anchors m = (b, i, j) of the
// NHWC input are GEMM rows; class q's tap (u, v) reads pixel m + shift,
// shift = (off_r + u) * n + (off_c + v), so every tap of every class is the
// same staged halo read from a different row.  A work unit is (pair tile of
// 256 anchors, feature tile of NT <= 256 outputs, class q):
//   D[m, f] = sum_{taps t of q} sum_ch X[m + shift_t, ch] * W_t[f, ch]
// with K = taps(q) * cin.
//
// B200 mapping.
//   * Two CTAs of a cluster (one TPC) run one M = 256 MMA (cta_group::2): CTA
//     r stages anchors [m0 + 128 r, +128) and features [NT/2 r, +NT/2) of the
//     tile, so each SM reads 4 KB of A and NT/2 * 32 B of B per K=16 step --
//     half the shared-memory and L2 traffic of a 1-SM tile -- while its TMEM
//     holds the full 128 x NT accumulator of its anchors.
//   * Halo and weights arrive by TMA as 128-byte rows (64 bf16 channels) with
//     the 128-byte swizzle; the MMA reads them through SW128 K-major
//     descriptors.  A row shift of the halo is a descriptor start offset with
//     base_offset 0 (known-answer test: scripts/sw128_test.cu).
//   * Weights come from the KMAJOR panels (class, f, u, v, ch): one 3-D
//     tensor map per class, box {64 ch, 1 tap, NT/2 features}.
//   * Both CTAs' TMA loads complete on the leader's mbarriers; the leader's
//     single MMA thread issues every MMA and multicasts its commits to both
//     CTAs' "empty" / "accumulator full" barriers; both epilogues release the
//     accumulator on the leader's barrier.
//   * D is double-buffered in TMEM (2 x NT columns), so the epilogue of one
//     unit overlaps the MMAs of the next.
//
// Warp roles (224 threads per CTA): 0-3 epilogue (lane = anchor: each thread
// stores its anchor's features contiguously, bias / ReLU / tanh fused),
// 4 A (activation) TMA producer, 5 MMA issuer (leader CTA), 6 B (weight) TMA
// producer and TMEM allocator; at one CTA per SM 352 threads, warps 7-10 a
// second set of epilogue warps (Params::epi8).
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <queue>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"
#include "tc_guard.cuh"

namespace segconv_b200 {
namespace tcw {

using namespace tc;

constexpr int NUM_THREADS = 224;  // 0-3 epilogue, 4 A producer, 5 MMA issuer, 6 B producer / TMEM owner
// One CTA per SM: four more epilogue warps (7-10; warp w drains TMEM lane
// quadrant w % 4 with warp w - 7 .. , alternate 32-column chunks each) -- a
// 256 x 256 unit's epilogue took longer than the MMAs of the short units
// queued behind it.  Two CTAs per SM keep 224 threads (register budget).
__host__ __device__ constexpr int wide_threads(int cps) { return cps == 2 ? NUM_THREADS : NUM_THREADS + 128; }
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int KB = 64;  // channels per stage: one 128-byte row
constexpr int WCH = 128;  // WGRAD: pixels (K) per chunk
constexpr int MAX_TAPS_Q = 25;  // 5x5: the input-gradient walk uses every tap as one class
constexpr int MAX_STAGES_A = 8, MAX_STAGES_B = 12;
constexpr int SMEM_PER_CTA2 = 113 * 1024;  // two CTAs per SM (Params::cps == 2)
// unit-schedule table entries (Params::sched): the parameters live in the
// constant bank, whose misses on a kernel's first reads are slow -- keep it small
constexpr int SCHED_MAX = 640;

struct Params {
  void* y;
  const float* bias;
  unsigned epi;
  int y_dtype;
  int batch, n, cin, cout, out_h, out_w;
  long long Mv;  // batch * n * n anchors (virtual positions, p_fused == 0)
  int NT, n_tiles, nkb;
  int S_rows;
  int a_stage_bytes, b_stage_bytes, stages_a, stages_b;
  int bprod;  // IM2COL: warp 6 issues the B loads (A and B on separate lanes)
  int taps[4];
  int shift[4][MAX_TAPS_Q];
  int rows[4], cols[4];
  long long pair_tiles, units;
  long long tail_full;  // IM2COL: units from here on are feature-tile halves (last partial wave)
  int tail_on;
  // TILE2D (p_fused > 0): each CTA stages TR rows of the padded (virtual) grid,
  // VW = n + 2 p_fused wide, as one 4-D TMA box whose out-of-image part is
  // zero-filled -- the padding is never materialised
  int tile2d, pf, VW, TR, TRH, tiles_per_img;
  int BW, BWo, col_tiles;  // TILE2D column blocks: box width (row pitch), anchors kept per block
  int allq;  // halo staging: one unit = all four classes of a tile (4 accumulators of NT <= 64)
  int wres;  // ALLQ with one feature tile: every (kb, class, tap) weight tile resident in SMEM
  int nacc;  // TMEM accumulator buffers (0 = 2; ALLQ with NT = 128 fills 512 columns with one)
  int tap_base[4];  // WRES: first tile of class q within a k-block
  // IM2COL (small images, where the halo-shift grid wastes rows): GEMM rows are
  // only class q's output anchors; each tap's A tile is gathered by an im2col
  // TMA (walk over the anchors, tap offset added per load)
  int im2col;
  long long unit_base[5];  // first unit of class q (units are class-major)
  int tap_off_r[4][MAX_TAPS_Q], tap_off_c[4][MAX_TAPS_Q];
  // walk origin of anchor (i, j): (wscale * i + wbase_r, wscale * j + wbase_c);
  // output pixel of anchor (i, j) of class (r, c): (ostride * i + r, ostride * j + c).
  // Forward: wscale 1, wbase -p_fused, ostride 2.  Input gradient (launch_tc_bwd_data):
  // wscale 2 (stride-2 im2col walk over gy), ostride 1, one class holding every tap.
  int wscale, wbase_r, wbase_c, ostride;
  int b_tap_last;  // B map coordinates (k, n, tap) instead of (k, tap, n)
  // SPLIT (fp32 layers, f16x3 math): x and w are stored as fp16 [hi | lo]
  // channel halves; the K loop runs three passes (xh.wh, xl.wh, xh.wl), pass
  // 1 reading A channels + split_off and pass 2 B channels + split_off
  int split, split_off;
  uint32_t ab_fmt;  // MMA operand format: 1 bf16, 0 fp16
  const float* split_inv_scale;  // SPLIT: the weights were scaled by 2^s; sums are multiplied by 2^-s
  int oscale;  // multiply the sums by *split_inv_scale without SPLIT's three passes (split-fp16 input gradient)
  const int* run_if;  // non-null: the whole grid exits at once unless *run_if != 0 (device-side range guard)
  // TF32 (fp32 data, math = tf32): fp32 operands, kind::tf32 MMAs (K = 8 per
  // instruction -- the same 32 bytes per step), 32 channels per 128-byte row
  int tf32;
  int kbc;  // channels per k-block (one 128-byte TMA row): 64 16-bit, 32 fp32
  // WGRAD (mode 1, launch_tc_bwd_weight): per unit (split s, tap t, 256-channel pair
  // tile ct, feature tile nt), D[ch, f] = sum over the split's 64-pixel chunks of
  // x[m, ch] * gy[b, 2i+p-U, 2j+p-V, f].  Both operands are MN-major (channels /
  // features contiguous, pixels = K): A from a 2-D map over x, B from the
  // stride-2 im2col walk over gy.  Results go to wout (+ s * ksz when split).
  int mode;
  int kstage;  // IM2COL forward: 64-channel k-blocks per pipeline stage (2 halves the handshakes)
  int cps;     // CTAs per SM (2: NT <= 128 forward, 256 TMEM columns each, two pipelines share the tensor pipe)
  int a_share;  // the stage's k-blocks multiply one A box (split-fp16 input gradient: [hi | lo] x two B halves)
  int w_kw, w_taps, w_ch_pairs, w_splits, w_cin, w_cout, w_direct, w_accumulate;
  int w_in_h, w_in_w;  // input map (anchor grid) of the kernel-gradient walk
  long long w_chunks, w_cps, w_ksz;
  float* wout;
  unsigned long long* trace;
  int debug;
  // IM2COL forward: per-pair unit lists from the host's balanced schedule
  // (launch_wide_t): entry = unit | (feature half << 14), 0xFFFF ends a list;
  // sched_slots == 0 keeps the round-robin order
  int epi8;  // one CTA per SM, forward: warps 7-10 join the epilogue (wide_threads)
  int sched_slots;
  int wh_ok;  // Maps::wh (half-width weight boxes) are encoded: half units may be scheduled
  uint16_t sched[SCHED_MAX];
};

struct Maps {
  CUtensorMap x;     // (cin, Mv) bf16, box {64, S_rows}; TILE2D: (cin, n, n, batch), box {64, VW, TRH, 1}
  CUtensorMap w[4];  // class q: (cin, taps_q, cout_pad) bf16, box {64, 1, NT/2}, 128B swizzle
  CUtensorMap xi[4]; // IM2COL class q: (cin, n, n, batch), walk over its anchors, 64 ch x 128 px
  CUtensorMap wh[4]; // as w, box {64, 1, NT/4}: a feature half unit's weights (Params::wh_ok)
};

// ---------------------------------------------------------------- PTX (pair)
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive (+ expect tx) on an mbarrier given by its shared::cluster address
__device__ __forceinline__ void mbar_arrive_expect_tx_cl(uint32_t bar_cl, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(
                   bar_cl),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl)
               : "memory");
}
// Relaxed form for the epilogue's "accumulator drained" arrive: only the TMEM
// reads (complete after tcgen05.wait::ld, ordered by the tcgen05 fences) must
// precede the MMA's reuse of the columns -- a release would also hold the warp
// until its outstanding global stores are acknowledged (an ERRBAR / membar
// stall in the epilogue, 4 % of the C5 layer-b samples)
__device__ __forceinline__ void mbar_arrive_cl_relaxed(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// TMA loads into this CTA's SMEM, completing on a (possibly peer) mbarrier
__device__ __forceinline__ void tma2_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                             uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                             int c2, uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma2_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                             int c2, int c3, uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma2_load_im2col(uint32_t dst, const CUtensorMap* map, int c, int w,
                                                 int h, int n, uint16_t ow, uint16_t oh,
                                                 uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow),
      "h"(oh)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma2_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// commit prior MMAs to the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// SW128 K-major descriptor: SBO = 1024 (8-row atoms), layout type 2, base offset 0
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16_m256(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
// kind::f16 with operand format fmt (1 bf16, 0 fp16), fp32 accumulate, M = 256
__host__ __device__ constexpr uint32_t idesc_f16_m256(uint32_t fmt, int n) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
// both operands MN-major (a_major bit 15, b_major bit 16)
__host__ __device__ constexpr uint32_t idesc_bf16_m256_mn(int n) {
  return idesc_bf16_m256(n) | (1u << 15) | (1u << 16);
}
// SW128 MN-major descriptor: 64-element (128-byte) rows along MN, one row per K;
// LBO = bytes between 64-element MN blocks, SBO = 1024 (8 K rows per atom)
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// WGRAD unit k of this pair -> (split, tap, channel pair tile, feature tile)
__device__ __forceinline__ bool wunit_of(const Params& p, int k, int& s, int& t, int& ct, int& nt) {
  const long long pairs = gridDim.x / 2;
  long long u = (long long)(blockIdx.x / 2) + (long long)k * pairs;
  if (u >= p.units) return false;
  nt = (int)(u % p.n_tiles);
  u /= p.n_tiles;
  ct = (int)(u % p.w_ch_pairs);
  u /= p.w_ch_pairs;
  t = (int)(u % p.w_taps);
  s = (int)(u / p.w_taps);
  return true;
}

// WGRAD segment k of this pair: tile (t, ct, nt), chunk range [c0, c1) of
// pixel split s, output slot s (0 when the sum is not split)
__device__ __forceinline__ bool wseg_of(const Params& p, int k, int& t, int& ct, int& nt, long long& c0,
                                        long long& c1, int& slot) {
  int s;
  if (!wunit_of(p, k, s, t, ct, nt)) return false;
  c0 = (long long)s * p.w_cps;
  c1 = min(p.w_chunks, c0 + p.w_cps);
  slot = p.w_direct ? 0 : s;
  return true;
}

__device__ __forceinline__ void trace_ev(const Params& p, int ev, int local) {
  if (p.trace == nullptr || blockIdx.x >= 160 || local >= 64) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  p.trace[(blockIdx.x * 16 + ev) * 64 + local] = t;
}

// unit k of this pair -> (pair tile, feature tile, class)
// hf: 0 = whole feature tile; 1 / 2 = its first / second half (tail units)
__device__ __forceinline__ bool unit_of(const Params& p, int k, long long& pt, int& nt, int& q, int& hf) {
  const long long pairs = gridDim.x / 2;
  long long u;
  hf = 0;
  if (p.sched_slots > 0) {
    if (k >= p.sched_slots) return false;
    const unsigned e = p.sched[(blockIdx.x >> 1) * p.sched_slots + k];
    if (e == 0xFFFFu) return false;
    u = e & 0x3FFFu;
    hf = (int)(e >> 14);
  } else {
    u = (long long)(blockIdx.x / 2) + (long long)k * pairs;
    if (u >= p.units) return false;
  }
  if (p.tail_on && u >= p.tail_full) {
    hf = 1 + (int)((u - p.tail_full) & 1);
    u = p.tail_full + ((u - p.tail_full) >> 1);
  }
  if (p.im2col) {  // class-major: [class q][pair tile][feature tile]
    q = 0;
    while (u >= p.unit_base[q + 1]) ++q;
    const long long v = u - p.unit_base[q];
    nt = (int)(v % p.n_tiles);
    pt = v / p.n_tiles;
    return true;
  }
  if (p.allq) {
    q = 0;
    nt = (int)(u % p.n_tiles);
    pt = u / p.n_tiles;
    return true;
  }
  q = (int)(u & 3);
  const long long t = u >> 2;
  nt = (int)(t % p.n_tiles);
  pt = t / p.n_tiles;
  return true;
}

template <int ACT>
__device__ __forceinline__ float finish(float v, const float* bias, unsigned epi, int f) {
  if (epi & SEGCONV_EPI_BIAS) v += __ldg(bias + f);
  if (ACT == 1) v = fmaxf(v, 0.0f);
  if (ACT == 2) v = tanhf(v);
  return v;
}
// bf16 outputs: the hardware tanh (max relative error ~2^-11) is below the bf16
// rounding of the result (2^-9); accurate tanhf dominated the epilogue of large
// bf16 tanh layers (EB-GAN preset, whose last layer writes 256^2 x 64 per image:
// 1.02 -> 0.80 ms per step)
template <int ACT>
__device__ __forceinline__ float finish_bf(float v, const float* bias, unsigned epi, int f) {
  if (epi & SEGCONV_EPI_BIAS) v += __ldg(bias + f);
  if (ACT == 1) v = fmaxf(v, 0.0f);
  if (ACT == 2) asm("tanh.approx.f32 %0, %1;" : "=f"(v) : "f"(v));
  return v;
}

template <typename YT, int ACT, int CPS>
__global__ void __launch_bounds__(wide_threads(CPS), CPS)
    wide_kernel(const __grid_constant__ Params p, const __grid_constant__ Maps maps) {
  if (threadIdx.x == 0) trace_ev(p, 14, 0);  // kernel entry (diagnostics)
  if (p.run_if != nullptr && *p.run_if == 0) return;  // every CTA alike: before any barrier or TMEM
  extern __shared__ __align__(1024) uint8_t smem[];
  const int SA = p.stages_a, SB = p.stages_b;
  uint8_t* a_base = smem;
  uint8_t* b_base = smem + (size_t)SA * p.a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_base + (size_t)SB * p.b_stage_bytes);
  uint64_t* a_full = bars;          // leader: both CTAs' halo bytes
  uint64_t* a_empty = a_full + SA;  // each CTA: MMAs done with the stage
  uint64_t* b_full = a_empty + SA;
  uint64_t* b_empty = b_full + SB;
  uint64_t* acc_full = b_empty + SB;  // each CTA: accumulator ready
  uint64_t* acc_empty = acc_full + 2;  // leader: both epilogues drained it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int kst = p.kstage > 0 ? p.kstage : 1;  // k-blocks per stage
  if (warp == 5 && lane == 0) {
    // IM2COL forward: one barrier pair per stage for A and B (both producers
    // arrive on a_full, both wait on a_empty) -- one wait and one commit per
    // stage in the MMA issuer
    const uint32_t full_count = (p.im2col && p.mode != 1 && p.bprod) ? 2u : 1u;
    for (int s = 0; s < SA; ++s) {
      mbar_init(&a_full[s], full_count);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], (CPS == 1 && p.epi8) ? 16 : 8);  // one arrive per epilogue warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    trace_ev(p, 15, 1);
  }
  if (warp == 4 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.x)) : "memory");
    for (int q = 0; q < 4; ++q) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[q])) : "memory");
      if (p.im2col)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.xi[q])) : "memory");
      if (p.wh_ok)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.wh[q])) : "memory");
    }
  }
  if (warp == 6) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(CPS == 2 ? 256 : 512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    if (lane == 0) trace_ev(p, 15, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_ev(p, 15, 2);
  cluster_sync_relaxed();  // both CTAs' barriers initialised before any remote arrive
  if (threadIdx.x == 0) trace_ev(p, 15, 3);
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) griddep_launch_dependents();  // next layer may start its prologue
  if (threadIdx.x == 0) trace_ev(p, 12, 0);

  const int NT2 = p.NT / 2;
  const int NACC = p.nacc > 0 ? p.nacc : 2;
  const uint32_t a_tx = (uint32_t)p.S_rows * 128, b_tx = (uint32_t)NT2 * 128;

  if (warp == 4 || (warp == 6 && p.mode == 1 && p.bprod)) {
    // ===== TMA producer (both CTAs): own halo rows and own half of the features
    // (WGRAD with bprod: warp 4 streams the x rows, warp 6 the gy im2col rows)
    const bool doA = warp == 4, doB = warp == 6 || !p.bprod;
    if (lane == 0 && p.mode == 1) {
      griddep_wait();
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int t, ct, nt, slot;
      long long cb, ce;
      const int img = p.w_in_h * p.w_in_w;
      const int di = WCH / p.w_in_w, dj = WCH - (WCH / p.w_in_w) * p.w_in_w;  // a chunk = di rows + dj pixels
      for (int k = 0; wseg_of(p, k, t, ct, nt, cb, ce, slot); ++k) {
        const int ch0 = ct * 256 + (int)rank * 128, f0 = nt * p.NT + (int)rank * NT2;
        // first anchor of the segment's first chunk; then advanced by 64 pixels per
        // chunk without divisions (the single producer lane is on the critical path)
        const long long mfirst = cb * WCH;
        int b0 = (int)(mfirst / img);
        int i0 = (int)(mfirst - (long long)b0 * img);
        int j0 = i0 % p.w_in_w;
        i0 /= p.w_in_w;
        for (long long c = cb; c < ce; ++c) {
          const long long m = c * WCH;
          if (doA) {
          mbar_wait(&a_empty[sa], pa ^ 1);
          const uint32_t af = mapa(smem_u32(&a_full[sa]), 0);
          if (rank == 0) mbar_arrive_expect_tx(&a_full[sa], 2 * 2 * WCH * 128);
          const uint32_t ad = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          tma2_load_2d(ad, &maps.x, ch0, (int)m, af);
          tma2_load_2d(ad + WCH * 128, &maps.x, ch0 + 64, (int)m, af);
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
          }
          if (doB) {
          mbar_wait(&b_empty[sb], pb ^ 1);
          const uint32_t bf = mapa(smem_u32(&b_full[sb]), 0);
          if (rank == 0) mbar_arrive_expect_tx(&b_full[sb], 2 * (uint32_t)(NT2 / 64) * WCH * 128);
          const uint32_t bd = smem_u32(b_base + (size_t)sb * p.b_stage_bytes);
          for (int h = 0; h < NT2 / 64; ++h)
            tma2_load_im2col(bd + h * WCH * 128, &maps.xi[0], f0 + 64 * h, p.wscale * j0 + p.wbase_c,
                             p.wscale * i0 + p.wbase_r,
                             b0, (uint16_t)p.tap_off_c[0][t], (uint16_t)p.tap_off_r[0][t], bf);
          if (++sb == SB) {
            sb = 0;
            pb ^= 1;
          }
          }
          j0 += dj;
          i0 += di;
          if (j0 >= p.w_in_w) {
            j0 -= p.w_in_w;
            ++i0;
          }
          if (i0 >= p.w_in_h) {
            const int q = i0 / p.w_in_h;
            b0 += q;
            i0 -= q * p.w_in_h;
          }
        }
      }
    } else if (p.mode != 1 && p.im2col && p.bprod && !p.wres) {
      // ===== IM2COL A producer, whole warp: the operands stay warp-uniform
      // (uniform registers, no per-lane R2UR / single-lane issue loop) and one
      // elected lane arrives and issues -- the single-lane form of this loop
      // took ~300 cycles per stage, more than a stage of N = 128 MMAs
      griddep_wait();
      int sa = 0, gsa = 0;
      uint32_t pa = 0;
      long long pt;
      int nt, q, hf;
      for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
        const int R = p.rows[q], C = p.cols[q];
        const long long a0 = pt * 256 + (long long)rank * 128;
        const int ib = (int)(a0 / ((long long)R * C));
        const int rem = (int)(a0 - (long long)ib * R * C);
        const int i0 = rem / C, j0 = rem - (rem / C) * C;
        const int xw = p.wscale * j0 + p.wbase_c, xh = p.wscale * i0 + p.wbase_r;
        const CUtensorMap* map = &maps.xi[q];
        const int taps = p.taps[q];
        for (int pass = 0; pass < (p.split ? 3 : 1); ++pass)
          for (int kb = 0; kb < p.nkb; ++kb) {
            const int ca = kb * p.kbc * kst + (pass == 1 ? p.split_off : 0);  // A: xl on pass 1
            for (int t = 0; t < taps; ++t) {
              mbar_wait(&a_empty[sa], pa ^ 1);
              if (lane == 0 && rank == 0) trace_ev(p, 10, gsa);
              ++gsa;
              if (elect_one()) {
                const uint32_t af = mapa(smem_u32(&a_full[sa]), 0);
                const int ka = p.a_share ? 1 : kst;  // A boxes per stage
                if (rank == 0)
                  mbar_arrive_expect_tx(&a_full[sa], (p.debug & 32) ? 0u : 2u * 128 * 128 * (uint32_t)ka);
                if (!(p.debug & 32))
                  for (int j = 0; j < ka; ++j)
                    tma2_load_im2col(smem_u32(a_base + (size_t)sa * p.a_stage_bytes) + (uint32_t)j * 16384u, map,
                                     ca + j * p.kbc, xw, xh, ib, (uint16_t)p.tap_off_c[q][t],
                                     (uint16_t)p.tap_off_r[q][t], af);
              }
              __syncwarp();
              if (++sa == SA) {
                sa = 0;
                pa ^= 1;
              }
            }
          }
      }
    } else if (lane == 0 && p.mode != 1) {
      griddep_wait();  // activations come from the previous kernel (stack layer)
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      if (p.wres && blockIdx.x / 2 < p.units) {  // all weight tiles once, on b_full[0]
        const uint32_t bf = mapa(smem_u32(&b_full[0]), 0);
        const int ntile = p.nkb * (p.taps[0] + p.taps[1] + p.taps[2] + p.taps[3]);
        if (rank == 0) mbar_arrive_expect_tx(&b_full[0], 2 * b_tx * (uint32_t)ntile);
        int idx = 0;
        for (int kb = 0; kb < p.nkb; ++kb)
          for (int qq = 0; qq < 4; ++qq)
            for (int t = 0; t < p.taps[qq]; ++t, ++idx)
              tma2_load_3d(smem_u32(b_base) + (uint32_t)idx * b_tx, &maps.w[qq], kb * KB, t, (int)rank * NT2, bf);
      }
      long long pt;
      int nt, q, hf;
      int gsa = 0;  // trace: global stage index
      for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
        const long long m0 = pt * 256 + (long long)rank * 128;
        const long long g = pt * 2 + rank;  // TILE2D: this CTA's row tile
        const int tb = p.tile2d ? (int)(g / p.tiles_per_img) : 0;
        const int trc = p.tile2d ? (int)(g - (long long)tb * p.tiles_per_img) : 0;  // (row tile, col block)
        const int trow = p.tile2d ? trc / p.col_tiles : 0;
        const int tvi0 = trow * p.TR, tvj0 = p.tile2d ? (trc - trow * p.col_tiles) * p.BWo : 0;
        const int f0 = hf ? nt * p.NT + (hf - 1) * NT2 + (int)rank * (NT2 / 2) : nt * p.NT + (int)rank * NT2;
        if (p.im2col) {
          // this CTA's first anchor of class q: (b, i, j) on the class's rows x cols grid
          const int R = p.rows[q], C = p.cols[q];
          const long long a0 = pt * 256 + (long long)rank * 128;
          const int ib = (int)(a0 / ((long long)R * C));
          const int rem = (int)(a0 - (long long)ib * R * C);
          const int i0 = rem / C, j0 = rem - (rem / C) * C;
          for (int pass = 0; pass < (p.split ? 3 : 1); ++pass)
          for (int kb = 0; kb < p.nkb; ++kb)
            for (int t = 0; t < p.taps[q]; ++t) {
              const int ca = kb * p.kbc + (pass == 1 ? p.split_off : 0);  // A: xl on pass 1
              const int cb = kb * p.kbc + (pass == 2 ? p.split_off : 0);  // B: wl on pass 2
              mbar_wait(&a_empty[sa], pa ^ 1);
              if (rank == 0) trace_ev(p, 10, gsa++);
              const uint32_t af = mapa(smem_u32(&a_full[sa]), 0);
              if (rank == 0) mbar_arrive_expect_tx(&a_full[sa], (p.debug & 32) ? 0u : 2 * 128 * 128);
              if (!(p.debug & 32))  // diagnostics: no activation loads
              tma2_load_im2col(smem_u32(a_base + (size_t)sa * p.a_stage_bytes), &maps.xi[q],
                               ca, p.wscale * j0 + p.wbase_c, p.wscale * i0 + p.wbase_r, ib,
                               (uint16_t)p.tap_off_c[q][t], (uint16_t)p.tap_off_r[q][t], af);
              if (++sa == SA) {
                sa = 0;
                pa ^= 1;
              }
              if (p.bprod) continue;  // warp 6 streams B
              mbar_wait(&b_empty[sb], pb ^ 1);
              const uint32_t bf = mapa(smem_u32(&b_full[sb]), 0);
              if (rank == 0) mbar_arrive_expect_tx(&b_full[sb], 2 * b_tx);
              if (p.b_tap_last)
                tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[q], cb, f0,
                             t, bf);
              else
                tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[q], cb, t,
                             f0, bf);
              if (++sb == SB) {
                sb = 0;
                pb ^= 1;
              }
            }
          if (rank == 0) trace_ev(p, 0, k);
          continue;
        }
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_empty[sa], pa ^ 1);
          // the leader expects both CTAs' bytes on its barrier; the peer only
          // issues its loads (they complete on the leader's barrier)
          const uint32_t af = mapa(smem_u32(&a_full[sa]), 0);
          if (rank == 0) mbar_arrive_expect_tx(&a_full[sa], (p.debug & 32) ? 0u : 2 * a_tx);
          if (!(p.debug & 32)) {  // diagnostics: no halo loads
            if (p.tile2d)
              tma2_load_4d(smem_u32(a_base + (size_t)sa * p.a_stage_bytes), &maps.x, kb * KB, tvj0 - p.pf,
                           tvi0 - p.pf, tb, af);
            else
              tma2_load_2d(smem_u32(a_base + (size_t)sa * p.a_stage_bytes), &maps.x, kb * KB,
                           (int)m0, af);
          }
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
          if (!p.wres && !p.bprod)
          for (int qq = p.allq ? 0 : q; qq < (p.allq ? 4 : q + 1); ++qq)
          for (int t = 0; t < p.taps[qq]; ++t) {
            mbar_wait(&b_empty[sb], pb ^ 1);
            const uint32_t bf = mapa(smem_u32(&b_full[sb]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&b_full[sb], (p.debug & 16) ? 0u : 2 * b_tx);
            if (!(p.debug & 16))  // diagnostics: no weight loads
              tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[qq], kb * KB, t,
                           f0, bf);
            if (++sb == SB) {
              sb = 0;
              pb ^= 1;
            }
          }
        }
        if (rank == 0) trace_ev(p, 0, k);
      }
    }
  } else if (warp == 6 && p.mode != 1) {
    // ===== IM2COL B producer (both CTAs): the weight tiles of every (pass, kb, tap)
    // step, in the A producer's order -- two serial issue chains instead of one
    if (p.im2col && p.bprod) {
      // whole warp, one elected lane issues (see the A producer)
      griddep_wait();
      int sb = 0, gsb = 0;
      uint32_t pb = 0;
      long long pt;
      int nt, q, hf;
      for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
        const int f0 = hf ? nt * p.NT + (hf - 1) * NT2 + (int)rank * (NT2 / 2) : nt * p.NT + (int)rank * NT2;
        // a scheduled feature half loads half-width weight boxes (the tail halves keep full boxes)
        const bool hb = hf && p.wh_ok && p.sched_slots > 0;
        const CUtensorMap* map = hb ? &maps.wh[q] : &maps.w[q];
        const uint32_t btx = hb ? b_tx / 2 : b_tx;
        const int taps = p.taps[q];
        for (int pass = 0; pass < (p.split ? 3 : 1); ++pass)
          for (int kb = 0; kb < p.nkb; ++kb) {
            const int cb = kb * p.kbc * kst + (pass == 2 ? p.split_off : 0);  // B: wl on pass 2
            for (int t = 0; t < taps; ++t) {
              // the stage's A and B share a_full / a_empty (SA == SB, lockstep)
              mbar_wait(&a_empty[sb], pb ^ 1);
              if (lane == 0 && rank == 0) trace_ev(p, 11, gsb);
              ++gsb;
              if (elect_one()) {
                const uint32_t bf = mapa(smem_u32(&a_full[sb]), 0);
                if (rank == 0) mbar_arrive_expect_tx(&a_full[sb], (p.debug & 16) ? 0u : 2 * btx * (uint32_t)kst);
                const uint32_t dst = smem_u32(b_base + (size_t)sb * p.b_stage_bytes);
                if (!(p.debug & 16))
                  for (int j = 0; j < kst; ++j) {
                    if (p.b_tap_last)
                      tma2_load_3d(dst + (uint32_t)j * b_tx, map, cb + j * p.kbc, f0, t, bf);
                    else
                      tma2_load_3d(dst + (uint32_t)j * b_tx, map, cb + j * p.kbc, t, f0, bf);
                  }
              }
              __syncwarp();
              if (++sb == SB) {
                sb = 0;
                pb ^= 1;
              }
            }
          }
      }
    } else if (lane == 0 && p.bprod) {
      griddep_wait();
      int sb = 0, gsb = 0;
      uint32_t pb = 0;
      long long pt;
      int nt, q, hf;
      for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
        const int f0 = hf ? nt * p.NT + (hf - 1) * NT2 + (int)rank * (NT2 / 2) : nt * p.NT + (int)rank * NT2;
        if (!p.im2col) {  // halo staging: (kb, class, tap) weight tiles in the MMA order
          for (int kb = 0; kb < p.nkb; ++kb)
            for (int qq = p.allq ? 0 : q; qq < (p.allq ? 4 : q + 1); ++qq)
              for (int t = 0; t < p.taps[qq]; ++t) {
                mbar_wait(&b_empty[sb], pb ^ 1);
                const uint32_t bf = mapa(smem_u32(&b_full[sb]), 0);
                if (rank == 0) mbar_arrive_expect_tx(&b_full[sb], 2 * b_tx);
                tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[qq], kb * KB, t, f0, bf);
                if (++sb == SB) {
                  sb = 0;
                  pb ^= 1;
                }
              }
          continue;
        }
        for (int pass = 0; pass < (p.split ? 3 : 1); ++pass)
          for (int kb = 0; kb < p.nkb; ++kb)
            for (int t = 0; t < p.taps[q]; ++t) {
              const int cb = kb * p.kbc + (pass == 2 ? p.split_off : 0);  // B: wl on pass 2
              // the stage's A and B share a_full / a_empty (SA == SB, lockstep)
              mbar_wait(&a_empty[sb], pb ^ 1);
              if (rank == 0) trace_ev(p, 11, gsb++);
              const uint32_t bf = mapa(smem_u32(&a_full[sb]), 0);
              if (rank == 0) mbar_arrive_expect_tx(&a_full[sb], (p.debug & 16) ? 0u : 2 * b_tx);
              if (p.debug & 16) {  // diagnostics: no weight loads
                if (++sb == SB) {
                  sb = 0;
                  pb ^= 1;
                }
                continue;
              }
              if (p.b_tap_last)
                tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[q], cb, f0, t, bf);
              else
                tma2_load_3d(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), &maps.w[q], cb, t, f0, bf);
              if (++sb == SB) {
                sb = 0;
                pb ^= 1;
              }
            }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===== MMA issuer (leader CTA; the whole warp runs the loop, one lane issues)
    if (rank == 0 && p.mode == 1) {
      const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
      int sa = 0, sb = 0, acc = 0;
      uint32_t pa = 0, pb = 0, pacc = 0;
      int t, ct, nt, slot;
      long long c0, c1;
      const uint32_t idesc = idesc_bf16_m256_mn(p.NT);
      for (int k = 0; wseg_of(p, k, t, ct, nt, c0, c1, slot); ++k) {
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        const uint32_t d = tb + (uint32_t)(acc * p.NT);
        for (long long c = c0; c < c1; ++c) {
          mbar_wait(&a_full[sa], pa);
          mbar_wait(&b_full[sb], pb);
          tc_fence_after();
          const uint64_t ad = sw128_mn_desc(smem_u32(a_base + (size_t)sa * p.a_stage_bytes), WCH * 128);
          const uint64_t bd = sw128_mn_desc(smem_u32(b_base + (size_t)sb * p.b_stage_bytes), WCH * 128);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < WCH / 16; ++ks)  // K = 16 pixels = 2 atoms of 8 rows: +2048 bytes
              mma2_bf16(d, ad + 128u * ks, bd + 128u * ks, idesc, (c == c0 && ks == 0) ? 0u : 1u);
          }
          __syncwarp();
          if (elect_one()) {
            commit2(&a_empty[sa]);
            commit2(&b_empty[sb]);
          }
          __syncwarp();
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
          if (++sb == SB) {
            sb = 0;
            pb ^= 1;
          }
        }
        if (elect_one()) commit2(&acc_full[acc]);
        __syncwarp();
        if (++acc == NACC) {
          acc = 0;
          pacc ^= 1;
        }
      }
    } else if (rank == 0) {
      const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
      int sa = 0, sb = 0, acc = 0;
      uint32_t pa = 0, pb = 0, pacc = 0;
      long long pt;
      int nt, q, hf;
      const uint32_t idesc_full = idesc_f16_m256(p.ab_fmt, p.NT), idesc_half = idesc_f16_m256(p.ab_fmt, p.NT / 2);
      int gst = 0;  // trace: global stage index
      if (p.wres && blockIdx.x / 2 < p.units) {  // resident weight tiles
        mbar_wait(&b_full[0], 0);
        tc_fence_after();
      }
      for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
        const uint32_t idesc = hf ? idesc_half : idesc_full;
        mbar_wait(&acc_empty[acc], pacc ^ 1);
        tc_fence_after();
        if (lane == 0) trace_ev(p, 2, k);
        // SPLIT: pass 0 (xh.wh) accumulates into its own columns, passes 1-2 (the
        // ~2^-11 smaller corrections) into the next NT -- the large sum then takes
        // only a third of the non-round-to-nearest accumulation steps
        const uint32_t d = tb + (uint32_t)(acc * p.NT * (p.split ? 2 : p.allq ? 4 : 1));
        if (p.im2col) {
          // Tight issue loop -- one barrier wait, the stage's MMAs, one commit,
          // descriptors advanced by constant strides.  A warp-uniform issue
          // loop costs ~370 cycles per stage before any MMA (wait 80, commit
          // 70, loop / elect / syncwarp ~220: scripts/mma2_bench.cu) and the
          // tensor pipe queues only about one MMA ahead, so a stage must hold
          // more MMA time than that: four N = 256 MMAs (512 cycles) do, four
          // N = 128 ones (276) do not -- hence two k-blocks per stage (kst).
          const int per_pass = p.nkb * p.taps[q];
          const int nst = (p.split ? 3 : 1) * per_pass;
          const uint64_t ad0 = sw128_desc(smem_u32(a_base)), bd0 = sw128_desc(smem_u32(b_base));
          const uint32_t astep = (uint32_t)p.a_stage_bytes >> 4, bstep = (uint32_t)p.b_stage_bytes >> 4;
          int in_pass = 0, pass = 0;
          for (int s = 0; s < nst; ++s) {
            mbar_wait(&a_full[sa], pa);
            tc_fence_after();
            if (lane == 0) trace_ev(p, 6, gst);
            const uint64_t ad = ad0 + (uint64_t)((uint32_t)sa * astep);
            const uint64_t bd = bd0 + (uint64_t)((uint32_t)sa * bstep);
            const uint32_t ds = d + (pass > 0 ? (uint32_t)p.NT : 0u);
            const uint32_t acc0 = (pass <= 1 && in_pass == 0) ? 0u : 1u;
            if (elect_one()) {
              if (p.debug & 8) {  // diagnostics: no MMAs
              } else if (p.tf32) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)  // 4 x (K = 8 fp32) = one 128-byte row
                  mma2_tf32(ds, ad + 2u * ks, bd + 2u * ks, idesc, ks == 0 ? acc0 : 1u);
              } else if (kst == 2) {
                // two 64-channel blocks: A 16 KB, B b_tx apart
#pragma unroll
                for (int ks = 0; ks < KB / 16; ++ks)
                  mma2_bf16(ds, ad + 2u * ks, bd + 2u * ks, idesc, ks == 0 ? acc0 : 1u);
#pragma unroll
                for (int ks = 0; ks < KB / 16; ++ks)
                  mma2_bf16(ds, ad + (p.a_share ? 0u : (16384u >> 4)) + 2u * ks, bd + (b_tx >> 4) + 2u * ks, idesc, 1u);
              } else {
#pragma unroll
                for (int ks = 0; ks < KB / 16; ++ks)
                  mma2_bf16(ds, ad + 2u * ks, bd + 2u * ks, idesc, ks == 0 ? acc0 : 1u);
              }
              commit2(&a_empty[sa]);
            }
            __syncwarp();
            if (lane == 0) trace_ev(p, 8, gst);
            ++gst;
            if (++sa == SA) {
              sa = 0;
              pa ^= 1;
            }
            if (++in_pass == per_pass) {
              in_pass = 0;
              ++pass;
            }
          }
        } else
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&a_full[sa], pa);
          tc_fence_after();
          const uint32_t xa = smem_u32(a_base + (size_t)sa * p.a_stage_bytes);
          for (int qq = p.allq ? 0 : q; qq < (p.allq ? 4 : q + 1); ++qq)
          for (int t = 0; t < p.taps[qq]; ++t) {
            if (!p.wres) {
              mbar_wait(&b_full[sb], pb);
              tc_fence_after();
            }
            const uint32_t wa = p.wres ? smem_u32(b_base) + (uint32_t)((kb * p.tap_base[3] + kb * p.taps[3] +
                                                                        p.tap_base[qq] + t) * NT2 * 128)
                                       : smem_u32(b_base + (size_t)sb * p.b_stage_bytes);
            const uint64_t ad = sw128_desc(xa + (uint32_t)p.shift[qq][t] * 128);
            const uint64_t bd = sw128_desc(wa);
            const uint32_t dq = d + (p.allq ? (uint32_t)(qq * p.NT) : 0u);
            if (!(p.debug & 8) && elect_one()) {
#pragma unroll
              for (int ks = 0; ks < KB / 16; ++ks)  // +32 bytes per K=16 step: +2 in the start field
                mma2_bf16(dq, ad + 2u * ks, bd + 2u * ks, idesc,
                          (kb == 0 && t == 0 && ks == 0) ? 0u : 1u);
            }
            __syncwarp();
            if (p.wres) continue;
            if (elect_one()) commit2(&b_empty[sb]);
            __syncwarp();
            if (++sb == SB) {
              sb = 0;
              pb ^= 1;
            }
          }
          if (elect_one()) commit2(&a_empty[sa]);
          __syncwarp();
          if (++sa == SA) {
            sa = 0;
            pa ^= 1;
          }
        }
        if (elect_one()) commit2(&acc_full[acc]);
        __syncwarp();
        if (lane == 0) trace_ev(p, 3, k);
        if (++acc == NACC) {
          acc = 0;
          pacc ^= 1;
        }
      }
    }
  } else if (warp < 4 && p.mode == 1) {
    // ===== WGRAD epilogue: lane = input channel; 32 features per TMEM load
    const uint32_t lane_base = tmem_base + ((uint32_t)(warp * 32) << 16);
    const uint32_t acc_empty_leader0 = mapa(smem_u32(&acc_empty[0]), 0);
    int acc = 0;
    uint32_t pacc = 0;
    int t, ct, nt, slot;
    long long c0, c1;
    for (int k = 0; wseg_of(p, k, t, ct, nt, c0, c1, slot); ++k) {
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      const int ch = ct * 256 + (int)rank * 128 + warp * 32 + lane;
      const bool ok = ch < p.w_cin;
      float* dst = p.wout + (long long)slot * p.w_ksz +
                   ((long long)t * p.w_cin + (ok ? ch : 0)) * p.w_cout + nt * p.NT;
#pragma unroll 1
      for (int c0 = 0; c0 < p.NT; c0 += 32) {
        float v[32];
        tmem_ld32(lane_base + (uint32_t)(acc * p.NT + c0), v);
        if (!ok) continue;
        float4* o = reinterpret_cast<float4*>(dst + c0);
        if (p.w_direct && p.w_accumulate) {
          if (aligned32(dst + c0)) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float a[8];
              ld_global_v8f(dst + c0 + 8 * e, a);
#pragma unroll
              for (int u = 0; u < 8; ++u) a[u] += v[8 * e + u];
              st_global_v8f(dst + c0 + 8 * e, a);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float4 a = o[e];
              o[e] = make_float4(a.x + v[4 * e], a.y + v[4 * e + 1], a.z + v[4 * e + 2], a.w + v[4 * e + 3]);
            }
          }
        } else if (aligned32(dst + c0)) {
#pragma unroll
          for (int e = 0; e < 4; ++e) st_global_v8f(dst + c0 + 8 * e, &v[8 * e]);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cl_relaxed(acc_empty_leader0 + (uint32_t)acc * 8);
      if (++acc == NACC) {
        acc = 0;
        pacc ^= 1;
      }
    }
  } else if (warp < 4 || (CPS == 1 && warp >= 7 && p.epi8)) {
    // ===== epilogue: lane = anchor; each thread writes its anchor's features
    // (one CTA per SM: two warps per TMEM lane quadrant, alternate column chunks)
    const int qd = warp & 3;
    const bool e8 = CPS == 1 && p.epi8;
    const int c_first = (e8 && warp >= 7) ? 32 : 0, c_step = e8 ? 64 : 32;
    const uint32_t lane_base = tmem_base + ((uint32_t)(qd * 32) << 16);
    const uint32_t acc_empty_leader0 = mapa(smem_u32(&acc_empty[0]), 0);
    const int img = p.n * p.n;
    int acc = 0;
    uint32_t pacc = 0;
    long long pt;
    int nt, q, hf;
    for (int k = 0; unit_of(p, k, pt, nt, q, hf); ++k) {
      mbar_wait(&acc_full[acc], pacc);
      tc_fence_after();
      if (threadIdx.x == 0 && rank == 0) trace_ev(p, 4, k);
      int b, i, j;
      bool in_range;
      if (p.im2col) {
        const int R = p.rows[q], C = p.cols[q];
        const long long a = pt * 256 + (long long)rank * 128 + qd * 32 + lane;
        b = (int)(a / ((long long)R * C));
        const int rem = (int)(a - (long long)b * R * C);
        i = rem / C;
        j = rem - (rem / C) * C;
        in_range = b < p.batch;
      } else if (p.tile2d) {
        const long long g = pt * 2 + rank;
        b = (int)(g / p.tiles_per_img);
        const int trc = (int)(g - (long long)b * p.tiles_per_img);
        const int trow = trc / p.col_tiles, tcol = trc - trow * p.col_tiles;
        const int t = qd * 32 + lane, jj = t % p.BW;
        i = trow * p.TR + t / p.BW;
        j = tcol * p.BWo + jj;
        in_range = b < p.batch && t < p.TR * p.BW && jj < p.BWo;
      } else {
        const long long m = pt * 256 + (long long)rank * 128 + qd * 32 + lane;
        b = (int)(m / img);
        const int rem = (int)(m - (long long)b * img);
        i = rem / p.n;
        j = rem - (rem / p.n) * p.n;
        in_range = m < p.Mv;
      }
      for (int qq = p.allq ? 0 : q; qq < (p.allq ? 4 : q + 1); ++qq) {
      const int r = qq >> 1, c = qq & 1;
      const int fbase = nt * p.NT + (hf ? (hf - 1) * (p.NT / 2) : 0);
      const bool ok = in_range && i < p.rows[qq] && j < p.cols[qq] && !(p.debug & 1);
      const uint32_t cbase = (uint32_t)(acc * p.NT * (p.split ? 2 : p.allq ? 4 : 1) + (p.allq ? qq * p.NT : 0));
      YT* dst = reinterpret_cast<YT*>(p.y) +
                ((long long)((long long)b * p.out_h + p.ostride * i + r) * p.out_w + p.ostride * j + c) *
                    p.cout +
                fbase;
      const int fmax = p.cout - fbase;  // features of this tile that exist
      const float osc = (p.split || p.oscale) ? __ldg(p.split_inv_scale) : 1.0f;
#pragma unroll 1
      for (int c0 = c_first; c0 < ((p.debug & 4) ? 0 : hf ? p.NT / 2 : p.NT); c0 += c_step) {  // 4: diagnostics, no epilogue
        float v[32];
        tmem_ld32(lane_base + cbase + (uint32_t)c0, v);
        if (p.split) {
          float w2[32];
          tmem_ld32(lane_base + (uint32_t)(acc * p.NT * 2 + p.NT + c0), w2);
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = (v[e] + w2[e]) * osc;  // scale: exact power of two
        } else if (p.oscale) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] *= osc;
        }
        if (!ok || c0 >= fmax) continue;
        if (c0 + 32 <= fmax) {
          if constexpr (sizeof(YT) == 2) {
            uint32_t w[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int f = fbase + c0 + 2 * e;
              const __nv_bfloat162 h = __floats2bfloat162_rn(finish_bf<ACT>(v[2 * e], p.bias, p.epi, f),
                                                             finish_bf<ACT>(v[2 * e + 1], p.bias, p.epi, f + 1));
              w[e] = *reinterpret_cast<const uint32_t*>(&h);
            }
            if (aligned32(dst + c0)) {
              // 256-bit stores (sm_100 STG.256): half the store instructions of
              // the scattered per-anchor epilogue writes
#pragma unroll
              for (int e = 0; e < 2; ++e) st_global_v8(dst + c0 + 16 * e, &w[8 * e]);
            } else {
              uint4* o = reinterpret_cast<uint4*>(dst + c0);
#pragma unroll
              for (int e = 0; e < 4; ++e) o[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = finish<ACT>(v[e], p.bias, p.epi, fbase + c0 + e);
            if (aligned32(dst + c0)) {
#pragma unroll
              for (int e = 0; e < 4; ++e) st_global_v8f(reinterpret_cast<float*>(dst + c0 + 8 * e), &v[8 * e]);
            } else {
              float4* o = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (c0 + e < fmax)
              dst[c0 + e] = from_f<YT>(sizeof(YT) == 2 ? finish_bf<ACT>(v[e], p.bias, p.epi, fbase + c0 + e)
                                                       : finish<ACT>(v[e], p.bias, p.epi, fbase + c0 + e));
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0 && rank == 0) trace_ev(p, 5, k);  // epilogue of the unit done (warp 0)
      if (lane == 0) mbar_arrive_cl_relaxed(acc_empty_leader0 + (uint32_t)acc * 8);
      if (++acc == NACC) {
        acc = 0;
        pacc ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the pair's MMAs and remote arrivals are over before TMEM is freed
  if (threadIdx.x == 0) trace_ev(p, 13, 0);
  if (warp == 6) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CPS == 2 ? 256 : 512)
                 : "memory");
  }
}

}  // namespace tcw

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFnW)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFnW encode_fn_w() {
  // magic static: thread-safe one-time lookup of the driver entry point
  static const EncodeTiledFnW fn = [] {
    EncodeTiledFnW fn = nullptr;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFnW)f;
    return fn;
  }();
  return fn;
}

typedef CUresult (*EncIm2colW)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncIm2colW encode_im2col_w() {
  // magic static: thread-safe one-time lookup of the driver entry point
  static const EncIm2colW fn = [] {
    EncIm2colW fn = nullptr;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncIm2colW)f;
    return fn;
  }();
  return fn;
}

// features per pair tile: the whole (32-padded) cout up to 256
int tc_wide_ntile(int cout) {
  const int c32 = (cout + 31) / 32 * 32;
  return std::min(256, c32);
}

// Must agree with make_wide (the KMAJOR panels it implies have no other consumer):
// every class has taps, at most MAX_TAPS_Q of them, and the im2col walk's
// corner offsets (-p_fused .. ) fit the rank-4 range [-128, 127].
bool tc_wide_fits(int kh, int kw, int p, int cin, int cout) {
  // narrow outputs (e.g. the 3-channel last layer of a GAN generator at p = 2,
  // which the folded / scatter kernels do not take) run with a 32-wide
  // feature tile: the MMA idles on the padding, the layer is bound by its
  // activation reads anyway
  if (cin % tcw::KB != 0 || cout < 1 || p < 0 || p / 2 > 120) return false;
  int ah[2], aw[2];
  for (int r = 0; r < 2; ++r) {
    const int u0 = (p + r) & 1;
    ah[r] = u0 >= kh ? 0 : (kh - u0 + 1) / 2;
    aw[r] = u0 >= kw ? 0 : (kw - u0 + 1) / 2;
    if (ah[r] == 0 || aw[r] == 0) return false;
  }
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c)
      if (ah[r] * aw[c] > tcw::MAX_TAPS_Q) return false;
  return true;
}

// xs: the [hi | lo] fp16 copy of an fp32 input (SPLIT); any aligned pointer
// when only checking support
// A and B streams on two producer lanes (measured: C3 81.3 -> 78.9 us)
static int wide_bprod() { return 1; }

static int wide_pairs();

static int wide_debug_bits() {
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  return dbg;
}
static bool make_wide(const FusedProblem& pr, tcw::Params& p, tcw::Maps& maps, const void* xs = nullptr) {
  p = tcw::Params{};
  const bool split = pr.x_dtype == SEGCONV_F32 && pr.panel_dtype == SEGCONV_F16_SPLIT;
  const bool tf32 = pr.x_dtype == SEGCONV_F32 && pr.panel_dtype == SEGCONV_F32;
  if (!split && !tf32 && (pr.x_dtype != SEGCONV_BF16 || pr.panel_dtype != SEGCONV_BF16)) return false;
  if (pr.panel_layout != SEGCONV_PANEL_KMAJOR) return false;
  if (split && !xs) return false;
  p.split = split ? 1 : 0;
  p.tf32 = tf32 ? 1 : 0;
  p.kbc = tf32 ? 32 : tcw::KB;
  const int esz = tf32 ? 4 : 2;  // operand element bytes
  p.split_off = pr.cin;
  if (split) {  // the scale slot follows the K-major panels: 4 classes x cout_pad x taps x 2 cin fp16
    long long main = 0;
    for (int q = 0; q < 4; ++q) main += (long long)pr.cls.kh[q] * pr.cls.kw[q] * 2 * pr.cin * pr.cout_pad;
    p.split_inv_scale = reinterpret_cast<const float*>(reinterpret_cast<const __half*>(pr.panels) + main) + 1;
  }
  p.ab_fmt = tf32 ? 2u : split ? 0u : 1u;  // instruction-descriptor operand format: tf32 / f16 / bf16
  const int kc = split ? 2 * pr.cin : pr.cin;  // channels of the staged tensors
  const void* xsrc = split ? xs : pr.x;
  const CUtensorMapDataType op_type = tf32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                      : split ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if (pr.y_dtype != SEGCONV_BF16 && pr.y_dtype != SEGCONV_F32) return false;
  if (!tc_wide_fits(pr.kh, pr.kw, pr.p, pr.cin, pr.cout)) return false;
  p.wscale = 1;
  p.wbase_r = p.wbase_c = -pr.pf;
  p.ostride = 2;
  p.y = pr.y;
  p.bias = pr.bias;
  p.epi = pr.epi;
  p.y_dtype = pr.y_dtype;
  p.batch = pr.batch;
  p.n = pr.n;
  p.cin = pr.cin;
  p.cout = pr.cout;
  p.out_h = pr.out_h;
  p.out_w = pr.out_w;
  p.Mv = (long long)pr.batch * pr.n * pr.n;
  p.NT = split ? std::min(128, tc_wide_ntile(pr.cout)) : tc_wide_ntile(pr.cout);  // SPLIT: 2 accumulators
  {
    // small batches of small maps (GAN generators' first layers): fewer 256-wide
    // units than CTA pairs leaves SMs idle -- halve the feature tile when the
    // doubled unit count still fits one wave (DCGAN 4x4 x 1024 -> 512: 34.8 -> 32.2 us)
    long long u = 0;
    for (int q = 0; q < 4; ++q) u += ((long long)pr.batch * pr.cls.rows[q] * pr.cls.cols[q] + 255) / 256;
    if (p.NT > 128 && 2 * u * ((pr.cout + p.NT - 1) / p.NT) <= wide_pairs()) p.NT = 128;
  }
  p.n_tiles = (pr.cout + p.NT - 1) / p.NT;
  if (p.n_tiles * p.NT > pr.cout_pad && p.n_tiles > 1) {
    // the last tile may run past cout_pad: the TMA box is zero-filled out of bounds
  }
  p.nkb = pr.cin / p.kbc;
  p.pf = pr.pf;
  p.tile2d = pr.pf > 0 ? 1 : 0;
  p.VW = pr.n + 2 * pr.pf;  // pitch of the staged rows (the padded grid in TILE2D)
  int max_shift = 0, max_dy = 0, max_dx = 0;
  for (int q = 0; q < 4; ++q) {
    p.taps[q] = pr.cls.kh[q] * pr.cls.kw[q];
    if (p.taps[q] > tcw::MAX_TAPS_Q) return false;
    for (int u = 0; u < pr.cls.kh[q]; ++u)
      for (int v = 0; v < pr.cls.kw[q]; ++v) {
        max_dy = std::max(max_dy, pr.cls.off_r[q] + u);
        max_dx = std::max(max_dx, pr.cls.off_c[q] + v);
      }
    p.rows[q] = pr.cls.rows[q];
    p.cols[q] = pr.cls.cols[q];
  }
  // IM2COL: GEMM rows are only output anchors (the halo-shift grid computes
  // every virtual position: C5 a 44 %, b 54 %, c 65 %, C3 77 % useful rows)
  {
    long long useful = 0, taps = 0;
    for (int q = 0; q < 4; ++q) {
      useful += (long long)pr.cls.rows[q] * pr.cls.cols[q] * p.taps[q];
      taps += p.taps[q];
    }
    const double eff = (double)useful / ((double)p.VW * p.VW * taps);
    (void)eff;
    // measured (B200, bench.py): im2col beats the halo-shift staging on every
    // BASELINE shape -- C3 89.7 -> 79.9 us (78 % useful rows), C5 237 -> 138 us
    // -- the extra per-tap A gathers are L2 hits, the saved MMA rows are not
    p.im2col = 1;
    // narrow outputs (<= 64 features) on large padded maps: stage each block of
    // rows once and run all four classes' taps on it as shifted descriptors (4
    // accumulators, ALLQ) instead of re-gathering the block per (class, tap) --
    // measured (B200, batch 64, 4x4, p = 2): 128^2 x 64 -> 64 561 -> 365 us,
    // 64^2 x 64 -> 64 152 -> 106 us; at 32^2 the im2col walk is still faster
    if (!split && !tf32 && p.tile2d && tc_wide_ntile(pr.cout) <= 64 && pr.n >= 64) p.im2col = 0;
    p.bprod = p.im2col ? wide_bprod() : 0;
  }
  // halo-shift staging (SEGCONV_WIDE_IM2COL=0) limits: the staged rows must fit
  // one TMA box; they do not constrain the im2col path (e.g. 128 x 128 maps)
  if (!p.im2col) {
    if (p.tile2d) {
      // column blocks of BW staged columns (the row pitch), BWo = BW - max_dx anchors
      // each (the rest read the next block's columns); BW = VW is one block per row.
      // Pick the width that needs the fewest 128-row tiles.
      const int vh = std::max(pr.cls.rows[0], pr.cls.rows[2]);
      const int vw = std::max(pr.cls.cols[0], pr.cls.cols[1]);
      long long best = -1;
      for (int bw : {p.VW, 128, 64, 32, 16}) {
        if (bw > p.VW || bw > 128 || (bw < p.VW && bw - max_dx < 8)) continue;
        const int bwo = bw == p.VW ? p.VW : bw - max_dx;
        const int tr = 128 / bw, ct = (vw + bwo - 1) / bwo;
        const int trh = tr + max_dy + 1;  // + one row: shifted reads of the last anchors wrap a row
        if (trh > 256 || bw * trh > 384) continue;
        const long long tiles = (long long)((vh + tr - 1) / tr) * ct;
        if (best < 0 || tiles < best) {
          best = tiles;
          p.BW = bw, p.BWo = bwo, p.TR = tr, p.col_tiles = ct, p.TRH = trh;
        }
      }
      if (best < 0) return false;
      p.tiles_per_img = (int)best;
      p.S_rows = p.BW * p.TRH;
    }
  }
  for (int q = 0; q < 4; ++q)  // halo shifts: row offset x staged pitch + column offset
    for (int u = 0; u < pr.cls.kh[q]; ++u)
      for (int v = 0; v < pr.cls.kw[q]; ++v) {
        const int pitch = p.tile2d ? p.BW : pr.n;
        const int sh = (pr.cls.off_r[q] + u) * pitch + (pr.cls.off_c[q] + v);
        p.shift[q][u * pr.cls.kw[q] + v] = sh;
        max_shift = std::max(max_shift, sh);
      }
  if (!p.im2col && !p.tile2d) {
    p.S_rows = (128 + max_shift + 7) / 8 * 8;
    if (p.S_rows > 256) return false;  // one TMA box
  }
  {
    p.allq = (!p.im2col && p.NT <= 128) ? 1 : 0;
    p.nacc = p.allq && 4 * p.NT > 256 ? 1 : 2;
    p.wres = (p.allq && p.n_tiles == 1) ? 1 : 0;
    p.bprod = (!p.im2col && !p.wres) ? wide_bprod() : p.bprod;
    int tb = 0;
    for (int q = 0; q < 4; ++q) {
      p.tap_base[q] = tb;
      tb += p.taps[q];
    }
  }
  if (p.im2col) {
    p.tile2d = 0;
    p.S_rows = 128;
    for (int q = 0; q < 4; ++q)
      for (int u = 0; u < pr.cls.kh[q]; ++u)
        for (int v = 0; v < pr.cls.kw[q]; ++v) {
          p.tap_off_r[q][u * pr.cls.kw[q] + v] = pr.cls.off_r[q] + u;
          p.tap_off_c[q][u * pr.cls.kw[q] + v] = pr.cls.off_c[q] + v;
        }
  }
  p.a_stage_bytes = (p.S_rows * 128 + 1023) / 1024 * 1024;
  p.b_stage_bytes = (p.NT / 2) * 128;
  if (p.b_stage_bytes % 1024) return false;
  const int bar_bytes = (2 * tcw::MAX_STAGES_A + 2 * tcw::MAX_STAGES_B + 4) * 8 + 16;
  int budget = tcw::SMEM_LIMIT - bar_bytes;
  if (p.im2col) {  // A and B both per (k-block, tap): paired rings
    // two 64-channel k-blocks per stage where cin allows: the producer / MMA
    // handshake costs a few hundred cycles per stage whatever its size, as
    // much as a stage of N = 128 MMAs (measured: the empty pipeline alone,
    // no loads / MMAs / epilogue, takes 27 us for C5 layer c at one k-block
    // per stage)
    // narrow feature tiles: two CTAs (two pipelines) per SM, 256 TMEM columns
    // each -- one CTA's per-stage handshakes run under the other's MMAs
    // (measured: C5 layer c 39.6 -> 35.1-37.3 us; the same for NT = 256 with one
    // accumulator per CTA made C3 77 -> 92 us)
    // only when the units fill twice as many CTA pairs (small batches keep one
    // pipeline with the whole ring: C5 at 128 images 50.8 -> 63.4 us otherwise)
    long long units = 0;
    for (int q = 0; q < 4; ++q)
      units += ((long long)pr.batch * pr.cls.rows[q] * pr.cls.cols[q] + 255) / 256 * p.n_tiles;
    p.cps = (!split && !tf32 && p.mode == 0 && p.NT <= 128 && units >= 4LL * wide_pairs()) ? 2 : 1;
    if (p.cps == 2) budget = tcw::SMEM_PER_CTA2 - bar_bytes;
    p.kstage = (p.cps == 1 && !split && !tf32 && p.mode == 0 && pr.cin % (2 * tcw::KB) == 0 &&
                2 * (p.a_stage_bytes + p.b_stage_bytes) * 3 <= budget) ? 2 : 1;
    p.nkb = pr.cin / (p.kbc * p.kstage);
    // eight epilogue warps where some class's units are short (< 12 stages), so
    // a unit's epilogue would outlast the MMAs of the next: C5 115.7 vs 117.3 us;
    // with only long units (C3: 16 stages each) four are faster (76.7 vs 77.2 us)
    {
      int min_st = 1 << 30;
      for (int q = 0; q < 4; ++q) min_st = std::min(min_st, p.taps[q] * p.nkb * (split ? 3 : 1));
      p.epi8 = (p.cps == 1 && p.mode == 0 && min_st < 12 && !(wide_debug_bits() & 256)) ? 1 : 0;  // debug 256: four
    }
    p.a_stage_bytes *= p.kstage;
    p.b_stage_bytes *= p.kstage;
    p.stages_a = p.stages_b = std::min(tcw::MAX_STAGES_A, budget / (p.a_stage_bytes + p.b_stage_bytes));
    if (p.stages_a < 2) return false;
  } else if (p.wres) {  // one "stage" holding every weight tile, A ring in the rest
    p.b_stage_bytes *= p.nkb * (p.tap_base[3] + p.taps[3]);
    p.stages_b = 1;
    p.stages_a = std::min(tcw::MAX_STAGES_A, (budget - p.b_stage_bytes) / p.a_stage_bytes);
    if (p.stages_a < 2) p.wres = 0, p.b_stage_bytes = (p.NT / 2) * 128, p.bprod = wide_bprod();
  }
  if (!p.im2col && !p.wres) {
    p.stages_a = 3;
    p.stages_b = std::min(tcw::MAX_STAGES_B, (budget - p.stages_a * p.a_stage_bytes) / p.b_stage_bytes);
    if (p.stages_b < 4) {
      p.stages_a = 2;
      p.stages_b = std::min(tcw::MAX_STAGES_B, (budget - p.stages_a * p.a_stage_bytes) / p.b_stage_bytes);
    }
    if (p.stages_b < 2) return false;
  }
  if (p.im2col) {
    p.unit_base[0] = 0;
    for (int q = 0; q < 4; ++q) {
      const long long aq = (long long)pr.batch * pr.cls.rows[q] * pr.cls.cols[q];
      p.unit_base[q + 1] = p.unit_base[q] + (aq + 255) / 256 * p.n_tiles;
    }
    p.units = p.unit_base[4];
    p.pair_tiles = 0;
  } else {
    p.pair_tiles = p.tile2d ? ((long long)pr.batch * p.tiles_per_img + 1) / 2 : (p.Mv + 255) / 256;
    p.units = p.pair_tiles * p.n_tiles * (p.allq ? 1 : 4);
  }
  if ((long long)pr.batch * pr.out_h * pr.out_w * pr.cout >= (1LL << 40)) return false;
  // tensor maps
  EncodeTiledFnW fn = encode_fn_w();
  if (!fn) return false;
  if (p.tile2d) {
    const cuuint64_t dims[4] = {(cuuint64_t)kc, (cuuint64_t)pr.n, (cuuint64_t)pr.n,
                                (cuuint64_t)pr.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)kc * esz, (cuuint64_t)pr.n * kc * esz,
                                   (cuuint64_t)pr.n * pr.n * kc * esz};
    const cuuint32_t box[4] = {(cuuint32_t)p.kbc, (cuuint32_t)p.BW, (cuuint32_t)p.TRH, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (fn(&maps.x, op_type, 4, const_cast<void*>(xsrc), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  } else {
    const cuuint64_t dims[2] = {(cuuint64_t)kc, (cuuint64_t)p.Mv};
    const cuuint64_t strides[1] = {(cuuint64_t)kc * esz};
    const cuuint32_t box[2] = {(cuuint32_t)p.kbc, (cuuint32_t)p.S_rows};
    const cuuint32_t es[2] = {1, 1};
    if (fn(&maps.x, op_type, 2, const_cast<void*>(xsrc), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  if (p.im2col) {
    typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                  cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncIm2col enc2 = nullptr;
    if (!enc2) {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult qr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &qr) !=
              cudaSuccess ||
          qr != cudaDriverEntryPointSuccess)
        return false;
      enc2 = (EncIm2col)f;
    }
    const cuuint64_t dims[4] = {(cuuint64_t)kc, (cuuint64_t)pr.n, (cuuint64_t)pr.n,
                                (cuuint64_t)pr.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)kc * esz, (cuuint64_t)pr.n * kc * esz,
                                   (cuuint64_t)pr.n * pr.n * kc * esz};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    for (int q = 0; q < 4; ++q) {
      // walk origins (anchor - p_fused) over [-pf, C-1-pf] x [-pf, R-1-pf] of every image
      const int lower[2] = {-pr.pf, -pr.pf};
      const int upper[2] = {pr.cls.cols[q] - pr.pf - pr.n, pr.cls.rows[q] - pr.pf - pr.n};
      if (enc2(&maps.xi[q], op_type, 4, const_cast<void*>(xsrc), dims,
               strides, lower, upper, (cuuint32_t)p.kbc, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    }
  }
  for (int q = 0; q < 4; ++q) {
    const cuuint64_t dims[3] = {(cuuint64_t)kc, (cuuint64_t)p.taps[q], (cuuint64_t)pr.cout_pad};
    const cuuint64_t strides[2] = {(cuuint64_t)kc * esz, (cuuint64_t)p.taps[q] * kc * esz};
    const cuuint32_t box[3] = {(cuuint32_t)p.kbc, 1, (cuuint32_t)(p.NT / 2)};
    const cuuint32_t es[3] = {1, 1, 1};
    void* base = (char*)const_cast<void*>(pr.panels) + pr.cls.sub_offset[q] * esz;
    if (fn(&maps.w[q], op_type, 3, base, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    if (p.im2col && p.mode == 0 && !split && p.NT == 256) {  // feature-half units (balanced schedule)
      const cuuint32_t hbox[3] = {(cuuint32_t)p.kbc, 1, (cuuint32_t)(p.NT / 4)};
      if (fn(&maps.wh[q], op_type, 3, base, dims, strides, hbox, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
      p.wh_ok = q == 3 ? 1 : 0;
    }
  }
  return true;
}

// Input gradient of the fused layer (reference netdemo/layers.hpp:171-211) on
// the same pair kernel: gx[m, ch] = sum_{U,V,f} gy[b, 2i+p-U, 2j+p-V, f] k[U,V,ch,f]
// is one "class" whose K loop runs over every tap (U, V) and cout in 64-feature
// blocks.  A = a stride-2 im2col walk over gy (origin (2i + p-kh+1, 2j + p-kw+1),
// tap offset (kh-1-U, kw-1-V); positions outside gy are zero-filled by the TMA),
// B = the original kernel, whose (U, V, ch, f) layout is already K-major for
// N = ch -- no flipped or re-laid-out copy is made.
// Input gradient on the pair kernel (stride-2 im2col walk over gy).  bf16: gy
// and the kernel as they are.  Split fp16 (fp32 data, f16x3, cout = 32):
// gy16 = gy's [hi | lo] halves as 64 channels (scaled by 2^t) and per tap
// w2 = [wh | wh | wl | 0] (scaled by 2^s): one stage per tap multiplies its A
// box by both 64-channel B halves, gh.wh + gl.wh + gh.wl; gx = 2^-s-t (sum).
static bool make_wide_dgrad(const BackwardProblem& pr, tcw::Params& p, tcw::Maps& maps,
                            const void* gy16 = nullptr, const void* w2 = nullptr) {
  p = tcw::Params{};
  const bool split = gy16 != nullptr;
  p.ab_fmt = split ? 0 : 1;  // fp16 / bf16 operands
  p.kbc = tcw::KB;
  if (pr.dtype != (split ? SEGCONV_F32 : SEGCONV_BF16)) return false;
  const int kch = split ? 2 * pr.cout : pr.cout;  // A (gy) channels per tap
  if (kch % tcw::KB != 0 || pr.cin < 64 || pr.cin % 8 != 0) return false;
  if (split && kch != tcw::KB) return false;  // one A box of [hi | lo] per tap (cout = 32)
  const int taps = pr.kh * pr.kw;
  if (taps > tcw::MAX_TAPS_Q) return false;
  // walk origin of input pixel (i, j): (stride*i + lo_r, stride*j + lo_c); the
  // corners bound the walk: [lo, stride*(in-1) + lo] in gy coordinates
  const int lo_r = pr.p - pr.kh + 1, lo_c = pr.p - pr.kw + 1;
  const int up_r = pr.stride * (pr.in_h - 1) + lo_r - (pr.out_h - 1);
  const int up_c = pr.stride * (pr.in_w - 1) + lo_c - (pr.out_w - 1);
  if (lo_r < -128 || lo_c < -128 || up_r < -128 || up_c < -128 || up_r > 127 || up_c > 127 || lo_r > 127 ||
      lo_c > 127)
    return false;  // rank-4 im2col corner range
  if ((long long)pr.batch * pr.in_h * pr.in_w * pr.cin >= (1LL << 40)) return false;
  p.y = pr.gx;
  p.y_dtype = split ? SEGCONV_F32 : SEGCONV_BF16;
  p.batch = pr.batch;
  p.n = pr.in_h;
  p.cin = split ? 2 * kch : kch;  // GEMM K channels
  p.cout = pr.cin;  // GEMM N: input-gradient channels
  p.out_h = pr.in_h;
  p.out_w = pr.in_w;
  p.Mv = (long long)pr.batch * pr.in_h * pr.in_w;
  p.NT = tc_wide_ntile(pr.cin);
  p.n_tiles = (pr.cin + p.NT - 1) / p.NT;
  // split: one stage per tap, its A box [gh | gl] multiplied by the two B
  // halves [wh | wh] and [wl | 0] (two k-blocks, one A box)
  p.kstage = split ? 2 : 1;
  p.a_share = split ? 1 : 0;
  p.nkb = split ? 1 : kch / tcw::KB;
  p.im2col = 1;
  p.bprod = wide_bprod();
  p.S_rows = 128;
  p.taps[0] = taps;
  for (int U = 0; U < pr.kh; ++U)
    for (int V = 0; V < pr.kw; ++V) {
      p.tap_off_r[0][U * pr.kw + V] = pr.kh - 1 - U;
      p.tap_off_c[0][U * pr.kw + V] = pr.kw - 1 - V;
    }
  p.rows[0] = pr.in_h;
  p.cols[0] = pr.in_w;
  p.wscale = pr.stride;
  p.wbase_r = lo_r;
  p.wbase_c = lo_c;
  p.ostride = 1;
  p.b_tap_last = 1;
  p.a_stage_bytes = 128 * 128;
  p.b_stage_bytes = (p.NT / 2) * 128 * p.kstage;
  if (p.b_stage_bytes % 1024) return false;
  const int bar_bytes = (2 * tcw::MAX_STAGES_A + 2 * tcw::MAX_STAGES_B + 4) * 8 + 16;
  p.stages_a = p.stages_b =
      std::min(tcw::MAX_STAGES_A, (tcw::SMEM_LIMIT - bar_bytes) / (p.a_stage_bytes + p.b_stage_bytes));
  if (p.stages_a < 2) return false;
  p.unit_base[0] = 0;
  const long long u1 = (p.Mv + 255) / 256 * p.n_tiles;
  for (int q = 1; q <= 4; ++q) p.unit_base[q] = u1;
  p.units = u1;
  EncodeTiledFnW fn = encode_fn_w();
  if (!fn) return false;
  typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncIm2col enc2 = nullptr;
  if (!enc2) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return false;
    enc2 = (EncIm2col)f;
  }
  const CUtensorMapDataType op = split ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)kch, (cuuint64_t)pr.out_w, (cuuint64_t)pr.out_h,
                                (cuuint64_t)pr.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)kch * 2, (cuuint64_t)pr.out_w * kch * 2,
                                   (cuuint64_t)pr.out_h * pr.out_w * kch * 2};
    // walk: origins lo, lo + stride, ... (in_h x in_w per image); corners {W, H}
    const int lower[2] = {lo_c, lo_r};
    const int upper[2] = {up_c, up_r};
    const cuuint32_t es[4] = {1, (cuuint32_t)pr.stride, (cuuint32_t)pr.stride, 1};
    if (enc2(&maps.xi[0], op, 4, const_cast<void*>(split ? gy16 : pr.gy), dims, strides, lower,
             upper, (cuuint32_t)tcw::KB, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    const int bch = p.cin;  // B channels per (tap, input channel): 2 kch for the split
    const cuuint64_t dims[3] = {(cuuint64_t)bch, (cuuint64_t)pr.cin, (cuuint64_t)taps};
    const cuuint64_t strides[2] = {(cuuint64_t)bch * 2, (cuuint64_t)pr.cin * bch * 2};
    const cuuint32_t box[3] = {(cuuint32_t)tcw::KB, (cuuint32_t)(p.NT / 2), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (fn(&maps.w[0], op, 3, const_cast<void*>(split ? w2 : pr.k), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  // every map the kernel prefetches must be valid
  maps.x = maps.xi[0];
  for (int q = 1; q < 4; ++q) {
    maps.w[q] = maps.w[0];
    maps.xi[q] = maps.xi[0];
  }
  return true;
}

// Kernel gradient (reference layers.hpp:196-199: gw[f] += ip[ch] * gp[f]) on the
// pair kernel, mode 1: gk[t, ch, f] = sum_m x[m, ch] gy[b, 2i+p-U, 2j+p-V, f],
// M = 256 channels per pair x N = 128/256 features, K = pixels in 64-pixel
// chunks, both operands MN-major SW128.  The pixel reduction is split so the
// units fill the pairs evenly; splits > 1 write fp32 partials that
// launch_wgrad_reduce sums in split order (deterministic).
static bool make_wide_wgrad(const BackwardProblem& pr, tcw::Params& p, tcw::Maps& maps, int pairs) {
  p = tcw::Params{};
  p.bprod = wide_bprod();
  p.ab_fmt = 1;  // bf16 operands
  p.kbc = tcw::KB;
  if (pr.dtype != SEGCONV_BF16 || pr.batch < 1) return false;
  if (pr.cin % 128 != 0 || pr.cout % 128 != 0) return false;
  const int taps = pr.kh * pr.kw;
  if (taps > tcw::MAX_TAPS_Q) return false;
  const int lo_r = pr.p - pr.kh + 1, lo_c = pr.p - pr.kw + 1;
  const int up_r = pr.stride * (pr.in_h - 1) + lo_r - (pr.out_h - 1);
  const int up_c = pr.stride * (pr.in_w - 1) + lo_c - (pr.out_w - 1);
  if (lo_r < -128 || lo_c < -128 || up_r < -128 || up_c < -128 || up_r > 127 || up_c > 127 || lo_r > 127 ||
      lo_c > 127)
    return false;
  const long long M = (long long)pr.batch * pr.in_h * pr.in_w;
  if (M + 64 >= (1LL << 31)) return false;
  p.mode = 1;
  p.n = pr.in_h;
  p.w_in_h = pr.in_h;
  p.w_in_w = pr.in_w;
  p.wscale = pr.stride;
  p.batch = pr.batch;
  p.NT = pr.cout % 256 == 0 ? 256 : 128;
  p.n_tiles = pr.cout / p.NT;
  p.w_kw = pr.kw;
  p.w_taps = taps;
  p.w_ch_pairs = (pr.cin + 255) / 256;
  p.w_cin = pr.cin;
  p.w_cout = pr.cout;
  p.w_ksz = (long long)taps * pr.cin * pr.cout;
  p.w_accumulate = pr.accumulate;
  p.wbase_r = lo_r;
  p.wbase_c = lo_c;
  for (int U = 0; U < pr.kh; ++U)
    for (int V = 0; V < pr.kw; ++V) {
      p.tap_off_r[0][U * pr.kw + V] = pr.kh - 1 - U;
      p.tap_off_c[0][U * pr.kw + V] = pr.kw - 1 - V;
    }
  p.w_chunks = (M + tcw::WCH - 1) / tcw::WCH;
  // splits: minimise modelled time = waves x chunks per unit x t_chunk + the
  // split-K round trip of the partials (write + reduce read, ~5 TB/s, + launch);
  // t_chunk ~ 0.6 us for a 256 x 256 x 64 pair chunk (measured, B200)
  const long long base = (long long)taps * p.w_ch_pairs * p.n_tiles;
  const double t_chunk = 0.6 * p.NT / 256.0 * tcw::WCH / 64.0;
  const double t_split = (double)taps * pr.cin * pr.cout * 8.0 / 5e6;  // us per split
  int best = 1;
  double best_t = 1e300;
  for (int sp = 1; sp <= 64; ++sp) {
    if (sp > 1 && p.w_chunks / sp < 8) break;
    const long long units = base * sp;
    const long long waves = (units + pairs - 1) / pairs;
    const double t = (double)waves * (double)((p.w_chunks + sp - 1) / sp) * t_chunk +
                     (sp > 1 ? sp * t_split + 3.0 : 0.0);
    if (t < best_t * 0.98) {
      best_t = t;
      best = sp;
    }
  }
  p.w_cps = (p.w_chunks + best - 1) / best;
  p.w_splits = (int)((p.w_chunks + p.w_cps - 1) / p.w_cps);
  p.w_direct = p.w_splits == 1;
  p.units = base * p.w_splits;
  p.a_stage_bytes = 2 * tcw::WCH * 128;
  p.b_stage_bytes = (p.NT / 2 / 64) * tcw::WCH * 128;
  const int bar_bytes = (2 * tcw::MAX_STAGES_A + 2 * tcw::MAX_STAGES_B + 4) * 8 + 16;
  p.stages_a = p.stages_b =
      std::min(tcw::MAX_STAGES_A, (tcw::SMEM_LIMIT - bar_bytes) / (p.a_stage_bytes + p.b_stage_bytes));
  EncodeTiledFnW fn = encode_fn_w();
  if (!fn) return false;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)pr.cin, (cuuint64_t)M};
    const cuuint64_t strides[1] = {(cuuint64_t)pr.cin * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)tcw::WCH};
    const cuuint32_t es[2] = {1, 1};
    if (fn(&maps.x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pr.x), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  EncIm2colW enc2 = encode_im2col_w();
  if (!enc2) return false;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)pr.cout, (cuuint64_t)pr.out_w, (cuuint64_t)pr.out_h,
                                (cuuint64_t)pr.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)pr.cout * 2, (cuuint64_t)pr.out_w * pr.cout * 2,
                                   (cuuint64_t)pr.out_h * pr.out_w * pr.cout * 2};
    const int lower[2] = {lo_c, lo_r};
    const int upper[2] = {up_c, up_r};
    const cuuint32_t es[4] = {1, (cuuint32_t)pr.stride, (cuuint32_t)pr.stride, 1};
    if (enc2(&maps.xi[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(pr.gy), dims, strides, lower,
             upper, 64, (cuuint32_t)tcw::WCH, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  for (int q = 0; q < 4; ++q) {
    maps.w[q] = maps.x;
    if (q) maps.xi[q] = maps.xi[0];
  }
  return true;
}

static int wide_pairs() {
  const int sms = device_sm_count();
  return sms / 2;
}

bool tc_bwd_weight_supported(const BackwardProblem& pr) {
  tcw::Params p;
  tcw::Maps m;
  return make_wide_wgrad(pr, p, m, wide_pairs());
}

// Valid correlation (reference reference_ops.hpp:86-102, conv2d_valid) on the
// pair kernel: one class, every tap (u, v) an im2col offset of the stride-1 walk
// over the output pixels; B = the kernel transposed to (cout, tap, cin) K-major
// (launch_kmajor_transpose); bias / ReLU / tanh epilogue as the fused op.
static bool make_wide_conv(const void* src, int batch, int h, int w, int cin, const void* kt, int kh, int kw,
                           int cout, const float* bias, unsigned epi, void* y, tcw::Params& p, tcw::Maps& maps) {
  p = tcw::Params{};
  p.ab_fmt = 1;  // bf16 operands
  p.kbc = tcw::KB;
  const int taps = kh * kw;
  if (cin % tcw::KB != 0 || cout < 64 || taps > tcw::MAX_TAPS_Q || kh > 128 || kw > 128) return false;
  const int oh = h - kh + 1, ow = w - kw + 1;
  if (oh < 1 || ow < 1 || batch < 1) return false;
  if ((long long)batch * oh * ow * cout >= (1LL << 40)) return false;
  p.y = y;
  p.bias = bias;
  p.epi = epi;
  p.y_dtype = SEGCONV_BF16;
  p.batch = batch;
  p.n = h;
  p.cin = cin;
  p.cout = cout;
  p.out_h = oh;
  p.out_w = ow;
  p.NT = tc_wide_ntile(cout);
  p.n_tiles = (cout + p.NT - 1) / p.NT;
  p.nkb = cin / tcw::KB;
  p.im2col = 1;
  p.bprod = wide_bprod();
  p.S_rows = 128;
  p.taps[0] = taps;
  for (int u = 0; u < kh; ++u)
    for (int v = 0; v < kw; ++v) {
      p.tap_off_r[0][u * kw + v] = u;
      p.tap_off_c[0][u * kw + v] = v;
    }
  p.rows[0] = oh;
  p.cols[0] = ow;
  p.wscale = 1;
  p.wbase_r = p.wbase_c = 0;
  p.ostride = 1;
  p.a_stage_bytes = 128 * 128;
  p.b_stage_bytes = (p.NT / 2) * 128;
  if (p.b_stage_bytes % 1024) return false;
  const int bar_bytes = (2 * tcw::MAX_STAGES_A + 2 * tcw::MAX_STAGES_B + 4) * 8 + 16;
  p.stages_a = p.stages_b =
      std::min(tcw::MAX_STAGES_A, (tcw::SMEM_LIMIT - bar_bytes) / (p.a_stage_bytes + p.b_stage_bytes));
  if (p.stages_a < 2) return false;
  const long long u1 = ((long long)batch * oh * ow + 255) / 256 * p.n_tiles;
  p.unit_base[0] = 0;
  for (int q = 1; q <= 4; ++q) p.unit_base[q] = u1;
  p.units = u1;
  EncodeTiledFnW fn = encode_fn_w();
  EncIm2colW enc2 = encode_im2col_w();
  if (!fn || !enc2) return false;
  {
    const cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
    const cuuint64_t strides[3] = {(cuuint64_t)cin * 2, (cuuint64_t)w * cin * 2, (cuuint64_t)h * w * cin * 2};
    const int lower[2] = {0, 0};
    const int upper[2] = {-(kw - 1), -(kh - 1)};  // walk origins: the output pixels
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc2(&maps.xi[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(src), dims, strides, lower,
             upper, (cuuint32_t)tcw::KB, 128, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    const cuuint64_t dims[3] = {(cuuint64_t)cin, (cuuint64_t)taps, (cuuint64_t)cout};
    const cuuint64_t strides[2] = {(cuuint64_t)cin * 2, (cuuint64_t)taps * cin * 2};
    const cuuint32_t box[3] = {(cuuint32_t)tcw::KB, 1, (cuuint32_t)(p.NT / 2)};
    const cuuint32_t es[3] = {1, 1, 1};
    if (fn(&maps.w[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(kt), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  maps.x = maps.xi[0];
  for (int q = 1; q < 4; ++q) {
    maps.w[q] = maps.w[0];
    maps.xi[q] = maps.xi[0];
  }
  return true;
}

bool tc_conv_valid_supported(int batch, int h, int w, int cin, int kh, int kw, int cout) {
  const int taps = kh * kw;
  return cin % tcw::KB == 0 && cout >= 64 && cout % 8 == 0 && taps <= tcw::MAX_TAPS_Q && h - kh + 1 >= 1 &&
         w - kw + 1 >= 1 && batch >= 1 && kh <= 128 && kw <= 128;
}

bool tc_bwd_data_supported(const BackwardProblem& pr) {
  tcw::Params p;
  tcw::Maps m;
  return make_wide_dgrad(pr, p, m);
}

bool tc_wide_supported(const FusedProblem& pr, int math) {
  if (math != SEGCONV_MATH_BF16 && math != SEGCONV_MATH_F16X3 && math != SEGCONV_MATH_TF32) return false;
  tcw::Params p;
  tcw::Maps m;
  return make_wide(pr, p, m, pr.x);  // pr.x stands in for the split copy (alignment only)
}

// Balanced unit schedule for the im2col forward (Params::sched).  Units are
// class-major and a unit's length is its class's taps x k-blocks, so the
// round-robin order leaves pairs with one long unit more than others (C5
// layer a: 128 k-steps on the busiest pair for a mean of 111).  Longest unit
// first onto the least-loaded pair; a unit of >= 12 stages that would
// overshoot the mean is run as two feature halves (N = NT/2, half-width weight
// boxes) on the two least-loaded pairs, costed at 0.65 of the unit each (half
// the MMAs, but the same A tile).  Used when it beats round-robin; cached per
// shape.  Measured on the C5 stack (eager layer times, 30 steps): layer a
// 60.6 -> 56.7 us; splitting shorter units (layer b's 4- and 8-stage ones)
// cost 1 us there, and with two CTAs per SM (layer c) the pairs sharing an SM
// already even out -- a balanced order was 1.5 us slower -- so neither is done
// (see balance_units for where it is used).
// unit_base: first unit of each class (class-major), cost = taps x k-block
// stages; returns the [pairs][slots] table, or empty when round-robin is as good
static std::vector<uint16_t> wide_schedule(const long long* unit_base, const int* taps, int nkb, int passes,
                                           bool halves, long long pairs) {
  std::vector<uint16_t> tab;
  const long long units = unit_base[4];
  if (units <= 0 || units > 0x3FFF || pairs <= 0 || units <= pairs) return tab;
  std::vector<std::pair<int, int>> us;  // (cost, unit)
  long long total = 0;
  for (int q = 0; q < 4; ++q)
    for (long long u = unit_base[q]; u < unit_base[q + 1]; ++u) {
      const int c = taps[q] * nkb * passes * 100;
      us.emplace_back(c, (int)u);
      total += c;
    }
  long long rr_max = 0;
  for (long long i = 0; i < pairs; ++i) {
    long long l = 0;
    for (long long u = i; u < (long long)us.size(); u += pairs) l += us[u].first;  // class-major = unit order
    rr_max = std::max(rr_max, l);
  }
  std::stable_sort(us.begin(), us.end(),
                   [](const std::pair<int, int>& a, const std::pair<int, int>& b) { return a.first > b.first; });
  const double target = 1.02 * (double)total / (double)pairs;
  using LP = std::pair<double, long long>;
  std::priority_queue<LP, std::vector<LP>, std::greater<LP>> heap;
  for (long long i = 0; i < pairs; ++i) heap.emplace(0.0, i);
  std::vector<std::vector<uint16_t>> lists((size_t)pairs);
  for (const auto& cu : us) {
    const LP a = heap.top();
    heap.pop();
    if (halves && cu.first >= 1200 && a.first + cu.first > target) {
      const LP b = heap.top();
      heap.pop();
      lists[(size_t)a.second].push_back((uint16_t)(cu.second | (1 << 14)));
      lists[(size_t)b.second].push_back((uint16_t)(cu.second | (2 << 14)));
      heap.emplace(a.first + 0.65 * cu.first, a.second);
      heap.emplace(b.first + 0.65 * cu.first, b.second);
    } else {
      lists[(size_t)a.second].push_back((uint16_t)cu.second);
      heap.emplace(a.first + cu.first, a.second);
    }
  }
  double mx = 0;
  while (!heap.empty()) {
    mx = std::max(mx, heap.top().first);
    heap.pop();
  }
  size_t sl = 0;
  for (const auto& l : lists) sl = std::max(sl, l.size());
  if (mx < 0.99 * (double)rr_max && (long long)sl * pairs <= tcw::SCHED_MAX) {
    tab.assign((size_t)pairs * sl, (uint16_t)0xFFFF);
    for (size_t i = 0; i < lists.size(); ++i)
      std::copy(lists[i].begin(), lists[i].end(), tab.begin() + (long long)i * (long long)sl);
  }
  return tab;
}

static bool balance_units(tcw::Params& pk, long long pairs) {
  // only with feature halves available and >= 2.5 waves of units: a longest-first
  // order without halves, or over fewer waves, measured slower than round-robin
  // (C5 at 512 images: 87.8 -> 92.0 us; layer c at 512: 25.9 -> 27.7 us) --
  // round-robin runs a pixel tile's feature tiles on neighbouring pairs at the
  // same time, and their shared A tiles then cost the L2 once
  if (!(pk.mode == 0 && pk.im2col) || pk.cps == 2 || pk.unit_base[4] != pk.units || !pk.wh_ok ||
      2 * pk.units < 5 * pairs)
    return false;
  struct Key {
    long long pairs, base[5];
    int taps[4], nkb, split, wh;
    bool operator<(const Key& o) const { return std::memcmp(this, &o, sizeof(Key)) < 0; }
  };
  Key key;
  std::memset(&key, 0, sizeof(key));
  key.pairs = pairs;
  for (int q = 0; q < 5; ++q) key.base[q] = pk.unit_base[q];
  for (int q = 0; q < 4; ++q) key.taps[q] = pk.taps[q];
  key.nkb = pk.nkb;
  key.split = pk.split;
  key.wh = pk.wh_ok;
  static std::mutex mu;
  static std::map<Key, std::vector<uint16_t>> cache;  // empty vector: round-robin is as good
  std::vector<uint16_t> tab;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it == cache.end())
      it = cache.emplace(key, wide_schedule(pk.unit_base, pk.taps, pk.nkb, pk.split ? 3 : 1, pk.wh_ok != 0, pairs))
               .first;
    tab = it->second;
  }
  if (tab.empty()) return false;
  std::copy(tab.begin(), tab.end(), pk.sched);
  pk.sched_slots = (int)(tab.size() / (size_t)pairs);
  return true;
}

// diagnostics / host-logic tests (segconv_debug_wide_schedule)
size_t debug_wide_schedule(const long long* unit_base, const int* taps, int nkb, long long pairs, int halves,
                           uint16_t* out, size_t cap) {
  const std::vector<uint16_t> t = wide_schedule(unit_base, taps, nkb, 1, halves != 0, pairs);
  if (t.empty() || out == nullptr || t.size() > cap) return 0;
  std::copy(t.begin(), t.end(), out);
  return t.size() / (size_t)pairs;
}

template <typename YT, int ACT>
static cudaError_t launch_wide_t(const tcw::Params& prm, const tcw::Maps& maps, cudaStream_t s) {
  auto kern = prm.cps == 2 ? tcw::wide_kernel<YT, ACT, 2> : tcw::wide_kernel<YT, ACT, 1>;
  static PerDeviceOnce once1, once2;
  {
    const cudaError_t e = prm.cps == 2 ? smem_attr_once(once2, kern, tcw::SMEM_PER_CTA2)
                                       : smem_attr_once(once1, kern, tcw::SMEM_LIMIT);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  long long pairs = std::min<long long>(prm.units, (long long)(sms / 2) * (prm.cps == 2 ? 2 : 1));
  tcw::Params pk = prm;
  const bool no_balance = (prm.debug & 64) != 0;  // diagnostics (SEGCONV_TC_DEBUG): round-robin order
  // last partial wave: when its T units fit twice over, run them as 2T feature
  // half-tiles (N = NT/2) so the wave takes half a unit instead of a whole one
  if (!no_balance && balance_units(pk, pairs)) {
  } else if (prm.mode == 0 && prm.im2col && prm.NT >= 128 && pairs > 0) {
    const long long T = prm.units % pairs;
    if (T > 0 && 2 * T <= pairs) {
      pk.tail_on = 1;
      pk.tail_full = prm.units - T;
      pk.units = prm.units + T;
    }
  }
  const size_t smem = (size_t)prm.stages_a * prm.a_stage_bytes + (size_t)prm.stages_b * prm.b_stage_bytes +
                      (2 * tcw::MAX_STAGES_A + 2 * tcw::MAX_STAGES_B + 4) * 8 + 16;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(tcw::wide_threads(prm.cps == 2 ? 2 : 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the previous
  at[1].val.programmaticStreamSerializationAllowed = 1;              // kernel's tail
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, pk, maps);
  if (e == cudaSuccess) note_launch();
  return e;
}

namespace tcw {
// fp32 x -> fp16 [hi | lo] channel halves, x * 2^t = hi + lo to ~22 bits.
// fp16 has a 5-bit exponent: a power of two t puts max |x * 2^t| at 2^14, so
// no finite input overflows and the split's subnormal floor (2^-25) sits 39
// binades below the largest activation (range guard, tc_guard.cuh).  The sums
// are of (x 2^t)(w 2^s): inv_out = 2^-s * 2^-t, applied in the epilogue.
__global__ void x_amax_kernel(const float* __restrict__ x, long long n, unsigned* __restrict__ amax_bits) {
  float m = 0.0f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {  // float4 body, scalar tail
    const long long n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    long long e = e0;
    for (; e + 3 * stride < n4; e += 4 * stride) {  // four loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + e + u * stride);  // read once: streaming
#pragma unroll
      for (int u = 0; u < 4; ++u)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
    }
    for (; e < n4; e += stride) {
      const float4 v = __ldcs(x4 + e);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    e0 += n4 * 4;
    if (e0 < n) m = fmaxf(m, fabsf(__ldg(x + e0)));  // < 4 left: the first threads take them
  } else {
    for (long long e = e0; e < n; e += stride) m = fmaxf(m, fabsf(__ldg(x + e)));
  }
  // one atomic per block: a thousand warps' atomics on one word serialise at L2
  __shared__ float wm[32];
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) atomicMax(amax_bits, __float_as_uint(m));
  }
}

__global__ void split_x_kernel(const float* __restrict__ x, __half* __restrict__ xs, long long npix, int cin,
                               const unsigned* __restrict__ amax_bits, const float* __restrict__ w_inv,
                               float* __restrict__ inv_out) {
  const int t = split_scale_exp(*amax_bits);
  const float scale = ldexpf(1.0f, t);
  if (blockIdx.x == 0 && threadIdx.x == 0) *inv_out = *w_inv * ldexpf(1.0f, -t);
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (cin % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(xs) & 15) == 0) {
    // 8 channels per thread: two float4 loads, two 16-byte stores (hi, lo)
    const int c8 = cin / 8;
    const long long total8 = npix * c8;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total8; e += stride) {
      const long long pix = e / c8;
      const int ch = (int)(e - pix * c8) * 8;
      const float4* src = reinterpret_cast<const float4*>(x + pix * cin + ch);
      const float4 a = __ldcs(src), b = __ldcs(src + 1);
      const float v[8] = {a.x * scale, a.y * scale, a.z * scale, a.w * scale,
                          b.x * scale, b.y * scale, b.z * scale, b.w * scale};
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __half2 h = __floats2half2_rn(v[2 * k], v[2 * k + 1]);
        const float2 hf = __half22float2(h);
        const __half2 l = __floats2half2_rn(v[2 * k] - hf.x, v[2 * k + 1] - hf.y);
        hi[k] = *reinterpret_cast<const uint32_t*>(&h);
        lo[k] = *reinterpret_cast<const uint32_t*>(&l);
      }
      __half* dst = xs + pix * 2 * cin + ch;
      *reinterpret_cast<uint4*>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(dst + cin) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
    return;
  }
  const long long total = npix * cin;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += stride) {
    const long long pix = e / cin;
    const int ch = (int)(e - pix * cin);
    const float v = x[e] * scale;
    const __half hi = __float2half_rn(v);
    xs[pix * 2 * cin + ch] = hi;
    xs[pix * 2 * cin + cin + ch] = __float2half_rn(v - __half2float(hi));
  }
}
// Split-fp16 input gradient: w2[taps][cin][4 cout] fp16 = [wh | wh | wl | 0]
// (make_wide_dgrad: two k-blocks against one A box [gh | gl]), weights scaled
// by 2^s (max |w'| = 2^14); *w_inv = 2^-s.
__global__ void split_w2_kernel(const float* __restrict__ k, int taps, int cin, int cout,
                                const unsigned* __restrict__ amax_bits, __half* __restrict__ w2,
                                float* __restrict__ w_inv, const unsigned* __restrict__ gy_amax_bits,
                                int* __restrict__ guard) {
  const int s = split_scale_exp(*amax_bits);
  const float scale = ldexpf(1.0f, s);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *w_inv = ldexpf(1.0f, -s);
    if (guard != nullptr) {
      // accuracy bound of the split: each fp16 hi/lo pair is within 2^-25 of
      // its scaled value (max 2^14), i.e. 2^-38 of the largest |gy| (|w|);
      // over K = taps x cout products the absolute error stays under a
      // quarter of the fp32 bar's 1e-5 floor when max|gy| max|w| K 2^-37
      // does.  Past it (dynamic ranges of ~10^9 and more) the SIMT kernels run.
      const float gmax = __uint_as_float(*gy_amax_bits), wmax = __uint_as_float(*amax_bits);
      const bool ok = (double)gmax * wmax * taps * cout * 0x1p-37 <= 2.5e-6 && isfinite(gmax) && isfinite(wmax);
      guard[0] = ok ? 1 : 0;
      guard[1] = ok ? 0 : 1;
    }
  }
  const int kch = 2 * cout;
  const long long total = (long long)taps * cin * cout;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / cout;  // (tap, ci)
    const int f = (int)(e - row * cout);
    const float v = k[e] * scale;
    const __half hi = __float2half_rn(v);
    const __half lo = __float2half_rn(v - __half2float(hi));
    __half* r = w2 + row * 2 * kch;  // [wh | wh | wl | 0]: k-block 0 x [gh | gl], k-block 1 x [gh | gl]
    r[f] = hi;
    r[cout + f] = hi;
    r[2 * cout + f] = lo;
    r[3 * cout + f] = __float2half_rn(0.0f);
  }
}
}  // namespace tcw

cudaError_t launch_tc_wide(const FusedProblem& pr, cudaStream_t s) {
  tcw::Params p;
  tcw::Maps maps;
  if (pr.x_dtype == SEGCONV_F32 && pr.panel_dtype == SEGCONV_F16_SPLIT) {
    const long long npix = (long long)pr.batch * pr.n * pr.n;
    if (npix == 0) return cudaSuccess;
    void* xs = nullptr;
    const size_t xs_bytes = ((size_t)npix * 2 * pr.cin * 2 + 15) / 16 * 16;
    cudaError_t e = workspace_alloc(&xs, xs_bytes + 16, s);
    if (e != cudaSuccess) return e;
    // after the halves: [max |x| bits][2^-s 2^-t]
    unsigned* xtail = reinterpret_cast<unsigned*>(static_cast<char*>(xs) + xs_bytes);
    const long long total = npix * pr.cin;
    const bool ok = make_wide(pr, p, maps, xs);
    e = ok ? cudaMemsetAsync(xtail, 0, 4, s) : cudaErrorNotSupported;
    if (e == cudaSuccess) {
      const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
      tcw::x_amax_kernel<<<std::min(blocks, 148u * 8), 256, 0, s>>>((const float*)pr.x, total, xtail);
      tcw::split_x_kernel<<<blocks, 256, 0, s>>>((const float*)pr.x, (__half*)xs, npix, pr.cin, xtail,
                                                  p.split_inv_scale, reinterpret_cast<float*>(xtail + 1));
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      note_launch(2);
      p.split_inv_scale = reinterpret_cast<const float*>(xtail + 1);
      {
        p.trace = tc_trace_buffer();
        const int act = (pr.epi & SEGCONV_EPI_RELU) ? 1 : (pr.epi & SEGCONV_EPI_TANH) ? 2 : 0;
        if (pr.y_dtype == SEGCONV_BF16)
          e = act == 1 ? launch_wide_t<__nv_bfloat16, 1>(p, maps, s)
                       : act == 2 ? launch_wide_t<__nv_bfloat16, 2>(p, maps, s)
                                  : launch_wide_t<__nv_bfloat16, 0>(p, maps, s);
        else
          e = act == 1 ? launch_wide_t<float, 1>(p, maps, s)
                       : act == 2 ? launch_wide_t<float, 2>(p, maps, s) : launch_wide_t<float, 0>(p, maps, s);
      }
    }
    const cudaError_t e2 = cudaFreeAsync(xs, s);
    return e != cudaSuccess ? e : e2;
  }
  if (!make_wide(pr, p, maps)) return cudaErrorNotSupported;
  if (p.units == 0) return cudaSuccess;
  p.trace = tc_trace_buffer();
  static const int dbg = getenv("SEGCONV_TC_DEBUG") ? atoi(getenv("SEGCONV_TC_DEBUG")) : 0;
  p.debug = dbg;
  const int act = (pr.epi & SEGCONV_EPI_RELU) ? 1 : (pr.epi & SEGCONV_EPI_TANH) ? 2 : 0;
  if (pr.y_dtype == SEGCONV_BF16) {
    if (act == 1) return launch_wide_t<__nv_bfloat16, 1>(p, maps, s);
    if (act == 2) return launch_wide_t<__nv_bfloat16, 2>(p, maps, s);
    return launch_wide_t<__nv_bfloat16, 0>(p, maps, s);
  }
  if (act == 1) return launch_wide_t<float, 1>(p, maps, s);
  if (act == 2) return launch_wide_t<float, 2>(p, maps, s);
  return launch_wide_t<float, 0>(p, maps, s);
}

cudaError_t launch_tc_bwd_weight(const BackwardProblem& pr, cudaStream_t s) {
  tcw::Params p;
  tcw::Maps maps;
  if (!make_wide_wgrad(pr, p, maps, wide_pairs())) return cudaErrorNotSupported;
  p.trace = nullptr;
  if (p.w_direct) {
    p.wout = (float*)pr.gk;
    return launch_wide_t<float, 0>(p, maps, s);
  }
  float* ws = nullptr;
  cudaError_t e = workspace_alloc((void**)&ws, (size_t)p.w_splits * p.w_ksz * sizeof(float), s);
  if (e != cudaSuccess) return e;
  p.wout = ws;
  e = launch_wide_t<float, 0>(p, maps, s);
  if (e == cudaSuccess) {
    e = launch_wgrad_reduce(ws, (float*)pr.gk, p.w_ksz, p.w_splits, pr.accumulate, s);
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  return e != cudaSuccess ? e : e2;
}

cudaError_t launch_tc_bwd_data(const BackwardProblem& pr, cudaStream_t s) {
  tcw::Params p;
  tcw::Maps maps;
  if (!make_wide_dgrad(pr, p, maps)) return cudaErrorNotSupported;
  if (p.units == 0) return cudaSuccess;
  p.trace = nullptr;
  return launch_wide_t<__nv_bfloat16, 0>(p, maps, s);
}

bool tc_bwd_data_split_supported(const BackwardProblem& pr) {
  tcw::Params p;
  tcw::Maps m;
  return make_wide_dgrad(pr, p, m, pr.gy, pr.k);  // stand-ins for the split copies (alignment only)
}

// fp32 input gradient in split-fp16 math on the pair kernel: pre-passes split gy
// (scaled by 2^t) into [hi | lo] channel halves and build the doubled tap list
// of the kernel (scaled by 2^s); the GEMM's sums are multiplied by 2^-s-t.
cudaError_t launch_tc_bwd_data_split(const BackwardProblem& pr, cudaStream_t s, bool guarded) {
  const long long npix = (long long)pr.batch * pr.out_h * pr.out_w;
  const int taps = pr.kh * pr.kw, kch = 2 * pr.cout;
  const size_t gy16_bytes = ((size_t)npix * kch * 2 + 255) / 256 * 256;
  const size_t w2_bytes = ((size_t)taps * pr.cin * 2 * kch * 2 + 255) / 256 * 256;
  void* ws = nullptr;
  cudaError_t e = workspace_alloc(&ws, gy16_bytes + w2_bytes + 32, s);
  if (e != cudaSuccess) return e;
  void* gy16 = ws;
  void* w2 = static_cast<char*>(ws) + gy16_bytes;
  // tail: [max |gy| bits][max |w| bits][2^-s][2^-s 2^-t][guard: tensor cores ran][SIMT must]
  unsigned* tail = reinterpret_cast<unsigned*>(static_cast<char*>(w2) + w2_bytes);
  float* tailf = reinterpret_cast<float*>(tail);
  int* gflags = reinterpret_cast<int*>(tail + 4);
  tcw::Params p;
  tcw::Maps maps;
  e = make_wide_dgrad(pr, p, maps, gy16, w2) ? cudaMemsetAsync(tail, 0, 8, s) : cudaErrorNotSupported;
  if (e == cudaSuccess && p.units > 0) {
    const long long ngy = npix * pr.cout, nk = (long long)taps * pr.cin * pr.cout;
    const unsigned bg = (unsigned)std::min<long long>((ngy + 255) / 256, 148LL * 16);
    const unsigned bk = (unsigned)std::min<long long>((nk + 255) / 256, 148LL * 4);
    tcw::x_amax_kernel<<<std::min(bg, 148u * 8), 256, 0, s>>>((const float*)pr.gy, ngy, tail);
    tcw::x_amax_kernel<<<bk, 256, 0, s>>>((const float*)pr.k, nk, tail + 1);
    tcw::split_w2_kernel<<<bk, 256, 0, s>>>((const float*)pr.k, taps, pr.cin, pr.cout, tail + 1, (__half*)w2,
                                            tailf + 2, tail, guarded ? gflags : nullptr);
    tcw::split_x_kernel<<<bg, 256, 0, s>>>((const float*)pr.gy, (__half*)gy16, npix, pr.cout, tail, tailf + 2,
                                           tailf + 3);
    e = cudaGetLastError();
    note_launch(4);
    if (e == cudaSuccess) {
      p.split_inv_scale = tailf + 3;
      p.oscale = 1;
      p.run_if = guarded ? gflags : nullptr;
      p.trace = nullptr;
      e = launch_wide_t<float, 0>(p, maps, s);
    }
  }
  if (guarded && e == cudaSuccess && p.units > 0) {
    // the SIMT kernels, gated on the other flag (exit at once when the tensor
    // cores took the gradient) -- decided on the device, nothing synchronises
    BackwardProblem pf = pr;
    pf.run_if = gflags + 1;
    e = launch_bwd_data_simt(pf, false, s);
  }
  const cudaError_t e2 = cudaFreeAsync(ws, s);
  return e != cudaSuccess ? e : e2;
}

cudaError_t launch_tc_conv_valid(const void* src, int batch, int h, int w, int cin, const void* kt, int kh,
                                 int kw, int cout, const float* bias, unsigned epi, void* y, cudaStream_t s) {
  tcw::Params p;
  tcw::Maps maps;
  if (!make_wide_conv(src, batch, h, w, cin, kt, kh, kw, cout, bias, epi, y, p, maps))
    return cudaErrorNotSupported;
  p.trace = nullptr;
  const int act = (epi & SEGCONV_EPI_RELU) ? 1 : (epi & SEGCONV_EPI_TANH) ? 2 : 0;
  if (act == 1) return launch_wide_t<__nv_bfloat16, 1>(p, maps, s);
  if (act == 2) return launch_wide_t<__nv_bfloat16, 2>(p, maps, s);
  return launch_wide_t<__nv_bfloat16, 0>(p, maps, s);
}

}  // namespace segconv_b200

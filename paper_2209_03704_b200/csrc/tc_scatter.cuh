// tc_scatter.cuh -- column layout shared by the pixel-scatter kernels
// (tc_ring.cu, tc_tile.cu) and their weight images.
#pragma once

namespace segconv_b200 {

// Column layout of D (= rows of the weight image) for even p_orig (p = 0 as
// written; an even p shifts every input offset by -p/2, which the kernels
// apply): per-axis parity r has act(r) = (KH - r + 1) / 2 taps starting at
// offset r, so the union window is U = max_r (r + act(r)) rows / cols (KH + 1)
// / 2 for odd KH, KH / 2 + 1 for even KH).  Columns: for dy, a group padded to
// a multiple of 16; inside it (q, dx, f) with f fastest.
template <int KH, int COUT>
struct ScatterLayout {
  static constexpr int act(int r) { return (KH - r + 1) / 2; }
  static constexpr int U = act(0) > 1 + act(1) ? act(0) : 1 + act(1);
  static constexpr bool has(int q, int dy, int dx) {
    return dy >= (q >> 1) && dy < (q >> 1) + act(q >> 1) && dx >= (q & 1) &&
           dx < (q & 1) + act(q & 1);
  }
  static constexpr bool has_dy(int q, int dy) {
    return dy >= (q >> 1) && dy < (q >> 1) + act(q >> 1);
  }
  static constexpr int group_len(int dy) {
    int n = 0;
    for (int q = 0; q < 4; ++q)
      for (int dx = 0; dx < U; ++dx)
        if (has(q, dy, dx)) n += COUT;
    return n;
  }
  static constexpr int group_pad(int dy) { return (group_len(dy) + 15) / 16 * 16; }
  static constexpr int group_off(int dy) {
    int o = 0;
    for (int d = 0; d < dy; ++d) o += group_pad(d);
    return o;
  }
  static constexpr int N = group_off(U);
  // column of (dy, q, dx, f) inside its group, -1 if absent
  static constexpr int col_in_group(int dy, int q, int dx, int f) {
    if (!has(q, dy, dx)) return -1;
    int c = 0;
    for (int qq = 0; qq < 4; ++qq)
      for (int xx = 0; xx < U; ++xx)
        if (has(qq, dy, xx)) {
          if (qq == q && xx == dx) return c + f;
          c += COUT;
        }
    return -1;
  }
  // useful columns only (the tile kernel's SMEM copy of D): (dy, q, dx, f) ->
  // column, group by group without the 16-column padding
  static constexpr int useful_off(int dy) {
    int o = 0;
    for (int d = 0; d < dy; ++d) o += group_len(d);
    return o;
  }
  static constexpr int NU = useful_off(U);
  static constexpr int ucol(int dy, int q, int dx, int f) {
    return has(q, dy, dx) ? useful_off(dy) + col_in_group(dy, q, dx, f) : -1;
  }
  // D (TMEM) column -> useful column, -1 for padding
  static constexpr int compact(int c) {
    int dy = 0;
    while (dy + 1 < U && c >= group_off(dy + 1)) ++dy;
    const int col = c - group_off(dy);
    return col < group_len(dy) ? useful_off(dy) + col : -1;
  }
};

}  // namespace segconv_b200

// px_layout.cuh — geometry of the pixel-major tensor-core SNO path (no_px_kernels.cu) and of the
// MMA-ready blobs its kernels exchange through HBM.
//
// A layer tile is 128 consecutive pixels of one system in row-major order (n = 64: two rows;
// n >= 128: a 128-column block of one row), so the channel GEMMs run with M = 128 pixels and
// N = NP output channels (w rounded up to 16) and no padding in M.  Blobs (bf16 hi + bf16 lo, the
// 3xBF16 split, each half in the canonical no-swizzle core-matrix layout its consumer reads):
//   V tile  [hi | lo], each [cgroup c/8][pgroup p/8][p%8][c%8] (2048 B per cgroup): the K-major A of
//           the next layer's bypass GEMM and, read MN-major, the A of this layer's x-analysis.
//           Only CGS = ceil(w/8) channel groups are stored; the stage's padding groups are zeros.
//   G       y-synthesised spectral term, the MN-major B of the x-synthesis (N = o, K = k' = (kappa2,
//           re|im) < 40, 5 k-groups; k-group 5 (k' 40..47) is zero in smem).  In smem a row is
//           [k'/8][o/8][k'%8][o%8]; in HBM the rows of a system are interleaved at 32-byte granularity,
//           [b][hi|lo][k'/8, o/8][k'%8 / 2][row i][32 B], so the y-synthesis writes 1 KB runs per warp
//           (32 consecutive rows) and the layer gathers one row with a 5-D TMA tensor copy whose box
//           lands in smem in exactly the row's canonical order.
//   T row   fp32 [kappa2][o][re|im] (40 w floats): x-analysed activations, read by the y-analysis.
#pragma once
#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace fcgno {

struct PxGeom {
  int n, w, NP, KCG, CGS, RT, CB, TPS, units, nF, nMT, LBO_G, D2W, MYT;
  __host__ __device__ PxGeom(int n_, int w_) : n(n_), w(w_) {
    NP = (w + 15) & ~15;          // N of the channel GEMMs (w rounded up to 16)
    KCG = NP / 8;                 // channel groups of a stage tile
    CGS = (w + 7) / 8;            // channel groups stored in HBM
    RT = n < 128 ? 128 / n : 1;   // rows per tile (n = 64: 2)
    CB = n < 128 ? 1 : n / 128;   // column blocks per row
    TPS = n * n / 128;            // tiles per system
    units = n / RT;               // row units (RT rows, CB tiles) per system
    nF = n < 128 ? 3 : CB;        // twiddle blobs: per column block; n = 64: unmasked + 2 row-masked
    nMT = (n + 127) / 128;        // y-synthesis M tiles of 128 rows
    LBO_G = (NP / 8) * 128;       // k-group stride of a G row
    D2W = RT * 48;                // x-analysis accumulator columns per tile
    MYT = (40 * w + 127) / 128;   // y-analysis M tiles of 128 (kappa2, o, re|im) rows
  }
  __host__ __device__ uint32_t v_half() const { return (uint32_t)CGS * 2048u; }      // stored hi (= lo) of a V tile
  __host__ __device__ uint32_t g_half() const { return 5u * (uint32_t)LBO_G; }      // stored hi (= lo) of a G row
  // smem hi (= lo) of a stage tile: the stored channel groups only; the bypass GEMM reads an odd last
  // group's partner (channels CGS*8 .. KCG*8) from a shared zero block instead
  __host__ __device__ uint32_t stage_half() const { return (uint32_t)CGS * 2048u; }
  __host__ __device__ size_t v_bytes(int B) const { return (size_t)B * TPS * 2 * v_half(); }
  __host__ __device__ size_t g_bytes(int B) const { return (size_t)B * n * 2 * g_half(); }
  __host__ __device__ size_t t_floats(int B) const { return (size_t)B * n * 40 * w + 256; }   // + over-read pad
  // byte offset of the 32-byte piece (system b, hi|lo hl, k-group kg, o-group og, k'%8 pair, row i) of G
  __host__ __device__ size_t g_off(int b, int hl, int kg, int og, int pair, int i) const {
    return (((((size_t)b * 2 + hl) * 5 + kg) * (NP / 8) + og) * 4 + pair) * (size_t)n * 32 + (size_t)i * 32;
  }
};

// Constant operand blobs, built once per NO apply / solve by k_px_prep ([hi][lo] each):
//   F[f]    twiddles F[p][k'] = (cos, -sin)(2 pi kappa2 j(p) / n) for k' < 40, k-group-major
//           [k'/8][p/8][p%8][k'%8] (5 k-groups of 2048 B; k' 40..47 read from the layer's zero block):
//           the x-synthesis A (K-major, M = p) and, read MN-major, the x-analysis B.  n = 64: f = 0
//           unmasked, f = 1 / 2 zero outside the tile's first / second row (per-row synthesis).
//   W[l]    layer weights W[o][c] (layers 2, 3), K-major B (N = o, K = c), NP x NP.
//   FP[mt]  y-synthesis A: Fp[i][(kappa1, re|im)], K-major (M = i, K = 48), per 128-row M tile.
//   FY      y-analysis B: F[i][(kappa1, x|y)], K-major (N = 48, K = i).
//   MX[l]   mode-mixing B per mode (layers 2, 3, and the layer-4/projection fold with cout = 1).
struct PxConst {
  size_t F, W[2], FP, FY, MX[3], total;
  uint32_t f_half, w_half, fp_half, fy_half, mx_half[3];
  int KM, NM[3];
  __host__ __device__ PxConst(const PxGeom& g) {
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 1023) & ~size_t(1023); return at; };
    f_half = 5u * 2048u;
    F = take((size_t)g.nF * 2 * f_half);
    w_half = (uint32_t)g.NP * g.NP * 2u;
    W[0] = take(2 * (size_t)w_half);
    W[1] = take(2 * (size_t)w_half);
    fp_half = 128u * 48u * 2u;
    FP = take((size_t)g.nMT * 2 * fp_half);
    fy_half = (uint32_t)g.n * 48u * 2u;
    FY = take(2 * (size_t)fy_half);
    KM = (2 * g.w + 15) & ~15;
    for (int l = 0; l < 3; ++l) {
      const int cout = l < 2 ? g.w : 1;
      NM[l] = (cout + 15) & ~15;
      mx_half[l] = (uint32_t)NM[l] * KM * 2;
      MX[l] = take((size_t)kModes2 * 2 * mx_half[l]);
    }
    total = o;
  }
};

}  // namespace fcgno

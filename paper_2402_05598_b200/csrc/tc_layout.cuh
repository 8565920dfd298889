// tc_layout.cuh — geometry of the tensor-core SNO path and of the MMA-ready "blobs" its kernels
// exchange through HBM.  Every inter-kernel tensor is stored already split into bf16 hi + lo in
// the canonical no-swizzle core-matrix layout its consumer's tcgen05.mma reads, one contiguous
// blob per consumer tile, so a consumer stages a tile with a single cp.async.bulk and a producer
// converts in its epilogue.
#pragma once
#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace fcgno {

constexpr int kKS = 48;   // x-synthesis / x-analysis width: 40 (20 modes x re|im) padded to 48

struct TcGeom {
  int n, w, WP, R, CP, KB, tiles_per_sys, mtiles;
  __host__ __device__ TcGeom(int n_, int w_) : n(n_), w(w_) {
    WP = w <= 32 ? 32 : (w <= 64 ? 64 : 128);   // padded channels per row in the 128 TMEM lanes
    R = 128 / WP;                               // rows per tile
    CP = (w + 7) & ~7;                          // channels per row in the K index (r, c)
    KB = (R * CP + 15) & ~15;                   // bypass K = R * CP padded to 16
    tiles_per_sys = n / R;
    mtiles = (w * kModes + 127) / 128;          // y-analysis M tiles of (o, kappa2) rows
  }
  // activation blob of a tile (B operand of the next layer): MN-major, N = j (n), K = (r, c) (KB)
  __host__ __device__ uint32_t v_half() const { return (uint32_t)KB * n * 2; }          // bytes of hi (= lo)
  __host__ __device__ uint32_t v_sbo() const { return (uint32_t)(KB / 8) * 128; }
  // G blob of a tile (A operand of the x-synthesis): K-major, M = (o, r) (lane o*R + r, 128), K = k' (48)
  __host__ __device__ uint32_t g_half() const { return 128u * kKS * 2; }
  __host__ __device__ uint32_t g_sbo() const { return (uint32_t)(kKS / 8) * 128; }
  // T blob of an (system, m-tile) (A operand of the y-analysis): MN-major, M = (o, kappa2) (128 per tile),
  // K = (i, re|im) (2n); m-groups adjacent (SBO = 128), k-groups at LBO = 16 * 128, so the 2R
  // consecutive k written by one layer tile form 2R*16-byte contiguous runs.
  __host__ __device__ uint32_t t_half() const { return 128u * (2 * n) * 2; }
  __host__ __device__ uint32_t t_sbo() const { return 128u; }
  __host__ __device__ uint32_t t_lbo() const { return 16u * 128u; }
  __host__ __device__ size_t v_bytes_total(int B) const { return (size_t)B * tiles_per_sys * 2 * v_half(); }
  __host__ __device__ size_t g_bytes_total(int B) const { return (size_t)B * tiles_per_sys * 2 * g_half(); }
  __host__ __device__ size_t t_bytes_total(int B) const { return (size_t)B * mtiles * 2 * t_half(); }
};

}  // namespace fcgno

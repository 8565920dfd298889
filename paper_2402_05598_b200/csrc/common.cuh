// common.cuh — device primitives shared by the FCG-NO kernels (sm_100a).
//
//  * double-double arithmetic built from error-free transformations (TwoSum, TwoProduct via
//    fma), used to make every inner product the correctly rounded value of the exact sum in
//    all but astronomically rare ties (reading R6);
//  * deterministic block reductions and the "last CTA of a system reduces the partials"
//    protocol, so no scalar-only kernel launch is needed per reduction;
//  * the harmonic face mean of the stencil (R1); the stencil itself (canonical op
//    order R5, explicit _rn intrinsics so nvcc cannot contract it into fma) is st_walk in
//    fcg_device.cuh.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fcgno {

constexpr int kThreads = 256;          // block size of the element-wise / stencil kernels
constexpr int kPerThread = 4;          // elements per thread
constexpr int kTile = kThreads * kPerThread;  // elements of one system per CTA
constexpr int kModes = 20;             // K
constexpr int kModes2 = kModes * kModes;
constexpr int kMmax = 64;              // FCGNO_MMAX
constexpr int kDotChunk = 6;           // window dots reduced together
constexpr int kRowSplitMax = 8;        // row parts per system of the FFMA NO layer (partial analyses)
// rows per CTA of k_dft_rows (= row groups of the input DFT partials): 4 up to n = 128 (more CTAs
// for the small grids), 8 above (fewer partials for k_lift_mix to sum); same-box A/B, DESIGN §5.7
__host__ __device__ __forceinline__ int dft_rows(int n) { return n <= 64 ? 4 : 8; }
constexpr int kStR = 16;               // rows of a 2-D stencil tile
constexpr int kStC = 128;              // columns of a 2-D stencil tile
constexpr int kStThreads = 256;        // block size of the stencil-tile kernels

// 2-D stencil tiles (fcg_device.cuh): C = min(n, kStC) columns, kStR rows, CTAs per system.
__host__ __device__ __forceinline__ int st_cols(int n) { return n < kStC ? n : kStC; }
__host__ __device__ __forceinline__ int st_tiles(int n) {
  return ((n + kStR - 1) / kStR) * ((n + st_cols(n) - 1) / st_cols(n));
}
// Elements per thread of the element-wise kernels: kPerThread for small batches (more CTAs, lower
// latency), kEptWide once a batch has >= 2^21 unknowns (fewer, fatter CTAs amortise the per-CTA
// double-double reduction and keep more loads in flight).
constexpr int kEptWide = 16;
__host__ __device__ __forceinline__ bool ew_wide(int n, int B) { return (size_t)n * n * B >= ((size_t)1 << 21); }
constexpr int kEptUpdate = 16;         // k_update streams two vectors (u is updated lazily)
__host__ __device__ __forceinline__ int ew_blocks(int n, int ept) { return (n * n + kThreads * ept - 1) / (kThreads * ept); }
// Capacity of the per-system partial arrays: the most CTAs any kernel launches per system.
__host__ __device__ __forceinline__ int part_cap(int n) {
  const int a = (n * n + kTile - 1) / kTile, b = st_tiles(n);
  return a > b ? a : b;
}

enum : int { SYS_RUNNING = 0, SYS_CONVERGED = 1, SYS_MAXIT = 2, SYS_BREAKDOWN = 3, SYS_NONFINITE = 4 };
enum : int { FLAG_NONFINITE = 1, FLAG_BREAKDOWN = 2 };

// ------------------------------------------------------------------ double-double
struct __align__(16) dd { double hi, lo; };

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void fast_two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  e = __dsub_rn(b, __dsub_rn(s, a));
}
// Accurate double-double addition (relative error <= 3u^2); commutative bit for bit.
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  double sh, sl, th, tl;
  two_sum(x.hi, y.hi, sh, sl);
  two_sum(x.lo, y.lo, th, tl);
  sl = __dadd_rn(sl, th);
  fast_two_sum(sh, sl, sh, sl);
  sl = __dadd_rn(sl, tl);
  fast_two_sum(sh, sl, sh, sl);
  return {sh, sl};
}
// Dot2 (Ogita-Rump-Oishi) accumulation of one exact product a*b into (s, c).
__device__ __forceinline__ void dot2_acc(double a, double b, double& s, double& c) {
  double p = __dmul_rn(a, b);
  double e = __fma_rn(a, b, -p);
  double q;
  two_sum(s, p, s, q);
  c = __dadd_rn(c, __dadd_rn(q, e));
}
__device__ __forceinline__ dd dot2_finish(double s, double c) {
  dd r;
  fast_two_sum(s, c, r.hi, r.lo);
  return r;
}
__device__ __forceinline__ double dd_round(dd x) { return __dadd_rn(x.hi, x.lo); }

__device__ __forceinline__ dd shfl_down_dd(dd x, int off) {
  return {__shfl_down_sync(0xffffffffu, x.hi, off), __shfl_down_sync(0xffffffffu, x.lo, off)};
}

// Block-reduce NV double-doubles; result valid in thread 0.  `sm` holds >= 8*NV dd.
template <int NV>
__device__ __forceinline__ void block_reduce_dd(dd (&v)[NV], dd* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = dd_add(v[q], shfl_down_dd(v[q], off));
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sm[warp * NV + q] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      dd acc = sm[q];
      for (int w = 1; w < nw; ++w) acc = dd_add(acc, sm[w * NV + q]);
      v[q] = acc;
    }
  }
}

// Deterministic reduction of `count` dd partials (stride `stride` in dd units) by the whole
// block; result returned to every thread.  Order depends only on count and blockDim.
__device__ __forceinline__ dd block_reduce_partials(const dd* part, int count, int stride, dd* sm) {
  dd acc = {0.0, 0.0};
  for (int t = threadIdx.x; t < count; t += blockDim.x) {
    const double2 pv = __ldcg(reinterpret_cast<const double2*>(part + (size_t)t * stride));
    acc = dd_add(acc, dd{pv.x, pv.y});
  }
  dd v[1] = {acc};
  block_reduce_dd<1>(v, sm);
  __shared__ dd bcast;
  if (threadIdx.x == 0) bcast = v[0];
  __syncthreads();
  dd out = bcast;
  __syncthreads();
  return out;
}

// Last-CTA protocol: called by every thread after thread 0 wrote this CTA's partials.
// Returns true in exactly one CTA per system (the last to arrive); that CTA re-arms the counter.
__device__ __forceinline__ bool arrive_last(unsigned* counter, int nblk) {
  __shared__ int last;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == (unsigned)(nblk - 1));
    if (last) *counter = 0u;  // every CTA of this round has arrived; safe to re-arm
  }
  __syncthreads();
  if (last) __threadfence();
  return last != 0;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels of one FCG iteration are launched with programmatic stream serialization: a kernel may
// start (and run its prologue) while its predecessor drains; pdl_wait() blocks until the
// predecessor grid has completed and its memory is visible.  No-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ------------------------------------------------------------------ schedule
__device__ __forceinline__ int m_schedule(int i, int m, int schedule) {
  if (schedule == 1) return i < m ? i : m;               // sliding
  int mod = i % (m + 1);
  int t = mod > 1 ? mod : 1;
  return i < t ? i : t;
}

// ------------------------------------------------------------------ stencil (fp64, canonical order)
__device__ __forceinline__ double harmonic(double a, double b) {
  return __ddiv_rn(2.0 * __dmul_rn(a, b), __dadd_rn(a, b));
}

}  // namespace fcgno

// fcg_small.cu — the whole identity-preconditioned FCG(m) solve of a small system in ONE kernel.
//
// BASELINE configs[0] (32 x 32, batch 1) is bound by latency, not bandwidth: the general path spends
// three dependent launches per iteration on 1,024 unknowns.  Here one CTA owns one
// system (N = n^2 <= 1024, up to four nodes per thread): u, r, the face coefficients and the new p, s live in
// registers, the (p, s) ring of Algorithm 1 in shared memory, and an iteration costs
// a few block-wide double-double reductions instead of launches.  No CTA ever waits on another one.
//
// Arithmetic is the general path's, operation for operation (R5, R6, R12-R14): stencil in
// the canonical order, p = w - sum beta_k p_k newest -> oldest, every inner product the rounded
// double-double sum of exact products, alpha = (p,r)/(p,s), r -= alpha s, u += alpha p.
#include "internal.h"
#include "fcg_device.cuh"

namespace fcgno {

namespace {

constexpr int kSmallRed = 4;   // inner products reduced together

// Sum of NV double-doubles over the block, returned to every thread.  `red` holds 33 * NV dd.
template <int NV>
__device__ __forceinline__ void block_sum_dd(dd (&v)[NV], dd* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = dd_add(v[q], shfl_down_dd(v[q], off));
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp * NV + q] = v[q];
  __syncthreads();
  if (warp == 0) {
    dd a[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) a[q] = lane < nw ? red[lane * NV + q] : dd{0.0, 0.0};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int q = 0; q < NV; ++q) a[q] = dd_add(a[q], shfl_down_dd(a[q], off));
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NV; ++q) red[32 * NV + q] = a[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = red[32 * NV + q];
  __syncthreads();   // red is reused by the next reduction
}

// exact product a * b as a double-double
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}

}  // namespace

// One CTA per system; thread t owns nodes t + q * blockDim.x, q < kSmallPT (blockDim.x = ceil(N / kSmallPT)
// rounded up to a warp), so that a reduction's shuffle tree and barriers are shared by kSmallPT products.
// Dynamic shared memory: ring_p [m+1][N], ring_s [m+1][N] doubles, then 33 * kSmallRed dd of scratch.
constexpr int kSmallPT = 4;
__global__ void __launch_bounds__(256, 1) k_fcg_small(FcgDev d) {
  extern __shared__ __align__(16) double smem[];
  const int n = d.n, N = d.N, m = d.m, b = blockIdx.x, T = blockDim.x;
  double* ring_p = smem;
  double* ring_s = smem + (size_t)(m + 1) * N;
  dd* red = reinterpret_cast<dd*>(smem + (size_t)2 * (m + 1) * N);
  __shared__ double sgamma[kMmax + 1];
  __shared__ double sbeta[kMmax];
  const size_t base = (size_t)b * N;
  int e[kSmallPT], i0[kSmallPT], j0[kSmallPT];
  bool on[kSmallPT];
  double kW[kSmallPT], kE[kSmallPT], kS[kSmallPT], kN[kSmallPT], dsum[kSmallPT], u[kSmallPT], r[kSmallPT];
#pragma unroll
  for (int q = 0; q < kSmallPT; ++q) {
    e[q] = threadIdx.x + q * T;
    on[q] = e[q] < N;
    if (!on[q]) e[q] = 0;
    i0[q] = e[q] / n;
    j0[q] = e[q] - i0[q] * n;
    // face coefficients, once (R1, R2): the adjacent nodal value on the boundary
    const double kc = d.k[base + e[q]];
    kW[q] = j0[q] > 0 ? harmonic(d.k[base + e[q] - 1], kc) : kc;
    kE[q] = j0[q] < n - 1 ? harmonic(kc, d.k[base + e[q] + 1]) : kc;
    kS[q] = i0[q] > 0 ? harmonic(d.k[base + e[q] - n], kc) : kc;
    kN[q] = i0[q] < n - 1 ? harmonic(kc, d.k[base + e[q] + n]) : kc;
    dsum[q] = __dadd_rn(__dadd_rn(kW[q], kE[q]), __dadd_rn(kS[q], kN[q]));
    u[q] = d.u[base + e[q]];
  }
  // (A x)_e for x held in shared memory (zero outside the grid), canonical order R5
  auto apply = [&](const double* x, int q) {
    const int ee = e[q];
    const double xc = x[ee];
    const double xW = j0[q] > 0 ? x[ee - 1] : 0.0, xE = j0[q] < n - 1 ? x[ee + 1] : 0.0;
    const double xS = i0[q] > 0 ? x[ee - n] : 0.0, xN = i0[q] < n - 1 ? x[ee + n] : 0.0;
    double t = __dmul_rn(dsum[q], xc);
    t = __dsub_rn(t, __dmul_rn(kW[q], xW));
    t = __dsub_rn(t, __dmul_rn(kE[q], xE));
    t = __dsub_rn(t, __dmul_rn(kS[q], xS));
    t = __dsub_rn(t, __dmul_rn(kN[q], xN));
    return __dmul_rn(t, d.scale);
  };
  // this thread's part of an inner product: exact products accumulated in double-double
  auto dot_part = [&](const double (&a)[kSmallPT], const double (&c)[kSmallPT]) {
    dd acc = on[0] ? two_prod(a[0], c[0]) : dd{0.0, 0.0};
#pragma unroll
    for (int q = 1; q < kSmallPT; ++q)
      if (on[q]) acc = dd_add(acc, two_prod(a[q], c[q]));
    return acc;
  };
  // r0 = f - A u0, rho0 = ||r0||
#pragma unroll
  for (int q = 0; q < kSmallPT; ++q)
    if (on[q]) ring_p[e[q]] = u[q];   // slot 0 as scratch for the stencil's neighbours
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSmallPT; ++q) r[q] = on[q] ? __dsub_rn(d.f[base + e[q]], apply(ring_p, q)) : 0.0;
  __syncthreads();
  double rho0;
  {
    dd v[1] = {dot_part(r, r)};
    block_sum_dd<1>(v, red);
    rho0 = __dsqrt_rn(dd_round(v[0]));
  }
  int status = (rho0 == 0.0) ? SYS_CONVERGED : (d.maxit == 0 ? SYS_MAXIT : SYS_RUNNING);
  int iters = 0;
  if (threadIdx.x == 0 && d.hist) d.hist[(size_t)b * (d.maxit + 1)] = 1.0;
  for (int i = 0; status == SYS_RUNNING; ++i) {
    const int mi = m_schedule(i, m, d.schedule), slot = ring_slot(i, m);
    // beta_k = (w, s_k) / (p_k, s_k) over the window, w = r
    for (int q0 = 0; q0 < mi; q0 += kSmallRed) {
      dd v[kSmallRed];
#pragma unroll
      for (int t = 0; t < kSmallRed; ++t) {
        v[t] = dd{0.0, 0.0};
        if (q0 + t < mi) {
          const double* sk = ring_s + (size_t)ring_slot(i - mi + q0 + t, m) * N;
          double sv[kSmallPT];
#pragma unroll
          for (int q = 0; q < kSmallPT; ++q) sv[q] = sk[e[q]];
          v[t] = dot_part(r, sv);
        }
      }
      block_sum_dd<kSmallRed>(v, red);
      if (threadIdx.x < kSmallRed && q0 + threadIdx.x < mi) {
        dd mine = v[0];
#pragma unroll
        for (int t = 1; t < kSmallRed; ++t)
          if ((int)threadIdx.x == t) mine = v[t];
        sbeta[q0 + threadIdx.x] = __ddiv_rn(dd_round(mine), sgamma[ring_slot(i - mi + q0 + threadIdx.x, m)]);
      }
    }
    __syncthreads();
    // p = w - sum beta_k p_k, newest -> oldest (R13); a non-finite w flags the system (R14)
    int bad = 0;
    double p[kSmallPT], s[kSmallPT];
#pragma unroll
    for (int q = 0; q < kSmallPT; ++q) {
      bad |= on[q] && !isfinite(r[q]);
      p[q] = r[q];
    }
    for (int t = mi - 1; t >= 0; --t) {
      const double* pk = ring_p + (size_t)ring_slot(i - mi + t, m) * N;
      const double bt = sbeta[t];
#pragma unroll
      for (int q = 0; q < kSmallPT; ++q) p[q] = __dsub_rn(p[q], __dmul_rn(bt, pk[e[q]]));
    }
#pragma unroll
    for (int q = 0; q < kSmallPT; ++q)
      if (on[q]) ring_p[(size_t)slot * N + e[q]] = p[q];   // slot i % (m+1) is outside the window: no reader
    bad = __syncthreads_or(bad);
    // s = A p; gamma = (p, s), alpha = (p, r) / gamma
#pragma unroll
    for (int q = 0; q < kSmallPT; ++q) {
      s[q] = on[q] ? apply(ring_p + (size_t)slot * N, q) : 0.0;
      if (on[q]) ring_s[(size_t)slot * N + e[q]] = s[q];
    }
    dd v[2] = {dot_part(p, s), dot_part(p, r)};
    block_sum_dd<2>(v, red);
    const double gamma = dd_round(v[0]);
    if (threadIdx.x == 0) sgamma[slot] = gamma;
    int fl = bad ? FLAG_NONFINITE : 0;
    if (!(gamma > 0.0) || !isfinite(gamma)) fl |= FLAG_BREAKDOWN;
    if (fl) {
      status = (fl & FLAG_NONFINITE) ? SYS_NONFINITE : SYS_BREAKDOWN;
      iters = i;
      break;
    }
    const double alpha = __ddiv_rn(dd_round(v[1]), gamma);
    // u += alpha p; r -= alpha s; ||r|| / ||r0||
#pragma unroll
    for (int q = 0; q < kSmallPT; ++q) {
      u[q] = __dadd_rn(u[q], __dmul_rn(alpha, p[q]));
      r[q] = __dsub_rn(r[q], __dmul_rn(alpha, s[q]));
    }
    dd w[1] = {dot_part(r, r)};
    block_sum_dd<1>(w, red);
    const double h = __ddiv_rn(__dsqrt_rn(dd_round(w[0])), rho0);
    if (threadIdx.x == 0 && d.hist) d.hist[(size_t)b * (d.maxit + 1) + i + 1] = h;
    if (h <= d.tol) { status = SYS_CONVERGED; iters = i + 1; }
    else if (i + 1 >= d.maxit) { status = SYS_MAXIT; iters = d.maxit; }
  }
#pragma unroll
  for (int q = 0; q < kSmallPT; ++q)
    if (on[q]) d.u[base + e[q]] = u[q];
  if (threadIdx.x == 0) {
    d.status[b] = status;
    d.iters[b] = iters;
  }
}

size_t fcg_small_smem(int n, int m) {
  const size_t N = (size_t)n * n;
  return 2 * (size_t)(m + 1) * N * sizeof(double) + 33 * kSmallRed * sizeof(dd);
}

// The persistent path applies to fp64 identity solves with n^2 <= 1024 whose ring fits shared memory.
bool fcg_small_applies(int n, int m) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("FCGNO_PERSISTENT");
    enabled = (e && e[0] == '0') ? 0 : 1;
  }
  return enabled && n * n <= 1024 && fcg_small_smem(n, m) <= 200u * 1024u;
}

cudaError_t launch_fcg_small(const FcgDev& d, cudaStream_t s) {
  static size_t attr = 0;
  const size_t smem = fcg_small_smem(d.n, d.m);
  if (smem > attr) {
    const cudaError_t e = cudaFuncSetAttribute((const void*)k_fcg_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int threads = ((d.N + kSmallPT - 1) / kSmallPT + 31) & ~31;
  k_fcg_small<<<d.B, threads, smem, s>>>(d);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace fcgno

// fcg_kernels.cu — matrix-free stencil, inner products and the FCG(m) step kernels.
//
// One FCG iteration (Algorithm 1) is split into five launches, each one
// HBM sweep over the vectors it touches; every reduction finishes inside the producing kernel
// (last CTA of a system reduces its partials in a fixed order), so the only scalar launch is
// k_finalize:
//   [NO output or k_window_dots]  (w, s_k) for the m_i window      -> beta_k = (w,s_k)/(p_k,s_k)
//   k_pform                        p = w - sum beta_k p_k            (newest -> oldest)
//   k_stencil_dots                 s = A p ; (p,s), (p,r)            -> alpha, breakdown
//   k_update                       u += alpha p ; r -= alpha s ; (r,r)
//   k_finalize                     ||r||/||r0||, status, iteration counter
// All arithmetic is fp64 in the oracle's operation order (R5, R6, R13) so identity
// runs reproduce the oracle's residual histories bit for bit.
#include "internal.h"
#include "fcg_device.cuh"

namespace fcgno {

uint64_t& launch_counter() {
  static uint64_t c = 0;
  return c;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FCGNO_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static inline dim3 sys_grid(int nblk, int B) { return dim3((unsigned)nblk, (unsigned)B, 1); }


// ------------------------------------------------------------------ apply_A
__global__ void __launch_bounds__(kThreads) k_apply_A(const double* __restrict__ k, const double* __restrict__ x,
                                                      double* __restrict__ y, int n, int N, double scale) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const double* kb = k + (size_t)b * N;
  const double* xb = x + (size_t)b * N;
  double* yb = y + (size_t)b * N;
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = blockIdx.x * kTile + q * kThreads + threadIdx.x;
    if (e < N) {
      const int i = e / n, j = e - i * n;
      yb[e] = stencil_at(kb, xb, n, i, j, scale);
    }
  }
}

cudaError_t launch_apply_A(const double* k, const double* x, double* y, int n, int B, cudaStream_t s) {
  const int N = n * n, nblk = (N + kTile - 1) / kTile;
  cudaError_t e = launch_k(k_apply_A, sys_grid(nblk, B), dim3(kThreads), 0, s, k, x, y, n, N, double(n + 1) * double(n + 1));
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ batched dot
__global__ void __launch_bounds__(kThreads) k_dot(const double* __restrict__ x, const double* __restrict__ y,
                                                  double* __restrict__ out, dd* part, unsigned* cnt, int N,
                                                  int nblk) {
  pdl_wait();
  pdl_trigger();
  __shared__ dd sm[8];
  const int b = blockIdx.y;
  double s = 0.0, c = 0.0;
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = blockIdx.x * kTile + q * kThreads + threadIdx.x;
    if (e < N) dot2_acc(x[(size_t)b * N + e], y[(size_t)b * N + e], s, c);
  }
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) part[(size_t)b * nblk + blockIdx.x] = v[0];
  if (arrive_last(cnt + b, nblk)) {
    const dd t = block_reduce_partials(part + (size_t)b * nblk, nblk, 1, sm);
    if (threadIdx.x == 0) out[b] = dd_round(t);
  }
}

cudaError_t launch_dot(const double* x, const double* y, double* out, dd* part, unsigned* cnt, int n, int B,
                       cudaStream_t s) {
  const int N = n * n, nblk = (N + kTile - 1) / kTile;
  cudaError_t e = launch_k(k_dot, sys_grid(nblk, B), dim3(kThreads), 0, s, x, y, out, part, cnt, N, nblk);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ k validation
__global__ void k_check_k(const double* __restrict__ k, size_t count, int* bad) {
  pdl_wait();
  pdl_trigger();
  int local = 0;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count; t += (size_t)gridDim.x * blockDim.x) {
    const double v = k[t];
    if (!(v > 0.0) || !isfinite(v)) local = 1;
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

cudaError_t launch_check_k(const double* k, size_t count, int* bad, cudaStream_t s) {
  k_check_k<<<296, kThreads, 0, s>>>(k, count, bad);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ r0 = f - A u0
__global__ void __launch_bounds__(kThreads) k_init_residual(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  __shared__ dd sm[8];
  const int b = blockIdx.y, N = d.N;
  const double* kb = d.k + (size_t)b * N;
  const double* ub = d.u + (size_t)b * N;
  double s = 0.0, c = 0.0;
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = blockIdx.x * kTile + q * kThreads + threadIdx.x;
    if (e < N) {
      const int i = e / d.n, j = e - i * d.n;
      const double rv = __dsub_rn(d.f[(size_t)b * N + e], stencil_at(kb, ub, d.n, i, j, d.scale));
      d.r[(size_t)b * N + e] = rv;
      dot2_acc(rv, rv, s, c);
    }
  }
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) d.part_rr[(size_t)b * d.nblk + blockIdx.x] = v[0];
  if (arrive_last(d.cnt + 2 * d.B + b, d.nblk)) {
    const dd t = block_reduce_partials(d.part_rr + (size_t)b * d.nblk, d.nblk, 1, sm);
    if (threadIdx.x == 0) {
      const double rr = dd_round(t);
      const double rho0 = __dsqrt_rn(rr);
      d.rr[b] = rr;
      d.rho0[b] = rho0;
      d.flags[b] = 0;
      d.iters[b] = 0;
      if (d.hist) d.hist[(size_t)b * (d.maxit + 1)] = 1.0;
      d.status[b] = (rho0 == 0.0) ? SYS_CONVERGED : (d.maxit == 0 ? SYS_MAXIT : SYS_RUNNING);
      if (d.status[b] == SYS_RUNNING) atomicAdd(d.active, 1);
    }
  }
}

cudaError_t launch_init_residual(const FcgDev& d, cudaStream_t s) {
  cudaError_t e = launch_k(k_init_residual, sys_grid(d.nblk, d.B), dim3(kThreads), 0, s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) k_window_dots(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  if (d.status[b] != SYS_RUNNING) return;
  const int i = *d.iter;
  const int mi = m_schedule(i, d.m, d.schedule);
  if (mi == 0) return;
  double wv[kPerThread];
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = blockIdx.x * kTile + q * kThreads + threadIdx.x;
    wv[q] = e < d.N ? d.w[(size_t)b * d.N + e] : 0.0;
  }
  window_dots_beta(d, b, blockIdx.x, i, mi, wv);
}

cudaError_t launch_window_dots(const FcgDev& d, cudaStream_t s) {
  cudaError_t e = launch_k(k_window_dots, sys_grid(d.nblk, d.B), dim3(kThreads), 0, s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ p = w - sum beta_k p_k ; s = A p ; (p,s), (p,r)
// One CTA per (tile of kTile elements, system).  p is formed for the tile plus a one-row halo on
// each side (the halo values are recomputed here, bit-identical to the owning CTA's), kept in
// shared memory for the stencil, and written to the ring for the tile only.
__global__ void __launch_bounds__(kThreads) k_pform_stencil(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double sp[];   // p over [lo, hi)
  __shared__ dd sm[16];
  __shared__ double sbeta[kMmax];
  __shared__ int sslot[kMmax];
  const int b = blockIdx.y;
  if (d.status[b] != SYS_RUNNING) return;
  const int i = *d.iter;
  const int mi = m_schedule(i, d.m, d.schedule);
  const int N = d.N, n = d.n, slot = ring_slot(i, d.m);
  const int e0 = blockIdx.x * kTile, e1 = min(N, e0 + kTile);
  const int lo = max(0, e0 - n), hi = min(N, e1 + n);
  for (int q = threadIdx.x; q < mi; q += blockDim.x) {
    sbeta[q] = d.beta[(size_t)b * kMmax + q];
    sslot[q] = ring_slot(i - mi + q, d.m);
  }
  __syncthreads();
  double* pout = d.ring_p + ((size_t)slot * d.B + b) * N;
  const double* wb = d.w + (size_t)b * N;
  int bad = 0;
  for (int e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    const double wv = wb[e];
    double p = wv;
    for (int t = mi - 1; t >= 0; --t)   // newest -> oldest (R13)
      p = __dsub_rn(p, __dmul_rn(sbeta[t], d.ring_p[((size_t)sslot[t] * d.B + b) * N + e]));
    sp[e - lo] = p;
    if (e >= e0 && e < e1) {
      if (!isfinite(wv)) bad = 1;
      pout[e] = p;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(d.flags + b, FLAG_NONFINITE);
  const double* kb = d.k + (size_t)b * N;
  double* sb = d.ring_s + ((size_t)slot * d.B + b) * N;
  double s0 = 0.0, c0 = 0.0, s1 = 0.0, c1 = 0.0;
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = e0 + q * kThreads + threadIdx.x;
    if (e < N) {
      const int ii = e / n, j = e - ii * n;
      const double sv = stencil_at(kb, sp, n, ii, j, d.scale, lo);
      sb[e] = sv;
      const double pv = sp[e - lo];
      dot2_acc(pv, sv, s0, c0);
      dot2_acc(pv, d.r[(size_t)b * N + e], s1, c1);
    }
  }
  dd v[2] = {dot2_finish(s0, c0), dot2_finish(s1, c1)};
  block_reduce_dd<2>(v, sm);
  if (threadIdx.x == 0) {
    d.part_step[((size_t)b * d.nblk + blockIdx.x) * 2 + 0] = v[0];
    d.part_step[((size_t)b * d.nblk + blockIdx.x) * 2 + 1] = v[1];
  }
  if (arrive_last(d.cnt + d.B + b, d.nblk)) {
    dd g, p;
    if (d.nblk <= kSerialPartials) {
      if (threadIdx.x == 0) {
        g = serial_partials(d.part_step + (size_t)b * d.nblk * 2 + 0, d.nblk, 2);
        p = serial_partials(d.part_step + (size_t)b * d.nblk * 2 + 1, d.nblk, 2);
      }
    } else {
      g = block_reduce_partials(d.part_step + (size_t)b * d.nblk * 2 + 0, d.nblk, 2, sm);
      p = block_reduce_partials(d.part_step + (size_t)b * d.nblk * 2 + 1, d.nblk, 2, sm);
    }
    if (threadIdx.x == 0) {
      const double gamma = dd_round(g);
      d.gamma[(size_t)slot * d.B + b] = gamma;
      if (!(gamma > 0.0) || !isfinite(gamma)) atomicOr(d.flags + b, FLAG_BREAKDOWN);
      d.alpha[b] = __ddiv_rn(dd_round(p), gamma);
    }
  }
}

size_t pform_stencil_smem(int n) { return (size_t)(kTile + 2 * n) * sizeof(double); }

cudaError_t launch_pform_stencil(const FcgDev& d, cudaStream_t s) {
  static size_t set = 0;
  const size_t smem = pform_stencil_smem(d.n);
  if (smem > 48 * 1024 && smem > set) {   // never during graph capture of a smaller size
    const cudaError_t e = cudaFuncSetAttribute((const void*)k_pform_stencil, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set = smem;
  }
  cudaError_t e = launch_k(k_pform_stencil, sys_grid(d.nblk, d.B), dim3(kThreads), smem, s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ u += alpha p ; r -= alpha s ; (r,r) ; bookkeeping
// The last CTA of each system reduces (r, r) and applies the system's convergence / breakdown
// bookkeeping (Algorithm 1's stopping test); the last system to arrive publishes the number of
// systems still running and advances the iteration counter.  Systems flagged this iteration
// skip the vector update but still take part in the arrival protocol.
__global__ void __launch_bounds__(kThreads) k_update(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  __shared__ dd sm[8];
  const int b = blockIdx.y;
  if (d.status[b] != SYS_RUNNING) return;
  const int i = *d.iter;
  const int fl = d.flags[b];
  const int N = d.N, slot = ring_slot(i, d.m);
  double s = 0.0, c = 0.0;
  if (fl == 0) {
    const double alpha = d.alpha[b];
    const double* pb = d.ring_p + ((size_t)slot * d.B + b) * N;
    const double* sb = d.ring_s + ((size_t)slot * d.B + b) * N;
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
      const int e = blockIdx.x * kTile + q * kThreads + threadIdx.x;
      if (e < N) {
        const size_t g = (size_t)b * N + e;
        d.u[g] = __dadd_rn(d.u[g], __dmul_rn(alpha, pb[e]));
        const double rv = __dsub_rn(d.r[g], __dmul_rn(alpha, sb[e]));
        d.r[g] = rv;
        dot2_acc(rv, rv, s, c);
      }
    }
  }
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) d.part_rr[(size_t)b * d.nblk + blockIdx.x] = v[0];
  if (!arrive_last(d.cnt + 2 * d.B + b, d.nblk)) return;
  bool running = false;
  if (fl == 0) {
    dd t;
    if (d.nblk <= kSerialPartials) {
      if (threadIdx.x == 0) t = serial_partials(d.part_rr + (size_t)b * d.nblk, d.nblk, 1);
    } else {
      t = block_reduce_partials(d.part_rr + (size_t)b * d.nblk, d.nblk, 1, sm);
    }
    if (threadIdx.x == 0) {
      const double rr = dd_round(t);
      d.rr[b] = rr;
      const double h = __ddiv_rn(__dsqrt_rn(rr), d.rho0[b]);
      if (d.hist) d.hist[(size_t)b * (d.maxit + 1) + i + 1] = h;
      if (h <= d.tol) { d.status[b] = SYS_CONVERGED; d.iters[b] = i + 1; }
      else if (i + 1 >= d.maxit) { d.status[b] = SYS_MAXIT; d.iters[b] = d.maxit; }
      else running = true;
    }
  } else if (threadIdx.x == 0) {
    d.status[b] = (fl & FLAG_NONFINITE) ? SYS_NONFINITE : SYS_BREAKDOWN;
    d.iters[b] = i;
  }
  if (threadIdx.x == 0) {
    const int expected = *d.active;          // systems running at the start of this iteration
    if (running) atomicAdd(d.gcnt + 1, 1u);
    __threadfence();
    const unsigned prev = atomicAdd(d.gcnt, 1u);
    if (prev == (unsigned)(expected - 1)) {  // last system: publish and re-arm
      __threadfence();
      *d.active = (int)atomicExch(d.gcnt + 1, 0u);
      *d.gcnt = 0u;
      *d.iter = i + 1;
    }
  }
}

cudaError_t launch_update(const FcgDev& d, cudaStream_t s) {
  cudaError_t e = launch_k(k_update, sys_grid(d.nblk, d.B), dim3(kThreads), 0, s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace fcgno

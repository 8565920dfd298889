// fcg_kernels.cu — matrix-free stencil, inner products and the FCG(m) step kernels.
//
// One FCG iteration (Algorithm 1) is two launches after the preconditioner, each
// one HBM sweep over the vectors it touches; every reduction finishes inside the producing kernel
// (the last CTA of a system reduces its partials in a fixed order), so there is no scalar-only
// launch:
//   [k_no_out* | k_window_dots]  w = B(r); (w, s_k) for the m_i window -> beta_k = (w,s_k)/(p_k,s_k)
//   k_pform_stencil           u += alpha_{i-1} p_{i-1} (lazy x update); p = w - sum beta_k p_k
//                             (newest -> oldest); s = A p; (p,s), (p,r) -> alpha, breakdown
//   k_update                  r -= alpha s; (r,r); ||r||/||r0||, status, iteration counter
//
//   k_flush_x (once, after the solve)  the last lazy x update of the stopped systems
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



// ------------------------------------------------------------------ apply_A
// 2-D tiles (fcg_device.cuh st_fill / st_walk): x and k staged once with a one-cell halo, every
// face computed once.  Grid (st_tiles(n), B), kStThreads threads, RG = st_rg(n) rows per thread.
#define ST_SMEM                                                   \
  __shared__ __align__(16) double sx[(kStR + 2) * kStSP];        \
  __shared__ __align__(16) double sk[(kStR + 2) * kStSP];        \
  __shared__ double sbnd[kStR * (kStThreads / 32 + 1)]

// launch KERNEL<RG, PAIRS, V> for the row-group size of n; PAIRS (column pairs) when n is even; V
// the storage type of the FCG vectors (double, or float with opts.vec_fp32, reading R21)
#define ST_LAUNCH2(err, PAIRS, V, n, KERNEL, grid, s, ...)                                                    \
  switch (st_rg(n)) {                                                                                         \
    case 1: err = launch_k(KERNEL<1, PAIRS, V>, grid, dim3(kStThreads), 0, s, __VA_ARGS__); break;            \
    case 2: err = launch_k(KERNEL<2, PAIRS, V>, grid, dim3(kStThreads), 0, s, __VA_ARGS__); break;            \
    case 4: err = launch_k(KERNEL<4, PAIRS, V>, grid, dim3(kStThreads), 0, s, __VA_ARGS__); break;            \
    default: err = launch_k(KERNEL<8, PAIRS, V>, grid, dim3(kStThreads), 0, s, __VA_ARGS__); break;           \
  }
#define ST_LAUNCH(err, n, V, KERNEL, grid, s, ...)                       \
  if ((n) % 2 == 0) {                                                   \
    ST_LAUNCH2(err, true, V, n, KERNEL, grid, s, __VA_ARGS__)           \
  } else {                                                              \
    ST_LAUNCH2(err, false, V, n, KERNEL, grid, s, __VA_ARGS__)          \
  }
#define ST_LAUNCH_VEC(err, d, KERNEL, grid, s, ...)                     \
  if ((d).vec32) {                                                      \
    ST_LAUNCH(err, (d).n, float, KERNEL, grid, s, __VA_ARGS__)          \
  } else {                                                              \
    ST_LAUNCH(err, (d).n, double, KERNEL, grid, s, __VA_ARGS__)         \
  }

template <int RG, bool PAIRS, typename V>   // V unused: apply_A works on caller fp64 vectors
__global__ void __launch_bounds__(kStThreads, 4) k_apply_A(const double* __restrict__ k, const double* __restrict__ x,
                                                           double* __restrict__ y, int n, double scale, int fast) {
  pdl_wait();
  pdl_trigger();
  ST_SMEM;
  const int b = blockIdx.y;
  const size_t N = (size_t)n * n;
  const StGeo g = st_geo(n);
  const double* xb = x + b * N;
  double* yb = y + b * N;
  st_copy<PAIRS>(g, n, k + b * N, sk);
  st_copy<PAIRS>(g, n, xb, sx);
  st_fill_end();
  const StWalk<RG> w(g);
  const double none[RG] = {};
  st_walk_any<RG>(fast, g, w, n, scale, sx, sk, sbnd, none, [&](bool ok, int e, double, double v, double, double) {
    if (ok) yb[e] = v;
  });
}

cudaError_t launch_apply_A(const double* k, const double* x, double* y, int n, int B, bool kfast, cudaStream_t s) {
  cudaError_t e;
  ST_LAUNCH(e, n, double, k_apply_A, dim3((unsigned)st_tiles(n), (unsigned)B), s, k, x, y, n, double(n + 1) * double(n + 1),
            kfast ? 1 : 0);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ classical stationary preconditioners
// Jacobi(k) (Eq. 15) and symmetric Gauss-Seidel(k) in red-black order (readings
// R22-R24) as stencil sweeps over the 2-D tiles.  One launch = one sweep over the nodes of `colour`
// (-1: every node, a Jacobi sweep x -> xout; 0 / 1: a red / black half sweep, in place):
//   x_e <- x_e + (z_e - (A x)_e) / a_ee                  (R23; x = 0 on the first sweep)
// and, on the last sweep, w = the new x at every node, stored in the FCG vector type V.
template <int RG, bool PAIRS, typename V>
__global__ void __launch_bounds__(kStThreads, 4) k_stationary(const double* __restrict__ k, const V* __restrict__ z,
                                                              const double* x, double* xout, V* __restrict__ w, int n,
                                                              double scale, int fast, int colour, int first,
                                                              const int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  ST_SMEM;
  const int b = blockIdx.y;
  if (status && status[b] != SYS_RUNNING) return;
  const size_t N = (size_t)n * n;
  const StGeo g = st_geo(n);
  st_copy<PAIRS>(g, n, k + b * N, sk);
  if (first) {
    for (int t = threadIdx.x; t < (kStR + 2) * kStSP; t += blockDim.x) sx[t] = 0.0;
  } else {
    st_copy<PAIRS>(g, n, x + b * N, sx);
  }
  st_fill_end();
  const StWalk<RG> wk(g);
  double zx[RG];
  st_rows<RG, V>(g, wk, n, z + b * N, zx);
  double* xo = xout + b * N;
  V* wo = w ? w + b * N : nullptr;
  st_walk_any<RG>(fast != 0, g, wk, n, scale, sx, sk, sbnd, zx, [&](bool ok, int e, double xc, double ax, double zv, double aee) {
    if (!ok) return;
    const int i = e / n, j = e - i * n;
    const bool upd = colour < 0 || ((i + j) & 1) == colour;
    const double v = upd ? __dadd_rn(xc, __ddiv_rn(__dsub_rn(zv, ax), aee)) : xc;
    if (upd || first) xo[e] = v;
    if (wo) wo[e] = (V)v;
  });
}

template <typename V>
static cudaError_t launch_stationary_t(const double* k, const V* z, double* xa, double* xb, V* w, int n, int B,
                                       bool kfast, int kind, int sweeps, const int* status, cudaStream_t s) {
  const dim3 grid((unsigned)st_tiles(n), (unsigned)B);
  const double scale = double(n + 1) * double(n + 1);
  cudaError_t e = cudaSuccess;
  if (kind == 1) {   // Jacobi: sweeps x_{s-1} -> x_s, ping-pong
    for (int sw = 0; sw < sweeps && e == cudaSuccess; ++sw) {
      const double* xin = (sw & 1) ? xa : xb;
      double* xo = (sw & 1) ? xb : xa;
      ST_LAUNCH(e, n, V, k_stationary, grid, s, k, z, xin, xo, sw == sweeps - 1 ? w : nullptr, n, scale, kfast ? 1 : 0,
                -1, sw == 0 ? 1 : 0, status);
      ++launch_counter();
    }
  } else {           // red-black SGS: per sweep L^-1 (red, black) then U^-1 (black, red), in place
    const int seq[4] = {0, 1, 1, 0};
    for (int sw = 0; sw < sweeps && e == cudaSuccess; ++sw)
      for (int h = 0; h < 4 && e == cudaSuccess; ++h) {
        const bool last = sw == sweeps - 1 && h == 3;
        ST_LAUNCH(e, n, V, k_stationary, grid, s, k, z, xa, xa, last ? w : nullptr, n, scale, kfast ? 1 : 0, seq[h],
                  (sw == 0 && h == 0) ? 1 : 0, status);
        ++launch_counter();
      }
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_stationary(const double* k, const void* z, double* xa, double* xb, void* w, bool v32, int n, int B,
                              bool kfast, int kind, int sweeps, const int* status, cudaStream_t s) {
  if (v32)
    return launch_stationary_t<float>(k, static_cast<const float*>(z), xa, xb, static_cast<float*>(w), n, B, kfast, kind,
                                      sweeps, status, s);
  return launch_stationary_t<double>(k, static_cast<const double*>(z), xa, xb, static_cast<double*>(w), n, B, kfast,
                                     kind, sweeps, status, s);
}

// ------------------------------------------------------------------ batched dot
template <int EPT>
__global__ void __launch_bounds__(kThreads) k_dot(const double* __restrict__ x, const double* __restrict__ y,
                                                  double* __restrict__ out, dd* part, unsigned* cnt, int N, int cap) {
  pdl_wait();
  pdl_trigger();
  __shared__ dd sm[8];
  const int b = blockIdx.y;
  const double* xb = x + (size_t)b * N;
  const double* yb = y + (size_t)b * N;
  double xv[EPT], yv[EPT];
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = (blockIdx.x * EPT + q) * kThreads + threadIdx.x;
    xv[q] = e < N ? xb[e] : 0.0;
    yv[q] = e < N ? yb[e] : 0.0;
  }
  double s = 0.0, c = 0.0;
#pragma unroll
  for (int q = 0; q < EPT; ++q) dot2_acc(xv[q], yv[q], s, c);
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) part[(size_t)b * cap + blockIdx.x] = v[0];
  const int nb = gridDim.x;
  if (arrive_last(cnt + b, nb)) {
    const dd t = block_reduce_partials(part + (size_t)b * cap, nb, 1, sm);
    if (threadIdx.x == 0) out[b] = dd_round(t);
  }
}

cudaError_t launch_dot(const double* x, const double* y, double* out, dd* part, unsigned* cnt, int n, int B,
                       cudaStream_t s) {
  const int N = n * n, cap = part_cap(n);
  cudaError_t e;
  if (ew_wide(n, B))
    e = launch_k(k_dot<kEptWide>, dim3((unsigned)ew_blocks(n, kEptWide), (unsigned)B), dim3(kThreads), 0, s, x, y,
                 out, part, cnt, N, cap);
  else
    e = launch_k(k_dot<kPerThread>, dim3((unsigned)ew_blocks(n, kPerThread), (unsigned)B), dim3(kThreads), 0, s, x,
                 y, out, part, cnt, N, cap);
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
    if (!(v > 0.0) || !isfinite(v)) local |= 1;
    if (!k_inrange(v)) local |= 2;   // outside the branch-free division's range (fcg_device.cuh)
  }
  const int any1 = __syncthreads_or(local & 1), any2 = __syncthreads_or(local & 2);
  if (threadIdx.x == 0 && (any1 || any2)) atomicOr(bad, (any1 ? 1 : 0) | (any2 ? 2 : 0));
}

cudaError_t launch_check_k(const double* k, size_t count, int* bad, cudaStream_t s) {
  k_check_k<<<296, kThreads, 0, s>>>(k, count, bad);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ r0 = f - A u0
template <int RG, bool PAIRS, typename V>
__global__ void __launch_bounds__(kStThreads, 3) k_init_residual(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  ST_SMEM;
  __shared__ dd sm[8];
  const int b = blockIdx.y, n = d.n;
  const size_t N = (size_t)d.N;
  const StGeo g = st_geo(n);
  const double* ub = d.u + b * N;
  V* rb = reinterpret_cast<V*>(d.r) + b * N;
  double* r64 = d.r64 ? d.r64 + b * N : nullptr;   // fp64 copy of an fp32 r for the NO input
  const bool fast = d.kfast != 0;
  st_copy<PAIRS>(g, n, d.k + b * N, sk);
  st_copy<PAIRS>(g, n, ub, sx);
  st_fill_end();
  const StWalk<RG> w(g);
  double fx[RG];
  st_rows(g, w, n, d.f + b * N, fx);
  double s = 0.0, c = 0.0;
  st_walk_any<RG>(fast, g, w, n, d.scale, sx, sk, sbnd, fx, [&](bool ok, int e, double, double v, double fv, double) {
    const double rv = ok ? rnd<V>(__dsub_rn(fv, v)) : 0.0;   // stored value (R21)
    if (ok) {
      rb[e] = (V)rv;
      if (r64) r64[e] = rv;
    }
    dot2_acc(rv, rv, s, c);
  });
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) d.part_rr[(size_t)b * d.nblk + blockIdx.x] = v[0];
  const int nb = gridDim.x;
  if (arrive_last(d.cnt + 2 * d.B + b, nb)) {
    const dd t = block_reduce_partials(d.part_rr + (size_t)b * d.nblk, nb, 1, sm);
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
  cudaError_t e;
  ST_LAUNCH_VEC(e, d, k_init_residual, dim3((unsigned)st_tiles(d.n), (unsigned)d.B), s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ (w, s_k) window dots (identity B)
template <int EPT, typename V>
__global__ void __launch_bounds__(kThreads, 2) k_window_dots(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  if (d.status[b] != SYS_RUNNING) return;
  const int i = *d.iter;
  const int mi = m_schedule(i, d.m, d.schedule);
  if (mi == 0) return;
  double wv[EPT];
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = (blockIdx.x * EPT + q) * kThreads + threadIdx.x;
    wv[q] = e < d.N ? (double)reinterpret_cast<const V*>(d.w)[(size_t)b * d.N + e] : 0.0;
  }
  window_dots_pairs<EPT, V>(d, b, blockIdx.x, i, mi, wv);
}

// Wide batches: 32 elements per thread, w kept in (dynamic) shared memory by its own thread.
constexpr int kEptWin = 32;
template <typename V>
__global__ void __launch_bounds__(kThreads, 2) k_window_dots_smem(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double wsm[];   // [kEptWin][kThreads]
  const int b = blockIdx.y;
  if (d.status[b] != SYS_RUNNING) return;
  const int i = *d.iter;
  const int mi = m_schedule(i, d.m, d.schedule);
  if (mi == 0) return;
  const V* wb = reinterpret_cast<const V*>(d.w) + (size_t)b * d.N;
#pragma unroll 8
  for (int q = 0; q < kEptWin; ++q) {
    const int e = (blockIdx.x * kEptWin + q) * kThreads + threadIdx.x;
    wsm[q * kThreads + threadIdx.x] = e < d.N ? (double)__ldg(wb + e) : 0.0;
  }
  window_dots_pairs_smem<kEptWin, V>(d, b, blockIdx.x, i, mi, wsm);
}

template <typename V>
static cudaError_t launch_window_dots_t(const FcgDev& d, cudaStream_t s) {
  if (ew_wide(d.n, d.B)) {
    static bool attr = false;
    const int smem = kEptWin * kThreads * (int)sizeof(double);
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute((const void*)k_window_dots_smem<float>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)k_window_dots_smem<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    return launch_k(k_window_dots_smem<V>, dim3((unsigned)ew_blocks(d.n, kEptWin), (unsigned)d.B), dim3(kThreads),
                    (size_t)smem, s, d);
  }
  return launch_k(k_window_dots<kPerThread, V>, dim3((unsigned)ew_blocks(d.n, kPerThread), (unsigned)d.B),
                  dim3(kThreads), 0, s, d);
}

cudaError_t launch_window_dots(const FcgDev& d, cudaStream_t s) {
  const cudaError_t e = d.vec32 ? launch_window_dots_t<float>(d, s) : launch_window_dots_t<double>(d, s);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ p = w - sum beta_k p_k ; s = A p ; (p,s), (p,r)
// One CTA per 2-D tile of one system.  Phase 1 forms p over the tile and its one-cell halo (halo
// values recomputed, bit-identical to the owning CTA's) into shared memory and writes the tile's
// p to the ring; phase 2 applies the stencil from shared memory, writes s and accumulates (p,s)
// and (p,r).  The system's last CTA forms gamma = (p,s), alpha = (p,r)/gamma and flags breakdown.
template <int RG, bool PAIRS, typename V>
__global__ void __launch_bounds__(kStThreads, 3) k_pform_stencil(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  ST_SMEM;
  __shared__ dd sm[2 * (kStThreads / 32)];
  __shared__ double sbeta[kMmax];
  __shared__ const V* sptr[kMmax];
  const int b = blockIdx.y;
  const int n = d.n;
  const size_t N = (size_t)d.N;
  const StGeo g = st_geo(n);
  st_copy<PAIRS>(g, n, d.k + b * N, sk);   // independent of the iteration state: in flight first
  if (d.status[b] != SYS_RUNNING) {
    cp_async_wait_all();
    return;
  }
  const int i = *d.iter;
  const int mi = m_schedule(i, d.m, d.schedule);
  const int slot = ring_slot(i, d.m);
  for (int q = threadIdx.x; q < mi; q += blockDim.x) {
    sbeta[q] = d.beta[(size_t)b * kMmax + q];
    sptr[q] = reinterpret_cast<const V*>(d.ring_p) + ((size_t)ring_slot(i - mi + q, d.m) * d.B + b) * N;
  }
  __syncthreads();
  V* pout = reinterpret_cast<V*>(d.ring_p) + ((size_t)slot * d.B + b) * N;
  const V* wb = reinterpret_cast<const V*>(d.w) + b * N;
  const bool fast = d.kfast != 0;
  // lazy x update of the previous iteration, u += alpha_{i-1} p_{i-1}, inside
  // the p-form's first batch of loads (p_{i-1} is the newest window vector): the same single rounding
  // as in k_update's place, one sweep of u fewer.  alpha[b] still holds alpha_{i-1}: this launch's
  // last CTA overwrites it only after every CTA has passed here.
  const int bad = st_pform<PAIRS, V>(g, n, wb, sptr, sbeta, mi, sx, pout, d.u + b * N, i > 0 ? d.alpha[b] : 0.0, i > 0);
  cp_async_wait_all();
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(d.flags + b, FLAG_NONFINITE);
  const StWalk<RG> w(g);
  double rx[RG];
  st_rows<RG, V>(g, w, n, reinterpret_cast<const V*>(d.r) + b * N, rx);
  V* sout = reinterpret_cast<V*>(d.ring_s) + ((size_t)slot * d.B + b) * N;
  double s0 = 0.0, c0 = 0.0, s1 = 0.0, c1 = 0.0;
  st_walk_any<RG>(fast, g, w, n, d.scale, sx, sk, sbnd, rx, [&](bool ok, int e, double pv, double sv, double rv, double) {
    const double sr = rnd<V>(sv);   // s as stored (R21)
    if (ok) sout[e] = (V)sr;
    const double p = ok ? pv : 0.0, q = ok ? sr : 0.0;
    dot2_acc(p, q, s0, c0);
    dot2_acc(p, rv, s1, c1);
  });
  // (p,s), (p,r): warp sums, then warp 0 alone finishes (the other warps retire: no block-wide wait on
  // the arrival's fence + atomic round trip)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const dd vs = warp_sum2_dd(dot2_finish(s0, c0), dot2_finish(s1, c1), lane);   // lane 0: (p,s), lane 16: (p,r)
  if (lane == 0) sm[warp * 2 + 0] = vs;
  if (lane == 16) sm[warp * 2 + 1] = vs;
  __syncthreads();
  if (warp != 0) return;
  const int nb = gridDim.x;
  int last = 0;
  if (lane == 0) {
    dd a0 = sm[0], a1 = sm[1];
    for (int q = 1; q < kStThreads / 32; ++q) {   // fixed order over the warps
      a0 = dd_add(a0, sm[q * 2 + 0]);
      a1 = dd_add(a1, sm[q * 2 + 1]);
    }
    d.part_step[((size_t)b * d.nblk + blockIdx.x) * 2 + 0] = a0;
    d.part_step[((size_t)b * d.nblk + blockIdx.x) * 2 + 1] = a1;
    __threadfence();
    unsigned* counter = d.cnt + d.B + b;
    const unsigned prev = atomicAdd(counter, 1u);
    last = prev == (unsigned)(nb - 1);
    if (last) *counter = 0u;   // every CTA of this launch has arrived; safe to re-arm
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  // the system's last CTA: gamma = (p,s), alpha = (p,r)/gamma, breakdown flag
  dd gsum = {0.0, 0.0}, psum = {0.0, 0.0};
  const dd* part = d.part_step + (size_t)b * d.nblk * 2;
  if (nb <= kSerialPartials) {
    if (lane == 0) {
      gsum = serial_partials(part + 0, nb, 2);
      psum = serial_partials(part + 1, nb, 2);
    }
  } else {   // lanes stride over the CTAs' partials, then a shuffle tree (fixed order)
    for (int t = lane; t < nb; t += 32) {
      const double2 ga = __ldcg(reinterpret_cast<const double2*>(part + (size_t)t * 2 + 0));
      const double2 pa = __ldcg(reinterpret_cast<const double2*>(part + (size_t)t * 2 + 1));
      gsum = dd_add(gsum, dd{ga.x, ga.y});
      psum = dd_add(psum, dd{pa.x, pa.y});
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      gsum = dd_add(gsum, shfl_down_dd(gsum, off));
      psum = dd_add(psum, shfl_down_dd(psum, off));
    }
  }
  if (lane == 0) {
    const double gamma = dd_round(gsum);
    d.gamma[(size_t)slot * d.B + b] = gamma;
    if (!(gamma > 0.0) || !isfinite(gamma)) atomicOr(d.flags + b, FLAG_BREAKDOWN);
    d.alpha[b] = __ddiv_rn(dd_round(psum), gamma);
  }
}

cudaError_t launch_pform_stencil(const FcgDev& d, cudaStream_t s) {
  cudaError_t e;
  ST_LAUNCH_VEC(e, d, k_pform_stencil, dim3((unsigned)st_tiles(d.n), (unsigned)d.B), s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ r -= alpha s ; (r,r) ; bookkeeping
// u += alpha p is applied lazily by the next k_pform_stencil (or by k_flush_x after the solve), so
// this kernel streams r and s only.  The last CTA of each system reduces (r, r) and applies the system's
// convergence / breakdown bookkeeping (Algorithm 1's stopping test); the last system to arrive
// publishes the number of systems still running and advances the iteration counter.  Systems
// flagged this iteration skip the vector update but still take part in the arrival protocol.
template <int EPT, typename V>
__global__ void __launch_bounds__(kThreads, 2) k_update(FcgDev d) {
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
    const V* sb = reinterpret_cast<const V*>(d.ring_s) + ((size_t)slot * d.B + b) * N;
    V* rb = reinterpret_cast<V*>(d.r) + (size_t)b * N;
    double* r64 = d.r64 ? d.r64 + (size_t)b * N : nullptr;
    double rv[EPT], sv[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) {   // all loads first: EPT x 2 in flight
      const int e = (blockIdx.x * EPT + q) * kThreads + threadIdx.x;
      const bool ok = e < N;
      rv[q] = ok ? (double)rb[e] : 0.0;
      sv[q] = ok ? (double)__ldg(sb + e) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      const int e = (blockIdx.x * EPT + q) * kThreads + threadIdx.x;
      rv[q] = rnd<V>(__dsub_rn(rv[q], __dmul_rn(alpha, sv[q])));   // stored value (R21)
      if (e < N) {
        rb[e] = (V)rv[q];
        if (r64) r64[e] = rv[q];
      }
    }
#pragma unroll
    for (int q = 0; q < EPT; ++q) dot2_acc(rv[q], rv[q], s, c);
  }
  dd v[1] = {dot2_finish(s, c)};
  block_reduce_dd<1>(v, sm);
  if (threadIdx.x == 0) d.part_rr[(size_t)b * d.nblk + blockIdx.x] = v[0];
  const int nb = gridDim.x;
  if (!arrive_last(d.cnt + 2 * d.B + b, nb)) return;
  bool running = false;
  if (fl == 0) {
    dd t;
    if (nb <= kSerialPartials) {
      if (threadIdx.x == 0) t = serial_partials(d.part_rr + (size_t)b * d.nblk, nb, 1);
    } else {
      t = block_reduce_partials(d.part_rr + (size_t)b * d.nblk, nb, 1, sm);
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

// Condition of the device-side iteration loop (a CUDA-graph WHILE node, api.cu): run another chunk
// of iterations while any system of the batch is still running.
__global__ void k_loop_cond(const int* __restrict__ active, cudaGraphConditionalHandle h) {
  pdl_wait();
  cudaGraphSetConditional(h, *active > 0 ? 1u : 0u);
}

cudaError_t launch_loop_cond(const int* active, cudaGraphConditionalHandle h, cudaStream_t s) {
  cudaError_t e = launch_k(k_loop_cond, dim3(1), dim3(1), 0, s, active, h);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// After the solve: the last lazy x update of every system that stopped in k_update (converged or
// at maxit after >= 1 iteration), u += alpha_{iters-1} p_{iters-1}.
template <int EPT, typename V>
__global__ void __launch_bounds__(kThreads) k_flush_x(FcgDev d) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const int st = d.status[b], it = d.iters[b];
  if (!((st == SYS_CONVERGED || st == SYS_MAXIT) && it >= 1)) return;
  const int N = d.N;
  const double al = d.alpha[b];
  const V* pb = reinterpret_cast<const V*>(d.ring_p) + ((size_t)ring_slot(it - 1, d.m) * d.B + b) * N;
  double* ub = d.u + (size_t)b * N;
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = (blockIdx.x * EPT + q) * kThreads + threadIdx.x;
    if (e < N) ub[e] = __dadd_rn(ub[e], __dmul_rn(al, (double)pb[e]));
  }
}

cudaError_t launch_flush_x(const FcgDev& d, cudaStream_t s) {
  const dim3 grid((unsigned)ew_blocks(d.n, kPerThread), (unsigned)d.B);
  cudaError_t e = d.vec32 ? launch_k(k_flush_x<kPerThread, float>, grid, dim3(kThreads), 0, s, d)
                          : launch_k(k_flush_x<kPerThread, double>, grid, dim3(kThreads), 0, s, d);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

template <typename V>
static cudaError_t launch_update_t(const FcgDev& d, cudaStream_t s) {
  if (ew_wide(d.n, d.B))
    return launch_k(k_update<kEptUpdate, V>, dim3((unsigned)ew_blocks(d.n, kEptUpdate), (unsigned)d.B), dim3(kThreads),
                    0, s, d);
  return launch_k(k_update<kPerThread, V>, dim3((unsigned)ew_blocks(d.n, kPerThread), (unsigned)d.B), dim3(kThreads),
                  0, s, d);
}

cudaError_t launch_update(const FcgDev& d, cudaStream_t s) {
  const cudaError_t e = d.vec32 ? launch_update_t<float>(d, s) : launch_update_t<double>(d, s);
  if (e != cudaSuccess) return e;
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace fcgno

// diag_kernels.cu — Theorem-1 / Notay diagnostics (Theorem 1; Eq. final_loss,
// P:146-150):
//   eps(r) = || B(r) - A^{-1} r ||_A / || A^{-1} r ||_A ,  ||v||_A = sqrt((v, A v)),
// evaluated in its direct form: the difference d = c B(r) - e is formed first (c = 1, or the
// scale-free minimiser c* = (w, A e) / (w, A w)), then ||d||_A and ||e||_A each from one stencil
// application and one correctly rounded inner product, in the oracle's operation order
// (oracle/notay.py), so that no cancellation enters beyond the one in d itself.
//   k_notay_form   d = c_b w - e              (standalone fcgno_notay_ratio)
//   k_diag_state   e = u* - u_i, d = w_i - e  (inside fcgno_fcg_solve_diag, once per iteration; u_i
//                  is the iterate the lazy x update is about to form, u + alpha_{i-1} p_{i-1})
//   k_notay_coef   c_b = (w, A e)_b / (w, A w)_b
//   k_notay_final  eps_b = sqrt((d, A d)_b) / sqrt((e, A e)_b), ||e||_A = sqrt((e, A e)_b)
#include <algorithm>

#include "internal.h"
#include "fcg_device.cuh"

namespace fcgno {

__global__ void __launch_bounds__(kThreads) k_notay_form(const double* __restrict__ w, const double* __restrict__ e,
                                                          const double* __restrict__ c, double* __restrict__ d, int N) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const size_t base = (size_t)b * N;
  const double cb = c ? c[b] : 1.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N; t += gridDim.x * blockDim.x) {
    const double wv = w[base + t];
    d[base + t] = __dsub_rn(c ? __dmul_rn(cb, wv) : wv, e[base + t]);
  }
}

template <typename V>
__global__ void __launch_bounds__(kThreads) k_diag_state(FcgDev dv) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  if (dv.status[b] != SYS_RUNNING) return;
  const int i = *dv.iter, N = dv.N;
  const size_t base = (size_t)b * N;
  const V* w = reinterpret_cast<const V*>(dv.w) + base;
  const V* pprev = i > 0 ? reinterpret_cast<const V*>(dv.ring_p) + ((size_t)ring_slot(i - 1, dv.m) * dv.B + b) * N : nullptr;
  const double al = i > 0 ? dv.alpha[b] : 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N; t += gridDim.x * blockDim.x) {
    double u = dv.u[base + t];
    if (i > 0) u = __dadd_rn(u, __dmul_rn(al, (double)pprev[t]));   // the lazy update's single rounding
    const double e = __dsub_rn(dv.dg_ustar[base + t], u);
    dv.dg_e[base + t] = e;
    dv.dg_d[base + t] = __dsub_rn((double)w[t], e);
  }
}

__global__ void k_notay_coef(const double* __restrict__ wAe, const double* __restrict__ wAw, double* __restrict__ c,
                             int B) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) c[b] = __ddiv_rn(wAe[b], wAw[b]);
}

// out[b * stride + (iter ? *iter : 0)]; status (optional) skips stopped systems
__global__ void k_notay_final(const double* __restrict__ dAd, const double* __restrict__ eAe, double* __restrict__ eps,
                              double* __restrict__ err_a, const int* __restrict__ iter, size_t stride,
                              const int* __restrict__ status, int B) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || (status && status[b] != SYS_RUNNING)) return;
  const size_t at = (size_t)b * stride + (iter ? (size_t)*iter : 0);
  const double ne = __dsqrt_rn(eAe[b]);
  if (eps) eps[at] = __ddiv_rn(__dsqrt_rn(dAd[b]), ne);
  if (err_a) err_a[at] = ne;
}

static dim3 ew_grid(int n, int B) { return dim3((unsigned)std::min(ew_blocks(n, kPerThread), 1024), (unsigned)B); }

cudaError_t launch_notay_form(const double* w, const double* e, const double* c, double* d, int n, int B, cudaStream_t s) {
  const cudaError_t err = launch_k(k_notay_form, ew_grid(n, B), dim3(kThreads), 0, s, w, e, c, d, n * n);
  ++launch_counter();
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_notay_coef(const double* wAe, const double* wAw, double* c, int B, cudaStream_t s) {
  const cudaError_t err = launch_k(k_notay_coef, dim3((unsigned)((B + 127) / 128)), dim3(128), 0, s, wAe, wAw, c, B);
  ++launch_counter();
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_notay_final(const double* dAd, const double* eAe, double* eps, double* err_a, const int* iter,
                               size_t stride, const int* status, int B, cudaStream_t s) {
  const cudaError_t err = launch_k(k_notay_final, dim3((unsigned)((B + 127) / 128)), dim3(128), 0, s, dAd, eAe, eps,
                                   err_a, iter, stride, status, B);
  ++launch_counter();
  return err != cudaSuccess ? err : cudaGetLastError();
}

// One in-solve diagnostic step (after w_i = B(r_i), before k_pform_stencil).  Returns the launches.
int enqueue_diag(const FcgDev& d, cudaStream_t s) {
  cudaError_t e = d.vec32 ? launch_k(k_diag_state<float>, ew_grid(d.n, d.B), dim3(kThreads), 0, s, d)
                          : launch_k(k_diag_state<double>, ew_grid(d.n, d.B), dim3(kThreads), 0, s, d);
  if (e != cudaSuccess) return -1;
  if (launch_apply_A(d.k, d.dg_e, d.dg_Ae, d.n, d.B, d.kfast != 0, s) != cudaSuccess) return -1;
  if (launch_apply_A(d.k, d.dg_d, d.dg_Ad, d.n, d.B, d.kfast != 0, s) != cudaSuccess) return -1;
  if (launch_dot(d.dg_e, d.dg_Ae, d.dg_sc, d.dg_part, d.dg_cnt, d.n, d.B, s) != cudaSuccess) return -1;
  if (launch_dot(d.dg_d, d.dg_Ad, d.dg_sc + d.B, d.dg_part, d.dg_cnt, d.n, d.B, s) != cudaSuccess) return -1;
  if (launch_notay_final(d.dg_sc + d.B, d.dg_sc, d.dg_eps, d.dg_erra, d.iter, (size_t)d.maxit, d.status, d.B, s) !=
      cudaSuccess)
    return -1;
  ++launch_counter();
  return 6;
}

}  // namespace fcgno

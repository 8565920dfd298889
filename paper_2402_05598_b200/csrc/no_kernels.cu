// no_kernels.cu — spectral neural operator forward (§2.4.2, App. A).
//
// Per layer: analysis c = DFT_M(v) (M = {-10..9}^2), mode-diagonal complex channel mixing
// g[o](kappa) = sum_c R[c][o](kappa) c[c](kappa), synthesis z = n^-2 Re iDFT_M(g), bypass W v + b,
// GELU (R7-R11).  Kernel split:
//   k_dft_rows    DFT_M of r/||r|| (row-group partials)
//   k_lift_mix    layer-1 mixing with the lift folded in: g1 = A0 R^ + A1 K^ + n^2 delta A2
//   k_no_layer    one CTA per (system, group of GO output channels) streams the system's rows:
//                 y-synthesis of g for the rows -> bypass GEMV + x-synthesis + bias + GELU ->
//                 store v -> x-analysis -> y-analysis accumulated in registers -> c[kappa][b][o]
//   k_mix         mode-diagonal mixing for layers 2, 3 and (folded with the projection) 4
//   k_no_out      out = dw.v3 + cst + S(g4), w = ||r|| out, fused FCG window dots (w, s_k)
// Templated on T = float (production) or double (trajectory-parity mode).
#include <cstdio>

#include "internal.h"
#include "fcg_device.cuh"
#include "tc_common.cuh"

namespace fcgno {

template <typename T> struct Cplx;
template <> struct Cplx<float> { using type = float2; };
template <> struct Cplx<double> { using type = double2; };

__device__ __forceinline__ float gelu_t(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ double gelu_t(double x) { return 0.5 * x * (1.0 + erf(x * 0.70710678118654752440)); }

constexpr int kGhStride = kModes2 + 1;  // padded row of the per-channel mode array in smem
constexpr int kMixBatch = 32;    // systems per CTA of k_mix
constexpr int kMaxDynSmem = 227 * 1024;

// ------------------------------------------------------------------ twiddles
// basis 0 (Fourier, R7-R8): exp(-2 pi i kappa j / n), kappa = kx - 10;
// basis 1 (Chebyshev, R25): (cos(pi k (j + 1/2) / n), 0), k = kx: the complex machinery then carries
// zero imaginary parts and the synthesis Re(g F*) reduces to the cosine sum
__global__ void k_twiddles(float2* F32, double2* F64, int n, int basis) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * kModes) return;
  const int j = t / kModes, kx = t - j * kModes;
  double sn, cs;
  if (basis == 0) {
    const long long kap = kx - kModes / 2;
    const long long q = ((kap * j) % n + n) % n;       // exact phase reduction
    sincospi(2.0 * (double)q / (double)n, &sn, &cs);
    sn = -sn;
  } else {
    const long long q = ((long long)kx * (2 * j + 1)) % (4LL * n);   // pi k (2j + 1) / (2n), reduced exactly
    cs = cospi((double)q / (2.0 * (double)n));
    sn = 0.0;
  }
  F64[t] = make_double2(cs, sn);
  F32[t] = make_float2((float)cs, (float)sn);
}

cudaError_t launch_twiddles(float* F32, double* F64, int n, int basis, cudaStream_t s) {
  const int cnt = n * kModes;
  k_twiddles<<<(cnt + 255) / 256, 256, 0, s>>>(reinterpret_cast<float2*>(F32), reinterpret_cast<double2*>(F64), n, basis);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ DFT_M of an input field
// grid (ngroups, B).  x is fp64; for FROM_R the field is x * (1/||x||) with ||x|| = sqrt(rr[b]).
template <typename T, bool FROM_R>
__global__ void __launch_bounds__(256) k_dft_rows(const double* __restrict__ x, const double* __restrict__ rr,
                                                  const typename Cplx<T>::type* __restrict__ F,
                                                  typename Cplx<T>::type* __restrict__ part, int n, int ngroups,
                                                  const int* __restrict__ status, double* __restrict__ rinv) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  const int b = blockIdx.y, g = blockIdx.x;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int DR = dft_rows(n);
  T* X = reinterpret_cast<T*>(smraw);                               // [DR][n]
  T2* Tx = reinterpret_cast<T2*>(X + ((DR * n + 3) & ~3));          // [DR][20]
  const int N = n * n, i0 = g * DR, rows = min(DR, n - i0);
  double inv = 1.0;
  if (FROM_R) {
    const double s = sqrt(rr[b]);
    inv = s > 0.0 ? 1.0 / s : 0.0;
    if (rinv && g == 0 && threadIdx.x == 0) rinv[b] = inv;   // 1/||r|| for the tensor-core layer 1
  }
  const double* xb = x + (size_t)b * N + (size_t)i0 * n;
  for (int t = threadIdx.x; t < rows * n; t += blockDim.x) X[t] = (T)(xb[t] * inv);
  __syncthreads();
  // x-direction: thread = (column slice js, mode k2); a twiddle is loaded once for every row of the group,
  // and a slice's chain is n / kDftSlices steps long; the slices' partial sums are added in a fixed order
  {
    constexpr int kDftSlices = 12;                                   // 12 x 20 modes = 240 of the 256 threads
    T2* Tp = reinterpret_cast<T2*>(Tx + DR * kModes);                // [kDftSlices][DR][20]
    const int js = threadIdx.x / kModes, k2 = threadIdx.x - js * kModes;
    if (js < kDftSlices) {
      const int per = (n + kDftSlices - 1) / kDftSlices, j0 = js * per, j1 = min(n, j0 + per);
      T ar[8], ai[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) { ar[r] = 0; ai[r] = 0; }
      for (int j = j0; j < j1; ++j) {
        const T2 f = __ldg(F + j * kModes + k2);
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < rows) {
            const T v = X[r * n + j];
            ar[r] += v * f.x; ai[r] += v * f.y;
          }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < rows) Tp[(js * DR + r) * kModes + k2] = T2{ar[r], ai[r]};
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * kModes; e += blockDim.x) {
      T sr = 0, si = 0;
      for (int q = 0; q < kDftSlices; ++q) {
        const T2 v = Tp[q * DR * kModes + e];
        sr += v.x; si += v.y;
      }
      Tx[e] = T2{sr, si};
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kModes2; e += blockDim.x) {
    const int k1 = e / kModes, k2 = e - k1 * kModes;
    T ar = 0, ai = 0;
    for (int r = 0; r < rows; ++r) {
      const T2 f = __ldg(F + (i0 + r) * kModes + k1);
      const T2 t = Tx[r * kModes + k2];
      ar += f.x * t.x - f.y * t.y;
      ai += f.x * t.y + f.y * t.x;
    }
    part[((size_t)b * ngroups + g) * kModes2 + e] = T2{ar, ai};
  }
}

template <typename T>
__global__ void k_reduce_groups(const typename Cplx<T>::type* __restrict__ part, typename Cplx<T>::type* __restrict__ out,
                                int ngroups) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  const int b = blockIdx.x;
  for (int e = threadIdx.x; e < kModes2; e += blockDim.x) {
    T ar = 0, ai = 0;
    for (int g = 0; g < ngroups; ++g) {
      const T2 v = part[((size_t)b * ngroups + g) * kModes2 + e];
      ar += v.x; ai += v.y;
    }
    out[(size_t)b * kModes2 + e] = T2{ar, ai};
  }
}

static size_t dft_smem(int n, size_t tsz) {   // X [DR][n], Tx [DR][20] complex, slice partials [12][DR][20] complex
  return ((size_t)((dft_rows(n) * n + 3) & ~3)) * tsz + (size_t)13 * dft_rows(n) * kModes * 2 * tsz;
}

template <typename T>
cudaError_t launch_khat(const double* k, const T* F, T* part, T* khat, int n, int B, int ngroups, cudaStream_t s) {
  using T2 = typename Cplx<T>::type;
  static bool attr = false;   // assemble runs before any NO call; sized for the largest NO grid (n = 512): the
                              // slice partials exceed 48 KB at n >= 256 in fp64
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute((const void*)k_dft_rows<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)dft_smem(512, sizeof(T)));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_dft_rows<T, false><<<dim3(ngroups, B), 256, dft_smem(n, sizeof(T)), s>>>(
      k, nullptr, reinterpret_cast<const T2*>(F), reinterpret_cast<T2*>(part), n, ngroups, nullptr, nullptr);
  k_reduce_groups<T><<<B, 256, 0, s>>>(reinterpret_cast<const T2*>(part), reinterpret_cast<T2*>(khat), ngroups);
  launch_counter() += 2;
  return cudaGetLastError();
}
template cudaError_t launch_khat<float>(const double*, const float*, float*, float*, int, int, int, cudaStream_t);
template cudaError_t launch_khat<double>(const double*, const double*, double*, double*, int, int, int, cudaStream_t);

// ------------------------------------------------------------------ layer-1 mixing with the lift folded in
// Output channels per CTA of k_lift_mix: every CTA of a system repeats the sum over the input DFT's row
// groups, so the channel chunk grows with the batch once the grid exceeds about eight CTAs per SM.
static int lift_channels(int w, int B) {
  const int ch = (w * B + 8 * 148 - 1) / (8 * 148);
  return ch < 4 ? 4 : (ch > w ? w : ch);
}
template <typename T>
__global__ void __launch_bounds__(256) k_lift_mix(const typename Cplx<T>::type* __restrict__ rpart, int ngroups,
                                                  const typename Cplx<T>::type* __restrict__ khat,
                                                  const typename Cplx<T>::type* __restrict__ A0,
                                                  const typename Cplx<T>::type* __restrict__ A1,
                                                  const typename Cplx<T>::type* __restrict__ A2,
                                                  typename Cplx<T>::type* __restrict__ ghat, int w, T n2, T inv_n2,
                                                  const int* __restrict__ status, int mode_major, int k0, int och) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  const int b = blockIdx.x, ochunk = blockIdx.y;   // och output channels per CTA
  if (status && status[b] != SYS_RUNNING) return;
  __shared__ T2 Rh[kModes2];
  for (int e = threadIdx.x; e < kModes2; e += blockDim.x) {
    T ar = 0, ai = 0;
    int g = 0;
    for (; g + 8 <= ngroups; g += 8) {          // 8 independent loads in flight
      T2 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = rpart[((size_t)b * ngroups + g + q) * kModes2 + e];
#pragma unroll
      for (int q = 0; q < 8; ++q) { ar += v[q].x; ai += v[q].y; }
    }
    for (; g < ngroups; ++g) {
      const T2 v = rpart[((size_t)b * ngroups + g) * kModes2 + e];
      ar += v.x; ai += v.y;
    }
    Rh[e] = T2{ar, ai};
  }
  __syncthreads();
  // k0: the mode of a constant field (the lift's bias bE transforms to n^2 at k0 only)
  // element e -> (o, kappa): kappa fastest for the [B][w][400] layout (FFMA path), o fastest for the
  // mode-major [400][B][w] layout of the tensor-core path, so the stores stay contiguous
  const int olo = ochunk * och, ohi = min(w, olo + och), no_ = ohi - olo, cnt = no_ * kModes2;
  auto decode = [&](int e, int& o, int& kk) {
    if (mode_major) { kk = e / no_; o = olo + (e - kk * no_); }
    else { o = olo + e / kModes2; kk = e % kModes2; }
  };
  for (int e0 = threadIdx.x; e0 < cnt; e0 += 4 * blockDim.x) {
    T2 a0[4], a1[4], kh[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = e0 + q * blockDim.x;
      int o, kk;
      decode(e < cnt ? e : 0, o, kk);
      const bool ok = e < cnt;
      a0[q] = ok ? A0[(size_t)kk * w + o] : T2{T(0), T(0)};
      a1[q] = ok ? A1[(size_t)kk * w + o] : T2{T(0), T(0)};
      kh[q] = ok ? khat[(size_t)b * kModes2 + kk] : T2{T(0), T(0)};
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = e0 + q * blockDim.x;
      if (e >= cnt) break;
      int o, kk;
      decode(e, o, kk);
      const T2 rh = Rh[kk];
      T gr = a0[q].x * rh.x - a0[q].y * rh.y + a1[q].x * kh[q].x - a1[q].y * kh[q].y;
      T gi = a0[q].x * rh.y + a0[q].y * rh.x + a1[q].x * kh[q].y + a1[q].y * kh[q].x;
      if (kk == k0) { gr += n2 * A2[o].x; gi += n2 * A2[o].y; }
      const size_t at = mode_major ? ((size_t)kk * gridDim.x + b) * ((w + 3) & ~3) + o : ((size_t)b * w + o) * kModes2 + kk;
      ghat[at] = T2{gr * inv_n2, gi * inv_n2};
    }
  }
}

// ------------------------------------------------------------------ mode-diagonal mixing
// grid (400, ceil(B / kMixBatch)).  chat [nparts][400][B][cin] (partial analyses summed here in a
// fixed order), R [400][cin][cout], ghat [B][cout][400].  Each thread owns 2 systems x 2 output
// channels, so every shared-memory read feeds two complex multiply-adds.
template <typename T>
__global__ void __launch_bounds__(256) k_mix(const typename Cplx<T>::type* __restrict__ chat,
                                             const typename Cplx<T>::type* __restrict__ R,
                                             typename Cplx<T>::type* __restrict__ ghat, int B, int cin, int cout,
                                             T inv_n2, const int* __restrict__ status, int nparts) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  extern __shared__ __align__(16) unsigned char smraw[];
  T2* Rs = reinterpret_cast<T2*>(smraw);             // [cin][cout]
  T2* Cs = Rs + (size_t)cin * cout;                  // [kMixBatch][cin]
  const int kk = blockIdx.x, b0 = blockIdx.y * kMixBatch, nb = min(kMixBatch, B - b0);
  const T2* Rk = R + (size_t)kk * cin * cout;
  for (int t = threadIdx.x; t < cin * cout; t += blockDim.x) Rs[t] = Rk[t];
  for (int t = threadIdx.x; t < nb * cin; t += blockDim.x) {
    T ar = 0, ai = 0;
    for (int p = 0; p < nparts; ++p) {
      const T2 v = chat[(((size_t)p * kModes2 + kk) * B + b0) * cin + t];
      ar += v.x; ai += v.y;
    }
    Cs[t] = T2{ar, ai};
  }
  __syncthreads();
  const int ob = (cout + 1) / 2, bbn = (nb + 1) / 2;
  for (int e = threadIdx.x; e < bbn * ob; e += blockDim.x) {
    const int o = (e % ob) * 2, bb = (e / ob) * 2;
    const bool o1 = o + 1 < cout, b1 = bb + 1 < nb;
    T a00r = 0, a00i = 0, a01r = 0, a01i = 0, a10r = 0, a10i = 0, a11r = 0, a11i = 0;
    for (int c = 0; c < cin; ++c) {
      const T2 r0 = Rs[c * cout + o], r1 = o1 ? Rs[c * cout + o + 1] : T2{T(0), T(0)};
      const T2 c0 = Cs[bb * cin + c], c1 = b1 ? Cs[(bb + 1) * cin + c] : T2{T(0), T(0)};
      a00r += r0.x * c0.x - r0.y * c0.y;  a00i += r0.x * c0.y + r0.y * c0.x;
      a01r += r1.x * c0.x - r1.y * c0.y;  a01i += r1.x * c0.y + r1.y * c0.x;
      a10r += r0.x * c1.x - r0.y * c1.y;  a10i += r0.x * c1.y + r0.y * c1.x;
      a11r += r1.x * c1.x - r1.y * c1.y;  a11i += r1.x * c1.y + r1.y * c1.x;
    }
    const int g0 = b0 + bb;
    const bool run0 = !status || status[g0] == SYS_RUNNING;
    const bool run1 = b1 && (!status || status[g0 + 1] == SYS_RUNNING);
    if (run0) {
      ghat[((size_t)g0 * cout + o) * kModes2 + kk] = T2{a00r * inv_n2, a00i * inv_n2};
      if (o1) ghat[((size_t)g0 * cout + o + 1) * kModes2 + kk] = T2{a01r * inv_n2, a01i * inv_n2};
    }
    if (run1) {
      ghat[((size_t)(g0 + 1) * cout + o) * kModes2 + kk] = T2{a10r * inv_n2, a10i * inv_n2};
      if (o1) ghat[((size_t)(g0 + 1) * cout + o + 1) * kModes2 + kk] = T2{a11r * inv_n2, a11i * inv_n2};
    }
  }
}

// ------------------------------------------------------------------ operator layer (layers 1-3)
template <typename T>
struct LayerArgs {
  int n, N, w, cin, B, rows, nbuf, use_gelu, fsm;
  const double* r; const double* rr; const double* k;   // FIRST layer inputs
  const T* vin;                                          // [B][cin][N] (layers 2, 3)
  const T* W;                                            // [w][cin]
  const T* bias;                                         // [w]
  const typename Cplx<T>::type* ghat;                    // [B][w][400], scaled by n^-2
  const typename Cplx<T>::type* F;                       // [n][20]
  T* vout;                                               // [B][w][N]
  typename Cplx<T>::type* chat;                          // [400][B][w]
  const int* status;
};


template <typename T, int GO>
struct LayerSmem {
  // element offsets (in T) of each region; complex regions are 2 T per entry
  size_t Wsm, bsm, gh, Fs, Vin, Vout, Gs, Tx, total;
  int nbuf;
  __host__ __device__ LayerSmem(int n, int cin, int rows, int nbuf_, int fs) {
    const int CH = rows * n;
    nbuf = nbuf_;                               // 2: double-buffered input rows (cp.async)
    size_t o = 0;
    auto al = [](size_t x) { return (x + 3) & ~size_t(3); };
    Wsm = o; o = al(o + (size_t)cin * GO);
    bsm = o; o = al(o + GO);
    gh = o; o = al(o + (size_t)2 * GO * kGhStride);
    Fs = o; o = al(o + (fs ? (size_t)2 * n * kModes : 0));
    Vin = o; o = al(o + (size_t)nbuf * cin * CH);
    Vout = o; o = al(o + (size_t)GO * CH);
    Gs = o; o = al(o + (size_t)2 * rows * kModes * GO);
    Tx = o; o = al(o + (size_t)2 * GO * (rows * kModes + 1));
    total = o;
  }
};

template <typename T> constexpr int layer_go() { return sizeof(T) == 4 ? 8 : 4; }

// Rows per chunk (up to 256 pixels) and input buffering: halve the rows, then drop the second
// buffer, until the CTA's shared memory fits the opt-in limit.
// The twiddle table is staged in shared memory whenever it fits (dropped last): for n >= 256 its
// global reads sat on the dependent x-analysis / y-synthesis loops.
template <typename T>
void layer_config(int n, int cin, bool first, size_t limit, int* rows_out, int* nbuf_out, int* fs_out) {
  int nbuf = first ? 1 : 2, fs = 1;
  int rows = n >= 256 ? 1 : 256 / n;
  auto bytes = [&]() { return LayerSmem<T, layer_go<T>()>(n, cin, rows, nbuf, fs).total * sizeof(T); };
  while (rows > 1 && bytes() > limit) rows = (rows + 1) / 2;
  if (bytes() > limit) nbuf = 1;
  if (bytes() > limit) fs = 0;
  *rows_out = rows;
  *nbuf_out = nbuf;
  *fs_out = fs;
}

__device__ __forceinline__ void cp_async_bytes16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(sdst)), "l"(gsrc),
               "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T, bool FIRST, int GO>
__global__ void __launch_bounds__(256) k_no_layer(const LayerArgs<T> a) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  constexpr int NACC = (GO * kModes2 + 255) / 256;
  constexpr int VEC = 16 / sizeof(T);
  const int b = blockIdx.y, og = blockIdx.x * GO;
  if (a.status && a.status[b] != SYS_RUNNING) return;
  const int n = a.n, N = a.N, cin = a.cin, w = a.w, RC = a.rows;
  // row split (gridDim.z parts): this CTA's rows [ia, ib); its y-analysis is partial z of chat,
  // summed by k_mix in a fixed order
  const int nrc = (n + RC - 1) / RC, z = blockIdx.z, nz = gridDim.z;
  const int ia = (int)(((long long)nrc * z / nz)) * RC, ib = min(n, (int)(((long long)nrc * (z + 1) / nz)) * RC);
  const int go = min(GO, w - og);
  const int nbuf = a.nbuf;
  const LayerSmem<T, GO> L(n, cin, RC, nbuf, a.fsm);
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  T* Wsm = sm + L.Wsm;           // [cin][GO]
  T* bsm = sm + L.bsm;           // [GO]
  T2* gh = reinterpret_cast<T2*>(sm + L.gh);      // [GO][kGhStride]
  T* VinB = sm + L.Vin;          // [nbuf][cin][CH]
  T* Vout = sm + L.Vout;         // [GO][CH]
  T2* Gs = reinterpret_cast<T2*>(sm + L.Gs);      // [RC][20][GO]
  T2* Tx = reinterpret_cast<T2*>(sm + L.Tx);      // [GO][RC*20+1]
  const int TXS = RC * kModes + 1;
  const int CH = RC * n;
  const bool fsm = a.fsm != 0;
  T2* Fsm = reinterpret_cast<T2*>(sm + L.Fs);
  const T2* Ft = fsm ? Fsm : a.F;                 // twiddles exp(-2 pi i kappa j / n), [n][20]

  // async staging of the input rows of chunk i0 into buffer `buf` (layers 2, 3)
  auto stage = [&](int i0, int buf) {
    const int rows = min(RC, n - i0), npix = rows * n;
    T* dst = VinB + (size_t)buf * cin * CH;
    const T* src = a.vin + (size_t)b * cin * N + (size_t)i0 * n;
    if (n % VEC == 0) {
      const int nv = npix / VEC;
      for (int t = threadIdx.x; t < cin * nv; t += blockDim.x) {
        const int c = t / nv, q = t - c * nv;
        cp_async_bytes16(dst + (size_t)c * npix + q * VEC, src + (size_t)c * N + q * VEC);
      }
    } else {
      for (int t = threadIdx.x; t < cin * npix; t += blockDim.x) {
        const int c = t / npix, q = t - c * npix;
        cp_async_small<sizeof(T)>(dst + (size_t)c * npix + q, src + (size_t)c * N + q);
      }
    }
    cp_async_commit();
  };
  if (!FIRST && nbuf == 2 && ia < ib) stage(ia, 0);

  for (int t = threadIdx.x; t < cin * GO; t += blockDim.x) {
    const int c = t / GO, o = t - c * GO;
    Wsm[t] = o < go ? a.W[(size_t)(og + o) * cin + c] : T(0);
  }
  for (int o = threadIdx.x; o < GO; o += blockDim.x) bsm[o] = o < go ? a.bias[og + o] : T(0);
  for (int t = threadIdx.x; t < GO * kModes2; t += blockDim.x) {
    const int o = t / kModes2, kk = t - o * kModes2;
    gh[o * kGhStride + kk] = o < go ? a.ghat[((size_t)b * w + og + o) * kModes2 + kk] : T2{T(0), T(0)};
  }
  if (fsm)
    for (int t = threadIdx.x; t < n * kModes; t += blockDim.x) Fsm[t] = a.F[t];
  double inv_s = 1.0;
  if (FIRST) {
    const double s = sqrt(a.rr[b]);
    inv_s = s > 0.0 ? 1.0 / s : 0.0;
  }
  T accr[NACC], acci[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) { accr[q] = 0; acci[q] = 0; }
  __syncthreads();

  int it = 0;
  for (int i0 = ia; i0 < ib; i0 += RC, ++it) {
    const int rows = min(RC, n - i0), npix = rows * n;
    const size_t base = (size_t)i0 * n;
    T* Vin = VinB + (size_t)((FIRST || nbuf == 1) ? 0 : (it & 1)) * cin * CH;
    // 1. input rows of every input channel (layer 1: r/||r|| and k converted on the fly)
    if (FIRST) {
      const double* rb = a.r + (size_t)b * N + base;
      const double* kb = a.k + (size_t)b * N + base;
      for (int t = threadIdx.x; t < npix; t += blockDim.x) {
        Vin[t] = (T)(rb[t] * inv_s);
        Vin[npix + t] = (T)kb[t];
      }
    } else if (nbuf == 2) {
      if (i0 + RC < ib) { stage(i0 + RC, (it + 1) & 1); cp_async_wait<1>(); }
      else cp_async_wait<0>();
    } else {
      stage(i0, 0);
      cp_async_wait<0>();
    }
    // 2. y-synthesis of this layer's spectral term for the rows: Gs[r][k2][o]
    for (int e = threadIdx.x; e < rows * kModes * GO; e += blockDim.x) {
      const int o = e % GO, rk = e / GO, r = rk / kModes, k2 = rk - r * kModes;
      T gr = 0, gi = 0;
      const T2* F1 = Ft + (size_t)(i0 + r) * kModes;
#pragma unroll 4
      for (int k1 = 0; k1 < kModes; ++k1) {
        const T2 g = gh[o * kGhStride + k1 * kModes + k2];
        const T2 f = F1[k1];                         // conj(f) = exp(+2 pi i kappa1 i / n)
        gr += g.x * f.x + g.y * f.y;
        gi += g.y * f.x - g.x * f.y;
      }
      Gs[(r * kModes + k2) * GO + o] = T2{gr, gi};
    }
    __syncthreads();
    // 3. bypass + x-synthesis + bias + GELU for every pixel of the rows
    for (int p = threadIdx.x; p < npix; p += blockDim.x) {
      const int r = p / n, j = p - r * n;
      T acc[GO];
#pragma unroll
      for (int o = 0; o < GO; ++o) acc[o] = bsm[o];
#pragma unroll 4
      for (int c = 0; c < cin; ++c) {
        const T x = Vin[c * npix + p];
#pragma unroll
        for (int o = 0; o < GO; ++o) acc[o] += Wsm[c * GO + o] * x;
      }
      const T2* Fj = Ft + (size_t)j * kModes;
      const T2* Gr = Gs + (size_t)r * kModes * GO;
#pragma unroll 4
      for (int k2 = 0; k2 < kModes; ++k2) {
        const T2 f = Fj[k2];                         // Re(G exp(+i th)) = G.x f.x + G.y f.y
#pragma unroll
        for (int o = 0; o < GO; ++o) {
          const T2 g = Gr[k2 * GO + o];
          acc[o] += g.x * f.x + g.y * f.y;
        }
      }
#pragma unroll
      for (int o = 0; o < GO; ++o) {
        const T v = a.use_gelu ? gelu_t(acc[o]) : acc[o];
        Vout[o * npix + p] = v;
        if (o < go) a.vout[((size_t)b * w + og + o) * N + base + p] = v;
      }
    }
    __syncthreads();
    // 4. x-analysis of the new activations: Tx[o][r][k2]
    for (int e = threadIdx.x; e < GO * rows * kModes; e += blockDim.x) {
      const int k2 = e % kModes, orr = e / kModes, r = orr % rows, o = orr / rows;
      const T* vrow = Vout + (size_t)o * npix + (size_t)r * n;
      T tr = 0, ti = 0;
#pragma unroll 4
      for (int j = 0; j < n; ++j) {
        const T2 f = Ft[(size_t)j * kModes + k2];
        const T v = vrow[j];
        tr += v * f.x; ti += v * f.y;
      }
      Tx[o * TXS + r * kModes + k2] = T2{tr, ti};
    }
    __syncthreads();
    // 5. y-analysis accumulated over the rows in registers: acc(kappa, o)
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
      const int e = threadIdx.x + q * 256;
      if (e < GO * kModes2) {
        const int o = e % GO, kk = e / GO, k1 = kk / kModes, k2 = kk - k1 * kModes;
        for (int r = 0; r < rows; ++r) {
          const T2 f = Ft[(size_t)(i0 + r) * kModes + k1];
          const T2 t = Tx[o * TXS + r * kModes + k2];
          accr[q] += f.x * t.x - f.y * t.y;
          acci[q] += f.x * t.y + f.y * t.x;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NACC; ++q) {
    const int e = threadIdx.x + q * 256;
    if (e < GO * kModes2) {
      const int o = e % GO, kk = e / GO;
      if (o < go) a.chat[(((size_t)z * kModes2 + kk) * a.B + b) * w + og + o] = T2{accr[q], acci[q]};
    }
  }
}

// ------------------------------------------------------------------ layer 4 + projection + FCG window dots
template <typename T>
struct OutArgs {
  int n, N, w, use_dots;
  const T* vin;                                   // [B][w][N]
  const float* p3;                                // tensor-core path: layer-3 projection bypass term [B][N]
  const T* dw;                                    // [w]
  const T* cst;                                   // [1]
  const typename Cplx<T>::type* gh4;              // [B][400] scaled by n^-2 (tensor-core path: [400][B])
  int B;
  const typename Cplx<T>::type* F;
  const double* rr;
  double* wout;                                   // [B][N]
  const int* status;
};


// V: storage type of the FCG vectors (w written, ring read; R21), fixed per launch.
template <typename T, typename V>
__global__ void __launch_bounds__(kThreads) k_no_out(const OutArgs<T> a, const FcgDev d) {
  pdl_wait();
  pdl_trigger();
  using T2 = typename Cplx<T>::type;
  const int b = blockIdx.y, blk = blockIdx.x;
  if (a.status && a.status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  T2* gh = reinterpret_cast<T2*>(smraw);          // [400]
  T2* Gs = gh + kModes2;                          // [nr][20]
  const int n = a.n, N = a.N, w = a.w;
  const int e0 = blk * kTile;
  const int rlo = e0 / n, rhi = min(n - 1, (e0 + kTile - 1) / n), nr = rhi - rlo + 1;
  T* dws = reinterpret_cast<T*>(Gs + (size_t)nr * kModes);   // [w]
  for (int t = threadIdx.x; t < kModes2; t += blockDim.x) gh[t] = a.gh4[(size_t)b * kModes2 + t];
  for (int t = threadIdx.x; t < w; t += blockDim.x) dws[t] = a.dw[t];
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kModes; e += blockDim.x) {
    const int r = e / kModes, k2 = e - r * kModes;
    T gr = 0, gi = 0;
    for (int k1 = 0; k1 < kModes; ++k1) {
      const T2 g = gh[k1 * kModes + k2];
      const T2 f = __ldg(a.F + (size_t)(rlo + r) * kModes + k1);
      gr += g.x * f.x + g.y * f.y;
      gi += g.y * f.x - g.x * f.y;
    }
    Gs[e] = T2{gr, gi};
  }
  __syncthreads();
  const double s = sqrt(a.rr[b]);
  const T cst = a.cst[0];
  T acc[kPerThread];
  const T* vb = a.vin + (size_t)b * w * N;
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) acc[q] = cst;
  // bypass: 8 channels x 4 pixels of independent loads in flight
  for (int c0 = 0; c0 < w; c0 += 8) {
    T x[8][kPerThread];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
#pragma unroll
      for (int q = 0; q < kPerThread; ++q) {
        const int e = e0 + q * kThreads + threadIdx.x;
        x[cc][q] = (c0 + cc < w && e < N) ? __ldg(vb + (size_t)(c0 + cc) * N + e) : T(0);
      }
#pragma unroll
    for (int cc = 0; cc < 8; ++cc)
#pragma unroll
      for (int q = 0; q < kPerThread; ++q) acc[q] += (c0 + cc < w ? dws[c0 + cc] : T(0)) * x[cc][q];
  }
  double wv[kPerThread];
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = e0 + q * kThreads + threadIdx.x;
    wv[q] = 0.0;
    if (e < N) {
      const int i = e / n, j = e - i * n;
      T z = acc[q];
      const T2* Gr = Gs + (size_t)(i - rlo) * kModes;
#pragma unroll 4
      for (int k2 = 0; k2 < kModes; ++k2) {
        const T2 f = __ldg(a.F + (size_t)j * kModes + k2);
        z += Gr[k2].x * f.x + Gr[k2].y * f.y;
      }
      wv[q] = rnd<V>(s * (double)z);   // w as stored (R21): the window dots see the stored value
      reinterpret_cast<V*>(a.wout)[(size_t)b * N + e] = (V)wv[q];
    }
  }
  if (a.use_dots) {
    const int i = *d.iter;
    const int mi = m_schedule(i, d.m, d.schedule);
    if (mi > 0) window_dots_beta<kPerThread, V>(d, b, blk, i, mi, wv);
  }
}

// Tensor-core path variant: the layer-4 bypass sum_o (D W4)[o] v3[o] arrives as one fp32 field
// reduced by layer 3's epilogue; this kernel adds cst + the 1-channel synthesis, scales by ||r||
// and computes the FCG window dots.
template <typename V>
__global__ void __launch_bounds__(kThreads, 2) k_no_out_blob(const OutArgs<float> a, const FcgDev d) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y, blk = blockIdx.x;
  if (a.status && a.status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int n = a.n, N = a.N;
  const int e0 = blk * kTile;
  const int rlo = e0 / n, rhi = min(n - 1, (e0 + kTile - 1) / n), nr = rhi - rlo + 1;
  const int nr_max = kTile / n + 2;
  float2* gh = reinterpret_cast<float2*>(smraw);              // [400] g4 of this system
  float2* Gs = gh + kModes2;                                   // [nr_max][20] y-synthesised rows
  float2* Fs = Gs + (size_t)nr_max * kModes;                   // [20][n] twiddles, transposed
  float* outs = reinterpret_cast<float*>(Fs + (size_t)kModes * n);
  // window vectors first: their loads are in flight during the synthesis below
  const int it = a.use_dots ? *d.iter : 0;
  const int mi = a.use_dots ? m_schedule(it, d.m, d.schedule) : 0;
  double rv[kWinPre][kPerThread];
  if (mi > 0) window_prefetch<V>(d, b, blk, it, mi, rv);
  for (int t = threadIdx.x; t < kModes2; t += blockDim.x) gh[t] = a.gh4[(size_t)t * a.B + b];   // mode-major
  for (int t = threadIdx.x; t < kModes * n; t += blockDim.x) {   // transposed: consecutive threads, consecutive j
    const int k = t / n, j = t - k * n;
    Fs[t] = __ldg(a.F + (size_t)j * kModes + k);
  }
  // the bypass term sum_o dw[o] v3[o] was reduced by layer 3 (k_tc_layer, fused projection)
  for (int t = threadIdx.x; t < kTile; t += blockDim.x) outs[t] = (e0 + t < N) ? a.p3[(size_t)b * N + e0 + t] : 0.f;
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kModes; e += blockDim.x) {
    const int r = e / kModes, k2 = e - r * kModes;
    float gr = 0, gi = 0;
#pragma unroll 4
    for (int k1 = 0; k1 < kModes; ++k1) {
      const float2 gg = gh[k1 * kModes + k2];
      const float2 f = Fs[k1 * n + rlo + r];
      gr += gg.x * f.x + gg.y * f.y;
      gi += gg.y * f.x - gg.x * f.y;
    }
    Gs[e] = make_float2(gr, gi);
  }
  __syncthreads();
  const double s = sqrt(a.rr[b]);
  const float cst = a.cst[0];
  double wv[kPerThread];
#pragma unroll
  for (int q = 0; q < kPerThread; ++q) {
    const int e = e0 + q * kThreads + threadIdx.x;
    wv[q] = 0.0;
    if (e < N) {
      const int i = e / n, j = e - i * n;
      float z = cst + outs[e - e0];
      const float2* Gr = Gs + (size_t)(i - rlo) * kModes;
#pragma unroll 4
      for (int k2 = 0; k2 < kModes; ++k2) {
        const float2 f = Fs[k2 * n + j];
        z += Gr[k2].x * f.x + Gr[k2].y * f.y;
      }
      wv[q] = rnd<V>(s * (double)z);   // w as stored (R21): the window dots see the stored value
      reinterpret_cast<V*>(a.wout)[(size_t)b * N + e] = (V)wv[q];
    }
  }
  if (mi > 0) window_dots_beta<true, kPerThread, V>(d, b, blk, it, mi, wv, rv);
}


// Wide-batch variant (B n^2 >= 2^21, no fused window dots): a CTA owns kOutRows rows of one system.  The
// twiddles F[j][.] of a thread's column stay in registers over its rows, the y-synthesised rows are
// built once per CTA, and a pixel costs 20 shared broadcasts and 40 FMAs (the tile variant above
// reloads the whole twiddle table and re-derives its rows per 1,024 pixels).
constexpr int kOutRows = 16;
template <typename V>
__global__ void __launch_bounds__(256) k_no_out_wide(const OutArgs<float> a) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y, n = a.n, N = a.N;
  if (a.status && a.status[b] != SYS_RUNNING) return;
  __shared__ float2 gh[kModes2];                 // g4 of this system
  __shared__ __align__(16) float2 Gs[kOutRows][kModes];   // y-synthesised rows
  const int rlo = blockIdx.x * kOutRows, nr = min(kOutRows, n - rlo);
  for (int t = threadIdx.x; t < kModes2; t += blockDim.x) gh[t] = a.gh4[(size_t)t * a.B + b];   // mode-major
  __syncthreads();
  for (int e = threadIdx.x; e < nr * kModes; e += blockDim.x) {
    const int r = e / kModes, k2 = e - r * kModes;
    const float2* Fi = a.F + (size_t)(rlo + r) * kModes;
    float gr = 0, gi = 0;
#pragma unroll 4
    for (int k1 = 0; k1 < kModes; ++k1) {
      const float2 gg = gh[k1 * kModes + k2];
      const float2 f = __ldg(Fi + k1);
      gr += gg.x * f.x + gg.y * f.y;
      gi += gg.y * f.x - gg.x * f.y;
    }
    Gs[r][k2] = make_float2(gr, gi);
  }
  __syncthreads();
  const double s = sqrt(a.rr[b]);
  const float cst = a.cst[0];
  const int cols = n < 256 ? n : 256, rsub = 256 / cols;   // n = 64: 4 row sets, 128: 2, >= 256: 1
  const int jl = threadIdx.x % cols, r0 = threadIdx.x / cols;
  for (int jb = 0; jb < n; jb += cols) {
    const int j = jb + jl;
    float2 fj[kModes];
    const float4* Fp = reinterpret_cast<const float4*>(a.F + (size_t)j * kModes);   // 160 bytes, 16-byte aligned
#pragma unroll
    for (int q = 0; q < kModes / 2; ++q) {
      const float4 v = __ldg(Fp + q);
      fj[2 * q] = make_float2(v.x, v.y);
      fj[2 * q + 1] = make_float2(v.z, v.w);
    }
    for (int r = r0; r < nr; r += rsub) {
      const size_t e = (size_t)b * N + (size_t)(rlo + r) * n + j;
      float z = cst + __ldg(a.p3 + e);
      const float4* Gr = reinterpret_cast<const float4*>(&Gs[r][0]);
#pragma unroll
      for (int q = 0; q < kModes / 2; ++q) {
        const float4 g2 = Gr[q];
        z += g2.x * fj[2 * q].x + g2.y * fj[2 * q].y;
        z += g2.z * fj[2 * q + 1].x + g2.w * fj[2 * q + 1].y;
      }
      reinterpret_cast<V*>(a.wout)[e] = (V)(s * (double)z);   // w as stored (R21)
    }
  }
}

// ------------------------------------------------------------------ launcher
// Largest dynamic shared memory a CTA may request on this device (opt-in limit).
static int optin_smem() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = kMaxDynSmem;
  }
  return v;
}

static cudaError_t set_smem(const void* fn) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin_smem() - (int)fa.sharedSizeBytes);
}

// Raise the dynamic shared-memory limit of every NO kernel once (never during graph capture).
template <typename T>
cudaError_t prepare_no_kernels() {
  static bool done = false;
  if (done) return cudaSuccess;
  constexpr int GO = layer_go<T>();
  cudaError_t e;
  if ((e = set_smem((const void*)k_no_layer<T, true, GO>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_no_layer<T, false, GO>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_mix<T>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_no_out<T, double>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_no_out<T, float>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_no_out_blob<double>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_no_out_blob<float>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_dft_rows<T, true>)) != cudaSuccess) return e;
  if ((e = set_smem((const void*)k_dft_rows<T, false>)) != cudaSuccess) return e;
  done = true;
  return cudaSuccess;
}
template cudaError_t prepare_no_kernels<float>();
template cudaError_t prepare_no_kernels<double>();

template <typename T>
size_t no_max_smem(int n, int w) {
  constexpr int GO = layer_go<T>();
  const size_t lim = (size_t)optin_smem() - 2048;
  int rows1, nbuf1, fs1;
  layer_config<T>(n, w, false, lim, &rows1, &nbuf1, &fs1);
  size_t m = LayerSmem<T, GO>(n, w, rows1, nbuf1, fs1).total * sizeof(T);
  const size_t msmem = ((size_t)w * w + (size_t)kMixBatch * w) * 2 * sizeof(T);
  return m > msmem ? m : msmem;
}
template size_t no_max_smem<float>(int, int);
template size_t no_max_smem<double>(int, int);

// Row split of the FFMA layer kernel: parts per system such that (CTAs x parts) fills the SMs
// once at the kernel's occupancy, at most kRowSplitMax and one row chunk per part.
static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static int layer_row_split(const void* fn, size_t smem, int ctas, int row_chunks) {
  const int sms = sm_count();
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess || per_sm < 1) {
    (void)cudaGetLastError();
    per_sm = 1;
  }
  int nz = (sms * per_sm) / (ctas > 0 ? ctas : 1);
  nz = nz < 1 ? 1 : (nz > kRowSplitMax ? kRowSplitMax : nz);
  return nz < row_chunks ? nz : row_chunks;
}

// The tensor-core path keeps the mixed spectra mode-major ([400][B][cout]); the FFMA path [B][cout][400].
template <typename T>
static bool tc_layout_modes(const NoDev<T>& no) {
  if constexpr (sizeof(T) == sizeof(float)) return no.tc != 0;
  return false;
}

template <typename T>
cudaError_t launch_no_forward(const NoDev<T>& no, const double* r, const double* rr, double* wout,
                              const FcgDev* fcg, const int* status, cudaStream_t s, int* nlaunch, ProfHook* prof) {
  auto pb = [&](int c) { if (prof) prof->begin(c, s); };
  auto pe = [&](int c) { if (prof) prof->end(c, s); };
  using T2 = typename Cplx<T>::type;
  constexpr int GO = layer_go<T>();
  const int n = no.n, B = no.B, w = no.w, N = n * n;
  const T n2 = (T)((double)n * n), inv_n2 = (T)(1.0 / ((double)n * n));
  const T* pk = no.pk;
  const T2* F = reinterpret_cast<const T2*>(no.F);
  T2* ghat = reinterpret_cast<T2*>(no.ghat);
  T2* chat = reinterpret_cast<T2*>(no.chat);
  int launches = 0;

  // 1. DFT_M of r/||r|| (row-group partials)
  pb(PROF_NO_INPUT);
  launch_k(k_dft_rows<T, true>, dim3(no.ngroups, B), dim3(256), dft_smem(n, sizeof(T)), s, r, rr, F,
           reinterpret_cast<T2*>(no.rpart), n, no.ngroups, status, no.rinv);
  ++launches;
  // 2. layer-1 mixing with the lift folded in
  const int och = lift_channels(w, B);
  launch_k(k_lift_mix<T>, dim3(B, (w + och - 1) / och), dim3(256), 0, s, reinterpret_cast<const T2*>(no.rpart), no.ngroups,
           reinterpret_cast<const T2*>(no.khat), reinterpret_cast<const T2*>(pk + no.L.A0),
           reinterpret_cast<const T2*>(pk + no.L.A1), reinterpret_cast<const T2*>(pk + no.L.A2), ghat, w, n2, inv_n2,
           status, (int)tc_layout_modes(no), no.k0, och);
  pe(PROF_NO_INPUT);
  ++launches;
  // 3. layers 1..3, each followed by the mixing of the next layer
  const size_t lim = (size_t)optin_smem() - 2048;
  const dim3 lgrid((w + GO - 1) / GO, B);
  T* vbuf[2] = {no.v0, no.v1};
  bool tc_path = false;
  if constexpr (sizeof(T) == sizeof(float)) tc_path = no.tc != 0;
  if (tc_path) {
    pb(PROF_NO_YDIR);
    launch_px_ysyn(reinterpret_cast<const float*>(ghat), no.cst, no.Gb, n, w, B, status, s);
    pe(PROF_NO_YDIR);
    launches += 1;
  }
  unsigned char* vblob[2] = {no.vb0, no.vb1};
  int nparts = 1;
  for (int l = 0; l < 3; ++l) {
    if (tc_path) {
      PxLayerHost h{};
      h.n = n; h.w = w; h.B = B; h.use_gelu = no.use_gelu; h.layer = l;
      h.r = r; h.rr = no.rinv; h.k = no.k;
      h.cst = no.cst;
      h.bias = reinterpret_cast<const float*>(pk + (l == 0 ? no.L.b1 : no.L.b[l - 1]));
      h.w1e = reinterpret_cast<const float*>(pk + no.L.W1E);
      h.vin = l == 0 ? nullptr : vblob[(l - 1) & 1];
      h.vout = l == 2 ? nullptr : vblob[l & 1];
      h.G = no.Gb; h.T = no.Tb; h.status = status;
      if (l == 2) { h.dw = reinterpret_cast<const float*>(pk + no.L.dw); h.p3 = no.p3; }
      pb(PROF_NO_LAYER);
      launch_px_layer(h, s);
      pe(PROF_NO_LAYER);
      pb(PROF_NO_YDIR);
      launch_px_yan(no.Tb, no.cst, reinterpret_cast<float*>(chat), n, w, B, status, s);
      pe(PROF_NO_YDIR);
      launches += 2;
    } else {
      LayerArgs<T> la{};
      int rows, nbuf, fs;
      layer_config<T>(n, l == 0 ? 2 : w, l == 0, lim, &rows, &nbuf, &fs);
      // tiny batches (config 1: one system): shorter row chunks, so that the row split below can
      // spread a system over up to kRowSplitMax CTAs
      while (rows > 1 && (int)(lgrid.x * lgrid.y) * ((n + rows - 1) / rows) < kRowSplitMax * (int)(lgrid.x * lgrid.y) &&
             (int)(lgrid.x * lgrid.y) * kRowSplitMax <= 2 * sm_count())
        rows /= 2;
      la.n = n; la.N = N; la.w = w; la.B = B; la.rows = rows; la.nbuf = nbuf; la.use_gelu = no.use_gelu; la.fsm = fs;
      la.r = r; la.rr = rr; la.k = no.k;
      la.ghat = ghat; la.F = F; la.chat = chat; la.status = status;
      la.vout = vbuf[l & 1];
      if (l == 0) {
        la.cin = 2; la.W = pk + no.L.W1E; la.bias = pk + no.L.b1; la.vin = nullptr;
      } else {
        la.cin = w; la.W = pk + no.L.W[l - 1]; la.bias = pk + no.L.b[l - 1]; la.vin = vbuf[(l - 1) & 1];
      }
      const size_t smem = LayerSmem<T, GO>(n, la.cin, rows, nbuf, fs).total * sizeof(T);
      // split the rows of each system over gridDim.z CTAs until the grid fills the SMs once
      // (large n, few systems: config 5 has 6 x 8 CTAs of one per SM otherwise)
      const void* fn = l == 0 ? (const void*)k_no_layer<T, true, GO> : (const void*)k_no_layer<T, false, GO>;
      const int nz = layer_row_split(fn, smem, (int)(lgrid.x * lgrid.y), (n + rows - 1) / rows);
      nparts = nz;
      const dim3 g3(lgrid.x, lgrid.y, nz);
      pb(PROF_NO_LAYER);
      if (l == 0) {
        launch_k(k_no_layer<T, true, GO>, g3, dim3(256), smem, s, la);
      } else {
        launch_k(k_no_layer<T, false, GO>, g3, dim3(256), smem, s, la);
      }
      pe(PROF_NO_LAYER);
      ++launches;
    }
    // mixing for the next layer (layers 2, 3) or layer 4 folded with the projection (cout = 1)
    const int cout = (l < 2) ? w : 1;
    const T2* Rm = reinterpret_cast<const T2*>(pk + (l < 2 ? no.L.R[l] : no.L.Q));
    const size_t msmem = ((size_t)w * cout + (size_t)kMixBatch * w) * sizeof(T2);
    pb(PROF_NO_MIX);
    if (tc_path)
      launch_mix_px(l, reinterpret_cast<const float*>(chat), no.cst, reinterpret_cast<float*>(ghat), n, w, B,
                    (float)inv_n2, status, s);
    else
      launch_k(k_mix<T>, dim3(kModes2, (B + kMixBatch - 1) / kMixBatch), dim3(256), msmem, s,
               (const T2*)chat, Rm, ghat, B, w, cout, inv_n2, status, nparts);
    pe(PROF_NO_MIX);
    ++launches;
    if (tc_path && l < 2) {
      pb(PROF_NO_YDIR);
      launch_px_ysyn(reinterpret_cast<const float*>(ghat), no.cst, no.Gb, n, w, B, status, s);
      pe(PROF_NO_YDIR);
      ++launches;
    }
  }
  // 4. layer 4 + projection (+ window dots when inside FCG)
  OutArgs<T> oa{};
  // wide batches: the window dots (w, s_k) run in the separate wide window kernel (16 elements per
  // thread, w staged in shared memory) after the output kernel; small ones keep them fused in it
  const bool split_dots = fcg != nullptr && ew_wide(n, B);
  oa.n = n; oa.N = N; oa.w = w; oa.use_dots = fcg != nullptr && !split_dots;
  oa.vin = vbuf[0];                       // layer 3 wrote vbuf[2 & 1] = vbuf[0]
  oa.dw = pk + no.L.dw; oa.cst = pk + no.L.cst;
  oa.gh4 = ghat; oa.F = F; oa.rr = rr; oa.wout = wout; oa.status = status; oa.B = B;
  const int nblk = (N + kTile - 1) / kTile;
  const int nr_max = kTile / n + 2;
  const size_t osmem = (size_t)(kModes2 + (size_t)nr_max * kModes) * sizeof(T2) + (size_t)((w + 3) & ~3) * sizeof(T);
  FcgDev dummy{};
  const bool v32 = fcg && fcg->vec32;
  pb(PROF_NO_OUT);
  if constexpr (sizeof(T) == sizeof(float)) {
    if (tc_path) {
      oa.p3 = no.p3;
      const size_t bsmem = (size_t)(kModes2 + (size_t)nr_max * kModes + (size_t)kModes * n) * sizeof(float2) + kTile * sizeof(float);
      if (ew_wide(n, B) && !oa.use_dots) {   // wide batches (also the standalone apply on them: same kernel, same bits)
        const dim3 wg((unsigned)((n + kOutRows - 1) / kOutRows), (unsigned)B);
        if (v32) launch_k(k_no_out_wide<float>, wg, dim3(256), 0, s, oa);
        else launch_k(k_no_out_wide<double>, wg, dim3(256), 0, s, oa);
      } else if (v32) launch_k(k_no_out_blob<float>, dim3(nblk, B), dim3(kThreads), bsmem, s, oa, *fcg);
      else launch_k(k_no_out_blob<double>, dim3(nblk, B), dim3(kThreads), bsmem, s, oa, fcg ? *fcg : dummy);
    } else {
      if (v32) launch_k(k_no_out<T, float>, dim3(nblk, B), dim3(kThreads), osmem, s, oa, *fcg);
      else launch_k(k_no_out<T, double>, dim3(nblk, B), dim3(kThreads), osmem, s, oa, fcg ? *fcg : dummy);
    }
  } else {
    if (v32) launch_k(k_no_out<T, float>, dim3(nblk, B), dim3(kThreads), osmem, s, oa, *fcg);
    else launch_k(k_no_out<T, double>, dim3(nblk, B), dim3(kThreads), osmem, s, oa, fcg ? *fcg : dummy);
  }
  pe(PROF_NO_OUT);
  ++launches;
  if (split_dots) {
    pb(PROF_WINDOW);
    const cudaError_t e = launch_window_dots(*fcg, s);   // adds itself to launch_counter()
    pe(PROF_WINDOW);
    if (e != cudaSuccess) return e;
  }
  launch_counter() += launches;
  if (nlaunch) *nlaunch = launches + (split_dots ? 1 : 0);
  return cudaGetLastError();
}

// Constant operand blobs of the tensor-core path (once per apply / solve, outside graphs).
cudaError_t prepare_no_constants(const NoDev<float>& no, cudaStream_t s) {
  if (!no.tc) return cudaSuccess;
  const float* pk = no.pk;
  return launch_px_prep(no.n, no.w, pk + no.L.W[0], pk + no.L.W[1], pk + no.L.R[0], pk + no.L.R[1], pk + no.L.Q, no.F,
                        no.cst, s);
}

template cudaError_t launch_no_forward<float>(const NoDev<float>&, const double*, const double*, double*,
                                              const FcgDev*, const int*, cudaStream_t, int*, ProfHook*);
template cudaError_t launch_no_forward<double>(const NoDev<double>&, const double*, const double*, double*,
                                               const FcgDev*, const int*, cudaStream_t, int*, ProfHook*);

}  // namespace fcgno

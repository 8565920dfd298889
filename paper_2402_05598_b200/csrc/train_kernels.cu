// train_kernels.cu — training the SNO preconditioner on the GPU.
//
// One minibatch step computes, for the samples (k_b, r_b, e_b) of the minibatch,
//   w_b = ||r_b|| NO([r_b/||r_b||, k_b])                       (forward, readings R7-R11)
//   L   = mean_b ||w_b - e_b||_A / ||e_b||_A                   (Notay loss in error form)
//         (or the L2 form with ||.||_2)
//   dL/dtheta for every weight of the canonical blob            (backward, the chain rule of oracle/train.py)
// and AdamW updates the fp32 weights (reading R26; Table 6).
//
// Layout (fp32, pixel-major: channels contiguous, the bypass is a [B n^2 x w] x [w x w] GEMM):
//   activations  X[b][i][j][c]                       (B, n, n, w)
//   spectra      C[b][part][kappa1][kappa2][c]        part 0 = Re, 1 = Im (kappa in {-10..9})
// The truncated 2-D transforms are separable and run as two batched real GEMMs each against
// constant twiddle matrices (complex products written as 2x2 real blocks):
//   analysis  T[b][i][part][kappa2][c] = sum_j Fj[(part,kappa2)][j] X[b][i][j][c]
//             C[b][(part,kappa1)][(kappa2,c)] = sum_(i,part') Fi[(part,kappa1)][(i,part')] T[b][(i,part')][(kappa2,c)]
//   synthesis U[b][(i,part)][(kappa2,o)] = sum_(part',kappa1) Gi[(i,part)][(part',kappa1)] G[b][(part',kappa1)][(kappa2,o)]
//             x[b][i][j][o] = alpha sum_(part,kappa2) Gj[j][(part,kappa2)] U[b][i][(part,kappa2)][o]
// (Fj/Fi hold exp(-i theta), Gi/Gj the real part of exp(+i theta)).  The adjoints are the same
// transforms (oracle/train.py): dg = analysis(dz)/n^2 and dv = n^2 synthesis(dc).  The mode-diagonal
// complex mixing and its two adjoints run per mode (one CTA per kappa).  Every reduction is a fixed-
// order sum (split-K partials summed in order), so a step is deterministic.
#include <cmath>

#include "internal.h"

namespace fcgno {

// ------------------------------------------------------------------ batched strided SGEMM
// C[z](m, n) = alpha sum_k A[z](m, k) B[z](k, n) + beta C[z](m, n)   (epilogues below)
// with element (m, k) of A at A + b0 sA0 + b1 sA1 + m sAm + k sAk (z = b0 nb1 + b1), likewise B and C.
// Any stride may be 0 (a broadcast operand, e.g. a vector of ones).
template <int BM, int BN>
__global__ void __launch_bounds__(256) k_tr_gemm(TrGemm g) {
  constexpr int BK = 16, TM = BM / 16, TN = BN / 16;
  __shared__ float As[BK][BM + 1];
  __shared__ float Bs[BK][BN + 1];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const long long z = blockIdx.z, b0 = z / g.nb1, b1 = z % g.nb1;
  const float* A = g.A + b0 * g.sA0 + b1 * g.sA1;
  const float* B = g.B + b0 * g.sB0 + b1 * g.sB1;
  float* C = g.C + b0 * g.sC0 + b1 * g.sC1;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const bool a_kfast = g.sAk == 1, b_kfast = g.sBk == 1 && g.sBn != 1;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    for (int e = tid; e < BM * BK; e += 256) {
      int mm, kk;
      if (a_kfast) { kk = e % BK; mm = e / BK; } else { mm = e % BM; kk = e / BM; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.M && k < g.K) ? A[m * g.sAm + k * g.sAk] : 0.f;
    }
    for (int e = tid; e < BK * BN; e += 256) {
      int kk, nn;
      if (b_kfast) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      const int nc = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (nc < g.N && k < g.K) ? B[k * g.sBk + nc * g.sBn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int nc = n0 + tx + 16 * j;
      if (nc >= g.N) continue;
      const long long off = m * g.sCm + nc * g.sCn;
      float v = g.alpha * acc[i][j];
      if (g.beta != 0.f) v += g.beta * C[off];
      if (g.epi != TR_EPI_STORE) v += g.bias[nc];
      C[off] = v;
      if (g.epi == TR_EPI_BIAS_GELU) {
        float* aux = g.aux + b0 * g.sC0 + b1 * g.sC1;
        aux[off] = 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
      }
    }
  }
}

cudaError_t launch_tr_gemm(const TrGemm& g, cudaStream_t s) {
  const long long nbatch = (long long)g.nb0 * g.nb1;
  if (nbatch < 1 || nbatch > 65535 || g.M < 1 || g.N < 1 || g.K < 0) return cudaErrorInvalidValue;
  const bool smallM = g.M <= 40, smallN = g.N <= 40;
  if (smallM && smallN)
    k_tr_gemm<32, 32><<<dim3((g.N + 31) / 32, (g.M + 31) / 32, (unsigned)nbatch), 256, 0, s>>>(g);
  else if (smallM)
    k_tr_gemm<32, 64><<<dim3((g.N + 63) / 64, (g.M + 31) / 32, (unsigned)nbatch), 256, 0, s>>>(g);
  else if (smallN)
    k_tr_gemm<64, 32><<<dim3((g.N + 31) / 32, (g.M + 63) / 64, (unsigned)nbatch), 256, 0, s>>>(g);
  else
    k_tr_gemm<64, 64><<<dim3((g.N + 63) / 64, (g.M + 63) / 64, (unsigned)nbatch), 256, 0, s>>>(g);
  ++launch_counter();
  return cudaGetLastError();
}

// Sum of split-K partials part[S][M][N] in split order into out(m, n) = out + m sOm + n sOn.
__global__ void k_tr_reduce(const float* __restrict__ part, int S, int M, int N, float* __restrict__ out,
                            long long sOm, long long sOn) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * N) return;
  float acc = 0.f;
  for (int s = 0; s < S; ++s) acc += part[(size_t)s * M * N + t];
  out[(t / N) * sOm + (t % N) * sOn] = acc;
}
cudaError_t launch_tr_reduce(const float* part, int S, int M, int N, float* out, long long sOm, long long sOn,
                             cudaStream_t s) {
  k_tr_reduce<<<(M * N + 255) / 256, 256, 0, s>>>(part, S, M, N, out, sOm, sOn);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ twiddle matrices
// kappa(k) = k - 10; theta = 2 pi kappa j / n, evaluated as sincospi(2 kappa j / n) in fp64 with
// kappa j reduced mod n (exact integers), then rounded to fp32.
__global__ void k_tr_twiddles(int n, float* Fj, float* Fi, float* Gi, float* Gj, float* one) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) *one = 1.f;   // the broadcast operand of the bias-gradient GEMMs
  if (t >= kModes * n) return;
  const int kk = t / n, j = t % n, kappa = kk - kModes / 2;
  const long long ph = (((long long)kappa * j) % n + n) % n;
  double sn, cs;
  sincospi(2.0 * (double)ph / (double)n, &sn, &cs);
  const float c = (float)cs, s = (float)sn;
  // analysis along j: rows (part, kappa2), exp(-i theta) = cos - i sin
  Fj[(0 * kModes + kk) * n + j] = c;
  Fj[(1 * kModes + kk) * n + j] = -s;
  // analysis along i: [Re; Im] = [[C, S], [-S, C]] [Tr; Ti], columns ordered (i, part')
  Fi[(0 * kModes + kk) * 2 * n + 2 * j + 0] = c;
  Fi[(0 * kModes + kk) * 2 * n + 2 * j + 1] = s;
  Fi[(1 * kModes + kk) * 2 * n + 2 * j + 0] = -s;
  Fi[(1 * kModes + kk) * 2 * n + 2 * j + 1] = c;
  // synthesis along i: rows (i, part): Ur = C Gr - S Gi, Ui = S Gr + C Gi
  Gi[(2 * j + 0) * 2 * kModes + 0 * kModes + kk] = c;
  Gi[(2 * j + 0) * 2 * kModes + 1 * kModes + kk] = -s;
  Gi[(2 * j + 1) * 2 * kModes + 0 * kModes + kk] = s;
  Gi[(2 * j + 1) * 2 * kModes + 1 * kModes + kk] = c;
  // synthesis along j: Re(U e^{+i theta}) = Ur cos - Ui sin
  Gj[j * 2 * kModes + 0 * kModes + kk] = c;
  Gj[j * 2 * kModes + 1 * kModes + kk] = -s;
}
cudaError_t launch_tr_twiddles(int n, float* Fj, float* Fi, float* Gi, float* Gj, float* one, cudaStream_t s) {
  k_tr_twiddles<<<(kModes * n + 127) / 128, 128, 0, s>>>(n, Fj, Fi, Gi, Gj, one);
  ++launch_counter();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ element-wise kernels
// Gather the minibatch: sample perm[b] of the dataset (k of system ksys[sample], or of the sample).
__global__ void k_tr_gather(const double* __restrict__ k, const double* __restrict__ r, const double* __restrict__ e,
                            const int* __restrict__ perm, const int* __restrict__ ksys, int N, double* kg, double* rg,
                            double* eg) {
  const int b = blockIdx.y;
  const int smp = perm ? perm[b] : b;
  const int ks = ksys ? ksys[smp] : smp;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    kg[(size_t)b * N + p] = k[(size_t)ks * N + p];
    rg[(size_t)b * N + p] = r[(size_t)smp * N + p];
    eg[(size_t)b * N + p] = e[(size_t)smp * N + p];
  }
}

// Lift (R10): x0 = [r/||r||, k] rounded to fp32 (R18), v0[c] = E[c][0] x0 + E[c][1] x1 + bE[c].
__global__ void k_tr_lift(const double* __restrict__ rg, const double* __restrict__ kg, const double* __restrict__ rr,
                          const float* __restrict__ E, const float* __restrict__ bE, int N, int w, float* X2,
                          float* v0) {
  const int b = blockIdx.y;
  const double nrm = sqrt(rr[b]);
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    const size_t q = (size_t)b * N + p;
    const float x0 = (float)(rg[q] * inv), x1 = (float)kg[q];
    X2[2 * q] = x0;
    X2[2 * q + 1] = x1;
    float* v = v0 + q * w;
    for (int c = 0; c < w; ++c) v[c] = fmaf(E[2 * c], x0, fmaf(E[2 * c + 1], x1, bE[c]));
  }
}

// Projection (R10) and the loss residual: w = ||r|| (sum_c D[c] v4[c] + bD), d = w - e (fp64).
__global__ void k_tr_proj(const float* __restrict__ v4, const float* __restrict__ D, const float* __restrict__ bD,
                          const double* __restrict__ rr, const double* __restrict__ eg, int N, int w, double* wout,
                          double* d) {
  const int b = blockIdx.y;
  const double nrm = sqrt(rr[b]);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    const size_t q = (size_t)b * N + p;
    const float* v = v4 + q * w;
    float acc = bD[0];
    for (int c = 0; c < w; ++c) acc = fmaf(D[c], v[c], acc);
    const double wv = nrm * (double)acc;
    if (wout) wout[q] = wv;
    d[q] = wv - eg[q];
  }
}

// Per-sample loss and the gradient coefficient: loss_b = sqrt(dd_b / ee_b);
// dL/dw_b = g_b / (Bm sqrt(dd_b) sqrt(ee_b)) with g_b = A d_b (Notay) or d_b (L2); coef folds ||r_b||.
__global__ void k_tr_loss(const double* __restrict__ dd, const double* __restrict__ ee, const double* __restrict__ rr,
                          int B, int Bmean, double* loss, double* coef) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double nd = sqrt(dd[b]), ne = sqrt(ee[b]);
  if (loss) loss[b] = nd / ne;
  coef[b] = sqrt(rr[b]) / ((double)Bmean * nd * ne);
}

// dout = coef_b g (fp32) and dL/dv4[c] = D[c] dout.
__global__ void k_tr_dout(const double* __restrict__ gvec, const double* __restrict__ coef,
                          const float* __restrict__ D, int N, int w, float* dout, float* dv) {
  const int b = blockIdx.y;
  const double cf = coef[b];
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    const size_t q = (size_t)b * N + p;
    const float g = (float)(cf * gvec[q]);
    dout[q] = g;
    float* o = dv + q * w;
    for (int c = 0; c < w; ++c) o[c] = D[c] * g;
  }
}

// dz = dv * GELU'(z) in place, GELU'(z) = Phi(z) + z phi(z).
__global__ void k_tr_gelu_bwd(float* __restrict__ dv, const float* __restrict__ z, size_t count) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count; t += (size_t)gridDim.x * blockDim.x) {
    const float x = z[t];
    const float g = 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * __expf(-0.5f * x * x);
    dv[t] *= g;
  }
}

// ------------------------------------------------------------------ mode-diagonal mixing
// (re, im) pair of the canonical blob: two scalar loads, the pair's offset is odd for odd w.
__device__ __forceinline__ float2 ldf2(const float* p) { return make_float2(p[0], p[1]); }
// Spectra C[b][part][kappa][c] (kappa = kappa1 * 20 + kappa2), weights R[c][o][kappa][re,im] (canonical blob).
// Forward: G[b][kappa][o] = sum_c R[c][o][kappa] C[b][kappa][c].  One CTA per kappa.
__global__ void k_tr_mix_fwd(const float* __restrict__ C, const float* __restrict__ R, int B, int w,
                             float* __restrict__ G) {
  extern __shared__ float2 sm[];
  float2* Rk = sm;            // [c][o]
  float2* Ck = sm + w * w;    // [b][c]
  const int kap = blockIdx.x;
  const size_t spec = (size_t)2 * kModes2 * w;   // floats per system of a spectrum
  for (int t = threadIdx.x; t < w * w; t += blockDim.x)
    Rk[t] = ldf2(R + ((size_t)t * kModes2 + kap) * 2);
  for (int t = threadIdx.x; t < B * w; t += blockDim.x) {
    const int b = t / w, c = t % w;
    const float* cb = C + b * spec + (size_t)kap * w + c;
    Ck[t] = make_float2(cb[0], cb[(size_t)kModes2 * w]);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < B * w; t += blockDim.x) {
    const int b = t / w, o = t % w;
    float re = 0.f, im = 0.f;
    for (int c = 0; c < w; ++c) {
      const float2 r = Rk[c * w + o], x = Ck[b * w + c];
      re = fmaf(r.x, x.x, fmaf(-r.y, x.y, re));
      im = fmaf(r.x, x.y, fmaf(r.y, x.x, im));
    }
    float* gb = G + b * spec + (size_t)kap * w + o;
    gb[0] = re;
    gb[(size_t)kModes2 * w] = im;
  }
}

// Backward: dR[c][o][kappa] = sum_b dG[b][o] conj(C[b][c]) (overwrites the gradient blob's R block)
// and dC[b][c] = sum_o conj(R[c][o]) dG[b][o].
__global__ void k_tr_mix_bwd(const float* __restrict__ C, const float* __restrict__ dG, const float* __restrict__ R,
                             int B, int w, float* __restrict__ dR, float* __restrict__ dC) {
  extern __shared__ float2 sm[];
  float2* Rk = sm;              // [c][o]
  float2* Ck = sm + w * w;      // [b][c]
  float2* Gk = Ck + B * w;      // [b][o]
  const int kap = blockIdx.x;
  const size_t spec = (size_t)2 * kModes2 * w;
  for (int t = threadIdx.x; t < w * w; t += blockDim.x)
    Rk[t] = ldf2(R + ((size_t)t * kModes2 + kap) * 2);
  for (int t = threadIdx.x; t < B * w; t += blockDim.x) {
    const int b = t / w, c = t % w;
    const size_t off = b * spec + (size_t)kap * w + c;
    Ck[t] = make_float2(C[off], C[off + (size_t)kModes2 * w]);
    Gk[t] = make_float2(dG[off], dG[off + (size_t)kModes2 * w]);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
    const int c = t / w, o = t % w;
    float re = 0.f, im = 0.f;
    for (int b = 0; b < B; ++b) {       // dG conj(C)
      const float2 g = Gk[b * w + o], x = Ck[b * w + c];
      re = fmaf(g.x, x.x, fmaf(g.y, x.y, re));
      im = fmaf(g.y, x.x, fmaf(-g.x, x.y, im));
    }
    float* dr = dR + ((size_t)t * kModes2 + kap) * 2;   // the R block's offset may be odd (odd w)
    dr[0] = re;
    dr[1] = im;
  }
  for (int t = threadIdx.x; t < B * w; t += blockDim.x) {
    const int b = t / w, c = t % w;
    float re = 0.f, im = 0.f;
    for (int o = 0; o < w; ++o) {       // conj(R) dG
      const float2 r = Rk[c * w + o], g = Gk[b * w + o];
      re = fmaf(r.x, g.x, fmaf(r.y, g.y, re));
      im = fmaf(r.x, g.y, fmaf(-r.y, g.x, im));
    }
    float* o = dC + b * spec + (size_t)kap * w + c;
    o[0] = re;
    o[(size_t)kModes2 * w] = im;
  }
}

// ------------------------------------------------------------------ AdamW (reading R26)
__global__ void k_tr_adamw(size_t count, float* __restrict__ th, const float* __restrict__ g, float* __restrict__ m,
                           float* __restrict__ v, float b1, float omb1, float b2, float omb2, float eps, float decay,
                           float step_size, float bc2_sqrt) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count; t += (size_t)gridDim.x * blockDim.x) {
    const float gt = g[t];
    float p = th[t] * decay;
    const float mt = b1 * m[t] + omb1 * gt;
    const float vt = b2 * v[t] + omb2 * gt * gt;
    p -= step_size * mt / (sqrtf(vt) / bc2_sqrt + eps);
    m[t] = mt;
    v[t] = vt;
    th[t] = p;
  }
}

// Krylov training pair (Eq. 8-9): r = f - A u_i (given Au), e = e_scale (u* - u_i)
// (e_scale: the unit of the target, R27).  Au may alias r (element-wise, read before write).
__global__ void k_tr_pair(const double* __restrict__ f, const double* Au, const double* __restrict__ ustar,
                          const double* __restrict__ u, size_t count, double e_scale, double* r,
                          double* __restrict__ e) {
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < count; t += (size_t)gridDim.x * blockDim.x) {
    r[t] = __dsub_rn(f[t], Au[t]);
    e[t] = __dmul_rn(e_scale, __dsub_rn(ustar[t], u[t]));
  }
}

// ------------------------------------------------------------------ launchers
namespace {
int ew_grid(size_t count) { return (int)std::min<size_t>((count + 255) / 256, 148 * 16); }
dim3 per_sys(int N, int B) { return dim3((unsigned)std::min(64, (N + 255) / 256), (unsigned)B); }
}  // namespace

cudaError_t launch_tr_gather(const double* k, const double* r, const double* e, const int* perm, const int* ksys, int N,
                             int B, double* kg, double* rg, double* eg, cudaStream_t s) {
  k_tr_gather<<<per_sys(N, B), 256, 0, s>>>(k, r, e, perm, ksys, N, kg, rg, eg);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_lift(const double* rg, const double* kg, const double* rr, const float* E, const float* bE, int N,
                           int B, int w, float* X2, float* v0, cudaStream_t s) {
  k_tr_lift<<<per_sys(N, B), 256, 0, s>>>(rg, kg, rr, E, bE, N, w, X2, v0);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_proj(const float* v4, const float* D, const float* bD, const double* rr, const double* eg, int N,
                           int B, int w, double* wout, double* d, cudaStream_t s) {
  k_tr_proj<<<per_sys(N, B), 256, 0, s>>>(v4, D, bD, rr, eg, N, w, wout, d);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_loss(const double* dd, const double* ee, const double* rr, int B, int Bmean, double* loss,
                           double* coef, cudaStream_t s) {
  k_tr_loss<<<(B + 127) / 128, 128, 0, s>>>(dd, ee, rr, B, Bmean, loss, coef);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_dout(const double* gvec, const double* coef, const float* D, int N, int B, int w, float* dout,
                           float* dv, cudaStream_t s) {
  k_tr_dout<<<per_sys(N, B), 256, 0, s>>>(gvec, coef, D, N, w, dout, dv);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_gelu_bwd(float* dv, const float* z, size_t count, cudaStream_t s) {
  k_tr_gelu_bwd<<<ew_grid(count), 256, 0, s>>>(dv, z, count);
  ++launch_counter();
  return cudaGetLastError();
}
size_t tr_mix_smem(int B, int w, bool bwd) { return sizeof(float2) * ((size_t)w * w + (size_t)(bwd ? 2 : 1) * B * w); }
cudaError_t prepare_tr_kernels() {
  static bool done = false;
  if (done) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_tr_mix_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_tr_mix_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  done = e == cudaSuccess;
  return e;
}
cudaError_t launch_tr_mix_fwd(const float* C, const float* R, int B, int w, float* G, cudaStream_t s) {
  k_tr_mix_fwd<<<kModes2, 256, tr_mix_smem(B, w, false), s>>>(C, R, B, w, G);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_mix_bwd(const float* C, const float* dG, const float* R, int B, int w, float* dR, float* dC,
                              cudaStream_t s) {
  k_tr_mix_bwd<<<kModes2, 256, tr_mix_smem(B, w, true), s>>>(C, dG, R, B, w, dR, dC);
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_adamw(size_t count, float* th, const float* g, float* m, float* v, double lr, double b1, double b2,
                            double eps, double wd, int t, cudaStream_t s) {
  const double bc1 = 1.0 - std::pow(b1, t), bc2 = 1.0 - std::pow(b2, t);
  // 1 - beta in fp64 then rounded (1.f - (float)0.999 is off by 1.3e-5 relative)
  k_tr_adamw<<<ew_grid(count), 256, 0, s>>>(count, th, g, m, v, (float)b1, (float)(1.0 - b1), (float)b2,
                                             (float)(1.0 - b2), (float)eps, (float)(1.0 - lr * wd), (float)(lr / bc1),
                                             (float)std::sqrt(bc2));
  ++launch_counter();
  return cudaGetLastError();
}
cudaError_t launch_tr_pair(const double* f, const double* Au, const double* ustar, const double* u, size_t count,
                           double e_scale, double* r, double* e, cudaStream_t s) {
  k_tr_pair<<<ew_grid(count), 256, 0, s>>>(f, Au, ustar, u, count, e_scale, r, e);
  ++launch_counter();
  return cudaGetLastError();
}

}  // namespace fcgno

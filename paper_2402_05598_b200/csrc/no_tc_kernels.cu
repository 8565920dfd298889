// no_tc_kernels.cu — tensor-core (tcgen05 / TMEM) SNO layers for the fp32 NO path.
//
// One layer (R7-R11) is
//   u[o][i][j] = sum_c W[o][c] v[c][i][j] + b[o] + n^-2 Re sum_kappa g[o](kappa) e^{+2 pi i kappa.(i,j)/n}
//   v'         = GELU(u)                                    (layers 1-3; layer 4 is folded away)
//   c'[o](k)   = sum_{i,j} v'[o][i][j] e^{-2 pi i k.(i,j)/n}
// The DFTs are separable; every contraction is a dense GEMM on the 5th-gen tensor cores:
//
//   k_ysyn_tc   per (system, 6 channels): G[i][(o,k')] = Fp[i][(k1,p)] . Gh[(k1,p)][(o,k')]          (y-synthesis)
//   k_tc_layer  tile = R rows of one system; TMEM lane = o * R + r (channel-major so padding channels fill whole warps), R * WP = 128
//     D1[(r,o)][j]  = sum_{(r',c)} Wbd[(r,o)][(r',c)] V[(r',c)][j]      bypass, block-diagonal in r
//                   + sum_{k'} G[(r,o)][k'] Basis[k'][j]                 x-synthesis (k' = (kappa2, re|im))
//     epilogue      v' = GELU(D1 + b) -> next layer's V blob, and into TMEM (A operand of D2)
//     D2[(r,o)][k'] = sum_j v'[(r,o)][j] F[j][k']                        x-analysis
//     epilogue      -> T blob
//   k_yan_tc    per (system, 128 (kappa2,o) rows): C^T[(k2,o)][(k1,p)] = T[(k2,o)][(i,p')] . Ap[(i,p')][(k1,p)]
//
// Every tensor passed between these kernels lives in HBM as a "blob" already split into bf16
// hi + lo in its consumer's canonical core-matrix layout (tc_layout.cuh), so consumers stage a
// tile with one cp.async.bulk on an mbarrier (prefetched during the previous tile's epilogue) and
// producers convert in their epilogues.
//
// Precision: each product is accumulated as hi*hi + hi*lo + lo*hi in fp32 (3xBF16, ~2^-16
// relative per product; the whole NO stays within ~1e-5 relative L2 of the fp64 oracle, inside
// the 1e-4 parity bound).
#include <algorithm>

#include "internal.h"
#include "tc_common.cuh"
#include "tc_layout.cuh"

namespace fcgno {

constexpr int kTcThreads = 256;

// GELU(x) = x/2 (1 + erf(x / sqrt 2)) (reading R11) with a branch-free erf: Abramowitz & Stegun 7.1.26,
// |erf error| <= 1.5e-7 (two orders below the 3xBF16 operand rounding of this path); CUDA's erff
// branches on |x| and executes both sides under divergence.  The reciprocal and the exponential
// are single MUFU operations (relative error ~2^-22, far inside the A&S bound).
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_f(float x) {
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752f, fabsf(x), 1.0f));   // 1 / (1 + p z), z = |x|/sqrt 2
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  const float pe = p * ex2_approx((x * x) * -0.72134752044448170f);   // erfc(z) = p e^{-z^2}, z^2 = x^2 / 2
  return 0.5f * x * (x >= 0.f ? 2.0f - pe : pe);                      // 1 + erf(x/sqrt 2)
}

// 8 consecutive values -> 16 bytes of bf16 hi and 16 bytes of bf16 lo in shared memory
__device__ __forceinline__ void store_split8(unsigned char* hi, unsigned char* lo, const float (&v)[8]) {
  uint4 h, l;
  tc::split8(v, h, l);
  *reinterpret_cast<uint4*>(hi) = h;
  *reinterpret_cast<uint4*>(lo) = l;
}

using tc::tmem_ld8;

// ------------------------------------------------------------------ constant operand blobs
// Built once per NO apply / solve by k_tc_prep (outside the iteration graph) and bulk-copied by
// every persistent CTA: twiddles for the x-direction (BF), the block-diagonal layer weights (AW),
// the y-synthesis twiddles (FP) and the y-analysis twiddles (AP), each as [hi][lo] bf16.
struct TcConst {
  size_t BF, AW[3], FP, AP, MX[3], total;
  uint32_t bf_half, aw_half[3], fp_half, ap_half, mx_half[3];
  int KB[3], KM, NM[3];
  __host__ __device__ TcConst(const TcGeom& g) {
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o = (o + bytes + 1023) & ~size_t(1023); return at; };
    bf_half = (uint32_t)g.n * kKS * 2;
    BF = take(2 * (size_t)bf_half);
    for (int l = 0; l < 3; ++l) {
      const int cin = l == 0 ? 2 : g.w, CP = (cin + 7) & ~7;
      KB[l] = (g.R * CP + 15) & ~15;
      aw_half[l] = 128u * KB[l] * 2;
      AW[l] = take(2 * (size_t)aw_half[l]);
    }
    fp_half = 128u * kKS * 2;
    FP = take(2 * (size_t)fp_half);
    ap_half = (uint32_t)kKS * (2 * g.n) * 2;
    AP = take(2 * (size_t)ap_half);
    // mode-mixing B operands per mode: rows o (NM), K = (c, re|im) (KM) holding (Rr, Ri) of R[c][o]
    // (the A side carries the complex structure, k_mix_tc); mixes for layers 2, 3 and the
    // layer-4/projection fold (cout = 1)
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

struct TcPrepArgs {
  int n, w;
  const float2* Rm[3];    // mixing weights [400][w][cout] (layers 2, 3; Q with cout = 1)
  const float* W[3];      // layer weights [w][cin] (layer 1: W1E [w][2])
  const float2* F;        // [n][20]
  unsigned char* out;
};

__global__ void __launch_bounds__(256) k_tc_prep(const TcPrepArgs a) {
  const TcGeom g(a.n, a.w);
  const TcConst C(g);
  const int n = a.n, w = a.w, WP = g.WP, R = g.R;
  const int nBF = n * (kKS / 8), nFP = 128 * (kKS / 8), nAP = kKS * (2 * n / 8);
  int nAW[3], nMX[3], tot = nBF + nFP + nAP;
  for (int l = 0; l < 3; ++l) { nAW[l] = 128 * (C.KB[l] / 8); tot += nAW[l]; }
  for (int l = 0; l < 3; ++l) { nMX[l] = kModes2 * C.NM[l] * (C.KM / 8); tot += nMX[l]; }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
    float v[8];
    unsigned char* dst;
    uint32_t half, off;
    int u = t;
    if (u < nBF) {                       // F[j][k'] K-major (N = j, K = k')
      const int j = u % n, kc = u / n;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kp = kc * 8 + q;
        v[q] = 0.f;
        if (kp < 2 * kModes) { const float2 f = a.F[(size_t)j * kModes + (kp >> 1)]; v[q] = (kp & 1) ? f.y : f.x; }
      }
      dst = a.out + C.BF; half = C.bf_half; off = tc::kmajor_off(j, kc * 8, (kKS / 8) * 128, 128);
    } else if ((u -= nBF) < nFP) {       // Fp[i][(k1,p)] (rows i < n), K-major
      const int i = u % 128, kc = u / 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = kc * 8 + q, k1 = k >> 1;
        v[q] = 0.f;
        if (i < n && k1 < kModes) { const float2 f = a.F[(size_t)i * kModes + k1]; v[q] = (k & 1) ? f.y : f.x; }
      }
      dst = a.out + C.FP; half = C.fp_half; off = tc::kmajor_off(i, kc * 8, (kKS / 8) * 128, 128);
    } else if ((u -= nFP) < nAP) {       // Ap^T: row (k1, pout), K = (i, pin)
      const int nn = u % kKS, kc = u / kKS, k1 = nn >> 1, pout = nn & 1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = kc * 4 + q;
        float2 f = make_float2(0.f, 0.f);
        if (k1 < kModes) f = a.F[(size_t)i * kModes + k1];
        v[2 * q] = pout ? f.y : f.x;
        v[2 * q + 1] = pout ? f.x : -f.y;
      }
      dst = a.out + C.AP; half = C.ap_half; off = tc::kmajor_off(nn, kc * 8, ((2 * n) / 8) * 128, 128);
    } else if ((u -= nAP) >= nAW[0] + nAW[1] + nAW[2]) {   // mixing B: row o, K = (c, re|im) = (Rr, Ri)
      u -= nAW[0] + nAW[1] + nAW[2];
      int l = 0;
      while (u >= nMX[l]) { u -= nMX[l]; ++l; }
      const int cout = l < 2 ? w : 1, NM = C.NM[l], KM = C.KM;
      const int per_mode = NM * (KM / 8), kk = u / per_mode, rem = u % per_mode, nn = rem % NM, kc = rem / NM;
      const int o = nn;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = kc * 4 + q;
        float rr = 0.f, ri = 0.f;
        if (c < w && o < cout) { const float2 R2 = a.Rm[l][((size_t)kk * w + c) * cout + o]; rr = R2.x; ri = R2.y; }
        v[2 * q] = rr;
        v[2 * q + 1] = ri;
      }
      dst = a.out + C.MX[l] + (size_t)kk * 2 * C.mx_half[l]; half = C.mx_half[l];
      off = tc::kmajor_off(nn, kc * 8, (KM / 8) * 128, 128);
    } else {                             // Wbd[(r,o)][(r',c)] per layer
      int l = 0;
      while (u >= nAW[l]) { u -= nAW[l]; ++l; }
      const int cin = l == 0 ? 2 : w, CP = (cin + 7) & ~7, KB = C.KB[l];
      const int Lr = u % 128, kc = u / 128, r = Lr % R, o = Lr / R;   // lane = (o, r): padding in whole warps
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kk = kc * 8 + q, rp = kk / CP, c = kk % CP;
        v[q] = (rp == r && rp < R && o < w && c < cin) ? a.W[l][(size_t)o * cin + c] : 0.f;
      }
      dst = a.out + C.AW[l]; half = C.aw_half[l]; off = tc::kmajor_off(Lr, kc * 8, (KB / 8) * 128, 128);
    }
    uint4 h, lo;
    tc::split8(v, h, lo);
    *reinterpret_cast<uint4*>(dst + off) = h;
    *reinterpret_cast<uint4*>(dst + half + off) = lo;
  }
}

// ------------------------------------------------------------------ k_tc_layer
constexpr int kTcMaxSys = 4096;   // running-system bitmask cached in shared memory up to this batch

struct TcSmem {
  // byte offsets; every region 1024-aligned; [hi][lo] back to back like their blobs
  uint32_t BV, AG, BF, RK, TS, PJ, bar, tptr, bias, runb, total;
  int KB, CP;
  __host__ __device__ TcSmem(const TcGeom& g, int cin) {
    CP = (cin + 7) & ~7;
    KB = (g.R * CP + 15) & ~15;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    BV = take(2u * (uint32_t)g.n * KB * 2);
    AG = take(2u * g.g_half());
    BF = take(2u * (uint32_t)g.n * kKS * 2);
    RK = take(cin == 2 ? 2u * g.R * g.n * 8 : 16u);   // layer 1: fp64 rows of r and k
    TS = take(2u * (2 * g.R) * (uint32_t)(g.mtiles * 128) * 2);   // T tile staging [hi|lo][k_local][m]
    PJ = take(4u * g.R * (uint32_t)g.n * 4);                      // layer 3: per-warp-quad projection partials
    bar = take(64);
    tptr = bar + 40;
    bias = take(128 * 4);
    runb = take(kTcMaxSys / 8);
    total = o;
  }
};

struct TcLayerArgs {
  int n, w, cin, B, use_gelu, layer;
  const double* r; const double* rr; const double* k;   // layer 1 inputs
  const unsigned char* vin;                              // V blobs (layers 2, 3)
  const float* W;                                        // [w][cin] (layer 1: W1E [w][2])
  const float* bias;                                     // [w]
  const unsigned char* G;                                // G blobs
  const unsigned char* cst;                              // constant blobs (TcConst)
  unsigned char* vout;                                   // V blobs of the next layer
  unsigned char* T;                                      // T blobs
  const float* dw;                                       // layer 3: projection weights (D W4) [w]
  float* pout;                                           // layer 3: sum_o dw[o] v3[o] per pixel [B][n][n]
  const int* status;
};

template <int WP, bool FIRST>
__global__ void __launch_bounds__(kTcThreads, 2) k_tc_layer(const TcLayerArgs a) {
  const TcGeom g(a.n, a.w);
  const TcConst C(g);
  constexpr int R = 128 / WP;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = n * n, w = a.w, cin = a.cin;
  const TcSmem L(g, cin);
  const int KB = L.KB, CP = L.CP;                     // of this layer's input (FIRST: cin = 2)
  const uint32_t SBO_AW = (KB / 8) * 128, SBO_BV = (KB / 8) * 128, SBO_AG = g.g_sbo(), SBO_F = (kKS / 8) * 128;
  const uint32_t aw_half = 128u * KB * 2, bv_half = (uint32_t)KB * n * 2, bf_half = (uint32_t)n * kKS * 2;
  const uint32_t vout_half = g.v_half(), vout_sbo = g.v_sbo();   // next layer's V blob geometry (cin = w)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0] tile loads, [1] D1, [2] D2, [3] constants
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  const double* rk = reinterpret_cast<const double*>(sm + L.RK);
  const bool proj = a.pout != nullptr;                  // layer 3 of the fused projection path
  float* pj = reinterpret_cast<float*>(sm + L.PJ);      // [4 warp quads][R][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // TMEM: D1 / D2 (aliased) [0, n), v' hi/lo (A of D2) [n, 2n), Wbd hi/lo (A of the bypass) [2n, 2n+KB)
  const uint32_t need = 2u * n + (uint32_t)KB;
  const uint32_t ncols = need <= 128 ? 128u : (need <= 256 ? 256u : 512u);
  const int ntiles = a.B * g.tiles_per_sys;
  uint32_t* runb = reinterpret_cast<uint32_t*>(sm + L.runb);   // running-system bitmask (B <= kTcMaxSys)
  const bool cached = a.status && a.B <= kTcMaxSys;
  auto running = [&](int t) {
    const int sb = t / g.tiles_per_sys;
    if (!a.status) return true;
    if (cached) return ((runb[sb >> 5] >> (sb & 31)) & 1u) != 0;
    return __ldcg(a.status + sb) == SYS_RUNNING;
  };
  auto next_tile = [&](int t) {
    while (t < ntiles && !running(t)) t += gridDim.x;
    return t;
  };
  const uint32_t rk_bytes = (uint32_t)R * n * 8;
  const uint32_t in_bytes = FIRST ? 2u * g.g_half() + 2u * rk_bytes : 2u * bv_half + 2u * g.g_half();
  // one thread: bulk copies of tile t's inputs.  V (or r, k) was produced before this kernel's
  // predecessor started; G is the predecessor's output (copied only after griddepcontrol.wait).
  auto prefetch_v = [&](int t) {
    const int tb = t / g.tiles_per_sys, ti0 = (t % g.tiles_per_sys) * R;
    tc::mbar_expect_tx(&bar[0], in_bytes);
    if (FIRST) {
      const size_t e = (size_t)tb * N + (size_t)ti0 * n;
      tc::bulk_g2s(sm + L.RK, a.r + e, rk_bytes, &bar[0]);
      tc::bulk_g2s(sm + L.RK + rk_bytes, a.k + e, rk_bytes, &bar[0]);
    } else {
      tc::bulk_g2s(sm + L.BV, a.vin + (size_t)t * 2 * bv_half, 2u * bv_half, &bar[0]);
    }
  };
  auto prefetch_g = [&](int t) { tc::bulk_g2s(sm + L.AG, a.G + (size_t)t * 2 * g.g_half(), 2u * g.g_half(), &bar[0]); };
  auto prefetch = [&](int t) { prefetch_v(t); prefetch_g(t); };

  // ---- one-time setup, overlapping the predecessor's tail (programmatic dependent launch): barriers,
  // constant operands, the running-system bitmask (status is written only by k_update, which
  // completed before the predecessor started; read through L2), the first tile's V operand, TMEM,
  // bias and the block-diagonal weights.  Only the G operand waits for griddepcontrol.wait.
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&bar[3], 2u * bf_half);
    tc::bulk_g2s(sm + L.BF, a.cst + C.BF, 2u * bf_half, &bar[3]);
  }
  if (cached) {
    for (int q = warp; q < (a.B + 31) / 32; q += blockDim.x / 32) {
      const int sb = q * 32 + lane;
      const unsigned bits = __ballot_sync(0xffffffffu, sb < a.B && __ldcg(a.status + sb) == SYS_RUNNING);
      if (lane == 0) runb[q] = bits;
    }
  }
  __syncthreads();
  int tile = next_tile(blockIdx.x);
  if (tid == 0 && tile < ntiles) prefetch_v(tile);
  if (warp == 0) tc::tmem_alloc(tptr, ncols);

  for (int t = tid; t < 128; t += blockDim.x) {
    const int o = t / R;
    sbias[t] = o < w ? a.bias[o] : 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t tD1 = tmem, tD2 = tmem;                 // D2 is issued after epilogue 1 drained D1
  const uint32_t tAh = tmem + (uint32_t)n, tAl = tAh + (uint32_t)(n / 2);
  const uint32_t tWh = tmem + 2u * n, tWl = tWh + (uint32_t)(KB / 2);
  // Wbd rows into TMEM (lane = (r, o)) from the prebuilt K-major blob: warps 0-3, one lane per row
  if (warp < 4) {
    const int Lr = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const unsigned char* aw = a.cst + C.AW[a.layer];
    for (int k0 = 0; k0 < KB; k0 += 16) {
      uint32_t hi8[8], lo8[8];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t off = tc::kmajor_off(Lr, k0 + 8 * hh, SBO_AW, 128);
        const uint4 h = __ldg(reinterpret_cast<const uint4*>(aw + off));
        const uint4 l = __ldg(reinterpret_cast<const uint4*>(aw + aw_half + off));
        hi8[4 * hh] = h.x; hi8[4 * hh + 1] = h.y; hi8[4 * hh + 2] = h.z; hi8[4 * hh + 3] = h.w;
        lo8[4 * hh] = l.x; lo8[4 * hh + 1] = l.y; lo8[4 * hh + 2] = l.z; lo8[4 * hh + 3] = l.w;
      }
      tc::tmem_st8(tWh + lane_off + k0 / 2, hi8);
      tc::tmem_st8(tWl + lane_off + k0 / 2, lo8);
    }
    tc::tmem_wait_st();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t id1 = tc::make_idesc_bf16(128, n, false, true);     // A (TMEM), B MN-major (bypass)
  const uint32_t id1s = tc::make_idesc_bf16(128, n, false, false);   // synthesis: both K-major
  const uint32_t id2 = tc::make_idesc_bf16(128, kKS, false, true);   // analysis: B = F viewed MN-major
  const uint32_t sm_base = tc::smem_u32(sm);
  pdl_wait();
  pdl_trigger();
  if (tid == 0 && tile < ntiles) prefetch_g(tile);
  if (tid == 0) tc::mbar_wait(&bar[3], 0);

  uint32_t ph = 0;
  for (; tile < ntiles; tile = next_tile(tile + gridDim.x)) {
    const int b = tile / g.tiles_per_sys, i0 = (tile % g.tiles_per_sys) * R;
    if (FIRST) {   // layer 1: V = [r/||r||, k] converted from the prefetched fp64 rows
      tc::mbar_wait(&bar[0], ph);
      const double s = sqrt(a.rr[b]);
      const double inv_s = s > 0.0 ? 1.0 / s : 0.0;
      for (int t = tid; t < KB * (n / 8); t += blockDim.x) {
        const int kk = t % KB, jc = t / KB;
        const int rp = kk / CP, c = kk % CP;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0.f;
        if (rp < R && c < cin) {
          const double* src = rk + (size_t)c * R * n + (size_t)rp * n + jc * 8;
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (float)(c == 0 ? src[q] * inv_s : src[q]);
        }
        const uint32_t off = tc::mnmajor_off(jc * 8, kk, SBO_BV, 128);
        store_split8(sm + L.BV + off, sm + L.BV + bv_half + off, v);
      }
      tc::fence_proxy_async_smem();
      __syncthreads();
    }
    // ---- D1 = Wbd V + G Basis   (3xBF16: hi*hi + hi*lo + lo*hi)
    if (tid == 0) {
      if (!FIRST) tc::mbar_wait(&bar[0], ph);
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < KB / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t at = (p == 2 ? tWl : tWh) + 8u * s, bo = L.BV + (p == 1 ? bv_half : 0u) + 256u * s;
          tc::mma_bf16_ts(tD1, at, tc::make_sdesc(sm_base + bo, 128, SBO_BV), id1, acc);
          acc = 1;
        }
      }
      for (int s = 0; s < kKS / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t ao = L.AG + (p == 2 ? g.g_half() : 0u) + 256u * s, bo = L.BF + (p == 1 ? bf_half : 0u) + 256u * s;
          tc::mma_bf16(tD1, tc::make_sdesc(sm_base + ao, 128, SBO_AG), tc::make_sdesc(sm_base + bo, 128, SBO_F), id1s, 1);
        }
      }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], ph);
    tc::fence_after_sync();
    // the MMAs have consumed BV / AG / RK: prefetch the next tile while the epilogues run
    if (tid == 0) {
      const int tn = next_tile(tile + gridDim.x);
      if (tn < ntiles) prefetch(tn);
    }
    // ---- epilogue 1: v' = GELU(D1 + b) -> next V blob (bf16 hi/lo) and -> TMEM (A operand of D2)
    // Lane = (o, r); warps whose 32 lanes are all padding channels skip (their D2 rows are unused).
    if ((32 * (warp & 3)) / R < g.CP) {
      const int q4 = warp & 3, half = warp >> 2;
      const int Lr = q4 * 32 + lane;
      const int r = Lr % R, o = Lr / R;
      const float bo = sbias[Lr];
      const float dwo = (proj && o < w) ? a.dw[o] : 0.f;
      const bool store = o < g.CP;                       // rows (r, o >= w) carry exact zeros
      unsigned char* vb = a.vout + (size_t)tile * 2 * vout_half;
      const uint32_t kk = (uint32_t)(r * g.CP + o);
      const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
      for (int c0 = half * (n / 2); c0 < (half + 1) * (n / 2); c0 += 16) {
        uint32_t u[16];
        tc::tmem_ld16(tD1 + lane_off + c0, u);
        tc::tmem_wait_ld();
        float v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float x = __uint_as_float(u[t]) + bo;
          v[t] = a.use_gelu ? gelu_f(x) : x;
        }
        uint32_t ph8[8], pl8[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) tc::split2(v[2 * t], v[2 * t + 1], ph8[t], pl8[t]);
        if (proj) {                                     // layer 3: sum_o dw[o] v3[(o, r)][j] instead of the blob
          float pp[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) pp[t] = dwo * v[t];
#pragma unroll
          for (int off = 16; off >= R; off >>= 1)
#pragma unroll
            for (int t = 0; t < 16; ++t) pp[t] += __shfl_xor_sync(0xffffffffu, pp[t], off);
          if (lane < R)
#pragma unroll
            for (int t = 0; t < 16; ++t) pj[((size_t)q4 * R + r) * n + c0 + t] = pp[t];
        } else if (store) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t off = tc::mnmajor_off(c0 + 8 * hh, kk, vout_sbo, 128);
            *reinterpret_cast<uint4*>(vb + off) = make_uint4(ph8[4 * hh], ph8[4 * hh + 1], ph8[4 * hh + 2], ph8[4 * hh + 3]);
            *reinterpret_cast<uint4*>(vb + vout_half + off) =
                make_uint4(pl8[4 * hh], pl8[4 * hh + 1], pl8[4 * hh + 2], pl8[4 * hh + 3]);
          }
        }
        tc::tmem_st8(tAh + lane_off + c0 / 2, ph8);
        tc::tmem_st8(tAl + lane_off + c0 / 2, pl8);
      }
      tc::tmem_wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    if (proj) {   // fixed-order sum over the 4 warp quads (quads made only of padding lanes wrote nothing)
      const int nq = min(4, (g.CP * R + 31) / 32);
      for (int e = tid; e < R * n; e += blockDim.x) {
        float acc = 0.f;
        for (int q = 0; q < nq; ++q) acc += pj[(size_t)q * R * n + e];
        a.pout[(size_t)b * N + (size_t)i0 * n + e] = acc;
      }
    }
    // ---- D2 = v' F  (x-analysis)
    if (tid == 0) {
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < n / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t at = (p == 2 ? tAl : tAh) + 8u * s;     // 16 bf16 of K = 8 TMEM columns
          // F viewed MN-major (N = k', K = j): LBO = K-group stride = SBO_F, SBO = N-group stride = 128
          const uint64_t bd = tc::make_sdesc(sm_base + L.BF + (p == 1 ? bf_half : 0u) + 2u * SBO_F * s, SBO_F, 128);
          tc::mma_bf16_ts(tD2, at, bd, id2, acc);
          acc = 1;
        }
      }
      tc::mma_commit(&bar[2]);
    }
    tc::mbar_wait(&bar[2], ph);
    tc::fence_after_sync();
    // ---- epilogue 2: D2 -> T blob.  Stage [hi|lo][k_local = (r, re|im)][m = (o, k2)] in smem, then
    // copy 2R*16-byte runs per 8-row m group into the MN-major T blob (tc_layout.cuh).
    {
      const int q4 = warp & 3, half = warp >> 2;
      const int Lr = q4 * 32 + lane;
      const int r = Lr % R, o = Lr / R;
      const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
      const int MT = g.mtiles * 128;
      __nv_bfloat16* ts = reinterpret_cast<__nv_bfloat16*>(sm + L.TS);
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {               // columns [24*half, 24*half + 24) in chunks of 8 (< 40)
        const int c0 = half * 24 + cc * 8;
        if (c0 >= 2 * kModes) break;
        uint32_t u[8];
        tmem_ld8(tD2 + lane_off + c0, u);
        tc::tmem_wait_ld();
        if (o < w) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int k2 = (c0 + q) >> 1, pin = (c0 + q) & 1, m = k2 * w + o, kl = 2 * r + pin;
            __nv_bfloat16 h, l;
            tc::split_bf16(__uint_as_float(u[q]), h, l);
            ts[(size_t)kl * MT + m] = h;
            ts[(size_t)(2 * R + kl) * MT + m] = l;
          }
        }
      }
      __syncthreads();
      const int KL = 2 * R, k0 = 2 * i0;                        // this tile's K range [k0, k0 + 2R)
      const int ngroups = (w * kModes + 7) / 8;
      const uint32_t t_half = g.t_half(), t_lbo = g.t_lbo();
      unsigned char* tb = a.T + (size_t)b * g.mtiles * 2 * t_half;
      for (int e = tid; e < 2 * ngroups; e += blockDim.x) {
        const int hl = e / ngroups, grp = e % ngroups, mt = grp / 16, gi = grp % 16;
        unsigned char* dst = tb + ((size_t)mt * 2 + hl) * t_half + (uint32_t)gi * 128 + (uint32_t)(k0 / 8) * t_lbo +
                             (uint32_t)(k0 % 8) * 16;
#pragma unroll 8
        for (int kl = 0; kl < KL; ++kl)
          *reinterpret_cast<uint4*>(dst + kl * 16) =
              *reinterpret_cast<const uint4*>(ts + (size_t)(hl * KL + kl) * MT + grp * 8);
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    ph ^= 1;
  }
  tc::fence_after_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ------------------------------------------------------------------ k_tc_layer_ws: pipelined layer
// Same arithmetic as k_tc_layer; one CTA (16 warps) per SM, split into two groups of 8 warps that
// take the CTA's tiles alternately (group e: tiles it = e, e+2, ...).  Each group's leader thread
// issues its own MMAs at the points its data is ready -- no dedicated producer / MMA warps, so no
// thread spins and all 16 warps keep the 128-register budget:
//   after epilogue 1 of tile it:  D2(it) and D1(it + 2) (separate TMEM accumulators)
//   after D1(it) completed:       bulk loads of tile it + S into the stage D1(it) consumed
// so the tensor pipe runs a group's next D1 under its epilogue 2, the other group's epilogues run
// under this group's MMAs, and loads run S tiles ahead.  TMEM (512 columns): per group e, D1 at
// e*n, D2 at 2n + 48e, v' hi|lo at 2n + 96 + e*n; Wbd hi|lo at 4n + 96 (needs 4n + 96 + KB <= 512).
constexpr int kWsGroupWarps = 8;
constexpr int kWsThreads = 2 * kWsGroupWarps * 32;
constexpr int kWsStages = 3;
constexpr int kWsMaxTiles = 2048;   // per-CTA tile list cached in shared memory

struct TcWsSmem {
  uint32_t BV, AG, RK, BF, TS, PJ, bar, tptr, bias, list, total;
  int KB, CP, stages;
  __host__ __device__ TcWsSmem(const TcGeom& g, int cin, int stages_) : stages(stages_) {
    CP = (cin + 7) & ~7;
    KB = (g.R * CP + 15) & ~15;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    BV = take((uint32_t)stages * bv_stage_bytes(g));
    AG = take((uint32_t)stages * 2u * g.g_half());
    RK = take(cin == 2 ? (uint32_t)stages * 2u * g.R * g.n * 8 : 16u);
    BF = take(2u * (uint32_t)g.n * kKS * 2);
    TS = take(2u * ts_bytes(g));
    PJ = take(2u * pj_bytes(g));
    bar = take(256);           // mbarriers + TMEM pointer + tile count
    tptr = bar + 192;
    bias = take(128 * 4);
    list = take(kWsMaxTiles * 4);
    total = o;
  }
  __host__ __device__ uint32_t bv_stage_bytes(const TcGeom& g) const { return 2u * (uint32_t)g.n * KB * 2; }
  __host__ __device__ static uint32_t ts_bytes(const TcGeom& g) { return 2u * (2 * g.R) * (uint32_t)(g.mtiles * 128) * 2; }
  __host__ __device__ static uint32_t pj_bytes(const TcGeom& g) { return 4u * g.R * (uint32_t)g.n * 4; }
};

__host__ __device__ inline bool ws_tmem_fits(const TcGeom& g, int KB) { return 4 * g.n + 2 * kKS + KB <= 512; }

template <int WP, bool FIRST>
__global__ void __launch_bounds__(kWsThreads, 1) k_tc_layer_ws(const TcLayerArgs a, const int stages) {
  const TcGeom g(a.n, a.w);
  const TcConst C(g);
  constexpr int R = 128 / WP;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = n * n, w = a.w, cin = a.cin;
  const TcWsSmem L(g, cin, stages);
  const int KB = L.KB, CP = L.CP;
  const uint32_t SBO_AW = (KB / 8) * 128, SBO_BV = (KB / 8) * 128, SBO_AG = g.g_sbo(), SBO_F = (kKS / 8) * 128;
  const uint32_t aw_half = 128u * KB * 2, bv_half = (uint32_t)KB * n * 2, bf_half = (uint32_t)n * kKS * 2;
  const uint32_t g_half = g.g_half(), rk_bytes = (uint32_t)R * n * 8;
  const uint32_t vout_half = g.v_half(), vout_sbo = g.v_sbo();
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);
  uint64_t* full = bar;          // [3] stage loaded (layer 1: raw fp64 rows and G landed)
  uint64_t* d1full = bar + 4;    // [2] D1 of group e's current tile complete
  uint64_t* d2full = bar + 6;    // [2] D2 complete
  uint64_t* cstb = bar + 8;      // constant x-direction twiddles landed
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  int* pcnt = reinterpret_cast<int*>(sm + L.tptr + 4);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  int* list = reinterpret_cast<int*>(sm + L.list);
  const bool proj = a.pout != nullptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = a.B * g.tiles_per_sys;
  const uint32_t sm_base = tc::smem_u32(sm);

  auto issue_loads = [&](int it) {   // one thread: bulk copies of list[it] into stage it % stages
    const int tile = list[it], s = it % stages;
    const int tb = tile / g.tiles_per_sys, ti0 = (tile % g.tiles_per_sys) * R;
    unsigned char* ag = sm + L.AG + (uint32_t)s * 2u * g_half;
    if (FIRST) {
      unsigned char* rk = sm + L.RK + (uint32_t)s * 2u * rk_bytes;
      const size_t e = (size_t)tb * N + (size_t)ti0 * n;
      tc::mbar_expect_tx(&full[s], 2u * rk_bytes + 2u * g_half);
      tc::bulk_g2s(rk, a.r + e, rk_bytes, &full[s]);
      tc::bulk_g2s(rk + rk_bytes, a.k + e, rk_bytes, &full[s]);
    } else {
      tc::mbar_expect_tx(&full[s], 2u * bv_half + 2u * g_half);
      tc::bulk_g2s(sm + L.BV + (uint32_t)s * L.bv_stage_bytes(g), a.vin + (size_t)tile * 2 * bv_half, 2u * bv_half, &full[s]);
    }
    tc::bulk_g2s(ag, a.G + (size_t)tile * 2 * g_half, 2u * g_half, &full[s]);
  };

  if (tid == 0) {
    for (int q = 0; q < 9; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(cstb, 2u * bf_half);
    tc::bulk_g2s(sm + L.BF, a.cst + C.BF, 2u * bf_half, cstb);
  }
  pdl_wait();
  if (tid == 0) {   // this CTA's tiles (running systems only), in order
    int cnt = 0;
    for (int t = blockIdx.x; t < ntiles && cnt < kWsMaxTiles; t += gridDim.x)
      if (!a.status || a.status[t / g.tiles_per_sys] == SYS_RUNNING) list[cnt++] = t;
    *pcnt = cnt;
    for (int it = 0; it < cnt && it < stages; ++it) issue_loads(it);
  }
  if (warp == 0) tc::tmem_alloc(tptr, 512);
  for (int t = tid; t < 128; t += blockDim.x) {
    const int o = t / R;
    sbias[t] = o < w ? a.bias[o] : 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  pdl_trigger();   // after the TMEM allocation: a dependent CTA placed on this SM cannot take the columns first
  const uint32_t tmem = *tptr;
  const int cnt = *pcnt;
  const uint32_t tWh = tmem + 4u * n + 2u * kKS, tWl = tWh + (uint32_t)(KB / 2);
  if (warp < 4) {   // Wbd rows into TMEM (lane = (o, r)) from the prebuilt K-major blob
    const int Lr = warp * 32 + lane;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const unsigned char* aw = a.cst + C.AW[a.layer];
    for (int k0 = 0; k0 < KB; k0 += 16) {
      uint32_t hi8[8], lo8[8];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t off = tc::kmajor_off(Lr, k0 + 8 * hh, SBO_AW, 128);
        const uint4 h = __ldg(reinterpret_cast<const uint4*>(aw + off));
        const uint4 l = __ldg(reinterpret_cast<const uint4*>(aw + aw_half + off));
        hi8[4 * hh] = h.x; hi8[4 * hh + 1] = h.y; hi8[4 * hh + 2] = h.z; hi8[4 * hh + 3] = h.w;
        lo8[4 * hh] = l.x; lo8[4 * hh + 1] = l.y; lo8[4 * hh + 2] = l.z; lo8[4 * hh + 3] = l.w;
      }
      tc::tmem_st8(tWh + lane_off + k0 / 2, hi8);
      tc::tmem_st8(tWl + lane_off + k0 / 2, lo8);
    }
    tc::tmem_wait_st();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();

  const int grp = warp / kWsGroupWarps, q4 = warp & 3, slice = (warp >> 2) & 1;
  const bool leader = (warp % kWsGroupWarps) == 0 && lane == 0;
  constexpr uint32_t kGrpThreads = kWsGroupWarps * 32;
  const uint32_t nbar = 1 + grp;
  const int gtid = tid - grp * (int)kGrpThreads;
  const uint32_t tD1 = tmem + (uint32_t)(grp * n), tD2 = tmem + 2u * n + (uint32_t)(grp * kKS);
  const uint32_t tA = tmem + 2u * n + 2u * kKS + (uint32_t)(grp * n), tAl = tA + (uint32_t)(n / 2);
  const uint32_t id1 = tc::make_idesc_bf16(128, n, false, true);
  const uint32_t id1s = tc::make_idesc_bf16(128, n, false, false);
  const uint32_t id2 = tc::make_idesc_bf16(128, kKS, false, true);

  // layer 1: V = [r/||r||, k] of tile list[it] from its raw fp64 rows, by the group's 256 threads
  auto convert = [&](int it) {
    const int s = it % stages, tile = list[it], tb = tile / g.tiles_per_sys;
    tc::mbar_wait(&full[s], (uint32_t)(it / stages) & 1);
    const double sr = sqrt(a.rr[tb]);
    const double inv_s = sr > 0.0 ? 1.0 / sr : 0.0;
    const double* rkd = reinterpret_cast<const double*>(sm + L.RK + (uint32_t)s * 2u * rk_bytes);
    unsigned char* bv = sm + L.BV + (uint32_t)s * L.bv_stage_bytes(g);
    for (int t = gtid; t < KB * (n / 8); t += kGrpThreads) {
      const int kk = t % KB, jc = t / KB, rp = kk / CP, c = kk % CP;
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = 0.f;
      if (rp < R && c < cin) {
        const double* src = rkd + (size_t)c * R * n + (size_t)rp * n + jc * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (float)(c == 0 ? src[q] * inv_s : src[q]);
      }
      const uint32_t off = tc::mnmajor_off(jc * 8, kk, SBO_BV, 128);
      store_split8(bv + off, bv + bv_half + off, v);
    }
    tc::fence_proxy_async_smem();
  };
  // leader: D1 = Wbd V + G Basis of tile list[it] into this group's D1 accumulator
  auto issue_d1 = [&](int it) {
    const int s = it % stages;
    if (!FIRST) tc::mbar_wait(&full[s], (uint32_t)(it / stages) & 1);
    tc::fence_after_sync();
    const uint32_t bvs = L.BV + (uint32_t)s * L.bv_stage_bytes(g), ags = L.AG + (uint32_t)s * 2u * g_half;
    uint32_t acc = 0;
    for (int q = 0; q < KB / 16; ++q) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t at = (p == 2 ? tWl : tWh) + 8u * q, bo = bvs + (p == 1 ? bv_half : 0u) + 256u * q;
        tc::mma_bf16_ts(tD1, at, tc::make_sdesc(sm_base + bo, 128, SBO_BV), id1, acc);
        acc = 1;
      }
    }
    for (int q = 0; q < kKS / 16; ++q) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t ao = ags + (p == 2 ? g_half : 0u) + 256u * q, bo = L.BF + (p == 1 ? bf_half : 0u) + 256u * q;
        tc::mma_bf16(tD1, tc::make_sdesc(sm_base + ao, 128, SBO_AG), tc::make_sdesc(sm_base + bo, 128, SBO_F), id1s, 1);
      }
    }
    tc::mma_commit(&d1full[grp]);
  };
  // leader: D2 = v' F (x-analysis) of the group's current tile
  auto issue_d2 = [&]() {
    tc::fence_after_sync();
    uint32_t acc = 0;
    for (int q = 0; q < n / 16; ++q) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t at = (p == 2 ? tAl : tA) + 8u * q;
        const uint64_t bd = tc::make_sdesc(sm_base + L.BF + (p == 1 ? bf_half : 0u) + 2u * SBO_F * q, SBO_F, 128);
        tc::mma_bf16_ts(tD2, at, bd, id2, acc);
        acc = 1;
      }
    }
    tc::mma_commit(&d2full[grp]);
  };

  const int Lr = q4 * 32 + lane, r = Lr % R, o = Lr / R;
  const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
  const bool live = (32 * q4) / R < g.CP;            // warp holds at least one real channel row
  const float bo = sbias[Lr];
  const float dwo = (proj && o < w) ? a.dw[o] : 0.f;
  const bool store = o < g.CP;
  const uint32_t kk = (uint32_t)(r * g.CP + o);
  const int nch = n / 8;                               // 8-column chunks of D1; slice takes c = slice + 2k
  const int MT = g.mtiles * 128;
  __nv_bfloat16* ts = reinterpret_cast<__nv_bfloat16*>(sm + L.TS + (uint32_t)grp * TcWsSmem::ts_bytes(g));
  float* pj = reinterpret_cast<float*>(sm + L.PJ + (uint32_t)grp * TcWsSmem::pj_bytes(g));

  if (grp < cnt) {   // the group's first tile: stage it and start its D1
    if (FIRST) {
      tc::mbar_wait(cstb, 0);
      convert(grp);
      tc::named_sync(nbar, kGrpThreads);
    }
    if (leader) {
      tc::mbar_wait(cstb, 0);
      issue_d1(grp);
    }
  }
  for (int it = grp; it < cnt; it += 2) {
    const int tile = list[it], b = tile / g.tiles_per_sys, i0 = (tile % g.tiles_per_sys) * R;
    const uint32_t par = (uint32_t)(it >> 1) & 1;
    tc::mbar_wait(&d1full[grp], par);
    tc::fence_after_sync();
    if (leader && it + stages < cnt) issue_loads(it + stages);   // D1(it) has consumed stage it % S
    // ---- epilogue 1: v' = GELU(D1 + b) -> next V blob and TMEM (A of D2); layer 3: projection partials
    if (live) {
      unsigned char* vb = a.vout + (size_t)tile * 2 * vout_half;
      for (int c00 = slice; c00 < nch; c00 += 8) {       // batches of up to 4 chunks: c00, c00 + 2, ...
        uint32_t u[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (c00 + 2 * k < nch) tmem_ld8(tD1 + lane_off + 8 * (c00 + 2 * k), u[k]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = c00 + 2 * k;
          if (c >= nch) break;
          float v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const float x = __uint_as_float(u[k][t]) + bo;
            v[t] = a.use_gelu ? gelu_f(x) : x;
          }
          uint32_t ph4[4], pl4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) tc::split2(v[2 * t], v[2 * t + 1], ph4[t], pl4[t]);
          if (proj) {
            float pp[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) pp[t] = dwo * v[t];
#pragma unroll
            for (int off = 16; off >= R; off >>= 1)
#pragma unroll
              for (int t = 0; t < 8; ++t) pp[t] += __shfl_xor_sync(0xffffffffu, pp[t], off);
            if (lane < R) {
              float4* dst = reinterpret_cast<float4*>(pj + ((size_t)q4 * R + r) * n + 8 * c);
              dst[0] = make_float4(pp[0], pp[1], pp[2], pp[3]);
              dst[1] = make_float4(pp[4], pp[5], pp[6], pp[7]);
            }
          } else if (store) {
            const uint32_t off = tc::mnmajor_off(8 * c, kk, vout_sbo, 128);
            *reinterpret_cast<uint4*>(vb + off) = make_uint4(ph4[0], ph4[1], ph4[2], ph4[3]);
            *reinterpret_cast<uint4*>(vb + vout_half + off) = make_uint4(pl4[0], pl4[1], pl4[2], pl4[3]);
          }
          tc::tmem_st4(tA + lane_off + 4 * c, ph4[0], ph4[1], ph4[2], ph4[3]);
          tc::tmem_st4(tAl + lane_off + 4 * c, pl4[0], pl4[1], pl4[2], pl4[3]);
        }
      }
      tc::tmem_wait_st();
    }
    if (FIRST && it + 2 < cnt) convert(it + 2);      // next tile's layer-1 operand, rows landed long ago
    tc::fence_before_sync();
    tc::named_sync(nbar, kGrpThreads);                // v' in TMEM, D1 drained, pj written
    if (leader) {
      issue_d2();
      if (it + 2 < cnt) issue_d1(it + 2);
    }
    if (proj) {   // fixed-order sum over the 4 lane quadrants
      const int nq = min(4, (g.CP * R + 31) / 32);
      for (int e = gtid; e < R * n; e += kGrpThreads) {
        float acc = 0.f;
        for (int q = 0; q < nq; ++q) acc += pj[(size_t)q * R * n + e];
        a.pout[(size_t)b * N + (size_t)i0 * n + e] = acc;
      }
    }
    // ---- epilogue 2: D2 -> T blob via the group's [hi|lo][k_local][m] staging buffer
    tc::mbar_wait(&d2full[grp], par);
    tc::fence_after_sync();
    {
      uint32_t u[3][8];                                // 8-column chunks of the 40 (k2, re|im) columns
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (slice + 2 * k < 5) tmem_ld8(tD2 + lane_off + 8 * (slice + 2 * k), u[k]);
      tc::tmem_wait_ld();
      if (o < w) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int c = slice + 2 * k;
          if (c >= 5) break;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int col = 8 * c + q, k2 = col >> 1, pin = col & 1, m = k2 * w + o, kl = 2 * r + pin;
            __nv_bfloat16 h, l;
            tc::split_bf16(__uint_as_float(u[k][q]), h, l);
            ts[(size_t)kl * MT + m] = h;
            ts[(size_t)(2 * R + kl) * MT + m] = l;
          }
        }
      }
    }
    tc::fence_before_sync();
    tc::named_sync(nbar, kGrpThreads);
    {
      const int KL = 2 * R, k0 = 2 * i0;
      const int ngroups = (w * kModes + 7) / 8;
      const uint32_t t_half = g.t_half(), t_lbo = g.t_lbo();
      unsigned char* tb = a.T + (size_t)b * g.mtiles * 2 * t_half;
      for (int e = gtid; e < 2 * ngroups; e += kGrpThreads) {
        const int hl = e / ngroups, gr = e % ngroups, mt = gr / 16, gi = gr % 16;
        unsigned char* dst = tb + ((size_t)mt * 2 + hl) * t_half + (uint32_t)gi * 128 + (uint32_t)(k0 / 8) * t_lbo +
                             (uint32_t)(k0 % 8) * 16;
#pragma unroll 8
        for (int kl = 0; kl < KL; ++kl)
          *reinterpret_cast<uint4*>(dst + kl * 16) =
              *reinterpret_cast<const uint4*>(ts + (size_t)(hl * KL + kl) * MT + gr * 8);
      }
    }
    tc::named_sync(nbar, kGrpThreads);   // staging buffers (ts, pj) free for the group's next tile
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------ y-direction transforms on tensor cores
// Complex products written as 2x2 real blocks (F = (Fx, Fy) = exp(-2 pi i kappa i / n)):
//   y-synthesis  G[i][(o,k2,re|im)] = sum_{(k1,p)} Fp[i][(k1,p)] * Gh[(k1,p)][(o,k2,re|im)]
//                Fp[i][(k1,0)] = Fx, Fp[i][(k1,1)] = Fy;  Gh rows (k1,0) = (gr | gi), (k1,1) = (gi | -gr)
//   y-analysis   C^T[(o,k2)][(k1,re|im)] = sum_{(i,p)} T[(o,k2)][(i,p)] * Ap[(i,p)][(k1,re|im)]
//                Ap[(i,0)][(k1,re)] = Fx, Ap[(i,1)][(k1,re)] = -Fy, Ap[(i,0)][(k1,im)] = Fy, Ap[(i,1)][(k1,im)] = Fx
constexpr int kYsynCh = 6;                 // channels per work item: N = 6 * 40 = 240
constexpr int kYsynN = kYsynCh * 2 * kModes;

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(tc::smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

struct YsynSmem {
  uint32_t A, B, GS, bar, tptr, total;
  __host__ __device__ YsynSmem() {
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    A = take(2u * 128 * kKS * 2);
    B = take(2u * kYsynN * kKS * 2);
    GS = take((uint32_t)kYsynCh * kModes2 * 8);
    bar = take(64);
    tptr = bar + 32;
    total = o;
  }
};

// persistent over work items (system, 6-channel chunk)
__global__ void __launch_bounds__(128, 2) k_ysyn_tc(const float2* __restrict__ ghat, const unsigned char* __restrict__ cst,
                                                    unsigned char* __restrict__ Gb, int n, int w, int B,
                                                    const int* status) {
  const TcGeom geo(n, w);
  const TcConst C(geo);
  const YsynSmem L;
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr uint32_t SBO = (kKS / 8) * 128;             // K = 48 for both operands (K-major)
  const uint32_t a_half = 128u * kKS * 2, b_half = (uint32_t)kYsynN * kKS * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0] staging, [1] MMA, [2] constants
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  const float2* gs = reinterpret_cast<const float2*>(sm + L.GS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nch = (w + kYsynCh - 1) / kYsynCh, nitems = B * nch;
  auto next_item = [&](int it) {
    while (it < nitems && status && status[it / nch] != SYS_RUNNING) it += gridDim.x;
    return it;
  };
  // all threads: gather g[kappa][b][oc .. oc + 6) of the mode-major ghat into GS [kappa][6] (async)
  auto prefetch = [&](int it) {
    const int b = it / nch, oc = (it % nch) * kYsynCh, nvalid = min(kYsynCh, w - oc);
    float2* gsw = reinterpret_cast<float2*>(sm + L.GS);
    for (int t = tid; t < kModes2 * nvalid; t += blockDim.x) {
      const int kk = t / nvalid, ol = t - kk * nvalid;
      cp_async8(gsw + kk * kYsynCh + ol, ghat + ((size_t)kk * B + b) * w + oc + ol);
    }
    cp_async_commit();
  };
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&bar[2], 2u * a_half);
    tc::bulk_g2s(sm + L.A, cst + C.FP, 2u * a_half, &bar[2]);
  }
  pdl_wait();
  pdl_trigger();
  int it = next_item(blockIdx.x);
  if (it < nitems) prefetch(it);
  if (warp == 0) tc::tmem_alloc(tptr, 256);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t id = tc::make_idesc_bf16(128, kYsynN, false, false);
  const uint32_t base = tc::smem_u32(sm);
  if (tid == 0) tc::mbar_wait(&bar[2], 0);
  uint32_t ph = 0;
  for (; it < nitems; it = next_item(it + gridDim.x)) {
    const int b = it / nch, oc = (it % nch) * kYsynCh;
    cp_async_wait_all();
    __syncthreads();
    // B = Gh rows (ol, k2, pout), K = (k1, pin), from the staged g of the chunk
    for (int t = tid; t < (kYsynN / 2) * (kKS / 8); t += blockDim.x) {
      const int m = t % (kYsynN / 2), kc = t / (kYsynN / 2);
      const int ol = m / kModes, k2 = m % kModes, o = oc + ol;
      float vr[8], vi[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k1 = kc * 4 + q;
        float2 gg = make_float2(0.f, 0.f);
        if (o < w && k1 < kModes) gg = gs[(k1 * kModes + k2) * kYsynCh + ol];
        vr[2 * q] = gg.x;  vr[2 * q + 1] = gg.y;
        vi[2 * q] = gg.y;  vi[2 * q + 1] = -gg.x;
      }
      const uint32_t offr = tc::kmajor_off(2 * m, kc * 8, SBO, 128), offi = tc::kmajor_off(2 * m + 1, kc * 8, SBO, 128);
      store_split8(sm + L.B + offr, sm + L.B + b_half + offr, vr);
      store_split8(sm + L.B + offi, sm + L.B + b_half + offi, vi);
    }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    {
      const int itn = next_item(it + gridDim.x);       // staging buffer is free again
      if (itn < nitems) prefetch(itn);
    }
    if (tid == 0) {
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < kKS / 16; ++s)
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t aa = base + L.A + (p == 2 ? a_half : 0u) + 256u * s, bb = base + L.B + (p == 1 ? b_half : 0u) + 256u * s;
          tc::mma_bf16(tmem, tc::make_sdesc(aa, 128, SBO), tc::make_sdesc(bb, 128, SBO), id, acc);
          acc = 1;
        }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], ph);
    tc::fence_after_sync();
    // epilogue: lane = row i -> G blob of tile (b, i / R), row Lr = (i % R, o), 16-byte hi/lo chunks of k'
    const int i = warp * 32 + lane;
    const uint32_t gh = geo.g_half(), gsb = geo.g_sbo();
    unsigned char* gt = Gb + ((size_t)b * geo.tiles_per_sys + (i < n ? i / geo.R : 0)) * 2 * gh;
    for (int ol = 0; ol < kYsynCh; ++ol) {
      const int o = oc + ol;
      const uint32_t Lr = (uint32_t)(o * geo.R + (i % geo.R));   // lane = (o, r)
#pragma unroll
      for (int c = 0; c < 2 * kModes; c += 8) {
        uint32_t u[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + ol * 2 * kModes + c, u);
        tc::tmem_wait_ld();
        if (i < n && o < w) {
          float v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = __uint_as_float(u[q]);
          uint4 h, l;
          tc::split8(v, h, l);
          const uint32_t off = tc::kmajor_off(Lr, c, gsb, 128);
          *reinterpret_cast<uint4*>(gt + off) = h;
          *reinterpret_cast<uint4*>(gt + gh + off) = l;
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    ph ^= 1;
  }
  tc::fence_after_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

constexpr int kYanN = kKS;                 // (k1, re|im) = 40 padded to 48

// persistent over work items (system, 128-row m tile)
__global__ void __launch_bounds__(128, 2) k_yan_tc(const unsigned char* __restrict__ Tb, const unsigned char* __restrict__ cst,
                                                   float2* __restrict__ chat, int n, int w, int B, const int* status) {
  const TcGeom geo(n, w);
  const TcConst C(geo);
  extern __shared__ __align__(1024) unsigned char sm[];
  const int K = 2 * n;
  const uint32_t SBO_A = geo.t_sbo(), LBO_A = geo.t_lbo(), SBO_B = (K / 8) * 128, th = geo.t_half(), bh = C.ap_half;
  const uint32_t A0 = 0, B0 = (2 * th + 1023) & ~1023u, BAR = (B0 + 2 * bh + 1023) & ~1023u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR);     // [0] tile load, [1] MMA, [2] constants
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + BAR + 32);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = w * kModes, nitems = B * geo.mtiles;
  auto next_item = [&](int it) {
    while (it < nitems && status && status[it / geo.mtiles] != SYS_RUNNING) it += gridDim.x;
    return it;
  };
  auto prefetch = [&](int it) {
    tc::mbar_expect_tx(&bar[0], 2 * th);
    tc::bulk_g2s(sm + A0, Tb + (size_t)it * 2 * th, 2 * th, &bar[0]);
  };
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&bar[2], 2 * bh);
    tc::bulk_g2s(sm + B0, cst + C.AP, 2 * bh, &bar[2]);
  }
  pdl_wait();
  pdl_trigger();
  int it = next_item(blockIdx.x);
  if (tid == 0 && it < nitems) prefetch(it);
  if (warp == 0) tc::tmem_alloc(tptr, 64);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t id = tc::make_idesc_bf16(128, kYanN, true, false);   // A (T) MN-major
  const uint32_t base = tc::smem_u32(sm);
  if (tid == 0) tc::mbar_wait(&bar[2], 0);
  uint32_t ph = 0;
  for (; it < nitems; it = next_item(it + gridDim.x)) {
    const int b = it / geo.mtiles, m0 = (it % geo.mtiles) * 128;
    if (tid == 0) {
      tc::mbar_wait(&bar[0], ph);
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < K / 16; ++s)
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t aa = base + A0 + (p == 2 ? th : 0u) + 2u * LBO_A * s, bb = base + B0 + (p == 1 ? bh : 0u) + 256u * s;
          tc::mma_bf16(tmem, tc::make_sdesc(aa, LBO_A, SBO_A), tc::make_sdesc(bb, 128, SBO_B), id, acc);
          acc = 1;
        }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], ph);
    tc::fence_after_sync();
    if (tid == 0) {                                   // A consumed: prefetch the next tile
      const int itn = next_item(it + gridDim.x);
      if (itn < nitems) prefetch(itn);
    }
    {
      const int m = m0 + warp * 32 + lane;
      const int k2 = m / w, o = m - k2 * w;          // T rows ordered (kappa2, o): stores coalesce over o
#pragma unroll
      for (int c = 0; c < 2 * kModes; c += 8) {
        uint32_t u[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, u);
        tc::tmem_wait_ld();
        if (m < M) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k1 = c / 2 + q;
            chat[((size_t)(k1 * kModes + k2) * B + b) * w + o] = make_float2(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]));
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    ph ^= 1;
  }
  tc::fence_after_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

// ------------------------------------------------------------------ mode-diagonal mixing on tensor cores
// per mode kappa: G[b][(o, re|im)] = sum_{(c, re|im)} C[b][(c, re|im)] * R'[(c, re|im)][(o, re|im)] / n^2,
// R' the 2x2-real form of R[c][o](kappa) (prebuilt per mode); M = systems (<= 128 per item).
struct MixSmem {
  uint32_t A, B, bar, tptr, total;
  __host__ __device__ MixSmem(int KM, int NM) {
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    A = take(2u * 128 * KM * 2);
    B = take(2u * NM * KM * 2);
    bar = take(64);
    tptr = bar + 32;
    total = o;
  }
};

// Mode-diagonal mixing, one work item = (mode kappa, 64 systems).  The complex product
// g[b][o] = sum_c c[b][c] R[c][o] runs as one real GEMM with two A rows per system,
//   row 2b   = (cr, -ci) per channel  ->  D = sum_c cr Rr - ci Ri = gr
//   row 2b+1 = (ci,  cr) per channel  ->  D = sum_c ci Rr + cr Ri = gi
// against B = (Rr, Ri) per channel (k_tc_prep), so the weight blob and N are not doubled.
constexpr int kMixSys = 64;   // systems per work item (2 A rows each)

__global__ void __launch_bounds__(128) k_mix_tc(const float2* __restrict__ chat, const unsigned char* __restrict__ cst,
                                               float2* __restrict__ ghat, int n, int w, int B, int mix, float inv_n2,
                                               const int* status) {
  const TcGeom geo(n, w);
  const TcConst C(geo);
  const int KM = C.KM, NM = C.NM[mix], cout = mix < 2 ? w : 1;
  const MixSmem L(KM, NM);
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t SBO = (KM / 8) * 128, a_half = 128u * KM * 2, b_half = C.mx_half[mix];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0] B load, [1] MMA
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbc = (B + kMixSys - 1) / kMixSys, nitems = kModes2 * nbc;
  auto prefetch = [&](int it) {
    const int kk = it / nbc;
    tc::mbar_expect_tx(&bar[0], 2 * b_half);
    tc::bulk_g2s(sm + L.B, cst + C.MX[mix] + (size_t)kk * 2 * b_half, 2 * b_half, &bar[0]);
  };
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
    if ((int)blockIdx.x < nitems) prefetch(blockIdx.x);   // weights do not depend on the predecessor
  }
  const uint32_t ncols = NM <= 32 ? 32u : (NM <= 64 ? 64u : 128u);
  if (warp == 0) tc::tmem_alloc(tptr, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t id = tc::make_idesc_bf16(128, NM, false, false);
  const uint32_t base = tc::smem_u32(sm);
  pdl_wait();
  pdl_trigger();
  uint32_t ph = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int kk = it / nbc, b0 = (it % nbc) * kMixSys, nb = min(kMixSys, B - b0);
    // A: rows (b, re|im), K = (c, re|im); all loads of a batch first
    {
      constexpr int kBatch = 8;
      const int ntask = kMixSys * (KM / 8);
      for (int t0 = tid; t0 < ntask; t0 += kBatch * blockDim.x) {
        float2 x[kBatch][4];
#pragma unroll
        for (int z = 0; z < kBatch; ++z) {
          const int t = t0 + z * blockDim.x, bl = t % kMixSys, kc = t / kMixSys;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = kc * 4 + q;
            x[z][q] = (t < ntask && bl < nb && c < w) ? __ldg(chat + ((size_t)kk * B + b0 + bl) * w + c)
                                                      : make_float2(0.f, 0.f);
          }
        }
#pragma unroll
        for (int z = 0; z < kBatch; ++z) {
          const int t = t0 + z * blockDim.x, bl = t % kMixSys, kc = t / kMixSys;
          if (t >= ntask) break;
          float vr[8], vi[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            vr[2 * q] = x[z][q].x;  vr[2 * q + 1] = -x[z][q].y;
            vi[2 * q] = x[z][q].y;  vi[2 * q + 1] = x[z][q].x;
          }
          const uint32_t offr = tc::kmajor_off(2 * bl, kc * 8, SBO, 128), offi = tc::kmajor_off(2 * bl + 1, kc * 8, SBO, 128);
          store_split8(sm + L.A + offr, sm + L.A + a_half + offr, vr);
          store_split8(sm + L.A + offi, sm + L.A + a_half + offi, vi);
        }
      }
    }
    tc::fence_proxy_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::mbar_wait(&bar[0], ph);
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < KM / 16; ++s)
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t aa = base + L.A + (p == 2 ? a_half : 0u) + 256u * s, bb = base + L.B + (p == 1 ? b_half : 0u) + 256u * s;
          tc::mma_bf16(tmem, tc::make_sdesc(aa, 128, SBO), tc::make_sdesc(bb, 128, SBO), id, acc);
          acc = 1;
        }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], ph);
    tc::fence_after_sync();
    if (tid == 0 && it + (int)gridDim.x < nitems) prefetch(it + gridDim.x);   // B consumed
    {
      // lane pair (2bl, 2bl+1) holds (gr, gi) of system bl: swap halves of each 8-column chunk so the
      // even lane writes o in [c0, c0+4) and the odd lane o in [c0+4, c0+8) as float2 runs
      const int row = warp * 32 + lane, bl = row >> 1, p = row & 1, b = b0 + bl;
      const bool ok = bl < nb && (!status || status[b] == SYS_RUNNING);
      for (int c0 = 0; c0 < cout; c0 += 8) {
        uint32_t u[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, u);
        tc::tmem_wait_ld();
        float mine[4], other[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float keep = __uint_as_float(u[p ? 4 + q : q]);      // my half
          const float give = __uint_as_float(u[p ? q : 4 + q]);      // partner's half
          mine[q] = keep;
          other[q] = __shfl_xor_sync(0xffffffffu, give, 1);
        }
        if (ok) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int o = c0 + 4 * p + q;
            if (o < cout) {
              const float gr = p ? other[q] : mine[q], gi = p ? mine[q] : other[q];
              ghat[((size_t)kk * B + b) * cout + o] = make_float2(gr * inv_n2, gi * inv_n2);
            }
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    ph ^= 1;
  }
  tc::fence_after_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

static size_t ysyn_tc_smem() { return YsynSmem().total; }
static size_t yan_tc_smem(int n) {
  const TcGeom g(n, 1);
  const uint32_t th = g.t_half(), bh = (uint32_t)kKS * (2 * n) * 2;
  return (((2 * th + 1023) & ~1023u) + 2 * bh + 1023 & ~1023u) + 64;
}

// ------------------------------------------------------------------ host side
static int optin_bytes() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 0;
  }
  return v;
}

bool tc_layer_supported(int n, int w) {
  if (w > 128 || w < 1 || n % 16 != 0 || n < 64 || n > 128) return false;
  const TcGeom g(n, w);
  if (n % g.R) return false;
  const int optin = optin_bytes();
  return TcSmem(g, w).total <= (uint32_t)optin && yan_tc_smem(n) <= (size_t)optin;
}

static int num_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  }
  return v;
}

template <int WP>
static cudaError_t prep_tc() {
  const void* fns[4] = {(const void*)k_tc_layer<WP, true>, (const void*)k_tc_layer<WP, false>,
                        (const void*)k_tc_layer_ws<WP, true>, (const void*)k_tc_layer_ws<WP, false>};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// FCGNO_TC_WS=1 selects the pipelined two-group layer kernel (k_tc_layer_ws).  Default: k_tc_layer
// with two CTAs per SM, measured faster on B200.
static bool ws_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FCGNO_TC_WS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

cudaError_t prepare_tc_kernels() {
  static bool done = false;
  if (done) return cudaSuccess;
  cudaError_t e;
  if ((e = prep_tc<32>()) != cudaSuccess) return e;
  if ((e = prep_tc<64>()) != cudaSuccess) return e;
  if ((e = prep_tc<128>()) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute((const void*)k_ysyn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute((const void*)k_yan_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute((const void*)k_mix_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess) return e;
  done = true;
  return cudaSuccess;
}

cudaError_t launch_tc_layer(const TcLayerArgsHost& h, cudaStream_t s) {
  TcLayerArgs a{};
  a.n = h.n; a.w = h.w; a.cin = h.cin; a.B = h.B; a.use_gelu = h.use_gelu; a.layer = h.layer;
  a.r = h.r; a.rr = h.rr; a.k = h.k; a.vin = h.vin; a.W = h.W; a.bias = h.bias; a.G = h.G; a.cst = h.cst;
  a.vout = h.vout; a.T = h.T; a.dw = h.dw; a.pout = h.pout; a.status = h.status;
  const TcGeom g(h.n, h.w);
  const int ntiles = h.B * g.tiles_per_sys;
  if (ws_enabled()) {
    int stages = kWsStages;
    while (stages > 1 && TcWsSmem(g, h.cin, stages).total > (uint32_t)optin_bytes()) --stages;
    const size_t wsmem = TcWsSmem(g, h.cin, stages).total;
    if (wsmem <= (size_t)optin_bytes() && ws_tmem_fits(g, TcWsSmem(g, h.cin, stages).KB) &&
        (ntiles + num_sms() - 1) / num_sms() <= kWsMaxTiles) {
      const int grid = std::min(ntiles, num_sms());
      if (g.WP == 32) {
        if (h.first) launch_k(k_tc_layer_ws<32, true>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
        else launch_k(k_tc_layer_ws<32, false>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
      } else if (g.WP == 64) {
        if (h.first) launch_k(k_tc_layer_ws<64, true>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
        else launch_k(k_tc_layer_ws<64, false>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
      } else {
        if (h.first) launch_k(k_tc_layer_ws<128, true>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
        else launch_k(k_tc_layer_ws<128, false>, dim3(grid), dim3(kWsThreads), wsmem, s, a, stages);
      }
      return cudaGetLastError();
    }
  }
  const size_t smem = TcSmem(g, h.cin).total;
  // persistent grid: as many CTAs as fit per SM by shared memory (<= 2) and TMEM columns
  const uint32_t need_cols = 2u * h.n + (uint32_t)TcSmem(g, h.cin).KB;
  const int by_tmem = need_cols <= 256 ? 2 : 1;
  const int by_smem = (int)((228u * 1024u) / (smem + 1024u));
  const int per_sm = std::max(1, std::min(by_tmem, std::min(by_smem, 2)));
  const int grid = std::min(ntiles, per_sm * num_sms());
  if (g.WP == 32) {
    if (h.first) launch_k(k_tc_layer<32, true>, dim3(grid), dim3(kTcThreads), smem, s, a);
    else launch_k(k_tc_layer<32, false>, dim3(grid), dim3(kTcThreads), smem, s, a);
  } else if (g.WP == 64) {
    if (h.first) launch_k(k_tc_layer<64, true>, dim3(grid), dim3(kTcThreads), smem, s, a);
    else launch_k(k_tc_layer<64, false>, dim3(grid), dim3(kTcThreads), smem, s, a);
  } else {
    if (h.first) launch_k(k_tc_layer<128, true>, dim3(grid), dim3(kTcThreads), smem, s, a);
    else launch_k(k_tc_layer<128, false>, dim3(grid), dim3(kTcThreads), smem, s, a);
  }
  return cudaGetLastError();
}

cudaError_t launch_ysyn(const float* ghat, const unsigned char* cst, unsigned char* Gb, int n, int w, int B,
                        const int* status, cudaStream_t s) {
  const int items = B * ((w + kYsynCh - 1) / kYsynCh);
  const int grid = std::min(items, 2 * num_sms());
  launch_k(k_ysyn_tc, dim3(grid), dim3(128), ysyn_tc_smem(), s, reinterpret_cast<const float2*>(ghat), cst, Gb, n, w, B,
           status);
  return cudaGetLastError();
}

cudaError_t launch_yan(const unsigned char* Tb, const unsigned char* cst, float* chat, int n, int w, int B,
                       const int* status, cudaStream_t s) {
  const TcGeom g(n, w);
  const int items = B * g.mtiles;
  const int per_sm = yan_tc_smem(n) <= 110 * 1024 ? 2 : 1;
  const int grid = std::min(items, per_sm * num_sms());
  launch_k(k_yan_tc, dim3(grid), dim3(128), yan_tc_smem(n), s, Tb, cst, reinterpret_cast<float2*>(chat), n, w, B, status);
  return cudaGetLastError();
}

size_t tc_const_bytes(int n, int w) { return TcConst(TcGeom(n, w)).total; }

static int mix_per_sm() {   // FCGNO_MIX_PER_SM (A/B experiments); default 3 (smem allows 3, measured best)
  static int v = -1;
  if (v < 0) { const char* e = getenv("FCGNO_MIX_PER_SM"); v = e ? std::max(1, atoi(e)) : 3; }
  return v;
}

cudaError_t launch_mix_tc(int mix, const float* chat, const unsigned char* cst, float* ghat, int n, int w, int B,
                          float inv_n2, const int* status, cudaStream_t s) {
  const TcGeom g(n, w);
  const TcConst C(g);
  const size_t smem = MixSmem(C.KM, C.NM[mix]).total;
  const int nitems = kModes2 * ((B + kMixSys - 1) / kMixSys);
  const int per_sm = std::max(1, std::min(mix_per_sm(), (int)((228u * 1024u) / (smem + 1024u))));
  const int grid = std::min(nitems, per_sm * num_sms());
  return launch_k(k_mix_tc, dim3(grid), dim3(128), smem, s, reinterpret_cast<const float2*>(chat), cst,
                  reinterpret_cast<float2*>(ghat), n, w, B, mix, inv_n2, status);
}

cudaError_t launch_tc_prep(int n, int w, const float* W1, const float* W2, const float* W3, const float* R2,
                           const float* R3, const float* Q, const float* F, unsigned char* out, cudaStream_t s) {
  TcPrepArgs a{};
  a.n = n; a.w = w; a.W[0] = W1; a.W[1] = W2; a.W[2] = W3; a.F = reinterpret_cast<const float2*>(F); a.out = out;
  a.Rm[0] = reinterpret_cast<const float2*>(R2); a.Rm[1] = reinterpret_cast<const float2*>(R3);
  a.Rm[2] = reinterpret_cast<const float2*>(Q);
  k_tc_prep<<<2 * num_sms(), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace fcgno

// no_px_kernels.cu — pixel-major tensor-core (tcgen05 / TMEM) SNO layers for the fp32 NO path,
// n = 64 or n a multiple of 128 up to 512 (BASELINE configs 2-5).
//
// One layer (§2.4.2, R7-R11), per system:
//   u[i][j][o] = sum_c W[o][c] v[i][j][c] + b[o] + n^-2 Re sum_kappa g[o](kappa) e^{+2 pi i kappa.(i,j)/n}
//   v'         = GELU(u)                               (layers 1-3; layer 4 is folded away)
//   c'[o](k)   = sum_{i,j} v'[i][j][o] e^{-2 pi i k.(i,j)/n}
// with the DFTs separable, so that every contraction is a dense GEMM on the tensor cores:
//   k_px_ysyn   per (system, 128 rows, kappa2 group):  G[i][(q,o)] = Fp[i][(k1,p)] . Gh_kappa2[(k1,p)][(q,o)]
//   k_px_layer  per tile of 128 pixels (M = pixels, N = channels):
//                 D1[p][o]  = sum_c V[p][c] W[o][c]                 bypass        (layers 2, 3)
//                           + sum_k' F[p][k'] G_row(p)[k'][o]       x-synthesis
//                 epilogue  v' = GELU(D1 + b (+ layer 1's 2-channel lift bypass on the CUDA cores))
//                           -> the tile in shared memory, bulk-stored as the next layer's V blob
//                           (layer 3: sum_o (D W4)[o] v'[o] per pixel instead)
//                 D2[o][k'] = sum_p v'[p][o] F[p][k']               x-analysis (the same smem tile read
//                           MN-major; n >= 256: accumulated over the row's column blocks)
//                 epilogue  -> T rows (fp32)
//   k_px_yan    per (system, 128 (kappa2, o, re|im) rows): C[(k2,o,p)][(k1,x|y)] = sum_i T[i][..] F[i][(k1,x|y)],
//               complex recombination of lane pairs in the epilogue -> c'[kappa][b][o]
// Precision: 3xBF16 split (hi*hi + hi*lo + lo*hi, fp32 accumulation), ~1e-5 relative L2 for the NO.
//
// k_px_layer is warp-specialised, one CTA per SM over its tiles: warp 0 issues the bulk loads (V
// tile or layer 1's fp64 r/k; G rows by TMA tensor copy) into a 2-stage ring; warp 1 issues the MMAs
// (D1 of tile t into one of two TMEM accumulators, then the x-analysis of tile t-1); warps 3-14 run
// epilogue 1 (three warpgroups splitting the channel columns, thread = pixel) and write v' in place
// into the stage the tile arrived in; warp 2 bulk-stores it and releases the stage; warps 15-18 run
// epilogue 2 (thread = channel) into T.
#include <algorithm>

#include <cuda.h>

#include "internal.h"
#include "px_layout.cuh"
#include "tc_common.cuh"

namespace fcgno {

namespace {

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
// packed fp32 pairs (FFMA2 / FMUL2 / FADD2 on sm_100a: one issue slot for two lanes of arithmetic)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// GELU(x) = x/2 (1 + erf(x / sqrt 2)) (reading R11) of two values, erf by Abramowitz & Stegun 7.1.26
// (|error| <= 1.5e-7, two orders below the 3xBF16 operand rounding) through erfc: with h = x/2 and
// pe = poly(t) exp(-x^2/2), t = 1/(1 + p|x|/sqrt 2),  GELU = h + |h| - |h| pe  (x >= 0: h (2 - pe);
// x < 0: h pe, the sum h + |h| being exactly 0).  Branch-free; the polynomial, the squares and the
// scalings run as packed pairs, the two MUFU operations (rcp, ex2) per value as scalars.
__device__ __forceinline__ void gelu_px2(float& x0, float& x1) {
  const float t0 = rcp_approx(fmaf(0.3275911f * 0.70710678118654752f, fabsf(x0), 1.0f));
  const float t1 = rcp_approx(fmaf(0.3275911f * 0.70710678118654752f, fabsf(x1), 1.0f));
  const uint64_t X = pk2(x0, x1), T = pk2(t0, t1);
  uint64_t P = fma2(pk2(1.061405429f, 1.061405429f), T, pk2(-1.453152027f, -1.453152027f));
  P = fma2(P, T, pk2(1.421413741f, 1.421413741f));
  P = fma2(P, T, pk2(-0.284496736f, -0.284496736f));
  P = fma2(P, T, pk2(0.254829592f, 0.254829592f));
  P = mul2(P, T);
  const uint64_t Z = mul2(mul2(X, X), pk2(-0.72134752044448170f, -0.72134752044448170f));
  float z0, z1;
  upk2(Z, z0, z1);
  const uint64_t PE = mul2(P, pk2(ex2_approx(z0), ex2_approx(z1)));
  const uint64_t H = mul2(X, pk2(0.5f, 0.5f));
  float h0, h1, pe0, pe1;
  upk2(H, h0, h1);
  upk2(PE, pe0, pe1);
  x0 = fmaf(-fabsf(h0), pe0, h0 + fabsf(h0));
  x1 = fmaf(-fabsf(h1), pe1, h1 + fabsf(h1));
}

__device__ __forceinline__ void st_split8(unsigned char* hi, unsigned char* lo, const float* v) {
  uint4 h, l;
  tc::split8(v, h, l);
  *reinterpret_cast<uint4*>(hi) = h;
  *reinterpret_cast<uint4*>(lo) = l;
}

__device__ __forceinline__ void store_split8(unsigned char* hi, unsigned char* lo, const float (&v)[8]) {
  st_split8(hi, lo, v);
}
using tc::tmem_ld8;

// 256-bit read-only global load (sm_100: LDG.256), 32-byte aligned
__device__ __forceinline__ void ld_global_256(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}
// 256-bit global store (sm_100: STG.256), 32-byte aligned
__device__ __forceinline__ void st_global_256(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

__host__ __device__ inline uint32_t pow2_cols(uint32_t c) { return c <= 32 ? 32u : c <= 64 ? 64u : c <= 128 ? 128u : c <= 256 ? 256u : 512u; }

}  // namespace

// ------------------------------------------------------------------ constant blobs
struct PxPrepArgs {
  int n, w;
  const float* W[2];      // layers 2, 3: [w][w]
  const float2* Rm[3];    // mixing weights [400][w][cout]
  const float2* F;        // [n][20] exp(-2 pi i kappa j / n)
  unsigned char* out;
};

__global__ void __launch_bounds__(256) k_px_prep(const PxPrepArgs a) {
  const PxGeom g(a.n, a.w);
  const PxConst C(g);
  const int n = a.n, w = a.w;
  const int nF = g.nF * 128 * 5, nW = 2 * g.NP * g.KCG, nFP = g.nMT * 128 * 6, nFY = 48 * (n / 8);
  int nMX[3], tot = nF + nW + nFP + nFY;
  for (int l = 0; l < 3; ++l) { nMX[l] = kModes2 * C.NM[l] * (C.KM / 8); tot += nMX[l]; }
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
    float v[8];
    unsigned char* dst;
    uint32_t half, off;
    int u = t;
    if (u < nF) {                                  // F[f][k'/8][p/8][p%8][k'%8] (k' < 40)
      const int f = u / (128 * 5), rem = u % (128 * 5), p = rem % 128, kg = rem / 128;
      const int j = n < 128 ? p % n : f * 128 + p;
      const int row = n < 128 ? p / n : 0;
      const bool keep = n >= 128 || f == 0 || (f == 1 && row == 0) || (f == 2 && row == 1);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int kp = kg * 8 + q;
        v[q] = 0.f;
        if (keep && kp < 2 * kModes) { const float2 z = a.F[(size_t)j * kModes + (kp >> 1)]; v[q] = (kp & 1) ? z.y : z.x; }
      }
      dst = a.out + C.F + (size_t)f * 2 * C.f_half; half = C.f_half;
      off = (uint32_t)kg * 2048u + (uint32_t)(p >> 3) * 128u + (uint32_t)(p & 7) * 16u;
    } else if ((u -= nF) < nW) {                   // W[l][o][c] K-major B (N = o, K = c)
      const int l = u / (g.NP * g.KCG), rem = u % (g.NP * g.KCG), o = rem % g.NP, cg = rem / g.NP;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = cg * 8 + q;
        v[q] = (o < w && c < w) ? a.W[l][(size_t)o * w + c] : 0.f;
      }
      dst = a.out + C.W[l]; half = C.w_half;
      off = (uint32_t)(o >> 3) * (uint32_t)(g.KCG * 128) + (uint32_t)cg * 128u + (uint32_t)(o & 7) * 16u;
    } else if ((u -= nW) < nFP) {                  // Fp[mt][i][(k1, p)] K-major (M = i, K = 48)
      const int mt = u / (128 * 6), rem = u % (128 * 6), i = rem % 128, kg = rem / 128, row = mt * 128 + i;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = kg * 8 + q, k1 = k >> 1;
        v[q] = 0.f;
        if (row < n && k1 < kModes) { const float2 z = a.F[(size_t)row * kModes + k1]; v[q] = (k & 1) ? z.y : z.x; }
      }
      dst = a.out + C.FP + (size_t)mt * 2 * C.fp_half; half = C.fp_half;
      off = (uint32_t)(i >> 3) * 768u + (uint32_t)kg * 128u + (uint32_t)(i & 7) * 16u;
    } else if ((u -= nFP) < nFY) {                 // Fy[i][(k1, x|y)] K-major B (N = 48, K = i)
      const int nn = u % 48, ig = u / 48, k1 = nn >> 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = ig * 8 + q;
        v[q] = 0.f;
        if (k1 < kModes) { const float2 z = a.F[(size_t)i * kModes + k1]; v[q] = (nn & 1) ? z.y : z.x; }
      }
      dst = a.out + C.FY; half = C.fy_half;
      off = (uint32_t)(nn >> 3) * (uint32_t)((n / 8) * 128) + (uint32_t)ig * 128u + (uint32_t)(nn & 7) * 16u;
    } else {                                       // mode-mixing B: row o, K = (c, re|im) = (Rr, Ri)
      u -= nFY;
      int l = 0;
      while (u >= nMX[l]) { u -= nMX[l]; ++l; }
      const int cout = l < 2 ? w : 1, NM = C.NM[l], KM = C.KM;
      const int per_mode = NM * (KM / 8), kk = u / per_mode, rem = u % per_mode, nn = rem % NM, kc = rem / NM;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = kc * 4 + q;
        float rr = 0.f, ri = 0.f;
        if (c < w && nn < cout) { const float2 R2 = a.Rm[l][((size_t)kk * w + c) * cout + nn]; rr = R2.x; ri = R2.y; }
        v[2 * q] = rr;
        v[2 * q + 1] = ri;
      }
      dst = a.out + C.MX[l] + (size_t)kk * 2 * C.mx_half[l]; half = C.mx_half[l];
      off = (uint32_t)(nn >> 3) * (uint32_t)((KM / 8) * 128) + (uint32_t)kc * 128u + (uint32_t)(nn & 7) * 16u;
    }
    uint4 h, lo;
    tc::split8(v, h, lo);
    *reinterpret_cast<uint4*>(dst + off) = h;
    *reinterpret_cast<uint4*>(dst + half + off) = lo;
  }
}

// ------------------------------------------------------------------ k_px_layer
// Diagnostics (FCGNO_PX_TRACE=<layer 1..3>): clock64 stamps of the pipeline events of CTA 0's first
// kPxTraceTiles tiles, read back with fcgno_debug_px_trace (scripts/px_trace.py).
constexpr int kPxTraceTiles = 64, kPxTraceEv = 34;   // 10 pipeline events + (start, done) of the 12 epilogue-1 warps
__device__ unsigned long long g_px_trace[kPxTraceTiles * kPxTraceEv];
#define PX_TRACE(t, ev)                                                                  \
  do {                                                                                   \
    if (a.trace && blockIdx.x == 0 && (t) < kPxTraceTiles)                               \
      g_px_trace[(t) * kPxTraceEv + (ev)] = clock64();                                   \
  } while (0)
constexpr int kPxE1Groups = 3;                                 // epilogue-1 warpgroups (column split)
constexpr int kPxE1Warps = 4 * kPxE1Groups;
// warp roles: 0 V loads, 1 D1 MMAs, 2 G loads, 3 x-analysis MMAs, 4-15 epilogue 1, 16-19 epilogue 2
constexpr int kPxE1First = 4, kPxE2First = kPxE1First + kPxE1Warps;
constexpr int kPxThreads = (kPxE2First + 4) * 32;
constexpr int kPxMaxSys = 4096;
constexpr uint32_t kPxSmemLimit = 227u * 1024u;

// Shared-memory plan: NST V stages (the tile's v' is written back in place) and GST G stages, 3 each
// when they fit the 227 KB opt-in limit, else 2.  Padding channel group CGS (w odd-eighths) and G's
// k-group 5 (k' 40..47) are read from one shared zero block (per-step descriptor LBO), not stored.
struct PxSmem {
  uint32_t ST, GS, RK, WB, FB, ZB, misc, bias, w1e, dw, bar, tptr, runb, pj, total, stage_bytes, gs_bytes;
  int NST, GST;
  __host__ __device__ PxSmem(const PxGeom& g, bool first, bool proj) {
    stage_bytes = 2u * g.stage_half();
    gs_bytes = (uint32_t)g.RT * 10u * (uint32_t)g.LBO_G;   // per stage: RT rows x [hi 5 k-groups | lo 5]
    for (NST = 3; NST >= 2; --NST) {
      for (GST = 3; GST >= 2; --GST) {
        plan(g, first, proj);
        if (total <= kPxSmemLimit) return;
      }
    }
    NST = GST = 2;
    plan(g, first, proj);
  }
  __host__ __device__ void plan(const PxGeom& g, bool first, bool proj) {
    uint32_t o = 0;
    auto take = [&](uint32_t bytes, uint32_t al) { const uint32_t at = (o + al - 1) & ~(al - 1); o = at + bytes; return at; };
    ST = take((uint32_t)NST * stage_bytes, 1024);
    GS = take((uint32_t)GST * gs_bytes, 1024);
    RK = first ? take((uint32_t)NST * 2048u, 128) : 0u;
    WB = first ? 0u : take(2u * (uint32_t)g.NP * g.NP * 2u, 1024);
    FB = take((uint32_t)g.nF * 2u * 5u * 2048u, 1024);
    ZB = take(2048, 1024);                     // zero block (after every descriptor start: LBO > 0)
    bias = take(128 * 4, 16);
    w1e = first ? take(256 * 4, 16) : 0u;
    dw = proj ? take(128 * 4, 16) : 0u;
    bar = take(256, 16);
    tptr = bar + 248;
    runb = take(kPxMaxSys / 8, 16);
    pj = proj ? take(2u * kPxE1Groups * 128u * 4u, 16) : 0u;   // layer 3: per-group projection partials
    total = (o + 15) & ~15u;
    // the x-analysis reads its A (a stage tile, MN-major, M = 128 channels) over 16 channel groups:
    // rows o >= NP read whatever follows (their results are ignored), which must lie inside the smem
    const uint32_t reach = ST + (uint32_t)(NST - 1) * stage_bytes + g.stage_half() + 16u * 2048u;
    if (reach > total) total = reach;
  }
};

struct PxLayerArgs {
  int n, w, B, layer, use_gelu;
  const double* r; const double* rr; const double* k;   // layer 1 inputs (fp64; rr = 1/||r|| per system)
  const unsigned char* vin;                              // V blobs (layers 2, 3)
  unsigned char* vout;                                   // V blobs of the next layer (layers 1, 2)
  const unsigned char* G;                                // G (interleaved rows; read by TMA through gmap)
  float* T;                                              // T rows
  const unsigned char* cst;                              // PxConst
  const float* bias;                                     // [w]
  const float* w1e;                                      // layer 1: lift folded into W1, [w][2]
  const float* dw;                                       // layer 3: projection (D W4) [w]
  float* p3;                                             // layer 3: sum_o dw[o] v3[o] per pixel [B][n][n]
  const int* status;
  int trace;                                             // diagnostics: record g_px_trace
};

// Pipeline (per CTA, tiles t of its row units in order; s = t % NST, gs = t % GST, d = t % 2):
//   warp 0  V loads     wait empty[s]   -> bulk-copy V(t) (layer 1: fp64 r, k) into stage s  -> full[s]
//   warp 2  G loads     wait gempty[gs] -> TMA-gather the tile's G row(s) into G stage gs    -> gfull[gs]
//   warp 1  D1 MMAs     D1(t) = bypass + x-synthesis into TMEM buffer d once full[s], gfull[gs] and
//                       d1empty[d] allow (commit -> d1full[d], gempty[gs])
//   warps 4-15 E1       v' = GELU(D1 + b) -> smem stage s in place (A of the x-analysis) and HBM (next
//                       layer's V, 16-byte coalesced stores); layer 3: the projection sum instead of HBM
//                       (-> d1empty[d], vfull[s])
//   warp 3  D2 MMAs     D2 += x-analysis of tile t once vfull[s] (commit -> empty[s]; last column block
//                       of the row -> d2full); a second MMA issuer, so the stage is released without
//                       waiting behind the next tile's D1 instructions
//   warps 16-19 E2      D2 -> T rows (fp32, coalesced over o)
template <bool FIRST, bool PROJ>
__global__ void __launch_bounds__(kPxThreads, 1) k_px_layer(const PxLayerArgs a, const __grid_constant__ CUtensorMap gmap) {
  const PxGeom g(a.n, a.w);
  const PxConst C(g);
  const PxSmem L(g, FIRST, PROJ);
  const int NST = L.NST, GST = L.GST;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = n * n, w = a.w, NP = g.NP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bar);
  uint64_t *full = bars, *empty = bars + 3, *vfull = bars + 6, *gfull = bars + 9, *gempty = bars + 12,
           *d1full = bars + 15, *d1empty = bars + 17, *d2full = bars + 19, *d2empty = bars + 21, *cstb = bars + 23;
  constexpr int kNumBars = 24;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  float* sw1e = reinterpret_cast<float*>(sm + L.w1e);
  float* sdw = reinterpret_cast<float*>(sm + L.dw);
  uint32_t* runb = reinterpret_cast<uint32_t*>(sm + L.runb);
  const int nunits = a.B * g.units;
  const bool cached = a.status && a.B <= kPxMaxSys;
  const uint32_t ncols = pow2_cols(2u * NP + 2u * g.D2W);

  // ---- prologue (overlaps the predecessor's tail under programmatic dependent launch)
  if (tid == 0) {
    // d1empty, vfull: the epilogue-1 threads; d2empty: the 128 epilogue-2 threads; all others one
    // arrival (expect_tx or an MMA commit)
    for (int q = 0; q < kNumBars; ++q) {
      const bool e1 = (q >= 6 && q < 9) || (q >= 17 && q < 19), e2 = q >= 21 && q < 23;
      tc::mbar_init(&bars[q], e1 ? 32u * kPxE1Warps : e2 ? 128u : 1u);
    }
    tc::fence_mbar_init();
    const uint32_t fbytes = (uint32_t)g.nF * 2u * C.f_half;
    tc::mbar_expect_tx(cstb, fbytes + (FIRST ? 0u : 2u * C.w_half));
    tc::bulk_g2s(sm + L.FB, a.cst + C.F, fbytes, cstb);
    if (!FIRST) tc::bulk_g2s(sm + L.WB, a.cst + C.W[a.layer - 1], 2u * C.w_half, cstb);
  }
  {   // stages zeroed (layer-1 tiles are produced in place) and the zero block
    uint4* z = reinterpret_cast<uint4*>(sm + L.ST);
    for (uint32_t t = tid; t < ((uint32_t)NST * L.stage_bytes) / 16u; t += blockDim.x) z[t] = make_uint4(0, 0, 0, 0);
    z = reinterpret_cast<uint4*>(sm + L.ZB);
    for (uint32_t t = tid; t < 2048u / 16u; t += blockDim.x) z[t] = make_uint4(0, 0, 0, 0);
  }
  for (int o = tid; o < 128; o += blockDim.x) {
    sbias[o] = o < w ? a.bias[o] : 0.f;
    if (FIRST) { sw1e[2 * o] = o < w ? a.w1e[2 * o] : 0.f; sw1e[2 * o + 1] = o < w ? a.w1e[2 * o + 1] : 0.f; }
    if (PROJ) sdw[o] = o < w ? a.dw[o] : 0.f;
  }
  if (cached)
    for (int q = warp; q < (a.B + 31) / 32; q += blockDim.x / 32) {
      const int sb = q * 32 + lane;
      const unsigned bits = __ballot_sync(0xffffffffu, sb < a.B && __ldcg(a.status + sb) == SYS_RUNNING);
      if (lane == 0) runb[q] = bits;
    }
  if (warp == 0) tc::tmem_alloc(tptr, ncols);
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  pdl_wait();
  pdl_trigger();

  auto running = [&](int u) {
    const int b = u / g.units;
    if (!a.status) return true;
    if (cached) return ((runb[b >> 5] >> (b & 31)) & 1u) != 0;
    return __ldcg(a.status + b) == SYS_RUNNING;
  };
  auto next_unit = [&](int u) {
    while (u < nunits && !running(u)) u += gridDim.x;
    return u;
  };
  const uint32_t base = tc::smem_u32(sm);
  const uint32_t sth0 = base + L.ST, fb0 = base + L.FB, gs0 = base + L.GS, wb0 = base + L.WB, zb0 = base + L.ZB;
  const uint32_t sh = g.stage_half(), fh = C.f_half, LG = (uint32_t)g.LBO_G, KCG = (uint32_t)g.KCG;

  if (warp == 0 || warp == 2) {
    // ================= producers: V tiles (warp 0) and G rows (warp 2)
    if (lane == 0) {
      int t = 0;
      for (int u = next_unit(blockIdx.x); u < nunits; u = next_unit(u + gridDim.x)) {
        const int b = u / g.units, ul = u % g.units;
        for (int cb = 0; cb < g.CB; ++cb, ++t) {
          if (warp == 0) {
            const int s = t % NST;
            tc::mbar_wait(&empty[s], ((uint32_t)(t / NST) & 1u) ^ 1u);
            PX_TRACE(t, 0);
            const int tt = ul * g.CB + cb;
            unsigned char* st = sm + L.ST + (uint32_t)s * L.stage_bytes;
            if (FIRST) {
              const size_t e = (size_t)b * N + (size_t)tt * 128;
              tc::mbar_expect_tx(&full[s], 2048u);
              tc::bulk_g2s(sm + L.RK + s * 2048, a.r + e, 1024u, &full[s]);
              tc::bulk_g2s(sm + L.RK + s * 2048 + 1024, a.k + e, 1024u, &full[s]);
            } else {
              const unsigned char* src = a.vin + ((size_t)b * g.TPS + tt) * 2 * g.v_half();
              tc::mbar_expect_tx(&full[s], 2u * g.v_half());
              tc::bulk_g2s(st, src, g.v_half(), &full[s]);
              tc::bulk_g2s(st + g.stage_half(), src + g.v_half(), g.v_half(), &full[s]);
            }
          } else {
            const int gs = t % GST;
            tc::mbar_wait(&gempty[gs], ((uint32_t)(t / GST) & 1u) ^ 1u);
            tc::mbar_expect_tx(&gfull[gs], (uint32_t)g.RT * 2u * g.g_half());
            for (int r = 0; r < g.RT; ++r) {   // G row i: hi and lo boxes of the interleaved layout
              unsigned char* gdst = sm + L.GS + (uint32_t)gs * L.gs_bytes + (uint32_t)r * 10u * g.LBO_G;
              const int i = ul * g.RT + r;
              tc::tma_load_5d(gdst, &gmap, 0, i, 0, 0, 2 * b, &gfull[gs]);
              tc::tma_load_5d(gdst + 5u * g.LBO_G, &gmap, 0, i, 0, 0, 2 * b + 1, &gfull[gs]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= D1 MMAs (one thread): bypass + x-synthesis
    if (tc::elect_one()) {
      tc::mbar_wait(cstb, 0);
      const uint32_t id1 = tc::make_idesc_bf16(128, NP, false, false);   // V (K-major) . W (K-major)
      const uint32_t id2 = tc::make_idesc_bf16(128, NP, false, true);    // F (K-major) . G (MN-major)
      int t = 0;
      for (int u = next_unit(blockIdx.x); u < nunits; u = next_unit(u + gridDim.x)) {
        for (int cb = 0; cb < g.CB; ++cb, ++t) {
          const int s = t % NST, gs = t % GST, d = t & 1;
          tc::mbar_wait(&full[s], (uint32_t)(t / NST) & 1u);
          tc::mbar_wait(&gfull[gs], (uint32_t)(t / GST) & 1u);
          tc::mbar_wait(&d1empty[d], ((uint32_t)(t >> 1) & 1u) ^ 1u);
          PX_TRACE(t, 1);
          tc::fence_after_sync();
          const uint32_t d1 = tmem + (uint32_t)d * NP;
          const uint32_t sth = sth0 + (uint32_t)s * L.stage_bytes, stl = sth + sh;
          uint32_t acc = 0;
          if (!FIRST) {   // bypass: K = channels, 16 per step (an odd last group pairs with the zero block)
            for (uint32_t ks = 0; ks < KCG / 2; ++ks)
#pragma unroll
              for (int p = 0; p < 3; ++p) {
                const uint32_t aa = (p == 2 ? stl : sth) + ks * 4096u;
                const uint32_t lbo = (2 * ks + 1 < (uint32_t)g.CGS) ? 2048u : zb0 - aa;
                const uint32_t bb = wb0 + (p == 1 ? C.w_half : 0u) + ks * 256u;
                tc::mma_bf16(d1, tc::make_sdesc(aa, lbo, 128), tc::make_sdesc(bb, 128, KCG * 128u), id1, acc);
                acc = 1;
              }
          }
          const uint32_t gsb = gs0 + (uint32_t)gs * L.gs_bytes;
          for (int r = 0; r < g.RT; ++r) {   // x-synthesis: K = k' (40 of 48; k-group 5 from the zero block)
            const uint32_t fbr = fb0 + (uint32_t)(g.RT == 2 ? 1 + r : cb) * 2u * fh;
            const uint32_t gh = gsb + (uint32_t)r * 10u * LG, gl = gh + 5u * LG;
            for (int ks = 0; ks < 3; ++ks)
#pragma unroll
              for (int p = 0; p < 3; ++p) {
                const uint32_t aa = fbr + (p == 2 ? fh : 0u) + (uint32_t)ks * 4096u;
                const uint32_t bb = (p == 1 ? gl : gh) + (uint32_t)ks * 2u * LG;
                tc::mma_bf16(d1, tc::make_sdesc(aa, ks < 2 ? 2048u : zb0 - aa, 128), tc::make_sdesc(bb, ks < 2 ? LG : zb0 - bb, 128),
                             id2, acc);
                acc = 1;
              }
          }
          tc::mma_commit(&d1full[d]);
          tc::mma_commit(&gempty[gs]);
          PX_TRACE(t, 2);
        }
      }
    }
  } else if (warp == 3) {
    // ================= x-analysis MMAs (one thread): D2[o][k'] += sum_p v'[p][o] F[p][k']
    if (tc::elect_one()) {
      tc::mbar_wait(cstb, 0);
      const uint32_t id3 = tc::make_idesc_bf16(128, 48, true, true);     // v'^T (MN-major) . F (MN-major)
      int t = 0, ui = 0;
      for (int u = next_unit(blockIdx.x); u < nunits; u = next_unit(u + gridDim.x), ++ui) {
        const int b2 = ui & 1;
        for (int cb = 0; cb < g.CB; ++cb, ++t) {
          const int s = t % NST;
          tc::mbar_wait(&vfull[s], (uint32_t)(t / NST) & 1u);
          PX_TRACE(t, 8);
          if (cb == 0) tc::mbar_wait(&d2empty[b2], ((uint32_t)(ui >> 1) & 1u) ^ 1u);
          PX_TRACE(t, 9);
          tc::fence_after_sync();
          const uint32_t sth = sth0 + (uint32_t)s * L.stage_bytes, stl = sth + sh;
          const uint32_t d2 = tmem + 2u * NP + (uint32_t)b2 * g.D2W;
          if (g.RT == 2) {        // two rows: pixels 0-63 -> columns [0, 48), pixels 64-127 -> [48, 96)
            for (int r = 0; r < 2; ++r)
              for (int ks = 0; ks < 4; ++ks)
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                  const int kk = r * 4 + ks;
                  const uint32_t aa = (p == 2 ? stl : sth) + (uint32_t)kk * 256u;
                  const uint32_t bb = fb0 + (p == 1 ? fh : 0u) + (uint32_t)kk * 256u;
                  tc::mma_bf16(d2 + (uint32_t)r * 48u, tc::make_sdesc(aa, 128, 2048), tc::make_sdesc(bb, 128, 2048), id3,
                               (ks | p) != 0);
                }
          } else {
            const uint32_t fbc = fb0 + (uint32_t)cb * 2u * fh;
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
              for (int p = 0; p < 3; ++p) {
                const uint32_t aa = (p == 2 ? stl : sth) + (uint32_t)ks * 256u;
                const uint32_t bb = fbc + (p == 1 ? fh : 0u) + (uint32_t)ks * 256u;
                tc::mma_bf16(d2, tc::make_sdesc(aa, 128, 2048), tc::make_sdesc(bb, 128, 2048), id3, (cb | ks | p) != 0);
              }
          }
          tc::mma_commit(&empty[s]);                       // stage t consumed
          PX_TRACE(t, 5);
          if (cb == g.CB - 1) tc::mma_commit(&d2full[b2]);
        }
      }
    }
  } else if (warp < kPxE2First) {
    // ================= epilogue 1: thread = pixel p of the tile (TMEM lane p); warpgroup eg takes the
    // 16-column chunks eg, eg + 3, ... of the NP channels
    const int q4 = warp & 3, p = q4 * 32 + lane, eg = (warp - kPxE1First) / 4;
    float* pj = reinterpret_cast<float*>(sm + L.pj);
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t poff = (uint32_t)(p >> 3) * 128u + (uint32_t)(p & 7) * 16u;
    int t = 0;
    int u = next_unit(blockIdx.x);
    const bool use_gelu = a.use_gelu != 0;
    double inv_next = (FIRST && u < nunits) ? __ldg(a.rr + u / g.units) : 0.0;   // 1/||r|| of the next unit, in flight
    for (int un; u < nunits; u = un) {
      const int b = u / g.units, ul = u % g.units;
      un = next_unit(u + gridDim.x);
      float rh = 0.f, kf = 0.f;
      const double inv_s = inv_next;
      if (FIRST && un < nunits) inv_next = __ldg(a.rr + un / g.units);
      for (int cb = 0; cb < g.CB; ++cb, ++t) {
        const int s = t % NST, d = t & 1;
        if (lane == 0 && q4 == 0 && eg == 0) PX_TRACE(t, 6);
        tc::mbar_wait(&d1full[d], (uint32_t)(t >> 1) & 1u);
        if (lane == 0 && q4 == 0 && eg == 0) PX_TRACE(t, 3);
        if (lane == 0) PX_TRACE(t, 10 + 2 * (warp - kPxE1First));
        tc::fence_after_sync();
        if (FIRST) {   // the lift's 2-channel bypass W1 (E [r/||r||, k] + bE) on the CUDA cores
          tc::mbar_wait(&full[s], (uint32_t)(t / NST) & 1u);
          const double* rk = reinterpret_cast<const double*>(sm + L.RK + s * 2048);
          rh = (float)(rk[p] * inv_s);
          kf = (float)rk[128 + p];
        }
        unsigned char* sth = sm + L.ST + (uint32_t)s * L.stage_bytes;
        unsigned char* stl = sth + g.stage_half();
        unsigned char* gv = PROJ ? nullptr : a.vout + ((size_t)b * g.TPS + ul * g.CB + cb) * 2 * g.v_half();
        float pacc = 0.f;
        for (int c0 = 16 * eg; c0 < NP; c0 += 16 * kPxE1Groups) {
          uint32_t uu[16];
          tc::tmem_ld16(tmem + (uint32_t)d * NP + lane_off + (uint32_t)c0, uu);
          tc::tmem_wait_ld();
          float v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int o = c0 + q;
            v[q] = __uint_as_float(uu[q]) + sbias[o];
            if (FIRST) v[q] = fmaf(sw1e[2 * o], rh, fmaf(sw1e[2 * o + 1], kf, v[q]));
          }
          if (use_gelu) {   // one uniform branch around 8 independent pairs
#pragma unroll
            for (int q = 0; q < 16; q += 2) gelu_px2(v[q], v[q + 1]);
          }
          if (PROJ) {
#pragma unroll
            for (int q = 0; q < 16; ++q) pacc = fmaf(sdw[c0 + q], v[q], pacc);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cg = c0 / 8 + h;
            const uint32_t off = (uint32_t)cg * 2048u + poff;
            uint4 hv, lv;
            tc::split8(v + 8 * h, hv, lv);
            if (cg < g.CGS) {   // stage (in place) and the next layer's V blob (16-byte stores, 512 B per warp)
              *reinterpret_cast<uint4*>(sth + off) = hv;
              *reinterpret_cast<uint4*>(stl + off) = lv;
              if (!PROJ) {
                *reinterpret_cast<uint4*>(gv + off) = hv;
                *reinterpret_cast<uint4*>(gv + g.v_half() + off) = lv;
              }
            }
          }
        }
        tc::fence_before_sync();
        tc::mbar_arrive(&d1empty[d]);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&vfull[s]);
        if (lane == 0 && q4 == 0 && eg == 0) PX_TRACE(t, 4);
        if (lane == 0) PX_TRACE(t, 11 + 2 * (warp - kPxE1First));
        if (PROJ) {   // sum_o (D W4)[o] v3[o]: the groups' partials added in a fixed order
          pj[((size_t)d * kPxE1Groups + eg) * 128 + p] = pacc;
          tc::named_sync(1, 32u * kPxE1Warps);
          if (eg == 0) {
            float acc = 0.f;
#pragma unroll
            for (int q = 0; q < kPxE1Groups; ++q) acc += pj[((size_t)d * kPxE1Groups + q) * 128 + p];
            a.p3[(size_t)b * N + (size_t)(ul * g.CB + cb) * 128 + p] = acc;
          }
        }
      }
    }
  } else {
    // ================= epilogue 2: thread = channel o (TMEM lane o) -> T rows [kappa2][o][re|im]
    const int q4 = warp & 3, o = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int ui = 0;
    for (int u = next_unit(blockIdx.x); u < nunits; u = next_unit(u + gridDim.x), ++ui) {
      const int b = u / g.units, ul = u % g.units, b2 = ui & 1;
      tc::mbar_wait(&d2full[b2], (uint32_t)(ui >> 1) & 1u);
      tc::fence_after_sync();
      for (int r = 0; r < g.RT; ++r) {
        uint32_t v[48];
        const uint32_t col = tmem + 2u * NP + (uint32_t)b2 * g.D2W + (uint32_t)r * 48u + lane_off;
        tc::tmem_ld16(col, *reinterpret_cast<uint32_t(*)[16]>(v));
        tc::tmem_ld16(col + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tc::tmem_ld16(col + 32, *reinterpret_cast<uint32_t(*)[16]>(v + 32));
        tc::tmem_wait_ld();
        if (o < w) {
          float2* dst = reinterpret_cast<float2*>(a.T + ((size_t)b * n + ul * g.RT + r) * 40 * w) + o;
#pragma unroll
          for (int k2 = 0; k2 < kModes; ++k2)
            dst[(size_t)k2 * w] = make_float2(__uint_as_float(v[2 * k2]), __uint_as_float(v[2 * k2 + 1]));
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&d2empty[b2]);
      if (lane == 0 && q4 == 0) PX_TRACE(ui, 7);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ------------------------------------------------------------------ k_px_ysyn: y-synthesis
// Work = (system b, M tile of 128 rows i, kappa2) steps; a CTA takes items (b, M tile, group of KG
// consecutive kappa2) and walks their steps in order.  For each kappa2 the B operand
// Gh[(k1, p)][(q, o)] (K = 48, N = 2 NP) is built from the mixed spectrum g[kappa][b][o]:
//   rows (k1, 0): (gr | gi),  rows (k1, 1): (gi | -gr)    so that  D[i][(q,o)] = (Gr | Gi)[i][kappa2][o]
// with Fp[i][(k1,0)] = cos, Fp[i][(k1,1)] = -sin: Gr = sum gr cos - gi sin, Gi = sum gi cos + gr sin
// (g e^{+i theta}).  Warp-specialised: warps 0-7 build B(step) into a double buffer (thread = (o, half
// of the kappa1 range), all its loads in flight at once), warp 8 issues the MMAs into a double-buffered
// TMEM accumulator, warps 9-16 write the G rows' bf16 hi/lo pieces (32 bytes per (row, o-group),
// consecutive rows adjacent: 1 KB per warp store).
constexpr int kYsynBuild = 8, kYsynEpi = 8, kYsynThreads = (kYsynBuild + 1 + kYsynEpi) * 32;
struct PxYsynSmem {
  uint32_t A, Bb, bar, tptr, runb, total, b_half;
  __host__ __device__ PxYsynSmem(const PxGeom& g) {
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    A = take((uint32_t)g.nMT * 2u * 128u * 48u * 2u);   // every M tile's Fp blob, resident
    b_half = 2u * (uint32_t)g.NP * 48u * 2u;
    Bb = take(2u * 2u * b_half);
    bar = take(128);
    tptr = bar + 120;
    runb = take(kPxMaxSys / 8);
    total = o;
  }
};

__global__ void __launch_bounds__(kYsynThreads, 1) k_px_ysyn(const float2* __restrict__ ghat, const unsigned char* __restrict__ cst,
                                                             unsigned char* __restrict__ Gb, int n, int w, int B, int kg,
                                                             const int* __restrict__ status) {
  const PxGeom g(n, w);
  const PxConst C(g);
  const PxYsynSmem L(g);
  extern __shared__ __align__(1024) unsigned char sm[];
  const int NP = g.NP, N2 = 2 * NP, nkg = kModes / kg, wp = (w + 3) & ~3;   // wp: row pitch of the spectra
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);
  uint64_t *bfull = bar, *bfree = bar + 2, *dfull = bar + 4, *dfree = bar + 6, *abar = bar + 8;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  const int nitems = B * g.nMT * nkg;
  const uint32_t LBO_B = (uint32_t)(N2 / 8) * 128u, ncols = pow2_cols(2u * N2);
  uint32_t* runb = reinterpret_cast<uint32_t*>(sm + L.runb);   // running-system bitmask (B <= kPxMaxSys)
  const bool cached = status && B <= kPxMaxSys;
  if (cached)
    for (int q = warp; q < (B + 31) / 32; q += blockDim.x / 32) {
      const int sb = q * 32 + lane;
      const unsigned bits = __ballot_sync(0xffffffffu, sb < B && __ldcg(status + sb) == SYS_RUNNING);
      if (lane == 0) runb[q] = bits;
    }
  auto next_item = [&](int it) {
    if (!status) return it;
    while (it < nitems) {
      const int sb = it / (g.nMT * nkg);
      if (cached ? ((runb[sb >> 5] >> (sb & 31)) & 1u) != 0 : __ldcg(status + sb) == SYS_RUNNING) break;
      it += gridDim.x;
    }
    return it;
  };
  if (tid == 0) {
    for (int q = 0; q < 9; ++q) tc::mbar_init(&bar[q], q < 2 ? 32u * kYsynBuild : (q >= 6 && q < 8) ? 32u * kYsynEpi : 1u);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(abar, (uint32_t)g.nMT * 2u * C.fp_half);
    tc::bulk_g2s(sm + L.A, cst + C.FP, (uint32_t)g.nMT * 2u * C.fp_half, abar);
  }
  if (warp == 0) tc::tmem_alloc(tptr, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  pdl_wait();
  pdl_trigger();

  if (warp < kYsynBuild) {
    // ================= B builders
    const int bt = tid;
    uint32_t c = 0;
    for (int it = next_item(blockIdx.x); it < nitems; it = next_item(it + gridDim.x)) {
      const int b = it / (g.nMT * nkg), k20 = (it % nkg) * kg;
      for (int kk = 0; kk < kg; ++kk, ++c) {
        const int k2 = k20 + kk;
        tc::mbar_wait(&bfree[c & 1u], ((c >> 1) & 1u) ^ 1u);
        unsigned char* bh = sm + L.Bb + (c & 1u) * 2u * L.b_half;
        for (int t = bt; t < 2 * NP; t += 32 * kYsynBuild) {   // task = (o, kappa1 half: k-groups 3h .. 3h+2)
          const int o = t % NP, hh = t / NP;
          float2 gg[12];
#pragma unroll
          for (int e = 0; e < 12; ++e) {
            const int k1 = hh * 12 + e;
            gg[e] = (k1 < kModes && o < w) ? __ldg(ghat + ((size_t)(k1 * kModes + k2) * B + b) * wp + o) : make_float2(0.f, 0.f);
          }
#pragma unroll
          for (int kq = 0; kq < 3; ++kq) {
            const int kgp = hh * 3 + kq;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 z = gg[kq * 4 + e];
                v[2 * e] = q == 0 ? z.x : z.y;
                v[2 * e + 1] = q == 0 ? z.y : -z.x;
              }
              const int nn = q * NP + o;
              const uint32_t off = (uint32_t)(nn >> 3) * 128u + (uint32_t)kgp * LBO_B + (uint32_t)(nn & 7) * 16u;
              st_split8(bh + off, bh + L.b_half + off, v);
            }
          }
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&bfull[c & 1u]);
      }
    }
  } else if (warp == kYsynBuild) {
    // ================= MMA issuer
    if (tc::elect_one()) {
      tc::mbar_wait(abar, 0);
      const uint32_t id = tc::make_idesc_bf16(128, N2, false, false);
      const uint32_t base = tc::smem_u32(sm);
      uint32_t c = 0;
      for (int it = next_item(blockIdx.x); it < nitems; it = next_item(it + gridDim.x)) {
        const int mt = (it / nkg) % g.nMT;
        const uint32_t ah = base + L.A + (uint32_t)mt * 2u * C.fp_half, al = ah + C.fp_half;
        for (int kk = 0; kk < kg; ++kk, ++c) {
          tc::mbar_wait(&bfull[c & 1u], (c >> 1) & 1u);
          tc::mbar_wait(&dfree[c & 1u], ((c >> 1) & 1u) ^ 1u);
          tc::fence_after_sync();
          const uint32_t bh = base + L.Bb + (c & 1u) * 2u * L.b_half, bl = bh + L.b_half;
          const uint32_t d = tmem + (c & 1u) * (uint32_t)N2;
          for (int ks = 0; ks < 3; ++ks)
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const uint32_t aa = (p == 2 ? al : ah) + (uint32_t)ks * 256u;
              const uint32_t bb = (p == 1 ? bl : bh) + (uint32_t)ks * 2u * LBO_B;
              tc::mma_bf16(d, tc::make_sdesc(aa, 128, 768), tc::make_sdesc(bb, LBO_B, 128), id, (ks | p) != 0);
            }
          tc::mma_commit(&dfull[c & 1u]);
          tc::mma_commit(&bfree[c & 1u]);
        }
      }
    }
  } else {
    // ================= epilogue: thread = row i of the M tile; the two warpgroups split the o-groups
    const int ew = warp - (kYsynBuild + 1), q4 = warp & 3, half = ew / 4;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    uint32_t c = 0;
    for (int it = next_item(blockIdx.x); it < nitems; it = next_item(it + gridDim.x)) {
      const int b = it / (g.nMT * nkg), mt = (it / nkg) % g.nMT, k20 = (it % nkg) * kg;
      const int i = mt * 128 + q4 * 32 + lane;
      for (int kk = 0; kk < kg; ++kk, ++c) {
        tc::mbar_wait(&dfull[c & 1u], (c >> 1) & 1u);
        tc::fence_after_sync();
        const int k2 = k20 + kk, kgi = k2 >> 2, pair = k2 & 3;   // k' = 2 k2 + q: k-group k2/4, pair k2%4
        const uint32_t dcol = tmem + (c & 1u) * (uint32_t)N2 + lane_off;
        // 32 bytes per (row, o-group): [k' = 2 k2 | 2 k2 + 1]; the TMEM loads of 3 o-groups issued together
        for (int og0 = half; og0 < NP / 8; og0 += 6) {
          uint32_t re[3][8], im[3][8];
#pragma unroll
          for (int z = 0; z < 3; ++z) {
            const int og = og0 + 2 * z;
            if (og < NP / 8) {
              tmem_ld8(dcol + (uint32_t)(og * 8), re[z]);
              tmem_ld8(dcol + (uint32_t)(NP + og * 8), im[z]);
            }
          }
          tc::tmem_wait_ld();
#pragma unroll
          for (int z = 0; z < 3; ++z) {
            const int og = og0 + 2 * z;
            if (i < n && og < NP / 8) {
              float vr[8], vi[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) { vr[e] = __uint_as_float(re[z][e]); vi[e] = __uint_as_float(im[z][e]); }
              uint4 hr, lr, hi, li;
              tc::split8(vr, hr, lr);
              tc::split8(vi, hi, li);
              // one 32-byte store per (row, o-group) piece: a warp writes 1 KB contiguous per instruction
              st_global_256(Gb + g.g_off(b, 0, kgi, og, pair, i), hr, hi);
              st_global_256(Gb + g.g_off(b, 1, kgi, og, pair, i), lr, li);
            }
          }
        }
        tc::fence_before_sync();
        tc::mbar_arrive(&dfree[c & 1u]);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ------------------------------------------------------------------ k_px_yan: y-analysis
// Item = (system b, M tile of 128 rows m = (kappa2 w + o) 2 + (re|im) of the T rows), K = i in chunks of
// 64 rows.  Each thread holds its part of the next chunk in registers (8 x 16-byte loads in flight)
// while the current one is converted fp32 -> bf16 hi/lo (MN-major A) into a double buffer and the
// previous chunk's MMAs run: one block barrier per chunk.  B = F[i][(k1, x|y)], resident.
// Epilogue: lane pairs (re, im) recombine  c_r = T_r.Fx - T_i.Fy,  c_i = T_i.Fx + T_r.Fy  (e^{-i theta}).
constexpr int kYanKC = 64, kYanTasks = kYanKC * 16 / 256;   // 16-row... 8-float tasks per thread per chunk
struct PxYanSmem {
  uint32_t A, Bf, bar, tptr, total;
  __host__ __device__ PxYanSmem(const PxGeom& g) {
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    A = take(2u * 2u * 128u * kYanKC * 2u);
    Bf = take(2u * (uint32_t)g.n * 48u * 2u);
    bar = take(64);
    tptr = bar + 56;
    total = o;
  }
};

__global__ void __launch_bounds__(256) k_px_yan(const float* __restrict__ T, const unsigned char* __restrict__ cst,
                                                float2* __restrict__ chat, int n, int w, int B,
                                                const int* __restrict__ status) {
  const PxGeom g(n, w);
  const PxConst C(g);
  const PxYanSmem L(g);
  extern __shared__ __align__(1024) unsigned char sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0,1] MMA of A buffer; [2] B landed
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  const int nitems = B * g.MYT, nK = n / kYanKC, M = 40 * w;
  const uint32_t a_half = 128u * kYanKC * 2u, SBO_Y = (uint32_t)(n / 8) * 128u;
  auto next_item = [&](int it) {
    while (it < nitems && status && __ldcg(status + it / g.MYT) != SYS_RUNNING) it += gridDim.x;
    return it;
  };
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&bar[2], 2u * C.fy_half);
    tc::bulk_g2s(sm + L.Bf, cst + C.FY, 2u * C.fy_half, &bar[2]);
  }
  if (warp == 0) tc::tmem_alloc(tptr, 64);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t base = tc::smem_u32(sm);
  const uint32_t id = tc::make_idesc_bf16(128, 48, true, false);
  pdl_wait();
  pdl_trigger();
  if (tid == 0) tc::mbar_wait(&bar[2], 0);
  // the CTA's chunk sequence (item, kc); registers x hold the next chunk's loads
  float4 x[kYanTasks][2];
  int lit = next_item(blockIdx.x), lkc = 0;
  auto load = [&]() {
    if (lit < nitems) {
      const int b = lit / g.MYT, m0 = (lit % g.MYT) * 128;
      const float* src = T + ((size_t)b * n + (size_t)lkc * kYanKC) * M + m0;
#pragma unroll
      for (int z = 0; z < kYanTasks; ++z) {   // task t = (row il, 8-float group mg): lanes cover 8 rows x 4 groups
        const int t = tid + z * 256, il = (t >> 7) * 8 + (t & 7), mg = (t >> 3) & 15;
        ld_global_256(src + (size_t)il * M + mg * 8, x[z][0], x[z][1]);   // 32 contiguous bytes, one load
      }
      if (++lkc == nK) { lkc = 0; lit = next_item(lit + gridDim.x); }
    }
  };
  load();
  uint32_t c = 0;
  for (int it = next_item(blockIdx.x); it < nitems; it = next_item(it + gridDim.x)) {
    const int b = it / g.MYT, m0 = (it % g.MYT) * 128;
    for (int kc = 0; kc < nK; ++kc, ++c) {
      if (c >= 2) tc::mbar_wait(&bar[c & 1u], ((c - 2u) >> 1) & 1u);    // MMA c - 2 done with A buffer c & 1
      unsigned char* ah = sm + L.A + (c & 1u) * 2u * a_half;
#pragma unroll
      for (int z = 0; z < kYanTasks; ++z) {   // a warp's 32 chunks are 512 contiguous bytes (no bank conflicts)
        const int t = tid + z * 256, ih = t >> 7, il7 = t & 7, mg = (t >> 3) & 15;
        const float v[8] = {x[z][0].x, x[z][0].y, x[z][0].z, x[z][0].w, x[z][1].x, x[z][1].y, x[z][1].z, x[z][1].w};
        const uint32_t off = (uint32_t)mg * 128u + (uint32_t)ih * 2048u + (uint32_t)il7 * 16u;
        st_split8(ah + off, ah + a_half + off, v);
      }
      load();                                                            // next chunk in flight from here
      tc::fence_proxy_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      tc::fence_after_sync();
      if (warp == 0 && tc::elect_one()) {
        const uint32_t aah = base + L.A + (c & 1u) * 2u * a_half, aal = aah + a_half;
        const uint32_t bh = base + L.Bf, bl = bh + C.fy_half;
        for (int ks = 0; ks < kYanKC / 16; ++ks)
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            const uint32_t aa = (p == 2 ? aal : aah) + (uint32_t)ks * 4096u;
            const uint32_t bb = (p == 1 ? bl : bh) + (uint32_t)((kc * kYanKC + ks * 16) / 8) * 128u;
            tc::mma_bf16(tmem, tc::make_sdesc(aa, 2048, 128), tc::make_sdesc(bb, 128, SBO_Y), id, (kc | ks | p) != 0);
          }
        tc::mma_commit(&bar[c & 1u]);
      }
    }
    // epilogue: all of this item's MMAs complete (the last commit covers the earlier ones); the next
    // item's first MMA is issued only after the next chunk's block barrier
    const uint32_t cl = c - 1u;
    tc::mbar_wait(&bar[cl & 1u], (cl >> 1) & 1u);
    tc::fence_after_sync();
    if (warp < 4) {
      uint32_t v[48];
      const uint32_t col = tmem + ((uint32_t)(warp * 32) << 16);
      tc::tmem_ld16(col, *reinterpret_cast<uint32_t(*)[16]>(v));
      tc::tmem_ld16(col + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
      tc::tmem_ld16(col + 32, *reinterpret_cast<uint32_t(*)[16]>(v + 32));
      tc::tmem_wait_ld();
      const int m = m0 + warp * 32 + lane, pr = m >> 1, k2 = pr / w, o = pr - k2 * w;
      const bool re = (lane & 1) == 0;
      const int wp = (w + 3) & ~3;                                    // row pitch of the mode-major spectra
      float2* dst = chat + ((size_t)k2 * B + b) * wp + o;           // mode (k1, k2) at dst + k1 * 20 B wp
      const size_t kstride = (size_t)kModes * B * wp;
#pragma unroll
      for (int k1 = 0; k1 < kModes; ++k1) {
        const float xv = __uint_as_float(v[2 * k1]), yv = __uint_as_float(v[2 * k1 + 1]);
        const float px = __shfl_xor_sync(0xffffffffu, xv, 1), py = __shfl_xor_sync(0xffffffffu, yv, 1);
        if (re && m < M) dst[k1 * kstride] = make_float2(xv - py, px + yv);
      }
    }
    tc::fence_before_sync();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
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

__global__ void __launch_bounds__(128) k_mix_tc(const float2* __restrict__ chat, const unsigned char* __restrict__ mx,
                                               float2* __restrict__ ghat, int w, int B, int cout, float inv_n2,
                                               const int* status) {
  const int KM = (2 * w + 15) & ~15, NM = (cout + 15) & ~15, wp = (w + 3) & ~3;   // wp: row pitch of the spectra
  const MixSmem L(KM, NM);
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t SBO = (KM / 8) * 128, a_half = 128u * KM * 2, b_half = (uint32_t)NM * KM * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0] B load, [1] MMA
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbc = (B + kMixSys - 1) / kMixSys, nitems = kModes2 * nbc;
  auto prefetch = [&](int it) {
    const int kk = it / nbc;
    tc::mbar_expect_tx(&bar[0], 2 * b_half);
    tc::bulk_g2s(sm + L.B, mx + (size_t)kk * 2 * b_half, 2 * b_half, &bar[0]);
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
    // A: rows (b, re|im), K = (c, re|im); all loads of a batch first.  A task's four channels are 32
    // contiguous, 32-byte aligned bytes (spectra rows are padded to wp = 4-channel multiples): one 256-bit
    // load per task instead of four 8-byte loads that each cost the load unit a pass over 32 scattered lines
    {
      constexpr int kBatch = 8;
      const int ntask = kMixSys * (KM / 8);
      for (int t0 = tid; t0 < ntask; t0 += kBatch * blockDim.x) {
        float4 x[kBatch][2];
#pragma unroll
        for (int z = 0; z < kBatch; ++z) {
          const int t = t0 + z * blockDim.x, bl = t % kMixSys, kc = t / kMixSys;
          if (t < ntask && bl < nb && kc * 4 < wp)
            ld_global_256(reinterpret_cast<const float*>(chat + ((size_t)kk * B + b0 + bl) * wp + kc * 4), x[z][0], x[z][1]);
          else
            x[z][0] = x[z][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int z = 0; z < kBatch; ++z) {
          const int t = t0 + z * blockDim.x, bl = t % kMixSys, kc = t / kMixSys;
          if (t >= ntask) break;
          const float cr[4] = {x[z][0].x, x[z][0].z, x[z][1].x, x[z][1].z}, ci[4] = {x[z][0].y, x[z][0].w, x[z][1].y, x[z][1].w};
          float vr[8], vi[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = kc * 4 + q < w;          // the row's padding holds no data
            const float re = in ? cr[q] : 0.f, im = in ? ci[q] : 0.f;
            vr[2 * q] = re;  vr[2 * q + 1] = -im;
            vi[2 * q] = im;  vi[2 * q + 1] = re;
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
    if (warp == 0 && tc::elect_one()) {
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
      const int coutp = cout == 1 ? 1 : wp;          // output row pitch (padded like the input's)
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
          float2 o4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float gr = p ? other[q] : mine[q], gi = p ? mine[q] : other[q];
            o4[q] = make_float2(gr * inv_n2, gi * inv_n2);
          }
          float2* dst = ghat + ((size_t)kk * B + b) * coutp + c0 + 4 * p;
          if (cout > 1) {   // 4 channels = 32 aligned bytes (columns >= cout of the padded row receive zeros)
            if (c0 + 4 * p < coutp)
              st_global_256(dst, make_uint4(__float_as_uint(o4[0].x), __float_as_uint(o4[0].y), __float_as_uint(o4[1].x), __float_as_uint(o4[1].y)),
                            make_uint4(__float_as_uint(o4[2].x), __float_as_uint(o4[2].y), __float_as_uint(o4[3].x), __float_as_uint(o4[3].y)));
          } else if (p == 0) {
            dst[0] = o4[0];
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

// ------------------------------------------------------------------ host side
static int px_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      v = 0;
  }
  return v;
}
static int px_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}


bool px_supported_shape(int n, int w) {
  if (w < 1 || w > 128) return false;
  if (!(n == 64 || (n % 128 == 0 && n >= 128 && n <= 512))) return false;
  const PxGeom g(n, w);
  return PxSmem(g, true, false).total <= kPxSmemLimit && PxSmem(g, false, false).total <= kPxSmemLimit &&
         PxSmem(g, false, true).total <= kPxSmemLimit &&
         PxYsynSmem(g).total <= kPxSmemLimit && PxYanSmem(g).total <= kPxSmemLimit;
}

bool px_supported(int n, int w) { return px_supported_shape(n, w) && px_optin() >= (int)kPxSmemLimit; }

size_t px_const_bytes(int n, int w) { return PxConst(PxGeom(n, w)).total; }
size_t px_v_bytes(int n, int w, int B) { return PxGeom(n, w).v_bytes(B); }
size_t px_g_bytes(int n, int w, int B) { return PxGeom(n, w).g_bytes(B); }
size_t px_t_floats(int n, int w, int B) { return PxGeom(n, w).t_floats(B); }
size_t px_mx_offset(int n, int w, int mix) { return PxConst(PxGeom(n, w)).MX[mix]; }

cudaError_t prepare_px_kernels() {
  static bool done = false;
  if (done) return cudaSuccess;
  const void* fns[6] = {(const void*)k_px_layer<true, false>, (const void*)k_px_layer<false, false>,
                        (const void*)k_px_layer<false, true>, (const void*)k_px_ysyn, (const void*)k_px_yan,
                        (const void*)k_px_layer<true, true>};
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPxSmemLimit);
    if (e != cudaSuccess) return e;
  }
  done = true;
  return cudaSuccess;
}

cudaError_t launch_px_prep(int n, int w, const float* W2, const float* W3, const float* R2, const float* R3,
                           const float* Q, const float* F, unsigned char* out, cudaStream_t s) {
  PxPrepArgs a{};
  a.n = n; a.w = w; a.W[0] = W2; a.W[1] = W3;
  a.Rm[0] = reinterpret_cast<const float2*>(R2); a.Rm[1] = reinterpret_cast<const float2*>(R3);
  a.Rm[2] = reinterpret_cast<const float2*>(Q);
  a.F = reinterpret_cast<const float2*>(F);
  a.out = out;
  k_px_prep<<<2 * px_sms(), 256, 0, s>>>(a);
  ++launch_counter();
  return cudaGetLastError();
}

// TMA tensor map of the interleaved G layout (px_layout.cuh): dims (innermost first) 8 x u32 (32 B),
// n rows, 4 pairs, 5 x NP/8 (k-group, o-group), 2 B (system, hi|lo); box = one row's hi or lo blob.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static cudaError_t make_g_map(CUtensorMap* m, const unsigned char* G, const PxGeom& g, int B) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t n = (cuuint64_t)g.n, kog = 5ull * (g.NP / 8);
  const cuuint64_t dims[5] = {8, n, 4, kog, 2ull * B};
  const cuuint64_t strides[4] = {32, 32 * n, 128 * n, 128 * n * kog};
  const cuuint32_t box[5] = {8, 1, 4, (cuuint32_t)kog, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, const_cast<unsigned char*>(G), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_px_layer(const PxLayerHost& h, cudaStream_t s) {
  PxLayerArgs a{};
  a.n = h.n; a.w = h.w; a.B = h.B; a.layer = h.layer; a.use_gelu = h.use_gelu;
  a.r = h.r; a.rr = h.rr; a.k = h.k; a.vin = h.vin; a.vout = h.vout; a.G = h.G; a.T = h.T; a.cst = h.cst;
  a.bias = h.bias; a.w1e = h.w1e; a.dw = h.dw; a.p3 = h.p3; a.status = h.status;
  static int trace_layer = -1;
  if (trace_layer < 0) { const char* e = getenv("FCGNO_PX_TRACE"); trace_layer = e ? atoi(e) : 0; }
  a.trace = trace_layer == h.layer + 1;
  const PxGeom g(h.n, h.w);
  const bool first = h.layer == 0, proj = h.layer == 2;
  const size_t smem = PxSmem(g, first, proj).total;
  const int grid = std::min(h.B * g.units, px_sms());
  alignas(64) CUtensorMap gmap;
  if (const cudaError_t e = make_g_map(&gmap, h.G, g, h.B)) return e;
  if (first) return launch_k(k_px_layer<true, false>, dim3(grid), dim3(kPxThreads), smem, s, a, gmap);
  if (proj) return launch_k(k_px_layer<false, true>, dim3(grid), dim3(kPxThreads), smem, s, a, gmap);
  return launch_k(k_px_layer<false, false>, dim3(grid), dim3(kPxThreads), smem, s, a, gmap);
}

cudaError_t launch_px_ysyn(const float* ghat, const unsigned char* cst, unsigned char* Gb, int n, int w, int B,
                           const int* status, cudaStream_t s) {
  const PxGeom g(n, w);
  const int sms = px_sms();
  // one kappa2 per item: the Fp blobs are resident, so finer items only improve the balance
  const int base_items = B * g.nMT;
  const int kg = 1;
  const PxYsynSmem L(g);
  const int items = base_items * (kModes / kg);
  const int grid = std::min(items, sms);
  return launch_k(k_px_ysyn, dim3(grid), dim3(kYsynThreads), (size_t)L.total, s, reinterpret_cast<const float2*>(ghat),
                  cst, Gb, n, w, B, kg, status);
}

cudaError_t launch_px_yan(const float* T, const unsigned char* cst, float* chat, int n, int w, int B, const int* status,
                          cudaStream_t s) {
  const PxGeom g(n, w);
  const PxYanSmem L(g);
  const int items = B * g.MYT;
  const int per_sm = std::max(1, std::min(3, (int)((228u * 1024u) / (L.total + 1024u))));
  const int grid = std::min(items, per_sm * px_sms());
  return launch_k(k_px_yan, dim3(grid), dim3(256), (size_t)L.total, s, T, cst, reinterpret_cast<float2*>(chat), n, w,
                  B, status);
}


cudaError_t launch_mix_px(int mix, const float* chat, const unsigned char* cst, float* ghat, int n, int w, int B,
                          float inv_n2, const int* status, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute((const void*)k_mix_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int cout = mix < 2 ? w : 1, KM = (2 * w + 15) & ~15, NM = (cout + 15) & ~15;
  const size_t smem = MixSmem(KM, NM).total;
  const int nitems = kModes2 * ((B + kMixSys - 1) / kMixSys);
  const int per_sm = std::max(1, std::min(3, (int)((228u * 1024u) / (smem + 1024u))));
  const int grid = std::min(nitems, per_sm * px_sms());
  return launch_k(k_mix_tc, dim3(grid), dim3(128), smem, s, reinterpret_cast<const float2*>(chat),
                  cst + px_mx_offset(n, w, mix), reinterpret_cast<float2*>(ghat), w, B, cout, inv_n2, status);
}

cudaError_t px_trace_read(unsigned long long* host, int count) {
  return cudaMemcpyFromSymbol(host, g_px_trace, sizeof(unsigned long long) * std::min(count, kPxTraceTiles * kPxTraceEv));
}

}  // namespace fcgno

// no_tc_kernels.cu — tensor-core (tcgen05 / TMEM) SNO operator layer for the fp32 NO path.
//
// One layer (R7-R11) is
//   u[o][i][j] = sum_c W[o][c] v[c][i][j] + b[o] + n^-2 Re sum_kappa g[o](kappa) e^{+2 pi i kappa.(i,j)/n}
//   v'         = GELU(u)                                    (layers 1-3; layer 4 is folded away)
//   c'[o](k)   = sum_{i,j} v'[o][i][j] e^{-2 pi i k.(i,j)/n}
// The x-direction parts are dense contractions and run on the 5th-gen tensor cores; the
// y-direction parts (K = 20 modes against n rows) run in two small CUDA-core kernels that
// materialise G (y-synthesised g, per row) and read back T (x-analysed v', per row):
//
//   k_tc_layer  tile = R rows of one system; TMEM lanes = (row r, padded channel o) (R * WP = 128)
//     D1[(r,o)][j]  = sum_{(r',c)} Wbd[(r,o)][(r',c)] V[(r',c)][j]      bypass, block-diagonal in r
//                   + sum_{k'} G[(r,o)][k'] Basis[k'][j]                 x-synthesis (k' = (kappa2, re/im))
//     epilogue      v' = GELU(D1 + b)  -> global, and bf16 hi/lo into smem (A operand of D2)
//     D2[(r,o)][k'] = sum_j v'[(r,o)][j] F[j][k']                        x-analysis
//     epilogue      T[b][i][o][k'] <- D2
//   k_yan       c[kappa][b][o]   = sum_i F[i][kappa1] T[b][i][o][kappa2]     (y-analysis)
//   k_ysyn      G[b][i][o][k']   = sum_kappa1 g[b][o][kappa1][kappa2] conj(F[i][kappa1])   (y-synthesis)
//
// Precision: every operand is split into bf16 hi + lo and each product is accumulated as
// hi*hi + hi*lo + lo*hi in fp32 (3xBF16, ~2^-16 relative per product; SURVEY.md §0.1 item 5
// measured 1e-5 relative L2 for the whole NO, inside the 1e-4 parity bound).
#include <algorithm>

#include "internal.h"
#include "tc_common.cuh"

namespace fcgno {

constexpr int kTcThreads = 256;
constexpr int kKS = 48;                  // x-synthesis / x-analysis width: 40 (20 modes x re/im) padded to 48

template <int WP>
struct TcShape {
  static constexpr int R = 128 / WP;     // rows per tile
};

struct TcSmem {
  // byte offsets; every region 1024-aligned
  uint32_t AW[2], BV[2], AG[2], BF[2], bar, tptr, bias, total;
  int KB, CP;
  __host__ __device__ TcSmem(int n, int cin, int WP) {
    const int R = 128 / WP;
    CP = (cin + 7) & ~7;
    KB = (R * CP + 15) & ~15;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    for (int h = 0; h < 2; ++h) AW[h] = take(128u * KB * 2);
    for (int h = 0; h < 2; ++h) BV[h] = take((uint32_t)n * KB * 2);
    for (int h = 0; h < 2; ++h) AG[h] = take(128u * kKS * 2);
    for (int h = 0; h < 2; ++h) BF[h] = take((uint32_t)n * kKS * 2);
    bar = take(64);
    tptr = bar + 16;
    bias = take(128 * 4);
    total = o;
  }
};

struct TcLayerArgs {
  int n, N, w, cin, B, use_gelu;
  const double* r; const double* rr; const double* k;   // layer 1 inputs
  const float* vin;                                      // [B][cin][N] (layers 2, 3)
  const float* W;                                        // [w][cin]
  const float* bias;                                     // [w]
  const float* G;                                        // [B][n][w][40]
  const float2* F;                                       // [n][20]
  float* vout;                                           // [B][w][N]
  float* T;                                              // [B][n][w][40]
  const int* status;
};

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// 8 consecutive values -> 16 bytes of bf16 hi and 16 bytes of bf16 lo
__device__ __forceinline__ void store_split8(unsigned char* hi, unsigned char* lo, const float (&v)[8]) {
  __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) tc::split_bf16(v[t], h[t], l[t]);
  *reinterpret_cast<uint4*>(hi) = *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(lo) = *reinterpret_cast<const uint4*>(l);
}

template <int WP, bool FIRST>
__global__ void __launch_bounds__(kTcThreads, 2) k_tc_layer(const TcLayerArgs a) {
  constexpr int R = TcShape<WP>::R;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = a.N, w = a.w, cin = a.cin;
  const TcSmem L(n, cin, WP);
  const int KB = L.KB, CP = L.CP;
  const uint32_t SBO_AW = (KB / 8) * 128, SBO_BV = (KB / 8) * 128, SBO_AG = (kKS / 8) * 128,
                 SBO_F = (kKS / 8) * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // TMEM columns: D1 [0, n), D2 [n, n+48), v' as the A operand of D2: hi [n+64, n+64+n/2), lo after it
  const uint32_t need = (uint32_t)n + 64u + (uint32_t)n;
  const uint32_t ncols = need <= 128 ? 128u : (need <= 256 ? 256u : 512u);

  // ---- one-time setup: barriers, TMEM, block-diagonal weights, twiddle operand, bias
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tptr, ncols);
  for (int t = tid; t < 128 * (KB / 8); t += blockDim.x) {        // Wbd[(r,o)][(r',c)]
    const int Lr = t % 128, kc = t / 128;
    const int r = Lr / WP, o = Lr % WP;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kk = kc * 8 + q, rp = kk / CP, c = kk % CP;
      v[q] = (rp == r && rp < R && o < w && c < cin) ? a.W[(size_t)o * cin + c] : 0.f;
    }
    const uint32_t off = tc::kmajor_off(Lr, kc * 8, SBO_AW, 128);
    store_split8(sm + L.AW[0] + off, sm + L.AW[1] + off, v);
  }
  for (int t = tid; t < n * (kKS / 8); t += blockDim.x) {         // F[j][k'] (K-major view: N = j, K = k')
    const int j = t % n, kc = t / n;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kp = kc * 8 + q;
      if (kp < 2 * kModes) {
        const float2 f = a.F[(size_t)j * kModes + (kp >> 1)];
        v[q] = (kp & 1) ? f.y : f.x;
      } else {
        v[q] = 0.f;
      }
    }
    const uint32_t off = tc::kmajor_off(j, kc * 8, SBO_F, 128);
    store_split8(sm + L.BF[0] + off, sm + L.BF[1] + off, v);
  }
  for (int t = tid; t < 128; t += blockDim.x) {
    const int o = t % WP;
    sbias[t] = o < w ? a.bias[o] : 0.f;
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  const uint32_t tD1 = tmem, tD2 = tmem + (uint32_t)n;
  const uint32_t tAh = tmem + (uint32_t)n + 64u, tAl = tAh + (uint32_t)(n / 2);
  const uint32_t id1 = tc::make_idesc_bf16(128, n, false, true);     // A K-major, B MN-major (bypass)
  const uint32_t id1s = tc::make_idesc_bf16(128, n, false, false);   // synthesis: both K-major
  const uint32_t id2 = tc::make_idesc_bf16(128, kKS, false, true);   // analysis: B = F viewed MN-major
  const uint32_t sm_base = tc::smem_u32(sm);

  const int tiles_per_sys = n / R;
  const int ntiles = a.B * tiles_per_sys;
  uint32_t phase = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int b = tile / tiles_per_sys, i0 = (tile % tiles_per_sys) * R;
    if (a.status && a.status[b] != SYS_RUNNING) continue;
    // ---- stage V (MN-major B operand, K = (r', c)) and G (K-major A operand)
    double inv_s = 1.0;
    if (FIRST) {
      const double s = sqrt(a.rr[b]);
      inv_s = s > 0.0 ? 1.0 / s : 0.0;
    }
    {
      // all of this thread's global loads first (up to kStage tasks of 8 values), then convert
      constexpr int kStage = 8;
      const int nv = KB * (n / 8), ntask = nv + 128 * (kKS / 8);
      for (int t0 = tid; t0 < ntask; t0 += kStage * blockDim.x) {
        float v[kStage][8];
#pragma unroll
        for (int q = 0; q < kStage; ++q) {
          const int t = t0 + q * blockDim.x;
#pragma unroll
          for (int e = 0; e < 8; ++e) v[q][e] = 0.f;
          if (t >= ntask) continue;
          if (t < nv) {
            const int kk = t % KB, jc = t / KB;
            const int rp = kk / CP, c = kk % CP;
            if (rp < R && c < cin) {
              const size_t e = (size_t)(i0 + rp) * n + jc * 8;
              if (FIRST) {
                const double* src = (c == 0 ? a.r : a.k) + (size_t)b * N + e;
#pragma unroll
                for (int z = 0; z < 8; ++z) v[q][z] = (float)(c == 0 ? src[z] * inv_s : src[z]);
              } else {
                const float4* src = reinterpret_cast<const float4*>(a.vin + ((size_t)b * cin + c) * N + e);
                const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
                v[q][0] = x0.x; v[q][1] = x0.y; v[q][2] = x0.z; v[q][3] = x0.w;
                v[q][4] = x1.x; v[q][5] = x1.y; v[q][6] = x1.z; v[q][7] = x1.w;
              }
            }
          } else {
            const int u = t - nv, Lr = u % 128, kc = u / 128;
            const int r = Lr / WP, o = Lr % WP;
            if (o < w) {
              const float4* src = reinterpret_cast<const float4*>(a.G + (((size_t)b * n + i0 + r) * w + o) * (2 * kModes) + kc * 8);
              if (kc * 8 < 2 * kModes) {
                const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
                v[q][0] = x0.x; v[q][1] = x0.y; v[q][2] = x0.z; v[q][3] = x0.w;
                v[q][4] = x1.x; v[q][5] = x1.y; v[q][6] = x1.z; v[q][7] = x1.w;
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kStage; ++q) {
          const int t = t0 + q * blockDim.x;
          if (t >= ntask) continue;
          if (t < nv) {
            const int kk = t % KB, jc = t / KB;
            const uint32_t off = tc::mnmajor_off(jc * 8, kk, SBO_BV, 128);
            store_split8(sm + L.BV[0] + off, sm + L.BV[1] + off, v[q]);
          } else {
            const int u = t - nv, Lr = u % 128, kc = u / 128;
            const uint32_t off = tc::kmajor_off(Lr, kc * 8, SBO_AG, 128);
            store_split8(sm + L.AG[0] + off, sm + L.AG[1] + off, v[q]);
          }
        }
      }
    }
    tc::fence_proxy_async_smem();
    __syncthreads();
    // ---- D1 = Wbd V + G Basis   (3xBF16: hi*hi + hi*lo + lo*hi)
    if (tid == 0) {
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < KB / 16; ++s) {
        const uint32_t ao = 256u * s, bo = 256u * s;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const int ah = (p == 2), bh = (p == 1);
          const uint64_t ad = tc::make_sdesc(sm_base + L.AW[ah] + ao, 128, SBO_AW);
          const uint64_t bd = tc::make_sdesc(sm_base + L.BV[bh] + bo, 128, SBO_BV);
          tc::mma_bf16(tD1, ad, bd, id1, acc);
          acc = 1;
        }
      }
      for (int s = 0; s < kKS / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const int ah = (p == 2), bh = (p == 1);
          const uint64_t ad = tc::make_sdesc(sm_base + L.AG[ah] + 256u * s, 128, SBO_AG);
          const uint64_t bd = tc::make_sdesc(sm_base + L.BF[bh] + 256u * s, 128, SBO_F);
          tc::mma_bf16(tD1, ad, bd, id1s, 1);
        }
      }
      tc::mma_commit(&bar[0]);
    }
    tc::mbar_wait(&bar[0], phase);
    tc::fence_after_sync();
    // ---- epilogue 1: v' = GELU(D1 + b) -> global and -> AV (K-major A operand of D2)
    {
      const int q4 = warp & 3, half = warp >> 2;
      const int Lr = q4 * 32 + lane;
      const int r = Lr / WP, o = Lr % WP;
      const float bo = sbias[Lr];
      const bool valid = o < w;
      float* dst = a.vout + ((size_t)b * w + (valid ? o : 0)) * N + (size_t)(i0 + r) * n;
      for (int c0 = half * (n / 2); c0 < (half + 1) * (n / 2); c0 += 16) {
        uint32_t u[16];
        tc::tmem_ld16(tD1 + ((uint32_t)(q4 * 32) << 16) + c0, u);
        tc::tmem_wait_ld();
        float v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const float x = __uint_as_float(u[t]) + bo;
          v[t] = valid ? (a.use_gelu ? gelu_f(x) : x) : 0.f;
        }
        if (valid) {
#pragma unroll
          for (int t = 0; t < 16; t += 4)
            *reinterpret_cast<float4*>(dst + c0 + t) = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
        }
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          __nv_bfloat16 h0, l0, h1, l1;
          tc::split_bf16(v[2 * t], h0, l0);
          tc::split_bf16(v[2 * t + 1], h1, l1);
          ph[t] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
          pl[t] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
        }
        const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
        tc::tmem_st8(tAh + lane_off + c0 / 2, ph);
        tc::tmem_st8(tAl + lane_off + c0 / 2, pl);
      }
      tc::tmem_wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    // ---- D2 = v' F  (x-analysis)
    if (tid == 0) {
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < n / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const int ah = (p == 2), bh = (p == 1);
          const uint32_t at = (ah ? tAl : tAh) + 8u * s;     // 16 bf16 of K = 8 TMEM columns
          // F viewed MN-major (N = k', K = j): LBO = K-group stride = SBO_F, SBO = N-group stride = 128
          const uint64_t bd = tc::make_sdesc(sm_base + L.BF[bh] + 2u * SBO_F * s, SBO_F, 128);
          tc::mma_bf16_ts(tD2, at, bd, id2, acc);
          acc = 1;
        }
      }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], phase);
    tc::fence_after_sync();
    // ---- epilogue 2: T[b][i0+r][o][0..39] <- D2
    if (warp < 4) {
      const int Lr = warp * 32 + lane;
      const int r = Lr / WP, o = Lr % WP;
      float* dst = a.T + (((size_t)b * n + i0 + r) * w + (o < w ? o : 0)) * (2 * kModes);
#pragma unroll
      for (int c0 = 0; c0 < kKS; c0 += 16) {
        uint32_t u[16];
        tc::tmem_ld16(tD2 + ((uint32_t)(warp * 32) << 16) + c0, u);
        tc::tmem_wait_ld();
        if (o < w) {
#pragma unroll
          for (int t = 0; t < 16; t += 4)
            if (c0 + t < 2 * kModes)
              *reinterpret_cast<float4*>(dst + c0 + t) =
                  make_float4(__uint_as_float(u[t]), __uint_as_float(u[t + 1]), __uint_as_float(u[t + 2]),
                              __uint_as_float(u[t + 3]));
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    phase ^= 1;
  }
  tc::fence_after_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ------------------------------------------------------------------ y-direction transforms (CUDA cores)
// One thread = (pair of channels, kappa2) for a group of rows: each twiddle read from shared
// memory feeds two complex MACs.  Rows are split across CTAs (grid.z) for parallelism: the
// y-synthesis rows are independent; the y-analysis writes one partial per row group, summed in a
// fixed order by k_mix.
constexpr int kYO = 12;          // channel pairs per CTA -> 24 channels, 240 threads

// k_ysyn: G[b][i][o][2*k2 + {0,1}] = (re, im) of sum_k1 g[b][o][k1][k2] conj(F[i][k1]);  g carries n^-2.
__global__ void __launch_bounds__(kYO * kModes) k_ysyn(const float2* __restrict__ ghat, const float2* __restrict__ F,
                                                       float* __restrict__ G, int n, int w, int rows_per,
                                                       const int* status) {
  const int b = blockIdx.y, k2 = threadIdx.x % kModes;
  const int o0 = (blockIdx.x * kYO + threadIdx.x / kModes) * 2;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ float2 Fs[];                     // [rows_per][20]
  const int i0 = blockIdx.z * rows_per, rows = min(rows_per, n - i0);
  for (int t = threadIdx.x; t < rows * kModes; t += blockDim.x) Fs[t] = F[(size_t)i0 * kModes + t];
  float2 g0[kModes], g1[kModes];
  const bool v0 = o0 < w, v1 = o0 + 1 < w;
#pragma unroll
  for (int k1 = 0; k1 < kModes; ++k1) {
    g0[k1] = v0 ? ghat[((size_t)b * w + o0) * kModes2 + k1 * kModes + k2] : make_float2(0.f, 0.f);
    g1[k1] = v1 ? ghat[((size_t)b * w + o0 + 1) * kModes2 + k1 * kModes + k2] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  if (!v0) return;
  for (int r = 0; r < rows; r += 2) {
    float a0r = 0.f, a0i = 0.f, a1r = 0.f, a1i = 0.f, b0r = 0.f, b0i = 0.f, b1r = 0.f, b1i = 0.f;
    const bool r1 = r + 1 < rows;
#pragma unroll
    for (int k1 = 0; k1 < kModes; ++k1) {
      const float2 f = Fs[r * kModes + k1];
      const float2 h = r1 ? Fs[(r + 1) * kModes + k1] : make_float2(0.f, 0.f);
      a0r += g0[k1].x * f.x + g0[k1].y * f.y;  a0i += g0[k1].y * f.x - g0[k1].x * f.y;
      a1r += g1[k1].x * f.x + g1[k1].y * f.y;  a1i += g1[k1].y * f.x - g1[k1].x * f.y;
      b0r += g0[k1].x * h.x + g0[k1].y * h.y;  b0i += g0[k1].y * h.x - g0[k1].x * h.y;
      b1r += g1[k1].x * h.x + g1[k1].y * h.y;  b1i += g1[k1].y * h.x - g1[k1].x * h.y;
    }
    float* row0 = G + (((size_t)b * n + i0 + r) * w + o0) * (2 * kModes) + 2 * k2;
    *reinterpret_cast<float2*>(row0) = make_float2(a0r, a0i);
    if (v1) *reinterpret_cast<float2*>(row0 + 2 * kModes) = make_float2(a1r, a1i);
    if (r1) {
      float* row1 = row0 + (size_t)w * (2 * kModes);
      *reinterpret_cast<float2*>(row1) = make_float2(b0r, b0i);
      if (v1) *reinterpret_cast<float2*>(row1 + 2 * kModes) = make_float2(b1r, b1i);
    }
  }
}

// k_yan: c_part[g][kappa][b][o] = sum_{i in group g} F[i][k1] * (T[b][i][o][2 k2], T[b][i][o][2 k2 + 1])
__global__ void __launch_bounds__(kYO * kModes) k_yan(const float* __restrict__ T, const float2* __restrict__ F,
                                                      float2* __restrict__ chat, int n, int w, int B, int rows_per,
                                                      const int* status) {
  const int b = blockIdx.y, k2 = threadIdx.x % kModes, g = blockIdx.z;
  const int o0 = (blockIdx.x * kYO + threadIdx.x / kModes) * 2;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ float2 Fs[];
  const int i0 = g * rows_per, rows = min(rows_per, n - i0);
  for (int t = threadIdx.x; t < rows * kModes; t += blockDim.x) Fs[t] = F[(size_t)i0 * kModes + t];
  __syncthreads();
  const bool v0 = o0 < w, v1 = o0 + 1 < w;
  if (!v0) return;
  float2 c0[kModes], c1[kModes];
#pragma unroll
  for (int k1 = 0; k1 < kModes; ++k1) { c0[k1] = make_float2(0.f, 0.f); c1[k1] = make_float2(0.f, 0.f); }
  const size_t rstride = (size_t)w * (2 * kModes);
  const float* base = T + (((size_t)b * n + i0) * w + o0) * (2 * kModes) + 2 * k2;
  for (int r = 0; r < rows; r += 4) {
    float2 t0[4], t1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = r + q < rows;
      t0[q] = ok ? __ldg(reinterpret_cast<const float2*>(base + (r + q) * rstride)) : make_float2(0.f, 0.f);
      t1[q] = (ok && v1) ? __ldg(reinterpret_cast<const float2*>(base + (r + q) * rstride + 2 * kModes))
                         : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (r + q >= rows) break;
#pragma unroll
      for (int k1 = 0; k1 < kModes; ++k1) {
        const float2 f = Fs[(r + q) * kModes + k1];
        c0[k1].x += f.x * t0[q].x - f.y * t0[q].y;  c0[k1].y += f.x * t0[q].y + f.y * t0[q].x;
        c1[k1].x += f.x * t1[q].x - f.y * t1[q].y;  c1[k1].y += f.x * t1[q].y + f.y * t1[q].x;
      }
    }
  }
#pragma unroll
  for (int k1 = 0; k1 < kModes; ++k1) {
    float2* dst = chat + (((size_t)g * kModes2 + k1 * kModes + k2) * B + b) * w + o0;
    dst[0] = c0[k1];
    if (v1) dst[1] = c1[k1];
  }
}

// ------------------------------------------------------------------ y-direction transforms on tensor cores
// Complex products written as 2x2 real blocks (F = (Fx, Fy) = exp(-2 pi i kappa i / n)):
//   y-synthesis  G[i][(o,k2,re|im)] = sum_{(k1,p)} Fp[i][(k1,p)] * Gh[(k1,p)][(o,k2,re|im)]
//                Fp[i][(k1,0)] = Fx, Fp[i][(k1,1)] = Fy;  Gh rows (k1,0) = (gr | gi), (k1,1) = (gi | -gr)
//   y-analysis   C^T[(o,k2)][(k1,re|im)] = sum_{(i,p)} T[(o,k2)][(i,p)] * Ap[(i,p)][(k1,re|im)]
//                Ap[(i,0)][(k1,re)] = Fx, Ap[(i,1)][(k1,re)] = -Fy, Ap[(i,0)][(k1,im)] = Fy, Ap[(i,1)][(k1,im)] = Fx
constexpr int kYsynCh = 6;                 // channels per CTA: N = 6 * 40 = 240
constexpr int kYsynN = kYsynCh * 2 * kModes;

__global__ void __launch_bounds__(128, 2) k_ysyn_tc(const float2* __restrict__ ghat, const float2* __restrict__ F,
                                                    float* __restrict__ G, int n, int w, const int* status) {
  const int b = blockIdx.y, oc = blockIdx.x * kYsynCh;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(1024) unsigned char sm[];
  constexpr uint32_t SBO = (kKS / 8) * 128;             // K = 48 for both operands (K-major)
  const uint32_t A0 = 0, A1 = 128 * kKS * 2, B0 = 2 * A1, B1 = B0 + kYsynN * kKS * 2, BAR = B1 + kYsynN * kKS * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + BAR + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) { tc::mbar_init(bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(tptr, 256);
  // A = Fp (rows i < n), K-major
  for (int t = tid; t < 128 * (kKS / 8); t += blockDim.x) {
    const int i = t % 128, kc = t / 128;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = kc * 8 + q, k1 = k >> 1;
      v[q] = 0.f;
      if (i < n && k1 < kModes) { const float2 f = F[(size_t)i * kModes + k1]; v[q] = (k & 1) ? f.y : f.x; }
    }
    const uint32_t off = tc::kmajor_off(i, kc * 8, SBO, 128);
    store_split8(sm + A0 + off, sm + A1 + off, v);
  }
  // B = Gh for channels [oc, oc+6): row nn = (ol*20 + k2)*2 + pout, K = (k1, pin), K-major
  for (int t = tid; t < (kYsynN / 2) * (kKS / 8); t += blockDim.x) {
    const int m = t % (kYsynN / 2), kc = t / (kYsynN / 2);
    const int ol = m / kModes, k2 = m % kModes, o = oc + ol;
    float vr[8], vi[8];                                 // pout = re / im rows
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k1 = kc * 4 + q;
      float2 g = make_float2(0.f, 0.f);
      if (o < w && k1 < kModes) g = ghat[((size_t)b * w + o) * kModes2 + k1 * kModes + k2];
      vr[2 * q] = g.x;  vr[2 * q + 1] = g.y;           // (k1,0): gr ; (k1,1): gi
      vi[2 * q] = g.y;  vi[2 * q + 1] = -g.x;          // (k1,0): gi ; (k1,1): -gr
    }
    const uint32_t offr = tc::kmajor_off(2 * m, kc * 8, SBO, 128), offi = tc::kmajor_off(2 * m + 1, kc * 8, SBO, 128);
    store_split8(sm + B0 + offr, sm + B1 + offr, vr);
    store_split8(sm + B0 + offi, sm + B1 + offi, vi);
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  if (tid == 0) {
    const uint32_t id = tc::make_idesc_bf16(128, kYsynN, false, false);
    const uint32_t base = tc::smem_u32(sm);
    uint32_t acc = 0;
    for (int s = 0; s < kKS / 16; ++s)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t aa = base + (p == 2 ? A1 : A0) + 256u * s, bb = base + (p == 1 ? B1 : B0) + 256u * s;
        tc::mma_bf16(tmem, tc::make_sdesc(aa, 128, SBO), tc::make_sdesc(bb, 128, SBO), id, acc);
        acc = 1;
      }
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after_sync();
  const int i = warp * 32 + lane;
  for (int ol = 0; ol < kYsynCh; ++ol) {
#pragma unroll
    for (int c = 0; c < 2 * kModes; c += 8) {
      uint32_t u[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + ol * 2 * kModes + c));
      tc::tmem_wait_ld();
      const int o = oc + ol;
      if (i < n && o < w) {
        float4* dst = reinterpret_cast<float4*>(G + (((size_t)b * n + i) * w + o) * (2 * kModes) + c);
        dst[0] = make_float4(__uint_as_float(u[0]), __uint_as_float(u[1]), __uint_as_float(u[2]), __uint_as_float(u[3]));
        dst[1] = make_float4(__uint_as_float(u[4]), __uint_as_float(u[5]), __uint_as_float(u[6]), __uint_as_float(u[7]));
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

constexpr int kYanN = kKS;                 // (k1, re|im) = 40 padded to 48

__global__ void __launch_bounds__(256, 1) k_yan_tc(const float* __restrict__ T, const float2* __restrict__ F,
                                                   float2* __restrict__ chat, int n, int w, int B, const int* status) {
  const int b = blockIdx.y, m0 = blockIdx.x * 128;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int K = 2 * n;
  const uint32_t SBO_A = (K / 8) * 128, SBO_B = (K / 8) * 128;
  const uint32_t A0 = 0, A1 = 128 * K * 2, B0 = 2 * A1, B1 = B0 + kYanN * K * 2, BAR = B1 + kYanN * K * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + BAR + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = w * kModes;                             // rows (o, k2)
  if (tid == 0) { tc::mbar_init(bar, 1); tc::fence_mbar_init(); }
  if (warp == 0) tc::tmem_alloc(tptr, 64);
  // B = Ap^T: row nn = (k1, pout), K = (i, pin), K-major
  for (int t = tid; t < kYanN * (K / 8); t += blockDim.x) {
    const int nn = t % kYanN, kc = t / kYanN, k1 = nn >> 1, pout = nn & 1;
    float v[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = kc * 4 + q;
      float2 f = make_float2(0.f, 0.f);
      if (k1 < kModes) f = F[(size_t)i * kModes + k1];
      v[2 * q] = pout ? f.y : f.x;            // pin = re
      v[2 * q + 1] = pout ? f.x : -f.y;       // pin = im
    }
    const uint32_t off = tc::kmajor_off(nn, kc * 8, SBO_B, 128);
    store_split8(sm + B0 + off, sm + B1 + off, v);
  }
  // A = T rows m = (o, k2), K = (i, pin): 4 rows i per 16-byte chunk
  const float* Tb = T + (size_t)b * n * w * (2 * kModes);
  const size_t rstride = (size_t)w * (2 * kModes);
  for (int t0 = tid; t0 < 128 * (K / 8); t0 += 4 * blockDim.x) {
    float v[4][8];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const int t = t0 + z * blockDim.x;
      const int m = t % 128, kc = t / 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) v[z][q] = 0.f;
      if (t < 128 * (K / 8) && m0 + m < M) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 x = __ldg(reinterpret_cast<const float2*>(Tb + (size_t)(kc * 4 + q) * rstride + (size_t)(m0 + m) * 2));
          v[z][2 * q] = x.x; v[z][2 * q + 1] = x.y;
        }
      }
    }
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const int t = t0 + z * blockDim.x;
      if (t >= 128 * (K / 8)) break;
      const int m = t % 128, kc = t / 128;
      const uint32_t off = tc::kmajor_off(m, kc * 8, SBO_A, 128);
      store_split8(sm + A0 + off, sm + A1 + off, v[z]);
    }
  }
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  if (tid == 0) {
    const uint32_t id = tc::make_idesc_bf16(128, kYanN, false, false);
    const uint32_t base = tc::smem_u32(sm);
    uint32_t acc = 0;
    for (int s = 0; s < K / 16; ++s)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t aa = base + (p == 2 ? A1 : A0) + 256u * s, bb = base + (p == 1 ? B1 : B0) + 256u * s;
        tc::mma_bf16(tmem, tc::make_sdesc(aa, 128, SBO_A), tc::make_sdesc(bb, 128, SBO_B), id, acc);
        acc = 1;
      }
    tc::mma_commit(bar);
  }
  tc::mbar_wait(bar, 0);
  tc::fence_after_sync();
  if (warp < 4) {
    const int m = m0 + warp * 32 + lane;
    const int o = m / kModes, k2 = m % kModes;
#pragma unroll
    for (int c = 0; c < 2 * kModes; c += 8) {
      uint32_t u[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
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
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

static size_t ysyn_tc_smem() { return (size_t)2 * 128 * kKS * 2 + (size_t)2 * kYsynN * kKS * 2 + 64; }
static size_t yan_tc_smem(int n) { return (size_t)2 * 128 * (2 * n) * 2 + (size_t)2 * kYanN * (2 * n) * 2 + 64; }

// ------------------------------------------------------------------ host side
bool tc_layer_supported(int n, int w) {
  if (w > 128 || n % 16 != 0 || n < 64 || n > 256) return false;
  const int WP = w <= 32 ? 32 : (w <= 64 ? 64 : 128);
  const int R = 128 / WP;
  if (n % R) return false;
  int optin = 0, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  return TcSmem(n, w, WP).total <= (uint32_t)optin;
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
  cudaError_t e = cudaFuncSetAttribute((const void*)k_tc_layer<WP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void*)k_tc_layer<WP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
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
  done = true;
  return cudaSuccess;
}

cudaError_t launch_tc_layer(const TcLayerArgsHost& h, cudaStream_t s) {
  TcLayerArgs a{};
  a.n = h.n; a.N = h.n * h.n; a.w = h.w; a.cin = h.cin; a.B = h.B; a.use_gelu = h.use_gelu;
  a.r = h.r; a.rr = h.rr; a.k = h.k; a.vin = h.vin; a.W = h.W; a.bias = h.bias; a.G = h.G;
  a.F = reinterpret_cast<const float2*>(h.F); a.vout = h.vout; a.T = h.T; a.status = h.status;
  const int WP = h.w <= 32 ? 32 : (h.w <= 64 ? 64 : 128);
  const int R = 128 / WP;
  const int ntiles = h.B * (h.n / R);
  const size_t smem = TcSmem(h.n, h.cin, WP).total;
  // persistent grid: as many CTAs as fit per SM by shared memory (<= 2) and TMEM columns
  const uint32_t need_cols = (uint32_t)h.n + 64u + (uint32_t)h.n;
  const int by_tmem = need_cols <= 256 ? 2 : 1;
  const int by_smem = (int)((228u * 1024u) / (smem + 1024u));
  const int per_sm = std::max(1, std::min(by_tmem, std::min(by_smem, 2)));
  const int grid = std::min(ntiles, per_sm * num_sms());
  if (WP == 32) {
    if (h.first) k_tc_layer<32, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<32, false><<<grid, kTcThreads, smem, s>>>(a);
  } else if (WP == 64) {
    if (h.first) k_tc_layer<64, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<64, false><<<grid, kTcThreads, smem, s>>>(a);
  } else {
    if (h.first) k_tc_layer<128, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<128, false><<<grid, kTcThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

// Row groups so that the grid covers the SMs ~4 times (at most kMaxYParts, at least 8 rows each).
int yan_parts(int n, int w, int B) {
  if (n <= 128) return 1;   // tensor-core y-analysis (k_yan_tc) writes the full sum
  const int wc = (w + 2 * kYO - 1) / (2 * kYO);
  int p = (4 * num_sms() + wc * B - 1) / (wc * B);
  p = std::max(1, std::min(p, std::min(kMaxYParts, n / 8)));
  return p;
}

cudaError_t launch_ysyn(const float* ghat, const float* F, float* G, int n, int w, int B, const int* status,
                        cudaStream_t s) {
  if (n <= 128) {
    k_ysyn_tc<<<dim3((w + kYsynCh - 1) / kYsynCh, B), 128, ysyn_tc_smem(), s>>>(
        reinterpret_cast<const float2*>(ghat), reinterpret_cast<const float2*>(F), G, n, w, status);
    return cudaGetLastError();
  }
  const int parts = yan_parts(n, w, B), rows_per = (n + parts - 1) / parts;
  k_ysyn<<<dim3((w + 2 * kYO - 1) / (2 * kYO), B, parts), kYO * kModes, rows_per * kModes * sizeof(float2), s>>>(
      reinterpret_cast<const float2*>(ghat), reinterpret_cast<const float2*>(F), G, n, w, rows_per, status);
  return cudaGetLastError();
}

cudaError_t launch_yan(const float* T, const float* F, float* chat, int n, int w, int B, int nparts, const int* status,
                       cudaStream_t s) {
  if (nparts == 1 && n <= 128) {
    k_yan_tc<<<dim3((w * kModes + 127) / 128, B), 256, yan_tc_smem(n), s>>>(
        T, reinterpret_cast<const float2*>(F), reinterpret_cast<float2*>(chat), n, w, B, status);
    return cudaGetLastError();
  }
  const int rows_per = (n + nparts - 1) / nparts;
  k_yan<<<dim3((w + 2 * kYO - 1) / (2 * kYO), B, nparts), kYO * kModes, rows_per * kModes * sizeof(float2), s>>>(
      T, reinterpret_cast<const float2*>(F), reinterpret_cast<float2*>(chat), n, w, B, rows_per, status);
  return cudaGetLastError();
}

}  // namespace fcgno

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
  uint32_t AW[2], BV[2], AG[2], BF[2], AV[2], bar, tptr, bias, total;
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
    for (int h = 0; h < 2; ++h) AV[h] = take(128u * n * 2);
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
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_layer(const TcLayerArgs a) {
  constexpr int R = TcShape<WP>::R;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = a.N, w = a.w, cin = a.cin;
  const TcSmem L(n, cin, WP);
  const int KB = L.KB, CP = L.CP;
  const uint32_t SBO_AW = (KB / 8) * 128, SBO_BV = (KB / 8) * 128, SBO_AG = (kKS / 8) * 128,
                 SBO_F = (kKS / 8) * 128, SBO_AV = (n / 8) * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t ncols = (n + kKS) <= 128 ? 128u : ((n + kKS) <= 256 ? 256u : 512u);

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
    for (int t = tid; t < KB * (n / 8); t += blockDim.x) {
      const int kk = t % KB, jc = t / KB;
      const int rp = kk / CP, c = kk % CP;
      float v[8];
      if (rp < R && c < cin) {
        const size_t e = (size_t)(i0 + rp) * n + jc * 8;
        if (FIRST) {
          const double* src = (c == 0 ? a.r : a.k) + (size_t)b * N + e;
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (float)(c == 0 ? src[q] * inv_s : src[q]);
        } else {
          const float4* src = reinterpret_cast<const float4*>(a.vin + ((size_t)b * cin + c) * N + e);
          const float4 x0 = src[0], x1 = src[1];
          v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w; v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0.f;
      }
      const uint32_t off = tc::mnmajor_off(jc * 8, kk, SBO_BV, 128);
      store_split8(sm + L.BV[0] + off, sm + L.BV[1] + off, v);
    }
    for (int t = tid; t < 128 * (kKS / 8); t += blockDim.x) {
      const int Lr = t % 128, kc = t / 128;
      const int r = Lr / WP, o = Lr % WP;
      float v[8];
      if (o < w) {
        const float* src = a.G + (((size_t)b * n + i0 + r) * w + o) * (2 * kModes) + kc * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (kc * 8 + q < 2 * kModes) ? src[q] : 0.f;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0.f;
      }
      const uint32_t off = tc::kmajor_off(Lr, kc * 8, SBO_AG, 128);
      store_split8(sm + L.AG[0] + off, sm + L.AG[1] + off, v);
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
        float v8[8];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
          for (int t = 0; t < 8; ++t) v8[t] = v[hh * 8 + t];
          const uint32_t off = tc::kmajor_off(Lr, c0 + hh * 8, SBO_AV, 128);
          store_split8(sm + L.AV[0] + off, sm + L.AV[1] + off, v8);
        }
      }
    }
    tc::fence_proxy_async_smem();
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
          const uint64_t ad = tc::make_sdesc(sm_base + L.AV[ah] + 256u * s, 128, SBO_AV);
          // F viewed MN-major (N = k', K = j): LBO = K-group stride = SBO_F, SBO = N-group stride = 128
          const uint64_t bd = tc::make_sdesc(sm_base + L.BF[bh] + 2u * SBO_F * s, SBO_F, 128);
          tc::mma_bf16(tD2, ad, bd, id2, acc);
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
// k_ysyn: G[b][i][o][2*k2 + {0,1}] = (re, im) of sum_k1 g[b][o][k1][k2] conj(F[i][k1]);  g already carries n^-2.
// grid (ceil(w / 12), B), 240 threads = 12 channels x 20 kappa2.
constexpr int kYO = 12;
__global__ void __launch_bounds__(kYO * kModes) k_ysyn(const float2* __restrict__ ghat, const float2* __restrict__ F,
                                                       float* __restrict__ G, int n, int w, const int* status) {
  const int b = blockIdx.y, o = blockIdx.x * kYO + threadIdx.x / kModes, k2 = threadIdx.x % kModes;
  if (status && status[b] != SYS_RUNNING) return;
  __shared__ float2 Fs[64 * kModes];
  float2 g[kModes];
  const bool valid = o < w;
#pragma unroll
  for (int k1 = 0; k1 < kModes; ++k1)
    g[k1] = valid ? ghat[((size_t)b * w + o) * kModes2 + k1 * kModes + k2] : make_float2(0.f, 0.f);
  for (int i0 = 0; i0 < n; i0 += 64) {
    const int rows = min(64, n - i0);
    __syncthreads();
    for (int t = threadIdx.x; t < rows * kModes; t += blockDim.x) Fs[t] = F[(size_t)i0 * kModes + t];
    __syncthreads();
    if (valid) {
      for (int r = 0; r < rows; ++r) {
        float gr = 0.f, gi = 0.f;
#pragma unroll
        for (int k1 = 0; k1 < kModes; ++k1) {
          const float2 f = Fs[r * kModes + k1];
          gr += g[k1].x * f.x + g[k1].y * f.y;
          gi += g[k1].y * f.x - g[k1].x * f.y;
        }
        *reinterpret_cast<float2*>(G + (((size_t)b * n + i0 + r) * w + o) * (2 * kModes) + 2 * k2) = make_float2(gr, gi);
      }
    }
  }
}

// k_yan: c[kappa][b][o] = sum_i F[i][k1] * (T[b][i][o][2 k2], T[b][i][o][2 k2 + 1])   (complex)
__global__ void __launch_bounds__(kYO * kModes) k_yan(const float* __restrict__ T, const float2* __restrict__ F,
                                                      float2* __restrict__ chat, int n, int w, int B,
                                                      const int* status) {
  const int b = blockIdx.y, o = blockIdx.x * kYO + threadIdx.x / kModes, k2 = threadIdx.x % kModes;
  if (status && status[b] != SYS_RUNNING) return;
  __shared__ float2 Fs[64 * kModes];
  float2 acc[kModes];
#pragma unroll
  for (int k1 = 0; k1 < kModes; ++k1) acc[k1] = make_float2(0.f, 0.f);
  const bool valid = o < w;
  for (int i0 = 0; i0 < n; i0 += 64) {
    const int rows = min(64, n - i0);
    __syncthreads();
    for (int t = threadIdx.x; t < rows * kModes; t += blockDim.x) Fs[t] = F[(size_t)i0 * kModes + t];
    __syncthreads();
    if (valid) {
      for (int r = 0; r < rows; ++r) {
        const float2 t2 = *reinterpret_cast<const float2*>(T + (((size_t)b * n + i0 + r) * w + o) * (2 * kModes) + 2 * k2);
#pragma unroll
        for (int k1 = 0; k1 < kModes; ++k1) {
          const float2 f = Fs[r * kModes + k1];
          acc[k1].x += f.x * t2.x - f.y * t2.y;
          acc[k1].y += f.x * t2.y + f.y * t2.x;
        }
      }
    }
  }
  if (valid)
#pragma unroll
    for (int k1 = 0; k1 < kModes; ++k1) chat[((size_t)(k1 * kModes + k2) * B + b) * w + o] = acc[k1];
}

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
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  const size_t smem = TcSmem(h.n, h.cin, WP).total;
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

cudaError_t launch_ysyn(const float* ghat, const float* F, float* G, int n, int w, int B, const int* status,
                        cudaStream_t s) {
  k_ysyn<<<dim3((w + kYO - 1) / kYO, B), kYO * kModes, 0, s>>>(reinterpret_cast<const float2*>(ghat),
                                                               reinterpret_cast<const float2*>(F), G, n, w, status);
  return cudaGetLastError();
}

cudaError_t launch_yan(const float* T, const float* F, float* chat, int n, int w, int B, const int* status,
                       cudaStream_t s) {
  k_yan<<<dim3((w + kYO - 1) / kYO, B), kYO * kModes, 0, s>>>(T, reinterpret_cast<const float2*>(F),
                                                              reinterpret_cast<float2*>(chat), n, w, B, status);
  return cudaGetLastError();
}

}  // namespace fcgno

// no_tc_kernels.cu — tensor-core (tcgen05 / TMEM) SNO layers for the fp32 NO path.
//
// One layer (R7-R11) is
//   u[o][i][j] = sum_c W[o][c] v[c][i][j] + b[o] + n^-2 Re sum_kappa g[o](kappa) e^{+2 pi i kappa.(i,j)/n}
//   v'         = GELU(u)                                    (layers 1-3; layer 4 is folded away)
//   c'[o](k)   = sum_{i,j} v'[o][i][j] e^{-2 pi i k.(i,j)/n}
// The DFTs are separable; every contraction is a dense GEMM on the 5th-gen tensor cores:
//
//   k_ysyn_tc   per (system, 6 channels): G[i][(o,k')] = Fp[i][(k1,p)] . Gh[(k1,p)][(o,k')]          (y-synthesis)
//   k_tc_layer  tile = R rows of one system; TMEM lanes = (row r, padded channel o), R * WP = 128
//     D1[(r,o)][j]  = sum_{(r',c)} Wbd[(r,o)][(r',c)] V[(r',c)][j]      bypass, block-diagonal in r
//                   + sum_{k'} G[(r,o)][k'] Basis[k'][j]                 x-synthesis (k' = (kappa2, re|im))
//     epilogue      v' = GELU(D1 + b) -> next layer's V blob, and into TMEM (A operand of D2)
//     D2[(r,o)][k'] = sum_j v'[(r,o)][j] F[j][k']                        x-analysis
//     epilogue      -> T blob
//   k_yan_tc    per (system, 128 (o,kappa2) rows): C^T[(o,k2)][(k1,p)] = T[(o,k2)][(i,p')] . Ap[(i,p')][(k1,p)]
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

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// 8 consecutive values -> 16 bytes of bf16 hi and 16 bytes of bf16 lo in shared memory
__device__ __forceinline__ void store_split8(unsigned char* hi, unsigned char* lo, const float (&v)[8]) {
  uint4 h, l;
  tc::split8(v, h, l);
  *reinterpret_cast<uint4*>(hi) = h;
  *reinterpret_cast<uint4*>(lo) = l;
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&u)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "r"(taddr));
}

// ------------------------------------------------------------------ k_tc_layer
struct TcSmem {
  // byte offsets; every region 1024-aligned; BV/AG hold [hi][lo] back to back like their blobs
  uint32_t AW[2], BV, AG, BF[2], bar, tptr, bias, total;
  int KB, CP;
  __host__ __device__ TcSmem(const TcGeom& g, int cin) {
    CP = (cin + 7) & ~7;
    KB = (g.R * CP + 15) & ~15;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t at = o; o = (o + bytes + 1023) & ~1023u; return at; };
    for (int h = 0; h < 2; ++h) AW[h] = take(128u * KB * 2);
    BV = take(2u * (uint32_t)g.n * KB * 2);
    AG = take(2u * g.g_half());
    for (int h = 0; h < 2; ++h) BF[h] = take((uint32_t)g.n * kKS * 2);
    bar = take(64);
    tptr = bar + 32;
    bias = take(128 * 4);
    total = o;
  }
};

struct TcLayerArgs {
  int n, w, cin, B, use_gelu;
  const double* r; const double* rr; const double* k;   // layer 1 inputs
  const unsigned char* vin;                              // V blobs (layers 2, 3)
  const float* W;                                        // [w][cin]
  const float* bias;                                     // [w]
  const unsigned char* G;                                // G blobs
  const float2* F;                                       // [n][20]
  unsigned char* vout;                                   // V blobs of the next layer
  unsigned char* T;                                      // T blobs
  const int* status;
};

template <int WP, bool FIRST>
__global__ void __launch_bounds__(kTcThreads, 2) k_tc_layer(const TcLayerArgs a) {
  const TcGeom g(a.n, a.w);
  constexpr int R = 128 / WP;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int n = a.n, N = n * n, w = a.w, cin = a.cin;
  const TcSmem L(g, cin);
  const int KB = L.KB, CP = L.CP;                     // of this layer's input (FIRST: cin = 2)
  const uint32_t SBO_AW = (KB / 8) * 128, SBO_BV = (KB / 8) * 128, SBO_AG = g.g_sbo(), SBO_F = (kKS / 8) * 128;
  const uint32_t vout_half = g.v_half(), vout_sbo = g.v_sbo();   // next layer's V blob geometry (cin = w)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L.bar);   // [0] loads, [1] D1, [2] D2
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + L.tptr);
  float* sbias = reinterpret_cast<float*>(sm + L.bias);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t need = (uint32_t)n + 64u + (uint32_t)n;
  const uint32_t ncols = need <= 128 ? 128u : (need <= 256 ? 256u : 512u);
  const int ntiles = a.B * g.tiles_per_sys;
  auto running = [&](int t) { return !a.status || a.status[t / g.tiles_per_sys] == SYS_RUNNING; };
  auto next_tile = [&](int t) {
    while (t < ntiles && !running(t)) t += gridDim.x;
    return t;
  };
  const uint32_t in_bytes = FIRST ? 2u * g.g_half() : 2u * (uint32_t)KB * n * 2 + 2u * g.g_half();
  auto prefetch = [&](int t) {   // one thread: bulk copies of tile t's blobs
    tc::mbar_expect_tx(&bar[0], in_bytes);
    if (!FIRST) tc::bulk_g2s(sm + L.BV, a.vin + (size_t)t * 2 * KB * n * 2, 2u * KB * n * 2, &bar[0]);
    tc::bulk_g2s(sm + L.AG, a.G + (size_t)t * 2 * g.g_half(), 2u * g.g_half(), &bar[0]);
  };

  // ---- one-time setup: barriers, TMEM, block-diagonal weights, twiddle operand, bias
  int tile = next_tile(blockIdx.x);
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) tc::mbar_init(&bar[q], 1);
    tc::fence_mbar_init();
    if (tile < ntiles) prefetch(tile);
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
      v[q] = 0.f;
      if (kp < 2 * kModes) {
        const float2 f = a.F[(size_t)j * kModes + (kp >> 1)];
        v[q] = (kp & 1) ? f.y : f.x;
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

  uint32_t ph = 0;
  for (; tile < ntiles; tile = next_tile(tile + gridDim.x)) {
    const int b = tile / g.tiles_per_sys, i0 = (tile % g.tiles_per_sys) * R;
    if (FIRST) {   // layer 1: V = [r/||r||, k] converted from fp64 in the block
      const double s = sqrt(a.rr[b]);
      const double inv_s = s > 0.0 ? 1.0 / s : 0.0;
      for (int t = tid; t < KB * (n / 8); t += blockDim.x) {
        const int kk = t % KB, jc = t / KB;
        const int rp = kk / CP, c = kk % CP;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0.f;
        if (rp < R && c < cin) {
          const double* src = (c == 0 ? a.r : a.k) + (size_t)b * N + (size_t)(i0 + rp) * n + jc * 8;
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (float)(c == 0 ? src[q] * inv_s : src[q]);
        }
        const uint32_t off = tc::mnmajor_off(jc * 8, kk, SBO_BV, 128);
        store_split8(sm + L.BV + off, sm + L.BV + (uint32_t)KB * n * 2 + off, v);
      }
      tc::fence_proxy_async_smem();
      __syncthreads();
    }
    // ---- D1 = Wbd V + G Basis   (3xBF16: hi*hi + hi*lo + lo*hi)
    if (tid == 0) {
      tc::mbar_wait(&bar[0], ph);
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < KB / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t ao = L.AW[p == 2] + 256u * s, bo = L.BV + (p == 1 ? (uint32_t)KB * n * 2 : 0u) + 256u * s;
          tc::mma_bf16(tD1, tc::make_sdesc(sm_base + ao, 128, SBO_AW), tc::make_sdesc(sm_base + bo, 128, SBO_BV), id1, acc);
          acc = 1;
        }
      }
      for (int s = 0; s < kKS / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t ao = L.AG + (p == 2 ? g.g_half() : 0u) + 256u * s, bo = L.BF[p == 1] + 256u * s;
          tc::mma_bf16(tD1, tc::make_sdesc(sm_base + ao, 128, SBO_AG), tc::make_sdesc(sm_base + bo, 128, SBO_F), id1s, 1);
        }
      }
      tc::mma_commit(&bar[1]);
    }
    tc::mbar_wait(&bar[1], ph);
    tc::fence_after_sync();
    // the MMAs have consumed BV / AG: prefetch the next tile while the epilogues run
    if (tid == 0) {
      const int tn = next_tile(tile + gridDim.x);
      if (tn < ntiles) prefetch(tn);
    }
    // ---- epilogue 1: v' = GELU(D1 + b) -> next V blob (bf16 hi/lo) and -> TMEM (A operand of D2)
    {
      const int q4 = warp & 3, half = warp >> 2;
      const int Lr = q4 * 32 + lane;
      const int r = Lr / WP, o = Lr % WP;
      const float bo = sbias[Lr];
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
        if (store) {
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
    // ---- D2 = v' F  (x-analysis)
    if (tid == 0) {
      tc::fence_after_sync();
      uint32_t acc = 0;
      for (int s = 0; s < n / 16; ++s) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const uint32_t at = (p == 2 ? tAl : tAh) + 8u * s;     // 16 bf16 of K = 8 TMEM columns
          // F viewed MN-major (N = k', K = j): LBO = K-group stride = SBO_F, SBO = N-group stride = 128
          const uint64_t bd = tc::make_sdesc(sm_base + L.BF[p == 1] + 2u * SBO_F * s, SBO_F, 128);
          tc::mma_bf16_ts(tD2, at, bd, id2, acc);
          acc = 1;
        }
      }
      tc::mma_commit(&bar[2]);
    }
    tc::mbar_wait(&bar[2], ph);
    tc::fence_after_sync();
    // ---- epilogue 2: D2 -> T blob: row m = (o, k2), K = (i, re|im) -> one 4-byte hi and lo word per k2
    {
      const int q4 = warp & 3, half = warp >> 2;
      const int Lr = q4 * 32 + lane;
      const int r = Lr / WP, o = Lr % WP;
      const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
      const int kcol = 2 * (i0 + r);
      const uint32_t t_half = g.t_half(), t_sbo = g.t_sbo();
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) {               // columns [24*half, 24*half + 24) in chunks of 8 (< 40)
        const int c0 = half * 24 + cc * 8;
        if (c0 >= 2 * kModes) break;
        uint32_t u[8];
        tmem_ld8(tD2 + lane_off + c0, u);
        tc::tmem_wait_ld();
        if (o < w) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k2 = c0 / 2 + q, m = o * kModes + k2;
            uint32_t hi, lo;
            tc::split2(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1]), hi, lo);
            unsigned char* tb = a.T + ((size_t)b * g.mtiles + m / 128) * 2 * t_half;
            const uint32_t off = tc::kmajor_off(m % 128, kcol, t_sbo, 128);
            *reinterpret_cast<uint32_t*>(tb + off) = hi;
            *reinterpret_cast<uint32_t*>(tb + t_half + off) = lo;
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

// ------------------------------------------------------------------ y-direction transforms on tensor cores
// Complex products written as 2x2 real blocks (F = (Fx, Fy) = exp(-2 pi i kappa i / n)):
//   y-synthesis  G[i][(o,k2,re|im)] = sum_{(k1,p)} Fp[i][(k1,p)] * Gh[(k1,p)][(o,k2,re|im)]
//                Fp[i][(k1,0)] = Fx, Fp[i][(k1,1)] = Fy;  Gh rows (k1,0) = (gr | gi), (k1,1) = (gi | -gr)
//   y-analysis   C^T[(o,k2)][(k1,re|im)] = sum_{(i,p)} T[(o,k2)][(i,p)] * Ap[(i,p)][(k1,re|im)]
//                Ap[(i,0)][(k1,re)] = Fx, Ap[(i,1)][(k1,re)] = -Fy, Ap[(i,0)][(k1,im)] = Fy, Ap[(i,1)][(k1,im)] = Fx
constexpr int kYsynCh = 6;                 // channels per CTA: N = 6 * 40 = 240
constexpr int kYsynN = kYsynCh * 2 * kModes;

__global__ void __launch_bounds__(128, 2) k_ysyn_tc(const float2* __restrict__ ghat, const float2* __restrict__ F,
                                                    unsigned char* __restrict__ Gb, int n, int w, const int* status) {
  const TcGeom geo(n, w);
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
  for (int t = tid; t < 128 * (kKS / 8); t += blockDim.x) {     // A = Fp (rows i < n), K-major
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
  for (int t = tid; t < (kYsynN / 2) * (kKS / 8); t += blockDim.x) {   // B = Gh, rows (ol, k2, pout)
    const int m = t % (kYsynN / 2), kc = t / (kYsynN / 2);
    const int ol = m / kModes, k2 = m % kModes, o = oc + ol;
    float vr[8], vi[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k1 = kc * 4 + q;
      float2 gg = make_float2(0.f, 0.f);
      if (o < w && k1 < kModes) gg = ghat[((size_t)b * w + o) * kModes2 + k1 * kModes + k2];
      vr[2 * q] = gg.x;  vr[2 * q + 1] = gg.y;
      vi[2 * q] = gg.y;  vi[2 * q + 1] = -gg.x;
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
  // epilogue: lane = row i -> G blob of tile (b, i / R), row Lr = (i % R, o), 16-byte hi/lo chunks of k'
  const int i = warp * 32 + lane;
  const uint32_t gh = geo.g_half(), gs = geo.g_sbo();
  unsigned char* gt = Gb + ((size_t)b * geo.tiles_per_sys + (i < n ? i / geo.R : 0)) * 2 * gh;
  for (int ol = 0; ol < kYsynCh; ++ol) {
    const int o = oc + ol;
    const uint32_t Lr = (uint32_t)((i % geo.R) * geo.WP + o);
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
        const uint32_t off = tc::kmajor_off(Lr, c, gs, 128);
        *reinterpret_cast<uint4*>(gt + off) = h;
        *reinterpret_cast<uint4*>(gt + gh + off) = l;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

constexpr int kYanN = kKS;                 // (k1, re|im) = 40 padded to 48

__global__ void __launch_bounds__(128, 2) k_yan_tc(const unsigned char* __restrict__ Tb, const float2* __restrict__ F,
                                                   float2* __restrict__ chat, int n, int w, int B, const int* status) {
  const TcGeom geo(n, w);
  const int b = blockIdx.y, mt = blockIdx.x, m0 = mt * 128;
  if (status && status[b] != SYS_RUNNING) return;
  extern __shared__ __align__(1024) unsigned char sm[];
  const int K = 2 * n;
  const uint32_t SBO_A = geo.t_sbo(), SBO_B = (K / 8) * 128, th = geo.t_half();
  const uint32_t A0 = 0, B0 = 2 * th, B1 = B0 + kYanN * K * 2, BAR = B1 + kYanN * K * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR);     // [0] load, [1] MMA
  uint32_t* tptr = reinterpret_cast<uint32_t*>(sm + BAR + 16);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = w * kModes;
  if (tid == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&bar[0], 2 * th);
    tc::bulk_g2s(sm + A0, Tb + ((size_t)b * geo.mtiles + mt) * 2 * th, 2 * th, &bar[0]);
  }
  if (warp == 0) tc::tmem_alloc(tptr, 64);
  for (int t = tid; t < kYanN * (K / 8); t += blockDim.x) {     // B = Ap^T: row (k1, pout), K = (i, pin)
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
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tptr;
  if (tid == 0) {
    tc::mbar_wait(&bar[0], 0);
    tc::fence_after_sync();
    const uint32_t id = tc::make_idesc_bf16(128, kYanN, false, false);
    const uint32_t base = tc::smem_u32(sm);
    uint32_t acc = 0;
    for (int s = 0; s < K / 16; ++s)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint32_t aa = base + A0 + (p == 2 ? th : 0u) + 256u * s, bb = base + (p == 1 ? B1 : B0) + 256u * s;
        tc::mma_bf16(tmem, tc::make_sdesc(aa, 128, SBO_A), tc::make_sdesc(bb, 128, SBO_B), id, acc);
        acc = 1;
      }
    tc::mma_commit(&bar[1]);
  }
  tc::mbar_wait(&bar[1], 0);
  tc::fence_after_sync();
  {
    const int m = m0 + warp * 32 + lane;
    const int o = m / kModes, k2 = m % kModes;
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
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

static size_t ysyn_tc_smem() { return (size_t)2 * 128 * kKS * 2 + (size_t)2 * kYsynN * kKS * 2 + 64; }
static size_t yan_tc_smem(int n) { return (size_t)2 * 128 * (2 * n) * 2 + (size_t)2 * kYanN * (2 * n) * 2 + 64; }

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
  a.n = h.n; a.w = h.w; a.cin = h.cin; a.B = h.B; a.use_gelu = h.use_gelu;
  a.r = h.r; a.rr = h.rr; a.k = h.k; a.vin = h.vin; a.W = h.W; a.bias = h.bias; a.G = h.G;
  a.F = reinterpret_cast<const float2*>(h.F); a.vout = h.vout; a.T = h.T; a.status = h.status;
  const TcGeom g(h.n, h.w);
  const int ntiles = h.B * g.tiles_per_sys;
  const size_t smem = TcSmem(g, h.cin).total;
  // persistent grid: as many CTAs as fit per SM by shared memory (<= 2) and TMEM columns
  const uint32_t need_cols = (uint32_t)h.n + 64u + (uint32_t)h.n;
  const int by_tmem = need_cols <= 256 ? 2 : 1;
  const int by_smem = (int)((228u * 1024u) / (smem + 1024u));
  const int per_sm = std::max(1, std::min(by_tmem, std::min(by_smem, 2)));
  const int grid = std::min(ntiles, per_sm * num_sms());
  if (g.WP == 32) {
    if (h.first) k_tc_layer<32, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<32, false><<<grid, kTcThreads, smem, s>>>(a);
  } else if (g.WP == 64) {
    if (h.first) k_tc_layer<64, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<64, false><<<grid, kTcThreads, smem, s>>>(a);
  } else {
    if (h.first) k_tc_layer<128, true><<<grid, kTcThreads, smem, s>>>(a);
    else k_tc_layer<128, false><<<grid, kTcThreads, smem, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_ysyn(const float* ghat, const float* F, unsigned char* Gb, int n, int w, int B, const int* status,
                        cudaStream_t s) {
  k_ysyn_tc<<<dim3((w + kYsynCh - 1) / kYsynCh, B), 128, ysyn_tc_smem(), s>>>(
      reinterpret_cast<const float2*>(ghat), reinterpret_cast<const float2*>(F), Gb, n, w, status);
  return cudaGetLastError();
}

cudaError_t launch_yan(const unsigned char* Tb, const float* F, float* chat, int n, int w, int B, const int* status,
                       cudaStream_t s) {
  const TcGeom g(n, w);
  k_yan_tc<<<dim3(g.mtiles, B), 128, yan_tc_smem(n), s>>>(Tb, reinterpret_cast<const float2*>(F),
                                                          reinterpret_cast<float2*>(chat), n, w, B, status);
  return cudaGetLastError();
}

}  // namespace fcgno

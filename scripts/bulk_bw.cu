// Microbenchmark: global -> shared streaming bandwidth of 1-D cp.async.bulk (TMA) rings versus
// plain 16-byte loads, one persistent CTA per SM (or `ctas` per SM).  Informs the staging design
// of the tensor-core kernels.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bulk_bw scripts/bulk_bw.cu && /tmp/bulk_bw
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(
                   smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

// each CTA streams chunks c = blockIdx.x, blockIdx.x + gridDim.x, ... through an S-stage ring
__global__ void k_bulk(const unsigned char* src, size_t nchunks, uint32_t chunk, int S, unsigned* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)S * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  size_t issued = 0, done = 0;
  const size_t mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (; issued < mine && issued < (size_t)S; ++issued) {
    const int s = issued % S;
    expect_tx(&bar[s], chunk);
    bulk(sm + (size_t)s * chunk, src + (blockIdx.x + issued * gridDim.x) * (size_t)chunk, chunk, &bar[s]);
  }
  for (; done < mine; ++done) {
    const int s = done % S;
    mbar_wait(&bar[s], (uint32_t)(done / S) & 1);
    acc += sm[(size_t)s * chunk];
    if (issued < mine) {
      expect_tx(&bar[s], chunk);
      bulk(sm + (size_t)s * chunk, src + (blockIdx.x + issued * gridDim.x) * (size_t)chunk, chunk, &bar[s]);
      ++issued;
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

__global__ void k_ldg(const uint4* src, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n16; t += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcg(src + t);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (argc > 1 ? (size_t)atoi(argv[1]) : 256ull) << 20;   // MB streamed
  const bool warm = argc > 2 && argv[2][0] == 'w';                          // L2-resident source
  unsigned char* src;
  unsigned* sink;
  cudaMalloc(&src, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(src, 1, bytes);
  unsigned char* flush;
  cudaMalloc(&flush, 512ull << 20);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto launch) {
    float best = 1e9f;
    for (int r = 0; r < 3; ++r) {
      if (warm) launch(); else cudaMemset(flush, r, 512ull << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  printf("SMs=%d, %zu MB %s\n", sms, bytes >> 20, warm ? "L2-warm (re-read right after a pass)" : "from HBM (L2 flushed)");
  for (int ctas : {1, 2})
    for (uint32_t chunk : {4096u, 8192u, 16384u, 32768u, 65536u})
      for (int S : {2, 4, 8}) {
        const size_t smem = (size_t)S * chunk + 256;
        if (smem * ctas > 220 * 1024) continue;
        const size_t nchunks = bytes / chunk;
        const double gbs = run([&] { k_bulk<<<sms * ctas, 32, smem>>>(src, nchunks, chunk, S, sink); });
        printf("bulk ctas/SM=%d chunk=%6u stages=%d in-flight/SM=%4zu KB : %7.0f GB/s\n", ctas, chunk, S,
               (size_t)S * chunk * ctas / 1024, gbs);
      }
  for (int tpb : {256, 512, 1024}) {
    const double gbs = run([&] { k_ldg<<<sms * 2, tpb>>>(reinterpret_cast<const uint4*>(src), bytes / 16, sink); });
    printf("ldg.cg 16B  grid=2x%d x %d threads : %7.0f GB/s\n", sms, tpb, gbs);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

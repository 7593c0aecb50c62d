// microbench_dsmem.cu — design probe (not product code): throughput of a
// 10^6-cell histogram held in the distributed shared memory of a thread-block
// cluster (u16 counter pairs), versus the local shared-memory histogram.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_dsmem tools/microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mixz(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void gen(uint32_t* k, uint64_t n, uint32_t bound) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    k[i] = mixz(0x1234 + (i + 1) * 0x9E3779B97F4A7C15ULL) % bound;
}

// Each cluster counts a contiguous share of the keys into its DSMEM grid of
// `cells` u16 counters (2 per word), spread over CS CTAs.
template <int CS, bool RED>
__global__ void k_dsmem_hist(const uint4* __restrict__ keys, uint64_t nvec, uint32_t cells, uint32_t* out_sink) {
  extern __shared__ uint32_t s[];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t per_cta = (cells + CS - 1) / CS;  // cells owned by one CTA
  const uint32_t words = (per_cta + 1) / 2;
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) s[i] = 0;
  cluster.sync();
  const uint64_t nclusters = gridDim.x / CS;
  const uint64_t cid = blockIdx.x / CS;
  const uint32_t rank = cluster.block_rank();
  const uint64_t per = (nvec + nclusters - 1) / nclusters;
  const uint64_t v0 = cid * per, v1 = v0 + per < nvec ? v0 + per : nvec;
  for (uint64_t i = v0 + rank * blockDim.x + threadIdx.x; i < v1; i += (uint64_t)CS * blockDim.x) {
    const uint4 q = __ldcs(keys + i);
    const uint32_t e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t owner = e[j] / per_cta;
      const uint32_t local = e[j] - owner * per_cta;
      uint32_t* remote = cluster.map_shared_rank(s + (local >> 1), owner);
      if (RED) atomicAdd(remote, 1u << ((local & 1) * 16));
      else {
        const uint32_t old = atomicAdd(remote, 1u << ((local & 1) * 16));
        if (old == 0xFFFFFFFFu) out_sink[0] = 1;
      }
    }
  }
  cluster.sync();
  uint32_t acc = 0;
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) acc += s[i];
  if (acc == 0x12345u) out_sink[1] = acc;
}

__global__ void k_local_hist(const uint4* __restrict__ keys, uint64_t nvec, uint32_t bins, uint32_t* sink) {
  extern __shared__ uint32_t s[];
  for (uint32_t i = threadIdx.x; i < bins; i += blockDim.x) s[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q = __ldcs(keys + i);
    atomicAdd(&s[q.x % bins], 1u);
    atomicAdd(&s[q.y % bins], 1u);
    atomicAdd(&s[q.z % bins], 1u);
    atomicAdd(&s[q.w % bins], 1u);
  }
  __syncthreads();
  if (s[threadIdx.x] == 0x12345u) sink[0] = 1;
}

template <int CS, bool RED>
int run(const uint32_t* k, uint64_t n, uint32_t cells, uint32_t* sink, int threads, int sms) {
  auto kern = k_dsmem_hist<CS, RED>;
  const uint32_t per_cta = (cells + CS - 1) / CS;
  const size_t smem = ((per_cta + 1) / 2) * 4;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (CS > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  int nclusters = 0;
  cfg.gridDim = dim3(CS);
  CK(cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg));
  cfg.gridDim = dim3(CS * nclusters);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, kern, (const uint4*)k, n / 4, cells, sink));
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) cudaLaunchKernelEx(&cfg, kern, (const uint4*)k, n / 4, cells, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("dsmem hist cells=%u cluster=%d red=%d threads=%d clusters=%d smem=%zuKB: %.3f ms  %.1f Gkeys/s  %.2f keys/clk/SM\n",
         cells, CS, RED, threads, nclusters, smem / 1024, ms, n / ms / 1e6, n / (ms * 1e-3) / 1.9e9 / sms);
  return 0;
}

int main() {
  const uint64_t n = 1ull << 28;
  uint32_t *k, *sink;
  CK(cudaMalloc(&k, n * 4));
  CK(cudaMalloc(&sink, 64));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  gen<<<sms * 8, 256>>>(k, n, 1000000);
  CK(cudaDeviceSynchronize());
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_local_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k_local_hist<<<sms * 8, 256, 4096 * 4>>>((const uint4*)k, n / 4, 4096, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_local_hist<<<sms * 8, 256, 4096 * 4>>>((const uint4*)k, n / 4, 4096, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("local smem hist 4096 bins: %.3f ms\n", ms / 5);
  }
  run<16, true>(k, n, 1000000, sink, 1024, sms);
  run<16, true>(k, n, 1000000, sink, 512, sms);
  run<16, false>(k, n, 1000000, sink, 1024, sms);
  run<8, true>(k, n, 400000, sink, 1024, sms);
  run<4, true>(k, n, 200000, sink, 1024, sms);
  run<2, true>(k, n, 100000, sink, 1024, sms);
  return 0;
}

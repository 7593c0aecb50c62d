// microbench.cu — design probes for the counting pass on B200 (not product
// code).  Times, with CUDA events, streaming reads, copies, and histogram
// variants over 2^28 uint32 keys, to choose between L2-atomic grids and
// shared-memory privatisation.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mixz(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void gen(uint32_t* k, uint64_t n, uint32_t bound, int zipfish) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = mixz(0x1234 + (i + 1) * 0x9E3779B97F4A7C15ULL);
    uint32_t v = x % bound;
    if (zipfish && (i & 1)) v = (x >> 40) % 16 == 0 ? 0 : v % 64;  // skewed half
    k[i] = v;
  }
}

__global__ void k_read(const uint4* __restrict__ p, uint64_t nv, unsigned* sink) {
  unsigned acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) atomicAdd(sink, 1);
}

__global__ void k_copy(const uint4* __restrict__ p, uint4* __restrict__ q, uint64_t nv) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(q + i, __ldcs(p + i));
}

template <int AGG>
__global__ void k_hist_global(const uint4* __restrict__ p, uint64_t nv, unsigned* __restrict__ h) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (nv + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + it * stride;
    bool ok = i < nv;
    uint4 v = ok ? __ldcs(p + i) : make_uint4(0, 0, 0, 0);
    unsigned e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (AGG) {
        unsigned tag = ok ? e[j] : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, tag);
        if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[e[j]], __popc(peers));
      } else if (ok) {
        atomicAdd(&h[e[j]], 1u);
      }
    }
  }
}

template <int AGG>
__global__ void k_hist_smem(const uint4* __restrict__ p, uint64_t nv, unsigned* __restrict__ h, unsigned bins) {
  extern __shared__ unsigned s[];
  for (unsigned i = threadIdx.x; i < bins; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t iters = (nv + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x + it * stride;
    bool ok = i < nv;
    uint4 v = ok ? __ldcs(p + i) : make_uint4(0, 0, 0, 0);
    unsigned e[4] = {v.x % bins, v.y % bins, v.z % bins, v.w % bins};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (AGG) {
        unsigned tag = ok ? e[j] : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, tag);
        if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&s[e[j]], __popc(peers));
      } else if (ok) {
        atomicAdd(&s[e[j]], 1u);
      }
    }
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < bins; i += blockDim.x)
    if (s[i]) atomicAdd(&h[i], s[i]);
}

int main() {
  const uint64_t n = 1ull << 28, nv = n / 4;
  uint32_t *k, *k2, *o;
  unsigned *h, *sink;
  CK(cudaMalloc(&k, n * 4));
  CK(cudaMalloc(&k2, n * 4));
  CK(cudaMalloc(&o, n * 4));
  CK(cudaMalloc(&h, 100000000ull * 4));
  CK(cudaMalloc(&sink, 4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    cudaError_t e = cudaGetLastError();
    printf("%-44s %8.3f ms  %8.1f GB/s  %7.1f Gkeys/s %s\n", name, ms, bytes / ms / 1e6, n / ms / 1e6,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  printf("SMs=%d n=%llu\n", sms, (unsigned long long)n);
  const unsigned bounds[] = {1000, 100000, 1000000, 10000000, 100000000};
  gen<<<sms * 8, 256>>>(k, n, 1000000, 0);
  for (int grid_mul : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "read 1GiB (uint4, grid %dxSM)", grid_mul);
    timeit(nm, n * 4.0, [&] { k_read<<<sms * grid_mul, 256>>>((const uint4*)k, nv, sink); });
  }
  timeit("copy 1GiB->1GiB", n * 8.0, [&] { k_copy<<<sms * 8, 256>>>((const uint4*)k, (uint4*)o, nv); });
  for (unsigned bound : bounds) {
    gen<<<sms * 8, 256>>>(k, n, bound, 0);
    char nm[64];
    snprintf(nm, 64, "global RED hist bins=%u", bound);
    timeit(nm, n * 4.0, [&] {
      cudaMemsetAsync(h, 0, bound * 4ull);
      k_hist_global<0><<<sms * 8, 256>>>((const uint4*)k, nv, h);
    });
    snprintf(nm, 64, "global RED+match hist bins=%u", bound);
    timeit(nm, n * 4.0, [&] {
      cudaMemsetAsync(h, 0, bound * 4ull);
      k_hist_global<1><<<sms * 8, 256>>>((const uint4*)k, nv, h);
    });
  }
  gen<<<sms * 8, 256>>>(k, n, 1000000, 1);
  timeit("global RED hist 1e6 skewed", n * 4.0, [&] {
    cudaMemsetAsync(h, 0, 4000000);
    k_hist_global<0><<<sms * 8, 256>>>((const uint4*)k, nv, h);
  });
  timeit("global RED+match hist 1e6 skewed", n * 4.0, [&] {
    cudaMemsetAsync(h, 0, 4000000);
    k_hist_global<1><<<sms * 8, 256>>>((const uint4*)k, nv, h);
  });
  gen<<<sms * 8, 256>>>(k, n, 1000000, 0);
  for (unsigned bins : {256u, 1000u, 4096u, 16384u, 50000u}) {
    char nm[64];
    size_t sm = bins * 4;
    cudaFuncSetAttribute(k_hist_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k_hist_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    for (int per : {2, 4, 8}) {
      snprintf(nm, 64, "smem hist bins=%u grid %dxSM", bins, per);
      timeit(nm, n * 4.0, [&] { k_hist_smem<0><<<sms * per, 256, sm>>>((const uint4*)k, nv, h, bins); });
    }
    snprintf(nm, 64, "smem+match hist bins=%u grid 4xSM", bins);
    timeit(nm, n * 4.0, [&] { k_hist_smem<1><<<sms * 4, 256, sm>>>((const uint4*)k, nv, h, bins); });
  }
  return 0;
}

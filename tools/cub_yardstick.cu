// cub_yardstick.cu — library yardstick, NOT part of the product: times CUB's
// DeviceRadixSort (the onesweep LSD radix sort torch.sort uses) on the cfg2
// shapes, so the repo's own kernels can be compared with a tuned library sort
// on the same box.  2^28 uint32 keys uniform in [0,10^6) (cfg2), key-only and
// stable key/value (payload = index), over the 20 bits 10^6 needs and over all
// 32 bits.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/cub_yardstick.cu -o tools/cub_yardstick
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__global__ void gen(uint32_t* k, uint32_t* v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = i + 0x9E3779B97F4A7C15ull;  // splitmix64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    k[i] = static_cast<uint32_t>(z % 1000000ull);
    v[i] = static_cast<uint32_t>(i);
  }
}

__global__ void check(const uint32_t* k, size_t n, unsigned* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x + 1; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (k[i - 1] > k[i]) *bad = 1;
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], nullptr, 0) : (1ull << 28);
  const int iters = 10;
  uint32_t *k0, *v0, *k1, *v1, *k2, *v2;
  unsigned* bad;
  CK(cudaMalloc(&k0, n * 4));
  CK(cudaMalloc(&v0, n * 4));
  CK(cudaMalloc(&k1, n * 4));
  CK(cudaMalloc(&v1, n * 4));
  CK(cudaMalloc(&k2, n * 4));
  CK(cudaMalloc(&v2, n * 4));
  CK(cudaMalloc(&bad, 4));
  gen<<<148 * 8, 256>>>(k0, v0, n);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int pairs = 0; pairs < 2; ++pairs)
    for (int end_bit : {20, 32}) {
      size_t tmp = 0;
      void* d_tmp = nullptr;
      auto run = [&](void* t) {
        if (pairs)
          CK(cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, v0, v1, n, 0, end_bit));
        else
          CK(cub::DeviceRadixSort::SortKeys(t, tmp, k0, k1, n, 0, end_bit));
      };
      run(nullptr);
      CK(cudaMalloc(&d_tmp, tmp));
      for (int w = 0; w < 3; ++w) run(d_tmp);
      float total = 0;
      for (int it = 0; it < iters; ++it) {
        CK(cudaMemcpyAsync(k2, v0, n * 4, cudaMemcpyDeviceToDevice));  // evict L2 between runs
        CK(cudaEventRecord(a));
        run(d_tmp);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        total += ms;
      }
      CK(cudaMemset(bad, 0, 4));
      check<<<148 * 8, 256>>>(k1, n, bad);
      unsigned h;
      CK(cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost));
      const double ms = total / iters;
      printf("{\"lib\": \"cub::DeviceRadixSort::%s\", \"n\": %zu, \"end_bit\": %d, \"ms\": %.4f, \"gkeys_s\": %.2f, \"sorted\": %s}\n",
             pairs ? "SortPairs" : "SortKeys", n, end_bit, ms, n / ms / 1e6, h ? "false" : "true");
      CK(cudaFree(d_tmp));
    }
  return 0;
}

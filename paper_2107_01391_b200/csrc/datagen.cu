// datagen.cu — seeded synthetic config inputs on the device (bench/test
// utility; not part of the sort).  Element i of Splitmix64(seed) is
// mix(seed + (i+1)*golden) (splitmix64.hpp:14-19), so these are
// bit-identical to oracle/oracle.cpp's or_gen_* on the host.
#include <cuda_runtime.h>

#include <cstdint>

#include "recsort_b200.h"
#include "rs_internal.cuh"

namespace rsb {
namespace {

__device__ __forceinline__ uint64_t sm64_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void k_gen_u32(uint64_t seed, uint64_t first, uint64_t n, uint64_t bound, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t x = sm64_at(seed, first + i);
    out[i] = bound ? static_cast<uint32_t>(x % bound) : static_cast<uint32_t>(x >> 32);
  }
}

__global__ void k_iota(uint64_t first, uint64_t n, uint32_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<uint32_t>(first + i);
}

// cfg3: even elements k uniform in [0, ranks), odd elements k = Zipf rank-1
// by inverse CDF (upper_bound on a host-computed table); x = k / 1000.
__global__ void k_gen_f64(uint64_t seed, uint64_t first, uint64_t n, const double* cdf,
                          uint32_t ranks, double* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t g = first + i;
    const uint64_t x = sm64_at(seed, g);
    uint64_t k;
    if ((g & 1) == 0) {
      k = x % ranks;
    } else {
      const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
      uint32_t lo = 0, hi = ranks;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cdf[mid] > u) hi = mid;
        else lo = mid + 1;
      }
      k = lo < ranks ? lo : ranks - 1;
    }
    out[i] = static_cast<double>(k) / 1000.0;
  }
}

__global__ void k_gen_str(uint64_t seed, uint64_t first, uint64_t n, uint8_t* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t w = 0;
    for (int j = 0; j < 8; ++j)
      w |= static_cast<uint64_t>('a' + sm64_at(seed, (first + i) * 8 + j) % 26) << (8 * j);
    reinterpret_cast<uint64_t*>(out)[i] = w;
  }
}

unsigned gen_grid(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace
}  // namespace rsb

using namespace rsb;

extern "C" {

rs_status rs_gen_u32(uint64_t seed, uint64_t first, uint64_t n, uint64_t bound, uint32_t* out,
                     void* stream) {
  return guarded([&] {
    ensure_device();
    if (n == 0) return;
    k_gen_u32<<<gen_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, first, n, bound, out);
    RS_LAUNCH_CHECK();
  });
}

rs_status rs_gen_iota_u32(uint64_t first, uint64_t n, uint32_t* out, void* stream) {
  return guarded([&] {
    ensure_device();
    if (n == 0) return;
    k_iota<<<gen_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(first, n, out);
    RS_LAUNCH_CHECK();
  });
}

rs_status rs_gen_f64_cfg3(uint64_t seed, uint64_t first, uint64_t n, const double* cdf,
                          uint32_t ranks, double* out, void* stream) {
  return guarded([&] {
    ensure_device();
    if (n == 0) return;
    if (ranks == 0) fail(RS_INVALID_ARGUMENT, "ranks must be positive");
    k_gen_f64<<<gen_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, first, n, cdf, ranks, out);
    RS_LAUNCH_CHECK();
  });
}

rs_status rs_gen_str_cfg4(uint64_t seed, uint64_t first, uint64_t n, uint8_t* out, void* stream) {
  return guarded([&] {
    ensure_device();
    if (n == 0) return;
    k_gen_str<<<gen_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, first, n, out);
    RS_LAUNCH_CHECK();
  });
}

}  // extern "C"

// kernels_msd.cuh — MSD bucket passes (K6) for keys too wide for one grid,
// and the range partition the multi-GPU exchange uses.  The reference has no
// such pass: it raises cell_budget_exceeded (key_model.cpp:72-76).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rs_internal.cuh"

namespace rsb {

constexpr int kMsdThreads = 256;  // also used by kernels_msd_engine.cuh
constexpr uint32_t kMsdSmemBuckets = 12288;

// Histogram of bucket = key / divisor (magic-number division, exact for
// 32-bit keys: see div_magic).  Buckets at or above `buckets` set overflow.
__global__ void __launch_bounds__(kMsdThreads) k_bucket_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                             unsigned long long magic, uint32_t buckets,
                                                             unsigned long long* __restrict__ hist,
                                                             DevStats* st) {
  extern __shared__ uint32_t s_h[];
  const bool smem = buckets <= kMsdSmemBuckets;
  if (smem) {
    for (uint32_t i = threadIdx.x; i < buckets; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
  }
  unsigned ovf = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = __ldcs(keys + i);
    const uint32_t b = magic ? static_cast<uint32_t>(__umul64hi((unsigned long long)k, magic)) : k;
    if (b >= buckets) {
      ovf = 1;
      continue;
    }
    if (smem) atomicAdd(&s_h[b], 1u);
    else atomicAdd(&hist[b], 1ull);
  }
  if (smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < buckets; i += blockDim.x)
      if (s_h[i]) atomicAdd(&hist[i], (unsigned long long)s_h[i]);
  }
  if (ovf) atomicOr(&st->overflow, 1u);
}

// Map a bucket to its part through the sorted part bounds (bounds[0] = 0,
// bounds[parts] = buckets).
__device__ __forceinline__ uint32_t part_of(uint32_t b, const uint32_t* s_bounds, uint32_t parts) {
  uint32_t lo = 0, hi = parts;  // last p with bounds[p] <= b
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s_bounds[mid] <= b) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Per-part counts (pass 1 of the partition).
__global__ void __launch_bounds__(kMsdThreads) k_part_count(const uint32_t* __restrict__ keys, uint64_t n,
                                                            unsigned long long magic,
                                                            const uint32_t* __restrict__ bounds, uint32_t parts,
                                                            unsigned long long* __restrict__ counts) {
  __shared__ uint32_t s_bounds[1025];
  __shared__ uint32_t s_c[1024];
  for (uint32_t i = threadIdx.x; i <= parts; i += blockDim.x) s_bounds[i] = bounds[i];
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) s_c[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = __ldcs(keys + i);
    const uint32_t b = magic ? static_cast<uint32_t>(__umul64hi((unsigned long long)k, magic)) : k;
    atomicAdd(&s_c[part_of(b, s_bounds, parts)], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x)
    if (s_c[i]) atomicAdd(&counts[i], (unsigned long long)s_c[i]);
}

// Scatter into part-contiguous order (pass 2).  Each CTA takes a chunk of
// keys, ranks them per part in shared memory and reserves its run in every
// part with one global atomic per (CTA chunk, part).  Part p is written at
// dst[p] + cursor: one buffer for a local partition, or — the multi-GPU
// exchange — each part straight into its destination rank's receive buffer
// through NVLink peer pointers (no separate all-to-all).
constexpr int kPartChunk = 4096;
__global__ void __launch_bounds__(kMsdThreads) k_part_scatter(const uint32_t* __restrict__ keys, uint64_t n,
                                                              unsigned long long magic,
                                                              const uint32_t* __restrict__ bounds, uint32_t parts,
                                                              unsigned long long* __restrict__ cursors,
                                                              uint32_t* const* __restrict__ dst) {
  __shared__ uint32_t s_bounds[1025];
  __shared__ uint32_t s_c[1024];
  __shared__ unsigned long long s_base[1024];
  __shared__ uint32_t* s_dst[1024];
  for (uint32_t i = threadIdx.x; i <= parts; i += blockDim.x) s_bounds[i] = bounds[i];
  for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) s_dst[i] = dst[i];
  for (uint64_t c0 = (uint64_t)blockIdx.x * kPartChunk; c0 < n; c0 += (uint64_t)gridDim.x * kPartChunk) {
    for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x) s_c[i] = 0;
    __syncthreads();
    uint32_t k[kPartChunk / kMsdThreads], p[kPartChunk / kMsdThreads], r[kPartChunk / kMsdThreads];
#pragma unroll
    for (int j = 0; j < kPartChunk / kMsdThreads; ++j) {
      const uint64_t i = c0 + j * kMsdThreads + threadIdx.x;
      p[j] = 0xffffffffu;
      if (i < n) {
        k[j] = __ldcs(keys + i);
        const uint32_t b = magic ? static_cast<uint32_t>(__umul64hi((unsigned long long)k[j], magic)) : k[j];
        p[j] = part_of(b, s_bounds, parts);
        r[j] = atomicAdd(&s_c[p[j]], 1u);
      }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < parts; i += blockDim.x)
      if (s_c[i]) s_base[i] = atomicAdd(&cursors[i], (unsigned long long)s_c[i]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPartChunk / kMsdThreads; ++j)
      if (p[j] != 0xffffffffu) s_dst[p[j]][s_base[p[j]] + r[j]] = k[j];
    __syncthreads();
  }
}


}  // namespace rsb

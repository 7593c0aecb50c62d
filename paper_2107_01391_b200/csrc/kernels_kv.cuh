// kernels_kv.cuh — stable key/value sort (K5).
//
// The reference has no record API; its stable order is rsort's
// originals_by_key (rsort.cpp:133-145) == baselines::radix_sort_lsd_by
// (baselines.hpp:24-46), which makes base-10 LSD passes.  Here a pass takes
// a group of three decimal digits (radix 1000 = a 10x10x10 sub-grid of the
// Cartesian count space), so a 6-digit key needs two stable passes instead
// of six.  Because stable order is unique, the output is bit-identical to
// the reference's for any stable schedule.
//
// Per pass (one kernel, single-pass "onesweep" structure):
//   * tiles of 4096 records get ordered ids from an atomic ticket;
//   * each warp ranks its records stably with __match_any_sync over the
//     group digit and a warp-private shared histogram;
//   * the tile's per-digit counts are published and each digit's prefix over
//     earlier tiles is found by decoupled look-back (32-bit descriptors:
//     [31:30] flag, [29:0] count; n < 2^30 per call);
//   * records are staged in shared memory in digit order and written out so
//     consecutive threads store consecutive addresses of a digit run.
// Digit offsets of every pass come from one histogram pre-pass over the keys.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rs_internal.cuh"

namespace rsb {

constexpr int kKvThreads = 256;
constexpr int kKvItems = 16;                        // records per thread
constexpr int kKvTile = kKvThreads * kKvItems;      // 4096 records per tile
constexpr int kKvBins = 1000;                       // three decimal digits
constexpr int kKvMaxPasses = 4;                     // 10-digit uint32 keys
constexpr size_t kKvSmemBytes = kKvBins * 8 + 2 * kKvTile * 4 + kKvBins * 4 +
                                (kKvThreads / 32) * kKvBins * 2 + kKvTile * 2;
constexpr uint32_t kKvAgg = 1u << 30, kKvPre = 2u << 30, kKvVal = (1u << 30) - 1;

// Exact floor(n / D) for 32-bit n with M = ceil(2^64 / D) (error n*e/2^64 <
// 1/D because n, e < 2^32).
__device__ __forceinline__ uint32_t div_magic(uint32_t n, unsigned long long m) {
  return static_cast<uint32_t>(__umul64hi(static_cast<unsigned long long>(n), m));
}

struct KvPass {
  unsigned long long magic_div;  // divides by 10^(3*pass)
  unsigned long long magic_1000; // divides by 1000
  uint32_t bins;                 // 1000, or 10^(remaining digits) on the top pass
};

__device__ __forceinline__ uint32_t kv_digit(uint32_t key, const KvPass& p) {
  const uint32_t q = p.magic_div ? div_magic(key, p.magic_div) : key;
  return q - 1000u * div_magic(q, p.magic_1000);
}

// Pre-pass: all group-digit histograms at once (+ max for the geometry).
__global__ void __launch_bounds__(kKvThreads) k_kv_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                        KvPass p0, KvPass p1, KvPass p2, KvPass p3,
                                                        uint32_t passes,
                                                        unsigned long long* __restrict__ hist,
                                                        DevStats* st) {
  __shared__ uint32_t s_hist[kKvMaxPasses * kKvBins];
  for (int i = threadIdx.x; i < kKvMaxPasses * kKvBins; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const KvPass ps[kKvMaxPasses] = {p0, p1, p2, p3};
  unsigned long long mx = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = __ldcs(keys + i);
    mx = k > mx ? k : mx;
    for (uint32_t p = 0; p < passes; ++p) atomicAdd(&s_hist[p * kKvBins + kv_digit(k, ps[p])], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)passes * kKvBins; i += blockDim.x)
    if (s_hist[i]) atomicAdd(&hist[i], (unsigned long long)s_hist[i]);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&st->max_key, mx);
}

// Exclusive scan of each pass's histogram into digit offsets (1 block/pass).
__global__ void k_kv_offsets(const unsigned long long* __restrict__ hist,
                             unsigned long long* __restrict__ offsets) {
  const int p = blockIdx.x;
  __shared__ unsigned long long s[kKvBins];
  for (int i = threadIdx.x; i < kKvBins; i += blockDim.x) s[i] = hist[p * kKvBins + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int i = 0; i < kKvBins; ++i) {
      const unsigned long long c = s[i];
      s[i] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kKvBins; i += blockDim.x) offsets[p * kKvBins + i] = s[i];
}

// One stable LSD pass.
__global__ void __launch_bounds__(kKvThreads) k_kv_pass(const uint32_t* __restrict__ keys_in,
                                                        const uint32_t* __restrict__ vals_in,
                                                        uint32_t* __restrict__ keys_out,
                                                        uint32_t* __restrict__ vals_out, uint64_t n,
                                                        KvPass pass,
                                                        const unsigned long long* __restrict__ offsets,
                                                        uint32_t* desc, unsigned* tile_counter) {
  // dynamic shared memory (kKvSmemBytes), carved:
  extern __shared__ __align__(16) unsigned char kv_smem[];
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(kv_smem);   // [kKvBins]
  uint32_t* s_keys = reinterpret_cast<uint32_t*>(s_base + kKvBins);             // [kKvTile]
  uint32_t* s_vals = s_keys + kKvTile;                                          // [kKvTile]
  uint32_t* s_cnt = s_vals + kKvTile;                                           // [kKvBins]
  uint16_t (*s_wh)[kKvBins] = reinterpret_cast<uint16_t (*)[kKvBins]>(s_cnt + kKvBins);  // [8][kKvBins]
  uint16_t* s_dig = &s_wh[kKvThreads / 32][0];                                  // [kKvTile]
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[kKvThreads];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < (kKvThreads / 32) * kKvBins; i += blockDim.x)
    (&s_wh[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * kKvTile;

  // striped load: record t0 + warp*512 + j*32 + lane
  uint32_t k[kKvItems], v[kKvItems], rank[kKvItems];
  uint16_t d[kKvItems];
#pragma unroll
  for (int j = 0; j < kKvItems; ++j) {
    const uint64_t i = t0 + warp * (kKvItems * 32) + j * 32 + lane;
    const bool ok = i < n;
    k[j] = ok ? __ldcs(keys_in + i) : 0u;
    v[j] = ok ? __ldcs(vals_in + i) : 0u;
    d[j] = ok ? static_cast<uint16_t>(kv_digit(k[j], pass)) : static_cast<uint16_t>(0xffff);
  }
  // warp-level stable ranks
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kKvItems; ++j) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[j]);
    const bool ok = d[j] != 0xffff;
    uint32_t base = 0;
    if (ok) base = s_wh[warp][d[j]];
    __syncwarp();
    if (ok && (peers & lt) == 0) s_wh[warp][d[j]] = static_cast<uint16_t>(base + __popc(peers));
    __syncwarp();
    rank[j] = base + __popc(peers & lt);
  }
  __syncthreads();
  // per digit: exclusive prefix across warps, tile count
  for (int b = threadIdx.x; b < kKvBins; b += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kKvThreads / 32; ++w) {
      const uint32_t c = s_wh[w][b];
      s_wh[w][b] = static_cast<uint16_t>(run);
      run += c;
    }
    s_cnt[b] = run;
  }
  __syncthreads();
  // publish aggregates, look back, publish inclusive prefixes
  volatile uint32_t* vdesc = desc;
  for (int b = threadIdx.x; b < (int)pass.bins; b += blockDim.x) {
    const uint32_t c = s_cnt[b];
    unsigned long long prefix = 0;
    if (tile == 0) {
      vdesc[b] = kKvPre | c;
    } else {
      vdesc[(uint64_t)tile * kKvBins + b] = kKvAgg | c;
      for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
        uint32_t x;
        do {
          x = vdesc[(uint64_t)t * kKvBins + b];
        } while ((x >> 30) == 0);
        prefix += x & kKvVal;
        if ((x >> 30) == 2) break;
      }
      vdesc[(uint64_t)tile * kKvBins + b] = kKvPre | static_cast<uint32_t>(prefix + c);
    }
    s_base[b] = offsets[b] + prefix;
  }
  // tile-local exclusive scan of s_cnt over digits (4 digits per thread)
  {
    uint32_t loc[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b = threadIdx.x * 4 + q;
      loc[q] = b < kKvBins ? s_cnt[b] : 0u;
      sum += loc[q];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_scan[warp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t r = 0;
      for (int w = 0; w < kKvThreads / 32; ++w) {
        const uint32_t c = s_scan[w];
        s_scan[w] = r;
        r += c;
      }
    }
    __syncthreads();
    uint32_t run = s_scan[warp] + inc - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b = threadIdx.x * 4 + q;
      if (b < kKvBins) s_cnt[b] = run;
      run += loc[q];
    }
  }
  __syncthreads();
  // stage in digit order
#pragma unroll
  for (int j = 0; j < kKvItems; ++j) {
    if (d[j] != 0xffff) {
      const uint32_t pos = s_cnt[d[j]] + s_wh[warp][d[j]] + rank[j];
      s_keys[pos] = k[j];
      s_vals[pos] = v[j];
      s_dig[pos] = d[j];
    }
  }
  __syncthreads();
  const uint64_t valid = n - t0 < (uint64_t)kKvTile ? n - t0 : (uint64_t)kKvTile;
  for (uint32_t i = threadIdx.x; i < valid; i += blockDim.x) {
    const uint32_t b = s_dig[i];
    const unsigned long long g = s_base[b] + (i - s_cnt[b]);
    keys_out[g] = s_keys[i];
    vals_out[g] = s_vals[i];
  }
}

}  // namespace rsb

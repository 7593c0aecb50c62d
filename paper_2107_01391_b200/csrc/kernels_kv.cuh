// kernels_kv.cuh — stable key/value sort (K5).
//
// The reference has no record API; its stable order is rsort's
// originals_by_key (rsort.cpp:133-145) == baselines::radix_sort_lsd_by
// (baselines.hpp:24-46), which makes base-10 LSD passes.  Here a pass takes a
// pair of decimal digits (radix 100: a 10x10 sub-grid of the Cartesian count
// space), so a 6-digit key needs three stable passes instead of six.  (Triples
// — radix 1000, two passes — measured 6 ms per pass on B200: the per-tile
// work over 1000 digit bins and 4-record write runs dominated.)  Stable order
// is unique, so the output is bit-identical to the reference's for any stable
// schedule.
//
// Per pass (reduce-then-scan, deterministic):
//   k_kv_chunk_hist     per-CTA digit counts over a contiguous chunk      R4
//   exscan              [bins][G] -> each CTA's start in every digit run
//   k_kv_chunk_scatter  the CTA walks its chunk tile by tile in order; each
//                       warp ranks its records stably with 7 ballots over
//                       the digit bits (no __match_any_sync, which measured
//                       ~10x slower on B200), the tile is staged in shared
//                       memory in digit order and written so consecutive
//                       threads store consecutive addresses of a run  R8 + W8
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rs_internal.cuh"

namespace rsb {

constexpr int kKvThreads = 256;
constexpr int kKvItems = 16;                    // records per thread per tile
constexpr int kKvTile = kKvThreads * kKvItems;  // 4096 records
constexpr int kKvBins = 100;                    // two decimal digits
constexpr int kKvBits = 7;                      // 100 < 2^7
constexpr int kKvMaxPasses = 5;                 // 10-digit uint32 keys
constexpr int kKvWarps = kKvThreads / 32;
constexpr size_t kKvSmemBytes = kKvWarps * kKvBins * 2  // s_wh
                                + kKvBins * 4 * 3        // s_cnt, s_start, s_cur
                                + kKvTile * 4 * 2        // s_keys, s_vals
                                + kKvTile * 2            // s_dig
                                + 64 * 4;

struct KvPass {
  unsigned long long magic_div;   // floor(k / 10^(2*pass)) = (k * magic_div) >> shift_div
  unsigned long long magic_1000;  // floor(q / 100) = (q * magic_1000) >> shift_1000
  uint32_t shift_div, shift_1000;
  uint32_t bins;                  // 100, or 10 on a top pass with one digit left
  uint64_t chunk;                 // records per CTA (multiple of kKvTile)
  uint32_t G;                     // CTAs
};

__device__ __forceinline__ uint32_t kv_digit(uint32_t key, const KvPass& p) {
  const uint32_t q = p.shift_div == 64
                         ? static_cast<uint32_t>(__umul64hi(static_cast<unsigned long long>(key), p.magic_div))
                         : static_cast<uint32_t>((static_cast<unsigned long long>(key) * p.magic_div) >> p.shift_div);
  return q - 100u * static_cast<uint32_t>((static_cast<unsigned long long>(q) * p.magic_1000) >> p.shift_1000);
}

// grid = G x kKvHistSplit: CTA (c, s) counts sub-range s of chunk c and adds
// its counts into hist[d][c] (zeroed by the host).
constexpr int kKvHistSplit = 4;
__global__ void __launch_bounds__(kKvThreads) k_kv_chunk_hist(const uint32_t* __restrict__ keys, uint64_t n,
                                                              KvPass p, bool aligned,
                                                              uint32_t* __restrict__ hist,  // [bins][G]
                                                              DevStats* st) {
  __shared__ uint32_t s_h[kKvBins];
  for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const uint32_t c = blockIdx.x / kKvHistSplit, sub = blockIdx.x % kKvHistSplit;
  const uint64_t span = p.chunk / kKvHistSplit;  // chunk is a multiple of kKvTile
  const uint64_t cend = (uint64_t)c * p.chunk + p.chunk < n ? (uint64_t)c * p.chunk + p.chunk : n;
  const uint64_t c0 = (uint64_t)c * p.chunk + sub * span;
  const uint64_t c1 = sub + 1 == kKvHistSplit ? cend : (c0 + span < cend ? c0 + span : cend);
  unsigned long long mx = 0;
  for (uint64_t base = c0; base < c1; base += kKvTile) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i0 = base + q * 1024 + threadIdx.x * 4;
      uint32_t v[4];
      if (aligned && i0 + 4 <= c1) {
        const uint4 w = __ldcs(reinterpret_cast<const uint4*>(keys + i0));
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
      } else {
        for (int e = 0; e < 4; ++e) v[e] = i0 + e < c1 ? keys[i0 + e] : 0u;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (i0 + e < c1) {
          mx = v[e] > mx ? v[e] : mx;
          atomicAdd(&s_h[kv_digit(v[e], p)], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x)
    if (s_h[b]) atomicAdd(&hist[(uint64_t)b * p.G + c], s_h[b]);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = w > mx ? w : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&st->max_key, mx);
}

__global__ void __launch_bounds__(kKvThreads) k_kv_chunk_scatter(const uint32_t* __restrict__ keys_in,
                                                                 const uint32_t* __restrict__ vals_in,
                                                                 uint32_t* __restrict__ keys_out,
                                                                 uint32_t* __restrict__ vals_out, uint64_t n,
                                                                 KvPass p, const uint32_t* __restrict__ off) {
  extern __shared__ __align__(16) unsigned char kv_smem[];
  uint32_t* s_keys = reinterpret_cast<uint32_t*>(kv_smem);  // [kKvTile]
  uint32_t* s_vals = s_keys + kKvTile;                      // [kKvTile]
  uint32_t* s_cnt = s_vals + kKvTile;                       // [kKvBins]
  uint32_t* s_start = s_cnt + kKvBins;                      // [kKvBins]
  uint32_t* s_cur = s_start + kKvBins;                      // [kKvBins]
  uint16_t* s_wh = reinterpret_cast<uint16_t*>(s_cur + kKvBins);  // [kKvWarps][kKvBins]
  uint16_t* s_dig = s_wh + kKvWarps * kKvBins;                    // [kKvTile]
  __shared__ uint32_t s_scan[kKvWarps];
  __shared__ uint32_t s_total;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x) s_cur[b] = off[(uint64_t)b * p.G + blockIdx.x];
  for (int i = threadIdx.x; i < kKvWarps * kKvBins; i += blockDim.x) s_wh[i] = 0;
  const uint64_t c0 = (uint64_t)blockIdx.x * p.chunk;
  const uint64_t c1 = c0 + p.chunk < n ? c0 + p.chunk : n;
  uint16_t* wh = s_wh + warp * kKvBins;
  __syncthreads();

  for (uint64_t t0 = c0; t0 < c1; t0 += kKvTile) {
    // striped load: record t0 + warp*512 + j*32 + lane (input order =
    // warp-major, then j, then lane)
    uint32_t k[kKvItems], v[kKvItems], rank[kKvItems];
    uint32_t d[kKvItems];
#pragma unroll
    for (int j = 0; j < kKvItems; ++j) {
      const uint64_t i = t0 + warp * (kKvItems * 32) + j * 32 + lane;
      const bool ok = i < c1;
      k[j] = ok ? __ldcs(keys_in + i) : 0u;
      v[j] = ok ? __ldcs(vals_in + i) : 0u;
      d[j] = ok ? kv_digit(k[j], p) : 0xffffu;
    }
    // stable warp ranks: peers = lanes with the same digit, from 10 ballots
#pragma unroll
    for (int j = 0; j < kKvItems; ++j) {
      const bool ok = d[j] != 0xffffu;
      unsigned peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
      for (int b = 0; b < kKvBits; ++b) {
        const bool bit = (d[j] >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
      uint32_t base = 0;
      if (ok) base = wh[d[j]];
      __syncwarp();
      if (ok && (peers & lt) == 0) wh[d[j]] = static_cast<uint16_t>(base + __popc(peers));
      __syncwarp();
      rank[j] = base + __popc(peers & lt);
    }
    __syncthreads();
    // per digit: exclusive prefix across warps (in s_wh) and tile count
    for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x) {
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kKvWarps; ++w) {
        const uint32_t c = s_wh[w * kKvBins + b];
        s_wh[w * kKvBins + b] = static_cast<uint16_t>(run);
        run += c;
      }
      s_cnt[b] = run;
    }
    __syncthreads();
    // tile-local exclusive scan over digits (warp 0..3, one digit per lane)
    if (threadIdx.x < 128) {
      const uint32_t b = threadIdx.x;
      const uint32_t c = b < p.bins ? s_cnt[b] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_scan[warp] = inc;
      __syncwarp();
      asm volatile("bar.sync 1, 128;");
      uint32_t before = 0;
      for (int w = 0; w < warp; ++w) before += s_scan[w];
      if (b < p.bins) s_start[b] = before + inc - c;
      if (b == 127) s_total = before + inc;
    }
    // s_cnt[b] becomes this tile's destination base: dest(i) = s_cnt[b] + i
    for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x) {
      const uint32_t c = s_cnt[b];
      s_cnt[b] = s_cur[b] - s_start[b];
      s_cur[b] += c;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kKvItems; ++j) {
      if (d[j] != 0xffffu) {
        const uint32_t pos = s_start[d[j]] + wh[d[j]] + rank[j];
        s_keys[pos] = k[j];
        s_vals[pos] = v[j];
      }
    }
    __syncthreads();
    const uint32_t total = s_total;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
      const uint32_t key = s_keys[i];
      const uint32_t g = s_cnt[kv_digit(key, p)] + i;
      keys_out[g] = key;
      vals_out[g] = s_vals[i];
    }
    for (int i = threadIdx.x; i < kKvWarps * kKvBins; i += blockDim.x) s_wh[i] = 0;
    __syncthreads();
  }
}

}  // namespace rsb

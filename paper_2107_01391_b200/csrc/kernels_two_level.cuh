// kernels_two_level.cuh — the counting pass for grids too large for one
// shared-memory histogram (10^6 cells at cfg2/cfg3).
//
// Measured on B200 (tools/microbench.cu, profiles/r1_microbench.txt): an
// L2-atomic histogram of 2^28 keys over 10^6 cells takes 1.49 ms (181 G
// atomics/s) while a shared-memory histogram of <= 4096 bins takes 0.20 ms at
// 5.3 TB/s.  So the Cartesian grid is split as outer x inner: the leading
// digits pick one of B outer buckets and the trailing digits one of S inner
// cells (10^6 = 1000 x 1000):
//
//   K1a outer_hist     per-CTA shared histogram of the outer digit over a
//                      contiguous chunk of keys (+ max / flags)        R4
//   scan               exclusive scan of the [B][G] per-CTA counts (look-back)
//   K1b outer_scatter  re-read the chunk, stage each tile in shared memory in
//                      bucket order, write the inner digit as uint16
//                      into bucket-contiguous order                     R4 + W2
//   K2  inner_count    slices of the partitioned inner digits, shared
//                      histogram over S cells, one flush per slice into
//                      the dense count grid                             R2
// after which the occupancy scan and the load-balanced emit run unchanged.
// The outer partition is unordered within a bucket: only counts matter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_grid.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kTlThreads = 256;
constexpr int kTlTile = 4096;               // keys per tile (16 per thread)
constexpr uint32_t kTlMaxBuckets = 4096;    // outer buckets (smem hist <= 16 KB)
constexpr uint32_t kTlMaxInner = 16384;     // inner cells (smem hist <= 64 KB)

struct TwoLevel {
  unsigned long long cells;  // grid size C
  uint32_t S;                // inner cells per bucket
  uint32_t B;                // outer buckets = ceil(C / S)
  unsigned long long magic;  // bucket = (cell * magic) >> shift, exact for cell < 2^32
  uint32_t shift;
  uint64_t chunk;            // keys per CTA (multiple of kTlTile)
  uint32_t G;                // CTAs in K1a / K1b
};

__device__ __forceinline__ uint32_t tl_bucket(uint32_t cell, const TwoLevel& t) {
  return static_cast<uint32_t>((static_cast<unsigned long long>(cell) * t.magic) >> t.shift);
}

// Loads element i of a tile: thread t owns elements 4t..4t+3 of each
// 1024-element quarter (16-byte vectors when the input is aligned).
__device__ __forceinline__ uint32_t from_bits32(uint32_t w, uint32_t*) { return w; }
__device__ __forceinline__ int32_t from_bits32(uint32_t w, int32_t*) { return static_cast<int32_t>(w); }
__device__ __forceinline__ double from_bits64(unsigned long long w, double*) { return __longlong_as_double(static_cast<long long>(w)); }
__device__ __forceinline__ unsigned long long from_bits64(unsigned long long w, unsigned long long*) { return w; }
__device__ __forceinline__ int64_t from_bits64(unsigned long long w, int64_t*) { return static_cast<int64_t>(w); }

template <class In>
struct Load4 {
  __device__ __forceinline__ static void run(const In* p, uint64_t i0, uint64_t n, bool aligned, In (&v)[4]) {
    if (aligned && i0 + 4 <= n) {
      if constexpr (sizeof(In) == 4) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(p + i0));
        v[0] = from_bits32(q.x, (In*)nullptr); v[1] = from_bits32(q.y, (In*)nullptr);
        v[2] = from_bits32(q.z, (In*)nullptr); v[3] = from_bits32(q.w, (In*)nullptr);
      } else {
        const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(p + i0));
        const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(p + i0 + 2));
        v[0] = from_bits64(a.x, (In*)nullptr); v[1] = from_bits64(a.y, (In*)nullptr);
        v[2] = from_bits64(b.x, (In*)nullptr); v[3] = from_bits64(b.y, (In*)nullptr);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = (i0 + e < n) ? p[i0 + e] : In{};
    }
  }
};

// ------------------------------------------------------------ K1a
template <class Map>
__global__ void __launch_bounds__(kTlThreads) k_outer_hist(const typename Map::In* __restrict__ in, uint64_t n,
                                                           Map map, TwoLevel t, bool aligned,
                                                           uint32_t* __restrict__ cta_hist,  // [B][G]
                                                           DevStats* st) {
  using In = typename Map::In;
  extern __shared__ uint32_t s_h[];  // [B]
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const uint64_t c0 = (uint64_t)blockIdx.x * t.chunk;
  const uint64_t c1 = c0 + t.chunk < n ? c0 + t.chunk : n;
  unsigned long long mx = 0;
  unsigned flags = 0, ovf = 0;
  // software pipeline: the next tile's four vectors are in flight while
  // the current tile is counted
  In cur[4][4], nxt[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) Load4<In>::run(in, c0 + q * 1024 + threadIdx.x * 4, c1, aligned, cur[q]);
  for (uint64_t base = c0; base < c1; base += kTlTile) {
    const uint64_t nb = base + kTlTile;
    if (nb < c1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) Load4<In>::run(in, nb + q * 1024 + threadIdx.x * 4, c1, aligned, nxt[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i0 = base + q * 1024 + threadIdx.x * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (i0 + e < c1) {
          const unsigned long long k = map(cur[q][e], flags);
          mx = k > mx ? k : mx;
          if (k < t.cells) atomicAdd(&s_h[tl_bucket(static_cast<uint32_t>(k), t)], 1u);
          else ovf = 1;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) cur[q][e] = nxt[q][e];
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) cta_hist[(uint64_t)b * t.G + blockIdx.x] = s_h[b];
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

// ---------------------------------------- exclusive scan (look-back), u32
// out[i] = sum(in[0..i)); also writes the grand total to *total.  Tiles of
// 4096 entries; one 64-bit descriptor per tile ([63:62] flag, [61:0] sum).
__global__ void __launch_bounds__(kThreads) k_exscan_u32(const uint32_t* __restrict__ in, uint64_t count,
                                                         uint32_t* __restrict__ out, unsigned long long* desc,
                                                         unsigned* tile_counter, unsigned long long* total,
                                                         uint32_t num_tiles) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_w[kThreads / 32];
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t i0 = (uint64_t)tile * kScanTile + threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    v[k] = (i0 + k < count) ? in[i0 + k] : 0u;
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const unsigned long long c = s_w[w];
      s_w[w] = r;
      r += c;
    }
    volatile unsigned long long* vd = desc;
    unsigned long long p = 0;
    if (tile == 0) {
      vd[0] = kDescPre | r;
    } else {
      vd[tile] = kDescAgg | r;
      p = lookback(vd, tile);
      vd[tile] = kDescPre | (p + r);
    }
    s_prefix = p;
    if (tile == num_tiles - 1) *total = p + r;
  }
  __syncthreads();
  unsigned long long run = s_prefix + s_w[warp] + inc - sum;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (i0 + k < count) out[i0 + k] = static_cast<uint32_t>(run);
    run += v[k];
  }
}

// ------------------------------------------------------------ K1b
// Dynamic shared layout (kOuterScatterSmem(B)): s_cur[B] running global
// cursor of this CTA per bucket, s_cnt[B+1] tile counts -> tile-local starts,
// s_low[kTlTile] inner digits staged in bucket order.  After staging, each
// warp copies whole bucket runs, lanes on consecutive elements.
__host__ __device__ constexpr size_t kOuterScatterSmem(uint32_t B) {
  return ((size_t)B * 4 * 2 + 16 + kTlTile * 2 + 15) & ~size_t(15);
}

template <class Map>
__global__ void __launch_bounds__(kTlThreads) k_outer_scatter(const typename Map::In* __restrict__ in, uint64_t n,
                                                              Map map, TwoLevel t, bool aligned,
                                                              const uint32_t* __restrict__ cta_off,  // [B][G]
                                                              uint16_t* __restrict__ lows) {
  using In = typename Map::In;
  extern __shared__ __align__(16) unsigned char tl_smem[];
  uint32_t* s_cur = reinterpret_cast<uint32_t*>(tl_smem);
  uint32_t* s_cnt = s_cur + t.B;  // [B+1]
  uint16_t* s_low = reinterpret_cast<uint16_t*>(tl_smem + (((size_t)t.B * 8 + 16 + 15) & ~size_t(15)));
  __shared__ uint32_t s_scan[kTlThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) s_cur[b] = cta_off[(uint64_t)b * t.G + blockIdx.x];
  const uint64_t c0 = (uint64_t)blockIdx.x * t.chunk;
  const uint64_t c1 = c0 + t.chunk < n ? c0 + t.chunk : n;
  const uint32_t per_thread_b = (t.B + kTlThreads - 1) / kTlThreads;
  In cur[4][4], nxt[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) Load4<In>::run(in, c0 + q * 1024 + threadIdx.x * 4, c1, aligned, cur[q]);
  for (uint64_t base = c0; base < c1; base += kTlTile) {
    for (uint32_t b = threadIdx.x; b <= t.B; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    const uint64_t nb = base + kTlTile;
    if (nb < c1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) Load4<In>::run(in, nb + q * 1024 + threadIdx.x * 4, c1, aligned, nxt[q]);
    }
    uint32_t bk[16], lo[16], rk[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i0 = base + q * 1024 + threadIdx.x * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bk[q * 4 + e] = 0xffffffffu;
        if (i0 + e < c1) {
          unsigned flags = 0;
          const unsigned long long k = map(cur[q][e], flags);
          if (k < t.cells) {
            const uint32_t b = tl_bucket(static_cast<uint32_t>(k), t);
            bk[q * 4 + e] = b;
            lo[q * 4 + e] = static_cast<uint32_t>(k) - b * t.S;
            rk[q * 4 + e] = atomicAdd(&s_cnt[b], 1u);
          }
        }
      }
    }
    __syncthreads();
    // exclusive scan of s_cnt over buckets (per_thread_b consecutive per
    // thread); s_cnt[B] becomes the number of staged keys
    {
      uint32_t sum = 0;
      const uint32_t b0 = threadIdx.x * per_thread_b;
      for (uint32_t j = 0; j < per_thread_b; ++j)
        if (b0 + j < t.B) sum += s_cnt[b0 + j];
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
        for (int w = 0; w < kTlThreads / 32; ++w) {
          const uint32_t c = s_scan[w];
          s_scan[w] = r;
          r += c;
        }
        s_cnt[t.B] = r;
      }
      __syncthreads();
      uint32_t run = s_scan[warp] + inc - sum;
      for (uint32_t j = 0; j < per_thread_b; ++j) {
        if (b0 + j < t.B) {
          const uint32_t c = s_cnt[b0 + j];
          s_cnt[b0 + j] = run;  // tile-local start of bucket
          run += c;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (bk[j] != 0xffffffffu) s_low[s_cnt[bk[j]] + rk[j]] = static_cast<uint16_t>(lo[j]);
    __syncthreads();
    // keys outside the grid were never staged (K1a flagged the overflow and
    // the sort is redone with the derived width).  One warp per bucket run.
    for (uint32_t b = warp; b < t.B; b += kTlThreads / 32) {
      const uint32_t s = s_cnt[b], e = s_cnt[b + 1];
      uint16_t* dst = lows + s_cur[b] - s;
      for (uint32_t i = s + lane; i < e; i += 32) dst[i] = s_low[i];
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) s_cur[b] += s_cnt[b + 1] - s_cnt[b];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) cur[q][e] = nxt[q][e];
    __syncthreads();
  }
}

// ------------------------------------------------------------- K2
// Slice j of the partitioned inner digits covers [j*L, (j+1)*L).  Buckets
// overlapping it are walked in order; each gets a shared histogram over its
// S cells, flushed once into counts[b*S + c].
__global__ void __launch_bounds__(kTlThreads) k_inner_count(const uint16_t* __restrict__ lows, uint64_t n,
                                                            const uint32_t* __restrict__ bucket_start,  // [B+1]
                                                            TwoLevel t, uint64_t slice,
                                                            uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_c[];  // [S]
  __shared__ uint32_t s_b0;
  const uint64_t p0 = (uint64_t)blockIdx.x * slice;
  const uint64_t p1 = p0 + slice < n ? p0 + slice : n;
  if (threadIdx.x == 0) {  // last bucket whose start <= p0
    uint32_t lo = 0, hi = t.B;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (bucket_start[mid] <= p0) lo = mid;
      else hi = mid;
    }
    s_b0 = lo;
  }
  __syncthreads();
  for (uint32_t b = s_b0; b < t.B && bucket_start[b] < p1; ++b) {
    const uint64_t a = bucket_start[b] > p0 ? bucket_start[b] : p0;
    const uint64_t e = bucket_start[b + 1] < p1 ? bucket_start[b + 1] : p1;
    if (a >= e) continue;
    for (uint32_t c = threadIdx.x; c < t.S; c += blockDim.x) s_c[c] = 0;
    __syncthreads();
    // 8 inner digits (16 bytes) per thread per step where aligned
    uint64_t i = a + threadIdx.x;
    const uint64_t a8 = (a + 7) & ~7ull;
    if (a8 < e) {
      for (uint64_t h = a + threadIdx.x; h < a8; h += blockDim.x) atomicAdd(&s_c[lows[h]], 1u);
      const uint64_t nv = (e - a8) / 8;
      const uint4* v = reinterpret_cast<const uint4*>(lows + a8);
      for (uint64_t q = threadIdx.x; q < nv; q += blockDim.x) {
        const uint4 w = __ldcs(v + q);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          atomicAdd(&s_c[ws[k] & 0xffffu], 1u);
          atomicAdd(&s_c[ws[k] >> 16], 1u);
        }
      }
      i = a8 + nv * 8 + threadIdx.x;
    }
    for (; i < e; i += blockDim.x) atomicAdd(&s_c[lows[i]], 1u);
    __syncthreads();
    const unsigned long long cb = (unsigned long long)b * t.S;
    for (uint32_t c = threadIdx.x; c < t.S; c += blockDim.x)
      if (s_c[c] && cb + c < t.cells) atomicAdd(&counts[cb + c], s_c[c]);
    __syncthreads();
  }
}

// bucket_start[b] = cta_off[b*G] (first CTA's offset), bucket_start[B] = total.
__global__ void k_bucket_starts(const uint32_t* __restrict__ cta_off, TwoLevel t,
                                const unsigned long long* total, uint32_t* __restrict__ bucket_start) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < t.B) bucket_start[b] = cta_off[(uint64_t)b * t.G];
  if (b == t.B) bucket_start[b] = static_cast<uint32_t>(*total);
}

}  // namespace rsb

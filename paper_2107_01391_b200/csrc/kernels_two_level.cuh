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
//   K1 tile_partition  one CTA per 8192-key tile: map each key to its cell,
//                      counting-sort the tile by outer bucket in shared
//                      memory and write the inner digits (uint16) back to
//                      the tile's own slot, fully coalesced; per-(bucket,
//                      tile) counts and in-tile starts go to two small
//                      tables; max / flags / overflow fused               R4 + W2
//   scan               exclusive scan of the bucket-major [B][T] counts
//   work list          each bucket cut into groups of ~target keys
//   K2 inner_gather    one CTA per group: gathers the bucket's runs (~80
//                      keys each) from consecutive tiles, shared histogram
//                      over the S inner cells, one flush into the dense
//                      count grid                                        R2
// after which the occupancy scan and the load-balanced emit run unchanged.
// No histogram pre-pass is needed: each tile sorts only itself.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_grid.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kTlThreads = 512;
constexpr int kTlPerThread = 16;
constexpr int kTlTile = kTlThreads * kTlPerThread;  // 8192 keys per tile
constexpr uint32_t kTlMaxBuckets = 4096;            // outer buckets
constexpr uint32_t kTlMaxInner = 16384;             // inner cells (smem hist <= 64 KB)
constexpr int kGatherThreads = 256;

struct TwoLevel {
  unsigned long long cells;  // grid size C
  uint32_t S;                // inner cells per bucket
  uint32_t B;                // outer buckets = ceil(C / S)
  unsigned long long magic;  // bucket = (cell * magic) >> shift, exact for cell < 2^32
  uint32_t shift;
  uint32_t T;                // tiles = ceil(n / kTlTile)
  uint64_t target;           // keys per K2 group
};

__device__ __forceinline__ uint32_t tl_bucket(uint32_t cell, const TwoLevel& t) {
  return static_cast<uint32_t>((static_cast<unsigned long long>(cell) * t.magic) >> t.shift);
}

__device__ __forceinline__ uint32_t from_bits32(uint32_t w, uint32_t*) { return w; }
__device__ __forceinline__ int32_t from_bits32(uint32_t w, int32_t*) { return static_cast<int32_t>(w); }
__device__ __forceinline__ double from_bits64(unsigned long long w, double*) { return __longlong_as_double(static_cast<long long>(w)); }
__device__ __forceinline__ unsigned long long from_bits64(unsigned long long w, unsigned long long*) { return w; }
__device__ __forceinline__ int64_t from_bits64(unsigned long long w, int64_t*) { return static_cast<int64_t>(w); }

// Elements i0..i0+3 (16-byte vector loads when the input is aligned).
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

// ------------------------------------------------------------- K1
// Shared layout (kTilePartitionSmem(B)): s_cnt[B+1] counts -> starts,
// s_low[kTlTile] inner digits in bucket order.
__host__ __device__ constexpr size_t kTilePartitionSmem(uint32_t B) {
  return (((size_t)B + 1) * 4 + 15) / 16 * 16 + (size_t)kTlTile * 2;
}

template <class Map>
__global__ void __launch_bounds__(kTlThreads) k_tile_partition(const typename Map::In* __restrict__ in, uint64_t n,
                                                               Map map, TwoLevel t, bool aligned,
                                                               uint16_t* __restrict__ lows,       // [T][kTlTile]
                                                               uint32_t* __restrict__ cnt_bm,     // [B][T]
                                                               uint16_t* __restrict__ start_tm,   // [T][B]
                                                               DevStats* st) {
  using In = typename Map::In;
  extern __shared__ __align__(16) unsigned char tl_smem[];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(tl_smem);
  uint16_t* s_low = reinterpret_cast<uint16_t*>(tl_smem + (((size_t)t.B + 1) * 4 + 15) / 16 * 16);
  __shared__ uint32_t s_scan[kTlThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tile = blockIdx.x;
  const uint64_t base = (uint64_t)tile * kTlTile;
  const uint64_t end = base + kTlTile < n ? base + kTlTile : n;
  for (uint32_t b = threadIdx.x; b <= t.B; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  unsigned long long mx = 0;
  unsigned flags = 0, ovf = 0;
  uint32_t pk[kTlPerThread];  // bucket << 16 | rank   (0xffffffff = not counted)
  uint16_t lo[kTlPerThread];
#pragma unroll
  for (int q = 0; q < kTlPerThread / 4; ++q) {
    const uint64_t i0 = base + q * (kTlThreads * 4) + threadIdx.x * 4;
    In v[4];
    Load4<In>::run(in, i0, end, aligned, v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pk[q * 4 + e] = 0xffffffffu;
      lo[q * 4 + e] = 0;
      if (i0 + e < end) {
        const unsigned long long k = map(v[e], flags);
        mx = k > mx ? k : mx;
        if (k < t.cells) {
          const uint32_t b = tl_bucket(static_cast<uint32_t>(k), t);
          lo[q * 4 + e] = static_cast<uint16_t>(static_cast<uint32_t>(k) - b * t.S);
          pk[q * 4 + e] = (b << 16) | atomicAdd(&s_cnt[b], 1u);
        } else {
          ovf = 1;
        }
      }
    }
  }
  __syncthreads();
  // counts out (bucket-major for the scan), then exclusive scan in place
  const uint32_t per = (t.B + kTlThreads - 1) / kTlThreads;
  const uint32_t b0 = threadIdx.x * per;
  uint32_t sum = 0;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t b = b0 + j;
    if (b < t.B) {
      const uint32_t c = s_cnt[b];
      cnt_bm[(uint64_t)b * t.T + tile] = c;
      sum += c;
    }
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
    for (int w = 0; w < kTlThreads / 32; ++w) {
      const uint32_t c = s_scan[w];
      s_scan[w] = r;
      r += c;
    }
  }
  __syncthreads();
  uint32_t run = s_scan[warp] + inc - sum;
  for (uint32_t j = 0; j < per; ++j) {
    const uint32_t b = b0 + j;
    if (b < t.B) {
      const uint32_t c = s_cnt[b];
      s_cnt[b] = run;
      start_tm[(uint64_t)tile * t.B + b] = static_cast<uint16_t>(run);
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kTlPerThread; ++j)
    if (pk[j] != 0xffffffffu) s_low[s_cnt[pk[j] >> 16] + (pk[j] & 0xffffu)] = lo[j];
  __syncthreads();
  // the whole tile slot, 16-byte stores (entries past the counted keys are
  // never read: K2 reads exactly each bucket's run)
  uint4* dst = reinterpret_cast<uint4*>(lows + base);
  const uint4* src = reinterpret_cast<const uint4*>(s_low);
  for (uint32_t i = threadIdx.x; i < kTlTile / 8; i += blockDim.x) __stcs(dst + i, src[i]);
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

// ------------------------------------------------------ K2 work list
// groups[b] = ceil(total_b / target); work_start = exclusive scan (one CTA,
// B <= 4096).  off_bm is the exclusive scan of cnt_bm, so bucket b's keys
// are [off_bm[b*T], off_bm[(b+1)*T]) in bucket-major order.
__global__ void k_work_list(const uint32_t* __restrict__ off_bm, const unsigned long long* total, TwoLevel t,
                            uint32_t* __restrict__ work_start) {
  __shared__ uint32_t s_w[1024];
  const uint32_t per = (t.B + blockDim.x - 1) / blockDim.x;
  uint32_t g[8];
  uint32_t sum = 0;
  for (uint32_t j = 0; j < per && j < 8; ++j) {
    const uint32_t b = threadIdx.x * per + j;
    g[j] = 0;
    if (b < t.B) {
      const unsigned long long lo = off_bm[(uint64_t)b * t.T];
      const unsigned long long hi = (b + 1 < t.B) ? off_bm[(uint64_t)(b + 1) * t.T] : *total;
      g[j] = static_cast<uint32_t>((hi - lo + t.target - 1) / t.target);
    }
    sum += g[j];
  }
  s_w[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < blockDim.x; ++i) {
      const uint32_t c = s_w[i];
      s_w[i] = r;
      r += c;
    }
    work_start[t.B] = r;
  }
  __syncthreads();
  uint32_t run = s_w[threadIdx.x];
  for (uint32_t j = 0; j < per && j < 8; ++j) {
    const uint32_t b = threadIdx.x * per + j;
    if (b < t.B) work_start[b] = run;
    run += g[j];
  }
}

// --------------------------------------------------------------- K2
// CTA w -> bucket b (work_start[b] <= w < work_start[b+1]), group g = w -
// work_start[b], bucket-local key range [g*target, (g+1)*target).  Tiles are
// found by binary search over off_bm[b][*]; each warp walks tiles and its
// lanes count the run's inner digits into the shared histogram.
__global__ void __launch_bounds__(kGatherThreads) k_inner_gather(const uint16_t* __restrict__ lows,
                                                                 const uint32_t* __restrict__ off_bm,
                                                                 const uint32_t* __restrict__ cnt_bm,
                                                                 const uint16_t* __restrict__ start_tm,
                                                                 const uint32_t* __restrict__ work_start,
                                                                 const unsigned long long* total, TwoLevel t,
                                                                 uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_c[];  // [S]
  __shared__ uint32_t s_b, s_t0, s_t1;
  __shared__ unsigned long long s_k0, s_k1;
  const uint32_t w = blockIdx.x;
  if (w >= work_start[t.B]) return;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = t.B;  // last b with work_start[b] <= w
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (work_start[mid] <= w) lo = mid;
      else hi = mid;
    }
    const uint32_t b = lo;
    const uint32_t g = w - work_start[b];
    const uint32_t* row = off_bm + (uint64_t)b * t.T;
    const unsigned long long bstart = row[0];
    const unsigned long long bend = (b + 1 < t.B) ? off_bm[(uint64_t)(b + 1) * t.T] : *total;
    unsigned long long k0 = bstart + (unsigned long long)g * t.target;
    unsigned long long k1 = k0 + t.target < bend ? k0 + t.target : bend;
    // first tile whose run ends after k0: last t with row[t] <= k0
    uint32_t a = 0, z = t.T;
    while (z - a > 1) {
      const uint32_t mid = (a + z) >> 1;
      if (row[mid] <= k0) a = mid;
      else z = mid;
    }
    uint32_t c = a, e = t.T;  // first t with row[t] >= k1
    while (c < e) {
      const uint32_t mid = (c + e) >> 1;
      if (row[mid] >= k1) e = mid;
      else c = mid + 1;
    }
    s_b = b;
    s_t0 = a;
    s_t1 = c;
    s_k0 = k0;
    s_k1 = k1;
  }
  for (uint32_t i = threadIdx.x; i < t.S; i += blockDim.x) s_c[i] = 0;
  __syncthreads();
  const uint32_t b = s_b;
  const unsigned long long k0 = s_k0, k1 = s_k1;
  const uint32_t* row = off_bm + (uint64_t)b * t.T;
  const uint32_t* crow = cnt_bm + (uint64_t)b * t.T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t tt = s_t0 + warp; tt < s_t1; tt += kGatherThreads / 32) {
    const unsigned long long r0 = row[tt];
    const unsigned long long r1 = r0 + crow[tt];
    const unsigned long long a = r0 > k0 ? r0 : k0;
    const unsigned long long z = r1 < k1 ? r1 : k1;
    if (a >= z) continue;
    const uint16_t* src = lows + (uint64_t)tt * kTlTile + start_tm[(uint64_t)tt * t.B + b] + (a - r0);
    const uint32_t len = static_cast<uint32_t>(z - a);
    for (uint32_t i = lane; i < len; i += 32) atomicAdd(&s_c[src[i]], 1u);
  }
  __syncthreads();
  const unsigned long long cb = (unsigned long long)b * t.S;
  for (uint32_t c = threadIdx.x; c < t.S; c += blockDim.x)
    if (s_c[c] && cb + c < t.cells) atomicAdd(&counts[cb + c], s_c[c]);
}

}  // namespace rsb

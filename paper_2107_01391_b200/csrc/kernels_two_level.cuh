// kernels_two_level.cuh — the counting pass for grids too large for one
// shared-memory histogram (10^6 cells at cfg2/cfg3).
//
// Measured on B200 (tools/microbench.cu, profiles/r1_microbench.txt): an
// L2-atomic histogram of 2^28 keys over 10^6 cells takes 1.49 ms (181 G
// atomics/s) while a shared-memory histogram of <= 4096 bins takes 0.20 ms at
// 5.3 TB/s.  So the Cartesian grid is split as outer x inner: the leading
// digits pick one of B outer buckets and the trailing digits one of S inner
// cells (10^6 = 100 x 10^4):
//
//   K1 page_partition  persistent CTAs stream tiles of 4096 keys: map each
//                      key to its cell, counting-sort the tile by outer
//                      bucket in shared memory and append each bucket's
//                      run of inner digits (uint16) to that bucket's current
//                      2 KB page in the CTA's private page region; pages are
//                      taken from a shared-memory counter (no global
//                      atomics, no pre-pass); max / flags / overflow fused  R4 + W2
//   page lists         per-(bucket, CTA) page counts scanned bucket-major,
//                      page ids listed per bucket
//   K2 page_count      one CTA per group of a bucket's pages: streams whole
//                      pages, shared histogram over the S inner cells, one
//                      flush into the dense count grid                   R2
// after which the occupancy scan and the load-balanced emit run unchanged.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "bulk_copy.cuh"
#include "kernels_grid.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kTlThreads = 256;
constexpr int kTlPerThread = 16;
constexpr int kTlTile = kTlThreads * kTlPerThread;  // 4096 keys per tile
constexpr uint32_t kTlMaxBuckets = 1024;            // outer buckets
constexpr uint32_t kTlMaxInner = 16384;             // inner cells (smem hist <= 64 KB)
constexpr uint32_t kPage = 1024;                    // inner digits per page (2 KB)
constexpr uint16_t kPagePad = 0xffff;               // padding entry (inner digits are < 16384)
constexpr int kGatherThreads = 256;
constexpr int kTlRep = 4;                           // lane replicas of a bucket's rank counter (skewed tiles)
constexpr uint32_t kMaxGroupPages = 256;            // pages per page-count work item (16 * S / kPage <= 256)

struct TwoLevel {
  unsigned long long cells;  // grid size C
  uint32_t S;                // inner cells per bucket
  uint32_t B;                // outer buckets = ceil(C / S)
  unsigned long long magic;  // bucket = (cell * magic) >> shift, exact for cell < 2^32
  uint32_t shift;
  uint32_t T;                // tiles = ceil(n / kTlTile)
  uint32_t G;                // persistent partition CTAs
  uint32_t pages_per_cta;    // page region of one CTA
  uint32_t group_pages;      // pages per K2 work item
  uint32_t negS;             // 0 - S: inner digit = cell + bucket * negS, one multiply-add from the constant bank
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
  unsigned long long r = 0, before = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    before += w < warp ? s_w[w] : 0ull;
    r += s_w[w];
  }
  if (warp == 0) {
    volatile unsigned long long* vd = desc;
    unsigned long long p = 0;
    if (tile == 0) {
      if (lane == 0) vd[0] = kDescPre | r;
    } else {
      if (lane == 0) vd[tile] = kDescAgg | r;
      p = warp_lookback(vd, tile);
      if (lane == 0) vd[tile] = kDescPre | (p + r);
    }
    if (lane == 0) {
      s_prefix = p;
      if (tile == num_tiles - 1) *total = p + r;
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + before + inc - sum;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (i0 + k < count) out[i0 + k] = static_cast<uint32_t>(run);
    run += v[k];
  }
}

// ------------------------------------------------------------- K1
// Dynamic shared layout (kPagePartitionSmem(B)): s_cnt[B+1] tile counts ->
// starts, s_page[B] current page per bucket, s_fill[B] its fill, s_np[B]
// pages opened per bucket, s_low[kTlTile] staged inner digits.
__host__ __device__ constexpr size_t kPagePartitionOffset(uint32_t B) {
  return (((size_t)B + 2) * 4 + (size_t)B * 12 + 15) / 16 * 16 + (size_t)B * 16;
}
__host__ __device__ constexpr size_t kPagePartitionSmem(uint32_t B) {
  return kPagePartitionOffset(B) + (size_t)kTlTile * 4;  // staged (bucket << 16 | inner digit)
}

template <class Map>
__global__ void __launch_bounds__(kTlThreads) k_page_partition(const typename Map::In* __restrict__ in, uint64_t n,
                                                               Map map, TwoLevel t, bool aligned,
                                                               uint16_t* __restrict__ pages,        // [G*ppc][kPage]
                                                               uint16_t* __restrict__ page_bucket,  // [G*ppc]
                                                               uint16_t* __restrict__ page_fill,    // [G*ppc]
                                                               uint32_t* __restrict__ pc_bm,        // [B][G]
                                                               DevStats* st) {
  using In = typename Map::In;
  extern __shared__ __align__(16) unsigned char tl_smem[];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(tl_smem);  // [B+2]: buckets, staged total, dummy
  uint32_t* s_page = s_cnt + t.B + 2;                       // [B]
  uint32_t* s_fill = s_page + t.B;                          // [B]
  uint32_t* s_np = s_fill + t.B;                            // [B]
  // per bucket, this tile: {run start in staging, dest of rank r < thr = A + r,
  // else Bv + r, thr} (dest = index into the CTA's page region)
  uint4* s_dst = reinterpret_cast<uint4*>(tl_smem + (((size_t)t.B + 2) * 4 + (size_t)t.B * 12 + 15) / 16 * 16);
  uint32_t* s_stage = reinterpret_cast<uint32_t*>(tl_smem + kPagePartitionOffset(t.B));
  __shared__ uint32_t s_scan[kTlThreads / 32];
  __shared__ uint32_t s_next;  // next free page of this CTA's region
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t page0 = blockIdx.x * t.pages_per_cta;
  uint16_t* my_pages = pages + (uint64_t)page0 * kPage;
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) {
    s_page[b] = 0xffffffffu;
    s_fill[b] = kPage;  // "full": the first key of a bucket opens a page
    s_np[b] = 0;
  }
  if (threadIdx.x == 0) s_next = 0;
  unsigned long long mx = 0;
  uint32_t mx32 = 0;
  const uint32_t cells32 = t.cells > 0xFFFFFFFFull ? 0xFFFFFFFFu : static_cast<uint32_t>(t.cells);
  unsigned flags = 0, ovf = 0;
  const uint32_t per = (t.B + kTlThreads - 1) / kTlThreads;
  In cur[4][4], nxt[4][4];
  uint32_t tile = blockIdx.x;
  if (tile < t.T) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      Load4<In>::run(in, (uint64_t)tile * kTlTile + q * 1024 + threadIdx.x * 4, n, aligned, cur[q]);
  }
  for (; tile < t.T; tile += gridDim.x) {
    const uint64_t base = (uint64_t)tile * kTlTile;
    const uint32_t nt = tile + gridDim.x;
    if (nt < t.T) {  // software pipeline: the next tile's loads are in flight
#pragma unroll
      for (int q = 0; q < 4; ++q)
        Load4<In>::run(in, (uint64_t)nt * kTlTile + q * 1024 + threadIdx.x * 4, n, aligned, nxt[q]);
    }
    for (uint32_t b = threadIdx.x; b <= t.B + 1; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    // Branch-free key loop: keys that are past the end or outside the grid
    // are counted in the dummy bin B+1 and never staged.
    uint32_t pk[kTlPerThread];  // bucket << 16 | rank in tile
    uint32_t lo2[kTlPerThread / 2];
    const bool full = base + kTlTile <= n;
    const uint32_t dummy = t.B + 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i0 = base + q * 1024 + threadIdx.x * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = full || i0 + e < n;
        uint32_t b, l;
        if constexpr (sizeof(typename Map::Key) == 4) {
          // 32-bit keys: compares, max and bucket math stay 32-bit
          const uint32_t kk = map.key32(cur[q][e], flags);
          const bool in = ok && kk < cells32;
          ovf |= ok && !in;
          mx32 = (ok && kk > mx32) ? kk : mx32;
          const uint32_t bk = tl_bucket(kk, t);
          b = in ? bk : dummy;
          l = kk - bk * t.S;
        } else {
          // 64-bit mapped keys (float64 / int64 mappers are heavy): branch so
          // the mapper and bucket math only run for real keys
          b = dummy;
          l = 0;
          if (ok) {
            const unsigned long long kk = map(cur[q][e], flags);
            mx = kk > mx ? kk : mx;
            if (kk < t.cells) {
              b = tl_bucket(static_cast<uint32_t>(kk), t);
              l = static_cast<uint32_t>(kk) - b * t.S;
            } else {
              ovf = 1;
            }
          }
        }
        pk[q * 4 + e] = (b << 16) | atomicAdd(&s_cnt[b], 1u);
        if (e & 1) lo2[(q * 4 + e) >> 1] |= (l & 0xffffu) << 16;
        else lo2[(q * 4 + e) >> 1] = l & 0xffffu;
      }
    }
    __syncthreads();
    {  // exclusive scan of s_cnt over buckets; s_cnt[B] = staged keys
      uint32_t sum = 0;
      const uint32_t b0 = threadIdx.x * per;
      for (uint32_t j = 0; j < per; ++j)
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
      for (uint32_t j = 0; j < per; ++j) {
        if (b0 + j < t.B) {
          const uint32_t c = s_cnt[b0 + j];
          s_cnt[b0 + j] = run;
          run += c;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kTlPerThread; ++j) {
      const uint32_t b = pk[j] >> 16;
      if (b != dummy)
        s_stage[s_cnt[b] + (pk[j] & 0xffffu)] = (b << 16) | ((lo2[j >> 1] >> ((j & 1) * 16)) & 0xffffu);
    }
    // page bookkeeping, one thread per bucket: a run that does not fit the
    // current page spills into freshly allocated consecutive pages
    for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) {
      const uint32_t len = s_cnt[b + 1] - s_cnt[b];
      if (len == 0) continue;
      uint32_t fill = s_fill[b], pg = s_page[b];
      const uint32_t room = (pg == 0xffffffffu) ? 0u : kPage - fill;
      uint32_t pa = pg, fa = fill, pb = 0;
      if (len > room) {
        const uint32_t extra = (len - room + kPage - 1) / kPage;
        const uint32_t first = atomicAdd(&s_next, extra);
        for (uint32_t j = 0; j < extra; ++j) page_bucket[page0 + first + j] = static_cast<uint16_t>(b);
        for (uint32_t j = 0; j + 1 < extra; ++j) page_fill[page0 + first + j] = static_cast<uint16_t>(kPage);
        if (pg != 0xffffffffu) page_fill[page0 + pg] = static_cast<uint16_t>(kPage);
        s_np[b] += extra;
        if (room == 0) {
          pa = first;
          fa = 0;
          pb = first + 1;
        } else {
          pb = first;
        }
        pg = first + extra - 1;
        fill = len - room - (extra - 1) * kPage;
      } else {
        fill += len;
      }
      s_fill[b] = fill;
      s_page[b] = pg;
      // continuation pages are consecutive, so rank r >= kPage - fa lands at
      // (pb - 1) * kPage + fa + r
      s_dst[b] = make_uint4(s_cnt[b], pa * kPage + fa, (pb - 1) * kPage + fa, kPage - fa);
    }
    __syncthreads();
    // element-parallel copy of the staged runs into their pages
    const uint32_t staged = s_cnt[t.B];
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < staged; i += blockDim.x) {
      const uint32_t w = s_stage[i];
      const uint4 d = s_dst[w >> 16];
      const uint32_t r = i - d.x;
      my_pages[(r < d.w ? d.y : d.z) + r] = static_cast<uint16_t>(w);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) cur[q][e] = nxt[q][e];
    __syncthreads();
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) {
    if (s_page[b] != 0xffffffffu) page_fill[page0 + s_page[b]] = static_cast<uint16_t>(s_fill[b]);
    pc_bm[(uint64_t)b * t.G + blockIdx.x] = s_np[b];
  }
  warp_max_to(mx > mx32 ? mx : mx32, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}


// ------------------------------------------------------- K1 (TMA-fed)
// Partition for 16-byte aligned inputs with B <= 256: tiles of 4096 inputs
// arrive by 1D TMA bulk copies one tile ahead (double buffer); each key is
// mapped straight from the shared tile (uint32 keys: four 16-byte vectors
// per thread; 8-byte inputs: one element per thread per step, so only the
// 32-bit cells stay in registers).  One thread per bucket scans and keeps
// the page bookkeeping; the tile is staged by bucket in the consumed input
// buffer, each bucket run padded to 16 bytes, and written to its page(s) by
// TMA bulk stores.  Same page contents as k_page_partition<Map> (plus pad
// entries, skipped by k_page_count).
template <class Map>
__host__ __device__ constexpr size_t page_tma_smem() {
  return 2 * (size_t)kTlTile * sizeof(typename Map::In)  // s_in[2]; the consumed buffer stages the tile
         + 256 * 16                                      // s_run: this tile's run geometry per bucket
         + 258 * 4 * 4                                   // s_cnt, s_page, s_fill, s_np
         + 258 * 4 * (size_t)kTlRep;                     // s_rep
}
template <class Map>
constexpr int page_tma_min_blocks() { return sizeof(typename Map::In) == 4 ? 4 : 2; }

template <class Map>
__global__ void __launch_bounds__(kTlThreads, page_tma_min_blocks<Map>())
    k_page_partition_tma(const typename Map::In* __restrict__ in, uint64_t n, Map map, TwoLevel t,
                         uint16_t* __restrict__ pages, uint16_t* __restrict__ page_bucket,
                         uint16_t* __restrict__ page_fill, uint32_t* __restrict__ pc_bm, DevStats* st) {
  using In = typename Map::In;
  constexpr bool k32 = sizeof(In) == 4;
  extern __shared__ __align__(128) unsigned char sm[];
  In* s_in = reinterpret_cast<In*>(sm);                         // [2][kTlTile]
  uint4* s_run = reinterpret_cast<uint4*>(s_in + 2 * kTlTile);       // [256]: start, plen, dst_a, dst_b
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_run + 256);        // [258]: bucket totals -> starts
  uint32_t* s_page = s_cnt + 258;
  uint32_t* s_fill = s_page + 258;
  uint32_t* s_np = s_fill + 258;
  // rank counters, replica-major [kTlRep][258].  A tile whose predecessor had
  // a hot bucket (> 1/8 of the tile) spreads every bucket's atomics over
  // kTlRep lane replicas (same-address atomics serialise: skewed keys, cfg3's
  // Zipf half); otherwise all lanes use replica 0, the plain layout.
  uint32_t* s_rep = s_np + 258;
  const uint32_t lane_rep = threadIdx.x & (kTlRep - 1);
  uint32_t rmask = 0;  // 0: one counter per bucket; kTlRep-1: replicas
  __shared__ uint32_t s_scan[kTlThreads / 32];
  __shared__ uint32_t s_next;
  __shared__ __align__(8) unsigned long long s_bar[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t B = t.B, dummy = t.B + 1;
  const uint32_t cells32 = static_cast<uint32_t>(t.cells);
  const uint32_t page0 = blockIdx.x * t.pages_per_cta;
  uint16_t* my_pages = pages + (uint64_t)page0 * kPage;
  const uint32_t full_tiles = static_cast<uint32_t>(n / kTlTile);
  for (uint32_t i = threadIdx.x; i < 258 * kTlRep; i += kTlThreads) s_rep[i] = 0;
  if (threadIdx.x < 258) {
    s_cnt[threadIdx.x] = 0;
    s_page[threadIdx.x] = 0xffffffffu;
    s_fill[threadIdx.x] = kPage;
    s_np[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    s_next = 0;
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t tile, int b) {  // one thread
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[b], kTlTile * sizeof(In));
    bulk_g2s(s_in + b * kTlTile, in + (uint64_t)tile * kTlTile, kTlTile * sizeof(In), &s_bar[b]);
  };
  if (threadIdx.x == 0 && blockIdx.x < full_tiles) issue(blockIdx.x, 0);
  uint32_t mx32 = 0;
  unsigned long long mx64 = 0;
  unsigned flags = 0;
  const uint32_t magic32 = static_cast<uint32_t>(t.magic), shift32 = t.shift - 32;
  unsigned phase = 0;  // bit b: parity of buffer b's barrier
  int buf = 0;
  // element of the tile handled by (thread, j): 16-byte vectors for uint32
  auto elem = [&](int j) -> uint32_t {
    return k32 ? (uint32_t)((j >> 2) * 1024 + threadIdx.x * 4 + (j & 3)) : (uint32_t)(j * kTlThreads + threadIdx.x);
  };
  for (uint32_t tile = blockIdx.x; tile < t.T; tile += gridDim.x, buf ^= 1) {
    const uint32_t nt = tile + gridDim.x;
    if (threadIdx.x == 0 && nt < full_tiles) issue(nt, buf ^ 1);
    const bool full = tile < full_tiles;
    uint32_t kreg[k32 ? kTlPerThread : 1];
    if (full) {
      mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
      if constexpr (k32) {
        const uint4* src = reinterpret_cast<const uint4*>(s_in + buf * kTlTile);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = src[q * kTlThreads + threadIdx.x];
          kreg[4 * q] = v.x; kreg[4 * q + 1] = v.y; kreg[4 * q + 2] = v.z; kreg[4 * q + 3] = v.w;
        }
      }
    }
    uint32_t pk[kTlPerThread], lo2[kTlPerThread / 2];
    const uint32_t prev_mask = rmask;  // this tile's replica mask (rmask is updated for the next tile below)
    uint32_t* const my_cnt = s_rep + (lane_rep & rmask) * 258;  // this lane's counters for this tile
    // bucket = floor(cell / S) as one 32-bit high product (magic < 2^32,
    // shift >= 32); keys outside the grid count in the dummy bin B+1 and
    // raise the overflow flag through the running max (checked at the end)
    auto rank = [&](auto full_tile) {
      constexpr bool kFull = decltype(full_tile)::value;
#pragma unroll
      for (int j = 0; j < kTlPerThread; ++j) {
        bool ok = true;
        In v;
        if constexpr (kFull) {
          if constexpr (k32) v = static_cast<In>(kreg[j]);
          else v = s_in[buf * kTlTile + elem(j)];
        } else {
          const uint64_t i = (uint64_t)tile * kTlTile + elem(j);
          ok = i < n;
          v = ok ? in[i] : In{};
        }
        uint32_t kk;
        bool ing;
        if constexpr (k32) {
          kk = map.key32(v, flags);
          mx32 = (ok && kk > mx32) ? kk : mx32;
          ing = ok && kk < cells32;
        } else {
          const unsigned long long k64 = ok ? map(v, flags) : 0ull;
          mx64 = k64 > mx64 ? k64 : mx64;
          ing = ok && k64 < t.cells;
          kk = static_cast<uint32_t>(k64);
        }
        const uint32_t bk = __umulhi(kk, magic32) >> shift32;
        const uint32_t b = ing ? bk : dummy;
        pk[j] = (b << 16) | atomicAdd(&my_cnt[b], 1u);
        const uint32_t l = (kk - bk * t.S) & 0xffffu;
        if (j & 1) lo2[j >> 1] |= l << 16;
        else lo2[j >> 1] = l;
      }
    };
    if (full) rank(std::true_type{});
    else rank(std::false_type{});
    __syncthreads();
    // One thread per bucket: exclusive scan of the runs padded to 8 entries
    // (16 bytes) + page bookkeeping.  Pages fill in 8-entry units, so every
    // run and every page split stays 16-byte aligned for the bulk stores.
    uint16_t* stage = reinterpret_cast<uint16_t*>(s_in + buf * kTlTile);  // the tile was consumed above
    const uint32_t b = threadIdx.x;
    // the bucket's length: its replica counts summed
    uint32_t len = 0;
    if (b < B) {
      len = s_rep[b];
      if (rmask)
#pragma unroll
        for (int r = 1; r < kTlRep; ++r) len += s_rep[r * 258 + b];
    }
    const uint32_t plen = (len + 7) & ~7u;
    {
      uint32_t start;
      uint32_t inc = plen;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_scan[warp] = inc;
      __syncthreads();
      uint32_t before = 0;
#pragma unroll
      for (int w = 0; w < kTlThreads / 32; ++w) before += w < warp ? s_scan[w] : 0u;
      start = before + inc - plen;
      if (b < B && len) {
        uint32_t fill = s_fill[b], pg = s_page[b];
        const uint32_t room = (pg == 0xffffffffu) ? 0u : kPage - fill;
        uint32_t pa = pg, fa = fill, pb = 0;
        if (plen > room) {
          const uint32_t extra = (plen - room + kPage - 1) / kPage;
          const uint32_t first = atomicAdd(&s_next, extra);
          for (uint32_t j = 0; j < extra; ++j) page_bucket[page0 + first + j] = static_cast<uint16_t>(b);
          for (uint32_t j = 0; j + 1 < extra; ++j) page_fill[page0 + first + j] = static_cast<uint16_t>(kPage);
          if (pg != 0xffffffffu) page_fill[page0 + pg] = static_cast<uint16_t>(kPage);
          s_np[b] += extra;
          if (room == 0) {
            pa = first;
            fa = 0;
            pb = first + 1;
          } else {
            pb = first;
          }
          pg = first + extra - 1;
          fill = plen - room - (extra - 1) * kPage;
        } else {
          fill += plen;
        }
        s_fill[b] = fill;
        s_page[b] = pg;
        // ranks < kPage - fa: the current page at pa*kPage + fa; the rest:
        // consecutive fresh pages from pb*kPage (parked in shared memory
        // across the staging step, which needs the registers)
        s_run[b] = make_uint4(start, plen, pa * kPage + fa, pb * kPage);
        for (uint32_t r = len; r < plen; ++r) stage[start + r] = kPagePad;
      }
      if (b < B) {  // replica counts become staging positions (exclusive, from the run start)
        if (rmask) {
          uint32_t run = start;
#pragma unroll
          for (int r = 0; r < kTlRep; ++r) {
            const uint32_t v = s_rep[r * 258 + b];
            s_rep[r * 258 + b] = run;
            run += v;
          }
        } else {
          s_rep[b] = start;
        }
      }
      __syncwarp();
      if (b < B) s_cnt[b] = start;
    }
    // the next tile spreads its atomics if this one had a hot bucket
    rmask = __syncthreads_or(b < B && len > kTlTile / 8) ? kTlRep - 1 : 0u;
    {  // branch-free: all 16 run starts are read up front (the dummy bin's counter is a valid read)
      uint32_t pos[kTlPerThread];
#pragma unroll
      for (int j = 0; j < kTlPerThread; ++j) pos[j] = my_cnt[pk[j] >> 16] + (pk[j] & 0xffffu);
#pragma unroll
      for (int j = 0; j < kTlPerThread; ++j)
        if ((pk[j] >> 16) != dummy) stage[pos[j]] = static_cast<uint16_t>(lo2[j >> 1] >> ((j & 1) * 16));
    }
    fence_proxy_async_smem();  // staged entries -> visible to the bulk stores
    __syncthreads();
    // every read of the counters is behind the barrier above: clear them for
    // the next tile (its atomics come after the barrier closing this tile)
    for (uint32_t i = threadIdx.x; i < 258 * (prev_mask + 1); i += kTlThreads) s_rep[i] = 0;
    if (b < B && len) {  // the run, as one or two TMA bulk stores
      const uint4 r = s_run[b];  // start, plen, dst_a, dst_b
      const uint32_t thr = kPage - (r.z & (kPage - 1));
      const uint32_t n1 = r.y < thr ? r.y : thr;
      bulk_s2g(my_pages + r.z, stage + r.x, n1 * 2);
      if (r.y > n1) bulk_s2g(my_pages + r.w, stage + r.x + n1, (r.y - n1) * 2);
      bulk_commit();
      bulk_wait_read();  // the buffer takes a later tile's load
    }
    __syncthreads();
  }
  for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
    if (s_page[b] != 0xffffffffu) page_fill[page0 + s_page[b]] = static_cast<uint16_t>(s_fill[b]);
    pc_bm[(uint64_t)b * t.G + blockIdx.x] = s_np[b];
  }
  const unsigned long long mx = k32 ? (unsigned long long)mx32 : mx64;
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (mx >= t.cells ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

// Page list grouped by bucket: CTA c walks its used pages (allocated densely
// from 0) and places page p of bucket b at list[po_bm[b][c] + rank].
__global__ void k_page_list(const uint16_t* __restrict__ page_bucket, const uint32_t* __restrict__ po_bm,
                            const uint32_t* __restrict__ pc_bm, TwoLevel t, uint32_t* __restrict__ list) {
  extern __shared__ uint32_t s_cur[];  // [B]
  __shared__ uint32_t s_used;
  const uint32_t c = blockIdx.x;
  if (threadIdx.x == 0) s_used = 0;
  __syncthreads();
  uint32_t used = 0;
  for (uint32_t b = threadIdx.x; b < t.B; b += blockDim.x) {
    s_cur[b] = po_bm[(uint64_t)b * t.G + c];
    used += pc_bm[(uint64_t)b * t.G + c];
  }
  atomicAdd(&s_used, used);
  __syncthreads();
  const uint32_t page0 = c * t.pages_per_cta;
  for (uint32_t p = threadIdx.x; p < s_used; p += blockDim.x) {
    const uint32_t b = page_bucket[page0 + p];
    list[atomicAdd(&s_cur[b], 1u)] = page0 + p;
  }
}

// The page table's scan and the page-count work list in one CTA, for page
// tables of at most kPageScanMax (bucket, CTA) entries (cfg2: 100 x 296):
// po_bm = exclusive scan of pc_bm, *total = the page count, and
// work_start = exclusive scan over buckets of ceil(pages_b / group_pages)
// (k_page_work's list) — in place of the look-back scan, its descriptor
// reset and k_page_work (three launches).
constexpr int kPageScanThreads = 1024;
constexpr uint32_t kPageScanPer = 32;
constexpr uint64_t kPageScanMax = (uint64_t)kPageScanThreads * kPageScanPer;
__global__ void __launch_bounds__(kPageScanThreads) k_page_scan(const uint32_t* __restrict__ pc_bm, uint32_t count,
                                                                 uint32_t* __restrict__ po_bm,
                                                                 unsigned long long* total, TwoLevel t,
                                                                 uint32_t* __restrict__ work_start) {
  __shared__ uint32_t s_w[kPageScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto block_scan = [&](uint32_t v, uint32_t& excl, uint32_t& all) {
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    const uint32_t tw = s_w[lane];
    uint32_t ti = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    excl = __shfl_sync(0xffffffffu, ti - tw, wid) + inc - v;
    all = __shfl_sync(0xffffffffu, ti, 31);
    __syncthreads();
  };
  // warp w scans entries [w*1024, (w+1)*1024) as 32 coalesced rows of 32
  const uint32_t base_e = wid * (32 * kPageScanPer);
  uint32_t ex[kPageScanPer];
  uint32_t carry = 0;
#pragma unroll
  for (uint32_t i = 0; i < kPageScanPer; ++i) {
    const uint32_t e = base_e + i * 32 + lane;
    ex[i] = e < count ? __ldcg(pc_bm + e) : 0u;
  }
#pragma unroll
  for (uint32_t i = 0; i < kPageScanPer; ++i) {
    const uint32_t x = ex[i];
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    ex[i] = carry + inc - x;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  uint32_t wbase, all;
  if (lane == 0) s_w[wid] = carry;
  __syncthreads();
  {
    const uint32_t tw = s_w[lane];
    uint32_t ti = tw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    wbase = __shfl_sync(0xffffffffu, ti - tw, wid);
    all = __shfl_sync(0xffffffffu, ti, 31);
  }
  __syncthreads();
#pragma unroll
  for (uint32_t i = 0; i < kPageScanPer; ++i) {
    const uint32_t e = base_e + i * 32 + lane;
    if (e < count) po_bm[e] = wbase + ex[i];
  }
  if (threadIdx.x == 0) *total = all;
  __syncthreads();  // po_bm visible to the CTA (global writes, same CTA)
  // bucket b's pages: [po_bm[b*G], po_bm[(b+1)*G]) -> groups of group_pages
  const uint32_t b = threadIdx.x;
  uint32_t g = 0;
  if (b < t.B) {
    const uint32_t lo = __ldcg(po_bm + (uint64_t)b * t.G);
    const uint32_t hi = (b + 1 < t.B) ? __ldcg(po_bm + (uint64_t)(b + 1) * t.G) : all;
    g = (hi - lo + t.group_pages - 1) / t.group_pages;
  }
  uint32_t ws, wall;
  block_scan(g, ws, wall);
  if (b < t.B) work_start[b] = ws;
  if (threadIdx.x == 0) work_start[t.B] = wall;
}

// Work list: bucket b owns list entries [po_bm[b*G], po_bm[(b+1)*G]), cut
// into groups of group_pages; work_start = exclusive scan of group counts.
__global__ void k_page_work(const uint32_t* __restrict__ po_bm, const unsigned long long* total, TwoLevel t,
                            uint32_t* __restrict__ work_start) {
  __shared__ uint32_t s_w[kTlMaxBuckets];
  const uint32_t b = threadIdx.x;
  uint32_t g = 0;
  if (b < t.B) {
    const uint32_t lo = po_bm[(uint64_t)b * t.G];
    const uint32_t hi = (b + 1 < t.B) ? po_bm[(uint64_t)(b + 1) * t.G] : static_cast<uint32_t>(*total);
    g = (hi - lo + t.group_pages - 1) / t.group_pages;
  }
  // exclusive scan of the group counts: warp scans, then the warp totals
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = g;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  uint32_t before = 0;
  for (uint32_t q = 0; q < wid; ++q) before += s_w[q];
  if (b < t.B) work_start[b] = before + inc - g;
  if (threadIdx.x == blockDim.x - 1) work_start[t.B] = before + inc;
}

// --------------------------------------------------------------- K2
// CTA w -> bucket b (work_start[b] <= w < work_start[b+1]) and its group of
// pages; streams the pages as a flat range of 16-byte slots (128 per page),
// shared histogram over the S inner cells, one flush into the grid.
__global__ void __launch_bounds__(kGatherThreads) k_page_count(const uint16_t* __restrict__ pages,
                                                               const uint16_t* __restrict__ page_fill,
                                                               const uint32_t* __restrict__ list,
                                                               const uint32_t* __restrict__ po_bm,
                                                               const uint32_t* __restrict__ work_start,
                                                               const unsigned long long* total, TwoLevel t,
                                                               uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_c[];  // [S + 1]
  __shared__ uint32_t s_b, s_p0, s_p1;
  __shared__ uint32_t s_pg[kMaxGroupPages], s_fl[kMaxGroupPages];  // the group's pages and fills
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
    const uint32_t first = po_bm[(uint64_t)b * t.G];
    const uint32_t last = (b + 1 < t.B) ? po_bm[(uint64_t)(b + 1) * t.G] : static_cast<uint32_t>(*total);
    const uint32_t p0 = first + (w - work_start[b]) * t.group_pages;
    s_b = b;
    s_p0 = p0;
    s_p1 = p0 + t.group_pages < last ? p0 + t.group_pages : last;
  }
  for (uint32_t i = threadIdx.x; i <= t.S; i += blockDim.x) s_c[i] = 0;  // [S]: dump bin of pad entries
  __syncthreads();
  const uint32_t np = s_p1 - s_p0;  // <= kMaxGroupPages
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
    const uint32_t page = list[s_p0 + i];
    s_pg[i] = page;
    s_fl[i] = page_fill[page];
  }
  __syncthreads();
  // 16-byte slots (8 entries); four independent loads in flight per thread
  constexpr uint32_t kSlots = kPage / 8;
  constexpr int kU = 4;
  const uint32_t nslots = np * kSlots;
  for (uint32_t s0 = threadIdx.x; s0 < nslots; s0 += kU * kGatherThreads) {
    uint4 v[kU];
    uint32_t lim[kU];  // valid entries in the slot
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t s = s0 + u * kGatherThreads;
      const uint32_t pi = s / kSlots, q = s % kSlots;
      const uint32_t fill = s < nslots ? s_fl[pi] : 0u;
      lim[u] = fill > q * 8 ? min(fill - q * 8, 8u) : 0u;
      v[u] = lim[u] ? __ldcs(reinterpret_cast<const uint4*>(pages + (uint64_t)s_pg[pi] * kPage) + q)
                    : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t ws[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      if (lim[u] == 8) {  // a full slot (all but a bucket's last page): pad entries land in the dump bin S
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          atomicAdd(&s_c[min(ws[j] & 0xffffu, t.S)], 1u);
          atomicAdd(&s_c[min(ws[j] >> 16, t.S)], 1u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t e0 = ws[j] & 0xffffu, e1 = ws[j] >> 16;
          if (2 * j < lim[u]) atomicAdd(&s_c[min(e0, t.S)], 1u);
          if (2 * j + 1 < lim[u]) atomicAdd(&s_c[min(e1, t.S)], 1u);
        }
      }
    }
  }
  __syncthreads();
  const unsigned long long cb = (unsigned long long)s_b * t.S;
  for (uint32_t c = threadIdx.x; c < t.S; c += blockDim.x)
    if (s_c[c] && cb + c < t.cells) atomicAdd(&counts[cb + c], s_c[c]);
}

}  // namespace rsb

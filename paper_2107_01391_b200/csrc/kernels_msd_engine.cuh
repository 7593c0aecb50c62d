// kernels_msd_engine.cuh — MSD bucket passes for keys too wide for one grid
// (the reference raises cell_budget_exceeded instead,
// key_model.cpp:72-76).
//
// Keys are 32- or 64-bit integers whose order is the sort order (uint32
// keys; fixed-width strings packed obits bits per symbol ordinal, which keeps
// lexicographic order because every ordinal < 32).  Each level splits every
// open segment by its next 8-bit digit — a 256-cell sub-grid of the
// Cartesian space:
//   k_msd_hist     per (segment, chunk) digit counts, layout per segment
//                  [digit][chunk]                                    R
//   exscan         ONE global look-back scan over all segments' tables:
//                  entry (s, d, c) minus entry (s, 0, 0) is the key's
//                  offset inside segment s
//   k_msd_scatter  tiles staged in shared memory by digit, runs written to
//                  the other buffer at their final positions           R + W
//   k_msd_classify each (segment, digit) run becomes a leaf or a segment
//                  of the next level
// Leaves (no key leaves its final position again):
//   k_leaf_grid    dense leaves (remaining bits <= 16, occupancy >= 1/16):
//                  the recombinant step itself — a shared-memory count grid
//                  over the remaining 2^bits cells, counts -> offsets, a
//                  counting-sort scatter through shared memory (run-length
//                  emit for segments too large to stage)                 R + W
//   k_leaf_radix   mid-size leaves (<= 4096 keys, <= 24 remaining bits):
//                  split by the top 11 remaining bits in shared memory,
//                  each key ranked by counting the smaller keys of its
//                  bucket and written straight to its place; skewed leaves:
//                  8-bit LSD passes (the first by returning atomics, then
//                  stable ballot ranks)                                  R + W
//   k_leaf_warp    tiny leaves (<= 32 keys): register bitonic network    R + W
//   k_leaf_bitonic small leaves of the last digit (<= 2048 keys)         R + W
//   k_leaf_copy    single keys / exhausted digits                        R + W
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels_grid.cuh"
#include "kernels_msd.cuh"
#include "bulk_copy.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kMsdDigitBits = 8;
constexpr int kMsdBins = 1 << kMsdDigitBits;
// keys per scatter tile: 32-bit keys 8192 (128-byte digit runs), 64-bit keys
// 4096 (the 64-bit register tile already costs ~120 registers at 4096)
template <class K>
__host__ __device__ constexpr int msd_tile() { return sizeof(K) == 4 ? 8192 : 4096; }
constexpr uint32_t kMsdChunk = 65536;   // keys per (segment, chunk) work item
constexpr uint32_t kLeafSmall = 2048;   // shared bitonic leaf capacity
constexpr uint32_t kLeafWarp = 32;      // warp (register) bitonic leaf capacity
constexpr uint32_t kLeafRadixMax = 4096;  // shared-memory LSD leaf: <= 4096 keys, <= 24 remaining bits
constexpr int kLeafRadixThreads = 256;     // one thread per top digit in the fast path
constexpr uint32_t kLeafRankMax = 32;       // largest bucket the fast path ranks by counting
static_assert(kLeafRadixThreads == 256, "the radix leaf's fast path keeps one top digit per thread");
constexpr int kLeafGridBits = 16;       // count-grid leaf: <= 2^16 cells (u16 pairs, 128 KB)
constexpr int kLeafGridThreads = 1024;  // one 128 KB CTA per SM: 32 warps to hide latency

struct MsdSeg {
  unsigned long long start;  // position in the array (final position)
  uint32_t size;
  uint32_t chunk0;           // first chunk of this segment in the level's chunk list
  uint32_t nchunks;
};

// ------------------------------------------------------------- loaders
// Level 0 reads the caller's input through a loader; deeper levels read keys
// from the ping-pong buffers.
template <class K>
struct LoadKeys {
  using Key = K;
  const K* p;
  unsigned long long n_total;  // readable elements at p (bulk copies never read past them)
  __device__ __forceinline__ K operator()(unsigned long long i) const { return __ldcs(p + i); }
  // A tile of up to kTile keys at a: 16-byte vectors when a is aligned
  // (thread t takes elements 4t..4t+3 of each 1024-element quarter), else
  // element j*256+t.  Order inside a tile is irrelevant to the partition.
  static constexpr int kTile = msd_tile<K>();
  __device__ __forceinline__ void load16(unsigned long long a, uint32_t tl, K (&k)[kTile / kMsdThreads]) {
    vec_ = (sizeof(K) == 4) && ((reinterpret_cast<uintptr_t>(p + a) & 15) == 0) && tl == kTile;
    if (vec_) {
#pragma unroll
      for (int q = 0; q < kTile / (4 * kMsdThreads); ++q) {
        const uint4 w = __ldcs(reinterpret_cast<const uint4*>(p + a) + q * kMsdThreads + threadIdx.x);
        k[4 * q] = static_cast<K>(w.x); k[4 * q + 1] = static_cast<K>(w.y);
        k[4 * q + 2] = static_cast<K>(w.z); k[4 * q + 3] = static_cast<K>(w.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kTile / kMsdThreads; ++j) {
        const uint32_t i = j * kMsdThreads + threadIdx.x;
        k[j] = i < tl ? __ldcs(p + a + i) : K(0);
      }
    }
  }
  __device__ __forceinline__ bool valid(int j, uint32_t tl) const {
    return vec_ || (uint32_t)(j * kMsdThreads + threadIdx.x) < tl;
  }
  bool vec_ = false;
};

// Fixed-width records -> packed key (obits bits per ordinal — the bit
// length of the largest ordinal, 5 for a-z — pad ordinal 0, first symbol
// most significant; width * obits <= 64).
struct LoadStr {
  using Key = unsigned long long;
  const uint8_t* recs;
  uint32_t width;
  const uint16_t* ord;  // device table (256 entries)
  static constexpr int kTile = msd_tile<Key>();
  __device__ __forceinline__ void load16(unsigned long long a, uint32_t tl, Key (&k)[kTile / kMsdThreads]) const {
#pragma unroll
    for (int j = 0; j < kTile / kMsdThreads; ++j) {
      const uint32_t i = j * kMsdThreads + threadIdx.x;
      k[j] = i < tl ? (*this)(a + i) : 0ull;
    }
  }
  __device__ __forceinline__ bool valid(int j, uint32_t tl) const { return (uint32_t)(j * kMsdThreads + threadIdx.x) < tl; }
  bool w8 = false;       // 8-byte records at an 8-byte aligned base: one 64-bit load each
  int lin = -1;          // contiguous alphabet: ordinal = byte - lin (symbols validated by k_str_scan)
  uint32_t obits = 5;
  __device__ __forceinline__ uint32_t ord_of(uint32_t c) const {
    return lin >= 0 ? c - static_cast<uint32_t>(lin) : __ldg(ord + c);
  }
  __device__ __forceinline__ unsigned long long operator()(unsigned long long i) const {
    if (w8) {
      const unsigned long long w = __ldcs(reinterpret_cast<const unsigned long long*>(recs) + i);
      unsigned long long k = 0;
      bool ended = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = static_cast<uint32_t>(w >> (8 * j)) & 0xffu;
        ended |= c == 0;
        const uint32_t o = ended ? 0u : ord_of(c);
        k = (k << obits) | o;
      }
      return k;
    }
    const uint8_t* r = recs + i * width;
    unsigned long long k = 0;
    bool ended = false;
    for (uint32_t j = 0; j < width; ++j) {
      uint32_t o = 0;
      if (!ended) {
        const uint8_t c = r[j];
        if (c == 0) ended = true;
        else o = ord_of(c);
      }
      k = (k << obits) | o;
    }
    return k;
  }
};

// ------------------------------------------------------------- emitters
template <class K>
struct EmitKey {
  K* out;
  __device__ __forceinline__ void operator()(unsigned long long pos, K key) const { out[pos] = key; }
};

// packed key -> record bytes (key_to_string, key_model.cpp:249-263: pad
// ordinals become NUL bytes)
struct EmitStr {
  uint8_t* out;
  uint32_t width;
  const uint8_t* sym;  // device: ordinal -> byte, sym[0] = 0
  int lin = -1;        // contiguous alphabet: byte = ordinal + lin (no table lookups)
  bool w8 = false;     // 8-byte records at an 8-byte aligned base: one 64-bit store each
  uint32_t obits = 5;  // bits per packed ordinal
  __device__ __forceinline__ uint32_t byte_of(uint32_t o) const {
    return lin >= 0 ? (o ? o + static_cast<uint32_t>(lin) : 0u) : sym[o];
  }
  __device__ __forceinline__ void operator()(unsigned long long pos, unsigned long long key) const {
    const uint32_t mask = (1u << obits) - 1u;
    if (w8) {
      unsigned long long w = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        w |= static_cast<unsigned long long>(byte_of(static_cast<uint32_t>(key >> (obits * (7 - j))) & mask)) << (8 * j);
      reinterpret_cast<unsigned long long*>(out)[pos] = w;
      return;
    }
    uint8_t* r = out + pos * width;
    for (int j = (int)width - 1; j >= 0; --j) {
      r[j] = static_cast<uint8_t>(byte_of(static_cast<uint32_t>(key) & mask));
      key >>= obits;
    }
  }
};

// ------------------------------------------------------------- level
// chunk -> (segment) map: chunk_seg[c] = s
__global__ void k_msd_chunks(const MsdSeg* __restrict__ segs, uint32_t nseg, uint32_t* __restrict__ chunk_seg) {
  const uint32_t s = blockIdx.x;
  if (s >= nseg) return;
  const MsdSeg g = segs[s];
  for (uint32_t c = threadIdx.x; c < g.nchunks; c += blockDim.x) chunk_seg[g.chunk0 + c] = s;
}

template <class Load>
__global__ void __launch_bounds__(kMsdThreads) k_msd_hist(Load ld, const MsdSeg* __restrict__ segs,
                                                          const uint32_t* __restrict__ chunk_seg, uint32_t shift,
                                                          uint32_t* __restrict__ table) {
  __shared__ uint32_t s_h[kMsdBins];
  const uint32_t c = blockIdx.x;
  const MsdSeg g = segs[chunk_seg[c]];
  const uint32_t ci = c - g.chunk0;
  for (int b = threadIdx.x; b < kMsdBins; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const unsigned long long a = g.start + (unsigned long long)ci * kMsdChunk;
  const uint32_t len = min(kMsdChunk, g.size - ci * kMsdChunk);
  for (uint32_t i = threadIdx.x; i < len; i += blockDim.x)
    atomicAdd(&s_h[(uint32_t)(ld(a + i) >> shift) & (kMsdBins - 1)], 1u);
  __syncthreads();
  uint32_t* t = table + (unsigned long long)g.chunk0 * kMsdBins;  // segment table [digit][chunk]
  for (int b = threadIdx.x; b < kMsdBins; b += blockDim.x) t[(unsigned long long)b * g.nchunks + ci] = s_h[b];
}

template <class Load>
constexpr size_t msd_scatter_smem() {  // tile buffers: two (TMA double buffer) for uint32 keys
  return (std::is_same<Load, LoadKeys<uint32_t>>::value ? 2 : 1) * (size_t)(msd_tile<typename Load::Key>() + 4) *
         sizeof(typename Load::Key);
}
template <class Load>
constexpr int msd_scatter_min_blocks() { return sizeof(typename Load::Key) == 4 ? 3 : 4; }

template <class Load>
__global__ void __launch_bounds__(kMsdThreads, msd_scatter_min_blocks<Load>()) k_msd_scatter(Load ld, const MsdSeg* __restrict__ segs,
                                                             const uint32_t* __restrict__ chunk_seg, uint32_t shift,
                                                             const uint32_t* __restrict__ off,
                                                             typename Load::Key* __restrict__ dst) {
  using K = typename Load::Key;
  constexpr int kTile = msd_tile<K>();
  // uint32 keys: tiles double-buffered by 1D TMA bulk copies (an aligned
  // superset of the tile, the offset skipped in shared memory); the consumed
  // buffer is reused as the output staging
  constexpr bool kBulk = std::is_same<Load, LoadKeys<uint32_t>>::value;
  constexpr int kPer = kTile / kMsdThreads;  // 16 keys per thread per tile
  __shared__ uint32_t s_base[kMsdBins];  // segment-relative destination of this tile's digit run, minus its start
  __shared__ uint32_t s_cur[kMsdBins];   // running segment-relative cursor per digit
  __shared__ uint32_t s_cnt[kMsdBins];
  extern __shared__ __align__(16) unsigned char msd_smem[];
  auto s_buf = reinterpret_cast<K(*)[kTile + 4]>(msd_smem);  // [kBulk ? 2 : 1][kTile + 4]
  __shared__ uint32_t s_scan[kMsdThreads / 32];
  __shared__ __align__(8) unsigned long long s_bar[2];
  const uint32_t c = blockIdx.x;
  const MsdSeg g = segs[chunk_seg[c]];
  const uint32_t ci = c - g.chunk0;
  const uint32_t* t = off + (unsigned long long)g.chunk0 * kMsdBins;
  const uint32_t base0 = t[0];
  for (int b = threadIdx.x; b < kMsdBins; b += blockDim.x) s_cur[b] = t[(unsigned long long)b * g.nchunks + ci] - base0;
  const unsigned long long a = g.start + (unsigned long long)ci * kMsdChunk;
  const uint32_t len = min(kMsdChunk, g.size - ci * kMsdChunk);
  const uint32_t ntiles = (len + kTile - 1) / kTile;
  K* seg_dst = dst + g.start;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tile u of this chunk: aligned superset [a+u*T - mis, ...) of round-up size
  auto tile_geo = [&](uint32_t u, uint32_t& mis, uint32_t& bytes, bool& ok) {
    if constexpr (kBulk) {
      const unsigned long long e0 = a + (unsigned long long)u * kTile;
      const uint32_t tl = min((uint32_t)kTile, len - u * kTile);
      mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(ld.p + e0) & 15) / sizeof(K));
      bytes = ((tl + mis) * (uint32_t)sizeof(K) + 15) & ~15u;
      ok = e0 - mis + bytes / sizeof(K) <= ld.n_total;
    } else {
      mis = bytes = 0;
      ok = false;
    }
  };
  unsigned phase = 0;  // bit b: parity of buffer b's barrier
  if constexpr (kBulk) {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t mis, bytes;
      bool ok;
      tile_geo(0, mis, bytes, ok);
      if (ok) {
        if constexpr (kBulk) {
          mbar_expect_tx(&s_bar[0], bytes);
          bulk_g2s(&s_buf[0][0], ld.p + a - mis, bytes, &s_bar[0]);
        }
      }
    }
  }
  for (uint32_t u = 0; u < ntiles; ++u) {
    const uint32_t t0 = u * kTile;
    const uint32_t tl = min((uint32_t)kTile, len - t0);
    const int buf = kBulk ? (u & 1) : 0;
    s_cnt[threadIdx.x] = 0;
    if constexpr (kBulk) {
      if (threadIdx.x == 0 && u + 1 < ntiles) {
        uint32_t mis, bytes;
        bool ok;
        tile_geo(u + 1, mis, bytes, ok);
        if (ok) {
          if constexpr (kBulk) {
            fence_proxy_async_smem();
            mbar_expect_tx(&s_bar[buf ^ 1], bytes);
            bulk_g2s(&s_buf[buf ^ 1][0], ld.p + a + t0 + kTile - mis, bytes, &s_bar[buf ^ 1]);
          }
        }
      }
    }
    __syncthreads();
    K k[kPer];
    uint32_t rk2[kPer / 2];  // ranks in the tile (< kTile), two per word; 0xffff = no key
    bool bulk_tile = false;
    if constexpr (kBulk) {
      uint32_t mis, bytes;
      tile_geo(u, mis, bytes, bulk_tile);
      if (bulk_tile) {
        mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const uint32_t i = j * kMsdThreads + threadIdx.x;
          k[j] = i < tl ? s_buf[buf][mis + i] : K(0);
        }
      }
    }
    if (!bulk_tile) ld.load16(a + t0, tl, k);  // element j*kMsdThreads + threadIdx.x (or a permutation)
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      uint32_t r = 0xffffu;
      const bool valid = bulk_tile ? (uint32_t)(j * kMsdThreads + threadIdx.x) < tl : ld.valid(j, tl);
      if (valid) r = atomicAdd(&s_cnt[(uint32_t)(k[j] >> shift) & (kMsdBins - 1)], 1u);
      if (j & 1) rk2[j >> 1] |= r << 16;
      else rk2[j >> 1] = r;
    }
    __syncthreads();
    {  // exclusive scan of 256 counts, one per thread
      const uint32_t v = s_cnt[threadIdx.x];
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_scan[warp] = inc;
      __syncthreads();
      uint32_t before = 0;
#pragma unroll
      for (int w = 0; w < kMsdThreads / 32; ++w) before += w < warp ? s_scan[w] : 0u;
      const uint32_t start = before + inc - v;
      s_base[threadIdx.x] = s_cur[threadIdx.x] - start;
      s_cur[threadIdx.x] += v;
      s_cnt[threadIdx.x] = start;
    }
    __syncthreads();
    K* stage = &s_buf[buf][0];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint32_t r = (rk2[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
      if (r != 0xffffu) stage[s_cnt[(uint32_t)(k[j] >> shift) & (kMsdBins - 1)] + r] = k[j];
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < tl; i += blockDim.x) {
      const K key = stage[i];
      seg_dst[s_base[(uint32_t)(key >> shift) & (kMsdBins - 1)] + i] = key;
    }
    __syncthreads();
  }
}

// Leaf / next-segment lists (device counters in cnt[0..3]: next, grid,
// small, copy).  Thread per (segment, digit).
struct MsdLists {
  MsdSeg* next;
  MsdSeg* leaf_grid;
  MsdSeg* leaf_small;
  MsdSeg* leaf_copy;
  MsdSeg* leaf_warp;
  MsdSeg* leaf_radix;
  unsigned* cnt;   // [6]: next, grid, small, copy, warp, radix
  unsigned* rmax;  // largest radix leaf
};

__global__ void k_msd_classify(const MsdSeg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ off,
                               uint32_t rem_bits, MsdLists L) {
  const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t s = static_cast<uint32_t>(idx / kMsdBins);
  const uint32_t d = static_cast<uint32_t>(idx % kMsdBins);
  if (s >= nseg) return;
  const MsdSeg g = segs[s];
  const uint32_t* t = off + (unsigned long long)g.chunk0 * kMsdBins;
  const uint32_t lo = t[(unsigned long long)d * g.nchunks] - t[0];
  const uint32_t hi = (d + 1 < kMsdBins) ? t[(unsigned long long)(d + 1) * g.nchunks] - t[0] : g.size;
  const uint32_t size = hi - lo;
  if (size == 0) return;
  const MsdSeg sub{g.start + lo, size, 0, 0};
  // rem_bits = bits below this level's digit
  if (rem_bits == 0 || size == 1) {
    L.leaf_copy[atomicAdd(&L.cnt[3], 1u)] = sub;
  } else if (rem_bits <= kLeafGridBits && size >= (1u << rem_bits) / 16 && size <= 65535u) {
    L.leaf_grid[atomicAdd(&L.cnt[1], 1u)] = sub;  // dense: the count grid
  } else if (size <= kLeafWarp) {
    L.leaf_warp[atomicAdd(&L.cnt[4], 1u)] = sub;  // small: one warp, registers
  } else if (size <= kLeafSmall && rem_bits <= kMsdDigitBits) {
    L.leaf_small[atomicAdd(&L.cnt[2], 1u)] = sub;  // last digit: shared bitonic
  } else if (size <= kLeafRadixMax && rem_bits <= 3 * kMsdDigitBits) {
    L.leaf_radix[atomicAdd(&L.cnt[5], 1u)] = sub;  // mid-size: shared-memory LSD passes
    atomicMax(L.rmax, size);
  } else {
    L.next[atomicAdd(&L.cnt[0], 1u)] = sub;  // split by the next 8-bit digit
  }
}

// Fill chunk0 / nchunks of a segment list (exclusive scan of chunk counts).
__global__ void k_msd_chunk_counts(const MsdSeg* __restrict__ segs, uint32_t nseg, uint32_t* __restrict__ counts) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) counts[s] = (segs[s].size + kMsdChunk - 1) / kMsdChunk;
}
__global__ void k_msd_chunk_assign(MsdSeg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ counts,
                                   const uint32_t* __restrict__ starts) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nseg) {
    segs[s].chunk0 = starts[s];
    segs[s].nchunks = counts[s];
  }
}

// ------------------------------------------------------------- leaves
template <class K, class Emit>
__global__ void k_leaf_copy(const K* __restrict__ src, const MsdSeg* __restrict__ segs, Emit emit) {
  const MsdSeg g = segs[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < g.size; i += blockDim.x) emit(g.start + i, src[g.start + i]);
}

// The recombinant step on a leaf: every key of the segment shares the bits
// above rem_bits, so a count grid over the 2^rem_bits remaining cells sorts
// it.  Counters are uint16 pairs in 32-bit words (segments hold < 65536
// keys); word w lives at w ^ ((w >> 5) & 31) so that threads scanning 32
// consecutive words each hit distinct banks.  Grid <= 2^16 cells = 128 KB.
//
// Segments up to `cap` keys (the shared memory left after the grid, as
// uint16 cells) are finished by a counting-sort scatter inside shared
// memory: counts become exclusive offsets in place, each key (re-read from
// L2) takes its rank with one returning shared atomic and drops its cell
// into the staging array, which is then written out in order — one coalesced
// store per key.  Larger segments walk the grid (run-length emit).
__host__ __device__ constexpr uint32_t leaf_grid_words(uint32_t rem_bits) { return ((1u << rem_bits) + 1) / 2; }
__device__ __forceinline__ uint32_t leaf_gw(uint32_t w) { return w ^ ((w >> 5) & 31u); }

template <class K, class Emit>
__global__ void __launch_bounds__(kLeafGridThreads) k_leaf_grid(const K* __restrict__ src,
                                                                const MsdSeg* __restrict__ segs, uint32_t rem_bits,
                                                                uint32_t cap, Emit emit, uint32_t nsegs,
                                                                uint32_t ahead) {
  extern __shared__ uint32_t s_w[];
  __shared__ uint32_t s_scan[kLeafGridThreads / 32];
  const MsdSeg g = segs[blockIdx.x];
  // One CTA per SM: the leaf `ahead` launches later (about the next wave on
  // this SM) is pulled into L2 now, one 128-byte line per thread, so its
  // first key loads hit L2 instead of waiting out DRAM latency.
  if (blockIdx.x + ahead < nsegs) {
    const MsdSeg h = segs[blockIdx.x + ahead];
    const char* base = reinterpret_cast<const char*>(src + h.start);
    const uint64_t bytes = (uint64_t)h.size * sizeof(K);
    for (uint64_t off = (uint64_t)threadIdx.x * 128; off < bytes; off += (uint64_t)kLeafGridThreads * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
  }
  const uint32_t cells = 1u << rem_bits;
  const uint32_t words = (cells + 1) / 2;
  uint16_t* s_out = reinterpret_cast<uint16_t*>(s_w + words);
  const bool scatter = g.size <= cap;
  const K mask = (K(1) << rem_bits) - 1;
  // One CTA per SM: the first batch of keys is in flight while the grid is
  // zeroed, later batches keep kB loads per thread outstanding.
  constexpr int kB = sizeof(K) == 4 ? 16 : 8;
  const K* sp = src + g.start;
  const K prefix = sp[0] & ~mask;
  K v[kB];
  auto load = [&](uint32_t i, bool last_use) {
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const uint32_t e = i + u * kLeafGridThreads;
      v[u] = e < g.size ? (last_use ? __ldcs(sp + e) : __ldcg(sp + e)) : K(0);
    }
  };
  uint32_t i = threadIdx.x;
  load(i, !scatter);
  if ((words & 3) == 0) {  // 16-byte stores (words is a power of two here)
    for (uint32_t z = threadIdx.x; z < words / 4; z += blockDim.x) reinterpret_cast<uint4*>(s_w)[z] = make_uint4(0, 0, 0, 0);
  } else {
    for (uint32_t z = threadIdx.x; z < words; z += blockDim.x) s_w[z] = 0;
  }
  __syncthreads();
  for (;;) {
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (i + u * kLeafGridThreads < g.size) {
        const uint32_t cell = static_cast<uint32_t>(v[u] & mask);
        atomicAdd(&s_w[leaf_gw(cell >> 1)], 1u << ((cell & 1) * 16));
      }
    i += kB * kLeafGridThreads;
    if (i >= g.size) break;
    load(i, !scatter);
  }
  if (scatter) load(threadIdx.x, true);  // the rank pass re-reads the segment (L2)
  __syncthreads();
  // exclusive scan over cells: each thread owns a contiguous run of words
  const uint32_t per = (words + kLeafGridThreads - 1) / kLeafGridThreads;
  const uint32_t w0 = threadIdx.x * per;
  // words >= threads: each thread owns whole words w0 .. w0+per-1 (per | 32,
  // w0 a multiple of per), whose swizzle is one XOR with xr; no bounds
  const bool whole = words >= kLeafGridThreads;
  const uint32_t xr = (w0 >> 5) & 31u;
  // 2^16 cells (cfg5's leaves): the thread's 32 words stay in registers
  // between the sum and the offsets pass (one shared read per word, not two)
  const bool fast32 = whole && per == 32;
  uint32_t xs[32];
  uint32_t sum = 0;
  if (fast32) {
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) {
      xs[j] = s_w[(w0 + j) ^ xr];
      sum += (xs[j] & 0xffffu) + (xs[j] >> 16);
    }
  } else if (whole) {
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t x = s_w[(w0 + j) ^ xr];
      sum += (x & 0xffffu) + (x >> 16);
    }
  } else {
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t w = w0 + j;
      if (w < words) {
        const uint32_t x = s_w[leaf_gw(w)];
        sum += (x & 0xffffu) + (x >> 16);
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_scan[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
  {  // exclusive prefix of the 32 warp totals: one load and a warp scan, not a 31-step loop
    const uint32_t t = s_scan[lane];
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    run += __shfl_sync(0xffffffffu, ti - t, warp);
  }
  if (scatter) {
    if (fast32) {
#pragma unroll
      for (uint32_t j = 0; j < 32; ++j) {  // counts -> exclusive offsets (< 65536: no carry between halves)
        const uint32_t c0 = xs[j] & 0xffffu, c1 = xs[j] >> 16;
        s_w[(w0 + j) ^ xr] = run | ((run + c0) << 16);
        run += c0 + c1;
      }
    }
    for (uint32_t j = 0; j < (fast32 ? 0u : per); ++j) {  // counts -> exclusive offsets (< 65536: no carry between halves)
      const uint32_t w = w0 + j;
      if (whole || w < words) {
        const uint32_t pw = whole ? (w ^ xr) : leaf_gw(w);
        const uint32_t x = s_w[pw];
        const uint32_t c0 = x & 0xffffu, c1 = x >> 16;
        s_w[pw] = run | ((run + c0) << 16);
        run += c0 + c1;
      }
    }
    __syncthreads();
    for (i = threadIdx.x;;) {
#pragma unroll
      for (int u = 0; u < kB; ++u)
        if (i + u * kLeafGridThreads < g.size) {
          const uint32_t cell = static_cast<uint32_t>(v[u] & mask);
          const uint32_t sh = (cell & 1) * 16;
          const uint32_t old = atomicAdd(&s_w[leaf_gw(cell >> 1)], 1u << sh);
          s_out[(old >> sh) & 0xffffu] = static_cast<uint16_t>(cell);
        }
      i += kB * kLeafGridThreads;
      if (i >= g.size) break;
      load(i, true);
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < g.size; p += kLeafGridThreads) emit(g.start + p, prefix | K(s_out[p]));
    return;
  }
  // Emit warp-cooperatively: the warp's 32 threads own a contiguous range of
  // cells and hence a contiguous output range starting at lane 0's offset.
  // Lanes take 32 consecutive cells at a time and write consecutive
  // positions (coalesced), instead of each thread streaming its own run.
  uint32_t out = __shfl_sync(0xffffffffu, run, 0);
  const uint32_t w_begin = warp * 32 * per;                 // first counter word of this warp
  const uint32_t w_end = min(words, w_begin + 32 * per);
  for (uint32_t wb = w_begin; wb < w_end; wb += 32) {       // lane: one word = two cells
    const uint32_t w = wb + lane;
    const uint32_t x = w < w_end ? s_w[leaf_gw(w)] : 0u;
    const uint32_t c0 = x & 0xffffu, c1 = x >> 16;
    uint32_t inc2 = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc2, o);
      if (lane >= o) inc2 += y;
    }
    const uint32_t at = out + inc2 - c0 - c1;
    for (uint32_t q = 0; q < c0; ++q) emit(g.start + at + q, prefix | K(2 * w));
    for (uint32_t q = 0; q < c1; ++q) emit(g.start + at + c0 + q, prefix | K(2 * w + 1));
    out += __shfl_sync(0xffffffffu, inc2, 31);
  }
}

// Small sparse leaf: shared bitonic sort of <= 2048 keys (padded with the
// maximum key), then emit.
template <class K, class Emit>
__global__ void __launch_bounds__(kMsdThreads) k_leaf_bitonic(const K* __restrict__ src, const MsdSeg* __restrict__ segs,
                                                              Emit emit) {
  __shared__ K s[kLeafSmall];
  const MsdSeg g = segs[blockIdx.x];
  uint32_t n2 = 1;
  while (n2 < g.size) n2 <<= 1;
  for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) s[i] = i < g.size ? src[g.start + i] : ~K(0);
  __syncthreads();
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const K a = s[i], b = s[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < g.size; i += blockDim.x) emit(g.start + i, s[i]);
}

// Tiny leaves (<= 32 keys): one warp per segment, lane i holds key i, a
// register bitonic network over shuffles; warps stride over the list.
template <class K, class Emit>
__global__ void __launch_bounds__(kMsdThreads) k_leaf_warp(const K* __restrict__ src, const MsdSeg* __restrict__ segs,
                                                           uint32_t nseg, Emit emit) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x / 32);
  for (uint32_t s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); s < nseg; s += nw) {
    const MsdSeg g = segs[s];
    K v = lane < g.size ? src[g.start + lane] : ~K(0);
#pragma unroll
    for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        const K o = __shfl_xor_sync(0xffffffffu, v, j);
        const bool up = (lane & k) == 0;
        const bool lower = (lane & j) == 0;
        v = (lower == up) ? (v < o ? v : o) : (v < o ? o : v);
      }
    }
    if (lane < g.size) emit(g.start + lane, v);
  }
}

// Mid-size leaves (<= kLeafRadixMax keys, <= 24 remaining bits): one CTA
// loads the segment into shared memory and sorts it by the remaining bits
// with stable 8-bit LSD passes, then writes it once.  Ranking: each warp owns
// a contiguous range of the segment; keys are counted per (digit, warp) with
// shared atomics, one exclusive scan over the table in (digit, warp) order
// gives every warp its start per digit, and the warp then walks its range 32
// keys at a time, the lanes sharing a digit found by 8 ballots (measured
// faster than __match_any_sync on B200) — the order inside a digit is (warp,
// group, lane), i.e. the input order, so the passes are stable.
template <class K>
__host__ __device__ constexpr size_t leaf_radix_smem(uint32_t cap) {  // two key buffers + two count tables
  return 2 * (size_t)cap * sizeof(K) + 2 * 256 * (kLeafRadixThreads / 32) * sizeof(uint32_t);
}

template <class K, class Emit>
__global__ void __launch_bounds__(kLeafRadixThreads) k_leaf_radix(const K* __restrict__ src,
                                                                  const MsdSeg* __restrict__ segs, uint32_t rem_bits,
                                                                  uint32_t cap, Emit emit) {
  constexpr int kW = kLeafRadixThreads / 32;
  extern __shared__ __align__(16) unsigned char lr_smem[];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(lr_smem);  // [2][kW warps][256 digits] (digit -> bank)
  K* in = reinterpret_cast<K*>(s_cnt + 2 * 256 * kW);
  K* out = in + cap;
  __shared__ uint32_t s_part[kLeafRadixThreads / 32];
  const MsdSeg g = segs[blockIdx.x];
  const uint32_t n = g.size;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t per = (n + kW * 32 - 1) / (kW * 32) * 32;  // contiguous range per warp, in groups of 32
  const uint32_t w0 = warp * per, w1 = min(n, w0 + per);
  const unsigned lt = (1u << lane) - 1;
  for (uint32_t i = threadIdx.x; i < 2 * 256 * kW; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  // Fast path: split by the top (up to) 11 remaining bits into 2048 buckets
  // (returning atomics — an MSD split needs no stability), then every key
  // finds its final place by counting the smaller keys of its bucket (1-2
  // keys on average) and leaves straight from there.  A bucket above
  // kLeafRankMax keys (skewed data, duplicates) sends the leaf down the LSD
  // passes below.
  constexpr int kFastBits = 11, kFastBins = 1 << kFastBits, kBinsPer = kFastBins / kLeafRadixThreads;
  const uint32_t top = rem_bits > kFastBits ? rem_bits - kFastBits : 0;
  const uint32_t dmask = (rem_bits < kFastBits ? (1u << rem_bits) : kFastBins) - 1u;
  uint32_t* hs = s_cnt;                 // [2048] bucket counts -> scatter cursors
  uint32_t* hstart = s_cnt + kFastBins; // [2048] bucket starts (the tables hold 2 * 256 * 8 words)
  static_assert(2 * 256 * kW >= 2 * kFastBins, "count tables too small for the fast split");
  for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 8 * kLeafRadixThreads) {  // 8 loads in flight per thread
    K k[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t i = i0 + u * kLeafRadixThreads;
      k[u] = i < n ? __ldcs(src + g.start + i) : K(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t i = i0 + u * kLeafRadixThreads;
      if (i < n) {
        in[i] = k[u];
        atomicAdd(&hs[static_cast<uint32_t>(k[u] >> top) & dmask], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t bc[kBinsPer], bsum = 0, bmax = 0;  // this thread's buckets: kBinsPer consecutive ones
#pragma unroll
  for (int q = 0; q < kBinsPer; ++q) {
    bc[q] = hs[threadIdx.x * kBinsPer + q];
    bsum += bc[q];
    bmax = bc[q] > bmax ? bc[q] : bmax;
  }
  if (!__syncthreads_or(bmax > kLeafRankMax)) {
    uint32_t inc = bsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_part[warp] = inc;
    __syncthreads();
    uint32_t run = inc - bsum;
    for (int w = 0; w < warp; ++w) run += s_part[w];
#pragma unroll
    for (int q = 0; q < kBinsPer; ++q) {
      hs[threadIdx.x * kBinsPer + q] = run;
      hstart[threadIdx.x * kBinsPer + q] = run;
      run += bc[q];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const K key = in[i];
      out[atomicAdd(&hs[static_cast<uint32_t>(key >> top) & dmask], 1u)] = key;
    }
    __syncthreads();
    // hs[d] is now the end of bucket d
    for (uint32_t p = threadIdx.x; p < n; p += blockDim.x) {
      const K x = out[p];
      const uint32_t d = static_cast<uint32_t>(x >> top) & dmask;
      const uint32_t s = hstart[d], e = hs[d];
      uint32_t r = s;
      for (uint32_t q = s; q < e; ++q) {
        const K y = out[q];
        r += (y < x || (y == x && q < p)) ? 1u : 0u;
      }
      emit(g.start + r, x);
    }
    return;
  }
  // LSD passes: count the first digit per (warp range, digit)
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kBinsPer; ++q) hs[threadIdx.x * kBinsPer + q] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
    atomicAdd(&s_cnt[(i / per) * 256 + (static_cast<uint32_t>(in[i]) & 255u)], 1u);
  __syncthreads();
  int cur = 0;
  for (uint32_t sh = 0; sh < rem_bits; sh += 8, cur ^= 1) {
    uint32_t* cnt = s_cnt + cur * 256 * kW;
    uint32_t* nxt = s_cnt + (cur ^ 1) * 256 * kW;
    const bool more = sh + 8 < rem_bits;
    {  // exclusive scan in (digit, warp) order: thread t takes entries t*kPer ..
      constexpr int kPer = 256 * kW / kLeafRadixThreads;
      auto at = [&](int j) -> uint32_t& {
        const uint32_t e = threadIdx.x * kPer + j;
        return cnt[(e % kW) * 256 + e / kW];
      };
      uint32_t v[kPer], sum = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        v[j] = at(j);
        sum += v[j];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_part[warp] = inc;
      __syncthreads();
      uint32_t run = inc - sum;
      for (int w = 0; w < warp; ++w) run += s_part[w];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        at(j) = run;
        run += v[j];
      }
    }
    __syncthreads();
    for (uint32_t base = w0; base < w1; base += 32) {  // stable scatter; counts the next digit
      const uint32_t i = base + lane;
      const bool v = i < w1;
      const K key = v ? in[i] : K(0);
      const uint32_t d = static_cast<uint32_t>(key >> sh) & 255u;
      uint32_t pos;
      if (sh == 0) {  // the first LSD pass may order equal digits freely: one returning atomic
        pos = v ? atomicAdd(&cnt[warp * 256 + d], 1u) : 0u;
      } else {        // later passes keep the previous order: same-digit lanes from 8 ballots
        unsigned pm = __ballot_sync(0xffffffffu, v);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const unsigned x = __ballot_sync(0xffffffffu, (d >> b) & 1u);
          pm &= ((d >> b) & 1u) ? x : ~x;
        }
        pos = v ? cnt[warp * 256 + d] + __popc(pm & lt) : 0u;
        __syncwarp();
        if (v && (pm & lt) == 0) cnt[warp * 256 + d] += __popc(pm);
        __syncwarp();
      }
      if (v) {
        out[pos] = key;
        if (more) atomicAdd(&nxt[(pos / per) * 256 + (static_cast<uint32_t>(key >> (sh + 8)) & 255u)], 1u);
      }
    }
    __syncthreads();
    // this table is next written two passes later (behind the next scan's barriers)
    for (uint32_t i = threadIdx.x; i < 256 * kW; i += blockDim.x) cnt[i] = 0;
    K* t = in;
    in = out;
    out = t;
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) emit(g.start + i, in[i]);
}

// ------------------------------------------------------------- report
// Single-grid report read directly off the sorted
// fixed-width records: row = ordinal of the first byte, suffix = base-radix
// value of bytes 1..w-1 (pad = 0).
__device__ __forceinline__ uint32_t rec_ord(const uint8_t* r, uint32_t j, uint32_t width, const uint16_t* ord) {
  for (uint32_t q = 0; q < j; ++q)
    if (r[q] == 0) return 0;
  return j < width && r[j] ? ord[r[j]] : 0;
}

__global__ void k_report_recs(const uint8_t* __restrict__ recs, uint64_t n, uint32_t width, uint32_t w,
                              uint32_t radix, const uint16_t* __restrict__ ord, DevStats* st) {
  // one warp: lane l finds the first record whose first ordinal is >= r
  // (r = base + l); the end of r's run is lane l + 1's answer, so each lane
  // makes one binary search (lane 31 only supplies lane 30's end)
  unsigned long long span = 0;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t base = 0; base < radix; base += 31) {
    const uint32_t r = base + lane;
    uint64_t a = 0, b = n;  // first record with first ordinal >= r
    while (a < b) {
      const uint64_t mid = (a + b) >> 1;
      if (rec_ord(recs + mid * width, 0, width, ord) >= r) b = mid;
      else a = mid + 1;
    }
    const uint64_t c = __shfl_down_sync(0xffffffffu, a, 1);  // first record with first ordinal >= r + 1
    if (lane < 31 && r < radix && a < c) {
      unsigned long long lo = 0, hi = 0;
      for (uint32_t j = 1; j < w; ++j) {
        lo = lo * radix + rec_ord(recs + a * width, j, width, ord);
        hi = hi * radix + rec_ord(recs + (c - 1) * width, j, width, ord);
      }
      span += hi - lo + 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) span += __shfl_xor_sync(0xffffffffu, span, o);
  if (threadIdx.x == 0) {
    st->cells_traversed = span;
    st->report_digits = w;
  }
}

}  // namespace rsb

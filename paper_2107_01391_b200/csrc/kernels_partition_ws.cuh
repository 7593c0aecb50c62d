// kernels_partition_ws.cuh — the counting pass's partition (K1 of
// kernels_two_level.cuh) with warp-specialised roles.
//
// Ranking warps (kWsRankThreads) stream tiles of 4096 keys (4-byte keys:
// 16-byte loads prefetched one tile ahead into registers; 8-byte keys: TMA
// bulk copies two tiles ahead into shared memory, mapped to saturated 32-bit
// cells as they are read out) and rank + stage every key with
// one shared atomic and one uint16 store: each bucket owns a slot range of the
// tile's staging buffer, sized from the bucket's count two tiles earlier
// (c + c/2 + 32 slots, a multiple of 8), and one shared word (range end << 16 |
// next slot) whose atomicAdd returns the key's slot.  A key that finds its
// bucket's range full is counted straight into the grid (global atomic); keys
// outside the grid rank into a dummy bucket whose range is empty.
// Store warps (kWsStoreThreads, one or two buckets per thread) take a ranked
// tile, pad each run to 16 bytes, keep the page bookkeeping in registers,
// copy the runs into the CTA's pages with 16-byte stores and size the slot
// ranges of the tile two ahead.  Two staging buffers alternate; named barriers
// hand a buffer to the store warps (RANKED) and back once it is copied out
// (FREE), so ranking never waits for the page work unless the store warps fall
// a whole tile behind.  When a bucket held more than 1/8 of a tile two tiles
// earlier (skewed keys), that bucket's keys in each warp instruction take one
// atomic (ballot + leader) instead of serialising on one shared word.  The
// pages are the same as k_page_partition_tma's.
#pragma once

#include "kernels_two_level.cuh"

namespace rsb {

constexpr int kWsRankThreads = 256;
constexpr int kWsStoreThreads = 128;
constexpr int kWsThreads = kWsRankThreads + kWsStoreThreads;

// Named barriers with immediate ids (id0 for buffer 0, id0 + 1 for buffer 1),
// so ptxas reserves only the ids used.
template <int kId0, int kCount>
__device__ __forceinline__ void nbar_sync(int buf) {
  if (buf) asm volatile("bar.sync %0, %1;" ::"n"(kId0 + 1), "n"(kCount) : "memory");
  else asm volatile("bar.sync %0, %1;" ::"n"(kId0), "n"(kCount) : "memory");
}
template <int kId0, int kCount>
__device__ __forceinline__ void nbar_arrive(int buf) {
  if (buf) asm volatile("bar.arrive %0, %1;" ::"n"(kId0 + 1), "n"(kCount) : "memory");
  else asm volatile("bar.arrive %0, %1;" ::"n"(kId0), "n"(kCount) : "memory");
}

// staging slots per buffer: the ranges sum to <= tile + tile/2 + B * (32 + 7)
__host__ __device__ constexpr uint32_t ws_stage_slots(uint32_t B) {
  return (uint32_t)kTlTile + (uint32_t)kTlTile / 2 + B * 40u;
}
// staging[2], s_w[2][260] (+ the dummy bucket), s_off[2][256], skew[2];
// 8-byte inputs add two 32 KB key tiles (filled by TMA bulk copies)
__host__ __device__ constexpr size_t page_ws_meta_end(uint32_t B) {
  return 2 * (size_t)ws_stage_slots(B) * 2 + 2 * 260 * 4 + 2 * 256 * 4 + 16;
}
__host__ __device__ constexpr size_t page_ws_smem(uint32_t B, uint32_t in_bytes = 4) {
  return in_bytes == 8 ? ((page_ws_meta_end(B) + 127) & ~(size_t)127) + 2 * (size_t)kTlTile * 8 : page_ws_meta_end(B);
}

template <class Map>
__global__ void __launch_bounds__(kWsThreads, 2)
    k_page_partition_ws(const typename Map::In* __restrict__ in, uint64_t n, Map map, TwoLevel t,
                        uint16_t* __restrict__ pages, uint16_t* __restrict__ page_bucket,
                        uint16_t* __restrict__ page_fill, uint32_t* __restrict__ pc_bm,
                        uint32_t* __restrict__ grid, DevStats* st) {
  using In = typename Map::In;
  constexpr bool k32 = sizeof(In) == 4;
  constexpr int kRanked = 1, kFree = 3, kScanBar = 5;  // named barrier ids (+ buffer for RANKED / FREE)
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t SLOTS = ws_stage_slots(t.B);
  uint16_t* s_stage = reinterpret_cast<uint16_t*>(sm);                      // [2][SLOTS]
  uint32_t* s_w = reinterpret_cast<uint32_t*>(sm + 2 * (size_t)SLOTS * 2);  // [2][260]: end << 16 | next slot
  uint32_t* s_off = s_w + 2 * 260;                                          // [2][256]: range start
  uint32_t* s_skew = s_off + 2 * 256;                                       // [2]
  // 8-byte keys: [2][kTlTile] tiles landing by TMA (4-byte keys are prefetched into registers)
  unsigned long long* s_in = reinterpret_cast<unsigned long long*>(sm + ((page_ws_meta_end(t.B) + 127) & ~(size_t)127));
  __shared__ uint32_t s_scan[kWsStoreThreads / 32];
  __shared__ uint32_t s_next;
  __shared__ __align__(8) unsigned long long s_inbar[2];
  const int lane = threadIdx.x & 31;
  const uint32_t B = t.B;
  const uint32_t ntiles = blockIdx.x < t.T ? (t.T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t page0 = blockIdx.x * t.pages_per_cta;

  // slot ranges of the first two tiles: the even split; the dummy bucket B
  // (keys outside the grid) has an empty range
  if (threadIdx.x < 260) {
    const uint32_t b = threadIdx.x;
    const uint32_t cap = ((kTlTile + kTlTile / 2) / B + 32 + 7) & ~7u;
    const uint32_t off = b < B ? b * cap : 0u;
    const uint32_t c = b < B ? cap : 0u;
    for (int q = 0; q < 2; ++q) {
      if (b < 256) s_off[q * 256 + b] = off;
      s_w[q * 260 + b] = ((off + c) << 16) | off;
    }
  }
  if (threadIdx.x == 0) {
    s_next = 0;
    s_skew[0] = s_skew[1] = 0xffffffffu;
    if constexpr (!k32) {
      mbar_init(&s_inbar[0], 1);
      mbar_init(&s_inbar[1], 1);
      fence_mbar_init();
    }
  }
  __syncthreads();

  if (threadIdx.x < kWsRankThreads) {
    // ------------------------------------------------------------ rankers
    const uint32_t cells32 = static_cast<uint32_t>(t.cells);
    const uint32_t magic32 = static_cast<uint32_t>(t.magic), shift32 = t.shift - 32;
    const uint32_t S = t.S;
    uint32_t mx32 = 0;
    unsigned long long mx64 = 0;
    unsigned flags = 0;
    In cur[4][4], nxt[4][4];
    // 8-byte keys: the tile's cells, mapped as the tile is read out of shared
    // memory (saturated at 0xFFFFFFFF, which no grid reaches: kc < cells is
    // the in-grid test, as for 4-byte keys)
    uint32_t kc[16];
    const uint64_t full_tiles = n / kTlTile;
    // the 16 keys of (tile, this thread): four 16-byte vectors (bounds-checked
    // only in the last, partial tile)
    auto load = [&](uint64_t tile, In (&v)[4][4]) {
      if (tile < full_tiles) {
        if constexpr (k32) {
          const uint4* p = reinterpret_cast<const uint4*>(in) + tile * (kTlTile / 4) + threadIdx.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = __ldcs(p + q * kWsRankThreads);
            v[q][0] = from_bits32(u.x, (In*)nullptr); v[q][1] = from_bits32(u.y, (In*)nullptr);
            v[q][2] = from_bits32(u.z, (In*)nullptr); v[q][3] = from_bits32(u.w, (In*)nullptr);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) Load4<In>::run(in, tile * kTlTile + q * 1024 + threadIdx.x * 4, n, true, v[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) Load4<In>::run(in, tile * kTlTile + q * 1024 + threadIdx.x * 4, n, false, v[q]);
      }
    };
    // rank + stage one tile; kSkew: warp-aggregated atomics; kFull: no bounds checks
    auto rank_tile = [&](auto skew_c, auto full_c, uint64_t tile, uint32_t* w, uint16_t* stage, uint32_t hot) {
      constexpr bool kSkew = decltype(skew_c)::value, kFull = decltype(full_c)::value;
      uint32_t r[16];
      uint32_t hot_mask = 0, hot_seen = 0;  // this thread's keys in the hot bucket; the warp's hot keys so far
      const unsigned lt = (1u << lane) - 1u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bool ok = true;
          if constexpr (!kFull) ok = tile * kTlTile + q * 1024 + threadIdx.x * 4 + e < n;
          uint32_t kk;
          bool ing;
          if constexpr (k32) {
            kk = map.key32(cur[q][e], flags);
            if constexpr (kFull) {
              mx32 = kk > mx32 ? kk : mx32;
              ing = kk < cells32;
            } else {
              mx32 = (ok && kk > mx32) ? kk : mx32;
              ing = ok && kk < cells32;
            }
          } else {
            kk = kc[q * 4 + e];
            ing = kk < cells32;
          }
          uint32_t bk = __umulhi(kk, magic32) >> shift32;
          bk = ing ? bk : B;  // the dummy bucket: an empty range, never staged
          uint32_t rr;
          if constexpr (!kSkew) {
            rr = atomicAdd(&w[bk], 1u);
          } else {
            // hot-bucket keys take a place in the warp's running hot count
            // (one atomic for the whole tile below); the others their own atomic
            const bool ish = bk == hot;
            const unsigned m = __ballot_sync(0xffffffffu, ish);
            rr = ish ? hot_seen + __popc(m & lt) : atomicAdd(&w[bk], 1u);
            hot_mask |= ish ? 1u << (q * 4 + e) : 0u;
            hot_seen += __popc(m);
          }
          r[q * 4 + e] = rr;
        }
      }
      if constexpr (kSkew) {
        uint32_t base = 0;
        if (lane == 0 && hot_seen) base = atomicAdd(&w[hot], hot_seen);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (hot_mask & (1u << j)) r[j] += base;  // (range end << 16 | next slot) + the key's place
      }
      // (the keys are re-read from registers: cheaper than holding them twice)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t rr = r[q * 4 + e], pos = rr & 0xffffu;
          uint32_t kk;
          if constexpr (k32) {
            unsigned f = 0;
            kk = map.key32(cur[q][e], f);
          } else {
            kk = kc[q * 4 + e];
          }
          if (pos < (rr >> 16)) {
            stage[pos] = static_cast<uint16_t>(kk - (__umulhi(kk, magic32) >> shift32) * S);
          } else {
            // the bucket's range is full: count the key directly (a key
            // outside the grid or past the input ranked into the dummy bucket)
            bool ing = kk < cells32;
            if constexpr (k32 && !kFull) ing = ing && tile * kTlTile + q * 1024 + threadIdx.x * 4 + e < n;
            if (ing && (rr >> 16) != 0) atomicAdd(&grid[kk], 1u);
          }
        }
      }
    };
    // 8-byte keys: a full tile lands in s_in[buf] by one TMA bulk copy, two
    // tiles ahead; each ranker maps its 16 keys out of it (conflict-free
    // 16-byte reads), then the rankers sync and the buffer is refilled
    auto issue = [&](uint64_t tl, int b) {  // one thread
      fence_proxy_async_smem();
      mbar_expect_tx(&s_inbar[b], kTlTile * 8);
      bulk_g2s(s_in + (size_t)b * kTlTile, in + tl * kTlTile, kTlTile * 8, &s_inbar[b]);
    };
    auto map_tile = [&](uint64_t tl, int b, unsigned& phase) {
      if constexpr (!k32) {
        if (tl < full_tiles) {
          mbar_wait(&s_inbar[b], (phase >> b) & 1u);
          phase ^= 1u << b;
          const ulonglong2* src = reinterpret_cast<const ulonglong2*>(s_in + (size_t)b * kTlTile);
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const ulonglong2 x = src[h * kWsRankThreads + threadIdx.x];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const unsigned long long k64 = map(from_bits64(e ? x.y : x.x, (In*)nullptr), flags);
              mx64 = k64 > mx64 ? k64 : mx64;
              kc[h * 2 + e] = k64 < 0xFFFFFFFFull ? static_cast<uint32_t>(k64) : 0xFFFFFFFFu;
            }
          }
          asm volatile("bar.sync 6, %0;" ::"n"(kWsRankThreads) : "memory");  // every ranker has read s_in[b]
          const uint64_t ahead = tl + 2ull * gridDim.x;
          if (threadIdx.x == 0 && ahead < full_tiles) issue(ahead, b);
        } else {  // the partial last tile, from global memory with bounds
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            In v[4];
            Load4<In>::run(in, tl * kTlTile + q * 1024 + threadIdx.x * 4, n, false, v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const bool ok = tl * kTlTile + q * 1024 + threadIdx.x * 4 + e < n;
              const unsigned long long k64 = ok ? map(v[e], flags) : 0ull;
              mx64 = k64 > mx64 ? k64 : mx64;
              kc[q * 4 + e] = ok && k64 < 0xFFFFFFFFull ? static_cast<uint32_t>(k64) : 0xFFFFFFFFu;
            }
          }
        }
      }
    };
    unsigned in_phase = 0;
    uint64_t tile = blockIdx.x;
    if constexpr (k32) {
      if (ntiles) load(tile, cur);
    } else if (threadIdx.x == 0) {
      for (uint32_t k = 0; k < 2 && k < ntiles; ++k)
        if (tile + (uint64_t)k * gridDim.x < full_tiles) issue(tile + (uint64_t)k * gridDim.x, k);
    }
    for (uint32_t i = 0; i < ntiles; ++i, tile += gridDim.x) {
      const int buf = i & 1;
      if constexpr (k32) {
        if (i + 1 < ntiles) load(tile + gridDim.x, nxt);
      } else {
        map_tile(tile, buf, in_phase);
      }
      if (i >= 2) nbar_sync<kFree, kWsThreads>(buf);  // the store warps set this buffer's ranges
      uint32_t* w = s_w + buf * 260;
      uint16_t* stage = s_stage + buf * SLOTS;
      const uint32_t hot = s_skew[buf];  // the hot bucket, or 0xffffffff
      if (tile < full_tiles) {
        if (hot == 0xffffffffu) rank_tile(std::false_type{}, std::true_type{}, tile, w, stage, hot);
        else rank_tile(std::true_type{}, std::true_type{}, tile, w, stage, hot);
      } else {
        rank_tile(std::false_type{}, std::false_type{}, tile, w, stage, hot);
      }
      nbar_arrive<kRanked, kWsThreads>(buf);
      if constexpr (k32) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) cur[q][e] = nxt[q][e];
      }
    }
    const unsigned long long mx = k32 ? (unsigned long long)mx32 : mx64;
    warp_max_to(mx, &st->max_key);
    flags = warp_or(flags | (mx >= t.cells ? 0x80000000u : 0u));
    if (lane == 0 && flags) {
      if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
      if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
    }
    return;
  }
  // ------------------------------------------------------------ store warps
  const uint32_t sid = threadIdx.x - kWsRankThreads;
  const int swarp = sid >> 5;
  uint16_t* my_pages = pages + (uint64_t)page0 * kPage;
  uint32_t pg[2] = {0xffffffffu, 0xffffffffu}, fill[2] = {kPage, kPage}, np[2] = {0, 0};
  for (uint32_t i = 0; i < ntiles; ++i) {
    const int buf = i & 1;
    nbar_sync<kRanked, kWsThreads>(buf);
    uint32_t* w = s_w + buf * 260;
    uint16_t* stage = s_stage + buf * SLOTS;
    uint32_t cap[2] = {0, 0};
    // runs longer than kOwn 16-byte pieces: the rest is copied by the whole warp below
    constexpr uint32_t kOwn = 16;
    uint32_t l_off[2] = {0, 0}, l_nch[2] = {0, 0}, l_n1c[2] = {0, 0};
    uint4* l_d1[2] = {nullptr, nullptr};
    uint4* l_d2[2] = {nullptr, nullptr};
    uint32_t hot = 0;  // (count << 16 | bucket) of this thread's hottest bucket above 1/8 of a tile
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint32_t b = sid + k * kWsStoreThreads;
      if (b >= B) continue;
      const uint32_t v = w[b];
      const uint32_t off = s_off[buf * 256 + b];
      const uint32_t nxt_slot = v & 0xffffu, end = v >> 16;
      const uint32_t cnt = nxt_slot - off;  // keys of this bucket in the tile (staged or not)
      const uint32_t staged = (nxt_slot < end ? nxt_slot : end) - off;
      const uint32_t run = (staged + 7) & ~7u;  // <= the range (a multiple of 8)
      cap[k] = (cnt + (cnt >> 1) + 32 + 7) & ~7u;
      if (cnt > kTlTile / 8 && (cnt << 16 | b) > hot) hot = cnt << 16 | b;
      for (uint32_t r = staged; r < run; ++r) stage[off + r] = kPagePad;
      if (run) {
        const uint32_t room = (pg[k] == 0xffffffffu) ? 0u : kPage - fill[k];
        uint32_t pa = pg[k], fa = fill[k], pb = 0;
        if (run > room) {
          const uint32_t extra = (run - room + kPage - 1) / kPage;
          const uint32_t first = atomicAdd(&s_next, extra);
          for (uint32_t j = 0; j < extra; ++j) page_bucket[page0 + first + j] = static_cast<uint16_t>(b);
          for (uint32_t j = 0; j + 1 < extra; ++j) page_fill[page0 + first + j] = static_cast<uint16_t>(kPage);
          if (pg[k] != 0xffffffffu) page_fill[page0 + pg[k]] = static_cast<uint16_t>(kPage);
          np[k] += extra;
          if (room == 0) {
            pa = first;
            fa = 0;
            pb = first + 1;
          } else {
            pb = first;
          }
          pg[k] = first + extra - 1;
          fill[k] = run - room - (extra - 1) * kPage;
        } else {
          fill[k] += run;
        }
        // the run in 16-byte pieces: [0, n1) to the current page at fa, the
        // rest to consecutive fresh pages from pb
        const uint32_t n1 = run < kPage - fa ? run : kPage - fa;
        const uint4* src = reinterpret_cast<const uint4*>(stage + off);
        uint4* d1 = reinterpret_cast<uint4*>(my_pages + (uint64_t)pa * kPage + fa);
        uint4* d2 = reinterpret_cast<uint4*>(my_pages + (uint64_t)pb * kPage) - n1 / 8;
        const uint32_t nch = run / 8, own = nch < kOwn ? nch : kOwn;
        for (uint32_t c = 0; c < own; ++c) {
          const uint4 x = src[c];
          if (c < n1 / 8) d1[c] = x;
          else d2[c] = x;
        }
        l_off[k] = off;
        l_nch[k] = nch;
        l_n1c[k] = n1 / 8;
        l_d1[k] = d1;
        l_d2[k] = d2;
      }
    }
    // long runs (a hot bucket): the warp copies the pieces past kOwn together
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      unsigned m = __ballot_sync(0xffffffffu, l_nch[k] > kOwn);
      while (m) {
        const int src_lane = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t so = __shfl_sync(0xffffffffu, l_off[k], src_lane);
        const uint32_t nc = __shfl_sync(0xffffffffu, l_nch[k], src_lane);
        const uint32_t n1c = __shfl_sync(0xffffffffu, l_n1c[k], src_lane);
        uint4* d1 = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(l_d1[k]), src_lane));
        uint4* d2 = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(l_d2[k]), src_lane));
        const uint4* src = reinterpret_cast<const uint4*>(stage + so);
        for (uint32_t c = kOwn + lane; c < nc; c += 32) {
          const uint4 x = src[c];
          if (c < n1c) d1[c] = x;
          else d2[c] = x;
        }
      }
    }
    // slot ranges of tile i+2 (this buffer) from this tile's counts: thread
    // sid's buckets sid and sid + 128 take consecutive ranges at its
    // exclusive prefix over the store threads
    const uint32_t v = cap[0] + cap[1];
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_scan[swarp] = inc;
    const uint32_t whot = __reduce_max_sync(0xffffffffu, hot);
    nbar_sync<kScanBar, kWsStoreThreads>(0);
    uint32_t before = 0;
#pragma unroll
    for (int q = 0; q < kWsStoreThreads / 32; ++q) before += q < swarp ? s_scan[q] : 0u;
    const uint32_t start = before + inc - v;
    if (lane == 0 && swarp == 0) s_skew[buf] = 0;
    nbar_sync<kScanBar, kWsStoreThreads>(0);  // s_scan read and s_skew cleared before the writes below
    if (lane == 0 && whot) atomicMax(&s_skew[buf], whot);
    nbar_sync<kScanBar, kWsStoreThreads>(0);
    if (sid == 0) s_skew[buf] = s_skew[buf] ? (s_skew[buf] & 0xffffu) : 0xffffffffu;
    if (sid < B) {
      s_off[buf * 256 + sid] = start;
      s_w[buf * 260 + sid] = ((start + cap[0]) << 16) | start;
    }
    if (sid + kWsStoreThreads < B) {
      const uint32_t o2 = start + cap[0];
      s_off[buf * 256 + sid + kWsStoreThreads] = o2;
      s_w[buf * 260 + sid + kWsStoreThreads] = ((o2 + cap[1]) << 16) | o2;
    }
    if (sid == 0) s_w[buf * 260 + B] = 0;  // the dummy bucket: empty range again
    if (i + 2 < ntiles) nbar_arrive<kFree, kWsThreads>(buf);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t b = sid + k * kWsStoreThreads;
    if (b >= B) continue;
    if (pg[k] != 0xffffffffu) page_fill[page0 + pg[k]] = static_cast<uint16_t>(fill[k]);
    pc_bm[(uint64_t)b * t.G + blockIdx.x] = np[k];
  }
}

}  // namespace rsb

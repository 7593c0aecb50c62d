// kernels_partition_direct.cuh — the counting pass's partition (K1 of
// kernels_two_level.cuh) for 4-byte keys, written straight into per-bucket
// page chunks in shared memory and flushed by TMA bulk stores.
//
// The page-count kernel only needs, per outer bucket, every inner digit of the
// bucket's keys in some 2 KB page; order is free.  So each bucket owns a ring
// of two 256-entry chunks (512 B each) in shared memory, and one shared word
// (limit << 16 | next slot).  A key's atomicAdd on that word returns its ring
// slot: one shared atomic and one uint16 store per key, no staging buffer, no
// run copies through registers.  After every 4096-key tile (one barrier) the
// thread owning a bucket bulk-stores each chunk that filled up into the
// bucket's current page (four chunks per 1024-entry page) with
// cp.async.bulk (UBLKCP: no LSU wavefronts for the page stores), and moves
// the bucket's limit: a chunk's buffer is handed back once the bulk store
// that reads it has been waited for, one tile later.  A bucket that takes more
// keys in one tile than its writable chunks hold (more than 256-511 keys of a
// 4096-key tile: skewed input) counts the rest straight into the grid with
// warp-aggregated global atomics — correct, slower; cfg3's Zipf-skewed mapped
// cells keep the TMA-fed partition.
//
// Replaces the loop of hashing.cpp:40-52 (hash_insert of every key) with the
// two-level grid of kernels_two_level.cuh; the pages are the same as
// k_page_partition_ws's, so k_page_list / k_page_count consume them unchanged.
#pragma once

#include "bulk_copy.cuh"
#include "kernels_two_level.cuh"

namespace rsb {

constexpr int kDirThreads = 512;
constexpr int kDirPer = kTlTile / kDirThreads;  // 8 keys per thread per tile
constexpr uint32_t kDirChunk = 256;             // entries per ring chunk (512 B)
constexpr uint32_t kDirRing = 2 * kDirChunk;    // entries per bucket ring (1 KB)
constexpr uint32_t kDirChunksPerPage = kPage / kDirChunk;
constexpr uint32_t kDirMaxBuckets = 104;        // rings <= 104 KB: two CTAs per SM

__host__ __device__ constexpr size_t page_dir_smem(uint32_t B) {
  return (size_t)B * kDirRing * sizeof(uint16_t) + 128 * sizeof(uint32_t);  // rings [B], words [B + 1]
}

template <class Map>
__global__ void __launch_bounds__(kDirThreads, 2)
    k_page_partition_direct(const typename Map::In* __restrict__ in, uint64_t n, Map map, TwoLevel t,
                            uint16_t* __restrict__ pages, uint16_t* __restrict__ page_bucket,
                            uint16_t* __restrict__ page_fill, uint32_t* __restrict__ pc_bm,
                            uint32_t* __restrict__ grid, DevStats* st) {
  using In = typename Map::In;
  static_assert(sizeof(In) == 4, "4-byte keys");
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t B = t.B;
  uint16_t* ring = reinterpret_cast<uint16_t*>(sm);                                           // [B][kDirRing]
  uint32_t* w = reinterpret_cast<uint32_t*>(sm + (size_t)B * kDirRing * sizeof(uint16_t));  // [B + 1]
  __shared__ uint32_t s_next;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t ntiles = blockIdx.x < t.T ? (t.T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t page0 = blockIdx.x * t.pages_per_cta;
  const uint32_t cells32 = static_cast<uint32_t>(t.cells);
  const uint32_t magic32 = static_cast<uint32_t>(t.magic), shift32 = t.shift - 32;
  const uint32_t S = t.S;
  const uint64_t full_tiles = n / kTlTile;

  // state of bucket tid (tid < B), in registers: chunks whose bulk store was
  // issued (ring-relative), the open page, its chunks, the pages taken
  uint32_t issued = 0, pg = 0, q = kDirChunksPerPage, np = 0;
  if (tid < B) w[tid] = kDirRing << 16;  // both chunks writable, next slot 0
  if (tid == B) w[B] = 0;                // the dummy word of keys outside the grid
  if (tid == 0) s_next = 0;
  __syncthreads();

  uint32_t mx = 0;
  unsigned flags = 0;
  In cur[kDirPer], nxt[kDirPer];
  auto load = [&](uint64_t tile, In (&v)[kDirPer]) {
#pragma unroll
    for (int h = 0; h < kDirPer / 4; ++h) {
      In x[4];
      Load4<In>::run(in, tile * kTlTile + (uint64_t)h * (kTlTile / 2) + tid * 4, n, tile < full_tiles, x);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[h * 4 + e] = x[e];
    }
  };
  // element index of key j of this thread in tile `tile`
  auto index_of = [&](uint64_t tile, int j) {
    return tile * kTlTile + (uint64_t)(j / 4) * (kTlTile / 2) + tid * 4 + (j & 3);
  };
  auto open_page = [&]() {
    if (q == kDirChunksPerPage) {
      pg = atomicAdd(&s_next, 1u);
      page_bucket[page0 + pg] = static_cast<uint16_t>(tid);
      page_fill[page0 + pg] = static_cast<uint16_t>(kPage);
      ++np;
      q = 0;
    }
  };

  // bucket tid's work after a tile: hand back the chunks whose bulk stores
  // have read them, bulk-store the chunks that filled up, move the limit
  auto flush = [&]() {
    const uint32_t v = w[tid];
    uint32_t next = v & 0xffffu;
    const uint32_t lim = v >> 16;
    if (next > lim) next = lim;  // the keys past the limit were counted in the grid
    bulk_wait_read();            // this thread's bulk stores of earlier tiles have read their chunks
    const uint32_t free_upto = issued;
    const uint32_t full = next / kDirChunk;
    if (full > issued) {
      fence_proxy_async_smem();  // the rankers' stores (ordered by the barrier) before the async-proxy reads
      for (uint32_t c = issued; c < full; ++c) {
        open_page();
        bulk_s2g(pages + (uint64_t)(page0 + pg) * kPage + q * kDirChunk, ring + tid * kDirRing + (c & 1) * kDirChunk,
                 kDirChunk * sizeof(uint16_t));
        ++q;
      }
      bulk_commit();
      issued = full;
    }
    uint32_t nlim = (free_upto + 2) * kDirChunk;
    if (free_upto >= 2) {  // keep the positions small; whole rings keep the chunk parity
      const uint32_t m = free_upto / 2;
      next -= m * kDirRing;
      nlim -= m * kDirRing;
      issued -= m * 2;
    }
    w[tid] = (nlim << 16) | next;
  };

  // rank + store one tile; kFull: no bounds checks.  Keys outside the grid
  // (or past n) take the dummy word B, whose limit is 0: never stored
  auto rank_tile = [&](auto full_c, uint64_t tile) {
    constexpr bool kFull = decltype(full_c)::value;
    uint32_t r[kDirPer];
#pragma unroll
    for (int j = 0; j < kDirPer; ++j) {
      const uint32_t kk = map.key32(cur[j], flags);
      bool ing;
      if constexpr (kFull) {
        mx = kk > mx ? kk : mx;
        ing = kk < cells32;
      } else {
        const bool ok = index_of(tile, j) < n;
        mx = (ok && kk > mx) ? kk : mx;
        ing = ok && kk < cells32;
      }
      const uint32_t bk = ing ? __umulhi(kk, magic32) >> shift32 : B;
      r[j] = atomicAdd(&w[bk], 1u);
    }
    unsigned fb = 0;  // keys whose bucket's writable chunks are full
#pragma unroll
    for (int j = 0; j < kDirPer; ++j) {
      unsigned f = 0;
      const uint32_t kk = map.key32(cur[j], f);
      const uint32_t pos = r[j] & 0xffffu, lim = r[j] >> 16;
      const uint32_t bk = __umulhi(kk, magic32) >> shift32;
      if (pos < lim) ring[bk * kDirRing + (pos & (kDirRing - 1))] = static_cast<uint16_t>(kk - bk * S);
      fb |= (pos >= lim && lim != 0) ? 1u << j : 0u;
    }
    if (__any_sync(0xffffffffu, fb)) {  // skewed tile: count those keys straight into the grid
#pragma unroll
      for (int j = 0; j < kDirPer; ++j) {
        const bool mine = (fb >> j) & 1u;
        unsigned f = 0;
        const uint32_t kk = map.key32(cur[j], f);
        const unsigned peers = __match_any_sync(0xffffffffu, mine ? kk : 0xffffffffu);
        if (mine && lane == static_cast<uint32_t>(__ffs(peers) - 1))
          atomicAdd(&grid[kk], static_cast<uint32_t>(__popc(peers)));
      }
    }
  };

  // keys stream two tiles ahead in registers (32 KB per CTA in flight)
  uint64_t tile = blockIdx.x;
  if (ntiles) load(tile, cur);
  if (ntiles > 1) load(tile + gridDim.x, nxt);
  for (uint32_t i = 0; i < ntiles; ++i, tile += gridDim.x) {
    In nx2[kDirPer];
    if (i + 2 < ntiles) load(tile + 2ull * gridDim.x, nx2);
    if (tile < full_tiles) rank_tile(std::true_type{}, tile);
    else rank_tile(std::false_type{}, tile);
    __syncthreads();
    if (tid < B) flush();
    if (tid == B) w[B] = 0;  // the dummy word: limit 0, slot counter reset
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kDirPer; ++j) {
      cur[j] = nxt[j];
      nxt[j] = nx2[j];
    }
  }

  // the last, partly filled chunk of every bucket (its tail padded with pad
  // entries, which k_page_count drops), then this CTA's page counts
  if (tid < B) {
    const uint32_t next = w[tid] & 0xffffu;  // <= the limit after the last flush
    const uint32_t rem = next - issued * kDirChunk;
    if (rem) {
      uint16_t* rc = ring + tid * kDirRing + (issued & 1) * kDirChunk;
      const uint32_t len = (rem + 7) & ~7u;
      for (uint32_t e = rem; e < len; ++e) rc[e] = kPagePad;
      open_page();
      fence_proxy_async_smem();
      bulk_s2g(pages + (uint64_t)(page0 + pg) * kPage + q * kDirChunk, rc, len * sizeof(uint16_t));
      bulk_commit();
      page_fill[page0 + pg] = static_cast<uint16_t>(q * kDirChunk + len);
    } else if (q < kDirChunksPerPage) {
      page_fill[page0 + pg] = static_cast<uint16_t>(q * kDirChunk);
    }
    pc_bm[(uint64_t)tid * t.G + blockIdx.x] = np;
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (mx >= t.cells ? 0x80000000u : 0u));
  if (lane == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

}  // namespace rsb

// kernels_partition_direct.cuh — the counting pass's partition (K1 of
// kernels_two_level.cuh) for 4-byte keys, written straight into per-bucket
// page chunks in shared memory and flushed by TMA bulk stores.
//
// The page-count kernel only needs, per outer bucket, every inner digit of the
// bucket's keys in some 2 KB page; order is free.  So each bucket owns a ring
// of two 128-entry chunks (256 B each) in shared memory and one shared word
// (limit and next slot, in ring bytes: dir_word below); a key's atomicAdd on
// that word returns its ring slot: one shared atomic and one uint16 store per
// key, no staging buffer and no run copies through registers.  The word's
// encoding keeps the ranker at ~15 instructions per key (was 23): the
// writable test is a shift and a compare, the slot address one LOP3 over a
// ring-size-aligned base, the inner digit one multiply-add by -S.
//
// Two warp roles.  Twelve ranking warps stream 3072-key tiles (8 keys per
// thread, 16-byte loads two tiles ahead in registers) and rank them into two
// alternating sets of rings and words (even / odd tiles); they never wait for
// each other.  Four owner warps (thread b owns bucket b) take a set once its
// tile is ranked (named barrier RANKED[s]: rankers arrive, owners sync),
// bulk-store every chunk that filled up into the bucket's current page (eight
// chunks per 1024-entry page) with cp.async.bulk (UBLKCP: no LSU wavefronts
// for the page stores), hand back the chunks whose earlier bulk stores have
// read them, move the bucket's limit, and release the set (FLUSHED[s]: owners
// arrive, rankers sync before ranking into it again two tiles later).
//
// A bucket that takes more keys in one tile than its writable chunks hold
// (more than 128-255 keys of a 3072-key tile: skewed input) counts the rest
// straight into the grid with warp-aggregated global atomics — correct,
// slower; cfg3's Zipf-skewed mapped cells run the hot variant below.  Keys
// outside the grid rank into the word of a spare ring (index B) whose limit
// never binds and whose contents nobody reads, so a ranker's only unwritable
// case is a full ring (the hot variant keeps limit 0 there: its in-place
// counted keys carry word 0).
//
// Replaces the loop of hashing.cpp:40-52 (hash_insert of every key) with the
// two-level grid of kernels_two_level.cuh; the pages are the same as
// k_page_partition_ws's, so k_page_list / k_page_count consume them unchanged.
#pragma once

#include "bulk_copy.cuh"
#include "kernels_partition_ws.cuh"  // nbar_sync / nbar_arrive
#include "kernels_two_level.cuh"

namespace rsb {

constexpr uint32_t kDirMaxBuckets = 104;  // owner threads 0..B-1 of 128; B + 1 words per set
constexpr int kDirRankers = 384;
constexpr int kDirOwners = 128;
constexpr int kDirThreads = kDirRankers + kDirOwners;
constexpr uint32_t kDirChunk = 128;
template <class In>
constexpr int kDirPerT = 32 / sizeof(In);  // 32 bytes of keys per ranker thread per tile
constexpr uint32_t kDirRing = 2 * kDirChunk;

// + one ring of slack: the kernel starts its rings on a ring-size boundary of
// the shared window, so a ring slot's address is (word & mask) | ring base
// B + 1 rings per set: ring B takes the keys outside the grid (never flushed)
__host__ __device__ constexpr size_t page_dir_smem(uint32_t B) {
  return 2 * (size_t)(B + 1) * kDirRing * sizeof(uint16_t) + 2 * 128 * sizeof(uint32_t) + kDirRing * sizeof(uint16_t);
}

// kHot (skewed inputs, e.g. cfg3's Zipf-hot mapped cells): a shared uint32
// histogram of one bucket's S inner cells: the first bucket whose ring
// overflows becomes the CTA's hot bucket and its keys are counted there
// directly (one shared atomic each, no ring, no page), the histogram flushed
// into the grid at the end.
// The hot variant's ring chunks are 64 entries, which leaves room for the
// histogram while two CTAs still share an SM.
template <bool kHot>
__host__ __device__ constexpr uint32_t dir_chunk() { return kHot ? 64u : kDirChunk; }
__host__ __device__ constexpr size_t page_dir_hot_smem(uint32_t B, uint32_t S) {
  return 2 * (size_t)(B + 1) * 2 * dir_chunk<true>() * sizeof(uint16_t) + 2 * 128 * sizeof(uint32_t) +
         (size_t)S * sizeof(uint32_t) + 2 * dir_chunk<true>() * sizeof(uint16_t);
}
constexpr uint32_t kDirNoHot = 0xffffffffu;

// A bucket's shared word counts ring BYTES: (2 * limit - 1) << 16 | 2 * next
// (0 for limit 0).  With r the value an atomicAdd of 2 returns, the slot is
// writable iff (r << 16) < r (next < limit, two instructions), its byte offset
// in the ring is r & (ring bytes - 1), and "limit != 0" is r > 0xffff.
__host__ __device__ constexpr uint32_t dir_word(uint32_t limit, uint32_t next) {
  return limit ? ((2u * limit - 1u) << 16) | (2u * next) : 0u;
}
__device__ __forceinline__ uint32_t dir_word_next(uint32_t v) { return (v & 0xffffu) >> 1; }
__device__ __forceinline__ uint32_t dir_word_limit(uint32_t v) { return ((v >> 16) + 1u) >> 1; }
__device__ __forceinline__ uint32_t atoms_add(uint32_t saddr, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(saddr), "r"(v));
  return r;
}
__device__ __forceinline__ void sts_u16(uint32_t saddr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(saddr), "h"(static_cast<uint16_t>(v)));
}

template <class Map, bool kHot = false>
__global__ void __launch_bounds__(kDirThreads, 2)
    k_page_partition_direct(const typename Map::In* __restrict__ in, uint64_t n, Map map, TwoLevel t,
                             uint16_t* __restrict__ pages, uint16_t* __restrict__ page_bucket,
                             uint16_t* __restrict__ page_fill, uint32_t* __restrict__ pc_bm,
                             uint32_t* __restrict__ grid, DevStats* st) {
  using In = typename Map::In;
  constexpr bool k32 = sizeof(In) == 4;
  constexpr int kRk = kDirRankers, kThr = kDirThreads;
  constexpr uint32_t kDirTile = kRk * kDirPerT<In>;    // 3072 4-byte or 1536 8-byte keys
  constexpr uint32_t kDirChunk = dir_chunk<kHot>();
  constexpr uint32_t kDirRing = 2 * kDirChunk;
  constexpr bool kInt64 = std::is_same_v<Map, MapI64> || std::is_same_v<Map, MapU64>;
  using Mx = std::conditional_t<k32 || kInt64, uint32_t, unsigned long long>;
  constexpr uint32_t kCPP = kPage / kDirChunk;
  constexpr int kRanked = 1, kFlushed = 3;  // named barrier ids (+ set)
  extern __shared__ __align__(128) unsigned char sm[];
  const uint32_t B = t.B;
  constexpr uint32_t kRingBytes = kDirRing * sizeof(uint16_t);
  const uint32_t sm_sa = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t pad = (0u - sm_sa) & (kRingBytes - 1);  // rings start on a ring-size boundary
  uint16_t* ring = reinterpret_cast<uint16_t*>(sm + pad);                                  // [2][B + 1][kDirRing]
  uint32_t* w = reinterpret_cast<uint32_t*>(sm + pad + 2 * (size_t)(B + 1) * kRingBytes);  // [2][128]
  const uint32_t ring_sa = sm_sa + pad, w_sa = ring_sa + 2 * (B + 1) * kRingBytes;
  // The word of "bucket" B takes the keys outside the grid.  Its limit never
  // binds (their digits go to ring B, which nobody reads), so "not writable"
  // alone means a full ring; the hot variant keeps limit 0 there instead (its
  // hot keys carry word 0: no store, no fallback).
  constexpr uint32_t kDummyWord = kHot ? 0u : dir_word(0x8000u, 0);
  uint32_t* s_hh = w + 2 * 128;  // kHot: [S] counts of the hot bucket's inner cells
  __shared__ uint32_t s_next, s_hot;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t T = static_cast<uint32_t>((n + kDirTile - 1) / kDirTile);
  const uint32_t ntiles = blockIdx.x < T ? (T - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t page0 = blockIdx.x * t.pages_per_cta;
  const uint32_t cells32 = static_cast<uint32_t>(t.cells);
  const uint32_t magic32 = static_cast<uint32_t>(t.magic), shift32 = t.shift - 32;
  const uint32_t S = t.S;
  const uint32_t full_tiles = static_cast<uint32_t>(n / kDirTile);
  if (tid < 2 * 128) {
    const uint32_t b = tid & 127;
    w[tid] = b < B ? dir_word(kDirRing, 0) : kDummyWord;  // both chunks writable
  }
  if (tid == 0) {
    s_next = 0;
    s_hot = kDirNoHot;
  }
  if constexpr (kHot)
    for (uint32_t c = tid; c < t.S; c += kThr) s_hh[c] = 0;
  __syncthreads();

  if (tid < kRk) {
    // ------------------------------------------------------------ rankers
    Mx mx = 0;
    unsigned flags = 0;
    uint32_t neg = 0;  // int64 keys: OR of the high halves (sign bit: a negative value)
    In cur[kDirPerT<In>], nxt[kDirPerT<In>];
    auto load = [&](uint32_t tile, In (&v)[kDirPerT<In>]) {
#pragma unroll
      for (int h = 0; h < kDirPerT<In> / 4; ++h) {
        In x[4];
        Load4<In>::run(in, (uint64_t)tile * kDirTile + h * (kDirTile / 2) + tid * 4, n, tile < full_tiles, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) v[h * 4 + e] = x[e];
      }
    };
    auto index_of = [&](uint32_t tile, int j) {
      return (uint64_t)tile * kDirTile + (j / 4) * (kDirTile / 2) + tid * 4 + (j & 3);
    };
    auto rank_tile = [&](auto full_c, uint32_t tile, int s, In (&cur)[kDirPerT<In>]) {
      constexpr bool kFull = decltype(full_c)::value;
      uint32_t ws_sa = w_sa + s * 512, rs_sa = ring_sa + s * (B + 1) * kRingBytes;
      asm volatile("" : "+r"(ws_sa), "+r"(rs_sa));  // once per tile, not per key
      // inner digit = cell + bucket * (-S): one multiply-add; the shuffle keeps
      // -S in a register (ptxas reloads a plain parameter for every key)
      const uint32_t negS = __shfl_sync(0xffffffffu, t.negS, 0);
      // each key's 32-bit cell (8-byte keys saturate at 0xFFFFFFFF, which no
      // grid reaches, so kc < cells is the in-grid test for both widths)
      uint32_t kc[kDirPerT<In>], r[kDirPerT<In>], bkv[kDirPerT<In>];
      const uint32_t hot = kHot ? *reinterpret_cast<volatile uint32_t*>(&s_hot) : kDirNoHot;
#pragma unroll
      for (int j = 0; j < kDirPerT<In>; ++j) {
        Mx k;
        if constexpr (k32) {
          k = map.key32(cur[j], flags);
          kc[j] = k;
        } else if constexpr (kInt64) {
          // from the two 32-bit halves: a nonzero high half saturates the
          // cell (and, signed, flags a negative value); the max is taken
          // over the saturated cells (the host asks for the exact max if
          // a redo needs it)
          const unsigned long long u = static_cast<unsigned long long>(cur[j]);
          const uint32_t hi = static_cast<uint32_t>(u >> 32), lo = static_cast<uint32_t>(u);
          if constexpr (std::is_same_v<Map, MapI64>) neg |= hi;
          kc[j] = hi ? 0xFFFFFFFFu : lo;
          k = kc[j];
        } else {
          k = map(cur[j], flags);
          kc[j] = k < 0xFFFFFFFFull ? static_cast<uint32_t>(k) : 0xFFFFFFFFu;
        }
        // a cell past the last bucket clamps to B; the few cells between the
        // grid's end and the last bucket's end stay in that bucket (the page
        // count drops them; the max flags the pass anyway)
        uint32_t bk = min(__umulhi(kc[j], magic32) >> shift32, B);
        if constexpr (kFull) {
          mx = k > mx ? k : mx;
        } else {
          const bool ok = index_of(tile, j) < n;
          mx = (ok && k > mx) ? k : mx;
          bk = ok ? bk : B;
        }
        bkv[j] = bk;
        if (kHot && bk == hot) {  // counted in place; r = 0 (limit 0): no ring store, no fallback
          atomicAdd(&s_hh[kc[j] - bk * S], 1u);
          r[j] = 0;
        } else {
          r[j] = atoms_add(ws_sa + bk * 4, 2u);
        }
      }
      bool nw[kDirPerT<In>];  // key j found its ring full
#pragma unroll
      for (int j = 0; j < kDirPerT<In>; ++j) {
        const uint32_t kk = kc[j], rr = r[j];
        const uint32_t bk = bkv[j];
        const bool writable = (rr << 16) < rr;
        if (writable) sts_u16((rr & (kRingBytes - 1)) | (rs_sa + bk * kRingBytes), kk + bk * negS);
        nw[j] = kHot ? !writable && rr > 0xffffu : !writable;
      }
      bool fb = false;
#pragma unroll
      for (int j = 0; j < kDirPerT<In>; ++j) fb = fb || nw[j];
      if (__any_sync(0xffffffffu, fb)) {
#pragma unroll
        for (int j = 0; j < kDirPerT<In>; ++j) {
          // past a (nonzero) limit; a cell beyond the grid in the last bucket is dropped
          const bool mine = !((r[j] << 16) < r[j]) && (!kHot || r[j] > 0xffffu) && kc[j] < cells32;
          if (!__any_sync(0xffffffffu, mine)) continue;  // a match only for the key slots that need one
          const uint32_t kk = kc[j];
          const unsigned peers = __match_any_sync(0xffffffffu, mine ? kk : 0xffffffffu);
          if (mine && lane == static_cast<uint32_t>(__ffs(peers) - 1))
            atomicAdd(&grid[kk], static_cast<uint32_t>(__popc(peers)));
        }
      }
    };
    uint32_t tile = blockIdx.x;
    if (ntiles) load(tile, cur);
    if (ntiles > 1) load(tile + gridDim.x, nxt);
    for (uint32_t i = 0; i < ntiles; ++i, tile += gridDim.x) {
      const int s = i & 1;
      In nx2[kDirPerT<In>];
      if (i + 2 < ntiles) load(tile + 2 * gridDim.x, nx2);
      if (i >= 2) nbar_sync<kFlushed, kThr>(s);  // set s flushed after tile i-2
      if (tile < full_tiles) rank_tile(std::true_type{}, tile, s, cur);
      else rank_tile(std::false_type{}, tile, s, cur);
      nbar_arrive<kRanked, kThr>(s);
#pragma unroll
      for (int j = 0; j < kDirPerT<In>; ++j) {
        cur[j] = nxt[j];
        nxt[j] = nx2[j];
      }
    }
    if (static_cast<int32_t>(neg) < 0) flags |= kFlagNegative;
    warp_max_to(static_cast<unsigned long long>(mx), &st->max_key);
    flags = warp_or(flags | (mx >= t.cells ? 0x80000000u : 0u));
    if (lane == 0 && flags) {
      if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
      if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
    }
    if constexpr (!kHot) return;
  } else {
  // -------------------------------------------------------------- owners
  const uint32_t b = tid - kRk;
  uint32_t issued0 = 0, issued1 = 0, pg = 0, q = kCPP, np = 0;
  auto open_page = [&]() {
    if (q == kCPP) {
      pg = atomicAdd(&s_next, 1u);
      page_bucket[page0 + pg] = static_cast<uint16_t>(b);
      page_fill[page0 + pg] = static_cast<uint16_t>(kPage);
      ++np;
      q = 0;
    }
  };
  auto flush = [&](auto s_c) {
    constexpr int s = decltype(s_c)::value;
    uint32_t& issued = s ? issued1 : issued0;
    uint32_t* ws = w + s * 128;
    const uint16_t* rs = ring + ((size_t)s * (B + 1) + b) * kDirRing;
    const uint32_t v = ws[b];
    uint32_t next = dir_word_next(v);
    const uint32_t lim = dir_word_limit(v);
    if (next > lim) {  // the keys past the limit were counted in the grid
      next = lim;
      if (kHot && s_hot == kDirNoHot) atomicCAS(&s_hot, kDirNoHot, b);  // skew: b's keys count in place from now on
    }
    bulk_wait_read1();  // set s's bulk stores of two tiles ago have read their chunks
    const uint32_t free_upto = issued;
    const uint32_t full = next / kDirChunk;
    if (full > issued) {
      fence_proxy_async_smem();
      for (uint32_t c = issued; c < full; ++c) {
        open_page();
        bulk_s2g(pages + (uint64_t)(page0 + pg) * kPage + q * kDirChunk, rs + (c & 1) * kDirChunk,
                 kDirChunk * sizeof(uint16_t));
        ++q;
      }
      issued = full;
    }
    bulk_commit();
    uint32_t nlim = (free_upto + 2) * kDirChunk;
    if (free_upto >= 2) {
      const uint32_t m = free_upto / 2;
      next -= m * kDirRing;
      nlim -= m * kDirRing;
      issued -= m * 2;
    }
    ws[b] = dir_word(nlim, next);
  };
  auto step = [&](auto s_c, uint32_t i) {
    constexpr int s = decltype(s_c)::value;
    nbar_sync<kRanked, kThr>(s);  // tile i ranked into set s
    if (b < B) flush(s_c);
    if (b == B) w[s * 128 + B] = kDummyWord;
    if (i + 2 < ntiles) nbar_arrive<kFlushed, kThr>(s);
  };
  for (uint32_t i = 0; i < ntiles; i += 2) {
    step(std::integral_constant<int, 0>{}, i);
    if (i + 1 < ntiles) step(std::integral_constant<int, 1>{}, i + 1);
  }
  if (b < B) {
    auto tail = [&](auto s_c) {
      constexpr int s = decltype(s_c)::value;
      const uint32_t is = s ? issued1 : issued0;
      const uint32_t next = dir_word_next(w[s * 128 + b]);
      const uint32_t rem = next - is * kDirChunk;
      if (rem) {
        uint16_t* rc = ring + ((size_t)s * (B + 1) + b) * kDirRing + (is & 1) * kDirChunk;
        for (uint32_t e = rem; e < kDirChunk; ++e) rc[e] = kPagePad;
        open_page();
        fence_proxy_async_smem();
        bulk_s2g(pages + (uint64_t)(page0 + pg) * kPage + q * kDirChunk, rc, kDirChunk * sizeof(uint16_t));
        ++q;
      }
    };
    tail(std::integral_constant<int, 0>{});
    tail(std::integral_constant<int, 1>{});
    bulk_commit();
    if (q < kCPP) page_fill[page0 + pg] = static_cast<uint16_t>(q * kDirChunk);
    pc_bm[(uint64_t)b * t.G + blockIdx.x] = np;
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  }  // owners
  if constexpr (kHot) {  // the hot bucket's counts into the grid
    __syncthreads();
    const uint32_t hot = s_hot;
    if (hot != kDirNoHot)
      for (uint32_t c = tid; c < S; c += kThr) {
        const uint32_t v = s_hh[c];
        if (v && (uint64_t)hot * S + c < t.cells) atomicAdd(&grid[hot * S + c], v);
      }
  }
}

}  // namespace rsb

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
//   k_kv_chunk_scatter  the CTA walks its chunk tile by tile in order (tiles
//                       double-buffered in shared memory by 1D TMA bulk
//                       copies, cp.async.bulk + mbarrier); each
//                       warp ranks its records stably: the lanes sharing a
//                       digit OR their bits into a per-warp shared bitmap
//                       word of that digit and read it back (3 shared ops;
//                       7 ballots over the digit bits measured 4.38 vs
//                       3.71 ms for the three scatters, __match_any_sync
//                       ~10x slower), the tile is staged in shared
//                       memory in digit order and written so consecutive
//                       threads store consecutive addresses of a run  R8 + W8
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bulk_copy.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kKvThreads = 256;
constexpr int kKvItems = 16;                    // records per thread per tile
constexpr int kKvTile = kKvThreads * kKvItems;  // 4096 records
constexpr int kKvHistThreads = 256;             // histogram CTA: 4 x 1024-key quarters per tile
constexpr int kKvBins = 100;                    // two decimal digits
constexpr int kKvMaxPasses = 5;                 // 10-digit uint32 keys
constexpr int kKvWarps = kKvThreads / 32;

struct KvPass {
  unsigned long long magic_div;   // floor(k / 10^(2*pass)) = (k * magic_div) >> shift_div
  unsigned long long magic_1000;  // floor(q / 100) = (q * magic_1000) >> shift_1000
  uint32_t shift_div, shift_1000;
  uint32_t bins;                  // 100, or 10 on a top pass with one digit left
  uint64_t chunk;                 // records per CTA (multiple of kKvTile)
  uint32_t G;                     // CTAs
};

// 32-bit high products (magic < 2^32, shift >= 32, exact for every uint32;
// capi.cu div_magic32); shift 0 = divisor 1, shift 64 = 64-bit fallback
__device__ __forceinline__ uint32_t kv_digit(uint32_t key, const KvPass& p) {
  uint32_t q;
  if (p.shift_div == 64) q = static_cast<uint32_t>(__umul64hi(static_cast<unsigned long long>(key), p.magic_div));
  else if (p.shift_div == 0) q = key;
  else q = __umulhi(key, static_cast<uint32_t>(p.magic_div)) >> (p.shift_div - 32);
  return q - 100u * (__umulhi(q, static_cast<uint32_t>(p.magic_1000)) >> (p.shift_1000 - 32));
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
  uint32_t mx = 0;
  uint64_t base = c0;
  if (aligned) {  // whole tiles: 4 vectors in flight per thread, no bounds checks
    for (; base + kKvTile <= c1; base += kKvTile) {
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = __ldcs(reinterpret_cast<const uint4*>(keys + base + q * 1024 + threadIdx.x * 4));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t v[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          mx = v[e] > mx ? v[e] : mx;
          atomicAdd(&s_h[kv_digit(v[e], p)], 1u);
        }
      }
    }
  }
  for (uint64_t i = base + threadIdx.x; i < c1; i += blockDim.x) {
    const uint32_t v = keys[i];
    mx = v > mx ? v : mx;
    atomicAdd(&s_h[kv_digit(v, p)], 1u);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x)
    if (s_h[b]) atomicAdd(&hist[(uint64_t)b * p.G + c], s_h[b]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(&st->max_key, static_cast<unsigned long long>(mx));
}

// Shared layout: two input buffers of one tile (keys then values, 32 KB
// each) filled by 1D TMA bulk copies one tile ahead; after a tile's records
// are in registers its buffer becomes that tile's output staging.
constexpr size_t kKvSmemBytes = 2 * (size_t)kKvTile * 8  // s_in[2] (keys | vals)
                                + kKvWarps * kKvBins * 2  // s_wh
                                + kKvBins * 4 * 2         // s_cnt, s_cur
                                + kKvTile                 // s_dig
                                + kKvWarps * kKvBins * 4;  // s_bm

__global__ void __launch_bounds__(kKvThreads, 3) k_kv_chunk_scatter(const uint32_t* __restrict__ keys_in,
                                                                 const uint32_t* __restrict__ vals_in,
                                                                 uint32_t* __restrict__ keys_out,
                                                                 uint32_t* __restrict__ vals_out, uint64_t n,
                                                                 KvPass p, const uint32_t* __restrict__ off,
                                                                 bool bulk_ok) {
  extern __shared__ __align__(128) unsigned char kv_smem[];
  uint32_t* s_in = reinterpret_cast<uint32_t*>(kv_smem);              // [2][2][kKvTile]
  uint16_t* s_wh = reinterpret_cast<uint16_t*>(s_in + 4 * kKvTile);   // [kKvWarps][kKvBins]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_wh + kKvWarps * kKvBins);
  uint32_t* s_cur = s_cnt + kKvBins;
  uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_cur + kKvBins);  // [kKvTile]
  uint32_t* s_bm = reinterpret_cast<uint32_t*>(s_dig + kKvTile);  // [kKvWarps][kKvBins] lane bitmaps
  __shared__ uint32_t s_scan[kKvWarps];
  __shared__ uint32_t s_total;
  __shared__ __align__(8) unsigned long long s_bar[2];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t b = threadIdx.x; b < p.bins; b += blockDim.x) s_cur[b] = off[(uint64_t)b * p.G + blockIdx.x];
  for (int i = threadIdx.x; i < kKvWarps * kKvBins; i += blockDim.x) s_wh[i] = 0;
  for (int i = threadIdx.x; i < kKvWarps * kKvBins; i += blockDim.x) s_bm[i] = 0;
  uint32_t* bm = s_bm + warp * kKvBins;
  const uint64_t c0 = (uint64_t)blockIdx.x * p.chunk;
  const uint64_t c1 = c0 + p.chunk < n ? c0 + p.chunk : n;
  uint16_t* wh = s_wh + warp * kKvBins;
  // a tile can be bulk-loaded when it is full and the inputs are 16-byte aligned
  auto full_tile = [&](uint64_t t0) { return bulk_ok && t0 + kKvTile <= c1; };
  auto issue = [&](uint64_t t0, int buf) {  // one thread
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[buf], 2 * kKvTile * 4);
    bulk_g2s(s_in + buf * 2 * kKvTile, keys_in + t0, kKvTile * 4, &s_bar[buf]);
    bulk_g2s(s_in + buf * 2 * kKvTile + kKvTile, vals_in + t0, kKvTile * 4, &s_bar[buf]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && c0 < c1 && full_tile(c0)) issue(c0, 0);
  unsigned phase = 0;  // bit b: parity of buffer b's barrier
  int buf = 0;
  for (uint64_t t0 = c0; t0 < c1; t0 += kKvTile, buf ^= 1) {
    const uint64_t nt = t0 + kKvTile;
    if (threadIdx.x == 0 && nt < c1 && full_tile(nt)) issue(nt, buf ^ 1);
    const bool full = full_tile(t0);  // block-uniform
    uint32_t* in_k = s_in + buf * 2 * kKvTile;
    uint32_t* in_v = in_k + kKvTile;
    // striped order: record t0 + warp*512 + j*32 + lane (input order =
    // warp-major, then j, then lane)
    uint32_t k[kKvItems], v[kKvItems];
    uint32_t d[kKvItems];  // digit (0xffff: no record) | the record's rank << 16 once ranked
    if (full) {
      mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
#pragma unroll
      for (int j = 0; j < kKvItems; ++j) {
        const uint32_t i = warp * (kKvItems * 32) + j * 32 + lane;
        k[j] = in_k[i];
        v[j] = in_v[i];
        d[j] = kv_digit(k[j], p);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kKvItems; ++j) {
        const uint64_t i = t0 + warp * (kKvItems * 32) + j * 32 + lane;
        const bool ok = i < c1;
        k[j] = ok ? __ldcs(keys_in + i) : 0u;
        v[j] = ok ? __ldcs(vals_in + i) : 0u;
        d[j] = ok ? kv_digit(k[j], p) : 0xffffu;
      }
    }
    // stable warp ranks: rank = the warp's running count of the digit + the
    // peers in lower lanes
#pragma unroll
    for (int j = 0; j < kKvItems; ++j) {
      const bool ok = full || d[j] != 0xffffu;
      // peers (lanes with the same digit) from the warp's shared lane bitmap
      // of that digit: one OR, one read, one reset by the leader
      if (ok) atomicOr(&bm[d[j]], 1u << lane);
      __syncwarp();
      const unsigned peers = ok ? bm[d[j]] : 0u;
      uint32_t base = 0;
      if (ok) base = wh[d[j]];
      __syncwarp();
      if (ok && (peers & lt) == 0) {
        wh[d[j]] = static_cast<uint16_t>(base + __popc(peers));
        bm[d[j]] = 0u;
      }
      __syncwarp();
      d[j] |= (base + __popc(peers & lt)) << 16;
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
    // tile-local exclusive scan over digits (warps 0..3, one digit per lane)
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
      if (b < p.bins) {
        const uint32_t start = before + inc - c;
        s_cnt[b] = s_cur[b] - start;  // this tile's destination base: dest(i) = s_cnt[b] + i
        s_cur[b] += c;
        // the digit's start in the tile folded into its warp prefixes: one
        // lookup per staged record
#pragma unroll 1
        for (int w = 0; w < kKvWarps; ++w) s_wh[w * kKvBins + b] += static_cast<uint16_t>(start);
      }
      if (b == 127) s_total = before + inc;
    }
    __syncthreads();
    // stage (key | value) in digit order into this tile's consumed input
    // buffer, and the digit as one byte
    unsigned long long* stage = reinterpret_cast<unsigned long long*>(in_k);
#pragma unroll
    for (int j = 0; j < kKvItems; ++j) {
      const uint32_t dj = d[j] & 0xffffu;
      if (dj != 0xffffu) {
        const uint32_t pos = wh[dj] + (d[j] >> 16);
        stage[pos] = (static_cast<unsigned long long>(v[j]) << 32) | k[j];
        s_dig[pos] = static_cast<uint8_t>(dj);
      }
    }
    __syncthreads();
    const uint32_t total = s_total;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
      const unsigned long long kv = stage[i];
      const uint32_t g = s_cnt[s_dig[i]] + i;
      keys_out[g] = static_cast<uint32_t>(kv);
      vals_out[g] = static_cast<uint32_t>(kv >> 32);
    }
    for (int i = threadIdx.x; i < kKvWarps * kKvBins; i += blockDim.x) s_wh[i] = 0;
    __syncthreads();
  }
}

// Multi-GPU stable key/value placement: records already in
// this rank's stable local order (record i, key k) go to their final global
// position P = cell_off[k] + i in the output slice of the rank owning cell k
// (cell_off folds in the global cell start, the earlier ranks' counts of k
// and this rank's local start of k, minus the owner's slice start).  The
// destination is a peer GPU's buffer mapped over NVLink, so the placement
// kernel is the all-to-all; records of one cell land as one contiguous run.
__global__ void __launch_bounds__(256) k_kv_place(const uint32_t* __restrict__ keys,
                                                  const uint32_t* __restrict__ vals, uint64_t n,
                                                  const long long* __restrict__ cell_off,
                                                  const uint8_t* __restrict__ cell_owner,
                                                  uint32_t* const* __restrict__ dst_k,
                                                  uint32_t* const* __restrict__ dst_v, uint32_t ranks,
                                                  uint64_t cells, unsigned* __restrict__ bad) {
  __shared__ uint32_t* s_k[64];
  __shared__ uint32_t* s_v[64];
  for (uint32_t r = threadIdx.x; r < ranks; r += blockDim.x) {
    s_k[r] = dst_k[r];
    s_v[r] = dst_v[r];
  }
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t k = __ldcs(keys + i);
    if (k >= cells) {  // outside the grid the placement tables cover: flagged, never stored
      *bad = 1u;
      continue;
    }
    const uint32_t r = __ldg(cell_owner + k);
    if (r >= ranks) {
      *bad = 1u;
      continue;
    }
    const uint64_t off = static_cast<uint64_t>(__ldg(cell_off + k) + static_cast<long long>(i));
    s_k[r][off] = k;
    s_v[r][off] = __ldcs(vals + i);
  }
}

}  // namespace rsb

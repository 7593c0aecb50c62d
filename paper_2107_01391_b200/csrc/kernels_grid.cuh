// kernels_grid.cuh — the single-grid hot path on sm_100a.
//
//   K1 map+count   hashing cycle: hash_insert / CountSpace::increment
//                  (hashing.cpp:27-38, hashing.hpp:71-75) fused with the
//                  mapper (sort.cpp:42-46, key_model.cpp:135-158).
//   K2+K3 scan     occupancy (TraverseMaps, hashing.hpp:21-48) as warp ballots
//                  over count>0, compacted with a single-pass decoupled
//                  look-back exclusive scan over cells.
//   K4 emit        extract's run-length copy loop (extraction.cpp:21-29) as a
//                  load-balanced expand over output positions.
//   report         ExtractionReport (extraction.hpp:12-15) from per-row
//                  first/last keys of the sorted output.
//
// Layout in HBM: keys are streamed once per pass with 16-byte vector loads;
// the grid is a dense uint32 array of radix^n counters (4 MB at 10^6 cells,
// L2-resident on B200's 126 MB L2); the occupied-cell list is two arrays
// (cell id u32, inclusive key prefix u64).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels_f64.cuh"
#include "rs_internal.cuh"

namespace rsb {

constexpr int kThreads = 256;
constexpr int kScanPerThread = 16;
constexpr int kScanTile = kThreads * kScanPerThread;  // 4096 cells per scan tile
constexpr int kEmitTile = 8192;                       // output positions per emit CTA
constexpr int kEmitCap = 2048;                        // occupied cells staged per emit tile
constexpr uint32_t kSmemCellsMax = 12288;             // smem-privatised grid limit (48 KB)

// ------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t d_digit_count(unsigned long long v) {
  uint32_t d = 1;
  while (v >= 10ull) {
    v /= 10ull;
    ++d;
  }
  return d;
}

__device__ __forceinline__ unsigned long long d_pow(unsigned long long radix, uint32_t e) {
  unsigned long long r = 1;
  for (uint32_t i = 0; i < e; ++i) r *= radix;
  return r;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ ulonglong2 ld_stream(const ulonglong2* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }

__device__ __forceinline__ void warp_max_to(unsigned long long v, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0 && v) atomicMax(dst, v);
}

__device__ __forceinline__ unsigned warp_or(unsigned v) { return __reduce_or_sync(0xffffffffu, v); }

// One hash_insert for a warp-uniform call site.  With kAggregate the lanes
// holding the same cell elect a leader (__match_any_sync) that adds the
// group's population, so a hot cell costs one L2 atomic per warp, not 32.
template <bool kAggregate>
__device__ __forceinline__ void count_cell_global(uint32_t* __restrict__ counts,
                                                  uint32_t cell, bool valid) {
  if constexpr (kAggregate) {
    const unsigned tag = valid ? cell : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, tag);
    const int leader = __ffs(peers) - 1;
    if (valid && (int)(threadIdx.x & 31) == leader) atomicAdd(&counts[cell], (unsigned)__popc(peers));
  } else {
    if (valid) atomicAdd(&counts[cell], 1u);
  }
}

// ------------------------------------------------------------- mappers
// A mapper turns one input element into (cell, valid, flags).  `cells` is
// the grid size; keys at or beyond it set overflow (hint too small or a key
// outside the spec, hashing.cpp:31-34).
struct MapU32 {
  using In = uint32_t;
  using Key = uint32_t;  // mapped keys fit 32 bits: the partition works in 32-bit arithmetic
  __device__ __forceinline__ unsigned long long operator()(uint32_t k, unsigned&) const { return k; }
  __device__ __forceinline__ uint32_t key32(uint32_t k, unsigned&) const { return k; }
};

struct MapI64 {
  using In = int64_t;
  using Key = unsigned long long;
  __device__ __forceinline__ unsigned long long operator()(int64_t v, unsigned& flags) const {
    if (v < 0) {
      flags |= kFlagNegative;
      return 0;
    }
    return static_cast<unsigned long long>(v);
  }
};

struct MapU64 {
  using In = unsigned long long;
  using Key = unsigned long long;
  __device__ __forceinline__ unsigned long long operator()(unsigned long long v, unsigned&) const { return v; }
};

// float_to_decimal(x, scale) (key_model.cpp:135-158) without a string round
// trip.  Let P = 10^scale and m = floor(x*P) computed exactly (fma residual).
// Inside the domain (x == 0 or x > 10^-(scale+3)) and x*P*100 < 2^53 the set of reals that round to x spans
// less than 0.02 in units of 1/P, so:
//  * if m/P or (m+1)/P rounds to x, the shortest round-trip numeral has at
//    most `scale` fractional digits and equals it  -> that mantissa;
//  * else if (m+1/2)/P rounds to x, the shortest numeral is exactly that
//    half-way point, which the reference rounds up -> m+1;
//  * else the shortest numeral and x lie on the same side of m+1/2, so the
//    half-up result is decided by x*P versus m+1/2, exactly.
// IEEE division of two exact doubles (m < 2^53, P <= 10^15) is correctly
// rounded, so every "rounds to x" test is exact.
// The exact float64 mapping out of line: the hot loops keep their registers
// for the fast tests and pay a call only for the keys those leave undecided.
template <class Map>
__device__ __noinline__ unsigned long long map_exact(const Map& map, double x, unsigned& flags) {
  return map.exact(x, flags);
}

// kGeneral = false: the lean mapper of the hot kernels — a value outside
// the fast domain raises kFlagDomain and the host redoes the sort with
// kGeneral = true, whose exact() takes the exact general search for
// those values (a call the hot kernels' register budget never pays for).
template <bool kGeneral>
struct MapF64T {
  using In = double;
  using Key = unsigned long long;
  static constexpr bool kMapFirst = true;  // a separate streaming map pass, then the uint32 partition
  double P;      // 10^scale
  double limit;  // 2^53 / 100
  double tiny;   // just above 10^-(scale+3)
  uint32_t scale;
  unsigned long long Pi;         // 10^scale; 0 outside the fast domain (scale > 15)
  unsigned long long xlim_bits;  // bits of the least x with RN(x * P) >= limit
  unsigned long long tiny_bits;  // bits of tiny
  unsigned long long zero_bits;  // 0: +0 is decided by fast(); ~0 (scale > 15): it is not
  // The mapping every kernel calls: the fast tests below, the exact path
  // (out of line) for the keys they leave undecided.
  __device__ __forceinline__ unsigned long long operator()(double x, unsigned& flags) const {
    bool und;
    const double kd = fast(x, und);
    return und ? map_exact(*this, x, flags) : static_cast<unsigned long long>(kd);
  }
  // The exact mapping (also classifies bad inputs).
  __device__ __forceinline__ unsigned long long exact(double x, unsigned& flags) const {
    if (!isfinite(x)) {
      flags |= kFlagNonFinite;
      return 0;
    }
    if (x < 0.0) {
      flags |= kFlagNegative;
      return 0;
    }
    const double p = x * P;
    // Outside the fast domain (tiny values, whose shortest numeral may have
    // >= scale+20 fractional digits, and x * 10^(scale+2) >= 2^53): the
    // exact general search (kernels_f64.cuh)
    if (!(p < limit) || (x > 0.0 && x < tiny)) {
      if constexpr (kGeneral) {
        uint32_t code;
        const unsigned long long k = f2d_general(x, scale, code);
        if (code != kF2dOk) flags |= kFlagBudget;
        return k;
      } else {
        flags |= kFlagDomain;
        return 0;
      }
    }
    const double err = fma(x, P, -p);  // x*P == p + err exactly
    double f = floor(p);
    if (p == f && err < 0.0) f -= 1.0;
    const unsigned long long m = static_cast<unsigned long long>(f);
    const double fr = p - f;  // exact, in [0, 1]
    // The reals that round to x span < 0.02 in units of 1/P and |err| is far
    // below 0.001, so an integer (or half-integer) candidate can only round
    // to x when p lies within 0.02 of it: test only the nearest candidate.
    if (fr < 0.02 || fr > 0.98) {
      const unsigned long long c = fr < 0.5 ? m : m + 1;
      if (static_cast<double>(c) / P == x) return c;
    } else if (fr > 0.48 && fr < 0.52) {
      if (static_cast<double>(2 * m + 1) / (2.0 * P) == x) return m + 1;
    }
    const bool up = fr > 0.5 || (fr == 0.5 && err > 0.0);
    return up ? m + 1 : m;
  }
  // The same mapping for the hot kernels.  Away from the half-way point the
  // candidate tests of exact() cannot change the result: with fr < 0.02
  // the integer candidate is m and the half-up rule also gives m, with
  // fr > 0.98 both give m + 1, and in between (|fr - 1/2| > 0.02) the
  // shortest numeral lies within 0.01 of x * P and rounds like it.  So the
  // mantissa is rint(x * P) unless |fr - 1/2| <= 0.02, where the half-integer
  // candidate (2m+1) / 2P is tested without a division: x == RN(c / d) iff
  // the exact residual c - x*d lies inside x's rounding interval, of
  // half-width h = d * ulp(x) / 2 (exact: an exponent shift of d's bits);
  // r = |fma(-x, d, c)| rounds it once, so r < h proves it and r > h refutes
  // it.  r == h and powers of two (narrower spacing below x) stay
  // undecided, as do keys outside the fast domain (one unsigned range check
  // on the bits of x: non-negative doubles order as their bit patterns):
  // those go through exact() (mirrored by
  // tests/test_f64_mapping.py::kernel_f64_fast).  +0 is decided (rint gives
  // 0) unless scale > 15 (zero_bits).  Returns the mantissa as a double
  // (exact: < 2^53 / 100); meaningless when undecided.
  __device__ __forceinline__ double fast(double x, bool& undecided) const {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    undecided = u - tiny_bits >= xlim_bits - tiny_bits && u != zero_bits;
    const double p = x * P;
    const double c = rint(p);
    const double d = p - c;  // exact, in [-1/2, 1/2]
    if ((__double2hiint(d) & 0x7FFFFFFF) < 0x3FDEB851) return c;  // |d| < 0.48 (widened by < 2^-20)
    const double m = d >= 0.0 ? c : c - 1.0;  // floor(p): p is no integer here
    const double dv = 2.0 * P;
    const long long hb = __double_as_longlong(dv) + (static_cast<long long>(static_cast<int>(u >> 52) - 1076) << 52);
    const long long rb = __double_as_longlong(fma(-x, dv, fma(m, 2.0, 1.0))) & 0x7FFFFFFFFFFFFFFFll;
    undecided = undecided || (u & ((1ull << 52) - 1)) == 0 || rb == hb;
    if (rb < hb) return m + 1.0;  // the shortest numeral is m + 1/2: half-up
    const double fr = p - m;      // exact
    const bool up = fr > 0.5 || (fr == 0.5 && fma(x, P, -p) > 0.0);
    return up ? m + 1.0 : m;
  }
};
using MapF64 = MapF64T<false>;
using MapF64G = MapF64T<true>;
template <class M>
struct is_f64_map : std::false_type {};
template <bool G>
struct is_f64_map<MapF64T<G>> : std::true_type {};

template <class M, class = void>
struct map_first : std::false_type {};
template <class M>
struct map_first<M, std::void_t<decltype(M::kMapFirst)>> : std::true_type {};

// Heavy mappers (float64): every input mapped once into a uint32 cell by a
// streaming pass at full occupancy (cells >= 2^32 clamp to 0xFFFFFFFF, which
// still lies outside any grid the two-level split serves), so the tuned
// uint32 partition runs on the cells; max key and flags as in the fused path.
template <class Map>
__global__ void __launch_bounds__(kThreads, 4) k_map_cells(const typename Map::In* __restrict__ in, uint64_t n, Map map,
                                                        bool aligned, uint32_t* __restrict__ out, DevStats* st) {
  using In = typename Map::In;
  unsigned long long mx = 0;
  unsigned flags = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (is_f64_map<Map>::value) {
    // float64: the fast tests, the exact path for the keys they leave
    // undecided; the converted cell saturates at 0xFFFFFFFF, the max runs
    // over the cells (the exact key only past the saturation, rarely)
    uint32_t mx32 = 0;
    auto cell = [&](double x) -> uint32_t {
      bool und;
      const double kd = map.fast(x, und);
      uint32_t c = __double2uint_rz(kd);
      if (und) {
        const unsigned long long k = map_exact(map, x, flags);
        mx = k > mx ? k : mx;
        c = k < 0xFFFFFFFFull ? static_cast<uint32_t>(k) : 0xFFFFFFFFu;
      } else if (c == 0xFFFFFFFFu) {
        const unsigned long long k = static_cast<unsigned long long>(kd);
        mx = k > mx ? k : mx;
      }
      mx32 = max(mx32, c);
      return c;
    };
    if (aligned) {  // two inputs per 16-byte load, four loads in flight, two cells per 8-byte store
      const uint64_t pairs = n / 2;
      const auto* src = reinterpret_cast<const double2*>(in);
      auto* dst = reinterpret_cast<uint2*>(out);
      uint64_t p = i;
      for (; p + 3 * stride < pairs; p += 4 * stride) {
        double2 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = __ldcs(src + p + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[p + u * stride] = make_uint2(cell(w[u].x), cell(w[u].y));
      }
      for (; p < pairs; p += stride) {
        const double2 w = __ldcs(src + p);
        dst[p] = make_uint2(cell(w.x), cell(w.y));
      }
      if ((n & 1) && i == 0) out[n - 1] = cell(in[n - 1]);
      i = n;  // done
    }
    for (; i < n; i += stride) out[i] = cell(in[i]);
    mx = mx32 > mx ? mx32 : mx;
  } else {
    auto cell = [&](In x) -> uint32_t {
      const unsigned long long k = map(x, flags);
      mx = k > mx ? k : mx;
      return k < 0xFFFFFFFFull ? static_cast<uint32_t>(k) : 0xFFFFFFFFu;
    };
    for (; i < n; i += stride) out[i] = cell(in[i]);
  }
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

// ----------------------------------------------------------- K0: max pass
// The reference derives the geometry from the dataset max (sort.cpp:31-40);
// without a declared width this pass runs first.
template <class Map>
__global__ void __launch_bounds__(kThreads) k_max(const typename Map::In* __restrict__ in,
                                                  uint64_t n, Map map, DevStats* st) {
  unsigned long long mx = 0;
  unsigned flags = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  using In = typename Map::In;
  if constexpr (!is_f64_map<Map>::value) {  // cheap maps: 16-byte vectors, four in flight per thread
    constexpr int kPer = 16 / sizeof(In);
    if ((reinterpret_cast<uintptr_t>(in) & 15) == 0) {
      const uint64_t nv = n / kPer;
      const auto* v4 = reinterpret_cast<const uint4*>(in);
      uint64_t p = i;
      for (; p + 3 * stride < nv; p += 4 * stride) {
        uint4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = __ldcs(v4 + p + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const In* e = reinterpret_cast<const In*>(&w[u]);
#pragma unroll
          for (int q = 0; q < kPer; ++q) {
            const unsigned long long k = map(e[q], flags);
            mx = k > mx ? k : mx;
          }
        }
      }
      for (; p < nv; p += stride) {
        const uint4 w = __ldcs(v4 + p);
        const In* e = reinterpret_cast<const In*>(&w);
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const unsigned long long k = map(e[q], flags);
          mx = k > mx ? k : mx;
        }
      }
      i = nv * kPer + i;  // the tail
    }
  }
  for (; i < n; i += stride) {
    const unsigned long long k = map(__ldcs(in + i), flags);
    mx = k > mx ? k : mx;
  }
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

// The max of an evenly strided sample of `samples` elements: the width the
// counting pass is planned for when the caller declares none.  The pass
// itself folds in the true max and flags a key outside the planned grid, so
// a sample that misses the max costs a second sort, never a wrong one.
template <class Map>
__global__ void __launch_bounds__(kThreads) k_max_sample(const typename Map::In* __restrict__ in, uint64_t n,
                                                         uint32_t samples, Map map, DevStats* st) {
  unsigned long long mx = 0;
  unsigned flags = 0;
  const uint64_t step = n / samples > 0 ? n / samples : 1;  // one 64-bit division, not one per sample
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < samples; s += gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)s * step < n ? (uint64_t)s * step : n - 1;
    const unsigned long long k = map(__ldg(in + i), flags);
    mx = k > mx ? k : mx;
  }
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

// ------------------------------------------------- K1: map + count (L2 grid)
// Grid-stride over 16-byte vectors of the input; every lane of a warp runs
// the same trip count so __match_any_sync always sees the full warp.
template <class Map, bool kAggregate>
__global__ void __launch_bounds__(kThreads) k_count_global(const typename Map::In* __restrict__ in,
                                                           uint64_t n, Map map,
                                                           uint32_t* __restrict__ counts,
                                                           unsigned long long cells, DevStats* st) {
  using In = typename Map::In;
  constexpr int kVec = 16 / sizeof(In);
  using Vec = typename std::conditional<sizeof(In) == 4, uint4,
              typename std::conditional<std::is_same<In, double>::value, double2, ulonglong2>::type>::type;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(in);
  const uint64_t head0 = ((16 - (addr & 15)) & 15) / sizeof(In);
  const uint64_t head = head0 < n ? head0 : n;
  const uint64_t nvec = (n - head) / kVec;
  const uint64_t tail0 = head + nvec * kVec;
  const Vec* v = reinterpret_cast<const Vec*>(in + head);

  unsigned long long mx = 0;
  unsigned flags = 0, ovf = 0;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  constexpr int kUnroll = 2;
  const uint64_t iters = (nvec + stride * kUnroll - 1) / (stride * kUnroll);
  for (uint64_t it = 0; it < iters; ++it) {
    Vec q[kUnroll];
    bool ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = tid + (it * kUnroll + u) * stride;
      ok[u] = i < nvec;
      if (ok[u]) q[u] = ld_stream(v + i);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const In* e = reinterpret_cast<const In*>(&q[u]);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        unsigned long long k = 0;
        if (ok[u]) k = map(e[j], flags);
        const bool in_grid = ok[u] && k < cells;
        ovf |= (ok[u] && k >= cells);
        mx = (ok[u] && k > mx) ? k : mx;
        count_cell_global<kAggregate>(counts, static_cast<uint32_t>(k), in_grid);
      }
    }
  }
  // unaligned head and tail elements (fewer than kVec of each)
  if (blockIdx.x == 0) {
    const uint64_t tcount = n - tail0;
    uint64_t i = ~0ull;
    if (threadIdx.x < head) i = threadIdx.x;
    else if (threadIdx.x - head < tcount) i = tail0 + (threadIdx.x - head);
    if (i < n) {
      const unsigned long long k = map(in[i], flags);
      if (k < cells) atomicAdd(&counts[k], 1u);
      else ovf = 1;
      mx = k > mx ? k : mx;
    }
  }
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

// ------------------------------------------ K1': map + count (smem grid)
// For grids of at most kSmemCellsMax cells: block-private shared-memory
// histogram, flushed once per CTA.
template <class Map>
__global__ void __launch_bounds__(kThreads) k_count_smem(const typename Map::In* __restrict__ in,
                                                         uint64_t n, Map map,
                                                         uint32_t* __restrict__ counts,
                                                         unsigned long long cells, DevStats* st) {
  extern __shared__ uint32_t s_hist[];
  for (uint32_t c = threadIdx.x; c < cells; c += blockDim.x) s_hist[c] = 0;
  __syncthreads();
  unsigned long long mx = 0;
  unsigned flags = 0, ovf = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t iters = (n + stride - 1) / stride;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t i = tid + it * stride;
    const bool ok = i < n;
    unsigned long long k = 0;
    if (ok) k = map(__ldcs(in + i), flags);
    const bool in_grid = ok && k < cells;
    ovf |= ok && k >= cells;
    mx = (ok && k > mx) ? k : mx;
    // plain shared atomics: __match_any_sync aggregation measured ~10x
    // slower on B200 for uniform keys (profiles/r1_microbench.txt)
    if (in_grid) atomicAdd(&s_hist[k], 1u);
  }
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < cells; c += blockDim.x)
    if (s_hist[c]) atomicAdd(&counts[c], s_hist[c]);
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if ((threadIdx.x & 31) == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
}

// ------------------------------------ K2+K3: occupancy + look-back scan
// Tile t covers cells [t*4096, (t+1)*4096).  Each warp ballots count>0 over
// its cells (the occupancy bitmap, one 32-bit word per ballot) and the block
// scans (occupied, keys) pairs; tiles chain through a decoupled look-back
// with one 64-bit descriptor per quantity: [63:62] flag (1 aggregate,
// 2 inclusive prefix), [61:0] value.
constexpr unsigned long long kDescAgg = 1ull << 62;
constexpr unsigned long long kDescPre = 2ull << 62;
constexpr unsigned long long kDescVal = (1ull << 62) - 1;

// Exclusive prefix of `tile` from its predecessors' descriptors, called by a
// whole warp: lane l reads descriptor tile-1-l, so one window of 32
// predecessors costs one round trip; the window's aggregates are summed up to
// the nearest inclusive prefix, else the warp moves 32 tiles back.
__device__ __forceinline__ unsigned long long warp_lookback(volatile unsigned long long* desc, uint32_t tile) {
  const int lane = threadIdx.x & 31;
  unsigned long long prefix = 0;
  for (int64_t base = (int64_t)tile - 1;; base -= 32) {
    const int64_t i = base - lane;
    unsigned long long d = kDescPre;  // before tile 0: an empty inclusive prefix
    if (i >= 0) {
      do {
        d = desc[i];
      } while ((d >> 62) == 0);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (d >> 62) == 2);
    const int stop = pre ? __ffs(pre) - 1 : 31;
    unsigned long long v = lane <= stop ? (d & kDescVal) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (pre) return prefix;
  }
}

template <class C>
__global__ void __launch_bounds__(kThreads) k_scan_cells(const C* __restrict__ counts,
                                                         unsigned long long cells,
                                                         uint32_t* __restrict__ occ_cell,
                                                         unsigned long long* __restrict__ occ_end,
                                                         unsigned long long* desc_occ,
                                                         unsigned long long* desc_sum,
                                                         uint32_t num_tiles, DevStats* st,
                                                         uint32_t etiles, uint32_t* __restrict__ tile_first,
                                                         uint4* __restrict__ spans) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wocc[kThreads / 32], s_wsum[kThreads / 32];
  __shared__ unsigned long long s_pocc, s_psum;
  if (threadIdx.x == 0) s_tile = atomicAdd(&st->tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const unsigned long long c0 = (unsigned long long)tile * kScanTile + threadIdx.x * kScanPerThread;
  C c[kScanPerThread];
  // 16-byte loads need a 16-byte aligned grid (rs_emit_u32 scans sub-ranges from any cell);
  // 64-bit counts (inputs of 2^32 keys or more) are read one by one
  if (sizeof(C) == 4 && c0 + kScanPerThread <= cells && (reinterpret_cast<uintptr_t>(counts) & 15) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(counts + c0);
#pragma unroll
    for (int q = 0; q < kScanPerThread / 4; ++q) {
      const uint4 w = p[q];
      c[4 * q] = w.x; c[4 * q + 1] = w.y; c[4 * q + 2] = w.z; c[4 * q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanPerThread; ++k) c[k] = (c0 + k < cells) ? counts[c0 + k] : C{0};
  }
  uint32_t occ = 0;
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    occ += c[k] != 0;
    sum += c[k];
  }
  // warp inclusive scans
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t iocc = occ;
  unsigned long long isum = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, iocc, o);
    const unsigned long long b = __shfl_up_sync(0xffffffffu, isum, o);
    if (lane >= o) {
      iocc += a;
      isum += b;
    }
  }
  if (lane == 31) {
    s_wocc[warp] = iocc;
    s_wsum[warp] = isum;
  }
  __syncthreads();
  // tile totals (every thread; the warp sums are in shared memory)
  unsigned long long ro = 0, rs = 0, bo = 0, bs = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const unsigned long long a = s_wocc[w], b = s_wsum[w];
    bo += w < warp ? a : 0ull;
    bs += w < warp ? b : 0ull;
    ro += a;
    rs += b;
  }
  // warp 0 chains the occupied count, warp 1 the key sum
  if (warp < 2) {
    volatile unsigned long long* vd = warp == 0 ? desc_occ : desc_sum;
    const unsigned long long r = warp == 0 ? ro : rs;
    unsigned long long p = 0;
    if (tile == 0) {
      if (lane == 0) vd[0] = kDescPre | r;
    } else {
      if (lane == 0) vd[tile] = kDescAgg | r;
      p = warp_lookback(vd, tile);
      if (lane == 0) vd[tile] = kDescPre | (p + r);
    }
    if (lane == 0) {
      if (warp == 0) s_pocc = p;
      else s_psum = p;
    }
  }
  __syncthreads();
  const unsigned long long m = s_pocc + ro, total = s_psum + rs;
  if (tile == num_tiles - 1 && threadIdx.x == 0) {
    st->n_occupied = m;
    st->total = total;
  }
  unsigned long long pos = s_pocc + bo + (iocc - occ);
  unsigned long long run = s_psum + bs + (isum - sum);
  // emit tile e starts at output position e*kEmitTile: the occupied cell
  // whose key run holds that position starts the tile (tile_first[e]).  A
  // cell spanning one or two tiles is written by its thread; longer spans
  // (hot cells, all in one scan tile under skew) go to a list that
  // k_fill_spans spreads over the whole GPU.
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (c[k]) {
      occ_cell[pos] = static_cast<uint32_t>(c0 + k);
      if (tile_first) {
        const unsigned long long e0 = (run + kEmitTile - 1) / kEmitTile;
        unsigned long long e1 = (run + c[k] + kEmitTile - 1) / kEmitTile;
        e1 = e1 < etiles ? e1 : etiles;
        if (e1 > e0 + 2) {
          spans[atomicAdd(&st->long_spans, 1u)] =
              make_uint4(static_cast<uint32_t>(e0), static_cast<uint32_t>(e1), static_cast<uint32_t>(pos), 0u);
        } else {
          for (unsigned long long e = e0; e < e1; ++e) tile_first[e] = static_cast<uint32_t>(pos);
        }
      }
      run += c[k];
      occ_end[pos] = run;
      ++pos;
    }
  }
  // sentinels: tiles past the counted keys (keys outside the grid) and entry etiles
  if (tile_first && tile == num_tiles - 1)
    for (unsigned long long e = (total + kEmitTile - 1) / kEmitTile + threadIdx.x; e <= etiles; e += blockDim.x)
      tile_first[e] = static_cast<uint32_t>(m);
}

// tile_first over the long spans listed by k_scan_cells (disjoint tile
// ranges, at most etiles/3 of them): one CTA per span, threads over tiles.
__global__ void k_fill_spans(const uint4* __restrict__ spans, const DevStats* st, uint32_t* __restrict__ tile_first) {
  const uint32_t count = st->long_spans;
  for (uint32_t s = blockIdx.x; s < count; s += gridDim.x) {
    const uint4 u = spans[s];
    for (uint32_t e = u.x + threadIdx.x; e < u.y; e += blockDim.x) tile_first[e] = u.z;
  }
}

// First occupied-cell index of every emit tile when the key total is only
// known after the scan (rs_emit_u32; grid sorts fill it inside k_scan_cells): tile_first[t] = first j with
// occ_end[j] > t*kEmitTile (t = 0..tiles; entry `tiles` is the sentinel M).
__global__ void k_tile_first(const unsigned long long* __restrict__ occ_end, const DevStats* st,
                             uint64_t n, uint32_t tiles, uint32_t* __restrict__ tile_first) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  const unsigned long long m = st->n_occupied;
  const unsigned long long p = (unsigned long long)t * kEmitTile;
  if (p >= n) {
    tile_first[t] = static_cast<uint32_t>(m);
    return;
  }
  unsigned long long lo = 0, hi = m;
  while (lo < hi) {
    const unsigned long long mid = (lo + hi) >> 1;
    if (occ_end[mid] > p) hi = mid;
    else lo = mid + 1;
  }
  tile_first[t] = static_cast<uint32_t>(lo);
}

// ----------------------------------------------------------- K4: emit
// Output writers: positions p..p+3 receive key values v[0..3].
struct OutU32 {
  static constexpr int kWordBytes = 4;
  uint32_t* out;
  uint32_t base;
  bool aligned;
  __device__ __forceinline__ void put1(uint64_t p, uint32_t c) const { out[p] = c + base; }
  // p..p+3 inside the output
  __device__ __forceinline__ void put4_full(uint64_t p, const uint32_t (&c)[4]) const {
    if (aligned) {
      __stcs(reinterpret_cast<uint4*>(out + p), make_uint4(c[0] + base, c[1] + base, c[2] + base, c[3] + base));
    } else {
      for (int e = 0; e < 4; ++e) out[p + e] = c[e] + base;
    }
  }
  __device__ __forceinline__ void put4(uint64_t p, const uint32_t (&c)[4], uint64_t end) const {
    if (aligned && p + 4 <= end) {
      __stcs(reinterpret_cast<uint4*>(out + p), make_uint4(c[0] + base, c[1] + base, c[2] + base, c[3] + base));
    } else {
      for (int e = 0; e < 4; ++e)
        if (p + e < end) out[p + e] = c[e] + base;
    }
  }
};

// 256-bit streaming store of four 64-bit values (sm_100: STG.E.EF.ENL2.256);
// p must be 32-byte aligned.
__device__ __forceinline__ void st_cs_v4_b64(unsigned long long* p, unsigned long long a, unsigned long long b,
                                             unsigned long long c, unsigned long long d) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

struct OutU64 {
  static constexpr int kWordBytes = 8;
  unsigned long long* out;
  unsigned long long base;
  bool aligned;  // 32-byte aligned: positions 4k take one 256-bit store
  __device__ __forceinline__ void put1(uint64_t p, uint32_t c) const { out[p] = c + base; }
  __device__ __forceinline__ void put4_full(uint64_t p, const uint32_t (&c)[4]) const {
    if (aligned) {
      st_cs_v4_b64(out + p, c[0] + base, c[1] + base, c[2] + base, c[3] + base);
    } else {
      for (int e = 0; e < 4; ++e) out[p + e] = c[e] + base;
    }
  }
  __device__ __forceinline__ void put4(uint64_t p, const uint32_t (&c)[4], uint64_t end) const {
    if (aligned && p + 4 <= end) {
      st_cs_v4_b64(out + p, c[0] + base, c[1] + base, c[2] + base, c[3] + base);
    } else {
      for (int e = 0; e < 4; ++e)
        if (p + e < end) out[p + e] = c[e] + base;
    }
  }
};

// Each CTA writes output positions [t*8192, (t+1)*8192).  Dense tile (at
// most kEmitCap occupied cells reach it): the cells' run ends are staged in
// shared memory (relative to the tile) and every warp writes 1024
// consecutive positions as 16-byte stores, lane-contiguous; a lane finds the
// cell of its first position by binary search and then walks forward (the
// positions only grow).  Sparse tile (more cells than kEmitCap, i.e. runs of
// ~4 keys or fewer): cell-driven, each thread writes whole runs.
template <class Out>
__global__ void __launch_bounds__(kThreads) k_emit(const uint32_t* __restrict__ occ_cell,
                                                   const unsigned long long* __restrict__ occ_end,
                                                   const uint32_t* __restrict__ tile_first,
                                                   const DevStats* st, uint64_t n, Out out) {
  __shared__ uint32_t s_end[kEmitCap + 1];  // occ_end - p0, clipped to the tile
  __shared__ uint32_t s_cell[kEmitCap + 1];
  const uint32_t t = blockIdx.x;
  const uint64_t p0 = (uint64_t)t * kEmitTile;
  const uint64_t pend = p0 + kEmitTile < n ? p0 + kEmitTile : n;
  const unsigned long long m = st->n_occupied;
  const uint32_t j0 = tile_first[t];
  uint32_t j1 = tile_first[t + 1];
  if (j1 >= m) j1 = static_cast<uint32_t>(m - 1);
  const uint32_t cnt = j1 - j0 + 1;
  if (cnt > kEmitCap) {
    for (uint32_t j = j0 + threadIdx.x; j <= j1; j += blockDim.x) {
      const unsigned long long a0 = j ? occ_end[j - 1] : 0ull;
      const unsigned long long a = a0 > p0 ? a0 : p0;
      const unsigned long long b0 = occ_end[j];
      const unsigned long long b = b0 < pend ? b0 : pend;
      const uint32_t cell = occ_cell[j];
      for (unsigned long long q = a; q < b; ++q) out.put1(q, cell);
    }
    return;
  }
  for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) {
    const unsigned long long e = occ_end[j0 + k] - p0;
    s_end[k] = static_cast<uint32_t>(e < (unsigned long long)kEmitTile ? e : kEmitTile);
    s_cell[k] = occ_cell[j0 + k];
  }
  if (threadIdx.x == 0) {  // sentinel: every position lies before it
    s_end[cnt] = 0xffffffffu;
    s_cell[cnt] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kPerWarp = kEmitTile / (kThreads / 32);  // 1024
  uint32_t k = 0;
  {
    const uint32_t rel = warp * kPerWarp + lane * 4;
    uint32_t lo = 0, hi = cnt;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_end[mid] > rel) hi = mid;
      else lo = mid + 1;
    }
    k = lo < cnt ? lo : cnt - 1;
  }
  const bool full = pend - p0 == (uint64_t)kEmitTile;
  if constexpr (Out::kWordBytes == 4) {
    // 4-byte outputs: the current cell's run end and id stay in registers
    // across groups (long runs cost no shared loads).  Every occupied cell
    // holds >= 1 key, so one position further is at most one cell further:
    // a group that crosses run ends needs no loops.
    uint32_t ek = s_end[k], ck = s_cell[k];
#pragma unroll
    for (int g = 0; g < kPerWarp / 128; ++g) {
      const uint32_t rel = warp * kPerWarp + g * 128 + lane * 4;  // position - p0
      if (!full && p0 + rel >= pend) break;
      while (ek <= rel) {
        ++k;
        ek = s_end[k];
        ck = s_cell[k];
      }
      uint32_t v[4];
      v[0] = v[1] = v[2] = v[3] = ck;
      if (ek < rel + 4) {  // a run ends inside the group
        uint32_t kk = k, e_kk = ek;
#pragma unroll
        for (int e = 1; e < 4; ++e) {
          if (e_kk <= rel + e) {
            ++kk;
            e_kk = s_end[kk];
          }
          v[e] = s_cell[kk];
        }
      }
      if (full) out.put4_full(p0 + rel, v);
      else out.put4(p0 + rel, v, pend);
    }
  } else {
    // wider outputs (64-bit keys, records): the store stream, not the walk,
    // sets the pace (measured: the tighter walk above floods the store queue
    // and starves the next CTAs' setup loads)
#pragma unroll
    for (int g = 0; g < kPerWarp / 128; ++g) {
      const uint32_t rel = warp * kPerWarp + g * 128 + lane * 4;
      const uint64_t base = p0 + rel;
      if (base >= pend) break;
      while (k + 1 < cnt && s_end[k] <= rel) ++k;  // single-cell tiles (hot cells) skip the load
      uint32_t v[4];
      const uint32_t c = s_cell[k];
      if (s_end[k] >= rel + 4 || k + 1 == cnt) {  // the four positions share a cell
        v[0] = v[1] = v[2] = v[3] = c;
      } else {
        uint32_t kk = k;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          while (kk + 1 < cnt && s_end[kk] <= rel + e) ++kk;
          v[e] = s_cell[kk];
        }
      }
      out.put4(base, v, pend);
    }
  }
}

// ------------------------------------------------------------- report
// cells_traversed = sum over occupied leading-digit rows of
// (max suffix - min suffix + 1) (extraction.cpp:16-30; exact by SURVEY F4),
// read off the sorted output with two binary searches per row.
// `sorted` is either the sorted output (n keys) or, with n_from_occupied,
// the ascending list of occupied cells from the scan (the span sum depends
// only on the distinct keys), which also serves outputs that are not keys.
template <class K>
__global__ void k_report(const K* __restrict__ sorted, uint64_t n, uint32_t radix,
                         uint32_t total_digits, uint32_t frac_digits,
                         unsigned long long key_add, DevStats* st, bool n_from_occupied = false) {
  if (n_from_occupied) n = st->n_occupied;
  if (n == 0) {
    if (threadIdx.x == 0) {
      st->cells_traversed = 0;
      st->report_digits = total_digits ? total_digits : 1;
    }
    return;
  }
  const unsigned long long top = static_cast<unsigned long long>(sorted[n - 1]) + key_add;
  // total_digits == 0: decimal geometry from the max, lambda + frac
  // (sort.cpp:31-40 for integers, key_model.cpp:122-124 for decimals).
  const uint32_t digits =
      total_digits ? total_digits : d_digit_count(top / d_pow(10, frac_digits)) + frac_digits;
  const unsigned long long mod = d_pow(radix, digits - 1);
  // one warp per leading digit (row): the row's first and last keys by two
  // warp-cooperative searches (32 probes per round trip)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  auto lower_bound = [&](uint64_t a, uint64_t b, unsigned long long key) {  // first i in [a,b) with sorted[i] >= key
    while (b - a > 32) {
      const uint64_t step = (b - a) / 32;
      const uint64_t idx = a + (uint64_t)(lane + 1) * step;
      const bool ge = idx < b ? (unsigned long long)sorted[idx] + key_add >= key : true;
      const unsigned m = __ballot_sync(0xffffffffu, ge);
      if (m == 0) {
        a = a + 32 * step + 1;
      } else {
        const int f = __ffs(m) - 1;
        b = a + (uint64_t)(f + 1) * step;
        a = f > 0 ? a + (uint64_t)f * step + 1 : a;
      }
    }
    const uint64_t idx = a + lane;
    const bool ge = idx < b ? (unsigned long long)sorted[idx] + key_add >= key : true;
    const unsigned m = __ballot_sync(0xffffffffu, ge);
    return m ? a + (uint64_t)(__ffs(m) - 1) : b;
  };
  unsigned long long span = 0;
  for (uint32_t r = warp; r < radix; r += nwarps) {
    const unsigned long long lo_key = (unsigned long long)r * mod;
    const uint64_t a = lower_bound(0, n, lo_key);
    const uint64_t c = lower_bound(a, n, lo_key + mod);
    if (a < c && lane == 0) span += (unsigned long long)sorted[c - 1] - (unsigned long long)sorted[a] + 1;
  }
  __shared__ unsigned long long s_span[32];
  if (lane == 0) s_span[warp] = span;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long total = 0;
    for (int w = 0; w < nwarps; ++w) total += s_span[w];
    st->cells_traversed = total;
    st->report_digits = digits;
  }
}

// ------------------------------------------------- small inputs, one launch
// Grids of at most kSmemCellsMax cells and inputs of at most kSmallMax keys
// (cfg1: 2^20 keys, 10^3 cells) are launch-bound on the multi-pass path.
// Here count, scan, emit and report are ONE cooperative launch (every CTA
// resident): each CTA counts a slice into a shared grid and flushes it into
// the global grid, a grid-wide barrier, then every CTA scans the global grid
// in shared memory and writes its share of output positions (each thread
// four consecutive positions: one binary search, then a walk), and CTA 0
// computes the report (per-row spans, as k_report).  A key outside the grid
// or a flagged input skips the emit (the host redoes or raises).
constexpr uint64_t kSmallMax = 1ull << 22;
constexpr int kSmallThreads = 1024;
constexpr uint64_t kSmallSample = 1024;  // keys of the strided sample that sizes an undeclared grid (one per thread)

// With auto_cells (decimal integers without a declared width) the grid is
// derived in the same launch: a max phase, a first barrier, cells =
// 10^digits(max); a grid above the shared limit or the budget stops the
// launch (st->overflow = 2) and the host takes the multi-pass path with the
// max it now knows.
__device__ __forceinline__ void grid_barrier(uint32_t* ctr) {  // all CTAs resident (cooperative launch)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (*reinterpret_cast<volatile uint32_t*>(ctr) < gridDim.x) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

template <class Map, class Out>
__global__ void __launch_bounds__(kSmallThreads) k_small_sort(const typename Map::In* __restrict__ in, uint64_t n,
                                                              Map map, uint32_t cells, Out out,
                                                              uint32_t* gcount,  // [kSmemCellsMax + 2] zeroed
                                                              DevStats* st, uint32_t radix, uint32_t total_digits,
                                                              uint32_t frac_digits, bool auto_cells, uint64_t budget) {
  extern __shared__ uint32_t s_c[];  // [cells + 1]: counts, then exclusive offsets (s_c[cells] = n)
  __shared__ uint32_t s_scan[kSmallThreads / 32];
  __shared__ unsigned long long s_span[kSmallThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* bar = gcount + kSmemCellsMax;  // two barrier counters
  if (auto_cells) {
    // the grid from the max of a strided sample that every CTA reads alike
    // (no grid-wide max pass and barrier); the count below folds in the
    // true max, and a key past the sampled grid makes the host redo the
    // sort with it (st->overflow = 1, no emit)
    unsigned long long m = 0;
    unsigned fl = 0;
    const uint64_t ns = n < kSmallSample ? n : kSmallSample, step = n / ns;
    for (uint64_t j = threadIdx.x; j < ns; j += blockDim.x) {
      const unsigned long long k = map(__ldcg(in + j * step), fl);
      m = k > m ? k : m;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the last key too (sorted or nearly sorted inputs)
      const unsigned long long k = map(__ldcg(in + n - 1), fl);
      m = k > m ? k : m;
    }
    m = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(m >> 32)) == 0
            ? __reduce_max_sync(0xffffffffu, static_cast<unsigned>(m))
            : (static_cast<unsigned long long>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(m >> 32))) << 32) |
                  0xffffffffu;
    if (lane == 0) s_span[warp] = m;
    __syncthreads();
    unsigned long long smax = 0;
    for (int w = 0; w < kSmallThreads / 32; ++w) smax = s_span[w] > smax ? s_span[w] : smax;
    __syncthreads();
    const uint32_t d = d_digit_count(smax);
    const unsigned long long need = d_pow(10, d);
    if (need > kSmemCellsMax || need > budget) {
      // the grid does not qualify: the exact max (and flags) for the host's multi-pass path
      unsigned long long mm = 0;
      unsigned ff = fl;
      const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
      for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const unsigned long long k = map(__ldcs(in + i), ff);
        mm = k > mm ? k : mm;
      }
      warp_max_to(mm, &st->max_key);
      ff = warp_or(ff);
      if (lane == 0 && ff) atomicOr(&st->flags, ff);
      if (blockIdx.x == 0 && threadIdx.x == 0) st->overflow = 2;  // multi-pass path (or the budget error)
      return;
    }
    cells = static_cast<uint32_t>(need);
  }
  for (uint32_t c = threadIdx.x; c <= cells; c += blockDim.x) s_c[c] = 0;
  __syncthreads();
  unsigned long long mx = 0;
  unsigned flags = 0;
  bool ovf = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto count = [&](typename Map::In x) {
    const unsigned long long k = map(x, flags);
    mx = k > mx ? k : mx;
    if (k < cells) atomicAdd(&s_c[k], 1u);
    else ovf = true;
  };
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  using In = typename Map::In;
  if constexpr (sizeof(In) == 4 && !is_f64_map<Map>::value) {  // 16-byte vectors, all of a thread's loads in flight
    if ((reinterpret_cast<uintptr_t>(in) & 15) == 0) {
      const uint64_t nv = n / 4;
      const auto* v4 = reinterpret_cast<const uint4*>(in);
      for (uint64_t p = i; p < nv; p += 2 * stride) {
        const uint4 a = __ldcs(v4 + p);
        const bool two = p + stride < nv;
        const uint4 b = two ? __ldcs(v4 + p + stride) : make_uint4(0, 0, 0, 0);
        count(static_cast<In>(a.x)); count(static_cast<In>(a.y)); count(static_cast<In>(a.z)); count(static_cast<In>(a.w));
        if (two) {
          count(static_cast<In>(b.x)); count(static_cast<In>(b.y)); count(static_cast<In>(b.z)); count(static_cast<In>(b.w));
        }
      }
      i = nv * 4 + i;
    }
  }
  for (; i < n; i += stride) count(__ldcs(in + i));
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < cells; c += blockDim.x)
    if (s_c[c]) atomicAdd(&gcount[c], s_c[c]);
  warp_max_to(mx, &st->max_key);
  flags = warp_or(flags | (ovf ? 0x80000000u : 0u));
  if (lane == 0 && flags) {
    if (flags & 0x7fffffffu) atomicOr(&st->flags, flags & 0x7fffffffu);
    if (flags & 0x80000000u) atomicOr(&st->overflow, 1u);
  }
  grid_barrier(bar);
  if (*reinterpret_cast<volatile unsigned*>(&st->overflow) || *reinterpret_cast<volatile unsigned*>(&st->flags))
    return;
  // exclusive offsets of the global grid, in every CTA
  const uint32_t per = (cells + blockDim.x - 1) / blockDim.x, c0 = threadIdx.x * per;
  uint32_t sum = 0;
  for (uint32_t j = 0; j < per; ++j)
    if (c0 + j < cells) {
      const uint32_t v = __ldcg(gcount + c0 + j);
      s_c[c0 + j] = v;
      sum += v;
    }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_scan[warp] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
  {
    const uint32_t t = s_scan[lane];
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    run += __shfl_sync(0xffffffffu, ti - t, warp);
  }
  for (uint32_t j = 0; j < per; ++j)
    if (c0 + j < cells) {
      const uint32_t v = s_c[c0 + j];
      s_c[c0 + j] = run;
      run += v;
    }
  if (threadIdx.x == blockDim.x - 1) s_c[cells] = run;
  __syncthreads();
  // emit: this CTA's share of positions, four per thread
  const uint64_t share = ((n + gridDim.x - 1) / gridDim.x + 3) & ~3ull;
  const uint64_t p0 = (uint64_t)blockIdx.x * share, p1 = p0 + share < n ? p0 + share : n;
  for (uint64_t p = p0 + 4ull * threadIdx.x; p < p1; p += 4ull * blockDim.x) {
    uint32_t lo = 0, hi = cells;  // the last cell whose offset is <= p (it is occupied)
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_c[mid] <= p) lo = mid;
      else hi = mid;
    }
    uint32_t cv[4];
    uint32_t cell = lo;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      while (cell + 1 < cells && s_c[cell + 1] <= p + e) ++cell;
      cv[e] = cell;
    }
    out.put4(p, cv, p1);
  }
  if (blockIdx.x != 0) return;
  // report (k_report's definition): per occupied leading-digit row, max - min + 1
  const unsigned long long top = *reinterpret_cast<volatile unsigned long long*>(&st->max_key);
  const uint32_t digits = total_digits ? total_digits : d_digit_count(top / d_pow(10, frac_digits)) + frac_digits;
  const unsigned long long mod = d_pow(radix, digits - 1);
  unsigned long long span = 0;
  for (uint32_t r = warp; r < radix && (unsigned long long)r * mod < cells; r += blockDim.x / 32) {
    const uint32_t a = static_cast<uint32_t>(r * mod);
    const uint32_t b = (unsigned long long)(r + 1) * mod < cells ? static_cast<uint32_t>((r + 1) * mod) : cells;
    uint32_t first = 0xffffffffu, last = 0;
    for (uint32_t c = a + lane; c < b; c += 32)
      if (s_c[c + 1] > s_c[c]) {
        first = c < first ? c : first;
        last = c;
      }
    first = __reduce_min_sync(0xffffffffu, first);
    last = __reduce_max_sync(0xffffffffu, last);
    if (first != 0xffffffffu) span += last - first + 1;
  }
  if (lane == 0) s_span[warp] = span;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long total = 0;
    for (int w = 0; w < kSmallThreads / 32; ++w) total += s_span[w];
    st->cells_traversed = total;
    st->report_digits = digits;
  }
}

}  // namespace rsb

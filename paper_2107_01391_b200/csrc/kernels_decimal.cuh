// kernels_decimal.cuh — decimal text on the GPU: the
// ingest side of sort_decimals (parse_decimal + normalize_dataset,
// key_model.cpp:80-133) and its render side (format_scaled_decimal,
// key_model.cpp:170-180), over an Arrow-style string column (bytes +
// n+1 offsets).
//
//   k_dec_parse   one thread per numeral: the reference grammar (digits,
//                 optional '.', digits; no sign, no exponent), mantissa with
//                 the reference's overflow rule, scale = fractional digits;
//                 dataset max scale / max integer part by atomics; the first
//                 failing numeral (lowest index, i.e. the one the reference's
//                 sequential loop stops at) by an atomicMin of (index, code)
//   k_dec_scale   key = mantissa * 10^(dataset scale - own scale)
//   k_dec_offsets rendered length per key, scanned into the output offsets
//   k_dec_format_staged  digits right to left into shared memory, the CTA's
//                 contiguous output range written with 16-byte stores
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rs_internal.cuh"

namespace rsb {

// Per-numeral outcome, in the order the reference checks (key_model.cpp:81-104
// then DecimalValue::integer_part, key_model.cpp:60-62, in normalize_dataset).
enum : uint32_t {
  kDecOk = 0,
  kDecEmpty = 1,          // parse_error "empty numeral"
  kDecNegative = 2,       // negative_value
  kDecMultiDot = 3,       // parse_error "multiple decimal points"
  kDecNoFrac = 4,         // parse_error "no digits after decimal point"
  kDecNoDigits = 5,       // parse_error "no digits"
  kDecBadChar = 6,        // parse_error "invalid character"
  kDecTooLong = 7,        // cell_budget_exceeded: mantissa overflows 64 bits
  kDecScaleOverflow = 8,  // cell_budget_exceeded: 10^scale overflows 64 bits (integer_part)
};

__device__ __constant__ unsigned long long c_pow10[20] = {
    1ull, 10ull, 100ull, 1000ull, 10000ull, 100000ull, 1000000ull, 10000000ull, 100000000ull, 1000000000ull,
    10000000000ull, 100000000000ull, 1000000000000ull, 10000000000000ull, 100000000000000ull,
    1000000000000000ull, 10000000000000000ull, 100000000000000000ull, 1000000000000000000ull,
    10000000000000000000ull};

struct DecStats {
  unsigned long long first_error;  // (index << 8) | code, ~0 if none
  unsigned long long max_integer;
  unsigned int max_scale;
  unsigned int pad;
};

__global__ void __launch_bounds__(kThreads) k_dec_parse(const char* __restrict__ chars,
                                                        const unsigned long long* __restrict__ offsets, uint64_t n,
                                                        unsigned long long* __restrict__ mant,
                                                        uint8_t* __restrict__ scale_out, DecStats* ds,
                                                        uint32_t* __restrict__ scale_u32 = nullptr) {
  // scale_u32 != nullptr: parse_decimal alone (rs_parse_decimals) — own scales
  // as uint32, and no integer_part check (normalize_dataset's, 10^scale)
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const auto* bytes = reinterpret_cast<const unsigned char*>(chars);
  unsigned long long mx_int = 0;
  uint32_t mx_scale = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long b = offsets[i];
    const uint32_t len = static_cast<uint32_t>(offsets[i + 1] - b);
    const unsigned char* s = bytes + b;
    // one sweep: digits counted and accumulated (wrapping), the first dot
    // (integer part = the value before it), a second dot, other bytes
    uint32_t dot = 0xffffffffu, ndig = 0;
    bool second_dot = false, bad = false;
    unsigned long long m = 0, ip = 0;
    for (uint32_t j = 0; j < len; ++j) {
      const uint32_t c = __ldg(s + j);
      const uint32_t d = c - '0';
      if (d < 10) {
        m = m * 10 + d;
        ++ndig;
      } else if (c == '.') {
        second_dot |= dot != 0xffffffffu;
        if (dot == 0xffffffffu) {
          dot = j;
          ip = m;
        }
      } else {
        bad = true;
      }
    }
    if (dot == 0xffffffffu) ip = m;
    // < 20 digits never overflow 64 bits; otherwise accumulate_digits' exact
    // rule (key_model.cpp:22-34), digit by digit
    bool overflow = false;
    if (ndig >= 20 && !bad) {
      unsigned long long acc = 0, acc_ip = 0;
      for (uint32_t j = 0; j < len && !overflow; ++j) {
        const uint32_t d = __ldg(s + j) - '0';
        if (d >= 10) continue;
        if (acc > (~0ull - d) / 10) overflow = true;
        else acc = acc * 10 + d;
        if (dot == 0xffffffffu || j < dot) acc_ip = acc;
      }
      m = acc;
      ip = acc_ip;
    }
    uint32_t code = kDecOk, frac = 0;
    if (len == 0) {
      code = kDecEmpty;
    } else if (s[0] == '-') {
      code = kDecNegative;
    } else {
      const uint32_t ilen = dot != 0xffffffffu ? dot : len;
      const uint32_t flen = dot != 0xffffffffu ? len - ilen - 1 : 0;
      if (second_dot) code = kDecMultiDot;
      else if (dot != 0xffffffffu && flen == 0) code = kDecNoFrac;
      else if (ilen == 0 && flen == 0) code = kDecNoDigits;
      else if (bad) code = kDecBadChar;
      else if (overflow) code = kDecTooLong;
      else if (flen > 19 && !scale_u32) code = kDecScaleOverflow;
      frac = flen;
    }
    if (code != kDecOk) {
      atomicMin(&ds->first_error, (static_cast<unsigned long long>(i) << 8) | code);
      m = 0;
      ip = 0;
      frac = 0;
    }
    mant[i] = m;
    if (scale_u32) scale_u32[i] = frac;
    else scale_out[i] = static_cast<uint8_t>(frac);
    mx_int = ip > mx_int ? ip : mx_int;
    mx_scale = frac > mx_scale ? frac : mx_scale;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mx_int, o);
    const uint32_t bb = __shfl_xor_sync(0xffffffffu, mx_scale, o);
    mx_int = a > mx_int ? a : mx_int;
    mx_scale = bb > mx_scale ? bb : mx_scale;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mx_int) atomicMax(&ds->max_integer, mx_int);
    if (mx_scale) atomicMax(&ds->max_scale, mx_scale);
  }
}

// keys[i] = mant[i] * 10^(scale - own scale) (in place)
__global__ void __launch_bounds__(kThreads) k_dec_scale(unsigned long long* __restrict__ mant,
                                                        const uint8_t* __restrict__ own, uint64_t n, uint32_t scale) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    mant[i] *= c_pow10[scale - own[i]];
}

__device__ __forceinline__ uint32_t dec_digits(unsigned long long v) {
  if (v == 0) return 1;
  const uint32_t t = (static_cast<uint32_t>(64 - __clzll(static_cast<long long>(v))) * 1233u) >> 12;  // ~log10(2^bits)
  return t + (v >= c_pow10[t] ? 1u : 0u);
}

// to_string(mantissa / p) [ '.' zero-padded(mantissa % p, scale) ] (format_scaled_decimal,
// key_model.cpp:170-180), staged: a CTA formats 256 consecutive keys into shared
// memory (their output bytes are one contiguous range of the column) and
// writes the range out with 16-byte stores — the per-byte global stores of
// k_dec_format become one vector store per 16 bytes.  The staging keeps the
// range's alignment (its start sits at `lead` = start mod 16).
constexpr int kDecFmtKeys = 256;
constexpr int kDecFmtMaxBytes = 41;  // 20 integer digits + '.' + 19 fractional digits (+1 slack)
__global__ void __launch_bounds__(kDecFmtKeys) k_dec_format_staged(const unsigned long long* __restrict__ keys,
                                                                   uint64_t n, uint32_t scale,
                                                                   const unsigned long long* __restrict__ offsets,
                                                                   char* __restrict__ out) {
  __shared__ __align__(16) char s_buf[kDecFmtKeys * kDecFmtMaxBytes + 32];
  for (uint64_t i0 = (uint64_t)blockIdx.x * kDecFmtKeys; i0 < n; i0 += (uint64_t)gridDim.x * kDecFmtKeys) {
    const uint64_t i1 = i0 + kDecFmtKeys < n ? i0 + kDecFmtKeys : n;
    const unsigned long long gbase = offsets[i0], gend = offsets[i1];
    const uint32_t lead = static_cast<uint32_t>(gbase & 15u);
    const uint64_t i = i0 + threadIdx.x;
    if (i < i1) {
      unsigned long long v = keys[i];
      char* end = s_buf + lead + (offsets[i + 1] - gbase);
      uint32_t j = 0;
      auto emit = [&](uint32_t dg) {
        if (scale != 0 && j == scale) *--end = '.';
        *--end = static_cast<char>('0' + dg);
        ++j;
      };
      while (v >> 32) {
        emit(static_cast<uint32_t>(v % 10));
        v /= 10;
      }
      uint32_t x = static_cast<uint32_t>(v);
      do {
        emit(x % 10);
        x /= 10;
      } while (x != 0 || j <= scale);
    }
    __syncthreads();
    const unsigned long long a16 = (gbase + 15) & ~15ull, e16 = gend & ~15ull;
    if (a16 >= e16) {  // short range: bytes
      for (unsigned long long p = gbase + threadIdx.x; p < gend; p += blockDim.x) out[p] = s_buf[lead + (p - gbase)];
    } else {
      for (unsigned long long p = gbase + threadIdx.x; p < a16; p += blockDim.x) out[p] = s_buf[lead + (p - gbase)];
      for (unsigned long long p = a16 + 16ull * threadIdx.x; p < e16; p += 16ull * blockDim.x)
        *reinterpret_cast<uint4*>(out + p) = *reinterpret_cast<const uint4*>(s_buf + lead + (p - gbase));
      for (unsigned long long p = e16 + threadIdx.x; p < gend; p += blockDim.x) out[p] = s_buf[lead + (p - gbase)];
    }
    __syncthreads();
  }
}

// Offsets of the rendered column: exclusive scan of the rendered lengths of
// format_scaled_decimal(key, scale) — the integer part key / 10^scale has
// max(1, digits(key) - scale) digits, so no division — computed while the
// keys stream in (striped, coalesced); out[n] = total.  Look-back over tiles
// of 4096 keys.
__global__ void __launch_bounds__(kThreads) k_dec_offsets(const unsigned long long* __restrict__ keys, uint64_t n,
                                                          uint32_t scale, unsigned long long* __restrict__ out,
                                                          unsigned long long* desc, unsigned* tile_counter,
                                                          uint32_t num_tiles) {
  __shared__ uint32_t s_len[kScanTile + kScanTile / 32];  // index r at r + r/32: both access orders conflict-free
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_w[kThreads / 32];
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t t0 = (uint64_t)tile * kScanTile;
  const uint32_t extra = scale ? 1 + scale : 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {  // striped: consecutive lanes, consecutive keys
    const uint32_t r = k * kThreads + threadIdx.x;
    uint32_t l = 0;
    if (t0 + r < n) {
      const uint32_t d = dec_digits(keys[t0 + r]);
      l = (d > scale ? d - scale : 1u) + extra;
    }
    s_len[r + (r >> 5)] = l;
  }
  __syncthreads();
  uint32_t v[kScanPerThread], sum = 0;  // blocked: thread t owns entries 16t .. 16t+15
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const uint32_t r = threadIdx.x * kScanPerThread + k;
    v[k] = s_len[r + (r >> 5)];
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
      if (tile == num_tiles - 1) out[n] = p + r;
    }
  }
  __syncthreads();
  // exclusive tile-relative offsets back into shared memory, then striped stores
  uint32_t run = static_cast<uint32_t>(before + inc - sum);
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const uint32_t r = threadIdx.x * kScanPerThread + k;
    s_len[r + (r >> 5)] = run;
    run += v[k];
  }
  __syncthreads();
  const unsigned long long base = s_prefix;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const uint32_t rr = k * kThreads + threadIdx.x;
    if (t0 + rr < n) out[t0 + rr] = base + s_len[rr + (rr >> 5)];
  }
}

}  // namespace rsb

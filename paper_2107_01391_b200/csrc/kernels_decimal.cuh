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
//   k_dec_len     rendered length per key; exclusive scan -> offsets
//   k_dec_format  digits written right to left into the output column
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
                                                        uint8_t* __restrict__ scale_out, DecStats* ds) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long mx_int = 0;
  uint32_t mx_scale = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long b = offsets[i], e = offsets[i + 1];
    const uint64_t len = e - b;
    const char* s = chars + b;
    uint32_t code = kDecOk;
    unsigned long long m = 0;
    uint32_t frac = 0;
    if (len == 0) {
      code = kDecEmpty;
    } else if (s[0] == '-') {
      code = kDecNegative;
    } else {
      // one sweep: the dot position, a second dot, non-digits, the mantissa
      int64_t dot = -1;
      bool second_dot = false, bad = false, overflow = false;
      for (uint64_t j = 0; j < len; ++j) {
        const unsigned c = static_cast<unsigned char>(s[j]);
        if (c == '.') {
          if (dot >= 0) second_dot = true;
          else dot = static_cast<int64_t>(j);
          continue;
        }
        if (c < '0' || c > '9') {
          bad = true;
          continue;
        }
        const unsigned long long d = c - '0';
        if (m > (~0ull - d) / 10) overflow = true;  // accumulate_digits (key_model.cpp:22-34)
        else if (!overflow) m = m * 10 + d;
      }
      const uint64_t ilen = dot >= 0 ? static_cast<uint64_t>(dot) : len;
      const uint64_t flen = dot >= 0 ? len - ilen - 1 : 0;
      if (second_dot) code = kDecMultiDot;
      else if (dot >= 0 && flen == 0) code = kDecNoFrac;
      else if (ilen == 0 && flen == 0) code = kDecNoDigits;
      else if (bad) code = kDecBadChar;
      else if (overflow) code = kDecTooLong;
      else if (flen > 19) code = kDecScaleOverflow;
      frac = static_cast<uint32_t>(flen);
    }
    if (code != kDecOk) {
      atomicMin(&ds->first_error, (static_cast<unsigned long long>(i) << 8) | code);
      m = 0;
      frac = 0;
    }
    mant[i] = m;
    scale_out[i] = static_cast<uint8_t>(frac);
    const unsigned long long ip = m / c_pow10[frac];
    mx_int = ip > mx_int ? ip : mx_int;
    mx_scale = frac > mx_scale ? frac : mx_scale;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mx_int, o);
    const uint32_t b = __shfl_xor_sync(0xffffffffu, mx_scale, o);
    mx_int = a > mx_int ? a : mx_int;
    mx_scale = b > mx_scale ? b : mx_scale;
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
  uint32_t d = 1;
  while (d < 20 && v >= c_pow10[d]) ++d;
  return d;
}

// rendered length of format_scaled_decimal(key, scale)
__global__ void __launch_bounds__(kThreads) k_dec_len(const unsigned long long* __restrict__ keys, uint64_t n,
                                                      uint32_t scale, unsigned long long* __restrict__ len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    len[i] = dec_digits(keys[i] / c_pow10[scale]) + (scale ? 1 + scale : 0);
}

// to_string(mantissa / p) [ '.' zero-padded(mantissa % p, scale) ]
__global__ void __launch_bounds__(kThreads) k_dec_format(const unsigned long long* __restrict__ keys, uint64_t n,
                                                         uint32_t scale,
                                                         const unsigned long long* __restrict__ offsets,
                                                         char* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned long long v = keys[i];
    char* end = out + offsets[i + 1];
    for (uint32_t j = 0; j < scale; ++j) {  // fractional digits, right to left
      *--end = static_cast<char>('0' + v % 10);
      v /= 10;
    }
    if (scale) *--end = '.';
    do {
      *--end = static_cast<char>('0' + v % 10);
      v /= 10;
    } while (v);
  }
}

// Exclusive scan of n uint64 values (look-back), out[n] = total.
__global__ void __launch_bounds__(kThreads) k_exscan_u64(const unsigned long long* __restrict__ in, uint64_t count,
                                                         unsigned long long* __restrict__ out,
                                                         unsigned long long* desc, unsigned* tile_counter,
                                                         uint32_t num_tiles) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_w[kThreads / 32];
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t i0 = (uint64_t)tile * kScanTile + threadIdx.x * kScanPerThread;
  unsigned long long v[kScanPerThread], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    v[k] = (i0 + k < count) ? in[i0 + k] : 0ull;
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
      if (tile == num_tiles - 1) out[count] = p + r;
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + before + inc - sum;
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (i0 + k < count) out[i0 + k] = run;
    run += v[k];
  }
}

}  // namespace rsb

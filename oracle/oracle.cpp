// oracle.cpp — CPU restatement of the Recombinant Sort reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  Each function restates the
// reference function cited beside it; it is checked against the reference's
// golden vectors and against the reference library itself (oracle/_ref) in
// tests/test_oracle.py.  Single-threaded, like the reference.
#include "oracle.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string_view>
#include <vector>

namespace {

constexpr uint64_t kMaxU64 = ~uint64_t{0};
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline uint64_t mix_out(uint64_t z) {  // splitmix64.hpp:17-19
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// parse_decimal restricted to what std::to_chars(fixed) emits
// (key_model.cpp:80-105, accumulate_digits 22-34).
int parse_fixed(std::string_view text, uint64_t* mantissa, uint32_t* scale) {
  const size_t dot = text.find('.');
  std::string_view ip = text.substr(0, dot);
  std::string_view fp = dot == std::string_view::npos ? std::string_view{}
                                                      : text.substr(dot + 1);
  uint64_t acc = 0;
  for (std::string_view part : {ip, fp}) {
    for (char c : part) {
      const uint64_t d = static_cast<uint64_t>(c - '0');
      if (acc > (kMaxU64 - d) / 10) return OR_CELL_BUDGET_EXCEEDED;
      acc = acc * 10 + d;
    }
  }
  *mantissa = acc;
  *scale = static_cast<uint32_t>(fp.size());
  return OR_OK;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- SplitMix64
uint64_t or_sm64_next(uint64_t* state) {  // splitmix64.hpp:14-19
  *state += kGolden;
  return mix_out(*state);
}

double or_sm64_next_unit(uint64_t* state) {  // splitmix64.hpp:22-24
  return static_cast<double>(or_sm64_next(state) >> 11) * 0x1.0p-53;
}

uint64_t or_sm64_mix(uint64_t seed, uint64_t index) {  // splitmix64.hpp:32-35
  uint64_t s = seed + index;
  return or_sm64_next(&s);
}

uint64_t or_sm64_at(uint64_t seed, uint64_t i) {
  return mix_out(seed + (i + 1) * kGolden);
}

// ----------------------------------------------------------------- key model
uint32_t or_decimal_digit_count(uint64_t v) {  // key_model.cpp:51-58
  uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

int or_checked_pow(uint64_t radix, uint32_t exp, uint64_t* out) {  // :38-49
  uint64_t r = 1;
  for (uint32_t i = 0; i < exp; ++i) {
    if (r > kMaxU64 / radix) return OR_CELL_BUDGET_EXCEEDED;
    r *= radix;
  }
  *out = r;
  return OR_OK;
}

int or_make_key_spec(uint32_t radix, uint32_t total, uint32_t integer,
                     uint64_t max_cells, or_key_spec* out) {  // :64-78
  if (radix < 2 || total < 1 || integer > total) return OR_INVALID_ARGUMENT;
  uint64_t cells = 0;
  if (int st = or_checked_pow(radix, total, &cells)) return st;
  if (cells > max_cells) return OR_CELL_BUDGET_EXCEEDED;
  *out = or_key_spec{radix, total, integer};
  return OR_OK;
}

int or_float_to_decimal(double x, uint32_t scale, uint64_t* mantissa) {
  // key_model.cpp:135-158
  if (std::isnan(x) || std::isinf(x)) return OR_NON_FINITE;
  if (x < 0.0) return OR_NEGATIVE_VALUE;
  if (std::signbit(x)) x = 0.0;
  char buf[512];
  const auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::fixed);
  if (res.ec != std::errc{}) return OR_NON_FINITE;
  uint64_t m = 0;
  uint32_t s = 0;
  if (int st = parse_fixed({buf, static_cast<size_t>(res.ptr - buf)}, &m, &s)) return st;
  if (s <= scale) {
    uint64_t p = 0;
    if (int st = or_checked_pow(10, scale - s, &p)) return st;
    *mantissa = m * p;  // the reference multiplies unchecked (key_model.cpp:152)
    return OR_OK;
  }
  uint64_t divisor = 0;
  if (int st = or_checked_pow(10, s - scale, &divisor)) return st;
  uint64_t q = m / divisor;
  if (m % divisor >= divisor / 2) ++q;  // half rounds up
  *mantissa = q;
  return OR_OK;
}

// -------------------------------------------- hashing + extraction cycles
int or_sort_keys(const uint64_t* keys, uint64_t n, or_key_spec spec,
                 uint64_t max_cells, uint64_t* out, uint64_t out_capacity,
                 or_report* report) {
  uint64_t cells = 0, mod = 0;
  if (int st = or_checked_pow(spec.radix, spec.total_digits, &cells)) return st;
  if (cells > max_cells) return OR_CELL_BUDGET_EXCEEDED;  // hashing.cpp:19-23
  if (int st = or_checked_pow(spec.radix, spec.total_digits - 1, &mod)) return st;
  // CountSpace (hashing.hpp:55-58) + TraverseMaps (hashing.hpp:21-48)
  std::vector<uint64_t> counts;
  try {
    counts.assign(cells, 0);
  } catch (...) {
    return OR_ALLOC_FAILED;
  }
  std::vector<uint8_t> occupied(spec.radix, 0);
  std::vector<uint64_t> h_min(spec.radix, 0);
  std::vector<int64_t> h_max(spec.radix, -1);
  for (uint64_t i = 0; i < n; ++i) {  // build_count_space, hashing.cpp:40-52
    const uint64_t key = keys[i];
    if (key >= cells) return OR_SPEC_MISMATCH;  // hash_insert :31-34
    ++counts[key];
    const uint32_t row = static_cast<uint32_t>(key / mod);
    const uint64_t suffix = key % mod;
    if (!occupied[row]) {
      occupied[row] = 1;
      h_min[row] = suffix;
    } else if (suffix < h_min[row]) {
      h_min[row] = suffix;
    }
    if (static_cast<int64_t>(suffix) > h_max[row]) h_max[row] = static_cast<int64_t>(suffix);
  }
  if (out_capacity < n) return OR_BUFFER_TOO_SMALL;  // extraction.cpp:8-12
  uint64_t written = 0, traversed = 0;
  for (uint32_t row = 0; row < spec.radix && written < n; ++row) {  // :16-31
    if (!occupied[row]) continue;
    const uint64_t hi = static_cast<uint64_t>(h_max[row]);
    const uint64_t base = static_cast<uint64_t>(row) * mod;
    for (uint64_t suffix = h_min[row]; suffix <= hi; ++suffix) {
      ++traversed;
      const uint64_t key = base + suffix;
      for (uint64_t c = counts[key]; c > 0; --c) out[written++] = key;
      if (written == n) break;
    }
  }
  if (report) *report = or_report{written, traversed, spec};
  return OR_OK;
}

// ------------------------------------------------------------------ facades
int or_sort_integers_i64(const int64_t* values, uint64_t n, uint64_t max_cells,
                         int64_t* out, or_report* report) {  // sort.cpp:29-59
  uint64_t max_value = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (values[i] < 0) return OR_NEGATIVE_VALUE;
    max_value = std::max<uint64_t>(max_value, static_cast<uint64_t>(values[i]));
  }
  const uint32_t d = or_decimal_digit_count(max_value);
  or_key_spec spec{};
  if (int st = or_make_key_spec(10, d, d, max_cells, &spec)) return st;
  std::vector<uint64_t> keys(values, values + n), sorted(n);
  if (int st = or_sort_keys(keys.data(), n, spec, max_cells, sorted.data(), n, report)) return st;
  for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<int64_t>(sorted[i]);
  return OR_OK;
}

int or_sort_integers_u32(const uint32_t* values, uint64_t n, uint64_t max_cells,
                         uint32_t* out, or_report* report) {
  uint64_t max_value = 0;
  for (uint64_t i = 0; i < n; ++i) max_value = std::max<uint64_t>(max_value, values[i]);
  const uint32_t d = or_decimal_digit_count(max_value);
  or_key_spec spec{};
  if (int st = or_make_key_spec(10, d, d, max_cells, &spec)) return st;
  std::vector<uint64_t> keys(values, values + n), sorted(n);
  if (int st = or_sort_keys(keys.data(), n, spec, max_cells, sorted.data(), n, report)) return st;
  for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(sorted[i]);
  return OR_OK;
}

int or_sort_f64(const double* x, uint64_t n, uint32_t scale, uint64_t max_cells,
                uint64_t* out, or_report* report) {
  std::vector<uint64_t> keys(n);
  uint64_t max_m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (int st = or_float_to_decimal(x[i], scale, &keys[i])) return st;
    max_m = std::max(max_m, keys[i]);
  }
  uint64_t p = 0;
  if (int st = or_checked_pow(10, scale, &p)) return st;
  const uint32_t lambda = or_decimal_digit_count(max_m / p);  // key_model.cpp:122
  or_key_spec spec{};
  if (int st = or_make_key_spec(10, lambda + scale, lambda, max_cells, &spec)) return st;
  return or_sort_keys(keys.data(), n, spec, max_cells, out, n, report);
}

static int alphabet_table(const char* alphabet, uint16_t* ord, uint32_t* radix) {
  // Alphabet ctor, key_model.cpp:190-201
  const size_t len = std::strlen(alphabet);
  if (len == 0 || len > 0xFFFE) return OR_INVALID_ARGUMENT;
  std::memset(ord, 0, 256 * sizeof(uint16_t));
  for (size_t i = 0; i < len; ++i) {
    const auto c = static_cast<unsigned char>(alphabet[i]);
    if (ord[c] != 0) return OR_INVALID_ARGUMENT;
    ord[c] = static_cast<uint16_t>(i + 1);
  }
  *radix = static_cast<uint32_t>(len) + 1;
  return OR_OK;
}

static inline uint32_t rec_len(const uint8_t* rec, uint32_t width) {
  uint32_t l = 0;
  while (l < width && rec[l] != 0) ++l;
  return l;
}

int or_strings_to_keys(const uint8_t* chars, uint64_t n, uint32_t width,
                       const char* alphabet, uint64_t max_cells, uint64_t* keys,
                       or_key_spec* spec_out) {  // key_model.cpp:225-247
  uint16_t ord[256];
  uint32_t radix = 0;
  if (int st = alphabet_table(alphabet, ord, &radix)) return st;
  uint32_t w = 1;
  for (uint64_t i = 0; i < n; ++i) w = std::max(w, rec_len(chars + i * width, width));
  or_key_spec spec{};
  if (int st = or_make_key_spec(radix, w, w, max_cells, &spec)) return st;
  for (uint64_t i = 0; i < n; ++i) {
    const uint8_t* rec = chars + i * width;
    const uint32_t l = rec_len(rec, width);
    uint64_t key = 0;
    for (uint32_t j = 0; j < w; ++j) {
      uint32_t o = 0;
      if (j < l) {
        o = ord[rec[j]];
        if (o == 0) return OR_SYMBOL_OUT_OF_ALPHABET;
      }
      key = key * radix + o;
    }
    keys[i] = key;
  }
  if (spec_out) *spec_out = spec;
  return OR_OK;
}

int or_sort_fixed_strings(const uint8_t* chars, uint64_t n, uint32_t width,
                          const char* alphabet, uint8_t* out, or_report* report) {
  uint16_t ord[256];
  uint32_t radix = 0;
  if (int st = alphabet_table(alphabet, ord, &radix)) return st;
  uint32_t w = 1;
  for (uint64_t i = 0; i < n; ++i) {
    const uint8_t* rec = chars + i * width;
    const uint32_t l = rec_len(rec, width);
    for (uint32_t j = 0; j < l; ++j)
      if (ord[rec[j]] == 0) return OR_SYMBOL_OUT_OF_ALPHABET;
    w = std::max(w, l);
  }
  // oracle_sort<std::string> (baselines.hpp:56-60): byte-lexicographic order.
  std::vector<uint64_t> idx(n);
  for (uint64_t i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
    return std::memcmp(chars + a * width, chars + b * width, width) < 0;
  });
  for (uint64_t i = 0; i < n; ++i) std::memcpy(out + i * width, chars + idx[i] * width, width);
  if (report) {
    // Single-grid report with an unlimited budget: per-row spans over the
    // base-radix keys of the sorted records (extraction.cpp:16-30, F4).
    uint64_t dummy = 0;
    if (int st = or_checked_pow(radix, w, &dummy)) return st;
    std::vector<uint64_t> keys(n);
    for (uint64_t i = 0; i < n; ++i) {
      const uint8_t* rec = out + i * width;
      const uint32_t l = rec_len(rec, width);
      uint64_t key = 0;
      for (uint32_t j = 0; j < w; ++j) key = key * radix + (j < l ? ord[rec[j]] : 0);
      keys[i] = key;
    }
    if (int st = or_report_from_sorted(keys.data(), n, radix, w, report)) return st;
  }
  return OR_OK;
}

// ------------------------------------------------------- stable key/value
int or_radix_sort_lsd_kv_u32(const uint32_t* keys, const uint32_t* vals, uint64_t n,
                             uint32_t* keys_out, uint32_t* vals_out) {
  // radix_sort_lsd_by (baselines.hpp:24-46) over (key, value) records.
  std::vector<uint64_t> items(n), scratch(n);
  for (uint64_t i = 0; i < n; ++i) items[i] = (static_cast<uint64_t>(keys[i]) << 32) | vals[i];
  if (n >= 2) {
    uint64_t max_key = 0;
    for (uint64_t i = 0; i < n; ++i) max_key = std::max<uint64_t>(max_key, keys[i]);
    const uint32_t passes = or_decimal_digit_count(max_key);
    uint64_t place = 1;
    for (uint32_t pass = 0; pass < passes; ++pass) {
      uint64_t counts[10] = {};
      for (uint64_t it : items) ++counts[((it >> 32) / place) % 10];
      uint64_t offsets[10], running = 0;
      for (int d = 0; d < 10; ++d) {
        offsets[d] = running;
        running += counts[d];
      }
      for (uint64_t it : items) scratch[offsets[((it >> 32) / place) % 10]++] = it;
      items.swap(scratch);
      if (pass + 1 < passes) place *= 10;
    }
  }
  for (uint64_t i = 0; i < n; ++i) {
    keys_out[i] = static_cast<uint32_t>(items[i] >> 32);
    vals_out[i] = static_cast<uint32_t>(items[i]);
  }
  return OR_OK;
}

int or_report_from_sorted(const uint64_t* sorted, uint64_t n, uint32_t radix,
                          uint32_t total_digits, or_report* report) {
  uint64_t mod = 0;
  if (int st = or_checked_pow(radix, total_digits - 1, &mod)) return st;
  uint64_t traversed = 0;
  uint64_t i = 0;
  while (i < n) {  // one occupied row at a time: span = last - first + 1
    const uint64_t row = sorted[i] / mod;
    uint64_t j = i;
    while (j + 1 < n && sorted[j + 1] / mod == row) ++j;
    traversed += (sorted[j] % mod) - (sorted[i] % mod) + 1;
    i = j + 1;
  }
  *report = or_report{n, traversed, or_key_spec{radix, total_digits, total_digits}};
  return OR_OK;
}

// --------------------------------------------------------------- generators
uint64_t or_config_seed(uint32_t cfg) {  // bench.cpp:149 pattern, base seed 42
  return or_sm64_mix(42, cfg);
}

void or_gen_u32_mod(uint64_t seed, uint64_t first, uint64_t n, uint64_t bound,
                    uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t x = or_sm64_at(seed, first + i);
    out[i] = bound ? static_cast<uint32_t>(x % bound) : static_cast<uint32_t>(x >> 32);
  }
}

int or_zipf_cdf(uint32_t ranks, double s, double* cdf) {
  double total = 0.0;
  for (uint32_t r = 1; r <= ranks; ++r) {
    total += std::pow(static_cast<double>(r), -s);
    cdf[r - 1] = total;
  }
  for (uint32_t r = 0; r < ranks; ++r) cdf[r] /= total;
  cdf[ranks - 1] = 1.0;
  return OR_OK;
}

void or_gen_f64_cfg3(uint64_t seed, uint64_t first, uint64_t n, const double* cdf,
                     uint32_t ranks, double* out) {
  // even elements: k uniform in [0, ranks); odd elements: k = Zipf rank - 1
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t g = first + i;
    const uint64_t x = or_sm64_at(seed, g);
    uint64_t k;
    if ((g & 1) == 0) {
      k = x % ranks;
    } else {
      const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
      k = static_cast<uint64_t>(std::upper_bound(cdf, cdf + ranks, u) - cdf);
      if (k >= ranks) k = ranks - 1;
    }
    out[i] = static_cast<double>(k) / 1000.0;
  }
}

void or_gen_str_cfg4(uint64_t seed, uint64_t first, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < 8; ++j)
      out[i * 8 + j] = static_cast<uint8_t>('a' + or_sm64_at(seed, (first + i) * 8 + j) % 26);
}

}  // extern "C"

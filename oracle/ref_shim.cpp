// ref_shim.cpp — extern "C" wrappers over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/librecsort_ref.so.  Nothing here re-implements the algorithm:
// each wrapper calls the reference's own public API and maps recsort::Error
// to (errc + 1) so tests can compare statuses with rs_status.
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "recsort/baselines.hpp"
#include "recsort/error.hpp"
#include "recsort/extraction.hpp"
#include "recsort/hashing.hpp"
#include "recsort/key_model.hpp"
#include "recsort/bench.hpp"
#include "recsort/sort.hpp"
#include "recsort/splitmix64.hpp"

using namespace recsort;

struct ref_report {
  uint64_t written, cells_traversed;
  uint32_t radix, total_digits, integer_digits;
};

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_msg = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::bad_alloc&) {
    g_msg = "allocation failed";
    return 99;
  }
}

void fill(ref_report* r, const ExtractionReport& rep, const KeySpec& spec) {
  if (!r) return;
  *r = ref_report{rep.written, rep.cells_traversed, spec.radix, spec.total_digits,
                  spec.integer_digits};
}

std::vector<std::string> records(const uint8_t* chars, uint64_t n, uint32_t width) {
  std::vector<std::string> v;
  v.reserve(n);
  for (uint64_t i = 0; i < n; ++i) {
    const char* rec = reinterpret_cast<const char*>(chars + i * width);
    v.emplace_back(rec, strnlen(rec, width));
  }
  return v;
}

}  // namespace

int copy_out(const std::string& s, char* out, uint64_t cap) {
  if (s.size() + 1 > cap) fail(errc::buffer_too_small, "shim buffer");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// sort_integers (sort.cpp:29-59)
int ref_sort_integers(const int64_t* values, uint64_t n, uint64_t max_cells,
                      int64_t* out, ref_report* report) {
  return guarded([&] {
    IntegerSortResult r = sort_integers(std::span<const int64_t>(values, n), max_cells);
    std::memcpy(out, r.values.data(), n * sizeof(int64_t));
    fill(report, r.report, r.spec);
  });
}

// Core only: build_count_space + extract over prebuilt DigitKeys
// (hashing.cpp:40-52, extraction.cpp:5-32).  Used by the CPU baseline timer.
int ref_sort_keys_core(const uint64_t* keys, uint64_t n, uint32_t radix,
                       uint32_t total_digits, uint32_t integer_digits,
                       uint64_t max_cells, uint64_t* out, ref_report* report) {
  return guarded([&] {
    const KeySpec spec = make_key_spec(radix, total_digits, integer_digits, max_cells);
    std::vector<DigitKey> dk;
    dk.reserve(n);
    for (uint64_t i = 0; i < n; ++i) dk.push_back(DigitKey{keys[i], spec});
    HashedSpace built = build_count_space(dk, spec, {}, max_cells);
    const ExtractionReport rep = extract(built.space, built.maps,
                                         std::span<uint64_t>(out, n));
    fill(report, rep, spec);
  });
}

int ref_float_to_decimal(double x, uint32_t scale, uint64_t* mantissa) {
  return guarded([&] { *mantissa = float_to_decimal(x, scale).mantissa; });
}

// float_to_decimal of every element: mantissa and status per element (the
// per-element statuses let the GPU parity tests sample every exponent).
int ref_float_to_decimal_many(const double* x, uint64_t n, uint32_t scale, uint64_t* mantissa,
                              int32_t* status) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t m = 0;
    status[i] = guarded([&] { m = float_to_decimal(x[i], scale).mantissa; });
    mantissa[i] = m;
  }
  return 0;
}

// float_to_decimal per element, then the core with KeySpec{10, lambda+cd, lambda}
// (key_model.cpp:122-124 for lambda).
int ref_sort_f64(const double* x, uint64_t n, uint32_t scale, uint64_t max_cells,
                 uint64_t* out, ref_report* report) {
  return guarded([&] {
    std::vector<uint64_t> m(n);
    uint64_t max_m = 0;
    for (uint64_t i = 0; i < n; ++i) {
      m[i] = float_to_decimal(x[i], scale).mantissa;
      if (m[i] > max_m) max_m = m[i];
    }
    const uint32_t lambda = decimal_digit_count(max_m / checked_pow(10, scale));
    const KeySpec spec = make_key_spec(10, lambda + scale, lambda, max_cells);
    std::vector<DigitKey> dk;
    dk.reserve(n);
    for (uint64_t v : m) dk.push_back(DigitKey{v, spec});
    HashedSpace built = build_count_space(dk, spec, {}, max_cells);
    const ExtractionReport rep = extract(built.space, built.maps,
                                         std::span<uint64_t>(out, n));
    fill(report, rep, spec);
  });
}

// sort_decimals (sort.cpp:16-27); inputs/outputs as NUL-separated text.
int ref_sort_decimals(const char* joined, uint64_t n, uint64_t max_cells,
                      char* out, uint64_t out_capacity, ref_report* report) {
  return guarded([&] {
    std::vector<std::string> v;
    const char* p = joined;
    for (uint64_t i = 0; i < n; ++i) {
      v.emplace_back(p);
      p += v.back().size() + 1;
    }
    DecimalSortResult r = sort_decimals(v, max_cells);
    std::string flat;
    for (const auto& s : r.values) {
      flat += s;
      flat += '\0';
    }
    if (flat.size() > out_capacity) fail(errc::buffer_too_small, "shim buffer");
    std::memcpy(out, flat.data(), flat.size());
    fill(report, r.report, r.spec);
  });
}

// sort_strings facade (sort.cpp:61-77) over fixed-width NUL-padded records.
int ref_sort_strings(const uint8_t* chars, uint64_t n, uint32_t width,
                     const char* alphabet, uint64_t max_cells, uint8_t* out,
                     ref_report* report) {
  return guarded([&] {
    const Alphabet a(alphabet);
    StringSortResult r = sort_strings(records(chars, n, width), a, max_cells);
    std::memset(out, 0, n * width);
    for (uint64_t i = 0; i < n; ++i)
      std::memcpy(out + i * width, r.values[i].data(), r.values[i].size());
    fill(report, r.report, r.spec);
  });
}

int ref_strings_to_keys(const uint8_t* chars, uint64_t n, uint32_t width,
                        const char* alphabet, uint64_t max_cells, uint64_t* keys) {
  return guarded([&] {
    const Alphabet a(alphabet);
    NormalizedDataset norm = strings_to_keys(records(chars, n, width), a, max_cells);
    for (uint64_t i = 0; i < n; ++i) keys[i] = norm.keys[i].key;
  });
}

// baselines::oracle_sort<std::string> (baselines.hpp:56-60): ground truth for
// string configs the facade cannot take.
int ref_oracle_sort_strings(const uint8_t* chars, uint64_t n, uint32_t width,
                            uint8_t* out) {
  return guarded([&] {
    std::vector<std::string> s = baselines::oracle_sort(records(chars, n, width));
    std::memset(out, 0, n * width);
    for (uint64_t i = 0; i < n; ++i) std::memcpy(out + i * width, s[i].data(), s[i].size());
  });
}

// radix_sort_lsd_by (baselines.hpp:24-46) over (key, value) pairs: the stable
// key/value oracle.
int ref_radix_sort_lsd_kv(const uint32_t* keys, const uint32_t* vals, uint64_t n,
                          uint32_t* keys_out, uint32_t* vals_out) {
  return guarded([&] {
    std::vector<std::pair<uint32_t, uint32_t>> items(n);
    for (uint64_t i = 0; i < n; ++i) items[i] = {keys[i], vals[i]};
    baselines::radix_sort_lsd_by(items, [](const auto& p) { return p.first; });
    for (uint64_t i = 0; i < n; ++i) {
      keys_out[i] = items[i].first;
      vals_out[i] = items[i].second;
    }
  });
}

int ref_radix_sort_lsd(const uint64_t* values, uint64_t n, uint64_t* out) {
  return guarded([&] {
    std::vector<uint64_t> r = baselines::radix_sort_lsd(std::span<const uint64_t>(values, n));
    std::memcpy(out, r.data(), n * sizeof(uint64_t));
  });
}

// bench::generate (bench.cpp:75-89): the values, NUL-separated.
int ref_generate(uint64_t n, double lo, double hi, uint32_t cd, uint64_t seed, char* out, uint64_t cap) {
  return guarded([&] {
    bench::DatasetSpec ds;
    ds.n_elements = n;
    ds.range_lo = lo;
    ds.range_hi = hi;
    ds.cd = cd;
    ds.seed = seed;
    std::string flat;
    for (const std::string& v : bench::generate(ds)) {
      flat += v;
      flat += '\0';
    }
    if (flat.size() > cap) fail(errc::buffer_too_small, "shim buffer");
    std::memcpy(out, flat.data(), flat.size());
  });
}

// bench::describe (bench.cpp:101-122) as "total,integer,cells,count_dims,h_min,h_max".
int ref_describe(double lo, double hi, uint32_t cd, char* out, uint64_t cap) {
  return guarded([&] {
    const bench::KeyShape s = bench::describe(bench::CaseSpec{lo, hi, cd});
    copy_out(std::to_string(s.total_digits) + "," + std::to_string(s.integer_digits) + "," +
                 std::to_string(s.cell_count) + "," + s.count_dims + "," + s.h_min_dims + "," + s.h_max_dims,
             out, cap);
  });
}

// bench::emit_csv (bench.cpp:312-334) of one record; case_label as well.
int ref_emit_csv_one(const char* alg, uint64_t n, double lo, double hi, uint32_t cd, uint32_t trial,
                     double seconds, int has_cost, uint64_t cost, char* out, uint64_t cap) {
  return guarded([&] {
    bench::BenchRecord r;
    r.algorithm = alg;
    r.dataset.n_elements = n;
    r.dataset.range_lo = lo;
    r.dataset.range_hi = hi;
    r.dataset.cd = cd;
    r.trial = trial;
    r.elapsed_seconds = seconds;
    if (has_cost) r.extraction_cost = cost;
    const std::vector<bench::BenchRecord> one{r};
    copy_out(bench::emit_csv(one) + "|" + bench::case_label(bench::CaseSpec{lo, hi, cd}), out, cap);
  });
}

// bench::parse_csv + bench::fit_scaling (bench.cpp:228-297, 365-393) of a
// one-group CSV; the worst-case constant table entry for d.
int ref_fit_scaling_csv(const char* csv, double* slope, double* intercept, double* r2) {
  return guarded([&] {
    const std::vector<bench::BenchRecord> recs = bench::parse_csv(csv);
    const bench::ScalingReport rep = bench::fit_scaling(recs);
    *slope = rep.slope;
    *intercept = rep.intercept;
    *r2 = rep.r_squared;
  });
}

int ref_worst_case_constant(uint32_t d, uint64_t* num, uint64_t* den, int* below) {
  return guarded([&] {
    const bench::WorstCaseConstant w = bench::worst_case_constant(d);
    *num = w.numerator;
    *den = w.denominator;
    *below = w.below_squared_bound() ? 1 : 0;
  });
}

uint64_t ref_splitmix64_next(uint64_t* state) {
  Splitmix64 g(*state);
  const uint64_t v = g.next();
  *state += 0x9E3779B97F4A7C15ULL;
  return v;
}

uint64_t ref_splitmix64_mix(uint64_t seed, uint64_t index) {
  return splitmix64_mix(seed, index);
}

}  // extern "C"

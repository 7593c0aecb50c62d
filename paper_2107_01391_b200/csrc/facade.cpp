// facade.cpp — recsort:: C++ facade (include/recsort/sort.hpp) over the C-ABI.
// Host-side only: text ingest/render and host<->device copies; every sort
// runs through an rs_sort_* entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "recsort/sort.hpp"
#include "recsort_b200.h"

namespace recsort {
namespace {

void throw_status(rs_status st) {
  if (st == RS_OK) return;
  const std::string msg = rs_last_error();
  if (st >= RS_PARSE_ERROR && st <= RS_INVALID_ARGUMENT) throw Error(static_cast<errc>(st - 1), msg);
  throw Error(errc::device_error, msg);
}

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw Error(errc::device_error, cudaGetErrorString(e));
}

// RAII device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) {
    if (n) cuda_ok(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

template <class T>
DevBuf<T> upload(const T* h, std::size_t n) {
  DevBuf<T> d(n);
  if (n) cuda_ok(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

rs_options opts(const SortOptions& o) { return rs_options{o.max_cells, o.key_digits, o.msd ? 1u : 0u}; }

ExtractionReport rep(const rs_report& r) { return ExtractionReport{r.written, r.cells_traversed}; }
KeySpec spec(const rs_report& r) { return KeySpec{r.spec.radix, r.spec.total_digits, r.spec.integer_digits}; }

// parse_decimal grammar (key_model.cpp:80-105).
void parse_decimal(const std::string& text, std::uint64_t& mantissa, std::uint32_t& scale) {
  if (text.empty()) throw Error(errc::parse_error, "empty numeral");
  if (text.front() == '-') throw Error(errc::negative_value, "negative values are not supported: '" + text + "'");
  const std::size_t dot = text.find('.');
  const std::string ip = text.substr(0, dot);
  const std::string fp = dot == std::string::npos ? std::string{} : text.substr(dot + 1);
  if (dot != std::string::npos && fp.find('.') != std::string::npos)
    throw Error(errc::parse_error, "multiple decimal points in '" + text + "'");
  if (dot != std::string::npos && fp.empty())
    throw Error(errc::parse_error, "no digits after decimal point in '" + text + "'");
  if (ip.empty() && fp.empty()) throw Error(errc::parse_error, "no digits in '" + text + "'");
  std::uint64_t acc = 0;
  for (const std::string* part : {&ip, &fp})
    for (char c : *part) {
      if (c < '0' || c > '9') throw Error(errc::parse_error, "invalid character in numeral '" + text + "'");
      const std::uint64_t d = static_cast<std::uint64_t>(c - '0');
      if (acc > (~std::uint64_t{0} - d) / 10)
        throw Error(errc::cell_budget_exceeded, "numeral '" + text + "' has more digits than any cell budget admits");
      acc = acc * 10 + d;
    }
  mantissa = acc;
  scale = static_cast<std::uint32_t>(fp.size());
}

std::uint64_t pow10(std::uint32_t e) {
  std::uint64_t r = 1;
  for (std::uint32_t i = 0; i < e; ++i) {
    if (r > ~std::uint64_t{0} / 10) throw Error(errc::cell_budget_exceeded, "key space overflows 64 bits");
    r *= 10;
  }
  return r;
}

std::uint32_t digits(std::uint64_t v) {
  std::uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

}  // namespace

const char* errc_name(errc code) noexcept {
  if (code == errc::device_error) return "device_error";
  return rs_status_name(static_cast<rs_status>(static_cast<int>(code) + 1));
}

Alphabet::Alphabet(std::string_view symbols) : symbols_(symbols) {
  if (symbols.empty()) throw Error(errc::invalid_argument, "alphabet is empty");
  bool seen[256] = {};
  for (unsigned char c : symbols_) {
    if (seen[c]) throw Error(errc::invalid_argument, std::string("duplicate symbol '") + char(c) + "' in alphabet");
    seen[c] = true;
  }
}

const Alphabet& Alphabet::lowercase() {
  static const Alphabet a("abcdefghijklmnopqrstuvwxyz");
  return a;
}

IntegerSortResult sort_integers(std::span<const std::int64_t> values, std::uint64_t max_cells) {
  const std::size_t n = values.size();
  DevBuf<std::int64_t> in = upload(values.data(), n), out(n);
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_i64(in.p, n, out.p, n, &o, &r, nullptr));
  IntegerSortResult res;
  res.values.resize(n);
  if (n) cuda_ok(cudaMemcpy(res.values.data(), out.p, n * sizeof(std::int64_t), cudaMemcpyDeviceToHost));
  res.spec = spec(r);
  res.report = rep(r);
  return res;
}

DecimalKeySortResult sort_decimal_keys(std::span<const std::string> values, std::uint64_t max_cells) {
  // normalize_dataset (key_model.cpp:107-133) on the host, the count grid on the device
  std::vector<std::uint64_t> mant(values.size());
  std::vector<std::uint32_t> scales(values.size());
  std::uint32_t scale = 0;
  std::uint64_t max_int = 0;
  for (std::size_t i = 0; i < values.size(); ++i) {
    parse_decimal(values[i], mant[i], scales[i]);
    scale = std::max(scale, scales[i]);
    max_int = std::max(max_int, mant[i] / pow10(scales[i]));
  }
  const std::uint32_t lambda = values.empty() ? 1 : digits(max_int);
  const std::uint32_t total = values.empty() ? 1 : lambda + scale;
  rs_key_spec ks{10, total, lambda};
  for (std::size_t i = 0; i < values.size(); ++i) mant[i] *= pow10(scale - scales[i]);
  const std::size_t n = mant.size();
  DevBuf<std::uint64_t> in = upload(mant.data(), n), out(n);
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_keys(in.p, n, ks, out.p, n, &o, &r, nullptr));
  DecimalKeySortResult res;
  res.keys.resize(n);
  if (n) cuda_ok(cudaMemcpy(res.keys.data(), out.p, n * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
  res.spec = KeySpec{10, total, lambda};
  res.report = rep(r);
  return res;
}

DecimalSortResult sort_decimals(std::span<const std::string> values, std::uint64_t max_cells) {
  DecimalKeySortResult k = sort_decimal_keys(values, max_cells);
  DecimalSortResult res;
  res.spec = k.spec;
  res.report = k.report;
  const std::uint64_t p = pow10(k.spec.scale());
  for (std::uint64_t key : k.keys) {  // format_scaled_decimal (key_model.cpp:170-180)
    std::string s = std::to_string(key / p);
    if (k.spec.scale()) {
      const std::string frac = std::to_string(key % p);
      s += '.';
      s.append(k.spec.scale() - frac.size(), '0');
      s += frac;
    }
    res.values.push_back(std::move(s));
  }
  return res;
}

StringSortResult sort_strings(std::span<const std::string> values, const Alphabet& alphabet,
                              std::uint64_t max_cells) {
  std::size_t width = 1;
  for (const std::string& v : values) width = std::max(width, v.size());
  if (width > 12) throw Error(errc::cell_budget_exceeded, "key space overflows the cell budget");
  const std::size_t n = values.size();
  std::vector<std::uint8_t> recs(n * width, 0);
  for (std::size_t i = 0; i < n; ++i) std::memcpy(recs.data() + i * width, values[i].data(), values[i].size());
  DevBuf<std::uint8_t> in = upload(recs.data(), recs.size()), out(recs.size());
  const std::string sym(alphabet.symbols());
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_fixed_str(in.p, n, static_cast<std::uint32_t>(width), sym.c_str(), out.p, n, &o, &r, nullptr));
  if (!recs.empty()) cuda_ok(cudaMemcpy(recs.data(), out.p, recs.size(), cudaMemcpyDeviceToHost));
  StringSortResult res;
  res.spec = spec(r);
  res.report = rep(r);
  for (std::size_t i = 0; i < n; ++i) {
    const char* p = reinterpret_cast<const char*>(recs.data() + i * width);
    res.values.emplace_back(p, strnlen(p, width));
  }
  return res;
}

ExtractionReport recombinant_sort(const std::uint32_t* d_keys, std::uint64_t n, std::uint32_t* d_out,
                                  const SortOptions& opt, void* stream) {
  rs_options o = opts(opt);
  rs_report r{};
  throw_status(rs_sort_u32(d_keys, n, d_out, n, &o, &r, stream));
  return rep(r);
}

ExtractionReport recombinant_sort(const std::uint32_t* d_keys, const std::uint32_t* d_vals, std::uint64_t n,
                                  std::uint32_t* d_keys_out, std::uint32_t* d_vals_out, const SortOptions& opt,
                                  void* stream) {
  rs_options o = opts(opt);
  rs_report r{};
  throw_status(rs_sort_u32_kv(d_keys, d_vals, n, d_keys_out, d_vals_out, n, &o, &r, stream));
  return rep(r);
}

ExtractionReport recombinant_sort(const double* d_x, std::uint64_t n, std::uint32_t scale,
                                  std::uint64_t* d_mantissas, const SortOptions& opt, void* stream) {
  rs_options o = opts(opt);
  rs_report r{};
  throw_status(rs_sort_f64(d_x, n, scale, d_mantissas, n, &o, &r, stream));
  return rep(r);
}

ExtractionReport recombinant_sort(const std::uint8_t* d_records, std::uint64_t n, std::uint32_t width,
                                  const Alphabet& alphabet, std::uint8_t* d_out, const SortOptions& opt,
                                  void* stream) {
  rs_options o = opts(opt);
  rs_report r{};
  const std::string sym(alphabet.symbols());
  throw_status(rs_sort_fixed_str(d_records, n, width, sym.c_str(), d_out, n, &o, &r, stream));
  return rep(r);
}

}  // namespace recsort

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

namespace {
// The numerals as a device string column (Arrow layout: bytes + n+1 offsets).
struct DecColumn {
  DevBuf<char> chars;
  DevBuf<std::uint64_t> offsets;
};
DecColumn upload_column(std::span<const std::string> values) {
  std::vector<std::uint64_t> off(values.size() + 1, 0);
  std::string flat;
  for (std::size_t i = 0; i < values.size(); ++i) {
    flat += values[i];
    off[i + 1] = flat.size();
  }
  return DecColumn{upload(flat.data(), std::max<std::size_t>(flat.size(), 1)), upload(off.data(), off.size())};
}
}  // namespace

DecimalKeySortResult sort_decimal_keys(std::span<const std::string> values, std::uint64_t max_cells) {
  // parse_decimal + normalize_dataset + count + extract, all on the device
  const std::size_t n = values.size();
  DecColumn col = upload_column(values);
  DevBuf<std::uint64_t> out(std::max<std::size_t>(n, 1));
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_decimal_strings(col.chars.p, col.offsets.p, n, out.p, n, &o, &r, nullptr));
  DecimalKeySortResult res;
  res.keys.resize(n);
  if (n) cuda_ok(cudaMemcpy(res.keys.data(), out.p, n * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
  res.spec = spec(r);
  res.report = rep(r);
  return res;
}

DecimalSortResult sort_decimals(std::span<const std::string> values, std::uint64_t max_cells) {
  // as sort_decimal_keys, then format_scaled_decimal on the device
  const std::size_t n = values.size();
  DecColumn col = upload_column(values);
  DevBuf<std::uint64_t> keys(std::max<std::size_t>(n, 1));
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_decimal_strings(col.chars.p, col.offsets.p, n, keys.p, n, &o, &r, nullptr));
  DecimalSortResult res;
  res.spec = spec(r);
  res.report = rep(r);
  DevBuf<std::uint64_t> off(n + 1);
  std::uint64_t need = 0;
  const rs_status st = rs_format_decimals(keys.p, n, res.spec.scale(), nullptr, 0, off.p, &need, nullptr);
  if (st != RS_OK && st != RS_BUFFER_TOO_SMALL) throw_status(st);
  DevBuf<char> chars(std::max<std::uint64_t>(need, 1));
  throw_status(rs_format_decimals(keys.p, n, res.spec.scale(), chars.p, need, off.p, &need, nullptr));
  std::string flat(need, '\0');
  std::vector<std::uint64_t> h_off(n + 1);
  if (need) cuda_ok(cudaMemcpy(flat.data(), chars.p, need, cudaMemcpyDeviceToHost));
  cuda_ok(cudaMemcpy(h_off.data(), off.p, (n + 1) * sizeof(std::uint64_t), cudaMemcpyDeviceToHost));
  res.values.reserve(n);
  for (std::size_t i = 0; i < n; ++i) res.values.emplace_back(flat.substr(h_off[i], h_off[i + 1] - h_off[i]));
  return res;
}

StringSortResult sort_strings(std::span<const std::string> values, const Alphabet& alphabet,
                              std::uint64_t max_cells) {
  std::size_t width = 1;
  for (const std::string& v : values) width = std::max(width, v.size());
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

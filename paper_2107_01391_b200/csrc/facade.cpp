// facade.cpp — the recsort:: C++ surface (include/recsort/{error,key_model,
// hashing,extraction,sort}.hpp) over the C-ABI.  Host-side only: packing of
// host inputs, host<->device copies and the single-key helpers the reference
// calls per key; every span-level step (normalize, strings_to_keys, the
// hashing cycle, extraction, the sorts) runs through an rs_* entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "recsort/sort.hpp"
#include "recsort_b200.h"

namespace recsort {

namespace detail {
// The library's bulk fill of the reference's host objects after a device
// build (the reference's loop fills them through increment()/update()).
struct SpaceAccess {
  static std::vector<std::uint64_t>& counts(CountSpace& s) { return s.counts_; }
  static const std::vector<std::uint64_t>& counts(const CountSpace& s) { return s.counts_; }
  static void set_totals(CountSpace& s, std::uint64_t inserted, std::uint64_t accesses) {
    s.total_inserted_ = inserted;
    s.cell_accesses_ = accesses;
  }
  static void add_accesses(const CountSpace& s, std::uint64_t k) { s.cell_accesses_ += k; }
  static std::vector<HMinEntry>& h_min(TraverseMaps& m) { return m.h_min_; }
  static std::vector<std::int64_t>& h_max(TraverseMaps& m) { return m.h_max_; }
  static const std::vector<HMinEntry>& h_min(const TraverseMaps& m) { return m.h_min_; }
  static const std::vector<std::int64_t>& h_max(const TraverseMaps& m) { return m.h_max_; }
};
}  // namespace detail

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

template <class T>
void download(T* h, const T* d, std::size_t n) {
  if (n) cuda_ok(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost));
}

rs_options opts(const SortOptions& o) { return rs_options{o.max_cells, o.key_digits, o.msd ? 1u : 0u}; }
rs_key_spec abi(const KeySpec& s) { return rs_key_spec{s.radix, s.total_digits, s.integer_digits}; }
KeySpec spec_of(const rs_key_spec& s) { return KeySpec{s.radix, s.total_digits, s.integer_digits}; }
ExtractionReport rep(const rs_report& r) { return ExtractionReport{r.written, r.cells_traversed}; }

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

// Strings as NUL-padded records of the longest string's width (>= 1), for the
// device; the first embedded NUL (the device reads NUL as the end of a
// string) by (string, position).
struct Records {
  std::vector<std::uint8_t> bytes;
  std::size_t width = 1;
  std::size_t nul_string = SIZE_MAX, nul_pos = 0;
};
Records pack(std::span<const std::string> values) {
  Records r;
  for (const std::string& v : values) r.width = std::max(r.width, v.size());
  r.bytes.assign(values.size() * r.width, 0);
  for (std::size_t i = 0; i < values.size(); ++i) {
    std::memcpy(r.bytes.data() + i * r.width, values[i].data(), values[i].size());
    if (r.nul_string == SIZE_MAX) {
      const std::size_t z = values[i].find('\0');
      if (z != std::string::npos) {
        r.nul_string = i;
        r.nul_pos = z;
      }
    }
  }
  return r;
}

// Alphabet::ordinal's error for the first symbol outside the alphabet
// (key_model.cpp:208-214): an embedded NUL the device cannot see is that
// symbol unless an earlier (string, position) failed first on the device.
void check_embedded_nul(const Records& r, std::span<const std::string> values, const Alphabet& alphabet) {
  if (r.nul_string == SIZE_MAX) return;
  if (alphabet.contains(0)) throw Error(errc::invalid_argument, "NUL as an alphabet symbol is not supported");
  for (std::size_t i = 0; i <= r.nul_string; ++i) {
    const std::size_t end = i == r.nul_string ? r.nul_pos : values[i].size();
    for (std::size_t j = 0; j < end; ++j) (void)alphabet.ordinal(static_cast<unsigned char>(values[i][j]));
  }
  (void)alphabet.ordinal(0);  // throws symbol_out_of_alphabet
}

std::uint64_t pow10(std::uint32_t e) { return checked_pow(10, e); }

}  // namespace

// ------------------------------------------------------------- error.hpp
const char* errc_name(errc code) noexcept {
  if (code == errc::device_error) return "device_error";
  return rs_status_name(static_cast<rs_status>(static_cast<int>(code) + 1));
}

// --------------------------------------------------------- key_model.hpp
std::uint64_t checked_pow(std::uint64_t radix, std::uint32_t exp) {
  std::uint64_t v = 0;
  throw_status(rs_checked_pow(radix, exp, &v));
  return v;
}

std::uint32_t decimal_digit_count(std::uint64_t v) noexcept {
  std::uint32_t d = 1;
  for (; v >= 10; v /= 10) ++d;
  return d;
}

std::uint64_t DecimalValue::integer_part() const { return mantissa / pow10(scale); }

KeySpec make_key_spec(std::uint32_t radix, std::uint32_t total_digits, std::uint32_t integer_digits,
                      std::uint64_t max_cells) {
  rs_key_spec s{};
  throw_status(rs_make_key_spec(radix, total_digits, integer_digits, max_cells, &s));
  return spec_of(s);
}

DecimalValue parse_decimal(std::string_view text) {
  const std::string one(text);
  DecColumn col = upload_column(std::span<const std::string>(&one, 1));
  DevBuf<std::uint64_t> m(1);
  DevBuf<std::uint32_t> sc(1);
  throw_status(rs_parse_decimals(col.chars.p, col.offsets.p, 1, m.p, sc.p, nullptr));
  DecimalValue v;
  download(&v.mantissa, m.p, 1);
  download(&v.scale, sc.p, 1);
  return v;
}

NormalizedDataset normalize_dataset(std::span<const std::string> values, std::uint64_t max_cells) {
  const std::size_t n = values.size();
  DecColumn col = upload_column(values);
  DevBuf<std::uint64_t> keys(n);
  rs_options o{max_cells, 0, 0};
  rs_key_spec s{};
  throw_status(rs_normalize_decimal_strings(col.chars.p, col.offsets.p, n, keys.p, &o, &s, nullptr));
  std::vector<std::uint64_t> h(n);
  download(h.data(), keys.p, n);
  NormalizedDataset out;
  out.spec = spec_of(s);
  out.keys.reserve(n);
  for (std::uint64_t k : h) out.keys.push_back(DigitKey{k, out.spec});
  return out;
}

DecimalValue float_to_decimal(double x, std::uint32_t scale) {
  DevBuf<double> d = upload(&x, 1);
  DevBuf<std::uint64_t> m(1);
  throw_status(rs_float_to_decimal(d.p, 1, scale, m.p, nullptr));
  DecimalValue v{0, scale};
  download(&v.mantissa, m.p, 1);
  return v;
}

std::vector<std::uint32_t> digits_of(const DigitKey& k) {
  std::vector<std::uint32_t> d(k.spec.total_digits);
  std::uint64_t rest = k.key;
  for (std::uint32_t i = k.spec.total_digits; i > 0; --i) {
    d[i - 1] = static_cast<std::uint32_t>(rest % k.spec.radix);
    rest /= k.spec.radix;
  }
  return d;
}

std::string format_scaled_decimal(std::uint64_t mantissa, std::uint32_t scale) {
  const std::uint64_t p = pow10(scale);
  std::string s = std::to_string(mantissa / p);
  if (scale == 0) return s;
  const std::string frac = std::to_string(mantissa % p);
  return s + '.' + std::string(scale - frac.size(), '0') + frac;
}

std::string reconstruct_value(std::uint64_t key, const KeySpec& spec) {
  return format_scaled_decimal(key, spec.scale());
}

std::string reconstruct_value(const DigitKey& k) { return reconstruct_value(k.key, k.spec); }

Alphabet::Alphabet(std::string_view symbols) : symbols_(symbols) {
  if (symbols_.empty()) fail(errc::invalid_argument, "alphabet is empty");
  if (symbols_.size() > 0xFFFE) fail(errc::invalid_argument, "alphabet too large");
  std::uint16_t ord = 0;
  for (const char ch : symbols_) {
    const auto c = static_cast<unsigned char>(ch);
    if (ordinal_of_[c] != 0) fail(errc::invalid_argument, std::string("duplicate symbol '") + ch + "' in alphabet");
    ordinal_of_[c] = ++ord;
  }
}

const Alphabet& Alphabet::lowercase() {
  static const Alphabet a("abcdefghijklmnopqrstuvwxyz");
  return a;
}

std::uint32_t Alphabet::ordinal(unsigned char c) const {
  if (ordinal_of_[c] == 0)
    fail(errc::symbol_out_of_alphabet, std::string("symbol '") + static_cast<char>(c) + "' is not in the alphabet");
  return ordinal_of_[c];
}

char Alphabet::symbol(std::uint32_t ordinal) const {
  if (ordinal == 0 || ordinal > symbols_.size())
    fail(errc::symbol_out_of_alphabet, "ordinal " + std::to_string(ordinal) + " has no symbol");
  return symbols_[ordinal - 1];
}

NormalizedDataset strings_to_keys(std::span<const std::string> values, const Alphabet& alphabet,
                                  std::uint64_t max_cells) {
  const Records r = pack(values);
  const auto w = static_cast<std::uint32_t>(r.width);
  make_key_spec(alphabet.radix(), w, w, max_cells);  // the budget first (key_model.cpp:230-231)
  check_embedded_nul(r, values, alphabet);
  const std::size_t n = values.size();
  DevBuf<std::uint8_t> in = upload(r.bytes.data(), r.bytes.size());
  DevBuf<std::uint64_t> keys(n);
  const std::string sym(alphabet.symbols());
  rs_options o{max_cells, 0, 0};
  rs_key_spec s{};
  throw_status(rs_strings_to_keys(in.p, n, w, sym.c_str(), keys.p, &o, &s, nullptr));
  std::vector<std::uint64_t> h(n);
  download(h.data(), keys.p, n);
  NormalizedDataset out;
  out.spec = spec_of(s);  // {radix, w, w}: no string holds a NUL past check_embedded_nul
  out.keys.reserve(n);
  for (std::uint64_t k : h) out.keys.push_back(DigitKey{k, out.spec});
  return out;
}

std::string key_to_string(std::uint64_t key, const KeySpec& spec, const Alphabet& alphabet) {
  std::vector<std::uint32_t> ords(spec.total_digits);
  for (std::uint32_t i = spec.total_digits; i > 0; --i) {
    ords[i - 1] = static_cast<std::uint32_t>(key % spec.radix);
    key /= spec.radix;
  }
  std::size_t len = ords.size();
  while (len > 0 && ords[len - 1] == 0) --len;
  std::string s;
  s.reserve(len);
  for (std::size_t i = 0; i < len; ++i) s += alphabet.symbol(ords[i]);
  return s;
}

// ----------------------------------------------------------- hashing.hpp
std::uint64_t CountSpace::sum_cells() const noexcept {
  std::uint64_t s = 0;
  for (std::uint64_t c : counts_) s += c;
  return s;
}

std::uint64_t CountSpace::occupied_cells() const noexcept {
  std::uint64_t s = 0;
  for (std::uint64_t c : counts_) s += c != 0;
  return s;
}

HashedSpace new_space(const KeySpec& spec, std::uint64_t max_cells) {
  const std::uint64_t cells = spec.cell_count();
  if (cells > max_cells)
    fail(errc::cell_budget_exceeded,
         "count space needs " + std::to_string(cells) + " cells, budget is " + std::to_string(max_cells));
  return HashedSpace{CountSpace(spec), TraverseMaps(spec)};
}

void hash_insert(CountSpace& space, TraverseMaps& maps, const DigitKey& k) {
  if (k.spec != space.spec()) fail(errc::spec_mismatch, "key was built under a different key spec");
  if (k.key >= space.cell_limit())
    fail(errc::spec_mismatch, "key " + std::to_string(k.key) + " is outside its spec's key space");
  space.increment(k.key);
  const std::uint64_t mod = space.suffix_modulus();
  maps.update(static_cast<std::uint32_t>(k.key / mod), k.key % mod);
}

namespace {
// The keys of a DigitKey span for the device, checked in the reference's
// per-key order (hashing.cpp:27-38): spec first, then range.
std::vector<std::uint64_t> pack_keys(std::span<const DigitKey> keys, const KeySpec& spec) {
  const std::uint64_t cells = spec.cell_count();
  std::vector<std::uint64_t> h(keys.size());
  for (std::size_t i = 0; i < keys.size(); ++i) {
    if (keys[i].spec != spec) fail(errc::spec_mismatch, "key was built under a different key spec");
    if (keys[i].key >= cells)
      fail(errc::spec_mismatch, "key " + std::to_string(keys[i].key) + " is outside its spec's key space");
    h[i] = keys[i].key;
  }
  return h;
}
}  // namespace

HashedSpace build_count_space(std::span<const DigitKey> keys, const KeySpec& spec, const InsertSnapshot& on_insert,
                              std::uint64_t max_cells) {
  HashedSpace built = new_space(spec, max_cells);
  if (on_insert) {  // the snapshot observes every intermediate state: key by key
    std::size_t inserted = 0;
    for (const DigitKey& k : keys) {
      hash_insert(built.space, built.maps, k);
      on_insert(++inserted, built.space, built.maps);
    }
    return built;
  }
  const std::vector<std::uint64_t> h = pack_keys(keys, spec);
  const std::uint64_t cells = spec.cell_count();
  DevBuf<std::uint64_t> d_keys = upload(h.data(), h.size());
  DevBuf<std::uint64_t> d_counts(cells);
  std::vector<std::uint64_t> row_min(spec.radix);
  std::vector<std::int64_t> row_max(spec.radix);
  throw_status(rs_build_count_space(d_keys.p, h.size(), abi(spec), max_cells, d_counts.p, row_min.data(),
                                    row_max.data(), nullptr));
  download(detail::SpaceAccess::counts(built.space).data(), d_counts.p, cells);
  detail::SpaceAccess::set_totals(built.space, h.size(), h.size());  // one cell access per insertion
  auto& lo = detail::SpaceAccess::h_min(built.maps);
  auto& hi = detail::SpaceAccess::h_max(built.maps);
  for (std::uint32_t r = 0; r < spec.radix; ++r) {
    hi[r] = row_max[r];
    lo[r] = row_max[r] >= 0 ? HMinEntry{true, row_min[r]} : HMinEntry{};
  }
  return built;
}

// -------------------------------------------------------- extraction.hpp
ExtractionReport extract(const CountSpace& space, const TraverseMaps& maps, std::span<std::uint64_t> out,
                         const EmitHook& on_emit) {
  const std::uint64_t total = space.total_inserted();
  if (out.size() < total)
    fail(errc::buffer_too_small,
         "output buffer holds " + std::to_string(out.size()) + " keys, need " + std::to_string(total));
  const KeySpec& spec = space.spec();
  const auto& counts = detail::SpaceAccess::counts(space);
  const auto& lo = detail::SpaceAccess::h_min(maps);
  const auto& hi = detail::SpaceAccess::h_max(maps);
  std::vector<std::uint64_t> row_min(spec.radix, ~std::uint64_t{0});
  std::vector<std::int64_t> row_max(spec.radix, -1);
  for (std::uint32_t r = 0; r < spec.radix && r < maps.rows(); ++r) {
    if (!lo[r].occupied) continue;  // untouched rows cost nothing
    row_min[r] = lo[r].min_suffix;
    row_max[r] = hi[r];
  }
  DevBuf<std::uint64_t> d_counts = upload(counts.data(), counts.size());
  DevBuf<std::uint64_t> d_out(std::max<std::uint64_t>(total, 1));
  rs_report r{};
  throw_status(rs_extract(d_counts.p, abi(spec), total, row_min.data(), row_max.data(), d_out.p, total, &r,
                          nullptr));
  download(out.data(), d_out.p, r.written);
  detail::SpaceAccess::add_accesses(space, r.cells_traversed);  // one read per traversed cell
  if (on_emit)
    for (std::uint64_t i = 0; i < r.written; ++i) on_emit(i + 1, out[i]);
  return ExtractionReport{r.written, r.cells_traversed};
}

SortedKeys sort_keys(std::span<const DigitKey> keys, const KeySpec& spec, std::uint64_t max_cells) {
  new_space(spec, max_cells);  // (hashing.cpp:17-25: the budget before anything else)
  const std::vector<std::uint64_t> h = pack_keys(keys, spec);
  const std::size_t n = h.size();
  DevBuf<std::uint64_t> d_in = upload(h.data(), n), d_out(n);
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_keys(d_in.p, n, abi(spec), d_out.p, n, &o, &r, nullptr));
  std::vector<std::uint64_t> sorted(n);
  download(sorted.data(), d_out.p, n);
  SortedKeys res;
  res.report = rep(r);
  res.keys.reserve(n);
  for (std::uint64_t k : sorted) res.keys.push_back(DigitKey{k, spec});
  return res;
}

// -------------------------------------------------------------- sort.hpp
IntegerSortResult sort_integers(std::span<const std::int64_t> values, std::uint64_t max_cells) {
  const std::size_t n = values.size();
  DevBuf<std::int64_t> in = upload(values.data(), n), out(n);
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_i64(in.p, n, out.p, n, &o, &r, nullptr));
  IntegerSortResult res;
  res.values.resize(n);
  download(res.values.data(), out.p, n);
  res.spec = spec_of(r.spec);
  res.report = rep(r);
  return res;
}

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
  download(res.keys.data(), out.p, n);
  res.spec = spec_of(r.spec);
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
  res.spec = spec_of(r.spec);
  res.report = rep(r);
  DevBuf<std::uint64_t> off(n + 1);
  std::uint64_t need = 0;
  const rs_status st = rs_format_decimals(keys.p, n, res.spec.scale(), nullptr, 0, off.p, &need, nullptr);
  if (st != RS_OK && st != RS_BUFFER_TOO_SMALL) throw_status(st);
  DevBuf<char> chars(std::max<std::uint64_t>(need, 1));
  throw_status(rs_format_decimals(keys.p, n, res.spec.scale(), chars.p, need, off.p, &need, nullptr));
  std::string flat(need, '\0');
  std::vector<std::uint64_t> h_off(n + 1);
  download(flat.data(), chars.p, need);
  download(h_off.data(), off.p, n + 1);
  res.values.reserve(n);
  for (std::size_t i = 0; i < n; ++i) res.values.emplace_back(flat.substr(h_off[i], h_off[i + 1] - h_off[i]));
  return res;
}

StringSortResult sort_strings(std::span<const std::string> values, const Alphabet& alphabet,
                              std::uint64_t max_cells) {
  const Records rec = pack(values);
  const std::size_t n = values.size(), width = rec.width;
  if (rec.nul_string != SIZE_MAX) {  // the reference's check order: budget, then symbols
    make_key_spec(alphabet.radix(), static_cast<std::uint32_t>(width), static_cast<std::uint32_t>(width), max_cells);
    check_embedded_nul(rec, values, alphabet);
  }
  DevBuf<std::uint8_t> in = upload(rec.bytes.data(), rec.bytes.size()), out(rec.bytes.size());
  const std::string sym(alphabet.symbols());
  rs_options o{max_cells, 0, 0};
  rs_report r{};
  throw_status(rs_sort_fixed_str(in.p, n, static_cast<std::uint32_t>(width), sym.c_str(), out.p, n, &o, &r, nullptr));
  std::vector<std::uint8_t> sorted(rec.bytes.size());
  download(sorted.data(), out.p, sorted.size());
  StringSortResult res;
  res.spec = spec_of(r.spec);
  res.report = rep(r);
  res.values.reserve(n);
  for (std::size_t i = 0; i < n; ++i) {
    const char* p = reinterpret_cast<const char*>(sorted.data() + i * width);
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

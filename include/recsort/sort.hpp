// recsort/sort.hpp — drop-in C++ facade of the B200 library.
//
// Same include path, namespace and names as the reference's public surface
// (proj/include/recsort/sort.hpp:19-61, error.hpp:10-40, key_model.hpp:16,
// 35-46, 93-121, extraction.hpp:12-15), implemented over the C-ABI in
// recsort_b200.h (csrc/facade.cpp).  Host spans in, std::vector out; the
// copies to and from the device happen inside.  Errors are thrown as
// recsort::Error with the reference's errc codes.  recombinant_sort()
// overloads are the device-pointer entry points (caller-owned device memory,
// a cudaStream_t passed as void*).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "recsort_b200.h"

namespace recsort {

enum class errc {
  parse_error,
  negative_value,
  non_finite,
  cell_budget_exceeded,
  symbol_out_of_alphabet,
  spec_mismatch,
  buffer_too_small,
  range_exceeded,
  out_of_range,
  invalid_range,
  insufficient_data,
  invalid_argument,
  device_error,  // not in the reference: CUDA failure or no device (there is no CPU path)
};

const char* errc_name(errc code) noexcept;

class Error : public std::runtime_error {
 public:
  Error(errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

inline constexpr std::uint64_t kDefaultCellBudget = RS_DEFAULT_CELL_BUDGET;

struct KeySpec {
  std::uint32_t radix = 10;
  std::uint32_t total_digits = 1;
  std::uint32_t integer_digits = 1;
  std::uint32_t scale() const noexcept { return total_digits - integer_digits; }
  bool operator==(const KeySpec&) const = default;
};

struct ExtractionReport {
  std::uint64_t written = 0;
  std::uint64_t cells_traversed = 0;
};

// An ordered set of distinct symbols; ordinal 0 is the end-of-string pad.
class Alphabet {
 public:
  explicit Alphabet(std::string_view symbols);
  static const Alphabet& lowercase();
  std::uint32_t radix() const noexcept { return static_cast<std::uint32_t>(symbols_.size()) + 1; }
  std::string_view symbols() const noexcept { return symbols_; }

 private:
  std::string symbols_;
};

struct DecimalKeySortResult {
  std::vector<std::uint64_t> keys;
  KeySpec spec;
  ExtractionReport report;
};
struct DecimalSortResult {
  std::vector<std::string> values;
  KeySpec spec;
  ExtractionReport report;
};
struct IntegerSortResult {
  std::vector<std::int64_t> values;
  KeySpec spec;
  ExtractionReport report;
};
struct StringSortResult {
  std::vector<std::string> values;
  KeySpec spec;
  ExtractionReport report;
};

// The reference facade (sort.hpp:44-61), same signatures.
DecimalKeySortResult sort_decimal_keys(std::span<const std::string> values,
                                       std::uint64_t max_cells = kDefaultCellBudget);
DecimalSortResult sort_decimals(std::span<const std::string> values,
                                std::uint64_t max_cells = kDefaultCellBudget);
IntegerSortResult sort_integers(std::span<const std::int64_t> values,
                                std::uint64_t max_cells = kDefaultCellBudget);
StringSortResult sort_strings(std::span<const std::string> values, const Alphabet& alphabet,
                              std::uint64_t max_cells = kDefaultCellBudget);

// recombinant_sort overload set over device memory.
struct SortOptions {
  std::uint64_t max_cells = kDefaultCellBudget;
  std::uint32_t key_digits = 0;  // declared decimal width (0 = derive)
  bool msd = false;              // split grids above the budget (MSD)
};
ExtractionReport recombinant_sort(const std::uint32_t* d_keys, std::uint64_t n, std::uint32_t* d_out,
                                  const SortOptions& opt = {}, void* stream = nullptr);
ExtractionReport recombinant_sort(const std::uint32_t* d_keys, const std::uint32_t* d_vals, std::uint64_t n,
                                  std::uint32_t* d_keys_out, std::uint32_t* d_vals_out,
                                  const SortOptions& opt = {}, void* stream = nullptr);
ExtractionReport recombinant_sort(const double* d_x, std::uint64_t n, std::uint32_t scale,
                                  std::uint64_t* d_mantissas, const SortOptions& opt = {},
                                  void* stream = nullptr);
ExtractionReport recombinant_sort(const std::uint8_t* d_records, std::uint64_t n, std::uint32_t width,
                                  const Alphabet& alphabet, std::uint8_t* d_out, const SortOptions& opt = {},
                                  void* stream = nullptr);

}  // namespace recsort

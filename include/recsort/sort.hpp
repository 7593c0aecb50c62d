// recsort/sort.hpp — the reference's public sorting surface (proj/include/
// recsort/sort.hpp:19-61) over the B200 library, with the same include
// path, namespace, names and signatures, built on error.hpp / key_model.hpp /
// extraction.hpp of this directory (the reference's own header set).  Host
// spans in, std::vector out; the copies to and from the device happen inside
// (csrc/facade.cpp).  Errors are thrown as recsort::Error with the
// reference's errc codes.  The recombinant_sort() overloads are the
// device-pointer entry points (caller-owned device memory, a cudaStream_t
// passed as void*).
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "recsort/extraction.hpp"
#include "recsort/key_model.hpp"
#include "recsort_b200.h"

namespace recsort {

struct DecimalKeySortResult {
  std::vector<std::uint64_t> keys;  // non-decreasing
  KeySpec spec;
  ExtractionReport report;
};

struct DecimalSortResult {
  std::vector<std::string> values;  // rendered at the dataset scale, non-decreasing
  KeySpec spec;
  ExtractionReport report;
};

struct IntegerSortResult {
  std::vector<std::int64_t> values;
  KeySpec spec;
  ExtractionReport report;
};

struct StringSortResult {
  std::vector<std::string> values;  // the original (unpadded) strings
  KeySpec spec;
  ExtractionReport report;
};

// normalize + hash + extract without rendering the keys back to text.
DecimalKeySortResult sort_decimal_keys(std::span<const std::string> values,
                                       std::uint64_t max_cells = kDefaultCellBudget);

// The full decimal pipeline; values come back at the dataset's common scale.
DecimalSortResult sort_decimals(std::span<const std::string> values,
                                std::uint64_t max_cells = kDefaultCellBudget);

// Integers (scale 0); a negative input raises errc::negative_value.
IntegerSortResult sort_integers(std::span<const std::int64_t> values,
                                std::uint64_t max_cells = kDefaultCellBudget);

// Lexicographic sort over a fixed alphabet.
StringSortResult sort_strings(std::span<const std::string> values, const Alphabet& alphabet,
                              std::uint64_t max_cells = kDefaultCellBudget);

// ---- device-pointer overloads (not in the reference) ----------
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

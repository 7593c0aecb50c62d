/*
 * oracle.h — CPU restatement of the Recombinant Sort reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2107_01391_b200/) may link, load or call this code.  It exists
 * so tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
 * check the GPU results against the reference algorithm on the same seeded
 * inputs.
 *
 * Pinning: every function below is cross-checked in tests/test_oracle.py
 * against (a) the golden vectors and known-answer tests of the reference's own
 * suites (proj/tests/*.cpp, proj/tests/python/test_smoke.py) and (b) the
 * reference library itself compiled from /root/reference/proj/src by
 * oracle/Makefile into oracle/_ref/ (see oracle/ref_shim.cpp).
 *
 * Status codes are errc order + 1 (proj/include/recsort/error.hpp:10-23),
 * identical to rs_status in include/recsort_b200.h.
 */
#ifndef RECSORT_ORACLE_H
#define RECSORT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OR_OK = 0,
  OR_PARSE_ERROR = 1,
  OR_NEGATIVE_VALUE = 2,
  OR_NON_FINITE = 3,
  OR_CELL_BUDGET_EXCEEDED = 4,
  OR_SYMBOL_OUT_OF_ALPHABET = 5,
  OR_SPEC_MISMATCH = 6,
  OR_BUFFER_TOO_SMALL = 7,
  OR_RANGE_EXCEEDED = 8,
  OR_OUT_OF_RANGE = 9,
  OR_INVALID_RANGE = 10,
  OR_INSUFFICIENT_DATA = 11,
  OR_INVALID_ARGUMENT = 12,
  OR_ALLOC_FAILED = 99
};

#define OR_DEFAULT_CELL_BUDGET 100000000ULL /* key_model.hpp:16 */

typedef struct or_key_spec {
  uint32_t radix, total_digits, integer_digits;
} or_key_spec;

typedef struct or_report {
  uint64_t written, cells_traversed;
  or_key_spec spec;
} or_report;

/* --- SplitMix64 (splitmix64.hpp:10-35) --------------------------------- */
uint64_t or_sm64_next(uint64_t* state);
double or_sm64_next_unit(uint64_t* state);
uint64_t or_sm64_mix(uint64_t seed, uint64_t index);
/* i-th output of Splitmix64(seed) (0-based), counter-addressed. */
uint64_t or_sm64_at(uint64_t seed, uint64_t i);

/* --- key model (key_model.cpp:38-78, 135-158, 225-263) ------------------ */
uint32_t or_decimal_digit_count(uint64_t v);
int or_checked_pow(uint64_t radix, uint32_t exp, uint64_t* out);
int or_make_key_spec(uint32_t radix, uint32_t total_digits,
                     uint32_t integer_digits, uint64_t max_cells,
                     or_key_spec* out);
int or_float_to_decimal(double x, uint32_t scale, uint64_t* mantissa);

/* --- hashing + extraction cycles (hashing.cpp:27-52, extraction.cpp:5-45) */
int or_sort_keys(const uint64_t* keys, uint64_t n, or_key_spec spec,
                 uint64_t max_cells, uint64_t* out, uint64_t out_capacity,
                 or_report* report);

/* --- facades (sort.cpp:7-77) ------------------------------------------- */
int or_sort_integers_i64(const int64_t* values, uint64_t n,
                         uint64_t max_cells, int64_t* out, or_report* report);
int or_sort_integers_u32(const uint32_t* values, uint64_t n,
                         uint64_t max_cells, uint32_t* out, or_report* report);
/* float_to_decimal(x, scale) per element, then the core on the mantissas
 * with KeySpec{10, lambda+scale, lambda}. */
int or_sort_f64(const double* x, uint64_t n, uint32_t scale,
                uint64_t max_cells, uint64_t* out, or_report* report);
/* strings_to_keys for fixed-width records: record i is chars[i*width ..],
 * length = first NUL or width.  Keys are base-(|alphabet|+1) Horner with
 * pad ordinal 0 (key_model.cpp:225-247). */
int or_strings_to_keys(const uint8_t* chars, uint64_t n, uint32_t width,
                       const char* alphabet, uint64_t max_cells,
                       uint64_t* keys, or_key_spec* spec);
/* Byte-lexicographic sort of fixed-width NUL-padded records: the reference's
 * oracle_sort<std::string> (baselines.hpp:56-60) for records without NULs.
 * Also returns the single-grid report the reference facade would give with
 * an unlimited budget (per-row spans) when report != NULL. */
int or_sort_fixed_strings(const uint8_t* chars, uint64_t n, uint32_t width,
                          const char* alphabet, uint8_t* out,
                          or_report* report);

/* --- stable key/value order (baselines.hpp:24-46, rsort.cpp:133-145) ---- */
int or_radix_sort_lsd_kv_u32(const uint32_t* keys, const uint32_t* vals,
                             uint64_t n, uint32_t* keys_out,
                             uint32_t* vals_out);
/* Single-grid report over already sorted u64 keys for a radix (the per-row
 * span sum of extraction.cpp:16-30; exact by SURVEY F4). */
int or_report_from_sorted(const uint64_t* sorted, uint64_t n, uint32_t radix,
                          uint32_t total_digits, or_report* report);

/* --- seeded config generators (SURVEY 7 "spec gaps") ------------------- */
uint64_t or_config_seed(uint32_t cfg);
void or_gen_u32_mod(uint64_t seed, uint64_t first, uint64_t n, uint64_t bound,
                    uint32_t* out); /* bound == 0: full 32-bit (next >> 32) */
int or_zipf_cdf(uint32_t ranks, double s, double* cdf);
void or_gen_f64_cfg3(uint64_t seed, uint64_t first, uint64_t n,
                     const double* cdf, uint32_t ranks, double* out);
void or_gen_str_cfg4(uint64_t seed, uint64_t first, uint64_t n,
                     uint8_t* out /* n*8 bytes */);

#ifdef __cplusplus
}
#endif
#endif

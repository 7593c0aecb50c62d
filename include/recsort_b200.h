/*
 * recsort_b200.h — C-ABI of the B200-native Recombinant Sort hot path.
 *
 * Every entry point is plain C: device pointers, sizes, a cudaStream_t passed
 * as `void*`, and an rs_status return.  No torch or C++ types cross this
 * boundary.  The C++ facade in include/recsort/sort.hpp (same names as the
 * reference's proj/include/recsort/sort.hpp) and the Python host mirror
 * (paper_2107_01391_b200/__init__.py, same names as proj/python/recsort) are
 * thin layers over these functions.  INTEGRATION.md shows the bindings.
 *
 * Pointer convention: unless a parameter is prefixed h_, it is a DEVICE
 * pointer on the current CUDA device.  Work is enqueued on `stream` (NULL =
 * legacy default stream); calls that return a report synchronise `stream`
 * once at the end to read it back.
 *
 * Errors: rs_status mirrors recsort::errc in declaration order
 * (proj/include/recsort/error.hpp:10-23) shifted by one so that RS_OK == 0,
 * plus CUDA/NCCL failure codes.  Budget checks happen before any device
 * allocation (acceptance.cpp:292-314, c09).  The thread-local message of
 * the last failure is available from rs_last_error().
 */
#ifndef RECSORT_B200_H
#define RECSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rs_status {
  RS_OK = 0,
  RS_PARSE_ERROR = 1,            /* errc::parse_error */
  RS_NEGATIVE_VALUE = 2,         /* errc::negative_value */
  RS_NON_FINITE = 3,             /* errc::non_finite */
  RS_CELL_BUDGET_EXCEEDED = 4,   /* errc::cell_budget_exceeded */
  RS_SYMBOL_OUT_OF_ALPHABET = 5, /* errc::symbol_out_of_alphabet */
  RS_SPEC_MISMATCH = 6,          /* errc::spec_mismatch */
  RS_BUFFER_TOO_SMALL = 7,       /* errc::buffer_too_small */
  RS_RANGE_EXCEEDED = 8,         /* errc::range_exceeded */
  RS_OUT_OF_RANGE = 9,           /* errc::out_of_range */
  RS_INVALID_RANGE = 10,         /* errc::invalid_range */
  RS_INSUFFICIENT_DATA = 11,     /* errc::insufficient_data */
  RS_INVALID_ARGUMENT = 12,      /* errc::invalid_argument */
  RS_CUDA_ERROR = 100,           /* a CUDA runtime call or kernel failed */
  RS_NCCL_ERROR = 101,           /* reserved for the collective layer */
  RS_NO_DEVICE = 102             /* no CUDA device: there is no CPU path */
} rs_status;

#define RS_DEFAULT_CELL_BUDGET 100000000ULL /* key_model.hpp:16 */

/* KeySpec (key_model.hpp:35-46). */
typedef struct rs_key_spec {
  uint32_t radix;
  uint32_t total_digits;
  uint32_t integer_digits;
} rs_key_spec;

/* ExtractionReport (extraction.hpp:12-15) + the KeySpec every facade result
 * carries (sort.hpp:19-41).  For multi-level (MSD) sorts, cells_traversed is
 * the single-grid value the reference would report for the same data with an
 * unlimited budget (sum over occupied leading-digit rows of max-min+1 suffix,
 * SURVEY F4); it does not depend on how the grid was split. */
typedef struct rs_report {
  uint64_t written;
  uint64_t cells_traversed;
  rs_key_spec spec;
} rs_report;

typedef struct rs_options {
  /* Per-grid cell budget; 0 means RS_DEFAULT_CELL_BUDGET. */
  uint64_t max_cells;
  /* Declared decimal width of the key domain (like a radix sort's bit
   * range).  0: derive it from the data with a separate max pass (exactly
   * the reference's sort.cpp:31-40).  >0: count directly into a
   * 10^key_digits grid and derive the exact spec from the max found by the
   * same pass; a key outside the declared width is detected on the device
   * and the sort is redone with the derived width, so the result never
   * depends on the hint. */
  uint32_t key_digits;
  /* 0: reference semantics — a grid above max_cells raises
   *    RS_CELL_BUDGET_EXCEEDED (key_model.cpp:72-76).
   * 1: split such grids with MSD bucket passes on the leading digits and
   *    apply max_cells per bucket grid. */
  uint32_t msd;
} rs_options;

/* ---- library / errors ------------------------------------------------- */
const char* rs_last_error(void);
const char* rs_status_name(rs_status status);       /* errc_name, key_model.cpp:265-281 */
const char* rs_version(void);
/* Frees the calling thread's cached workspaces on every device. */
void rs_release_workspaces(void);

/* ---- instrumentation ---------------------------------------------------
 * Every kernel the library launches is counted (rs_launch_count).  With
 * profiling on, each pass is bracketed by CUDA events recorded on the stream
 * it runs on and its device time accumulated per pass id; reading the totals
 * is valid after the sort returned (the call synchronised its stream). */
enum {
  RS_PASS_MAX = 0, RS_PASS_COUNT = 1, RS_PASS_SCAN = 2, RS_PASS_EMIT = 3,
  RS_PASS_REPORT = 4, RS_PASS_KV_HIST = 5, RS_PASS_KV_SCATTER = 6,
  RS_PASS_MSD_HIST = 7, RS_PASS_MSD_SCATTER = 8, RS_PASS_BUCKET = 9,
  RS_PASS_COPY = 10, RS_PASS_OTHER = 11, RS_PASS_PARTITION = 12, RS_NUM_PASSES = 13
};
uint64_t rs_launch_count(void);
void rs_profile_enable(int on);
void rs_profile_reset(void);
/* Fills ms[RS_NUM_PASSES] (accumulated device milliseconds) and
 * launches[RS_NUM_PASSES]; returns RS_NUM_PASSES. */
int rs_profile_read(double* h_ms, uint64_t* h_launches);
const char* rs_pass_name(int pass);

/* ---- sorts (device pointers) ------------------------------------------ */

/* sort_integers (sort.hpp:52-53, sort.cpp:29-59) for uint32 keys: identity
 * mapper, KeySpec{10, d, d} with d = digits(max).  out needs n slots. */
rs_status rs_sort_u32(const uint32_t* keys, uint64_t n, uint32_t* out,
                      uint64_t out_capacity, const rs_options* opt,
                      rs_report* report, void* stream);

/* sort_integers with the reference's int64 element type; negative inputs
 * raise RS_NEGATIVE_VALUE (sort.cpp:31-37). */
rs_status rs_sort_i64(const int64_t* values, uint64_t n, int64_t* out,
                      uint64_t out_capacity, const rs_options* opt,
                      rs_report* report, void* stream);

/* sort_integers over keys spread across several GPUs of one process
 * ("rs_sort_u32_multi"): shard g = h_keys[g][0 .. h_n[g]) on
 * device h_devices[g].  One max over all shards fixes KeySpec{10, d, d}
 * (sort.cpp:31-40, budget-checked before any grid); every GPU counts its
 * shard, the first GPU gathers and sums the grids over NVLink, cuts the
 * cells into ngpus contiguous ranges of ~total/ngpus keys, and GPU g emits
 * range g into h_out[g] (h_written[g] keys): the concatenation of the
 * outputs in device order is the sorted whole.  The report is the
 * single-grid one.  Fewer than 2^32 keys in total; synchronous. */
rs_status rs_sort_u32_multi(uint32_t ngpus, const int* h_devices, const uint32_t* const* h_keys,
                            const uint64_t* h_n, uint32_t* const* h_out,
                            const uint64_t* h_out_capacity, uint64_t* h_written,
                            const rs_options* opt, rs_report* report);

/* Stable key/value sort of uint32 keys with uint32 payloads.  The reference
 * library has no record API; its stable order is rsort's originals_by_key
 * (rsort.cpp:133-145) == baselines::radix_sort_lsd_by (baselines.hpp:24-46):
 * equal keys keep their input order. */
rs_status rs_sort_u32_kv(const uint32_t* keys, const uint32_t* vals, uint64_t n,
                         uint32_t* keys_out, uint32_t* vals_out,
                         uint64_t out_capacity, const rs_options* opt,
                         rs_report* report, void* stream);

/* float64 decimals: float_to_decimal(x, scale) per element (key_model.cpp:
 * 135-158: shortest round-trip numeral rounded half-up), then KeySpec
 * {10, lambda+scale, lambda}, lambda = digits(max_mantissa / 10^scale)
 * (key_model.cpp:122-124).  Emits the sorted mantissas
 * (DecimalKeySortResult::keys, sort.hpp:19-23).  Bit-identical to the
 * reference for every double (fast IEEE tests on the common domain, an exact
 * shortest-numeral search elsewhere; kernels_f64.cuh).  Errors are the
 * reference's for the first failing element in input order (non_finite,
 * negative_value, cell_budget_exceeded); scale <= 40, and scale > 19 fails
 * as the reference's 10^scale does.  The composition (per-element
 * float_to_decimal, then the grid) is SURVEY 8c's cfg3 oracle. */
rs_status rs_sort_f64(const double* x, uint64_t n, uint32_t scale,
                      uint64_t* mantissas_out, uint64_t out_capacity,
                      const rs_options* opt, rs_report* report, void* stream);

/* float_to_decimal(x[i], scale).mantissa for every element (key_model.cpp:
 * 135-158, DecimalValue::mantissa; the vectorised form of the reference's
 * per-value call): shortest round-trip fixed numeral, rescaled to `scale`
 * places (half up; an unchecked upscale wraps modulo 2^64 as in the
 * reference).  The first failing element (input order) sets the status and
 * the reference's message.  scale <= 40. */
rs_status rs_float_to_decimal(const double* x, uint64_t n, uint32_t scale,
                              uint64_t* mantissas_out, void* stream);

/* sort_strings (sort.hpp:57-60, sort.cpp:61-77) over fixed-width records:
 * record i is chars[i*width .. i*width+width), its string ends at the first
 * NUL byte or at width.  h_alphabet is a host NUL-terminated symbol list
 * (Alphabet, key_model.hpp:93-121); NULL = "abcdefghijklmnopqrstuvwxyz".
 * Output records are the sorted originals, NUL-padded.  Checks in the
 * reference's order: KeySpec{radix, w, w} for the longest string w
 * (make_key_spec: cell budget, radix^w overflow), then the first symbol
 * outside the alphabet.  With rs_options.msd a key space above the budget is
 * sorted by MSD passes over keys packed b bits per ordinal (b = bit length
 * of the alphabet size: 5 for a-z, 6 for <= 63 symbols, 8 for <= 255) when
 * width * b <= 64 (12 a-z characters, 16 of a 15-symbol alphabet, 8 of any
 * byte alphabet); wider records keep the reference's budget error. */
rs_status rs_sort_fixed_str(const uint8_t* chars, uint64_t n, uint32_t width,
                            const char* h_alphabet, uint8_t* out,
                            uint64_t out_capacity, const rs_options* opt,
                            rs_report* report, void* stream);

/* sort_keys (extraction.hpp:31-36, extraction.cpp:34-45): keys already in
 * [0, radix^total_digits) of `spec`; a key outside raises RS_SPEC_MISMATCH
 * (hashing.cpp:31-34). */
rs_status rs_sort_keys(const uint64_t* keys, uint64_t n, rs_key_spec spec,
                       uint64_t* out, uint64_t out_capacity,
                       const rs_options* opt, rs_report* report, void* stream);

/* ---- the reference's lower-level surface (key_model.hpp, hashing.hpp,
 * extraction.hpp), what include/recsort/{key_model,hashing,extraction}.hpp
 * implement over this ABI ---------------------------------------------- */
/* checked_pow / make_key_spec (key_model.hpp:19-51, key_model.cpp:38-78):
 * host geometry with the reference's errors; no device needed. */
rs_status rs_checked_pow(uint64_t radix, uint32_t exp, uint64_t* h_out);
rs_status rs_make_key_spec(uint32_t radix, uint32_t total_digits, uint32_t integer_digits,
                           uint64_t max_cells, rs_key_spec* h_spec);

/* strings_to_keys (key_model.hpp:118-121, key_model.cpp:225-247) over n
 * NUL-padded records of `width` bytes: keys_out[i] = sum ord_j *
 * radix^(w-1-j) at the data width w (longest string, >= 1), pad ordinal 0.
 * Checks in the reference's order: KeySpec{radix, w, w} (budget), then the
 * first symbol outside the alphabet.  *h_spec receives the spec. */
rs_status rs_strings_to_keys(const uint8_t* chars, uint64_t n, uint32_t width, const char* h_alphabet,
                             uint64_t* keys_out, const rs_options* opt, rs_key_spec* h_spec, void* stream);

/* build_count_space without snapshots (hashing.hpp:107-113,
 * hashing.cpp:40-52): counts[radix^total_digits] (uint64, device) receive
 * the multiplicity of every key (CountSpace, hashing.hpp:53-89) and
 * h_row_min / h_row_max (host, `radix` entries each) the TraverseMaps
 * (hashing.hpp:12-48): per leading digit the least / greatest occupied
 * suffix, ~0 / -1 for an untouched row.  The budget is new_space's
 * (hashing.cpp:17-25, checked before anything is allocated); a key outside
 * the spec's key space raises RS_SPEC_MISMATCH. */
rs_status rs_build_count_space(const uint64_t* keys, uint64_t n, rs_key_spec spec, uint64_t max_cells,
                               uint64_t* counts, uint64_t* h_row_min, int64_t* h_row_max, void* stream);

/* extract (extraction.hpp:24-27, extraction.cpp:5-32): the raster scan of
 * every occupied row's span [h_row_min, h_row_max] of a uint64 count grid,
 * emitting each cell's multiplicity until `total` keys (total_inserted) are
 * written.  RS_BUFFER_TOO_SMALL when out_capacity < total (checked first).
 * report->cells_traversed counts the cells the raster visits. */
rs_status rs_extract(const uint64_t* counts, rs_key_spec spec, uint64_t total, const uint64_t* h_row_min,
                     const int64_t* h_row_max, uint64_t* out, uint64_t out_capacity, rs_report* report,
                     void* stream);

/* ---- decimal text ------------------------------------ */
/* sort_decimal_keys (sort.hpp:44-47, sort.cpp:7-14) over a device string
 * column in Arrow layout: numeral i is chars[offsets[i] .. offsets[i+1]),
 * offsets has n+1 entries.  Parsing follows parse_decimal
 * (key_model.cpp:80-105) and normalize_dataset (key_model.cpp:107-133) on the
 * GPU: the error is that of the first failing numeral (the one the
 * reference's sequential loop stops at), with the reference's message.
 * keys_out[n] receive the sorted mantissas at the dataset scale; report->spec
 * is the dataset KeySpec {10, lambda + scale, lambda}. */
rs_status rs_sort_decimal_strings(const char* chars, const uint64_t* offsets, uint64_t n,
                                  uint64_t* keys_out, uint64_t out_capacity,
                                  const rs_options* opt, rs_report* report, void* stream);

/* parse_decimal (key_model.hpp:78-80, key_model.cpp:80-105) for every
 * numeral of a device string column: mantissas[i] and scales[i] (fractional
 * digits).  The error is that of the first failing numeral in input order. */
rs_status rs_parse_decimals(const char* chars, const uint64_t* offsets, uint64_t n, uint64_t* mantissas,
                            uint32_t* scales, void* stream);

/* normalize_dataset (key_model.hpp:82-87, key_model.cpp:107-133): keys_out[i]
 * = mantissa_i * 10^(scale - scale_i) at the dataset's common scale;
 * *h_spec = {10, lambda + scale, lambda}. */
rs_status rs_normalize_decimal_strings(const char* chars, const uint64_t* offsets, uint64_t n,
                                       uint64_t* keys_out, const rs_options* opt, rs_key_spec* h_spec,
                                       void* stream);

/* format_scaled_decimal (key_model.cpp:170-180) / reconstruct_value for n
 * keys at `scale` (<= 19), into a device string column: out_offsets[0..n]
 * (n+1 entries) and out_chars.  *h_chars_needed (host) receives the total
 * length; RS_BUFFER_TOO_SMALL when it exceeds out_chars_capacity (the
 * offsets are written either way). */
rs_status rs_format_decimals(const uint64_t* keys, uint64_t n, uint32_t scale, char* out_chars,
                             uint64_t out_chars_capacity, uint64_t* out_offsets,
                             uint64_t* h_chars_needed, void* stream);

/* ---- host-buffer entry points (H2D / sort / D2H inside one call) -------- */
/* Same semantics as rs_sort_u32 / rs_sort_u32_kv on HOST buffers: one
 * host->device copy of the input, the device sort, one device->host copy of
 * the output, all on `stream`, returning after the stream synchronises.  The
 * device staging buffers belong to the call (no pass of the sort reuses
 * them).  A sort cannot emit before it has counted every key, so within one
 * call the copies do not overlap; callers sorting a stream of batches overlap
 * consecutive calls on two streams (H2D of batch k+1 beside D2H of batch k,
 * PCIe being full duplex), as bench.py's e2e figure does. */
rs_status rs_sort_u32_host(const uint32_t* h_keys, uint64_t n, uint32_t* h_out,
                           const rs_options* opt, rs_report* report, void* stream);
rs_status rs_sort_u32_kv_host(const uint32_t* h_keys, const uint32_t* h_vals,
                              uint64_t n, uint32_t* h_keys_out,
                              uint32_t* h_vals_out, const rs_options* opt,
                              rs_report* report, void* stream);

/* ---- phase API (multi-GPU orchestration) -------------------- */
/* Multi-GPU stable key/value placement ("within a cell, rank =
 * sum of earlier ranks' counts + local rank"): keys/vals hold this rank's
 * records in stable local order; record i with key k is written at
 * h_dst_keys[o] / h_dst_vals[o] + cell_off[k] + i, o = cell_owner[k] — device
 * addresses of the owners' output slices (peer buffers over NVLink), so the
 * placement is the exchange and the slices come out in the reference's
 * unique stable order (radix_sort_lsd_by, baselines.hpp:24-46).  cell_off
 * (int64) and cell_owner (uint8) are device arrays of `cells` entries. */
rs_status rs_kv_place_u32(const uint32_t* keys, const uint32_t* vals, uint64_t n,
                          const int64_t* cell_off, const uint8_t* cell_owner, uint64_t cells,
                          const uint64_t* h_dst_keys, const uint64_t* h_dst_vals,
                          uint32_t ranks, void* stream);

/* Count uint32 keys into a caller-owned grid of `cells` uint32 counters
 * (overwritten; the same counting pass as rs_sort_u32).  Keys >= cells are
 * not counted; h_max, if not NULL, receives the maximum key (host pointer;
 * the call then synchronises). */
rs_status rs_count_u32(const uint32_t* keys, uint64_t n, uint32_t* counts,
                       uint64_t cells, uint32_t* h_max, void* stream);
/* Emit the run-length expansion of cells [cell_lo, cell_hi) of a (globally
 * reduced) count grid into out, which must hold exactly the keys of that
 * cell range.  Keys are cell indices + key_base. */
rs_status rs_emit_u32(const uint32_t* counts, uint64_t cells, uint64_t cell_lo,
                      uint64_t cell_hi, uint32_t key_base, uint32_t* out,
                      uint64_t out_capacity, uint64_t* h_written, void* stream);

/* The small-grid sharding's emit in one call: over the global
 * (all-reduced) grid, the cells are cut into `parts` contiguous ranges of
 * about total/parts keys, on cell boundaries (cut r, 1 <= r < parts, = 1 + the
 * cell whose inclusive prefix first reaches ceil(r * total / parts);
 * dist.cell_ranges), and range `part` is emitted into out (its keys in
 * order; *h_written, host, receives how many).  h_cells (host, optional)
 * receives the range [lo, hi). */
rs_status rs_emit_part_u32(const uint32_t* counts, uint64_t cells, uint32_t part, uint32_t parts,
                           uint32_t* out, uint64_t out_capacity, uint64_t* h_written,
                           uint64_t* h_cells, void* stream);
/* Histogram of key / divisor into `buckets` uint64 counters (MSD splitters). */
rs_status rs_bucket_hist_u32(const uint32_t* keys, uint64_t n, uint64_t divisor,
                             uint64_t* hist, uint32_t buckets, void* stream);
/* Stable partition of keys into `parts` ranges of buckets (bucket =
 * key/divisor; part p holds buckets [bounds[p], bounds[p+1]) ); h_counts
 * receives the per-part key counts (host pointer). */
rs_status rs_partition_u32(const uint32_t* keys, uint64_t n, uint64_t divisor,
                           const uint32_t* h_bounds, uint32_t parts,
                           uint32_t* out, uint64_t* h_counts, void* stream);

/* The two passes of rs_partition_u32 apart, for the multi-GPU exchange of
 * SURVEY 8e (wide keys): per-part counts of this rank's keys, then the
 * scatter with part p written at h_dst[p] + h_offsets[p] + rank-in-part —
 * h_dst[p] a device address (a peer GPU's receive buffer mapped over NVLink,
 * e.g. torch symmetric memory), so the partition kernel itself performs the
 * all-to-all.  h_dst / h_offsets: `parts` host values. */
rs_status rs_part_counts_u32(const uint32_t* keys, uint64_t n, uint64_t divisor,
                             const uint32_t* h_bounds, uint32_t parts,
                             uint64_t* h_counts, void* stream);
rs_status rs_partition_u32_to(const uint32_t* keys, uint64_t n, uint64_t divisor,
                              const uint32_t* h_bounds, uint32_t parts,
                              const uint64_t* h_dst, const uint64_t* h_offsets,
                              void* stream);

/* ---- synthetic config inputs (bench/test utility, not part of the sort) --
 * Counter-addressed SplitMix64 (splitmix64.hpp:14-19): element i
 * of Splitmix64(seed).  Bit-identical to the host generators in oracle/. */
rs_status rs_gen_u32(uint64_t seed, uint64_t first, uint64_t n, uint64_t bound,
                     uint32_t* out, void* stream); /* bound 0 = next()>>32 */
rs_status rs_gen_iota_u32(uint64_t first, uint64_t n, uint32_t* out, void* stream);
rs_status rs_gen_f64_cfg3(uint64_t seed, uint64_t first, uint64_t n,
                          const double* zipf_cdf, uint32_t ranks, double* out,
                          void* stream);
rs_status rs_gen_str_cfg4(uint64_t seed, uint64_t first, uint64_t n, uint8_t* out,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RECSORT_B200_H */

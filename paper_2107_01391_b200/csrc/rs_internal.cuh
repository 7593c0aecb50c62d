// rs_internal.cuh — shared host/device plumbing for the B200 hot path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "recsort_b200.h"

namespace rsb {

// ---------------------------------------------------------------- errors
struct Failure {
  rs_status status;
  std::string message;
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(rs_status st, const std::string& msg) {
  throw Failure{st, msg};
}

#define RS_CUDA(call)                                                     \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      ::rsb::fail(RS_CUDA_ERROR, std::string(#call) + ": " +              \
                                     cudaGetErrorString(e_));             \
  } while (0)

#define RS_LAUNCH_CHECK() RS_CUDA(cudaGetLastError())

// Runs f, mapping Failure / bad_alloc to an rs_status and a message.
template <class F>
rs_status guarded(F&& f) {
  try {
    f();
    return RS_OK;
  } catch (const Failure& e) {
    set_last_error(e.message);
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return RS_CUDA_ERROR;
  }
}

// -------------------------------------------------------- host arithmetic
constexpr uint64_t kMaxU64 = ~uint64_t{0};

inline uint32_t digit_count(uint64_t v) {  // decimal_digit_count, key_model.cpp:51-58
  uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

// checked_pow (key_model.cpp:38-49); fails with the reference's code.
inline uint64_t checked_pow(uint64_t radix, uint32_t exp) {
  uint64_t r = 1;
  for (uint32_t i = 0; i < exp; ++i) {
    if (r > kMaxU64 / radix)
      fail(RS_CELL_BUDGET_EXCEEDED, "key space " + std::to_string(radix) + "^" +
                                        std::to_string(exp) + " overflows 64 bits");
    r *= radix;
  }
  return r;
}

// make_key_spec (key_model.cpp:64-78): geometry + budget, before allocation.
inline rs_key_spec make_key_spec(uint32_t radix, uint32_t total, uint32_t integer,
                                 uint64_t max_cells) {
  if (radix < 2) fail(RS_INVALID_ARGUMENT, "radix must be at least 2");
  if (total < 1) fail(RS_INVALID_ARGUMENT, "need at least one digit");
  if (integer > total) fail(RS_INVALID_ARGUMENT, "integer digits exceed total digits");
  const uint64_t cells = checked_pow(radix, total);
  if (cells > max_cells)
    fail(RS_CELL_BUDGET_EXCEEDED, "key space needs " + std::to_string(cells) +
                                      " cells, budget is " + std::to_string(max_cells));
  return rs_key_spec{radix, total, integer};
}

inline uint64_t budget_of(const rs_options* opt) {
  return (opt && opt->max_cells) ? opt->max_cells : RS_DEFAULT_CELL_BUDGET;
}

// ------------------------------------------------------------ device side
// Counters the passes share; one per workspace, reset per sort.
struct DevStats {
  unsigned long long max_key;    // atomicMax over mapped keys
  unsigned long long n_occupied; // occupied cells (written by the last scan tile)
  unsigned long long total;      // keys counted (written by the last scan tile)
  unsigned int overflow;         // a key fell outside the grid
  unsigned int flags;            // kFlag* bits
  unsigned int tile_counter;     // dynamic tile ids for the look-back scan
  unsigned int long_spans;        // hot cells spanning >= 3 emit tiles (k_scan_cells -> k_fill_spans)
  unsigned long long cells_traversed;  // report (per-row spans)
  unsigned long long report_digits;    // total_digits found by the report kernel
};

// kFlagBudget: float_to_decimal raised cell_budget_exceeded (mantissa or 10^e overflow)
enum : unsigned { kFlagNegative = 1u, kFlagNonFinite = 2u, kFlagDomain = 4u, kFlagBudget = 8u };

// Per-(device, stream) scratch cache.  Buffers only grow; each stream owns
// its own so concurrent calls on different streams never share scratch.
struct Workspace {
  int device = -1;
  cudaStream_t stream = nullptr;
  static constexpr int kSlots = 25;
  void* buf[kSlots] = {};
  size_t cap[kSlots] = {};
  DevStats* stats = nullptr;   // device
  DevStats* h_stats = nullptr; // pinned host mirror
  // a second stream for work that overlaps the main one inside a call (the
  // report beside the emit), forked and joined with the two events
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  void ensure_side();

  void* raw(int slot, size_t bytes);
  template <class T>
  T* get(int slot, size_t count) {
    return static_cast<T*>(raw(slot, count * sizeof(T) + 16));
  }
  void release();
};

Workspace& workspace_for(cudaStream_t stream);

// ------------------------------------------------------ instrumentation
// Pass bracket: counts launches always; with profiling on, records a CUDA
// event pair on the pass's stream and queues it for accumulation at the
// next synchronisation point (flush_profile).
void note_launch(int pass, int launches = 1);
struct PassTimer {
  int pass;
  cudaStream_t stream;
  cudaEvent_t a = nullptr, b = nullptr;
  int launches;
  PassTimer(int p, cudaStream_t s, int nl = 1);
  ~PassTimer();
};
void flush_profile();
void ensure_device();

// Slot assignment (fixed so phases can hand buffers to each other).
enum Slot : int {
  kSlotCounts = 0,   // grid counters
  kSlotOccCell = 1,  // compacted occupied cell ids
  kSlotOccEnd = 2,   // inclusive key prefix per occupied cell
  kSlotTileDesc = 3, // look-back descriptors
  kSlotTileFirst = 4,// first occupied cell of each emit tile
  kSlotTmpKeys = 5,  // key/value ping-pong or MSD buckets
  kSlotTmpVals = 6,
  kSlotHist = 7,     // digit histograms
  kSlotMapped = 8,   // mapped keys (f64 / strings)
  kSlotMisc = 9,
  kSlotTmpKeys2 = 10,
  kSlotTmpVals2 = 11,
  kSlotCtaHist = 12,    // per-CTA outer histograms [B][G]
  kSlotCtaOff = 13,     // their exclusive scan
  kSlotBucketStart = 14,
  kSlotLows = 15,       // partitioned inner digits (uint16)
  kSlotDesc2 = 16,      // look-back descriptors of the second scan
  kSlotScratch = 17,
  kSlotAlphabet = 18,   // string ordinal / symbol tables
  kSlotExtra1 = 19,     // MSD radix-leaf list
  kSlotSpans = 20,      // long emit-tile spans of hot cells
  kSlotMisc2 = 21,      // packed string keys (MSD)
  kSlotCounts64 = 22,   // 64-bit grid of inputs with 2^32 keys or more
  kSlotHostIn = 23,     // device staging of the host-buffer entry points (no internal pass uses it)
  kSlotHostOut = 24,
};

}  // namespace rsb

// capi.cu — the extern "C" boundary (include/recsort_b200.h) and the host
// orchestration of the single-grid passes.  No CPU path exists: without a
// CUDA device every entry point returns RS_NO_DEVICE.
#include <cuda_runtime.h>

#include <charconv>
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "kernels_grid.cuh"
#include "kernels_kv.cuh"
#include "kernels_two_level.cuh"
#include "kernels_partition_ws.cuh"
#include "kernels_partition_direct.cuh"
#include "kernels_msd.cuh"
#include "kernels_msd_engine.cuh"
#include "kernels_decimal.cuh"
#include "recsort_b200.h"
#include "rs_internal.cuh"

namespace rsb {

// ------------------------------------------------------------- errors
namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// ------------------------------------------------------ instrumentation
namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_profile{0};
std::mutex g_prof_mutex;
double g_ms[RS_NUM_PASSES] = {};
uint64_t g_pass_launches[RS_NUM_PASSES] = {};
std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> g_pending;
}  // namespace

void note_launch(int pass, int launches) {
  g_launches += launches;
  std::lock_guard<std::mutex> lock(g_prof_mutex);
  g_pass_launches[pass] += launches;
}

PassTimer::PassTimer(int p, cudaStream_t s, int nl) : pass(p), stream(s), launches(nl) {
  if (g_profile.load()) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, stream);
  }
}

PassTimer::~PassTimer() {
  note_launch(pass, launches);
  if (a) {
    cudaEventRecord(b, stream);
    std::lock_guard<std::mutex> lock(g_prof_mutex);
    g_pending.push_back({pass, {a, b}});
  }
}

void flush_profile() {
  std::lock_guard<std::mutex> lock(g_prof_mutex);
  for (auto& e : g_pending) {
    float ms = 0.f;
    cudaEventSynchronize(e.second.second);
    cudaEventElapsedTime(&ms, e.second.first, e.second.second);
    g_ms[e.first] += ms;
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  g_pending.clear();
}

// --------------------------------------------------------- workspaces
void* Workspace::raw(int slot, size_t bytes) {
  if (cap[slot] < bytes) {
    if (buf[slot]) RS_CUDA(cudaFreeAsync(buf[slot], stream));
    buf[slot] = nullptr;
    cap[slot] = 0;
    const size_t want = bytes + bytes / 8;  // grow with headroom
    RS_CUDA(cudaMallocAsync(&buf[slot], want, stream));
    cap[slot] = want;
  }
  return buf[slot];
}

void Workspace::release() {
  for (int i = 0; i < kSlots; ++i) {
    if (buf[i]) cudaFreeAsync(buf[i], stream);
    buf[i] = nullptr;
    cap[i] = 0;
  }
  if (stats) cudaFree(stats);
  if (h_stats) cudaFreeHost(h_stats);
  stats = nullptr;
  h_stats = nullptr;
  if (side) cudaStreamDestroy(side);
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
  side = nullptr;
  fork = join = nullptr;
}

void Workspace::ensure_side() {
  if (side) return;
  int lo = 0, hi = 0;  // the highest priority: its small CTAs start ahead of the main stream's waiting ones
  RS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  RS_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
  RS_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  RS_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
}

namespace {
std::mutex g_ws_mutex;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;
}  // namespace

void ensure_device() {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    fail(RS_NO_DEVICE, "no CUDA device is visible; recsort_b200 has no CPU path");
}

Workspace& workspace_for(cudaStream_t stream) {
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  Workspace*& w = g_ws[{dev, stream}];
  if (!w) {
    w = new Workspace();
    w->device = dev;
    w->stream = stream;
    RS_CUDA(cudaMalloc(&w->stats, sizeof(DevStats)));
    RS_CUDA(cudaMallocHost(&w->h_stats, sizeof(DevStats)));
  }
  return *w;
}

// The dynamic shared memory limit of a kernel, raised once per (kernel,
// device): function attributes belong to a device's context, so a process
// driving several GPUs (rs_sort_u32_multi) sets them on each.
void set_smem(const void* fn, size_t bytes) {
  int dev = 0;
  RS_CUDA(cudaGetDevice(&dev));
  static std::mutex m;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lock(m);
  size_t& cur = done[{fn, dev}];
  if (cur >= bytes) return;
  RS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  cur = bytes;
}
template <class F>
void set_smem(F* fn, size_t bytes) {
  set_smem(reinterpret_cast<const void*>(fn), bytes);
}

int sm_count() {
  static int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return sms;
}

// k_report: one warp per leading digit, at most 32 warps
unsigned report_threads(uint32_t radix) { return 32u * (radix < 32 ? (radix ? radix : 1) : 32); }

size_t smem_optin() {  // opt-in dynamic shared memory per block
  static size_t b = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v > 0 ? static_cast<size_t>(v) : static_cast<size_t>(232448);
  }();
  return b;
}

// Persistent-style grid for streaming passes: up to `per_sm` CTAs per SM,
// never more than there are 16-byte vectors to read.
unsigned stream_grid(uint64_t n_elems, int elems_per_cta, int per_sm = 8) {
  const uint64_t want = (n_elems + elems_per_cta - 1) / elems_per_cta;
  const uint64_t cap = (uint64_t)sm_count() * per_sm;
  return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

void reset_stats(Workspace& ws) {
  RS_CUDA(cudaMemsetAsync(ws.stats, 0, sizeof(DevStats), ws.stream));
}

void pull_stats(Workspace& ws) {
  RS_CUDA(cudaMemcpyAsync(ws.h_stats, ws.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, ws.stream));
  RS_CUDA(cudaStreamSynchronize(ws.stream));
}

void check_flags(unsigned flags) {
  if (flags & kFlagNonFinite) fail(RS_NON_FINITE, "value is not finite");
  if (flags & kFlagNegative) fail(RS_NEGATIVE_VALUE, "negative values are not supported");
  if (flags & kFlagBudget) fail(RS_CELL_BUDGET_EXCEEDED, "a value's numeral exceeds every cell budget");
}

// ---------------------------------------------------------------- passes
template <class Map>
unsigned long long device_max(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, bool check = true) {
  reset_stats(ws);
  {
    PassTimer pt_(RS_PASS_MAX, ws.stream);
    k_max<Map><<<stream_grid(n, kThreads * 8), kThreads, 0, ws.stream>>>(in, n, map, ws.stats);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
  if (check) check_flags(ws.h_stats->flags);
  return ws.h_stats->max_key;
}

// ------------------------------------------------------ float64 mapping
template <bool G>
MapF64T<G> make_map_f64(uint32_t scale) {
  // the fast tests need 10^(scale+2) * x < 2^53 (scale <= 15); above that
  // every element leaves the fast domain (limit -1)
  const bool fast = scale <= 15;
  const double P = fast ? static_cast<double>(checked_pow(10, scale)) : 1.0;
  const double limit = fast ? 9007199254740992.0 / 100.0 : -1.0;
  const double tiny = fast ? 1.0000001 * std::pow(10.0, -static_cast<double>(scale + 3)) : 0.0;
  MapF64T<G> m{P, limit, tiny, scale, 0, 0, 0, ~0ull};
  if (fast) {
    // the integer fast path tests bit patterns: positive doubles order as
    // their bits, so x * P < limit <=> bits(x) < bits(xlim) for the least
    // such xlim (found from limit / P by stepping, exact IEEE products)
    double xl = limit / P;
    while (xl * P >= limit) xl = std::nextafter(xl, 0.0);
    while (xl * P < limit) xl = std::nextafter(xl, INFINITY);
    std::memcpy(&m.xlim_bits, &xl, 8);
    std::memcpy(&m.tiny_bits, &tiny, 8);
    m.Pi = checked_pow(10, scale);
    m.zero_bits = 0;
  }
  return m;
}
constexpr unsigned kF64Errors = kFlagNegative | kFlagNonFinite | kFlagBudget;

// The first failing element in input order (the one the reference's
// sequential float_to_decimal loop stops at).
__global__ void k_f64_first_error(const double* __restrict__ x, uint64_t n, MapF64G map,
                                  unsigned long long* first) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned fl = 0;
    (void)map(x[i], fl);
    if (fl) atomicMin(first, static_cast<unsigned long long>(i));
  }
}

// The reference's error for x (key_model.cpp:135-158): non_finite, negative,
// or cell_budget_exceeded from parse_decimal / checked_pow on x's shortest
// fixed numeral.  Host-side formatting of the one failing element's message
// (std::to_chars as the reference); the values themselves never come here.
[[noreturn]] void fail_f64(double x, uint32_t scale) {
  if (!std::isfinite(x)) fail(RS_NON_FINITE, "value is not finite");
  if (x < 0.0) fail(RS_NEGATIVE_VALUE, "negative values are not supported");
  if (std::signbit(x)) x = 0.0;
  char buf[512];
  const auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::fixed);
  const std::string text(buf, res.ptr);
  unsigned long long M = 0;
  uint32_t F = 0;
  bool frac = false;
  for (const char ch : text) {
    if (ch == '.') {
      frac = true;
      continue;
    }
    const unsigned d = static_cast<unsigned>(ch - '0');
    if (M > (~0ull - d) / 10)
      fail(RS_CELL_BUDGET_EXCEEDED, "numeral '" + text + "' has more digits than any cell budget admits");
    M = M * 10 + d;
    F += frac ? 1 : 0;
  }
  const uint32_t e = F <= scale ? scale - F : F - scale;
  if (e <= 19) fail(RS_CUDA_ERROR, "float_to_decimal: device flagged " + text + " but it maps");
  fail(RS_CELL_BUDGET_EXCEEDED, "key space 10^" + std::to_string(e) + " overflows 64 bits");
}

// After a pass whose flags hold no kFlagDomain: the first element error.
void check_f64(Workspace& ws, const double* x, uint64_t n, uint32_t scale) {
  if (!(ws.h_stats->flags & kF64Errors)) return;
  const MapF64G map = make_map_f64<true>(scale);
  auto* first = ws.get<unsigned long long>(kSlotScratch, 4);
  RS_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), ws.stream));
  k_f64_first_error<<<stream_grid(n, kThreads * 8), kThreads, 0, ws.stream>>>(x, n, map, first);
  RS_LAUNCH_CHECK();
  unsigned long long i = 0;
  RS_CUDA(cudaMemcpyAsync(&i, first, sizeof(i), cudaMemcpyDeviceToHost, ws.stream));
  RS_CUDA(cudaStreamSynchronize(ws.stream));
  if (i >= n) fail(RS_CUDA_ERROR, "float_to_decimal: flagged element not found");
  double xi = 0.0;
  RS_CUDA(cudaMemcpy(&xi, x + i, sizeof(double), cudaMemcpyDeviceToHost));
  fail_f64(xi, scale);
}

// out[i] = float_to_decimal(x[i], scale).mantissa: the fast tests, the exact
// search for the keys they cannot decide
template <class Map>
__global__ void __launch_bounds__(kThreads) k_f64_map_u64(const double* __restrict__ x, uint64_t n, Map map,
                                                          unsigned long long* __restrict__ out, DevStats* st) {
  unsigned flags = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = __ldcs(x + i);
    out[i] = map(v, flags);
  }
  flags = warp_or(flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&st->flags, flags);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

// Exclusive scan of `count` uint32 values (decoupled look-back); the grand
// total lands in *total (device).
void exscan_u32(Workspace& ws, const uint32_t* in, uint64_t count, uint32_t* out,
                unsigned long long* total) {
  const uint32_t tiles = static_cast<uint32_t>((count + kScanTile - 1) / kScanTile);
  auto* desc = ws.get<unsigned long long>(kSlotDesc2, tiles + 1ull);
  RS_CUDA(cudaMemsetAsync(desc, 0, (tiles + 1ull) * sizeof(unsigned long long), ws.stream));
  auto* ticket = reinterpret_cast<unsigned*>(desc + tiles);
  PassTimer pt_(RS_PASS_SCAN, ws.stream);
  k_exscan_u32<<<tiles, kThreads, 0, ws.stream>>>(in, count, out, desc, ticket, total, tiles);
  RS_LAUNCH_CHECK();
}

// floor(x / d) == (x * magic) >> shift for every 32-bit x, with magic < 2^32
// so the product is one 32x32->64 multiply (exact when the rounding excess
// magic*d - 2^shift stays below 2^(shift-32)).
bool div_magic32(uint64_t d, unsigned long long& magic, uint32_t& shift) {
  if (d == 1) {
    magic = 1;
    shift = 0;
    return true;
  }
  for (uint32_t L = 32; L < 64; ++L) {
    const unsigned __int128 p = (unsigned __int128)1 << L;
    const unsigned __int128 m = (p + d - 1) / d;
    if (m >= ((unsigned __int128)1 << 32)) break;
    if (m * d - p < ((unsigned __int128)1 << (L - 32))) {
      magic = static_cast<unsigned long long>(m);
      shift = L;
      return true;
    }
  }
  return false;
}

// Which partition kernel a two-level count uses.  The warp-specialised kernel
// (kernels_partition_ws.cuh) is the faster one on keys as the caller gives
// them (cfg2: 0.53 vs 0.575 ms at 2^28; the same keys as int64: 0.73 vs
// 0.93 ms); the TMA-fed kernel, whose lane replicas absorb a hot bucket, on
// cfg3's Zipf-skewed mapped cells (0.64 vs ~0.97 ms; profiles/r02_summary.md).
template <class Map>
bool use_ws_partition(bool mapped) {
  return !mapped;
}

// Geometry of the two-level split: ~10^4 inner cells per outer bucket
// (10^6 = 100 x 10^4).  Few outer buckets keep each tile's bucket runs long
// (~40 keys per 4096-key tile); 10^4 inner counters (40 KB) still fit a
// shared histogram.
template <class Map>
bool plan_two_level(uint64_t cells, uint64_t n, TwoLevel& t, bool ws) {
  if (cells <= kSmemCellsMax || cells > 0xFFFFFFFFull || n >= 0x7FFFFFFFull * 16) return false;
  uint64_t B = (cells + 9999) / 10000;
  if (B > kTlMaxBuckets) B = kTlMaxBuckets;
  const uint64_t S = (cells + B - 1) / B;
  if (S > kTlMaxInner) return false;
  t.cells = cells;
  t.S = static_cast<uint32_t>(S);
  t.negS = 0u - t.S;
  t.B = static_cast<uint32_t>((cells + S - 1) / S);
  if (!div_magic32(S, t.magic, t.shift) || t.shift < 32) return false;  // S == 1: never (cells > smem grid)
  t.T = static_cast<uint32_t>((n + kTlTile - 1) / kTlTile);
  // CTAs per SM of each partition kernel, once per mapper (one device type per process)
  static const int per_sm_tma = [] {
    int b = 0;
    set_smem(k_page_partition_tma<Map>, page_tma_smem<Map>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_page_partition_tma<Map>, kTlThreads, page_tma_smem<Map>());
    return b < 1 ? 1 : b;
  }();
  static const int per_sm_ws = [] {
    int b = 0;
    constexpr uint32_t kIn = sizeof(typename Map::In);
    set_smem(k_page_partition_ws<Map>, page_ws_smem(256, kIn));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_page_partition_ws<Map>, kWsThreads, page_ws_smem(100, kIn));
    return b < 1 ? 1 : b;
  }();
  uint64_t G = (uint64_t)sm_count() * (ws ? per_sm_ws : per_sm_tma);  // one persistent wave
  if (G > t.T) G = t.T;
  t.G = static_cast<uint32_t>(G);
  const uint64_t tiles_per = (t.T + G - 1) / G;
  // entries per tile <= kTlTile + 7 pads per bucket run (uint32 partition),
  // plus one partly filled page per bucket
  t.pages_per_cta = static_cast<uint32_t>((tiles_per * (kTlTile + 7ull * t.B) + kPage - 1) / kPage + t.B);
  // groups of ~16*S keys keep the per-group flush of S counters small
  t.group_pages = static_cast<uint32_t>(std::min<uint64_t>(kMaxGroupPages, std::max<uint64_t>(128, 16ull * S / kPage)));
  return true;
}

template <class Map>
void two_level_count(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, const TwoLevel& t0,
                     uint32_t* counts, bool use_ws) {
  const bool al = aligned16(in);
  const bool direct = al && t0.B <= kDirMaxBuckets;
  TwoLevel t = t0;
  if (direct && t.G != 2u * sm_count()) {  // the direct partition: two CTAs per SM, one persistent wave
    t.G = static_cast<uint32_t>(std::min<uint64_t>(2ull * sm_count(), t.T));
    const uint64_t tiles_per = (t.T + t.G - 1) / t.G;
    t.pages_per_cta = static_cast<uint32_t>((tiles_per * (kTlTile + 7ull * t.B) + kPage - 1) / kPage + t.B);
  }
  const uint64_t P = (uint64_t)t.G * t.pages_per_cta;
  const uint64_t bg = (uint64_t)t.B * t.G;
  auto* pages = ws.get<uint16_t>(kSlotLows, P * kPage);
  auto* page_bucket = ws.get<uint16_t>(kSlotBucketStart, P);
  auto* page_fill = ws.get<uint16_t>(kSlotTmpVals2, P);
  auto* pc_bm = ws.get<uint32_t>(kSlotCtaHist, bg);
  auto* po_bm = ws.get<uint32_t>(kSlotCtaOff, bg);
  auto* list = ws.get<uint32_t>(kSlotTmpKeys2, P);
  auto* total = ws.get<unsigned long long>(kSlotScratch, 4);
  auto* work = ws.get<uint32_t>(kSlotMisc, t.B + 1ull);
  const size_t smem = kPagePartitionSmem(t.B);
  if (smem > 48 * 1024) set_smem(k_page_partition<Map>, smem);
  // zeroed before the partition: keys whose staging range is full are counted straight into it
  RS_CUDA(cudaMemsetAsync(counts, 0, t.cells * sizeof(uint32_t), ws.stream));
  {
    PassTimer pt_(RS_PASS_PARTITION, ws.stream);
    bool launched = false;
    if constexpr (!map_first<Map>::value) {  // (mapped float64 cells arrive as MapU32)
      if (direct) {  // keys straight into shared page chunks, TMA bulk-stored
        launched = true;
        if (use_ws) {
          set_smem(k_page_partition_direct<Map>, page_dir_smem(t.B));
          k_page_partition_direct<Map><<<t.G, kDirThreads, page_dir_smem(t.B), ws.stream>>>(
              in, n, map, t, pages, page_bucket, page_fill, pc_bm, counts, ws.stats);
        } else {  // mapped float64 cells (cfg3: a Zipf-hot bucket): the variant that counts a hot bucket in place
          set_smem(k_page_partition_direct<Map, true>, page_dir_hot_smem(t.B, t.S));
          k_page_partition_direct<Map, true><<<t.G, kDirThreads, page_dir_hot_smem(t.B, t.S),
                                               ws.stream>>>(in, n, map, t, pages, page_bucket, page_fill, pc_bm,
                                                            counts, ws.stats);
        }
      }
    }
    if (launched) {
    } else if (al && t.B <= 256 && use_ws) {  // warp-specialised: rankers + page-store warps
      set_smem(k_page_partition_ws<Map>, page_ws_smem(t.B, sizeof(typename Map::In)));
      k_page_partition_ws<Map><<<t.G, kWsThreads, page_ws_smem(t.B, sizeof(typename Map::In)), ws.stream>>>(
          in, n, map, t, pages, page_bucket, page_fill, pc_bm, counts, ws.stats);
    } else if (al && t.B <= 256) {  // TMA-fed tiles, bulk-stored pages
      set_smem(k_page_partition_tma<Map>, page_tma_smem<Map>());
      k_page_partition_tma<Map><<<t.G, kTlThreads, page_tma_smem<Map>(), ws.stream>>>(
          in, n, map, t, pages, page_bucket, page_fill, pc_bm, ws.stats);
    } else {
      k_page_partition<Map><<<t.G, kTlThreads, smem, ws.stream>>>(in, n, map, t, al, pages, page_bucket,
                                                                  page_fill, pc_bm, ws.stats);
    }
    RS_LAUNCH_CHECK();
  }
  if (bg <= kPageScanMax && t.B <= (uint32_t)kPageScanThreads) {  // one CTA: scan + work list
    PassTimer pt_(RS_PASS_SCAN, ws.stream, 2);
    k_page_scan<<<1, kPageScanThreads, 0, ws.stream>>>(pc_bm, static_cast<uint32_t>(bg), po_bm, total, t, work);
    RS_LAUNCH_CHECK();
    k_page_list<<<t.G, 256, t.B * sizeof(uint32_t), ws.stream>>>(page_bucket, po_bm, pc_bm, t, list);
    RS_LAUNCH_CHECK();
  } else {
    exscan_u32(ws, pc_bm, bg, po_bm, total);
    PassTimer pt_(RS_PASS_SCAN, ws.stream, 2);
    k_page_list<<<t.G, 256, t.B * sizeof(uint32_t), ws.stream>>>(page_bucket, po_bm, pc_bm, t, list);
    RS_LAUNCH_CHECK();
    k_page_work<<<1, kTlMaxBuckets, 0, ws.stream>>>(po_bm, total, t, work);
    RS_LAUNCH_CHECK();
  }
  const uint64_t max_groups = P / t.group_pages + t.B + 1;
  const size_t cnt_smem = (t.S + 1) * sizeof(uint32_t);  // + the dump bin of pad entries
  if (cnt_smem > 48 * 1024) set_smem(k_page_count, cnt_smem);
  {
    PassTimer pt_(RS_PASS_COUNT, ws.stream);
    k_page_count<<<static_cast<unsigned>(max_groups), kGatherThreads, cnt_smem, ws.stream>>>(
        pages, page_fill, list, po_bm, work, total, t, counts);
    RS_LAUNCH_CHECK();
  }
}

// Counting pass into ws counts[cells] (zeroed here): a shared-memory grid
// when it fits, the two-level split up to 4096 x 16384 cells, L2 atomics
// beyond that.
template <class Map>
void count_pass(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, uint64_t cells,
                uint32_t* counts) {
  if (n == 0) {
    RS_CUDA(cudaMemsetAsync(counts, 0, cells * sizeof(uint32_t), ws.stream));
    return;
  }
  TwoLevel t{};
  if constexpr (map_first<Map>::value) {
    if (plan_two_level<MapU32>(cells, n, t, use_ws_partition<MapU32>(true))) {  // map pass, then the uint32 partition
      auto* mapped = ws.get<uint32_t>(kSlotMapped, n);
      {
        PassTimer pt_(RS_PASS_PARTITION, ws.stream);
        k_map_cells<Map><<<stream_grid(n, kThreads * 8, 8), kThreads, 0, ws.stream>>>(in, n, map, aligned16(in),
                                                                                        mapped, ws.stats);
        RS_LAUNCH_CHECK();
      }
      two_level_count(ws, mapped, n, MapU32{}, t, counts, use_ws_partition<MapU32>(true));
      return;
    }
  }
  if (plan_two_level<Map>(cells, n, t, use_ws_partition<Map>(false))) {
    two_level_count(ws, in, n, map, t, counts, use_ws_partition<Map>(false));
    return;
  }
  RS_CUDA(cudaMemsetAsync(counts, 0, cells * sizeof(uint32_t), ws.stream));
  PassTimer pt_(RS_PASS_COUNT, ws.stream);
  if (cells <= kSmemCellsMax) {
    // Few CTAs so the per-CTA flush of `cells` counters stays small
    // against the keys each CTA counts.
    const uint64_t per_cta_min = cells * 8 > 8192 ? cells * 8 : 8192;
    const unsigned grid = stream_grid(n, static_cast<int>(per_cta_min), 8);
    k_count_smem<Map><<<grid, kThreads, cells * sizeof(uint32_t), ws.stream>>>(in, n, map, counts,
                                                                               cells, ws.stats);
  } else {
    const unsigned grid = stream_grid(n, kThreads * 8, 8);
    k_count_global<Map, false><<<grid, kThreads, 0, ws.stream>>>(in, n, map, counts, cells, ws.stats);
  }
  RS_LAUNCH_CHECK();
}

// Occupancy + look-back scan + tile starts; returns nothing, results live in
// ws slots kSlotOccCell/kSlotOccEnd/kSlotTileFirst and stats->n_occupied.
template <class C>
void scan_pass(Workspace& ws, const C* counts, uint64_t cells, uint64_t n) {
  const uint32_t tiles = static_cast<uint32_t>((cells + kScanTile - 1) / kScanTile);
  auto* desc = ws.get<unsigned long long>(kSlotTileDesc, 2ull * tiles);
  auto* occ_cell = ws.get<uint32_t>(kSlotOccCell, cells);
  auto* occ_end = ws.get<unsigned long long>(kSlotOccEnd, cells);
  RS_CUDA(cudaMemsetAsync(desc, 0, 2ull * tiles * sizeof(unsigned long long), ws.stream));
  RS_CUDA(cudaMemsetAsync(&ws.stats->tile_counter, 0, sizeof(unsigned), ws.stream));
  const uint32_t etiles = static_cast<uint32_t>((n + kEmitTile - 1) / kEmitTile);
  auto* tile_first = ws.get<uint32_t>(kSlotTileFirst, etiles + 1ull);
  {
    PassTimer pt_(RS_PASS_SCAN, ws.stream, 2);  // k_scan_cells + k_fill_spans
    auto* spans = ws.get<uint4>(kSlotSpans, etiles / 3 + 1ull);  // a long span covers >= 3 tiles
    k_scan_cells<<<tiles, kThreads, 0, ws.stream>>>(counts, cells, occ_cell, occ_end, desc, desc + tiles,
                                                     tiles, ws.stats, etiles, tile_first, spans);
    RS_LAUNCH_CHECK();
    k_fill_spans<<<sm_count() * 4, kThreads, 0, ws.stream>>>(spans, ws.stats, tile_first);
    RS_LAUNCH_CHECK();
  }
}

template <class Out>
void emit_pass(Workspace& ws, uint64_t n, Out out) {
  const uint32_t etiles = static_cast<uint32_t>((n + kEmitTile - 1) / kEmitTile);
  {
    PassTimer pt_(RS_PASS_EMIT, ws.stream);
    k_emit<Out><<<etiles, kThreads, 0, ws.stream>>>(static_cast<uint32_t*>(ws.buf[kSlotOccCell]),
                                                    static_cast<unsigned long long*>(ws.buf[kSlotOccEnd]),
                                                    static_cast<uint32_t*>(ws.buf[kSlotTileFirst]),
                                                    ws.stats, n, out);
    RS_LAUNCH_CHECK();
  }
}

// The one-launch path for small inputs (k_small_sort); with auto_cells the
// grid comes from the max inside the launch.  Stats pulled on return;
// h_stats->overflow == 2: the grid did not qualify (max known).
template <class Map, class Out>
void small_sort(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, uint32_t cells, Out out,
                uint32_t radix, uint32_t total_digits, uint32_t frac_digits, bool auto_cells, uint64_t budget) {
  reset_stats(ws);
  auto* g = ws.get<uint32_t>(kSlotCounts, kSmemCellsMax + 2);
  RS_CUDA(cudaMemsetAsync(g, 0, (kSmemCellsMax + 2) * sizeof(uint32_t), ws.stream));
  auto* kern = k_small_sort<Map, Out>;
  const size_t smem = (kSmemCellsMax + 1) * sizeof(uint32_t);
  set_smem(kern, smem);
  // at most one CTA per SM: the flush into the global grid is cells x CTAs atomics
  const uint64_t want = (n + 4 * kSmallThreads - 1) / (4 * kSmallThreads);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(want, (uint64_t)sm_count()));
  DevStats* stp = ws.stats;
  void* args[] = {const_cast<typename Map::In**>(&in), &n, &map, &cells, &out, &g, &stp, &radix, &total_digits,
                  &frac_digits, &auto_cells, &budget};
  {
    PassTimer pt_(RS_PASS_COUNT, ws.stream);
    RS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kSmallThreads), args, smem,
                                        ws.stream));
  }
  pull_stats(ws);
}

// Keys counted per uint32 grid pass: below 2^32, so no counter can wrap.
constexpr uint64_t kCountChunk = 0xFFFFFFFFull;

__global__ void k_grid_acc64(unsigned long long* __restrict__ wide, const uint32_t* __restrict__ counts,
                             uint64_t cells) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += stride) wide[c] += counts[c];
}

// One full single-grid sort: count -> scan -> emit -> report.  Leaves the
// stats (max, overflow, flags, report) in ws.h_stats after one sync.
template <class Map, class Out, class K>
void grid_sort(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, uint64_t cells,
               Out out, const K* sorted, uint32_t radix, uint32_t total_digits,
               uint32_t frac_digits) {
  if (cells > 0xFFFFFFFFull)
    fail(RS_CELL_BUDGET_EXCEEDED, "a single grid holds at most 2^32-1 cells");
  reset_stats(ws);
  if constexpr (Out::kWordBytes > 0) {
    if (n > 0 && n <= kSmallMax && cells <= kSmemCellsMax) {  // one cooperative launch
      small_sort(ws, in, n, map, static_cast<uint32_t>(cells), out, radix, total_digits, frac_digits, false, 0);
      return;
    }
  }
  auto* counts = ws.get<uint32_t>(kSlotCounts, cells);
  if (n <= kCountChunk) {
    count_pass(ws, in, n, map, cells, counts);
    scan_pass(ws, counts, cells, n);
  } else {
    // 2^32 keys or more: one cell may hold more than a uint32 counter can
    // (the reference's CountSpace counts in uint64, hashing.hpp:86).  Chunks
    // of kCountChunk keys are counted into the uint32 grid (no chunk can wrap
    // a counter) and accumulated into a uint64 grid, which the scan reads.
    auto* wide = ws.get<unsigned long long>(kSlotCounts64, cells);
    RS_CUDA(cudaMemsetAsync(wide, 0, cells * sizeof(unsigned long long), ws.stream));
    for (uint64_t off = 0; off < n; off += kCountChunk) {
      const uint64_t len = std::min<uint64_t>(kCountChunk, n - off);
      count_pass(ws, in + off, len, map, cells, counts);
      PassTimer pt_(RS_PASS_COUNT, ws.stream);
      k_grid_acc64<<<stream_grid(cells, kThreads * 4), kThreads, 0, ws.stream>>>(wide, counts, cells);
      RS_LAUNCH_CHECK();
    }
    scan_pass(ws, static_cast<const unsigned long long*>(wide), cells, n);
  }
  // the report (one small latency-bound CTA over the occupied-cell list)
  // runs on the side stream beside the emit, which reads the same list and
  // writes only the output
  ws.ensure_side();
  RS_CUDA(cudaEventRecord(ws.fork, ws.stream));
  RS_CUDA(cudaStreamWaitEvent(ws.side, ws.fork, 0));
  {
    PassTimer pt_(RS_PASS_REPORT, ws.side);
    k_report<uint32_t><<<1, report_threads(radix), 0, ws.side>>>(static_cast<const uint32_t*>(ws.buf[kSlotOccCell]), 0,
                                                radix, total_digits, frac_digits, 0, ws.stats, true);
    RS_LAUNCH_CHECK();
  }
  RS_CUDA(cudaEventRecord(ws.join, ws.side));
  emit_pass(ws, n, out);
  (void)sorted;
  RS_CUDA(cudaStreamWaitEvent(ws.stream, ws.join, 0));
  pull_stats(ws);
}

uint64_t pow10u(uint32_t e) { return checked_pow(10, e); }

void msd_u32_entry(Workspace& ws, const uint32_t* in, uint64_t n, const uint32_t* out, uint32_t key_bits);
void msd_i64_entry(Workspace& ws, const int64_t* in, uint64_t n, const uint64_t* out, uint32_t key_bits);

constexpr uint32_t kMaxSamples = 65536;  // strided sample that plans an undeclared width

// Shared driver for the decimal-integer paths (u32 and i64).
template <class Map, class Out, class K>
void integer_sort(const typename Map::In* in, uint64_t n, Map map, Out out, const K* sorted,
                  uint64_t out_capacity, const rs_options* opt, rs_report* report,
                  cudaStream_t stream, uint32_t max_digits,
                  void (*msd_u32)(Workspace&, const typename Map::In*, uint64_t, const K*, uint32_t) = nullptr) {
  ensure_device();
  const uint64_t budget = budget_of(opt);
  if (n > 0 && (!in || !sorted)) fail(RS_INVALID_ARGUMENT, "null device pointer");
  if (n == 0) {  // empty input: KeySpec{10,1,1}, nothing written
    const rs_key_spec spec = make_key_spec(10, 1, 1, budget);
    if (report) *report = rs_report{0, 0, spec};
    return;
  }
  Workspace& ws = workspace_for(stream);
  const uint32_t hint = opt ? opt->key_digits : 0;
  const bool hinted = hint >= 1 && hint <= max_digits && pow10u(hint) <= budget;
  uint32_t digits = hint;
  // a declared width already above the budget goes to the 32-bit MSD path
  // without the max pass (the MSD sort does not need the geometry up front;
  // int64 input keeps the pass, it rejects negative values)
  const bool msd_declared = msd_u32 && opt && opt->msd && hint >= 1 && hint <= max_digits &&
                            pow10u(hint) > budget && sizeof(typename Map::In) == 4;
  uint32_t key_bits = 8 * sizeof(typename Map::In);
  bool speculative = false;  // digits from a sample: the grid sort confirms or redoes
  if (!hinted && !msd_declared) {
    unsigned long long mx;
    if (n > kSmallMax && out_capacity >= n) {
      // plan the grid from the max of a strided sample instead of a full
      // max pass (0.18 ms at 2^28 keys); the counting pass folds in the true
      // max and flags keys outside the planned grid
      reset_stats(ws);
      {
        PassTimer pt_(RS_PASS_MAX, ws.stream);
        k_max_sample<Map><<<64, kThreads, 0, ws.stream>>>(in, n, kMaxSamples, map, ws.stats);
        RS_LAUNCH_CHECK();
      }
      pull_stats(ws);
      check_flags(ws.h_stats->flags);
      const uint32_t d = digit_count(ws.h_stats->max_key);
      speculative = pow10u(d) <= budget;  // else: the full max pass decides (budget vs. MSD, error order)
    }
    if (speculative) {
      digits = digit_count(ws.h_stats->max_key);
    } else if (Out::kWordBytes > 0 && n <= kSmallMax && out_capacity >= n) {
      // small input: max, grid, count, scan, emit and report in one launch when
      // the grid fits shared memory and the budget
      small_sort(ws, in, n, map, 0u, out, 10u, 0u, 0u, true, budget);
      check_flags(ws.h_stats->flags);
      // 1: a key past the sampled grid, 2: the grid does not qualify; either
      // way the exact max is known and the general path below takes over
      if (ws.h_stats->overflow == 0) {
        const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
        if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d}};
        return;
      }
      mx = ws.h_stats->max_key;
      digits = digit_count(mx);
    } else {
      mx = device_max(ws, in, n, map);
      digits = digit_count(mx);
    }
    if (!speculative) {
      mx = ws.h_stats->max_key;
      key_bits = 1;  // MSD digits cover the max's bit width only
      while (key_bits < 64 && (mx >> key_bits)) ++key_bits;
    }
  }
  if (msd_u32 && opt && opt->msd && pow10u(digits) > budget) {
    // wide keys: MSD bucket passes + per-bucket grids
    if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
    msd_u32(ws, in, n, sorted, key_bits);
    const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
    if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d}};
    return;
  }
  make_key_spec(10, digits, digits, budget);  // budget gate before the grid exists
  if (out_capacity < n)
    fail(RS_BUFFER_TOO_SMALL, "output buffer holds " + std::to_string(out_capacity) +
                                  " keys, need " + std::to_string(n));
  grid_sort(ws, in, n, map, pow10u(digits), out, sorted, 10, 0, 0);
  check_flags(ws.h_stats->flags);
  if (ws.h_stats->overflow) {  // declared (or sampled) width too small: redo with the derived one
    unsigned long long mx = ws.h_stats->max_key;
    // the direct partition reports 8-byte keys' max as a saturated 32-bit
    // cell; a key at or past 2^32 - 1 needs the exact max
    if (sizeof(typename Map::In) == 8 && mx >= 0xFFFFFFFFull) mx = device_max(ws, in, n, map);
    digits = digit_count(mx);
    if (msd_u32 && opt && opt->msd && pow10u(digits) > budget) {
      key_bits = 1;
      while (key_bits < 64 && (mx >> key_bits)) ++key_bits;
      if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
      msd_u32(ws, in, n, sorted, key_bits);
      const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
      if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d}};
      return;
    }
    make_key_spec(10, digits, digits, budget);
    grid_sort(ws, in, n, map, pow10u(digits), out, sorted, 10, 0, 0);
  }
  const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
  if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d}};
}


// ------------------------------------------------------ stable key/value
unsigned long long magic_div(uint64_t d) { return ~0ull / d + 1ull; }  // ceil(2^64/d), d = 10^k

KvPass kv_pass(uint32_t g, uint32_t digits, uint64_t n) {
  KvPass p{};
  if (!div_magic32(pow10u(2 * g), p.magic_div, p.shift_div)) {  // no 32-bit magic: 64-bit high product
    p.magic_div = magic_div(pow10u(2 * g));
    p.shift_div = 64;
  }
  div_magic32(100, p.magic_1000, p.shift_1000);
  const uint32_t rem = digits - 2 * g;
  p.bins = rem >= 2 ? 100u : static_cast<uint32_t>(pow10u(rem));
  const uint64_t tiles = (n + kKvTile - 1) / kKvTile;
  static int per_sm = 0;
  if (!per_sm) {
    set_smem(k_kv_chunk_scatter, kKvSmemBytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kv_chunk_scatter, kKvThreads, kKvSmemBytes);
    if (per_sm < 1) per_sm = 1;
  }
  uint64_t G = (uint64_t)sm_count() * per_sm;  // one persistent wave
  if (G > tiles) G = tiles ? tiles : 1;
  p.chunk = ((tiles + G - 1) / G) * kKvTile;
  p.G = static_cast<uint32_t>((n + p.chunk - 1) / p.chunk);
  return p;
}

void kv_sort(Workspace& ws, const uint32_t* keys, const uint32_t* vals, uint64_t n, uint32_t digits,
             uint32_t* keys_out, uint32_t* vals_out) {
  const uint32_t passes = (digits + 1) / 2;
  reset_stats(ws);
  uint32_t* tk = ws.get<uint32_t>(kSlotTmpKeys, n);
  uint32_t* tv = ws.get<uint32_t>(kSlotTmpVals, n);
  set_smem(k_kv_chunk_scatter, kKvSmemBytes);
  auto* total = ws.get<unsigned long long>(kSlotScratch, 4);
  const uint32_t* sk = keys;
  const uint32_t* sv = vals;
  for (uint32_t g = 0; g < passes; ++g) {
    const KvPass p = kv_pass(g, digits, n);
    const uint64_t bg = (uint64_t)p.bins * p.G;
    auto* hist = ws.get<uint32_t>(kSlotCtaHist, bg);
    auto* off = ws.get<uint32_t>(kSlotCtaOff, bg);
    const bool to_out = ((passes - 1 - g) % 2) == 0;
    uint32_t* dk = to_out ? keys_out : tk;
    uint32_t* dv = to_out ? vals_out : tv;
    {
      PassTimer pt_(RS_PASS_KV_HIST, ws.stream);
      RS_CUDA(cudaMemsetAsync(hist, 0, bg * sizeof(uint32_t), ws.stream));
      k_kv_chunk_hist<<<p.G * kKvHistSplit, kKvHistThreads, 0, ws.stream>>>(sk, n, p, aligned16(sk), hist, ws.stats);
      RS_LAUNCH_CHECK();
    }
    exscan_u32(ws, hist, bg, off, total);
    {
      PassTimer pt_(RS_PASS_KV_SCATTER, ws.stream);
      k_kv_chunk_scatter<<<p.G, kKvThreads, kKvSmemBytes, ws.stream>>>(sk, sv, dk, dv, n, p, off,
                                                                        aligned16(sk) && aligned16(sv));
      RS_LAUNCH_CHECK();
    }
    sk = dk;
    sv = dv;
  }
  {
    PassTimer pt_(RS_PASS_REPORT, ws.stream);
    k_report<uint32_t><<<1, report_threads(10), 0, ws.stream>>>(keys_out, n, 10, 0, 0, 0, ws.stats);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
}

// ------------------------------------------------------- fixed strings
// strings_to_keys (key_model.cpp:225-247): ordinal via a 256-entry table
// (0 = not in the alphabet), Horner in base radix over `digits` positions,
// pad ordinal 0 after the string's end (first NUL or the record width).
struct StrTable {
  uint16_t ord[256];
  uint8_t sym[256];  // ordinal -> byte
  uint32_t radix;
};


__global__ void __launch_bounds__(kThreads) k_str_keys(const uint8_t* __restrict__ recs, uint64_t n,
                                                       uint32_t width, uint32_t digits,
                                                       uint32_t radix, const uint16_t* __restrict__ ord_g,
                                                       unsigned long long* __restrict__ keys,
                                                       DevStats* st) {
  __shared__ uint16_t ord[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ord[i] = ord_g[i];
  __syncthreads();
  unsigned bad = 0;
  unsigned long long mxlen = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint8_t* r = recs + i * width;
    unsigned long long key = 0;
    bool ended = false;
    uint32_t len = 0;
    for (uint32_t j = 0; j < digits; ++j) {
      uint32_t o = 0;
      if (j < width && !ended) {
        const uint8_t c = r[j];
        if (c == 0) ended = true;
        else {
          o = ord[c];
          if (o == 0) bad = 1;
          ++len;
        }
      }
      key = key * radix + o;
    }
    for (uint32_t j = digits; j < width && !ended; ++j) {  // longer than digits
      if (r[j] == 0) break;
      ++len;
      if (ord[r[j]] == 0) bad = 1;
    }
    mxlen = len > mxlen ? len : mxlen;
    keys[i] = key;
  }
  if (bad) atomicOr(&st->flags, 8u);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mxlen, o);
    mxlen = w > mxlen ? w : mxlen;
  }
  if ((threadIdx.x & 31) == 0 && mxlen) atomicMax(&st->max_key, mxlen);
}


// Width (longest string) and symbol validation for the MSD path, optionally
// writing each record's packed key (obits bits per ordinal, first symbol
// most significant, pad 0 — the MSD key order); 8-byte records read as two
// 16-byte loads per thread per round.
template <int kBits>  // bits per packed ordinal; 0 = the runtime obits
__global__ void __launch_bounds__(kThreads) k_str_scan(const uint8_t* __restrict__ recs, uint64_t n, uint32_t width,
                                                       bool w8, const uint16_t* __restrict__ ord_g, DevStats* st,
                                                       unsigned long long* __restrict__ packed, int lin,
                                                       uint32_t alen, uint32_t obits_rt) {
  const uint32_t obits = kBits ? kBits : obits_rt;
  __shared__ uint16_t ord[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) ord[i] = ord_g[i];
  __syncthreads();
  unsigned bad = 0;
  unsigned long long mxlen = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // 5-bit ordinals of a contiguous alphabet, SWAR on the record's two 32-bit
  // halves: first NUL from the zero-byte mask, per-byte ordinal and range
  // check with the byte-SIMD intrinsics, fields merged pairwise (first
  // character most significant).  Same results as the byte loop below.
  const uint32_t lin4 = 0x01010101u * static_cast<uint32_t>(lin + 1), alen4 = 0x01010101u * alen;
  auto pack20 = [](uint32_t o) {  // bytes o0..o3 (o0 first) -> o0<<15 | o1<<10 | o2<<5 | o3
    const uint32_t a = __byte_perm(o, 0, 0x0123);  // o3 | o2<<8 | o1<<16 | o0<<24
    const uint32_t p = (a & 0x00FF00FFu) | ((a & 0xFF00FF00u) >> 3);
    return (p & 0xFFFFu) | ((p >> 16) << 10);
  };
  auto scan8_lin5 = [&](unsigned long long w) {
    const unsigned long long z = (w - 0x0101010101010101ull) & ~w & 0x8080808080808080ull;
    const uint32_t len = z ? static_cast<uint32_t>(__ffsll(static_cast<long long>(z)) - 1) >> 3 : 8u;
    const unsigned long long vm = len == 8 ? ~0ull : ((1ull << (8 * len)) - 1ull);
    const uint32_t lo = static_cast<uint32_t>(w), hi = static_cast<uint32_t>(w >> 32);
    const uint32_t vlo = static_cast<uint32_t>(vm), vhi = static_cast<uint32_t>(vm >> 32);
    const uint32_t dlo = __vsub4(lo, lin4), dhi = __vsub4(hi, lin4);  // ordinal - 1 per byte
    bad |= ((__vcmpgeu4(dlo, alen4) & vlo) | (__vcmpgeu4(dhi, alen4) & vhi)) != 0u;
    const uint32_t olo = __vadd4(dlo, 0x01010101u) & vlo, ohi = __vadd4(dhi, 0x01010101u) & vhi;
    mxlen = len > mxlen ? len : mxlen;
    return (static_cast<unsigned long long>(pack20(olo)) << 20) | pack20(ohi);
  };
  auto scan8 = [&](unsigned long long w) {
    if (kBits == 5 && lin >= 0) return scan8_lin5(w);
    uint32_t len = 0;
    bool ended = false;
    unsigned long long k = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t c = static_cast<uint32_t>(w >> (8 * j)) & 0xffu;
      ended |= c == 0;
      // contiguous alphabet: ordinal = byte - lin when inside [lin+1, lin+alen], else 0 (bad)
      const uint32_t lo = c - static_cast<uint32_t>(lin);
      const uint32_t o = ended ? 0u : (lin >= 0 ? (lo - 1u < alen ? lo : 0u) : ord[c]);
      len += ended ? 0u : 1u;
      bad |= !ended && o == 0;
      k = (k << obits) | o;
    }
    mxlen = len > mxlen ? len : mxlen;
    return k;
  };
  if (w8) {
    const auto* r2 = reinterpret_cast<const ulonglong2*>(recs);
    auto* p2 = reinterpret_cast<ulonglong2*>(packed);
    const uint64_t pairs = n >> 1;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < pairs; i += 2 * stride) {
      const ulonglong2 a = __ldcs(r2 + i), b = __ldcs(r2 + i + stride);
      const ulonglong2 ka = make_ulonglong2(scan8(a.x), scan8(a.y)), kb = make_ulonglong2(scan8(b.x), scan8(b.y));
      if (packed) {
        p2[i] = ka;
        p2[i + stride] = kb;
      }
    }
    if (i < pairs) {
      const ulonglong2 a = __ldcs(r2 + i);
      const ulonglong2 ka = make_ulonglong2(scan8(a.x), scan8(a.y));
      if (packed) p2[i] = ka;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned long long k = scan8(reinterpret_cast<const unsigned long long*>(recs)[n - 1]);
      if (packed) packed[n - 1] = k;
    }
  } else {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      uint32_t len = 0;
      bool ended = false;
      unsigned long long k = 0;
      const uint8_t* r = recs + i * width;
      for (uint32_t j = 0; j < width; ++j) {
        uint32_t o = 0;
        if (!ended) {
          const uint8_t c = r[j];
          if (c == 0) ended = true;
          else {
            ++len;
            o = ord[c];
            bad |= o == 0;
          }
        }
        k = (k << obits) | o;
      }
      mxlen = len > mxlen ? len : mxlen;
      if (packed) packed[i] = k;
    }
  }
  if (bad) atomicOr(&st->flags, 8u);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mxlen, o);
    mxlen = w > mxlen ? w : mxlen;
  }
  if ((threadIdx.x & 31) == 0 && mxlen) atomicMax(&st->max_key, mxlen);
}

// The first symbol outside the alphabet in (record, position) order — the
// one Alphabet::ordinal raises for in strings_to_keys (key_model.cpp:
// 208-214, 233-241).
__global__ void k_str_first_bad(const uint8_t* __restrict__ recs, uint64_t n, uint32_t width,
                                const uint16_t* __restrict__ ord, unsigned long long* first) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint8_t* r = recs + i * width;
    for (uint32_t j = 0; j < width && r[j] != 0; ++j)
      if (__ldg(ord + r[j]) == 0) {
        atomicMin(first, i * width + j);
        break;
      }
  }
}

// Emit writer for strings: key -> record bytes (key_to_string,
// key_model.cpp:249-263; pad ordinals become NUL bytes).
struct OutStr {
  static constexpr int kWordBytes = 0;  // records
  uint8_t* out;
  uint32_t width, digits, radix;
  const uint8_t* sym;  // device: ordinal -> byte, sym[0] = 0
  unsigned long long base;
  __device__ __forceinline__ void put_key(uint64_t p, unsigned long long key) const {
    uint8_t buf[32];  // a single grid has < 2^32 cells and radix >= 2, so digits <= 31
    for (int j = (int)digits - 1; j >= 0; --j) {
      const unsigned long long q = key / radix;
      buf[j] = sym[key - q * radix];
      key = q;
    }
    uint8_t* r = out + p * width;
    for (uint32_t j = 0; j < width; ++j) r[j] = j < digits ? buf[j] : 0;
  }
  __device__ __forceinline__ void put1(uint64_t p, uint32_t c) const { put_key(p, base + c); }
  __device__ __forceinline__ void put4(uint64_t p, const uint32_t (&c)[4], uint64_t end) const {
    for (int e = 0; e < 4; ++e)
      if (p + e < end) put_key(p + e, base + c[e]);
  }
  __device__ __forceinline__ void put4_full(uint64_t p, const uint32_t (&c)[4]) const {
    for (int e = 0; e < 4; ++e) put_key(p + e, base + c[e]);
  }
};


// ------------------------------------------------------------ MSD engine
// Segmented MSD over 8-bit digit sub-grids (kernels_msd_engine.cuh).  Levels
// run until every segment became a leaf; each level synchronises once to
// size the next one.  Leaves write the final output through `emit`.
template <class Load, class Emit>
void msd_sort(Workspace& ws, Load load0, uint64_t n, uint32_t key_bits, Emit emit) {
  using K = typename Load::Key;
  if (n == 0) return;
  if (n >= 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "the MSD path sorts fewer than 2^32 keys per call");
  K* buf[2] = {ws.get<K>(kSlotTmpKeys, n), ws.get<K>(kSlotTmpVals, n)};
  const uint64_t cap = std::min<uint64_t>(n, 1ull << 26) + 256;
  auto* segs_a = ws.get<MsdSeg>(kSlotCtaHist, cap);
  auto* segs_b = ws.get<MsdSeg>(kSlotCtaOff, cap);
  auto* leaf_grid = ws.get<MsdSeg>(kSlotBucketStart, cap);
  auto* leaf_small = ws.get<MsdSeg>(kSlotLows, cap);
  auto* leaf_copy = ws.get<MsdSeg>(kSlotTmpKeys2, cap);
  auto* leaf_warp = ws.get<MsdSeg>(kSlotTmpVals2, cap);
  auto* leaf_radix = ws.get<MsdSeg>(kSlotExtra1, cap);
  auto* cnt = ws.get<unsigned>(kSlotScratch, 10);  // [0..5] list counts, [6..7] u64 total, [8] largest radix leaf
  auto* total = reinterpret_cast<unsigned long long*>(cnt + 6);
  // the first level's one segment, its chunks already assigned (no count,
  // scan and read-back for it)
  const uint32_t first_chunks = static_cast<uint32_t>((n + kMsdChunk - 1) / kMsdChunk);
  MsdSeg first{0, static_cast<uint32_t>(n), 0, first_chunks};
  RS_CUDA(cudaMemcpyAsync(segs_a, &first, sizeof(MsdSeg), cudaMemcpyHostToDevice, ws.stream));
  uint32_t nseg = 1;
  uint32_t shift = key_bits > kMsdDigitBits ? key_bits - kMsdDigitBits : 0;
  MsdSeg* segs_in = segs_a;
  MsdSeg* segs_out = segs_b;
  for (int level = 0; nseg > 0; ++level) {
    // chunks of every open segment
    unsigned long long nchunks = first_chunks;
    if (level > 0) {
      auto* ccount = ws.get<uint32_t>(kSlotMisc, 2ull * nseg + 2);
      uint32_t* cstart = ccount + nseg + 1;
      k_msd_chunk_counts<<<(nseg + 255) / 256, 256, 0, ws.stream>>>(segs_in, nseg, ccount);
      RS_LAUNCH_CHECK();
      exscan_u32(ws, ccount, nseg, cstart, total);
      k_msd_chunk_assign<<<(nseg + 255) / 256, 256, 0, ws.stream>>>(segs_in, nseg, ccount, cstart);
      RS_LAUNCH_CHECK();
      RS_CUDA(cudaMemcpyAsync(&nchunks, total, sizeof(nchunks), cudaMemcpyDeviceToHost, ws.stream));
      RS_CUDA(cudaStreamSynchronize(ws.stream));
    }
    auto* chunk_seg = ws.get<uint32_t>(kSlotTileFirst, nchunks);
    auto* table = ws.get<uint32_t>(kSlotCounts, nchunks * kMsdBins);
    auto* off = ws.get<uint32_t>(kSlotOccEnd, nchunks * kMsdBins);
    k_msd_chunks<<<nseg, 256, 0, ws.stream>>>(segs_in, nseg, chunk_seg);
    RS_LAUNCH_CHECK();
    K* dst = buf[level & 1];
    {
      PassTimer pt_(RS_PASS_MSD_HIST, ws.stream);
      if (level == 0) k_msd_hist<<<nchunks, kMsdThreads, 0, ws.stream>>>(load0, segs_in, chunk_seg, shift, table);
      else k_msd_hist<<<nchunks, kMsdThreads, 0, ws.stream>>>(LoadKeys<K>{buf[(level - 1) & 1], n}, segs_in,
                                                              chunk_seg, shift, table);
      RS_LAUNCH_CHECK();
    }
    exscan_u32(ws, table, nchunks * kMsdBins, off, total);
    {
      PassTimer pt_(RS_PASS_MSD_SCATTER, ws.stream);
      set_smem(k_msd_scatter<Load>, msd_scatter_smem<Load>());
      set_smem(k_msd_scatter<LoadKeys<K>>, msd_scatter_smem<LoadKeys<K>>());
      if (level == 0)
        k_msd_scatter<<<nchunks, kMsdThreads, msd_scatter_smem<Load>(), ws.stream>>>(load0, segs_in, chunk_seg, shift,
                                                                                      off, dst);
      else k_msd_scatter<<<nchunks, kMsdThreads, msd_scatter_smem<LoadKeys<K>>(), ws.stream>>>(LoadKeys<K>{buf[(level - 1) & 1], n}, segs_in,
                                                                 chunk_seg, shift, off, dst);
      RS_LAUNCH_CHECK();
    }
    RS_CUDA(cudaMemsetAsync(cnt, 0, 6 * sizeof(unsigned), ws.stream));
    RS_CUDA(cudaMemsetAsync(cnt + 8, 0, sizeof(unsigned), ws.stream));
    MsdLists L{segs_out, leaf_grid, leaf_small, leaf_copy, leaf_warp, leaf_radix, cnt, cnt + 8};
    const unsigned long long pairs = (unsigned long long)nseg * kMsdBins;
    k_msd_classify<<<static_cast<unsigned>((pairs + 255) / 256), 256, 0, ws.stream>>>(segs_in, nseg, off, shift, L);
    RS_LAUNCH_CHECK();
    unsigned h[9] = {};
    RS_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, ws.stream));
    RS_CUDA(cudaStreamSynchronize(ws.stream));
    for (int i = 0; i < 6; ++i)
      if ((uint64_t)h[i] > cap) fail(RS_CUDA_ERROR, "MSD segment list overflow");
    {
      PassTimer pt_(RS_PASS_BUCKET, ws.stream,
                    (h[1] ? 1 : 0) + (h[2] ? 1 : 0) + (h[3] ? 1 : 0) + (h[4] ? 1 : 0) + (h[5] ? 1 : 0));
      if (h[5]) {  // buffers sized to the largest leaf of the list
        set_smem(k_leaf_radix<K, Emit>, leaf_radix_smem<K>(kLeafRadixMax));
        const uint32_t lcap = (h[8] + 15) & ~15u;
        k_leaf_radix<K, Emit><<<h[5], kLeafRadixThreads, leaf_radix_smem<K>(lcap), ws.stream>>>(dst, leaf_radix, shift,
                                                                                                 lcap, emit);
      }
      if (h[4]) {
        const unsigned blocks = std::min<unsigned>((h[4] + 7) / 8, sm_count() * 16);
        k_leaf_warp<K, Emit><<<blocks, kMsdThreads, 0, ws.stream>>>(dst, leaf_warp, h[4], emit);
      }
      if (h[3]) k_leaf_copy<K, Emit><<<h[3], 256, 0, ws.stream>>>(dst, leaf_copy, emit);
      if (h[1]) {
        // grid + uint16 staging for segments up to `lcap` keys (the rest: run-length emit)
        const size_t grid_b = leaf_grid_words(shift) * sizeof(uint32_t);
        const size_t smem = std::min<size_t>(grid_b + 2 * 65536, smem_optin() - 1024);
        const uint32_t lcap = static_cast<uint32_t>(std::min<size_t>((smem - grid_b) / 2, 65535));
        set_smem(k_leaf_grid<K, Emit>, smem);
        k_leaf_grid<K, Emit><<<h[1], kLeafGridThreads, smem, ws.stream>>>(dst, leaf_grid, shift, lcap, emit, h[1],
                                                                           static_cast<uint32_t>(sm_count()));
      }
      if (h[2]) k_leaf_bitonic<K, Emit><<<h[2], kMsdThreads, 0, ws.stream>>>(dst, leaf_small, emit);
      RS_LAUNCH_CHECK();
    }
    nseg = h[0];
    std::swap(segs_in, segs_out);
    if (shift == 0 && nseg) fail(RS_CUDA_ERROR, "MSD: segments left after the last digit");
    shift = shift > kMsdDigitBits ? shift - kMsdDigitBits : 0;
  }
}
void msd_u32_entry(Workspace& ws, const uint32_t* in, uint64_t n, const uint32_t* out, uint32_t key_bits) {
  reset_stats(ws);
  msd_sort(ws, LoadKeys<uint32_t>{in, n}, n, key_bits, EmitKey<uint32_t>{const_cast<uint32_t*>(out)});
  {
    PassTimer pt_(RS_PASS_REPORT, ws.stream);
    k_report<uint32_t><<<1, report_threads(10), 0, ws.stream>>>(out, n, 10, 0, 0, 0, ws.stats);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
}

// int64 input (non-negative, checked by the max pass): the same engine over
// 64-bit keys, digits over the max's bit width
void msd_i64_entry(Workspace& ws, const int64_t* in, uint64_t n, const uint64_t* out, uint32_t key_bits) {
  reset_stats(ws);
  msd_sort(ws, LoadKeys<uint64_t>{reinterpret_cast<const uint64_t*>(in), n}, n, key_bits,
           EmitKey<uint64_t>{const_cast<uint64_t*>(out)});
  {
    PassTimer pt_(RS_PASS_REPORT, ws.stream);
    k_report<uint64_t><<<1, report_threads(10), 0, ws.stream>>>(out, n, 10, 0, 0, 0, ws.stats);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
}

void msd_sort_str(Workspace& ws, const uint8_t* chars, uint64_t n, uint32_t width, uint32_t w, uint32_t radix,
                  const uint16_t* d_ord, const uint8_t* d_sym, uint8_t* out, int lin,
                  const unsigned long long* packed, uint32_t obits) {
  reset_stats(ws);
  EmitStr em{out, width, d_sym};
  em.lin = lin;
  em.obits = obits;
  em.w8 = width == 8 && (reinterpret_cast<uintptr_t>(out) & 7) == 0;
  if (packed) {  // keys packed by k_str_scan
    msd_sort(ws, LoadKeys<unsigned long long>{packed, n}, n, obits * width, em);
  } else {
    LoadStr ld{chars, width, d_ord};
    ld.w8 = width == 8 && (reinterpret_cast<uintptr_t>(chars) & 7) == 0;
    ld.lin = lin;
    ld.obits = obits;
    msd_sort(ws, ld, n, obits * width, em);
  }
  {
    PassTimer pt_(RS_PASS_REPORT, ws.stream);
    k_report_recs<<<1, 32, 0, ws.stream>>>(out, n, width, w, radix, d_ord, ws.stats);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
}

// ---------------------------------------------- single-process multi-GPU
// rs_sort_u32_multi: the per-GPU grids summed on the first device...
__global__ void k_grid_add(uint32_t* __restrict__ acc, const uint32_t* __restrict__ other, uint32_t parts,
                           uint64_t cells) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += stride) {
    uint32_t s = acc[c];
    for (uint32_t p = 0; p < parts; ++p) s += other[(uint64_t)p * cells + c];
    acc[c] = s;
  }
}

// ...and cut into `parts` contiguous cell ranges of about total/parts keys:
// cut r (1 <= r < parts) = 1 + the cell where the inclusive prefix first
// reaches ceil(r * total / parts) (dist.cell_bounds_device's rule).
__global__ void k_grid_cuts(const uint32_t* __restrict__ excl, const uint32_t* __restrict__ cnt, uint64_t cells,
                            const unsigned long long* __restrict__ total, uint32_t parts,
                            unsigned long long* __restrict__ cuts) {
  const unsigned long long tot = *total;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += stride) {
    const unsigned long long lo = excl[c], hi = lo + cnt[c];
    for (uint32_t r = 1; r < parts; ++r) {
      const unsigned long long t = (r * tot + parts - 1) / parts;
      if (lo < t && t <= hi) cuts[r - 1] = c + 1;
    }
  }
}

}  // namespace rsb

using namespace rsb;

// ------------------------------------------------------- decimal text
// The reference's message for a numeral's first failing check
// (key_model.cpp:22-34, 38-49, 80-105).
[[noreturn]] void fail_numeral(uint32_t code, const std::string& text, uint32_t frac_digits) {
  switch (code) {
    case kDecEmpty: fail(RS_PARSE_ERROR, "empty numeral");
    case kDecNegative: fail(RS_NEGATIVE_VALUE, "negative values are not supported: '" + text + "'");
    case kDecMultiDot: fail(RS_PARSE_ERROR, "multiple decimal points in '" + text + "'");
    case kDecNoFrac: fail(RS_PARSE_ERROR, "no digits after decimal point in '" + text + "'");
    case kDecNoDigits: fail(RS_PARSE_ERROR, "no digits in '" + text + "'");
    case kDecBadChar: fail(RS_PARSE_ERROR, "invalid character in numeral '" + text + "'");
    case kDecTooLong:
      fail(RS_CELL_BUDGET_EXCEEDED, "numeral '" + text + "' has more digits than any cell budget admits");
    default:
      fail(RS_CELL_BUDGET_EXCEEDED, "key space 10^" + std::to_string(frac_digits) + " overflows 64 bits");
  }
}

// =================================================================== C-ABI
extern "C" {

const char* rs_last_error(void) { return g_last_error.c_str(); }

const char* rs_status_name(rs_status s) {
  switch (s) {
    case RS_OK: return "ok";
    case RS_PARSE_ERROR: return "parse_error";
    case RS_NEGATIVE_VALUE: return "negative_value";
    case RS_NON_FINITE: return "non_finite";
    case RS_CELL_BUDGET_EXCEEDED: return "cell_budget_exceeded";
    case RS_SYMBOL_OUT_OF_ALPHABET: return "symbol_out_of_alphabet";
    case RS_SPEC_MISMATCH: return "spec_mismatch";
    case RS_BUFFER_TOO_SMALL: return "buffer_too_small";
    case RS_RANGE_EXCEEDED: return "range_exceeded";
    case RS_OUT_OF_RANGE: return "out_of_range";
    case RS_INVALID_RANGE: return "invalid_range";
    case RS_INSUFFICIENT_DATA: return "insufficient_data";
    case RS_INVALID_ARGUMENT: return "invalid_argument";
    case RS_CUDA_ERROR: return "cuda_error";
    case RS_NCCL_ERROR: return "nccl_error";
    case RS_NO_DEVICE: return "no_device";
  }
  return "unknown";
}

const char* rs_version(void) { return "recsort_b200 0.1.0 (sm_100a)"; }

uint64_t rs_launch_count(void) { return g_launches.load(); }
void rs_profile_enable(int on) { g_profile.store(on ? 1 : 0); }
void rs_profile_reset(void) {
  flush_profile();
  std::lock_guard<std::mutex> lock(g_prof_mutex);
  for (int i = 0; i < RS_NUM_PASSES; ++i) {
    g_ms[i] = 0.0;
    g_pass_launches[i] = 0;
  }
}
int rs_profile_read(double* h_ms, uint64_t* h_launches) {
  flush_profile();
  std::lock_guard<std::mutex> lock(g_prof_mutex);
  for (int i = 0; i < RS_NUM_PASSES; ++i) {
    if (h_ms) h_ms[i] = g_ms[i];
    if (h_launches) h_launches[i] = g_pass_launches[i];
  }
  return RS_NUM_PASSES;
}
const char* rs_pass_name(int pass) {
  static const char* names[RS_NUM_PASSES] = {"max",      "count",       "scan",   "emit", "report",
                                             "kv_hist",  "kv_scatter",  "msd_hist", "msd_scatter",
                                             "bucket",   "copy",        "other",  "partition"};
  return (pass >= 0 && pass < RS_NUM_PASSES) ? names[pass] : "unknown";
}


void rs_release_workspaces(void) {
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  for (auto& kv : g_ws) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(kv.first.first);
    cudaStreamSynchronize(kv.second->stream);
    kv.second->release();
    delete kv.second;
    cudaSetDevice(prev);
  }
  g_ws.clear();
}

rs_status rs_sort_u32(const uint32_t* keys, uint64_t n, uint32_t* out, uint64_t out_capacity,
                      const rs_options* opt, rs_report* report, void* stream) {
  return guarded([&] {
    OutU32 o{out, 0u, aligned16(out)};
    integer_sort(keys, n, MapU32{}, o, out, out_capacity, opt, report,
                 static_cast<cudaStream_t>(stream), 10, &msd_u32_entry);
  });
}

rs_status rs_sort_i64(const int64_t* values, uint64_t n, int64_t* out, uint64_t out_capacity,
                      const rs_options* opt, rs_report* report, void* stream) {
  return guarded([&] {
    OutU64 o{reinterpret_cast<unsigned long long*>(out), 0ull, aligned32(out)};
    integer_sort(values, n, MapI64{}, o, reinterpret_cast<const uint64_t*>(out), out_capacity, opt,
                 report, static_cast<cudaStream_t>(stream), 19, &msd_i64_entry);
  });
}

rs_status rs_sort_keys(const uint64_t* keys, uint64_t n, rs_key_spec spec, uint64_t* out,
                       uint64_t out_capacity, const rs_options* opt, rs_report* report,
                       void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    make_key_spec(spec.radix, spec.total_digits, spec.integer_digits, budget);
    const uint64_t cells = checked_pow(spec.radix, spec.total_digits);
    if (n > 0 && (!keys || !out)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    if (n == 0) {
      if (report) *report = rs_report{0, 0, spec};
      return;
    }
    if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    OutU64 o{reinterpret_cast<unsigned long long*>(out), 0ull, aligned32(out)};
    grid_sort(ws, reinterpret_cast<const unsigned long long*>(keys), n, MapU64{}, cells, o, out,
              spec.radix, spec.total_digits, 0);
    if (ws.h_stats->overflow)
      fail(RS_SPEC_MISMATCH, "a key is outside its spec's key space");
    if (report) *report = rs_report{n, ws.h_stats->cells_traversed, spec};
  });
}

// One float64 sort with mapper `map`; false when a value left the lean
// mapper's fast domain (nothing is reported, the caller redoes the sort
// with the general mapper).
extern "C++" {
template <class Map>
bool sort_f64_with(Workspace& ws, const double* x, uint64_t n, uint32_t scale, Map map, uint64_t* out,
                   uint64_t out_capacity, const rs_options* opt, uint64_t budget, rs_report* report) {
  const uint64_t P = pow10u(scale);
  const uint32_t hint = opt ? opt->key_digits : 0;
  const bool hinted = hint > scale && hint <= 19 && pow10u(hint) <= budget;
  uint32_t total = hint;
  if (!hinted) {
    const unsigned long long mx = device_max(ws, x, n, map, false);
    if (ws.h_stats->flags & kFlagDomain) return false;
    check_f64(ws, x, n, scale);
    total = digit_count(mx / P) + scale;
  }
  make_key_spec(10, total, total - scale, budget);
  if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
  OutU64 o{reinterpret_cast<unsigned long long*>(out), 0ull, aligned32(out)};
  grid_sort(ws, x, n, map, pow10u(total), o, out, 10, 0, scale);
  if (ws.h_stats->flags & kFlagDomain) return false;
  check_f64(ws, x, n, scale);
  if (ws.h_stats->overflow) {
    total = digit_count(ws.h_stats->max_key / P) + scale;
    make_key_spec(10, total, total - scale, budget);
    grid_sort(ws, x, n, map, pow10u(total), o, out, 10, 0, scale);
  }
  const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
  if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d - scale}};
  return true;
}
}  // extern "C++"

rs_status rs_sort_f64(const double* x, uint64_t n, uint32_t scale, uint64_t* out,
                      uint64_t out_capacity, const rs_options* opt, rs_report* report,
                      void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (scale > kF2dMaxScale) fail(RS_OUT_OF_RANGE, "float_to_decimal on the device supports scale <= 40");
    if (n > 0 && (!x || !out)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    // lambda = digits(max / 10^scale) (key_model.cpp:122-124): 10^scale itself must fit
    const std::string pow_msg = "key space 10^" + std::to_string(scale) + " overflows 64 bits";
    if (n == 0) {
      if (scale > 19) fail(RS_CELL_BUDGET_EXCEEDED, pow_msg);
      if (report) *report = rs_report{0, 0, make_key_spec(10, 1, 1, budget)};
      return;
    }
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    if (scale > 19) {  // the element errors come first (in input order), then the geometry's
      device_max(ws, x, n, make_map_f64<true>(scale), false);
      check_f64(ws, x, n, scale);
      fail(RS_CELL_BUDGET_EXCEEDED, pow_msg);
    }
    // the lean mapper first; a value outside its domain redoes the sort with the general one
    if (scale > 15 || !sort_f64_with(ws, x, n, scale, make_map_f64<false>(scale), out, out_capacity, opt, budget,
                                     report))
      sort_f64_with(ws, x, n, scale, make_map_f64<true>(scale), out, out_capacity, opt, budget, report);
  });
}


rs_status rs_float_to_decimal(const double* x, uint64_t n, uint32_t scale, uint64_t* out, void* stream) {
  return guarded([&] {
    ensure_device();
    if (scale > kF2dMaxScale) fail(RS_OUT_OF_RANGE, "float_to_decimal on the device supports scale <= 40");
    if (n == 0) return;
    if (!x || !out) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    auto run = [&](auto map) {
      reset_stats(ws);
      PassTimer pt_(RS_PASS_MAX, ws.stream);
      k_f64_map_u64<<<stream_grid(n, kThreads * 8), kThreads, 0, ws.stream>>>(
          x, n, map, reinterpret_cast<unsigned long long*>(out), ws.stats);
      RS_LAUNCH_CHECK();
    };
    run(make_map_f64<false>(scale));  // lean; values outside its domain: again with the general mapper
    pull_stats(ws);
    if (ws.h_stats->flags & kFlagDomain) {
      run(make_map_f64<true>(scale));
      pull_stats(ws);
    }
    check_f64(ws, x, n, scale);
  });
}


rs_status rs_sort_u32_multi(uint32_t ngpus, const int* h_devices, const uint32_t* const* h_keys,
                            const uint64_t* h_n, uint32_t* const* h_out, const uint64_t* h_out_capacity,
                            uint64_t* h_written, const rs_options* opt, rs_report* report) {
  return guarded([&] {
    if (ngpus == 0 || ngpus > 64 || !h_devices || !h_keys || !h_n || !h_out || !h_out_capacity || !h_written)
      fail(RS_INVALID_ARGUMENT, "bad multi-GPU arguments");
    int prev = 0;
    RS_CUDA(cudaGetDevice(&prev));
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    const uint64_t budget = budget_of(opt);
    uint64_t n_total = 0;
    unsigned long long mx = 0;
    for (uint32_t g = 0; g < ngpus; ++g) {  // the max (sort.cpp:31-38) over every shard
      RS_CUDA(cudaSetDevice(h_devices[g]));
      ensure_device();
      n_total += h_n[g];
      if (h_n[g] > 0) {
        if (!h_keys[g] || !h_out[g]) fail(RS_INVALID_ARGUMENT, "null device pointer");
        Workspace& ws = workspace_for(nullptr);
        const unsigned long long m = device_max(ws, h_keys[g], h_n[g], MapU32{});
        mx = m > mx ? m : mx;
      }
    }
    if (n_total >= 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "rs_sort_u32_multi sorts fewer than 2^32 keys");
    if (n_total == 0) {
      for (uint32_t g = 0; g < ngpus; ++g) h_written[g] = 0;
      if (report) *report = rs_report{0, 0, make_key_spec(10, 1, 1, budget)};
      return;
    }
    const uint32_t digits = digit_count(mx);
    const rs_key_spec spec = make_key_spec(10, digits, digits, budget);
    const uint64_t cells = pow10u(digits);
    // every GPU counts its shard into its own grid (allocated per shard: a
    // device may hold several shards)
    struct Grids {
      std::vector<uint32_t*> p;
      std::vector<int> dev;
      ~Grids() {
        for (size_t i = 0; i < p.size(); ++i)
          if (p[i]) {
            cudaSetDevice(dev[i]);
            cudaFree(p[i]);
          }
      }
    } gr;
    gr.p.assign(ngpus, nullptr);
    gr.dev.assign(h_devices, h_devices + ngpus);
    std::vector<uint32_t*>& grids = gr.p;
    for (uint32_t g = 0; g < ngpus; ++g) {
      RS_CUDA(cudaSetDevice(h_devices[g]));
      RS_CUDA(cudaMalloc(&grids[g], cells * sizeof(uint32_t)));
      Workspace& ws = workspace_for(nullptr);
      reset_stats(ws);
      count_pass(ws, h_keys[g], h_n[g], MapU32{}, cells, grids[g]);
    }
    for (uint32_t g = 0; g < ngpus; ++g) {
      RS_CUDA(cudaSetDevice(h_devices[g]));
      RS_CUDA(cudaDeviceSynchronize());
    }
    // the first GPU gathers the other grids over NVLink and sums them
    RS_CUDA(cudaSetDevice(h_devices[0]));
    Workspace& w0 = workspace_for(nullptr);
    if (ngpus > 1) {
      auto* gather = w0.get<uint32_t>(kSlotExtra1, (ngpus - 1) * cells);
      for (uint32_t g = 1; g < ngpus; ++g)
        RS_CUDA(cudaMemcpyPeerAsync(gather + (g - 1) * cells, h_devices[0], grids[g], h_devices[g],
                                    cells * sizeof(uint32_t), w0.stream));
      k_grid_add<<<stream_grid(cells, kThreads * 4), kThreads, 0, w0.stream>>>(grids[0], gather, ngpus - 1, cells);
      RS_LAUNCH_CHECK();
    }
    // cell cuts from the global prefix
    auto* excl = w0.get<uint32_t>(kSlotTmpKeys, cells);
    auto* tot = w0.get<unsigned long long>(kSlotScratch, 4 + 64);
    auto* cuts = tot + 4;
    exscan_u32(w0, grids[0], cells, excl, tot);
    std::vector<unsigned long long> hcuts(ngpus > 1 ? ngpus - 1 : 1, cells);
    if (ngpus > 1) {
      RS_CUDA(cudaMemcpyAsync(cuts, hcuts.data(), (ngpus - 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                              w0.stream));
      k_grid_cuts<<<stream_grid(cells, kThreads * 4), kThreads, 0, w0.stream>>>(excl, grids[0], cells, tot, ngpus,
                                                                              cuts);
      RS_LAUNCH_CHECK();
      RS_CUDA(cudaMemcpyAsync(hcuts.data(), cuts, (ngpus - 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              w0.stream));
    }
    RS_CUDA(cudaStreamSynchronize(w0.stream));
    std::vector<uint64_t> bounds(ngpus + 1, 0);
    bounds[ngpus] = cells;
    for (uint32_t r = 1; r < ngpus; ++r) bounds[r] = std::max<uint64_t>(bounds[r - 1], std::min<uint64_t>(hcuts[r - 1], cells));
    // the global grid to every GPU, each emits its own cell range
    for (uint32_t g = 1; g < ngpus; ++g)
      RS_CUDA(cudaMemcpyPeer(grids[g], h_devices[g], grids[0], h_devices[0], cells * sizeof(uint32_t)));
    for (uint32_t g = 0; g < ngpus; ++g) {
      RS_CUDA(cudaSetDevice(h_devices[g]));
      uint64_t wr = 0;
      const rs_status st = rs_emit_u32(grids[g], cells, bounds[g], bounds[g + 1], 0, h_out[g], h_out_capacity[g], &wr,
                                       nullptr);
      if (st != RS_OK) fail(st, rs_last_error());
      h_written[g] = wr;
    }
    // the report from the global grid (first GPU)
    RS_CUDA(cudaSetDevice(h_devices[0]));
    reset_stats(w0);
    scan_pass(w0, grids[0], cells, n_total);
    {
      PassTimer pt_(RS_PASS_REPORT, w0.stream);
      k_report<uint32_t><<<1, report_threads(10), 0, w0.stream>>>(static_cast<const uint32_t*>(w0.buf[kSlotOccCell]),
                                                                  0, 10, digits, 0, 0, w0.stats, true);
      RS_LAUNCH_CHECK();
    }
    pull_stats(w0);
    if (report) *report = rs_report{n_total, w0.h_stats->cells_traversed, spec};
  });
}

rs_status rs_sort_u32_kv(const uint32_t* keys, const uint32_t* vals, uint64_t n, uint32_t* keys_out,
                         uint32_t* vals_out, uint64_t out_capacity, const rs_options* opt,
                         rs_report* report, void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (n == 0) {
      if (report) *report = rs_report{0, 0, make_key_spec(10, 1, 1, budget)};
      return;
    }
    if (!keys || !vals || !keys_out || !vals_out) fail(RS_INVALID_ARGUMENT, "null device pointer");
    // positions and per-chunk offsets are uint32: fewer than 2^32 records per call
    if (n > 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "rs_sort_u32_kv takes fewer than 2^32 records per call");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const uint32_t hint = opt ? opt->key_digits : 0;
    const bool hinted = hint >= 1 && hint <= 10 && pow10u(hint) <= budget;
    uint32_t digits = hinted ? hint : digit_count(device_max(ws, keys, n, MapU32{}));
    make_key_spec(10, digits, digits, budget);
    if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
    kv_sort(ws, keys, vals, n, digits, keys_out, vals_out);
    if (digit_count(ws.h_stats->max_key) > digits) {
      digits = digit_count(ws.h_stats->max_key);
      make_key_spec(10, digits, digits, budget);
      kv_sort(ws, keys, vals, n, digits, keys_out, vals_out);
    }
    const uint32_t d = static_cast<uint32_t>(ws.h_stats->report_digits);
    if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{10, d, d}};
  });
}

extern "C++" {
// Alphabet (key_model.cpp:190-223) as a device table in ws kSlotAlphabet, the
// data's width (longest record, key_model.cpp:228-230) and symbol check by
// one scan; `packed` (optional) receives the MSD-packed keys.
struct StrSetup {
  StrTable t;
  size_t alen;
  int lin;            // contiguous alphabet: ordinal = byte - lin
  uint32_t obits;     // bits of the largest ordinal
  const uint16_t* d_ord;
  const uint8_t* d_sym;
  uint32_t w;         // width of the data (>= 1)
  bool bad;           // a symbol outside the alphabet
};

StrSetup str_setup(Workspace& ws, const uint8_t* chars, uint64_t n, uint32_t width, const char* h_alphabet,
                   unsigned long long* packed) {
  StrSetup r{};
  const char* alpha = h_alphabet ? h_alphabet : "abcdefghijklmnopqrstuvwxyz";
  r.alen = strlen(alpha);
  if (r.alen == 0) fail(RS_INVALID_ARGUMENT, "alphabet is empty");  // Alphabet(), key_model.cpp:190-201
  for (size_t i = 0; i < r.alen; ++i) {
    const auto c = static_cast<unsigned char>(alpha[i]);
    if (r.t.ord[c] != 0) fail(RS_INVALID_ARGUMENT, std::string("duplicate symbol '") + alpha[i] + "' in alphabet");
    r.t.ord[c] = static_cast<uint16_t>(i + 1);
    r.t.sym[i + 1] = c;
  }
  r.t.radix = static_cast<uint32_t>(r.alen) + 1;
  r.lin = static_cast<int>(static_cast<unsigned char>(alpha[0])) - 1;
  for (size_t i = 1; i < r.alen; ++i)
    if (static_cast<unsigned char>(alpha[i]) != static_cast<unsigned char>(alpha[0]) + i) r.lin = -1;
  if (static_cast<unsigned char>(alpha[0]) == 0) r.lin = -1;
  r.obits = 1;
  while ((r.alen >> r.obits) != 0) ++r.obits;
  auto* tab = ws.get<uint8_t>(kSlotAlphabet, sizeof(StrTable));
  RS_CUDA(cudaMemcpyAsync(tab, &r.t, sizeof(StrTable), cudaMemcpyHostToDevice, ws.stream));
  r.d_ord = reinterpret_cast<const uint16_t*>(tab);
  r.d_sym = tab + offsetof(StrTable, sym);
  r.w = 1;
  if (n == 0) return r;
  reset_stats(ws);
  {
    PassTimer pt_(RS_PASS_OTHER, ws.stream);
    const bool w8 = width == 8 && (reinterpret_cast<uintptr_t>(chars) & 15) == 0;
    auto scan = r.obits == 5 ? k_str_scan<5> : k_str_scan<0>;
    scan<<<stream_grid(n, kThreads * 4, 8), kThreads, 0, ws.stream>>>(chars, n, width, w8, r.d_ord, ws.stats, packed,
                                                                      r.lin, static_cast<uint32_t>(r.alen), r.obits);
    RS_LAUNCH_CHECK();
  }
  pull_stats(ws);
  r.bad = (ws.h_stats->flags & 8u) != 0;
  r.w = ws.h_stats->max_key ? static_cast<uint32_t>(ws.h_stats->max_key) : 1u;
  return r;
}

// The first symbol outside the alphabet in (record, position) order, raised
// as Alphabet::ordinal does (key_model.cpp:208-214, 233-241).
[[noreturn]] void fail_first_symbol(Workspace& ws, const uint8_t* chars, uint64_t n, uint32_t width,
                                    const uint16_t* d_ord) {
  auto* first = ws.get<unsigned long long>(kSlotScratch, 4);
  RS_CUDA(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), ws.stream));
  k_str_first_bad<<<stream_grid(n, kThreads * 4, 8), kThreads, 0, ws.stream>>>(chars, n, width, d_ord, first);
  RS_LAUNCH_CHECK();
  unsigned long long at = 0;
  RS_CUDA(cudaMemcpyAsync(&at, first, sizeof(at), cudaMemcpyDeviceToHost, ws.stream));
  RS_CUDA(cudaStreamSynchronize(ws.stream));
  uint8_t c = 0;
  if (at < n * width) RS_CUDA(cudaMemcpy(&c, chars + at, 1, cudaMemcpyDeviceToHost));
  fail(RS_SYMBOL_OUT_OF_ALPHABET, std::string("symbol '") + static_cast<char>(c) + "' is not in the alphabet");
}

// strings_to_keys' keys at width w into `keys` (base-radix, pad ordinal 0)
void str_keys(Workspace& ws, const uint8_t* chars, uint64_t n, uint32_t width, const StrSetup& su,
              unsigned long long* keys) {
  PassTimer pt_(RS_PASS_OTHER, ws.stream);
  k_str_keys<<<stream_grid(n, kThreads * 4, 8), kThreads, 0, ws.stream>>>(chars, n, width, su.w, su.t.radix, su.d_ord,
                                                                            keys, ws.stats);
  RS_LAUNCH_CHECK();
}
}  // extern "C++"

rs_status rs_sort_fixed_str(const uint8_t* chars, uint64_t n, uint32_t width, const char* h_alphabet,
                            uint8_t* out, uint64_t out_capacity, const rs_options* opt,
                            rs_report* report, void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (width == 0) fail(RS_INVALID_ARGUMENT, "record width must be at least 1");
    if (n > 0 && (!chars || !out)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    // width of the data = longest string (key_model.cpp:228-230), symbols checked;
    // with msd the same pass packs the keys the MSD levels read
    size_t alen = h_alphabet ? strlen(h_alphabet) : 26;
    uint32_t obits = 1;
    while ((alen >> obits) != 0) ++obits;
    const bool want_msd = opt && opt->msd && width * obits <= 64;
    unsigned long long* packed = want_msd && n ? ws.get<unsigned long long>(kSlotMisc2, n) : nullptr;
    const StrSetup su = str_setup(ws, chars, n, width, h_alphabet, packed);
    if (n == 0) {
      if (report) *report = rs_report{0, 0, make_key_spec(su.t.radix, 1, 1, budget)};
      return;
    }
    const uint32_t w = su.w;
    const uint64_t total_cells = [&] {
      try { return checked_pow(su.t.radix, w); } catch (const Failure&) { return ~uint64_t{0}; }
    }();
    const bool msd = want_msd;  // MSD needs the packed key to fit 64 bits; else the reference's budget error
    if (!msd || total_cells <= budget) {
      const rs_key_spec spec = make_key_spec(su.t.radix, w, w, budget);
      if (su.bad) fail_first_symbol(ws, chars, n, width, su.d_ord);  // after the key spec, as strings_to_keys orders them
      if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
      auto* keys = ws.get<unsigned long long>(kSlotMapped, n);
      str_keys(ws, chars, n, width, su, keys);
      OutStr o{out, width, w, su.t.radix, su.d_sym, 0ull};
      grid_sort(ws, keys, n, MapU64{}, total_cells, o, keys, su.t.radix, w, 0);
      if (report) *report = rs_report{n, ws.h_stats->cells_traversed, spec};
      return;
    }
    if (su.bad) fail_first_symbol(ws, chars, n, width, su.d_ord);
    if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
    msd_sort_str(ws, chars, n, width, w, su.t.radix, su.d_ord, su.d_sym, out, su.lin, packed, su.obits);
    if (report) *report = rs_report{n, ws.h_stats->cells_traversed, rs_key_spec{su.t.radix, w, w}};
  });
}

rs_status rs_strings_to_keys(const uint8_t* chars, uint64_t n, uint32_t width, const char* h_alphabet,
                             uint64_t* keys_out, const rs_options* opt, rs_key_spec* h_spec, void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (width == 0) fail(RS_INVALID_ARGUMENT, "record width must be at least 1");
    if (n > 0 && (!chars || !keys_out)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const StrSetup su = str_setup(ws, chars, n, width, h_alphabet, nullptr);
    const rs_key_spec spec = make_key_spec(su.t.radix, su.w, su.w, budget);  // budget before symbols
    if (n > 0) {
      if (su.bad) fail_first_symbol(ws, chars, n, width, su.d_ord);
      str_keys(ws, chars, n, width, su, reinterpret_cast<unsigned long long*>(keys_out));
      RS_CUDA(cudaStreamSynchronize(ws.stream));
    }
    if (h_spec) *h_spec = spec;
  });
}

extern "C++" {
// TraverseMaps (hashing.hpp:12-48) of a count grid: per leading-digit row the
// least and greatest occupied suffix (row_min ~0 / row_max -1 while a row is
// untouched).  A warp's cells mostly share a row: its lanes reduce first.
__global__ void k_row_bounds(const unsigned long long* __restrict__ counts, uint64_t cells, unsigned long long mod,
                             unsigned long long* __restrict__ row_min, long long* __restrict__ row_max) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t base0 = (uint64_t)blockIdx.x * blockDim.x;
  for (uint64_t b = base0; b < cells; b += stride) {  // warp-uniform trip count
    const uint64_t c = b + threadIdx.x;
    const bool occ = c < cells && counts[c] != 0;
    const unsigned long long row = occ ? c / mod : ~0ull;
    const unsigned long long suf = occ ? c - row * mod : 0ull;
    const unsigned long long r0 = __shfl_sync(0xffffffffu, row, 0);
    const bool same = __all_sync(0xffffffffu, !occ || row == r0);
    if (same && r0 != ~0ull) {
      unsigned long long mn = occ ? suf : ~0ull, mx = occ ? suf : 0ull;
      bool any = occ;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), d = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = d > mx ? d : mx;
      }
      any = __any_sync(0xffffffffu, any);
      if ((threadIdx.x & 31) == 0 && any) {
        atomicMin(&row_min[r0], mn);
        atomicMax(&row_max[r0], static_cast<long long>(mx));
      }
    } else if (occ) {
      atomicMin(&row_min[row], suf);
      atomicMax(&row_max[row], static_cast<long long>(suf));
    }
  }
}

// extract's traversal set (extraction.cpp:16-30): cells inside their row's
// [min, max] span of an occupied row keep their count, the rest read as 0.
__global__ void k_mask_counts(const unsigned long long* __restrict__ counts, uint64_t cells, unsigned long long mod,
                              const unsigned long long* __restrict__ row_min, const long long* __restrict__ row_max,
                              unsigned long long* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += stride) {
    const unsigned long long row = c / mod, suf = c - row * mod;
    const long long hi = row_max[row];
    out[c] = (hi >= 0 && suf >= row_min[row] && suf <= static_cast<unsigned long long>(hi)) ? counts[c] : 0ull;
  }
}

// The occupied cell holding output position pos (the cell whose emission
// completes `pos + 1` keys).
__global__ void k_cell_at(const uint32_t* __restrict__ occ_cell, const unsigned long long* __restrict__ occ_end,
                          const DevStats* st, unsigned long long pos, unsigned long long* out) {
  unsigned long long lo = 0, hi = st->n_occupied;
  while (lo < hi) {
    const unsigned long long mid = (lo + hi) >> 1;
    if (occ_end[mid] > pos) hi = mid;
    else lo = mid + 1;
  }
  *out = lo < st->n_occupied ? occ_cell[lo] : ~0ull;
}

// counts (uint64 grid) += the keys' cells, chunk by chunk through the uint32
// counting pass (fewer than 2^32 keys per chunk: no counter wraps)
template <class Map>
void count_into_u64(Workspace& ws, const typename Map::In* in, uint64_t n, Map map, uint64_t cells,
                    unsigned long long* wide) {
  auto* counts = ws.get<uint32_t>(kSlotCounts, cells);
  for (uint64_t off = 0; off < n; off += kCountChunk) {
    const uint64_t len = std::min<uint64_t>(kCountChunk, n - off);
    count_pass(ws, in + off, len, map, cells, counts);
    PassTimer pt_(RS_PASS_COUNT, ws.stream);
    k_grid_acc64<<<stream_grid(cells, kThreads * 4), kThreads, 0, ws.stream>>>(wide, counts, cells);
    RS_LAUNCH_CHECK();
  }
}
}  // extern "C++"

rs_status rs_build_count_space(const uint64_t* keys, uint64_t n, rs_key_spec spec, uint64_t max_cells,
                               uint64_t* counts, uint64_t* h_row_min, int64_t* h_row_max, void* stream) {
  return guarded([&] {
    ensure_device();
    make_key_spec(spec.radix, spec.total_digits, spec.integer_digits, ~uint64_t{0});  // the geometry itself
    const uint64_t cells = checked_pow(spec.radix, spec.total_digits);
    if (cells > max_cells)  // new_space (hashing.cpp:17-25): the budget before any allocation
      fail(RS_CELL_BUDGET_EXCEEDED,
           "count space needs " + std::to_string(cells) + " cells, budget is " + std::to_string(max_cells));
    if (cells > 0xFFFFFFFFull) fail(RS_CELL_BUDGET_EXCEEDED, "a single grid holds at most 2^32-1 cells");
    if (!counts || (n > 0 && !keys)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    reset_stats(ws);
    auto* wide = reinterpret_cast<unsigned long long*>(counts);
    RS_CUDA(cudaMemsetAsync(wide, 0, cells * sizeof(uint64_t), ws.stream));
    if (n > 0) count_into_u64(ws, reinterpret_cast<const unsigned long long*>(keys), n, MapU64{}, cells, wide);
    const unsigned long long mod = checked_pow(spec.radix, spec.total_digits - 1);
    auto* rows = ws.get<unsigned long long>(kSlotHist, 2ull * spec.radix);
    auto* rmax = reinterpret_cast<long long*>(rows + spec.radix);
    RS_CUDA(cudaMemsetAsync(rows, 0xff, 2ull * spec.radix * sizeof(uint64_t), ws.stream));  // min ~0, max -1
    {
      PassTimer pt_(RS_PASS_SCAN, ws.stream);
      k_row_bounds<<<stream_grid(cells, kThreads * 4), kThreads, 0, ws.stream>>>(wide, cells, mod, rows, rmax);
      RS_LAUNCH_CHECK();
    }
    if (h_row_min) RS_CUDA(cudaMemcpyAsync(h_row_min, rows, spec.radix * sizeof(uint64_t), cudaMemcpyDeviceToHost, ws.stream));
    if (h_row_max) RS_CUDA(cudaMemcpyAsync(h_row_max, rmax, spec.radix * sizeof(int64_t), cudaMemcpyDeviceToHost, ws.stream));
    pull_stats(ws);
    if (ws.h_stats->overflow) fail(RS_SPEC_MISMATCH, "a key is outside its spec's key space");
  });
}

rs_status rs_extract(const uint64_t* counts, rs_key_spec spec, uint64_t total, const uint64_t* h_row_min,
                     const int64_t* h_row_max, uint64_t* out, uint64_t out_capacity, rs_report* report,
                     void* stream) {
  return guarded([&] {
    ensure_device();
    make_key_spec(spec.radix, spec.total_digits, spec.integer_digits, ~uint64_t{0});
    const uint64_t cells = checked_pow(spec.radix, spec.total_digits);
    if (cells > 0xFFFFFFFFull) fail(RS_CELL_BUDGET_EXCEEDED, "a single grid holds at most 2^32-1 cells");
    if (out_capacity < total)  // extraction.cpp:8-12
      fail(RS_BUFFER_TOO_SMALL, "output buffer holds " + std::to_string(out_capacity) + " keys, need " +
                                    std::to_string(total));
    if (!counts || !h_row_min || !h_row_max || (total > 0 && !out)) fail(RS_INVALID_ARGUMENT, "null pointer");
    const unsigned long long mod = checked_pow(spec.radix, spec.total_digits - 1);
    // cells_traversed: every occupied row's span, unless the output fills up
    // inside one (then up to the cell that completes it)
    unsigned long long spans = 0;
    for (uint32_t r = 0; r < spec.radix; ++r)
      if (h_row_max[r] >= 0) spans += static_cast<unsigned long long>(h_row_max[r]) - h_row_min[r] + 1;
    if (total == 0) {
      if (report) *report = rs_report{0, 0, spec};
      return;
    }
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    reset_stats(ws);
    auto* rows = ws.get<unsigned long long>(kSlotHist, 2ull * spec.radix + 1);
    auto* rmax = reinterpret_cast<long long*>(rows + spec.radix);
    RS_CUDA(cudaMemcpyAsync(rows, h_row_min, spec.radix * sizeof(uint64_t), cudaMemcpyHostToDevice, ws.stream));
    RS_CUDA(cudaMemcpyAsync(rmax, h_row_max, spec.radix * sizeof(int64_t), cudaMemcpyHostToDevice, ws.stream));
    auto* masked = ws.get<unsigned long long>(kSlotCounts64, cells);
    k_mask_counts<<<stream_grid(cells, kThreads * 4), kThreads, 0, ws.stream>>>(
        reinterpret_cast<const unsigned long long*>(counts), cells, mod, rows, rmax, masked);
    RS_LAUNCH_CHECK();
    scan_pass(ws, static_cast<const unsigned long long*>(masked), cells, total);
    pull_stats(ws);  // (also orders the host arrays above)
    const unsigned long long sum = ws.h_stats->total;
    const uint64_t written = std::min<uint64_t>(total, sum);
    unsigned long long traversed = spans;
    if (sum > total) {
      // more keys in the spans than were inserted: the raster stops at the
      // cell that completes `total` (extraction.cpp:27); tile starts for that length
      const uint32_t etiles = static_cast<uint32_t>((total + kEmitTile - 1) / kEmitTile);
      k_tile_first<<<(etiles + 1 + 255) / 256, 256, 0, ws.stream>>>(
          static_cast<unsigned long long*>(ws.buf[kSlotOccEnd]), ws.stats, total, etiles,
          static_cast<uint32_t*>(ws.buf[kSlotTileFirst]));
      auto* at = ws.get<unsigned long long>(kSlotScratch, 4);
      k_cell_at<<<1, 1, 0, ws.stream>>>(static_cast<uint32_t*>(ws.buf[kSlotOccCell]),
                                        static_cast<unsigned long long*>(ws.buf[kSlotOccEnd]), ws.stats, total - 1, at);
      RS_LAUNCH_CHECK();
      unsigned long long stop = 0;
      RS_CUDA(cudaMemcpyAsync(&stop, at, sizeof(stop), cudaMemcpyDeviceToHost, ws.stream));
      RS_CUDA(cudaStreamSynchronize(ws.stream));
      const unsigned long long srow = stop / mod, ssuf = stop - srow * mod;
      traversed = 0;
      for (uint32_t r = 0; r < srow; ++r)
        if (h_row_max[r] >= 0) traversed += static_cast<unsigned long long>(h_row_max[r]) - h_row_min[r] + 1;
      traversed += ssuf - h_row_min[srow] + 1;
    }
    if (written > 0) {
      OutU64 o{reinterpret_cast<unsigned long long*>(out), 0ull, aligned32(out)};
      emit_pass(ws, written, o);
    }
    RS_CUDA(cudaStreamSynchronize(ws.stream));
    if (report) *report = rs_report{written, traversed, spec};
  });
}

rs_status rs_checked_pow(uint64_t radix, uint32_t exp, uint64_t* h_out) {
  return guarded([&] {
    const uint64_t v = checked_pow(radix, exp);
    if (h_out) *h_out = v;
  });
}

rs_status rs_make_key_spec(uint32_t radix, uint32_t total_digits, uint32_t integer_digits, uint64_t max_cells,
                           rs_key_spec* h_spec) {
  return guarded([&] {
    const rs_key_spec s = make_key_spec(radix, total_digits, integer_digits, max_cells);
    if (h_spec) *h_spec = s;
  });
}

rs_status rs_bucket_hist_u32(const uint32_t* keys, uint64_t n, uint64_t divisor, uint64_t* hist,
                             uint32_t buckets, void* stream) {
  return guarded([&] {
    ensure_device();
    if (divisor == 0 || buckets == 0) fail(RS_INVALID_ARGUMENT, "divisor and buckets must be positive");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    reset_stats(ws);
    RS_CUDA(cudaMemsetAsync(hist, 0, buckets * sizeof(uint64_t), ws.stream));
    if (n > 0) {
      const unsigned long long magic = divisor == 1 ? 0ull : magic_div(divisor);
      const size_t smem = buckets <= kMsdSmemBuckets ? buckets * sizeof(uint32_t) : 0;
      {
        PassTimer pt_(RS_PASS_MSD_HIST, ws.stream);
        k_bucket_hist<<<stream_grid(n, kMsdThreads * 16, 8), kMsdThreads, smem, ws.stream>>>(
            keys, n, magic, buckets, reinterpret_cast<unsigned long long*>(hist), ws.stats);
        RS_LAUNCH_CHECK();
      }
    }
    pull_stats(ws);
    if (ws.h_stats->overflow) fail(RS_OUT_OF_RANGE, "a key's bucket is beyond `buckets`");
  });
}

// Per-part counts and the scatter of rs_partition_u32, shared with the
// multi-GPU exchange (rs_part_counts_u32 / rs_partition_u32_to).
extern "C++" {
struct PartSetup {
  unsigned long long magic;
  uint32_t* d_bounds;
  unsigned long long* counts;
  unsigned long long* cursors;
  uint32_t** d_dst;
};

PartSetup part_setup(Workspace& ws, uint64_t divisor, const uint32_t* h_bounds, uint32_t parts) {
  if (parts == 0 || parts > 1024) fail(RS_INVALID_ARGUMENT, "parts must be in [1, 1024]");
  if (divisor == 0) fail(RS_INVALID_ARGUMENT, "divisor must be positive");
  for (uint32_t p = 0; p < parts; ++p)
    if (h_bounds[p] > h_bounds[p + 1]) fail(RS_INVALID_RANGE, "part bounds must be non-decreasing");
  auto* scratch = ws.get<unsigned long long>(kSlotHist, 2048 + 1024 + 1025);
  PartSetup s;
  s.counts = scratch;
  s.cursors = scratch + 1024;
  s.d_dst = reinterpret_cast<uint32_t**>(scratch + 2048);
  s.d_bounds = reinterpret_cast<uint32_t*>(scratch + 3072);
  s.magic = divisor == 1 ? 0ull : magic_div(divisor);
  RS_CUDA(cudaMemcpyAsync(s.d_bounds, h_bounds, (parts + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, ws.stream));
  return s;
}

std::vector<unsigned long long> part_counts(Workspace& ws, const uint32_t* keys, uint64_t n, const PartSetup& s,
                                            uint32_t parts) {
  std::vector<unsigned long long> hc(parts, 0);
  RS_CUDA(cudaMemsetAsync(s.counts, 0, parts * sizeof(unsigned long long), ws.stream));
  if (n > 0) {
    PassTimer pt_(RS_PASS_MSD_HIST, ws.stream);
    k_part_count<<<stream_grid(n, kMsdThreads * 16, 8), kMsdThreads, 0, ws.stream>>>(keys, n, s.magic, s.d_bounds,
                                                                                     parts, s.counts);
    RS_LAUNCH_CHECK();
  }
  RS_CUDA(cudaMemcpyAsync(hc.data(), s.counts, parts * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ws.stream));
  RS_CUDA(cudaStreamSynchronize(ws.stream));
  return hc;
}

void part_scatter(Workspace& ws, const uint32_t* keys, uint64_t n, const PartSetup& s, uint32_t parts,
                  const uint64_t* h_dst, const unsigned long long* h_cursor0) {
  RS_CUDA(cudaMemcpyAsync(s.cursors, h_cursor0, parts * sizeof(unsigned long long), cudaMemcpyHostToDevice, ws.stream));
  RS_CUDA(cudaMemcpyAsync(s.d_dst, h_dst, parts * sizeof(uint64_t), cudaMemcpyHostToDevice, ws.stream));
  if (n > 0) {
    PassTimer pt_(RS_PASS_MSD_SCATTER, ws.stream);
    k_part_scatter<<<stream_grid(n, kPartChunk, 4), kMsdThreads, 0, ws.stream>>>(keys, n, s.magic, s.d_bounds, parts,
                                                                                 s.cursors, s.d_dst);
    RS_LAUNCH_CHECK();
  }
  RS_CUDA(cudaStreamSynchronize(ws.stream));  // the host arrays above are stack memory
}
}  // extern "C++"

rs_status rs_partition_u32(const uint32_t* keys, uint64_t n, uint64_t divisor, const uint32_t* h_bounds,
                           uint32_t parts, uint32_t* out, uint64_t* h_counts, void* stream) {
  return guarded([&] {
    ensure_device();
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const PartSetup s = part_setup(ws, divisor, h_bounds, parts);
    const std::vector<unsigned long long> hc = part_counts(ws, keys, n, s, parts);
    std::vector<unsigned long long> starts(parts, 0);
    std::vector<uint64_t> dst(parts, reinterpret_cast<uint64_t>(out));
    unsigned long long run = 0;
    for (uint32_t p = 0; p < parts; ++p) {
      starts[p] = run;
      run += hc[p];
    }
    if (n > 0) part_scatter(ws, keys, n, s, parts, dst.data(), starts.data());
    if (h_counts)
      for (uint32_t p = 0; p < parts; ++p) h_counts[p] = hc[p];
  });
}

rs_status rs_part_counts_u32(const uint32_t* keys, uint64_t n, uint64_t divisor, const uint32_t* h_bounds,
                             uint32_t parts, uint64_t* h_counts, void* stream) {
  return guarded([&] {
    ensure_device();
    if (!h_counts) fail(RS_INVALID_ARGUMENT, "null counts");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const PartSetup s = part_setup(ws, divisor, h_bounds, parts);
    const std::vector<unsigned long long> hc = part_counts(ws, keys, n, s, parts);
    for (uint32_t p = 0; p < parts; ++p) h_counts[p] = hc[p];
  });
}

rs_status rs_partition_u32_to(const uint32_t* keys, uint64_t n, uint64_t divisor, const uint32_t* h_bounds,
                              uint32_t parts, const uint64_t* h_dst, const uint64_t* h_offsets, void* stream) {
  return guarded([&] {
    ensure_device();
    if (!h_dst || !h_offsets) fail(RS_INVALID_ARGUMENT, "null destination arrays");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const PartSetup s = part_setup(ws, divisor, h_bounds, parts);
    std::vector<unsigned long long> cur(h_offsets, h_offsets + parts);
    part_scatter(ws, keys, n, s, parts, h_dst, cur.data());
  });
}

// Host-buffer entry points: H2D, sort, D2H in one call on `stream`.
rs_status rs_sort_u32_host(const uint32_t* h_keys, uint64_t n, uint32_t* h_out, const rs_options* opt,
                           rs_report* report, void* stream) {
  return guarded([&] {
    ensure_device();
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    // staging slots of their own: no internal pass of the sort reuses them
    uint32_t* d_in = ws.get<uint32_t>(kSlotHostIn, n ? n : 1);
    uint32_t* d_out = ws.get<uint32_t>(kSlotHostOut, n ? n : 1);
    if (n) RS_CUDA(cudaMemcpyAsync(d_in, h_keys, n * 4, cudaMemcpyHostToDevice, ws.stream));
    const rs_status st = rs_sort_u32(d_in, n, d_out, n, opt, report, stream);
    if (st != RS_OK) throw Failure{st, g_last_error};
    if (n) RS_CUDA(cudaMemcpyAsync(h_out, d_out, n * 4, cudaMemcpyDeviceToHost, ws.stream));
    RS_CUDA(cudaStreamSynchronize(ws.stream));
  });
}

rs_status rs_sort_u32_kv_host(const uint32_t* h_keys, const uint32_t* h_vals, uint64_t n, uint32_t* h_keys_out,
                              uint32_t* h_vals_out, const rs_options* opt, rs_report* report, void* stream) {
  return guarded([&] {
    ensure_device();
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const uint64_t m = n ? n : 1;
    uint32_t* d_k = ws.get<uint32_t>(kSlotHostIn, 2 * m);
    uint32_t* d_v = d_k + m;
    uint32_t* d_ko = ws.get<uint32_t>(kSlotHostOut, 2 * m);
    uint32_t* d_vo = d_ko + m;
    if (n) {
      RS_CUDA(cudaMemcpyAsync(d_k, h_keys, n * 4, cudaMemcpyHostToDevice, ws.stream));
      RS_CUDA(cudaMemcpyAsync(d_v, h_vals, n * 4, cudaMemcpyHostToDevice, ws.stream));
    }
    const rs_status st = rs_sort_u32_kv(d_k, d_v, n, d_ko, d_vo, n, opt, report, stream);
    if (st != RS_OK) throw Failure{st, g_last_error};
    if (n) {
      RS_CUDA(cudaMemcpyAsync(h_keys_out, d_ko, n * 4, cudaMemcpyDeviceToHost, ws.stream));
      RS_CUDA(cudaMemcpyAsync(h_vals_out, d_vo, n * 4, cudaMemcpyDeviceToHost, ws.stream));
    }
    RS_CUDA(cudaStreamSynchronize(ws.stream));
  });
}

// ------------------------------------------------------------- phase API
rs_status rs_kv_place_u32(const uint32_t* keys, const uint32_t* vals, uint64_t n, const int64_t* cell_off,
                          const uint8_t* cell_owner, uint64_t cells, const uint64_t* h_dst_keys,
                          const uint64_t* h_dst_vals, uint32_t ranks, void* stream) {
  return guarded([&] {
    ensure_device();
    if (ranks == 0 || ranks > 64) fail(RS_INVALID_ARGUMENT, "ranks must be in [1, 64]");
    if (n > 0 && (!keys || !vals || !cell_off || !cell_owner)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    if (!h_dst_keys || !h_dst_vals) fail(RS_INVALID_ARGUMENT, "null destination arrays");
    if (cells == 0 || cells > 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "cells out of range");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    auto* d = ws.get<unsigned long long>(kSlotMisc, 129);
    auto* bad = reinterpret_cast<unsigned*>(d + 128);
    RS_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), ws.stream));
    RS_CUDA(cudaMemcpyAsync(d, h_dst_keys, ranks * sizeof(uint64_t), cudaMemcpyHostToDevice, ws.stream));
    RS_CUDA(cudaMemcpyAsync(d + 64, h_dst_vals, ranks * sizeof(uint64_t), cudaMemcpyHostToDevice, ws.stream));
    if (n > 0) {
      PassTimer pt_(RS_PASS_KV_SCATTER, ws.stream);
      k_kv_place<<<stream_grid(n, 256 * 8, 8), 256, 0, ws.stream>>>(
          keys, vals, n, reinterpret_cast<const long long*>(cell_off), cell_owner, reinterpret_cast<uint32_t* const*>(d),
          reinterpret_cast<uint32_t* const*>(d + 64), ranks, cells, bad);
      RS_LAUNCH_CHECK();
    }
    unsigned h_bad = 0;
    RS_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, ws.stream));
    RS_CUDA(cudaStreamSynchronize(ws.stream));  // the host pointer arrays are the caller's
    if (h_bad) fail(RS_OUT_OF_RANGE, "a key lies outside the placement grid or its owner is not a rank");
  });
}

rs_status rs_count_u32(const uint32_t* keys, uint64_t n, uint32_t* counts, uint64_t cells,
                       uint32_t* h_max, void* stream) {
  return guarded([&] {
    ensure_device();
    if (cells == 0 || cells > 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "cells out of range");
    // uint32 counters: fewer than 2^32 keys per call, so no cell can wrap
    if (n > kCountChunk) fail(RS_INVALID_ARGUMENT, "rs_count_u32 counts fewer than 2^32 keys per call");
    if (n > 0 && (!keys || !counts)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    reset_stats(ws);
    count_pass(ws, keys, n, MapU32{}, cells, counts);  // same counting pass as rs_sort_u32
    pull_stats(ws);
    if (h_max) *h_max = static_cast<uint32_t>(ws.h_stats->max_key);
    // a key outside the grid would silently drop out of the counts
    if (ws.h_stats->overflow) fail(RS_OUT_OF_RANGE, "a key lies outside the grid of " + std::to_string(cells) + " cells");
  });
}

rs_status rs_emit_part_u32(const uint32_t* counts, uint64_t cells, uint32_t part, uint32_t parts, uint32_t* out,
                           uint64_t out_capacity, uint64_t* h_written, uint64_t* h_cells, void* stream) {
  return guarded([&] {
    ensure_device();
    if (parts == 0 || part >= parts || parts > 1024) fail(RS_INVALID_ARGUMENT, "part must be < parts <= 1024");
    if (cells == 0 || cells > 0xFFFFFFFFull) fail(RS_INVALID_ARGUMENT, "cells out of range");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    // cut r (1 <= r < parts) = 1 + the cell whose inclusive prefix first
    // reaches ceil(r * total / parts): the global prefix and the cuts on the
    // device, two cut values back to the host
    uint64_t lo = 0, hi = cells;
    if (parts > 1) {
      auto* excl = ws.get<uint32_t>(kSlotTmpKeys, cells);
      auto* tot = ws.get<unsigned long long>(kSlotScratch, 4 + 1024);
      auto* cuts = tot + 4;
      RS_CUDA(cudaMemsetAsync(cuts, 0xff, (parts - 1) * sizeof(unsigned long long), ws.stream));  // ~0: past the grid
      exscan_u32(ws, counts, cells, excl, tot);
      k_grid_cuts<<<stream_grid(cells, kThreads * 4), kThreads, 0, ws.stream>>>(excl, counts, cells, tot, parts, cuts);
      RS_LAUNCH_CHECK();
      std::vector<unsigned long long> h(parts - 1);
      RS_CUDA(cudaMemcpyAsync(h.data(), cuts, (parts - 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              ws.stream));
      RS_CUDA(cudaStreamSynchronize(ws.stream));
      // monotone and inside the grid (dist.cell_ranges' clamping)
      uint64_t prev = 0;
      for (uint32_t r = 1; r < parts; ++r) {
        const uint64_t c = std::max<uint64_t>(prev, std::min<uint64_t>(h[r - 1], cells));
        if (r == part) lo = c;
        if (r == part + 1) hi = c;
        prev = c;
      }
    }
    if (h_cells) {
      h_cells[0] = lo;
      h_cells[1] = hi;
    }
    const rs_status st = rs_emit_u32(counts, cells, lo, hi, 0, out, out_capacity, h_written, stream);
    if (st != RS_OK) throw Failure{st, g_last_error};
  });
}

rs_status rs_emit_u32(const uint32_t* counts, uint64_t cells, uint64_t cell_lo, uint64_t cell_hi,
                      uint32_t key_base, uint32_t* out, uint64_t out_capacity,
                      uint64_t* h_written, void* stream) {
  return guarded([&] {
    ensure_device();
    if (cell_lo > cell_hi || cell_hi > cells) fail(RS_INVALID_RANGE, "bad cell range");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    reset_stats(ws);
    const uint64_t span = cell_hi - cell_lo;
    uint64_t written = 0;
    if (span > 0) {
      // scan the sub-range to learn how many keys it holds
      const uint32_t tiles = static_cast<uint32_t>((span + kScanTile - 1) / kScanTile);
      auto* desc = ws.get<unsigned long long>(kSlotTileDesc, 2ull * tiles);
      auto* occ_cell = ws.get<uint32_t>(kSlotOccCell, span);
      auto* occ_end = ws.get<unsigned long long>(kSlotOccEnd, span);
      RS_CUDA(cudaMemsetAsync(desc, 0, 2ull * tiles * 8, ws.stream));
      {
        PassTimer pt_(RS_PASS_SCAN, ws.stream);
        k_scan_cells<<<tiles, kThreads, 0, ws.stream>>>(counts + cell_lo, span, occ_cell, occ_end, desc,
                                                         desc + tiles, tiles, ws.stats, 0, nullptr, nullptr);
        RS_LAUNCH_CHECK();
      }
      pull_stats(ws);
      written = ws.h_stats->total;
      if (written > out_capacity) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
      if (written > 0) {
        const uint32_t etiles = static_cast<uint32_t>((written + kEmitTile - 1) / kEmitTile);
        auto* tile_first = ws.get<uint32_t>(kSlotTileFirst, etiles + 1ull);
        {
          PassTimer pt_(RS_PASS_SCAN, ws.stream);
          k_tile_first<<<(etiles + 1 + 255) / 256, 256, 0, ws.stream>>>(occ_end, ws.stats, written,
                                                                        etiles, tile_first);
          RS_LAUNCH_CHECK();
        }
        OutU32 o{out, static_cast<uint32_t>(key_base + cell_lo), aligned16(out)};
        emit_pass(ws, written, o);
      }
    }
    if (h_written) *h_written = written;
  });
}


extern "C++" {
// parse_decimal over a device string column into ws mant (kSlotMapped) /
// own scales (kSlotTmpKeys); the first failing numeral in input order raises
// the reference's error.  Returns the dataset's max scale / max integer part.
DecStats decimal_parse(Workspace& ws, const char* chars, const uint64_t* offsets, uint64_t n,
                       uint32_t* scale_u32 = nullptr) {
  auto* mant = ws.get<unsigned long long>(kSlotMapped, n);
  auto* own = ws.get<uint8_t>(kSlotTmpKeys, n);
  auto* ds = reinterpret_cast<DecStats*>(ws.get<uint8_t>(kSlotAlphabet, sizeof(StrTable)));
  const auto* off = reinterpret_cast<const unsigned long long*>(offsets);
  RS_CUDA(cudaMemsetAsync(ds, 0, sizeof(DecStats), ws.stream));
  RS_CUDA(cudaMemsetAsync(&ds->first_error, 0xff, sizeof(unsigned long long), ws.stream));
  {
    PassTimer pt_(RS_PASS_OTHER, ws.stream);
    k_dec_parse<<<stream_grid(n, kThreads * 4, 8), kThreads, 0, ws.stream>>>(chars, off, n, mant, own, ds, scale_u32);
    RS_LAUNCH_CHECK();
  }
  DecStats h{};
  RS_CUDA(cudaMemcpyAsync(&h, ds, sizeof(h), cudaMemcpyDeviceToHost, ws.stream));
  RS_CUDA(cudaStreamSynchronize(ws.stream));
  if (h.first_error != ~0ull) {  // the numeral the reference's loop stops at
    const uint64_t i = h.first_error >> 8;
    unsigned long long be[2];
    RS_CUDA(cudaMemcpy(be, off + i, sizeof(be), cudaMemcpyDeviceToHost));
    std::string text(be[1] - be[0], '\0');
    if (!text.empty()) RS_CUDA(cudaMemcpy(text.data(), chars + be[0], text.size(), cudaMemcpyDeviceToHost));
    const size_t dot = text.find('.');
    fail_numeral(static_cast<uint32_t>(h.first_error & 0xff), text,
                 dot == std::string::npos ? 0u : static_cast<uint32_t>(text.size() - dot - 1));
  }
  return h;
}

// normalize_dataset (key_model.cpp:107-133): lambda from the largest integer
// part, the dataset scale from the longest fraction; keys (in ws kSlotMapped)
// = mantissa * 10^(scale - own scale).
rs_key_spec decimal_normalize(Workspace& ws, const char* chars, const uint64_t* offsets, uint64_t n,
                              uint64_t budget) {
  const DecStats h = decimal_parse(ws, chars, offsets, n);
  const uint32_t scale = h.max_scale;
  const uint32_t lambda = digit_count(h.max_integer);
  const rs_key_spec spec = make_key_spec(10, lambda + scale, lambda, budget);
  PassTimer pt_(RS_PASS_OTHER, ws.stream);
  k_dec_scale<<<stream_grid(n, kThreads * 4, 8), kThreads, 0, ws.stream>>>(
      static_cast<unsigned long long*>(ws.buf[kSlotMapped]), static_cast<const uint8_t*>(ws.buf[kSlotTmpKeys]), n,
      scale);
  RS_LAUNCH_CHECK();
  return spec;
}
}  // extern "C++"

rs_status rs_sort_decimal_strings(const char* chars, const uint64_t* offsets, uint64_t n, uint64_t* keys_out,
                                  uint64_t out_capacity, const rs_options* opt, rs_report* report, void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (n == 0) {
      if (report) *report = rs_report{0, 0, make_key_spec(10, 1, 1, budget)};
      return;
    }
    if (!offsets || !keys_out || !chars) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const rs_key_spec spec = decimal_normalize(ws, chars, offsets, n, budget);
    if (out_capacity < n) fail(RS_BUFFER_TOO_SMALL, "output buffer too small");
    auto* mant = static_cast<const unsigned long long*>(ws.buf[kSlotMapped]);
    OutU64 o{reinterpret_cast<unsigned long long*>(keys_out), 0ull, aligned32(keys_out)};
    grid_sort(ws, mant, n, MapU64{}, checked_pow(10, spec.total_digits), o, keys_out, 10, spec.total_digits, 0);
    if (report) *report = rs_report{n, ws.h_stats->cells_traversed, spec};
  });
}

rs_status rs_normalize_decimal_strings(const char* chars, const uint64_t* offsets, uint64_t n, uint64_t* keys_out,
                                       const rs_options* opt, rs_key_spec* h_spec, void* stream) {
  return guarded([&] {
    ensure_device();
    const uint64_t budget = budget_of(opt);
    if (n == 0) {
      if (h_spec) *h_spec = make_key_spec(10, 1, 1, budget);
      return;
    }
    if (!offsets || !keys_out || !chars) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    const rs_key_spec spec = decimal_normalize(ws, chars, offsets, n, budget);
    RS_CUDA(cudaMemcpyAsync(keys_out, ws.buf[kSlotMapped], n * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                            ws.stream));
    RS_CUDA(cudaStreamSynchronize(ws.stream));
    if (h_spec) *h_spec = spec;
  });
}

rs_status rs_parse_decimals(const char* chars, const uint64_t* offsets, uint64_t n, uint64_t* mantissas,
                            uint32_t* scales, void* stream) {
  return guarded([&] {
    ensure_device();
    if (n == 0) return;
    if (!offsets || !chars || !mantissas || !scales) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    decimal_parse(ws, chars, offsets, n, scales);
    RS_CUDA(cudaMemcpyAsync(mantissas, ws.buf[kSlotMapped], n * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                            ws.stream));
    RS_CUDA(cudaStreamSynchronize(ws.stream));
  });
}

rs_status rs_format_decimals(const uint64_t* keys, uint64_t n, uint32_t scale, char* out_chars,
                             uint64_t out_chars_capacity, uint64_t* out_offsets, uint64_t* h_chars_needed,
                             void* stream) {
  return guarded([&] {
    ensure_device();
    if (scale > 19) fail(RS_INVALID_ARGUMENT, "scale must be at most 19");
    if (!out_offsets || (n && !keys)) fail(RS_INVALID_ARGUMENT, "null device pointer");
    Workspace& ws = workspace_for(static_cast<cudaStream_t>(stream));
    auto* off = reinterpret_cast<unsigned long long*>(out_offsets);
    unsigned long long total = 0;
    if (n == 0) {
      RS_CUDA(cudaMemsetAsync(off, 0, sizeof(unsigned long long), ws.stream));
    } else {
      const auto* k = reinterpret_cast<const unsigned long long*>(keys);
      const uint32_t tiles = static_cast<uint32_t>((n + kScanTile - 1) / kScanTile);
      auto* desc = ws.get<unsigned long long>(kSlotDesc2, tiles + 1ull);
      RS_CUDA(cudaMemsetAsync(desc, 0, (tiles + 1ull) * sizeof(unsigned long long), ws.stream));
      PassTimer pt_(RS_PASS_OTHER, ws.stream);
      k_dec_offsets<<<tiles, kThreads, 0, ws.stream>>>(k, n, scale, off, desc, reinterpret_cast<unsigned*>(desc + tiles),
                                                       tiles);
      RS_LAUNCH_CHECK();
      RS_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(total), cudaMemcpyDeviceToHost, ws.stream));
    }
    RS_CUDA(cudaStreamSynchronize(ws.stream));
    if (h_chars_needed) *h_chars_needed = total;
    if (total > out_chars_capacity) fail(RS_BUFFER_TOO_SMALL, "output character buffer too small");
    if (n) {
      if (!out_chars) fail(RS_INVALID_ARGUMENT, "null device pointer");
      PassTimer pt_(RS_PASS_OTHER, ws.stream);
      k_dec_format_staged<<<stream_grid(n, kDecFmtKeys * 4, 8), kDecFmtKeys, 0, ws.stream>>>(
          reinterpret_cast<const unsigned long long*>(keys), n, scale, off, out_chars);
      RS_LAUNCH_CHECK();
      RS_CUDA(cudaStreamSynchronize(ws.stream));
    }
  });
}

}  // extern "C"


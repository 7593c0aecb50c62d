// test_facade.cpp — the reference's facade cases (proj/tests/test_facade.cpp,
// test_extraction.cpp, acceptance.cpp c01/c09, test_smoke.py) restated against
// the B200 library through the drop-in header recsort/sort.hpp.  Built and
// run by tests/test_cpp_facade.py on a GPU box.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "recsort/sort.hpp"

static int g_fail = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                      \
    }                                                                \
  } while (0)
#define CHECK_FAILS_WITH(expr, want_code)                            \
  do {                                                               \
    bool threw_ = false;                                             \
    try {                                                            \
      (void)(expr);                                                  \
    } catch (const recsort::Error& e_) {                             \
      threw_ = true;                                                 \
      CHECK(e_.code() == (want_code));                               \
    }                                                                \
    CHECK(threw_);                                                   \
  } while (0)

using namespace recsort;

int main() {
  // worked example, cost 17 (test_extraction.cpp:30-40, acceptance.cpp:46-69)
  {
    const std::vector<std::string> in{"4.5", "0.3", "2.3", "8.8", "7", "9.2", "4.5", "4.3", "8", "3.2"};
    const DecimalSortResult r = sort_decimals(in);
    const std::vector<std::string> want{"0.3", "2.3", "3.2", "4.3", "4.5", "4.5", "7.0", "8.0", "8.8", "9.2"};
    CHECK(r.values == want);
    CHECK(r.report.written == 10);
    CHECK(r.report.cells_traversed == 17);
    CHECK((r.spec == KeySpec{10, 2, 1}));
  }
  // integers (test_facade.cpp)
  {
    const std::vector<std::int64_t> in{45, 3, 23, 88, 70, 92, 45, 43, 80, 32};
    const IntegerSortResult r = sort_integers(in);
    CHECK((r.values == std::vector<std::int64_t>{3, 23, 32, 43, 45, 45, 70, 80, 88, 92}));
    CHECK(r.report.cells_traversed == 17);
    const std::vector<std::int64_t> neg{3, -1};
    CHECK_FAILS_WITH(sort_integers(neg), errc::negative_value);
    const std::vector<std::int64_t> empty{};
    CHECK(sort_integers(empty).report.written == 0);
    std::vector<std::int64_t> big(10000);
    unsigned s = 7;
    for (auto& v : big) v = (s = s * 1103515245u + 12345u) % 100;
    IntegerSortResult rb = sort_integers(big);
    std::sort(big.begin(), big.end());
    CHECK(rb.values == big);
  }
  // strings (test_facade.cpp:74-79, test_smoke.py)
  {
    const std::vector<std::string> in{"ba", "ab", "aa", "b"};
    const StringSortResult r = sort_strings(in, Alphabet::lowercase());
    CHECK((r.values == std::vector<std::string>{"aa", "ab", "b", "ba"}));
    const std::vector<std::string> bad{"aZ"};
    CHECK_FAILS_WITH(sort_strings(bad, Alphabet::lowercase()), errc::symbol_out_of_alphabet);
    const std::vector<std::string> wide{"zzzzzz"};
    CHECK_FAILS_WITH(sort_strings(wide, Alphabet::lowercase()), errc::cell_budget_exceeded);
    CHECK_FAILS_WITH(Alphabet("aa"), errc::invalid_argument);
  }
  // budget and parse errors (acceptance.cpp:292-314 c09, test_key_model.cpp:67-78)
  {
    const std::vector<std::string> wide{"123456789012"};
    CHECK_FAILS_WITH(sort_decimals(wide), errc::cell_budget_exceeded);
    const std::vector<std::string> bad{"1.2.3"};
    CHECK_FAILS_WITH(sort_decimals(bad), errc::parse_error);
    const std::vector<std::string> neg{"-3"};
    CHECK_FAILS_WITH(sort_decimals(neg), errc::negative_value);
  }
  // recombinant_sort over device memory: uint32 keys, key/value, MSD
  {
    const std::uint64_t n = 1 << 20;
    std::vector<std::uint32_t> h(n), v(n);
    unsigned s = 11;
    for (std::uint64_t i = 0; i < n; ++i) {
      h[i] = (s = s * 1664525u + 1013904223u) % 1000000u;
      v[i] = static_cast<std::uint32_t>(i);
    }
    std::uint32_t *dk, *dv, *dko, *dvo;
    cudaMalloc(&dk, n * 4);
    cudaMalloc(&dv, n * 4);
    cudaMalloc(&dko, n * 4);
    cudaMalloc(&dvo, n * 4);
    cudaMemcpy(dk, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), n * 4, cudaMemcpyHostToDevice);
    const ExtractionReport r = recombinant_sort(dk, n, dko);
    std::vector<std::uint32_t> got(n), gotv(n);
    cudaMemcpy(got.data(), dko, n * 4, cudaMemcpyDeviceToHost);
    std::vector<std::uint32_t> want = h;
    std::sort(want.begin(), want.end());
    CHECK(got == want);
    CHECK(r.written == n);
    recombinant_sort(dk, dv, n, dko, dvo);
    cudaMemcpy(got.data(), dko, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(gotv.data(), dvo, n * 4, cudaMemcpyDeviceToHost);
    CHECK(got == want);
    bool stable = true;
    for (std::uint64_t i = 1; i < n; ++i)
      if (got[i] == got[i - 1] && gotv[i] < gotv[i - 1]) stable = false;
    CHECK(stable);
    for (std::uint64_t i = 0; i < n; ++i) h[i] = (s = s * 1664525u + 1013904223u);
    cudaMemcpy(dk, h.data(), n * 4, cudaMemcpyHostToDevice);
    CHECK_FAILS_WITH(recombinant_sort(dk, n, dko), errc::cell_budget_exceeded);
    SortOptions msd;
    msd.msd = true;
    recombinant_sort(dk, n, dko, msd);
    cudaMemcpy(got.data(), dko, n * 4, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    CHECK(got == h);
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dko);
    cudaFree(dvo);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}

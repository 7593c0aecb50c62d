"""Pins the CPU oracle (oracle/oracle.cpp) before it is trusted as the GPU
checker: the reference's own known answers and golden vectors, the committed
fixtures generated from the reference library, and — where oracle/_ref was
built — a live differential against the reference."""
import numpy as np
import pytest

from oracle import OracleError

ST_CELL_BUDGET_EXCEEDED = 4
ST_NEGATIVE = 2
ST_NON_FINITE = 3
ST_SPEC_MISMATCH = 6
ST_SYMBOL = 5


# ------------------------------------------------------ known answers
def test_splitmix_known_answers(oracle, golden):
    # test_bench.cpp:16-22
    assert oracle.splitmix_stream(42, 1)[0] == 0xBDD732262FEB6E95
    assert oracle.next_unit(42) == 0.7415648787718233
    assert oracle.splitmix_stream(42, 8) == [int(x) for x in golden["splitmix42_first8"]]


def test_splitmix_counter_addressable(oracle):
    # element i == mix(seed + (i+1)*golden)
    seq = oracle.splitmix_stream(123456789, 5000)
    assert [oracle.L.or_sm64_at(123456789, i) for i in range(5000)] == seq


def test_worked_example_extracts_with_cost_17(oracle):
    # test_extraction.cpp:30-40, acceptance.cpp:46-69
    out, rep = oracle.sort_keys(np.array([45, 3, 23, 88, 70, 92, 45, 43, 80, 32]), (10, 2, 1))
    assert out.tolist() == [3, 23, 32, 43, 45, 45, 70, 80, 88, 92]
    assert rep[:2] == (10, 17)


def test_single_and_all_equal_cost_one_cell(oracle):
    # test_extraction.cpp:42-56
    assert oracle.sort_keys(np.array([57]), (10, 2, 1))[1][1] == 1
    out, rep = oracle.sort_keys(np.full(23, 66), (10, 2, 1))
    assert out.tolist() == [66] * 23 and rep[1] == 1


def test_sorted_input_is_identity(oracle):
    keys = np.array([3, 23, 32, 43, 45, 45, 70, 80, 88, 92])
    assert oracle.sort_keys(keys, (10, 2, 1))[0].tolist() == keys.tolist()


def test_differential_10k_four_digit(oracle):
    # test_extraction.cpp:65-71
    keys = oracle.gen_u32(0x4D16, 0, 10000, 10**4).astype(np.uint64)
    out, rep = oracle.sort_keys(keys, (10, 4, 4))
    assert np.array_equal(out, np.sort(keys))
    assert rep[1] == oracle.report_from_sorted(out, 10, 4)[1]


def test_spans_equal_traversal_cost(oracle):
    # test_extraction.cpp:135-154 (F4): k == sum of occupied row spans
    for inst in range(20):
        keys = oracle.gen_u32(0xC057 + inst, 0, 1 + inst * 2, 100).astype(np.uint64)
        out, rep = oracle.sort_keys(keys, (10, 2, 1))
        rows = {}
        for k in keys.tolist():
            r, s = divmod(k, 10)
            lo, hi = rows.get(r, (s, s))
            rows[r] = (min(lo, s), max(hi, s))
        assert rep[1] == sum(hi - lo + 1 for lo, hi in rows.values())


def test_float_to_decimal_half_up(oracle):
    # test_key_model.cpp:80-93
    assert oracle.float_to_decimal(4.5, 1) == 45
    assert oracle.float_to_decimal(0.0, 3) == 0
    assert oracle.float_to_decimal(2.345, 2) == 235
    assert oracle.float_to_decimal(0.285, 2) == 29
    assert oracle.float_to_decimal(2.344, 2) == 234
    assert oracle.float_to_decimal(7.0, 0) == 7
    assert oracle.float_to_decimal_status(-1.0, 2)[0] == ST_NEGATIVE
    assert oracle.float_to_decimal_status(float("nan"), 1)[0] == ST_NON_FINITE
    assert oracle.float_to_decimal_status(float("inf"), 1)[0] == ST_NON_FINITE


def test_float_to_decimal_matches_golden(oracle, golden):
    xs = golden["f2d_x"]
    for scale in (0, 1, 2, 3, 4, 6):
        want = golden[f"f2d_scale{scale}"]
        got = np.array([oracle.float_to_decimal(float(x), scale) for x in xs], dtype=np.uint64)
        assert np.array_equal(got, want), scale


def test_budget_guards(oracle):
    # test_key_model.cpp:211-222, acceptance.cpp:292-314 (c09)
    with pytest.raises(OracleError) as e:
        oracle.sort_keys(np.array([1]), (10, 9, 9))
    assert e.value.status == ST_CELL_BUDGET_EXCEEDED
    with pytest.raises(OracleError) as e:
        oracle.sort_integers_i64(np.array([123456789012]))
    assert e.value.status == ST_CELL_BUDGET_EXCEEDED
    with pytest.raises(OracleError) as e:
        oracle.strings_to_keys(np.frombuffer(b"zzzzzz", dtype=np.uint8).reshape(1, 6))
    assert e.value.status == ST_CELL_BUDGET_EXCEEDED


def test_errors(oracle):
    with pytest.raises(OracleError) as e:
        oracle.sort_integers_i64(np.array([3, -1]))
    assert e.value.status == ST_NEGATIVE
    with pytest.raises(OracleError) as e:
        oracle.sort_keys(np.array([100]), (10, 2, 1))
    assert e.value.status == ST_SPEC_MISMATCH  # hashing.cpp:31-34
    with pytest.raises(OracleError) as e:
        oracle.strings_to_keys(np.frombuffer(b"aZ", dtype=np.uint8).reshape(1, 2))
    assert e.value.status == ST_SYMBOL


def test_string_keys_order_and_pad(oracle):
    # test_key_model.cpp:158-180
    recs = np.zeros((3, 2), dtype=np.uint8)
    for i, s in enumerate([b"ba", b"ab", b"aa"]):
        recs[i, : len(s)] = list(s)
    keys, spec = oracle.strings_to_keys(recs)
    assert spec == (27, 2, 2)
    assert keys[2] < keys[1] < keys[0]
    recs = np.zeros((2, 2), dtype=np.uint8)
    recs[0, 0] = ord("b")
    recs[1, :] = [ord("b"), ord("a")]
    keys, _ = oracle.strings_to_keys(recs)
    assert keys[0] < keys[1]  # end padding keeps the prefix first


def test_kv_stability(oracle):
    # test_baselines.cpp:41-56
    k = oracle.gen_u32(0x57AB, 0, 2000, 50)
    v = np.arange(2000, dtype=np.uint32)
    ko, vo = oracle.radix_sort_lsd_kv(k, v)
    assert np.all(ko[1:] >= ko[:-1])
    same = ko[1:] == ko[:-1]
    assert np.all(vo[1:][same] > vo[:-1][same])


# ------------------------------------------------------ golden fixtures
def test_oracle_matches_reference_golden(oracle, golden):
    for cfg in ("cfg1", "cfg2"):
        out, rep = oracle.sort_integers_u32(golden[f"{cfg}_keys"])
        assert np.array_equal(out, golden[f"{cfg}_sorted"])
        assert list(rep[:2]) + list(rep[2]) == golden[f"{cfg}_report"].tolist()
    ko, vo = oracle.radix_sort_lsd_kv(golden["kv_keys"], golden["kv_vals"])
    assert np.array_equal(ko, golden["kv_sorted_keys"]) and np.array_equal(vo, golden["kv_sorted_vals"])
    out, rep = oracle.sort_f64(golden["cfg3_x"], 3)
    assert np.array_equal(out, golden["cfg3_sorted"])
    assert list(rep[:2]) + list(rep[2]) == golden["cfg3_report"].tolist()
    keys, _ = oracle.strings_to_keys(golden["str_recs"], "abc")
    assert np.array_equal(keys, golden["str_keys"])
    out, rep = oracle.sort_fixed_strings(golden["str_recs"], "abc")
    assert np.array_equal(out, golden["str_sorted"])
    assert list(rep[:2]) + list(rep[2]) == golden["str_report"].tolist()
    out, _ = oracle.sort_fixed_strings(golden["cfg4_recs"])
    assert np.array_equal(out, golden["cfg4_sorted"])


def test_generators_match_golden(oracle, golden):
    assert np.array_equal(oracle.gen_u32(oracle.config_seed(1), 0, 4096, 1000), golden["cfg1_keys"])
    cdf = oracle.zipf_cdf()
    assert np.array_equal(oracle.gen_f64_cfg3(oracle.config_seed(3), 0, 4096, cdf), golden["cfg3_x"])
    assert np.array_equal(oracle.gen_str_cfg4(oracle.config_seed(4), 0, 3000), golden["cfg4_recs"])


# ------------------------------------------- live reference differential
def test_oracle_vs_reference_integers(oracle, ref):
    for inst, (n, bound) in enumerate([(1, 10), (7, 10), (1000, 100), (5000, 10**4), (30000, 10**6),
                                       (3000, 10**7)]):
        keys = oracle.gen_u32(0xD1FF + inst, 0, n, bound)
        a, ra = oracle.sort_integers_u32(keys)
        b, rb = ref.sort_integers(keys.astype(np.int64))
        assert np.array_equal(a.astype(np.int64), b) and ra == rb


def test_oracle_vs_reference_float_to_decimal(oracle, ref):
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.random(20000) * 1000, rng.random(5000) * 1e-3,
                         np.exp(rng.uniform(-40, 40, 5000)), [1e-300, 1e300, 2.0**64]])
    for scale in (0, 2, 3, 5):
        for x in xs:
            assert oracle.float_to_decimal_status(float(x), scale) == ref.float_to_decimal_status(float(x), scale)


def test_oracle_vs_reference_strings_and_kv(oracle, ref):
    recs = oracle.gen_str_cfg4(99, 0, 5000)
    assert np.array_equal(oracle.sort_fixed_strings(recs)[0], ref.oracle_sort_strings(recs))
    short = recs[:, :4].copy()
    short[::3, 3] = 0
    a, ra = oracle.sort_fixed_strings(short)
    b, rb = ref.sort_strings(short)
    assert np.array_equal(a, b) and ra == rb
    k = oracle.gen_u32(5, 0, 20000, 10**6)
    v = np.arange(20000, dtype=np.uint32)
    ka, va = oracle.radix_sort_lsd_kv(k, v)
    kb, vb = ref.radix_sort_lsd_kv(k, v)
    assert np.array_equal(ka, kb) and np.array_equal(va, vb)

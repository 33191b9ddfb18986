"""Pin the C restatement (oracle/kvq_oracle.c) before trusting it as the parity checker.

CPU only. Three anchors:
  1. the reference's own known-answer tests (tests/test_bitpack.cpp, test_quantize.cpp,
     test_kernels.cpp, test_calibrate.cpp, test_kvcache.cpp; cited per test);
  2. the golden fixtures in tests/golden/ generated from the unmodified reference
     (tests/golden/make_golden.py) — compared BIT-EXACTLY;
  3. the live reference build (oracle/_ref/libkvq_ref.so) where it exists, on random
     sweeps, plus the documented reference defect at kernels.hpp:220.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def bits_eq(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.uint32)
    b = np.ascontiguousarray(b, np.float32).view(np.uint32)
    return a.shape == b.shape and np.array_equal(a, b)


# ---- 1. reference known answers ----------------------------------------------------------

def test_pack_worked_examples(oracle):
    # test_bitpack.cpp:12-52
    assert oracle.pack([3, 1, 0, 2], 2, 8)[1].tolist() == [210]
    assert oracle.pack([1, 0, 1, 1, 0, 0, 1, 0], 1, 8)[1].tolist() == [178]
    assert oracle.pack([1, 2, 3], 4, 16)[1].tolist() == [0x30, 0x12]
    assert oracle.pack([3, 3, 3, 3, 3], 2, 8)[1].tolist() == [0xFF, 0xC0]
    assert oracle.pack([4], 2, 8)[0] == 2  # domain error (test_bitpack.cpp:126-131)
    assert oracle.pack([1], 3, 8)[0] == 1  # config error (133-140)


def test_pack_word_count_law(oracle):
    # test_bitpack.cpp:54-67
    for count, n, m, words in [(17, 4, 8, 9), (33, 1, 32, 2), (8, 8, 8, 8), (16, 2, 16, 2), (1, 1, 8, 1)]:
        st, out = oracle.pack(np.ones(count, np.uint32), n, m)
        assert st == 0 and out.size == words * (m // 8)


def test_pack_exhaustive_single_word(oracle):
    # acceptance.cpp:47-75: every word value round-trips for (1,8),(2,8),(4,8),(8,8),(1,16),(2,16)
    for n, m in [(1, 8), (2, 8), (4, 8), (8, 8), (1, 16), (2, 16)]:
        g = m // n
        words = np.arange(1 << m, dtype=np.uint32)
        codes = np.stack([(words >> (m - n * (k + 1))) & ((1 << n) - 1) for k in range(g)], 1).reshape(-1)
        st, packed = oracle.pack(codes, n, m)
        assert st == 0
        back = packed.view(np.uint8 if m == 8 else np.uint16)
        assert np.array_equal(back.astype(np.uint32), words)
        assert np.array_equal(oracle.unpack(packed, codes.size, n, m), codes)


def test_quantize_hand_values(oracle):
    # test_quantize.cpp:47-67
    def q1(x, a, b, bits):
        return int(oracle.unpack(oracle.quantize(np.array([[x]], np.float32), [a], [b], bits), 1, bits)[0])

    assert q1(1.4, 0.0, 3.0, 2) == 1
    assert q1(0.1, -2.0, 2.0, 1) == 1
    assert [q1(x, 0.0, 3.0, 2) for x in (0.5, 1.5, 2.5)] == [1, 2, 3]  # ties away from zero
    for bits in (1, 2, 4, 8):
        L = (1 << bits) - 1
        assert q1(-1.5, -1.5, 2.5, bits) == 0 and q1(2.5, -1.5, 2.5, bits) == L
        assert q1(99.0, -1.5, 2.5, bits) == L and q1(-99.0, -1.5, 2.5, bits) == 0


def test_stats_and_degenerate_channel(oracle):
    # test_quantize.cpp:34-45, 69-80
    a, b = oracle.compute_stats(np.array([[1, 5], [3, 2]], np.float32), 0)
    assert a.tolist() == [1, 2] and b.tolist() == [3, 5]
    a, b = oracle.compute_stats(np.array([[1, 5], [3, 2]], np.float32), 1)
    assert a.tolist() == [1, 1] and b.tolist() == [5, 5]
    m = np.array([[4, 1], [4, 2], [4, 3]], np.float32)
    a, b = oracle.compute_stats(m, 0)
    codes = oracle.unpack(oracle.quantize(m, a, b, 2), 12, 2)
    assert codes.reshape(3, 4)[:, 0].tolist() == [0, 0, 0]
    assert oracle.dequantize(oracle.quantize(m, a, b, 2), 3, 2, a, b, 2)[:, 0].tolist() == [4, 4, 4]


def test_kernel_hand_values(oracle):
    # test_kernels.cpp:37-46: 1-bit q=(2,3), codes (1,0) -> 2
    k = np.array([[1.0, 0.0]], np.float32)
    codes = oracle.quantize(k, [0, 0], [1, 1], 1)
    assert oracle.qk_scores([2, 3], codes, 1, 2, [0, 0], [1, 1], 1).tolist() == [2.0]
    # integer-valued inputs make the fused paths exact (94-109)
    rng = np.random.default_rng(5)
    kk = rng.integers(0, 4, size=(12, 8)).astype(np.float32)
    q = rng.integers(-4, 5, size=8).astype(np.float32)
    codes = oracle.quantize(kk, np.zeros(8), np.full(8, 3.0), 2)
    deq = oracle.dequantize(codes, 12, 8, np.zeros(8), np.full(8, 3.0), 2)
    assert np.array_equal(oracle.qk_scores(q, codes, 12, 8, np.zeros(8), np.full(8, 3.0), 2), deq @ q)


def test_calibration_hand_values(oracle):
    # test_calibrate.cpp:60-66, 90-95, 134-147
    assert oracle.g_apply(0.0, 0.0, 10.0, 2.0, 1.0) == -2.0
    assert oracle.g_apply(10.0, 0.0, 10.0, 2.0, 1.0) == 9.0
    assert oracle.g_apply(5.0, 0.0, 10.0, 2.0, 1.0) == 3.5
    assert oracle.g_apply(7.0, 4.0, 4.0, 2.0, 1.0) == 5.0
    row, _ = oracle.calibrated_softmax_concat([0.0, 10.0], [9.0], 2.0, 1.0)
    e = np.exp(np.array([-2.0, 9.0, 9.0], np.float32) - np.float32(9.0))
    assert np.allclose(row, e / e.sum(), rtol=1e-6)
    _, viol = oracle.calibrated_softmax_concat([0.0, 1e-4], [], 0.0, 3.0)
    assert viol == 1


# ---- 2. golden fixtures (bit-exact) ------------------------------------------------------

def test_quant_fixtures(oracle):
    z = np.load(GOLD / "quant_cases.npz")
    for i in range(int(z["count"])):
        bits, wb, mode = z[f"c{i}_meta"].tolist()
        x = z[f"c{i}_x"]
        if mode >= 0:
            a, b = oracle.compute_stats(x, mode)
            assert bits_eq(a, z[f"c{i}_alpha"]) and bits_eq(b, z[f"c{i}_beta"]), f"stats case {i}"
        codes = oracle.quantize(x, z[f"c{i}_alpha"], z[f"c{i}_beta"], bits, wb)
        assert np.array_equal(codes, z[f"c{i}_codes"]), f"codes case {i}"


def test_kernel_fixtures(oracle):
    z = np.load(GOLD / "kernels.npz")
    for i in range(int(z["count"])):
        bits, wb, tokens, dim = z[f"k{i}_meta"].tolist()
        args = (z[f"k{i}_codes"], tokens, dim, z[f"k{i}_alpha"], z[f"k{i}_beta"], bits, wb)
        assert bits_eq(oracle.qk_scores(z[f"k{i}_q"], *args), z[f"k{i}_scores"]), f"qk case {i}"
        assert bits_eq(oracle.wv_output(z[f"k{i}_w"], *args), z[f"k{i}_wv"]), f"wv case {i}"
    for j in range(int(z["scount"])):
        t1, t2 = z[f"s{j}_tau"].tolist()
        row, viol = oracle.calibrated_softmax_concat(z[f"s{j}_vis"], z[f"s{j}_tail"], t1, t2)
        assert bits_eq(row, z[f"s{j}_row"]) and viol == int(z[f"s{j}_viol"]), f"softmax case {j}"


def load_inputs(z, oracle):
    h, n, d = z["meta"][:3].tolist()
    if "k" in z:
        return z["k"], z["v"]
    seed = int(z["seed"])
    ks, vs = [], []
    for hh in range(h):
        k, v, _ = oracle.generate_head(seed, hh, n, d)
        ks.append(k)
        vs.append(v)
    k, v = np.stack(ks), np.stack(vs)
    assert hashlib.sha256(k.tobytes() + v.tobytes()).hexdigest() == str(z["sha256"]), "generator drift"
    return k, v


DECODE_FIXTURES = sorted(p.name for p in GOLD.glob("decode_*.npz"))


@pytest.mark.parametrize("name", DECODE_FIXTURES)
def test_decode_fixtures(oracle, name):
    z = np.load(GOLD / name)
    h, n, d, bits, wb, steps = z["meta"].tolist()
    t1, t2 = z["tau"].tolist()
    k, v = load_inputs(z, oracle)
    segs = []
    for hh in range(h):
        if bits == 16:
            segs.append(None)
            continue
        ka, kb = oracle.compute_stats(k[hh], 0) if n else (np.zeros(d), np.zeros(d))
        va, vb = oracle.compute_stats(v[hh], 0) if n else (np.zeros(d), np.zeros(d))
        kc = oracle.quantize(k[hh], ka, kb, bits, wb) if n else np.zeros(0, np.uint8)
        vc = oracle.quantize(v[hh], va, vb, bits, wb) if n else np.zeros(0, np.uint8)
        if n:
            assert np.array_equal(kc, z[f"kcodes{hh}"]) and np.array_equal(vc, z[f"vcodes{hh}"])
            assert bits_eq(ka, z[f"kalpha{hh}"]) and bits_eq(vb, z[f"vbeta{hh}"])
        segs.append((kc, ka, kb, vc, va, vb))
    tails_k = [[] for _ in range(h)]
    tails_v = [[] for _ in range(h)]
    for t in range(steps):
        q = z[f"q{t}"]
        for hh in range(h):
            if bits == 16:  # full precision: prefill lives in the tail
                kt = np.concatenate([k[hh]] + [np.array(tails_k[hh]).reshape(-1, d)])
                vt = np.concatenate([v[hh]] + [np.array(tails_v[hh]).reshape(-1, d)])
                o, w, viol = oracle.decode_head(q[hh], 0, 8, 8, [], [], [], [], [], [], kt, vt, t1, t2)
            else:
                kc, ka, kb, vc, va, vb = segs[hh]
                o, w, viol = oracle.decode_head(q[hh], n, bits, wb, kc, ka, kb, vc, va, vb,
                                                np.array(tails_k[hh]), np.array(tails_v[hh]), t1, t2)
            assert bits_eq(o, z[f"out{t}"][hh]), f"{name} step {t} head {hh} output"
            assert bits_eq(w, z[f"w{t}"][hh]), f"{name} step {t} head {hh} weights"
        for hh in range(h):
            tails_k[hh].append(z[f"knew{t}"][hh])
            tails_v[hh].append(z[f"vnew{t}"][hh])


# ---- 3. live reference ----------------------------------------------------------------------

def test_generator_matches_reference(oracle, ref):
    k, v, q = ref.generate(99, 3, 17, 9)
    for h in range(3):
        ok, ov, oq = oracle.generate_head(99, h, 17, 9)
        assert bits_eq(ok, k[h]) and bits_eq(ov, v[h]) and bits_eq(oq, q[h])
    sq, sk, sv = ref.generate_step(99, 3, 9, 5)
    for h in range(3):
        oq, ok, ov = oracle.generate_step_head(99, h, 5, 9)
        assert bits_eq(oq, sq[h]) and bits_eq(ok, sk[h]) and bits_eq(ov, sv[h])


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("wb", [8, 16, 32])
def test_random_sweep_vs_reference(oracle, ref, bits, wb):
    if wb % bits:
        pytest.skip("invalid width pair")
    rng = np.random.default_rng(bits * 100 + wb)
    for _ in range(6):
        n, d = int(rng.integers(1, 200)), int(rng.integers(1, 70))
        m = rng.uniform(-4, 4, size=(n, d)).astype(np.float32)
        a, b = oracle.compute_stats(m, 0)
        ra, rb = ref.compute_stats(m, 0)
        assert bits_eq(a, ra) and bits_eq(b, rb)
        codes = oracle.quantize(m, a, b, bits, wb)
        assert np.array_equal(codes, ref.quantize(m, a, b, bits, wb))
        q = rng.uniform(-1, 1, size=d).astype(np.float32)
        w = rng.uniform(0, 1, size=n).astype(np.float32)
        assert bits_eq(oracle.qk_scores(q, codes, n, d, a, b, bits, wb), ref.qk_scores(q, codes, n, d, a, b, bits, wb))
        assert bits_eq(oracle.wv_output(w, codes, n, d, a, b, bits, wb), ref.wv_output(w, codes, n, d, a, b, bits, wb))


def test_table_path_b1_matches_reference(oracle, ref):
    # n >= 512 at M = 8 takes the reference's byte-table path (kernels.hpp:252); for
    # b = 1 its w*8 stride is correct, so the oracle must agree bit for bit.
    rng = np.random.default_rng(3)
    m = rng.normal(size=(700, 128)).astype(np.float32)
    a, b = oracle.compute_stats(m, 0)
    codes = oracle.quantize(m, a, b, 1, 8)
    q = rng.normal(size=128).astype(np.float32)
    assert bits_eq(oracle.qk_scores(q, codes, 700, 128, a, b, 1, 8), ref.qk_scores(q, codes, 700, 128, a, b, 1, 8))


@pytest.mark.parametrize("bits", [2, 4])
def test_reference_table_path_defect_documented(oracle, ref, bits):
    """kernels.hpp:220 strides the scaled query by 8 instead of codes-per-word: for
    b >= 2, M = 8, n >= 512 every reference score is wrong. The oracle
    implements the intended math, which the reference's own M = 32 path and its
    dequantize-then-dense product both confirm."""
    rng = np.random.default_rng(bits)
    n, d = 600, 128
    m = rng.normal(size=(n, d)).astype(np.float32)
    a, b = oracle.compute_stats(m, 0)
    q = rng.normal(size=d).astype(np.float32)
    c8 = oracle.quantize(m, a, b, bits, 8)
    c32 = oracle.quantize(m, a, b, bits, 32)
    mine = oracle.qk_scores(q, c8, n, d, a, b, bits, 8)
    wide = ref.qk_scores(q, c32, n, d, a, b, bits, 32)
    dense = ref.dequantize(c8, n, d, a, b, bits, 8) @ q
    assert np.allclose(mine, wide, rtol=1e-5, atol=1e-4 * np.abs(wide).max())
    assert np.allclose(mine, dense, rtol=1e-5, atol=1e-4 * np.abs(dense).max())
    buggy = ref.qk_scores(q, c8, n, d, a, b, bits, 8)
    # The defect is real: garbage (often NaN/inf) scores from the over-read.
    assert not np.allclose(buggy, wide, rtol=1e-2, atol=1e-2 * np.abs(wide).max())


def test_decode_matches_reference_cache(oracle, ref):
    rng = np.random.default_rng(17)
    for bits, wb in [(1, 8), (2, 8), (4, 16), (8, 32)]:
        h, n, d = 2, 50, 12
        k = rng.uniform(-2, 2, size=(h, n, d)).astype(np.float32)
        v = rng.uniform(-2, 2, size=(h, n, d)).astype(np.float32)
        cache = ref.cache_build(k, v, bits, wb, 2.0, 0.5)
        kt, vt = [[] for _ in range(h)], [[] for _ in range(h)]
        for t in range(3):
            q = rng.uniform(-1, 1, size=(h, d)).astype(np.float32)
            ro, rw, _ = cache.decode(q, n + t)
            for hh in range(h):
                ka, kb = oracle.compute_stats(k[hh])
                va, vb = oracle.compute_stats(v[hh])
                o, w, _ = oracle.decode_head(q[hh], n, bits, wb, oracle.quantize(k[hh], ka, kb, bits, wb), ka, kb,
                                             oracle.quantize(v[hh], va, vb, bits, wb), va, vb,
                                             np.array(kt[hh]), np.array(vt[hh]), 2.0, 0.5)
                assert bits_eq(o, ro[hh]) and bits_eq(w, rw[hh])
            kn = rng.uniform(-2, 2, size=(h, d)).astype(np.float32)
            vn = rng.uniform(-2, 2, size=(h, d)).astype(np.float32)
            cache.append(kn, vn)
            for hh in range(h):
                kt[hh].append(kn[hh])
                vt[hh].append(vn[hh])


def test_grid_search_oracle_matches_reference_fixture(oracle):
    """The C restatement of grid_mse_table / grid_search against the unmodified reference's
    outputs (tests/golden/grid_search.npz, calibrate.hpp:195-234)."""
    z = np.load(GOLD / "grid_search.npz")
    for bits in (1, 2, 4):
        mse, best = oracle.grid_mse_table(z[f"b{bits}_q"], z[f"b{bits}_keys"], z[f"b{bits}_codes"],
                                          z[f"b{bits}_alpha"], z[f"b{bits}_beta"], bits, 8, z["tau1"], z["tau2"])
        np.testing.assert_allclose(mse, z[f"b{bits}_mse"], rtol=1e-6)
        assert best == tuple(z[f"b{bits}_best"].tolist())


REPORT_CASES = [("t41", 1, 0, (1.0, 0.0), 12), ("t43", 8, 0, (0.0, 0.0), 40), ("t47", 2, 0, (0.0, 0.0), 40),
                ("g2", 2, 1, (2.0, 1.0), 40), ("b1", 1, 0, (3.0, 0.0), 7), ("one", 4, 0, (1.0, 2.0), 1),
                ("wide", 1, 0, (1.0, 0.0), 5000)]


@pytest.mark.parametrize("name,bits,mode,tau,bins", REPORT_CASES)
def test_mse_report_oracle_matches_reference_fixture(oracle, name, bits, mode, tau, bins):
    """The C restatement of mse_report (calibrate.hpp:300-351) against the unmodified
    reference (tests/golden/mse_report.npz): edges and histograms bit-identical, MSEs equal."""
    z = np.load(GOLD / "mse_report.npz")
    r = oracle.mse_report(z[f"{name}_q"], z[f"{name}_keys"], bits, mode, 8, tau, bins)
    assert np.array_equal(r["edges"], z[f"{name}_edges"])
    assert np.array_equal(r["counts"], z[f"{name}_counts"])
    np.testing.assert_allclose(r["mse_quant"], z[f"{name}_mse_quant"], rtol=1e-12)
    np.testing.assert_allclose(r["mse_quant_c"], z[f"{name}_mse_quant_c"], rtol=1e-12)
    # the reference's own invariants (test_calibrate.cpp:272-305)
    assert np.all(z[f"{name}_counts"].sum(axis=2) == z[f"{name}_keys"].shape[1])
    np.testing.assert_allclose(z[f"{name}_means"], [z[f"{name}_mse_quant"].mean(), z[f"{name}_mse_quant_c"].mean()],
                               rtol=1e-12)


def test_report_csv_writers(tmp_path):
    """write_mse_csv / write_histogram_csv (calibrate.hpp:369-397): host formatting of a
    report, the line layout of the reference's tests (test_calibrate.cpp:307-352)."""
    from paper_2502_14882_b200 import kvq
    rep = kvq.MseReport(rows=[kvq.MseRow(0, 0.125, 1e-7), kvq.MseRow(1, 2.0 / 3.0, 0.0)],
                        histograms=[kvq.HeadHistogram(h, np.array([-1.0, 0.5, 2.0], np.float32),
                                                      np.array([[1, 2], [3, 0], [0, 3]], np.uint64)) for h in (0, 1)])
    kvq.write_mse_csv(tmp_path / "mse.csv", rep)
    lines = (tmp_path / "mse.csv").read_text().splitlines()
    assert lines == ["variant,head,mse", "exact,0,0", "exact,1,0", "quant,0,0.125", "quant,1,0.666666667",
                     "quant_c,0,1e-07", "quant_c,1,0"]
    kvq.write_histogram_csv(tmp_path / "hist.csv", rep)
    lines = (tmp_path / "hist.csv").read_text().splitlines()
    assert len(lines) == 1 + 2 * 3 * 2
    assert lines[0] == "variant,head,bin_left,bin_right,count"
    assert lines[1:4] == ["exact,0,-1,0.5,1", "exact,0,0.5,2,2", "quant,0,-1,0.5,3"]
    with pytest.raises(kvq.FormatError):
        kvq.write_mse_csv(tmp_path / "missing" / "x.csv", rep)


def test_reference_dequant_then_dot_arm_matches_post_scaled(ref):
    """The bench's "without post-scaling" CPU arm (dequantize + naive_qk / naive_wv around the
    calibrated softmax, BASELINE config 3) computes the same attention as the reference's
    post-scaled decode_step, up to fp32 reassociation."""
    rng = np.random.default_rng(33)
    R, H, G, n, d = 2, 2, 2, 300, 32
    k = rng.normal(size=(R, H, n, d)).astype(np.float32)
    v = rng.normal(size=(R, H, n, d)).astype(np.float32)
    q = rng.normal(size=(R, H, G, d)).astype(np.float32)
    kn = rng.normal(size=(R, H, d)).astype(np.float32)
    for bits, wb in ((1, 8), (2, 32), (4, 32)):
        _, post = ref.bench_decode(k, v, R, H, G, n, d, bits, wb, 1.0, 0.0, q, kn, kn, 2, 2, prefill_tail=3)
        _, deq = ref.bench_decode(k, v, R, H, G, n, d, bits, wb, 1.0, 0.0, q, kn, kn, 2, 2, prefill_tail=3,
                                  dequant=True)
        assert np.linalg.norm(post - deq) / np.linalg.norm(post) < 1e-5, bits

"""Opt-in token-wise V (KVQ_MODE_V_TOKEN_WISE; north_star "token-wise min/max for V").

PARITY UNPINNED against the reference (which quantizes V channel-wise, kvcache.hpp:60-61):
the checker is oracle/tokenwise.py, the reference quantizer (quantize.hpp:64-146) restated
with the reduction axis swapped.

  * K1: V codes and per-token (alpha, beta) bit-exact with the restatement; K unchanged
    (channel-wise, bit-exact with the reference restatement oracle/kvq_oracle.c);
  * K2: the IMMA decode with the per-token V steps folded into the probabilities
    (out_c = sum_j p_j alpha_j + sum_j (p_j s_j) code_jc) against float64 math on the cache's
    own codes and stats, at the launch geometries the decode plans (split clusters,
    balanced 4-warp launch, 8-warp solo CTAs, head-group split), with fp32 tail rows and
    through the fused step;
  * what the mode does not support raises config_error instead of computing wrong numbers.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# The IMMA weights are e_j s_j (the token's V step folded in) as 16-bit integers per 128-token
# group and head, and the alpha term rides on the same integer weights (v_jc = s_j (code_jc +
# alpha_j / s_j)), so numerator terms stay consistent: the channel-wise bar (1e-4) holds.
TOL = 1e-4


def _unpack(raw, n, bits):
    b = np.asarray(raw, np.uint8).reshape(n, 16 * bits)
    shifts = 8 - bits * (np.arange(8 // bits) + 1)
    return ((b[..., None] >> shifts) & ((1 << bits) - 1)).reshape(n, 128)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("B,H,G,n,bits", [(2, 2, 4, 256, 1), (1, 2, 6, 1024, 2), (40, 8, 4, 1024, 1),
                                           (20, 8, 4, 2048, 4), (4, 8, 4, 4096, 8)])
def test_token_wise_v_codes_and_decode(kvq, B, H, G, n, bits):
    from oracle import tokenwise as tw
    from oracle.oracle import C_Oracle

    oracle = C_Oracle()
    rng = np.random.default_rng(100 + bits)
    k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    v = (rng.normal(size=(B, H, n, 128)) * rng.uniform(0.2, 3.0, size=(B, H, n, 1))).astype(np.float32)
    v[0, 0, 3] = 0.0  # a flat token (zero range)
    v[0, 0, 5, :2] = (-0.0, 0.0)  # signed-zero ties
    cfg = kvq.QuantizationConfig(bits, kvq.QuantMode.v_token_wise)
    cal = kvq.CalibrationParams(1.0, 0.0)
    cache = kvq.BatchedCache.build(k, v, cfg, cal, group=G)
    kn = rng.normal(size=(B, H, 128)).astype(np.float32)
    vn = rng.normal(size=(B, H, 128)).astype(np.float32)
    cache.append(kn, vn)
    q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
    out, _, _ = cache.decode(q)
    units = sorted({0, (B * H) // 2, B * H - 1})
    worst = 0.0
    for u in units:
        b, h = divmod(u, H)
        ka, kb = oracle.compute_stats(k[b, h])
        kseg = cache.segment(u, 0)
        assert np.array_equal(kseg.stats.alpha.view(np.uint32), ka.view(np.uint32))
        assert np.array_equal(kseg.codes.bytes, oracle.quantize(k[b, h], ka, kb, bits))
        codes, va, vb = tw.quantize_tokenwise(v[b, h], bits)
        ga, gb = cache.value_token_stats(u)
        assert np.array_equal(ga.view(np.uint32), va.view(np.uint32)), "token alpha"
        assert np.array_equal(gb.view(np.uint32), vb.view(np.uint32)), "token beta"
        vseg = cache.segment(u, 1)
        assert np.array_equal(_unpack(vseg.codes.bytes, n, bits), codes), "token-wise V codes"
        kc = _unpack(kseg.codes.bytes, n, bits)
        for g in range(G):
            want = tw.decode_f64(kc, ka, kb, codes, va, vb, q[b, h, g], kn[b, h][None], vn[b, h][None], bits,
                                 (1.0, 0.0))
            worst = max(worst, _rel(out[b, h, g], want))
    assert worst <= TOL, worst


def test_token_wise_v_fused_step_and_device_build(kvq):
    torch = pytest.importorskip("torch")
    B, H, G, n = 64, 8, 4, 1024  # 512 units: the balanced 4-warp launch
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(9)
    k = torch.randn((B, H, n, 128), device=dev, generator=gen)
    v = torch.randn((B, H, n, 128), device=dev, generator=gen)
    cfg = kvq.QuantizationConfig(1, kvq.QuantMode.v_token_wise)
    mk = lambda: kvq.BatchedCache.build_device(k, v, cfg, kvq.CalibrationParams(1.0, 0.0), group=G)
    a, b = mk(), mk()
    for c in (a, b):
        c.reserve_tail(8)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs come from the current stream
    for step in range(3):
        q = torch.randn((B, H, G, 128), device=dev, generator=gen)
        kn = torch.randn((B, H, 128), device=dev, generator=gen)
        o1, o2 = torch.empty_like(q), torch.empty_like(q)
        s.wait_stream(torch.cuda.current_stream())
        a.step_device(q, o1, kn, kn, s.cuda_stream)
        b.decode_device(q, o2, s.cuda_stream)
        b.append_device(kn, kn, s.cuda_stream)
        s.synchronize()
        assert torch.equal(o1, o2), step
    # one unit against float64 math
    from oracle import tokenwise as tw
    u = 333
    bq, hq = divmod(u, H)
    ks, vs = a.segment(u, 0), a.segment(u, 1)
    va, vb = a.value_token_stats(u)
    q = torch.randn((B, H, G, 128), device=dev, generator=gen)
    out = torch.empty_like(q)
    s.wait_stream(torch.cuda.current_stream())
    a.decode_device(q, out, s.cuda_stream)
    s.synchronize()
    kt, vt = a.tail(u, 0), a.tail(u, 1)
    qh = q.cpu().numpy()
    for g in range(G):
        want = tw.decode_f64(_unpack(ks.codes.bytes, n, 1), ks.stats.alpha, ks.stats.beta, _unpack(vs.codes.bytes, n, 1),
                             va, vb, qh[bq, hq, g], kt, vt, 1, (1.0, 0.0))
        assert _rel(out.cpu().numpy()[bq, hq, g], want) <= TOL


def test_token_wise_v_unsupported_uses_raise(kvq):
    rng = np.random.default_rng(1)
    k = rng.normal(size=(1, 2, 64, 128)).astype(np.float32)
    cache = kvq.BatchedCache.build(k, k, kvq.QuantizationConfig(1, kvq.QuantMode.v_token_wise),
                                   kvq.CalibrationParams(1.0, 0.0), group=4)
    q = rng.normal(size=(1, 2, 4, 128)).astype(np.float32)
    cache.set_path(kvq.PATH_GENERIC)
    with pytest.raises(kvq.ConfigError):
        cache.decode(q)
    cache.set_path(kvq.PATH_AUTO)
    with pytest.raises(kvq.ConfigError):
        cache.save_image()
    with pytest.raises(kvq.ConfigError):
        kvq.BatchedCache.build(rng.normal(size=(1, 1, 16, 64)).astype(np.float32),
                               rng.normal(size=(1, 1, 16, 64)).astype(np.float32),
                               kvq.QuantizationConfig(1, kvq.QuantMode.v_token_wise), kvq.CalibrationParams(), group=1)


def test_token_wise_v_long_tail_and_host_step(kvq):
    """Token-wise V through the fp32 tail pass (tail capacity > 64 rows: the decode writes its
    log-sum-exp, the tail pass merges) and through the chunked host-buffer step
    (kvq_cache_step: per-chunk stats offsets), against the same cache decoded directly."""
    from oracle import tokenwise as tw
    B, H, G, n = 32, 8, 4, 512  # 256 units: the host step runs 2 request chunks
    rng = np.random.default_rng(21)
    k = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    v = rng.normal(size=(B, H, n, 128)).astype(np.float32)
    cfg = kvq.QuantizationConfig(1, kvq.QuantMode.v_token_wise)
    a = kvq.BatchedCache.build(k, v, cfg, kvq.CalibrationParams(1.0, 0.0), group=G)
    b = kvq.BatchedCache.build(k, v, cfg, kvq.CalibrationParams(1.0, 0.0), group=G)
    a.reserve_tail(100)  # tail pass path
    for step in range(3):
        q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
        kn = rng.normal(size=(B, H, 128)).astype(np.float32)
        vn = rng.normal(size=(B, H, 128)).astype(np.float32)
        out_a, _, _ = a.decode(q)
        a.append(kn, vn)
        out_b = np.empty_like(q)
        b.step(q, kn, vn, out_b)
        assert np.allclose(out_a, out_b, rtol=0, atol=5e-5 * np.abs(out_a).max()), step
    u = 77
    bq, hq = divmod(u, H)
    ks, vs = a.segment(u, 0), a.segment(u, 1)
    va, vb = a.value_token_stats(u)
    q = rng.normal(size=(B, H, G, 128)).astype(np.float32)
    out, _, _ = a.decode(q)
    for g in range(G):
        want = tw.decode_f64(_unpack(ks.codes.bytes, n, 1), ks.stats.alpha, ks.stats.beta, _unpack(vs.codes.bytes, n, 1),
                             va, vb, q[bq, hq, g], a.tail(u, 0), a.tail(u, 1), 1, (1.0, 0.0))
        assert _rel(out[bq, hq, g], want) <= TOL

"""Oracle (test infrastructure only) for the opt-in token-wise V mode (KVQ_MODE_V_TOKEN_WISE).

PARITY UNPINNED: the reference has no token-wise quantizer (V is channel-wise there,
kvcache.hpp:45-46, 60-61) and no test or golden vector covers it. This
is the reference's own quantizer restated with the reduction axis swapped - the checker the
GPU tests compare the device path with, never part of the product:

  compute_stats   quantize.hpp:64-89   min / max folded in index order with std::min /
                                       std::max semantics (the first of equal values wins),
                                       here over the d channels of each token
  quantize        quantize.hpp:91-127  inv_step = L / (beta - alpha) (0 for a flat token),
                                       code = clamp(round((x - alpha) * inv_step), 0, L),
                                       round half away from zero, separately rounded fp32 ops
  dequantize      quantize.hpp:129-146 alpha + code * (beta - alpha) / L, per token
"""
from __future__ import annotations

import numpy as np


def stats_tokenwise(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Per-row (token) min / max of x [n][d] float32, folded in channel order, first wins."""
    x = np.asarray(x, np.float32)
    lo = x[:, 0].copy()
    hi = x[:, 0].copy()
    for c in range(1, x.shape[1]):
        v = x[:, c]
        lo = np.where(v < lo, v, lo)   # std::min(lo, v): v only if strictly smaller
        hi = np.where(hi < v, v, hi)   # std::max(hi, v): v only if strictly larger
    return lo.astype(np.float32), hi.astype(np.float32)


def quantize_tokenwise(x: np.ndarray, bits: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(codes [n][d] uint8, alpha [n], beta [n]) - quantize.hpp:91-127 with per-token stats."""
    x = np.asarray(x, np.float32)
    L = np.float32((1 << bits) - 1)
    lo, hi = stats_tokenwise(x)
    rng = (hi - lo).astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = np.where(rng > 0, L / np.where(rng > 0, rng, np.float32(1)), np.float32(0)).astype(np.float32)
    t = ((x - lo[:, None]).astype(np.float32) * inv[:, None]).astype(np.float32)
    r = np.floor(t.astype(np.float64) + 0.5)  # roundf for t >= 0 (x >= alpha by construction)
    codes = np.clip(r, 0, float(L)).astype(np.uint8)
    return codes, lo, hi


def dequantize_tokenwise(codes: np.ndarray, alpha: np.ndarray, beta: np.ndarray, bits: int) -> np.ndarray:
    """float64 values alpha_j + code_jc (beta_j - alpha_j) / L (quantize.hpp:129-146, per token)."""
    L = float((1 << bits) - 1)
    a = np.asarray(alpha, np.float64)
    s = np.where(np.asarray(beta, np.float64) > a, (np.asarray(beta, np.float64) - a) / L, 0.0)
    return a[:, None] + np.asarray(codes, np.float64) * s[:, None]


def decode_f64(k_codes, ka, kb, v_codes, va_tok, vb_tok, q, k_tail, v_tail, bits, tau) -> np.ndarray:
    """One decode row in float64 (kvcache.hpp:263-311: post-scaled K scores, calibrated softmax
    over [g(vis) | tail], w.V) with channel-wise K and token-wise V."""
    f = np.float64
    L = float((1 << bits) - 1)
    ka, kb, q = (np.asarray(x, f) for x in (ka, kb, q))
    sk = np.where(kb > ka, (kb - ka) / L, 0.0)
    isd = 1.0 / np.sqrt(f(q.size))
    vis = (np.asarray(k_codes, f) @ (q * sk) + q @ ka) * isd
    tail = (np.asarray(k_tail, f) @ q) * isd
    gamma, delta = vis.min(), vis.max()
    if delta > gamma:
        t = (vis - gamma) / (delta - gamma)
        vis = vis - (tau[0] * (1 - t) + tau[1] * t)
    else:
        vis = vis - tau[0]
    row = np.concatenate([vis, tail])
    p = np.exp(row - row.max())
    p /= p.sum()
    vdeq = dequantize_tokenwise(v_codes, va_tok, vb_tok, bits)
    return p[:vis.size] @ vdeq + p[vis.size:] @ np.asarray(v_tail, f)

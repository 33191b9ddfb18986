"""ctypes bindings for the parity checkers — TEST INFRASTRUCTURE ONLY.

  * ``C``   — the plain-C restatement (oracle/kvq_oracle.c -> _ref/libkvq_oracle.so)
  * ``Ref`` — the unmodified reference headers behind a C shim
              (oracle/ref_shim.cpp -> _ref/libkvq_ref.so)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module. Both classes expose the same method names so a test can run the
same check against either.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
_F = C.POINTER(C.c_float)
_U8 = C.POINTER(C.c_uint8)
_U32 = C.POINTER(C.c_uint32)
_SZ = C.c_size_t
_SZP = C.POINTER(C.c_size_t)
_VP = C.c_void_p


def build() -> None:
    """Compile the checkers (needs only gcc/g++; the reference shim also needs
    /root/reference, so on the GPU box the prebuilt .so is used)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a):
    return a.ctypes.data_as(_F)


def _u8(a):
    return a.ctypes.data_as(_U8)


def _row_bytes(dim: int, bits: int, word_bits: int) -> int:
    g = word_bits // bits
    return (dim + g - 1) // g * g // g * (word_bits // 8)


class C_Oracle:
    """The C restatement (kvq_oracle.h)."""

    name = "oracle"

    def __init__(self, path: Path | None = None):
        path = path or REF_DIR / "libkvq_oracle.so"
        if not path.exists():
            build()
        L = C.CDLL(str(path))
        sigs = {
            "kvqo_pack": (C.c_int, [_U32, _SZ, C.c_int, C.c_int, _U8]),
            "kvqo_unpack": (C.c_int, [_U8, _SZ, C.c_int, C.c_int, _U32]),
            "kvqo_compute_stats": (C.c_int, [_F, _SZ, _SZ, C.c_int, _F, _F]),
            "kvqo_quantize": (C.c_int, [_F, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _U8]),
            "kvqo_dequantize": (None, [_U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqo_qk_scores": (None, [_F, _U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqo_wv_output": (None, [_F, _U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqo_naive_qk": (None, [_F, _F, _SZ, _SZ, _F]),
            "kvqo_naive_wv": (None, [_F, _F, _SZ, _SZ, _F]),
            "kvqo_g_apply": (C.c_float, [C.c_float] * 5),
            "kvqo_softmax_inplace": (None, [_F, _SZ]),
            "kvqo_calibrated_softmax_concat": (None, [_F, _SZ, _F, _SZ, C.c_float, C.c_float, _F, _SZP]),
            "kvqo_decode_head": (None, [_F, _SZ, _SZ, C.c_int, C.c_int, _U8, _F, _F, _U8, _F, _F, _F, _F, _SZ,
                                        C.c_float, C.c_float, _F, _F, _SZP]),
            "kvqo_generate_head": (None, [C.c_uint64, C.c_uint64, _SZ, _SZ, C.c_double, C.c_double, _F, _F, _F]),
            "kvqo_generate_step_head": (None, [C.c_uint64, C.c_uint64, C.c_uint64, _SZ, C.c_double, C.c_double,
                                               _F, _F, _F]),
            "kvqo_oracle_attention": (None, [_F, _F, _F, _SZ, _SZ, _F]),
            "kvqo_grid_mse_table": (None, [_F, _F, _U8, _F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, _F, _F, _SZ,
                                           C.POINTER(C.c_double), _F]),
            "kvqo_mse_report": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                                          _SZ, C.POINTER(C.c_double), C.POINTER(C.c_double), _F,
                                          C.POINTER(C.c_uint64)]),
        }
        for n, (r, a) in sigs.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        self.L = L

    def pack(self, codes, bits, word_bits=8):
        c = np.ascontiguousarray(codes, np.uint32)
        g = word_bits // bits
        out = np.zeros(max((c.size + g - 1) // g * (word_bits // 8), 1), np.uint8)
        st = self.L.kvqo_pack(c.ctypes.data_as(_U32), c.size, bits, word_bits, _u8(out))
        return st, out[:(c.size + g - 1) // g * (word_bits // 8)]

    def unpack(self, data, count, bits, word_bits=8):
        b = np.ascontiguousarray(data, np.uint8)
        out = np.zeros(max(count, 1), np.uint32)
        self.L.kvqo_unpack(_u8(b if b.size else np.zeros(1, np.uint8)), count, bits, word_bits,
                           out.ctypes.data_as(_U32))
        return out[:count]

    def compute_stats(self, m, mode=0):
        m = _f32(m)
        a = np.zeros(m.shape[1], np.float32)
        b = np.zeros(m.shape[1], np.float32)
        st = self.L.kvqo_compute_stats(_fp(m), m.shape[0], m.shape[1], mode, _fp(a), _fp(b))
        assert st == 0
        return a, b

    def quantize(self, m, alpha, beta, bits, word_bits=8):
        m = _f32(m)
        out = np.zeros(max(m.shape[0] * _row_bytes(m.shape[1], bits, word_bits), 1), np.uint8)
        st = self.L.kvqo_quantize(_fp(m), m.shape[0], m.shape[1], _fp(_f32(alpha)), _fp(_f32(beta)), bits,
                                  word_bits, _u8(out))
        assert st == 0
        return out[:m.shape[0] * _row_bytes(m.shape[1], bits, word_bits)]

    def dequantize(self, data, rows, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros((rows, dim), np.float32)
        self.L.kvqo_dequantize(_u8(np.ascontiguousarray(data, np.uint8)), rows, dim, _fp(_f32(alpha)),
                               _fp(_f32(beta)), bits, word_bits, _fp(out))
        return out

    def qk_scores(self, q, data, tokens, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros(max(tokens, 1), np.float32)
        self.L.kvqo_qk_scores(_fp(_f32(q)), _u8(np.ascontiguousarray(data, np.uint8)), tokens, dim,
                              _fp(_f32(alpha)), _fp(_f32(beta)), bits, word_bits, _fp(out))
        return out[:tokens]

    def wv_output(self, w, data, tokens, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros(dim, np.float32)
        self.L.kvqo_wv_output(_fp(_f32(w)), _u8(np.ascontiguousarray(data, np.uint8)), tokens, dim,
                              _fp(_f32(alpha)), _fp(_f32(beta)), bits, word_bits, _fp(out))
        return out

    def g_apply(self, x, gamma, delta, tau1, tau2):
        return self.L.kvqo_g_apply(x, gamma, delta, tau1, tau2)

    def calibrated_softmax_concat(self, vis, tail, tau1, tau2):
        vis, tail = _f32(vis), _f32(tail)
        out = np.zeros(max(vis.size + tail.size, 1), np.float32)
        viol = C.c_size_t(0)
        self.L.kvqo_calibrated_softmax_concat(_fp(vis if vis.size else np.zeros(1, np.float32)), vis.size,
                                              _fp(tail if tail.size else np.zeros(1, np.float32)), tail.size,
                                              tau1, tau2, _fp(out), C.byref(viol))
        return out[:vis.size + tail.size], int(viol.value)

    def decode_head(self, q, n_vis, bits, word_bits, kb, ka, kbeta, vb, va, vbeta, ktail, vtail, tau1, tau2):
        """One head of HybridKVCache::run_decode. Returns (out, weights, violations)."""
        dim = q.size
        ktail = _f32(ktail).reshape(-1, dim) if np.size(ktail) else np.zeros((0, dim), np.float32)
        vtail = _f32(vtail).reshape(-1, dim) if np.size(vtail) else np.zeros((0, dim), np.float32)
        nt = ktail.shape[0]
        out = np.zeros(dim, np.float32)
        w = np.zeros(max(n_vis + nt, 1), np.float32)
        viol = C.c_size_t(0)
        z8 = np.zeros(1, np.uint8)
        zf = np.zeros(max(dim, 1), np.float32)
        self.L.kvqo_decode_head(
            _fp(_f32(q)), dim, n_vis, bits, word_bits,
            _u8(np.ascontiguousarray(kb, np.uint8) if np.size(kb) else z8), _fp(_f32(ka) if np.size(ka) else zf),
            _fp(_f32(kbeta) if np.size(kbeta) else zf),
            _u8(np.ascontiguousarray(vb, np.uint8) if np.size(vb) else z8), _fp(_f32(va) if np.size(va) else zf),
            _fp(_f32(vbeta) if np.size(vbeta) else zf),
            _fp(ktail if nt else zf), _fp(vtail if nt else zf), nt, tau1, tau2, _fp(out), _fp(w), C.byref(viol))
        return out, w[:n_vis + nt], int(viol.value)

    def generate_head(self, seed, head, tokens, dim, mean=0.0, stddev=1.0):
        k = np.zeros((tokens, dim), np.float32)
        v = np.zeros((tokens, dim), np.float32)
        q = np.zeros(dim, np.float32)
        self.L.kvqo_generate_head(seed, head, tokens, dim, mean, stddev, _fp(k), _fp(v), _fp(q))
        return k, v, q

    def generate_step_head(self, seed, head, step, dim, mean=0.0, stddev=1.0):
        q = np.zeros(dim, np.float32)
        k = np.zeros(dim, np.float32)
        v = np.zeros(dim, np.float32)
        self.L.kvqo_generate_step_head(seed, head, step, dim, mean, stddev, _fp(q), _fp(k), _fp(v))
        return q, k, v

    def naive_qk(self, q, k):
        k = _f32(k)
        out = np.zeros(k.shape[0], np.float32)
        self.L.kvqo_naive_qk(_fp(_f32(q)), _fp(k), k.shape[0], k.shape[1], _fp(out))
        return out

    def naive_wv(self, w, v):
        v = _f32(v)
        out = np.zeros(v.shape[1], np.float32)
        self.L.kvqo_naive_wv(_fp(_f32(w)), _fp(v), v.shape[0], v.shape[1], _fp(out))
        return out

    def oracle_attention(self, q, k, v):
        k, v = _f32(k), _f32(v)
        out = np.zeros(k.shape[1], np.float32)
        self.L.kvqo_oracle_attention(_fp(_f32(q)), _fp(k), _fp(v), k.shape[0], k.shape[1], _fp(out))
        return out


    def grid_mse_table(self, queries, keys_exact, codes, alpha, beta, bits, word_bits, tau1, tau2):
        """calibrate.hpp:195-234 -> (mse[cells] float64, best (tau1, tau2))."""
        q, ke = _f32(queries), _f32(keys_exact)
        S, n, d = ke.shape
        cb = np.ascontiguousarray(codes, np.uint8)
        t1, t2 = _f32(tau1), _f32(tau2)
        mse = np.zeros(t1.size, np.float64)
        best = np.zeros(2, np.float32)
        self.L.kvqo_grid_mse_table(_fp(q), _fp(ke), _u8(cb), _fp(_f32(alpha)), _fp(_f32(beta)), S, n, d, bits,
                                   word_bits, _fp(t1), _fp(t2), t1.size, mse.ctypes.data_as(C.POINTER(C.c_double)),
                                   _fp(best))
        return mse, (float(best[0]), float(best[1]))

    def mse_report(self, queries, keys, bits, mode=0, word_bits=8, tau=(0.0, 0.0), bins=40):
        """calibrate.hpp:300-351 -> dict(mse_quant, mse_quant_c [H], edges [H][bins+1],
        counts [H][3][bins], means (quant, quant_c))."""
        q, k = _f32(queries), _f32(keys)
        H, n, d = k.shape
        out = _report_buffers(H, bins)
        st = self.L.kvqo_mse_report(_fp(q), _fp(k), H, n, d, mode, bits, word_bits, tau[0], tau[1], bins,
                                    *_report_ptrs(out))
        if st != 0:
            raise ValueError("compute_stats: empty matrix")
        out["means"] = (float(np.mean(out["mse_quant"])), float(np.mean(out["mse_quant_c"])))
        return out


def _report_buffers(H, bins):
    return {"mse_quant": np.zeros(H, np.float64), "mse_quant_c": np.zeros(H, np.float64),
            "edges": np.zeros((H, bins + 1), np.float32), "counts": np.zeros((H, 3, bins), np.uint64)}


def _report_ptrs(out):
    return (out["mse_quant"].ctypes.data_as(C.POINTER(C.c_double)),
            out["mse_quant_c"].ctypes.data_as(C.POINTER(C.c_double)), _fp(out["edges"]),
            out["counts"].ctypes.data_as(C.POINTER(C.c_uint64)))


class Ref:
    """The unmodified reference behind oracle/ref_shim.cpp."""

    name = "reference"

    def __init__(self, path: Path | None = None):
        path = path or REF_DIR / "libkvq_ref.so"
        if not path.exists():
            build()
        if not path.exists():
            raise FileNotFoundError(f"{path}: reference shim not built (needs /root/reference)")
        L = C.CDLL(str(path))
        sigs = {
            "kvqr_last_error": (C.c_char_p, []),
            "kvqr_pack": (C.c_int, [_U32, _SZ, C.c_int, C.c_int, _U8, _SZP]),
            "kvqr_unpack": (C.c_int, [_U8, _SZ, C.c_int, C.c_int, _U32]),
            "kvqr_compute_stats": (C.c_int, [_F, _SZ, _SZ, C.c_int, _F, _F]),
            "kvqr_quantize": (C.c_int, [_F, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _U8, _SZP]),
            "kvqr_dequantize": (C.c_int, [_U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqr_qk_scores": (C.c_int, [_F, _U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqr_wv_output": (C.c_int, [_F, _U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvqr_calibrated_softmax_concat": (C.c_int, [_F, _SZ, _F, _SZ, C.c_float, C.c_float, _F, _SZP]),
            "kvqr_g_apply": (C.c_float, [C.c_float] * 5),
            "kvqr_generate": (C.c_int, [C.c_uint64, _SZ, _SZ, _SZ, _F, _F, _F]),
            "kvqr_generate_step": (C.c_int, [C.c_uint64, _SZ, _SZ, C.c_uint64, _F, _F, _F]),
            "kvqr_oracle_attention": (None, [_F, _F, _F, _SZ, _SZ, _F]),
            "kvqr_cache_build": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                                           C.POINTER(_VP)]),
            "kvqr_cache_free": (None, [_VP]),
            "kvqr_cache_append": (C.c_int, [_VP, _F, _F]),
            "kvqr_cache_decode": (C.c_int, [_VP, _F, _F, _F, _SZP]),
            "kvqr_cache_segment": (C.c_int, [_VP, _SZ, C.c_int, _U8, _F, _F]),
            "kvqr_cache_memory": (C.c_int, [_VP, _SZP]),
            "kvqr_bench_decode": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_float, C.c_float,
                                            _F, _F, _F, C.c_int, C.c_int, _SZ, C.POINTER(C.c_double), _F]),
            "kvqr_bench_decode_dequant": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_float,
                                                    C.c_float, _F, _F, _F, C.c_int, C.c_int, _SZ,
                                                    C.POINTER(C.c_double), _F]),
            "kvqr_cache_save": (C.c_int, [C.c_void_p, C.c_void_p, _SZ, _SZP]),
            "kvqr_cache_load": (C.c_int, [C.c_void_p, _SZ, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
            "kvqr_grid_mse_table": (C.c_int, [_F, _F, _U8, _F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, _F, _F, _SZ,
                                              C.POINTER(C.c_double), _F]),
            "kvqr_mse_report": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float,
                                          _SZ, C.POINTER(C.c_double), C.POINTER(C.c_double), _F,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
        }
        for n, (r, a) in sigs.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        self.L = L

    def _ok(self, st):
        if st != 0:
            raise RuntimeError(f"reference error {st}: {self.L.kvqr_last_error().decode()}")

    def pack(self, codes, bits, word_bits=8):
        c = np.ascontiguousarray(codes, np.uint32)
        out = np.zeros(c.size * 4 + 8, np.uint8)
        n = C.c_size_t(0)
        st = self.L.kvqr_pack(c.ctypes.data_as(_U32), c.size, bits, word_bits, _u8(out), C.byref(n))
        return st, out[:n.value]

    def unpack(self, data, count, bits, word_bits=8):
        out = np.zeros(max(count, 1), np.uint32)
        b = np.ascontiguousarray(data, np.uint8)
        self._ok(self.L.kvqr_unpack(_u8(b if b.size else np.zeros(1, np.uint8)), count, bits, word_bits,
                                    out.ctypes.data_as(_U32)))
        return out[:count]

    def compute_stats(self, m, mode=0):
        m = _f32(m)
        a = np.zeros(m.shape[1], np.float32)
        b = np.zeros(m.shape[1], np.float32)
        self._ok(self.L.kvqr_compute_stats(_fp(m), m.shape[0], m.shape[1], mode, _fp(a), _fp(b)))
        return a, b

    def quantize(self, m, alpha, beta, bits, word_bits=8):
        m = _f32(m)
        out = np.zeros(m.size * 4 + 64, np.uint8)
        n = C.c_size_t(0)
        self._ok(self.L.kvqr_quantize(_fp(m), m.shape[0], m.shape[1], _fp(_f32(alpha)), _fp(_f32(beta)), bits,
                                      word_bits, _u8(out), C.byref(n)))
        return out[:n.value]

    def dequantize(self, data, rows, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros((rows, dim), np.float32)
        self._ok(self.L.kvqr_dequantize(_u8(np.ascontiguousarray(data, np.uint8)), rows, dim, _fp(_f32(alpha)),
                                        _fp(_f32(beta)), bits, word_bits, _fp(out)))
        return out

    def qk_scores(self, q, data, tokens, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros(max(tokens, 1), np.float32)
        self._ok(self.L.kvqr_qk_scores(_fp(_f32(q)), _u8(np.ascontiguousarray(data, np.uint8)), tokens, dim,
                                       _fp(_f32(alpha)), _fp(_f32(beta)), bits, word_bits, _fp(out)))
        return out[:tokens]

    def wv_output(self, w, data, tokens, dim, alpha, beta, bits, word_bits=8):
        out = np.zeros(dim, np.float32)
        self._ok(self.L.kvqr_wv_output(_fp(_f32(w)), _u8(np.ascontiguousarray(data, np.uint8)), tokens, dim,
                                       _fp(_f32(alpha)), _fp(_f32(beta)), bits, word_bits, _fp(out)))
        return out

    def g_apply(self, x, gamma, delta, tau1, tau2):
        return self.L.kvqr_g_apply(x, gamma, delta, tau1, tau2)

    def calibrated_softmax_concat(self, vis, tail, tau1, tau2):
        vis, tail = _f32(vis), _f32(tail)
        out = np.zeros(max(vis.size + tail.size, 1), np.float32)
        viol = C.c_size_t(0)
        self._ok(self.L.kvqr_calibrated_softmax_concat(_fp(vis if vis.size else np.zeros(1, np.float32)),
                                                       vis.size, _fp(tail if tail.size else np.zeros(1, np.float32)),
                                                       tail.size, tau1, tau2, _fp(out), C.byref(viol)))
        return out[:vis.size + tail.size], int(viol.value)

    def generate(self, seed, heads, tokens, dim):
        k = np.zeros((heads, tokens, dim), np.float32)
        v = np.zeros((heads, tokens, dim), np.float32)
        q = np.zeros((heads, dim), np.float32)
        self._ok(self.L.kvqr_generate(seed, heads, tokens, dim, _fp(k), _fp(v), _fp(q)))
        return k, v, q

    def generate_step(self, seed, heads, dim, step):
        q = np.zeros((heads, dim), np.float32)
        k = np.zeros((heads, dim), np.float32)
        v = np.zeros((heads, dim), np.float32)
        self._ok(self.L.kvqr_generate_step(seed, heads, dim, step, _fp(q), _fp(k), _fp(v)))
        return q, k, v

    def oracle_attention(self, q, k, v):
        k, v = _f32(k), _f32(v)
        out = np.zeros(k.shape[1], np.float32)
        self.L.kvqr_oracle_attention(_fp(_f32(q)), _fp(k), _fp(v), k.shape[0], k.shape[1], _fp(out))
        return out

    # -- HybridKVCache
    def cache_load(self, image: bytes, heads: int, dim: int):
        """HybridKVCache::load -> (RefCache, None) or (None, (status, message, offset))."""
        out = C.c_void_p()
        off = C.c_uint64(0)
        buf = (C.c_uint8 * max(len(image), 1)).from_buffer_copy(image or b"\0")
        st = self.L.kvqr_cache_load(buf, len(image), C.byref(out), C.byref(off))
        if st != 0:
            return None, (st, self.L.kvqr_last_error().decode(), int(off.value))
        return RefCache(self, out.value, heads, dim), None

    def cache_build(self, k, v, bits, word_bits=8, tau1=0.0, tau2=0.0, mode=0):
        """k, v: [heads][n][dim]."""
        k, v = _f32(k), _f32(v)
        h, n, d = k.shape
        out = C.c_void_p()
        kb = k if k.size else np.zeros(1, np.float32)
        vb = v if v.size else np.zeros(1, np.float32)
        self._ok(self.L.kvqr_cache_build(_fp(kb), _fp(vb), h, n, d, bits, mode, word_bits, tau1, tau2,
                                         C.byref(out)))
        return RefCache(self, out.value, h, d)

    def bench_decode(self, k, v, requests, kv_heads, group, n, dim, bits, word_bits, tau1, tau2, q, k_new, v_new,
                     threads, steps, prefill_tail=0, dequant=False):
        """The reference's decode on host threads; dequant=True: the dequantize-then-dot
        ablation (dequantize + naive_qk / naive_wv around the calibrated softmax)."""
        secs = (C.c_double * steps)()
        out = np.zeros_like(_f32(q))
        fn = self.L.kvqr_bench_decode_dequant if dequant else self.L.kvqr_bench_decode
        self._ok(fn(_fp(_f32(k)), _fp(_f32(v)), requests, kv_heads, group, n, dim, bits,
                                          word_bits, tau1, tau2, _fp(_f32(q)), _fp(_f32(k_new)), _fp(_f32(v_new)),
                                          threads, steps, prefill_tail, secs, _fp(out)))
        return list(secs), out


    def grid_mse_table(self, queries, keys_exact, codes, alpha, beta, bits, word_bits, tau1, tau2):
        """calibrate.hpp:195-234 -> (mse[cells] float64, best (tau1, tau2))."""
        q, ke = _f32(queries), _f32(keys_exact)
        S, n, d = ke.shape
        cb = np.ascontiguousarray(codes, np.uint8)
        t1, t2 = _f32(tau1), _f32(tau2)
        mse = np.zeros(t1.size, np.float64)
        best = np.zeros(2, np.float32)
        self._ok(self.L.kvqr_grid_mse_table(_fp(q), _fp(ke), _u8(cb), _fp(_f32(alpha)), _fp(_f32(beta)), S, n, d, bits,
                                   word_bits, _fp(t1), _fp(t2), t1.size, mse.ctypes.data_as(C.POINTER(C.c_double)),
                                   _fp(best)))
        return mse, (float(best[0]), float(best[1]))

    def mse_report(self, queries, keys, bits, mode=0, word_bits=8, tau=(0.0, 0.0), bins=40):
        q, k = _f32(queries), _f32(keys)
        H, n, d = k.shape
        out = _report_buffers(H, bins)
        means = np.zeros(2, np.float64)
        self._ok(self.L.kvqr_mse_report(_fp(q), _fp(k), H, n, d, mode, bits, word_bits, tau[0], tau[1], bins,
                                        *_report_ptrs(out), means.ctypes.data_as(C.POINTER(C.c_double))))
        out["means"] = (float(means[0]), float(means[1]))
        return out


class RefCache:
    def __init__(self, ref: Ref, handle, heads, dim):
        self.ref, self.h, self.heads, self.dim = ref, C.c_void_p(handle), heads, dim
        self.n_total = None

    def __del__(self):
        if self.h:
            self.ref.L.kvqr_cache_free(self.h)
            self.h = None

    def append(self, k_new, v_new):
        self.ref._ok(self.ref.L.kvqr_cache_append(self.h, _fp(_f32(k_new)), _fp(_f32(v_new))))

    def decode(self, q, n_total):
        out = np.zeros((self.heads, self.dim), np.float32)
        w = np.zeros((self.heads, max(n_total, 1)), np.float32)
        viol = C.c_size_t(0)
        self.ref._ok(self.ref.L.kvqr_cache_decode(self.h, _fp(_f32(q)), _fp(out), _fp(w), C.byref(viol)))
        return out, w[:, :n_total], int(viol.value)

    def segment(self, head, which, nbytes):
        b = np.zeros(max(nbytes, 1), np.uint8)
        a = np.zeros(self.dim, np.float32)
        be = np.zeros(self.dim, np.float32)
        self.ref.L.kvqr_cache_segment(self.h, head, which, _u8(b), _fp(a), _fp(be))
        return b[:nbytes], a, be

    def memory(self):
        m = (C.c_size_t * 6)()
        self.ref.L.kvqr_cache_memory(self.h, m)
        return [int(x) for x in m]

    def save(self) -> bytes:
        n = C.c_size_t(0)
        self.ref._ok(self.ref.L.kvqr_cache_save(self.h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        self.ref._ok(self.ref.L.kvqr_cache_save(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

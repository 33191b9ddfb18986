"""Python mirror of the reference `kvq` hot-path API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/kvq/*.hpp, cited per function) so parity tests read like
the reference's own tests. Every numeric result is computed by the CUDA kernels in
libkvq_b200.so (include/kvq_capi.h); there is no CPU fallback - without the library or a
GPU every call raises.

Host arrays are numpy; the `*_device` methods of :class:`BatchedCache` take torch CUDA
tensors (torch is only plumbing for device memory and streams).
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field
from enum import IntEnum
from pathlib import Path
from typing import Sequence

import numpy as np

_LIB_PATH = Path(os.environ.get("KVQ_LIB_PATH") or Path(__file__).resolve().parent / "libkvq_b200.so")
_lib = None

# ---- errors (errors.hpp:11-33) ------------------------------------------------------


class KvqError(RuntimeError):
    """Base of the error classes below."""


class ConfigError(KvqError):
    """kvq::config_error: unsupported bitwidth / word width / kernel config."""


class DomainError(KvqError):
    """kvq::domain_error: shape mismatch, empty input, code out of range."""


class FormatError(KvqError):
    """kvq::format_error: malformed serialized data; `offset` = the byte where parsing failed."""

    def __init__(self, msg: str, offset: int = 0):
        super().__init__(f"{msg} (byte offset {offset})")
        self.message, self.offset = msg, offset


class CudaError(KvqError):
    """Device failure or no usable GPU (the library has no CPU fallback)."""


_ERRS = {1: ConfigError, 2: DomainError, 3: FormatError, 4: CudaError}

_F = C.POINTER(C.c_float)
_F32 = np.dtype(np.float32)
_U8 = C.POINTER(C.c_uint8)
_U32 = C.POINTER(C.c_uint32)
_SZ = C.c_size_t
_SZP = C.POINTER(C.c_size_t)
_VP = C.c_void_p


def lib() -> C.CDLL:
    """Load libkvq_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise CudaError(f"{_LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(str(_LIB_PATH))
        sig = {
            "kvq_last_error": (_SZ, [C.c_char_p, _SZ]),
            "kvq_launch_count": (C.c_ulonglong, []),
            "kvq_device_available": (C.c_int, []),
            "kvq_set_device": (C.c_int, [C.c_int]),
            "kvq_cache_sync_tail": (C.c_int, [_VP]),
            "kvq_packed_bytes": (_SZ, [_SZ, C.c_int, C.c_int]),
            "kvq_pack": (C.c_int, [_U32, _SZ, C.c_int, C.c_int, _U8, _SZ]),
            "kvq_unpack": (C.c_int, [_U8, _SZ, _SZ, C.c_int, C.c_int, _U32]),
            "kvq_segment_bytes": (_SZ, [_SZ, _SZ, C.c_int, C.c_int]),
            "kvq_compute_stats": (C.c_int, [_F, _SZ, _SZ, C.c_int, _F, _F]),
            "kvq_quantize": (C.c_int, [_F, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _U8, _SZ]),
            "kvq_dequantize": (C.c_int, [_U8, _SZ, _SZ, _F, _F, C.c_int, C.c_int, _F]),
            "kvq_quantize_device": (C.c_int, [_VP, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int, _VP, _VP, _VP, _VP]),
            "kvq_qk_scores": (C.c_int, [_F, _U8, _F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, _F]),
            "kvq_naive_qk": (C.c_int, [_F, _F, _SZ, _SZ, _F]),
            "kvq_naive_wv": (C.c_int, [_F, _F, _SZ, _SZ, _F]),
            "kvq_wv_output": (C.c_int, [_F, _U8, _F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, _F]),
            "kvq_calibrated_softmax_concat": (C.c_int, [_F, _SZ, _F, _SZ, _SZ, C.c_float, C.c_float, _F, _SZP]),
            "kvq_grid_mse_table": (C.c_int, [_F, _F, _U8, _F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, _F, _F, _SZ,
                                             C.POINTER(C.c_double), _F]),
            "kvq_mse_report": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float, _SZ,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double), _F, C.POINTER(C.c_uint64)]),
            "kvq_cache_build": (C.c_int, [_F, _F, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int,
                                          C.c_float, C.c_float, C.POINTER(_VP)]),
            "kvq_cache_build_device": (C.c_int, [_VP, _VP, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, C.c_int, C.c_int,
                                                 C.c_float, C.c_float, _VP, C.POINTER(_VP)]),
            "kvq_cache_free": (None, [_VP]),
            "kvq_cache_reserve_tail": (C.c_int, [_VP, _SZ]),
            "kvq_cache_set_path": (C.c_int, [_VP, C.c_int]),
            "kvq_cache_append": (C.c_int, [_VP, _F, _F]),
            "kvq_cache_append_device": (C.c_int, [_VP, _VP, _VP, _VP]),
            "kvq_cache_decode": (C.c_int, [_VP, _F, _F, _F, _SZP]),
            "kvq_cache_decode_device": (C.c_int, [_VP, _VP, _VP, _VP]),
            "kvq_cache_step_device": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
            "kvq_cache_step": (C.c_int, [_VP, _VP, _VP, _VP, _VP]),
            "kvq_cache_info": (C.c_int, [_VP, _SZP]),
            "kvq_cache_calibration": (C.c_int, [_VP, _F]),
            "kvq_cache_memory": (C.c_int, [_VP, _SZP]),
            "kvq_cache_resident_bytes": (C.c_int, [_VP, _SZP]),
            "kvq_cache_read_segment": (C.c_int, [_VP, _SZ, C.c_int, _U8, _F, _F]),
            "kvq_cache_read_tail": (C.c_int, [_VP, _SZ, C.c_int, _F]),
            "kvq_cache_read_value_token_stats": (C.c_int, [_VP, _SZ, _F, _F]),
            "kvq_cache_device_pointers": (C.c_int, [_VP, C.POINTER(_VP)]),
            "kvq_last_error_offset": (C.c_ulonglong, []),
            "kvq_cache_image_bytes": (C.c_int, [_VP, _SZP]),
            "kvq_cache_save_image": (C.c_int, [_VP, _VP, _SZ, C.c_int, _VP]),
            "kvq_cache_load_image": (C.c_int, [_VP, _SZ, _SZ, _SZ, _SZP, C.POINTER(_VP)]),
            "kvq_shard_assign": (C.c_int, [_SZ, _SZ, C.c_int, C.c_int, C.POINTER(C.c_longlong), _SZ, _SZP]),
            "kvq_shard_place": (C.c_int, [_VP, C.c_int, _SZ, _SZ, _SZ, _SZ, _VP, C.c_int, _VP]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        buf = C.create_string_buffer(1024)
        lib().kvq_last_error(buf, 1024)
        msg = buf.value.decode(errors="replace")
        if status == 3:
            raise FormatError(msg, int(lib().kvq_last_error_offset()))
        raise _ERRS.get(status, KvqError)(msg)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_F)


def _u8p(a: np.ndarray):
    return a.ctypes.data_as(_U8)


def launch_count() -> int:
    """Kernels launched by libkvq_b200.so in this process."""
    return int(lib().kvq_launch_count())


def device_available() -> bool:
    return bool(lib().kvq_device_available())


def set_device(device: int) -> None:
    """Bind this thread's CUDA device for the library (one process per GPU)."""
    _check(lib().kvq_set_device(int(device)))


def shard_assign(batch: int, kv_heads: int, world: int, rank: int) -> np.ndarray:
    """Global unit indices (b * H + h) rank `rank` owns (kvq_shard_assign):
    contiguous request slices when batch >= world, else round-robin. Host-only."""
    n = C.c_size_t(0)
    _check(lib().kvq_shard_assign(batch, kv_heads, world, rank, None, 0, C.byref(n)))
    out = np.empty(n.value, np.int64)
    _check(lib().kvq_shard_assign(batch, kv_heads, world, rank, out.ctypes.data_as(C.POINTER(C.c_longlong)),
                                  out.size, C.byref(n)))
    return out


def shard_place(parts_ptr: int, world: int, width: int, batch: int, kv_heads: int, row: int, out,
                stream: int = 0) -> None:
    """kvq_shard_place: scatter the gathered [world][width] device rows into the global
    [batch * kv_heads][row] order. `out` is a float32 numpy array (host) or a device pointer."""
    if isinstance(out, np.ndarray):
        if out.dtype != np.float32 or not out.flags.c_contiguous or out.size < batch * kv_heads * row:
            raise DomainError("shard_place: out must be a contiguous float32 array of batch * kv_heads * row")
        _check(lib().kvq_shard_place(parts_ptr, world, width, batch, kv_heads, row, out.ctypes.data, 0, stream))
    else:
        _check(lib().kvq_shard_place(parts_ptr, world, width, batch, kv_heads, row, int(out), 1, stream))


# ---- bitpack.hpp -----------------------------------------------------------------------


@dataclass
class PackedBuffer:
    """bitpack.hpp:15-40."""

    bytes: np.ndarray  # uint8, LE words of word_bits
    code_bits: int = 0
    word_bits: int = 8
    logical_count: int = 0

    def codes_per_word(self) -> int:
        return self.word_bits // self.code_bits

    def word_count(self) -> int:
        g = self.codes_per_word()
        return (self.logical_count + g - 1) // g

    def byte_size(self) -> int:
        return int(self.bytes.size)

    def word_at(self, i: int) -> int:
        nb = self.word_bits // 8
        return int.from_bytes(bytes(self.bytes[i * nb:(i + 1) * nb]), "little")


def pack(codes, code_bits: int, word_bits: int = 8) -> PackedBuffer:
    """kvq::pack (bitpack.hpp:161-187), on the GPU."""
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    n = lib().kvq_packed_bytes(c.size, code_bits, word_bits)
    out = np.zeros(max(n, 1), dtype=np.uint8)
    _check(lib().kvq_pack(c.ctypes.data_as(_U32), c.size, code_bits, word_bits, _u8p(out), out.size))
    return PackedBuffer(out[:n].copy(), code_bits, word_bits, int(c.size))


def unpack(buf: PackedBuffer) -> np.ndarray:
    """kvq::unpack (bitpack.hpp:189-203), on the GPU."""
    out = np.zeros(max(buf.logical_count, 1), dtype=np.uint32)
    b = np.ascontiguousarray(buf.bytes, dtype=np.uint8)
    if b.size == 0:
        b = np.zeros(1, dtype=np.uint8)
    _check(lib().kvq_unpack(_u8p(b), buf.byte_size(), buf.logical_count, buf.code_bits, buf.word_bits,
                            out.ctypes.data_as(_U32)))
    return out[:buf.logical_count].copy()


# ---- quantize.hpp ----------------------------------------------------------------------


class QuantMode(IntEnum):
    channel_wise = 0
    global_ = 1
    # Opt-in extension (not in the reference): K channel-wise, V token-wise (north_star;
    # KVQ_MODE_V_TOKEN_WISE) - BatchedCache only, d = 128, tensor-core decode.
    v_token_wise = 2


@dataclass
class ChannelStats:
    """quantize.hpp:24-29."""

    alpha: np.ndarray
    beta: np.ndarray

    def dim(self) -> int:
        return int(self.alpha.size)


@dataclass
class QuantizationConfig:
    """quantize.hpp:33-44."""

    bitwidth: int = 8
    mode: QuantMode = QuantMode.channel_wise
    word_bits: int = 8


@dataclass
class QuantizedSegment:
    """quantize.hpp:46-62."""

    codes: PackedBuffer
    stats: ChannelStats
    tokens: int = 0
    dim: int = 0
    bitwidth: int = 0

    def codes_per_row(self) -> int:
        g = self.codes.codes_per_word()
        return (self.dim + g - 1) // g * g

    def words_per_row(self) -> int:
        return self.codes_per_row() // self.codes.codes_per_word()

    def row_bytes(self) -> int:
        return self.words_per_row() * self.codes.word_bits // 8


# ---- file records: KVQP segments (quantize.hpp:148-230), KVQT tensors (tensor_io.hpp) -------
# Host formatting; byte-identical to the reference's writers. Readers raise FormatError with
# the reference's messages and byte offsets (relative to the start of the record + `off`).

def _read(buf: bytes, off: int, n: int, what: str) -> bytes:
    if len(buf) - off < n:
        raise FormatError(f"truncated while reading {what}", off)
    return buf[off:off + n]


def _magic(buf: bytes, off: int, magic: bytes, name: str) -> int:
    if len(buf) - off < 4:
        raise FormatError(f"truncated before {name} magic", off)
    if buf[off:off + 4] != magic:
        raise FormatError(f"bad {name} magic", off)
    return off + 4


def write_segment(seg: QuantizedSegment) -> bytes:
    """write_segment (quantize.hpp:155-168): the KVQP record of `seg`."""
    c = seg.codes
    return (b"KVQP" + struct.pack("<IBBHQ", 1, c.code_bits, c.word_bits, 0, c.logical_count)
            + np.ascontiguousarray(c.bytes, np.uint8).tobytes() + struct.pack("<Q", seg.dim)
            + _f32(seg.stats.alpha).astype("<f4").tobytes() + _f32(seg.stats.beta).astype("<f4").tobytes())


def read_segment(buf: bytes, off: int = 0) -> tuple[QuantizedSegment, int]:
    """read_segment (quantize.hpp:177-222) -> (segment, offset after it)."""
    off = _magic(buf, off, b"KVQP", "packed segment")
    (version,) = struct.unpack("<I", _read(buf, off, 4, "version"))
    off += 4
    if version != 1:
        raise FormatError(f"unsupported segment version {version}", off - 4)
    if len(buf) - off < 4:
        raise FormatError("truncated while reading width header", off)
    n, m = buf[off], buf[off + 1]
    off += 4
    if n < 1 or m < 8 or m > 32 or m % 8:
        raise FormatError("stored widths invalid: word bits must be 8, 16, or 32 and code bits >= 1", off - 4)
    if m % n:
        raise FormatError(f"stored widths invalid: code bits {n} must divide word bits {m}", off - 4)
    (logical,) = struct.unpack("<Q", _read(buf, off, 8, "logical_count"))
    off += 8
    g = m // n
    nbytes = (logical + g - 1) // g * (m // 8)
    if len(buf) - off < nbytes:
        raise FormatError("truncated packed words", off)
    codes = np.frombuffer(buf, np.uint8, nbytes, off).copy()
    off += nbytes
    (dim,) = struct.unpack("<Q", _read(buf, off, 8, "dim"))
    off += 8
    stats = []
    for what in ("alpha", "beta"):
        have = min(dim, (len(buf) - off) // 4)
        if have < dim:
            raise FormatError(f"truncated while reading {what}", off + 4 * have)
        stats.append(np.frombuffer(buf, "<f4", dim, off).astype(np.float32))
        off += 4 * dim
    stride = (dim + g - 1) // g * g
    if (logical != 0) if stride == 0 else (logical % stride != 0):
        raise FormatError("logical_count does not cover whole rows", off)
    seg = QuantizedSegment(PackedBuffer(codes, n, m, logical), ChannelStats(stats[0], stats[1]),
                           0 if stride == 0 else logical // stride, dim, n)
    return seg, off


def write_tensor(m) -> bytes:
    """write_tensor (tensor_io.hpp:66-72): the KVQT record of a [rows][cols] fp32 matrix."""
    a = _f32(m)
    a = a.reshape(a.shape[0], -1) if a.ndim != 2 else a
    return b"KVQT" + struct.pack("<IQQ", 1, a.shape[0], a.shape[1]) + a.astype("<f4").tobytes()


def read_tensor(buf: bytes, off: int = 0) -> tuple[np.ndarray, int]:
    """read_tensor (tensor_io.hpp:84-107) -> (matrix, offset after it)."""
    off = _magic(buf, off, b"KVQT", "tensor")
    (version,) = struct.unpack("<I", _read(buf, off, 4, "version"))
    off += 4
    if version != 1:
        raise FormatError(f"unsupported tensor version {version}", off - 4)
    (rows,) = struct.unpack("<Q", _read(buf, off, 8, "rows"))
    off += 8
    (cols,) = struct.unpack("<Q", _read(buf, off, 8, "cols"))
    off += 8
    count = rows * cols
    if len(buf) - off < 4 * count:
        raise FormatError("truncated while reading tensor data", off + (len(buf) - off) // 4 * 4)
    a = np.frombuffer(buf, "<f4", count, off).astype(np.float32).reshape(rows, cols)
    off += 4 * count
    if not np.all(np.isfinite(a)):
        raise FormatError("tensor contains non-finite values", off)
    return a, off


def compute_stats(m, mode: QuantMode = QuantMode.channel_wise) -> ChannelStats:
    """kvq::compute_stats (quantize.hpp:64-89)."""
    m = _f32(np.atleast_2d(m)) if np.ndim(m) else _f32(m)
    rows, cols = (m.shape if m.ndim == 2 else (0, 0))
    a = np.zeros(max(cols, 1), np.float32)
    b = np.zeros(max(cols, 1), np.float32)
    _check(lib().kvq_compute_stats(_fp(m), rows, cols, int(mode), _fp(a), _fp(b)))
    return ChannelStats(a[:cols].copy(), b[:cols].copy())


def quantize(m, stats: ChannelStats, bitwidth: int, word_bits: int = 8) -> QuantizedSegment:
    """kvq::quantize (quantize.hpp:91-127)."""
    m = _f32(m)
    rows, cols = m.shape
    if stats.alpha.size != cols or stats.beta.size != cols:
        raise DomainError(f"quantize: stats dim {stats.alpha.size} does not match matrix cols {cols}")
    alpha, beta = _f32(stats.alpha), _f32(stats.beta)
    n = lib().kvq_segment_bytes(rows, cols, bitwidth, word_bits)
    out = np.zeros(max(n, 1), np.uint8)
    _check(lib().kvq_quantize(_fp(m), rows, cols, _fp(alpha), _fp(beta), bitwidth, word_bits, _u8p(out), out.size))
    g = word_bits // bitwidth
    cpr = (cols + g - 1) // g * g
    buf = PackedBuffer(out[:n].copy(), bitwidth, word_bits, rows * cpr)
    return QuantizedSegment(buf, ChannelStats(alpha.copy(), beta.copy()), rows, cols, bitwidth)


def dequantize(seg: QuantizedSegment) -> np.ndarray:
    """kvq::dequantize (quantize.hpp:129-146)."""
    out = np.zeros((seg.tokens, seg.dim), np.float32)
    if seg.tokens == 0 or seg.dim == 0:
        return out
    codes = np.ascontiguousarray(seg.codes.bytes)
    _check(lib().kvq_dequantize(_u8p(codes), seg.tokens, seg.dim, _fp(_f32(seg.stats.alpha)),
                                _fp(_f32(seg.stats.beta)), seg.bitwidth, seg.codes.word_bits, _fp(out)))
    return out


# ---- kernels.hpp -----------------------------------------------------------------------


@dataclass
class KernelConfig:
    """kernels.hpp:30-40. Validated like the reference; never changes results."""

    head_block: int = 32
    token_block: int = 64
    workers: int = 1

    def validate(self) -> None:
        if self.head_block < 1 or self.token_block < 1 or self.workers < 1:
            raise ConfigError("kernel blocks and workers must be >= 1")


def naive_qk(q, k) -> np.ndarray:
    """kvq::naive_qk (kernels.hpp:401-413): q K^T over an unquantized matrix, the reference's
    scalar loop (same order, separately rounded)."""
    q, k = _f32(q).reshape(-1), _f32(k)
    if q.size != k.shape[1]:
        raise DomainError("naive_qk: query length does not match key cols")
    out = np.zeros(k.shape[0], np.float32)
    if k.shape[0]:
        _check(lib().kvq_naive_qk(_fp(q), _fp(k), k.shape[0], k.shape[1], _fp(out)))
    return out


def naive_wv(w, v) -> np.ndarray:
    """kvq::naive_wv (kernels.hpp:415-426): w V, accumulated over rows in order."""
    w, v = _f32(w).reshape(-1), _f32(v)
    if w.size != v.shape[0]:
        raise DomainError("naive_wv: weight length does not match value rows")
    out = np.zeros(v.shape[1], np.float32)
    if v.shape[1]:
        _check(lib().kvq_naive_wv(_fp(w), _fp(v), v.shape[0], v.shape[1], _fp(out)))
    return out


def _check_uniform(segs: Sequence[QuantizedSegment], who: str) -> None:
    s0 = segs[0]
    for s in segs[1:]:
        if (s.tokens, s.dim, s.bitwidth, s.codes.word_bits) != (s0.tokens, s0.dim, s0.bitwidth, s0.codes.word_bits):
            raise DomainError(f"{who}: head segments have mismatched shapes")


def _stack_segments(segs: Sequence[QuantizedSegment]):
    codes = np.concatenate([np.ascontiguousarray(s.codes.bytes) for s in segs] + [np.zeros(1, np.uint8)])
    alpha = _f32(np.concatenate([s.stats.alpha for s in segs]))
    beta = _f32(np.concatenate([s.stats.beta for s in segs]))
    return codes, alpha, beta


def qk_scores(q, keys, cfg: KernelConfig | None = None) -> np.ndarray:
    """kvq::qk_scores: single form (kernels.hpp:302-314) when `keys` is a segment,
    batched form (342-363) when it is a sequence of per-head segments."""
    cfg = cfg or KernelConfig()
    cfg.validate()
    single = isinstance(keys, QuantizedSegment)
    segs = [keys] if single else list(keys)
    q = _f32(q)
    q2 = q.reshape(1, -1) if single else q
    if single and q.size != keys.dim:
        raise DomainError(f"qk_scores: query length {q.size} does not match segment dim {keys.dim}")
    if not single:
        if q2.shape[0] != len(segs):
            raise DomainError("qk_scores: query rows != head count")
        if not segs:
            return np.zeros((0, 0), np.float32)
        _check_uniform(segs, "qk_scores")
        if q2.shape[1] != segs[0].dim:
            raise DomainError("qk_scores: query cols do not match segment dim")
    s0 = segs[0]
    out = np.zeros((len(segs), max(s0.tokens, 1)), np.float32)
    codes, alpha, beta = _stack_segments(segs)
    _check(lib().kvq_qk_scores(_fp(q2), _u8p(codes), _fp(alpha), _fp(beta), len(segs), s0.tokens, s0.dim,
                               s0.bitwidth, s0.codes.word_bits, _fp(out)))
    out = out[:, :s0.tokens]
    return out[0].copy() if single else out.copy()


def wv_output(w, values, cfg: KernelConfig | None = None) -> np.ndarray:
    """kvq::wv_output: single (kernels.hpp:316-336) or batched (365-396) form."""
    cfg = cfg or KernelConfig()
    cfg.validate()
    single = isinstance(values, QuantizedSegment)
    segs = [values] if single else list(values)
    w = _f32(w)
    w2 = w.reshape(1, -1) if single else w
    if single and w.size != values.tokens:
        raise DomainError(f"wv_output: weight length {w.size} does not match segment tokens {values.tokens}")
    if not single:
        if w2.shape[0] != len(segs):
            raise DomainError("wv_output: weight rows != head count")
        if not segs:
            return np.zeros((0, 0), np.float32)
        _check_uniform(segs, "wv_output")
        if w2.shape[1] != segs[0].tokens:
            raise DomainError("wv_output: weight cols do not match segment tokens")
    s0 = segs[0]
    out = np.zeros((len(segs), s0.dim), np.float32)
    codes, alpha, beta = _stack_segments(segs)
    wbuf = w2 if w2.size else np.zeros((len(segs), 1), np.float32)
    _check(lib().kvq_wv_output(_fp(wbuf), _u8p(codes), _fp(alpha), _fp(beta), len(segs), s0.tokens, s0.dim,
                               s0.bitwidth, s0.codes.word_bits, _fp(out)))
    return out[0].copy() if single else out


# ---- calibrate.hpp ---------------------------------------------------------------------


@dataclass
class CalibrationParams:
    """calibrate.hpp:26-32."""

    tau1: float = 0.0
    tau2: float = 0.0

    def identity(self) -> bool:
        return self.tau1 == 0.0 and self.tau2 == 0.0


def calibrated_softmax_concat(vis, tail, p: CalibrationParams, with_violations: bool = False):
    """kvq::calibrated_softmax_concat (calibrate.hpp:100-114) on the GPU. Accepts one
    row (1-D) or a batch of rows (2-D). Returns the probability row(s), plus the slope
    violation count when with_violations."""
    vis, tail = _f32(vis), _f32(tail)
    single = vis.ndim == 1 and tail.ndim == 1
    v2 = vis.reshape(1, -1) if vis.ndim == 1 else vis
    t2 = tail.reshape(1, -1) if tail.ndim == 1 else tail
    rows = max(v2.shape[0], t2.shape[0])
    if v2.shape[1] == 0:
        v2 = np.zeros((rows, 0), np.float32)
    if t2.shape[1] == 0:
        t2 = np.zeros((rows, 0), np.float32)
    n = v2.shape[1] + t2.shape[1]
    out = np.zeros((rows, max(n, 1)), np.float32)
    viol = C.c_size_t(0)
    vb = v2 if v2.size else np.zeros(1, np.float32)
    tb = t2 if t2.size else np.zeros(1, np.float32)
    _check(lib().kvq_calibrated_softmax_concat(_fp(vb), v2.shape[1], _fp(tb), t2.shape[1], rows, p.tau1, p.tau2,
                                               _fp(out), C.byref(viol)))
    out = out[:, :n]
    res = out[0].copy() if single else out
    return (res, int(viol.value)) if with_violations else res


def g_apply(x: float, gamma: float, delta: float, p: CalibrationParams) -> float:
    """calibrate.hpp:62-67 — scalar form of g for API parity (fp32 arithmetic)."""
    f = np.float32
    x, gamma, delta = f(x), f(gamma), f(delta)
    width = f(delta - gamma)
    if width <= 0:
        return float(f(x - f(p.tau1)))
    t = f(f(x - gamma) / width)
    return float(f(x - f(f(f(p.tau1) * f(f(1) - t)) + f(f(p.tau2) * t))))


@dataclass
class CalibrationSample:
    """calibrate.hpp:127-131: one query, its exact keys and the same keys quantized."""

    query: np.ndarray              # [d]
    keys_exact: np.ndarray         # [n][d] fp32
    keys_quant: QuantizedSegment   # same tokens, packed


@dataclass
class GridCell:
    """calibrate.hpp:148-151."""

    params: CalibrationParams
    mse: float = 0.0


def make_grid(values) -> list[CalibrationParams]:
    """calibrate.hpp:133-142: the sorted cartesian square of `values`."""
    vals = sorted(float(v) for v in values)
    if not vals:
        raise DomainError("make_grid: empty value list")
    return [CalibrationParams(t1, t2) for t1 in vals for t2 in vals]


def default_grid() -> list[CalibrationParams]:
    """calibrate.hpp:144-146: {0, 1, 2, 3}^2."""
    return make_grid([0.0, 1.0, 2.0, 3.0])


def _grid_call(samples: Sequence[CalibrationSample], cells: Sequence[CalibrationParams]):
    if not samples:
        raise DomainError("grid_mse_table: empty calibration set")
    if not cells:
        raise DomainError("grid_mse_table: empty grid")
    s0 = samples[0]
    n, d = s0.keys_exact.shape
    bits, wb = s0.keys_quant.bitwidth, s0.keys_quant.codes.word_bits
    for i, s in enumerate(samples):
        if (np.asarray(s.query).size != d or s.keys_exact.shape != (n, d) or s.keys_quant.dim != d
                or s.keys_quant.tokens != n or s.keys_quant.bitwidth != bits or s.keys_quant.codes.word_bits != wb):
            raise DomainError(f"calibration sample {i} has inconsistent shapes")
    q = np.stack([_f32(s.query) for s in samples])
    ke = np.stack([_f32(s.keys_exact) for s in samples])
    codes = np.stack([np.ascontiguousarray(s.keys_quant.codes.bytes, np.uint8) for s in samples])
    alpha = np.stack([_f32(s.keys_quant.stats.alpha) for s in samples])
    beta = np.stack([_f32(s.keys_quant.stats.beta) for s in samples])
    t1 = _f32([c.tau1 for c in cells])
    t2 = _f32([c.tau2 for c in cells])
    mse = np.zeros(len(cells), np.float64)
    best = np.zeros(2, np.float32)
    _check(lib().kvq_grid_mse_table(_fp(q), _fp(ke), codes.ctypes.data_as(_U8), _fp(alpha), _fp(beta), len(samples),
                                    n, d, bits, wb, _fp(t1), _fp(t2), len(cells),
                                    mse.ctypes.data_as(C.POINTER(C.c_double)), _fp(best)))
    return mse, CalibrationParams(float(best[0]), float(best[1]))


def grid_mse_table(samples: Sequence[CalibrationSample], cells: Sequence[CalibrationParams]) -> list[GridCell]:
    """kvq::grid_mse_table (calibrate.hpp:195-210) on the GPU: mean softmax MSE per cell."""
    mse, _ = _grid_call(samples, cells)
    return [GridCell(c, float(m)) for c, m in zip(cells, mse)]


def grid_search(samples: Sequence[CalibrationSample], cells: Sequence[CalibrationParams] | None = None
                ) -> CalibrationParams:
    """kvq::grid_search (calibrate.hpp:213-234): argmin, ties to the smaller tau1, then tau2."""
    _, best = _grid_call(samples, default_grid() if cells is None else cells)
    return best


# ---- diagnostics: mse_report (calibrate.hpp:236-397) -----------------------------------

class ScoreVariant(IntEnum):
    """calibrate.hpp:241."""

    exact = 0
    quant = 1
    quant_c = 2


def variant_name(v: ScoreVariant) -> str:
    return ("exact", "quant", "quant_c")[int(v)]


@dataclass
class HeadWorkload:
    """workload.hpp:68-72 (values are carried but unused by mse_report)."""

    keys: np.ndarray    # [tokens][d]
    values: np.ndarray  # [tokens][d]
    query: np.ndarray   # [1][d] or [d]


@dataclass
class MseRow:
    """calibrate.hpp:251-255."""

    head: int = 0
    mse_quant: float = 0.0
    mse_quant_c: float = 0.0


@dataclass
class HeadHistogram:
    """calibrate.hpp:257-261: bins + 1 shared edges, counts per ScoreVariant."""

    head: int = 0
    edges: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    counts: np.ndarray = field(default_factory=lambda: np.zeros((3, 0), np.uint64))


@dataclass
class MseReport:
    """calibrate.hpp:263-268."""

    rows: list = field(default_factory=list)
    histograms: list = field(default_factory=list)
    mean_mse_quant: float = 0.0
    mean_mse_quant_c: float = 0.0


def _report_call(keys: np.ndarray, queries: np.ndarray, cfg: QuantizationConfig, p: CalibrationParams, bins: int):
    H, n, d = keys.shape
    mq, mc = np.zeros(H, np.float64), np.zeros(H, np.float64)
    edges = np.zeros((H, bins + 1), np.float32)
    counts = np.zeros((H, 3, bins), np.uint64)
    _check(lib().kvq_mse_report(_fp(queries), _fp(keys), H, n, d, cfg.bitwidth, int(cfg.mode), cfg.word_bits,
                                p.tau1, p.tau2, bins, mq.ctypes.data_as(C.POINTER(C.c_double)),
                                mc.ctypes.data_as(C.POINTER(C.c_double)), _fp(edges),
                                counts.ctypes.data_as(C.POINTER(C.c_uint64))))
    return mq, mc, edges, counts


def mse_report(heads: Sequence[HeadWorkload], qcfg: QuantizationConfig, p: CalibrationParams, bins: int = 40,
               kcfg: KernelConfig | None = None) -> MseReport:
    """kvq::mse_report (calibrate.hpp:300-351) on the GPU: per head, quantize the keys with
    their own stats, then compare the exact, quantized and calibrated pre-softmax rows
    (softmax MSE vs exact; shared-edge histograms). Heads of equal shape go in one call."""
    if not heads:
        raise DomainError("mse_report: no heads")
    if bins < 1:
        raise ConfigError("mse_report: bins must be >= 1")
    if kcfg is not None:
        kcfg.validate()
    keys = [_f32(h.keys) for h in heads]
    queries = [_f32(h.query).reshape(-1) for h in heads]
    for k, q in zip(keys, queries):
        if k.ndim != 2 or q.size != k.shape[1]:
            raise DomainError("naive_qk: query length does not match key cols")
    report = MseReport()
    i = 0
    while i < len(heads):  # runs of equal-shape heads share one device call
        j = i + 1
        while j < len(heads) and keys[j].shape == keys[i].shape:
            j += 1
        mq, mc, edges, counts = _report_call(np.stack(keys[i:j]), np.stack(queries[i:j]), qcfg, p, bins)
        for h in range(j - i):
            report.rows.append(MseRow(i + h, float(mq[h]), float(mc[h])))
            report.histograms.append(HeadHistogram(i + h, edges[h], counts[h]))
        i = j
    for r in report.rows:  # in head order, as the reference accumulates
        report.mean_mse_quant += r.mse_quant
        report.mean_mse_quant_c += r.mse_quant_c
    report.mean_mse_quant /= len(heads)
    report.mean_mse_quant_c /= len(heads)
    return report


def _fmt_real(v: float) -> str:
    return "%.9g" % v  # calibrate.hpp:355-359


def write_mse_csv(path, report: MseReport) -> None:
    """calibrate.hpp:369-381; columns variant,head,mse."""
    try:
        with open(path, "w") as f:
            f.write("variant,head,mse\n")
            for r in report.rows:
                f.write(f"exact,{r.head},0\n")
            for r in report.rows:
                f.write(f"quant,{r.head},{_fmt_real(r.mse_quant)}\n")
            for r in report.rows:
                f.write(f"quant_c,{r.head},{_fmt_real(r.mse_quant_c)}\n")
    except OSError as e:
        raise FormatError(f"cannot open for writing: {path}") from e


def write_histogram_csv(path, report: MseReport) -> None:
    """calibrate.hpp:383-397; columns variant,head,bin_left,bin_right,count."""
    try:
        with open(path, "w") as f:
            f.write("variant,head,bin_left,bin_right,count\n")
            for h in report.histograms:
                for v in range(3):
                    for b in range(len(h.edges) - 1):
                        f.write(f"{variant_name(ScoreVariant(v))},{h.head},{_fmt_real(float(h.edges[b]))},"
                                f"{_fmt_real(float(h.edges[b + 1]))},{int(h.counts[v][b])}\n")
    except OSError as e:
        raise FormatError(f"cannot open for writing: {path}") from e


# ---- kvcache.hpp -----------------------------------------------------------------------

FULL_PRECISION_BITS = 16


@dataclass
class CacheMemory:
    """kvcache.hpp:28-35."""

    code_bytes: int = 0
    stats_bytes: int = 0
    quantized_bytes: int = 0
    tail_bytes: int = 0
    fp32_vis_bytes: int = 0
    total_bytes: int = 0


@dataclass
class DecodeDetail:
    """kvcache.hpp:37-41."""

    outputs: np.ndarray
    weights: np.ndarray
    slope_violations: int = 0


PATH_AUTO, PATH_GENERIC, PATH_TC, PATH_UMMA, PATH_DEQUANT = 0, 1, 2, 3, 4


class BatchedCache:
    """A device-resident batch of hybrid caches: `batch` sequences x `kv_heads` KV heads,
    each KV head serving `group` query heads (GQA). batch = group = 1 is exactly one
    reference HybridKVCache (kvcache.hpp:43-319)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = (C.c_size_t * 10)()
        _check(lib().kvq_cache_info(self._h, info))
        (self.batch, self.kv_heads, self.group, self.dim, self._n_vis, _, self.bitwidth, self.word_bits,
         self.mode, _) = [int(x) for x in info]
        tau = (C.c_float * 2)()
        lib().kvq_cache_calibration(self._h, tau)
        self.calibration = CalibrationParams(float(tau[0]), float(tau[1]))

    # -- construction
    @classmethod
    def build(cls, k_vis, v_vis, cfg: QuantizationConfig, cal: CalibrationParams, group: int = 1) -> "BatchedCache":
        """k_vis/v_vis: [batch][kv_heads][n][dim] fp32 host arrays."""
        k, v = _f32(k_vis), _f32(v_vis)
        if k.shape != v.shape or k.ndim != 4:
            raise DomainError("cache build: need matching [batch][kv_heads][n][dim] key/value arrays")
        b, h, n, d = k.shape
        kb = k if k.size else np.zeros(1, np.float32)
        vb = v if v.size else np.zeros(1, np.float32)
        out = C.c_void_p()
        _check(lib().kvq_cache_build(_fp(kb), _fp(vb), b, h, group, n, d, int(cfg.bitwidth), int(cfg.mode),
                                     int(cfg.word_bits), cal.tau1, cal.tau2, C.byref(out)))
        return cls(out.value)

    @classmethod
    def build_device(cls, k_vis, v_vis, cfg: QuantizationConfig, cal: CalibrationParams, group: int = 1,
                     stream: int = 0) -> "BatchedCache":
        """Same, from torch CUDA tensors [batch][kv_heads][n][dim] (no host round trip)."""
        b, h, n, d = k_vis.shape
        out = C.c_void_p()
        _check(lib().kvq_cache_build_device(k_vis.data_ptr(), v_vis.data_ptr(), b, h, group, n, d,
                                            int(cfg.bitwidth), int(cfg.mode), int(cfg.word_bits), cal.tau1,
                                            cal.tau2, stream, C.byref(out)))
        return cls(out.value)

    # -- snapshots: the reference's KVQC bytes (kvcache.hpp:137-218), every unit a "head"
    def image_bytes(self) -> int:
        n = C.c_size_t(0)
        _check(lib().kvq_cache_image_bytes(self._h, C.byref(n)))
        return n.value

    def save_image(self) -> bytes:
        """The cache as one KVQC image (host bytes)."""
        n = self.image_bytes()
        buf = (C.c_uint8 * n)()
        _check(lib().kvq_cache_save_image(self._h, C.cast(buf, _VP), n, 0, None))
        return bytes(buf)

    def save_image_device(self, out, stream: int = 0) -> None:
        """The image into a torch CUDA uint8 tensor of image_bytes() (checkpoint or migrate
        a cache without a host round trip)."""
        _check(lib().kvq_cache_save_image(self._h, out.data_ptr(), out.numel(), 1, stream or None))

    @classmethod
    def load_image(cls, image: bytes, batch: int = 1, group: int = 1) -> tuple["BatchedCache", int]:
        """Parse a KVQC image (heads = batch x kv_heads units); returns (cache, bytes used)."""
        data = bytes(image)
        buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
        used = C.c_size_t(0)
        out = C.c_void_p()
        _check(lib().kvq_cache_load_image(C.cast(buf, _VP), len(data), batch, group, C.byref(used), C.byref(out)))
        return cls(out.value), used.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.kvq_cache_free(h)
            self._h = None

    # -- accessors
    def _info(self):
        info = (C.c_size_t * 10)()
        _check(lib().kvq_cache_info(self._h, info))
        return [int(x) for x in info]

    @property
    def units(self) -> int:
        return self.batch * self.kv_heads

    def vis_tokens(self) -> int:
        return self._info()[4]

    def tail_tokens(self) -> int:
        return self._info()[5]

    def total_tokens(self) -> int:
        return self.vis_tokens() + self.tail_tokens()

    def set_path(self, path: int) -> None:
        _check(lib().kvq_cache_set_path(self._h, path))

    def reserve_tail(self, rows: int) -> None:
        _check(lib().kvq_cache_reserve_tail(self._h, rows))

    def memory(self) -> CacheMemory:
        m = (C.c_size_t * 6)()
        _check(lib().kvq_cache_memory(self._h, m))
        return CacheMemory(*[int(x) for x in m])

    def resident_bytes(self) -> dict:
        """Device bytes held for the codes: K rows, V rows (0 when V lives only in the
        decode's operand layout), the V operand layout, derived layouts built on demand."""
        m = (C.c_size_t * 4)()
        _check(lib().kvq_cache_resident_bytes(self._h, m))
        return dict(zip(("k_rows", "v_rows", "v_operand", "derived"), (int(x) for x in m)))

    def segment(self, unit: int, which: int) -> QuantizedSegment:
        """Packed codes and per-channel stats of one unit's K (0) or V (1) segment. A token-wise
        V cache's V segment carries no per-channel stats (zeros here; value_token_stats)."""
        n, d = self.vis_tokens(), self.dim
        bits = self.bitwidth if self.bitwidth != FULL_PRECISION_BITS else 8
        nbytes = lib().kvq_segment_bytes(n, d, bits, self.word_bits)
        raw = np.zeros(max(nbytes, 1), np.uint8)
        a = np.zeros(d, np.float32)
        b = np.zeros(d, np.float32)
        tokwise_v = which == 1 and self._info()[8] == int(QuantMode.v_token_wise)
        _check(lib().kvq_cache_read_segment(self._h, unit, which, _u8p(raw), None if tokwise_v else _fp(a),
                                            None if tokwise_v else _fp(b)))
        g = self.word_bits // bits
        cpr = (d + g - 1) // g * g
        return QuantizedSegment(PackedBuffer(raw[:nbytes].copy(), bits, self.word_bits, n * cpr),
                                ChannelStats(a, b), n, d, bits)

    def tail(self, unit: int, which: int) -> np.ndarray:
        out = np.zeros((max(self.tail_tokens(), 1), self.dim), np.float32)
        _check(lib().kvq_cache_read_tail(self._h, unit, which, _fp(out)))
        return out[:self.tail_tokens()].copy()

    def value_token_stats(self, unit: int) -> tuple[np.ndarray, np.ndarray]:
        """Token-wise V caches: the V (alpha, beta) of every visual token of one unit."""
        n = self._info()[4]
        a, b = np.zeros(max(n, 1), np.float32), np.zeros(max(n, 1), np.float32)
        _check(lib().kvq_cache_read_value_token_stats(self._h, unit, _fp(a), _fp(b)))
        return a[:n], b[:n]

    def device_pointers(self) -> list[int]:
        p = (C.c_void_p * 9)()
        _check(lib().kvq_cache_device_pointers(self._h, p))
        return [int(x or 0) for x in p]

    # -- hot path (host buffers)
    def append(self, k_new, v_new) -> None:
        """[batch][kv_heads][dim] each (kvcache.hpp:99-109)."""
        k, v = _f32(k_new), _f32(v_new)
        if k.size != self.units * self.dim or v.size != self.units * self.dim:
            raise DomainError(f"append: expected {self.units} x {self.dim} new key/value rows")
        _check(lib().kvq_cache_append(self._h, _fp(k), _fp(v)))

    def decode(self, queries, weights: bool = False, violations: bool = False):
        """queries [batch][kv_heads][group][dim] -> out, same shape (kvcache.hpp:111-121)."""
        q = _f32(queries)
        if q.size != self.units * self.group * self.dim:
            raise DomainError(f"decode_step: expected {self.units * self.group} x {self.dim} queries")
        out = np.zeros((self.batch, self.kv_heads, self.group, self.dim), np.float32)
        w = None
        if weights:
            w = np.zeros((self.batch, self.kv_heads, self.group, max(self.total_tokens(), 1)), np.float32)
        viol = C.c_size_t(0)
        _check(lib().kvq_cache_decode(self._h, _fp(q), _fp(out), _fp(w) if w is not None else None,
                                      C.byref(viol) if violations else None))
        if w is not None:
            w = w[..., :self.total_tokens()]
        return out, w, int(viol.value)

    def step(self, queries, k_new, v_new, out: np.ndarray) -> None:
        """decode then append through host buffers, one synchronization (kvq_cache_step).
        The buffers are used in place (and a CUDA graph of the step is cached per buffer
        set), so they must be C-contiguous float32 of exactly the step's sizes."""
        nq, nkv = self.units * self.group * self.dim, self.units * self.dim
        arrs = (queries, k_new, v_new, out)
        for name, arr, n in zip(("queries", "k_new", "v_new", "out"), arrs, (nq, nkv, nkv, nq)):
            if not (isinstance(arr, np.ndarray) and arr.dtype == _F32 and arr.flags.c_contiguous):
                raise DomainError(f"step: {name} must be a C-contiguous float32 numpy array")
            if arr.size != n:
                raise DomainError(f"step: {name} has {arr.size} elements, expected {n}")
        # a serving loop passes the same buffers every step: their addresses are looked up once
        # (numpy's ctypes bridge costs ~2-5 us per array - a fifth of a C2 host-buffer step)
        cached = getattr(self, "_step_bufs", None)
        if cached is not None and all(x is y for x, y in zip(arrs, cached[0])):
            ptrs = cached[1]
        else:
            ptrs = tuple(a.ctypes.data for a in arrs)
            self._step_bufs = (arrs, ptrs)
        _check(lib().kvq_cache_step(self._h, *ptrs))

    def sync_tail(self) -> None:
        """Reconcile the host tail counter with the device (after graph replays)."""
        _check(lib().kvq_cache_sync_tail(self._h))

    # -- hot path (device tensors)
    def decode_device(self, q, out, stream: int = 0) -> None:
        _check(lib().kvq_cache_decode_device(self._h, q.data_ptr(), out.data_ptr(), stream))

    def append_device(self, k_new, v_new, stream: int = 0) -> None:
        _check(lib().kvq_cache_append_device(self._h, k_new.data_ptr(), v_new.data_ptr(), stream))

    def step_device(self, q, out, k_new, v_new, stream: int = 0) -> None:
        """decode_device(q, out) then append_device(k_new, v_new), fused into one kernel when
        the tensor-core decode owns the fp32 tail (graph-capturable, same results)."""
        _check(lib().kvq_cache_step_device(self._h, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                                           out.data_ptr(), stream))


class HybridKVCache:
    """Drop-in for kvq::HybridKVCache (kvcache.hpp:43-319): one sequence, `heads` heads,
    one query row per head, device-resident state."""

    def __init__(self, cache: BatchedCache):
        self._c = cache

    @staticmethod
    def _stack(mats):
        mats = [_f32(m) for m in mats]
        if not mats or len(mats) == 0:
            raise DomainError("cache build: need matching per-head key/value lists")
        return mats

    @classmethod
    def build(cls, k_vis: Sequence, v_vis: Sequence, cfg: QuantizationConfig,
              cal: CalibrationParams) -> "HybridKVCache":
        """kvcache.hpp:48-66."""
        if cfg.bitwidth not in (1, 2, 4, 8):
            raise ConfigError("bitwidth must be 1, 2, 4, or 8")
        return cls._build(k_vis, v_vis, cfg, cal)

    @classmethod
    def build_full_precision(cls, k: Sequence, v: Sequence) -> "HybridKVCache":
        """kvcache.hpp:69-83."""
        return cls._build(k, v, QuantizationConfig(FULL_PRECISION_BITS, QuantMode.channel_wise, 8),
                          CalibrationParams())

    @classmethod
    def _build(cls, k_vis, v_vis, cfg, cal):
        if len(k_vis) == 0 or len(k_vis) != len(v_vis):
            raise DomainError("cache build: need matching per-head key/value lists")
        ks = [_f32(m).reshape(_f32(m).shape if _f32(m).ndim == 2 else (0, 0)) for m in k_vis]
        vs = [_f32(m) for m in v_vis]
        r0, c0 = ks[0].shape
        for h, (kk, vv) in enumerate(zip(ks, vs)):
            if kk.shape != (r0, c0) or vv.shape != (r0, c0):
                raise DomainError(f"cache build: head {h} shape differs from head 0")
        if c0 == 0:
            raise DomainError("cache build: head dim must be positive")
        k = np.stack(ks)[None]
        v = np.stack(vs)[None]
        return cls(BatchedCache.build(k, v, cfg, cal, group=1))

    def heads(self) -> int:
        return self._c.kv_heads

    def dim(self) -> int:
        return self._c.dim

    def bitwidth(self) -> int:
        return self._c.bitwidth

    def calibration(self) -> CalibrationParams:
        return self._c.calibration

    def vis_tokens(self) -> int:
        return self._c.vis_tokens()

    def tail_tokens(self) -> int:
        return self._c.tail_tokens()

    def total_tokens(self) -> int:
        return self._c.total_tokens()

    def key_segment(self, h: int) -> QuantizedSegment:
        return self._c.segment(h, 0)

    def value_segment(self, h: int) -> QuantizedSegment:
        return self._c.segment(h, 1)

    def key_tail(self, h: int) -> np.ndarray:
        return self._c.tail(h, 0)

    def value_tail(self, h: int) -> np.ndarray:
        return self._c.tail(h, 1)

    def append(self, k_new, v_new) -> None:
        k, v = _f32(k_new), _f32(v_new)
        if k.shape != (self.heads(), self.dim()) or v.shape != (self.heads(), self.dim()):
            raise DomainError(f"append: expected {self.heads()} x {self.dim()} new key/value rows")
        self._c.append(k, v)

    def _check_q(self, queries):
        q = _f32(queries)
        if q.shape != (self.heads(), self.dim()):
            raise DomainError(f"decode_step: expected {self.heads()} x {self.dim()} queries")
        return q

    def decode_step(self, queries, cfg: KernelConfig | None = None) -> np.ndarray:
        (cfg or KernelConfig()).validate()
        out, _, _ = self._c.decode(self._check_q(queries))
        return out.reshape(self.heads(), self.dim())

    def decode_step_detailed(self, queries, cfg: KernelConfig | None = None) -> DecodeDetail:
        (cfg or KernelConfig()).validate()
        out, w, viol = self._c.decode(self._check_q(queries), weights=True, violations=True)
        return DecodeDetail(out.reshape(self.heads(), self.dim()), w.reshape(self.heads(), -1), viol)

    def memory(self) -> CacheMemory:
        return self._c.memory()

    def save(self, path) -> None:
        """HybridKVCache::save (kvcache.hpp:137-161): the reference's KVQC bytes."""
        data = self._c.save_image()
        try:
            with open(path, "wb") as f:
                f.write(data)
        except OSError as e:
            raise FormatError(f"cannot open for writing: {path}") from e

    @classmethod
    def load(cls, path) -> "HybridKVCache":
        """HybridKVCache::load (kvcache.hpp:163-218); trailing bytes are a format error."""
        try:
            with open(path, "rb") as f:
                data = f.read()
        except OSError as e:
            raise FormatError(f"cannot open for reading: {path}") from e
        c, used = BatchedCache.load_image(data)
        if used != len(data):
            raise FormatError("trailing bytes after cache data", used)
        return cls(c)

    @classmethod
    def from_bytes(cls, image: bytes) -> tuple["HybridKVCache", int]:
        c, used = BatchedCache.load_image(image)
        return cls(c), used

    def to_bytes(self) -> bytes:
        return self._c.save_image()

    @property
    def batched(self) -> BatchedCache:
        return self._c

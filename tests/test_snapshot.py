"""Cache snapshots: the reference's KVQC / KVQP / KVQT byte format
(kvcache.hpp:137-218, quantize.hpp:148-230, tensor_io.hpp:11-128), pinned on images and
load errors produced by the unmodified reference (tests/golden/cache_io.npz,
make_golden.py cache_io)."""
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"
CASES = ["q4", "fp", "d128", "m16", "empty"]
META = {  # name: (bits, word_bits, tau)
    "q4": (4, 8, (2.0, 1.0)), "fp": (16, 8, (0.0, 0.0)), "d128": (1, 8, (1.0, 0.0)),
    "m16": (2, 16, (0.0, 0.0)), "empty": (2, 8, (1.0, 0.0)),
}


def _mutated(z, i):
    base = bytearray(z["q4_image"].tobytes())
    at, val = int(z["mut_at"][i]), int(z["mut_val"][i])
    if at == -1:
        return bytes(base[:val])
    if at == -2:  # NaN in head 0's K tail (after two 188-byte segments and a 24-byte header)
        seg = 20 + 96 + 8 + 64
        base[52 + 2 * seg + 24: 52 + 2 * seg + 28] = np.array([np.nan], np.float32).tobytes()
        return bytes(base)
    base[at] = val
    return bytes(base)


def test_load_rejects_malformed_images_like_the_reference(kvq_host):
    """Every corruption the reference rejects is a FormatError with its message and byte
    offset (test_kvcache.cpp:353-395); validation runs on the host before any device work."""
    z = np.load(GOLD / "cache_io.npz")
    for i, label in enumerate(z["mut_labels"]):
        with pytest.raises(kvq_host.FormatError) as e:
            kvq_host.BatchedCache.load_image(_mutated(z, i))
        assert str(e.value) == str(z["mut_msg"][i]), label  # message incl. " (byte offset N)"
        assert e.value.offset == int(z["mut_off"][i]), label


def _build(kvq, z, name):
    bits, wb, tau = META[name]
    k, v = z[f"{name}_k"], z[f"{name}_v"]
    if bits == 16:
        c = kvq.HybridKVCache.build_full_precision(list(k), list(v))
    else:
        c = kvq.HybridKVCache.build(list(k), list(v), kvq.QuantizationConfig(bits, kvq.QuantMode.channel_wise, wb),
                                    kvq.CalibrationParams(*tau))
    for t in range(z[f"{name}_kn"].shape[0]):
        c.append(z[f"{name}_kn"][t], z[f"{name}_vn"][t])
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_save_is_byte_identical_to_the_reference(kvq, name):
    """A device cache built and appended like the reference's saves to the same bytes."""
    z = np.load(GOLD / "cache_io.npz")
    c = _build(kvq, z, name)
    assert c.to_bytes() == z[f"{name}_image"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_load_reference_image_decodes_like_the_reference(kvq, name, tmp_path):
    """load(reference image) -> the reference's segments, tails and decode output; the
    file round trip and re-save are byte-identical (test_kvcache.cpp:307-351)."""
    z = np.load(GOLD / "cache_io.npz")
    img = z[f"{name}_image"].tobytes()
    c, used = kvq.HybridKVCache.from_bytes(img)
    assert used == len(img)
    assert c.to_bytes() == img
    bits, wb, tau = META[name]
    h = z[f"{name}_k"].shape[0]
    assert c.heads() == h and c.bitwidth() == bits
    assert (c.calibration().tau1, c.calibration().tau2) == (tau if bits != 16 else (0.0, 0.0))
    assert c.tail_tokens() == z[f"{name}_kn"].shape[0] + (z[f"{name}_k"].shape[1] if bits == 16 else 0)
    out = c.decode_step(z[f"{name}_q"])
    want = z[f"{name}_out"]
    err = np.linalg.norm(out - want) / max(np.linalg.norm(want), 1e-30)
    assert err <= 1e-4, err
    p = tmp_path / "cache.kvqc"
    c.save(p)
    assert p.read_bytes() == img
    assert kvq.HybridKVCache.load(p).to_bytes() == img
    p.write_bytes(img + b"x")
    with pytest.raises(kvq.FormatError) as e:
        kvq.HybridKVCache.load(p)
    assert e.value.offset == len(img)


@pytest.mark.gpu
def test_device_image_and_batched_load(kvq):
    """The image gathered in device memory equals the host image; a 3-head image loads as
    3 requests x 1 KV head or 1 x 3 (any batch dividing the heads), not as 2 x ..."""
    import torch
    z = np.load(GOLD / "cache_io.npz")
    img = z["d128_image"].tobytes()
    c, _ = kvq.BatchedCache.load_image(img, batch=3, group=1)
    assert (c.batch, c.kv_heads) == (3, 1)
    dev = torch.empty(c.image_bytes(), dtype=torch.uint8, device="cuda")
    c.save_image_device(dev)
    torch.cuda.synchronize()
    assert dev.cpu().numpy().tobytes() == img
    g, _ = kvq.BatchedCache.load_image(img, batch=1, group=2)
    assert (g.batch, g.kv_heads, g.group) == (1, 3, 2)
    with pytest.raises(kvq.DomainError):
        kvq.BatchedCache.load_image(img, batch=2)


def test_segment_and_tensor_records_roundtrip_reference_bytes(kvq_host):
    """The KVQP / KVQT records inside a reference KVQC image read back and re-serialize to
    the same bytes (quantize.hpp:148-230, tensor_io.hpp:66-107); short reads raise the
    reference's messages."""
    k = kvq_host
    for name in CASES:
        img = np.load(GOLD / "cache_io.npz")[f"{name}_image"].tobytes()
        off = 52
        heads = int.from_bytes(img[8:16], "little")
        for _ in range(heads):
            for _ in range(2):
                seg, end = k.read_segment(img, off)
                assert k.write_segment(seg) == img[off:end]
                off = end
            for _ in range(2):
                t, end = k.read_tensor(img, off)
                assert k.write_tensor(t) == img[off:end]
                off = end
        assert off == len(img)
    img = np.load(GOLD / "cache_io.npz")["q4_image"].tobytes()
    with pytest.raises(k.FormatError) as e:
        k.read_segment(img[:52 + 20 + 96 + 8 + 10], 52)
    assert e.value.message == "truncated while reading alpha" and e.value.offset == 184
    with pytest.raises(k.FormatError) as e:
        k.read_segment(img[:100], 52)
    assert e.value.message == "truncated packed words" and e.value.offset == 72

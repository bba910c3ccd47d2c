"""FIC1 container on the device (proj/src/format.cpp:105-185): records packed
/ unpacked by csrc/fic1.cu, byte-exact against the reference's own FIC1 bytes (golden vectors
from the compiled reference and, where oracle/_ref is built, ref serialize on random
encodings), round trips, the device-to-device entry and the error cases."""
import os

import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200.abi import MAPPING_DTYPE
from paper_1404_0774_b200.fic1 import deserialize, record_layout, serialize, serialize_device

pytestmark = pytest.mark.gpu


def _random_encoding(rng, side=64, height=None):
    height = side if height is None else height
    n = int(rng.choice([2, 4, 8]))
    step = int(rng.integers(1, 2 * n + 1))
    p = fic.CodecParams(n=n, step=step, s_bits=int(rng.integers(1, 17)), o_bits=int(rng.integers(1, 17)),
                        s_max=float(rng.uniform(0.1, 2.0)))
    px, py, _, _ = record_layout(side, height, p)
    count = (side // n) * (height // n)
    m = np.zeros(count, MAPPING_DTYPE)
    m["x"] = rng.integers(0, px, count) * step
    m["y"] = rng.integers(0, py, count) * step
    m["sym"] = rng.integers(0, 8, count)
    m["qs"] = rng.integers(0, 1 << p.s_bits, count)
    m["qo"] = rng.integers(0, 1 << p.o_bits, count)
    return fic.EncodedImage(side, height, p, m)


def test_fic1_golden_bytes(golden):
    # the reference's FIC1 bytes of its own encodes (tests/golden/make_golden.py)
    variants = [dict(), dict(step=2, s_max=0.75), dict(o_bits=6, s_bits=4)]
    for i, pv in enumerate(variants):
        enc = fic.EncodedImage(32, 32, fic.CodecParams(**pv), golden[f"noise32_v{i}_maps"])
        assert serialize(enc) == golden[f"noise32_v{i}_fic1"].tobytes()
        back = deserialize(golden[f"noise32_v{i}_fic1"].tobytes())
        assert back == enc


def test_fic1_round_trip_random():
    rng = np.random.default_rng(7)
    have_ref = os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "oracle", "_ref", "libfic_ref.so"))
    ref = None
    if have_ref:
        from oracle import Reference
        ref = Reference()
    for k in range(60):
        enc = _random_encoding(rng, height=[64, 32, 128][k % 3] if k % 4 == 0 else None)
        blob = serialize(enc)
        assert blob[:4] == b"FIC1"
        back = deserialize(blob)
        assert back == enc
        assert serialize(back) == blob
        if ref is not None and enc.width == enc.height:
            p = enc.params
            want = ref.serialize(enc.mappings, enc.width, dict(n=p.n, step=p.step, s_bits=p.s_bits, o_bits=p.o_bits,
                                                               s_max=p.s_max))
            assert blob == want


def test_fic1_device_entry():
    import torch
    rng = np.random.default_rng(11)
    enc = _random_encoding(rng, side=512)
    blob = serialize(enc)
    d_maps = torch.from_numpy(enc.mappings.view(np.uint8).copy()).cuda()
    size = serialize_device(d_maps.data_ptr(), enc.width, enc.height, enc.params)
    assert size == len(blob)
    d_out = torch.zeros(size, dtype=torch.uint8, device="cuda")
    serialize_device(d_maps.data_ptr(), enc.width, enc.height, enc.params, d_out.data_ptr(), size,
                     torch.cuda.current_stream().cuda_stream)
    assert d_out.cpu().numpy().tobytes() == blob


def test_fic1_errors():
    enc = _random_encoding(np.random.default_rng(1))
    blob = serialize(enc)
    with pytest.raises(fic.CodecError, match="TruncatedData"):
        deserialize(blob[:10])
    with pytest.raises(fic.CodecError, match="MalformedHeader"):
        deserialize(b"XXXX" + blob[4:])
    with pytest.raises(fic.CodecError, match="TruncatedData"):
        deserialize(blob[:-1])
    bad = fic.EncodedImage(enc.width, enc.height, enc.params, enc.mappings.copy())
    bad.mappings["x"][3] += 1
    if enc.params.step > 1:
        with pytest.raises(fic.CodecError, match="OutOfRange: domain position off the step grid"):
            serialize(bad)
    with pytest.raises(fic.CodecError, match="BadParams"):
        serialize(fic.EncodedImage(enc.width, enc.height, enc.params, enc.mappings[:-1].copy()))
    # a record whose x index lies outside the grid (format.cpp:174-177)
    p = fic.CodecParams(n=4, step=3)
    px, py, widths, nb = record_layout(32, 32, p)
    assert px < (1 << widths[0])
    m = np.zeros(64, MAPPING_DTYPE)
    blob = bytearray(serialize(fic.EncodedImage(32, 32, p, m)))
    blob[20 + 5 * nb] = 0xFF  # record 5: x index all ones
    with pytest.raises(fic.CodecError, match="domain index outside the grid in record 5"):
        deserialize(bytes(blob))

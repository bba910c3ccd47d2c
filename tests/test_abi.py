"""CPU: the C-ABI library loads, exports exactly what include/fic_b200.h declares, and its
host-side entry points (no device work) follow the reference's validation semantics."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "fic_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fic_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), f"libfic_b200.so does not export {name}"
    assert sorted(_lib.EXPORTS) == declared


def test_library_is_sm100a():
    # the in-tree library carries sm_100a SASS with tcgen05 / bulk-copy instructions
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "UTCHMMA" in out and "LDTM" in out and "UBLKCP" in out


def test_struct_layouts():
    assert ctypes.sizeof(abi.FicMapping) == 32
    assert ctypes.sizeof(abi.FicParams) == 32
    assert ctypes.sizeof(abi.FicStats) == 24
    assert abi.MAPPING_DTYPE.itemsize == 32


def test_errc_names_match_reference_enum():
    L = _lib.lib()
    for code, name in enumerate(abi.ERRC_NAMES, start=1):
        assert L.fic_errc_name(code).decode() == name
    assert L.fic_errc_name(0).decode() == "Ok"


def test_params_normalisation():
    # params.cpp:9-23: step 0 tracks n, s_max snapped to milli precision, invariants raise BadParams
    p = fic.CodecParams(n=8)
    assert p.step == 8 and p.s_max == 1.0 and p.s_bits == 5 and p.o_bits == 7
    assert fic.CodecParams(s_max=0.12345).s_max == 0.123
    assert repr(fic.CodecParams()) == "CodecParams(n=4, step=4, s_bits=5, o_bits=7, s_max=1.000000)"
    for bad in [dict(n=3), dict(n=1), dict(step=-1), dict(s_bits=0), dict(s_bits=17), dict(o_bits=0),
                dict(s_max=0.0), dict(s_max=70.0), dict(s_max=0.0004), dict(shadow_eps=-1.0)]:
        with pytest.raises(fic.CodecError, match="BadParams"):
            fic.CodecParams(**bad)


def test_geometry_validation():
    # image.cpp:138-149, surfaced like the reference bindings (test_smoke.py:66-71)
    with pytest.raises(fic.CodecError, match="NotSquare"):
        fic.validate_geometry(np.zeros((16, 32), np.uint8))
    with pytest.raises(fic.CodecError, match="NotPowerOfTwo"):
        fic.validate_geometry(np.zeros((96, 96), np.uint8))
    with pytest.raises(fic.CodecError, match="TooSmallForDomain"):
        fic.validate_geometry(np.zeros((8, 8), np.uint8), fic.CodecParams(n=8))
    with pytest.raises(fic.CodecError, match="IndivisibleByRange"):
        fic.validate_geometry(np.zeros((4, 4), np.uint8), fic.CodecParams(n=8))
    fic.validate_geometry(np.zeros((64, 64), np.uint8))


def test_encode_validation_precedes_device_work():
    # validation errors are reported before any CUDA call, so they surface on CPU too
    with pytest.raises(fic.CodecError, match="NotSquare"):
        fic.encode(np.zeros((16, 32), np.uint8))
    with pytest.raises(fic.CodecError, match="BadParams"):
        fic.encode(np.zeros((16, 16), np.uint8), workers=2, chunk=(0, 1))
    with pytest.raises(fic.CodecError, match="GeometryError"):
        fic.encode_range(np.zeros((16, 16), np.uint8), 3, 0)
    with pytest.raises(fic.CodecError, match="BadParams"):
        fic.encode_rows(np.zeros((16, 16), np.uint8), 2, 9)


def test_decoded_error_bound():
    assert fic.decoded_error_bound(2.0, 0.5) == 4.0
    with pytest.raises(fic.CodecError, match="NonContractive"):
        fic.decoded_error_bound(1.0, 1.0)


def test_no_silent_cpu_fallback_without_a_gpu():
    # with no usable device the compute entry points fail loudly (FIC_ERR_CUDA)
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(fic.CodecError, match="CudaError"):
        fic.encode(np.zeros((16, 16), np.uint8))


def test_missing_extension_raises(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_lib.ExtensionMissing):
        _lib.lib()

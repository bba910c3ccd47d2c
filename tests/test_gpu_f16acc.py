"""The fp16-accumulator pruning bound (scan_threshold, f16acc) rests on how tcgen05.mma kind::f16
rounds into an fp16 D on this hardware: to nearest even, once per K=16 step, with the
.pack::16b load layout the epilogue assumes.  tools/f16acc_probe.cu measures exactly that;
this test builds and runs it on the box and holds it to the bound's assumptions, so a device
or driver that behaved differently fails here instead of silently mis-pruning."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_f16_accumulator_matches_bound_assumptions(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "f16acc_probe")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "f16acc_probe.cu")], check=True, capture_output=True, timeout=600)
    out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=120).stdout
    assert "status no error" in out, out
    m = re.search(r"register j == columns \(2j, 2j\+1\): (\d+) of (\d+)", out)
    assert m and m.group(1) == m.group(2), out  # the epilogue's packed-register layout
    K = 64
    e32 = float(re.search(r"fp32 D: max \|D - exact\| / sum\|ab\| = ([0-9.e+-]+)", out).group(1))
    assert e32 <= K * 2.0 ** -21, out  # scan_threshold: K * 2^-21 |u||b| for fp32 accumulation
    e16 = float(re.search(r"fp16 D, one element per column: max err / sum\|ab\| = ([0-9.e+-]+)", out).group(1))
    # fp16 accumulation: (K/16) roundings of at most 2^-11 |u||b| each (the bound adds the first
    # K/16 - 1 this way and the last one relative to the result, which is smaller)
    assert e16 <= (K // 16) * 2.0 ** -11 * 1.05 + K * 2.0 ** -21, out
    # 16 products inside one step: summed, then rounded once (each within the bound)
    m = re.search(r"many-term step: exact-then-round (\d+), per-product rounding \d+, within the bound (\d+) of (\d+)", out)
    assert m and m.group(2) == m.group(3), out
    for k2 in (1, 16):  # round to nearest even, inside a K=16 step and across steps
        m = re.search(rf"rounding probe \(second term at k={k2}\): matches RNE (\d+), RZ \d+, neither (\d+) of (\d+)",
                      out)
        assert m and m.group(1) == m.group(3) and m.group(2) == "0", out

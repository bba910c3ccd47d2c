"""Host-API encode overheads (GPU analysis tool): the Python wrapper, the bare C-ABI call, with
pageable or pinned host buffers, and the device-resident encode, each averaged over warm calls
(no L2 flush).  Usage: python tools/e2e_probe.py [cfg]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402
from paper_1404_0774_b200._lib import lib  # noqa: E402
from paper_1404_0774_b200.abi import MAPPING_DTYPE, FicStats, ptr  # noqa: E402


def tm(f, n=300):
    for _ in range(30):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
gen, n, step = images.CONFIGS[cfg]
img = np.ascontiguousarray(gen())
h, w = img.shape
p = fic.CodecParams(n=n, step=step)
R = (w // n) * (h // n)
L = lib()
pin_img = torch.empty(img.shape, dtype=torch.uint8, pin_memory=True).numpy()
pin_img[:] = img
out = np.zeros(R, MAPPING_DTYPE)
pin_out = torch.empty(R * MAPPING_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(MAPPING_DTYPE)
st = FicStats()
d_img = torch.from_numpy(img).cuda()
d_out = torch.empty(R * MAPPING_DTYPE.itemsize, dtype=torch.uint8, device="cuda")


def c_call(src, dst):
    return lambda: L.fic_encode(ptr(src), w, h, ctypes.byref(p.struct), ptr(dst), ctypes.byref(st))


res = {
    "python fic.encode (pageable in)": tm(lambda: fic.encode(img, p)),
    "python fic.encode (pinned in)": tm(lambda: fic.encode(pin_img, p)),
    "C-ABI fic_encode pageable in / pageable out": tm(c_call(img, out)),
    "C-ABI fic_encode pinned in / pageable out": tm(c_call(pin_img, out)),
    "C-ABI fic_encode pinned in / pinned out": tm(c_call(pin_img, pin_out)),
    "device encode (fic_encode_device, synchronised)": tm(
        lambda: fic.encode_device(d_img.data_ptr(), w, h, d_out.data_ptr(), p)),
}
assert (pin_out.view(np.uint8) == out.view(np.uint8)).all()
for k, v in res.items():
    print(f"{k:50s} {v:8.1f} us")

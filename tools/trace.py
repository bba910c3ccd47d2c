"""Per-tile pipeline timeline of scan CTA 0 (FIC_DEBUG=32, read with fic_debug_trace): how long
the MMA issuer waited for a TMEM buffer / a pool tile, the tile period, and how long the
epilogue warps took per tile.  GPU analysis tool; needs a trace build of the library:
    FIC_TRACE=1 FIC_LIB=$PWD/paper_1404_0774_b200/libfic_trace.so python -m paper_1404_0774_b200.build
    FIC_LIB=$PWD/paper_1404_0774_b200/libfic_trace.so python tools/trace.py cfg2 [extra FIC_DEBUG bits]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402
from paper_1404_0774_b200._lib import lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
gen, n, step = images.CONFIGS[cfg]
img = gen()
fic.encode(img, fic.CodecParams(n=n, step=step))
os.environ["FIC_DEBUG"] = str(32 | (int(sys.argv[2]) if len(sys.argv) > 2 else 0))
os.environ["FIC_NO_GRAPH"] = "1"
os.environ["FIC_PREPASS"] = "0"  # the full level only: its trace is what stays in the buffer
fic.encode(img, fic.CodecParams(n=n, step=step))
T, S = 256, 51
buf = np.zeros(T * S, np.int64)
assert lib().fic_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), T * S) == 0
t = buf.reshape(T, S)
valid = t[:, 2] > 0
t = t[valid]
print(f"{cfg}: {len(t)} tiles traced (CTA 0)")
period = np.diff(t[:, 2])
wait_buf = t[:, 1] - t[:, 0]
wait_tile = t[:, 2] - t[:, 1]
rel = t[:, 3:19]
done = t[:-1, 19:35]
proc = done - rel[:-1]
spread = rel.max(1) - rel.min(1)
print(f"tile period (MMA start to start): median {np.median(period):.0f} cycles, p90 {np.quantile(period, .9):.0f}")
print(f"MMA wait for a TMEM buffer: median {np.median(wait_buf):.0f}, for the pool tile: median {np.median(wait_tile):.0f}")
print(f"epilogue: release spread across warps median {np.median(spread):.0f}; per-warp processing median "
      f"{np.median(proc):.0f}, p90 {np.quantile(proc, .9):.0f}, slowest warp per tile median {np.median(proc.max(1)):.0f}")
test = t[:, 35:51] - rel
print(f"epilogue release -> past the per-range test: median {np.median(test):.0f}, p90 {np.quantile(test, .9):.0f}")
print(f"MMA start -> first release median {np.median(rel.min(1) - t[:, 2]):.0f}, -> last release "
      f"{np.median(rel.max(1) - t[:, 2]):.0f}")

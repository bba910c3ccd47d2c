"""Real (non-serialised, warm) per-kernel device times and inter-kernel gaps of one encode,
from CUPTI via torch.profiler (captures the library's kernels too).  GPU analysis tool."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
gen, n, step = images.CONFIGS[cfg]
img = gen()
p = fic.CodecParams(n=n, step=step)
torch.cuda.init()
for _ in range(3):
    fic.encode(img, p)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        fic.encode(img, p)
path = "/tmp/kineto.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
# last encode: from the last pool kernel on
starts = [i for i, e in enumerate(ev) if "pool_v3" in e["name"]]
seg = ev[starts[-1]:]
t0 = seg[0]["ts"]
busy = 0.0
prev_end = None
rows = []
for e in seg:
    gap = e["ts"] - prev_end if prev_end is not None else 0.0
    rows.append((e["ts"] - t0, e["dur"], gap, e["name"][:60]))
    busy += e["dur"]
    prev_end = e["ts"] + e["dur"]
for r in rows:
    print(f"{r[0]:9.1f} {r[1]:8.1f} gap {r[2]:6.1f}  {r[3]}")
span = prev_end - t0
print(f"span {span:.1f} us, busy {busy:.1f} us, gaps {span - busy:.1f} us")

"""Host-side breakdown of one host-API encode (fic.encode): CUDA runtime API calls and device
activity from CUPTI (torch.profiler), to see where the end-to-end time beyond the device encode
goes.  GPU analysis tool."""
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
for _ in range(5):
    fic.encode(img, p)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        fic.encode(img, p)
path = "/tmp/kineto_e2e.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
rt = [e for e in ev if e.get("cat") in ("cuda_runtime", "cuda_driver") and "dur" in e]
dev = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
rt.sort(key=lambda e: e["ts"])
dev.sort(key=lambda e: e["ts"])
# the last encode: from the last graph launch
gl = [i for i, e in enumerate(rt) if "GraphLaunch" in e["name"]]
t0 = rt[gl[-1] - 3]["ts"] if gl else rt[0]["ts"]
print("host API calls (last encode), us from first:")
for e in rt:
    if e["ts"] >= t0:
        print(f"  {e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['name']}")
print("device activity:")
for e in dev:
    if e["ts"] >= t0:
        print(f"  {e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['name'][:70]}")

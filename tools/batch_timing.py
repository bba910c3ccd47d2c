"""Volume (cfg5) encode throughput: stacked batch passes vs one encode per slice.
   python tools/batch_timing.py [slices] [chunk]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import paper_1404_0774_b200 as fic
from paper_1404_0774_b200 import images
from paper_1404_0774_b200.abi import MAPPING_DTYPE

count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
vol = images.volume(count=count, side=512)
p = fic.CodecParams(n=8, step=4)
per = (512 // 8) ** 2
d_img = torch.from_numpy(vol).cuda()
d_out = torch.zeros(count * per * MAPPING_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
d_ref = torch.zeros_like(d_out)


def batched():
    fic.encode_batch_device(d_img.data_ptr(), count, 512, 512, d_out.data_ptr(), p)


def looped():
    for i in range(count):
        fic.encode_device(d_img[i].data_ptr(), 512, 512, d_ref.data_ptr() + i * per * MAPPING_DTYPE.itemsize, p)
    torch.cuda.synchronize()


for name, f in [("per-slice", looped), ("batched", batched)]:
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 3
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    print(f"{name:10s} chunk={os.environ.get('FIC_BATCH_CHUNK', '64')}: {dt * 1e3:8.2f} ms for {count} slices "
          f"= {count / dt:8.1f} slices/s")
same = torch.equal(d_out, d_ref)
print("batched == per-slice:", same)
sys.exit(0 if same else 1)

"""Prints the matcher's pruning counters (FIC_DEBUG=4) and wall time per config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

os.environ["FIC_DEBUG"] = "4"
for cfg in (sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]):
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    t = time.time()
    enc = fic.encode(img, fic.CodecParams(n=n, step=step))
    print(cfg, f"{time.time() - t:.3f}s", flush=True)

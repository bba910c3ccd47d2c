"""Encode one configured synthetic image once (used under ncu by tools/profile.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
gen, n, step = images.CONFIGS[cfg]
img = gen()
for _ in range(reps):
    enc = fic.encode(img, fic.CodecParams(n=n, step=step))
print(cfg, enc.stats)

"""Per-tile pipeline timestamps of CTA (0,0) of the tcgen05 matcher (FIC_DEBUG=32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
gen, n, step = images.CONFIGS[cfg]
img = gen()
fic.encode(img, fic.CodecParams(n=n, step=step))
os.environ["FIC_DEBUG"] = str(32 | extra)
fic.encode(img, fic.CodecParams(n=n, step=step))

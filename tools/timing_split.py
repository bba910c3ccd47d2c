"""Matcher time with the epilogue skipped (FIC_DEBUG=8) / MMAs skipped (16) / normal."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

for cfg in sys.argv[1:] or ["cfg2", "cfg4"]:
    gen, n, step = images.CONFIGS[cfg]
    img = gen()
    for flags in ["0", "8"]:
        os.environ["FIC_DEBUG"] = str(int(flags) | int(os.environ.get("FIC_DEBUG_BASE", "0")))
        fic.set_matcher_timing(True)
        fic.encode(img, fic.CodecParams(n=n, step=step))
        fic.matcher_timing(reset=True)
        for _ in range(3):
            fic.encode(img, fic.CodecParams(n=n, step=step))
        ms, k = fic.matcher_timing(reset=True)
        print(cfg, "flags", flags, f"matcher {ms:.3f} ms", flush=True)

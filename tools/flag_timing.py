"""Full-level scan time under debug flags (FIC_DEBUG): 0 normal, 8 no per-column test,
16 no MMAs, 128 no TMEM reads, 144 neither MMAs nor TMEM reads.  GPU analysis tool; the
codes of a debug run are meaningless (errors from the record self-check are ignored)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_0774_b200 as fic  # noqa: E402
from paper_1404_0774_b200 import images  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
gen, n, step = images.CONFIGS[cfg]
img = gen()
p = fic.CodecParams(n=n, step=step)
fic.encode(img, p)
for flags in sys.argv[2:] or ["0", "8", "16", "128", "144"]:
    os.environ["FIC_DEBUG"] = flags
    fic.set_matcher_timing(True)
    fic.scan_timing(reset=True)
    for _ in range(2):
        try:
            fic.encode(img, p)
        except Exception as e:  # noqa: BLE001
            print("  error:", str(e)[:160], flush=True)
    ms, k = fic.scan_timing(reset=True)
    fic.set_matcher_timing(False)
    print(f"{cfg} FIC_DEBUG={flags}: full-level scan {ms:.3f} ms ({k} launches)", flush=True)

"""Per-source-line instruction counts and warp-stall samples of one kernel in an ncu report
(`--import-source on`, built with -lineinfo).  Usage: python tools/ncu_lines.py REP [kernel-regex] [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kern=None, top=30):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kern:
        cmd += ["-k", "regex:" + kern, "--launch-count", "1"]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    his = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
    agg, aex = collections.Counter(), collections.Counter()
    for hi in his:
        h = rows[hi]
        isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        cur = None
        for r in rows[hi + 1:]:
            if "Warp Stall Sampling (All Samples)" in r:
                break
            if len(r) <= iex:
                continue
            if r[0].strip() and not r[0].startswith("0x"):
                cur = (r[0], r[isrc].strip()[:110])
                continue
            try:
                agg[cur] += int(r[iss] or 0)
                aex[cur] += int(float(r[iex] or 0))
            except ValueError:
                pass
    print(f"{'stall samples':>13} {'instructions':>12}  line  source")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:13d} {aex[k]:12d}  {k[0]:>5} {k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, int(sys.argv[3]) if len(sys.argv) > 3 else 30)

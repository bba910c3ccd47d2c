"""Print the raw ncu metrics of a report whose names match any of the given regexes."""
import csv
import io
import re
import subprocess
import sys

if __name__ == "__main__":
    rep, pats = sys.argv[1], [re.compile(p) for p in sys.argv[2:]]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        for n, un, x in zip(h, u, v):
            if any(p.search(n) for p in pats):
                try:
                    if float(x.replace(",", "")) == 0.0:
                        continue
                except ValueError:
                    pass
                print(f"{n:90s} {x} {un}")

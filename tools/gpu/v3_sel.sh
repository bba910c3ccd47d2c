# cfg3 timeline with the branch-free first-level selection, GPU suite
for C in cfg3 cfg3 cfg2; do echo "== $C"; timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep -v -i warn | cut -c1-62; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2

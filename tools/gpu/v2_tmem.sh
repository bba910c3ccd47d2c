# full-level scan time under debug switches: 8 = TMEM loads without the test, 128 = no TMEM
# reads, 16 = no MMAs; F16ACC = fp16 accumulators (packed loads)
k() { echo "== $*"; env "$@" timeout 300 python tools/kineto_gaps.py $C 2>&1 | grep "scan_kernel" | cut -c1-60; }
for C in cfg2 cfg3; do
  k X=0; k FIC_DEBUG=8; k FIC_DEBUG=128; k FIC_DEBUG=24; k FIC_F16ACC=1; k FIC_F16ACC=1 FIC_DEBUG=8
done

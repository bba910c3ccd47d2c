for l in libfic_b200.so libfic_b200_c2.so; do for c in cfg2 cfg3; do echo "== $c $l"; FIC_LIB=$PWD/paper_1404_0774_b200/$l timeout 300 python tools/kineto_gaps.py $c 2>&1 | cut -c1-90; done; done

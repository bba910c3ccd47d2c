for l in libfic_b200_old.so libfic_b200.so; do echo "== $l"; FIC_LIB=$PWD/paper_1404_0774_b200/$l timeout 300 python tools/e2e_probe.py cfg2; done

timeout 300 python tools/kineto_gaps.py cfg1 2>&1 | grep -v -i warn
FIC_DEBUG=4 timeout 60 python tools/encode_once.py cfg1 2>&1 | tail -3

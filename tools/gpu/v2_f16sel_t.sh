timeout 900 python -m pytest tests/test_gpu_encode.py -x -q -m gpu 2>&1 | grep -v "^\.\|passed" | tail -40
timeout 900 python -m pytest tests/test_gpu_encode.py -q -m gpu 2>&1 | tail -3

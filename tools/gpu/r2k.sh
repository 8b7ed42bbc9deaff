python tools/gpu/ts_ab.py "" 2>&1 | tail -8
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4

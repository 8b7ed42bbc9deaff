python tools/gpu/ts_ab.py "" 2>&1 | tail -8
WPM_DEBUG_LIB=debug timeout 600 python tools/time_n.py 2 3 4 5 6 2>&1 | tail -5 | cut -c1-120
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_synthetic.py -q -x 2>&1 | tail -2

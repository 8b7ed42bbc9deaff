for n in 2 3 4; do python tools/gpu/n2.py $n 2>&1 | tail -1; done
python tools/gpu/ts_ab.py "" 2>&1 | tail -8
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthetic.py -q -x 2>&1 | tail -2

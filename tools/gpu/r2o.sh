python tools/time_n.py 2 4 5 8 11 2>&1 | tail -5 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], 'sort', d['ms_sort'], 'search', d['ms_search'], 'total', d['ms_total'], 'dups', d['dups'], d['wpms'])"
python tools/e2e_trace.py 5 2>&1 | grep call
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthetic.py tests/test_gpu_multi.py -q -x 2>&1 | tail -2

python tools/time_n.py 4 5 6 7 8 9 10 11 2>&1 | tail -8 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], 'sort', d['ms_sort'], 'search', d['ms_search'], 'total', d['ms_total'], 'dups', d['dups'])"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line13.py tests/test_gpu_alg1.py tests/test_gpu_multi.py -q -x 2>&1 | tail -2

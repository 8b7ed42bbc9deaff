for t in 1024 2048 4096; do WPM_SORT_TILE=$t python tools/time_n.py 5 8 11 2>&1 | tail -3 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print('tile', $t, d['n'], 'sort', d['ms_sort'], 'search', d['ms_search'], 'total', d['ms_total'])"; done
python -m pytest tests/test_gpu_parity.py -q -x -k "digest or counts" 2>&1 | tail -2
python tools/gpu/claim_ab.py 2>&1 | grep claim

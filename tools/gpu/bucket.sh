cd $GRAFT_REPO_ROOT
timeout 200 python tools/gpu/sort_probe.py 2 3 4 5 6 7 8 9 10 11 2>&1
WPM_SORT=merge timeout 200 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed 's/^/merge /'
timeout 300 python tools/gpu/mapq.py 2 3 4 5 6 7 8 9 10 11 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5

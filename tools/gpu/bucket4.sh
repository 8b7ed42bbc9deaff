cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/mapq.py 2 3 4 5 8 11 2>&1
WPM_SORT=bucket timeout 300 python tools/gpu/mapq.py 4 5 6 8 11 2>&1 | sed 's/^/bucket /'
timeout 100 python tools/gpu/sort_probe.py 4 5 6 7 8 9 10 11 2>&1
WPM_SORT=bucket WPM_BUCKET_TILE=1024 timeout 100 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed 's/^/bucket /'
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -x -q 2>&1 | tail -3

cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/mapq.py 2 3 4 5 6 7 8 9 10 11 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5

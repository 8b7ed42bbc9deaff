set -x
cd $GRAFT_REPO_ROOT
timeout 120 python tools/gpu/mapq.py 7 8 6 5 9 2>&1
WPM_MAPQ=0 timeout 120 python tools/gpu/mapq.py 7 8 2>&1
for h in 8 16 64 128; do WPM_HUNGRY=$h timeout 120 python tools/gpu/mapq.py 7 8 2>&1; done
timeout 600 python -m pytest tests -m gpu -x -q -k "multi or split or progress or parity" 2>&1 | tail -5

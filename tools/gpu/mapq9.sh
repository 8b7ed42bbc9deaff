cd $GRAFT_REPO_ROOT
timeout 120 python tools/gpu/mapq.py 9 10 2>&1
for h in 32 128 512; do WPM_MAPQ9=1 WPM_HUNGRY=$h timeout 120 python tools/gpu/mapq.py 9 10 2>&1 | sed "s/^/q9 h$h /"; done

cd $GRAFT_REPO_ROOT
for st in 4 5 0; do WPM_BUCKET_STOP=$st timeout 100 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed "s/^/stop $st /"; done
for st in 4 5 0; do WPM_BUCKET_TILE=1024 WPM_BUCKET_STOP=$st timeout 100 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed "s/^/T1024 stop $st /"; done

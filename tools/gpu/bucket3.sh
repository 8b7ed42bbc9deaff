cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/mapq.py 2 3 4 5 8 11 2>&1
for t in 512 1024 2048 4096; do WPM_BUCKET_TILE=$t timeout 100 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed "s/^/T $t /"; done
for st in 1 2 3 4; do WPM_BUCKET_TILE=1024 WPM_BUCKET_STOP=$st timeout 100 python tools/gpu/sort_probe.py 5 8 11 2>&1 | sed "s/^/T1024 stop $st /"; done

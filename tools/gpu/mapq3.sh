cd $GRAFT_REPO_ROOT
for w in 20 10 8; do for h in 32 128; do WPM_MAPQ_WPB=$w WPM_HUNGRY=$h timeout 120 python tools/gpu/mapq.py 7 8 2>&1 | sed "s/^/wpb $w /"; done; done
WPM_MAPQ=0 timeout 120 python tools/gpu/mapq.py 7 8 2>&1

cd $GRAFT_REPO_ROOT
for q in 1 0; do WPM_MAPQ=$q WPM_DEBUG_LIB=prof WPM_PROFILE=1 timeout 120 python tools/gpu/mapq.py 8 7 9 2>&1 | grep -v "^\[wpm\] poll"; done
WPM_DEBUG_LIB=prof WPM_PROFILE=1 timeout 120 python tools/gpu/c8t.py 2>&1 | tail -12

cd $GRAFT_REPO_ROOT
for v in "" r64 r80; do WPM_DEBUG_LIB=$v timeout 120 python tools/time_n.py 5 8 11 > gpurun_out/sw_v$v.log 2>&1; done

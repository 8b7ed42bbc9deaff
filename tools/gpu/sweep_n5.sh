cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 60 python tools/gpu/sort_probe.py 5 2>&1 | sed "s/^/$* /"; }
run X=0
for v in 8 64 256 1024; do run WPM_BACKOFF_MIN=$v; done
for v in 1024 4096 32768; do run WPM_BACKOFF_MAX=$v; done
for v in 256 1024 6000 20000; do run WPM_HUNGRY=$v; done
for v in 8 12 24 32; do run WPM_CHECK_EVERY=$v; done
run WPM_BLOCKS_PER_SM=1
run WPM_DONATE_MAX=2
run WPM_DONATE_MAX=4

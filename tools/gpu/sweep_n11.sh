cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 60 python tools/gpu/sort_probe.py 11 2>&1 | sed "s/^/$* /"; }
run X=0
for v in 128 512 2048; do run WPM_BACKOFF_MIN=$v; done
for v in 2048 16384 65536; do run WPM_BACKOFF_MAX=$v; done
for v in 256 1024 4000; do run WPM_HUNGRY=$v; done
for v in 16 24 48 64; do run WPM_CHECK_EVERY=$v; done
run WPM_DONATE_MAX=2
run WPM_TS=0

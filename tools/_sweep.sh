cd $GRAFT_REPO_ROOT
timeout 120 python tools/time_n.py 5 8 11 > gpurun_out/sw_default.log 2>&1
for h in 1 32 256; do WPM_HUNGRY=$h timeout 120 python tools/time_n.py 5 8 11 > gpurun_out/sw_h$h.log 2>&1; done
WPM_BACKOFF_MAX=2048 timeout 120 python tools/time_n.py 5 8 11 > gpurun_out/sw_b2048.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "counts_and_nodes or random or constrained or full_subset or shards or small or octa" > gpurun_out/t6.log 2>&1

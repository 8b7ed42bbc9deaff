# poll backoff at n = 7, 8 (map queues): first sleep 32 (default) / 256 / 1024 ns, cap 8 / 32 us
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=7 timeout 1200 python tools/ab_k3.py 5,7,8,9 ":" ":WPM_BACKOFF_MIN=256" ":WPM_BACKOFF_MIN=1024" ":WPM_BACKOFF_MAX=32768" ":WPM_BACKOFF_MIN=256,WPM_BACKOFF_MAX=32768" ":" > gpurun_out/r3i_ab_backoff.jsonl 2>&1; cat gpurun_out/r3i_ab_backoff.jsonl

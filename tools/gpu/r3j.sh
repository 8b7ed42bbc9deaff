# poll backoff first sleep 32 (default) / 1024 / 2048 / 4096 ns at n = 4, 5, 6, 10, 11
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=9 timeout 1200 python tools/ab_k3.py 4,5,6,10,11 ":" ":WPM_BACKOFF_MIN=1024" ":WPM_BACKOFF_MIN=2048" ":WPM_BACKOFF_MIN=4096" ":" ":WPM_BACKOFF_MIN=1024" ":WPM_BACKOFF_MIN=2048" ":WPM_BACKOFF_MIN=4096" > gpurun_out/r3j_ab_backoff2.jsonl 2>&1; cat gpurun_out/r3j_ab_backoff2.jsonl

# first donation check of a task after 1 / 2 / 4 / 8 nodes (default: check_every = 16 at n <= 6, 32 above)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=9 timeout 1200 python tools/ab_k3.py 4,5,6,8,11 ":" ":WPM_FIRST_CHECK=1" ":WPM_FIRST_CHECK=2" ":WPM_FIRST_CHECK=4" ":WPM_FIRST_CHECK=8" ":" ":WPM_FIRST_CHECK=2" ":WPM_FIRST_CHECK=4" > gpurun_out/r3k_ab_first.jsonl 2>&1; cat gpurun_out/r3k_ab_first.jsonl

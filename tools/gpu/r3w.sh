# donation check interval and hunger threshold at small n with the 1 us first poll sleep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=9 timeout 1200 python tools/ab_k3.py 4,5,6 ":" ":WPM_CHECK_EVERY=8" ":WPM_CHECK_EVERY=24" ":WPM_CHECK_EVERY=32" ":WPM_HUNGRY=256" ":WPM_HUNGRY=4096" ":" > gpurun_out/r3w_ab_check.jsonl 2>&1; cat gpurun_out/r3w_ab_check.jsonl

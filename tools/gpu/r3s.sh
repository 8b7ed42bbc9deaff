# starvation-adaptive donation checks: direct runs and the shard-run projection
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=7 timeout 1200 python tools/ab_k3.py 5,8,11 ":" ":WPM_STARVE_AT=512,WPM_STARVE_CHECK=4" ":WPM_STARVE_AT=512,WPM_STARVE_CHECK=8" ":WPM_STARVE_AT=1024,WPM_STARVE_CHECK=4" ":WPM_STARVE_AT=256,WPM_STARVE_CHECK=8" ":" > gpurun_out/r3s_ab.jsonl 2>&1; cat gpurun_out/r3s_ab.jsonl
WPM_STARVE_AT=512 WPM_STARVE_CHECK=8 timeout 900 python tools/gpu/proj_probe.py 640 > gpurun_out/r3s_proj_a.jsonl 2>/dev/null; cat gpurun_out/r3s_proj_a.jsonl
WPM_STARVE_AT=512 WPM_STARVE_CHECK=4 timeout 900 python tools/gpu/proj_probe.py 640 > gpurun_out/r3s_proj_b.jsonl 2>/dev/null; cat gpurun_out/r3s_proj_b.jsonl

# for_pairs (exact n-lane packing for the n >= 9 classes): parity + timing; per-call e2e trace
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "orbit or synthetic or universe" > gpurun_out/r3c_parity.log 2>&1; tail -3 gpurun_out/r3c_parity.log
AB_REPS=9 timeout 900 python tools/ab_k3.py 5,8,9,10,11 ":" > gpurun_out/r3c_ab.jsonl 2>&1; cat gpurun_out/r3c_ab.jsonl
WPM_TRACE=2 timeout 120 python tools/e2e_trace.py 5 > gpurun_out/r3c_e2e_trace.txt 2>&1; tail -60 gpurun_out/r3c_e2e_trace.txt

# run_claim on a plan that did not split (fix + test); shard-run projection; fresh ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r3q_multi.log 2>&1; tail -2 gpurun_out/r3q_multi.log
timeout 1500 python tools/gpu/proj_probe.py 640 2048 > gpurun_out/r3q_proj.jsonl 2> gpurun_out/r3q_proj.err; cat gpurun_out/r3q_proj.jsonl; tail -3 gpurun_out/r3q_proj.err
bash tools/gpu/r3p.sh

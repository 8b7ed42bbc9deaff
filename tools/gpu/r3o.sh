# shard-run projection (each W-GPU shard's claim phase timed on its own) at per-GPU targets 640 / 2048 / 4096
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/gpu/proj_probe.py 640 2048 4096 > gpurun_out/r3o_proj.jsonl 2> gpurun_out/r3o_proj.err; cat gpurun_out/r3o_proj.jsonl; tail -3 gpurun_out/r3o_proj.err

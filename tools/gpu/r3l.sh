# multi-GPU projection at per-GPU frontier targets 96 / 160 / 256 / 400 / 640
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/gpu/proj_probe.py 96 160 256 400 640 > gpurun_out/r3l_proj.jsonl 2> gpurun_out/r3l_proj.err; cat gpurun_out/r3l_proj.jsonl; tail -3 gpurun_out/r3l_proj.err

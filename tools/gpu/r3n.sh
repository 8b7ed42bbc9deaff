# multi-GPU projection, list-schedule and static columns, per-GPU frontier targets 32 .. 640
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/gpu/proj_probe.py 32 64 96 160 320 640 > gpurun_out/r3n_proj.jsonl 2> gpurun_out/r3n_proj.err; cat gpurun_out/r3n_proj.jsonl; tail -3 gpurun_out/r3n_proj.err

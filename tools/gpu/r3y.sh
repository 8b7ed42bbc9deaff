# final validation: the GPU suite, then profiles + bench + reference arm (r3z.sh, TAG=r02f)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_gpu_tests.log 2>&1; tail -3 gpurun_out/r02f_gpu_tests.log
TAG=r02f bash tools/gpu/r3z.sh

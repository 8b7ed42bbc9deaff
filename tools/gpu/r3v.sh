# final GPU suite + smoke, then more exhaustive Algorithm-1 chunks at n = 10
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3v_smoke.log 2>&1; tail -1 gpurun_out/r3v_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3v_gpu_tests.log 2>&1; tail -3 gpurun_out/r3v_gpu_tests.log
ALG1_BUDGET=1380 bash tools/gpu/alg1_n10.sh

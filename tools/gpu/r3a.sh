# session re-entry check: smoke, the GPU suite, a short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; tail -1 gpurun_out/r3a_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-per-n > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err; tail -c 1500 gpurun_out/r3a_bench.json
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_gpu_tests.log 2>&1; tail -5 gpurun_out/r3a_gpu_tests.log

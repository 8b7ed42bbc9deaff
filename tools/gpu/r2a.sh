set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests.log 2>&1; tail -30 gpurun_out/multi_tests.log
timeout 600 oracle/_ref/adapter_check > gpurun_out/adapter.log 2>&1; tail -5 gpurun_out/adapter.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reach.py -x -q > gpurun_out/parity_tests.log 2>&1; tail -15 gpurun_out/parity_tests.log
python bench.py --steps 20 --warmup 5 --no-per-n --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -c 1500 gpurun_out/bench_quick.json

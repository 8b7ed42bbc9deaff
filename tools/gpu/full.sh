python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; tail -1 gpurun_out/full_smoke.log
timeout 1500 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; tail -c 300 gpurun_out/full_bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/full_bench_ref.json 2>&1; tail -c 400 gpurun_out/full_bench_ref.json
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/full_gpu_tests.log 2>&1; tail -3 gpurun_out/full_gpu_tests.log

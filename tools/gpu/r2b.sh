set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_reach.py -x -q > gpurun_out/multi_tests.log 2>&1; tail -5 gpurun_out/multi_tests.log
python bench.py --steps 20 --warmup 5 --no-per-n --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print(d['ms_per_step'], d['breakdown_ms'], d['e2e']['wall_ms'], d['parity'])"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log

# staging + block cache + cached occupancy + orbit bitmap: e2e trace, bench, full GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e_smoke.log 2>&1; tail -1 gpurun_out/r3e_smoke.log
WPM_TRACE=2 timeout 120 python tools/e2e_trace.py 5 > gpurun_out/r3e_e2e_trace.txt 2>&1; tail -42 gpurun_out/r3e_e2e_trace.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-per-n --no-cpu-baseline > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r3e_bench.json')); print(d['ms_per_step'], d['e2e']['wall_ms'], d['e2e']['samples_ms'], d['e2e_dropin'])"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3e_gpu_tests.log 2>&1; tail -5 gpurun_out/r3e_gpu_tests.log

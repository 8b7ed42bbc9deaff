# pinned staging of the small copies: smoke, multi-GPU protocol tests, per-call e2e trace, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3d_smoke.log 2>&1; tail -1 gpurun_out/r3d_smoke.log
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_synthetic.py -x -q > gpurun_out/r3d_tests.log 2>&1; tail -3 gpurun_out/r3d_tests.log
WPM_TRACE=2 timeout 120 python tools/e2e_trace.py 5 > gpurun_out/r3d_e2e_trace.txt 2>&1; tail -45 gpurun_out/r3d_e2e_trace.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-per-n --no-cpu-baseline > gpurun_out/r3d_bench.json 2> gpurun_out/r3d_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r3d_bench.json')); print(d['ms_per_step'], d['e2e']['wall_ms'], d['e2e']['samples_ms'], d['e2e_dropin'])"

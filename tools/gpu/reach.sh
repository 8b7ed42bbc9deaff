set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_reach.py -x -q -k "not pinned" > gpurun_out/reach_tests.log 2>&1; tail -15 gpurun_out/reach_tests.log
timeout 1200 python tests/golden/make_golden_reach.py gpurun_out/reach.json > gpurun_out/reach_golden.log 2>&1; tail -5 gpurun_out/reach_golden.log

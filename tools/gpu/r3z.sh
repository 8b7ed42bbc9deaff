# final profiles of this session's code (summaries travel back), then the full bench and the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r02e}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reach.py tests/test_gpu_multi.py -x -q -k "11 or multi or reach" > gpurun_out/${TAG}_n11_tests.log 2>&1; tail -2 gpurun_out/${TAG}_n11_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
for n in 5 8 11; do
  nodes=$(python -c "import json; print(json.load(open('tests/golden/golden.json'))['dfs']['$n']['nodes'])")
  ncu -f --set full --import-source on -k regex:k3_search -s 1 -c 1 -o /tmp/k3_n$n python tools/gpu/k3_probe.py $n 2 > /tmp/k3_n$n.log 2>&1
  python tools/ncu_summary.py /tmp/k3_n$n.ncu-rep $nodes gpurun_out/${TAG}_k3_n${n}_ncu.txt "search node"
done
ncu -f --set full --import-source on -k regex:k4_sort -s 2 -c 1 -o /tmp/k4_n5 python tools/gpu/sort_probe.py 5 > /tmp/k4_n5.log 2>&1
python tools/ncu_summary.py /tmp/k4_n5.ncu-rep 0 gpurun_out/${TAG}_k4_n5_ncu.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-per-n --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv 2 gpurun_out/${TAG}_bench_n5_launches.txt
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 300 gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; tail -c 300 gpurun_out/${TAG}_bench_ref.json

# the full bench with this session's final code (r02h), the reference arm, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; tail -1 gpurun_out/r02h_smoke.log
timeout 1500 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; tail -c 300 gpurun_out/r02h_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r02h_bench.json')); print(d['ms_per_step'], d['e2e']['wall_ms'], d['e2e_dropin']['wall_ms'], d['roofline'])
for c in d['scaling_projection']['cases']: print(c['case'], [(w['W'], w['projected_speedup'], w['list_schedule_bound_speedup'], w['claim_ms_slowest_shard'], w['claim_ms_mean_shard']) for w in c['by_W']])"
timeout 900 python bench.py --impl reference > gpurun_out/r02h_bench_ref.json 2> gpurun_out/r02h_bench_ref.err; tail -c 200 gpurun_out/r02h_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches.csv python bench.py --steps 2 --warmup 3 --no-per-n --no-cpu-baseline > gpurun_out/r02h_ncu_bench.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/r02h_launches.csv 2 gpurun_out/r02h_bench_n5_launches.txt

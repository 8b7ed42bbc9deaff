# the full bench once more (bench.py's projection rewrite), then the exhaustive Algorithm 1 at n = 10 in chunks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; tail -c 400 gpurun_out/r02g_bench.err; python -c "
import json; d=json.load(open('gpurun_out/r02g_bench.json')); print(d['ms_per_step'], d['e2e']['wall_ms'])
for c in d['scaling_projection']['cases']: print(c['case'], [(w['W'], w['projected_speedup'], w['list_schedule_bound_speedup']) for w in c['by_W']])"
ALG1_BUDGET=${ALG1_BUDGET:-3600} bash tools/gpu/alg1_n10.sh

set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for t in 2048 4096 8192; do for c in 512 1024 2048; do WPM_SORT_TILE=$t WPM_SORT_CHUNK=$c python tools/time_n.py 5 8 > gpurun_out/sort_${t}_${c}.txt 2>&1; echo "tile $t chunk $c"; cat gpurun_out/sort_${t}_${c}.txt | tail -3; done; done
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 600 gpurun_out/bench_full.err; python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); print(d['ms_per_step'], d['breakdown_ms'], d['e2e']['wall_ms'], d['e2e_dropin'], d['parity']); print(json.dumps(d['scaling_projection'])[:3000]); print(json.dumps(d['cpu_baseline']))"

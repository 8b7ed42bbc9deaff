python -c "
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench, torch
import paper_2301_00806_b200 as wpm
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda:0')
r = bench.scaling_projection(wpm, 0, flush)
for c in r['cases']: print(c['case'], c['frontier_records'], c['split_ms_by_W'], c['claim_ms'], c['one_gpu_run_ms'], [(w['W'], round(w['static_max_over_mean'],3), round(w['dynamic_makespan_over_mean'],4), float(w['projected_speedup']), float(w['projected_speedup_static_split'])) for w in c['by_W']])
"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2

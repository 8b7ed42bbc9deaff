python -c "
import os, sys, json
sys.path.insert(0, os.getcwd())
import bench, torch
import paper_2301_00806_b200 as wpm
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda:0')
r = bench.scaling_projection(wpm, 0, flush)
for c in r['cases']: print(c['case'], c['frontier_records'], c['split_ms_host'], c['claim_ms'], c['one_gpu_run_ms'], [(w['W'], round(w['static_max_over_mean'],3), round(w['dynamic_makespan_over_mean'],4), w['projected_speedup'], w['projected_speedup_static_split']) for w in c['by_W']])
"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x -k "multi or claim or split or kernel1 or kernel2 or shuffled" 2>&1 | tail -2

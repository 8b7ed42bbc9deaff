"""Scaling projection (bench.scaling_projection) at several per-GPU frontier targets (dev tool)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2301_00806_b200 as wpm  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda:0")
for per in [int(x) for x in sys.argv[1:]] or [640]:
    r = bench.scaling_projection(wpm, 0, flush, per_gpu=per)
    for c in r["cases"]:
        w8 = [w for w in c["by_W"] if w["W"] == 8][0]
        print(json.dumps({"per_gpu": per, "case": c["case"], "records": c["frontier_records"],
                          "split_ms_W8": c["split_ms_host"], "largest_record_frac": c["largest_record_frac"],
                          "one_gpu_ms": c["one_gpu_run_ms"], "claim_ms": c["claim_ms"],
                          "W8_makespan_over_mean": w8["dynamic_makespan_over_mean"],
                          "W8_static_max_over_mean": w8["static_max_over_mean"],
                          "speedup": {w["W"]: w["projected_speedup"] for w in c["by_W"]},
                          "speedup_static": {w["W"]: w["projected_speedup_static_split"] for w in c["by_W"]}}), flush=True)

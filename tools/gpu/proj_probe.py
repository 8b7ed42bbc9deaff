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
        print(json.dumps({"per_gpu": per, "case": c["case"], "records": c["frontier_records"],
                          "split_ms": c["split_ms_by_W"], "one_gpu_ms": c["one_gpu_run_ms"],
                          "claim_all_ms": c["claim_ms_one_gpu_all_records"],
                          "claim_slowest": {w["W"]: w["claim_ms_slowest_shard"] for w in c["by_W"]},
                          "speedup": {w["W"]: w["projected_speedup"] for w in c["by_W"]},
                          "list_bound": {w["W"]: w["list_schedule_bound_speedup"] for w in c["by_W"]}}), flush=True)

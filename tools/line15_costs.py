"""Per-survivor cost of the line-15 canonical-labeling search on the GPU:
prints the distribution and dumps the most expensive complexes (facet masks,
placements) to gpurun_out/l15_heavy_n{n}.json.  Development tool."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2301_00806_b200 as wpm  # noqa: E402

for n in [int(x) for x in sys.argv[1:]]:
    with wpm.Plan.orbits(n) as p:
        p.run()
        p.line13()
        p.line15()
        st = p.line15_stats()
        cost = p.line15_costs()
        surv = p.fetch_complexes(13)
        order = np.argsort(-cost)
        tot = int(cost.sum())
        q = np.percentile(cost, [50, 90, 99, 99.9]).tolist()
        print(json.dumps({"n": n, **st, "total": tot, "max": int(cost.max()), "pct50_90_99_999": q,
                          "top10_share": float(cost[order[:10]].sum() / max(tot, 1))}), flush=True)
        heavy = [{"i": int(i), "cost": int(cost[i]), "facets": surv.complex(int(i))} for i in order[:40]]
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump({"n": n, "m": n + 4, "heavy": heavy}, open(os.path.join(ROOT, "gpurun_out", f"l15_heavy_n{n}.json"), "w"))

"""A/B of the claim phase vs the seeded frontier vs the root tasks (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm

def run(n, mode, depth=3, target=4096):
    with wpm.Plan.orbits(n) as p:
        best = None
        for _ in range(3):
            if mode == "roots":
                p.run(); ms = p.timing()["ms_total"]; st = p.stats()
            elif mode == "seeded":
                p.set_split(depth); p.run(); ms = p.timing()["ms_total"]; st = p.stats()
            else:
                ctr, _ = wpm.claim_counter_create(0)
                t0 = time.perf_counter()
                f = p.split(depth, target)
                p.run_claim(ctr)
                ms = (time.perf_counter() - t0) * 1e3
                wpm.claim_counter_close(0, ctr, False)
                st = p.stats()
            best = min(best or 1e9, ms)
        return {"n": n, "mode": mode, "env": os.environ.get("WPM_CLAIM_LOW"), "depth": depth, "target": target,
                "ms": round(best, 3), "ms_search": round(st["ms_search"], 3), "nodes": st["nodes"], "tasks": st["tasks"]}

for n in (5, 8, 11):
    print(json.dumps(run(n, "roots")), flush=True)
    for d in (2, 3, 4, 5):
        print(json.dumps(run(n, "seeded", d)), flush=True)
    print(json.dumps(run(n, "claim")), flush=True)

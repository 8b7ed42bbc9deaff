import os, sys, time, json
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
for n in (8, 11):
    with wpm.Plan.orbits(n) as p:
        p.run(); t_run = p.timing()["ms_total"]
        for d in (3, 5, 7, 9, 11, 13):
            ctr, _ = wpm.claim_counter_create(0)
            best = None
            for _ in range(2):
                wpm.claim_counter_reset(0, ctr)
                t0 = time.perf_counter(); F = p.split(d, 1); t1 = time.perf_counter()
                p.run_claim(ctr); t2 = time.perf_counter()
                r = ((t1 - t0) * 1e3, (t2 - t1) * 1e3, F, p.stats()["nodes"])
                best = r if best is None or r[0] + r[1] < best[0] + best[1] else best
            wpm.claim_counter_close(0, ctr, False)
            print(json.dumps({"n": n, "depth": d, "split_ms": round(best[0], 3), "claim_ms": round(best[1], 3), "records": best[2], "nodes": best[3], "direct_ms": round(t_run, 3)}), flush=True)

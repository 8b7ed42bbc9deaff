"""A/B of kernel-3 variants via env knobs (dev tool): median search ms of 5 runs."""
import json, os, statistics, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2301_00806_b200 as wpm
import catalog as C
cases = [("5", None), ("6", None), ("8", None), ("9", None), ("10", None), ("11", None), ("syn", 0.80)]
knobs = [dict(x.split("=") for x in a.split(",")) if a else {} for a in sys.argv[1:]] or [{}]
g = json.load(open("tests/golden/golden.json"))
for name, d in cases:
    for k in knobs:
        for kk in ("WPM_TS", "WPM_BACKOFF_MIN", "WPM_BACKOFF_MAX", "WPM_BLOCKS_PER_SM", "WPM_CHECK_EVERY"):
            os.environ.pop(kk, None)
        os.environ.update(k)
        p = wpm.Plan.universes(15, 11, [C.synthetic_universe(1, d)], facet_cap=252) if d else wpm.Plan.orbits(int(name))
        with p:
            ms = []
            for _ in range(6):
                p.run()
                st = p.stats()
                ms.append(st["ms_search"])
            ok = None if d else (st["nodes"] == g["dfs"][name]["nodes"] and p.fetch().total == g["dfs"][name]["sum"])
            print(json.dumps({"case": name, "knobs": k, "ms": round(statistics.median(ms[1:]), 3), "nodes": st["nodes"],
                              "Gn/s": round(st["nodes"] / statistics.median(ms[1:]) / 1e6, 3), "ok": ok,
                              "warps": p.timing()["warps"]}), flush=True)

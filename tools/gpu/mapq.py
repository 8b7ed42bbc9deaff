"""Map-queue A/B: full-orbit n = 6..9 plans, WPM_MAPQ / WPM_HUNGRY from the env
(set per child process by mapq.sh); median search ms and the golden check."""
import json, os, sys, statistics
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
g = json.load(open("tests/golden/golden.json"))
for n in [int(x) for x in sys.argv[1:]]:
    with wpm.Plan.orbits(n) as p:
        ms = []
        for _ in range(6):
            tot = p.run()
            ms.append(p.stats()["ms_search"])
        st = p.stats()
        res = p.fetch()
        ok = tot == g["dfs"][str(n)]["sum"] and st["nodes"] == g["dfs"][str(n)]["nodes"] and res.counts == [m["wpms"] for m in g["dfs"][str(n)]["maps"]]
        med = statistics.median(ms[1:])
        print("mapq", os.environ.get("WPM_MAPQ", "1"), "hungry", os.environ.get("WPM_HUNGRY", "-"), "n", n, "warps", p.timing()["warps"],
              "ms", round(med, 3), "min", round(min(ms[1:]), 3), "Gn/s", round(st["nodes"] / med / 1e6, 3), "OK" if ok else "MISMATCH", flush=True)

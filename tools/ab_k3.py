"""A/B of kernel-3 builds and launch knobs (dev tool).

Each setting runs in its own process (the library variant is chosen at
import time by WPM_DEBUG_LIB): median search ms over R runs per n, with the
WPM total and node count checked against tests/golden/golden.json.

  python tools/ab_k3.py 5,8,11 base: WPM_CARVEOUT=75,WPM_BLOCKS_PER_SM=6 ...
  (a setting is LIB:ENV1=V1,ENV2=V2; empty LIB = the product build)
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, statistics, sys
sys.path.insert(0, %r)
import paper_2301_00806_b200 as wpm
g = json.load(open(os.path.join(%r, "tests", "golden", "golden.json")))["dfs"]
reps = int(os.environ.get("AB_REPS", "7"))
for n in [int(x) for x in sys.argv[1].split(",")]:
    with wpm.Plan.orbits(n) as p:
        ms, tot = [], []
        for _ in range(reps + 1):
            p.run()
            st, tm = p.stats(), p.timing()
            ms.append(st["ms_search"]); tot.append(tm["ms_total"])
        r = p.fetch()
    ok = r.total == g[str(n)]["sum"] and st["nodes"] == g[str(n)]["nodes"]
    print(json.dumps({"n": n, "ok": ok, "wpms": r.total, "nodes": st["nodes"],
                      "ms_search_med": round(statistics.median(ms[1:]), 3), "ms_search_min": round(min(ms[1:]), 3),
                      "ms_total_med": round(statistics.median(tot[1:]), 3)}), flush=True)
"""


def main():
    ns = sys.argv[1]
    for setting in sys.argv[2:]:
        lib, _, envs = setting.partition(":")
        env = dict(os.environ)
        env.pop("WPM_DEBUG_LIB", None)
        if lib:
            env["WPM_DEBUG_LIB"] = lib
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, ROOT), ns], env=env, capture_output=True,
                             text=True, timeout=900)
        for line in out.stdout.splitlines():
            print(json.dumps({"setting": setting, **json.loads(line)}), flush=True)
        if out.returncode:
            print(json.dumps({"setting": setting, "error": out.stderr[-800:]}), flush=True)


if __name__ == "__main__":
    main()

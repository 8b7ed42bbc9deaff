"""Prints DESIGN.md's per-n table from a bench.py JSON line (dev tool).
usage: python tools/design_tables.py profiles/<bench>.json """
import json
import sys

d = json.load(open(sys.argv[1]))
# round-1 step ms (the driver's BENCH_r01 per_n)
r1 = {2: 0.24, 3: 0.45, 4: 0.91, 5: 2.25, 6: 10.07, 7: 28.0, 8: 44.7, 9: 46.2, 10: 37.3, 11: 22.6}
maps = {2: 7, 3: 16, 4: 28, 5: 35, 6: 35, 7: 28, 8: 16, 9: 7, 10: 3, 11: 1}
print("| n | maps | WPMs | search nodes | k3 ms | sort ms | step ms | Gnodes/s (k3) | e2e ms | round 1 step ms |")
print("|---|---|---|---|---|---|---|---|---|---|")
for e in d["per_n"]:
    n = e["n"]
    g = e["nodes"] / (e["ms_search"] * 1e-3) / 1e9
    prev = r1.get(n, "")
    print(f"| {n} | {e.get('maps', maps.get(n))} | {e['wpms']:,} | {e['nodes']:,} | {e['ms_search']:.2f} | "
          f"{e['ms_sort']:.2f} | {e['ms_step']:.2f} | {g:.2f} | {e['e2e_ms']:.2f} | {prev} |")

"""Writes golden.json["reach"] for n = 10, 11 -- the SURVEY 8(c)(2)-(3)
protocol run on the B200 (needs a GPU; run once, the record is committed):

  python tests/golden/make_golden_reach.py [out.json]

Per n: rows, unsound / unreachable counts (must be 0), and for each of the
sampled prefixes the map, the fixed reference candidates of the outer
blocks, the inner space's leaves, the reference odometer's accepted count,
the DFS count sharing the prefix and the two-sided equality."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2301_00806_b200 as wpm  # noqa: E402
from reach_protocol import run_protocol  # noqa: E402

SAMPLES, SEED = 200, 2301
MAX_LEAVES = {10: 1 << 32, 11: 1 << 32}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "reach.json")
    rec = {}
    for n in (10, 11):
        t0 = time.time()
        r = run_protocol(wpm, n, SAMPLES, MAX_LEAVES[n], seed=SEED)
        r.update({"samples_requested": SAMPLES, "max_leaves": MAX_LEAVES[n], "seed": SEED,
                  "seconds": round(time.time() - t0, 1),
                  "all_equal": all(s["equal"] for s in r["samples"]),
                  "leaves_total": sum(s["leaves"] for s in r["samples"]),
                  "wpms_compared": sum(s["dfs"] for s in r["samples"])})
        rec[str(n)] = r
        print(n, r["rows"], r["unsound"], r["unreachable"], r["all_equal"], r["seconds"], flush=True)
    json.dump(rec, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()

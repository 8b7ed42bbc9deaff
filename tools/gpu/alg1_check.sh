cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f /tmp/a6.jsonl /tmp/a7.jsonl
timeout 300 python tools/alg1_full.py 6 /tmp/a6.jsonl --chunk-leaves 1e7 2>&1 | tail -2
python - <<'PY'
import json
for f in ("/tmp/a6.jsonl",):
    r=[json.loads(l) for l in open(f)]
    print(f, len(r), "chunks, all equal:", all(x["equal"] for x in r), "odometer sum", sum(x["odometer"] for x in r), "dfs sum", sum(x["dfs"] for x in r), "leaves", sum(x["leaves"] for x in r), "s", round(sum(x["s"] for x in r),1))
PY
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
import paper_2301_00806_b200 as wpm
from reach_protocol import ncand
sys.path.insert(0, "tools")
from alg1_full import chunks_of
for n in (9, 10, 11):
    with wpm.Plan.orbits(n) as p:
        p.run()
        for i in range(p.num_maps):
            w = p.space_blocks(i)
            tot = 1
            for x in w: tot *= ncand(x)
            j, pre = chunks_of(w, 2e13)
            print("n", n, "map", i, "blocks", len(w), "widths", w[:8], "leaves %.3e" % tot, "chunks@2e13", len(pre), "nfixed", j, flush=True)
PY

"""Line-15 probe on the GPU: per n, the device pipeline (search, line 13,
line 15) with counts, device times and the labeling-search sizes, checked
against golden.json["line15"] where present.  Development tool."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2301_00806_b200 as wpm  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
ns = [int(x) for x in sys.argv[1:]] or list(range(2, 12))
for n in ns:
    with wpm.Plan.orbits(n) as p:
        p.run()
        l7, l13 = p.line13()
        t0 = time.perf_counter()
        l15 = p.line15()
        wall = (time.perf_counter() - t0) * 1e3
        st = p.line15_stats()
        reps = p.fetch_complexes(15)
        sha = hashlib.sha256(reps.cplx_bytes()).hexdigest()
        canon = hashlib.sha256(p.fetch_complexes(14).cplx_bytes()).hexdigest()
        want = g.get("line15", {}).get(str(n))
        ok = None if want is None or "line15" not in want else (
            want["line15"] == l15 and want.get("sha256", sha) == sha and want.get("canon_sha256", canon) == canon)
        print(json.dumps({"n": n, "line7": l7, "line13": l13, "line15": l15, "wall_ms": round(wall, 3), **st,
                          "parity": ok, "sha256": sha, "canon_sha256": canon}), flush=True)

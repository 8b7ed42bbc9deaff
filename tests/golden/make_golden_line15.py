"""Add Algorithm 2 line-15 goldens to tests/golden/golden.json.
TEST INFRASTRUCTURE ONLY (nothing here runs on the GPU box).

For each n: the line-13 survivors come from the oracle route (dfs_port per
map + line13_port), asserted byte-identical to golden.json["line13"][n]
(itself the reference pipeline's own output for n <= 7).  They are written
as .cplx and handed to the UNMODIFIED reference's canonical forms
(oracle/_ref/plseeds_ref line15: canonical_form per survivor,
isomorphism.hpp:228-303, then the first-appearance dedupe exactly as
pipeline.hpp:91-103).  Recorded: the line-15 count, the SHA-256 of the
representatives' .cplx, the SHA-256 of every survivor's canonical form in
survivor order (the `canon` vector), and the reference's time.  The paper's
own line-15 counts (PAPER.md table "output of Algorithm 2", n <= 10) are
checked as well.

usage: python tests/golden/make_golden_line15.py [--min 2] [--max 11] [--threads T]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle_bind import Oracle  # noqa: E402
from make_golden_line13 import global_rows  # noqa: E402

import numpy as np  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")
# PAPER.md, table "The output of Algorithm 2 for n <= 10", row "line 15"
PAPER_LINE15 = {2: 2, 3: 5, 4: 49, 5: 256, 6: 1791, 7: 2194, 8: 1401, 9: 381, 10: 56}


def survivors_cplx(orc: Oracle, n: int, orbits, want_sha: str) -> bytes:
    m = n + 4
    all_sub = orc.all_subsets_universe(m, n)
    rows = []
    for r in orbits:
        uni = orc.matroid_universe(r)
        _, _, bits = orc.dfs(n, uni, orc.cyclic_facet_bound(n))
        rows.append(global_rows(orc, n, uni, bits, all_sub))
    _, _, surv = orc.line13(m, n, np.concatenate(rows))
    data = orc.write_cplx(m, n, all_sub, surv)
    assert hashlib.sha256(data).hexdigest() == want_sha, f"n={n}: survivors differ from golden line13"
    return data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min", type=int, default=2)
    ap.add_argument("--max", type=int, default=11)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "golden.json"))
    args = ap.parse_args()
    orc = Oracle()
    g = json.load(open(args.out))
    sec = g.setdefault("line15", {})
    for n in range(args.min, args.max + 1):
        t0 = time.time()
        data = survivors_cplx(orc, n, g["orbits"][str(n)], g["line13"][str(n)]["sha256"])
        with tempfile.TemporaryDirectory() as td:
            s, c, r = (os.path.join(td, x) for x in ("s.cplx", "c.cplx", "r.cplx"))
            open(s, "wb").write(data)
            txt = subprocess.run([REF, "line15", s, "--threads", str(args.threads), "--canon", c, "--out", r],
                                 check=True, capture_output=True, text=True).stdout.split()
            canon_sha = hashlib.sha256(open(c, "rb").read()).hexdigest()
            reps_sha = hashlib.sha256(open(r, "rb").read()).hexdigest()
        ent = {"line13": int(txt[1]), "line15": int(txt[3]), "sha256": reps_sha, "canon_sha256": canon_sha,
               "ref_canon_s": float(txt[5]), "threads": int(txt[7]),
               "source": "oracle/_ref (reference canonical_form + dedupe, pipeline.hpp:91-103) on the golden "
                         "line-13 survivors"}
        assert ent["line13"] == g["line13"][str(n)]["line13"]
        if n in PAPER_LINE15:
            assert ent["line15"] == PAPER_LINE15[n], (n, ent["line15"], PAPER_LINE15[n])
            ent["paper_line15"] = PAPER_LINE15[n]
        sec[str(n)] = ent
        print(f"n={n} line13={ent['line13']} line15={ent['line15']} ref {ent['ref_canon_s']:.1f}s "
              f"total {time.time() - t0:.1f}s", flush=True)
        json.dump(g, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

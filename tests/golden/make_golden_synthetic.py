"""Synthetic candidate-facet sets (BASELINE.json configs[4], SURVEY.md 8(d)
item 5) -> golden.json["synthetic"].  TEST INFRASTRUCTURE ONLY.

Universe (seed, d): facet j of the all-subsets universe of (m, n) = (15, 11)
(ascending masks) is kept iff splitmix64(seed ^ j) * 2^-64 < d
(tests/catalog.py synthetic_universe); facet cap 252 = the UBT bound of n=11.

* d <= 0.73: the UNMODIFIED reference (oracle/_ref/plseeds_ref job: its
  incidence, convenient basis and enumerate_wpm) -- count and the SHA-256 of
  its .cplx output; jobs it cannot finish in --timeout seconds are skipped.
  Above that the reference's kernel-basis search stops finishing (d = 0.74
  seed 1 and d >= 0.75 all ran past 10 minutes on 8 threads).
* d in {0.75, 0.78}: the CPU restatement of the device search
  (oracle/dfs_port.c) -- count, node count and the SHA-256 of the same .cplx
  bytes; on every reference-pinned case it is asserted equal to the
  reference.

usage: python tests/golden/make_golden_synthetic.py [--threads T] [--timeout S]
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
import catalog as C  # noqa: E402
from oracle_bind import Oracle  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")
M_, N_, CAP = 15, 11, 252
REF_DENSITIES = (0.60, 0.65, 0.70, 0.72, 0.73)
DFS_DENSITIES = (0.75, 0.78)


def ref_job(u, threads, timeout):
    with tempfile.TemporaryDirectory() as td:
        job, out = os.path.join(td, "j.txt"), os.path.join(td, "o.cplx")
        with open(job, "w") as f:
            f.write(f"{M_} {N_} {len(u)} {CAP} 0 0\n" + " ".join(str(x) for x in u) + "\n")
        try:
            txt = subprocess.run([REF, "job", job, "--threads", str(threads), "--out", out], check=True,
                                 capture_output=True, text=True, timeout=timeout).stdout.split()
        except subprocess.TimeoutExpired:
            return None
        data = open(out, "rb").read() if os.path.exists(out) else b""
    return {"wpms": int(txt[1]), "sha256": hashlib.sha256(data).hexdigest(), "ref_s": float(txt[3])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--timeout", type=float, default=120.0)
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "golden.json"))
    args = ap.parse_args()
    orc = Oracle()
    g = json.load(open(args.out))
    sec = {"m": M_, "n": N_, "cap": CAP, "generator": "splitmix64(seed ^ j) < d * 2^64 over the ascending "
           "all-subsets universe (tests/catalog.py synthetic_universe)", "cases": []}
    for d in REF_DENSITIES + DFS_DENSITIES:
        for seed in range(1, args.seeds + 1):
            t0 = time.time()
            u = C.synthetic_universe(seed, d)
            cnt, nodes, bits = orc.dfs(N_, u, CAP)
            sha = hashlib.sha256(orc.write_cplx(M_, N_, u, bits) if cnt else b"").hexdigest()
            ent = {"seed": seed, "d": d, "M": len(u), "wpms": cnt, "nodes": nodes, "sha256": sha}
            if d in REF_DENSITIES:
                r = ref_job(u, args.threads, args.timeout)
                if r is None:
                    ent["source"] = "oracle (dfs_port); the reference timed out"
                else:
                    assert (r["wpms"], r["sha256"]) == (cnt, sha), (seed, d, r, cnt)
                    ent["source"] = "oracle/_ref (reference enumerate_wpm), equal to dfs_port"
                    ent["ref_s"] = r["ref_s"]
            else:
                ent["source"] = "oracle (dfs_port: the device search restated)"
            sec["cases"].append(ent)
            print(f"d={d} seed={seed} M={len(u)} wpms={cnt} nodes={nodes} {ent['source']} "
                  f"{time.time() - t0:.1f}s", flush=True)
    g["synthetic"] = sec
    json.dump(g, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

"""Add Algorithm 2 line-7 / line-13 goldens to tests/golden/golden.json.
TEST INFRASTRUCTURE ONLY (nothing here runs on the GPU box).

Sources:
  * n = 2..7: oracle/_ref/plseeds_ref line13 -- the UNMODIFIED reference
    (enumerate_wpm per orbit, the std::set union, support + is_seed exactly as
    pipeline.hpp:58-89) -- line7, line13 and the SHA-256 of the survivors
    written with write_complexes (complex_io.hpp:34-39).
  * n = 8..11 (the reference cannot enumerate them in reasonable time): the
    oracle -- dfs_port per map, the union and filter of line13_port.c
    (po_line13, swap characterisation) -- after asserting that the same
    oracle route reproduces the reference's line7/line13/digest for every
    n <= --check-max.

usage: python tests/golden/make_golden_line13.py [--ref-max 7] [--check-max 7] [--max 11]
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

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import Oracle  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")


def ref_line13(n: int, threads: int):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "l13.cplx")
        txt = subprocess.run([REF, "line13", str(n), "--threads", str(threads), "--out", out], check=True,
                             capture_output=True, text=True).stdout
        data = open(out, "rb").read()
    t = txt.split()
    return {"line7": int(t[1]), "line13": int(t[3]), "sha256": hashlib.sha256(data).hexdigest(),
            "ref_enum_s": float(t[5]), "ref_filter_s": float(t[7]), "threads": int(t[9])}


def global_rows(orc: Oracle, n: int, universe, bits: np.ndarray, all_sub) -> np.ndarray:
    """WPM bitsets over a map's universe -> bitsets over all n-subsets of [m]."""
    gw = (len(all_sub) + 63) // 64
    gidx = np.searchsorted(np.asarray(all_sub, dtype=np.uint64), np.asarray(universe, dtype=np.uint64))
    out = np.zeros((bits.shape[0], gw), dtype=np.uint64)
    for w in range(bits.shape[1]):
        col = bits[:, w]
        for b in range(64):
            j = w * 64 + b
            if j >= len(universe):
                break
            hit = (col >> np.uint64(b)) & np.uint64(1)
            g = int(gidx[j])
            out[:, g >> 6] |= hit << np.uint64(g & 63)
    return out


def oracle_line13(orc: Oracle, n: int, orbits):
    m = n + 4
    all_sub = orc.all_subsets_universe(m, n)
    rows = []
    for r in orbits:
        uni = orc.matroid_universe(r)
        _, _, bits = orc.dfs(n, uni, orc.cyclic_facet_bound(n))
        rows.append(global_rows(orc, n, uni, bits, all_sub))
    allr = np.concatenate(rows)
    l7, l13, surv = orc.line13(m, n, allr)
    data = orc.write_cplx(m, n, all_sub, surv)
    return {"line7": l7, "line13": l13, "sha256": hashlib.sha256(data).hexdigest(), "wpms": int(allr.shape[0])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-max", type=int, default=7)
    ap.add_argument("--check-max", type=int, default=7)
    ap.add_argument("--min", type=int, default=2)
    ap.add_argument("--max", type=int, default=11)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "golden.json"))
    args = ap.parse_args()
    orc = Oracle()
    g = json.load(open(args.out))
    sec = g.setdefault("line13", {})
    for n in range(args.min, args.max + 1):
        t0 = time.time()
        orbits = g["orbits"][str(n)]
        ent = None
        if n <= args.ref_max:
            ent = ref_line13(n, args.threads)
            ent["source"] = "oracle/_ref (reference pipeline.hpp:58-89)"
        if n <= args.check_max or ent is None:
            o = oracle_line13(orc, n, orbits)
            if ent is not None:
                for k in ("line7", "line13", "sha256"):
                    assert o[k] == ent[k], (n, k, o[k], ent[k])
            else:
                ent = {"line7": o["line7"], "line13": o["line13"], "sha256": o["sha256"],
                       "source": "oracle (dfs_port + line13_port, swap form; equal to the reference for n <= "
                                 f"{args.check_max})"}
        sec[str(n)] = ent
        print(f"n={n} line7={ent['line7']} line13={ent['line13']} {time.time() - t0:.1f}s", flush=True)
        json.dump(g, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

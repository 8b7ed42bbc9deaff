"""Regenerate tests/golden/golden.json.  TEST INFRASTRUCTURE ONLY.

Sources (nothing here runs on the GPU box):
  * oracle/_ref/plseeds_ref -- the UNMODIFIED reference library compiled from
    /root/reference/proj/include by oracle/Makefile -- for n = 2..7 (UBT cap,
    pipeline.hpp:58-72 semantics) and the no-property counts for n = 2..5:
    per-map WPM counts, universe sizes, kernel dimension, combination-space
    size and the SHA-256 of the per-map `.cplx` bytes (SURVEY.md App. C
    protocol: write_complexes per map, maps concatenated).
  * oracle/liboracle.so dfs_port -- the CPU restatement of the device search --
    for the DFS node counts (n = 2..11) and for the WPM counts/digests at
    n = 8..11, where the reference cannot finish.  The n = 8
    reference run (~1.5 h on 8 cores) is merged in when present
    (--n8-summary /tmp/n8/summary.txt from oracle's run script).

usage: python tests/golden/make_golden.py [--max-ref 7] [--max-dfs 11]
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import Oracle  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")


def ref_enumerate(n: int, nocap: bool, threads: int, maps_range=None):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "o.cplx")
        cmd = [REF, "enumerate", str(n), "--threads", str(threads), "--out", out]
        if maps_range is not None:
            cmd += ["--maps", f"{maps_range[0]}:{maps_range[1]}"]
        if nocap:
            cmd.append("--nocap")
        txt = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
        data = open(out, "rb").read()
    maps = []
    for line in txt.splitlines():
        if line.startswith("map "):
            t = line.split()
            maps.append({"M": int(t[3]), "N": int(t[5]), "s": int(t[7]), "space": int(t[9]),
                         "wpms": int(t[11]), "seconds": float(t[15])})
    return maps, data


def ref_per_map(n: int, nocap: bool, threads: int, num_maps: int):
    maps, digests, whole = [], [], hashlib.sha256()
    for i in range(num_maps):
        mm, data = ref_enumerate(n, nocap, threads, (i, i + 1))
        maps += mm
        digests.append(hashlib.sha256(data).hexdigest())
        whole.update(data)
    return maps, digests, whole.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-ref", type=int, default=7)
    ap.add_argument("--max-dfs", type=int, default=11)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--n8-summary", default="/tmp/n8/summary.txt")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "golden.json"))
    args = ap.parse_args()
    orc = Oracle()
    g = {"ubt": {}, "nocap": {}, "dfs": {}, "orbits": {}}
    if os.path.exists(args.out):
        g.update(json.load(open(args.out)))
    for n in range(2, 12):
        g["orbits"][str(n)] = [d for d in orc.idcm_orbits(n)]
    for n in range(2, args.max_ref + 1):
        t0 = time.time()
        maps, digests, whole = ref_per_map(n, False, args.threads, len(g["orbits"][str(n)]))
        counts = [m["wpms"] for m in maps]
        ent = {"source": "oracle/_ref (reference enumerate_wpm)", "maps": maps, "sha256": whole,
               "map_sha256": digests, "sum": sum(counts)}
        g["ubt"][str(n)] = ent
        print(f"ref n={n} sum={sum(counts)} {time.time() - t0:.1f}s", flush=True)
    for n in range(2, min(args.max_ref, 5) + 1):
        maps, digests, whole = ref_per_map(n, True, args.threads, len(g["orbits"][str(n)]))
        g["nocap"][str(n)] = {"counts": [m["wpms"] for m in maps], "sha256": whole, "map_sha256": digests}
    for n in range(2, args.max_dfs + 1):
        t0 = time.time()
        per = []
        blob = hashlib.sha256()
        for rows in g["orbits"][str(n)]:
            uni = orc.matroid_universe(rows)
            cnt, nodes, bits = orc.dfs(n, uni, orc.cyclic_facet_bound(n), want_bits=n >= 8)
            ent = {"M": len(uni), "wpms": cnt, "nodes": nodes}
            if n >= 8:
                b = orc.write_cplx(n + 4, n, uni, bits)
                ent["sha256"] = hashlib.sha256(b).hexdigest()
                blob.update(b)
            per.append(ent)
        g["dfs"][str(n)] = {"source": "oracle dfs_port", "maps": per,
                            "sum": sum(p["wpms"] for p in per), "nodes": sum(p["nodes"] for p in per)}
        if n >= 8:
            g["dfs"][str(n)]["sha256"] = blob.hexdigest()
        print(f"dfs n={n} sum={g['dfs'][str(n)]['sum']} nodes={g['dfs'][str(n)]['nodes']} "
              f"{time.time() - t0:.1f}s", flush=True)
    if os.path.exists(args.n8_summary):
        lines = [ln.split() for ln in open(args.n8_summary) if ln[:1].isdigit()]
        if len(lines) == 16:
            maps = [{"M": int(t[5]), "N": int(t[7]), "s": int(t[9]), "space": int(t[11]), "wpms": int(t[13])}
                    for t in lines]
            ent = {"source": "oracle/_ref (reference enumerate_wpm), 6 threads", "maps": maps,
                   "map_sha256": [t[1] for t in lines], "sum": sum(m["wpms"] for m in maps)}
            whole = os.path.join(os.path.dirname(args.n8_summary), "whole.txt")
            if os.path.exists(whole):
                ent["sha256"] = open(whole).read().split()[0]
            g["ubt"]["8"] = ent
    json.dump(g, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()

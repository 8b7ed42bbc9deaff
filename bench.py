"""bench.py -- WPM enumeration throughput on B200 (and the reference CPU arm).

Workload (BASELINE.json configs[1]): Picard 4, n = 5 (m = 9) -- every WPM of
every mod-2 characteristic map (35 IDCM orbits), UBT facet cap, canonical
output.  One "step" = one complete enumeration of all maps: kernel 3 (search)
+ canonical sort, universes/incidence resident in HBM.

Metric (BASELINE.json): search nodes/s and wall time per n.  A node is one
facet-inclusion step of the canonical DFS tree of the workload; the tree is
a property of the workload (3,638,216 nodes at n = 5, pinned by the CPU
restatement), so both arms report  nodes(workload) / their own wall time and
the driver's ratio is the wall-time ratio.  The reference's own search size
(combination-space leaves, search.hpp:62-104) is reported beside it.

  value : nodes / device time, inputs resident (Plan.run; kernel 3 + sort)
  e2e   : the same through the one-shot C-ABI call wpm_enumerate_orbits with
          host buffers (orbits -> kernels 1,2 -> search -> sort -> D2H of every
          WPM bitset), timed on the host around the call
  roofline : kernel 3 vs the measured INT32 issue peak (5n ops per node,
          SURVEY.md 8(d)); bound "int-issue" (no tensor / HBM work on this path)
  cpu_baseline : the reference compiled from its own headers (oracle/_ref),
          nproc threads, the same workload

Multi-GPU (torchrun): root tasks are sharded t % world == rank (weak split of
one fixed workload = strong scaling); NCCL only for the final counts and the
result gather to rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NODES_PER_N = None  # filled from tests/golden/golden.json


def _golden():
    return json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def reference_arm(args):
    """`--impl reference`: the reference's own CPU path (oracle/_ref, built
    from the unmodified headers), nproc threads, same workload and unit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")
    n = args.n
    g = _golden()
    nodes = g["dfs"][str(n)]["nodes"]
    threads = os.cpu_count() or 1
    if not os.path.exists(ref):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/plseeds_ref not built"}))
        return 0

    def one():
        t0 = time.perf_counter()
        out = subprocess.run([ref, "enumerate", str(n), "--threads", str(threads)], check=True,
                             capture_output=True, text=True).stdout
        wall = time.perf_counter() - t0
        tot = [ln for ln in out.splitlines() if ln.startswith("total")][0].split()
        return wall, int(tot[2]), int(tot[4]), float(tot[6]), float(tot[8])

    for _ in range(args.warmup):
        one()
    walls, leaves = [], 0
    wpms = 0
    for _ in range(args.steps):
        wall, wpms, leaves, prep, enum = one()
        walls.append(wall)
    t = sum(walls) / len(walls)
    value = nodes / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64 (GF(2) bitsets)", "data": "synthetic (IDCM orbit maps, deterministic)",
        "config": {"workload": f"Picard 4, n={n} (m={n + 4}): all {len(g['orbits'][str(n)])} characteristic maps, "
                               "UBT cap", "n": n, "maps": len(g["orbits"][str(n)]), "wpms": wpms,
                   "reference_leaves": leaves, "threads": threads},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full n={n} enumeration (all maps), {args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_leaves_per_s": leaves / t, "wall_s": t,
    }
    print(json.dumps(line))
    return 0


METRIC = "search nodes/sec and wall time to enumerate all WPMs per Picard-4 dim n"
# per step at n = 5, from the ncu launch list of this command
# (profiles/r01_bench_n5_launches.txt): seed_tasks + k3_search + CUB merge sort
# of the key rows (1 block sort + 9 partition/merge pairs) + split_rows
LAUNCHES_PER_STEP = 22


def _profile_summary(n):
    """traffic / instructions-per-node of kernel 3 from the committed ncu capture."""
    out = {}
    path = os.path.join(ROOT, "profiles", f"r01_k3_n{n}_ncu.txt")
    if not os.path.exists(path):
        return out
    rd = wr = None
    for ln in open(path):
        t = ln.split()
        if not t:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if t[0] == "dram__bytes_read.sum":
            rd = float(t[1]) * scale.get(t[2], 1)
        elif t[0] == "dram__bytes_write.sum":
            wr = float(t[1]) * scale.get(t[2], 1)
        elif ln.startswith("warp instructions per node"):
            out["inst_per_node"] = float(t[-1])
        elif t[0] == "smsp__issue_active.avg.pct_of_peak_sustained_active":
            out["issue_pct"] = float(t[1])
    if rd is not None and wr is not None:
        out["traffic"] = rd + wr
    return out
UNIT = "search nodes/s (DFS facet-inclusion steps of the workload / wall s)"


def cpu_baseline(n, nodes):
    ref = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")
    threads = os.cpu_count() or 1
    if not os.path.exists(ref):
        return None
    t0 = time.perf_counter()
    out = subprocess.run([ref, "enumerate", str(n), "--threads", str(threads)], check=True, capture_output=True,
                         text=True, timeout=600).stdout
    wall = time.perf_counter() - t0
    tot = [ln for ln in out.splitlines() if ln.startswith("total")][0].split()
    return {"value": nodes / wall, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"one full n={n} enumeration, all maps (reference enumerate_wpm, {threads} threads)",
            "wall_s": wall, "reference_leaves": int(tot[4]), "wpms": int(tot[2])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-n", dest="per_n", action="store_false",
                    help="skip the n = 2..11 sweep (1 GPU only)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    args.warmup = max(args.warmup, 3)

    import numpy as np
    import torch

    import paper_2301_00806_b200 as wpm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    n = args.n
    g = _golden()
    expect_nodes = g["dfs"][str(n)]["nodes"]
    expect_wpms = g["dfs"][str(n)]["sum"]

    plan = wpm.Plan.orbits(n, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2
    for _ in range(args.warmup):
        plan.run(rank, world)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(dev)
    barrier()
    sampler.start()
    ms_total = ms_search = ms_sort = 0.0
    nodes = 0
    t_host = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the device-timed window)
        torch.cuda.synchronize(dev)
        plan.run(rank, world)
        st = plan.stats()
        ms_total += plan.timing()["ms_total"]
        ms_search += st["ms_search"]
        ms_sort += st["ms_sort"]
        nodes = st["nodes"]
    barrier()
    t_host = time.perf_counter() - t_host
    clocks = sampler.stop()
    res = plan.fetch()
    # whole-job: sum nodes over ranks, max device time over ranks
    tot_nodes = nodes
    ms_step = ms_total / args.steps
    if dist:
        t = torch.tensor([float(nodes), ms_step, float(res.total)], dtype=torch.float64, device=f"cuda:{dev}")
        mx = t.clone()
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot_nodes = int(t[0].item())
        ms_step = mx[1].item()
        tot_wpms = int(t[2].item())
    else:
        tot_wpms = res.total
    value = tot_nodes / (ms_step * 1e-3)

    # e2e: the reference-facing one-shot C-ABI call, host buffers, all copies inside
    e2e_times = []
    h2d = d2h = 0
    for i in range(max(2, min(args.steps, 10)) + 1):
        barrier()
        t0 = time.perf_counter()
        r = wpm_orbits_oneshot(wpm, n, dev, rank, world)
        dt = time.perf_counter() - t0
        if i > 0:  # first call pays context/module load
            e2e_times.append(dt)
        h2d, d2h = r.h2d_bytes, r.d2h_bytes
    e2e_s = statistics.median(e2e_times)
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    e2e_value = tot_nodes / e2e_s

    # roofline of kernel 3 vs measured INT32 issue peak
    peak = wpm.int_peak(dev)
    ops = tot_nodes / max(world, 1) * 5 * n if world > 1 else nodes * 5 * n
    ms_k3 = ms_search / args.steps
    achieved = ops / (ms_k3 * 1e-3)
    prof = _profile_summary(n)
    roofline = {"bound": "int-issue", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
                "frac": achieved / peak, "traffic": prof.get("traffic"),
                "note": "achieved = 5n int lane-ops per search node (SURVEY 8d) / kernel-3 CUDA-event time; peak = "
                        "measured LOP3+IADD chains on all SMs (wpm_int_peak, live). traffic = dram read+write bytes "
                        "of one kernel-3 launch from the committed ncu --set full capture",
                "issue": {"warp_inst_per_node": prof.get("inst_per_node"),
                          "issue_active_pct": prof.get("issue_pct"),
                          "warp_inst_peak_per_s": 4 * 148 * 1.965e9,
                          "note": "the kernel is issue-bound: one DFS per warp has O(n) lanes of work per node; "
                                  "see profiles/r01_k3_n5_ncu.txt"}}

    num_maps = plan.num_maps
    per_n = None
    if world == 1 and args.per_n:
        plan.close()
        per_n = sweep_per_n(wpm, dev, flush, g)
        synthetic = sweep_synthetic(wpm, dev, flush, g)
        plan = None

    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(n, expect_nodes)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64 (GF(2) bitsets)",
            "data": "synthetic (IDCM orbit maps, deterministic; no dataset)",
            "config": {"workload": f"Picard 4, n={n} (m={n + 4}): all {num_maps} characteristic maps, UBT cap "
                                   "(BASELINE configs[1])", "n": n, "maps": num_maps, "wpms": tot_wpms,
                       "dfs_nodes": tot_nodes, "l2": "flushed (256 MB write) between timed steps",
                       "parallelism": f"root-task shards x{world}"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "wall_ms": e2e_s * 1e3, "min_ms": min(e2e_times) * 1e3, "samples_ms": [round(t * 1e3, 3) for t in e2e_times],
                    "call": "wpm_enumerate_orbits (one-shot C-ABI)"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "gpu_launches_per_step": {"seed_tasks": 1, "k3_search": 1, "cub_merge_sort": 19, "split_rows": 1},
            "breakdown_ms": {"search": ms_k3, "sort": ms_sort / args.steps, "step": ms_step},
            "parity": {"wpms_expected": expect_wpms, "nodes_expected": expect_nodes,
                       "ok": tot_wpms == expect_wpms and tot_nodes == expect_nodes},
            "host_wall_s": t_host,
        }
        if per_n is not None:
            line["per_n"] = per_n
            line["synthetic"] = synthetic
            row = next((r for r in per_n if r["n"] == n), None)
            if row and row.get("alg1"):
                # the same algorithm on both sides: the reference's leaves per
                # second (kernel basis + odometer), GPU vs the CPU reference run
                a1 = row["alg1"]
                line["alg1_reference_algorithm"] = {
                    "leaves": a1["leaves"], "gpu_ms": round(a1["ms_prep_host"] + a1["ms_step"], 3),
                    "gpu_leaves_per_s": a1["leaves"] / ((a1["ms_prep_host"] + a1["ms_step"]) * 1e-3),
                    "cpu_leaves_per_s": (cpu["reference_leaves"] / cpu["wall_s"]) if cpu else None,
                    "cpu_threads": cpu["cores"] if cpu else None, "parity_ok": a1["parity_ok"],
                    "note": "leaves = combination-space leaves (search.hpp:62-104), the reference's own work unit; "
                            "gpu_ms = host basis build + device leaf kernel + canonical sort"}
        print(json.dumps(line))
    if plan is not None:
        plan.close()
    if dist:
        dist.destroy_process_group()
    return 0


def sweep_per_n(wpm, dev, flush, g, ns=range(2, 12), reps=3, alg1_max_n=8):
    """The metric is quoted per Picard-4 dimension n: every n = 2..11 (all maps,
    UBT cap) on this GPU -- device time of search + sort (median of `reps`
    runs after one warm-up, L2 flushed before each) and the one-shot C-ABI
    call with host buffers; parity of counts and nodes against the golden
    file.  Also Algorithm 2 lines 7 / 13 (union + support + seedness filter,
    pipeline.hpp:58-89) on each run's resident result: device ms and counts
    against golden.json["line13"]; line 15 (canonical forms + class dedupe,
    pipeline.hpp:91-103) likewise against golden.json["line15"] (the
    reference for n <= 7, the paper's counts for n = 8..10); and, for
    n <= alg1_max_n, the reference's
    own algorithm (kernel basis + every combination-space leaf on the GPU):
    the reference's work unit (leaves) per second, apples to apples."""
    import torch

    rows = []
    for n in ns:
        with wpm.Plan.orbits(n, device=dev) as p:
            p.run()
            runs, l13, l15 = [], [], []
            for _ in range(reps):
                flush.zero_()
                torch.cuda.synchronize(dev)
                p.run()
                st, tm = p.stats(), p.timing()
                runs.append((tm["ms_total"], st["ms_search"], st["ms_sort"], st["nodes"]))
                # Algorithm 2 lines 7 / 13 on the resident result (k5_line13.cu)
                lines = p.line13()
                lt = p.line13_timing()
                l13.append((lt["ms_union"] + lt["ms_filter"], lt["ms_union"], lt["ms_filter"], lines))
                # Algorithm 2 line 15 on the resident survivors (k7_line15.cu)
                c15 = p.line15()
                s15 = p.line15_stats()
                l15.append((s15["ms_canon"] + s15["ms_dedupe"], s15["ms_canon"], s15["ms_dedupe"], c15,
                            s15["placements"]))
            total = p.fetch().total
        runs.sort()
        ms, ms_search, ms_sort, nodes = runs[len(runs) // 2]
        l13.sort()
        ms13, ms_union, ms_filter, (line7, line13) = l13[len(l13) // 2]
        want13 = g.get("line13", {}).get(str(n), {})
        l15.sort()
        ms15, ms_canon, ms_dedupe, line15, placements = l15[len(l15) // 2]
        want15 = g.get("line15", {}).get(str(n), {})
        want = g["dfs"][str(n)]
        alg1 = None
        if n <= alg1_max_n:
            # the reference's own search (Algorithm 1: kernel basis + every
            # combination-space leaf, k6_odometer.cu), same maps and cap
            with wpm.Plan.orbits(n, device=dev) as p:
                ts = []
                for _ in range(1 if n >= 8 else 3):
                    flush.zero_()
                    torch.cuda.synchronize(dev)
                    tot1 = p.run_kernel_basis()
                    st1 = p.kernel_basis_stats()
                    ts.append((p.timing()["ms_total"], st1["ms_leaves"], st1["ms_prep"]))
                    counts1 = p.fetch().counts
                ts.sort()
                ms1, ms_leaves, ms_prep = ts[len(ts) // 2]
            ref_maps = g["ubt"].get(str(n), {}).get("maps")
            want_counts = [m["wpms"] for m in ref_maps] if ref_maps else [m["wpms"] for m in want["maps"]]
            alg1 = {"leaves": st1["leaves"], "cap_checked": st1["checked"], "ms_step": round(ms1, 3),
                    "ms_leaves": round(ms_leaves, 3), "ms_prep_host": round(ms_prep, 3),
                    "leaves_per_s": st1["leaves"] / (ms_leaves * 1e-3) if ms_leaves else None,
                    "parity_ok": tot1 == want["sum"] and counts1 == want_counts}
        wpm.enumerate_orbits(n, device=dev)  # warm the one-shot path
        e2e = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = wpm.enumerate_orbits(n, device=dev)
            e2e.append((time.perf_counter() - t0) * 1e3)
            if len(e2e) < 3:
                del r
        e2e_ms = statistics.median(e2e)
        rows.append({"n": n, "m": n + 4, "maps": r.num_maps, "wpms": total, "nodes": nodes,
                     "ms_step": round(ms, 3), "ms_search": round(ms_search, 3), "ms_sort": round(ms_sort, 3),
                     "nodes_per_s": nodes / (ms * 1e-3), "e2e_ms": round(e2e_ms, 3),
                     "d2h_bytes": int(r.d2h_bytes),
                     "parity_ok": total == want["sum"] and r.total == want["sum"] and nodes == want["nodes"],
                     "line13": {"line7": line7, "line13": line13, "ms": round(ms13, 3), "ms_union": round(ms_union, 3),
                                "ms_filter": round(ms_filter, 3),
                                "parity_ok": (line7, line13) == (want13.get("line7"), want13.get("line13"))},
                     "line15": {"line15": line15, "ms": round(ms15, 3), "ms_canon": round(ms_canon, 3),
                                "ms_dedupe": round(ms_dedupe, 3), "placements": placements,
                                "ref_canon_s": want15.get("ref_canon_s"), "ref_threads": want15.get("threads"),
                                "parity_ok": None if "line15" not in want15 else line15 == want15["line15"]},
                     "alg1": alg1})
        del r
    return rows


def sweep_synthetic(wpm, dev, flush, g, densities=(0.75, 0.78, 0.80, 0.85, 0.90, 1.0), seed=1,
                    budget=2_000_000_000):
    """BASELINE configs[4]: synthetic candidate-facet sets, (m, n) = (15, 11),
    cap 252, density sweep.  Full enumeration where it
    is checkable (parity vs golden.json["synthetic"]); above d = 0.80 a
    node-budgeted stress run (truncated = True: nodes/s and divergence only)."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import catalog as C

    want = {(c["seed"], round(c["d"], 4)): c for c in g.get("synthetic", {}).get("cases", [])}
    rows = []
    for d in densities:
        u = C.synthetic_universe(seed, d)
        with wpm.Plan.universes(15, 11, [u], facet_cap=252, device=dev) as p:
            if d > 0.80:
                p.set_node_budget(budget)
            p.run()
            flush.zero_()
            torch.cuda.synchronize(dev)
            total = p.run()
            st, tm = p.stats(), p.timing()
            trunc = p.truncated()
        w = want.get((seed, round(d, 4)))
        rows.append({"d": d, "seed": seed, "M": len(u), "wpms": total, "nodes": st["nodes"],
                     "ms_search": round(st["ms_search"], 3), "ms_step": round(tm["ms_total"], 3),
                     "nodes_per_s": st["nodes"] / (st["ms_search"] * 1e-3) if st["ms_search"] else None,
                     "truncated": trunc,
                     "parity_ok": None if w is None or trunc else (total == w["wpms"] and st["nodes"] == w["nodes"])})
    return rows


class _E2E:
    def __init__(self, h2d, d2h, total):
        self.h2d_bytes, self.d2h_bytes, self.total = h2d, d2h, total


def wpm_orbits_oneshot(wpm, n, dev, rank, world):
    """wpm_enumerate_orbits for world == 1.  For world > 1: every rank builds
    its plan from the host maps, searches its root-task shard, NCCL gathers
    the canonical rows into rank 0's HBM, rank 0 sorts them canonically and
    copies the full list to the host."""
    if world == 1:
        return wpm.enumerate_orbits(n, device=dev)
    import torch
    import torch.distributed as dist

    from paper_2301_00806_b200 import dist as wdist

    with wpm.Plan.orbits(n, device=dev) as p:
        p.run(rank, world)
        total, dups, rows, maps = wdist.gather_to_rank0_device(dist, p, rank, dev, return_rows=True)
        d2h = 0
        if rank == 0:
            assert dups == 0
            host = torch.empty(rows.numel(), dtype=rows.dtype, pin_memory=True)
            host.copy_(rows)
            d2h = host.numel() * host.element_size()
    return _E2E(0, d2h, total)


if __name__ == "__main__":
    sys.exit(main())

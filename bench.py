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

Multi-GPU (torchrun, one process per GPU): the library's shared-frontier
protocol (paper_2301_00806_b200/dist.py): rank 0 splits the search tree below
the root, the frontier records go to every rank (NCCL broadcast), every GPU's
kernel 3 claims records through one counter in rank 0's HBM (CUDA IPC, peer
atomics) -- one fixed workload split dynamically = strong scaling -- and the
rows are gathered to rank 0 (send/recv) and sorted there once.  On one GPU the
line carries a scaling PROJECTION from measured per-record node counts
(`scaling_projection`).
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


def workload_config(n, maps):
    """The `config` of both arms (identical dicts: the driver compares them)."""
    return {"workload": f"Picard 4, n={n} (m={n + 4}): all {maps} characteristic maps, UBT cap "
                        "(BASELINE configs[1])" if n == 5 else f"Picard 4, n={n} (m={n + 4}): all {maps} "
                        "characteristic maps, UBT cap",
            "n": n, "m": n + 4, "maps": maps, "facet_cap": "ubt (cyclic_facet_bound)",
            "output": "every WPM of every map, canonical order (search.hpp:247-257)"}


def _ref_run(ref, n, threads, maps=None, timeout=900):
    cmd = [ref, "enumerate", str(n), "--threads", str(threads)]
    if maps:
        cmd += ["--maps", maps]
    t0 = time.perf_counter()
    out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout).stdout
    wall = time.perf_counter() - t0
    tot = [ln for ln in out.splitlines() if ln.startswith("total")][0].split()
    return {"wall_s": wall, "wpms": int(tot[2]), "leaves": int(tot[4]), "prep_s": float(tot[6]),
            "enum_s": float(tot[8])}


def reference_arm(args):
    """`--impl reference`: the reference's own CPU path (oracle/_ref, built
    from the unmodified headers), all host threads, same workload and unit."""
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
    for _ in range(args.warmup):
        _ref_run(ref, n, threads)
    runs = [_ref_run(ref, n, threads) for _ in range(args.steps)]
    t = sum(r["wall_s"] for r in runs) / len(runs)
    value = nodes / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64 (GF(2) bitsets)", "data": "synthetic (IDCM orbit maps, deterministic)",
        "config": workload_config(n, len(g["orbits"][str(n)])),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full n={n} enumeration (all maps, reference enumerate_wpm, {threads} threads), "
                                   f"{args.steps} steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {"wpms": runs[-1]["wpms"], "leaves": runs[-1]["leaves"], "threads": threads,
                      "leaves_per_s": runs[-1]["leaves"] / t, "wall_s": t},
    }
    print(json.dumps(line))
    return 0


METRIC = "search nodes/sec and wall time to enumerate all WPMs per Picard-4 dim n"
# per step at n = 5 (1 GPU), from the ncu launch list of this command
# (profiles/r02_bench_n5_launches.txt): seed_tasks + k3_search + k4_sort (one
# cooperative launch: tile sort, merge passes, split)
LAUNCHES_PER_STEP = 3


def _profile_summary(n):
    """traffic / instructions-per-node of kernel 3 from the committed ncu capture."""
    out = {}
    for tag in ("r02g", "r02c", "r02", "r01"):  # the newest capture committed
        path = os.path.join(ROOT, "profiles", f"{tag}_k3_n{n}_ncu.txt")
        if os.path.exists(path):
            out["source"] = f"profiles/{tag}_k3_n{n}_ncu.txt"
            break
    else:
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
        elif ln.startswith("warp instructions per"):
            out["inst_per_node"] = float(t[-1])
        elif t[0] == "smsp__issue_active.avg.pct_of_peak_sustained_active":
            out["issue_pct"] = float(t[1])
    if rd is not None and wr is not None:
        out["traffic"] = rd + wr
    return out
UNIT = "search nodes/s (DFS facet-inclusion steps of the workload / wall s)"


def cpu_baseline(n, nodes):
    """The reference on this host, same run: nproc threads and 1 thread on the
    full n workload, plus the reference's leaves/s at n = 6 (all maps) and
    n = 7 (map 0) for the labelled n = 8..11 projections."""
    import psutil

    ref = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")
    threads = os.cpu_count() or 1
    if not os.path.exists(ref):
        return None
    full = _ref_run(ref, n, threads, timeout=600)
    one = _ref_run(ref, n, 1, timeout=600)
    g = _golden()
    rate = {}
    for nn, maps in ((6, None), (7, "0:1")):
        r = _ref_run(ref, nn, threads, maps, timeout=600)
        rate[nn] = {"leaves": r["leaves"], "enum_s": r["enum_s"], "leaves_per_s": r["leaves"] / r["enum_s"],
                    "maps": maps or "all"}
    lps = rate[7]["leaves_per_s"]
    proj = {}
    for nn in range(8, 12):
        leaves = g.get("leaves", {}).get(str(nn))
        if leaves:
            proj[str(nn)] = {"leaves": leaves, "projected_s": leaves / lps,
                             "projected_days": leaves / lps / 86400.0}
    return {"value": nodes / full["wall_s"], "unit": UNIT, "cores": threads, "kind": "reference",
            "physical_cores": psutil.cpu_count(logical=False),
            "sample": f"one full n={n} enumeration, all maps (reference enumerate_wpm, {threads} threads); "
                      f"also 1 thread, n=6 all maps and n=7 map 0 for the projections",
            "wall_s": full["wall_s"], "reference_leaves": full["leaves"], "wpms": full["wpms"],
            "one_thread": {"wall_s": one["wall_s"], "value": nodes / one["wall_s"], "cores": 1},
            "leaves_per_s_by_n": rate,
            "projection": {"note": f"PROJECTION, not a run: combination-space leaves (search.hpp:62-104) / the "
                                   f"reference's measured leaves/s at n=7 on {threads} threads ({lps:.3g}/s); the "
                                   "per-leaf cost grows with the word count, so these are lower bounds",
                           "by_n": proj}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-n", dest="per_n", action="store_false",
                    help="skip the n = 2..11 sweep, the synthetic band and the scaling projection (1 GPU only)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    args.warmup = max(args.warmup, 3)

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
    counter = None
    if world > 1:
        from paper_2301_00806_b200 import dist as wdist

        counter = wdist.share_claim_counter(dist, rank, dev)

    def step():
        """one full enumeration of the workload: 1 GPU = kernel 3 + the sort;
        N GPUs = split, frontier broadcast, shared claims, gather + sort on rank 0"""
        if world == 1:
            plan.run()
            return
        wdist.run_job(dist, plan, rank, world, dev, counter)
        wdist.gather_to_rank0_device(dist, plan, rank, dev)

    for _ in range(args.warmup):
        step()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(dev)
    barrier()
    sampler.start()
    ms_total = ms_search = ms_sort = 0.0
    nodes = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the device-timed window)
        torch.cuda.synchronize(dev)
        if world == 1:
            step()
            ms_total += plan.timing()["ms_total"]  # plan-stream CUDA events: first to last op of the run
        else:
            # every library call blocks on its own stream, so the events on
            # torch's stream bracket the whole step (NCCL included)
            ev0.record()
            step()
            ev1.record()
            torch.cuda.synchronize(dev)
            ms_total += ev0.elapsed_time(ev1)
        st = plan.stats()
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
        t = torch.tensor([float(nodes), float(res.total)], dtype=torch.float64, device=f"cuda:{dev}")
        mx = torch.tensor([ms_step], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot_nodes = int(t[0].item())
        ms_step = mx[0].item()
        tot_wpms = int(t[1].item())
    else:
        tot_wpms = res.total
    value = tot_nodes / (ms_step * 1e-3)

    # e2e: the reference-facing call, host buffers, all copies inside
    e2e_times = []
    h2d = d2h = 0
    for i in range(max(2, min(args.steps, 10)) + 1):
        barrier()
        t0 = time.perf_counter()
        r = wpm_orbits_oneshot(wpm, n, dev, rank, world, counter)
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
    dropin = e2e_dropin(n, dev) if world == 1 else None

    # roofline of kernel 3 vs measured INT32 issue peak
    peak = wpm.int_peak(dev)
    ms_k3 = ms_search / args.steps
    achieved = nodes * 5 * n / (ms_k3 * 1e-3)
    prof = _profile_summary(n)
    roofline = {"bound": "int-issue", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
                "frac": achieved / peak, "traffic": prof.get("traffic"),
                "note": "achieved = 5n int lane-ops per search node (SURVEY 8d) / kernel-3 CUDA-event time; peak = "
                        "measured LOP3+IADD chains on all SMs (wpm_int_peak, live). traffic = dram read+write bytes "
                        "of one kernel-3 launch from the committed ncu --set full capture",
                "issue": {"warp_inst_per_node": prof.get("inst_per_node"),
                          "issue_active_pct": prof.get("issue_pct"),
                          "warp_inst_peak_per_s": 4 * 148 * 1.965e9,
                          "profile": prof.get("source"),
                          "note": "the kernel is issue-bound: one DFS per warp has O(n) lanes of work per node; "
                                  "see profiles/ (k3 ncu summaries)"}}

    num_maps = plan.num_maps
    per_n = synthetic = scaling = None
    if world == 1 and args.per_n:
        plan.close()
        plan = None
        per_n = sweep_per_n(wpm, dev, flush, g)
        synthetic = sweep_synthetic(wpm, dev, flush, g)
        scaling = scaling_projection(wpm, dev, flush)

    if rank == 0:
        cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(n, expect_nodes)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64 (GF(2) bitsets)",
            "data": "synthetic (IDCM orbit maps, deterministic; no dataset)",
            "config": workload_config(n, num_maps),
            "run": {"wpms": tot_wpms, "dfs_nodes": tot_nodes, "l2": "flushed (256 MB write) between timed steps",
                    "parallelism": "1 GPU: persistent kernel 3, in-GPU work queue" if world == 1 else
                    f"{world} GPUs: split below the root + shared-frontier claims (dist.run_job)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "wall_ms": e2e_s * 1e3, "min_ms": min(e2e_times) * 1e3,
                    "samples_ms": [round(t * 1e3, 3) for t in e2e_times],
                    "call": "wpm_enumerate_orbits (one-shot C-ABI)" if world == 1 else
                            "Plan.orbits + dist.run_job + gather to rank 0 + D2H"},
            "e2e_dropin": dropin,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "gpu_launches_per_step": {"seed_tasks": 1, "k3_search": 1, "k4_sort": 1},
            "breakdown_ms": {"search": ms_k3, "sort": ms_sort / args.steps, "step": ms_step},
            "parity": {"wpms_expected": expect_wpms, "nodes_expected": expect_nodes,
                       "ok": tot_wpms == expect_wpms and tot_nodes == expect_nodes},
            "host_wall_s": t_host,
        }
        if per_n is not None:
            line["per_n"] = per_n
            line["synthetic"] = synthetic
            line["scaling_projection"] = scaling
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
        if counter is not None:
            dist.barrier()
            wpm.claim_counter_close(dev, counter[0], counter[1])
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


def wpm_orbits_oneshot(wpm, n, dev, rank, world, counter=None):
    """wpm_enumerate_orbits for world == 1.  For world > 1: every rank builds
    its plan from the host maps, the ranks run the shared-frontier job
    (dist.run_job), the canonical rows go to rank 0 (send/recv), rank 0 sorts
    them and copies the full list to the host."""
    if world == 1:
        return wpm.enumerate_orbits(n, device=dev)
    import torch
    import torch.distributed as dist

    from paper_2301_00806_b200 import dist as wdist

    with wpm.Plan.orbits(n, device=dev) as p:
        wdist.run_job(dist, p, rank, world, dev, counter)
        total, dups, rows, maps = wdist.gather_to_rank0_device(dist, p, rank, dev, return_rows=True)
        d2h = 0
        if rank == 0:
            assert dups == 0
            host = torch.empty(rows.numel(), dtype=rows.dtype, pin_memory=True)
            host.copy_(rows)
            d2h = host.numel() * host.element_size()
    return _E2E(0, d2h, total)


def e2e_dropin(n, dev):
    """The drop-in's own return type, timed: tools/dropin_e2e (C++,
    include/plseeds_b200.hpp) runs the Algorithm-2 per-orbit loop
    (pipeline.hpp:58-72) through plseeds_b200::enumerate_orbits and builds
    every std::vector<PureComplex> -- the reference arm's output objects."""
    exe = os.path.join(ROOT, "build", "dropin_e2e")
    if not os.path.exists(exe):
        return None
    out = subprocess.run([exe, str(n), str(dev), "7"], capture_output=True, text=True, timeout=300)
    if out.returncode != 0:
        return {"error": out.stderr[-300:]}
    return json.loads(out.stdout.strip().splitlines()[-1])


def scaling_projection(wpm, dev, flush, cases=((8, None), (11, None), (11, 0.80)), max_w=8, per_gpu=None):
    """1-GPU PROJECTION of the multi-GPU job (labelled as such; the driver's
    SCALE run measures the real thing), built from measured pieces:
      * t_split(W): every GPU splits its share of the root tasks below the
        root until >= per_gpu records (the library's frontier target); the
        W shards are timed one after another here, the slowest counts;
      * t_claim(W): with ~5 k records and ~4 k warps per GPU, every record is
        claimed at launch, so each GPU works through about 1/W of the
        frontier with only donation to spread it over its warps.  Each of the
        W strided shards of the concatenated frontier is run as a claim phase
        on its own (a fresh plan: one GPU, its shard only, kernel-3 device
        time), and the slowest shard counts.
    projected T_W = t_split(W) + max_s t_claim(W, s); speed-ups are against the
    measured direct 1-GPU run.  Also reported: the per-record node counts'
    static max/mean and a list schedule in claim order (the bound if GPUs
    could keep claiming single records), both at the 1-GPU claim rate."""
    import heapq
    import sys as _sys

    import numpy as np
    import torch

    _sys.path.insert(0, os.path.join(ROOT, "tests"))
    import catalog as C

    from paper_2301_00806_b200 import dist as wpm_dist

    if per_gpu is None:
        per_gpu = int(os.environ.get("WPM_SPLIT_PER_GPU", "640"))
    out = []
    for n, d in cases:
        if d is None:
            mk = lambda: wpm.Plan.orbits(n, device=dev)  # noqa: E731
            name = f"n={n}, all maps"
        else:
            u = C.synthetic_universe(1, d)
            mk = lambda: wpm.Plan.universes(15, 11, [u], facet_cap=252, device=dev)  # noqa: E731
            name = f"synthetic (15, 11) d={d} seed 1"
        with mk() as p, mk() as q:
            p.run()
            flush.zero_()
            torch.cuda.synchronize(dev)
            p.run()
            t_one = p.timing()["ms_total"]
            # the split as W GPUs run it: every GPU splits its share of the
            # root tasks; the shards run one after another here, timed apiece
            t_shard = {}
            for W in (1, 2, 4, 8):
                times = []
                for sidx in range(W):
                    for rep in range(2):  # the first pass sizes the frontier / queue buffers
                        torch.cuda.synchronize(dev)
                        t0 = time.perf_counter()
                        p.split(0, per_gpu, sidx, W)
                        dt = (time.perf_counter() - t0) * 1e3
                    times.append(dt)
                t_shard[W] = max(times)
            parts = []
            for sidx in range(max_w):
                p.split(0, per_gpu, sidx, max_w)
                ptr, cnt, recw = p.frontier()
                parts.append(torch.as_tensor(wpm_dist._wrap_device(ptr, cnt * recw, torch.int32, dev)).clone())
            recs = torch.cat(parts)
            F = recs.numel() // recw
            rv = recs.view(F, recw)
            ctr, _ = wpm.claim_counter_create(dev)
            try:
                # per-record nodes: the whole frontier claimed by one GPU
                q.set_root_stats(True)
                q.load_frontier(recs.data_ptr(), F)
                wpm.claim_counter_reset(dev, ctr)
                q.run_claim(ctr)
                t_main = q.stats()["ms_search"]
                per, _ = q.root_nodes()
                q.set_root_stats(False)
                # the W-GPU claim phase: each GPU's 1/W of the records on its own
                t_claim = {}
                for W in (1, 2, 4, 8):
                    ts = []
                    for sidx in range(W):
                        sub = rv[sidx::W].contiguous()
                        q.load_frontier(sub.data_ptr(), sub.shape[0])
                        wpm.claim_counter_reset(dev, ctr)
                        q.run_claim(ctr)
                        ts.append(q.stats()["ms_search"])
                    t_claim[W] = (max(ts), float(np.mean(ts)))
            finally:
                wpm.claim_counter_close(dev, ctr, False)
        per = per.astype(np.float64)
        tot = per.sum()
        rate = tot / max(t_main, 1e-3)  # nodes per ms, one GPU claiming the whole frontier
        rows = []
        for W in (1, 2, 4, 8):
            loads = np.zeros(W)
            for i, x in enumerate(per):
                loads[i % W] += x
            h = [(0.0, i) for i in range(W)]
            for x in per:
                t, i = heapq.heappop(h)
                heapq.heappush(h, (t + x, i))
            mk_nodes = max(t for t, _ in h)
            t_w = t_shard[W] + t_claim[W][0]
            rows.append({"W": W, "claim_ms_slowest_shard": round(t_claim[W][0], 3),
                         "claim_ms_mean_shard": round(t_claim[W][1], 3),
                         "static_max_over_mean": float(loads.max() / loads.mean()),
                         "dynamic_makespan_over_mean": float(mk_nodes / (tot / W)),
                         "projected_ms": round(t_w, 3), "projected_speedup": round(t_one / t_w, 3),
                         "list_schedule_bound_speedup": round(t_one / (t_shard[W] + mk_nodes / rate), 3)})
        out.append({"case": name, "per_gpu_target": per_gpu, "frontier_records": int(F),
                    "split_ms_host": round(t_shard[max_w], 3),
                    "split_ms_by_W": {str(k): round(v, 3) for k, v in t_shard.items()},
                    "claim_ms_one_gpu_all_records": round(t_main, 3), "one_gpu_run_ms": round(t_one, 3),
                    "claim_nodes": int(tot),
                    "largest_record_frac": float(per.max() / tot) if tot else None, "by_W": rows})
    return {"note": "PROJECTION from 1-B200 runs (not a multi-GPU run): each W-GPU shard's split and claim "
                    "phase timed on its own; excludes the NCCL frontier broadcast and the rank-0 gather",
            "cases": out}


if __name__ == "__main__":
    sys.exit(main())

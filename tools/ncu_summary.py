"""Summarise an ncu report / launch list into profiles/ (dev tool).

usage: python tools/ncu_summary.py REPORT.ncu-rep UNITS OUT.txt [UNIT_NAME]
       (UNITS = work units in the launch, e.g. search nodes; 0 = per launch)
       python tools/ncu_summary.py --launches launches.csv STEPS OUT.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__maximum_warps_per_active_cycle_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
]


def ncu_csv(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def report(rep, nodes, out, unit="search node"):
    raw = list(csv.reader(io.StringIO(ncu_csv(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    lines = [f"ncu --set full summary of {rep} (kernel: {vals[hdr.index('Kernel Name')]})", ""]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            lines.append(f"{h:60s} {v:>18s} {u}")
            d[h] = v
    inst = float(d.get("smsp__inst_executed.sum", "0").replace(",", ""))
    dur = float(d.get("gpu__time_duration.sum", "0").replace(",", ""))
    lines.append("")
    if nodes:
        lines.append(f"{unit}s in this launch{'':<10s} {nodes}")
        lines.append(f"warp instructions per {unit:<14s} {inst / nodes:.1f}")
        lines.append(f"{unit}s/s in this (profiled) launch {nodes / (dur * 1e-3):.3e}  (ncu replay: not a bench number)")
    else:
        nodes = 1
        unit = "launch"
    st = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and
          not h.endswith("not_issued")]
    tot = sum(float(v or 0) for _, v in st)
    lines.append("")
    lines.append("warp stall sampling (share of samples):")
    for h, v in sorted(st, key=lambda x: -float(x[1] or 0))[:10]:
        lines.append(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * float(v or 0) / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source",
                                                "cuda,sass"]))))
    if len(src) > 3:
        h = src[2]
        ie = h.index("Instructions Executed")
        agg = []
        for r in src[3:]:
            if len(r) > ie and r[0] and r[2] == "-":
                try:
                    agg.append((int(r[ie] or 0), int(r[0]), r[1].strip()[:88]))
                except ValueError:
                    pass
        lines.append("")
        lines.append(f"top CUDA source lines by warp instructions executed (per {unit}):")
        for c, ln, s in sorted(agg, reverse=True)[:25]:
            lines.append(f"  {c / nodes:7.1f}  L{ln:<5d} {s}")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, steps, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    c, t = collections.Counter(), collections.defaultdict(float)
    for d in data:
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:70]
            c[k] += 1
            t[k] += float(d["Metric Value"])
    tot = sum(t.values())
    lines = [f"ncu launch list ({path}): gpu__time_duration.sum, --clock-control none, cold-cache, serialised",
             f"{'launches':>8s} {'total us':>10s} {'share':>6s}  kernel"]
    for k in sorted(t, key=lambda k: -t[k]):
        lines.append(f"{c[k]:8d} {t[k] / 1e3:10.1f} {100 * t[k] / tot:5.1f}%  {k}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], int(sys.argv[3]), sys.argv[4])
    else:
        report(sys.argv[1], int(sys.argv[2]), sys.argv[3], *(sys.argv[4:5] or ["search node"]))

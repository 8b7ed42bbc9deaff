"""Per-function warp-instruction breakdown of kernel 3 from an ncu report (dev tool).
usage: python tools/ncu_breakdown.py REPORT.ncu-rep NODES"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, N = sys.argv[1], int(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
secs, cur = [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = {"file": r[1], "rows": []}
        secs.append(cur)
        continue
    if cur is not None:
        cur["rows"].append(r)
src = open("paper_2301_00806_b200/csrc/k3_search.cu").read().split("\n")
starts = []
for i, l in enumerate(src):
    m = re.match(r".*__device__ (?:__forceinline__ )?\S+\s+(\w+)\(", l) or re.match(r"__global__ .*?(\w+)\(", l)
    if m:
        starts.append((i + 1, m.group(1)))


def fn(line):
    name = "top"
    for s, nm in starts:
        if s <= line:
            name = nm
    return name


agg, hdr_lines, stall = collections.Counter(), collections.Counter(), collections.Counter()
for sec in secs:
    h = next((r for r in sec["rows"] if "Instructions Executed" in r), None)
    if not h:
        continue
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    for r in sec["rows"]:
        if len(r) > ie and r[0].isdigit() and r[2] == "-":
            c = int(r[ie] or 0)
            if "k3_search.cu" in sec["file"]:
                agg[fn(int(r[0]))] += c
                stall[fn(int(r[0]))] += int(r[ss] or 0)
            else:
                hdr_lines[(sec["file"].split("/")[-1], r[1].strip()[:50])] += c
tot = sum(agg.values()) + sum(hdr_lines.values())
st = sum(stall.values()) or 1
print(f"total warp instructions per node: {tot / N:.1f}")
for k, v in agg.most_common():
    print(f"{v / N:7.1f}  stall {100 * stall[k] / st:5.1f}%  {k}")
print("-- inlined CUDA-header intrinsics")
for k, v in hdr_lines.most_common(8):
    print(f"{v / N:7.1f}  {k}")

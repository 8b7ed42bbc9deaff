import os, sys, time, json
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
n = int(sys.argv[1]); nfix = int(sys.argv[2])
with wpm.Plan.orbits(n) as p:
    w = p.space_blocks(0)
    print("blocks", w, flush=True)
    t0 = time.perf_counter()
    tot = p.run_kernel_basis_prefix(0, [0] * nfix)
    dt = time.perf_counter() - t0
    st = p.kernel_basis_stats()
    print(json.dumps({"n": n, "nfix": nfix, "accepted": tot, "leaves": st["leaves"], "s": dt, "ms_leaves": st["ms_leaves"], "leaves_per_s": st["leaves"] / (st["ms_leaves"] * 1e-3)}), flush=True)

"""Runs kernel 3 on one workload (for ncu captures): n, or 'syn' for the d=0.80 synthetic."""
import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2301_00806_b200 as wpm
arg = sys.argv[1] if len(sys.argv) > 1 else "5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if arg == "syn":
    import catalog as C
    p = wpm.Plan.universes(15, 11, [C.synthetic_universe(1, 0.80)], facet_cap=252)
else:
    p = wpm.Plan.orbits(int(arg))
with p:
    for _ in range(reps):
        p.run()
    print(p.stats(), p.timing())

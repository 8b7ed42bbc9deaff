import os, sys
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
with wpm.Plan.orbits(n) as p:
    for _ in range(2):
        p.run()
    print(p.stats())

import os, sys
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
n = int(sys.argv[1])
with wpm.Plan.orbits(n) as p:
    print(n, p.run(), p.stats())

import os, sys
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
for n in (2, 3, 4):
    with wpm.Plan.orbits(n) as p:
        p.run(); print(n, p.line13(), flush=True)
        try:
            print(n, "line15", p.line15(), flush=True)
        except Exception as e:
            print(n, "ERR", e, flush=True)
            break

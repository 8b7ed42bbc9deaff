import sys, time
sys.path.insert(0, '.')
import paper_2301_00806_b200 as wpm
n = int(sys.argv[1]); b = int(sys.argv[2])
with wpm.Plan.orbits(n) as p:
    print('plan', flush=True)
    p.set_node_budget(b)
    t = time.time(); tot = p.run(); print('run1', tot, p.truncated(), p.stats(), round(time.time() - t, 3), flush=True)
    p.set_node_budget(0)
    t = time.time(); tot = p.run(); print('run2', tot, p.truncated(), p.stats(), round(time.time() - t, 3), flush=True)

import os, sys
sys.path.insert(0, os.getcwd())
os.environ["WPM_TRACE"] = "1"
import paper_2301_00806_b200 as wpm
for n, nd in ((5, 2), (8, 3), (11, 2)):
    with wpm.Plan.orbits(n, devices=[0] * nd) as p:
        t = p.run()
        print(n, nd, t, p.fetch().nodes, p.device_stats(), flush=True)
    with wpm.Plan.orbits(n) as p:
        print("single", p.run(), flush=True)

"""One workload per kernel family for the ncu captures (dev tool)."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
what = sys.argv[1]
if what == "k3":
    with wpm.Plan.orbits(int(sys.argv[2])) as p:
        p.run(); p.run()
elif what == "line13":
    with wpm.Plan.orbits(int(sys.argv[2])) as p:
        p.run(); p.line13(); p.line13()
elif what == "alg1":
    with wpm.Plan.orbits(int(sys.argv[2])) as p:
        p.run_kernel_basis(); p.run_kernel_basis()
elif what == "verify":
    with wpm.Plan.orbits(int(sys.argv[2])) as p:
        p.run(); p.verify(reach=True); p.verify(reach=True)
elif what == "create":
    for _ in range(2):
        with wpm.Plan.orbits(int(sys.argv[2])) as p:
            pass
print("ok", what)

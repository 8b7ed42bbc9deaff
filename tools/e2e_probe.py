"""e2e one-shot timing probe: wall vs device time of wpm_enumerate_orbits
before/after other plan kinds ran in the process.  Development tool."""
import sys
import time

sys.path.insert(0, '.')
import paper_2301_00806_b200 as wpm  # noqa: E402


def t(n, k=6):
    out = []
    for _ in range(k):
        t0 = time.perf_counter()
        r = wpm.enumerate_orbits(n)
        w = (time.perf_counter() - t0) * 1e3
        out.append(f"{w:.2f}/{r.ms_total:.2f}/{r.ms_search:.2f}")
        del r
    return out


print('fresh', t(5))
with wpm.Plan.orbits(5) as p:
    p.run(); p.line13(); p.line15()
print('after line15', t(5))
with wpm.Plan.orbits(5) as p:
    p.run(); p.line13(); p.line15()
    print('inside plan', t(5))
print('after line15 again', t(5, 10))

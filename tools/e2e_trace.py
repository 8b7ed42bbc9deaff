"""Phase trace of the one-shot C-ABI call (dev tool): WPM_TRACE=1."""
import os
import sys
import time

os.environ.setdefault("WPM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_00806_b200 as wpm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for i in range(4):
    t0 = time.perf_counter()
    r = wpm.enumerate_orbits(n)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.2f} ms  total={r.total} h2d={r.h2d_bytes} d2h={r.d2h_bytes}",
          file=sys.stderr, flush=True)

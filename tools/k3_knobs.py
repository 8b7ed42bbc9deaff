"""Kernel-3 launch/queue knob sweep at one n (dev tool): median search ms over
5 runs per setting, settings via the env knobs plan_search reads per run."""
import itertools
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_00806_b200 as wpm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
grid = {
    "WPM_DONATE_MAX": ["", "2", "4", "8"],
    "WPM_HUNGRY": ["", "256"],
    "WPM_CHECK_EVERY": ["", "8", "32"],
    "WPM_BACKOFF_MIN": ["", "512"],
}
with wpm.Plan.orbits(n) as p:
    p.run()
    res = []
    for combo in itertools.product(*grid.values()):
        for k, v in zip(grid, combo):
            if v:
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        ms = []
        for _ in range(5):
            p.run()
            ms.append(p.stats()["ms_search"])
        res.append((statistics.median(ms), dict(zip(grid, combo)), p.stats()["tasks"]))
    res.sort(key=lambda r: r[0])
    for r in res[:12] + res[-3:]:
        print(json.dumps({"ms": round(r[0], 3), "tasks": r[2], **r[1]}))

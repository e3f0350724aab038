"""Run bench.py's paper experiments (ADR + Riccati whole-integration
wall-clock vs the published MATLAB numbers) alone; prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2304_02327_b200 as kp  # noqa: E402

only = sys.argv[1] if len(sys.argv) > 1 else ""
if only:
    bench.PAPER_RUNS = [r for r in bench.PAPER_RUNS if only in r[0]]
print(json.dumps(bench.run_paper_experiments(kp), indent=1))

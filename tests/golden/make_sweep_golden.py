"""Golden output of the REFERENCE sweep harness (rsvdkit 0.1.0
experiment.run_experiment, experiment.py:197-263) on a small synthetic
spec, for the GPU harness parity test. Build container only:

    RSVDKIT_SRC=/root/reference/pkg/src RSVD_BACKEND=python python tests/golden/make_sweep_golden.py
"""

import json
import os
import sys

os.environ.setdefault("RSVD_BACKEND", "python")
sys.path.insert(0, os.environ.get("RSVDKIT_SRC", "/root/reference/pkg/src"))
import numpy as np  # noqa: E402
import rsvdkit as rk  # noqa: E402

SPEC = {"algorithms": ["bk", "si"], "k": 5, "q_list": [1, 2, 4], "seeds": [0, 3],
        "synthetic": {"n": 300, "d": 120, "spectrum": [1.0 / (i ** 0.7) for i in range(1, 121)], "seed": 7}}
rows, summary = rk.run_experiment(rk.ExperimentSpec.from_dict(SPEC))
for r in rows:
    r.pop("wall_ms")
out = {"spec": SPEC, "rows": rows, "oracle_top": summary["oracle_top_singular_values"], "csv_header":
       rk.rows_to_csv(rows[:0]).strip()}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sweep_golden.json")
json.dump(out, open(path, "w"), indent=1)
print("wrote", path, len(rows))

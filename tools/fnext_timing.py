"""Wall-clock of the SURVEY §8f two-level runs on the device (step-level drivers), against
the reference's own wall time recorded in the golden files (same configs, build container)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P  # noqa: E402

G = ROOT / "tests" / "golden"
rows = []
for name in ("cfg1_twoway", "cfg1_tdep", "cfg1_tdep_twoway", "cfg1_full", "cfg1_tdep_full", "cfg1_gsrc"):
    cfg = P.load_config(ROOT / "configs" / f"{name}.cfg")
    P.two_level_run(cfg, n_steps=1)                      # warm-up (library load, workspaces)
    t0 = time.perf_counter()
    _, stats = P.two_level_run(cfg)
    dt = time.perf_counter() - t0
    z = np.load(G / f"run_{name}.npz")
    rows.append({"config": name, "device_s": dt, "reference_s": float(z["wall"]),
                 "speedup": float(z["wall"]) / dt, "counters": stats.counters})
print(json.dumps(rows, indent=1))

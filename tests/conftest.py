import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

GOLDEN = ROOT / "tests" / "golden"
CONFIGS = ROOT / "configs"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtlgpu.so")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


def has_reference() -> bool:
    return (REFERENCE_SRC / "lpbfsim" / "__init__.py").exists()


# ---- melt-mask margins (SURVEY §7 hard part 4) ------------------------------------------
# Every bit-exact mask assertion records the minimum |T - T_liquidus| over the nodes it
# compared, the number of melted nodes and the field error, so "bit-exact" is shown to be
# non-trivial: a mask can only be equal by construction when margin > error.
MARGINS: dict = {}


def assert_mask(tag: str, T, ref, TL: float, ref_is_packed: bool = False, err: float | None = None):
    """Melt masks T > TL equal to the reference's (a field or np.packbits of its mask);
    records the margin under `tag`.  `err`: max |T - T_ref| (K) when known."""
    import numpy as np
    if tag is None:
        tag = os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0].split("::")[-1]
    T = np.asarray(T)
    mine = T > TL
    if ref_is_packed:
        np.testing.assert_array_equal(np.packbits(mine), ref)
    else:
        ref = np.asarray(ref)
        np.testing.assert_array_equal(mine, ref > TL)
        e = float(np.abs(T - ref).max())
        err = e if err is None else max(err, e)
    margin = float(np.min(np.abs(T - TL))) if T.size else float("inf")
    rec = MARGINS.setdefault(tag, {"min_margin_K": float("inf"), "melt_nodes_max": 0, "masks": 0,
                                   "max_abs_err_K": 0.0})
    rec["min_margin_K"] = min(rec["min_margin_K"], margin)
    rec["melt_nodes_max"] = max(rec["melt_nodes_max"], int(mine.sum()))
    rec["masks"] += 1
    if err is not None:
        rec["max_abs_err_K"] = max(rec["max_abs_err_K"], float(err))
        # margin > error: the mask agreement follows from the error bound, not from luck
        assert margin > err, (tag, margin, err)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    if not MARGINS:
        return
    import json
    terminalreporter.write_sep("-", "melt-mask margins (min |T - T_liquidus| over compared nodes)")
    for tag, r in sorted(MARGINS.items()):
        terminalreporter.write_line(f"{tag}: margin {r['min_margin_K']:.4g} K, max field error "
                                    f"{r['max_abs_err_K']:.3g} K, melted nodes <= {r['melt_nodes_max']}, "
                                    f"{r['masks']} masks")
    out = ROOT / "gpurun_out"
    if out.is_dir():
        (out / "mask_margins.json").write_text(json.dumps(MARGINS, indent=1))

"""Experiment modes over the device solves (``lpbfsim/runner.py:186-440``).

``run_experiment(cfg, out_dir)`` dispatches a config to its mode — ``reference``
(monolithic fine-grid run), ``two-level-space`` / ``two-level-spacetime``,
``convergence-study`` (reference + a sweep of multirate runs, errors per run) and
``compare`` (multirate against uniform-step timing) — and writes the reference's output
files: ``errors.csv``, ``timing.csv``, ``summary.json``, ``centerline.csv``,
``study_matrix.csv``.  Every solve runs on the GPU (``run_reference``,
``two_level_run``); error norms use the device metrics (``metrics.error_metrics``).
VTK snapshots are not written: a cadence other than ``none`` raises
``UnsupportedOnDevice``.  2D control-line temperatures do not arise (3D only).
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import UnsupportedOnDevice
from .metrics import ErrorReport, RunLog, composite_sampler, centerline_profile, error_metrics
from .runner import build_problem, convert_config, run_reference
from .stats import RunStats

__all__ = ["RunArtifacts", "run_experiment", "run_study", "run_compare", "study_pairs", "write_csv"]


@dataclass
class RunArtifacts:
    """``runner.py:36-46``."""

    out_dir: Path
    log: RunLog
    stats: RunStats
    report: ErrorReport | None = None
    summary: dict | None = None
    reports: dict | None = None
    reference: object | None = None


def _fmt(v):
    if isinstance(v, (float, np.floating)):
        return f"{float(v):.12g}"
    return v


def write_csv(path, header: list, rows):
    """``vtkio.write_csv`` (``vtkio.py:47-61``): fixed header, %.12g floats."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with path.open("w", newline="") as f:
        w = csv.writer(f)
        w.writerow(header)
        for row in rows:
            w.writerow([_fmt(v) for v in row])


def _cadence(cfg, override):
    cadence = override if override is not None else cfg.snapshots
    if cadence != "none":
        raise UnsupportedOnDevice(f"VTK snapshots (cadence {cadence!r}) are not written by the device "
                                  "package; set 'snapshots none'")
    return cadence


def _write_errors_csv(out: Path, report: ErrorReport):
    rows = [(t, kind, rel, "" if np.isnan(ts) else ts)
            for t, kind, rel, ts in zip(report.times, report.kinds, report.rel_l2, report.t_star)]
    write_csv(out / "errors.csv", ["t", "step_kind", "rel_l2_local", "T_star"], rows)


def _write_timing_csv(out: Path, stats: RunStats):
    sec, cnt = stats.seconds, stats.counters
    rows = [
        ("total", stats.total_seconds, 1),
        ("global_solve", sec.get("global_solve", 0.0), cnt.get("global_solves", 0)),
        ("local_solve", sec.get("local_solve", 0.0), cnt.get("local_solves", 0)),
        ("assembly", sec.get("assembly", 0.0), cnt.get("picard_iterations", 0)),
        ("coupling_overhead", sec.get("coupling_overhead", 0.0), cnt.get("coupling_iterations", 0)),
        ("reference_solve", sec.get("reference_solve", 0.0), cnt.get("reference_solves", 0)),
        ("predictor", sec.get("predictor", 0.0), cnt.get("predictor_solves", 0)),
    ]
    write_csv(out / "timing.csv", ["phase", "seconds", "count"], rows)


def _two_level_run(cfg, spacetime: bool, dt_macro=None, micro=None):
    """``runner._two_level_run`` (``runner.py:236-257``): (log, stats, state)."""
    from .runner import two_level_run
    log = RunLog()
    state, stats = two_level_run(cfg, spacetime=spacetime, dt_macro=dt_macro, micro=micro, recorder=log.record)
    return log, stats, state


def _centerline(cfg, sample, out: Path, dx: float):
    y, z = cfg.centerline_y, cfg.centerline_z
    if y is None:
        return None
    gb = convert_config(cfg)["global_box"]
    xs, Ts = centerline_profile(sample, y, z, (gb.lo[0], gb.hi[0]), dx)
    write_csv(out / "centerline.csv", ["x", "temperature"], list(zip(xs, Ts)))
    return xs, Ts


def run_experiment(cfg, out_dir, snapshots: str | None = None, threads: int = 1) -> RunArtifacts:
    """``runner.run_experiment`` (``runner.py:270-284``)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    _cadence(cfg, snapshots)
    if cfg.mode == "reference":
        return _run_reference_mode(cfg, out)
    if cfg.mode in ("two-level-space", "two-level-spacetime"):
        return _run_two_level_mode(cfg, out, cfg.mode == "two-level-spacetime")
    if cfg.mode == "convergence-study":
        return run_study(cfg, out, snapshots, threads)
    if cfg.mode == "compare":
        return run_compare(cfg, out, snapshots)
    raise ValueError(f"unhandled mode {cfg.mode}")


def _run_reference_mode(cfg, out: Path) -> RunArtifacts:
    """``runner.py:287-315``."""
    from .grid import build_structured_grid
    stats = RunStats()
    mesh = build_structured_grid(convert_config(cfg)["global_box"], cfg.h_reference)
    rows = []

    def observer(state):
        rows.append((state.time, "macro", 0.0, ""))

    traj = run_reference(cfg, stats=stats, mesh=mesh, observer=observer)
    write_csv(out / "errors.csv", ["t", "step_kind", "rel_l2_local", "T_star"], rows)
    _write_timing_csv(out, stats)
    final = traj.state(len(traj) - 1)
    _centerline(cfg, final, out, mesh.spacing[0])
    summary = {"mode": "reference", "steps": len(traj) - 1, **stats.report()}
    (out / "summary.json").write_text(json.dumps(summary, indent=2))
    return RunArtifacts(out, RunLog(), stats, None, summary)


def _run_two_level_mode(cfg, out: Path, spacetime: bool) -> RunArtifacts:
    """``runner.py:318-339``."""
    log, stats, state = _two_level_run(cfg, spacetime)
    rows = [(r.time, r.kind, "", "") for r in log.of_kind("initial", "micro", "macro")]
    write_csv(out / "errors.csv", ["t", "step_kind", "rel_l2_local", "T_star"], rows)
    _write_timing_csv(out, stats)
    final = log.of_kind("macro")[-1]
    _centerline(cfg, composite_sampler(final.local, final.global_field), out, cfg.h_reference)
    summary = {"mode": cfg.mode, "macro_steps": len(log.of_kind("macro")),
               "local_solves_expected": len(log.of_kind("macro")) * cfg.micro_steps, **stats.report()}
    (out / "summary.json").write_text(json.dumps(summary, indent=2))
    return RunArtifacts(out, log, stats, None, summary)


def study_pairs(cfg) -> list:
    """(dt_macro, micro_steps) pairs of the sweep (``runner.py:342-353``)."""
    dts = cfg.dt_macro_list or [cfg.dt_macro]
    micros = cfg.dt_micro_list or [cfg.dt_micro]
    pairs = []
    for dt in dts:
        for dmu in micros:
            ratio = dt / dmu
            if abs(ratio - round(ratio)) > 1e-9 * ratio:
                raise ValueError(f"micro step {dmu:g} does not divide macro step {dt:g}")
            pairs.append((dt, int(round(ratio))))
    return pairs


def run_study(cfg, out: Path, snapshots=None, threads: int = 1) -> RunArtifacts:
    """Reference solve plus a sweep of multirate runs, errors per run (``runner.py:356-403``).
    The runs share one GPU, so they execute one after another whatever ``threads`` says."""
    out = Path(out)
    stats = RunStats()
    with stats.timer("reference_total"):
        reference = run_reference(cfg, stats=stats)
    pairs = study_pairs(cfg)
    matrix_rows, reports = [], {}
    for dt, micro in pairs:
        log, run_stats, _ = _two_level_run(cfg, True, dt_macro=dt, micro=micro)
        report = error_metrics(log, reference)
        sub = out / f"dt_{dt:g}" / f"micro_{dt / micro:g}"
        sub.mkdir(parents=True, exist_ok=True)
        _write_errors_csv(sub, report)
        _write_timing_csv(sub, run_stats)
        matrix_rows.append((dt, dt / micro, report.mean_rel_l2))
        reports[(dt, micro)] = report
    write_csv(out / "study_matrix.csv", ["dt_global", "dt_local", "mean_rel_l2"], matrix_rows)
    summary = {"mode": "convergence-study", "pairs": [[dt, dt / m] for dt, m in pairs],
               "mean_rel_l2": {f"{dt:g}/{dt / m:g}": reports[(dt, m)].mean_rel_l2 for dt, m in pairs},
               **stats.report()}
    (out / "summary.json").write_text(json.dumps(summary, indent=2))
    return RunArtifacts(out, RunLog(), stats, None, summary, reports=reports, reference=reference)


def run_compare(cfg, out: Path, snapshots=None) -> RunArtifacts:
    """Multirate against uniform-step two-level timing (``runner.py:406-440``)."""
    out = Path(out)
    log_st, stats_st, _ = _two_level_run(cfg, True)
    wall_st = stats_st.total_seconds
    _write_timing_csv(out / "spacetime", stats_st)
    log_sp, stats_sp, _ = _two_level_run(cfg, False)
    wall_sp = stats_sp.total_seconds
    _write_timing_csv(out / "spaceonly", stats_sp)
    summary = {
        "mode": "compare", "wall_spacetime": wall_st, "wall_spaceonly": wall_sp,
        "speedup": wall_sp / wall_st if wall_st > 0 else float("inf"),
        "global_solves_spacetime": stats_st.counters.get("global_solves", 0),
        "global_solves_spaceonly": stats_sp.counters.get("global_solves", 0),
        "local_solves_spacetime": stats_st.counters.get("local_solves", 0),
        "local_solves_spaceonly": stats_sp.counters.get("local_solves", 0),
    }
    (out / "summary.json").write_text(json.dumps(summary, indent=2))
    return RunArtifacts(out, log_st, stats_st, None, summary)

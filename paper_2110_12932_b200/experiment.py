"""Experiment modes over the device solves (``lpbfsim/runner.py:186-440``).

``run_experiment(cfg, out_dir)`` dispatches a config to its mode — ``reference``
(monolithic fine-grid run), ``two-level-space`` / ``two-level-spacetime``,
``convergence-study`` (reference + a sweep of multirate runs, errors per run) and
``compare`` (multirate against uniform-step timing) — and writes the reference's output
files: ``errors.csv``, ``timing.csv``, ``summary.json``, ``centerline.csv``,
``study_matrix.csv``.  Every solve runs on the GPU (``run_reference``,
``two_level_run``); error norms use the device metrics (``metrics.error_metrics``).
Field snapshots are written as the reference's legacy ASCII VTK files
(``vtkio.write_vtk``: every macro record, every 10th micro record for ``all`` in 3D).
2D control-line temperatures do not arise (3D only).
"""

from __future__ import annotations

import csv
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .metrics import ErrorReport, RunLog, composite_sampler, centerline_profile, error_metrics
from .runner import build_problem, convert_config, run_reference
from .stats import RunStats

__all__ = ["RunArtifacts", "run_experiment", "run_study", "run_compare", "study_pairs", "write_csv", "write_vtk"]


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
    """``runner._snapshot_cadence`` (``runner.py:212-213``)."""
    return override if override is not None else cfg.snapshots


def write_vtk(path, mesh, point_data: dict | None = None, title: str = "lpbfsim"):
    """``vtkio.write_vtk`` (``vtkio.py:15-44``): legacy ASCII unstructured grid of the Kuhn
    tets (3D) or the triangles (2D, z = 0) with nodal scalars."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    pts = mesh.coords
    if mesh.dim == 2:
        pts = np.column_stack([pts, np.zeros(len(pts))])
    nv = mesh.dim + 1
    elems = mesh.elems
    ne = len(elems)
    with path.open("w") as f:
        f.write("# vtk DataFile Version 2.0\n")
        f.write(f"{title}\n")
        f.write("ASCII\n")
        f.write("DATASET UNSTRUCTURED_GRID\n")
        f.write(f"POINTS {mesh.n_nodes} double\n")
        for p in pts:
            f.write(f"{p[0]:.10g} {p[1]:.10g} {p[2]:.10g}\n")
        f.write(f"\nCELLS {ne} {ne * (nv + 1)}\n")
        for e in elems:
            f.write(f"{nv} " + " ".join(str(int(v)) for v in e) + "\n")
        f.write(f"\nCELL_TYPES {ne}\n")
        f.write(("5\n" if mesh.dim == 2 else "10\n") * ne)
        if point_data:
            f.write(f"\nPOINT_DATA {mesh.n_nodes}\n")
            for name, values in point_data.items():
                f.write(f"SCALARS {name} double\n")
                f.write("LOOKUP_TABLE default\n")
                for v in np.asarray(values):
                    f.write(f"{v:.10g}\n")


def _write_snapshots(out: Path, cfg, log: RunLog, cadence: str):
    """``runner._write_snapshots`` (``runner.py:216-233``)."""
    if cadence == "none":
        return
    every = 10 if cfg.dimension == 3 and cadence == "all" else 1
    micro_seen = 0
    for r in log.records:
        if r.kind in ("initial", "macro"):
            if r.global_field is not None:
                write_vtk(out / "vtk" / f"global_{r.time:.6e}.vtk", r.global_field.mesh,
                          {"temperature": r.global_field.values})
            if r.local is not None:
                write_vtk(out / "vtk" / f"local_{r.time:.6e}.vtk", r.local.mesh, {"temperature": r.local.values})
        elif r.kind == "micro" and cadence == "all":
            micro_seen += 1                 # decimated records (local None) count too
            if micro_seen % every == 0 and r.local is not None:
                write_vtk(out / "vtk" / f"local_{r.time:.6e}.vtk", r.local.mesh, {"temperature": r.local.values})


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


class DecimatingRecorder:
    """Recorder for the experiment modes that reads only the micro fields its outputs need
    (snapshot decimation on the device, ``runner.py:216-233``): ``micro_every`` = 1 every
    micro field (error metrics), k > 1 every k-th one (VTK cadence "all" in 3D), 0 none
    (cadences "macro" / "none").  The drivers ask ``wants`` once per micro record, in order;
    records whose field is not wanted arrive with ``local=None`` and are logged as such."""

    def __init__(self, log: RunLog, micro_every: int = 1):
        self.log = log
        self.micro_every = int(micro_every)
        self._seen = 0

    def wants(self, kind: str, time: float) -> bool:
        if kind != "micro":
            return True
        self._seen += 1
        return self.micro_every > 0 and self._seen % self.micro_every == 0

    def __call__(self, kind, time, local, global_field, iterations):
        self.log.record(kind, time, local, global_field, iterations)


def _micro_every(cfg, cadence: str) -> int:
    """Which micro fields ``_write_snapshots`` reads for a cadence (``runner.py:219-233``)."""
    if cadence != "all":
        return 0
    return 10 if cfg.dimension == 3 else 1


def _two_level_run(cfg, spacetime: bool, dt_macro=None, micro=None, micro_every: int = 1):
    """``runner._two_level_run`` (``runner.py:236-257``): (log, stats, state).  ``micro_every``:
    the micro fields the caller will read (DecimatingRecorder)."""
    from .runner import two_level_run
    log = RunLog()
    rec = log.record if micro_every == 1 else DecimatingRecorder(log, micro_every)
    state, stats = two_level_run(cfg, spacetime=spacetime, dt_macro=dt_macro, micro=micro, recorder=rec)
    return log, stats, state


def _t_star_fn(cfg, log: RunLog):
    """``runner._t_star_fn`` (``runner.py:166-178``): the 2D studies' control-line temperature
    of a record, sampled from the fine field where it covers and the coarse one elsewhere."""
    if cfg.dimension != 2 or cfg.control_line_y is None:
        return None
    from .metrics import control_temperature
    gb = convert_config(cfg)["global_box"]
    x0, x1 = gb.lo[0], gb.hi[0]
    dx = cfg.h_global / 2

    def t_star(record):
        glob = record.global_field or log.latest_global_at(record.time)
        return control_temperature(composite_sampler(record.local, glob), cfg.control_line_y, (x0, x1), dx)

    return t_star


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
    if cfg.mode == "reference":
        return _run_reference_mode(cfg, out, snapshots)
    if cfg.mode in ("two-level-space", "two-level-spacetime"):
        return _run_two_level_mode(cfg, out, cfg.mode == "two-level-spacetime", snapshots)
    if cfg.mode == "convergence-study":
        return run_study(cfg, out, snapshots, threads)
    if cfg.mode == "compare":
        return run_compare(cfg, out, snapshots)
    raise ValueError(f"unhandled mode {cfg.mode}")


def _run_reference_mode(cfg, out: Path, snapshots=None) -> RunArtifacts:
    """``runner.py:287-315``."""
    from .grid import build_structured_grid
    stats = RunStats()
    mesh = build_structured_grid(convert_config(cfg)["global_box"], cfg.h_reference)
    cadence = _cadence(cfg, snapshots)
    rows = []
    count = [0]

    def observer(state):
        count[0] += 1
        rows.append((state.time, "macro", 0.0, ""))
        if cadence == "all" and count[0] % (1 if cfg.dimension == 2 else 10) == 0:
            write_vtk(out / "vtk" / f"reference_{state.time:.6e}.vtk", mesh, {"temperature": state.values})

    traj = run_reference(cfg, stats=stats, mesh=mesh, observer=observer)
    if cadence == "macro":
        fr = traj.state(len(traj) - 1)
        write_vtk(out / "vtk" / f"reference_{fr.time:.6e}.vtk", mesh, {"temperature": fr.values})
    write_csv(out / "errors.csv", ["t", "step_kind", "rel_l2_local", "T_star"], rows)
    _write_timing_csv(out, stats)
    final = traj.state(len(traj) - 1)
    _centerline(cfg, final, out, mesh.spacing[0])
    summary = {"mode": "reference", "steps": len(traj) - 1, **stats.report()}
    (out / "summary.json").write_text(json.dumps(summary, indent=2))
    return RunArtifacts(out, RunLog(), stats, None, summary)


def _run_two_level_mode(cfg, out: Path, spacetime: bool, snapshots=None) -> RunArtifacts:
    """``runner.py:318-339``."""
    cadence = _cadence(cfg, snapshots)
    log, stats, state = _two_level_run(cfg, spacetime, micro_every=_micro_every(cfg, cadence))
    rows = [(r.time, r.kind, "", "") for r in log.of_kind("initial", "micro", "macro")]
    write_csv(out / "errors.csv", ["t", "step_kind", "rel_l2_local", "T_star"], rows)
    _write_timing_csv(out, stats)
    _write_snapshots(out, cfg, log, _cadence(cfg, snapshots))
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
        report = error_metrics(log, reference, t_star_of=_t_star_fn(cfg, log))
        sub = out / f"dt_{dt:g}" / f"micro_{dt / micro:g}"
        sub.mkdir(parents=True, exist_ok=True)
        _write_errors_csv(sub, report)
        _write_timing_csv(sub, run_stats)
        _write_snapshots(sub, cfg, log, _cadence(cfg, snapshots))
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
    log_st, stats_st, _ = _two_level_run(cfg, True, micro_every=_micro_every(cfg, _cadence(cfg, snapshots)))
    wall_st = stats_st.total_seconds
    _write_timing_csv(out / "spacetime", stats_st)
    _write_snapshots(out / "spacetime", cfg, log_st, _cadence(cfg, snapshots))
    log_sp, stats_sp, _ = _two_level_run(cfg, False, micro_every=0)
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

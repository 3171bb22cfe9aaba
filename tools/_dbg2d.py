import sys, json, numpy as np, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2110_12932_b200 as P
from paper_2110_12932_b200.multirate import predictor_global
z = np.load(ROOT / "tests/golden/run_run2d_twoway.npz")
tmp = Path(tempfile.mkdtemp())
rho, chi, Ts, Tl, S = (float(v) for v in z["mat_scalars"])
lines = ["units K", f"rho {rho!r}", f"chi {chi!r}", f"T_solidus {Ts!r}", f"T_liquidus {Tl!r}", f"S {S!r}",
         "[conductivity]"] + [f"{float(a)!r} {float(b)!r}" for a, b in z["k_table"]] + ["[heat_capacity]"] + \
        [f"{float(a)!r} {float(b)!r}" for a, b in z["c_table"]]
(tmp / "in625.mat").write_text("\n".join(lines) + "\n")
for name in ("run2d", "run2d_twoway"):
    (tmp / f"{name}.cfg").write_text((ROOT / f"configs/{name}.cfg").read_text())
    cfg = P.load_config(tmp / f"{name}.cfg")
    prob, lm = P.build_problem(cfg)
    print(name, "k_l[0:2]", prob.mat_local.conductivity_table[:2].tolist(), "k_g[0:2]", prob.mat_global.conductivity_table[:2].tolist(),
          "c_l", prob.mat_local.heat_capacity_table[:2].tolist(), "rho", prob.mat_local.rho, prob.mat_global.rho, "chi", prob.mat_local.chi)
    T0 = P.uniform_field(prob.global_mesh, cfg.T_initial, time=0.0)
    state = P.initial_state(prob, lm, T0)
    pred = predictor_global(prob, state, cfg.dt_macro)
    print(name, "predictor max", pred.values.max())
    out = P.solve_local(prob, state.local_field, 0.01, state.gamma, state.trace)
    print(name, "first local max", out.values.max(), "solver", prob.solver)

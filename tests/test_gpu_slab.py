"""z-slab multi-rank global solve against the single-GPU solve and the oracle.

The box the GPU tests run on has one GPU, so the multi-rank cases run 2 and 3
processes over gloo on the same device: the halos and partial sums go through the
host (the NCCL path differs only in moving the same planes device to device), and
no kernel waits on another rank's kernel.  Tolerance: 1e-12 relative L-inf (the
slab solve mirrors scipy's cg; only the summation order of the dot products
differs), CG iteration counts equal to the single-GPU solve's.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2110_12932_b200 as P
from paper_2110_12932_b200 import _native as N
from paper_2110_12932_b200 import ops
from paper_2110_12932_b200 import slab as SL

from .conftest import CONFIGS
from .conftest import assert_mask
from .test_gpu_parity import _oracle_step, rel

pytestmark = pytest.mark.gpu


def _case(name, seed, gaussian):
    cfg = P.load_config(CONFIGS / f"{name}.cfg")
    problem, _ = P.build_problem(cfg)
    grid = problem.global_mesh
    rng = np.random.default_rng(seed)
    T = rng.uniform(293.0, 2293.0, grid.n_nodes)
    if gaussian:
        src = problem.local_source(cfg.dt_macro)
        return cfg, grid, T, None, src
    pts, pw = problem.global_source(0.0, cfg.dt_macro)
    return cfg, grid, T, ops.deposit_load(grid, pts, pw), None


def _slab_solve(name, seed, gaussian, rank, world):
    import torch
    cfg, grid, T, load, src = _case(name, seed, gaussian)
    S = SL.SlabGlobalSolver(grid, 9.8, 8440 * 410.0, rank=rank, world=world, device="cuda:0", rtol=1e-12)
    S.set_own(S.x, T)
    if load is not None:
        S.set_own(S.load, load)
    info = S.step(cfg.dt_macro, 293.0, with_load=load is not None,
                  gaussian=src.device_args() if src is not None else None)
    torch.cuda.synchronize()
    return S.gather_field(), info


def _worker(rank, world, port, name, seed, gaussian, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, info = _slab_solve(name, seed, gaussian, rank, world)
        q.put((rank, x, info.iterations, info.status))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(world, name, seed, gaussian):
    if world == 1:
        x, info = _slab_solve(name, seed, gaussian, 0, 1)
        return x, [info.iterations], [info.status]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, seed, gaussian, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=600) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out[0][1], [o[2] for o in out], [o[3] for o in out]


def _single(name, seed, gaussian):
    cfg, grid, T, load, src = _case(name, seed, gaussian)
    x, info = ops.step(grid, 9.8, 8440 * 410.0, cfg.dt_macro, N.TL_DIRICHLET_BOTTOM, T, g_const=293.0,
                       load=load, gaussian=src.device_args() if src is not None else None, rtol=1e-12)
    return x, info, (grid, T, cfg, load, src)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_global_step_matches_single_gpu_cfg2(world):
    ref, info, _ = _single("cfg2", 0, False)
    x, its, sts = _run_ranks(world, "cfg2", 0, False)
    assert sts == [0] * world and len(set(its)) == 1
    assert its[0] == info.iterations
    assert rel(x, ref) <= 1e-12


def test_slab_global_step_gaussian_vs_oracle_cfg1():
    """Space-mode global step (Gaussian source in the RHS), 2 ranks, against the oracle."""
    _, info, (grid, T, cfg, _, src) = _single("cfg1_m4", 3, True)
    x, its, sts = _run_ranks(2, "cfg1_m4", 3, True)
    g = np.full(grid.n_nodes, 293.0)
    ref, oits = _oracle_step(grid, N.TL_DIRICHLET_BOTTOM, T, cfg.dt_macro, g, gauss=(cfg.beam, src.center))
    assert sts == [0, 0] and its[0] == its[1] and abs(its[0] - oits) <= 1
    assert rel(x, ref) <= 1e-12


def test_slab_single_rank_cfg3_streaming_size():
    """HBM-sized grid (cfg3 global, 6.9M nodes) on one rank: same result as the fused solve."""
    ref, info, _ = _single("cfg3", 0, False)
    x, its, sts = _run_ranks(1, "cfg3", 0, False)
    assert sts == [0] and its[0] == info.iterations
    assert rel(x, ref) <= 1e-12


def test_slab_solve_at_the_iteration_limit_follows_scipy():
    """The device-resident slab CG stops like scipy's cg: with maxiter = the iterations the
    solve needs it reports failure, with one more it converges (same rule as the fused
    kernels, tests/test_gpu_parity.py::test_linear_cg_at_the_iteration_limit_follows_scipy)."""
    import torch
    cfg, grid, T, load, _ = _case("cfg1_m4", 0, False)
    _, info, _ = _single("cfg1_m4", 0, False)
    its = info.iterations
    for maxiter, status in ((its, N.TL_SOLVE_MAXITER), (its + 1, N.TL_SOLVE_OK), (2, N.TL_SOLVE_MAXITER)):
        S = SL.SlabGlobalSolver(grid, 9.8, 8440 * 410.0, rank=0, world=1, device="cuda:0", rtol=1e-12,
                                maxiter=maxiter)
        S.set_own(S.x, T)
        S.set_own(S.load, load)
        got = S.step(cfg.dt_macro, 293.0, with_load=True)
        torch.cuda.synchronize()
        assert got.status == status and got.iterations == min(maxiter, its), (maxiter, its, got)


# ---- whole multirate runs with the global grid on slabs ----------------------------

def _run_worker(rank, world, port, name, n_steps, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = P.load_config(CONFIGS / f"{name}.cfg")
        state, stats = P.two_level_run_slabs(cfg, n_steps=n_steps, device=0)
        if state is None:
            q.put((rank, None))
        else:
            q.put((rank, (state.global_field.values, state.local_field.values,
                          tuple(state.local_field.mesh.placement.offset), dict(stats.counters))))
    finally:
        dist.destroy_process_group()


def _slab_run(world, name, n_steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_worker, args=(r, world, port, name, n_steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=1200) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    have = [r for r in range(world) if out[r] is not None]
    assert len(have) == 1          # the rank that ran the last step's local part
    return out[have[0]]


@pytest.mark.parametrize("world,name,n_steps", [(1, "cfg1_m4", 12), (2, "cfg1_m4", None), (3, "cfg2", 6)])
def test_slab_multirate_run_matches_single_gpu(world, name, n_steps):
    """Global grid split over ranks (device-resident CG), local steps pipelined over the
    ranks in time (chain c on rank c mod world, re-anchored from the global planes): same
    fields, relocations and RunStats counters as the single-GPU run; melt masks."""
    cfg = P.load_config(CONFIGS / f"{name}.cfg")
    ref, ref_stats = P.two_level_run(cfg, n_steps=n_steps)
    gv, lv, off, counters = _slab_run(world, name, n_steps)
    assert off == tuple(ref.local_field.mesh.placement.offset)
    assert counters == dict(ref_stats.counters)
    assert rel(gv, ref.global_field.values) <= 1e-11
    assert rel(lv, ref.local_field.values) <= 1e-11
    TL = cfg.material.T_liquidus
    assert_mask(f"slab run {name} x{world} local", lv, ref.local_field.values, TL)
    assert_mask(f"slab run {name} x{world} global", gv, ref.global_field.values, TL)

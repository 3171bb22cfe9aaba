"""Host-side multi-rank logic on CPU (gloo, world_size 2): scenario sharding (config 5)
and the max-over-ranks timing reduction bench.py uses (bench.env_rank / all_reduce MAX)."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import torch
from paper_2110_12932_b200 import scenarios as S


def test_cfg5_draw_matches_survey_probe():
    """SURVEY Probe P10: seed 0 gives m counts {5: 24, 10: 23, 20: 17}, 418-980 macro
    steps per scenario, 37,853 in total, 2.31e11 DOF-timesteps."""
    sc = S.draw(0, 64)
    counts = {m: sum(s.micro == m for s in sc) for m in (5, 10, 20)}
    assert counts == {5: 24, 10: 23, 20: 17}
    assert min(s.n_macro for s in sc) == 418 and max(s.n_macro for s in sc) == 980
    assert sum(s.n_macro for s in sc) == 37853
    assert sum(s.dof_timesteps for s in sc) == pytest.approx(2.31e11, rel=5e-3)


def test_scenario_config_loads():
    s = S.draw()[7]
    cfg = s.config()
    assert cfg.micro_steps == s.micro and cfg.beam.power == s.power
    assert abs(cfg.path.segments[0].start[1] - (1.5e-3 - 2 * s.hatch)) < 1e-15
    assert abs(cfg.t_end / 2e-5 - s.n_macro) < 1e-9


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_is_a_balanced_partition(world):
    sc = S.draw()
    parts = [S.shard(sc, r, world) for r in range(world)]
    idx = sorted(s.index for p in parts for s in p)
    assert idx == list(range(64))
    loads = [sum(s.dof_timesteps for s in p) for p in parts]
    assert max(loads) - min(loads) <= max(s.dof_timesteps for s in sc)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        r, w, lr = bench.env_rank()
        mine = S.shard(S.draw(), r, w)
        gathered = [None] * w
        dist.all_gather_object(gathered, [s.index for s in mine])
        t = torch.tensor([10.0 * (r + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tmax = float(t.item())
        t = torch.tensor([float(sum(s.dof_timesteps for s in mine))], dtype=torch.float64)
        dist.all_reduce(t)
        total = float(t.item())
        q.put((r, gathered, tmax, total))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_reduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, gathered, tmax, total in out:
        assert sorted(i for g in gathered for i in g) == list(range(64))
        assert tmax == 20.0
        assert total == sum(s.dof_timesteps for s in S.draw())


# ---- z-slab decomposition of the global solve: host logic (partition, halos, sums) ----

from paper_2110_12932_b200 import slab as SL  # noqa: E402


@pytest.mark.parametrize("planes,world", [(41, 1), (41, 2), (41, 3), (201, 8), (8, 8)])
def test_plane_partition_covers_and_balances(planes, world):
    parts = SL.plane_partition(planes, world)
    assert parts[0][0] == 0 and parts[-1][1] == planes
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    sizes = [k1 - k0 for k0, k1 in parts]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    for r, (k0, k1) in enumerate(parts):
        h0, h1 = SL.stored_planes(k0, k1, planes)
        assert h0 == (k0 - 1 if r > 0 else 0) and h1 == (k1 + 1 if r < world - 1 else planes)


def test_plane_partition_rejects_more_ranks_than_planes():
    with pytest.raises(ValueError):
        SL.plane_partition(4, 5)


def _halo_worker(rank, world, port, q):
    import numpy as np
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, nxy = 11, 6
        k0, k1 = SL.plane_partition(nz, world)[rank]
        h0, h1 = SL.stored_planes(k0, k1, nz)
        buf = torch.full(((h1 - h0) * nxy,), -1.0, dtype=torch.float64)
        for k in range(k0, k1):   # own plane k holds 100 k + column index
            buf[(k - h0) * nxy:(k - h0 + 1) * nxy] = 100.0 * k + torch.arange(nxy, dtype=torch.float64)
        SL.HaloExchange(rank, world, k0, k1, h0, nxy).exchange(buf)
        planes = buf.view(h1 - h0, nxy).numpy()
        ok = all(np.array_equal(planes[k - h0], 100.0 * k + np.arange(nxy)) for k in range(h0, h1))
        # rank-ordered sums: rank r contributes (r + 1) * [1e16, 1, -1e16, 0.5]
        sums = torch.tensor([1e16, 1.0, -1e16, 0.5], dtype=torch.float64) * (rank + 1)
        tot = SL.rank_sum(sums, world)
        q.put((rank, ok, tot.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange_and_rank_ordered_sums(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in out)
    tots = [tot for _, _, tot in out]
    assert all(t == tots[0] for t in tots)          # bitwise the same on every rank
    expect = [0.0] * 4
    for r in range(world):                            # the rank order is the summation order
        expect = [e + v * (r + 1) for e, v in zip(expect, [1e16, 1.0, -1e16, 0.5])]
    assert tots[0] == expect


# ---- the multi-GPU two-level driver: chains, super-steps, device-side sums -------------

from paper_2110_12932_b200 import multirate_dist as MD  # noqa: E402


def test_chain_ranks_every_step_relocates():
    """BASELINE configs move the box after every step: every step starts a chain and the
    chains go round-robin over the ranks."""
    starts, ranks, used = MD.chain_ranks(True, [True] * 5, 0, 3)
    assert starts == [True] * 5 and ranks == [0, 1, 2, 0, 1] and used == 5
    starts, ranks, used = MD.chain_ranks(True, [True] * 3, 7, 4)
    assert ranks == [3, 0, 1] and used == 3


def test_chain_ranks_keep_non_relocating_steps_together():
    """A step after which the box does not move continues its chain on the same rank (its
    local field carries over, multirate.py:184-190)."""
    starts, ranks, used = MD.chain_ranks(True, [False, True, False, False, True], 0, 2)
    assert starts == [True, False, True, False, False]
    assert ranks == [0, 0, 1, 1, 1] and used == 2
    starts, ranks, used = MD.chain_ranks(False, [True, True], 4, 2)   # continues chain 3
    assert starts == [False, True] and ranks == [1, 0] and used == 1


@pytest.mark.parametrize("world", [1, 2, 4])
def test_plan_superstep_covers_world_chains(world):
    """A super-step holds exactly `world` whole chains (one per rank) and consecutive
    super-steps tile the schedule with the same plans as one-step planning."""
    import paper_2110_12932_b200 as P
    from paper_2110_12932_b200.schedule import plan_spacetime
    from .conftest import CONFIGS
    cfg = P.load_config(CONFIGS / "cfg1_m4.cfg")
    problem, lm = P.build_problem(cfg)
    sched = P.MacroSchedule(cfg.dt_macro, cfg.micro_steps, 0.0, cfg.t_end)
    state, moved_before, got = (lm.placement, 0.0, 0.0, 0), True, []
    while True:
        plans, nxt = MD.plan_superstep(problem, sched, cfg.path, cfg.policy, *state, world, moved_before)
        if not plans:
            break
        starts, ranks, used = MD.chain_ranks(moved_before, [bool(p.moved[0]) for p in plans], 0, world)
        assert used <= world and (used == world or nxt[3] == sched.n_macro)
        assert sorted(set(ranks)) == list(range(used))
        got.extend(plans)
        moved_before = bool(plans[-1].moved[0])
        state = nxt
    assert len(got) == sched.n_macro
    placement, tg, tl = lm.placement, 0.0, 0.0
    for k, pl in enumerate(got):
        ref = plan_spacetime(problem, sched, placement, cfg.path, cfg.policy, tg, tl, k0=k, nsteps=1)
        assert pl.macro.tobytes() == ref.macro.tobytes() and pl.micro.tobytes() == ref.micro.tobytes()
        placement, tg, tl = ref.final_placement, ref.final_t_global, ref.final_t_local


def _comm_worker(rank, world, port, q):
    import numpy as np
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz, nxy = 9, 4
        k0, k1 = SL.plane_partition(nz, world)[rank]
        h0, h1 = SL.stored_planes(k0, k1, nz)
        comm = SL.SlabComm(rank, world, k0, k1, h0, nxy)
        sums = torch.arange(SL.SUMS, dtype=torch.float64) + 10.0 * rank
        gath = torch.zeros(world * SL.SUMS, dtype=torch.float64)
        comm.allgather(sums, gath)
        ok_g = np.array_equal(gath.numpy().reshape(world, SL.SUMS),
                              np.stack([np.arange(SL.SUMS) + 10.0 * r for r in range(world)]))
        buf = torch.full(((h1 - h0) * nxy,), -1.0, dtype=torch.float64)
        for k in range(k0, k1):
            buf[(k - h0) * nxy:(k - h0 + 1) * nxy] = float(k)
        comm.halo_wait(comm.halo_start(buf))
        ok_h = all(np.all(buf.view(h1 - h0, nxy).numpy()[k - h0] == k) for k in range(h0, h1))
        q.put((rank, ok_g, ok_h))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_comm_allgather_rank_order_and_halo(world):
    """SlabComm: every rank's 8 partial sums land in rank order in the gather buffer the
    kernels read; halo start/wait fills each stored halo plane with the neighbour's plane."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(g and h for _, g, h in out)

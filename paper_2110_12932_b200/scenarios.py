"""BASELINE config 5: batched scan scenarios and their sharding across ranks.

64 independent runs of the config-2 geometry with parameters drawn from
``numpy.random.default_rng(0)`` in the order fixed by SURVEY.md §8(d):
P ~ U[150, 300] W, v ~ U[0.5, 1.2] m/s, r ~ U[35, 70] um, eta ~ U[0.30, 0.45],
hatch ~ U[80, 120] um, m = rng.choice([5, 10, 20]); the path starts at
(0.5, 1.5 - 2 hatch, 1.0) mm and t_end = ceil((10 mm / v) / 20 us) * 20 us
(``lpbfsim/config.py:457-459`` requires whole macro steps).

Scenarios are independent, so multi-GPU execution is scenario sharding (one group
per GPU, no data-path collective): ``shard`` balances DOF-timestep work across
ranks with a deterministic longest-processing-time assignment.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .config import ExperimentConfig, config_from_text

CFG2_NODES = (600_281, 520_251)          # global, local nodes of the config-2 geometry
DT_MACRO = 2e-5


@dataclass(frozen=True)
class Scenario:
    index: int
    power: float
    speed: float
    radius: float
    absorptivity: float
    hatch: float
    micro: int

    @property
    def t_end(self) -> float:
        n = math.ceil((10e-3 / self.speed) / DT_MACRO - 1e-9)
        return n * DT_MACRO

    @property
    def n_macro(self) -> int:
        return int(round(self.t_end / DT_MACRO))

    @property
    def dof_timesteps(self) -> int:
        ng, nl = CFG2_NODES
        return self.n_macro * (ng + self.micro * nl)

    def config(self, base_dir=None) -> ExperimentConfig:
        """The scenario as an ExperimentConfig (config-2 geometry, reference .cfg format)."""
        base = Path(base_dir) if base_dir is not None else Path(__file__).resolve().parent.parent / "configs"
        return config_from_text(self.config_text(base), base, f"cfg5_{self.index}")

    def config_text(self, base_dir=None) -> str:
        """The scenario's .cfg text (readable by the reference's own ``load_config`` too)."""
        base = Path(base_dir) if base_dir is not None else Path(__file__).resolve().parent.parent / "configs"
        text = (base / "cfg2.cfg").read_text()
        y0 = 1.5 - 2 * self.hatch * 1e3
        repl = {
            "power 200": f"power {self.power!r}",
            "absorptivity 0.35": f"absorptivity {self.absorptivity!r}",
            "radius 0.05 mm": f"radius {self.radius!r}",
            "speed 800 mm/s": f"speed {self.speed!r}",
            "hatch 0.1 mm": f"hatch {self.hatch!r}",
            "origin 0.5 1.3 1.0 mm": f"origin 0.5 {y0!r} 1.0 mm",
            "t_end 12.5 ms": f"t_end {self.t_end!r}",
            "micro_steps 10": f"micro_steps {self.micro}",
        }
        for a, b in repl.items():
            assert a in text, a
            text = text.replace(a, b)
        return text


def draw(seed: int = 0, n: int = 64) -> list[Scenario]:
    rng = np.random.default_rng(seed)
    P = rng.uniform(150.0, 300.0, n)
    v = rng.uniform(0.5, 1.2, n)
    r = rng.uniform(35e-6, 70e-6, n)
    eta = rng.uniform(0.30, 0.45, n)
    hatch = rng.uniform(80e-6, 120e-6, n)
    m = rng.choice([5, 10, 20], n)
    return [Scenario(i, float(P[i]), float(v[i]), float(r[i]), float(eta[i]), float(hatch[i]), int(m[i]))
            for i in range(n)]


def shard(scenarios: list[Scenario], rank: int, world: int) -> list[Scenario]:
    """Deterministic LPT assignment by DOF-timestep work; every scenario on exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    load = [0] * world
    owner = {}
    for s in sorted(scenarios, key=lambda s: (-s.dof_timesteps, s.index)):
        k = min(range(world), key=lambda w: (load[w], w))
        owner[s.index] = k
        load[k] += s.dof_timesteps
    return [s for s in scenarios if owner[s.index] == rank]

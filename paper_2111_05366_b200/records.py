"""Option and result records of the drop-in API.

Same field names, defaults and validation errors as the reference records
(MatchOptions matcher.py:32-66, MatchResult :69-78, SeedSet :81-97,
SinkhornParams sinkhorn.py:21-40, SinkhornResult :43-50, LapSolution
lap.py:32-36), so code written against ``otmatch`` constructs them unchanged.
Two fields are added *after* the reference's, with defaults that keep the
reference's arithmetic: ``MatchOptions.precision`` ("fp64" = float64
throughout, "fp32" = fp32 iterate with fp64 potentials/accumulators) and
``MatchOptions.device`` (CUDA ordinal).  ``MatchResult.diagnostics`` carries
what the reference computes but discards (per-LOT sweeps, phase times).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

STEP_SOLVERS = ("exact_lap", "lot")
SENSES = ("minimize", "maximize")
INITS = ("barycenter", "randomized_blend")
PRECISIONS = ("fp64", "fp32")


@dataclass(frozen=True)
class SinkhornParams:
    """Entropic regularisation (reg = 1/lam on the unit-range cost) and stopping rule."""

    lam: float = 100.0
    max_sweeps: int = 1000
    tol: float = 1e-8

    def __post_init__(self):
        if not self.lam > 0:
            raise ValueError("lam must be positive")
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be at least 1")
        if not self.tol > 0:
            raise ValueError("tol must be positive")


@dataclass(frozen=True)
class SinkhornResult:
    matrix: np.ndarray
    converged: bool
    sweeps: int
    deviation: float


@dataclass(frozen=True)
class LapSolution:
    assignment: np.ndarray
    objective: float


@dataclass(frozen=True)
class MatchOptions:
    """FAQ (step_solver="exact_lap") or GOAT (step_solver="lot") configuration."""

    step_solver: str = "exact_lap"
    sinkhorn: SinkhornParams = field(default_factory=SinkhornParams)
    init: object = "barycenter"
    max_iters: int = 30
    fw_tol: float = 1e-2
    n_restarts: int = 1
    shuffle_input: bool = False
    rng_seed: int = 0
    objective_sense: str = "maximize"
    precision: str = "fp64"
    device: int = 0

    def __post_init__(self):
        if self.step_solver not in STEP_SOLVERS:
            raise ValueError(f"step_solver must be one of {STEP_SOLVERS}")
        if self.objective_sense not in SENSES:
            raise ValueError(f"objective_sense must be one of {SENSES}")
        if isinstance(self.init, str) and self.init not in INITS:
            raise ValueError(f"init must be one of {INITS} or a doubly stochastic matrix")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if not self.fw_tol > 0:
            raise ValueError("fw_tol must be positive")
        if self.n_restarts < 1:
            raise ValueError("n_restarts must be at least 1")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")


@dataclass(frozen=True)
class MatchResult:
    alignment: np.ndarray
    objective: float
    iterations: int
    iterate_history: list
    converged: bool
    wall_time: float
    diagnostics: dict = field(default=None, compare=False, repr=False)


@dataclass(frozen=True)
class SeedSet:
    """Known (G1 vertex, G2 vertex) correspondences."""

    pairs: np.ndarray

    def __post_init__(self):
        pairs = np.asarray(self.pairs, dtype=np.intp).reshape(-1, 2)
        object.__setattr__(self, "pairs", pairs)
        for side in range(2):
            if np.unique(pairs[:, side]).size != pairs.shape[0]:
                raise ValueError("duplicate vertex in seed set")

    @property
    def count(self) -> int:
        return int(self.pairs.shape[0])

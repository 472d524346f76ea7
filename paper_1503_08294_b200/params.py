"""Run parameters and small value types shared by the host API.

Mirrors the reference's host-side types field for field so existing calling
code keeps working:
  EngineParams   pkg/src/growsurf/engine.py:38-95
  WinnerResult   pkg/src/growsurf/engine.py:122-146
  BatchOutcome   pkg/src/growsurf/multi.py:35-41
  batch_size     pkg/src/growsurf/multi.py:44-55
  RingClass      pkg/src/growsurf/network.py:34-44
  StateError / UnknownUnitError   pkg/src/growsurf/network.py:26-31
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

__all__ = [
    "EngineParams",
    "WinnerResult",
    "BatchOutcome",
    "batch_size",
    "RingClass",
    "StateError",
    "UnknownUnitError",
]


class UnknownUnitError(KeyError):
    """An operation referenced an id that is not alive in the network."""


class StateError(RuntimeError):
    """The operation is invalid for the current network state."""


class RingClass(Enum):
    """Shape of the subgraph induced on a unit's neighbours."""

    DISK = "disk"
    HALF_DISK = "half-disk"
    INCONSISTENT = "inconsistent"


# device encoding of RingClass (csrc/growsurf_b200.cuh RING_*)
RING_FROM_CODE = (RingClass.DISK, RingClass.HALF_DISK, RingClass.INCONSISTENT)


@dataclass
class EngineParams:
    """Run parameters; validation identical to engine.py:71-91."""

    eps_b: float = 0.1
    eps_n: float = 0.01
    theta0: float = 0.2
    max_age: int = 200
    tau_b: float = 0.05
    tau_n: float = 0.005
    h_t: float = 0.3
    rho: float = 0.8
    ring_patience: int = 500
    max_signals: int = 5_000_000
    allow_boundary: bool = False
    batch_cap: int = 8192
    batch_floor: int = 64
    cube: float | None = None
    stale_factor: int = 30

    def __post_init__(self):
        if not (0.0 <= self.eps_n < self.eps_b <= 1.0):
            raise ValueError("need 0 <= eps_n < eps_b <= 1")
        if not (self.theta0 > 0.0 and math.isfinite(self.theta0)):
            raise ValueError("theta0 must be positive and finite")
        if self.max_age < 0:
            raise ValueError("max_age must be >= 0")
        for name in ("tau_b", "tau_n", "h_t", "rho"):
            v = getattr(self, name)
            if not (0.0 < v < 1.0):
                raise ValueError(f"{name} must lie in (0, 1), got {v}")
        if self.ring_patience < 1:
            raise ValueError("ring_patience must be >= 1")
        if self.max_signals < 1:
            raise ValueError("max_signals must be >= 1")
        if not (1 <= self.batch_floor <= self.batch_cap):
            raise ValueError("need 1 <= batch_floor <= batch_cap")
        if self.cube is not None and not (self.cube > 0.0):
            raise ValueError("cube must be positive")
        if self.stale_factor < 1:
            raise ValueError("stale_factor must be >= 1")

    @property
    def grid_cube(self) -> float:
        return self.theta0 if self.cube is None else self.cube


class WinnerResult:
    """Nearest (winner) and second-nearest unit ids with Euclidean distances."""

    __slots__ = ("winner", "second", "d_winner", "d_second")

    def __init__(self, winner: int, second: int, d_winner: float, d_second: float):
        self.winner = winner
        self.second = second
        self.d_winner = d_winner
        self.d_second = d_second

    def __repr__(self):
        return (
            f"WinnerResult(winner={self.winner}, second={self.second}, "
            f"d_winner={self.d_winner!r}, d_second={self.d_second!r})"
        )

    def __eq__(self, other):
        return (
            isinstance(other, WinnerResult)
            and self.winner == other.winner
            and self.second == other.second
            and self.d_winner == other.d_winner
            and self.d_second == other.d_second
        )


@dataclass(frozen=True)
class BatchOutcome:
    """Accounting for one resolved batch: processed + discarded = m."""

    processed: int
    discarded: int
    inserted_units: int


def batch_size(units: int, cap: int = 8192, floor: int = 64) -> int:
    """Smallest power of two strictly above ``units``, clamped to [floor, cap]."""
    if units < 0:
        raise ValueError("unit count must be >= 0")
    if not (1 <= floor <= cap):
        raise ValueError("need 1 <= floor <= cap")
    return min(max(1 << int(units).bit_length(), floor), cap)

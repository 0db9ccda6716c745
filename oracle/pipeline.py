"""SM-pool slowdown model of the oracle (test infrastructure only).

Restates SPEC.md:481-499 / 535-536: ``gemm_duration = base / (1 - Σ
reservations)``, ``NoSmAvailable`` when nothing is left.  The build measures the
slowdown of a concurrent cuBLAS GEMM instead of modelling it; this is the
reference's *prediction* the measurement is reported against (NCCL-style
intra-host P2P reserves 0.232 of the SMs -> +30%).
"""
from __future__ import annotations

from typing import Dict

from .des import SimulationError

P2P_SM_FRACTION_INTRA_HOST = 0.232
P2P_SM_FRACTION_INTER_HOST = 0.032


class NoSmAvailable(SimulationError):
    """Reservations leave no SMs."""


def gemm_duration(base: float, reservations: Dict[str, float]) -> float:
    avail = 1.0 - sum(reservations.values())
    if avail <= 0:
        raise NoSmAvailable(f"available fraction {avail}")
    return base / avail

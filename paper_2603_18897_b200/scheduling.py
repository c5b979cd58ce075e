"""Admission-scoring surface of the speculation scheduler.

Mirrors the parts of ``spectool/scheduling.py`` on the hot path: ``Job``
with its utility ``U = (p * T) / (c * d)`` (scheduling.py:34-60), the EWMA
``EstimateBook`` (:187-225) and ``greedy_speculative_selection``
(:242-258), which runs on the device (K6).  The event-driven Scheduler state
machine itself is sequential by contract and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Any, Iterable

from .policy import SpecLevel


class JobKind(str, Enum):
    AUTHORITATIVE = "authoritative"
    SPECULATIVE = "speculative"


class JobState(str, Enum):
    PENDING = "pending"
    RUNNING = "running"
    PROMOTED = "promoted"
    COMPLETED = "completed"
    ABORTED = "aborted"


@dataclass
class Job:
    id: int
    kind: JobKind
    tool_type: str
    args: Any
    arg_hash: str
    session_id: str
    p: float
    benefit_ms: float
    cost: int
    duration_est_ms: float
    submitted_at: float
    level: SpecLevel | None = None
    no_commit: bool = False
    state: JobState = JobState.PENDING
    preemptible: bool = False
    dispatched_at: float | None = None
    finished_at: float | None = None
    result: Any = None
    ok: bool = False
    consumed: bool = False

    def utility(self) -> float:
        return (self.p * self.benefit_ms) / (self.cost * self.duration_est_ms)


class EstimateBook:
    """Per-tool EWMA duration estimates (alpha * sample + (1 - alpha) * current)."""

    def __init__(self, alpha: float = 0.5, default_duration_ms: float = 1000.0,
                 warm_fraction: float = 0.2, costs: dict[str, int] | None = None):
        if not 0 < alpha <= 1:
            raise ValueError("alpha must be in (0, 1]")
        self.alpha = alpha
        self.default_duration_ms = default_duration_ms
        self.warm_fraction = warm_fraction
        self.costs = dict(costs or {})
        self._duration: dict[str, float] = {}
        self._stall_saved: dict[str, float] = {}

    def update(self, tool_type: str, duration_ms: float | None = None,
               stall_saved_ms: float | None = None) -> None:
        if duration_ms is not None:
            self._duration[tool_type] = self._ewma(self._duration.get(tool_type), duration_ms)
        if stall_saved_ms is not None:
            self._stall_saved[tool_type] = self._ewma(self._stall_saved.get(tool_type),
                                                      stall_saved_ms)

    def _ewma(self, current: float | None, sample: float) -> float:
        return sample if current is None else self.alpha * sample + (1 - self.alpha) * current

    def duration(self, tool_type: str) -> float:
        return self._duration.get(tool_type, self.default_duration_ms)

    def stall_saved(self, tool_type: str) -> float:
        return self._stall_saved.get(tool_type, 0.0)

    def cost(self, tool_type: str) -> int:
        return self.costs.get(tool_type, 1)


def greedy_speculative_selection(jobs: Iterable[Job], slack: int, budget: int) -> list[Job]:
    """Jobs in (-U, -p, id) order, taken while cost fits both the remaining
    slack and budget (device top-k + scan, K6)."""
    from .select import greedy_select_jobs

    return greedy_select_jobs(list(jobs), slack, budget)

"""Runtime prediction surface: windows, predicted invocations, Predictor.

Mirrors ``spectool/prediction.py``.  ``Predictor.predict`` (prediction.py:76-118)
and ``score_accuracy`` (:133-169) run through the device predict kernel (K4):
the pool is compiled once per Predictor into a device-resident image whose
buckets are pre-ranked by ``(-p, pattern_id)``, and every call ships the
window's tokens and payload tapes to the GPU.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from enum import Enum
from typing import Any, Sequence

from .events import Event, EventKind, Session

DEFAULT_WINDOW_CAPACITY = 16


class Completeness(str, Enum):
    FULL = "full"
    PARTIAL = "partial"
    TOOL_ONLY = "tool_only"


@dataclass(frozen=True)
class PredictedInvocation:
    tool_type: str
    args: dict[str, Any]
    completeness: Completeness
    probability: float
    source_pattern: str
    created_at: float


class PredictionWindow:
    """Bounded per-session view of recent events (deque with maxlen)."""

    def __init__(self, capacity: int = DEFAULT_WINDOW_CAPACITY):
        if capacity < 1:
            raise ValueError("window capacity must be >= 1")
        self._events: deque[Event] = deque(maxlen=capacity)

    @property
    def capacity(self) -> int:
        return self._events.maxlen  # type: ignore[return-value]

    def observe(self, event: Event) -> None:
        self._events.append(event)

    def events(self) -> tuple[Event, ...]:
        return tuple(self._events)

    def tool_events(self) -> tuple[Event, ...]:
        return tuple(e for e in self._events if e.kind is EventKind.TOOL_CALL)

    def __len__(self) -> int:
        return len(self._events)


@dataclass
class PredictDiagnostics:
    structural_errors: int = 0


class Predictor:
    """Matches a pattern pool against session windows on the device."""

    def __init__(self, pool):
        from .device_ops import DevicePool

        self.pool = pool
        self.diagnostics = PredictDiagnostics()
        self._device = DevicePool(pool)

    def predict(self, window: PredictionWindow, now: float | None = None,
                max_candidates: int | None = None) -> list[PredictedInvocation]:
        return self.predict_batch([window], now=now, max_candidates=max_candidates)[0]

    def predict_batch(self, windows: Sequence[PredictionWindow], now: float | None = None,
                      max_candidates: int | None = None) -> list[list[PredictedInvocation]]:
        """One kernel launch for many windows; same result as calling
        :meth:`predict` on each."""
        preds, errs = self._device.predict_windows([w.events() for w in windows], now,
                                                   max_candidates)
        self.diagnostics.structural_errors += errs
        return preds

    def predict_admit_batch(self, windows: Sequence[PredictionWindow], policy, estimates,
                            now: float | None = None, max_candidates: int | None = 8):
        """Fused predict + admit with ``benefit = estimates.duration(tool)``
        (the simulator's live path, simulation.py:425-429)."""
        preds, actions, errs = self._device.predict_admit_windows(
            [w.events() for w in windows], policy, estimates, now, max_candidates)
        self.diagnostics.structural_errors += errs
        return preds, actions


@dataclass(frozen=True)
class AccuracyReport:
    top1: float
    top3: float
    hit_rate: float
    scored_calls: int

    def to_json(self) -> dict[str, Any]:
        return {"top1": self.top1, "top3": self.top3, "hit_rate": self.hit_rate,
                "scored_calls": self.scored_calls}


def score_accuracy(traces: Sequence[Session], pool, window_capacity: int = DEFAULT_WINDOW_CAPACITY,
                   max_candidates: int | None = None) -> AccuracyReport:
    """Replay: before each tool call after the first, predict from the window
    (LLM steps occupy window slots); score top-1 / top-3 / full-argument hit
    (prediction.py:133-169).  All windows of the corpus are predicted in one
    device batch; the hit test compares canonical argument forms."""
    from .device_ops import score_replay

    return score_replay(traces, pool, window_capacity, max_candidates)

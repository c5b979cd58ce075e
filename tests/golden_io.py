"""Rebuild this package's objects from the golden fixtures (tests/golden/)."""

from __future__ import annotations

import io
import json
import os

from paper_2603_18897_b200.events import Event, EventKind, Session, Status
from paper_2603_18897_b200.mining import load_pool
from paper_2603_18897_b200.policy import SpecLevel, SpeculationPolicy, ToolRule
from paper_2603_18897_b200.scheduling import EstimateBook

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache: dict[str, dict] = {}


def golden(name: str) -> dict:
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".gz"):
            import gzip
            with gzip.open(path, "rt", encoding="utf-8") as fh:
                _cache[name] = json.load(fh)
        else:
            with open(path, encoding="utf-8") as fh:
                _cache[name] = json.load(fh)
    return _cache[name]


def event(d: dict) -> Event:
    return Event(d["session_id"], d["seq"], EventKind(d["kind"]), d["tool"], Status(d["status"]),
                 d["args"], d["result"], d["t_start_ms"], d["t_end_ms"])


def session(d: dict) -> Session:
    return Session(d["id"], tuple(event(e) for e in d["events"]))


def pool(obj: dict):
    return load_pool(io.StringIO(json.dumps(obj)))


def policy(obj: dict | None) -> SpeculationPolicy | None:
    if obj is None:
        return None
    return SpeculationPolicy(default_allow=obj["default_allow"],
                             default_level=SpecLevel(obj["default_level"]),
                             tool_rules={t: ToolRule(a, SpecLevel(l))
                                         for t, (a, l) in obj["tools"].items()})


def estimates(obj: dict | None) -> EstimateBook | None:
    if obj is None:
        return None
    book = EstimateBook(default_duration_ms=obj["default"])
    book._duration.update(obj["tools"])
    return book


def pred_dict(p) -> dict:
    return {"tool": p.tool_type, "args": p.args, "completeness": p.completeness.value,
            "p": p.probability, "pattern": p.source_pattern, "created_at": p.created_at}


def same(a, b) -> bool:
    """Structural equality that also distinguishes 1 / 1.0 / True (JSON
    round trips keep the distinction; Python == does not)."""
    if type(a) is not type(b):
        return False
    if isinstance(a, dict):
        return list(a) == list(b) and all(same(a[k], b[k]) for k in a)
    if isinstance(a, list):
        return len(a) == len(b) and all(same(x, y) for x, y in zip(a, b))
    if isinstance(a, float) and a != a:
        return b != b
    return a == b

"""Value mappings: expression types, serialization and device-backed evaluation.

Mirrors ``spectool/mappings.py``.  The expression dataclasses and their JSON /
alias forms (mappings.py:26-133, 431-528) are host-side descriptions; the work
of resolving them against payloads (``evaluate``, mappings.py:207-223), of
enumerating matching leaves (``candidate_paths``, :237-266) and of counting
hypothesis hits (``_holds``, :326-335) runs in libpaste over payload tapes
(:mod:`.tape`).
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from enum import Enum
from typing import Any, Sequence

from .events import Event, EventSignature, Status

DEFAULT_VALIDATION_FRACTION = 0.9
DEFAULT_PATH_NODE_BUDGET = 10_000

PathStep = str | int
Path = tuple[PathStep, ...]


class MappingStructureError(ValueError):
    """A mapping references a context position outside the matched context."""


class Normalization(str, Enum):
    NONE = "none"
    TRIM = "trim"
    LOWERCASE = "lowercase"

    def apply(self, text: str) -> str:
        if self is Normalization.TRIM:
            return text.strip()
        if self is Normalization.LOWERCASE:
            return text.lower()
        return text


@dataclass(frozen=True)
class PathLookup:
    ctx_pos: int
    path: Path

    def __post_init__(self) -> None:
        if not self.path:
            raise ValueError("PathLookup path must be non-empty")


@dataclass(frozen=True)
class IndexedFallback:
    ctx_pos: int
    path_prefix: Path
    start_index: int
    path_suffix: Path
    fail_tool: str

    def __post_init__(self) -> None:
        if self.start_index < 0:
            raise ValueError("IndexedFallback start_index must be >= 0")


@dataclass(frozen=True)
class FormatTemplate:
    prefix: str
    hole: PathLookup
    suffix: str
    normalization: Normalization = Normalization.NONE


MappingExpr = PathLookup | IndexedFallback | FormatTemplate


@dataclass(frozen=True)
class ArgBinding:
    arg_name: str
    expr: MappingExpr


@dataclass(frozen=True)
class ValueMapping:
    bindings: tuple[ArgBinding, ...]

    def arg_names(self) -> tuple[str, ...]:
        return tuple(b.arg_name for b in self.bindings)


class _Unbound:
    def __repr__(self) -> str:  # pragma: no cover
        return "UNBOUND"


UNBOUND = _Unbound()


@dataclass(frozen=True)
class MatchedContext:
    """Matched events (aligned with the context) and the contiguous history
    slice from the first matched event through the anchor."""

    events: tuple[Event, ...]
    history: tuple[Event, ...] = ()

    def __post_init__(self) -> None:
        if not self.history:
            object.__setattr__(self, "history", self.events)


@dataclass(frozen=True)
class MappingResult:
    args: dict[str, Any]
    unbound: tuple[str, ...]

    @property
    def complete(self) -> bool:
        return not self.unbound


@dataclass(frozen=True)
class PathSearch:
    paths: tuple[Path, ...]
    truncated: bool


def expr_ctx_pos(expr: MappingExpr) -> int:
    return expr.hole.ctx_pos if isinstance(expr, FormatTemplate) else expr.ctx_pos


# ---------------------------------------------------------------------------
# Device-backed operations (implemented in .device_ops)
# ---------------------------------------------------------------------------


def evaluate(mapping: ValueMapping, matched: MatchedContext | Sequence[Event]) -> MappingResult:
    """Resolve every binding against the matched events on the device."""
    from .device_ops import evaluate_mapping

    ctx = matched if isinstance(matched, MatchedContext) else MatchedContext(events=tuple(matched))
    return evaluate_mapping(mapping, ctx)


def candidate_paths(payload: Any, target_value: Any,
                    node_budget: int = DEFAULT_PATH_NODE_BUDGET) -> PathSearch:
    """All pre-order paths whose scalar leaf equals ``target_value`` (device leaf scan)."""
    from .device_ops import candidate_paths_batch

    return candidate_paths_batch([payload], [target_value], node_budget)[0]


Occurrence = tuple[MatchedContext, Event]


def infer_mapping(occurrences: Sequence[Occurrence],
                  validation_fraction: float = DEFAULT_VALIDATION_FRACTION) -> ValueMapping | None:
    """Search PathLookup -> IndexedFallback -> FormatTemplate per common scalar
    argument; the first hypothesis holding on >= ``validation_fraction`` of the
    occurrences wins (mappings.py:276-417).  Hypothesis hit counts run on the
    device (:mod:`.phase2`)."""
    from .phase2_device import infer_mapping as _infer

    return _infer(occurrences, validation_fraction)


# ---------------------------------------------------------------------------
# Serialization (host-side wire format; mappings.py:435-528)
# ---------------------------------------------------------------------------

_ALIAS_RE = re.compile(r"^\s*([A-Za-z_][A-Za-z0-9_]*)Res\s*((?:\[[^\]]+\])+)\s*$")
_STEP_RE = re.compile(r"\[([^\]]+)\]")


def expr_to_json(expr: MappingExpr) -> dict[str, Any]:
    if isinstance(expr, PathLookup):
        return {"kind": "path", "ctx": expr.ctx_pos, "path": list(expr.path)}
    if isinstance(expr, IndexedFallback):
        return {"kind": "indexed_fallback", "ctx": expr.ctx_pos,
                "prefix": list(expr.path_prefix), "start": expr.start_index,
                "suffix": list(expr.path_suffix), "fail_tool": expr.fail_tool}
    if isinstance(expr, FormatTemplate):
        return {"kind": "format", "prefix": expr.prefix, "hole": expr_to_json(expr.hole),
                "suffix": expr.suffix, "normalize": expr.normalization.value}
    raise TypeError(f"unknown expression type: {type(expr)!r}")


def _steps_from_json(steps: Sequence[Any]) -> Path:
    return tuple(int(s) if isinstance(s, (int, float)) and not isinstance(s, bool) else str(s)
                 for s in steps)


def expr_from_json(obj: Any, context: Sequence[EventSignature] = ()) -> MappingExpr:
    if isinstance(obj, str):
        return parse_path_alias(obj, context)
    kind = obj.get("kind")
    if kind == "path":
        return PathLookup(ctx_pos=int(obj["ctx"]), path=_steps_from_json(obj["path"]))
    if kind == "indexed_fallback":
        return IndexedFallback(ctx_pos=int(obj["ctx"]), path_prefix=_steps_from_json(obj["prefix"]),
                               start_index=int(obj["start"]),
                               path_suffix=_steps_from_json(obj["suffix"]),
                               fail_tool=str(obj["fail_tool"]))
    if kind == "format":
        hole = expr_from_json(obj["hole"], context)
        if not isinstance(hole, PathLookup):
            raise ValueError("format template hole must be a path lookup")
        return FormatTemplate(prefix=str(obj.get("prefix", "")), hole=hole,
                              suffix=str(obj.get("suffix", "")),
                              normalization=Normalization(obj.get("normalize", "none")))
    raise ValueError(f"unknown mapping expression kind: {kind!r}")


def parse_path_alias(text: str, context: Sequence[EventSignature]) -> PathLookup:
    """``<Tool>Res["key"][0]`` -> PathLookup on the last context position of that
    tool (case-insensitive), successful positions preferred."""
    m = _ALIAS_RE.match(text)
    if m is None:
        raise ValueError(f"unrecognized mapping alias: {text!r}")
    tool, steps_text = m.groups()
    positions = [i for i, sig in enumerate(context) if sig.tool_type.lower() == tool.lower()]
    if not positions:
        raise ValueError(f"alias tool {tool!r} not found in pattern context")
    ok = [i for i in positions if context[i].status is Status.SUCCESS]
    path: list[PathStep] = []
    for raw in _STEP_RE.findall(steps_text):
        raw = raw.strip()
        if any(raw.startswith(q) and raw.endswith(q) for q in "\"'"):
            path.append(raw[1:-1])
        else:
            path.append(int(raw))
    return PathLookup(ctx_pos=(ok or positions)[-1], path=tuple(path))


def mapping_to_json(mapping: ValueMapping) -> list[dict[str, Any]]:
    return [{"arg": b.arg_name, "expr": expr_to_json(b.expr)} for b in mapping.bindings]


def mapping_from_json(obj: Any, context: Sequence[EventSignature] = ()) -> ValueMapping:
    bindings = [ArgBinding(str(item["arg"]), expr_from_json(item["expr"], context)) for item in obj]
    return ValueMapping(bindings=tuple(sorted(bindings, key=lambda b: b.arg_name)))

"""Mining Phase II: value-mapping inference over a candidate's occurrences.

Host-side in this round (SURVEY.md 8(f) row 1 moves the hypothesis hit
counting onto the device).  Semantics follow the reference's search order
exactly (mappings.py:276-417): arguments common to every occurrence and
scalar everywhere, sorted by name; per argument the searchers PathLookup ->
IndexedFallback -> FormatTemplate, each enumerating hypotheses from a seed
occurrence in DFS-leaf order and keeping the first one that reproduces the
actual argument on at least ``fraction`` of the occurrences.
"""

from __future__ import annotations

from typing import Any, Iterator, Sequence

from .events import Event, Status, values_equal
from .mappings import (UNBOUND, ArgBinding, FormatTemplate, IndexedFallback, MappingExpr,
                       MappingStructureError, MatchedContext, Normalization, PathLookup,
                       PathSearch, ValueMapping)
from .tape import leaf_str_of

Occurrence = tuple[MatchedContext, Event]
_NORMS = (Normalization.NONE, Normalization.TRIM, Normalization.LOWERCASE)


# ---------------------------------------------------------------------------
# expression evaluation against concrete events (mappings.py:143-223)
# ---------------------------------------------------------------------------

def walk(payload: Any, path) -> Any:
    node = payload
    for step in path:
        if isinstance(step, int):
            if not (isinstance(node, list) and 0 <= step < len(node)):
                return UNBOUND
        elif not (isinstance(node, dict) and step in node):
            return UNBOUND
        node = node[step]
    return node


def fails_after(history: Sequence[Event], source: Event, fail_tool: str) -> int:
    """FAIL events of ``fail_tool`` after ``source`` (by identity) in history."""
    seen, n = False, 0
    for ev in history:
        if ev is source:
            seen = True
        elif seen and ev.tool_type == fail_tool and ev.status is Status.FAIL:
            n += 1
    return n


def resolve(expr: MappingExpr, ctx: MatchedContext) -> Any:
    if isinstance(expr, FormatTemplate):
        leaf = resolve(expr.hole, ctx)
        text = None if leaf is UNBOUND else leaf_str_of(leaf)
        if text is None:
            return UNBOUND
        return expr.prefix + expr.normalization.apply(text) + expr.suffix
    if not 0 <= expr.ctx_pos < len(ctx.events):
        raise MappingStructureError(f"ctx_pos {expr.ctx_pos} out of range")
    src = ctx.events[expr.ctx_pos]
    if isinstance(expr, PathLookup):
        return walk(src.result, expr.path)
    if isinstance(expr, IndexedFallback):
        idx = expr.start_index + fails_after(ctx.history, src, expr.fail_tool)
        return walk(src.result, expr.path_prefix + (idx,) + expr.path_suffix)
    raise TypeError(f"unknown expression type: {type(expr)!r}")


def holds_fraction(expr: MappingExpr, name: str, occurrences: Sequence[Occurrence]) -> float:
    hits = 0
    for ctx, actual in occurrences:
        try:
            value = resolve(expr, ctx)
        except MappingStructureError:
            return 0.0
        if value is not UNBOUND and values_equal(value, actual.args[name]):
            hits += 1
    return hits / len(occurrences)


def mapping_holds(mapping: ValueMapping, ctx: MatchedContext, actual: Event) -> bool:
    """Every binding resolves and equals the actual argument (mining.py:202-212)."""
    values: dict[str, Any] = {}
    unbound = False
    for b in mapping.bindings:  # evaluate(): later bindings of a name win
        value = resolve(b.expr, ctx)
        if value is UNBOUND:
            unbound = True
        else:
            values[b.arg_name] = value
    args = actual.args
    if unbound or not isinstance(args, dict):
        return False
    return all(name in args and values_equal(v, args[name]) for name, v in values.items())


# ---------------------------------------------------------------------------
# hypothesis generation
# ---------------------------------------------------------------------------

def leaf_paths(payload: Any, target: Any, budget: int = 10_000) -> PathSearch:
    """Pre-order paths to scalar leaves equal to target, node budget as in the
    reference's candidate_paths (mappings.py:237-266)."""
    paths: list = []
    visited = 0
    stack: list[tuple[Any, tuple]] = [(payload, ())]
    while stack:
        node, path = stack.pop()
        visited += 1
        if visited > budget:
            return PathSearch(tuple(paths), True)
        if isinstance(node, dict):
            stack.extend(reversed([(node[k], path + (k,)) for k in node]))
        elif isinstance(node, list):
            stack.extend(reversed([(v, path + (i,)) for i, v in enumerate(node)]))
        elif values_equal(node, target):
            paths.append(path)
    return PathSearch(tuple(paths), False)


def scalar_leaves(payload: Any, path: tuple = ()) -> Iterator[tuple[tuple, Any]]:
    if isinstance(payload, dict):
        for k in payload:
            yield from scalar_leaves(payload[k], path + (k,))
    elif isinstance(payload, list):
        for i, v in enumerate(payload):
            yield from scalar_leaves(v, path + (i,))
    elif path:
        yield path, payload


def source_positions(ctx: MatchedContext) -> Iterator[int]:
    return (i for i, ev in enumerate(ctx.events) if ev.status is Status.SUCCESS)


def _path_lookup(name, occ, fraction):
    ctx0, act0 = occ[0]
    for pos in source_positions(ctx0):
        for path in leaf_paths(ctx0.events[pos].result, act0.args[name]).paths:
            expr = PathLookup(ctx_pos=pos, path=path)  # raises on path == () like the reference
            if holds_fraction(expr, name, occ) >= fraction:
                return expr
    return None


def _indexed_fallback(name, occ, fraction):
    target_tool = occ[0][1].tool_type
    fails = [[fails_after(ctx.history, ev, target_tool) for ev in ctx.events] for ctx, _ in occ]
    seed = min(range(len(occ)), key=lambda i: min(fails[i]) if fails[i] else 0)
    ctx_s, act_s = occ[seed]
    for pos in source_positions(ctx_s):
        n_fail = fails[seed][pos]
        for path in leaf_paths(ctx_s.events[pos].result, act_s.args[name]).paths:
            for cut, step in enumerate(path):
                if not isinstance(step, int) or step - n_fail < 0:
                    continue
                expr = IndexedFallback(ctx_pos=pos, path_prefix=path[:cut],
                                       start_index=step - n_fail, path_suffix=path[cut + 1:],
                                       fail_tool=target_tool)
                if holds_fraction(expr, name, occ) >= fraction:
                    return expr
    return None


def _format_template(name, occ, fraction):
    ctx0, act0 = occ[0]
    actual = act0.args[name]
    if not isinstance(actual, str):
        return None
    for pos in source_positions(ctx0):
        for path, leaf in scalar_leaves(ctx0.events[pos].result):
            text = leaf_str_of(leaf)
            if text is None:
                continue
            for norm in _NORMS:
                hole = norm.apply(text)
                if not hole:
                    continue
                at = actual.find(hole)
                while at != -1:
                    expr = FormatTemplate(prefix=actual[:at], hole=PathLookup(ctx_pos=pos, path=path),
                                          suffix=actual[at + len(hole):], normalization=norm)
                    if holds_fraction(expr, name, occ) >= fraction:
                        return expr
                    at = actual.find(hole, at + 1)
    return None


def common_scalar_args(occ: Sequence[Occurrence]) -> list[str]:
    first = occ[0][1].args
    if not isinstance(first, dict):
        return []
    names = []
    for name in sorted(first):
        if all(isinstance(a.args, dict) and name in a.args
               and not isinstance(a.args[name], (dict, list)) for _, a in occ):
            names.append(name)
    return names


def infer_mapping(occurrences: Sequence[Occurrence], validation_fraction: float = 0.9
                  ) -> ValueMapping | None:
    if len(occurrences) < 2:
        return None
    bindings = []
    for name in common_scalar_args(occurrences):
        for search in (_path_lookup, _indexed_fallback, _format_template):
            expr = search(name, occurrences, validation_fraction)
            if expr is not None:
                bindings.append(ArgBinding(name, expr))
                break
    if not bindings:
        return None
    return ValueMapping(bindings=tuple(sorted(bindings, key=lambda b: b.arg_name)))

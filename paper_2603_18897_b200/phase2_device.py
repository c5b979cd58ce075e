"""Phase II on the device: infer_mapping with K7 hypothesis hit counting.

The reference's search (mappings.py:276-417) is kept verbatim in structure:
common scalar argument names, then per name PathLookup -> IndexedFallback ->
FormatTemplate, each enumerating hypotheses from a seed occurrence in the
reference's order and accepting the first whose hit fraction reaches the
validation fraction.  What moves to the device is the expensive part -- the
hit counts of every hypothesis over every occurrence (``_holds``, K7
``paste_holds``) and the seed's ``candidate_paths`` (K5).  Hypotheses whose
FormatTemplate comparisons involve non-ASCII text come back "unsure" and are
re-evaluated with Python string semantics (phase2.holds_fraction), so the
result is exact.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _native, phase2
from ._native import BINDING_DTYPE, HoldsDesc, check, ptr
from .events import Status
from .mappings import (ArgBinding, FormatTemplate, IndexedFallback, PathLookup, ValueMapping)
from .packing import SigTable, encode_binding
from .tape import KeyTable, TapeArena, scalar_bytes

_NORM_CODE = {"none": 0, "trim": 1, "lowercase": 2}


class OccurrenceSet:
    """One candidate's occurrences packed for the device (tapes of the
    matched events' results, histories, actual arguments)."""

    def __init__(self, occ: Sequence, target_tool: str):
        from .device_ops import to_dev

        self.occ = list(occ)
        self.M = len(self.occ)
        self.n_ctx = len(self.occ[0][0].events)
        self.sigs, self.keys = SigTable(), KeyTable()
        self.sigs.tool(target_tool)
        self.arena = TapeArena(self.keys, keep_objects=False)
        slot: dict[int, int] = {}
        occ_event, src_pos, hist_off, hist_tok = [], [], [0], []
        for ctx, _ in self.occ:
            for ev in ctx.events:
                if id(ev) not in slot:
                    slot[id(ev)] = self.arena.add(ev.result)
                occ_event.append(slot[id(ev)])
                src_pos.append(next((j for j, h in enumerate(ctx.history) if h is ev), -1))
            hist_tok += [self.sigs.sig(h.tool_type, h.status) for h in ctx.history]
            hist_off.append(len(hist_tok))
        nodes, data, refs = self.arena.arrays()
        self.dev = {k: to_dev(v) for k, v in dict(
            nodes=nodes, data=data, refs=refs, occ_event=np.array(occ_event, np.int32),
            src_pos=np.array(src_pos, np.int32), hist_off=np.array(hist_off, np.int32),
            hist_tok=np.array(hist_tok or [0], np.int32)).items()}
        self._actual: dict[str, dict] = {}

    def actual(self, name: str):
        """Canonical form of every occurrence's ``args[name]`` on the device."""
        from .device_ops import to_dev

        if name not in self._actual:
            import unicodedata

            types, nans, chunks = [], [], []
            for _, act in self.occ:
                v = act.args[name]
                try:
                    t, f, b = scalar_bytes(v)
                    if isinstance(v, str):
                        b = unicodedata.normalize("NFC", v).encode("utf-8", "surrogatepass")
                except TypeError:
                    t, f, b = -1, 0, b""
                types.append(t)
                nans.append(1 if f & 4 else 0)
                chunks.append(b)
            off = np.zeros(self.M + 1, np.int64)
            off[1:] = np.cumsum([len(b) for b in chunks])
            self._actual[name] = {k: to_dev(v) for k, v in dict(
                act_type=np.array(types, np.int32), act_nan=np.array(nans, np.uint8),
                act_off=off, act_bytes=np.frombuffer(b"".join(chunks) + b"\0", np.uint8)).items()}
        return self._actual[name]

    def holds(self, exprs: Sequence, name: str, want_eq: bool = False):
        """(hits[H], unsure[H], eq[H, M] or None) for hypotheses ``exprs``."""
        import torch

        from .device_ops import stream_handle, to_dev

        lib = _native.lib()
        H = len(exprs)
        steps: list[int] = []
        rows, fmt, fbytes = [], [], bytearray()
        for e in exprs:
            rows.append(encode_binding(e, self.sigs, self.keys, steps))
            if isinstance(e, FormatTemplate):
                pre = e.prefix.encode("utf-8", "surrogatepass")
                suf = e.suffix.encode("utf-8", "surrogatepass")
                fmt += [len(fbytes), len(pre), len(fbytes) + len(pre), len(suf),
                        _NORM_CODE[e.normalization.value]]
                fbytes += pre + suf
            else:
                fmt += [0, 0, 0, 0, 0]
        a = self.actual(name)
        d = {k: to_dev(v) for k, v in dict(
            hyp=np.array(rows, dtype=BINDING_DTYPE), steps=np.array(steps or [0, 0], np.int32),
            fmt=np.array(fmt, np.int32), fbytes=np.frombuffer(bytes(fbytes) + b"\0", np.uint8)).items()}
        hits = torch.zeros(H, dtype=torch.int64, device="cuda")
        unsure = torch.zeros(H, dtype=torch.int64, device="cuda")
        eq = torch.zeros(H * self.M, dtype=torch.uint8, device="cuda") if want_eq else None
        dv = self.dev
        desc = HoldsDesc(H, self.M, self.n_ctx, 0, ptr(d["hyp"]), ptr(d["steps"]), ptr(d["fmt"]),
                         ptr(d["fbytes"]), ptr(dv["nodes"]), ptr(dv["data"]), ptr(dv["refs"]),
                         ptr(dv["occ_event"]), ptr(dv["src_pos"]), ptr(dv["hist_off"]),
                         ptr(dv["hist_tok"]), ptr(a["act_type"]), ptr(a["act_nan"]),
                         ptr(a["act_off"]), ptr(a["act_bytes"]), ptr(hits), ptr(unsure), ptr(eq))
        check(lib.paste_holds(ctypes.byref(desc), stream_handle()), lib)
        return (hits.cpu().numpy(), unsure.cpu().numpy(),
                eq.view(H, self.M).cpu().numpy() if want_eq else None)


def _first_passing(exprs, err, name, occs: OccurrenceSet, fraction: float):
    """The reference's "first hypothesis with _holds >= fraction"; ``err`` is
    an exception the enumeration hit after the listed hypotheses."""
    if exprs:
        hits, unsure, _ = occs.holds(exprs, name)
        for i, e in enumerate(exprs):
            if unsure[i]:
                frac = phase2.holds_fraction(e, name, occs.occ)  # Unicode string semantics
            else:
                frac = hits[i] / occs.M
            if frac >= fraction:
                return e
    if err is not None:
        raise err
    return None


def _path_hypotheses(name, occs: OccurrenceSet):
    from .device_ops import candidate_paths_batch

    ctx0, act0 = occs.occ[0]
    positions = list(phase2.source_positions(ctx0))
    searches = candidate_paths_batch([ctx0.events[p].result for p in positions],
                                     [act0.args[name]] * len(positions), 10_000)
    out = []
    for pos, search in zip(positions, searches):
        for path in search.paths:
            try:
                out.append(PathLookup(ctx_pos=pos, path=path))
            except ValueError as exc:  # bare scalar result: the reference raises here
                return out, exc
    return out, None


def _fallback_hypotheses(name, occs: OccurrenceSet):
    from .device_ops import candidate_paths_batch

    occ = occs.occ
    target_tool = occ[0][1].tool_type
    fails = [[phase2.fails_after(ctx.history, ev, target_tool) for ev in ctx.events]
             for ctx, _ in occ]
    seed = min(range(len(occ)), key=lambda i: min(fails[i]) if fails[i] else 0)
    ctx_s, act_s = occ[seed]
    positions = list(phase2.source_positions(ctx_s))
    searches = candidate_paths_batch([ctx_s.events[p].result for p in positions],
                                     [act_s.args[name]] * len(positions), 10_000)
    out = []
    for pos, search in zip(positions, searches):
        n_fail = fails[seed][pos]
        for path in search.paths:
            for cut, step in enumerate(path):
                if not isinstance(step, int) or step - n_fail < 0:
                    continue
                out.append(IndexedFallback(ctx_pos=pos, path_prefix=path[:cut],
                                           start_index=step - n_fail, path_suffix=path[cut + 1:],
                                           fail_tool=target_tool))
    return out, None


def _format_hypotheses(name, occs: OccurrenceSet):
    ctx0, act0 = occs.occ[0]
    actual = act0.args[name]
    if not isinstance(actual, str):
        return [], None
    out = []
    for pos in phase2.source_positions(ctx0):
        for path, leaf in phase2.scalar_leaves(ctx0.events[pos].result):
            text = phase2.leaf_str_of(leaf)
            if text is None:
                continue
            for norm in phase2._NORMS:
                hole = norm.apply(text)
                if not hole:
                    continue
                at = actual.find(hole)
                while at != -1:
                    out.append(FormatTemplate(prefix=actual[:at],
                                              hole=PathLookup(ctx_pos=pos, path=path),
                                              suffix=actual[at + len(hole):], normalization=norm))
                    at = actual.find(hole, at + 1)
    return out, None


def _aliased_histories(occurrences) -> bool:
    """True when some history holds the same event object twice (possible only
    in hand-built contexts); _failures_after's identity skip then needs the
    host semantics."""
    for ctx, _ in occurrences:
        ids = [id(e) for e in ctx.history]
        if len(ids) != len(set(ids)):
            return True
    return False


def infer_mapping(occurrences: Sequence, validation_fraction: float = 0.9,
                  occs: OccurrenceSet | None = None) -> ValueMapping | None:
    if len(occurrences) < 2:
        return None
    names = phase2.common_scalar_args(occurrences)
    if not names:
        return None
    if _aliased_histories(occurrences):
        return phase2.infer_mapping(occurrences, validation_fraction)
    occs = occs or OccurrenceSet(occurrences, occurrences[0][1].tool_type)
    bindings = []
    for name in names:
        for gen in (_path_hypotheses, _fallback_hypotheses, _format_hypotheses):
            exprs, err = gen(name, occs)
            expr = _first_passing(exprs, err, name, occs, validation_fraction)
            if expr is not None:
                bindings.append(ArgBinding(name, expr))
                break
    if not bindings:
        return None
    return ValueMapping(bindings=tuple(sorted(bindings, key=lambda b: b.arg_name)))


def count_mapping_hits(mapping: ValueMapping, occs: OccurrenceSet) -> int:
    """sum(mapping_holds(...)) over the occurrences (mining.py:282-285):
    every binding must resolve and equal its argument.  Per-binding equality
    flags come from K7; occurrences with an unsure flag or a missing argument
    are checked with the host semantics."""
    occ = occs.occ
    ok = np.ones(occs.M, bool)
    check_host = np.zeros(occs.M, bool)
    for b in mapping.bindings:
        present = np.array([isinstance(a.args, dict) and b.arg_name in a.args for _, a in occ])
        if not present.all():
            check_host |= ~present
        idx = np.flatnonzero(present)
        if len(idx) == 0:
            continue
        sub = OccurrenceSet([occ[i] for i in idx], occ[0][1].tool_type) if len(idx) < occs.M else occs
        _, _, eq = sub.holds([b.expr], b.arg_name, want_eq=True)
        flags = np.zeros(occs.M, np.uint8)
        flags[idx] = eq[0]
        ok &= flags == 1
        check_host |= flags == 2
    hits = int((ok & ~check_host).sum())
    for i in np.flatnonzero(check_host):
        ctx, act = occ[i]
        hits += phase2.mapping_holds(mapping, ctx, act)
    return hits

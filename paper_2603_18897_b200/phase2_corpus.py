"""Phase II over one corpus tape: mapping inference for every mined candidate
with the occurrences, histories and actual arguments read in HBM (SURVEY.md
8(f) row 1).

mine() (mining.py:248-292) keeps, per candidate, the followed occurrences of
its target and runs infer_mapping / mapping_holds on them
(mappings.py:276-417, mining.py:202-212,277-285).  Here:

* every tool event's ``result`` and ``args`` are payload tapes of one corpus
  arena in HBM, written once per mine() call (tape 2p = result of stream
  position p, 2p + 1 = its args);
* the occurrences come from the device occurrence pass
  (paste_mine_occurrences) as stream positions: anchor, matched events,
  history = [first matched, anchor] of the corpus token stream;
* the common scalar argument test (_common_scalar_args) is a device key
  lookup over the occurrences' argument tapes (paste_tape_key_lookup);
* every hypothesis is scored over every occurrence by K7 (paste_holds in
  corpus mode: histories are ranges of the token stream, actuals are nodes
  of the argument tapes), and mapping_holds counts use K7's per-binding
  equality flags;
* the IndexedFallback seed (the occurrence with the fewest failures after a
  source, mappings.py:353-362) is an argmin over prefix counts of the
  target's FAIL tokens;
* the host keeps the reference's enumeration order: it
  materialises the seed occurrence only, generates its hypotheses in the
  reference's order and takes the first one whose device hit fraction
  passes.  Pairs the device cannot decide exactly (non-ASCII
  FormatTemplate text) are re-evaluated with Python string semantics on
  Python objects built for those occurrences only.
"""

from __future__ import annotations

import ctypes
from typing import Any, Sequence

import numpy as np

from . import _native, phase2
from ._native import BINDING_DTYPE, HoldsDesc, KeyLookupDesc, check, ptr
from .mappings import (ArgBinding, FormatTemplate, IndexedFallback, MatchedContext, PathLookup,
                       ValueMapping)
from .packing import SigTable, encode_binding
from .tape import KeyTable, TapeArena

_NORM_CODE = {"none": 0, "trim": 1, "lowercase": 2}
SEG_FLAG = np.int32(-2**31)


def _torch():
    import torch

    return torch


class CorpusTapes:
    """The corpus in HBM for Phase II: token stream + result / args tapes."""

    def __init__(self, nodes, data, refs, keys: KeyTable, tok_host: np.ndarray, tok_dev,
                 sigs: SigTable, events: Sequence, res_tape=None, args_tape=None):
        from .device_ops import to_dev

        self.keys, self.sigs, self.events = keys, sigs, events
        self.tok, self.tok_dev = tok_host, tok_dev
        self.dev = {"nodes": to_dev(nodes), "data": to_dev(data), "refs": to_dev(refs)}
        n = len(tok_host)
        # tape of stream position p's result / args (default: 2p, 2p + 1)
        self.res_tape = (2 * np.arange(n, dtype=np.int64) if res_tape is None
                         else np.asarray(res_tape, np.int64))
        self.args_tape = self.res_tape + 1 if args_tape is None else np.asarray(args_tape, np.int64)
        self._fail_prefix: dict[int, np.ndarray] = {}

    @classmethod
    def from_events(cls, flat: Sequence, tok_host: np.ndarray, tok_dev, sigs: SigTable
                    ) -> "CorpusTapes":
        keys = KeyTable()
        arena = TapeArena(keys, keep_objects=False)
        payloads = [None] * (2 * len(flat))
        payloads[0::2] = [ev.result for ev in flat]
        payloads[1::2] = [ev.args for ev in flat]
        arena.add_many(payloads)
        nodes, data, refs = arena.arrays()
        return cls(nodes, data, refs, keys, tok_host, tok_dev, sigs, flat)

    def fail_prefix(self, tool: int) -> np.ndarray:
        """F[p] = FAIL events of `tool` at stream positions < p."""
        f = self._fail_prefix.get(tool)
        if f is None:
            t = self.tok & 0x7fffffff
            hit = ((t >> 1) == tool) & ((t & 1) == 0)
            f = np.zeros(len(t) + 1, np.int64)
            np.cumsum(hit, out=f[1:])
            self._fail_prefix[tool] = f
        return f


class TapeEvents:
    """Stream position -> Event decoded from the corpus tapes (the JSONL path
    has no Python events): built once per position, so histories keep the
    identity _failures_after relies on (mappings.py:197-206)."""

    def __init__(self, ct_arrays: tuple, keys: KeyTable, sigs: SigTable, tok: np.ndarray,
                 res_tape: np.ndarray, args_tape: np.ndarray, cols: dict):
        self.nodes, self.data, self.refs = ct_arrays
        self.keys, self.sigs, self.tok = keys, sigs, tok
        self.res_tape, self.args_tape, self.cols = res_tape, args_tape, cols
        self._cache: dict[int, Any] = {}

    def __len__(self) -> int:
        return len(self.tok)

    def _decode(self, tape: int) -> Any:
        from .tape import decode_node

        return decode_node(self.nodes, self.data, int(self.refs[tape, 0]),
                           int(self.refs[tape, 1]), 0, self.keys)

    def __getitem__(self, p: int):
        ev = self._cache.get(p)
        if ev is None:
            from .events import Event, EventKind, Status

            t = int(self.tok[p]) & 0x7fffffff
            ev = Event("", int(self.cols["seq"][p]), EventKind.TOOL_CALL, self.sigs.tools[t >> 1],
                       Status.SUCCESS if t & 1 else Status.FAIL,
                       self._decode(int(self.args_tape[p])), self._decode(int(self.res_tape[p])),
                       float(self.cols["t_start"][p]), float(self.cols["t_end"][p]))
            self._cache[p] = ev
        return ev


class CorpusOccurrences:
    """One candidate's occurrences as stream positions (anchors [M], matched
    event positions [M, n_ctx]) over a CorpusTapes."""

    def __init__(self, ct: CorpusTapes, anchors: np.ndarray, picked: np.ndarray,
                 target_tool: str):
        from .device_ops import to_dev_many

        self.ct = ct
        self.anchors = np.asarray(anchors, np.int64)
        self.picked = np.asarray(picked, np.int32)
        self.M, self.n_ctx = self.picked.shape
        self.target_tool = target_tool
        self.act_tape = ct.args_tape[self.anchors + 1].astype(np.int32)
        self.dev = to_dev_many(dict(
            occ_event=ct.res_tape[self.picked].reshape(-1).astype(np.int32),
            src_pos=(self.picked - self.picked[:, :1]).reshape(-1).astype(np.int32),
            hist_off=self.picked[:, 0].astype(np.int32),
            hist_end=(self.anchors + 1).astype(np.int32), act_tape=self.act_tape))
        self._objs: dict[int, tuple] = {}
        self._act: dict[str, tuple] = {}

    # -- Python objects (seeds, host re-checks) ------------------------------

    def occ(self, i: int):
        """(MatchedContext, next event) of occurrence i, as the reference builds it."""
        o = self._objs.get(i)
        if o is None:
            ev = self.ct.events
            pk = self.picked[i].tolist()
            a = int(self.anchors[i])
            m = MatchedContext(events=tuple(ev[p] for p in pk),
                               history=tuple(ev[p] for p in range(pk[0], a + 1)))
            o = self._objs[i] = (m, ev[a + 1])
        return o

    def occ_list(self) -> list:
        return [self.occ(i) for i in range(self.M)]

    # -- device -----------------------------------------------------------------

    def actual(self, name: str):
        """(node of args[name] per occurrence on the device, #scalar values)."""
        from .device_ops import stream_handle

        got = self._act.get(name)
        if got is None:
            torch = _torch()
            lib = _native.lib()
            key = self.ct.keys.ids.get(name)
            node = torch.full((self.M,), -1, dtype=torch.int32, device="cuda")
            n_scalar = 0
            if key is not None:
                cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                dv = self.ct.dev
                d = KeyLookupDesc(self.M, ptr(dv["nodes"]), ptr(dv["refs"]),
                                  ptr(self.dev["act_tape"]), key, 0, ptr(node), ptr(cnt))
                check(lib.paste_tape_key_lookup(ctypes.byref(d), stream_handle()), lib)
                n_scalar = int(cnt.item())
            got = self._act[name] = (node, n_scalar)
        return got

    def holds(self, exprs: Sequence, name: str, want_eq: bool = False):
        """(hits[H], unsure[H], eq[H, M] or None) of hypotheses over every occurrence."""
        from .device_ops import stream_handle, to_dev_many

        torch = _torch()
        lib = _native.lib()
        H = len(exprs)
        steps: list[int] = []
        rows, fmt, fbytes = [], [], bytearray()
        for e in exprs:
            rows.append(encode_binding(e, self.ct.sigs, self.ct.keys, steps))
            if isinstance(e, FormatTemplate):
                pre = e.prefix.encode("utf-8", "surrogatepass")
                suf = e.suffix.encode("utf-8", "surrogatepass")
                fmt += [len(fbytes), len(pre), len(fbytes) + len(pre), len(suf),
                        _NORM_CODE[e.normalization.value]]
                fbytes += pre + suf
            else:
                fmt += [0, 0, 0, 0, 0]
        node, _ = self.actual(name)
        d = to_dev_many(dict(
            hyp=np.array(rows, dtype=BINDING_DTYPE), steps=np.array(steps or [0, 0], np.int32),
            fmt=np.array(fmt, np.int32),
            fbytes=np.frombuffer(bytes(fbytes) + b"\0", np.uint8)))
        hits = torch.zeros(H, dtype=torch.int64, device="cuda")
        unsure = torch.zeros(H, dtype=torch.int64, device="cuda")
        eq = torch.zeros(H * self.M, dtype=torch.uint8, device="cuda") if want_eq else None
        dv, ov = self.ct.dev, self.dev
        desc = HoldsDesc(H, self.M, self.n_ctx, 0, ptr(d["hyp"]), ptr(d["steps"]), ptr(d["fmt"]),
                         ptr(d["fbytes"]), ptr(dv["nodes"]), ptr(dv["data"]), ptr(dv["refs"]),
                         ptr(ov["occ_event"]), ptr(ov["src_pos"]), ptr(ov["hist_off"]),
                         ptr(self.ct.tok_dev), 0, 0, 0, 0, ptr(hits), ptr(unsure), ptr(eq),
                         ptr(ov["hist_end"]), ptr(ov["act_tape"]), ptr(node))
        check(lib.paste_holds(ctypes.byref(desc), stream_handle()), lib)
        return (hits.cpu().numpy(), unsure.cpu().numpy(),
                eq.view(H, self.M).cpu().numpy() if want_eq else None)

    def fails(self) -> np.ndarray:
        """[M, n_ctx]: FAIL events of the target tool after each matched event
        in the occurrence's history (_failures_after, mappings.py:197-206)."""
        f = self.ct.fail_prefix(self.ct.sigs.tool(self.target_tool))
        return f[self.anchors + 1][:, None] - f[self.picked.astype(np.int64) + 1]


# ---------------------------------------------------------------------------
# the reference's search (mappings.py:276-417) over CorpusOccurrences
# ---------------------------------------------------------------------------

def _first_passing(exprs, err, name, co: CorpusOccurrences, fraction: float):
    if exprs:
        hits, unsure, _ = co.holds(exprs, name)
        for i, e in enumerate(exprs):
            if unsure[i]:  # Unicode string semantics on the host
                frac = phase2.holds_fraction(e, name, co.occ_list())
            else:
                frac = hits[i] / co.M
            if frac >= fraction:
                return e
    if err is not None:
        raise err
    return None


def _path_hypotheses(name, co: CorpusOccurrences, seed: int = 0):
    from .device_ops import candidate_paths_batch

    ctx0, act0 = co.occ(seed)
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


def _fallback_hypotheses(name, co: CorpusOccurrences):
    from .device_ops import candidate_paths_batch

    fails = co.fails()
    seed = int(np.argmin(fails.min(axis=1))) if co.n_ctx else 0  # first minimum, as min()
    ctx_s, act_s = co.occ(seed)
    positions = list(phase2.source_positions(ctx_s))
    searches = candidate_paths_batch([ctx_s.events[p].result for p in positions],
                                     [act_s.args[name]] * len(positions), 10_000)
    out = []
    for pos, search in zip(positions, searches):
        n_fail = int(fails[seed, pos])
        for path in search.paths:
            for cut, step in enumerate(path):
                if not isinstance(step, int) or step - n_fail < 0:
                    continue
                out.append(IndexedFallback(ctx_pos=pos, path_prefix=path[:cut],
                                           start_index=step - n_fail, path_suffix=path[cut + 1:],
                                           fail_tool=co.target_tool))
    return out, None


def _format_hypotheses(name, co: CorpusOccurrences):
    ctx0, act0 = co.occ(0)
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


def common_scalar_args(co: CorpusOccurrences) -> list[str]:
    """_common_scalar_args (mappings.py:299-315): the first occurrence's
    argument names, sorted, that every occurrence holds with a scalar value."""
    first = co.occ(0)[1].args
    if not isinstance(first, dict):
        return []
    return [name for name in sorted(first) if co.actual(name)[1] == co.M]


def infer_mapping(co: CorpusOccurrences, validation_fraction: float = 0.9
                  ) -> ValueMapping | None:
    if co.M < 2:
        return None
    bindings = []
    for name in common_scalar_args(co):
        for gen in (_path_hypotheses, _fallback_hypotheses, _format_hypotheses):
            exprs, err = gen(name, co)
            expr = _first_passing(exprs, err, name, co, validation_fraction)
            if expr is not None:
                bindings.append(ArgBinding(name, expr))
                break
    if not bindings:
        return None
    return ValueMapping(bindings=tuple(sorted(bindings, key=lambda b: b.arg_name)))


def count_mapping_hits(mapping: ValueMapping, co: CorpusOccurrences) -> int:
    """sum(mapping_holds(mapping, m, nxt)) over the occurrences (mining.py:
    202-212,282-285) from K7's per-binding equality flags (an absent argument
    or a non-dict args compares unequal, as mapping_holds returns False);
    occurrences with an undecided flag are re-checked on the host."""
    ok = np.ones(co.M, bool)
    check_host = np.zeros(co.M, bool)
    for b in mapping.bindings:
        _, _, eq = co.holds([b.expr], b.arg_name, want_eq=True)
        ok &= eq[0] == 1
        check_host |= eq[0] == 2
    hits = int((ok & ~check_host).sum())
    for i in np.flatnonzero(check_host):
        ctx, act = co.occ(int(i))
        hits += phase2.mapping_holds(mapping, ctx, act)
    return hits

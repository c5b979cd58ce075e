"""Device execution of the reference-shaped API calls.

Each function here packs host objects (:mod:`.packing`), moves the arrays to
HBM with torch, calls one libpaste entry point through the C ABI, copies the
compact result records back and rebuilds reference objects.  torch is used
for device memory and streams only.
"""

from __future__ import annotations

import ctypes
import os
from typing import Any, Callable, Sequence

import numpy as np

from . import _native
from ._native import AdmitDesc, AdmitListsDesc, PoolDesc, PredictOut, WindowsDesc, check, ptr
from .packing import (C_FULL, PoolImage, PredictResult, SigTable, admit_tables, decode_actions,
                      decode_predictions, pack_windows)
from .tape import KeyTable


def _torch():
    import torch

    return torch


def to_dev_many(arrays: dict) -> dict:
    """Several small numpy arrays -> CUDA tensors in ONE host-to-device copy:
    packed at 16-byte aligned offsets of one buffer; every result is a view
    of it with the array's dtype (structured arrays as uint8 bytes)."""
    torch = _torch()
    parts, off = [], 0
    for k, arr in arrays.items():
        a = np.ascontiguousarray(arr)
        raw = a.view(np.uint8).reshape(-1) if a.size else np.zeros(0, np.uint8)
        parts.append((k, a, off, raw.nbytes))
        off = (off + raw.nbytes + 15) & ~15
    host = np.zeros(max(off, 16), np.uint8)
    for k, a, o, nb in parts:
        if nb:
            host[o:o + nb] = a.view(np.uint8).reshape(-1)
    dev = torch.from_numpy(host).to("cuda", non_blocking=False)
    out = {"__buf__": dev, "__span__": {k: (o, nb) for k, _a, o, nb in parts}}
    for k, a, o, nb in parts:
        view = dev[o:o + nb]
        if a.dtype.names is not None or a.dtype == np.uint8:
            out[k] = view
        else:
            out[k] = view.view(getattr(torch, a.dtype.name))
    return out


def to_dev(arr: np.ndarray):
    """numpy (incl. structured) -> contiguous CUDA tensor with the same bytes."""
    torch = _torch()
    a = np.ascontiguousarray(arr)
    if not a.flags.writeable:
        a = a.copy()
    if a.dtype.names is not None or a.dtype == np.uint8:
        t = torch.from_numpy(a.view(np.uint8).reshape(-1))
    else:
        t = torch.from_numpy(a)
    return t.to("cuda", non_blocking=False)


def stream_handle() -> int:
    return _torch().cuda.current_stream().cuda_stream


class DevicePool:
    """A pattern pool compiled into a device-resident PoolImage."""

    def __init__(self, pool, sigs: SigTable | None = None, keys: KeyTable | None = None):
        self.pool = pool
        self.sigs = SigTable() if sigs is None else sigs
        self.keys = KeyTable() if keys is None else keys
        self.image = PoolImage.compile(pool, self.sigs, self.keys)
        self._dev: dict[str, Any] | None = None
        self._tables: dict[tuple[int, int], tuple[Any, int]] = {}
        self.table_budget = 256 << 20  # bytes of HBM a pool's match tables may use

    def device_arrays(self) -> dict[str, Any]:
        if self._dev is None:
            _native.lib()  # fail loudly without the library / a device
            im = self.image
            self._dev = {name: to_dev(getattr(im, name)) for name in
                         ("patterns", "bindings", "ctx_sig", "steps", "bucket_off", "bucket_pat")}
            self._dev["bucket_scan_all"] = to_dev(
                im.bucket_scan_all if len(im.bucket_scan_all) else np.zeros(1, np.uint8))
        return self._dev

    def desc(self, max_candidates: int | None = None, capacity: int | None = None) -> PoolDesc:
        """Pool descriptor; with (max_candidates, capacity) it carries the
        compiled match table for that request shape when the pool fits."""
        d = self.device_arrays()
        im = self.image
        desc = PoolDesc(len(im.pool.patterns), im.n_bucket_sigs, im.k, im.relation, im.max_ctx,
                        im.max_bindings, ptr(d["patterns"]), ptr(d["bindings"]), ptr(d["ctx_sig"]),
                        ptr(d["steps"]), ptr(d["bucket_off"]), ptr(d["bucket_pat"]),
                        ptr(d["bucket_scan_all"]), 0, 0, 0)
        if max_candidates is not None and capacity is not None:
            table, g = self.match_table(desc, max_candidates, capacity)
            if table is not None:
                desc.match_table, desc.mt_k, desc.mt_g = ptr(table), max_candidates, g
        return desc

    def match_table(self, desc: PoolDesc, K: int, W: int):
        """Device-built match table for (K, W), cached per pool (K4 compile step)."""
        key = (K, W)
        if key not in self._tables:
            torch = _torch()
            lib = _native.lib()
            nbytes = lib.paste_match_table_bytes(ctypes.byref(desc), K, W)
            table = None
            if nbytes > 0 and nbytes <= self.table_budget and not os.environ.get("PASTE_NO_MATCH_TABLE"):
                table = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                check(lib.paste_build_match_table(ctypes.byref(desc), K, W, ptr(table),
                                                  stream_handle()), lib)
            g = min(self.image.k if self.image.relation == 0 else self.image.max_ctx, W)
            self._tables[key] = (table, g)
        return self._tables[key]

    # -- predict -------------------------------------------------------------

    def _run(self, batch, K: int, admit: tuple[np.ndarray, np.ndarray, np.ndarray] | None
             ) -> PredictResult:
        torch = _torch()
        lib = _native.lib()
        n = batch.n
        B = max(self.image.max_bindings, 1)
        nodes, data, refs = batch.arena.arrays()
        tok, evt, count = to_dev(batch.tok), to_dev(batch.evt), to_dev(batch.count)
        d_nodes, d_data, d_refs = to_dev(nodes), to_dev(data), to_dev(refs)
        win = WindowsDesc(n, batch.capacity, 0, ptr(tok), ptr(evt), ptr(count), ptr(d_nodes),
                          ptr(d_data), ptr(d_refs), 0, 0, 0, 0)
        dev = torch.device("cuda")
        o = {"n_pred": torch.zeros(n, dtype=torch.int32, device=dev),
             "pred_pat": torch.zeros(n * K, dtype=torch.int32, device=dev),
             "pred_comp": torch.zeros(n * K, dtype=torch.uint8, device=dev),
             "pred_arg": torch.full((n * K * B,), -1, dtype=torch.int64, device=dev),
             "struct_err": torch.zeros(n, dtype=torch.int32, device=dev)}
        if admit is not None:
            o["n_act"] = torch.zeros(n, dtype=torch.int32, device=dev)
            o["act_pred"] = torch.zeros(n * K, dtype=torch.int16, device=dev)
            o["act_level"] = torch.zeros(n * K, dtype=torch.uint8, device=dev)
            o["act_util"] = torch.zeros(n * K, dtype=torch.float64, device=dev)
            allow, level, bene = (to_dev(x) for x in admit)
            adm = AdmitDesc(1, len(admit[0]), ptr(allow), ptr(level), ptr(bene))
        else:
            adm = AdmitDesc(0, 0, 0, 0, 0)
        out = PredictOut(K, B, 0, 0, ptr(o["n_pred"]), ptr(o["pred_pat"]), ptr(o["pred_comp"]),
                         ptr(o["pred_arg"]), ptr(o.get("n_act")), ptr(o.get("act_pred")),
                         ptr(o.get("act_level")), ptr(o.get("act_util")), ptr(o["struct_err"]))
        pool = self.desc(K, batch.capacity)
        check(lib.paste_predict_batch(ctypes.byref(pool), ctypes.byref(win), ctypes.byref(adm),
                                      ctypes.byref(out), stream_handle()), lib)
        h = {k: v.cpu().numpy() for k, v in o.items()}
        return PredictResult(K, B, h["n_pred"], h["pred_pat"], h["pred_comp"], h["pred_arg"],
                             h.get("n_act"), h.get("act_pred"), h.get("act_level"),
                             h.get("act_util"), h["struct_err"])

    def _k_for(self, max_candidates: int | None) -> tuple[int, bool]:
        """Kernel slot count; truncation with Python slice semantics for
        non-positive values is applied on the host."""
        if max_candidates is not None and max_candidates > 0:
            return max_candidates, False
        return max(self.image.max_bucket, 1), max_candidates is not None

    def predict_windows(self, windows: Sequence[Sequence], now: float | None,
                        max_candidates: int | None):
        K, slice_after = self._k_for(max_candidates)
        batch = pack_windows(windows, self.sigs, self.keys)
        res = self._run(batch, K, None)
        preds = decode_predictions(res, self.image, batch.arena, batch.created, now)
        if slice_after:
            preds = [p[:max_candidates] for p in preds]
        return preds, int(res.struct_err.sum())

    def predict_admit_windows(self, windows: Sequence[Sequence], policy, estimates,
                              now: float | None, max_candidates: int | None):
        K, slice_after = self._k_for(max_candidates)
        if slice_after:
            raise ValueError("predict_admit_batch needs a positive max_candidates")
        batch = pack_windows(windows, self.sigs, self.keys)
        tables = admit_tables(self.sigs, policy, estimates.duration)
        res = self._run(batch, K, tables)
        preds = decode_predictions(res, self.image, batch.arena, batch.created, now)
        return preds, decode_actions(res, preds), int(res.struct_err.sum())


# ---------------------------------------------------------------------------
# standalone admit
# ---------------------------------------------------------------------------


def admit_lists(lists: Sequence[Sequence], policy, benefit_of: Callable[[Any], float]):
    from .policy import SpecLevel, SpeculativeAction
    from .prediction import Completeness

    torch = _torch()
    lib = _native.lib()
    sigs = SigTable()
    flat = [p for lst in lists for p in lst]
    off = np.zeros(len(lists) + 1, np.int64)
    off[1:] = np.cumsum([len(lst) for lst in lists])
    tool = np.array([sigs.tool(p.tool_type) for p in flat] or [0], np.int32)
    full = np.array([p.completeness is Completeness.FULL for p in flat] or [0], np.uint8)
    prob = np.array([p.probability for p in flat] or [0], np.float64)
    bene = np.array([benefit_of(p) for p in flat] or [0], np.float64)
    created = np.array([p.created_at for p in flat] or [0], np.float64)
    allow, level, _ = admit_tables(sigs, policy, lambda name: 0.0)
    d = {k: to_dev(v) for k, v in dict(off=off, tool=tool, full=full, prob=prob, bene=bene,
                                       created=created, allow=allow, level=level).items()}
    N = max(len(flat), 1)
    dev = torch.device("cuda")
    n_act = torch.zeros(len(lists) or 1, dtype=torch.int32, device=dev)
    act_pred = torch.zeros(N, dtype=torch.int32, device=dev)
    act_level = torch.zeros(N, dtype=torch.uint8, device=dev)
    act_util = torch.zeros(N, dtype=torch.float64, device=dev)
    adm = AdmitDesc(1, len(allow), ptr(d["allow"]), ptr(d["level"]), 0)
    desc = AdmitListsDesc(len(lists), ptr(d["off"]), ptr(d["tool"]), ptr(d["full"]),
                          ptr(d["prob"]), ptr(d["bene"]), ptr(d["created"]), ptr(n_act),
                          ptr(act_pred), ptr(act_level), ptr(act_util))
    check(lib.paste_admit_lists(ctypes.byref(adm), ctypes.byref(desc), stream_handle()), lib)
    n_act, act_pred = n_act.cpu().numpy(), act_pred.cpu().numpy()
    act_level, act_util = act_level.cpu().numpy(), act_util.cpu().numpy()
    out = []
    for li, lst in enumerate(lists):
        b0 = int(off[li])
        out.append([SpeculativeAction(prediction=lst[int(act_pred[b0 + j])],
                                      level=SpecLevel(int(act_level[b0 + j])),
                                      expected_utility=float(act_util[b0 + j]))
                    for j in range(int(n_act[li]))])
    return out


# ---------------------------------------------------------------------------
# K5: candidate_paths (leaf scan) and evaluate (resolve)
# ---------------------------------------------------------------------------


def _target_scalar(value):
    """(tape type or -1, is_nan, canonical bytes) of a candidate_paths target."""
    import unicodedata

    from .tape import T_STR, scalar_bytes

    try:
        typ, flags, data = scalar_bytes(value)
    except TypeError:
        return -1, 0, b""  # containers / non-JSON objects never equal a scalar leaf
    if typ == T_STR:
        data = unicodedata.normalize("NFC", value).encode("utf-8", "surrogatepass")
    return typ, 1 if (flags & 4) else 0, data


def candidate_paths_batch(payloads: Sequence[Any], targets: Sequence[Any], node_budget: int):
    from ._native import LeafScanDesc
    from .mappings import PathSearch
    from .tape import TapeArena

    torch = _torch()
    lib = _native.lib()
    arena = TapeArena(keep_objects=False)
    events = np.array(arena.add_many(payloads) or [0], np.int32)
    nodes, data, refs = arena.arrays()
    n = len(payloads)
    sizes = []
    for e in range(n):
        root = nodes[int(refs[e, 0])]
        sizes.append(int(root["b"]) if root["type"] >= 6 else 1)
    cap = np.minimum(np.array(sizes or [0], np.int64), max(node_budget, 0))
    out_off = np.zeros(n + 1, np.int64)
    out_off[1:] = np.cumsum(cap[:n])
    tt, tn, tb = zip(*[_target_scalar(t) for t in targets]) if n else ((), (), ())
    target_off = np.zeros(n + 1, np.int64)
    target_off[1:] = np.cumsum([len(b) for b in tb])
    tbytes = np.frombuffer(b"".join(tb) + b"\0", np.uint8)
    d = to_dev_many(dict(
        nodes=nodes, data=data, refs=refs, events=events,
        tt=np.array(list(tt) or [0], np.int32), tn=np.array(list(tn) or [0], np.uint8),
        toff=target_off, tbytes=tbytes, out_off=out_off,
        out_nodes=np.zeros(max(int(out_off[-1]), 1), np.int32),
        n_out=np.zeros(max(n, 1), np.int64), trunc=np.zeros(max(n, 1), np.uint8)))
    out_nodes, n_out, trunc = d["out_nodes"], d["n_out"], d["trunc"]
    desc = LeafScanDesc(n, int(node_budget), ptr(d["nodes"]), ptr(d["data"]), ptr(d["refs"]),
                        ptr(d["events"]), ptr(d["tt"]), ptr(d["tn"]), ptr(d["toff"]),
                        ptr(d["tbytes"]), ptr(d["out_off"]), ptr(out_nodes), ptr(n_out), ptr(trunc))
    check(lib.paste_leaf_scan(ctypes.byref(desc), stream_handle()), lib)
    # the three results are the tail of the packed buffer: one device-to-host copy
    span = d["__span__"]
    lo = span["out_nodes"][0]
    hi = span["trunc"][0] + span["trunc"][1]
    back = d["__buf__"][lo:hi].cpu().numpy()
    o, nb = span["out_nodes"]
    out_nodes = back[o - lo:o - lo + nb].view(np.int32)
    o, nb = span["n_out"]
    n_out = back[o - lo:o - lo + nb].view(np.int64)
    o, nb = span["trunc"]
    trunc = back[o - lo:o - lo + nb]
    res = []
    for q in range(n):
        found = out_nodes[out_off[q]:out_off[q] + min(int(n_out[q]), int(cap[q]))]
        res.append(PathSearch(paths=tuple(arena.path_of(q, int(x)) for x in found),
                              truncated=bool(trunc[q])))
    return res


def evaluate_mapping(mapping, ctx):
    """evaluate() (mappings.py:207-223) with the resolution on the device."""
    from ._native import BINDING_DTYPE, ResolveDesc
    from .mappings import FormatTemplate, MappingResult, MappingStructureError, expr_ctx_pos
    from .packing import encode_binding
    from .tape import TapeArena, leaf_str_of

    torch = _torch()
    lib = _native.lib()
    for b in mapping.bindings:  # structural errors raise before any work
        pos = expr_ctx_pos(b.expr)
        if not 0 <= pos < len(ctx.events):
            raise MappingStructureError(f"ctx_pos {pos} out of range")
    if not mapping.bindings:
        return MappingResult(args={}, unbound=())
    sigs, keys = SigTable(), KeyTable()
    arena = TapeArena(keys)
    slot_of: dict[int, int] = {}
    steps: list[int] = []
    rows, src_event, src_pos, hist_tok, hist_off = [], [], [], [], [0]
    for b in mapping.bindings:
        rows.append(encode_binding(b.expr, sigs, keys, steps))
        src = ctx.events[expr_ctx_pos(b.expr)]
        if id(src) not in slot_of:
            slot_of[id(src)] = arena.add(src.result)
        src_event.append(slot_of[id(src)])
        first = next((j for j, ev in enumerate(ctx.history) if ev is src), -1)
        src_pos.append(first)
        for j, ev in enumerate(ctx.history):
            hist_tok.append(-1 if (ev is src or ev.kind.value != "tool_call")
                            else sigs.sig(ev.tool_type, ev.status))
        hist_off.append(len(hist_tok))
    nodes, data, refs = arena.arrays()
    d = {k: to_dev(v) for k, v in dict(
        bindings=np.array(rows, dtype=BINDING_DTYPE), steps=np.array(steps or [0, 0], np.int32),
        nodes=nodes, refs=refs, src_event=np.array(src_event, np.int32),
        hist_off=np.array(hist_off, np.int32), hist_tok=np.array(hist_tok or [0], np.int32),
        src_pos=np.array(src_pos, np.int32)).items()}
    result = torch.zeros(len(rows), dtype=torch.int64, device="cuda")
    desc = ResolveDesc(len(rows), ptr(d["bindings"]), ptr(d["steps"]), ptr(d["nodes"]),
                       ptr(d["refs"]), ptr(d["src_event"]), ptr(d["hist_off"]), ptr(d["hist_tok"]),
                       ptr(d["src_pos"]), ptr(result))
    check(lib.paste_resolve(ctypes.byref(desc), stream_handle()), lib)
    res = result.cpu().numpy()
    args, unbound = {}, []
    for b, ev, node in zip(mapping.bindings, src_event, res.tolist()):
        if node < 0:
            unbound.append(b.arg_name)
            continue
        value = arena.node_object(ev, node)
        if isinstance(b.expr, FormatTemplate):
            value = b.expr.prefix + b.expr.normalization.apply(leaf_str_of(value)) + b.expr.suffix
        args[b.arg_name] = value
    return MappingResult(args=args, unbound=tuple(unbound))


# ---------------------------------------------------------------------------
# score_accuracy replay (prediction.py:133-169)
# ---------------------------------------------------------------------------


def score_replay(traces, pool, window_capacity: int, max_candidates):
    """Device replay with the hit check on the device (replay.py, C2)."""
    from .replay import score_replay as _score

    return _score(traces, pool, window_capacity, max_candidates)


class LeafScanBatch:
    """Device-resident K5 batch: one (payload, target) query per session.

    Queries whose payloads share a node array (shape-interned tapes) and
    whose targets share type and canonical length are grouped when the batch
    is built; when groups are few the shape-shared scan runs (candidates
    listed once per group, compared per query), else the per-query scan."""

    def __init__(self, nodes, data, refs, target_off, target_bytes, node_budget: int = 10_000,
                 target_type: int = 5, max_matches: int = 4, shared: bool | None = None):
        torch = _torch()
        self.lib = _native.lib()
        n = len(refs)
        self.n = n
        self.nodes, self.data, self.refs = to_dev(nodes), to_dev(data), to_dev(refs)
        self.events = torch.arange(n, dtype=torch.int32, device="cuda")
        self.tt = torch.full((n,), target_type, dtype=torch.int32, device="cuda")
        self.tn = torch.zeros(n, dtype=torch.uint8, device="cuda")
        self.toff, self.tbytes = to_dev(target_off), to_dev(target_bytes)
        self.out_off = torch.arange(n + 1, dtype=torch.int64, device="cuda") * max_matches
        self.out_nodes = torch.zeros(n * max_matches, dtype=torch.int32, device="cuda")
        self.n_out = torch.zeros(n, dtype=torch.int64, device="cuda")
        self.trunc = torch.zeros(n, dtype=torch.uint8, device="cuda")
        self.budget = node_budget
        # shape groups: (node array, target type, target length)
        refs_np = np.asarray(refs).reshape(-1, 2)
        tlen = np.diff(np.asarray(target_off, np.int64))
        keys = np.stack([refs_np[:, 0], np.full(n, target_type, np.int64), tlen], axis=1)
        uniq, rep, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
        self.n_groups = len(uniq)
        self.shared = (self.n_groups * 8 <= n) if shared is None else shared
        if self.shared:
            self.group = torch.from_numpy(inv.reshape(-1).astype(np.int32)).cuda()
            self.group_rep = torch.from_numpy(rep.astype(np.int32)).cuda()
            self.scratch = torch.empty(
                max(self.lib.paste_leaf_scan_shared_bytes(self.n_groups, node_budget), 4),
                dtype=torch.uint8, device="cuda")

    def desc(self):
        from ._native import LeafScanDesc

        return LeafScanDesc(self.n, self.budget, ptr(self.nodes), ptr(self.data), ptr(self.refs),
                            ptr(self.events), ptr(self.tt), ptr(self.tn), ptr(self.toff),
                            ptr(self.tbytes), ptr(self.out_off), ptr(self.out_nodes),
                            ptr(self.n_out), ptr(self.trunc))

    def launch(self) -> None:
        d = self.desc()
        if self.shared:
            check(self.lib.paste_leaf_scan_shared(ctypes.byref(d), ptr(self.group), self.n_groups,
                                                  ptr(self.group_rep), ptr(self.scratch),
                                                  stream_handle()), self.lib)
        else:
            check(self.lib.paste_leaf_scan(ctypes.byref(d), stream_handle()), self.lib)

    def launch_count(self) -> int:
        return 2 if self.shared else 1

"""Device-resident live sessions: the batched predict + admit serving path.

One ``LiveSessionTable`` holds, in HBM, the prediction windows of N live
sessions (a ring of W (token, event) slots each, ``PredictionWindow``
prediction.py:40-58), the payload arena of the events those windows can
still see, and the compact output records.  Each :meth:`step` is what the
reference does once per tool completion per session (simulation.py:402-442:
observe -> predict(max_candidates) -> admit(benefit = EWMA duration)), for all
N sessions in one kernel launch.

Arena: the events observed at step s form batch region ``s mod (W+1)``; a
window only reaches W events back, so a region is never overwritten while a
window still references it.  Payload node arrays are shape-interned
(:mod:`.synth`), so a batch ships its tokens, directory entries and scalar
bytes only.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import AdmitDesc, LivePlan, PredictOut, WindowsDesc, check, ptr
from .device_ops import DevicePool, stream_handle, to_dev
from .packing import PredictResult, admit_tables


def wire8_layout(n: int, node_bytes: int = 2) -> tuple[int, int]:
    """(byte offset of the node half, total bytes) of the packed narrow wire
    form: tok8 [n] | pad to 16 | node16 [n] (node_bytes 2) or node8 [n] (1)."""
    off = (n + 15) // 16 * 16
    return off, off + node_bytes * n


class NodeCodes:
    """u8 codes for the node arrays (payload shapes) of a live table's
    events: the 2-byte wire form (u8 token + u8 node code), decoded on the
    device through a 256-entry code -> node_base table.  Codes are only ever
    appended, so steps in flight keep their meaning; past 256 node arrays
    encode() returns None and batches keep the 3-byte form."""

    def __init__(self):
        import torch

        self.lut = np.full(1 << 16, -1, np.int16)  # node_base -> code
        gpu = torch.cuda.is_available()  # (the host encoding alone runs without one)
        self.host = torch.zeros(256, dtype=torch.int32)
        self.host = self.host.pin_memory() if gpu else self.host
        self.dev = torch.zeros(256, dtype=torch.int32, device="cuda") if gpu else None
        self.n = 0
        self.uploaded = 0

    def encode(self, node: np.ndarray) -> np.ndarray | None:
        code = self.lut[node]
        missing = code < 0
        if missing.any():
            new = np.unique(node[missing])
            if self.n + len(new) > 256:
                return None
            self.lut[new] = np.arange(self.n, self.n + len(new), dtype=np.int16)
            self.host.numpy()[self.n:self.n + len(new)] = new
            self.n += len(new)
            code = self.lut[node]
        return code.astype(np.uint8)

    def upload(self, stream) -> None:
        """Queue the table's new entries host -> device on `stream`."""
        import torch

        if self.n > self.uploaded:
            with torch.cuda.stream(stream):
                self.dev[:self.n].copy_(self.host[:self.n], non_blocking=True)
            self.uploaded = self.n


class EventCodes:
    """u8 codes for the (token, node array) pairs of a live table's events:
    the 1-byte wire form, decoded on the device through a 256-entry code ->
    (token, node_base) table (paste_windows.event_codes).  Pairs are keyed
    by (u8 token, NodeCodes node code); codes are only ever appended, so
    steps in flight keep their meaning; past 256 pairs encode() returns
    None and batches keep the 2-byte form."""

    def __init__(self, nodes: NodeCodes):
        import torch

        self.nodes = nodes
        self.lut = np.full(1 << 16, -1, np.int16)  # tok8 << 8 | node code -> code
        gpu = torch.cuda.is_available()
        self.host = torch.zeros(512, dtype=torch.int32)  # (token, node_base) per code
        self.host = self.host.pin_memory() if gpu else self.host
        self.dev = torch.zeros(512, dtype=torch.int32, device="cuda") if gpu else None
        self.n = 0
        self.uploaded = 0

    def encode(self, tok8: np.ndarray, node8: np.ndarray) -> np.ndarray | None:
        key = (tok8.astype(np.int32) << 8) | node8
        code = self.lut[key]
        missing = code < 0
        if missing.any():
            new = np.unique(key[missing])
            if self.n + len(new) > 256:
                return None
            self.lut[new] = np.arange(self.n, self.n + len(new), dtype=np.int16)
            pairs = self.host.numpy().reshape(256, 2)
            t = new >> 8
            pairs[self.n:self.n + len(new), 0] = np.where(t == 255, -1, t)
            pairs[self.n:self.n + len(new), 1] = self.nodes.host.numpy()[new & 0xFF]
            self.n += len(new)
            code = self.lut[key]
        return code.astype(np.uint8)

    def upload(self, stream) -> None:
        """Queue the table's new entries host -> device on `stream`."""
        import torch

        if self.n > self.uploaded:
            with torch.cuda.stream(stream):
                self.dev[:2 * self.n].copy_(self.host[:2 * self.n], non_blocking=True)
            self.uploaded = self.n


@dataclass
class EventBatch:
    """One new tool event per session: tokens, batch-relative directory
    entries (node_base, byte_base) and the batch's scalar bytes."""

    tok: object   # i32[n]      (numpy or torch, host or device)
    ref: object   # i64[n, 2]
    data: object  # u8[bytes]
    node: object = None  # optional i32[n]: node_base only (the narrow wire form)
    tok8: object = None    # optional u8[n]: token, 255 = LLM step (the narrow wire forms)
    node16: object = None  # optional u16[n]: node_base (3-byte form)
    packed: object = None  # optional u8: tok8 and node16 / node8 in one buffer (wire8_layout)
    node8: object = None   # optional u8[n]: node code (2-byte form, NodeCodes of the table)
    ev8: object = None     # optional u8[n]: event code (1-byte form, EventCodes of the table)

    def narrowed(self, codes: "NodeCodes | None" = None,
                 events: "EventCodes | None" = None) -> "EventBatch":
        """The narrow wire form alongside the others, when the values fit
        (signature ids < 255, node bases < 2^16): u8 token + u16 node_base
        (3 bytes), or with a live table's ``codes`` u8 token + u8 node code
        (2 bytes) while the table has seen at most 256 node arrays.  Both
        halves sit in one buffer (`packed`, wire8_layout), so a step uploads
        them with one copy.  With the table's ``events`` as well, a u8 event
        code per session (1 byte) while the table has seen at most 256
        (token, node array) pairs; `packed` is then that code array."""
        tok = np.asarray(self.tok)
        node = np.asarray(self.node if self.node is not None else np.asarray(self.ref)[:, 0])
        if tok.size and (tok.max() >= 255 or node.max() >= (1 << 16) or node.min() < 0):
            return self
        n = len(tok)
        code = codes.encode(node) if codes is not None else None
        off, size = wire8_layout(n, 1 if code is not None else 2)
        packed = np.zeros(size, np.uint8)
        tok8 = packed[:n]
        tok8[:] = np.where(tok < 0, 255, tok)
        if code is not None:
            node8 = packed[off:off + n]
            node8[:] = code
            ev = events.encode(tok8, node8) if events is not None else None
            if ev is not None:
                return EventBatch(self.tok, self.ref, self.data, self.node, tok8, None, ev,
                                  node8, ev)
            return EventBatch(self.tok, self.ref, self.data, self.node, tok8, None, packed, node8)
        node16 = packed[off:off + 2 * n].view(np.uint16)
        node16[:] = node
        return EventBatch(self.tok, self.ref, self.data, self.node, tok8, node16, packed)

    def pin(self) -> "EventBatch":
        """Move the narrow wire form into pinned host memory (one buffer, with
        tok8 / node16 / node8 as views), for the asynchronous single-copy
        upload."""
        import torch

        if self.ev8 is not None and isinstance(self.ev8, np.ndarray):
            self.ev8 = self.packed = torch.from_numpy(self.ev8).pin_memory()
        elif self.packed is not None and isinstance(self.packed, np.ndarray):
            n = len(self.tok8)
            off, _ = wire8_layout(n)
            self.packed = torch.from_numpy(self.packed).pin_memory()
            self.tok8 = self.packed[:n]
            if self.node8 is not None:
                self.node8 = self.packed[off:off + n]
            else:
                self.node16 = self.packed[off:off + 2 * n].view(torch.int16)
        return self

    def wire(self, ship_bytes: bool, narrow8: bool = False) -> tuple:
        """The arrays a step copies host -> device."""
        if ship_bytes:
            return (self.tok, self.ref, self.data)
        if narrow8 and self.packed is not None:
            return (self.packed,)
        if narrow8 and self.tok8 is not None:
            return (self.tok8, self.node16)
        return (self.tok, self.node) if self.node is not None else (self.tok, self.ref)

    def nbytes(self, with_data: bool = True, narrow8: bool = False) -> int:
        return sum(int(x.nbytes) if isinstance(x, np.ndarray) else x.numel() * x.element_size()
                   for x in self.wire(with_data, narrow8))


class LiveSessionTable:
    def __init__(self, dpool: DevicePool, n_sessions: int, nodes: np.ndarray,
                 max_batch_bytes: int, policy, estimates, capacity: int = 16,
                 max_candidates: int = 8, ship_bytes: bool = False):
        import torch

        _native.lib()
        self.torch = torch
        self.dpool = dpool
        self.n = n_sessions
        self.W = capacity
        self.K = max_candidates
        self.B = max(dpool.image.max_bindings, 1)
        self.regions = capacity + 1
        # predict resolves argument *node references*; the scalar bytes stay in
        # the host's copy of the payload unless a consumer on the device needs them
        self.ship_bytes = ship_bytes
        self.max_batch_bytes = int(max_batch_bytes) if ship_bytes else 0
        dev = torch.device("cuda")
        n, W, K, B = self.n, self.W, self.K, self.B
        self.tok = torch.full((n * W,), -1, dtype=torch.int32, device=dev)
        self.evt = torch.full((n * W,), -1, dtype=torch.int32, device=dev)
        self.count = torch.zeros(n, dtype=torch.int64, device=dev)
        self.nodes = to_dev(nodes)
        self.host_nodes = nodes
        self.bytes = torch.zeros(max(self.regions * self.max_batch_bytes, 1), dtype=torch.uint8,
                                 device=dev)
        self.refs = torch.zeros(self.regions * n * 2, dtype=torch.int64, device=dev)
        self.new_tok = torch.zeros(n, dtype=torch.int32, device=dev)
        self.new_ref = torch.zeros(n * 2, dtype=torch.int64, device=dev)
        self.new_node = torch.zeros(n, dtype=torch.int32, device=dev)
        self.narrow = False  # last staged batch came in the narrow (node-only) form
        # serve(): one fused predict + compaction kernel (True) or the K-slot
        # kernel + the compaction kernel (False)
        self.serve_fused = True
        if self.regions > 31 or len(nodes) >= (1 << 27):
            raise ValueError("live table needs capacity <= 30 and < 2^27 template nodes")
        allow, level, bene = admit_tables(dpool.sigs, policy, estimates.duration)
        self.benefit = np.asarray(bene, np.float64)
        # narrowest record-stream widths this table's geometry allows
        self.cformat = ((_native.PASTE_CF_HDR8 if max_candidates <= 15 else 0)
                        | (_native.PASTE_CF_PRED8 if len(dpool.image.patterns) <= 64 else 0)
                        | (_native.PASTE_CF_ARG16 if len(nodes) < (1 << 11) else 0))
        self.adm_arrays = (to_dev(allow), to_dev(level), to_dev(bene))
        self.adm = AdmitDesc(1, len(allow), *[ptr(a) for a in self.adm_arrays])
        self.out = {"n_pred": torch.zeros(n, dtype=torch.int32, device=dev),
                    "pred_pat": torch.zeros(n * K, dtype=torch.int32, device=dev),
                    "pred_comp": torch.zeros(n * K, dtype=torch.uint8, device=dev),
                    "pred_arg": torch.full((n * K * B,), -1, dtype=torch.int64, device=dev),
                    "n_act": torch.zeros(n, dtype=torch.int32, device=dev),
                    "act_pred": torch.zeros(n * K, dtype=torch.int16, device=dev),
                    "act_level": torch.zeros(n * K, dtype=torch.uint8, device=dev),
                    "act_util": torch.zeros(n * K, dtype=torch.float64, device=dev),
                    "struct_err": torch.zeros(n, dtype=torch.int32, device=dev)}
        o = self.out
        # slot-major ring and records: a step touches contiguous 128-byte lines
        self.out_desc = PredictOut(K, B, 1, 0, *[ptr(o[k]) for k in (
            "n_pred", "pred_pat", "pred_comp", "pred_arg", "n_act", "act_pred", "act_level",
            "act_util", "struct_err")])
        self.pool_desc = dpool.desc(max_candidates, capacity)
        self.steps = 0
        self.lib = _native.lib()
        # serve() format: with the fused kernel the prediction list ships as
        # the session's match-table key (PASTE_CF_ENTRY16) when keys fit u16
        ef = self.cformat | _native.PASTE_CF_ENTRY16
        self.sformat = ef if self.lib.paste_predict_compact_supported(
            ctypes.byref(self.pool_desc), capacity, K, B, ef) else self.cformat
        self._entries = None
        self.plan = None
        self._plan_host = None
        self.plan_codes = None
        self._build_plan()
        # the 3-byte observe input and the key + argument serving streams
        # need the live-plan kernels
        self.narrow8 = (self.plan is not None and not ship_bytes and len(nodes) < (1 << 16)
                        and 2 * len(dpool.sigs) < 255)
        self.codes = NodeCodes() if self.narrow8 else None  # the 2-byte wire form
        self.ecodes = EventCodes(self.codes) if self.narrow8 else None  # the 1-byte form
        self.new_tok8 = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.new_node16 = torch.zeros(n, dtype=torch.int16, device=dev)
        self.staged8 = False
        if self.plan is not None and self.sformat & _native.PASTE_CF_ENTRY16:
            self.sformat |= _native.PASTE_CF_KEYS
            # one reference per distinct resolution (PASTE_CF_UNIQ)
            if os.environ.get("PASTE_NO_UNIQ") != "1":
                self.sformat |= _native.PASTE_CF_UNIQ
            # u8 plan codes instead of u16 keys when the distinct non-empty
            # entries fit (PASTE_CF_KEY8): 1 B per session less to download
            if self.plan_codes is not None and os.environ.get("PASTE_NO_KEY8") != "1":
                self.sformat |= _native.PASTE_CF_KEY8

    def _build_plan(self) -> None:
        """Compile the live plan (paste_build_live_plan: per match-table key,
        the step's records and admit decisions) and the walk table (per
        (binding, template node): the resolved argument node).  None when the
        request shape is outside the plan's envelope (the step then runs the
        general kernel)."""
        t = self.torch
        lib = self.lib
        if os.environ.get("PASTE_NO_LIVE_PLAN"):
            return
        nbytes = lib.paste_live_plan_bytes(ctypes.byref(self.pool_desc), self.K, self.W)
        if nbytes <= 0:
            return
        buf = t.empty(nbytes, dtype=t.uint8, device="cuda")
        check(lib.paste_build_live_plan(ctypes.byref(self.pool_desc), ctypes.byref(self.adm),
                                        self.K, self.W, ptr(buf), stream_handle()), lib)
        walk = None
        n_bind = len(self.dpool.image.bindings)
        wbytes = lib.paste_live_walk_bytes(n_bind, len(self.host_nodes)) if n_bind else -1
        if wbytes > 0:
            walk = t.empty(wbytes // 4, dtype=t.int32, device="cuda")
            check(lib.paste_build_live_walk(ctypes.byref(self.pool_desc), n_bind, ptr(self.nodes),
                                            len(self.host_nodes), ptr(walk), stream_handle()), lib)
        self._plan_bufs = (buf, walk)
        self.plan = LivePlan(ptr(buf), self.K, self.dpool.image.max_bindings, ptr(walk),
                             len(self.host_nodes) if walk is not None else 0)
        self._assign_plan_codes()

    def _assign_plan_codes(self) -> None:
        """Number the plan's distinct non-empty entries (PASTE_CF_KEY8).
        Everything the host expands from a key -- counts, pattern ids,
        completeness, action codes, utilities, binding map words -- is the
        entry's content, so keys with equal content may share one u8 code;
        entries without predictions, actions or bindings all read as 0xFF,
        like a session without a key.  The code goes into byte 8 of each
        entry's header, which the serving kernels write to the key stream;
        the host keeps one representative key per code (``plan_host()[6]``).
        None (and the u16 key stream) when more than 255 codes are needed."""
        self._plan_host = None
        self.plan_codes = None
        K, M = self.K, self.K * max(self.dpool.image.max_bindings, 1)
        L = plan_layout_host(K, M)
        got = plan_codes(self._plan_bufs[0].cpu().numpy().reshape(-1, L["stride"]), K, M)
        if got is None:
            return
        codes, rep = got
        t = self.torch
        view = self._plan_bufs[0].view(-1, L["stride"])
        view[:, 8].copy_(t.from_numpy(codes))
        self.plan_codes = (codes, rep)

    def refresh_estimates(self, estimates) -> None:
        """Re-read ``benefit_of = estimates.duration`` for every tool (the
        reference reads the current EWMA at every prediction,
        simulation.py:428-429): call after ``EstimateBook.update`` so the
        device admit tables and ``CompactRecords.expand`` see the new values."""
        bene = np.array([float(estimates.duration(name)) for name in self.dpool.sigs.tools]
                        or [0.0], np.float64)
        self.benefit = bene
        self.adm_arrays[2].copy_(self.torch.from_numpy(bene))
        if self.plan is not None:  # utilities / per-tool winners live in the plan
            check(self.lib.paste_build_live_plan(ctypes.byref(self.pool_desc),
                                                 ctypes.byref(self.adm), self.K, self.W,
                                                 self.plan.plan, stream_handle()), self.lib)
            self._entries = None
            fmt8 = self.sformat & _native.PASTE_CF_KEY8
            self._assign_plan_codes()  # entry contents changed: codes and host copy
            if fmt8 and self.plan_codes is None:
                self.sformat &= ~_native.PASTE_CF_KEY8

    # -- state upload ---------------------------------------------------------

    def region_bytes(self, region: int):
        b0 = region * self.max_batch_bytes
        return self.bytes[b0:b0 + self.max_batch_bytes]

    def stage(self, batch: EventBatch, region: int, non_blocking: bool = True):
        """Copy a batch into the staging inputs and its arena region."""
        t = self.torch
        tok = batch.tok if isinstance(batch.tok, t.Tensor) else t.from_numpy(batch.tok)
        ref = batch.ref if isinstance(batch.ref, t.Tensor) else t.from_numpy(batch.ref)
        data = batch.data if isinstance(batch.data, t.Tensor) else t.from_numpy(batch.data)
        self.staged8 = self.narrow8 and batch.tok8 is not None
        if self.staged8:
            node16 = batch.node16
            if batch.node8 is not None:  # the 2-byte form: node codes -> node_base here
                code = batch.node8.cpu().numpy() if isinstance(batch.node8, t.Tensor) \
                    else np.asarray(batch.node8)
                node16 = self.codes.host.numpy()[code.astype(np.int64)].astype(np.uint16)
            for d, x in ((self.new_tok8, batch.tok8), (self.new_node16, node16)):
                x = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(x))
                d.copy_(x.reshape(-1).view(d.dtype), non_blocking=non_blocking)
            return
        self.new_tok.copy_(tok.reshape(-1), non_blocking=non_blocking)
        self.narrow = batch.node is not None and not self.ship_bytes
        if self.narrow:  # node_base only: 8 B/session on the wire with the token
            node = batch.node if isinstance(batch.node, t.Tensor) else t.from_numpy(batch.node)
            self.new_node.copy_(node.reshape(-1), non_blocking=non_blocking)
        else:
            self.new_ref.copy_(ref.reshape(-1), non_blocking=non_blocking)
        if self.ship_bytes:
            if data.numel() > self.max_batch_bytes:
                raise ValueError("event batch exceeds the arena region size")
            self.region_bytes(region)[:data.numel()].copy_(data.reshape(-1),
                                                           non_blocking=non_blocking)

    def launch(self, region: int, new_tok=None, new_ref=None, new_node=None) -> None:
        """observe (new event per session) + predict + admit, one kernel."""
        staged8 = new_tok is None and new_ref is None and new_node is None and self.staged8
        if new_tok is None and new_ref is None and new_node is None and self.narrow:
            new_node = self.new_node
        ref = None if new_node is not None else (self.new_ref if new_ref is None else new_ref)
        win = WindowsDesc(self.n, self.W, 1, ptr(self.tok), ptr(self.evt), ptr(self.count),
                          ptr(self.nodes), ptr(self.bytes), ptr(self.refs),
                          ptr(self.new_tok if new_tok is None else new_tok), ptr(ref),
                          region * self.n, region * self.max_batch_bytes, 0, ptr(new_node))
        if staged8:
            win.new_tok, win.new_ref, win.new_node = None, None, None
            win.new_tok8, win.new_node16 = ptr(self.new_tok8), ptr(self.new_node16)
        if self.plan is not None:
            check(self.lib.paste_predict_live(ctypes.byref(self.pool_desc), ctypes.byref(win),
                                              ctypes.byref(self.adm), ctypes.byref(self.plan),
                                              ctypes.byref(self.out_desc), stream_handle()),
                  self.lib)
            return
        check(self.lib.paste_predict_batch(ctypes.byref(self.pool_desc), ctypes.byref(win),
                                           ctypes.byref(self.adm), ctypes.byref(self.out_desc),
                                           stream_handle()), self.lib)

    def compact_scratch_bytes(self) -> int:
        """Scratch for launch_compact (either serving kernel) and the
        compaction kernel."""
        return max(self.lib.paste_compact_scratch_bytes(self.n),
                   self.lib.paste_predict_compact_scratch_bytes(self.n),
                   self.lib.paste_predict_live_compact_scratch_bytes(self.n, self.K, self.B))

    def launch_compact(self, region: int, cdesc, scratch, new_tok=None, new_node=None,
                       new_ref=None) -> bool:
        """observe + predict + admit writing the narrow record streams
        directly (paste_predict_compact); False when the pool / envelope
        needs the two-kernel path (launch + paste_compact_records)."""
        if new_tok is None:
            new_tok = self.new_tok
            if self.narrow:
                new_node = self.new_node
        ref = None if new_node is not None else (self.new_ref if new_ref is None else new_ref)
        win = WindowsDesc(self.n, self.W, 1, ptr(self.tok), ptr(self.evt), ptr(self.count),
                          ptr(self.nodes), ptr(self.bytes), ptr(self.refs), ptr(new_tok),
                          ptr(ref), region * self.n, region * self.max_batch_bytes, 0,
                          ptr(new_node))
        if self.plan is not None:
            rc = self.lib.paste_predict_live_compact(
                ctypes.byref(self.pool_desc), ctypes.byref(win), ctypes.byref(self.adm),
                ctypes.byref(self.plan), self.B, ctypes.byref(cdesc), ptr(scratch),
                scratch.numel(), stream_handle())
            if rc != _native.PASTE_ERR_UNSUPPORTED:
                check(rc, self.lib)
                return True
        rc = self.lib.paste_predict_compact(ctypes.byref(self.pool_desc), ctypes.byref(win),
                                            ctypes.byref(self.adm), self.K, self.B,
                                            ctypes.byref(cdesc), ptr(scratch), stream_handle())
        if rc == _native.PASTE_ERR_UNSUPPORTED:
            return False
        check(rc, self.lib)
        return True

    def step(self, batch: EventBatch) -> None:
        """Stage one batch of new events and run the fused step (async)."""
        region = self.steps % self.regions
        self.stage(batch, region)
        self.launch(region)
        self.steps += 1

    # -- results ----------------------------------------------------------------

    def action_keys(self):
        """Scheduler cache keys of this step's admitted actions, computed on
        the device from the K-slot records (paste_action_keys): (keys
        u8[n*K, 16], state u8[n*K]) device tensors in action-slot order;
        state 0 = key, 1 = WARM_ONLY (no argument key), 2 = decide on the
        host (``canonical_arg_hash`` of the decoded arguments)."""
        from ._native import ActionKeysDesc
        from .hashing import key_tables
        from .replay import KeysetTable, pool_hit_tables

        t = self.torch
        if not self.ship_bytes:
            raise ValueError("action keys hash argument values: build the table with "
                             "ship_bytes=True so payload bytes live on the device")
        if getattr(self, "_keys", None) is None:
            _, bind_key, fmt, fbytes = pool_hit_tables(self.dpool, KeysetTable())
            self._keys = {"bind_key": to_dev(bind_key), "fmt": to_dev(fmt), "fbytes": to_dev(fbytes),
                          "keys": t.zeros(self.n * self.K * 16, dtype=t.uint8, device="cuda"),
                          "state": t.zeros(self.n * self.K, dtype=t.uint8, device="cuda")}
        k = self._keys
        kb, ko, kr = (to_dev(a) for a in key_tables(self.dpool.keys))
        d = ActionKeysDesc(self.n, self.pool_desc, self.out_desc, ptr(self.nodes), ptr(self.bytes),
                           ptr(self.refs), ptr(kb), ptr(ko), ptr(kr), ptr(k["bind_key"]),
                           ptr(k["fmt"]), ptr(k["fbytes"]), ptr(k["keys"]), ptr(k["state"]))
        check(self.lib.paste_action_keys(ctypes.byref(d), stream_handle()), self.lib)
        t.cuda.current_stream().synchronize()  # the key tables above are temporaries
        return k["keys"].view(self.n * self.K, 16), k["state"]

    def entries(self):
        """Host copy of the match table's prediction lists (for
        PASTE_CF_ENTRY16 records): (n_match[keys], pattern ids[keys, K])."""
        if self._entries is None:
            table, _ = self.dpool.match_table(self.pool_desc, self.K, self.W)
            raw = table.cpu().numpy()
            stride = 16 + 32 * self.K
            rows = raw.reshape(-1, stride)
            n_match = rows[:, :4].copy().view(np.int32)[:, 0]
            recs = rows[:, 16:].copy().view(np.int32).reshape(len(rows), self.K, 8)
            self._entries = (n_match, recs[:, :, 0].copy())
        return self._entries

    def plan_host(self):
        """Host copy of the live plan for expanding PASTE_CF_KEYS streams:
        per key (n_pred, n_act, action codes [keys, K] = slot | level if
        complete << 8 | level if PARTIAL << 12, n_map, n_units, map words
        [keys, M] = binding | rank << 32 | bslot << 40 | age << 48 | unit
        << 56, representative key per u8 plan code [256] (-1 = none) or
        None)."""
        if self._plan_host is None:
            buf = self._plan_bufs[0].cpu().numpy()
            K, M = self.K, self.K * max(self.dpool.image.max_bindings, 1)
            L = plan_layout_host(K, M)
            off_act, off_map = L["off_act"], L["off_map"]
            rows = buf.reshape(-1, L["stride"])
            self._plan_host = (rows[:, 0].astype(np.int64), rows[:, 1].astype(np.int64),
                               rows[:, off_act:off_act + 2 * K].copy().view(np.uint16),
                               rows[:, 2].astype(np.int64), rows[:, 3].astype(np.int64),
                               rows[:, off_map:off_map + 8 * M].copy().view(np.uint64),
                               self.plan_codes[1] if self.plan_codes is not None else None)
        return self._plan_host

    def output_nbytes(self) -> int:
        return sum(v.numel() * v.element_size() for v in self.out.values())

    def fetch(self, pinned: dict | None = None) -> PredictResult:
        """D2H copy of the output records (into pinned buffers if given)."""
        if pinned is not None:
            for k, v in self.out.items():
                pinned[k].copy_(v, non_blocking=True)
            self.torch.cuda.current_stream().synchronize()
            h = {k: v.numpy() for k, v in pinned.items()}
        else:
            h = {k: v.cpu().numpy() for k, v in self.out.items()}
        return PredictResult(self.K, self.B, h["n_pred"], h["pred_pat"], h["pred_comp"],
                             h["pred_arg"], h["n_act"], h["act_pred"], h["act_level"],
                             h["act_util"], h["struct_err"], 1)

    def pinned_outputs(self) -> dict:
        t = self.torch
        return {k: t.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in self.out.items()}

    def host_state(self) -> dict:
        """Copies of the window rings / directory (for oracle cross-checks)."""
        return {"tok": self.tok.cpu().numpy(), "evt": self.evt.cpu().numpy(),
                "count": self.count.cpu().numpy(),
                "refs": self.refs.cpu().numpy().reshape(-1, 2),
                "bytes": self.bytes.cpu().numpy()}


@dataclass
class CompactRecords:
    """Host copy of the narrow CSR record streams of one live step
    (compact.cu; element widths per ``fmt``, PASTE_CF_* bits)."""

    K: int
    B: int
    hdr: np.ndarray    # n_pred | n_act << 8 (u16), or << 4 (u8, HDR8)
    pred: np.ndarray   # pattern | completeness << 14 (u16), or << 6 (u8, PRED8)
    arg: np.ndarray    # region << 27 | node (u32), or << 11 (u16, ARG16); all-ones = unresolved
    act: np.ndarray    # u8: slot | level << 5
    fmt: int = 0
    entries: tuple | None = None  # (n_match, pattern ids [keys, K]) for PASTE_CF_ENTRY16
    plan: tuple | None = None     # LiveSessionTable.plan_host() for PASTE_CF_KEYS

    @property
    def nbytes(self) -> int:
        return 32 + sum(a.nbytes for a in (self.hdr, self.pred, self.arg, self.act))

    def expand(self, patterns: np.ndarray, benefit: np.ndarray) -> PredictResult:
        """Back to fixed per-session records (for decoding / comparisons).
        Utilities are p(pattern) * benefit(target tool): the same IEEE
        multiply the device did (policy.py:224-232)."""
        K, B = self.K, self.B
        keys = bool(self.fmt & _native.PASTE_CF_KEYS)
        if keys:  # counts from the key's live-plan entry
            if self.fmt & _native.PASTE_CF_KEY8:  # u8 plan code -> a key with its content
                key = self.plan[6][self.pred.astype(np.int64)]
                valid = key >= 0
            else:
                key = self.pred.astype(np.int64)
                valid = key != 0xFFFF
            kk = np.where(valid, key, 0)
            n_pred = np.where(valid, self.plan[0][kk], 0)
            n_act = np.where(valid, self.plan[1][kk], 0)
        else:
            hdr = self.hdr.astype(np.int64)
            hshift = 4 if self.fmt & _native.PASTE_CF_HDR8 else 8
            n_pred, n_act = hdr & ((1 << hshift) - 1), hdr >> hshift
        n = len(n_pred)
        res = PredictResult.empty(n, K, B, True)
        res.n_pred[:] = n_pred
        res.n_act[:] = n_act
        sess = np.repeat(np.arange(n), n_pred)
        slot = np.arange(len(sess)) - np.repeat(np.cumsum(n_pred) - n_pred, n_pred)
        a16 = bool(self.fmt & _native.PASTE_CF_ARG16)
        ashift = 11 if a16 else 27
        a = self.arg.astype(np.int64)
        unresolved = a == (0xFFFF if a16 else 0xFFFFFFFF)
        if self.fmt & _native.PASTE_CF_ENTRY16:
            # the session's match-table entry lists its predictions; PARTIAL =
            # a mapped prediction with an unresolved reference
            kidx = kk if keys else self.pred.astype(np.int64)
            pid = self.entries[1][kidx[sess], slot].astype(np.int64)
            mapped = (patterns["flags"][pid] & 1) != 0
            nb = np.where(mapped, patterns["n_bind"][pid], 0)
            res.pred_pat[sess * K + slot] = pid
            if not self.fmt & _native.PASTE_CF_UNIQ:  # (else from the units, below)
                cu = np.concatenate([[0], np.cumsum(unresolved)])
                start = np.cumsum(nb) - nb
                partial = (cu[start + nb] - cu[start]) > 0
                comp = np.where(mapped, np.where(partial, 1, 0), 2)
                res.pred_comp[sess * K + slot] = comp.astype(np.uint8)
                part_at = np.zeros(n * K, bool)
                part_at[sess * K + slot] = mapped & partial
        else:
            pshift = 6 if self.fmt & _native.PASTE_CF_PRED8 else 14
            pred = self.pred.astype(np.int64)
            pid = pred & ((1 << pshift) - 1)
            res.pred_pat[sess * K + slot] = pid
            res.pred_comp[sess * K + slot] = (pred >> pshift).astype(np.uint8)
            mapped = (patterns["flags"][pid] & 1) != 0
            nb = np.where(mapped, patterns["n_bind"][pid], 0)
        if self.fmt & _native.PASTE_CF_UNIQ:
            # one reference per resolution unit: binding q of the entry reads
            # its unit's reference (map word bits 56-63)
            nmap = np.where(valid, self.plan[3][kk], 0)
            nu = np.where(valid, self.plan[4][kk], 0)
            q_sess = np.repeat(np.arange(n), nmap)
            q_idx = np.arange(len(q_sess)) - np.repeat(np.cumsum(nmap) - nmap, nmap)
            w = self.plan[5][kk[q_sess], q_idx]
            rank = ((w >> np.uint64(32)) & np.uint64(0xFF)).astype(np.int64)
            bslot = ((w >> np.uint64(40)) & np.uint64(0xFF)).astype(np.int64)
            unit = (w >> np.uint64(56)).astype(np.int64)
            word = a[(np.cumsum(nu) - nu)[q_sess] + unit]
            bad = word == (0xFFFF if a16 else 0xFFFFFFFF)
            part_q = np.zeros(n * K, bool)
            part_q[(q_sess * K + rank)[bad]] = True
            comp = np.where(mapped, np.where(part_q[sess * K + slot], 1, 0), 2)
            res.pred_comp[sess * K + slot] = comp.astype(np.uint8)
            part_at = part_q
            ev = (word >> ashift) * n + q_sess
            res.pred_arg[(q_sess * K + rank) * B + bslot] = np.where(
                bad, -1, (ev << 32) | (word & ((1 << ashift) - 1)))
        else:
            p_sess, p_slot = np.repeat(sess, nb), np.repeat(slot, nb)
            b_idx = np.arange(int(nb.sum())) - np.repeat(np.cumsum(nb) - nb, nb)
            ev = (a >> ashift) * n + p_sess
            res.pred_arg[(p_sess * K + p_slot) * B + b_idx] = np.where(
                unresolved, -1, (ev << 32) | (a & ((1 << ashift) - 1)))
        a_sess = np.repeat(np.arange(n), n_act)
        a_slot = np.arange(len(a_sess)) - np.repeat(np.cumsum(n_act) - n_act, n_act)
        if keys:  # the entry's admit decisions; PARTIAL predictions at their partial level
            code = self.plan[2][kk[a_sess], a_slot].astype(np.int64)
            a_pred = code & 0xFF
            lv = np.where(part_at[a_sess * K + a_pred], (code >> 12) & 15, (code >> 8) & 15)
            res.act_pred[a_sess * K + a_slot] = a_pred
            res.act_level[a_sess * K + a_slot] = lv.astype(np.uint8)
        else:
            a_pred = (self.act & 31).astype(np.int64)
            res.act_pred[a_sess * K + a_slot] = a_pred
            res.act_level[a_sess * K + a_slot] = self.act >> 5
        a_pid = res.pred_pat[a_sess * K + a_pred]
        res.act_util[a_sess * K + a_slot] = (patterns["p"][a_pid]
                                             * benefit[patterns["target_tool"][a_pid]])
        return res


def _compact_buffers(table: "LiveSessionTable", f: int | None = None):
    t = table.torch
    n, K, B = table.n, table.K, table.B
    f = table.cformat if f is None else f
    dev = t.device("cuda")
    entry = bool(f & _native.PASTE_CF_ENTRY16)
    if f & _native.PASTE_CF_KEYS:  # totals | keys | args in one buffer: one download copy
        return _keys_buffers(t, n * K * B, n, bool(f & _native.PASTE_CF_ARG16), dev,
                             kb=_key_bytes(f))
    return {"hdr": t.zeros(n, dtype=t.uint8 if f & _native.PASTE_CF_HDR8 else t.int16, device=dev),
            "pred": t.zeros(n if entry else n * K,
                            dtype=t.uint8 if f & _native.PASTE_CF_PRED8 and not entry else t.int16,
                            device=dev),
            "arg": t.zeros(n * K * B, dtype=t.int16 if f & _native.PASTE_CF_ARG16 else t.int32,
                           device=dev),
            "act": t.zeros(n * K, dtype=t.uint8, device=dev),
            "totals": t.zeros(5, dtype=t.int64, device=dev)}


def keys_layout(n: int, arg_cap: int, a16: bool, kb: int = 2) -> tuple[int, int, int]:
    """Byte offsets of the key-stream buffer: totals (5 x i64) at 0, the
    keys (u16, or u8 plan codes: kb = 1) at `k_off`, the argument words at
    `a_off`; `size` in total."""
    k_off = 64
    a_off = (k_off + kb * n + 63) // 64 * 64
    return k_off, a_off, a_off + arg_cap * (2 if a16 else 4)


def plan_codes(rows: np.ndarray, K: int, M: int):
    """u8 plan codes of live-plan entries ``rows`` [keys, stride] (raw
    bytes, plan_layout_host): one code per distinct non-empty content in
    first-key order of np.unique, 0xFF for entries without predictions,
    actions or bindings.  Returns (codes [keys], representative key per
    code [256], -1 = unused), or None when more than 255 codes are needed."""
    L = plan_layout_host(K, M)
    nm, na, nmap = (rows[:, j].astype(np.int64) for j in (0, 1, 2))
    live = (nm > 0) | (na > 0) | (nmap > 0)

    def cols(off, width, slots, count):  # slots past an entry's count are never written
        keep = np.arange(slots)[None, :] < count[:, None]
        return np.where(np.repeat(keep, width, axis=1), rows[:, off:off + width * slots], 0)

    content = np.concatenate([
        rows[:, :4], cols(L["off_pid"], 4, K, nm), cols(L["off_comp"], 1, K, nm),
        cols(L["off_act"], 2, K, na), cols(L["off_util"], 8, K, na),
        cols(L["off_map"], 8, M, nmap)], axis=1)
    idx = np.flatnonzero(live)
    codes = np.full(len(rows), 0xFF, np.uint8)
    rep = np.full(256, -1, np.int64)
    if len(idx):
        uniq, first, inv = np.unique(content[idx], axis=0, return_index=True,
                                     return_inverse=True)
        if len(uniq) > 255:
            return None
        codes[idx] = inv.reshape(-1).astype(np.uint8)
        rep[:len(uniq)] = idx[first]
    return codes, rep


def _key_bytes(fmt: int) -> int:
    """Bytes per session of the key stream: u8 plan codes or u16 keys."""
    return 1 if fmt & _native.PASTE_CF_KEY8 else 2


def plan_layout_host(K: int, M: int) -> dict:
    """Byte offsets of a live-plan entry (live_plan.cu plan_layout): header
    (n_pred, n_act, n_map, n_units bytes, i32 structural errors, u8 plan
    code at 8), pattern ids, completeness, action codes, utilities, map
    words."""
    al = lambda x, a: (x + a - 1) // a * a  # noqa: E731
    off_comp = 16 + 4 * K
    off_act = al(off_comp + K, 16)
    off_util = al(off_act + 2 * K, 8)
    off_map = off_util + 8 * K
    return {"off_pid": 16, "off_comp": off_comp, "off_act": off_act, "off_util": off_util,
            "off_map": off_map, "stride": al(off_map + 8 * M, 16)}


def _keys_buffers(t, arg_cap: int, n: int, a16: bool, dev, pinned: bool = False,
                  kb: int = 2) -> dict:
    k_off, a_off, size = keys_layout(n, arg_cap, a16, kb)
    blob = (t.empty(size, dtype=t.uint8, pin_memory=True) if pinned
            else t.zeros(size, dtype=t.uint8, device=dev))
    z = (lambda m, dt: t.empty(m, dtype=dt, pin_memory=True)) if pinned else \
        (lambda m, dt: t.zeros(m, dtype=dt, device=dev))
    return {"blob": blob, "totals": blob[:40].view(t.int64),
            "pred": blob[k_off:k_off + kb * n].view(t.int16 if kb == 2 else t.uint8),
            "arg": blob[a_off:a_off + arg_cap * (2 if a16 else 4)].view(t.int16 if a16 else t.int32),
            "hdr": z(16, t.int16), "act": z(16, t.uint8)}  # not written in this form


def _compact_desc(c: dict, fmt: int = 0):
    from ._native import CompactDesc

    return CompactDesc(ptr(c["hdr"]), ptr(c["pred"]), ptr(c["arg"]), ptr(c["act"]),
                       ptr(c["totals"]), fmt, 0)


def _compact_init(table: "LiveSessionTable") -> None:
    t = table.torch
    table.cbuf = _compact_buffers(table)
    table.cscratch = t.empty(table.lib.paste_compact_scratch_bytes(table.n), dtype=t.uint8,
                             device="cuda")
    table.cdesc = _compact_desc(table.cbuf, table.cformat)


def _records(table, h: dict, f: int | None = None) -> CompactRecords:
    f = table.cformat if f is None else f
    entry = bool(f & _native.PASTE_CF_ENTRY16)
    return CompactRecords(
        table.K, table.B, h["hdr"].view(np.uint8 if f & _native.PASTE_CF_HDR8 else np.uint16),
        h["pred"].view(np.uint8 if f & _native.PASTE_CF_PRED8 and not entry else np.uint16),
        h["arg"].view(np.uint16 if f & _native.PASTE_CF_ARG16 else np.uint32), h["act"], f,
        table.entries() if entry else None)


def _sizes(table, totals, f: int | None = None) -> dict:
    P, A, Q, wide, _err = (int(x) for x in totals.tolist())
    if wide:
        raise _native.PasteError(f"{wide} argument refs outside the live table's event form: "
                                 "use fetch()")
    f = table.cformat if f is None else f
    return {"hdr": table.n, "pred": table.n if f & _native.PASTE_CF_ENTRY16 else P, "arg": A,
            "act": Q}


def fetch_compact(table: "LiveSessionTable", pinned: dict | None = None) -> CompactRecords:
    """Compact the step's records on the device (one scan kernel) and copy
    only the produced bytes back: totals first, then the sized streams."""
    t = table.torch
    if not hasattr(table, "cbuf"):
        _compact_init(table)
    check(table.lib.paste_compact_records(ctypes.byref(table.out_desc), table.n,
                                          ctypes.byref(table.pool_desc), ctypes.byref(table.cdesc),
                                          ptr(table.cscratch), stream_handle()), table.lib)
    c = table.cbuf
    if pinned is None:
        pinned = {k: t.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in c.items()}
    pinned["totals"].copy_(c["totals"], non_blocking=True)
    t.cuda.current_stream().synchronize()
    sizes = _sizes(table, pinned["totals"])
    for k, m in sizes.items():
        pinned[k][:m].copy_(c[k][:m], non_blocking=True)
    t.cuda.current_stream().synchronize()
    return _records(table, {k: pinned[k][:m].numpy() for k, m in sizes.items()})


_STREAMS = ("hdr", "pred", "arg", "act")


def _serve_state(table, depth: int, fmt: int) -> dict:
    """Buffer sets, pinned mirrors, numpy views, copy lists and reusable
    events of the serving loop (built once per (depth, format)): `depth`
    device sets, `2 * depth` pinned host sets (records are handed out
    depth - 1 steps behind the launches, and a yielded record's pinned set
    is not overwritten until the generator has advanced depth - 1 more
    steps)."""
    t = table.torch
    bufs = [_compact_buffers(table, fmt) for _ in range(depth)]
    keys = bool(fmt & _native.PASTE_CF_KEYS)
    if keys:
        pinned = [_keys_buffers(t, bufs[0]["arg"].numel(), table.n,
                                bool(fmt & _native.PASTE_CF_ARG16), None, pinned=True,
                                kb=_key_bytes(fmt))
                  for _ in range(2 * depth)]
    else:
        pinned = [{k: t.empty(v.shape, dtype=v.dtype, pin_memory=True)
                   for k, v in bufs[0].items()} for _ in range(2 * depth)]
    entry = bool(fmt & _native.PASTE_CF_ENTRY16)
    vdt = {"hdr": np.uint8 if fmt & _native.PASTE_CF_HDR8 else np.uint16,
           "pred": (np.uint8 if (fmt & _native.PASTE_CF_PRED8 and not entry)
                    or fmt & _native.PASTE_CF_KEY8 else np.uint16),
           "arg": np.uint16 if fmt & _native.PASTE_CF_ARG16 else np.uint32, "act": np.uint8}
    names = ("totals",) + _STREAMS
    hsets = [{"views": {k: h[k].numpy().view(vdt[k]) for k in _STREAMS},
              "totals": h["totals"].numpy(),
              "dst": (ctypes.c_void_p * 5)(*[h[k].data_ptr() for k in names]),
              "ptr": {k: h[k].data_ptr() for k in names},
              "base": h["blob"].data_ptr() if keys else None}
             for h in pinned]
    dsets = [{"src": (ctypes.c_void_p * 5)(*[c[k].data_ptr() for k in names]),
              "ptr": {k: c[k].data_ptr() for k in names},
              "esize": [c[k].element_size() for k in _STREAMS],
              "cap": [c[k].numel() for k in _STREAMS],
              "base": c["blob"].data_ptr() if keys else None}
             for c in bufs]
    return {
        "fmt": fmt, "bufs": bufs, "descs": [_compact_desc(c, fmt) for c in bufs],
        "pinned": pinned, "hsets": hsets, "dsets": dsets,
        "bytes": (ctypes.c_int64 * 5)(),
        "bound": [None] * 4,  # per variable stream: elements the async download copies
        "scratch": [t.empty(table.compact_scratch_bytes(),
                            dtype=t.uint8, device="cuda") for _ in range(depth)],
        "copy": t.cuda.Stream(), "up": t.cuda.Stream(), "sup": t.cuda.Stream(),
        "free": [None] * depth, "in_free": [None] * depth,
        "ev_ready": [t.cuda.Event() for _ in range(depth)],
        "ev_up": [t.cuda.Event() for _ in range(depth)],
        "wins": {},
        "in": [_in_set(t, table.n) for _ in range(depth)]}


def _in_set(t, n: int) -> dict:
    off, size = wire8_layout(n)
    packed = t.zeros(size, dtype=t.uint8, device="cuda")
    return {"packed": packed, "tok8": packed[:n], "node16": packed[off:off + 2 * n].view(t.int16),
            "node8": packed[off:off + n], "n2": wire8_layout(n, 1)[1],
            "tok": t.zeros(n, dtype=t.int32, device="cuda"),
            "node": t.zeros(n, dtype=t.int32, device="cuda"),
            "ref": t.zeros(2 * n, dtype=t.int64, device="cuda")}


def serve(table: "LiveSessionTable", batches, depth: int = 4):
    """Pipelined live steps (the serving loop).  Step i+1's inputs upload on
    an upload stream into their own staging set while step i's fused
    predict + compaction kernel runs on the compute stream; step i's
    download is queued on a copy stream right behind its kernel, with no
    host round trip: the variable-length streams are copied up to a bound
    (the largest recent count plus a margin) together with the step's
    totals, and the rare step that outgrows its bound fetches the rest when
    it is handed out.  So the two copy engines and the SMs overlap and the
    host only waits for records it hands out.  The host side is kept thin:
    each step's copies go out as one ``paste_memcpy_batch`` call per
    direction, window descriptors are cached per (buffer set, arena region)
    and events are reused.  Yields each step's CompactRecords in order
    (``records.downloaded`` is the device event of its download); a yielded
    record's arrays are pinned-buffer views, valid until the generator has
    advanced ``depth - 1`` more steps."""
    from collections import deque

    if depth < 3:
        raise ValueError("serve() needs depth >= 3 buffer sets")
    t = table.torch
    lib = table.lib
    fmt = table.sformat if table.serve_fused else table.cformat
    if (getattr(table, "_serve", None) is None or len(table._serve["bufs"]) != depth
            or table._serve["fmt"] != fmt):
        table._serve = _serve_state(table, depth, fmt)
    sv = table._serve
    comp, copy, up = t.cuda.current_stream(), sv["copy"], sv["up"]
    comp_h, copy_h, up_h = (s.cuda_stream for s in (comp, copy, up))
    entries = table.entries() if fmt & _native.PASTE_CF_ENTRY16 else None
    plan = table.plan_host() if fmt & _native.PASTE_CF_KEYS else None
    n = table.n
    keys = bool(fmt & _native.PASTE_CF_KEYS)  # counts / actions follow from the key
    # stream sizes fixed by the format (None = variable, from the totals)
    fixed = (0 if keys else n, n if fmt & _native.PASTE_CF_ENTRY16 else None, None,
             0 if keys else None)
    bound = sv["bound"]
    margin = getattr(table, "serve_bound_margin", None)
    copy_q = deque()
    H2D, D2H = _native.PASTE_COPY_H2D, _native.PASTE_COPY_D2H
    nh = 2 * depth  # pinned sets: a handed-out record outlives depth - 1 more steps
    a_off = keys_layout(n, 0, True, _key_bytes(fmt))[1] if keys else 0

    def actual_sizes(tot):
        P, A, Q = int(tot[0]), int(tot[1]), int(tot[2])
        return [fixed[0], fixed[1] if fixed[1] is not None else P, A,
                fixed[3] if fixed[3] is not None else Q]

    def download(k, h, step):
        """Queue step's download (device set k -> pinned set h) behind its
        kernel on the copy stream."""
        ds, hs = sv["dsets"][k], sv["hsets"][h]
        copy.wait_event(sv["ev_ready"][k])
        nb = sv["bytes"]
        nb[0] = 5 * 8
        if any(bound[j] is None for j in range(4) if fixed[j] is None):
            # no bound yet: the sizes come from this step's totals (host round trip)
            check(lib.paste_memcpy_batch(1, hs["dst"], ds["src"], nb, D2H, copy_h), lib)
            copy.synchronize()
            sizes = actual_sizes(hs["totals"])
        else:
            sizes = [fixed[j] if fixed[j] is not None else min(bound[j], ds["cap"][j])
                     for j in range(4)]
        for j in range(4):
            nb[1 + j] = sizes[j] * ds["esize"][j]
        if trace is not None:
            trace[step]["d0"] = _tev(t, copy)
        if keys:  # totals | keys | args[:bound]: one contiguous copy
            one = (ctypes.c_int64 * 1)(a_off + nb[3])
            copied = int(one[0])
            check(lib.paste_memcpy_batch(1, (ctypes.c_void_p * 1)(hs["base"]),
                                         (ctypes.c_void_p * 1)(ds["base"]), one, D2H, copy_h), lib)
        else:
            check(lib.paste_memcpy_batch(5, hs["dst"], ds["src"], nb, D2H, copy_h), lib)
            copied = sum(int(nb[j]) for j in range(5))
        done = t.cuda.Event(enable_timing=True)
        done.record(copy)
        if trace is not None:
            trace[step]["d1"] = done
        sv["free"][k] = done
        copy_q.append((k, h, sizes, done, copied))

    def hand_out():
        k, h, sizes, done, copied = copy_q.popleft()
        if spin:  # poll: a sleeping wait wakes tens of microseconds late
            while not done.query():
                pass
        else:
            done.synchronize()
        hs, ds = sv["hsets"][h], sv["dsets"][k]
        tot = hs["totals"]
        if int(tot[3]):
            raise _native.PasteError(f"{int(tot[3])} argument refs outside the live table's "
                                     "event form: use fetch()")
        need = actual_sizes(tot)
        for j, name in enumerate(_STREAMS):
            if fixed[j] is not None:
                continue
            if need[j] > sizes[j]:  # outgrew the bound: fetch the rest (device set k is
                es = ds["esize"][j]  # not reused before this step's download is done)
                nb1 = (ctypes.c_int64 * 1)((need[j] - sizes[j]) * es)
                sup = sv["sup"]  # its own stream: not behind later steps' downloads
                check(lib.paste_memcpy_batch(
                    1, (ctypes.c_void_p * 1)(hs["ptr"][name] + sizes[j] * es),
                    (ctypes.c_void_p * 1)(ds["ptr"][name] + sizes[j] * es), nb1, D2H,
                    sup.cuda_stream), lib)
                sup.synchronize()
                copied += int(nb1[0])
                sv["supplements"] = sv.get("supplements", 0) + 1
            # the bound follows the largest recent count with 1/32 headroom
            # (a step past it costs a synchronous fetch of the rest, on a
            # side stream; the headroom is D2H bytes every step)
            grow = need[j] + (need[j] >> 5) + 1024 if margin is None else int(margin)
            bound[j] = grow if bound[j] is None else max(grow, (bound[j] * 127) // 128)
        v = hs["views"]
        rec = CompactRecords(table.K, table.B, v["hdr"][:need[0]], v["pred"][:need[1]],
                             v["arg"][:need[2]], v["act"][:need[3]], fmt, entries, plan)
        rec.downloaded = done  # device event: this step's records are on the host
        rec.wire_bytes = copied  # bytes this step's download moved (bound slack included)
        return rec

    def upload(i, b):
        """Stage step i's inputs into set i % depth on the upload stream, once
        the kernel that last read that set is done; returns the event."""
        k = i % depth
        region = (steps0 + i) % table.regions  # the arena region step i will use
        if sv["in_free"][k] is not None:
            up.wait_event(sv["in_free"][k])
        if trace is not None:
            trace.append({"u0": _tev(t, up)})
        st = sv["in"][k]
        narrow = b.node is not None and not table.ship_bytes
        if table.narrow8 and table.serve_fused and b.ev8 is not None:  # 1 B: event code
            narrow = "event"  # (not 1: True == 1 is the 8 B/session node form's flag)
            table.codes.upload(up)
            table.ecodes.upload(up)
            wire = [(st["tok8"], b.ev8)]
        elif (table.narrow8 and table.serve_fused and b.tok8 is not None
                and b.node8 is not None):  # 2 B per session: token + node code
            narrow = 2
            table.codes.upload(up)
            wire = ([(st["packed"][:b.packed.numel()], b.packed)]
                    if isinstance(b.packed, t.Tensor) and b.packed.numel() == st["n2"]
                    else [(st["tok8"], b.tok8), (st["node8"], b.node8)])
        elif table.narrow8 and table.serve_fused and b.tok8 is not None:  # 3 B per session
            narrow = 8
            wire = ([(st["packed"], b.packed)]
                    if isinstance(b.packed, t.Tensor) and b.packed.numel() == st["packed"].numel()
                    else [(st["tok8"], b.tok8), (st["node16"], b.node16)])
        else:
            wire = [(st["tok"], b.tok), (st["node"], b.node) if narrow else (st["ref"], b.ref)]
        if all(isinstance(x, t.Tensor) and not x.is_cuda and x.is_pinned() for _, x in wire):
            nw = len(wire)
            check(lib.paste_memcpy_batch(
                nw, (ctypes.c_void_p * nw)(*[d.data_ptr() for d, _ in wire]),
                (ctypes.c_void_p * nw)(*[x.data_ptr() for _, x in wire]),
                (ctypes.c_int64 * nw)(*[x.numel() * x.element_size() for _, x in wire]),
                H2D, up_h), lib)
        else:
            with t.cuda.stream(up):
                for d, x in wire:
                    x = x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(x))
                    d.copy_(x.reshape(-1).view(d.dtype), non_blocking=True)
        if table.ship_bytes:
            with t.cuda.stream(up):
                data = b.data if isinstance(b.data, t.Tensor) else t.from_numpy(b.data)
                table.region_bytes(region)[:data.numel()].copy_(data.reshape(-1),
                                                                non_blocking=True)
        ev = sv["ev_up"][k]
        ev.record(up)
        if trace is not None:
            trace[-1]["u1"] = _tev(t, up)
        return ev, narrow

    def launch_fused(k, region, st, narrow) -> bool:
        key = (k, region, narrow)
        win = sv["wins"].get(key)
        if win is None:
            win = WindowsDesc(n, table.W, 1, ptr(table.tok), ptr(table.evt), ptr(table.count),
                              ptr(table.nodes), ptr(table.bytes), ptr(table.refs), ptr(st["tok"]),
                              None if narrow else ptr(st["ref"]), region * n,
                              region * table.max_batch_bytes, 0,
                              ptr(st["node"]) if narrow else None)
            if narrow == 8:
                win.new_tok, win.new_node = None, None
                win.new_tok8, win.new_node16 = ptr(st["tok8"]), ptr(st["node16"])
            elif narrow == 2:
                win.new_tok, win.new_node = None, None
                win.new_tok8, win.new_node16 = ptr(st["tok8"]), None
                win.new_node8, win.node_codes = ptr(st["node8"]), ptr(table.codes.dev)
            elif narrow == "event":
                win.new_tok, win.new_node = None, None
                win.new_tok8, win.new_node16 = ptr(st["tok8"]), None
                win.event_codes = ptr(table.ecodes.dev)
            sv["wins"][key] = win
        if table.plan is not None:
            scr = sv["scratch"][k]
            rc = lib.paste_predict_live_compact(ctypes.byref(table.pool_desc), ctypes.byref(win),
                                                ctypes.byref(table.adm), ctypes.byref(table.plan),
                                                table.B, ctypes.byref(sv["descs"][k]), ptr(scr),
                                                scr.numel(), comp_h)
            if rc != _native.PASTE_ERR_UNSUPPORTED:
                check(rc, lib)
                return True
        rc = lib.paste_predict_compact(ctypes.byref(table.pool_desc), ctypes.byref(win),
                                       ctypes.byref(table.adm), table.K, table.B,
                                       ctypes.byref(sv["descs"][k]), ptr(sv["scratch"][k]),
                                       comp_h)
        if rc == _native.PASTE_ERR_UNSUPPORTED:
            return False
        check(rc, lib)
        return True

    trace = getattr(table, "serve_trace", None)  # development: per-step timing events
    spin = os.environ.get("PASTE_SERVE_SPIN", "0") == "1"  # measured no faster
    it = iter(batches)
    steps0 = table.steps
    # uploads run `ahead` steps in front of the kernels, so the H2D engine
    # always has queued work whatever the host is doing
    ahead = max(1, min(int(os.environ.get("PASTE_SERVE_AHEAD", "2")), depth - 2))
    staged = deque()
    n_up = 0
    while len(staged) < ahead:
        nxt = next(it, None)
        if nxt is None:
            break
        staged.append(upload(n_up, nxt))
        n_up += 1
    i = 0
    while staged:
        k = i % depth
        h = sv.setdefault("hnext", 0)  # pinned sets rotate across serve() calls
        sv["hnext"] = (h + 1) % nh
        uploaded, narrow = staged.popleft()
        region = table.steps % table.regions
        st = sv["in"][k]
        if sv["free"][k] is not None:  # the set's previous download has finished
            comp.wait_event(sv["free"][k])
        comp.wait_event(uploaded)
        node_in = st["node"] if narrow else None
        ref_in = None if narrow else st["ref"]
        if trace is not None:
            trace[i]["k0"] = _tev(t, comp)
        fused = table.serve_fused and launch_fused(k, region, st, narrow)
        if not fused:
            if fmt & _native.PASTE_CF_ENTRY16:
                raise _native.PasteError("PASTE_CF_ENTRY16 needs the fused serving kernel")
            table.launch(region, st["tok"], ref_in, node_in)
            check(lib.paste_compact_records(ctypes.byref(table.out_desc), n,
                                            ctypes.byref(table.pool_desc),
                                            ctypes.byref(sv["descs"][k]),
                                            ptr(sv["scratch"][k]), comp_h), lib)
        table.steps += 1
        if trace is not None:
            trace[i]["k1"] = _tev(t, comp)
        ready = sv["ev_ready"][k]
        ready.record(comp)
        sv["in_free"][k] = ready
        download(k, h, i)
        # the next upload goes out now, before the host waits on anything
        nxt = next(it, None)
        if nxt is not None:
            staged.append(upload(n_up, nxt))
            n_up += 1
        i += 1
        if len(copy_q) > depth - 1:  # hand out step i - depth + 1
            yield hand_out()
    while copy_q:
        yield hand_out()


def _tev(t, stream):
    e = t.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


LiveSessionTable.serve = serve
LiveSessionTable.fetch_compact = fetch_compact

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
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import AdmitDesc, PredictOut, WindowsDesc, check, ptr
from .device_ops import DevicePool, stream_handle, to_dev
from .packing import PredictResult, admit_tables


@dataclass
class EventBatch:
    """One new tool event per session: tokens, batch-relative directory
    entries (node_base, byte_base) and the batch's scalar bytes."""

    tok: object   # i32[n]      (numpy or torch, host or device)
    ref: object   # i64[n, 2]
    data: object  # u8[bytes]

    def nbytes(self, with_data: bool = True) -> int:
        parts = (self.tok, self.ref, self.data) if with_data else (self.tok, self.ref)
        return sum(int(x.nbytes) if isinstance(x, np.ndarray) else x.numel() * x.element_size()
                   for x in parts)


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
        self.bytes = torch.zeros(max(self.regions * self.max_batch_bytes, 1), dtype=torch.uint8,
                                 device=dev)
        self.refs = torch.zeros(self.regions * n * 2, dtype=torch.int64, device=dev)
        self.new_tok = torch.zeros(n, dtype=torch.int32, device=dev)
        self.new_ref = torch.zeros(n * 2, dtype=torch.int64, device=dev)
        allow, level, bene = admit_tables(dpool.sigs, policy, estimates.duration)
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
        self.new_tok.copy_(tok.reshape(-1), non_blocking=non_blocking)
        self.new_ref.copy_(ref.reshape(-1), non_blocking=non_blocking)
        if self.ship_bytes:
            if data.numel() > self.max_batch_bytes:
                raise ValueError("event batch exceeds the arena region size")
            self.region_bytes(region)[:data.numel()].copy_(data.reshape(-1),
                                                           non_blocking=non_blocking)

    def launch(self, region: int, new_tok=None, new_ref=None) -> None:
        """observe (new event per session) + predict + admit, one kernel."""
        win = WindowsDesc(self.n, self.W, 1, ptr(self.tok), ptr(self.evt), ptr(self.count),
                          ptr(self.nodes), ptr(self.bytes), ptr(self.refs),
                          ptr(self.new_tok if new_tok is None else new_tok),
                          ptr(self.new_ref if new_ref is None else new_ref),
                          region * self.n, region * self.max_batch_bytes)
        check(self.lib.paste_predict_batch(ctypes.byref(self.pool_desc), ctypes.byref(win),
                                           ctypes.byref(self.adm), ctypes.byref(self.out_desc),
                                           stream_handle()), self.lib)

    def step(self, batch: EventBatch) -> None:
        """Stage one batch of new events and run the fused step (async)."""
        region = self.steps % self.regions
        self.stage(batch, region)
        self.launch(region)
        self.steps += 1

    # -- results ----------------------------------------------------------------

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

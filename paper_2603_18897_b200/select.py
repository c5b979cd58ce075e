"""K6: batched admission selection (greedy_speculative_selection) on the device."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import SelectDesc, check, ptr


def _torch():
    import torch

    return torch


def select_greedy_arrays(p, benefit, duration, cost, ids, slack: int, budget: int):
    """Device greedy selection over job columns (numpy or CUDA tensors);
    returns the chosen job indices in selection order (numpy int32)."""
    from .device_ops import stream_handle

    torch = _torch()
    lib = _native.lib()

    def dev(a, dt):
        if isinstance(a, torch.Tensor):
            return a.to(device="cuda", dtype=dt).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dt)

    n = int(len(p))
    cols = [dev(p, torch.float64), dev(benefit, torch.float64), dev(duration, torch.float64),
            dev(cost, torch.int32), dev(ids, torch.int64)]
    cap = max(min(slack, budget), 0)
    selected = torch.zeros(max(min(cap, n), 1), dtype=torch.int32, device="cuda")
    n_sel = torch.zeros(1, dtype=torch.int64, device="cuda")
    need = lib.paste_select_scratch_bytes(n)
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    d = SelectDesc(n, *[ptr(c) for c in cols], ptr(selected), ptr(n_sel))
    check(lib.paste_select_greedy(ctypes.byref(d), int(slack), int(budget), ptr(scratch), need,
                                  stream_handle()), lib)
    return selected[:int(n_sel.item())].cpu().numpy()


def greedy_select_jobs(jobs, slack: int, budget: int):
    """greedy_speculative_selection(jobs, slack, budget) with Job objects."""
    if not jobs:
        return []
    for j in jobs:  # the reference's Job.utility() divides by cost * duration
        if j.cost * j.duration_est_ms == 0:
            raise ZeroDivisionError("float division by zero")
    p = np.array([j.p for j in jobs], np.float64)
    bene = np.array([j.benefit_ms for j in jobs], np.float64)
    dur = np.array([j.duration_est_ms for j in jobs], np.float64)
    cost = np.array([j.cost for j in jobs], np.int64)
    if (cost < 1).any() or (cost > 2**31 - 1).any():
        raise ValueError("job costs must be positive int32 values")
    ids = np.array([j.id for j in jobs], np.int64)
    idx = select_greedy_arrays(p, bene, dur, cost.astype(np.int32), ids, slack, budget)
    return [jobs[i] for i in idx.tolist()]


def preemption_victim(jobs):
    """The job Stage 2 of schedule_tick aborts first (scheduling.py:571-578):
    ``min(victims, key=lambda j: (j.utility(), -j.id))`` on the device."""
    from .device_ops import stream_handle

    if not jobs:
        return None
    torch = _torch()
    lib = _native.lib()
    for j in jobs:
        if j.cost * j.duration_est_ms == 0:
            raise ZeroDivisionError("float division by zero")
    cols = [torch.tensor([getattr(j, f) for j in jobs], dtype=dt, device="cuda") for f, dt in (
        ("p", torch.float64), ("benefit_ms", torch.float64), ("duration_est_ms", torch.float64),
        ("cost", torch.int32), ("id", torch.int64))]
    out = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")
    d = SelectDesc(len(jobs), *[ptr(c) for c in cols], 0, 0)
    check(lib.paste_select_victim(ctypes.byref(d), ptr(out), ptr(scratch), stream_handle()), lib)
    i = int(out.item())
    return jobs[i] if i >= 0 else None

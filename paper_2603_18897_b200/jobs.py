"""A16: admitted speculative actions -> scheduler jobs, on the device.

``Scheduler._admit_action`` (scheduling.py:464-511) turns each admitted
``SpeculativeAction`` into a ``Job`` whose utility ``U = (p*T)/(c*d)``
(scheduling.py:59-60) drives greedy selection.  Per level, with mean =
``EstimateBook.duration(tool)`` and wf = ``warm_fraction``:

* WARM_ONLY: key ``(tool, "warm")``, d = max(wf*mean, 1e-9), T = wf*mean;
* DRY_RUN:   key ``(tool, canonical_arg_hash(args))``, d = max(mean, 1e-9), T = wf*mean;
* FULL:      same key, d = max(mean, 1e-9), T = mean;

an action whose key an earlier job of the batch holds is coalesced (no id);
the others take consecutive ids, and a job costing more than ``r_total`` is
dropped after taking its id.  ``paste_action_jobs`` computes all of this for
a batch entering a fresh scheduler (the cache / in-flight state of a running
``Scheduler`` is the sequential state machine, out of scope), and
``paste_live_actions`` feeds it straight from a live step's records, so a
live step -> job columns -> ``paste_select_greedy`` never leaves the GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from ._native import ActionsDesc, JobsOut, LiveActionsDesc, SelectDesc, check, ptr
from .policy import SpecLevel
from .scheduling import Job, JobKind


def _torch():
    import torch

    return torch


@dataclass
class JobColumns:
    """Device job columns in batch order (the K6 inputs)."""

    p: object
    benefit: object
    duration: object
    cost: object
    id: object
    action: object   # i64: source action index of each job
    n: int
    next_id: int

    def host(self) -> dict:
        return {k: getattr(self, k)[:self.n].cpu().numpy()
                for k in ("p", "benefit", "duration", "cost", "id", "action")}

    def select(self, slack: int, budget: int) -> np.ndarray:
        """greedy_speculative_selection over these jobs on the device:
        the chosen job indices in selection order."""
        from .select import select_greedy_arrays

        n = self.n
        return select_greedy_arrays(self.p[:n], self.benefit[:n], self.duration[:n],
                                    self.cost[:n], self.id[:n], slack, budget)


def tool_tables(tools: Sequence[str], estimates) -> tuple[np.ndarray, np.ndarray]:
    """Per-tool EstimateBook.duration / cost, read at call time (so EWMA
    updates are seen, as the reference reads them per action)."""
    mean = np.array([float(estimates.duration(t)) for t in tools] or [0.0], np.float64)
    cost = np.array([int(estimates.cost(t)) for t in tools] or [1], np.int64)
    if (cost < -2**31).any() or (cost > 2**31 - 1).any():
        raise ValueError("tool costs must fit int32")
    return mean, cost.astype(np.int32)


def action_jobs_arrays(tool, level, p, key, mean, cost, warm_fraction: float, r_total: int,
                       id_base: int = 1) -> JobColumns:
    """Job columns for action columns in batch order (numpy or CUDA
    tensors): tool i32, level u8 (SpecLevel), p f64, key u8[n,16]
    (canonical_arg_hash digests; ignored for WARM_ONLY); per-tool mean
    duration f64 and cost i32."""
    from .device_ops import stream_handle

    torch = _torch()
    lib = _native.lib()

    def dev(a, dt):
        if isinstance(a, torch.Tensor):
            return a.to(device="cuda", dtype=dt).contiguous()
        return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dt)

    n = int(len(p))
    cols = [dev(tool, torch.int32), dev(level, torch.uint8), dev(p, torch.float64),
            dev(key, torch.uint8).reshape(-1)]
    if cols[3].numel() < 16 * n:
        raise ValueError("key needs 16 bytes per action")
    tabs = [dev(mean, torch.float64), dev(cost, torch.int32)]
    m = max(n, 1)
    out = {"p": torch.empty(m, dtype=torch.float64, device="cuda"),
           "benefit": torch.empty(m, dtype=torch.float64, device="cuda"),
           "duration": torch.empty(m, dtype=torch.float64, device="cuda"),
           "cost": torch.empty(m, dtype=torch.int32, device="cuda"),
           "id": torch.empty(m, dtype=torch.int64, device="cuda"),
           "action": torch.empty(m, dtype=torch.int64, device="cuda"),
           "tot": torch.zeros(2, dtype=torch.int64, device="cuda")}
    a = ActionsDesc(n, *[ptr(c) for c in cols], len(tabs[0]), 0, ptr(tabs[0]), ptr(tabs[1]),
                    float(warm_fraction), int(r_total), int(id_base))
    tot = out["tot"]
    j = JobsOut(*[ptr(out[k]) for k in ("p", "benefit", "duration", "cost", "id", "action")],
                tot.data_ptr(), tot.data_ptr() + 8)
    need = lib.paste_action_jobs_scratch_bytes(n)
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    check(lib.paste_action_jobs(ctypes.byref(a), ctypes.byref(j), ptr(scratch), need,
                                stream_handle()), lib)
    n_jobs, next_id = (int(v) for v in tot.cpu().tolist())
    return JobColumns(out["p"], out["benefit"], out["duration"], out["cost"], out["id"],
                      out["action"], n_jobs, next_id)


def admit_action_batch(batches: Sequence[tuple[str, Sequence]], estimates, r_total: int,
                       id_base: int = 1, now: float = 0.0) -> tuple[list[Job | None], int]:
    """``Scheduler._admit_action`` for every action of ``batches`` (pairs of
    session id and that session's admitted ``SpeculativeAction`` list, in
    submission order) entering a fresh scheduler whose next id is
    ``id_base``.  Returns one ``Job`` or ``None`` (coalesced / over r_total)
    per action, in order, and the scheduler's next id."""
    from .hashing import canonical_arg_hash_batch

    acts = [(sid, a) for sid, lst in batches for a in lst]
    tools = sorted({a.prediction.tool_type for _, a in acts})
    tid = {t: i for i, t in enumerate(tools)}
    n = len(acts)
    level = np.array([int(a.level) for _, a in acts], np.uint8)
    nonwarm = [i for i in range(n) if level[i] != int(SpecLevel.WARM_ONLY)]
    hexes = canonical_arg_hash_batch([acts[i][1].prediction.args for i in nonwarm]) if nonwarm \
        else []
    key = np.zeros((max(n, 1), 16), np.uint8)
    arg_hash = ["warm"] * n
    for i, h in zip(nonwarm, hexes):
        key[i] = np.frombuffer(bytes.fromhex(h), np.uint8)
        arg_hash[i] = h
    mean, cost = tool_tables(tools, estimates)
    cols = action_jobs_arrays(np.array([tid[a.prediction.tool_type] for _, a in acts], np.int32),
                              level, np.array([a.prediction.probability for _, a in acts],
                                              np.float64),
                              key, mean, cost, estimates.warm_fraction, r_total, id_base)
    h = cols.host()
    jobs: list[Job | None] = [None] * n
    for r in range(cols.n):
        i = int(h["action"][r])
        sid, act = acts[i]
        warm = act.level is SpecLevel.WARM_ONLY or int(act.level) == int(SpecLevel.WARM_ONLY)
        jobs[i] = Job(id=int(h["id"][r]), kind=JobKind.SPECULATIVE,
                      tool_type=act.prediction.tool_type,
                      args={} if warm else act.prediction.args, arg_hash=arg_hash[i],
                      session_id=sid, p=float(h["p"][r]), benefit_ms=float(h["benefit"][r]),
                      cost=int(h["cost"][r]), duration_est_ms=float(h["duration"][r]),
                      submitted_at=now, level=SpecLevel(int(act.level)),
                      no_commit=bool(getattr(act, "no_commit", False)), preemptible=True)
    return jobs, cols.next_id


def live_action_columns(table) -> dict:
    """Flatten a live step's admitted actions (``LiveSessionTable`` K-slot
    records) into batch-order device columns, with the scheduler cache keys
    of ``paste_action_keys`` (unsure keys re-hashed on the host)."""
    from .device_ops import stream_handle

    torch = _torch()
    lib = table.lib
    keys, state = table.action_keys()
    st = state.cpu().numpy()
    if (st == 2).any():  # decide on the host: decode the arguments, hash them
        from .events import canonical_arg_hash
        from .packing import decode_actions, decode_predictions
        from .tape import ArrayTapes

        res = table.fetch().session_major()
        hs = table.host_state()
        arena = ArrayTapes(table.host_nodes, hs["bytes"], hs["refs"], table.dpool.keys)
        acts = decode_actions(res, decode_predictions(res, table.dpool.image, arena,
                                                      [0.0] * table.n, 0.0))
        kh = keys.cpu().numpy()
        for slot in np.nonzero(st == 2)[0]:
            j, s = divmod(int(slot), table.n)  # slot-major action records
            args = acts[s][j].prediction.args
            kh[slot] = np.frombuffer(bytes.fromhex(canonical_arg_hash(args)), np.uint8)
        keys = torch.from_numpy(kh).cuda()
    n, K = table.n, table.K
    m = n * K
    c = {"tool": torch.empty(m, dtype=torch.int32, device="cuda"),
         "level": torch.empty(m, dtype=torch.uint8, device="cuda"),
         "p": torch.empty(m, dtype=torch.float64, device="cuda"),
         "key": torch.empty(m * 16, dtype=torch.uint8, device="cuda"),
         "session": torch.empty(m, dtype=torch.int64, device="cuda"),
         "slot": torch.empty(m, dtype=torch.int32, device="cuda"),
         "n": torch.zeros(1, dtype=torch.int64, device="cuda")}
    d = LiveActionsDesc(n, table.pool_desc, table.out_desc, ptr(keys),
                        *[ptr(c[k]) for k in ("tool", "level", "p", "key", "session", "slot", "n")])
    need = lib.paste_live_actions_scratch_bytes(n)
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    check(lib.paste_live_actions(ctypes.byref(d), ptr(scratch), need, stream_handle()), lib)
    c["n"] = int(c["n"].item())
    c["_keys"] = keys  # keep the key buffer alive with the columns
    return c


def live_step_jobs(table, estimates, r_total: int, id_base: int = 1) -> tuple[dict, JobColumns]:
    """A live step's admitted actions -> job columns, all on the device:
    (action columns, JobColumns); ``JobColumns.select`` finishes the
    admission with K6."""
    c = live_action_columns(table)
    mean, cost = tool_tables(table.dpool.sigs.tools, estimates)
    n = c["n"]
    jobs = action_jobs_arrays(c["tool"][:n], c["level"][:n], c["p"][:n], c["key"][:16 * n],
                              mean, cost, estimates.warm_fraction, r_total, id_base)
    return c, jobs


def select_jobs_desc(cols: JobColumns, selected, n_sel) -> SelectDesc:
    return SelectDesc(cols.n, ptr(cols.p), ptr(cols.benefit), ptr(cols.duration), ptr(cols.cost),
                      ptr(cols.id), ptr(selected), ptr(n_sel))

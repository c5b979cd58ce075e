"""CPU restatement of Scheduler._admit_action for a batch (TEST INFRASTRUCTURE
ONLY: imported by tests/ as the checker, never by the product package).

Follows /root/reference/pkg/src/spectool/scheduling.py:464-511 literally for
a batch of admitted actions entering a fresh scheduler (empty cache, no
running jobs): per action, in order, the key is (tool, "warm") for WARM_ONLY
and (tool, arg_hash) otherwise (:468-480); an action whose key a job of the
batch already holds is coalesced (:490-493); otherwise a job takes the next
id (:495) with duration / benefit from the estimates (:471-481) and is
dropped if its cost exceeds r_total (:501-502).  Job.utility is :59-60.
"""

from __future__ import annotations


def admit_jobs(actions, mean_of, cost_of, warm_fraction: float, r_total: int, id_base: int = 1):
    """actions: iterable of (tool, level, p, arg_hash) with level 1/2/3
    (WARM_ONLY / DRY_RUN / FULL).  Returns (per-action job tuple
    (id, p, benefit, cost, duration, arg_hash) or None, next id)."""
    next_id = id_base
    held = set()
    out = []
    for tool, level, p, arg_hash in actions:
        mean = mean_of(tool)
        if level == 1:
            key = (tool, "warm")
            duration = max(warm_fraction * mean, 1e-9)
            benefit = warm_fraction * mean
        else:
            key = (tool, arg_hash)
            duration = max(mean, 1e-9)
            benefit = mean if level == 3 else warm_fraction * mean
        if key in held:
            out.append(None)
            continue
        jid = next_id
        next_id += 1
        cost = cost_of(tool)
        if cost > r_total:
            out.append(None)
            continue
        held.add(key)
        out.append((jid, p, benefit, cost, duration, key[1]))
    return out, next_id


def utility(p: float, benefit: float, cost: int, duration: float) -> float:
    return (p * benefit) / (cost * duration)

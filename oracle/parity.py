"""Parity drivers (TEST INFRASTRUCTURE ONLY): run the device path and the C
oracle side by side on the same seeded inputs and report mismatches.

Used by tests/ and by bench.py's parity leg (the benchmarked sizes: 1M live
sessions, the 100M-event mining corpus).  The oracle here is the checker,
never the thing measured; the product package never imports this module.
"""

from __future__ import annotations

import os

import numpy as np

from . import bridge


def compare_records(dev, ora) -> list[str]:
    """Field names where two PredictResults (session-major) differ; fp64
    utilities are compared by bit pattern."""
    bad = []
    if not np.array_equal(dev.n_pred, ora.n_pred):
        return ["n_pred"]
    if not np.array_equal(dev.struct_err, ora.struct_err):
        bad.append("struct_err")
    K, B = dev.K, dev.B
    slot_valid = (np.arange(K)[None, :] < dev.n_pred[:, None]).reshape(-1)
    if not np.array_equal(dev.pred_pat[slot_valid], ora.pred_pat[slot_valid]):
        bad.append("pred_pat")
    if not np.array_equal(dev.pred_comp[slot_valid], ora.pred_comp[slot_valid]):
        bad.append("pred_comp")
    arg_valid = np.repeat(slot_valid & (dev.pred_comp != 2), B)
    if not np.array_equal(dev.pred_arg[arg_valid], ora.pred_arg[arg_valid]):
        bad.append("pred_arg")
    if not np.array_equal(dev.n_act, ora.n_act):
        bad.append("n_act")
        return bad
    act_valid = (np.arange(K)[None, :] < dev.n_act[:, None]).reshape(-1)
    if not np.array_equal(dev.act_pred[act_valid], ora.act_pred[act_valid]):
        bad.append("act_pred")
    if not np.array_equal(dev.act_level[act_valid], ora.act_level[act_valid]):
        bad.append("act_level")
    if not np.array_equal(dev.act_util[act_valid].view(np.int64),
                          ora.act_util[act_valid].view(np.int64)):
        bad.append("act_util")
    return bad


def live_parity(dp, policy, book, n: int, steps: int, K: int = 8, seed: int = 7,
                threads: int | None = None, workload_cls=None, serve: bool = True,
                alternate_wide: bool = True) -> dict:
    """Run ``steps`` live steps over n sessions three ways on one seeded
    workload -- the K-slot kernel (LiveSessionTable.step + fetch), the
    pipelined serving loop (fused predict + narrow-stream kernel,
    LiveSessionTable.serve, records expanded) and the oracle
    (oracle_predict_batch over mirrored host rings) -- and compare every
    record of every step.  Returns {"sessions", "steps", "predictions",
    "kslot_ok", "serve_ok", "mismatch"}."""
    import torch

    from paper_2603_18897_b200.live import LiveSessionTable
    from paper_2603_18897_b200.packing import WindowBatch, admit_tables
    from paper_2603_18897_b200.synth import LiveWorkload

    threads = threads or os.cpu_count() or 1
    make = workload_cls or (lambda: LiveWorkload(dp.sigs, dp.keys, n, seed=seed))
    wl_a, wl_b = make(), make()
    seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, book,
                           max_candidates=K)
    W, R = seq.W, seq.regions
    host = WindowBatch(W, np.full(n * W, -1, np.int32), np.full(n * W, -1, np.int32),
                       np.zeros(n, np.int64), None, [], slot_major=1)
    host.arena = (wl_a.tmpl.nodes, np.zeros(1, np.uint8), np.zeros((R * n, 2), np.int64))
    tables = admit_tables(dp.sigs, policy, book.duration)
    expected: dict[int, object] = {}
    mismatch: list[str] = []
    total = 0

    def kslot_and_oracle():
        nonlocal total
        for step in range(steps):
            b = wl_a.next_batch()
            if alternate_wide and step % 2:
                b.node = None  # the wide (16-B directory entry) observe input
            seq.step(b)
            dev = seq.fetch().session_major()
            ora = bridge.predict(dp.image, host, K, tables, new_tok=b.tok,
                                 new_ref=np.ascontiguousarray(b.ref),
                                 new_evt_base=(step % R) * n,
                                 new_byte_base=(step % R) * seq.max_batch_bytes, threads=threads)
            bad = compare_records(dev, ora)
            if bad:
                mismatch.append(f"kslot step {step}: {','.join(bad)}")
            total += int(dev.n_pred.sum())
            expected[step] = ora
            del dev
            yield wl_b.next_batch()

    if serve:
        pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, book,
                               max_candidates=K)
        for i, r in enumerate(pip.serve(kslot_and_oracle())):
            got = r.expand(dp.image.patterns, pip.benefit)
            bad = compare_records(got, expected.pop(i))
            if bad:
                mismatch.append(f"serve step {i}: {','.join(bad)}")
        fused = pip.serve_fused
        del pip
    else:
        for _ in kslot_and_oracle():
            expected.clear()
        fused = None
    state = seq.host_state()
    if not (np.array_equal(state["tok"], host.tok) and np.array_equal(state["count"], host.count)):
        mismatch.append("window rings differ after the run")
    del seq
    torch.cuda.empty_cache()
    return {"sessions": n, "steps": steps, "predictions": total,
            "kslot_ok": not any(m.startswith("kslot") or m.startswith("window") for m in mismatch),
            "serve_ok": serve and not any(m.startswith("serve") for m in mismatch),
            "serve_kernel": "fused predict + narrow streams" if fused else "K-slot + compaction",
            "mismatch": mismatch[:8]}


def mining_parity(tables, host_columns: dict, n_sigs: int, k: int, relation: int,
                  threads: int | None = None) -> dict:
    """Device count tables (after expand) against oracle_mine_counts on the
    host token stream (gap split restated on the host), bit for bit."""
    from paper_2603_18897_b200.synth import columnar_flags

    threads = threads or os.cpu_count() or 1
    tok = host_columns["sig"].astype(np.int32, copy=True)
    tok[columnar_flags(host_columns)] |= np.int32(-2**31)
    ora = bridge.mine_counts(tok, n_sigs, k, relation, threads=threads)
    names = ("tool_count", "support", "match", "follow")
    bad = [nm for nm, dev, ref in zip(names, (tables.tool_count, tables.support, tables.match,
                                              tables.follow), ora)
           if not np.array_equal(dev.cpu().numpy().astype(np.uint64), ref)]
    return {"events": int(len(tok)), "relation": "suffix" if relation else "anchored",
            "ok": not bad, "mismatch": bad, "oracle_tables": ora}

"""The UNMODIFIED reference (``spectool``), timed on this host and used as a
parity check of the live path (CPU BASELINE / TEST INFRASTRUCTURE ONLY:
imported by bench.py's baseline legs, never by the product package).

``baseline/_ref`` holds the reference installed as-is:

    cp -r /root/reference/pkg /tmp/refsrc
    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref /tmp/refsrc

(``--no-deps``: its one dependency, pyyaml, is in the image but not in the
wheelhouse).  The directory is git-ignored and travels to the GPU box, so
nothing here reads /root/reference.  BASELINE.md section 3 plans exactly this:
the reference's own predict + admit (prediction.py:76-118, policy.py:207-236)
on the C3 workload, one core and all cores (session-sharded processes, each
generating its own shard), and its outputs compared with ours.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
W = 16  # suffix window (C3)


def available() -> str | None:
    """None when spectool imports from baseline/_ref, else why not."""
    if not os.path.isdir(os.path.join(REF_DIR, "spectool")):
        return "baseline/_ref/spectool not installed"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import spectool  # noqa: F401
    except Exception as e:  # pragma: no cover - reported, not raised
        return f"import spectool failed: {e!r}"
    if not os.path.dirname(sys.modules["spectool"].__file__).startswith(REF_DIR):
        return "spectool resolved outside baseline/_ref"
    return None


def _setup(pool_file: str, policy_text: str, durations: dict):
    from spectool.mining import load_pool
    from spectool.policy import parse_policy
    from spectool.prediction import Predictor
    from spectool.scheduling import EstimateBook

    pool = load_pool(pool_file)
    book = EstimateBook()
    for tool, ms in durations.items():
        book.update(tool, ms)
    return Predictor(pool), parse_policy(policy_text).policy, book


def c3_sample(m: int, n_steps: int, seed: int, pool_file: str):
    """n_steps batches of the C3 workload (synth.LiveWorkload over the same
    pool tables) for m sessions, and the same batches as reference Events:
    (batches, events[step][session])."""
    from spectool.events import Event, EventKind, Status

    from paper_2603_18897_b200.device_ops import DevicePool
    from paper_2603_18897_b200.mining import load_pool
    from paper_2603_18897_b200.synth import LiveWorkload
    from paper_2603_18897_b200.tape import decode_node

    dp = DevicePool(load_pool(pool_file))
    wl = LiveWorkload(dp.sigs, dp.keys, m, seed=seed)
    batches, events = [], []
    for step in range(n_steps):
        b = wl.next_batch()
        batches.append(b)
        row = []
        for s in range(m):
            sig = int(b.tok[s])
            row.append(Event(session_id=f"s{s}", seq=step, kind=EventKind.TOOL_CALL,
                             tool_type=dp.sigs.tools[sig >> 1],
                             status=Status.SUCCESS if sig & 1 else Status.FAIL, args={},
                             result=decode_node(wl.tmpl.nodes, b.data, int(b.ref[s, 0]),
                                                int(b.ref[s, 1]), 0, dp.keys),
                             t_start=float(step), t_end=float(step)))
        events.append(row)
    return dp, wl, batches, events


def run_c3(events, pool_file, policy_text, durations, max_candidates=8, record=False):
    """Feed every step's events through the reference: observe, then (for the
    steps after the first W) predict(max_candidates) + admit(benefit =
    EstimateBook.duration).  Returns (session-steps timed, seconds, outputs
    of the timed steps when ``record``)."""
    from spectool.policy import admit
    from spectool.prediction import PredictionWindow

    predictor, policy, book = _setup(pool_file, policy_text, durations)

    def benefit(pr):
        return book.duration(pr.tool_type)

    m = len(events[0])
    windows = [PredictionWindow(W) for _ in range(m)]
    for row in events[:W]:  # fill the windows (untimed)
        for w, ev in zip(windows, row):
            w.observe(ev)
    outs = []
    done, spent = 0, 0.0
    for row in events[W:]:
        step_out = [] if record else None
        t0 = time.perf_counter()
        for w, ev in zip(windows, row):
            w.observe(ev)
            preds = predictor.predict(w, max_candidates=max_candidates)
            acts = admit(preds, policy, benefit)
            if record:
                step_out.append((preds, acts))
        spent += time.perf_counter() - t0
        done += m
        if record:
            outs.append(step_out)
    return done, spent, outs


def _worker(a):
    """One core's shard: its own sessions (seed + worker id), timed alone."""
    err = available()
    if err:
        raise RuntimeError(err)
    m, n_steps, seed, pool_file, policy_text, durations = a
    _, _, _, events = c3_sample(m, n_steps, seed, pool_file)
    done, spent, _ = run_c3(events, pool_file, policy_text, durations)
    return done, spent


def c3_all_cores(procs, m, n_steps, pool_file, policy_text, durations, seed=2603):
    """Session-sharded processes (spawned: the parent holds a CUDA context),
    each generating and timing its own shard; aggregate = all session-steps
    / the slowest worker's time (they run concurrently)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as p:
        res = p.map(_worker, [(m, n_steps, seed + 1000 * i, pool_file, policy_text, durations)
                              for i in range(procs)])
    done = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    return done / slowest, done, slowest


def _pred_key(p):
    return (p.tool_type, json.dumps(p.args, sort_keys=True), p.completeness.value,
            p.probability, p.source_pattern)


def _act_key(a):
    return (a.prediction.source_pattern, int(a.level), a.expected_utility)


def c3_parity(dp, wl, batches, ref_outs, policy, book, max_candidates=8):
    """Run our live path (LiveSessionTable, the C3 device step) over the same
    batches and compare every timed step's decoded predictions and admitted
    actions with the reference's, session by session."""
    from paper_2603_18897_b200.live import LiveSessionTable
    from paper_2603_18897_b200.packing import decode_actions, decode_predictions
    from paper_2603_18897_b200.tape import ArrayTapes

    m = len(batches[0].tok)
    table = LiveSessionTable(dp, m, wl.tmpl.nodes, wl.max_batch_bytes, policy, book,
                             max_candidates=max_candidates, ship_bytes=True)
    bad, n_pred, n_act, first = 0, 0, 0, None
    for step, b in enumerate(batches):
        table.step(b)
        if step < W:
            continue
        res = table.fetch().session_major()
        hs = table.host_state()
        arena = ArrayTapes(wl.tmpl.nodes, hs["bytes"], hs["refs"], dp.keys)
        preds = decode_predictions(res, dp.image, arena, [0.0] * m, 0.0)
        acts = decode_actions(res, preds)
        for s, (rp, ra) in enumerate(ref_outs[step - W]):
            n_pred += len(rp)
            n_act += len(ra)
            if ([_pred_key(p) for p in preds[s]] != [_pred_key(p) for p in rp]
                    or [_act_key(a) for a in acts[s]] != [_act_key(a) for a in ra]):
                bad += 1
                if first is None:
                    first = {"step": step, "session": s,
                             "ours": [_pred_key(p) for p in preds[s]],
                             "reference": [_pred_key(p) for p in rp]}
    return {"sessions": m, "steps": len(batches) - W, "predictions": n_pred, "actions": n_act,
            "mismatched_session_steps": bad, "first_mismatch": first, "ok": bad == 0}


def mine_text(text: str, tau: float, k: int = 3, sigma: int = 5, relation: str | None = None):
    """The reference end to end on JSONL text: ingest_trace (events.py:196)
    + mine (mining.py:248) with MiningConfig(k, sigma, tau, relation).
    Returns (patterns as pool JSON, sessions, events, seconds)."""
    from spectool.events import ingest_trace
    from spectool.mining import MatchRelation, MiningConfig, _pattern_to_json, mine

    cfg = MiningConfig(k=k, sigma=sigma, tau=tau)
    if relation is not None:
        cfg = MiningConfig(k=k, sigma=sigma, tau=tau, match_relation=MatchRelation(relation))
    t0 = time.perf_counter()
    sessions = ingest_trace(text).sessions
    pats = mine(sessions, cfg)
    dt = time.perf_counter() - t0
    return ([_pattern_to_json(p) for p in pats], len(sessions),
            sum(len(s.events) for s in sessions), dt)


def ours_as_json(patterns):
    from paper_2603_18897_b200.mining import _pattern_to_json

    return [_pattern_to_json(p) for p in patterns]


def score_text(text: str, pool_file: str, window: int, max_candidates):
    """The reference's score_accuracy (prediction.py:133-169) over the
    sessions of JSONL text, with a reference-format pool file.  Returns
    (report dict, scored calls, seconds of score_accuracy alone)."""
    from spectool.events import ingest_trace
    from spectool.mining import load_pool
    from spectool.prediction import score_accuracy

    sessions = ingest_trace(text).sessions
    pool = load_pool(pool_file)
    t0 = time.perf_counter()
    rep = score_accuracy(sessions, pool, window, max_candidates)
    dt = time.perf_counter() - t0
    return rep.to_json(), rep.scored_calls, dt


def candidate_paths_sample(c: dict, m: int):
    """The reference's candidate_paths (mappings.py:237-266, default node
    budget) over the first m C5 payloads (synth.long_output_corpus),
    decoded to Python objects; the target is the next call's argument
    string.  Returns (paths per session, truncated flags, seconds of the
    candidate_paths calls alone)."""
    from spectool.mappings import candidate_paths

    from paper_2603_18897_b200.tape import decode_node

    payloads, targets = [], []
    for s in range(m):
        payloads.append(decode_node(c["nodes"], c["bytes"], int(c["refs"][s, 0]),
                                    int(c["refs"][s, 1]), 0, c["keys"]))
        t0, t1 = int(c["target_off"][s]), int(c["target_off"][s + 1])
        targets.append(bytes(c["target_bytes"][t0:t1]).decode("utf-8"))
    t0 = time.perf_counter()
    res = [candidate_paths(p, t) for p, t in zip(payloads, targets)]
    dt = time.perf_counter() - t0
    return [r.paths for r in res], [r.truncated for r in res], dt


def columnar_to_jsonl(c: dict, tools) -> str:
    """A columnar corpus (synth.columnar_corpus) as the reference's JSONL
    records (events.py:162-184: session_id, seq, kind, tool, status,
    t_start_ms, t_end_ms), one line per event in file order."""
    sess, seq, sig = c["session"].tolist(), c["seq"].tolist(), c["sig"].tolist()
    ts, te = c["t_start"].tolist(), c["t_end"].tolist()
    return "".join(
        '{"session_id": "c%d", "seq": %d, "kind": "tool_call", "tool": "%s", "status": "%s", '
        '"t_start_ms": %r, "t_end_ms": %r}\n'
        % (a, q, tools[g >> 1], "success" if g & 1 else "fail", x, y)
        for a, q, g, x, y in zip(sess, seq, sig, ts, te))

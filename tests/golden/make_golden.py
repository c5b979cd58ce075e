"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is not available on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden.py

Every fixture records inputs (sessions / pools / windows / jobs / payloads)
and the reference's outputs for them, so the oracle and the CUDA path can be
pinned to the reference without importing it at test time.
"""

from __future__ import annotations

import io
import json
import os
import random
import sys

import spectool
from spectool.events import Event, EventKind, EventSignature, Session, Status, event_to_record
from spectool.mappings import (ArgBinding, FormatTemplate, IndexedFallback, Normalization,
                               PathLookup, ValueMapping, candidate_paths)
from spectool.mining import (MatchRelation, MiningConfig, PatternPool, PatternTuple, load_pool,
                             mine, mine_pool, pool_to_json, save_pool)
from spectool.policy import SpecLevel, SpeculationPolicy, ToolRule, admit, parse_policy
from spectool.prediction import (Completeness, PredictedInvocation, PredictionWindow, Predictor,
                                 score_accuracy)
from spectool.scheduling import EstimateBook, Job, JobKind, greedy_speculative_selection
from spectool.simulation import ToolModel, LatencySpec, tool_result
from spectool.workloads import generate_corpus

assert "/root/reference" in os.path.dirname(spectool.__file__), spectool.__file__

OUT = os.path.dirname(os.path.abspath(__file__))
S, F = Status.SUCCESS, Status.FAIL

MOTIF_POLICY = """\
speculation_policy:
  default:
    allow: false
  tools:
    web_fetch: {allow: true, max_speculation: full}
    terminal: {allow: true, max_speculation: dry_run}
    search: {allow: true, max_speculation: full}
    file_editor: {allow: true, max_speculation: dry_run}
"""
EXAMPLE_POLICY = """\
speculation_policy:
  default: {allow: false}
  tools:
    web_search: {allow: true, max_speculation: full}
    pip_install: {allow: true, max_speculation: dry_run}
"""


def sig(tool, status=S):
    return EventSignature(tool, status)


def ev(tool, status=S, result=None, args=None, seq=0, kind=EventKind.TOOL_CALL, session="s"):
    return Event(session, seq, kind, tool if kind is EventKind.TOOL_CALL else "", status, args,
                 result, float(seq), float(seq) + 1.5)


def llm(seq=0):
    return ev("", kind=EventKind.LLM_STEP, seq=seq)


def rec(e: Event) -> dict:
    return event_to_record(e)


def pred_json(p: PredictedInvocation) -> dict:
    return {"tool": p.tool_type, "args": p.args, "completeness": p.completeness.value,
            "p": p.probability, "pattern": p.source_pattern, "created_at": p.created_at}


def policy_json(policy: SpeculationPolicy | None):
    if policy is None:
        return None
    return {"default_allow": policy.default_allow, "default_level": int(policy.default_level),
            "tools": {t: [r.allow, int(r.max_speculation)] for t, r in policy.tool_rules.items()}}


def estimates_json(book: EstimateBook) -> dict:
    return {"default": book.default_duration_ms, "tools": dict(book._duration)}


# ---------------------------------------------------------------------------
# prediction + admit
# ---------------------------------------------------------------------------

SEARCH_RESULT = {"list": [{"url": "a.com"}, {"url": "b.com"}]}


def fetch_pool(k=3, relation=MatchRelation.ANCHORED_SUBSEQUENCE):
    first = PatternTuple((sig("search"),), "web_fetch",
                         ValueMapping((ArgBinding("url", PathLookup(0, ("list", 0, "url"))),)), 0.9, 10)
    retry = PatternTuple((sig("search"), sig("web_fetch", F)), "web_fetch",
                         ValueMapping((ArgBinding("url", PathLookup(0, ("list", 1, "url"))),)), 0.8, 8)
    return PatternPool(MiningConfig(k=k, tau=0.5, match_relation=relation), (first, retry))


def edge_pool():
    """Hand-built pool covering every expression class and edge."""
    pats = [
        # PathLookup to scalar / container / missing key
        PatternTuple((sig("search"),), "web_fetch",
                     ValueMapping((ArgBinding("url", PathLookup(0, ("list", 0, "url"))),)), 0.9, 10),
        PatternTuple((sig("search"),), "summarize",
                     ValueMapping((ArgBinding("doc", PathLookup(0, ("list", 1))),
                                   ArgBinding("n", PathLookup(0, ("total",))))), 0.9, 10),
        PatternTuple((sig("search"),), "archive",
                     ValueMapping((ArgBinding("x", PathLookup(0, ("nope",))),)), 0.7, 4),
        # FormatTemplate with each normalization; bool / None / container holes
        PatternTuple((sig("file_editor"),), "terminal",
                     ValueMapping((ArgBinding("cmd", FormatTemplate("pytest ", PathLookup(0, ("path",)), " -q")),)), 0.6, 6),
        PatternTuple((sig("file_editor"),), "shell",
                     ValueMapping((ArgBinding("cmd", FormatTemplate("echo ", PathLookup(0, ("title",)), "", Normalization.TRIM)),
                                   ArgBinding("low", FormatTemplate("", PathLookup(0, ("title",)), "!", Normalization.LOWERCASE)))), 0.6, 6),
        PatternTuple((sig("file_editor"),), "flag",
                     ValueMapping((ArgBinding("v", FormatTemplate("v=", PathLookup(0, ("applied",)), "")),
                                   ArgBinding("w", FormatTemplate("w=", PathLookup(0, ("size",)), "")),
                                   ArgBinding("z", FormatTemplate("z=", PathLookup(0, ("ratio",)), "")))), 0.55, 6),
        PatternTuple((sig("file_editor"),), "nullish",
                     ValueMapping((ArgBinding("v", FormatTemplate("", PathLookup(0, ("none",)), "")),
                                   ArgBinding("c", FormatTemplate("", PathLookup(0, ("meta",)), "")))), 0.55, 6),
        # IndexedFallback with prefix/suffix and failures of the target tool
        PatternTuple((sig("search"), sig("web_fetch", F)), "web_fetch",
                     ValueMapping((ArgBinding("url", IndexedFallback(0, ("list",), 0, ("url",), "web_fetch")),)), 0.8, 8),
        PatternTuple((sig("search"), sig("grep", F)), "web_fetch",
                     ValueMapping((ArgBinding("url", IndexedFallback(0, ("list",), 1, ("url",), "web_fetch")),)), 0.8, 8),
        # struct error (ctx_pos out of range)
        PatternTuple((sig("search"),), "broken",
                     ValueMapping((ArgBinding("x", PathLookup(5, ("y",))),)), 0.95, 5),
        # tool-only and ties on p (pattern_id decides)
        PatternTuple((sig("search"),), "tie_a", None, 0.7, 5),
        PatternTuple((sig("search"),), "tie_b", None, 0.7, 5),
        PatternTuple((sig("grep"), sig("search")), "tie_c", None, 0.7, 5),
        PatternTuple((sig("grep", F), sig("grep"), sig("search")), "deep", None, 0.65, 5),
        PatternTuple((sig("grep"), sig("grep"), sig("grep"), sig("search")), "too_long", None, 0.99, 5),
        # duplicate content, different p (same pattern_id)
        PatternTuple((sig("search"),), "dup", None, 0.5, 5),
        PatternTuple((sig("search"),), "dup", None, 0.6, 5),
        # empty mapping -> FULL with no args
        PatternTuple((sig("grep"),), "emptymap", ValueMapping(()), 0.4, 5),
        # source at a failed position (evaluate still reads it)
        PatternTuple((sig("web_fetch", F),), "web_fetch",
                     ValueMapping((ArgBinding("token", PathLookup(0, ("token",))),)), 0.45, 5),
    ]
    return pats


def edge_windows():
    edit = {"path": "src/ÅmÅ.py", "applied": True, "title": "  Hello World ", "size": 2.0,
            "ratio": 0.25, "none": None, "meta": {"k": [1, 2]}}
    edit_nfc = {"path": "src/ÅmÅ.py", "applied": False, "title": "ÉCOLE",
                "size": 10 ** 30, "ratio": float("1e300"), "none": None, "meta": []}
    sr = {"list": [{"url": "a.com", "rank": 0}, {"url": "b.com", "rank": 1},
                   {"url": "c.com", "rank": 2}], "total": 3}
    wins = [
        [],
        [ev("search", result=sr)],
        [ev("search", result={"list": []})],
        [ev("search", result=sr), ev("web_fetch", F, result={"ok": False, "token": "t0"})],
        [ev("search", result=sr), ev("web_fetch", F, result={"ok": False, "token": "t0"}),
         ev("web_fetch", F, result={"ok": False, "token": "t1"})],
        [ev("search", result=sr), ev("web_fetch", F, result={"token": "x"}), ev("grep", F, result={}),
         ev("web_fetch", F, result={"token": "y"})],
        [ev("search", result=sr), ev("grep", F, result=None)],
        [ev("grep", F, result={}), ev("grep", result={}), ev("search", result=sr)],
        [ev("grep", result={}), ev("grep", F, result={}), ev("grep", result={}), ev("search", result=sr)],
        [ev("grep", F, result={}), llm(1), ev("grep", result={}), llm(2), ev("search", result=sr)],
        [ev("file_editor", result=edit)],
        [ev("file_editor", result=edit_nfc)],
        [ev("file_editor", result={"path": 7, "title": "", "applied": True})],
        [ev("file_editor", result="scalar-result")],
        [ev("unknown_tool", result={}), ev("search", result=sr)],
        [ev("search", result=sr), ev("unknown_tool", result={})],
        [ev("grep", result={"x": 1})],
        [llm(0)],
        [ev("web_fetch", F, result={"token": 3.5})],
        [ev("search", result=sr)] + [ev("noise", result={}) for _ in range(3)] + [ev("search", result=sr)],
    ]
    return wins


def roundtrip(pool):
    """Fixtures carry pools as pool JSON; predict on the pool as the reference
    itself loads it back (mapping_from_json sorts bindings by arg name)."""
    buf = io.StringIO()
    save_pool(pool, buf)
    buf.seek(0)
    return load_pool(buf)


def predict_case(name, pool, windows, max_candidates, policy=None, book=None, tool_only=False):
    pool = roundtrip(pool)
    predictor = Predictor(pool)
    out_preds, out_acts = [], []
    for w in windows:
        win = PredictionWindow(16)
        for e in w:
            win.observe(e)
        preds = predictor.predict(win, max_candidates=max_candidates)
        out_preds.append([pred_json(p) for p in preds])
        if policy is not None:
            acts = admit(preds, policy, benefit_of=lambda p: book.duration(p.tool_type))
            out_acts.append([{"pred": next(i for i, q in enumerate(preds) if q is a.prediction),
                              "level": int(a.level), "utility": a.expected_utility} for a in acts])
    return {"name": name, "pool": pool_to_json(pool), "max_candidates": max_candidates,
            "policy": policy_json(policy), "estimates": estimates_json(book) if book else None,
            "windows": [[rec(e) for e in w] for w in windows],
            "expected": out_preds, "expected_actions": out_acts if policy is not None else None,
            "structural_errors": predictor.diagnostics.structural_errors}


def stress_pool(seed=1001, n=1000, n_tools=20):
    rng = random.Random(seed)
    tools = [f"tool{i}" for i in range(n_tools)]
    pats, seen = [], set()
    while len(pats) < n:
        ctx = tuple(sig(rng.choice(tools), rng.choice([S, F])) for _ in range(rng.randint(1, 3)))
        target = rng.choice(tools)
        if (ctx, target) in seen:
            continue
        seen.add((ctx, target))
        pats.append(PatternTuple(ctx, target, None, round(rng.uniform(0.3, 1.0), 4), 5))
    return PatternPool(MiningConfig(), tuple(pats)), tools


def motif_corpus(n, seed):
    return generate_corpus({"search_visit": 0.25, "edit_verify": 0.25, "locate_examine": 0.25,
                            "batch_fetch": 0.25}, n, seed=seed,
                           params={"search_visit": {"rounds": 4}, "edit_verify": {"rounds": 4},
                                   "locate_examine": {"rounds": 4},
                                   "batch_fetch": {"fetch_count": 6}})


def make_predict():
    cases = []
    cases.append(predict_case("fetch_pool", fetch_pool(), edge_windows(), None))
    base = edge_pool()
    for k in (1, 2, 3, 4):
        pool = PatternPool(MiningConfig(k=k, tau=0.3), tuple(base))
        for K in (None, 1, 3, 8):
            book = EstimateBook()
            book.update("web_fetch", 900.0)
            book.update("terminal", 1500.0)
            cases.append(predict_case(f"edge_k{k}_K{K}", pool, edge_windows(), K,
                                      SpeculationPolicy(default_allow=True,
                                                        tool_rules={"terminal": ToolRule(True, SpecLevel.DRY_RUN),
                                                                    "tie_b": ToolRule(False)}),
                                      book))
    pool = PatternPool(MiningConfig(k=3, tau=0.3, match_relation=MatchRelation.CONTIGUOUS_SUFFIX), tuple(base))
    cases.append(predict_case("edge_suffix", pool, edge_windows(), None,
                              SpeculationPolicy(default_allow=True), EstimateBook()))
    cases.append(predict_case("fetch_suffix", fetch_pool(relation=MatchRelation.CONTIGUOUS_SUFFIX),
                              edge_windows(), 8))

    # stress pool, random windows
    pool, tools = stress_pool()
    rng = random.Random(77)
    wins = []
    for i in range(300):
        n = rng.randint(0, 16)
        w = []
        for j in range(n):
            if rng.random() < 0.1:
                w.append(llm(j))
            else:
                w.append(ev(rng.choice(tools), rng.choice([S, S, F]), result={"i": j}, seq=j))
        wins.append(w)
    book = EstimateBook()
    for t in tools[::3]:
        book.update(t, 100.0 + 7 * len(t))
    pol = SpeculationPolicy(default_allow=True, tool_rules={t: ToolRule(i % 3 != 0, SpecLevel(1 + i % 3))
                                                            for i, t in enumerate(tools[::2])})
    for K in (None, 3, 8):
        cases.append(predict_case(f"stress_K{K}", pool, wins, K, pol if K == 8 else None,
                                  book if K == 8 else None))

    # mined motif pool on held-out motif sessions (simulator semantics: tool-only windows)
    train = motif_corpus(300, 11)
    for tau in (0.3, 0.5):
        mpool = mine_pool(train.sessions, MiningConfig(k=3, sigma=5, tau=tau))
        held = motif_corpus(40, 12)
        wins = []
        for s in held.sessions:
            tool_events = s.tool_events()
            for e in range(1, len(tool_events) + 1):
                wins.append(list(tool_events[max(0, e - 16):e]))
        book = EstimateBook()
        book.update("search", 700.0)
        book.update("web_fetch", 1100.0)
        cases.append(predict_case(f"motif_tau{tau}", mpool, wins, 8,
                                  parse_policy(MOTIF_POLICY).policy, book))
    return {"cases": cases}


def make_admit():
    rng = random.Random(5)
    tools = ["a", "b", "c", "d"]
    lists = []
    for i in range(200):
        preds = []
        for j in range(rng.randint(0, 12)):
            preds.append(PredictedInvocation(
                tool_type=rng.choice(tools), args={"i": j},
                completeness=rng.choice(list(Completeness)),
                probability=rng.choice([0.5, 0.9, rng.uniform(0.05, 1.0)]),
                source_pattern=f"p{j}", created_at=rng.choice([1.0, 2.0, 3.0])))
        lists.append(preds)
    pol = SpeculationPolicy(default_allow=True, tool_rules={"a": ToolRule(True, SpecLevel.DRY_RUN),
                                                            "b": ToolRule(True, SpecLevel.WARM_ONLY),
                                                            "d": ToolRule(False)})
    bene = {t: 10.0 * (i + 1) for i, t in enumerate(tools)}
    out = []
    for preds in lists:
        acts = admit(preds, pol, benefit_of=lambda p: bene[p.tool_type] * (1 + p.created_at % 2))
        out.append({"preds": [pred_json(p) for p in preds],
                    "actions": [{"pred": next(i for i, q in enumerate(preds) if q is a.prediction),
                                 "level": int(a.level), "utility": a.expected_utility} for a in acts]})
    return {"policy": policy_json(pol), "benefit": bene, "lists": out}


# ---------------------------------------------------------------------------
# mining
# ---------------------------------------------------------------------------

def _session(sid, calls):
    events, t = [], 0.0
    for seq, (tool, status, args, result) in enumerate(calls):
        events.append(Event(sid, seq, EventKind.TOOL_CALL, tool, status, args, result, t, t + 10))
        t += 20
    return Session(sid, tuple(events))


def sess_json(s: Session) -> dict:
    return {"id": s.session_id, "events": [rec(e) for e in s.events]}


def pattern_json(p: PatternTuple) -> dict:
    from spectool.mining import _pattern_to_json
    d = _pattern_to_json(p)
    d["pattern_id"] = p.pattern_id
    return d


def make_mine():
    rng = random.Random(20_250_101)
    corpora = []
    for ci in range(40):
        tools = ["alpha", "beta", "gamma", "delta"][:rng.randint(2, 4)]
        sessions = []
        for i in range(rng.randint(15, 60)):
            calls = [(rng.choice(tools), S if rng.random() < 0.8 else F,
                      {"token": f"{rng.getrandbits(48):012x}"},
                      {"echo": f"{rng.getrandbits(48):012x}"}) for _ in range(rng.randint(1, 9))]
            sessions.append(_session(f"c{ci}-s{i}", calls))
        cfg = MiningConfig(k=rng.choice([1, 2, 3, 4]), sigma=rng.choice([1, 2, 3]),
                           tau=rng.choice([0.3, 0.5, 1.0]),
                           match_relation=rng.choice(list(MatchRelation)))
        mined = mine(sessions, cfg)
        corpora.append({"config": {"k": cfg.k, "sigma": cfg.sigma, "tau": cfg.tau,
                                   "match_relation": cfg.match_relation.value},
                        "sessions": [sess_json(s) for s in sessions],
                        "expected": [pattern_json(p) for p in mined]})
    # motif corpora with mappings (PathLookup / FormatTemplate / IndexedFallback)
    mapped = []
    for seed, mix, params, cfg in [
        (7, {"search_visit": 0.5, "batch_fetch": 0.5}, None, MiningConfig()),
        (7, {"search_visit": 0.5, "batch_fetch": 0.5}, None, MiningConfig(tau=0.3)),
        (1, {"edit_verify": 0.5, "locate_examine": 0.5}, None, MiningConfig(tau=0.3)),
        (3, {"search_visit": 1.0}, {"search_visit": {"rounds": 3}}, MiningConfig(k=2, tau=0.3)),
    ]:
        corpus = generate_corpus(mix, 150, seed=seed, params=params)
        mined = mine(corpus.sessions, cfg)
        mapped.append({"config": {"k": cfg.k, "sigma": cfg.sigma, "tau": cfg.tau,
                                  "match_relation": cfg.match_relation.value},
                       "sessions": [sess_json(s) for s in corpus.sessions],
                       "expected": [pattern_json(p) for p in mined]})
    return {"corpora": corpora, "mapped": mapped}


# ---------------------------------------------------------------------------
# greedy selection
# ---------------------------------------------------------------------------

def make_greedy():
    rng = random.Random(404)
    cases = []
    for inst in range(300):
        n = rng.randint(0, 40 if inst % 3 else 12)
        jobs = [Job(id=i + 1, kind=JobKind.SPECULATIVE, tool_type=f"t{i}", args={}, arg_hash="",
                    session_id="s", p=rng.choice([0.5, round(rng.uniform(0.05, 1.0), 2)]),
                    benefit_ms=rng.choice([1000.0, 200.0, rng.uniform(100, 10_000)]),
                    cost=rng.randint(1, 4),
                    duration_est_ms=rng.choice([1000.0, rng.uniform(100, 5000)]),
                    submitted_at=0.0) for i in range(n)]
        rng.shuffle(jobs)
        slack, budget = rng.randint(0, 10), rng.randint(0, 10)
        chosen = greedy_speculative_selection(jobs, slack, budget)
        cases.append({"jobs": [[j.id, j.p, j.benefit_ms, j.cost, j.duration_est_ms] for j in jobs],
                      "slack": slack, "budget": budget, "expected": [j.id for j in chosen]})
    return {"cases": cases}


def make_jobs():
    """Scheduler._admit_action (scheduling.py:464-511) on batches of admitted
    actions from many sessions, into a fresh scheduler: the job terms
    (benefit / duration by level, the 1e-9 clamp, warm_fraction, per-tool
    cost), key coalescing (warm key (tool, "warm"), others (tool, arg hash)),
    ids, the cost > r_total drop; then greedy_speculative_selection over the
    admitted jobs (Job.utility, scheduling.py:59-60, 242-258)."""
    from spectool.policy import SpeculativeAction
    from spectool.scheduling import ResourceState, Scheduler

    rng = random.Random(1616)
    tools = ["search", "web_fetch", "terminal", "file_editor", "grep", "big"]
    cases = []
    for inst in range(120):
        n_sess = rng.randint(0, 30 if inst % 4 else 6)
        wf = rng.choice([0.2, 0.2, 0.35, 0.0, 1e-12])
        book = EstimateBook(warm_fraction=wf, costs={"terminal": 2, "grep": 3, "big": 9},
                            default_duration_ms=rng.choice([1000.0, 1000.0, 0.0, 5e-10]))
        for t in tools:
            r = rng.random()
            if r < 0.5:
                book.update(t, rng.choice([700.0, 1100.0, rng.uniform(1, 5000), 3e-9, 0.0]))
            if r < 0.2:
                book.update(t, rng.uniform(1, 5000))
        r_total = rng.choice([4, 8, 24])
        sched = Scheduler(ResourceState(r_total, 1 << 30), launcher=lambda j: None,
                          estimates=book)
        actions, jobs = [], []
        for s in range(n_sess):
            for a in range(rng.randint(0, 8)):
                tool = rng.choice(tools)
                args = {"u": rng.randint(0, 6)} if rng.random() < 0.8 else {"q": "x", "n": [1, 2]}
                level = rng.choice([SpecLevel.FULL, SpecLevel.DRY_RUN, SpecLevel.WARM_ONLY])
                p = rng.choice([0.5, 0.9, rng.uniform(0.01, 1.0)])
                pred = PredictedInvocation(tool, args, Completeness.FULL, p, f"pat{a}", 0.0)
                act = SpeculativeAction(pred, level, p * 1.0)
                job = sched._admit_action(act, f"s{s}", 0.0)
                actions.append({"session": s, "tool": tool, "args": args, "level": int(level),
                                "p": p})
                jobs.append(None if job is None else
                            [job.id, job.p, job.benefit_ms, job.cost, job.duration_est_ms,
                             job.arg_hash, job.utility() if job.cost * job.duration_est_ms
                             else None])
        admitted = [sched.jobs[j[0]] for j in jobs if j is not None]
        sel = []
        for slack, budget in ((rng.randint(0, 12), rng.randint(0, 12)), (200, 150)):
            try:
                chosen = [j.id for j in greedy_speculative_selection(admitted, slack, budget)]
            except ZeroDivisionError:
                chosen = "ZeroDivisionError"
            sel.append({"slack": slack, "budget": budget, "expected": chosen})
        cases.append({"tools": tools, "estimates": {
            "default": book.default_duration_ms, "warm_fraction": wf, "costs": book.costs,
            "durations": dict(book._duration)}, "r_total": r_total, "next_id": next(sched._ids),
            "actions": actions, "jobs": jobs, "select": sel})
    return {"cases": cases}


# ---------------------------------------------------------------------------
# candidate_paths
# ---------------------------------------------------------------------------

def make_paths():
    url_list = tool_result(ToolModel("search", LatencySpec("fixed", ms=1.0), result_kind="url_list",
                                     result_size=1120), {"query": "q-long"}, 0)[1]
    payloads = [
        ({"a": {"b": 1}, "c": 1, "d": [1, 1.0, True, "1"]}, 1),
        ({"a": {"b": 1}, "c": 1}, 1.0),
        ({"x": [True, 1, "true"]}, True),
        ({"s": "Å", "t": "Å", "u": ["Å"]}, "Å"),
        ({"n": None, "m": [None]}, None),
        ({"f": 0.1, "g": [0.1, 0.30000000000000004]}, 0.1),
        ({"big": 10 ** 20, "bf": 1e20}, 10 ** 20),
        ({"nan": float("nan")}, float("nan")),
        ("root-scalar", "root-scalar"),
        ([["deep", ["deeper", {"k": "deep"}]]], "deep"),
        ({"list": [{"url": f"u{i}"} for i in range(30)]}, "u17"),
        (url_list, url_list["list"][37 * 5 % 1120]["url"]),
        ({"k": list(range(12000))}, 11999),
        ({"k": list(range(12000))}, 5),
        ({"d": {f"k{i}": i for i in range(50)}}, 49),
        ({}, 1),
    ]
    cases = []
    for payload, target in payloads:
        for budget in (10_000, 5, 1, 0):
            res = candidate_paths(payload, target, budget)
            cases.append({"payload": payload, "target": target, "budget": budget,
                          "paths": [list(p) for p in res.paths], "truncated": res.truncated})
    return {"cases": cases}


# ---------------------------------------------------------------------------
# score_accuracy
# ---------------------------------------------------------------------------

def make_score():
    out = []
    train = motif_corpus(200, 21)
    pool = mine_pool(train.sessions, MiningConfig(k=3, sigma=5, tau=0.3))
    held = motif_corpus(60, 22)
    for W, K in ((16, None), (4, 3), (16, 8)):
        rep = score_accuracy(held.sessions, pool, window_capacity=W, max_candidates=K)
        out.append({"pool": pool_to_json(pool), "window": W, "max_candidates": K,
                    "sessions": [sess_json(s) for s in held.sessions], "expected": rep.to_json()})
    return {"cases": out}


# ---------------------------------------------------------------------------
# canonical_arg_hash (events.py:94-122)
# ---------------------------------------------------------------------------

def make_hash():
    """Values and the reference's canonical_arg_hash of each ("error" when the
    reference raises): key order, NFC (keys and values, incl. colliding
    keys), JSON escapes, integral / special floats, bool vs int, deep and
    wide containers, multi-block serialisations, lone surrogates."""
    from spectool.events import canonical_arg_hash

    rng = random.Random(7)
    alphabet = ["a", "b", "Z", "0", " ", '"', "\\", "\n", "\t", "\x00", "\x1f", "\x7f", "é",
                "e\u0301", "\u00c5", "A\u030a", "\u4e2d", "\U0001F600", "/", "<", "\u2028"]

    def rstr(n):
        return "".join(rng.choice(alphabet) for _ in range(n))

    def rscalar():
        r = rng.random()
        if r < 0.3:
            return rstr(rng.randint(0, 12))
        if r < 0.45:
            return rng.randint(-10 ** 6, 10 ** 6)
        if r < 0.6:
            return rng.choice([0.5, -1.25, 1e16, 1e-7, 3.0, -0.0, 2.5e300, 1.0 / 3.0,
                               float("nan"), float("inf"), float("-inf"), 123456789.0])
        if r < 0.7:
            return rng.choice([True, False, None])
        return rng.choice([2 ** 70, -(2 ** 64), 0, 1])

    def rvalue(depth=0):
        r = rng.random()
        if depth > 3 or r < 0.45:
            return rscalar()
        if r < 0.7:
            return [rvalue(depth + 1) for _ in range(rng.randint(0, 4))]
        return {rstr(rng.randint(1, 6)): rvalue(depth + 1) for _ in range(rng.randint(0, 5))}

    values = [
        {}, [], "", 0, None, True, 1.0, -0.0, {"b": 1, "a": 2}, {"a": [1, 2.0, True, None]},
        {"url": "https://example.org/a?b=c&d=\"e\""}, {"path": "C:\\tmp\\x", "n": 3},
        {"e\u0301": 1, "\u00e9": 2}, {"\u00e9": 1, "e\u0301": 2},  # keys colliding under NFC
        {"k": "\ud800"}, "a\udfffb",  # lone surrogates: the reference raises
        {"x" * 60: "y" * 60}, "z" * 121, "z" * 122, "z" * 254, "z" * 500,
        {"d%03d" % i: i for i in range(300)},  # wide dict
        [[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[[["deep"]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]]],
        {"cmd": "pytest -q tests/test_x.py::test_y", "timeout": 30.0, "env": {"CI": "1"}},
    ]
    values += [rvalue() for _ in range(400)]
    cases = []
    for v in values:
        try:
            h = canonical_arg_hash(v)
        except (UnicodeEncodeError, ValueError):
            h = "error"
        cases.append({"value": v, "hash": h})
    path = os.path.join(OUT, "hash_golden.json")
    with open(path, "w", encoding="utf-8") as fh:  # ASCII escapes keep lone surrogates
        json.dump({"cases": cases}, fh, ensure_ascii=True, separators=(",", ":"))
    print(f"hash_golden.json: {len(cases)} values", file=sys.stderr)


# ---------------------------------------------------------------------------
# ingestion (events.py:196-252) and the pool wire format (mining.py:300-398)
# ---------------------------------------------------------------------------

def _ingest_json(text, threshold=None):
    from spectool.events import ingest_trace
    res = ingest_trace(text) if threshold is None else ingest_trace(text, threshold)
    return {"text": text, "threshold": threshold,
            "expected": {"sessions": [sess_json(s) for s in res.sessions],
                         "errors": [[e.line, e.message] for e in res.errors],
                         "reordered": res.reordered_sessions}}


def _line(sid, seq, kind="tool_call", tool="a", status="success", t0=0.0, t1=None, **extra):
    d = {"session_id": sid, "seq": seq, "kind": kind, "tool": tool, "status": status,
         "t_start_ms": t0, "t_end_ms": t0 + 1.0 if t1 is None else t1}
    d.update(extra)
    return json.dumps(d, ensure_ascii=False)


def make_ingest():
    """The reference's ingest_trace on hand-made edge traces and on random
    interleaved traces: first-appearance grouping, the stable (t_start, seq)
    sort and the reorder tally, gap splits at exactly / just past / just
    under the threshold (incl. gaps measured from an LLM step), #n segment
    ids, per-line errors (bad JSON, non-objects, missing fields, bad enums,
    t_start > t_end, empty tool), coerced field types and custom thresholds."""
    T = 300_000.0
    hand = []
    # exact-threshold gaps: > splits, == does not; +-0.5
    hand.append("\n".join([_line("g", 0, t0=0.0, t1=10.0), _line("g", 1, t0=10.0 + T),
                           _line("g", 2, t0=11.0 + T + T + 0.5), _line("g", 3, t0=2 * T + 12.0 + T - 0.5 + 0.5),
                           _line("g", 4, t0=4 * T + 100.0, tool="b"),
                           _line("g", 5, kind="llm_step", tool="", t0=5 * T + 200.0),
                           _line("g", 6, t0=5 * T + 201.0 + T)]))
    # interleaving + reorders + ties on t_start broken by seq, duplicate (t, seq) kept stable
    hand.append("\n".join([_line("x", 3, t0=5.0, tool="c"), _line("y", 0, t0=1.0),
                           _line("x", 1, t0=5.0, tool="b"), _line("x", 0, t0=9.0),
                           _line("y", 1, t0=1.0, tool="d"), _line("y", 1, t0=1.0, tool="e"),
                           _line("z", 0, t0=0.0, kind="llm_step", tool=""),
                           _line("x", 2, t0=2.0, status="fail")]))
    # malformed lines of every kind the reference tallies
    hand.append("\n".join([
        _line("m", 0), "{broken", "[1, 2]", "42", '"str"', "null",
        json.dumps({"session_id": "m", "seq": 1, "kind": "tool_call", "tool": "a"}),
        _line("m", 2, kind="bogus"), _line("m", 3, status="ok"),
        _line("m", 4, t0=10.0, t1=5.0), _line("m", 5, tool=""),
        _line("m", 6, kind="llm_step", tool=""), "   ", "",
        _line("m", 7, t0=3.0, t1=3.0, tool="f"),
        '{"session_id": "m", "seq": "x", "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": 1, "t_end_ms": 2}',
        '{"session_id": "m", "seq": 8, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": "abc", "t_end_ms": 2}',
        _line("m", 9, t0=20.0)]))
    # coercions: numeric / escaped / unicode ids, seq as float or numeric string,
    # times as strings or ints, -0.0, tools that are numbers, extra keys and payloads
    hand.append("\n".join([
        '{"session_id": 7, "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": 1, "t_end_ms": 2}',
        '{"session_id": "7", "seq": 1.9, "kind": "tool_call", "tool": 5, "status": "fail", '
        '"t_start_ms": "3", "t_end_ms": "4.5"}',
        '{"session_id": "s\\"q", "seq": "2", "kind": "tool_call", "tool": "\\u00e9t\\u00e9", '
        '"status": "success", "t_start_ms": -0.0, "t_end_ms": 0.0, "args": {"q": [1, {"k": null}]}}',
        '{"session_id": "s\\"q", "seq": 3, "kind": "tool_call", "tool": "b", "status": "success", '
        '"t_start_ms": 0.0, "t_end_ms": 0.0, "result": "r", "extra": true}',
        _line("ü#1", 0, t0=1e15, t1=1e15 + 1), _line("ü", 0, t0=-5.0, t1=-4.0),
        _line("ü", 1, t0=-1e-300, t1=1e-300, tool="z"),
        '{"session_id": "n", "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": 1e308, "t_end_ms": Infinity}',
        '{"session_id": "n", "seq": 1, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": true, "t_end_ms": 2}']))
    cases = [_ingest_json(t) for t in hand]
    cases.append(_ingest_json(hand[0], 1000.0))
    cases.append(_ingest_json(hand[1], 0.0))
    cases.append(_ingest_json(hand[0], 299_999.5))
    # random interleaved traces
    rng = random.Random(5196)
    tools = ["search", "web_fetch", "file_editor", "terminal", "grep", "Zeta", "été"]
    for ci in range(24):
        lines = []
        n_sess = rng.randint(1, 40)
        for s in range(n_sess):
            t = rng.choice([0.0, rng.uniform(0, 1e6)])
            sid = rng.choice([f"s{s}", f"sess-{s}", f"s{s}#1", f"é{s}"])
            for q in range(rng.randint(1, 12)):
                kind = "llm_step" if rng.random() < 0.2 else "tool_call"
                t += rng.choice([0.0, 10.0, 500.0, T - 0.5, T, T + 0.5, 400_000.0, 1e6])
                dur = rng.choice([0.0, 1.0, rng.uniform(1, 2000)])
                extra = {}
                if rng.random() < 0.3:
                    extra["args"] = {"q": rng.randint(0, 9)}
                if rng.random() < 0.3:
                    extra["result"] = {"r": [1, 2.5, None, True]}
                lines.append(_line(sid, q, kind=kind,
                                   tool="" if kind == "llm_step" else rng.choice(tools),
                                   status="fail" if rng.random() < 0.1 else "success",
                                   t0=t, t1=t + dur, **extra))
            if rng.random() < 0.3 and len(lines) > 2:  # swap timestamps -> reorder
                i = rng.randrange(len(lines) - 1)
                a, b = json.loads(lines[i]), json.loads(lines[i + 1])
                if a["session_id"] == b["session_id"]:
                    for key in ("t_start_ms", "t_end_ms"):
                        a[key], b[key] = b[key], a[key]
                    lines[i], lines[i + 1] = json.dumps(a), json.dumps(b)
        if ci % 2:
            rng.shuffle(lines)
        for _ in range(rng.randint(0, 4)):
            lines.insert(rng.randrange(len(lines) + 1), rng.choice(["{", "[]", "   ", _line(
                "bad", 0, t0=5.0, t1=1.0), _line("bad", 1, tool="")]))
        cases.append(_ingest_json("\n".join(lines) + rng.choice(["", "\n"]),
                                  rng.choice([None, None, 1000.0, 5e5])))
    return {"cases": cases}


def make_pool_bytes():
    """save_pool text written by the reference: the random 1000-pattern pool of
    pkg/tests/test_mining.py:253-276 (its generator, seed 21), pools with every
    mapping kind and normalisation, and pools the reference mined from the
    mapped motif corpora -- the load -> save byte-identity gate and the
    serialisation of device-mined pools."""
    from spectool.mining import MatchRelation
    rng = random.Random(21)
    tools = ["a", "b", "c"]
    patterns = []
    for _ in range(1000):
        ctx = tuple(sig(rng.choice(tools), rng.choice([S, F])) for _ in range(rng.randint(1, 3)))
        mapping = None
        if rng.random() < 0.5:
            mapping = ValueMapping((ArgBinding("arg0", PathLookup(
                rng.randrange(len(ctx)), ("list", rng.randint(0, 3), "url"))),))
        patterns.append(PatternTuple(context=ctx, target=rng.choice(tools), mapping=mapping,
                                     p=round(rng.uniform(0.1, 1.0), 6), support=rng.randint(1, 50)))
    pools = {"random_1000": PatternPool(config=MiningConfig(), patterns=tuple(patterns))}
    pools["edge"] = PatternPool(config=MiningConfig(k=2, sigma=3, tau=0.25,
                                                    match_relation=MatchRelation.CONTIGUOUS_SUFFIX),
                                patterns=tuple(edge_pool()))
    for name, (seed, mix, cfg) in {
            "mined_search_batch_t03": (7, {"search_visit": 0.5, "batch_fetch": 0.5},
                                       MiningConfig(tau=0.3)),
            "mined_coding_t03": (1, {"edit_verify": 0.5, "locate_examine": 0.5},
                                 MiningConfig(tau=0.3))}.items():
        corpus = generate_corpus(mix, 150, seed=seed)
        pools[name] = mine_pool(corpus.sessions, cfg)
    out = {}
    for name, pool in pools.items():
        buf = io.StringIO()
        save_pool(pool, buf)
        again = io.StringIO()  # the reference's own load -> save of that text
        save_pool(load_pool(io.StringIO(buf.getvalue())), again)
        out[name] = {"saved": buf.getvalue(), "resaved": again.getvalue()}
    return {"pools": out}


def make_c1():
    """C1 at its stated size: generate_corpus(search_visit /
    batch_fetch 0.5 / 0.5, 1000 sessions, seed 7) mined at the default
    MiningConfig (tau 0.5) and at tau 0.3, and score_accuracy(W=16) of each
    pool on the held-out seed-8 corpus (1000 sessions)."""
    import gzip
    mix = {"search_visit": 0.5, "batch_fetch": 0.5}
    train = generate_corpus(mix, 1000, seed=7)
    held = generate_corpus(mix, 1000, seed=8)
    out = {"train": [sess_json(s) for s in train.sessions],
           "held": [sess_json(s) for s in held.sessions], "cases": []}
    for cfg in (MiningConfig(), MiningConfig(tau=0.3)):
        pool = mine_pool(train.sessions, cfg)
        rep = score_accuracy(held.sessions, pool, window_capacity=16)
        out["cases"].append({"config": {"k": cfg.k, "sigma": cfg.sigma, "tau": cfg.tau,
                                        "match_relation": cfg.match_relation.value},
                             "expected": [pattern_json(p) for p in pool.patterns],
                             "score": rep.to_json()})
        print(f"C1 tau={cfg.tau}: {len(pool)} patterns, {rep.to_json()}", file=sys.stderr)
    path = os.path.join(OUT, "c1_golden.json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(out, fh, ensure_ascii=False, separators=(",", ":"))
    print(f"c1_golden.json.gz: {os.path.getsize(path) / 1e6:.2f} MB", file=sys.stderr)


def dump(name, obj):
    path = os.path.join(OUT, name)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(obj, fh, ensure_ascii=False, separators=(",", ":"))
    print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB", file=sys.stderr)


def main(which):
    if "c3pool" in which:
        make_c3_pool()
    if "c2" in which:
        make_c2()
    if "hash" in which:
        make_hash()
    if "jobs" in which:
        dump("jobs_golden.json", make_jobs())
    if "c1" in which:
        make_c1()
    if "ingest" in which:
        dump("ingest_golden.json", make_ingest())
    if "poolbytes" in which:
        dump("pool_bytes_golden.json", make_pool_bytes())
    if "fixtures" not in which:
        return
    dump("predict_golden.json", make_predict())
    dump("admit_golden.json", make_admit())
    dump("mine_golden.json", make_mine())
    dump("greedy_golden.json", make_greedy())
    dump("paths_golden.json", make_paths())
    dump("score_golden.json", make_score())


def make_c3_pool():
    """The C3 pool: mined by the reference from a 1k-session training mix of the
    four motifs (rounds=16, fetch_count=15), tau = 0.3."""
    corpus = generate_corpus({"search_visit": 0.25, "edit_verify": 0.25, "locate_examine": 0.25,
                              "batch_fetch": 0.25}, 1000, seed=2603,
                             params={"search_visit": {"rounds": 16}, "edit_verify": {"rounds": 16},
                                     "locate_examine": {"rounds": 16},
                                     "batch_fetch": {"fetch_count": 15}})
    pool = mine_pool(corpus.sessions, MiningConfig(k=3, sigma=5, tau=0.3))
    path = os.path.join(os.path.dirname(os.path.dirname(OUT)), "paper_2603_18897_b200", "data",
                        "pool_motif_c3.json")
    save_pool(pool, path)
    print(f"pool_motif_c3.json: {len(pool)} patterns", file=sys.stderr)


CODING_MIX = {"edit_verify": 0.5, "locate_examine": 0.5}


def make_c2():
    """C2: pools mined by the reference from
    generate_corpus(edit_verify/locate_examine, 1000, seed=1) with the default
    MiningConfig (tau 0.5) and with tau 0.3 (FormatTemplate bindings), plus
    the reference's score_accuracy on a 400-session replay corpus (seed=2)."""
    data = os.path.join(os.path.dirname(os.path.dirname(OUT)), "paper_2603_18897_b200", "data")
    train = generate_corpus(CODING_MIX, 1000, seed=1)
    pools = {"pool_coding_c2.json": mine_pool(train.sessions, MiningConfig()),
             "pool_coding_c2_t03.json": mine_pool(train.sessions, MiningConfig(tau=0.3))}
    for name, pool in pools.items():
        save_pool(pool, os.path.join(data, name))
        print(f"{name}: {len(pool)} patterns", file=sys.stderr)
    held = generate_corpus(CODING_MIX, 400, seed=2)
    cases = []
    for name, pool in pools.items():
        pool = roundtrip(pool)
        for W, K in ((16, 8), (16, None), (2, 1)):
            rep = score_accuracy(held.sessions, pool, window_capacity=W, max_candidates=K)
            cases.append({"pool_file": name, "window": W, "max_candidates": K,
                          "expected": rep.to_json()})
    dump("score_c2_golden.json", {"sessions": [sess_json(s) for s in held.sessions],
                                  "cases": cases})


if __name__ == "__main__":
    main(sys.argv[1:] or ["fixtures", "c3pool"])

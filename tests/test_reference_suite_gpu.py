"""The reference's own hot-path tests, restated against this package's public
API (the drop-in surface, every call running on the device):

  * pkg/tests/test_prediction.py:45-247   PredictionWindow, Predictor.predict,
                                          score_accuracy, the < 1 ms per-call
                                          budget on the 1,000-pattern pool
  * pkg/tests/test_policy.py:103-170      admit (caps, PARTIAL -> WARM_ONLY,
                                          arbitration, tie-breaks, deny-all)
  * pkg/tests/test_scheduling.py:224-270  greedy_speculative_selection
  * pkg/tests/test_mining.py:53-216       mine() on hand-made corpora

Expected values are the ones those tests assert; where they compare with a
brute force, the brute force is restated here from the reference's
pkg/tests/oracles.py."""

import itertools
import random
import time

import pytest

from paper_2603_18897_b200 import (ArgBinding, Completeness, Event, EventKind, EventSignature,
                                   Job, JobKind, MiningConfig, PathLookup, PatternPool,
                                   PatternTuple, PredictedInvocation, PredictionWindow, Predictor,
                                   Session, SpecLevel, SpeculationPolicy, Status, ValueMapping,
                                   admit, greedy_speculative_selection, mine, parse_policy,
                                   score_accuracy)
from paper_2603_18897_b200.mining import MatchRelation
from paper_2603_18897_b200.policy import ToolRule

pytestmark = pytest.mark.gpu
S, F = Status.SUCCESS, Status.FAIL
SEARCH_RESULT = {"list": [{"url": "a.com"}, {"url": "b.com"}]}
EXAMPLE_POLICY = """\
speculation_policy:
  default: {allow: false}
  tools:
    web_search: {allow: true, max_speculation: full}
    pip_install: {allow: true, max_speculation: dry_run}
"""


def sig(tool, status=S):
    return EventSignature(tool, status)


def ev(tool, status=S, result=None, args=None, seq=0, session="s"):
    return Event(session, seq, EventKind.TOOL_CALL, tool, status, args, result, float(seq),
                 float(seq) + 1)


def fetch_pool(tau=0.5, relation=MatchRelation.ANCHORED_SUBSEQUENCE):
    first = PatternTuple((sig("search"),), "web_fetch",
                         ValueMapping((ArgBinding("url", PathLookup(0, ("list", 0, "url"))),)),
                         0.9, 10)
    retry = PatternTuple((sig("search"), sig("web_fetch", F)), "web_fetch",
                         ValueMapping((ArgBinding("url", PathLookup(0, ("list", 1, "url"))),)),
                         0.8, 8)
    return PatternPool(MiningConfig(tau=tau, match_relation=relation), (first, retry))


def window(*events, capacity=8):
    w = PredictionWindow(capacity)
    for e in events:
        w.observe(e)
    return w


# --------------------------------------------------------------------------
# prediction (test_prediction.py:45-171)
# --------------------------------------------------------------------------

def test_window_capacity_evicts_oldest():
    w = window(*(ev("t", seq=i) for i in range(4)), capacity=3)
    assert [e.seq for e in w.events()] == [1, 2, 3]


def test_new_event_visible_to_predict():
    w = PredictionWindow(8)
    pr = Predictor(fetch_pool())
    assert pr.predict(w) == []
    w.observe(ev("search", result=SEARCH_RESULT))
    preds = pr.predict(w)
    assert len(preds) == 1 and preds[0].tool_type == "web_fetch"


def test_first_result_pattern_fires():
    preds = Predictor(fetch_pool()).predict(window(ev("search", result=SEARCH_RESULT)))
    assert len(preds) == 1
    p = preds[0]
    assert (p.tool_type, p.args, p.probability, p.completeness) == (
        "web_fetch", {"url": "a.com"}, 0.9, Completeness.FULL)


def test_fallback_pattern_fires_after_failure():
    w = window(ev("search", result=SEARCH_RESULT, seq=0),
               ev("web_fetch", F, args={"url": "a.com"}, seq=1))
    preds = Predictor(fetch_pool()).predict(w)
    assert [p.probability for p in preds] == [0.8]
    assert preds[0].args == {"url": "b.com"}


def test_empty_pool_predicts_nothing():
    pr = Predictor(PatternPool(MiningConfig(), ()))
    assert pr.predict(window(ev("search", result=SEARCH_RESULT))) == []


def test_predict_does_not_mutate_window():
    w = window(ev("search", result=SEARCH_RESULT))
    before = w.events()
    Predictor(fetch_pool()).predict(w)
    assert w.events() == before


def test_adding_pattern_is_monotone():
    w = window(ev("search", result=SEARCH_RESULT))
    base = fetch_pool()
    bigger = PatternPool(base.config, base.patterns + (
        PatternTuple((sig("search"),), "summarize", None, 0.6, 7),))
    before = {p.source_pattern for p in Predictor(base).predict(w)}
    after = {p.source_pattern for p in Predictor(bigger).predict(w)}
    assert before <= after and len(after) == 2


def test_partial_when_path_absent():
    preds = Predictor(fetch_pool()).predict(window(ev("search", result={"list": []})))
    assert preds[0].completeness is Completeness.PARTIAL and preds[0].args == {}


def test_max_candidates_truncates():
    pats = tuple(PatternTuple((sig("search"),), f"tool{i}", None, 0.5 + i / 100, 5)
                 for i in range(10))
    preds = Predictor(PatternPool(MiningConfig(), pats)).predict(
        window(ev("search", result={})), max_candidates=3)
    assert len(preds) == 3
    assert preds[0].probability >= preds[1].probability >= preds[2].probability
    assert [p.tool_type for p in preds] == ["tool9", "tool8", "tool7"]


def test_corrupted_pattern_skipped_and_tallied():
    bad = PatternTuple((sig("search"),), "summarize",
                       ValueMapping((ArgBinding("x", PathLookup(5, ("y",))),)), 0.95, 5)
    pr = Predictor(PatternPool(MiningConfig(), fetch_pool().patterns + (bad,)))
    preds = pr.predict(window(ev("search", result=SEARCH_RESULT)))
    assert [p.tool_type for p in preds] == ["web_fetch"]
    assert pr.diagnostics.structural_errors == 1


def test_contiguous_suffix_relation_requires_adjacency():
    pool = PatternPool(MiningConfig(tau=0.5, match_relation=MatchRelation.CONTIGUOUS_SUFFIX),
                       (PatternTuple((sig("a"), sig("b")), "c", None, 0.7, 5),))
    pr = Predictor(pool)
    assert pr.predict(window(*(ev(t, seq=i) for i, t in enumerate("axb")))) == []
    assert [p.tool_type for p in pr.predict(window(ev("a", seq=0), ev("b", seq=1)))] == ["c"]


def stress_pool(seed=123, n=1000, n_tools=20):
    """test_prediction.py:173-199 / test_acceptance.py:511-527: 1,000 distinct
    (context, target) patterns over 20 tools."""
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


def test_latency_budget_on_large_pool():
    """Per-call Predictor.predict on the 1,000-pattern pool: the reference's
    acceptance budget is < 1 ms per call."""
    pool, tools = stress_pool()
    pr = Predictor(pool)
    w = window(*(ev(tools[i % len(tools)], seq=i, result={"x": i}) for i in range(16)),
               capacity=16)
    for _ in range(50):
        pr.predict(w)
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        pr.predict(w)
    per_call_ms = (time.perf_counter() - t0) * 1000 / n
    print(f"Predictor.predict per call: {per_call_ms:.3f} ms")
    assert per_call_ms < 1.0


# --------------------------------------------------------------------------
# score_accuracy (test_prediction.py:202-247)
# --------------------------------------------------------------------------

def perfect_corpus(n=30):
    out = []
    for i in range(n):
        result = {"list": [{"url": f"https://d{i}.example"}]}
        out.append(Session(f"s{i}", (
            ev("search", result=result, args={"q": str(i)}, seq=0, session=f"s{i}"),
            ev("web_fetch", args={"url": result["list"][0]["url"]}, result={"ok": 1}, seq=1,
               session=f"s{i}"))))
    return out


def perfect_pool():
    return PatternPool(MiningConfig(), (PatternTuple(
        (sig("search"),), "web_fetch",
        ValueMapping((ArgBinding("url", PathLookup(0, ("list", 0, "url"))),)), 1.0, 30),))


def test_deterministic_corpus_scores_one():
    rep = score_accuracy(perfect_corpus(), perfect_pool())
    assert (rep.top1, rep.top3, rep.hit_rate) == (1.0, 1.0, 1.0)


def test_empty_pool_scores_zero():
    rep = score_accuracy(perfect_corpus(), PatternPool(MiningConfig(), ()))
    assert (rep.top1, rep.top3, rep.hit_rate) == (0.0, 0.0, 0.0) and rep.scored_calls > 0


# --------------------------------------------------------------------------
# admit (test_policy.py:103-170)
# --------------------------------------------------------------------------

def pred(tool="web_search", completeness=Completeness.FULL, p=0.9, args=None, created_at=0.0):
    return PredictedInvocation(tool, args or {"q": "x"}, completeness, p, "pat", created_at)


def test_allowed_full_prediction():
    acts = admit([pred(p=0.9)], parse_policy(EXAMPLE_POLICY).policy, lambda pr: 10.0)
    assert len(acts) == 1 and acts[0].level is SpecLevel.FULL
    assert acts[0].expected_utility == pytest.approx(9.0)


def test_policy_cap_applies_to_full_prediction():
    acts = admit([pred(tool="pip_install", p=0.8)], parse_policy(EXAMPLE_POLICY).policy,
                 lambda pr: 10.0)
    assert acts[0].level is SpecLevel.DRY_RUN


def test_partial_prediction_warms_only():
    acts = admit([pred(completeness=Completeness.PARTIAL)], parse_policy(EXAMPLE_POLICY).policy,
                 lambda pr: 10.0)
    assert acts[0].level is SpecLevel.WARM_ONLY


def test_disallowed_tool_dropped():
    assert admit([pred(tool="rm_rf")], parse_policy(EXAMPLE_POLICY).policy, lambda pr: 10.0) == []


def test_utility_arbitration_keeps_higher_product():
    a = pred(tool="web_fetch", p=0.9, args={"u": "a"})
    b = pred(tool="web_fetch", p=0.8, args={"u": "b"})
    benefits = {id(a): 10.0, id(b): 20.0}
    acts = admit([a, b], SpeculationPolicy(default_allow=True), lambda pr: benefits[id(pr)])
    assert len(acts) == 1 and acts[0].prediction is b
    assert acts[0].expected_utility == pytest.approx(16.0)


def test_tie_break_prefers_probability_then_earlier():
    early = pred(tool="t", p=0.9, args={"u": 1}, created_at=1.0)
    late = pred(tool="t", p=0.9, args={"u": 2}, created_at=2.0)
    acts = admit([late, early], SpeculationPolicy(default_allow=True), lambda pr: 5.0)
    assert acts[0].prediction is early


def test_at_most_one_action_per_tool_and_caps_respected():
    policy = SpeculationPolicy(default_allow=True,
                               tool_rules={"a": ToolRule(True, SpecLevel.DRY_RUN),
                                           "b": ToolRule(True, SpecLevel.WARM_ONLY)})
    rng = random.Random(11)
    for _ in range(60):
        preds = [pred(tool=rng.choice("abc"), p=rng.uniform(0.05, 1.0),
                      completeness=rng.choice(list(Completeness)), args={"i": i})
                 for i in range(rng.randint(0, 12))]
        acts = admit(preds, policy, lambda pr: 7.0)
        tools = [a.tool_type for a in acts]
        assert len(tools) == len(set(tools))
        for a in acts:
            assert a.level <= policy.rule_for(a.tool_type).max_speculation
            if a.prediction.completeness is not Completeness.FULL:
                assert a.level is SpecLevel.WARM_ONLY


def test_deny_all_admits_nothing():
    deny = SpeculationPolicy(default_allow=False)
    assert admit([pred(tool=f"t{i}") for i in range(5)], deny, lambda pr: 1.0) == []


# --------------------------------------------------------------------------
# greedy selection (test_scheduling.py:224-270)
# --------------------------------------------------------------------------

def job(i, p, benefit, cost, duration):
    return Job(id=i, kind=JobKind.SPECULATIVE, tool_type=f"t{i}", args={}, arg_hash=f"h{i}",
               session_id="s", p=p, benefit_ms=benefit, cost=cost, duration_est_ms=duration,
               submitted_at=0.0, level=SpecLevel.FULL, preemptible=True)


def test_greedy_documented_example():
    a, b = job(1, 0.9, 10_000, 1, 2_000), job(2, 0.5, 30_000, 2, 3_000)
    assert a.utility() == pytest.approx(4.5) and b.utility() == pytest.approx(2.5)
    assert [j.id for j in greedy_speculative_selection([a, b], slack=2, budget=2)] == [1]


def test_greedy_selection_is_descending_utility():
    rng = random.Random(5)
    jobs = [job(i, rng.uniform(0.1, 1), rng.uniform(100, 10_000), rng.randint(1, 3),
                rng.uniform(100, 5_000)) for i in range(10)]
    u = [j.utility() for j in greedy_speculative_selection(jobs, slack=6, budget=6)]
    assert u == sorted(u, reverse=True) and u


def test_greedy_never_exceeds_min_of_slack_and_budget():
    rng = random.Random(6)
    for _ in range(100):
        jobs = [job(i, rng.uniform(0.05, 1), rng.uniform(100, 10_000), rng.randint(1, 4),
                    rng.uniform(100, 5_000)) for i in range(rng.randint(0, 12))]
        slack, budget = rng.randint(0, 8), rng.randint(0, 8)
        chosen = greedy_speculative_selection(jobs, slack, budget)
        assert sum(j.cost for j in chosen) <= min(slack, budget)


def test_greedy_against_exhaustive_optimum():
    def best(jobs, cap):  # pkg/tests/oracles.py:120-133
        top = 0.0
        for mask in range(1 << len(jobs)):
            sel = [j for i, j in enumerate(jobs) if mask >> i & 1]
            if sum(j.cost for j in sel) <= cap:
                top = max(top, sum(j.p * j.benefit_ms for j in sel))
        return top

    rng = random.Random(7)
    ratios = []
    for _ in range(50):
        jobs = [job(i, rng.uniform(0.05, 1), rng.uniform(100, 10_000), rng.randint(1, 3),
                    rng.uniform(100, 5_000)) for i in range(10)]
        cap = min(rng.randint(1, 6), rng.randint(1, 6))
        got = sum(j.p * j.benefit_ms for j in greedy_speculative_selection(jobs, cap, cap))
        b = best(jobs, cap)
        assert got <= b + 1e-9
        if b > 0:
            ratios.append(got / b)
    assert sum(ratios) / len(ratios) > 0.5


# --------------------------------------------------------------------------
# mining (test_mining.py:53-216)
# --------------------------------------------------------------------------

def session(sid, calls):
    return Session(sid, tuple(Event(sid, i, EventKind.TOOL_CALL, t, st, None, None, 20.0 * i,
                                    20.0 * i + 10) for i, (t, st) in enumerate(calls)))


def brute_force_mine(sessions, cfg):
    """pkg/tests/oracles.py brute_force_mine restated: every (context,
    target) with support >= sigma whose p = follow / match >= tau (anchored
    subsequence within the k events before the target)."""
    streams = [[sig(e.tool_type, e.status) for e in s.tool_events()] for s in sessions]
    tool_count = {}
    for st in streams:
        for s_ in st:
            tool_count[s_.tool_type] = tool_count.get(s_.tool_type, 0) + 1
    support = {}
    for st in streams:
        for i, s_ in enumerate(st):
            window_ = st[max(0, i - cfg.k):i]
            seen = set()
            for r in range(1, len(window_) + 1):
                for idx in itertools.combinations(range(len(window_)), r):
                    seen.add(tuple(window_[j] for j in idx))
            for ctx in seen:
                support[(ctx, s_.tool_type)] = support.get((ctx, s_.tool_type), 0) + 1

    def matches(st, a, ctx):
        if st[a] != ctx[-1]:
            return False
        lo = max(0, a - cfg.k + 1)
        j = len(ctx) - 1
        for q in range(a, lo - 1, -1):
            if j >= 0 and st[q] == ctx[j]:
                j -= 1
        return j < 0

    out = {}
    for (ctx, tgt), sup in support.items():
        if sup < cfg.sigma or tool_count[tgt] < cfg.sigma:
            continue
        m = hit = 0
        for st in streams:
            for a in range(len(st)):
                if matches(st, a, ctx):
                    m += 1
                    hit += a + 1 < len(st) and st[a + 1].tool_type == tgt
        if m and hit / m >= cfg.tau:
            out[(ctx, tgt)] = (hit / m, sup)
    return out


def test_mine_planted_chain_probability():
    rng = random.Random(3)
    sessions = []
    for i in range(80):
        calls = []
        for _ in range(6):
            calls.append(("search", S))
            calls.append(("fetch", S) if rng.random() < 0.75 else ("reply", S))
        sessions.append(session(f"s{i}", calls))
    pats = mine(sessions, MiningConfig(k=1, sigma=5, tau=0.3))
    by = {(p.context, p.target): p for p in pats}
    exp = brute_force_mine(sessions, MiningConfig(k=1, sigma=5, tau=0.3))
    assert set(by) == set(exp)
    for key, (p, sup) in exp.items():
        assert by[key].p == p and by[key].support == sup


@pytest.mark.parametrize("seed", range(12))
def test_mine_equals_brute_force_on_random_corpora(seed):
    rng = random.Random(seed)
    tools = ["a", "b", "c"][:rng.randint(2, 3)]
    sessions = [session(f"s{i}", [(rng.choice(tools), S if rng.random() < 0.8 else F)
                                  for _ in range(rng.randint(1, 8))]) for i in range(30)]
    cfg = MiningConfig(k=rng.choice([1, 2, 3]), sigma=rng.choice([1, 2, 3]),
                       tau=rng.choice([0.2, 0.5]))
    got = {(p.context, p.target): (p.p, p.support) for p in mine(sessions, cfg)}
    assert got == brute_force_mine(sessions, cfg)


def test_mine_empty_traces_raise():
    with pytest.raises(ValueError):
        mine([], MiningConfig())

"""C2 replay (score_accuracy, prediction.py:133-169).

* CPU: the oracle replay (C oracle predictions + canonical_arg_hash) is pinned
  to the reference's own score_accuracy outputs (score_golden.json,
  score_c2_golden.json);
* GPU: the device replay (paste_replay_score: windows -> K4 -> on-device hit
  check) equals the oracle replay call for call on synthetic coding corpora,
  and the public score_accuracy equals the reference's goldens.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import golden_io as G
from oracle import bridge
from paper_2603_18897_b200.device_ops import DevicePool
from paper_2603_18897_b200.mining import load_pool
from paper_2603_18897_b200.replay import KeysetTable, corpus_from_traces

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_2603_18897_b200", "data")


def c2_pool(name):
    return load_pool(os.path.join(DATA, name))


def _golden_cases():
    g = G.golden("score_c2_golden.json")
    sessions = [G.session(s) for s in g["sessions"]]
    for case in g["cases"]:
        yield sessions, c2_pool(case["pool_file"]), case
    for case in G.golden("score_golden.json")["cases"]:
        yield [G.session(s) for s in case["sessions"]], G.pool(case["pool"]), case


def _report(top1, top3, hits, n):
    return {"top1": top1 / n, "top3": top3 / n, "hit_rate": hits / n, "scored_calls": n}


def test_oracle_replay_matches_reference():
    for sessions, pool, case in _golden_cases():
        dp = DevicePool(pool)
        corpus, _, arena = corpus_from_traces(sessions, dp, case["window"], KeysetTable())
        got = bridge.score_corpus(dp.image, corpus, dp.keys, case["window"],
                                  case["max_candidates"])
        assert _report(*got) == case["expected"], case.get("pool_file")


def test_coding_corpus_shape():
    from paper_2603_18897_b200.synth import coding_replay_corpus

    dp = DevicePool(c2_pool("pool_coding_c2_t03.json"))
    c = coding_replay_corpus(dp, 500, seed=3)
    assert (c.ev_tok[c.call_pos] >= 0).all()
    assert (c.call_len >= 1).all() and (c.call_len <= 16).all()
    # every scored call's window stays inside its session (>= 1 tool call)
    assert ((c.ev_tok[c.call_pos - c.call_len] == -1)).all()  # windows start at an LLM step
    top1, top3, hits, n = bridge.score_corpus(dp.image, c, dp.keys, 16, 8)
    assert n == c.n_calls and hits > 0 and top3 >= top1
    # stream-mode windows (read in place) == gathered rings
    assert bridge.score_corpus(dp.image, c, dp.keys, 16, 8, stream=False) == (top1, top3, hits, n)
    assert bridge.score_corpus(dp.image, c, dp.keys, 3, None, calls=slice(100, 900)) == \
        bridge.score_corpus(dp.image, c, dp.keys, 3, None, calls=slice(100, 900), stream=False)


@pytest.mark.gpu
def test_score_accuracy_c2_matches_reference():
    from paper_2603_18897_b200.prediction import score_accuracy

    for sessions, pool, case in _golden_cases():
        rep = score_accuracy(sessions, pool, window_capacity=case["window"],
                             max_candidates=case["max_candidates"])
        assert rep.to_json() == case["expected"]


@pytest.mark.gpu
@pytest.mark.parametrize("pool_file,W,K", [("pool_coding_c2_t03.json", 16, 8),
                                           ("pool_coding_c2_t03.json", 4, None),
                                           ("pool_coding_c2_t03.json", 16, -2),
                                           ("pool_coding_c2.json", 16, 8),
                                           ("pool_coding_c2.json", 2, 1)])
def test_device_replay_matches_oracle(pool_file, W, K):
    from paper_2603_18897_b200.replay import ReplayBatch
    from paper_2603_18897_b200.synth import coding_replay_corpus

    dp = DevicePool(c2_pool(pool_file))
    ks = KeysetTable()
    c = coding_replay_corpus(dp, 4000, window_capacity=W, seed=11, ksets=ks)
    rb = ReplayBatch(dp, c, W, K, ks)
    rb.launch()
    top1, top3, hits, unsure = rb.tallies.cpu().numpy().tolist()
    assert unsure == 0  # ASCII corpus: every hit decided on the device
    exp = bridge.score_corpus(dp.image, c, dp.keys, W, K, threads=8)
    assert (top1, top3, hits, c.n_calls) == exp
    # the fused replay (one kernel, no records) gives the same tallies
    assert rb.launch_fused()
    assert rb.tallies.cpu().numpy().tolist() == [top1, top3, hits, 0]


@pytest.mark.gpu
def test_device_replay_unsure_calls_go_to_the_host():
    """Non-ASCII FormatTemplate text and container-valued arguments come back
    unsure; the public API re-checks them and still equals the oracle."""
    from paper_2603_18897_b200.events import Event, EventKind, Session, Status
    from paper_2603_18897_b200.mappings import (ArgBinding, FormatTemplate, Normalization,
                                                PathLookup, ValueMapping)
    from paper_2603_18897_b200.mining import MiningConfig, PatternPool, PatternTuple
    from paper_2603_18897_b200.events import EventSignature
    from paper_2603_18897_b200.prediction import score_accuracy

    S = Status.SUCCESS
    fmt = FormatTemplate(prefix="ré ", hole=PathLookup(0, ("path",)), suffix="",
                         normalization=Normalization.NONE)
    pats = (PatternTuple((EventSignature("a", S),), "b",
                         ValueMapping((ArgBinding("cmd", fmt),)), 0.9, 5),
            PatternTuple((EventSignature("a", S),), "c",
                         ValueMapping((ArgBinding("obj", PathLookup(0, ("obj",))),)), 0.8, 5))
    pool = PatternPool(MiningConfig(k=1), pats)
    sessions = []
    for i in range(40):
        p = f"p{i}"
        evs = [Event(f"s{i}", 0, EventKind.TOOL_CALL, "a", S, {}, {"path": p, "obj": [i, {"x": i}]},
                     0, 1),
               Event(f"s{i}", 1, EventKind.TOOL_CALL, "b" if i % 2 else "c", S,
                     {"cmd": f"ré {p}"} if i % 2 else {"obj": [i, {"x": i + (i % 4 == 0)}]},
                     None, 1, 2)]
        sessions.append(Session(f"s{i}", tuple(evs)))
    dp = DevicePool(pool)
    corpus, _, _ = corpus_from_traces(sessions, dp, 16, KeysetTable())
    expect = bridge.score_corpus(dp.image, corpus, dp.keys, 16, None)
    rep = score_accuracy(sessions, pool, window_capacity=16)
    assert rep.to_json() == _report(*expect)
    assert 0 < expect[2] < 40


@pytest.mark.gpu
def test_device_hit_check_fuzz_matches_oracle():
    """Word-wise byte comparison at every length / alignment, lowercase and
    strip normalizations, numbers vs strings, near-miss mutations."""
    import random

    from paper_2603_18897_b200.events import Event, EventKind, EventSignature, Session, Status
    from paper_2603_18897_b200.mappings import (ArgBinding, FormatTemplate, Normalization,
                                                PathLookup, ValueMapping)
    from paper_2603_18897_b200.mining import MiningConfig, PatternPool, PatternTuple
    from paper_2603_18897_b200.replay import ReplayBatch

    S = Status.SUCCESS
    rng = random.Random(7)
    alphabet = "abcXYZ019 _-/."

    def mutate(s):
        r = rng.random()
        if r < 0.5 or not s:
            return s
        if r < 0.7:
            i = rng.randrange(len(s))
            return s[:i] + ("q" if s[i] != "q" else "r") + s[i + 1:]
        if r < 0.85:
            return s + "z"
        return s[:-1]

    def mapping(norm, pre, suf):
        return ValueMapping((ArgBinding("a", PathLookup(0, ("v",))),
                             ArgBinding("b", FormatTemplate(pre, PathLookup(0, ("v",)), suf, norm))))

    pats = (PatternTuple((EventSignature("t0", S),), "t1", mapping(Normalization.LOWERCASE, "P:", ""), 0.9, 5),
            PatternTuple((EventSignature("t0", S),), "t2", mapping(Normalization.TRIM, "", "?x=1"), 0.8, 5),
            PatternTuple((EventSignature("t0", S),), "t3", mapping(Normalization.NONE, "pre ", " suf"), 0.7, 5))
    pool = PatternPool(MiningConfig(k=1), pats)
    norms = {"t1": lambda s: "P:" + s.lower(), "t2": lambda s: s.strip() + "?x=1",
             "t3": lambda s: "pre " + s + " suf"}
    sessions = []
    for i in range(3000):
        kind = rng.random()
        if kind < 0.8:
            v = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 41)))
        elif kind < 0.9:
            v = rng.randrange(-10**6, 10**6)
        else:
            v = rng.choice([1.5, 2.0, -0.25, True, None])
        tgt = rng.choice(["t1", "t2", "t3"])
        a_val = mutate(v) if isinstance(v, str) else (v if rng.random() < 0.7 else str(v))
        text = v if isinstance(v, str) else (str(int(v)) if isinstance(v, float) and v.is_integer()
                                             else str(v))
        b_val = mutate(norms[tgt](text)) if isinstance(v, (str, int, float)) and v is not True \
            else "P:true"
        evs = [Event(f"s{i}", 0, EventKind.TOOL_CALL, "t0", S, {}, {"v": v}, 0, 1),
               Event(f"s{i}", 1, EventKind.LLM_STEP, "", S, None, None, 1, 2),
               Event(f"s{i}", 2, EventKind.TOOL_CALL, tgt, S, {"a": a_val, "b": b_val}, None, 2, 3)]
        sessions.append(Session(f"s{i}", tuple(evs)))
    dp = DevicePool(pool)
    ks = KeysetTable()
    corpus, _, _ = corpus_from_traces(sessions, dp, 16, ks)
    rb = ReplayBatch(dp, corpus, 16, 3, ks)
    rb.launch()
    top1, top3, hits, unsure = rb.tallies.cpu().numpy().tolist()
    assert unsure == 0
    expect = bridge.score_corpus(dp.image, corpus, dp.keys, 16, 3)
    assert (top1, top3, hits, corpus.n_calls) == expect
    assert 200 < hits < 2800

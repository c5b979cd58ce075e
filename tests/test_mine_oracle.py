"""Mining counts: the CPU oracle (literal match_at / window restatement) must
reproduce the reference's mine() on the golden corpora, and the host Phase II
must reproduce the reference's inferred mappings."""

import pytest

import golden_io as G
from oracle import bridge
from paper_2603_18897_b200.mine_engine import decode_context, pack_streams
from paper_2603_18897_b200.mining import MatchRelation, MiningConfig, pattern_sort_key
from paper_2603_18897_b200.packing import SigTable

MINE = G.golden("mine_golden.json")


def _cfg(d):
    return MiningConfig(k=d["k"], sigma=d["sigma"], tau=d["tau"],
                        match_relation=MatchRelation(d["match_relation"]))


def _oracle_mine_mapping_free(sessions, cfg):
    streams = [s.tool_events() for s in sessions]
    sigs = SigTable(sorted({e.tool_type for st in streams for e in st}))
    S = max(sigs.n_sigs, 2)
    rel = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    tables = bridge.mine_counts(pack_streams(streams, sigs), S, cfg.k, rel)
    rows = []
    for t, c, sup, m, f in bridge.select_candidates(*tables, S, cfg.k, cfg.sigma, cfg.tau):
        ctx = tuple(sigs.signature(x) for x in decode_context(c, S, cfg.k))
        rows.append((ctx, sigs.tools[t], f / m, sup))
    rows.sort(key=lambda r: (-r[2], -len(r[0]), r[1],
                             tuple((s.tool_type, s.status.value) for s in r[0])))
    return [([[s.tool_type, s.status.value] for s in ctx], tgt, p, sup) for ctx, tgt, p, sup in rows]


@pytest.mark.parametrize("idx", range(len(MINE["corpora"])))
def test_oracle_counts_reproduce_reference_mine(idx):
    corpus = MINE["corpora"][idx]
    sessions = [G.session(s) for s in corpus["sessions"]]
    cfg = _cfg(corpus["config"])
    got = _oracle_mine_mapping_free(sessions, cfg)
    exp = [([[c["tool"], c["status"]] for c in p["context"]], p["target"], p["p"], p["support"])
           for p in corpus["expected"]]
    assert all(p["mapping"] is None for p in corpus["expected"])
    assert got == exp


def test_phase2_reproduces_reference_mappings():
    """Host Phase II over reference-identical occurrences (the occurrence
    lists come from the host matcher, the counts from the oracle)."""
    from paper_2603_18897_b200 import phase2
    from paper_2603_18897_b200.mine_engine import _occurrences
    from paper_2603_18897_b200.events import signature_of
    from paper_2603_18897_b200.mappings import mapping_to_json

    for corpus in MINE["mapped"]:
        sessions = [G.session(s) for s in corpus["sessions"]]
        cfg = _cfg(corpus["config"])
        streams = [s.tool_events() for s in sessions]
        sig_streams = [[signature_of(e) for e in st] for st in streams]
        for p in corpus["expected"]:
            ctx = tuple(G.session({"id": "x", "events": []}).events) or ()
            from paper_2603_18897_b200.events import EventSignature, Status
            ctx = tuple(EventSignature(c["tool"], Status(c["status"])) for c in p["context"])
            occ = _occurrences(streams, sig_streams, ctx, p["target"], cfg)
            mapping = phase2.infer_mapping(occ, cfg.validation_fraction) if len(occ) >= 2 else None
            got = mapping_to_json(mapping) if mapping is not None else None
            assert got == p["mapping"], (p["context"], p["target"])


def test_vectorised_pattern_order_equals_reference_sort_key():
    import numpy as np

    from paper_2603_18897_b200.mine_engine import (decode_context, encode_context,
                                                   patterns_from_candidates)
    from paper_2603_18897_b200.mining import PatternTuple

    rng = np.random.default_rng(0)
    S, k = 10, 3
    sigs = SigTable([f"t{i}" for i in range(5)])
    rows = set()
    while len(rows) < 400:
        n = int(rng.integers(1, k + 1))
        ctx = tuple(int(x) for x in rng.integers(0, S, n))
        match = int(rng.integers(1, 6))
        rows.add((int(rng.integers(0, 5)), encode_context(ctx, S, k), int(rng.integers(5, 50)),
                  match, int(rng.integers(0, match + 1))))
    cands = np.array(sorted(rows), np.int64)
    cfg = MiningConfig(k=k, sigma=1, tau=0.3)
    got = patterns_from_candidates(cands, sigs, S, cfg)
    exp = []
    for t, c, sup, m, f in cands.tolist():
        if f / m >= cfg.tau:
            exp.append(PatternTuple(tuple(sigs.signature(x) for x in decode_context(c, S, k)),
                                    sigs.tools[t], None, f / m, sup))
    exp.sort(key=pattern_sort_key)
    assert got == exp

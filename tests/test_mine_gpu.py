"""K2 parity on the GPU: mine() against the reference's golden outputs, and
the device count tables against the CPU oracle (bit-exact) at larger sizes."""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import bridge  # noqa: E402
from paper_2603_18897_b200 import mine, mine_frequent_subsequences, validate  # noqa: E402
from paper_2603_18897_b200.events import EventSignature, Status  # noqa: E402
from paper_2603_18897_b200.mappings import mapping_to_json  # noqa: E402
from paper_2603_18897_b200.mine_engine import MineTables  # noqa: E402
from paper_2603_18897_b200.mining import MatchRelation, MiningConfig  # noqa: E402

MINE = G.golden("mine_golden.json")


def _cfg(d):
    return MiningConfig(k=d["k"], sigma=d["sigma"], tau=d["tau"],
                        match_relation=MatchRelation(d["match_relation"]))


def _as_json(p):
    return {"context": [{"tool": s.tool_type, "status": s.status.value} for s in p.context],
            "target": p.target, "mapping": mapping_to_json(p.mapping) if p.mapping else None,
            "p": p.p, "support": p.support, "pattern_id": p.pattern_id}


@pytest.mark.parametrize("group,idx", [("corpora", i) for i in range(len(MINE["corpora"]))]
                         + [("mapped", i) for i in range(len(MINE["mapped"]))])
def test_mine_matches_reference_golden(group, idx):
    corpus = MINE[group][idx]
    sessions = [G.session(s) for s in corpus["sessions"]]
    got = [_as_json(p) for p in mine(sessions, _cfg(corpus["config"]))]
    assert got == corpus["expected"]


def _random_stream(n_sessions, n_sigs, seed, mean_len=8, planted=True):
    rng = np.random.default_rng(seed)
    lens = rng.geometric(1.0 / mean_len, n_sessions)
    total = int(lens.sum())
    tok = rng.integers(0, n_sigs, total, dtype=np.int32)
    if planted:  # skew: a first-order chain so some grams repeat a lot
        nxt = rng.integers(0, n_sigs, n_sigs)
        follow = rng.random(total) < 0.5
        tok[1:][follow[1:]] = nxt[tok[:-1][follow[1:]]]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    tok[starts] |= np.int32(-2**31)
    return tok


@pytest.mark.parametrize("n_sigs,k,rel", [(32, 3, 0), (32, 3, 1), (8, 4, 0), (8, 4, 1),
                                          (16, 1, 0), (12, 2, 1), (6, 5, 0)])
def test_count_tables_match_oracle(n_sigs, k, rel):
    tok = _random_stream(20_000, n_sigs, seed=n_sigs * 10 + k)
    t = MineTables.allocate(n_sigs, k, rel)
    t.count(torch.from_numpy(tok).cuda())
    t.expand()
    ora = bridge.mine_counts(tok, n_sigs, k, rel)
    for dev, ref in zip((t.tool_count, t.support, t.match, t.follow), ora):
        assert np.array_equal(dev.cpu().numpy().astype(np.uint64), ref)


@pytest.mark.parametrize("n_sigs,k,rel,tau", [(32, 3, 0, 0.3), (32, 3, 1, 0.1), (8, 4, 0, 0.05),
                                              (12, 2, 1, 0.5), (6, 5, 0, 1.0), (16, 1, 0, 0.2)])
def test_select_sorted_matches_oracle_order(n_sigs, k, rel, tau):
    """Device selection + rank sort == the oracle's candidates in mine()'s
    output order (mining.py:105-111), including the capacity retry."""
    from paper_2603_18897_b200.mine_engine import patterns_from_candidates
    from paper_2603_18897_b200.packing import SigTable

    tok = _random_stream(20_000, n_sigs, seed=n_sigs * 7 + k)
    t = MineTables.allocate(n_sigs, k, rel)
    t.count(torch.from_numpy(tok).cuda())
    t.expand()
    sigs = SigTable([f"tool{i:02d}" for i in range((n_sigs + 1) // 2)])
    cfg = MiningConfig(k=k, sigma=2, tau=tau,
                       match_relation=MatchRelation.ANCHORED_SUBSEQUENCE if rel == 0
                       else MatchRelation.CONTIGUOUS_SUFFIX)
    ora = bridge.mine_counts(tok, n_sigs, k, rel)
    cands = np.array(bridge.select_candidates(*ora, n_sigs, k, cfg.sigma, cfg.tau), np.int64)
    exp = patterns_from_candidates(cands.reshape(-1, 5), sigs, n_sigs, cfg)
    got = t.select_sorted(cfg.sigma, cfg.tau, cap=7)  # forces the retry path
    assert len(got) == len(exp) > 0
    assert got.patterns(sigs) == exp
    assert np.array_equal(got.p, [p.p for p in exp])


def test_count_is_additive_across_shards():
    """Shards counted into one histogram == the whole corpus (K3 merge basis)."""
    tok = _random_stream(50_000, 32, seed=5)
    cut = int(np.flatnonzero(tok < 0)[len(np.flatnonzero(tok < 0)) // 2])
    whole = MineTables.allocate(32, 3, 0)
    whole.count(torch.from_numpy(tok).cuda())
    parts = MineTables.allocate(32, 3, 0)
    parts.count(torch.from_numpy(tok[:cut]).cuda())
    parts.count(torch.from_numpy(tok[cut:]).cuda())
    assert torch.equal(whole.hist, parts.hist)


def test_frequent_subsequences_spec_example():
    A, B, C = (EventSignature(t, Status.SUCCESS) for t in "ABC")
    got = mine_frequent_subsequences([[A, B], [A, C], [A, B]], 2)
    assert got == {(A,): 3, (B,): 2, (A, B): 2}


def test_frequent_subsequences_random_vs_bruteforce():
    import itertools
    import random

    rng = random.Random(3)
    sigs = [EventSignature(t, s) for t in "abc" for s in (Status.SUCCESS, Status.FAIL)]
    windows = [[rng.choice(sigs) for _ in range(rng.randint(0, 5))] for _ in range(300)]
    exp: dict = {}
    for w in windows:
        subs = {tuple(w[i] for i in range(len(w)) if m >> i & 1) for m in range(1, 1 << len(w))}
        for s in subs:
            exp[s] = exp.get(s, 0) + 1
    exp = {s: c for s, c in exp.items() if c >= 4}
    assert mine_frequent_subsequences(windows, 4) == exp


def test_validate_matches_counts():
    corpus = MINE["corpora"][0]
    sessions = [G.session(s) for s in corpus["sessions"]]
    cfg = _cfg(corpus["config"])
    for p in corpus["expected"][:5]:
        ctx = tuple(EventSignature(c["tool"], Status(c["status"])) for c in p["context"])
        assert validate(ctx, p["target"], None, sessions, cfg) == p["p"]


def _host_tokens(c):
    from paper_2603_18897_b200.synth import columnar_flags

    tok = c["sig"].copy()
    tok[columnar_flags(c)] |= np.int32(-2**31)
    return tok


def _dev(c):
    return {k: torch.from_numpy(v).cuda() for k, v in c.items()}


def test_columnar_ingest_count_matches_oracle():
    from paper_2603_18897_b200.mine_engine import ingest_count
    from paper_2603_18897_b200.synth import columnar_corpus

    c = columnar_corpus(300_000, seed=11)
    tok = _host_tokens(c)
    for k, rel in ((3, 0), (3, 1), (2, 0)):
        t = MineTables.allocate(32, k, rel)
        out = torch.empty(len(tok), dtype=torch.int32, device="cuda")
        counters = ingest_count(t, _dev(c), tokens_out=out)
        assert np.array_equal(out.cpu().numpy(), tok)
        assert int(counters[0]) == int((tok < 0).sum()) and int(counters[1]) == 0
        t.expand()
        ora = bridge.mine_counts(tok, 32, k, rel)
        for dev, ref in zip((t.tool_count, t.support, t.match, t.follow), ora):
            assert np.array_equal(dev.cpu().numpy().astype(np.uint64), ref)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_columnar_staged_count_equals_single_pass(k):
    """Two-pass (staged words + L2 pass) histogram == the fused single pass ==
    the oracle's tables, including a ragged tail (n not a multiple of 4)."""
    from paper_2603_18897_b200.mine_engine import ingest_count
    from paper_2603_18897_b200.synth import columnar_corpus

    c = columnar_corpus(123_457, seed=20 + k)
    dev = _dev(c)
    a = MineTables.allocate(32, k, 0)
    b = MineTables.allocate(32, k, 0)
    ca = ingest_count(a, dev, staged=True)
    cb = ingest_count(b, dev, staged=False)
    assert torch.equal(a.hist, b.hist) and torch.equal(ca, cb)
    a.expand()
    ora = bridge.mine_counts(_host_tokens(c), 32, k, 0)
    for dev_t, ref in zip((a.tool_count, a.support, a.match, a.follow), ora):
        assert np.array_equal(dev_t.cpu().numpy().astype(np.uint64), ref)


def test_columnar_staged_count_spills_skewed_grams():
    """A corpus dominated by one all-success gram and one third-event gram:
    the 16-bit shared-memory counters of the staged pass (success lattice,
    dense block) spill many times per CTA; the histogram still equals the
    plain RED pass."""
    from paper_2603_18897_b200.mine_engine import ingest_count

    rng = np.random.default_rng(5)
    short, long_ = 6_000_000, 14_000_000
    sess = np.concatenate([np.arange(short) // 3, short // 3 + np.arange(long_) // 1000])
    seq = np.concatenate([np.arange(short) % 3, np.arange(long_) % 1000]).astype(np.int32)
    sig = np.where(rng.random(short + long_) < 0.03, rng.integers(0, 32, short + long_), 7)
    t = seq.astype(np.float64) * 10.0
    c = dict(session=sess.astype(np.int32), seq=seq, t_start=t, t_end=t + 1.0,
             sig=sig.astype(np.int32))
    dev = _dev(c)
    for k in (3, 2):
        a = MineTables.allocate(32, k, 0)
        b = MineTables.allocate(32, k, 0)
        ca = ingest_count(a, dev, staged=True)
        cb = ingest_count(b, dev, staged=False)
        assert torch.equal(a.hist, b.hist) and torch.equal(ca, cb)
        assert int(a.hist.max()) > 10_000_000  # the hot cells spilled many times


def test_mine_columnar_patterns_match_oracle_selection():
    from paper_2603_18897_b200.mine_engine import mine_columnar, patterns_from_candidates
    from paper_2603_18897_b200.packing import SigTable
    from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

    c = columnar_corpus(200_000, seed=12)
    sigs = SigTable(C4_TOOLS)
    cfg = MiningConfig(k=3, sigma=5, tau=0.3)
    got = mine_columnar(_dev(c), sigs, cfg)
    ora = bridge.mine_counts(_host_tokens(c), 32, 3, 0)
    cands = np.array(bridge.select_candidates(*ora, 32, 3, cfg.sigma, cfg.tau), np.int64)
    exp = patterns_from_candidates(cands.reshape(-1, 5), sigs, 32, cfg)
    assert got == exp and len(got) > 0


@pytest.mark.parametrize("rel", [0, 1])
def test_columnar_count_at_scale_matches_oracle(rel):
    """25M events of the C4 corpus (a quarter of the benchmarked size; the
    bench checks the full 100M) through the staged two-pass count: tables
    and the selected pattern list against the oracle, both relations."""
    from oracle.parity import mining_parity
    from paper_2603_18897_b200.mine_engine import ingest_count, patterns_from_candidates
    from paper_2603_18897_b200.packing import SigTable
    from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

    c = columnar_corpus(25_000_000, seed=40 + rel)
    sigs = SigTable(C4_TOOLS)
    cfg = MiningConfig(k=3, sigma=5, tau=0.3, match_relation=MatchRelation.CONTIGUOUS_SUFFIX
                       if rel else MatchRelation.ANCHORED_SUBSEQUENCE)
    t = MineTables.allocate(32, 3, rel)
    ingest_count(t, _dev(c))
    t.expand()
    got = t.select_sorted(cfg.sigma, cfg.tau).patterns(sigs)
    r = mining_parity(t, c, 32, 3, rel)
    assert r["ok"], r["mismatch"]
    cands = np.array(bridge.select_candidates(*r["oracle_tables"], 32, 3, cfg.sigma, cfg.tau),
                     np.int64).reshape(-1, 5)
    assert got == patterns_from_candidates(cands, sigs, 32, cfg) and len(got) > 0


def test_sharded_mining_equals_single_device(tmp_path):
    """mine_columnar over 2 ranks (whole-session shards, histogram merged by
    all-reduce; gloo ranks sharing this GPU, launched by torchrun) == the
    single-device result."""
    import json
    import os
    import socket
    import subprocess
    import sys

    from paper_2603_18897_b200.mine_engine import mine_columnar
    from paper_2603_18897_b200.packing import SigTable
    from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "ranks.json"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(root, "tests", "sharded_mine_worker.py"), str(out)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-3000:]
    got = json.loads(out.read_text())
    c = columnar_corpus(400_000, seed=31)
    whole = mine_columnar(_dev(c), SigTable(C4_TOOLS), MiningConfig(k=3, sigma=5, tau=0.3))
    exp = [[[[s.tool_type, s.status.value] for s in p.context], p.target, p.p, p.support]
           for p in whole]
    assert got["0"] == exp and got["1"] == exp and len(exp) > 0


@pytest.mark.parametrize("seed", [1, 2])
def test_mine_jsonl_equals_mine_of_ingested_sessions(seed):
    """JSONL -> native columnar ingest -> device counts == mine() over the
    reference-semantics ingest_trace sessions (payload-free trace, so no
    mapping can be inferred and p = follow / match on both paths)."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_ingest import _trace

    from paper_2603_18897_b200.events import ingest_trace
    from paper_2603_18897_b200.ingest import mine_jsonl

    text = _trace(seed, n_sessions=2000, payloads=False)
    cfg = MiningConfig(k=3, sigma=5, tau=0.3)
    got = mine_jsonl(text, cfg)
    exp = mine(ingest_trace(text).sessions, cfg)
    assert got == exp and len(got) > 0


def test_sharded_session_mining_with_mappings(tmp_path):
    """mine(shard, cfg, group=...) over 2 ranks (contiguous session shards,
    gloo ranks sharing this GPU): counts merged by all-reduce, Phase II over
    the gathered occurrences -- both ranks return the reference's golden
    patterns, mappings included."""
    import json
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "ranks.json"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(root, "tests", "sharded_mine_worker.py"), str(out), "sessions"]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-3000:]
    got = json.loads(out.read_text())
    for i, corpus in enumerate(MINE["mapped"]):
        exp = [[p["context"], p["target"], p["mapping"], p["p"], p["support"]]
               for p in corpus["expected"]]
        exp = [[[[c["tool"], c["status"]] for c in e[0]]] + e[1:] for e in exp]
        assert got["0"][i] == exp and got["1"][i] == exp


@pytest.mark.parametrize("rel,k", [(MatchRelation.ANCHORED_SUBSEQUENCE, 3),
                                   (MatchRelation.ANCHORED_SUBSEQUENCE, 4),
                                   (MatchRelation.CONTIGUOUS_SUFFIX, 3)])
def test_device_occurrences_equal_host_rescan(rel, k):
    """paste_mine_occurrences + the K1 sort == the host rescan of every
    stream (_collect_occurrences filtered to the target, mining.py:215-227,
    277-279) for every selected candidate: same occurrences, stream order,
    matched events and histories."""
    from paper_2603_18897_b200.events import Event, EventKind, Session, signature_of
    from paper_2603_18897_b200.mine_engine import (_count_corpus, _occurrences, decode_context,
                                                   device_occurrences)

    rng = np.random.default_rng(k + 10 * rel.value.__len__())
    tools = ["a", "b", "c", "d"]
    sessions = []
    for i in range(400):
        evs = []
        for j in range(int(rng.integers(1, 14))):
            evs.append(Event(f"s{i}", j, EventKind.TOOL_CALL, tools[int(rng.integers(0, 4))],
                             Status.FAIL if rng.random() < 0.2 else Status.SUCCESS, None, None,
                             float(j), float(j) + 0.5))
        sessions.append(Session(f"s{i}", tuple(evs)))
    cfg = MiningConfig(k=k, sigma=2, tau=1e-9, match_relation=rel)
    streams = [s.tool_events() for s in sessions]
    sigs, tables, tok_dev = _count_corpus(streams, cfg)
    rows = [r for r in tables.select(cfg.sigma, cfg.tau).tolist() if r[4] >= 2]
    assert len(rows) > 50
    S = tables.n_sigs
    cands = [(decode_context(r[1], S, cfg.k), r[0], r[4]) for r in rows]
    flat = [e for st in streams for e in st]
    got = device_occurrences(tok_dev, flat, sigs, cands, cfg)
    # positions against the oracle restatement (oracle/occurrences.py)
    from oracle.occurrences import occurrences as oracle_occurrences
    from paper_2603_18897_b200.mine_engine import occurrence_positions
    tok_host = tok_dev.cpu().numpy()
    for (cs, tool, f), (anc, pk) in zip(cands, occurrence_positions(tok_dev, sigs, cands, cfg)):
        exp = oracle_occurrences(tok_host, cs, tool, cfg.k,
                                 rel is MatchRelation.CONTIGUOUS_SUFFIX)
        assert [(int(a), tuple(int(x) for x in p)) for a, p in zip(anc, pk)] == exp
    sig_streams = [[signature_of(e) for e in st] for st in streams]
    for (cs, tool, f), occ in zip(cands, got):
        ctx = tuple(sigs.signature(x) for x in cs)
        exp = _occurrences(streams, sig_streams, ctx, sigs.tools[tool], cfg)
        assert len(occ) == len(exp) == f
        for (m1, n1), (m2, n2) in zip(occ, exp):
            assert n1 is n2
            assert all(x is y for x, y in zip(m1.events, m2.events))
            assert len(m1.history) == len(m2.history)
            assert all(x is y for x, y in zip(m1.history, m2.history))


def test_mine_with_non_json_payload_outside_mappings():
    """A payload the tape cannot hold (a tuple) on an event no mapping needs:
    mine() still equals the reference semantics (per-candidate occurrence
    sets instead of the corpus tape)."""
    from paper_2603_18897_b200.events import Event, EventKind, Session

    sessions = []
    for i in range(20):
        url = f"https://x{i}.example"
        evs = (Event(f"s{i}", 0, EventKind.TOOL_CALL, "search", Status.SUCCESS, {"q": str(i)},
                     {"list": [{"url": url}]}, 0.0, 1.0),
               Event(f"s{i}", 1, EventKind.TOOL_CALL, "web_fetch", Status.SUCCESS, {"url": url},
                     {"ok": 1}, 2.0, 3.0),
               Event(f"s{i}", 2, EventKind.TOOL_CALL, "note", Status.SUCCESS, None,
                     ("opaque", i), 4.0, 5.0))
        sessions.append(Session(f"s{i}", evs))
    pats = mine(sessions, MiningConfig(k=1, sigma=5, tau=0.5))
    m = [p for p in pats if p.target == "web_fetch"]
    assert m and m[0].mapping is not None and m[0].p == 1.0


@pytest.mark.parametrize("slices,rel,k", [(1, 0, 3), (2, 0, 3), (3, 1, 3), (8, 0, 3), (5, 0, 2),
                                          (4, 1, 4)])
def test_sliced_expand_sums_to_full_expand(slices, rel, k):
    """The target-sliced tail (paste_mine_transpose_slices + expand_slice):
    for every slice count the per-block tables -- tools of the block, match
    of the contexts anchored in it -- add up to the full expansion exactly,
    and each block's selection is the full selection restricted to its
    tools."""
    import ctypes

    from paper_2603_18897_b200 import _native
    from paper_2603_18897_b200._native import check, ptr
    from paper_2603_18897_b200.synth import columnar_corpus

    lib = _native.lib()
    c = columnar_corpus(300_000, seed=70 + slices)
    full = MineTables.allocate(32, k, rel)
    from paper_2603_18897_b200.mine_engine import ingest_count
    ingest_count(full, _dev(c))
    part = MineTables.allocate(32, k, rel)
    part.hist.copy_(full.hist)
    full.expand()
    w = int(lib.paste_mine_slice_cols(32, slices))
    n_win = full.n_bins // 34
    hist_t = torch.empty(slices * w * n_win, dtype=torch.int32, device="cuda")
    d = part.desc()
    check(lib.paste_mine_transpose_slices(ctypes.byref(d), slices, ptr(hist_t), None), lib)
    acc = {n: torch.zeros_like(getattr(full, n)) for n in ("tool_count", "support", "match",
                                                           "follow")}
    for r in range(slices):
        for n in acc:
            getattr(part, n).zero_()
        block = hist_t[r * w * n_win:(r + 1) * w * n_win].contiguous()
        check(lib.paste_mine_expand_slice(ctypes.byref(d), ptr(block), r * w, w, None), lib)
        for n in acc:
            acc[n] += getattr(part, n)
    for n in acc:
        assert torch.equal(acc[n], getattr(full, n)), n

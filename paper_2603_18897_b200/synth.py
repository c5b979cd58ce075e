"""Columnar synthetic agent traces for the benchmark configurations.

The reference generates traces object by object (workloads.py:297-331, about
0.3 s per 1k sessions); 1M live sessions need a vectorised generator.  This
one reproduces the reference's motif structure and payload shapes:

* motifs (workloads.py:102-214): search -> web_fetch (+ retry after a
  failure), file_editor -> terminal, grep -> file_editor, search -> batch of
  web_fetch;
* results use the shapes of ``tool_result`` (simulation.py:150-178): url_list
  ``{"list": [{"url", "rank"}...], "total"}``, file_hits ``{"hits": [{"path",
  "line"}...], "count"}``, edit ``{"path", "applied"}``, echo ``{"ok",
  "token"}`` and the failure form ``{"ok": false, "error", "token"}``.

Payload tapes are *shape-interned*: every payload of one kind has the same
node array (only its scalar bytes differ), so events share one node template
and carry only their own bytes -- ``paste_event_ref.node_base`` points at the
template, ``byte_base`` at the event's bytes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tape import KeyTable, TapeArena

TOOLS = ("search", "web_fetch", "file_editor", "terminal", "grep")
SEARCH, FETCH, EDITOR, TERMINAL, GREP = range(5)
MOTIFS = ("search_visit", "edit_verify", "locate_examine", "batch_fetch")

# payload kinds
K_SEARCH, K_GREP, K_EDIT, K_ECHO, K_FAIL = range(5)
_HEX = np.frombuffer(b"0123456789abcdef", dtype=np.uint8)


def _sample_payloads() -> dict[int, tuple[object, bool]]:
    """Payload samples with 'X' placeholders; bool = all runs share one value."""
    return {
        K_SEARCH: ({"list": [{"url": f"https://XXXXXXXX-{i}.example/doc", "rank": i}
                             for i in range(5)], "total": 5}, True),
        K_GREP: ({"hits": [{"path": f"src/mXXXXXXXX_{i}.py", "line": 10 * (i + 1)}
                           for i in range(4)], "count": 4}, True),
        K_EDIT: ({"path": "src/fix_XXXXXXXXXX.py", "applied": True}, False),
        K_ECHO: ({"ok": True, "token": "XXXXXXXXXXXXXXXX"}, False),
        K_FAIL: ({"ok": False, "error": "execution_failed", "token": "XXXXXXXXXXXXXXXX"}, False),
    }


@dataclass
class ShapeTemplates:
    nodes: np.ndarray              # NODE_DTYPE, all templates back to back
    node_base: np.ndarray          # i64[kind]
    byte_tmpl: list[np.ndarray]    # per kind template bytes
    runs: list[np.ndarray]         # per kind: [n_runs, run_len] byte positions of 'X'
    shared: list[bool]


def make_templates(keys: KeyTable) -> ShapeTemplates:
    arena = TapeArena(keys, keep_objects=False)
    samples = _sample_payloads()
    for k in range(len(samples)):
        arena.add(samples[k][0])
    nodes, data, refs = arena.arrays()
    byte_tmpl, runs, shared = [], [], []
    for k in range(len(samples)):
        b0 = int(refs[k, 1])
        b1 = int(refs[k + 1, 1]) if k + 1 < len(samples) else len(data)
        tmpl = data[b0:b1].copy()
        pos = np.flatnonzero(tmpl == ord("X"))
        # split into runs of consecutive positions
        cuts = np.flatnonzero(np.diff(pos) != 1) + 1
        groups = np.split(pos, cuts) if len(pos) else []
        runs.append(np.stack(groups) if groups else np.zeros((0, 0), np.int64))
        byte_tmpl.append(tmpl)
        shared.append(samples[k][1])
    return ShapeTemplates(nodes, refs[:, 0].copy(), byte_tmpl, runs, shared)


def payload_kind(tool: np.ndarray, ok: np.ndarray) -> np.ndarray:
    kind = np.full(tool.shape, K_ECHO, np.int8)
    kind[tool == SEARCH] = K_SEARCH
    kind[tool == GREP] = K_GREP
    kind[tool == EDITOR] = K_EDIT
    kind[~ok] = K_FAIL
    return kind


def fill_payloads(tmpl: ShapeTemplates, kind: np.ndarray, rng: np.random.Generator,
                  byte_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Bytes for a batch of payloads: returns (bytes u8[], refs i64[n,2])."""
    n = len(kind)
    # bytes are laid out grouped by kind (refs carry each event's byte base)
    starts = np.zeros(n, np.int64)
    blocks = []
    at = 0
    for k in range(len(tmpl.byte_tmpl)):
        idx = np.flatnonzero(kind == k)
        if not len(idx):
            continue
        t = tmpl.byte_tmpl[k]
        block = np.broadcast_to(t, (len(idx), len(t))).copy()
        runs = tmpl.runs[k]
        if runs.size:
            n_runs, run_len = runs.shape
            if tmpl.shared[k]:
                hexes = _HEX[rng.integers(0, 16, (len(idx), run_len), dtype=np.uint8)]
                for r in range(n_runs):
                    block[:, runs[r]] = hexes
            else:
                hexes = _HEX[rng.integers(0, 16, (len(idx), n_runs * run_len), dtype=np.uint8)]
                block[:, runs.reshape(-1)] = hexes
        starts[idx] = at + np.arange(len(idx), dtype=np.int64) * len(t)
        at += block.size
        blocks.append(block.reshape(-1))
    out = np.concatenate(blocks) if blocks else np.zeros(1, np.uint8)
    refs = np.empty((n, 2), np.int64)
    refs[:, 0] = tmpl.node_base[kind]
    refs[:, 1] = starts + byte_offset
    return out, refs


class MotifStream:
    """Per-session motif state machines advanced one tool call at a time.

    Transitions follow the reference's scripts with its default rates
    (visit 0.51, verify 0.55, open 0.38; batch_fetch issues ``fetch_count``
    fetches after one search); web_fetch / terminal fail with probability
    ``fail_rate`` and a failed fetch is retried once (search_visit retry).
    """

    def __init__(self, n_sessions: int, seed: int, fail_rate: float = 0.05,
                 fetch_count: int = 15):
        self.n = n_sessions
        self.rng = np.random.default_rng(seed)
        self.motif = self.rng.integers(0, len(MOTIFS), n_sessions, dtype=np.int8)
        self.prev = np.full(n_sessions, -1, np.int8)
        self.prev_ok = np.ones(n_sessions, bool)
        self.run = np.zeros(n_sessions, np.int16)  # fetches since last search (batch)
        self.fail_rate = fail_rate
        self.fetch_count = fetch_count

    def step(self) -> tuple[np.ndarray, np.ndarray]:
        """Next (tool id in TOOLS, ok) per session."""
        u = self.rng.random(self.n)
        m, prev, ok_prev = self.motif, self.prev, self.prev_ok
        nxt = np.empty(self.n, np.int8)
        # search_visit: search -> fetch (0.51) | search; failed fetch -> retry fetch
        sv = m == 0
        nxt[sv] = SEARCH
        sel = sv & (prev == SEARCH) & (u < 0.51)
        nxt[sel] = FETCH
        nxt[sv & (prev == FETCH) & ~ok_prev] = FETCH
        # edit_verify: editor -> terminal (0.55) | editor
        ev = m == 1
        nxt[ev] = EDITOR
        nxt[ev & (prev == EDITOR) & (u < 0.55)] = TERMINAL
        # locate_examine: grep -> editor (0.38) | grep
        le = m == 2
        nxt[le] = GREP
        nxt[le & (prev == GREP) & (u < 0.38)] = EDITOR
        # batch_fetch: search then fetch_count fetches, repeat
        bf = m == 3
        nxt[bf] = FETCH
        restart = bf & ((prev == -1) | (self.run >= self.fetch_count))
        nxt[restart] = SEARCH
        self.run[bf & (nxt == SEARCH)] = 0
        self.run[bf & (nxt == FETCH)] += 1
        ok = np.ones(self.n, bool)
        may_fail = (nxt == FETCH) | (nxt == TERMINAL)
        ok[may_fail] = self.rng.random(int(may_fail.sum())) >= self.fail_rate
        self.prev, self.prev_ok = nxt, ok
        return nxt, ok


def sig_map(sigs) -> np.ndarray:
    """TOOLS index -> tool id in a SigTable (interning missing tools)."""
    return np.array([sigs.tool(t) for t in TOOLS], np.int32)


def tokens(tool: np.ndarray, ok: np.ndarray, tool_ids: np.ndarray) -> np.ndarray:
    return (2 * tool_ids[tool] + ok.astype(np.int32)).astype(np.int32)


class LiveWorkload:
    """C3 generator: N sessions, one new tool event per session per batch."""

    def __init__(self, sigs, keys, n_sessions: int, seed: int = 2603, fail_rate: float = 0.05):
        self.n = n_sessions
        self.tmpl = make_templates(keys)
        self.stream = MotifStream(n_sessions, seed, fail_rate=fail_rate)
        self.tool_ids = sig_map(sigs)
        self.rng = np.random.default_rng(seed + 1)
        self.max_batch_bytes = n_sessions * max(len(t) for t in self.tmpl.byte_tmpl)

    def next_batch(self):
        from .live import EventBatch

        tool, ok = self.stream.step()
        kind = payload_kind(tool, ok)
        data, ref = fill_payloads(self.tmpl, kind, self.rng)
        # the narrow wire form (node_base only) is produced with the batch
        return EventBatch(tokens(tool, ok, self.tool_ids), ref, data,
                          np.ascontiguousarray(ref[:, 0], dtype=np.int32))


class StressWorkload:
    """C3 on the 1,000-pattern / 20-tool stress pool (SURVEY.md 8(d) pool ii):
    every session observes one tool call per step, a uniformly drawn tool of
    the pool (as the reference's latency test cycles through its 20 tools,
    test_prediction.py:186-199) that fails with probability ``fail_rate``;
    the pool has no mappings, so payloads are the small echo shape."""

    def __init__(self, sigs, keys, n_sessions: int, seed: int = 2603, n_tools: int = 20,
                 fail_rate: float = 0.2):
        self.n = n_sessions
        self.tmpl = make_templates(keys)
        self.rng = np.random.default_rng(seed)
        self.tool_ids = np.array([sigs.tool(f"tool{i}") for i in range(n_tools)], np.int32)
        self.fail_rate = fail_rate
        self.max_batch_bytes = n_sessions * max(len(t) for t in self.tmpl.byte_tmpl)

    def next_batch(self):
        from .live import EventBatch

        tool = self.rng.integers(0, len(self.tool_ids), self.n)
        ok = self.rng.random(self.n) >= self.fail_rate
        kind = np.where(ok, K_ECHO, K_FAIL).astype(np.int8)
        data, ref = fill_payloads(self.tmpl, kind, self.rng)
        tok = (2 * self.tool_ids[tool] + ok.astype(np.int32)).astype(np.int32)
        return EventBatch(tok, ref, data, np.ascontiguousarray(ref[:, 0], dtype=np.int32))


def stress_pool(seed: int = 1001, n_patterns: int = 1000, n_tools: int = 20):
    """The 1,000-pattern / 20-tool stress pool of the reference's runtime
    overhead criterion (test_acceptance.py:507-527), regenerated from its
    recipe: random contexts of 1-3 signatures, distinct (context, target)."""
    import random

    from .events import EventSignature, Status
    from .mining import MiningConfig, PatternPool, PatternTuple

    rng = random.Random(seed)
    tools = [f"tool{i}" for i in range(n_tools)]
    pats, seen = [], set()
    while len(pats) < n_patterns:
        ctx = tuple(EventSignature(rng.choice(tools), rng.choice([Status.SUCCESS, Status.FAIL]))
                    for _ in range(rng.randint(1, 3)))
        target = rng.choice(tools)
        if (ctx, target) in seen:
            continue
        seen.add((ctx, target))
        pats.append(PatternTuple(context=ctx, target=target, mapping=None,
                                 p=round(rng.uniform(0.3, 1.0), 4), support=5))
    return PatternPool(config=MiningConfig(), patterns=tuple(pats))


# ---------------------------------------------------------------------------
# C4: columnar mining corpus
# ---------------------------------------------------------------------------

C4_TOOLS = tuple(f"tool{i:02d}" for i in range(16))
# planted motifs at the paper's transition rates:
# edit -> verify 0.55, grep -> editor 0.38, search -> fetch 0.51
C4_PLANTED = ((0, 1, 0.55), (2, 0, 0.38), (3, 4, 0.51))


def columnar_corpus(n_events: int, seed: int = 2603, mean_len: float = 8.0,
                    fail_rate: float = 0.05, split_rate: float = 0.01, max_len: int = 64):
    """Columnar trace of ``n_events`` tool events: session idx (first-appearance
    order), seq, t_start / t_end (ms), sig over the 16 C4 tools (interned in
    sorted order, so sig = 2 * tool + success).  Tools follow a first-order
    chain with the planted motifs; ``split_rate`` of the think gaps exceed the
    300 s inactivity threshold (ingest splits them into new segments)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.geometric(1.0 / mean_len, int(n_events / mean_len * 1.2) + 16), max_len)
    csum = np.cumsum(lens)
    n_sess = int(np.searchsorted(csum, n_events)) + 1
    lens = lens[:n_sess].copy()
    lens[-1] -= int(csum[n_sess - 1] - n_events)
    starts = np.zeros(n_sess, np.int64)
    starts[1:] = np.cumsum(lens)[:-1]
    session = np.repeat(np.arange(n_sess, dtype=np.int32), lens)
    seq = (np.arange(n_events, dtype=np.int64) - np.repeat(starts, lens)).astype(np.int32)

    # tool chain, vectorised across sessions (longest first so active = prefix)
    order = np.argsort(-lens, kind="stable")
    olens, ostarts = lens[order], starts[order]
    tool = np.empty(n_events, np.int8)
    nxt_planted = np.full(16, -1, np.int8)
    p_planted = np.zeros(16)
    for a, b, p in C4_PLANTED:
        nxt_planted[a], p_planted[a] = b, p
    prev = rng.integers(0, 16, n_sess, dtype=np.int8)
    for pos in range(int(olens.max())):
        m = int(np.searchsorted(-olens, -pos, side="left"))  # sessions longer than pos
        if m == 0:
            break
        pv = prev[:m]
        u = rng.random(m)
        t = rng.integers(0, 16, m, dtype=np.int8)
        planted = (nxt_planted[pv] >= 0) & (u < p_planted[pv])
        t[planted] = nxt_planted[pv][planted]
        tool[ostarts[:m] + pos] = t
        prev[:m] = t
    ok = rng.random(n_events) >= fail_rate
    sig = (2 * tool.astype(np.int32) + ok).astype(np.int32)

    dur = rng.exponential(800.0, n_events)
    think = rng.exponential(2000.0, n_events)
    think[rng.random(n_events) < split_rate] += 400_000.0
    think[starts] = 0.0
    step = think + dur
    cum = np.cumsum(step)
    cum -= np.repeat(cum[starts] - step[starts], lens)  # restart per session
    t0 = np.repeat(rng.uniform(0, 1e9, n_sess), lens)
    t_end = t0 + cum
    t_start = t_end - dur
    return {"session": session, "seq": seq, "t_start": t_start, "t_end": t_end, "sig": sig}


def columnar_flags(c, inactivity_ms: float = 300_000.0) -> np.ndarray:
    """Segment-start flags of a columnar corpus (host restatement of the gap
    split, used by the CPU baseline and tests)."""
    s, ts, te = c["session"], c["t_start"], c["t_end"]
    b = np.ones(len(s), bool)
    b[1:] = (s[1:] != s[:-1]) | ((ts[1:] - te[:-1]) > inactivity_ms)
    return b


# ---------------------------------------------------------------------------
# C5: long tool outputs (64 KB url_list results)
# ---------------------------------------------------------------------------

def long_output_corpus(n_sessions: int, seed: int = 2603, result_size: int = 1120):
    """Per session one ``tool_result(url_list, result_size)`` payload
    (simulation.py:150-178; 65,005 B of canonical JSON at 1120 entries) and
    the next call's argument ``list[(37 * s) % result_size].url``
    (SURVEY.md 8(d) C5).  Payloads are shape-interned: one node template,
    per-session bytes."""
    from .tape import KeyTable, TapeArena

    keys = KeyTable()
    arena = TapeArena(keys, keep_objects=False)
    sample = {"list": [{"url": f"https://XXXXXXXX-{i}.example/doc", "rank": i}
                       for i in range(result_size)], "total": result_size}
    arena.add(sample)
    nodes, data, refs = arena.arrays()
    tmpl = data.copy()
    pos = np.flatnonzero(tmpl == ord("X"))
    runs = pos.reshape(-1, 8)
    rng = np.random.default_rng(seed)
    L = len(tmpl)
    out = np.broadcast_to(tmpl, (n_sessions, L)).copy()
    hexes = _HEX[rng.integers(0, 16, (n_sessions, 8), dtype=np.uint8)]
    for r in range(len(runs)):
        out[:, runs[r]] = hexes
    byte_base = np.arange(n_sessions, dtype=np.int64) * L
    ev_refs = np.stack([np.zeros(n_sessions, np.int64), byte_base], axis=1)
    j = (37 * np.arange(n_sessions)) % result_size
    url_node = 3 + 3 * j  # root dict, "list", then (dict, url, rank) per entry
    a = nodes["a"][url_node].astype(np.int64)
    b = nodes["b"][url_node].astype(np.int64)
    t_off = np.zeros(n_sessions + 1, np.int64)
    t_off[1:] = np.cumsum(b)
    flat = out.reshape(-1)
    gather = np.repeat(byte_base + a, b) + (np.arange(int(b.sum())) - np.repeat(t_off[:-1], b))
    return {"nodes": nodes, "bytes": flat, "refs": ev_refs, "target_off": t_off,
            "target_bytes": flat[gather], "expected_node": url_node, "keys": keys,
            "payload_bytes": L, "canonical_json_bytes": None}


# ---------------------------------------------------------------------------
# C2: coding-agent replay corpus (edit_verify / locate_examine)
# ---------------------------------------------------------------------------

class FieldTemplates:
    """Shape-interned payload templates whose variable text is marked by runs
    of one uppercase placeholder letter per field ('A', 'B', ...)."""

    def __init__(self, keys: KeyTable, samples: list):
        arena = TapeArena(keys, keep_objects=False)
        for s in samples:
            arena.add(s)
        self.nodes, data, refs = arena.arrays()
        self.node_base = refs[:, 0].copy()
        self.byte_tmpl, self.fields = [], []
        for k in range(len(samples)):
            b0 = int(refs[k, 1])
            b1 = int(refs[k + 1, 1]) if k + 1 < len(samples) else len(data)
            t = data[b0:b1].copy()
            f = {}
            for letter in b"ABCDEFGH":
                pos = np.flatnonzero(t == letter)
                if len(pos):
                    cuts = np.flatnonzero(np.diff(pos) != 1) + 1
                    f[chr(letter)] = np.stack(np.split(pos, cuts))  # [n_runs, run_len]
            self.byte_tmpl.append(t)
            self.fields.append(f)

    def fill(self, kind: int, values: dict[str, np.ndarray]) -> np.ndarray:
        """[n, len] payload bytes of template ``kind``; values[letter] is [n, run_len]
        (every run of a field gets the same text)."""
        n = len(next(iter(values.values())))
        t = self.byte_tmpl[kind]
        block = np.broadcast_to(t, (n, len(t))).copy()
        for letter, runs in self.fields[kind].items():
            for r in range(len(runs)):
                block[:, runs[r]] = values[letter]
        return block


# payload templates of the two coding motifs (workloads.py:139-193, shapes of
# simulation.py:150-178): edit / verify / grep / open, args then results
_C2_SAMPLES = [
    {"path": "src/fix_AAAAAAAAAA.py", "change": "BBBBBBBBBB"},          # 0 edit args
    {"path": "src/fix_AAAAAAAAAA.py", "applied": True},                 # 1 edit result
    {"cmd": "pytest src/fix_AAAAAAAAAA.py"},                            # 2 verify args
    {"ok": True, "token": "CCCCCCCCCCCCCCCC"},                          # 3 verify result
    {"pattern": "sym_AAAAAAAAAA"},                                      # 4 grep args
    {"hits": [{"path": f"src/mBBBBBBBB_{i}.py", "line": 10 * (i + 1)} for i in range(4)],
     "count": 4},                                                       # 5 grep result
    {"path": "src/mBBBBBBBB_0.py"},                                     # 6 open args
    {"path": "src/mBBBBBBBB_0.py", "applied": True},                    # 7 open result
]
C2_EDIT, C2_VERIFY, C2_GREP, C2_OPEN = range(4)
_C2_TOOL = ("file_editor", "terminal", "grep", "file_editor")


def _hex(rng: np.random.Generator, n: int, width: int) -> np.ndarray:
    return _HEX[rng.integers(0, 16, (n, width), dtype=np.uint8)]


def coding_replay_corpus(dp, n_sessions: int, window_capacity: int = 16, seed: int = 2,
                         ksets=None, rounds: int = 4, verify_rate: float = 0.55,
                         open_rate: float = 0.38):
    """C2 replay corpus as a ReplayCorpus: ``n_sessions`` coding sessions, half
    edit_verify (file_editor -> terminal "pytest <path>" at ``verify_rate``),
    half locate_examine (grep -> file_editor hits[0].path at ``open_rate``),
    ``rounds`` rounds each, every tool call preceded by an LLM step
    (workloads.py:297-366).  Token / path text is random hex; the planted
    dependencies are exact, so mined PathLookup / FormatTemplate bindings hit."""
    from .events import Status
    from .replay import KeysetTable, ReplayCorpus

    ksets = KeysetTable() if ksets is None else ksets
    rng = np.random.default_rng(seed)
    n = n_sessions
    motif = rng.random(n) < 0.5                       # True = locate_examine
    fired = rng.random((n, rounds)) < np.where(motif, open_rate, verify_rate)[:, None]
    kind = np.empty((n, rounds, 2), np.int8)
    kind[:, :, 0] = np.where(motif, C2_GREP, C2_EDIT)[:, None]
    kind[:, :, 1] = np.where(motif, C2_OPEN, C2_VERIFY)[:, None]
    valid = np.ones((n, rounds, 2), bool)
    valid[:, :, 1] = fired
    # per-round field text: A (10 hex), B (10 hex: edit change / 8 hex: grep hash)
    a_txt = _hex(rng, n * rounds, 10).reshape(n, rounds, 10)
    b_txt = _hex(rng, n * rounds, 10).reshape(n, rounds, 10)
    flat_valid = valid.reshape(-1)
    call_kind = kind.reshape(-1)[flat_valid]
    call_round = np.broadcast_to(np.arange(n * rounds).reshape(n, rounds, 1),
                                 (n, rounds, 2)).reshape(-1)[flat_valid]
    call_sess = call_round // rounds
    n_calls_s = valid.reshape(n, -1).sum(axis=1)
    T = len(call_kind)
    call_start = np.zeros(n + 1, np.int64)
    call_start[1:] = np.cumsum(n_calls_s)
    j = np.arange(T, dtype=np.int64) - call_start[call_sess]     # call index in session
    sess_ev0 = 2 * call_start[:-1]                               # LLM + tool per call
    tool_pos = sess_ev0[call_sess] + 2 * j + 1

    tmpl = FieldTemplates(dp.keys, _C2_SAMPLES)
    tool_ids = np.array([dp.sigs.sig(t, Status.SUCCESS) for t in _C2_TOOL], np.int32)
    E = int(2 * T)
    ev_tok = np.full(E, -1, np.int32)
    ev_tok[tool_pos] = tool_ids[call_kind]
    scored = np.flatnonzero(j >= 1)
    C = len(scored)
    # payload ids: results 0..T-1 (call order), then args of scored calls
    ev_evt = np.full(E, -1, np.int32)
    ev_evt[tool_pos] = np.arange(T, dtype=np.int32)

    blocks, bases, node_base = [], np.zeros(T + C, np.int64), np.zeros(T + C, np.int64)
    at = 0

    def emit(tk: int, pids: np.ndarray, values: dict[str, np.ndarray]):
        nonlocal at
        if not len(pids):
            return
        blk = tmpl.fill(tk, values)
        bases[pids] = at + np.arange(len(pids), dtype=np.int64) * blk.shape[1]
        node_base[pids] = tmpl.node_base[tk]
        at += blk.size
        blocks.append(blk.reshape(-1))

    a_of = a_txt.reshape(-1, 10)[call_round]
    b_of = b_txt.reshape(-1, 10)[call_round]
    for ck in range(4):
        ids = np.flatnonzero(call_kind == ck)
        res_vals = {C2_EDIT: {"A": a_of[ids]}, C2_VERIFY: {"C": _hex(rng, len(ids), 16)},
                    C2_GREP: {"B": b_of[ids, :8]}, C2_OPEN: {"B": b_of[ids, :8]}}[ck]
        emit(2 * ck + 1, ids, res_vals)
        sc = np.intersect1d(ids, scored, assume_unique=True)
        args_pid = T + np.searchsorted(scored, sc)
        arg_vals = {C2_EDIT: {"A": a_of[sc], "B": b_of[sc]}, C2_VERIFY: {"A": a_of[sc]},
                    C2_GREP: {"A": a_of[sc]}, C2_OPEN: {"B": b_of[sc, :8]}}[ck]
        emit(2 * ck, args_pid, arg_vals)
    refs = np.stack([node_base, bases], axis=1)
    keysets = np.array([ksets.of_args(s) for s in _C2_SAMPLES[0::2]], np.int32)
    sk = call_kind[scored]
    return ReplayCorpus(
        ev_tok=ev_tok, ev_evt=ev_evt, call_pos=tool_pos[scored].astype(np.int64),
        call_len=np.minimum(window_capacity, 2 * j[scored] + 1).astype(np.int64),
        call_tool=(tool_ids[sk] >> 1).astype(np.int32),
        call_args=(T + np.arange(C)).astype(np.int32), call_keyset=keysets[sk],
        nodes=tmpl.nodes, data=np.concatenate(blocks) if blocks else np.zeros(1, np.uint8),
        refs=refs)

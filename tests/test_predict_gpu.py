"""K4 parity on the GPU: the CUDA predict / admit path against the reference's
golden vectors and, at scale, against the pinned CPU oracle (bit-exact)."""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import bridge  # noqa: E402
from paper_2603_18897_b200 import admit  # noqa: E402
from paper_2603_18897_b200._native import (PASTE_CF_ENTRY16, PASTE_CF_KEY8, PASTE_CF_KEYS,  # noqa: E402
                                           PASTE_CF_UNIQ)
from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.live import LiveSessionTable  # noqa: E402
from paper_2603_18897_b200.mining import load_pool  # noqa: E402
from paper_2603_18897_b200.packing import PredictResult, WindowBatch, admit_tables  # noqa: E402
from paper_2603_18897_b200.policy import parse_policy  # noqa: E402
from paper_2603_18897_b200.prediction import PredictionWindow, Predictor  # noqa: E402
from paper_2603_18897_b200.scheduling import EstimateBook  # noqa: E402
from paper_2603_18897_b200.synth import LiveWorkload, stress_pool  # noqa: E402

CASES = G.golden("predict_golden.json")["cases"]
MOTIF_POLICY = """
speculation_policy:
  default: {allow: false}
  tools:
    web_fetch: {allow: true, max_speculation: full}
    terminal: {allow: true, max_speculation: dry_run}
    search: {allow: true, max_speculation: full}
    file_editor: {allow: true, max_speculation: dry_run}
"""


def _windows(case):
    out = []
    for w in case["windows"]:
        win = PredictionWindow(16)
        for e in w:
            win.observe(G.event(e))
        out.append(win)
    return out


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_predict_matches_reference_golden(case):
    pool = G.pool(case["pool"])
    predictor = Predictor(pool)
    wins = _windows(case)
    K = case["max_candidates"]
    preds = predictor.predict_batch(wins, max_candidates=K)
    for got, exp in zip(preds, case["expected"]):
        assert G.same([G.pred_dict(p) for p in got], exp)
    assert predictor.diagnostics.structural_errors == case["structural_errors"]
    pol = G.policy(case["policy"])
    if pol is None:
        return
    book = G.estimates(case["estimates"])
    if K is not None and K <= 32:  # fused predict + admit kernel
        preds2, acts = predictor.predict_admit_batch(wins, pol, book, max_candidates=K)
    else:  # standalone admit kernel on the predictions
        preds2 = preds
        acts = [admit(p, pol, lambda pr: book.duration(pr.tool_type)) for p in preds]
    for s, (got, exp) in enumerate(zip(acts, case["expected_actions"])):
        assert [(preds2[s].index(a.prediction), int(a.level), a.expected_utility)
                for a in got] == [(e["pred"], e["level"], e["utility"]) for e in exp]


def test_single_window_predict_api():
    case = next(c for c in CASES if c["name"] == "fetch_pool")
    predictor = Predictor(G.pool(case["pool"]))
    for win, exp in zip(_windows(case), case["expected"]):
        assert G.same([G.pred_dict(p) for p in predictor.predict(win)], exp)


def test_admit_matches_reference_golden():
    from paper_2603_18897_b200.prediction import Completeness, PredictedInvocation

    g = G.golden("admit_golden.json")
    pol = G.policy(g["policy"])
    bene = g["benefit"]
    for item in g["lists"]:
        preds = [PredictedInvocation(p["tool"], p["args"], Completeness(p["completeness"]), p["p"],
                                     p["pattern"], p["created_at"]) for p in item["preds"]]
        acts = admit(preds, pol, lambda p: bene[p.tool_type] * (1 + p.created_at % 2))
        assert [(preds.index(a.prediction), int(a.level), a.expected_utility) for a in acts] == \
            [(a["pred"], a["level"], a["utility"]) for a in item["actions"]]


def _compare(dev: PredictResult, ora: PredictResult):
    assert np.array_equal(dev.n_pred, ora.n_pred)
    assert np.array_equal(dev.struct_err, ora.struct_err)
    K, B = dev.K, dev.B
    slot_valid = (np.arange(K)[None, :] < dev.n_pred[:, None]).reshape(-1)
    assert np.array_equal(dev.pred_pat[slot_valid], ora.pred_pat[slot_valid])
    assert np.array_equal(dev.pred_comp[slot_valid], ora.pred_comp[slot_valid])
    arg_valid = np.repeat(slot_valid & (dev.pred_comp != 2), B)
    assert np.array_equal(dev.pred_arg[arg_valid], ora.pred_arg[arg_valid])
    assert np.array_equal(dev.n_act, ora.n_act)
    act_valid = (np.arange(K)[None, :] < dev.n_act[:, None]).reshape(-1)
    assert np.array_equal(dev.act_pred[act_valid], ora.act_pred[act_valid])
    assert np.array_equal(dev.act_level[act_valid], ora.act_level[act_valid])
    # fp64 utilities: same single multiply -> bit-exact (tolerance 1e-6 rel not needed)
    assert np.array_equal(dev.act_util[act_valid].view(np.int64),
                          ora.act_util[act_valid].view(np.int64))


def _live_vs_oracle(dp, n, steps, seed, policy, book, K=8, workload=None, updates=None):
    wl = workload or LiveWorkload(dp.sigs, dp.keys, n, seed=seed)
    table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes, policy, book,
                             max_candidates=K)
    W, R = table.W, table.regions
    host = WindowBatch(W, np.full(n * W, -1, np.int32), np.full(n * W, -1, np.int32),
                       np.zeros(n, np.int64), None, [], slot_major=1)
    refs = np.zeros((R * n, 2), np.int64)
    host.arena = (wl.tmpl.nodes, np.zeros(1, np.uint8), refs)
    tables = admit_tables(dp.sigs, policy, book.duration)
    total_preds = 0
    for step in range(steps):
        if updates and step in updates:  # EWMA moves: the device tables follow
            for tool, ms in updates[step]:
                book.update(tool, ms)
            table.refresh_estimates(book)
            tables = admit_tables(dp.sigs, policy, book.duration)
        batch = wl.next_batch()
        if step % 2:
            batch.node = None  # alternate the wide (16-B directory entry) observe input
        region = step % R
        table.step(batch)
        dev = table.fetch()
        ora = bridge.predict(dp.image, host, K, tables, new_tok=batch.tok,
                             new_ref=np.ascontiguousarray(batch.ref), new_evt_base=region * n,
                             new_byte_base=region * table.max_batch_bytes, threads=8)
        _compare(dev.session_major(), ora)
        total_preds += int(dev.n_pred.sum())
    state = table.host_state()
    assert np.array_equal(state["tok"], host.tok) and np.array_equal(state["count"], host.count)
    return total_preds


@pytest.mark.parametrize("plan", [True, False])
def test_live_c3_pool_matches_oracle(plan, monkeypatch):
    """The live-plan kernel (default) and the general match-table kernel."""
    if not plan:
        monkeypatch.setenv("PASTE_NO_LIVE_PLAN", "1")
    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    book = EstimateBook()
    for tool, ms in (("search", 700.0), ("web_fetch", 1080.0), ("file_editor", 300.0),
                     ("terminal", 1420.0), ("grep", 400.0)):
        book.update(tool, ms)
    n_preds = _live_vs_oracle(DevicePool(pool), 20_000, 24, 7, parse_policy(MOTIF_POLICY).policy, book)
    assert n_preds > 20_000 * 24  # the pool fires on this workload


def test_live_follows_estimate_updates():
    """EstimateBook.update between steps + refresh_estimates: utilities and
    per-tool arbitration use the current EWMA, as the reference reads
    estimates.duration at every prediction (simulation.py:428-429)."""
    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    book = EstimateBook()
    ups = {3: [("search", 700.0), ("web_fetch", 5000.0)], 9: [("terminal", 1.5), ("search", 3.0)],
           14: [("web_fetch", 0.0)]}
    n_preds = _live_vs_oracle(DevicePool(pool), 5_000, 18, 11, parse_policy(MOTIF_POLICY).policy,
                              book, updates=ups)
    assert n_preds > 0


@pytest.mark.parametrize("plan", [True, False])
def test_live_stress_pool_matches_oracle(plan, monkeypatch):
    """1,000-pattern pool; the synthetic tools are renamed onto the pool's tools."""
    from paper_2603_18897_b200 import synth
    from paper_2603_18897_b200.policy import SpeculationPolicy

    if not plan:
        monkeypatch.setenv("PASTE_NO_LIVE_PLAN", "1")
    pool = stress_pool()
    dp = DevicePool(pool)

    class Renamed(LiveWorkload):
        def __init__(self):
            super().__init__(dp.sigs, dp.keys, 10_000, seed=3)
            self.rng2 = np.random.default_rng(9)

        def next_batch(self):
            b = super().next_batch()
            tools = self.rng2.integers(0, 20, len(b.tok))
            ok = self.rng2.random(len(b.tok)) < 0.7
            b.tok = (2 * np.array([dp.sigs.tool(f"tool{t}") for t in range(20)])[tools]
                     + ok).astype(np.int32)
            return b

    n = _live_vs_oracle(dp, 10_000, 20, 3, SpeculationPolicy(default_allow=True), EstimateBook(),
                        K=8, workload=Renamed())
    assert n > 0


def test_generic_kernel_path_matches_too():
    """Re-run the golden and live parity tests with the generic (non-fast)
    kernel pinned, so both device code paths stay parity-checked."""
    import os
    import subprocess
    import sys

    if os.environ.get("PASTE_FORCE_GENERIC") or os.environ.get("PASTE_NO_MATCH_TABLE"):
        pytest.skip("already running pinned to an alternative kernel path")
    for var in ("PASTE_FORCE_GENERIC", "PASTE_NO_MATCH_TABLE"):
        env = dict(os.environ, **{var: "1"})
        proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__,
                               "-k", "golden or live"], env=env, capture_output=True, text=True,
                              cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert proc.returncode == 0, var + proc.stdout[-3000:] + proc.stderr[-3000:]


@pytest.mark.parametrize("fmt", [None, 0, 1, 2, 4])
def test_compact_records_expand_to_the_full_records(fmt):
    """Compaction of the K-slot records into the narrow streams, at the
    table's narrowest widths (None) and each width flag alone / none."""
    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    book = EstimateBook()
    dp = DevicePool(pool)
    n = 50_000
    wl = LiveWorkload(dp.sigs, dp.keys, n, seed=21)
    table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes,
                             parse_policy(MOTIF_POLICY).policy, book, max_candidates=8)
    if fmt is not None:
        table.cformat = fmt
    for step in range(20):
        table.step(wl.next_batch())
        full = table.fetch().session_major()
        comp = table.fetch_compact()
        _compare(comp.expand(dp.image.patterns, table.benefit), full)
        assert comp.nbytes < 0.2 * table.output_nbytes()


@pytest.mark.parametrize("variant", ["motif", "negative_benefit", "allow_all_k3", "wide_format",
                                     "ship_bytes", "pred_stream", "pinned_inputs", "no_plan",
                                     "no_plan_pred_stream", "narrow8", "narrow8_pinned",
                                     "no_keys", "no_uniq", "tight_bound", "narrow2",
                                     "narrow2_pinned", "key16", "narrow1", "narrow1_pinned"])
def test_serve_pipeline_yields_the_step_records(variant, monkeypatch):
    """The pipelined serving loop (fused predict + compaction kernel, step
    i+1's upload / compute overlapping step i's download) returns exactly
    what the sequential step (K-slot records) returns: expanded records
    equal the full records, and in the same stream format the streams equal
    the compaction kernel's.  The serving format ships match-table keys
    (PASTE_CF_ENTRY16) unless the variant turns it off."""
    from paper_2603_18897_b200.policy import SpeculationPolicy

    if variant.startswith("no_plan"):  # the general fused kernel
        monkeypatch.setenv("PASTE_NO_LIVE_PLAN", "1")
        variant = variant[len("no_plan_"):] or "motif"
    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    dp = DevicePool(pool)
    n = 30_000
    policy = parse_policy(MOTIF_POLICY).policy
    book = EstimateBook()
    K = 8
    if variant == "negative_benefit":  # exact _beats arbitration path
        book.update("search", -700.0)
        book.update("terminal", -5.0)
    if variant == "allow_all_k3":
        policy, K = SpeculationPolicy(default_allow=True), 3
    wl_a = LiveWorkload(dp.sigs, dp.keys, n, seed=31)
    wl_b = LiveWorkload(dp.sigs, dp.keys, n, seed=31)
    seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, book,
                           max_candidates=K)
    pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, book,
                           max_candidates=K)
    if variant == "ship_bytes":  # payload bytes uploaded into the arena regions too
        seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, book,
                               max_candidates=K, ship_bytes=True)
        pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, book,
                               max_candidates=K, ship_bytes=True)
    if variant == "wide_format":
        seq.cformat = pip.cformat = 0
        pip.sformat = PASTE_CF_ENTRY16
    if variant == "pred_stream":
        pip.sformat = pip.cformat
    else:
        assert pip.sformat & PASTE_CF_ENTRY16
    if variant == "no_keys":
        pip.sformat &= ~(PASTE_CF_KEYS | PASTE_CF_UNIQ | PASTE_CF_KEY8)
    if variant == "no_uniq":
        pip.sformat &= ~PASTE_CF_UNIQ
    if variant == "key16":  # u16 match-table keys instead of u8 plan codes
        assert pip.sformat & PASTE_CF_KEY8
        pip.sformat &= ~PASTE_CF_KEY8
    if variant == "tight_bound":  # every step outgrows its download bound: the rest is fetched
        pip.serve_bound_margin = 64
    steps = 20
    expect, full = [], []
    for _ in range(steps):
        seq.step(wl_a.next_batch())
        full.append(seq.fetch().session_major())
        r = seq.fetch_compact()
        expect.append(tuple(a.copy() for a in (r.hdr, r.pred, r.arg, r.act)))
    def feed():
        for _ in range(steps):
            b = wl_b.next_batch()
            if variant.startswith("narrow8"):  # u8 token + u16 node on the wire
                b = b.narrowed()
                assert b.tok8 is not None and pip.narrow8
            if variant.startswith("narrow2"):  # u8 token + u8 node code on the wire
                b = b.narrowed(pip.codes)
                assert b.node8 is not None and pip.narrow8
            if variant.startswith("narrow1"):  # u8 event code on the wire
                b = b.narrowed(pip.codes, pip.ecodes)
                assert b.ev8 is not None and pip.narrow8
            if variant in ("pinned_inputs", "narrow8_pinned", "narrow2_pinned",
                           "narrow1_pinned"):  # batched copies
                b.tok = torch.from_numpy(b.tok).pin_memory()
                b.node = torch.from_numpy(b.node).pin_memory()
                b.ref = torch.from_numpy(np.ascontiguousarray(b.ref)).pin_memory()
                if b.tok8 is not None:
                    b.pin()
            yield b

    got = []
    for r in pip.serve(feed()):
        got.append((tuple(a.copy() for a in (r.hdr, r.pred, r.arg, r.act)),
                    r.expand(dp.image.patterns, pip.benefit)))
    assert len(got) == steps
    for e, f, (g, g_exp) in zip(expect, full, got):
        _compare(g_exp, f)
        for i, (x, y) in enumerate(zip(e, g)):
            if i == 1 and pip.sformat != seq.cformat:  # pred stream: keys in ENTRY16
                continue
            if i in (0, 3) and pip.sformat & PASTE_CF_KEYS:  # no hdr / act streams
                assert len(y) == 0
                continue
            if i == 2 and pip.sformat & PASTE_CF_UNIQ:  # one reference per unit
                assert len(y) <= len(x)
                continue
            assert np.array_equal(x, y)
    if variant == "ship_bytes":  # same arena contents
        assert torch.equal(seq.bytes, pip.bytes) and torch.equal(seq.refs, pip.refs)


def test_action_keys_match_canonical_arg_hash():
    """Device scheduler keys of admitted actions (paste_action_keys) ==
    canonical_arg_hash of the decoded prediction arguments (the host mirror,
    pinned to the reference's hashes in test_hash.py), for every non-warm
    action; warm-only actions carry no argument key."""
    from paper_2603_18897_b200.events import canonical_arg_hash
    from paper_2603_18897_b200.packing import decode_actions, decode_predictions
    from paper_2603_18897_b200.tape import ArrayTapes

    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    dp = DevicePool(pool)
    n = 4000
    wl = LiveWorkload(dp.sigs, dp.keys, n, seed=41)
    table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes,
                             parse_policy(MOTIF_POLICY).policy, EstimateBook(), max_candidates=8,
                             ship_bytes=True)
    checked = warm = 0
    for step in range(20):
        table.step(wl.next_batch())
        if step < 16:
            continue
        keys, state = table.action_keys()
        keys, state = keys.cpu().numpy(), state.cpu().numpy()
        res = table.fetch().session_major()
        hs = table.host_state()
        arena = ArrayTapes(wl.tmpl.nodes, hs["bytes"], hs["refs"], dp.keys)
        preds = decode_predictions(res, dp.image, arena, [0.0] * n, 0.0)
        acts = decode_actions(res, preds)
        K = table.K
        for s in range(n):
            for j, a in enumerate(acts[s]):
                slot = j * n + s  # slot-major action records
                if a.level.value == 1:
                    assert state[slot] == 1
                    warm += 1
                    continue
                assert state[slot] == 0
                assert keys[slot].tobytes().hex() == canonical_arg_hash(a.prediction.args)
                checked += 1
    assert checked > 1000 and warm > 0


@pytest.mark.parametrize("n,steps", [(400_000, 6), (1_000_000, 18)])
def test_live_beyond_one_persistent_sweep(n, steps):
    """Sizes past one persistent-CTA sweep (grid SMs x resident CTAs x 128
    threads = 151,552 sessions on a B200): the multi-chunk CTA loop with
    walk-memo reuse across chunks (predict_fast_kernel) and the fused
    serving kernel's multi-thousand-tile look-back (predict_compact_kernel),
    every record of every step against the oracle.  The 1M x 18 case is the
    benchmarked C3 configuration with every window full."""
    from oracle.parity import live_parity

    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    book = EstimateBook()
    for tool, ms in (("search", 700.0), ("web_fetch", 1078.8), ("file_editor", 300.0),
                     ("terminal", 1424.2), ("grep", 400.0)):
        book.update(tool, ms)
    r = live_parity(DevicePool(pool), parse_policy(MOTIF_POLICY).policy, book, n, steps, K=8,
                    seed=n + steps)
    assert r["kslot_ok"] and r["serve_ok"], r["mismatch"]
    assert r["serve_kernel"].startswith("fused")
    assert r["predictions"] > n * steps


def test_node_codes_append_only_and_bounded():
    """NodeCodes: new node arrays get the next codes (in sorted order within a
    batch) and codes never change;
    past 256 node arrays encode() declines (the 3-byte form is kept)."""
    from paper_2603_18897_b200.live import NodeCodes

    c = NodeCodes()
    a = c.encode(np.array([700, 5, 700, 9], np.int64))
    assert a.tolist() == [2, 0, 2, 1] and c.n == 3
    b = c.encode(np.array([9, 11, 5], np.int64))
    assert b.tolist() == [1, 3, 0] and c.host.numpy()[:4].tolist() == [5, 9, 700, 11]
    assert c.encode(np.arange(1000, 1300)) is None and c.n == 4
    assert c.encode(np.arange(1000, 1252)).max() == 255 and c.n == 256


def test_serve_follows_estimate_updates():
    """refresh_estimates between serve() calls: the plan's utilities and
    per-tool winners change, so its u8 plan codes (PASTE_CF_KEY8) and the
    host's copy of the plan are rebuilt; every served step still equals the
    K-slot step under the same estimates."""
    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    dp = DevicePool(pool)
    policy = parse_policy(MOTIF_POLICY).policy
    n = 4096
    books = EstimateBook(), EstimateBook()
    wl_a, wl_b = (LiveWorkload(dp.sigs, dp.keys, n, seed=13) for _ in range(2))
    seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, books[0])
    pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, books[1])
    assert pip.sformat & PASTE_CF_KEY8
    phases = [[], [("search", 700.0), ("web_fetch", 5000.0)], [("terminal", 1.5), ("search", 3.0)],
              [("web_fetch", 0.0)]]
    n_act = 0
    for ups in phases:
        for tool, ms in ups:
            for b in books:
                b.update(tool, ms)
        if ups:
            seq.refresh_estimates(books[0])
            pip.refresh_estimates(books[1])
        full = []
        for _ in range(6):
            seq.step(wl_a.next_batch())
            full.append(seq.fetch().session_major())
        got = [r.expand(dp.image.patterns, pip.benefit)
               for r in pip.serve(wl_b.next_batch() for _ in range(6))]
        assert len(got) == 6
        for f, g in zip(full, got):
            _compare(g, f)
            n_act += int(f.n_act.sum())
    assert n_act > 0

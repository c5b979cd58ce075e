"""K5 leaf scan (candidate_paths), device evaluate() and the score_accuracy
replay against the reference's golden outputs."""

import random

import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_18897_b200 import candidate_paths, evaluate, score_accuracy  # noqa: E402
from paper_2603_18897_b200 import phase2  # noqa: E402
from paper_2603_18897_b200.device_ops import candidate_paths_batch  # noqa: E402
from paper_2603_18897_b200.events import Event, EventKind, Status  # noqa: E402
from paper_2603_18897_b200.mappings import (ArgBinding, FormatTemplate, IndexedFallback,  # noqa: E402
                                            MatchedContext, MappingStructureError, Normalization,
                                            PathLookup, ValueMapping)

PATHS = G.golden("paths_golden.json")["cases"]


def test_candidate_paths_matches_reference():
    for case in PATHS:
        got = candidate_paths(case["payload"], case["target"], case["budget"])
        assert [list(p) for p in got.paths] == case["paths"], (case["target"], case["budget"])
        assert got.truncated == case["truncated"]


def test_candidate_paths_batch_equals_single_calls():
    payloads = [c["payload"] for c in PATHS]
    targets = [c["target"] for c in PATHS]
    batch = candidate_paths_batch(payloads, targets, 10_000)
    for c, b in zip(PATHS, batch):
        single = candidate_paths(c["payload"], c["target"], 10_000)
        assert b == single


def _ev(tool, status=Status.SUCCESS, result=None, seq=0):
    return Event("s", seq, EventKind.TOOL_CALL, tool, status, {"i": seq}, result, 0.0, 1.0)


def test_evaluate_matches_host_restatement_on_random_contexts():
    rng = random.Random(17)
    for trial in range(300):
        lst = [{"url": f"u{trial}-{j}", "n": j, "flag": j % 2 == 0} for j in range(rng.randint(0, 5))]
        src = _ev("search", result={"list": lst, "total": float(len(lst)), "title": " Mixed CASE "})
        hist = [src] + [_ev(rng.choice(["web_fetch", "grep"]), rng.choice(list(Status)), {}, j + 1)
                        for j in range(rng.randint(0, 4))]
        ctx = MatchedContext(events=(src, hist[-1]), history=tuple(hist))
        mapping = ValueMapping((
            ArgBinding("a", PathLookup(0, ("list", rng.randint(0, 5), "url"))),
            ArgBinding("b", IndexedFallback(0, ("list",), rng.randint(0, 3), ("url",), "web_fetch")),
            ArgBinding("c", FormatTemplate("x ", PathLookup(0, ("title",)), "!",
                                           rng.choice(list(Normalization)))),
            ArgBinding("d", FormatTemplate("", PathLookup(0, ("list", 0, "flag")), "")),
            ArgBinding("e", PathLookup(0, ("total",))),
            ArgBinding("f", PathLookup(1, ("missing",))),
        ))
        got = evaluate(mapping, ctx)
        exp_args, exp_unbound = {}, []
        for b in mapping.bindings:
            v = phase2.resolve(b.expr, ctx)
            if v is phase2.UNBOUND:
                exp_unbound.append(b.arg_name)
            else:
                exp_args[b.arg_name] = v
        assert got.args == exp_args and got.unbound == tuple(exp_unbound)
        assert all(type(got.args[k]) is type(exp_args[k]) for k in exp_args)


def test_evaluate_structural_error_raises():
    src = _ev("search", result={"x": 1})
    with pytest.raises(MappingStructureError):
        evaluate(ValueMapping((ArgBinding("x", PathLookup(3, ("x",))),)), [src])


def test_score_accuracy_matches_reference():
    for case in G.golden("score_golden.json")["cases"]:
        sessions = [G.session(s) for s in case["sessions"]]
        rep = score_accuracy(sessions, G.pool(case["pool"]), window_capacity=case["window"],
                             max_candidates=case["max_candidates"])
        assert rep.to_json() == case["expected"]


@pytest.mark.parametrize("shared", [True, False])
@pytest.mark.parametrize("budget", [10_000, 2_000, 1, 0])
def test_long_output_leaf_scan_matches_oracle(budget, shared):
    """Both the per-query scan and the shape-shared scan (candidates listed
    once per payload shape) against the oracle's candidate_paths."""
    import numpy as np

    from oracle import bridge
    from paper_2603_18897_b200.device_ops import LeafScanBatch
    from paper_2603_18897_b200.synth import long_output_corpus

    c = long_output_corpus(3000, seed=5)
    b = LeafScanBatch(c["nodes"], c["bytes"], c["refs"], c["target_off"], c["target_bytes"],
                      node_budget=budget, shared=shared)
    b.launch()
    n_out, out, tr = bridge.leaf_scan(c["nodes"], c["bytes"], c["refs"], c["target_off"],
                                      c["target_bytes"], node_budget=budget, threads=8)
    assert np.array_equal(b.n_out.cpu().numpy(), n_out)
    assert np.array_equal(b.trunc.cpu().numpy(), tr)
    dev = b.out_nodes.view(3000, -1).cpu().numpy()
    for q in range(3000):
        k = min(int(n_out[q]), 4)
        assert np.array_equal(dev[q, :k], out[q, :k])


def _occ(context_tool, target_tool, result, actual_args, fails=0, seq0=0):
    src = Event("s", seq0, EventKind.TOOL_CALL, context_tool, Status.SUCCESS, {"q": seq0}, result,
                0.0, 1.0)
    history = [src]
    for j in range(fails):
        history.append(Event("s", seq0 + 1 + j, EventKind.TOOL_CALL, target_tool, Status.FAIL,
                             {"r": j}, {"ok": False}, 2.0 + j, 3.0 + j))
    ctx_events = (src,) if fails == 0 else (src, history[-1])
    actual = Event("s", seq0 + 1 + fails, EventKind.TOOL_CALL, target_tool, Status.SUCCESS,
                   actual_args, {"ok": True}, 9.0, 10.0)
    return (MatchedContext(events=ctx_events, history=tuple(history)), actual)


def test_device_infer_mapping_matches_host_search():
    """K7 inference == the host restatement (pinned by the reference goldens)
    over the acceptance criterion's occurrence families, incl. Unicode."""
    from paper_2603_18897_b200 import infer_mapping

    fams = [
        [_occ("grep", "file_editor", {"hits": [{"path": f"src/м{i}.py"}], "n": 1},
              {"path": f"src/м{i}.py"}, seq0=i) for i in range(10)],
        [_occ("search", "web_fetch", {"list": [{"url": f"u{i}-{j}.example"} for j in range(4)]},
              {"url": f"u{i}-{1 + i % 2}.example"}, fails=1 + i % 2, seq0=i * 10) for i in range(10)],
        [_occ("file_editor", "terminal", {"path": f"pkg/x{i}.py"}, {"cmd": f"pytest pkg/x{i}.py"},
              seq0=i) for i in range(10)],
        [_occ("file_editor", "terminal", {"title": f"  Ünïcode {i} "},
              {"cmd": f"open ünïcode {i}!"}, seq0=i) for i in range(10)],
        [_occ("file_editor", "terminal", {"t": f" Name{i} "}, {"cmd": f"name{i}", "x": i},
              seq0=i) for i in range(10)],
        [_occ("search", "web_fetch", {"v": 1.0 * i, "w": str(i)}, {"a": i, "b": f"id-{i}"},
              seq0=i) for i in range(12)],
    ]
    for occ in fams:
        got = infer_mapping(occ)
        exp = phase2.infer_mapping(occ)
        assert got == exp, (got, exp)

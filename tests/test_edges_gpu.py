"""Edge sizes on the device paths: traces shorter than one tile (or empty),
single sessions, partial warps / tiles in the serving kernels, selection with
no candidates."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import bridge  # noqa: E402
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count  # noqa: E402
from paper_2603_18897_b200.synth import columnar_corpus, columnar_flags  # noqa: E402


def _dev(c):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in c.items()}


@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 33, 511, 513, 1025])
@pytest.mark.parametrize("staged", [True, False])
def test_tiny_columnar_traces_match_oracle(n, staged):
    c = columnar_corpus(4096, seed=n)
    c = {k: np.ascontiguousarray(v[:n]) for k, v in c.items()}
    tok = c["sig"].copy()
    tok[columnar_flags(c)] |= np.int32(-2**31)
    t = MineTables.allocate(32, 3, 0)
    counters = ingest_count(t, _dev(c), staged=staged)
    t.expand()
    ora = bridge.mine_counts(tok, 32, 3, 0)
    for dev_t, ref in zip((t.tool_count, t.support, t.match, t.follow), ora):
        assert np.array_equal(dev_t.cpu().numpy().astype(np.uint64), ref)
    assert int(counters[0]) == int((tok < 0).sum())


def test_empty_trace_and_no_candidates():
    t = MineTables.allocate(32, 3, 0)
    empty = {k: torch.empty(0, dtype=v.dtype, device="cuda")
             for k, v in _dev(columnar_corpus(8, seed=1)).items()}
    ingest_count(t, empty)
    t.expand()
    assert int(t.hist.sum()) == 0
    table = t.select_sorted(5, 0.3)
    assert len(table) == 0


@pytest.mark.parametrize("n", [1, 31, 33, 129])
def test_serving_partial_tiles(n):
    """The fused serving kernel and the compaction at session counts that
    leave partial warps / tiles == the sequential K-slot path."""
    from paper_2603_18897_b200.device_ops import DevicePool
    from paper_2603_18897_b200.live import LiveSessionTable
    from paper_2603_18897_b200.mining import load_pool
    from paper_2603_18897_b200.policy import parse_policy
    from paper_2603_18897_b200.scheduling import EstimateBook
    from paper_2603_18897_b200.synth import LiveWorkload
    from test_predict_gpu import MOTIF_POLICY

    pool = load_pool("paper_2603_18897_b200/data/pool_motif_c3.json")
    dp = DevicePool(pool)
    policy = parse_policy(MOTIF_POLICY).policy
    wl_a, wl_b = (LiveWorkload(dp.sigs, dp.keys, n, seed=5) for _ in range(2))
    seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, EstimateBook())
    pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, EstimateBook())
    from paper_2603_18897_b200._native import PASTE_CF_KEYS, PASTE_CF_UNIQ
    from test_predict_gpu import _compare

    expect, full = [], []
    for _ in range(18):
        seq.step(wl_a.next_batch())
        full.append(seq.fetch().session_major())
        r = seq.fetch_compact()
        expect.append([a.copy() for a in (r.hdr, r.pred, r.arg, r.act)])
    got = [([a.copy() for a in (r.hdr, r.pred, r.arg, r.act)],
            r.expand(dp.image.patterns, pip.benefit))
           for r in pip.serve(wl_b.next_batch() for _ in range(18))]
    for e, f, (g, g_exp) in zip(expect, full, got):
        _compare(g_exp, f)
        for i, (x, y) in enumerate(zip(e, g)):
            if i == 1 and pip.sformat != seq.cformat:  # ENTRY16 ships keys, not patterns
                continue
            if i in (0, 3) and pip.sformat & PASTE_CF_KEYS:  # no hdr / act streams
                continue
            if i == 2 and pip.sformat & PASTE_CF_UNIQ:  # one reference per resolution unit
                assert len(y) <= len(x)
                continue
            assert np.array_equal(x, y)

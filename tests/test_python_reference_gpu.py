"""The live C3 step == the UNMODIFIED reference's predict + admit
(spectool installed into baseline/_ref, prediction.py:76-118,
policy.py:207-236) on the same event batches: every session's decoded
PredictedInvocation list (tool, args, completeness, probability, pattern id)
and SpeculativeAction list (pattern, level, expected utility) compared
exactly, over several steps after the windows fill."""

import pytest

import bench
import spectool_ref as R

pytestmark = pytest.mark.gpu

WHY = R.available()


@pytest.mark.skipif(WHY is not None, reason=str(WHY))
@pytest.mark.parametrize("m,timed,seed", [(700, 4, 11), (3000, 2, 12)])
def test_live_step_equals_reference(m, timed, seed):
    from paper_2603_18897_b200.mining import load_pool
    from paper_2603_18897_b200.policy import parse_policy
    from paper_2603_18897_b200.scheduling import EstimateBook

    pf = "paper_2603_18897_b200/data/pool_motif_c3.json"
    assert len(load_pool(pf).patterns) > 0
    dp, wl, batches, events = R.c3_sample(m, R.W + timed, seed, pf)
    _, _, outs = R.run_c3(events, pf, bench.MOTIF_POLICY, bench.DURATIONS, record=True)
    book = EstimateBook()
    for tool, ms in bench.DURATIONS.items():
        book.update(tool, ms)
    r = R.c3_parity(dp, wl, batches, outs, parse_policy(bench.MOTIF_POLICY).policy, book)
    assert r["ok"], r["first_mismatch"]
    assert r["predictions"] > 3 * m * timed and r["actions"] > m * timed

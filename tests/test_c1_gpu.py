"""C1 at its stated size (BASELINE.json configs[0]): the
reference's deep-research corpus (generate_corpus search_visit / batch_fetch,
1000 sessions, seed 7) mined on the device at tau 0.5 and 0.3 equals the
reference's mine() tuple for tuple (mappings and pattern ids included), and
score_accuracy(W=16) of each device-mined pool on the held-out seed-8 corpus
equals the reference's report (tests/golden/c1_golden.json.gz, written by
running the reference: make_golden.py c1)."""

import pytest

import golden_io as G
from paper_2603_18897_b200 import mine
from paper_2603_18897_b200.mining import MatchRelation, MiningConfig, PatternPool
from paper_2603_18897_b200.prediction import score_accuracy
from test_mine_gpu import _as_json

pytestmark = pytest.mark.gpu

C1 = G.golden("c1_golden.json.gz")


@pytest.mark.parametrize("i", range(len(C1["cases"])))
def test_c1_mine_and_score_match_reference(i):
    case = C1["cases"][i]
    c = case["config"]
    cfg = MiningConfig(k=c["k"], sigma=c["sigma"], tau=c["tau"],
                       match_relation=MatchRelation(c["match_relation"]))
    train = [G.session(s) for s in C1["train"]]
    assert sum(len(s.tool_events()) for s in train) == 4288
    pats = mine(train, cfg)
    assert [_as_json(p) for p in pats] == case["expected"]
    held = [G.session(s) for s in C1["held"]]
    rep = score_accuracy(held, PatternPool(cfg, tuple(pats)), window_capacity=16)
    assert rep.to_json() == case["score"]

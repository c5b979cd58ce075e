"""mine_jsonl end to end on the device: native
parallel parse with payload tapes -> K1 device ordering -> count -> Phase II
over the corpus tapes == mine(ingest_trace(text).sessions) and, where the
ingest leaves the sessions as generated, == the REFERENCE's mine() output
(mine_golden.json mapped corpora, c1_golden.json.gz) tuple for tuple,
mappings and pattern ids included."""

import io

import pytest

import golden_io as G
from paper_2603_18897_b200 import mine
from paper_2603_18897_b200.events import ingest_trace, write_trace
from paper_2603_18897_b200.ingest import mine_jsonl, parse_jsonl_raw
from paper_2603_18897_b200.mining import MatchRelation, MiningConfig
from test_mine_gpu import _as_json

pytestmark = pytest.mark.gpu


def _cfg(d):
    return MiningConfig(k=d["k"], sigma=d["sigma"], tau=d["tau"],
                        match_relation=MatchRelation(d["match_relation"]))


def _jsonl(sessions):
    buf = io.StringIO()
    write_trace(sessions, buf)
    return buf.getvalue()


def _cases():
    mined = G.golden("mine_golden.json")
    out = [(f"mapped{i}", c["sessions"], c["config"], c["expected"])
           for i, c in enumerate(mined["mapped"])]
    c1 = G.golden("c1_golden.json.gz")
    out += [(f"c1-{i}", c1["train"], c["config"], c["expected"])
            for i, c in enumerate(c1["cases"])]
    out += [(f"corpus{i}", c["sessions"], c["config"], c["expected"])
            for i, c in enumerate(mined["corpora"][:8])]
    return out


CASES = _cases()


@pytest.mark.parametrize("i", range(len(CASES)))
def test_mine_jsonl_matches_reference(i):
    name, sess, cfg_d, expected = CASES[i]
    sessions = [G.session(s) for s in sess]
    text = _jsonl(sessions)
    assert parse_jsonl_raw(text, payloads=False) is not None  # the native path runs
    cfg = _cfg(cfg_d)
    got = [_as_json(p) for p in mine_jsonl(text, cfg)]
    ingested = ingest_trace(text).sessions
    assert got == [_as_json(p) for p in mine(ingested, cfg)]
    if [s.session_id for s in ingested] == [s.session_id for s in sessions]:
        assert got == expected
    if name.startswith(("mapped", "c1")):
        assert any(p["mapping"] for p in got)

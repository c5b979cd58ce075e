"""Pool wire format: pool files the REFERENCE wrote
(tests/golden/pool_bytes_golden.json, save_pool in mining.py:318-324) load and
re-serialise byte-identically through this package (the gate of
pkg/tests/test_mining.py:253-276), and pools MINED ON THE DEVICE from the same
corpora serialise to the reference's bytes."""

import io
import json

import pytest

from golden_io import golden, session
from paper_2603_18897_b200.mining import (MiningConfig, PoolFormatError, load_pool, mine_pool,
                                          save_pool)
from paper_2603_18897_b200.mining import MatchRelation

POOLS = golden("pool_bytes_golden.json")["pools"]


@pytest.mark.parametrize("name", sorted(POOLS))
def test_reference_pool_reserialises_byte_identically(name):
    """load -> save gives the reference's own load -> save bytes, and those
    are a fixed point (the edge pool was written from hand-built objects with
    unsorted bindings, which load_pool sorts in both implementations)."""
    saved, resaved = POOLS[name]["saved"], POOLS[name]["resaved"]
    out = io.StringIO()
    save_pool(load_pool(io.StringIO(saved)), out)
    assert out.getvalue() == resaved
    again = io.StringIO()
    save_pool(load_pool(io.StringIO(resaved)), again)
    assert again.getvalue() == resaved
    if name != "edge":
        assert resaved == saved


def test_random_pool_is_the_reference_tests_pool():
    pool = load_pool(io.StringIO(POOLS["random_1000"]["saved"]))
    assert len(pool) == 1000
    kinds = {type(p.mapping.bindings[0].expr).__name__ for p in pool.patterns if p.mapping}
    assert kinds == {"PathLookup"}


@pytest.mark.parametrize("text", ["{broken", '{"version": 99, "patterns": []}', "[]"])
def test_malformed_pools_rejected(text):
    with pytest.raises(PoolFormatError):
        load_pool(io.StringIO(text))


# (pool name, index into mine_golden's mapped corpora): the same generate_corpus
# seed / mix / size / MiningConfig the reference mined the golden pool from
MINED = {"mined_search_batch_t03": 1, "mined_coding_t03": 2}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(MINED))
def test_device_mined_pool_serialises_to_reference_bytes(name):
    corpus = golden("mine_golden.json")["mapped"][MINED[name]]
    c = corpus["config"]
    cfg = MiningConfig(k=c["k"], sigma=c["sigma"], tau=c["tau"],
                       match_relation=MatchRelation(c["match_relation"]))
    ref = json.loads(POOLS[name]["saved"])["config"]
    assert (ref["k"], ref["sigma"], ref["tau"]) == (cfg.k, cfg.sigma, cfg.tau)
    pool = mine_pool([session(s) for s in corpus["sessions"]], cfg)
    out = io.StringIO()
    save_pool(pool, out)
    assert out.getvalue() == POOLS[name]["saved"]

"""K6 greedy admission selection: oracle pinned to the reference's golden
selections (CPU) and the device path against both (GPU)."""

import numpy as np
import pytest

import golden_io as G
from oracle import bridge

CASES = G.golden("greedy_golden.json")["cases"]


def _cols(case):
    jobs = np.array(case["jobs"], dtype=object).reshape(-1, 5)
    ids = np.array([int(j[0]) for j in jobs], np.int64)
    p = np.array([j[1] for j in jobs], np.float64)
    bene = np.array([j[2] for j in jobs], np.float64)
    cost = np.array([int(j[3]) for j in jobs], np.int32)
    dur = np.array([j[4] for j in jobs], np.float64)
    return p, bene, dur, cost, ids


def test_oracle_greedy_matches_reference():
    for case in CASES:
        p, bene, dur, cost, ids = _cols(case)
        got = bridge.greedy(p, bene, dur, cost, ids, case["slack"], case["budget"])
        assert [int(ids[i]) for i in got] == case["expected"]


@pytest.mark.gpu
def test_device_greedy_matches_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_18897_b200.scheduling import Job, JobKind, greedy_speculative_selection

    for case in CASES:
        jobs = [Job(id=int(j[0]), kind=JobKind.SPECULATIVE, tool_type="t", args={}, arg_hash="",
                    session_id="s", p=j[1], benefit_ms=j[2], cost=int(j[3]),
                    duration_est_ms=j[4], submitted_at=0.0) for j in case["jobs"]]
        got = greedy_speculative_selection(jobs, case["slack"], case["budget"])
        assert [j.id for j in got] == case["expected"]


@pytest.mark.gpu
@pytest.mark.parametrize("n,cap,ties", [(2_000_000, 24, False), (1_000_000, 64, True),
                                        (300_000, 8, True), (50, 64, False),
                                        # general path: caps past the radix-select envelope
                                        (2_000_000, 128, False), (1_000_000, 4_000, True),
                                        (100_000, 10**9, True), (70, 65, False)])
def test_device_greedy_matches_oracle_at_scale(n, cap, ties):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_18897_b200.select import select_greedy_arrays

    rng = np.random.default_rng(n + cap)
    if ties:  # few distinct values -> many exact utility ties, id decides
        p = rng.choice([0.25, 0.5, 0.75, 1.0], n)
        bene = rng.choice([100.0, 200.0, 1000.0], n)
        dur = rng.choice([100.0, 1000.0], n)
    else:
        p = rng.uniform(0.05, 1.0, n)
        bene = rng.uniform(100, 10_000, n)
        dur = rng.uniform(100, 5_000, n)
    cost = rng.integers(1, 6, n).astype(np.int32)
    if cap > 1000:
        cost = rng.integers(1, 300, n).astype(np.int32)
    ids = rng.permutation(n).astype(np.int64) + 1
    slack, budget = cap + 3, cap
    got = select_greedy_arrays(p, bene, dur, cost, ids, slack, budget).tolist()
    assert got == bridge.greedy(p, bene, dur, cost, ids, slack, budget)


@pytest.mark.gpu
def test_device_greedy_many_tied_candidates():
    """More than the on-chip sort's 4,096 candidates (every job tied on
    U and p, cost 1, cap 64 -> the radix select is exact, but a cap-64 class
    of all-equal keys with duplicate ids overflows it): the general path
    takes over and still matches the oracle."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_18897_b200.select import select_greedy_arrays

    n = 50_000
    p = np.full(n, 0.5)
    bene = np.full(n, 100.0)
    dur = np.full(n, 100.0)
    cost = np.ones(n, np.int32)
    ids = np.full(n, 7, np.int64)  # duplicate ids: the threshold cannot split the tie
    got = select_greedy_arrays(p, bene, dur, cost, ids, 64, 64).tolist()
    assert got == bridge.greedy(p, bene, dur, cost, ids, 64, 64)


@pytest.mark.gpu
def test_preemption_victim_matches_reference_expression():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import random

    from paper_2603_18897_b200.scheduling import Job, JobKind
    from paper_2603_18897_b200.select import preemption_victim

    rng = random.Random(7)
    for trial in range(200):
        jobs = [Job(id=rng.randint(1, 10_000), kind=JobKind.SPECULATIVE, tool_type="t", args={},
                    arg_hash="", session_id="s", p=rng.choice([0.5, 0.25, rng.random() + 0.01]),
                    benefit_ms=rng.choice([100.0, 50.0]), cost=rng.randint(1, 3),
                    duration_est_ms=rng.choice([100.0, 200.0]), submitted_at=0.0)
                for _ in range(rng.randint(1, 3000 if trial % 10 == 0 else 30))]
        exp = min(jobs, key=lambda j: (j.utility(), -j.id))  # scheduling.py:577
        assert preemption_victim(jobs) is exp

"""N > 1 sharded mining on CPU: two gloo ranks each count a shard of whole
sessions and merge their (k+1)-gram histograms with the engine's merge
(mine_engine.merge_shard_histograms); the merged histogram must equal the
single-process histogram of the whole corpus."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_18897_b200.mine_engine import merge_shard_histograms


def gram_histogram(tok: np.ndarray, S: int, k: int) -> np.ndarray:
    """Host restatement of the (k+1)-gram histogram (mine.cu): one gram per
    event, BEGIN (= S) before a segment's first event; base S + 2."""
    base = S + 2
    start = tok < 0
    sig = (tok & 0x7FFFFFFF).astype(np.int64)
    n = len(tok)
    seg = np.cumsum(start) - 1
    seg_start = np.flatnonzero(start)[seg]
    pos = np.arange(n) - seg_start
    hist = np.zeros(base ** (k + 1), np.int64)
    key = sig.copy()
    mult = base
    for d in range(1, k + 1):
        prev = np.where(pos >= d, sig[np.maximum(np.arange(n) - d, 0)], S)
        key += prev * mult
        mult *= base
    np.add.at(hist, key, 1)
    return hist


def _corpus(seed=0, n_sessions=400, S=10):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 12, n_sessions)
    tok = rng.integers(0, S, int(lens.sum())).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    tok[starts] |= np.int32(-2**31)
    return tok, starts


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tok, starts = _corpus()
    cuts = [0, int(starts[len(starts) // 2]), len(tok)]  # whole sessions per rank
    shard = tok[cuts[rank]:cuts[rank + 1]]
    hist = torch.from_numpy(gram_histogram(shard, 10, 3))
    counters = torch.tensor([int((shard < 0).sum()), 0], dtype=torch.int64)
    merge_shard_histograms(hist, counters, dist.group.WORLD)
    if rank == 0:
        out_q.put((hist.numpy(), counters.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_merge_equals_whole_corpus():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, counters = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    tok, starts = _corpus()
    assert np.array_equal(merged, gram_histogram(tok, 10, 3))
    assert counters[0] == len(starts)


def test_gram_histogram_marginal_counts_every_anchor():
    """The identity expand relies on instead of END grams: summing the
    histogram over the oldest symbol, H[(x, w)] over x, counts the events
    whose newest k symbols (BEGIN-padded) are w -- every anchor, including a
    segment's last event."""
    S, k = 10, 3
    tok, starts = _corpus(seed=3)
    h = gram_histogram(tok, S, k)
    assert h.sum() == len(tok)
    base = S + 2
    marg = h.reshape(base, base ** k).sum(axis=0)  # key = w + base^k * x
    anchors = gram_histogram(tok, S, k - 1)          # k-grams ending at each event
    w_keys = np.arange(base ** k)
    assert np.array_equal(marg, anchors[w_keys])


def _merge_worker(rank, world, port, out_q):
    """The sliced tail's row merge (mine_engine.merge_sorted_tables) over two
    gloo ranks, each holding the sorted rows of its own tools."""
    from paper_2603_18897_b200.mine_engine import merge_sorted_tables

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = _sorted_rows()
    mine = rows[(rows[:, 0] % world) == rank]  # a rank's tools, still in order
    merged = merge_sorted_tables(mine, 10, 3, dist.group.WORLD)
    if rank == 0:
        out_q.put(merged.rows)
    dist.barrier()
    dist.destroy_process_group()


def _sorted_rows():
    """Random selection rows in mine()'s order: (-p, -len, tool, context)."""
    from paper_2603_18897_b200.mine_engine import ctx_offsets

    rng = np.random.default_rng(3)
    S, k = 10, 3
    off = ctx_offsets(S, k)
    n = 400
    length = rng.integers(1, k + 1, n)
    local = np.array([rng.integers(0, S ** int(L)) for L in length])
    ctx = np.array(off)[length] + local
    tool = rng.integers(0, S // 2, n)
    p = rng.choice([0.25, 0.5, 0.75, 1.0, 1 / 3], n)
    rows = np.stack([tool, ctx, rng.integers(5, 50, n), rng.integers(1, 9, n),
                     rng.integers(1, 9, n), p.view(np.int64)], axis=1).astype(np.int64)
    keep = np.unique(rows[:, :2], axis=0, return_index=True)[1]  # (tool, ctx) unique
    rows = rows[np.sort(keep)]
    L = np.searchsorted(np.array(off)[1:], rows[:, 1], side="right")
    return rows[np.lexsort((rows[:, 1] - np.array(off)[L], rows[:, 0], -L,
                            -rows[:, 5].view(np.float64)))]


def test_sliced_tail_row_merge_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(merged, _sorted_rows())

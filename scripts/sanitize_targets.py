"""compute-sanitizer targets (racecheck / synccheck / memcheck / initcheck):
small but multi-CTA instances of the kernels with the riskiest
synchronisation, each checked against the oracle so a sanitizer run also
shows the results stayed right under its serialising scheduler.

  mine   columnar_count_kernel (TMA bulk staging + mbarrier producer /
         consumer ring) and stage_hist_kernel (16-bit packed shared counters
         with guard-bit spills, CTA-pair DSMEM flush) on a corpus with hot
         cells that spill, tables vs the oracle
  live   predict_live_kernel, the two-pass serving step (stage + scatter),
         the look-back serving kernels (PASTE_LIVE_MODE=ticket / pipe) and
         compact.cu's look-back compaction, vs the K-slot records
  order  the K1 general path (order.cu): warp bitonic, CTA chunk sort +
         merge-path passes, warp-aggregated placement
  select sel_greedy_kernel / victim_kernel

usage: python scripts/sanitize_targets.py {mine,live,select,all}
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def mine():
    from oracle import bridge
    from paper_2603_18897_b200.mine_engine import MineTables, ingest_count
    from paper_2603_18897_b200.synth import columnar_corpus

    c = columnar_corpus(300_000, seed=77)
    # a hot cell: one long run of the same signature spills the 16-bit counters
    c["sig"][1000:80_000] = 7
    c["session"][1000:80_000] = c["session"][1000]
    c["seq"][1000:80_000] = np.arange(79_000, dtype=np.int32) + 10_000
    t = np.arange(79_000, dtype=np.float64) * 10.0 + 1e9
    c["t_start"][1000:80_000], c["t_end"][1000:80_000] = t, t + 1.0
    order = np.lexsort((c["seq"], c["t_start"], c["session"]))
    c = {k: np.ascontiguousarray(v[order]) for k, v in c.items()}
    dev = {k: torch.from_numpy(v).cuda() for k, v in c.items()}
    for staged in (True, False):
        tab = MineTables.allocate(32, 3, 0)
        ingest_count(tab, dev, staged=staged)
        tab.expand()
        torch.cuda.synchronize()
    from oracle.parity import mining_parity
    r = mining_parity(tab, c, 32, 3, 0)
    assert r["ok"], r["mismatch"]
    print("mine ok")


def live():
    from paper_2603_18897_b200.device_ops import DevicePool
    from paper_2603_18897_b200.live import LiveSessionTable
    from paper_2603_18897_b200.mining import load_pool
    from paper_2603_18897_b200.policy import parse_policy
    from paper_2603_18897_b200.scheduling import EstimateBook
    from paper_2603_18897_b200.synth import LiveWorkload
    from test_predict_gpu import MOTIF_POLICY, _compare

    pool = load_pool(os.path.join(ROOT, "paper_2603_18897_b200", "data", "pool_motif_c3.json"))
    dp = DevicePool(pool)
    policy = parse_policy(MOTIF_POLICY).policy
    n = int(os.environ.get("SAN_SESSIONS", "20000"))
    steps = int(os.environ.get("SAN_STEPS", "4"))
    wl_a, wl_b = (LiveWorkload(dp.sigs, dp.keys, n, seed=9) for _ in range(2))
    seq = LiveSessionTable(dp, n, wl_a.tmpl.nodes, wl_a.max_batch_bytes, policy, EstimateBook())
    pip = LiveSessionTable(dp, n, wl_b.tmpl.nodes, wl_b.max_batch_bytes, policy, EstimateBook())
    full = []
    for _ in range(steps):
        seq.step(wl_a.next_batch())
        full.append(seq.fetch().session_major())
        seq.fetch_compact()  # compact.cu look-back compaction
    wire2 = os.environ.get("SAN_WIRE2") == "1"  # the 2-byte input (node codes), pinned
    wire1 = os.environ.get("SAN_WIRE1") == "1"  # the 1-byte input (event codes), pinned
    batches = (wl_b.next_batch().narrowed(pip.codes, pip.ecodes).pin() if wire1
               else wl_b.next_batch().narrowed(pip.codes).pin() if wire2 else wl_b.next_batch()
               for _ in range(steps))
    got = [r.expand(dp.image.patterns, pip.benefit) for r in pip.serve(batches)]
    for g, f in zip(got, full):
        _compare(g, f)
    print("live ok", os.environ.get("PASTE_LIVE_MODE", "two-pass"))


def replay():
    from paper_2603_18897_b200.device_ops import DevicePool
    from paper_2603_18897_b200.mining import load_pool
    from paper_2603_18897_b200.replay import KeysetTable, ReplayBatch
    from paper_2603_18897_b200.synth import coding_replay_corpus

    pool = load_pool(os.path.join(ROOT, "paper_2603_18897_b200", "data", "pool_coding_c2_t03.json"))
    dp = DevicePool(pool)
    ks = KeysetTable()
    c = coding_replay_corpus(dp, int(os.environ.get("SAN_SESSIONS", "3000")), window_capacity=16,
                             seed=2, ksets=ks)
    rb = ReplayBatch(dp, c, 16, 8, ks)
    rb.launch()
    two = rb.tallies.cpu().tolist()
    assert rb.launch_fused()
    assert rb.tallies.cpu().tolist() == two
    print("replay ok", two)


def order():
    from oracle.order import order_trace
    from order_cases import random_trace
    from paper_2603_18897_b200.mine_engine import order_columnar

    keys = ("session", "seq", "t_start", "t_end", "sig")
    for il, ls in ((False, ()), (True, (64, 3000))):
        raw = random_trace(3000, seed=5, long_sessions=ls, interleave=il)
        got = order_columnar({k: torch.from_numpy(v).cuda() for k, v in raw.items()}, 3000,
                             300_000.0, with_order=True)
        cols, n_seg, reord, order_ = order_trace(*(raw[k] for k in keys), 3000, 300_000.0)
        assert got.n_segments == n_seg and got.reordered_sessions == reord
        assert np.array_equal(got.order.cpu().numpy(), order_)
        for k in keys:
            assert np.array_equal(got.columns[k].cpu().numpy(), cols[k]), k
    print("order ok")


def select():
    from paper_2603_18897_b200.select import select_greedy_arrays
    rng = np.random.default_rng(5)
    n = 50_000
    p = rng.choice([0.5, 0.25, 0.75], n)
    ben = rng.choice([1000.0, 200.0], n)
    cost = rng.integers(1, 4, n)
    dur = rng.choice([1000.0, 500.0], n)
    ids = np.arange(1, n + 1)
    for slack, budget in ((24, 8), (200, 150)):
        got = ids[select_greedy_arrays(p, ben, dur, cost.astype(np.int32), ids, slack, budget)]
        u = (p * ben) / (cost * dur)
        order = np.lexsort((ids, -p, -u))
        r, b, exp = slack, budget, []
        for i in order:
            if cost[i] <= r and cost[i] <= b:
                exp.append(ids[i])
                r -= cost[i]
                b -= cost[i]
        assert list(got) == exp, (slack, budget)
    print("select ok")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for name, fn in (("mine", mine), ("live", live), ("order", order), ("select", select),
                     ("replay", replay)):
        if which in (name, "all"):
            fn()

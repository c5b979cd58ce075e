"""Per-stage device times of the C4 mining step as it runs on one rank of
N (strong scaling, 100M events in total), measured on one GPU: the count of
100M / N events, the s0-major transpose, the expansion of every column
block (the slowest block bounds the step), the block's sorted selection,
and the row merge.  The collectives (reduce-scatter of the histogram,
all-reduce of the match array, all-gather of the rows) are not measurable
on one GPU and are listed with their sizes."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200 import _native  # noqa: E402
from paper_2603_18897_b200._native import check, ptr  # noqa: E402
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count  # noqa: E402
from paper_2603_18897_b200.mining import MiningConfig  # noqa: E402
from paper_2603_18897_b200.synth import columnar_corpus  # noqa: E402

lib = _native.lib()
total = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cfg = MiningConfig(k=3, sigma=5, tau=0.3)


def dev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


full = columnar_corpus(total)
for N in (1, 2, 4, 8):
    n = total // N
    dev = {k: torch.from_numpy(np.ascontiguousarray(v[:n])).cuda() for k, v in full.items()}
    t = MineTables.allocate(32, 3, 0)
    t_count = dev_time(lambda: (t.hist.zero_(), ingest_count(t, dev)))
    w = int(lib.paste_mine_slice_cols(32, N))
    n_win = t.n_bins // 34
    hist_t = torch.empty(N * w * n_win, dtype=torch.int32, device="cuda")
    d = t.desc()
    t_tr = dev_time(lambda: check(lib.paste_mine_transpose_slices(ctypes.byref(d), N, ptr(hist_t),
                                                                  None), lib))
    blocks = [hist_t[r * w * n_win:(r + 1) * w * n_win].contiguous() for r in range(N)]
    t_exp, t_sel, rows = [], [], []
    for r in range(N):
        def exp(r=r):
            for x in (t.tool_count, t.support, t.match, t.follow):
                x.zero_()
            check(lib.paste_mine_expand_slice(ctypes.byref(d), ptr(blocks[r]), r * w, w, None), lib)
        t_exp.append(dev_time(exp))
        exp()
        w0 = time.perf_counter()
        tab = t.select_sorted(cfg.sigma, cfg.tau)
        t_sel.append((time.perf_counter() - w0) * 1e3)
        rows.append(len(tab))
    full_exp = dev_time(lambda: t.expand()) if N == 1 else None
    print(f"N={N}: count {t_count:.3f} ms, transpose {t_tr:.3f} ms, expand max block "
          f"{max(t_exp):.3f} ms (blocks {['%.3f' % x for x in t_exp]}), select+sort+readback "
          f"max {max(t_sel):.3f} ms (wall), rows per block {rows}"
          + (f", full expand {full_exp:.3f} ms" if full_exp else "")
          + f"; collectives: reduce-scatter {N * w * n_win * 4 / 1e6:.1f} MB, "
            f"match all-reduce {t.match.numel() * 8 / 1e6:.2f} MB")

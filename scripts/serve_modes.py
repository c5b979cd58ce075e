"""C3 serving loop (LiveSessionTable.serve) timed in steady state on 1M
sessions with the 3-byte observe input: device ms per step between
download-complete events.  PASTE_LIVE_MODE picks the serving kernel(s)
(two-pass default, ticket, pipe); run once per mode.  With --ncu, runs a
few steps only (for an ncu capture of the serving kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.live import LiveSessionTable  # noqa: E402
from paper_2603_18897_b200.synth import LiveWorkload  # noqa: E402


class A:
    pool = "c3"


def main():
    ncu = "--ncu" in sys.argv
    if os.environ.get("NOGC") == "1":
        import gc
        gc.disable()
    pool, policy, book = bench.load_setup(A)
    dp = DevicePool(pool)
    n = 1_000_000
    wl = LiveWorkload(dp.sigs, dp.keys, n, seed=2603)
    table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes, policy, book,
                             max_candidates=8)
    for _ in range(table.W + 2):
        table.step(wl.next_batch())
    steps = 6 if ncu else 40
    batches = []
    for _ in range(steps + 4):
        b = wl.next_batch().narrowed(None if os.environ.get("WIRE3") == "1" else table.codes,
                                     table.ecodes if os.environ.get("WIRE1") == "1" else None)
        b.tok = torch.from_numpy(b.tok).pin_memory()
        b.node = torch.from_numpy(b.node).pin_memory()
        b.pin()
        batches.append(b)
    for _ in table.serve(batches[:4], depth=int(os.environ.get("SERVE_DEPTH", "4"))):
        pass
    torch.cuda.synchronize()
    done = []
    if "--trace" in sys.argv:
        table.serve_trace = []
    depth = int(os.environ.get("SERVE_DEPTH", "4"))
    import time
    wall = []
    for r in table.serve(batches[4:], depth=depth):
        done.append(r.downloaded)
        wall.append(time.perf_counter())
    torch.cuda.synchronize()
    tr = getattr(table, "serve_trace", None)
    if tr:
        t0 = tr[10]["u0"]
        for j in range(10, 16):
            e = tr[j]
            print(" ".join(f"{k}={t0.elapsed_time(e[k]) * 1e3:8.1f}" for k in
                           ("u0", "u1", "k0", "k1", "d0", "d1") if k in e))
    import numpy as np
    dw = np.diff(wall) * 1e6
    print(f"host yield gaps us: p50 {np.median(dw):.1f} p90 {np.percentile(dw, 90):.1f} "
          f"max {dw.max():.1f}; supplements {table._serve.get('supplements', 0)}; "
          f"bound {table._serve['bound']}")
    k = len(done) - 1
    ms = done[0].elapsed_time(done[-1]) / k
    print(f"mode={os.environ.get('PASTE_LIVE_MODE', 'two-pass')} uniq={os.environ.get('PASTE_NO_UNIQ') != '1'} "
          f"depth={os.environ.get('SERVE_DEPTH', '4')} fmt={table.sformat} {ms:.4f} ms/step -> {n / ms / 1e6:.2f} G sessions/s")


if __name__ == "__main__":
    main()

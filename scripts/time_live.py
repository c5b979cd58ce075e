"""K4 (predict_live_kernel) device time per 1M-session C3 step, timed as
bench.py times it (L2 flushed between steps), plus a digest of the last
step's records so builds selected by PASTE_LIVE_MINB can be compared for
both speed and identical output (development helper)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.live import LiveSessionTable  # noqa: E402
from paper_2603_18897_b200.synth import LiveWorkload  # noqa: E402


class A:
    pool = "c3"


pool, policy, book = bench.load_setup(A)
dp = DevicePool(pool)
n = 1_000_000
wl = LiveWorkload(dp.sigs, dp.keys, n, seed=2603)
table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes, policy, book, max_candidates=8)
for _ in range(table.W):
    table.step(wl.next_batch())
flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
staged = []
for _ in range(43):
    b = wl.next_batch()
    staged.append((table.steps % table.regions, torch.from_numpy(b.tok).cuda(),
                   torch.from_numpy(b.node).cuda()))
    table.steps += 1
torch.cuda.synchronize()
stream = torch.cuda.current_stream()
for region, tok, node in staged[:3]:
    if os.environ.get("WARM_FLUSH") == "1":  # warm-up steps exactly as the timed ones
        bench.l2_flush(flush)
    table.launch(region, tok, new_node=node)
ts = []
for region, tok, node in staged[3:]:
    bench.l2_flush(flush)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    table.launch(region, tok, new_node=node)
    e1.record(stream)
    ts.append((e0, e1))
torch.cuda.synchronize()
us = [e0.elapsed_time(e1) * 1e3 for e0, e1 in ts]
dig = [int(v.to(torch.int64).sum()) if v.dtype != torch.float64 else float(v.sum())
       for v in table.out.values()]
print(f"MINB={os.environ.get('PASTE_LIVE_MINB', '7')} "
      f"median {statistics.median(us):.1f} us mean {statistics.mean(us):.1f} us min {min(us):.1f}; "
      f"digest {dig}")
if os.environ.get("PER_STEP") == "1":
    print("per step us:", " ".join(f"{u:.1f}" for u in us))

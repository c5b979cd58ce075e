"""C3 live predict+admit: fill windows, then a few steps (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.live import LiveSessionTable  # noqa: E402
from paper_2603_18897_b200.synth import LiveWorkload  # noqa: E402


class A:
    pool = os.environ.get("POOL", "c3")


pool, policy, book = bench.load_setup(A)
dp = DevicePool(pool)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
wl = LiveWorkload(dp.sigs, dp.keys, n, seed=2603)
table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes, policy, book, max_candidates=8)
for _ in range(table.W + 3):
    table.step(wl.next_batch())
torch.cuda.synchronize()
# the fused serving kernel (paste_predict_compact), a few steps
for _ in table.serve([wl.next_batch() for _ in range(4)]):
    pass
torch.cuda.synchronize()

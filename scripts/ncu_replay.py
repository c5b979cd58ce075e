"""Warm C2 replay launches (ncu target): ReplayBatch over the bench corpus."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.mining import load_pool  # noqa: E402
from paper_2603_18897_b200.replay import KeysetTable, ReplayBatch  # noqa: E402
from paper_2603_18897_b200.synth import coding_replay_corpus  # noqa: E402

pool = load_pool(os.path.join("paper_2603_18897_b200", "data", "pool_coding_c2_t03.json"))
dp = DevicePool(pool)
ks = KeysetTable()
c = coding_replay_corpus(dp, 100_000, window_capacity=16, seed=2, ksets=ks)
rb = ReplayBatch(dp, c, 16, 8, ks)
for _ in range(3):
    rb.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    rb.launch()
e1.record()
e1.synchronize()
print("replay step ms", e0.elapsed_time(e1) / 20, "calls", c.n_calls)

"""C2 fused replay launches (ncu -k replay_fused target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_18897_b200.device_ops import DevicePool  # noqa: E402
from paper_2603_18897_b200.mining import load_pool  # noqa: E402
from paper_2603_18897_b200.replay import KeysetTable, ReplayBatch  # noqa: E402
from paper_2603_18897_b200.synth import coding_replay_corpus  # noqa: E402

n_sess = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
pool = load_pool(os.path.join(os.path.dirname(__file__), "..", "paper_2603_18897_b200", "data",
                              "pool_coding_c2_t03.json"))
dp = DevicePool(pool)
ks = KeysetTable()
c = coding_replay_corpus(dp, n_sess, window_capacity=16, seed=2, ksets=ks)
rb = ReplayBatch(dp, c, 16, 8, ks)
for _ in range(3):
    assert rb.launch_fused()
torch.cuda.synchronize()
print(c.n_calls, rb.tallies.cpu().numpy().tolist())

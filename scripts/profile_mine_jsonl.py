"""Host profile of mine_jsonl on the Phase II bench corpus (development helper)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_18897_b200.ingest import mine_jsonl  # noqa: E402
from paper_2603_18897_b200.mining import MiningConfig  # noqa: E402

tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 160
text, ns, ne = bench.coding_jsonl(tiles)
cfg = MiningConfig(tau=0.3)
mine_jsonl(text, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
mine_jsonl(text, cfg)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
mine_jsonl(text, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)

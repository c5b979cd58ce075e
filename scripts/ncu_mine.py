"""One warm columnar ingest+count launch on the C4 corpus (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count
from paper_2603_18897_b200.packing import SigTable
from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = {k: torch.from_numpy(v).cuda() for k, v in columnar_corpus(n).items()}
t = MineTables.allocate(SigTable(C4_TOOLS).n_sigs, 3, 0)
for _ in range(2):
    t.hist.zero_()
    ingest_count(t, dev)
t.expand()
t.select_sorted(5, 0.3)
torch.cuda.synchronize()

"""Event-timed columnar ingest+count launches on the C4 corpus (dev helper)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count
from paper_2603_18897_b200.packing import SigTable
from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
STAGED = len(sys.argv) <= 2 or sys.argv[2] != "single"
dev = {k: torch.from_numpy(v).cuda() for k, v in columnar_corpus(n).items()}
t = MineTables.allocate(SigTable(C4_TOOLS).n_sigs, 3, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
times = []
for i in range(12):
    flush.sum()
    t.hist.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(3_000_000)  # GPU busy while the host enqueues: events bracket the kernel only
    e0.record()
    ingest_count(t, dev, staged=STAGED)
    e1.record()
    e1.synchronize()
    times.append(e0.elapsed_time(e1))
times = sorted(times[2:])
print(f"ingest_count staged={STAGED} n={n}: median {times[len(times)//2]:.3f} ms  min {times[0]:.3f} ms  "
      f"-> {28 * n / times[len(times)//2] / 1e6:.0f} GB/s")

import sys, torch
sys.path.insert(0, ".")
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count
from paper_2603_18897_b200.packing import SigTable
from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus
n = 100_000_000
dev = {k: torch.from_numpy(v).cuda() for k, v in columnar_corpus(n).items()}
t = MineTables.allocate(32, 3, 0)
ingest_count(t, dev, staged=True)
torch.cuda.synchronize()
w = t._stage[:4 * n].view(torch.int32)
key = (w & 0x3fffffff).long()
cold = key[(w >= 0)]   # bit 31 clear
print("cold", cold.numel())
rnd = torch.randint(0, 1336336, (cold.numel(),), device="cuda")
perm = cold[torch.randperm(cold.numel(), device="cuda")]
def tm(name, x):
    for _ in range(2): torch.bincount(x, minlength=1336336)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): torch.bincount(x, minlength=1336336)
    e1.record(); e1.synchronize(); print(name, e0.elapsed_time(e1) / 5, "ms")
tm("cold keys (event order)", cold)
tm("cold keys (shuffled)", perm)
tm("uniform random", rnd)

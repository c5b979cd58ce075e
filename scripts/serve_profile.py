import sys, time, cProfile, pstats
import torch
sys.path.insert(0, ".")
import bench
from paper_2603_18897_b200.device_ops import DevicePool
from paper_2603_18897_b200.live import LiveSessionTable
from paper_2603_18897_b200.synth import LiveWorkload
class A: pool = "c3"
pool, policy, book = bench.load_setup(A)
dp = DevicePool(pool)
n = 1_000_000
wl = LiveWorkload(dp.sigs, dp.keys, n, seed=2603)
table = LiveSessionTable(dp, n, wl.tmpl.nodes, wl.max_batch_bytes, policy, book, max_candidates=8)
for _ in range(table.W + 2):
    table.step(wl.next_batch())
batches = [wl.next_batch() for _ in range(42)]
for b in batches:
    b.tok = torch.from_numpy(b.tok).pin_memory(); b.node = torch.from_numpy(b.node).pin_memory()
for _ in table.serve(batches[:2]): pass
torch.cuda.synchronize()
t = time.perf_counter()
for _ in table.serve(batches[2:]): pass
torch.cuda.synchronize()
print("wall per step ms", (time.perf_counter() - t) / 40 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in table.serve(batches[2:22]): pass
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)

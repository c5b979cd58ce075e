"""Per-stage timing of the C4 mining step (development helper)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2603_18897_b200.mine_engine import MineTables, ingest_count, patterns_from_candidates
from paper_2603_18897_b200.mining import MiningConfig
from paper_2603_18897_b200.packing import SigTable
from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
c = columnar_corpus(n)
dev = {k: torch.from_numpy(v).cuda() for k, v in c.items()}
cfg = MiningConfig(k=3, sigma=5, tau=0.3)
sigs = SigTable(C4_TOOLS)
t = MineTables.allocate(sigs.n_sigs, 3, 0)


def timed(name, fn, reps=3):
    for _ in range(1):
        out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    e1.synchronize()
    print(f"{name:22s} dev {e0.elapsed_time(e1) / reps:8.3f} ms  wall {(time.perf_counter() - w0) / reps * 1e3:8.3f} ms")
    return out


timed("hist zero", lambda: t.hist.zero_())
timed("ingest_count", lambda: (t.hist.zero_(), ingest_count(t, dev)))
timed("expand", lambda: t.expand())
cands = timed("select", lambda: t.select(cfg.sigma, cfg.tau))
print("candidates", len(cands), "nonzero bins", int((t.hist != 0).sum()))
timed("patterns (host)", lambda: patterns_from_candidates(cands, sigs, t.n_sigs, cfg))
tab = timed("select_sorted", lambda: t.select_sorted(cfg.sigma, cfg.tau))
print("sorted rows", len(tab))
timed("materialize", lambda: tab.patterns(sigs))
ref = patterns_from_candidates(cands, sigs, t.n_sigs, cfg)
print("sorted == host", tab.patterns(sigs) == ref)

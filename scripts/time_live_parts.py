"""Per-part timing of one C3 live step (development helper)."""
import sys
import time

import torch

sys.path.insert(0, ".")
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
for _ in range(table.W + 2):
    table.step(wl.next_batch())
comp = table.fetch_compact()
b = wl.next_batch()
tok = torch.from_numpy(b.tok).pin_memory()
node = torch.from_numpy(b.node).pin_memory()
pinned = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in table.cbuf.items()}
sizes = {"hdr": n, "pred": len(comp.pred), "arg": len(comp.arg), "act": len(comp.act)}
s = torch.cuda.current_stream()


def timed(name, fn, reps=10):
    fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    print(f"{name:28s} dev {e0.elapsed_time(e1) / reps:7.3f} ms  host {(time.perf_counter() - w0) / reps * 1e3:7.3f} ms")


timed("H2D tok+node (8 MB)", lambda: (table.new_tok.copy_(tok, non_blocking=True),
                                      table.new_node.copy_(node, non_blocking=True)))
timed("kernel (launch)", lambda: table.launch(table.steps % table.regions, new_node=table.new_node,
                                              new_tok=table.new_tok))
from paper_2603_18897_b200.live import _compact_init  # noqa: E402
import ctypes  # noqa: E402
from paper_2603_18897_b200._native import ptr  # noqa: E402
from paper_2603_18897_b200.device_ops import stream_handle  # noqa: E402
timed("compaction", lambda: table.lib.paste_compact_records(
    ctypes.byref(table.out_desc), table.n, ctypes.byref(table.pool_desc), ctypes.byref(table.cdesc),
    ptr(table.cscratch), stream_handle()))
timed("D2H sized (%.1f MB)" % (comp.nbytes / 1e6), lambda: [pinned[k][:m].copy_(table.cbuf[k][:m], non_blocking=True) for k, m in sizes.items()])
big = torch.empty(24_000_000, dtype=torch.uint8, device="cuda")
bigh = torch.empty(24_000_000, dtype=torch.uint8, pin_memory=True)
timed("D2H one 24 MB copy", lambda: bigh.copy_(big, non_blocking=True))
timed("H2D one 24 MB copy", lambda: big.copy_(bigh, non_blocking=True))
timed("fetch_compact (full)", lambda: table.fetch_compact(pinned), reps=5)
batches = [wl.next_batch() for _ in range(42)]
for bb in batches:
    bb.tok = torch.from_numpy(bb.tok).pin_memory()
    bb.node = torch.from_numpy(bb.node).pin_memory()
for depth, fused in ((3, True), (4, True), (6, True), (3, False)):
    table.serve_fused = fused
    for _ in table.serve(batches[:2], depth=depth):
        pass
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cnt = 0
    for r in table.serve(batches[2:], depth=depth):
        cnt += 1
    e1.record()
    e1.synchronize()
    print(f"serve depth {depth} fused={fused}: {e0.elapsed_time(e1) / cnt:.3f} ms/step over {cnt} steps")

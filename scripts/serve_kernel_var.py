"""Device time of the serving step's kernels alone (development helper):
paste_predict_live_compact on fixed inputs, back to back, with and without
concurrent PCIe copies of the serving sizes on other streams."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
batches = [wl.next_batch().narrowed(table.codes, table.ecodes).pin() for _ in range(8)]
for _ in table.serve(batches[:6]):
    pass
torch.cuda.synchronize()
sv = table._serve
# the window descriptor and buffers of set 0 as serve() left them
key = next(k for k in sv["wins"] if k[0] == 0)
win = sv["wins"][key]
lib = table.lib
comp = torch.cuda.current_stream()


def launch():
    rc = lib.paste_predict_live_compact(ctypes.byref(table.pool_desc), ctypes.byref(win),
                                        ctypes.byref(table.adm), ctypes.byref(table.plan),
                                        table.B, ctypes.byref(sv["descs"][0]),
                                        sv["scratch"][0].data_ptr(), sv["scratch"][0].numel(),
                                        comp.cuda_stream)
    assert rc == 0, rc


def timed(reps=50, copies=False, up=True, down=True):
    up_h = torch.empty(1_000_000, dtype=torch.uint8, pin_memory=True)
    up_d = torch.empty(1_000_000, dtype=torch.uint8, device="cuda")
    dn_h = torch.empty(2_500_000, dtype=torch.uint8, pin_memory=True)
    dn_d = torch.empty(2_500_000, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ts = []
    for _ in range(reps):
        if copies and up:
            with torch.cuda.stream(s1):
                up_d.copy_(up_h, non_blocking=True)
        if copies and down:
            with torch.cuda.stream(s2):
                dn_h.copy_(dn_d, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        launch()
        e1.record(comp)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    torch.cuda.synchronize()
    ts = np.array(ts[5:])
    return f"p50 {np.median(ts):.1f} p90 {np.percentile(ts, 90):.1f} max {ts.max():.1f} us"


print("kernels alone      ", timed())
print("with PCIe copies   ", timed(copies=True))
print("with H2D only      ", timed(copies=True, down=False))
print("with D2H only      ", timed(copies=True, up=False))
print("kernels alone again", timed())
# queue pre-filled: host submission out of the timed path
torch.cuda._sleep(5_000_000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(comp)
for _ in range(40):
    launch()
e1.record(comp)
e1.synchronize()
print(f"40 back to back (queued)  {e0.elapsed_time(e1) / 40 * 1e3:.1f} us each")


def queued_with_copies(up=True, down=True, reps=40):
    """40 kernels back to back on the compute stream while 40 uploads / 40
    downloads of the serving sizes run on two other streams, all queued
    behind a sleep so host submission is out of the timed path."""
    up_h = torch.empty(1_000_000, dtype=torch.uint8, pin_memory=True)
    up_d = torch.empty(1_000_000, dtype=torch.uint8, device="cuda")
    dn_h = torch.empty(2_500_000, dtype=torch.uint8, pin_memory=True)
    dn_d = torch.empty(2_500_000, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    gate = torch.cuda.Event()
    torch.cuda._sleep(5_000_000)
    gate.record(comp)
    s1.wait_event(gate)
    s2.wait_event(gate)
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s1):
                up_d.copy_(up_h, non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                dn_h.copy_(dn_d, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(reps):
        launch()
    e1.record(comp)
    torch.cuda.synchronize()
    return f"{e0.elapsed_time(e1) / reps * 1e3:.1f} us each"


print("queued, with both copies   ", queued_with_copies())
print("queued, with H2D copies    ", queued_with_copies(down=False))
print("queued, with D2H copies    ", queued_with_copies(up=False))

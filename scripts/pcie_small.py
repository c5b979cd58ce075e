"""PCIe copy rates at the serving step's sizes (development helper): H2D of
3 MB and D2H of 3.2 MB, alone and concurrently, as one copy or split into
the serving loop's pieces, timed over back-to-back repetitions with CUDA
events on each copy stream."""
import torch

MB = 1_000_000


def bufs(sizes):
    return ([torch.empty(s, dtype=torch.uint8, pin_memory=True) for s in sizes],
            [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes])


up_h, up_d = bufs([3 * MB])
up2_h, up2_d = bufs([1 * MB, 2 * MB])
dn_h, dn_d = bufs([3_200_000])
dn3_h, dn3_d = bufs([40, 2 * MB, 1_200_000])
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=200):
    for _ in range(3):
        step(h2d, d2h)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(s1)
    e[2].record(s2)
    for _ in range(reps):
        step(h2d, d2h)
    e[1].record(s1)
    e[3].record(s2)
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps * 1e3, e[2].elapsed_time(e[3]) / reps * 1e3


def step(h2d, d2h):
    if h2d:
        with torch.cuda.stream(s1):
            for d, h in zip(*h2d[::-1]):
                d.copy_(h, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            for h, d in zip(*d2h):
                h.copy_(d, non_blocking=True)


for name, a, b in (("H2D 3 MB x1", (up_h, up_d), None), ("H2D 1+2 MB", (up2_h, up2_d), None),
                   ("D2H 3.2 MB x1", None, (dn_h, dn_d)), ("D2H 40B+2+1.2 MB", None, (dn3_h, dn3_d)),
                   ("both x1", (up_h, up_d), (dn_h, dn_d)),
                   ("both split", (up2_h, up2_d), (dn3_h, dn3_d))):
    u, d = run(a, b)
    print(f"{name:20s} up-stream {u:7.1f} us  down-stream {d:7.1f} us")

# the same copies while a memory-bound kernel stream runs beside them
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s3 = torch.cuda.Stream()


def busy(reps):
    with torch.cuda.stream(s3):
        for _ in range(reps):
            big.add_(1)


torch.cuda.synchronize()
busy(400)
u, d = run((up_h, up_d), (dn_h, dn_d), reps=100)
print(f"{'both x1 + kernel':20s} up-stream {u:7.1f} us  down-stream {d:7.1f} us")
torch.cuda.synchronize()
up2m_h, up2m_d = bufs([2 * MB])
dn35_h, dn35_d = bufs([3_500_000])
u, d = run((up2m_h, up2m_d), (dn35_h, dn35_d))
print(f"{'up 2 MB, down 3.5 MB':20s} up-stream {u:7.1f} us  down-stream {d:7.1f} us")

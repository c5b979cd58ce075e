import torch, time
n = 24_000_000
a_h = torch.empty(n, dtype=torch.uint8, pin_memory=True); a_d = torch.empty(n, dtype=torch.uint8, device="cuda")
b_h = torch.empty(n, dtype=torch.uint8, pin_memory=True); b_d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    a_d.copy_(a_h, non_blocking=True); b_h.copy_(b_d, non_blocking=True)
torch.cuda.synchronize()
def run(h2d, d2h, reps=20):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): a_d.copy_(a_h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): b_h.copy_(b_d, non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e3
print("h2d only %.3f ms, d2h only %.3f ms, both %.3f ms" % (run(1,0), run(0,1), run(1,1)))

"""Host<->device copy bandwidth on the box: H2D alone, D2H alone, both at once (pinned buffers)."""
import torch, time
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n // 3, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n // 3, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / reps
    return dt
for h2d, d2h in ((1, 0), (0, 1), (1, 1)):
    run(h2d, d2h, 1); dt = run(h2d, d2h)
    print(f"h2d={h2d} d2h={d2h}: {dt*1e3:.1f} ms  H2D {n/dt/1e9 if h2d else 0:.1f} GB/s  D2H {(n//3)/dt/1e9 if d2h else 0:.1f} GB/s")

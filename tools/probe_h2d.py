"""Host-link probe: pinned H2D / D2H bandwidth for one and two concurrent copies
(the e2e leg's 480 MB-in / 160 MB-out per 20 M MS step)."""
import torch
N = 480 * 2**20 // 8
h = torch.empty(N, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(N // 3, dtype=torch.float64, pin_memory=True)
d = torch.empty(N, dtype=torch.float64, device="cuda")
d2 = torch.empty(N // 3, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=10):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def one():
    d.copy_(h, non_blocking=True)
def two():
    half = N // 2
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
def duplex():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
def d2h():
    h2.copy_(d2, non_blocking=True)
for name, f, b in (("h2d 1 copy", one, N * 8), ("h2d 2 streams", two, N * 8), ("d2h", d2h, N // 3 * 8),
                   ("h2d 480MB + d2h 160MB concurrent", duplex, N * 8)):
    ms = t(f)
    print(f"{name}: {ms:.3f} ms, {b / ms / 1e6:.1f} GB/s (H2D bytes)")

"""Experiment: host<->device copy bandwidth of 64 MiB pinned buffers, alone and both
directions at once (the e2e leg's ceiling)."""
import torch
n = 64 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    ev = torch.cuda.Event(); ev.record()
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    e = torch.cuda.Event(); e.record(s1); torch.cuda.current_stream().wait_event(e)
    e = torch.cuda.Event(); e.record(s2); torch.cuda.current_stream().wait_event(e)
bi = t(both)
print("H2D %.1f GB/s  D2H %.1f GB/s  both %.1f GB/s each" % (n / h2d / 1e6, n / d2h / 1e6, n / bi / 1e6))

"""Pinned host<->device copy bandwidth on the GPU box (diagnostics)."""
import torch
n = 1 << 26
h = torch.empty(n, dtype=torch.int32).pin_memory()
h2 = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device='cuda')
d2 = torch.empty(n, dtype=torch.int32, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
mb = n * 4 / 1e9
print('H2D GB/s %.1f' % (mb / (t(lambda: d.copy_(h, non_blocking=True)) / 1e3)))
print('D2H GB/s %.1f' % (mb / (t(lambda: h.copy_(d, non_blocking=True)) / 1e3)))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
print('H2D+D2H concurrent aggregate GB/s %.1f' % (2 * mb / (t(both) / 1e3)))

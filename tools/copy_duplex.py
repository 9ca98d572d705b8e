"""Pinned H2D and D2H copies of the e2e workload's sizes, alone and
concurrently on two streams: the PCIe bound of bench.py's e2e step.
usage: python tools/copy_duplex.py"""
import torch
dev = torch.device('cuda', 0)
n = 1 << 24
h_in = torch.empty(n, dtype=torch.int32).pin_memory()
h_out = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
d_in = torch.empty(n, dtype=torch.int32, device=dev)
d_out = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                for j in range(2):
                    h_out[j].copy_(d_out[j], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


run(True, True, 3)
for name, h, d in (("H2D 64 MB", True, False), ("D2H 128 MB", False, True), ("both", True, True)):
    print("%-12s %.3f ms per step" % (name, run(h, d)))

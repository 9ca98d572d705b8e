"""Pinned H2D and D2H copies of the e2e workload's sizes, alone and
concurrently on two streams: the PCIe bound of bench.py's e2e step.
usage: python tools/copy_duplex.py [log2 n]   (24: cfg2, 31: cfg5)"""
import sys

import torch
dev = torch.device('cuda', 0)
n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 24)
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


reps = 20 if n <= (1 << 26) else 3
run(True, True, 1)
for name, h, d in (("H2D %d MB" % (4 * n >> 20), True, False), ("D2H %d MB" % (8 * n >> 20), False, True),
                   ("both", True, True)):
    ms = run(h, d, reps)
    print("%-12s %.3f ms per step (%.1f GB/s H2D, %.1f GB/s D2H)" % (
        name, ms, 4 * n / ms / 1e6 if h else 0, 8 * n / ms / 1e6 if d else 0), flush=True)

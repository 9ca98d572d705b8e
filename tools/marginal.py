"""Median time of one sort (CUDA events, L2 flushed, input restored outside
the timed interval).  With PS_DEBUG_STAGES=s only the first s merge stages
run, so a sweep over s gives each stage's marginal cost under PDL overlap.
usage: PS_DEBUG_STAGES=s python tools/marginal.py [cfg2]"""
import os, sys
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor

name = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
dev = torch.device('cuda', 0)
src = torch.from_numpy(workloads.generate(name)).to(dev)
keys = torch.empty_like(src)
perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ts = []
for it in range(25):
    keys.copy_(src)
    flush.fill_(it & 255)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _sort_tensor(keys, perm, SortConfig(), _lib.VALUES_ARGSORT, collect_runs=False)
    b.record()
    torch.cuda.synchronize()
    if it >= 5:
        ts.append(a.elapsed_time(b))
ts.sort()
print('%s stages=%s median %.1f us  min %.1f us' % (name, os.environ.get('PS_DEBUG_STAGES', 'all'),
                                                   1e3 * ts[len(ts) // 2], 1e3 * ts[0]))

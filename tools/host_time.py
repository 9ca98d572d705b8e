"""Host time spent inside one ps_sort call vs the device time of the same sort
(is the host's launch rate the bottleneck?).  PS_DEBUG_STAGES limits the phases.
usage: PS_DEBUG_STAGES=-2 python tools/host_time.py cfg2"""
import os, sys, time
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor

name = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
dev = torch.device('cuda', 0)
COUNT = os.environ.get("PS_COUNT", "1") == "1"
src = torch.from_numpy(workloads.generate(name)).to(dev)
keys = torch.empty_like(src)
perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
hs, ds = [], []
for it in range(25):
    keys.copy_(src)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    _sort_tensor(keys, perm, SortConfig(count_comparisons=COUNT), _lib.VALUES_ARGSORT, collect_runs=False,
                 asynchronous=True)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    if it >= 5:
        hs.append((t1 - t0) * 1e6)
        ds.append(a.elapsed_time(b) * 1e3)
hs.sort(); ds.sort()
print('%s count=%d stages=%s host %.1f us  device %.1f us  launches/sort %s' % (
    name, COUNT, os.environ.get('PS_DEBUG_STAGES', 'all'), hs[len(hs) // 2], ds[len(ds) // 2], _lib.launch_count() if hasattr(_lib, 'launch_count') else '?'))

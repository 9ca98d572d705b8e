"""Per-stage CUDA-event profile of one sort (diagnostics; run on the GPU box).
usage: python tools/stage_profile.py [cfg2] [n] [nocount]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor

name = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
count = not (len(sys.argv) > 3 and sys.argv[3] == "nocount")
keys_np = workloads.generate(name, n=n)
dev = torch.device('cuda', 0)
src = torch.from_numpy(keys_np).to(dev)
keys = torch.empty_like(src)
perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
lib = _lib.load()
for it in range(3):
    keys.copy_(src)
    torch.cuda.synchronize()
    lib.ps_profile_enable(1)
    _sort_tensor(keys, perm, SortConfig(count_comparisons=count), _lib.VALUES_ARGSORT, collect_runs=False)
    lib.ps_profile_enable(0)
prof = _lib.profile_read()
tot = 0
for e in prof:
    gbs = e['bytes'] / (e['ms'] * 1e6) if e['ms'] > 0 else 0
    tot += e['ms']
    print('%-15s stage %3d nodes %8d chunks %8d  %8.3f ms  %9.1f MB  %7.0f GB/s' % (
        e['kind'], e['stage'], e['nodes'], e['chunks'], e['ms'], e['bytes'] / 1e6, gbs))
print('sum of entries %.3f ms' % tot)
import numpy as np
ok = np.array_equal(perm.cpu().numpy(), np.argsort(keys_np, kind='stable'))
print('parity vs numpy stable argsort:', 'OK' if ok else 'MISMATCH')

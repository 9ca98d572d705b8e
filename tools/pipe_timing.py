"""Phase cycle counters of merge_pipe_kernel (needs the PS_PIPE_TIMING build:
   nvcc ... -DPS_PIPE_TIMING -o /tmp/libps_timing.so; PS_LIB=/tmp/libps_timing.so python tools/pipe_timing.py cfg2)"""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor
name = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
lib = _lib.load()
lib.ps_debug_pipe_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
keys_np = workloads.generate(name)
dev = torch.device('cuda', 0)
src = torch.from_numpy(keys_np).to(dev)
keys = torch.empty_like(src)
perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
buf = np.zeros(40, dtype=np.uint64)
for it in range(2):
    keys.copy_(src)
    lib.ps_debug_pipe_timing(buf.ctypes.data, 1)
    _sort_tensor(keys, perm, SortConfig(), _lib.VALUES_ARGSORT, collect_runs=False)
    lib.ps_debug_pipe_timing(buf.ctypes.data, 1)
names = ['P.batch', 'P.wait_empty', 'P.stage', 'P.units', 'C.wait_full', 'C.pass1', 'C.pass2', 'C.store', 'C.units']
pu, cu = max(int(buf[3]), 1), max(int(buf[8]), 1)
for i, nm in enumerate(names):
    v = int(buf[i])
    per = v / (pu if nm.startswith('P') else cu)
    print('%-14s total %14d   per unit %10.1f cycles' % (nm, v, per))
print('per-warp pass1 work (cycles/unit, to the barrier):', ' '.join('%6.0f' % (int(buf[16 + w]) / cu) for w in range(8)))
print('per-warp pass2 work (cycles/unit, since unit start):', ' '.join('%6.0f' % (int(buf[24 + w]) / cu) for w in range(8)))
# per-CTA stamps of the last pipe launch of the sort (the root merge)
cta = np.zeros((1024, 5), dtype=np.uint64)
lib.ps_debug_cta_timing.argtypes = [ctypes.c_void_p]
lib.ps_debug_cta_timing(cta.ctypes.data)
g = int(np.count_nonzero(cta[:, 0]))
c = cta[:g].astype(np.int64)
t0 = c[:, 0].min()
print('last launch: %d CTAs; us from the first CTA start:' % g)
for j, nm in enumerate(['start', 'after partition', 'first unit ready', 'consumers done', 'producer done']):
    v = (c[:, j] - t0) / 1e3
    print('  %-18s min %7.2f  median %7.2f  max %7.2f' % (nm, v.min(), np.median(v), v.max()))

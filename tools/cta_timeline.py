"""Per-CTA timeline of the last merge_pipe_kernel launch (PS_PIPE_TIMING build):
start, after partition, first unit ready, consumers done, producer done (globaltimer ns).
usage: nvcc ... -DPS_PIPE_TIMING -o /tmp/libps_timing.so;
       PS_LIB=/tmp/libps_timing.so PS_DEBUG_STAGES=s python tools/cta_timeline.py cfg2"""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor
name = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
lib = _lib.load()
lib.ps_debug_cta_timing.argtypes = [ctypes.c_void_p]
keys_np = workloads.generate(name)
dev = torch.device('cuda', 0)
src = torch.from_numpy(keys_np).to(dev)
keys = torch.empty_like(src)
perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
for it in range(3):
    keys.copy_(src)
    _sort_tensor(keys, perm, SortConfig(), _lib.VALUES_ARGSORT, collect_runs=False)
    torch.cuda.synchronize()
buf = np.zeros((1024, 5), dtype=np.uint64)
lib.ps_debug_cta_timing(buf.ctypes.data)
b = buf[buf[:, 0] > 0].astype(np.float64)
t0 = b[:, 0].min()
b = (b - t0) / 1e3  # us
for i, nm in enumerate(['start', 'partition done', 'first unit ready', 'consumers done', 'producer done']):
    col = b[:, i]
    print('%-18s min %7.1f  median %7.1f  max %7.1f us' % (nm, col.min(), np.median(col), col.max()))
print('CTAs', len(b))

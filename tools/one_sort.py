"""One warm sort of a workload (for ncu captures of a single stage's kernels).
usage: python tools/one_sort.py [cfg2]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2209_06909_b200 import SortConfig, _lib, workloads
from paper_2209_06909_b200.policy import _sort_tensor

keys_np = workloads.generate(sys.argv[1] if len(sys.argv) > 1 else 'cfg2')
dev = torch.device('cuda', 0)
keys = torch.from_numpy(keys_np).to(dev)
perm = torch.empty(keys.numel(), dtype=torch.int32, device=dev)
_sort_tensor(keys, perm, SortConfig(), _lib.VALUES_ARGSORT, collect_runs=False)
torch.cuda.synchronize()

"""One asynchronous sort of a config (for ncu captures); prints the index of
the merge_pipe_kernel launch of the biggest merge stage.
usage: python tools/one_sort.py cfg5 [--pick]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import SortConfig, _lib, workloads  # noqa: E402
from paper_2209_06909_b200.policy import _sort_tensor, check  # noqa: E402

name = sys.argv[1]
dev = torch.device("cuda", 0)
x = workloads.generate(name, seed=0)
keys = torch.from_numpy(x).to(dev)
perm = torch.empty(keys.numel(), dtype=torch.int32, device=dev)
lib = _lib.load()
if "--pick" in sys.argv:
    lib.ps_profile_enable(1)
_sort_tensor(keys, perm, SortConfig(), _lib.VALUES_ARGSORT, collect_runs=False, asynchronous=True)
check(dev)
if "--pick" in sys.argv:
    prof = _lib.profile_read()
    pipe = [e for e in prof if e["kind"] == "merge" and e["chunks"] > 0]
    best = max(range(len(pipe)), key=lambda i: pipe[i]["bytes"])
    for i, e in enumerate(pipe):
        print("pipe launch %d: stage %d nodes %d chunks %d %.1f MB %.3f ms" % (
            i, e["stage"], e["nodes"], e["chunks"], e["bytes"] / 1e6, e["ms"]), file=sys.stderr)
    print(best)

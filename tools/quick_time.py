"""Median device time of one sort per config, with and without the
CountingOrder counters (count_comparisons), and the phase split.
usage: python tools/quick_time.py cfg2 cfg4 cfg5 ..."""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import SortConfig, _lib, workloads  # noqa: E402
from paper_2209_06909_b200.policy import _sort_tensor, check  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
for name in sys.argv[1:]:
    x = workloads.generate(name, seed=0)
    src = torch.from_numpy(x).to(dev)
    keys = torch.empty_like(src)
    perm = torch.empty(src.numel(), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for count in (False, True):
        cfg = SortConfig(count_comparisons=count)
        ts = []
        for i in range(12):
            keys.copy_(src)
            flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _sort_tensor(keys, perm, cfg, _lib.VALUES_ARGSORT, collect_runs=False, asynchronous=True)
            b.record()
            check(dev)
            if i >= 2:
                ts.append(a.elapsed_time(b))
        lib.ps_profile_enable(1)
        keys.copy_(src)
        _sort_tensor(keys, perm, cfg, _lib.VALUES_ARGSORT, collect_runs=False, asynchronous=True)
        ph = _lib.profile_read()
        lib.ps_profile_enable(0)
        agg = {}
        for e in ph:
            agg[e["kind"]] = agg.get(e["kind"], 0.0) + e["ms"]
        print("%s count=%d median %.3f ms  %s" % (name, count, statistics.median(ts),
              " ".join("%s=%.3f" % kv for kv in agg.items())), flush=True)
    del src, keys, perm, flush
    torch.cuda.empty_cache()

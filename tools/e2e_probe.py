"""Where does the cfg5 e2e step go?  The bench's pipelined H2D / sort / D2H
ring (bench.run_e2e) in variants: copies only, synchronous sorts (the bench),
asynchronous sorts, and more steps.  usage: python tools/e2e_probe.py [log2 n] [steps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import SortConfig, _lib, stable_argsort, workloads  # noqa: E402
from paper_2209_06909_b200.policy import _sort_tensor, check, finish_counters  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 31
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
keys_np = workloads.generate("cfg5", n=1 << lg, seed=0)
n = keys_np.shape[0]
NB = 3
h_in = [torch.from_numpy(keys_np).pin_memory() for _ in range(NB)]
h_out = [torch.empty_like(h_in[0]).pin_memory() for _ in range(NB)]
h_perm = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(NB)]
d_in = [torch.empty(n, dtype=h_in[0].dtype, device=dev) for _ in range(NB)]
d_perm = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(NB)]
s_h2d, s_cmp, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
cfg = SortConfig()


def pipeline(K, mode):
    ev_h2d, d2h_done = {}, {}
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s_h2d)

    def h2d(i):
        b = i % NB
        if b in d2h_done:
            s_h2d.wait_event(d2h_done[b])
        with torch.cuda.stream(s_h2d):
            d_in[b].copy_(h_in[b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_h2d)
        ev_h2d[i] = e

    h2d(0)
    for i in range(K):
        if i + 1 < K:
            h2d(i + 1)
        b = i % NB
        s_cmp.wait_event(ev_h2d[i])
        with torch.cuda.stream(s_cmp):
            if mode == "sync":
                _, p, _ = stable_argsort(d_in[b], cfg, collect_runs=False)
            elif mode in ("async", "async+finish"):
                p = d_perm[b]
                st = _sort_tensor(d_in[b], p, cfg, _lib.VALUES_ARGSORT, collect_runs=False, asynchronous=True)
            else:
                p = d_perm[b]
            done = torch.cuda.Event()
            done.record(s_cmp)
        s_d2h.wait_event(done)
        with torch.cuda.stream(s_d2h):
            h_out[b].copy_(d_in[b], non_blocking=True)
            h_perm[b].copy_(p, non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_d2h)
        d2h_done[b] = e
        if mode == "async+finish":
            with torch.cuda.stream(s_cmp):
                finish_counters(st)  # the step's SortStats, after its D2H is queued
    t1.record(s_d2h)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1)


pipeline(2, "copies")
for mode in ("copies", "sync", "async", "async+finish"):
    ms = pipeline(K, mode)
    print("%-7s K=%d: %.1f ms per step" % (mode, K, ms / K), flush=True)

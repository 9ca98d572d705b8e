"""Stress of concurrent sorts whose merge stages are mostly fused-partition
(cooperative, grid-barrier) pipe launches: small inputs, several host threads.
usage: python tools/stress_fused.py [threads] [reps]"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import SortConfig, stable_argsort, workloads  # noqa: E402

nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
dev = torch.device("cuda", 0)
inputs = [workloads.generate("cfg2", n=1 << 19, seed=1), workloads.generate("cfg5", n=1 << 20, seed=2),
          workloads.generate("cfg3", n=1 << 19, seed=3), workloads.generate("cfg2", n=1 << 21, seed=4)]
refs = [np.argsort(x, kind="stable").astype(np.int32) for x in inputs]
errors, slow = [], []


def worker(idx):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        dkeys = [torch.from_numpy(x).to(dev) for x in inputs]
        for rep in range(reps):
            q = (idx + rep) % len(inputs)
            try:
                t0 = time.perf_counter()
                out, perm, _ = stable_argsort(dkeys[q].clone(), SortConfig())
                s.synchronize()
                dt = time.perf_counter() - t0
                if dt > 0.3:
                    slow.append((idx, rep, q, round(dt, 3)))
                if rep % 10 == 0 and int(np.count_nonzero(perm.cpu().numpy() != refs[q])):
                    errors.append((idx, rep, q, "mismatch"))
            except Exception as e:  # noqa: BLE001
                errors.append((idx, rep, q, repr(e)[:300]))


ts = [threading.Thread(target=worker, args=(i,)) for i in range(nthr)]
t0 = time.perf_counter()
for t in ts:
    t.start()
for t in ts:
    t.join()
print("threads", nthr, "reps", reps, "errors", len(errors), "slow (>0.3 s)", len(slow), "wall %.1f s" % (time.perf_counter() - t0))
for e in (errors + slow)[:10]:
    print(e)

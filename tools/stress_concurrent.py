"""Stress of concurrent sorts on several host threads / streams (the scenario of
tests/test_gpu_parity.py::test_concurrent_sorts_on_two_streams, more repeats).
usage: python tools/stress_concurrent.py [threads] [reps]"""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import SortConfig, stable_argsort, workloads  # noqa: E402

nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
dev = torch.device("cuda", 0)
inputs = [workloads.generate("cfg2", n=1 << 22, seed=41), workloads.generate("cfg3", n=1 << 21, seed=42),
          workloads.generate("cfg5", n=1 << 22, seed=43), workloads.generate("cfg1", n=1 << 20, seed=44)]
refs = [np.argsort(x, kind="stable").astype(np.int32) for x in inputs]  # the stable order is unique
errors = []


def worker(idx):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for rep in range(reps):
            q = (idx + 2 * rep + rep // 7) % len(inputs)
            try:
                keys = torch.from_numpy(inputs[q]).to(dev)
                out, perm, _ = stable_argsort(keys, SortConfig())
                s.synchronize()
                bad = int(np.count_nonzero(perm.cpu().numpy() != refs[q]))
                if bad:
                    errors.append((idx, rep, q, "mismatches", bad))
            except Exception as e:  # noqa: BLE001
                errors.append((idx, rep, q, repr(e)[:300]))


ts = [threading.Thread(target=worker, args=(i,)) for i in range(nthr)]
for t in ts:
    t.start()
for t in ts:
    t.join()
print("threads", nthr, "reps", reps, "errors", len(errors))
for e in errors[:10]:
    print(e)

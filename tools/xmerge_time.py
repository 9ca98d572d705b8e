"""Device time of the single-pass cross-shard merge (ps_shard_merge) with G
shards emulated on one GPU (local pointers instead of peer mappings): slab g
of N = G * shard keys, float32 keys uniform in [-1e6, 1e6], sorted shards.
usage: python tools/xmerge_time.py [shard_len] [G ...]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2209_06909_b200 import multigpu  # noqa: E402

dev = torch.device("cuda", 0)
shard = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
Gs = [int(x) for x in sys.argv[2:]] or [2, 4, 8]
g = torch.Generator(device=dev)
g.manual_seed(0)
for G in Gs:
    sk, sv = [], []
    for h in range(G):
        k = (torch.rand(shard, device=dev, generator=g) * 2e6 - 1e6).sort().values
        sk.append(k)
        sv.append(torch.arange(h * shard, (h + 1) * shard, dtype=torch.int32, device=dev))
    smp = [multigpu.shard_samples(k) for k in sk]
    N = G * shard
    t0, t1 = multigpu.slab_bounds(N, G, G // 2)
    out_k = torch.empty(t1 - t0, dtype=torch.float32, device=dev)
    out_v = torch.empty(t1 - t0, dtype=torch.int32, device=dev)
    ws = None
    ts = []
    for i in range(6):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        multigpu.shard_merge(sk, sv, t0, t1, out_k, out_v, samples=smp, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    byts = (t1 - t0) * 8 * 2
    ok = bool((out_k[1:] >= out_k[:-1]).all())
    print("G=%d slab=%d keys: %.3f ms, %.1f GB/s (slab bytes read + written), sorted=%s" % (
        G, t1 - t0, ms, byts / ms / 1e6, ok), flush=True)
    del sk, sv, smp, out_k, out_v
    torch.cuda.empty_cache()

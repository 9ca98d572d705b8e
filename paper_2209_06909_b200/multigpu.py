"""Multi-GPU sorting: shard, sort locally, cross-shard merge.

One process per GPU.  Every rank holds a contiguous shard of the global input
(shard g = global indices [off_g, off_g + n_g)).  The sort runs in two steps.

1. Each rank sorts its shard with the single-GPU hot path.  The payload is
   the global index, so stability is carried across shards.  The shard is
   its own array: its run powers use the shard length, so its merge tree
   differs from the 1-GPU tree.  Tree parity is defined at G = 1 only.
2. ``ps_shard_merge`` produces this rank's slab of the global stable order,
   ranks [g*N/G, (g+1)*N/G).  It finds the slab's co-ranks in all G sorted
   shards and reads the peer shards directly over NVLink (CUDA IPC mappings,
   peer loads in the gather kernel).  It then merges the G windows locally.

``torch.distributed`` is used only as plumbing: sizes and IPC handles are
exchanged as Python objects, plus barriers.  No collective touches the key
data, and there is no NCCL on the data path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .policy import SortConfig, _dtype_id, _sort_tensor


def slab_bounds(total, world, rank):
    """Global rank range [t0, t1) of ``rank``'s output slab."""
    return (total * rank) // world, (total * (rank + 1)) // world


def plan(sizes, rank):
    """Host plan for one rank: shard offsets, global size and slab bounds."""
    sizes = [int(s) for s in sizes]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64).tolist()
    total = offs[-1]
    t0, t1 = slab_bounds(total, len(sizes), rank)
    return {"sizes": sizes, "offsets": offs[:-1], "total": total, "slab": (t0, t1)}


def shard_merge(shard_keys, shard_vals, t0, t1, out_keys=None, out_vals=None):
    """Slab [t0, t1) of the stable merge of the sorted shards (all tensors
    addressable from the current device: local or peer-mapped)."""
    import torch

    lib = _lib.load()
    G = len(shard_keys)
    if G != len(shard_vals) or not 1 <= G <= 8:
        raise ValueError("need 1..8 shards with matching value arrays")
    dt = _dtype_id(shard_keys[0])
    dev = torch.device("cuda", torch.cuda.current_device())
    n = t1 - t0
    if out_keys is None:
        out_keys = torch.empty(n, dtype=shard_keys[0].dtype, device=dev)
    if out_vals is None:
        out_vals = torch.empty(n, dtype=torch.int32, device=dev)
    kp = (ctypes.c_void_p * G)(*[k.data_ptr() for k in shard_keys])
    vp = (ctypes.c_void_p * G)(*[v.data_ptr() for v in shard_vals])
    ns = (ctypes.c_int64 * G)(*[k.numel() for k in shard_keys])
    nbytes = lib.ps_shard_merge_workspace_size(G, n)
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.ps_shard_merge(dt, G, kp, vp, ns, t0, t1, out_keys.data_ptr(), out_vals.data_ptr(),
                                  ws.data_ptr(), ws.numel(), stream))
    return out_keys, out_vals


def sort_distributed(keys, config=None, group=None):
    """Sort a globally sharded array: ``keys`` is this rank's contiguous shard
    (CUDA tensor).  Returns (slab_keys, slab_global_indices) of this rank's
    slab of the global stable order."""
    import torch
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    if config is None:
        config = SortConfig()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sizes = [None] * world
    if world > 1:
        dist.all_gather_object(sizes, int(keys.numel()), group=group)
    else:
        sizes = [int(keys.numel())]
    p = plan(sizes, rank)
    off = p["offsets"][rank]
    vals = torch.arange(off, off + keys.numel(), dtype=torch.int32, device=keys.device)
    _sort_tensor(keys, vals, config, _lib.VALUES_PERMUTE, collect_runs=False)
    if world == 1:
        return keys, vals
    torch.cuda.synchronize(keys.device)
    handles = [None] * world
    dist.all_gather_object(handles, (reduce_tensor(keys), reduce_tensor(vals)), group=group)
    peers_k, peers_v = [], []
    for g, ((fk, ak), (fv, av)) in enumerate(handles):
        if g == rank:
            peers_k.append(keys)
            peers_v.append(vals)
        else:
            peers_k.append(fk(*ak))
            peers_v.append(fv(*av))
    t0, t1 = p["slab"]
    out = shard_merge(peers_k, peers_v, t0, t1)
    torch.cuda.synchronize(keys.device)
    dist.barrier(group=group)  # peers keep their shards alive until every slab is merged
    del peers_k, peers_v
    return out

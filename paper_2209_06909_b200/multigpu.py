"""Multi-GPU sorting: shard, sort locally, cross-shard merge.

One process per GPU.  Every rank holds a contiguous shard of the global input
(shard g = global indices [off_g, off_g + n_g)).  The sort runs in two steps.

1. Each rank sorts its shard with the single-GPU hot path.  The payload is
   the global index, so stability is carried across shards.  The shard is
   its own array: its run powers use the shard length, so its merge tree
   differs from the 1-GPU tree.  Tree parity is defined at G = 1 only.
2. ``ps_shard_merge`` produces this rank's slab of the global stable order,
   ranks [g*N/G, (g+1)*N/G), in one pass: it finds the slab's co-ranks in
   all G sorted shards and loads the peer shards' windows directly over
   NVLink (CUDA IPC mappings opened in this device's context with lazy peer
   access, ``ps_ipc_open``) into the merge kernel's shared memory.

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


def shard_samples(keys, out=None):
    """Sample array of a sorted shard (every 128 bytes of keys), the input
    ps_shard_merge uses to cut the slab without peer searches."""
    import torch

    lib = _lib.load()
    dt = _dtype_id(keys)
    ns = int(lib.ps_shard_sample_count(dt, keys.numel()))
    if out is None:
        out = torch.empty(max(ns, 1), dtype=keys.dtype, device=keys.device)
    stream = torch.cuda.current_stream(keys.device).cuda_stream
    _lib.check(lib.ps_shard_samples(dt, keys.data_ptr(), keys.numel(), out.data_ptr(), stream))
    return out


def shard_merge(shard_keys, shard_vals, t0, t1, out_keys=None, out_vals=None, samples=None, workspace=None):
    """Slab [t0, t1) of the stable merge of the sorted shards (all tensors
    addressable from the current device: local or peer-mapped).  ``samples``
    are the shards' sample arrays (shard_samples) or None."""
    import torch

    G = len(shard_keys)
    if G != len(shard_vals) or not 1 <= G <= 8:
        raise ValueError("need 1..8 shards with matching value arrays")
    sp = None if samples is None else [
        (s.data_ptr() if s is not None and s.numel() else None) for s in samples]
    return _shard_merge_ptrs(shard_keys[0].dtype, [k.data_ptr() for k in shard_keys],
                             [v.data_ptr() for v in shard_vals], sp, [k.numel() for k in shard_keys], t0, t1,
                             torch.device("cuda", torch.cuda.current_device()), out_keys, out_vals, workspace)


def _shard_merge_ptrs(dtype, kptrs, vptrs, sptrs, sizes, t0, t1, dev, out_keys=None, out_vals=None, workspace=None):
    """shard_merge over raw device pointers (local or peer-mapped)."""
    import torch

    lib = _lib.load()
    G = len(kptrs)
    dt = _dtype_id(torch.empty(0, dtype=dtype))
    n = t1 - t0
    if out_keys is None:
        out_keys = torch.empty(n, dtype=dtype, device=dev)
    if out_vals is None:
        out_vals = torch.empty(n, dtype=torch.int32, device=dev)
    kp = (ctypes.c_void_p * G)(*kptrs)
    vp = (ctypes.c_void_p * G)(*vptrs)
    sp = None if sptrs is None else (ctypes.c_void_p * G)(*sptrs)
    ns = (ctypes.c_int64 * G)(*[int(x) for x in sizes])
    nbytes = int(lib.ps_shard_merge_workspace_size(G, n))
    ws = workspace
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.ps_shard_merge(dt, G, kp, vp, sp, ns, t0, t1, out_keys.data_ptr(), out_vals.data_ptr(),
                                  ws.data_ptr(), ws.numel(), stream))
    return out_keys, out_vals


def _ipc_export(t):
    """(CUDA IPC handle of the allocation holding ``t``, byte offset of ``t``
    in it, element count): plain bytes and ints, exchanged as plumbing."""
    lib = _lib.load()
    handle = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _lib.check(lib.ps_ipc_export(t.device.index, t.data_ptr(), handle, ctypes.byref(off)))
    return handle.raw, int(off.value), t.numel()


class DistributedSorter:
    """Persistent multi-GPU sorter for one rank (one process per GPU).

    Owns the rank's shard buffers (``keys``: fill it, then call ``sort``), the
    global-index payload, the shard's sample array and the output slab.  The
    CUDA IPC handles of the shard, payload and samples are exchanged once at
    construction (``all_gather_object``, plumbing only) and the peers' buffers
    stay mapped, so a sort is: local sort of the shard, its samples, a host
    barrier, the single-pass cross-shard merge of this rank's slab (peer loads
    over NVLink), and a closing barrier (peers keep their shards until every
    slab is merged)."""

    def __init__(self, n_local, dtype, config=None, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.config = config or SortConfig()
        self.group = group
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        sizes = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(sizes, int(n_local), group=group)
        else:
            sizes = [int(n_local)]
        self.plan = plan(sizes, self.rank)
        off = self.plan["offsets"][self.rank]
        self.keys = torch.empty(n_local, dtype=dtype, device=dev)
        self.vals = torch.empty(n_local, dtype=torch.int32, device=dev)
        self._iota = torch.arange(off, off + n_local, dtype=torch.int32, device=dev)
        lib = _lib.load()
        ns = int(lib.ps_shard_sample_count(_dtype_id(self.keys), n_local))
        self.samples = torch.empty(max(ns, 1), dtype=dtype, device=dev)
        t0, t1 = self.plan["slab"]
        self.out_keys = torch.empty(t1 - t0, dtype=dtype, device=dev)
        self.out_vals = torch.empty(t1 - t0, dtype=torch.int32, device=dev)
        self.ws = torch.empty(max(int(lib.ps_shard_merge_workspace_size(self.world, t1 - t0)), 1),
                              dtype=torch.uint8, device=dev)
        self.device = dev
        self.peers = None
        self._mapped = []
        if self.world > 1:
            # each rank's shard, payload and samples are opened in THIS device's
            # context (ps_ipc_open: lazy peer access), not the peer's, so the
            # shard-merge kernel here loads them over NVLink
            handles = [None] * self.world
            dist.all_gather_object(handles, tuple(_ipc_export(t) for t in (self.keys, self.vals, self.samples)),
                                   group=group)
            self.peers = []
            for g, hs in enumerate(handles):
                if g == self.rank:
                    self.peers.append(tuple(t.data_ptr() for t in (self.keys, self.vals, self.samples)))
                    continue
                ptrs = []
                for handle, off, _ in hs:
                    base = ctypes.c_void_p()
                    _lib.check(lib.ps_ipc_open(dev.index, handle, ctypes.byref(base)))
                    self._mapped.append(base.value)
                    ptrs.append(base.value + off)
                self.peers.append(tuple(ptrs))

    def close(self):
        """Unmap the peers' buffers (after a closing barrier of every rank)."""
        lib = _lib.load()
        while self._mapped:
            _lib.check(lib.ps_ipc_close(self.device.index, self._mapped.pop()))

    def sort(self):
        """Sort the global array whose shard this rank holds in ``keys``;
        returns (slab keys, slab global indices) views of this rank's slab."""
        import torch

        self.vals.copy_(self._iota)
        if self.keys.numel():
            _sort_tensor(self.keys, self.vals, self.config, _lib.VALUES_PERMUTE, collect_runs=False)
        if self.world == 1:
            return self.keys, self.vals
        shard_samples(self.keys, self.samples)
        torch.cuda.synchronize(self.keys.device)
        self.dist.barrier(group=self.group)
        t0, t1 = self.plan["slab"]
        sizes = self.plan["sizes"]
        _shard_merge_ptrs(self.keys.dtype, [p[0] for p in self.peers], [p[1] for p in self.peers],
                          [p[2] if sizes[g] else None for g, p in enumerate(self.peers)], sizes, t0, t1,
                          self.device, self.out_keys, self.out_vals, self.ws)
        torch.cuda.synchronize(self.keys.device)
        self.dist.barrier(group=self.group)  # peers keep their shards alive until every slab is merged
        return self.out_keys, self.out_vals


def sort_distributed(keys, config=None, group=None):
    """Sort a globally sharded array: ``keys`` is this rank's contiguous shard
    (CUDA tensor).  Returns (slab_keys, slab_global_indices) of this rank's
    slab of the global stable order.  One-shot form of DistributedSorter."""
    sorter = DistributedSorter(keys.numel(), keys.dtype, config, group, keys.device)
    sorter.keys.copy_(keys)
    k, v = sorter.sort()
    k, v = k.clone(), v.clone()
    sorter.close()
    return k, v

"""O(n) certificate of a stable sort, on the device.

A stable sort's output is unique, so for keys ``src`` and the pair
(``keys``, ``perm``) returned by :func:`stable_argsort` these four checks are
equivalent to bit-exactness against the reference (policy.py:201-262):

1. ``perm`` is a permutation of 0..n-1;
2. ``keys == src[perm]`` bit for bit (so -0.0 / +0.0 are told apart);
3. ``keys`` is nondecreasing under the reference's ``<=`` (statskit.py:68-72);
4. equal keys keep increasing source index (stability).

Used by bench.py and the full-size tests where the CPU oracle cannot run the
whole sort (cfg5, n = 2^31).
"""

from __future__ import annotations

_BITS = None


def _bits(t):
    import torch

    global _BITS
    if _BITS is None:
        _BITS = {torch.float32: torch.int32, torch.float64: torch.int64}
    return t.view(_BITS[t.dtype]) if t.dtype in _BITS else t


def certify(src, keys, perm, chunk=1 << 28):
    """Raises AssertionError unless (keys, perm) is the stable sort of src.
    Works in chunks of ``chunk`` elements to bound the temporaries."""
    import torch

    n = src.numel()
    assert keys.numel() == n and perm.numel() == n, "length mismatch"
    if n == 0:
        return
    dev = src.device
    seen = torch.zeros(n, dtype=torch.uint8, device=dev)
    for a in range(0, n, chunk):
        p = perm[a:a + chunk].long()
        assert int(p.min()) >= 0 and int(p.max()) < n, "perm out of range"
        seen.index_fill_(0, p, 1)
        assert torch.equal(_bits(src[p]), _bits(keys[a:a + chunk])), "keys != src[perm]"
        b = min(n, a + chunk + 1)  # one element of overlap with the next chunk
        k0, k1 = keys[a:b - 1], keys[a + 1:b]
        assert bool((k0 <= k1).all()), "keys not sorted"
        p0, p1 = perm[a:b - 1], perm[a + 1:b]
        assert not bool(((k0 == k1) & (p0 > p1)).any()), "equal keys out of source order"
        del p
    assert int(seen.sum(dtype=torch.int64)) == n, "perm is not a permutation"


_M1, _M2, _M3 = 0x9E3779B97F4A7C15 - 2**64, 0xBF58476D1CE4E5B9 - 2**64, 0x94D049BB133111EB - 2**64


def _pair_hash(kbits, idx):
    """A 64-bit mix of (key bits, index) per element (int64, wrapping)."""
    h = kbits.long() * _M1 + idx.long() * _M2
    h = h ^ (h >> 31)  # arithmetic shift: still a fixed bijection-like mix
    h = h * _M3
    return h ^ (h >> 29)


def distributed_certify(src_shard, src_off, slab_keys, slab_idx, slab, red_dev, group=None):
    """Certificate of a multi-GPU stable sort (bench.py --gpus N): this rank's
    slab [t0, t1) is sorted with equal keys in increasing global index, its
    first record follows the previous slab's last one, and the (key, global
    index) pairs of all slabs together equal those of all input shards
    (all-reduced sums of a 64-bit pair hash, and of the index sums)."""
    import torch
    import torch.distributed as dist

    t0, t1 = slab
    assert slab_keys.numel() == t1 - t0 == slab_idx.numel(), "slab length"
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bad = []  # collected, so that every rank reaches every collective
    if slab_keys.numel() > 1:
        k0, k1 = slab_keys[:-1], slab_keys[1:]
        if not bool((k0 <= k1).all()):
            bad.append("slab not sorted")
        elif bool(((k0 == k1) & (slab_idx[:-1] > slab_idx[1:])).any()):
            bad.append("slab not stable")
    # slab boundaries: every rank's (first key, last key, first index, last
    # index, length), keys exact as float64 (float keys) or int64 (int keys)
    is_f = slab_keys.dtype in (torch.float32, torch.float64)
    wide = torch.float64 if is_f else torch.int64
    m = slab_keys.numel()
    edge_k = torch.tensor([slab_keys[0].item() if m else 0, slab_keys[-1].item() if m else 0], dtype=wide)
    edge_i = torch.tensor([int(slab_idx[0]) if m else -1, int(slab_idx[-1]) if m else -1, m], dtype=torch.int64)
    ek = [torch.zeros_like(edge_k).to(red_dev) for _ in range(world)]
    ei = [torch.zeros_like(edge_i).to(red_dev) for _ in range(world)]
    dist.all_gather(ek, edge_k.to(red_dev), group=group)
    dist.all_gather(ei, edge_i.to(red_dev), group=group)
    prev = [g for g in range(rank) if int(ei[g][2]) > 0]
    if m and prev:
        g = prev[-1]
        pk, fk = ek[g][1].item(), ek[rank][0].item()
        pi, fi = int(ei[g][1]), int(ei[rank][0])
        if not (pk < fk or (pk == fk and pi < fi)):
            bad.append("slab boundary out of order")
    n_src = src_shard.numel()
    gidx = torch.arange(src_off, src_off + n_src, dtype=torch.int64, device=src_shard.device)
    h_in = _pair_hash(_bits(src_shard), gidx).sum()
    h_out = _pair_hash(_bits(slab_keys), slab_idx).sum()
    v = torch.stack([h_in, h_out, gidx.sum(), slab_idx.long().sum()]).to(red_dev)
    dist.all_reduce(v, group=group)
    if int(v[0]) != int(v[1]):
        bad.append("output (key, index) pairs differ from the input")
    if int(v[2]) != int(v[3]):
        bad.append("output indices are not the input indices")
    nbad = torch.tensor([len(bad)], dtype=torch.int64, device=red_dev)
    dist.all_reduce(nbad, group=group)
    assert int(nbad) == 0, "rank %d: %s (%d failures over all ranks)" % (rank, "; ".join(bad) or "ok", int(nbad))


"""Multi-GPU mode.

CPU tests cover the host logic: the slab plan exchanged over a world-size-2
gloo group, and a pure-Python restatement of the parallel bracketing co-rank
selection that ps_shard_merge runs on the device (shard_select_kernel).
GPU tests run ps_shard_merge with G shards emulated on one device, and a
two-process sort_distributed over CUDA IPC on one GPU (gloo for plumbing).
"""

import os
import socket

import numpy as np
import pytest

from paper_2209_06909_b200 import multigpu

SEL_CANDIDATES = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan_worker(rank, world, port, sizes, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = [None] * world
    dist.all_gather_object(got, sizes[rank])
    q.put((rank, multigpu.plan(got, rank)))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_plan_over_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    sizes = [1000, 777]
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["offsets"] == [0, 1000] and res[1]["total"] == 1777
    assert res[0]["slab"] == (0, 888) and res[1]["slab"] == (888, 1777)


@pytest.mark.parametrize("total,world", [(0, 1), (10, 3), (2**31, 8), (12345, 7)])
def test_slabs_partition_the_ranks(total, world):
    slabs = [multigpu.slab_bounds(total, world, g) for g in range(world)]
    assert slabs[0][0] == 0 and slabs[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))


def bracket_select(shards, t, rounds=None):
    """Restatement of shard_select_kernel: co-rank of global rank t in the
    stable merge of sorted shards (order (key, shard, position))."""
    G = len(shards)
    n = [len(s) for s in shards]
    N = sum(n)
    lo = [max(0, t - (N - n[h])) for h in range(G)]
    hi = [min(n[h], t) for h in range(G)]
    for _ in range(rounds or 64):
        if lo == hi:
            break
        cur_lo, cur_hi = list(lo), list(hi)
        for g in range(G):
            w = cur_hi[g] - cur_lo[g]
            if w <= 0:
                continue
            for ci in range(SEL_CANDIDATES):
                p = cur_lo[g] + (w * (ci + 1)) // (SEL_CANDIDATES + 1)
                if p >= cur_hi[g]:
                    continue
                y = shards[g][p]
                r = []
                for h in range(G):
                    if h == g:
                        r.append(p)
                        continue
                    side = "right" if h < g else "left"  # <= for earlier shards, < for later
                    pos = int(np.searchsorted(shards[h][cur_lo[h]:cur_hi[h]], y, side=side)) + cur_lo[h]
                    r.append(pos)
                R = sum(r)
                for h in range(G):
                    if R < t:
                        lo[h] = max(lo[h], p + 1 if h == g else r[h])
                    else:
                        hi[h] = min(hi[h], p if h == g else r[h])
    assert lo == hi
    return lo


def test_bracketing_selection_matches_stable_merge():
    rng = np.random.default_rng(4)
    for trial in range(60):
        G = int(rng.integers(1, 9))
        shards = []
        for _ in range(G):
            m = int(rng.integers(0, 400))
            hi = int(rng.choice([3, 50, 10**6]))
            shards.append(np.sort(rng.integers(0, hi, size=m)))
        allk = np.concatenate(shards) if shards else np.array([])
        shard_id = np.concatenate([np.full(len(s), h) for h, s in enumerate(shards)])
        order = np.lexsort((shard_id, allk))  # stable (key, shard, position)
        N = len(allk)
        for t in sorted(set([0, N, N // 2, int(rng.integers(0, N + 1))])):
            c = bracket_select(shards, t)
            first_t = shard_id[order[:t]]
            expect = [int(np.sum(first_t == h)) for h in range(G)]
            assert c == expect, (trial, t)


def _precedes(z, b, y, a):
    """(b, key z) before (a, key y) in (key, shard) order (xs_precedes)."""
    return z < y or (not (y < z) and b < a)


def sample_cut_rows(shards, t0, t1, m, s):
    """Python restatement of the device plan of ps_shard_merge (ps_shard.cuh:
    xs_plan_kernel, xs_cuts_kernel): boundary rows (lo[], hi[], cut) in merged
    order, from the exact co-ranks of t0 / t1 and rank searches among samples."""
    G = len(shards)
    c0 = bracket_select(shards, t0)
    c1 = bracket_select(shards, t1)
    cd = lambda a, b: -(-a // b)  # noqa: E731
    w0 = [cd(c, s) for c in c0]
    w1 = [cd(c, s) for c in c1]
    j0 = [cd(w, m) for w in w0]
    rows = {}
    for a in range(G):
        for j in range(j0[a], cd(w1[a], m)):
            i = j * m
            x = shards[a][i * s]
            lo, hi, idx = [], [], 0
            for b in range(G):
                if b == a:
                    rb = i
                    lo.append(i * s)
                    hi.append(i * s)
                else:
                    smp = shards[b][::s][w0[b]:w1[b]]
                    r = 0
                    while r < len(smp) and _precedes(smp[r], b, x, a):
                        r += 1
                    rb = w0[b] + r
                    l_, h_ = ((rb - 1) * s + 1 if rb else 0), rb * s
                    lo.append(min(max(l_, c0[b]), c1[b]))
                    hi.append(min(max(h_, c0[b]), c1[b]))
                idx += cd(rb, m) - j0[b]
            assert idx not in rows
            rows[idx] = (lo, hi, (x, a, i * s))
    out = [(list(c0), list(c0), None)] + [rows[i] for i in range(len(rows))] + [(list(c1), list(c1), None)]
    return out


def _exact(shard, b, lo, hi, cut):
    if cut is None or cut[1] == b:
        return lo
    x, a, _ = cut
    q = lo
    while q < hi and _precedes(shard[q], b, x, a):
        q += 1
    return q


def test_sample_cuts_partition_the_slab():
    """The rows of the device plan cut every slab into chunks whose bracketed
    windows fit one unit, and the chunks' exact boundaries (resolved inside
    the brackets, as xs_merge_kernel does in shared memory) reproduce the
    stable merge."""
    rng = np.random.default_rng(11)
    for trial in range(40):
        G = int(rng.integers(1, 9))
        s = int(rng.choice([2, 4, 8]))
        m = int(rng.integers(1, 5))
        shards = []
        for _ in range(G):
            n = int(rng.integers(0, 300))
            hi = int(rng.choice([3, 40, 10**6]))
            shards.append(np.sort(rng.integers(0, hi, size=n)))
        allk = np.concatenate(shards)
        sid = np.concatenate([np.full(len(x), h) for h, x in enumerate(shards)])
        pos = np.concatenate([np.arange(len(x)) for x in shards])
        order = np.lexsort((sid, allk))
        N = len(allk)
        for W in (1, 2, 3):
            for g in range(W):
                t0, t1 = multigpu.slab_bounds(N, W, g)
                rows = sample_cut_rows(shards, t0, t1, m, s)
                E = [[_exact(shards[b], b, lo[b], hi[b], cut) for b in range(G)] for lo, hi, cut in rows]
                got = []
                for r in range(len(rows) - 1):
                    loaded = sum(rows[r + 1][1][b] - rows[r][0][b] for b in range(G))
                    assert loaded <= G * (m + 2) * s, (trial, loaded)
                    part = [(shards[b][q], b, q) for b in range(G) for q in range(E[r][b], E[r + 1][b])]
                    got += sorted(part, key=lambda t: (t[0], t[1], t[2]))
                exp = [(allk[o], sid[o], pos[o]) for o in order[t0:t1]]
                assert [(int(a), int(b), int(c)) for a, b, c in got] == [(int(a), int(b), int(c)) for a, b, c in exp]


# --------------------------------------------------------------------- GPU
torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("kind", ["cfg2", "dups", "disjoint"])
def test_shard_merge_emulated_on_one_gpu(G, kind):
    from paper_2209_06909_b200 import SortConfig, stable_sort_with, workloads

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(G * 7 + len(kind))
    n = 200_000 + int(rng.integers(0, 1000))
    if kind == "cfg2":
        keys = workloads.cfg2(n=n, seed=G)
    elif kind == "dups":
        keys = rng.integers(0, 5, size=n).astype(np.int32)
    else:
        keys = np.arange(n, dtype=np.int32)[::-1].copy()  # each shard's keys disjoint from the others
    cuts = np.sort(rng.integers(0, n, size=G - 1)) if G > 1 else np.array([], dtype=np.int64)
    bounds = [0] + cuts.tolist() + [n]
    sk, sv = [], []
    for g in range(G):
        a, b = bounds[g], bounds[g + 1]
        k = torch.from_numpy(keys[a:b].copy()).to(dev)
        v = torch.arange(a, b, dtype=torch.int32, device=dev)
        if k.numel():
            stable_sort_with(k, SortConfig(), values=v)
        sk.append(k)
        sv.append(v)
    smp = [multigpu.shard_samples(k) if k.numel() else None for k in sk] if G % 2 == 0 else None
    out_k, out_v = [], []
    for g in range(G):
        t0, t1 = multigpu.slab_bounds(n, G, g)
        k, v = multigpu.shard_merge(sk, sv, t0, t1, samples=smp)
        out_k.append(k.cpu().numpy())
        out_v.append(v.cpu().numpy())
    perm = np.argsort(keys, kind="stable")
    assert np.array_equal(np.concatenate(out_v), perm)
    assert np.array_equal(np.concatenate(out_k), keys[perm])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "int64", "float64", "int32"])
@pytest.mark.parametrize("G", [2, 7, 8])
def test_shard_merge_dtypes_sizes_and_empty_shards(dtype, G):
    """Slabs of 8 shards (some empty, some tiny) with many units per slab;
    published samples; ties across shards; odd slab bounds."""
    from paper_2209_06909_b200 import SortConfig, stable_sort_with

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(G * 31 + len(dtype))
    sizes = rng.integers(0, 700_000, size=G)
    sizes[rng.integers(0, G)] = 0
    if G > 2:
        sizes[(rng.integers(0, G) + 1) % G] = 17
    n = int(sizes.sum())
    if dtype.startswith("float"):
        keys = (rng.integers(-5000, 5000, size=n) * 0.25).astype(dtype)
    else:
        keys = rng.integers(-3000, 3000, size=n).astype(dtype) * np.array(2**33 if dtype == "int64" else 1,
                                                                          dtype=dtype)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    sk, sv = [], []
    for g in range(G):
        a, b = int(bounds[g]), int(bounds[g + 1])
        k = torch.from_numpy(keys[a:b].copy()).to(dev)
        v = torch.arange(a, b, dtype=torch.int32, device=dev)
        if k.numel():
            stable_sort_with(k, SortConfig(), values=v)
        sk.append(k)
        sv.append(v)
    smp = [multigpu.shard_samples(k) if k.numel() else None for k in sk]
    perm = np.argsort(keys, kind="stable")
    cuts = [0, 1, n // 3 + 5, n // 2, n - 1, n]
    for t0, t1 in zip(cuts[:-1], cuts[1:]):
        k, v = multigpu.shard_merge(sk, sv, t0, t1, samples=smp)
        assert np.array_equal(v.cpu().numpy(), perm[t0:t1]), (t0, t1)
        assert np.array_equal(k.cpu().numpy().view(np.uint8), keys[perm[t0:t1]].view(np.uint8)), (t0, t1)


def _dist_worker(rank, world, port, n, q):
    import torch.distributed as dist

    from paper_2209_06909_b200 import workloads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)  # both ranks share the single test GPU (host barriers only)
    keys = workloads.cfg5(n=n, seed=1)
    a, b = multigpu.slab_bounds(n, world, rank)
    shard = torch.from_numpy(keys[a:b].copy()).cuda()
    k, v = multigpu.sort_distributed(shard)
    q.put((rank, k.cpu().numpy(), v.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sort_distributed_two_processes_one_gpu():
    import torch.multiprocessing as mp

    from paper_2209_06909_b200 import workloads

    n = 300_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (k, v)) for r, k, v in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    keys = workloads.cfg5(n=n, seed=1)
    perm = np.argsort(keys, kind="stable")
    assert np.array_equal(np.concatenate([res[0][1], res[1][1]]), perm)
    assert np.array_equal(np.concatenate([res[0][0], res[1][0]]).view(np.uint32), keys[perm].view(np.uint32))


def _certify_worker(rank, world, port, q, tamper):
    import torch
    import torch.distributed as dist

    from paper_2209_06909_b200.certify import distributed_certify

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    N = 5000
    keys = rng.integers(0, 300, size=N).astype(np.float32)  # many ties
    order = np.argsort(keys, kind="stable")
    lo, hi = multigpu.slab_bounds(N, world, rank)
    src = torch.from_numpy(keys[lo:hi].copy())
    t0, t1 = multigpu.slab_bounds(N, world, rank)
    sk = torch.from_numpy(keys[order][t0:t1].copy())
    si = torch.from_numpy(order[t0:t1].astype(np.int32))
    if tamper == "swap" and rank == 1:
        si[[3, 4]] = si[[4, 3]]  # breaks stability (or order) within the slab
        sk[[3, 4]] = sk[[4, 3]]
    if tamper == "dup" and rank == 0:
        si[-1] = si[-2]  # duplicate index: multiset differs
    try:
        distributed_certify(src, lo, sk, si, (t0, t1), torch.device("cpu"))
        q.put((rank, "ok"))
    except AssertionError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


@pytest.mark.parametrize("tamper", [None, "swap", "dup"])
def test_distributed_certificate_gloo_world2(tamper):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_certify_worker, args=(r, 2, port, q, tamper)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    if tamper is None:
        assert res == {0: "ok", 1: "ok"}
    else:
        assert any(v != "ok" for v in res.values()), res


@pytest.mark.gpu
def test_shard_merge_eight_shards_at_scale():
    """8 shards of 2^23 cfg5-recipe keys (2^26 in all), every slab merged with
    published samples and checked against numpy's stable argsort of the whole
    input: thousands of units and cuts per slab."""
    from paper_2209_06909_b200 import SortConfig, stable_sort_with, workloads

    dev = torch.device("cuda", 0)
    G, m = 8, 1 << 23
    keys = workloads.cfg5(n=G * m, seed=3)
    sk, sv = [], []
    for g in range(G):
        k = torch.from_numpy(keys[g * m:(g + 1) * m].copy()).to(dev)
        v = torch.arange(g * m, (g + 1) * m, dtype=torch.int32, device=dev)
        stable_sort_with(k, SortConfig(), values=v)
        sk.append(k)
        sv.append(v)
    smp = [multigpu.shard_samples(k) for k in sk]
    out_v = []
    for g in range(G):
        t0, t1 = multigpu.slab_bounds(G * m, G, g)
        _, v = multigpu.shard_merge(sk, sv, t0, t1, samples=smp)
        out_v.append(v.cpu().numpy())
    assert np.array_equal(np.concatenate(out_v), np.argsort(keys, kind="stable"))

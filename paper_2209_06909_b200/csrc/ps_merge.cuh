// ps_merge.cuh -- N3: batched stable k-way merges (one launch per tree level).
//
// Replaces merges.py:75-500 (merge_2way_*, merge_3way, merge_4way_*).  A stable
// k-way merge has a unique output (ties go to the lower-index run,
// merges.py:1-8), i.e. the merge under the strict order (key, run, position).
//
// Big nodes are cut into chunks: cut (a, j) is the record at position j*S of
// run a (S = cut_cap / arity); its rank in every other run b is a search
// (<= for b < a, < for b > a) and its index in the merged cut order follows
// directly from those ranks.  Between consecutive cuts there are at most S
// records of each run, so every chunk holds <= cut_cap records.
//
// merge_pipe_kernel (persistent, warp-specialized):
//   producer warp  -- reads the descriptors of 32 chunks at once, packs
//                     consecutive chunks of a node into units of <= cut_cap
//                     records and stages each unit's k input windows (keys
//                     and values) into a free smem slot with TMA bulk copies
//                     (cp.async.bulk + mbarrier complete_tx), double-buffered;
//   consumer warps -- merge the unit with branch-light merge-path passes:
//                     4-way = merge(merge(A,B), merge(C,D)), 3-way =
//                     merge(merge(A,B), C), 2-way = merge(A,B); ties go left
//                     in every pass, so the result is the stable k-way merge.
//                     Outputs land in a bank-padded smem layout and leave with
//                     16-byte coalesced stores.
// Children are read from buffer (depth+1)&1 and the node writes depth&1.
#pragma once

#include "ps_common.cuh"
#include "ps_form.cuh"

namespace ps {

// consumer threads per merge_pipe_kernel CTA, per key width.  4-byte keys: 288
// consumers x VT 15 (units of 4320 records, ~111 KB of shared memory), so two
// CTAs share an SM and each fills the other's barrier and load waits: the merge
// kernels of cfg5 run 7% faster than with one CTA of 576 x 15 per SM (the
// geometry until round 2; 0.8% faster than 512 x 17 on cfg2), at twice the
// cuts (cfg5 partition 4.3 -> 7.3 ms; cfg5 -2.8%, cfg4 -4%, cfg2 +1.6% per sort).
// 8-byte keys: one CTA of 352 x 13 per SM (2.8% faster than 512 x 9 on cfg3; two
// CTAs of 160 x 13 are 1% slower).
#ifndef PS_CONSUMERS4
#define PS_CONSUMERS4 288
#endif
#ifndef PS_CONSUMERS8
#define PS_CONSUMERS8 352
#endif
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_consumers() {
    return sizeof(K) == 4 ? PS_CONSUMERS4 : PS_CONSUMERS8;
}
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_threads() {
    return 32 + pipe_consumers<K>();
}

// Consumer thread t produces the VT outputs [VT*t, VT*t + VT) of every merge
// pass.  VT is odd (15 records of 8 bytes, 13 of 16 bytes): the k-th output of
// the lanes of a warp lands in distinct banks (2 or 4 wavefronts per warp
// store, the minimum), and the data-dependent read positions of balanced
// merges (~VT/2 * t) spread over all banks as well.  No padding is needed.
#ifndef PS_VT4
#define PS_VT4 15
#endif
#ifndef PS_VT8
#define PS_VT8 13
#endif
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_vt() {
    return sizeof(K) == 4 ? PS_VT4 : PS_VT8;
}
// segments per unit (bounds the slot's window-alignment slack: two CTAs of
// 4-byte keys must fit an SM)
#ifndef PS_MAXSEG4
#define PS_MAXSEG4 8
#endif
#ifndef PS_MAXSEG8
#define PS_MAXSEG8 32
#endif
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_maxseg() {
    return sizeof(K) == 4 ? PS_MAXSEG4 : PS_MAXSEG8;
}
// records per unit (smem slot capacity)
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_cap() {
    return pipe_vt<K>() * pipe_consumers<K>();
}
// Cut spacing budget: units hold <= CAP - VT records, so pass 1 can start Y
// at a VT-aligned offset (no thread straddles X and Y) within NC threads.
template <class K>
PS_DEV __host__ constexpr uint32_t cut_cap() {
    return pipe_cap<K>() - pipe_vt<K>();
}
PS_DEV __host__ constexpr uint32_t align16c(uint32_t x) { return (x + 15u) & ~15u; }
PS_DEV __host__ constexpr uint32_t cmax(uint32_t a, uint32_t b) { return a > b ? a : b; }

// smallest cut spacing of any key type (bounds the chunk count)
constexpr uint32_t MIN_CUT_SPACING =
    (cut_cap<int32_t>() < cut_cap<int64_t>() ? cut_cap<int32_t>() : cut_cap<int64_t>()) / MAX_WAY;

// # of a[0..len) that are <= x (LE) or < x (!LE): branch-free binary lifting
// (the predicate holds on a prefix; add the largest powers of two that keep it)
template <class K, bool LE>
PS_DEV uint32_t count_pred(const K* __restrict__ a, uint32_t len, K x) {
    uint32_t lo = 0;
    for (uint32_t step = len ? (1u << (31 - __clz(len))) : 0u; step; step >>= 1) {
        const uint32_t probe = lo + step;
        if (probe <= len) {
            const K y = a[probe - 1];
            const bool p = LE ? !(x < y) : (y < x);
            lo = p ? probe : lo;
        }
    }
    return lo;
}

// Warp-cooperative count of a[0..len) <= x (LE) or < x: 32-ary search, one
// coalesced probe round per factor of 33 (all lanes return the result).
template <class K, bool LE>
PS_DEV uint32_t warp_count_pred(const K* __restrict__ a, uint32_t len, K x) {
    const uint32_t lane = lane_id();
    uint32_t lo = 0, hi = len;  // answer in [lo, hi]; pred true on [0, ans)
    while (hi - lo > 32) {
        const uint32_t span = hi - lo;
        const uint32_t probe = lo + (uint32_t)(((uint64_t)span * (lane + 1)) / 33);
        const K y = a[probe];
        const bool p = LE ? !(x < y) : (y < x);
        const uint32_t bal = __ballot_sync(PS_FULL, p);
        // pred is monotone: true for lanes < c
        const uint32_t c = __popc(bal);
        const uint32_t nlo = c ? lo + (uint32_t)(((uint64_t)span * c) / 33) + 1 : lo;
        const uint32_t nhi = c < 32 ? lo + (uint32_t)(((uint64_t)span * (c + 1)) / 33) : hi;
        lo = nlo;
        hi = nhi;
    }
    // final <= 32 candidates [lo, hi): one probe each
    const uint32_t idx = lo + lane;
    bool p = false;
    if (idx < hi) {
        const K y = a[idx];
        p = LE ? !(x < y) : (y < x);
    }
    return lo + __popc(__ballot_sync(PS_FULL, p));
}

// Up to three counts at once (one per other run): lanes 10g..10g+9 run an
// 11-ary search in array g, all groups in the same rounds (~8 rounds for 2^22
// elements instead of three sequential searches).  le[g]: count <= x, else < x.
template <class K>
PS_DEV void warp_count3(const K* r0, const K* r1, const K* r2, uint32_t l0, uint32_t l1, uint32_t l2, bool le0,
                        bool le1, bool le2, uint32_t nsearch, K x, uint32_t* out) {
    const uint32_t lane = lane_id();
    const uint32_t grp = lane / 10, sub = lane % 10;
    const bool active = grp < nsearch;
    const K* run = grp == 0 ? r0 : (grp == 1 ? r1 : r2);
    const bool le = grp == 0 ? le0 : (grp == 1 ? le1 : le2);
    uint32_t lo = 0, hi = active ? (grp == 0 ? l0 : (grp == 1 ? l1 : l2)) : 0;
    const uint32_t gshift = grp < 3 ? grp * 10 : 0;
    while (__any_sync(PS_FULL, hi - lo > 10)) {
        const uint32_t span = hi - lo;
        const bool probing = span > 10;
        bool p = false;
        if (probing) {
            const uint32_t probe = lo + (uint32_t)(((uint64_t)span * (sub + 1)) / 11);
            const K y = run[probe];
            p = le ? !(x < y) : (y < x);
        }
        const uint32_t bal = __ballot_sync(PS_FULL, p);
        if (probing) {
            const uint32_t c = __popc((bal >> gshift) & 0x3FFu);
            const uint32_t nlo = c ? lo + (uint32_t)(((uint64_t)span * c) / 11) + 1 : lo;
            const uint32_t nhi = c < 10 ? lo + (uint32_t)(((uint64_t)span * (c + 1)) / 11) : hi;
            lo = nlo;
            hi = nhi;
        }
    }
    const uint32_t idx = lo + sub;
    bool p = false;
    if (active && idx < hi) {
        const K y = run[idx];
        p = le ? !(x < y) : (y < x);
    }
    const uint32_t bal = __ballot_sync(PS_FULL, p);
    const uint32_t res = lo + __popc((bal >> gshift) & 0x3FFu);
    out[0] = __shfl_sync(PS_FULL, res, 0);
    out[1] = __shfl_sync(PS_FULL, res, 10);
    out[2] = __shfl_sync(PS_FULL, res, 20);
}

// Partition: the cut of chunk c's (run, j) pair (whole warp; every chunk index
// of a node past its first maps to one (a, j) with j*S < L[a]); the cut lands at
// its index in the merged cut order.  The first chunk of each node gets the
// zero cut.
template <class K>
PS_DEV void partition_chunk(const Bufs<K>& bufs, const Node* __restrict__ nodes, const uint32_t* __restrict__ chunk2node,
                            uint32_t c, uint4* __restrict__ cuts) {
    const uint32_t lane = lane_id();
    const Node nd = nodes[chunk2node[c]];
    uint32_t q = c - nd.chunk_base;
    if (q == 0) {
        if (lane == 0) cuts[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    q -= 1;
    const uint32_t w = nd.arity;
    const uint32_t S = node_spacing(nd, cut_cap<K>());
    const K* src = bufs.kb(nd.parity ^ 1);
    uint32_t L[4];
#pragma unroll
    for (uint32_t a = 0; a < 4; ++a) L[a] = a < w ? nd.pos[a + 1] - nd.pos[a] : 0;
    uint32_t a = 0;
    for (; a < w; ++a) {
        const uint32_t nc = (L[a] - 1) / S;
        if (q < nc) break;
        q -= nc;
    }
    const uint32_t j = q + 1;
    const K y = src[(uint64_t)nd.pos[a] + (uint64_t)j * S];
    // the other runs, in order: o = index among them, run bb = o + (o >= a)
    const uint32_t b0 = a == 0 ? 1 : 0, b1 = a <= 1 ? 2 : 1, b2 = a == 3 ? 2 : 3;
    uint32_t got[3];
    warp_count3<K>(src + nd.pos[b0], src + nd.pos[b1], src + nd.pos[b2 < w ? b2 : 0], L[b0],
                   b1 < w ? L[b1] : 0, b2 < w ? L[b2] : 0, b0 < a, b1 < a, b2 < a, w - 1, y, got);
    uint32_t rk[4] = {0, 0, 0, 0};
    rk[a] = j * S;
    uint32_t mm = j - 1;
#pragma unroll
    for (uint32_t o = 0; o < 3; ++o) {
        if (o + 1 >= w) break;
        const uint32_t bb = o + (o >= a ? 1 : 0);
        rk[bb] = got[o];
        mm += got[o] ? (got[o] - 1) / S : 0;
    }
    if (lane == 0) cuts[nd.chunk_base + 1 + mm] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
}

constexpr uint32_t COUNT_SMALL = 512;  // nodes counted by one thread

// Up to three counts at once by one thread (the scalar twin of warp_count3).
template <class K>
PS_DEV void thread_count3(const K* r0, const K* r1, const K* r2, uint32_t l0, uint32_t l1, uint32_t l2, bool le0,
                          bool le1, bool le2, uint32_t nsearch, K x, uint32_t* out) {
    out[0] = nsearch > 0 ? (le0 ? count_pred<K, true>(r0, l0, x) : count_pred<K, false>(r0, l0, x)) : 0u;
    out[1] = nsearch > 1 ? (le1 ? count_pred<K, true>(r1, l1, x) : count_pred<K, false>(r1, l1, x)) : 0u;
    out[2] = nsearch > 2 ? (le2 ? count_pred<K, true>(r2, l2, x) : count_pred<K, false>(r2, l2, x)) : 0u;
}

// The counters of one node (see merge_counters_kernel); WARP: the whole warp
// cooperates in every rank search (big nodes), else one thread per node.
template <class K, bool WARP>
PS_DEV void node_counters(const Bufs<K>& bufs, const Node& nd, int variant, unsigned long long& cmp,
                          unsigned long long& wr) {
    auto cnt3 = [](const K* r0, const K* r1, const K* r2, uint32_t l0, uint32_t l1, uint32_t l2, bool le0,
                   bool le1, bool le2, uint32_t nsearch, K x, uint32_t* out) {
        if (WARP)
            warp_count3<K>(r0, r1, r2, l0, l1, l2, le0, le1, le2, nsearch, x, out);
        else
            thread_count3<K>(r0, r1, r2, l0, l1, l2, le0, le1, le2, nsearch, x, out);
    };
    const uint32_t w = nd.arity, T = nd.pos[w] - nd.pos[0];
    const K* src = bufs.kb(nd.parity ^ 1);
    uint32_t L[4], e[4], g[4][3];
#pragma unroll
    for (uint32_t a = 0; a < 4; ++a) L[a] = a < w ? nd.pos[a + 1] - nd.pos[a] : 0;
#pragma unroll
    for (uint32_t a = 0; a < 4; ++a) {
        e[a] = 0;
        g[a][0] = g[a][1] = g[a][2] = 0;
        if (a >= w) continue;
        // records of the other runs (in order) before run a's last record
        const uint32_t b0 = a == 0 ? 1 : 0, b1 = a <= 1 ? 2 : 1, b2 = a == 3 ? 2 : 3;
        const K y = src[(uint64_t)nd.pos[a + 1] - 1];
        cnt3(src + nd.pos[b0], src + nd.pos[b1], src + nd.pos[b2 < w ? b2 : 0], L[b0],
                       b1 < w ? L[b1] : 0, b2 < w ? L[b2] : 0, b0 < a, b1 < a, b2 < a, w - 1, y, g[a]);
        e[a] = L[a] - 1 + g[a][0] + (w > 2 ? g[a][1] : 0) + (w > 3 ? g[a][2] : 0);
    }
    if (w == 2) {
        if (variant == 1 && L[0] > L[1]) {
            // backward: first records' positions, f0 = run 1 before run 0's first
            // record (strictly smaller), f1 = run 0 not after run 1's first (<=)
            uint32_t f[3];
            cnt3(src + nd.pos[1], src, src, L[1], 0, 0, false, false, false, 1, src[nd.pos[0]], f);
            const uint32_t f0 = f[0];
            uint32_t h[3];
            cnt3(src + nd.pos[0], src, src, L[0], 0, 0, true, false, false, 1, src[nd.pos[1]], h);
            const uint32_t f1 = h[0];
            cmp = T - max(f0, f1);
            wr = T - f1;
        } else {
            cmp = min(e[0], e[1]) + 1;
            wr = e[0] + 1;
        }
    } else if (variant == 4) {
        // stages kernels (merges.py:337-545): a tournament over the live runs
        // until the first of them ends, then again over the rest, then a
        // 2-way stage.  In a tournament every output costs its z compare plus
        // the refetch compare of its side when that side holds two runs,
        // except while the other side's pending head is the last record of
        // its run (safe = 0): then the output costs the unfetch + refetch of
        // both sides, 2 + [four] compares; the run-ending output costs none.
        // Merged positions: mpos(c, i) of record i of run c; cnt(x, c) = run c
        // records before run x's last (merged position e[x]).
        auto slot = [](uint32_t c, uint32_t a) { return c < a ? c : c - 1; };
        auto before_last = [&](uint32_t x, uint32_t c) -> uint32_t {
            return c == x ? L[x] - 1 : g[x][slot(c, x)];
        };
        auto mpos = [&](uint32_t c, uint32_t i) -> int64_t {
            const uint32_t b0 = c == 0 ? 1 : 0, b1 = c <= 1 ? 2 : 1, b2 = c == 3 ? 2 : 3;
            uint32_t h[3];
            cnt3(src + nd.pos[b0], src + nd.pos[b1], src + nd.pos[b2 < w ? b2 : 0], L[b0],
                           b1 < w ? L[b1] : 0, b2 < w ? L[b2] : 0, b0 < c, b1 < c, b2 < c, w - 1,
                           src[(uint64_t)nd.pos[c] + i], h);
            return (int64_t)i + h[0] + (w > 2 ? h[1] : 0) + (w > 3 ? h[2] : 0);
        };
        uint32_t alive[4] = {0, 1, 2, 3}, na = w;
        int64_t os = 0;
        int32_t bprev = -1;
        while (na >= 3) {
            const bool four = na == 4;
            uint32_t be = alive[0];
            for (uint32_t i = 1; i < na; ++i) be = e[alive[i]] < e[be] ? alive[i] : be;
            const int64_t oe = e[be];
            cmp += 2 + (four ? 1 : 0) + (uint64_t)(oe - os);
            if (four) {
                cmp += (uint64_t)(oe - os);
            } else {
                for (uint32_t i = 0; i < 2; ++i) {  // left-side outputs in [os, oe)
                    const uint32_t c = alive[i];
                    cmp += before_last(be, c) - (bprev < 0 ? 0u : before_last((uint32_t)bprev, c));
                }
            }
            for (uint32_t i = 0; i < na; ++i) {
                const uint32_t b = alive[i];
                const bool left = i < 2;
                if (!four && !left) continue;  // a right-side pending head costs the same either way
                // q: merged position of the last record of b's side before b's last
                int64_t q = -1;
                if (L[b] >= 2) q = mpos(b, L[b] - 2);
                const int32_t sib = left ? (int32_t)alive[1 - i] : (int32_t)alive[5 - i];
                const uint32_t gc = before_last(b, (uint32_t)sib);
                if (gc >= 1) q = max(q, mpos((uint32_t)sib, gc - 1));
                const int64_t lo = max(q, os - 1), hi = min((int64_t)e[b], oe);
                if (hi > lo + 1) cmp += (uint64_t)(hi - lo - 1);
            }
            uint32_t k2 = 0;  // drop the ended run, keep the order
            for (uint32_t i = 0; i < na; ++i)
                if (alive[i] != be) alive[k2++] = alive[i];
            na = k2;
            bprev = (int32_t)be;
            os = oe + 1;
        }
        if (na == 2) cmp += (uint64_t)(min(e[alive[0]], e[alive[1]]) - os + 1);
    } else {
        const uint32_t MX = max(e[0], e[1]), MY = w == 4 ? max(e[2], e[3]) : e[2];
        // side X outputs before its first run ends: g[0][0] = run 1 before run 0's last
        const uint32_t CX = e[0] < e[1] ? L[0] - 1 + g[0][0] : L[1] - 1 + g[1][0];
        // side Y: g[2][2] = run 3 before run 2's last, g[3][2] = run 2 before run 3's last
        const uint32_t CY = w == 4 ? (e[2] < e[3] ? L[2] - 1 + g[2][2] : L[3] - 1 + g[3][2]) : 0;
        cmp = 1 + (w == 4 ? 1 : 0) + (min(MX, MY) + 1) + CX + CY;
    }
    if (variant != 1) wr = 0;
}

// CountingOrder comparisons of the reference's merge kernels (merges.py:75-334)
// and the written count of merge_2way_copy_smaller (:145-201) for the nodes of
// one stage, from the merged positions e_a of every run's last record (and, for
// a backward copy-smaller merge, of its first records); one warp per node.
// Sentinel compares are not counted (statskit.py:64-67):
//   2-way (sentinel, no-sentinel, copy-smaller forward): min(e0, e1) + 1
//   copy-smaller backward (n1 > n2): T - max(f0, f1)
//   3/4-way tournament: the two first-level compares (one for 3-way), the root
//     compares while both sides hold records, min(MX, MY) + 1, and the refills
//     of a side while both its runs hold records: the side's outputs before its
//     first run ends.
// Variant ids follow ps_variant; 3/4-way nodes of the stages kernels (4): see
// the simulation below.
template <class K>
__global__ void __launch_bounds__(256) merge_counters_kernel(Bufs<K> bufs, const Node* __restrict__ nodes, uint32_t nlo,
                                                             uint32_t nhi, int variant, Summary* sum) {
    pdl_wait();
    const uint32_t idx = nlo + blockIdx.x * 8 + warp_id();
    unsigned long long cmp = 0, wr = 0;
    const Node nd = nodes[idx < nhi ? idx : nlo];
    // big nodes only (the others: merge_counters_small_kernel)
    if (idx < nhi && nd.pos[nd.arity] - nd.pos[0] > COUNT_SMALL) node_counters<K, true>(bufs, nd, variant, cmp, wr);
    if (lane_id() != 0) cmp = wr = 0;
    for (int dd = 16; dd; dd >>= 1) {
        cmp += __shfl_xor_sync(PS_FULL, cmp, dd);
        wr += __shfl_xor_sync(PS_FULL, wr, dd);
    }
    if (lane_id() == 0) {
        if (cmp) atomicAdd(&sum->comparisons, cmp);
        if (wr) atomicAdd(&sum->cs_written, wr);
    }
}

// Nodes of at most COUNT_SMALL records: one thread per node (scalar rank
// searches over runs that are a few cache lines long).
template <class K>
__global__ void __launch_bounds__(256) merge_counters_small_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                   uint32_t nlo, uint32_t nhi, int variant,
                                                                   Summary* sum) {
    pdl_wait();
    const uint32_t idx = nlo + blockIdx.x * 256 + threadIdx.x;
    unsigned long long cmp = 0, wr = 0;
    if (idx < nhi) {
        const Node nd = nodes[idx];
        if (nd.pos[nd.arity] - nd.pos[0] <= COUNT_SMALL) node_counters<K, false>(bufs, nd, variant, cmp, wr);
    }
    for (int dd = 16; dd; dd >>= 1) {
        cmp += __shfl_xor_sync(PS_FULL, cmp, dd);
        wr += __shfl_xor_sync(PS_FULL, wr, dd);
    }
    if (lane_id() == 0) {
        if (cmp) atomicAdd(&sum->comparisons, cmp);
        if (wr) atomicAdd(&sum->cs_written, wr);
    }
}

// Stand-alone partition launch: one warp per chunk of [c0, c1).
template <class K>
__global__ void __launch_bounds__(256) merge_partition_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                              const uint32_t* __restrict__ chunk2node, uint32_t c0,
                                                              uint32_t c1, uint4* __restrict__ cuts) {
    pdl_wait();
    const uint32_t c = c0 + blockIdx.x * 8 + warp_id();
    if (c >= c1) return;
    partition_chunk<K>(bufs, nodes, chunk2node, c, cuts);
}

// Thin partition for stages with many cuts: three lanes per cut (one per other
// run), ten cuts per warp, each lane a plain binary search.  A warp-wide 11-ary
// search reads ~4x the DRAM sectors per search (ten probes per round past the
// shared top of the search tree); once the cuts fill more than one wave of
// warps the stage is bound by those sectors, not by the search depth.
template <class K>
__global__ void __launch_bounds__(256) merge_partition_thin_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                   const uint32_t* __restrict__ chunk2node,
                                                                   uint32_t c0, uint32_t c1,
                                                                   uint4* __restrict__ cuts) {
    pdl_wait();
    const uint32_t lane = lane_id();
    const uint32_t slot = lane / 3, o = lane % 3;  // lanes 30, 31 idle
    const uint32_t c = c0 + (blockIdx.x * 8 + warp_id()) * 10 + slot;
    const bool live = slot < 10 && c < c1;
    uint32_t got = 0, a = 0, j = 0, w = 0, S = 0, q = 1;
    Node nd;
    if (live) {
        nd = nodes[chunk2node[c]];
        q = c - nd.chunk_base;
        if (q > 0) {
            q -= 1;
            w = nd.arity;
            S = node_spacing(nd, cut_cap<K>());
            for (; a < w; ++a) {
                const uint32_t nc = (nd.pos[a + 1] - nd.pos[a] - 1) / S;
                if (q < nc) break;
                q -= nc;
            }
            j = q + 1;
            const K* src = bufs.kb(nd.parity ^ 1);
            const K y = src[(uint64_t)nd.pos[a] + (uint64_t)j * S];
            const uint32_t bb = o + (o >= a ? 1u : 0u);  // the o-th other run
            if (o + 1 < w) {
                const K* run = src + nd.pos[bb];
                const uint32_t len = nd.pos[bb + 1] - nd.pos[bb];
                got = bb < a ? count_pred<K, true>(run, len, y) : count_pred<K, false>(run, len, y);
            }
            q = 1;  // (marks a real cut below)
        } else {
            q = 0;
        }
    }
    // gather the cut's three counts on its first lane
    const uint32_t base = slot * 3 < 32 ? slot * 3 : 0;
    const uint32_t g0 = __shfl_sync(PS_FULL, got, base), g1 = __shfl_sync(PS_FULL, got, base + 1),
                   g2 = __shfl_sync(PS_FULL, got, base + 2);
    if (!live || o != 0) return;
    if (q == 0) {
        cuts[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    const uint32_t gg[3] = {g0, g1, g2};
    uint32_t rk[4] = {0, 0, 0, 0};
    rk[a] = j * S;
    uint32_t mm = j - 1;
#pragma unroll
    for (uint32_t oo = 0; oo < 3; ++oo) {
        if (oo + 1 >= w) break;
        const uint32_t bb = oo + (oo >= a ? 1 : 0);
        rk[bb] = gg[oo];
        mm += gg[oo] ? (gg[oo] - 1) / S : 0;
    }
    cuts[nd.chunk_base + 1 + mm] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP).
PS_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

PS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PS_DEV void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
PS_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
PS_DEV void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
PS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
PS_DEV void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// TMA bulk store smem -> global (bulk async-group), its commit and waits
PS_DEV void tma_store_1d(void* gmem_dst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}
PS_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
PS_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
PS_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (TMA)
PS_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// named barrier 1 over the consumer warps only
#ifndef PS_SLOTS
#define PS_SLOTS 2
#endif
constexpr uint32_t PIPE_SLOTS = PS_SLOTS;  // input slots per CTA (TMA multi-buffering)
template <uint32_t NC>
PS_DEV void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// ---------------------------------------------------------------------------
// Small nodes (size <= SMALL_NODE): one warp per group of G consecutive nodes
// of the batch (G * largest small node <= SMALL_NODE, chosen by the host per
// level), packed into the warp's shared-memory window.  Loads are batched;
// each node is then merged by the warp's lanes with merge-path passes like the
// pipe's (4-way = merge(merge(A,B), merge(C,D)), ties to the left).
constexpr uint32_t SMALL_WARPS = 8;

template <class K>
size_t merge_small_smem_bytes() {
    return (size_t)SMALL_WARPS * SMALL_NODE * (3 * (sizeof(K) + 4) + 1);
}

// outputs [0, la + lb) of merge(A, B) (ties to A) into (okk, ovv), the lanes of
// a warp taking equal consecutive slices (diagonal search, then a serial merge)
template <class K>
PS_DEV void warp_merge2(const K* ak, const int32_t* av, uint32_t la, const K* bk, const int32_t* bv, uint32_t lb,
                        K* okk, int32_t* ovv) {
    const uint32_t lane = lane_id(), tot = la + lb;
    const uint32_t per = (tot + 31) / 32;
    const uint32_t o0 = min(tot, lane * per), o1 = min(tot, o0 + per);
    if (o0 >= o1) return;
    uint32_t lo = o0 > lb ? o0 - lb : 0, hi = o0 < la ? o0 : la;
    while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        const bool le = !(bk[o0 - 1 - m] < ak[m]);
        lo = le ? m + 1 : lo;
        hi = le ? hi : m;
    }
    uint32_t i = lo, j = o0 - lo;
    for (uint32_t o = o0; o < o1; ++o) {
        const bool takeA = i < la && (j >= lb || !(bk[j] < ak[i]));
        okk[o] = takeA ? ak[i] : bk[j];
        ovv[o] = takeA ? av[i] : bv[j];
        i += takeA;
        j += !takeA;
    }
}

template <class K>
__global__ void __launch_bounds__(SMALL_WARPS * 32) merge_small_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                       uint32_t nlo, uint32_t nhi, uint32_t G) {
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    // per node of the group: packed start, global start, run starts (relative), size, parity
    __shared__ uint32_t s_pre[SMALL_WARPS][33];
    __shared__ uint32_t s_p0[SMALL_WARPS][32];
    __shared__ uint32_t s_off[SMALL_WARPS][32][4];
    __shared__ uint8_t s_par[SMALL_WARPS][32];
    const uint32_t warp = warp_id(), lane = lane_id();
    const uint64_t first64 = (uint64_t)nlo + ((uint64_t)blockIdx.x * SMALL_WARPS + warp) * G;
    if (first64 >= nhi) return;
    const uint32_t first = (uint32_t)first64;
    const uint32_t cnt = min(G, nhi - first);
    uint8_t* base = smem + (size_t)warp * SMALL_NODE * (3 * (sizeof(K) + 4) + 1);
    K* sk = reinterpret_cast<K*>(base);
    K* ok = sk + SMALL_NODE;
    K* xk = ok + SMALL_NODE;
    int32_t* sv = reinterpret_cast<int32_t*>(xk + SMALL_NODE);
    int32_t* ov = sv + SMALL_NODE;
    int32_t* xv = ov + SMALL_NODE;
    uint8_t* snid = reinterpret_cast<uint8_t*>(xv + SMALL_NODE);
    uint32_t sz = 0;
    if (lane < cnt) {
        const Node nd = nodes[first + lane];
        const uint32_t w = nd.arity, p0 = nd.pos[0], size = nd.pos[w] - p0;
        if (size <= SMALL_KERNEL_MAX) {  // bigger nodes of the batch belong to the pipe kernel
            sz = size;
            s_p0[warp][lane] = p0;
            s_par[warp][lane] = nd.parity;
#pragma unroll
            for (uint32_t a = 0; a < 4; ++a) s_off[warp][lane][a] = a < w ? nd.pos[a] - p0 : size;
        }
    }
    uint32_t inc = sz;
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(PS_FULL, inc, d);
        if (lane >= (uint32_t)d) inc += y;
    }
    s_pre[warp][lane + 1] = inc;
    if (lane == 0) s_pre[warp][0] = 0;
    const uint32_t total = __shfl_sync(PS_FULL, inc, 31);
    __syncwarp();
    const uint32_t* pre = s_pre[warp];
    if (total > SMALL_NODE) return;  // host chose G too large (cannot happen)
    constexpr uint32_t PER = SMALL_NODE / 32;
    {
        K kk[PER];
        int32_t vv[PER];
#pragma unroll
        for (uint32_t u = 0; u < PER; ++u) {
            const uint32_t i = lane + 32 * u;
            if (i < total) {
                uint32_t lo = 0, hi = cnt;  // pre[lo] <= i < pre[hi]
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (pre[mid] <= i) lo = mid; else hi = mid;
                }
                snid[i] = (uint8_t)lo;
                const uint64_t p = (uint64_t)s_p0[warp][lo] + (i - pre[lo]);
                const uint32_t sp = s_par[warp][lo] ^ 1u;
                kk[u] = bufs.kb(sp)[p];
                vv[u] = bufs.vb(sp)[p];
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < PER; ++u) {
            const uint32_t i = lane + 32 * u;
            if (i < total) {
                sk[i] = kk[u];
                sv[i] = vv[u];
            }
        }
    }
    __syncwarp();
    for (uint32_t jn = 0; jn < cnt; ++jn) {
        const uint32_t nb = pre[jn], S = pre[jn + 1] - nb;
        if (S == 0) continue;  // a big node of the batch
        const uint32_t* off = s_off[warp][jn];
        const uint32_t o1 = off[1], o2 = off[2], o3 = off[3];
        const K* k0 = sk + nb;
        const int32_t* v0 = sv + nb;
        if (o2 >= S) {  // 2-way
            warp_merge2<K>(k0, v0, o1, k0 + o1, v0 + o1, S - o1, ok + nb, ov + nb);
        } else {  // 3/4-way: X = A+B, Y = C+D (D empty for 3-way), then X+Y
            warp_merge2<K>(k0, v0, o1, k0 + o1, v0 + o1, o2 - o1, xk + nb, xv + nb);
            warp_merge2<K>(k0 + o2, v0 + o2, o3 - o2, k0 + o3, v0 + o3, S - o3, xk + nb + o2, xv + nb + o2);
            __syncwarp();
            warp_merge2<K>(xk + nb, xv + nb, o2, xk + nb + o2, xv + nb + o2, S - o2, ok + nb, ov + nb);
        }
        __syncwarp();
    }
#pragma unroll 4
    for (uint32_t i = lane; i < total; i += 32) {
        const uint32_t j = snid[i];
        const uint64_t p = (uint64_t)s_p0[warp][j] + (i - pre[j]);
        bufs.kb(s_par[warp][j])[p] = ok[i];
        bufs.vb(s_par[warp][j])[p] = ov[i];
    }
}

// 4- or 8-byte asynchronous global -> shared copy (LDGSTS)
template <class T>
PS_DEV void cp_async_small(T* smem_dst, const T* gmem_src) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4 or 8 bytes");
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gmem_src), "n"(sizeof(T))
                 : "memory");
}

// Merge-path outputs [o, oe) of merge(A, B) (ties to A) into (ok, ov)[o...]:
// diagonal search, then one record per step with the heads in registers.  A
// read one past a run's end stays inside the CTA's shared memory.
template <class K>
PS_DEV void smem_merge_piece(const K* ak, const int32_t* av, uint32_t la, const K* bk, const int32_t* bv,
                           uint32_t lb, uint32_t o, uint32_t oe, K* ok, int32_t* ov) {
    uint32_t lo = o > lb ? o - lb : 0, hi = o < la ? o : la;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const bool le = !(bk[o - 1 - mid] < ak[mid]);
        lo = le ? mid + 1 : lo;
        hi = le ? hi : mid;
    }
    uint32_t i = lo, j = o - lo;
    K a = ak[i], b = bk[j];
    for (; o < oe; ++o) {
        const bool ta = i < la && (j >= lb || !(b < a));
        ok[o] = ta ? a : b;
        ov[o] = *(ta ? av + i : bv + j);
        i += ta;
        j += !ta;
        const K nk = *(ta ? ak + i : bk + j);
        a = ta ? nk : a;
        b = ta ? b : nk;
    }
}


// ---------------------------------------------------------------------------
// Mid-size nodes (<= SMALL_KERNEL_MAX records): a CTA per batch of G
// consecutive nodes of the stage (G * largest <= MID_CAP), packed into shared
// memory with asynchronous copies (a warp per node, coalesced), merged by
// the pipe's two passes with VT consecutive outputs per thread (odd VT:
// conflict-free stores) -- X = merge(A,B), Y = merge(C,D) into buffer 1,
// then merge(X,Y) back into buffer 0 (2-way nodes: merge(A,B) into buffer 1,
// which their first pass leaves unused) -- and stored a warp per node.  Two
// buffers, so three CTAs fit an SM.  Ties go to the lower run in every pass
// (merges.py:204-334).
constexpr uint32_t MID_THREADS = 256;
constexpr uint32_t MID_MAXG = 64;
template <class K>
PS_DEV __host__ constexpr uint32_t mid_vt() {
    return sizeof(K) == 4 ? 15u : 9u;
}
template <class K>
PS_DEV __host__ constexpr uint32_t mid_cap() {
    return mid_vt<K>() * MID_THREADS;
}
template <class K>
PS_DEV __host__ constexpr size_t mid_smem_bytes() {  // two SoA record buffers
    return 2 * (size_t)mid_cap<K>() * (sizeof(K) + 4) + 128;
}
// nodes per CTA for a stage whose largest small node has `maxsz` records
template <class K>
inline uint32_t mid_group(uint32_t maxsz) {
    const uint32_t g = maxsz ? mid_cap<K>() / maxsz : MID_MAXG;
    return g < 1 ? 1 : (g > MID_MAXG ? MID_MAXG : g);
}

template <class K>
__global__ void __launch_bounds__(MID_THREADS) merge_mid_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                               uint32_t nlo, uint32_t nhi, uint32_t G) {
    pdl_wait();
    constexpr uint32_t CAP = mid_cap<K>(), VT = mid_vt<K>();
    extern __shared__ __align__(128) uint8_t smem[];
    auto KB = [&](uint32_t q) { return reinterpret_cast<K*>(smem + (size_t)q * CAP * (sizeof(K) + 4)); };
    auto VB = [&](uint32_t q) {
        return reinterpret_cast<int32_t*>(smem + (size_t)q * CAP * (sizeof(K) + 4) + (size_t)CAP * sizeof(K));
    };
    __shared__ uint32_t s_pre[MID_MAXG + 1], s_p0[MID_MAXG], s_rel[MID_MAXG][4];
    __shared__ uint8_t s_par[MID_MAXG], s_w[MID_MAXG];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t first64 = (uint64_t)nlo + (uint64_t)blockIdx.x * G;
    if (first64 >= nhi) return;
    const uint32_t first = (uint32_t)first64, cnt = min(G, nhi - first);
    if (warp == 0) {
        uint32_t sz = 0;
        for (uint32_t base = 0; base < cnt; base += 32) {  // (cnt <= 64: two rounds)
            const uint32_t j = base + lane;
            uint32_t size = 0;
            if (j < cnt) {
                const Node nd = nodes[first + j];
                const uint32_t w = nd.arity, p0 = nd.pos[0];
                size = nd.pos[w] - p0;
                if (size > SMALL_KERNEL_MAX) size = 0;  // a big node of the stage: the pipe's
                s_p0[j] = p0;
                s_par[j] = nd.parity;
                s_w[j] = (uint8_t)w;
#pragma unroll
                for (uint32_t a = 0; a < 4; ++a) s_rel[j][a] = a + 1 <= w ? nd.pos[a + 1] - p0 : size;
            }
            uint32_t inc = size;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(PS_FULL, inc, d);
                if (lane >= (uint32_t)d) inc += y;
            }
            if (j < cnt) s_pre[j + 1] = sz + inc;
            if (base == 0 && lane == 0) s_pre[0] = 0;
            sz += __shfl_sync(PS_FULL, inc, 31);
        }
    }
    __syncthreads();
    const uint32_t total = s_pre[cnt];
    if (total == 0) return;
    // ---- load: a warp per node, records of buffer parity ^ 1 into buffer 0
    for (uint32_t j = warp; j < cnt; j += MID_THREADS / 32) {
        const uint32_t o = s_pre[j], size = s_pre[j + 1] - o;
        if (!size) continue;
        const uint32_t sp = s_par[j] ^ 1u;
        const K* gk = bufs.kb(sp) + s_p0[j];
        const int32_t* gv = bufs.vb(sp) + s_p0[j];
        for (uint32_t t = lane; t < size; t += 32) {
            cp_async_small(KB(0) + o + t, gk + t);
            cp_async_small(VB(0) + o + t, gv + t);
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // ---- two passes over the packed nodes, VT outputs per thread (pieces may
    //      span nodes and X / Y halves)
    for (uint32_t pass = 0; pass < 2; ++pass) {
        for (uint32_t o = tid * VT, oe = min(o + VT, total); o < oe;) {
            uint32_t lo = 0, hi = cnt;  // last node with s_pre <= o
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_pre[mid] <= o)
                    lo = mid;
                else
                    hi = mid;
            }
            const uint32_t j = lo, nb = s_pre[j], ne = s_pre[j + 1], w = s_w[j];
            const uint32_t r1 = s_rel[j][0], r2 = s_rel[j][1], r3 = s_rel[j][2];
            const uint32_t q = o - nb;
            if (pass == 0) {
                if (w < 3) {  // 2-way nodes merge in pass 2
                    o = min(oe, ne);
                    continue;
                }
                if (q < r2) {  // X = merge(A, B)
                    const uint32_t pe = min(oe, nb + r2);
                    smem_merge_piece<K>(KB(0) + nb, VB(0) + nb, r1, KB(0) + nb + r1, VB(0) + nb + r1, r2 - r1, q,
                                        pe - nb, KB(1) + nb, VB(1) + nb);
                    o = pe;
                } else {  // Y = merge(C, D) (3-way: C)
                    const uint32_t pe = min(oe, ne), r4 = ne - nb;
                    const uint32_t c1 = w == 4 ? r3 : r4;
                    smem_merge_piece<K>(KB(0) + nb + r2, VB(0) + nb + r2, c1 - r2, KB(0) + nb + c1, VB(0) + nb + c1,
                                        r4 - c1, q - r2, pe - nb - r2, KB(1) + nb + r2, VB(1) + nb + r2);
                    o = pe;
                }
            } else {
                const uint32_t pe = min(oe, ne), r4 = ne - nb;
                const uint32_t src = w >= 3 ? 1u : 0u, m = w >= 3 ? r2 : r1;
                smem_merge_piece<K>(KB(src) + nb, VB(src) + nb, m, KB(src) + nb + m, VB(src) + nb + m, r4 - m, q,
                                    pe - nb, KB(src ^ 1u) + nb, VB(src ^ 1u) + nb);
                o = pe;
            }
        }
        __syncthreads();
    }
    // ---- store: a warp per node
    for (uint32_t j = warp; j < cnt; j += MID_THREADS / 32) {
        const uint32_t o = s_pre[j], size = s_pre[j + 1] - o;
        if (!size) continue;
        K* dk = bufs.kb(s_par[j]) + s_p0[j];
        int32_t* dv = bufs.vb(s_par[j]) + s_p0[j];
        const uint32_t q = s_w[j] >= 3 ? 0u : 1u;  // the buffer its second pass wrote
        const K* sk = KB(q) + o;
        const int32_t* sv = VB(q) + o;
        for (uint32_t t = lane; t < size; t += 32) {
            dk[t] = sk[t];
            dv[t] = sv[t];
        }
    }
}

// ---------------------------------------------------------------------------
// Tiny nodes (every small node of the stage <= TINY records): one node per
// thread.  A warp stages its 32 nodes' keys as rows of TINY+1 elements (odd
// stride: the lanes' row-wise accesses spread over the banks), each lane then
// runs the node's stable k-way tournament sequentially (ties to the lower run,
// as merges.py:229-269) and records the source offset of every output; the
// store pass gathers keys from the rows and payloads from global memory, one
// coalesced store per node and row segment.  No merge-path searches, no
// per-node barrier: ~15 instructions per output and 32 independent merges per
// warp, where the warp-per-node kernel spends most of its time in diagonal
// searches for two outputs per lane.

template <class K, uint32_t TINY>
struct TinyCfg {
    static constexpr uint32_t RK = TINY + 1;                      // key / payload row stride (elements)
    static constexpr uint32_t RI = (TINY + 4) & ~3u;              // offset row stride (bytes)
    static constexpr uint32_t KEY_BYTES = align16c(32 * RK * (uint32_t)sizeof(K));
    static constexpr uint32_t VAL_BYTES = align16c(32 * RK * 4u);
    static constexpr uint32_t WARP_BYTES = KEY_BYTES + VAL_BYTES + align16c(32 * RI);
    static constexpr uint32_t WARPS = cmax(1u, (uint32_t)(112 * 1024) / WARP_BYTES);  // two CTAs per SM
};
template <class K, uint32_t TINY>
size_t merge_tiny_smem_bytes() {
    return (size_t)TinyCfg<K, TINY>::WARPS * TinyCfg<K, TINY>::WARP_BYTES;
}

// With `sum` (merge variants 2way, 2way-nosentinel, 4way), each lane also
// counts its node's CountingOrder comparisons from the positions its
// tournament observes -- where every run's last record lands (e_a) and where
// within its side (CX, CY) -- by node_counters' closed forms, so the stage
// needs no separate counters launch.
template <class K, uint32_t TINY>
__global__ void __launch_bounds__(TinyCfg<K, TINY>::WARPS * 32) merge_tiny_kernel(Bufs<K> bufs,
                                                                                  const Node* __restrict__ nodes,
                                                                                  uint32_t nlo, uint32_t nhi,
                                                                                  Summary* __restrict__ sum) {
    static_assert(TINY <= 256, "offsets are bytes");
    using C = TinyCfg<K, TINY>;
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t warp = warp_id(), lane = lane_id();
    uint8_t* wbase = smem + (size_t)warp * C::WARP_BYTES;
    K* rows = reinterpret_cast<K*>(wbase);
    int32_t* vrows = reinterpret_cast<int32_t*>(wbase + C::KEY_BYTES);
    uint8_t* outi = wbase + C::KEY_BYTES + C::VAL_BYTES;
    const uint64_t i64 = (uint64_t)nlo + ((uint64_t)blockIdx.x * C::WARPS + warp) * 32 + lane;
    uint32_t p0 = 0, T = 0, par = 0, w = 0;
    uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0;  // run ends (row offsets); run a starts at e_{a-1}
    if (i64 < nhi) {
        const Node nd = nodes[(uint32_t)i64];
        w = nd.arity;
        p0 = nd.pos[0];
        const uint32_t size = nd.pos[w] - p0;
        if (size <= TINY) {  // (bigger: the pipe kernel's)
            T = size;
            par = nd.parity;
            e0 = nd.pos[1] - p0;
            e1 = w > 1 ? nd.pos[2] - p0 : T;
            e2 = w > 2 ? nd.pos[3] - p0 : T;
            e3 = T;
        }
    }
    if (__ballot_sync(PS_FULL, T != 0) == 0) return;
    // ---- rows: every node's keys and payloads (buffer parity ^ 1) with
    // asynchronous copies, all in flight at once, coalesced per node ----
    for (uint32_t j = 0; j < 32; ++j) {  // node-major: no division, empty tails skipped
        const uint32_t tj = __shfl_sync(PS_FULL, T, j);
        if (tj == 0) continue;
        const uint32_t sp = __shfl_sync(PS_FULL, par, j) ^ 1u, bj = __shfl_sync(PS_FULL, p0, j);
        const K* gk = bufs.kb(sp) + bj;
        const int32_t* gv = bufs.vb(sp) + bj;
        K* rk = rows + j * C::RK;
        int32_t* rv = vrows + j * C::RK;
        for (uint32_t t = lane; t < tj; t += 32) {
            cp_async_small(rk + t, gk + t);
            cp_async_small(rv + t, gv + t);
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    // ---- the lane's tournament ----
    unsigned long long cmp = 0;
    auto tournament = [&](auto count) {
        constexpr bool COUNT = decltype(count)::value;
        const K* row = rows + lane * C::RK;
        uint8_t* oi = outi + lane * C::RI;
        uint32_t i0 = 0, i1 = e0, i2 = e1, i3 = e2;
        K h0 = row[0], h1 = row[i1], h2 = row[i2], h3 = row[i3];
        uint32_t E0 = 0, E1 = 0, E2 = 0, E3 = 0, P0 = 0, P1 = 0, P2 = 0, P3 = 0, xo = 0, yo = 0;
        for (uint32_t o = 0; o < T; ++o) {
            const bool v0 = i0 < e0, v1 = i1 < e1, v2 = i2 < e2, v3 = i3 < e3;
            const bool b1 = v1 && (!v0 || h1 < h0);  // ties to the lower run
            const bool b3 = v3 && (!v2 || h3 < h2);
            const K kl = b1 ? h1 : h0, kr = b3 ? h3 : h2;
            const bool vl = v0 || v1, vr = v2 || v3;
            const bool right = vr && (!vl || kr < kl);
            const uint32_t src = right ? (b3 ? i3 : i2) : (b1 ? i1 : i0);
            oi[o] = (uint8_t)src;
            const K nk = row[src + 1];  // (one past a run reads its neighbour or the row's slack)
            const bool s0 = !right && !b1, s1 = !right && b1, s2 = right && !b3, s3 = right && b3;
            if (COUNT) {  // the last record of a run: its merged position and its side position
                const uint32_t side = right ? yo : xo;
                if (s0 && src + 1 == e0) { E0 = o; P0 = side; }
                if (s1 && src + 1 == e1) { E1 = o; P1 = side; }
                if (s2 && src + 1 == e2) { E2 = o; P2 = side; }
                if (s3 && src + 1 == e3) { E3 = o; P3 = side; }
                xo += !right;
                yo += right;
            }
            i0 += s0;
            i1 += s1;
            i2 += s2;
            i3 += s3;
            h0 = s0 ? nk : h0;
            h1 = s1 ? nk : h1;
            h2 = s2 ? nk : h2;
            h3 = s3 ? nk : h3;
        }
        if (COUNT) {
            if (w == 2) {
                cmp = min(E0, E1) + 1;  // merges.py:75-142 (sentinel compares uncounted)
            } else {                    // merges.py:204-334: node_counters' 3/4-way closed form
                const uint32_t MX = max(E0, E1), MY = w == 4 ? max(E2, E3) : E2;
                const uint32_t CX = E0 < E1 ? P0 : P1;
                const uint32_t CY = w == 4 ? (E2 < E3 ? P2 : P3) : 0u;
                cmp = 1 + (w == 4 ? 1 : 0) + (min(MX, MY) + 1) + CX + CY;
            }
        }
    };
    if (T) {
        if (sum)
            tournament(std::true_type{});
        else
            tournament(std::false_type{});
    }
    if (sum) {
        for (int dd = 16; dd; dd >>= 1) cmp += __shfl_xor_sync(PS_FULL, cmp, dd);
        if (lane == 0 && cmp) atomicAdd(&sum->comparisons, cmp);
    }
    __syncwarp();
    // ---- stores: keys and payloads from the rows, one coalesced store per node ----
    for (uint32_t j = 0; j < 32; ++j) {
        const uint32_t tj = __shfl_sync(PS_FULL, T, j);
        if (tj == 0) continue;
        const uint32_t pj = __shfl_sync(PS_FULL, par, j), bj = __shfl_sync(PS_FULL, p0, j);
        K* dk = bufs.kb(pj) + bj;
        int32_t* dv = bufs.vb(pj) + bj;
        const K* rk = rows + j * C::RK;
        const int32_t* rv = vrows + j * C::RK;
        const uint8_t* oj = outi + j * C::RI;
        for (uint32_t t = lane; t < tj; t += 32) {
            const uint32_t sidx = oj[t];
            dk[t] = rk[sidx];
            dv[t] = rv[sidx];
        }
    }
}

// nodes per warp for a batch whose largest small node has `maxsz` records
inline uint32_t small_group(uint32_t maxsz) {
    if (maxsz == 0) return 1;
    const uint32_t g = SMALL_NODE / maxsz;
    return g < 1 ? 1 : (g > 32 ? 32 : g);
}

// ---------------------------------------------------------------------------
// Optional clock64 phase counters of the pipe kernel (build with -DPS_PIPE_TIMING)
#ifdef PS_PIPE_TIMING
__device__ unsigned long long g_pipe_tim[40];
// per-CTA globaltimer stamps of the last pipe launch: start, after the fused
// partition, first unit ready (consumer 0), consumers done, producer done
__device__ unsigned long long g_cta_tim[1024][5];
PS_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define PT_CTA(idx) \
    if (blockIdx.x < 1024) g_cta_tim[blockIdx.x][idx] = gtimer();
#define PT_START(on) long long _pt0 = clock64(); const bool _pton = (on);
#define PT_MARK(idx)                                                         \
    if (_pton) {                                                             \
        const long long _t = clock64();                                      \
        atomicAdd(&g_pipe_tim[idx], (unsigned long long)(_t - _pt0));        \
        _pt0 = _t;                                                           \
    }
#define PT_COUNT(idx) \
    if (_pton) atomicAdd(&g_pipe_tim[idx], 1ull);
// per-consumer-warp work time since the unit started (before the barrier)
#define PT_USTART long long _ptu = clock64();
#define PT_WARP(idx) \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_pipe_tim[(idx) + ((threadIdx.x - 32) >> 5)], clock64() - _ptu);
#else
#define PT_USTART
#define PT_WARP(idx)
#define PT_CTA(idx)
#define PT_START(on)
#define PT_MARK(idx)
#define PT_COUNT(idx)
#endif

// ---------------------------------------------------------------------------
// Big-node chunks: persistent, warp-specialized, TMA-bulk double-buffered.


// (key, value) record in shared memory: 8 bytes for 4-byte keys, 16 for 8-byte
template <class K>
struct alignas(sizeof(K) == 4 ? 8 : 16) Rec {
    K k;
    int32_t v;
};


// Units hold up to pipe_maxseg<K>() <= MAXSEG segments; a segment is a contiguous chunk range of
// one node (a unit of one segment may be several chunks of one node; several
// segments pack consecutive whole small-to-mid nodes or chunk ranges).
constexpr uint32_t MAXSEG = 32;
// PS_XR2=1: two first-pass scratch buffers used alternately, so a unit's end
// needs no CTA barrier (needs fewer consumers to fit shared memory)
#ifndef PS_XR2
#define PS_XR2 0
#endif
// PS_BULK_STORE=1: single-segment 3/4-way units leave through TMA bulk stores
// issued by the producer warp (the consumers only write SoA outputs to the slot)
#ifndef PS_BULK_STORE
#define PS_BULK_STORE 1
#endif
// PS_SOA_X=1: the first pass writes X || Y as SoA (a key array and a value
// array) instead of (key, value) records, so the second pass's diagonal probes
// read 4- or 8-byte keys at unit stride (fewer bank conflicts than key fields
// of 8- or 16-byte records)
#ifndef PS_SOA_X
#define PS_SOA_X 1
#endif

template <class K>
struct PipeLayout {
    static constexpr uint32_t CAP = pipe_cap<K>();
    static constexpr uint32_t PADN = (CAP + pipe_vt<K>() + 16 + 3) & ~3u;  // record capacity (+ over-read / don't-care slack)
    static_assert(PADN >= CAP + pipe_vt<K>() - 1, "record slack must hold a thread's don't-care outputs");
    static constexpr uint32_t RECB = (uint32_t)sizeof(Rec<K>);
    // slot = TMA landing zone of the key windows + value windows of all segments
    // (SoA, <= 31 bytes of 16-byte alignment slack per window), and afterwards
    // the records of the last pass
    static constexpr uint32_t KEY_BYTES = align16c(CAP * (uint32_t)sizeof(K)) + pipe_maxseg<K>() * MAX_WAY * 32u;
    static constexpr uint32_t VAL_BYTES = align16c(CAP * 4u) + pipe_maxseg<K>() * MAX_WAY * 32u;
    static constexpr uint32_t SLOT = align16c(cmax(KEY_BYTES + VAL_BYTES, PADN * RECB));
    // scratch: first-pass records X || Y of every segment (or the 2-way output)
    static constexpr uint32_t SCRATCH = align16c(PADN * RECB);
    // SoA scratch (PS_SOA_X): keys at 0, values at XV
    static constexpr uint32_t XV = align16c(PADN * (uint32_t)sizeof(K));
    static_assert(XV + PADN * 4 <= SCRATCH, "SoA scratch must fit");
    static constexpr uint32_t NXR = PS_XR2 ? 2 : 1;  // scratch buffers (2: alternate by unit)
    // SoA output of a bulk-stored unit inside its slot: keys at 0, values at OV
    static constexpr uint32_t EPK = 16 / (uint32_t)sizeof(K);  // keys per 16 bytes
    static constexpr uint32_t OV = align16c((PADN + 4) * (uint32_t)sizeof(K));
    static_assert(OV + (PADN + 4) * 4 <= SLOT, "SoA outputs must fit the slot");
};

struct PipeSeg {
    uint64_t out;  // global element index of the segment's first output
    uint32_t koff[4], voff[4], len[4];  // window byte offsets in the slot, lengths (0 past the arity)
    uint32_t w, par, T, lx;             // arity, output parity, records, |X| = len[0] + len[1]
};

struct PipeDesc {
    uint32_t nseg, done, end1, end2;
    uint32_t s1[2 * MAXSEG];  // pass-1 layout: X of segment s at s1[2s], Y at s1[2s+1] (VT-aligned)
    uint32_t s2[MAXSEG];      // pass-2 layout: output of segment s at s2[s] (VT-aligned)
    PipeSeg seg[MAXSEG];
};

template <class K>
size_t merge_pipe_smem_bytes() {
    return PIPE_SLOTS * (size_t)PipeLayout<K>::SLOT + PipeLayout<K>::NXR * (size_t)PipeLayout<K>::SCRATCH +
           PIPE_SLOTS * sizeof(PipeDesc) + 64;
}

// Merge-path cursors.  WinCur merges two TMA-landed SoA windows, RecCur two padded record runs;
// ties always go to the A side.  Outputs go to padded records out[base + o].
template <class K>
struct WinCur {
    const K *ak, *bk;
    const int32_t *av, *bv;
    uint32_t la, lb, i, j, o, oe, base;
    K a, b;
    // one-past-the-end reads stay inside shared memory (the next window, the
    // slot's alignment slack or the padded capacity), so no clamping is needed
    PS_DEV uint32_t ca(uint32_t x) const { return x; }
    PS_DEV uint32_t cb(uint32_t x) const { return x; }
    PS_DEV K keyA(uint32_t x) const { return ak[ca(x)]; }
    PS_DEV K keyB(uint32_t x) const { return bk[cb(x)]; }
    PS_DEV void heads() {
        a = ak[ca(i)];
        b = bk[cb(j)];
    }
    // one output to outp[t]; no end check (see single_merge)
    PS_DEV void step(Rec<K>* outp, uint32_t t) {
        const bool takeA = i < la && (j >= lb || !(b < a));
        Rec<K> r;
        r.k = takeA ? a : b;
        r.v = *(takeA ? av + i : bv + j);
        outp[t] = r;
        i += takeA;
        j += !takeA;
        const K nk = *(takeA ? ak + ca(i) : bk + cb(j));
        a = takeA ? nk : a;
        b = takeA ? b : nk;
    }
};

template <class K>
struct RecCur {
    const Rec<K>* r;
    uint32_t offa, offb, la, lb, i, j, o, oe, base;
    Rec<K> a, b;
    PS_DEV uint32_t ia(uint32_t x) const { return (offa + x); }
    PS_DEV uint32_t ib(uint32_t x) const { return (offb + x); }
    PS_DEV K keyA(uint32_t x) const { return r[ia(x)].k; }
    PS_DEV K keyB(uint32_t x) const { return r[ib(x)].k; }
    PS_DEV void heads() {
        a = r[ia(i)];
        b = r[ib(j)];
    }
    PS_DEV void step(Rec<K>* outp, uint32_t t) {
        const bool takeA = i < la && (j >= lb || !(b.k < a.k));
        outp[t] = takeA ? a : b;
        i += takeA;
        j += !takeA;
        const Rec<K> nx = r[takeA ? ia(i) : ib(j)];
        a = takeA ? nx : a;
        b = takeA ? b : nx;
    }
};

// One cursor: diagonal search, then the serial branch-free merge of exactly
// VT steps (fully unrolled, no per-step end check).  A thread with fewer than
// VT outputs (the last one of a merge) writes up to VT - 1 don't-care records
// past its range: they land in the slack between X and Y (Y starts VT-aligned)
// or past the unit's last output, inside the record capacity (PADN >= CAP + VT
// - 1), and are never read.  Its extra reads stay inside shared memory too.
// Merge-path diagonal: # of A among the first c.o outputs (ties to A).  With
// PS_SEARCH4 the first rounds probe three points at once (4-ary), halving the
// dependent shared-memory round trips for twice the probes.
#ifndef PS_SEARCH4
#define PS_SEARCH4 0
#endif
template <class C>
PS_DEV uint32_t diag_search(const C& c) {
    uint32_t lo = c.o > c.lb ? c.o - c.lb : 0, hi = c.o < c.la ? c.o : c.la;
    if (PS_SEARCH4) {
        while (hi - lo > 3) {
            const uint32_t span = hi - lo;
            const uint32_t q1 = lo + (span >> 2), q2 = lo + (span >> 1), q3 = lo + ((3 * span) >> 2);
            const bool p1 = !(c.keyB(c.o - 1 - q1) < c.keyA(q1));
            const bool p2 = !(c.keyB(c.o - 1 - q2) < c.keyA(q2));
            const bool p3 = !(c.keyB(c.o - 1 - q3) < c.keyA(q3));
            const uint32_t nlo = p3 ? q3 + 1 : p2 ? q2 + 1 : p1 ? q1 + 1 : lo;
            const uint32_t nhi = p3 ? hi : p2 ? q3 : p1 ? q2 : q1;
            lo = nlo;
            hi = nhi;
        }
    }
    while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        const bool le = !(c.keyB(c.o - 1 - m) < c.keyA(m));
        lo = le ? m + 1 : lo;
        hi = le ? hi : m;
    }
    return lo;
}

// PS_LOADS_FIRST=1: the merge step of a WinCur issues its two shared-memory
// loads (the value of the record it emits and the key behind it, one address
// register: the new head is the next element of the run just consumed) before
// its two stores.  The stores may alias the loads as far as the compiler knows,
// so source order is issue order: with the value load, its store and only then
// the key load (the order until round 2) every step waits for two dependent
// shared-memory round trips instead of one.
#ifndef PS_LOADS_FIRST
#define PS_LOADS_FIRST 1
#endif

// One merge chain over two SoA windows, heads in registers, pointer cursors.
// 4-byte keys: a value sits at a fixed byte offset dv from its key in both
// windows (TMA slot: KEY_BYTES, windows share their 16-byte phases; scratch:
// XV), so one selected pointer serves both loads.
template <class K>
struct MChain {
    const K *pa, *pb, *ea, *eb;
    const int32_t *va, *vb;  // 8-byte keys: value cursors
    K a, b;
    PS_DEV void init(const WinCur<K>& c, uint32_t i, uint32_t j) {
        pa = c.ak + i;
        pb = c.bk + j;
        ea = c.ak + c.la;
        eb = c.bk + c.lb;
        va = c.av + i;
        vb = c.bv + j;
        a = *pa;
        b = *pb;
    }
    // emits one record: returns its key, loads its value into v
    PS_DEV K step(ptrdiff_t dv, int32_t& v) {
        const bool tA = pa < ea && (pb >= eb || !(b < a));
        const K k = tA ? a : b;
        const K* p = tA ? pa : pb;
        const K nk = p[1];
        if constexpr (sizeof(K) == 4) {
            v = *reinterpret_cast<const int32_t*>(reinterpret_cast<const uint8_t*>(p) + dv);
        } else {
            v = *(tA ? va : vb);
            va += tA;
            vb += !tA;
        }
        pa = tA ? p + 1 : pa;
        pb = tA ? pb : p + 1;
        a = tA ? nk : a;
        b = tA ? b : nk;
        return k;
    }
};

// The VT outputs [o, o + VT) of a WinCur merge, written by put(t, key, value)
// with t relative to o (a thread with fewer outputs writes don't-care records,
// see single_merge).
template <class K, class Put>
PS_DEV void win_merge(const WinCur<K>& c, Put put) {
    const ptrdiff_t dv = reinterpret_cast<const uint8_t*>(c.av) - reinterpret_cast<const uint8_t*>(c.ak);
    const uint32_t i0 = diag_search(c);
    MChain<K> A;
    A.init(c, i0, c.o - i0);
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) {
        int32_t v;
        const K k = A.step(dv, v);
        put(t, k, v);
    }
}

template <class K>
PS_DEV void single_merge(WinCur<K>& c, Rec<K>* out) {
    if (c.o >= c.oe) return;
    if (PS_LOADS_FIRST) {
        Rec<K>* outp = out + c.base + c.o;
        win_merge<K>(c, [&](uint32_t t, K k, int32_t v) {
            Rec<K> r;
            r.k = k;
            r.v = v;
            outp[t] = r;
        });
        return;
    }
    const uint32_t lo = diag_search(c);
    c.i = lo;
    c.j = c.o - lo;
    c.heads();
    Rec<K>* outp = out + c.base + c.o;
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) c.step(outp, t);
}

template <class C, class K>
PS_DEV void single_merge(C& c, Rec<K>* out) {
    if (c.o >= c.oe) return;
    const uint32_t lo = diag_search(c);
    c.i = lo;
    c.j = c.o - lo;
    c.heads();
    Rec<K>* outp = out + c.base + c.o;
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) c.step(outp, t);
}

// Pass 2 into SoA outputs (keys[o], vals[o]) for the bulk-store path.
template <class K>
PS_DEV void single_merge_soa(RecCur<K>& c, K* outk, int32_t* outv) {
    if (c.o >= c.oe) return;
    const uint32_t lo = diag_search(c);
    c.i = lo;
    c.j = c.o - lo;
    c.heads();
    K* ok = outk + c.o;
    int32_t* ov = outv + c.o;
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) {
        const bool takeA = c.i < c.la && (c.j >= c.lb || !(c.b.k < c.a.k));
        const Rec<K> r = takeA ? c.a : c.b;
        ok[t] = r.k;
        ov[t] = r.v;
        c.i += takeA;
        c.j += !takeA;
        const Rec<K> nx = c.r[takeA ? c.ia(c.i) : c.ib(c.j)];
        c.a = takeA ? nx : c.a;
        c.b = takeA ? c.b : nx;
    }
}

// Pass into SoA outputs from SoA inputs (keys ok[t], values ov[t]).
template <class K>
PS_DEV void single_merge_soa(WinCur<K>& c, K* outk, int32_t* outv) {
    if (c.o >= c.oe) return;
    if (PS_LOADS_FIRST) {
        K* ok2 = outk + c.base + c.o;
        int32_t* ov2 = outv + c.base + c.o;
        win_merge<K>(c, [&](uint32_t t, K k, int32_t v) {
            ok2[t] = k;
            ov2[t] = v;
        });
        return;
    }
    const uint32_t lo = diag_search(c);
    c.i = lo;
    c.j = c.o - lo;
    c.heads();
    K* ok = outk + c.base + c.o;
    int32_t* ov = outv + c.base + c.o;
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) {
        const bool takeA = c.i < c.la && (c.j >= c.lb || !(c.b < c.a));
        ok[t] = takeA ? c.a : c.b;
        ov[t] = *(takeA ? c.av + c.i : c.bv + c.j);
        c.i += takeA;
        c.j += !takeA;
        const K nk = *(takeA ? c.ak + c.i : c.bk + c.j);
        c.a = takeA ? nk : c.a;
        c.b = takeA ? c.b : nk;
    }
}

// A TMA-landed input window: SoA keys / values, unpadded.
template <class K>
struct Win {
    const K* k;
    const int32_t* v;
    uint32_t len;
};

// largest p in [0, n) with tab[p] <= x (tab ascending, tab[0] == 0 <= x)
PS_DEV uint32_t last_le(const uint32_t* tab, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tab[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

template <class K>
__global__ void __launch_bounds__(pipe_threads<K>()) merge_pipe_kernel(Bufs<K> bufs, uint64_t nelem,
                                                                  const Node* __restrict__ nodes,
                                                                  const uint32_t* __restrict__ chunk2node,
                                                                  uint4* __restrict__ cuts, uint32_t c0,
                                                                  uint32_t nchunks, uint32_t* err,
                                                                  uint32_t* __restrict__ bar_ctr) {
    pdl_wait();
    using LY = PipeLayout<K>;
    constexpr uint32_t VT = pipe_vt<K>();
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* scratch = smem + PIPE_SLOTS * LY::SLOT;
    PipeDesc* desc = reinterpret_cast<PipeDesc*>(scratch + LY::NXR * LY::SCRATCH);
    uint64_t* bars = reinterpret_cast<uint64_t*>(desc + PIPE_SLOTS);
    uint64_t* full = bars;                // [PIPE_SLOTS]
    uint64_t* empty = bars + PIPE_SLOTS;  // [PIPE_SLOTS]
    __shared__ uint64_t s_e0[MAXSEG][MAX_WAY];  // producer: global element index of each window
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        PT_CTA(0)
        for (uint32_t sl = 0; sl < PIPE_SLOTS; ++sl) {
            mbar_init(&full[sl], 1);
            mbar_init(&empty[sl], pipe_consumers<K>() / 32);
        }
        mbar_fence_init();
    }
    if (bar_ctr) {
        // fused partition: all warps of the grid compute the stage's cuts, then a
        // grid barrier (a cut lands at its merged index, possibly in another
        // CTA's chunk range)
        const uint32_t nw = gridDim.x * (pipe_threads<K>() / 32);
        for (uint32_t c = blockIdx.x * (pipe_threads<K>() / 32) + (tid >> 5); c < nchunks; c += nw)
            partition_chunk<K>(bufs, nodes, chunk2node, c0 + c, cuts);
        grid_barrier(bar_ctr, gridDim.x, err);
    } else {
        __syncthreads();
    }
    if (tid == 0) {
        PT_CTA(1)
    }

    if (tid < 32) {
        // ------------------------------ producer ------------------------------
        const uint32_t lane = tid;
        const uint32_t cbeg = c0 + (uint32_t)(((uint64_t)nchunks * blockIdx.x) / gridDim.x);
        const uint32_t cend = c0 + (uint32_t)(((uint64_t)nchunks * (blockIdx.x + 1)) / gridDim.x);
        uint32_t unit = 0;
        uint32_t pend = 0;  // slots whose (bulk-store) unit still has to leave
        // Stores the bulk unit that occupied slot sl (its descriptor is still there):
        // the 16-byte-aligned middle of the keys and of the values with one TMA
        // bulk store each, the <= 3 edge elements at each end with lane stores.
        auto bulk_store = [&](uint32_t sl) {
            const PipeSeg& g = desc[sl].seg[0];
            const uint8_t* sb = smem + sl * LY::SLOT;
            const K* sk = reinterpret_cast<const K*>(sb);
            const int32_t* sv = reinterpret_cast<const int32_t*>(sb + LY::OV);
            K* dk = bufs.kb(g.par);
            int32_t* dv = bufs.vb(g.par);
            const uint64_t out = g.out;
            const uint32_t T = g.T;
            const uint32_t pk = (uint32_t)(out % LY::EPK), pv = (uint32_t)(out % 4);
            const uint32_t k0 = min(T, (LY::EPK - pk) % LY::EPK), v0 = min(T, (4 - pv) % 4);
            const uint32_t kt = (uint32_t)((out + T) % LY::EPK), vt = (uint32_t)((out + T) % 4);
            const uint32_t k1 = max(k0, T >= kt ? T - kt : 0u), v1 = max(v0, T >= vt ? T - vt : 0u);
            if (lane == 0) {
                if (k1 > k0) tma_store_1d(dk + out + k0, sk + pk + k0, (k1 - k0) * (uint32_t)sizeof(K));
                if (v1 > v0) tma_store_1d(dv + out + v0, sv + pv + v0, (v1 - v0) * 4u);
                bulk_commit();
            }
            const uint32_t q = lane & 3;
            const uint32_t e = (lane & 4) ? k1 + q : q;  // keys: head lanes 0-3, tail 4-7
            if (lane < 8 && e < ((lane & 4) ? T : k0)) dk[out + e] = sk[pk + e];
            const uint32_t f = (lane & 4) ? v1 + q : q;  // values: head lanes 8-11, tail 12-15
            if (lane >= 8 && lane < 16 && f < ((lane & 4) ? T : v0)) dv[out + f] = sv[pv + f];
            if (lane == 0) bulk_wait_read_all();  // the slot may be overwritten afterwards
            __syncwarp();
        };
        PT_START(lane == 0)
        for (uint32_t c = cbeg; c < cend;) {
            // batch descriptors of chunks c .. c+31 (lane l <-> chunk c+l)
            const uint32_t x = c + lane;
            const uint32_t nvalid = min(32u, cend - c);
            const bool xv = lane < nvalid;
            uint32_t nid = xv ? chunk2node[x] : INF32;
            Node nd;
            uint4 st = make_uint4(0, 0, 0, 0), en = make_uint4(0, 0, 0, 0);
            if (xv) {
                nd = nodes[nid];
                const uint32_t q = x - nd.chunk_base;
                if (q > 0) st = cuts[x];
                if (q + 1 < nd.nchunks) {
                    en = cuts[x + 1];
                } else {
                    en.x = nd.pos[1] - nd.pos[0];
                    en.y = nd.arity > 1 ? nd.pos[2] - nd.pos[1] : 0;
                    en.z = nd.arity > 2 ? nd.pos[3] - nd.pos[2] : 0;
                    en.w = nd.arity > 3 ? nd.pos[4] - nd.pos[3] : 0;
                }
            } else {
                nd.arity = 2;
                nd.parity = 0;
#pragma unroll
                for (int t = 0; t < 5; ++t) nd.pos[t] = 0;
            }
            const uint32_t tot = (en.x - st.x) + (en.y - st.y) + (en.z - st.z) + (en.w - st.w);
            // records per unit of this chunk's node (arity * cut spacing <= cut_cap)
            const uint32_t ucap = xv ? (uint32_t)nd.arity * node_spacing(nd, cut_cap<K>()) : cut_cap<K>();
            // segment starts (node changes) and inclusive prefixes over the batch:
            // PT records, PC records + 2 VT per segment (pass layout slack), PS segments
            const uint32_t nid_prev = __shfl_up_sync(PS_FULL, nid, 1);
            const uint32_t sgs = (lane == 0 || nid != nid_prev) ? 1u : 0u;
            uint32_t PT = tot, PC = tot + sgs * 2 * VT, PS = sgs;
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t a1 = __shfl_up_sync(PS_FULL, PT, d), a2 = __shfl_up_sync(PS_FULL, PC, d);
                const uint32_t a3 = __shfl_up_sync(PS_FULL, PS, d);
                if (lane >= (uint32_t)d) {
                    PT += a1;
                    PC += a2;
                    PS += a3;
                }
            }
            const uint32_t XT = PT - tot, XC = PC - (tot + sgs * 2 * VT), XS = PS - sgs;
            PT_MARK(0)
            uint32_t u = 0;
            while (u < nvalid) {
                // unit = lanes u..V: chunks of one node with <= cut_cap records, or
                // several segments with sum(records + 2 VT) <= CAP, <= MAXSEG of them
                const uint32_t nid_u = __shfl_sync(PS_FULL, nid, u);
                const uint32_t XTu = __shfl_sync(PS_FULL, XT, u), XCu = __shfl_sync(PS_FULL, XC, u);
                const uint32_t XSu = __shfl_sync(PS_FULL, XS, u), sgsu = __shfl_sync(PS_FULL, sgs, u);
                const uint32_t ucapu = __shfl_sync(PS_FULL, ucap, u);
                const bool same = nid == nid_u;
                const uint32_t sumT = PT - XTu;
                const uint32_t sumC = PC - XCu + (sgsu ? 0u : 2 * VT);
                const uint32_t nsg = PS - XSu + (sgsu ? 0u : 1u);
                const bool ok = lane >= u && lane < nvalid &&
                                (same ? sumT <= ucapu : (sumC <= LY::CAP && nsg <= pipe_maxseg<K>()));
                const uint32_t bal = __ballot_sync(PS_FULL, ok) >> u;
                const uint32_t runlen = __ffs(~bal) ? __ffs(~bal) - 1 : 32 - u;
                const uint32_t V = u + max(runlen, 1u) - 1;
                // segments of the unit: starts at u and at node changes in (u, V]
                const uint32_t mseg = __ballot_sync(PS_FULL, lane >= u && lane <= V && (lane == u || sgs));
                const uint32_t nseg = __popc(mseg);
                const bool has = lane < nseg;
                const uint32_t as = has ? __fns(mseg, 0, lane + 1) : u;
                const uint32_t bs = (lane + 1 < nseg) ? __fns(mseg, 0, lane + 2) - 1 : V;
                uint32_t sv4[4], ev4[4], npos[5];
                sv4[0] = __shfl_sync(PS_FULL, st.x, as);
                sv4[1] = __shfl_sync(PS_FULL, st.y, as);
                sv4[2] = __shfl_sync(PS_FULL, st.z, as);
                sv4[3] = __shfl_sync(PS_FULL, st.w, as);
                ev4[0] = __shfl_sync(PS_FULL, en.x, bs);
                ev4[1] = __shfl_sync(PS_FULL, en.y, bs);
                ev4[2] = __shfl_sync(PS_FULL, en.z, bs);
                ev4[3] = __shfl_sync(PS_FULL, en.w, bs);
#pragma unroll
                for (int t = 0; t < 5; ++t) npos[t] = __shfl_sync(PS_FULL, nd.pos[t], as);
                const uint32_t w = __shfl_sync(PS_FULL, (uint32_t)nd.arity, as);
                const uint32_t par = __shfl_sync(PS_FULL, (uint32_t)nd.parity, as);
                // per segment (lane s < nseg): windows, region sizes, pass layouts
                uint32_t len[4], kph[4], vph[4], kb[4], vb[4];
                uint32_t T = 0, kreg = 0, vreg = 0;
#pragma unroll
                for (uint32_t t = 0; t < 4; ++t) {
                    len[t] = (has && t < w) ? ev4[t] - sv4[t] : 0;
                    const uint64_t e0 = (uint64_t)npos[t] + sv4[t];
                    kph[t] = (uint32_t)((e0 * sizeof(K)) & 15);
                    vph[t] = (uint32_t)((e0 * 4) & 15);
                    kb[t] = len[t] ? align16c(kph[t] + len[t] * (uint32_t)sizeof(K)) : 0;
                    vb[t] = len[t] ? align16c(vph[t] + len[t] * 4u) : 0;
                    T += len[t];
                    kreg += kb[t];
                    vreg += vb[t];
                }
                const uint32_t LXs = len[0] + len[1], LYs = T - LXs;
                const bool last = lane + 1 == nseg;
                const uint32_t px = (LXs + VT - 1) / VT * VT, py = (LYs + VT - 1) / VT * VT;
                const uint32_t size1 = !has ? 0u : !last ? px + py : (LYs ? px + LYs : LXs);
                const uint32_t size2 = !has ? 0u : !last ? (T + VT - 1) / VT * VT : T;
                uint32_t ek = kreg, ev = vreg, e1 = size1, e2 = size2;  // inclusive scans over segments
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t b1 = __shfl_up_sync(PS_FULL, ek, d), b2 = __shfl_up_sync(PS_FULL, ev, d);
                    const uint32_t b3 = __shfl_up_sync(PS_FULL, e1, d), b4 = __shfl_up_sync(PS_FULL, e2, d);
                    if (lane >= (uint32_t)d) {
                        ek += b1;
                        ev += b2;
                        e1 += b3;
                        e2 += b4;
                    }
                }
                const uint32_t end1 = __shfl_sync(PS_FULL, e1, 31), end2 = __shfl_sync(PS_FULL, e2, 31);
                // ---- stage the unit into slot (unit % PIPE_SLOTS) ----
                const uint32_t slot = unit % PIPE_SLOTS;
                if (unit >= PIPE_SLOTS) mbar_wait(&empty[slot], ((unit / PIPE_SLOTS) - 1) & 1);
                if (pend & (1u << slot)) {
                    bulk_store(slot);
                    pend &= ~(1u << slot);
                }
                PT_MARK(1)
                uint8_t* sbase = smem + slot * LY::SLOT;
                PipeDesc& d = desc[slot];
                if (has) {
                    PipeSeg& g = d.seg[lane];
                    uint32_t ko = ek - kreg, vo = LY::KEY_BYTES + (ev - vreg);
                    uint64_t out = npos[0];
#pragma unroll
                    for (uint32_t t = 0; t < 4; ++t) {
                        g.koff[t] = ko + kph[t];
                        g.voff[t] = vo + vph[t];
                        g.len[t] = len[t];
                        s_e0[lane][t] = (uint64_t)npos[t] + sv4[t];
                        ko += kb[t];
                        vo += vb[t];
                        out += (t < w) ? sv4[t] : 0u;
                    }
                    g.out = out;
                    g.w = w;
                    g.par = par;
                    g.T = T;
                    g.lx = LXs;
                    const uint32_t b1s = e1 - size1;
                    d.s1[2 * lane] = b1s;
                    d.s1[2 * lane + 1] = b1s + px;
                    d.s2[lane] = e2 - size2;
                }
                if (lane == 0) {
                    d.nseg = nseg;
                    d.done = 0;
                    d.end1 = end1;
                    d.end2 = end2;
                    if (end1 > LY::CAP + VT - 1 || end2 > LY::CAP + VT - 1) atomicOr(err, ERR_CUT);
                }
                __syncwarp();
                // window copies: op = (segment, window, keys|values), spread over the lanes
                uint32_t tx = 0;
                for (uint32_t op = lane; op < nseg * 8; op += 32) {
                    const uint32_t sg = op >> 3, t = op & 3;
                    const bool is_val = (op & 4) != 0;
                    const PipeSeg& g = d.seg[sg];
                    const uint32_t ln = g.len[t];
                    if (ln == 0) continue;
                    const uint32_t eb = is_val ? 4u : (uint32_t)sizeof(K);
                    const uint32_t doff = is_val ? g.voff[t] : g.koff[t];  // includes the phase
                    const uint64_t e0 = s_e0[sg][t];
                    const uint8_t* src = is_val ? reinterpret_cast<const uint8_t*>(bufs.vb(g.par ^ 1))
                                                : reinterpret_cast<const uint8_t*>(bufs.kb(g.par ^ 1));
                    const uint64_t b0 = e0 * eb, b1 = (e0 + ln) * eb;
                    const uint64_t a0 = b0 & ~15ull, a1 = b1 & ~15ull;
                    uint8_t* dst = sbase + doff - (uint32_t)(b0 & 15);  // 16-byte aligned region start
                    const uint64_t r1 = (b1 + 15) & ~15ull;
                    if (r1 <= nelem * eb) {
                        // whole region [a0, r1) in one copy: the bytes past the window stay
                        // inside the source array and land in this window's own slack
                        tma_load_1d(dst, src + a0, (uint32_t)(r1 - a0), &full[slot]);
                        tx += (uint32_t)(r1 - a0);
                        continue;
                    }
                    if (a1 > a0) {
                        tma_load_1d(dst, src + a0, (uint32_t)(a1 - a0), &full[slot]);
                        tx += (uint32_t)(a1 - a0);
                    }
                    // tail bytes [max(a1, b0), b1) at the array end with ordinary loads
                    for (uint64_t bb = (a1 > b0 ? a1 : b0); bb < b1; bb += eb) {
                        if (is_val)
                            *reinterpret_cast<int32_t*>(dst + (bb - a0)) = *reinterpret_cast<const int32_t*>(src + bb);
                        else
                            *reinterpret_cast<K*>(dst + (bb - a0)) = *reinterpret_cast<const K*>(src + bb);
                    }
                }
                for (int dd = 16; dd; dd >>= 1) tx += __shfl_xor_sync(PS_FULL, tx, dd);
                __syncwarp();
                if (PS_BULK_STORE && nseg == 1 && __shfl_sync(PS_FULL, w, 0) >= 3) pend |= 1u << slot;
                if (lane == 0) mbar_arrive_tx(&full[slot], tx);
                PT_MARK(2)
                PT_COUNT(3)
                unit++;
                u = V + 1;
            }
            c += nvalid;
        }
        // termination marker, then the units still in flight leave
        const uint32_t slot = unit % PIPE_SLOTS;
        if (unit >= PIPE_SLOTS) mbar_wait(&empty[slot], ((unit / PIPE_SLOTS) - 1) & 1);
        if (pend & (1u << slot)) bulk_store(slot);
        pend &= ~(1u << slot);
        __syncwarp();
        if (lane == 0) {
            desc[slot].done = 1;
            mbar_arrive(&full[slot]);
        }
        for (uint32_t v = unit >= PIPE_SLOTS - 1 ? unit - (PIPE_SLOTS - 1) : 0; v < unit; ++v) {
            const uint32_t sl = v % PIPE_SLOTS;
            if (!(pend & (1u << sl))) continue;
            mbar_wait(&empty[sl], (v / PIPE_SLOTS) & 1);
            bulk_store(sl);
        }
        if (lane == 0) bulk_wait_all();
        if (lane == 0) {
            PT_CTA(4)
        }
        return;
    }

    // ------------------------------ consumers ---------------------------------
    const uint32_t ctid = tid - 32;
    const uint32_t clane = ctid & 31, wid = ctid >> 5;
    Rec<K>* const xr0 = reinterpret_cast<Rec<K>*>(scratch);
    constexpr uint32_t ER = sizeof(K) == 4 ? 4 : 2;  // records per 16-byte store group
    const uint32_t ob = VT * ctid;                   // this thread's first output of a pass layout
    const uint32_t r0w = VT * 32 * wid, r1w = VT * 32 * (wid + 1);  // this warp's outputs
    PT_START(ctid == 0)
    for (uint32_t i = 0;; ++i) {
        const uint32_t slot = i % PIPE_SLOTS;
        mbar_wait(&full[slot], (i / PIPE_SLOTS) & 1);
        if (i == 0 && ctid == 0) {
            PT_CTA(2)
        }
        PT_MARK(4)
        PT_USTART
        const PipeDesc& d = desc[slot];
        if (d.done) {
            if (ctid == 0) {
                PT_CTA(3)
            }
            break;
        }
        Rec<K>* const xr = xr0 + (LY::NXR == 2 ? (i & 1) * (LY::SCRATCH / LY::RECB) : 0);
        const bool single_pass = d.nseg == 1 && d.seg[0].w < 3;  // read before the slot is released
        uint8_t* sbase = smem + slot * LY::SLOT;
        Rec<K>* const orec = reinterpret_cast<Rec<K>*>(sbase);
        // SoA first-pass scratch (PS_SOA_X): X || Y keys at xk, values at xv
        K* const xk = reinterpret_cast<K*>(xr);
        int32_t* const xv = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(xr) + LY::XV);
        auto xcur = [&](uint32_t offa, uint32_t offb, uint32_t la, uint32_t lb, uint32_t base, uint32_t o,
                        uint32_t oe) {
            WinCur<K> c;
            c.ak = xk + offa;
            c.bk = xk + offb;
            c.av = xv + offa;
            c.bv = xv + offb;
            c.la = la;
            c.lb = lb;
            c.o = o;
            c.oe = oe;
            c.base = base;
            return c;
        };
        (void)xcur;
        auto wincur = [&](const PipeSeg& g, uint32_t a, uint32_t base, uint32_t o, uint32_t oe) {
            WinCur<K> c;
            c.ak = reinterpret_cast<const K*>(sbase + g.koff[a]);
            c.bk = reinterpret_cast<const K*>(sbase + g.koff[a + 1]);
            c.av = reinterpret_cast<const int32_t*>(sbase + g.voff[a]);
            c.bv = reinterpret_cast<const int32_t*>(sbase + g.voff[a + 1]);
            c.la = g.len[a];
            c.lb = g.len[a + 1];
            c.o = o;
            c.oe = oe;
            c.base = base;
            return c;
        };
        if (d.nseg == 1) {
            // ---- one segment: pass 2 output phase-shifted for 16-byte stores ----
            const PipeSeg& g = d.seg[0];
            const uint32_t T = g.T, par = g.par;
            const uint64_t out = g.out;
            const uint32_t al = (uint32_t)(out % ER);
            const uint32_t o0 = min(T, ob), o1 = min(T, ob + VT);
            Rec<K>* res;
            if (g.w >= 3) {
                // pass 1: X = merge(A, B) -> xr[0, LX);  Y = merge(C, D) (3-way: C) -> xr[LXp, LXp + LY)
                // (LXp = LX rounded up to VT: every thread works inside X or inside Y)
                const uint32_t LX = g.lx, LYn = T - LX, LXp = d.s1[1];
                const bool isY = ob >= LXp;
                WinCur<K> c = isY ? wincur(g, 2, LXp, ob - LXp, min(ob + VT - LXp, LYn))
                                  : wincur(g, 0, 0, ob, min(ob + VT, LX));
                if (PS_SOA_X)
                    single_merge_soa(c, xk, xv);
                else
                    single_merge(c, xr);
                PT_WARP(16)
                consumer_sync<pipe_consumers<K>()>();
                PT_MARK(5)
                if (PS_SOA_X) {
                    if (PS_BULK_STORE) {
                        WinCur<K> q = xcur(0, LXp, LX, LYn, 0, o0, o1);
                        single_merge_soa(q, reinterpret_cast<K*>(sbase) + (uint32_t)(out % LY::EPK),
                                         reinterpret_cast<int32_t*>(sbase + LY::OV) + (uint32_t)(out % 4));
                        fence_proxy_async_smem();
                        PT_WARP(24)
                        __syncwarp();
                        PT_MARK(6)
                        goto unit_done;
                    }
                    WinCur<K> q = xcur(0, LXp, LX, LYn, al, o0, o1);
                    single_merge(q, orec);
                    res = orec;
                } else {
                // pass 2: merge X and Y into the slot (its input windows are consumed)
                RecCur<K> p0;
                p0.r = xr;
                p0.offa = 0;
                p0.offb = LXp;
                p0.la = LX;
                p0.lb = LYn;
                p0.base = al;
                p0.o = o0;
                p0.oe = o1;
                if (PS_BULK_STORE) {
                    // SoA outputs phase-aligned with their destinations; the producer
                    // stores them with TMA once every warp has arrived on empty[slot]
                    single_merge_soa(p0, reinterpret_cast<K*>(sbase) + (uint32_t)(out % LY::EPK),
                                     reinterpret_cast<int32_t*>(sbase + LY::OV) + (uint32_t)(out % 4));
                    fence_proxy_async_smem();
                    PT_WARP(24)
                    __syncwarp();
                    PT_MARK(6)
                    goto unit_done;
                }
                single_merge(p0, orec);
                res = orec;
                }
            } else {
                // 2-way: merge(A, B) straight into scratch
                WinCur<K> c = wincur(g, 0, al, o0, o1);
                single_merge(c, xr);
                res = xr;
            }
            PT_WARP(24)
            // store: every warp moves its own outputs as soon as they are written:
            // full ER-groups of the phase-shifted layout as 16-byte vectors, the
            // partial groups at both ends record by record
            __syncwarp();
            PT_MARK(6)
            K* __restrict__ dstK = bufs.kb(par);
            int32_t* __restrict__ dstV = bufs.vb(par);
            const uint32_t rs = al + min(T, r0w), re = al + min(T, r1w);
            const uint64_t gbase = out - al;  // global element of record index 0
            if (rs < re) {
                const uint32_t g0 = (rs + ER - 1) / ER, g1 = re / ER;
                for (uint32_t j = g0 + clane; j < g1; j += 32) {
                    const uint32_t r0 = j * ER;
                    const uint4* src = reinterpret_cast<const uint4*>(res + r0);
                    if (sizeof(K) == 4) {
                        const uint4 q0 = src[0], q1 = src[1];  // (k0,v0,k1,v1) (k2,v2,k3,v3)
                        *reinterpret_cast<uint4*>(dstK + gbase + r0) = make_uint4(q0.x, q0.z, q1.x, q1.z);
                        *reinterpret_cast<uint4*>(dstV + gbase + r0) = make_uint4(q0.y, q0.w, q1.y, q1.w);
                    } else {
                        const uint4 q0 = src[0], q1 = src[1];  // (k0 lo, k0 hi, v0, pad) (k1 lo, k1 hi, v1, pad)
                        *reinterpret_cast<uint4*>(dstK + gbase + r0) = make_uint4(q0.x, q0.y, q1.x, q1.y);
                        *reinterpret_cast<uint2*>(dstV + gbase + r0) = make_uint2(q0.z, q1.z);
                    }
                }
                // head [rs, min(re, g0*ER)) on lanes 0..ER-1, tail [max(rs, g1*ER), re) on lanes 16..
                // (a range inside one group is written twice, with the same data)
                uint32_t rr = INF32;
                if (clane < ER) rr = rs + clane < min(re, g0 * ER) ? rs + clane : INF32;
                if (clane >= 16 && clane < 16 + ER) {
                    const uint32_t t0 = max(rs, g1 * ER) + (clane - 16);
                    rr = t0 < re ? t0 : INF32;
                }
                if (rr != INF32) {
                    const Rec<K> rec = res[rr];
                    dstK[gbase + rr] = rec.k;
                    dstV[gbase + rr] = rec.v;
                }
            }
        } else {
            // ---- several segments: both passes through the VT-aligned part layouts ----
            const uint32_t nseg = d.nseg;
            if (ob < d.end1) {
                const uint32_t pp = last_le(d.s1, 2 * nseg, ob);
                const PipeSeg& g = d.seg[pp >> 1];
                const bool isY = pp & 1;
                const uint32_t Lp = isY ? g.T - g.lx : g.lx;
                const uint32_t o = ob - d.s1[pp];
                if (o < Lp) {
                    WinCur<K> c = wincur(g, isY ? 2 : 0, d.s1[pp], o, min(o + VT, Lp));
                    if (PS_SOA_X)
                        single_merge_soa(c, xk, xv);
                    else
                        single_merge(c, xr);
                }
            }
            PT_WARP(16)
            consumer_sync<pipe_consumers<K>()>();
            PT_MARK(5)
            if (ob < d.end2) {
                const uint32_t sg = last_le(d.s2, nseg, ob);
                const PipeSeg& g = d.seg[sg];
                const uint32_t o = ob - d.s2[sg];
                if (o < g.T && PS_SOA_X) {
                    WinCur<K> q = xcur(d.s1[2 * sg], d.s1[2 * sg + 1], g.lx, g.T - g.lx, d.s2[sg], o,
                                       min(o + VT, g.T));
                    single_merge(q, orec);
                } else if (o < g.T) {
                    RecCur<K> p0;
                    p0.r = xr;
                    p0.offa = d.s1[2 * sg];
                    p0.offb = d.s1[2 * sg + 1];
                    p0.la = g.lx;
                    p0.lb = g.T - g.lx;
                    p0.base = d.s2[sg];
                    p0.o = o;
                    p0.oe = min(o + VT, g.T);
                    single_merge(p0, orec);
                }
            }
            PT_WARP(24)
            __syncwarp();
            PT_MARK(6)
            // store this warp's outputs segment by segment (coalesced 4-byte stores)
            const uint32_t re = min(r1w, d.end2);
            if (r0w < re) {
                for (uint32_t sg = last_le(d.s2, nseg, r0w); sg < nseg && d.s2[sg] < re; ++sg) {
                    const PipeSeg& g = d.seg[sg];
                    const uint32_t lo = max(r0w, d.s2[sg]), hi = min(re, d.s2[sg] + g.T);
                    K* __restrict__ dstK = bufs.kb(g.par);
                    int32_t* __restrict__ dstV = bufs.vb(g.par);
                    const uint64_t gb = g.out - d.s2[sg];
                    for (uint32_t r = lo + clane; r < hi; r += 32) {
                        const Rec<K> rec = orec[r];
                        dstK[gb + r] = rec.k;
                        dstV[gb + r] = rec.v;
                    }
                }
            }
        }
        __syncwarp();
    unit_done:
        if (clane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
        // scratch xr is rewritten by the next unit's first pass (with two scratch
        // buffers only single-pass units, which have no barrier of their own, need it)
        if (LY::NXR == 1 || single_pass) consumer_sync<pipe_consumers<K>()>();
        PT_MARK(7)
        PT_COUNT(8)
    }
}

}  // namespace ps

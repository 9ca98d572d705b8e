// ps_shard.cuh -- N6: cross-shard merge for the multi-GPU mode.
//
// Rank g of G has sorted its contiguous shard (shard h holds global indices
// [off_h, off_h + n_h)).  Its output slab is global ranks [t0, t1) of the
// stable order (key, shard, position) == (key, global index).  The slab's
// start and end co-ranks in the G shards are found by *parallel bracketing*:
// every round, P evenly spaced candidates of every shard's current window are
// ranked against all shards at once (one warp per candidate, one lane per
// shard doing a binary search clamped to that shard's window) and the
// windows shrink by ~P+1; shards may live on other GPUs (peer pointers,
// NVLink loads).  The co-ranked windows are then gathered with direct peer
// loads and merged locally with the same kernels as the single-GPU tree.
#pragma once

#include "ps_common.cuh"

namespace ps {

constexpr uint32_t MAX_SHARDS = 8;
constexpr uint32_t SEL_CANDIDATES = 64;  // per shard per round

template <class K>
struct ShardSet {
    const K* k[MAX_SHARDS];
    const int32_t* v[MAX_SHARDS];
    uint64_t n[MAX_SHARDS];
    uint64_t off[MAX_SHARDS];  // global index of each shard's first element
    uint32_t G;
};

// bounds layout: [which target (0: slab start, 1: slab end)][2][MAX_SHARDS]
//   lo = bounds[t*2*MAX_SHARDS + h], hi = bounds[t*2*MAX_SHARDS + MAX_SHARDS + h]
// Invariant: the true co-rank c_h of the target rank lies in [lo_h, hi_h].

// # of shard-h elements before element (g, key y) in (key, shard, pos) order,
// searched within [lo, hi] (valid by the clamping argument).
template <class K>
PS_DEV uint64_t shard_count_before(const K* __restrict__ a, uint64_t lo, uint64_t hi, K y, bool le) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const K z = a[mid];
        const bool before = le ? !(y < z) : (z < y);
        lo = before ? mid + 1 : lo;
        hi = before ? hi : mid;
    }
    return lo;
}

// One bracketing round for up to two targets (blockIdx.y).  Grid.x =
// G * SEL_CANDIDATES / warps-per-block; one warp per candidate.
template <class K>
__global__ void __launch_bounds__(256) shard_select_kernel(ShardSet<K> S, const uint64_t* __restrict__ targets,
                                                           unsigned long long* bounds) {
    pdl_wait();
    const uint32_t tgt = blockIdx.y;
    const uint32_t wid = blockIdx.x * 8 + warp_id();
    const uint32_t lane = lane_id();
    const uint32_t G = S.G;
    if (wid >= G * SEL_CANDIDATES) return;
    const uint32_t g = wid / SEL_CANDIDATES, ci = wid % SEL_CANDIDATES;
    unsigned long long* lo = bounds + (size_t)tgt * 2 * MAX_SHARDS;
    unsigned long long* hi = lo + MAX_SHARDS;
    const uint64_t t = targets[tgt];
    const uint64_t glo = lo[g], ghi = hi[g];
    if (ghi <= glo) return;
    const uint64_t w = ghi - glo;
    const uint64_t p = glo + (w * (ci + 1)) / (SEL_CANDIDATES + 1);  // candidate position in shard g
    if (p >= ghi) return;
    const K y = S.k[g][p];
    uint64_t r = 0;
    if (lane < G) {
        if (lane == g) {
            r = p;
        } else {
            const uint64_t l = lo[lane], h = hi[lane];
            r = shard_count_before<K>(S.k[lane], l, h, y, lane < g);
        }
    }
    uint64_t R = r;
    for (int d = 16; d; d >>= 1) R += __shfl_xor_sync(PS_FULL, R, d);
    // element (g, p) precedes the target element iff its global rank R < t
    if (lane < G) {
        if (R < t) {
            atomicMax(&lo[lane], (unsigned long long)(lane == g ? p + 1 : r));
        } else {
            atomicMin(&hi[lane], (unsigned long long)(lane == g ? p : r));
        }
    }
}

// Gather the co-ranked windows [cb[h], ce[h]) of every shard (peer loads)
// into the local buffers at the window offsets dst_off[h].
template <class K>
__global__ void shard_gather_kernel(ShardSet<K> S, const unsigned long long* __restrict__ bounds_begin,
                                    const unsigned long long* __restrict__ bounds_end, K* __restrict__ dk,
                                    int32_t* __restrict__ dv, uint64_t total) {
    pdl_wait();
    __shared__ uint64_t s_cb[MAX_SHARDS], s_off[MAX_SHARDS + 1];
    if (threadIdx.x == 0) {
        uint64_t acc = 0;
        for (uint32_t h = 0; h < S.G; ++h) {
            s_cb[h] = bounds_begin[h];  // lo == hi after convergence
            s_off[h] = acc;
            acc += bounds_end[h] - bounds_begin[h];
        }
        for (uint32_t h = S.G; h <= MAX_SHARDS; ++h) s_off[h] = acc;
    }
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = 0;
        while (h + 1 < S.G && i >= s_off[h + 1]) ++h;
        const uint64_t src = s_cb[h] + (i - s_off[h]);
        dk[i] = S.k[h][src];
        dv[i] = S.v[h][src];
    }
}

}  // namespace ps

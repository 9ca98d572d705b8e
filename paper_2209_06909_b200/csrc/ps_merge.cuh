// ps_merge.cuh -- N3: batched stable k-way merges (one launch per tree level).
//
// Replaces merges.py:75-500 (merge_2way_*, merge_3way, merge_4way_*).  A stable
// k-way merge has a unique output (ties go to the lower-index run,
// merges.py:1-8), which is the merge under the strict composite order
// (key, run index, position).  Big nodes are cut into chunks: cut (a, j) is
// the element at position j*S of run a (S = CHUNK_CAP / arity); its rank in
// every other run b is a binary search (<= for b < a, < for b > a), and its
// index in the merged cut order follows directly from those ranks.  Between
// consecutive cuts there are at most S elements of each run, so each chunk is
// at most CHUNK_CAP records and is merged in shared memory by one CTA: every
// record computes its output rank within the chunk (its own index plus its
// galloping co-rank in each other window) and is scattered once.  Children
// are read from buffer (depth+1)&1 and the node is written to depth&1.
#pragma once

#include "ps_common.cuh"
#include "ps_form.cuh"

namespace ps {

// # of a[0..len) that are <= x (LE) or < x (!LE)
template <class K, bool LE>
PS_DEV uint32_t count_pred(const K* __restrict__ a, uint32_t len, K x) {
    uint32_t lo = 0;
    while (len > 0) {
        const uint32_t half = len >> 1;
        const K y = a[lo + half];
        const bool p = LE ? !(x < y) : (y < x);
        if (p) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return lo;
}

// Advance cursor cur in window w[0..len) to the first index where the
// predicate (w[i] <= x, or w[i] < x) fails; galloping from cur.
template <class K, bool LE>
PS_DEV uint32_t gallop(const K* w, uint32_t len, uint32_t cur, K x) {
    auto pred = [&](uint32_t i) {
        const K y = w[i];
        return LE ? !(x < y) : (y < x);
    };
    if (cur >= len || !pred(cur)) return cur;
    uint32_t lo = cur, hi, step = 1;
    for (;;) {
        hi = lo + step;
        if (hi >= len) {
            hi = len;
            break;
        }
        if (!pred(hi)) break;
        lo = hi;
        step <<= 1;
    }
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pred(mid))
            lo = mid;
        else
            hi = mid;
    }
    return hi;
}

// Partition: one thread per chunk of the stage [c0, c1).
template <class K>
__global__ void merge_partition_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                       const uint32_t* __restrict__ chunk2node, uint32_t c0, uint32_t c1,
                                       uint4* __restrict__ cuts) {
    const uint32_t c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c1) return;
    const Node nd = nodes[chunk2node[c]];
    uint32_t q = c - nd.chunk_base;
    if (q == 0) {
        cuts[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    q -= 1;
    const uint32_t w = nd.arity;
    const uint32_t S = CHUNK_CAP / w;
    const K* src = bufs.k[nd.parity ^ 1];
    uint32_t L[4];
    for (uint32_t a = 0; a < 4; ++a) L[a] = a < w ? nd.pos[a + 1] - nd.pos[a] : 0;
    uint32_t a = 0;
    for (; a < w; ++a) {
        const uint32_t nc = (L[a] - 1) / S;
        if (q < nc) break;
        q -= nc;
    }
    const uint32_t j = q + 1;
    const K y = src[(uint64_t)nd.pos[a] + (uint64_t)j * S];
    uint32_t rk[4] = {0, 0, 0, 0};
    uint32_t mm = j - 1;
    for (uint32_t bb = 0; bb < w; ++bb) {
        if (bb == a) {
            rk[bb] = j * S;
            continue;
        }
        const K* run = src + nd.pos[bb];
        rk[bb] = bb < a ? count_pred<K, true>(run, L[bb], y) : count_pred<K, false>(run, L[bb], y);
        mm += rk[bb] ? (rk[bb] - 1) / S : 0;
    }
    cuts[nd.chunk_base + 1 + mm] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
}

template <class K>
size_t merge_smem_bytes() {
    return (size_t)CHUNK_CAP * (sizeof(K) + 4);
}

// Merge: one CTA per chunk of the stage starting at c0.
template <class K>
__global__ void __launch_bounds__(MERGE_THREADS) merge_chunks_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                     const uint32_t* __restrict__ chunk2node,
                                                                     const uint4* __restrict__ cuts, uint32_t c0,
                                                                     uint32_t* err) {
    extern __shared__ __align__(16) uint8_t smem[];
    K* sk = reinterpret_cast<K*>(smem);
    int32_t* sv = reinterpret_cast<int32_t*>(sk + CHUNK_CAP);
    __shared__ uint32_t s_off[5], s_len[4];
    __shared__ uint64_t s_src[4], s_out;
    __shared__ uint32_t s_w, s_T, s_par;
    const uint32_t c = c0 + blockIdx.x;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        const Node nd = nodes[chunk2node[c]];
        const uint32_t q = c - nd.chunk_base;
        const uint32_t w = nd.arity;
        uint32_t st[4] = {0, 0, 0, 0}, en[4] = {0, 0, 0, 0};
        for (uint32_t a = 0; a < w; ++a) en[a] = nd.pos[a + 1] - nd.pos[a];
        if (q > 0) {
            const uint4 v = cuts[c];
            st[0] = v.x;
            st[1] = v.y;
            st[2] = v.z;
            st[3] = v.w;
        }
        if (q + 1 < nd.nchunks) {
            const uint4 v = cuts[c + 1];
            en[0] = v.x;
            en[1] = v.y;
            en[2] = v.z;
            en[3] = v.w;
        }
        uint32_t acc = 0;
        uint64_t out = nd.pos[0];
        for (uint32_t a = 0; a < 4; ++a) {
            s_off[a] = acc;
            const uint32_t len = a < w ? en[a] - st[a] : 0;
            s_len[a] = len;
            s_src[a] = a < w ? (uint64_t)nd.pos[a] + st[a] : 0;
            acc += len;
            out += a < w ? st[a] : 0;
        }
        s_off[4] = acc;
        if (acc > CHUNK_CAP) {
            atomicOr(err, ERR_CUT);
            acc = 0;
        }
        s_T = acc;
        s_w = w;
        s_out = out;
        s_par = nd.parity;
    }
    __syncthreads();
    const uint32_t T = s_T, w = s_w;
    const uint32_t par = s_par;
    const K* __restrict__ srcK = bufs.k[par ^ 1];
    const int32_t* __restrict__ srcV = bufs.v[par ^ 1];
    for (uint32_t i = tid; i < T; i += MERGE_THREADS) {
        const uint32_t a = (i >= s_off[1]) + (i >= s_off[2]) + (i >= s_off[3]);
        const uint64_t g = s_src[a] + (i - s_off[a]);
        sk[i] = srcK[g];
        sv[i] = srcV[g];
    }
    __syncthreads();
    K xk[MERGE_VT];
    int32_t xv[MERGE_VT];
    uint32_t xr[MERGE_VT];
    uint32_t cur[4] = {0, 0, 0, 0};
    int cur_a = -1;
#pragma unroll
    for (uint32_t v = 0; v < MERGE_VT; ++v) {
        const uint32_t i = tid * MERGE_VT + v;
        xr[v] = INF32;
        if (i < T) {
            const uint32_t a = (i >= s_off[1]) + (i >= s_off[2]) + (i >= s_off[3]);
            if ((int)a != cur_a) {
                cur_a = (int)a;
                cur[0] = cur[1] = cur[2] = cur[3] = 0;
            }
            const K x = sk[i];
            uint32_t rank = i - s_off[a];
#pragma unroll
            for (uint32_t bb = 0; bb < 4; ++bb) {
                if (bb < w && bb != a) {
                    const K* wb = sk + s_off[bb];
                    cur[bb] = bb < a ? gallop<K, true>(wb, s_len[bb], cur[bb], x)
                                     : gallop<K, false>(wb, s_len[bb], cur[bb], x);
                    rank += cur[bb];
                }
            }
            xk[v] = x;
            xv[v] = sv[i];
            xr[v] = rank;
        }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t v = 0; v < MERGE_VT; ++v) {
        if (xr[v] != INF32) {
            sk[xr[v]] = xk[v];
            sv[xr[v]] = xv[v];
        }
    }
    __syncthreads();
    K* __restrict__ dstK = bufs.k[par];
    int32_t* __restrict__ dstV = bufs.v[par];
    const uint64_t out = s_out;
    for (uint32_t i = tid; i < T; i += MERGE_THREADS) {
        dstK[out + i] = sk[i];
        dstV[out + i] = sv[i];
    }
}

}  // namespace ps

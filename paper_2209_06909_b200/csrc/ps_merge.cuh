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
PS_DEV void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(256) : "memory"); }

// ---------------------------------------------------------------------------
// Small nodes (size <= SMALL_NODE): one warp per node, straight from global.
constexpr uint32_t SMALL_WARPS = 8;

template <class K>
size_t merge_small_smem_bytes() {
    return (size_t)SMALL_WARPS * SMALL_NODE * 2 * (sizeof(K) + 4);
}

template <class K>
__global__ void __launch_bounds__(SMALL_WARPS * 32) merge_small_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                       uint32_t nlo, uint32_t nhi) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t idx = nlo + blockIdx.x * SMALL_WARPS + warp;
    if (idx >= nhi) return;
    const Node nd = nodes[idx];
    const uint32_t w = nd.arity;
    const uint32_t p0 = nd.pos[0];
    const uint32_t size = nd.pos[w] - p0;
    if (size > SMALL_NODE) return;
    uint8_t* base = smem + (size_t)warp * SMALL_NODE * 2 * (sizeof(K) + 4);
    K* sk = reinterpret_cast<K*>(base);
    K* ok = sk + SMALL_NODE;
    int32_t* sv = reinterpret_cast<int32_t*>(ok + SMALL_NODE);
    int32_t* ov = sv + SMALL_NODE;
    const K* __restrict__ srcK = bufs.k[nd.parity ^ 1];
    const int32_t* __restrict__ srcV = bufs.v[nd.parity ^ 1];
    for (uint32_t i = lane; i < size; i += 32) {
        sk[i] = srcK[(uint64_t)p0 + i];
        sv[i] = srcV[(uint64_t)p0 + i];
    }
    __syncwarp();
    __shared__ uint32_t s_off[SMALL_WARPS][8];
    if (lane < 5) s_off[warp][lane] = lane <= w ? nd.pos[lane] - p0 : size;
    __syncwarp();
    const uint32_t* off = s_off[warp];
    const uint32_t o1 = off[1], o2 = w > 2 ? off[2] : size, o3 = w > 3 ? off[3] : size;
    for (uint32_t i = lane; i < size; i += 32) {
        const uint32_t a = (i >= o1) + (i >= o2) + (i >= o3);
        const K x = sk[i];
        uint32_t rank = i - off[a];
#pragma unroll
        for (uint32_t b = 0; b < 4; ++b) {
            if (b < w && b != a) {
                const uint32_t ob = off[b], lb = off[b + 1] - ob;
                rank += b < a ? count_pred<K, true>(sk + ob, lb, x) : count_pred<K, false>(sk + ob, lb, x);
            }
        }
        ok[rank] = x;
        ov[rank] = sv[i];
    }
    __syncwarp();
    K* __restrict__ dstK = bufs.k[nd.parity];
    int32_t* __restrict__ dstV = bufs.v[nd.parity];
    for (uint32_t i = lane; i < size; i += 32) {
        dstK[(uint64_t)p0 + i] = ok[i];
        dstV[(uint64_t)p0 + i] = ov[i];
    }
}

// ---------------------------------------------------------------------------
// Big-node chunks: persistent, warp-specialized, TMA-bulk double-buffered.
//   warp 0      producer: chunk descriptor (node, cuts) + cp.async.bulk of the
//               k input windows (keys and values) into the next smem slot;
//   warps 1..8  consumers: rank every record of the chunk (own index plus
//               galloping co-ranks in the other windows), scatter in place
//               into a bank-padded layout, then 16-byte coalesced stores.
constexpr uint32_t PIPE_CONSUMERS = 256;
constexpr uint32_t PIPE_THREADS = 32 + PIPE_CONSUMERS;
constexpr uint32_t PIPE_VT = CHUNK_CAP / PIPE_CONSUMERS;

PS_DEV __host__ constexpr uint32_t align16c(uint32_t x) { return (x + 15u) & ~15u; }

template <class K>
struct PipeLayout {
    static constexpr uint32_t KEY_BYTES = align16c(CHUNK_CAP * (uint32_t)sizeof(K) * 33u / 32u) + 4u * 32u;
    static constexpr uint32_t VAL_BYTES = align16c(CHUNK_CAP * 4u * 33u / 32u) + 4u * 32u;
    static constexpr uint32_t SLOT = KEY_BYTES + VAL_BYTES;
};

struct PipeDesc {
    uint64_t out;
    uint32_t koff[4], voff[4];
    uint32_t woff[5];
    uint32_t len[4];
    uint32_t T, w, par, done;
};

template <class K>
size_t merge_pipe_smem_bytes() {
    return 2 * (size_t)PipeLayout<K>::SLOT + 2 * sizeof(PipeDesc) + 64;
}

template <class K>
PS_DEV uint32_t pad_idx(uint32_t o) {
    return o + (o >> 5);
}

template <class K>
__global__ void __launch_bounds__(PIPE_THREADS) merge_pipe_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                  const uint32_t* __restrict__ chunk2node,
                                                                  const uint4* __restrict__ cuts, uint32_t c0,
                                                                  uint32_t nunits, uint32_t* err) {
    using LY = PipeLayout<K>;
    extern __shared__ __align__(128) uint8_t smem[];
    PipeDesc* desc = reinterpret_cast<PipeDesc*>(smem + 2 * LY::SLOT);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * LY::SLOT + 2 * sizeof(PipeDesc));
    uint64_t* full = bars;       // [2]
    uint64_t* empty = bars + 2;  // [2]
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], PIPE_CONSUMERS / 32);
        mbar_init(&empty[1], PIPE_CONSUMERS / 32);
        mbar_fence_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ------------------------------ producer ------------------------------
        const uint32_t lane = tid;
        for (uint32_t i = 0;; ++i) {
            const uint32_t slot = i & 1;
            const uint32_t u = blockIdx.x + i * gridDim.x;
            if (i >= 2) mbar_wait(&empty[slot], ((i >> 1) - 1) & 1);
            if (lane == 0) {
                PipeDesc& d = desc[slot];
                if (u >= nunits) {
                    d.done = 1;
                    mbar_arrive(&full[slot]);
                } else {
                    const uint32_t c = c0 + u;
                    const Node nd = nodes[chunk2node[c]];
                    const uint32_t q = c - nd.chunk_base;
                    const uint32_t w = nd.arity;
                    uint32_t st[4] = {0, 0, 0, 0}, en[4] = {0, 0, 0, 0};
                    for (uint32_t a = 0; a < w; ++a) en[a] = nd.pos[a + 1] - nd.pos[a];
                    if (q > 0) {
                        const uint4 v = cuts[c];
                        st[0] = v.x; st[1] = v.y; st[2] = v.z; st[3] = v.w;
                    }
                    if (q + 1 < nd.nchunks) {
                        const uint4 v = cuts[c + 1];
                        en[0] = v.x; en[1] = v.y; en[2] = v.z; en[3] = v.w;
                    }
                    const uint32_t par = nd.parity;
                    const K* srcK = bufs.k[par ^ 1];
                    const int32_t* srcV = bufs.v[par ^ 1];
                    uint8_t* sbase = smem + slot * LY::SLOT;
                    uint32_t kcur = 0, vcur = LY::KEY_BYTES, tx = 0, acc = 0;
                    uint64_t out = nd.pos[0];
                    for (uint32_t a = 0; a < 4; ++a) {
                        d.woff[a] = acc;
                        const uint32_t len = a < w ? en[a] - st[a] : 0;
                        d.len[a] = len;
                        if (a < w) out += st[a];
                        if (len == 0) {
                            d.koff[a] = kcur;
                            d.voff[a] = vcur;
                            continue;
                        }
                        const uint64_t e0 = (uint64_t)nd.pos[a] + st[a], e1 = e0 + len;
                        // keys
                        {
                            const uint64_t b0 = e0 * sizeof(K), b1 = e1 * sizeof(K);
                            const uint64_t a0 = b0 & ~15ull, a1 = b1 & ~15ull;
                            d.koff[a] = kcur + (uint32_t)(b0 - a0);
                            if (a1 > a0) {
                                tma_load_1d(sbase + kcur, reinterpret_cast<const uint8_t*>(srcK) + a0,
                                            (uint32_t)(a1 - a0), &full[slot]);
                                tx += (uint32_t)(a1 - a0);
                            }
                            const uint64_t t0 = a1 / sizeof(K) > e0 ? a1 / sizeof(K) : e0;
                            for (uint64_t e = t0; e < e1; ++e)
                                *reinterpret_cast<K*>(sbase + kcur + (e * sizeof(K) - a0)) = srcK[e];
                            kcur += align16c((uint32_t)(b1 - a0));
                        }
                        // values
                        {
                            const uint64_t b0 = e0 * 4, b1 = e1 * 4;
                            const uint64_t a0 = b0 & ~15ull, a1 = b1 & ~15ull;
                            d.voff[a] = vcur + (uint32_t)(b0 - a0);
                            if (a1 > a0) {
                                tma_load_1d(sbase + vcur, reinterpret_cast<const uint8_t*>(srcV) + a0,
                                            (uint32_t)(a1 - a0), &full[slot]);
                                tx += (uint32_t)(a1 - a0);
                            }
                            const uint64_t t0 = a1 / 4 > e0 ? a1 / 4 : e0;
                            for (uint64_t e = t0; e < e1; ++e)
                                *reinterpret_cast<int32_t*>(sbase + vcur + (e * 4 - a0)) = srcV[e];
                            vcur += align16c((uint32_t)(b1 - a0));
                        }
                        acc += len;
                    }
                    d.woff[4] = acc;
                    if (acc > CHUNK_CAP || kcur > LY::KEY_BYTES || vcur > LY::SLOT) {
                        atomicOr(err, ERR_CUT);
                        acc = 0;
                        d.woff[0] = d.woff[1] = d.woff[2] = d.woff[3] = d.woff[4] = 0;
                    }
                    d.T = acc;
                    d.w = w;
                    d.par = par;
                    d.out = out;
                    d.done = 0;
                    mbar_arrive_tx(&full[slot], tx);
                }
            }
            const uint32_t stop = __shfl_sync(PS_FULL, u >= nunits ? 1u : 0u, 0);
            if (stop) break;
        }
        return;
    }

    // ------------------------------ consumers ---------------------------------
    const uint32_t ctid = tid - 32;
    const uint32_t clane = ctid & 31;
    for (uint32_t i = 0;; ++i) {
        const uint32_t slot = i & 1;
        mbar_wait(&full[slot], (i >> 1) & 1);
        const PipeDesc& d = desc[slot];
        if (d.done) break;
        const uint32_t T = d.T, w = d.w, par = d.par;
        const uint64_t out = d.out;
        const uint32_t* woff = d.woff;  // shared memory (dynamic window index)
        const uint32_t* len = d.len;
        const uint32_t* koff = d.koff;
        const uint32_t* voff = d.voff;
        const uint32_t wo1 = woff[1], wo2 = woff[2], wo3 = woff[3];
        uint8_t* sbase = smem + slot * LY::SLOT;
        const uint32_t i0 = (ctid * T) / PIPE_CONSUMERS;
        const uint32_t i1 = ((ctid + 1) * T) / PIPE_CONSUMERS;
        K xk[PIPE_VT];
        int32_t xv[PIPE_VT];
        uint32_t xr[PIPE_VT];
        uint32_t cur[4] = {0, 0, 0, 0};
        int cur_a = -1;
#pragma unroll
        for (uint32_t v = 0; v < PIPE_VT; ++v) {
            const uint32_t e = i0 + v;
            xr[v] = INF32;
            if (e < i1) {
                const uint32_t a = (e >= wo1) + (e >= wo2) + (e >= wo3);
                if ((int)a != cur_a) {
                    cur_a = (int)a;
                    cur[0] = cur[1] = cur[2] = cur[3] = 0;
                }
                const uint32_t p = e - woff[a];
                const K x = reinterpret_cast<const K*>(sbase + koff[a])[p];
                uint32_t rank = p;
#pragma unroll
                for (uint32_t b = 0; b < 4; ++b) {
                    if (b < w && b != a) {
                        const K* wb = reinterpret_cast<const K*>(sbase + koff[b]);
                        cur[b] = b < a ? gallop<K, true>(wb, len[b], cur[b], x) : gallop<K, false>(wb, len[b], cur[b], x);
                        rank += cur[b];
                    }
                }
                xk[v] = x;
                xv[v] = reinterpret_cast<const int32_t*>(sbase + voff[a])[p];
                xr[v] = rank;
            }
        }
        consumer_sync();
        K* ok = reinterpret_cast<K*>(sbase);
        int32_t* ov = reinterpret_cast<int32_t*>(sbase + LY::KEY_BYTES);
#pragma unroll
        for (uint32_t v = 0; v < PIPE_VT; ++v) {
            if (xr[v] != INF32) {
                const uint32_t o = pad_idx<K>(xr[v]);
                ok[o] = xk[v];
                ov[o] = xv[v];
            }
        }
        consumer_sync();
        // 16-byte stores aligned in global memory
        K* __restrict__ dstK = bufs.k[par];
        int32_t* __restrict__ dstV = bufs.v[par];
        {
            constexpr uint32_t E = 16 / sizeof(K);
            const uint32_t al = (uint32_t)(out % E);
            const uint32_t ngroups = (al + T + E - 1) / E;
            for (uint32_t j = ctid; j < ngroups; j += PIPE_CONSUMERS) {
                const int32_t o0 = (int32_t)(j * E) - (int32_t)al;  // chunk index of the group's first element
                if (o0 >= 0 && o0 + (int32_t)E <= (int32_t)T) {
                    if (E == 4) {
                        uint4 vv;
                        uint32_t* pv = reinterpret_cast<uint32_t*>(&vv);
#pragma unroll
                        for (uint32_t t = 0; t < E; ++t) {
                            const K kk = ok[pad_idx<K>(o0 + t)];
                            pv[t] = *reinterpret_cast<const uint32_t*>(&kk);
                        }
                        *reinterpret_cast<uint4*>(dstK + out + o0) = vv;
                    } else {
                        uint4 vv;
                        unsigned long long* pv = reinterpret_cast<unsigned long long*>(&vv);
#pragma unroll
                        for (uint32_t t = 0; t < E; ++t) {
                            const K kk = ok[pad_idx<K>(o0 + t)];
                            pv[t] = *reinterpret_cast<const unsigned long long*>(&kk);
                        }
                        *reinterpret_cast<uint4*>(dstK + out + o0) = vv;
                    }
                } else {
                    for (uint32_t t = 0; t < E; ++t) {
                        const int32_t o = o0 + (int32_t)t;
                        if (o >= 0 && o < (int32_t)T) dstK[out + o] = ok[pad_idx<K>(o)];
                    }
                }
            }
            const uint32_t alv = (uint32_t)(out % 4);
            const uint32_t ngv = (alv + T + 3) / 4;
            for (uint32_t j = ctid; j < ngv; j += PIPE_CONSUMERS) {
                const int32_t o0 = (int32_t)(j * 4) - (int32_t)alv;
                if (o0 >= 0 && o0 + 4 <= (int32_t)T) {
                    int4 vv;
                    vv.x = ov[pad_idx<K>(o0)];
                    vv.y = ov[pad_idx<K>(o0 + 1)];
                    vv.z = ov[pad_idx<K>(o0 + 2)];
                    vv.w = ov[pad_idx<K>(o0 + 3)];
                    *reinterpret_cast<int4*>(dstV + out + o0) = vv;
                } else {
                    for (int32_t t = 0; t < 4; ++t) {
                        const int32_t o = o0 + t;
                        if (o >= 0 && o < (int32_t)T) dstV[out + o] = ov[pad_idx<K>(o)];
                    }
                }
            }
        }
        __syncwarp();
        if (clane == 0) mbar_arrive(&empty[slot]);
    }
}

}  // namespace ps

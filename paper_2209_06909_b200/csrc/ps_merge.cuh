// ps_merge.cuh -- N3: batched stable k-way merges (one launch per tree level).
//
// Replaces merges.py:75-500 (merge_2way_*, merge_3way, merge_4way_*).  A stable
// k-way merge has a unique output (ties go to the lower-index run,
// merges.py:1-8), i.e. the merge under the strict order (key, run, position).
//
// Big nodes are cut into chunks: cut (a, j) is the record at position j*S of
// run a (S = CHUNK_CAP / arity); its rank in every other run b is a search
// (<= for b < a, < for b > a) and its index in the merged cut order follows
// directly from those ranks.  Between consecutive cuts there are at most S
// records of each run, so every chunk holds <= CHUNK_CAP records.
//
// merge_pipe_kernel (persistent, warp-specialized):
//   producer warp  -- reads the descriptors of 32 chunks at once, packs
//                     consecutive chunks of a node into units of <= CHUNK_CAP
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

// Partition: one warp per chunk of the stage [c0, c1); the first chunk of each
// node gets the zero cut.
template <class K>
__global__ void __launch_bounds__(256) merge_partition_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                              const uint32_t* __restrict__ chunk2node, uint32_t c0,
                                                              uint32_t c1, uint4* __restrict__ cuts) {
    const uint32_t c = c0 + blockIdx.x * 8 + warp_id();
    if (c >= c1) return;
    const uint32_t lane = lane_id();
    const Node nd = nodes[chunk2node[c]];
    uint32_t q = c - nd.chunk_base;
    if (q == 0) {
        if (lane == 0) cuts[c] = make_uint4(0, 0, 0, 0);
        return;
    }
    q -= 1;
    const uint32_t w = nd.arity;
    const uint32_t S = CHUNK_CAP / w;
    const K* src = bufs.k[nd.parity ^ 1];
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
    uint32_t rk[4] = {0, 0, 0, 0};
    uint32_t mm = j - 1;
#pragma unroll
    for (uint32_t bb = 0; bb < 4; ++bb) {
        if (bb >= w) break;
        if (bb == a) {
            rk[bb] = j * S;
            continue;
        }
        const K* run = src + nd.pos[bb];
        rk[bb] = bb < a ? warp_count_pred<K, true>(run, L[bb], y) : warp_count_pred<K, false>(run, L[bb], y);
        mm += rk[bb] ? (rk[bb] - 1) / S : 0;
    }
    if (lane == 0) cuts[nd.chunk_base + 1 + mm] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
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
// named barrier 1 over the consumer warps only
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
    __shared__ uint32_t s_off[SMALL_WARPS][8];
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
constexpr uint32_t PIPE_CONSUMERS = 256;
constexpr uint32_t PIPE_THREADS = 32 + PIPE_CONSUMERS;

PS_DEV __host__ constexpr uint32_t align16c(uint32_t x) { return (x + 15u) & ~15u; }
PS_DEV uint32_t padi(uint32_t o) { return o + (o >> 5); }  // bank padding: one slot per 32

template <class K>
struct PipeLayout {
    static constexpr uint32_t PADN = CHUNK_CAP + CHUNK_CAP / 32 + 8;
    // slot = TMA landing zone for the k windows (with 16B alignment slack), and
    // afterwards the padded output of the last pass
    static constexpr uint32_t KEY_BYTES = align16c(PADN * (uint32_t)sizeof(K)) + MAX_WAY * 32u;
    static constexpr uint32_t VAL_BYTES = align16c(PADN * 4u) + MAX_WAY * 32u;
    static constexpr uint32_t SLOT = KEY_BYTES + VAL_BYTES;
    // scratch for the first-pass results X || Y (padded)
    static constexpr uint32_t SKEY = align16c(PADN * (uint32_t)sizeof(K));
    static constexpr uint32_t SCRATCH = SKEY + align16c(PADN * 4u);
};

struct PipeDesc {
    uint64_t out;  // global element index of the unit's first output
    uint32_t koff[4], voff[4], len[4];
    uint32_t T, w, par, done;
};

template <class K>
size_t merge_pipe_smem_bytes() {
    return 2 * (size_t)PipeLayout<K>::SLOT + PipeLayout<K>::SCRATCH + 2 * sizeof(PipeDesc) + 64;
}

// A read-only sorted sequence in shared memory (optionally bank-padded).
template <class K>
struct SeqView {
    const K* k;
    const int32_t* v;
    uint32_t len;
    bool pad;
    PS_DEV uint32_t at(uint32_t i) const { return pad ? padi(i) : i; }
};

// Merge-path: produce outputs [o0, o1) of merge(A, B) (ties to A) into the
// padded arrays ok/ov at positions base + o.
template <class K>
PS_DEV void merge_range(const SeqView<K>& A, const SeqView<K>& B, K* ok, int32_t* ov, uint32_t base, uint32_t o0,
                        uint32_t o1) {
    if (o0 >= o1) return;
    // diagonal search: i = # of A among the first o0 outputs
    uint32_t lo = o0 > B.len ? o0 - B.len : 0;
    uint32_t hi = o0 < A.len ? o0 : A.len;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (!(B.k[B.at(o0 - 1 - mid)] < A.k[A.at(mid)]))  // A[mid] <= B[o0-1-mid]
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = o0 - lo;
    K a = i < A.len ? A.k[A.at(i)] : K(0);
    K b = j < B.len ? B.k[B.at(j)] : K(0);
    for (uint32_t o = o0; o < o1; ++o) {
        const bool takeA = j >= B.len || (i < A.len && !(b < a));
        const uint32_t po = padi(base + o);
        if (takeA) {
            ok[po] = a;
            ov[po] = A.v[A.at(i)];
            ++i;
            if (i < A.len) a = A.k[A.at(i)];
        } else {
            ok[po] = b;
            ov[po] = B.v[B.at(j)];
            ++j;
            if (j < B.len) b = B.k[B.at(j)];
        }
    }
}

template <class K>
__global__ void __launch_bounds__(PIPE_THREADS) merge_pipe_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                  const uint32_t* __restrict__ chunk2node,
                                                                  const uint4* __restrict__ cuts, uint32_t c0,
                                                                  uint32_t nchunks, uint32_t* err) {
    using LY = PipeLayout<K>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* scratch = smem + 2 * LY::SLOT;
    PipeDesc* desc = reinterpret_cast<PipeDesc*>(scratch + LY::SCRATCH);
    uint64_t* bars = reinterpret_cast<uint64_t*>(desc + 2);
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
        const uint32_t cbeg = c0 + (uint32_t)(((uint64_t)nchunks * blockIdx.x) / gridDim.x);
        const uint32_t cend = c0 + (uint32_t)(((uint64_t)nchunks * (blockIdx.x + 1)) / gridDim.x);
        uint32_t unit = 0;
        for (uint32_t c = cbeg; c < cend;) {
            // batch descriptors of chunks c .. c+31 (lane l <-> chunk c+l)
            const uint32_t x = c + lane;
            const bool xv = x < cend;
            uint32_t nid = xv ? chunk2node[x] : 0;
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
                nid = INF32;
            }
            const uint32_t nvalid = min(32u, cend - c);
            uint32_t u = 0;
            while (u < nvalid) {
                // unit = lanes u..V of the same node with total <= CHUNK_CAP
                const uint32_t nid_u = __shfl_sync(PS_FULL, nid, u);
                const uint32_t sx = __shfl_sync(PS_FULL, st.x, u), sy = __shfl_sync(PS_FULL, st.y, u);
                const uint32_t sz = __shfl_sync(PS_FULL, st.z, u), sw = __shfl_sync(PS_FULL, st.w, u);
                const uint32_t tot = (en.x - sx) + (en.y - sy) + (en.z - sz) + (en.w - sw);
                const bool ok = lane >= u && lane < nvalid && nid == nid_u && tot <= CHUNK_CAP;
                uint32_t bal = __ballot_sync(PS_FULL, ok) >> u;
                // contiguous run of ok lanes starting at u
                const uint32_t runlen = __ffs(~bal) ? __ffs(~bal) - 1 : 32 - u;
                const uint32_t V = u + max(runlen, 1u) - 1;
                const uint32_t ex = __shfl_sync(PS_FULL, en.x, V), ey = __shfl_sync(PS_FULL, en.y, V);
                const uint32_t ez = __shfl_sync(PS_FULL, en.z, V), ew = __shfl_sync(PS_FULL, en.w, V);
                // node fields of lane u
                uint32_t npos[5];
#pragma unroll
                for (int t = 0; t < 5; ++t) npos[t] = __shfl_sync(PS_FULL, nd.pos[t], u);
                const uint32_t w = __shfl_sync(PS_FULL, (uint32_t)nd.arity, u);
                const uint32_t par = __shfl_sync(PS_FULL, (uint32_t)nd.parity, u);
                // ---- stage the unit into slot (unit & 1) ----
                const uint32_t slot = unit & 1;
                if (unit >= 2) mbar_wait(&empty[slot], ((unit >> 1) - 1) & 1);
                uint8_t* sbase = smem + slot * LY::SLOT;
                const uint32_t sv4[4] = {sx, sy, sz, sw};
                const uint32_t ev4[4] = {ex, ey, ez, ew};
                // lane a (< w) handles keys of window a, lane 4+a values of window a
                const uint32_t wa = lane & 3;
                const bool is_val = lane >= 4;
                uint32_t len = 0, phase = 0, bytes_region = 0, tx = 0;
                uint64_t e0 = 0;
                const uint32_t ebytes = is_val ? 4u : (uint32_t)sizeof(K);
                if (lane < 8 && wa < w) {
                    len = ev4[wa] - sv4[wa];
                    e0 = (uint64_t)npos[wa] + sv4[wa];
                    const uint64_t b0 = e0 * ebytes;
                    phase = (uint32_t)(b0 & 15);
                    bytes_region = len ? align16c(phase + len * ebytes) : 0;
                }
                // exclusive prefix of region sizes within the key lanes (0..3) and value lanes (4..7)
                uint32_t pre = 0;
#pragma unroll
                for (uint32_t t = 0; t < 4; ++t) {
                    const uint32_t r = __shfl_sync(PS_FULL, bytes_region, (lane & 4) + t);
                    if (t < wa) pre += r;
                }
                const uint32_t region = (is_val ? LY::KEY_BYTES : 0u) + pre;
                if (lane < 8 && wa < w && len) {
                    const uint8_t* src = is_val ? reinterpret_cast<const uint8_t*>(bufs.v[par ^ 1])
                                                : reinterpret_cast<const uint8_t*>(bufs.k[par ^ 1]);
                    const uint64_t b0 = e0 * ebytes, b1 = (e0 + len) * ebytes;
                    const uint64_t a0 = b0 & ~15ull, a1 = b1 & ~15ull;
                    if (a1 > a0) {
                        tma_load_1d(sbase + region, src + a0, (uint32_t)(a1 - a0), &full[slot]);
                        tx = (uint32_t)(a1 - a0);
                    }
                    // tail bytes [max(a1, b0), b1) with ordinary loads
                    for (uint64_t bb = (a1 > b0 ? a1 : b0); bb < b1; bb += ebytes) {
                        if (is_val)
                            *reinterpret_cast<int32_t*>(sbase + region + (bb - a0)) =
                                *reinterpret_cast<const int32_t*>(src + bb);
                        else
                            *reinterpret_cast<K*>(sbase + region + (bb - a0)) = *reinterpret_cast<const K*>(src + bb);
                    }
                }
                uint32_t txs = tx;
                for (int d = 16; d; d >>= 1) txs += __shfl_xor_sync(PS_FULL, txs, d);
                uint32_t total = 0;  // window lengths live in key lanes 0..3
#pragma unroll
                for (uint32_t t = 0; t < 4; ++t) total += __shfl_sync(PS_FULL, len, t);
                if (lane < 8) {
                    PipeDesc& d = desc[slot];
                    if (lane < 4) {
                        d.koff[wa] = region + phase;
                        d.len[wa] = len;
                    } else {
                        d.voff[wa] = region + phase;
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    PipeDesc& d = desc[slot];
                    uint64_t out = npos[0];
                    for (uint32_t t = 0; t < w; ++t) out += sv4[t];
                    d.out = out;
                    d.T = total;
                    d.w = w;
                    d.par = par;
                    d.done = 0;
                    if (total > CHUNK_CAP) atomicOr(err, ERR_CUT);
                    mbar_arrive_tx(&full[slot], txs);
                }
                unit++;
                u = V + 1;
            }
            c += nvalid;
        }
        // termination marker
        const uint32_t slot = unit & 1;
        if (unit >= 2) mbar_wait(&empty[slot], ((unit >> 1) - 1) & 1);
        if (lane == 0) {
            desc[slot].done = 1;
            mbar_arrive(&full[slot]);
        }
        return;
    }

    // ------------------------------ consumers ---------------------------------
    const uint32_t ctid = tid - 32;
    const uint32_t clane = ctid & 31;
    K* const xk = reinterpret_cast<K*>(scratch);
    int32_t* const xv = reinterpret_cast<int32_t*>(scratch + LY::SKEY);
    for (uint32_t i = 0;; ++i) {
        const uint32_t slot = i & 1;
        mbar_wait(&full[slot], (i >> 1) & 1);
        const PipeDesc& d = desc[slot];
        if (d.done) break;
        const uint32_t T = d.T, w = d.w, par = d.par;
        const uint64_t out = d.out;
        uint8_t* sbase = smem + slot * LY::SLOT;
        SeqView<K> win[4];
#pragma unroll
        for (uint32_t a = 0; a < 4; ++a) {
            win[a].k = reinterpret_cast<const K*>(sbase + d.koff[a]);
            win[a].v = reinterpret_cast<const int32_t*>(sbase + d.voff[a]);
            win[a].len = a < w ? d.len[a] : 0;
            win[a].pad = false;
        }
        const uint32_t o0 = (uint32_t)(((uint64_t)T * ctid) / PIPE_CONSUMERS);
        const uint32_t o1 = (uint32_t)(((uint64_t)T * (ctid + 1)) / PIPE_CONSUMERS);
        K* ok;
        int32_t* ov;
        if (w >= 3) {
            // pass 1: X = merge(A, B) -> scratch[0, LA+LB); Y = merge(C, D) (or C) -> scratch[LA+LB, T)
            const uint32_t LX = win[0].len + win[1].len;
            merge_range<K>(win[0], win[1], xk, xv, 0, o0, min(o1, LX));
            merge_range<K>(win[2], win[3], xk, xv, LX, o0 > LX ? o0 - LX : 0, o1 > LX ? o1 - LX : 0);
            consumer_sync();
            // pass 2: merge X (scratch[0, LX)) and Y (scratch[LX, T)) into the
            // slot, whose input windows are fully consumed
            ok = reinterpret_cast<K*>(sbase);
            ov = reinterpret_cast<int32_t*>(sbase + LY::KEY_BYTES);
            // merge X and Y where Y element j lives at padded index LX + j
            {
                uint32_t lo = o0 > (T - LX) ? o0 - (T - LX) : 0;
                uint32_t hi = o0 < LX ? o0 : LX;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (!(xk[padi(LX + o0 - 1 - mid)] < xk[padi(mid)]))
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                uint32_t ii = lo, jj = o0 - lo;
                const uint32_t LY_ = T - LX;
                K a = ii < LX ? xk[padi(ii)] : K(0);
                K b = jj < LY_ ? xk[padi(LX + jj)] : K(0);
                for (uint32_t o = o0; o < o1; ++o) {
                    const bool takeA = jj >= LY_ || (ii < LX && !(b < a));
                    const uint32_t po = padi(o);
                    if (takeA) {
                        ok[po] = a;
                        ov[po] = xv[padi(ii)];
                        ++ii;
                        if (ii < LX) a = xk[padi(ii)];
                    } else {
                        ok[po] = b;
                        ov[po] = xv[padi(LX + jj)];
                        ++jj;
                        if (jj < LY_) b = xk[padi(LX + jj)];
                    }
                }
            }
        } else {
            // 2-way: merge(A, B) straight into scratch
            ok = xk;
            ov = xv;
            merge_range<K>(win[0], win[1], ok, ov, 0, o0, o1);
        }
        consumer_sync();
        // 16-byte stores aligned in global memory
        K* __restrict__ dstK = bufs.k[par];
        int32_t* __restrict__ dstV = bufs.v[par];
        {
            constexpr uint32_t E = 16 / sizeof(K);
            const uint32_t al = (uint32_t)(out % E);
            const uint32_t ng = (al + T + E - 1) / E;
            for (uint32_t j = ctid; j < ng; j += PIPE_CONSUMERS) {
                const int32_t g0 = (int32_t)(j * E) - (int32_t)al;
                if (g0 >= 0 && g0 + (int32_t)E <= (int32_t)T) {
                    uint4 vv;
                    K* pv = reinterpret_cast<K*>(&vv);
#pragma unroll
                    for (uint32_t t = 0; t < E; ++t) pv[t] = ok[padi(g0 + t)];
                    *reinterpret_cast<uint4*>(dstK + out + g0) = vv;
                } else {
                    for (uint32_t t = 0; t < E; ++t) {
                        const int32_t o = g0 + (int32_t)t;
                        if (o >= 0 && o < (int32_t)T) dstK[out + o] = ok[padi(o)];
                    }
                }
            }
            const uint32_t alv = (uint32_t)(out % 4);
            const uint32_t ngv = (alv + T + 3) / 4;
            for (uint32_t j = ctid; j < ngv; j += PIPE_CONSUMERS) {
                const int32_t g0 = (int32_t)(j * 4) - (int32_t)alv;
                if (g0 >= 0 && g0 + 4 <= (int32_t)T) {
                    int4 vv;
                    vv.x = ov[padi(g0)];
                    vv.y = ov[padi(g0 + 1)];
                    vv.z = ov[padi(g0 + 2)];
                    vv.w = ov[padi(g0 + 3)];
                    *reinterpret_cast<int4*>(dstV + out + g0) = vv;
                } else {
                    for (int32_t t = 0; t < 4; ++t) {
                        const int32_t o = g0 + t;
                        if (o >= 0 && o < (int32_t)T) dstV[out + o] = ov[padi(o)];
                    }
                }
            }
        }
        consumer_sync();  // scratch / slot reads done before the next unit
        if (clane == 0) mbar_arrive(&empty[slot]);
    }
}

}  // namespace ps

// ps_shard.cuh -- N6: single-pass cross-shard merge for the multi-GPU mode.
//
// Rank g of G has sorted its contiguous shard (shard h holds global indices
// [off_h, off_h + n_h)); the payload carried through the local sort is the
// global index.  Its output slab is global ranks [t0, t1) of the stable order
// (key, shard, position) == (key, global index).  The slab is produced in one
// pass over the peer shards (NVLink loads, no NCCL, no gathered copy):
//
//  1. co-ranks of t0 and t1 by parallel bracketing (shard_select_kernel):
//     every round, SEL_CANDIDATES evenly spaced candidates of every shard's
//     current window are ranked against all shards at once and the windows
//     shrink by ~65x; a fixed number of rounds, no host round trip;
//  2. every shard publishes a sample array (every XS_STRIDE-th key, 128
//     bytes apart); the slab's sample windows are copied to local memory;
//  3. cuts: every m-th sample of every shard inside the slab is a cut
//     element x.  Its rank among the other shards' samples (local binary
//     searches) brackets its exact rank in each shard to a window of
//     XS_STRIDE positions, and fixes its index in the merged cut order
//     exactly (cuts are samples), so every cut writes its boundary row
//     directly; between consecutive cuts each shard holds <= m*XS_STRIDE
//     records;
//  4. xs_merge_kernel: consecutive chunks are packed into units; a unit's
//     bracketed shard windows are loaded once (asynchronous copies from the
//     peers into shared memory), the exact boundaries are found inside the
//     loaded windows (shared-memory binary searches against the cut
//     elements), the G windows are merged by ceil(log2 G) stable pairwise
//     merge-path passes in shared memory, and the unit leaves with coalesced
//     stores into the local slab.
// Everything after the launch is stream-ordered on the device.
#pragma once

#include "ps_common.cuh"
#include "ps_merge.cuh"

namespace ps {

constexpr uint32_t MAX_SHARDS = 8;
constexpr uint32_t SEL_CANDIDATES = 64;  // per shard per bracketing round

// sample stride: 128 bytes of keys (32 4-byte keys, 16 8-byte keys)
template <class K>
PS_DEV __host__ constexpr uint32_t xs_stride() {
    return 128u / (uint32_t)sizeof(K);
}
// merge geometry: two CTAs per SM (one loads while the other merges).  A
// thread produces VT consecutive outputs of every pass; VT is odd, so the
// k-th outputs of a warp's lanes land in distinct banks.
constexpr uint32_t XM_THREADS = 256;
template <class K>
PS_DEV __host__ constexpr uint32_t xm_vt() {
    return sizeof(K) == 4 ? 15u : 9u;
}
template <class K>
PS_DEV __host__ constexpr uint32_t xm_cap() {  // loaded records per unit
    return xm_vt<K>() * XM_THREADS;
}
template <class K>
PS_DEV __host__ constexpr size_t xm_smem_bytes() {  // three SoA record buffers (+ over-read slack)
    return 3 * (size_t)xm_cap<K>() * (sizeof(K) + 4) + 128;
}

template <class K>
struct ShardSet {
    const K* k[MAX_SHARDS];
    const int32_t* v[MAX_SHARDS];
    const K* smp[MAX_SHARDS];  // published sample arrays (NULL: read keys[i * stride])
    uint64_t n[MAX_SHARDS];
    uint32_t G;
};

// Boundary row: the exact rank E_b of the boundary element in shard b lies in
// [lo[b], hi[b]] (lo == hi for exact rows: the slab ends and the cut's own
// shard).  key/shard/pos identify the cut element (shard = INF32: exact row).
template <class K>
struct XRow {
    uint32_t lo[MAX_SHARDS];
    uint32_t hi[MAX_SHARDS];
    K key;
    uint32_t shard;
    uint32_t pos;
};

// Device plan of one slab (written by xs_plan_kernel).
struct XPlan {
    uint32_t c0[MAX_SHARDS], c1[MAX_SHARDS];  // exact co-ranks of t0 and t1
    uint32_t w0[MAX_SHARDS], w1[MAX_SHARDS];  // sample window [w0, w1) of each shard
    uint32_t sbase[MAX_SHARDS + 1];           // local sample copy offsets
    uint32_t cbase[MAX_SHARDS + 1];           // cut candidate offsets (cuts of shard a)
    uint32_t j0[MAX_SHARDS];                  // first cut ordinal of each shard (ceil(w0 / m))
    uint32_t ncuts, nrows, m, ok;
};

// element (b, q) with key z precedes element (a, .) with key y in (key, shard) order
template <class K>
PS_DEV bool xs_precedes(K z, uint32_t b, K y, uint32_t a) {
    return z < y || (!(y < z) && b < a);
}

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

// bounds layout: [target (0: t0, 1: t1)][lo | hi][MAX_SHARDS]; the true
// co-rank c_h of the target lies in [lo_h, hi_h].
template <class K>
__global__ void xs_init_kernel(ShardSet<K> S, uint64_t t0, uint64_t t1, unsigned long long* bounds,
                               uint64_t* targets) {
    pdl_wait();
    const uint32_t h = threadIdx.x;
    uint64_t N = 0;
    for (uint32_t g = 0; g < S.G; ++g) N += S.n[g];
    for (uint32_t t = 0; t < 2; ++t) {
        const uint64_t tg = t ? t1 : t0;
        uint64_t lo = 0, hi = 0;
        if (h < S.G) {
            const uint64_t rest = N - S.n[h];
            lo = tg > rest ? tg - rest : 0;
            hi = tg < S.n[h] ? tg : S.n[h];
        }
        if (h < MAX_SHARDS) {
            bounds[t * 2 * MAX_SHARDS + h] = lo;
            bounds[t * 2 * MAX_SHARDS + MAX_SHARDS + h] = hi;
        }
    }
    if (h == 0) {
        targets[0] = t0;
        targets[1] = t1;
    }
}

// One bracketing round for both targets (blockIdx.y).  Grid.x =
// G * SEL_CANDIDATES / warps-per-block; one warp per candidate, lane = shard.
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

PS_DEV uint32_t cdiv32(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// One thread: check convergence of the bracketing and lay out the slab's
// samples and cuts (m = samples per cut).
template <class K>
__global__ void xs_plan_kernel(ShardSet<K> S, const unsigned long long* __restrict__ bounds, uint64_t t0,
                               uint64_t t1, uint32_t m, XPlan* plan, uint32_t* err) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    constexpr uint32_t s = xs_stride<K>();
    XPlan P;
    uint64_t sum0 = 0, sum1 = 0;
    bool ok = true;
    P.sbase[0] = 0;
    P.cbase[0] = 0;
    for (uint32_t h = 0; h < MAX_SHARDS; ++h) {
        uint32_t c0 = 0, c1 = 0;
        if (h < S.G) {
            ok &= bounds[h] == bounds[MAX_SHARDS + h] && bounds[2 * MAX_SHARDS + h] == bounds[3 * MAX_SHARDS + h];
            c0 = (uint32_t)bounds[h];
            c1 = (uint32_t)bounds[2 * MAX_SHARDS + h];
            ok &= c0 <= c1;
        }
        sum0 += c0;
        sum1 += c1;
        P.c0[h] = c0;
        P.c1[h] = c1;
        P.w0[h] = cdiv32(c0, s);
        P.w1[h] = cdiv32(c1, s);
        P.j0[h] = cdiv32(P.w0[h], m);
        const uint32_t ncut = cdiv32(P.w1[h], m) - P.j0[h];
        P.sbase[h + 1] = P.sbase[h] + (P.w1[h] - P.w0[h]);
        P.cbase[h + 1] = P.cbase[h] + ncut;
    }
    ok &= sum0 == t0 && sum1 == t1;
    P.ncuts = P.cbase[MAX_SHARDS];
    P.nrows = P.ncuts + 2;
    P.m = m;
    P.ok = ok ? 1u : 0u;
    if (!ok) atomicOr(err, ERR_CUT);
    *plan = P;
}

// Local copy of the slab's sample windows (peer reads of the published
// samples, or strided reads of the keys when a shard published none).
template <class K>
__global__ void __launch_bounds__(256) xs_sample_copy_kernel(ShardSet<K> S, const XPlan* __restrict__ plan,
                                                             K* __restrict__ smp) {
    pdl_wait();
    __shared__ uint32_t sb[MAX_SHARDS + 1], w0[MAX_SHARDS];
    if (threadIdx.x <= MAX_SHARDS) sb[threadIdx.x] = plan->sbase[threadIdx.x];
    if (threadIdx.x < MAX_SHARDS) w0[threadIdx.x] = plan->w0[threadIdx.x];
    __syncthreads();
    const uint32_t total = sb[MAX_SHARDS];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        uint32_t h = 0;
        while (h + 1 < S.G && i >= sb[h + 1]) ++h;
        const uint64_t q = (uint64_t)w0[h] + (i - sb[h]);
        smp[i] = S.smp[h] ? S.smp[h][q] : S.k[h][q * xs_stride<K>()];
    }
}

// One thread per cut: cut (a, j) is the sample of shard a with index j*m,
// element (a, p = j*m*stride).  Writes boundary row 1 + (its index in the
// merged cut order); thread 0 also writes the exact rows 0 and nrows-1.
template <class K>
__global__ void __launch_bounds__(256) xs_cuts_kernel(ShardSet<K> S, const XPlan* __restrict__ plan,
                                                      const K* __restrict__ smp, XRow<K>* __restrict__ rows) {
    pdl_wait();
    constexpr uint32_t s = xs_stride<K>();
    __shared__ XPlan P;
    if (threadIdx.x == 0) P = *plan;
    __syncthreads();
    if (!P.ok) return;
    const uint32_t G = S.G;
    const uint32_t m = P.m;
    if (blockIdx.x == 0 && threadIdx.x < 2) {
        XRow<K> r;
        for (uint32_t h = 0; h < MAX_SHARDS; ++h) r.lo[h] = r.hi[h] = threadIdx.x ? P.c1[h] : P.c0[h];
        r.key = K(0);
        r.shard = INF32;
        r.pos = 0;
        rows[threadIdx.x ? P.nrows - 1 : 0] = r;
    }
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < P.ncuts; c += gridDim.x * blockDim.x) {
        uint32_t a = 0;
        while (a + 1 < G && c >= P.cbase[a + 1]) ++a;
        const uint32_t i = (P.j0[a] + (c - P.cbase[a])) * m;  // sample index of the cut
        const K x = smp[P.sbase[a] + (i - P.w0[a])];
        XRow<K> r;
        uint32_t idx = 0;
        for (uint32_t b = 0; b < MAX_SHARDS; ++b) {
            uint32_t lo = 0, hi = 0;
            if (b < G) {
                uint32_t rb;  // samples of shard b preceding x
                if (b == a) {
                    rb = i;
                    lo = hi = i * s;
                } else {
                    const K* sw = smp + P.sbase[b];
                    uint32_t l = 0, h = P.w1[b] - P.w0[b];
                    while (l < h) {
                        const uint32_t mid = (l + h) >> 1;
                        const bool pre = xs_precedes<K>(sw[mid], b, x, a);
                        l = pre ? mid + 1 : l;
                        h = pre ? h : mid;
                    }
                    rb = P.w0[b] + l;
                    // exact rank E in ((rb - 1) * s, rb * s], inside the slab's [c0, c1]
                    lo = rb ? (rb - 1) * s + 1 : 0;
                    hi = rb * s;
                    lo = min(max(lo, P.c0[b]), P.c1[b]);
                    hi = min(max(hi, P.c0[b]), P.c1[b]);
                }
                idx += cdiv32(rb, m) - P.j0[b];
            }
            r.lo[b] = lo;
            r.hi[b] = hi;
        }
        r.key = x;
        r.shard = a;
        r.pos = i * s;
        rows[1 + idx] = r;
    }
}

PS_DEV void cp_async4(void* dst, const void* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
PS_DEV void cp_async8(void* dst, const void* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
PS_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Persistent unit loop over the boundary rows (chunks [row c, row c+1]).
template <class K>
__global__ void __launch_bounds__(XM_THREADS) xs_merge_kernel(ShardSet<K> S, const XPlan* __restrict__ plan,
                                                              const XRow<K>* __restrict__ rows, K* __restrict__ out_k,
                                                              int32_t* __restrict__ out_v, uint64_t t0,
                                                              uint32_t* err) {
    pdl_wait();
    constexpr uint32_t CAP = xm_cap<K>(), VT = xm_vt<K>();
    extern __shared__ __align__(128) uint8_t smem[];
    // buffer q: CAP keys then CAP values
    auto BK = [&](uint32_t q) { return reinterpret_cast<K*>(smem + (size_t)q * CAP * (sizeof(K) + 4)); };
    auto BV = [&](uint32_t q) {
        return reinterpret_cast<int32_t*>(smem + (size_t)q * CAP * (sizeof(K) + 4) + (size_t)CAP * sizeof(K));
    };
    __shared__ uint32_t s_L[MAX_SHARDS], s_off[MAX_SHARDS + 1], s_E0[MAX_SHARDS], s_E1[MAX_SHARDS];
    __shared__ uint32_t s_ro[MAX_SHARDS + 1], s_rl[MAX_SHARDS];  // runs of the current pass: offset, length
    __shared__ uint32_t s_next;
    __shared__ unsigned long long s_out;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    const uint32_t G = S.G;
    const uint32_t nrows = plan->nrows;
    if (!plan->ok) return;
    const uint32_t nch = nrows - 1;
    const uint32_t cbeg = (uint32_t)(((uint64_t)nch * blockIdx.x) / gridDim.x);
    const uint32_t cend = (uint32_t)(((uint64_t)nch * (blockIdx.x + 1)) / gridDim.x);
    // warp 0: pack chunks c .. c2-1 (rows c .. c2) into a unit of <= CAP loaded
    // records; its bracketed window of shard b is [s_L[b], s_L[b] + len) at
    // buffer offset s_off[b]
    auto pack = [&](uint32_t c) {
        const uint32_t r = c + 1 + lane;
        uint32_t tot = INF32;
        if (r <= cend) {
            tot = 0;
            for (uint32_t b = 0; b < G; ++b) tot += rows[r].hi[b] - rows[c].lo[b];
        }
        const uint32_t fit = __ballot_sync(PS_FULL, tot <= CAP);
        const uint32_t nfit = __ffs(~fit) ? __ffs(~fit) - 1 : 32;  // leading chunks that fit
        const uint32_t c2 = c + max(nfit, 1u);
        if (lane == 0) {
            if (nfit == 0) atomicOr(err, ERR_CUT);
            s_next = c2;
        }
        if (lane < MAX_SHARDS) {
            const uint32_t L = lane < G ? rows[c].lo[lane] : 0;
            const uint32_t H = lane < G ? rows[c2].hi[lane] : 0;
            s_L[lane] = L;
            uint32_t inc = H - L;
            for (int d = 1; d < 8; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFu, inc, d);
                if (lane >= (uint32_t)d) inc += y;
            }
            s_off[lane + 1] = min(inc, CAP);
            if (lane == 0) s_off[0] = 0;
        }
    };
    // all threads: asynchronous copies of the packed windows into buffer 0
    auto issue_loads = [&]() {
        for (uint32_t b = 0; b < G; ++b) {
            const uint32_t e0 = s_off[b], e1 = s_off[b + 1];
            const int64_t sh = (int64_t)s_L[b] - (int64_t)e0;  // shard position of buffer slot e: e + sh
            const K* __restrict__ gk = S.k[b] + sh;
            const int32_t* __restrict__ gv = S.v[b] + sh;
            for (uint32_t e = e0 + tid; e < e1; e += XM_THREADS) {
                if (sizeof(K) == 4)
                    cp_async4(BK(0) + e, gk + e);
                else
                    cp_async8(BK(0) + e, gk + e);
                cp_async4(BV(0) + e, gv + e);
            }
        }
    };
    if (cbeg < cend) {
        if (tid < 32) pack(cbeg);
        __syncthreads();
        issue_loads();
    }
    // Software pipeline: the next unit's windows are loaded into buffer 0 as
    // soon as the first pass has consumed it, while the later passes and the
    // store of the current unit run on buffers 1 and 2.
    for (uint32_t c = cbeg; c < cend;) {
        const uint32_t c2 = s_next;
        cp_async_wait_all();
        __syncthreads();
        // ---- exact boundaries inside the loaded windows (threads 0..G-1: row c,
        //      threads 8..8+G-1: row c2)
        if (tid < 16 && (tid & 7) < G) {
            const uint32_t b = tid & 7;
            const XRow<K>& R = rows[tid < 8 ? c : c2];
            uint32_t E = R.lo[b];
            if (R.shard != INF32 && b != R.shard && R.hi[b] > R.lo[b]) {
                const K* w = BK(0) + s_off[b];  // w[q - L] = shard b element q
                const uint32_t L = s_L[b];
                uint32_t l = R.lo[b], h = R.hi[b];
                while (l < h) {
                    const uint32_t mid = (l + h) >> 1;
                    const bool pre = xs_precedes<K>(w[mid - L], b, R.key, R.shard);
                    l = pre ? mid + 1 : l;
                    h = pre ? h : mid;
                }
                E = l;
            }
            (tid < 8 ? s_E0 : s_E1)[b] = E;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t pos = 0;
            uint32_t acc = 0;
            for (uint32_t b = 0; b < G; ++b) {
                pos += s_E0[b];
                s_ro[b] = s_off[b] + (s_E0[b] - s_L[b]);  // run b inside buffer 0
                s_rl[b] = s_E1[b] - s_E0[b];
                acc += s_rl[b];
            }
            s_ro[G] = acc;
            s_out = pos - t0;
        }
        __syncthreads();
        // ---- pairwise merge passes: buffer 0 -> 1 -> 2 -> 1 ...
        uint32_t R = G, src = 0, dst = 1;
        const uint32_t U = s_ro[G];
        bool prefetched = false;
        while (R > 1) {
            const uint32_t Rn = (R + 1) / 2;
            // output pair q at compact offset sum(len of runs < 2q)
            for (uint32_t o = tid * VT, oe = min(o + VT, U); o < oe;) {
                uint32_t q = 0, base = 0;
                for (;; ++q) {
                    const uint32_t pl = s_rl[2 * q] + (2 * q + 1 < R ? s_rl[2 * q + 1] : 0);
                    if (o < base + pl || q + 1 == Rn) break;
                    base += pl;
                }
                const uint32_t la = s_rl[2 * q], lb = 2 * q + 1 < R ? s_rl[2 * q + 1] : 0;
                const uint32_t pe = min(oe, base + la + lb);
                if (pe <= o) {  // no pair holds o: the unit's descriptors are inconsistent
                    atomicOr(err, ERR_CUT);
                    break;
                }
                const uint32_t ra = s_ro[2 * q], rb = 2 * q + 1 < R ? s_ro[2 * q + 1] : ra;
                smem_merge_piece<K>(BK(src) + ra, BV(src) + ra, la, BK(src) + rb, BV(src) + rb, lb, o - base,
                                  pe - base, BK(dst) + base, BV(dst) + base);
                o = pe;
            }
            __syncthreads();
            if (tid == 0) {
                uint32_t base = 0;
                for (uint32_t q = 0; q < Rn; ++q) {
                    const uint32_t pl = s_rl[2 * q] + (2 * q + 1 < R ? s_rl[2 * q + 1] : 0);
                    s_ro[q] = base;
                    s_rl[q] = pl;
                    base += pl;
                }
            }
            if (!prefetched) {  // buffer 0 is consumed: pack and load the next unit
                prefetched = true;
                if (tid < 32 && c2 < cend) pack(c2);
                __syncthreads();
                if (c2 < cend) issue_loads();
            } else {
                __syncthreads();
            }
            R = Rn;
            src = dst;
            dst = dst == 1 ? 2 : 1;
        }
        if (!prefetched) {  // G == 1: the unit is stored straight from buffer 0
            const uint64_t ob = s_out;
            const uint32_t r0 = s_ro[0];
            for (uint32_t e = tid; e < U; e += XM_THREADS) {
                out_k[ob + e] = BK(0)[r0 + e];
                out_v[ob + e] = BV(0)[r0 + e];
            }
            __syncthreads();
            if (tid < 32 && c2 < cend) pack(c2);
            __syncthreads();
            if (c2 < cend) issue_loads();
        } else {
            // ---- store the unit (src holds the merged records, compact from s_ro[0])
            const uint64_t ob = s_out;
            const uint32_t r0 = s_ro[0];
            for (uint32_t e = tid; e < U; e += XM_THREADS) {
                out_k[ob + e] = BK(src)[r0 + e];
                out_v[ob + e] = BV(src)[r0 + e];
            }
        }
        c = c2;
    }
}

// samples[i] = keys[i * stride] of one shard
template <class K>
__global__ void __launch_bounds__(256) xs_samples_kernel(const K* __restrict__ keys, uint64_t n,
                                                         K* __restrict__ smp) {
    pdl_wait();
    const uint64_t ns = (n + xs_stride<K>() - 1) / xs_stride<K>();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x)
        smp[i] = keys[i * xs_stride<K>()];
}

}  // namespace ps

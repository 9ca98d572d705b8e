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

// consumer threads per merge_pipe_kernel CTA
#ifndef PS_CONSUMERS
#define PS_CONSUMERS 512
#endif
constexpr uint32_t PIPE_CONSUMERS = PS_CONSUMERS;

// Consumer thread t produces the VT outputs [VT*t, VT*t + VT) of every merge
// pass.  VT is odd (17 records of 8 bytes, 9 of 16 bytes): the k-th output of
// the lanes of a warp lands in distinct banks (2 or 4 wavefronts per warp
// store, the minimum), and the data-dependent read positions of balanced
// merges (~VT/2 * t) spread over all banks as well.  No padding is needed.
#ifndef PS_VT4
#define PS_VT4 17
#endif
#ifndef PS_VT8
#define PS_VT8 9
#endif
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_vt() {
    return sizeof(K) == 4 ? PS_VT4 : PS_VT8;
}
// records per unit (smem slot capacity)
template <class K>
PS_DEV __host__ constexpr uint32_t pipe_cap() {
    return pipe_vt<K>() * PIPE_CONSUMERS;
}
// Cut spacing budget: units hold <= CAP - VT records, so pass 1 can start Y
// at a VT-aligned offset (no thread straddles X and Y) within NC threads.
template <class K>
PS_DEV __host__ constexpr uint32_t cut_cap() {
    return pipe_cap<K>() - pipe_vt<K>();
}
// smallest cut spacing of any key type (bounds the chunk count)
constexpr uint32_t MIN_CUT_SPACING =
    (cut_cap<int32_t>() < cut_cap<int64_t>() ? cut_cap<int32_t>() : cut_cap<int64_t>()) / MAX_WAY;

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
    const uint32_t S = cut_cap<K>() / w;
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
#ifndef PS_SLOTS
#define PS_SLOTS 2
#endif
constexpr uint32_t PIPE_SLOTS = PS_SLOTS;  // input slots per CTA (TMA multi-buffering)
PS_DEV void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(PIPE_CONSUMERS) : "memory"); }

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
    const K* __restrict__ srcK = bufs.kb(nd.parity ^ 1);
    const int32_t* __restrict__ srcV = bufs.vb(nd.parity ^ 1);
    {
        // all loads issued before the shared-memory stores
        constexpr uint32_t PER = SMALL_NODE / 32;
        K kk[PER];
        int32_t vv[PER];
#pragma unroll
        for (uint32_t u = 0; u < PER; ++u) {
            const uint32_t i = lane + 32 * u;
            if (i < size) {
                kk[u] = srcK[(uint64_t)p0 + i];
                vv[u] = srcV[(uint64_t)p0 + i];
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < PER; ++u) {
            const uint32_t i = lane + 32 * u;
            if (i < size) {
                sk[i] = kk[u];
                sv[i] = vv[u];
            }
        }
    }
    if (lane < 5) s_off[warp][lane] = lane <= w ? nd.pos[lane] - p0 : size;
    __syncwarp();
    const uint32_t* off = s_off[warp];
    const uint32_t o1 = off[1], o2 = w > 2 ? off[2] : size, o3 = w > 3 ? off[3] : size;
#pragma unroll 4
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
    K* __restrict__ dstK = bufs.kb(nd.parity);
    int32_t* __restrict__ dstV = bufs.vb(nd.parity);
    for (uint32_t i = lane; i < size; i += 32) {
        dstK[(uint64_t)p0 + i] = ok[i];
        dstV[(uint64_t)p0 + i] = ov[i];
    }
}

// ---------------------------------------------------------------------------
// Optional clock64 phase counters of the pipe kernel (build with -DPS_PIPE_TIMING)
#ifdef PS_PIPE_TIMING
__device__ unsigned long long g_pipe_tim[40];
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
#define PT_START(on)
#define PT_MARK(idx)
#define PT_COUNT(idx)
#endif

// ---------------------------------------------------------------------------
// Big-node chunks: persistent, warp-specialized, TMA-bulk double-buffered.
constexpr uint32_t PIPE_THREADS = 32 + PIPE_CONSUMERS;

PS_DEV __host__ constexpr uint32_t align16c(uint32_t x) { return (x + 15u) & ~15u; }
PS_DEV __host__ constexpr uint32_t cmax(uint32_t a, uint32_t b) { return a > b ? a : b; }

// (key, value) record in shared memory: 8 bytes for 4-byte keys, 16 for 8-byte
template <class K>
struct alignas(sizeof(K) == 4 ? 8 : 16) Rec {
    K k;
    int32_t v;
};


template <class K>
struct PipeLayout {
    static constexpr uint32_t CAP = pipe_cap<K>();
    static constexpr uint32_t PADN = CAP + pipe_vt<K>() + 16;  // record capacity (+ over-read / don't-care slack)
    static_assert(PADN >= CAP + pipe_vt<K>() - 1, "record slack must hold a thread's don't-care outputs");
    static constexpr uint32_t RECB = (uint32_t)sizeof(Rec<K>);
    // slot = TMA landing zone of the k key windows + k value windows (SoA, 16B
    // alignment slack each), and afterwards the padded records of the last pass
    static constexpr uint32_t KEY_BYTES = align16c(CAP * (uint32_t)sizeof(K)) + MAX_WAY * 32u;
    static constexpr uint32_t VAL_BYTES = align16c(CAP * 4u) + MAX_WAY * 32u;
    static constexpr uint32_t SLOT = align16c(cmax(KEY_BYTES + VAL_BYTES, PADN * RECB));
    // scratch: first-pass records X || Y (or the 2-way output)
    static constexpr uint32_t SCRATCH = align16c(PADN * RECB);
};

struct PipeDesc {
    uint64_t out;  // global element index of the unit's first output
    uint32_t koff[4], voff[4], len[4];
    uint32_t T, w, par, done;
};

template <class K>
size_t merge_pipe_smem_bytes() {
    return PIPE_SLOTS * (size_t)PipeLayout<K>::SLOT + PipeLayout<K>::SCRATCH + PIPE_SLOTS * sizeof(PipeDesc) + 64;
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
template <class C, class K>
PS_DEV void single_merge(C& c, Rec<K>* out) {
    if (c.o >= c.oe) return;
    uint32_t lo = c.o > c.lb ? c.o - c.lb : 0, hi = c.o < c.la ? c.o : c.la;
    while (lo < hi) {
        const uint32_t m = (lo + hi) >> 1;
        const bool le = !(c.keyB(c.o - 1 - m) < c.keyA(m));
        lo = le ? m + 1 : lo;
        hi = le ? hi : m;
    }
    c.i = lo;
    c.j = c.o - lo;
    c.heads();
    Rec<K>* outp = out + c.base + c.o;
#pragma unroll
    for (uint32_t t = 0; t < pipe_vt<K>(); ++t) c.step(outp, t);
}

// A TMA-landed input window: SoA keys / values, unpadded.
template <class K>
struct Win {
    const K* k;
    const int32_t* v;
    uint32_t len;
};

template <class K>
__global__ void __launch_bounds__(PIPE_THREADS) merge_pipe_kernel(Bufs<K> bufs, const Node* __restrict__ nodes,
                                                                  const uint32_t* __restrict__ chunk2node,
                                                                  const uint4* __restrict__ cuts, uint32_t c0,
                                                                  uint32_t nchunks, uint32_t* err) {
    using LY = PipeLayout<K>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* scratch = smem + PIPE_SLOTS * LY::SLOT;
    PipeDesc* desc = reinterpret_cast<PipeDesc*>(scratch + LY::SCRATCH);
    uint64_t* bars = reinterpret_cast<uint64_t*>(desc + PIPE_SLOTS);
    uint64_t* full = bars;                // [PIPE_SLOTS]
    uint64_t* empty = bars + PIPE_SLOTS;  // [PIPE_SLOTS]
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (uint32_t sl = 0; sl < PIPE_SLOTS; ++sl) {
            mbar_init(&full[sl], 1);
            mbar_init(&empty[sl], PIPE_CONSUMERS / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (tid < 32) {
        // ------------------------------ producer ------------------------------
        const uint32_t lane = tid;
        const uint32_t cbeg = c0 + (uint32_t)(((uint64_t)nchunks * blockIdx.x) / gridDim.x);
        const uint32_t cend = c0 + (uint32_t)(((uint64_t)nchunks * (blockIdx.x + 1)) / gridDim.x);
        uint32_t unit = 0;
        PT_START(lane == 0)
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
            PT_MARK(0)
            uint32_t u = 0;
            while (u < nvalid) {
                // unit = lanes u..V of the same node with total <= cut_cap
                const uint32_t nid_u = __shfl_sync(PS_FULL, nid, u);
                const uint32_t sx = __shfl_sync(PS_FULL, st.x, u), sy = __shfl_sync(PS_FULL, st.y, u);
                const uint32_t sz = __shfl_sync(PS_FULL, st.z, u), sw = __shfl_sync(PS_FULL, st.w, u);
                const uint32_t tot = (en.x - sx) + (en.y - sy) + (en.z - sz) + (en.w - sw);
                const bool ok = lane >= u && lane < nvalid && nid == nid_u && tot <= cut_cap<K>();
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
                const uint32_t slot = unit % PIPE_SLOTS;
                if (unit >= PIPE_SLOTS) mbar_wait(&empty[slot], ((unit / PIPE_SLOTS) - 1) & 1);
                PT_MARK(1)
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
                    const uint8_t* src = is_val ? reinterpret_cast<const uint8_t*>(bufs.vb(par ^ 1))
                                                : reinterpret_cast<const uint8_t*>(bufs.kb(par ^ 1));
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
                    if (total > cut_cap<K>()) atomicOr(err, ERR_CUT);
                    mbar_arrive_tx(&full[slot], txs);
                }
                PT_MARK(2)
                PT_COUNT(3)
                unit++;
                u = V + 1;
            }
            c += nvalid;
        }
        // termination marker
        const uint32_t slot = unit % PIPE_SLOTS;
        if (unit >= PIPE_SLOTS) mbar_wait(&empty[slot], ((unit / PIPE_SLOTS) - 1) & 1);
        if (lane == 0) {
            desc[slot].done = 1;
            mbar_arrive(&full[slot]);
        }
        return;
    }

    // ------------------------------ consumers ---------------------------------
    const uint32_t ctid = tid - 32;
    const uint32_t clane = ctid & 31;
    Rec<K>* const xr = reinterpret_cast<Rec<K>*>(scratch);
    PT_START(ctid == 0)
    for (uint32_t i = 0;; ++i) {
        const uint32_t slot = i % PIPE_SLOTS;
        mbar_wait(&full[slot], (i / PIPE_SLOTS) & 1);
        PT_MARK(4)
        PT_USTART
        const PipeDesc& d = desc[slot];
        if (d.done) break;
        const uint32_t T = d.T, w = d.w, par = d.par;
        const uint64_t out = d.out;
        uint8_t* sbase = smem + slot * LY::SLOT;
        Win<K> win[4];
#pragma unroll
        for (uint32_t a = 0; a < 4; ++a) {
            win[a].k = reinterpret_cast<const K*>(sbase + d.koff[a]);
            win[a].v = reinterpret_cast<const int32_t*>(sbase + d.voff[a]);
            win[a].len = a < w ? d.len[a] : 0;
        }
        auto wincur = [&](uint32_t a, uint32_t b, uint32_t base, uint32_t o0, uint32_t o1) {
            WinCur<K> c;
            c.ak = win[a].k;
            c.bk = win[b].k;
            c.av = win[a].v;
            c.bv = win[b].v;
            c.la = win[a].len;
            c.lb = win[b].len;
            c.o = o0;
            c.oe = o1;
            c.base = base;
            return c;
        };
        Rec<K>* orec;
        constexpr uint32_t NC = PIPE_CONSUMERS;
        // final records are placed with the global 16-byte phase of the
        // destination so the store phase moves aligned 16-byte vectors
        constexpr uint32_t ER = sizeof(K) == 4 ? 4 : 2;  // records per store group
        const uint32_t al = (uint32_t)(out % ER);
        constexpr uint32_t VT = pipe_vt<K>();
        const uint32_t o0 = min(T, VT * ctid), o1 = min(T, VT * ctid + VT);
        if (w >= 3) {
            // pass 1: X = merge(A, B) -> xr[0, LX);  Y = merge(C, D) (3-way: C) -> xr[LXp, LXp + LY)
            // with LXp = LX rounded up to VT: thread t takes outputs [VT*t, VT*t + VT)
            // of that layout, so every warp runs one merge (no X/Y divergence)
            const uint32_t LX = win[0].len + win[1].len, LYn = T - LX;
            const uint32_t LXp = (LX + VT - 1) / VT * VT;
            const uint32_t ob = VT * ctid;
            const bool isY = ob >= LXp;
            WinCur<K> c;
            c.ak = isY ? win[2].k : win[0].k;
            c.bk = isY ? win[3].k : win[1].k;
            c.av = isY ? win[2].v : win[0].v;
            c.bv = isY ? win[3].v : win[1].v;
            c.la = isY ? win[2].len : win[0].len;
            c.lb = isY ? win[3].len : win[1].len;
            c.o = isY ? ob - LXp : ob;
            c.oe = isY ? min(ob + VT - LXp, LYn) : min(ob + VT, LX);
            c.base = isY ? LXp : 0;
            single_merge(c, xr);
            PT_WARP(16)
            consumer_sync();
            PT_MARK(5)
            // pass 2: merge X and Y into the slot (its input windows are consumed)
            orec = reinterpret_cast<Rec<K>*>(sbase);
            RecCur<K> p0;
            p0.r = xr;
            p0.offa = 0;
            p0.offb = LXp;
            p0.la = LX;
            p0.lb = LYn;
            p0.base = al;
            p0.o = o0;
            p0.oe = o1;
            single_merge(p0, orec);
        } else {
            // 2-way: merge(A, B) straight into scratch
            orec = xr;
            WinCur<K> c0 = wincur(0, 1, al, o0, o1);
            single_merge(c0, orec);
        }
        PT_WARP(24)
        // store: every warp moves its own outputs [VT*32*w, VT*32*(w+1)) as soon as
        // they are written (no CTA barrier): full ER-groups of the phase-shifted
        // layout as 16-byte vectors, the partial groups at both ends record by record
        __syncwarp();
        PT_MARK(6)
        K* __restrict__ dstK = bufs.kb(par);
        int32_t* __restrict__ dstV = bufs.vb(par);
        {
            const uint32_t wid = ctid >> 5;
            const uint32_t rs = al + min(T, VT * 32 * wid), re = al + min(T, VT * 32 * (wid + 1));
            const uint64_t gbase = out - al;  // global element of record index 0
            if (rs < re) {
                const uint32_t g0 = (rs + ER - 1) / ER, g1 = re / ER;
                for (uint32_t j = g0 + clane; j < g1; j += 32) {
                    const uint32_t r0 = j * ER;
                    const uint4* src = reinterpret_cast<const uint4*>(orec + r0);
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
                    const Rec<K> rec = orec[rr];
                    dstK[gbase + rr] = rec.k;
                    dstV[gbase + rr] = rec.v;
                }
            }
        }
        __syncwarp();
        if (clane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
        // scratch xr is rewritten by the next unit's first pass
        consumer_sync();
        PT_MARK(7)
        PT_COUNT(8)
    }
}

}  // namespace ps

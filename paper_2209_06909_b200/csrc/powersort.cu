// powersort.cu -- host orchestration + C ABI (include/powersort_b200.h).
//
// ps_sort = stable_sort_with (policy.py:201-262) as a stream of kernels:
//   N1 pass 1  rd_types -> suffix-min(F) -> rd_tables -> chain scan -> rd_emit
//   N2         powers -> min tree -> nearest<= -> classify (x2) -> spine
//              -> depth / stack scans -> node finalize -> chunk plan
//   N1 pass 2  form_leaves (into buffer depth&1)
//   N3/N4      per stage (power levels high..low, then merge_down nodes):
//              partition (big nodes) + merge_chunks
// Two host synchronisations read the run count and the tree summary.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/powersort_b200.h"
#include "ps_common.cuh"
#include "ps_form.cuh"
#include "ps_merge.cuh"
#include "ps_runs.cuh"
#include "ps_scan.cuh"
#include "ps_shard.cuh"
#include "ps_tree.cuh"

using namespace ps;

namespace {

thread_local std::string g_last_error;
thread_local bool g_prof_on = false;
thread_local std::vector<ps_prof_entry> g_prof_last;

// CUDA-event phase timer (only active when ps_profile_enable(1) was called).
struct Prof {
    struct Rec {
        ps_prof_entry e;
        cudaEvent_t a, b;
    };
    bool on;
    cudaStream_t s;
    std::vector<Rec> recs;
    explicit Prof(cudaStream_t st) : on(g_prof_on), s(st) {}
    ~Prof() {
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
    int begin(int kind, int stage, int64_t nodes, int64_t chunks, int64_t bytes) {
        if (!on) return -1;
        Rec r;
        memset(&r.e, 0, sizeof(r.e));
        r.e.kind = kind;
        r.e.stage = stage;
        r.e.nodes = nodes;
        r.e.chunks = chunks;
        r.e.bytes = bytes;
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, s);
        recs.push_back(r);
        return (int)recs.size() - 1;
    }
    void end(int i) {
        if (i >= 0) cudaEventRecord(recs[i].b, s);
    }
    void finish() {
        if (!on) return;
        cudaStreamSynchronize(s);
        g_prof_last.clear();
        for (auto& r : recs) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.a, r.b);
            r.e.ms = ms;
            g_prof_last.push_back(r.e);
        }
    }
};


int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define PS_CUDA(call)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(PS_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                                      __FILE__ + ":" + std::to_string(__LINE__));                  \
    } while (0)

// after every kernel launch: count it and surface launch errors
#define PS_LAUNCH_CHECK()            \
    do {                             \
        launch_counter()++;          \
        PS_CUDA(cudaGetLastError()); \
    } while (0)

constexpr uint32_t NBARS = NPOW + MAX_SPINE + 8;  // fused-partition stages per sort
constexpr uint64_t WS_MAGIC = 0x5053423230304b31ull;  // "PSB200K1"

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Workspace header (device memory at offset 0; copied to host by ps_result_*).
struct WsHeader {
    uint64_t magic;
    int64_t n;
    int64_t m;
    int32_t k, dtype;
    uint32_t r;
    uint32_t nmain, nspine_nodes;
    uint32_t counters_pending;  // comparisons / moves of an asynchronous sort still on the device
    uint64_t off_sum, off_b, off_nat, off_nodes;
    int64_t moves_base;         // tree-determined part of `moves` (pending counters)
    int32_t counters_exact, pad2;
};

// Small device->host reads go through a host-mapped pinned buffer written by a
// kernel: a cudaMemcpyAsync would queue behind bulk transfers of other streams
// on the copy engines (the pipelined end-to-end path), a kernel store does not.
struct HostMap {
    uint8_t* h = nullptr;
    uint8_t* d = nullptr;
    size_t size = 0;
    uint32_t seq = 0;   // last publish sequence number
};
thread_local HostMap g_map;

// Copies the 32-bit words of a || b (each zero-padded to 16 bytes) to mapped
// host memory, three per 16-byte store with the sequence number as the fourth,
// then one more record with two checksums of all the words.  The host waits
// until every record carries seq and the checksums match: a 16-byte store that
// reached the host torn (tag before data) is caught and re-read.  (No
// system-scope fence: it would wait behind the bulk host copies other streams
// keep on the link.)
__host__ __device__ inline void publish_mix(uint32_t w, uint32_t i, uint32_t& s1, uint32_t& s2) {
    s1 += w * (2u * i + 1u);
    s2 ^= (w << (i & 15u)) | (w >> ((32u - (i & 15u)) & 31u));
}
__global__ void publish_kernel(const uint32_t* __restrict__ a, uint32_t na, const uint32_t* __restrict__ b,
                               uint32_t nb, uint4* __restrict__ dst, uint32_t seq) {
    pdl_wait();
    const uint32_t nw = na + nb, ns = (nw + 2) / 3;
    uint32_t s1 = 0, s2 = 0;
    for (uint32_t q = threadIdx.x; q < ns; q += blockDim.x) {
        uint32_t v[3];
#pragma unroll
        for (uint32_t t = 0; t < 3; ++t) {
            const uint32_t w = 3 * q + t;
            v[t] = w < na ? a[w] : (w < nw ? b[w - na] : 0u);
            publish_mix(v[t], w, s1, s2);
        }
        dst[q] = make_uint4(v[0], v[1], v[2], seq);
    }
    __shared__ uint32_t r1[32], r2[32];
    for (int d = 16; d; d >>= 1) {
        s1 += __shfl_xor_sync(PS_FULL, s1, d);
        s2 ^= __shfl_xor_sync(PS_FULL, s2, d);
    }
    if ((threadIdx.x & 31) == 0) {
        r1[threadIdx.x >> 5] = s1;
        r2[threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t1 = 0, t2 = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
            t1 += r1[w];
            t2 ^= r2[w];
        }
        dst[ns] = make_uint4(t1, t2, ns, seq);
    }
}

__global__ void write_header_kernel(WsHeader h, WsHeader* dst) {
    pdl_wait();
    if (threadIdx.x == 0) *dst = h;
}

int host_map_ensure(size_t bytes) {
    if (g_map.size >= bytes) return PS_OK;
    if (g_map.h) cudaFreeHost(g_map.h);
    const uint32_t seq = g_map.seq;
    g_map = HostMap();
    g_map.seq = seq;
    void* h = nullptr;
    PS_CUDA(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    void* d = nullptr;
    PS_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    memset(h, 0, bytes);
    g_map.h = (uint8_t*)h;
    g_map.d = (uint8_t*)d;
    g_map.size = bytes;
    return PS_OK;
}

// Device ranges a (and b) to host memory, in two halves so that the host can
// enqueue more work before it waits: publish_begin enqueues the copy;
// publish_wait spins until every store carries the sequence number (no stream
// synchronization: later work may already be queued behind the copy) and
// unpacks the bytes.  Sources are 16-byte aligned workspace regions.
struct Pending {
    uint32_t seq = 0;
    const void* a_src = nullptr;  // device sources (the fallback copy)
    const void* b_src = nullptr;
    size_t abytes = 0, bbytes = 0;
    void* a_out = nullptr;
    void* b_out = nullptr;
};
int publish_begin(const void* a, size_t abytes, void* a_out, const void* b, size_t bbytes, void* b_out,
                  cudaStream_t s, Pending& pend) {
    const size_t na = (abytes + 15) / 16 * 4, nb = (bbytes + 15) / 16 * 4;
    const size_t ns = (na + nb + 2) / 3;
    int rc = host_map_ensure((ns + 1) * 16);
    if (rc) return rc;
    const uint32_t seq = ++g_map.seq;
    PS_CUDA(launch_k(publish_kernel, 1, 256, 0, s, (const uint32_t*)a, (uint32_t)na, (const uint32_t*)b,
                     (uint32_t)nb, (uint4*)g_map.d, seq));
    pend.seq = seq;
    pend.a_src = a;
    pend.b_src = b;
    pend.abytes = abytes;
    pend.bbytes = bbytes;
    pend.a_out = a_out;
    pend.b_out = b_out;
    return PS_OK;
}
int publish_wait(const Pending& pend, cudaStream_t s) {
    const size_t na = (pend.abytes + 15) / 16 * 4, nb = (pend.bbytes + 15) / 16 * 4;
    const size_t ns = (na + nb + 2) / 3;
    const volatile uint32_t* hw = reinterpret_cast<const volatile uint32_t*>(g_map.h);
    auto arrived = [&]() {
        for (size_t q = ns + 1; q-- > 0;)  // the last stores are the likeliest to be missing
            if (hw[4 * q + 3] != pend.seq) return false;
        return true;
    };
    std::vector<uint32_t> tmp(na + nb);
    auto consistent = [&]() {  // every word read once, against the checksum record
        std::atomic_thread_fence(std::memory_order_acquire);
        uint32_t s1 = 0, s2 = 0;
        for (size_t w = 0; w < ns * 3; ++w) {
            const uint32_t v = hw[4 * (w / 3) + (w % 3)];
            if (w < na + nb) tmp[w] = v;
            publish_mix(v, (uint32_t)w, s1, s2);
        }
        return s1 == hw[4 * ns] && s2 == hw[4 * ns + 1];
    };
    bool ok = false;
    for (uint32_t spins = 1;; ++spins) {
        if (arrived() && consistent()) {
            ok = true;
            break;
        }
        if ((spins & 255u) == 0) {  // a failed stream never delivers
            const cudaError_t e = cudaStreamQuery(s);
            if (e != cudaSuccess && e != cudaErrorNotReady) PS_CUDA(e);
            if (e == cudaSuccess && !(arrived() && consistent())) break;  // done, but not (yet) coherent here
        }
    }
    if (!ok) {
        // the stream has finished: read the device sources directly
        PS_CUDA(cudaStreamSynchronize(s));
        PS_CUDA(cudaMemcpy(tmp.data(), pend.a_src, na * 4, cudaMemcpyDeviceToHost));
        if (nb) PS_CUDA(cudaMemcpy(tmp.data() + na, pend.b_src, nb * 4, cudaMemcpyDeviceToHost));
    }
    memcpy(pend.a_out, tmp.data(), pend.abytes);
    if (pend.bbytes) memcpy(pend.b_out, tmp.data() + na, pend.bbytes);
    return PS_OK;
}
int publish(const void* a, size_t abytes, void* a_out, const void* b, size_t bbytes, void* b_out, cudaStream_t s) {
    Pending pend;
    int rc = publish_begin(a, abytes, a_out, b, bbytes, b_out, s, pend);
    if (rc) return rc;
    return publish_wait(pend, s);
}

// leading Summary fields the host needs at each synchronization point
constexpr size_t SUM_HEAD = offsetof(Summary, level_off);    // r, err, node counts, max_stack
constexpr size_t SUM_STATS = offsetof(Summary, level_cost);  // + level offsets and the counters

struct Layout {
    uint64_t n, m, kb, rmax, ngroups, ntiles, chunks_max, scan_tmp;
    uint32_t nlev;
    uint64_t lev_size[8];
    uint64_t tab_levels;  // number of chain-scan levels
    uint64_t lvlP[16];
    // offsets
    uint64_t header, sum, k1, v1, ty, cg, Fg, Ft, tile_tab, lvl_tab[16], lvl_ent[16], b, nat, leafpar, P,
        minlev[8], Rle, Lle, Dd, Sd, hist, hist_off, hist_tot, spine, nodes, nch, chunk_base, stage_chunk, chunk2node, cuts, bars, tile_first,
        pdelta,
        scantmp_u32, scantmp_i32, total;
};

Layout make_layout(uint64_t n, uint64_t kb, uint64_t m, bool sort_buffers, uint64_t rmax_override = 0) {
    Layout L;
    memset(&L, 0, sizeof(L));
    L.n = n;
    L.m = m;
    L.kb = kb;
    uint64_t rmax = rmax_override ? rmax_override : std::min<uint64_t>(n, cdiv(n, std::max<uint64_t>(m, 1)));
    L.rmax = rmax + 2;
    L.ngroups = std::max<uint64_t>(1, cdiv(n, GROUP));
    L.ntiles = L.ngroups * TILES_PER_GROUP;
    // total chunks <= nodes + merge_cost / (cut spacing); merge_cost <= 64 n
    L.chunks_max = L.rmax + cdiv(64 * n, MIN_CUT_SPACING) + 16;
    // min tree levels over P (size rmax + 1)
    uint64_t s = align_up(L.rmax + 1, 32);
    L.nlev = 0;
    for (;;) {
        L.lev_size[L.nlev++] = s;
        if (s <= 32 || L.nlev == 8) break;
        s = align_up(cdiv(s, 32), 32);
    }
    // chain-scan levels
    uint64_t P = L.ngroups;
    L.tab_levels = 0;
    for (;;) {
        L.lvlP[L.tab_levels++] = P;
        if (P <= TSCAN_FAN) break;
        P = cdiv(P, TSCAN_FAN);
    }
    uint64_t big = std::max<uint64_t>({L.rmax + MAX_SPINE + 2, L.ngroups + 2, (uint64_t)NPOW * cdiv(L.rmax, CLS_THREADS) + 2,
                                       (uint64_t)NSTAGE * cdiv(L.rmax + MAX_SPINE, FIN_THREADS) + 2, L.rmax});
    L.scan_tmp = scan_tmp_elems(big);

    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t o = off;
        off = align_up(off + std::max<uint64_t>(bytes, 1), 256);
        return o;
    };
    const uint64_t M1 = std::min<uint64_t>(m, MAX_M_TILED) + 1;
    L.header = take(sizeof(WsHeader));
    L.sum = take(sizeof(Summary));
    if (sort_buffers) {
        L.k1 = take(n * kb);
        L.v1 = take(n * 4);
        L.ty = take((L.ngroups * GROUP_WORDS + 64) * 4);
        L.cg = take((L.ngroups + 1) * 4);
        L.Fg = take((L.ngroups + 1) * 4);
        L.Ft = take((L.ntiles + 1) * 4);
        L.tile_first = take((L.ntiles + 1) * 4);
        if (m <= MAX_M_TILED) {
            L.tile_tab = take(L.ntiles * M1 * 8);
            for (uint64_t l = 0; l < L.tab_levels; ++l) {
                L.lvl_tab[l] = take(L.lvlP[l] * M1 * 8);
                L.lvl_ent[l] = take((L.lvlP[l] + 1) * 8);
            }
        }
        L.nat = take(L.rmax * 4);
        L.leafpar = take(L.rmax);
        L.cuts = take(L.chunks_max * 16);
        L.bars = take(NBARS * 4);
    }
    L.b = take((L.rmax + 2) * 4);
    for (uint32_t l = 0; l < L.nlev; ++l) L.minlev[l] = take(L.lev_size[l] + 32);
    L.P = L.minlev[0];
    L.Rle = take(L.rmax * 4);
    L.Lle = take(L.rmax * 4);
    L.Dd = take((L.rmax + 2) * 4);
    L.Sd = take((L.rmax + 2) * 4);
    L.hist = take(((uint64_t)NPOW * cdiv(L.rmax, CLS_THREADS) + 2) * 4);
    L.hist_off = take(((uint64_t)NPOW * cdiv(L.rmax, CLS_THREADS) + 2) * 4);
    L.hist_tot = take(16);
    L.spine = take(MAX_SPINE * 4);
    L.nodes = take((L.rmax + MAX_SPINE) * sizeof(Node));
    L.pdelta = take(NPOW * 4);
    L.nch = take((L.rmax + MAX_SPINE + 2) * 4);
    L.chunk_base = take((L.rmax + MAX_SPINE + 2) * 4);
    L.stage_chunk = take((NSTAGE + 2) * 4);
    L.chunk2node = take(L.chunks_max * 4);
    L.scantmp_u32 = take(L.scan_tmp * 4);
    L.scantmp_i32 = take(L.scan_tmp * 4);
    L.total = off;
    return L;
}

// Host copy of the summary plus the per-stage chunk ranges.
struct TreeInfo {
    Summary s;
    // chunk_base at the stage offsets [0..NSTAGE], total [NSTAGE+1]
    uint32_t stage_chunk[NSTAGE + 2];
    uint32_t level_chunk(uint32_t h) const { return stage_chunk[h]; }
    uint32_t total_chunks() const { return stage_chunk[NSTAGE + 1]; }
};

template <class T>
T* at(uint8_t* ws, uint64_t off) {
    return reinterpret_cast<T*>(ws + off);
}

inline unsigned grid_for(uint64_t n, unsigned t) { return (unsigned)std::max<uint64_t>(1, cdiv(n, t)); }

// End of the tree phase: the chunk -> node map (its size is read on the
// device), then one publish of the summary and the stage chunk offsets (the
// host schedules the merges from them).  The publish is only enqueued here;
// tree_wait() collects it, so the caller can queue leaf formation first.
int finish_tree(uint8_t* ws, const Layout& L, TreeInfo& info, cudaStream_t s, Pending& pend, bool chunk_map = true) {
    Summary* sum = at<Summary>(ws, L.sum);
    if (chunk_map) {  // (the multi-kernel path builds it in tree_chunks_kernel)
        launch_k(tree_chunk_map_kernel, CHUNK_MAP_CTAS, 256, 0, s, (const Node*)at<Node>(ws, L.nodes),
                 (const Summary*)sum, (const uint32_t*)at<uint32_t>(ws, L.stage_chunk),
                 (uint32_t)std::min<uint64_t>(L.chunks_max, 0xFFFFFFFFull), at<uint32_t>(ws, L.chunk2node));
        PS_LAUNCH_CHECK();
    }
    return publish_begin(sum, sizeof(Summary), &info.s, at<uint32_t>(ws, L.stage_chunk), sizeof(info.stage_chunk),
                         info.stage_chunk, s, pend);
}

int tree_wait(const Layout& L, TreeInfo& info, cudaStream_t s, const Pending& pend) {
    int rc = publish_wait(pend, s);
    if (rc) return rc;
    if (info.total_chunks() > L.chunks_max) return fail(PS_ENOMEM, "merge chunk table exceeds workspace bound");
    if (info.s.err & ERR_STACK) return fail(PS_EOVERFLOW, "run stack exceeded its height bound");
    if (info.s.err) return fail(PS_EINVARIANT, "device invariant violated (flags " + std::to_string(info.s.err) + ")");
    return PS_OK;
}

// Builds the merge tree of the run boundaries b[0..r] (device, already in
// place) for an array of n elements.  Leaves leaf parities when leafpar != 0.
int build_tree(uint8_t* ws, const Layout& L, uint32_t r, uint64_t n, int k, int strict, int slack_mode,
               uint8_t* leafpar, TreeInfo& info, cudaStream_t s, Pending& pend, uint32_t cap = CHUNK_CAP) {
    Summary* sum = at<Summary>(ws, L.sum);
    uint32_t* err = &sum->err;
    const uint32_t* b = at<uint32_t>(ws, L.b);
    uint8_t* P = at<uint8_t>(ws, L.P);
    const uint32_t log2k = k == 4 ? 2 : 1;
    // P over [0, padded): r + 1 boundaries and 0xFF up to the next multiple of 32
    const uint32_t padded = (uint32_t)align_up((uint64_t)r + 1, 32);
    static const bool no_small_tree = knob_set("PS_NO_SMALL_TREE");  // A/B: multi-kernel path
    // A/B: PS_TREE_SMALL_R=x moves the one-CTA / multi-kernel crossover
    static const uint32_t small_r = (uint32_t)knob("PS_TREE_SMALL_R", TREE_SMALL_R);
    if (r <= small_r && !no_small_tree) {
        // the whole build in one CTA (tree_small_kernel), then one publish
        TreeSmallArgs a;
        memset(&a, 0, sizeof(a));
        a.b = b;
        a.r = r;
        a.n = n;
        a.log2k = log2k;
        a.k = (uint32_t)k;
        a.strict = strict;
        a.slack_mode = slack_mode;
        a.cap = cap;
        a.stack_cap = (uint32_t)ps_run_stack_capacity(k, (int64_t)n);
        a.P = P;
        a.padded = padded;
        a.mt.lev[0] = P;
        uint32_t nlev = 1;
        uint64_t size = align_up((uint64_t)r + 1, 32);
        while (size > 32 && nlev < L.nlev) {
            const uint64_t groups = size / 32;
            const uint64_t outp = align_up(groups, 32);
            a.mt.lev[nlev] = at<uint8_t>(ws, L.minlev[nlev]);
            a.lev_groups[nlev] = (uint32_t)groups;
            a.lev_padded[nlev] = (uint32_t)outp;
            nlev++;
            size = outp;
        }
        a.mt.nlev = nlev;
        a.Rle = at<uint32_t>(ws, L.Rle);
        a.Lle = at<uint32_t>(ws, L.Lle);
        a.Dd = at<int32_t>(ws, L.Dd);
        a.Sd = at<int32_t>(ws, L.Sd);
        a.nblocks = (uint32_t)std::max<uint64_t>(1, cdiv(r > 1 ? r - 1 : 1, CLS_THREADS));
        a.hist = at<uint32_t>(ws, L.hist);
        a.hoff = at<uint32_t>(ws, L.hist_off);
        a.htot = at<uint32_t>(ws, L.hist_tot);
        a.spine = at<uint32_t>(ws, L.spine);
        a.nodes = at<Node>(ws, L.nodes);
        a.pdelta = at<int32_t>(ws, L.pdelta);
        a.leafpar = leafpar;
        a.nmax = r + MAX_SPINE;
        a.nch = at<uint32_t>(ws, L.nch);
        a.cb = at<uint32_t>(ws, L.chunk_base);
        a.stage_chunk = at<uint32_t>(ws, L.stage_chunk);
        a.sum = sum;
        PS_CUDA(launch_k(tree_small_kernel, 1, CLS_THREADS, 0, s, a));
        launch_counter()++;
        return finish_tree(ws, L, info, s, pend);
    }
    // T1 powers (array over 0..padded) with min-tree level 1, T2 the other levels
    int32_t* Dd = at<int32_t>(ws, L.Dd);
    int32_t* Sd = at<int32_t>(ws, L.Sd);
    MinTree mt;
    memset(&mt, 0, sizeof(mt));
    mt.lev[0] = P;
    uint32_t nlev = 1;
    uint32_t lev_groups[8] = {0}, lev_padded[8] = {0};
    {
        uint64_t size = align_up((uint64_t)r + 1, 32);
        while (size > 32 && nlev < L.nlev) {
            const uint64_t groups = size / 32;
            const uint64_t outp = align_up(groups, 32);
            lev_groups[nlev] = (uint32_t)groups;
            lev_padded[nlev] = (uint32_t)outp;
            mt.lev[nlev] = at<uint8_t>(ws, L.minlev[nlev]);
            nlev++;
            size = outp;
        }
    }
    mt.nlev = nlev;
    {
        uint8_t* lev1 = nlev > 1 ? const_cast<uint8_t*>(mt.lev[1]) : nullptr;
        const uint64_t nthr = std::max<uint64_t>({padded, (uint64_t)lev_padded[1] * 32, (uint64_t)r + 2});
        launch_k(tree_powers_kernel, grid_for(nthr, 256), 256, 0, s, b, r, n, log2k, P, padded, err, Dd, Sd, lev1,
                 lev_padded[1]);
        PS_LAUNCH_CHECK();
    }
    for (uint32_t l = 2; l < nlev; ++l) {
        launch_k(tree_minlevel_kernel, grid_for(lev_padded[l], 256), 256, 0, s, mt.lev[l - 1], lev_groups[l],
                 const_cast<uint8_t*>(mt.lev[l]), lev_padded[l]);
        PS_LAUNCH_CHECK();
    }
    uint32_t* Rle = at<uint32_t>(ws, L.Rle);
    uint32_t* Lle = at<uint32_t>(ws, L.Lle);
    launch_k(tree_nearest_kernel, grid_for(r, 256), 256, 0, s, mt, P, r, Rle, Lle);
    PS_LAUNCH_CHECK();
    // T3 classify
    const uint32_t nblocks = (uint32_t)std::max<uint64_t>(1, cdiv(r > 1 ? r - 1 : 1, CLS_THREADS));
    uint32_t* hist = at<uint32_t>(ws, L.hist);
    uint32_t* hoff = at<uint32_t>(ws, L.hist_off);
    uint32_t* htot = at<uint32_t>(ws, L.hist_tot);
    uint32_t* spine = at<uint32_t>(ws, L.spine);
    Node* nodes = at<Node>(ws, L.nodes);  // written at their merge-stage slots (tree_spine_cta)
    int32_t* pdelta = at<int32_t>(ws, L.pdelta);
    launch_k(tree_classify_kernel<0>, nblocks, CLS_THREADS, 0, s, P, Rle, Lle, b, r, k, nblocks, hist, nullptr, Dd, Sd,
                                                            spine, nodes, sum, (const int32_t*)pdelta);
    PS_LAUNCH_CHECK();
    PS_CUDA((device_scan<uint32_t, OpSum<uint32_t>>(hist, hoff, (int64_t)NPOW * nblocks, false, true,
                                                   at<uint32_t>(ws, L.scantmp_u32), htot, s)));
    launch_k(tree_spine_kernel, 1, 256, 0, s, b, r, k, strict, spine, nodes, Dd, sum, mt, (const uint32_t*)hoff,
             (const uint32_t*)htot, nblocks, pdelta);
    PS_LAUNCH_CHECK();
    launch_k(tree_classify_kernel<1>, nblocks, CLS_THREADS, 0, s, P, Rle, Lle, b, r, k, nblocks, nullptr, hoff, Dd, Sd,
                                                            spine, nodes, sum, (const int32_t*)pdelta);
    PS_LAUNCH_CHECK();
    // depth (inclusive prefix of Dd) and stack height (inclusive prefix of Sd)
    PS_CUDA((device_scan2<int32_t, OpSum<int32_t>>(Dd, Dd, Sd, Sd, (int64_t)r + 1, false, false,
                                                  at<int32_t>(ws, L.scantmp_i32), s)));
    // node-indexed kernels run over the bound nmax and read the node count on the device
    const uint32_t nmax = r + MAX_SPINE;
    const int64_t stack_cap = (int64_t)ps_run_stack_capacity(k, (int64_t)n);
    uint32_t* nch = at<uint32_t>(ws, L.nch);
    uint32_t* cb = at<uint32_t>(ws, L.chunk_base);
    const uint32_t nfb = (uint32_t)cdiv(nmax, FIN_THREADS);
    static_assert(FIN_THREADS == 256, "finalize blocks also cover the r + 1 stack heights");
    launch_k(tree_nodes_finalize_kernel, nfb, FIN_THREADS, 0, s, nodes, nmax, Dd, slack_mode, cap, sum, nch,
             (const int32_t*)Sd, r, (uint32_t)stack_cap, leafpar);
    PS_LAUNCH_CHECK();
    PS_CUDA((device_scan<uint32_t, OpSum<uint32_t>>(nch, cb, nmax, false, true, at<uint32_t>(ws, L.scantmp_u32),
                                                   cb + nmax, s)));
    launch_k(tree_chunks_kernel, CHUNK_MAP_CTAS, 256, 0, s, nodes, (const uint32_t*)cb, nmax, sum,
             at<uint32_t>(ws, L.stage_chunk), (uint32_t)std::min<uint64_t>(L.chunks_max, 0xFFFFFFFFull),
             at<uint32_t>(ws, L.chunk2node));
    PS_LAUNCH_CHECK();
    return finish_tree(ws, L, info, s, pend, false);
}

// stages with at least this many cuts use the thin partition kernel
constexpr uint32_t THIN_CUTS = 12000;

// Runs one batch of disjoint merge nodes [nlo, nhi) whose chunks are
// [c0, c1): small nodes by warps, big ones by partition + the TMA pipeline.
template <class K>
struct MergeRunner {
    Bufs<K> bufs;
    const Node* nodes;
    const uint32_t* c2n;
    uint4* cuts;
    uint32_t* err;
    cudaStream_t s;
    size_t psmem, ssmem;
    uint32_t pipe_grid_max;

    uint64_t nelem;  // elements in each buffer
    int count_variant = -1;  // >= 0: CountingOrder counters of this merge variant per stage
    Summary* sum = nullptr;
    uint32_t* bars;  // grid-barrier counters, one per fused-partition pipe launch
    uint32_t nbars, bar_next;
    bool fuse;
    static inline bool coop_pdl = true;  // cooperative launches also take PDL until the driver refuses

    int init(Bufs<K> b, uint64_t n, const Node* nd, const uint32_t* chunk2node, uint4* ct, uint32_t* e,
             uint32_t* bar, uint32_t nbar, cudaStream_t st) {
        bufs = b;
        nelem = n;
        bars = bar;
        nbars = nbar;
        bar_next = 0;
        static const bool no_fuse = knob_set("PS_NO_FUSE");  // A/B: stand-alone partition launches
        fuse = !no_fuse && bar != nullptr;
        if (fuse) PS_CUDA(cudaMemsetAsync(bar, 0, (size_t)nbar * 4, st));
        nodes = nd;
        c2n = chunk2node;
        cuts = ct;
        err = e;
        s = st;
        psmem = merge_pipe_smem_bytes<K>();
        ssmem = merge_small_smem_bytes<K>();
        PS_CUDA(cudaFuncSetAttribute(merge_pipe_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
        // 4-byte keys: two CTAs per SM need the largest shared-memory carve-out
        PS_CUDA(cudaFuncSetAttribute(merge_pipe_kernel<K>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
        PS_CUDA(cudaFuncSetAttribute(merge_small_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
        PS_CUDA(cudaFuncSetAttribute(merge_mid_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)mid_smem_bytes<K>()));
        int dev = 0, sms = 148, occ = 1;
        PS_CUDA(cudaGetDevice(&dev));
        PS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        PS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, merge_pipe_kernel<K>, pipe_threads<K>(), psmem));
        pipe_grid_max = (uint32_t)std::max(1, sms * std::max(occ, 1));
        return PS_OK;
    }

    // the side stream of the counters and its events (sort-local; see stage())
    cudaStream_t side = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    bool join_pending = false;

    // one side stream and event pair per host thread and device, kept for the
    // thread's lifetime
    struct SideRes {
        int dev = -1;
        cudaStream_t st = nullptr;
        cudaEvent_t a = nullptr, b = nullptr;
    };
    static SideRes& side_res() {
        thread_local SideRes r;
        return r;
    }
    int use_side_stream() {
        int dev = 0;
        PS_CUDA(cudaGetDevice(&dev));
        SideRes& r = side_res();
        if (r.dev != dev) {
            if (r.st) {  // another device: release the old set (after its work)
                cudaStreamSynchronize(r.st);
                cudaEventDestroy(r.a);
                cudaEventDestroy(r.b);
                cudaStreamDestroy(r.st);
            }
            r = SideRes();
            PS_CUDA(cudaStreamCreateWithFlags(&r.st, cudaStreamNonBlocking));
            PS_CUDA(cudaEventCreateWithFlags(&r.a, cudaEventDisableTiming));
            PS_CUDA(cudaEventCreateWithFlags(&r.b, cudaEventDisableTiming));
            r.dev = dev;
        }
        side = r.st;
        ev_in = r.a;
        ev_out = r.b;
        return PS_OK;
    }
    // the previous stage's counters are done before anything overwrites their inputs
    int join() {
        if (join_pending) {
            PS_CUDA(cudaStreamWaitEvent(s, ev_out, 0));
            join_pending = false;
        }
        return PS_OK;
    }

    int stage(uint32_t nlo, uint32_t nhi, uint32_t c0, uint32_t c1, uint32_t nsmall, uint32_t small_max, Prof* prof,
              int stage_id) {
        if (nhi <= nlo) return PS_OK;
        {
            int rc = join();
            if (rc) return rc;
        }
        const uint32_t nbig = (nhi - nlo) - nsmall;
        // the tiny kernel counts its own nodes' comparisons for the sentinel /
        // no-sentinel 2-way and 4-way variants (every small node of such a stage is its)
        static const bool old_small = knob_set("PS_OLD_SMALL");  // A/B: warp-per-group kernel only
        static const uint32_t tiny_min = (uint32_t)knob("PS_TINY_MIN", 32768);
        const bool use_tiny = nsmall && !old_small && nsmall >= tiny_min && small_max <= 256;
        const bool tiny_counts = use_tiny && (count_variant == 0 || count_variant == 2 || count_variant == 3);
        if (count_variant >= 0) {
            // The counters read the stage's inputs, which no merge of this stage
            // overwrites: they run on a side stream next to the stage's merges
            // and the next stage waits for them.
            static_assert(COUNT_SMALL == SMALL_KERNEL_MAX, "level_small counts the thread-counted nodes");
            cudaStream_t cs = s;
            if (side) {
                PS_CUDA(cudaEventRecord(ev_in, s));
                PS_CUDA(cudaStreamWaitEvent(side, ev_in, 0));
                cs = side;
            }
            if (nsmall && !tiny_counts) {
                launch_k(merge_counters_small_kernel<K>, grid_for(nhi - nlo, 256), 256, 0, cs, bufs, nodes, nlo, nhi,
                         count_variant, sum);
                PS_LAUNCH_CHECK();
            }
            if (nbig) {
                launch_k(merge_counters_kernel<K>, grid_for(nhi - nlo, 8), 256, 0, cs, bufs, nodes, nlo, nhi,
                         count_variant, sum);
                PS_LAUNCH_CHECK();
            }
            if (side) {
                PS_CUDA(cudaEventRecord(ev_out, side));
                join_pending = true;
            }
        }
        if (nsmall) {
            // a thread per node while there are enough nodes to fill the GPU (a
            // warp per 32 nodes); otherwise the warp-per-group kernel
            auto tiny = [&](auto kern, size_t tsm, uint32_t warps) -> int {
                PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
                launch_k(kern, grid_for(nhi - nlo, 32ull * warps), warps * 32, tsm, s, bufs, nodes, nlo, nhi,
                         tiny_counts ? sum : nullptr);
                return PS_OK;
            };
            if (use_tiny && small_max <= 64)
                tiny(merge_tiny_kernel<K, 64>, merge_tiny_smem_bytes<K, 64>(), TinyCfg<K, 64>::WARPS);
            else if (use_tiny && small_max <= 96)
                tiny(merge_tiny_kernel<K, 96>, merge_tiny_smem_bytes<K, 96>(), TinyCfg<K, 96>::WARPS);
            else if (use_tiny && small_max <= 128)
                tiny(merge_tiny_kernel<K, 128>, merge_tiny_smem_bytes<K, 128>(), TinyCfg<K, 128>::WARPS);
            else if (use_tiny && small_max <= 256)
                tiny(merge_tiny_kernel<K, 256>, merge_tiny_smem_bytes<K, 256>(), TinyCfg<K, 256>::WARPS);
            else {
                static const bool warp_small = knob_set("PS_WARP_SMALL");  // A/B: the warp-per-group kernel
                if (warp_small) {
                    const uint32_t G = small_group(small_max);
                    launch_k(merge_small_kernel<K>, grid_for(cdiv(nhi - nlo, G), SMALL_WARPS), SMALL_WARPS * 32,
                             ssmem, s, bufs, nodes, nlo, nhi, G);
                } else {
                    const uint32_t G = mid_group<K>(small_max);
                    launch_k(merge_mid_kernel<K>, (unsigned)cdiv(nhi - nlo, G), MID_THREADS, mid_smem_bytes<K>(), s,
                             bufs, nodes, nlo, nhi, G);
                }
            }
            PS_LAUNCH_CHECK();
        }
        if (c1 > c0) {
            uint32_t* bar = nullptr;
            const uint32_t grid = std::min(c1 - c0, pipe_grid_max);
            if (c1 - c0 > nbig) {  // some node has several chunks: cuts needed
                // fused into the pipe launch while each of its warps has <= 1 cut to
                // find (the searches are latency-bound; more cuts need the wide grid)
                if (fuse && bar_next < nbars && c1 - c0 <= grid * (pipe_threads<K>() / 32)) {
                    bar = bars + bar_next++;  // partition fused into the pipe launch
                } else {
                    const int pp = prof ? prof->begin(3, stage_id, nbig, c1 - c0, 0) : -1;
                    // many cuts: three lanes per cut (fewer DRAM sectors); else a warp per cut
                    static const uint32_t thin_min =
                        (uint32_t)knob("PS_THIN_CUTS", THIN_CUTS);
                    if (c1 - c0 >= thin_min)
                        launch_k(merge_partition_thin_kernel<K>, grid_for(c1 - c0, 80), 256, 0, s, bufs, nodes, c2n,
                                 c0, c1, cuts);
                    else
                        launch_k(merge_partition_kernel<K>, grid_for(c1 - c0, 8), 256, 0, s, bufs, nodes, c2n, c0, c1,
                                 cuts);
                    PS_LAUNCH_CHECK();
                    if (prof) prof->end(pp);
                }
            }
            const uint32_t units = c1 - c0;
            if (bar) {
                // the fused partition's grid barrier needs every CTA resident:
                // a cooperative launch guarantees it (also against concurrent
                // sorts on other streams) or fails, and then the stage takes
                // the stand-alone partition
                cudaError_t e = launch_coop(coop_pdl, merge_pipe_kernel<K>, grid, pipe_threads<K>(), psmem, s, bufs,
                                            nelem, nodes, c2n, cuts, c0, units, err, bar);
                if (e != cudaSuccess && coop_pdl) {
                    (void)cudaGetLastError();
                    coop_pdl = false;  // this driver rejects cooperative + PDL
                    e = launch_coop(false, merge_pipe_kernel<K>, grid, pipe_threads<K>(), psmem, s, bufs, nelem,
                                    nodes, c2n, cuts, c0, units, err, bar);
                }
                if (e == cudaSuccess) {
                    PS_LAUNCH_CHECK();
                    return PS_OK;
                }
                (void)cudaGetLastError();
                launch_k(merge_partition_kernel<K>, grid_for(c1 - c0, 8), 256, 0, s, bufs, nodes, c2n, c0, c1, cuts);
                PS_LAUNCH_CHECK();
                bar = nullptr;
            }
            launch_k(merge_pipe_kernel<K>, grid, pipe_threads<K>(), psmem, s, bufs, nelem, nodes,
                     c2n, cuts, c0, units, err, bar);
            PS_LAUNCH_CHECK();
        }
        return PS_OK;
    }
};

int write_header(uint8_t* ws, const Layout& L, int64_t n, int64_t m, int k, int dtype, uint32_t r, uint32_t nmain,
                 uint32_t nspine, cudaStream_t s, int64_t moves_base = -1, bool exact = false) {
    WsHeader h;
    memset(&h, 0, sizeof(h));
    h.counters_pending = moves_base >= 0 ? 1u : 0u;
    h.moves_base = moves_base;
    h.counters_exact = exact ? 1 : 0;
    h.magic = WS_MAGIC;
    h.n = n;
    h.m = m;
    h.k = k;
    h.dtype = dtype;
    h.r = r;
    h.nmain = nmain;
    h.nspine_nodes = nspine;
    h.off_sum = L.sum;
    h.off_b = L.b;
    h.off_nat = L.nat;
    h.off_nodes = L.nodes;
    PS_CUDA(launch_k(write_header_kernel, 1, 32, 0, s, h, reinterpret_cast<WsHeader*>(ws + L.header)));
    return PS_OK;
}

int validate_cfg(const ps_config* cfg) {
    if (!cfg) return fail(PS_EINVAL, "config is NULL");
    if (cfg->k != 2 && cfg->k != 4) return fail(PS_EINVAL, "k must be 2 or 4, got " + std::to_string(cfg->k));
    int vk;
    switch (cfg->variant) {
        case PS_VARIANT_2WAY:
        case PS_VARIANT_2WAY_COPY_SMALLER:
        case PS_VARIANT_2WAY_NOSENTINEL:
            vk = 2;
            break;
        case PS_VARIANT_4WAY:
        case PS_VARIANT_4WAY_NOSENTINEL:
            vk = 4;
            break;
        default:
            return fail(PS_EINVAL, "unknown merge variant " + std::to_string(cfg->variant));
    }
    if (vk != cfg->k)
        return fail(PS_EINVAL, "variant implements k=" + std::to_string(vk) + ", but config asks for k=" +
                                   std::to_string(cfg->k));
    if (cfg->min_run_len < 1) return fail(PS_EINVAL, "min_run_len must be >= 1");
    return PS_OK;
}

int slack_mode_of(int variant) {
    switch (variant) {
        case PS_VARIANT_4WAY:
        case PS_VARIANT_2WAY:
            return 0;  // sentinel kernels: +arity writes per merge
        case PS_VARIANT_4WAY_NOSENTINEL:
            return 1;  // 2-way no-sentinel +0, stages +1
        default:
            return 2;
    }
}

template <class K>
int sort_impl(K* keys, int32_t* values, int64_t n, const ps_config& cfg, uint8_t* ws, size_t wsb, ps_stats* st,
              cudaStream_t s) {
    const uint64_t m = (uint64_t)cfg.min_run_len;
    const Layout L = make_layout((uint64_t)n, sizeof(K), m, true);
    if (wsb < L.total)
        return fail(PS_ENOMEM, "workspace too small: need " + std::to_string(L.total) + " bytes");
    const bool argsort = cfg.values_mode == PS_VALUES_ARGSORT;
    // PS_DEBUG_STAGES=s (measurement only): enqueue the first s merge stages;
    // -1 / -2 / -3: stop after run detection / the tree / leaf formation
    static const int stage_limit = (int)knob("PS_DEBUG_STAGES", 1 << 30);
    // data-dependent counters: comparisons / moves on request; copy-smaller's
    // buffer and scan counters always (both need a sync after the merges)
    const bool counting = cfg.count_comparisons != 0;
    const bool need_counts = counting || cfg.variant == PS_VARIANT_2WAY_COPY_SMALLER;
    Summary* sum = at<Summary>(ws, L.sum);
    PS_CUDA(cudaMemsetAsync(sum, 0, sizeof(Summary), s));
    uint32_t* err = &sum->err;
    uint32_t* ty = at<uint32_t>(ws, L.ty);
    uint32_t* cg = at<uint32_t>(ws, L.cg);
    uint32_t* Fg = at<uint32_t>(ws, L.Fg);
    uint32_t* Ft = at<uint32_t>(ws, L.Ft);
    uint32_t* b = at<uint32_t>(ws, L.b);
    uint32_t* nat = at<uint32_t>(ws, L.nat);
    const uint32_t ngroups = (uint32_t)L.ngroups;
    const int64_t rec_bytes = (int64_t)sizeof(K) + 4;
    Prof prof(s);

    // ---- N1 pass 1: run detection ------------------------------------------
    const int ph_rd = prof.begin(0, -1, 0, 0, n * (int64_t)sizeof(K));
    launch_k(rd_types_kernel<K>, ngroups, RD_THREADS, 0, s, keys, (uint64_t)n, ty, cg);
    PS_LAUNCH_CHECK();
    PS_CUDA((device_scan<uint32_t, OpMin<uint32_t>>(cg, Fg, ngroups, true, false, at<uint32_t>(ws, L.scantmp_u32),
                                                   nullptr, s)));
    if (m <= MAX_M_TILED) {
        const uint32_t M1 = (uint32_t)m + 1;
        uint64_t* tile_tab = at<uint64_t>(ws, L.tile_tab);
        uint64_t* gtab = at<uint64_t>(ws, L.lvl_tab[0]);
        const size_t smem = (size_t)TILES_PER_GROUP * M1 * 8;
        const size_t fan_smem = (size_t)TSCAN_FAN * M1 * 8;  // up to 64.3 KB at m = 256
        if (fan_smem > 48 * 1024) {
            PS_CUDA(cudaFuncSetAttribute(rd_compose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fan_smem));
            PS_CUDA(cudaFuncSetAttribute(rd_top_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fan_smem));
            PS_CUDA(cudaFuncSetAttribute(rd_down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fan_smem));
        }
        PS_CUDA(cudaFuncSetAttribute(rd_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        PS_CUDA(cudaFuncSetAttribute(rd_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch_k(rd_tables_kernel, ngroups, RD_THREADS, smem, s, ty, (uint64_t)n, (uint32_t)m, Fg, ngroups, tile_tab, Ft, gtab,
                                                   err);
        PS_LAUNCH_CHECK();
        const size_t c2smem = rd_chain2_smem((uint32_t)L.lvlP[0], (uint32_t)m);
        static const size_t c2max = (size_t)knob("PS_CHAIN2_MAX", 64 * 1024);
        if (L.tab_levels == 2 && c2smem <= c2max) {  // (bigger: one SM staging every table loses)
            // two levels: compose, top and down in one CTA
            PS_CUDA(cudaFuncSetAttribute(rd_chain2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2smem));
            launch_k(rd_chain2_kernel, 1, (unsigned)(32 * cdiv(L.lvlP[0], TSCAN_FAN)), c2smem, s,
                     (const uint64_t*)at<uint64_t>(ws, L.lvl_tab[0]), (uint32_t)L.lvlP[0], (const uint32_t*)Ft,
                     (uint64_t)n, (uint32_t)m, at<uint64_t>(ws, L.lvl_ent[0]), b, sum, err);
            PS_LAUNCH_CHECK();
        } else {
            uint64_t span = GROUP;
            std::vector<uint64_t> spans(L.tab_levels);
            for (uint64_t l = 0; l < L.tab_levels; ++l) {
                spans[l] = span;
                if (l + 1 < L.tab_levels) {
                    launch_k(rd_compose_kernel, (unsigned)L.lvlP[l + 1], 32, fan_smem, s, 
                        at<uint64_t>(ws, L.lvl_tab[l]), (uint32_t)L.lvlP[l], span, Ft, (uint64_t)n, (uint32_t)m,
                        at<uint64_t>(ws, L.lvl_tab[l + 1]), err);
                    PS_LAUNCH_CHECK();
                    span *= TSCAN_FAN;
                }
            }
            const uint64_t top = L.tab_levels - 1;
            launch_k(rd_top_kernel, 1, 32, fan_smem, s, at<uint64_t>(ws, L.lvl_tab[top]), (uint32_t)L.lvlP[top], spans[top], Ft,
                                           (uint64_t)n, (uint32_t)m, at<uint64_t>(ws, L.lvl_ent[top]), b, sum, err);
            PS_LAUNCH_CHECK();
            for (int64_t l = (int64_t)top - 1; l >= 0; --l) {
                launch_k(rd_down_kernel, (unsigned)L.lvlP[l + 1], 32, fan_smem, s, 
                    at<uint64_t>(ws, L.lvl_tab[l]), (uint32_t)L.lvlP[l], spans[l], Ft, (uint64_t)n, (uint32_t)m,
                    at<uint64_t>(ws, L.lvl_ent[l + 1]), at<uint64_t>(ws, L.lvl_ent[l]), err);
                PS_LAUNCH_CHECK();
            }
        }
        launch_k(rd_emit_kernel, ngroups, RD_THREADS, smem, s, ty, (uint64_t)n, (uint32_t)m, Fg, ngroups, tile_tab, Ft,
                 at<uint64_t>(ws, L.lvl_ent[0]), b, nat, at<uint32_t>(ws, L.tile_first), err);
        PS_LAUNCH_CHECK();
    } else {
        launch_k(rd_serial_kernel, 1, 32, 0, s, ty, (uint64_t)n, m, b, nat, sum);
        PS_LAUNCH_CHECK();
    }
    prof.end(ph_rd);
    Summary h;
    {
        int rc = publish(sum, SUM_HEAD, &h, nullptr, 0, nullptr, s);
        if (rc) return rc;
    }
    if (h.err) return fail(PS_EINVARIANT, "run detection invariant violated (flags " + std::to_string(h.err) + ")");
    const uint32_t r = h.r;
    if (r < 1 || r + 2 > L.rmax) return fail(PS_EINVARIANT, "run count out of range: " + std::to_string(r));
    if (stage_limit == -1) return PS_OK;

    // ---- N2: merge tree --------------------------------------------------------
    uint8_t* leafpar = at<uint8_t>(ws, L.leafpar);
    TreeInfo info;
    memset(&info.s, 0, sizeof(info.s));
    uint32_t nnodes = 0;
    Pending tree_pend;  // the tree summary, collected after leaf formation is queued
    const int ph_tree = prof.begin(1, -1, 0, 0, 0);
    if (r >= 2) {
        int rc = build_tree(ws, L, r, (uint64_t)n, cfg.k, cfg.strict_merge_down, slack_mode_of(cfg.variant), leafpar,
                            info, s, tree_pend, cut_cap<K>());
        if (rc) return rc;
    } else {
        PS_CUDA(cudaMemsetAsync(leafpar, 0, 1, s));
    }
    prof.end(ph_tree);
    if (stage_limit == -2) return PS_OK;

    // ---- N1 pass 2: leaves -----------------------------------------------------
    Bufs<K> bufs;
    bufs.k[0] = keys;
    bufs.v[0] = values;
    bufs.k[1] = at<K>(ws, L.k1);
    bufs.v[1] = at<int32_t>(ws, L.v1);
    {
        const size_t smem = form_smem_bytes<K>((uint32_t)std::min<uint64_t>(m, MAX_FORM_M), net_windows(m));
        const unsigned grid = grid_for((uint64_t)n, (uint64_t)FORM_TILE * FORM_TPC);
        static_assert(FORM_TILE == TILE, "leaf formation tiles are run detection's chain tiles");
        // per-tile first leaf, written by rd_emit_kernel (tiled detector only)
        const uint32_t* tile_first = m <= MAX_M_TILED ? at<uint32_t>(ws, L.tile_first) : nullptr;
        const int ph = prof.begin(2, -1, r, 0, n * ((int64_t)sizeof(K) + rec_bytes));
        if (argsort) {
            PS_CUDA(cudaFuncSetAttribute(form_leaves_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            launch_k(form_leaves_kernel<K, true>, grid, FORM_THREADS, smem, s, bufs, (uint64_t)n, b, nat, leafpar, r, ty,
                     (uint32_t)m, tile_first, counting ? sum : nullptr);
        } else {
            PS_CUDA(cudaFuncSetAttribute(form_leaves_kernel<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            launch_k(form_leaves_kernel<K, false>, grid, FORM_THREADS, smem, s, bufs, (uint64_t)n, b, nat, leafpar, r,
                     ty, (uint32_t)m, tile_first, counting ? sum : nullptr);
        }
        PS_LAUNCH_CHECK();
        if (net_windows(m)) {
            // extended windows: a register sorting network per window (ps_form.cuh)
            const unsigned wg = grid_for(r, FORM_THREADS);  // a warp per 32 leaves
            auto go = [&](auto kern, size_t wsm) -> int {
                PS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
                launch_k(kern, wg, FORM_THREADS, wsm, s, bufs, (const uint32_t*)b, (const uint32_t*)nat,
                         (const uint8_t*)leafpar, r, (const uint32_t*)ty, (uint64_t)n, counting ? sum : nullptr);
                return PS_OK;
            };
            if (argsort) {
                if (m <= 8) go(form_windows_kernel<K, 8, true>, form_windows_smem<K, 8>());
                else if (m <= 16) go(form_windows_kernel<K, 16, true>, form_windows_smem<K, 16>());
                else if (m <= 24) go(form_windows_kernel<K, 24, true>, form_windows_smem<K, 24>());
                else go(form_windows_kernel<K, 32, true>, form_windows_smem<K, 32>());
            } else {
                if (m <= 8) go(form_windows_kernel<K, 8, false>, form_windows_smem<K, 8>());
                else if (m <= 16) go(form_windows_kernel<K, 16, false>, form_windows_smem<K, 16>());
                else if (m <= 24) go(form_windows_kernel<K, 24, false>, form_windows_smem<K, 24>());
                else go(form_windows_kernel<K, 32, false>, form_windows_smem<K, 32>());
            }
            PS_LAUNCH_CHECK();
        }
        if (m > MAX_FORM_M && (uint64_t)n > MAX_FORM_M) {
            // windows longer than a tile's staging capacity: one CTA per window
            const size_t bsm = big_window_smem_bytes<K>();
            if (argsort)
                launch_k(form_big_windows_kernel<K, true>, BIGW_CTAS, BIGW_THREADS, bsm, s, bufs, (const uint32_t*)b,
                         (const uint32_t*)nat, (const uint8_t*)leafpar, r);
            else
                launch_k(form_big_windows_kernel<K, false>, BIGW_CTAS, BIGW_THREADS, bsm, s, bufs, (const uint32_t*)b,
                         (const uint32_t*)nat, (const uint8_t*)leafpar, r);
            PS_LAUNCH_CHECK();
        }
        prof.end(ph);
    }

    if (r >= 2) {
        int rc = tree_wait(L, info, s, tree_pend);
        if (rc) return rc;
        nnodes = info.s.nmain + info.s.nspine_nodes;
    }
    if (stage_limit == -3) return PS_OK;
    {
        int rc = write_header(ws, L, n, (int64_t)m, cfg.k, 0, r, info.s.nmain, info.s.nspine_nodes, s);
        if (rc) return rc;
    }

    // ---- N3/N4: merges, stage by stage ------------------------------------------
    // enqueued without a final synchronization: the counters are known from the
    // tree; merge-phase invariant flags are read by ps_check()
    if (nnodes) {
        MergeRunner<K> mr;
        int rc = mr.init(bufs, (uint64_t)n, at<Node>(ws, L.nodes), at<uint32_t>(ws, L.chunk2node), at<uint4>(ws, L.cuts),
                         err, at<uint32_t>(ws, L.bars), NBARS, s);
        if (rc) return rc;
        mr.count_variant = need_counts ? cfg.variant : -1;
        mr.sum = sum;
        if (need_counts) {
            rc = mr.use_side_stream();
            if (rc) return rc;
        }
        int stage = 0;
        auto run_stage = [&](uint32_t nlo, uint32_t nhi, uint32_t c0, uint32_t c1, uint64_t cost, uint32_t nsmall,
                             uint32_t small_max) -> int {
            if (nhi <= nlo || stage >= stage_limit) return PS_OK;
            const int ph = prof.begin(4, stage, nhi - nlo, c1 - c0, 2 * (int64_t)cost * rec_bytes);
            int rc2 = mr.stage(nlo, nhi, c0, c1, nsmall, small_max, &prof, stage);
            prof.end(ph);
            stage++;
            return rc2;
        };
        // one launch per merge stage (T6): power levels, higher first, with the
        // merge_down nodes one stage after their last input
        for (uint32_t h = 1; h < NSTAGE; ++h) {
            rc = run_stage(info.s.level_off[h], info.s.level_off[h + 1], info.level_chunk(h), info.level_chunk(h + 1),
                           info.s.level_cost[h], info.s.level_small[h], info.s.level_small_max[h]);
            if (rc) return rc;
        }
        rc = mr.join();  // the last counters land before the summary is read
        if (rc) return rc;
    }
    prof.finish();  // synchronizes only while profiling

    // ---- N5: SortStats (statskit.py:75-98), from the tree summary ----------------
    // The data-dependent counters and the merge-phase invariant flags arrive
    // after the merges (unless the caller asked for PS_FLAG_ASYNC).
    Summary c;
    memset(&c, 0, sizeof(c));
    // An asynchronous counting sort (not copy-smaller, whose buffer and scan
    // counters are data-dependent too) leaves comparisons / moves on the
    // device: ps_result_counters() reads them once the stream has finished.
    const bool defer = counting && (cfg.flags & PS_FLAG_ASYNC) && cfg.variant != PS_VARIANT_2WAY_COPY_SMALLER;
    if (!defer && (need_counts || !(cfg.flags & PS_FLAG_ASYNC))) {
        int rc = publish(sum, need_counts ? SUM_STATS : SUM_HEAD, &c, nullptr, 0, nullptr, s);
        if (rc) return rc;
        if (c.err & ERR_STACK) return fail(PS_EOVERFLOW, "run stack exceeded its height bound");
        if (c.err)
            return fail(PS_EINVARIANT, "merge-phase device invariant violated (flags " + std::to_string(c.err) + ")");
    }
    h = info.s;
    memset(st, 0, sizeof(*st));
    const int64_t M = (int64_t)h.merge_cost;
    st->merge_cost = M;
    st->merges2 = (int64_t)h.merges[2];
    st->merges3 = (int64_t)h.merges[3];
    st->merges4 = (int64_t)h.merges[4];
    st->runs_detected = r;
    st->max_stack_height = h.max_stack;
    st->buffer_cost = M;
    st->scan_reads = n + 2 * M;
    st->scan_writes = n + 2 * M + (int64_t)h.scan_slack;
    st->comparisons = -1;
    st->moves = -1;
    st->comparisons_valid = 0;
    st->moves_valid = 0;
    const bool sentinel_tournament = cfg.variant == PS_VARIANT_4WAY;
    const int64_t m34 = (int64_t)(h.merges[3] + h.merges[4]);
    if (cfg.variant == PS_VARIANT_2WAY_COPY_SMALLER) {
        // merges.py:145-201: only the smaller run is buffered; copied + written moves
        const int64_t cw = (int64_t)(c.cs_copied + c.cs_written);
        st->buffer_cost = (int64_t)c.cs_copied;
        st->scan_reads = n + cw;
        st->scan_writes = n + cw;
    }
    if (counting) {
        // comparisons: detection + extension + merges
        // (the insertion shifts of windows longer than MAX_FORM_M are not counted)
        const bool exact = !(m > MAX_FORM_M && (uint64_t)n > MAX_FORM_M);
        st->comparisons_valid = exact;
        st->comparisons = exact ? (int64_t)c.comparisons : -1;
        // moves: reversals + insertions, then per merge 2 * size (buffer out and
        // back), + 1 for a stages merge, copied + written for copy-smaller
        int64_t mv = (int64_t)c.moves;
        if (cfg.variant == PS_VARIANT_2WAY_COPY_SMALLER)
            mv += (int64_t)(c.cs_copied + c.cs_written);
        else
            mv += 2 * M + (sentinel_tournament ? 0 : m34);
        st->moves = exact ? mv : -1;
        st->moves_valid = exact;
        if (defer) {
            // the header records what ps_result_counters needs (written behind the merges)
            const int64_t base = mv - (int64_t)c.moves;  // (c is zero here: the tree part)
            int rc = write_header(ws, L, n, (int64_t)m, cfg.k, 0, r, info.s.nmain, info.s.nspine_nodes, s, base,
                                  exact);
            if (rc) return rc;
            PS_LAUNCH_CHECK();
            st->comparisons = st->moves = -1;
            st->comparisons_valid = st->moves_valid = exact ? 2 : 0;  // 2: pending (ps_result_counters)
        }
    }
    return PS_OK;
}

// ---------------------------------------------------------------------------
// Synchronizes `stream` and reports the device invariant flags of the last
// ps_sort on `workspace` (merge-phase chunk bounds, grid barriers).
int check_impl(void* workspace, cudaStream_t s) {
    WsHeader hd;
    PS_CUDA(cudaStreamSynchronize(s));
    PS_CUDA(cudaMemcpy(&hd, workspace, sizeof(hd), cudaMemcpyDeviceToHost));
    if (hd.magic != WS_MAGIC) return fail(PS_EINVAL, "workspace holds no sort");
    uint32_t err = 0;
    PS_CUDA(cudaMemcpy(&err, (const uint8_t*)workspace + hd.off_sum + offsetof(Summary, err), 4,
                       cudaMemcpyDeviceToHost));
    if (err) return fail(PS_EINVARIANT, "device invariant violated (flags " + std::to_string(err) + ")");
    return PS_OK;
}

// ---------------------------------------------------------------------------
// N6 cross-shard merge (ps_shard_merge): bracketing selection of the slab's
// ends, sample cuts, one merge launch (ps_shard.cuh).  No host round trip
// until the final error check.
struct ShardLayout {
    uint64_t bounds, targets, err, plan, smp, rows, total, rows_cap, smp_cap;
};

// samples per cut for G shards: a chunk's bracketed windows, G * (m + 2) *
// stride records, fit one unit of xm_cap records
template <class K>
uint32_t shard_cut_samples(uint32_t G) {
    const int m = (int)(xm_cap<K>() / (G * xs_stride<K>())) - 2;
    return (uint32_t)std::max(m, 1);
}

template <class K>
ShardLayout shard_layout(uint64_t slab_n) {
    ShardLayout L;
    memset(&L, 0, sizeof(L));
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t o = off;
        off = align_up(off + std::max<uint64_t>(bytes, 1), 256);
        return o;
    };
    L.smp_cap = slab_n / xs_stride<K>() + MAX_SHARDS + 1;
    L.rows_cap = slab_n / ((uint64_t)shard_cut_samples<K>(MAX_SHARDS) * xs_stride<K>()) + 2 * MAX_SHARDS + 2;
    L.bounds = take(2 * 2 * MAX_SHARDS * 8);
    L.targets = take(16);
    L.err = take(16);
    L.plan = take(sizeof(XPlan));
    L.smp = take(L.smp_cap * sizeof(K));
    L.rows = take(L.rows_cap * sizeof(XRow<K>));
    L.total = off;
    return L;
}

template <class K>
int shard_merge_impl(int32_t G, const void* const* shard_keys, const int32_t* const* shard_vals,
                     const void* const* shard_samples, const int64_t* shard_n, int64_t t0, int64_t t1, K* out_k,
                     int32_t* out_v, uint8_t* ws, size_t wsb, cudaStream_t s) {
    if (G < 1 || G > (int32_t)MAX_SHARDS) return fail(PS_EINVAL, "nshards must be in 1..8");
    if (!shard_keys || !shard_vals || !shard_n || !ws) return fail(PS_EINVAL, "NULL pointer argument");
    ShardSet<K> S;
    memset(&S, 0, sizeof(S));
    S.G = (uint32_t)G;
    uint64_t N = 0;
    for (int32_t h = 0; h < G; ++h) {
        if (shard_n[h] < 0 || shard_n[h] > ((int64_t)1 << 31)) return fail(PS_EINVAL, "shard length outside [0, 2^31]");
        S.k[h] = reinterpret_cast<const K*>(shard_keys[h]);
        S.v[h] = shard_vals[h];
        S.smp[h] = shard_samples ? reinterpret_cast<const K*>(shard_samples[h]) : nullptr;
        S.n[h] = (uint64_t)shard_n[h];
        N += (uint64_t)shard_n[h];
    }
    if (t0 < 0 || t1 < t0 || (uint64_t)t1 > N) return fail(PS_EINVAL, "slab range outside [0, sum(shard_n)]");
    const uint64_t slab = (uint64_t)(t1 - t0);
    if (slab > ((uint64_t)1 << 31)) return fail(PS_EINVAL, "slab longer than 2^31");
    const ShardLayout L = shard_layout<K>(slab);
    if (wsb < L.total) return fail(PS_ENOMEM, "shard-merge workspace too small");
    if (slab == 0) return PS_OK;
    unsigned long long* bounds = at<unsigned long long>(ws, L.bounds);
    uint64_t* targets = at<uint64_t>(ws, L.targets);
    uint32_t* d_err = at<uint32_t>(ws, L.err);
    XPlan* plan = at<XPlan>(ws, L.plan);
    K* smp = at<K>(ws, L.smp);
    XRow<K>* rows = at<XRow<K>>(ws, L.rows);
    PS_CUDA(cudaMemsetAsync(d_err, 0, 4, s));

    // ---- co-ranks of t0 and t1: fixed rounds of parallel bracketing ----------------
    launch_k(xs_init_kernel<K>, 1, 32, 0, s, S, (uint64_t)t0, (uint64_t)t1, bounds, targets);
    PS_LAUNCH_CHECK();
    uint64_t maxw = 1;
    for (int32_t h = 0; h < G; ++h) maxw = std::max<uint64_t>(maxw, S.n[h]);
    int rounds = 2;  // a window of w <= SEL_CANDIDATES + 1 positions is resolved in one round
    for (uint64_t w = maxw; w > SEL_CANDIDATES + 1; w = w / (SEL_CANDIDATES + 1) + 1) rounds++;
    const dim3 sgrid((unsigned)cdiv((uint64_t)G * SEL_CANDIDATES, 8), 2);
    for (int it = 0; it < rounds; ++it) {
        launch_k(shard_select_kernel<K>, sgrid, 256, 0, s, S, (const uint64_t*)targets, bounds);
        PS_LAUNCH_CHECK();
    }
    // ---- plan, local sample windows, cuts -----------------------------------------
    const uint32_t m = shard_cut_samples<K>((uint32_t)G);
    launch_k(xs_plan_kernel<K>, 1, 32, 0, s, S, (const unsigned long long*)bounds, (uint64_t)t0, (uint64_t)t1, m,
             plan, d_err);
    PS_LAUNCH_CHECK();
    const unsigned sgrid2 = (unsigned)std::min<uint64_t>(cdiv(slab / xs_stride<K>() + 1, 256), 148 * 8);
    launch_k(xs_sample_copy_kernel<K>, sgrid2, 256, 0, s, S, (const XPlan*)plan, smp);
    PS_LAUNCH_CHECK();
    const uint64_t max_cuts = L.rows_cap;
    launch_k(xs_cuts_kernel<K>, (unsigned)std::min<uint64_t>(cdiv(max_cuts, 256), 148 * 8), 256, 0, s, S,
             (const XPlan*)plan, (const K*)smp, rows);
    PS_LAUNCH_CHECK();
    // ---- one merge launch: two CTAs per SM ------------------------------------------
    static bool attr_set = false;
    const size_t smem = xm_smem_bytes<K>();
    if (!attr_set) {
        PS_CUDA(cudaFuncSetAttribute(xs_merge_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    int dev = 0, nsm = 148;
    PS_CUDA(cudaGetDevice(&dev));
    PS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const unsigned mgrid = (unsigned)std::min<uint64_t>(2 * (uint64_t)nsm, cdiv(slab, xm_cap<K>() / 2) + 1);
    launch_k(xs_merge_kernel<K>, mgrid, XM_THREADS, smem, s, S, (const XPlan*)plan, (const XRow<K>*)rows, out_k,
             out_v, (uint64_t)t0, d_err);
    PS_LAUNCH_CHECK();
    uint32_t herr = 0;
    PS_CUDA(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, s));
    PS_CUDA(cudaStreamSynchronize(s));
    if (herr) return fail(PS_EINVARIANT, "shard merge invariant violated (flags " + std::to_string(herr) + ")");
    return PS_OK;
}

template <class K>
int shard_samples_impl(const void* keys, int64_t n, void* samples, cudaStream_t s) {
    if (n < 0) return fail(PS_EINVAL, "n must be >= 0");
    if (n == 0) return PS_OK;
    if (!keys || !samples) return fail(PS_EINVAL, "NULL pointer argument");
    const uint64_t ns = cdiv((uint64_t)n, xs_stride<K>());
    launch_k(xs_samples_kernel<K>, (unsigned)std::min<uint64_t>(cdiv(ns, 256), 148 * 8), 256, 0, s,
             (const K*)keys, (uint64_t)n, (K*)samples);
    PS_LAUNCH_CHECK();
    return PS_OK;
}

}  // namespace

// =============================================================================
namespace {
// dst row i = src row perm[i]: thread per (row, W-byte word), words of a row
// consecutive across threads (coalesced stores, row-contiguous loads)
template <class W>
__global__ void gather_rows_kernel(const W* __restrict__ src, const int32_t* __restrict__ perm, W* __restrict__ dst,
                                   uint64_t n, uint64_t wpr) {
    pdl_wait();
    const uint64_t tot = n * wpr;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < tot; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t row = t / wpr, w = t - row * wpr;
        dst[t] = src[(uint64_t)perm[row] * wpr + w];
    }
}

}  // namespace

extern "C" {

const char* ps_last_error(void) { return g_last_error.c_str(); }

const char* ps_version(void) { return "powersort-b200 0.1.0 (sm_100a)"; }

int ps_profile_enable(int32_t on) {
    g_prof_on = on != 0;
    return PS_OK;
}

int ps_profile_read(ps_prof_entry* out, int32_t cap, int32_t* count) {
    const int32_t n = (int32_t)g_prof_last.size();
    if (count) *count = n;
    if (out)
        for (int32_t i = 0; i < n && i < cap; ++i) out[i] = g_prof_last[i];
    return PS_OK;
}

int64_t ps_launch_count(void) { return launch_counter().load(); }

size_t ps_workspace_size(int64_t n, int32_t dtype, const ps_config* cfg) {
    if (n < 0 || !cfg || cfg->min_run_len < 1) return 0;
    uint64_t kb = dtype == PS_INT32 || dtype == PS_FLOAT32 ? 4 : (dtype == PS_INT64 || dtype == PS_FLOAT64 ? 8 : 0);
    if (!kb) return 0;
    return (size_t)make_layout((uint64_t)n, kb, (uint64_t)cfg->min_run_len, true).total;
}

int ps_check(void* workspace, void* stream) {
    if (!workspace) return fail(PS_EINVAL, "NULL pointer argument");
    return check_impl(workspace, (cudaStream_t)stream);
}

int ps_sort(int32_t dtype, void* keys, int32_t* values, int64_t n, const ps_config* cfg, void* workspace,
            size_t workspace_bytes, ps_stats* stats, void* stream) {
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (n < 0) return fail(PS_EINVAL, "n must be >= 0");
    if (n > ((int64_t)1 << 31)) return fail(PS_EINVAL, "n > 2^31 is not supported (int32 payload)");
    if (!stats) return fail(PS_EINVAL, "stats is NULL");
    memset(stats, 0, sizeof(*stats));
    if (n == 0) return PS_OK;  // policy.py:207-209
    if (!keys || !values || !workspace) return fail(PS_EINVAL, "NULL pointer argument");
    if (((uintptr_t)keys | (uintptr_t)values | (uintptr_t)workspace) & 15)
        return fail(PS_EINVAL, "keys, values and workspace must be 16-byte aligned (TMA and vector access)");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    switch (dtype) {
        case PS_INT32:
            return sort_impl<int32_t>((int32_t*)keys, values, n, *cfg, ws, workspace_bytes, stats, s);
        case PS_INT64:
            return sort_impl<int64_t>((int64_t*)keys, values, n, *cfg, ws, workspace_bytes, stats, s);
        case PS_FLOAT32:
            return sort_impl<float>((float*)keys, values, n, *cfg, ws, workspace_bytes, stats, s);
        case PS_FLOAT64:
            return sort_impl<double>((double*)keys, values, n, *cfg, ws, workspace_bytes, stats, s);
        default:
            return fail(PS_EINVAL, "unsupported dtype " + std::to_string(dtype));
    }
}

static int read_header(const void* workspace, WsHeader& h) {
    if (!workspace) return fail(PS_EINVAL, "workspace is NULL");
    // ps_sort returns with work queued on its stream, which may be any stream
    PS_CUDA(cudaDeviceSynchronize());
    PS_CUDA(cudaMemcpy(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost));
    if (h.magic != WS_MAGIC) return fail(PS_EINVAL, "workspace holds no sort result");
    return PS_OK;
}

int ps_result_counters(void* workspace, void* stream, int64_t* comparisons, int64_t* moves) {
    if (!workspace) return fail(PS_EINVAL, "NULL pointer argument");
    // the header and the summary's flags and counters through the host-mapped
    // publish, stream-ordered behind the sort: no device-wide synchronization
    // and no copy-engine transfer, which would queue behind bulk copies of
    // other streams (a pipelined caller's)
    static_assert(sizeof(WsHeader) <= 256, "the summary follows the header at byte 256");
    WsHeader h;
    Summary* sp = new Summary;
    memset(sp, 0, sizeof(Summary));
    const uint8_t* ws = (const uint8_t*)workspace;
    int rc = publish(ws, sizeof(WsHeader), &h, ws + 256, offsetof(Summary, moves) + 8, sp, (cudaStream_t)stream);
    const uint32_t err = sp->err;
    const unsigned long long cm = sp->comparisons, mv = sp->moves;
    delete sp;
    if (rc) return rc;
    if (h.magic != WS_MAGIC || h.off_sum != 256) return fail(PS_EINVAL, "workspace holds no sort result");
    if (!h.counters_pending) return fail(PS_EINVAL, "the last sort on this workspace has no pending counters");
    if (err) return fail(PS_EINVARIANT, "device invariant violated (flags " + std::to_string(err) + ")");
    if (comparisons) *comparisons = h.counters_exact ? (int64_t)cm : -1;
    if (moves) *moves = h.counters_exact ? (int64_t)mv + h.moves_base : -1;
    return PS_OK;
}

int ps_result_counts(const void* workspace, int64_t* runs, int64_t* merges) {
    WsHeader h;
    int rc = read_header(workspace, h);
    if (rc) return rc;
    if (runs) *runs = h.r;
    if (merges) *merges = (int64_t)h.nmain + h.nspine_nodes;
    return PS_OK;
}

int ps_result_runs(const void* workspace, int64_t* run_lengths, int64_t* natural_run_lengths, int64_t cap) {
    WsHeader h;
    int rc = read_header(workspace, h);
    if (rc) return rc;
    if (cap < (int64_t)h.r) return fail(PS_EINVAL, "capacity below the run count");
    const uint8_t* ws = (const uint8_t*)workspace;
    std::vector<uint32_t> b(h.r + 1), nat(h.r);
    PS_CUDA(cudaMemcpy(b.data(), ws + h.off_b, (h.r + 1) * 4, cudaMemcpyDeviceToHost));
    if (natural_run_lengths && h.off_nat)
        PS_CUDA(cudaMemcpy(nat.data(), ws + h.off_nat, h.r * 4, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < h.r; ++i) {
        if (run_lengths) run_lengths[i] = (int64_t)b[i + 1] - b[i];
        if (natural_run_lengths) natural_run_lengths[i] = h.off_nat ? nat[i] : (int64_t)b[i + 1] - b[i];
    }
    return PS_OK;
}

int ps_result_trace(const void* workspace, int64_t* rows, int64_t cap) {
    WsHeader h;
    int rc = read_header(workspace, h);
    if (rc) return rc;
    const uint32_t nn = h.nmain + h.nspine_nodes;
    if (cap < (int64_t)nn) return fail(PS_EINVAL, "capacity below the merge count");
    std::vector<Node> nodes(nn);
    if (nn)
        PS_CUDA(cudaMemcpy(nodes.data(), (const uint8_t*)workspace + h.off_nodes, nn * sizeof(Node),
                           cudaMemcpyDeviceToHost));
    // main-loop merges execute when boundary R arrives, higher powers first
    // (policy.py:250-259); then _merge_down in sequence (policy.py:146-175).
    // (the node table is grouped by height, T6: the order is rebuilt here)
    std::vector<uint32_t> idx, spine;
    for (uint32_t i = 0; i < nn; ++i) (nodes[i].flags & 1 ? spine : idx).push_back(i);
    std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
        const Node &x = nodes[a], &y = nodes[b];
        const uint32_t ex = x.pos[x.arity], ey = y.pos[y.arity];
        if (ex != ey) return ex < ey;
        return x.power > y.power;
    });
    std::sort(spine.begin(), spine.end(), [&](uint32_t a, uint32_t b) { return nodes[a].order < nodes[b].order; });
    idx.insert(idx.end(), spine.begin(), spine.end());
    for (uint32_t i = 0; i < nn; ++i) {
        const Node& x = nodes[idx[i]];
        int64_t* row = rows + 7 * i;
        row[0] = x.arity;
        for (int j = 0; j < 5; ++j) row[1 + j] = -1;
        for (int j = 0; j <= x.arity; ++j) row[1 + j] = x.pos[j];
        row[6] = (int64_t)x.pos[x.arity] - x.pos[0];
    }
    return PS_OK;
}

size_t ps_profile_workspace_size(int64_t r, int64_t n) {
    if (r < 1 || n < r) return 0;
    return (size_t)make_layout((uint64_t)n, 4, 1, false, (uint64_t)r).total;
}

int ps_tree_from_profile(const int64_t* lengths, int64_t r, int32_t k, int32_t strict_merge_down, void* workspace,
                         size_t workspace_bytes, int64_t* merge_cost, int64_t* max_stack_height, void* stream) {
    if (k != 2 && k != 4) return fail(PS_EINVAL, "k must be 2 or 4, got " + std::to_string(k));
    if (r < 1 || !lengths) return fail(PS_EINVAL, "a run profile has at least one run");
    uint64_t n = 0;
    std::vector<uint32_t> b(r + 1);
    for (int64_t i = 0; i < r; ++i) {
        if (lengths[i] < 1) return fail(PS_EINVAL, "run lengths must be positive");
        b[i] = (uint32_t)n;
        n += (uint64_t)lengths[i];
        if (n > ((uint64_t)1 << 31)) return fail(PS_EINVAL, "profile longer than 2^31");
    }
    b[r] = (uint32_t)n;
    const Layout L = make_layout(n, 4, 1, false, (uint64_t)r);
    if (workspace_bytes < L.total) return fail(PS_ENOMEM, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
    PS_CUDA(cudaMemsetAsync(ws + L.sum, 0, sizeof(Summary), s));
    PS_CUDA(cudaMemcpyAsync(ws + L.b, b.data(), (r + 1) * 4, cudaMemcpyHostToDevice, s));
    TreeInfo info;
    memset(&info.s, 0, sizeof(info.s));
    if (r >= 2) {
        Pending pend;
        int rc = build_tree(ws, L, (uint32_t)r, n, k, strict_merge_down, 0, nullptr, info, s, pend);
        if (rc) return rc;
        rc = tree_wait(L, info, s, pend);
        if (rc) return rc;
    }
    int rc = write_header(ws, L, (int64_t)n, 1, k, 0, (uint32_t)r, info.s.nmain, info.s.nspine_nodes, s);
    if (rc) return rc;
    PS_CUDA(cudaStreamSynchronize(s));
    if (merge_cost) *merge_cost = (int64_t)info.s.merge_cost;
    if (max_stack_height) *max_stack_height = info.s.max_stack;
    return PS_OK;
}

int ps_node_power(int32_t k, int64_t n, int64_t b1, int64_t e1, int64_t b2, int64_t e2, int32_t any_k) {
    // power.py:47-74, exact in 128-bit integers
    if (!any_k && k != 2 && k != 3 && k != 4) return fail(-PS_EINVAL, "node_power supports k in {2, 3, 4}");
    if (k < 2) return fail(-PS_EINVAL, "boundary power needs k >= 2");
    if (!(0 <= b1 && b1 < e1 && e1 == b2 && b2 < e2 && e2 <= n)) return fail(-PS_EINVAL, "malformed run bounds");
    const unsigned __int128 A = (unsigned __int128)(b1 + e1), B = (unsigned __int128)(b2 + e2);
    const unsigned __int128 two_n = (unsigned __int128)2 * (unsigned __int128)n;
    unsigned __int128 kp = (unsigned __int128)k;
    int p = 1;
    while ((A * kp) / two_n == (B * kp) / two_n) {
        p++;
        kp *= (unsigned __int128)k;
    }
    return p;
}

int64_t ps_run_stack_capacity(int64_t k, int64_t n) {
    if (k < 2 || n < 1) return -PS_EINVAL;
    int64_t m = 0;
    unsigned __int128 p = 1;
    while (p < (unsigned __int128)n) {
        p *= (unsigned __int128)k;
        m++;
    }
    return (k - 1) * (m + 1);
}

size_t ps_shard_merge_workspace_size(int32_t nshards, int64_t slab_n) {
    if (nshards < 1 || nshards > (int32_t)MAX_SHARDS || slab_n < 0) return 0;
    return (size_t)std::max(shard_layout<int32_t>((uint64_t)slab_n).total, shard_layout<int64_t>((uint64_t)slab_n).total);
}

int64_t ps_shard_sample_count(int32_t dtype, int64_t n) {
    if (n < 0) return -PS_EINVAL;
    const int64_t s = (dtype == PS_INT64 || dtype == PS_FLOAT64) ? 16 : (dtype == PS_INT32 || dtype == PS_FLOAT32) ? 32 : 0;
    if (!s) return -PS_EINVAL;
    return (n + s - 1) / s;
}

int ps_shard_samples(int32_t dtype, const void* keys, int64_t n, void* samples, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
        case PS_INT32: return shard_samples_impl<int32_t>(keys, n, samples, s);
        case PS_INT64: return shard_samples_impl<int64_t>(keys, n, samples, s);
        case PS_FLOAT32: return shard_samples_impl<float>(keys, n, samples, s);
        case PS_FLOAT64: return shard_samples_impl<double>(keys, n, samples, s);
        default: return fail(PS_EINVAL, "unsupported dtype " + std::to_string(dtype));
    }
}

int ps_gather_rows(const void* src, const int32_t* perm, void* dst, int64_t n, int64_t row_bytes, void* stream) {
    if (n < 0 || row_bytes < 1) return fail(PS_EINVAL, "n must be >= 0 and row_bytes >= 1");
    if (n == 0) return PS_OK;
    if (!src || !perm || !dst) return fail(PS_EINVAL, "NULL pointer argument");
    cudaStream_t s = (cudaStream_t)stream;
    const uintptr_t al = (uintptr_t)src | (uintptr_t)dst | (uintptr_t)row_bytes;
    const unsigned grid = (unsigned)std::min<uint64_t>(cdiv((uint64_t)n * (uint64_t)row_bytes, 256 * 4), 148 * 32);
    if (al % 16 == 0)
        launch_k(gather_rows_kernel<uint4>, grid, 256, 0, s, (const uint4*)src, perm, (uint4*)dst, (uint64_t)n,
                 (uint64_t)row_bytes / 16);
    else if (al % 8 == 0)
        launch_k(gather_rows_kernel<uint2>, grid, 256, 0, s, (const uint2*)src, perm, (uint2*)dst, (uint64_t)n,
                 (uint64_t)row_bytes / 8);
    else if (al % 4 == 0)
        launch_k(gather_rows_kernel<uint32_t>, grid, 256, 0, s, (const uint32_t*)src, perm, (uint32_t*)dst,
                 (uint64_t)n, (uint64_t)row_bytes / 4);
    else
        launch_k(gather_rows_kernel<uint8_t>, grid, 256, 0, s, (const uint8_t*)src, perm, (uint8_t*)dst,
                 (uint64_t)n, (uint64_t)row_bytes);
    launch_counter()++;
    PS_CUDA(cudaGetLastError());
    return PS_OK;
}

// Peer shards: a CUDA IPC handle of another rank's allocation is opened in the
// CALLER's device context with lazy peer access, so the shard-merge kernel on
// this device can load from it over NVLink (an allocation opened in the peer
// device's own context would need cudaDeviceEnablePeerAccess as well).
int ps_ipc_export(int32_t device, const void* ptr, void* handle, int64_t* offset) {
    if (!ptr || !handle || !offset) return fail(PS_EINVAL, "NULL pointer argument");
    PS_CUDA(cudaSetDevice(device));
    // allocation base of ptr (cuMemGetAddressRange through the runtime's
    // driver entry point: no link-time libcuda dependency)
    using range_fn = int (*)(unsigned long long*, size_t*, unsigned long long);
    static range_fn range = nullptr;
    if (!range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        PS_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) return fail(PS_ECUDA, "cuMemGetAddressRange not found");
        range = (range_fn)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
        return fail(PS_ECUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    PS_CUDA(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return PS_OK;
}

int ps_ipc_open(int32_t device, const void* handle, void** base) {
    if (!handle || !base) return fail(PS_EINVAL, "NULL pointer argument");
    PS_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    *base = nullptr;
    PS_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    return PS_OK;
}

int ps_ipc_close(int32_t device, void* base) {
    if (!base) return PS_OK;
    PS_CUDA(cudaSetDevice(device));
    PS_CUDA(cudaIpcCloseMemHandle(base));
    return PS_OK;
}

int ps_shard_merge(int32_t dtype, int32_t nshards, const void* const* shard_keys, const int32_t* const* shard_vals,
                   const void* const* shard_samples, const int64_t* shard_n, int64_t out_begin, int64_t out_end,
                   void* out_keys, int32_t* out_vals, void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* ws = (uint8_t*)workspace;
#define PS_SM(K)                                                                                              \
    return shard_merge_impl<K>(nshards, shard_keys, shard_vals, shard_samples, shard_n, out_begin, out_end, \
                               (K*)out_keys, out_vals, ws, workspace_bytes, s)
    switch (dtype) {
        case PS_INT32: PS_SM(int32_t);
        case PS_INT64: PS_SM(int64_t);
        case PS_FLOAT32: PS_SM(float);
        case PS_FLOAT64: PS_SM(double);
        default: return fail(PS_EINVAL, "unsupported dtype " + std::to_string(dtype));
    }
#undef PS_SM
}

}  // extern "C"

#ifdef PS_PIPE_TIMING
// Diagnostics build only: clock64 phase counters of merge_pipe_kernel
// (producer: batch, wait-empty, stage, units; consumer: wait-full, pass 1,
// pass 2, store, units).
extern "C" int ps_debug_pipe_timing(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ps::g_pipe_tim, 40 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[40] = {0};
        cudaMemcpyToSymbol(ps::g_pipe_tim, z, sizeof(z));
    }
    return PS_OK;
}
extern "C" int ps_debug_cta_timing(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, ps::g_cta_tim, sizeof(ps::g_cta_tim));
    return PS_OK;
}
#endif

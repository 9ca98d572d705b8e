// ps_form.cuh -- N1 pass 2: leaf-run formation.
//
// Every leaf run of the reference is, after find_first_run's reversal
// (runs.py:41-47) and extend_run's insertion sort (runs.py:50-82), the stable
// sort of the original elements of its window.  Natural runs are
// copied (ascending) or reversed (strictly descending); extended windows
// (natural length < run length <= min_run_len) are ranked by (key, position).
// Each leaf is written straight into ping-pong buffer (leaf depth & 1), so
// no merge ever copies back.  Buffer 0 is the caller's array:
// parity-0 leaves are formed in place (reversals swap mirrored pairs owned by
// one thread; windows are staged in shared memory before being written).
#pragma once

#include "ps_common.cuh"
#include "ps_scan.cuh"

namespace ps {

constexpr uint32_t FORM_TILE = 2048;
constexpr uint32_t FORM_THREADS = 256;
#ifndef PS_FORM_TPC
#define PS_FORM_TPC 8
#endif
constexpr uint32_t FORM_TPC = PS_FORM_TPC;  // detection tiles per leaf-formation CTA
constexpr uint32_t MAX_FORM_M = 1024;
// PS_NO_NET=1 (A/B builds): short windows take the rank loop too
#ifndef PS_NO_NET
#define PS_NO_NET 0
#endif

template <class K>
struct Bufs {
    K* k[2];
    int32_t* v[2];
    // select, not an indexed access: a runtime index into the by-value kernel
    // parameter would spill the struct to local memory
    PS_DEV K* kb(uint32_t p) const { return p ? k[1] : k[0]; }
    PS_DEV int32_t* vb(uint32_t p) const { return p ? v[1] : v[0]; }
};

// shared layout: sb[FORM_TILE+2] u32, snat[FORM_TILE+1] u32, spar[FORM_TILE+1] u8,
//   wlist[FORM_TILE+1] u32 (window leaf ids), woff[FORM_TILE+2] u32,
//   wk[FORM_TILE+MAX_M] K, wv[...] i32
template <class K>
size_t form_smem_bytes(uint32_t m, bool net) {
    size_t s = 0;
    s += (FORM_TILE + 2) * 4;
    s += (FORM_TILE + 1) * 4;
    s += ((FORM_TILE + 1) + 15) / 16 * 16;
    if (net) return s;  // windows go to form_windows_kernel: no staging
    s += (FORM_TILE + 1) * 4;
    s += (FORM_TILE + 2) * 4;
    s = (s + 15) / 16 * 16;
    const size_t cap = FORM_TILE + (m < MAX_FORM_M ? m : MAX_FORM_M);
    s += cap * sizeof(K);
    s += cap * 4;
    s += (cap * 2 + 15) / 16 * 16;  // window index of every staged element
    return s;
}

// ---------------------------------------------------------------------------
// Short extended windows (min_run_len <= 32): one thread sorts a whole window
// in registers with Batcher's odd-even merge-sort network over (key, offset)
// pairs.  The offset breaks key ties, so the network's output is the stable
// sort of the window's original elements -- the leaf extend_run's insertion
// sort produces (runs.py:50-82).  Padding lanes (offset >= len)
// hold the largest key and a larger offset, so they sort past the window.
template <int S>
struct OddEvenNet {
    int cnt = 0;
    int a[S * 8] = {};
    int b[S * 8] = {};
    constexpr OddEvenNet() {
        for (int p = 1; p < S; p <<= 1)
            for (int k = p; k >= 1; k >>= 1)
                for (int j = k % p; j + k < S; j += 2 * k)
                    for (int i = 0; i < k && i + j + k < S; ++i)
                        if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
                            a[cnt] = i + j;
                            b[cnt] = i + j + k;
                            ++cnt;
                        }
    }
};
static_assert(OddEvenNet<32>().cnt == 191, "Batcher network size for 32 inputs");

// The power-of-two network restricted to L real inputs: wires L.. carry the
// padding (larger than every input), so a comparator whose upper wire is
// padding is a no-op and one whose lower wire is padding is a fixed swap --
// a relabelling of physical registers.  Only real-vs-real comparators remain
// (L = 24: 132 of 191); sorted wire j ends in physical register out[j].
template <int L>
struct PrunedNet {
    static constexpr int P = L <= 8 ? 8 : L <= 16 ? 16 : 32;
    int cnt = 0;
    int a[P * 8] = {};
    int b[P * 8] = {};
    int out[P] = {};
    constexpr PrunedNet() {
        const OddEvenNet<P> net{};
        int map[P] = {};
        bool real[P] = {};
        for (int w = 0; w < P; ++w) {
            map[w] = w;
            real[w] = w < L;
        }
        for (int c = 0; c < net.cnt; ++c) {
            const int x = net.a[c], y = net.b[c];
            if (!real[y]) continue;
            if (!real[x]) {
                const int t = map[x];
                map[x] = map[y];
                map[y] = t;
                real[x] = true;
                real[y] = false;
                continue;
            }
            a[cnt] = map[x];
            b[cnt] = map[y];
            ++cnt;
        }
        for (int w = 0; w < P; ++w) out[w] = map[w];
    }
};
static_assert(OddEvenNet<16>().cnt == 63, "Batcher network size for 16 inputs");

template <class K>
PS_DEV K key_pad();
template <>
PS_DEV int32_t key_pad<int32_t>() { return 0x7FFFFFFF; }
template <>
PS_DEV int64_t key_pad<int64_t>() { return 0x7FFFFFFFFFFFFFFFll; }
template <>
PS_DEV float key_pad<float>() { return __int_as_float(0x7F800000); }
template <>
PS_DEV double key_pad<double>() { return __longlong_as_double(0x7FF0000000000000ll); }

// Sorts k[0..S) (padding past the window) carrying the original offsets o[].
template <class K, int S>
PS_DEV void net_sort(K (&k)[S], uint32_t (&o)[S]) {
    constexpr PrunedNet<S> net{};
#pragma unroll
    for (int c = 0; c < net.cnt; ++c) {
        const int x = net.a[c], y = net.b[c];
        const K kx = k[x], ky = k[y];
        const uint32_t ox = o[x], oy = o[y];
        const bool sw = (ky < kx) || (!(kx < ky) && oy < ox);
        k[x] = sw ? ky : kx;
        k[y] = sw ? kx : ky;
        o[x] = sw ? oy : ox;
        o[y] = sw ? ox : oy;
    }
}

// Extended windows go to form_windows_kernel when they fit a network (it also
// counts the insertion sort's compares and moves when asked).
__host__ __device__ inline bool net_windows(uint64_t m) { return !PS_NO_NET && m <= 32; }

template <class K, int S>
constexpr size_t form_windows_smem() {
    return (size_t)(FORM_THREADS / 32) * 32 * (S + 1) * (sizeof(K) + 4);
}

// A warp per 32 consecutive leaves; each extended window (natural length <
// leaf length) is sorted by its lane's network, natural leaves are left to
// form_leaves_kernel.  Windows move through a per-warp shared-memory
// transpose (row w = window w, stride S+1 elements: conflict-free lane rows),
// so global loads and stores are one coalesced instruction per window.
//
// With `counters`, each lane also counts its window's insertion sort
// (runs.py:50-68): the element at offset q past the natural prefix, with s
// earlier window elements greater than it, costs s + [s < q] compares and
// s + 1 moves when s > 0 (statskit.py:49-72).
template <class K, int S, bool ARGSORT>
__global__ void __launch_bounds__(FORM_THREADS) form_windows_kernel(Bufs<K> bufs, const uint32_t* __restrict__ b,
                                                                    const uint32_t* __restrict__ nat,
                                                                    const uint8_t* __restrict__ leafpar, uint32_t r,
                                                                    const uint32_t* __restrict__ ty, uint64_t n,
                                                                    Summary* __restrict__ counters) {
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr uint32_t RW = S + 1;
    const uint32_t lane = lane_id(), warp = warp_id();
    K* sk = reinterpret_cast<K*>(smem) + (size_t)warp * 32 * RW;
    uint32_t* so = reinterpret_cast<uint32_t*>(reinterpret_cast<K*>(smem) + (size_t)(FORM_THREADS / 32) * 32 * RW) +
                   (size_t)warp * 32 * RW;
    const uint32_t i = (blockIdx.x * (FORM_THREADS / 32) + warp) * 32 + lane;
    uint32_t b0 = 0, len = 0, par = 0, nprefix = 0;
    if (i < r) {
        b0 = b[i];
        const uint32_t l = b[i + 1] - b0;
        nprefix = nat[i];
        if (nprefix < l) {
            len = l;
            par = leafpar[i];
        }
    }
    if (__ballot_sync(PS_FULL, len != 0) == 0) return;
    const K* K0 = bufs.k[0];
    const int32_t* V0 = bufs.v[0];
#pragma unroll 8
    for (uint32_t w = 0; w < 32; ++w) {  // window w -> row w
        const uint32_t bw = __shfl_sync(PS_FULL, b0, w), lw = __shfl_sync(PS_FULL, len, w);
        if (lane < lw) sk[w * RW + lane] = K0[bw + lane];
    }
    __syncwarp();
    K k[S];
    uint32_t o[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
        o[j] = (uint32_t)j;
        k[j] = (uint32_t)j < len ? sk[lane * RW + j] : key_pad<K>();
    }
    if (counters) {
        unsigned long long c_cmp = 0, c_mov = 0;
        // the window's natural run (runs.py:23-47): its pair compares plus the
        // failing one before the array end; a strictly descending one is reversed
        if (len && nprefix >= 2) {
            c_cmp += nprefix - 1 + ((uint64_t)b0 + nprefix < n ? 1 : 0);
            const uint64_t q = (uint64_t)b0 + 1;
            if (!((ty[q >> 5] >> (q & 31)) & 1u)) c_mov += nprefix;
        }
#pragma unroll
        for (int q = 1; q < S; ++q) {
            uint32_t sh = 0;
#pragma unroll
            for (int f = 0; f < q; ++f) sh += (uint32_t)(k[q] < k[f]);
            if ((uint32_t)q < len && (uint32_t)q >= nprefix) {
                c_cmp += sh + (sh < (uint32_t)q ? 1u : 0u);
                c_mov += sh ? sh + 1u : 0u;
            }
        }
        for (int dd = 16; dd; dd >>= 1) {
            c_cmp += __shfl_xor_sync(PS_FULL, c_cmp, dd);
            c_mov += __shfl_xor_sync(PS_FULL, c_mov, dd);
        }
        if (lane == 0) {
            if (c_cmp) atomicAdd(&counters->comparisons, c_cmp);
            if (c_mov) atomicAdd(&counters->moves, c_mov);
        }
    }
    net_sort<K, S>(k, o);
    constexpr PrunedNet<S> net{};
#pragma unroll
    for (int j = 0; j < S; ++j) {
        sk[lane * RW + j] = k[net.out[j]];
        so[lane * RW + j] = o[net.out[j]];
    }
    __syncwarp();
    if (!ARGSORT) {  // gather every payload before any store: parity-0 leaves are formed in place
#pragma unroll 8
        for (uint32_t w = 0; w < 32; ++w) {
            const uint32_t bw = __shfl_sync(PS_FULL, b0, w), lw = __shfl_sync(PS_FULL, len, w);
            if (lane < lw) so[w * RW + lane] = (uint32_t)V0[bw + so[w * RW + lane]];
        }
        __syncwarp();
    }
#pragma unroll 8
    for (uint32_t w = 0; w < 32; ++w) {
        const uint32_t bw = __shfl_sync(PS_FULL, b0, w), lw = __shfl_sync(PS_FULL, len, w);
        const uint32_t pw = __shfl_sync(PS_FULL, par, w);
        if (lane < lw) {
            const uint32_t ov = so[w * RW + lane];
            bufs.kb(pw)[bw + lane] = sk[w * RW + lane];
            bufs.vb(pw)[bw + lane] = ARGSORT ? (int32_t)(bw + ov) : (int32_t)ov;
        }
    }
}

// four consecutive keys: one (4-byte keys) or two (8-byte) 16-byte accesses
template <class K>
struct alignas(16) K4 {
    K e[4];
};

// Largest j in [0, r) with b[j] <= x (b ascending, b[0] = 0 <= x), by a warp
// (33-ary search: one probe per lane and round; all lanes return j).
PS_DEV uint32_t warp_last_le(const uint32_t* __restrict__ b, uint32_t r, uint32_t x) {
    const uint32_t lane = lane_id();
    uint32_t lo = 0, hi = r;  // b[lo] <= x, answer in [lo, hi)
    while (hi - lo > 32) {
        const uint32_t span = hi - lo;
        const uint32_t probe = lo + (uint32_t)(((uint64_t)span * (lane + 1)) / 33);
        const uint32_t c = __popc(__ballot_sync(PS_FULL, b[probe] <= x));
        // probes 0..c-1 satisfy b <= x
        const uint32_t nlo = c ? lo + (uint32_t)(((uint64_t)span * c) / 33) : lo;
        const uint32_t nhi = c < 32 ? lo + (uint32_t)(((uint64_t)span * (c + 1)) / 33) : hi;
        lo = nlo;
        hi = nhi;
    }
    const uint32_t idx = lo + lane;
    const bool p = idx < hi && b[idx] <= x;
    return lo + __popc(__ballot_sync(PS_FULL, p)) - 1;
}

template <class K, bool ARGSORT>
__global__ void __launch_bounds__(FORM_THREADS, 3) form_leaves_kernel(Bufs<K> bufs, uint64_t n,
                                                                   const uint32_t* __restrict__ b,
                                                                   const uint32_t* __restrict__ nat,
                                                                   const uint8_t* __restrict__ leafpar, uint32_t r,
                                                                   const uint32_t* __restrict__ ty, uint32_t m,
                                                                   const uint32_t* __restrict__ tile_first,
                                                                   Summary* __restrict__ counters) {
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t* sb = reinterpret_cast<uint32_t*>(smem);
    uint32_t* snat = sb + (FORM_TILE + 2);
    uint8_t* spar = reinterpret_cast<uint8_t*>(snat + (FORM_TILE + 1));
    uint32_t* wlist = reinterpret_cast<uint32_t*>(spar + ((FORM_TILE + 1) + 15) / 16 * 16);
    uint32_t* woff = wlist + (FORM_TILE + 1);
    size_t off = (reinterpret_cast<uint8_t*>(woff + (FORM_TILE + 2)) - smem + 15) / 16 * 16;
    const uint32_t cap = FORM_TILE + (m < MAX_FORM_M ? m : MAX_FORM_M);
    K* wk = reinterpret_cast<K*>(smem + off);
    int32_t* wv = reinterpret_cast<int32_t*>(wk + cap);
    uint16_t* widx = reinterpret_cast<uint16_t*>(wv + cap);
    __shared__ uint32_t s_first, s_cnt, s_nwin, s_wtot;
    __shared__ uint32_t sw32[32];

    K* const K0 = bufs.k[0];
    int32_t* const V0 = bufs.v[0];
    const uint32_t tid = threadIdx.x;
    // leaves covering positions lo_pos and hi_pos - 1 (tiles [tb, te) of run detection)
    auto locate = [&](uint32_t tb, uint32_t te, uint64_t lo_pos, uint64_t hi_pos) {
        __syncthreads();  // the previous tile's shared arrays are consumed
        if (tile_first) {
            if (tid == 0) {
                const uint32_t lo = tile_first[tb];
                uint32_t lo2 = r - 1;
                if (hi_pos < n) {
                    const uint32_t nx = tile_first[te];  // covers hi_pos
                    lo2 = b[nx] == hi_pos ? nx - 1 : nx;
                }
                s_first = lo;
                s_cnt = lo2 - lo + 1;
            }
        } else if (tid < 32) {
            // last leaf with b <= lo_pos and last leaf with b <= hi_pos-1: 32-ary warp searches
            const uint32_t lo = warp_last_le(b, r, (uint32_t)lo_pos);
            const uint32_t lo2 = warp_last_le(b, r, (uint32_t)(hi_pos - 1));
            if (tid == 0) {
                s_first = lo;
                s_cnt = lo2 - lo + 1;
            }
        }
        __syncthreads();
    };
    // A CTA covers FORM_TPC detection tiles.  When few (long) leaves cover the
    // whole span and windows are left to form_windows_kernel, it is formed in
    // one pass; otherwise tile by tile (the shared arrays hold one tile).
    const bool net = net_windows(m);
    const uint32_t ntiles = (uint32_t)((n + FORM_TILE - 1) / FORM_TILE);
    const uint32_t tb = blockIdx.x * FORM_TPC, te = min(tb + FORM_TPC, ntiles);
    const uint64_t span0 = (uint64_t)tb * FORM_TILE, span1 = min((uint64_t)te * FORM_TILE, n);
    locate(tb, te, span0, span1);
    const bool whole = net && s_cnt <= 16;
    if (net && !whole) {
        // spans made only of extended windows (form_windows_kernel's, which also
        // counts their detection compares) have nothing to do
        bool anynat = false;
        for (uint32_t i = tid; i < s_cnt; i += FORM_THREADS) {
            const uint32_t j = s_first + i;
            anynat |= nat[j] >= b[j + 1] - b[j];
        }
        if (!__syncthreads_or(anynat)) return;
    }
    for (uint32_t tl = tb; tl < te; ++tl) {
    const uint64_t t0 = whole ? span0 : (uint64_t)tl * FORM_TILE;
    const uint64_t t1 = whole ? span1 : min(t0 + FORM_TILE, n);
    if (!whole && te - tb > 1) locate(tl, tl + 1, t0, t1);
    [&]() {
    const uint32_t first = s_first, cnt = s_cnt;
    for (uint32_t i = tid; i <= cnt; i += FORM_THREADS) sb[i] = b[first + i];
    for (uint32_t i = tid; i < cnt; i += FORM_THREADS) {
        snat[i] = nat[first + i];
        spar[i] = leafpar[first + i];
    }
    __syncthreads();

    // ---- CountingOrder counters (statskit.py:49-72), when requested ---------
    // detection of every leaf starting in this tile (runs.py:23-47): the natural
    // run's pair compares plus the failing one before the array end; a reversal
    // moves its natural length.  Extension compares / moves are per element below.
    unsigned long long c_cmp = 0, c_mov = 0;
    auto flush_counters = [&]() {  // all threads; warp sums, one atomic pair per warp
        if (!counters) return;
        for (int dd = 16; dd; dd >>= 1) {
            c_cmp += __shfl_xor_sync(PS_FULL, c_cmp, dd);
            c_mov += __shfl_xor_sync(PS_FULL, c_mov, dd);
        }
        if (lane_id() == 0) {
            if (c_cmp) atomicAdd(&counters->comparisons, c_cmp);
            if (c_mov) atomicAdd(&counters->moves, c_mov);
        }
    };
    if (counters) {
        for (uint32_t i = tid; i < cnt; i += FORM_THREADS) {
            const uint64_t bj = sb[i];
            if (bj < t0) continue;  // counted by the tile it starts in
            const uint32_t nj = snat[i];
            if (net && nj < sb[i + 1] - bj) continue;  // an extended window: form_windows_kernel counts it
            if (nj >= 2) {
                c_cmp += nj - 1 + (bj + nj < n ? 1 : 0);
                const uint64_t q = bj + 1;
                if (!((ty[q >> 5] >> (q & 31)) & 1u)) c_mov += nj;  // strictly descending: reversed
            }
        }
    }

    // ---- natural leaves: copy / mirrored swap ------------------------------
    // Positions are handled FORM_BATCH at a time per thread: all loads of a
    // batch are issued before its stores (memory-level parallelism).  Every
    // address a thread reads is written only by that thread (a mirrored pair
    // belongs to the owner of its lower position), so the reordering is safe.
    constexpr uint32_t FORM_BATCH = 4;
    enum : uint8_t { F_NONE = 0, F_COPY = 1, F_ARGV = 2, F_SWAP = 3 };
    bool anynat = false;  // tiles made only of extended windows skip this pass
    for (uint32_t i = tid; i < cnt; i += FORM_THREADS) anynat |= !(snat[i] < sb[i + 1] - sb[i]);
    if (!__syncthreads_or(anynat)) {
    } else if (cnt <= 16) {
        // few (long) leaves: leaf by leaf, all threads striding over its positions
        for (uint32_t li = 0; li < cnt; ++li) {
            const uint64_t bj = sb[li], ej = sb[li + 1];
            const uint32_t len = (uint32_t)(ej - bj);
            if (snat[li] < len) continue;  // extended window, below
            const uint32_t par = spar[li];
            bool desc = false;
            if (len >= 2) {
                const uint64_t q = bj + 1;
                desc = !((ty[q >> 5] >> (q & 31)) & 1u);
            }
            K* dk = bufs.kb(par);
            int32_t* dv = bufs.vb(par);
            const uint64_t lo = bj > t0 ? bj : t0, hi = ej < t1 ? ej : t1;
            if (!desc) {
                if (!par && !ARGSORT) continue;  // in place already
                // 4-element groups with 16-byte accesses (the arrays are 16-byte
                // aligned), FORM_BATCH groups in flight per thread; the unaligned
                // edges element by element below
                const uint64_t lo4 = (lo + 3) & ~3ull, hi4 = hi & ~3ull;
                const uint64_t a0 = lo4 < hi ? lo4 : hi, a1 = hi4 > a0 ? hi4 : a0;
                for (uint64_t g0 = a0 / 4 + tid; g0 < a1 / 4; g0 += FORM_THREADS * FORM_BATCH) {
                    K4<K> kq[FORM_BATCH];
                    uint4 vq[FORM_BATCH];
#pragma unroll
                    for (uint32_t u = 0; u < FORM_BATCH; ++u) {
                        const uint64_t g = g0 + (uint64_t)u * FORM_THREADS;
                        if (g < a1 / 4) {
                            if (par) kq[u] = reinterpret_cast<const K4<K>*>(K0)[g];
                            if (!ARGSORT) vq[u] = reinterpret_cast<const uint4*>(V0)[g];
                        }
                    }
#pragma unroll
                    for (uint32_t u = 0; u < FORM_BATCH; ++u) {
                        const uint64_t g = g0 + (uint64_t)u * FORM_THREADS;
                        if (g < a1 / 4) {
                            if (par) reinterpret_cast<K4<K>*>(dk)[g] = kq[u];
                            const uint32_t q = (uint32_t)(4 * g);
                            reinterpret_cast<uint4*>(dv)[g] = ARGSORT ? make_uint4(q, q + 1, q + 2, q + 3) : vq[u];
                        }
                    }
                }
                for (uint64_t p = tid; p < (a0 - lo) + (hi - a1); p += FORM_THREADS) {
                    const uint64_t q = p < a0 - lo ? lo + p : a1 + (p - (a0 - lo));
                    if (par) dk[q] = K0[q];
                    dv[q] = ARGSORT ? (int32_t)q : V0[q];
                }
            } else {
                // mirrored pairs (p, s - p) belong to the owner of p <= s - p
                const uint64_t sm = bj + ej - 1;
                const uint64_t hi2 = hi < sm / 2 + 1 ? hi : sm / 2 + 1;
                for (uint64_t p0 = lo + tid; p0 < hi2; p0 += FORM_THREADS * FORM_BATCH) {
                    K ka[FORM_BATCH], kb[FORM_BATCH];
                    int32_t va[FORM_BATCH], vb[FORM_BATCH];
#pragma unroll
                    for (uint32_t u = 0; u < FORM_BATCH; ++u) {
                        const uint64_t p = p0 + (uint64_t)u * FORM_THREADS;
                        if (p < hi2) {
                            const uint64_t mr = sm - p;
                            ka[u] = K0[p];
                            kb[u] = K0[mr];
                            va[u] = ARGSORT ? (int32_t)p : V0[p];
                            vb[u] = ARGSORT ? (int32_t)mr : V0[mr];
                        }
                    }
#pragma unroll
                    for (uint32_t u = 0; u < FORM_BATCH; ++u) {
                        const uint64_t p = p0 + (uint64_t)u * FORM_THREADS;
                        if (p < hi2) {
                            const uint64_t mr = sm - p;
                            if (p < mr) {
                                dk[p] = kb[u];
                                dv[p] = vb[u];
                                dk[mr] = ka[u];
                                dv[mr] = va[u];
                            } else if (par || ARGSORT) {  // the center of an odd-length run
                                dk[p] = ka[u];
                                dv[p] = va[u];
                            }
                        }
                    }
                }
            }
        }
    } else
    for (uint64_t pos0 = t0 + tid; pos0 < t1; pos0 += FORM_THREADS * FORM_BATCH) {
        uint8_t act[FORM_BATCH];
        uint8_t parb[FORM_BATCH];
        uint64_t mir[FORM_BATCH];
        K ka[FORM_BATCH], kb[FORM_BATCH];
        int32_t va[FORM_BATCH], vb[FORM_BATCH];
#pragma unroll
        for (uint32_t u = 0; u < FORM_BATCH; ++u) {
            const uint64_t pos = pos0 + (uint64_t)u * FORM_THREADS;
            act[u] = F_NONE;
            parb[u] = 0;
            mir[u] = pos;
            if (pos >= t1) continue;
            uint32_t lo = 0, hi = cnt;  // sb[lo] <= pos < sb[hi]
            while (hi - lo > 1) {
                uint32_t mid = (lo + hi) >> 1;
                if (sb[mid] <= pos) lo = mid; else hi = mid;
            }
            const uint64_t bj = sb[lo], ej = sb[lo + 1];
            const uint32_t len = (uint32_t)(ej - bj);
            if (snat[lo] < len) continue;  // extended window, below
            const uint32_t par = spar[lo];
            parb[u] = (uint8_t)par;
            bool desc = false;
            if (len >= 2) {
                const uint64_t q = bj + 1;
                desc = !((ty[q >> 5] >> (q & 31)) & 1u);
            }
            const uint64_t mirror = desc ? bj + ej - 1 - pos : pos;
            mir[u] = mirror;
            if (pos < mirror) {
                act[u] = F_SWAP;
                ka[u] = K0[pos];
                kb[u] = K0[mirror];
                va[u] = ARGSORT ? (int32_t)pos : V0[pos];
                vb[u] = ARGSORT ? (int32_t)mirror : V0[mirror];
            } else if (pos == mirror) {
                if (par) {
                    act[u] = F_COPY;
                    ka[u] = K0[pos];
                    va[u] = ARGSORT ? (int32_t)pos : V0[pos];
                } else if (ARGSORT) {
                    act[u] = F_ARGV;
                }
            }
        }
#pragma unroll
        for (uint32_t u = 0; u < FORM_BATCH; ++u) {
            const uint64_t pos = pos0 + (uint64_t)u * FORM_THREADS;
            K* dk = bufs.kb(parb[u]);
            int32_t* dv = bufs.vb(parb[u]);
            if (act[u] == F_SWAP) {
                dk[pos] = kb[u];
                dv[pos] = vb[u];
                dk[mir[u]] = ka[u];
                dv[mir[u]] = va[u];
            } else if (act[u] == F_COPY) {
                dk[pos] = ka[u];
                dv[pos] = va[u];
            } else if (act[u] == F_ARGV) {
                V0[pos] = (int32_t)pos;
            }
        }
    }

    // ---- extended windows starting in this tile: stable rank ---------------
    if (net_windows(m)) {  // form_windows_kernel sorts them
        flush_counters();
        return;
    }
    bool anywin = false;
    // (windows longer than MAX_FORM_M are sorted by form_big_windows_kernel)
    for (uint32_t i = tid; i < cnt; i += FORM_THREADS) {
        const uint32_t len = sb[i + 1] - sb[i];
        anywin |= (snat[i] < len) && (len <= MAX_FORM_M) && (sb[i] >= t0);
    }
    if (!__syncthreads_or(anywin)) {
        flush_counters();
        return;
    }
    // compact the window leaf ids (block scan of flags, several rounds)
    uint32_t nwin = 0;
    for (uint32_t base = 0; base < cnt; base += FORM_THREADS) {
        const uint32_t i = base + tid;
        uint32_t flag = 0;
        if (i < cnt) {
            const uint32_t len = sb[i + 1] - sb[i];
            flag = (snat[i] < len) && (len <= MAX_FORM_M) && (sb[i] >= t0);
        }
        uint32_t tot;
        const uint32_t ex = block_exclusive<uint32_t, OpSum<uint32_t>>(flag, tot, sw32);
        if (flag) wlist[nwin + ex] = i;
        nwin += tot;
    }
    if (nwin == 0) {
        flush_counters();
        return;
    }
    // element offsets of the windows
    uint32_t wtot = 0;
    for (uint32_t base = 0; base < nwin; base += FORM_THREADS) {
        const uint32_t i = base + tid;
        uint32_t len = 0;
        if (i < nwin) len = sb[wlist[i] + 1] - sb[wlist[i]];
        uint32_t tot;
        const uint32_t ex = block_exclusive<uint32_t, OpSum<uint32_t>>(len, tot, sw32);
        if (i < nwin) woff[i] = wtot + ex;
        wtot += tot;
    }
    if (tid == 0) woff[nwin] = wtot;
    __syncthreads();
    // window index of every staged element (a thread per window)
    for (uint32_t i = tid; i < nwin; i += FORM_THREADS)
        for (uint32_t e = woff[i]; e < woff[i + 1]; ++e) widx[e] = (uint16_t)i;
    __syncthreads();
    // stage
    for (uint32_t e0 = tid; e0 < wtot; e0 += FORM_THREADS * 4) {
        K kk[4];
        int32_t vv[4];
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
            const uint32_t e = e0 + u * FORM_THREADS;
            if (e >= wtot) continue;
            const uint32_t lo = widx[e];
            const uint64_t p = (uint64_t)sb[wlist[lo]] + (e - woff[lo]);
            kk[u] = K0[p];
            vv[u] = ARGSORT ? (int32_t)p : V0[p];
        }
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
            const uint32_t e = e0 + u * FORM_THREADS;
            if (e < wtot) {
                wk[e] = kk[u];
                wv[e] = vv[u];
            }
        }
    }
    __syncthreads();
    for (uint32_t e = tid; e < wtot; e += FORM_THREADS) {
        const uint32_t lo = widx[e];
        const uint32_t wb = woff[lo], we = woff[lo + 1];
        const K x = wk[e];
        // stable rank in the window: earlier elements <= x, later elements < x
        // (one loop over the whole window: the same trip count on every lane)
        uint32_t rank = 0, shifts = 0;
#pragma unroll 4
        for (uint32_t f = wb; f < we; ++f) {
            const K y = wk[f];
            rank += (uint32_t)(y < x) | ((uint32_t)(f < e) & (uint32_t)!(x < y));
            if (counters) shifts += (uint32_t)(f < e) & (uint32_t)(x < y);
        }
        const uint32_t leaf = wlist[lo];
        if (counters && e - wb >= snat[leaf]) {
            // insertion of element q past the sorted natural prefix (runs.py:50-68):
            // it shifts the earlier elements > x, compares each of them plus the
            // first <= x if there is one, and moves shifts + 1 when it shifts
            const uint32_t q = e - wb;
            c_cmp += shifts + (shifts < q ? 1u : 0u);
            c_mov += shifts ? shifts + 1u : 0u;
        }
        const uint32_t par = spar[leaf];
        const uint64_t dst = (uint64_t)sb[leaf] + rank;
        bufs.kb(par)[dst] = x;
        bufs.vb(par)[dst] = wv[e];
    }
    flush_counters();
    }();
    if (whole) break;
    }
}

// ---------------------------------------------------------------------------
// Extended windows longer than MAX_FORM_M (min_run_len > 1024): each is the
// stable sort of its original records, done by one CTA: chunks of
// BIGW_CHUNK records are sorted in shared memory (4-record insertion sorts,
// then merge passes), then merge passes over global memory ping-pong between
// the window's ranges of the two buffers, ending in the leaf's parity buffer.
constexpr uint32_t BIGW_THREADS = 512;
constexpr uint32_t BIGW_CHUNK = 2048;  // = BIGW_THREADS * 4
constexpr uint32_t BIGW_CTAS = 2 * 148;

template <class K>
size_t big_window_smem_bytes() {
    return 2 * (size_t)BIGW_CHUNK * (sizeof(K) + 4);
}

// one stable merge pass: sorted runs of width w -> 2w over [0, len), VT
// consecutive outputs per thread (VT divides 2w, so a thread stays in its pair)
template <class K, uint32_t VT>
PS_DEV void bigw_merge_pass(const K* sk, const int32_t* sv, K* dk, int32_t* dv, uint32_t len, uint32_t w) {
    for (uint32_t o0 = threadIdx.x * VT; o0 < len; o0 += blockDim.x * VT) {
        const uint32_t a0 = o0 / (2 * w) * (2 * w);
        const uint32_t a1 = min(a0 + w, len), b1 = min(a0 + 2 * w, len);
        const uint32_t la = a1 - a0, lb = b1 - a1, d = o0 - a0;
        uint32_t lo = d > lb ? d - lb : 0, hi = min(d, la);  // # of A records among the first d outputs
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            const bool le = !(sk[a1 + d - 1 - mid] < sk[a0 + mid]);
            lo = le ? mid + 1 : lo;
            hi = le ? hi : mid;
        }
        uint32_t i = lo, j = d - lo;
        for (uint32_t t = 0; t < VT && o0 + t < b1; ++t) {
            const bool takeA = i < la && (j >= lb || !(sk[a1 + j] < sk[a0 + i]));
            const uint32_t src = takeA ? a0 + i : a1 + j;
            dk[o0 + t] = sk[src];
            dv[o0 + t] = sv[src];
            i += takeA;
            j += !takeA;
        }
    }
}

template <class K, bool ARGSORT>
__global__ void __launch_bounds__(BIGW_THREADS) form_big_windows_kernel(Bufs<K> bufs, const uint32_t* __restrict__ b,
                                                                        const uint32_t* __restrict__ nat,
                                                                        const uint8_t* __restrict__ leafpar,
                                                                        uint32_t r) {
    pdl_wait();
    extern __shared__ __align__(128) uint8_t smem[];
    K* sk[2];
    int32_t* sv[2];
    sk[0] = reinterpret_cast<K*>(smem);
    sk[1] = sk[0] + BIGW_CHUNK;
    sv[0] = reinterpret_cast<int32_t*>(sk[1] + BIGW_CHUNK);
    sv[1] = sv[0] + BIGW_CHUNK;
    const uint32_t tid = threadIdx.x;
    for (uint32_t leaf = blockIdx.x; leaf < r; leaf += gridDim.x) {
        const uint64_t base = b[leaf];
        const uint32_t len = b[leaf + 1] - (uint32_t)base;
        if (!(nat[leaf] < len && len > MAX_FORM_M)) continue;
        const uint32_t par = leafpar[leaf];
        uint32_t passes = 0;  // global merge passes after the chunk sorts
        for (uint64_t w = BIGW_CHUNK; w < len; w *= 2) ++passes;
        const uint32_t first = par ^ (passes & 1);  // so that the last pass lands in par
        K* K0 = bufs.k[0];
        int32_t* V0 = bufs.v[0];
        for (uint32_t c0 = 0; c0 < len; c0 += BIGW_CHUNK) {
            const uint32_t cl = min(BIGW_CHUNK, len - c0);
            // 4 consecutive records per thread, insertion-sorted (stable)
            K kk[4];
            int32_t vv[4];
            const uint32_t e0 = tid * 4;
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
                const uint32_t e = e0 + u;
                if (e < cl) {
                    const uint64_t p = base + c0 + e;
                    kk[u] = K0[p];
                    vv[u] = ARGSORT ? (int32_t)p : V0[p];
                }
            }
            const uint32_t mine = e0 < cl ? min(4u, cl - e0) : 0u;
            for (uint32_t u = 1; u < mine; ++u) {
                const K x = kk[u];
                const int32_t xv = vv[u];
                uint32_t q = u;
                while (q > 0 && x < kk[q - 1]) {
                    kk[q] = kk[q - 1];
                    vv[q] = vv[q - 1];
                    --q;
                }
                kk[q] = x;
                vv[q] = xv;
            }
            for (uint32_t u = 0; u < mine; ++u) {
                sk[0][e0 + u] = kk[u];
                sv[0][e0 + u] = vv[u];
            }
            __syncthreads();
            uint32_t cur = 0;
            for (uint32_t w = 4; w < cl; w *= 2) {
                bigw_merge_pass<K, 4>(sk[cur], sv[cur], sk[cur ^ 1], sv[cur ^ 1], cl, w);
                cur ^= 1;
                __syncthreads();
            }
            K* dk = bufs.kb(first) + base + c0;
            int32_t* dv = bufs.vb(first) + base + c0;
            for (uint32_t e = tid; e < cl; e += BIGW_THREADS) {
                dk[e] = sk[cur][e];
                dv[e] = sv[cur][e];
            }
            __syncthreads();
        }
        uint32_t src = first;
        for (uint64_t w = BIGW_CHUNK; w < len; w *= 2) {
            __syncthreads();  // the previous pass (or the chunk writes) is complete
            __threadfence_block();
            bigw_merge_pass<K, 8>(bufs.kb(src) + base, bufs.vb(src) + base, bufs.kb(src ^ 1) + base,
                                  bufs.vb(src ^ 1) + base, len, (uint32_t)w);
            src ^= 1;
        }
        __syncthreads();
    }
}

}  // namespace ps

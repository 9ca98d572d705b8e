// ps_runs.cuh -- N1 pass 1: parallel run detection.
//
// The reference detects runs left to right (policy.py:241-248 next_run ->
// runs.py:23-47 find_first_run, runs.py:71-82 extend_run): from position p
// the natural run ends at E(p) (maximal weakly increasing or strictly
// decreasing stretch starting with pair (p, p+1)) and the next run starts at
//     next(p) = max(E(p), min(n, p + m)),   m = min_run_len.
// This chain is inherently sequential; we make it parallel with SURVEY F6:
//   * pair types t(q) = [a[q-1] <= a[q]] are packed into bit words (RD1), and
//     E(p) = first "type change" position > p+1 (or n).
//   * For a tile starting at t, the first chain node >= t lies in the
//     candidate set C(t) = {t, ..., t+m-1} U {F(t)}, F(t) = first change > t.
//   * Each tile therefore has an (m+1)-entry transfer table
//     candidate -> (first chain node >= next tile start, #nodes in tile);
//     tables compose associatively (function composition with pass-through),
//     so the chain is a scan over tables (hierarchical, fan-out 32).
//   * Once every tile knows its entry node, one lane re-walks the tile and
//     emits the run boundaries b[] and natural lengths (policy.py:243,247).
#pragma once

#include "ps_common.cuh"

namespace ps {

// Bits j of the returned mask are set iff lo <= q0 + j < hi.
PS_DEV uint32_t range_mask(uint64_t q0, uint64_t lo, uint64_t hi) {
    if (q0 + 32 <= lo || q0 >= hi || lo >= hi) return 0u;
    uint32_t m = PS_FULL;
    if (q0 < lo) m &= PS_FULL << (uint32_t)(lo - q0);
    if (q0 + 32 > hi) m &= PS_FULL >> (uint32_t)(q0 + 32 - hi);
    return m;
}

// ---------------------------------------------------------------------------
// RD1: type bits t(q) for q in the group, plus c_g = first change position in
// (G, G+GROUP] (2 <= q <= n-1), INF if none.  One CTA per group; each warp
// streams 1024 keys per round with coalesced loads, ballots give the words.
template <class K>
__global__ void __launch_bounds__(RD_THREADS) rd_types_kernel(const K* __restrict__ a, uint64_t n,
                                                       uint32_t* __restrict__ ty, uint32_t* __restrict__ cg) {
    pdl_wait();
    __shared__ uint32_t sw[GROUP_WORDS];
    __shared__ uint32_t smin[TILES_PER_GROUP];
    const uint32_t g = blockIdx.x;
    const uint64_t G = (uint64_t)g * GROUP;
    const uint32_t lane = lane_id(), warp = warp_id();
    // each lane loads 16 bytes (EPL keys) per step: a warp step covers KPI keys
    // = EPL type words, gathered from 32 / EPL lanes each (the keys are 16-byte
    // aligned, ps_sort checks it)
    constexpr uint32_t EPL = 16 / sizeof(K), KPI = 32 * EPL, LPW = 32 / EPL;
    static_assert(TILE % KPI == 0, "a warp's tile is whole steps");
    const uint64_t p0 = G + (uint64_t)warp * TILE;
    K carry = (p0 >= 1 && p0 - 1 < n) ? a[p0 - 1] : K(0);
#pragma unroll 4
    for (uint32_t it = 0; it < TILE / KPI; ++it) {
        const uint64_t q0 = p0 + (uint64_t)it * KPI + lane * EPL;
        K x[EPL];
        if (q0 + EPL <= n) {
            const uint4 v = *reinterpret_cast<const uint4*>(a + q0);
            memcpy(x, &v, 16);
        } else {
#pragma unroll
            for (uint32_t e = 0; e < EPL; ++e) x[e] = q0 + e < n ? a[q0 + e] : K(0);
        }
        K prev = shfl_up(x[EPL - 1], 1);
        if (lane == 0) prev = carry;
        uint32_t nib = 0;
#pragma unroll
        for (uint32_t e = 0; e < EPL; ++e) {
            const uint64_t q = q0 + e;
            const bool bit = q >= 1 && q < n && key_le(e == 0 ? prev : x[e - 1], x[e]);
            nib |= (uint32_t)bit << e;
        }
        carry = shfl(x[EPL - 1], 31);
        uint32_t wv = nib << (EPL * (lane % LPW));
#pragma unroll
        for (uint32_t d = 1; d < LPW; d <<= 1) wv |= __shfl_xor_sync(PS_FULL, wv, d);
        if (lane % LPW == 0) sw[warp * (TILE / 32) + it * EPL + lane / LPW] = wv;
    }
    __syncthreads();
    uint32_t best = INF32;
    const uint64_t Gend = G + GROUP;
    for (uint32_t w = threadIdx.x; w < GROUP_WORDS; w += blockDim.x) {
        uint32_t cur = sw[w];
        ty[(uint64_t)g * GROUP_WORDS + w] = cur;
        uint32_t prevbit = w ? (sw[w - 1] >> 31) : 0u;
        uint32_t chg = cur ^ ((cur << 1) | prevbit);
        if (w == 0) chg &= ~1u;  // q = G is not in (G, Gend]
        const uint64_t q0 = G + 32ull * w;
        chg &= range_mask(q0, 2, n);
        if (chg) best = min(best, (uint32_t)(q0 + __ffs(chg) - 1));
    }
    if (threadIdx.x == 0 && Gend >= 2 && Gend < n) {
        // q = Gend: t(Gend) ^ t(Gend - 1)
        uint32_t tend = key_le(a[Gend - 1], a[Gend]) ? 1u : 0u;
        uint32_t tprev = sw[GROUP_WORDS - 1] >> 31;
        if (tend != tprev) best = min(best, (uint32_t)Gend);
    }
    for (int d = 16; d; d >>= 1) best = min(best, __shfl_xor_sync(PS_FULL, best, d));
    if (lane == 0) smin[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = INF32;
        for (uint32_t i = 0; i < TILES_PER_GROUP; ++i) m = min(m, smin[i]);
        cg[g] = m;
    }
}

// ---------------------------------------------------------------------------
// Per-CTA view of one group's change bits, with O(1) "next change" lookup.
struct ChainView {
    const uint32_t* chg;  // GROUP_WORDS + 1 words; bit j of word w = change at G + 32w + j
    const uint16_t* nzn;  // nzn[w] = first w' >= w with chg[w'] != 0, else 0xFFFF (size GROUP_WORDS+2)
    uint64_t G, Gend, n;
    uint64_t Fnext;  // first change > Gend (or n)
    uint64_t m;

    // First change position >= y (y >= G + 1), or n.
    PS_DEV uint64_t next_change_ge(uint64_t y) const {
        if (y > Gend) return Fnext;
        const uint32_t off = (uint32_t)(y - G);
        const uint32_t w = off >> 5;
        const uint32_t bits = chg[w] & (PS_FULL << (off & 31));
        if (bits) return G + 32ull * w + (__ffs(bits) - 1);
        const uint32_t w2 = nzn[w + 1];
        if (w2 != 0xFFFFu) return G + 32ull * w2 + (__ffs(chg[w2]) - 1);
        return Fnext;
    }
    // E(p): end of the natural run starting at p (runs.py:23-47).
    PS_DEV uint64_t E(uint64_t p) const {
        const uint64_t q = p + 1;
        if (q >= n) return n;
        uint64_t c = next_change_ge(q + 1);
        return c < n ? c : n;
    }
    // next(p) = max(E(p), min(n, p+m))  (policy.py:241-248 with runs.py:71-82)
    PS_DEV uint64_t next(uint64_t p, uint64_t* e_out = nullptr) const {
        const uint64_t e = E(p);
        if (e_out) *e_out = e;
        uint64_t s = p + m;
        if (s > n) s = n;
        return e > s ? e : s;
    }
};

// Chain walk from x (absolute, in the group) while x < lim, in 32-bit offsets
// from G.  For 3 <= m <= 32 a step whose natural run is shorter than m costs
// one funnel shift of two change words (next = x + m, E = the first change);
// other steps go through ChainView::next.  visit(x, e) is called per node.
template <class F>
PS_DEV uint64_t chain_walk(const ChainView& cv, uint64_t x, uint64_t lim, F&& visit) {
    const uint64_t G = cv.G;
    const uint32_t m = (uint32_t)cv.m;
    const uint32_t n_o = (uint32_t)min(cv.n - G, (uint64_t)0xFFFFFFFFu);
    const uint32_t lim_o = (uint32_t)(lim - G);
    const bool fast = m >= 3 && m <= 32;
    const uint32_t mask = fast ? (1u << (m - 1)) - 1u : 0u;
    uint32_t xo = (uint32_t)(x - G);
    while (xo < lim_o) {
        const uint32_t off2 = xo + 2, w = off2 >> 5;
        const uint32_t win = __funnelshift_r(cv.chg[w], cv.chg[w + 1], off2 & 31) & mask;
        if (win && xo + 1 < n_o) {
            visit(G + xo, G + off2 + (uint32_t)(__ffs(win) - 1));
            xo = min(xo + m, n_o);
        } else {
            uint64_t e;
            const uint64_t nx = cv.next(G + xo, &e);
            visit(G + xo, e);
            if (nx - G >= (uint64_t)lim_o) return nx;
            xo = (uint32_t)(nx - G);
        }
    }
    return G + xo;
}

// Build chg / nzn in shared memory for group g (all threads of the CTA).
PS_DEV void build_chain_view(const uint32_t* __restrict__ ty, uint64_t n, uint32_t g, uint32_t ngroups,
                             const uint32_t* __restrict__ Fg, uint32_t* s_chg, uint16_t* s_nzn, ChainView& cv,
                             uint64_t m) {
    const uint64_t G = (uint64_t)g * GROUP;
    const uint64_t wg0 = (uint64_t)g * GROUP_WORDS;
    const uint64_t nwords_total = (uint64_t)ngroups * GROUP_WORDS;
    // chg words 0..GROUP_WORDS (inclusive; the last only for position Gend)
    for (uint32_t w = threadIdx.x; w <= GROUP_WORDS; w += blockDim.x) {
        const uint64_t gw = wg0 + w;
        uint32_t cur = gw < nwords_total ? ty[gw] : 0u;
        uint32_t prv = (gw >= 1 && gw - 1 < nwords_total) ? ty[gw - 1] : 0u;
        uint32_t chg = cur ^ ((cur << 1) | (prv >> 31));
        const uint64_t q0 = G + 32ull * w;
        uint64_t hi = n;
        if (w == GROUP_WORDS) hi = min(hi, q0 + 1);  // only position Gend
        chg &= range_mask(q0, 2, hi);
        if (w == 0) chg &= ~1u;
        s_chg[w] = chg;
    }
    if (threadIdx.x == 0) s_chg[GROUP_WORDS + 1] = 0;  // (chain_walk's window past the group)
    __syncthreads();
    // nzn: suffix "first nonzero word" -- each thread owns 2 words of 0..511,
    // word 512 handled by all (cheap), then a block suffix-min over threads.
    __shared__ uint32_t s_red[32];
    const uint32_t t = threadIdx.x;  // blockDim.x == GROUP_WORDS / 2
    static_assert(RD_THREADS * 2 == GROUP_WORDS, "two change words per thread");
    const uint32_t w0 = 2 * t, w1 = 2 * t + 1;
    const uint32_t NONE = 0xFFFFu;
    uint32_t v0 = s_chg[w0] ? w0 : NONE;
    uint32_t v1 = s_chg[w1] ? w1 : NONE;
    uint32_t vlast = s_chg[GROUP_WORDS] ? GROUP_WORDS : NONE;
    uint32_t loc = min(v0, v1);
    // exclusive suffix-min over threads t' > t
    const uint32_t lane = lane_id(), warp = warp_id();
    uint32_t x = loc;
    for (int d = 1; d < 32; d <<= 1) {
        uint32_t y = __shfl_down_sync(PS_FULL, x, d);
        if (lane + d < 32) x = min(x, y);
    }
    // x = inclusive suffix-min within warp from this lane
    if (lane == 0) s_red[warp] = x;
    __syncthreads();
    uint32_t after_warp = vlast;
    for (uint32_t ww = warp + 1; ww < TILES_PER_GROUP; ++ww) after_warp = min(after_warp, s_red[ww]);
    uint32_t excl = __shfl_down_sync(PS_FULL, x, 1);
    if (lane == 31) excl = NONE;
    excl = min(excl, after_warp);
    s_nzn[w1] = (uint16_t)min(v1, excl);
    s_nzn[w0] = (uint16_t)min(v0, min(v1, excl));
    if (t == 0) {
        s_nzn[GROUP_WORDS] = (uint16_t)vlast;
        s_nzn[GROUP_WORDS + 1] = (uint16_t)NONE;
    }
    __syncthreads();
    cv.chg = s_chg;
    cv.nzn = s_nzn;
    cv.G = G;
    cv.Gend = G + GROUP;
    cv.n = n;
    uint64_t fn = (g + 1 < ngroups) ? (uint64_t)Fg[g + 1] : (uint64_t)n;
    cv.Fnext = fn < n ? fn : n;
    cv.m = m;
}

// Candidate index of position x in the table of a span starting at t with
// F(t) = Ft:  x - t if < m, else the F(t) slot m.
PS_DEV void tab_apply(const uint64_t* tab, uint64_t t, uint64_t tnext, uint64_t Ft, uint64_t m, uint64_t n,
                      uint64_t& x, uint64_t& c, uint32_t* err) {
    if (x >= tnext || x >= n) return;  // pass-through
    const uint64_t d = x - t;
    uint32_t idx = d < m ? (uint32_t)d : (uint32_t)m;
    if (idx == m && x != Ft) atomicOr(err, ERR_CHAIN);
    const uint64_t v = tab[idx];
    x = unpack_x(v);
    c += unpack_c(v);
}

// ---------------------------------------------------------------------------
// RD2a: per-tile transfer tables (one warp per tile, lanes over the m+1
// candidates) and their composition into one table per group.
// Dynamic smem: TILES_PER_GROUP * (m+1) uint64.
__global__ void __launch_bounds__(RD_THREADS) rd_tables_kernel(const uint32_t* __restrict__ ty, uint64_t n, uint32_t m,
                                                        const uint32_t* __restrict__ Fg, uint32_t ngroups,
                                                        uint64_t* __restrict__ tile_tab, uint32_t* __restrict__ Ft,
                                                        uint64_t* __restrict__ group_tab, uint32_t* err) {
    pdl_wait();
    __shared__ uint32_t s_chg[GROUP_WORDS + 2];
    __shared__ uint16_t s_nzn[GROUP_WORDS + 2];
    __shared__ uint64_t s_Ft[TILES_PER_GROUP];
    extern __shared__ uint64_t s_tab[];  // [TILES_PER_GROUP][m+1]
    const uint32_t g = blockIdx.x;
    ChainView cv;
    build_chain_view(ty, n, g, ngroups, Fg, s_chg, s_nzn, cv, m);
    const uint32_t lane = lane_id(), w = warp_id();
    const uint32_t M1 = m + 1;
    const uint64_t t = cv.G + (uint64_t)w * TILE;
    const uint64_t tend = t + TILE;
    const uint64_t lim = tend < n ? tend : n;
    uint64_t F_t = cv.next_change_ge(t + 1);
    if (F_t > n) F_t = n;
    if (lane == 0) s_Ft[w] = F_t;
    for (uint32_t e = lane; e < M1; e += 32) {
        uint64_t x = e < m ? t + e : F_t;
        uint32_t cnt = 0;
        if (x < lim) x = chain_walk(cv, x, lim, [&](uint64_t, uint64_t) { cnt++; });
        s_tab[w * M1 + e] = pack_xc((uint32_t)x, (uint32_t)cnt);
    }
    __syncthreads();
    const uint64_t tile0 = (uint64_t)g * TILES_PER_GROUP;
    for (uint32_t i = threadIdx.x; i < TILES_PER_GROUP * M1; i += blockDim.x)
        tile_tab[tile0 * M1 + i] = s_tab[i];
    if (threadIdx.x < TILES_PER_GROUP) Ft[tile0 + threadIdx.x] = (uint32_t)s_Ft[threadIdx.x];
    if (w == 0) {
        for (uint32_t e = lane; e < M1; e += 32) {
            uint64_t x = e < m ? cv.G + e : s_Ft[0];
            uint64_t c = 0;
            for (uint32_t k = 0; k < TILES_PER_GROUP; ++k) {
                const uint64_t tk = cv.G + (uint64_t)k * TILE;
                tab_apply(s_tab + k * M1, tk, tk + TILE, s_Ft[k], m, n, x, c, err);
            }
            group_tab[(uint64_t)g * M1 + e] = pack_xc((uint32_t)x, (uint32_t)c);
        }
    }
}

// ---------------------------------------------------------------------------
// Chain scan over tables (hierarchical, fan-out TSCAN_FAN).  Level-L table j
// spans [j*span, (j+1)*span); F at its start is Ft[j*span/TILE].  Every kernel
// stages its tables and F values in shared memory first, so the serial walks
// below only pay shared-memory latency.
// Dynamic smem of compose/top/down: TSCAN_FAN*(m+1) uint64.
PS_DEV uint32_t stage_tables(const uint64_t* __restrict__ in, uint32_t j0, uint32_t cnt, uint32_t M1,
                             uint64_t span, const uint32_t* __restrict__ Ft, uint64_t* s_tab, uint64_t* s_F) {
    // batches of 8 independent loads per thread (a plain load->store loop would
    // wait one memory latency per element)
    const uint32_t tot = cnt * M1;
    const uint64_t* src = in + (uint64_t)j0 * M1;
    for (uint32_t base = 0; base < tot; base += 8 * blockDim.x) {
        uint64_t v[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = base + u * blockDim.x + threadIdx.x;
            v[u] = i < tot ? src[i] : 0;
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = base + u * blockDim.x + threadIdx.x;
            if (i < tot) s_tab[i] = v[u];
        }
    }
    for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) s_F[k] = Ft[((uint64_t)(j0 + k) * span) / TILE];
    return cnt;
}

// compose: one warp per output table.
__global__ void __launch_bounds__(32) rd_compose_kernel(const uint64_t* __restrict__ in, uint32_t P, uint64_t span,
                                                        const uint32_t* __restrict__ Ft, uint64_t n, uint32_t m,
                                                        uint64_t* __restrict__ out, uint32_t* err) {
    pdl_wait();
    extern __shared__ uint64_t s_tab[];
    __shared__ uint64_t s_F[TSCAN_FAN];
    const uint32_t o = blockIdx.x;
    const uint32_t j0 = o * TSCAN_FAN;
    const uint32_t cnt = min(TSCAN_FAN, P - j0);
    const uint32_t M1 = m + 1;
    stage_tables(in, j0, cnt, M1, span, Ft, s_tab, s_F);
    __syncwarp();
    const uint64_t t0 = (uint64_t)j0 * span;
    for (uint32_t e = threadIdx.x; e < M1; e += 32) {
        uint64_t x = e < m ? t0 + e : s_F[0];
        uint64_t c = 0;
        for (uint32_t k = 0; k < cnt; ++k) {
            const uint64_t tk = t0 + (uint64_t)k * span;
            tab_apply(s_tab + k * M1, tk, tk + span, s_F[k], m, n, x, c, err);
        }
        out[(uint64_t)o * M1 + e] = pack_xc((uint32_t)x, (uint32_t)c);
    }
}

// top: P <= TSCAN_FAN tables, entry (0, 0); writes each table's entry and the
// total run count r (b[r] = n).
__global__ void __launch_bounds__(32) rd_top_kernel(const uint64_t* __restrict__ in, uint32_t P, uint64_t span,
                                                    const uint32_t* __restrict__ Ft, uint64_t n, uint32_t m,
                                                    uint64_t* __restrict__ entries, uint32_t* __restrict__ b,
                                                    Summary* sum, uint32_t* err) {
    pdl_wait();
    extern __shared__ uint64_t s_tab[];
    __shared__ uint64_t s_F[TSCAN_FAN];
    const uint32_t M1 = m + 1;
    stage_tables(in, 0, P, M1, span, Ft, s_tab, s_F);
    __syncwarp();
    if (threadIdx.x != 0) return;
    uint64_t x = 0, c = 0;
    for (uint32_t j = 0; j < P; ++j) {
        entries[j] = pack_xc((uint32_t)x, (uint32_t)c);
        const uint64_t tj = (uint64_t)j * span;
        tab_apply(s_tab + j * M1, tj, tj + span, s_F[j], m, n, x, c, err);
    }
    if (x != n) atomicOr(err, ERR_CHAIN);
    sum->r = (uint32_t)c;
    b[c] = (uint32_t)n;
}

// down: given the entry of each level-(L+1) table, derive level-L entries.
__global__ void __launch_bounds__(32) rd_down_kernel(const uint64_t* __restrict__ in, uint32_t P, uint64_t span,
                                                     const uint32_t* __restrict__ Ft, uint64_t n, uint32_t m,
                                                     const uint64_t* __restrict__ up_entries,
                                                     uint64_t* __restrict__ entries, uint32_t* err) {
    pdl_wait();
    extern __shared__ uint64_t s_tab[];
    __shared__ uint64_t s_F[TSCAN_FAN];
    const uint32_t o = blockIdx.x;
    const uint32_t j0 = o * TSCAN_FAN;
    const uint32_t cnt = min(TSCAN_FAN, P - j0);
    const uint32_t M1 = m + 1;
    stage_tables(in, j0, cnt, M1, span, Ft, s_tab, s_F);
    __syncwarp();
    if (threadIdx.x != 0) return;
    const uint64_t v = up_entries[o];
    uint64_t x = unpack_x(v), c = unpack_c(v);
    for (uint32_t k = 0; k < cnt; ++k) {
        entries[j0 + k] = pack_xc((uint32_t)x, (uint32_t)c);
        const uint64_t tk = (uint64_t)(j0 + k) * span;
        tab_apply(s_tab + k * M1, tk, tk + span, s_F[k], m, n, x, c, err);
    }
}

// Two-level chain scan in one CTA (TSCAN_FAN < P <= TSCAN_FAN^2 group tables):
// warp w composes group tables [32w, 32w+32) into a level-1 table, thread 0
// walks the level-1 tables from (0, 0) (the top: run count, b[r] = n), then
// lane 0 of each warp walks its group tables from its level-1 entry and writes
// the group entries (the compose / top / down kernels' work, one launch).
// Dynamic smem: (nw + 1) * TSCAN_FAN * (m+1) uint64, nw = ceil(P / TSCAN_FAN).
__global__ void __launch_bounds__(1024) rd_chain2_kernel(const uint64_t* __restrict__ in, uint32_t P,
                                                         const uint32_t* __restrict__ Ft, uint64_t n, uint32_t m,
                                                         uint64_t* __restrict__ entries, uint32_t* __restrict__ b,
                                                         Summary* sum, uint32_t* err) {
    pdl_wait();
    extern __shared__ uint64_t sm[];
    __shared__ uint64_t s_F[TSCAN_FAN * TSCAN_FAN];
    __shared__ uint64_t s_up[TSCAN_FAN];
    const uint32_t M1 = m + 1, lane = lane_id(), w = warp_id(), nw = blockDim.x / 32;
    uint64_t* s_tab = sm + (uint64_t)w * TSCAN_FAN * M1;
    uint64_t* s_l1 = sm + (uint64_t)nw * TSCAN_FAN * M1;
    const uint32_t j0 = w * TSCAN_FAN;
    const uint32_t cnt = P > j0 ? min(TSCAN_FAN, P - j0) : 0u;
    const uint64_t* src = in + (uint64_t)j0 * M1;
    for (uint32_t base = 0; base < cnt * M1; base += 8 * 32) {  // 8 independent loads per lane
        uint64_t v[8];
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            v[u] = i < cnt * M1 ? src[i] : 0;
        }
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = base + u * 32 + lane;
            if (i < cnt * M1) s_tab[i] = v[u];
        }
    }
    for (uint32_t k = lane; k < cnt; k += 32) s_F[j0 + k] = Ft[((uint64_t)(j0 + k) * GROUP) / TILE];
    __syncwarp();
    const uint64_t t0 = (uint64_t)j0 * GROUP;
    if (cnt) {
        for (uint32_t e = lane; e < M1; e += 32) {
            uint64_t x = e < m ? t0 + e : s_F[j0];
            uint64_t c = 0;
            for (uint32_t k = 0; k < cnt; ++k) {
                const uint64_t tk = t0 + (uint64_t)k * GROUP;
                tab_apply(s_tab + k * M1, tk, tk + GROUP, s_F[j0 + k], m, n, x, c, err);
            }
            s_l1[w * M1 + e] = pack_xc((uint32_t)x, (uint32_t)c);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t P1 = (P + TSCAN_FAN - 1) / TSCAN_FAN;
        const uint64_t span1 = (uint64_t)GROUP * TSCAN_FAN;
        uint64_t x = 0, c = 0;
        for (uint32_t j = 0; j < P1; ++j) {
            s_up[j] = pack_xc((uint32_t)x, (uint32_t)c);
            const uint64_t tj = (uint64_t)j * span1;
            tab_apply(s_l1 + j * M1, tj, tj + span1, s_F[j * TSCAN_FAN], m, n, x, c, err);
        }
        if (x != n) atomicOr(err, ERR_CHAIN);
        sum->r = (uint32_t)c;
        b[c] = (uint32_t)n;
    }
    __syncthreads();
    if (lane == 0 && cnt) {
        const uint64_t v = s_up[w];
        uint64_t x = unpack_x(v), c = unpack_c(v);
        for (uint32_t k = 0; k < cnt; ++k) {
            entries[j0 + k] = pack_xc((uint32_t)x, (uint32_t)c);
            const uint64_t tk = t0 + (uint64_t)k * GROUP;
            tab_apply(s_tab + k * M1, tk, tk + GROUP, s_F[j0 + k], m, n, x, c, err);
        }
    }
}
inline size_t rd_chain2_smem(uint32_t P, uint32_t m) {
    const size_t nw = (P + TSCAN_FAN - 1) / TSCAN_FAN;
    return (nw + 1) * TSCAN_FAN * (size_t)(m + 1) * 8;
}

// ---------------------------------------------------------------------------
// RD2c: emit the run boundaries b[c] and natural lengths nat[c].
// Dynamic smem: TILES_PER_GROUP * (m+1) uint64 (the group's tile tables).
__global__ void __launch_bounds__(RD_THREADS) rd_emit_kernel(const uint32_t* __restrict__ ty, uint64_t n, uint32_t m,
                                                      const uint32_t* __restrict__ Fg, uint32_t ngroups,
                                                      const uint64_t* __restrict__ tile_tab,
                                                      const uint32_t* __restrict__ Ft,
                                                      const uint64_t* __restrict__ group_entries,
                                                      uint32_t* __restrict__ b, uint32_t* __restrict__ nat,
                                                      uint32_t* __restrict__ tile_first, uint32_t* err) {
    pdl_wait();
    __shared__ uint32_t s_chg[GROUP_WORDS + 2];
    __shared__ uint16_t s_nzn[GROUP_WORDS + 2];
    __shared__ uint64_t s_entry[TILES_PER_GROUP];
    __shared__ uint64_t s_F[TILES_PER_GROUP];
    extern __shared__ uint64_t s_tab[];  // [TILES_PER_GROUP][m+1]
    const uint32_t g = blockIdx.x;
    ChainView cv;
    build_chain_view(ty, n, g, ngroups, Fg, s_chg, s_nzn, cv, m);
    const uint32_t M1 = m + 1;
    const uint64_t tile0 = (uint64_t)g * TILES_PER_GROUP;
    for (uint32_t i = threadIdx.x; i < TILES_PER_GROUP * M1; i += blockDim.x) s_tab[i] = tile_tab[tile0 * M1 + i];  // <= 8 per thread
    if (threadIdx.x < TILES_PER_GROUP) s_F[threadIdx.x] = Ft[tile0 + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t v = group_entries[g];
        uint64_t x = unpack_x(v), c = unpack_c(v);
        for (uint32_t k = 0; k < TILES_PER_GROUP; ++k) {
            s_entry[k] = pack_xc((uint32_t)x, (uint32_t)c);
            const uint64_t tk = cv.G + (uint64_t)k * TILE;
            tab_apply(s_tab + k * M1, tk, tk + TILE, s_F[k], m, n, x, c, err);
        }
    }
    __syncthreads();
    // tile w is walked by lane w of warp 0 (one warp issues all eight walks)
    const uint32_t w = threadIdx.x;
    if (w >= TILES_PER_GROUP) return;
    const uint64_t t = cv.G + (uint64_t)w * TILE;
    const uint64_t lim = min(t + TILE, n);
    const uint64_t v = s_entry[w];
    uint64_t x = unpack_x(v);
    uint32_t c = unpack_c(v);
    // the run covering the tile's first position (leaf formation's tile = TILE)
    if (t < n) tile_first[tile0 + w] = (uint32_t)(x == t ? c : c - 1);
    if (x < lim)
        chain_walk(cv, x, lim, [&](uint64_t p, uint64_t e) {
            b[c] = (uint32_t)p;
            nat[c] = (uint32_t)(e - p);
            c++;
        });
}

// ---------------------------------------------------------------------------
// Serial chain walker for min_run_len > MAX_M_TILED (chain steps are >= m
// apart, so at most n/m steps); one warp scans change bits 1024 at a time.
__global__ void rd_serial_kernel(const uint32_t* __restrict__ ty, uint64_t n, uint64_t m,
                                 uint32_t* __restrict__ b, uint32_t* __restrict__ nat, Summary* sum) {
    pdl_wait();
    const uint32_t lane = lane_id();
    const uint64_t nwords = (n + 31) / 32;
    uint64_t p = 0, c = 0;
    while (p < n) {
        const uint64_t q = p + 1;
        uint64_t E = n;
        if (q < n) {
            const uint64_t y = q + 1;
            const uint64_t lo = y > 2 ? y : 2;
            for (uint64_t w0 = y / 32; w0 < nwords; w0 += 32) {
                const uint64_t w = w0 + lane;
                uint32_t chg = 0;
                if (w < nwords) {
                    const uint32_t tcur = ty[w];
                    const uint32_t tprv = w ? ty[w - 1] : 0u;
                    chg = (tcur ^ ((tcur << 1) | (tprv >> 31))) & range_mask(w * 32, lo, n);
                }
                const uint32_t bal = __ballot_sync(PS_FULL, chg != 0);
                if (bal) {
                    const int l = __ffs(bal) - 1;
                    const uint32_t cw = __shfl_sync(PS_FULL, chg, l);
                    E = (w0 + l) * 32 + (__ffs(cw) - 1);
                    break;
                }
            }
        }
        uint64_t s = p + m;
        if (s > n) s = n;
        const uint64_t nx = E > s ? E : s;
        if (lane == 0) {
            b[c] = (uint32_t)p;
            nat[c] = (uint32_t)(E - p);
        }
        c++;
        p = nx;
    }
    if (lane == 0) {
        b[c] = (uint32_t)n;
        sum->r = (uint32_t)c;
    }
}

}  // namespace ps

// ps_tree.cuh -- N2: boundary powers and the stack-free merge tree.
//
// The reference runs a stack over the run boundaries (policy.py:250-259,
// RunStack :94-129, _merge_one_group :132-143, _merge_down :146-175).  Its
// merge tree is a function of the boundary powers alone:
//   * boundary j (between runs j-1 and j), power P[j] (power.py:58-74,
//     computed exactly with a clz on 32-bit fixed-point midpoints, F4);
//   * R(j) = next boundary to the right with strictly smaller power; the
//     boundaries sharing (R, P) form one main-loop merge whose left end is
//     the previous boundary with strictly smaller power;
//   * boundaries with no R form the "spine" that _merge_down collapses.
// With sentinels P[0] = P[r] = 0 every query "nearest <= to the right/left"
// is answered by a 32-ary min tree over the uint8 powers.
#pragma once

#include "ps_common.cuh"
#include "ps_scan.cuh"

namespace ps {

// ---------------------------------------------------------------------------
// T1: powers.  P[j] for j in [0, padded): P[0] = P[r] = 0, j > r -> 0xFF.
PS_DEV void tree_power_one(uint32_t j, const uint32_t* __restrict__ b, uint32_t r, uint64_t n, uint32_t log2k,
                           uint8_t* __restrict__ P, uint32_t* err) {
    uint32_t v;
    if (j == 0 || j == r) {
        v = 0;
    } else if (j > r) {
        v = 0xFF;
    } else {
        // doubled midpoints A = b1+e1, B = b2+e2 of runs j-1 and j (power.py:67-68)
        const uint64_t A = (uint64_t)b[j - 1] + b[j];
        const uint64_t B = (uint64_t)b[j] + b[j + 1];
        // floor(A * 2^32 / 2n) < 2^32 since A < 2n
        const uint32_t x = (uint32_t)((A << 31) / n);
        const uint32_t y = (uint32_t)((B << 31) / n);
        const uint32_t d = __clz(x ^ y) + 1;  // first differing fraction bit
        v = (d + log2k - 1) / log2k;        // least p with d <= p*log2(k)
        if (v >= NPOW) {
            atomicOr(err, ERR_POWER);
            v = NPOW - 1;
        }
    }
    P[j] = (uint8_t)v;
}
// grid over nthreads >= max(padded, 32 * lev1_padded, r + 2): also zeroes the
// depth / stack-height difference arrays and writes min-tree level 1 (warp minima)
__global__ void tree_powers_kernel(const uint32_t* __restrict__ b, uint32_t r, uint64_t n, uint32_t log2k,
                                   uint8_t* __restrict__ P, uint32_t padded, uint32_t* err, int32_t* __restrict__ Dd,
                                   int32_t* __restrict__ Sd, uint8_t* __restrict__ lev1, uint32_t lev1_padded) {
    pdl_wait();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < r + 2) {
        Dd[j] = 0;
        Sd[j] = 0;
    }
    uint32_t v = 0xFF;
    if (j < padded) {
        tree_power_one(j, b, r, n, log2k, P, err);
        v = P[j];
    }
    if (lev1) {
        for (int d = 16; d; d >>= 1) v = min(v, __shfl_xor_sync(PS_FULL, v, d));
        if (lane_id() == 0 && j / 32 < lev1_padded) lev1[j / 32] = (uint8_t)v;
    }
}

// T2: one level of the 32-ary min tree (bytes).
PS_DEV void tree_minlevel_one(uint32_t i, const uint8_t* __restrict__ in, uint32_t in_groups,
                              uint8_t* __restrict__ out) {
    uint32_t v = 0xFF;
    if (i < in_groups) {
        const uint4* p = reinterpret_cast<const uint4*>(in + (uint64_t)i * 32);
        uint4 a = p[0], c = p[1];
        uint32_t m = __vminu4(__vminu4(__vminu4(a.x, a.y), __vminu4(a.z, a.w)),
                              __vminu4(__vminu4(c.x, c.y), __vminu4(c.z, c.w)));
        m = __vminu4(m, m >> 16);
        m = __vminu4(m, m >> 8);
        v = m & 0xFF;
    }
    out[i] = (uint8_t)v;
}
__global__ void tree_minlevel_kernel(const uint8_t* __restrict__ in, uint32_t in_groups, uint8_t* __restrict__ out,
                                     uint32_t out_padded) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < out_padded) tree_minlevel_one(i, in, in_groups, out);
}

struct MinTree {
    const uint8_t* lev[8];
    uint32_t nlev;
};

// bit i set iff arr[grp*32 + i] <= v
PS_DEV uint32_t group_le_mask(const uint8_t* arr, uint32_t grp, uint32_t v) {
    const uint4* p = reinterpret_cast<const uint4*>(arr + (uint64_t)grp * 32);
    const uint4 a = __ldg(p), c = __ldg(p + 1);
    const uint32_t vv = v * 0x01010101u;
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    uint32_t mask = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t cm = __vcmpleu4(w[i], vv);
        mask |= (((cm & 0x80808080u) * 0x00204081u) >> 28) << (4 * i);
    }
    return mask;
}

// first index > j with P <= v
PS_DEV uint32_t find_right_le(const MinTree& t, uint32_t j, uint32_t v) {
    uint32_t idx = j, L = 0, f;
    for (;;) {
        const uint32_t grp = idx >> 5, off = idx & 31;
        uint32_t mask = group_le_mask(t.lev[L], grp, v);
        mask &= off == 31 ? 0u : (PS_FULL << (off + 1));
        if (mask) {
            f = grp * 32 + (__ffs(mask) - 1);
            break;
        }
        if (L + 1 >= t.nlev) return INF32;
        idx = grp;
        L++;
    }
    while (L > 0) {
        L--;
        const uint32_t mask = group_le_mask(t.lev[L], f, v);
        f = f * 32 + (__ffs(mask) - 1);
    }
    return f;
}

// last index < j with P <= v
PS_DEV uint32_t find_left_le(const MinTree& t, uint32_t j, uint32_t v) {
    uint32_t idx = j, L = 0, f;
    for (;;) {
        const uint32_t grp = idx >> 5, off = idx & 31;
        uint32_t mask = group_le_mask(t.lev[L], grp, v);
        mask &= off == 0 ? 0u : (PS_FULL >> (32 - off));
        if (mask) {
            f = grp * 32 + (31 - __clz(mask));
            break;
        }
        if (L + 1 >= t.nlev) return INF32;
        idx = grp;
        L++;
    }
    while (L > 0) {
        L--;
        const uint32_t mask = group_le_mask(t.lev[L], f, v);
        f = f * 32 + (31 - __clz(mask));
    }
    return f;
}

// T3a: Rle[j] = first j' > j with P[j'] <= P[j]; Lle[j] = last j' < j with P[j'] <= P[j].
__global__ void tree_nearest_kernel(MinTree t, const uint8_t* __restrict__ P, uint32_t r, uint32_t* __restrict__ Rle,
                                    uint32_t* __restrict__ Lle) {
    pdl_wait();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (j >= r) return;
    const uint32_t v = P[j];
    Rle[j] = find_right_le(t, j, v);
    Lle[j] = find_left_le(t, j, v);
}

// Classification of boundary j (1 <= j <= r-1).
struct BoundaryClass {
    bool head;        // rightmost member of a main-loop merge node
    bool spine;       // never popped by the main loop
    uint32_t rstrict; // R(j) (strictly smaller to the right) or INF32
    uint32_t nmem;    // head only: members
    uint32_t bidx[5]; // head only: begin, members..., end (boundary indices)
};

PS_DEV BoundaryClass classify(uint32_t j, const uint8_t* __restrict__ P, const uint32_t* __restrict__ Rle,
                              const uint32_t* __restrict__ Lle, uint32_t r, uint32_t k, uint32_t* err) {
    BoundaryClass c;
    const uint32_t v = P[j];
    const uint32_t rr = Rle[j];
    c.head = rr < r && P[rr] < v;
    c.spine = false;
    c.rstrict = INF32;
    c.nmem = 0;
    if (c.head) {
        c.rstrict = rr;
        uint32_t mem[4];
        uint32_t cnt = 0;
        mem[cnt++] = j;
        uint32_t ll = Lle[j];
        while (ll >= 1 && P[ll] == v) {
            if (cnt >= k - 1) {
                atomicOr(err, ERR_GROUP);
                break;
            }
            mem[cnt++] = ll;
            ll = Lle[ll];
        }
        c.nmem = cnt;
        c.bidx[0] = ll;
        for (uint32_t i = 0; i < cnt; ++i) c.bidx[1 + i] = mem[cnt - 1 - i];
        c.bidx[1 + cnt] = rr;
    } else {
        // follow the equal-power chain to the right (<= k-2 steps)
        uint32_t x = j;
        uint32_t steps = 0;
        while (Rle[x] < r && P[Rle[x]] == v) {
            x = Rle[x];
            if (++steps > 8) {
                atomicOr(err, ERR_GROUP);
                break;
            }
        }
        if (Rle[x] >= r) {
            c.spine = true;
        } else {
            c.rstrict = Rle[x];
        }
    }
    return c;
}

constexpr uint32_t CLS_THREADS = 1024;

// T3b (PASS 0): per-block / per-warp histogram of head powers, spine list,
// depth and stack-height difference arrays.  (PASS 1): stable scatter of the
// main-loop nodes into per-power buckets (ascending power, position order).
// One block of CLS_THREADS boundaries (vb: the block's index); all threads of
// a CLS_THREADS-thread CTA call it.
template <int PASS>
PS_DEV void tree_classify_block(uint32_t vb, const uint8_t* __restrict__ P, const uint32_t* __restrict__ Rle,
                                const uint32_t* __restrict__ Lle, const uint32_t* __restrict__ b, uint32_t r,
                                uint32_t k, uint32_t nblocks, uint32_t* __restrict__ blockHist,
                                const uint32_t* __restrict__ blockOff, int32_t* __restrict__ Ddiff,
                                int32_t* __restrict__ Sdiff, uint32_t* __restrict__ spine_list,
                                Node* __restrict__ nodes, Summary* sum, const int32_t* __restrict__ pdelta) {
    __shared__ uint32_t whist[32][NPOW];
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    for (uint32_t i = tid; i < 32 * NPOW; i += blockDim.x) (&whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t j = vb * CLS_THREADS + tid + 1;
    const bool valid = j < r;
    BoundaryClass c;
    c.head = false;
    uint32_t p = 0xFF;
    if (valid) {
        c = classify(j, P, Rle, Lle, r, k, &sum->err);
        if (c.head) p = P[j];
    }
    const uint32_t peers = __match_any_sync(PS_FULL, p);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1));
    if (c.head && rank == 0) whist[warp][p] = __popc(peers);
    __syncthreads();
    // exclusive scan over warps per power bucket
    if (tid < NPOW) {
        uint32_t acc = 0;
        for (int w = 0; w < 32; ++w) {
            const uint32_t x = whist[w][tid];
            whist[w][tid] = acc;
            acc += x;
        }
        if (PASS == 0) blockHist[(uint64_t)tid * nblocks + vb] = acc;
    }
    __syncthreads();
    if (PASS == 0) {
        if (valid) {
            // stack height: boundary j is on the stack from its push until R(j)
            atomicAdd(&Sdiff[j], 1);
            if (c.rstrict != INF32) atomicAdd(&Sdiff[c.rstrict], -1);
            if (c.head) {
                // depth: the node strictly contains boundaries (begin, end)
                atomicAdd(&Ddiff[c.bidx[0] + 1], 1);
                atomicAdd(&Ddiff[c.bidx[1 + c.nmem]], -1);
            }
            if (c.spine) {
                const uint32_t s = atomicAdd(&sum->nspine, 1u);
                if (s < MAX_SPINE)
                    spine_list[s] = j;
                else
                    atomicOr(&sum->err, ERR_SPINE);
            }
        }
    } else if (c.head) {
        // power-bucket position, moved to the node's merge stage (tree_spine_cta)
        const uint32_t slot = blockOff[(uint64_t)p * nblocks + vb] + whist[warp][p] + rank + pdelta[p];
        Node nd;
        const uint32_t arity = c.nmem + 1;
        for (uint32_t i = 0; i < 5; ++i) nd.pos[i] = i <= arity ? b[c.bidx[i]] : 0u;
        nd.arity = (uint8_t)arity;
        nd.parity = 0;
        nd.power = (uint8_t)p;
        nd.flags = 0;
        nd.probe = c.bidx[1];
        nd.chunk_base = 0;
        nd.nchunks = 0;
        nd.order = c.bidx[1 + c.nmem];  // R's boundary index
        nodes[slot] = nd;
    }
    __syncthreads();  // whist is reused by the next call
}

template <int PASS>
__global__ void __launch_bounds__(CLS_THREADS) tree_classify_kernel(
    const uint8_t* __restrict__ P, const uint32_t* __restrict__ Rle, const uint32_t* __restrict__ Lle,
    const uint32_t* __restrict__ b, uint32_t r, uint32_t k, uint32_t nblocks, uint32_t* __restrict__ blockHist,
    const uint32_t* __restrict__ blockOff, int32_t* __restrict__ Ddiff, int32_t* __restrict__ Sdiff,
    uint32_t* __restrict__ spine_list, Node* __restrict__ nodes, Summary* sum, const int32_t* __restrict__ pdelta) {
    pdl_wait();
    tree_classify_block<PASS>(blockIdx.x, P, Rle, Lle, b, r, k, nblocks, blockHist, blockOff, Ddiff, Sdiff, spine_list,
                              nodes, sum, pdelta);
}

// T4: the spine and _merge_down (policy.py:146-175): staged by the CTA, replayed by one thread.
// min of level 0 over [lo, hi) of a 32-ary min tree: partial groups at each
// level, whole groups one level up
PS_DEV uint32_t range_min(const MinTree& t, uint32_t lo, uint32_t hi) {
    uint32_t m = 0xFF;
    for (uint32_t L = 0; lo < hi; ++L) {
        const uint8_t* a = t.lev[L];
        const uint32_t lo2 = (lo + 31) & ~31u, hi2 = hi & ~31u;
        if (L + 1 >= t.nlev || lo2 >= hi2) {
            for (uint32_t x = lo; x < hi; ++x) m = min(m, (uint32_t)a[x]);
            break;
        }
        for (uint32_t x = lo; x < lo2; ++x) m = min(m, (uint32_t)a[x]);
        for (uint32_t x = hi2; x < hi; ++x) m = min(m, (uint32_t)a[x]);
        lo = lo2 >> 5;
        hi = hi2 >> 5;
    }
    return m;
}

PS_DEV void tree_level_offsets_cta(const uint32_t* __restrict__ blockOff, const uint32_t* __restrict__ total,
                                   uint32_t nblocks, Summary* sum);

// Merge stage of a main-loop node: its power level, higher powers first.
PS_DEV uint32_t main_stage(uint32_t power) { return NPOW - power; }

// T6: the merge schedule is fixed here.  Stage h holds the main nodes of power
// NPOW - h (one contiguous power bucket, position order) followed by the
// merge_down nodes of stage h.  Writes the stage offsets into level_off (the
// power offsets it replaces are read first), each power bucket's shift
// pdelta[p] for classification pass 1, and the merge_down nodes at their
// final slots; so no regrouping pass is needed.
PS_DEV void tree_spine_cta(const uint32_t* __restrict__ b, uint32_t r, uint32_t k, int strict,
                           uint32_t* __restrict__ spine_list, Node* __restrict__ nodes, int32_t* __restrict__ Ddiff,
                           Summary* sum, const MinTree& mt, int32_t* __restrict__ pdelta) {
    __shared__ Node s_sn[MAX_SPINE];
    __shared__ uint32_t s_nn;
    __shared__ uint32_t s_cnt[NSTAGE + 1], s_soff[NSTAGE + 1], s_pow[NPOW + 1];
    // the stack entries are staged and sorted by the CTA, their run starts are
    // gathered in parallel; one thread then replays _merge_down from shared memory
    __shared__ uint32_t s_list[MAX_SPINE];
    __shared__ uint32_t s_beta[MAX_SPINE + 2];  // beta[1] = 0, beta[h] = s_{h-1}; [H+1] = first run_begin
    __shared__ uint32_t s_bval[MAX_SPINE + 2];  // b[beta[h]]
    __shared__ uint32_t s_br;
    __shared__ uint8_t s_key[MAX_SPINE + 2];  // merge stage of stack entry h's subtree (0: a single run)
    const uint32_t t = threadIdx.x;
    uint32_t H = sum->nspine;
    if (H > MAX_SPINE) {
        if (t == 0) atomicOr(&sum->err, ERR_SPINE);
        H = MAX_SPINE;
    }
    if (t < H) {  // rank sort of distinct boundary indices
        const uint32_t x = spine_list[t];
        uint32_t rank = 0;
        for (uint32_t i = 0; i < H; ++i) rank += spine_list[i] < x;
        s_list[rank] = x;
    }
    __syncthreads();
    for (uint32_t h = t + 1; h <= H + 1; h += blockDim.x)
        s_beta[h] = h == 1 ? 0u : (h <= H ? s_list[h - 2] : (H ? s_list[H - 1] : 0u));
    __syncthreads();
    for (uint32_t h = t + 1; h <= H + 1; h += blockDim.x) {
        s_bval[h] = b[s_beta[h]];
        // entry h spans boundaries [beta_h, end); its subtree's root is the main
        // node of the smallest power strictly inside
        const uint32_t lo = s_beta[h] + 1, hi = h <= H ? s_beta[h + 1] : r;
        s_key[h] = (uint8_t)(lo < hi ? main_stage(range_min(mt, lo, hi)) : 0u);
    }
    if (t == 0) s_br = b[r];
    for (uint32_t p = t; p <= NPOW; p += blockDim.x) s_pow[p] = sum->level_off[p];
    __syncthreads();
    if (t == 0) {
    uint32_t nn = 0;
    uint32_t height = H;
    uint32_t run_begin = H + 1;  // index into s_beta / s_bval
    uint32_t cur_key = s_key[H + 1];  // stage of the accumulated last run
    auto emit = [&](const uint32_t* hh, uint32_t w) {
        // a merge_down node runs after the last of its inputs (earliest stage here)
        uint32_t key = cur_key;
        for (uint32_t i = 0; i + 1 < w; ++i) key = max(key, (uint32_t)s_key[hh[i]]);
        key += 1;
        if (key >= NSTAGE) {
            atomicOr(&sum->err, ERR_SPINE);
            key = NSTAGE - 1;
        }
        cur_key = key;
        Node nd;
        for (uint32_t i = 0; i < 5; ++i) nd.pos[i] = 0;
        for (uint32_t i = 0; i < w; ++i) nd.pos[i] = s_bval[hh[i]];
        nd.pos[w] = s_br;
        nd.arity = (uint8_t)w;
        nd.parity = 0;
        nd.power = 0;
        nd.flags = (uint8_t)(1u | (key << 1));
        nd.probe = s_beta[hh[1]];
        nd.chunk_base = 0;
        nd.nchunks = 0;
        nd.order = nn;
        s_sn[nn] = nd;
        nn++;
        atomicAdd(&Ddiff[s_beta[hh[0]] + 1], 1);
        atomicAdd(&Ddiff[r], -1);
    };
    if (H > 0) {
        if (k == 4 && !strict) {
            const uint32_t n_runs = height + 1;
            const uint32_t rem = n_runs % 3;
            if (rem == 0) {
                const uint32_t h2 = height--;
                const uint32_t h1 = height--;
                const uint32_t hh[3] = {h1, h2, run_begin};
                emit(hh, 3);
                run_begin = h1;
            } else if (rem == 2) {
                const uint32_t h1 = height--;
                const uint32_t hh[2] = {h1, run_begin};
                emit(hh, 2);
                run_begin = h1;
            }
            while (height) {
                const uint32_t h3 = height--;
                const uint32_t h2 = height--;
                const uint32_t h1 = height--;
                const uint32_t hh[4] = {h1, h2, h3, run_begin};
                emit(hh, 4);
                run_begin = h1;
            }
        } else {
            while (height) {
                const uint32_t cnt = (k - 1) < height ? (k - 1) : height;
                uint32_t hh[4];
                for (uint32_t i = 0; i < cnt; ++i) hh[cnt - 1 - i] = height--;
                hh[cnt] = run_begin;
                emit(hh, cnt + 1);
                run_begin = hh[0];
            }
        }
    }
    // as late as possible: the chain ends at the root's stage, each node one
    // stage before its consumer (>= its earliest stage, which is at least one
    // less per step), so the chain shares the last main-loop launches
    for (uint32_t i = 0; i < nn; ++i) {
        const uint32_t key = cur_key - (nn - 1 - i);
        s_sn[i].flags = (uint8_t)(1u | (key << 1));
    }
    sum->nspine_nodes = nn;
    s_nn = nn;
    }
    __syncthreads();
    const uint32_t nn = s_nn;
    // nodes per stage: the power bucket NPOW - h plus the merge_down nodes of stage h
    for (uint32_t h = t; h <= NSTAGE; h += blockDim.x) {
        uint32_t c = 0;
        if (h >= 1 && h < NPOW) c = s_pow[NPOW - h + 1] - s_pow[NPOW - h];
        for (uint32_t i = 0; i < nn; ++i) c += (uint32_t)(s_sn[i].flags >> 1) == h;
        s_cnt[h] = c;
    }
    __syncthreads();
    if (t == 0) {
        uint32_t acc = 0;
        for (uint32_t h = 0; h <= NSTAGE; ++h) {
            s_soff[h] = acc;
            acc += s_cnt[h];
        }
    }
    __syncthreads();
    for (uint32_t h = t; h <= NSTAGE; h += blockDim.x) sum->level_off[h] = s_soff[h];
    for (uint32_t p = t; p < NPOW; p += blockDim.x)
        pdelta[p] = p >= 1 ? (int32_t)s_soff[NPOW - p] - (int32_t)s_pow[p] : 0;
    for (uint32_t i = t; i < nn; i += blockDim.x) {
        const uint32_t h = s_sn[i].flags >> 1;
        uint32_t rank = 0;
        for (uint32_t j = 0; j < i; ++j) rank += (uint32_t)(s_sn[j].flags >> 1) == h;
        const uint32_t pm = (h >= 1 && h < NPOW) ? s_pow[NPOW - h + 1] - s_pow[NPOW - h] : 0u;
        nodes[s_soff[h] + pm + rank] = s_sn[i];
    }
}
// (also the power-bucket offsets and nmain, from the scanned histograms)
__global__ void tree_spine_kernel(const uint32_t* __restrict__ b, uint32_t r, uint32_t k, int strict,
                                  uint32_t* __restrict__ spine_list, Node* __restrict__ nodes,
                                  int32_t* __restrict__ Ddiff, Summary* sum, MinTree mt,
                                  const uint32_t* __restrict__ hoff, const uint32_t* __restrict__ htot,
                                  uint32_t nblocks, int32_t* __restrict__ pdelta) {
    pdl_wait();
    tree_level_offsets_cta(hoff, htot, nblocks, sum);
    __syncthreads();
    tree_spine_cta(b, r, k, strict, spine_list, nodes, Ddiff, sum, mt, pdelta);
}

// T5: per-node depth/parity, chunk counts and merge statistics; leaf parity.
// slack_mode: 0 -> slack = arity ("4way"/"2way" sentinel kernels),
//             1 -> 2-way 0, 3/4-way 1 ("4way-nosentinel"), 2 -> 0.
// node count is read on the device (nmain + nspine_nodes, <= nmax): no host sync
PS_DEV uint32_t node_count(const Summary* sum, uint32_t nmax) {
    const uint32_t c = sum->nmain + sum->nspine_nodes;
    return c < nmax ? c : nmax;
}

// ---- T6: the merge schedule ---------------------------------------------------
// Every node carries a merge stage (flags >> 1): a main-loop node its power
// level (main_stage, higher powers first), a merge_down node one stage after
// the last of its inputs (tree_spine_cta).  Children always come in earlier
// stages, so the merge_down chain shares the main-loop levels' launches instead
// of running as a tail of single-node launches.  (Any topological order is
// valid: a node writes buffer depth & 1 over its own range, which only its
// ancestors read afterwards.)  Nodes are regrouped by stage, one launch each.
constexpr uint32_t FIN_THREADS = 256;

// T5: per-node depth/parity, merge stage, chunk counts, merge statistics and
// per-stage statistics; the block's stage histogram (hist[h * nblocks + blk])
// for the stable regrouping.
PS_DEV void tree_finalize_block(uint32_t i0, Node* __restrict__ nodes, uint32_t nmax, const int32_t* __restrict__ S,
                                int slack_mode, uint32_t cap, Summary* sum, uint32_t* __restrict__ nch) {
    __shared__ uint32_t s_hh[NSTAGE];
    __shared__ unsigned long long s_cost[NSTAGE];
    __shared__ uint32_t s_small[NSTAGE], s_smax[NSTAGE];
    const uint32_t nnodes = node_count(sum, nmax);
    const uint32_t i = i0 + threadIdx.x;
    for (uint32_t t = threadIdx.x; t < NSTAGE; t += blockDim.x) {
        s_hh[t] = 0;
        s_cost[t] = 0;
        s_small[t] = 0;
        s_smax[t] = 0;
    }
    __syncthreads();
    unsigned long long cost = 0, m2 = 0, m3 = 0, m4 = 0, slack = 0, copied = 0;
    uint32_t key = 0xFFFFFFFFu, sz = 0, sm = 0;
    if (i < nnodes) {
        Node nd = nodes[i];
        const int32_t depth = S[nd.probe] - 1;
        nd.parity = (uint8_t)(depth & 1);
        const uint32_t w = nd.arity;
        const uint32_t size = nd.pos[w] - nd.pos[0];
        nd.nchunks = node_chunks(nd, cap, SMALL_KERNEL_MAX);
        if (!(nd.flags & 1)) nd.flags = (uint8_t)(main_stage(nd.power) << 1);  // (spine: set by tree_spine_cta)
        const uint32_t stage = nd.flags >> 1;
        nodes[i] = nd;
        nch[i] = nd.nchunks;
        atomicAdd(&s_hh[stage], 1u);
        cost = size;
        if (w == 2) copied = min(nd.pos[1] - nd.pos[0], nd.pos[2] - nd.pos[1]);  // copy-smaller's buffer
        m2 = w == 2;
        m3 = w == 3;
        m4 = w == 4;
        slack = slack_mode == 0 ? w : (slack_mode == 1 ? (w == 2 ? 0 : 1) : 0);
        if (depth < 0) atomicOr(&sum->err, ERR_CHAIN);
        key = stage;
        sz = size;
        sm = size <= SMALL_KERNEL_MAX;
    } else if (i < nmax) {
        nch[i] = 0;  // (the chunk scan runs over nmax)
    }
    // per-stage cost / small counts: shared-memory atomics per distinct stage
    // per warp, then one global atomic per stage per block (the nodes arrive
    // grouped by power, so most blocks touch one or two stages; per-warp global
    // atomics on a handful of addresses serialised in L2)
    {
        const uint32_t grp = __match_any_sync(PS_FULL, key);
        const uint32_t gsz = __reduce_add_sync(grp, sz), gsm = __reduce_add_sync(grp, sm);
        const uint32_t gmx = __reduce_max_sync(grp, sm ? sz : 0u);
        if (key != 0xFFFFFFFFu && lane_id() == (uint32_t)(__ffs(grp) - 1)) {
            atomicAdd(&s_cost[key], (unsigned long long)gsz);
            if (gsm) {
                atomicAdd(&s_small[key], gsm);
                atomicMax(&s_smax[key], gmx);
            }
        }
    }
    for (int d = 16; d; d >>= 1) {
        cost += __shfl_xor_sync(PS_FULL, cost, d);
        m2 += __shfl_xor_sync(PS_FULL, m2, d);
        m3 += __shfl_xor_sync(PS_FULL, m3, d);
        m4 += __shfl_xor_sync(PS_FULL, m4, d);
        slack += __shfl_xor_sync(PS_FULL, slack, d);
        copied += __shfl_xor_sync(PS_FULL, copied, d);
    }
    // block reduction, then one set of atomics per block
    __shared__ unsigned long long s_red[6][32];
    const uint32_t wv = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s_red[0][wv] = cost;
        s_red[1][wv] = m2;
        s_red[2][wv] = m3;
        s_red[3][wv] = m4;
        s_red[4][wv] = slack;
        s_red[5][wv] = copied;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        unsigned long long t = 0;
        for (uint32_t q = 0; q < (blockDim.x + 31) / 32; ++q) t += s_red[threadIdx.x][q];
        if (t) {
            unsigned long long* dst = threadIdx.x == 0   ? &sum->merge_cost
                                    : threadIdx.x == 4 ? &sum->scan_slack
                                    : threadIdx.x == 5 ? &sum->cs_copied
                                                       : &sum->merges[threadIdx.x + 1];
            atomicAdd(dst, t);
        }
    }
    for (uint32_t t = threadIdx.x; t < NSTAGE; t += blockDim.x) {
        if (s_hh[t]) {
            atomicAdd(&sum->level_cost[t], s_cost[t]);
            if (s_small[t]) {
                atomicAdd(&sum->level_small[t], s_small[t]);
                atomicMax(&sum->level_small_max[t], s_smax[t]);
            }
        }
    }
    __syncthreads();  // s_red / s_hh are reused by the next call
}
// (grid over nmax >= r + 1 threads: also the max stack height from the
// stack-height prefix H and the leaf parities from the depths S)
__global__ void __launch_bounds__(FIN_THREADS) tree_nodes_finalize_kernel(
    Node* __restrict__ nodes, uint32_t nmax, const int32_t* __restrict__ S, int slack_mode, uint32_t cap,
    Summary* sum, uint32_t* __restrict__ nch, const int32_t* __restrict__ H, uint32_t r,
    uint32_t stack_cap, uint8_t* __restrict__ leafpar) {
    pdl_wait();
    {
        const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x + 1;
        if (leafpar && j - 1 < r) {
            const uint32_t jl = j - 1;
            const int32_t a = jl == 0 ? 0 : S[jl];
            const int32_t c = jl + 1 >= r ? 0 : S[jl + 1];
            leafpar[jl] = (uint8_t)((a > c ? a : c) & 1);
        }
        // block maximum, one atomic per block (per-warp atomics on one address serialise)
        __shared__ int32_t s_hmax[FIN_THREADS / 32];
        int32_t v = (j < r) ? H[j] : 0;
        for (int d = 16; d; d >>= 1) v = max(v, __shfl_xor_sync(PS_FULL, v, d));
        if (lane_id() == 0) s_hmax[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (uint32_t w = 1; w < FIN_THREADS / 32; ++w) v = max(v, s_hmax[w]);
            if (v > 0) {
                atomicMax(&sum->max_stack, (uint32_t)v);
                if ((uint32_t)v > stack_cap) atomicOr(&sum->err, ERR_STACK);
            }
        }
    }
    tree_finalize_block(blockIdx.x * blockDim.x, nodes, nmax, S, slack_mode, cap, sum, nch);
}

// chunk_base at the node indices the host schedules stages by: the stage
// offsets (out[0..NSTAGE]) and the total (out[NSTAGE+1]); cb has nnodes+1
// entries.
PS_DEV void tree_stage_chunks_cta(const uint32_t* __restrict__ cb, const Summary* __restrict__ sum, uint32_t nmax,
                                   uint32_t* __restrict__ out) {
    const uint32_t nnodes = node_count(sum, nmax);
    const uint32_t t = threadIdx.x;
    for (uint32_t h = t; h <= NSTAGE; h += blockDim.x) {
        const uint32_t i = sum->level_off[h];
        out[h] = cb[i < nnodes ? i : nnodes];
    }
    if (t == 0) out[NSTAGE + 1] = cb[nnodes];
}
__global__ void tree_stage_chunks_kernel(const uint32_t* __restrict__ cb, const Summary* __restrict__ sum,
                                         uint32_t nmax, uint32_t* __restrict__ out) {
    pdl_wait();
    tree_stage_chunks_cta(cb, sum, nmax, out);
}

__global__ void tree_leaf_parity_kernel(const int32_t* __restrict__ S, uint32_t r, uint8_t* __restrict__ leafpar) {
    pdl_wait();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= r) return;
    const int32_t a = j == 0 ? 0 : S[j];
    const int32_t c = j + 1 >= r ? 0 : S[j + 1];
    leafpar[j] = (uint8_t)((a > c ? a : c) & 1);
}

// max stack height (H = inclusive scan of the stack difference array) and, with
// leafpar, the leaf parities from the depths S
__global__ void tree_stack_max_kernel(const int32_t* __restrict__ H, uint32_t r, Summary* sum, uint32_t cap,
                                      const int32_t* __restrict__ S, uint8_t* __restrict__ leafpar) {
    pdl_wait();
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (leafpar && j - 1 < r) {
        const uint32_t jl = j - 1;
        const int32_t a = jl == 0 ? 0 : S[jl];
        const int32_t c = jl + 1 >= r ? 0 : S[jl + 1];
        leafpar[jl] = (uint8_t)((a > c ? a : c) & 1);
    }
    int32_t v = (j < r) ? H[j] : 0;
    for (int d = 16; d; d >>= 1) v = max(v, __shfl_xor_sync(PS_FULL, v, d));
    if (lane_id() == 0 && v > 0) {
        atomicMax(&sum->max_stack, (uint32_t)v);
        if ((uint32_t)v > cap) atomicOr(&sum->err, ERR_STACK);
    }
}

// level offsets of the power buckets from the scanned block histograms
PS_DEV void tree_level_offsets_cta(const uint32_t* __restrict__ blockOff, const uint32_t* __restrict__ total,
                                   uint32_t nblocks, Summary* sum) {
    const uint32_t p = threadIdx.x;
    if (p < NPOW) sum->level_off[p] = blockOff[(uint64_t)p * nblocks];
    if (p == 0) {
        sum->level_off[NPOW] = *total;
        sum->nmain = *total;
    }
}
__global__ void tree_level_offsets_kernel(const uint32_t* __restrict__ blockOff, const uint32_t* __restrict__ total,
                                          uint32_t nblocks, Summary* sum) {
    pdl_wait();
    tree_level_offsets_cta(blockOff, total, nblocks, sum);
}

// chunk_base into the nodes; block 0 also gathers the stage chunk offsets
__global__ void tree_copy_chunk_base_kernel(Node* __restrict__ nodes, const uint32_t* __restrict__ base,
                                            uint32_t nmax, const Summary* __restrict__ sum,
                                            uint32_t* __restrict__ stage_chunk) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < node_count(sum, nmax)) nodes[i].chunk_base = base[i];
    if (blockIdx.x == 0) tree_stage_chunks_cta(base, sum, nmax, stage_chunk);
}

// chunk_base into the nodes, the stage chunk offsets (block 0) and the chunk
// -> node map (the last node whose chunk base is <= c, searched in cb), grid-
// stride over CHUNK_MAP_CTAS CTAs; the counts are read on the device.
__global__ void tree_chunks_kernel(Node* __restrict__ nodes, const uint32_t* __restrict__ cb, uint32_t nmax,
                                   Summary* sum, uint32_t* __restrict__ stage_chunk, uint32_t chunks_max,
                                   uint32_t* __restrict__ chunk2node) {
    pdl_wait();
    const uint32_t nn = node_count(sum, nmax);
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    for (uint32_t i = gt; i < nn; i += gs) nodes[i].chunk_base = cb[i];
    if (blockIdx.x == 0) tree_stage_chunks_cta(cb, sum, nmax, stage_chunk);
    const uint32_t total = cb[nn];
    if (nn == 0 || total > chunks_max) return;  // (the host fails on the published total)
    for (uint32_t c = gt; c < total; c += gs) {
        uint32_t lo = 0, hi = nn;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (cb[mid] <= c)
                lo = mid;
            else
                hi = mid;
        }
        chunk2node[c] = lo;
    }
}

// nchunks per node, zero for the padding up to nmax (the scan runs over nmax)
__global__ void tree_nchunks_kernel(const Node* __restrict__ nodes, uint32_t nmax, const Summary* __restrict__ sum,
                                    uint32_t* __restrict__ out) {
    pdl_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nmax) out[i] = i < node_count(sum, nmax) ? nodes[i].nchunks : 0u;
}

// chunk -> node map by binary search over the nodes' chunk_base; the node and
// chunk counts are read on the device (grid-stride over CHUNK_MAP_CTAS CTAs).
constexpr uint32_t CHUNK_MAP_CTAS = 4 * 148;
__global__ void tree_chunk_map_kernel(const Node* __restrict__ nodes, const Summary* __restrict__ sum,
                                      const uint32_t* __restrict__ stage_chunk, uint32_t chunks_max,
                                      uint32_t* __restrict__ chunk2node) {
    pdl_wait();
    const uint32_t nnodes = sum->nmain + sum->nspine_nodes;
    const uint32_t total = stage_chunk[NSTAGE + 1];
    if (nnodes == 0 || total > chunks_max) return;  // (the host fails on the published total)
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < total; c += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nnodes;  // find last node with chunk_base <= c
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (nodes[mid].chunk_base <= c)
                lo = mid;
            else
                hi = mid;
        }
        chunk2node[c] = lo;
    }
}

// ---------------------------------------------------------------------------
// The whole tree build (T1-T5) for r <= TREE_SMALL_R boundaries in ONE CTA of
// CLS_THREADS threads: the phases of the multi-kernel path back to back with
// CTA barriers instead of ~20 dependent launches.
#ifndef PS_TREE_SMALL_R
#define PS_TREE_SMALL_R 1024
#endif
constexpr uint32_t TREE_SMALL_R = PS_TREE_SMALL_R;

struct TreeSmallArgs {
    const uint32_t* b;
    uint32_t r;
    uint64_t n;
    uint32_t log2k, k;
    int strict, slack_mode;
    uint32_t cap, stack_cap;
    uint8_t* P;
    uint32_t padded;
    MinTree mt;
    uint32_t lev_groups[8], lev_padded[8];  // level l >= 1: input groups, padded size
    uint32_t* Rle;
    uint32_t* Lle;
    int32_t* Dd;
    int32_t* Sd;
    uint32_t nblocks;
    uint32_t* hist;
    uint32_t* hoff;
    uint32_t* htot;
    uint32_t* spine;
    Node* nodes;
    uint8_t* leafpar;  // nullable
    uint32_t nmax;
    uint32_t* nch;
    uint32_t* cb;
    uint32_t* stage_chunk;
    Summary* sum;
    int32_t* pdelta;                        // per-power shift to the merge-stage order
};

__global__ void __launch_bounds__(CLS_THREADS) tree_small_kernel(TreeSmallArgs a) {
    pdl_wait();
    __shared__ uint32_t s_items[CLS_THREADS * 2];  // (static shared memory: the spine stages its nodes too)
    __shared__ uint32_t s_sw[32];
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    uint32_t* err = &a.sum->err;
    for (uint32_t i = tid; i < a.r + 2; i += nt) {
        a.Dd[i] = 0;
        a.Sd[i] = 0;
    }
    for (uint32_t j = tid; j < a.padded; j += nt) tree_power_one(j, a.b, a.r, a.n, a.log2k, a.P, err);
    __syncthreads();
    for (uint32_t l = 1; l < a.mt.nlev; ++l) {
        uint8_t* out = const_cast<uint8_t*>(a.mt.lev[l]);
        for (uint32_t i = tid; i < a.lev_padded[l]; i += nt) tree_minlevel_one(i, a.mt.lev[l - 1], a.lev_groups[l], out);
        __syncthreads();
    }
    for (uint32_t j = tid + 1; j < a.r; j += nt) {
        const uint32_t v = a.P[j];
        a.Rle[j] = find_right_le(a.mt, j, v);
        a.Lle[j] = find_left_le(a.mt, j, v);
    }
    __syncthreads();
    for (uint32_t vb = 0; vb < a.nblocks; ++vb)
        tree_classify_block<0>(vb, a.P, a.Rle, a.Lle, a.b, a.r, a.k, a.nblocks, a.hist, nullptr, a.Dd, a.Sd, a.spine,
                               a.nodes, a.sum, a.pdelta);
    cta_scan<uint32_t, OpSum<uint32_t>, 2>(a.hist, a.hoff, (int64_t)NPOW * a.nblocks, false, true, a.htot, s_items,
                                           s_sw);
    tree_level_offsets_cta(a.hoff, a.htot, a.nblocks, a.sum);
    __syncthreads();
    tree_spine_cta(a.b, a.r, a.k, a.strict, a.spine, a.nodes, a.Dd, a.sum, a.mt, a.pdelta);
    __syncthreads();
    for (uint32_t vb = 0; vb < a.nblocks; ++vb)
        tree_classify_block<1>(vb, a.P, a.Rle, a.Lle, a.b, a.r, a.k, a.nblocks, nullptr, a.hoff, a.Dd, a.Sd, a.spine,
                               a.nodes, a.sum, a.pdelta);
    cta_scan<int32_t, OpSum<int32_t>, 2>(a.Dd, a.Dd, (int64_t)a.r + 1, false, false, nullptr,
                                         reinterpret_cast<int32_t*>(s_items), reinterpret_cast<int32_t*>(s_sw));
    cta_scan<int32_t, OpSum<int32_t>, 2>(a.Sd, a.Sd, (int64_t)a.r + 1, false, false, nullptr,
                                         reinterpret_cast<int32_t*>(s_items), reinterpret_cast<int32_t*>(s_sw));
    for (uint32_t j0 = 0; j0 < a.r; j0 += nt) {  // max stack height
        const uint32_t j = j0 + tid + 1;
        int32_t v = j < a.r ? a.Sd[j] : 0;
        for (int d = 16; d; d >>= 1) v = max(v, __shfl_xor_sync(PS_FULL, v, d));
        if (lane_id() == 0 && v > 0) {
            atomicMax(&a.sum->max_stack, (uint32_t)v);
            if ((uint32_t)v > a.stack_cap) atomicOr(err, ERR_STACK);
        }
    }
    if (a.leafpar) {
        for (uint32_t j = tid; j < a.r; j += nt) {
            const int32_t x = j == 0 ? 0 : a.Dd[j];
            const int32_t y = j + 1 >= a.r ? 0 : a.Dd[j + 1];
            a.leafpar[j] = (uint8_t)((x > y ? x : y) & 1);
        }
    }
    __syncthreads();
    for (uint32_t i0 = 0; i0 < a.nmax; i0 += nt)
        tree_finalize_block(i0, a.nodes, a.nmax, a.Dd, a.slack_mode, a.cap, a.sum, a.nch);
    __syncthreads();
    cta_scan<uint32_t, OpSum<uint32_t>, 2>(a.nch, a.cb, a.nmax, false, true, a.cb + a.nmax, s_items, s_sw);
    {
        const uint32_t nn = node_count(a.sum, a.nmax);
        for (uint32_t i = tid; i < nn; i += nt) a.nodes[i].chunk_base = a.cb[i];
    }
    __syncthreads();
    tree_stage_chunks_cta(a.cb, a.sum, a.nmax, a.stage_chunk);
}

}  // namespace ps

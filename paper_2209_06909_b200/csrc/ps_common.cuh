// ps_common.cuh -- shared constants, types and device helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <utility>

#define PS_DEV __device__ __forceinline__
#define PS_FULL 0xFFFFFFFFu

namespace ps {

// ---- run detection geometry --------------------------------
constexpr uint32_t TILE = 2048;                   // positions per chain tile (one warp)
#ifndef PS_TPG
#define PS_TPG 8
#endif
constexpr uint32_t TILES_PER_GROUP = PS_TPG;      // tiles per CTA (a warp each)
constexpr uint32_t RD_THREADS = TILES_PER_GROUP * 32;  // run-detection CTA size
constexpr uint32_t GROUP = TILE * TILES_PER_GROUP; // positions per CTA
constexpr uint32_t GROUP_WORDS = GROUP / 32;      // type-bit words per CTA
constexpr uint32_t MAX_M_TILED = 256;             // larger min_run_len -> serial chain walker
constexpr uint32_t TSCAN_FAN = 32;                // tables composed per warp in the chain scan

// ---- merge geometry ------------------------------------------------------
constexpr uint32_t CHUNK_CAP = 4096;  // max records per merge chunk (k * cut spacing), 4-byte keys
// per key width: 8-byte keys use half the records so two CTAs still fit per SM
template <class K>
__host__ __device__ constexpr uint32_t chunk_cap() {
#ifdef PS_CAP4
    return sizeof(K) == 4 ? PS_CAP4 : CHUNK_CAP / 2;
#else
    return sizeof(K) == 4 ? CHUNK_CAP : CHUNK_CAP / 2;
#endif
}
constexpr uint32_t MERGE_THREADS = 256;
constexpr uint32_t MERGE_VT = CHUNK_CAP / MERGE_THREADS;  // 16 records per thread
constexpr uint32_t MAX_WAY = 4;
constexpr uint32_t SMALL_NODE = 512;  // nodes up to this size: one warp each (no chunking)
// nodes of at most SMALL_KERNEL_MAX records are merged by merge_small_kernel
// (<= SMALL_NODE); all others by the TMA pipeline (0: the pipeline takes all).
// Tiny nodes stay on the warp kernel: a pipeline unit holds at most MAXSEG of
// them and its producer then dominates.
#ifndef PS_SMALL_MAX
#define PS_SMALL_MAX 512
#endif
constexpr uint32_t SMALL_KERNEL_MAX = PS_SMALL_MAX;
static_assert(SMALL_KERNEL_MAX <= SMALL_NODE, "small-kernel threshold exceeds its capacity");

constexpr uint32_t INF32 = 0xFFFFFFFFu;
constexpr uint32_t MAX_SPINE = 256;
constexpr uint32_t NPOW = 64;  // power buckets (powers are <= 33 for n <= 2^31)
constexpr uint32_t NSTAGE = 128;  // merge stages: NPOW - power, merge_down nodes after their inputs (< 2^7)

// Error flags raised on the device (bitmask in Summary.err).
enum : uint32_t {
    ERR_CHAIN = 1u,      // run-chain candidate lemma violated
    ERR_GROUP = 2u,      // more than k-1 equal powers in a group (policy.py:139)
    ERR_SPINE = 4u,      // spine larger than MAX_SPINE
    ERR_STACK = 8u,      // run stack above run_stack_capacity (policy.py:117-120)
    ERR_CUT = 16u,       // merge chunk larger than CHUNK_CAP
    ERR_POWER = 32u,     // power outside 1..NPOW-1
    ERR_BARRIER = 64u,   // grid barrier timed out (CTAs not co-resident)
};

// One merge of the tree.  pos[0..arity] are the run boundaries (positions):
// children are [pos[a], pos[a+1]).
struct Node {
    uint32_t pos[5];
    uint8_t arity;
    uint8_t parity;   // output buffer (depth & 1)
    uint8_t power;    // boundary power (0 for merge_down/spine nodes)
    uint8_t flags;
    uint32_t probe;   // a member boundary index (depth lookup)
    uint32_t chunk_base;
    uint32_t nchunks;
    uint32_t order;   // reference execution order key helper
};
static_assert(sizeof(Node) == 40, "Node layout");

// Cut spacing of a node's runs (ps_merge.cuh): cap / arity, so that a chunk
// holds <= cap records.  (Finer cuts for the single-node merge_down stages were
// measured: no gain, their time is the partition search and the first load.)
PS_DEV __host__ uint32_t node_spacing(const Node& nd, uint32_t cap) { return cap / nd.arity; }
// chunks of a node: 0 for the small-node kernel, else 1 + its cut points
PS_DEV __host__ uint32_t node_chunks(const Node& nd, uint32_t cap, uint32_t small_max) {
    const uint32_t w = nd.arity, size = nd.pos[w] - nd.pos[0];
    if (size <= small_max) return 0;
    const uint32_t S = node_spacing(nd, cap);
    uint32_t nch = 1;
    if (size > w * S)
        for (uint32_t a = 0; a < w; ++a) nch += (nd.pos[a + 1] - nd.pos[a] - 1) / S;
    return nch;
}

// Device -> host summary, read once after the tree is built.
struct Summary {
    uint32_t r;              // runs
    uint32_t err;            // ERR_* bitmask
    uint32_t nmain;          // main-loop merge nodes
    uint32_t nspine;         // spine boundaries
    uint32_t nspine_nodes;   // merge_down nodes
    uint32_t max_stack;      // max_stack_height
    uint32_t total_chunks;
    uint32_t pad0;
    uint32_t level_off[NSTAGE + 1];  // node offsets per power bucket, then (T6) per merge stage
    unsigned long long merge_cost;
    unsigned long long merges[5];      // by arity
    unsigned long long scan_slack;     // sum of per-merge slack (variant-specific)
    unsigned long long buffer_cost;
    // CountingOrder counters (ps_config.count_comparisons): comparisons and the
    // data-dependent moves of detection / extension; copy-smaller's copied and
    // written element totals (merges.py:145-201)
    unsigned long long comparisons;
    unsigned long long moves;
    unsigned long long cs_copied;
    unsigned long long cs_written;
    unsigned long long level_cost[NSTAGE];     // merge cost per merge stage
    uint32_t level_small[NSTAGE];               // nodes <= SMALL_NODE per stage
    uint32_t level_small_max[NSTAGE];           // largest small node per stage
};

// Programmatic dependent launch (PDL).  Every kernel is launched with
// programmatic stream serialization, so its launch overlaps the tail of the
// previous kernel in the stream; pdl_wait() (first statement of every kernel)
// blocks until that predecessor has completed and its writes are visible.
PS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Measurement knobs for A/B runs.  Only a -DPS_DEBUG_KNOBS build (tools/,
// libpowersort_b200_debug.so) reads them from the environment; the product
// library ignores the environment, so no variable can change what ps_sort does.
inline long knob(const char* name, long dflt) {
#ifdef PS_DEBUG_KNOBS
    const char* v = getenv(name);
    return v ? atol(v) : dflt;
#else
    (void)name;
    return dflt;
#endif
}
inline bool knob_set(const char* name) {
#ifdef PS_DEBUG_KNOBS
    return getenv(name) != nullptr;
#else
    (void)name;
    return false;
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    static const bool pdl = !knob_set("PS_NO_PDL");  // PS_NO_PDL=1: plain stream order (A/B runs)
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Cooperative launch (all CTAs co-resident, or the launch fails), for kernels
// with a grid barrier; `pdl` adds programmatic stream serialization.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_coop(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Barrier over all CTAs of a grid whose CTAs are co-resident (persistent
// grids of <= occupancy x SMs CTAs, launched cooperatively).  ctr is zeroed before the launch; the k-th
// barrier of a launch waits for target = k * gridDim.x arrivals.  A bounded
// spin turns a missing CTA into ERR_BARRIER instead of a hang.
PS_DEV void grid_barrier(uint32_t* ctr, uint32_t target, uint32_t* err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        for (uint32_t spins = 0;; ++spins) {
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            __nanosleep(100);
            if (spins > (1u << 23)) {
                atomicOr(err, ERR_BARRIER);
                break;
            }
        }
        __threadfence();
    }
    __syncthreads();
}


PS_DEV uint32_t lane_id() { return threadIdx.x & 31u; }
PS_DEV uint32_t warp_id() { return threadIdx.x >> 5; }

PS_DEV uint64_t pack_xc(uint32_t x, uint32_t c) { return ((uint64_t)c << 32) | x; }
PS_DEV uint32_t unpack_x(uint64_t v) { return (uint32_t)v; }
PS_DEV uint32_t unpack_c(uint64_t v) { return (uint32_t)(v >> 32); }

template <class T>
PS_DEV T shfl(T v, int src) {
    return __shfl_sync(PS_FULL, v, src);
}
template <class T>
PS_DEV T shfl_up(T v, int d) {
    return __shfl_up_sync(PS_FULL, v, d);
}

// Key comparisons: the reference's `le` is `key(a) <= key(b)` (statskit.py:68-72).
template <class K>
PS_DEV bool key_le(K a, K b) {
    return a <= b;
}
template <class K>
PS_DEV bool key_lt(K a, K b) {
    return a < b;
}

}  // namespace ps

// ps_scan.cuh -- device-wide reduce-then-scan for small auxiliary arrays
// (run counts, power histograms, depth / stack-height difference arrays).
// Forward or reverse, inclusive or exclusive, any commutative monoid.
#pragma once

#include <atomic>

#include "ps_common.cuh"

namespace ps {

// Host-side count of kernels launched by this library (bench evidence).
inline std::atomic<int64_t>& launch_counter() {
    static std::atomic<int64_t> c{0};
    return c;
}

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_BLK = SCAN_THREADS * SCAN_ITEMS;

template <class T>
struct OpSum {
    PS_DEV T operator()(T a, T b) const { return a + b; }
    PS_DEV static T id() { return T(0); }
};
template <class T>
struct OpMin {
    PS_DEV T operator()(T a, T b) const { return a < b ? a : b; }
    PS_DEV static T id() { return T(~T(0)) > T(0) ? T(~T(0)) : T(0x7FFFFFFF); }
};
template <class T>
struct OpMax {
    PS_DEV T operator()(T a, T b) const { return a > b ? a : b; }
    PS_DEV static T id() { return T(0); }
};

// Exclusive block scan of one value per thread (thread order); returns the
// exclusive prefix, writes the block total.
template <class T, class Op>
PS_DEV T block_exclusive(T v, T& total, T* sw /* >= 32 */) {
    Op op;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    T x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(PS_FULL, x, d);
        if (lane >= d) x = op(y, x);
    }
    if (lane == 31) sw[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nw ? sw[lane] : Op::id();
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            T y = __shfl_up_sync(PS_FULL, w, d);
            if (lane >= d) w = op(y, w);
        }
        sw[lane] = w;
    }
    __syncthreads();
    T wpre = warp ? sw[warp - 1] : Op::id();
    total = sw[nw - 1];
    T ex = __shfl_up_sync(PS_FULL, x, 1);
    if (lane == 0) ex = Op::id();
    T r = op(wpre, ex);
    __syncthreads();
    return r;
}

// Single-pass scan with decoupled look-back: CTA t scans tile t (SCAN_BLK
// items), publishes its aggregate, then walks back over its predecessors'
// status words until it meets an inclusive prefix.  Status word = epoch (30
// bits, unique per launch, so no zeroing pass is needed) | flag (2) | value
// (32).  Tiles are indexed by blockIdx.x; the hardware dispatches blocks in
// index order, so every predecessor a CTA waits on is already running.
// gridDim.y = 2 scans a second array of the same length (status words follow).
constexpr uint32_t SCAN_AGG = 1, SCAN_PREFIX = 2;

PS_DEV unsigned long long scan_word(uint32_t epoch, uint32_t flag, uint32_t v) {
    return ((unsigned long long)epoch << 34) | ((unsigned long long)flag << 32) | v;
}
PS_DEV void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
PS_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <class T, class Op>
__global__ void __launch_bounds__(SCAN_THREADS) scan_onepass_kernel(const T* in, T* out, int64_t n, int reverse,
                                                                    int exclusive, T* total_out,
                                                                    unsigned long long* status, uint32_t epoch,
                                                                    const T* in2, T* out2) {
    static_assert(sizeof(T) == 4, "status words carry 32-bit values");
    pdl_wait();
    if (blockIdx.y == 1) {  // a second, independent array of the same length
        in = in2;
        out = out2;
        total_out = nullptr;
        status += gridDim.x;
    }
    __shared__ T items[SCAN_BLK];
    __shared__ T sw[32];
    __shared__ T s_prefix;
    Op op;
    const uint32_t tile = blockIdx.x;
    const int64_t base = (int64_t)tile * SCAN_BLK;
    for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
        const int64_t g = base + i;
        items[i] = g < n ? in[reverse ? n - 1 - g : g] : Op::id();
    }
    __syncthreads();
    T loc[SCAN_ITEMS];
    T acc = Op::id();
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        loc[j] = items[threadIdx.x * SCAN_ITEMS + j];
        acc = op(acc, loc[j]);
    }
    T total;
    T pre = block_exclusive<T, Op>(acc, total, sw);
    if (threadIdx.x < 32) {
        // warp look-back: 32 predecessors per round; stop at the nearest prefix
        const uint32_t lane = threadIdx.x;
        T prefix = Op::id();
        if (tile == 0) {
            if (lane == 0) st_release_u64(&status[0], scan_word(epoch, SCAN_PREFIX, (uint32_t)total));
        } else {
            if (lane == 0) st_release_u64(&status[tile], scan_word(epoch, SCAN_AGG, (uint32_t)total));
            for (int64_t top = (int64_t)tile - 1;; top -= 32) {
                const int64_t j = top - (int64_t)lane;
                T x = Op::id();
                uint32_t f = SCAN_PREFIX;
                if (j >= 0) {
                    unsigned long long v;
                    do {  // predecessor j publishes its aggregate without waiting on anything
                        v = ld_acquire_u64(&status[j]);
                        f = (uint32_t)(v >> 32) & 3u;
                    } while ((uint32_t)(v >> 34) != epoch || f == 0);
                    x = (T)(uint32_t)v;
                }
                const uint32_t pm = __ballot_sync(PS_FULL, f == SCAN_PREFIX);
                const uint32_t first = pm ? (uint32_t)(__ffs(pm) - 1) : 32u;  // nearest prefix
                if (lane > first) x = Op::id();
                for (int d = 16; d; d >>= 1) x = op(x, __shfl_xor_sync(PS_FULL, x, d));  // (Op is commutative)
                prefix = op(x, prefix);
                if (pm) break;
            }
            if (lane == 0) st_release_u64(&status[tile], scan_word(epoch, SCAN_PREFIX, (uint32_t)op(prefix, total)));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    pre = op(s_prefix, pre);
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const T inc = op(pre, loc[j]);
        items[threadIdx.x * SCAN_ITEMS + j] = exclusive ? pre : inc;
        pre = inc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
        const int64_t g = base + i;
        if (g < n) out[reverse ? n - 1 - g : g] = items[i];
    }
    if (total_out && threadIdx.x == 0 && tile == gridDim.x - 1) *total_out = op(s_prefix, total);
}

inline uint32_t scan_next_epoch() {
    // unique per launch within the process; the random start keeps stale status
    // words of another process in reused device memory from matching
    static std::atomic<uint32_t> e{(uint32_t)(((uintptr_t)&e >> 4) ^ (uint32_t)clock()) & 0x3FFFFFFFu};
    uint32_t v;
    do v = e.fetch_add(1) & 0x3FFFFFFFu; while (v == 0);
    return v;
}

// Whole-CTA scan (any blockDim <= 1024) for fused single-CTA kernels: tiles of
// blockDim * ITEMS items with a running carry.  items: blockDim * ITEMS
// elements of shared memory, sw: 32.  Ends with a CTA barrier.
template <class T, class Op, int ITEMS>
PS_DEV void cta_scan(const T* in, T* out, int64_t n, bool reverse, bool exclusive, T* total_out, T* items, T* sw,
                     T carry = Op::id()) {
    Op op;
    const int TB = (int)blockDim.x * ITEMS;
    for (int64_t base = 0; base < n; base += TB) {
        for (int i = threadIdx.x; i < TB; i += blockDim.x) {
            const int64_t g = base + i;
            items[i] = g < n ? in[reverse ? n - 1 - g : g] : Op::id();
        }
        __syncthreads();
        T loc[ITEMS];
        T acc = Op::id();
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            loc[j] = items[threadIdx.x * ITEMS + j];
            acc = op(acc, loc[j]);
        }
        T total;
        T pre = op(carry, block_exclusive<T, Op>(acc, total, sw));
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const T inc = op(pre, loc[j]);
            items[threadIdx.x * ITEMS + j] = exclusive ? pre : inc;
            pre = inc;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < TB; i += blockDim.x) {
            const int64_t g = base + i;
            if (g < n) out[reverse ? n - 1 - g : g] = items[i];
        }
        carry = op(carry, total);
        __syncthreads();
    }
    if (total_out && threadIdx.x == 0) *total_out = carry;
    __syncthreads();
}

// Elements (4-byte) of temporary storage device_scan / device_scan2 need for n
// items: the status words of two arrays' tiles.
inline int64_t scan_tmp_elems(int64_t n) { return 4 * ((n + SCAN_BLK - 1) / SCAN_BLK + 1) + 64; }

// out may alias in.  tmp: scan_tmp_elems(n) elements (8-byte aligned).
// total_out (device, nullable) receives the reduction of all n items.  in2 /
// out2 (nullable): a second array of n items scanned the same way, same launch.
template <class T, class Op>
cudaError_t device_scan(const T* in, T* out, int64_t n, bool reverse, bool exclusive, T* tmp, T* total_out,
                        cudaStream_t s, const T* in2 = nullptr, T* out2 = nullptr) {
    if (n <= 0) return cudaSuccess;
    const int64_t nb = (n + SCAN_BLK - 1) / SCAN_BLK;
    const dim3 grid((unsigned)nb, in2 ? 2u : 1u);
    launch_k(scan_onepass_kernel<T, Op>, grid, SCAN_THREADS, 0, s, in, out, n, (int)reverse, (int)exclusive, total_out,
             reinterpret_cast<unsigned long long*>(tmp), scan_next_epoch(), in2, out2);
    launch_counter()++;
    return cudaGetLastError();
}

template <class T, class Op>
cudaError_t device_scan2(const T* in, T* out, const T* in2, T* out2, int64_t n, bool reverse, bool exclusive, T* tmp,
                         cudaStream_t s) {
    return device_scan<T, Op>(in, out, n, reverse, exclusive, tmp, nullptr, s, in2, out2);
}

}  // namespace ps

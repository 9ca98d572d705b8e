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

template <class T, class Op>
__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const T* __restrict__ in, T* __restrict__ partial,
                                                                   int64_t n, int reverse) {
    pdl_wait();
    __shared__ T sw[32];
    Op op;
    const int64_t base = (int64_t)blockIdx.x * SCAN_BLK;
    T acc = Op::id();
    for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
        int64_t g = base + i;
        if (g < n) acc = op(acc, in[reverse ? n - 1 - g : g]);
    }
    T total;
    block_exclusive<T, Op>(acc, total, sw);
    if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

template <class T, class Op>
__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(const T* in, T* out, int64_t n,
                                                                  const T* __restrict__ carry, int reverse,
                                                                  int exclusive, T* total_out) {
    pdl_wait();
    __shared__ T items[SCAN_BLK];
    __shared__ T sw[32];
    Op op;
    const int64_t base = (int64_t)blockIdx.x * SCAN_BLK;
    for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
        int64_t g = base + i;
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
    T c = carry ? carry[blockIdx.x] : Op::id();
    pre = op(c, pre);
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        T inc = op(pre, loc[j]);
        items[threadIdx.x * SCAN_ITEMS + j] = exclusive ? pre : inc;
        pre = inc;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
        int64_t g = base + i;
        if (g < n) out[reverse ? n - 1 - g : g] = items[i];
    }
    if (total_out && threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) *total_out = op(c, total);
}

// Small n: one CTA walks the tiles in order with a running carry (one launch
// instead of reduce + recursive scan + apply).
constexpr int64_t SCAN_SEQ_MAX = 8 * SCAN_BLK;

template <class T, class Op>
__global__ void __launch_bounds__(SCAN_THREADS) scan_seq_kernel(const T* in, T* out, int64_t n, int reverse,
                                                                int exclusive, T* total_out, const T* in2, T* out2) {
    pdl_wait();
    if (blockIdx.x == 1) {  // a second, independent array of the same length (one launch for both)
        in = in2;
        out = out2;
        total_out = nullptr;
    }
    __shared__ T items[SCAN_BLK];
    __shared__ T sw[32];
    Op op;
    T carry = Op::id();
    for (int64_t base = 0; base < n; base += SCAN_BLK) {
        for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
            int64_t g = base + i;
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
        T pre = op(carry, block_exclusive<T, Op>(acc, total, sw));
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; ++j) {
            T inc = op(pre, loc[j]);
            items[threadIdx.x * SCAN_ITEMS + j] = exclusive ? pre : inc;
            pre = inc;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < SCAN_BLK; i += SCAN_THREADS) {
            int64_t g = base + i;
            if (g < n) out[reverse ? n - 1 - g : g] = items[i];
        }
        carry = op(carry, total);
        __syncthreads();
    }
    if (total_out && threadIdx.x == 0) *total_out = carry;
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

// Two independent arrays of n items each, scanned the same way; one launch when
// small.  tmp as for device_scan.
template <class T, class Op>
cudaError_t device_scan2(const T* in, T* out, const T* in2, T* out2, int64_t n, bool reverse, bool exclusive, T* tmp,
                         cudaStream_t s);

// Elements of temporary storage device_scan needs for n items.
inline int64_t scan_tmp_elems(int64_t n) {
    int64_t t = 0;
    while (n > SCAN_BLK) {
        n = (n + SCAN_BLK - 1) / SCAN_BLK;
        t += n + 32;
    }
    return t + 64;
}

// out may alias in.  tmp: scan_tmp_elems(n) elements.  total_out (device,
// nullable) receives the reduction of all n items.
template <class T, class Op>
cudaError_t device_scan(const T* in, T* out, int64_t n, bool reverse, bool exclusive, T* tmp, T* total_out,
                        cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t nb = (n + SCAN_BLK - 1) / SCAN_BLK;
    if (n <= SCAN_SEQ_MAX) {
        launch_k(scan_seq_kernel<T, Op>, 1, SCAN_THREADS, 0, s, in, out, n, (int)reverse, (int)exclusive, total_out,
                 (const T*)nullptr, (T*)nullptr);
        launch_counter()++;
        return cudaGetLastError();
    }
    T* partial = tmp;
    T* rest = tmp + nb + 32;
    launch_k(scan_reduce_kernel<T, Op>, (unsigned)nb, SCAN_THREADS, 0, s, in, partial, n, reverse);
    launch_counter() += 2;
    cudaError_t e = device_scan<T, Op>(partial, partial, nb, false, true, rest, nullptr, s);
    if (e != cudaSuccess) return e;
    launch_k(scan_apply_kernel<T, Op>, (unsigned)nb, SCAN_THREADS, 0, s, in, out, n, partial, reverse, exclusive,
                                                                    total_out);
    return cudaGetLastError();
}

template <class T, class Op>
cudaError_t device_scan2(const T* in, T* out, const T* in2, T* out2, int64_t n, bool reverse, bool exclusive, T* tmp,
                         cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (n <= SCAN_SEQ_MAX) {
        launch_k(scan_seq_kernel<T, Op>, 2, SCAN_THREADS, 0, s, in, out, n, (int)reverse, (int)exclusive, (T*)nullptr,
                 in2, out2);
        launch_counter()++;
        return cudaGetLastError();
    }
    cudaError_t e = device_scan<T, Op>(in, out, n, reverse, exclusive, tmp, nullptr, s);
    if (e != cudaSuccess) return e;
    return device_scan<T, Op>(in2, out2, n, reverse, exclusive, tmp, nullptr, s);
}

}  // namespace ps

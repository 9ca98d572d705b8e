// Microbenchmark of the in-shared-memory merge-path loop used by
// merge_pipe_kernel (diagnostics only, not part of the library).
// Each CTA holds two sorted SoA windows of N/2 keys+values in smem and merges
// them into padded records, `reps` times; prints cycles per record per CTA.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "../paper_2209_06909_b200/csrc/ps_merge.cuh"

using namespace ps;

template <int NT, int N>
__global__ void __launch_bounds__(NT) bench_kernel(const int* __restrict__ gk, int reps, unsigned long long* cyc,
                                                   int mode) {
    extern __shared__ __align__(16) uint8_t smem[];
    int* ak = reinterpret_cast<int*>(smem);
    int* bk = ak + N / 2;
    int* av = bk + N / 2;
    int* bv = av + N / 2;
    Rec<int>* out = reinterpret_cast<Rec<int>*>(bv + N / 2);
    for (int i = threadIdx.x; i < N / 2; i += NT) {
        ak[i] = gk[i];
        bk[i] = gk[2304 + i];
        av[i] = i;
        bv[i] = N / 2 + i;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const uint32_t t = threadIdx.x;
        WinCur<int> c;
        c.ak = ak;
        c.bk = bk;
        c.av = av;
        c.bv = bv;
        c.la = N / 2;
        c.lb = N / 2;
        c.o = (uint32_t)((uint64_t)N * t / NT);
        c.oe = (uint32_t)((uint64_t)N * (t + 1) / NT);
        c.base = 0;
        if (mode == 0) {
            single_merge(c, out);
        } else {
            // search only
            uint32_t lo = c.o > c.lb ? c.o - c.lb : 0, hi = c.o < c.la ? c.o : c.la;
            while (lo < hi) {
                const uint32_t m = (lo + hi) >> 1;
                const bool le = !(c.keyB(c.o - 1 - m) < c.keyA(m));
                lo = le ? m + 1 : lo;
                hi = le ? hi : m;
            }
            if (lo == 0xFFFFFFFF) out[0].k = lo;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}

// composite u64 records: one LDS.64 per head, 64-bit compares
template <int NT, int N>
__global__ void __launch_bounds__(NT) bench64_kernel(const int* __restrict__ gk, int reps, unsigned long long* cyc) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* A = reinterpret_cast<uint64_t*>(smem);
    uint64_t* B = A + N / 2;
    uint64_t* out = B + N / 2;
    for (int i = threadIdx.x; i < N / 2; i += NT) {
        A[i] = ((uint64_t)(uint32_t)gk[i] << 32) | (uint32_t)i;
        B[i] = ((uint64_t)(uint32_t)gk[2304 + i] << 32) | (uint32_t)(N / 2 + i);
    }
    __syncthreads();
    long long t0 = clock64();
    const uint32_t la = N / 2, lb = N / 2;
    for (int r = 0; r < reps; ++r) {
        const uint32_t t = threadIdx.x;
        const uint32_t o0 = (uint32_t)((uint64_t)N * t / NT), o1 = (uint32_t)((uint64_t)N * (t + 1) / NT);
        uint32_t lo = o0 > lb ? o0 - lb : 0, hi = o0 < la ? o0 : la;
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            const bool le = A[m] < B[o0 - 1 - m];
            lo = le ? m + 1 : lo;
            hi = le ? hi : m;
        }
        uint32_t i = lo, j = o0 - lo;
        uint64_t a = A[i < la ? i : la - 1], b = B[j < lb ? j : lb - 1];
#pragma unroll 4
        for (uint32_t o = o0; o < o1; ++o) {
            const bool takeA = i < la && (j >= lb || a < b);
            out[padr<int>(o)] = takeA ? a : b;
            i += takeA;
            j += !takeA;
            const uint64_t nx = takeA ? A[i < la ? i : la - 1] : B[j < lb ? j : lb - 1];
            a = takeA ? nx : a;
            b = takeA ? b : nx;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}

template <int NT, int N>
void run64(const int* dk, int blocks) {
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    cudaMemset(dc, 0, 8);
    size_t smem = N * 8 + (N + N / 8 + 16) * 8;
    cudaFuncSetAttribute(bench64_kernel<NT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 200;
    bench64_kernel<NT, N><<<blocks, NT, smem>>>(dk, reps, dc);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    double per_cta_rep = (double)c / blocks / reps;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bench64_kernel<NT, N>, NT, smem);
    printf("u64  NT %4d N %5d blocks %5d occ %d : %8.0f cycles/rep/CTA  %.3f cycles/record/CTA  err=%s\n", NT, N,
           blocks, occ, per_cta_rep, per_cta_rep / N, cudaGetErrorString(cudaGetLastError()));
    cudaFree(dc);
}

template <int NT, int N>
void run(const int* dk, int blocks, int mode) {
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    cudaMemset(dc, 0, 8);
    size_t smem = N * 4 * 2 + (N + N / 8 + 16) * 8;
    cudaFuncSetAttribute(bench_kernel<NT, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int reps = 200;
    bench_kernel<NT, N><<<blocks, NT, smem>>>(dk, reps, dc, mode);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    double per_cta_rep = (double)c / blocks / reps;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bench_kernel<NT, N>, NT, smem);
    printf("mode %d NT %4d N %5d blocks %5d occ %d : %8.0f cycles/rep/CTA  %.3f cycles/record/CTA  err=%s\n", mode,
           NT, N, blocks, occ, per_cta_rep, per_cta_rep / N, cudaGetErrorString(cudaGetLastError()));
    cudaFree(dc);
}

int main() {
    const int N = 8192;
    std::vector<int> h(N);
    srand(1);
    for (int i = 0; i < N; ++i) h[i] = rand();
    std::sort(h.begin(), h.begin() + 2304);
    std::sort(h.begin() + 2304, h.begin() + 4608);
    int* dk;
    cudaMalloc(&dk, N * 4);
    cudaMemcpy(dk, h.data(), N * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 1; ++mode) {
        run<256, 4096>(dk, 148 * 2, mode);   // VT 16
        run<256, 4352>(dk, 148 * 2, mode);   // VT 17
        run<256, 3840>(dk, 148 * 2, mode);   // VT 15
        run<256, 3328>(dk, 148 * 2, mode);   // VT 13
        run<128, 4352>(dk, 148 * 2, mode);   // VT 34
        run<128, 4224>(dk, 148 * 2, mode);   // VT 33
        run<512, 4608>(dk, 148 * 2, mode);   // VT 9
    }
    run64<256, 4096>(dk, 148 * 2);
    run64<256, 4096>(dk, 148 * 3);
    run64<512, 4096>(dk, 148 * 2);
    run64<128, 4096>(dk, 148 * 2);
    return 0;
}

// Microbenchmark (tooling, not product): tcgen05.ld throughput per SM.
// W warps (W/4 per TMEM lane quadrant) each issue `iters` rounds of four
// 32x32b.x32 loads (4 KB each, 16 KB per round) and one wait; cycles by
// clock64 around the loop. Prints bytes/cycle/SM for W = 4, 8, 16.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2411_15871_b200/csrc/cuda -I include tools/micro/tmem_bw.cu -o /tmp/tmem_bw -lcuda
#include <cstdio>

#include "common.cuh"

using namespace dh;

__global__ void tmem_read(int iters, long long* cycles, unsigned* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col0 = ((warp >> 2) * 128) & 511;
    unsigned acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t a[32], b[32], c[32], d[32];
        tmem_ld32(tmem + lane_off + col0, a);
        tmem_ld32(tmem + lane_off + col0 + 32, b);
        tmem_ld32(tmem + lane_off + col0 + 64, c);
        tmem_ld32(tmem + lane_off + col0 + 96, d);
        tmem_ld_wait();
        // static indices only (a dynamic index would put the arrays in local memory)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= a[j] + b[j] + c[j] + d[j];
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main() {
    long long* cyc;
    unsigned* sink;
    cudaMalloc(&cyc, 148 * sizeof(long long));
    cudaMalloc(&sink, 148 * 1024 * sizeof(unsigned));
    const int iters = 4096;
    for (int w : {4, 8, 16}) {
        tmem_read<<<148, 32 * w>>>(iters, cyc, sink);
        tmem_read<<<148, 32 * w>>>(iters, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (long long x : h) mx = x > mx ? x : mx;
        const double bytes = static_cast<double>(w) * iters * 4 * 4096;
        std::printf("warps %2d: %s  %.1f bytes/cycle/SM (%lld cycles)\n", w, cudaGetErrorString(e), bytes / mx,
                    static_cast<long long>(mx));
    }
    return 0;
}

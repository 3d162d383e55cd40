// Microbenchmark (tooling, not product): RMSNorm forward / backward kernel
// variants of csrc/cuda/elementwise.cu at the Llama-3-8B row width (4096) for
// the TP=1 (4096 rows) and TP=8 (512 rows) shapes; each variant launched 50x
// back to back between CUDA events after warm-up (warm L2 as in the step).
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I include \
//        -I paper_2411_15871_b200/csrc/cuda tools/micro/rmsnorm_var.cu \
//        paper_2411_15871_b200/csrc/cuda/errors.cu -o tools/micro/rmsnorm_var -lcuda
#include "../../paper_2411_15871_b200/csrc/cuda/elementwise.cu"

#include <cstdio>
#include <functional>

using namespace dh;

static float time_us(const std::function<void()>& f, int n = 50) {
    for (int i = 0; i < 5; ++i) f();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < n; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / n;
}

int main() {
    const int cols = 4096, vc = cols / 8;
    for (int rows : {4096, 512}) {
        const size_t n = static_cast<size_t>(rows) * cols;
        uint4 *x, *y, *dy, *dx, *g, *res;
        float *rstd, *dg;
        cudaMalloc(&x, n * 2);
        cudaMalloc(&y, n * 2);
        cudaMalloc(&dy, n * 2);
        cudaMalloc(&dx, n * 2);
        cudaMalloc(&res, n * 2);
        cudaMalloc(&g, cols * 2);
        cudaMalloc(&rstd, rows * 4);
        cudaMalloc(&dg, cols * 4);
        cudaMemset(x, 0x3c, n * 2);
        cudaMemset(dy, 0x3c, n * 2);
        cudaMemset(res, 0x3c, n * 2);
        cudaMemset(g, 0x3c, cols * 2);
        cudaMemset(dg, 0, cols * 4);
        const float ic = 1.f / cols, eps = 1e-5f;
        const double mb2 = 2.0 * n * 2 / 1e6, mb3 = 1.5 * mb2;
        auto rep = [&](const char* name, double mb, float us) {
            printf("rows %4d %-34s %7.2f us %6.0f GB/s\n", rows, name, us, mb * 1e3 / us);
        };
        rep("fwd split<4,128,2> (current)", mb2, time_us([&] {
                rmsnorm_fwd_split<4, 128, 2><<<(rows + 1) / 2, 256>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd split<4,128,4>", mb2, time_us([&] {
                rmsnorm_fwd_split<4, 128, 4><<<(rows + 3) / 4, 512>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd split<4,128,1>", mb2, time_us([&] {
                rmsnorm_fwd_split<4, 128, 1><<<rows, 128>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd split<2,256,1>", mb2, time_us([&] {
                rmsnorm_fwd_split<2, 256, 1><<<rows, 256>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd split<8,64,2>", mb2, time_us([&] {
                rmsnorm_fwd_split<8, 64, 2><<<(rows + 1) / 2, 128>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd split<8,64,4>", mb2, time_us([&] {
                rmsnorm_fwd_split<8, 64, 4><<<(rows + 3) / 4, 256>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("fwd reg-warp<16> (1 warp/row)", mb2, time_us([&] {
                rmsnorm_fwd_split<16, 32, 8><<<(rows + 7) / 8, 256>>>(x, g, y, rstd, rows, ic, eps);
            }));
        rep("add+fwd split<4,128,2> (current)", 2 * mb2, time_us([&] {
                rmsnorm_fwd_split<4, 128, 2><<<(rows + 1) / 2, 256>>>(x, g, y, rstd, rows, ic, eps, res, dx);
            }));
        rep("add+fwd split<2,256,1>", 2 * mb2, time_us([&] {
                rmsnorm_fwd_split<2, 256, 1><<<rows, 256>>>(x, g, y, rstd, rows, ic, eps, res, dx);
            }));
        auto bwd = [&](auto kern, int cv, int rpb) {
            const int n_dg = cols / (8 * cv);
            return time_us([&] {
                kern<<<n_dg + (rows + rpb - 1) / rpb, vc>>>(x, g, rstd, dy, res, dx, dg, rows, vc, ic, n_dg);
            });
        };
        rep("bwd fused<8,4,1> (current)", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<8, 4, 1>, 8, 1));
        rep("bwd fused<8,8,1>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<8, 8, 1>, 8, 1));
        rep("bwd fused<8,4,2>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<8, 4, 2>, 8, 2));
        rep("bwd fused<8,8,2>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<8, 8, 2>, 8, 2));
        rep("bwd fused<8,8,4>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<8, 8, 4>, 8, 4));
        rep("bwd fused<4,8,2>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<4, 8, 2>, 4, 2));
        rep("bwd fused<16,8,2>", mb3 + mb2 / 2, bwd(rmsnorm_bwd_fused<16, 8, 2>, 16, 2));
        rep("bwd dx rows only <8,4,1>", mb3 + mb2 / 2, time_us([&] {
                rmsnorm_bwd_fused<8, 4, 1><<<64 + rows, vc>>>(x, g, rstd, dy, res, dx, nullptr, rows, vc, ic, 64);
            }));
        rep("bwd dx rows only <8,4,2>", mb3 + mb2 / 2, time_us([&] {
                rmsnorm_bwd_fused<8, 4, 2><<<64 + rows / 2, vc>>>(x, g, rstd, dy, res, dx, nullptr, rows, vc, ic, 64);
            }));
        {  // RoPE over the q and k heads of the fused qkv rows (TP=1: 32 + 8 heads, TP=8: 4 + 1)
            const int heads = rows == 4096 ? 40 : 5, D = 128, ldq = (heads + (rows == 4096 ? 8 : 1)) * D;
            __nv_bfloat16* qkv;
            cudaMalloc(&qkv, static_cast<size_t>(rows) * ldq * 2);
            cudaMemset(qkv, 0x3c, static_cast<size_t>(rows) * ldq * 2);
            const double mb = 2.0 * rows * heads * D * 2 / 1e6, lt = std::log(500000.0);
            rep("rope", mb, time_us([&] { rope_vec_kernel<<<rows, 128>>>(qkv, ldq, rows, heads, D, lt, 0, 1.f); }));
            cudaFree(qkv);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
        cudaFree(x); cudaFree(y); cudaFree(dy); cudaFree(dx); cudaFree(res); cudaFree(g); cudaFree(rstd); cudaFree(dg);
    }
    return 0;
}

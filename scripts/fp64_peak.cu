// FP64 throughput microbenchmark for the roofline denominators:
//   dfma  : independent DFMA chains, 8 per thread, enough warps to fill every SM
//   dmma  : legacy warp MMA m8n8k4 f64 (mma.sync), to see whether the FP64 tensor path adds throughput
//   both  : half the warps on each in the same kernel (co-issue test)
//   ffma  : the same chains in fp32 (fp32 mode's ALU roof)
// Timed with CUDA events over a launch long enough (>= 200 ms) for the clocks to settle.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b, int reps) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 64
        for (int i = 0; i < ITERS; ++i) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ffma(double* out, double a, double b, int reps) {
    const float af = (float)a, bf = (float)b;
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 64
        for (int i = 0; i < ITERS; ++i) {
            x0 = fmaf(x0, af, bf); x1 = fmaf(x1, af, bf); x2 = fmaf(x2, af, bf); x3 = fmaf(x3, af, bf);
            x4 = fmaf(x4, af, bf); x5 = fmaf(x5, af, bf); x6 = fmaf(x6, af, bf); x7 = fmaf(x7, af, bf);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ffma2(double* out, double a, double b, int reps) {
    const float2 af = make_float2((float)a, (float)a), bf = make_float2((float)b, (float)b);
    float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
    for (int r = 0; r < reps; ++r) {
#pragma unroll 64
        for (int i = 0; i < ITERS; ++i) {
            x0 = __ffma2_rn(x0, af, bf); x1 = __ffma2_rn(x1, af, bf); x2 = __ffma2_rn(x2, af, bf); x3 = __ffma2_rn(x3, af, bf);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x1.x + x2.x + x3.x + x0.y + x1.y + x2.y + x3.y;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, double a, double b, int reps) {
    double c0[2] = {0, 0}, c1[2] = {1, 0}, c2[2] = {2, 0}, c3[2] = {3, 0};
    const double av = a * (threadIdx.x & 3), bv = b;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 16
        for (int i = 0; i < ITERS / 4; ++i) {
            dmma(c0, av, bv); dmma(c1, av, bv); dmma(c2, av, bv); dmma(c3, av, bv);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
}

__global__ void k_both(double* out, double a, double b, int reps) {
    if ((threadIdx.x >> 5) & 1) {
        double c0[2] = {0, 0}, c1[2] = {1, 0}, c2[2] = {2, 0}, c3[2] = {3, 0};
        for (int r = 0; r < reps; ++r) {
#pragma unroll 16
            for (int i = 0; i < ITERS / 4; ++i) {
                dmma(c0, a, b); dmma(c1, a, b); dmma(c2, a, b); dmma(c3, a, b);
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = c0[0] + c1[0] + c2[0] + c3[0] + c0[1] + c1[1] + c2[1] + c3[1];
    } else {
        double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
        for (int r = 0; r < reps; ++r) {
#pragma unroll 64
            for (int i = 0; i < ITERS; ++i) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    }
}

int main(int argc, char** argv) {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256, blocks = nsm * 8;
    double* out;
    cudaMalloc(&out, sizeof(double) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double a = 0.999999, b = 1e-7;
    auto run = [&](const char* name, void (*k)(double*, double, double, int), double flop_per_rep_thread, int reps) {
        k<<<blocks, threads>>>(out, a, b, 1);   // warm-up
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(e0);
            k<<<blocks, threads>>>(out, a, b, reps);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double flops = flop_per_rep_thread * reps * (double)threads * blocks;
        printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.3f, \"blocks\": %d, \"threads\": %d, \"sms\": %d}\n", name,
               best, flops / (best * 1e-3) / 1e12, blocks, threads, nsm);
        fflush(stdout);
    };
    const int reps = argc > 1 ? atoi(argv[1]) : 24;
    // dfma: 8 chains x ITERS FMAs x 2 flops per thread
    run("dfma", k_dfma, 8.0 * ITERS * 2.0, reps);
    // dmma m8n8k4: 2*8*8*4 = 512 flops per warp-instruction = 16 per thread; 4 x ITERS/4 per rep
    run("dmma_m8n8k4", k_dmma, 16.0 * ITERS, reps);
    // both: half the threads each (counted at their own rates)
    run("dfma+dmma (half the warps each)", k_both, 0.5 * (8.0 * ITERS * 2.0) + 0.5 * (16.0 * ITERS), reps);
    // ffma: fp32 mode's ALU roof (same chains in fp32)
    run("ffma", k_ffma, 8.0 * ITERS * 2.0, reps * 2);
    run("ffma2 (packed fp32x2)", k_ffma2, 8.0 * ITERS * 2.0, reps * 2);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}

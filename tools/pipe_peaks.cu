// pipe_peaks.cu -- SURVEY §7 step 1: measured per-SM throughput of the pipes the ALU-bound
// kernels' rooflines divide by (MUFU sin/cos, FP32 FMA, integer VABSDIFF4 and LOP3, IMAD, FP64
// DFMA).  Each kernel runs 8 independent dependency chains per thread over a grid of 8 blocks x
// 256 threads per SM, so the pipe, not latency, is the bound; the host reports warp-lane
// operations per SM clock (the SM clock from %clock64 deltas inside the kernel).
// Build + run: tools/pipe_peaks.sh (nvcc on the GPU box).  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

__device__ unsigned long long g_cycles[1024];

template <int OP>
__global__ void __launch_bounds__(256) k_pipe(float* out, uint32_t* iout, double* dout, float seed) {
    const unsigned long long c0 = clock64();
    const uint32_t mul = 2654435761u + (uint32_t)(seed * 1000.0f);   // run-time: no affine folding
    float f[kChains];
    uint32_t u[kChains];
    double d[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        f[c] = seed + threadIdx.x * 1e-3f + c;
        u[c] = threadIdx.x * 2654435761u + c;
        d[c] = seed + c;
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == 0) {            // MUFU: one sin + one cos (2 MUFU ops)
                float s, co;
                __sincosf(f[c], &s, &co);
                f[c] = s + co;
            } else if (OP == 1) {     // FFMA
                f[c] = fmaf(f[c], 1.0001f, 0.5f);
            } else if (OP == 2) {     // VABSDIFF4 (integer ALU pipe)
                uint32_t r;
                asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(r) : "r"(u[c]), "r"(0x01020304u), "r"(u[c]));
                u[c] = r;
            } else if (OP == 3) {     // LOP3 (integer ALU pipe)
                uint32_t r;
                asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(u[c]), "r"(0x9E3779B9u), "r"(u[(c + 1) % kChains]));
                u[c] = r;
            } else if (OP == 4) {     // IMAD
                u[c] = u[c] * mul + 12345u;
            } else {                  // DFMA
                d[c] = fma(d[c], 1.0001, 0.5);
            }
        }
    }
    float fs = 0.f;
    uint32_t us = 0;
    double ds = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        fs += f[c];
        us ^= u[c];
        ds += d[c];
    }
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    out[t] = fs;
    iout[t] = us;
    dout[t] = ds;
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_cycles[blockIdx.x] = clock64() - c0;
}

template <int OP>
double run(const char* name, double ops_per_iter_chain, int n_sm, float* o, uint32_t* io, double* dd) {
    const int blocks = 8 * n_sm;
    k_pipe<OP><<<blocks, 256>>>(o, io, dd, 0.25f);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_pipe<OP><<<blocks, 256>>>(o, io, dd, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc[1024];
    cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(cyc));
    double cmax = 0.0;
    for (int i = 0; i < blocks && i < 1024; ++i) cmax = cyc[i] > cmax ? (double)cyc[i] : cmax;
    const double ops = (double)blocks * 256 * kIters * kChains * ops_per_iter_chain;
    const double sm_mhz = cmax / (ms * 1e3);            // block cycles over the kernel's time
    const double per_clk_sm = ops / (ms * 1e-3) / (sm_mhz * 1e6) / n_sm;
    std::printf("  \"%s\": {\"ms\": %.4f, \"ops\": %.6e, \"sm_mhz\": %.1f, \"lane_ops_per_clk_per_sm\": %.2f},\n",
                name, ms, ops, sm_mhz, per_clk_sm);
    return per_clk_sm;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int n_sm = p.multiProcessorCount, n = 8 * n_sm * 256;
    float* o;
    uint32_t* io;
    double* dd;
    cudaMalloc(&o, n * sizeof(float));
    cudaMalloc(&io, n * sizeof(uint32_t));
    cudaMalloc(&dd, n * sizeof(double));
    std::printf("{\n  \"device\": \"%s\", \"n_sm\": %d,\n", p.name, n_sm);
    run<0>("mufu_sincos", 2.0, n_sm, o, io, dd);
    run<1>("ffma", 1.0, n_sm, o, io, dd);
    run<2>("vabsdiff4", 1.0, n_sm, o, io, dd);
    run<3>("lop3", 1.0, n_sm, o, io, dd);
    run<4>("imad", 1.0, n_sm, o, io, dd);
    run<5>("dfma", 1.0, n_sm, o, io, dd);
    std::printf("  \"how\": \"8 independent chains per thread, 8 x 256-thread blocks per SM, %d iterations; lane ops per SM clock from events + clock64\"\n}\n", kIters);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}

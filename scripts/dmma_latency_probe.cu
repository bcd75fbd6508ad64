// DMMA.8x8x4 latency and per-SM throughput vs (warps per SM, independent chains per warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dlp scripts/dmma_latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(int iters, double *out, long long *cyc) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[CH][2];
    for (int t = 0; t < CH; ++t) c[t][0] = c[t][1] = t;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < CH; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1])
                         : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0;
    for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
    if (s == 42.0) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run(int warps_per_sm, int sms, double *out, long long *cyc) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<CH><<<sms, 32 * warps_per_sm>>>(16, out, cyc);
    cudaEventRecord(e0);
    chains<CH><<<sms, 32 * warps_per_sm>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double fl = 512.0 * CH * iters * warps_per_sm * sms;
    printf("warps/SM %2d chains %d : %6.1f TF  %.2f clk/dmma/warp-chain\n", warps_per_sm, CH,
           fl / ms / 1e9, double(h) / iters);
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1 << 16);
    cudaMalloc(&cyc, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {1, 4, 8, 12, 16, 32}) {
        run<1>(w, sms, out, cyc);
        run<2>(w, sms, out, cyc);
        run<4>(w, sms, out, cyc);
        run<8>(w, sms, out, cyc);
    }
}

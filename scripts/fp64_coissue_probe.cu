// Does FP64 DFMA (CUDA-core pipe) run concurrently with DMMA (tensor pipe) on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0 dmma only, 1 dfma only, 2 both interleaved
__global__ void probe(int iters, double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2]; double f[8];
    for (int t = 0; t < 8; ++t) { c[t][0] = c[t][1] = 0; f[t] = t; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            if (MODE != 1)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
            if (MODE != 0) {
#pragma unroll
                for (int u = 0; u < 8; ++u) f[u] = fma(f[u], 0.9999999, 1e-9);
            }
        }
    }
    double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + f[t];
    if (s == 42.0) out[threadIdx.x] = s;
}
int main() {
    double* out; cudaMalloc(&out, 8192);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 2, threads = 512, iters = 2048;
    float ms[3];
    void (*k[3])(int, double*) = {probe<0>, probe<1>, probe<2>};
    for (int m = 0; m < 3; ++m) {
        k[m]<<<blocks, threads>>>(8, out);
        cudaEventRecord(e0); k[m]<<<blocks, threads>>>(iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms[m], e0, e1);
    }
    double warps = blocks * threads / 32.0;
    double dmma_fl = 2.0 * 256 * 8 * iters * warps, dfma_fl = 2.0 * 32 * 64 * iters * warps;
    printf("dmma only: %.1f TF  (%.2f ms)\n", dmma_fl / ms[0] / 1e9, ms[0]);
    printf("dfma only: %.1f TF  (%.2f ms)\n", dfma_fl / ms[1] / 1e9, ms[1]);
    printf("both:      %.1f TF  combined (%.2f ms; serial would be %.2f ms)\n", (dmma_fl + dfma_fl) / ms[2] / 1e9, ms[2], ms[0] + ms[1]);
}

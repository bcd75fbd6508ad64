#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_probe(int iters, double* out) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    if (s == 42.0) out[threadIdx.x] = s;
}
__global__ void dfma_probe(int iters, double* out) {
    double a[8]; for (int t=0;t<8;++t) a[t]=threadIdx.x+t;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u=0;u<16;++u) for (int t=0;t<8;++t) a[t]=fma(a[t],0.999999,1e-9);
    double s=0; for(int t=0;t<8;++t) s+=a[t]; if (s==42.0) out[threadIdx.x]=s;
}
int main() {
    double* out; cudaMalloc(&out, 1024*8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int wpb : {4, 8, 16}) {
      int blocks = sms*2, iters=4096;
      dmma_probe<<<blocks, wpb*32>>>(16, out);
      cudaEventRecord(e0); dmma_probe<<<blocks, wpb*32>>>(iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double fl = 2.0*256*8*(double)iters*blocks*wpb; 
      printf("DMMA m8n8k4 warps/blk %d: %.2f TFLOP/s  (%s)\n", wpb, fl/ms/1e9, cudaGetErrorString(cudaGetLastError()));
    }
    int blocks=sms*8, iters=2048;
    dfma_probe<<<blocks,256>>>(16,out);
    cudaEventRecord(e0); dfma_probe<<<blocks,256>>>(iters,out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    printf("DFMA: %.2f TFLOP/s\n", 2.0*8*16*(double)iters*blocks*256/ms/1e9);
}

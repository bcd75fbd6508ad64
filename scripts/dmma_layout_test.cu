// Verifies the mma.sync.m8n8k4 f64 fragment layout assumed by coal_dmma.cuh.
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
    int l = threadIdx.x;
    double a = A[(l >> 2) * 4 + (l & 3)];      // A[row=l/4][col=l%4]  (8x4 row-major)
    double b = B[(l & 3) * 8 + (l >> 2)];      // B[row=l%4][col=l/4]  (4x8)
    double c0 = 0, c1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[(l >> 2) * 8 + 2 * (l & 3)] = c0;        // C[row=l/4][col=2*(l%4)+{0,1}]
    C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1 + i * 0.37; hB[i] = 2 - i * 0.11; }
    for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
        double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c]; ref[r * 8 + c] = s; }
    double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC); cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
    printf("dmma layout max err %g -> %s\n", err, err < 1e-12 ? "LAYOUT OK" : "LAYOUT MISMATCH");
}

// Latency of the A4 epilogue math (eig3_sym + regularize) on one thread, in SM clocks:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/eig_latency.cu -o tools/eig_latency
#include <cstdio>
#include "../paper_2403_12550_b200/csrc/gsicp_internal.cuh"
using namespace gsicp;
__global__ void k(double *io, long long *cyc, int reps) {
    double A[6] = {io[0], io[1], io[2], io[3], io[4], io[5]};
    double acc = 0.0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        A[0] += acc * 1e-30;  // serial dependency between repetitions
        const Eig3 e = eig3_sym(A);
        double R[6];
        regularize(A, e, GSICP_REG_ELLIPSE, 1e-3, R);
        acc = R[0] + e.lam[0];
    }
    const long long t1 = clock64();
    io[6] = acc;
    cyc[0] = (t1 - t0) / reps;
}
int main() {
    double h[7] = {2.0e-4, 3e-5, -1e-5, 1.5e-4, 2e-6, 1e-6, 0};
    double *d;
    long long *c, hc;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&c, sizeof(long long));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    k<<<1, 1>>>(d, c, 10);
    k<<<1, 1>>>(d, c, 100);
    cudaMemcpy(&hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
    printf("eig3_sym + regularize: %lld cycles per call (one thread)\n", hc);
    return 0;
}

// Dev micro-benchmark: dependent fp64 add chain latency on B200 (sets the floor of the
// exact sequential signal_std: one dependent add per sample and pass).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* x, int n, double* out, long long* cyc) {
    double s = 0.0;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) s += x[i & 1023];
    long long t1 = clock64();
    out[0] = s;
    cyc[0] = t1 - t0;
}
__global__ void chain_smem(const double* x, int n, double* out, long long* cyc) {
    __shared__ double b[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) b[i] = x[i];
    __syncthreads();
    if (threadIdx.x) return;
    double s = 0.0;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) s += b[i & 1023];
    long long t1 = clock64();
    out[0] = s;
    cyc[0] = t1 - t0;
}
int main() {
    double *x, *o; long long* c;
    cudaMalloc(&x, 8192 * 8); cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    cudaMemset(x, 0, 8192 * 8);
    const int n = 1 << 20;
    long long h;
    chain<<<1, 1>>>(x, n, o, c); cudaDeviceSynchronize();
    chain<<<1, 1>>>(x, n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("global-fed chain: %.2f cycles/add\n", (double)h / n);
    chain_smem<<<1, 32>>>(x, n, o, c); cudaDeviceSynchronize();
    chain_smem<<<1, 32>>>(x, n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("smem-fed chain: %.2f cycles/add\n", (double)h / n);
    return 0;
}

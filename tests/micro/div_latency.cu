// Dev micro-benchmark: latency of the forward-sweep row d' = c - (h/d)*h (emd.cpp:64-69) with
// IEEE division vs a division seeded by the fp32 reciprocal (2 fp64 Newton steps + the same
// final correction), and a check that the seeded division equals IEEE on many operands.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_seeded(double a, double b) {
    const float bf = (float)b;
    double y = (double)__frcp_rn(bf);          // ~24 bits
    double e = fma(-b, y, 1.0);
    y = fma(y, e, y);                          // ~48 bits
    e = fma(-b, y, 1.0);
    y = fma(y, e, y);                          // ~full
    const double q = a * y;
    const double r = fma(-b, q, a);
    return fma(y, r, q);
}

__global__ void chain(int n, double h, double c, double* out, long long* cyc, int mode) {
    double d = c + threadIdx.x * 1e-3;
    const long long t0 = clock64();
    if (mode == 0) {
#pragma unroll 4
        for (int i = 0; i < n; ++i) d = c - (h / d) * h;
    } else if (mode == 1) {
#pragma unroll 4
        for (int i = 0; i < n; ++i) d = c - div_seeded(h, d) * h;
    } else {
#pragma unroll 4
        for (int i = 0; i < n; ++i) d = c - (h * d) * h;  // no division: dmul+dadd chain
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = d;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void check(unsigned long long seed, long long n, unsigned long long* bad) {
    unsigned long long s = seed + blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    for (long long i = 0; i < n; ++i) {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        const double a = (double)((s >> 40) & 0xFFFF) + 1.0;                 // small integer numerator (h)
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        const double b = __longlong_as_double((long long)(0x3FF0000000000000ULL | (s >> 12))) * (double)((s >> 2) & 0xFFF);
        if (b == 0.0) continue;
        if (__double_as_longlong(a / b) != __double_as_longlong(div_seeded(a, b))) ++nb;
    }
    atomicAdd(bad, nb);
}

int main() {
    double* o; long long* c; unsigned long long* bad;
    cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8); cudaMalloc(&bad, 8);
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {1, 8, 16}) {
            chain<<<1, 32 * warps>>>(4096, 3.0, 20.0, o, c, mode);
            cudaDeviceSynchronize();
            long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
            printf("mode %d (%s) warps %2d: %.1f cycles per row\n", mode, mode == 0 ? "IEEE div" : mode == 1 ? "seeded div" : "no div",
                   warps, cy / 4096.0);
        }
    }
    cudaMemset(bad, 0, 8);
    check<<<1184, 256>>>(12345, 20000, bad);
    cudaDeviceSynchronize();
    unsigned long long nb; cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    printf("seeded vs IEEE mismatches over %lld operand pairs: %llu\n", 1184LL * 256 * 20000, nb);
    return 0;
}

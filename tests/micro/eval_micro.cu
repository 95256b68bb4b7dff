// Microbenchmark (dev aid): throughput of the bit-exact spline-evaluation
// arithmetic on B200 under different work decompositions.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2106_15319_b200/csrc/semd_device.cuh"
using namespace semd::dev;

// variant 1: S samples per thread, segment fixed per thread (no search), 2 envelopes
template <int S>
__global__ void __launch_bounds__(256) v_fixed(const double* __restrict__ in, double* out, int n, double h, double rh) {
    const int t0 = (blockIdx.x * blockDim.x + threadIdx.x) * S;
    if (t0 + S > n) return;
    double x0 = t0 - 1.0, x1 = t0 + S + 1.0;
    double y0 = in[t0], y1 = in[t0 + 1], m0 = 0.3, m1 = -0.2;
    double acc[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const double tt = (double)(t0 + k);
        const double hh = h * h;
        const double u = spline_eval_fast(x0, x1, y0, y1, m0, m1, h, rh, hh, tt);
        const double l = spline_eval_fast(x0 + 0.5, x1 + 0.5, y1, y0, m1, m0, h, rh, hh, tt);
        const double mean = 0.5 * (u + l);
        acc[k] = in[t0 + k] - mean;
    }
#pragma unroll
    for (int k = 0; k < S; ++k) out[t0 + k] = acc[k];
}

// variant 1b: same, occupancy limited to 2 blocks x 256 threads per SM (128 regs)
template <int S>
__global__ void __launch_bounds__(256, 2) v_fixed_lo(const double* __restrict__ in, double* out, int n, double h, double rh) {
    const int t0 = (blockIdx.x * blockDim.x + threadIdx.x) * S;
    if (t0 + S > n) return;
    double x0 = t0 - 1.0, x1 = t0 + S + 1.0;
    double y0 = in[t0], y1 = in[t0 + 1], m0 = 0.3, m1 = -0.2;
    double acc[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const double tt = (double)(t0 + k);
        const double hh = h * h;
        const double u = spline_eval_fast(x0, x1, y0, y1, m0, m1, h, rh, hh, tt);
        const double l = spline_eval_fast(x0 + 0.5, x1 + 0.5, y1, y0, m1, m0, h, rh, hh, tt);
        acc[k] = in[t0 + k] - 0.5 * (u + l);
    }
#pragma unroll
    for (int k = 0; k < S; ++k) out[t0 + k] = acc[k];
}
// variant 1c: grid-stride persistent, 2 blocks/SM of 256, 128 regs forced via dummy smem
template <int S>
__global__ void __launch_bounds__(256, 2) v_persist(const double* __restrict__ in, double* out, int n, double h, double rh) {
    __shared__ double pad[6000];
    if (n < 0) pad[threadIdx.x] = 1.0;
    for (int t0 = (blockIdx.x * blockDim.x + threadIdx.x) * S; t0 + S <= n; t0 += gridDim.x * blockDim.x * S) {
        double x0 = t0 - 1.0, x1 = t0 + S + 1.0;
        double y0 = in[t0], y1 = in[t0 + 1], m0 = 0.3, m1 = -0.2;
        double acc[S];
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const double tt = (double)(t0 + k);
            const double hh = h * h;
            const double u = spline_eval_fast(x0, x1, y0, y1, m0, m1, h, rh, hh, tt);
            const double l = spline_eval_fast(x0 + 0.5, x1 + 0.5, y1, y0, m1, m0, h, rh, hh, tt);
            acc[k] = in[t0 + k] - 0.5 * (u + l);
        }
#pragma unroll
        for (int k = 0; k < S; ++k) out[t0 + k] = acc[k];
    }
}

// variant 2: reference form with IEEE divisions
template <int S>
__global__ void __launch_bounds__(256) v_ref(const double* __restrict__ in, double* out, int n) {
    const int t0 = (blockIdx.x * blockDim.x + threadIdx.x) * S;
    if (t0 + S > n) return;
    double x0 = t0 - 1.0, x1 = t0 + S + 1.0;
    double y0 = in[t0], y1 = in[t0 + 1], m0 = 0.3, m1 = -0.2;
    double acc[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        const double tt = (double)(t0 + k);
        const double u = spline_eval_ref(x0, x1, y0, y1, m0, m1, tt);
        const double l = spline_eval_ref(x0 + 0.5, x1 + 0.5, y1, y0, m1, m0, tt);
        acc[k] = in[t0 + k] - 0.5 * (u + l);
    }
#pragma unroll
    for (int k = 0; k < S; ++k) out[t0 + k] = acc[k];
}

// variant 3: pure DFMA throughput
__global__ void v_dfma(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.999, d = 1e-7, e = 2.0, f = 3.0, g = 4.0, h = 5.0;
    for (int i = 0; i < iters; ++i) {
        a = fma(a, b, d); c = fma(c, b, d); e = fma(e, b, d); f = fma(f, b, d);
        g = fma(g, b, d); h = fma(h, b, d);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + c + e + f + g + h;
}

int main() {
    const int n = 1 << 26;
    double *in, *out;
    cudaMalloc(&in, n * 8);
    cudaMalloc(&out, n * 8);
    cudaMemset(in, 0, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    auto run = [&](const char* name, auto launch, double work, const char* unit) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%-24s %8.3f ms  %.3e %s\n", name, ms / 5, work / (ms / 5 / 1e3), unit);
    };
    run("fixed S=4", [&] { v_fixed<4><<<n / 4 / 256, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("fixed S=8", [&] { v_fixed<8><<<n / 8 / 256, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("fixed S=2", [&] { v_fixed<2><<<n / 2 / 256, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("fixed_lo S=4", [&] { v_fixed_lo<4><<<n / 4 / 256, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("persist 2x256 S=4", [&] { v_persist<4><<<148 * 2, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("persist 2x256 S=8", [&] { v_persist<8><<<148 * 2, 256>>>(in, out, n, 7.0, 1.0 / 7.0); }, n, "samples/s");
    run("ref S=4", [&] { v_ref<4><<<n / 4 / 256, 256>>>(in, out, n); }, n, "samples/s");
    run("dfma", [&] { v_dfma<<<148 * 8, 256>>>(out, 4096); }, 148.0 * 8 * 256 * 4096 * 6 * 2, "flop/s");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

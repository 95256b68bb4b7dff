// semd_launch.h -- host-side entry points into semd_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "semd_types.cuh"

namespace semd {
namespace dev {

struct RngJob {
    uint64_t seed;
    uint64_t* out;
    long long n;
};

size_t eval_smem_bytes();
cudaError_t eval_setup();
void launch_eval(const Arena& A, int sms, cudaStream_t st);
size_t solve_smem_bytes();
cudaError_t launch_setup();
void launch_step(const Arena& A, int sms, cudaStream_t st);
// programmatic dependent launch of the step kernels (default on; SEMD_PDL=0 disables)
bool pdl_enabled();
unsigned long long launch_count();  // kernels launched by this library (all contexts)
void count_launches(int n);
void launch_rng(const RngJob* jobs, int njobs, cudaStream_t st);
void launch_rng_ensemble(uint64_t base, long long m0, int count, uint64_t* out, long long stride, long long n,
                         cudaStream_t st);
void launch_box_muller(uint64_t* draws, long long n, double stdv, cudaStream_t st);
void launch_signal_std(const double* x, long long n, double* out, double scale, cudaStream_t st);
void launch_ensemble_finish(double* sums, int K, long long L, const double* x, double* residue, double inv,
                            cudaStream_t st);
void launch_concatenate(const double* x, long long M, long long N, long long D, const double* a, double* out,
                        int naive, cudaStream_t st);
void launch_transition_weights(long long d, double* a, cudaStream_t st);
void launch_deconcatenate(const double* modes, long long K, long long Lm, long long M, long long N, long long D,
                          double* out, cudaStream_t st);
void launch_envelope(const double* xs, const double* ys, int n, double* mom, double* work, long long length,
                     double* out, cudaStream_t st);
void launch_stage_scale(double* mode, long long n, double inv, int* nonzero, cudaStream_t st);
void launch_count_extrema(const double* x, long long n, unsigned long long* cnt, cudaStream_t st);
void launch_sub(double* residue, const double* mode, long long n, cudaStream_t st);
void launch_envelope_knots(const unsigned long long* idx, const double* val, long long n, long long length,
                           double* xs, double* ys, cudaStream_t st);
void launch_fill(double* p, long long n, double v, cudaStream_t st);
void launch_copy(const double* src, double* dst, long long n, cudaStream_t st);
void launch_gather(const int* idx, unsigned n, const double* src, double* out, cudaStream_t st);
void launch_signal_std_batch(const double* x, long long n, int B, double* out, double scale, cudaStream_t st);
void launch_slicewise_tensor(const double* sums, int kc, const int* kj, const double* res, long long M, int N,
                             int common, double scale, int scaled, double* out, cudaStream_t st);
void launch_slicewise_finish(const double* x, const double* sums, int kc, long long M, int N, double inv, double* res,
                             cudaStream_t st);
void launch_axpy(const double* a, const double* b, double beta, double* out, long long n, cudaStream_t st);

}  // namespace dev
}  // namespace semd

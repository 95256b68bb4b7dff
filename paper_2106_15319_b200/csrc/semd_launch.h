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
void launch_spec_decay(int* spec_hist, cudaStream_t st);  // halve the speculation statistics
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
size_t signal_std_workspace(long long n);  // 0: the signal is short, no workspace used
void launch_signal_std(const double* x, long long n, double* out, double scale, cudaStream_t st, void* ws = nullptr);
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
void launch_fill_i32(int* p, long long n, int v, cudaStream_t st);
void launch_copy(const double* src, double* dst, long long n, cudaStream_t st);
void launch_gather(const int* idx, unsigned n, const double* src, double* out, cudaStream_t st);
void launch_signal_std_batch(const double* x, long long n, int B, double* out, double scale, cudaStream_t st);
void launch_slicewise_tensor(const double* sums, int kc, const int* kj, const double* res, long long M, int N,
                             int common, double scale, int scaled, double* out, cudaStream_t st);
void launch_slicewise_finish(const double* x, const double* sums, int kc, long long M, int N, double inv, double* res,
                             cudaStream_t st);
void launch_axpy(const double* a, const double* b, double beta, double* out, long long n, cudaStream_t st);


// ---- the resident engine (semd_resident.cu): one CTA per job for short signals
constexpr int kResThreads = 512;
constexpr int kResMaxL = 8188;  // longest signal (samples) the resident engine takes
struct RJob {  // one job = JobSpec of the host driver (emd / EEMD realization / CEEMDAN task)
    int m, task, k, kmax, k0, init_kind, write_imf, detect_only;
    double beta;
    const double* a;
    const double* b;
    double* imf_out;    // every IMF also written here (single-IMF CEEMDAN noise tasks)
    double* res_out;    // every residue also written here
    double* res_final;  // the job's final residue
};
struct RResult {
    int k, produced, ended_insufficient, smem_overflow, k_overflow, hazards;
    unsigned n0, n1;
    long long sifted;
};
struct ResArgs {
    const RJob* jobs;
    RResult* res;
    int njobs, L;
    double* store;     // [njobs][kc][Lp] IMFs of write_imf jobs (accumulated in job order afterwards)
    int kc;            // IMF rows per job
    int* sifts;        // [njobs][kc] sift count of every produced IMF
    double* scratch;   // [grid][2][Lp] per-CTA residue and pre-sift candidate
    unsigned* ticket;  // job queue
    int max_iters;
    double sd_thr;
    int tab_rows;      // shared-memory segment-table capacity (16-byte rows)
    TraceRec* trace;
    int trace_cap;
    int* trace_count;
    int* sd_rechecks;
    int debug;         // bit 2: every SD decision by the sequential sums; bit 1: phase cycle profile
    int chain_div;     // tuning (SEMD_RES_CHAINS): solve chains per side aimed at (0: default)
    unsigned long long* prof;  // [16] SM cycles per phase (debug bit 1): detect, tables, solve, eval, sums, final, init, -, solve: rhs, fwd, back, table
};
size_t resident_smem_bytes(int L, int rows);
cudaError_t resident_setup();  // per device (launch_setup)
int resident_max_smem();
void launch_resident(const ResArgs& P, int grid, cudaStream_t st);

// The whole CEEMDAN (emd.cpp:264-344) in one cooperative launch of the resident engine.
struct CeeCtl {              // zeroed by the host before the launch
    unsigned bar_count, bar_gen;  // grid barrier
    unsigned ticket[64];     // per-stage job queues
    int beta_stage;          // highest stage whose beta is published
    int K;                   // modes produced
    int status;              // 1: segment tables outgrew the shared memory, 2: mode rows exhausted
    int stop[64];            // per stage: the residue check ended the loop
    int nonzero[64];         // per stage: the averaged mode has a nonzero sample
    double beta[64];
    unsigned long long sifted;
    int hazards;
};
struct CeeArgs {
    const double* x;     // the signal
    double* residue;     // running residue (starts as x)
    double* nres;        // [nr][Ls] noise residues (white noise at the start), updated in place
    long long Ls;
    double* e1;          // [nr][Lp] first modes of the stage
    int* e1_ok;          // [nr] first mode present (0: InsufficientExtrema -> zeros)
    int* alive;          // [nr] noise still yields modes (emd.cpp:318-324)
    double* E;           // [nr][Lp] this stage's noise modes E_K(w_m) (noise item -> first-mode item)
    int* e_have;         // [nr] E_K(w_m) present (0: exhausted, zeros)
    int* edone;          // [nr] stage whose noise item has finished (stage-tagged, zeroed at launch)
    double* modes;       // [kcap][L] the averaged modes
    int kcap, nr, m0, max_imfs;
    double nstd, beta0, inv_nr;
    CeeCtl* ctl;
};
int launch_res_ceemdan(const ResArgs& P, const CeeArgs& Q, int grid, cudaStream_t st);  // cudaError_t
void launch_res_accum(const RJob* jobs, const RResult* res, const int* rowj, const double* store, int kc, long long Lp,
                      int L, double* sums, int rows, cudaStream_t st);

}  // namespace dev
}  // namespace semd

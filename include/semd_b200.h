/*
 * semd_b200.h -- C ABI of the B200-native serial-EMD hot path.
 *
 * Drop-in boundary for the reference's free-function API in namespace semd
 * (/root/reference/proj/include/semd/emd.hpp:45-118 and serialize.hpp:10-50).
 * Each entry point below names the reference declaration it replaces. Plain
 * pointers and sizes only; no C++ or torch types cross this boundary. The
 * C++ mirror of the reference signatures (with the reference's exception
 * classes and messages) is include/semd/*.hpp, implemented over this ABI.
 *
 * All compute runs on the GPU (sm_100a). There is no CPU fallback: if no
 * CUDA device is usable, semd_ctx_create fails with SEMD_CUDA_ERROR.
 *
 * Buffers: host-pointer entry points take caller-owned host memory and copy
 * in/out; *_device entry points take device pointers on the context's GPU.
 * Calls are synchronous at the ABI (stream-ordered inside). One context per
 * host thread, or external locking.
 */
#ifndef SEMD_B200_H
#define SEMD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. SEMD_INVALID_INPUT maps to semd::InvalidInput and
 * SEMD_INSUFFICIENT_EXTREMA to semd::InsufficientExtrema (types.hpp:15-36),
 * with the reference's message in semd_last_error(). */
#define SEMD_OK 0
#define SEMD_INVALID_INPUT 1
#define SEMD_INSUFFICIENT_EXTREMA 2
#define SEMD_CAPACITY 3 /* output capacity too small; *k_out holds what is needed */
#define SEMD_CUDA_ERROR 4
#define SEMD_NO_MEMORY 5

#define SEMD_ALGO_EMD 0
#define SEMD_ALGO_EEMD 1
#define SEMD_ALGO_CEEMDAN 2

/* emd.hpp:10-18 SiftConfig */
typedef struct semd_sift_cfg {
    double sd_threshold; /* default 0.2 */
    int32_t max_sift_iters; /* default 300 (MaxIter) */
    int32_t max_imfs; /* default 0 = unlimited */
} semd_sift_cfg;

/* emd.hpp:21-28 EnsembleConfig */
typedef struct semd_ens_cfg {
    double nstd; /* default 0.2 (NSTD) */
    int32_t nr; /* default 100 (NR) */
    int32_t reserved;
    uint64_t base_seed; /* default 0 */
} semd_ens_cfg;

/* One record per find_extrema call made by the sifting machinery: the parity
 * trace (IMF index, sift iteration, extrema counts and an order-sensitive hash
 * of both index lists). Identical layout to the oracle's so_trace_rec. */
typedef struct semd_trace_rec {
    int32_t task; /* 0 emd sift, 1 ceemdan noise IMF, 2 ceemdan first mode, 3 ceemdan stage check */
    int32_t m;    /* realization */
    int32_t k;    /* IMF / stage index */
    int32_t iter; /* find_extrema call within extract_imf */
    uint32_t n_max, n_min;
    uint64_t hash;
} semd_trace_rec;

typedef struct semd_trace {
    semd_trace_rec* rec; /* host array of `cap` records (may be NULL with cap 0) */
    size_t cap;
    size_t count; /* records produced (may exceed cap; extra records dropped) */
} semd_trace;

/* Counters of the last decomposition run on a context. */
typedef struct semd_stats {
    uint64_t sifted_samples; /* sum over executed sift iterations of L */
    uint64_t sift_iterations;
    uint64_t steps;          /* lockstep engine steps */
    uint64_t kernel_launches;
    uint64_t solve_hazards;  /* speculative-solve block boundaries that disagreed; each such envelope
                                was re-solved by the exact sequential fallback (results stay bit-exact) */
    int32_t slots;           /* concurrent sift jobs used */
    int32_t waves;
    double eval_ms;          /* optional (timing enabled): device time of the sift kernel -- k_eval on the
                                lockstep engine, k_resident / k_res_ceemdan on the resident engine */
    uint64_t eval_launches;
    uint64_t sd_rechecks;    /* SD stop tests whose tree-summed ratio was too close to sd_threshold to certify
                                and were redone with the reference's sequential sums */
    uint64_t resident_jobs;  /* jobs run by the resident (one CTA per job, shared-memory) engine */
} semd_stats;

typedef struct semd_ctx semd_ctx;

/* ---- context ---------------------------------------------------------- */
int semd_ctx_create(int device, semd_ctx** out);
void semd_ctx_destroy(semd_ctx* ctx);
const char* semd_last_error(void); /* thread-local message of the last failure */
int semd_get_stats(semd_ctx* ctx, semd_stats* out);
/* Run subsequent work on this CUDA stream (cudaStream_t as void*); NULL = the context's own. */
int semd_set_stream(semd_ctx* ctx, void* cuda_stream);
/* Enable CUDA-event timing of the sift kernel (fills semd_stats.eval_ms). */
int semd_set_timing(semd_ctx* ctx, int enable);
/* Maximum concurrent sift jobs (0 = automatic from L and memory). */
int semd_set_max_slots(semd_ctx* ctx, int slots);
/* Sift engine: SEMD_ENGINE_AUTO (default; the SEMD_ENGINE environment variable "lockstep" /
 * "resident" overrides it) runs signals of at most SEMD_RESIDENT_MAX_L samples on the resident
 * engine (one persistent CTA per job, candidate and segment tables in shared memory) and longer
 * ones on the lockstep engine (G jobs per five-kernel step, state in HBM). Both are bit-identical
 * to the reference; RESIDENT still falls back to LOCKSTEP for signals it cannot hold. */
#define SEMD_ENGINE_AUTO 0
#define SEMD_ENGINE_LOCKSTEP 1
#define SEMD_ENGINE_RESIDENT 2
#define SEMD_RESIDENT_MAX_L 8188
int semd_set_engine(semd_ctx* ctx, int engine);

/* ---- emd.hpp ---------------------------------------------------------- */
/* emd.hpp:41 find_extrema (emd.cpp:10-35). Arrays hold up to n entries. */
int semd_find_extrema(semd_ctx* ctx, const double* x, size_t n, size_t* max_idx, double* max_val, size_t* n_max,
                      size_t* min_idx, double* min_val, size_t* n_min);
/* emd.hpp:49-50 envelope (emd.cpp:91-125) */
int semd_envelope(semd_ctx* ctx, const size_t* idx, const double* val, size_t n, size_t length, double* out);
/* emd.hpp:62 extract_imf (emd.cpp:127-153) */
int semd_extract_imf(semd_ctx* ctx, const double* x, size_t n, const semd_sift_cfg* cfg, double* imf,
                     int32_t* sift_count);
/* emd.hpp:68 emd, :91-92 eemd, :99-100 ceemdan, :113-114 decompose (emd.cpp:155-373).
 * imfs: k_cap x n (row k contiguous); residue: n. sift_counts (optional, k_cap):
 * per-IMF sift iterations (EMD only). trace optional. */
int semd_decompose(semd_ctx* ctx, int algo, const double* x, size_t n, const semd_sift_cfg* cfg,
                   const semd_ens_cfg* ens, double* imfs, size_t k_cap, size_t* k_out, double* residue,
                   int32_t* sift_counts, semd_trace* trace);
/* emd.hpp:73 white_noise (emd.cpp:181-200) */
int semd_white_noise(semd_ctx* ctx, size_t n, uint64_t seed, double std, double* out);
/* emd.hpp:77 derive_seed (emd.cpp:174-179): pure integer function of its arguments */
uint64_t semd_derive_seed(uint64_t base, uint64_t index);
/* emd.hpp:81 noise_mode (emd.cpp:202-207) */
int semd_noise_mode(semd_ctx* ctx, const double* w, size_t n, size_t i, const semd_sift_cfg* cfg, double* out);
/* emd.hpp:84 signal_std (emd.cpp:209-217) */
int semd_signal_std(semd_ctx* ctx, const double* x, size_t n, double* out);
/* emd.hpp:107 parse_algorithm (emd.cpp:346-354): 0 emd, 1 eemd, 2 ceemdan */
int semd_parse_algorithm(const char* name, int* algo);

/* ---- serialize.hpp ---------------------------------------------------- */
/* serialize.hpp:12 transition_weights (serialize.cpp:7-13) */
int semd_transition_weights(semd_ctx* ctx, size_t d, double* out);
/* serialize.hpp:16 default_transition_length (serialize.cpp:15-18) */
size_t semd_default_transition_length(size_t rows);
/* serialize.hpp:25 concatenate / :31 concatenate_naive (serialize.cpp:30-71).
 * x is channel-contiguous M x N (types.hpp:61-62); out has M*N + D*(N-1). */
int semd_concatenate(semd_ctx* ctx, const double* x, size_t M, size_t N, size_t D, double* out);
int semd_concatenate_naive(semd_ctx* ctx, const double* x, size_t M, size_t N, size_t D, double* out);
/* serialize.hpp:37-38 deconcatenate (serialize.cpp:73-95): modes K x L (row k
 * contiguous); out is the ImfTensor layout (k*N + j)*M + i (types.hpp:105-110). */
int semd_deconcatenate(semd_ctx* ctx, const double* modes, size_t K, size_t L, size_t M, size_t N, size_t D,
                       double* out);
/* serialize.hpp:44-45 serial_decompose (serialize.cpp:97-105): tensor has
 * room for k_cap modes (IMFs + residue) of M*N; *modes_out = K+1. */
int semd_serial_decompose(semd_ctx* ctx, int algo, const double* x, size_t M, size_t N, size_t D,
                          const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* tensor, size_t k_cap,
                          size_t* modes_out, semd_trace* trace);

/* ---- device-resident entry points (benchmarks, multi-GPU drivers) ------- */
/* Same as semd_decompose with device buffers. */
int semd_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t n, const semd_sift_cfg* cfg,
                          const semd_ens_cfg* ens, double* d_imfs, size_t k_cap, size_t* k_out, double* d_residue);
/* EEMD realization shard [m_begin, m_end): UNSCALED per-IMF sums over the
 * shard (row k contiguous, k_cap rows, zero-padded) and the shard's max K.
 * Combine shards by summing (e.g. an NCCL all-reduce), then call
 * semd_ensemble_finish_device with the total nr. */
int semd_eemd_partial_device(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg,
                             const semd_ens_cfg* ens, int32_t m_begin, int32_t m_end, double* d_sums,
                             size_t k_cap, size_t* k_out);
/* The same, plus the parity trace of the shard's realizations (one record per find_extrema
 * call, task 0, field m = global realization index; trace may be NULL). */
int semd_eemd_partial_traced_device(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg,
                                    const semd_ens_cfg* ens, int32_t m_begin, int32_t m_end, double* d_sums,
                                    size_t k_cap, size_t* k_out, semd_trace* trace);
/* imfs *= 1/nr; residue = x - sum_k imfs_k (emd.cpp:252-260). */
int semd_ensemble_finish_device(semd_ctx* ctx, const double* d_x, size_t n, double* d_sums, size_t K, int32_t nr,
                                double* d_residue);
/* serialize.cpp:30-50 / :73-95 on device buffers (same layouts as the host versions). */
int semd_concatenate_device(semd_ctx* ctx, const double* d_x, size_t M, size_t N, size_t D, double* d_out);
int semd_deconcatenate_device(semd_ctx* ctx, const double* d_modes, size_t K, size_t L, size_t M, size_t N, size_t D,
                              double* d_out);
int semd_serial_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t M, size_t N, size_t D,
                                 const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* d_tensor,
                                 size_t k_cap, size_t* modes_out);

/* baseline.hpp / baseline.cpp:5-29 slicewise_decompose: each channel of the channel-contiguous
 * M x N multi-signal decomposed independently; the ImfTensor (k*N + j)*M + i holds each channel's
 * IMFs zero-padded to a common mode count, residue last. EMD and EEMD run all channels (x all
 * realizations) as one batched engine pass. *modes_out = common mode count (SEMD_CAPACITY and
 * the needed count when it exceeds k_cap). */
int semd_slicewise_decompose(semd_ctx* ctx, int algo, const double* x, size_t M, size_t N, const semd_sift_cfg* cfg,
                             const semd_ens_cfg* ens, double* tensor, size_t k_cap, size_t* modes_out);
int semd_slicewise_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t M, size_t N,
                                    const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* d_tensor,
                                    size_t k_cap, size_t* modes_out);

/* recognition.cpp:281-298's decompositions batched: B independent serial_decompose calls
 * (serialize.cpp:97-105) on same-shape multi-signals (e.g. images as channels) in one engine pass.
 * x: B blocks of M x N (channel-contiguous); tensor: B blocks of k_cap x N x M in the ImfTensor
 * layout, item b holding K_b IMFs then its residue (zero modes after); modes_out[b] = K_b + 1.
 * SEMD_CAPACITY when some K_b + 1 > k_cap. */
int semd_serial_decompose_batch(semd_ctx* ctx, int algo, const double* x, size_t B, size_t M, size_t N, size_t D,
                                const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* tensor, size_t k_cap,
                                size_t* modes_out);

/* ---- CEEMDAN across GPUs: stages over a realization shard (emd.cpp:264-344) ----------
 * Rank r owns realizations [m_begin, m_end) (seeds from the global index). Driver loop:
 *   begin; stage(partial); all-reduce(partial) -> total; finish_stage(total, nr, 0, ...);
 *   while (max_imfs == 0 || K < max_imfs) {
 *     residue_extrema(&t); if (t < 3) break;                       (emd.cpp:311)
 *     stage(partial); all-reduce; finish_stage(total, nr, 1, mode, &ok); if (!ok) break;
 *   }
 *   residue(out).
 * stage() writes the UNSCALED sum over the shard of this stage's first modes (n doubles);
 * finish_stage scales the global total by 1/nr, stops on an all-zero mode (ok = 0;
 * emd.cpp:332-337) or subtracts it from the residue. With one shard [0, nr) this is
 * bit-identical to semd_decompose(SEMD_ALGO_CEEMDAN). One active shard per context. */
int semd_ceemdan_shard_begin(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg,
                             const semd_ens_cfg* ens, int32_t m_begin, int32_t m_end);
int semd_ceemdan_shard_residue_extrema(semd_ctx* ctx, size_t* total);
int semd_ceemdan_shard_stage(semd_ctx* ctx, double* d_partial);
int semd_ceemdan_shard_finish_stage(semd_ctx* ctx, const double* d_total, int32_t nr, int32_t check_zero,
                                    double* d_mode_out, int32_t* accepted);
int semd_ceemdan_shard_residue(semd_ctx* ctx, double* d_res_out);

/* ---- multi-GPU (B200 extension; the reference is single-process) -------------------------
 * One process (or thread) per GPU, one context each, joined by an NCCL communicator over
 * NVLink/NVSwitch. Rank 0 makes the id with semd_comm_unique_id and ships its bytes to the
 * other ranks (any side channel); every rank calls semd_comm_init collectively. After that,
 * EEMD and CEEMDAN calls on the context (semd_decompose, semd_serial_decompose and their
 * *_device forms) are collective: every rank passes the same input, rank r sifts realizations
 * shard_range(nr, r, W) (contiguous; seeds from the global index, emd.cpp:238), and
 *   EEMD:    ncclAllReduce(max) of K, one ncclReduce/ncclAllReduce(sum) of the K x n sums,
 *            then the finish (emd.cpp:246-261);
 *   CEEMDAN: one ncclAllReduce(sum) of n doubles per stage (emd.cpp:301-306, :331-339).
 * Across ranks the ensemble sum is not realization-ordered, so N > 1 results equal the
 * single-GPU ones to rounding (not bit-for-bit); a 1-rank communicator is bit-identical.
 * EMD calls are replicated (every rank computes the same result). */
#define SEMD_COMM_ID_BYTES 128
int semd_comm_unique_id(void* id_out, size_t bytes);
int semd_comm_init(semd_ctx* ctx, const void* id, size_t bytes, int rank, int world);
/* root >= 0: the EEMD sums are reduced to that rank only (others get K and no outputs);
 * root < 0 (default): every rank receives the full result. */
int semd_comm_set_root(semd_ctx* ctx, int root);
int semd_comm_info(semd_ctx* ctx, int* rank, int* world);
/* Small host-side reductions over the communicator (op 0 sum, 1 max); no-op without one. */
int semd_comm_allreduce_host(semd_ctx* ctx, double* vals, size_t n, int op);
int semd_comm_destroy(semd_ctx* ctx);

/* ---- device memory and timing on the context's stream (driver / benchmark plumbing) ------ */
int semd_device_alloc(semd_ctx* ctx, size_t bytes, void** d_out);
int semd_device_free(semd_ctx* ctx, void* d);
int semd_host_alloc(semd_ctx* ctx, size_t bytes, void** h_out); /* pinned host memory */
int semd_host_free(semd_ctx* ctx, void* h);
int semd_memcpy(semd_ctx* ctx, void* dst, const void* src, size_t bytes); /* any direction, synchronous */
/* CUDA events on the context stream: device milliseconds between start and stop. */
int semd_timer_start(semd_ctx* ctx);
int semd_timer_stop(semd_ctx* ctx, double* ms);

#ifdef __cplusplus
}
#endif
#endif

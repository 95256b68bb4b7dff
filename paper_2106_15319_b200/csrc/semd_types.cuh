// semd_types.cuh -- device-side data layout of the serial-EMD sift engine.
//
// One "slot" runs one sifting job (the IMF loop of emd(), emd.cpp:155-172, on
// one signal: a plain EMD input, one EEMD realization x + beta*w_m, or one
// CEEMDAN task). G slots advance together, one phase per kernel launch
// ("lockstep steps"); all per-slot state lives in HBM so no host round trip is
// needed between sift iterations.
//
// HBM layout per engine (L = serialized length, G = slots, T = eval tile):
//   bufs    f64 [G][4][L]        rotating X (IMF input), C (candidate), D (new candidate), R (residue of a
//                                speculative last sift, see ST_PRIMED)
//   tflags  u32 [2 par][G][tiles][32]     k_eval's detection word per lane: window flags + tile ranks
//   scnt    u32 [2 side][G][tiles]        extrema per tile
//   kidx    i32 [2 par][2 side][G][cap]   compacted extrema indices (cap = L/2+2)
//   (extremum values are not stored: value r = candidate[idx[r]], gathered by k_solve)
//   toff    u32 [2][2][G][tiles+1]        per-tile knot offsets, local to a scan chunk
//   tbase   u32 [2][2][G][chunks]         knot offset of each scan chunk (toff_at adds it)
//   ctot/cnum/cden [2 side][G][chunks]    per-chunk extrema totals and SD partials
//   ktab    f64x4 [2 side][G][cap+8]      segment table of the mirrored knot system {x, y, m, 1/h}
//   tnum/tden/thash [G][tiles]            per-tile SD and trace-hash partials
//   sums    f64 [kcap][L]                 ensemble / IMF accumulators
#pragma once
#include <cstdint>
#include <cstdio>

// Bounds checks of the checked build (-DSEMD_CHECK, build.py --checked; the GPU pool offers no
// compute-sanitizer): a failed check prints its condition and traps the kernel.
#ifdef SEMD_CHECK
#define SEMD_ASSERT(c)                                                                       \
    do {                                                                                     \
        if (!(c)) {                                                                          \
            printf("SEMD_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                       \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define SEMD_ASSERT(c) \
    do {               \
    } while (0)
#endif
#include <vector_types.h>

namespace semd {
namespace dev {

constexpr int kEvalTile = 128;                  // samples per eval tile (one warp)
constexpr int kEvalThreads = 256;              // 8 independent warps per CTA
constexpr int kSpt = kEvalTile / 32;            // samples per lane (consecutive)

constexpr int kSolveChains = 64;                         // speculative chains per block
constexpr int kSolveChunk = 16;                          // rows per chain
constexpr int kSolveWarm = 32;                           // per-chain warm-up rows
constexpr int kSolveBlock = kSolveChains * kSolveChunk;  // rows per CTA
constexpr int kSolveHalo = 64;                           // cross-block warm-up rows (front and back halo chains)
constexpr int kSolveThreads = 128;                       // >= kSolveMaxChains (the rest help staging)
constexpr int kSolveCtasPerSm = 4;
constexpr int kSolveMaxChains = (kSolveBlock + 2 * kSolveHalo) / kSolveChunk;  // chains tiling a block + halos
constexpr int kSolveSeqMax = 96;                         // rows solved by one exact thread
constexpr int kSolveWin = kSolveBlock + 2 * kSolveHalo + kSolveWarm + 4;  // staged knot window per block
constexpr int kSolvePadWin = kSolveWin + kSolveWin / 16 + 2;               // + one pad double per 16 rows

constexpr int kFinalTile = 1024;

constexpr int kScanShift = 12;
constexpr int kScanChunk = 1 << kScanShift;  // tiles per k_scan CTA
constexpr int kScanThreads = 256;
constexpr int kScanPer = kScanChunk / kScanThreads;

enum State : int {
    ST_FREE = 0,
    ST_INIT = 1,    // materialise X from the job's input, then detect (iteration 0)
    ST_DETECT = 2,  // detect extrema of X (iteration 0 of the next IMF)
    ST_SIFT = 3,    // one sift per step
    ST_WAITK = 4,   // IMF converged; waiting for every slot to reach the same IMF (lockstep)
    ST_FINAL = 5,   // residue update + accumulation this step
    ST_DONE = 6,
    // Speculative last sift (Slot::spec): a sift that is likely the IMF's last also writes the
    // residue R' = X - new (emd.cpp:167) and detects R''s extrema instead of new's. When the SD
    // test then stops, R' and its extrema are the next IMF's input and its find_extrema, so the
    // next IMF starts in ST_PRIMED (decide + compact only; no DETECT pass) and k_final only
    // accumulates. When it does not stop, the candidate's extrema are detected in ST_REDETECT.
    ST_PRIMED = 7,    // the next IMF's input extrema were detected by the previous IMF's last sift
    ST_REDETECT = 8,  // detect the candidate's extrema (a speculative sift that did not stop)
};

enum EvalMode : int { EM_NONE = 0, EM_INIT = 1, EM_DETECT = 2, EM_SIFT = 3, EM_SPEC = 4 };

// slot states that take part in a step's eval / scan / decide phase
__host__ __device__ inline bool eval_state(int st) {
    return st == ST_INIT || st == ST_DETECT || st == ST_SIFT || st == ST_PRIMED || st == ST_REDETECT;
}
constexpr int kBufs = 4;        // slot buffers (X, C, D, R')
constexpr int kSpecK = 16;      // speculation statistics: IMF index (last row: all later IMFs)
constexpr int kSpecS = 8;       // ... and sift count (last column: all longer IMFs)

struct Slot {
    // ---- job description (host-written before ST_INIT) ----
    int m;          // realization index (trace id)
    int task;       // trace task id (0 emd, 1 ceemdan noise IMF, 2 ceemdan first mode)
    int kmax;       // IMF limit of this job (0: unlimited)
    int k0;         // IMF k accumulates into sums row k0 + k
    int init_kind;  // 0: X = a ; 1: X = a + beta*b ; 2: X = a (zero IMFs allowed) ...
    int write_imf;  // 1: IMFs are accumulated (sums[k0+k] += imf)
    double beta;
    const double* init_a;
    const double* init_b;
    double* imf_out;      // single-IMF jobs: the IMF is also written here by k_final
    double* res_out;      // single-IMF jobs: the residue x - imf is also written here
    int detect_only;      // job = one find_extrema call (CEEMDAN stage check), then DONE
    // ---- dynamic state (device-written) ----
    int state;
    int k;       // IMFs completed
    int iter;    // sifts done on the current IMF
    int par;     // knot-set parity holding the current extrema
    int xb;      // buffer id of X
    int cb;      // buffer id of the current candidate (-1: X)
    int db;      // destination buffer of this step's eval
    unsigned epoch;
    unsigned n[2];       // extrema counts (max, min) of the current knot set
    int ended_insufficient;
    int last_imf_b;      // buffer id that held the last finalised IMF
    int trace_iter;      // find_extrema record due after compaction (-1: none)
    int cpar;            // parity the stage knots are compacted into this step
    unsigned tn[2];      // extrema counts of this step's detect
    int hazards;         // speculative-solve boundary mismatches observed
    int spec;            // this SIFT pass is a speculative last sift (writes R' into rb, detects R')
    int rb;              // buffer id of R'
    int spec_hit;        // the finished IMF's residue R' is in rb and its extrema are detected
    long long sifted;    // sifted samples (L per completed sift)
    double num, den;
};

struct TraceRec {
    int32_t task, m, k, iter;
    uint32_t n_max, n_min;
    uint64_t hash;
};

// Control block: work lists and kernel bookkeeping (device memory).
struct Ctrl {
    unsigned ticket[8];  // 0 eval, 1 compact, 2 solve, 3 final
    unsigned done[8];    // same, 4 scan
    int n_eval;    // slots with an eval-phase job this step
    int n_final;   // slots finalising this step
    int n_compact; // slots whose detect output is compacted this step
    int n_solve;   // (slot, side) solve items
    int solve_blocks;  // total blocks over solve items
    int active;    // slots not FREE/DONE
    int trace_count;
    int hazards;
    int k_overflow;
    int step;
    int hz_count;  // hazard log records produced
    int finished;  // the run's last step has published active == 0: later steps return at once
    int sd_rechecks;  // SD stop tests redone with the reference's sequential sums (uncertified decisions)
    int spec_pass, spec_hits, spec_misses;  // speculative last sifts: run, stopped, continued
    int n_eval_pass;  // eval_list[0, n_eval_pass): slots with an eval pass (ST_PRIMED slots follow)
    unsigned long long ev_t0;  // k_eval span of this step (globaltimer): min CTA start, max CTA end
    unsigned long long ev_t1;
    unsigned long long ev_ns;  // accumulated k_eval spans of this run (timing mode)
    // per-kernel device spans (globaltimer), double-buffered by step parity: [p][kernel][0] = max
    // of ~start over CTAs (i.e. ~min start), [1] = max end; the next step's k_solve folds the
    // previous step's spans into kns (profiling: semd_kernel_spans)
    unsigned long long kt[2][5][2];
    unsigned long long kns[5];     // solve, eval, scan, compact, final
    unsigned long long strips[2];  // eval strips in DETECT/INIT mode, in SIFT mode
    unsigned long long strip_cyc[2];  // SM cycles spent on those strips (clock64, per warp)
};

enum KernelId : int { KID_SOLVE = 0, KID_EVAL = 1, KID_SCAN = 2, KID_COMPACT = 3, KID_FINAL = 4 };

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// thread 0 of every CTA, after pdl_begin() / at the end of the kernel
__device__ __forceinline__ void span_begin(Ctrl* C, int id) {
    atomicMax(&C->kt[C->step & 1][id][0], ~gtimer());
}
__device__ __forceinline__ void span_end(Ctrl* C, int id, int step) {
    atomicMax(&C->kt[step & 1][id][1], gtimer());
}
// fold parity p's spans into kns and clear them (all of that step's kernels have completed)
__device__ __forceinline__ void span_fold(Ctrl* C, int p) {
    for (int id = 0; id < 5; ++id) {
        const unsigned long long a = C->kt[p][id][0], b = C->kt[p][id][1];
        if (a && b && b > ~a) C->kns[id] += b - ~a;
        C->kt[p][id][0] = 0;
        C->kt[p][id][1] = 0;
    }
}

// Programmatic dependent launch: every step kernel starts with pdl_begin(): the grid
// may be launched while its predecessor drains (launch latency and ramp overlap the
// tail); griddepcontrol.wait then holds it until the predecessor completed and its
// memory is visible. The trigger lets this grid's successor launch once all of this
// grid's CTAs have started. Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

struct Arena {
    int L, G, tiles, cap, kcap;
    int strip;     // tiles per eval strip (one warp work item, one SD partial): 16, or 4 for short signals
    int kper;      // > 0: IMF rows per job (batched jobs own rows [k0, k0 + kper)); 0: all kcap rows
    long long Lp;  // slot-buffer stride = tiles * kEvalTile (16-byte aligned; whole tiles readable)
    double sd_threshold;
    int max_sift_iters;
    int trace_cap;
    double* bufs;
    int* kidx;
    unsigned* toff;
    unsigned* tbase;
    unsigned* ctot;
    double* cnum;
    double* cden;
    int chunks;  // scan chunks per (slot, side): ceil(tiles / kScanChunk)
    double4* ktab;
    unsigned* scnt;
    double* tnum;
    double* tden;
    unsigned long long* thash;
    unsigned* tflags;  // [2 par][G][tiles][32 lanes] per detection lane: flags (max | min << 4) | max rank << 8 | min rank << 16
    Slot* slots;
    double* sums;
    int* imf_sifts;   // [kcap] sift count per IMF of slot 0 (plain EMD / extract_imf)
    Ctrl* ctrl;
    int* eval_list;   // [G]
    int* final_list;  // [G]
    int* compact_list; // [G]
    int* solve_item;  // [2G] (slot << 1 | side)
    int* solve_off;   // [2G+1] block prefix
    double* sb;       // [2][G][max_blocks][6] solve block boundary values
    int max_blocks;
    TraceRec* trace;
    int* hzlog;       // [hzlog_cap][8] solve-hazard records {m, k, iter, side, n, block, blocks, 0}
    int hzlog_cap;
    int debug;        // test hooks: bit 0 treat every solve block boundary as a hazard (exercise the repair);
                      // bit 2 redo every SD stop test with the sequential sums; bit 3 no speculative
                      // last sifts; bit 4 every sift speculative
                      // bit 1: accumulate k_solve per-phase clock cycles into prof[]
    unsigned long long* prof;  // [16]
    int* spec_hist;   // [kSpecK][kSpecS] IMFs that stopped after s sifts, per IMF index: the speculation policy's
                      // memory, kept across waves and calls of a context (halved at each decomposition's start)
    int* status_host; // mapped pinned: [0] active slots after this step, [1] step counter
};

// sums row k0 + k of a job is writable (its IMF fits the job's rows)
__host__ __device__ inline bool imf_row_ok(const Arena& a, int k0, int k) {
    return k0 + k < a.kcap && (a.kper == 0 || k < a.kper);
}
__host__ __device__ inline size_t buf_off(const Arena& a, int slot, int b) {
    return ((size_t)slot * kBufs + (size_t)b) * (size_t)a.Lp;
}
__host__ __device__ inline size_t knot_off(const Arena& a, int par, int side, int slot) {
    return (((size_t)par * 2 + side) * a.G + slot) * (size_t)a.cap;
}
// per-tile rows are padded to a multiple of 4 entries (16-byte aligned vector access in k_scan)
__host__ __device__ inline size_t tiles4(const Arena& a) { return ((size_t)a.tiles + 3) & ~(size_t)3; }
__host__ __device__ inline size_t toff_off(const Arena& a, int par, int side, int slot) {
    return (((size_t)par * 2 + side) * a.G + slot) * (((size_t)a.tiles + 4) & ~(size_t)3);
}
__host__ __device__ inline size_t tsd_off(const Arena& a, int slot) { return (size_t)slot * tiles4(a); }
__host__ __device__ inline size_t tbase_off(const Arena& a, int par, int side, int slot) {
    return (((size_t)par * 2 + side) * a.G + slot) * (size_t)a.chunks;
}
__host__ __device__ inline size_t chunk_off(const Arena& a, int side, int slot) {
    return ((size_t)side * a.G + slot) * (size_t)a.chunks;
}
// Knot offset of tile j (0 <= j <= tiles) of one (parity, side, slot): chunk-local
// prefix + chunk base. Tile `tiles` (the total) belongs to the last chunk.
struct ToffView {
    const unsigned* to;
    const unsigned* tb;
    int last;  // chunks - 1
    __device__ __forceinline__ unsigned operator[](int j) const {
        const int c = (j >> kScanShift) < last ? (j >> kScanShift) : last;
        return to[j] + tb[c];
    }
    // L1-bypassing read (last-CTA epilogues read values other CTAs of the same kernel wrote)
    __device__ __forceinline__ unsigned cg(int j) const {
        const int c = (j >> kScanShift) < last ? (j >> kScanShift) : last;
        return __ldcg(to + j) + __ldcg(tb + c);
    }
};
__device__ __forceinline__ ToffView toff_view(const Arena& a, int par, int side, int slot) {
    return ToffView{a.toff + toff_off(a, par, side, slot), a.tbase + tbase_off(a, par, side, slot), a.chunks - 1};
}
__host__ __device__ inline size_t tfl_off(const Arena& a, int par, int slot) {
    return ((size_t)par * a.G + slot) * (size_t)a.tiles * 32;
}
__host__ __device__ inline size_t tab_off(const Arena& a, int side, int slot) {
    return ((size_t)side * a.G + slot) * (size_t)(a.cap + 8);
}
__host__ __device__ inline size_t scnt_off(const Arena& a, int side, int slot) {
    return ((size_t)side * a.G + slot) * tiles4(a);
}

}  // namespace dev
}  // namespace semd

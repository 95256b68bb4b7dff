// semd_capi.cu -- host engine and C ABI (include/semd_b200.h).
//
// The host side only stages buffers, seeds realizations and sequences kernel
// launches; every numeric operation of the hot path runs in semd_kernels.cu
// on the GPU. Control flow that the reference resolves per sift iteration
// (stop tests, IMF completion, extrema counts) is decided on the device by
// the epilogues of k_eval / k_final; the host only polls a mapped pinned word
// a few steps behind to learn when every slot is done.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/semd_b200.h"
#include "semd_launch.h"
#include "semd_types.cuh"

using semd::dev::Arena;
using semd::dev::Ctrl;
using semd::dev::Slot;
using semd::dev::TraceRec;

namespace {

thread_local std::string g_err;

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void raise(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Error{code, buf};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(SEMD_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return SEMD_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return SEMD_NO_MEMORY;
    }
}

uint64_t derive_seed(uint64_t base, uint64_t index) {  // emd.cpp:174-179
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// ---- NCCL, loaded on first use (single-GPU contexts never touch it) ----------------------
// The library is resolved by soname, so a process that already loaded one (e.g. torch's
// bundled copy) shares it. SEMD_NCCL_LIB overrides the path.
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        const char* names[] = {std::getenv("SEMD_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        for (const char* nm : names)
            if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
        if (!h) {
            const char* e = dlerror();
            a.err = e ? e : "libnccl.so.2 not found";
            return a;
        }
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.Reduce = reinterpret_cast<decltype(a.Reduce)>(dlsym(h, "ncclReduce"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.Reduce && a.GetErrorString;
        if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

const NcclApi& nccl() {
    const NcclApi& a = nccl_api();
    if (!a.ok) raise(SEMD_CUDA_ERROR, "NCCL unavailable: %s", a.err.c_str());
    return a;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(SEMD_CUDA_ERROR, "%s: %s", what, nccl_api().GetErrorString(r));
}

// Contiguous realization shard of rank r of W (the same split as paper_2106_15319_b200/parallel.py).
void shard_range(int nr, int rank, int world, int* mb, int* me) {
    const int per = (nr + world - 1) / world;
    *mb = std::min(nr, rank * per);
    *me = std::min(nr, *mb + per);
}

// Device allocation helper that frees on scope exit.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    explicit DBuf(size_t b) { alloc(b); }
    ~DBuf() {
        if (p) cudaFree(p);
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    void alloc(size_t b) {
        if (p && bytes >= b) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (b == 0) b = 8;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            raise(SEMD_NO_MEMORY, "cudaMalloc(%zu bytes) failed: %s", b, cudaGetErrorString(e));
        }
        bytes = b;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct JobSpec {
    int m = 0, task = 0, k = 0, kmax = 0, k0 = 0, init_kind = 0, write_imf = 1, detect_only = 0;
    double beta = 0.0;
    const double* a = nullptr;
    const double* b = nullptr;
    double* imf_out = nullptr;
    double* res_out = nullptr;
};

}  // namespace

struct semd_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    int max_slots = 0;
    bool timing = false;
    semd_stats stats{};
    // engine arena
    Arena A{};
    int cfg_L = -1, cfg_G = -1, cfg_kcap = -1, cfg_trace = -1;
    DBuf bufs, kidx, toff, tbase, ctot, cnum, cden, ktab, scnt, tnum, tden, thash, tflags, slots, sums, imf_sifts, ctrl, lists, sb, trace, hzlog, prof;
    int* status_host = nullptr;
    int* status_host_dev = nullptr;
    unsigned char* pin_jobs = nullptr;  // pinned staging of a run's slots, control block and eval list
    size_t pin_jobs_bytes = 0;
    std::vector<Slot> h_slots;
    std::vector<TraceRec> h_trace;
    // scratch
    DBuf in_x, in_y, noise, scratch, scratch2, scalar, rng_jobs, std_ws, spec_hist;
    cudaEvent_t ev[16]{};
    cudaStream_t rng_stream = nullptr;  // noise for the next wave is generated here, overlapping the sift
    cudaEvent_t noise_ready[2]{};
    cudaEvent_t res_ready{};  // CEEMDAN: the stage residue is final (its std runs on the side stream)
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    cudaEvent_t tm0 = nullptr, tm1 = nullptr;  // semd_timer_start / semd_timer_stop
    // multi-GPU: an NCCL communicator over one context per rank (semd_comm_init)
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, root = -1;  // root < 0: every rank receives the ensemble result
    DBuf comm_buf, comm_red;

    ~semd_ctx() {
        if (comm) nccl_api().CommDestroy(comm);
        if (tm0) cudaEventDestroy(tm0);
        if (tm1) cudaEventDestroy(tm1);
        if (status_host) cudaFreeHost(status_host);
        if (pin_jobs) cudaFreeHost(pin_jobs);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (t0) cudaEventDestroy(t0);
        if (t1) cudaEventDestroy(t1);
        for (auto& e : noise_ready)
            if (e) cudaEventDestroy(e);
        if (res_ready) cudaEventDestroy(res_ready);
        if (rng_stream) cudaStreamDestroy(rng_stream);
        if (own) cudaStreamDestroy(own);
    }

    void use() { ck(cudaSetDevice(device), "cudaSetDevice"); }

    // ---- arena --------------------------------------------------------------
    void configure(long long L, int G, int kcap, int trace_cap) {
        if (L >= (1LL << 30)) raise(SEMD_INVALID_INPUT, "signal too long for the engine (%lld samples)", L);
        A.kper = 0;  // batched drivers set it after configuring
        if (L == cfg_L && G == cfg_G && kcap == cfg_kcap && trace_cap == cfg_trace) return;
        const int tiles = (int)((L + semd::dev::kEvalTile - 1) / semd::dev::kEvalTile);
        const int cap = (int)((L / 2 + 2 + 3) / 4 * 4);  // 16-byte aligned knot rows (bulk TMA staging)
        const int rows_max = cap + 2;
        const int max_blocks = rows_max / semd::dev::kSolveBlock + 2;
        const long long Lp = (long long)tiles * semd::dev::kEvalTile;  // whole tiles: bulk copies stay inside
        bufs.alloc((size_t)G * semd::dev::kBufs * Lp * 8);
        kidx.alloc(((size_t)4 * G * cap + 16) * 4);
        const size_t t4 = ((size_t)tiles + 3) & ~(size_t)3, t4p = ((size_t)tiles + 4) & ~(size_t)3;
        const int chunks = (tiles + semd::dev::kScanChunk - 1) / semd::dev::kScanChunk;
        toff.alloc((size_t)4 * G * t4p * 4);
        tbase.alloc((size_t)4 * G * chunks * 4);
        ctot.alloc((size_t)2 * G * chunks * 4);
        cnum.alloc((size_t)G * chunks * 8);
        cden.alloc((size_t)G * chunks * 8);
        ktab.alloc(((size_t)2 * G * (cap + 8) + 16) * 32);
        scnt.alloc((size_t)2 * G * t4 * 4);
        tnum.alloc((size_t)G * t4 * 8);
        tden.alloc((size_t)G * t4 * 8);
        thash.alloc((size_t)2 * G * tiles * 8);
        tflags.alloc((size_t)2 * G * tiles * 32 * 4);
        slots.alloc((size_t)G * sizeof(Slot));
        sums.alloc((size_t)kcap * L * 8);
        imf_sifts.alloc((size_t)kcap * 4);
        ctrl.alloc(sizeof(Ctrl));
        lists.alloc((size_t)(G + G + G + 2 * G + 2 * G + 1) * 4);
        sb.alloc((size_t)2 * G * max_blocks * 6 * 8);
        if (trace_cap > 0) trace.alloc((size_t)trace_cap * sizeof(TraceRec));
        A = Arena{};
        A.L = (int)L;
        A.Lp = Lp;
        A.G = G;
        A.tiles = tiles;
        // short signals (C2/C3: ~50 tiles, hundreds of slots): shorter strips spread a step's
        // work over more warps (the step is as long as its longest strip)
        A.strip = tiles < 128 ? 4 : 16;
        A.cap = cap;
        A.kcap = kcap;
        A.bufs = bufs.as<double>();
        A.kidx = kidx.as<int>();
        A.toff = toff.as<unsigned>();
        A.tbase = tbase.as<unsigned>();
        A.ctot = ctot.as<unsigned>();
        A.cnum = cnum.as<double>();
        A.cden = cden.as<double>();
        A.chunks = chunks;
        A.ktab = ktab.as<double4>();
        A.scnt = scnt.as<unsigned>();
        A.tnum = tnum.as<double>();
        A.tden = tden.as<double>();
        A.thash = thash.as<unsigned long long>();
        A.tflags = tflags.as<unsigned>();
        A.slots = slots.as<Slot>();
        A.sums = sums.as<double>();
        A.imf_sifts = imf_sifts.as<int>();
        A.ctrl = ctrl.as<Ctrl>();
        int* l = lists.as<int>();
        A.eval_list = l;
        A.final_list = l + G;
        A.compact_list = l + 2 * G;
        A.solve_item = l + 3 * G;
        A.solve_off = l + 5 * G;
        A.sb = sb.as<double>();
        A.max_blocks = max_blocks;
        A.trace = trace_cap > 0 ? trace.as<TraceRec>() : nullptr;
        A.trace_cap = trace_cap;
        A.status_host = status_host_dev;
        hzlog.alloc((size_t)kHzCap * 8 * 4);
        A.hzlog = hzlog.as<int>();
        A.hzlog_cap = kHzCap;
        A.debug = debug_flags;
        prof.alloc(16 * 8);
        A.prof = prof.as<unsigned long long>();
        if (!spec_hist.p) {  // once per context: the statistics outlive reconfigurations
            spec_hist.alloc((size_t)semd::dev::kSpecK * semd::dev::kSpecS * 4);
            ck(cudaMemsetAsync(spec_hist.p, 0, spec_hist.bytes, stream), "memset spec_hist");
        }
        A.spec_hist = spec_hist.as<int>();
        ck(cudaMemsetAsync(toff.p, 0, toff.bytes, stream), "memset toff");
        ck(cudaMemsetAsync(tbase.p, 0, tbase.bytes, stream), "memset tbase");
        ck(cudaMemsetAsync(sb.p, 0, sb.bytes, stream), "memset sb");
        cfg_L = (int)L;
        cfg_G = G;
        cfg_kcap = kcap;
        cfg_trace = trace_cap;
        h_slots.assign(G, Slot{});
        for (auto& s : h_slots) s.epoch = 1;
    }

    // samples per lockstep step the slot count aims at (SEMD_STEP_SAMPLES overrides; tuning)
    static long long step_samples() {
        static const long long v = [] {
            const char* e = std::getenv("SEMD_STEP_SAMPLES");
            const long long x = e ? std::atoll(e) : 0;
            return x > 0 ? x : (512LL << 20);  // C5: 31 realizations per wave (fewer steps, amortised fixed costs)
        }();
        return v;
    }
    int auto_slots(long long L, int jobs) {
        long long g = step_samples() / std::max(1LL, L);
        g = std::max(1LL, std::min<long long>(g, 1024));
        if (max_slots > 0) g = std::min<long long>(g, max_slots);
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        // the engine's own slot-scaled buffers count as available (they are reused or regrown)
        const size_t held = bufs.bytes + kidx.bytes + toff.bytes + ktab.bytes + scnt.bytes + tnum.bytes + tden.bytes +
                            thash.bytes + tflags.bytes + sb.bytes + noise.bytes;
        const long long per_slot = 102LL * L + 4096;  // slot buffers, knot lists, tables, detection words, noise
        const long long mem_g = (long long)(0.5 * (double)(free_b + held)) / per_slot;
        g = std::max(1LL, std::min(g, mem_g));
        g = std::min<long long>(g, std::max(1, jobs));
        const long long waves = (std::max(1, jobs) + g - 1) / g;  // the same wave count, evenly filled
        return (int)((std::max(1, jobs) + waves - 1) / waves);
    }

    static int default_kcap(long long L, int max_imfs) {
        if (max_imfs > 0) return max_imfs;
        int lg = 0;
        while ((1LL << lg) < L) ++lg;
        return lg + 6;
    }

    // ---- one lockstep run over the configured slots -------------------------
    // Pinned staging: [G slots][Ctrl][G eval-list ints][a reset Ctrl, never modified]
    void ensure_pin(int G) {
        const size_t sb = (size_t)G * sizeof(Slot), cb = sizeof(Ctrl), lb = (size_t)G * 4;
        if (pin_jobs_bytes >= sb + 2 * cb + lb) return;
        if (pin_jobs) cudaFreeHost(pin_jobs);
        pin_jobs = nullptr;
        pin_jobs_bytes = 0;
        ck(cudaHostAlloc(reinterpret_cast<void**>(&pin_jobs), sb + 2 * cb + lb, cudaHostAllocDefault), "pinned jobs");
        pin_jobs_bytes = sb + 2 * cb + lb;
        Ctrl& z = *reinterpret_cast<Ctrl*>(pin_jobs + pin_jobs_bytes - cb);
        z = Ctrl{};
        z.ev_t0 = ~0ull;
    }
    const Ctrl* pin_reset_ctrl() const {
        return reinterpret_cast<const Ctrl*>(pin_jobs + pin_jobs_bytes - sizeof(Ctrl));
    }

    void set_jobs(const std::vector<JobSpec>& jobs) {
        const int G = A.G;
        for (int s = 0; s < G; ++s) {
            Slot& S = h_slots[s];
            const unsigned epoch = S.epoch;
            S = Slot{};
            S.epoch = epoch + 1;
            if (s < (int)jobs.size()) {
                const JobSpec& J = jobs[s];
                S.m = J.m;
                S.task = J.task;
                S.k = J.k;
                S.kmax = J.kmax;
                S.k0 = J.k0;
                S.init_kind = J.init_kind;
                S.write_imf = J.write_imf;
                S.detect_only = J.detect_only;
                S.beta = J.beta;
                S.init_a = J.a;
                S.init_b = J.b;
                S.imf_out = J.imf_out;
                S.res_out = J.res_out;
                S.state = semd::dev::ST_INIT;
                S.xb = 0;
                S.cb = -1;
                S.par = 0;
            } else {
                S.state = semd::dev::ST_FREE;
            }
        }
        // one pinned staging block: the uploads are truly asynchronous and the first step is
        // launched right behind them (the previous run's kernels have completed: run() synced)
        const size_t sb = (size_t)G * sizeof(Slot), cb = sizeof(Ctrl), lb = (size_t)G * 4;
        ensure_pin(G);
        std::memcpy(pin_jobs, h_slots.data(), sb);
        Ctrl& c = *reinterpret_cast<Ctrl*>(pin_jobs + sb);
        c = Ctrl{};
        c.ev_t0 = ~0ull;
        int* el = reinterpret_cast<int*>(pin_jobs + sb + cb);
        const int ne = std::min((int)jobs.size(), G);
        for (int s = 0; s < ne; ++s) el[s] = s;
        c.n_eval = ne;
        c.n_eval_pass = ne;
        c.active = ne;
        ck(cudaMemcpyAsync(A.slots, pin_jobs, sb, cudaMemcpyHostToDevice, stream), "upload slots");
        ck(cudaMemcpyAsync(A.ctrl, &c, cb, cudaMemcpyHostToDevice, stream), "upload ctrl");
        if (ne) ck(cudaMemcpyAsync(A.eval_list, el, (size_t)ne * 4, cudaMemcpyHostToDevice, stream), "lists");
        ck(cudaMemsetAsync(A.solve_off, 0, 4, stream), "lists");
        status_host[1] = 0;
        *(volatile int*)status_host = c.active;
    }

    // Block until the device has completed `target` steps of this run (the last CTA of
    // k_final publishes {active slots, completed steps} to mapped pinned memory). No
    // per-step events: they would break the programmatic-dependent-launch chain.
    void wait_steps(int target) {
        volatile int* hs = status_host;
        for (unsigned spin = 0; hs[1] < target; ++spin) {
            if ((spin & 1023u) == 1023u) {
                const cudaError_t e = cudaStreamQuery(stream);
                if (e == cudaSuccess) {  // drained: the counter is final
                    if (hs[1] < target) break;
                } else if (e != cudaErrorNotReady) {
                    ck(e, "engine step");
                }
            }
        }
    }

    // steps launched ahead of the one the host waits for (SEMD_LAG overrides; tuning)
    static int lag_steps() {
        static const int v = [] {
            const char* e = std::getenv("SEMD_LAG");
            const int x = e ? std::atoi(e) : 0;
            return x > 0 ? x : 2;
        }();
        return v;
    }
    // SEMD_SPEC=0 turns the speculative last sifts off, =2 makes every sift speculative (A/B runs)
    static int spec_env_bits() {
        static const int v = [] {
            const char* e = std::getenv("SEMD_SPEC");
            return !e ? 0 : (e[0] == '0' ? 8 : (e[0] == '2' ? 16 : 0));
        }();
        return v;
    }
    void run(int max_steps) {
        A.debug = debug_flags | spec_env_bits();
        const int LAG = lag_steps();
        int step = 0;
        for (;; ++step) {
            semd::dev::launch_step(A, sms, stream);
            stats.eval_launches += 1;
            ck(cudaGetLastError(), "launch step");
            if (step >= LAG) {
                wait_steps(step - LAG + 1);
                if (*(volatile int*)status_host == 0) break;
            }
            if (step > max_steps) {
                cudaStreamSynchronize(stream);
                std::string d;
                if (cudaMemcpy(h_slots.data(), A.slots, (size_t)A.G * sizeof(Slot), cudaMemcpyDeviceToHost) ==
                    cudaSuccess) {
                    char b[160];
                    for (int i = 0; i < A.G && i < 8; ++i) {
                        const Slot& S = h_slots[i];
                        std::snprintf(b, sizeof b, " [m%d st%d k%d it%d n%u/%u par%d xb%d cb%d]", S.m, S.state, S.k,
                                      S.iter, S.n[0], S.n[1], S.par, S.xb, S.cb);
                        d += b;
                    }
                }
                raise(SEMD_CUDA_ERROR, "engine did not converge within %d steps;%s", max_steps, d.c_str());
            }
        }
        // slots and control block back through the pinned block, one synchronisation
        ensure_pin(A.G);
        const size_t sb = (size_t)A.G * sizeof(Slot);
        ck(cudaMemcpyAsync(pin_jobs, A.slots, sb, cudaMemcpyDeviceToHost, stream), "download slots");
        ck(cudaMemcpyAsync(pin_jobs + sb, A.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream), "download ctrl");
        ck(cudaStreamSynchronize(stream), "engine run");
        stats.steps += step + 1;
        std::memcpy(h_slots.data(), pin_jobs, sb);
        Ctrl c;
        std::memcpy(&c, pin_jobs + sb, sizeof(Ctrl));
        for (const Slot& S : h_slots) {
            stats.sifted_samples += (uint64_t)S.sifted;
            stats.sift_iterations += (uint64_t)(S.sifted / std::max(1, A.L));
        }
        stats.solve_hazards += (uint64_t)c.hazards;
        spec_stats[0] += (unsigned long long)c.spec_pass;
        spec_stats[1] += (unsigned long long)c.spec_hits;
        spec_stats[2] += (unsigned long long)c.spec_misses;
        spec_stats[3] += (unsigned long long)(step + 1);
        stats.sd_rechecks += (uint64_t)c.sd_rechecks;
        if (timing) stats.eval_ms += (double)c.ev_ns * 1e-6;
        for (int id = 0; id < 5; ++id) {  // the spans the last two steps left unfolded
            unsigned long long ns = c.kns[id];
            for (int p = 0; p < 2; ++p) {
                const unsigned long long a = c.kt[p][id][0], b = c.kt[p][id][1];
                if (a && b && b > ~a) ns += b - ~a;
            }
            span_ms[id] += (double)ns * 1e-6;
        }
        span_strips[0] += c.strips[0];
        span_strips[1] += c.strips[1];
        span_strips[2] += c.strip_cyc[0];
        span_strips[3] += c.strip_cyc[1];
        if (c.hz_count > 0) {
            const int n = std::min(c.hz_count, kHzCap);
            const size_t old = h_hz.size();
            h_hz.resize(old + (size_t)n * 8);
            ck(cudaMemcpy(h_hz.data() + old, A.hzlog, (size_t)n * 8 * 4, cudaMemcpyDeviceToHost), "hazard log");
        }
        if (c.k_overflow) raise(SEMD_CAPACITY, "IMF capacity exceeded (%d rows)", A.kcap);
        if (A.trace) {
            const int n = std::min(c.trace_count, A.trace_cap);
            const size_t old = h_trace.size();
            h_trace.resize(old + n);
            if (n) ck(cudaMemcpy(h_trace.data() + old, A.trace, (size_t)n * sizeof(TraceRec), cudaMemcpyDeviceToHost),
                      "trace");
            trace_total += c.trace_count;
        }
        // reset counters for the next run
        ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
    }
    long long trace_total = 0;
    double span_ms[5] = {};                 // device spans of the step kernels (semd_kernel_spans)
    unsigned long long span_strips[4] = {};  // eval strips: DETECT/INIT mode, SIFT mode; their warp cycles
    unsigned long long spec_stats[4] = {};   // speculative last sifts: run, stopped, continued; lockstep steps
    static constexpr int kHzCap = 4096;
    int debug_flags = 0;
    std::vector<int> h_hz;  // solve-hazard records since reset_stats (test hook)

    int max_steps_for(const semd_sift_cfg& cfg) const {
        const long long it = 2LL * std::max(1, cfg.max_sift_iters) + 2;  // + a detection step per speculative miss
        return (int)std::min<long long>((long long)(A.kcap + 2) * it + 64, 1LL << 30);
    }

    // ---- the resident engine (semd_resident.cu): short signals, one persistent CTA per job ----
    int engine = SEMD_ENGINE_AUTO;
    DBuf r_jobs, r_res, r_store, r_sifts, r_scratch, r_ticket, r_noise, r_prof, r_rows;
    DBuf ser_sig, ser_modes, ser_out;  // serial_decompose scratch (grow-only)
    bool r_prof_init = false;
    cudaEvent_t r_t0 = nullptr, r_t1 = nullptr;  // SEMD_RES_LOG timing
    std::vector<semd::dev::RResult> r_out;
    static int env_engine() {
        static const int v = [] {
            const char* e = std::getenv("SEMD_ENGINE");
            if (e && std::strcmp(e, "lockstep") == 0) return (int)SEMD_ENGINE_LOCKSTEP;
            if (e && std::strcmp(e, "resident") == 0) return (int)SEMD_ENGINE_RESIDENT;
            return (int)SEMD_ENGINE_AUTO;
        }();
        return v;
    }
    // segment-table rows (16 B) the resident kernel's shared memory holds next to a length-L candidate
    static int res_tab_rows(long long L) {
        const long long fixed = (long long)semd::dev::resident_smem_bytes((int)L, 0);
        return (int)std::max(0LL, ((long long)semd::dev::resident_max_smem() - fixed) / 16);
    }
    static int res_chain_div() {
        static const int v = [] {
            const char* e = std::getenv("SEMD_RES_CHAINS");
            return e ? std::atoi(e) : 0;
        }();
        return v;
    }
    void res_timer_start() {
        if (!r_t0) {
            ck(cudaEventCreate(&r_t0), "event");
            ck(cudaEventCreate(&r_t1), "event");
        }
        ck(cudaEventRecord(r_t0, stream), "ev");
    }
    bool resident_for(long long L) const {
        const int mode = engine != SEMD_ENGINE_AUTO ? engine : env_engine();
        if (mode == SEMD_ENGINE_LOCKSTEP) return false;
        if (L < 4 || L > semd::dev::kResMaxL) return false;
        return res_tab_rows(L) >= 64;
    }
    static Slot slot_from(const semd::dev::RResult& r) {
        Slot S{};
        S.k = r.k;
        S.ended_insufficient = r.ended_insufficient;
        S.n[0] = r.n0;
        S.n[1] = r.n1;
        S.sifted = r.sifted;
        S.state = semd::dev::ST_DONE;
        return S;
    }
    // All jobs in one launch of the resident engine (the arena must be configured for L: its sums,
    // trace and control block are used). write_imf jobs keep up to kc IMFs each, accumulated into
    // A.sums in job order afterwards (k_res_accum); job 0's sift counts go to A.imf_sifts and its
    // final residue to res_final0. Results per job in r_out. Jobs whose segment tables outgrow the
    // shared memory are listed in *failed; when one of them accumulates IMFs nothing is accumulated
    // and false is returned (the caller reruns the whole call on the lockstep engine, keeping the
    // realization order of the sums).
    bool run_resident(const std::vector<JobSpec>& js, int kc, std::vector<int>* failed, double* res_final0 = nullptr) {
        using namespace semd::dev;
        failed->clear();
        ensure_pin(A.G);
        const int nj = (int)js.size();
        const int L = A.L;
        const long long Lp = (L + 3) & ~3;
        std::vector<RJob> h(nj);
        bool any_write = false;
        for (int i = 0; i < nj; ++i) {
            const JobSpec& J = js[i];
            RJob R{};
            R.m = J.m;
            R.task = J.task;
            R.k = J.k;
            R.kmax = J.kmax;
            R.k0 = J.k0;
            R.init_kind = J.init_kind;
            R.write_imf = J.write_imf;
            R.detect_only = J.detect_only;
            R.beta = J.beta;
            R.a = J.a;
            R.b = J.b;
            R.imf_out = J.imf_out;
            R.res_out = J.res_out;
            R.res_final = i == 0 ? res_final0 : nullptr;
            h[i] = R;
            any_write = any_write || (J.write_imf && !J.detect_only);
        }
        kc = std::max(1, kc);
        const int grid = std::max(1, std::min(nj, sms));
        r_jobs.alloc((size_t)nj * sizeof(RJob));
        r_res.alloc((size_t)nj * sizeof(RResult));
        r_sifts.alloc((size_t)nj * kc * 4);
        if (any_write) r_store.alloc((size_t)nj * kc * Lp * 8);
        r_scratch.alloc((size_t)grid * 2 * Lp * 8);
        r_ticket.alloc(16);
        ck(cudaMemcpyAsync(r_jobs.p, h.data(), (size_t)nj * sizeof(RJob), cudaMemcpyHostToDevice, stream), "jobs");
        ck(cudaMemsetAsync(r_ticket.p, 0, 16, stream), "ticket");
        // the trace and SD-recheck counters live in the control block: start from a reset one (the
        // lockstep engine uploads its own per run; a fresh context's block is uninitialised)
        ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
        ResArgs P{};
        P.jobs = r_jobs.as<RJob>();
        P.res = r_res.as<RResult>();
        P.njobs = nj;
        P.L = L;
        P.store = any_write ? r_store.as<double>() : nullptr;
        P.kc = kc;
        P.sifts = r_sifts.as<int>();
        P.scratch = r_scratch.as<double>();
        P.ticket = r_ticket.as<unsigned>();
        P.max_iters = A.max_sift_iters;
        P.sd_thr = A.sd_threshold;
        P.tab_rows = res_tab_rows(L);
        P.trace = A.trace_cap > 0 ? A.trace : nullptr;
        P.trace_cap = A.trace_cap;
        P.trace_count = &A.ctrl->trace_count;
        P.sd_rechecks = &A.ctrl->sd_rechecks;
        P.debug = debug_flags;
        P.chain_div = res_chain_div();
        if (debug_flags & 2) {
            r_prof.alloc(128);
            if (!r_prof_init) {
                ck(cudaMemsetAsync(r_prof.p, 0, 128, stream), "prof");
                r_prof_init = true;
            }
            P.prof = r_prof.as<unsigned long long>();
        }
        static const bool res_log = std::getenv("SEMD_RES_LOG") != nullptr;
        const bool timed = res_log || timing;
        if (timed) res_timer_start();
        launch_resident(P, grid, stream);
        ck(cudaGetLastError(), "resident launch");
        if (timed) ck(cudaEventRecord(r_t1, stream), "ev");
        r_out.resize(nj);
        ck(cudaMemcpyAsync(r_out.data(), r_res.p, (size_t)nj * sizeof(RResult), cudaMemcpyDeviceToHost, stream),
           "resident results");
        ck(cudaStreamSynchronize(stream), "resident run");  // also keeps h alive for the upload
        if (timed) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r_t0, r_t1);
            stats.eval_ms += ms;  // the dominant (sift) kernel's device time
        }
        if (res_log) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r_t0, r_t1);
            long long sifts = 0;
            int maxs = 0;
            for (int i = 0; i < nj; ++i) {
                sifts += r_out[i].sifted / std::max(1, L);
                maxs = std::max(maxs, (int)(r_out[i].sifted / std::max(1, L)));
            }
            std::fprintf(stderr, "[resident] jobs %d task %d L %d: %.3f ms, sifts %lld (max per job %d)\n", nj,
                         js[0].task, L, ms, sifts, maxs);
        }
        bool fail_write = false, overflow = false;
        for (int i = 0; i < nj; ++i) {
            if (r_out[i].smem_overflow) {
                failed->push_back(i);
                fail_write = fail_write || (h[i].write_imf && !h[i].detect_only);
            }
            overflow = overflow || r_out[i].k_overflow;
        }
        if (fail_write || overflow) {  // nothing of this run is kept (its traces neither)
            ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
            ck(cudaStreamSynchronize(stream), "ctrl reset");
            if (overflow && !fail_write) raise(SEMD_CAPACITY, "IMF capacity exceeded (%d rows)", kc);
            return false;
        }
        if (any_write) {  // per sums row, the range of jobs that can write it (job rows non-decreasing)
            const int rows = A.kcap;
            std::vector<int> rj(2 * (size_t)rows);
            bool sorted = true;
            for (int i = 1; i < nj; ++i) sorted = sorted && h[i].k0 + h[i].k >= h[i - 1].k0 + h[i - 1].k;
            int lo = 0, hi = 0;
            for (int r = 0; r < rows; ++r) {
                while (sorted && lo < nj && h[lo].k0 + h[lo].k + kc <= r) ++lo;
                while (sorted && hi < nj && h[hi].k0 + h[hi].k <= r) ++hi;
                rj[2 * (size_t)r] = sorted ? lo : 0;
                rj[2 * (size_t)r + 1] = sorted ? std::max(lo, hi) : nj;
            }
            r_rows.alloc(rj.size() * 4);
            ck(cudaMemcpyAsync(r_rows.p, rj.data(), rj.size() * 4, cudaMemcpyHostToDevice, stream), "rows");
            launch_res_accum(P.jobs, P.res, r_rows.as<int>(), P.store, kc, Lp, L, A.sums, rows, stream);
            ck(cudaStreamSynchronize(stream), "accumulate");  // rj lifetime
        }
        if (A.imf_sifts && js[0].write_imf && !js[0].detect_only) {
            const int base = js[0].k0 + js[0].k;
            const int cnt = std::min(r_out[0].produced, std::max(0, A.kcap - base));
            if (cnt > 0)
                ck(cudaMemcpyAsync(A.imf_sifts + base, r_sifts.p, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, stream),
                   "sift counts");
        }
        ck(cudaGetLastError(), "resident accumulate");
        Ctrl c;
        ck(cudaMemcpyAsync(pin_jobs, A.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream), "ctrl");
        ck(cudaStreamSynchronize(stream), "resident");
        std::memcpy(&c, pin_jobs, sizeof(Ctrl));
        for (int i = 0; i < nj; ++i) {
            stats.sifted_samples += (uint64_t)r_out[i].sifted;
            stats.sift_iterations += (uint64_t)(r_out[i].sifted / std::max(1, L));
            stats.solve_hazards += (uint64_t)r_out[i].hazards;
        }
        stats.resident_jobs += (uint64_t)nj;
        stats.sd_rechecks += (uint64_t)c.sd_rechecks;
        if (A.trace) {
            const int n = std::min(c.trace_count, A.trace_cap);
            const size_t old = h_trace.size();
            h_trace.resize(old + n);
            if (n) ck(cudaMemcpy(h_trace.data() + old, A.trace, (size_t)n * sizeof(TraceRec), cudaMemcpyDeviceToHost),
                      "trace");
            trace_total += c.trace_count;
        }
        ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
        return true;
    }

    unsigned long long launches_at_reset = 0;
    void reset_stats(int slots_used) {
        stats = semd_stats{};
        h_hz.clear();
        stats.slots = slots_used;
        launches_at_reset = semd::dev::launch_count();
    }

    double* buf(int slot, int b) { return A.bufs + semd::dev::buf_off(A, slot, b); }

    // host out[i] = src[idx[i]] (extremum values: the samples at the extrema), gathered on the device
    void gather_values(const int* d_idx, unsigned n, const double* d_src, double* out) {
        scratch2.alloc((size_t)n * 8 + 8);
        semd::dev::launch_gather(d_idx, n, d_src, scratch2.as<double>(), stream);
        ck(cudaGetLastError(), "gather");
        ck(cudaMemcpyAsync(out, scratch2.p, (size_t)n * 8, cudaMemcpyDeviceToHost, stream), "values");
        ck(cudaStreamSynchronize(stream), "values");
    }

    void fill_sums(int rows, double value) {
        // +0.0 for ensembles (the reference's Signal(n, 0.0)), -0.0 where the
        // accumulator must reproduce the IMF bit-for-bit (-0.0 + v == v).
        const long long n = (long long)rows * A.L;
        if (value == 0.0 && !std::signbit(value)) ck(cudaMemsetAsync(A.sums, 0, (size_t)n * 8, stream), "memset sums");
        else semd::dev::launch_fill(A.sums, n, value, stream);
    }

    // ---- multi-GPU collectives (NCCL on the engine stream: stream-ordered with the kernels) ----
    long long comm_max(long long v) {
        if (!comm) return v;
        comm_buf.alloc(64);
        long long* d = comm_buf.as<long long>();
        ck(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, stream), "comm max");
        nck(nccl().AllReduce(d, d, 1, ncclInt64, ncclMax, comm, stream), "ncclAllReduce(max)");
        ck(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, stream), "comm max");
        ck(cudaStreamSynchronize(stream), "comm max");
        return v;
    }
    // in-place sum over ranks: to the root only when root >= 0 and root_only, else to every rank
    void comm_sum(double* d, size_t count, bool root_only) {
        if (!comm || count == 0) return;
        if (root_only && root >= 0)
            nck(nccl().Reduce(d, d, count, ncclDouble, ncclSum, root, comm, stream), "ncclReduce(sum)");
        else
            nck(nccl().AllReduce(d, d, count, ncclDouble, ncclSum, comm, stream), "ncclAllReduce(sum)");
    }
    bool has_result() const { return !comm || root < 0 || rank == root; }

    // more IMF rows for the configured engine, keeping rows [0, kcap) (CEEMDAN stages past the
    // initial estimate; the reference's IMF list is unbounded when max_imfs == 0)
    void grow_sums(int newk) {
        if (newk <= A.kcap) return;
        const size_t n = (size_t)A.L, old = (size_t)A.kcap;
        DBuf t((size_t)newk * n * 8);
        ck(cudaMemsetAsync(t.p, 0, t.bytes, stream), "grow sums");
        ck(cudaMemcpyAsync(t.p, sums.p, old * n * 8, cudaMemcpyDeviceToDevice, stream), "grow sums");
        DBuf c((size_t)newk * 4);
        ck(cudaMemsetAsync(c.p, 0, c.bytes, stream), "grow counts");
        ck(cudaMemcpyAsync(c.p, imf_sifts.p, old * 4, cudaMemcpyDeviceToDevice, stream), "grow counts");
        ck(cudaStreamSynchronize(stream), "grow sums");
        std::swap(sums.p, t.p);
        std::swap(sums.bytes, t.bytes);
        std::swap(imf_sifts.p, c.p);
        std::swap(imf_sifts.bytes, c.bytes);
        A.sums = sums.as<double>();
        A.imf_sifts = imf_sifts.as<int>();
        A.kcap = newk;
        cfg_kcap = newk;
    }

    // ---- drivers ---------------------------------------------------------------
    // emd.cpp:155-172 on a device signal; returns K. IMFs in sums rows, residue in buffer.
    int emd_device(const double* d_x, long long n, const semd_sift_cfg& cfg, semd_trace* tr, int m = 0) {
        if (n < 4) raise(SEMD_INVALID_INPUT, "emd: signal too short (need at least 4 samples)");
        int kcap = default_kcap(n, cfg.max_imfs);
        for (int attempt = 0;; ++attempt) {
            configure(n, 1, kcap, tr ? trace_cap_for(tr) : 0);
            A.sd_threshold = cfg.sd_threshold;
            A.max_sift_iters = cfg.max_sift_iters;
            fill_sums(kcap, -0.0);
            JobSpec J;
            J.m = m;
            J.task = 0;
            J.kmax = cfg.max_imfs;
            J.a = d_x;
            h_trace.clear();
            trace_total = 0;
            try {
                if (resident_for(n)) {
                    std::vector<int> failed;
                    if (run_resident({J}, kcap, &failed, buf(0, 0))) {
                        h_slots[0] = slot_from(r_out[0]);
                        h_slots[0].xb = 0;
                        return h_slots[0].k;
                    }
                    fill_sums(kcap, -0.0);  // the tables outgrew the resident engine: lockstep below
                }
                set_jobs({J});
                run(max_steps_for(cfg));
            } catch (const Error& e) {
                if (e.code == SEMD_CAPACITY && attempt < 3 && cfg.max_imfs == 0) {
                    kcap *= 2;
                    continue;
                }
                throw;
            }
            return h_slots[0].k;
        }
    }
    int trace_cap_for(const semd_trace* tr) const { return tr && tr->cap ? (int)std::min<size_t>(tr->cap, 1u << 26) : 0; }

    void export_trace(semd_trace* tr) {
        if (!tr) return;
        tr->count = (size_t)trace_total;
        const size_t n = std::min(tr->cap, h_trace.size());
        if (n && tr->rec) std::memcpy(tr->rec, h_trace.data(), n * sizeof(semd_trace_rec));
    }

    // white noise for realizations ms[0..g) into the noise buffer (stride Ls), std 1.
    void gen_noise(const std::vector<uint64_t>& seeds, long long n, long long Ls, double* dst, double stdv = 1.0) {
        const int g = (int)seeds.size();
        std::vector<semd::dev::RngJob> jobs(g);
        for (int i = 0; i < g; ++i) {
            jobs[i].seed = seeds[i];
            jobs[i].out = reinterpret_cast<uint64_t*>(dst + (size_t)i * Ls);
            jobs[i].n = n;
        }
        rng_jobs.alloc(jobs.size() * sizeof(semd::dev::RngJob));
        ck(cudaMemcpyAsync(rng_jobs.p, jobs.data(), jobs.size() * sizeof(semd::dev::RngJob), cudaMemcpyHostToDevice,
                           stream),
           "rng jobs");
        semd::dev::launch_rng(rng_jobs.as<semd::dev::RngJob>(), g, stream);
        semd::dev::launch_box_muller(reinterpret_cast<uint64_t*>(dst), (long long)g * Ls, stdv, stream);
        ck(cudaGetLastError(), "rng");
        ck(cudaStreamSynchronize(stream), "rng sync");  // jobs vector lifetime
    }

    // Workspace of the parallel (still reference-ordered) signal_std; null for short signals and
    // under debug bit 32, which keeps the single-thread kernel (tests compare the two).
    long long std_last_n = 0;
    void* std_workspace(long long n) {
        const size_t b = (debug_flags & 32) ? 0 : semd::dev::signal_std_workspace(n);
        std_last_n = b ? n : 0;
        if (!b) return nullptr;
        std_ws.alloc(b);
        return std_ws.p;
    }
    double device_std(const double* d_x, long long n, double scale) {
        scalar.alloc((2 + 2 * 256 + 8) * 8);
        semd::dev::launch_signal_std(d_x, n, scalar.as<double>(), scale, stream, std_workspace(n));
        double v = 0.0;
        ck(cudaMemcpyAsync(&v, scalar.p, 8, cudaMemcpyDeviceToHost, stream), "std");
        ck(cudaStreamSynchronize(stream), "std");
        return v;
    }

    // EEMD realizations [m_begin, m_end): unscaled sums in A.sums rows; returns max K.
    const double* noise_override = nullptr;  // test hook: nr x n noise (device)
    int eemd_partial_device(const double* d_x, long long n, const semd_sift_cfg& cfg, const semd_ens_cfg& ens,
                            int m_begin, int m_end, semd_trace* tr) {
        if (n < 4) raise(SEMD_INVALID_INPUT, "emd: signal too short (need at least 4 samples)");
        const int jobs = std::max(0, m_end - m_begin);
        bool res = jobs > 0 && resident_for(n);
        int G = res ? 1 : auto_slots(n, jobs);  // the resident engine needs no lockstep slots
        // W balanced waves (sizes differ by at most one): a short last wave would cost nearly a
        // full wave of lockstep steps
        int W = jobs > 0 ? (jobs + G - 1) / G : 0;
        auto wave = [&](int i, int& w0, int& g) {
            const int base = jobs / W, extra = jobs % W;
            w0 = m_begin + i * base + std::min(i, extra);
            g = base + (i < extra ? 1 : 0);
        };
        int kcap = default_kcap(n, cfg.max_imfs);
        const long long Ls = (n + 1) / 2 * 2;
        if (res && !noise_override) {  // every realization's noise (side stream), overlapping the std
            r_noise.alloc((size_t)jobs * Ls * 8);
            semd::dev::launch_rng_ensemble(ens.base_seed, m_begin, jobs, reinterpret_cast<uint64_t*>(r_noise.as<double>()),
                                           Ls, n, rng_stream);
            semd::dev::launch_box_muller(reinterpret_cast<uint64_t*>(r_noise.as<double>()), (long long)jobs * Ls, 1.0,
                                         rng_stream);
            ck(cudaGetLastError(), "rng");
            ck(cudaEventRecord(noise_ready[1], rng_stream), "rng event");
        }
        // the first wave's noise (side stream) overlaps the sequential std on the main stream
        bool first_noise_ready = false;
        if (!noise_override && jobs > 0 && !res) {
            int fw0, fg;
            wave(0, fw0, fg);
            noise.alloc((size_t)2 * G * Ls * 8);
            semd::dev::launch_rng_ensemble(ens.base_seed, fw0, fg, reinterpret_cast<uint64_t*>(noise.as<double>()), Ls,
                                           n, rng_stream);
            semd::dev::launch_box_muller(reinterpret_cast<uint64_t*>(noise.as<double>()), (long long)fg * Ls, 1.0,
                                         rng_stream);
            ck(cudaGetLastError(), "rng");
            ck(cudaEventRecord(noise_ready[0], rng_stream), "rng event");
            first_noise_ready = true;
        }
        const double beta = device_std(d_x, n, ens.nstd);  // emd.cpp:233
        for (int attempt = 0;; ++attempt) {
            configure(n, G, kcap, tr ? trace_cap_for(tr) : 0);
            A.sd_threshold = cfg.sd_threshold;
            A.max_sift_iters = cfg.max_sift_iters;
            semd::dev::launch_spec_decay(A.spec_hist, stream);  // the speculation policy's memory fades per call
            noise.alloc((size_t)2 * G * Ls * 8);  // double-buffered: wave i+1's noise is made during wave i
            fill_sums(kcap, 0.0);
            h_trace.clear();
            trace_total = 0;
            int kmax_seen = 0, waves = 0;
            auto nbuf = [&](int b) { return noise.as<double>() + (size_t)b * G * Ls; };
            // noise of wave i lives in buffer i%2; generated on rng_stream (buffer i%2 was last read
            // by wave i-2, whose run() the host has already synchronized), signalled by noise_ready
            auto make_noise = [&](int wi, int b) {
                int w0, g;
                wave(wi, w0, g);
                semd::dev::launch_rng_ensemble(ens.base_seed, w0, g, reinterpret_cast<uint64_t*>(nbuf(b)), Ls, n,
                                               rng_stream);
                semd::dev::launch_box_muller(reinterpret_cast<uint64_t*>(nbuf(b)), (long long)g * Ls, 1.0, rng_stream);
                ck(cudaGetLastError(), "rng");
                ck(cudaEventRecord(noise_ready[b], rng_stream), "rng event");
            };
            try {
                if (res) {  // every realization in one resident-engine launch, summed in m order
                    if (!noise_override) ck(cudaStreamWaitEvent(stream, noise_ready[1], 0), "noise wait");
                    std::vector<JobSpec> js(jobs);
                    for (int i = 0; i < jobs; ++i) {
                        JobSpec& J = js[i];
                        J.m = m_begin + i;
                        J.task = 0;
                        J.kmax = cfg.max_imfs;
                        J.init_kind = 1;
                        J.beta = beta;
                        J.a = d_x;
                        J.b = noise_override ? noise_override + (size_t)(m_begin + i) * n
                                             : r_noise.as<double>() + (size_t)i * Ls;
                    }
                    std::vector<int> failed;
                    if (run_resident(js, kcap, &failed)) {
                        for (int i = 0; i < jobs; ++i) kmax_seen = std::max(kmax_seen, r_out[i].k);
                        stats.waves += 1;
                        stats.slots = std::min(jobs, sms);
                        return kmax_seen;
                    }
                    // the tables outgrew the resident engine: the lockstep engine, sized for it
                    res = false;
                    G = auto_slots(n, jobs);
                    W = (jobs + G - 1) / G;
                    --attempt;
                    continue;
                }
                if (!noise_override && !first_noise_ready && W > 0) make_noise(0, 0);
                first_noise_ready = false;  // a capacity retry regenerates it
                for (int wi = 0; wi < W; ++wi) {
                    int w0, g;
                    wave(wi, w0, g);
                    const int b = wi & 1;
                    std::vector<JobSpec> js(g);
                    if (!noise_override) {
                        if (wi + 1 < W) make_noise(wi + 1, b ^ 1);  // overlaps this wave's sifting
                        ck(cudaStreamWaitEvent(stream, noise_ready[b], 0), "noise wait");
                    }
                    for (int i = 0; i < g; ++i) {
                        JobSpec& J = js[i];
                        J.m = w0 + i;
                        J.task = 0;
                        J.kmax = cfg.max_imfs;
                        J.init_kind = 1;
                        J.beta = beta;
                        J.a = d_x;
                        J.b = noise_override ? noise_override + (size_t)(w0 + i) * n : nbuf(b) + (size_t)i * Ls;
                    }
                    set_jobs(js);
                    run(max_steps_for(cfg));
                    ++waves;
                    for (int i = 0; i < g; ++i) kmax_seen = std::max(kmax_seen, h_slots[i].k);
                }
                ck(cudaStreamSynchronize(rng_stream), "rng");
            } catch (const Error& e) {
                cudaStreamSynchronize(rng_stream);
                if (e.code == SEMD_CAPACITY && attempt < 3 && cfg.max_imfs == 0) {
                    kcap *= 2;
                    continue;
                }
                throw;
            }
            stats.waves += waves;
            stats.slots = G;
            return kmax_seen;
        }
    }

    // ---- CEEMDAN (emd.cpp:264-344) as stages over a realization shard [m0, m1) ----------
    // begin -> stage 0 -> finish -> { residue_extrema >= 3 ? stage K -> finish : stop }.
    // A stage leaves the UNSCALED sum of the shard's first modes (realization order) in
    // sums row K; finish takes the all-shard total (this row on one GPU, an all-reduced
    // copy across GPUs), scales it by 1/nr, applies the all-zero stop (emd.cpp:332-337) and
    // updates the residue. Every rank holds the same residue, so beta_i, the stop tests and
    // the modes are identical on all ranks.
    struct CeemdanShard {
        bool active = false;
        const double* x = nullptr;
        long long n = 0, Ls = 0;
        semd_sift_cfg cfg{};
        semd_ens_cfg ens{};
        int m0 = 0, m1 = 0, G = 1, kcap = 0, K = 0, waves = 0;
        double beta0 = 0.0;
        std::vector<char> alive;
    } cs;
    double* cs_noise() { return noise.as<double>(); }         // shard noise residues (Ls stride)
    double* cs_E() { return scratch.as<double>(); }           // E_i(w^(m)) of the shard (n stride)
    double* cs_residue() { return scratch2.as<double>(); }
    int* cs_flag() { return reinterpret_cast<int*>(scratch2.as<double>() + cs.n); }

    void ceemdan_begin(const double* d_x, long long n, const semd_sift_cfg& cfg, const semd_ens_cfg& ens, int m0,
                       int m1, semd_trace* tr) {
        if (n < 4) raise(SEMD_INVALID_INPUT, "ceemdan: signal too short (need at least 4 samples)");
        if (m0 < 0 || m1 < m0 || m1 > ens.nr) raise(SEMD_INVALID_INPUT, "invalid realization range");
        cs = CeemdanShard{};
        cs.x = d_x;
        cs.n = n;
        cs.Ls = (n + 1) / 2 * 2;
        cs.cfg = cfg;
        cs.ens = ens;
        cs.m0 = m0;
        cs.m1 = m1;
        const int cnt = m1 - m0;
        // lockstep slots only when the stage jobs can run on the lockstep engine (the resident
        // engine needs none; auto_slots queries the free memory)
        cs.G = resident_for(n) ? 1 : auto_slots(n, std::max(1, cnt));
        cs.kcap = default_kcap(n, cfg.max_imfs);
        configure(n, cs.G, cs.kcap, tr ? trace_cap_for(tr) : 0);
        A.sd_threshold = cfg.sd_threshold;
        A.max_sift_iters = cfg.max_sift_iters;
        h_trace.clear();
        trace_total = 0;
        noise.alloc((size_t)std::max(1, cnt) * cs.Ls * 8);
        scratch.alloc((size_t)std::max(1, cnt) * n * 8);
        scratch2.alloc((size_t)n * 8 * 2);
        if (noise_override) {
            for (int i = 0; i < cnt; ++i)
                ck(cudaMemcpyAsync(cs_noise() + (size_t)i * cs.Ls, noise_override + (size_t)(m0 + i) * n, n * 8,
                                   cudaMemcpyDeviceToDevice, stream),
                   "noise override");
        } else if (cnt > 0) {  // w^(m) on the side stream (seeds derive_seed(base, m) on the device),
            // overlapping the sequential std below
            semd::dev::launch_rng_ensemble(ens.base_seed, m0, cnt, reinterpret_cast<uint64_t*>(cs_noise()), cs.Ls, n,
                                           rng_stream);
            semd::dev::launch_box_muller(reinterpret_cast<uint64_t*>(cs_noise()), (long long)cnt * cs.Ls, 1.0,
                                         rng_stream);
            ck(cudaGetLastError(), "rng");
            ck(cudaEventRecord(noise_ready[1], rng_stream), "rng event");
        }
        cs.alive.assign(cnt, 1);
        semd::dev::launch_copy(d_x, cs_residue(), n, stream);
        fill_sums(cs.kcap, 0.0);
        cs.beta0 = device_std(d_x, n, ens.nstd);  // emd.cpp:293
        if (!noise_override && cnt > 0) ck(cudaStreamWaitEvent(stream, noise_ready[1], 0), "noise wait");
        cs.active = true;
    }

    void cs_run_tasks(std::vector<JobSpec>& all, std::vector<Slot>* results) {
        results->resize(all.size());
        if (!all.empty() && resident_for(cs.n)) {
            std::vector<int> failed;
            if (run_resident(all, 1, &failed)) {
                for (size_t i = 0; i < all.size(); ++i) (*results)[i] = slot_from(r_out[i]);
                cs.waves += 1;
                if (failed.empty()) return;
                // jobs whose tables outgrew the shared memory (none of them accumulates): lockstep
                std::vector<JobSpec> rest;
                for (int i : failed) rest.push_back(all[i]);
                std::vector<Slot> rr;
                cs_run_lockstep(rest, &rr);
                for (size_t q = 0; q < failed.size(); ++q) (*results)[failed[q]] = rr[q];
                return;
            }
        }
        cs_run_lockstep(all, results);
    }
    void cs_run_lockstep(std::vector<JobSpec>& all, std::vector<Slot>* results) {
        results->resize(all.size());
        for (size_t w0 = 0; w0 < all.size(); w0 += cs.G) {
            const size_t g = std::min<size_t>(cs.G, all.size() - w0);
            std::vector<JobSpec> js(all.begin() + w0, all.begin() + w0 + g);
            set_jobs(js);
            run(max_steps_for(cs.cfg));
            ++cs.waves;
            for (size_t i = 0; i < g; ++i) (*results)[w0 + i] = h_slots[i];
        }
    }

    // find_extrema(residue).total() (emd.cpp:311)
    long long ceemdan_residue_extrema() {
        if (!cs.active) raise(SEMD_INVALID_INPUT, "ceemdan: no active shard (call begin)");
        if (!A.trace) {  // untraced: one counting kernel instead of an engine run
            const long long n = cs.n;
            if (n < 3) raise(SEMD_INVALID_INPUT, "find_extrema: signal too short (need at least 3 samples)");
            scalar.alloc((2 + 2 * 256 + 8) * 8);
            unsigned long long* d = reinterpret_cast<unsigned long long*>(scalar.p) + (2 + 2 * 256);  // spare tail
            ck(cudaMemsetAsync(d, 0, 16, stream), "count");
            semd::dev::launch_count_extrema(cs_residue(), n, d, stream);
            unsigned long long h[2] = {0, 0};
            ck(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, stream), "count");
            ck(cudaStreamSynchronize(stream), "count");
            return (long long)(h[0] + h[1]);
        }
        JobSpec J;
        J.m = -1;
        J.task = 3;
        J.k = cs.K;
        J.a = cs_residue();
        J.detect_only = 1;
        std::vector<JobSpec> js{J};
        std::vector<Slot> res;
        cs_run_tasks(js, &res);
        return (long long)res[0].n[0] + (long long)res[0].n[1];
    }

    // the shard's unscaled first-mode sum of stage K into sums row K
    void ceemdan_stage() {
        if (!cs.active) raise(SEMD_INVALID_INPUT, "ceemdan: no active shard (call begin)");
        if (cs.K >= cs.kcap) {
            grow_sums(2 * cs.kcap);
            cs.kcap = A.kcap;
        }
        const int cnt = cs.m1 - cs.m0;
        const long long n = cs.n;
        if (cs.K == 0) {  // mode 1 (emd.cpp:292-307): first modes of x + beta0 w^(m)
            std::vector<JobSpec> js(cnt);
            for (int i = 0; i < cnt; ++i) {
                JobSpec& J = js[i];
                J.m = cs.m0 + i;
                J.task = 2;
                J.k = 0;
                J.kmax = 1;
                J.init_kind = 1;
                J.beta = cs.beta0;
                J.a = cs.x;
                J.b = cs_noise() + (size_t)i * cs.Ls;
            }
            std::vector<Slot> res;
            cs_run_tasks(js, &res);
            return;
        }
        // beta_i = nstd * std(r_i) (emd.cpp:312): the sequential std (one SM) runs on the side stream
        // while the noise residues' modes E_i are extracted; the first modes need it afterwards
        scalar.alloc((2 + 2 * 256 + 8) * 8);
        ck(cudaEventRecord(res_ready, stream), "residue event");
        ck(cudaStreamWaitEvent(rng_stream, res_ready, 0), "residue wait");
        semd::dev::launch_signal_std(cs_residue(), n, scalar.as<double>(), cs.ens.nstd, rng_stream, std_workspace(n));
        double* beta_host = reinterpret_cast<double*>(status_host + 8);  // pinned
        ck(cudaMemcpyAsync(beta_host, scalar.p, 8, cudaMemcpyDeviceToHost, rng_stream), "std");
        {  // E_i(w^(m)) for the living noise residues (emd.cpp:316-325)
            std::vector<JobSpec> js;
            std::vector<int> idx;
            for (int i = 0; i < cnt; ++i) {
                if (!cs.alive[i]) continue;
                JobSpec J;
                J.m = cs.m0 + i;
                J.task = 1;
                J.k = cs.K;
                J.kmax = cs.K + 1;
                J.write_imf = 0;
                J.a = cs_noise() + (size_t)i * cs.Ls;
                J.imf_out = cs_E() + (size_t)i * n;
                J.res_out = cs_noise() + (size_t)i * cs.Ls;
                js.push_back(J);
                idx.push_back(i);
            }
            std::vector<Slot> res;
            cs_run_tasks(js, &res);
            for (size_t q = 0; q < idx.size(); ++q) {
                if (res[q].ended_insufficient) {
                    cs.alive[idx[q]] = 0;
                    ck(cudaMemsetAsync(cs_E() + (size_t)idx[q] * n, 0, n * 8, stream), "E zero");
                }
            }
        }
        ck(cudaStreamSynchronize(rng_stream), "std");
        const double beta_i = *beta_host;
        {  // first modes of r_i + beta_i E_i (emd.cpp:326-329)
            std::vector<JobSpec> js(cnt);
            for (int i = 0; i < cnt; ++i) {
                JobSpec& J = js[i];
                J.m = cs.m0 + i;
                J.task = 2;
                J.k = cs.K;
                J.kmax = cs.K + 1;
                J.init_kind = 1;
                J.beta = beta_i;
                J.a = cs_residue();
                J.b = cs_E() + (size_t)i * n;
            }
            std::vector<Slot> res;
            cs_run_tasks(js, &res);
        }
    }

    // The whole CEEMDAN in one cooperative launch of the resident engine (single GPU): stages,
    // ordered stage means, residue checks and beta_K on the device, no host round trip. False
    // (nothing produced) when it cannot run or a stage outgrew it; the caller then runs the
    // per-stage drivers.
    DBuf ce_e1, ce_ok, ce_alive, ce_ctl, ce_E, ce_flags;
    bool ceemdan_fused(const double* d_x, long long n, const semd_sift_cfg& cfg, const semd_ens_cfg& ens,
                       semd_trace* tr) {
        using namespace semd::dev;
        ceemdan_begin(d_x, n, cfg, ens, 0, ens.nr, tr);
        const int nr = ens.nr;
        const long long Lp = (n + 3) & ~3LL;
        ce_e1.alloc((size_t)nr * Lp * 8);
        ce_ok.alloc((size_t)nr * 4);
        ce_alive.alloc((size_t)nr * 4);
        ce_E.alloc((size_t)nr * Lp * 8);
        ce_flags.alloc((size_t)nr * 8);
        ck(cudaMemsetAsync(ce_flags.p, 0, (size_t)nr * 8, stream), "flags");
        ce_ctl.alloc(sizeof(CeeCtl));
        semd::dev::launch_fill_i32(ce_alive.as<int>(), nr, 1, stream);
        ck(cudaMemsetAsync(ce_ctl.p, 0, sizeof(CeeCtl), stream), "ctl");
        const int grid = std::max(1, std::min(nr, sms));
        r_scratch.alloc((size_t)grid * 2 * Lp * 8);
        ensure_pin(A.G);
        ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
        ResArgs P{};
        P.L = (int)n;
        P.scratch = r_scratch.as<double>();
        P.max_iters = A.max_sift_iters;
        P.sd_thr = A.sd_threshold;
        P.tab_rows = res_tab_rows(n);
        P.trace = A.trace_cap > 0 ? A.trace : nullptr;
        P.trace_cap = A.trace_cap;
        P.trace_count = &A.ctrl->trace_count;
        P.sd_rechecks = &A.ctrl->sd_rechecks;
        P.debug = debug_flags;
        P.chain_div = res_chain_div();
        if (debug_flags & 2) {
            r_prof.alloc(128);
            if (!r_prof_init) {
                ck(cudaMemsetAsync(r_prof.p, 0, 128, stream), "prof");
                r_prof_init = true;
            }
            P.prof = r_prof.as<unsigned long long>();
        }
        CeeArgs Q{};
        Q.x = d_x;
        Q.residue = cs_residue();
        Q.nres = cs_noise();
        Q.Ls = cs.Ls;
        Q.e1 = ce_e1.as<double>();
        Q.e1_ok = ce_ok.as<int>();
        Q.alive = ce_alive.as<int>();
        Q.E = ce_E.as<double>();
        Q.e_have = ce_flags.as<int>();
        Q.edone = ce_flags.as<int>() + nr;
        Q.modes = A.sums;
        Q.kcap = A.kcap;
        Q.nr = nr;
        Q.m0 = 0;
        Q.max_imfs = cfg.max_imfs;
        Q.nstd = ens.nstd;
        Q.beta0 = cs.beta0;
        Q.inv_nr = 1.0 / (double)nr;
        Q.ctl = ce_ctl.as<CeeCtl>();
        if (timing) res_timer_start();
        const cudaError_t e = (cudaError_t)launch_res_ceemdan(P, Q, grid, stream);
        if (timing && e == cudaSuccess) ck(cudaEventRecord(r_t1, stream), "ev");
        if (e != cudaSuccess) {  // e.g. the grid cannot be co-resident: per-stage drivers instead
            cudaGetLastError();
            cs.active = false;
            return false;
        }
        CeeCtl h{};
        Ctrl c;
        ck(cudaMemcpyAsync(&h, ce_ctl.p, sizeof(CeeCtl), cudaMemcpyDeviceToHost, stream), "ceemdan ctl");
        ck(cudaMemcpyAsync(pin_jobs, A.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream), "ctrl");
        ck(cudaStreamSynchronize(stream), "ceemdan (resident)");
        std::memcpy(&c, pin_jobs, sizeof(Ctrl));
        ck(cudaMemcpyAsync(A.ctrl, pin_reset_ctrl(), sizeof(Ctrl), cudaMemcpyHostToDevice, stream), "ctrl reset");
        if (h.status) {  // outgrew the shared memory or the mode rows: rerun per stage (new noise)
            ck(cudaStreamSynchronize(stream), "ctrl reset");
            cs.active = false;
            h_trace.clear();
            trace_total = 0;
            return false;
        }
        if (timing) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r_t0, r_t1);
            stats.eval_ms += ms;
        }
        stats.sifted_samples += h.sifted;
        stats.sift_iterations += h.sifted / (uint64_t)std::max(1LL, n);
        stats.solve_hazards += (uint64_t)h.hazards;
        stats.sd_rechecks += (uint64_t)c.sd_rechecks;
        stats.resident_jobs += (uint64_t)nr * (uint64_t)(h.K + 1);
        if (A.trace) {
            const int cnt = std::min(c.trace_count, A.trace_cap);
            const size_t old = h_trace.size();
            h_trace.resize(old + cnt);
            if (cnt)
                ck(cudaMemcpy(h_trace.data() + old, A.trace, (size_t)cnt * sizeof(TraceRec), cudaMemcpyDeviceToHost),
                   "trace");
            trace_total += c.trace_count;
        }
        cs.K = h.K;
        cs.waves += 1;
        return true;
    }

    // mode_K = total / nr; false (and no update) when check_zero and the mode is all zero.
    bool ceemdan_finish(const double* d_total, int nr, bool check_zero, double* d_mode_out) {
        if (!cs.active) raise(SEMD_INVALID_INPUT, "ceemdan: no active shard (call begin)");
        if (nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
        const long long n = cs.n;
        double* mode = A.sums + (size_t)cs.K * n;
        if (d_total && d_total != mode)
            ck(cudaMemcpyAsync(mode, d_total, n * 8, cudaMemcpyDeviceToDevice, stream), "stage total");
        ck(cudaMemsetAsync(cs_flag(), 0, 4, stream), "flag");
        semd::dev::launch_stage_scale(mode, n, 1.0 / (double)nr, cs_flag(), stream);
        int nz = 0;
        ck(cudaMemcpyAsync(&nz, cs_flag(), 4, cudaMemcpyDeviceToHost, stream), "flag");
        ck(cudaStreamSynchronize(stream), "stage");
        if (check_zero && !nz) return false;  // emd.cpp:332-337
        semd::dev::launch_sub(cs_residue(), mode, n, stream);
        if (d_mode_out) ck(cudaMemcpyAsync(d_mode_out, mode, n * 8, cudaMemcpyDeviceToDevice, stream), "mode");
        ++cs.K;
        return true;
    }

    // emd.cpp:264-344. Returns K; IMFs in `out_imfs` (device, k_cap rows), residue in out_res.
    // With a communicator the realizations are sharded over the ranks and every stage's first-mode
    // sum is all-reduced (NCCL, in place on the engine stream) before the identical finish on each
    // rank (emd.cpp:301-306, :331-339): residues, beta_i and the stop decisions agree everywhere.
    int ceemdan_device(const double* d_x, long long n, const semd_sift_cfg& cfg, const semd_ens_cfg& ens,
                       double* out_imfs, int k_cap, double* out_res, semd_trace* tr, int* k_needed) {
        int mb = 0, me = ens.nr;
        if (comm) shard_range(ens.nr, rank, world, &mb, &me);
        // the fused device loop has no stage exchange: single GPU (or a 1-rank communicator) only
        if ((comm && world > 1) || !resident_for(n) || !ceemdan_fused(d_x, n, cfg, ens, tr)) {
            ceemdan_begin(d_x, n, cfg, ens, mb, me, tr);
            auto stage_total = [&] {
                ceemdan_stage();
                comm_sum(A.sums + (size_t)cs.K * n, (size_t)n, false);
            };
            stage_total();
            ceemdan_finish(nullptr, ens.nr, false, nullptr);
            while (cfg.max_imfs == 0 || cs.K < cfg.max_imfs) {  // emd.cpp:310
                if (ceemdan_residue_extrema() < 3) break;        // emd.cpp:311
                stage_total();                                   // grows the IMF rows when needed
                if (!ceemdan_finish(nullptr, ens.nr, true, nullptr)) break;
            }
        }
        const int K = cs.K;
        stats.waves += cs.waves;
        stats.slots = cs.G;
        *k_needed = K;
        cs.active = false;
        if (K > k_cap) return K;
        if (out_imfs && K)
            ck(cudaMemcpyAsync(out_imfs, A.sums, (size_t)K * n * 8, cudaMemcpyDeviceToDevice, stream), "imfs");
        if (out_res) ck(cudaMemcpyAsync(out_res, cs_residue(), n * 8, cudaMemcpyDeviceToDevice, stream), "residue");
        ck(cudaStreamSynchronize(stream), "ceemdan");
        return K;
    }

    // ---- slicewise_decompose (baseline.cpp:5-29) on N same-length channels ----------------
    // EMD / EEMD: every channel (EEMD: channel x realization, channel-major) is a job of ONE
    // batched engine run; job j owns IMF rows [j*kc, (j+1)*kc). CEEMDAN: channel by channel.
    DBuf sl_imfs, sl_res, sl_kj, sl_beta;
    std::vector<int> sl_kj_host;  // IMF count of every channel of the last slicewise run
    void slicewise_device(int algo, const double* d_x, long long M, int N, const semd_sift_cfg& cfg,
                          const semd_ens_cfg& ens, double* d_tensor, size_t cap_modes, size_t* modes_out) {
        if (M == 0 || N == 0) raise(SEMD_INVALID_INPUT, "slicewise_decompose: empty input");
        if (algo != SEMD_ALGO_EMD) {  // emd.cpp:223-226, :229-230, :266-267
            if (ens.nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
            if (ens.nstd < 0.0) raise(SEMD_INVALID_INPUT, "ensemble: nstd must be non-negative");
            if (ens.nstd == 0.0) algo = SEMD_ALGO_EMD;
        }
        if (M < 4)
            raise(SEMD_INVALID_INPUT, algo == SEMD_ALGO_CEEMDAN ? "ceemdan: signal too short (need at least 4 samples)"
                                                               : "emd: signal too short (need at least 4 samples)");
        std::vector<int> kj(N, 0);
        int kc = default_kcap(M, cfg.max_imfs);
        sl_res.alloc((size_t)N * M * 8);
        double* res = sl_res.as<double>();
        const double* imf_rows = nullptr;  // [N][kc][M]
        bool scaled = false;
        if (algo == SEMD_ALGO_CEEMDAN) {
            sl_imfs.alloc((size_t)N * kc * M * 8);
            for (int j = 0; j < N; ++j) {
                int need = 0;
                const int K = ceemdan_device(d_x + (size_t)j * M, M, cfg, ens, sl_imfs.as<double>() + (size_t)j * kc * M,
                                             kc, res + (size_t)j * M, nullptr, &need);
                if (K > kc) raise(SEMD_CAPACITY, "IMF capacity exceeded (%d rows)", kc);
                kj[j] = K;
            }
            imf_rows = sl_imfs.as<double>();
        } else {
            const bool ens_mode = algo == SEMD_ALGO_EEMD;
            const int nr = ens_mode ? ens.nr : 1;
            const long long Ls = (M + 1) / 2 * 2;
            std::vector<double> beta(N, 0.0);
            if (ens_mode) {  // beta_j = nstd * std(x_j) (emd.cpp:233), exact sequential sums per channel
                sl_beta.alloc((size_t)N * 8);
                semd::dev::launch_signal_std_batch(d_x, M, N, sl_beta.as<double>(), ens.nstd, stream);
                ck(cudaMemcpyAsync(beta.data(), sl_beta.p, (size_t)N * 8, cudaMemcpyDeviceToHost, stream), "betas");
                noise.alloc((size_t)nr * Ls * 8);  // w_m, shared by every channel (emd.cpp:238)
                for (int m0 = 0; m0 < nr; m0 += 1024) {
                    const int g = std::min(1024, nr - m0);
                    std::vector<uint64_t> seeds(g);
                    for (int i = 0; i < g; ++i) seeds[i] = derive_seed(ens.base_seed, (uint64_t)(m0 + i));
                    gen_noise(seeds, M, Ls, noise.as<double>() + (size_t)m0 * Ls);
                }
            }
            const long long jobs = (long long)N * nr;
            bool res_engine = resident_for(M);
            for (int attempt = 0;; ++attempt) {
                if (res_engine) {  // every (channel, realization) job on the resident engine, in job order
                    configure(M, 1, N * kc, 0);
                    A.kper = kc;
                    A.sd_threshold = cfg.sd_threshold;
                    A.max_sift_iters = cfg.max_sift_iters;
                    fill_sums(N * kc, ens_mode ? 0.0 : -0.0);
                    if (!ens_mode)
                        ck(cudaMemcpyAsync(res, d_x, (size_t)N * M * 8, cudaMemcpyDeviceToDevice, stream), "res");
                    std::fill(kj.begin(), kj.end(), 0);
                    // batches bounded by the IMF store (jobs x kc x M doubles), kept in job order
                    const long long per = std::max<long long>(1, (1LL << 31) / ((long long)kc * ((M + 3) & ~3LL) * 8));
                    bool ok = true;
                    try {
                        for (long long w0 = 0; w0 < jobs && ok; w0 += per) {
                            const int g = (int)std::min<long long>(per, jobs - w0);
                            std::vector<JobSpec> js(g);
                            for (int i = 0; i < g; ++i) {
                                const long long q = w0 + i;
                                const int j = (int)(q / nr), m = (int)(q % nr);
                                JobSpec& J = js[i];
                                J.m = ens_mode ? m : j;
                                J.task = 0;
                                J.kmax = cfg.max_imfs;
                                J.k0 = j * kc;
                                J.a = d_x + (size_t)j * M;
                                if (ens_mode) {
                                    J.init_kind = 1;
                                    J.beta = beta[j];
                                    J.b = noise.as<double>() + (size_t)m * Ls;
                                } else {
                                    J.res_out = res + (size_t)j * M;
                                }
                            }
                            std::vector<int> failed;
                            ok = run_resident(js, kc, &failed);
                            if (ok && !failed.empty()) ok = false;  // (EMD residues: rerun all on the lockstep engine)
                            if (ok)
                                for (int i = 0; i < g; ++i) {
                                    const int j = (int)((w0 + i) / nr);
                                    kj[j] = std::max(kj[j], r_out[i].k);
                                }
                        }
                    } catch (const Error& e) {
                        A.kper = 0;
                        if (e.code == SEMD_CAPACITY && attempt < 3 && cfg.max_imfs == 0) {
                            kc *= 2;
                            continue;
                        }
                        throw;
                    }
                    A.kper = 0;
                    if (ok) break;
                    res_engine = false;  // tables outgrew the shared memory: the lockstep engine below
                    --attempt;
                    continue;
                }
                const int G = auto_slots(M, (int)std::min<long long>(jobs, 1 << 20));
                if ((long long)N * kc * M * 8 > (1LL << 40)) raise(SEMD_NO_MEMORY, "slicewise IMF store too large");
                configure(M, G, N * kc, 0);
                A.kper = kc;
                A.sd_threshold = cfg.sd_threshold;
                A.max_sift_iters = cfg.max_sift_iters;
                fill_sums(N * kc, ens_mode ? 0.0 : -0.0);
                if (!ens_mode)  // channels without IMFs keep x as residue; k_final overwrites the rest
                    ck(cudaMemcpyAsync(res, d_x, (size_t)N * M * 8, cudaMemcpyDeviceToDevice, stream), "res");
                std::fill(kj.begin(), kj.end(), 0);
                try {
                    for (long long w0 = 0; w0 < jobs; w0 += G) {
                        const int g = (int)std::min<long long>(G, jobs - w0);
                        std::vector<JobSpec> js(g);
                        for (int i = 0; i < g; ++i) {
                            const long long q = w0 + i;
                            const int j = (int)(q / nr), m = (int)(q % nr);
                            JobSpec& J = js[i];
                            J.m = ens_mode ? m : j;
                            J.task = 0;
                            J.kmax = cfg.max_imfs;
                            J.k0 = j * kc;
                            J.a = d_x + (size_t)j * M;
                            if (ens_mode) {
                                J.init_kind = 1;
                                J.beta = beta[j];
                                J.b = noise.as<double>() + (size_t)m * Ls;
                            } else {
                                J.res_out = res + (size_t)j * M;
                            }
                        }
                        set_jobs(js);
                        run(max_steps_for(cfg));
                        for (int i = 0; i < g; ++i) {
                            const int j = (int)((w0 + i) / nr);
                            kj[j] = std::max(kj[j], h_slots[i].k);
                        }
                    }
                } catch (const Error& e) {
                    A.kper = 0;
                    if (e.code == SEMD_CAPACITY && attempt < 3 && cfg.max_imfs == 0) {
                        kc *= 2;
                        continue;
                    }
                    throw;
                }
                A.kper = 0;
                break;
            }
            if (ens_mode) semd::dev::launch_slicewise_finish(d_x, A.sums, kc, M, N, 1.0 / (double)nr, res, stream);
            imf_rows = A.sums;
            scaled = ens_mode;
        }
        int common = 1;
        for (int j = 0; j < N; ++j) common = std::max(common, kj[j] + 1);
        sl_kj_host = kj;
        *modes_out = (size_t)common;
        if ((size_t)common > cap_modes) raise(SEMD_CAPACITY, "output holds %zu modes, decomposition has %d", cap_modes, common);
        sl_kj.alloc((size_t)N * 4);
        ck(cudaMemcpyAsync(sl_kj.p, kj.data(), (size_t)N * 4, cudaMemcpyHostToDevice, stream), "kj");
        semd::dev::launch_slicewise_tensor(imf_rows, kc, sl_kj.as<int>(), res, M, N, common,
                                           scaled ? 1.0 / (double)ens.nr : 1.0, scaled ? 1 : 0, d_tensor, stream);
        ck(cudaGetLastError(), "slicewise");
        ck(cudaStreamSynchronize(stream), "slicewise");
    }

    // B independent serial_decompose calls (serialize.cpp:97-105) on same-shape multi-signals, as
    // one batched engine pass: every multi-signal is serialized (x_b -> s_b of length L), the B
    // signals are decomposed like slicewise channels (EMD: one job each; EEMD: B x nr jobs sharing
    // the realizations' noise w_m, beta_b from s_b; CEEMDAN: one after another), and each result is
    // deconcatenated into its own ImfTensor: K_b IMFs then the residue, zero modes after.
    DBuf sb_ser, sb_tens;
    void serial_batch_device(int algo, const double* d_x, long long B, long long M, long long N, long long D,
                             const semd_sift_cfg& cfg, const semd_ens_cfg& ens, double* d_out, size_t k_cap,
                             size_t* modes_out) {
        if (B < 1) raise(SEMD_INVALID_INPUT, "serial_decompose_batch: empty batch");
        if (M == 0 || N == 0) raise(SEMD_INVALID_INPUT, "concatenate: empty input");
        if (D < 1) raise(SEMD_INVALID_INPUT, "concatenate: D must be at least 1");
        if (D > M) raise(SEMD_INVALID_INPUT, "concatenate: transition longer than channel");
        const long long L = M * N + D * (N - 1);
        sb_ser.alloc((size_t)B * L * 8);
        scratch2.alloc((size_t)D * 8);
        semd::dev::launch_transition_weights(D, scratch2.as<double>(), stream);
        for (long long b = 0; b < B; ++b)
            semd::dev::launch_concatenate(d_x + (size_t)b * M * N, M, N, D, scratch2.as<double>(),
                                          sb_ser.as<double>() + (size_t)b * L, 0, stream);
        ck(cudaGetLastError(), "concatenate");
        size_t cap = std::max<size_t>(k_cap, 2), common = 0;
        for (;;) {  // the slicewise tensor holds the common mode count; grow to fit it
            sb_tens.alloc(cap * (size_t)B * L * 8);
            try {
                slicewise_device(algo, sb_ser.as<double>(), L, (int)B, cfg, ens, sb_tens.as<double>(), cap, &common);
                break;
            } catch (const Error& e) {
                if (e.code != SEMD_CAPACITY || common <= cap) throw;
                cap = common;
            }
        }
        bool fits = true;
        for (long long b = 0; b < B; ++b) {
            modes_out[b] = (size_t)sl_kj_host[b] + 1;
            fits = fits && modes_out[b] <= k_cap;
        }
        if (!fits) raise(SEMD_CAPACITY, "output holds %zu modes per item, a decomposition has more", k_cap);
        // slicewise layout (k*B + b)*L + i, residue at k = common-1 -> per item K_b IMFs + residue
        DBuf modes((size_t)(common + 1) * L * 8);
        for (long long b = 0; b < B; ++b) {
            const int Kb = sl_kj_host[b];
            double* mrow = modes.as<double>();
            const double* t = sb_tens.as<double>();
            if (Kb)
                ck(cudaMemcpy2DAsync(mrow, (size_t)L * 8, t + (size_t)b * L, (size_t)B * L * 8, (size_t)L * 8, (size_t)Kb,
                                     cudaMemcpyDeviceToDevice, stream),
                   "modes");
            ck(cudaMemcpyAsync(mrow + (size_t)Kb * L, t + ((size_t)(common - 1) * B + b) * L, (size_t)L * 8,
                               cudaMemcpyDeviceToDevice, stream),
               "residue");
            double* dst = d_out + (size_t)b * k_cap * N * M;
            if ((size_t)Kb + 1 < k_cap)
                ck(cudaMemsetAsync(dst + (size_t)(Kb + 1) * N * M, 0, (k_cap - Kb - 1) * (size_t)N * M * 8, stream),
                   "zero modes");
            semd::dev::launch_deconcatenate(mrow, Kb + 1, L, M, N, D, dst, stream);
        }
        ck(cudaGetLastError(), "deconcatenate");
        ck(cudaStreamSynchronize(stream), "serial batch");
    }

    // Full decomposition with device buffers. Returns K via *k_out; SEMD_CAPACITY if K > k_cap.
    void decompose_device(int algo, const double* d_x, long long n, const semd_sift_cfg& cfg, const semd_ens_cfg& ens,
                          double* d_imfs, size_t k_cap, size_t* k_out, double* d_res, int32_t* sift_counts_host,
                          semd_trace* tr) {
        if (algo < 0 || algo > 2) raise(SEMD_INVALID_INPUT, "unknown algorithm value");
        if (algo != SEMD_ALGO_EMD) {
            if (ens.nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
            if (ens.nstd < 0.0) raise(SEMD_INVALID_INPUT, "ensemble: nstd must be non-negative");
            if (ens.nstd == 0.0) algo = SEMD_ALGO_EMD;  // degenerate ensemble is plain emd
        }
        reset_stats(1);
        if (algo != SEMD_ALGO_CEEMDAN && cfg.max_sift_iters <= 0 && cfg.max_imfs == 0)
            raise(SEMD_INVALID_INPUT,
                  "emd: max_sift_iters <= 0 with max_imfs == 0 never terminates (every IMF is the whole residue)");
        if (algo == SEMD_ALGO_EMD) {
            const int K = emd_device(d_x, n, cfg, tr);
            *k_out = (size_t)K;
            stats.slots = 1;
            stats.waves = 1;
            export_trace(tr);
            if ((size_t)K > k_cap) raise(SEMD_CAPACITY, "output holds %zu IMFs, decomposition has %d", k_cap, K);
            if (K && d_imfs)
                ck(cudaMemcpyAsync(d_imfs, A.sums, (size_t)K * n * 8, cudaMemcpyDeviceToDevice, stream), "imfs");
            if (d_res)
                ck(cudaMemcpyAsync(d_res, buf(0, h_slots[0].xb), n * 8, cudaMemcpyDeviceToDevice, stream), "residue");
            if (sift_counts_host && K) {
                std::vector<int> c(K);
                ck(cudaMemcpy(c.data(), A.imf_sifts, (size_t)K * 4, cudaMemcpyDeviceToHost), "counts");
                for (int k = 0; k < K; ++k) sift_counts_host[k] = c[k];
            }
            ck(cudaStreamSynchronize(stream), "emd");
            return;
        }
        if (algo == SEMD_ALGO_EEMD) {
            if (n < 4) raise(SEMD_INVALID_INPUT, "emd: signal too short (need at least 4 samples)");
            // realization shard of this rank (all of [0, nr) without a communicator)
            int mb = 0, me = ens.nr;
            if (comm) shard_range(ens.nr, rank, world, &mb, &me);
            int K = 0;
            if (me > mb) {
                K = eemd_partial_device(d_x, n, cfg, ens, mb, me, tr);
            } else {  // more ranks than realizations: this rank contributes zeros
                configure(n, 1, default_kcap(n, cfg.max_imfs), tr ? trace_cap_for(tr) : 0);
                fill_sums(A.kcap, 0.0);
                h_trace.clear();
                trace_total = 0;
            }
            double* sums_d = A.sums;
            if (comm) {  // emd.cpp:246-251 across ranks: K = max K_m, then the ensemble sum
                const int k_local = K;
                K = (int)comm_max(K);
                if (K > A.kcap) {  // another rank needed more IMF rows than this one holds
                    comm_red.alloc((size_t)K * n * 8);
                    ck(cudaMemsetAsync(comm_red.p, 0, (size_t)K * n * 8, stream), "reduce rows");
                    if (k_local)
                        ck(cudaMemcpyAsync(comm_red.p, A.sums, (size_t)k_local * n * 8, cudaMemcpyDeviceToDevice,
                                           stream),
                           "reduce rows");
                    sums_d = comm_red.as<double>();
                }
                comm_sum(sums_d, (size_t)K * n, true);
            }
            *k_out = (size_t)K;
            export_trace(tr);
            if (!has_result()) {  // root-only reduction: the ensemble lives on the root rank
                ck(cudaStreamSynchronize(stream), "eemd");
                return;
            }
            if ((size_t)K > k_cap) raise(SEMD_CAPACITY, "output holds %zu IMFs, decomposition has %d", k_cap, K);
            semd::dev::launch_ensemble_finish(sums_d, K, n, d_x, d_res ? d_res : buf(0, 1), 1.0 / (double)ens.nr,
                                              stream);
            if (K && d_imfs)
                ck(cudaMemcpyAsync(d_imfs, sums_d, (size_t)K * n * 8, cudaMemcpyDeviceToDevice, stream), "imfs");
            if (sift_counts_host)
                for (int k = 0; k < K; ++k) sift_counts_host[k] = 0;
            ck(cudaStreamSynchronize(stream), "eemd");
            return;
        }
        int need = 0;
        ceemdan_device(d_x, n, cfg, ens, d_imfs, (int)k_cap, d_res, tr, &need);
        *k_out = (size_t)need;
        export_trace(tr);
        if ((size_t)need > k_cap) raise(SEMD_CAPACITY, "output holds %zu IMFs, decomposition has %d", k_cap, need);
        if (sift_counts_host)
            for (int k = 0; k < need; ++k) sift_counts_host[k] = 0;
    }

    double* upload(DBuf& d, const double* h, size_t n) {
        d.alloc(n * 8);
        if (n) ck(cudaMemcpyAsync(d.p, h, n * 8, cudaMemcpyHostToDevice, stream), "upload");
        return d.as<double>();
    }
    void download(double* h, const double* d, size_t n) {
        if (n) ck(cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost, stream), "download");
        ck(cudaStreamSynchronize(stream), "download");
    }
};

namespace {

semd_sift_cfg sift_or_default(const semd_sift_cfg* c) {
    if (c) return *c;
    return semd_sift_cfg{0.2, 300, 0};
}
semd_ens_cfg ens_or_default(const semd_ens_cfg* e) {
    if (e) return *e;
    return semd_ens_cfg{0.2, 100, 0, 0};
}

void need_ctx(semd_ctx* ctx) {
    if (!ctx) raise(SEMD_INVALID_INPUT, "null semd_ctx");
    ctx->use();
}

void validate_serial(size_t M, size_t N, size_t D) {  // serialize.cpp:22-26
    if (M == 0 || N == 0) raise(SEMD_INVALID_INPUT, "concatenate: empty input");
    if (D < 1) raise(SEMD_INVALID_INPUT, "concatenate: D must be at least 1");
    if (D > M) raise(SEMD_INVALID_INPUT, "concatenate: transition longer than channel");
}

void concat_device(semd_ctx* c, const double* d_x, size_t M, size_t N, size_t D, double* d_out, int naive) {
    validate_serial(M, N, D);
    c->scratch2.alloc(std::max<size_t>(D, 1) * 8);
    semd::dev::launch_transition_weights((long long)D, c->scratch2.as<double>(), c->stream);
    semd::dev::launch_concatenate(d_x, (long long)M, (long long)N, (long long)D, c->scratch2.as<double>(), d_out, naive,
                                  c->stream);
    ck(cudaGetLastError(), "concatenate");
}

void validate_deconcat(size_t K, size_t L, size_t M, size_t N, size_t D) {  // serialize.cpp:75-81
    if (K == 0) raise(SEMD_INVALID_INPUT, "deconcatenate: no modes given");
    if (M == 0 || N == 0) raise(SEMD_INVALID_INPUT, "deconcatenate: empty target shape");
    const size_t expect = M * N + D * (N - 1);
    if (L != expect)
        raise(SEMD_INVALID_INPUT, "deconcatenate: mode length %zu does not match M*N + D*(N-1) = %zu", L, expect);
}

}  // namespace

extern "C" {

const char* semd_last_error(void) { return g_err.c_str(); }

int semd_ctx_create(int device, semd_ctx** out) {
    return guard([&] {
        if (!out) raise(SEMD_INVALID_INPUT, "null output pointer");
        *out = nullptr;
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            raise(SEMD_CUDA_ERROR, "no CUDA device available (%s); the B200 sift engine has no CPU fallback",
                  cudaGetErrorString(e));
        }
        if (device < 0 || device >= ndev) raise(SEMD_INVALID_INPUT, "device %d out of range (%d devices)", device, ndev);
        auto* c = new semd_ctx();
        try {
            c->device = device;
            c->use();
            cudaDeviceProp prop{};
            ck(cudaGetDeviceProperties(&prop, device), "device properties");
            if (prop.major < 10) raise(SEMD_CUDA_ERROR, "device %s (sm_%d%d) is not sm_100", prop.name, prop.major, prop.minor);
            c->sms = prop.multiProcessorCount;
            ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "stream");
            ck(cudaStreamCreateWithFlags(&c->rng_stream, cudaStreamNonBlocking), "stream");
            for (auto& e : c->noise_ready) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&c->res_ready, cudaEventDisableTiming), "event");
            c->stream = c->own;
            for (auto& ev : c->ev) ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
            ck(cudaEventCreate(&c->t0), "event");
            ck(cudaEventCreate(&c->t1), "event");
            ck(cudaHostAlloc(&c->status_host, 64, cudaHostAllocMapped), "pinned status");
            ck(cudaHostGetDevicePointer(&c->status_host_dev, c->status_host, 0), "mapped status");
            ck(semd::dev::launch_setup(), "kernel attributes");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void semd_ctx_destroy(semd_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
}

int semd_get_stats(semd_ctx* ctx, semd_stats* out) {
    return guard([&] {
        if (!ctx || !out) raise(SEMD_INVALID_INPUT, "null argument");
        ctx->stats.kernel_launches = semd::dev::launch_count() - ctx->launches_at_reset;
        *out = ctx->stats;
    });
}

int semd_set_stream(semd_ctx* ctx, void* s) {
    return guard([&] {
        need_ctx(ctx);
        ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    });
}

int semd_set_timing(semd_ctx* ctx, int enable) {
    return guard([&] {
        need_ctx(ctx);
        ctx->timing = enable != 0;
    });
}

int semd_set_max_slots(semd_ctx* ctx, int slots) {
    return guard([&] {
        need_ctx(ctx);
        ctx->max_slots = std::max(0, slots);
    });
}

int semd_set_engine(semd_ctx* ctx, int engine) {
    return guard([&] {
        need_ctx(ctx);
        if (engine < SEMD_ENGINE_AUTO || engine > SEMD_ENGINE_RESIDENT) raise(SEMD_INVALID_INPUT, "unknown engine %d", engine);
        ctx->engine = engine;
    });
}

// Test hook: nr x n host noise used instead of the device RNG (NULL clears).
int semd_set_noise_override(semd_ctx* ctx, const double* noise, size_t nr, size_t n) {
    return guard([&] {
        need_ctx(ctx);
        if (!noise) {
            ctx->noise_override = nullptr;
            return;
        }
        ctx->in_y.alloc(nr * n * 8);
        ck(cudaMemcpy(ctx->in_y.p, noise, nr * n * 8, cudaMemcpyHostToDevice), "noise override");
        ctx->noise_override = ctx->in_y.as<double>();
    });
}

// ---- CEEMDAN stages over a realization shard (multi-GPU drivers) ----------------------
int semd_ceemdan_shard_begin(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg_,
                             const semd_ens_cfg* ens_, int32_t m_begin, int32_t m_end) {
    return guard([&] {
        need_ctx(ctx);
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        const semd_ens_cfg ens = ens_or_default(ens_);
        if (ens.nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
        if (ens.nstd < 0.0) raise(SEMD_INVALID_INPUT, "ensemble: nstd must be non-negative");
        ctx->reset_stats(1);
        ctx->ceemdan_begin(d_x, (long long)n, cfg, ens, m_begin, m_end, nullptr);
    });
}
int semd_ceemdan_shard_residue_extrema(semd_ctx* ctx, size_t* total) {
    return guard([&] {
        need_ctx(ctx);
        const long long t = ctx->ceemdan_residue_extrema();
        if (total) *total = (size_t)t;
    });
}
int semd_ceemdan_shard_stage(semd_ctx* ctx, double* d_partial) {
    return guard([&] {
        need_ctx(ctx);
        ctx->ceemdan_stage();
        if (d_partial)
            ck(cudaMemcpyAsync(d_partial, ctx->A.sums + (size_t)ctx->cs.K * ctx->cs.n, ctx->cs.n * 8,
                               cudaMemcpyDeviceToDevice, ctx->stream),
               "partial");
        ck(cudaStreamSynchronize(ctx->stream), "stage");
    });
}
int semd_ceemdan_shard_finish_stage(semd_ctx* ctx, const double* d_total, int32_t nr, int32_t check_zero,
                                    double* d_mode_out, int32_t* accepted) {
    return guard([&] {
        need_ctx(ctx);
        const bool ok = ctx->ceemdan_finish(d_total, nr, check_zero != 0, d_mode_out);
        if (accepted) *accepted = ok ? 1 : 0;
        ck(cudaStreamSynchronize(ctx->stream), "finish");
    });
}
int semd_ceemdan_shard_residue(semd_ctx* ctx, double* d_res_out) {
    return guard([&] {
        need_ctx(ctx);
        if (!ctx->cs.active) raise(SEMD_INVALID_INPUT, "ceemdan: no active shard (call begin)");
        ck(cudaMemcpyAsync(d_res_out, ctx->cs_residue(), ctx->cs.n * 8, cudaMemcpyDeviceToDevice, ctx->stream),
           "residue");
        ck(cudaStreamSynchronize(ctx->stream), "residue");
    });
}

// Test hook: debug flags (bit 0: force the exact sequential solve repair on every multi-block envelope).
int semd_set_debug(semd_ctx* ctx, int flags) {
    return guard([&] {
        need_ctx(ctx);
        ctx->debug_flags = flags;
        ctx->A.debug = flags;
    });
}

// Dev hook: the resident engine's per-phase SM cycles (debug bit 1), 8 u64; reset after reading.
int semd_resident_profile(semd_ctx* ctx, uint64_t* out) {
    return guard([&] {
        need_ctx(ctx);
        for (int i = 0; i < 16; ++i) out[i] = 0;
        if (!ctx->r_prof_init) return;
        ck(cudaMemcpy(out, ctx->r_prof.p, 128, cudaMemcpyDeviceToHost), "prof");
        ck(cudaMemset(ctx->r_prof.p, 0, 128), "prof");
    });
}

// Test hook: k_solve per-phase cycle counters (debug bit 1), 16 u64; reset after reading.
int semd_solve_profile(semd_ctx* ctx, uint64_t* out) {
    return guard([&] {
        need_ctx(ctx);
        if (!ctx->prof.p) raise(SEMD_INVALID_INPUT, "no engine configured");
        ck(cudaMemcpy(out, ctx->prof.p, 16 * 8, cudaMemcpyDeviceToHost), "prof");
        ck(cudaMemset(ctx->prof.p, 0, 16 * 8), "prof");
    });
}

// Profiling hook: device spans (ms) of k_solve, k_eval, k_scan, k_compact, k_final summed over
// the steps since the last call, and the eval strips processed in DETECT/INIT and SIFT mode
// and their summed warp cycles (strips[4]).
int semd_kernel_spans(semd_ctx* ctx, double* ms, uint64_t* strips) {
    return guard([&] {
        need_ctx(ctx);
        for (int i = 0; i < 5; ++i) {
            ms[i] = ctx->span_ms[i];
            ctx->span_ms[i] = 0.0;
        }
        for (int i = 0; i < 4; ++i) {
            strips[i] = ctx->span_strips[i];
            ctx->span_strips[i] = 0;
        }
    });
}

// Profiling hook: speculative last sifts since the last call -- run, stopped (the next IMF skipped
// its DETECT pass and k_final its residue update), continued (an extra detection step) -- and the
// lockstep steps (out[4]). Debug bit 8 (semd_set_debug) turns speculation off, bit 16 makes every
// sift speculative.
int semd_spec_stats(semd_ctx* ctx, uint64_t* out) {
    return guard([&] {
        need_ctx(ctx);
        for (int i = 0; i < 4; ++i) {
            out[i] = ctx->spec_stats[i];
            ctx->spec_stats[i] = 0;
        }
    });
}

// Test hook: segments of the last parallel signal_std that were added term by term (the slow,
// reference-literal path), per pass: out[0] mean pass, out[1] variance pass, out[2] segments per pass
// (0: the last call used the single-thread kernel). Debug bit 32 forces the single-thread kernel.
int semd_std_stats(semd_ctx* ctx, uint64_t* out) {
    return guard([&] {
        need_ctx(ctx);
        out[0] = out[1] = out[2] = 0;
        if (!ctx->std_ws.p || !ctx->std_last_n) return;
        unsigned h[6];
        ck(cudaMemcpy(h, ctx->std_ws.p, sizeof(h), cudaMemcpyDeviceToHost), "std stats");
        out[0] = h[2];
        out[1] = h[3];
        out[2] = (uint64_t)((ctx->std_last_n + 511) / 512);
    });
}

// Test hook: solve-hazard records of the last call, 8 int32 each
// {m, k, iter, side, knots, block, blocks, 1 forward / 2 back-substitution}.
int semd_hazard_log(semd_ctx* ctx, int32_t* out, size_t cap, size_t* count) {
    return guard([&] {
        need_ctx(ctx);
        const size_t n = ctx->h_hz.size() / 8;
        if (count) *count = n;
        if (out) std::memcpy(out, ctx->h_hz.data(), std::min(n, cap) * 8 * 4);
    });
}

// Test hook: the raw std::mt19937_64 stream generated on the device.
int semd_mt19937_64_device_test(semd_ctx* ctx, uint64_t seed, size_t n, uint64_t* out) {
    return guard([&] {
        need_ctx(ctx);
        const size_t n2 = (n + 1) / 2 * 2;
        DBuf d(std::max<size_t>(n2, 2) * 8);
        semd::dev::RngJob job{seed, d.as<uint64_t>(), (long long)n2};
        DBuf dj(sizeof(job));
        ck(cudaMemcpy(dj.p, &job, sizeof(job), cudaMemcpyHostToDevice), "job");
        semd::dev::launch_rng(dj.as<semd::dev::RngJob>(), 1, ctx->stream);
        ck(cudaGetLastError(), "rng");
        ck(cudaStreamSynchronize(ctx->stream), "rng");
        if (n) ck(cudaMemcpy(out, d.p, n * 8, cudaMemcpyDeviceToHost), "draws");
    });
}

uint64_t semd_derive_seed(uint64_t base, uint64_t index) { return derive_seed(base, index); }

size_t semd_default_transition_length(size_t rows) {  // serialize.cpp:15-18
    const long long d = std::llround(0.2 * (double)rows);
    const size_t v = d < 1 ? 1 : (size_t)d;
    return std::min(v, rows);
}

int semd_parse_algorithm(const char* name, int* algo) {
    return guard([&] {
        if (!name || !algo) raise(SEMD_INVALID_INPUT, "null argument");
        std::string s;
        for (const char* p = name; *p; ++p) s.push_back((char)std::tolower((unsigned char)*p));
        if (s == "emd") *algo = 0;
        else if (s == "eemd") *algo = 1;
        else if (s == "ceemdan" || s == "eemdan") *algo = 2;
        else raise(SEMD_INVALID_INPUT, "unknown algorithm '%s' (expected emd, eemd, or ceemdan)", name);
    });
}

int semd_find_extrema(semd_ctx* ctx, const double* x, size_t n, size_t* max_idx, double* max_val, size_t* n_max,
                      size_t* min_idx, double* min_val, size_t* n_min) {
    return guard([&] {
        need_ctx(ctx);
        if (n < 3) raise(SEMD_INVALID_INPUT, "find_extrema: signal too short (need at least 3 samples)");
        const double* d_x = ctx->upload(ctx->in_x, x, n);
        ctx->reset_stats(1);
        ctx->configure((long long)n, 1, 1, 0);
        ctx->A.sd_threshold = 0.2;
        ctx->A.max_sift_iters = 1;
        JobSpec J;
        J.a = d_x;
        J.detect_only = 1;
        ctx->set_jobs({J});
        ctx->run(8);
        const Slot& S = ctx->h_slots[0];
        const unsigned nm = S.n[0], nn = S.n[1];
        std::vector<int> idx(std::max(nm, nn));
        const semd::dev::Arena& A = ctx->A;
        // the detect wrote parity 1 (slot started at parity 0)
        if (nm) {
            ck(cudaMemcpy(idx.data(), A.kidx + semd::dev::knot_off(A, 1, 0, 0), nm * 4, cudaMemcpyDeviceToHost), "idx");
            for (unsigned i = 0; i < nm; ++i) max_idx[i] = (size_t)idx[i];
            ctx->gather_values(A.kidx + semd::dev::knot_off(A, 1, 0, 0), nm, d_x, max_val);
        }
        if (nn) {
            ck(cudaMemcpy(idx.data(), A.kidx + semd::dev::knot_off(A, 1, 1, 0), nn * 4, cudaMemcpyDeviceToHost), "idx");
            for (unsigned i = 0; i < nn; ++i) min_idx[i] = (size_t)idx[i];
            ctx->gather_values(A.kidx + semd::dev::knot_off(A, 1, 1, 0), nn, d_x, min_val);
        }
        *n_max = nm;
        *n_min = nn;
    });
}

int semd_envelope(semd_ctx* ctx, const size_t* idx, const double* val, size_t n, size_t length, double* out) {
    return guard([&] {
        need_ctx(ctx);
        if (n < 2) raise(SEMD_INSUFFICIENT_EXTREMA, "envelope: need at least 2 extrema, got %zu", n);
        const size_t N = n + 4;
        ctx->scratch.alloc((N * 4 + length + n * 2) * 8);
        double* xs = ctx->scratch.as<double>();
        double* ys = xs + N;
        double* mom = ys + N;
        double* work = mom + N;
        double* d_out = work + N;
        unsigned long long* d_idx = reinterpret_cast<unsigned long long*>(d_out + length);
        double* d_val = reinterpret_cast<double*>(d_idx + n);
        static_assert(sizeof(size_t) == 8, "size_t must be 64-bit");
        ck(cudaMemcpyAsync(d_idx, idx, n * 8, cudaMemcpyHostToDevice, ctx->stream), "idx");
        ck(cudaMemcpyAsync(d_val, val, n * 8, cudaMemcpyHostToDevice, ctx->stream), "val");
        const bool left = idx[0] != 0, right = idx[n - 1] != length - 1;
        const int Nk = (int)(n + (left ? 2 : 0) + (right ? 2 : 0));
        semd::dev::launch_envelope_knots(d_idx, d_val, (long long)n, (long long)length, xs, ys, ctx->stream);
        semd::dev::launch_envelope(xs, ys, Nk, mom, work, (long long)length, d_out, ctx->stream);
        ck(cudaGetLastError(), "envelope");
        ctx->download(out, d_out, length);
    });
}

int semd_extract_imf(semd_ctx* ctx, const double* x, size_t n, const semd_sift_cfg* cfg_, double* imf,
                     int32_t* sift_count) {
    return guard([&] {
        need_ctx(ctx);
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        if (cfg.max_sift_iters <= 0) {  // the sift loop never runs: the IMF is x itself, 0 sifts
            const double* d_x0 = ctx->upload(ctx->in_x, x, n);
            if (sift_count) *sift_count = 0;
            ctx->download(imf, d_x0, n);
            return;
        }
        if (n < 3) raise(SEMD_INVALID_INPUT, "find_extrema: signal too short (need at least 3 samples)");
        const double* d_x = ctx->upload(ctx->in_x, x, n);
        ctx->reset_stats(1);
        ctx->configure((long long)n, 1, 1, 0);
        ctx->A.sd_threshold = cfg.sd_threshold;
        ctx->A.max_sift_iters = cfg.max_sift_iters;
        ctx->fill_sums(1, -0.0);
        JobSpec J;
        J.kmax = 1;
        J.a = d_x;
        ctx->set_jobs({J});
        ctx->run(ctx->max_steps_for(cfg));
        const Slot& S = ctx->h_slots[0];
        if (S.ended_insufficient) {
            const unsigned bad = S.n[0] < 2 ? S.n[0] : S.n[1];
            raise(SEMD_INSUFFICIENT_EXTREMA, "envelope: need at least 2 extrema, got %u", bad);
        }
        int c = 0;
        ck(cudaMemcpy(&c, ctx->A.imf_sifts, 4, cudaMemcpyDeviceToHost), "count");
        if (sift_count) *sift_count = c;
        ctx->download(imf, ctx->A.sums, n);
    });
}

int semd_decompose(semd_ctx* ctx, int algo, const double* x, size_t n, const semd_sift_cfg* cfg,
                   const semd_ens_cfg* ens, double* imfs, size_t k_cap, size_t* k_out, double* residue,
                   int32_t* sift_counts, semd_trace* trace) {
    return guard([&] {
        need_ctx(ctx);
        size_t K = 0;
        const double* d_x = ctx->upload(ctx->in_x, x, n);
        DBuf& outb = ctx->ser_out;  // context scratch (grow-only)
        outb.alloc((k_cap + 1) * std::max<size_t>(n, 1) * 8);
        double* d_imfs = outb.as<double>();
        double* d_res = d_imfs + k_cap * n;
        int rc = SEMD_OK;
        std::string msg;
        try {
            ctx->decompose_device(algo, d_x, (long long)n, sift_or_default(cfg), ens_or_default(ens), d_imfs, k_cap, &K,
                                  d_res, sift_counts, trace);
        } catch (const Error& e) {
            if (e.code != SEMD_CAPACITY) throw;
            rc = e.code;
            msg = e.msg;
        }
        if (k_out) *k_out = K;
        if (rc) raise(rc, "%s", msg.c_str());
        if (!ctx->has_result()) return;  // root-only ensemble reduction on another rank
        if (imfs && K) ctx->download(imfs, d_imfs, K * n);
        if (residue) ctx->download(residue, d_res, n);
    });
}

int semd_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t n, const semd_sift_cfg* cfg,
                          const semd_ens_cfg* ens, double* d_imfs, size_t k_cap, size_t* k_out, double* d_residue) {
    return guard([&] {
        need_ctx(ctx);
        size_t K = 0;
        try {
            ctx->decompose_device(algo, d_x, (long long)n, sift_or_default(cfg), ens_or_default(ens), d_imfs, k_cap, &K,
                                  d_residue, nullptr, nullptr);
        } catch (...) {
            if (k_out) *k_out = K;
            throw;
        }
        if (k_out) *k_out = K;
    });
}

int semd_eemd_partial_device(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg_,
                             const semd_ens_cfg* ens_, int32_t m_begin, int32_t m_end, double* d_sums, size_t k_cap,
                             size_t* k_out) {
    return semd_eemd_partial_traced_device(ctx, d_x, n, cfg_, ens_, m_begin, m_end, d_sums, k_cap, k_out, nullptr);
}

int semd_eemd_partial_traced_device(semd_ctx* ctx, const double* d_x, size_t n, const semd_sift_cfg* cfg_,
                                    const semd_ens_cfg* ens_, int32_t m_begin, int32_t m_end, double* d_sums,
                                    size_t k_cap, size_t* k_out, semd_trace* trace) {
    return guard([&] {
        need_ctx(ctx);
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        const semd_ens_cfg ens = ens_or_default(ens_);
        if (ens.nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
        if (ens.nstd < 0.0) raise(SEMD_INVALID_INPUT, "ensemble: nstd must be non-negative");
        if (m_begin < 0 || m_end < m_begin) raise(SEMD_INVALID_INPUT, "invalid realization range");
        // emd.cpp:230: a zero-noise ensemble is plain EMD, which ensemble sums cannot reproduce
        // bit-for-bit (sum of nr copies x 1/nr); the caller runs semd_decompose(SEMD_ALGO_EMD).
        if (ens.nstd == 0.0) raise(SEMD_INVALID_INPUT, "eemd shard: nstd == 0 is plain EMD (use semd_decompose)");
        ctx->reset_stats(1);
        const int K =
            m_end > m_begin ? ctx->eemd_partial_device(d_x, (long long)n, cfg, ens, m_begin, m_end, trace) : 0;
        if (m_end > m_begin) ctx->export_trace(trace);
        else if (trace) trace->count = 0;
        if (k_out) *k_out = (size_t)K;
        if ((size_t)K > k_cap) raise(SEMD_CAPACITY, "output holds %zu IMFs, shard has %d", k_cap, K);
        if (k_cap) ck(cudaMemsetAsync(d_sums, 0, k_cap * n * 8, ctx->stream), "zero sums");
        if (K) ck(cudaMemcpyAsync(d_sums, ctx->A.sums, (size_t)K * n * 8, cudaMemcpyDeviceToDevice, ctx->stream), "sums");
        ck(cudaStreamSynchronize(ctx->stream), "partial");
    });
}

int semd_ensemble_finish_device(semd_ctx* ctx, const double* d_x, size_t n, double* d_sums, size_t K, int32_t nr,
                                double* d_residue) {
    return guard([&] {
        need_ctx(ctx);
        if (nr < 1) raise(SEMD_INVALID_INPUT, "ensemble: nr must be at least 1");
        semd::dev::launch_ensemble_finish(d_sums, (int)K, (long long)n, d_x, d_residue, 1.0 / (double)nr, ctx->stream);
        ck(cudaGetLastError(), "finish");
        ck(cudaStreamSynchronize(ctx->stream), "finish");
    });
}

int semd_white_noise(semd_ctx* ctx, size_t n, uint64_t seed, double std, double* out) {
    return guard([&] {
        need_ctx(ctx);
        if (std < 0.0) raise(SEMD_INVALID_INPUT, "white_noise: std must be non-negative");
        if (n == 0) return;
        if (std == 0.0) {
            std::fill(out, out + n, 0.0);  // the reference's Signal(n, 0.0)
            return;
        }
        const long long Ls = ((long long)n + 1) / 2 * 2;
        ctx->scratch.alloc((size_t)Ls * 8);
        ctx->gen_noise({seed}, (long long)n, Ls, ctx->scratch.as<double>(), std);
        ctx->download(out, ctx->scratch.as<double>(), n);
    });
}

int semd_signal_std(semd_ctx* ctx, const double* x, size_t n, double* out) {
    return guard([&] {
        need_ctx(ctx);
        if (n == 0) {
            *out = 0.0;
            return;
        }
        const double* d_x = ctx->upload(ctx->in_x, x, n);
        *out = ctx->device_std(d_x, (long long)n, 1.0);
    });
}

int semd_noise_mode(semd_ctx* ctx, const double* w, size_t n, size_t i, const semd_sift_cfg* cfg, double* out) {
    return guard([&] {
        need_ctx(ctx);
        if (i == 0) raise(SEMD_INVALID_INPUT, "noise_mode: mode index is 1-based");
        const double* d_w = ctx->upload(ctx->in_x, w, n);
        ctx->reset_stats(1);
        const int K = ctx->emd_device(d_w, (long long)n, sift_or_default(cfg), nullptr);
        if (i - 1 < (size_t)K) ctx->download(out, ctx->A.sums + (i - 1) * n, n);
        else std::fill(out, out + n, 0.0);
    });
}

int semd_transition_weights(semd_ctx* ctx, size_t d, double* out) {
    return guard([&] {
        need_ctx(ctx);
        if (d < 1) raise(SEMD_INVALID_INPUT, "transition_weights: D must be at least 1");
        ctx->scratch2.alloc(d * 8);
        semd::dev::launch_transition_weights((long long)d, ctx->scratch2.as<double>(), ctx->stream);
        ctx->download(out, ctx->scratch2.as<double>(), d);
    });
}

static int concat_host(semd_ctx* ctx, const double* x, size_t M, size_t N, size_t D, double* out, int naive) {
    return guard([&] {
        need_ctx(ctx);
        validate_serial(M, N, D);
        const size_t L = M * N + D * (N - 1);
        const double* d_x = ctx->upload(ctx->in_x, x, M * N);
        ctx->scratch.alloc(L * 8);
        concat_device(ctx, d_x, M, N, D, ctx->scratch.as<double>(), naive);
        ctx->download(out, ctx->scratch.as<double>(), L);
    });
}

int semd_concatenate(semd_ctx* ctx, const double* x, size_t M, size_t N, size_t D, double* out) {
    return concat_host(ctx, x, M, N, D, out, 0);
}
int semd_concatenate_naive(semd_ctx* ctx, const double* x, size_t M, size_t N, size_t D, double* out) {
    return concat_host(ctx, x, M, N, D, out, 1);
}

int semd_concatenate_device(semd_ctx* ctx, const double* d_x, size_t M, size_t N, size_t D, double* d_out) {
    return guard([&] {
        need_ctx(ctx);
        concat_device(ctx, d_x, M, N, D, d_out, 0);
        ck(cudaStreamSynchronize(ctx->stream), "concatenate");
    });
}

int semd_deconcatenate_device(semd_ctx* ctx, const double* d_modes, size_t K, size_t L, size_t M, size_t N, size_t D,
                              double* d_out) {
    return guard([&] {
        need_ctx(ctx);
        validate_deconcat(K, L, M, N, D);
        semd::dev::launch_deconcatenate(d_modes, (long long)K, (long long)L, (long long)M, (long long)N, (long long)D,
                                        d_out, ctx->stream);
        ck(cudaGetLastError(), "deconcatenate");
        ck(cudaStreamSynchronize(ctx->stream), "deconcatenate");
    });
}

int semd_deconcatenate(semd_ctx* ctx, const double* modes, size_t K, size_t L, size_t M, size_t N, size_t D,
                       double* out) {
    return guard([&] {
        need_ctx(ctx);
        validate_deconcat(K, L, M, N, D);
        const double* d_m = ctx->upload(ctx->in_x, modes, K * L);
        ctx->scratch.alloc(K * M * N * 8);
        semd::dev::launch_deconcatenate(d_m, (long long)K, (long long)L, (long long)M, (long long)N, (long long)D,
                                        ctx->scratch.as<double>(), ctx->stream);
        ck(cudaGetLastError(), "deconcatenate");
        ctx->download(out, ctx->scratch.as<double>(), K * M * N);
    });
}

static void serial_device(semd_ctx* ctx, int algo, const double* d_x, size_t M, size_t N, size_t D,
                          const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* d_tensor, size_t k_cap,
                          size_t* modes_out, semd_trace* trace) {
    validate_serial(M, N, D);
    const size_t L = M * N + D * (N - 1);
    DBuf& sig = ctx->ser_sig;  // context scratch (grow-only): no cudaMalloc / cudaFree per call
    sig.alloc(L * 8);
    concat_device(ctx, d_x, M, N, D, sig.as<double>(), 0);
    // modes = imfs + residue, row k contiguous
    size_t kc = std::max<size_t>(k_cap, 1);
    DBuf& modes = ctx->ser_modes;
    size_t K = 0;
    for (int attempt = 0;; ++attempt) {
        modes.alloc((kc + 1) * L * 8);
        try {
            ctx->decompose_device(algo, sig.as<double>(), (long long)L, sift_or_default(cfg), ens_or_default(ens),
                                  modes.as<double>(), kc, &K, modes.as<double>() + kc * L, nullptr, trace);
            break;
        } catch (const Error& e) {
            if (e.code != SEMD_CAPACITY || attempt == 3 || K <= kc) throw;  // only an output-capacity miss retries
            kc = std::max(kc * 2, K);
        }
    }
    if (!ctx->has_result()) {  // root-only ensemble reduction: the tensor is produced on the root rank
        *modes_out = K + 1;
        return;
    }
    if (K != kc)  // move the residue right after the K IMFs
        ck(cudaMemcpyAsync(modes.as<double>() + K * L, modes.as<double>() + kc * L, L * 8, cudaMemcpyDeviceToDevice,
                           ctx->stream),
           "residue");
    *modes_out = K + 1;
    if (K + 1 > k_cap) raise(SEMD_CAPACITY, "output holds %zu modes, decomposition has %zu", k_cap, K + 1);
    validate_deconcat(K + 1, L, M, N, D);
    semd::dev::launch_deconcatenate(modes.as<double>(), (long long)(K + 1), (long long)L, (long long)M, (long long)N,
                                    (long long)D, d_tensor, ctx->stream);
    ck(cudaGetLastError(), "deconcatenate");
    ck(cudaStreamSynchronize(ctx->stream), "serial");
}

int semd_serial_decompose(semd_ctx* ctx, int algo, const double* x, size_t M, size_t N, size_t D,
                          const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* tensor, size_t k_cap,
                          size_t* modes_out, semd_trace* trace) {
    return guard([&] {
        need_ctx(ctx);
        validate_serial(M, N, D);
        const double* d_x = ctx->upload(ctx->in_x, x, M * N);
        DBuf& t = ctx->ser_out;
        t.alloc(std::max<size_t>(k_cap, 1) * M * N * 8);
        size_t mo = 0;
        try {
            serial_device(ctx, algo, d_x, M, N, D, cfg, ens, t.as<double>(), k_cap, &mo, trace);
        } catch (...) {
            if (modes_out) *modes_out = mo;
            throw;
        }
        if (modes_out) *modes_out = mo;
        if (ctx->has_result()) ctx->download(tensor, t.as<double>(), mo * M * N);
    });
}

int semd_serial_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t M, size_t N, size_t D,
                                 const semd_sift_cfg* cfg, const semd_ens_cfg* ens, double* d_tensor, size_t k_cap,
                                 size_t* modes_out) {
    return guard([&] {
        need_ctx(ctx);
        size_t mo = 0;
        try {
            serial_device(ctx, algo, d_x, M, N, D, cfg, ens, d_tensor, k_cap, &mo, nullptr);
        } catch (...) {
            if (modes_out) *modes_out = mo;
            throw;
        }
        if (modes_out) *modes_out = mo;
    });
}

int semd_slicewise_decompose(semd_ctx* ctx, int algo, const double* x, size_t M, size_t N, const semd_sift_cfg* cfg_,
                             const semd_ens_cfg* ens_, double* tensor, size_t k_cap, size_t* modes_out) {
    return guard([&] {
        need_ctx(ctx);
        if (algo < 0 || algo > 2) raise(SEMD_INVALID_INPUT, "unknown algorithm");
        if (M == 0 || N == 0) raise(SEMD_INVALID_INPUT, "slicewise_decompose: empty input");
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        const semd_ens_cfg ens = ens_or_default(ens_);
        const double* d_x = ctx->upload(ctx->in_x, x, M * N);
        ctx->reset_stats(1);
        DBuf t(std::max<size_t>(k_cap, 1) * M * N * 8);
        size_t mo = 0;
        try {
            ctx->slicewise_device(algo, d_x, (long long)M, (int)N, cfg, ens, t.as<double>(), k_cap, &mo);
        } catch (...) {
            if (modes_out) *modes_out = mo;
            throw;
        }
        if (modes_out) *modes_out = mo;
        ctx->download(tensor, t.as<double>(), mo * M * N);
    });
}

int semd_slicewise_decompose_device(semd_ctx* ctx, int algo, const double* d_x, size_t M, size_t N,
                                    const semd_sift_cfg* cfg_, const semd_ens_cfg* ens_, double* d_tensor,
                                    size_t k_cap, size_t* modes_out) {
    return guard([&] {
        need_ctx(ctx);
        if (algo < 0 || algo > 2) raise(SEMD_INVALID_INPUT, "unknown algorithm");
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        const semd_ens_cfg ens = ens_or_default(ens_);
        ctx->reset_stats(1);
        size_t mo = 0;
        try {
            ctx->slicewise_device(algo, d_x, (long long)M, (int)N, cfg, ens, d_tensor, k_cap, &mo);
        } catch (...) {
            if (modes_out) *modes_out = mo;
            throw;
        }
        if (modes_out) *modes_out = mo;
    });
}

// ---- device memory and timing on the context stream (bench / driver plumbing) -----------------
int semd_device_alloc(semd_ctx* ctx, size_t bytes, void** d_out) {
    return guard([&] {
        need_ctx(ctx);
        if (!d_out) raise(SEMD_INVALID_INPUT, "null output pointer");
        *d_out = nullptr;
        const cudaError_t e = cudaMalloc(d_out, std::max<size_t>(bytes, 8));
        if (e != cudaSuccess) {
            cudaGetLastError();
            raise(SEMD_NO_MEMORY, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        }
    });
}

int semd_device_free(semd_ctx* ctx, void* d) {
    return guard([&] {
        need_ctx(ctx);
        if (d) ck(cudaFree(d), "cudaFree");
    });
}

int semd_memcpy(semd_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] {
        need_ctx(ctx);
        if (bytes) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream), "memcpy");
        ck(cudaStreamSynchronize(ctx->stream), "memcpy");
    });
}

int semd_host_alloc(semd_ctx* ctx, size_t bytes, void** h_out) {
    return guard([&] {
        need_ctx(ctx);
        if (!h_out) raise(SEMD_INVALID_INPUT, "null output pointer");
        ck(cudaHostAlloc(h_out, std::max<size_t>(bytes, 8), cudaHostAllocDefault), "cudaHostAlloc");
    });
}

int semd_host_free(semd_ctx* ctx, void* h) {
    return guard([&] {
        need_ctx(ctx);
        if (h) ck(cudaFreeHost(h), "cudaFreeHost");
    });
}

int semd_timer_start(semd_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        if (!ctx->tm0) ck(cudaEventCreate(&ctx->tm0), "event");
        if (!ctx->tm1) ck(cudaEventCreate(&ctx->tm1), "event");
        ck(cudaStreamSynchronize(ctx->stream), "timer");
        ck(cudaEventRecord(ctx->tm0, ctx->stream), "timer");
    });
}

int semd_timer_stop(semd_ctx* ctx, double* ms) {
    return guard([&] {
        need_ctx(ctx);
        if (!ctx->tm0 || !ctx->tm1) raise(SEMD_INVALID_INPUT, "semd_timer_stop without semd_timer_start");
        ck(cudaEventRecord(ctx->tm1, ctx->stream), "timer");
        ck(cudaEventSynchronize(ctx->tm1), "timer");
        float f = 0.f;
        ck(cudaEventElapsedTime(&f, ctx->tm0, ctx->tm1), "timer");
        if (ms) *ms = (double)f;
    });
}

// ---- multi-GPU: one context per rank joined by an NCCL communicator ---------------------------
int semd_comm_unique_id(void* id_out, size_t bytes) {
    return guard([&] {
        if (!id_out || bytes < sizeof(ncclUniqueId)) raise(SEMD_INVALID_INPUT, "unique id buffer needs %zu bytes",
                                                           sizeof(ncclUniqueId));
        ncclUniqueId id;
        nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int semd_comm_init(semd_ctx* ctx, const void* id, size_t bytes, int rank, int world) {
    return guard([&] {
        need_ctx(ctx);
        if (!id || bytes < sizeof(ncclUniqueId)) raise(SEMD_INVALID_INPUT, "unique id needs %zu bytes",
                                                       sizeof(ncclUniqueId));
        if (world < 1 || rank < 0 || rank >= world) raise(SEMD_INVALID_INPUT, "rank %d out of range (world %d)", rank,
                                                          world);
        if (ctx->comm) {
            nccl_api().CommDestroy(ctx->comm);
            ctx->comm = nullptr;
        }
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        ncclComm_t c = nullptr;
        nck(nccl().CommInitRank(&c, world, uid, rank), "ncclCommInitRank");
        ctx->comm = c;
        ctx->rank = rank;
        ctx->world = world;
        ctx->root = -1;
    });
}

int semd_comm_set_root(semd_ctx* ctx, int root) {
    return guard([&] {
        need_ctx(ctx);
        if (root >= ctx->world) raise(SEMD_INVALID_INPUT, "root %d out of range (world %d)", root, ctx->world);
        ctx->root = root < 0 ? -1 : root;
    });
}

int semd_comm_info(semd_ctx* ctx, int* rank, int* world) {
    return guard([&] {
        need_ctx(ctx);
        if (rank) *rank = ctx->comm ? ctx->rank : 0;
        if (world) *world = ctx->comm ? ctx->world : 1;
    });
}

int semd_comm_allreduce_host(semd_ctx* ctx, double* vals, size_t n, int op) {
    return guard([&] {
        need_ctx(ctx);
        if (!ctx->comm || n == 0) return;
        if (op != 0 && op != 1) raise(SEMD_INVALID_INPUT, "op must be 0 (sum) or 1 (max)");
        ctx->comm_buf.alloc(std::max<size_t>(64, n * 8));
        double* d = ctx->comm_buf.as<double>();
        ck(cudaMemcpyAsync(d, vals, n * 8, cudaMemcpyHostToDevice, ctx->stream), "allreduce");
        nck(nccl().AllReduce(d, d, n, ncclDouble, op ? ncclMax : ncclSum, ctx->comm, ctx->stream), "ncclAllReduce");
        ck(cudaMemcpyAsync(vals, d, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "allreduce");
        ck(cudaStreamSynchronize(ctx->stream), "allreduce");
    });
}

int semd_comm_destroy(semd_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        if (ctx->comm) {
            ck(cudaStreamSynchronize(ctx->stream), "comm");
            nck(nccl_api().CommDestroy(ctx->comm), "ncclCommDestroy");
        }
        ctx->comm = nullptr;
        ctx->rank = 0;
        ctx->world = 1;
        ctx->root = -1;
    });
}

// ---- recognition.cpp:281-298: the feature bank's decompositions, batched ---------------------
int semd_serial_decompose_batch(semd_ctx* ctx, int algo, const double* x, size_t B, size_t M, size_t N, size_t D,
                                const semd_sift_cfg* cfg_, const semd_ens_cfg* ens_, double* tensor, size_t k_cap,
                                size_t* modes_out) {
    return guard([&] {
        need_ctx(ctx);
        if (algo < 0 || algo > 2) raise(SEMD_INVALID_INPUT, "unknown algorithm");
        if (!modes_out) raise(SEMD_INVALID_INPUT, "null modes_out");
        const semd_sift_cfg cfg = sift_or_default(cfg_);
        const semd_ens_cfg ens = ens_or_default(ens_);
        const double* d_x = ctx->upload(ctx->in_x, x, B * M * N);
        ctx->reset_stats(1);
        DBuf t(std::max<size_t>(k_cap, 1) * B * M * N * 8);
        ctx->serial_batch_device(algo, d_x, (long long)B, (long long)M, (long long)N, (long long)D, cfg, ens,
                                 t.as<double>(), k_cap, modes_out);
        ctx->download(tensor, t.as<double>(), k_cap * B * M * N);
    });
}

}  // extern "C"

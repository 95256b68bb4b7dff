// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile from the sources where they lie under
// /root/reference/proj/src into oracle/_ref/libsemd_ref.so. It lets the
// Python tests and the bench's CPU-baseline leg call the reference itself.
// It also holds the trace replayer: the extract_imf loop (emd.cpp:127-153)
// re-driven through the reference's public find_extrema / envelope so that
// every find_extrema call's extrema lists can be hashed; ref_emd_traced checks
// its own output against semd::emd bit-for-bit and reports any divergence.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <filesystem>
#include <fstream>

#include "semd/emd.hpp"
#include "semd/io.hpp"
#include "semd/recognition.hpp"
#include "semd/serialize.hpp"
#include "semd/synth.hpp"
#ifdef REF_HAVE_JSON
#include "nlohmann/json.hpp"
#endif

namespace {

thread_local std::string g_err;

struct TraceRec {
    int32_t task, m, k, iter;
    uint32_t n_max, n_min;
    uint64_t hash;
};

uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t hash_extrema(const semd::Extrema& e) {
    uint64_t h = 0;
    for (std::size_t j = 0; j < e.max_idx.size(); ++j) h += mix64((uint64_t(j) << 32) ^ uint64_t(e.max_idx[j]));
    for (std::size_t j = 0; j < e.min_idx.size(); ++j)
        h += mix64(0x8000000000000000ULL ^ (uint64_t(j) << 32) ^ uint64_t(e.min_idx[j]));
    return h;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const semd::InsufficientExtrema& e) {
        g_err = e.what();
        return 2;
    } catch (const semd::InvalidInput& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

struct Out {
    std::vector<double> imfs;  // K x n
    std::vector<double> residue;
    std::vector<int32_t> counts;
    std::vector<TraceRec> trace;
    std::size_t K = 0;
};

void store(Out* o, const semd::Decomposition& d) {
    o->K = d.imfs.size();
    const std::size_t n = d.residue.size();
    o->imfs.resize(o->K * n);
    for (std::size_t k = 0; k < o->K; ++k) std::memcpy(o->imfs.data() + k * n, d.imfs[k].data(), n * 8);
    o->residue = d.residue;
}

// The replayer: emd.cpp:127-153 through the public API, with per-call traces.
semd::SiftResult replay_extract(const semd::Signal& x, const semd::SiftConfig& cfg, std::vector<TraceRec>* tr,
                                int task, int m, int k) {
    semd::SiftResult res{x, 0};
    semd::Signal& cur = res.imf;
    for (int iter = 0; iter < cfg.max_sift_iters; ++iter) {
        semd::Extrema ext = semd::find_extrema(cur);
        tr->push_back({task, m, k, iter, uint32_t(ext.max_idx.size()), uint32_t(ext.min_idx.size()), hash_extrema(ext)});
        semd::Signal upper, lower;
        try {
            upper = semd::envelope(ext.max_idx, ext.max_val, cur.size());
            lower = semd::envelope(ext.min_idx, ext.min_val, cur.size());
        } catch (const semd::InsufficientExtrema&) {
            if (res.sift_count == 0) throw;
            return res;
        }
        double num = 0.0, den = 0.0;
        for (std::size_t i = 0; i < cur.size(); ++i) {
            const double mean = 0.5 * (upper[i] + lower[i]);
            num += mean * mean;
            den += cur[i] * cur[i];
            cur[i] -= mean;
        }
        ++res.sift_count;
        if (den == 0.0 || num / den < cfg.sd_threshold) return res;
    }
    return res;
}

semd::Decomposition replay_emd(const semd::Signal& x, const semd::SiftConfig& cfg, std::vector<TraceRec>* tr,
                               std::vector<int32_t>* counts, int m) {
    if (x.size() < 4) throw semd::InvalidInput("emd: signal too short (need at least 4 samples)");
    semd::Decomposition d;
    semd::Signal residue = x;
    while (cfg.max_imfs == 0 || d.imfs.size() < std::size_t(cfg.max_imfs)) {
        semd::SiftResult r;
        try {
            r = replay_extract(residue, cfg, tr, 0, m, int(d.imfs.size()));
        } catch (const semd::InsufficientExtrema&) {
            break;
        }
        for (std::size_t i = 0; i < residue.size(); ++i) residue[i] -= r.imf[i];
        if (counts) counts->push_back(r.sift_count);
        d.imfs.push_back(std::move(r.imf));
    }
    d.residue = std::move(residue);
    return d;
}

bool same(const semd::Decomposition& a, const semd::Decomposition& b) {
    if (a.imfs.size() != b.imfs.size()) return false;
    for (std::size_t k = 0; k < a.imfs.size(); ++k)
        if (a.imfs[k] != b.imfs[k]) return false;
    return a.residue == b.residue;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_out_new() { return new Out(); }
void ref_out_free(void* o) { delete static_cast<Out*>(o); }
std::size_t ref_out_K(void* o) { return static_cast<Out*>(o)->K; }
const double* ref_out_imfs(void* o) { return static_cast<Out*>(o)->imfs.data(); }
const double* ref_out_residue(void* o) { return static_cast<Out*>(o)->residue.data(); }
std::size_t ref_out_ncounts(void* o) { return static_cast<Out*>(o)->counts.size(); }
const int32_t* ref_out_counts(void* o) { return static_cast<Out*>(o)->counts.data(); }
std::size_t ref_out_ntrace(void* o) { return static_cast<Out*>(o)->trace.size(); }
const void* ref_out_trace(void* o) { return static_cast<Out*>(o)->trace.data(); }

uint64_t ref_derive_seed(uint64_t base, uint64_t index) { return semd::derive_seed(base, index); }

void ref_mt19937_64(uint64_t seed, std::size_t n, uint64_t* out) {
    std::mt19937_64 g(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = g();
}

int ref_white_noise(std::size_t n, uint64_t seed, double std, double* out) {
    return guard([&] {
        const semd::Signal w = semd::white_noise(n, seed, std);
        std::memcpy(out, w.data(), n * 8);
    });
}

double ref_signal_std(const double* x, std::size_t n) { return semd::signal_std(semd::Signal(x, x + n)); }

int ref_find_extrema(const double* x, std::size_t n, std::size_t* max_idx, double* max_val, std::size_t* n_max,
                     std::size_t* min_idx, double* min_val, std::size_t* n_min) {
    return guard([&] {
        const semd::Extrema e = semd::find_extrema(semd::Signal(x, x + n));
        *n_max = e.max_idx.size();
        *n_min = e.min_idx.size();
        std::memcpy(max_idx, e.max_idx.data(), *n_max * sizeof(std::size_t));
        std::memcpy(max_val, e.max_val.data(), *n_max * 8);
        std::memcpy(min_idx, e.min_idx.data(), *n_min * sizeof(std::size_t));
        std::memcpy(min_val, e.min_val.data(), *n_min * 8);
    });
}

int ref_envelope(const std::size_t* idx, const double* val, std::size_t n, std::size_t length, double* out) {
    return guard([&] {
        const semd::Signal e = semd::envelope(std::vector<std::size_t>(idx, idx + n), semd::Signal(val, val + n), length);
        std::memcpy(out, e.data(), length * 8);
    });
}

int ref_extract_imf(const double* x, std::size_t n, double sd, int iters, int imfs, double* out, int32_t* count) {
    return guard([&] {
        const semd::SiftResult r = semd::extract_imf(semd::Signal(x, x + n), {sd, iters, imfs});
        std::memcpy(out, r.imf.data(), n * 8);
        *count = r.sift_count;
    });
}

// The reference's own decompose (algo 0/1/2), bit-for-bit its output.
int ref_decompose(const double* x, std::size_t n, int algo, double sd, int iters, int imfs, double nstd, int nr,
                  uint64_t seed, void* out) {
    return guard([&] {
        const semd::Decomposition d = semd::decompose(semd::Signal(x, x + n), static_cast<semd::Algorithm>(algo),
                                                      {sd, iters, imfs}, {nstd, nr, seed});
        store(static_cast<Out*>(out), d);
    });
}

// EMD via the replayer; returns 3 if the replay is not bit-identical to semd::emd.
int ref_emd_traced(const double* x, std::size_t n, double sd, int iters, int imfs, void* out) {
    int mismatch = 0;
    int rc = guard([&] {
        Out* o = static_cast<Out*>(out);
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const semd::Decomposition d = replay_emd(s, cfg, &o->trace, &o->counts, 0);
        if (!same(d, semd::emd(s, cfg))) mismatch = 1;
        store(o, d);
    });
    if (rc == 0 && mismatch) {
        g_err = "replay diverged from semd::emd";
        return 3;
    }
    return rc;
}

// EEMD realizations [m_begin, m_end) through the replayer (per-realization
// traces and sift counts; counts are concatenated in realization order), with
// the per-realization emd checked against semd::emd. Sums are unscaled.
int ref_eemd_traced(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd, int nr,
                    uint64_t seed, int m_begin, int m_end, void* out) {
    int mismatch = 0;
    int rc = guard([&] {
        Out* o = static_cast<Out*>(out);
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        if (nr < 1) throw semd::InvalidInput("ensemble: nr must be at least 1");
        const double beta = nstd * semd::signal_std(s);
        std::vector<semd::Signal> sums;
        for (int m = m_begin; m < m_end; ++m) {
            const semd::Signal w = semd::white_noise(n, semd::derive_seed(seed, std::uint64_t(m)));
            semd::Signal xm(n);
            for (std::size_t i = 0; i < n; ++i) xm[i] = s[i] + beta * w[i];
            std::vector<int32_t> counts;
            const semd::Decomposition d = replay_emd(xm, cfg, &o->trace, &counts, m);
            if (!same(d, semd::emd(xm, cfg))) mismatch = 1;
            o->counts.push_back(int32_t(d.imfs.size()));  // K_m, then its sift counts
            o->counts.insert(o->counts.end(), counts.begin(), counts.end());
            while (sums.size() < d.imfs.size()) sums.emplace_back(n, 0.0);
            for (std::size_t k = 0; k < d.imfs.size(); ++k)
                for (std::size_t i = 0; i < n; ++i) sums[k][i] += d.imfs[k][i];
        }
        o->K = sums.size();
        o->imfs.resize(o->K * n);
        for (std::size_t k = 0; k < o->K; ++k) std::memcpy(o->imfs.data() + k * n, sums[k].data(), n * 8);
        o->residue.assign(n, 0.0);
    });
    if (rc == 0 && mismatch) {
        g_err = "replay diverged from semd::emd";
        return 3;
    }
    return rc;
}

// All-core realization-parallel reference EEMD work (the CPU baseline of
// BASELINE.md): realizations [m_begin, m_begin+count) of x + beta*w_m, each
// decomposed by the reference's own semd::emd, on `threads` threads. This is
// exactly eemd()'s per-realization work (emd.cpp:237-244) without its
// NR x K x L store; the sifted-sample count is taken from the parity-checked
// GPU run of the same realizations.
int ref_emd_realizations(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd,
                         uint64_t seed, int m_begin, int count, int threads, double* checksum) {
    return guard([&] {
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const double beta = nstd * semd::signal_std(s);
        std::vector<double> part(std::size_t(threads > 0 ? threads : 1), 0.0);
        auto work = [&](int tid) {
            for (int q = tid; q < count; q += threads) {
                const int m = m_begin + q;
                const semd::Signal w = semd::white_noise(n, semd::derive_seed(seed, std::uint64_t(m)));
                semd::Signal xm(n);
                for (std::size_t i = 0; i < n; ++i) xm[i] = s[i] + beta * w[i];
                const semd::Decomposition d = semd::emd(xm, cfg);
                part[std::size_t(tid)] += d.imfs.empty() ? 0.0 : d.imfs[0][n / 2];
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
        for (auto& t : pool) t.join();
        double c = 0.0;
        for (double v : part) c += v;
        *checksum = c;
    });
}

// CEEMDAN (emd.cpp:264-344) re-driven through the replayer so every
// find_extrema call is traced (task 1 noise IMF, 2 first mode, 3 stage check);
// the result is checked bit-for-bit against semd::ceemdan.
int ref_ceemdan_traced(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd, int nr,
                       uint64_t seed, void* out) {
    int mismatch = 0;
    int rc = guard([&] {
        Out* o = static_cast<Out*>(out);
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const semd::EnsembleConfig ens{nstd, nr, seed};
        std::vector<TraceRec>* tr = &o->trace;
        const std::size_t nrr = std::size_t(nr);
        std::vector<semd::Signal> noise_res(nrr);
        std::vector<bool> alive(nrr, true);
        for (std::size_t m = 0; m < nrr; ++m) noise_res[m] = semd::white_noise(n, semd::derive_seed(seed, m));
        auto first_mode = [&](const semd::Signal& v, int m, int k) {
            try {
                return replay_extract(v, cfg, tr, 2, m, k).imf;
            } catch (const semd::InsufficientExtrema&) {
                return semd::Signal(n, 0.0);
            }
        };
        semd::Decomposition d;
        semd::Signal residue = s;
        {
            const double beta0 = nstd * semd::signal_std(s);
            semd::Signal mode(n, 0.0);
            for (std::size_t m = 0; m < nrr; ++m) {
                semd::Signal xm(n);
                for (std::size_t i = 0; i < n; ++i) xm[i] = s[i] + beta0 * noise_res[m][i];
                const semd::Signal e1 = first_mode(xm, int(m), 0);
                for (std::size_t i = 0; i < n; ++i) mode[i] += e1[i];
            }
            const double inv = 1.0 / double(nrr);
            for (std::size_t i = 0; i < n; ++i) {
                mode[i] *= inv;
                residue[i] -= mode[i];
            }
            d.imfs.push_back(std::move(mode));
        }
        while (cfg.max_imfs == 0 || d.imfs.size() < std::size_t(cfg.max_imfs)) {
            const semd::Extrema ext = semd::find_extrema(residue);
            const int k = int(d.imfs.size());
            tr->push_back({3, -1, k, 0, uint32_t(ext.max_idx.size()), uint32_t(ext.min_idx.size()), hash_extrema(ext)});
            if (ext.total() < 3) break;
            const double beta_i = nstd * semd::signal_std(residue);
            semd::Signal mode(n, 0.0);
            for (std::size_t m = 0; m < nrr; ++m) {
                semd::Signal ei(n, 0.0);
                if (alive[m]) {
                    try {
                        semd::SiftResult r = replay_extract(noise_res[m], cfg, tr, 1, int(m), k);
                        ei = std::move(r.imf);
                        for (std::size_t i = 0; i < n; ++i) noise_res[m][i] -= ei[i];
                    } catch (const semd::InsufficientExtrema&) {
                        alive[m] = false;
                    }
                }
                semd::Signal sm(n);
                for (std::size_t i = 0; i < n; ++i) sm[i] = residue[i] + beta_i * ei[i];
                const semd::Signal e1 = first_mode(sm, int(m), k);
                for (std::size_t i = 0; i < n; ++i) mode[i] += e1[i];
            }
            const double inv = 1.0 / double(nrr);
            bool all_zero = true;
            for (std::size_t i = 0; i < n; ++i) {
                mode[i] *= inv;
                if (mode[i] != 0.0) all_zero = false;
            }
            if (all_zero) break;
            for (std::size_t i = 0; i < n; ++i) residue[i] -= mode[i];
            d.imfs.push_back(std::move(mode));
        }
        d.residue = std::move(residue);
        if (!same(d, semd::ceemdan(s, cfg, ens))) mismatch = 1;
        store(o, d);
    });
    if (rc == 0 && mismatch) {
        g_err = "replay diverged from semd::ceemdan";
        return 3;
    }
    return rc;
}


// ---- full-size ensemble goldens (tests/golden/make_golden_ensembles.py) ------------------

// One EEMD realization m of x (emd.cpp:237-244: w = white_noise(n, derive_seed(seed, m)),
// xm = x + beta*w, emd(xm)) through the replayer: per-IMF sift counts, the trace, and a
// compact summary of the IMFs (per-IMF sequential L2 norm, values at `ns` fixed indices).
// check != 0 also runs semd::emd and fails (3) unless the replay is bit-identical.
// Out: K, counts = sift counts, trace, imfs = K x ns sampled values, residue = K norms.
int ref_realization_summary(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd,
                            uint64_t seed, int m, int check, const uint64_t* sidx, std::size_t ns, void* out) {
    int mismatch = 0;
    int rc = guard([&] {
        Out* o = static_cast<Out*>(out);
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const double beta = nstd * semd::signal_std(s);
        semd::Signal xm(n);
        {
            const semd::Signal w = semd::white_noise(n, semd::derive_seed(seed, std::uint64_t(m)));
            for (std::size_t i = 0; i < n; ++i) xm[i] = s[i] + beta * w[i];
        }
        const semd::Decomposition d = replay_emd(xm, cfg, &o->trace, &o->counts, m);
        if (check && !same(d, semd::emd(xm, cfg))) mismatch = 1;
        o->K = d.imfs.size();
        o->imfs.assign(o->K * ns, 0.0);
        o->residue.assign(o->K, 0.0);
        for (std::size_t k = 0; k < o->K; ++k) {
            double acc = 0.0;
            for (double v : d.imfs[k]) acc += v * v;
            o->residue[k] = std::sqrt(acc);
            for (std::size_t j = 0; j < ns; ++j) o->imfs[k * ns + j] = d.imfs[k][sidx[j]];
        }
    });
    if (rc == 0 && mismatch) {
        g_err = "replay diverged from semd::emd";
        return 3;
    }
    return rc;
}

// The reference eemd() (emd.cpp:228-262) with its NR x K x L realization store replaced by
// in-order streaming: realizations are decomposed by the UNMODIFIED semd::emd on `threads`
// workers and added to the sums strictly in realization order, so the result is bit-identical
// to semd::eemd (skipping a missing IMF equals adding eemd()'s zero padding). Needed where
// eemd() itself cannot run (C5 would store 2.2 TB). Out: K, imfs (means), residue,
// counts = per-realization K.
int ref_eemd_stream(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd, int nr,
                    uint64_t seed, int threads, void* out) {
    return guard([&] {
        Out* o = static_cast<Out*>(out);
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        if (nr < 1) throw semd::InvalidInput("ensemble: nr must be at least 1");
        if (nstd == 0.0) {
            store(o, semd::emd(s, cfg));
            return;
        }
        const double beta = nstd * semd::signal_std(s);
        const int T = std::max(1, threads);
        std::mutex mu;
        std::condition_variable cv;
        std::map<int, std::vector<semd::Signal>> ready;
        int next_add = 0;
        std::atomic<int> next_m{0};
        std::string err;
        auto work = [&] {
            for (;;) {
                const int m = next_m.fetch_add(1);
                if (m >= nr) return;
                {
                    std::unique_lock<std::mutex> lk(mu);  // bound the realizations held in memory
                    cv.wait(lk, [&] { return m < next_add + T + 1 || !err.empty(); });
                    if (!err.empty()) return;
                }
                try {
                    const semd::Signal w = semd::white_noise(n, semd::derive_seed(seed, std::uint64_t(m)));
                    semd::Signal xm(n);
                    for (std::size_t i = 0; i < n; ++i) xm[i] = s[i] + beta * w[i];
                    semd::Decomposition d = semd::emd(xm, cfg);
                    std::lock_guard<std::mutex> lk(mu);
                    ready[m] = std::move(d.imfs);
                } catch (const std::exception& e) {
                    std::lock_guard<std::mutex> lk(mu);
                    err = e.what();
                }
                cv.notify_all();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(work);
        std::vector<semd::Signal> sums;
        o->counts.clear();
        for (int m = 0; m < nr; ++m) {
            std::vector<semd::Signal> r;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return ready.count(m) || !err.empty(); });
                if (!err.empty()) break;
                r = std::move(ready[m]);
                ready.erase(m);
            }
            o->counts.push_back(int32_t(r.size()));
            while (sums.size() < r.size()) sums.emplace_back(n, 0.0);
            for (std::size_t k = 0; k < r.size(); ++k)
                for (std::size_t i = 0; i < n; ++i) sums[k][i] += r[k][i];
            {
                std::lock_guard<std::mutex> lk(mu);
                next_add = m + 1;
            }
            cv.notify_all();
        }
        for (auto& t : pool) t.join();
        if (!err.empty()) throw std::runtime_error(err);
        const double inv = 1.0 / static_cast<double>(nr);
        for (auto& imf : sums)
            for (double& v : imf) v *= inv;
        semd::Decomposition d;
        d.residue = s;
        for (const auto& imf : sums)
            for (std::size_t i = 0; i < n; ++i) d.residue[i] -= imf[i];
        d.imfs = std::move(sums);
        store(o, d);
    });
}

// Sift counts of EEMD realizations [m_begin, m_begin+count) on `threads` threads: emd()'s
// loop (emd.cpp:155-172) over the reference's public extract_imf (emd.hpp:62), which
// returns the sift count emd() discards. *sifted = n * total sift iterations. The CPU
// baseline times semd::emd and takes its sifted-sample count from here (computed on the CPU).
int ref_realization_sifts(const double* x, std::size_t n, double sd, int iters, int imfs, double nstd,
                          uint64_t seed, int m_begin, int count, int threads, uint64_t* sifted, int32_t* per_m) {
    return guard([&] {
        const semd::Signal s(x, x + n);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const double beta = nstd * semd::signal_std(s);
        const int T = std::max(1, threads);
        std::vector<uint64_t> part(std::size_t(T), 0);
        std::vector<std::string> errs(static_cast<std::size_t>(T));
        auto work = [&](int tid) {
            try {
                for (int q = tid; q < count; q += T) {
                    const int m = m_begin + q;
                    const semd::Signal w = semd::white_noise(n, semd::derive_seed(seed, std::uint64_t(m)));
                    semd::Signal residue(n);
                    for (std::size_t i = 0; i < n; ++i) residue[i] = s[i] + beta * w[i];
                    int32_t sifts = 0, k = 0;
                    while (cfg.max_imfs == 0 || k < cfg.max_imfs) {
                        semd::SiftResult r;
                        try {
                            r = semd::extract_imf(residue, cfg);
                        } catch (const semd::InsufficientExtrema&) {
                            break;
                        }
                        for (std::size_t i = 0; i < n; ++i) residue[i] -= r.imf[i];
                        sifts += r.sift_count;
                        ++k;
                    }
                    if (per_m) per_m[q] = sifts;
                    part[std::size_t(tid)] += uint64_t(sifts) * n;
                }
            } catch (const std::exception& e) {
                errs[std::size_t(tid)] = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(work, t);
        for (auto& t : pool) t.join();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        uint64_t tot = 0;
        for (uint64_t v : part) tot += v;
        *sifted = tot;
    });
}

int ref_concatenate(const double* x, std::size_t M, std::size_t N, std::size_t D, int naive, double* out) {
    return guard([&] {
        semd::MultiSignal ms(M, N);
        for (std::size_t j = 0; j < N; ++j)
            for (std::size_t i = 0; i < M; ++i) ms(i, j) = x[j * M + i];
        const semd::Signal s = naive ? semd::concatenate_naive(ms, D) : semd::concatenate(ms, D);
        std::memcpy(out, s.data(), s.size() * 8);
    });
}

int ref_deconcatenate(const double* modes, std::size_t K, std::size_t L, std::size_t M, std::size_t N,
                      std::size_t D, double* out) {
    return guard([&] {
        std::vector<semd::Signal> v;
        for (std::size_t k = 0; k < K; ++k) v.emplace_back(modes + k * L, modes + (k + 1) * L);
        const semd::ImfTensor t = semd::deconcatenate(v, M, N, D);
        std::memcpy(out, t.data().data(), t.data().size() * 8);
    });
}

int ref_serial_decompose(const double* x, std::size_t M, std::size_t N, std::size_t D, int algo, double sd,
                         int iters, int imfs, double nstd, int nr, uint64_t seed, void* out) {
    return guard([&] {
        semd::MultiSignal ms(M, N);
        for (std::size_t j = 0; j < N; ++j)
            for (std::size_t i = 0; i < M; ++i) ms(i, j) = x[j * M + i];
        const semd::ImfTensor t = semd::serial_decompose(ms, D, static_cast<semd::Algorithm>(algo),
                                                         {sd, iters, imfs}, {nstd, nr, seed});
        Out* o = static_cast<Out*>(out);
        o->K = t.modes();
        o->imfs = t.data();
    });
}

int ref_multivariate_sinusoids(std::size_t n, double fs, double* out) {
    return guard([&] {
        const semd::MultiSignal s = semd::multivariate_sinusoids(semd::PickupMask::standard(), n, fs);
        std::memcpy(out, s.data().data(), s.data().size() * 8);
    });
}

std::size_t ref_default_transition_length(std::size_t rows) { return semd::default_transition_length(rows); }

// The reference CLI's `decompose` (cli.cpp:93-134) restated over the reference's own library
// functions (read_csv / read_pgm / image_to_multisignal, serial_decompose, write_csv / write_pgm)
// and nlohmann::json for the sidecar (cli.cpp:51-64): the golden outputs for semd-cli. cli.cpp
// itself needs CLI11, which is not in this image.
int ref_cli_decompose(const char* input, const char* algo_name, const char* d_flag, double nstd, int nr,
                      uint64_t seed, double sd, int iters, int imfs, const char* out_dir) {
    return guard([&] {
        namespace fs = std::filesystem;
        const semd::Algorithm algo = semd::parse_algorithm(algo_name);
        const semd::SiftConfig cfg{sd, iters, imfs};
        const semd::EnsembleConfig ens{nstd, nr, seed};
        fs::create_directories(out_dir);
        std::string ext = fs::path(input).extension().string();
        for (char& c : ext) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
        const bool is_pgm = ext == ".pgm";
        const std::string stem = fs::path(input).stem().string();
        semd::MultiSignal data;
        std::vector<std::string> header;
        if (is_pgm) {
            data = semd::image_to_multisignal(semd::read_pgm(input));
            for (std::size_t j = 0; j < data.channels(); ++j) header.push_back("c" + std::to_string(j + 1));
        } else {
            semd::CsvData csv = semd::read_csv(input);
            data = std::move(csv.data);
            header = std::move(csv.header);
        }
        const std::string dfl(d_flag);
        const std::size_t d = dfl == "auto" ? semd::default_transition_length(data.rows()) : std::stoul(dfl);
        const semd::ImfTensor t = semd::serial_decompose(data, d, algo, cfg, ens);
        for (std::size_t k = 0; k < t.modes(); ++k) {
            char nb[16];
            std::snprintf(nb, sizeof nb, "imf_%02zu", k + 1);
            const std::string name = stem + "_" + (k + 1 == t.modes() ? std::string("residue") : std::string(nb));
            semd::MultiSignal mode(t.rows(), t.channels());
            for (std::size_t j = 0; j < t.channels(); ++j)
                for (std::size_t i = 0; i < t.rows(); ++i) mode(i, j) = t(i, j, k);
            semd::write_csv((fs::path(out_dir) / (name + ".csv")).string(), mode, header);
            if (is_pgm) {
                semd::Image img(t.rows(), t.channels());
                for (std::size_t c = 0; c < t.channels(); ++c)
                    for (std::size_t r = 0; r < t.rows(); ++r) img(r, c) = t(r, c, k);
                semd::write_pgm((fs::path(out_dir) / (name + ".pgm")).string(), img, true);
            }
        }
#ifdef REF_HAVE_JSON
        nlohmann::json j{{"M", data.rows()}, {"N", data.channels()}, {"D", d}, {"K", t.modes()},
                         {"algorithm", semd::algorithm_name(algo)}, {"seed", ens.base_seed},
                         {"nstd", ens.nstd}, {"nr", ens.nr}};
        std::ofstream(fs::path(out_dir) / (stem + "_decomposition.json")) << j.dump(2) << '\n';
#else
        throw std::runtime_error("built without nlohmann::json");
#endif
    });
}

// nlohmann::json's text for one double (the sidecar's nstd), for the formatter test.
int ref_json_double(double v, char* out, std::size_t cap) {
#ifdef REF_HAVE_JSON
    const std::string s = nlohmann::json(v).dump();
    std::snprintf(out, cap, "%s", s.c_str());
    return 0;
#else
    return 4;
#endif
}

int ref_synth_signals_csv(std::size_t n, double fs, const char* path) {
    return guard([&] {
        const semd::MultiSignal s = semd::multivariate_sinusoids(semd::PickupMask::standard(), n, fs);
        std::vector<std::string> header;
        for (const char* name : semd::PickupMask::names()) header.push_back(name);
        semd::write_csv(path, s, header);
    });
}

// recognition.cpp:281-298 build_feature_bank on B images (row-major rows x cols each); out gets
// bank.features(1, k) for k = 1..target: B x target x (rows*cols) doubles.
int ref_feature_bank(const double* imgs, std::size_t B, std::size_t rows, std::size_t cols, int algo, std::size_t d,
                     double nstd, int nr, uint64_t seed, double snr_db, uint64_t speckle_seed, std::size_t target,
                     double* out) {
    return guard([&] {
        semd::FaceDataset ds;
        for (std::size_t b = 0; b < B; ++b) {
            semd::Image img(rows, cols);
            for (std::size_t p = 0; p < rows * cols; ++p) img.data()[p] = imgs[b * rows * cols + p];
            ds.images.push_back(std::move(img));
            ds.labels.push_back(int(b) + 1);
        }
        const semd::FaceFeatureBank bank = semd::build_feature_bank(
            ds, static_cast<semd::Algorithm>(algo), d, semd::SiftConfig{}, {nstd, nr, seed}, snr_db, speckle_seed, target);
        const std::size_t dim = rows * cols;
        for (std::size_t k = 1; k <= target; ++k) {
            const auto f = bank.features(1, k);
            for (std::size_t b = 0; b < B; ++b)
                std::memcpy(out + (b * target + (k - 1)) * dim, f[b].data(), dim * 8);
        }
    });
}

int ref_write_pgm(const double* px, std::size_t rows, std::size_t cols, int rescale, const char* path) {
    return guard([&] {
        semd::Image img(rows, cols);
        for (std::size_t p = 0; p < rows * cols; ++p) img.data()[p] = px[p];
        semd::write_pgm(path, img, rescale != 0);
    });
}


}  // extern "C"

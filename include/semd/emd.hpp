// semd/emd.hpp -- the reference's 1-D decomposition API
// (proj/include/semd/emd.hpp:1-120) with identical signatures, defaults,
// exception types and messages, implemented over the B200 C ABI
// (include/semd_b200.h). Link with libsemd_b200.so.
#pragma once

#include <cctype>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#include "../semd_b200.h"
#include "types.hpp"

namespace semd {

struct SiftConfig {
    double sd_threshold = 0.2;
    int max_sift_iters = 300;
    int max_imfs = 0;
};

struct EnsembleConfig {
    double nstd = 0.2;
    int nr = 100;
    std::uint64_t base_seed = 0;
};

struct Extrema {
    std::vector<std::size_t> max_idx;
    Signal max_val;
    std::vector<std::size_t> min_idx;
    Signal min_val;
    std::size_t total() const { return max_idx.size() + min_idx.size(); }
};

struct SiftResult {
    Signal imf;
    int sift_count = 0;
};

enum class Algorithm { Emd, Eemd, Ceemdan };

namespace detail {

/// One engine context per host thread (device from SEMD_DEVICE, default 0).
struct ThreadContext {
    semd_ctx* ctx = nullptr;
    ~ThreadContext() {
        if (ctx) semd_ctx_destroy(ctx);
    }
};

inline void check(int rc) {
    if (rc == SEMD_OK) return;
    const std::string msg = semd_last_error();
    if (rc == SEMD_INSUFFICIENT_EXTREMA) throw InsufficientExtrema(msg);
    if (rc == SEMD_INVALID_INPUT || rc == SEMD_CAPACITY) throw InvalidInput(msg);
    throw EngineError(msg);
}

inline semd_ctx* ctx() {
    thread_local ThreadContext tc;
    if (!tc.ctx) {
        const char* d = std::getenv("SEMD_DEVICE");
        check(semd_ctx_create(d ? std::atoi(d) : 0, &tc.ctx));
    }
    return tc.ctx;
}

inline semd_sift_cfg sift(const SiftConfig& c) { return semd_sift_cfg{c.sd_threshold, c.max_sift_iters, c.max_imfs}; }
inline semd_ens_cfg ens(const EnsembleConfig& e) { return semd_ens_cfg{e.nstd, e.nr, 0, e.base_seed}; }

inline Decomposition run(int algo, const Signal& x, const SiftConfig& cfg, const EnsembleConfig& en) {
    const semd_sift_cfg c = sift(cfg);
    const semd_ens_cfg e = ens(en);
    std::size_t cap = cfg.max_imfs > 0 ? std::size_t(cfg.max_imfs) : 32;
    for (;;) {
        std::vector<double> imfs(cap * x.size());
        Decomposition d;
        d.residue.resize(x.size());
        std::size_t K = 0;
        const int rc = semd_decompose(ctx(), algo, x.data(), x.size(), &c, &e, imfs.data(), cap, &K,
                                      d.residue.data(), nullptr, nullptr);
        if (rc == SEMD_CAPACITY && K > cap) {
            cap = K;
            continue;
        }
        check(rc);
        for (std::size_t k = 0; k < K; ++k)
            d.imfs.emplace_back(imfs.begin() + k * x.size(), imfs.begin() + (k + 1) * x.size());
        return d;
    }
}

}  // namespace detail

inline Extrema find_extrema(const Signal& x) {
    Extrema e;
    const std::size_t n = x.size();
    e.max_idx.resize(n);
    e.max_val.resize(n);
    e.min_idx.resize(n);
    e.min_val.resize(n);
    std::size_t a = 0, b = 0;
    detail::check(semd_find_extrema(detail::ctx(), x.data(), n, e.max_idx.data(), e.max_val.data(), &a,
                                    e.min_idx.data(), e.min_val.data(), &b));
    e.max_idx.resize(a);
    e.max_val.resize(a);
    e.min_idx.resize(b);
    e.min_val.resize(b);
    return e;
}

inline Signal envelope(const std::vector<std::size_t>& idx, const Signal& val, std::size_t length) {
    if (idx.size() >= 2 && val.size() != idx.size()) throw InvalidInput("envelope: index/value size mismatch");
    Signal out(length);
    detail::check(semd_envelope(detail::ctx(), idx.data(), val.data(), idx.size(), length, out.data()));
    return out;
}

inline SiftResult extract_imf(const Signal& x, const SiftConfig& cfg = {}) {
    const semd_sift_cfg c = detail::sift(cfg);
    SiftResult r;
    r.imf.resize(x.size());
    int32_t count = 0;
    detail::check(semd_extract_imf(detail::ctx(), x.data(), x.size(), &c, r.imf.data(), &count));
    r.sift_count = count;
    return r;
}

inline Decomposition emd(const Signal& x, const SiftConfig& cfg = {}) {
    return detail::run(SEMD_ALGO_EMD, x, cfg, {});
}

inline Signal white_noise(std::size_t n, std::uint64_t seed, double std = 1.0) {
    Signal out(n);
    detail::check(semd_white_noise(detail::ctx(), n, seed, std, out.data()));
    return out;
}

inline std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index) { return semd_derive_seed(base, index); }

inline Signal noise_mode(const Signal& w, std::size_t i, const SiftConfig& cfg = {}) {
    const semd_sift_cfg c = detail::sift(cfg);
    Signal out(w.size());
    detail::check(semd_noise_mode(detail::ctx(), w.data(), w.size(), i, &c, out.data()));
    return out;
}

inline double signal_std(const Signal& x) {
    double v = 0.0;
    detail::check(semd_signal_std(detail::ctx(), x.data(), x.size(), &v));
    return v;
}

inline Decomposition eemd(const Signal& x, const SiftConfig& cfg = {}, const EnsembleConfig& ens = {}) {
    return detail::run(SEMD_ALGO_EEMD, x, cfg, ens);
}

inline Decomposition ceemdan(const Signal& x, const SiftConfig& cfg = {}, const EnsembleConfig& ens = {}) {
    return detail::run(SEMD_ALGO_CEEMDAN, x, cfg, ens);
}

inline Algorithm parse_algorithm(const std::string& name) {
    int a = 0;
    detail::check(semd_parse_algorithm(name.c_str(), &a));
    return static_cast<Algorithm>(a);
}

inline std::string algorithm_name(Algorithm algo) {
    switch (algo) {
        case Algorithm::Emd: return "emd";
        case Algorithm::Eemd: return "eemd";
        case Algorithm::Ceemdan: return "ceemdan";
    }
    throw InvalidInput("unknown algorithm value");
}

inline Decomposition decompose(const Signal& x, Algorithm algo, const SiftConfig& cfg = {},
                               const EnsembleConfig& ens = {}) {
    return detail::run(static_cast<int>(algo), x, cfg, ens);
}

// ---- multi-GPU (B200 extension; the reference is single-process) ----------------------------
// One process or thread per GPU (SEMD_DEVICE selects it). Rank 0 calls comm_unique_id() and
// ships the bytes to the other ranks; every rank then calls comm_init(). From then on eemd,
// ceemdan, decompose and serial_decompose on this thread are collective: each rank passes the
// same input, sifts its shard of the realizations, and NCCL combines the ensemble sums
// (include/semd_b200.h, semd_comm_*). root >= 0 delivers EEMD results to that rank only.
inline std::vector<unsigned char> comm_unique_id() {
    std::vector<unsigned char> id(SEMD_COMM_ID_BYTES);
    detail::check(semd_comm_unique_id(id.data(), id.size()));
    return id;
}

inline void comm_init(const std::vector<unsigned char>& id, int rank, int world, int root = -1) {
    detail::check(semd_comm_init(detail::ctx(), id.data(), id.size(), rank, world));
    detail::check(semd_comm_set_root(detail::ctx(), root));
}

inline void comm_destroy() { detail::check(semd_comm_destroy(detail::ctx())); }

}  // namespace semd

// semd/serialize.hpp -- the reference's serializer API
// (proj/include/semd/serialize.hpp:1-52) with identical signatures and error
// messages, implemented over the B200 C ABI (include/semd_b200.h).
#pragma once

#include <vector>

#include "emd.hpp"
#include "types.hpp"

namespace semd {

inline std::vector<double> transition_weights(std::size_t d) {
    std::vector<double> a(d);
    detail::check(semd_transition_weights(detail::ctx(), d, a.data()));
    return a;
}

inline std::size_t default_transition_length(std::size_t rows) { return semd_default_transition_length(rows); }

inline Signal concatenate(const MultiSignal& x, std::size_t d) {
    const std::size_t m = x.rows(), n = x.channels();
    Signal out(m && n ? m * n + d * (n - 1) : 0);
    detail::check(semd_concatenate(detail::ctx(), x.data().data(), m, n, d, out.data()));
    return out;
}

inline Signal concatenate_naive(const MultiSignal& x, std::size_t d) {
    const std::size_t m = x.rows(), n = x.channels();
    Signal out(m && n ? m * n + d * (n - 1) : 0);
    detail::check(semd_concatenate_naive(detail::ctx(), x.data().data(), m, n, d, out.data()));
    return out;
}

inline ImfTensor deconcatenate(const std::vector<Signal>& modes, std::size_t rows, std::size_t channels,
                               std::size_t d) {
    if (modes.empty()) throw InvalidInput("deconcatenate: no modes given");
    const std::size_t L = modes.front().size();
    std::vector<double> flat;
    flat.reserve(modes.size() * L);
    for (const Signal& m : modes) {
        if (m.size() != L) {  // report the offending length exactly like serialize.cpp:77-81
            const std::size_t expect = rows * channels + d * (channels - 1);
            throw InvalidInput("deconcatenate: mode length " + std::to_string(m.size()) +
                               " does not match M*N + D*(N-1) = " + std::to_string(expect));
        }
        flat.insert(flat.end(), m.begin(), m.end());
    }
    ImfTensor t(rows, channels, modes.size());
    detail::check(semd_deconcatenate(detail::ctx(), flat.data(), modes.size(), L, rows, channels, d,
                                     t.mutable_data().data()));
    return t;
}

inline ImfTensor serial_decompose(const MultiSignal& x, std::size_t d, Algorithm algo, const SiftConfig& cfg = {},
                                  const EnsembleConfig& ens = {}) {
    const semd_sift_cfg c = detail::sift(cfg);
    const semd_ens_cfg e = detail::ens(ens);
    std::size_t cap = cfg.max_imfs > 0 ? std::size_t(cfg.max_imfs) + 1 : 33;
    for (;;) {
        std::vector<double> t(cap * x.rows() * x.channels());
        std::size_t modes = 0;
        const int rc = semd_serial_decompose(detail::ctx(), static_cast<int>(algo), x.data().data(), x.rows(),
                                             x.channels(), d, &c, &e, t.data(), cap, &modes, nullptr);
        if (rc == SEMD_CAPACITY && modes > cap) {
            cap = modes;
            continue;
        }
        detail::check(rc);
        ImfTensor out(x.rows(), x.channels(), modes);
        std::copy(t.begin(), t.begin() + modes * x.rows() * x.channels(), out.mutable_data().begin());
        return out;
    }
}

/// Image adapter (serialize.cpp:107-113): columns become channels.
inline MultiSignal image_to_multisignal(const Image& img) {
    if (img.rows() == 0 || img.cols() == 0) throw InvalidInput("image_to_multisignal: empty image");
    MultiSignal m(img.rows(), img.cols());
    for (std::size_t c = 0; c < img.cols(); ++c)
        for (std::size_t r = 0; r < img.rows(); ++r) m(r, c) = img(r, c);
    return m;
}

/// Inverse adapter (serialize.cpp:115-125): one image per mode.
inline std::vector<Image> imf_tensor_to_images(const ImfTensor& t) {
    std::vector<Image> out;
    for (std::size_t k = 0; k < t.modes(); ++k) {
        Image img(t.rows(), t.channels());
        for (std::size_t c = 0; c < t.channels(); ++c)
            for (std::size_t r = 0; r < t.rows(); ++r) img(r, c) = t(r, c, k);
        out.push_back(std::move(img));
    }
    return out;
}

}  // namespace semd

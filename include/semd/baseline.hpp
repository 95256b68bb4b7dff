// semd/baseline.hpp -- the reference's standard-version comparator
// (proj/include/semd/baseline.hpp, baseline.cpp:5-29) with the identical
// signature, implemented over the B200 C ABI: EMD / EEMD run every channel
// (x every realization) as one batched engine pass.
#pragma once

#include <vector>

#include "emd.hpp"
#include "types.hpp"

namespace semd {

inline ImfTensor slicewise_decompose(const MultiSignal& x, Algorithm algo, const SiftConfig& cfg = {},
                                     const EnsembleConfig& ens = {}) {
    if (x.rows() == 0 || x.channels() == 0) throw InvalidInput("slicewise_decompose: empty input");
    const semd_sift_cfg c = detail::sift(cfg);
    const semd_ens_cfg e = detail::ens(ens);
    std::size_t cap = cfg.max_imfs > 0 ? std::size_t(cfg.max_imfs) + 1 : 33;
    for (;;) {
        std::vector<double> t(cap * x.rows() * x.channels());
        std::size_t modes = 0;
        const int rc = semd_slicewise_decompose(detail::ctx(), static_cast<int>(algo), x.data().data(), x.rows(),
                                                x.channels(), &c, &e, t.data(), cap, &modes);
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

}  // namespace semd

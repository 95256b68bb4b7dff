// semd/recognition.hpp -- the face-recognition feature bank's decomposition side
// (proj/include/semd/recognition.hpp, proj/src/recognition.cpp:18-88, :238-298, synth.cpp:68-96)
// with the reference's signatures, over the B200 library: build_feature_bank decomposes every image
// in ONE batched engine pass (semd_serial_decompose_batch) instead of one serial_decompose per
// image. The classifier side (knn_classify, kfold_cv, knn_cv, heatmap_sweep) is host-only scoring
// outside the decomposition path and is not mirrored (out of scope).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <random>
#include <string>
#include <vector>

#include "emd.hpp"
#include "io.hpp"
#include "serialize.hpp"
#include "types.hpp"

namespace semd {

struct FaceDataset {
    std::vector<Image> images;  // grouped by subject, then image number
    std::vector<int> labels;    // 1-based subject labels, parallel to images
    std::size_t subjects = 0;
    std::size_t per_subject = 0;
};

/// recognition.cpp:18-23
inline std::string face_dataset_root(const std::string& explicit_root = "") {
    if (!explicit_root.empty()) return explicit_root;
    if (const char* env = std::getenv("SERIAL_EMD_DATASET"); env && *env) return env;
    throw DatasetNotFound("dataset not found: no path given and SERIAL_EMD_DATASET is not set");
}

/// recognition.cpp:25-62: root/sN/M.pgm, balanced subjects, equal dimensions.
inline FaceDataset load_face_dataset(const std::string& root) {
    namespace fs = std::filesystem;
    std::error_code ec;
    if (!fs::is_directory(root, ec)) throw DatasetNotFound("dataset not found: '" + root + "' is not a directory");
    FaceDataset ds;
    for (std::size_t s = 1;; ++s) {
        const fs::path dir = fs::path(root) / ("s" + std::to_string(s));
        if (!fs::is_directory(dir, ec)) break;
        std::size_t count = 0;
        for (std::size_t i = 1;; ++i) {
            const fs::path f = dir / (std::to_string(i) + ".pgm");
            if (!fs::is_regular_file(f, ec)) break;
            ds.images.push_back(read_pgm(f.string()));
            ds.labels.push_back(static_cast<int>(s));
            ++count;
        }
        if (count == 0) throw InvalidInput("face dataset: '" + dir.string() + "' contains no 1.pgm");
        if (s == 1) ds.per_subject = count;
        else if (count != ds.per_subject)
            throw InvalidInput("face dataset: unbalanced subject s" + std::to_string(s) + " (" + std::to_string(count) +
                               " images, expected " + std::to_string(ds.per_subject) + ")");
        ds.subjects = s;
    }
    if (ds.subjects == 0) throw DatasetNotFound("dataset not found: '" + root + "' has no s1/ subdirectory");
    for (const Image& img : ds.images)
        if (img.rows() != ds.images.front().rows() || img.cols() != ds.images.front().cols())
            throw InvalidInput("face dataset: images have differing dimensions");
    return ds;
}

/// recognition.cpp:64-75: pad with zero modes at the end, or drop trailing modes.
inline ImfTensor normalize_imf_count(const ImfTensor& t, std::size_t target = 10) {
    if (t.modes() == 0 || target == 0) throw InvalidInput("normalize_imf_count: mode counts must be positive");
    if (t.modes() == target) return t;
    ImfTensor out(t.rows(), t.channels(), target);
    const std::size_t keep = std::min(t.modes(), target), slice = t.rows() * t.channels();
    std::copy(t.data().begin(), t.data().begin() + static_cast<std::ptrdiff_t>(keep * slice), out.mode_channel(0, 0));
    return out;
}

/// recognition.cpp:77-88: elementwise sum of modes first..last, row-major over (row, channel).
inline std::vector<double> sum_imf_range(const ImfTensor& t, std::size_t first, std::size_t last) {
    if (first < 1 || first > last || last > t.modes())
        throw InvalidInput("sum_imf_range: invalid mode range " + std::to_string(first) + ".." + std::to_string(last) +
                           " for K=" + std::to_string(t.modes()));
    std::vector<double> f(t.rows() * t.channels(), 0.0);
    for (std::size_t k = first - 1; k < last; ++k)
        for (std::size_t r = 0; r < t.rows(); ++r)
            for (std::size_t c = 0; c < t.channels(); ++c) f[r * t.channels() + c] += t(r, c, k);
    return f;
}

/// synth.cpp:68-96: multiplicative speckle I + c I U, U ~ uniform[-1, 1] from mt19937_64(seed),
/// c chosen so the realized SNR is snr_db. Host-side image preparation.
inline Image add_speckle(const Image& img, double snr_db, std::uint64_t seed) {
    if (img.rows() == 0 || img.cols() == 0) throw InvalidInput("add_speckle: empty image");
    double ps = 0.0;
    for (double v : img.data()) ps += v * v;
    if (ps == 0.0) throw InvalidInput("add_speckle: all-zero image, SNR undefined");
    if (std::isinf(snr_db) && snr_db > 0) return img;
    std::mt19937_64 eng(seed);
    std::vector<double> noise(img.data().size());
    double pn = 0.0;
    for (std::size_t p = 0; p < noise.size(); ++p) {
        const double u = 2.0 * (static_cast<double>(eng() >> 11) * 0x1.0p-53) - 1.0;
        noise[p] = img.data()[p] * u;
        pn += noise[p] * noise[p];
    }
    if (pn == 0.0) throw InvalidInput("add_speckle: degenerate noise draw");
    const double c = std::sqrt(ps / (std::pow(10.0, snr_db / 10.0) * pn));
    Image out = img;
    for (std::size_t p = 0; p < noise.size(); ++p) out.data()[p] += c * noise[p];
    return out;
}

/// recognition.hpp:73-97 / recognition.cpp:238-278: per-image cumulative mode sums (float storage).
class FaceFeatureBank {
public:
    FaceFeatureBank() = default;
    FaceFeatureBank(std::size_t feature_dim, std::size_t modes) : dim_(feature_dim), modes_(modes) {}
    std::size_t size() const { return cum_.size(); }
    std::size_t feature_dim() const { return dim_; }
    std::size_t modes() const { return modes_; }

    void add(const ImfTensor& t) {
        if (t.rows() * t.channels() != dim_ || t.modes() != modes_)
            throw InvalidInput("FaceFeatureBank: tensor shape does not match the bank");
        std::vector<float> cum(modes_ * dim_, 0.0f);
        std::vector<double> run(dim_, 0.0);
        for (std::size_t k = 0; k < modes_; ++k) {
            for (std::size_t r = 0; r < t.rows(); ++r)
                for (std::size_t c = 0; c < t.channels(); ++c) run[r * t.channels() + c] += t(r, c, k);
            for (std::size_t p = 0; p < dim_; ++p) cum[k * dim_ + p] = static_cast<float>(run[p]);
        }
        cum_.push_back(std::move(cum));
    }

    std::vector<std::vector<double>> features(std::size_t first, std::size_t last) const {
        if (first < 1 || first > last || last > modes_) throw InvalidInput("FaceFeatureBank: invalid mode range");
        std::vector<std::vector<double>> out(cum_.size());
        for (std::size_t i = 0; i < cum_.size(); ++i) {
            const float* hi = cum_[i].data() + (last - 1) * dim_;
            const float* lo = first >= 2 ? cum_[i].data() + (first - 2) * dim_ : nullptr;
            out[i].resize(dim_);
            for (std::size_t p = 0; p < dim_; ++p)
                out[i][p] = static_cast<double>(hi[p]) - (lo ? static_cast<double>(lo[p]) : 0.0);
        }
        return out;
    }

private:
    std::size_t dim_ = 0, modes_ = 0;
    std::vector<std::vector<float>> cum_;
};

/// recognition.cpp:281-298: speckle each image (seed derive_seed(speckle_seed, i)), serial-decompose
/// it (image_to_multisignal, interval d), normalize to target_modes and bank it. All images go
/// through the GPU as one batch; each decomposition equals serial_decompose of that image alone.
inline FaceFeatureBank build_feature_bank(const FaceDataset& ds, Algorithm algo, std::size_t d,
                                          const SiftConfig& cfg, const EnsembleConfig& ens, double speckle_snr_db,
                                          std::uint64_t speckle_seed, std::size_t target_modes = 10) {
    if (ds.images.empty()) throw InvalidInput("build_feature_bank: empty dataset");
    const Image& first = ds.images.front();
    const std::size_t rows = first.rows(), cols = first.cols(), B = ds.images.size(), plane = rows * cols;
    FaceFeatureBank bank(plane, target_modes);
    std::vector<double> x(B * plane);  // B channel-contiguous multi-signals (M = rows, N = cols)
    for (std::size_t i = 0; i < B; ++i) {
        Image img = ds.images[i];
        if (std::isfinite(speckle_snr_db)) img = add_speckle(img, speckle_snr_db, derive_seed(speckle_seed, i));
        const MultiSignal ms = image_to_multisignal(img);
        std::copy(ms.data().begin(), ms.data().end(), x.begin() + static_cast<std::ptrdiff_t>(i * plane));
    }
    const semd_sift_cfg c = detail::sift(cfg);
    const semd_ens_cfg e = detail::ens(ens);
    std::size_t cap = std::max<std::size_t>(target_modes + 1, 16);
    std::vector<std::size_t> modes(B);
    std::vector<double> t;
    for (;;) {
        t.assign(cap * B * plane, 0.0);
        const int rc = semd_serial_decompose_batch(detail::ctx(), static_cast<int>(algo), x.data(), B, rows, cols, d, &c,
                                                   &e, t.data(), cap, modes.data());
        if (rc == SEMD_CAPACITY) {
            std::size_t need = cap;
            for (std::size_t m : modes) need = std::max(need, m);
            if (need > cap) {
                cap = need;
                continue;
            }
        }
        detail::check(rc);
        break;
    }
    for (std::size_t i = 0; i < B; ++i) {
        ImfTensor ti(rows, cols, modes[i]);
        std::copy(t.begin() + static_cast<std::ptrdiff_t>(i * cap * plane),
                  t.begin() + static_cast<std::ptrdiff_t>(i * cap * plane + modes[i] * plane), ti.mode_channel(0, 0));
        bank.add(normalize_imf_count(ti, target_modes));
    }
    return bank;
}

}  // namespace semd

// Harness for tests/test_feature_bank.py: build_feature_bank (include/semd/recognition.hpp, the
// batched-GPU mirror of recognition.cpp:281-298) on images read from a raw file; writes
// bank.features(1, k) for k = 1..target as B x target x (rows*cols) doubles.
//   feature_bank IN OUT B ROWS COLS ALGO D NSTD NR SEED SNR_DB|inf SPECKLE_SEED TARGET
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "semd/recognition.hpp"

int main(int argc, char** argv) {
    if (argc != 14) return 2;
    const std::size_t B = std::strtoull(argv[3], nullptr, 10), rows = std::strtoull(argv[4], nullptr, 10),
                      cols = std::strtoull(argv[5], nullptr, 10);
    const int algo = std::atoi(argv[6]);
    const std::size_t d = std::strtoull(argv[7], nullptr, 10);
    const double nstd = std::strtod(argv[8], nullptr);
    const int nr = std::atoi(argv[9]);
    const std::uint64_t seed = std::strtoull(argv[10], nullptr, 10);
    const double snr = std::string(argv[11]) == "inf" ? INFINITY : std::strtod(argv[11], nullptr);
    const std::uint64_t sseed = std::strtoull(argv[12], nullptr, 10);
    const std::size_t target = std::strtoull(argv[13], nullptr, 10);
    std::vector<double> px(B * rows * cols);
    std::ifstream(argv[1], std::ios::binary).read(reinterpret_cast<char*>(px.data()), px.size() * 8);
    semd::FaceDataset ds;
    for (std::size_t b = 0; b < B; ++b) {
        semd::Image img(rows, cols);
        for (std::size_t p = 0; p < rows * cols; ++p) img.data()[p] = px[b * rows * cols + p];
        ds.images.push_back(img);
        ds.labels.push_back(int(b) + 1);
    }
    const semd::FaceFeatureBank bank = semd::build_feature_bank(ds, static_cast<semd::Algorithm>(algo), d, {},
                                                                {nstd, nr, seed}, snr, sseed, target);
    const std::size_t dim = rows * cols;
    std::vector<double> out(B * target * dim);
    for (std::size_t k = 1; k <= target; ++k) {
        const auto f = bank.features(1, k);
        for (std::size_t b = 0; b < B; ++b)
            for (std::size_t p = 0; p < dim; ++p) out[(b * target + k - 1) * dim + p] = f[b][p];
    }
    std::ofstream(argv[2], std::ios::binary).write(reinterpret_cast<const char*>(out.data()), out.size() * 8);
    std::printf("OK %zu\n", bank.size());
    return 0;
}

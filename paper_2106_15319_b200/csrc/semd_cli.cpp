// semd_cli.cpp -- the reference's `decompose` front-end (proj/src/cli.cpp:93-134) over the B200
// library through the reference-signature C++ mirror (include/semd/*.hpp).
//
//   semd-cli decompose INPUT(.csv|.pgm) [--algo emd|eemd|ceemdan] [--d N|auto] [--nstd X] [--nr N]
//            [--seed N] [--sd-threshold X] [--max-sift-iters N] [--max-imfs N] [--out DIR]
//   semd-cli synth signals [--samples N] [--fs X] [--out DIR]
//
// Same options, defaults, output files and exit codes as the reference (CLI11 is not in this
// image, so a small parser stands in for it): per mode k a CSV <stem>_imf_KK.csv / <stem>_residue.csv
// written with %.17g (plus a rescaled PGM for PGM inputs) and <stem>_decomposition.json, the
// sidecar with M, N, D, K, algorithm, seed, nstd, nr (keys sorted, two-space indent: the layout of
// the reference's nlohmann::json dump(2)). Exit codes: 0 ok, 2 usage / invalid input, 1 internal.
// The remaining reference subcommands (bench, recognize, synth ati/speckle) are outside the hot
// path (out of scope).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "semd/emd.hpp"
#include "semd/io.hpp"
#include "semd/serialize.hpp"

namespace fs = std::filesystem;
using namespace semd;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --d: 'auto' -> round(0.2 M) (serialize.cpp:15-18), else a positive integer (cli.cpp:30-37)
std::size_t resolve_d(const std::string& flag, std::size_t rows) {
    if (flag == "auto") return default_transition_length(rows);
    char* end = nullptr;
    const unsigned long v = std::strtoul(flag.c_str(), &end, 10);
    if (end != flag.c_str() + flag.size() || v == 0)
        throw InvalidInput("--d must be a positive integer or 'auto', got '" + flag + "'");
    return static_cast<std::size_t>(v);
}

std::string lower_ext(const std::string& path) {
    std::string e = fs::path(path).extension().string();
    for (char& c : e) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return e;
}

std::string mode_name(std::size_t k, std::size_t modes) {
    if (k + 1 == modes) return "residue";
    char buf[16];
    std::snprintf(buf, sizeof buf, "imf_%02zu", k + 1);
    return buf;
}

void write_sidecar(const fs::path& path, std::size_t m, std::size_t n, std::size_t d, std::size_t k,
                   Algorithm algo, const EnsembleConfig& ens) {
    std::ofstream out(path);
    if (!out) throw InvalidInput("cannot open file for writing: " + path.string());
    out << "{\n"
        << "  \"D\": " << d << ",\n"
        << "  \"K\": " << k << ",\n"
        << "  \"M\": " << m << ",\n"
        << "  \"N\": " << n << ",\n"
        << "  \"algorithm\": \"" << algorithm_name(algo) << "\",\n"
        << "  \"nr\": " << ens.nr << ",\n"
        << "  \"nstd\": " << io_detail::json_double(ens.nstd) << ",\n"
        << "  \"seed\": " << ens.base_seed << "\n"
        << "}\n";
}

// cli.cpp:93-134
int cmd_decompose(const std::map<std::string, std::string>& o, const std::string& input) {
    auto get = [&](const char* key, const char* def) {
        const auto it = o.find(key);
        return it == o.end() ? std::string(def) : it->second;
    };
    auto num = [&](const char* key, const char* def) {
        const std::string v = get(key, def);
        char* end = nullptr;
        const double x = std::strtod(v.c_str(), &end);
        if (v.empty() || end != v.c_str() + v.size()) throw Usage(std::string("--") + key + ": invalid number '" + v + "'");
        return x;
    };
    auto integer = [&](const char* key, const char* def) {
        const std::string v = get(key, def);
        char* end = nullptr;
        const long long x = std::strtoll(v.c_str(), &end, 10);
        if (v.empty() || end != v.c_str() + v.size()) throw Usage(std::string("--") + key + ": invalid integer '" + v + "'");
        return x;
    };
    const Algorithm algo = parse_algorithm(get("algo", "emd"));
    const SiftConfig cfg{num("sd-threshold", "0.2"), (int)integer("max-sift-iters", "300"), (int)integer("max-imfs", "0")};
    const EnsembleConfig ens{num("nstd", "0.2"), (int)integer("nr", "100"),
                             (std::uint64_t)std::strtoull(get("seed", "0").c_str(), nullptr, 10)};
    const std::string out_dir = get("out", ".");
    fs::create_directories(out_dir);

    const bool is_pgm = lower_ext(input) == ".pgm";
    const std::string stem = fs::path(input).stem().string();
    MultiSignal data;
    std::vector<std::string> header;
    if (is_pgm) {
        data = image_to_multisignal(read_pgm(input));
        for (std::size_t j = 0; j < data.channels(); ++j) header.push_back("c" + std::to_string(j + 1));
    } else {
        CsvData csv = read_csv(input);
        data = std::move(csv.data);
        header = std::move(csv.header);
    }
    const std::size_t d = resolve_d(get("d", "auto"), data.rows());
    const ImfTensor t = serial_decompose(data, d, algo, cfg, ens);

    for (std::size_t k = 0; k < t.modes(); ++k) {
        const std::string name = stem + "_" + mode_name(k, t.modes());
        MultiSignal mode(t.rows(), t.channels());
        for (std::size_t j = 0; j < t.channels(); ++j)
            for (std::size_t i = 0; i < t.rows(); ++i) mode(i, j) = t(i, j, k);
        write_csv((fs::path(out_dir) / (name + ".csv")).string(), mode, header);
        if (is_pgm) {
            Image img(t.rows(), t.channels());
            for (std::size_t c = 0; c < t.channels(); ++c)
                for (std::size_t r = 0; r < t.rows(); ++r) img(r, c) = t(r, c, k);
            write_pgm((fs::path(out_dir) / (name + ".pgm")).string(), img, /*rescale=*/true);
        }
    }
    write_sidecar(fs::path(out_dir) / (stem + "_decomposition.json"), data.rows(), data.channels(), d, t.modes(), algo,
                  ens);
    std::cout << "decomposed " << input << ": M=" << data.rows() << " N=" << data.channels() << " D=" << d
              << " K=" << t.modes() << " algorithm=" << algorithm_name(algo) << " -> " << out_dir << "\n";
    return 0;
}

// cli.cpp:147-158 with synth.cpp:26-45: the pick-up-mask sinusoid mixture, header U..Z
int cmd_synth_signals(const std::map<std::string, std::string>& o) {
    const std::size_t samples = o.count("samples") ? std::strtoull(o.at("samples").c_str(), nullptr, 10) : 1000;
    const double fsr = o.count("fs") ? std::strtod(o.at("fs").c_str(), nullptr) : 1000.0;
    const std::string out_dir = o.count("out") ? o.at("out") : ".";
    if (fsr <= 2.0 * 32.0)
        throw InvalidInput("multivariate_sinusoids: fs must exceed twice the highest tone (aliasing)");
    if (samples < 2) throw InvalidInput("multivariate_sinusoids: need at least 2 samples");
    fs::create_directories(out_dir);
    static const int mask[4][6] = {{1, 1, 0, 1, 0, 0}, {1, 1, 1, 0, 1, 0}, {1, 1, 1, 1, 1, 1}, {1, 0, 1, 1, 0, 1}};
    static const double freqs[4] = {32.0, 16.0, 8.0, 2.0};
    constexpr double two_pi = 6.283185307179586476925286766559;
    MultiSignal data(samples, 6);
    for (std::size_t j = 0; j < 6; ++j)
        for (int i = 0; i < 4; ++i) {
            if (!mask[i][j]) continue;
            for (std::size_t t = 0; t < samples; ++t) data(t, j) += std::sin(two_pi * freqs[i] * double(t) / fsr);
        }
    const fs::path path = fs::path(out_dir) / "signals.csv";
    write_csv(path.string(), data, {"U", "V", "W", "X", "Y", "Z"});
    std::cout << "wrote " << path.string() << " (" << data.rows() << "x" << data.channels() << ")\n";
    return 0;
}

const char* kUsage =
    "serial-EMD (B200): 1D EMD/EEMD/CEEMDAN with multi-signal serialization\n"
    "Usage: semd-cli decompose INPUT [--algo A] [--d N|auto] [--nstd X] [--nr N] [--seed N]\n"
    "                 [--sd-threshold X] [--max-sift-iters N] [--max-imfs N] [--out DIR]\n"
    "       semd-cli synth signals [--samples N] [--fs X] [--out DIR]\n";

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    try {
        for (int i = 1; i < argc; ++i) {
            std::string a = argv[i];
            if (a == "-h" || a == "--help") {
                std::cout << kUsage;
                return 0;
            }
            if (a.rfind("--", 0) == 0) {
                std::string key = a.substr(2), val;
                const std::size_t eq = key.find('=');
                if (eq != std::string::npos) {
                    val = key.substr(eq + 1);
                    key = key.substr(0, eq);
                } else {
                    if (i + 1 >= argc) throw Usage("--" + key + " requires an argument");
                    val = argv[++i];
                }
                opt[key] = val;
            } else {
                pos.push_back(a);
            }
        }
        if (pos.empty()) throw Usage("a subcommand is required");
        static const char* dec_keys[] = {"algo", "d", "nstd", "nr", "seed", "sd-threshold", "max-sift-iters",
                                         "max-imfs", "out"};
        static const char* sig_keys[] = {"samples", "fs", "out"};
        auto check_keys = [&](const char* const* keys, std::size_t nk) {
            for (const auto& kv : opt) {
                bool ok = false;
                for (std::size_t q = 0; q < nk; ++q) ok = ok || kv.first == keys[q];
                if (!ok) throw Usage("unknown option --" + kv.first);
            }
        };
        if (pos[0] == "decompose") {
            if (pos.size() != 2) throw Usage("decompose: exactly one input file is required");
            check_keys(dec_keys, sizeof dec_keys / sizeof *dec_keys);
            return cmd_decompose(opt, pos[1]);
        }
        if (pos[0] == "synth" && pos.size() == 2 && pos[1] == "signals") {
            check_keys(sig_keys, sizeof sig_keys / sizeof *sig_keys);
            return cmd_synth_signals(opt);
        }
        throw Usage("unknown subcommand '" + pos[0] + "'");
    } catch (const Usage& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 2;
    } catch (const InvalidInput& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "internal error: " << e.what() << "\n";
        return 1;
    }
}

// C++ drop-in check: the reference's own unit-test idioms (proj/tests/test_emd.cpp,
// test_serialize.cpp) against the B200 library through include/semd/*.hpp.
// Prints "OK <n>" and exits 0 when every check passes.
#include <cmath>
#include <cstdio>
#include <string>

#include "semd/baseline.hpp"
#include "semd/emd.hpp"
#include "semd/serialize.hpp"

using namespace semd;

static int fails = 0, checks = 0;
#define CHECK(c)                                                         \
    do {                                                                 \
        ++checks;                                                        \
        if (!(c)) {                                                      \
            ++fails;                                                     \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
        }                                                                \
    } while (0)

template <class E, class F>
static bool throws_with(F f, const std::string& msg) {
    try {
        f();
    } catch (const E& e) {
        return msg.empty() || msg == e.what();
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    {  // test_emd.cpp:13-21
        const Extrema e = find_extrema({0.0, 1.0, 0.0, -1.0, 0.0});
        CHECK(e.max_idx.size() == 1 && e.max_idx[0] == 1 && e.max_val[0] == 1.0);
        CHECK(e.min_idx.size() == 1 && e.min_idx[0] == 3 && e.min_val[0] == -1.0);
    }
    {  // plateaus :38-53
        CHECK(find_extrema({0.0, 1.0, 1.0, 0.0}).max_idx.at(0) == 1);
        CHECK(find_extrema({0.0, 2.0, 2.0, 2.0, 0.0}).max_idx.at(0) == 2);
        CHECK(find_extrema({0.0, 1.0, 1.0, 2.0, 0.0}).max_idx.at(0) == 3);
    }
    CHECK(throws_with<InvalidInput>([] { find_extrema({1.0, 2.0}); },
                                    "find_extrema: signal too short (need at least 3 samples)"));
    CHECK(throws_with<InsufficientExtrema>([] { envelope({4}, {1.0}, 10); },
                                           "envelope: need at least 2 extrema, got 1"));
    {  // collinear anchored knots give the exact line :90-97
        const Signal env = envelope({0, 5, 10}, {0.0, 5.0, 10.0}, 11);
        for (std::size_t t = 0; t < env.size(); ++t) CHECK(std::abs(env[t] - double(t)) <= 1e-12);
    }
    {  // reconstruction and ramp
        Signal x(600);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.05 * i) + 0.3 * std::sin(0.7 * i) + 1e-3 * i;
        const Decomposition d = emd(x);
        double err = 0.0;
        for (std::size_t i = 0; i < x.size(); ++i) {
            double s = d.residue[i];
            for (const Signal& imf : d.imfs) s += imf[i];
            err = std::max(err, std::abs(s - x[i]));
        }
        CHECK(err <= 1e-8);
        Signal ramp(64);
        for (std::size_t i = 0; i < ramp.size(); ++i) ramp[i] = 0.25 * i;
        const Decomposition r = emd(ramp);
        CHECK(r.imfs.empty() && r.residue == ramp);
    }
    CHECK(throws_with<InvalidInput>([] { emd({1.0, 2.0, 1.0}); }, "emd: signal too short (need at least 4 samples)"));
    {  // ensembles: nstd = 0 degenerates to emd exactly
        Signal x(300);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.3 * i) * std::cos(0.011 * i);
        const Decomposition a = emd(x);
        const Decomposition b = eemd(x, {}, {0.0, 3, 0});
        CHECK(a.imfs == b.imfs && a.residue == b.residue);
        const Decomposition c = ceemdan(x, {}, {0.2, 4, 1});
        const Decomposition c2 = ceemdan(x, {}, {0.2, 4, 1});
        CHECK(c.imfs == c2.imfs && !c.imfs.empty());
    }
    CHECK(throws_with<InvalidInput>([] { eemd({1.0, 2.0, 3.0, 4.0, 5.0}, {}, {0.2, 0, 0}); },
                                    "ensemble: nr must be at least 1"));
    CHECK(parse_algorithm("EEMDAN") == Algorithm::Ceemdan);
    CHECK(throws_with<InvalidInput>([] { parse_algorithm("vmd"); },
                                    "unknown algorithm 'vmd' (expected emd, eemd, or ceemdan)"));
    {  // serializer (test_serialize.cpp)
        CHECK(transition_weights(4) == (std::vector<double>{0.2, 0.4, 0.6, 0.8}));
        CHECK(default_transition_length(1000) == 200 && default_transition_length(2) == 1);
        const MultiSignal x = MultiSignal::from_channels({{0.0, 3.0}, {6.0, 9.0}});
        const Signal s = concatenate(x, 2);
        CHECK(s == (Signal{0.0, 3.0, 5.0, 4.0, 6.0, 9.0}));
        CHECK(s == concatenate_naive(x, 2));
        const MultiSignal y = MultiSignal::from_channels({Signal(10, 1.0), Signal(10, 2.0)});
        CHECK(throws_with<InvalidInput>([&] { concatenate(y, 11); }, "concatenate: transition longer than channel"));
        const ImfTensor t = deconcatenate({concatenate(y, 3)}, 10, 2, 3);
        CHECK(t(4, 1, 0) == 2.0 && t(9, 0, 0) == 1.0);
        CHECK(throws_with<InvalidInput>([] { deconcatenate({Signal(11, 0.0)}, 10, 1, 2); },
                                        "deconcatenate: mode length 11 does not match M*N + D*(N-1) = 10"));
        MultiSignal z(200, 3);
        for (std::size_t j = 0; j < 3; ++j)
            for (std::size_t i = 0; i < 200; ++i) z(i, j) = std::sin(0.2 * (j + 1) * i) + 0.1 * j;
        const ImfTensor st = serial_decompose(z, 40, Algorithm::Emd);
        double err = 0.0;
        for (std::size_t j = 0; j < 3; ++j)
            for (std::size_t i = 0; i < 200; ++i) {
                double sum = 0.0;
                for (std::size_t k = 0; k < st.modes(); ++k) sum += st(i, j, k);
                err = std::max(err, std::abs(sum - z(i, j)));
            }
        CHECK(err <= 1e-8);
        // baseline.cpp:5-29: per-channel decompositions, residue last (test_baseline idioms)
        const ImfTensor sw = slicewise_decompose(z, Algorithm::Emd);
        const Decomposition d1 = emd(z.channel(1));
        CHECK(sw.modes() >= d1.imfs.size() + 1);
        bool same = true;
        for (std::size_t i = 0; i < 200; ++i) {
            if (!d1.imfs.empty() && sw(i, 1, 0) != d1.imfs[0][i]) same = false;
            if (sw(i, 1, sw.modes() - 1) != d1.residue[i]) same = false;
        }
        CHECK(same);
        CHECK(throws_with<InvalidInput>([] { slicewise_decompose(MultiSignal(), Algorithm::Emd); },
                                        "slicewise_decompose: empty input"));
    }
    {  // multi-GPU API on a 1-rank NCCL communicator: bit-identical to the single-GPU engine
        Signal x(900);
        for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.21 * i) + 0.4 * std::cos(0.047 * i);
        const Decomposition e1 = eemd(x, {}, {0.2, 7, 3});
        const Decomposition c1 = ceemdan(x, {}, {0.2, 5, 2});
        comm_init(comm_unique_id(), 0, 1);
        const Decomposition e2 = eemd(x, {}, {0.2, 7, 3});
        const Decomposition c2 = ceemdan(x, {}, {0.2, 5, 2});
        CHECK(e1.imfs == e2.imfs && e1.residue == e2.residue);
        CHECK(c1.imfs == c2.imfs && c1.residue == c2.residue);
        comm_destroy();
    }
    std::printf("%s %d/%d\n", fails ? "FAILED" : "OK", checks - fails, checks);
    return fails ? 1 : 0;
}

// Facade-level checks of verify_theory / write_theory_csv (bench.hpp:84-99),
// written against the adsann facade the reference's callers compile with:
// the properties the reference's bench tests state for the study (an
// unreachable threshold never fails and scans all dims; reliability and
// sampled dims grow with epsilon0; the CSV header), on the B200 engine.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <filesystem>
#include <fstream>
#include <string>

#include "adsann/bench.hpp"

using namespace adsann;

namespace {

struct Study {
    Dataset t, qt;
};

Study make_study(std::int32_t n, std::int32_t d, std::int32_t blobs, std::int32_t nq, std::uint64_t seed) {
    const Dataset all = synth_dataset(n + nq, d, blobs, 1.0, seed);
    Dataset raw, q;
    raw.n = n;
    raw.d = d;
    raw.data.assign(all.data.begin(), all.data.begin() + std::size_t(n) * d);
    q.n = nq;
    q.d = d;
    q.data.assign(all.data.begin() + std::size_t(n) * d, all.data.end());
    const TransformMatrix m = generate_orthogonal(d, seed + 1);
    return Study{apply_dataset(m, raw), apply_dataset(m, q)};
}

}  // namespace

TEST_CASE("verify_theory: an unreachable threshold scans every dimension and never fails") {
    const Study s = make_study(1000, 48, 8, 20, 513);
    const auto rows = verify_theory(s.t, s.qt, 20, {1e6});
    REQUIRE(rows.size() == 1);
    CHECK(rows[0].failures == 0);
    CHECK(rows[0].avg_dims == doctest::Approx(48.0));
    CHECK(rows[0].positives >= 20u * 20u);
}

TEST_CASE("verify_theory: failure rate falls and sampled dims grow with epsilon0") {
    const Study s = make_study(4000, 64, 16, 60, 515);
    const std::vector<double> grid = {3.0, 0.5, 2.0, 1.0, 2.5, 1.5};  // sorted by the call
    const auto rows = verify_theory(s.t, s.qt, 50, grid);
    REQUIRE(rows.size() == grid.size());
    CHECK(rows[0].epsilon0 == 0.5);
    CHECK(rows[0].failure_rate > 0.0);
    for (std::size_t i = 1; i < rows.size(); ++i) {
        CHECK(rows[i].epsilon0 > rows[i - 1].epsilon0);
        CHECK(rows[i].failure_rate <= rows[i - 1].failure_rate);
        CHECK(rows[i].avg_dims >= rows[i - 1].avg_dims);
        CHECK(rows[i].positives == rows[0].positives);
    }
    const auto path = std::filesystem::temp_directory_path() / "adsann_theory_facade.csv";
    write_theory_csv(rows, path);
    std::ifstream in(path);
    std::string header, first;
    std::getline(in, header);
    std::getline(in, first);
    CHECK(header == "epsilon0,failure_rate,avg_dims,failures,positives");
    CHECK(first.rfind("0.500,", 0) == 0);
}

TEST_CASE("verify_theory: argument errors are std::invalid_argument") {
    const Study s = make_study(200, 16, 4, 3, 7);
    CHECK_THROWS_AS(verify_theory(s.t, s.qt, 0, {2.1}), std::invalid_argument);
    CHECK_THROWS_AS(verify_theory(s.t, s.qt, 201, {2.1}), std::invalid_argument);
    Dataset wrong = s.qt;
    wrong.d = 8;
    CHECK_THROWS_AS(verify_theory(s.t, wrong, 5, {2.1}), std::invalid_argument);
}

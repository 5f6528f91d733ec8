// Drives the header-only C++ mirror (include/abmx_cuda.hpp) the way a reference user would:
// PredationModel / TrafficModel / FinanceModel step + collect_metrics, and the run_batch
// helpers. Prints every metrics row; tests/test_cpp_mirror_gpu.py compares with the oracle.
#include <cstdio>
#include <vector>

#include "abmx_cuda.hpp"

int main() {
    using namespace abmx::cuda;
    const auto seeds = replica_seeds(7, 1);
    {
        abmx_predation_config c = default_predation_config();
        c.sheep_capacity = 1024;
        c.wolf_capacity = 1024;
        PredationModel m(c, seeds[0]);
        std::vector<std::vector<double>> rows;
        for (std::int64_t t = 1; t <= 20; ++t) {
            m.step(t);
            m.collect_metrics(rows);
        }
        for (const auto& r : rows) std::printf("P %.17g %.17g %.17g %.17g\n", r[0], r[1], r[2], r[3]);
    }
    {
        abmx_traffic_config c = default_traffic_config();
        c.length = 30;
        TrafficModel m(c, seeds[0]);
        std::vector<std::vector<double>> rows;
        for (std::int64_t t = 1; t <= 40; ++t) {
            m.step(t);
            m.collect_metrics(rows);
        }
        for (const auto& r : rows) std::printf("T %.17g %.17g %.17g %.17g\n", r[0], r[1], r[2], r[3]);
        std::printf("TT %lld %lld\n", static_cast<long long>(m.spawned_total()), static_cast<long long>(m.exited_total()));
    }
    {
        abmx_finance_config c = default_finance_config();
        c.book_capacity = 64;
        FinanceModel m(c, seeds[0]);
        std::vector<std::vector<double>> rows;
        for (std::int64_t t = 1; t <= 10; ++t) {
            m.step(t);
            m.collect_metrics(rows);
        }
        for (const auto& r : rows)
            std::printf("F %.17g %.17g %.17g %.17g %.17g %.17g\n", r[0], r[1], r[2], r[3], r[4], r[5]);
    }
    try {
        abmx_traffic_config bad{0, 10, 0.5};
        TrafficModel m(bad, 1);
        std::printf("E none\n");
    } catch (const DomainError&) {
        std::printf("E DomainError\n");
    }
    return 0;
}

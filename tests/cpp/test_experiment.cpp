// test_experiment.cpp -- the reference's UNMODIFIED experiment harness
// (/root/reference/proj/include/xqr/experiment.hpp, the hot path's caller,
// SURVEY.md §8b) compiled against the drop-in headers (include/xqr: every
// other xqr header resolves there), so its mgs_qr / residual_max_entry /
// par_mgs_qr calls run on the B200 and its own R arithmetic runs on the
// drop-in value types.  Built by __graft_entry__.build() where the reference
// tree exists; run by tests/test_dropin_gpu.py.
//   test_experiment accuracy <cd|cdd|cqd> m n trials seed g...  -> accuracy_csv
//   test_experiment overhead m n reps                           -> bench_csv
#include <cstdio>
#include <cstdlib>
#include <string>

#include "xqr/experiment.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argv[1];
    try {
        if (mode == "accuracy" && argc >= 8) {
            xqr::accuracy_config cfg;
            cfg.precision = xqr::parse_precision(argv[2]);
            cfg.m = std::strtoull(argv[3], nullptr, 10);
            cfg.n = std::strtoull(argv[4], nullptr, 10);
            cfg.trials = std::strtoull(argv[5], nullptr, 10);
            cfg.seed = std::strtoull(argv[6], nullptr, 10);
            cfg.g_values.clear();
            for (int i = 7; i < argc; ++i) cfg.g_values.push_back(std::strtod(argv[i], nullptr));
            std::fputs(xqr::accuracy_csv(xqr::run_accuracy_sweep(cfg)).c_str(), stdout);
            return 0;
        }
        if (mode == "overhead" && argc >= 5) {
            xqr::overhead_config cfg;
            cfg.m = std::strtoull(argv[2], nullptr, 10);
            cfg.n = std::strtoull(argv[3], nullptr, 10);
            cfg.repetitions = std::strtoull(argv[4], nullptr, 10);
            std::fputs(xqr::bench_csv(xqr::run_overhead_bench(cfg)).c_str(), stdout);
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 4;
    }
    return 2;
}

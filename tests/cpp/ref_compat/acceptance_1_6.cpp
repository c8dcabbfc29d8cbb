// TEST INFRASTRUCTURE ONLY.  Runs acceptance criteria 1-6 of the reference's
// own acceptance suite (/root/reference/proj/tests/acceptance.cpp:64-365,
// compiled IN PLACE -- its path comes from the build recipe, the file is never
// copied) against THIS repo's include/ and libpf_b200.so:
//   1 schedule/formula agreement      4 utilization improvement, period identity
//   2 utilization values              5 analytic-model monotonicity, speedup bounds
//   3 bubble-fill soundness           6 step-time and training-time calculators
// Criteria 7-9 exercise the FP64 toy trainer and the trace IO, which this
// repo does not ship; the reference's main() is renamed to an
// unused static function so they are compiled but never referenced.
#include "pipefill/kfac/kfac.hpp"
#ifndef PF_WITH_REF_HEADERS  // the reference's own kfac.hpp declares the toy API itself
#include "toy_decls.hpp"
#endif

#define main static pfref_acceptance_main_unused
#include PF_REF_ACCEPTANCE
#undef main

int main() {
    const std::vector<Criterion> criteria = {
        {1, "schedule/formula agreement", 1.0, criterion_schedule_formula},
        {2, "utilization values", 1.0, criterion_utilization_values},
        {3, "bubble-fill soundness", 30.0, criterion_bubble_fill_soundness},
        {4, "utilization improvement and period identity", 30.0, criterion_utilization_improvement},
        {5, "analytic-model monotonicity and speedup bounds", 10.0, criterion_monotonicity},
        {6, "step-time and training-time calculators", 1.0, criterion_time_calculators},
    };
    int failed = 0;
    for (const auto& c : criteria) {
        Checker check;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            c.fn(check);
        } catch (const std::exception& e) {
            check.failures.push_back(std::string("exception: ") + e.what());
        }
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (dt > c.budget_s) check.failures.push_back("runtime budget exceeded");
        const bool ok = check.failures.empty();
        failed += ok ? 0 : 1;
        std::printf("[%s] criterion %d: %s (%.2fs)\n", ok ? "PASS" : "FAIL", c.id, c.name, dt);
        for (std::size_t i = 0; i < check.failures.size() && i < 8; ++i)
            std::printf("       - %s\n", check.failures[i].c_str());
    }
    return failed == 0 ? 0 : 1;
}

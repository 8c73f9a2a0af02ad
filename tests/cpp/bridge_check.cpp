// Compiles the drop-in bridge (include/migplan_b200_procedures.hpp) against the reference's
// own headers and, when a GPU is present, checks GPU fast_algo / crossover against the
// reference's on the slos_day-like workload.  Built by tests/test_bridge.py.
#include <cstdio>

#include "migplan/ga.hpp"
#include "migplan_b200_procedures.hpp"

using namespace migplan;

int main(int argc, char** argv) {
    ProfileStore ps;
    ModelProfile cnn;
    cnn.model_name = "cnn-a";
    cnn.entries[1] = {{1, 30, 25}, {4, 45, 45}, {8, 50, 70}, {16, 52, 130}};
    cnn.entries[2] = {{1, 34, 22}, {4, 60, 38}, {8, 80, 60}, {16, 85, 120}};
    cnn.entries[3] = {{1, 36, 20}, {4, 70, 33}, {8, 105, 52}, {16, 112, 105}};
    cnn.entries[4] = {{1, 38, 18}, {4, 80, 30}, {8, 120, 48}, {16, 130, 110}};
    cnn.entries[7] = {{1, 40, 15}, {4, 90, 25}, {8, 140, 40}, {16, 155, 120}, {32, 165, 200}};
    ps["cnn-a"] = cnn;
    std::vector<ServiceSpec> svcs{{"a", "cnn-a", 700.0, 100.0}, {"b", "cnn-a", 450.0, 100.0}, {"c", "cnn-a", 1300.0, 100.0}};
    validate_services(svcs, ps);
    PlanContext ctx = make_plan_context(svcs, ps, PartitionRuleSet::defaults());
    if (argc > 1 && std::string(argv[1]) == "--compile-only") return 0;
    b200::GpuContext g(ctx);
    auto ref = fast_algo(zero_completion(3), ctx);
    auto gpu = g.fast_algo(zero_completion(3));
    if (ref != gpu) {
        std::printf("fast_algo mismatch\n");
        return 1;
    }
    Chromosome parent = evaluate_chromosome(ref, ctx);
    GaParams gp;
    gp.slow.budget_iters = 24;
    Rng r1(7), r2(7);
    MctsProcedure slow_ref(gp.slow);
    b200::GpuMctsProcedure slow_gpu(g, gp.slow);
    Chromosome a = crossover(mutate(parent, gp, r1), slow_ref, ctx, gp, r1);
    Chromosome b = crossover(mutate(parent, gp, r2), slow_gpu, ctx, gp, r2);
    if (a.gpus != b.gpus) {
        std::printf("crossover mismatch\n");
        return 1;
    }
    std::printf("bridge ok: %zu GPUs\n", gpu.size());
    return 0;
}

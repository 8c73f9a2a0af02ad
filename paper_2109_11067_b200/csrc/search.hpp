// search.hpp — host drivers of the slow algorithms (MCTS, GA) over the device engine.
//
// "Parity mode": the control flow, RNG consumption (std::mt19937_64, util.hpp:27-51)
// and floating-point expressions restate mcts.hpp / ga.hpp one for one, so that under a
// matched seed the plans are identical to the reference's; every scoring pass (greedy
// fast_algo, top-K) runs on the B200 through Engine.
#pragma once

#include <cmath>
#include <functional>
#include <memory>
#include <random>
#include <unordered_map>
#include <vector>

#include "engine.hpp"

namespace mgb {

using Rng = std::mt19937_64;

inline uint64_t mix_seed(uint64_t a, uint64_t b) {  // util.hpp:30-35
    uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline size_t pick_index(Rng& rng, size_t n) {  // util.hpp:39-47
    if (n <= 1) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t r;
    do {
        r = rng();
    } while (r >= limit);
    return static_cast<size_t>(r % n);
}

inline bool satisfied(const std::vector<double>& c) {  // core.hpp:217-221
    for (double v : c)
        if (v < 1.0 - kSatisfyEps) return false;
    return true;
}

struct MctsParams {  // mcts.hpp:13-18
    int budget_iters = 200;
    int topk = 10;
    int pick_services = 5;
    double ucb_c = 1.4142135623730951;
};

struct GaParams {  // ga.hpp:24-36
    int population = 16;
    double erase_fraction = 0.10;
    int mutation_pairs = 2;
    int stall_rounds = 10;
    double time_budget_s = 0.0;
    uint64_t seed = 0;
    int max_rounds = 1 << 30;
    int workers = 1;
    MctsParams slow{48, 10, 5, 1.4142135623730951};
};

struct RolloutCache {  // mcts.hpp:47-50, keyed by the unsatisfied-service bitmap
    struct Hash {
        size_t operator()(const std::vector<uint64_t>& v) const {
            uint64_t h = 1469598103934665603ULL;
            for (uint64_t w : v) h = (h ^ w) * 1099511628211ULL;
            return static_cast<size_t>(h);
        }
    };
    std::unordered_map<std::vector<uint64_t>, std::vector<long long>, Hash> pools;
    int builds = 0;
};

// The searches take the candidate pool through this interface (Engine on the device).
std::vector<Config> fast_plan(Engine& e, const std::vector<double>& comp);
void add_util(const Engine& e, long long idx, std::vector<double>& comp);

std::vector<long long> expand_children(Engine& e, const std::vector<double>& comp, const MctsParams& p, Rng& rng);
int rollout(Engine& e, const std::vector<double>& comp, const MctsParams& p, RolloutCache& cache, Rng& rng,
            int max_depth, std::vector<long long>* picked);
std::vector<Config> mcts_solve(Engine& e, const std::vector<double>& comp, const MctsParams& p, uint64_t seed,
                               const std::function<void(int, int, int, int)>& trace);

struct Chromosome {  // ga.hpp:13-17
    std::vector<Config> gpus;
    int gpu_count = 0;
    double slack = 0.0;
};
struct Procedure {  // OptimizerProcedure, greedy.hpp:155-158
    virtual ~Procedure() = default;
    virtual std::vector<Config> solve(const std::vector<double>& comp, Engine& e, Rng& rng) const = 0;
};
struct FastProc final : Procedure {  // greedy.hpp:160-164
    std::vector<Config> solve(const std::vector<double>& comp, Engine& e, Rng&) const override {
        return fast_plan(e, comp);
    }
};
struct MctsProc final : Procedure {  // mcts.hpp:254-260
    MctsParams params;
    explicit MctsProc(MctsParams p) : params(p) {}
    std::vector<Config> solve(const std::vector<double>& comp, Engine& e, Rng& rng) const override {
        return mcts_solve(e, comp, params, rng(), nullptr);
    }
};

Chromosome evaluate_chromosome(std::vector<Config> gpus, const Engine& e);
Chromosome mutate(const Chromosome& parent, const GaParams& p, Rng& rng);
Chromosome crossover(const Chromosome& parent, const Procedure& slow, Engine& e, const GaParams& p, Rng& rng);
// Throughput mode: device population generations with Philox draws (ga.cu).
std::vector<Config> two_phase_parallel(Engine& e, const GaParams& p,
                                       const std::function<void(int, int, double, bool, double)>& log,
                                       const RolloutRefill* slow = nullptr);
std::vector<Config> two_phase(Engine& e, const GaParams& p,
                              const std::function<void(int, int, double, bool, double)>& log);
std::vector<Config> sorted_deployment(std::vector<Config> cfgs);

}  // namespace mgb

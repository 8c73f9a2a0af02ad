// search.cpp — MCTS (mcts.hpp) and GA (ga.hpp) drivers; see search.hpp.
#include "search.hpp"

#include <algorithm>
#include <chrono>
#include <exception>
#include <map>
#include <thread>
#include <cstdio>
#include <cstdlib>

namespace mgb {

std::vector<Config> fast_plan(Engine& e, const std::vector<double>& comp) {
    std::vector<uint64_t> rows;
    std::vector<double> scores;
    e.fast_algo(comp, rows, scores);
    std::vector<Config> out;
    out.reserve(rows.size());
    for (uint64_t r : rows) out.push_back(e.config_of(r));
    return out;
}

void add_util(const Engine& e, long long idx, std::vector<double>& comp) {
    const Model& m = e.model();
    int svc[kRowK], pat[kRowK];
    int k = m.members(e.base_rows()[idx], svc, pat);
    for (int j = 0; j < k; ++j) comp[svc[j]] = comp[svc[j]] + m.U[static_cast<size_t>(svc[j]) * m.PP + pat[j]];
}

namespace {

std::vector<int> unsatisfied(const std::vector<double>& c) {  // mcts.hpp:78-83
    std::vector<int> u;
    for (size_t i = 0; i < c.size(); ++i)
        if (c[i] < 1.0 - kSatisfyEps) u.push_back(static_cast<int>(i));
    return u;
}

std::vector<uint64_t> type_key(const std::vector<double>& c) {  // completion_type_key, mcts.hpp:38-43
    std::vector<uint64_t> k((c.size() + 63) / 64, 0);
    for (size_t i = 0; i < c.size(); ++i)
        if (c[i] < 1.0 - kSatisfyEps) k[i >> 6] |= 1ull << (i & 63);
    return k;
}

struct Node {  // SearchNode, mcts.hpp:22-35
    std::vector<double> comp;
    bool leaf = false;
    bool expanded = false;
    int visits = 0;
    double value_sum = 0.0;
    struct Edge {
        long long cand = -1;
        std::unique_ptr<Node> node;
    };
    std::vector<Edge> children;
    explicit Node(std::vector<double> c) : comp(std::move(c)) { leaf = satisfied(comp); }
};

void expand(Engine& e, Node& node, const MctsParams& p, Rng& rng) {
    std::vector<long long> top = expand_children(e, node.comp, p, rng);
    node.children.clear();
    for (long long idx : top) {
        std::vector<double> child = node.comp;
        add_util(e, idx, child);
        node.children.push_back(Node::Edge{idx, std::make_unique<Node>(std::move(child))});
    }
    node.expanded = true;
}

}  // namespace

// expand, mcts.hpp:89-116: partial Fisher-Yates sample of min(5, |unsat|) unsatisfied
// services; children = top-K over the base rows touching any sampled service.
std::vector<long long> expand_children(Engine& e, const std::vector<double>& comp, const MctsParams& p, Rng& rng) {
    if (satisfied(comp)) throw PlanningError("expand: node is already satisfied");
    std::vector<int> unsat = unsatisfied(comp);
    size_t take = std::min<size_t>(static_cast<size_t>(std::max(p.pick_services, 0)), unsat.size());
    for (size_t i = 0; i < take; ++i) {
        size_t j = i + pick_index(rng, unsat.size() - i);
        std::swap(unsat[i], unsat[j]);
    }
    std::vector<uint64_t> mask(4, 0);
    for (size_t i = 0; i < take; ++i) mask[unsat[i] >> 6] |= 1ull << (unsat[i] & 63);
    if (take == 0) return {};
    return e.topk(comp, p.topk, nullptr, &mask);
}

// rollout, mcts.hpp:122-143.
int rollout(Engine& e, const std::vector<double>& comp, const MctsParams& p, RolloutCache& cache, Rng& rng,
            int max_depth, std::vector<long long>* picked) {
    std::vector<double> cur = comp;
    int steps = 0;
    while (!satisfied(cur)) {
        if (steps >= max_depth) return max_depth;
        auto key = type_key(cur);
        auto it = cache.pools.find(key);
        if (it == cache.pools.end()) {
            ++cache.builds;
            it = cache.pools.emplace(std::move(key), e.topk(cur, p.topk, nullptr, nullptr)).first;
        }
        const std::vector<long long>& pool = it->second;
        if (pool.empty()) throw PlanningError("rollout: no candidate config serves the remaining demand");
        long long idx = pool[pick_index(rng, pool.size())];
        add_util(e, idx, cur);
        if (picked) picked->push_back(idx);
        ++steps;
    }
    return steps;
}

// mcts_solve, mcts.hpp:148-252: fast_ref and the descent completion on the greedy kernel, the
// search loop itself device-resident (mcts.cu: one CTA, the reference's mt19937_64 stream on
// the device).  The device top-K holds k <= 32 candidates: larger k is rejected (ArgumentError)
// rather than run on a host loop.
std::vector<Config> mcts_solve(Engine& e, const std::vector<double>& comp, const MctsParams& p, uint64_t seed,
                               const std::function<void(int, int, int, int)>& trace) {
    if (satisfied(comp)) return {};
    std::vector<Config> fast_ref = fast_plan(e, comp);
    if (p.budget_iters <= 0) return fast_ref;
    if (p.topk < 1 || p.topk > 32) throw ArgumentError("mcts_solve: topk must be in [1, 32] (device top-K)");
    const int l_ref = static_cast<int>(fast_ref.size());
    MctsDeviceResult r = e.mcts_device(comp, p.budget_iters, p.topk, p.pick_services, p.ucb_c, seed, l_ref);
    if (trace)
        for (int i = 0; i < r.iterations; ++i)
            trace(r.trace[4 * i], r.trace[4 * i + 1], r.trace[4 * i + 2], r.trace[4 * i + 3]);
    if (r.status == 1) throw PlanningError("rollout: no candidate config serves the remaining demand");
    if (r.status != 0) throw DeviceError("mcts: device search storage exhausted");
    std::vector<Config> via_descent;
    for (long long idx : r.descent) via_descent.push_back(e.config_of(e.base_rows()[idx]));
    if (!r.descent_leaf)
        for (auto& c : fast_plan(e, r.descent_comp)) via_descent.push_back(c);
    std::vector<Config> answer = std::move(fast_ref);
    if (via_descent.size() < answer.size()) answer = std::move(via_descent);
    if (r.best_len >= 0 && static_cast<size_t>(r.best_len) < answer.size()) {
        answer.clear();
        for (long long idx : r.best) answer.push_back(e.config_of(e.base_rows()[idx]));
    }
    return answer;
}

namespace {
double slack_of(const std::vector<double>& c) {  // core.hpp:232-236
    double s = 0.0;
    for (double v : c) s += std::max(0.0, v - 1.0);
    return s;
}
bool fitter(const Chromosome& a, const Chromosome& b) {  // ga.hpp:19-22
    if (a.gpu_count != b.gpu_count) return a.gpu_count < b.gpu_count;
    return a.slack < b.slack;
}
}  // namespace

Chromosome evaluate_chromosome(std::vector<Config> gpus, const Engine& e) {  // ga.hpp:38-46
    Chromosome c;
    std::vector<double> comp = e.completion_of(gpus);
    if (!satisfied(comp)) throw PlanningError("chromosome violates the deployment validity invariant");
    c.slack = slack_of(comp);
    c.gpu_count = static_cast<int>(gpus.size());
    c.gpus = std::move(gpus);
    return c;
}

// crossover, ga.hpp:51-77.
Chromosome crossover(const Chromosome& parent, const Procedure& slow, Engine& e, const GaParams& p, Rng& rng) {
    size_t n = parent.gpus.size();
    size_t erase = n == 0 ? 0 : static_cast<size_t>(std::ceil(p.erase_fraction * static_cast<double>(n)));
    if (erase == 0) return parent;
    std::vector<size_t> order(n);
    for (size_t i = 0; i < n; ++i) order[i] = i;
    for (size_t i = 0; i < erase; ++i) {
        size_t j = i + pick_index(rng, n - i);
        std::swap(order[i], order[j]);
    }
    std::vector<bool> erased(n, false);
    for (size_t i = 0; i < erase; ++i) erased[order[i]] = true;
    std::vector<Config> survivors;
    survivors.reserve(n);
    for (size_t i = 0; i < n; ++i)
        if (!erased[i]) survivors.push_back(parent.gpus[i]);
    try {
        std::vector<double> residual = e.completion_of(survivors);
        std::vector<Config> refill = slow.solve(residual, e, rng);
        for (auto& c : refill) survivors.push_back(c);
        return evaluate_chromosome(std::move(survivors), e);
    } catch (const PlanningError&) {
        return parent;
    }
}

// mutate, ga.hpp:83-113: swap (service, batch) of equal-size instances.
Chromosome mutate(const Chromosome& parent, const GaParams& p, Rng& rng) {
    Chromosome child = parent;
    struct Ref {
        size_t gpu, inst;
    };
    // instances by size, sizes ascending (the reference's std::map order); sizes are small
    // slice counts, so a flat table replaces the map
    int max_size = 0;
    for (const auto& g : child.gpus)
        for (int k = 0; k < g.n; ++k) max_size = std::max(max_size, g.inst[k].slices);
    std::vector<std::vector<Ref>> by_size(static_cast<size_t>(max_size) + 1);
    for (size_t g = 0; g < child.gpus.size(); ++g)
        for (int k = 0; k < child.gpus[g].n; ++k) by_size[child.gpus[g].inst[k].slices].push_back(Ref{g, size_t(k)});
    std::vector<int> sizes;
    for (int size = 0; size <= max_size; ++size)
        if (by_size[size].size() >= 2) sizes.push_back(size);
    if (sizes.empty()) return child;
    for (int pair = 0; pair < p.mutation_pairs; ++pair) {
        for (int attempt = 0; attempt < 64; ++attempt) {
            int size = sizes[pick_index(rng, sizes.size())];
            const auto& refs = by_size[size];
            Ref a = refs[pick_index(rng, refs.size())];
            Ref b = refs[pick_index(rng, refs.size())];
            auto& ia = child.gpus[a.gpu].inst[a.inst];
            auto& ib = child.gpus[b.gpu].inst[b.inst];
            if (ia.svc == ib.svc) continue;
            std::swap(ia.svc, ib.svc);
            std::swap(ia.batch, ib.batch);
            break;
        }
    }
    return child;
}

std::vector<Config> sorted_deployment(std::vector<Config> cfgs);

// Throughput-mode two_phase (ga.cu): every generation's mutation, crossover (erase +
// FastProcedure refill, all children in one greedy launch) and fitness run on the device
// over the whole population, with Philox draws (child i of round r: stream (r << 20) + i).
// Host: elitist stable selection over (gpu count, slack) as ga.hpp:165-175.
std::vector<Config> two_phase_parallel(Engine& e, const GaParams& p,
                                       const std::function<void(int, int, double, bool, double)>& log,
                                       const RolloutRefill* slow) {
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    std::vector<Config> seed_cfg = fast_plan(e, std::vector<double>(e.n(), 0.0));
    if (p.time_budget_s <= 0.0 || p.max_rounds <= 0) return sorted_deployment(std::move(seed_cfg));
    if (p.population < 1) throw ArgumentError("two_phase_parallel: population must be >= 1");
    Chromosome seed = evaluate_chromosome(seed_cfg, e);
    const int L_cap = 2 * seed.gpu_count + 64;
    std::vector<uint64_t> g0;
    for (const auto& c : seed_cfg) g0.push_back(e.model().genome_of(c.inst, c.n));
    const double tb0 = elapsed();
    GaRun* run = e.ga_begin(p.population, L_cap);
    if (std::getenv("MIGPLAN_GA_TIMERS"))
        std::fprintf(stderr, "[ga] seed %.2f ms, setup %.2f ms\n", 1e3 * tb0, 1e3 * (elapsed() - tb0));
    struct End {
        Engine& e;
        GaRun* r;
        ~End() { e.ga_end(r); }
    } end{e, run};
    e.ga_put(run, 0, 0, g0);
    struct Ent {
        int len;
        double slack;
    };
    std::vector<Ent> pop{{seed.gpu_count, seed.slack}};
    Ent best = pop[0];
    std::vector<uint64_t> best_g = g0;
    int buf = 0, stall = 0;
    auto fitter = [](const Ent& a, const Ent& b) { return a.len != b.len ? a.len < b.len : a.slack < b.slack; };
    for (int round = 1; round <= p.max_rounds; ++round) {
        if (elapsed() >= p.time_budget_s) break;
        if (stall >= p.stall_rounds) break;
        const size_t npar = std::min(pop.size(), (static_cast<size_t>(p.population) + 1) / 2);
        std::vector<int> plen(npar), clen;
        std::vector<double> cslack;
        for (size_t i = 0; i < npar; ++i) plen[i] = pop[i].len;
        const double tg0 = elapsed();
        e.ga_generation(run, buf, plen, round, p, clen, cslack, slow);
        if (std::getenv("MIGPLAN_GA_TIMERS"))
            std::fprintf(stderr, "[ga] round %d: generation %.2f ms\n", round, 1e3 * (elapsed() - tg0));
        struct Cand {
            bool child;
            int idx;
            Ent f;
        };
        std::vector<Cand> all;
        for (size_t i = 0; i < pop.size(); ++i) all.push_back({false, static_cast<int>(i), pop[i]});
        for (size_t c = 0; c < npar; ++c) all.push_back({true, static_cast<int>(c), {clen[c], cslack[c]}});
        std::stable_sort(all.begin(), all.end(), [&](const Cand& a, const Cand& b) { return fitter(a.f, b.f); });
        if (all.size() > static_cast<size_t>(p.population)) all.resize(p.population);
        std::vector<std::tuple<bool, int, int>> order;
        pop.clear();
        for (const auto& c : all) {
            order.emplace_back(c.child, c.idx, c.f.len);
            pop.push_back(c.f);
        }
        e.ga_select(run, buf, order);
        buf ^= 1;
        const bool improved = fitter(pop[0], best);
        if (improved) {
            best = pop[0];
            best_g = e.ga_get(run, buf, 0, best.len, false);
            stall = 0;
        } else {
            ++stall;
        }
        if (log) log(round, best.len, best.slack, improved, elapsed());
    }
    std::vector<Config> out;
    for (uint64_t g : best_g) {
        Config c;
        c.n = e.model().decode_genome(g, c.inst);
        out.push_back(c);
    }
    return sorted_deployment(std::move(out));
}

std::vector<Config> sorted_deployment(std::vector<Config> cfgs) {  // make_deployment, core.hpp:305-312
    std::sort(cfgs.begin(), cfgs.end(), config_less);
    return cfgs;
}

namespace {

// One GA round's children (ga.hpp:147-151: child i = crossover(mutate(pop[i]), MctsProcedure)),
// computed PHASE BY PHASE across the children so that each device stage is one grouped launch
// over all of them: every child keeps its own mt19937_64 stream and its own sequence of steps,
// so the children are exactly the reference's.
//   host    mutate; crossover's erase draws, survivors, residual; MctsProcedure's seed = rng()
//   device  fast_ref = fast_algo(residual) for all children       (grouped greedy)
//   device  the mcts_solve search loops                            (grouped mcts_kernel)
//   device  fast_algo completions of the visit-count descents      (grouped greedy)
//   host    answer precedence (mcts.hpp:245-251), evaluate_chromosome; PlanningError -> parent
// MIGPLAN_GA_TIMERS=1: host-side timeline of the parity GA (phase durations to stderr).
struct Timeline {
    bool on = std::getenv("MIGPLAN_GA_TIMERS") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ga] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

std::vector<Chromosome> breed_round(Engine& e, const std::vector<Chromosome>& pop, size_t n_parents, int round,
                                    const GaParams& p) {
    Timeline tl;
    struct Child {
        Chromosome c;  // the mutated parent (crossover's fallback)
        std::vector<Config> survivors, fast_ref, refill;
        std::vector<double> residual;
        uint64_t seed = 0;
        bool done = false;       // crossover fell back to the parent (result)
        bool no_refill = false;  // the survivors already satisfy every service
        Chromosome result;
        MctsDeviceResult mr;
    };
    std::vector<Child> ch(n_parents);
    auto fail = [&](Child& x) {  // crossover: catch (PlanningError) { return parent; }
        x.result = x.c;
        x.done = true;
    };
    for (size_t i = 0; i < n_parents; ++i) {
        Child& x = ch[i];
        Rng rng(mix_seed(p.seed, (static_cast<uint64_t>(round) << 20) + i));
        x.c = mutate(pop[i], p, rng);
        const size_t n = x.c.gpus.size();
        const size_t erase = n == 0 ? 0 : static_cast<size_t>(std::ceil(p.erase_fraction * static_cast<double>(n)));
        if (erase == 0) {
            fail(x);  // crossover returns its parent unchanged (ga.hpp:55)
            continue;
        }
        std::vector<size_t> order(n);
        for (size_t k = 0; k < n; ++k) order[k] = k;
        for (size_t k = 0; k < erase; ++k) std::swap(order[k], order[k + pick_index(rng, n - k)]);
        std::vector<bool> erased(n, false);
        for (size_t k = 0; k < erase; ++k) erased[order[k]] = true;
        for (size_t k = 0; k < n; ++k)
            if (!erased[k]) x.survivors.push_back(x.c.gpus[k]);
        try {
            x.residual = e.completion_of(x.survivors);
        } catch (const PlanningError&) {
            fail(x);
            continue;
        }
        x.seed = rng();  // MctsProcedure::solve: mcts_solve(comp, ctx, params, rng()) (mcts.hpp:258)
        if (satisfied(x.residual)) x.no_refill = true;  // mcts_solve returns {} (mcts.hpp:151)
    }
    tl.mark("mutate+erase (host)");
    // fast_ref for every child still searching
    std::vector<size_t> live;
    std::vector<std::vector<double>> comps;
    for (size_t i = 0; i < n_parents; ++i)
        if (!ch[i].done && !ch[i].no_refill) {
            live.push_back(i);
            comps.push_back(ch[i].residual);
        }
    std::vector<std::vector<uint64_t>> rows;
    std::vector<int> st;
    e.fast_algo_batch(comps, rows, st);
    tl.mark("fast_ref batch");
    std::vector<size_t> search;
    for (size_t q = 0; q < live.size(); ++q) {
        Child& x = ch[live[q]];
        if (st[q]) {
            fail(x);
            continue;
        }
        for (uint64_t r : rows[q]) x.fast_ref.push_back(e.config_of(r));
        if (p.slow.budget_iters <= 0 || p.slow.topk < 1) x.refill = x.fast_ref;
        else search.push_back(live[q]);
    }
    // the searches, one CTA each, one launch
    {
        std::vector<std::vector<double>> sc;
        std::vector<uint64_t> seeds;
        std::vector<int> lrefs;
        for (size_t i : search) {
            sc.push_back(ch[i].residual);
            seeds.push_back(ch[i].seed);
            lrefs.push_back(static_cast<int>(ch[i].fast_ref.size()));
        }
        tl.mark("configs (host)");
        auto res = e.mcts_device_group(sc, p.slow.budget_iters, p.slow.topk, p.slow.pick_services, p.slow.ucb_c, seeds,
                                       lrefs);
        tl.mark("mcts group");
        for (size_t q = 0; q < search.size(); ++q) {
            if (res[q].status == 1) {
                fail(ch[search[q]]);  // rollout: empty pool -> PlanningError
                continue;
            }
            if (res[q].status != 0) throw DeviceError("mcts: device search storage exhausted");
            ch[search[q]].mr = std::move(res[q]);
        }
    }
    // descent completions
    std::vector<size_t> desc;
    std::vector<std::vector<double>> dc;
    for (size_t i : search)
        if (!ch[i].done && !ch[i].mr.descent_leaf) {
            desc.push_back(i);
            dc.push_back(ch[i].mr.descent_comp);
        }
    std::vector<std::vector<uint64_t>> drows;
    std::vector<int> dst;
    e.fast_algo_batch(dc, drows, dst);
    tl.mark("descent batch");
    std::vector<std::vector<Config>> tail(n_parents);
    for (size_t q = 0; q < desc.size(); ++q) {
        if (dst[q]) {
            fail(ch[desc[q]]);
            continue;
        }
        for (uint64_t r : drows[q]) tail[desc[q]].push_back(e.config_of(r));
    }
    for (size_t i : search) {
        Child& x = ch[i];
        if (x.done) continue;
        std::vector<Config> via;
        for (long long idx : x.mr.descent) via.push_back(e.config_of(e.base_rows()[idx]));
        for (auto& c : tail[i]) via.push_back(c);
        std::vector<Config> answer = x.fast_ref;
        if (via.size() < answer.size()) answer = std::move(via);
        if (x.mr.best_len >= 0 && static_cast<size_t>(x.mr.best_len) < answer.size()) {
            answer.clear();
            for (long long idx : x.mr.best) answer.push_back(e.config_of(e.base_rows()[idx]));
        }
        x.refill = std::move(answer);
    }
    tl.mark("answers (host)");
    std::vector<Chromosome> out(n_parents);
    for (size_t i = 0; i < n_parents; ++i) {
        Child& x = ch[i];
        if (x.done) {
            out[i] = x.result;
            continue;
        }
        std::vector<Config> full = x.survivors;
        for (auto& c : x.refill) full.push_back(c);
        try {
            out[i] = evaluate_chromosome(std::move(full), e);
        } catch (const PlanningError&) {
            out[i] = x.c;
        }
    }
    tl.mark("evaluate (host)");
    return out;
}

}  // namespace

// two_phase, ga.hpp:126-179 (on an existing max_mix-2 context).
std::vector<Config> two_phase(Engine& e, const GaParams& p,
                              const std::function<void(int, int, double, bool, double)>& log) {
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    Timeline tl;
    std::vector<Config> seed_cfg = fast_plan(e, std::vector<double>(e.n(), 0.0));
    tl.mark("seed fast_algo");
    if (p.time_budget_s <= 0.0 || p.max_rounds <= 0) return sorted_deployment(std::move(seed_cfg));

    std::vector<Chromosome> pop;
    pop.push_back(evaluate_chromosome(std::move(seed_cfg), e));
    tl.mark("seed evaluate");
    Chromosome best = pop[0];
    MctsProc slow(p.slow);
    int stall = 0;
    for (int round = 1; round <= p.max_rounds; ++round) {
        if (elapsed() >= p.time_budget_s) break;
        if (stall >= p.stall_rounds) break;
        size_t n_parents = std::min(pop.size(), (static_cast<size_t>(p.population) + 1) / 2);
        if (p.slow.topk >= 1 && p.slow.topk <= 32) {  // phased, device-batched children
            std::vector<Chromosome> children = breed_round(e, pop, n_parents, round, p);
            for (auto& c : children) pop.push_back(std::move(c));
            std::stable_sort(pop.begin(), pop.end(), fitter);
            if (pop.size() > static_cast<size_t>(p.population)) pop.resize(p.population);
            bool improved = fitter(pop[0], best);
            if (improved) {
                best = pop[0];
                stall = 0;
            } else {
                ++stall;
            }
            if (log) log(round, best.gpu_count, best.slack, improved, elapsed());
            continue;
        }
        std::vector<Chromosome> children(n_parents);
        std::vector<std::exception_ptr> errs(n_parents);
        auto work = [&](size_t i) {
            try {
                Rng rng(mix_seed(p.seed, (static_cast<uint64_t>(round) << 20) + i));
                Chromosome c = mutate(pop[i], p, rng);
                children[i] = crossover(c, slow, e, p, rng);
            } catch (...) {
                errs[i] = std::current_exception();
            }
        };
        if (p.workers > 1 && n_parents > 1) {
            std::vector<std::thread> threads;
            size_t w = std::min<size_t>(static_cast<size_t>(p.workers), n_parents);
            for (size_t t = 0; t < w; ++t)
                threads.emplace_back([&, t] {
                    for (size_t i = t; i < n_parents; i += w) work(i);
                });
            for (auto& th : threads) th.join();
        } else {
            for (size_t i = 0; i < n_parents; ++i) work(i);
        }
        for (auto& ep : errs)
            if (ep) std::rethrow_exception(ep);
        for (auto& c : children) pop.push_back(std::move(c));
        std::stable_sort(pop.begin(), pop.end(), fitter);
        if (pop.size() > static_cast<size_t>(p.population)) pop.resize(p.population);
        bool improved = fitter(pop[0], best);
        if (improved) {
            best = pop[0];
            stall = 0;
        } else {
            ++stall;
        }
        if (log) log(round, best.gpu_count, best.slack, improved, elapsed());
    }
    return sorted_deployment(std::move(best.gpus));
}

}  // namespace mgb

// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Puts the UNMODIFIED reference implementation (`/root/reference/proj/include/migplan/*.hpp`,
// compiled from where it lies via -I, see oracle/Makefile) behind the same C-ABI as the
// product (`include/migplan_b200.h`).  The result, oracle/_ref/libmigref.so, is
//   * the checker that pins the CPU restatement (oracle/oracle.cpp),
//   * the generator of tests/golden/*.json (oracle/gen_golden.py),
//   * the `cpu_baseline` / `--impl reference` arm of bench.py.
// Build rule: -O3 -DNDEBUG, no -march=native, -ffp-contract=off.
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "migplan/bench.hpp"
#include "migplan/config_enum.hpp"
#include "migplan/core.hpp"
#include "migplan/ga.hpp"
#include "migplan/greedy.hpp"
#include "migplan/mcts.hpp"
#include "migplan/mig_rules.hpp"
#include "migplan_b200.h"
#ifdef MIGREF_WITH_IO
#include "migplan/io.hpp"
#include "migplan/transition_planner.hpp"
#endif

using namespace migplan;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return MIG_OK;
    } catch (const PlanningError& e) {
        g_err = e.what();
        return MIG_ERR_PLANNING;
    } catch (const SchemaError& e) {
        g_err = e.what();
        return MIG_ERR_SCHEMA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return MIG_ERR_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MIG_ERR_PLANNING;
    }
}

PartitionRuleSet rules_of(const mig_rules* r) {
    if (!r) return PartitionRuleSet::defaults();
    PartitionRuleSet out;
    for (int i = 0; i < r->n_sizes; ++i) {
        auto& v = out.slot_positions[r->size[i]];
        for (int k = 0; k < r->n_slots[i]; ++k) v.push_back(r->slots[i][k]);
        std::sort(v.begin(), v.end());
    }
    for (int i = 0; i < r->n_weights; ++i) out.memory_weight[r->weight_size[i]] = r->weight[i];
    for (int i = 0; i < r->n_exclusions; ++i)
        out.hard_exclusions.insert(normalized_pair(r->exclusion[i][0], r->exclusion[i][1]));
    out.memory_budget = r->memory_budget;
    return out;
}

ProfileStore store_of(const mig_model_profile* models, int n_models) {
    ProfileStore ps;
    for (int m = 0; m < n_models; ++m) {
        ModelProfile p;
        p.model_name = models[m].model_name ? models[m].model_name : "";
        for (int e = 0; e < models[m].n_entries; ++e) {
            const auto& x = models[m].entries[e];
            p.entries[x.size].push_back(ProfileEntry{x.batch, x.throughput_rps, x.p90_ms});
        }
        for (auto& [size, list] : p.entries)
            std::sort(list.begin(), list.end(),
                      [](const ProfileEntry& a, const ProfileEntry& b) { return a.batch < b.batch; });
        validate_profile(p);
        if (ps.count(p.model_name)) throw SchemaError("duplicate model '" + p.model_name + "'");
        ps[p.model_name] = std::move(p);
    }
    return ps;
}

std::vector<ServiceSpec> services_of(const mig_service* s, int n) {
    std::vector<ServiceSpec> out;
    for (int i = 0; i < n; ++i)
        out.push_back(ServiceSpec{s[i].service_id ? s[i].service_id : "", s[i].model_name ? s[i].model_name : "",
                                  s[i].required_rps, s[i].max_p90_ms});
    return out;
}

}  // namespace

struct mig_ctx {
    ProfileStore profiles;
    PartitionRuleSet rules;
    std::vector<ServiceSpec> services;
    PlanContext plan;
    std::vector<double> last_comp;  // start of the last mig_fast_algo (mig_ctx_step_rows replays it)
    bool have_last = false;
};

struct mig_rng {
    Rng rng;
};

struct mig_rollout_cache {
    RolloutCache cache;
};

namespace {

void to_c(const GpuConfig& cfg, const std::vector<ServiceSpec>& services, mig_config* out) {
    if (cfg.instances.size() > MIG_MAX_INSTANCES) throw std::invalid_argument("config has more than 7 instances");
    std::memset(out, 0, sizeof *out);
    out->n_instances = static_cast<int32_t>(cfg.instances.size());
    for (size_t k = 0; k < cfg.instances.size(); ++k) {
        const auto& in = cfg.instances[k];
        out->inst[k] = mig_instance{in.placement.slices, in.placement.start_slot,
                                    service_index(services, in.service_id), in.batch};
    }
}

GpuConfig from_c(const mig_config& c, const std::vector<ServiceSpec>& services) {
    GpuConfig g;
    for (int k = 0; k < c.n_instances; ++k) {
        const auto& in = c.inst[k];
        if (in.service < 0 || in.service >= static_cast<int>(services.size()))
            throw PlanningError("unknown service index " + std::to_string(in.service));
        g.instances.push_back(AssignedInstance{Placement{in.slices, in.slot}, services[in.service].service_id, in.batch});
    }
    return g;
}

void cand_to_c(const Candidate& c, const std::vector<ServiceSpec>& services, mig_candidate* out) {
    std::memset(out, 0, sizeof *out);
    to_c(c.config, services, &out->config);
    out->nnz = static_cast<int32_t>(c.util.size());
    for (size_t k = 0; k < c.util.size() && k < MIG_MAX_INSTANCES; ++k) {
        out->util_idx[k] = c.util[k].first;
        out->util_val[k] = c.util[k].second;
    }
    out->util_sum = c.util_sum;
}

CompletionRates comp_of(const double* comp, int n, const mig_ctx* ctx) {
    if (n != static_cast<int>(ctx->services.size()))
        throw PlanningError("completion vector length mismatch");
    return CompletionRates{std::vector<double>(comp, comp + n)};
}

thread_local std::vector<mig_config> g_pending;  // a plan that did not fit its caller's buffer
int emit_plan(const std::vector<GpuConfig>& plan, const std::vector<ServiceSpec>& services, mig_config* out,
              int32_t cap, int32_t* n_out) {
    *n_out = static_cast<int32_t>(plan.size());
    for (size_t i = 0; i < plan.size() && static_cast<int32_t>(i) < cap; ++i) to_c(plan[i], services, &out[i]);
    if (static_cast<int32_t>(plan.size()) > cap) {
        g_pending.resize(plan.size());
        for (size_t i = 0; i < plan.size(); ++i) to_c(plan[i], services, &g_pending[i]);
        g_err = "output capacity too small";
        return MIG_ERR_ARGUMENT;
    }
    return MIG_OK;
}

MctsParams mcts_of(const mig_mcts_params* p) {
    MctsParams m;
    if (p) {
        m.budget_iters = p->budget_iters;
        m.topk = p->topk;
        m.pick_services = p->pick_services;
        m.ucb_c = p->ucb_c;
    }
    return m;
}

GaParams ga_of(const mig_ga_params* p) {
    GaParams g;
    if (p) {
        g.population = p->population;
        g.erase_fraction = p->erase_fraction;
        g.mutation_pairs = p->mutation_pairs;
        g.stall_rounds = p->stall_rounds;
        g.time_budget_s = p->time_budget_s;
        g.seed = p->seed;
        g.max_rounds = p->max_rounds;
        g.workers = p->workers;
        g.slow = mcts_of(&p->slow);
    }
    return g;
}

// Instrumented replica of fast_algo's working-set growth (greedy.hpp:95-145), used
// only to count rows scored for bench.py's reference arm; results equal fast_algo.
// max_steps >= 0 stops after that many steps (a plan prefix); step_rows, if given,
// receives each step's working-set size and ext_rows each extension event's added rows.
int64_t count_rows(const CompletionRates& comp, const PlanContext& ctx, int64_t max_steps = -1,
                   std::vector<int64_t>* step_rows = nullptr, std::vector<int64_t>* ext_rows = nullptr) {
    int64_t rows = 0;
    int64_t steps = 0;
    CompletionRates cur = comp;
    if (is_satisfied(cur)) return 0;
    detail::WorkingSet ws(ctx.pool);
    std::vector<bool> almost(ctx.services.size(), false);
    auto maybe_extend = [&] {
        std::set<int> unsat;
        for (size_t i = 0; i < cur.values.size(); ++i)
            if (cur.values[i] < 1.0 - kSatisfyEps) unsat.insert(static_cast<int>(i));
        for (int i : unsat) {
            if (almost[i]) continue;
            if (1.0 - cur.values[i] < ctx.pool.best_single_util[i]) {
                almost[i] = true;
                size_t before = ws.extra.items.size();
                extend_candidate_pool(ws.extra, ctx.services, *ctx.profiles, ctx.rules, i, unsat, 4);
                if (ext_rows) ext_rows->push_back(static_cast<int64_t>(ws.extra.items.size() - before));
            }
        }
    };
    maybe_extend();
    while (!is_satisfied(cur) && (max_steps < 0 || steps < max_steps)) {
        ++steps;
        rows += static_cast<int64_t>(ws.size());
        if (step_rows) step_rows->push_back(static_cast<int64_t>(ws.size()));
        int best = -1;
        double best_score = 0.0;
        for (size_t i = 0; i < ws.size(); ++i) {
            double s = score(ws.at(i), cur);
            if (s <= 0.0) continue;
            if (best < 0 || candidate_preferred(ws.at(i), s, ws.at(best), best_score)) {
                best = static_cast<int>(i);
                best_score = s;
            }
        }
        if (best < 0) throw PlanningError("fast_algo: no config with positive score while services remain unsatisfied");
        for (const auto& [idx, u] : ws.at(best).util) cur.values[idx] += u;
        maybe_extend();
    }
    return rows;
}

}  // namespace

extern "C" {

const char* mig_last_error(void) { return g_err.c_str(); }
int32_t mig_abi_version(void) { return 1; }
const char* mig_impl_name(void) { return "reference"; }

void mig_rules_defaults(mig_rules* out) {
    std::memset(out, 0, sizeof *out);
    PartitionRuleSet d = PartitionRuleSet::defaults();
    for (const auto& [size, slots] : d.slot_positions) {
        int i = out->n_sizes++;
        out->size[i] = size;
        out->n_slots[i] = static_cast<int32_t>(slots.size());
        for (size_t k = 0; k < slots.size(); ++k) out->slots[i][k] = slots[k];
    }
    for (const auto& [size, w] : d.memory_weight) {
        int i = out->n_weights++;
        out->weight_size[i] = size;
        out->weight[i] = w;
    }
    for (const auto& [a, b] : d.hard_exclusions) {
        int i = out->n_exclusions++;
        out->exclusion[i][0] = a;
        out->exclusion[i][1] = b;
    }
    out->memory_budget = d.memory_budget;
}

int mig_is_legal_partition(const mig_rules* rules, const int32_t* slices, const int32_t* slots, int32_t n,
                           int32_t* legal) {
    return guarded([&] {
        std::vector<Placement> ps;
        for (int i = 0; i < n; ++i) ps.push_back(Placement{slices[i], slots[i]});
        *legal = is_legal_partition(ps, rules_of(rules)) ? 1 : 0;
    });
}

int mig_enumerate_maximal_partitions(const mig_rules* rules, mig_partition* out, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        auto parts = enumerate_maximal_partitions(rules_of(rules));
        *n_out = static_cast<int32_t>(parts.size());
        if (*n_out > cap) throw std::invalid_argument("output capacity too small");
        for (size_t i = 0; i < parts.size(); ++i) {
            std::memset(&out[i], 0, sizeof out[i]);
            out[i].n = static_cast<int32_t>(parts[i].placements.size());
            for (size_t k = 0; k < parts[i].placements.size(); ++k) {
                out[i].slices[k] = parts[i].placements[k].slices;
                out[i].slot[k] = parts[i].placements[k].start_slot;
            }
        }
    });
}

int mig_validate_services(const mig_model_profile* models, int32_t n_models, const mig_service* services,
                          int32_t n_services, int32_t* perm) {
    return guarded([&] {
        ProfileStore ps = store_of(models, n_models);
        auto svcs = services_of(services, n_services);
        validate_services(svcs, ps);
        std::vector<bool> used(n_services, false);
        for (int i = 0; i < n_services; ++i)
            for (int j = 0; j < n_services; ++j)
                if (!used[j] && svcs[i].service_id == (services[j].service_id ? services[j].service_id : "")) {
                    perm[i] = j;
                    used[j] = true;
                    break;
                }
    });
}

int mig_ctx_create(const mig_rules* rules, const mig_model_profile* models, int32_t n_models,
                   const mig_service* services, int32_t n_services, int32_t max_mix, int32_t, mig_ctx** out) {
    return guarded([&] {
        auto ctx = std::make_unique<mig_ctx>();
        ctx->profiles = store_of(models, n_models);
        ctx->rules = rules_of(rules);
        ctx->services = services_of(services, n_services);
        ctx->plan = make_plan_context(ctx->services, ctx->profiles, ctx->rules, max_mix);
        *out = ctx.release();
    });
}

void mig_ctx_destroy(mig_ctx* ctx) { delete ctx; }
int32_t mig_ctx_n_services(const mig_ctx* ctx) { return static_cast<int32_t>(ctx->services.size()); }

int mig_pool_size(const mig_ctx* ctx, int64_t* out) {
    *out = static_cast<int64_t>(ctx->plan.pool.items.size());
    return MIG_OK;
}

int mig_pool_candidate(const mig_ctx* ctx, int64_t idx, mig_candidate* out) {
    return guarded([&] {
        if (idx < 0 || idx >= static_cast<int64_t>(ctx->plan.pool.items.size()))
            throw std::invalid_argument("pool index out of range");
        cand_to_c(ctx->plan.pool.items[idx], ctx->services, out);
    });
}

int mig_pool_best_single_util(const mig_ctx* ctx, double* out) {
    for (size_t i = 0; i < ctx->services.size(); ++i) out[i] = ctx->plan.pool.best_single_util[i];
    return MIG_OK;
}

int mig_score(const mig_ctx* ctx, int64_t idx, const double* comp, int32_t n, double* out) {
    return guarded([&] {
        if (idx < 0 || idx >= static_cast<int64_t>(ctx->plan.pool.items.size()))
            throw std::invalid_argument("pool index out of range");
        *out = score(ctx->plan.pool.items[idx], comp_of(comp, n, ctx));
    });
}

int mig_topk_candidates(mig_ctx* ctx, const double* comp, int32_t n, int32_t k, const int64_t* from,
                        int64_t n_from, int64_t* out_idx, int32_t* n_out) {
    return guarded([&] {
        CompletionRates c = comp_of(comp, n, ctx);
        std::vector<int> f;
        if (from && n_from >= 0)
            for (int64_t i = 0; i < n_from; ++i) f.push_back(static_cast<int>(from[i]));
        auto top = detail::topk_candidates(ctx->plan.pool, c, k, (from && n_from >= 0) ? &f : nullptr);
        *n_out = static_cast<int32_t>(top.size());
        for (size_t i = 0; i < top.size(); ++i) out_idx[i] = top[i];
    });
}

int mig_fast_algo(mig_ctx* ctx, const double* comp, int32_t n, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_greedy_trace_fn trace, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        CompletionRates c = comp_of(comp, n, ctx);
        std::function<void(int, const Candidate&, double, const CompletionRates&)> tr = nullptr;
        if (trace)
            tr = [&](int iter, const Candidate& cand, double s, const CompletionRates& cur) {
                mig_candidate mc;
                cand_to_c(cand, ctx->services, &mc);
                trace(user, iter, &mc, s, cur.values.data(), static_cast<int32_t>(cur.values.size()));
            };
        auto plan = fast_algo(c, ctx->plan, tr);
        ctx->last_comp = c.values;
        ctx->have_last = true;
        rc = emit_plan(plan, ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_rng_create(uint64_t seed, mig_rng** out) {
    *out = new mig_rng{Rng(seed)};
    return MIG_OK;
}
void mig_rng_destroy(mig_rng* rng) { delete rng; }
uint64_t mig_rng_next(mig_rng* rng) { return rng->rng(); }
uint64_t mig_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }
uint64_t mig_pick_index(mig_rng* rng, uint64_t n) { return pick_index(rng->rng, n); }

void mig_mcts_params_defaults(mig_mcts_params* out) {
    MctsParams m;
    *out = mig_mcts_params{m.budget_iters, m.topk, m.pick_services, m.ucb_c};
}

int mig_expand(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params, mig_rng* rng,
               int64_t* children, int32_t cap, int32_t* n_children) {
    return guarded([&] {
        SearchNode node(comp_of(comp, n, ctx));
        auto top = expand(node, ctx->plan, mcts_of(params), rng->rng);
        *n_children = static_cast<int32_t>(top.size());
        if (*n_children > cap) throw std::invalid_argument("output capacity too small");
        for (size_t i = 0; i < top.size(); ++i) children[i] = top[i];
    });
}

int mig_rollout_cache_create(mig_rollout_cache** out) {
    *out = new mig_rollout_cache{};
    return MIG_OK;
}
void mig_rollout_cache_destroy(mig_rollout_cache* cache) { delete cache; }
int32_t mig_rollout_cache_builds(const mig_rollout_cache* cache) { return cache->cache.builds; }

int mig_rollout(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params,
                mig_rollout_cache* cache, mig_rng* rng, int32_t max_depth, int64_t* picked, int32_t cap,
                int32_t* steps) {
    return guarded([&] {
        std::vector<int> p;
        *steps = rollout(comp_of(comp, n, ctx), ctx->plan, mcts_of(params), cache->cache, rng->rng, max_depth,
                         picked ? &p : nullptr);
        if (picked) {
            if (static_cast<int32_t>(p.size()) > cap) throw std::invalid_argument("output capacity too small");
            for (size_t i = 0; i < p.size(); ++i) picked[i] = p[i];
        }
    });
}

int mig_mcts_solve(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params, uint64_t seed,
                   mig_config* out, int32_t cap, int32_t* n_out, mig_mcts_trace_fn trace, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::function<void(int, int, int, int)> tr = nullptr;
        if (trace) tr = [&](int a, int b, int c, int d) { trace(user, a, b, c, d); };
        auto plan = mcts_solve(comp_of(comp, n, ctx), ctx->plan, mcts_of(params), seed, tr);
        rc = emit_plan(plan, ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

}  // extern "C"

namespace {
// Throughput-mode rollouts (include/migplan_b200.h, mig_rollouts) assembled from the
// reference's own primitives: completion_type_key, detail::topk_candidates over ctx.pool,
// is_satisfied and the util add of rollout (mcts.hpp:38-43,56-76,122-143).  Only the
// schedule (lock-step rounds, lowest-index claims, Philox draws) is the product's.
uint64_t philox64_ref(uint64_t seed, uint64_t stream, uint64_t step) {
    uint32_t c[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        uint64_t a = (uint64_t)0xD2511F53u * c[0], b = (uint64_t)0xCD9E8D57u * c[2];
        c[0] = (uint32_t)(b >> 32) ^ c[1] ^ k0;
        c[1] = (uint32_t)b;
        c[2] = (uint32_t)(a >> 32) ^ c[3] ^ k1;
        c[3] = (uint32_t)a;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return ((uint64_t)c[1] << 32) | c[0];
}
struct RefPar {
    int best_len = -1;
    long long best_id = -1;
    std::vector<int> path;
    long long completed = 0, capped = 0, failed = 0, steps = 0, keys = 0;
    int rounds = 0;
};
RefPar ref_par(const PlanContext& ctx, const CompletionRates& comp, long long R, int K, int depth, uint64_t seed,
               long long id0, long long batch, int32_t* lengths) {
    RefPar res;
    RolloutCache cache;
    if (batch <= 0 || batch > R) batch = R;
    for (long long b0 = 0; b0 < R; b0 += batch) {
        long long nb = std::min(batch, R - b0);
        std::vector<CompletionRates> cur(nb, comp);
        std::vector<std::vector<int>> picks(nb);
        auto finish = [&](long long r) {
            int L = (int)picks[r].size();
            if (is_satisfied(cur[r])) {
                res.completed++;
                if (lengths) lengths[b0 + r] = L;
                long long id = id0 + b0 + r;
                if (res.best_len < 0 || L < res.best_len || (L == res.best_len && id < res.best_id))
                    res.best_len = L, res.best_id = id, res.path = picks[r];
                return true;
            }
            if (L >= depth) {
                res.capped++;
                if (lengths) lengths[b0 + r] = depth;
                return true;
            }
            return false;
        };
        std::vector<long long> act;
        for (long long r = 0; r < nb; ++r)
            if (!finish(r)) act.push_back(r);
        int rounds = 0;
        while (!act.empty()) {
            ++rounds;
            for (long long r : act) {  // ascending: the lowest index claims a new key
                std::string key = completion_type_key(cur[r]);
                if (!cache.pools.count(key)) {
                    ++cache.builds;
                    cache.pools.emplace(key, detail::topk_candidates(ctx.pool, cur[r], K, nullptr));
                }
            }
            std::vector<long long> next;
            for (long long r : act) {
                const std::vector<int>& pool = cache.pools.at(completion_type_key(cur[r]));
                if (pool.empty()) {
                    res.failed++;
                    if (lengths) lengths[b0 + r] = -1;
                    continue;
                }
                uint64_t x = philox64_ref(seed, (uint64_t)(id0 + b0 + r), (uint64_t)picks[r].size());
                int idx = pool[(size_t)(((unsigned __int128)x * pool.size()) >> 64)];
                for (const auto& [svc, u] : ctx.pool.items[idx].util) cur[r].values[svc] += u;
                picks[r].push_back(idx);
                res.steps++;
                if (!finish(r)) next.push_back(r);
            }
            act = std::move(next);
        }
        res.rounds = std::max(res.rounds, rounds);
    }
    res.keys = cache.builds;
    return res;
}
// Throughput-mode two_phase (mig_two_phase_parallel) on the reference's own operators'
// building blocks (GpuConfig, fast_algo, completion_of, evaluate_chromosome, fitter,
// make_deployment; ga.hpp, greedy.hpp, core.hpp).  The draws are the product's Philox
// stream instead of mt19937_64, so mutate/crossover are restated around them.
Chromosome mutate_philox(const Chromosome& parent, const GaParams& params, const std::function<size_t(size_t)>& dr) {
    Chromosome child = parent;  // ga.hpp:83-113
    struct Ref {
        size_t gpu, inst;
    };
    std::map<int, std::vector<Ref>> by_size;
    for (size_t g = 0; g < child.gpus.size(); ++g)
        for (size_t k = 0; k < child.gpus[g].instances.size(); ++k)
            by_size[child.gpus[g].instances[k].placement.slices].push_back(Ref{g, k});
    std::vector<int> sizes;
    for (const auto& [size, refs] : by_size)
        if (refs.size() >= 2) sizes.push_back(size);
    if (sizes.empty()) return child;
    for (int pair = 0; pair < params.mutation_pairs; ++pair)
        for (int attempt = 0; attempt < 64; ++attempt) {
            int size = sizes[dr(sizes.size())];
            const auto& refs = by_size[size];
            Ref a = refs[dr(refs.size())];
            Ref b = refs[dr(refs.size())];
            AssignedInstance& ia = child.gpus[a.gpu].instances[a.inst];
            AssignedInstance& ib = child.gpus[b.gpu].instances[b.inst];
            if (ia.service_id == ib.service_id) continue;
            std::swap(ia.service_id, ib.service_id);
            std::swap(ia.batch, ib.batch);
            break;
        }
    return child;
}

RefPar ref_par(const PlanContext& ctx, const CompletionRates& comp, long long R, int K, int depth, uint64_t seed,
              long long id0, long long batch, int32_t* lengths);

// slow == nullptr: FastProcedure refill.  Otherwise the throughput mcts_solve
// (mig_mcts_solve_parallel): the shorter of fast_algo(residual) and the best of
// slow->n_rollouts root-parallel rollouts under Philox key `rseed` (fast wins ties).
Chromosome crossover_philox(const Chromosome& parent, const PlanContext& ctx, const GaParams& params,
                            const std::function<size_t(size_t)>& dr, size_t lcap,
                            const mig_rollout_params* slow = nullptr, uint64_t rseed = 0) {  // ga.hpp:51-77
    size_t n = parent.gpus.size();
    size_t erase = n == 0 ? 0 : static_cast<size_t>(std::ceil(params.erase_fraction * static_cast<double>(n)));
    if (erase == 0) return parent;
    std::vector<size_t> order(n);
    for (size_t i = 0; i < n; ++i) order[i] = i;
    for (size_t i = 0; i < erase; ++i) std::swap(order[i], order[i + dr(n - i)]);
    std::vector<bool> erased(n, false);
    for (size_t i = 0; i < erase; ++i) erased[order[i]] = true;
    std::vector<GpuConfig> survivors;
    for (size_t i = 0; i < n; ++i)
        if (!erased[i]) survivors.push_back(parent.gpus[i]);
    try {
        CompletionRates residual = completion_of(survivors, ctx.services, *ctx.profiles);
        std::vector<GpuConfig> refill = fast_algo(residual, ctx);
        if (slow && !is_satisfied(residual)) {
            RefPar r = ref_par(ctx, residual, slow->n_rollouts, slow->topk, 2 * static_cast<int>(refill.size()), rseed,
                               slow->id_offset, slow->batch, nullptr);
            if (r.best_len >= 0 && static_cast<size_t>(r.best_len) < refill.size()) {
                refill.clear();
                for (int i : r.path) refill.push_back(ctx.pool.items[i].config);
            }
        }
        for (auto& cfg : refill) survivors.push_back(std::move(cfg));
        if (survivors.size() > lcap) return parent;
        return evaluate_chromosome(std::move(survivors), ctx);
    } catch (const PlanningError&) {
        return parent;
    }
}

std::vector<GpuConfig> two_phase_philox(const PlanContext& ctx, const GaParams& params,
                                        const std::function<void(const GaRoundLog&)>& log,
                                        const mig_rollout_params* slow = nullptr) {
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    std::vector<GpuConfig> seed_cfg = fast_algo(zero_completion(ctx.services.size()), ctx);
    if (params.time_budget_s <= 0.0 || params.max_rounds <= 0) {
        std::sort(seed_cfg.begin(), seed_cfg.end());
        return seed_cfg;
    }
    const size_t lcap = 2 * seed_cfg.size() + 64;
    std::vector<Chromosome> pop;
    pop.push_back(evaluate_chromosome(std::move(seed_cfg), ctx));
    Chromosome best = pop[0];
    int stall = 0;
    for (int round = 1; round <= params.max_rounds; ++round) {
        if (elapsed() >= params.time_budget_s) break;
        if (stall >= params.stall_rounds) break;
        size_t n_parents = std::min(pop.size(), (static_cast<size_t>(params.population) + 1) / 2);
        std::vector<Chromosome> children(n_parents);
        for (size_t i = 0; i < n_parents; ++i) {
            uint64_t t = 0;
            const uint64_t stream = (static_cast<uint64_t>(round) << 20) + i;
            std::function<size_t(size_t)> dr = [&](size_t m) {
                return static_cast<size_t>(((unsigned __int128)philox64_ref(params.seed, stream, t++) * m) >> 64);
            };
            children[i] = crossover_philox(mutate_philox(pop[i], params, dr), ctx, params, dr, lcap, slow,
                                           mix_seed(params.seed, stream));
        }
        for (auto& c : children) pop.push_back(std::move(c));
        std::stable_sort(pop.begin(), pop.end(), fitter);
        if (pop.size() > static_cast<size_t>(params.population)) pop.resize(params.population);
        bool improved = fitter(pop[0], best);
        if (improved) {
            best = pop[0];
            stall = 0;
        } else {
            ++stall;
        }
        if (log) log(GaRoundLog{round, best.gpu_count, best.slack, improved, elapsed()});
    }
    std::sort(best.gpus.begin(), best.gpus.end());
    return best.gpus;
}

void ref_par_out(const RefPar& r, int depth, mig_rollout_result* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->best_len = r.best_len;
    o->max_depth = depth;
    o->best_id = r.best_id;
    o->completed = r.completed;
    o->capped = r.capped;
    o->failed = r.failed;
    o->steps = r.steps;
    o->keys = r.keys;
    o->rounds = r.rounds;
    o->path_len = (int32_t)r.path.size();
}
}  // namespace

extern "C" {

int mig_rollouts(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* p, int32_t* lengths,
                 int64_t* best_path, int32_t cap, mig_rollout_result* out) {
    return guarded([&] {
        if (!p) throw std::invalid_argument("null rollout params");
        if (p->topk < 1 || p->topk > 32) throw std::invalid_argument("rollouts: topk must be in [1, 32]");
        CompletionRates c = comp_of(comp, n, ctx);
        int depth = p->max_depth < 0 ? 2 * (int)fast_algo(c, ctx->plan).size() : p->max_depth;
        RefPar r = ref_par(ctx->plan, c, p->n_rollouts, p->topk, depth, p->seed, p->id_offset, p->batch, lengths);
        if (best_path) {
            if ((int)r.path.size() > cap) throw std::invalid_argument("output capacity too small");
            for (size_t i = 0; i < r.path.size(); ++i) best_path[i] = r.path[i];
        }
        ref_par_out(r, depth, out);
    });
}

int mig_mcts_solve_parallel(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* p,
                            mig_config* out, int32_t cap, int32_t* n_out, mig_rollout_result* res) {
    int rc = MIG_OK;
    int g = guarded([&] {
        if (!p) throw std::invalid_argument("null rollout params");
        CompletionRates c = comp_of(comp, n, ctx);
        if (is_satisfied(c)) {
            ref_par_out(RefPar{}, 0, res);
            rc = emit_plan({}, ctx->services, out, cap, n_out);
            return;
        }
        std::vector<GpuConfig> fast = fast_algo(c, ctx->plan);
        int depth = 2 * (int)fast.size();
        RefPar r = ref_par(ctx->plan, c, p->n_rollouts, p->topk, depth, p->seed, p->id_offset, p->batch, nullptr);
        ref_par_out(r, depth, res);
        std::vector<GpuConfig> ans = fast;
        if (r.best_len >= 0 && (size_t)r.best_len < ans.size()) {
            ans.clear();
            for (int i : r.path) ans.push_back(ctx->plan.pool.items[i].config);
        }
        rc = emit_plan(ans, ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

// Sharding is a device feature of the product (include/migplan_b200.h); the CPU checkers
// plan unsharded, so only the trivial single-rank shard is accepted.
int mig_board_bytes(int32_t n_ranks, int64_t* bytes) {
    return guarded([&] { *bytes = (int64_t)(32 * 2 * (n_ranks > 0 ? n_ranks : 1)); });
}
int mig_board_alloc(int32_t, int32_t, void**, uint8_t*) {
    return guarded([&] { throw std::invalid_argument("exchange boards are device memory (product only)"); });
}
int mig_board_open(int32_t, const uint8_t*, void**) {
    return guarded([&] { throw std::invalid_argument("exchange boards are device memory (product only)"); });
}
int mig_board_free(void*, int32_t) { return MIG_OK; }
int mig_fast_algo_group(mig_ctx* const* ctxs, int32_t n_ctx, const double* comp, int32_t n, mig_config* out,
                        int32_t cap, int32_t* n_out) {
    if (n_ctx == 1 && ctxs) return mig_fast_algo(ctxs[0], comp, n, out, cap, n_out, nullptr, nullptr);
    return guarded([&] { throw std::invalid_argument("sharded greedy is a device feature (product only)"); });
}
int mig_ctx_set_shard(mig_ctx*, int32_t rank, int32_t n_ranks, void* const*, int32_t) {
    return guarded([&] {
        if (n_ranks != 1 || rank != 0) throw std::invalid_argument("sharded greedy is a device feature (product only)");
    });
}
void mig_ga_params_defaults(mig_ga_params* out) {
    GaParams g;
    std::memset(out, 0, sizeof *out);
    out->population = g.population;
    out->erase_fraction = g.erase_fraction;
    out->mutation_pairs = g.mutation_pairs;
    out->stall_rounds = g.stall_rounds;
    out->time_budget_s = g.time_budget_s;
    out->seed = g.seed;
    out->max_rounds = g.max_rounds;
    out->workers = g.workers;
    out->slow = mig_mcts_params{g.slow.budget_iters, g.slow.topk, g.slow.pick_services, g.slow.ucb_c};
}

int mig_completion_of(const mig_ctx* ctx, const mig_config* configs, int32_t n_configs, double* comp_out) {
    return guarded([&] {
        std::vector<GpuConfig> cfgs;
        for (int i = 0; i < n_configs; ++i) cfgs.push_back(from_c(configs[i], ctx->services));
        auto c = completion_of(cfgs, ctx->services, ctx->profiles);
        for (size_t i = 0; i < c.values.size(); ++i) comp_out[i] = c.values[i];
    });
}

int mig_mutate(const mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, const mig_ga_params* params,
               mig_rng* rng, mig_config* child) {
    return guarded([&] {
        Chromosome p;
        for (int i = 0; i < n_gpus; ++i) p.gpus.push_back(from_c(parent[i], ctx->services));
        p.gpu_count = n_gpus;
        Chromosome c = mutate(p, ga_of(params), rng->rng);
        for (size_t i = 0; i < c.gpus.size(); ++i) to_c(c.gpus[i], ctx->services, &child[i]);
    });
}

int mig_crossover(mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, int32_t slow_kind,
                  const mig_ga_params* params, mig_rng* rng, mig_config* child, int32_t cap, int32_t* n_child) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::vector<GpuConfig> gpus;
        for (int i = 0; i < n_gpus; ++i) gpus.push_back(from_c(parent[i], ctx->services));
        Chromosome p = gpus.empty() ? Chromosome{} : evaluate_chromosome(gpus, ctx->plan);
        GaParams gp = ga_of(params);
        FastProcedure fast;
        MctsProcedure slow(gp.slow);
        const OptimizerProcedure& proc = slow_kind == 0 ? static_cast<const OptimizerProcedure&>(fast) : slow;
        Chromosome c = crossover(p, proc, ctx->plan, gp, rng->rng);
        rc = emit_plan(c.gpus, ctx->services, child, cap, n_child);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::function<void(const GaRoundLog&)> lg = nullptr;
        if (log)
            lg = [&](const GaRoundLog& r) {
                log(user, r.round, r.best_gpus, r.best_slack, r.improved ? 1 : 0, r.elapsed_s);
            };
        Deployment dep = two_phase(ctx->services, ctx->profiles, ctx->rules, ga_of(params), lg);
        std::vector<GpuConfig> cfgs;
        for (auto& gpu : dep.gpus) cfgs.push_back(gpu.config);
        rc = emit_plan(cfgs, ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase_parallel(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                           mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::function<void(const GaRoundLog&)> lg = nullptr;
        if (log)
            lg = [&](const GaRoundLog& r) {
                log(user, r.round, r.best_gpus, r.best_slack, r.improved ? 1 : 0, r.elapsed_s);
            };
        rc = emit_plan(two_phase_philox(ctx->plan, ga_of(params), lg), ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase_parallel_mcts(mig_ctx* ctx, const mig_ga_params* params, const mig_rollout_params* slow,
                                mig_config* out, int32_t cap, int32_t* n_out, mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        if (!slow) throw std::invalid_argument("null rollout params");
        if (slow->topk < 1 || slow->topk > 32) throw std::invalid_argument("rollouts: topk must be in [1, 32]");
        std::function<void(const GaRoundLog&)> lg = nullptr;
        if (log)
            lg = [&](const GaRoundLog& r) {
                log(user, r.round, r.best_gpus, r.best_slack, r.improved ? 1 : 0, r.elapsed_s);
            };
        rc = emit_plan(two_phase_philox(ctx->plan, ga_of(params), lg, slow), ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_lower_bound(const mig_ctx* ctx, int32_t* out) {
    return guarded([&] { *out = lower_bound(ctx->services, ctx->profiles); });
}

int mig_baseline(const mig_ctx* ctx, int32_t kind, mig_config* out, int32_t cap, int32_t* n_out) {
    int rc = MIG_OK;
    *n_out = 0;
    int g = guarded([&] {  // the reference's baseline (bench.hpp:42-90), in construction order
        if (kind < 0 || kind > 2) throw std::invalid_argument("baseline kind must be 0, 1 or 2");
        const BaselineKind k = kind == 0 ? BaselineKind::WholeGpu : kind == 1 ? BaselineKind::SevenSlices
                                                                              : BaselineKind::Mix421;
        Deployment dep = baseline(k, ctx->services, ctx->profiles);
        std::vector<GpuConfig> plan;
        for (const auto& d : dep.gpus) plan.push_back(d.config);
        rc = emit_plan(plan, ctx->services, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_brute_force_optimum(mig_ctx* ctx, int32_t cap, int64_t node_budget, mig_config* out, int32_t out_cap,
                            int32_t* n_out, int32_t* found) {
    int rc = MIG_OK;
    *found = 0;
    *n_out = 0;
    int g = guarded([&] {  // the reference's own oracle (bench.hpp:160-219)
        if (cap < 0) throw std::invalid_argument("brute_force_optimum: cap must be >= 0");
        auto dep = brute_force_optimum(ctx->services, ctx->profiles, ctx->rules, cap, node_budget);
        if (!dep) return;
        *found = 1;
        std::vector<GpuConfig> plan;
        for (const auto& g : dep->gpus) plan.push_back(g.config);
        rc = emit_plan(plan, ctx->services, out, out_cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_ctx_stats(const mig_ctx*, mig_stats* out) {
    std::memset(out, 0, sizeof *out);
    return MIG_OK;
}
void mig_ctx_reset_stats(mig_ctx*) {}
int mig_device_cache_release(int32_t) { return MIG_OK; }
int mig_last_plan(mig_config* out, int32_t cap, int32_t* n_out) {
    *n_out = static_cast<int32_t>(g_pending.size());
    if (*n_out > cap) return MIG_ERR_ARGUMENT;
    std::copy(g_pending.begin(), g_pending.end(), out);
    return MIG_OK;
}
int mig_philox_u64(uint64_t seed, uint64_t stream, uint64_t step, int32_t, uint64_t* out) {
    *out = philox64_ref(seed, stream, step);
    return MIG_OK;
}

// The reference keeps no per-step record: the instrumented replica re-runs the last
// mig_fast_algo call's working-set growth (count_rows above).
int mig_ctx_step_rows(const mig_ctx* ctx, int64_t* out, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        std::vector<int64_t> sr;
        if (ctx->have_last) {
            CompletionRates c;
            c.values = ctx->last_comp;
            count_rows(c, ctx->plan, -1, &sr);
        }
        *n_out = static_cast<int32_t>(sr.size());
        for (int32_t i = 0; i < *n_out && i < cap; ++i) out[i] = sr[i];
    });
}

// Reference-arm extras (not in the product header): rows a fast_algo scans, and
// gen_workload (bench.hpp:125-156) so generated workloads come from the reference itself.
/* deployment_to_json(make_deployment(configs)).dump(2) + "\n" — the reference's own output
 * file bytes (io.hpp:44-48,196-208; core.hpp:305-312).  *len = bytes (NUL excluded). */
int mig_ref_deployment_json(mig_ctx* ctx, const mig_config* cfgs, int32_t n, char* buf, int32_t cap, int32_t* len) {
    return guarded([&] {
#ifdef MIGREF_WITH_IO
        std::vector<GpuConfig> v;
        for (int i = 0; i < n; ++i) v.push_back(from_c(cfgs[i], ctx->services));
        std::string out = deployment_to_json(make_deployment(std::move(v))).dump(2) + "\n";
        *len = static_cast<int32_t>(out.size());
        if (static_cast<int32_t>(out.size()) + 1 > cap) throw std::invalid_argument("output capacity too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
#else
        (void)ctx, (void)cfgs, (void)n, (void)buf, (void)cap, (void)len;
        throw std::invalid_argument("built without nlohmann/json (io.hpp)");
#endif
    });
}

/* The reference's transition planner (transition_planner.hpp:658-697) on deployment / SLO /
 * profile FILES read by its own loaders (io.hpp:85-190): plan_to_json(plan).dump(2) + "\n".
 * the planner must consume the product's plan output unchanged. */
int mig_ref_plan_transition(const char* old_dep, const char* new_dep, const char* old_slos, const char* new_slos,
                            const char* profiles, int32_t extra_budget, char* buf, int32_t cap, int32_t* len) {
    return guarded([&] {
#ifdef MIGREF_WITH_IO
        ProfileStore ps = load_profiles(profiles);
        auto os = load_services(old_slos, ps);
        auto ns = load_services(new_slos, ps);
        TransitionPlan plan = plan_transition(load_deployment(old_dep), load_deployment(new_dep), os, ns, ps,
                                              PartitionRuleSet::defaults(), extra_budget);
        std::string out = plan_to_json(plan).dump(2) + "\n";
        *len = static_cast<int32_t>(out.size());
        if (static_cast<int32_t>(out.size()) + 1 > cap) throw std::invalid_argument("output capacity too small");
        std::memcpy(buf, out.c_str(), out.size() + 1);
#else
        (void)old_dep, (void)new_dep, (void)old_slos, (void)new_slos, (void)profiles, (void)extra_budget;
        (void)buf, (void)cap, (void)len;
        throw std::invalid_argument("built without nlohmann/json (io.hpp)");
#endif
    });
}

int mig_ref_count_rows(mig_ctx* ctx, const double* comp, int32_t n, int64_t* rows) {
    return guarded([&] { *rows = count_rows(comp_of(comp, n, ctx), ctx->plan); });
}

// Per-step working-set sizes and per-event extension sizes of the first max_steps steps of
// fast_algo (the instrumented replica above).  Returns the counts written in *n_steps / *n_ext.
int mig_ref_step_rows(mig_ctx* ctx, const double* comp, int32_t n, int64_t max_steps, int64_t* step_rows,
                      int32_t step_cap, int32_t* n_steps, int64_t* ext_rows, int32_t ext_cap, int32_t* n_ext) {
    return guarded([&] {
        std::vector<int64_t> sr, er;
        count_rows(comp_of(comp, n, ctx), ctx->plan, max_steps, &sr, &er);
        *n_steps = static_cast<int32_t>(sr.size());
        *n_ext = static_cast<int32_t>(er.size());
        for (int i = 0; i < *n_steps && i < step_cap; ++i) step_rows[i] = sr[i];
        for (int i = 0; i < *n_ext && i < ext_cap; ++i) ext_rows[i] = er[i];
    });
}

// The reference's own fast_algo (greedy.hpp:95-145), stopped after its first max_steps steps,
// or (steps_after_ext >= 0) that many steps after the step following which maybe_extend
// first fires (greedy.hpp:107-119's trigger, evaluated on the traced completion; -1 = the
// call before step 0).  The trace callback throws a sentinel at the cap, so every step
// reported is the unmodified reference's.  *n_steps = steps traced.
struct PrefixStop {};
int mig_ref_fast_algo_prefix(mig_ctx* ctx, const double* comp, int32_t n, int64_t max_steps,
                             int64_t steps_after_ext, mig_greedy_trace_fn trace, void* user, int32_t* n_steps,
                             int32_t* first_ext_step) {
    int32_t steps = 0;
    int32_t ext_at = -2;
    int rc = guarded([&] {
        CompletionRates c = comp_of(comp, n, ctx);
        const auto& bsu = ctx->plan.pool.best_single_util;
        auto fires = [&](const CompletionRates& cur) {
            for (size_t i = 0; i < cur.values.size(); ++i)
                if (cur.values[i] < 1.0 - kSatisfyEps && 1.0 - cur.values[i] < bsu[i]) return true;
            return false;
        };
        if (fires(c)) ext_at = -1;
        std::function<void(int, const Candidate&, double, const CompletionRates&)> tr =
            [&](int iter, const Candidate& cand, double s, const CompletionRates& cur) {
                mig_candidate mc;
                cand_to_c(cand, ctx->services, &mc);
                if (trace) trace(user, iter, &mc, s, cur.values.data(), static_cast<int32_t>(cur.values.size()));
                ++steps;
                if (ext_at == -2 && fires(cur)) ext_at = iter;
                if (max_steps >= 0 && steps >= max_steps) throw PrefixStop{};
                if (steps_after_ext >= 0 && ext_at != -2 && iter >= ext_at + steps_after_ext) throw PrefixStop{};
            };
        try {
            fast_algo(c, ctx->plan, tr);
        } catch (const PrefixStop&) {
        }
    });
    *first_ext_step = ext_at;
    *n_steps = steps;
    return rc;
}

// Writes n services (id/model as indices into caller-owned string tables is awkward in C,
// so ids follow svc-%03d and models are returned as profile-store indices).
int mig_ref_gen_workload(const mig_model_profile* models, int32_t n_models, int32_t n, int32_t normal, double mu,
                         double sigma, double latency_ms, uint64_t seed, int32_t* model_idx, double* required_rps) {
    return guarded([&] {
        ProfileStore ps = store_of(models, n_models);
        WorkloadSpec w = gen_workload(n, normal ? Distribution::Normal : Distribution::Lognormal, mu, sigma,
                                      latency_ms, seed, ps);
        std::vector<std::string> names;
        for (const auto& [name, p] : ps) names.push_back(name);
        for (int i = 0; i < n; ++i) {
            const auto& s = w.services[i];
            model_idx[i] = -1;
            for (int m = 0; m < n_models; ++m)
                if (s.model_name == models[m].model_name) model_idx[i] = m;
            required_rps[i] = s.required_rps;
        }
    });
}

}  // extern "C"

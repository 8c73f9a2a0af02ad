// capi.cpp — the product's implementation of include/migplan_b200.h.
// Exceptions are mapped to status codes (util.hpp:12-25, migplan.cpp:414-426).
#include <cstring>
#include <string>

#include "engine.hpp"
#include "migplan_b200.h"
#include "philox.cuh"
#include "search.hpp"

using namespace mgb;

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
    } catch (const DeviceError& e) {
        g_err = e.what();
        return MIG_ERR_DEVICE;
    } catch (const ArgumentError& e) {
        g_err = e.what();
        return MIG_ERR_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MIG_ERR_ARGUMENT;
    }
}

Rules rules_of(const mig_rules* r) {
    if (!r) return Rules::defaults();
    Rules out;
    if (r->n_sizes < 0 || r->n_sizes > MIG_MAX_RULE_SIZES || r->n_weights < 0 || r->n_weights > MIG_MAX_RULE_SIZES ||
        r->n_exclusions < 0 || r->n_exclusions > MIG_MAX_EXCLUSIONS)
        throw SchemaError("partition rules out of range");
    for (int i = 0; i < r->n_sizes; ++i) {
        auto& v = out.slot_positions[r->size[i]];
        for (int k = 0; k < r->n_slots[i] && k < MIG_MAX_RULE_SLOTS; ++k) v.push_back(r->slots[i][k]);
        std::sort(v.begin(), v.end());
    }
    for (int i = 0; i < r->n_weights; ++i) out.memory_weight[r->weight_size[i]] = r->weight[i];
    for (int i = 0; i < r->n_exclusions; ++i) {
        int a = r->exclusion[i][0], b = r->exclusion[i][1];
        out.hard_exclusions.insert(a <= b ? std::pair{a, b} : std::pair{b, a});
    }
    out.memory_budget = r->memory_budget;
    return out;
}

std::map<std::string, ModelProfile> profiles_of(const mig_model_profile* models, int n) {
    std::map<std::string, ModelProfile> ps;
    for (int m = 0; m < n; ++m) {
        ModelProfile p;
        p.name = models[m].model_name ? models[m].model_name : "";
        for (int e = 0; e < models[m].n_entries; ++e) {
            const auto& x = models[m].entries[e];
            if (!valid_slices(x.size)) throw SchemaError("invalid instance size " + std::to_string(x.size));
            p.entries[x.size].push_back(ProfileEntry{x.batch, x.throughput_rps, x.p90_ms});
        }
        for (auto& [size, list] : p.entries)
            std::sort(list.begin(), list.end(), [](const ProfileEntry& a, const ProfileEntry& b) { return a.batch < b.batch; });
        validate_profile(p);
        if (ps.count(p.name)) throw SchemaError("duplicate model '" + p.name + "'");
        ps[p.name] = std::move(p);
    }
    return ps;
}

std::vector<Service> services_of(const mig_service* s, int n) {
    std::vector<Service> out;
    for (int i = 0; i < n; ++i)
        out.push_back(Service{s[i].service_id ? s[i].service_id : "", s[i].model_name ? s[i].model_name : "",
                              s[i].required_rps, s[i].max_p90_ms});
    return out;
}

void to_c(const Config& c, mig_config* out) {
    std::memset(out, 0, sizeof *out);
    out->n_instances = c.n;
    for (int k = 0; k < c.n; ++k) out->inst[k] = mig_instance{c.inst[k].slices, c.inst[k].slot, c.inst[k].svc, c.inst[k].batch};
}

Config from_c(const mig_config& c, int n_services) {
    if (c.n_instances < 0 || c.n_instances > MIG_MAX_INSTANCES) throw ArgumentError("bad instance count");
    Config g;
    g.n = c.n_instances;
    for (int k = 0; k < c.n_instances; ++k) {
        const auto& in = c.inst[k];
        if (in.service < 0 || in.service >= n_services)
            throw PlanningError("unknown service index " + std::to_string(in.service));
        g.inst[k] = Model::Inst{in.slices, in.slot, in.service, in.batch};
    }
    return g;
}

thread_local std::vector<mig_config> g_pending;  // a plan that did not fit its caller's buffer

int emit(const std::vector<Config>& plan, mig_config* out, int32_t cap, int32_t* n_out) {
    *n_out = static_cast<int32_t>(plan.size());
    for (size_t i = 0; i < plan.size() && static_cast<int32_t>(i) < cap; ++i) to_c(plan[i], &out[i]);
    if (static_cast<int32_t>(plan.size()) > cap) {
        g_pending.resize(plan.size());
        for (size_t i = 0; i < plan.size(); ++i) to_c(plan[i], &g_pending[i]);
        g_err = "output capacity too small";
        return MIG_ERR_ARGUMENT;
    }
    return MIG_OK;
}

MctsParams mcts_of(const mig_mcts_params* p) {
    MctsParams m;
    if (p) m = MctsParams{p->budget_iters, p->topk, p->pick_services, p->ucb_c};
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

}  // namespace

struct mig_ctx {
    std::unique_ptr<Engine> e;
};
struct mig_rng {
    Rng rng;
};
struct mig_rollout_cache {
    RolloutCache cache;
};

namespace {
std::vector<double> comp_of(const mig_ctx* ctx, const double* comp, int n) {
    if (n != ctx->e->n()) throw PlanningError("completion vector length mismatch");
    return std::vector<double>(comp, comp + n);
}
void cand_of(const Engine& e, uint64_t row, mig_candidate* out) {
    std::memset(out, 0, sizeof *out);
    to_c(e.config_of(row), &out->config);
    const Model& m = e.model();
    int svc[kRowK], pat[kRowK];
    int k = m.members(row, svc, pat);
    out->nnz = k;
    for (int j = 0; j < k; ++j) {
        out->util_idx[j] = svc[j];
        out->util_val[j] = m.U[static_cast<size_t>(svc[j]) * m.PP + pat[j]];
    }
    out->util_sum = m.util_sum(row);
}
}  // namespace

extern "C" {

const char* mig_last_error(void) { return g_err.c_str(); }
int32_t mig_abi_version(void) { return 1; }
const char* mig_impl_name(void) { return "product"; }

void mig_rules_defaults(mig_rules* out) {
    std::memset(out, 0, sizeof *out);
    Rules d = Rules::defaults();
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
        std::vector<Place> ps;
        for (int i = 0; i < n; ++i) ps.push_back(Place{slices[i], slots[i]});
        *legal = is_legal(ps, rules_of(rules)) ? 1 : 0;
    });
}

int mig_enumerate_maximal_partitions(const mig_rules* rules, mig_partition* out, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        auto parts = maximal_partitions(rules_of(rules));
        *n_out = static_cast<int32_t>(parts.size());
        if (*n_out > cap) throw ArgumentError("output capacity too small");
        for (size_t i = 0; i < parts.size(); ++i) {
            std::memset(&out[i], 0, sizeof out[i]);
            out[i].n = static_cast<int32_t>(parts[i].size());
            for (size_t k = 0; k < parts[i].size() && k < MIG_MAX_INSTANCES; ++k) {
                out[i].slices[k] = parts[i][k].slices;
                out[i].slot[k] = parts[i][k].slot;
            }
        }
    });
}

int mig_validate_services(const mig_model_profile* models, int32_t n_models, const mig_service* services,
                          int32_t n_services, int32_t* perm) {
    return guarded([&] {  // core.hpp:151-171
        auto ps = profiles_of(models, n_models);
        auto sv = services_of(services, n_services);
        std::vector<int> idx(n_services);
        for (int i = 0; i < n_services; ++i) idx[i] = i;
        std::sort(idx.begin(), idx.end(), [&](int a, int b) { return sv[a].id < sv[b].id; });
        for (int i = 0; i + 1 < n_services; ++i)
            if (sv[idx[i]].id == sv[idx[i + 1]].id) throw SchemaError("duplicate service id '" + sv[idx[i]].id + "'");
        for (int i : idx) {
            const auto& s = sv[i];
            if (s.id.empty()) throw SchemaError("service with empty id");
            if (s.req <= 0.0) throw PlanningError("service '" + s.id + "': required throughput must be positive");
            if (s.p90 <= 0.0) throw PlanningError("service '" + s.id + "': latency ceiling must be positive");
            auto it = ps.find(s.model);
            if (it == ps.end()) throw PlanningError("no profile for model '" + s.model + "'");
            bool feasible = false;
            for (const auto& [size, list] : it->second.entries)
                for (const auto& e : list)
                    if (valid_slices(size) && e.p90 <= s.p90) feasible = true;
            if (!feasible)
                throw PlanningError("service '" + s.id + "' is unschedulable: no (size, batch) of model '" + s.model +
                                    "' meets p90 <= " + std::to_string(s.p90) + " ms");
        }
        for (int i = 0; i < n_services; ++i) perm[i] = idx[i];
    });
}

int mig_ctx_create(const mig_rules* rules, const mig_model_profile* models, int32_t n_models,
                   const mig_service* services, int32_t n_services, int32_t max_mix, int32_t device, mig_ctx** out) {
    return guarded([&] {
        if (!out) throw ArgumentError("null output");
        auto c = std::make_unique<mig_ctx>();
        c->e = std::make_unique<Engine>(rules_of(rules), profiles_of(models, n_models), services_of(services, n_services),
                                        max_mix, device);
        *out = c.release();
    });
}

void mig_ctx_destroy(mig_ctx* ctx) { delete ctx; }
int32_t mig_ctx_n_services(const mig_ctx* ctx) { return ctx->e->n(); }

int mig_pool_size(const mig_ctx* ctx, int64_t* out) {
    *out = ctx->e->pool_size();
    return MIG_OK;
}

int mig_pool_candidate(const mig_ctx* ctx, int64_t idx, mig_candidate* out) {
    return guarded([&] {
        if (idx < 0 || idx >= ctx->e->pool_size()) throw ArgumentError("pool index out of range");
        cand_of(*ctx->e, ctx->e->base_rows()[idx], out);
    });
}

int mig_pool_best_single_util(const mig_ctx* ctx, double* out) {
    for (int i = 0; i < ctx->e->n(); ++i) out[i] = ctx->e->model().best_single[i];
    return MIG_OK;
}

int mig_score(const mig_ctx* ctx, int64_t idx, const double* comp, int32_t n, double* out) {
    return guarded([&] {
        if (idx < 0 || idx >= ctx->e->pool_size()) throw ArgumentError("pool index out of range");
        auto c = comp_of(ctx, comp, n);
        *out = ctx->e->model().score(ctx->e->base_rows()[idx], c.data());
    });
}

int mig_topk_candidates(mig_ctx* ctx, const double* comp, int32_t n, int32_t k, const int64_t* from, int64_t n_from,
                        int64_t* out_idx, int32_t* n_out) {
    return guarded([&] {
        auto c = comp_of(ctx, comp, n);
        std::vector<long long> idx;
        if (from && n_from >= 0) {
            for (int64_t i = 0; i < n_from; ++i) {
                if (from[i] < 0 || from[i] >= ctx->e->pool_size()) throw ArgumentError("pool index out of range");
                idx.push_back(from[i]);
            }
        }
        std::vector<long long> top;
        if (from && n_from == 0) top = {};
        else top = ctx->e->topk(c, k, (from && n_from >= 0) ? &idx : nullptr, nullptr);
        *n_out = static_cast<int32_t>(top.size());
        for (size_t i = 0; i < top.size(); ++i) out_idx[i] = top[i];
    });
}

int mig_fast_algo(mig_ctx* ctx, const double* comp, int32_t n, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_greedy_trace_fn trace, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        auto c = comp_of(ctx, comp, n);
        std::vector<uint64_t> rows;
        std::vector<double> scores;
        ctx->e->fast_algo(c, rows, scores);
        std::vector<Config> plan;
        const Model& m = ctx->e->model();
        for (size_t i = 0; i < rows.size(); ++i) {
            plan.push_back(ctx->e->config_of(rows[i]));
            if (trace) {  // replay greedy.hpp:139-140: comp after the pick, then trace
                int svc[kRowK], pat[kRowK];
                int k = m.members(rows[i], svc, pat);
                for (int j = 0; j < k; ++j) c[svc[j]] = c[svc[j]] + m.U[static_cast<size_t>(svc[j]) * m.PP + pat[j]];
                mig_candidate mc;
                cand_of(*ctx->e, rows[i], &mc);
                trace(user, static_cast<int32_t>(i), &mc, scores[i], c.data(), n);
            }
        }
        rc = emit(plan, out, cap, n_out);
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
        auto top = expand_children(*ctx->e, comp_of(ctx, comp, n), mcts_of(params), rng->rng);
        *n_children = static_cast<int32_t>(top.size());
        if (*n_children > cap) throw ArgumentError("output capacity too small");
        for (size_t i = 0; i < top.size(); ++i) children[i] = top[i];
    });
}

int mig_rollout_cache_create(mig_rollout_cache** out) {
    *out = new mig_rollout_cache{};
    return MIG_OK;
}
void mig_rollout_cache_destroy(mig_rollout_cache* cache) { delete cache; }
int32_t mig_rollout_cache_builds(const mig_rollout_cache* cache) { return cache->cache.builds; }

int mig_rollout(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params, mig_rollout_cache* cache,
                mig_rng* rng, int32_t max_depth, int64_t* picked, int32_t cap, int32_t* steps) {
    return guarded([&] {
        std::vector<long long> p;
        *steps = rollout(*ctx->e, comp_of(ctx, comp, n), mcts_of(params), cache->cache, rng->rng, max_depth,
                         picked ? &p : nullptr);
        if (picked) {
            if (static_cast<int32_t>(p.size()) > cap) throw ArgumentError("output capacity too small");
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
        auto plan = mcts_solve(*ctx->e, comp_of(ctx, comp, n), mcts_of(params), seed, tr);
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
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

}  // extern "C"

namespace {
// mig_rollouts body: resolves max_depth < 0 through the device greedy (mcts.hpp:152-155).
RolloutResult run_rollouts(mig_ctx* ctx, const std::vector<double>& c, const mig_rollout_params* p, int32_t* lengths,
                           int* depth_used, int* fast_len) {
    if (!p) throw ArgumentError("null rollout params");
    int depth = p->max_depth;
    *fast_len = -1;
    if (depth < 0) {
        std::vector<Config> ref = fast_plan(*ctx->e, c);
        *fast_len = static_cast<int>(ref.size());
        depth = 2 * *fast_len;
    }
    *depth_used = depth;
    RolloutResult r = ctx->e->rollouts(c, p->n_rollouts, p->topk, depth, p->seed, p->id_offset, p->batch,
                                       p->table_log2, lengths);
    // every pool build is one top-K over the whole base pool (mcts.hpp:129-133)
    ctx->e->stats.topk_calls += r.keys;
    ctx->e->stats.topk_rows += r.keys * ctx->e->pool_size();
    return r;
}
void result_of(const RolloutResult& r, int depth, mig_rollout_result* out) {
    if (!out) return;
    out->best_len = r.best_len;
    out->max_depth = depth;
    out->best_id = r.best_id;
    out->completed = r.completed;
    out->capped = r.capped;
    out->failed = r.failed;
    out->steps = r.steps;
    out->keys = r.keys;
    out->rounds = r.rounds;
    out->path_len = static_cast<int32_t>(r.path.size());
    out->device_ms = r.ms;
}
}  // namespace

extern "C" {

int mig_rollouts(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* params, int32_t* lengths,
                 int64_t* best_path, int32_t cap, mig_rollout_result* out) {
    return guarded([&] {
        int depth = 0, fl = 0;
        RolloutResult r = run_rollouts(ctx, comp_of(ctx, comp, n), params, lengths, &depth, &fl);
        if (best_path) {
            if (static_cast<int32_t>(r.path.size()) > cap) throw ArgumentError("output capacity too small");
            for (size_t i = 0; i < r.path.size(); ++i) best_path[i] = r.path[i];
        }
        result_of(r, depth, out);
    });
}

int mig_mcts_solve_parallel(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* params,
                            mig_config* out, int32_t cap, int32_t* n_out, mig_rollout_result* result) {
    int rc = MIG_OK;
    int g = guarded([&] {
        auto c = comp_of(ctx, comp, n);
        if (satisfied(c)) {  // mcts.hpp:151
            result_of(RolloutResult{}, 0, result);
            rc = emit({}, out, cap, n_out);
            return;
        }
        std::vector<Config> fast_ref = fast_plan(*ctx->e, c);
        mig_rollout_params p = *params;
        p.max_depth = 2 * static_cast<int32_t>(fast_ref.size());
        int depth = 0, fl = 0;
        RolloutResult r = run_rollouts(ctx, c, &p, nullptr, &depth, &fl);
        result_of(r, depth, result);
        std::vector<Config> answer = std::move(fast_ref);
        if (r.best_len >= 0 && static_cast<size_t>(r.best_len) < answer.size()) {
            answer.clear();
            for (long long idx : r.path) answer.push_back(ctx->e->config_of(ctx->e->base_rows()[idx]));
        }
        rc = emit(answer, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_board_bytes(int32_t n_ranks, int64_t* bytes) {
    return guarded([&] { *bytes = static_cast<int64_t>(board_bytes(n_ranks)); });
}
int mig_board_alloc(int32_t device, int32_t n_ranks, void** board, uint8_t* ipc_handle) {
    return guarded([&] { *board = board_alloc(device, n_ranks, ipc_handle); });
}
int mig_board_open(int32_t device, const uint8_t* ipc_handle, void** board) {
    return guarded([&] { *board = board_open(device, ipc_handle); });
}
int mig_philox_u64(uint64_t seed, uint64_t stream, uint64_t step, int32_t on_device, uint64_t* out) {
    return guarded([&] {
        if (on_device) {
            device_info(0);  // a CUDA device or MIG_ERR_DEVICE
            *out = philox_on_device(0, seed, stream, step);
        } else {
            *out = philox_u64(seed, stream, step);
        }
    });
}
int mig_last_plan(mig_config* out, int32_t cap, int32_t* n_out) {
    *n_out = static_cast<int32_t>(g_pending.size());
    if (*n_out > cap) return MIG_ERR_ARGUMENT;
    std::copy(g_pending.begin(), g_pending.end(), out);
    return MIG_OK;
}
int mig_device_cache_release(int32_t device) {
    return guarded([&] { release_device_cache(device); });
}
int mig_board_free(void* board, int32_t opened) {
    return guarded([&] { board_close(board, opened != 0); });
}
int mig_ctx_set_shard(mig_ctx* ctx, int32_t rank, int32_t n_ranks, void* const* boards, int32_t max_ctas) {
    return guarded([&] {
        std::vector<void*> b;
        if (n_ranks > 1) {
            if (!boards) throw ArgumentError("set_shard: null boards");
            b.assign(boards, boards + n_ranks);
        }
        ctx->e->set_shard(rank, n_ranks, b, max_ctas);
    });
}

int mig_fast_algo_group(mig_ctx* const* ctxs, int32_t n_ctx, const double* comp, int32_t n, mig_config* out,
                        int32_t cap, int32_t* n_out) {
    int rc = MIG_OK;
    int g = guarded([&] {
        if (!ctxs || n_ctx < 1) throw ArgumentError("fast_algo_group: no contexts");
        std::vector<Engine*> es;
        for (int i = 0; i < n_ctx; ++i) es.push_back(ctxs[i]->e.get());
        auto c = comp_of(ctxs[0], comp, n);
        std::vector<uint64_t> rows;
        std::vector<double> scores;
        Engine::fast_algo_group(es, c, rows, scores);
        std::vector<Config> plan;
        for (uint64_t r : rows) plan.push_back(es[0]->config_of(r));
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_completion_of(const mig_ctx* ctx, const mig_config* configs, int32_t n_configs, double* comp_out) {
    return guarded([&] {
        std::vector<Config> cfgs;
        for (int i = 0; i < n_configs; ++i) cfgs.push_back(from_c(configs[i], ctx->e->n()));
        auto c = ctx->e->completion_of(cfgs);
        for (size_t i = 0; i < c.size(); ++i) comp_out[i] = c[i];
    });
}

int mig_mutate(const mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, const mig_ga_params* params, mig_rng* rng,
               mig_config* child) {
    return guarded([&] {
        Chromosome p;
        for (int i = 0; i < n_gpus; ++i) p.gpus.push_back(from_c(parent[i], ctx->e->n()));
        p.gpu_count = n_gpus;
        Chromosome c = mutate(p, ga_of(params), rng->rng);
        for (size_t i = 0; i < c.gpus.size(); ++i) to_c(c.gpus[i], &child[i]);
    });
}

int mig_crossover(mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, int32_t slow_kind,
                  const mig_ga_params* params, mig_rng* rng, mig_config* child, int32_t cap, int32_t* n_child) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::vector<Config> gpus;
        for (int i = 0; i < n_gpus; ++i) gpus.push_back(from_c(parent[i], ctx->e->n()));
        Chromosome p = gpus.empty() ? Chromosome{} : evaluate_chromosome(gpus, *ctx->e);
        GaParams gp = ga_of(params);
        FastProc fast;
        MctsProc slow(gp.slow);
        const Procedure& proc = slow_kind == 0 ? static_cast<const Procedure&>(fast) : slow;
        Chromosome c = crossover(p, proc, *ctx->e, gp, rng->rng);
        rc = emit(c.gpus, child, cap, n_child);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::function<void(int, int, double, bool, double)> lg = nullptr;
        if (log) lg = [&](int r, int b, double s, bool imp, double el) { log(user, r, b, s, imp ? 1 : 0, el); };
        auto plan = two_phase(*ctx->e, ga_of(params), lg);
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase_parallel(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        std::function<void(int, int, double, bool, double)> lg = nullptr;
        if (log) lg = [&](int r, int b, double s, bool imp, double el) { log(user, r, b, s, imp ? 1 : 0, el); };
        auto plan = two_phase_parallel(*ctx->e, ga_of(params), lg);
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_two_phase_parallel_mcts(mig_ctx* ctx, const mig_ga_params* params, const mig_rollout_params* slow,
                                mig_config* out, int32_t cap, int32_t* n_out, mig_ga_log_fn log, void* user) {
    int rc = MIG_OK;
    int g = guarded([&] {
        if (!slow) throw ArgumentError("null rollout params");
        if (slow->topk < 1 || slow->topk > 32) throw ArgumentError("rollouts: topk must be in [1, 32]");
        std::function<void(int, int, double, bool, double)> lg = nullptr;
        if (log) lg = [&](int r, int b, double s, bool imp, double el) { log(user, r, b, s, imp ? 1 : 0, el); };
        RolloutRefill rf;
        rf.n_rollouts = slow->n_rollouts;
        rf.topk = slow->topk;
        rf.id_offset = slow->id_offset;
        rf.batch = slow->batch;
        rf.table_log2 = slow->table_log2;
        auto plan = two_phase_parallel(*ctx->e, ga_of(params), lg, &rf);
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_lower_bound(const mig_ctx* ctx, int32_t* out) {
    return guarded([&] {  // bench.hpp:93-108 over every constructible size {1,2,3,4,7}
        const Model& m = ctx->e->model();
        if (m.n == 0) {
            *out = 0;
            return;
        }
        double total = 0.0;
        for (int i = 0; i < m.n; ++i) {
            const auto& prof = ctx->e->profiles().at(m.services[i].model);
            double best = 0.0;
            for (int size : {1, 2, 3, 4, 7}) {
                auto it = prof.entries.find(size);
                if (it == prof.entries.end()) continue;
                const ProfileEntry* sel = nullptr;
                for (const auto& pe : it->second)
                    if (pe.p90 <= m.services[i].p90) sel = &pe;
                if (sel) best = std::max(best, sel->thr / size);
            }
            if (best <= 0.0) throw PlanningError("service '" + m.services[i].id + "' has no feasible instance size");
            total += m.services[i].req / best;
        }
        *out = static_cast<int32_t>(std::ceil(total / 7.0 - 1e-9));
    });
}

int mig_baseline(const mig_ctx* ctx, int32_t kind, mig_config* out, int32_t cap, int32_t* n_out) {
    int rc = MIG_OK;
    *n_out = 0;
    int g = guarded([&] {  // bench.hpp:42-90
        if (kind < 0 || kind > 2) throw ArgumentError("baseline kind must be 0 (7/7), 1 (7x1/7) or 2 (mix)");
        const Model& m = ctx->e->model();
        auto entry = [&](int i, int size) -> std::pair<int, double> {  // entry_or_throw, bench.hpp:26-31
            const auto& prof = ctx->e->profiles().at(m.services[i].model);
            const ProfileEntry* sel = nullptr;
            auto it = prof.entries.find(size);
            if (it != prof.entries.end())
                for (const auto& pe : it->second)
                    if (pe.p90 <= m.services[i].p90) sel = &pe;  // select_entry: largest feasible batch
            if (!sel)
                throw PlanningError("service '" + m.services[i].id + "' is infeasible on a " + std::to_string(size) +
                                    "/7 instance under its latency ceiling");
            return {sel->batch, sel->thr};
        };
        auto count = [](double need, double per) { return static_cast<int>(std::ceil(need / per - 1e-9)); };
        std::vector<Config> plan;
        auto one = [](std::initializer_list<Model::Inst> in) {
            Config c;
            c.n = 0;
            for (const auto& x : in) c.inst[c.n++] = x;
            return c;
        };
        if (kind == 0) {
            for (int i = 0; i < m.n; ++i) {
                auto [b, t] = entry(i, 7);
                for (int k = count(m.services[i].req, t); k > 0; --k) plan.push_back(one({{7, 0, i, b}}));
            }
        } else if (kind == 1) {
            Config cur;
            cur.n = 0;
            for (int i = 0; i < m.n; ++i) {
                auto [b, t] = entry(i, 1);
                for (int k = count(m.services[i].req, t); k > 0; --k) {
                    cur.inst[cur.n] = Model::Inst{1, cur.n, i, b};
                    if (++cur.n == 7) {
                        plan.push_back(cur);
                        cur.n = 0;
                    }
                }
            }
            if (cur.n) plan.push_back(cur);
        } else {
            for (int i = 0; i < m.n; ++i) {
                auto [b4, t4] = entry(i, 4);
                auto [b2, t2] = entry(i, 2);
                auto [b1, t1] = entry(i, 1);
                for (int k = count(m.services[i].req, t4 + t2 + t1); k > 0; --k)
                    plan.push_back(one({{4, 0, i, b4}, {2, 4, i, b2}, {1, 6, i, b1}}));
            }
        }
        rc = emit(plan, out, cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_brute_force_optimum(mig_ctx* ctx, int32_t cap, int64_t node_budget, mig_config* out, int32_t out_cap,
                            int32_t* n_out, int32_t* found) {
    int rc = MIG_OK;
    *found = 0;
    *n_out = 0;
    int g = guarded([&] {
        if (cap < 0) throw ArgumentError("brute_force_optimum: cap must be >= 0");
        bool f = false;
        auto plan = ctx->e->brute_force(cap, node_budget, f);
        *found = f ? 1 : 0;
        rc = emit(plan, out, out_cap, n_out);
    });
    return g != MIG_OK ? g : rc;
}

int mig_ctx_stats(const mig_ctx* ctx, mig_stats* out) {
    std::memset(out, 0, sizeof *out);
    const Stats& s = ctx->e->stats;
    out->greedy_rows = s.greedy_rows.load();
    out->topk_rows = s.topk_rows.load();
    out->rows_scored = out->greedy_rows + out->topk_rows;
    out->greedy_calls = s.greedy_calls.load();
    out->topk_calls = s.topk_calls.load();
    out->greedy_steps = s.greedy_steps.load();
    out->ext_events = s.ext_events.load();
    out->ext_rows = s.ext_rows.load();
    out->kernel_launches = s.launches.load();
    out->h2d_bytes = s.h2d.load();
    out->d2h_bytes = s.d2h.load();
    out->greedy_ms = s.greedy_ns.load() / 1e6;
    out->topk_ms = s.topk_ns.load() / 1e6;
    for (int k = 0; k < 5; ++k) out->phase_ms[k] = s.phase_ns[k].load() / 1e6;
    out->rollout_steps = s.rollout_steps.load();
    out->rollout_calls = s.rollout_calls.load();
    out->rollout_ms = s.rollout_ns.load() / 1e6;
    out->mcts_ms = s.mcts_ns.load() / 1e6;
    out->mcts_launches = s.mcts_launches.load();
    out->mcts_rows = s.mcts_rows.load();
    out->mcts_topk_calls = s.mcts_topk_calls.load();
    return MIG_OK;
}

void mig_ctx_reset_stats(mig_ctx* ctx) { ctx->e->stats.reset(); }

int mig_ctx_step_rows(const mig_ctx* ctx, int64_t* out, int32_t cap, int32_t* n_out) {
    return guarded([&] {
        auto v = ctx->e->last_step_rows();
        *n_out = static_cast<int32_t>(v.size());
        for (int32_t i = 0; i < *n_out && i < cap; ++i) out[i] = v[i];
    });
}

}  // extern "C"

// migplan_b200_procedures.hpp — drop-in GPU procedures for a codebase that uses the
// reference `migplan` headers (proj/include/migplan/*.hpp).
//
// Header-only bridge over the C-ABI (migplan_b200.h): it converts the reference's own
// types (ServiceSpec, ProfileStore, PartitionRuleSet, CompletionRates, GpuConfig) to the
// ABI structs and back, and rethrows ABI status codes as the reference's exceptions
// (util.hpp:12-25).  Usage inside the reference code base:
//
//     #include "migplan/ga.hpp"
//     #include "migplan_b200_procedures.hpp"
//     migplan::b200::GpuContext gctx(ctx);                  // mirrors make_plan_context
//     auto plan = gctx.fast_algo(zero_completion(n));       // == migplan::fast_algo(...)
//     migplan::b200::GpuFastProcedure fast(gctx);           // an OptimizerProcedure
//     migplan::b200::GpuMctsProcedure slow(gctx, params);   // an OptimizerProcedure
//     Chromosome child = crossover(parent, slow, ctx, ga_params, rng);  // ga.hpp:51
//
// Link with -lmigplan_b200 (paper_2109_11067_b200/_native/libmigplan_b200.so).
#pragma once

#include <string>
#include <vector>

#include "migplan/greedy.hpp"
#include "migplan/mcts.hpp"
#include "migplan_b200.h"

namespace migplan::b200 {

inline void check(int rc) {
    if (rc == MIG_OK) return;
    std::string msg = mig_last_error();
    if (rc == MIG_ERR_PLANNING) throw PlanningError(msg);
    if (rc == MIG_ERR_SCHEMA) throw SchemaError(msg);
    throw std::runtime_error("migplan_b200: " + msg);
}

// A device-resident PlanContext (greedy.hpp:16-31): same services (id-sorted), same
// profile store and rules; the candidate pool lives in HBM.
class GpuContext {
  public:
    explicit GpuContext(const PlanContext& ctx, int max_mix = 2, int device = 0) : services_(ctx.services) {
        mig_rules r{};
        for (const auto& [size, slots] : ctx.rules.slot_positions) {
            int i = r.n_sizes++;
            r.size[i] = size;
            r.n_slots[i] = static_cast<int32_t>(slots.size());
            for (size_t k = 0; k < slots.size() && k < MIG_MAX_RULE_SLOTS; ++k) r.slots[i][k] = slots[k];
        }
        for (const auto& [size, w] : ctx.rules.memory_weight) {
            int i = r.n_weights++;
            r.weight_size[i] = size;
            r.weight[i] = w;
        }
        for (const auto& [a, b] : ctx.rules.hard_exclusions) {
            int i = r.n_exclusions++;
            r.exclusion[i][0] = a;
            r.exclusion[i][1] = b;
        }
        r.memory_budget = ctx.rules.memory_budget;
        std::vector<std::vector<mig_profile_entry>> entries;
        std::vector<mig_model_profile> models;
        for (const auto& [name, prof] : *ctx.profiles) {
            std::vector<mig_profile_entry> e;
            for (const auto& [size, list] : prof.entries)
                for (const auto& pe : list) e.push_back(mig_profile_entry{size, pe.batch, pe.throughput_rps, pe.p90_ms});
            entries.push_back(std::move(e));
        }
        size_t m = 0;
        for (const auto& [name, prof] : *ctx.profiles) {
            models.push_back(mig_model_profile{name.c_str(), entries[m].data(), static_cast<int32_t>(entries[m].size())});
            ++m;
        }
        std::vector<mig_service> svcs;
        for (const auto& s : services_)
            svcs.push_back(mig_service{s.service_id.c_str(), s.model_name.c_str(), s.required_rps, s.max_p90_ms});
        check(mig_ctx_create(&r, models.data(), static_cast<int32_t>(models.size()), svcs.data(),
                             static_cast<int32_t>(svcs.size()), max_mix, device, &ctx_));
    }
    ~GpuContext() { mig_ctx_destroy(ctx_); }
    GpuContext(const GpuContext&) = delete;
    GpuContext& operator=(const GpuContext&) = delete;

    mig_ctx* raw() const { return ctx_; }

    GpuConfig to_config(const mig_config& c) const {
        GpuConfig g;
        for (int k = 0; k < c.n_instances; ++k)
            g.instances.push_back(AssignedInstance{Placement{c.inst[k].slices, c.inst[k].slot},
                                                   services_[c.inst[k].service].service_id, c.inst[k].batch});
        return g;
    }

    template <class Call>
    std::vector<GpuConfig> plan(Call&& call) const {
        std::vector<mig_config> buf(4096);
        int32_t n = 0;
        int rc = call(buf.data(), static_cast<int32_t>(buf.size()), &n);
        if (rc == MIG_ERR_ARGUMENT && n > static_cast<int32_t>(buf.size())) {
            buf.resize(n);
            rc = call(buf.data(), n, &n);
        }
        check(rc);
        std::vector<GpuConfig> out;
        for (int i = 0; i < n; ++i) out.push_back(to_config(buf[i]));
        return out;
    }

    // fast_algo(comp, ctx), greedy.hpp:95-145 — bit-exact, one persistent B200 kernel.
    std::vector<GpuConfig> fast_algo(const CompletionRates& comp) const {
        return plan([&](mig_config* o, int32_t cap, int32_t* n) {
            return mig_fast_algo(ctx_, comp.values.data(), static_cast<int32_t>(comp.values.size()), o, cap, n,
                                 nullptr, nullptr);
        });
    }

    // mcts_solve(comp, ctx, params, seed), mcts.hpp:148-252 — identical plan under a matched seed.
    std::vector<GpuConfig> mcts_solve(const CompletionRates& comp, const MctsParams& p, uint64_t seed) const {
        mig_mcts_params mp{p.budget_iters, p.topk, p.pick_services, p.ucb_c};
        return plan([&](mig_config* o, int32_t cap, int32_t* n) {
            return mig_mcts_solve(ctx_, comp.values.data(), static_cast<int32_t>(comp.values.size()), &mp, seed, o,
                                  cap, n, nullptr, nullptr);
        });
    }

  private:
    std::vector<ServiceSpec> services_;
    mig_ctx* ctx_ = nullptr;
};

// OptimizerProcedure plugins (greedy.hpp:155-164, mcts.hpp:254-260) backed by the B200.
struct GpuFastProcedure final : OptimizerProcedure {
    explicit GpuFastProcedure(const GpuContext& g) : gpu(g) {}
    std::vector<GpuConfig> solve(const CompletionRates& comp, const PlanContext&, Rng&) const override {
        return gpu.fast_algo(comp);
    }
    const GpuContext& gpu;
};

struct GpuMctsProcedure final : OptimizerProcedure {
    GpuMctsProcedure(const GpuContext& g, MctsParams p = {}) : gpu(g), params(p) {}
    std::vector<GpuConfig> solve(const CompletionRates& comp, const PlanContext&, Rng& rng) const override {
        return gpu.mcts_solve(comp, params, rng());  // same seed draw as MctsProcedure (mcts.hpp:258)
    }
    const GpuContext& gpu;
    MctsParams params;
};

}  // namespace migplan::b200

/*
 * migplan_b200.h — the C-ABI boundary of the B200-native MIG-SERVING optimizer.
 *
 * The reference (the headers under /root/reference/proj/include/migplan, header-only C++20) has
 * no FFI of its own; its public surface is C++ free functions and the
 * `OptimizerProcedure` plugin class.  Every entry point below is the plain-C
 * rendering of one of those functions (cited per declaration), with
 *   - plain pointers and sizes, no C++ or torch types,
 *   - C++ exceptions mapped onto status codes (util.hpp:12-25, migplan.cpp:414-426),
 *   - service indices instead of service-id strings (index i == services[i],
 *     services sorted by id exactly as `validate_services` leaves them,
 *     core.hpp:151-171).
 *
 * Three libraries implement this header:
 *   libmigplan_b200.so  — the product (CUDA sm_100a kernels + native runtime),
 *   oracle/liboracle.so — CPU restatement used only by tests/bench as checker,
 *   oracle/_ref/libmigref.so — the unmodified reference headers behind a shim.
 */
#ifndef MIGPLAN_B200_H
#define MIGPLAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (util.hpp:12-25; CLI exit codes migplan.cpp:414-426) ---- */
#define MIG_OK 0
#define MIG_ERR_PLANNING 1 /* migplan::PlanningError  */
#define MIG_ERR_SCHEMA 2   /* migplan::SchemaError    */
#define MIG_ERR_DEVICE 3   /* CUDA / NCCL failure     */
#define MIG_ERR_ARGUMENT 4 /* null pointer, too-small output capacity, limits */

#define MIG_MAX_INSTANCES 7 /* a GPU has 7 compute slots (core.hpp:126)        */
#define MIG_MAX_RULE_SIZES 8
#define MIG_MAX_RULE_SLOTS 16
#define MIG_MAX_EXCLUSIONS 16

/* Thread-local message of the last failing call (the exception's what()). */
const char* mig_last_error(void);
int32_t mig_abi_version(void);
/* "product" / "oracle" / "reference": which implementation this library is. */
const char* mig_impl_name(void);

/* ---- L1/L2 domain types (core.hpp:57-78,113-118,174-200; mig_rules.hpp:15-34) ---- */

typedef struct mig_profile_entry { /* ProfileEntry, core.hpp:57-61 (+ its size key) */
    int32_t size;
    int32_t batch;
    double throughput_rps;
    double p90_ms;
} mig_profile_entry;

typedef struct mig_model_profile { /* ModelProfile, core.hpp:64-76 */
    const char* model_name;
    const mig_profile_entry* entries; /* any order; grouped by size, sorted by batch inside */
    int32_t n_entries;
} mig_model_profile;

typedef struct mig_service { /* ServiceSpec, core.hpp:113-118 */
    const char* service_id;
    const char* model_name;
    double required_rps;
    double max_p90_ms;
} mig_service;

typedef struct mig_rules { /* PartitionRuleSet, mig_rules.hpp:15-34 */
    int32_t n_sizes;                                    /* slot_positions entries   */
    int32_t size[MIG_MAX_RULE_SIZES];
    int32_t n_slots[MIG_MAX_RULE_SIZES];
    int32_t slots[MIG_MAX_RULE_SIZES][MIG_MAX_RULE_SLOTS];
    int32_t n_weights;                                  /* memory_weight entries    */
    int32_t weight_size[MIG_MAX_RULE_SIZES];
    int32_t weight[MIG_MAX_RULE_SIZES];
    int32_t n_exclusions;                               /* hard_exclusions pairs    */
    int32_t exclusion[MIG_MAX_EXCLUSIONS][2];
    int32_t memory_budget;
} mig_rules;

typedef struct mig_instance { /* AssignedInstance, core.hpp:174-180 */
    int32_t slices;
    int32_t slot;
    int32_t service; /* index into the context's services */
    int32_t batch;
} mig_instance;

typedef struct mig_config { /* GpuConfig (normalized: sorted by (slices, slot)), core.hpp:184-200 */
    int32_t n_instances;
    mig_instance inst[MIG_MAX_INSTANCES];
} mig_config;

typedef struct mig_candidate { /* Candidate, config_enum.hpp:13-18 */
    mig_config config;
    int32_t nnz;                          /* util entries, ascending service index */
    int32_t util_idx[MIG_MAX_INSTANCES];
    double util_val[MIG_MAX_INSTANCES];
    double util_sum;
} mig_candidate;

typedef struct mig_partition { /* LegalPartition, mig_rules.hpp:62-65 */
    int32_t n;
    int32_t slices[MIG_MAX_INSTANCES];
    int32_t slot[MIG_MAX_INSTANCES];
} mig_partition;

void mig_rules_defaults(mig_rules* out); /* PartitionRuleSet::defaults, mig_rules.hpp:21-33 */

/* is_legal_partition, mig_rules.hpp:38-59 */
int mig_is_legal_partition(const mig_rules* rules, const int32_t* slices, const int32_t* slots, int32_t n,
                           int32_t* legal);
/* enumerate_maximal_partitions, mig_rules.hpp:116-135 (18 under defaults) */
int mig_enumerate_maximal_partitions(const mig_rules* rules, mig_partition* out, int32_t cap, int32_t* n_out);

/* validate_services, core.hpp:151-171: writes the id-sorted order into perm[n]
 * (perm[i] = caller index of the i-th service) and throws the reference's errors. */
int mig_validate_services(const mig_model_profile* models, int32_t n_models, const mig_service* services,
                          int32_t n_services, int32_t* perm);

/* ---- PlanContext (greedy.hpp:16-31) ---- */
typedef struct mig_ctx mig_ctx;

/* make_plan_context(services, profiles, rules, max_mix), greedy.hpp:23-31.
 * `services` must already be sorted by id (as validate_services leaves them).
 * `device` selects the CUDA device (product only; ignored by CPU libraries). */
int mig_ctx_create(const mig_rules* rules, const mig_model_profile* models, int32_t n_models,
                   const mig_service* services, int32_t n_services, int32_t max_mix, int32_t device,
                   mig_ctx** out);
void mig_ctx_destroy(mig_ctx* ctx);
int32_t mig_ctx_n_services(const mig_ctx* ctx);

/* CandidatePool view (config_enum.hpp:20-32).  Pool order is implementation
 * defined; every optimizer result is a function of the pool as a SET because
 * the preference order (greedy.hpp:63-67) is total. */
int mig_pool_size(const mig_ctx* ctx, int64_t* out);
int mig_pool_candidate(const mig_ctx* ctx, int64_t idx, mig_candidate* out);
int mig_pool_best_single_util(const mig_ctx* ctx, double* out /* n_services */);

/* score(const Candidate&, const CompletionRates&), greedy.hpp:36-43 */
int mig_score(const mig_ctx* ctx, int64_t idx, const double* comp, int32_t n, double* out);

/* detail::topk_candidates, mcts.hpp:56-76.  from == NULL (n_from < 0): whole base pool. */
int mig_topk_candidates(mig_ctx* ctx, const double* comp, int32_t n, int32_t k, const int64_t* from,
                        int64_t n_from, int64_t* out_idx, int32_t* n_out);

/* ---- fast algorithm (greedy.hpp:95-145) ----
 * trace(iter, chosen, best_score, comp-after-pick) exactly as greedy.hpp:140.
 * *n_out is always the plan length; MIG_ERR_ARGUMENT when it exceeds cap. */
typedef void (*mig_greedy_trace_fn)(void* user, int32_t iter, const mig_candidate* chosen, double score,
                                    const double* comp, int32_t n);
int mig_fast_algo(mig_ctx* ctx, const double* comp, int32_t n, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_greedy_trace_fn trace, void* user);

/* ---- RNG (util.hpp:27-51): std::mt19937_64 streams, splitmix64 seed mixing ---- */
typedef struct mig_rng mig_rng;
int mig_rng_create(uint64_t seed, mig_rng** out);
void mig_rng_destroy(mig_rng* rng);
uint64_t mig_rng_next(mig_rng* rng);
uint64_t mig_mix_seed(uint64_t a, uint64_t b);
uint64_t mig_pick_index(mig_rng* rng, uint64_t n);

/* ---- MCTS slow algorithm (mcts.hpp) ---- */
typedef struct mig_mcts_params { /* MctsParams, mcts.hpp:13-18 */
    int32_t budget_iters;
    int32_t topk;
    int32_t pick_services;
    double ucb_c;
} mig_mcts_params;
void mig_mcts_params_defaults(mig_mcts_params* out);

/* expand(node, ctx, params, rng), mcts.hpp:89-116: children = top-K pool indices */
int mig_expand(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params, mig_rng* rng,
               int64_t* children, int32_t cap, int32_t* n_children);

typedef struct mig_rollout_cache mig_rollout_cache; /* RolloutCache, mcts.hpp:47-50 */
int mig_rollout_cache_create(mig_rollout_cache** out);
void mig_rollout_cache_destroy(mig_rollout_cache* cache);
int32_t mig_rollout_cache_builds(const mig_rollout_cache* cache);

/* rollout(comp, ctx, params, cache, rng, max_depth, picked), mcts.hpp:122-143 */
int mig_rollout(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params,
                mig_rollout_cache* cache, mig_rng* rng, int32_t max_depth, int64_t* picked, int32_t cap,
                int32_t* steps);

typedef void (*mig_mcts_trace_fn)(void* user, int32_t iter, int32_t depth, int32_t estimate, int32_t best_len);
/* mcts_solve(comp, ctx, params, seed, trace), mcts.hpp:148-252 */
int mig_mcts_solve(mig_ctx* ctx, const double* comp, int32_t n, const mig_mcts_params* params, uint64_t seed,
                   mig_config* out, int32_t cap, int32_t* n_out, mig_mcts_trace_fn trace, void* user);

/* ---- MCTS throughput mode: root-parallel rollouts (product extension, rollout.cu) ----
 * The reference runs rollouts one at a time from a sequential mt19937_64 stream
 * (rollout, mcts.hpp:122-143; memoized per unsatisfied-set key, RolloutCache
 * mcts.hpp:47-50).  mig_rollouts runs n_rollouts of them from one root concurrently:
 *   - each step is the reference's rollout step (top-K of the BASE pool under the
 *     current completion, memoized by the unsatisfied bitmap, uniform pick, add);
 *   - draw t of rollout r is Philox4x32-10(key = seed, counter = (t, id_offset + r)),
 *     index = floor(draw * |pool| / 2^64);
 *   - rollouts advance in lock-step rounds; a key first reached in round d takes its pool
 *     from the completion vector of the lowest-indexed rollout that reached it in round d;
 *     the cache persists across the call's batches (rollouts [0,batch), [batch,2 batch)..).
 * The result is a deterministic function of (comp, params): oracle/oracle.cpp restates
 * the same schedule on the CPU.  Root-parallel sharding over GPUs gives each rank a
 * disjoint id range (its own cache), then a MIN-reduction of (best_len, best_id). */
typedef struct mig_rollout_params {
    int64_t n_rollouts;
    int32_t topk;       /* pool size per key, 1..32 (MctsParams.topk, mcts.hpp:15)          */
    int32_t max_depth;  /* < 0: 2 * |fast_algo(comp)|, as mcts_solve (mcts.hpp:154-155)     */
    uint64_t seed;      /* Philox key                                                       */
    int64_t id_offset;  /* global id of rollout 0 (its Philox stream)                       */
    int64_t batch;      /* rollouts per synchronous batch; <= 0: all in one batch           */
    int32_t table_log2; /* key-cache capacity 2^table_log2; <= 0: automatic                 */
} mig_rollout_params;

typedef struct mig_rollout_result {
    int32_t best_len;  /* steps of the shortest completed rollout; -1 if none completed     */
    int32_t max_depth; /* the depth cap used                                               */
    int64_t best_id;   /* its global id (ties: lowest id)                                  */
    int64_t completed, capped, failed; /* failed: reached a key with an empty pool         */
    int64_t steps;     /* rollout steps taken (all rollouts)                               */
    int64_t keys;      /* distinct keys cached (= top-K pool builds)                       */
    int32_t rounds;
    int32_t path_len;
    double device_ms;  /* product: device time of the rollout launches                    */
} mig_rollout_result;

/* lengths[n_rollouts] (optional): steps per rollout (capped: max_depth; empty pool: -1).
 * best_path[cap] (optional): the best rollout's picks (pool indices). */
int mig_rollouts(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* params, int32_t* lengths,
                 int64_t* best_path, int32_t cap, mig_rollout_result* out);

/* Throughput-mode mcts_solve: answer = the shorter of fast_algo(comp) and the best
 * root-parallel rollout (fast_ref wins ties, as mcts.hpp:245-251); max_depth = 2|fast_ref|. */
int mig_mcts_solve_parallel(mig_ctx* ctx, const double* comp, int32_t n, const mig_rollout_params* params,
                            mig_config* out, int32_t cap, int32_t* n_out, mig_rollout_result* result);

/* ---- sharded greedy across ranks (product) ----
 * The reference's fast_algo scans one working set on one core.  Sharded, every rank's
 * context keeps 1/n_ranks of every working set (base supports by index mod n_ranks,
 * extension supports by a fixed hash) and the persistent greedy kernel exchanges its
 * per-step winner with the other ranks through EXCHANGE BOARDS: small device buffers, one
 * per rank, written by every rank with peer stores (CUDA IPC over NVLink/NVSwitch, or
 * plain device pointers for ranks sharing a GPU).  Every rank applies the same global
 * winner, so plans are bit-identical to the unsharded fast_algo at any rank count.
 * Protocol: each rank allocates its board (mig_board_alloc), the ranks exchange the IPC
 * handles, open the peers' boards (mig_board_open), call mig_ctx_set_shard with all
 * n_ranks board pointers (boards[rank] = own), BARRIER, then call mig_fast_algo SPMD.
 * A missing peer fails the call with MIG_ERR_DEVICE after a watchdog (no hang). */
int mig_board_bytes(int32_t n_ranks, int64_t* bytes);
int mig_board_alloc(int32_t device, int32_t n_ranks, void** board, uint8_t* ipc_handle /* 64 bytes, or NULL */);
int mig_board_open(int32_t device, const uint8_t* ipc_handle /* 64 bytes */, void** board);
int mig_board_free(void* board, int32_t opened /* 1: from mig_board_open */);
/* Per-call device resources (streams, working-set arenas, pinned step buffers, scratch) are
 * pooled per device for the process, so a new context reuses them.  This frees every pooled
 * resource of `device` that no live call holds; the next call allocates cold.  CPU
 * implementations: no-op. */
int mig_device_cache_release(int32_t device);
/* Every plan-returning call that fails with MIG_ERR_ARGUMENT because `cap` is too small sets
 * *n_out to the plan's length and keeps the plan (per thread): this copies it out, so a caller
 * never re-runs a stateful call (mig_crossover's Rng, mig_two_phase's time budget) to fetch a
 * long plan. */
int mig_last_plan(mig_config* out, int32_t cap, int32_t* n_out);
/* Draw `step` of Philox stream `stream` under `seed` (the throughput-mode RNG: Philox4x32-10
 * with counter (step, stream) and key seed, draw = word1 << 32 | word0).  on_device = 1
 * evaluates it in a kernel (the product's device code path), 0 on the host; CPU
 * implementations ignore on_device.  For known-answer tests. */
int mig_philox_u64(uint64_t seed, uint64_t stream, uint64_t step, int32_t on_device, uint64_t* out);
/* max_ctas > 0 caps the greedy grid of this context. */
int mig_ctx_set_shard(mig_ctx* ctx, int32_t rank, int32_t n_ranks, void* const* boards, int32_t max_ctas);
/* fast_algo on ALL ranks of a shard whose contexts share one GPU (ctxs in rank order):
 * their instances run as CTA ranges of one cooperative launch and exchange through the
 * boards exactly as ranks on different GPUs do.  n_ctx == 1: plain mig_fast_algo. */
int mig_fast_algo_group(mig_ctx* const* ctxs, int32_t n_ctx, const double* comp, int32_t n, mig_config* out,
                        int32_t cap, int32_t* n_out);

/* ---- GA (ga.hpp) ---- */
typedef struct mig_ga_params { /* GaParams, ga.hpp:24-36 */
    int32_t population;
    double erase_fraction;
    int32_t mutation_pairs;
    int32_t stall_rounds;
    double time_budget_s;
    uint64_t seed;
    int32_t max_rounds;
    int32_t workers;
    mig_mcts_params slow;
} mig_ga_params;
void mig_ga_params_defaults(mig_ga_params* out);

/* completion_of(configs, services, profiles), core.hpp:291-302 */
int mig_completion_of(const mig_ctx* ctx, const mig_config* configs, int32_t n_configs, double* comp_out);

/* mutate(parent, params, rng), ga.hpp:83-113 (out may alias nothing; same length as parent) */
int mig_mutate(const mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, const mig_ga_params* params,
               mig_rng* rng, mig_config* child);

/* crossover(parent, MctsProcedure(params.slow), ctx, params, rng), ga.hpp:51-77.
 * slow_kind: 0 = FastProcedure (greedy.hpp:160-164), 1 = MctsProcedure (mcts.hpp:254-260). */
int mig_crossover(mig_ctx* ctx, const mig_config* parent, int32_t n_gpus, int32_t slow_kind,
                  const mig_ga_params* params, mig_rng* rng, mig_config* child, int32_t cap, int32_t* n_child);

typedef void (*mig_ga_log_fn)(void* user, int32_t round, int32_t best_gpus, double best_slack, int32_t improved,
                              double elapsed_s);
/* two_phase(ctx.services, profiles, rules, params, log), ga.hpp:126-179, on a context
 * built with max_mix = 2 (as two_phase builds its own, ga.hpp:129).  The output is
 * make_deployment order (sorted configs, core.hpp:305-312). */
int mig_two_phase(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                  mig_ga_log_fn log, void* user);

/* Throughput-mode two_phase (product extension, ga.cu): the same rounds, elitism and stop
 * rules as two_phase, with crossover's slow procedure = FastProcedure (greedy.hpp:160-164)
 * and Philox draws — draw t of child i in round r is Philox4x32-10(key = seed, counter =
 * (t, (r << 20) + i)), index = floor(draw * n / 2^64).  Every generation's mutation,
 * crossover and fitness run on the device over the whole population; children longer than
 * 2 * |seed plan| + 64 GPUs count as failed crossovers.  params->workers and ->slow are
 * ignored.  oracle/ and the reference shim restate the same rule on the CPU. */
int mig_two_phase_parallel(mig_ctx* ctx, const mig_ga_params* params, mig_config* out, int32_t cap, int32_t* n_out,
                           mig_ga_log_fn log, void* user);

/* The same throughput-mode two_phase with crossover's slow procedure = the throughput
 * mcts_solve (mig_mcts_solve_parallel) instead of FastProcedure — BASELINE config #3's
 * "greedy -> GA -> MCTS" pipeline with a fixed Philox seed: child i of round r refills its
 * residual with the shorter of fast_algo(residual) and the best of slow->n_rollouts
 * root-parallel rollouts (pool size slow->topk, depth cap 2 x |fast refill|, batches of
 * slow->batch, ids from slow->id_offset) under Philox key mix_seed(params->seed,
 * (r << 20) + i); the fast refill wins ties (mcts.hpp:245-251).  slow->seed, ->max_depth
 * and ->table_log2 are ignored. */
int mig_two_phase_parallel_mcts(mig_ctx* ctx, const mig_ga_params* params, const mig_rollout_params* slow,
                                mig_config* out, int32_t cap, int32_t* n_out, mig_ga_log_fn log, void* user);

/* ---- eval bench helpers (bench.hpp) ---- */
/* lower_bound(services, profiles), bench.hpp:93-108 */
int mig_lower_bound(const mig_ctx* ctx, int32_t* out);

/* baseline(kind, services, profiles), bench.hpp:42-90: the static-partition deployments.
 * kind: 0 = A100-7/7 (whole GPUs), 1 = A100-7x1/7 (1/7 instances packed seven to a GPU),
 * 2 = A100-MIX (4/7 + 2/7 + 1/7 per GPU).  Configs in construction order (make_deployment
 * sorts them); PlanningError "service '<id>' is infeasible on a <s>/7 instance under its
 * latency ceiling" when a needed size has no feasible batch. */
int mig_baseline(const mig_ctx* ctx, int32_t kind, mig_config* out, int32_t cap, int32_t* n_out);

/* brute_force_optimum(services, profiles, rules, cap, node_budget), bench.hpp:160-219: the
 * exhaustive minimum-GPU search over config multisets (iterative deepening, admissible bound).
 * Like the reference (bench.hpp:164-165) it builds the pool it searches — every config with
 * at most min(n, 7) distinct services, in the reference's emission order — independently of
 * the context's max_mix; the product's device search takes n <= 16 services and cap <= 8
 * (MIG_ERR_ARGUMENT beyond).  *found = 0 (and *n_out = 0) when the optimum exceeds cap;
 * PlanningError "oracle: node budget exceeded; ..." when more than node_budget DFS nodes are
 * visited and "oracle: service cannot be served by any config" when a service has no utility
 * anywhere.  The plan is the reference's first solution in its DFS order, and the budget
 * guard trips at exactly the reference's node count. */
int mig_brute_force_optimum(mig_ctx* ctx, int32_t cap, int64_t node_budget, mig_config* out, int32_t out_cap,
                            int32_t* n_out, int32_t* found);

/* ---- instrumentation (product only; CPU libraries report zeros) ---- */
/* Work counters.  "Rows scored" is implementation-independent (the oracle counts the same
 * numbers): every greedy step scores its whole working set (greedy.hpp:126-134) and every
 * top-K call scores its candidate set once (mcts.hpp:59-67). */
typedef struct mig_stats {
    int64_t rows_scored;      /* greedy_rows + topk_rows                                 */
    int64_t greedy_rows;      /* Σ over greedy steps of the working-set size             */
    int64_t topk_rows;        /* Σ over top-K calls of the candidate-set size            */
    int64_t greedy_calls;
    int64_t topk_calls;
    int64_t greedy_steps;     /* argmax steps executed                                   */
    int64_t ext_events;       /* extension events (greedy.hpp:107-119)                   */
    int64_t ext_rows;         /* rows appended by extension enumeration                  */
    int64_t kernel_launches;  /* CUDA kernels launched by this context (product only)    */
    int64_t h2d_bytes;        /* host->device bytes copied (product only)                */
    int64_t d2h_bytes;        /* device->host bytes copied (product only)                */
    double greedy_ms;         /* device time of greedy launches, CUDA events (product)   */
    double topk_ms;           /* device time of top-K launches, CUDA events (product)    */
    /* greedy-kernel phase split seen by CTA 0 (%globaltimer, product): scan+block argmax,
     * grid barrier, grid argmax+update, maybe_extend, extension enumeration+barrier     */
    double phase_ms[5];
    int64_t rollout_steps;    /* throughput-mode rollout steps (mig_rollouts)            */
    int64_t rollout_calls;
    double rollout_ms;        /* device time of rollout launches (product)               */
    double mcts_ms;           /* device time of the device-resident MCTS searches        */
    int64_t mcts_launches;
    int64_t mcts_rows;        /* rows scored by those searches' top-Ks (part of topk_rows) */
    int64_t mcts_topk_calls;  /* their top-K calls (part of topk_calls)                   */
} mig_stats;
int mig_ctx_stats(const mig_ctx* ctx, mig_stats* out);
void mig_ctx_reset_stats(mig_ctx* ctx);
/* Diagnostic: the working-set size (base pool + extension rows; this rank's share when
 * sharded) scanned at each step of the most recent greedy plan completed on this context
 * (greedy.hpp:123-134's ws.size()).  Writes min(cap, steps) values; *n_out = steps. */
int mig_ctx_step_rows(const mig_ctx* ctx, int64_t* out, int32_t cap, int32_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* MIGPLAN_B200_H */

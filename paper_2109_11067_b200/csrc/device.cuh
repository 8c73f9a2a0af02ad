// device.cuh — device-side tables and helpers shared by the sm_100a kernels.
#pragma once

#include <cstdint>

namespace mgb {

constexpr uint64_t kNoRow = ~0ull;

// Read-only model tables (uploaded once per PlanContext).  See model.hpp for meaning.
struct DevModel {
    int n;         // services
    int PP;        // patterns; row code = svc * PP + pattern, sentinel n * PP
    unsigned pp_magic;  // ceil(2^32 / PP): svc_of(code) = umulhi(code, pp_magic), exact for code < 2^16
    int n_sizes;
    int n_layouts;
    int max_mix;
    int n_tmpl[5];           // templates per member count k = 0..4
    const uint64_t* tmpl[5]; // layout(8) | pat0 << 8 | pat1 << 16 | pat2 << 24 | pat3 << 32
    const double* U;         // (n+1) * PP utilities, row n zeros
    const double* best_single;  // n
    const uint8_t* feas_mask;   // n
    const uint8_t* pat_mask;    // PP
    const uint8_t* pat_count;   // PP * 5
    const uint8_t* layout_count;  // n_layouts * 5
    const int8_t* layout_slots;   // n_layouts * 5 * 7 (ascending slots per size index)
    const int* sizes;             // n_sizes (ascending)
    const double* thr;            // n * 5: selected throughput per (service, size index), 0 if infeasible
    const double* req;            // n: required rps
    // row_key tables (common.cuh): per code (svc << 8 | pattern), per pattern its size counts
    // packed 3 bits per size index, and the layout of every packed count vector (0xFF: none)
    const uint16_t* key_code;     // (n + 1) * PP
    const uint32_t* pat_packed;   // PP
    const uint8_t* layout_of;     // 1 << 15
};

// code / PP by a multiply: for code < 2^16 and PP < 2^16 the error of ceil(2^32 / PP) stays
// below 1/PP, so the quotient is exact (the scan loops called the integer-division routine).
__device__ __forceinline__ int svc_of(const DevModel& M, unsigned code) {
    return M.pp_magic ? static_cast<int>(__umulhi(code, M.pp_magic)) : static_cast<int>(code);  // 0: PP == 1
}

// One argmax candidate: score, util_sum, packed row.
struct Best {
    double s;
    double u;
    uint64_t row;
};

// Per-call device state of the persistent greedy kernel.
struct GreedyState {
    unsigned int bar_count;
    unsigned int bar_gen;
    int status;        // 0 ok, 1 no positive score, 2 extension overflow, 3 step overflow
    int n_steps;
    unsigned long long ext_count;
    int n_events;
    unsigned int arrive;  // all-reduce argmax: arrivals so far (step s completes at (s + 1) * G)
    long long rows_scored;
    // CTA-0 %globaltimer phase totals (ns): 0 build W + scan + block reduce, 1 grid barrier,
    // 2 grid reduce + completion update, 3 maybe_extend, 4 extension enumeration + barrier
    unsigned long long phase_ns[5];
    unsigned long long last_seq;  // sharded greedy: exchange sequence number of the last step
};

enum GreedyStatus { kOk = 0, kNoPositive = 1, kExtOverflow = 2, kStepOverflow = 3, kExchTimeout = 4 };

// One record of the sharded greedy's per-step exchange board (kernels.cu exchange_best).
// A board is [2 parities][n_ranks] slots; seq = global step counter + 1 (monotonic).
struct ExchSlot {
    double s;
    double u;
    unsigned long long row;
    unsigned long long seq;
};
constexpr int kMaxRanks = 8;

struct GreedyArgs {
    DevModel M;
    uint64_t* rows;       // arena: base pool rows [0, n_base), extension rows appended after
    long long n_base;
    long long cap;        // arena capacity (rows)
    int cache_units;      // 16-byte row units of shared-memory cache per CTA
    int phase_timers;     // 1: CTA 0 records %globaltimer phase totals (diagnostics)
    int prefetch;         // bulk L2 prefetch distance of the streaming scan (iterations; 0 off)
    int pipeline;         // streaming scan: load the next 4 units before scoring these (1) or not
    int load_mode;        // streaming row load flavour (kernels.cu ld_row4)
    int interleave;       // units dealt to CTAs in 32-unit blocks (working set fits on chip)
    int ring_stages;      // TMA ring stages (32 KB each) for rows beyond the cache; 0: direct loads
    const double* comp0;  // host-mapped pinned
    GreedyState* st;      // device (barrier + atomics)
    GreedyState* out;     // host-mapped pinned: final state written by CTA 0
    Best* partials;       // 2 * gridDim.x (double buffered by step parity)
    uint64_t* pick_row;   // cap_steps (device)
    double* pick_score;   // cap_steps (device)
    long long* pick_rows; // rows in the working set at that step (device)
    uint64_t* host_pick_row;    // host-mapped copies written once at the end
    double* host_pick_score;
    long long* host_pick_rows;
    int* ev_svc;          // events recorded (service, in order)
    int cap_steps;
    // sharded greedy: this rank scans 1/n_ranks of every working set
    int n_ranks;          // 1: unsharded
    int rank;
    ExchSlot* boards[kMaxRanks];  // every rank's exchange board (peer or local device memory)
    unsigned long long exch_seq0; // step counter base of this call (monotonic across calls)
    long long exch_timeout_ns;
};

// A greedy launch: n_groups independent instances (ranks sharing this GPU), each on
// ctas_per_group consecutive CTAs.
constexpr int kMaxGroups = 8;  // instances per launch (param space: 8 x 368 B)
struct GreedyLaunch {
    int n_groups;
    int ctas_per_group;
    int cluster;  // each group is one thread-block cluster (<= 16 CTAs): DSMEM argmax, cluster barriers
    GreedyArgs g[kMaxGroups];
};

struct TopkArgs {
    DevModel M;
    const uint64_t* rows;     // base rows
    long long n_rows;
    const long long* index;   // optional: candidate indices to consider (NULL: all rows)
    long long n_index;
    const uint64_t* svc_mask; // optional: 4 words; a row qualifies if any member is in the mask
    const double* comp;
    int k;
    unsigned int* bar;        // 2 words
    Best* partials;           // 2 * gridDim.x
    uint64_t* out_row;        // k
    int* n_out;
};

// Single-launch top-K (topk.cu), k <= 32.  The completion vector and the service mask
// travel inside the launch parameters: no host-mapped reads on the latency path.
struct Topk1Args {
    DevModel M;
    const uint64_t* rows;
    long long n_rows;
    const long long* index;
    long long n_index;
    int use_mask;
    int k;
    long long rows_per_cta;
    Best* partials;     // gridDim.x * 32 per-CTA lists
    unsigned* ticket;   // zero before launch; reset by the last CTA
    uint64_t* out_row;  // k (host-mapped)
    int* n_out;         // host-mapped
    unsigned long long* n_scored;  // host-mapped: rows passing the service mask (zeroed by the host)
    uint64_t svc_mask[4];
    double comp[256];
};

// Throughput-mode GA (ga.cu).  A chromosome is a list of GPU GENOMES (8 bytes each):
// byte 0 = canonical layout id, byte 1 + k = service of the layout's k-th instance in
// normalized order (size ascending, slot ascending; core.hpp:187-190), 0xFF = none.
// Batch is a function of (service, size), so swaps of equal-size instances keep it exact.
struct GaBreedArgs {
    DevModel M;
    const uint64_t* pop;   // parents: [n_children][L_cap] genomes
    const int* pop_len;
    uint64_t* work;        // [n_children][L_cap] mutated parents (crossover's fallback)
    uint64_t* child;       // [n_children][L_cap] survivors, then refill
    int* n_surv;
    double* residual;      // [n_children][n] completion of the survivors
    unsigned* scratch;     // [n_children][8 * L_cap] erase order / size refs
    int L_cap;
    int round;
    int mutation_pairs;
    double erase_fraction;
    uint64_t seed;
};

struct GaFinishArgs {
    DevModel M;
    const uint64_t* work;
    uint64_t* child;
    const int* n_surv;
    const uint64_t* const* refill;  // [n_children] device pointers to picked rows
    const int* refill_n;            // [n_children] picks, -1: the refill failed
    int* child_len;
    double* child_slack;
    int L_cap;
};

// Device-resident parity mcts_solve (mcts.cu): one CTA per search.
struct MctsSolveArgs {
    const double* comp0;     // start completion (n, device)
    uint64_t seed;           // mt19937_64 seed = mix_seed(seed, 0x6d637473) (mcts.hpp:157)
    int l_ref;               // |fast_algo(comp0)|
    int max_nodes;
    double* node_comp;       // max_nodes * n
    int* node_visits;
    double* node_value;
    int* node_first;
    int* node_nch;
    int* node_cand;          // base-pool index of the edge into the node
    unsigned char* node_flags;
    int* pathnodes;          // selection path (node ids)
    int* edges;              // candidate ids along the path
    int* picked;             // rollout picks
    int* unsat;              // n
    unsigned tab_mask;       // rollout cache (open addressing over the unsat bitmap)
    unsigned* tag;
    uint64_t* key;
    int* pool_n;
    unsigned* pool;          // (tab_mask + 1) * topk
    int* trace;              // budget * 4: iter, depth, estimate, best_len (mcts.hpp:226)
    int* best_out;           // best complete path (candidate ids)
    int* descent_out;        // visit-count descent (candidate ids)
    double* descent_comp;    // n: completion at the end of the descent
    int* out;                // status, best_len, descent_len, descent_leaf, builds, nodes, iterations
};

struct MctsLaunch {
    DevModel M;
    const uint64_t* base;
    long long n_base;
    const unsigned* keyrank; // rank of each base row in the config order (tie-break)
    const double* logtab;    // std::log(v) for v = 0..budget (host-computed, bit-exact)
    int budget, topk, pick_services;
    double ucb_c;
    int node_smem;           // node metadata in shared memory (all solves: same max_nodes)
    int rows_smem;           // the base pool copied into shared memory
    int timers;              // accumulate top-K phase cycles (MIGPLAN_MCTS_TIMERS)
    int pair;                // every base row has <= 2 members: on-chip copy as 32-bit rows
    const unsigned* base32;  // pair pool too large for shared memory: its 32-bit rows in global memory
    // the base pool's supports (K1 order: each a contiguous row range): a top-K scans only the
    // supports that can hold a candidate (a service with need > 0, or a sampled service)
    int n_sup;               // 0: scan every row
    const int* sup_begin;    // n_sup + 1 row offsets
    const unsigned short* sup_svc;  // service a | b << 8 (b = 0xFF: single-service support)
    int l1_slots;            // on-chip rollout-cache slots (power of two; 0: global table only)
    MctsSolveArgs s[kMaxGroups];
};

// Device brute_force_optimum (bf.cu): one launch per iterative-deepening depth, over the
// max_mix = min(n, 7) pool that bf_enum_kernel builds in the reference's emission order.
constexpr int kBfMaxDepth = 8;   // cap
constexpr int kBfMaxN = 16;      // services (the max_mix = 7 pool of 16 services is ~1 M rows)
constexpr int kBfCodes = 8;      // member codes per wide row (<= 7 distinct services)
struct BfArgs {
    DevModel M;
    const uint4* rows;           // the pool: 8 u16 member codes per row (svc ascending, sentinel n*PP)
    long long n_rows;
    const double* best_any;      // n: best utility any config gives each service
    int depth;
    long long rank0, rank_end;   // this launch's DFS prefixes (lexicographic ranks)
    long long replay;            // >= 0: only this prefix rank, writes its tuple
    unsigned long long remaining;  // node budget left before this launch
    unsigned long long* cnt;     // per prefix: reference-order DFS nodes in its subtree
    unsigned long long* best_key;  // smallest solving rank
    unsigned long long* overrun;   // smallest rank whose own subtree exceeded `remaining`
    unsigned long long* sum;       // bf_sum_kernel: Σ cnt[rank0 .. min(best_key, rank_end-1)]
    long long* tuple;            // replay: picks (pool indices), tuple[kBfMaxDepth] = length
};

// The pool enumerator (config_enum.hpp:108-188 with max_mix = min(n, 7)): index t of layout
// li is a mixed-radix number over the layout's groups (group 0 most significant), each digit
// the lexicographic rank of a nondecreasing service sequence of the group's length.
struct BfEnumArgs {
    int n, PP, max_mix, n_layouts;
    int n_groups[32];
    int8_t g_len[32][5];          // slots per group
    int8_t g_size[32][5];         // size index per group
    long long g_cnt[32][5];       // C(n + len - 1, len): nondecreasing sequences per group
    long long lay_off[33];        // flat index of each layout's first combination
    uint8_t feas_mask[kBfMaxN];   // bit z: feasible at size index z
    const uint8_t* pat_of;        // 1 << 15: count vector (3 bits per size index) -> pattern (0xFF none)
    unsigned* block_cnt;          // per 256-index block: valid configs (mode 0) / write offset (mode 1)
    uint4* rows;                  // mode 1 output
    int* error;                   // a member pattern missing from pat_of
};

// Throughput-mode root-parallel rollouts (rollout.cu).
struct RolloutCounters {
    unsigned long long n_act[2];  // active-list lengths (ping-pong by round parity)
    unsigned long long n_pend[2]; // key-cache slots created per round (ping-pong)
    int done;                     // a round found no active rollout (its build kernel sets it)
    unsigned int bar_count, bar_gen;  // grid barrier of the persistent small-batch kernel
    int status;                   // 0 ok, 1 key cache full
    int rounds;
    unsigned long long best;      // min over completed rollouts of (steps << 32 | batch index)
    unsigned long long steps, completed, capped, failed, keys;
};

struct RolloutArgs {
    DevModel M;
    const uint64_t* base;   // base pool rows (the rollout pool, mcts.hpp:129-133)
    long long n_base;
    long long n_roll;       // rollouts in this batch
    long long id0;          // global id of the batch's rollout 0 (Philox stream id)
    uint64_t seed;          // Philox key
    int k;                  // pool size per key (MctsParams.topk), <= 32
    int max_depth;
    double* comp;           // n_roll * n: per-rollout completion vectors
    int* len;               // n_roll: steps taken
    uint8_t* status;        // n_roll: 0 active, 1 satisfied, 2 depth cap, 3 empty pool
    unsigned* rslot;        // n_roll: key-cache slot of the current key
    long long* act0;        // active lists (ping-pong)
    long long* act1;
    uint64_t* keys;         // n <= 64: n_roll type keys (the unsatisfied bitmap), kept per rollout
    // key cache (RolloutCache, mcts.hpp:47-50): open addressing over the unsat bitmap
    unsigned tab_mask;      // capacity - 1 (power of two)
    unsigned* tag;          // 0 empty, 1 key being written, 2 key ready
    uint64_t* key;          // capacity * 4
    unsigned long long* claimer;  // lowest batch index that probed the slot in its first round
    int* pool_n;            // -1 until the pool is built
    unsigned* pool;         // capacity * k base-pool indices, preferred first
    unsigned* pend0;        // slots created in the round (ping-pong)
    unsigned* pend1;
    RolloutCounters* cnt;
    long long* path;        // host-mapped: winner replay (base-pool indices), max_depth
    int* path_len;          // host-mapped
    int* lengths;           // optional, n_roll: steps (capped: max_depth, empty pool: -1)
    // the base pool's supports (pair pools): a pool build scans only supports with a member
    // whose need is > 0 (0: scan every row)
    int n_sup;
    const int* sup_begin;
    const unsigned short* sup_svc;
    const unsigned* base32;   // pair pools: the rows' low 32 bits (the pair top-K), else nullptr
    const unsigned* keyrank;  // config-order key rank of every base row (pair top-K tie-break)
    int timers;             // diagnostics (unused by the split kernels)
    double comp0[256];      // start completion (travels with the launch)
};

}  // namespace mgb

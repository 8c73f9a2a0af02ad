// engine.hpp — the native runtime behind the C-ABI: one PlanContext on one B200.
//
// Owns the device-resident tables (model + packed base pool), a pool of per-call
// "slots" (stream, extension arena, step buffers) so that concurrent GA workers can
// run independent greedy / top-K calls on one context (the reference's functions are
// reentrant over a const PlanContext, ga.hpp:153-163), and the host-side search
// drivers (MCTS, GA) that call the kernels.
#pragma once

#include <atomic>
#include <map>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "device.cuh"
#include "model.hpp"

namespace mgb {

struct Config {  // normalized GpuConfig with service indices (mig_config)
    int n = 0;
    Model::Inst inst[kMaxInst];
};

bool config_less(const Config& a, const Config& b);

// Exchange boards of the sharded greedy (device memory, IPC-shareable across processes).
size_t board_bytes(int n_ranks);
void* board_alloc(int device, int n_ranks, unsigned char ipc_handle[64]);
void* board_open(int device, const unsigned char ipc_handle[64]);
void board_close(void* board, bool opened);
void release_device_cache(int device);
uint64_t philox_on_device(int device, uint64_t seed, uint64_t stream, uint64_t step);
bool config_equal(const Config& a, const Config& b);

struct Slot;
struct GreedyCall;
struct GaRun;
struct GaParams;

struct DeviceInfo {
    int num_sms = 0;
    long long smem_optin = 0;
    long long mcts_static_smem = 0;  // static shared memory of mcts_kernel
    long long greedy_static_smem = 0;  // static shared memory of greedy_kernel
};
const DeviceInfo& device_info(int device);

struct Stats {
    std::atomic<long long> greedy_rows{0}, topk_rows{0}, greedy_calls{0}, topk_calls{0}, greedy_steps{0};
    std::atomic<long long> ext_events{0}, ext_rows{0}, launches{0}, h2d{0}, d2h{0};
    std::atomic<long long> greedy_ns{0}, topk_ns{0}, rollout_ns{0}, rollout_steps{0}, rollout_calls{0};
    std::atomic<long long> mcts_ns{0}, mcts_launches{0}, mcts_rows{0}, mcts_topk_calls{0};
    std::atomic<long long> phase_ns[5] = {0, 0, 0, 0, 0};
    void reset() {
        for (auto* a : {&greedy_rows, &topk_rows, &greedy_calls, &topk_calls, &greedy_steps, &ext_events, &ext_rows,
                        &launches, &h2d, &d2h, &greedy_ns, &topk_ns, &rollout_ns, &rollout_steps, &rollout_calls,
                        &mcts_ns, &mcts_launches, &mcts_rows, &mcts_topk_calls})
            a->store(0);
        for (auto& p : phase_ns) p.store(0);
    }
};

// Device-resident parity mcts_solve (mcts.cu): what the kernel returns to the host driver.
struct MctsDeviceResult {
    int status = 0;                  // 0 ok, 1 rollout found an empty pool (PlanningError), 2/3 capacity
    int iterations = 0;
    std::vector<int> trace;          // 4 per iteration: iter, depth, estimate, best_len
    std::vector<long long> best;     // best complete path (base-pool indices); empty + best_len -1: none
    int best_len = -1;
    std::vector<long long> descent;  // visit-count descent
    std::vector<double> descent_comp;
    bool descent_leaf = false;
    int builds = 0, expands = 0;
    long long expand_rows = 0;
};

// Throughput-mode root-parallel rollouts (rollout.cu): the result of one mig_rollouts call.
// Throughput mcts_solve as the GA's crossover refill (mig_two_phase_parallel_mcts).
struct RolloutRefill {
    long long n_rollouts = 0;
    int topk = 10;
    long long id_offset = 0;
    long long batch = 0;
    int table_log2 = 0;
};

struct RolloutResult {
    int best_len = -1;        // shortest completed rollout (steps); -1: none completed
    long long best_id = -1;   // its global id (ties: lowest id)
    std::vector<long long> path;  // its picks (base-pool indices)
    long long completed = 0, capped = 0, failed = 0, steps = 0, keys = 0;
    int rounds = 0, launches = 0;
    double ms = 0.0;          // device time (CUDA events)
};

// A device buffer from the process-wide scratch pool (returned on destruction).
class Scratch {
  public:
    Scratch(int device, size_t bytes);
    ~Scratch();
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    void* get() const { return p_; }

  private:
    int device_ = 0;
    size_t bytes_ = 0;
    void* p_ = nullptr;
};

class Engine {
  public:
    Engine(const Rules& rules, std::map<std::string, ModelProfile> profiles, std::vector<Service> services,
           int max_mix, int device);
    ~Engine();

    const Model& model() const { return m_; }
    int n() const { return m_.n; }
    const std::vector<uint64_t>& base_rows() const { return base_rows_; }
    long long pool_size() const { return static_cast<long long>(base_rows_.size()); }
    long long index_of(uint64_t row) const;
    Config config_of(uint64_t row) const;
    Config config_of_wide(const uint4& row) const;  // brute_force_optimum's 8-code rows

    // fast_algo (greedy.hpp:95-145) on the device.  Returns picked rows and their scores.
    void fast_algo(const std::vector<double>& comp, std::vector<uint64_t>& rows, std::vector<double>& scores);
    // The same on the ranks (in rank order) of a sharded greedy that share one GPU: one launch.
    static void fast_algo_group(const std::vector<Engine*>& es, const std::vector<double>& comp,
                                std::vector<uint64_t>& rows, std::vector<double>& scores);
    // topk_candidates (mcts.hpp:56-76) over the base pool; filter by explicit indices or a
    // service mask (rows touching any masked service).  Returns pool indices, preferred first.
    std::vector<long long> topk(const std::vector<double>& comp, int k, const std::vector<long long>* index,
                                const std::vector<uint64_t>* svc_mask);

    // n_roll root-parallel rollouts from comp (rollout.cu), processed in synchronous batches
    // of `batch` rollouts sharing one key cache; rollout r has global id id_offset + r.
    RolloutResult rollouts(const std::vector<double>& comp, long long n_roll, int k, int max_depth, uint64_t seed,
                           long long id_offset, long long batch, int table_log2, int* lengths);

    // Sharded greedy: from now on fast_algo scans only this rank's 1/n_ranks of
    // every working set and exchanges per-step winners through the boards (every rank's
    // board, device pointers valid on this device: peer memory or local).  All ranks must
    // call fast_algo with identical inputs (SPMD); their plans are identical.
    // max_ctas > 0 caps this context's greedy grid (ranks sharing one GPU).
    void set_shard(int rank, int n_ranks, const std::vector<void*>& boards, int max_ctas);
    int n_ranks() const { return n_ranks_; }

    // mcts_solve's search loop on the device (one CTA); l_ref = |fast_algo(comp)|.
    MctsDeviceResult mcts_device(const std::vector<double>& comp, int budget, int topk, int pick_services, double ucb_c,
                                 uint64_t seed, int l_ref);

    // brute_force_optimum (bench.hpp:160-219) on the device over the max_mix = min(n, 7) pool
    // it enumerates itself (bench.hpp:164-165; n <= 16).  found = false: the optimum exceeds cap.
    std::vector<Config> brute_force(int cap, long long node_budget, bool& found);

    // Slots kept past greedy_batch so the device picked rows it returns stay valid: released
    // when the lease is destroyed (after the caller has consumed the rows).
    struct SlotLease {
        Engine* e = nullptr;
        std::vector<Slot*> slots;
        SlotLease() = default;
        SlotLease(const SlotLease&) = delete;
        SlotLease& operator=(const SlotLease&) = delete;
        ~SlotLease() {
            for (Slot* s : slots) e->release(s);
        }
    };
    // Independent single-CTA greedy instances in one launch (the GA's refills).  With `lease`
    // every instance's slot (and so its device picked rows) is held by the lease; without
    // one, the device pointers in `rows` are only valid until the next batch of 8 starts,
    // so callers that read them must pass a lease (or ask for host_rows).
    void greedy_batch(const double* d_comps, int count, long long cap_steps, long long rows_bound,
                      std::vector<const uint64_t*>& rows,
                      std::vector<int>& n_steps, std::vector<std::vector<uint64_t>>* host_rows = nullptr,
                      SlotLease* lease = nullptr, const double* h_comps = nullptr);
    void fast_algo_batch(const std::vector<std::vector<double>>& comps, std::vector<std::vector<uint64_t>>& rows,
                         std::vector<int>& status);
    std::vector<MctsDeviceResult> mcts_device_group(const std::vector<std::vector<double>>& comps, int budget, int topk,
                                                    int pick_services, double ucb_c, const std::vector<uint64_t>& seeds,
                                                    const std::vector<int>& l_refs);
    // Throughput-mode GA device state and one generation (ga.cu; driver in search.cpp).
    GaRun* ga_begin(int population, int L_cap);
    void ga_end(GaRun* r);
    void ga_put(GaRun* r, int buf, int idx, const std::vector<uint64_t>& genomes);
    std::vector<uint64_t> ga_get(GaRun* r, int buf, int idx, int len, bool from_child);
    void ga_generation(GaRun* r, int buf, const std::vector<int>& parent_len, int round, const GaParams& p,
                       std::vector<int>& child_len, std::vector<double>& child_slack,
                       const RolloutRefill* slow = nullptr);
    void ga_select(GaRun* r, int buf, const std::vector<std::tuple<bool, int, int>>& order);

    // completion_of (core.hpp:291-302), count-based, on the host (control logic, not hot).
    std::vector<double> completion_of(const std::vector<Config>& cfgs) const;
    const std::map<std::string, ModelProfile>& profiles() const { return profiles_; }

    Stats stats;
    int device() const { return device_; }
    // working-set size at each step of the most recent greedy plan finished on this context
    std::vector<long long> last_step_rows() const {
        std::lock_guard<std::mutex> g(diag_mu_);
        return last_step_rows_;
    }

  private:
    mutable std::mutex diag_mu_;
    std::vector<long long> last_step_rows_;
    Slot* acquire();
    void release(Slot*);
    void ensure_ext(Slot* s, long long rows);
    long long step_bound(const std::vector<double>& comp) const;
    void greedy_prepare(GreedyCall& c, const double* comp_host, const double* comp_dev, long long cap_steps,
                        cudaStream_t st = nullptr, bool defer_init = false);
    // environment knobs of greedy_prepare, read once per context (greedy_prepare ran five
    // getenv calls per instance)
    struct GreedyKnobs {
        int phase_timers = 0, prefetch = 4, pipeline = 1, load_mode = 2;
        long long exch_timeout_ns = 10'000'000'000ll;
    } gk_;
    bool greedy_finish(GreedyCall& c, float ms, int attempt, std::vector<uint64_t>& rows, std::vector<double>& scores);

    Model m_;
    std::map<std::string, ModelProfile> profiles_;
    int device_ = 0;
    int num_sms_ = 0;
    int greedy_blocks_per_sm_ = 0;
    int topk_blocks_per_sm_ = 0;
    int rollout_blocks_per_sm_ = 0;      // pool-build kernel
    int rollout_adv_blocks_per_sm_ = 0;  // advance kernel
    DevModel dm_{};
    std::vector<void*> dev_allocs_;
    std::unique_ptr<Scratch> ctx_buf_;  // model tables + resident base pool (pooled, see engine.cu)
    // per-call rollout buffers (device and host-mapped) and streams, cached per device across
    // calls and contexts (engine.cu ro_cache): a rollout call that cudaMalloc'd / cudaHostAlloc'd
    // / freed its tables cost milliseconds of host time (config #3 runs hundreds of small calls)
    void* ro_get(size_t bytes, bool host);
    void ro_put(void* p);
    int ro_stream();
    void ro_stream_put(int i);
    uint64_t* d_base_ = nullptr;
    std::vector<uint64_t> base_rows_;
    mutable std::unordered_map<uint64_t, long long> row_index_;
    mutable std::once_flag row_index_once_;
    // rank of every base row in the config order (core.hpp:174-200), for the device
    // top-Ks' last tie-break (built on first use)
    unsigned* d_keyrank_ = nullptr;
    std::unique_ptr<Scratch> keyrank_buf_;
    std::once_flag keyrank_once_;
    const unsigned* keyrank();
    int greedy_cluster_ctas(size_t smem, long long rows_bound = -1) const;  // 0: cooperative launch
    long long working_set_bound(const double* comp) const;
    mutable std::atomic<int> cluster_ctas_{-1};  // its cached answer (no env override)
    // base-pool supports for the MCTS top-K (built on first use; pair pools only)
    std::once_flag sup_once_;
    std::unique_ptr<Scratch> sup_buf_;
    int n_sup_ = 0;
    const int* d_sup_begin_ = nullptr;
    const unsigned short* d_sup_svc_ = nullptr;
    void support_tables();
    // the base pool's rows as 32-bit pairs (max_mix <= 2: the two high codes are sentinels),
    // for the pool builds' pair top-K (built on first use)
    std::once_flag base32_once_;
    std::unique_ptr<Scratch> base32_buf_;
    const unsigned* base32();
    // supports the pool-build scans may list (pair pools), for shared-memory sizing
    int max_sup() const {
        const long long ns = m_.n + static_cast<long long>(m_.n) * (m_.n - 1) / 2;  // <= 2-member supports
        return m_.max_mix <= 2 && ns <= 4096 ? static_cast<int>(ns) : 0;
    }
    int greedy_interleave(int G) const;
    std::vector<double> min_u_;  // smallest positive utility per service (step bound)
    long long ext_bound_ = 0;
    int cache_units_ = 0;  // greedy shared-memory row cache per CTA (16-byte units)
    int ring_stages_ = 0;  // greedy TMA ring stages
    std::vector<long long> support_off_;  // base pool: row offset of every support (K1 order) + total
    int rank_ = 0, n_ranks_ = 1, max_ctas_ = 0;
    std::vector<void*> boards_;
    uint64_t* d_shard_ = nullptr;  // this rank's base rows (sharded greedy)
    long long n_shard_ = 0;
    unsigned long long exch_seq_ = 0;

};

}  // namespace mgb

// engine.cu — device memory, launches and per-call slots for one PlanContext.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <functional>

#include <nvtx3/nvtx3.hpp>

#include "engine.hpp"
#include "search.hpp"

namespace mgb {

namespace {
// MIGPLAN_HOST_TIMERS=1: host-side split of the grouped launches (set-up / launch to sync / after)
struct HostTimer {
    bool on = std::getenv("MIGPLAN_HOST_TIMERS") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
    double parts[4] = {0, 0, 0, 0};
    void mark(int k) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        parts[k] += std::chrono::duration<double, std::micro>(now - t).count();
        t = now;
    }
    void print(const char* what) const {
        if (on) std::fprintf(stderr, "[host] %-14s set-up %.1f us, launch->sync %.1f us, after %.1f us\n", what, parts[0], parts[1], parts[2]);
    }
};
}  // namespace


size_t greedy_smem_bytes(int n, int PP, int cache_units, int stages);
size_t topk_smem_bytes(int n, int PP);
const void* greedy_kernel_ptr();
const void* topk_kernel_ptr();
const void* enum_base_kernel_ptr();
int kernel_threads();
size_t topk1_smem_bytes(int n, int PP, int km);
int topk1_threads();
int topk1_rows_per_cta();
int topk1_max_ctas();
constexpr int kTopkMaxCtas = 4096;  // partial-list capacity (Best x 32 per CTA)
const void* topk1_kernel_ptr(int km);
size_t rollout_smem_bytes(int n, int PP, int n_sup);
size_t mcts_smem_bytes(int n, int PP, int max_nodes, long long n_base, bool node_smem, bool rows_smem, bool pair,
                       int n_sup);
const void* bf_kernel_ptr();
const void* bf_enum_kernel_ptr();
const void* bf_scan_kernel_ptr();
const void* bf_best_any_kernel_ptr();
const void* bf_sum_kernel_ptr();
const void* bf_warp_kernel_ptr();
int bf_threads();
const void* mcts_kernel_ptr(int n);  // the key-width variant for n services
void mcts_set_dense_pct(int pct);
void mcts_read_topk_timers(unsigned long long* h);
void greedy_read_diag(unsigned long long* skew_ns, unsigned long long* release_ns);
size_t keyrank_scratch_bytes(long long P);
cudaError_t build_keyrank(const DevModel& M, const uint64_t* rows, long long P, unsigned* rank, void* scratch,
                          size_t scratch_bytes, cudaStream_t stream, int* launches);
int mcts_threads();
const void* rollout_build_ptr();
const void* rollout_advance_ptr(int n);
const void* rollout_replay_ptr(int n);
const void* rollout_persistent_ptr(int n);
int rollout_per_warp(int n);
void rollout_set_dense_pct(int pct);
int rollout_threads();
int rollout_advance_threads();

namespace {

uint64_t mix_seed_u64(uint64_t a, uint64_t b) {  // util.hpp:30-35
    uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)
// NVTX ranges (header-only NVTX v3: free unless a profiler is attached) around every device
// entry point, so nsys/ncu timelines show plans, top-Ks, searches and generations by name.
#define MGB_RANGE(name) nvtx3::scoped_range mgb_nvtx_range_{name}

template <class T>
T* dalloc(std::vector<void*>& owned, size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    owned.push_back(p);
    return static_cast<T*>(p);
}

thread_local std::atomic<long long>* g_h2d = nullptr;  // set while an Engine is being constructed

template <class T>
T* upload(std::vector<void*>& owned, const std::vector<T>& v) {
    T* p = dalloc<T>(owned, v.size());
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    if (g_h2d) *g_h2d += static_cast<long long>(v.size() * sizeof(T));
    return p;
}

long long binom(long long a, int k) {
    if (k < 0 || a < k) return 0;
    long long r = 1;
    for (int i = 1; i <= k; ++i) r = r * (a - k + i) / i;
    return r;
}

}  // namespace

// Per-call resources.  Small inputs/outputs live in host-mapped pinned memory that the
// kernels read/write directly, so a greedy or top-K call costs one launch and one
// stream synchronisation (no separate H2D/D2H copies on the latency path).
struct HostIO {
    GreedyState res;       // final greedy state (written by CTA 0)
    int top_n;             // top-K result count
    int pad;
    double comp[256];      // completion vector input
    uint64_t mask[4];      // top-K service filter
    uint64_t top_rows[1024];
    unsigned long long n_scored;  // top-K: rows passing the service mask
};

struct Slot {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    uint64_t* ext = nullptr;
    long long ext_cap = 0;
    GreedyState* st = nullptr;
    Best* partials = nullptr;
    int cap_steps = 0;
    uint64_t* pick_row = nullptr;  // host-mapped
    double* pick_score = nullptr;  // host-mapped
    long long* pick_rows = nullptr;  // host-mapped
    int* ev_svc = nullptr;
    unsigned* bar = nullptr;
    unsigned* ticket = nullptr;  // single-pass top-K last-CTA ticket
    Best* tpart = nullptr;       // single-pass top-K per-CTA lists (32 x 16)
    long long* index = nullptr;
    long long index_cap = 0;
    HostIO* io = nullptr;  // host-mapped

    // device MCTS scratch (mcts.cu), grown on demand, and its pinned host staging (inputs in,
    // the search's outputs back, all on the launch stream: one synchronisation per launch)
    void* mcts_mem = nullptr;
    size_t mcts_bytes = 0;
    unsigned char* mcts_host = nullptr;
    size_t mcts_host_bytes = 0;
    double* logtab = nullptr;
    int logtab_n = 0;

    uint64_t* d_pick_row = nullptr;  // device-side step records
    double* d_pick_score = nullptr;
    long long* d_pick_rows = nullptr;

    void free_picks() {
        for (void* p : {(void*)pick_row, (void*)pick_score, (void*)pick_rows})
            if (p) cudaFreeHost(p);
        for (void* p : {(void*)d_pick_row, (void*)d_pick_score, (void*)d_pick_rows})
            if (p) cudaFree(p);
        pick_row = nullptr;
        pick_score = nullptr;
        pick_rows = nullptr;
        d_pick_row = nullptr;
        d_pick_score = nullptr;
        d_pick_rows = nullptr;
    }
    ~Slot() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (void* p : {(void*)ext, (void*)st, (void*)partials, (void*)ev_svc, (void*)bar, (void*)index,
                        (void*)ticket, (void*)tpart, mcts_mem, (void*)logtab})
            if (p) cudaFree(p);
        free_picks();
        if (io) cudaFreeHost(io);
        if (mcts_host) cudaFreeHost(mcts_host);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (stream) cudaStreamDestroy(stream);
    }
};

bool config_less(const Config& a, const Config& b) {  // GpuConfig operator<, core.hpp:199
    const int m = std::min(a.n, b.n);
    for (int i = 0; i < m; ++i) {
        const auto& x = a.inst[i];
        const auto& y = b.inst[i];
        if (x.slices != y.slices) return x.slices < y.slices;
        if (x.slot != y.slot) return x.slot < y.slot;
        if (x.svc != y.svc) return x.svc < y.svc;
        if (x.batch != y.batch) return x.batch < y.batch;
    }
    return a.n < b.n;
}

bool config_equal(const Config& a, const Config& b) { return !config_less(a, b) && !config_less(b, a); }

Engine::Engine(const Rules& rules, std::map<std::string, ModelProfile> profiles, std::vector<Service> services,
               int max_mix, int device)
    : profiles_(std::move(profiles)), device_(device) {
    MGB_RANGE("migplan: context build");
    const auto tb = std::chrono::steady_clock::now();
    for (const auto& [name, p] : profiles_) validate_profile(p);
    m_ = build_model(rules, profiles_, services, max_mix);

    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    const DeviceInfo& info = device_info(device);  // process-wide: properties + kernel attributes, once
    num_sms_ = info.num_sms;
    const auto t1 = clk::now();

    const int T = kernel_threads();
    // greedy: everything but the row cache is fixed; the cache takes the rest of the
    // opt-in shared memory (one CTA per SM), rounded to whole units per thread.
    // Per-warp TMA slots for rows beyond the on-chip cache (kernels.cu, streaming scan):
    // measured slower at n = 128 than the software-pipelined, L2-prefetched direct loads
    // (4.79 vs 5.1 TB/s on one box, identical plans), so off; MIGPLAN_RING=k enables k stages.
    ring_stages_ = 0;
    if (const char* e = std::getenv("MIGPLAN_RING")) ring_stages_ = std::max(0, std::min(8, std::atoi(e)));
    {
        const long long fixed = static_cast<long long>(greedy_smem_bytes(m_.n, m_.PP, 0, ring_stages_)) + 128;
        long long room = static_cast<long long>(info.smem_optin) - info.greedy_static_smem - 256 - fixed;
        cache_units_ = static_cast<int>(std::max<long long>(0, room / 16) / T * T);
        if (const char* e = std::getenv("MIGPLAN_ROW_CACHE_UNITS"))
            cache_units_ = std::max(0, std::min(cache_units_, std::atoi(e) / T * T));
    }
    const size_t gsm = greedy_smem_bytes(m_.n, m_.PP, cache_units_, ring_stages_), tsm = topk_smem_bytes(m_.n, m_.PP);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&greedy_blocks_per_sm_, greedy_kernel_ptr(), T, gsm));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&topk_blocks_per_sm_, topk_kernel_ptr(), T, tsm));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rollout_blocks_per_sm_, rollout_build_ptr(), rollout_threads(),
                                                     rollout_smem_bytes(m_.n, m_.PP, max_sup())));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rollout_adv_blocks_per_sm_, rollout_advance_ptr(m_.n),
                                                     rollout_advance_threads(), 0));
    if (greedy_blocks_per_sm_ < 1 || topk_blocks_per_sm_ < 1 || rollout_blocks_per_sm_ < 1 || rollout_adv_blocks_per_sm_ < 1)
        throw DeviceError("kernel does not fit on an SM");

    // ---- K1 input: every support with 1..max_mix members and its row offset (pool order)
    std::vector<uint32_t> supports;
    std::vector<long long> offsets;
    long long total = 0;
    {
        std::vector<int> sv(kRowK);
        for (int k = 1; k <= max_mix; ++k) {
            std::function<void(int, int)> rec = [&](int from, int d) {
                if (d == k) {
                    long long c = m_.rows_for_support(sv.data(), k);
                    if (c == 0) return;
                    uint32_t packed = 0xFFFFFFFFu;
                    for (int j = 0; j < k; ++j) packed = (packed & ~(0xFFu << (8 * j))) | (uint32_t(sv[j]) << (8 * j));
                    supports.push_back(packed);
                    offsets.push_back(total);
                    total += c;
                    return;
                }
                for (int v = from; v < m_.n; ++v) {
                    sv[d] = v;
                    rec(v + 1, d + 1);
                }
            };
            rec(0, 0);
        }
    }
    support_off_ = offsets;
    support_off_.push_back(total);

    // ---- device model tables + K1 inputs: one host blob, one allocation, one copy
    std::vector<unsigned char> blob;
    auto put = [&](const void* p, size_t bytes) {
        size_t at = (blob.size() + 15) & ~size_t{15};
        blob.resize(at + std::max<size_t>(bytes, 1));
        if (bytes) std::memcpy(blob.data() + at, p, bytes);
        return at;
    };
    dm_.n = m_.n;
    dm_.PP = m_.PP;
    gk_.phase_timers = std::getenv("MIGPLAN_PHASE_TIMERS") ? 1 : 0;
    if (const char* e = std::getenv("MIGPLAN_PREFETCH")) gk_.prefetch = std::atoi(e);
    if (const char* e = std::getenv("MIGPLAN_PIPE")) gk_.pipeline = std::atoi(e);
    if (const char* e = std::getenv("MIGPLAN_LOAD_MODE")) gk_.load_mode = std::atoi(e);
    if (const char* e = std::getenv("MIGPLAN_EXCH_TIMEOUT_MS")) gk_.exch_timeout_ns = std::atoll(e) * 1'000'000ll;
    dm_.pp_magic = m_.PP > 1 ? static_cast<unsigned>(((1ull << 32) + static_cast<unsigned long long>(m_.PP) - 1) /
                                                     static_cast<unsigned long long>(m_.PP))
                             : 0u;
    dm_.n_sizes = static_cast<int>(m_.sizes.size());
    dm_.n_layouts = static_cast<int>(m_.layouts.size());
    dm_.max_mix = m_.max_mix;
    size_t o_tmpl[kRowK + 1];
    for (int k = 0; k <= kRowK; ++k) {
        std::vector<uint64_t> t;
        for (const auto& tp : m_.templates[k]) {
            uint64_t v = static_cast<uint64_t>(tp.layout);
            for (int j = 0; j < kRowK; ++j) v |= static_cast<uint64_t>(tp.pat[j]) << (8 * (j + 1));
            t.push_back(v);
        }
        dm_.n_tmpl[k] = static_cast<int>(t.size());
        o_tmpl[k] = put(t.data(), t.size() * 8);
    }
    std::vector<uint8_t> pc(static_cast<size_t>(m_.PP) * 5, 0), lc(m_.layouts.size() * 5, 0);
    std::vector<int8_t> ls(m_.layouts.size() * 5 * 7, -1);
    for (int p = 0; p < m_.PP; ++p)
        for (int q = 0; q < kMaxSizes; ++q) pc[p * 5 + q] = m_.patterns[p][q];
    for (size_t l = 0; l < m_.layouts.size(); ++l) {
        for (int q = 0; q < kMaxSizes; ++q) lc[l * 5 + q] = m_.layouts[l].count[q];
        for (const auto& g : m_.layouts[l].groups)
            for (size_t t = 0; t < g.slots.size() && t < 7; ++t)
                ls[(l * 5 + g.size_idx) * 7 + t] = static_cast<int8_t>(g.slots[t]);
    }
    const size_t o_U = put(m_.U.data(), m_.U.size() * 8), o_best = put(m_.best_single.data(), m_.best_single.size() * 8),
                 o_feas = put(m_.feas_mask.data(), m_.feas_mask.size()), o_pm = put(m_.pat_mask.data(), m_.pat_mask.size()),
                 o_pc = put(pc.data(), pc.size()), o_lc = put(lc.data(), lc.size()), o_ls = put(ls.data(), ls.size()),
                 o_sz = put(m_.sizes.data(), m_.sizes.size() * 4), o_sup = put(supports.data(), supports.size() * 4),
                 o_off = put(offsets.data(), offsets.size() * 8);
    std::vector<double> thr(static_cast<size_t>(m_.n) * kMaxSizes, 0.0), req(m_.n, 0.0);
    for (int i = 0; i < m_.n; ++i) {
        req[i] = m_.services[i].req;
        for (size_t si = 0; si < m_.sizes.size(); ++si)
            if (m_.feas[i][si].ok) thr[static_cast<size_t>(i) * kMaxSizes + si] = m_.feas[i][si].thr;
    }
    const size_t o_thr = put(thr.data(), thr.size() * 8), o_req = put(req.data(), req.size() * 8);
    // row_key tables: code -> (service, pattern), pattern -> packed size counts, packed -> layout
    if (m_.PP > 255) throw ArgumentError("partition rules with more than 255 member patterns are not supported");
    std::vector<uint16_t> kcode(static_cast<size_t>(m_.n + 1) * m_.PP, 0);
    for (int c = 0; c < (m_.n + 1) * m_.PP; ++c)
        kcode[c] = static_cast<uint16_t>(((c / m_.PP) << 8) | (c % m_.PP));
    std::vector<uint32_t> ppk(m_.PP, 0u);
    for (int p = 0; p < m_.PP; ++p)
        for (int q = 0; q < kMaxSizes; ++q) ppk[p] |= static_cast<uint32_t>(m_.patterns[p][q] & 7) << (3 * q);
    std::vector<uint8_t> lof(1u << 15, 0xFF);
    for (size_t l = 0; l < m_.layouts.size(); ++l) {
        uint32_t v = 0;
        for (int q = 0; q < kMaxSizes; ++q) v |= static_cast<uint32_t>(m_.layouts[l].count[q] & 7) << (3 * q);
        if (lof[v] == 0xFF) lof[v] = static_cast<uint8_t>(l);
    }
    const size_t o_kc = put(kcode.data(), kcode.size() * 2), o_ppk = put(ppk.data(), ppk.size() * 4),
                 o_lof = put(lof.data(), lof.size());
    const size_t o_base = (blob.size() + 15) & ~size_t{15};
    // from the process-wide scratch pool: closing a context hands it back instead of cudaFree
    // (measured: a cudaFree here took 1-375 ms while the process holds the large greedy arenas)
    ctx_buf_ = std::make_unique<Scratch>(device_, o_base + (static_cast<size_t>(total) + 2) * 8);
    unsigned char* d = static_cast<unsigned char*>(ctx_buf_->get());
    CK(cudaMemcpy(d, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    stats.h2d += static_cast<long long>(blob.size());
    for (int k = 0; k <= kRowK; ++k) dm_.tmpl[k] = reinterpret_cast<const uint64_t*>(d + o_tmpl[k]);
    dm_.U = reinterpret_cast<const double*>(d + o_U);
    dm_.best_single = reinterpret_cast<const double*>(d + o_best);
    dm_.feas_mask = d + o_feas;
    dm_.pat_mask = d + o_pm;
    dm_.pat_count = d + o_pc;
    dm_.layout_count = d + o_lc;
    dm_.layout_slots = reinterpret_cast<const int8_t*>(d + o_ls);
    dm_.sizes = reinterpret_cast<const int*>(d + o_sz);
    dm_.thr = reinterpret_cast<const double*>(d + o_thr);
    dm_.req = reinterpret_cast<const double*>(d + o_req);
    dm_.key_code = reinterpret_cast<const uint16_t*>(d + o_kc);
    dm_.pat_packed = reinterpret_cast<const uint32_t*>(d + o_ppk);
    dm_.layout_of = d + o_lof;
    d_base_ = reinterpret_cast<uint64_t*>(d + o_base);
    const auto t2 = clk::now();

    // ---- K1: base pool rows, deterministic (support, template) order
    if (!supports.empty()) {
        const uint32_t* d_sup = reinterpret_cast<const uint32_t*>(d + o_sup);
        const long long* d_off = reinterpret_cast<const long long*>(d + o_off);
        int n_sup = static_cast<int>(supports.size());
        int threads = 256;
        int blocks = static_cast<int>((static_cast<long long>(n_sup) * 32 + threads - 1) / threads);
        void* args[] = {&dm_, &d_sup, &d_off, &n_sup, &d_base_};
        CK(cudaLaunchKernel(enum_base_kernel_ptr(), blocks, threads, args, 0, nullptr));
        stats.launches++;
        CK(cudaGetLastError());
    }
    base_rows_.resize(static_cast<size_t>(total));
    if (total) CK(cudaMemcpy(base_rows_.data(), d_base_, total * 8, cudaMemcpyDeviceToHost));
    stats.d2h += total * 8;
    const auto t3 = clk::now();
    if (std::getenv("MIGPLAN_CTX_TIMERS")) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "[migplan ctx] n=%d model %.0f us, device info %.0f us, tables %.0f us, K1+base %.0f us\n",
                     m_.n, us(tb, t0), us(t0, t1), us(t1, t2), us(t2, t3));
    }

    min_u_.assign(m_.n, 0.0);
    for (int i = 0; i < m_.n; ++i) {
        double mu = 0.0;
        for (int p = 0; p < m_.PP; ++p) {
            double u = m_.U[static_cast<size_t>(i) * m_.PP + p];
            if (u > 0.0 && (mu == 0.0 || u < mu)) mu = u;
        }
        min_u_[i] = mu;
    }
    // extension arena bound: every support with max_mix < |S| <= 4 (all templates).
    long double eb = 0;
    for (int k = max_mix + 1; k <= kRowK; ++k) eb += static_cast<long double>(binom(m_.n, k)) * m_.templates[k].size();
    ext_bound_ = static_cast<long long>(std::min<long double>(eb, 1ll << 31)) + 64;
}

// Working-set bound of a plan started from `comp`: the base pool plus every extension support
// over the services still unsatisfied there (an extension only ever adds supports inside the
// unsatisfied set, greedy.hpp:107-119).
long long Engine::working_set_bound(const double* comp) const {
    int u = 0;
    for (int i = 0; i < m_.n; ++i) u += comp[i] < 1.0 - kSatisfyEps ? 1 : 0;
    long double eb = 0;
    for (int k = m_.max_mix + 1; k <= kRowK; ++k) eb += static_cast<long double>(binom(u, k)) * m_.templates[k].size();
    return pool_size() + static_cast<long long>(std::min<long double>(eb, 1ll << 40));
}

const unsigned* Engine::keyrank() {
    std::call_once(keyrank_once_, [&] {
        const long long P = static_cast<long long>(base_rows_.size());
        CK(cudaSetDevice(device_));
        keyrank_buf_ = std::make_unique<Scratch>(device_, sizeof(unsigned) * std::max<long long>(P, 1));
        d_keyrank_ = static_cast<unsigned*>(keyrank_buf_->get());
        int l = 0;
        const size_t need = keyrank_scratch_bytes(P);
        Scratch tmp(device_, need);
        CK(build_keyrank(dm_, d_base_, P, d_keyrank_, tmp.get(), need, nullptr, &l));
        stats.launches += l;
    });
    return d_keyrank_;
}

void Engine::support_tables() {
    std::call_once(sup_once_, [&] {
        const int ns = static_cast<int>(support_off_.size()) - 1;
        if (ns <= 0 || m_.max_mix > 2) return;
        std::vector<int> begin(ns + 1);
        std::vector<unsigned short> svc(ns);
        for (int i = 0; i <= ns; ++i) begin[i] = static_cast<int>(support_off_[i]);
        for (int i = 0; i < ns; ++i) {
            int sv[kRowK], pt[kRowK];
            const int k = support_off_[i] < support_off_[i + 1] ? m_.members(base_rows_[support_off_[i]], sv, pt) : 0;
            if (k < 1 || k > 2) return;  // not a pair pool: scan every row
            svc[i] = static_cast<unsigned short>(sv[0] | ((k == 2 ? sv[1] : 0xFF) << 8));
        }
        const size_t bb = sizeof(int) * (ns + 1), sb = sizeof(unsigned short) * ns;
        sup_buf_ = std::make_unique<Scratch>(device_, bb + sb + 16);
        unsigned char* d = static_cast<unsigned char*>(sup_buf_->get());
        CK(cudaSetDevice(device_));
        CK(cudaMemcpy(d, begin.data(), bb, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d + bb, svc.data(), sb, cudaMemcpyHostToDevice));
        d_sup_begin_ = reinterpret_cast<const int*>(d);
        d_sup_svc_ = reinterpret_cast<const unsigned short*>(d + bb);
        n_sup_ = ns;
    });
}

const unsigned* Engine::base32() {
    std::call_once(base32_once_, [&] {
        const size_t P = base_rows_.size();
        std::vector<unsigned> lo(std::max<size_t>(P, 1));
        for (size_t i = 0; i < P; ++i) lo[i] = static_cast<unsigned>(base_rows_[i]);
        CK(cudaSetDevice(device_));
        base32_buf_ = std::make_unique<Scratch>(device_, sizeof(unsigned) * lo.size());
        CK(cudaMemcpy(base32_buf_->get(), lo.data(), sizeof(unsigned) * lo.size(), cudaMemcpyHostToDevice));
    });
    return static_cast<const unsigned*>(base32_buf_->get());
}

Engine::~Engine() {
    const auto t0 = std::chrono::steady_clock::now();
    cudaSetDevice(device_);
    if (d_shard_) cudaFree(d_shard_);
    for (void* p : dev_allocs_) cudaFree(p);
    if (std::getenv("MIGPLAN_HOST_TIMERS"))
        std::fprintf(stderr, "[host] context free: %.1f us (%zu device buffers)\n",
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(), dev_allocs_.size());
}

long long Engine::index_of(uint64_t row) const {
    std::call_once(row_index_once_, [this] {  // built on first use: not on the context-creation path
        row_index_.reserve(base_rows_.size() * 2);
        for (size_t i = 0; i < base_rows_.size(); ++i) row_index_.emplace(base_rows_[i], static_cast<long long>(i));
    });
    auto it = row_index_.find(row);
    if (it == row_index_.end()) throw ArgumentError("row not in the base pool");
    return it->second;
}

Config Engine::config_of(uint64_t row) const {
    Config c;
    c.n = m_.decode(row, c.inst);
    return c;
}

Config Engine::config_of_wide(const uint4& row) const {  // bf.cu's 8-code rows
    const unsigned w[4] = {row.x, row.y, row.z, row.w};
    int svc[kBfCodes], pat[kBfCodes], k = 0;
    for (int j = 0; j < kBfCodes; ++j) {
        const int code = static_cast<int>((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        if (code >= m_.n * m_.PP) break;
        svc[k] = code / m_.PP;
        pat[k++] = code % m_.PP;
    }
    Config c;
    c.n = m_.decode_members(svc, pat, k, c.inst);
    return c;
}

const DeviceInfo& device_info(int device) {
    static std::mutex mu;
    static std::map<int, DeviceInfo> cache;  // one entry per device for the process lifetime
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(device);
    if (it != cache.end()) {
        CK(cudaSetDevice(device));
        return it->second;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw DeviceError("no CUDA device available: the B200 planner has no CPU fallback");
    if (device < 0 || device >= ndev) throw DeviceError("CUDA device index out of range");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw DeviceError(std::string("device ") + prop.name + " is not sm_100-class (B200)");
    DeviceInfo info;
    info.num_sms = prop.multiProcessorCount;
    info.smem_optin = static_cast<long long>(prop.sharedMemPerBlockOptin);
    // every kernel may use all the opt-in shared memory its static allocation leaves
    CK(cudaFuncSetAttribute(topk1_kernel_ptr(32), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(mcts_kernel_ptr(1), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(mcts_kernel_ptr(255), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(greedy_kernel_ptr(), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (const void* k : {greedy_kernel_ptr(), topk_kernel_ptr(), topk1_kernel_ptr(32), rollout_build_ptr(), rollout_persistent_ptr(1), rollout_persistent_ptr(256),
                          mcts_kernel_ptr(1), mcts_kernel_ptr(255)}) {
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, k));
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(prop.sharedMemPerBlockOptin - fa.sharedSizeBytes)));
        if (k == mcts_kernel_ptr(1) || k == mcts_kernel_ptr(255))  // the larger of the two variants
            info.mcts_static_smem = std::max(info.mcts_static_smem, static_cast<long long>(fa.sharedSizeBytes));
        if (k == greedy_kernel_ptr()) info.greedy_static_smem = static_cast<long long>(fa.sharedSizeBytes);
    }
    return cache.emplace(device, info).first->second;
}

namespace {

// Per-call resources are context-independent (sized for n <= 255 and any grid), so they are
// pooled per device for the whole process: creating a PlanContext (the e2e path) never
// pays for stream creation, pinned-mapped host allocations or arena cudaMallocs twice.
struct SlotPool {
    std::mutex mu;
    std::vector<Slot*> free;
};
SlotPool& slot_pool(int device) {
    static std::mutex m;
    static std::map<int, SlotPool*> pools;  // intentionally leaked: lives until process exit
    std::lock_guard<std::mutex> g(m);
    auto& p = pools[device];
    if (!p) p = new SlotPool;
    return *p;
}

}  // namespace

namespace {

// Process-wide pool of device scratch buffers (per device, power-of-two size classes): the
// per-call temporaries of the GA phases and the per-context key ranks never pay cudaMalloc /
// cudaFree (a device-wide synchronization) inside a plan.
struct ScratchPool {
    std::mutex mu;
    std::multimap<size_t, void*> free;
};
ScratchPool& scratch_pool(int device) {
    static std::mutex m;
    static std::map<int, ScratchPool*> pools;  // intentionally leaked: lives until process exit
    std::lock_guard<std::mutex> g(m);
    auto& p = pools[device];
    if (!p) p = new ScratchPool;
    return *p;
}

}  // namespace

// Frees every pooled slot and scratch buffer of `device` not in use by a live call (the
// next context pays the cold allocations again: bench.py's cold e2e).
const void* philox_kat_kernel_ptr();
uint64_t philox_on_device(int device, uint64_t seed, uint64_t stream, uint64_t step) {
    CK(cudaSetDevice(device));
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof *d));
    void* args[] = {&seed, &stream, &step, &d};
    CK(cudaLaunchKernel(philox_kat_kernel_ptr(), 1, 1, args, 0, nullptr));
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return h;
}

// The rollout calls' cached buffers and streams, per device (process lifetime, like the slots).
struct RoCache {
    std::mutex mu;
    struct Blk {
        void* p;
        size_t n;
        bool host, used;
    };
    std::vector<Blk> blocks;
    struct Strm {
        cudaStream_t s;
        cudaEvent_t e0, e1;
        bool used;
    };
    std::deque<Strm> streams;  // deque: entries stay put while others are added
};
RoCache& ro_cache(int device) {
    static std::mutex m;
    static std::map<int, RoCache*> caches;  // intentionally leaked: lives until process exit
    std::lock_guard<std::mutex> g(m);
    auto& c = caches[device];
    if (!c) c = new RoCache;
    return *c;
}

void release_device_cache(int device) {
    {  // unused rollout buffers
        RoCache& rc = ro_cache(device);
        std::lock_guard<std::mutex> g(rc.mu);
        CK(cudaSetDevice(device));
        std::vector<RoCache::Blk> keep;
        for (auto& b : rc.blocks) {
            if (b.used)
                keep.push_back(b);
            else
                b.host ? cudaFreeHost(b.p) : cudaFree(b.p);
        }
        rc.blocks.swap(keep);
    }
    std::vector<Slot*> slots;
    {
        SlotPool& pool = slot_pool(device);
        std::lock_guard<std::mutex> g(pool.mu);
        slots.swap(pool.free);
    }
    for (Slot* s : slots) delete s;
    std::vector<void*> bufs;
    {
        ScratchPool& pool = scratch_pool(device);
        std::lock_guard<std::mutex> g(pool.mu);
        for (auto& [k, p] : pool.free) bufs.push_back(p);
        pool.free.clear();
    }
    CK(cudaSetDevice(device));
    for (void* p : bufs) cudaFree(p);
}

Scratch::Scratch(int device, size_t bytes) : device_(device) {
    size_t cls = 4096;
    while (cls < bytes) cls <<= 1;
    bytes_ = cls;
    ScratchPool& pool = scratch_pool(device);
    {
        std::lock_guard<std::mutex> g(pool.mu);
        auto it = pool.free.lower_bound(cls);
        if (it != pool.free.end() && it->first == cls) {
            p_ = it->second;
            pool.free.erase(it);
            return;
        }
    }
    CK(cudaMalloc(&p_, cls));
}

Scratch::~Scratch() {
    if (!p_) return;
    ScratchPool& pool = scratch_pool(device_);
    std::lock_guard<std::mutex> g(pool.mu);
    pool.free.emplace(bytes_, p_);
}

Slot* Engine::acquire() {
    SlotPool& pool = slot_pool(device_);
    {
        std::lock_guard<std::mutex> g(pool.mu);
        if (!pool.free.empty()) {
            Slot* s = pool.free.back();
            pool.free.pop_back();
            return s;
        }
    }
    CK(cudaSetDevice(device_));
    auto s = std::make_unique<Slot>();
    s->device = device_;
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&s->e0));
    CK(cudaEventCreate(&s->e1));
    CK(cudaMalloc(&s->st, sizeof(GreedyState)));
    CK(cudaMalloc(&s->partials, sizeof(Best) * 2 * 1024));
    CK(cudaMalloc(&s->ev_svc, sizeof(int) * (kMaxServices + 1)));
    CK(cudaMalloc(&s->bar, sizeof(unsigned) * 2));
    CK(cudaMemset(s->bar, 0, sizeof(unsigned) * 2));
    CK(cudaMalloc(&s->ticket, sizeof(unsigned)));
    CK(cudaMemset(s->ticket, 0, sizeof(unsigned)));
    CK(cudaMalloc(&s->tpart, sizeof(Best) * kTopkMaxCtas * 32));
    CK(cudaHostAlloc(&s->io, sizeof(HostIO), cudaHostAllocMapped));
    std::memset(s->io, 0, sizeof(HostIO));
    return s.release();
}

void Engine::release(Slot* s) {
    SlotPool& pool = slot_pool(device_);
    std::lock_guard<std::mutex> g(pool.mu);
    pool.free.push_back(s);
}

void Engine::ensure_ext(Slot* s, long long rows) {
    if (s->ext_cap >= rows) return;
    if (s->ext) CK(cudaFree(s->ext));
    s->ext = nullptr;
    CK(cudaMalloc(&s->ext, static_cast<size_t>(rows + 2) * sizeof(uint64_t)));
    s->ext_cap = rows;
}

long long Engine::step_bound(const std::vector<double>& comp) const {
    long long b = 1;
    for (int i = 0; i < m_.n; ++i) {
        double need = 1.0 - comp[i];
        if (need <= 0.0 || min_u_[i] <= 0.0) continue;
        b += static_cast<long long>(std::ceil(need / min_u_[i])) + 1;
    }
    return b;
}

void Engine::fast_algo(const std::vector<double>& comp, std::vector<uint64_t>& rows, std::vector<double>& scores) {
    fast_algo_group({this}, comp, rows, scores);
}

// Per-call resources and arguments of one greedy instance.
struct GreedyCall {
    Engine* e = nullptr;
    Slot* s = nullptr;
    long long n_base = 0;
    const uint64_t* base_src = nullptr;
    GreedyArgs a{};
};

void Engine::greedy_prepare(GreedyCall& c, const double* comp_host, const double* comp_dev, long long cap_steps,
                            cudaStream_t st, bool defer_init) {
    Slot* s = c.s;
    if (!st) st = s->stream;
    CK(cudaSetDevice(device_));
    if (s->cap_steps < cap_steps) {
        s->free_picks();
        CK(cudaHostAlloc(&s->pick_row, sizeof(uint64_t) * cap_steps, cudaHostAllocMapped));
        CK(cudaHostAlloc(&s->pick_score, sizeof(double) * cap_steps, cudaHostAllocMapped));
        CK(cudaHostAlloc(&s->pick_rows, sizeof(long long) * cap_steps, cudaHostAllocMapped));
        CK(cudaMalloc(&s->d_pick_row, sizeof(uint64_t) * cap_steps));
        CK(cudaMalloc(&s->d_pick_score, sizeof(double) * cap_steps));
        CK(cudaMalloc(&s->d_pick_rows, sizeof(long long) * cap_steps));
        s->cap_steps = static_cast<int>(cap_steps);
    }
    c.n_base = n_ranks_ > 1 ? n_shard_ : static_cast<long long>(base_rows_.size());
    c.base_src = n_ranks_ > 1 ? d_shard_ : d_base_;
    // Arena = base + the all-feasible extension bound (every support with max_mix < |S| <= 4),
    // capped at 3G rows (24 GB); the kernel reports overflow and the call is retried larger.
    ensure_ext(s, c.n_base + std::min<long long>(ext_bound_, 3ll << 30));
    if (comp_host) std::memcpy(s->io->comp, comp_host, sizeof(double) * m_.n);
    if (!defer_init) {  // (greedy_batch: one launch_greedy_batch_init for every instance instead)
        CK(cudaMemsetAsync(s->st, 0, sizeof(GreedyState), st));
        // the working-set arena starts as a copy of the resident base pool (device to device)
        if (c.n_base) CK(cudaMemcpyAsync(s->ext, c.base_src, c.n_base * 8, cudaMemcpyDeviceToDevice, st));
    }
    GreedyArgs& a = c.a;
    a = GreedyArgs{};
    a.M = dm_;
    a.rows = s->ext;
    a.n_base = c.n_base;
    a.cap = s->ext_cap;
    a.cache_units = cache_units_;
    a.ring_stages = ring_stages_;
    a.phase_timers = gk_.phase_timers;
    a.prefetch = gk_.prefetch;
    a.pipeline = gk_.pipeline;  // software-pipelined streaming loads (MIGPLAN_PIPE=0: off)
    a.load_mode = gk_.load_mode;  // ld.global.cs: measured best for the streaming scan (profiles/)
    a.comp0 = comp_host ? s->io->comp : comp_dev;
    a.st = s->st;
    a.out = &s->io->res;
    a.partials = s->partials;
    a.pick_row = s->d_pick_row;
    a.pick_score = s->d_pick_score;
    a.pick_rows = s->d_pick_rows;
    a.host_pick_row = s->pick_row;
    a.host_pick_score = s->pick_score;
    a.host_pick_rows = s->pick_rows;
    a.ev_svc = s->ev_svc;
    a.cap_steps = s->cap_steps;
    a.n_ranks = n_ranks_;
    a.rank = rank_;
    for (int q = 0; q < n_ranks_ && n_ranks_ > 1; ++q) a.boards[q] = static_cast<ExchSlot*>(boards_[q]);
    a.exch_seq0 = exch_seq_;
    a.exch_timeout_ns = gk_.exch_timeout_ns;
}

// Returns false when the arena overflowed and was grown (the caller relaunches).
bool Engine::greedy_finish(GreedyCall& c, float ms, int attempt, std::vector<uint64_t>& rows, std::vector<double>& scores) {
    Slot* s = c.s;
    const GreedyState h = s->io->res;
    if (n_ranks_ > 1) {
        if (h.status == kExtOverflow || h.status == kExchTimeout) {
            n_ranks_ = 1;  // the ranks' exchange sequences diverged: the shard must be set again
            throw DeviceError(h.status == kExchTimeout ? "sharded greedy: exchange with a peer rank timed out"
                                                       : "sharded greedy: extension arena overflow");
        }
        exch_seq_ = h.last_seq;
    }
    if (h.status == kExtOverflow && attempt < 4) {
        long long need = c.n_base + static_cast<long long>(h.ext_count) * 4 + (1 << 20);
        ensure_ext(s, std::max(need, s->ext_cap * 2));
        return false;
    }
    if (h.status == kExtOverflow) throw DeviceError("extension arena overflow");
    if (h.status == kStepOverflow) throw DeviceError("greedy step buffer overflow");
    rows.assign(s->pick_row, s->pick_row + h.n_steps);
    scores.assign(s->pick_score, s->pick_score + h.n_steps);
    {
        std::lock_guard<std::mutex> g(diag_mu_);
        last_step_rows_.assign(s->pick_rows, s->pick_rows + h.n_steps);
    }
    stats.greedy_ns += static_cast<long long>(ms * 1e6f);
    stats.h2d += static_cast<long long>(sizeof(double) * m_.n);
    stats.d2h += static_cast<long long>(sizeof(GreedyState) + (sizeof(uint64_t) + sizeof(double) + sizeof(long long)) *
                                                                  h.n_steps);
    stats.greedy_rows += h.rows_scored;
    stats.greedy_calls++;
    stats.greedy_steps += h.n_steps;
    stats.ext_events += h.n_events;
    stats.ext_rows += static_cast<long long>(h.ext_count);
    for (int k = 0; k < 5; ++k) stats.phase_ns[k] += static_cast<long long>(h.phase_ns[k]);
    if (std::getenv("MIGPLAN_PHASE_TIMERS")) {
        unsigned long long sk = 0, rl = 0;
        greedy_read_diag(&sk, &rl);
        std::fprintf(stderr, "[greedy] cumulative arrival skew (last CTA - CTA 0) %.3f ms, reduce+release %.3f ms\n",
                     sk * 1e-6, rl * 1e-6);
    }
    if (h.status == kNoPositive)
        throw PlanningError("fast_algo: no config with positive score while services remain unsatisfied");
    return true;
}
// Greedy launch: cooperative (grid-wide barriers over every SM) or, for small working sets,
// one thread-block cluster per instance (DSMEM argmax and cluster barriers: a step costs a
// few microseconds instead of a grid-wide barrier over 148 CTAs).
void launch_greedy_batch_init(const GreedyLaunch& L, const uint64_t* base, long long n_base, cudaStream_t st);
void launch_greedy(const GreedyLaunch& L, int T, size_t smem, cudaStream_t st) {
    void* args[] = {const_cast<GreedyLaunch*>(&L)};
    if (!L.cluster) {
        CK(cudaLaunchCooperativeKernel(greedy_kernel_ptr(), L.n_groups * L.ctas_per_group, T, args, smem, st));
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.n_groups * L.ctas_per_group);
    cfg.blockDim = dim3(T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = L.ctas_per_group;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelExC(&cfg, greedy_kernel_ptr(), args));
}

// Deal 32-unit blocks round-robin over the G CTAs instead of 512 contiguous units per CTA
// (MIGPLAN_INTERLEAVE=1, only when the working-set bound fits the G row caches).  Measured
// neutral at n = 24 (the per-step CTA skew is not a row-distribution effect), so off.
int Engine::greedy_interleave(int G) const {
    const char* v = std::getenv("MIGPLAN_INTERLEAVE");
    if (!v || std::atoi(v) == 0) return 0;
    const long long cap_rows = 2ll * cache_units_ * G;
    return n_ranks_ == 1 && ring_stages_ == 0 && pool_size() + ext_bound_ <= cap_rows ? 1 : 0;
}

// CTAs per instance in cluster mode (0: cooperative).  Cluster mode when the working set
// stays small: the base pool plus the extension bound (bench.hpp-style closed form) under
// kClusterRows; MIGPLAN_GREEDY_CLUSTER=0 disables it, =k forces k CTAs.
int Engine::greedy_cluster_ctas(size_t smem, long long rows_bound) const {
    if (n_ranks_ > 1) return 0;
    constexpr long long kClusterRows = 256ll << 10;
    if (rows_bound < 0) rows_bound = pool_size() + ext_bound_;
    static const int small = [] {  // CTAs per small instance (MIGPLAN_GREEDY_CLUSTER_SMALL: A/B)
        const char* e = std::getenv("MIGPLAN_GREEDY_CLUSTER_SMALL");
        return e ? std::max(2, std::min(16, std::atoi(e))) : 8;  // 8: GA refills 5.5 -> 5.0 ms per GA10 (16 and 4 slower)
    }();
    int want = rows_bound <= kClusterRows ? small : 0;
    const char* v = std::getenv("MIGPLAN_GREEDY_CLUSTER");
    if (v) want = std::max(0, std::min(16, std::atoi(v)));
    if (want == 0) return 0;
    const bool cacheable = !v;
    if (cacheable && cluster_ctas_ >= 0) return cluster_ctas_;  // the occupancy query is per context
    auto done = [&](int r) {
        if (cacheable) cluster_ctas_ = r;
        return r;
    };
    for (; want >= 2; want >>= 1) {  // the largest size the GPU can co-schedule
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(want);
        cfg.blockDim = dim3(kernel_threads());
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = want;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, greedy_kernel_ptr(), &cfg) == cudaSuccess && nc > 0)
            return done(want);
        cudaGetLastError();
    }
    return done(0);
}


// fast_algo on one engine, or on the ranks of a sharded greedy that share this GPU: their
// instances run as CTA ranges of ONE cooperative launch (GreedyLaunch), so the per-step
// exchange between them never waits on a kernel that is not resident.
void Engine::fast_algo_group(const std::vector<Engine*>& es, const std::vector<double>& comp,
                             std::vector<uint64_t>& rows, std::vector<double>& scores) {
    MGB_RANGE("migplan: fast_algo");
    rows.clear();
    scores.clear();
    const int P = static_cast<int>(es.size());
    if (P < 1 || P > kMaxRanks) throw ArgumentError("fast_algo: 1..8 contexts per group");
    Engine* e0 = es[0];
    for (Engine* e : es) {
        if (e->device_ != e0->device_) throw ArgumentError("fast_algo group: contexts on different devices");
        if (P > 1 && (e->n_ranks_ != P || e->max_ctas_ != es[0]->max_ctas_))
            throw ArgumentError("fast_algo group: every context must be one rank of a P-way shard");
    }
    for (int r = 0; r < P && P > 1; ++r)
        if (es[r]->rank_ != r) throw ArgumentError("fast_algo group: contexts must be in rank order");
    if (static_cast<int>(comp.size()) != e0->m_.n) throw PlanningError("fast_algo: completion vector length mismatch");
    bool sat = true;
    for (double c : comp)
        if (c < 1.0 - kSatisfyEps) sat = false;
    if (sat) return;  // greedy.hpp:101

    std::vector<GreedyCall> calls(P);
    struct Rel {
        std::vector<GreedyCall>& c;
        ~Rel() {
            for (auto& x : c)
                if (x.s) x.e->release(x.s);
        }
    } rel{calls};
    for (int r = 0; r < P; ++r) {
        calls[r].e = es[r];
        calls[r].s = es[r]->acquire();
    }
    const int T = kernel_threads();
    const size_t smem = greedy_smem_bytes(e0->m_.n, e0->m_.PP, e0->cache_units_, e0->ring_stages_);
    int G = e0->num_sms_ * e0->greedy_blocks_per_sm_ / P;
    if (e0->max_ctas_ > 0) G = std::min(G, e0->max_ctas_);
    if (const char* v = std::getenv("MIGPLAN_GREEDY_CTAS")) G = std::max(1, std::min(G, std::atoi(v)));
    const int GC = P == 1 ? e0->greedy_cluster_ctas(smem, e0->working_set_bound(comp.data())) : 0;
    if (GC) G = GC;
    Slot* s0 = calls[0].s;
    for (int attempt = 0;; ++attempt) {
        GreedyLaunch L{};
        L.n_groups = P;
        L.ctas_per_group = G;
        L.cluster = GC ? 1 : 0;
        const long long cap_steps = std::min<long long>(e0->step_bound(comp), 1 << 24);
        for (int r = 0; r < P; ++r) {
            es[r]->greedy_prepare(calls[r], comp.data(), nullptr, cap_steps);
            calls[r].a.interleave = es[r]->greedy_interleave(G);
            L.g[r] = calls[r].a;
        }
        for (int r = 1; r < P; ++r) CK(cudaStreamSynchronize(calls[r].s->stream));  // their arena copies
        CK(cudaEventRecord(s0->e0, s0->stream));
        launch_greedy(L, T, smem, s0->stream);
        for (Engine* e : es) e->stats.launches++;
        CK(cudaEventRecord(s0->e1, s0->stream));
        CK(cudaStreamSynchronize(s0->stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, s0->e0, s0->e1));
        bool done = true;
        for (int r = 0; r < P; ++r) {
            std::vector<uint64_t> rr;
            std::vector<double> ss;
            if (!es[r]->greedy_finish(calls[r], ms, attempt, rr, ss)) done = false;
            if (r == 0) {
                rows = std::move(rr);
                scores = std::move(ss);
            } else if (done && rr != rows) {
                throw DeviceError("sharded greedy: ranks disagree on the plan");
            }
        }
        if (done) return;
        if (P > 1) throw DeviceError("sharded greedy: extension arena overflow");
    }
}

std::vector<long long> Engine::topk(const std::vector<double>& comp, int k, const std::vector<long long>* index,
                                    const std::vector<uint64_t>* svc_mask) {
    MGB_RANGE("migplan: topk_candidates");
    if (static_cast<int>(comp.size()) != m_.n) throw PlanningError("completion vector length mismatch");
    std::vector<long long> out;
    if (k <= 0) return out;
    k = std::min(k, 1024);
    const long long total = index ? static_cast<long long>(index->size()) : pool_size();
    if (total == 0) return out;
    Slot* s = acquire();
    struct Rel {
        Engine* e;
        Slot* s;
        ~Rel() { e->release(s); }
    } rel{this, s};
    CK(cudaSetDevice(device_));
    std::memcpy(s->io->comp, comp.data(), sizeof(double) * m_.n);
    if (svc_mask) std::memcpy(s->io->mask, svc_mask->data(), sizeof(uint64_t) * 4);
    if (index) {
        if (s->index_cap < total) {
            if (s->index) CK(cudaFree(s->index));
            CK(cudaMalloc(&s->index, sizeof(long long) * total));
            s->index_cap = total;
        }
        CK(cudaMemcpyAsync(s->index, index->data(), sizeof(long long) * total, cudaMemcpyHostToDevice, s->stream));
    }
    CK(cudaEventRecord(s->e0, s->stream));
    // spread the scan over many SMs (one SM alone is issue-bound: ~30 us for 17K rows);
    // the last-CTA merge ranks only rows above the per-CTA K-th scores
    long long per = std::max<long long>(topk1_rows_per_cta(), (total + topk1_max_ctas() - 1) / topk1_max_ctas());
    if (total > (1ll << 22)) per = total + 1;  // huge explicit lists: the exact k-round kernel below
    if (const char* e = std::getenv("MIGPLAN_TOPK_ROWS_PER_CTA")) per = std::max(256ll, std::atoll(e));
    const long long g1 = (total + per - 1) / per;
    bool single = k <= 32 && g1 <= topk1_max_ctas();
    if (single) {  // one launch: per-CTA threshold + parallel rank, last-CTA merge (topk.cu)
        Topk1Args a{};
        a.M = dm_;
        a.rows = d_base_;
        a.n_rows = pool_size();
        a.index = index ? s->index : nullptr;
        a.n_index = index ? total : 0;
        a.use_mask = svc_mask ? 1 : 0;
        if (svc_mask) std::memcpy(a.svc_mask, svc_mask->data(), sizeof(uint64_t) * 4);
        std::memcpy(a.comp, comp.data(), sizeof(double) * m_.n);
        a.k = k;
        a.rows_per_cta = per;
        a.partials = s->tpart;
        a.ticket = s->ticket;
        a.out_row = s->io->top_rows;
        a.n_out = &s->io->top_n;
        a.n_scored = &s->io->n_scored;
        s->io->n_scored = 0;
        const int G = static_cast<int>(std::max<long long>(g1, 1));
        a.rows_per_cta = (total + G - 1) / G;
        void* args[] = {&a};
        // the grid is one thread-block cluster: the CTAs merge their winners over DSMEM
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(topk1_threads());
        cfg.dynamicSmemBytes = topk1_smem_bytes(m_.n, m_.PP, 32);
        cfg.stream = s->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelExC(&cfg, topk1_kernel_ptr(32), args));
        stats.launches++;
        CK(cudaEventRecord(s->e1, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        // *n_out == -1: a CTA's rows tied at its threshold beyond the candidate capacity;
        // the exact k-round kernel below answers instead.
        single = s->io->top_n >= 0;
        if (!single) CK(cudaMemsetAsync(s->ticket, 0, sizeof(unsigned), s->stream));
    }
    if (!single) {  // k rounds with grid barriers (k > 32, huge lists, or tie overflow)
        TopkArgs a{};
        a.M = dm_;
        a.rows = d_base_;
        a.n_rows = pool_size();
        a.index = index ? s->index : nullptr;
        a.n_index = index ? total : 0;
        a.svc_mask = svc_mask ? s->io->mask : nullptr;
        a.comp = s->io->comp;
        a.k = k;
        a.bar = s->bar;
        a.partials = s->partials;
        a.out_row = s->io->top_rows;
        a.n_out = &s->io->top_n;
        const int T = kernel_threads();
        int G = static_cast<int>(std::min<long long>((total + 4 * T - 1) / (4 * T), num_sms_ * topk_blocks_per_sm_));
        G = std::max(G, 1);
        void* args[] = {&a};
        CK(cudaLaunchCooperativeKernel(topk_kernel_ptr(), G, T, args, topk_smem_bytes(m_.n, m_.PP), s->stream));
        stats.launches++;
        CK(cudaEventRecord(s->e1, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    }
    const int got = s->io->top_n;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s->e0, s->e1));
    stats.topk_ns += static_cast<long long>(ms * 1e6f);
    // rows scored (mcts.hpp:59-67): the candidate list, or for expand's service filter the
    // rows touching a sampled service (the union of by_service lists, mcts.hpp:98-107)
    long long scored = total;
    if (svc_mask && single) {
        scored = static_cast<long long>(s->io->n_scored);
    } else if (svc_mask) {  // exact k-round fallback: count the filtered set on the host
        scored = 0;
        for (uint64_t row : base_rows_) {
            int svc[kRowK], pat[kRowK];
            const int k2 = m_.members(row, svc, pat);
            bool hit = false;
            for (int j = 0; j < k2; ++j) hit |= (((*svc_mask)[svc[j] >> 6] >> (svc[j] & 63)) & 1ull) != 0;
            scored += hit;
        }
    }
    stats.topk_rows += scored;
    stats.topk_calls++;
    stats.h2d += static_cast<long long>(sizeof(double) * m_.n + (index ? sizeof(long long) * total : 0) +
                                        (svc_mask ? 32 : 0));
    stats.d2h += static_cast<long long>(sizeof(int) + sizeof(uint64_t) * got);
    for (int i = 0; i < got; ++i) out.push_back(index_of(s->io->top_rows[i]));
    return out;
}

// Root-parallel rollouts (rollout.cu).  Device buffers live for the call; the key cache
// persists across the call's batches (the reference's RolloutCache lives for one
// mcts_solve call, mcts.hpp:158).  A full key cache restarts the call with 4x capacity.
void* Engine::ro_get(size_t bytes, bool host) {
    bytes = std::max<size_t>(bytes, 16);
    RoCache& rc = ro_cache(device_);
    {
        std::lock_guard<std::mutex> g(rc.mu);
        int best = -1;
        for (int i = 0; i < static_cast<int>(rc.blocks.size()); ++i) {  // best fit, at most 4x the request
            const RoCache::Blk& b = rc.blocks[i];
            if (!b.used && b.host == host && b.n >= bytes && b.n <= 4 * bytes + (1 << 20) &&
                (best < 0 || b.n < rc.blocks[best].n))
                best = i;
        }
        if (best >= 0) {
            rc.blocks[best].used = true;
            return rc.blocks[best].p;
        }
    }
    void* p = nullptr;
    if (host)
        CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped));
    else
        CK(cudaMalloc(&p, bytes));
    std::lock_guard<std::mutex> g(rc.mu);
    rc.blocks.push_back(RoCache::Blk{p, bytes, host, true});
    return p;
}
void Engine::ro_put(void* p) {
    RoCache& rc = ro_cache(device_);
    std::lock_guard<std::mutex> g(rc.mu);
    for (auto& b : rc.blocks)
        if (b.p == p) b.used = false;
}
int Engine::ro_stream() {
    RoCache& rc = ro_cache(device_);
    {
        std::lock_guard<std::mutex> g(rc.mu);
        for (int i = 0; i < static_cast<int>(rc.streams.size()); ++i)
            if (!rc.streams[i].used) {
                rc.streams[i].used = true;
                return i;
            }
    }
    RoCache::Strm x{};
    CK(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
    CK(cudaEventCreate(&x.e0));
    CK(cudaEventCreate(&x.e1));
    x.used = true;
    std::lock_guard<std::mutex> g(rc.mu);
    rc.streams.push_back(x);
    return static_cast<int>(rc.streams.size()) - 1;
}
void Engine::ro_stream_put(int i) {
    RoCache& rc = ro_cache(device_);
    std::lock_guard<std::mutex> g(rc.mu);
    rc.streams[i].used = false;
}

RolloutResult Engine::rollouts(const std::vector<double>& comp, long long n_roll, int k, int max_depth, uint64_t seed,
                               long long id_offset, long long batch, int table_log2, int* lengths) {
    MGB_RANGE("migplan: rollouts");
    if (static_cast<int>(comp.size()) != m_.n) throw PlanningError("completion vector length mismatch");
    if (k < 1 || k > 32) throw ArgumentError("rollouts: topk must be in [1, 32]");
    if (n_roll < 0 || max_depth < 0) throw ArgumentError("rollouts: negative count or depth");
    if (batch <= 0 || batch > n_roll) batch = n_roll;
    batch = std::min<long long>(batch, 1ll << 31);
    RolloutResult res;
    if (n_roll == 0) return res;
    CK(cudaSetDevice(device_));
    int L2 = table_log2;
    if (L2 <= 0) {
        long long want = std::max<long long>(1 << 16, std::min<long long>(1ll << 24, 4 * n_roll));
        L2 = 0;
        while ((1ll << L2) < want) ++L2;
    }
    L2 = std::min(std::max(L2, 4), 30);
    const int n = m_.n;
    std::vector<void*> owned;  // cached blocks (ro_get), handed back when the call ends
    struct Free {
        Engine* e;
        std::vector<void*>& v;
        ~Free() {
            for (void* p : v) e->ro_put(p);
        }
    } fr{this, owned};
    auto alloc = [&](size_t bytes) {
        void* p = ro_get(bytes, false);
        owned.push_back(p);
        return p;
    };
    struct HostOut {
        int path_len;
        int pad;
        double comp[256];
    };
    HostOut* ho = static_cast<HostOut*>(ro_get(sizeof(HostOut), true));
    owned.push_back(ho);
    long long* hpath = static_cast<long long*>(ro_get(sizeof(long long) * (max_depth + 1), true));
    owned.push_back(hpath);
    std::memcpy(ho->comp, comp.data(), sizeof(double) * n);

    RolloutArgs a{};
    a.M = dm_;
    a.base = d_base_;
    a.n_base = pool_size();
    std::memcpy(a.comp0, comp.data(), sizeof(double) * n);
    a.seed = seed;
    a.k = k;
    a.max_depth = max_depth;
    a.timers = 0;
    if (const char* v = std::getenv("MIGPLAN_ROLLOUT_DENSE_PCT")) rollout_set_dense_pct(std::atoi(v));  // A/B
    a.comp = static_cast<double*>(alloc(sizeof(double) * n * batch));
    a.len = static_cast<int*>(alloc(sizeof(int) * batch));
    a.status = static_cast<uint8_t*>(alloc(batch));
    a.rslot = static_cast<unsigned*>(alloc(sizeof(unsigned) * batch));
    a.act0 = static_cast<long long*>(alloc(sizeof(long long) * batch));
    a.act1 = static_cast<long long*>(alloc(sizeof(long long) * batch));
    a.keys = n <= 64 ? static_cast<uint64_t*>(alloc(sizeof(uint64_t) * batch)) : nullptr;
    a.cnt = static_cast<RolloutCounters*>(alloc(sizeof(RolloutCounters)));
    a.path = hpath;
    a.path_len = &ho->path_len;
    int* d_len = lengths ? static_cast<int*>(alloc(sizeof(int) * batch)) : nullptr;
    a.lengths = d_len;
    if (max_sup() > 0) support_tables();
    a.n_sup = n_sup_ > 0 && n_sup_ <= max_sup() ? n_sup_ : 0;
    a.sup_begin = a.n_sup ? d_sup_begin_ : nullptr;
    a.sup_svc = a.n_sup ? d_sup_svc_ : nullptr;
    // pair pools: pool builds run the FP32-bounded pair top-K (topk_pair.cuh) on 32-bit rows
    a.base32 = a.n_sup ? base32() : nullptr;
    a.keyrank = a.n_sup ? keyrank() : nullptr;
    const int si = ro_stream();  // cached stream + events (handed back at the end of the call)
    cudaStream_t st;
    cudaEvent_t e0, e1;
    {
        RoCache& rc = ro_cache(device_);
        std::lock_guard<std::mutex> g(rc.mu);
        st = rc.streams[si].s;
        e0 = rc.streams[si].e0;
        e1 = rc.streams[si].e1;
    }
    struct PutStream {
        Engine* e;
        int i;
        cudaStream_t s;
        ~PutStream() {
            cudaStreamSynchronize(s);
            e->ro_stream_put(i);
        }
    } ps{this, si, st};
    const int G = num_sms_ * rollout_blocks_per_sm_;
    const size_t smem = rollout_smem_bytes(n, m_.PP, max_sup());

    for (int attempt = 0;; ++attempt) {
        const size_t cap = size_t{1} << L2;
        std::vector<void*> table;
        auto talloc = [&](size_t bytes) {
            void* p = alloc(bytes);
            table.push_back(p);
            return p;
        };
        a.tab_mask = static_cast<unsigned>(cap - 1);
        a.tag = static_cast<unsigned*>(talloc(sizeof(unsigned) * cap));
        a.key = static_cast<uint64_t*>(talloc(sizeof(uint64_t) * 4 * cap));
        a.claimer = static_cast<unsigned long long*>(talloc(sizeof(unsigned long long) * cap));
        a.pool_n = static_cast<int*>(talloc(sizeof(int) * cap));
        a.pool = static_cast<unsigned*>(talloc(sizeof(unsigned) * k * cap));
        a.pend0 = static_cast<unsigned*>(talloc(sizeof(unsigned) * cap));
        a.pend1 = static_cast<unsigned*>(talloc(sizeof(unsigned) * cap));
        CK(cudaMemsetAsync(a.tag, 0, sizeof(unsigned) * cap, st));
        CK(cudaMemsetAsync(a.claimer, 0xFF, sizeof(unsigned long long) * cap, st));
        CK(cudaMemsetAsync(a.pool_n, 0xFF, sizeof(int) * cap, st));
        RolloutResult r;
        bool full = false;
        unsigned long long best_key = ~0ull;
        for (long long done = 0; done < n_roll; done += batch) {
            a.n_roll = std::min(batch, n_roll - done);
            a.id0 = id_offset + done;
            CK(cudaMemsetAsync(a.cnt, 0, sizeof(RolloutCounters), st));
            CK(cudaMemsetAsync(&a.cnt->best, 0xFF, sizeof(unsigned long long), st));
            // the start, then per round a pool-build launch and an advance launch, enqueued in
            // growing chunks; a round with no active rollout makes every later launch a no-op
            const int GA = num_sms_ * rollout_adv_blocks_per_sm_;
            const void* kb = rollout_build_ptr();
            const void* ka = rollout_advance_ptr(m_.n);
            auto adv = [&](int round) {
                void* args[] = {&a, &round};
                CK(cudaLaunchKernel(ka, GA, rollout_advance_threads(), args, 0, st));
            };
            auto bld = [&](int round) {
                void* args[] = {&a, &round};
                CK(cudaLaunchKernel(kb, G, rollout_threads(), args, smem, st));
            };
            // every round a rollout can need (a rollout takes at most max_depth steps) is enqueued
            // up front: the host never waits between rounds (a synchronisation per chunk left the
            // GPU idle while the next chunk was enqueued), and the rounds past the last one are
            // no-op launches (C->done)
            CK(cudaEventRecord(e0, st));
            int launches = 0;
            RolloutCounters c{};
            // small batches (one advance pass per round fits the grid once): one cooperative
            // launch runs every round with grid barriers (MIGPLAN_ROLLOUT_PERSIST=0/1 forces)
            const long long per_pass = static_cast<long long>(num_sms_) * (rollout_threads() / 32) * rollout_per_warp(m_.n);
            bool persist = a.n_roll <= per_pass;
            if (const char* v = std::getenv("MIGPLAN_ROLLOUT_PERSIST")) persist = std::atoi(v) != 0;
            if (persist) {
                void* args[] = {&a};
                CK(cudaLaunchCooperativeKernel(rollout_persistent_ptr(m_.n), num_sms_, rollout_threads(), args, smem, st));
                launches = 1;
            } else {
                adv(-1);
                launches = 1;
                for (int round = 0; round <= max_depth + 1; ++round) {
                    bld(round);
                    adv(round);
                    launches += 2;
                }
            }
            if (!persist) {
                void* args[] = {&a};
                CK(cudaLaunchKernel(rollout_replay_ptr(m_.n), 1, 32, args, 0, st));
                ++launches;
            }
            CK(cudaEventRecord(e1, st));
            stats.launches += launches;
            r.launches += launches;
            CK(cudaMemcpyAsync(&c, a.cnt, sizeof c, cudaMemcpyDeviceToHost, st));
            if (lengths)
                CK(cudaMemcpyAsync(lengths + done, d_len, sizeof(int) * a.n_roll, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            r.ms += ms;
            if (c.status != 0) {
                full = true;
                break;
            }
            r.completed += static_cast<long long>(c.completed);
            r.capped += static_cast<long long>(c.capped);
            r.failed += static_cast<long long>(c.failed);
            r.steps += static_cast<long long>(c.steps);
            r.keys += static_cast<long long>(c.keys);
            r.rounds = std::max(r.rounds, c.rounds);
            if (c.best != ~0ull) {  // (steps, global id): batches are in id order
                const unsigned long long len = c.best >> 32;
                const unsigned long long key = (len << 40) | static_cast<unsigned long long>(done + (c.best & 0xFFFFFFFFull));
                if (key < best_key) {
                    best_key = key;
                    r.best_len = static_cast<int>(len);
                    r.best_id = id_offset + done + static_cast<long long>(c.best & 0xFFFFFFFFull);
                    r.path.assign(hpath, hpath + ho->path_len);
                }
            }
        }
        if (full && attempt < 3 && L2 < 30) {
            for (void* p : table) {
                ro_put(p);
                owned.erase(std::find(owned.begin(), owned.end(), p));
            }
            L2 = std::min(L2 + 2, 30);
            continue;
        }
        if (full) throw DeviceError("rollouts: key cache full");
        res = std::move(r);
        break;
    }
    stats.rollout_ns += static_cast<long long>(res.ms * 1e6);
    stats.rollout_steps += res.steps;
    stats.rollout_calls++;
    stats.h2d += static_cast<long long>(sizeof(double) * n);
    stats.d2h += static_cast<long long>(sizeof(RolloutCounters) + sizeof(long long) * res.path.size() +
                                        (lengths ? sizeof(int) * n_roll : 0));
    return res;
}

// Independent greedy instances, one CTA each, in one launch: the GA's refills
// (FastProcedure, greedy.hpp:160-164) from `count` device-resident completion vectors.
// n_steps[i] = plan length, or -1 when fast_algo raised PlanningError (no positive score)
// or the plan would exceed cap_steps.  rows[i] = device pointer to the picked rows.
void Engine::greedy_batch(const double* d_comps, int count, long long cap_steps, long long rows_bound,
                          std::vector<const uint64_t*>& rows,
                          std::vector<int>& n_steps, std::vector<std::vector<uint64_t>>* host_rows,
                          SlotLease* lease, const double* h_comps) {
    MGB_RANGE("migplan: greedy batch (GA refills)");
    if (lease) lease->e = this;
    rows.assign(count, nullptr);
    n_steps.assign(count, -1);
    if (count <= 0) return;
    if (n_ranks_ > 1) throw ArgumentError("greedy_batch on a sharded context");
    const int T = kernel_threads();
    const size_t smem = greedy_smem_bytes(m_.n, m_.PP, cache_units_, ring_stages_);
    HostTimer ht;
    struct PrintT {
        HostTimer& h;
        ~PrintT() { h.print("greedy batch"); }
    } pt{ht};
    for (int b0 = 0; b0 < count; b0 += kMaxGroups) {
        const int nb = std::min(kMaxGroups, count - b0);
        std::vector<GreedyCall> calls(nb);
        struct Rel {
            std::vector<GreedyCall>& c;
            ~Rel() {
                for (auto& x : c)
                    if (x.s) x.e->release(x.s);
            }
        } rel{calls};
        // the SMs are split between the instances (each a complete fast_algo on its CTAs)
        int gpc = std::max(1, num_sms_ * greedy_blocks_per_sm_ / nb);
        if (const char* v = std::getenv("MIGPLAN_GREEDY_CTAS")) gpc = std::max(1, std::min(gpc, std::atoi(v)));
        const int GC = greedy_cluster_ctas(smem, rows_bound);
        if (GC && GC * nb <= num_sms_) gpc = GC;
        std::unique_ptr<GreedyLaunch> L(new GreedyLaunch{});
        L->n_groups = nb;
        L->ctas_per_group = gpc;
        L->cluster = GC && GC * nb <= num_sms_ ? 1 : 0;
        for (int i = 0; i < nb; ++i) {  // every instance's set-up on the launch stream: no cross-stream waits
            calls[i].e = this;
            calls[i].s = acquire();
            // host completions go through each slot's host-mapped input (no staging copy)
            greedy_prepare(calls[i], h_comps ? h_comps + static_cast<size_t>(b0 + i) * m_.n : nullptr,
                           h_comps ? nullptr : d_comps + static_cast<size_t>(b0 + i) * m_.n, cap_steps,
                           calls[0].s->stream, true);
            calls[i].a.interleave = greedy_interleave(gpc);
            L->g[i] = calls[i].a;
        }
        Slot* s0 = calls[0].s;
        launch_greedy_batch_init(*L, calls[0].base_src, calls[0].n_base, s0->stream);  // states + arenas
        CK(cudaGetLastError());
        stats.launches++;
        CK(cudaEventRecord(s0->e0, s0->stream));
        ht.mark(0);
        launch_greedy(*L, T, smem, s0->stream);
        stats.launches++;
        CK(cudaEventRecord(s0->e1, s0->stream));
        CK(cudaStreamSynchronize(s0->stream));
        ht.mark(1);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, s0->e0, s0->e1));
        stats.greedy_ns += static_cast<long long>(ms * 1e6f);
        for (int i = 0; i < nb; ++i) {
            const GreedyState h = calls[i].s->io->res;
            if (h.status == kExtOverflow) throw DeviceError("greedy_batch: extension arena overflow");
            stats.greedy_rows += h.rows_scored;
            stats.greedy_calls++;
            stats.greedy_steps += h.n_steps;
            stats.ext_events += h.n_events;
            stats.ext_rows += static_cast<long long>(h.ext_count);
            for (int k = 0; k < 5; ++k) stats.phase_ns[k] += static_cast<long long>(h.phase_ns[k]);
            if (h.status == kOk) {
                n_steps[b0 + i] = h.n_steps;
                rows[b0 + i] = calls[i].s->d_pick_row;
                if (host_rows) (*host_rows)[b0 + i].assign(calls[i].s->pick_row, calls[i].s->pick_row + h.n_steps);
            }
            stats.d2h += static_cast<long long>(sizeof(GreedyState) + sizeof(uint64_t) * std::max(h.n_steps, 0));
        }
        // with a lease the slots (and the device picked rows in `rows`) are held until the
        // caller has consumed them; the next batch then takes different slots
        for (auto& x : calls) {
            if (lease)
                lease->slots.push_back(x.s);
            else
                x.e->release(x.s);
            x.s = nullptr;
        }
        ht.mark(2);
    }
}

// ---- device-resident parity mcts_solve (mcts.cu)
MctsDeviceResult Engine::mcts_device(const std::vector<double>& comp, int budget, int topk, int pick_services,
                                     double ucb_c, uint64_t seed, int l_ref) {
    return mcts_device_group({comp}, budget, topk, pick_services, ucb_c, {seed}, {l_ref})[0];
}

// Several independent searches (the GA's children) as CTAs of one launch; each search has
// its own slot (scratch + rollout cache).
std::vector<MctsDeviceResult> Engine::mcts_device_group(const std::vector<std::vector<double>>& comps, int budget,
                                                        int topk, int pick_services, double ucb_c,
                                                        const std::vector<uint64_t>& seeds,
                                                        const std::vector<int>& l_refs) {
    MGB_RANGE("migplan: mcts search");
    if (topk < 1 || topk > 32) throw ArgumentError("mcts: topk must be in [1, 32] on the device path");
    if (n_ranks_ > 1) throw ArgumentError("mcts on a sharded context");
    const int n = m_.n;
    const int count = static_cast<int>(comps.size());
    std::vector<MctsDeviceResult> results(count);
    CK(cudaSetDevice(device_));
    HostTimer ht;
    struct PrintT {
        HostTimer& h;
        ~PrintT() { h.print("mcts group"); }
    } pt{ht};
    for (int b0 = 0; b0 < count; b0 += kMaxGroups) {
        const int nb = std::min(kMaxGroups, count - b0);
        std::vector<Slot*> slots;
        struct Rel {
            Engine* e;
            std::vector<Slot*>& v;
            ~Rel() {
                for (Slot* s : v) e->release(s);
            }
        } rel{this, slots};
        std::unique_ptr<MctsLaunch> L(new MctsLaunch{});
        L->M = dm_;
        L->base = d_base_;
        L->n_base = pool_size();
        L->keyrank = keyrank();
        L->budget = budget;
        L->topk = topk;
        L->pick_services = pick_services;
        L->ucb_c = ucb_c;
        struct Off {
            size_t comp0, ncomp, vis, val, first, nch, cand, flags, path, edges, picked, unsat, tag, key, pn, pool,
                trace, best, desc, dcomp, out;
            long long cap, max_nodes;
        };
        std::vector<Off> offs(nb);
        for (int q = 0; q < nb; ++q) {
            const int l_ref = l_refs[b0 + q];
            const int max_depth = 2 * l_ref;
            const long long max_nodes = 1 + static_cast<long long>(budget) * topk;
            const long long path_cap = max_nodes + max_depth + 8;
            long long want = std::max<long long>(1024, 2ll * budget * (max_depth + 1));
            long long cap = 1;
            while (cap < want) cap <<= 1;
            Slot* s = acquire();
            slots.push_back(s);
            size_t off = 0;
            auto take = [&](size_t bytes) {
                size_t at = (off + 15) & ~size_t{15};
                off = at + bytes;
                return at;
            };
            Off& o = offs[q];
            o.cap = cap;
            o.max_nodes = max_nodes;
            o.comp0 = take(sizeof(double) * n);
            o.ncomp = take(sizeof(double) * max_nodes * n);
            o.vis = take(sizeof(int) * max_nodes);
            o.val = take(sizeof(double) * max_nodes);
            o.first = take(sizeof(int) * max_nodes);
            o.nch = take(sizeof(int) * max_nodes);
            o.cand = take(sizeof(int) * max_nodes);
            o.flags = take(max_nodes);
            o.path = take(sizeof(int) * path_cap);
            o.edges = take(sizeof(int) * path_cap);
            o.picked = take(sizeof(int) * (max_depth + 8));
            o.unsat = take(sizeof(int) * (n + 1));
            o.tag = take(sizeof(unsigned) * cap);
            o.key = take(sizeof(uint64_t) * 4 * cap);
            o.pn = take(sizeof(int) * cap);
            o.pool = take(sizeof(unsigned) * topk * cap);
            o.trace = take(sizeof(int) * 4 * std::max(budget, 1));
            o.best = take(sizeof(int) * path_cap);
            o.desc = take(sizeof(int) * path_cap);
            o.dcomp = take(sizeof(double) * n);
            o.out = take(sizeof(int) * 32);
            if (s->mcts_bytes < off) {
                if (s->mcts_mem) CK(cudaFree(s->mcts_mem));
                s->mcts_mem = nullptr;
                CK(cudaMalloc(&s->mcts_mem, off));
                s->mcts_bytes = off;
            }
            if (s->logtab_n < budget + 2) {  // std::log(v), v = 0..budget+1 (the reference's own libm values)
                if (s->logtab) CK(cudaFree(s->logtab));
                std::vector<double> lt(budget + 2);
                for (int v = 0; v < budget + 2; ++v) lt[v] = std::log(static_cast<double>(std::max(1, v)));
                CK(cudaMalloc(&s->logtab, sizeof(double) * lt.size()));
                CK(cudaMemcpy(s->logtab, lt.data(), sizeof(double) * lt.size(), cudaMemcpyHostToDevice));
                s->logtab_n = static_cast<int>(lt.size());
            }
            unsigned char* b = static_cast<unsigned char*>(s->mcts_mem);
            // pinned staging: the completion in, the outputs (trace .. out, carved contiguously) back
            const size_t hb_bytes = std::max(sizeof(double) * n, o.out + sizeof(int) * 32 - o.trace);
            if (s->mcts_host_bytes < hb_bytes) {
                if (s->mcts_host) CK(cudaFreeHost(s->mcts_host));
                s->mcts_host = nullptr;
                CK(cudaMallocHost(&s->mcts_host, hb_bytes));
                s->mcts_host_bytes = hb_bytes;
            }
            // the kernel reads its start completion from the pinned staging (mapped) and zeroes its
            // own cache tags: no per-search copy or memset enqueued
            std::memcpy(s->mcts_host, comps[b0 + q].data(), sizeof(double) * n);
            MctsSolveArgs& a = L->s[q];
            a.comp0 = reinterpret_cast<const double*>(s->mcts_host);
            a.seed = mix_seed_u64(seeds[b0 + q], 0x6d637473);
            a.l_ref = l_ref;
            a.max_nodes = static_cast<int>(max_nodes);
            a.node_comp = reinterpret_cast<double*>(b + o.ncomp);
            a.node_visits = reinterpret_cast<int*>(b + o.vis);
            a.node_value = reinterpret_cast<double*>(b + o.val);
            a.node_first = reinterpret_cast<int*>(b + o.first);
            a.node_nch = reinterpret_cast<int*>(b + o.nch);
            a.node_cand = reinterpret_cast<int*>(b + o.cand);
            a.node_flags = b + o.flags;
            a.pathnodes = reinterpret_cast<int*>(b + o.path);
            a.edges = reinterpret_cast<int*>(b + o.edges);
            a.picked = reinterpret_cast<int*>(b + o.picked);
            a.unsat = reinterpret_cast<int*>(b + o.unsat);
            a.tab_mask = static_cast<unsigned>(cap - 1);
            a.tag = reinterpret_cast<unsigned*>(b + o.tag);
            a.key = reinterpret_cast<uint64_t*>(b + o.key);
            a.pool_n = reinterpret_cast<int*>(b + o.pn);
            a.pool = reinterpret_cast<unsigned*>(b + o.pool);
            a.trace = reinterpret_cast<int*>(b + o.trace);
            a.best_out = reinterpret_cast<int*>(b + o.best);
            a.descent_out = reinterpret_cast<int*>(b + o.desc);
            a.descent_comp = reinterpret_cast<double*>(b + o.dcomp);
            a.out = reinterpret_cast<int*>(b + o.out);
        }
        L->logtab = slots[0]->logtab;  // identical tables; slot 0's is >= budget + 2 long
        // one thread-block cluster per search: C ranks each scan 1/C of the base pool per top-K
        // (measured: the per-top-K fixed costs — cluster barriers, DSMEM merge — outweigh the
        // 1/C scan at the pool sizes of the GA workloads, so one CTA per search by default)
        int C = 1;
        if (const char* v = std::getenv("MIGPLAN_MCTS_CLUSTER")) C = std::max(1, std::min(16, std::atoi(v)));
        const bool pair = m_.max_mix <= 2 && !(std::getenv("MIGPLAN_MCTS_PAIR") && std::atoi(std::getenv("MIGPLAN_MCTS_PAIR")) == 0);
        L->pair = pair ? 1 : 0;
        const long long slice = pair ? (((pool_size() + C - 1) / C + 3) & ~3ll) : (((pool_size() + C - 1) / C + 1) & ~1ll);
        // on-chip placement: the slice first (every top-K scans it twice), then the nodes
        {
            const DeviceInfo& di = device_info(device_);
            const long long room = di.smem_optin - di.mcts_static_smem - 1024;
            const int mn = static_cast<int>(offs[0].max_nodes);
            // supports (skip the ones that cannot hold a candidate): one CTA over the whole pool
            int ns = 0;
            const char* sv_env = std::getenv("MIGPLAN_MCTS_SUPPORTS");
            if (pair && C == 1 && !(sv_env && std::atoi(sv_env) == 0)) {
                support_tables();
                ns = n_sup_;
            }
            L->rows_smem = static_cast<long long>(mcts_smem_bytes(n, m_.PP, mn, slice, false, true, pair, ns)) <= room;
            // a pair pool too large for shared memory: the pair top-K reads its 32-bit rows from
            // global memory (L2), with the support tables still on chip when they fit
            const bool pair_global = pair && !L->rows_smem && C == 1;
            L->base32 = pair_global ? base32() : nullptr;
            const bool sup_fit = static_cast<long long>(mcts_smem_bytes(n, m_.PP, mn, slice, false, L->rows_smem != 0, pair, ns)) <= room;
            if (!((L->rows_smem && pair) || pair_global) || !sup_fit) ns = 0;
            L->timers = std::getenv("MIGPLAN_MCTS_TIMERS") ? 1 : 0;
            if (const char* v = std::getenv("MIGPLAN_MCTS_DENSE_PCT")) mcts_set_dense_pct(std::atoi(v));
            L->node_smem =
                static_cast<long long>(mcts_smem_bytes(n, m_.PP, mn, slice, true, L->rows_smem != 0, pair, ns)) <= room;
            L->n_sup = ns;
            L->sup_begin = ns ? d_sup_begin_ : nullptr;
            L->sup_svc = ns ? d_sup_svc_ : nullptr;
        }
        size_t msm = mcts_smem_bytes(n, m_.PP, static_cast<int>(offs[0].max_nodes), slice, L->node_smem != 0,
                                     L->rows_smem != 0, pair, L->n_sup);
        {  // the on-chip rollout cache takes what is left (key words, pool size, K (index, row) pairs per slot)
            const DeviceInfo& di = device_info(device_);
            const long long left = di.smem_optin - di.mcts_static_smem - 1024 - static_cast<long long>(msm) - 64;
            const long long per = 8ll * ((n + 63) / 64) + 4 + 8ll * topk;
            int slots = 4096;
            while (slots >= 32 && slots * per > left) slots >>= 1;
            if (const char* v = std::getenv("MIGPLAN_MCTS_L1")) slots = std::min(slots, std::atoi(v));
            L->l1_slots = slots >= 32 ? slots : 0;
            msm += L->l1_slots ? static_cast<size_t>(L->l1_slots * per + 48) : 0;
        }
        Slot* s0 = slots[0];
        void* args[] = {L.get()};
        ht.mark(0);
        CK(cudaEventRecord(s0->e0, s0->stream));
        {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(nb * C);
            cfg.blockDim = dim3(mcts_threads());
            cfg.dynamicSmemBytes = msm;
            cfg.stream = s0->stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = C;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelExC(&cfg, mcts_kernel_ptr(n), args));
        }
        stats.launches++;
        CK(cudaEventRecord(s0->e1, s0->stream));
        for (int q = 0; q < nb; ++q) {  // the outputs are carved contiguously (trace, best, desc, dcomp, out)
            const Off& o = offs[q];
            CK(cudaMemcpyAsync(slots[q]->mcts_host, static_cast<unsigned char*>(slots[q]->mcts_mem) + o.trace,
                               o.out + sizeof(int) * 32 - o.trace, cudaMemcpyDeviceToHost, s0->stream));
        }
        CK(cudaStreamSynchronize(s0->stream));
        ht.mark(1);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, s0->e0, s0->e1));
        stats.mcts_ns += static_cast<long long>(ms * 1e6);
        stats.mcts_launches++;
        for (int q = 0; q < nb; ++q) {
            const Off& o = offs[q];
            const unsigned char* hbd = slots[q]->mcts_host;
            const size_t hb_size = o.out + sizeof(int) * 32 - o.trace;
            auto at = [&](size_t off) { return hbd + (off - o.trace); };
            int out[32];
            std::memcpy(out, at(o.out), sizeof(out));
            MctsDeviceResult& r = results[b0 + q];
            r.status = out[0];
            r.best_len = out[1];
            r.descent_leaf = out[3] != 0;
            r.builds = out[4];
            r.iterations = out[6];
            r.expands = out[7];
            std::memcpy(&r.expand_rows, &out[8], sizeof(long long));
            if (std::getenv("MIGPLAN_MCTS_TIMERS")) {
                long long t[5];
                std::memcpy(t, &out[10], sizeof t);
                unsigned long long tk[12];
                mcts_read_topk_timers(tk);
                if (tk[5])
                    std::fprintf(stderr, "[mcts] top-K (cumulative) calls %llu, cycles/call: tables %.0f scan %.0f tree %.0f pass2 %.0f "
                                 "rank %.0f, candidates/call %.1f; warps' scan end (from call start) max %.0f mean %.0f min %.0f, "
                                 "by-support %llu\n", tk[5], double(tk[0]) / tk[5], double(tk[7]) / tk[5],
                                 double(tk[1]) / tk[5], double(tk[2]) / tk[5], double(tk[3]) / tk[5], double(tk[4]) / tk[5],
                                 double(tk[8]) / tk[5], double(tk[9]) / tk[5], double(tk[10]) / tk[5], tk[11]);
                std::fprintf(stderr, "[mcts] solve %d: %.1f ms device, cycles sel %lld expand-host %lld miss-host %lld topk %lld "
                             "rollout-ctl %lld, builds %d expands %d iters %d, exact-path top-Ks (cumulative) %d, walk steps %d "
                             "cycles %lld, probes %d cycles %lld, entries %d\n",
                             b0 + q, ms, t[0], t[1], t[2], t[3], t[4], out[4], out[7], out[6], out[20], out[21],
                             *reinterpret_cast<const long long*>(&out[22]), out[24], *reinterpret_cast<const long long*>(&out[26]),
                             out[25]);
            }
            r.trace.resize(4 * static_cast<size_t>(r.iterations));
            std::vector<int> best(std::max(r.best_len, 0)), desc(out[2]);
            if (!r.trace.empty()) std::memcpy(r.trace.data(), at(o.trace), sizeof(int) * r.trace.size());
            if (!best.empty()) std::memcpy(best.data(), at(o.best), sizeof(int) * best.size());
            if (!desc.empty()) std::memcpy(desc.data(), at(o.desc), sizeof(int) * desc.size());
            r.descent_comp.resize(n);
            std::memcpy(r.descent_comp.data(), at(o.dcomp), sizeof(double) * n);
            r.best.assign(best.begin(), best.end());
            r.descent.assign(desc.begin(), desc.end());
            // work counters with the reference's definitions (mcts.hpp:59-67): every expansion
            // scores its filtered set, every rollout-cache miss the whole base pool
            stats.topk_calls += r.expands + r.builds;
            stats.topk_rows += r.expand_rows + static_cast<long long>(r.builds) * pool_size();
            stats.mcts_topk_calls += r.expands + r.builds;
            stats.mcts_rows += r.expand_rows + static_cast<long long>(r.builds) * pool_size();
            stats.h2d += static_cast<long long>(sizeof(double) * n);
            stats.d2h += static_cast<long long>(hb_size);
        }
        ht.mark(2);
    }
    return results;
}

// fast_algo on several host completion vectors, all in one grouped launch (CTA groups).
// status[i] = 0 ok, 1 PlanningError (no positive score).
void Engine::fast_algo_batch(const std::vector<std::vector<double>>& comps, std::vector<std::vector<uint64_t>>& rows,
                             std::vector<int>& status) {
    const int count = static_cast<int>(comps.size());
    rows.assign(count, {});
    status.assign(count, 0);
    if (count == 0) return;
    CK(cudaSetDevice(device_));
    long long cap_steps = 1;
    for (const auto& c : comps) {
        if (static_cast<int>(c.size()) != m_.n) throw PlanningError("fast_algo: completion vector length mismatch");
        cap_steps = std::max(cap_steps, std::min<long long>(step_bound(c), 1 << 24));
    }
    std::vector<double> flat;
    for (const auto& c : comps) flat.insert(flat.end(), c.begin(), c.end());
    // one staged copy (measured: every CTA reading its instance's completion from host-mapped
    // memory instead costs ~12 us per grouped launch)
    Scratch buf(device_, sizeof(double) * flat.size());
    double* d = static_cast<double*>(buf.get());
    CK(cudaMemcpy(d, flat.data(), sizeof(double) * flat.size(), cudaMemcpyHostToDevice));
    stats.h2d += static_cast<long long>(sizeof(double) * flat.size());
    std::vector<const uint64_t*> drows;
    std::vector<int> steps;
    long long wsb = 0;
    for (const auto& c : comps) wsb = std::max(wsb, working_set_bound(c.data()));
    greedy_batch(d, count, cap_steps, wsb, drows, steps, &rows);
    for (int i = 0; i < count; ++i)
        if (steps[i] < 0) status[i] = 1;
}

// ---- brute_force_optimum (bf.cu)
std::vector<Config> Engine::brute_force(int cap, long long node_budget, bool& found) {
    MGB_RANGE("migplan: brute_force_optimum");
    found = false;
    const int n = m_.n;
    if (n == 0) {
        found = true;
        return {};
    }
    if (n > kBfMaxN)
        throw ArgumentError("device brute_force_optimum: n <= " + std::to_string(kBfMaxN) + " services");
    if (cap > kBfMaxDepth) throw ArgumentError("brute_force_optimum: cap <= 8 on the device");
    CK(cudaSetDevice(device_));
    // The pool the reference searches: build_candidate_pool(..., max_mix = min(n, 7))
    // (bench.hpp:164-165), enumerated on the device in its emission order (config_enum.hpp:
    // 108-150: layouts in canonical order, then the per-group nondecreasing service sequences
    // in lexicographic order), so the DFS's first solution and node count are the reference's.
    BfEnumArgs ea{};
    ea.n = n;
    ea.PP = m_.PP;
    ea.max_mix = std::min(n, 7);
    ea.n_layouts = static_cast<int>(m_.layouts.size());
    long long space = 0;
    for (int li = 0; li < ea.n_layouts; ++li) {
        const Layout& L = m_.layouts[li];
        ea.lay_off[li] = space;
        ea.n_groups[li] = static_cast<int>(L.groups.size());
        long long c = 1;
        for (size_t g = 0; g < L.groups.size(); ++g) {
            const int len = static_cast<int>(L.groups[g].slots.size());
            ea.g_len[li][g] = static_cast<int8_t>(len);
            ea.g_size[li][g] = static_cast<int8_t>(L.groups[g].size_idx);
            long long mc = 1;
            for (int i = 1; i <= len; ++i) mc = mc * (n + i - 1) / i;
            ea.g_cnt[li][g] = mc;
            c *= mc;
        }
        space += c;
    }
    ea.lay_off[ea.n_layouts] = space;
    if (space > (1ll << 31)) throw ArgumentError("brute_force_optimum: enumeration space too large");
    for (int i = 0; i < n; ++i) ea.feas_mask[i] = m_.feas_mask[i];
    std::vector<uint8_t> pat_of(1u << 15, 0xFF);
    for (int p = 0; p < m_.PP; ++p) {
        unsigned key = 0;
        for (int z = 0; z < kMaxSizes; ++z) key |= static_cast<unsigned>(m_.patterns[p][z]) << (3 * z);
        pat_of[key] = static_cast<uint8_t>(p);
    }
    const int nb = static_cast<int>((space + 255) / 256);
    const size_t off_cnt0 = 256, off_lut = off_cnt0 + ((sizeof(unsigned) * (nb + 1) + 255) & ~size_t(255));
    void* emem = nullptr;
    CK(cudaMalloc(&emem, off_lut + pat_of.size()));
    struct EFree {
        void* p;
        ~EFree() { cudaFree(p); }
    } efr{emem};
    unsigned char* e8 = static_cast<unsigned char*>(emem);
    CK(cudaMemset(e8, 0, 256));
    CK(cudaMemcpy(e8 + off_lut, pat_of.data(), pat_of.size(), cudaMemcpyHostToDevice));
    ea.error = reinterpret_cast<int*>(e8);
    ea.block_cnt = reinterpret_cast<unsigned*>(e8 + off_cnt0);
    ea.pat_of = e8 + off_lut;
    int mode = 0;
    {
        void* args[] = {&ea, &mode};
        CK(cudaLaunchKernel(bf_enum_kernel_ptr(), nb, 256, args, 0, nullptr));
        void* sargs[] = {&ea.block_cnt, const_cast<int*>(&nb)};
        CK(cudaLaunchKernel(bf_scan_kernel_ptr(), 1, 1024, sargs, 0, nullptr));
        stats.launches += 2;
    }
    unsigned total = 0;
    CK(cudaMemcpy(&total, ea.block_cnt + nb, sizeof total, cudaMemcpyDeviceToHost));
    const long long P = total;
    // depth 1-2: a thread per prefix; depth >= 3: a warp per two-pick prefix (bf.cu)
    const long long chunk_t = static_cast<long long>(num_sms_) * bf_threads() * 4;
    const long long chunk_w = static_cast<long long>(num_sms_) * 64 * 8;
    const long long max_ranks = std::min(std::max(P * (P + 1) / 2, 1ll), std::max(chunk_t, chunk_w));
    struct Words {
        unsigned long long best_key, overrun, sum, pad;
    };
    const size_t off_tuple = sizeof(Words), off_any = off_tuple + sizeof(long long) * (kBfMaxDepth + 1);
    const size_t off_rows = (off_any + sizeof(double) * n + 255) & ~size_t(255);
    const size_t off_cnt = (off_rows + sizeof(uint4) * static_cast<size_t>(std::max(P, 1ll)) + 255) & ~size_t(255);
    void* mem = nullptr;
    CK(cudaMalloc(&mem, off_cnt + sizeof(unsigned long long) * std::max<long long>(max_ranks, 1)));
    struct Free {
        void* p;
        ~Free() { cudaFree(p); }
    } fr{mem};
    unsigned char* m8 = static_cast<unsigned char*>(mem);
    Words* w = reinterpret_cast<Words*>(m8);
    const uint4* rows = reinterpret_cast<const uint4*>(m8 + off_rows);
    std::vector<double> best_any(n, 0.0);  // bench.hpp:167-171
    CK(cudaMemset(m8 + off_any, 0, sizeof(double) * n));
    if (P > 0) {
        ea.rows = reinterpret_cast<uint4*>(m8 + off_rows);
        mode = 1;
        void* args[] = {&ea, &mode};
        CK(cudaLaunchKernel(bf_enum_kernel_ptr(), nb, 256, args, 0, nullptr));
        DevModel dm = dm_;
        long long Pv = P;
        unsigned long long* bits = reinterpret_cast<unsigned long long*>(m8 + off_any);
        void* bargs[] = {&dm, const_cast<uint4**>(&rows), &Pv, &bits};
        CK(cudaLaunchKernel(bf_best_any_kernel_ptr(), static_cast<unsigned>(std::min<long long>((P + 255) / 256, num_sms_ * 8)),
                            256, bargs, 0, nullptr));
        stats.launches += 2;
    }
    int enum_err = 0;
    CK(cudaMemcpy(&enum_err, ea.error, sizeof enum_err, cudaMemcpyDeviceToHost));
    if (enum_err) throw DeviceError("brute_force_optimum: a member pattern is missing from the model");
    CK(cudaMemcpy(best_any.data(), m8 + off_any, sizeof(double) * n, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i)
        if (best_any[i] <= 0.0) throw PlanningError("oracle: service cannot be served by any config");
    const unsigned long long budget = static_cast<unsigned long long>(std::max<long long>(node_budget, 0));
    auto over = [] { throw PlanningError("oracle: node budget exceeded; shrink the instance or raise the budget"); };
    unsigned long long nodes = 0;  // the reference's ++nodes, cumulative over depths
    int root_bound = 0;            // bound(zero completion), bench.hpp:179-187
    for (int i = 0; i < n; ++i) root_bound = std::max(root_bound, static_cast<int>(std::ceil(1.0 / best_any[i] - 1e-12)));
    const int T = bf_threads();
    for (int d = 0; d <= cap; ++d) {
        if (++nodes > budget) over();  // dfs root; satisfied only for an empty workload (above)
        if (d == 0 || root_bound > d) continue;  // bench.hpp:197
        BfArgs a{};
        a.M = dm_;
        a.rows = rows;
        a.n_rows = P;
        a.best_any = reinterpret_cast<const double*>(m8 + off_any);
        a.depth = d;
        a.replay = -1;
        a.cnt = reinterpret_cast<unsigned long long*>(m8 + off_cnt);
        a.best_key = &w->best_key;
        a.overrun = &w->overrun;
        a.sum = &w->sum;
        a.tuple = reinterpret_cast<long long*>(m8 + off_tuple);
        const Words init{~0ull, ~0ull, 0ull, 0ull};
        CK(cudaMemcpy(w, &init, sizeof init, cudaMemcpyHostToDevice));
        const long long ranks = d == 1 ? P : P * (P + 1) / 2;
        const bool warp = d >= 3;
        const long long chunk = warp ? chunk_w : chunk_t;
        const void* kern = warp ? bf_warp_kernel_ptr() : bf_kernel_ptr();
        for (long long r0 = 0; r0 < ranks; r0 += chunk) {
            a.rank0 = r0;
            a.rank_end = std::min(ranks, r0 + chunk);
            a.remaining = budget - nodes;
            void* args[] = {&a};
            const long long lanes = (a.rank_end - r0) * (warp ? 32 : 1);
            const unsigned grid = static_cast<unsigned>((lanes + T - 1) / T);
            CK(cudaLaunchKernel(kern, grid, T, args, 0, nullptr));
            CK(cudaLaunchKernel(bf_sum_kernel_ptr(), std::min<unsigned>(grid, num_sms_ * 4), T, args, 0, nullptr));
            stats.launches += 2;
            Words got{};
            CK(cudaMemcpy(&got, w, sizeof got, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(&w->sum, &init.sum, sizeof init.sum, cudaMemcpyHostToDevice));
            const bool hit = got.best_key != ~0ull;
            const unsigned long long stop_rank = hit ? got.best_key : static_cast<unsigned long long>(a.rank_end - 1);
            if (got.overrun <= stop_rank) over();
            nodes += got.sum;
            if (nodes > budget) over();
            if (hit) {
                a.replay = static_cast<long long>(got.best_key);
                CK(cudaLaunchKernel(kern, 1, T, args, 0, nullptr));
                stats.launches++;
                long long tup[kBfMaxDepth + 1];
                CK(cudaMemcpy(tup, a.tuple, sizeof tup, cudaMemcpyDeviceToHost));
                std::vector<Config> out;
                for (long long q = 0; q < tup[kBfMaxDepth]; ++q) {
                    uint4 r;
                    CK(cudaMemcpy(&r, rows + tup[q], sizeof r, cudaMemcpyDeviceToHost));
                    out.push_back(config_of_wide(r));
                }
                found = true;
                return out;
            }
        }
    }
    return {};
}

// ---- throughput-mode GA device state (ga.cu)
size_t ga_breed_smem_bytes(int n);
size_t ga_finish_smem_bytes(int n);
const void* ga_breed_kernel_ptr();
const void* ga_finish_kernel_ptr();
int ga_threads();

struct GaRun {
    int P = 0, nch = 0, L_cap = 0;
    uint64_t* pop[2] = {nullptr, nullptr};
    int* pop_len = nullptr;
    uint64_t* work = nullptr;
    uint64_t* child = nullptr;
    int* n_surv = nullptr;
    double* residual = nullptr;
    unsigned* scratch = nullptr;
    const uint64_t** refill = nullptr;
    int* refill_n = nullptr;
    uint64_t* alt = nullptr;  // per-child refill rows taken from a rollout (throughput MCTS refill)
    int* child_len = nullptr;
    double* child_slack = nullptr;
    std::vector<void*> owned;
    ~GaRun() {
        for (void* p : owned) cudaFree(p);
    }
};

GaRun* Engine::ga_begin(int P, int L_cap) {
    CK(cudaSetDevice(device_));
    auto r = std::make_unique<GaRun>();
    r->P = P;
    r->nch = (P + 1) / 2;
    r->L_cap = L_cap;
    auto al = [&](size_t bytes) {
        void* p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        r->owned.push_back(p);
        return p;
    };
    const size_t rowb = sizeof(uint64_t) * L_cap;
    for (auto& p : r->pop) p = static_cast<uint64_t*>(al(rowb * std::max(P, 1)));
    r->pop_len = static_cast<int*>(al(sizeof(int) * r->nch));
    r->work = static_cast<uint64_t*>(al(rowb * r->nch));
    r->child = static_cast<uint64_t*>(al(rowb * r->nch));
    r->n_surv = static_cast<int*>(al(sizeof(int) * r->nch));
    r->residual = static_cast<double*>(al(sizeof(double) * m_.n * r->nch));
    r->scratch = static_cast<unsigned*>(al(sizeof(unsigned) * 8 * L_cap * r->nch));
    r->refill = static_cast<const uint64_t**>(al(sizeof(void*) * r->nch));
    r->refill_n = static_cast<int*>(al(sizeof(int) * r->nch));
    r->alt = static_cast<uint64_t*>(al(rowb * r->nch));
    r->child_len = static_cast<int*>(al(sizeof(int) * r->nch));
    r->child_slack = static_cast<double*>(al(sizeof(double) * r->nch));
    static std::once_flag attrs;
    std::call_once(attrs, [] {
        for (const void* k : {ga_breed_kernel_ptr(), ga_finish_kernel_ptr()})
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    });
    return r.release();
}

void Engine::ga_end(GaRun* r) { delete r; }

void Engine::ga_put(GaRun* r, int buf, int idx, const std::vector<uint64_t>& genomes) {
    if (static_cast<int>(genomes.size()) > r->L_cap) throw ArgumentError("GA: chromosome longer than L_cap");
    CK(cudaMemcpy(r->pop[buf] + static_cast<size_t>(idx) * r->L_cap, genomes.data(), genomes.size() * 8,
                  cudaMemcpyHostToDevice));
}

std::vector<uint64_t> Engine::ga_get(GaRun* r, int buf, int idx, int len, bool from_child) {
    std::vector<uint64_t> g(len);
    const uint64_t* src = (from_child ? r->child : r->pop[buf]) + static_cast<size_t>(idx) * r->L_cap;
    if (len) CK(cudaMemcpy(g.data(), src, len * 8ull, cudaMemcpyDeviceToHost));
    return g;
}

// One generation: children of pop[buf][0..npar) (parents in fitness order, ga.hpp:146-151).
void Engine::ga_generation(GaRun* r, int buf, const std::vector<int>& parent_len, int round, const GaParams& p,
                           std::vector<int>& child_len, std::vector<double>& child_slack, const RolloutRefill* slow) {
    MGB_RANGE("migplan: GA generation");
    const int npar = static_cast<int>(parent_len.size());
    CK(cudaSetDevice(device_));
    CK(cudaMemcpy(r->pop_len, parent_len.data(), sizeof(int) * npar, cudaMemcpyHostToDevice));
    GaBreedArgs b{};
    b.M = dm_;
    b.pop = r->pop[buf];
    b.pop_len = r->pop_len;
    b.work = r->work;
    b.child = r->child;
    b.n_surv = r->n_surv;
    b.residual = r->residual;
    b.scratch = r->scratch;
    b.L_cap = r->L_cap;
    b.round = round;
    b.mutation_pairs = p.mutation_pairs;
    b.erase_fraction = p.erase_fraction;
    b.seed = p.seed;
    {
        void* args[] = {&b};
        CK(cudaLaunchKernel(ga_breed_kernel_ptr(), npar, ga_threads(), args, ga_breed_smem_bytes(m_.n), nullptr));
        stats.launches++;
        CK(cudaDeviceSynchronize());
    }
    // refill every child's residual with the device greedy, all children in one launch
    std::vector<const uint64_t*> rows;
    std::vector<int> steps;
    SlotLease lease;  // keeps every child's picked rows alive until ga_finish has read them
    greedy_batch(r->residual, npar, r->L_cap, -1, rows, steps, nullptr, &lease);
    std::vector<int> ns(npar);
    CK(cudaMemcpy(ns.data(), r->n_surv, sizeof(int) * npar, cudaMemcpyDeviceToHost));
    for (int i = 0; i < npar; ++i)
        if (ns[i] < 0) steps[i] = -1;  // no crossover: the child is the mutated parent
    if (slow) {
        // the throughput mcts_solve refill (mig_mcts_solve_parallel): each child whose greedy
        // refill succeeded also runs slow->n_rollouts root-parallel rollouts (K5) from its
        // residual, depth cap 2 x |greedy refill|; a strictly shorter best rollout replaces it
        std::vector<double> res(static_cast<size_t>(npar) * m_.n);
        CK(cudaMemcpy(res.data(), r->residual, sizeof(double) * res.size(), cudaMemcpyDeviceToHost));
        stats.d2h += static_cast<long long>(sizeof(double) * res.size());
        for (int i = 0; i < npar; ++i) {
            if (steps[i] <= 0) continue;  // failed crossover, or a satisfied residual (empty refill)
            const std::vector<double> c(res.begin() + static_cast<size_t>(i) * m_.n,
                                        res.begin() + static_cast<size_t>(i + 1) * m_.n);
            const uint64_t seed = mix_seed_u64(p.seed, (static_cast<uint64_t>(round) << 20) + static_cast<uint64_t>(i));
            RolloutResult rr = rollouts(c, slow->n_rollouts, slow->topk, 2 * steps[i], seed, slow->id_offset,
                                        slow->batch, slow->table_log2, nullptr);
            if (rr.best_len >= 0 && rr.best_len < steps[i]) {
                std::vector<uint64_t> rows_h;
                for (long long idx : rr.path) rows_h.push_back(base_rows_[static_cast<size_t>(idx)]);
                uint64_t* dst = r->alt + static_cast<size_t>(i) * r->L_cap;
                CK(cudaMemcpy(dst, rows_h.data(), sizeof(uint64_t) * rows_h.size(), cudaMemcpyHostToDevice));
                stats.h2d += static_cast<long long>(sizeof(uint64_t) * rows_h.size());
                rows[i] = dst;
                steps[i] = rr.best_len;
            }
        }
    }
    CK(cudaMemcpy(r->refill, rows.data(), sizeof(void*) * npar, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r->refill_n, steps.data(), sizeof(int) * npar, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(r->child_len, parent_len.data(), sizeof(int) * npar, cudaMemcpyHostToDevice));
    GaFinishArgs f{};
    f.M = dm_;
    f.work = r->work;
    f.child = r->child;
    f.n_surv = r->n_surv;
    f.refill = r->refill;
    f.refill_n = r->refill_n;
    f.child_len = r->child_len;
    f.child_slack = r->child_slack;
    f.L_cap = r->L_cap;
    {
        void* args[] = {&f};
        CK(cudaLaunchKernel(ga_finish_kernel_ptr(), npar, ga_threads(), args, ga_finish_smem_bytes(m_.n), nullptr));
        stats.launches++;
        CK(cudaDeviceSynchronize());
    }
    child_len.resize(npar);
    child_slack.resize(npar);
    CK(cudaMemcpy(child_len.data(), r->child_len, sizeof(int) * npar, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(child_slack.data(), r->child_slack, sizeof(double) * npar, cudaMemcpyDeviceToHost));
    stats.h2d += static_cast<long long>(sizeof(int) * 3 * npar + sizeof(void*) * npar);
    stats.d2h += static_cast<long long>((sizeof(int) * 2 + sizeof(double)) * npar);
}

// Next population buffer: entry j is (from_child ? child[idx] : pop[buf][idx]) of length len.
void Engine::ga_select(GaRun* r, int buf, const std::vector<std::tuple<bool, int, int>>& order) {
    const int nxt = buf ^ 1;
    for (size_t j = 0; j < order.size(); ++j) {
        const auto& [from_child, idx, len] = order[j];
        const uint64_t* src = (from_child ? r->child : r->pop[buf]) + static_cast<size_t>(idx) * r->L_cap;
        if (len) CK(cudaMemcpyAsync(r->pop[nxt] + j * static_cast<size_t>(r->L_cap), src, len * 8ull,
                                    cudaMemcpyDeviceToDevice, nullptr));
    }
    CK(cudaDeviceSynchronize());
}

void Engine::set_shard(int rank, int n_ranks, const std::vector<void*>& boards, int max_ctas) {
    MGB_RANGE("migplan: set_shard");
    if (n_ranks < 1 || n_ranks > kMaxRanks || rank < 0 || rank >= n_ranks)
        throw ArgumentError("set_shard: rank/n_ranks out of range (1..8 ranks)");
    if (n_ranks > 1 && static_cast<int>(boards.size()) != n_ranks) throw ArgumentError("set_shard: one board per rank");
    CK(cudaSetDevice(device_));
    if (d_shard_) {
        CK(cudaFree(d_shard_));
        d_shard_ = nullptr;
    }
    n_shard_ = 0;
    max_ctas_ = max_ctas;
    rank_ = rank;
    n_ranks_ = 1;
    boards_.clear();
    if (n_ranks == 1) return;
    // base rows by support, balanced by row count: supports in pool order, each to the rank
    // holding the fewest rows so far (ties: lowest rank) — the same deal on every rank
    std::vector<uint64_t> mine;
    std::vector<long long> load(n_ranks, 0);
    for (size_t i = 0; i + 1 < support_off_.size(); ++i) {
        const int q = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
        load[q] += support_off_[i + 1] - support_off_[i];
        if (q == rank)
            mine.insert(mine.end(), base_rows_.begin() + support_off_[i], base_rows_.begin() + support_off_[i + 1]);
    }
    CK(cudaMalloc(&d_shard_, std::max<size_t>(mine.size(), 1) * 8 + 16));
    if (!mine.empty()) CK(cudaMemcpy(d_shard_, mine.data(), mine.size() * 8, cudaMemcpyHostToDevice));
    stats.h2d += static_cast<long long>(mine.size() * 8);
    n_shard_ = static_cast<long long>(mine.size());
    // the own board starts empty (every rank zeroes its own before the group's first call)
    CK(cudaMemset(boards[rank], 0, board_bytes(n_ranks)));
    CK(cudaDeviceSynchronize());
    boards_ = boards;
    n_ranks_ = n_ranks;
    exch_seq_ = 0;
}

size_t board_bytes(int n_ranks) { return sizeof(ExchSlot) * 2 * static_cast<size_t>(std::max(n_ranks, 1)); }

void* board_alloc(int device, int n_ranks, unsigned char ipc_handle[64]) {
    CK(cudaSetDevice(device));
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(board_bytes(n_ranks), 256)));
    CK(cudaMemset(p, 0, board_bytes(n_ranks)));
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        CK(cudaIpcGetMemHandle(&h, p));
        std::memcpy(ipc_handle, &h, 64);
    }
    return p;
}

void* board_open(int device, const unsigned char ipc_handle[64]) {
    CK(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, 64);
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    return p;
}

void board_close(void* board, bool opened) {
    if (!board) return;
    if (opened) cudaIpcCloseMemHandle(board);
    else cudaFree(board);
}

// completion_of / detail::sum_rates (core.hpp:245-269): counts keyed by (svc, size, batch)
// in key order, total += count * thr, one division per service.
std::vector<double> Engine::completion_of(const std::vector<Config>& cfgs) const {
    // Fast path (every configuration the optimizer itself builds): each instance runs its
    // service's selected batch for its size, so the reference's per-(service, size, batch)
    // sums (core.hpp:245-269) are dense counts summed in ascending size order — the same
    // additions in the same order as the general path below, without its ordered map.
    {
        const int S = static_cast<int>(m_.sizes.size());
        thread_local std::vector<long long> cnt;
        cnt.assign(static_cast<size_t>(m_.n) * S, 0);
        int sidx[16];
        for (int& v : sidx) v = -1;
        for (int i = 0; i < S; ++i)
            if (m_.sizes[i] >= 0 && m_.sizes[i] < 16) sidx[m_.sizes[i]] = i;
        bool fast = true;
        for (const auto& c : cfgs) {
            for (int k = 0; k < c.n && fast; ++k) {
                const auto& in = c.inst[k];
                const int si = in.slices >= 0 && in.slices < 16 ? sidx[in.slices] : -1;
                if (in.svc < 0 || in.svc >= m_.n || si < 0 || !m_.feas[in.svc][si].ok || m_.feas[in.svc][si].batch != in.batch) {
                    fast = false;
                    break;
                }
                ++cnt[static_cast<size_t>(in.svc) * S + si];
            }
            if (!fast) break;
        }
        if (fast) {
            std::vector<double> out(m_.n);
            for (int i = 0; i < m_.n; ++i) {
                double total = 0.0;
                for (int si = 0; si < S; ++si) {
                    const long long c = cnt[static_cast<size_t>(i) * S + si];
                    if (c == 0) continue;
                    volatile double prod = static_cast<double>(c) * m_.feas[i][si].thr;
                    total = total + prod;
                }
                out[i] = total / m_.services[i].req;
            }
            return out;
        }
    }
    std::map<std::tuple<int, int, int>, long long> counts;
    for (const auto& c : cfgs)
        for (int k = 0; k < c.n; ++k) {
            const auto& in = c.inst[k];
            if (in.svc < 0 || in.svc >= m_.n) throw PlanningError("unknown service index in configuration");
            counts[{in.svc, in.slices, in.batch}] += 1;
        }
    std::vector<double> total(m_.n, 0.0);
    for (const auto& [key, count] : counts) {
        auto [idx, size, batch] = key;
        const auto& prof = profiles_.at(m_.services[idx].model);
        const ProfileEntry* e = nullptr;
        auto it = prof.entries.find(size);
        if (it != prof.entries.end())
            for (const auto& pe : it->second)
                if (pe.batch == batch) e = &pe;
        if (!e)
            throw PlanningError("profile '" + m_.services[idx].model + "' has no entry for size " +
                                std::to_string(size) + " batch " + std::to_string(batch));
        volatile double prod = static_cast<double>(count) * e->thr;
        total[idx] = total[idx] + prod;
    }
    std::vector<double> out(m_.n);
    for (int i = 0; i < m_.n; ++i) out[i] = total[i] / m_.services[i].req;
    return out;
}

}  // namespace mgb

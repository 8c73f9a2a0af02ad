// model.hpp — host-side domain model of the B200 optimizer.
//
// Turns the reference's inputs (PartitionRuleSet, ProfileStore, ServiceSpec[]) into the
// small dense tables the sm_100a kernels consume, and encodes/decodes the packed
// 8-byte candidate row.  Reference semantics restated here (file:line under
// /root/reference/proj/include/migplan):
//   is_legal_partition            mig_rules.hpp:38-59
//   enumerate_maximal_partitions  mig_rules.hpp:67-135
//   canonical_size_multisets      config_enum.hpp:41-64
//   select_batch / select_entry   core.hpp:122-138, feasibility_table config_enum.hpp:73-84
//   sum_rates / utility_of        core.hpp:245-276
//   fill_group / materialize      config_enum.hpp:119-183
//   GpuConfig total order         core.hpp:174-200, candidate_preferred greedy.hpp:63-67
//
// The packed row.  A candidate config with support S = {s0 < s1 < s2 < s3} (|S| <= 4) is
// fully determined by, for every member, its per-instance-size COUNT VECTOR ("pattern"):
// the layout is the sum of the patterns (one canonical layout per size multiset) and
// inside each size group the lower service index takes the lower slots.  Its utility for
// member j is U[s_j][p_j] = (sum_{size asc} count * thr) / req — a function of
// (service, pattern) only.  So a row is four u16 codes  code_j = s_j * PP + p_j  (unused
// positions hold the sentinel code n*PP whose utility is 0), i.e. 8 bytes instead of the
// 44-byte (4 x f64 util, 4 x u8 svc, f64 util_sum) record, and a greedy step reads
// 8 B/row from HBM plus a (n+1) x PP table of need*U products held in shared memory.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgb {

struct PlanningError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SchemaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ArgumentError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

constexpr double kSatisfyEps = 1e-9;  // core.hpp:18
constexpr int kMaxInst = 7;
constexpr int kRowK = 4;              // members per packed row (extensions mix <= 4, greedy.hpp:116)
constexpr int kMaxServices = 255;     // u8 service index in the 128-bit order key
constexpr int kMaxSizes = 5;          // {1,2,3,4,7}
constexpr int kMaxLayouts = 32;
constexpr int kMaxPatterns = 64;

inline bool valid_slices(int s) { return s == 1 || s == 2 || s == 3 || s == 4 || s == 7; }

struct Place {
    int slices = 1;
    int slot = 0;
    auto operator<=>(const Place&) const = default;
};

struct Rules {  // PartitionRuleSet, mig_rules.hpp:15-34
    std::map<int, std::vector<int>> slot_positions;
    std::map<int, int> memory_weight;
    std::set<std::pair<int, int>> hard_exclusions;
    int memory_budget = 8;
    static Rules defaults();
};

bool is_legal(const std::vector<Place>& ps, const Rules& r);
std::vector<std::vector<Place>> maximal_partitions(const Rules& r);  // sorted by start slot, key-ordered

struct ProfileEntry {
    int batch = 1;
    double thr = 0.0;
    double p90 = 0.0;
};
struct ModelProfile {
    std::string name;
    std::map<int, std::vector<ProfileEntry>> entries;  // size -> sorted by batch
};
struct Service {
    std::string id, model;
    double req = 0.0, p90 = 0.0;
};

void validate_profile(const ModelProfile& p);  // core.hpp:81-104

struct Layout {  // one canonical layout: groups by size descending, slots ascending
    struct Group {
        int size = 0;
        int size_idx = 0;
        std::vector<int> slots;
    };
    std::vector<Group> groups;
    std::array<uint8_t, kMaxSizes> count{};  // placements per size index
};

// A support template: k labelled members (positions in ascending service order) and
// one pattern id per position.
struct Template {
    int layout = 0;
    std::array<uint8_t, kRowK> pat{};
};

struct Feasible {
    bool ok = false;
    int batch = 1;
    double thr = 0.0;
};

// Dense model of one PlanContext.
struct Model {
    int n = 0;  // services
    int max_mix = 2;
    std::vector<Service> services;
    std::vector<int> sizes;  // distinct instance sizes used by layouts, ascending
    std::vector<Layout> layouts;
    int PP = 0;  // pattern count (row code = svc * PP + pattern)
    std::vector<std::array<uint8_t, kMaxSizes>> patterns;  // per-size-index counts
    std::vector<uint8_t> pat_mask;                         // bit i = size index i used
    std::vector<std::vector<Template>> templates;          // [k] for k = 0..kRowK
    std::vector<std::vector<Feasible>> feas;               // [svc][size idx]
    std::vector<uint8_t> feas_mask;                        // [svc]
    std::vector<double> U;                                 // (n+1) * PP, row n = 0
    std::vector<double> best_single;                       // [svc], config_enum.hpp:179-180
    uint16_t sentinel() const { return static_cast<uint16_t>(n * PP); }

    // row codec
    int members(uint64_t row, int* svc, int* pat) const;
    struct Inst {
        int slices, slot, svc, batch;
    };
    int decode(uint64_t row, Inst* out) const;  // normalized instances, returns count
    // the config of members (svc ascending, pattern ids; any k <= 7): canonical layout of the
    // summed patterns, lower service index on the lower slots of each size group
    int decode_members(const int* svc, const int* pat, int k, Inst* out) const;
    std::array<uint64_t, 2> key(uint64_t row) const;
    double util_sum(uint64_t row) const;
    double score(uint64_t row, const double* comp) const;
    int64_t rows_for_support(const int* s, int k) const;
    // GPU genome of the throughput-mode GA (device.cuh GaBreedArgs): layout id + the service
    // of each instance in normalized order.  genome_of throws if no canonical layout has
    // exactly these placements.
    uint64_t genome_of(const Inst* inst, int n) const;
    int decode_genome(uint64_t g, Inst* out) const;
    void emit_support(const int* s, int k, std::vector<uint64_t>& out) const;
};

Model build_model(const Rules& rules, const std::map<std::string, ModelProfile>& profiles,
                  const std::vector<Service>& services, int max_mix);

// 128-bit lexicographic key of an arbitrary normalized instance list (core.hpp:174-200).
std::array<uint64_t, 2> key_of(const Model::Inst* inst, int n);

inline bool key_less(const std::array<uint64_t, 2>& a, const std::array<uint64_t, 2>& b) {
    return a[0] != b[0] ? a[0] < b[0] : a[1] < b[1];
}

}  // namespace mgb

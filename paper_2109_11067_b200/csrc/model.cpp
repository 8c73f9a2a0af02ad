// model.cpp — see model.hpp.  Host-side only; builds the tables the kernels stream.
#include "model.hpp"

#include <algorithm>
#include <functional>

namespace mgb {

Rules Rules::defaults() {  // mig_rules.hpp:21-33
    Rules r;
    r.slot_positions = {{1, {0, 1, 2, 3, 4, 5, 6}}, {2, {0, 2, 4}}, {3, {0, 4}}, {4, {0}}, {7, {0}}};
    r.memory_weight = {{1, 1}, {2, 2}, {3, 4}, {4, 4}, {7, 8}};
    r.hard_exclusions = {{3, 4}};
    r.memory_budget = 8;
    return r;
}

// is_legal_partition, mig_rules.hpp:38-59: legal start slot, 7-slot mask without overlap,
// memory budget in eighths, no hard-excluded size pair.
bool is_legal(const std::vector<Place>& ps, const Rules& r) {
    unsigned occupied = 0;
    int memory = 0;
    for (const auto& p : ps) {
        auto pos = r.slot_positions.find(p.slices);
        if (pos == r.slot_positions.end()) return false;
        if (std::find(pos->second.begin(), pos->second.end(), p.slot) == pos->second.end()) return false;
        if (p.slot < 0 || p.slices < 1 || p.slot + p.slices > 7) return false;
        unsigned mask = ((1u << p.slices) - 1u) << p.slot;
        if (occupied & mask) return false;
        occupied |= mask;
        auto w = r.memory_weight.find(p.slices);
        if (w == r.memory_weight.end()) return false;
        memory += w->second;
    }
    if (memory > r.memory_budget) return false;
    for (size_t i = 0; i < ps.size(); ++i)
        for (size_t j = i + 1; j < ps.size(); ++j) {
            auto pr = ps[i].slices <= ps[j].slices ? std::pair{ps[i].slices, ps[j].slices}
                                                   : std::pair{ps[j].slices, ps[i].slices};
            if (r.hard_exclusions.count(pr)) return false;
        }
    return true;
}

// enumerate_maximal_partitions, mig_rules.hpp:67-135.  The universe is every (size, slot)
// with slot+size <= 7, sorted; legal subsets are grown in index order (each subset once),
// maximal ones kept, then ordered by (sizes descending, slots ascending).
std::vector<std::vector<Place>> maximal_partitions(const Rules& r) {
    std::vector<Place> universe;
    for (const auto& [size, slots] : r.slot_positions)
        for (int s : slots)
            if (s + size <= 7) universe.push_back(Place{size, s});
    std::sort(universe.begin(), universe.end());

    std::vector<std::vector<Place>> legal;
    std::vector<Place> cur;
    std::function<void(size_t)> grow = [&](size_t from) {
        legal.push_back(cur);
        for (size_t i = from; i < universe.size(); ++i) {
            cur.push_back(universe[i]);
            if (is_legal(cur, r)) grow(i + 1);
            cur.pop_back();
        }
    };
    grow(0);

    auto maximal = [&](const std::vector<Place>& p) {
        std::vector<Place> t = p;
        for (const auto& extra : universe) {
            if (std::find(t.begin(), t.end(), extra) != t.end()) continue;
            t.push_back(extra);
            bool ok = is_legal(t, r);
            t.pop_back();
            if (ok) return false;
        }
        return true;
    };
    using Key = std::pair<std::vector<int>, std::vector<int>>;
    auto key = [](const std::vector<Place>& p) {
        Key k;
        for (const auto& x : p) k.first.push_back(x.slices), k.second.push_back(x.slot);
        std::sort(k.first.begin(), k.first.end(), std::greater<>());
        std::sort(k.second.begin(), k.second.end());
        return k;
    };
    std::vector<std::pair<Key, std::vector<Place>>> out;
    for (auto& p : legal) {
        if (p.empty() && !universe.empty()) continue;
        if (!maximal(p)) continue;
        std::sort(p.begin(), p.end(), [](const Place& a, const Place& b) { return a.slot < b.slot; });
        out.emplace_back(key(p), p);
    }
    std::stable_sort(out.begin(), out.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<std::vector<Place>> res;
    for (auto& [k, p] : out) res.push_back(std::move(p));
    return res;
}

void validate_profile(const ModelProfile& p) {  // core.hpp:81-104
    if (p.name.empty()) throw SchemaError("profile with empty model name");
    for (const auto& [size, list] : p.entries) {
        if (!valid_slices(size))
            throw SchemaError("profile " + p.name + ": invalid instance size " + std::to_string(size));
        double prev_p90 = 0.0;
        int prev_batch = 0;
        for (const auto& e : list) {
            if (e.batch <= 0) throw SchemaError("profile " + p.name + ": non-positive batch");
            if (e.batch <= prev_batch)
                throw SchemaError("profile " + p.name + ": duplicate or unsorted batch " + std::to_string(e.batch) +
                                  " for size " + std::to_string(size));
            if (e.thr <= 0.0 || e.p90 <= 0.0)
                throw SchemaError("profile " + p.name + ": non-positive measurement at size " +
                                  std::to_string(size) + " batch " + std::to_string(e.batch));
            if (e.p90 < prev_p90)
                throw SchemaError("profile " + p.name + ": p90 decreases with batch at size " + std::to_string(size));
            prev_p90 = e.p90;
            prev_batch = e.batch;
        }
    }
}

namespace {

// All ways to split `total` identical slots among k labelled members (compositions).
void compositions(int total, int k, std::vector<int>& cur, std::vector<std::vector<int>>& out) {
    if (static_cast<int>(cur.size()) == k - 1) {
        cur.push_back(total);
        out.push_back(cur);
        cur.pop_back();
        return;
    }
    for (int c = 0; c <= total; ++c) {
        cur.push_back(c);
        compositions(total - c, k, cur, out);
        cur.pop_back();
    }
}

}  // namespace

Model build_model(const Rules& rules, const std::map<std::string, ModelProfile>& profiles,
                  const std::vector<Service>& services, int max_mix) {
    Model m;
    m.n = static_cast<int>(services.size());
    m.max_mix = max_mix;
    m.services = services;
    if (m.n > kMaxServices)
        throw ArgumentError("the B200 planner supports at most " + std::to_string(kMaxServices) + " services");
    if (max_mix < 1 || max_mix > kRowK)
        throw ArgumentError("the B200 planner supports max_mix in [1, 4] (packed 4-member rows)");
    for (const auto& [size, slots] : rules.slot_positions)
        if (!valid_slices(size)) throw SchemaError("invalid size '" + std::to_string(size) + "'");

    // canonical_size_multisets, config_enum.hpp:41-64: first maximal partition per size
    // multiset (in partition_key order); groups by size descending, placements ascending.
    std::set<std::vector<int>> seen;
    std::vector<std::map<int, std::vector<int>, std::greater<>>> raw;
    for (const auto& part : maximal_partitions(rules)) {
        std::vector<int> sizes;
        for (const auto& p : part) sizes.push_back(p.slices);
        std::sort(sizes.begin(), sizes.end(), std::greater<>());
        if (!seen.insert(sizes).second) continue;
        std::map<int, std::vector<int>, std::greater<>> g;
        for (const auto& p : part) g[p.slices].push_back(p.slot);
        for (auto& [s, v] : g) std::sort(v.begin(), v.end());
        raw.push_back(std::move(g));
    }
    std::set<int> size_set;
    for (const auto& g : raw)
        for (const auto& [s, v] : g) size_set.insert(s);
    m.sizes.assign(size_set.begin(), size_set.end());
    auto size_idx = [&](int s) { return static_cast<int>(std::find(m.sizes.begin(), m.sizes.end(), s) - m.sizes.begin()); };
    if (raw.size() > kMaxLayouts) throw ArgumentError("too many canonical layouts");
    for (const auto& g : raw) {
        Layout L;
        for (const auto& [s, v] : g) {
            L.groups.push_back(Layout::Group{s, size_idx(s), v});
            L.count[size_idx(s)] = static_cast<uint8_t>(v.size());
        }
        m.layouts.push_back(std::move(L));
    }

    // Templates: every count matrix (k labelled members x groups) whose row sums are the
    // group sizes and in which every member holds >= 1 instance.  Equivalent to the
    // reference's nondecreasing per-group service sequences (config_enum.hpp:140) with
    // support exactly the k members.
    std::map<std::array<uint8_t, kMaxSizes>, int> pat_id;
    std::vector<std::vector<std::pair<int, std::vector<std::array<uint8_t, kMaxSizes>>>>> raw_t(kRowK + 1);
    for (int k = 1; k <= kRowK; ++k) {
        for (size_t li = 0; li < m.layouts.size(); ++li) {
            const Layout& L = m.layouts[li];
            std::vector<std::vector<std::vector<int>>> per_group;
            for (const auto& g : L.groups) {
                std::vector<std::vector<int>> comps;
                std::vector<int> cur;
                compositions(static_cast<int>(g.slots.size()), k, cur, comps);
                per_group.push_back(std::move(comps));
            }
            std::vector<size_t> choice(L.groups.size(), 0);
            std::function<void(size_t)> rec = [&](size_t gi) {
                if (gi == L.groups.size()) {
                    std::vector<std::array<uint8_t, kMaxSizes>> pats(k);
                    for (size_t g = 0; g < L.groups.size(); ++g)
                        for (int j = 0; j < k; ++j)
                            pats[j][L.groups[g].size_idx] = static_cast<uint8_t>(per_group[g][choice[g]][j]);
                    for (int j = 0; j < k; ++j) {
                        int tot = 0;
                        for (int s = 0; s < kMaxSizes; ++s) tot += pats[j][s];
                        if (tot == 0) return;
                    }
                    for (auto& p : pats) pat_id.emplace(p, 0);
                    raw_t[k].emplace_back(static_cast<int>(li), pats);
                    return;
                }
                for (size_t c = 0; c < per_group[gi].size(); ++c) {
                    choice[gi] = c;
                    rec(gi + 1);
                }
            };
            rec(0);
        }
    }
    int next = 0;
    for (auto& [p, id] : pat_id) {
        id = next++;
        m.patterns.push_back(p);
        uint8_t mask = 0;
        for (int s = 0; s < kMaxSizes; ++s)
            if (p[s]) mask |= static_cast<uint8_t>(1u << s);
        m.pat_mask.push_back(mask);
    }
    m.PP = next;
    if (m.PP > kMaxPatterns) throw ArgumentError("too many instance-count patterns");
    // codes < 2^14: the greedy scan gathers Wf at byte offset 4 * code, formed for two codes of
    // a 32-bit row half with one shift (kernels.cu ub2); kMaxServices/kMaxPatterns keep it so
    static_assert((kMaxServices + 1) * kMaxPatterns <= 16384);
    if ((m.n + 1) * m.PP > 16384) throw ArgumentError("service x pattern codes exceed 14 bits");
    m.templates.assign(kRowK + 1, {});
    for (int k = 1; k <= kRowK; ++k)
        for (const auto& [li, pats] : raw_t[k]) {
            Template t;
            t.layout = li;
            for (int j = 0; j < k; ++j) t.pat[j] = static_cast<uint8_t>(pat_id.at(pats[j]));
            m.templates[k].push_back(t);
        }
    // Template order fixes the arena order inside a support block (K1/K2 emit rows
    // template-major).  Sorting by (p0, p1, p2, p3) makes the rows a warp scans together share
    // their leading members' patterns, so the W-table gathers of those members mostly hit
    // one shared-memory address (broadcast) instead of conflicting banks.  The optimizer's
    // results do not depend on row order (the preference order is total, greedy.hpp:63-67).
    for (int k = 1; k <= kRowK; ++k)
        std::stable_sort(m.templates[k].begin(), m.templates[k].end(),
                         [](const Template& a, const Template& b) { return a.pat < b.pat; });

    // feasibility_table (config_enum.hpp:73-84) via select_entry (core.hpp:122-138).
    m.feas.assign(m.n, std::vector<Feasible>(m.sizes.size()));
    m.feas_mask.assign(m.n, 0);
    for (int i = 0; i < m.n; ++i) {
        auto it = profiles.find(services[i].model);
        if (it == profiles.end()) throw PlanningError("no profile for model '" + services[i].model + "'");
        for (size_t si = 0; si < m.sizes.size(); ++si) {
            auto e = it->second.entries.find(m.sizes[si]);
            if (e == it->second.entries.end()) continue;
            const ProfileEntry* best = nullptr;
            for (const auto& pe : e->second)
                if (pe.p90 <= services[i].p90) best = &pe;
            if (!best) continue;
            m.feas[i][si] = Feasible{true, best->batch, best->thr};
            m.feas_mask[i] |= static_cast<uint8_t>(1u << si);
        }
    }

    // Utility table: core.hpp:257-267 — per service, sizes ascending, total += count*thr,
    // then one division by the requirement.  Invalid (infeasible) cells stay 0 and are
    // never referenced by a row.
    m.U.assign(static_cast<size_t>(m.n + 1) * m.PP, 0.0);
    for (int i = 0; i < m.n; ++i)
        for (int p = 0; p < m.PP; ++p) {
            if (m.pat_mask[p] & ~m.feas_mask[i]) continue;
            double total = 0.0;
            for (size_t si = 0; si < m.sizes.size(); ++si)
                if (m.patterns[p][si]) {
                    volatile double prod = static_cast<double>(m.patterns[p][si]) * m.feas[i][si].thr;
                    total = total + prod;
                }
            m.U[static_cast<size_t>(i) * m.PP + p] = total / services[i].req;
        }
    // best_single_util: max utility over single-service configs (config_enum.hpp:177-181).
    m.best_single.assign(m.n, 0.0);
    for (int i = 0; i < m.n; ++i)
        for (const auto& t : m.templates[1])
            if (!(m.pat_mask[t.pat[0]] & ~m.feas_mask[i]))
                m.best_single[i] = std::max(m.best_single[i], m.U[static_cast<size_t>(i) * m.PP + t.pat[0]]);
    return m;
}

int Model::members(uint64_t row, int* svc, int* pat) const {
    int k = 0;
    for (int j = 0; j < kRowK; ++j) {
        int code = static_cast<int>((row >> (16 * j)) & 0xFFFF);
        if (code == sentinel()) break;
        svc[k] = code / PP;
        pat[k] = code % PP;
        ++k;
    }
    return k;
}

int Model::decode(uint64_t row, Inst* out) const {
    int svc[kRowK], pat[kRowK];
    const int k = members(row, svc, pat);
    return decode_members(svc, pat, k, out);
}

int Model::decode_members(const int* svc, const int* pat, int k, Inst* out) const {
    std::array<uint8_t, kMaxSizes> tot{};
    for (int j = 0; j < k; ++j)
        for (int s = 0; s < kMaxSizes; ++s) tot[s] = static_cast<uint8_t>(tot[s] + patterns[pat[j]][s]);
    int li = -1;
    for (size_t l = 0; l < layouts.size(); ++l)
        if (layouts[l].count == tot) li = static_cast<int>(l);
    if (li < 0) throw ArgumentError("row does not decode to a canonical layout");
    int n_inst = 0;
    for (const auto& g : layouts[li].groups) {
        size_t slot = 0;
        for (int j = 0; j < k; ++j)
            for (int c = 0; c < patterns[pat[j]][g.size_idx]; ++c)
                out[n_inst++] = Inst{g.size, g.slots[slot++], svc[j], feas[svc[j]][g.size_idx].batch};
    }
    std::sort(out, out + n_inst, [](const Inst& a, const Inst& b) {
        return a.slices != b.slices ? a.slices < b.slices : a.slot < b.slot;
    });
    return n_inst;
}

std::array<uint64_t, 2> key_of(const Model::Inst* inst, int n) {
    unsigned __int128 k = 0;
    for (int i = 0; i < kMaxInst; ++i) {
        unsigned f = 0;
        if (i < n) f = (1u << 14) | (static_cast<unsigned>(inst[i].slices) << 11) |
                       (static_cast<unsigned>(inst[i].slot) << 8) | static_cast<unsigned>(inst[i].svc);
        k = (k << 15) | f;
    }
    return {static_cast<uint64_t>(k >> 64), static_cast<uint64_t>(k)};
}

std::array<uint64_t, 2> Model::key(uint64_t row) const {
    Inst in[kMaxInst];
    int c = decode(row, in);
    return key_of(in, c);
}

double Model::util_sum(uint64_t row) const {  // config_enum.hpp:173
    int svc[kRowK], pat[kRowK];
    int k = members(row, svc, pat);
    double s = 0.0;
    for (int j = 0; j < k; ++j) s = s + U[static_cast<size_t>(svc[j]) * PP + pat[j]];
    return s;
}

double Model::score(uint64_t row, const double* comp) const {  // greedy.hpp:36-43
    int svc[kRowK], pat[kRowK];
    int k = members(row, svc, pat);
    double s = 0.0;
    for (int j = 0; j < k; ++j) {
        double need = 1.0 - comp[svc[j]];
        if (need > 0.0) {
            volatile double prod = need * U[static_cast<size_t>(svc[j]) * PP + pat[j]];
            s = s + prod;
        }
    }
    return s;
}

namespace {
// normalized (slices, slot) placements of a layout: size ascending, slot ascending
std::vector<std::pair<int, int>> layout_places(const Layout& L) {
    std::vector<std::pair<int, int>> v;
    for (const auto& g : L.groups)
        for (int slot : g.slots) v.emplace_back(g.size, slot);
    std::sort(v.begin(), v.end());
    return v;
}
}  // namespace

uint64_t Model::genome_of(const Inst* inst, int n) const {
    std::vector<std::pair<int, int>> want;
    for (int i = 0; i < n; ++i) want.emplace_back(inst[i].slices, inst[i].slot);
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return want[a] < want[b]; });
    std::vector<std::pair<int, int>> sorted;
    for (int i : order) sorted.push_back(want[i]);
    for (size_t l = 0; l < layouts.size(); ++l) {
        if (layout_places(layouts[l]) != sorted) continue;
        uint64_t g = static_cast<uint64_t>(l);
        int pos = 0;
        for (int i : order) g |= static_cast<uint64_t>(inst[i].svc) << (8 * (1 + pos++));
        for (; pos < kMaxInst; ++pos) g |= 0xFFull << (8 * (1 + pos));
        return g;
    }
    throw ArgumentError("configuration is not a canonical layout");
}

int Model::decode_genome(uint64_t g, Inst* out) const {
    const int l = static_cast<int>(g & 0xFF);
    if (l >= static_cast<int>(layouts.size())) throw ArgumentError("genome: bad layout");
    auto places = layout_places(layouts[l]);
    int n = 0;
    for (const auto& [size, slot] : places) {
        const int svc = static_cast<int>((g >> (8 * (1 + n))) & 0xFF);
        int si = 0;
        while (sizes[si] != size) ++si;
        out[n] = Inst{size, slot, svc, feas[svc][si].batch};
        ++n;
    }
    return n;
}

int64_t Model::rows_for_support(const int* s, int k) const {
    int64_t c = 0;
    for (const auto& t : templates[k]) {
        bool ok = true;
        for (int j = 0; j < k && ok; ++j) ok = !(pat_mask[t.pat[j]] & ~feas_mask[s[j]]);
        c += ok;
    }
    return c;
}

void Model::emit_support(const int* s, int k, std::vector<uint64_t>& out) const {
    for (const auto& t : templates[k]) {
        bool ok = true;
        for (int j = 0; j < k && ok; ++j) ok = !(pat_mask[t.pat[j]] & ~feas_mask[s[j]]);
        if (!ok) continue;
        uint64_t row = 0;
        for (int j = 0; j < kRowK; ++j) {
            uint64_t code = j < k ? static_cast<uint64_t>(s[j] * PP + t.pat[j]) : sentinel();
            row |= code << (16 * j);
        }
        out.push_back(row);
    }
}

}  // namespace mgb

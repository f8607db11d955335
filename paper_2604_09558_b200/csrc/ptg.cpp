// VTOG construction, points-to-graph validation, elimination and byte
// accounting (proj/src/vtog.cpp, proj/src/cost_model.cpp), plus the
// max-elimination strategy used where the reference planner cannot compose.
#include <algorithm>
#include <functional>

#include "lower.hpp"
#include "vtc/plan.hpp"

#include "kernels.hpp"
#include "lower.hpp"

namespace vtc {

std::vector<int> Vtog::out_edges(const std::string& node) const {
    std::vector<int> out;
    for (const auto& e : edges)
        if (e.src == node) out.push_back(e.id);
    return out;
}

bool Vtog::conflicting(int e1, int e2) const {
    if (e1 == e2) return false;
    const std::string& src = edges[size_t(e1)].src;
    if (edges[size_t(e2)].src != src) return false;
    auto it = conflicts.find(src);
    if (it == conflicts.end()) return false;
    auto pr = std::minmax(e1, e2);
    return it->second.count({pr.first, pr.second}) > 0;
}

// vtog.cpp:31-78: one edge per (candidate, base target); conflicts = pairs of
// out-edges of a node that overlap without agreeing.
Vtog build_vtog(const CompGraph& g) {
    Vtog v;
    v.graph = &g;
    for (const auto& t : g.tensors()) v.nodes.push_back(t.id);
    int cand_idx = 0;
    for (const auto& n : g.nodes()) {
        if (!is_data_movement(n)) continue;
        for (const auto& c : vt_rules(n, g)) {
            const TensorSpec& vt = g.tensor(c.virtual_tensor);
            int64_t dom = c.map.domain_volume();
            for (const auto& base : c.map.targets()) {
                std::vector<VPiece> ps;
                for (const auto& p : c.map.pieces())
                    if (p.target == base) ps.push_back(p);
                VtEdge e;
                e.id = int(v.edges.size());
                e.src = c.virtual_tensor;
                e.dst = base;
                e.map = VMap(vt.shape, std::move(ps));
                e.partial = e.map.covered_volume() < dom;
                e.direction = c.direction;
                e.static_class = c.static_class;
                e.eliminated_op = c.eliminated_op;
                e.candidate = cand_idx;
                v.edges.push_back(std::move(e));
            }
            ++cand_idx;
        }
    }
    for (size_t i = 0; i < v.edges.size(); ++i)
        for (size_t j = i + 1; j < v.edges.size(); ++j) {
            const auto &a = v.edges[i], &b = v.edges[j];
            if (a.src != b.src) continue;
            // overlap volume on the virtual index space
            int64_t overlap = 0;
            for (const auto& p : a.map.pieces())
                for (const auto& q : b.map.pieces()) {
                    int64_t vol = 1;
                    for (size_t d = 0; d < p.lo.size(); ++d) {
                        int64_t lo = std::max(p.lo[d], q.lo[d]), hi = std::min(p.hi[d], q.hi[d]);
                        vol *= std::max<int64_t>(0, hi - lo);
                    }
                    overlap += vol;
                }
            if (overlap > 0 && a.map.agree_volume(b.map) != overlap) v.conflicts[a.src].insert({int(i), int(j)});
        }
    return v;
}

bool PointsToGraph::is_virtual(const std::string& t) const {
    return std::find(roots.begin(), roots.end(), t) == roots.end();
}

const VMap& PointsToGraph::map_of(const std::string& t) const {
    auto it = resolved.find(t);
    if (it == resolved.end()) throw SchemaError("no resolved map for tensor " + t);
    return it->second;
}

namespace {

std::function<const VMap*(const std::string&)> virtual_lookup(const std::map<std::string, VMap>& resolved,
                                                             const std::vector<std::string>& roots) {
    return [&resolved, &roots](const std::string& t) -> const VMap* {
        if (std::find(roots.begin(), roots.end(), t) != roots.end()) return nullptr;
        auto it = resolved.find(t);
        return it == resolved.end() ? nullptr : &it->second;
    };
}

}  // namespace

// vtog.cpp:90-121: a DM node needs no kernel when each output's resolved map
// already equals the gather map composed over its inputs' resolved maps.
std::vector<std::string> eliminated_nodes(const CompGraph& g, const std::map<std::string, VMap>& resolved,
                                          const std::vector<std::string>& roots) {
    std::vector<std::string> out;
    auto lookup = virtual_lookup(resolved, roots);
    for (const auto& n : g.nodes()) {
        if (!is_data_movement(n)) continue;
        bool all = true;
        for (const auto& o : n.outputs) {
            VMap expected = gather_map(n, o, g).compose(lookup);
            if (resolved.at(o).agree_volume(expected) != g.tensor(o).elems()) {
                all = false;
                break;
            }
        }
        if (all) out.push_back(n.id);
    }
    return out;
}

PointsToGraph all_physical_ptg(const CompGraph& g) {
    PointsToGraph p;
    for (const auto& t : g.tensors()) {
        p.roots.push_back(t.id);
        p.resolved.emplace(t.id, VMap::identity(t.id, t.shape));
    }
    p.eliminated_ops = eliminated_nodes(g, p.resolved, p.roots);
    return p;
}

// vtog.cpp:123-207
PointsToGraph validate_ptg(const Vtog& v, const std::vector<int>& selected) {
    const CompGraph& g = *v.graph;
    PointsToGraph ptg;
    ptg.selected = selected;
    std::sort(ptg.selected.begin(), ptg.selected.end());
    ptg.selected.erase(std::unique(ptg.selected.begin(), ptg.selected.end()), ptg.selected.end());

    std::map<std::string, std::vector<int>> groups;
    for (int e : ptg.selected) {
        if (e < 0 || e >= int(v.edges.size())) throw InvalidVtogError("selected edge id out of range");
        groups[v.edges[size_t(e)].src].push_back(e);
    }
    std::map<std::string, VMap> merged;
    for (const auto& [src, eids] : groups) {
        for (size_t i = 0; i < eids.size(); ++i)
            for (size_t j = i + 1; j < eids.size(); ++j)
                if (v.conflicting(eids[i], eids[j]))
                    throw ConflictViolationError("edges " + std::to_string(eids[i]) + " and " +
                                                 std::to_string(eids[j]) + " conflict at " + src);
        std::vector<VPiece> ps;
        for (int e : eids)
            for (const auto& p : v.edges[size_t(e)].map.pieces()) ps.push_back(p);
        VMap m(g.tensor(src).shape, std::move(ps));
        if (m.has_overlap()) throw ConflictViolationError("merged maps overlap at " + src);
        if (!m.is_total()) throw IncompleteSelectionError("selection at " + src + " does not cover the whole index space");
        merged.emplace(src, std::move(m));
    }

    std::map<std::string, int> color;
    std::vector<std::string> order;
    std::function<void(const std::string&)> visit = [&](const std::string& t) {
        auto it = merged.find(t);
        if (it == merged.end()) return;
        int& c = color[t];
        if (c == 2) return;
        if (c == 1) throw CycleDetectedError("virtual tensors form a cycle near " + t);
        c = 1;
        for (const auto& b : it->second.targets()) visit(b);
        color[t] = 2;
        order.push_back(t);
    };
    for (const auto& [src, m] : merged) visit(src);

    for (const auto& t : g.tensors())
        if (!merged.count(t.id)) {
            ptg.roots.push_back(t.id);
            ptg.resolved.emplace(t.id, VMap::identity(t.id, t.shape));
        }
    for (const auto& t : order) {
        auto lookup = [&](const std::string& b) -> const VMap* {
            if (!merged.count(b)) return nullptr;
            auto it = ptg.resolved.find(b);
            if (it == ptg.resolved.end()) throw MissingBaseMapError("base map for " + b + " not resolved yet");
            return &it->second;
        };
        ptg.resolved.emplace(t, merged.at(t).compose(lookup));
    }
    ptg.eliminated_ops = eliminated_nodes(g, ptg.resolved, ptg.roots);
    std::set<std::string> elim(ptg.eliminated_ops.begin(), ptg.eliminated_ops.end());
    for (const auto& n : g.nodes()) {
        if (is_data_movement(n) && elim.count(n.id)) continue;
        for (const auto& o : n.outputs)
            if (!ptg.resolved.at(o).injective())
                throw WriteAliasingError("node " + n.id + " writes " + o + " through a non-injective map");
    }
    return ptg;
}

std::vector<int> plan_max_elimination(const Vtog& v) {
    const CompGraph& g = *v.graph;
    // candidates: id -> edges
    std::map<int, std::vector<int>> cand_edges;
    for (const auto& e : v.edges) cand_edges[e.candidate].push_back(e.id);
    auto cand_of = [&](const std::string& virt, VtDirection dir, const std::string& op,
                       const std::string& base_has) -> int {
        for (const auto& [c, es] : cand_edges) {
            const VtEdge& e0 = v.edges[size_t(es[0])];
            if (e0.src != virt || e0.direction != dir || e0.eliminated_op != op) continue;
            if (!base_has.empty()) {
                bool found = false;
                for (int e : es) found |= v.edges[size_t(e)].dst == base_has;
                if (!found) continue;
            }
            return c;
        }
        return -1;
    };

    std::vector<int> selected;
    std::set<std::string> assigned;
    std::map<std::string, int> chosen;  // virtual tensor -> candidate
    auto try_select = [&](int c) -> bool {
        if (c < 0) return false;
        const std::string& virt = v.edges[size_t(cand_edges[c][0])].src;
        if (assigned.count(virt)) return false;
        std::vector<int> trial = selected;
        for (int e : cand_edges[c]) trial.push_back(e);
        try {
            PointsToGraph p = validate_ptg(v, trial);
            // the device descriptor must hold every resolved map (<= VTC_MAX_PIECES pieces)
            for (const auto& [id, m] : p.resolved)
                lower_map(m, [](const std::string&) { return TargetInfo{0, 0}; });
        } catch (const Error&) {
            return false;
        }
        selected = std::move(trial);
        assigned.insert(virt);
        chosen[virt] = c;
        return true;
    };
    auto unselect = [&](const std::string& virt) {
        auto it = chosen.find(virt);
        if (it == chosen.end()) return;
        for (int e : cand_edges[it->second]) selected.erase(std::remove(selected.begin(), selected.end(), e), selected.end());
        assigned.erase(virt);
        chosen.erase(it);
    };

    // Phase 1: write-side chains.  A ScatterND output aliases its data in place
    // (rule i) and its updates become slabs of the output (rule ii); the
    // updates' producing data-movement chain is pulled back so the compute
    // producer writes straight into the destination.
    std::function<void(const std::string&)> pull_back = [&](const std::string& u) {
        const OpNode* p = g.producer(u);
        if (!p || !is_data_movement(*p)) return;
        if (p->kind == OpKind::Concat) {
            for (const auto& in : p->inputs)
                if (try_select(cand_of(in, VtDirection::InputOverOutput, p->id, u))) pull_back(in);
            return;
        }
        if (p->kind == OpKind::ScatterND || p->kind == OpKind::Slice) return;
        const std::string& x = p->inputs[0];
        if (try_select(cand_of(x, VtDirection::InputOverOutput, p->id, u))) pull_back(x);
    };
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        if (n.kind == OpKind::ScatterND) {
            try_select(cand_of(n.outputs[0], VtDirection::OutputOverInput, n.id, n.inputs[0]));
            if (try_select(cand_of(n.inputs[1], VtDirection::InputOverOutput, n.id, n.outputs[0])))
                pull_back(n.inputs[1]);
        } else if (n.kind == OpKind::Concat && g.tensor(n.outputs[0]).kind != TensorKind::Intermediate) {
            // a physical concat destination: inputs become windows of it
            pull_back(n.outputs[0]);
        }
    }
    // Phase 2: read-side gathers for every remaining data-movement output.
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        if (!is_data_movement(n) || n.kind == OpKind::ScatterND) continue;
        for (const auto& o : n.outputs) try_select(cand_of(o, VtDirection::OutputOverInput, n.id, ""));
        // graph-output destinations: let the producer write through the inverse map
        bool any_phys_out = false;
        for (const auto& o : n.outputs) any_phys_out |= g.tensor(o).kind != TensorKind::Intermediate;
        if (any_phys_out && n.kind != OpKind::Concat && n.kind != OpKind::Slice) {
            const std::string& x = n.inputs[0];
            const OpNode* px = g.producer(x);
            if (px && !is_data_movement(*px)) try_select(cand_of(x, VtDirection::InputOverOutput, n.id, ""));
        }
    }
    // Phase 3: a data-movement op still left as a copy (its gather map composed
    // with the upstream views does not lower, e.g. Roll after a window-reverse
    // chain) -- re-plan its upstream single-input DM chain in the other
    // direction: its output stays physical and the chain's tensors become
    // views of it, so the compute producer writes straight through the
    // composed (lowerable) inverse map.
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        if (!is_data_movement(n) || n.kind == OpKind::ScatterND || n.kind == OpKind::Concat || n.kind == OpKind::Split)
            continue;
        if (n.outputs.size() != 1 || assigned.count(n.outputs[0])) continue;
        std::vector<std::string> chain;  // tensors upstream of n's output through single-input DM ops
        std::string t = n.inputs[0];
        const OpNode* p = &n;
        while (true) {
            chain.push_back(t);
            const OpNode* q = g.producer(t);
            if (!q || !is_data_movement(*q) || q->inputs.size() != 1 || q->outputs.size() != 1 ||
                q->kind == OpKind::ScatterND || g.consumers(t).size() != 1)
                break;
            p = q;
            t = q->inputs[0];
        }
        (void)p;
        std::vector<int> saved = selected;
        std::set<std::string> saved_assigned = assigned;
        std::map<std::string, int> saved_chosen = chosen;
        for (const auto& c : chain) unselect(c);
        pull_back(n.outputs[0]);
        // keep the re-plan only if it eliminated more operators
        auto count_elim = [&](const std::vector<int>& sel) -> size_t {
            try {
                return validate_ptg(v, sel).eliminated_ops.size();
            } catch (const Error&) {
                return 0;
            }
        };
        if (count_elim(selected) <= count_elim(saved)) {
            selected = saved;
            assigned = saved_assigned;
            chosen = saved_chosen;
        }
    }
    // Phase 4: a bf16 MatMul whose A operand is a view the tensor-core GEMM cannot
    // read by TMA (e.g. Swin's roll + window partition, a head transpose whose
    // K digits are narrower than a 64-wide K tile): make A physical instead and
    // let the producer write through the inverse chain (LayerNorm / attention
    // store through any map), when that eliminates as many operators.
    auto count_elim = [&](const std::vector<int>& sel) -> size_t {
        try {
            return validate_ptg(v, sel).eliminated_ops.size();
        } catch (const Error&) {
            return 0;
        }
    };
    auto tma_ok = [&](const std::string& a) -> bool {
        try {
            PointsToGraph p = validate_ptg(v, selected);
            auto it = p.resolved.find(a);
            if (it == p.resolved.end()) return true;  // physical
            vtc_map d = lower_map(it->second, [](const std::string&) { return TargetInfo{0, 0}; });
            const TensorSpec& t = g.tensor(a);
            GemmTcParams probe{};
            int64_t dims[5], strides[5];
            const void* base = nullptr;
            return gemm_tc_a_dims(d, t.shape[0], t.shape[1], probe, dims, strides, &base);
        } catch (const Error&) {
            return true;
        }
    };
    // A plain 2-D operand (one TMA box per stage) also beats an N-D view when the
    // producer is an attention kernel, which stores rows through any map for free.
    auto tma_plain = [&](const std::string& a) -> bool {
        try {
            PointsToGraph p = validate_ptg(v, selected);
            auto it = p.resolved.find(a);
            if (it == p.resolved.end()) return true;
            vtc_map d = lower_map(it->second, [](const std::string&) { return TargetInfo{0, 0}; });
            const TensorSpec& t = g.tensor(a);
            GemmTcParams probe{};
            int64_t dims[5], strides[5];
            const void* base = nullptr;
            return gemm_tc_a_dims(d, t.shape[0], t.shape[1], probe, dims, strides, &base) && probe.a_ndims == 2;
        } catch (const Error&) {
            return true;
        }
    };
    auto attention_fed = [&](const std::string& a) -> bool {
        std::string t = a;
        for (int hop = 0; hop < 8; ++hop) {
            const OpNode* q = g.producer(t);
            if (!q) return false;
            if (!is_data_movement(*q)) return q->kind == OpKind::Attention;
            if (q->inputs.size() != 1) return false;
            t = q->inputs[0];
        }
        return false;
    };
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        if (n.kind != OpKind::MatMul) continue;
        const std::string& a = n.inputs[0];
        const TensorSpec& at = g.tensor(a);
        if (at.dtype != DType::BF16 || at.shape.size() != 2 || at.shape[0] <= 16 || !assigned.count(a)) continue;
        if (tma_ok(a) && (tma_plain(a) || !attention_fed(a))) continue;
        std::vector<std::string> chain;
        std::string t = a;
        while (true) {
            const OpNode* q = g.producer(t);
            if (!q || !is_data_movement(*q) || q->inputs.size() != 1 || q->outputs.size() != 1 ||
                q->kind == OpKind::ScatterND)
                break;
            chain.push_back(t);
            t = q->inputs[0];
            if (g.consumers(t).size() != 1) break;
            if (!g.producer(t) || !is_data_movement(*g.producer(t))) {
                chain.push_back(t);  // the compute producer's output becomes a view too
                break;
            }
        }
        std::vector<int> saved = selected;
        std::set<std::string> saved_assigned = assigned;
        std::map<std::string, int> saved_chosen = chosen;
        size_t before = count_elim(selected);
        for (const auto& c : chain) unselect(c);
        pull_back(a);
        if (count_elim(selected) < before || !tma_ok(a) || !tma_plain(a)) {
            selected = saved;
            assigned = saved_assigned;
            chosen = saved_chosen;
        }
    }
    std::sort(selected.begin(), selected.end());
    return selected;
}

std::vector<int> plan_inplace_updates(const Vtog& v) {
    const CompGraph& g = *v.graph;
    std::vector<int> selected;
    for (const auto& n : g.nodes()) {
        if (n.kind != OpKind::ScatterND) continue;
        for (const auto& e : v.edges) {
            if (e.src != n.outputs[0] || e.dst != n.inputs[0] || e.direction != VtDirection::OutputOverInput ||
                e.eliminated_op != n.id)
                continue;
            std::vector<int> trial = selected;
            trial.push_back(e.id);
            try {
                validate_ptg(v, trial);
                selected = std::move(trial);
            } catch (const Error&) {
            }
            break;
        }
    }
    std::sort(selected.begin(), selected.end());
    return selected;
}

int64_t KernelBytes::total() const {
    int64_t t = 0;
    for (const auto& r : reads) t += r.bytes;
    for (const auto& w : writes) t += w.bytes;
    return t;
}

int64_t TrafficEstimate::total_bytes() const {
    int64_t t = 0;
    for (const auto& k : kernels) t += k.total();
    return t;
}

int64_t TrafficEstimate::data_movement_bytes() const {
    int64_t t = 0;
    for (const auto& k : kernels)
        if (k.data_movement) t += k.total();
    return t;
}

TrafficEstimate estimate(const CompGraph& g, const PointsToGraph& ptg) {
    TrafficEstimate est;
    std::set<std::string> elim(ptg.eliminated_ops.begin(), ptg.eliminated_ops.end());
    auto lookup = virtual_lookup(ptg.resolved, ptg.roots);
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        bool dm = is_data_movement(n);
        if (dm && elim.count(n.id)) continue;
        KernelBytes k;
        k.node = n.id;
        k.data_movement = dm;
        if (!dm) {
            for (const auto& in : n.inputs) {
                const TensorSpec& t = g.tensor(in);
                k.reads.push_back({in, ptg.map_of(in).unique_elems() * dtype_size(t.dtype)});
            }
            for (const auto& o : n.outputs) k.writes.push_back({o, g.tensor(o).bytes()});
        } else {
            for (const auto& o : n.outputs) {
                int64_t es = dtype_size(g.tensor(o).dtype);
                const VMap& out_map = ptg.map_of(o);
                VMap full = gather_map(n, o, g);
                for (const auto& in : n.inputs) {
                    std::vector<VPiece> ps;
                    for (const auto& p : full.pieces())
                        if (p.target == in) ps.push_back(p);
                    if (ps.empty()) continue;
                    VMap flow = VMap(full.shape(), std::move(ps)).compose(lookup);
                    int64_t region = flow.covered_volume();
                    int64_t moved = region - out_map.agree_volume(flow);
                    if (moved <= 0) continue;
                    k.reads.push_back({in, std::min(moved, flow.unique_elems()) * es});
                    k.writes.push_back({o, moved * es});
                }
            }
        }
        (dm ? est.data_movement_kernels : est.compute_kernels) += 1;
        est.kernels.push_back(std::move(k));
    }
    return est;
}

}  // namespace vtc

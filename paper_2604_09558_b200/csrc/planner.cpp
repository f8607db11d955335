// Cost model, saving oracles, enumeration and the global greedy planner
// (include/vtc/planner.hpp).  The analytic model restates the reference's
// three-stage traffic model (proj/src/cost_model.cpp:81-176) over vtc::VMap;
// greedy_build is Alg. 2, which the reference snapshot
// does not ship (proj/CMakeLists.txt:21).
#include "vtc/planner.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <set>
#include <sstream>

#include <cuda_runtime.h>

#include "json.hpp"
#include "vtc/exec.hpp"

namespace vtc {

void MachineParams::validate() const {
    if (!(bandwidth > 0) || coalesce_unit <= 0 || !(kernel_launch_overhead > 0) || !(noncoalesced_penalty >= 1) ||
        !(partial_penalty >= 1))
        throw SchemaError("machine parameters must be positive (penalties >= 1)");
}

MachineParams MachineParams::from_json(const std::string& text) {
    MachineParams p;
    json::Value j = json::parse(text);
    if (j.contains("bandwidth")) p.bandwidth = j.at("bandwidth").as_double();
    if (j.contains("coalesce_unit")) p.coalesce_unit = j.at("coalesce_unit").as_int();
    if (j.contains("kernel_launch_overhead")) p.kernel_launch_overhead = j.at("kernel_launch_overhead").as_double();
    if (j.contains("noncoalesced_penalty")) p.noncoalesced_penalty = j.at("noncoalesced_penalty").as_double();
    if (j.contains("partial_penalty")) p.partial_penalty = j.at("partial_penalty").as_double();
    p.validate();
    return p;
}

std::string MachineParams::to_json() const {
    json::Value j = json::Value::object();
    j.set("bandwidth", json::Value::number(bandwidth));
    j.set("coalesce_unit", json::Value::integer(coalesce_unit));
    j.set("kernel_launch_overhead", json::Value::number(kernel_launch_overhead));
    j.set("noncoalesced_penalty", json::Value::number(noncoalesced_penalty));
    j.set("partial_penalty", json::Value::number(partial_penalty));
    return json::dump(j);
}

MachineParams MachineParams::b200() {
    // Fitted on one B200 by scripts/calibrate.py (profiles/r2_calibration.json),
    // time unit = microseconds: the executor's copy kernel (gather_copy) moves
    // 1.66 TB/s through contiguous maps (64 MB .. 1 GB), runs of >= 16 bytes
    // cost the same as contiguous ones (1.02x), 4-8 byte runs / element-
    // scattered transposes 2.6-2.9x, and each dependent launch inside a CUDA
    // graph adds 2.1 us.
    MachineParams p;
    p.bandwidth = 1.66e6;
    p.coalesce_unit = 16;
    p.kernel_launch_overhead = 2.1;
    p.noncoalesced_penalty = 2.86;
    p.partial_penalty = 1.02;
    return p;
}

double bandwidth_factor(const VMap& m, int64_t elem_size, const MachineParams& params) {
    switch (m.contiguity(elem_size, params.coalesce_unit).cls) {
        case ContiguityClass::FullyContiguous: return 1.0;
        case ContiguityClass::PartiallyContiguous: return 1.0 / params.partial_penalty;
        case ContiguityClass::NonContiguous: return 1.0 / params.noncoalesced_penalty;
    }
    return 1.0;
}

namespace {

std::function<const VMap*(const std::string&)> virtual_lookup(const PointsToGraph& ptg) {
    return [&ptg](const std::string& t) -> const VMap* {
        if (std::find(ptg.roots.begin(), ptg.roots.end(), t) != ptg.roots.end()) return nullptr;
        auto it = ptg.resolved.find(t);
        return it == ptg.resolved.end() ? nullptr : &it->second;
    };
}

}  // namespace

// cost_model.cpp:117-176: compute kernels read every operand's unique physical
// bytes and write every output in full; a data-movement kernel moves only the
// elements whose destination differs from where the source already lives.
TrafficEstimate estimate(const CompGraph& g, const PointsToGraph& ptg, const MachineParams& params) {
    params.validate();
    TrafficEstimate est;
    std::set<std::string> elim(ptg.eliminated_ops.begin(), ptg.eliminated_ops.end());
    auto lookup = virtual_lookup(ptg);
    for (int ni : g.topo_order()) {
        const OpNode& n = g.nodes()[size_t(ni)];
        bool dm = is_data_movement(n);
        if (dm && elim.count(n.id)) continue;
        KernelBytes k;
        k.node = n.id;
        k.data_movement = dm;
        if (!dm) {
            for (const auto& in : n.inputs) {
                int64_t es = dtype_size(g.tensor(in).dtype);
                const VMap& m = ptg.map_of(in);
                k.reads.push_back({in, m.unique_elems() * es, bandwidth_factor(m, es, params)});
            }
            for (const auto& o : n.outputs) {
                int64_t es = dtype_size(g.tensor(o).dtype);
                k.writes.push_back({o, g.tensor(o).bytes(), bandwidth_factor(ptg.map_of(o), es, params)});
            }
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
                    int64_t moved = flow.covered_volume() - out_map.agree_volume(flow);
                    if (moved <= 0) continue;
                    k.reads.push_back({in, std::min(moved, flow.unique_elems()) * es, bandwidth_factor(flow, es, params)});
                    k.writes.push_back({o, moved * es, bandwidth_factor(out_map, es, params)});
                }
            }
        }
        k.time = params.kernel_launch_overhead;
        for (const auto& r : k.reads) k.time += double(r.bytes) / (params.bandwidth * r.bandwidth_factor);
        for (const auto& w : k.writes) k.time += double(w.bytes) / (params.bandwidth * w.bandwidth_factor);
        est.total_time += k.time;
        (dm ? est.data_movement_kernels : est.compute_kernels) += 1;
        est.kernels.push_back(std::move(k));
    }
    return est;
}

LatencyBreakdown breakdown(const TrafficEstimate& est) {
    LatencyBreakdown b;
    for (const auto& k : est.kernels) {
        if (k.data_movement) {
            b.data_movement_time += k.time;
            ++b.data_movement_kernels;
        } else {
            b.compute_time += k.time;
            ++b.compute_kernels;
        }
    }
    return b;
}

namespace {

class AnalyticOracle final : public SavingOracle {
public:
    explicit AnalyticOracle(MachineParams p) : params_(p) { params_.validate(); }
    double evaluate(const CompGraph& g, const PointsToGraph& ptg) override {
        ++calls;
        if (base_graph_ != &g) {
            base_ = estimate(g, all_physical_ptg(g), params_).total_time;
            base_graph_ = &g;
        }
        return base_ - estimate(g, ptg, params_).total_time;
    }

private:
    MachineParams params_;
    const CompGraph* base_graph_ = nullptr;
    double base_ = 0.0;
};

#define VTC_CUDA_OK(x)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Device time (us) of one CUDA-graph replay of the strategy: median of `trials`.
double device_step_us(const CompGraph& g, const PointsToGraph& ptg, int trials, uint64_t seed) {
    Executor ex(g, ptg);
    ex.prepare();
    // deterministic small-magnitude bytes in every root (timing only; no NaN/Inf patterns)
    for (const auto& r : ex.roots())
        if (r.ptr && r.bytes > 0) VTC_CUDA_OK(cudaMemset(r.ptr, int(seed & 0x1f), size_t(r.bytes)));
    cudaStream_t s;
    VTC_CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    VTC_CUDA_OK(cudaEventCreate(&a));
    VTC_CUDA_OK(cudaEventCreate(&b));
    std::vector<double> ts;
    for (int t = 0; t < trials + 2; ++t) {
        VTC_CUDA_OK(cudaEventRecord(a, s));
        ex.run_graph(s);
        VTC_CUDA_OK(cudaEventRecord(b, s));
        VTC_CUDA_OK(cudaEventSynchronize(b));
        float ms = 0;
        VTC_CUDA_OK(cudaEventElapsedTime(&ms, a, b));
        if (t >= 2) ts.push_back(double(ms) * 1e3);  // two warm-ups (graph capture, first touch)
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

class DeviceTimedOracle final : public SavingOracle {
public:
    DeviceTimedOracle(int trials, uint64_t seed) : trials_(trials), seed_(seed) {
        if (trials_ < 3) throw ExecutionError("device-timed oracle needs at least 3 trials");
    }
    double evaluate(const CompGraph& g, const PointsToGraph& ptg) override {
        ++calls;
        if (base_graph_ != &g) {
            base_ = device_step_us(g, all_physical_ptg(g), trials_, seed_);
            base_graph_ = &g;
        }
        return base_ - device_step_us(g, ptg, trials_, seed_);
    }

private:
    int trials_;
    uint64_t seed_;
    const CompGraph* base_graph_ = nullptr;
    double base_ = 0.0;
};

}  // namespace

std::unique_ptr<SavingOracle> saving_oracle(const MachineParams& params) {
    return std::make_unique<AnalyticOracle>(params);
}

std::unique_ptr<SavingOracle> device_timed_oracle(int trials, uint64_t seed) {
    return std::make_unique<DeviceTimedOracle>(trials, seed);
}

// vtog.cpp:209-237: DFS over edges in id order, "skip" before "take", pruning
// a take that conflicts with an edge already taken at the same node; every
// leaf is validated and kept when valid.
std::vector<PointsToGraph> enumerate_ptgs(const Vtog& v, int64_t limit) {
    size_t ne = v.edges.size();
    if (limit < 0 && ne > 20)
        throw SpaceTooLargeError("VTOG has " + std::to_string(ne) + " edges; enumeration requires a limit");
    std::vector<PointsToGraph> out;
    std::vector<int> picked;
    std::function<void(size_t)> dfs = [&](size_t next) {
        if (limit >= 0 && int64_t(out.size()) >= limit) return;
        if (next == ne) {
            try {
                out.push_back(validate_ptg(v, picked));
            } catch (const Error&) {
            }
            return;
        }
        dfs(next + 1);
        for (int e : picked)
            if (v.conflicting(e, int(next))) return;
        picked.push_back(int(next));
        dfs(next + 1);
        picked.pop_back();
    };
    dfs(0);
    return out;
}

std::pair<std::vector<int>, double> max_edges(const Vtog& v, const std::vector<int>& cands,
                                              const std::function<double(const std::vector<int>&)>& w,
                                              const std::function<bool(const std::vector<int>&)>& feasible) {
    if (cands.size() > 16) throw BudgetExceededError("MaxEdges: more than 16 candidate edges at one node");
    std::vector<int> best;
    double best_s = 0.0;  // the empty set is always feasible
    size_t n = cands.size();
    for (uint32_t mask = 1; mask < (1u << n); ++mask) {
        std::vector<int> P;
        bool ok = true;
        for (size_t i = 0; i < n && ok; ++i) {
            if (!(mask >> i & 1)) continue;
            for (int e : P)
                if (v.conflicting(e, cands[i])) {
                    ok = false;
                    break;
                }
            P.push_back(cands[i]);
        }
        if (!ok || !feasible(P)) continue;
        double s = w(P);
        if (s > best_s) {
            best_s = s;
            best = std::move(P);
        }
    }
    return {best, best_s};
}

GreedyResult greedy_build(const Vtog& v, SavingOracle& oracle,
                          const std::function<bool(const PointsToGraph&)>& accept) {
    const CompGraph& g = *v.graph;
    GreedyResult res;
    int64_t calls0 = oracle.calls;
    std::set<std::string> A;
    std::vector<int> C;
    for (const auto& t : v.nodes)
        if (v.out_edges(t).empty()) A.insert(t);

    // Validity of C u P, memoised per selection.
    std::map<std::vector<int>, bool> valid_cache;
    auto sel_key = [&](const std::vector<int>& P) {
        std::vector<int> k = C;
        k.insert(k.end(), P.begin(), P.end());
        std::sort(k.begin(), k.end());
        return k;
    };
    auto valid = [&](const std::vector<int>& P) {
        auto k = sel_key(P);
        auto it = valid_cache.find(k);
        if (it != valid_cache.end()) return it->second;
        bool ok = true;
        try {
            PointsToGraph p = validate_ptg(v, k);
            if (accept) ok = accept(p);
        } catch (const Error&) {
            ok = false;
        }
        valid_cache.emplace(k, ok);
        return ok;
    };
    // l(C), refreshed when C changes.
    double lC = 0.0;  // l(empty) = 0 by definition
    // w(P) = l(C u P) - l(C), profiled once and re-profiled for subsets that
    // contain an edge into the node anchored last (Alg. 2 lines 7 and 24).
    std::map<std::vector<int>, double> w_cache;
    auto profile = [&](const std::vector<int>& P) {
        double l = oracle.evaluate(g, validate_ptg(v, sel_key(P)));
        return l - lC;
    };
    auto w = [&](const std::vector<int>& P) {
        std::vector<int> k = P;
        std::sort(k.begin(), k.end());
        auto it = w_cache.find(k);
        if (it != w_cache.end()) return it->second;
        double s = profile(P);
        w_cache.emplace(k, s);
        return s;
    };

    // ties between nodes with equal saving go to the lowest tensor
    // id lexicographically (this also decides which node is anchored as a
    // physical tensor when no edge into A saves anything yet).
    std::vector<std::string> order = v.nodes;
    std::sort(order.begin(), order.end());
    while (A.size() < v.nodes.size()) {
        double max_s = -1.0;
        std::string vc;
        std::vector<int> Pc;
        for (const auto& t : order) {
            if (A.count(t)) continue;
            std::vector<int> cands;
            for (int e : v.out_edges(t))
                if (A.count(v.edges[size_t(e)].dst)) cands.push_back(e);
            auto [P, s] = max_edges(v, cands, w, valid);
            if (s > max_s) {
                max_s = s;
                vc = t;
                Pc = P;
            }
        }
        if (vc.empty() || max_s < 0) break;
        A.insert(vc);
        if (!Pc.empty()) {
            C.insert(C.end(), Pc.begin(), Pc.end());
            std::sort(C.begin(), C.end());
            lC = oracle.evaluate(g, validate_ptg(v, C));
        }
        res.total_saving += max_s;
        res.decisions.push_back({res.iterations, vc, Pc, max_s});
        ++res.iterations;
        // re-profile every cached subset containing an edge into vc
        for (auto it = w_cache.begin(); it != w_cache.end();) {
            bool into = false;
            for (int e : it->first) into |= v.edges[size_t(e)].dst == vc;
            it = into ? w_cache.erase(it) : std::next(it);
        }
    }
    res.ptg = validate_ptg(v, C);
    res.oracle_calls = oracle.calls - calls0;
    return res;
}

}  // namespace vtc

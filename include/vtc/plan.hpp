// Virtualization rules, VTOG, points-to graphs and the byte accountant.
//
// Mirrors the reference's planner-facing API so a planned graph and its
// virtual-vs-materialize decision drop in unchanged:
//   gather_map / vt_rules        proj/include/vtelim/vt_rules.hpp:15-38
//   Vtog / build_vtog / PointsToGraph / validate_ptg / eliminated_nodes
//                                proj/include/vtelim/vtog.hpp:17-72
//   estimate / all_physical_ptg  proj/include/vtelim/cost_model.hpp:18-82
// Maps are vtc::VMap (div/mod form) so validate_ptg composes at full
// north-star sizes where the reference throws ComposeLimitError.
#pragma once

#include <map>
#include <set>
#include <string>
#include <vector>

#include "vtc/graph.hpp"
#include "vtc/vmap.hpp"

namespace vtc {

enum class VtDirection { OutputOverInput, InputOverOutput };
const char* to_string(VtDirection d);

struct VtRuleCandidate {
    std::string virtual_tensor;
    std::vector<std::string> base_tensors;
    VMap map;
    VtDirection direction = VtDirection::OutputOverInput;
    TypeClass static_class = TypeClass::TypeII;
    std::string eliminated_op;
};

// Defining element map F of a data-movement operator (vt_rules.cpp:161-223).
VMap gather_map(const OpNode& node, const std::string& output_id, const CompGraph& g);
// Legal virtualization candidates (vt_rules.cpp:242-383).
std::vector<VtRuleCandidate> vt_rules(const OpNode& node, const CompGraph& g);

struct VtEdge {
    int id = -1;
    std::string src, dst;
    VMap map;
    bool partial = false;
    VtDirection direction = VtDirection::OutputOverInput;
    TypeClass static_class = TypeClass::TypeII;
    std::string eliminated_op;
    int candidate = -1;
};

struct Vtog {
    const CompGraph* graph = nullptr;
    std::vector<std::string> nodes;
    std::vector<VtEdge> edges;
    std::map<std::string, std::set<std::pair<int, int>>> conflicts;
    std::vector<int> out_edges(const std::string& node) const;
    bool conflicting(int e1, int e2) const;
};

Vtog build_vtog(const CompGraph& g);

struct PointsToGraph {
    std::vector<int> selected;
    std::map<std::string, VMap> resolved;
    std::vector<std::string> roots;
    std::vector<std::string> eliminated_ops;
    bool is_virtual(const std::string& t) const;
    const VMap& map_of(const std::string& t) const;
};

PointsToGraph validate_ptg(const Vtog& v, const std::vector<int>& selected);
PointsToGraph all_physical_ptg(const CompGraph& g);
std::vector<std::string> eliminated_nodes(const CompGraph& g, const std::map<std::string, VMap>& resolved,
                                          const std::vector<std::string>& roots);

// Strategy: maximal data-movement elimination (write-side chains pulled back
// from ScatterND/Concat into producers, read-side gathers elsewhere), each
// selection validated incrementally.  Stand-in for Alg. 2 (absent from the
// reference snapshot: proj/CMakeLists.txt:21).
std::vector<int> plan_max_elimination(const Vtog& v);

// Strong materialising comparator (SURVEY.md §8 d): only the ScatterND in-place
// rule (i) (proj/src/vt_rules.cpp:346-349) -- a KV-cache update writes its slab
// into the cache instead of cloning it -- and every other data-movement
// operator materialised by a copy kernel.
std::vector<int> plan_inplace_updates(const Vtog& v);

// Byte accounting of the three-stage kernel model (cost_model.cpp:117-176).
struct OperandBytes {
    std::string tensor;
    int64_t bytes = 0;
    double bandwidth_factor = 1.0;  // set by estimate(g, ptg, MachineParams)
};
struct KernelBytes {
    std::string node;
    bool data_movement = false;
    std::vector<OperandBytes> reads, writes;
    double time = 0.0;  // set by estimate(g, ptg, MachineParams)
    int64_t total() const;
};
struct TrafficEstimate {
    std::vector<KernelBytes> kernels;
    int data_movement_kernels = 0;
    int compute_kernels = 0;
    double total_time = 0.0;  // set by estimate(g, ptg, MachineParams)
    int64_t total_bytes() const;
    int64_t data_movement_bytes() const;
};
TrafficEstimate estimate(const CompGraph& g, const PointsToGraph& ptg);

}  // namespace vtc

// Points-to-graph construction: the analytic cost model, saving oracles, the
// exhaustive enumeration and the global greedy algorithm (Alg. 2).
//
//   MachineParams / bandwidth_factor / estimate(params)   proj/include/vtelim/cost_model.hpp:18-62,
//                                                         proj/src/cost_model.cpp:14-176
//   SavingOracle / saving_oracle / executor_timed_oracle  proj/include/vtelim/cost_model.hpp:64-73,
//                                                         proj/src/cost_model.cpp:188-246
//   breakdown                                             proj/src/cost_model.cpp:248-261
//   enumerate_ptgs                                        proj/src/vtog.cpp:209-237
//   greedy_build / max_edges                              PAPER.md:570-608 (Alg. 2)
//                                                         (absent from the reference snapshot:
//                                                         proj/CMakeLists.txt:21 lists src/greedy.cpp)
//
// The timed oracle here measures strategies on the B200 itself (CUDA-graph
// replay of the planned step, CUDA events) instead of the reference's
// single-threaded CPU interpreter.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "vtc/plan.hpp"

namespace vtc {

struct MachineParams {
    double bandwidth = 1.0;                  // bytes per time unit
    int64_t coalesce_unit = 128;             // minimal memory transfer unit, bytes
    double kernel_launch_overhead = 5000.0;  // time units per kernel
    double noncoalesced_penalty = 8.0;       // effective-bandwidth divisor
    double partial_penalty = 1.0;            // > 1: conservative mode

    void validate() const;
    static MachineParams from_json(const std::string& text);
    std::string to_json() const;
    // Fitted on a B200 by scripts/calibrate.py (bandwidth in bytes/us, overhead in us).
    static MachineParams b200();
};

double bandwidth_factor(const VMap& m, int64_t elem_size, const MachineParams& params);

// estimate() with per-operand bandwidth factors and kernel times (cost_model.cpp:117-176).
TrafficEstimate estimate(const CompGraph& g, const PointsToGraph& ptg, const MachineParams& params);

struct LatencyBreakdown {
    double data_movement_time = 0.0, compute_time = 0.0;
    int data_movement_kernels = 0, compute_kernels = 0;
};
LatencyBreakdown breakdown(const TrafficEstimate& est);

class SavingOracle {
public:
    virtual ~SavingOracle() = default;
    // Time saved by the strategy relative to the all-physical baseline.
    virtual double evaluate(const CompGraph& g, const PointsToGraph& ptg) = 0;
    int64_t calls = 0;
};

std::unique_ptr<SavingOracle> saving_oracle(const MachineParams& params);
// Median (baseline - strategy) device time of `trials` CUDA-graph replays on
// the current GPU, in microseconds; trials >= 3 (cost_model.cpp:205-233).
std::unique_ptr<SavingOracle> device_timed_oracle(int trials, uint64_t seed = 1);

// All valid points-to graphs in the reference's DFS order (exclude before
// include), or the first `limit`.  Unbounded enumeration is refused beyond 20 edges.
std::vector<PointsToGraph> enumerate_ptgs(const Vtog& v, int64_t limit = -1);

struct GreedyDecision {
    int iteration = 0;
    std::string node;
    std::vector<int> edges;
    double saving = 0.0;
};

struct GreedyResult {
    PointsToGraph ptg;
    double total_saving = 0.0;
    int iterations = 0;
    int64_t oracle_calls = 0;
    std::vector<GreedyDecision> decisions;
};

// Alg. 2 MaxEdges: the conflict-free subset of `cands` (edges of one node into
// the anchor set) with the largest sum of w; exact over all subsets (<= 16
// candidates).  `feasible` rejects subsets that do not form a valid selection
// (incomplete multi-target candidates).  Returns the empty set and 0 when no
// subset beats it.
std::pair<std::vector<int>, double> max_edges(const Vtog& v, const std::vector<int>& cands,
                                              const std::function<double(const std::vector<int>&)>& w,
                                              const std::function<bool(const std::vector<int>&)>& feasible);

// Alg. 2.  w(P) = l(C u P) - l(C), profiled when P becomes a candidate and
// re-profiled for the edges into each newly anchored node.
// `accept` (optional) further restricts which selections are feasible (the
// executor's descriptor limits when the result is to be run).
GreedyResult greedy_build(const Vtog& v, SavingOracle& oracle,
                          const std::function<bool(const PointsToGraph&)>& accept = {});

}  // namespace vtc

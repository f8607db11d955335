// vtelim_b200.hpp -- the reference-side adapter a vtelim maintainer adds next
// to proj/src/executor.cpp to run a planned graph on a B200 through libvtc.so
// (this repo's C ABI, include/vtc.h).  Header-only; compiled and run against
// the unmodified reference by tests/cpp/test_boundary.cpp.
//
//   execute_b200(g, ptg, inputs)      drop-in for vtelim::execute
//                                     (proj/include/vtelim/executor.hpp:77-83)
//   B200Session                       the serving form: plan once, bind the
//                                     weights once, one vtc_run per step
#pragma once

#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "vtc.h"
#include "vtelim/errors.hpp"
#include "vtelim/executor.hpp"
#include "vtelim/graph_ir.hpp"
#include "vtelim/vtog.hpp"

namespace vtelim {

inline void vtc_check(int rc) {
    if (rc == VTC_OK) return;
    std::string msg = vtc_last_error();
    switch (rc) {  // the classes the CPU executor throws (proj/include/vtelim/errors.hpp:14-38)
        case VTC_ERR_MISSING_INPUT: throw MissingInputError(msg);
        case VTC_ERR_SHAPE_MISMATCH: throw ShapeMismatchError(msg);
        case VTC_ERR_WRITE_ALIASING: throw WriteAliasingError(msg);
        case VTC_ERR_COMPOSE_LIMIT: throw ComposeLimitError(msg);
        case VTC_ERR_CONFLICT: throw ConflictViolationError(msg);
        case VTC_ERR_INCOMPLETE_SELECTION: throw IncompleteSelectionError(msg);
        default: throw ExecutionError(msg);
    }
}

class B200Session {
public:
    // Plans `ptg` (its selected VTOG edge ids: the VTOG edge order is the
    // reference's) once.  Inputs named in `resident` (weights, KV caches) are
    // uploaded by bind_resident() and stay on the device across steps.
    B200Session(const CompGraph& g, const PointsToGraph& ptg) : g_(g) {
        vtc_check(vtc_graph_parse(serialize_graph(g).c_str(), &graph_));
        std::vector<int32_t> sel(ptg.selected.begin(), ptg.selected.end());
        vtc_check(vtc_plan_create(graph_, VTC_PLAN_SELECTED, sel.data(), int32_t(sel.size()), 0, &plan_));
    }
    ~B200Session() {
        if (plan_) vtc_plan_free(plan_);
        if (graph_) vtc_graph_free(graph_);
    }
    B200Session(const B200Session&) = delete;
    B200Session& operator=(const B200Session&) = delete;

    void bind_resident(const std::map<std::string, DenseArray>& resident) {
        for (const auto& [id, a] : resident) {
            vtc_check(vtc_plan_upload(plan_, id.c_str(), a.raw(), a.raw_bytes(), nullptr));
            resident_.insert(id);
        }
    }

    // One step: the per-step inputs (resident ones may be omitted) in, every
    // graph output back; synchronous, as vtelim::execute.
    std::map<std::string, DenseArray> step(const std::map<std::string, DenseArray>& inputs, void* stream = nullptr) {
        std::vector<const char*> in_ids, out_ids;
        std::vector<const void*> in_ptrs;
        std::vector<void*> out_ptrs;
        std::vector<int64_t> in_bytes, out_bytes;
        for (const auto& [id, a] : inputs) {
            if (resident_.count(id)) continue;
            in_ids.push_back(id.c_str());
            in_ptrs.push_back(a.raw());
            in_bytes.push_back(a.raw_bytes());
        }
        std::map<std::string, DenseArray> out;
        for (const auto& id : g_.graph_outputs())
            out.emplace(id, DenseArray::zeros(g_.tensor(id).dtype, g_.tensor(id).shape));
        for (auto& [id, a] : out) {
            out_ids.push_back(id.c_str());
            out_ptrs.push_back(a.raw());
            out_bytes.push_back(a.raw_bytes());
        }
        vtc_check(vtc_run(plan_, int32_t(in_ids.size()), in_ids.data(), in_ptrs.data(), in_bytes.data(),
                          int32_t(out_ids.size()), out_ids.data(), out_ptrs.data(), out_bytes.data(), stream));
        return out;
    }

    vtc_plan* plan() { return plan_; }

private:
    const CompGraph& g_;
    vtc_graph* graph_ = nullptr;
    vtc_plan* plan_ = nullptr;
    std::set<std::string> resident_;
};

// Drop-in for execute(g, ptg, inputs): same arguments, same result.
inline std::map<std::string, DenseArray> execute_b200(const CompGraph& g, const PointsToGraph& ptg,
                                                      const std::map<std::string, DenseArray>& inputs) {
    B200Session s(g, ptg);
    return s.step(inputs);
}

}  // namespace vtelim

// C-ABI test harness around the UNMODIFIED reference library (vtelim).
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against the
// reference headers in /root/reference/proj/include and linked with the
// reference sources compiled in place (never copied).  Output goes to
// oracle/_ref/libvtelim_ref.so, which travels to the GPU box.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu/reference arm load it, and only
// as the checker or the timed CPU baseline -- never as the product path.
//
// Every entry point mirrors one reference API:
//   parse_graph            proj/src/graph_ir.cpp:455-485
//   make_random_inputs     proj/src/executor.cpp:508-528
//   all_physical_ptg       proj/src/cost_model.cpp:178-186
//   build_vtog/validate_ptg proj/src/vtog.cpp:31-78, 123-207
//   execute_detailed       proj/src/executor.cpp:448-498
//   gather_map             proj/src/vt_rules.cpp:161-223
//   IndexMap::eval         proj/src/mapping.cpp:103-116
//   estimate               proj/src/cost_model.cpp:117-176 (default or given MachineParams)
//   saving_oracle          proj/src/cost_model.cpp:188-203
//   enumerate_ptgs         proj/src/vtog.cpp:209-237
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "vtelim/cost_model.hpp"
#include "vtelim/executor.hpp"
#include "vtelim/graph_ir.hpp"
#include "vtelim/mapping.hpp"
#include "vtelim/vt_rules.hpp"
#include "vtelim/vtog.hpp"

using namespace vtelim;

namespace {

thread_local std::string g_err;
thread_local std::string g_str;

struct Graph {
    CompGraph g;
    std::unique_ptr<Vtog> vtog;  // built lazily; holds a pointer to g
};

struct Tensors {
    std::map<std::string, DenseArray> arrays;
};

struct Plan {
    PointsToGraph ptg;
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

const char* dup(const std::string& s) {
    g_str = s;
    return g_str.c_str();
}

Vtog& vtog_of(Graph* gr) {
    if (!gr->vtog) gr->vtog = std::make_unique<Vtog>(build_vtog(gr->g));
    return *gr->vtog;
}

nlohmann::json ptg_json(const PointsToGraph& p) {
    nlohmann::json j;
    j["selected"] = p.selected;
    j["roots"] = p.roots;
    j["eliminated_ops"] = p.eliminated_ops;
    nlohmann::json res = nlohmann::json::object();
    for (const auto& [k, m] : p.resolved) res[k] = m.to_json();
    j["resolved"] = res;
    return j;
}

}  // namespace

extern "C" {

const char* vref_last_error() { return g_err.c_str(); }

void* vref_graph_parse(const char* json_text) {
    Graph* gr = nullptr;
    if (guard([&] {
            auto p = std::make_unique<Graph>();
            p->g = parse_graph(json_text);
            gr = p.release();
        }))
        return nullptr;
    return gr;
}

void vref_graph_free(void* g) { delete static_cast<Graph*>(g); }

const char* vref_graph_serialize(void* g) {
    return dup(serialize_graph(static_cast<Graph*>(g)->g));
}

// Edges of the VTOG as JSON: [{id, src, dst, candidate, eliminated_op, direction, partial}]
const char* vref_vtog_json(void* g) {
    std::string out;
    if (guard([&] {
            Vtog& v = vtog_of(static_cast<Graph*>(g));
            nlohmann::json arr = nlohmann::json::array();
            for (const auto& e : v.edges)
                arr.push_back({{"id", e.id},
                               {"src", e.src},
                               {"dst", e.dst},
                               {"candidate", e.candidate},
                               {"eliminated_op", e.eliminated_op},
                               {"direction", to_string(e.direction)},
                               {"type", to_string(e.static_class)},
                               {"partial", e.partial},
                               {"map", e.map.to_json()}});
            nlohmann::json conf = nlohmann::json::array();
            for (const auto& [src, pairs] : v.conflicts)
                for (const auto& pr : pairs) conf.push_back({pr.first, pr.second});
            out = nlohmann::json{{"edges", arr}, {"conflicts", conf}}.dump();
        }))
        return nullptr;
    return dup(out);
}

void* vref_ptg_all_physical(void* g) {
    Plan* p = nullptr;
    if (guard([&] {
            auto pl = std::make_unique<Plan>();
            pl->ptg = all_physical_ptg(static_cast<Graph*>(g)->g);
            p = pl.release();
        }))
        return nullptr;
    return p;
}

void* vref_ptg_validate(void* g, const int* selected, int n) {
    Plan* p = nullptr;
    if (guard([&] {
            auto pl = std::make_unique<Plan>();
            std::vector<int> sel(selected, selected + n);
            pl->ptg = validate_ptg(vtog_of(static_cast<Graph*>(g)), sel);
            p = pl.release();
        }))
        return nullptr;
    return p;
}

void vref_ptg_free(void* p) { delete static_cast<Plan*>(p); }

const char* vref_ptg_json(void* p) { return dup(ptg_json(static_cast<Plan*>(p)->ptg).dump()); }

const char* vref_estimate_json(void* g, void* p) {
    std::string out;
    if (guard([&] {
            MachineParams mp;
            auto est = estimate(static_cast<Graph*>(g)->g, static_cast<Plan*>(p)->ptg, mp);
            out = est.to_json().dump();
        }))
        return nullptr;
    return dup(out);
}

const char* vref_estimate_params_json(void* g, void* p, const char* params_json) {
    std::string out;
    if (guard([&] {
            MachineParams mp = MachineParams::from_json(nlohmann::json::parse(params_json));
            auto est = estimate(static_cast<Graph*>(g)->g, static_cast<Plan*>(p)->ptg, mp);
            out = est.to_json().dump();
        }))
        return nullptr;
    return dup(out);
}

// saving_oracle(params).evaluate(g, ptg)
int vref_saving(void* g, void* p, const char* params_json, double* out) {
    return guard([&] {
        auto o = saving_oracle(MachineParams::from_json(nlohmann::json::parse(params_json)));
        *out = o->evaluate(static_cast<Graph*>(g)->g, static_cast<Plan*>(p)->ptg);
    });
}

// enumerate_ptgs(vtog, limit): [{selected, roots, eliminated_ops}] in the reference's order.
const char* vref_enumerate_json(void* g, int64_t limit) {
    std::string out;
    if (guard([&] {
            nlohmann::json arr = nlohmann::json::array();
            for (const auto& p : enumerate_ptgs(vtog_of(static_cast<Graph*>(g)), limit))
                arr.push_back({{"selected", p.selected}, {"roots", p.roots}, {"eliminated_ops", p.eliminated_ops}});
            out = arr.dump();
        }))
        return nullptr;
    return dup(out);
}

const char* vref_gather_map_json(void* g, const char* node_id, const char* output_id) {
    std::string out;
    if (guard([&] {
            const CompGraph& cg = static_cast<Graph*>(g)->g;
            const OpNode* n = nullptr;
            for (const auto& nd : cg.nodes())
                if (nd.id == node_id) n = &nd;
            if (!n) throw SchemaError(std::string("no node ") + node_id);
            out = gather_map(*n, output_id, cg).to_json().dump();
        }))
        return nullptr;
    return dup(out);
}

// Evaluate an IndexMap (JSON) at every index of its virtual shape in row-major
// order.  targets[i] receives the position of the piece's target inside the
// sorted `targets()` list, offsets[i] the element offset.
int vref_map_eval_all(const char* map_json, int32_t* targets, int64_t* offsets, int64_t cap) {
    return guard([&] {
        IndexMap m = IndexMap::from_json(nlohmann::json::parse(map_json));
        auto tl = m.targets();
        const Index& shape = m.virtual_shape();
        int64_t vol = volume(shape);
        if (vol > cap) throw ExecutionError("eval buffer too small");
        Index idx(shape.size(), 0);
        for (int64_t f = 0; f < vol; ++f) {
            auto [t, off] = m.eval(idx);
            targets[f] = int32_t(std::lower_bound(tl.begin(), tl.end(), t) - tl.begin());
            offsets[f] = off;
            for (int i = int(shape.size()) - 1; i >= 0; --i) {
                if (++idx[i] < shape[i]) break;
                idx[i] = 0;
            }
        }
    });
}

// Composition through the reference algebra: outer over base (single base target name).
const char* vref_map_compose(const char* outer_json, const char* base_name, const char* base_json,
                             int piece_cap) {
    std::string out;
    if (guard([&] {
            IndexMap outer = IndexMap::from_json(nlohmann::json::parse(outer_json));
            IndexMap base = IndexMap::from_json(nlohmann::json::parse(base_json));
            std::string bn = base_name;
            IndexMap c = outer.compose(
                [&](const std::string& t) -> const IndexMap* { return t == bn ? &base : nullptr; },
                piece_cap);
            out = c.to_json().dump();
        }))
        return nullptr;
    return dup(out);
}

// Map queries used to pin the descriptor compiler's analyses.
const char* vref_map_analyze(const char* map_json, int64_t elem_size, int64_t coalesce) {
    std::string out;
    if (guard([&] {
            IndexMap m = IndexMap::from_json(nlohmann::json::parse(map_json));
            auto r = m.contiguity(elem_size, coalesce);
            out = nlohmann::json{{"injective", m.injective()},
                                 {"unique_elems", m.unique_elems()},
                                 {"is_total", m.is_total()},
                                 {"single_valued", m.single_valued()},
                                 {"min_contiguous_dim", r.min_contiguous_dim},
                                 {"contiguous_run_elems", r.contiguous_run_elems},
                                 {"class", to_string(r.cls)},
                                 {"type", to_string(r.type_class)}}
                      .dump();
        }))
        return nullptr;
    return dup(out);
}

// ---- tensors -------------------------------------------------------------

void* vref_inputs_random(void* g, uint64_t seed) {
    Tensors* t = nullptr;
    if (guard([&] {
            auto tt = std::make_unique<Tensors>();
            tt->arrays = make_random_inputs(static_cast<Graph*>(g)->g, seed);
            t = tt.release();
        }))
        return nullptr;
    return t;
}

void* vref_tensors_new() { return new Tensors(); }
void vref_tensors_free(void* t) { delete static_cast<Tensors*>(t); }

// dtype code: 0 f64, 1 f32, 2 i64 (VTT1 codes, proj/src/executor.cpp:534)
int vref_tensor_set(void* t, const char* id, int dtype_code, const int64_t* shape, int ndim,
                    const void* data) {
    return guard([&] {
        DType dt = dtype_code == 0 ? DType::F64 : dtype_code == 1 ? DType::F32 : DType::I64;
        Index s(shape, shape + ndim);
        DenseArray a = DenseArray::zeros(dt, s);
        std::memcpy(a.raw(), data, size_t(a.raw_bytes()));
        static_cast<Tensors*>(t)->arrays[id] = std::move(a);
    });
}

int64_t vref_tensor_bytes(void* t, const char* id) {
    auto& m = static_cast<Tensors*>(t)->arrays;
    auto it = m.find(id);
    return it == m.end() ? -1 : it->second.raw_bytes();
}

int vref_tensor_get(void* t, const char* id, void* dst, int64_t cap) {
    return guard([&] {
        auto& m = static_cast<Tensors*>(t)->arrays;
        auto it = m.find(id);
        if (it == m.end()) throw ExecutionError(std::string("no tensor ") + id);
        if (it->second.raw_bytes() > cap) throw ExecutionError("buffer too small");
        std::memcpy(dst, it->second.raw(), size_t(it->second.raw_bytes()));
    });
}

uint64_t vref_tensor_digest(void* t, const char* id) {
    auto& m = static_cast<Tensors*>(t)->arrays;
    auto it = m.find(id);
    return it == m.end() ? 0 : array_digest(it->second);
}

// execute(g, ptg, inputs) -> outputs (graph outputs) plus every physical root
// written (mutated caches) under "root:<id>".  Wall time in ns -> *ns.
void* vref_execute(void* g, void* p, void* inputs, int with_roots, double* ns) {
    Tensors* out = nullptr;
    if (guard([&] {
            const CompGraph& cg = static_cast<Graph*>(g)->g;
            const PointsToGraph& ptg = static_cast<Plan*>(p)->ptg;
            auto t0 = std::chrono::steady_clock::now();
            ExecutionResult res = execute_detailed(cg, ptg, static_cast<Tensors*>(inputs)->arrays);
            auto o = std::make_unique<Tensors>();
            for (const auto& id : cg.graph_outputs()) o->arrays.emplace(id, res.materialize(id));
            auto t1 = std::chrono::steady_clock::now();
            if (ns) *ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
            if (with_roots)
                for (const auto& [id, arr] : res.store.buffers) o->arrays.emplace("root:" + id, arr);
            std::string skipped;
            for (const auto& s : res.skipped_ops) skipped += s + "\n";
            g_str = skipped;
            out = o.release();
        }))
        return nullptr;
    return out;
}

const char* vref_last_skipped() { return g_str.c_str(); }

}  // extern "C"

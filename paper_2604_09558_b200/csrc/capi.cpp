// extern "C" boundary (include/vtc.h).  Exceptions are caught here and
// turned into the status codes of the reference error classes.
#include <cstring>
#include <memory>
#include <string>

#include <cuda_runtime.h>

#include "json.hpp"
#include "kernels.hpp"
#include "lower.hpp"
#include "vtc.h"
#include "comm.hpp"
#include "vtc/exec.hpp"
#include "vtc/planner.hpp"

struct vtc_graph {
    vtc::CompGraph g;
    std::unique_ptr<vtc::Vtog> vtog;
};

struct vtc_comm {
    std::unique_ptr<vtc::Comm> c;
};

struct vtc_plan {
    vtc_graph* graph;
    std::unique_ptr<vtc::Executor> exec;
    uint32_t flags = 0;
    int mode = 0;
};

namespace {

thread_local std::string g_err;
thread_local std::string g_out;

template <class F>
int guard(F&& f) {
    try {
        f();
        return VTC_OK;
    } catch (const vtc::Error& e) {
        g_err = e.what();
        return e.code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return VTC_ERR_GENERIC;
    }
}

vtc::Vtog& vtog_of(vtc_graph* g) {
    if (!g->vtog) g->vtog = std::make_unique<vtc::Vtog>(vtc::build_vtog(g->g));
    return *g->vtog;
}

vtc::json::Value str(const std::string& s) { return vtc::json::Value::string(s); }
vtc::json::Value strs(const std::vector<std::string>& v) {
    auto a = vtc::json::Value::array();
    for (const auto& s : v) a.push(str(s));
    return a;
}

vtc::json::Value estimate_json(const vtc::TrafficEstimate& e) {
    using vtc::json::Value;
    Value j = Value::object();
    j.set("total_bytes", Value::integer(e.total_bytes()));
    j.set("data_movement_bytes", Value::integer(e.data_movement_bytes()));
    j.set("data_movement_kernels", Value::integer(e.data_movement_kernels));
    j.set("compute_kernels", Value::integer(e.compute_kernels));
    Value ks = Value::array();
    for (const auto& k : e.kernels) {
        Value kj = Value::object();
        kj.set("node", str(k.node));
        kj.set("data_movement", Value::boolean(k.data_movement));
        int64_t rb = 0, wb = 0;
        for (const auto& r : k.reads) rb += r.bytes;
        for (const auto& w : k.writes) wb += w.bytes;
        kj.set("read_bytes", Value::integer(rb));
        kj.set("write_bytes", Value::integer(wb));
        ks.push(kj);
    }
    j.set("kernels", ks);
    return j;
}

vtc::MachineParams params_of(const char* text) {
    if (!text || !*text) return vtc::MachineParams{};
    if (std::string(text) == "b200") return vtc::MachineParams::b200();
    return vtc::MachineParams::from_json(text);
}

vtc::json::Value ints_of(const std::vector<int>& v) {
    auto a = vtc::json::Value::array();
    for (int e : v) a.push(vtc::json::Value::integer(e));
    return a;
}

vtc::json::Value timed_estimate_json(const vtc::TrafficEstimate& e) {
    using vtc::json::Value;
    Value j = Value::object();
    j.set("total_time", Value::number(e.total_time));
    j.set("total_bytes", Value::integer(e.total_bytes()));
    j.set("data_movement_kernels", Value::integer(e.data_movement_kernels));
    j.set("compute_kernels", Value::integer(e.compute_kernels));
    Value ks = Value::array();
    for (const auto& k : e.kernels) {
        Value kj = Value::object();
        kj.set("node", str(k.node));
        kj.set("data_movement", Value::boolean(k.data_movement));
        kj.set("time", Value::number(k.time));
        for (int side = 0; side < 2; ++side) {
            Value ops = Value::array();
            for (const auto& o : side ? k.writes : k.reads) {
                Value oj = Value::object();
                oj.set("tensor", str(o.tensor));
                oj.set("bytes", Value::integer(o.bytes));
                oj.set("factor", Value::number(o.bandwidth_factor));
                ops.push(oj);
            }
            kj.set(side ? "writes" : "reads", ops);
        }
        ks.push(kj);
    }
    j.set("kernels", ks);
    vtc::LatencyBreakdown b = vtc::breakdown(e);
    Value bj = Value::object();
    bj.set("data_movement_time", Value::number(b.data_movement_time));
    bj.set("compute_time", Value::number(b.compute_time));
    bj.set("data_movement_kernels", Value::integer(b.data_movement_kernels));
    bj.set("compute_kernels", Value::integer(b.compute_kernels));
    j.set("breakdown", bj);
    return j;
}

// Can the executor run this strategy?  (every resolved map fits the device descriptor)
bool executable(const vtc::PointsToGraph& p) {
    try {
        for (const auto& [id, m] : p.resolved) vtc::lower_map(m, [](const std::string&) { return vtc::TargetInfo{0, 0}; });
    } catch (const vtc::Error&) {
        return false;
    }
    return true;
}

}  // namespace

extern "C" {

const char* vtc_last_error(void) { return g_err.c_str(); }
const char* vtc_version(void) { return "vtc-b200 0.1 (sm_100a)"; }

int vtc_graph_parse(const char* json_text, vtc_graph** out) {
    return guard([&] {
        auto g = std::make_unique<vtc_graph>();
        g->g = vtc::parse_graph(json_text);
        *out = g.release();
    });
}

void vtc_graph_free(vtc_graph* g) { delete g; }

int vtc_graph_serialize(vtc_graph* g, const char** json_out) {
    return guard([&] {
        g_out = vtc::serialize_graph(g->g);
        *json_out = g_out.c_str();
    });
}

int vtc_graph_vtog(vtc_graph* g, const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        vtc::Vtog& v = vtog_of(g);
        Value edges = Value::array();
        for (const auto& e : v.edges) {
            Value ej = Value::object();
            ej.set("id", Value::integer(e.id));
            ej.set("src", str(e.src));
            ej.set("dst", str(e.dst));
            ej.set("candidate", Value::integer(e.candidate));
            ej.set("eliminated_op", str(e.eliminated_op));
            ej.set("direction", str(vtc::to_string(e.direction)));
            ej.set("type", str(vtc::to_string(e.static_class)));
            ej.set("partial", Value::boolean(e.partial));
            ej.set("map", str(e.map.to_string()));
            edges.push(ej);
        }
        Value conf = Value::array();
        for (const auto& [src, pairs] : v.conflicts)
            for (const auto& pr : pairs) {
                Value c = Value::array();
                c.push(Value::integer(pr.first));
                c.push(Value::integer(pr.second));
                conf.push(c);
            }
        Value j = Value::object();
        j.set("edges", edges);
        j.set("conflicts", conf);
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_graph_estimate(vtc_graph* g, const int32_t* selected, int32_t n_selected, const char* params_json,
                       const char** json_out) {
    return guard([&] {
        vtc::MachineParams mp = params_of(params_json);
        vtc::PointsToGraph ptg = (!selected && n_selected < 0)
                                     ? vtc::all_physical_ptg(g->g)
                                     : vtc::validate_ptg(vtog_of(g), std::vector<int>(selected, selected + std::max(0, n_selected)));
        g_out = vtc::json::dump(timed_estimate_json(vtc::estimate(g->g, ptg, mp)));
        *json_out = g_out.c_str();
    });
}

int vtc_graph_enumerate(vtc_graph* g, int64_t limit, const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        Value arr = Value::array();
        for (const auto& p : vtc::enumerate_ptgs(vtog_of(g), limit)) {
            Value pj = Value::object();
            pj.set("selected", ints_of(p.selected));
            pj.set("roots", strs(p.roots));
            pj.set("eliminated_ops", strs(p.eliminated_ops));
            arr.push(pj);
        }
        Value j = Value::object();
        j.set("ptgs", arr);
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_graph_greedy(vtc_graph* g, const char* config_json, const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        Value cfg = (config_json && *config_json) ? vtc::json::parse(config_json) : Value::object();
        std::string oracle_kind = cfg.contains("oracle") ? cfg.at("oracle").as_string() : "analytic";
        std::string params_text;
        if (cfg.contains("params")) {
            const Value& pv = cfg.at("params");
            params_text = pv.is_string() ? pv.as_string() : vtc::json::dump(pv);
        }
        std::unique_ptr<vtc::SavingOracle> oracle;
        if (oracle_kind == "analytic") {
            oracle = vtc::saving_oracle(params_of(params_text.c_str()));
        } else if (oracle_kind == "device") {
            int trials = cfg.contains("trials") ? int(cfg.at("trials").as_int()) : 5;
            oracle = vtc::device_timed_oracle(trials);
        } else {
            throw vtc::SchemaError("unknown oracle " + oracle_kind);
        }
        bool exe = oracle_kind == "device" || (cfg.contains("executable") && cfg.at("executable").as_bool());
        vtc::Vtog& v = vtog_of(g);
        vtc::GreedyResult r = vtc::greedy_build(v, *oracle, exe ? std::function<bool(const vtc::PointsToGraph&)>(executable)
                                                                : std::function<bool(const vtc::PointsToGraph&)>());
        Value j = Value::object();
        j.set("selected", ints_of(r.ptg.selected));
        j.set("roots", strs(r.ptg.roots));
        j.set("eliminated_ops", strs(r.ptg.eliminated_ops));
        j.set("total_saving", Value::number(r.total_saving));
        j.set("final_saving", Value::number(oracle->evaluate(g->g, r.ptg)));
        j.set("iterations", Value::integer(r.iterations));
        j.set("oracle_calls", Value::integer(r.oracle_calls));
        Value ds = Value::array();
        for (const auto& d : r.decisions) {
            Value dj = Value::object();
            dj.set("iteration", Value::integer(d.iteration));
            dj.set("node", str(d.node));
            dj.set("edges", ints_of(d.edges));
            dj.set("saving", Value::number(d.saving));
            ds.push(dj);
        }
        j.set("decisions", ds);
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_plan_create(vtc_graph* g, int mode, const int32_t* selected, int32_t n_selected, uint32_t flags,
                    vtc_plan** out) {
    return guard([&] {
        vtc::PointsToGraph ptg;
        if (mode == VTC_PLAN_MATERIALIZE) {
            ptg = vtc::all_physical_ptg(g->g);
        } else if (mode == VTC_PLAN_SELECTED) {
            std::vector<int> sel(selected, selected + n_selected);
            ptg = vtc::validate_ptg(vtog_of(g), sel);
        } else if (mode == VTC_PLAN_MAX_ELIMINATION) {
            ptg = vtc::validate_ptg(vtog_of(g), vtc::plan_max_elimination(vtog_of(g)));
        } else if (mode == VTC_PLAN_INPLACE_UPDATES) {
            ptg = vtc::validate_ptg(vtog_of(g), vtc::plan_inplace_updates(vtog_of(g)));
        } else if (mode == VTC_PLAN_GREEDY) {
            auto oracle = vtc::saving_oracle(vtc::MachineParams::b200());
            ptg = vtc::greedy_build(vtog_of(g), *oracle, executable).ptg;
        } else {
            throw vtc::SchemaError("unknown plan mode");
        }
        vtc::ExecOptions opt;
        opt.exact_fp = !(flags & VTC_FLAG_FAST_FP);
        opt.use_gemv = !(flags & VTC_FLAG_NO_GEMV);
        opt.fuse = !(flags & VTC_FLAG_NO_FUSE);
        opt.gemv_stream = (flags & VTC_FLAG_GEMV_LDG) == 0;
        opt.use_tc = (flags & VTC_FLAG_NO_TC) == 0;
        opt.dynamic_pos = (flags & VTC_FLAG_DYNAMIC_POS) != 0;
        auto p = std::make_unique<vtc_plan>();
        p->graph = g;
        p->flags = flags;
        p->mode = mode;
        p->exec = std::make_unique<vtc::Executor>(g->g, std::move(ptg), opt);
        *out = p.release();
    });
}

void vtc_plan_free(vtc_plan* p) { delete p; }

int vtc_plan_info(vtc_plan* p, int dry, const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        const auto& ptg = p->exec->ptg();
        if (dry) p->exec->prepare(true);
        Value j = Value::object();
        j.set("mode", Value::integer(p->mode));
        j.set("roots", strs(ptg.roots));
        j.set("eliminated_ops", strs(ptg.eliminated_ops));
        Value sel = Value::array();
        for (int e : ptg.selected) sel.push(Value::integer(e));
        j.set("selected", sel);
        Value maps = Value::object();
        for (const auto& [id, m] : ptg.resolved)
            if (!m.is_identity_of(id)) maps.set(id, str(m.to_string()));
        j.set("virtual_maps", maps);
        Value ls = Value::array();
        int dm = 0;
        for (const auto& l : p->exec->launches()) {
            Value lj = Value::object();
            lj.set("node", str(l.node));
            lj.set("kernel", str(l.kernel));
            lj.set("bytes", Value::integer(l.bytes));
            ls.push(lj);
            if (l.kernel == "gather_copy") ++dm;
        }
        j.set("launches", ls);
        j.set("kernel_launches", Value::integer(p->exec->num_kernel_launches()));
        j.set("data_movement_launches", Value::integer(dm));
        auto est = vtc::estimate(p->exec->graph(), ptg);
        auto phys = vtc::estimate(p->exec->graph(), vtc::all_physical_ptg(p->exec->graph()));
        j.set("estimate", estimate_json(est));
        j.set("estimate_all_physical", estimate_json(phys));
        j.set("bytes_eliminated", Value::integer(phys.total_bytes() - est.total_bytes()));
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_plan_bind_root(vtc_plan* p, const char* tensor, void* dev_ptr) {
    return guard([&] { p->exec->bind_root(tensor, dev_ptr); });
}

int vtc_plan_root_ptr(vtc_plan* p, const char* tensor, void** dev_ptr) {
    return guard([&] { *dev_ptr = p->exec->root_ptr(tensor); });
}

int vtc_plan_upload(vtc_plan* p, const char* tensor, const void* host, int64_t bytes, void* stream) {
    return guard([&] { p->exec->upload(tensor, host, bytes, stream); });
}

int vtc_plan_download(vtc_plan* p, const char* tensor, void* host, int64_t bytes, void* stream) {
    return guard([&] { p->exec->download(tensor, host, bytes, stream); });
}

int vtc_run(vtc_plan* p, int32_t n_in, const char* const* in_ids, const void* const* in_host, const int64_t* in_bytes,
            int32_t n_out, const char* const* out_ids, void* const* out_host, const int64_t* out_bytes, void* stream) {
    return guard([&] {
        std::vector<vtc::Executor::HostIn> ins;
        std::vector<vtc::Executor::HostOut> outs;
        for (int32_t i = 0; i < n_in; ++i) ins.push_back({in_ids[i], in_host[i], in_bytes[i]});
        for (int32_t i = 0; i < n_out; ++i) outs.push_back({out_ids[i], out_host[i], out_bytes[i]});
        p->exec->run_host(ins, outs, stream);
    });
}

int vtc_comm_unique_id(void* out, int32_t bytes) {
    return guard([&] {
        if (bytes < 128) throw vtc::ExecutionError("vtc_comm_unique_id: buffer must hold 128 bytes");
        vtc::comm_unique_id(out);
    });
}

int vtc_comm_init(const void* unique_id, int32_t bytes, int32_t nranks, int32_t rank, vtc_comm** out) {
    return guard([&] {
        if (bytes < 128) throw vtc::ExecutionError("vtc_comm_init: unique id must be 128 bytes");
        auto* c = new vtc_comm;
        try {
            c->c = std::make_unique<vtc::Comm>(unique_id, nranks, rank);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int vtc_comm_init_host(vtc_allreduce_fn fn, void* user, int32_t nranks, int32_t rank, vtc_comm** out) {
    return guard([&] {
        auto* c = new vtc_comm;
        try {
            c->c = std::make_unique<vtc::Comm>(reinterpret_cast<vtc::HostAllReduceFn>(fn), user, nranks, rank);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void vtc_comm_free(vtc_comm* c) { delete c; }

int vtc_plan_set_comm(vtc_plan* p, vtc_comm* c) {
    return guard([&] { p->exec->set_comm(c ? c->c.get() : nullptr); });
}

int vtc_plan_set_position(vtc_plan* p, int64_t pos, void* stream) {
    return guard([&] { p->exec->set_position(pos, stream); });
}

int vtc_plan_prepare(vtc_plan* p) {
    return guard([&] { p->exec->prepare(false); });
}

int vtc_execute(vtc_plan* p, void* stream) {
    return guard([&] { p->exec->run(stream); });
}

int vtc_execute_graph(vtc_plan* p, void* stream) {
    return guard([&] { p->exec->run_graph(stream); });
}

int vtc_plan_num_launches(vtc_plan* p) { return p->exec->num_kernel_launches(); }

int vtc_execute_timed(vtc_plan* p, void* stream, float* ms, int32_t n) {
    return guard([&] { p->exec->run_timed(stream, ms, n); });
}

int vtc_plan_trace(vtc_plan* p, uint64_t* out, int32_t n) {
    int count = 0;
    int st = guard([&] { count = p->exec->read_trace(reinterpret_cast<unsigned long long*>(out), n); });
    return st == VTC_OK ? count : -st;
}

int vtc_map_eval(vtc_plan* p, const char* tensor, int lowered, int32_t* targets, int64_t* offsets, int64_t cap) {
    return guard([&] {
        const vtc::VMap& m = p->exec->ptg().map_of(tensor);
        auto tl = m.targets();
        int64_t vol = m.domain_volume();
        if (vol > cap) throw vtc::ExecutionError("eval buffer too small");
        vtc_map d{};
        if (lowered)
            d = vtc::lower_map(m, [&](const std::string& t) {
                return vtc::TargetInfo{int(std::lower_bound(tl.begin(), tl.end(), t) - tl.begin()), 0};
            });
        vtc::Index idx(m.shape().size(), 0);
        for (int64_t f = 0; f < vol; ++f) {
            if (lowered) {
                int pi = -1;
                offsets[f] = vtc::desc_eval(d, idx.data(), &pi);
                if (pi < 0) throw vtc::OutOfBoundsError("descriptor does not cover index");
                targets[f] = d.piece[pi].target;
            } else {
                auto [t, off] = m.eval(idx);
                targets[f] = int32_t(std::lower_bound(tl.begin(), tl.end(), t) - tl.begin());
                offsets[f] = off;
            }
            for (int i = int(idx.size()) - 1; i >= 0; --i) {
                if (++idx[size_t(i)] < m.shape()[size_t(i)]) break;
                idx[size_t(i)] = 0;
            }
        }
    });
}

int vtc_plan_map_json(vtc_plan* p, const char* tensor, const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        const vtc::VMap& m = p->exec->ptg().map_of(tensor);
        Value j = Value::object();
        j.set("shape", Value::ints(m.shape()));
        j.set("targets", strs(m.targets()));
        j.set("pieces", Value::integer(int64_t(m.pieces().size())));
        j.set("text", str(m.to_string()));
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_plan_map_analyze(vtc_plan* p, const char* tensor, int64_t elem_size, int64_t coalesce_unit,
                         const char** json_out) {
    return guard([&] {
        using vtc::json::Value;
        const vtc::VMap& m = p->exec->ptg().map_of(tensor);
        vtc::ContiguityReport r = m.contiguity(elem_size, coalesce_unit);
        Value j = Value::object();
        j.set("injective", Value::boolean(m.injective()));
        j.set("unique_elems", Value::integer(m.unique_elems()));
        j.set("is_total", Value::boolean(m.is_total()));
        j.set("min_contiguous_dim", Value::integer(r.min_contiguous_dim));
        j.set("contiguous_run_elems", Value::integer(r.contiguous_run_elems));
        j.set("class", str(vtc::to_string(r.cls)));
        j.set("type", str(vtc::to_string(r.type_class)));
        g_out = vtc::json::dump(j);
        *json_out = g_out.c_str();
    });
}

int vtc_launch_gather_copy(const vtc_map* dst, const vtc_map* src, int32_t elem_bytes, void* stream) {
    return guard([&] {
        vtc::EwParams p;
        std::memset(&p, 0, sizeof(p));
        p.rank = dst->rank;
        int64_t n = 1;
        for (int i = 0; i < dst->rank; ++i) {
            p.shape[i] = dst->shape[i];
            n *= dst->shape[i];
        }
        p.vec = 1;
        p.copy_only = 1;
        p.esize = elem_bytes;
        p.dt = elem_bytes == 8 ? vtc::KDType::I64 : elem_bytes == 4 ? vtc::KDType::F32 : vtc::KDType::BF16;
        p.nvec = n;
        p.nin = 1;
        p.out.m = *dst;
        p.in[0].m = *src;
        vtc::EwParams* dp = nullptr;
        cudaError_t e = cudaMalloc(&dp, sizeof(p));
        if (e == cudaSuccess) e = cudaMemcpy(dp, &p, sizeof(p), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) {
            vtc::launch_eltwise(p, dp, static_cast<cudaStream_t>(stream));
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        cudaFree(dp);
        if (e != cudaSuccess) throw vtc::CudaError(cudaGetErrorString(e));
    });
}

}  // extern "C"

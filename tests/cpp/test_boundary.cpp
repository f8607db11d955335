// The drop-in check: the UNMODIFIED reference
// (oracle/_ref objects, /root/reference/proj/include) and this repo's C ABI in
// one program.  For each graph the reference plans the points-to graph
// (validate_ptg over the VTOG edges vtc's planner picked, and all_physical_ptg),
// runs vtelim::execute on the CPU, and runs integration/vtelim_b200.hpp's
// execute_b200 / B200Session on the GPU; outputs must be arrays_bit_equal
// (proj/include/vtelim/executor.hpp:32).
// Usage: test_boundary <graph.json>...   (prints one line per graph, exit 0 = all equal)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "../../integration/vtelim_b200.hpp"
#include "vtelim/cost_model.hpp"

using namespace vtelim;

static std::vector<int> greedy_selection(const std::string& json) {
    vtc_graph* vg = nullptr;
    vtc_check(vtc_graph_parse(json.c_str(), &vg));
    const char* out = nullptr;
    vtc_check(vtc_graph_greedy(vg, "{\"oracle\":\"analytic\",\"executable\":true}", &out));
    std::string s = out;
    vtc_graph_free(vg);
    // "selected":[a,b,...]
    std::vector<int> sel;
    size_t p = s.find("\"selected\":[");
    if (p == std::string::npos) return sel;
    p += 12;
    while (s[p] != ']') {
        size_t q = p;
        while (s[q] != ',' && s[q] != ']') ++q;
        sel.push_back(std::stoi(s.substr(p, q - p)));
        p = s[q] == ',' ? q + 1 : q;
    }
    return sel;
}

int main(int argc, char** argv) {
    int bad = 0;
    for (int i = 1; i < argc; ++i) {
        std::ifstream f(argv[i]);
        std::stringstream ss;
        ss << f.rdbuf();
        CompGraph g = parse_graph(ss.str());
        Vtog v = build_vtog(g);
        auto inputs = make_random_inputs(g, 1);
        std::vector<int> sel = greedy_selection(ss.str());
        PointsToGraph planned = validate_ptg(v, sel);
        PointsToGraph phys = all_physical_ptg(g);
        auto want = execute(g, phys, inputs);
        auto want_v = execute(g, planned, inputs);
        auto got_p = execute_b200(g, phys, inputs);
        auto got_v = execute_b200(g, planned, inputs);
        // serving form: weights (every input but the first) resident, two steps
        B200Session sess(g, planned);
        std::map<std::string, DenseArray> resident, step_in;
        bool first = true;
        for (const auto& [id, a] : inputs) {
            (first ? step_in : resident).emplace(id, a);
            first = false;
        }
        sess.bind_resident(resident);
        auto got_s1 = sess.step(step_in);
        auto got_s2 = sess.step(step_in);
        // SiLU evaluates exp with the device libm (the reference: the host's), so
        // graphs with SiLU are held to a last-ulp bound instead of bit equality
        bool silu = false;
        for (const auto& n : g.nodes()) silu |= n.kind == OpKind::SiLU;
        auto rel = [](const DenseArray& x, const DenseArray& y) {
            double num = 0, den = 0;
            for (int64_t k = 0; k < x.elems(); ++k) {
                double a = x.dtype == DType::F64 ? x.f64[size_t(k)] : x.dtype == DType::F32 ? x.f32[size_t(k)] : double(x.i64[size_t(k)]);
                double b = y.dtype == DType::F64 ? y.f64[size_t(k)] : y.dtype == DType::F32 ? y.f32[size_t(k)] : double(y.i64[size_t(k)]);
                num = std::max(num, std::fabs(a - b));
                den = std::max(den, std::fabs(a));
            }
            return den > 0 ? num / den : num;
        };
        if (silu) {
            double worst = 0;
            for (const auto& [id, a] : want)
                for (const auto* o : {&want_v, &got_p, &got_v, &got_s1, &got_s2}) worst = std::max(worst, rel(a, o->at(id)));
            bool ok = worst <= 1e-14;
            printf("%s: %zu selected edges, %zu eliminated ops, outputs %s (max rel err %.3g, SiLU)\n", argv[i], sel.size(),
                   planned.eliminated_ops.size(), ok ? "within-1e-14" : "DIFFER", worst);
            bad += !ok;
            continue;
        }
        int ok = 1;
        for (const auto& [id, a] : want) {
            ok &= arrays_bit_equal(a, want_v.at(id));
            ok &= arrays_bit_equal(a, got_p.at(id));
            ok &= arrays_bit_equal(a, got_v.at(id));
            ok &= arrays_bit_equal(a, got_s1.at(id));
            ok &= arrays_bit_equal(a, got_s2.at(id));
            if (!ok)
                printf("  %s: first difference at %lld (planned %lld, session %lld)\n", id.c_str(),
                       (long long)first_difference(a, got_p.at(id)), (long long)first_difference(a, got_v.at(id)),
                       (long long)first_difference(a, got_s1.at(id)));
        }
        printf("%s: %zu selected edges, %zu eliminated ops, outputs %s, digest %016llx\n", argv[i], sel.size(),
               planned.eliminated_ops.size(), ok ? "bit-identical" : "DIFFER",
               (unsigned long long)array_digest(want.begin()->second));
        bad += !ok;
    }
    return bad ? 1 : 0;
}

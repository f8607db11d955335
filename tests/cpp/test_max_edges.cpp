// Alg. 2 MaxEdges on the Fig. 7 conflict structure, through
// the C++ API of libvtc.so.  Prints "chosen=<paper labels> s=<sum>" per case.
// Usage: test_max_edges <fig7 graph json file> w1 w2 w3
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>

#include "vtc/planner.hpp"

int main(int argc, char** argv) {
    if (argc != 5) return 2;
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    vtc::CompGraph g = vtc::parse_graph(ss.str());
    vtc::Vtog v = vtc::build_vtog(g);
    // paper labels: 1 = c over a, 2 = c over b, 3 = c over d
    std::map<int, int> label;
    std::vector<int> cands;
    for (const auto& e : v.edges) {
        if (e.src != "c") continue;
        int l = e.dst == "a" ? 1 : e.dst == "b" ? 2 : e.dst == "d" ? 3 : 0;
        if (!l) continue;
        label[e.id] = l;
        cands.push_back(e.id);
    }
    double w[4] = {0, atof(argv[2]), atof(argv[3]), atof(argv[4])};
    auto weight = [&](const std::vector<int>& P) {
        double s = 0;
        for (int e : P) s += w[label[e]];
        return s;
    };
    auto feasible = [](const std::vector<int>&) { return true; };  // conflicts only
    auto [P, s] = vtc::max_edges(v, cands, weight, feasible);
    std::vector<int> ls;
    for (int e : P) ls.push_back(label[e]);
    std::sort(ls.begin(), ls.end());
    printf("chosen=");
    for (size_t i = 0; i < ls.size(); ++i) printf(i ? ",%d" : "%d", ls[i]);
    printf(" s=%g\n", s);
    return 0;
}

// Div/mod index-map algebra (see include/vtc/vmap.hpp for the design).
//
// Reference semantics reproduced here (proj/src/mapping.cpp):
//   AffinePiece::eval / IndexMap::eval / find_piece   :53-57, 103-116
//   is_total / has_overlap                            :118-150
//   injective (lattice test + exhaustive fallback)    :172-238
//   unique_elems                                      :240-275
//   contiguity (Paper §4.3 classification)            :277-328
//   compose (F_outer o F_base, unflatten into base)   :330-461
// The composition differs in *how* boxes are handled: the reference bisects
// until every box is carry-free; here div/mod atoms absorb the carries, and
// boxes are split only at base-piece boundaries.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <functional>
#include <cassert>
#include <map>
#include <mutex>
#include <numeric>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

#include "vtc/vmap.hpp"

namespace vtc {

int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

int64_t floormod(int64_t a, int64_t b) {
    int64_t r = a % b;
    if (r != 0 && ((r < 0) != (b < 0))) r += b;
    return r;
}

namespace {

std::mutex g_intern_mu;
std::unordered_map<std::string, AtomP>& intern_table() {
    static std::unordered_map<std::string, AtomP> t;
    return t;
}

AtomP intern(Atom&& a) {
    std::lock_guard<std::mutex> lk(g_intern_mu);
    auto& tab = intern_table();
    auto it = tab.find(a.key);
    if (it != tab.end()) return it->second;
    auto p = std::make_shared<const Atom>(std::move(a));
    tab.emplace(p->key, p);
    return p;
}

AtomP make_axis_atom(int ax, int64_t lo, int64_t hi) {
    Atom a;
    a.kind = AtomKind::Axis;
    a.axis = ax;
    a.lo = lo;
    a.hi = hi;
    a.axes_mask = uint64_t(1) << ax;
    a.key = "i" + std::to_string(ax) + "[" + std::to_string(lo) + ":" + std::to_string(hi) + "]";
    return intern(std::move(a));
}

AtomP make_op_atom(AtomKind kind, const Lin& arg, int64_t k) {
    Atom a;
    a.kind = kind;
    a.arg = arg;
    a.k = k;
    int64_t lo = arg.lo(), hi = arg.hi();
    if (kind == AtomKind::Div) {
        a.lo = floordiv(lo, k);
        a.hi = floordiv(hi, k);
        a.key = "(" + arg.key() + ")/" + std::to_string(k);
    } else {
        if (floordiv(lo, k) == floordiv(hi, k)) {
            a.lo = floormod(lo, k);
            a.hi = floormod(hi, k);
        } else {
            a.lo = 0;
            a.hi = k - 1;
        }
        a.key = "(" + arg.key() + ")%" + std::to_string(k);
    }
    a.axes_mask = axes_mask(arg);
    return intern(std::move(a));
}

void add_term(Lin& l, int64_t c, const AtomP& a) {
    if (c == 0) return;
    // keep sorted by key
    auto it = std::lower_bound(l.t.begin(), l.t.end(), a->key,
                               [](const Term& t, const std::string& k) { return t.a->key < k; });
    if (it != l.t.end() && it->a == a) {
        it->c += c;
        if (it->c == 0) l.t.erase(it);
        return;
    }
    l.t.insert(it, Term{c, a});
}

Lin opaque(AtomKind kind, Lin r, int64_t k) {
    // Normalise so the atom argument is non-negative (device uses unsigned math).
    int64_t lo = r.lo();
    int64_t shift = 0;
    if (lo < 0) {
        shift = (-lo + k - 1) / k;
        r = r + shift * k;
    }
    AtomP a = make_op_atom(kind, r, k);
    Lin out = Lin::atom(a);
    if (kind == AtomKind::Div && shift) out = out + (-shift);
    return out;
}

}  // namespace

Lin Lin::axis(int ax, int64_t lo, int64_t hi) {
    if (lo == hi) return constant(lo);
    return atom(make_axis_atom(ax, lo, hi));
}

Lin Lin::atom(AtomP a, int64_t c) {
    Lin l;
    if (c != 0) l.t.push_back(Term{c, std::move(a)});
    return l;
}

int64_t Lin::lo() const {
    int64_t v = c0;
    for (const auto& tm : t) v += tm.c > 0 ? tm.c * tm.a->lo : tm.c * tm.a->hi;
    return v;
}

int64_t Lin::hi() const {
    int64_t v = c0;
    for (const auto& tm : t) v += tm.c > 0 ? tm.c * tm.a->hi : tm.c * tm.a->lo;
    return v;
}

std::string Lin::key() const {
    std::string s = std::to_string(c0);
    for (const auto& tm : t) s += "+" + std::to_string(tm.c) + "*" + tm.a->key;
    return s;
}

int64_t Atom::eval(const int64_t* idx) const {
    switch (kind) {
        case AtomKind::Axis: return idx[axis];
        case AtomKind::Div: return floordiv(arg.eval(idx), k);
        case AtomKind::Mod: return floormod(arg.eval(idx), k);
    }
    return 0;
}

int64_t Lin::eval(const int64_t* idx) const {
    int64_t v = c0;
    for (const auto& tm : t) v += tm.c * tm.a->eval(idx);
    return v;
}

bool Lin::depends_on(int axis) const { return (axes_mask(*this) >> axis) & 1; }

uint64_t axes_mask(const Lin& l) {
    uint64_t m = 0;
    for (const auto& tm : l.t) m |= tm.a->axes_mask;
    return m;
}

Lin operator+(const Lin& a, const Lin& b) {
    Lin r = a;
    r.c0 += b.c0;
    for (const auto& tm : b.t) add_term(r, tm.c, tm.a);
    return r;
}

Lin operator-(const Lin& a, const Lin& b) { return a + b * -1; }

Lin operator*(const Lin& a, int64_t s) {
    if (s == 0) return Lin::constant(0);
    Lin r = a;
    r.c0 *= s;
    for (auto& tm : r.t) tm.c *= s;
    return r;
}

Lin operator+(const Lin& a, int64_t c) {
    Lin r = a;
    r.c0 += c;
    return r;
}

namespace {

Lin atom_div(const AtomP& a, int64_t k);
Lin atom_mod(const AtomP& a, int64_t k);

}  // namespace

Lin fdiv(const Lin& L, int64_t k) {
    if (k <= 0) throw Error("fdiv by non-positive constant");
    if (k == 1) return L;
    int64_t lo = L.lo(), hi = L.hi();
    if (floordiv(lo, k) == floordiv(hi, k)) return Lin::constant(floordiv(lo, k));
    if (L.c0 == 0 && L.t.size() == 1 && L.t[0].c == 1) return atom_div(L.t[0].a, k);
    // L = k*q + r, with r as small as the term structure allows.
    Lin q = Lin::constant(floordiv(L.c0, k));
    Lin r = Lin::constant(floormod(L.c0, k));
    for (const auto& tm : L.t) {
        const int64_t c = tm.c;
        if (c % k == 0) {
            add_term(q, c / k, tm.a);
        } else if (c > 0 && k % c == 0 && tm.a->lo >= 0 && tm.a->hi >= k / c) {
            // c*a = k*(a div f) + c*(a mod f), f = k / c
            int64_t f = k / c;
            q = q + atom_div(tm.a, f);
            r = r + atom_mod(tm.a, f) * c;
        } else {
            add_term(r, c, tm.a);
        }
    }
    int64_t rlo = r.lo(), rhi = r.hi();
    if (floordiv(rlo, k) == floordiv(rhi, k)) return q + floordiv(rlo, k);
    if (r.t.size() == 1 && r.t[0].c == 1) {
        const Atom& a = *r.t[0].a;
        // floor((floor(x/a) + c)/k) == floor((x + a*c)/(a*k))
        if (a.kind == AtomKind::Div) return q + fdiv(a.arg + a.k * r.c0, a.k * k);
        if (r.c0 == 0) return q + atom_div(r.t[0].a, k);
    }
    return q + opaque(AtomKind::Div, r, k);
}

Lin fmod(const Lin& L, int64_t k) {
    if (k <= 0) throw Error("fmod by non-positive constant");
    if (k == 1) return Lin::constant(0);
    int64_t lo = L.lo(), hi = L.hi();
    if (floordiv(lo, k) == floordiv(hi, k)) return L + (-k * floordiv(lo, k));
    if (L.c0 == 0 && L.t.size() == 1 && L.t[0].c == 1) return atom_mod(L.t[0].a, k);
    Lin r = Lin::constant(floormod(L.c0, k));
    for (const auto& tm : L.t) {
        int64_t c = tm.c;
        if (floormod(c, k) == 0) continue;
        if (c > 0 && k % c == 0 && tm.a->lo >= 0 && tm.a->hi >= k / c) {
            r = r + atom_mod(tm.a, k / c) * c;  // c*a mod k == c*(a mod k/c)
        } else if (tm.a->kind == AtomKind::Mod && floormod(c * tm.a->k, k) == 0) {
            r = r + tm.a->arg * c;  // c*(x mod m) == c*x (mod k) when k | c*m
        } else {
            if (c > k) c = floormod(c, k);
            add_term(r, c, tm.a);
        }
    }
    int64_t rlo = r.lo(), rhi = r.hi();
    if (floordiv(rlo, k) == floordiv(rhi, k)) return r + (-k * floordiv(rlo, k));
    if (r.c0 == 0 && r.t.size() == 1 && r.t[0].c == 1) return atom_mod(r.t[0].a, k);
    return opaque(AtomKind::Mod, r, k);
}

namespace {

Lin atom_div(const AtomP& a, int64_t k) {
    if (k == 1) return Lin::atom(a);
    if (floordiv(a->lo, k) == floordiv(a->hi, k)) return Lin::constant(floordiv(a->lo, k));
    if (a->kind == AtomKind::Div) return fdiv(a->arg, a->k * k);                       // (x div m) div k
    if (a->kind == AtomKind::Mod && a->k % k == 0) return fmod(fdiv(a->arg, k), a->k / k);  // (x mod m) div k
    return opaque(AtomKind::Div, Lin::atom(a), k);
}

Lin atom_mod(const AtomP& a, int64_t k) {
    if (k == 1) return Lin::constant(0);
    if (floordiv(a->lo, k) == floordiv(a->hi, k)) return Lin::atom(a) + (-k * floordiv(a->lo, k));
    if (a->kind == AtomKind::Mod && a->k % k == 0) return fmod(a->arg, k);  // (x mod m) mod k
    return opaque(AtomKind::Mod, Lin::atom(a), k);
}

}  // namespace

namespace {

Lin subst_atom(const Atom& a, const std::vector<Lin>& vals, std::unordered_map<const Atom*, Lin>& memo) {
    auto it = memo.find(&a);
    if (it != memo.end()) return it->second;
    Lin out;
    switch (a.kind) {
        case AtomKind::Axis:
            out = size_t(a.axis) < vals.size() ? vals[size_t(a.axis)] : Lin::axis(a.axis, a.lo, a.hi);
            break;
        case AtomKind::Div:
        case AtomKind::Mod: {
            Lin arg = Lin::constant(a.arg.c0);
            for (const auto& tm : a.arg.t) arg = arg + subst_atom(*tm.a, vals, memo) * tm.c;
            out = a.kind == AtomKind::Div ? fdiv(arg, a.k) : fmod(arg, a.k);
            break;
        }
    }
    memo.emplace(&a, out);
    return out;
}

}  // namespace

// c*(x mod m) + c*m*(x div m) == c*x : undo digit splits that a later
// composition made redundant (e.g. a Split window re-read through a Reshape).
Lin recombine(Lin l) {
    bool changed = true;
    while (changed) {
        changed = false;
        for (size_t i = 0; i < l.t.size() && !changed; ++i) {
            const Atom& md = *l.t[i].a;
            if (md.kind != AtomKind::Mod) continue;
            for (size_t j = 0; j < l.t.size(); ++j) {
                const Atom& dv = *l.t[j].a;
                if (dv.kind != AtomKind::Div || dv.k != md.k || dv.arg.key() != md.arg.key()) continue;
                if (l.t[j].c != l.t[i].c * md.k) continue;
                int64_t c = l.t[i].c;
                Lin x = md.arg;
                Lin rest = Lin::constant(l.c0);
                for (size_t t = 0; t < l.t.size(); ++t)
                    if (t != i && t != j) rest = rest + Lin::atom(l.t[t].a, l.t[t].c);
                l = rest + x * c;
                changed = true;
                break;
            }
        }
    }
    return l;
}

Lin subst(const Lin& l, const std::vector<Lin>& vals) {
    std::unordered_map<const Atom*, Lin> memo;
    Lin out = Lin::constant(l.c0);
    for (const auto& tm : l.t) out = out + subst_atom(*tm.a, vals, memo) * tm.c;
    return recombine(out);
}

Lin restrict_to(const Lin& l, const Index& lo, const Index& hi) {
    std::vector<Lin> vals;
    for (size_t i = 0; i < lo.size(); ++i) vals.push_back(Lin::axis(int(i), lo[i], hi[i] - 1));
    return subst(l, vals);
}

std::string to_string(const Lin& l) { return l.key(); }

// ---------------------------------------------------------------------------

int64_t VPiece::box_volume() const {
    int64_t v = 1;
    for (size_t i = 0; i < lo.size(); ++i) v *= hi[i] - lo[i];
    return v;
}

bool VPiece::contains(const int64_t* idx) const {
    for (size_t i = 0; i < lo.size(); ++i)
        if (idx[i] < lo[i] || idx[i] >= hi[i]) return false;
    return true;
}

const char* to_string(ContiguityClass c) {
    switch (c) {
        case ContiguityClass::FullyContiguous: return "fully_contiguous";
        case ContiguityClass::PartiallyContiguous: return "partially_contiguous";
        case ContiguityClass::NonContiguous: return "non_contiguous";
    }
    return "?";
}

const char* to_string(TypeClass t) { return t == TypeClass::TypeI ? "type_i" : "type_ii"; }

VMap::VMap(Index shape, std::vector<VPiece> pieces) : shape_(std::move(shape)), pieces_(std::move(pieces)) {
    for (const auto& p : pieces_) {
        if (p.lo.size() != shape_.size() || p.hi.size() != shape_.size())
            throw OutOfBoundsError("piece rank does not match virtual shape");
        for (size_t i = 0; i < shape_.size(); ++i)
            if (p.lo[i] < 0 || p.hi[i] > shape_[i] || p.lo[i] >= p.hi[i])
                throw OutOfBoundsError("piece region outside virtual shape");
    }
}

VPiece VMap::affine_piece(const Index& lo, const Index& hi, const Index& strides, int64_t offset,
                          const std::string& target) {
    VPiece p;
    p.lo = lo;
    p.hi = hi;
    p.target = target;
    Lin off = Lin::constant(offset);
    for (size_t i = 0; i < lo.size(); ++i) off = off + Lin::axis(int(i), lo[i], hi[i] - 1) * strides[i];
    p.off = off;
    return p;
}

VMap VMap::affine(const Index& shape, const Index& strides, int64_t offset, const std::string& target) {
    return VMap(shape, {affine_piece(Index(shape.size(), 0), shape, strides, offset, target)});
}

VMap VMap::identity(const std::string& target, const Index& shape) {
    return affine(shape, default_strides(shape), 0, target);
}

std::vector<std::string> VMap::targets() const {
    std::vector<std::string> t;
    for (const auto& p : pieces_) t.push_back(p.target);
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    return t;
}

const VPiece* VMap::find_piece(const int64_t* idx) const {
    for (const auto& p : pieces_)
        if (p.contains(idx)) return &p;
    return nullptr;
}

std::pair<std::string, int64_t> VMap::eval(const Index& idx) const {
    if (idx.size() != shape_.size()) throw OutOfBoundsError("index rank mismatch");
    for (size_t i = 0; i < idx.size(); ++i)
        if (idx[i] < 0 || idx[i] >= shape_[i]) throw OutOfBoundsError("index outside virtual shape");
    const VPiece* p = find_piece(idx.data());
    if (!p) throw OutOfBoundsError("index not covered by any piece");
    return {p->target, p->off.eval(idx.data())};
}

int64_t VMap::covered_volume() const {
    int64_t v = 0;
    for (const auto& p : pieces_) v += p.box_volume();
    return v;
}

namespace {

bool box_intersect(const Index& alo, const Index& ahi, const Index& blo, const Index& bhi, Index& lo, Index& hi) {
    size_t n = alo.size();
    lo.resize(n);
    hi.resize(n);
    for (size_t i = 0; i < n; ++i) {
        lo[i] = std::max(alo[i], blo[i]);
        hi[i] = std::min(ahi[i], bhi[i]);
        if (lo[i] >= hi[i]) return false;
    }
    return true;
}

template <class F>
void for_each_in_box(const Index& lo, const Index& hi, F&& f) {
    Index idx = lo;
    size_t n = lo.size();
    if (n == 0) {
        f(idx);
        return;
    }
    while (true) {
        f(idx);
        int i = int(n) - 1;
        for (; i >= 0; --i) {
            if (++idx[size_t(i)] < hi[size_t(i)]) break;
            idx[size_t(i)] = lo[size_t(i)];
        }
        if (i < 0) break;
    }
}

// Digit view of an atom: ((axis + shift) div d) mod m.  m == 0: no mod.
struct Digit {
    int axis = -1;
    int64_t shift = 0, d = 1, m = 0;
};

std::optional<Digit> as_digit(const Atom& a) {
    if (a.kind == AtomKind::Axis) return Digit{a.axis, 0, 1, 0};
    auto inner_axis = [](const Lin& l, Digit& dg) -> bool {
        if (l.t.size() != 1 || l.t[0].c != 1 || l.t[0].a->kind != AtomKind::Axis) return false;
        dg.axis = l.t[0].a->axis;
        dg.shift = l.c0;
        return true;
    };
    Digit dg;
    if (a.kind == AtomKind::Div) {
        if (!inner_axis(a.arg, dg)) return std::nullopt;
        dg.d = a.k;
        return dg;
    }
    // Mod
    if (inner_axis(a.arg, dg)) {
        dg.m = a.k;
        return dg;
    }
    if (a.arg.t.size() == 1 && a.arg.t[0].c == 1 && a.arg.c0 == 0 && a.arg.t[0].a->kind == AtomKind::Div) {
        const Atom& dv = *a.arg.t[0].a;
        if (!inner_axis(dv.arg, dg)) return std::nullopt;
        dg.d = dv.k;
        dg.m = a.k;
        return dg;
    }
    return std::nullopt;
}

// Sufficient injectivity of sum(c_i * v_i) over independent variables v_i in
// [0, ext_i): the reference's lattice condition (mapping.cpp:176-193).
bool lattice_injective(std::vector<std::pair<int64_t, int64_t>> se) {
    std::sort(se.begin(), se.end(), std::greater<>());
    int64_t reach = 0;
    for (int i = int(se.size()) - 1; i >= 0; --i) {
        if (se[size_t(i)].first <= reach) return false;
        reach += se[size_t(i)].first * (se[size_t(i)].second - 1);
    }
    return true;
}

// Collect (|coeff|, extent) of a piece's atoms when the atoms are independent
// digits of the box axes; `complete` additionally requires that the digits
// determine every non-degenerate axis (so the map is injective iff the lattice
// condition holds).  Returns false when the structure is not digit-like.
bool digit_structure(const VPiece& p, std::vector<std::pair<int64_t, int64_t>>& se, bool complete) {
    std::map<int, std::vector<Digit>> per_axis;
    std::vector<std::pair<int64_t, int64_t>> out;
    for (const auto& tm : p.off.t) {
        auto dg = as_digit(*tm.a);
        if (!dg || dg->shift != 0) {
            // roll-style atom on one axis: ((x + s) mod m) with x range < m is a bijection
            const Atom& a = *tm.a;
            if (a.kind == AtomKind::Mod && __builtin_popcountll(a.axes_mask) == 1 && a.arg.t.size() == 1 &&
                a.arg.t[0].c == 1 && a.arg.t[0].a->kind == AtomKind::Axis) {
                int ax = a.arg.t[0].a->axis;
                int64_t ext = p.hi[size_t(ax)] - p.lo[size_t(ax)];
                if (ext <= a.k) {
                    per_axis[ax].push_back(Digit{ax, 0, 1, 0});
                    out.emplace_back(std::llabs(tm.c), ext);
                    continue;
                }
            }
            // composite roll: ((sum_i c_i * digit_i + s) mod k) where the digits form an
            // exact mixed-radix number x in [0, prod ext_i) <= k: x -> (x + s) mod k is a
            // bijection, so the atom is one digit of extent k built from its constituents
            // (Swin's roll after window partition: (7 * (t div 392 mod 8) + t div 7 mod 7 + 3) mod 56)
            if (a.kind == AtomKind::Mod && !a.arg.t.empty()) {
                struct Term {
                    int64_t c, ext;
                    Digit d;
                };
                std::vector<Term> ts;
                bool ok = true;
                for (const auto& at : a.arg.t) {
                    auto sub = as_digit(*at.a);
                    if (!sub || sub->shift != 0 || at.c <= 0) {
                        ok = false;
                        break;
                    }
                    Term t{at.c, at.a->hi - at.a->lo + 1, *sub};
                    // c * x mod k only sees x mod (k / c): an unbounded digit is cut there
                    if (a.k % at.c == 0 && t.ext > a.k / at.c) {
                        t.ext = a.k / at.c;
                        if (t.d.m == 0) t.d.m = t.ext;
                        else if (t.d.m % t.ext == 0) t.d.m = t.ext;
                        else {
                            ok = false;
                            break;
                        }
                    }
                    ts.push_back(t);
                }
                if (ok) {
                    std::sort(ts.begin(), ts.end(), [](const Term& x, const Term& y) { return x.c < y.c; });
                    int64_t radix = 1;
                    for (const auto& t : ts) {
                        if (t.c != radix) {
                            ok = false;
                            break;
                        }
                        radix *= t.ext;
                    }
                    if (ok && radix <= a.k) {
                        for (const auto& t : ts) per_axis[t.d.axis].push_back(t.d);
                        out.emplace_back(std::llabs(tm.c), a.k);
                        continue;
                    }
                }
            }
            return false;
        }
        per_axis[dg->axis].push_back(*dg);
        out.emplace_back(std::llabs(tm.c), tm.a->hi - tm.a->lo + 1);
    }
    // Digits of one axis must be disjoint slices of a mixed radix.
    for (auto& [ax, ds] : per_axis) {
        std::sort(ds.begin(), ds.end(), [](const Digit& a, const Digit& b) { return a.d < b.d; });
        int64_t next = ds[0].d;
        for (const auto& d : ds) {
            if (d.d < next) return false;  // overlapping slices
            if (complete && d.d != next) return false;
            if (d.m == 0) next = INT64_MAX;
            else next = d.d * d.m;
        }
        if (complete && ds[0].d != 1) return false;
        if (complete && next != INT64_MAX) {
            int64_t ext = p.hi[size_t(ax)];
            if (next < ext) return false;
        }
    }
    if (complete)
        for (size_t a = 0; a < p.lo.size(); ++a)
            if (p.hi[a] - p.lo[a] > 1 && !per_axis.count(int(a))) return false;
    se = std::move(out);
    return true;
}

}  // namespace

bool VMap::has_overlap() const {
    Index lo, hi;
    for (size_t i = 0; i < pieces_.size(); ++i)
        for (size_t j = i + 1; j < pieces_.size(); ++j)
            if (box_intersect(pieces_[i].lo, pieces_[i].hi, pieces_[j].lo, pieces_[j].hi, lo, hi)) return true;
    return false;
}

bool VMap::is_total() const { return !has_overlap() && covered_volume() == domain_volume(); }

bool VMap::injective(int64_t exhaustive_limit) const {
    bool analytic = true;
    for (const auto& p : pieces_) {
        std::vector<std::pair<int64_t, int64_t>> se;
        if (!digit_structure(p, se, true) || !lattice_injective(se)) {
            analytic = false;
            break;
        }
    }
    if (analytic) {
        for (size_t i = 0; i < pieces_.size() && analytic; ++i)
            for (size_t j = i + 1; j < pieces_.size(); ++j) {
                if (pieces_[i].target != pieces_[j].target) continue;
                const auto &a = pieces_[i], &b = pieces_[j];
                if (a.off.hi() >= b.off.lo() && b.off.hi() >= a.off.lo()) {
                    analytic = false;
                    break;
                }
            }
    }
    if (analytic) return true;
    if (covered_volume() > exhaustive_limit) return false;  // conservative
    auto tl = targets();
    std::vector<std::pair<int, int64_t>> addrs;
    addrs.reserve(size_t(covered_volume()));
    for (const auto& p : pieces_) {
        int ti = int(std::lower_bound(tl.begin(), tl.end(), p.target) - tl.begin());
        for_each_in_box(p.lo, p.hi, [&](const Index& idx) { addrs.emplace_back(ti, p.off.eval(idx.data())); });
    }
    std::sort(addrs.begin(), addrs.end());
    return std::adjacent_find(addrs.begin(), addrs.end()) == addrs.end();
}

int64_t VMap::unique_elems(int64_t exhaustive_limit) const {
    // Canonical image per piece: target, lowest address, sorted (|c|, extent)
    // of the digits the offset uses; identical images are counted once.
    struct Image {
        std::string target;
        int64_t base;
        std::vector<std::pair<int64_t, int64_t>> steps;
        bool operator<(const Image& o) const {
            return std::tie(target, base, steps) < std::tie(o.target, o.base, o.steps);
        }
        bool operator==(const Image& o) const {
            return target == o.target && base == o.base && steps == o.steps;
        }
    };
    std::vector<Image> ims;
    bool analytic = true;
    for (const auto& p : pieces_) {
        std::vector<std::pair<int64_t, int64_t>> se;
        if (!digit_structure(p, se, false) || !lattice_injective(se)) {
            analytic = false;
            break;
        }
        Image im{p.target, p.off.lo(), {}};
        for (auto& s : se)
            if (s.second > 1 && s.first != 0) im.steps.push_back(s);
        std::sort(im.steps.begin(), im.steps.end());
        ims.push_back(std::move(im));
    }
    if (analytic) {
        std::sort(ims.begin(), ims.end());
        ims.erase(std::unique(ims.begin(), ims.end()), ims.end());
        int64_t total = 0;
        for (const auto& im : ims) {
            int64_t v = 1;
            for (auto& s : im.steps) v *= s.second;
            total += v;
        }
        return total;
    }
    if (covered_volume() > exhaustive_limit) return covered_volume();  // upper bound
    auto tl = targets();
    std::vector<std::pair<int, int64_t>> addrs;
    for (const auto& p : pieces_) {
        int ti = int(std::lower_bound(tl.begin(), tl.end(), p.target) - tl.begin());
        for_each_in_box(p.lo, p.hi, [&](const Index& idx) { addrs.emplace_back(ti, p.off.eval(idx.data())); });
    }
    std::sort(addrs.begin(), addrs.end());
    addrs.erase(std::unique(addrs.begin(), addrs.end()), addrs.end());
    return int64_t(addrs.size());
}

namespace {

// Coefficient of axis a when it appears only as a plain Axis atom; else nullopt.
std::optional<int64_t> plain_stride(const VPiece& p, int a) {
    int64_t s = 0;
    for (const auto& tm : p.off.t) {
        if (!((tm.a->axes_mask >> a) & 1)) continue;
        if (tm.a->kind != AtomKind::Axis) return std::nullopt;
        s += tm.c;
    }
    return s;
}

}  // namespace

namespace {

// A box with a plain affine offset (the reference's AffinePiece).
struct AffBox {
    Index lo, hi, strides;
    int64_t c0 = 0;
    std::string target;
    const Lin* off = nullptr;  // the piece's offset (exact values at the box's points)
};

bool affine_strides(const Lin& l, int n, Index& strides) {
    strides.assign(size_t(n), 0);
    for (const auto& tm : l.t) {
        if (tm.a->kind != AtomKind::Axis) return false;
        strides[size_t(tm.a->axis)] += tm.c;
    }
    return true;
}

// Bisect (at the midpoint, the reference's Composer::emit_box split rule,
// mapping.cpp:402-417) the largest axis a div/mod atom depends on until the
// offset is affine over the box,
// then merge abutting boxes with equal strides and offset (IndexMap::normalize,
// mapping.cpp:495-537).  Returns false past `cap` boxes.
bool refine_affine(const VPiece& p, int n, std::vector<AffBox>& out, size_t cap) {
    std::function<bool(const Index&, const Index&)> rec = [&](const Index& lo, const Index& hi) -> bool {
        Lin r = restrict_to(p.off, lo, hi);
        Index st;
        if (affine_strides(r, n, st)) {
            if (out.size() >= cap) return false;
            // restrict_to re-bases nothing: axis atoms keep absolute indices, so c0 is the offset at 0
            out.push_back({lo, hi, st, r.c0, p.target, &p.off});
            return true;
        }
        // split only along axes a non-affine atom depends on (largest first)
        uint64_t mask = 0;
        for (const auto& tm : r.t)
            if (tm.a->kind != AtomKind::Axis) mask |= tm.a->axes_mask;
        int axis = -1;
        int64_t best = 1;
        for (int i = 0; i < n; ++i)
            if (((mask >> i) & 1) && hi[size_t(i)] - lo[size_t(i)] > best) {
                best = hi[size_t(i)] - lo[size_t(i)];
                axis = i;
            }
        if (axis < 0) {  // a single point always resolves
            if (out.size() >= cap) return false;
            out.push_back({lo, hi, Index(size_t(n), 0), r.eval(lo.data()), p.target, &p.off});
            return true;
        }
        Index mhi = hi, mlo = lo;
        int64_t mid = lo[size_t(axis)] + (hi[size_t(axis)] - lo[size_t(axis)]) / 2;
        mhi[size_t(axis)] = mid;
        mlo[size_t(axis)] = mid;
        return rec(lo, mhi) && rec(mlo, hi);
    };
    return rec(p.lo, p.hi);
}

// Merge abutting boxes of one piece whose union is still affine (the
// reference's IndexMap::normalize, mapping.cpp:495-537).  A stride along an
// axis where a box has extent 1 is undetermined; the merge derives it from the
// two boxes' origins, so boxes split by the bisection re-merge whenever the
// offset really is affine across the cut.
void merge_boxes(std::vector<AffBox>& b) {
    auto F = [](const AffBox& x, const Index& idx) { return x.off->eval(idx.data()); };
    bool merged = true;
    while (merged) {
        merged = false;
        for (size_t i = 0; i < b.size() && !merged; ++i)
            for (size_t j = 0; j < b.size(); ++j) {
                if (i == j) continue;
                AffBox &x = b[i], &y = b[j];
                if (x.target != y.target) continue;
                int k = -1;
                bool ok = true;
                for (size_t d = 0; d < x.lo.size(); ++d) {
                    if (x.lo[d] == y.lo[d] && x.hi[d] == y.hi[d]) continue;
                    if (k >= 0) { ok = false; break; }
                    k = int(d);
                }
                if (!ok || k < 0 || x.hi[size_t(k)] != y.lo[size_t(k)]) continue;  // y directly after x along k
                for (size_t d = 0; d < x.lo.size() && ok; ++d)
                    if (int(d) != k && x.hi[d] - x.lo[d] > 1 && x.strides[d] != y.strides[d]) ok = false;
                if (!ok) continue;
                int64_t dk = y.lo[size_t(k)] - x.lo[size_t(k)];
                int64_t df = F(y, y.lo) - F(x, x.lo);
                if (df % dk) continue;
                int64_t sk = df / dk;
                if (x.hi[size_t(k)] - x.lo[size_t(k)] > 1 && x.strides[size_t(k)] != sk) continue;
                if (y.hi[size_t(k)] - y.lo[size_t(k)] > 1 && y.strides[size_t(k)] != sk) continue;
                x.strides[size_t(k)] = sk;
                x.hi[size_t(k)] = y.hi[size_t(k)];
                x.c0 = F(x, x.lo);
                for (size_t d = 0; d < x.lo.size(); ++d) x.c0 -= x.strides[d] * x.lo[d];
                b.erase(b.begin() + long(j));
                merged = true;
                break;
            }
    }
}

// Boxes of one target that tile a box region and agree on one affine function
// become that single box (the reference composes such chains carry-free into
// one piece even when the symbolic form needed several).
void fuse_affine_tiling(std::vector<AffBox>& boxes) {
    std::map<std::string, std::vector<size_t>> by_target;
    for (size_t i = 0; i < boxes.size(); ++i) by_target[boxes[i].target].push_back(i);
    std::vector<AffBox> out;
    std::vector<bool> used(boxes.size(), false);
    for (auto& [t, ids] : by_target) {
        if (ids.size() < 2) continue;
        size_t n = boxes[ids[0]].lo.size();
        Index lo = boxes[ids[0]].lo, hi = boxes[ids[0]].hi;
        int64_t vol = 0;
        for (size_t i : ids) {
            const AffBox& b = boxes[i];
            int64_t v = 1;
            for (size_t d = 0; d < n; ++d) {
                lo[d] = std::min(lo[d], b.lo[d]);
                hi[d] = std::max(hi[d], b.hi[d]);
                v *= b.hi[d] - b.lo[d];
            }
            vol += v;
        }
        int64_t bvol = 1;
        for (size_t d = 0; d < n; ++d) bvol *= hi[d] - lo[d];
        if (vol != bvol) continue;
        Index st(n, 0);
        std::vector<bool> known(n, false);
        bool ok = true;
        for (size_t i : ids)
            for (size_t d = 0; d < n && ok; ++d) {
                const AffBox& b = boxes[i];
                if (b.hi[d] - b.lo[d] <= 1) continue;
                if (known[d] && st[d] != b.strides[d]) ok = false;
                st[d] = b.strides[d];
                known[d] = true;
            }
        if (!ok) continue;
        auto c0_of = [&](const AffBox& b) {
            int64_t c = b.off->eval(b.lo.data());
            for (size_t d = 0; d < n; ++d) c -= st[d] * b.lo[d];
            return c;
        };
        int64_t c0 = c0_of(boxes[ids[0]]);
        for (size_t i : ids) ok = ok && c0_of(boxes[i]) == c0;
        if (!ok) continue;
        AffBox f = boxes[ids[0]];
        f.lo = lo;
        f.hi = hi;
        f.strides = st;
        f.c0 = c0;
        out.push_back(f);
        for (size_t i : ids) used[i] = true;
    }
    for (size_t i = 0; i < boxes.size(); ++i)
        if (!used[i]) out.push_back(boxes[i]);
    boxes = std::move(out);
}

int64_t box_vol(const AffBox& b) {
    int64_t v = 1;
    for (size_t i = 0; i < b.lo.size(); ++i) v *= b.hi[i] - b.lo[i];
    return v;
}

}  // namespace

// proj/src/mapping.cpp:277-328, evaluated over the map's affine boxes: each
// div/mod piece is first refined into the boxes on which its offset is affine
// (what the reference's bisecting compose would have produced), so the report
// describes the same access pattern the reference's piece list describes.
bool VMap::images_disjoint(const VMap& other) const {
    for (const auto& p : pieces_)
        for (const auto& q : other.pieces_) {
            if (p.target != q.target) continue;
            // residue test: image of an affine piece modulo G (gcd of the non-unit
            // strides of both pieces) is one interval spanned by its unit-stride axis
            int n = int(p.lo.size()), m = int(q.lo.size());
            Index sp = Index(static_cast<size_t>(n), 0), sq = Index(static_cast<size_t>(m), 0);
            bool affine = true;
            for (int i = 0; i < n && affine; ++i) {
                auto s = plain_stride(p, i);
                if (!s) affine = false;
                else sp[size_t(i)] = p.hi[size_t(i)] - p.lo[size_t(i)] > 1 ? *s : 0;
            }
            for (int i = 0; i < m && affine; ++i) {
                auto s = plain_stride(q, i);
                if (!s) affine = false;
                else sq[size_t(i)] = q.hi[size_t(i)] - q.lo[size_t(i)] > 1 ? *s : 0;
            }
            bool proved = false;
            if (affine) {  // 1) the two images' address ranges do not overlap
                auto range = [](const VPiece& pc, const Index& st, int64_t& lo, int64_t& hi) {
                    int64_t c = pc.off.eval(pc.lo.data());
                    lo = hi = c;
                    for (size_t i = 0; i < st.size(); ++i) {
                        int64_t span = st[i] * (pc.hi[i] - pc.lo[i] - 1);
                        (span < 0 ? lo : hi) += span;
                    }
                };
                int64_t a_lo, a_hi, b_lo, b_hi;
                range(p, sp, a_lo, a_hi);
                range(q, sq, b_lo, b_hi);
                proved = a_hi < b_lo || b_hi < a_lo;
            }
            if (affine && !proved) {  // 2) residues modulo the common stride lattice
                int64_t G = 0;
                for (auto s : sp) if (s != 0 && s != 1) G = std::gcd(G, std::abs(s));
                for (auto s : sq) if (s != 0 && s != 1) G = std::gcd(G, std::abs(s));
                auto interval = [&](const VPiece& pc, const Index& st, int64_t& r0, int64_t& len) {
                    Index lo = pc.lo;
                    int64_t c = pc.off.eval(lo.data());  // value at the box origin
                    len = 1;
                    int units = 0;
                    for (size_t i = 0; i < st.size(); ++i)
                        if (st[i] == 1) {
                            len = pc.hi[i] - pc.lo[i];
                            ++units;
                        }
                    r0 = floormod(c, G);
                    return units <= 1;
                };
                int64_t a0, alen, b0, blen;
                if (G > 1 && interval(p, sp, a0, alen) && interval(q, sq, b0, blen) && alen + blen <= G) {
                    // intervals [a0, a0+alen) and [b0, b0+blen) on the circle Z_G
                    auto inside = [&](int64_t x, int64_t s0, int64_t len) { return floormod(x - s0, G) < len; };
                    proved = !inside(b0, a0, alen) && !inside(a0, b0, blen);
                }
            }
            if (!proved) {
                if (p.box_volume() > (int64_t(1) << 20) || q.box_volume() > (int64_t(1) << 20)) return false;
                std::vector<int64_t> a, b;
                auto collect = [](const VPiece& pc, std::vector<int64_t>& out) {
                    Index idx = pc.lo;
                    const size_t r = idx.size();
                    while (true) {
                        out.push_back(pc.off.eval(idx.data()));
                        size_t d = r;
                        while (d > 0) {
                            --d;
                            if (++idx[d] < pc.hi[d]) break;
                            idx[d] = pc.lo[d];
                            if (d == 0) return;
                        }
                        if (r == 0) return;
                    }
                };
                collect(p, a);
                collect(q, b);
                std::sort(a.begin(), a.end());
                std::sort(b.begin(), b.end());
                size_t i = 0, j = 0;
                while (i < a.size() && j < b.size()) {
                    if (a[i] == b[j]) return false;
                    if (a[i] < b[j]) ++i;
                    else ++j;
                }
            }
        }
    return true;
}

ContiguityReport VMap::contiguity(int64_t elem_size, int64_t coalesce_unit) const {
    ContiguityReport r;
    int n = rank();
    Index suffix = default_strides(shape_);
    std::vector<AffBox> boxes;
    bool refined = true;
    for (const auto& p : pieces_) {
        std::vector<AffBox> pb;
        if (!refine_affine(p, n, pb, 4096)) {
            refined = false;
            break;
        }
        boxes.insert(boxes.end(), pb.begin(), pb.end());
    }
    if (refined) {
        merge_boxes(boxes);
        fuse_affine_tiling(boxes);
    }
    int d = n + 1;
    for (int cand = n; cand >= 1; --cand) {
        bool ok = true;
        for (const auto& b : boxes) {
            if (b.hi[size_t(cand - 1)] - b.lo[size_t(cand - 1)] <= 1) continue;
            if (b.strides[size_t(cand - 1)] != suffix[size_t(cand - 1)]) {
                ok = false;
                break;
            }
        }
        if (!ok) break;
        d = cand;
    }
    r.min_contiguous_dim = d;
    int64_t min_run = INT64_MAX;
    for (const auto& b : boxes) {
        int64_t run = 1, step = 1;
        for (int i = n - 1; i >= 0; --i) {
            if (shape_[size_t(i)] == 1) continue;
            int64_t ext = b.hi[size_t(i)] - b.lo[size_t(i)];
            if (ext == 1) break;
            if (b.strides[size_t(i)] != step) break;
            run *= ext;
            if (ext != shape_[size_t(i)]) break;
            step *= shape_[size_t(i)];
        }
        min_run = std::min(min_run, run);
    }
    if (boxes.empty()) min_run = 0;
    r.contiguous_run_elems = min_run;
    bool fully = boxes.size() == 1 && d == 1 && box_vol(boxes[0]) == domain_volume();
    if (fully) r.cls = ContiguityClass::FullyContiguous;
    else if (min_run * elem_size >= coalesce_unit) r.cls = ContiguityClass::PartiallyContiguous;
    else r.cls = ContiguityClass::NonContiguous;
    r.type_class = fully ? TypeClass::TypeI : TypeClass::TypeII;
    return r;
}

namespace {

struct Composer {
    const VMap& base;
    Index suffix;
    std::vector<VPiece>& out;
    int cap;
    // Distinct base-piece boundaries per base axis.
    std::vector<std::vector<int64_t>> cuts;

    Composer(const VMap& b, std::vector<VPiece>& o, int c) : base(b), out(o), cap(c) {
        suffix = default_strides(b.shape());
        cuts.resize(b.shape().size());
        for (const auto& q : b.pieces())
            for (size_t j = 0; j < q.lo.size(); ++j) {
                cuts[j].push_back(q.lo[j]);
                cuts[j].push_back(q.hi[j]);
            }
        for (auto& c2 : cuts) {
            std::sort(c2.begin(), c2.end());
            c2.erase(std::unique(c2.begin(), c2.end()), c2.end());
        }
    }

    void push(VPiece&& p) {
        if (int(out.size()) >= cap) throw ComposeLimitError("composed map exceeds piece cap");
        out.push_back(std::move(p));
    }

    int cut_class(size_t j, int64_t v) const {
        return int(std::upper_bound(cuts[j].begin(), cuts[j].end(), v) - cuts[j].begin());
    }

    void emit(const VPiece& P, const Index& lo, const Index& hi) {
        Lin off = restrict_to(P.off, lo, hi);
        const Index& S = base.shape();
        int64_t total = volume(S);
        if (off.lo() < 0 || off.hi() >= total) throw OutOfBoundsError("composed address outside base tensor");
        std::vector<Lin> y(S.size());
        for (size_t j = 0; j < S.size(); ++j) {
            Lin v = fdiv(off, suffix[j]);
            y[j] = j == 0 ? v : fmod(v, S[j]);
        }
        // A base piece containing the whole range box of y?
        for (const auto& q : base.pieces()) {
            bool inside = true;
            for (size_t j = 0; j < S.size() && inside; ++j)
                if (y[j].lo() < q.lo[j] || y[j].hi() >= q.hi[j]) inside = false;
            if (!inside) continue;
            VPiece np;
            np.lo = lo;
            np.hi = hi;
            np.target = q.target;
            np.off = subst(q.off, y);
            push(std::move(np));
            return;
        }
        // Split along an axis that drives a base coordinate across a base cut.
        for (size_t j = 0; j < S.size(); ++j) {
            if (cut_class(j, y[j].lo()) == cut_class(j, y[j].hi())) continue;
            uint64_t m = axes_mask(y[j]);
            if (__builtin_popcountll(m) == 1) {
                int a = __builtin_ctzll(m);
                int64_t ext = hi[size_t(a)] - lo[size_t(a)];
                if (ext <= (int64_t(1) << 20)) {
                    Index probe = lo;
                    std::vector<int64_t> splits;
                    int prev = -1;
                    for (int64_t v = lo[size_t(a)]; v < hi[size_t(a)]; ++v) {
                        probe[size_t(a)] = v;
                        int cls = cut_class(j, y[j].eval(probe.data()));
                        if (prev >= 0 && cls != prev) splits.push_back(v);
                        prev = cls;
                    }
                    if (!splits.empty()) {
                        int64_t start = lo[size_t(a)];
                        splits.push_back(hi[size_t(a)]);
                        for (int64_t s : splits) {
                            Index l2 = lo, h2 = hi;
                            l2[size_t(a)] = start;
                            h2[size_t(a)] = s;
                            emit(P, l2, h2);
                            start = s;
                        }
                        return;
                    }
                }
            }
            // multi-axis dependence: bisect the largest contributing axis
            int best = -1;
            int64_t bext = 1;
            for (size_t a = 0; a < lo.size(); ++a)
                if (((m >> a) & 1) && hi[a] - lo[a] > bext) {
                    bext = hi[a] - lo[a];
                    best = int(a);
                }
            if (best >= 0) {
                bisect(P, lo, hi, best);
                return;
            }
        }
        // Range boxes are conservative (correlated coordinates); bisect the largest axis.
        int best = -1;
        int64_t bext = 1;
        for (size_t a = 0; a < lo.size(); ++a)
            if (hi[a] - lo[a] > bext) {
                bext = hi[a] - lo[a];
                best = int(a);
            }
        if (best < 0) {
            // a single point: evaluate through the base map directly
            Index pt = lo;
            int64_t o = off.eval(pt.data());
            Index yb = unflatten(o, S);
            const VPiece* q = base.find_piece(yb.data());
            if (!q) throw OutOfBoundsError("composed index not covered by base map");
            VPiece np;
            np.lo = lo;
            np.hi = hi;
            np.target = q->target;
            np.off = Lin::constant(q->off.eval(yb.data()));
            push(std::move(np));
            return;
        }
        bisect(P, lo, hi, best);
    }

    void bisect(const VPiece& P, const Index& lo, const Index& hi, int axis) {
        int64_t mid = lo[size_t(axis)] + (hi[size_t(axis)] - lo[size_t(axis)]) / 2;
        Index h1 = hi, l2 = lo;
        h1[size_t(axis)] = mid;
        l2[size_t(axis)] = mid;
        emit(P, lo, h1);
        emit(P, l2, hi);
    }
};

// Merge abutting pieces whose offset formula is the same function.
void normalize_pieces(std::vector<VPiece>& ps) {
    if (ps.size() > 512) return;
    bool merged = true;
    while (merged) {
        merged = false;
        for (size_t i = 0; i < ps.size() && !merged; ++i)
            for (size_t j = i + 1; j < ps.size() && !merged; ++j) {
                auto &a = ps[i], &b = ps[j];
                if (a.target != b.target) continue;
                int diff = -1;
                bool ok = true;
                for (size_t k = 0; k < a.lo.size(); ++k) {
                    if (a.lo[k] == b.lo[k] && a.hi[k] == b.hi[k]) continue;
                    if (diff >= 0) { ok = false; break; }
                    diff = int(k);
                }
                if (!ok || diff < 0) continue;
                if (!(a.hi[size_t(diff)] == b.lo[size_t(diff)] || b.hi[size_t(diff)] == a.lo[size_t(diff)])) continue;
                if (restrict_to(a.off, b.lo, b.hi).key() != b.off.key()) continue;
                Index lo = a.lo, hi = a.hi;
                lo[size_t(diff)] = std::min(a.lo[size_t(diff)], b.lo[size_t(diff)]);
                hi[size_t(diff)] = std::max(a.hi[size_t(diff)], b.hi[size_t(diff)]);
                Lin off = restrict_to(a.off, lo, hi);
                a.lo = lo;
                a.hi = hi;
                a.off = off;
                ps.erase(ps.begin() + int64_t(j));
                merged = true;
            }
    }
    std::sort(ps.begin(), ps.end(), [](const VPiece& a, const VPiece& b) { return a.lo < b.lo; });
}

}  // namespace

VMap VMap::compose(const std::function<const VMap*(const std::string&)>& base, int piece_cap) const {
    std::vector<VPiece> out;
    for (const auto& p : pieces_) {
        const VMap* bm = base(p.target);
        if (!bm) {
            if (int(out.size()) >= piece_cap) throw ComposeLimitError("composed map exceeds piece cap");
            out.push_back(p);
            continue;
        }
        Composer c(*bm, out, piece_cap);
        c.emit(p, p.lo, p.hi);
    }
    normalize_pieces(out);
    VMap m(shape_, std::move(out));
    for (const auto& t : m.targets())
        if (base(t) != nullptr) throw MissingBaseMapError("base map targets a non-physical tensor: " + t);
    return m;
}

namespace {

// Change of `l` when axis `ax` advances by P, if that change is the same for
// every index (atoms see the shift only through whole periods); nullopt else.
std::optional<int64_t> shift_delta(const Lin& l, int ax, int64_t P);

std::optional<int64_t> atom_delta(const Atom& a, int ax, int64_t P) {
    if (!(a.axes_mask & (uint64_t(1) << ax))) return 0;
    if (a.kind == AtomKind::Axis) return a.axis == ax ? P : 0;
    auto d = shift_delta(a.arg, ax, P);
    if (!d) return std::nullopt;
    if (a.kind == AtomKind::Div) {
        if (*d % a.k != 0) return std::nullopt;
        return *d / a.k;
    }
    if (*d % a.k != 0) return std::nullopt;  // Mod: whole periods only
    return 0;
}

std::optional<int64_t> shift_delta(const Lin& l, int ax, int64_t P) {
    int64_t s = 0;
    for (const auto& tm : l.t) {
        auto d = atom_delta(*tm.a, ax, P);
        if (!d) return std::nullopt;
        s += tm.c * *d;
    }
    return s;
}

// Smallest period P (a multiple of every divisor / modulus on the way to `ax`)
// after which every atom of `l` changes by a constant; 0 if none is found.
int64_t clean_period(const Lin& p, const Lin& q, int ax, int64_t extent) {
    std::set<int64_t> ks;
    std::function<void(const Lin&)> walk = [&](const Lin& l) {
        for (const auto& tm : l.t) {
            const Atom& a = *tm.a;
            if (a.kind == AtomKind::Axis || !(a.axes_mask & (uint64_t(1) << ax))) continue;
            ks.insert(a.k);
            walk(a.arg);
        }
    };
    walk(p);
    walk(q);
    int64_t P = 1;
    for (int64_t k : ks) {
        P = std::lcm(P, k);
        if (P > extent) return 0;
    }
    // coefficients inside the atoms may need a multiple of the lcm
    for (int64_t m = 1; m * P <= extent / 2; ++m) {
        auto dp = shift_delta(p, ax, m * P), dq = shift_delta(q, ax, m * P);
        if (dp && dq) return *dp == *dq ? m * P : -1;
    }
    return 0;
}

}  // namespace

int64_t VMap::agree_volume(const VMap& other, int64_t exhaustive_limit) const {
    int64_t agree = 0;
    Index lo, hi;
    for (const auto& p : pieces_)
        for (const auto& q : other.pieces_) {
            if (!box_intersect(p.lo, p.hi, q.lo, q.hi, lo, hi)) continue;
            if (p.target != q.target) continue;
            int64_t v = volume(Index([&] {
                Index e(lo.size());
                for (size_t i = 0; i < lo.size(); ++i) e[i] = hi[i] - lo[i];
                return e;
            }()));
            if (restrict_to(p.off, lo, hi).key() == restrict_to(q.off, lo, hi).key()) {
                agree += v;
                continue;
            }
            // Periodic reduction: when advancing an axis by a period P changes both
            // offsets by the same constant, they agree on the box iff they agree on
            // its first P slices along that axis (and disagreement repeats).
            Index rhi = hi;
            int64_t reps = 1;
            bool differ_const = false;
            for (size_t ax = 0; ax < lo.size() && volume([&] {
                     Index e(lo.size());
                     for (size_t i = 0; i < lo.size(); ++i) e[i] = rhi[i] - lo[i];
                     return e;
                 }()) > exhaustive_limit;
                 ++ax) {
                int64_t ext = rhi[ax] - lo[ax];
                if (ext < 4 || (rhi[ax] - lo[ax]) != (hi[ax] - lo[ax])) continue;
                int64_t P = clean_period(p.off, q.off, int(ax), ext);
                if (P < 0) {
                    differ_const = true;  // both periodic with different steps: disagree beyond the first period
                    break;
                }
                if (P == 0 || ext % P != 0) continue;
                reps *= ext / P;
                rhi[ax] = lo[ax] + P;
            }
            int64_t rv = 1;
            for (size_t i = 0; i < lo.size(); ++i) rv *= rhi[i] - lo[i];
            if (differ_const || rv > exhaustive_limit) continue;  // conservative: counted as disagreeing
            int64_t part = 0;
            for_each_in_box(lo, rhi, [&](const Index& idx) {
                if (p.off.eval(idx.data()) == q.off.eval(idx.data())) ++part;
            });
            agree += part == rv ? v : (reps == 1 ? part : 0);
        }
    return agree;
}

bool VMap::equivalent(const VMap& other, int64_t exhaustive_limit) const {
    if (shape_ != other.shape_) return false;
    int64_t dom = domain_volume();
    return covered_volume() == dom && other.covered_volume() == dom &&
           agree_volume(other, exhaustive_limit) == dom;
}

bool VMap::is_identity_of(const std::string& target) const {
    if (pieces_.size() != 1 || pieces_[0].target != target) return false;
    VMap id = identity(target, shape_);
    return pieces_[0].lo == id.pieces_[0].lo && pieces_[0].hi == id.pieces_[0].hi &&
           pieces_[0].off.key() == id.pieces_[0].off.key();
}

std::optional<int64_t> VMap::tile_stride(const VPiece& p, int axis, int64_t tile) {
    if (tile <= 1) {
        // per-element: only plain axis atoms are affine without a tile guarantee
        tile = 1;
    }
    int64_t stride = 0;
    for (const auto& tm : p.off.t) {
        if (!((tm.a->axes_mask >> axis) & 1)) continue;
        auto dg = as_digit(*tm.a);
        if (!dg) return std::nullopt;
        if (dg->axis != axis) return std::nullopt;
        if (dg->shift % tile != 0) return std::nullopt;
        if (dg->d == 1 && dg->m == 0) {
            stride += tm.c;
        } else if (dg->d == 1) {  // (x mod m): linear inside tiles when tile | m
            if (dg->m % tile != 0) return std::nullopt;
            stride += tm.c;
        } else {  // div: constant inside tiles when tile | d
            if (dg->d % tile != 0) return std::nullopt;
        }
    }
    return stride;
}

std::string VMap::to_string() const {
    std::ostringstream os;
    os << "VMap[";
    for (size_t i = 0; i < shape_.size(); ++i) os << (i ? "," : "") << shape_[i];
    os << "]{";
    for (const auto& p : pieces_) {
        os << " box(";
        for (size_t i = 0; i < p.lo.size(); ++i) os << (i ? "," : "") << p.lo[i] << ":" << p.hi[i];
        os << ")->" << p.target << "@" << p.off.key() << ";";
    }
    os << " }";
    return os.str();
}

}  // namespace vtc

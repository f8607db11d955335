// VMap -> vtc_map lowering.  Each piece's offset (an affine sum of atoms) is
// matched against the two-level descriptor form: top-level digits
// ((I[a] / d) % m) and up to two groups ((((shift + sum digits) % m1) / d) % m2).
// Atoms nested deeper than that are removed by splitting the piece's box
// (on a smaller box the range analysis in vmap.cpp drops the inner mods).
#include <algorithm>
#include <climits>

#include "lower.hpp"

namespace vtc {

namespace {

bool digit_of(const Atom& a, vtc_digit& d) {
    auto axis_only = [](const Lin& l, int& ax) {
        if (l.c0 != 0 || l.t.size() != 1 || l.t[0].c != 1 || l.t[0].a->kind != AtomKind::Axis) return false;
        ax = l.t[0].a->axis;
        return true;
    };
    d.div = 1;
    d.mod = 0;
    d.group = -1;
    int ax = -1;
    switch (a.kind) {
        case AtomKind::Axis: d.axis = int8_t(a.axis); return true;
        case AtomKind::Div:
            if (!axis_only(a.arg, ax) || a.k > UINT32_MAX) return false;
            d.axis = int8_t(ax);
            d.div = uint32_t(a.k);
            return true;
        case AtomKind::Mod:
            if (a.k > UINT32_MAX) return false;
            if (axis_only(a.arg, ax)) {
                d.axis = int8_t(ax);
                d.mod = uint32_t(a.k);
                return true;
            }
            if (a.arg.c0 == 0 && a.arg.t.size() == 1 && a.arg.t[0].c == 1 && a.arg.t[0].a->kind == AtomKind::Div) {
                const Atom& dv = *a.arg.t[0].a;
                if (!axis_only(dv.arg, ax) || dv.k > UINT32_MAX) return false;
                d.axis = int8_t(ax);
                d.div = uint32_t(dv.k);
                d.mod = uint32_t(a.k);
                return true;
            }
            return false;
    }
    return false;
}

const Atom* single_atom(const Lin& l) {
    if (l.c0 != 0 || l.t.size() != 1 || l.t[0].c != 1) return nullptr;
    return l.t[0].a.get();
}

// Lower one piece; false when an atom does not fit the two-level form or the
// digit/group budget is exceeded.  `bad_axes` collects axes of failing atoms.
bool lower_piece(const VPiece& p, vtc_piece& out, uint64_t& bad_axes) {
    out = vtc_piece{};
    int nd = 0, ng = 0;
    out.base = p.off.c0;
    for (size_t a = 0; a < p.lo.size(); ++a) {
        out.lo[a] = int32_t(p.lo[a]);
        out.hi[a] = int32_t(p.hi[a]);
    }
    bool ok = true;
    for (const auto& tm : p.off.t) {
        vtc_digit d{};
        if (digit_of(*tm.a, d)) {
            if (nd >= VTC_MAX_DIGITS) { ok = false; bad_axes |= tm.a->axes_mask; continue; }
            d.coeff = tm.c;
            out.dig[nd++] = d;
            continue;
        }
        // group form: peel Mod(m2) / Div(d) / Mod(m1) around an inner sum of digits
        const Atom* A = tm.a.get();
        uint32_t m1 = 0, dv = 1, m2 = 0;
        const Lin* inner = nullptr;
        if (A->kind == AtomKind::Mod) {
            const Atom* x = single_atom(A->arg);
            if (x && x->kind == AtomKind::Div) {
                m2 = uint32_t(A->k);
                dv = uint32_t(x->k);
                const Atom* y = single_atom(x->arg);
                if (y && y->kind == AtomKind::Mod) {
                    m1 = uint32_t(y->k);
                    inner = &y->arg;
                } else {
                    inner = &x->arg;
                }
            } else {
                m1 = uint32_t(A->k);
                inner = &A->arg;
            }
        } else if (A->kind == AtomKind::Div) {
            dv = uint32_t(A->k);
            const Atom* y = single_atom(A->arg);
            if (y && y->kind == AtomKind::Mod) {
                m1 = uint32_t(y->k);
                inner = &y->arg;
            } else {
                inner = &A->arg;
            }
        }
        bool gok = inner != nullptr && ng < VTC_MAX_GROUPS && inner->lo() >= 0;
        int nd_save = nd;
        if (gok) {
            for (const auto& it : inner->t) {
                vtc_digit gd{};
                if (!digit_of(*it.a, gd) || nd >= VTC_MAX_DIGITS) { gok = false; break; }
                gd.coeff = it.c;
                gd.group = int8_t(ng);
                out.dig[nd++] = gd;
            }
        }
        if (!gok) {
            nd = nd_save;
            ok = false;
            bad_axes |= tm.a->axes_mask;
            continue;
        }
        vtc_group& g = out.grp[ng++];
        g.coeff = tm.c;
        g.shift = inner->c0;
        g.m1 = m1;
        g.d = dv;
        g.m2 = m2;
    }
    for (int t = 0; t < nd; ++t) {
        vtc_digit& d = out.dig[t];
        d.div_shift = int8_t((d.div & (d.div - 1)) == 0 ? __builtin_ctz(d.div) : -1);
        d.mod_shift = int8_t(d.mod && (d.mod & (d.mod - 1)) == 0 ? __builtin_ctz(d.mod) : -1);
    }
    out.ndigits = int16_t(nd);
    out.ngroups = int16_t(ng);
    out.affine = ng == 0 ? 1 : 0;
    for (int a = 0; a < VTC_MAX_RANK; ++a) out.aff[a] = 0;
    for (int t = 0; t < nd; ++t) {
        const vtc_digit& d = out.dig[t];
        if (d.div != 1 || d.mod != 0 || d.group >= 0) out.affine = 0;
        else out.aff[d.axis] += d.coeff;
    }
    return ok;
}

}  // namespace

vtc_map lower_map(const VMap& m, const std::function<TargetInfo(const std::string&)>& target) {
    if (m.rank() > VTC_MAX_RANK) throw UnsupportedError("map rank exceeds VTC_MAX_RANK");
    for (auto s : m.shape())
        if (s > INT32_MAX) throw UnsupportedError("dimension exceeds int32 range");
    vtc_map d{};
    d.rank = m.rank();
    for (int i = 0; i < m.rank(); ++i) d.shape[i] = int32_t(m.shape()[size_t(i)]);
    std::vector<VPiece> work(m.pieces().rbegin(), m.pieces().rend());
    std::vector<vtc_piece> done;
    int guard = 0;
    while (!work.empty()) {
        VPiece p = work.back();
        work.pop_back();
        vtc_piece lp;
        uint64_t bad = 0;
        if (lower_piece(p, lp, bad)) {
            TargetInfo ti = target(p.target);
            lp.target = ti.index;
            lp.ptr = ti.ptr;
            done.push_back(lp);
            continue;
        }
        if (++guard > 4096) throw UnsupportedError("map does not lower to the device descriptor: " + m.to_string());
        // split the widest failing axis
        int best = -1;
        int64_t ext = 1;
        for (size_t a = 0; a < p.lo.size(); ++a)
            if (((bad >> a) & 1) && p.hi[a] - p.lo[a] > ext) {
                ext = p.hi[a] - p.lo[a];
                best = int(a);
            }
        if (best < 0) throw UnsupportedError("map does not lower to the device descriptor: " + m.to_string());
        int64_t mid = p.lo[size_t(best)] + ext / 2;
        VPiece a = p, b = p;
        a.hi[size_t(best)] = mid;
        b.lo[size_t(best)] = mid;
        a.off = restrict_to(p.off, a.lo, a.hi);
        b.off = restrict_to(p.off, b.lo, b.hi);
        work.push_back(b);
        work.push_back(a);
    }
    if (done.size() > VTC_MAX_PIECES)
        throw UnsupportedError("map needs " + std::to_string(done.size()) + " pieces (max " +
                               std::to_string(VTC_MAX_PIECES) + "): " + m.to_string());
    d.npieces = int32_t(done.size());
    for (size_t i = 0; i < done.size(); ++i) d.piece[i] = done[i];
    return d;
}

int64_t desc_eval(const vtc_map& d, const int64_t* idx, int* piece_out) {
    for (int pi = 0; pi < d.npieces; ++pi) {
        const vtc_piece& p = d.piece[pi];
        bool in = true;
        for (int a = 0; a < d.rank; ++a) in = in && idx[a] >= p.lo[a] && idx[a] < p.hi[a];
        if (!in) continue;
        int64_t off = p.base;
        int64_t acc[VTC_MAX_GROUPS] = {};
        for (int g = 0; g < p.ngroups; ++g) acc[g] = p.grp[g].shift;
        for (int t = 0; t < p.ndigits; ++t) {
            const vtc_digit& dg = p.dig[t];
            uint64_t v = uint64_t(idx[dg.axis]) / dg.div;
            if (dg.mod) v %= dg.mod;
            int64_t c = dg.coeff * int64_t(v);
            if (dg.group < 0) off += c;
            else acc[dg.group] += c;
        }
        for (int g = 0; g < p.ngroups; ++g) {
            const vtc_group& G = p.grp[g];
            uint64_t u = uint64_t(acc[g]);
            if (G.m1) u %= G.m1;
            u /= G.d;
            if (G.m2) u %= G.m2;
            off += G.coeff * int64_t(u);
        }
        if (piece_out) *piece_out = pi;
        return off;
    }
    if (piece_out) *piece_out = -1;
    return 0;
}

int64_t desc_tile_stride(const vtc_piece& p, int axis, int64_t tile) {
    int64_t stride = 0;
    for (int t = 0; t < p.ndigits; ++t) {
        const vtc_digit& d = p.dig[t];
        if (d.axis != axis) continue;
        if (d.group >= 0) return INT64_MIN;
        if (d.div == 1 && d.mod == 0) stride += d.coeff;
        else if (d.div == 1) {
            if (d.mod % tile != 0) return INT64_MIN;
            stride += d.coeff;
        } else if (d.div % tile != 0) {
            return INT64_MIN;
        }
    }
    return stride;
}

bool desc_pieces_aligned(const vtc_map& d, int axis, int64_t tile) {
    for (int pi = 0; pi < d.npieces; ++pi) {
        const vtc_piece& p = d.piece[pi];
        if (p.lo[axis] % tile != 0) return false;
        if (p.hi[axis] % tile != 0 && p.hi[axis] != d.shape[axis]) return false;
    }
    return true;
}

}  // namespace vtc

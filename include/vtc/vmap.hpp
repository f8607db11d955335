// Virtual-tensor index maps in closed div/mod form.
//
// The reference represents a virtual tensor's map F (Def. 4.1, PAPER.md) as a
// list of box-shaped affine pieces (proj/include/vtelim/mapping.hpp:31-123):
// every non-affine bias (Expand's modular term, a reshape of a transposed
// view, a roll) is realised by cutting the index space into more boxes, and
// IndexMap::compose bisects boxes until each is carry-free
// (proj/src/mapping.cpp:340-418).  That explodes beyond the 4096-piece cap on
// the north-star chains (SURVEY.md §0 finding 2: GQA at KV >= 512, Swin 56x56).
//
// vtc keeps the reference's piece structure (boxes -> target tensors) but each
// piece's offset is an affine sum over *atoms*, where an atom is a virtual
// axis or a floor-div / mod of an affine sum.  Composition substitutes the
// unflattened outer offset into the base map and simplifies with interval
// arithmetic (carry-free splitting of div/mod over sums), so the GQA chain
// composes to one piece with a (h div 4) digit and roll/window partitions
// compose to a few mod atoms.  Evaluation is exact integer arithmetic and is
// the same formula the device descriptor (include/vtc_desc.h) evaluates.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "vtc/graph.hpp"

namespace vtc {

int64_t floordiv(int64_t a, int64_t b);
int64_t floormod(int64_t a, int64_t b);

struct Atom;
using AtomP = std::shared_ptr<const Atom>;

struct Term {
    int64_t c;
    AtomP a;
};

// c0 + sum(c_i * atom_i); canonical: terms sorted by atom key, merged, non-zero.
struct Lin {
    int64_t c0 = 0;
    std::vector<Term> t;

    static Lin constant(int64_t c) { Lin l; l.c0 = c; return l; }
    static Lin axis(int ax, int64_t lo, int64_t hi);  // hi inclusive; constant when lo == hi
    static Lin atom(AtomP a, int64_t c = 1);

    bool is_const() const { return t.empty(); }
    int64_t lo() const;
    int64_t hi() const;
    std::string key() const;
    int64_t eval(const int64_t* idx) const;
    bool depends_on(int axis) const;
};

enum class AtomKind { Axis, Div, Mod };

struct Atom {
    AtomKind kind = AtomKind::Axis;
    int axis = -1;      // Axis
    Lin arg;            // Div / Mod
    int64_t k = 1;      // divisor / modulus
    int64_t lo = 0, hi = 0;  // value range (inclusive)
    std::string key;
    uint64_t axes_mask = 0;  // virtual axes this atom depends on

    int64_t eval(const int64_t* idx) const;
};

Lin operator+(const Lin& a, const Lin& b);
Lin operator-(const Lin& a, const Lin& b);
Lin operator*(const Lin& a, int64_t s);
Lin operator+(const Lin& a, int64_t c);
Lin fdiv(const Lin& a, int64_t k);
Lin fmod(const Lin& a, int64_t k);
// Replace every Axis(i) atom by vals[i] and re-simplify.
Lin subst(const Lin& l, const std::vector<Lin>& vals);
// Re-simplify with axis ranges narrowed to the box [lo, hi).
Lin restrict_to(const Lin& l, const Index& lo, const Index& hi);
uint64_t axes_mask(const Lin& l);

// One box of the virtual index space mapped into one target tensor.
struct VPiece {
    Index lo, hi;  // [lo, hi)
    std::string target;
    Lin off;       // element offset into target (row-major linear)

    int64_t box_volume() const;
    bool contains(const int64_t* idx) const;
};

enum class ContiguityClass { FullyContiguous, PartiallyContiguous, NonContiguous };
enum class TypeClass { TypeI, TypeII };
const char* to_string(ContiguityClass c);
const char* to_string(TypeClass t);

struct ContiguityReport {
    int min_contiguous_dim = 1;
    int64_t contiguous_run_elems = 0;
    ContiguityClass cls = ContiguityClass::NonContiguous;
    TypeClass type_class = TypeClass::TypeII;
};

class VMap {
public:
    VMap() = default;
    VMap(Index shape, std::vector<VPiece> pieces);

    static VMap identity(const std::string& target, const Index& shape);
    // One full-box affine piece: offset + sum(strides[i] * I_i).
    static VMap affine(const Index& shape, const Index& strides, int64_t offset, const std::string& target);
    // A box-affine piece (reference AffinePiece semantics, mapping.hpp:31-41).
    static VPiece affine_piece(const Index& lo, const Index& hi, const Index& strides, int64_t offset,
                               const std::string& target);

    const Index& shape() const { return shape_; }
    const std::vector<VPiece>& pieces() const { return pieces_; }
    std::vector<VPiece>& pieces_mut() { return pieces_; }
    int64_t domain_volume() const { return volume(shape_); }
    int rank() const { return int(shape_.size()); }
    std::vector<std::string> targets() const;

    const VPiece* find_piece(const int64_t* idx) const;
    std::pair<std::string, int64_t> eval(const Index& idx) const;

    int64_t covered_volume() const;
    bool has_overlap() const;
    bool is_total() const;

    // One-to-one onto (target, offset); required before writing through the map.
    bool injective(int64_t exhaustive_limit = int64_t(1) << 22) const;
    // Distinct physical elements the map touches.
    int64_t unique_elems(int64_t exhaustive_limit = int64_t(1) << 22) const;
    ContiguityReport contiguity(int64_t elem_size, int64_t coalesce_unit) const;

    // F_outer o F_base: pieces whose target has a base map are rewritten onto
    // the base map's targets.  Splits boxes only where a base piece boundary
    // (concat / scatter selection) or an unlowerable nesting requires it.
    VMap compose(const std::function<const VMap*(const std::string&)>& base, int piece_cap = 4096) const;

    // True when both maps send every index to the same (target, offset).
    // Structural first; exhaustive below `exhaustive_limit`; otherwise false.
    bool equivalent(const VMap& other, int64_t exhaustive_limit = int64_t(1) << 22) const;
    // Volume on which the maps agree (used for "coinciding" data movement).
    int64_t agree_volume(const VMap& other, int64_t exhaustive_limit = int64_t(1) << 22) const;

    // True when no physical element is in both maps' images (proved by a
    // residue test on affine pieces, or exhaustively on small maps); false
    // when disjointness cannot be shown.
    bool images_disjoint(const VMap& other) const;

    // True when the map is the identity layout of `target` with `shape`.
    bool is_identity_of(const std::string& target) const;

    // Strides of a piece along an axis for tiles of `tile` elements aligned
    // at multiples of `tile`: the offset is affine with this stride inside
    // every such tile of the piece.  nullopt when not tile-affine.
    static std::optional<int64_t> tile_stride(const VPiece& p, int axis, int64_t tile);

    std::string to_string() const;

private:
    Index shape_;
    std::vector<VPiece> pieces_;
};

std::string to_string(const Lin& l);

}  // namespace vtc

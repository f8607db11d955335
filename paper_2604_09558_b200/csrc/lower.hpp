// Lowering of vtc::VMap to the device descriptor (include/vtc_desc.h) and
// the host-side evaluator of that descriptor (same formula as the device).
#pragma once

#include <functional>
#include <string>
#include <utility>

#include "vtc/vmap.hpp"
#include "vtc_desc.h"

namespace vtc {

struct TargetInfo {
    int index = -1;     // root index in the plan
    uint64_t ptr = 0;   // device address (0 while unbound)
};

// Throws UnsupportedError when the map needs more than VTC_MAX_PIECES pieces
// after splitting unlowerable nestings.
vtc_map lower_map(const VMap& m, const std::function<TargetInfo(const std::string&)>& target);

// Host restatement of the device evaluator; returns the element offset and
// the piece index (or -1 when no piece contains idx).
int64_t desc_eval(const vtc_map& d, const int64_t* idx, int* piece_out);

// Tile-affine stride of a lowered piece along `axis` for aligned tiles of
// `tile` elements, or INT64_MIN when the descriptor is not affine there.
int64_t desc_tile_stride(const vtc_piece& p, int axis, int64_t tile);

// Smallest tile along `axis` at which every piece boundary is aligned.
bool desc_pieces_aligned(const vtc_map& d, int axis, int64_t tile);

}  // namespace vtc

/* Device-side VirtualTensor descriptor (POD, shared by host and device code).
 *
 * A lowered vtc::VMap (include/vtc/vmap.hpp).  It replaces the reference's
 * AffinePiece list (proj/include/vtelim/mapping.hpp:31-41) as the thing a
 * consumer kernel evaluates inside its own loads and stores:
 *
 *   piece  = first box with lo <= I < hi
 *   offset = base
 *          + sum_{digits t, group<0}  coeff_t * ((I[axis_t] / div_t) % mod_t)
 *          + sum_{groups g} coeff_g * ((((shift_g + sum_{digits in g} coeff*digit) % m1) / d) % m2)
 *   address = (char*)ptr + offset * elem_bytes
 *
 * Pieces without any division, modulus or group carry affine = 1 and the
 * per-axis strides aff[] (the same offset, evaluated without the digit walk).
 * mod == 0 / m1 == 0 / m2 == 0 mean "no modulus"; div/d == 1 mean "no
 * division".  All digit and group arguments are non-negative by
 * construction, so the device uses unsigned arithmetic.
 */
#ifndef VTC_DESC_H
#define VTC_DESC_H

#include <stdint.h>

#define VTC_MAX_RANK 8
#define VTC_MAX_PIECES 8
#define VTC_MAX_DIGITS 8
#define VTC_MAX_GROUPS 4

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vtc_digit {
    int64_t coeff;
    uint32_t div;      /* >= 1 */
    uint32_t mod;      /* 0: none */
    int8_t axis;
    int8_t group;      /* -1: top level */
    int8_t div_shift;  /* log2(div) when div is a power of two, else -1 */
    int8_t mod_shift;  /* log2(mod) when mod is a power of two, else -1 */
    int32_t pad;
} vtc_digit;

typedef struct vtc_group {
    int64_t coeff;
    int64_t shift;
    uint32_t m1, d, m2, pad; /* ((s % m1) / d) % m2 */
} vtc_group;

typedef struct vtc_piece {
    int32_t lo[VTC_MAX_RANK];
    int32_t hi[VTC_MAX_RANK];
    int64_t base;      /* element offset */
    uint64_t ptr;      /* device address of the target root */
    int32_t target;    /* root index inside the owning plan */
    int16_t ndigits;
    int16_t ngroups;
    int32_t affine;    /* 1: no div / mod / groups -- offset = base + sum_a aff[a] * I[a] */
    int32_t pad2;
    int64_t aff[VTC_MAX_RANK];
    vtc_digit dig[VTC_MAX_DIGITS];
    vtc_group grp[VTC_MAX_GROUPS];
} vtc_piece;

typedef struct vtc_map {
    int32_t rank;
    int32_t npieces;
    int32_t shape[VTC_MAX_RANK];
    vtc_piece piece[VTC_MAX_PIECES];
} vtc_map;

#ifdef __cplusplus
}
#endif

#endif /* VTC_DESC_H */

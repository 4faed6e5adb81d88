// tc_form.cuh — encoding of one row-block in the tensor-core "window" form (include/vnm.h values_tc /
// meta_tc).  The block's two kept values sit at their own channels (block columns
// c0 < c1, 0..M-1, M <= 8) of an 8-channel window split into two 2:4 groups (channels 0-3 and 4-7); each
// group is completed to exactly two entries with zero values at its lowest free positions.
#pragma once
#include <cstdint>

namespace vnm {

struct TcBlock {
    uint32_t nibs;     // lo-group nibble | hi-group nibble << 4 (each pos_a | pos_b << 2, pos_a < pos_b)
    uint16_t val[4];   // stored values: lo pair, hi pair
};

__device__ __forceinline__ TcBlock tc_encode_block(int c0, int c1, uint16_t v0, uint16_t v1) {
    TcBlock t;
    t.nibs = 0;
#pragma unroll
    for (int gi = 0; gi < 2; ++gi) {
        const int base = 4 * gi;
        const bool in0 = c0 >= base && c0 < base + 4, in1 = c1 >= base && c1 < base + 4;
        uint32_t nib = 0x4u;
        uint16_t a = 0, b = 0;
        if (in0 && in1) {
            nib = static_cast<uint32_t>(c0 - base) | (static_cast<uint32_t>(c1 - base) << 2);
            a = v0;
            b = v1;
        } else if (in0 || in1) {
            const int p = (in0 ? c0 : c1) - base;
            const uint16_t v = in0 ? v0 : v1;
            const int f = p == 0 ? 1 : 0;
            nib = static_cast<uint32_t>(p < f ? p : f) | (static_cast<uint32_t>(p < f ? f : p) << 2);
            if (p < f) a = v; else b = v;
        }
        t.nibs |= nib << (4 * gi);
        t.val[2 * gi] = a;
        t.val[2 * gi + 1] = b;
    }
    return t;
}

// The 16-channel window (8 < M <= 16, M % 4 != 0; include/vnm.h "window-16 form"): the block's M channels
// followed by 16-M channels of the next block, as four 2:4 groups (channels 0-3, 4-7, 8-11, 12-15), each
// completed to exactly two entries with zero values at its lowest free positions (the rule of tc_encode_block).
// nibs: group q's nibble at bits 4q; val[2q], val[2q+1]: group q's stored pair.  Half h (groups 2h, 2h+1) is
// what MMA (block group, h) reads: byte h of nibs and val[4h .. 4h+3].
struct TcBlock16 {
    uint32_t nibs;
    uint16_t val[8];
};

__device__ __forceinline__ TcBlock16 tc_encode_block16(int c0, int c1, uint16_t v0, uint16_t v1) {
    TcBlock16 t;
    t.nibs = 0;
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
        const int base = 4 * gi;
        const bool in0 = c0 >= base && c0 < base + 4, in1 = c1 >= base && c1 < base + 4;
        uint32_t nib = 0x4u;
        uint16_t a = 0, b = 0;
        if (in0 && in1) {
            nib = static_cast<uint32_t>(c0 - base) | (static_cast<uint32_t>(c1 - base) << 2);
            a = v0;
            b = v1;
        } else if (in0 || in1) {
            const int p = (in0 ? c0 : c1) - base;
            const uint16_t v = in0 ? v0 : v1;
            const int f = p == 0 ? 1 : 0;
            nib = static_cast<uint32_t>(p < f ? p : f) | (static_cast<uint32_t>(p < f ? f : p) << 2);
            if (p < f) a = v; else b = v;
        }
        t.nibs |= nib << (4 * gi);
        t.val[2 * gi] = a;
        t.val[2 * gi + 1] = b;
    }
    return t;
}

}  // namespace vnm

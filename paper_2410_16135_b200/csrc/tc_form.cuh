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

}  // namespace vnm

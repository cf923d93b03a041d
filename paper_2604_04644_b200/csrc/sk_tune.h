// Tile width EB (elements per CTA = payload lane width) per (shape, order),
// picked from B200 sweeps of 14 variants (EB x threads-divisor x min-blocks,
// tools/build_variants.sh + tools/tune_eb.py; profiles/r01/tune_helm.jsonl).
// 0 = default rule (largest power of two <= 16 whose three
// quad-point planes fit in 100 KB of shared memory).
#pragma once

namespace sk {

constexpr int kTunedEB[4][11] = {
    //  P: 0  1  2  3  4  5  6  7  8  9  10
    {0, 16, 16, 16, 8, 2, 2, 4, 1, 1, 2},  // hex
    {0, 16, 16, 16, 8, 8, 4, 4, 4, 4, 1},  // prism
    {0, 16, 16, 8, 8, 4, 4, 2, 1, 1, 2},  // pyr
    {0, 16, 16, 16, 8, 8, 4, 4, 4, 4, 2},  // tet
};

// threads per CTA = EB x (largest sweep item count) / divisor
constexpr int kTunedNTDiv[4][11] = {
    {1, 2, 1, 2, 1, 1, 1, 1, 1, 1, 1},  // hex
    {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},  // prism
    {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},  // pyr
    {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},  // tet
};

// 1: __launch_bounds__ min blocks = CTAs/SM allowed by shared memory
constexpr int kTunedMinB[4][11] = {
    {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},  // hex
    {0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1},  // prism
    {0, 1, 0, 1, 1, 1, 1, 1, 1, 1, 1},  // pyr
    {0, 0, 0, 1, 1, 1, 1, 1, 1, 0, 0},  // tet
};

#ifdef SK_EB_FIXED
constexpr int tuned_eb(int, int) { return SK_EB_FIXED; }
#else
constexpr int tuned_eb(int S, int P) { return kTunedEB[S][P]; }
#endif
#ifdef SK_NT_DIV
constexpr int tuned_nt_div(int, int) { return SK_NT_DIV; }
#else
constexpr int tuned_nt_div(int S, int P) { return kTunedNTDiv[S][P]; }
#endif
#ifdef SK_MINB
constexpr int tuned_minb(int, int) { return SK_MINB; }
#else
constexpr int tuned_minb(int S, int P) { return kTunedMinB[S][P]; }
#endif

}  // namespace sk

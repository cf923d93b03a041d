// Tile width EB (elements per CTA = payload lane width) per (shape, order),
// picked from B200 sweeps of 14 variants (EB x threads-divisor x min-blocks,
// tools/build_variants.sh + tools/tune_eb.py; profiles/r01/tune_helm.jsonl).
// 0 = default rule (largest power of two <= 16 whose three
// quad-point planes fit in 100 KB of shared memory).
#pragma once

#ifdef __CUDACC__
#define SK_HD __host__ __device__
#else
#define SK_HD
#endif

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

// 1: __launch_bounds__ min blocks = CTAs/SM allowed by shared memory, capped
// at kMinBCap (Helmholtz/stiffness kernels)
constexpr int kTunedMinB[4][11] = {
    {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},  // hex
    {0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1},  // prism
    {0, 1, 0, 1, 1, 1, 1, 1, 1, 1, 1},  // pyr
    {0, 0, 0, 1, 1, 1, 1, 1, 1, 0, 0},  // tet
};

// CTAs/SM cap of the min-blocks rule, per operator class (0 Helmholtz and
// stiffness, 1 mass, 2 the stand-alone transforms) x shape x order
constexpr int kMinBCap[3][4][11] = {
    {{4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4}},
    {{4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4}},
    {{4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4}},
};

// pyr/tet ragged r <-> k sweeps: compile-time slice dispatch up to this
// order (uniform table operands), L1 table reads above it (code size);
// per operator class x shape
constexpr int kRaggedMaxP[3][4] = {
    {0, 0, 6, 5},  // Helmholtz / stiffness
    {0, 0, 8, 8},  // mass
    {0, 0, 8, 8},  // transforms
};

// points of geometry loads in flight ahead of the metric in the Helmholtz
// middle sweep (lines longer than 6 points)
#ifdef SK_GEO_PD
constexpr int kGeoPipeDepth = SK_GEO_PD;
#else
constexpr int kGeoPipeDepth = 2;
#endif

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
#ifdef SK_MINB_CAP
constexpr int tuned_minb_cap(int, int, int) { return SK_MINB_CAP; }
#else
constexpr int tuned_minb_cap(int cls, int S, int P) { return kMinBCap[cls][S][P]; }
#endif

#ifdef SK_RAGGED_MAXP
SK_HD constexpr bool ragged_dispatch(int, int, int P) { return P <= SK_RAGGED_MAXP; }
#else
SK_HD constexpr bool ragged_dispatch(int cls, int S, int P) { return P <= kRaggedMaxP[cls][S]; }
#endif

}  // namespace sk

// Launch tuning tables per operator class x shape x order, picked from B200
// sweeps of variant builds (tools/build_variants.sh + tools/tune_eb.py;
// profiles/).  Operator classes: 0 Helmholtz / stiffness, 1 mass, 2 the
// stand-alone transforms.  Tile widths come in two families that own a
// geometry payload layout each: the Helmholtz family (Helmholtz, stiffness,
// non-collocated Helmholtz, phys_deriv) and the W family (mass, iproduct,
// iproduct-deriv, bwd_trans).
#pragma once

#ifdef __CUDACC__
#define SK_HD __host__ __device__
#else
#define SK_HD
#endif

namespace sk {

// EB = elements per CTA tile (= payload lane width of the family's payload);
// 0 = default rule (largest power of two <= 16 whose three quad-point
// planes fit in 100 KB of shared memory)
constexpr int kTunedEB[2][4][11] = {
    // Helmholtz family            P: 0  1   2   3   4  5  6  7  8  9  10
    {{0, 16, 8, 16, 8, 2, 2, 1, 1, 1, 2},    // hex
     {0, 16, 16, 16, 4, 8, 4, 2, 2, 1, 1},   // prism
     {0, 16, 8, 16, 8, 4, 4, 1, 1, 1, 1},    // pyr
     {0, 16, 16, 8, 8, 8, 4, 4, 4, 4, 2}},   // tet
    // W family (mass, iproduct, iproduct-deriv, bwd_trans)
    {{0, 16, 16, 16, 16, 8, 2, 8, 1, 1, 2},
     {0, 16, 16, 16, 16, 16, 8, 4, 4, 16, 1},
     {0, 16, 16, 8, 16, 8, 8, 8, 4, 2, 1},
     {0, 16, 16, 16, 16, 8, 8, 16, 16, 8, 8}},
};

// regular-geometry collocated Helmholtz / stiffness tile width (0 = the
// deformed table's); its payload has a fixed lane width (kRegPW), so the
// tile is tuned on its own (profiles/r01c/tune_regular_eb*.jsonl)
constexpr int kTunedEBReg[4][11] = {
    // P: 0  1  2  3  4  5  6  7  8  9  10
    {0, 0, 0, 0, 0, 0, 4, 4, 2, 0, 0},  // hex
    {0, 0, 0, 8, 0, 16, 8, 1, 4, 0, 2},  // prism
    {0, 0, 0, 0, 0, 0, 8, 0, 0, 0, 2},  // pyr
    {0, 0, 0, 0, 0, 0, 8, 0, 0, 0, 0},  // tet
};

// regular-geometry thread divisor (0 = the class table's): two items per
// thread measured +9-17 % at hex P=1, prism P=3/4, tet P=3
// (profiles/r01c/tune_regular_nt.jsonl)
constexpr int kTunedNTDivReg[4][11] = {
    {0, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // hex
    {0, 0, 0, 2, 2, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0},  // tet
};

// threads per CTA = EB x (largest sweep item count) / divisor
constexpr int kTunedNTDiv[3][4][11] = {
    {{1, 1, 1, 2, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 1, 2, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1}},
    {{1, 2, 2, 2, 1, 2, 1, 2, 1, 1, 1},
     {1, 2, 2, 2, 2, 2, 2, 1, 2, 1, 1},
     {1, 2, 1, 2, 1, 1, 1, 1, 1, 1, 1},
     {1, 1, 2, 1, 1, 1, 1, 1, 2, 1, 1}},
    {{1, 2, 1, 2, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1},
     {1, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1}},
};

// 1: __launch_bounds__ min blocks = CTAs/SM allowed by shared memory, capped
// at kMinBCap; 0: no min-blocks bound
constexpr int kTunedMinB[3][4][11] = {
    {{0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 0, 0, 1, 1, 1, 1, 1, 1, 0, 1}},
    {{0, 1, 1, 1, 1, 1, 1, 1, 0, 1, 1},
     {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0}},
    {{0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 1, 0, 1, 1, 1, 1, 1, 1, 1, 1},
     {0, 0, 0, 1, 1, 1, 1, 1, 1, 0, 0}},
};

// CTAs/SM cap of the min-blocks rule
constexpr int kMinBCap[3][4][11] = {
    {{4, 4, 8, 4, 4, 5, 4, 5, 4, 4, 4},
     {4, 4, 4, 5, 8, 6, 8, 8, 8, 4, 4},
     {4, 4, 8, 4, 4, 4, 8, 8, 5, 4, 4},
     {4, 4, 4, 8, 5, 4, 4, 4, 8, 4, 4}},
    {{4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 8, 4, 4, 4},
     {4, 4, 8, 4, 4, 4, 4, 8, 8, 4, 4},
     {4, 8, 4, 8, 4, 8, 4, 4, 4, 4, 4}},
    {{4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4},
     {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4}},
};

// Helmholtz geometry L2 prefetch of a tile: 1 = at tile start (bulk TMA
// prefetch, SASS UBLKPF), 2 = after the F2 sweep, 3 = both, 0 = none
// per shape x order; after F2 measured +1-7 % at P=6 (every shape), P=10
// (hex, prism, pyr) and tet P=9, for Helmholtz and stiffness alike
// (profiles/r01c/tune_geo_prefetch_pf2.jsonl); at tile start elsewhere
constexpr int kGeoPF[4][11] = {
    {1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 2},  // hex
    {1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 2},  // prism
    {1, 1, 1, 1, 1, 1, 2, 1, 1, 1, 2},  // pyr
    {1, 1, 1, 1, 1, 1, 2, 1, 1, 2, 1},  // tet
};
#ifdef SK_GEO_PF
SK_HD constexpr int geo_prefetch(int, int) { return SK_GEO_PF; }
#else
SK_HD constexpr int geo_prefetch(int S, int P) { return kGeoPF[S][P]; }
#endif

// Deformed Helmholtz (lam != 0) metric sweep in the low-register form
// (sk_ops.cuh M2, bit-identical arithmetic: lam W u staged through the U
// plane instead of keeping u live, the D2^T accumulator loaded after the
// metric loop).  Measured on B200, two A/B runs against the default form,
// 1 GB deformed (profiles/r02/m2_lowreg_ab*.jsonl, drift control <= 1.2 %):
// hex P=10 +27 / +26 %, pyr P=10 +8 / +9 %, prism P=10 +7 / +7 %, prism
// P=7 +3 / +3 %; other orders within noise or losing (tet -2 .. -11 % in
// the first run), and stiffness (lam = 0, no u term) gains nowhere, so the
// form is used for lam != 0 only.  Build-time override for A/B:
// -DSK_M2_LOWREG=0/1 (every Helmholtz instantiation).
constexpr bool kM2LowRegT[4][11] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},  // hex
    {0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};
#ifdef SK_M2_LOWREG
SK_HD constexpr bool m2_lowreg(int, int) { return SK_M2_LOWREG; }
#else
SK_HD constexpr bool m2_lowreg(int S, int P) { return kM2LowRegT[S][P]; }
#endif

// points per geometry-load chunk in the Helmholtz metric sweep (lines longer
// than 6 points): 7*CH doubles in flight per thread
#ifdef SK_GEO_CH
constexpr int kGeoChunk = SK_GEO_CH;
#else
constexpr int kGeoChunk = 4;
#endif

// 1: persistent CTAs (one resident wave striding over the tiles, next tile's
// coefficients register-prefetched, its geometry L2-prefetched after the
// metric sweep); Helmholtz class only, where measured faster
constexpr int kPersist[4][11] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0},  // hex
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};

// prism/pyr/tet ragged r <-> k sweeps: one item per (element, p, q) pair
// with the slice dispatched to compile-time constants up to this order
// (uniform table operands), L1 table reads above it (code size).  Prism
// without dispatch: one item per (element, q), all p unrolled, up to
// kPrismUniformMaxP.  Dispatch measured slower for Helmholtz at P >= 7 on
// every shape and for prism at every order but 7 (+5 %) (c3_tune_helm)
constexpr int kRaggedMaxP[3][4] = {
    {0, 0, 6, 5},  // Helmholtz / stiffness
    {0, 0, 9, 8},  // mass (pyr P=9: +12 %, c3_tune_mass)
    {0, 0, 8, 8},  // transforms
};

// r <-> k sweeps split over two threads per line when the lines fill at most
// half the CTA (pyr/tet (p,q) pairs: halves of k / r parity; prism (e, q)
// lines: p parity), from this order on, per operator class x shape.
// Measured: tet Helmholtz P=9/10 +3 %/+15 % (P=3-8 -2..-7 %), prism mass
// P>=5 +2..5 %, elsewhere no gain (tune14_op1.jsonl)
constexpr int kSplitMinP[3][4] = {
    {99, 99, 99, 9},  // Helmholtz / stiffness
    {99, 5, 99, 99},  // mass
    {99, 99, 99, 99},  // transforms
};

// prism r <-> k sweeps with warp-uniform slice pairs (sk_stages.cuh
// prism_slice_pairs) at these orders, per operator class: measured +3-4 %
// Helmholtz/stiffness P=6/7, mass +9/+6/+4 % P=6/7/9, slower at P=8/10
// (c5_tune_wp_*.jsonl)
constexpr bool kPrismWP[3][11] = {
    {0, 0, 0, 0, 0, 0, 1, 1, 0, 0, 0},
    {0, 0, 0, 0, 0, 0, 1, 1, 0, 1, 0},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
};

// Deformed Helmholtz geometry through a shared-memory ring fed by TMA bulk
// copies (cp.async.bulk + mbarrier, sk_ops.cuh k_helm): the ring holds this
// many k-slices of the tile's metric payload (0 = off: per-thread streaming
// loads after a tile-start L2 prefetch).  The first slices are issued at
// tile start and land during the F and M1 sweeps; the metric sweep refills
// each slot as soon as every warp is done with it.
constexpr int kGeoRing[4][11] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // hex
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};
#ifdef SK_GEO_RING
SK_HD constexpr int geo_ring(int, int) { return SK_GEO_RING; }
#else
SK_HD constexpr int geo_ring(int S, int P) { return kGeoRing[S][P]; }
#endif

// Deformed sum-factorised mass with TMA-moved tile inputs (sk_ops.cuh
// k_mass_tma) instead of k_mass, per shape x order.  Measured on B200, two
// A/B runs (profiles/r02/mass_tma_ab.jsonl, mass_tma_grid.jsonl; roofline
// fraction k_mass -> k_mass_tma): pyr P=3 0.45 -> 0.61, P=4 0.51 -> 0.54,
// P=5 0.44 -> 0.48, P=6 0.46 -> 0.49; prism P=2 0.59 -> 0.66, P=3 0.59 ->
// 0.72; tet P=4 0.43 -> 0.50, P=5 0.40 -> 0.43; hex P=6 0.69 -> 0.74.  It
// loses at tet P=3, prism P>=4, hex P=3..5 and P>=7 (one resident wave with
// the larger footprint), and the DMMA StdMat kernel stays ahead at P=1 and
// pyr / tet P=2; tile widths 4 / 8 and halved thread counts were no better.
// Build-time override for A/B: -DSK_MASS_TMA=0/1 (every order); run-time:
// SK_MASS_TMA=0.
constexpr bool kMassTma[4][11] = {
    // P: 0  1  2  3  4  5  6  7  8  9 10
    {0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0},  // hex
    {0, 0, 1, 1, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 0},  // tet
};
#ifdef SK_MASS_TMA
SK_HD constexpr bool mass_tma(int, int) { return SK_MASS_TMA; }
#else
SK_HD constexpr bool mass_tma(int S, int P) { return kMassTma[S][P]; }
#endif

// Deformed Helmholtz / stiffness through the persistent TMA-staged driver
// (sk_ops.cuh k_persist_tma) instead of k_tile / k_persist, per shape x
// order.  Measured on B200 (profiles/r02/helm_tma_ab*.jsonl, roofline
// fraction Helmholtz / stiffness, default -> TMA): hex P=6 0.86 -> 0.92 /
// 0.81 -> 0.85, P=7 0.65 -> 0.72, P=8 0.65 -> 0.68 / 0.64 -> 0.67, P=9
// 0.70 -> 0.77; prism P=2 0.90 -> 0.94; pyr P=2 0.88 -> 0.92 / 0.80 -> 0.84,
// P=3 stiffness 0.69 -> 0.74, P=5 0.65 -> 0.72.  It loses at prism / pyr /
// tet P>=6 and hex P<=5, P=10: one resident wave, the register-capped tile
// spills a little.  Build-time override for A/B: -DSK_HELM_TMA=0/1;
// run-time: SK_HELM_TMA=0.
constexpr bool kHelmTma[4][11] = {
    // P: 0  1  2  3  4  5  6  7  8  9 10
    {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 0},  // hex
    {0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 1, 1, 0, 1, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};
// the same driver for regular-geometry Helmholtz / stiffness (sum-factorised
// orders; the StdMat kernels take the low orders).  Measured
// (profiles/r02/helm_tma_regular.jsonl, FP64 roofline fraction Helmholtz /
// stiffness): tet P=9 0.30 -> 0.40 / 0.34 -> 0.35, prism P=5 0.42 -> 0.44 /
// 0.43 -> 0.48; it loses at most other orders (hex P=6-8 -15-30 %).
constexpr bool kHelmTmaReg[4][11] = {
    // P: 0  1  2  3  4  5  6  7  8  9 10
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // hex
    {0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0},  // tet
};
#ifdef SK_HELM_TMA_REG
SK_HD constexpr bool helm_tma_reg(int, int) { return SK_HELM_TMA_REG; }
#else
SK_HD constexpr bool helm_tma_reg(int S, int P) { return kHelmTmaReg[S][P]; }
#endif
#ifdef SK_HELM_TMA
SK_HD constexpr bool helm_tma(int, int) { return SK_HELM_TMA; }
#else
SK_HD constexpr bool helm_tma(int S, int P) { return kHelmTma[S][P]; }
#endif

// Sum-factorised mass with one warp per tile (sk_ops.cuh k_mass_warp, no CTA
// barriers) instead of the CTA-tile k_mass: elements per warp tile G and
// warps per CTA, per shape x order (G = 0: CTA tiles).  Build-time
// overrides for A/B: -DSK_MASS_WARP_G=<G> (every order), -DSK_MASS_WARP_WPC.
// Run-time override: SK_MASS_WARP=0 (never).
constexpr int kMassWarpG[4][11] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // hex
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};
#ifdef SK_MASS_WARP_G
SK_HD constexpr int mass_warp_g(int, int) { return SK_MASS_WARP_G; }
#else
SK_HD constexpr int mass_warp_g(int S, int P) { return kMassWarpG[S][P]; }
#endif
#ifdef SK_MASS_WARP_WPC
constexpr int kMassWarpWPC = SK_MASS_WARP_WPC;
#else
constexpr int kMassWarpWPC = 8;
#endif
#ifdef SK_MASS_WARP_MINB
constexpr int kMassWarpMinB = SK_MASS_WARP_MINB;
#else
constexpr int kMassWarpMinB = 1;
#endif

// Mass by the StdMat strategy on the FP64 tensor cores (sk_dense.cuh)
// instead of sum factorisation, per geometry class (0 regular, 1 deformed)
// x shape x order; instantiated up to kDenseMaxP.  Run-time override:
// SK_MASS_DENSE=0 (never) / 1 (wherever instantiated).
constexpr int kDenseMaxP = 6;
// Measured on B200 (roofline fraction sum-fac -> dense): deformed
// (profiles/r02/mass_dense_def_*.jsonl) P=1 every shape (hex 0.60 -> 0.70,
// prism 0.56 -> 0.74, pyr 0.46 -> 0.69, tet 0.41 -> 0.73), pyr / tet P=2
// (0.46 -> 0.62, 0.48 -> 0.53), tet P=3 (0.47 -> 0.54, re-measured with the
// register-bounded dense kernel, profiles/r02/dense_vs_sumfac_p2to4.txt);
// regular (|J| M_ref, one GEMM;
// profiles/r02/dense_mass_regular_*.jsonl) hex P<=2 (0.23/0.35 ->
// 0.76/0.58), prism P<=4 (0.22-0.38 -> 0.48-0.69), pyr P<=5 (0.17-0.37 ->
// 0.59-0.89), tet P<=6 (0.19-0.33 -> 0.65-1.16); slower elsewhere.
constexpr bool kDenseMass[2][4][11] = {
    // regular   P: 0  1  2  3  4  5  6
    {{0, 1, 1, 1, 0, 0, 0},   // hex (P=3: 0.38 -> 0.49, profiles/r02/dense_vs_sumfac_regular.txt)
     {0, 1, 1, 1, 1, 0, 0},   // prism
     {0, 1, 1, 1, 1, 1, 0},   // pyr
     {0, 1, 1, 1, 1, 1, 1}},  // tet
    // deformed
    {{0, 1, 0, 0, 0, 0, 0},
     {0, 1, 0, 0, 0, 0, 0},
     {0, 1, 1, 0, 0, 0, 0},
     {0, 1, 1, 1, 0, 0, 0}},
};

// Regular-geometry collocated Helmholtz / stiffness by StdMat on DMMA
// (sk_dense.cuh k_helm_dense: seven NM x NM element-independent matrices
// combined with the element's Lam and |J|) instead of sum factorisation,
// per shape x order (instantiated where the fragments fit, P <= kDenseMaxP).
// Run-time override: SK_HELM_DENSE=0 / 1.
// Measured (profiles/r02/dense_helm_regular_*.jsonl, roofline fraction of
// the reference flop count, Helmholtz / stiffness): hex P<=2 (0.30/0.41 ->
// 1.30/0.46), prism P<=3 (0.32-0.47 -> 0.55-0.99), pyr P<=3 (0.27-0.40 ->
// 0.86-1.18), tet P<=4 (0.26-0.43 -> 1.00-1.35); the dense form does fewer
// flops than the sum-factorised count there.  P>=4 (hex, prism, pyr) and P>=5
// (tet): fragments beyond 100 KB of shared memory or slower.
constexpr bool kDenseHelm[4][11] = {
    // P: 0  1  2  3  4
    {0, 1, 1, 0, 0},  // hex
    {0, 1, 1, 1, 0},  // prism
    {0, 1, 1, 1, 0},  // pyr
    {0, 1, 1, 1, 1},  // tet
};

// Overrides for tuning builds (-DSK_EB_FIXED=... etc.) apply to every class.
#ifdef SK_EB_FIXED
SK_HD constexpr int tuned_eb(int, int, int) { return SK_EB_FIXED; }
#else
SK_HD constexpr int tuned_eb(int fam, int S, int P) { return kTunedEB[fam][S][P]; }
#endif
// bwd_trans tile width (it reads no payload, so it need not match the W
// family's lane width); 0 = the W family's.  From a tile-width grid
// (profiles/r02/bwd_eb_grid.jsonl), adopted where >= 8 % faster: e.g. hex
// P=4 0.45 -> 0.69, tet P=3 0.27 -> 0.41, prism P=3 0.51 -> 0.66.
constexpr int kTunedEBBwd[4][11] = {
    { 0,  0,  8,  8,  4,  0,  0,  1,  0,  0,  0},  // hex
    { 0,  0,  8,  8,  4,  4,  2,  0,  0,  1,  0},  // prism
    { 0,  0,  8,  0,  4,  0,  2,  4,  0,  0,  0},  // pyr
    { 0,  0,  0,  8,  4,  0,  0,  4,  0,  0,  0}  // tet
};
// non-collocated Helmholtz tile width = its payload's lane width (kind 3);
// 0 = the Helmholtz family's.  From a tile-width grid with the five-plane
// fit (profiles/r02/nc_eb_grid*.jsonl), adopted where >= 8 % faster: e.g.
// pyr P=4 0.33 -> 0.44, tet P=6 0.25 -> 0.36, prism P=8 0.21 -> 0.32.
constexpr int kTunedEBNc[4][11] = {
    { 0,  0,  0,  0,  2, 16,  0,  4,  0,  0,  0},  // hex
    { 0,  0,  0,  0,  0,  0,  0,  0, 16,  0,  4},  // prism
    { 0,  0, 16,  0, 16,  0,  0,  4,  4,  0,  0},  // pyr
    { 0,  0,  0,  0,  0,  0,  8,  0,  0,  0,  0},  // tet
};
// phys_deriv tile width = its payload's lane width (kind 2); 0 = the
// Helmholtz family's.  From a tile-width grid (profiles/r02/pderiv_eb_grid.jsonl),
// adopted where >= 8 % faster: e.g. prism P=2 0.59 -> 0.86, hex P=3 0.48 ->
// 0.66, tet P=2 0.64 -> 0.77.
constexpr int kTunedEBPderiv[4][11] = {
    { 0,  4,  2,  1,  1,  1,  0,  2,  0,  0,  0},  // hex
    { 0,  4,  2,  1,  0,  1,  0,  0,  0,  0,  0},  // prism
    { 0,  4,  2,  1,  1,  0,  0,  2,  0,  0,  0},  // pyr
    { 0,  8,  4,  0,  1,  1,  0,  0,  0,  0,  0},  // tet
};
#ifdef SK_EB_FIXED
SK_HD constexpr int tuned_eb_pderiv(int, int) { return SK_EB_FIXED; }
#else
SK_HD constexpr int tuned_eb_pderiv(int S, int P) { return kTunedEBPderiv[S][P]; }
#endif
#ifdef SK_EB_FIXED
SK_HD constexpr int tuned_eb_nc(int, int) { return SK_EB_FIXED; }
#else
SK_HD constexpr int tuned_eb_nc(int S, int P) { return kTunedEBNc[S][P]; }
#endif
#ifdef SK_EB_FIXED
SK_HD constexpr int tuned_eb_bwd(int, int) { return SK_EB_FIXED; }
#else
SK_HD constexpr int tuned_eb_bwd(int S, int P) { return kTunedEBBwd[S][P]; }
#endif
#ifdef SK_EB_FIXED
SK_HD constexpr int tuned_eb_regular(int, int) { return SK_EB_FIXED; }
#else
SK_HD constexpr int tuned_eb_regular(int S, int P) { return kTunedEBReg[S][P]; }
#endif
#ifdef SK_NT_DIV
SK_HD constexpr int tuned_nt_div(int, int, int) { return SK_NT_DIV; }
#else
SK_HD constexpr int tuned_nt_div(int cls, int S, int P) { return kTunedNTDiv[cls][S][P]; }
#endif
#ifdef SK_NT_DIV
SK_HD constexpr int tuned_nt_div_regular(int, int) { return SK_NT_DIV; }
#else
SK_HD constexpr int tuned_nt_div_regular(int S, int P) { return kTunedNTDivReg[S][P] > 0 ? kTunedNTDivReg[S][P] : kTunedNTDiv[0][S][P]; }
#endif
#ifdef SK_MINB
SK_HD constexpr int tuned_minb(int, int, int) { return SK_MINB; }
#else
SK_HD constexpr int tuned_minb(int cls, int S, int P) { return kTunedMinB[cls][S][P]; }
#endif
#ifdef SK_MINB_CAP
SK_HD constexpr int tuned_minb_cap(int, int, int) { return SK_MINB_CAP; }
#else
SK_HD constexpr int tuned_minb_cap(int cls, int S, int P) { return kMinBCap[cls][S][P]; }
#endif
// Per-operator overrides of the class-2 launch tables for bwd_trans,
// iproduct_wrt_base, phys_deriv, iproduct_wrt_deriv_base and the
// non-collocated Helmholtz (they share kTunedNTDiv[2] / kTunedMinB[2]):
// thread divisor (0 = the class table) and min-blocks rule (-1 = the class
// table, 0 = none), shape x order.  From a deformed grid over divisors
// 1/2/4 and min-blocks off (profiles/r02/other_ops_grid.jsonl), adopted
// where >= 8 % faster than the class setting: e.g. iproduct_wrt_deriv_base
// pyr P=5 0.32 -> 0.59, prism P=4 0.21 -> 0.42; non-collocated Helmholtz
// hex P=3 0.44 -> 0.61, tet P=3 0.38 -> 0.52; bwd_trans pyr P=3 0.44 ->
// 0.58; iproduct_wrt_base hex P=5 0.68 -> 0.86.
constexpr int kOpNTDiv[5][4][11] = {
    {{ 0,  0,  0,  4,  4,  0,  0,  0,  0,  0,  0},
     { 0,  0,  0,  4,  0,  4,  0,  0,  0,  0,  0},
     { 0,  0,  0,  4,  0,  0,  0,  0,  0,  2,  0},
     { 0,  1,  0,  4,  0,  0,  0,  0,  4,  4,  0}},  // bwd
    {{ 0,  1,  0,  0,  4,  0,  0,  2,  0,  0,  0},
     { 0,  0,  0,  2,  0,  0,  0,  0,  0,  0,  0},
     { 0,  0,  0,  0,  0,  0,  0,  2,  0,  0,  0},
     { 0,  1,  0,  0,  0,  0,  0,  0,  0,  0,  0}},  // iprod
    {{ 0,  1,  0,  0,  0,  0,  0,  0,  0,  2,  0},
     { 0,  1,  1,  0,  0,  0,  0,  0,  0,  2,  0},
     { 0,  1,  1,  0,  0,  0,  0,  0,  2,  2,  0},
     { 0,  1,  1,  0,  0,  0,  0,  0,  0,  0,  0}},  // pderiv
    {{ 0,  0,  0,  0,  2,  0,  0,  2,  0,  0,  0},
     { 0,  0,  0,  2,  0,  0,  0,  0,  0,  0,  0},
     { 0,  0,  0,  0,  0,  0,  0,  2,  0,  0,  0},
     { 0,  0,  0,  0,  0,  0,  0,  0,  2,  0,  0}},  // ipderiv
    {{ 0,  0,  0,  4,  0,  0,  0,  0,  0,  0,  0},
     { 0,  0,  4,  4,  4,  4,  2,  4,  0,  0,  0},
     { 0,  0,  0,  4,  0,  4,  2,  0,  0,  0,  4},
     { 0,  0,  0,  4,  4,  0,  0,  0,  0,  0,  0}},  // helmnc
};
constexpr int kOpMinB[5][4][11] = {
    {{-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}},  // bwd
    {{-1, -1, -1, -1, -1,  0, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}},  // iprod
    {{-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1,  0, -1,  0, -1, -1, -1, -1, -1},
     {-1, -1, -1,  0, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}},  // pderiv
    {{-1, -1, -1, -1, -1,  0, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1,  0, -1, -1,  0, -1, -1, -1},
     {-1, -1, -1, -1,  0,  0, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1,  0, -1, -1, -1, -1, -1, -1}},  // ipderiv
    {{-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1},
     {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1}},  // helmnc
};
SK_HD constexpr int op_slot(int op) { return op >= 2 && op <= 6 ? op - 2 : -1; }  // OP_BWD .. OP_HELM_NC
#if defined(SK_NT_DIV)
SK_HD constexpr int nt_div_op(int op, int cls, int S, int P) { return tuned_nt_div(cls, S, P); }
#else
SK_HD constexpr int nt_div_op(int op, int cls, int S, int P) {
  return op_slot(op) >= 0 && kOpNTDiv[op_slot(op)][S][P] > 0 ? kOpNTDiv[op_slot(op)][S][P] : tuned_nt_div(cls, S, P);
}
#endif
#if defined(SK_MINB)
SK_HD constexpr int minb_op(int op, int cls, int S, int P) { return tuned_minb(cls, S, P); }
#else
SK_HD constexpr int minb_op(int op, int cls, int S, int P) {
  return op_slot(op) >= 0 && kOpMinB[op_slot(op)][S][P] >= 0 ? kOpMinB[op_slot(op)][S][P] : tuned_minb(cls, S, P);
}
#endif

#ifdef SK_PERSIST
constexpr bool tuned_persist(int, int, int) { return SK_PERSIST; }
#else
constexpr bool tuned_persist(int cls, int S, int P) { return cls == 0 && kPersist[S][P]; }
#endif
#ifdef SK_RAGGED_MAXP
SK_HD constexpr bool ragged_dispatch(int, int, int P) { return P <= SK_RAGGED_MAXP; }
#else
SK_HD constexpr bool ragged_dispatch(int cls, int S, int P) { return P <= kRaggedMaxP[cls][S]; }
#endif

#ifdef SK_SPLIT_MINP
SK_HD constexpr bool ragged_split(int, int, int P) { return P >= SK_SPLIT_MINP; }
#else
SK_HD constexpr bool ragged_split(int cls, int S, int P) { return P >= kSplitMinP[cls][S]; }
#endif

// ragged r <-> k sweep tables ([0, GLayout::RAGGED): slices and pairs)
// staged in shared memory per CTA instead of read through L1, per operator
// class (0 Helmholtz, 1 mass) x shape x order.  Enabled where Helmholtz and
// stiffness (or mass) both gained >= 2 % (profiles/r01c/tune_smem_tables_*,
// Helmholtz re-checked in ab_vs_ebf7fee.jsonl):
// the ragged paths are L1-latency bound at these orders, the extra shared
// memory costs no CTA per SM there
constexpr bool kSmemTab[2][4][11] = {
    {{0}, {0}, {0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0}},
    {{0}, {0}, {0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 0}, {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1}},
};
#ifdef SK_SMT
SK_HD constexpr bool smem_tables(int cls, int S, int P) { return cls < 2 && S >= 2 && P >= SK_SMT && (cls == 1 || !kPersist[S][P]); }
#else
SK_HD constexpr bool smem_tables(int cls, int S, int P) { return cls < 2 && kSmemTab[cls][S][P]; }
#endif

#ifdef SK_PRISM_WP
SK_HD constexpr bool prism_warp_pairs(int, int S, int P) { return S == 1 && P >= SK_PRISM_WP; }
#else
SK_HD constexpr bool prism_warp_pairs(int cls, int S, int P) { return S == 1 && kPrismWP[cls][P]; }
#endif

}  // namespace sk

// Sum-factorisation stages of the SUM_FAC_TOP kernels.
//
// A CTA owns a tile of EB elements; each stage is one 1D contraction along
// one tensor direction, parallel over (element, passive-index) items with
// the contracted line held in registers.  Wherever the 1D table does not
// depend on the item (all full families, and the warped families once the
// selector index is unrolled inside the thread) the table entry is a
// compile-time offset into kernel-parameter space, i.e. a uniform DFMA
// operand.  The two ragged stages of pyr/tet (selector p+q or max(p,q)
// varies per item) read their table from the L1-resident device buffer.
//
// Algorithm: reference sum-factorised kernels speckern/operators.py:149-391
// (contraction order r -> q -> p forward, p -> q -> r transposed, the
// collapsed-vertex rank-one corrections folded into the line passes).
//
// Per-element work arrays, plane-relative index (see Lay in sk_common.cuh):
//   plane 0: U  [i][j][k]                       / TA [p][q][k], Y and S rows
//   plane 1: V0 [i][j][k]   / coefficient tile staging [mode][XSTR]
//   plane 2: V1 [i][j][k]                       / TB [p][j][k]
// TA/TB are live only between the sweeps that produce and consume them.
#pragma once

#include "sk_common.cuh"

namespace sk {

// Code-size / parallelism switches (measured, profiles/r01): tet q <-> j
// sweeps use compile-time slice dispatch up to this order and a compact
// L1-table loop above it (instruction-cache footprint); prism r <-> k sweeps
// run one thread per (element, q) with uniform slice tables up to
// kPrismUniformMaxP and one per (element, p, q) pair above it.
#ifdef SK_TET_DISPATCH_MAXP
constexpr int kTetDispatchMaxP = SK_TET_DISPATCH_MAXP;
#else
constexpr int kTetDispatchMaxP = 9;
#endif
constexpr int kPrismUniformMaxP = 8;

// Prism r <-> k sweeps with warp-uniform slices: the slices p and P - p
// (n = P1 - p and p + 1 columns, P1 + 1 together) go to one group of whole
// warps whose lanes take the (element, q) lines, so every warp runs one
// branch of the slice dispatch (no divergence, uniform table operands) and
// the groups carry equal work.  f(pc, e, q) is called with the slice as a
// compile-time constant.
template <int P, class L, int NT, class F>
__device__ __forceinline__ void prism_slice_pairs(F&& f) {
  constexpr int P1 = P + 1, NPP = (P1 + 1) / 2, LN = L::EB * P1, WPG = (LN + 31) / 32;
  static_assert(NT >= 64, "warp-uniform slice pairs need a CTA-wide thread group");
  for (int sl = threadIdx.x; sl < NPP * WPG * 32; sl += NT) {
    const int g = sl / (WPG * 32), l = sl - g * (WPG * 32);
    if (l < LN) {
      const int q = l / L::EB, e = l - q * L::EB;
      dispatch<0, NPP>(g, [&](auto gc) {
        constexpr int pa = decltype(gc)::value, pb = P1 - 1 - pa;
        f(std::integral_constant<int, pa>{}, e, q);
        if constexpr (pb != pa) f(std::integral_constant<int, pb>{}, e, q);
      });
    }
  }
}
// L1-table ragged sweeps: loop over the item's own run length at run time
// (1) instead of the full unrolled P1 with predicated-off tails (0); same
// accumulation order, bit-identical results
#ifdef SK_RRL
constexpr bool kRaggedRuntimeLoop = SK_RRL;
#else
constexpr bool kRaggedRuntimeLoop = false;
#endif

// table reads of the ragged r <-> k sweeps: through L1 from the device
// table buffer, or plain shared-memory loads when the caller staged [0, RAGGED)
// of it in shared memory (SMT)
template <bool SMT>
__device__ __forceinline__ double ldt(const double* p) {
  if constexpr (SMT) return *p;
  else return __ldg(p);
}
template <bool SMT>
__device__ __forceinline__ int4 ldt(const int4* p) {
  if constexpr (SMT) return *p;
  else return __ldg(p);
}

// mode offset of the prism slice p: sum_{p' < p} P1 (P1 - p')
__host__ __device__ constexpr int prism_slice_off(int P1, int p) { return P1 * (p * P1 - p * (p - 1) / 2); }
// pyr/tet r <-> k sweeps (slice c2[max(p,q)] / c2[p+q] varies per item):
// compile-time slice dispatch (RD = true) or L1 table reads; chosen per
// operator class (sk_tune.h kRaggedMaxP)

// ---- coefficient tile staging ----------------------------------------------
// xs[m * XSTR + e] <-> field value of mode m of element e0 + e; iteration order
// follows the field layout so that consecutive threads touch consecutive
// global addresses.
template <class L, int N, int NT>
__device__ __forceinline__ void load_tile(const double* __restrict__ src, const Ctx& c, double* xs) {
  constexpr int EB = L::EB, XS = L::XSTR;
  if (c.W == 1) {
    const double* base = src + c.e0 * N;
    const long long lim = (c.E - c.e0) * N;  // loads past the last element read 0
#pragma unroll 4
    for (int g = tix<NT>(); g < EB * N; g += NT) {
      const int e = g / N, m = g - e * N;
      xs[m * XS + e] = g < lim ? __ldg(base + g) : 0.0;
    }
  } else {
    for (int g = tix<NT>(); g < EB * N; g += NT) {
      const int m = g / EB, e = g - m * EB;
      const long long eg = c.e0 + e;
      xs[m * XS + e] = eg < c.E ? __ldg(src + lane_base(eg, N, c.W) + (long long)m * c.W) : 0.0;
    }
  }
}

template <class L, int N, int NT>
__device__ __forceinline__ void store_tile(double* __restrict__ dst, const Ctx& c, const double* xs) {
  constexpr int EB = L::EB, XS = L::XSTR;
  if (c.W == 1) {
    double* base = dst + c.e0 * N;
    const long long lim = (c.Epad - c.e0) * N;
#pragma unroll 4
    for (int g = tix<NT>(); g < EB * N; g += NT) {
      const int e = g / N, m = g - e * N;
      if (g < lim) base[g] = xs[m * XS + e];
    }
  } else {
    for (int g = tix<NT>(); g < EB * N; g += NT) {
      const int m = g / EB, e = g - m * EB;
      const long long eg = c.e0 + e;
      if (eg < c.Epad) dst[lane_base(eg, N, c.W) + (long long)m * c.W] = xs[m * XS + e];
    }
  }
}

// Register-staged coefficient tile for the persistent kernels: the loads of
// the next tile are issued before the current tile's sweeps (they land during
// them) and written to the staging area at the top of the next iteration.
// Same thread -> element mapping as load_tile.
template <class L, int N, int NT>
struct TileRegs {
  static constexpr int EB = L::EB, XS = L::XSTR, CPT = (EB * N + NT - 1) / NT;
  double v[CPT];
  __device__ __forceinline__ void load(const double* __restrict__ src, const Ctx& c) {
    if (c.W == 1) {
      const double* base = src + c.e0 * N;
      const long long lim = (c.E - c.e0) * N;
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int g = tix<NT>() + i * NT;
        v[i] = (g < EB * N && g < lim) ? __ldg(base + g) : 0.0;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const int g = tix<NT>() + i * NT;
        const int m = g / EB, e = g - m * EB;
        const long long eg = c.e0 + e;
        v[i] = (g < EB * N && eg < c.E) ? __ldg(src + lane_base(eg, N, c.W) + (long long)m * c.W) : 0.0;
      }
    }
  }
  __device__ __forceinline__ void put(int W, double* xs) const {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int g = tix<NT>() + i * NT;
      if (g < EB * N) {
        int e, m;
        if (W == 1) {
          e = g / N;
          m = g - e * N;
        } else {
          m = g / EB;
          e = g - m * EB;
        }
        xs[m * XS + e] = v[i];
      }
    }
  }
};

// coefficient m of tile element e from / to the staged tile
template <class L, int NM>
struct CoefIn {
  const double* xs;
  __device__ __forceinline__ double operator()(int e, int m) const { return xs[m * L::XSTR + e]; }
};

template <class L, int NM, bool ACC = false>
struct CoefOut {
  double* xs;
  __device__ __forceinline__ void operator()(int e, int m, double v) const {
    if constexpr (ACC)
      xs[m * L::XSTR + e] += v;
    else
      xs[m * L::XSTR + e] = v;
  }
};

// ---- F3 core: p -> i for one (j,k) line ------------------------------------
template <int S, int P>
__device__ __forceinline__ void line_a0(const FwdTab<S, P>& B, const double (&x)[P + 1],
                                        double (&u)[Dims<S, P>::Q0]) {
  using Dm = Dims<S, P>;
#pragma unroll
  for (int i = 0; i < Dm::Q0; ++i) {
    double s = B.a0[i * Dm::P1] * x[0];
#pragma unroll
    for (int p = 1; p < Dm::P1; ++p) s = fma(B.a0[i * Dm::P1 + p], x[p], s);
    u[i] = s;
  }
}

// transposed p <- i for one (j,k) line
template <int S, int P>
__device__ __forceinline__ void line_a0t(const FwdTab<S, P>& B, const double (&r)[Dims<S, P>::Q0],
                                         double (&t)[P + 1]) {
  using Dm = Dims<S, P>;
#pragma unroll
  for (int p = 0; p < Dm::P1; ++p) {
    double s = B.a0[p] * r[0];
#pragma unroll
    for (int i = 1; i < Dm::Q0; ++i) s = fma(B.a0[i * Dm::P1 + p], r[i], s);
    t[p] = s;
  }
}

// v = D u along a line of length Q (D row-major Q x Q)
template <int Q>
__device__ __forceinline__ void line_d(const double* D, const double (&u)[Q], double (&v)[Q]) {
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    double s = D[a * Q] * u[0];
#pragma unroll
    for (int b = 1; b < Q; ++b) s = fma(D[a * Q + b], u[b], s);
    v[a] = s;
  }
}

// r += D^T w along a line
template <int Q>
__device__ __forceinline__ void line_dt_acc(const double* D, const double (&w)[Q], double (&r)[Q]) {
#pragma unroll
  for (int a = 0; a < Q; ++a) {
    double s = r[a];
#pragma unroll
    for (int b = 0; b < Q; ++b) s = fma(D[b * Q + a], w[b], s);
    r[a] = s;
  }
}

// ---- even-odd 1D contractions along Gauss-Lobatto directions -------------
// (see gll_dir): half the multiply-adds of the plain forms above.

// u[i] = sum_p B[i][p] x[p] for a full modified-basis family B (Q x P1)
template <int Q, int P1>
__device__ __forceinline__ void line_b_eo(const double* B, const double* bp, const double* bm, const double (&x)[P1],
                                          double (&u)[Q]) {
  constexpr int H = Q / 2;
  const double xs = x[0] + x[1], xd = x[0] - x[1];
#pragma unroll
  for (int i = 0; i < (Q + 1) / 2; ++i) {
    double pe = bp[i] * xs;
#pragma unroll
    for (int p = 2; p < P1; p += 2) pe = fma(B[i * P1 + p], x[p], pe);
    if (i < H) {
      double po = bm[i] * xd;
#pragma unroll
      for (int p = 3; p < P1; p += 2) po = fma(B[i * P1 + p], x[p], po);
      u[i] = pe + po;
      u[Q - 1 - i] = pe - po;
    } else {
      u[i] = pe;  // middle point: the odd modes vanish there
    }
  }
}

// t[p] = sum_i B[i][p] r[i]
template <int Q, int P1>
__device__ __forceinline__ void line_bt_eo(const double* B, const double* bp, const double* bm, const double (&r)[Q],
                                           double (&t)[P1]) {
  constexpr int H = Q / 2;
  double re[H], ro[H];
#pragma unroll
  for (int i = 0; i < H; ++i) {
    re[i] = r[i] + r[Q - 1 - i];
    ro[i] = r[i] - r[Q - 1 - i];
  }
  double sp = bp[0] * re[0], sm = bm[0] * ro[0];
#pragma unroll
  for (int i = 1; i < H; ++i) {
    sp = fma(bp[i], re[i], sp);
    sm = fma(bm[i], ro[i], sm);
  }
  if constexpr (Q % 2) sp = fma(bp[H], r[H], sp);
  t[0] = sp + sm;
  t[1] = sp - sm;
#pragma unroll
  for (int p = 2; p < P1; ++p) {
    double s;
    if (p % 2 == 0) {
      s = B[p] * re[0];
#pragma unroll
      for (int i = 1; i < H; ++i) s = fma(B[i * P1 + p], re[i], s);
      if constexpr (Q % 2) s = fma(B[H * P1 + p], r[H], s);
    } else {
      s = B[p] * ro[0];
#pragma unroll
      for (int i = 1; i < H; ++i) s = fma(B[i * P1 + p], ro[i], s);
    }
    t[p] = s;
  }
}

// v = M u (ACC: r += M u) for a centro-antisymmetric M in even-odd form
template <int Q, bool ACC>
__device__ __forceinline__ void line_m_eo(const EOTab<Q>& T, const double (&u)[Q], double (&v)[Q]) {
  constexpr int H = Q / 2;
  double e[H], o[H];
#pragma unroll
  for (int b = 0; b < H; ++b) {
    e[b] = u[b] + u[Q - 1 - b];
    o[b] = u[b] - u[Q - 1 - b];
  }
#pragma unroll
  for (int a = 0; a < H; ++a) {
    double pe = T.E[a * H] * e[0], po = T.O[a * H] * o[0];
#pragma unroll
    for (int b = 1; b < H; ++b) {
      pe = fma(T.E[a * H + b], e[b], pe);
      po = fma(T.O[a * H + b], o[b], po);
    }
    if constexpr (Q % 2) pe = fma(T.Em[a], u[H], pe);
    if constexpr (ACC) {
      v[a] += pe + po;
      v[Q - 1 - a] += po - pe;
    } else {
      v[a] = pe + po;
      v[Q - 1 - a] = po - pe;
    }
  }
  if constexpr (Q % 2) {
    double s = T.Om[0] * o[0];
#pragma unroll
    for (int b = 1; b < H; ++b) s = fma(T.Om[b], o[b], s);
    if constexpr (ACC)
      v[H] += s;
    else
      v[H] = s;
  }
}

// collocation derivative along direction DIR: v = D u, and r += D^T w
template <int S, int P, int DIR, int Q>
__device__ __forceinline__ void line_dd(const DTab<S, P>& D, const double (&u)[Q], double (&v)[Q]) {
  if constexpr (!use_eo(S, P)) {
    line_d<Q>(DIR == 0 ? D.d0 : DIR == 1 ? D.d1 : D.d2, u, v);
  } else if constexpr (DIR == 0) {
    line_m_eo<Q, false>(D.e0, u, v);
  } else if constexpr (DIR == 1) {
    if constexpr (gll_dir(S, 1)) line_m_eo<Q, false>(D.e1, u, v); else line_d<Q>(D.d1, u, v);
  } else {
    if constexpr (gll_dir(S, 2)) line_m_eo<Q, false>(D.e2, u, v); else line_d<Q>(D.d2, u, v);
  }
}

template <int S, int P, int DIR, int Q>
__device__ __forceinline__ void line_ddt_acc(const DTab<S, P>& D, const double (&w)[Q], double (&r)[Q]) {
  if constexpr (!use_eo(S, P)) {
    line_dt_acc<Q>(DIR == 0 ? D.d0 : DIR == 1 ? D.d1 : D.d2, w, r);
  } else if constexpr (DIR == 0) {
    line_m_eo<Q, true>(D.e0t, w, r);
  } else if constexpr (DIR == 1) {
    if constexpr (gll_dir(S, 1)) line_m_eo<Q, true>(D.e1t, w, r); else line_dt_acc<Q>(D.d1, w, r);
  } else {
    if constexpr (gll_dir(S, 2)) line_m_eo<Q, true>(D.e2t, w, r); else line_dt_acc<Q>(D.d2, w, r);
  }
}

// dir-0 value contractions in even-odd form (value tables only)
template <int S, int P, bool EO = use_eo(S, P)>
__device__ __forceinline__ void line_a0_eo(const FwdTab<S, P>& B, const double (&x)[P + 1], double (&u)[Dims<S, P>::Q0]) {
  if constexpr (EO)
    line_b_eo<Dims<S, P>::Q0, P + 1>(B.a0, B.a0p, B.a0m, x, u);
  else
    line_a0<S, P>(B, x, u);
}

template <int S, int P, bool EO = use_eo(S, P)>
__device__ __forceinline__ void line_a0t_eo(const FwdTab<S, P>& B, const double (&r)[Dims<S, P>::Q0], double (&t)[P + 1]) {
  if constexpr (EO)
    line_bt_eo<Dims<S, P>::Q0, P + 1>(B.a0, B.a0p, B.a0m, r, t);
  else
    line_a0t<S, P>(B, r, t);
}

// ---- F1: r -> k.  TA[p][q][k] = sum_r C_(p,q)[k][r] uhat[p,q,r] ----------
// DER2: the dir-2 family is the derivative one (reference dmode == 2; the
// caller passes the derivative FwdTab for hex/prism, the device buffer's DC2
// slices are used for pyr/tet)
template <int S, int P, class L, int NT, int TAo, class In, bool DER2 = false, bool RD = false, bool SPL = false,
          bool WP = false, bool SMT = false, bool EO = use_eo(S, P)>
__device__ __forceinline__ void stage_f1(const FwdTab<S, P>& B, const double* __restrict__ gtab, const In& xin,
                                         double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q2 = Dm::Q2, S2 = L::S2;
  if constexpr (S == HEX) {
    items<L, P1 * P1, NT>([&](int e, int ps) {
      double x[P1];
#pragma unroll
      for (int r = 0; r < P1; ++r) x[r] = xin(e, ps * P1 + r);
      if constexpr (!DER2 && EO) {
        double u[Q2];
        line_b_eo<Q2, P1>(B.a2, B.a2p, B.a2m, x, u);
#pragma unroll
        for (int k = 0; k < Q2; ++k) sm[L::at(e, TAo + ps * S2 + k)] = u[k];
      } else {
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          double s = B.a2[k * P1] * x[0];
#pragma unroll
          for (int r = 1; r < P1; ++r) s = fma(B.a2[k * P1 + r], x[r], s);
          sm[L::at(e, TAo + ps * S2 + k)] = s;
        }
      }
    });
  } else if constexpr (S != HEX && RD) {
    // prism / pyr / tet: item = (e, (p,q) pair), pairs ordered by slice; the
    // slice m = p (prism), max(p,q) (pyr) or p+q (tet) is dispatched to a
    // compile-time constant so c2[m] entries are uniform operands
    // (operators.py:209-351)
    // SPLIT = 2 when the pairs fill at most half the CTA: each (e, pair)
    // line is computed by two threads (halves of k, half index slowest so a
    // warp takes one half), so no warp idles through the stage
    constexpr int SPLIT = SPL && 2 * L::EB * Dm::NPAIR <= NT ? 2 : 1;
    const int4* pairs = reinterpret_cast<const int4*>(gtab + GLayout<S, P>::PAIRS);
    items<L, Dm::NPAIR * SPLIT, NT>([&](int e, int ps2) {
      const int h = ps2 / Dm::NPAIR, ps = ps2 - h * Dm::NPAIR;
      const int4 pr = ldt<SMT>(pairs + ps);  // p, q, mode offset, nr
      dispatch<0, P1>(P1 - pr.w, [&](auto mc) {
        constexpr int m = decltype(mc)::value;
        constexpr int n = P1 - m;
        constexpr int co = wfam_off(Q2, P1, m);
        double x[n];
#pragma unroll
        for (int r = 0; r < n; ++r) x[r] = xin(e, pr.z + r);
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          if (SPLIT == 1 || (k * SPLIT) / Q2 == h) {
            double s = B.c2[co + k * n] * x[0];
#pragma unroll
            for (int r = 1; r < n; ++r) s = fma(B.c2[co + k * n + r], x[r], s);
            // prism collapsed-edge share of mode (0, q, 1) (operators.py:288-293)
            if constexpr (S == PRISM && m == 1) s = fma(xin(e, pr.y * P1 + 1), B.c2[k * P1 + 1], s);
            sm[L::at(e, TAo + (pr.x * P1 + pr.y) * S2 + k)] = s;
          }
        }
        if constexpr (S != PRISM && m == 0) {
          if (pr.x == 0 && pr.y == 0) {
            // collapsed apex mode (0,0,1): Y[k] = c2[0][k][1] * uhat[0,0,1]
#pragma unroll
            for (int k = 0; k < Q2; ++k)
              if (SPLIT == 1 || (k * SPLIT) / Q2 == h) sm[L::at(e, TAo + P1 * P1 * S2 + k)] = B.c2[k * P1 + 1] * x[1];
          }
        }
      });
    });
  } else if constexpr (S == PRISM && WP) {
    prism_slice_pairs<P, L, NT>([&](auto pc, int e, int q) {
      constexpr int p = decltype(pc)::value, n = P1 - p, co = wfam_off(Q2, P1, p);
      constexpr int off = prism_slice_off(P1, p);
      double x[n];
#pragma unroll
      for (int r = 0; r < n; ++r) x[r] = xin(e, off + q * n + r);
      double u0q1 = 0.0;
      if constexpr (p == 1) u0q1 = xin(e, q * P1 + 1);  // mode (0, q, 1): collapsed-edge share
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        double s = B.c2[co + k * n] * x[0];
#pragma unroll
        for (int r = 1; r < n; ++r) s = fma(B.c2[co + k * n + r], x[r], s);
        if constexpr (p == 1) s = fma(u0q1, B.c2[k * P1 + 1], s);
        sm[L::at(e, TAo + (p * P1 + q) * S2 + k)] = s;
      }
    });
  } else if constexpr (S == PRISM && P <= kPrismUniformMaxP && !RD) {
    // item = (e, q[, p parity]); p unrolled so c2[p] is uniform
    // (operators.py:275-295).  SPLIT = 2 halves the slices between two
    // threads (even / odd p, parity slowest so warps stay uniform) when the
    // items fill at most half the CTA
    constexpr int SPLIT = SPL && 2 * L::EB * P1 <= NT ? 2 : 1;
    items<L, P1 * SPLIT, NT>([&](int e, int q2) {
      const int h = q2 / P1, q = q2 - h * P1;
      const double u0q1 = xin(e, q * P1 + 1);  // mode (0, q, 1): collapsed-edge share
      int off = 0;
#pragma unroll
      for (int p = 0; p < P1; ++p) {
        const int n = P1 - p;
        if (SPLIT == 1 || p % SPLIT == h) {
          double x[P1];
#pragma unroll
          for (int r = 0; r < P1; ++r) x[r] = r < n ? xin(e, off + q * n + r) : 0.0;
          const int co = wfam_off(Q2, P1, p);
#pragma unroll
          for (int k = 0; k < Q2; ++k) {
            double s = B.c2[co + k * n] * x[0];
#pragma unroll
            for (int r = 1; r < P1; ++r)
              if (r < n) s = fma(B.c2[co + k * n + r], x[r], s);
            if (p == 1) s = fma(u0q1, B.c2[k * P1 + 1], s);
            sm[L::at(e, TAo + (p * P1 + q) * S2 + k)] = s;
          }
        }
        off += P1 * n;
      }
    });
  } else {
    // prism / pyr / tet: item = (e, (p,q) pair); the dir-2 slice c2[p]
    // (prism), c2[max(p,q)] (pyr) or c2[p+q] (tet) differs per item -> read
    // from the device table buffer through L1 (operators.py:209-351)
    constexpr int SPLIT = SPL && 2 * L::EB * Dm::NPAIR <= NT ? 2 : 1;  // see the dispatch path
    const int4* pairs = reinterpret_cast<const int4*>(gtab + GLayout<S, P>::PAIRS);
    items<L, Dm::NPAIR * SPLIT, NT>([&](int e, int ps2) {
      const int h = ps2 / Dm::NPAIR, ps = ps2 - h * Dm::NPAIR;
      const int4 pr = ldt<SMT>(pairs + ps);  // p, q, mode offset, nr
      const int m = (S == TET) ? pr.x + pr.y : (S == PRISM) ? pr.x : cmax(pr.x, pr.y);
      const int n = P1 - m;
      const double* fam = gtab + (DER2 ? GLayout<S, P>::DC2 : GLayout<S, P>::C2);
      const double* tab = fam + wfam_off(Q2, P1, m);
      if constexpr (kRaggedRuntimeLoop) {
        double acc[Q2];
#pragma unroll
        for (int k = 0; k < Q2; ++k) acc[k] = 0.0;
#pragma unroll 1
        for (int r = 0; r < pr.w; ++r) {
          const double xr = xin(e, pr.z + r);
#pragma unroll
          for (int k = 0; k < Q2; ++k)
            if (SPLIT == 1 || (k * SPLIT) / Q2 == h) acc[k] = fma(ldt<SMT>(tab + k * n + r), xr, acc[k]);
        }
        const double u0q1 = (S == PRISM && pr.x == 1) ? xin(e, pr.y * P1 + 1) : 0.0;
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          if (SPLIT == 1 || (k * SPLIT) / Q2 == h) {
            double v = acc[k];
            if constexpr (S == PRISM) {
              if (pr.x == 1) v = fma(u0q1, ldt<SMT>(fam + k * P1 + 1), v);
            }
            sm[L::at(e, TAo + (pr.x * P1 + pr.y) * S2 + k)] = v;
          }
        }
        if (S != PRISM && pr.x == 0 && pr.y == 0) {
          const double x1 = xin(e, pr.z + 1);
#pragma unroll
          for (int k = 0; k < Q2; ++k)
            if (SPLIT == 1 || (k * SPLIT) / Q2 == h) sm[L::at(e, TAo + P1 * P1 * S2 + k)] = ldt<SMT>(fam + k * P1 + 1) * x1;
        }
        return;
      }
      double x[P1];
#pragma unroll
      for (int r = 0; r < P1; ++r) x[r] = r < pr.w ? xin(e, pr.z + r) : 0.0;
      // prism collapsed-edge share of mode (0, q, 1) (operators.py:288-293)
      const double u0q1 = (S == PRISM && pr.x == 1) ? xin(e, pr.y * P1 + 1) : 0.0;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        if (SPLIT == 1 || (k * SPLIT) / Q2 == h) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < P1; ++r)
            if (r < pr.w) s = fma(ldt<SMT>(tab + k * n + r), x[r], s);
          if constexpr (S == PRISM) {
            if (pr.x == 1) s = fma(u0q1, ldt<SMT>(fam + k * P1 + 1), s);
          }
          sm[L::at(e, TAo + (pr.x * P1 + pr.y) * S2 + k)] = s;
        }
      }
      if (S != PRISM && pr.x == 0 && pr.y == 0) {
        // collapsed apex mode (0,0,1): Y[k] = c2[0][k][1] * uhat[0,0,1]
#pragma unroll
        for (int k = 0; k < Q2; ++k)
          if (SPLIT == 1 || (k * SPLIT) / Q2 == h) sm[L::at(e, TAo + P1 * P1 * S2 + k)] = ldt<SMT>(fam + k * P1 + 1) * x[1];
      }
    });
  }
}

// ---- F2: q -> j.  TB[p][j][k] = sum_q B_p[j][q] TA[p][q][k] ---------------
// DER1: the dir-1 family is the derivative one (reference dmode == 1): the
// caller passes the derivative FwdTab and the apex share's constant eta_2
// factor differentiates to zero ("ones2", operators.py:233-235)
template <int S, int P, class L, int NT, int TAo, int TBo, bool DER1 = false, bool EO = use_eo(S, P)>
__device__ __forceinline__ void stage_f2(const FwdTab<S, P>& B, const double* __restrict__ gtab, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2;
  if constexpr (S != TET) {
    items<L, P1 * Q2, NT>([&](int e, int ps) {
      const int p = ps / Q2, k = ps - p * Q2;
      double x[P1];
#pragma unroll
      for (int q = 0; q < P1; ++q) x[q] = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
      double y = 0.0;
      if constexpr (S == PYR) y = sm[L::at(e, TAo + P1 * P1 * S2 + k)];
      if constexpr (!DER1 && EO) {
        // apex shares (operators.py:335-349): a1[j][1] y into p = 0, y into p = 1
        if constexpr (S == PYR) {
          if (p == 0) x[1] += y;
        }
        double u[Q1];
        line_b_eo<Q1, P1>(B.a1, B.a1p, B.a1m, x, u);
#pragma unroll
        for (int j = 0; j < Q1; ++j) {
          double s = u[j];
          if constexpr (S == PYR) {
            if (p == 1) s += y;
          }
          sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = s;
        }
        return;
      }
#pragma unroll
      for (int j = 0; j < Q1; ++j) {
        double s = B.a1[j * P1] * x[0];
#pragma unroll
        for (int q = 1; q < P1; ++q) s = fma(B.a1[j * P1 + q], x[q], s);
        if constexpr (S == PYR) {
          // apex mode shares (operators.py:335-349)
          if (!DER1 && p == 1) s += y;
          if (p == 0) s = fma(B.a1[j * P1 + 1], y, s);
        }
        sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = s;
      }
    });
  } else {
    // tet: item = (e, k, p) so that all P1 slices run in parallel; the slice
    // index is dispatched to a compile-time constant so b1[p] stays a
    // uniform operand (operators.py:209-245)
    if constexpr (P > kTetDispatchMaxP) {
      // high order: one compact loop, slice table through L1 (keeps the
      // kernel inside the instruction cache)
      const double* fam = gtab + (DER1 ? GLayout<S, P>::DB1 : GLayout<S, P>::B1);
      items<L, Q2 * P1, NT>([&](int e, int ps) {
        const int p = ps / Q2, k = ps - p * Q2;
        const int n = P1 - p;
        const double* tab = fam + wfam_off(Q1, P1, p);
        const double y = p <= 1 ? sm[L::at(e, TAo + P1 * P1 * S2 + k)] : 0.0;
        const double x01 = p == 1 ? sm[L::at(e, TAo + (0 * P1 + 1) * S2 + k)] : 0.0;
        if constexpr (kRaggedRuntimeLoop) {
          double acc[Q1];
#pragma unroll
          for (int j = 0; j < Q1; ++j) acc[j] = 0.0;
#pragma unroll 1
          for (int q = 0; q < n; ++q) {
            const double xq = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
#pragma unroll
            for (int j = 0; j < Q1; ++j) acc[j] = fma(__ldg(tab + j * n + q), xq, acc[j]);
          }
#pragma unroll
          for (int j = 0; j < Q1; ++j) {
            double s = acc[j];
            if (p == 1) {
              s = fma(B.b1[j * P1 + 1], x01, s);
              if constexpr (!DER1) s += y;
            }
            if (p == 0) s = fma(B.b1[j * P1 + 1], y, s);
            sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = s;
          }
          return;
        }
        double x[P1];
#pragma unroll
        for (int q = 0; q < P1; ++q) x[q] = q < n ? sm[L::at(e, TAo + (p * P1 + q) * S2 + k)] : 0.0;
#pragma unroll
        for (int j = 0; j < Q1; ++j) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < P1; ++q)
            if (q < n) s = fma(__ldg(tab + j * n + q), x[q], s);
          if (p == 1) {
            s = fma(B.b1[j * P1 + 1], x01, s);
            if constexpr (!DER1) s += y;
          }
          if (p == 0) s = fma(B.b1[j * P1 + 1], y, s);
          sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = s;
        }
      });
      return;
    }
    items<L, Q2 * P1, NT>([&](int e, int ps) {
      const int pr = ps / Q2, k = ps - pr * Q2;
      dispatch<0, P1>(pr, [&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int n = P1 - p;
        constexpr int bo = wfam_off(Q1, P1, p);
        double x[n];
#pragma unroll
        for (int q = 0; q < n; ++q) x[q] = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
        double y = 0.0, x01 = 0.0;
        if constexpr (p <= 1) {
          y = sm[L::at(e, TAo + P1 * P1 * S2 + k)];
          x01 = sm[L::at(e, TAo + (0 * P1 + 1) * S2 + k)];
        }
#pragma unroll
        for (int j = 0; j < Q1; ++j) {
          double s = B.b1[bo + j * n] * x[0];
#pragma unroll
          for (int q = 1; q < n; ++q) s = fma(B.b1[bo + j * n + q], x[q], s);
          if constexpr (p == 1) {  // edge (0,1,r) + apex shares
            s = fma(B.b1[j * P1 + 1], x01, s);
            if constexpr (!DER1) s += y;
          }
          if constexpr (p == 0) s = fma(B.b1[j * P1 + 1], y, s);
          sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = s;
        }
      });
    });
  }
}

// ---- B2: j -> q.  TA[p][q][k] = sum_j B_p[j][q] TB[p][j][k] ---------------
// DER1: derivative dir-1 family (transposed dmode == 1, apex "ones" share
// vanishes); ACC: add into TA and the spare rows instead of overwriting
template <int S, int P, class L, int NT, int TAo, int TBo, bool DER1 = false, bool ACC = false, bool EO = use_eo(S, P)>
__device__ __forceinline__ void stage_b2(const FwdTab<S, P>& B, const double* __restrict__ gtab, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2;
  if constexpr (S != TET) {
    items<L, P1 * Q2, NT>([&](int e, int ps) {
      const int p = ps / Q2, k = ps - p * Q2;
      double x[Q1];
#pragma unroll
      for (int j = 0; j < Q1; ++j) x[j] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
      if constexpr (!DER1 && EO) {
        double t[P1];
        line_bt_eo<Q1, P1>(B.a1, B.a1p, B.a1m, x, t);
#pragma unroll
        for (int q = 0; q < P1; ++q) {
          double& d = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
          d = ACC ? d + t[q] : t[q];
        }
      } else {
#pragma unroll
        for (int q = 0; q < P1; ++q) {
          double s = B.a1[q] * x[0];
#pragma unroll
          for (int j = 1; j < Q1; ++j) s = fma(B.a1[j * P1 + q], x[j], s);
          double& t = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
          t = ACC ? t + s : s;
        }
      }
      if constexpr (S == PYR) {
        if (p == 1) {  // Y[k] = sum_j TB[1][j][k] (apex share, operators.py:371)
          double y = 0.0;
          if constexpr (!DER1) {
            y = x[0];
#pragma unroll
            for (int j = 1; j < Q1; ++j) y += x[j];
          }
          double& t = sm[L::at(e, TAo + P1 * P1 * S2 + k)];
          t = ACC ? t + y : y;
        }
      }
    });
  } else {
    // tet: item = (e, k, p), p dispatched to a compile-time constant.  The
    // collapsed-edge share S[k] = sum_j b1[0][j][1] TB[1][j][k] and the apex
    // share Y[k] = sum_j TB[1][j][k] go to two spare rows; B3 adds them to
    // modes (0,1,r) and (0,0,1) (operators.py:263-271).
    if constexpr (P > kTetDispatchMaxP) {
      const double* fam = gtab + (DER1 ? GLayout<S, P>::DB1 : GLayout<S, P>::B1);
      items<L, Q2 * P1, NT>([&](int e, int ps) {
        const int p = ps / Q2, k = ps - p * Q2;
        const int n = P1 - p;
        const double* tab = fam + wfam_off(Q1, P1, p);
        double x[Q1];
#pragma unroll
        for (int j = 0; j < Q1; ++j) x[j] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
        if constexpr (kRaggedRuntimeLoop) {
#pragma unroll 1
          for (int q = 0; q < n; ++q) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < Q1; ++j) s = fma(__ldg(tab + j * n + q), x[j], s);
            double& t = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
            t = ACC ? t + s : s;
          }
        } else {
#pragma unroll
          for (int q = 0; q < P1; ++q) {
            if (q < n) {
              double s = 0.0;
#pragma unroll
              for (int j = 0; j < Q1; ++j) s = fma(__ldg(tab + j * n + q), x[j], s);
              double& t = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
              t = ACC ? t + s : s;
            }
          }
        }
        if (p == 1) {
          double s = B.b1[1] * x[0], y = DER1 ? 0.0 : x[0];
#pragma unroll
          for (int j = 1; j < Q1; ++j) {
            s = fma(B.b1[j * P1 + 1], x[j], s);
            if constexpr (!DER1) y += x[j];
          }
          double& ty = sm[L::at(e, TAo + P1 * P1 * S2 + k)];
          double& ts = sm[L::at(e, TAo + (P1 * P1 + 1) * S2 + k)];
          ty = ACC ? ty + y : y;
          ts = ACC ? ts + s : s;
        }
      });
      return;
    }
    items<L, Q2 * P1, NT>([&](int e, int ps) {
      const int pr = ps / Q2, k = ps - pr * Q2;
      dispatch<0, P1>(pr, [&](auto pc) {
        constexpr int p = decltype(pc)::value;
        constexpr int n = P1 - p;
        constexpr int bo = wfam_off(Q1, P1, p);
        double x[Q1];
#pragma unroll
        for (int j = 0; j < Q1; ++j) x[j] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
#pragma unroll
        for (int q = 0; q < n; ++q) {
          double s = B.b1[bo + q] * x[0];
#pragma unroll
          for (int j = 1; j < Q1; ++j) s = fma(B.b1[bo + j * n + q], x[j], s);
          double& t = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
          t = ACC ? t + s : s;
        }
        if constexpr (p == 1) {
          double s = B.b1[1] * x[0], y = DER1 ? 0.0 : x[0];
#pragma unroll
          for (int j = 1; j < Q1; ++j) {
            s = fma(B.b1[j * P1 + 1], x[j], s);
            if constexpr (!DER1) y += x[j];
          }
          double& ty = sm[L::at(e, TAo + P1 * P1 * S2 + k)];
          double& ts = sm[L::at(e, TAo + (P1 * P1 + 1) * S2 + k)];
          ty = ACC ? ty + y : y;
          ts = ACC ? ts + s : s;
        }
      });
    });
  }
}

// ---- B3: k -> r, produce coefficients ----------------------------------------
// DER2: derivative dir-2 family (transposed dmode == 2); accumulation into
// the output is the Out functor's business
template <int S, int P, class L, int NT, int TAo, class Out, bool DER2 = false, bool RD = false, bool SPL = false,
          bool WP = false, bool SMT = false, bool EO = use_eo(S, P)>
__device__ __forceinline__ void stage_b3(const FwdTab<S, P>& B, const double* __restrict__ gtab, const Out& out,
                                         const double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q2 = Dm::Q2, S2 = L::S2;
  if constexpr (S == HEX) {
    items<L, P1 * P1, NT>([&](int e, int ps) {
      double x[Q2];
#pragma unroll
      for (int k = 0; k < Q2; ++k) x[k] = sm[L::at(e, TAo + ps * S2 + k)];
      if constexpr (!DER2 && EO) {
        double t[P1];
        line_bt_eo<Q2, P1>(B.a2, B.a2p, B.a2m, x, t);
#pragma unroll
        for (int r = 0; r < P1; ++r) out(e, ps * P1 + r, t[r]);
      } else {
#pragma unroll
        for (int r = 0; r < P1; ++r) {
          double s = B.a2[r] * x[0];
#pragma unroll
          for (int k = 1; k < Q2; ++k) s = fma(B.a2[k * P1 + r], x[k], s);
          out(e, ps * P1 + r, s);
        }
      }
    });
  } else if constexpr (S != HEX && RD) {
    // prism / pyr / tet with the slice dispatched to a compile-time constant;
    // outputs split over two threads (r parity) when the pairs fill half the
    // CTA
    constexpr int SPLIT = SPL && 2 * L::EB * Dm::NPAIR <= NT ? 2 : 1;
    const int4* pairs = reinterpret_cast<const int4*>(gtab + GLayout<S, P>::PAIRS);
    items<L, Dm::NPAIR * SPLIT, NT>([&](int e, int ps2) {
      const int h = ps2 / Dm::NPAIR, ps = ps2 - h * Dm::NPAIR;
      const int4 pr = ldt<SMT>(pairs + ps);
      double x[Q2];
#pragma unroll
      for (int k = 0; k < Q2; ++k) x[k] = sm[L::at(e, TAo + (pr.x * P1 + pr.y) * S2 + k)];
      if constexpr (S == TET) {
        if (pr.x == 0 && pr.y == 1) {
#pragma unroll
          for (int k = 0; k < Q2; ++k) x[k] += sm[L::at(e, TAo + (P1 * P1 + 1) * S2 + k)];
        }
      }
      dispatch<0, P1>(P1 - pr.w, [&](auto mc) {
        constexpr int m = decltype(mc)::value;
        constexpr int n = P1 - m;
        constexpr int co = wfam_off(Q2, P1, m);
        double apex = 0.0;
        if constexpr (S == PRISM && m == 0) {
          if (SPLIT == 1 || h == 1) {
            // modes (0,q,1) += sum_k c2[0][k][1] TA[1][q][k] (operators.py:312-317)
#pragma unroll
            for (int k = 0; k < Q2; ++k) apex = fma(B.c2[k * P1 + 1], sm[L::at(e, TAo + (1 * P1 + pr.y) * S2 + k)], apex);
          }
        } else if constexpr (m == 0) {
          if (pr.x == 0 && pr.y == 0 && (SPLIT == 1 || h == 1)) {
#pragma unroll
            for (int k = 0; k < Q2; ++k) {
              const double y = sm[L::at(e, TAo + P1 * P1 * S2 + k)] + sm[L::at(e, TAo + (0 * P1 + 1) * S2 + k)];
              apex = fma(B.c2[k * P1 + 1], y, apex);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < n; ++r) {
          if (SPLIT == 1 || r % SPLIT == h) {
            double s = B.c2[co + r] * x[0];
#pragma unroll
            for (int k = 1; k < Q2; ++k) s = fma(B.c2[co + k * n + r], x[k], s);
            if (r == 1) s += apex;
            out(e, pr.z + r, s);
          }
        }
      });
    });
  } else if constexpr (S == PRISM && WP) {
    prism_slice_pairs<P, L, NT>([&](auto pc, int e, int q) {
      constexpr int p = decltype(pc)::value, n = P1 - p, co = wfam_off(Q2, P1, p);
      constexpr int off = prism_slice_off(P1, p);
      double x[Q2];
#pragma unroll
      for (int k = 0; k < Q2; ++k) x[k] = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
      double corr = 0.0;
      if constexpr (p == 0) {
        // modes (0,q,1) += sum_k c2[0][k][1] TA[1][q][k] (operators.py:312-317)
#pragma unroll
        for (int k = 0; k < Q2; ++k) corr = fma(B.c2[k * P1 + 1], sm[L::at(e, TAo + (1 * P1 + q) * S2 + k)], corr);
      }
#pragma unroll
      for (int r = 0; r < n; ++r) {
        double s = B.c2[co + r] * x[0];
#pragma unroll
        for (int k = 1; k < Q2; ++k) s = fma(B.c2[co + k * n + r], x[k], s);
        if (p == 0 && r == 1) s += corr;
        out(e, off + q * n + r, s);
      }
    });
  } else if constexpr (S == PRISM && P <= kPrismUniformMaxP && !RD) {
    constexpr int SPLIT = SPL && 2 * L::EB * P1 <= NT ? 2 : 1;  // see stage_f1
    items<L, P1 * SPLIT, NT>([&](int e, int q2) {
      const int h = q2 / P1, q = q2 - h * P1;
      int off = 0;
#pragma unroll
      for (int p = 0; p < P1; ++p) {
        const int n = P1 - p;
        if (SPLIT > 1 && p % SPLIT != h) {
          off += P1 * n;
          continue;
        }
        const int co = wfam_off(Q2, P1, p);
        double x[Q2];
#pragma unroll
        for (int k = 0; k < Q2; ++k) x[k] = sm[L::at(e, TAo + (p * P1 + q) * S2 + k)];
#pragma unroll
        for (int r = 0; r < P1; ++r) {
          if (r < n) {
            double s = B.c2[co + r] * x[0];
#pragma unroll
            for (int k = 1; k < Q2; ++k) s = fma(B.c2[co + k * n + r], x[k], s);
            if (p == 0 && r == 1) {
              // modes (0,q,1) += sum_k c2[0][k][1] TA[1][q][k] (operators.py:312-317)
              double corr = 0.0;
#pragma unroll
              for (int k = 0; k < Q2; ++k)
                corr = fma(B.c2[k * P1 + 1], sm[L::at(e, TAo + (1 * P1 + q) * S2 + k)], corr);
              s += corr;
            }
            out(e, off + q * n + r, s);
          }
        }
        off += P1 * n;
      }
    });
  } else {
    constexpr int SPLIT = SPL && 2 * L::EB * Dm::NPAIR <= NT ? 2 : 1;  // see the dispatch path
    const int4* pairs = reinterpret_cast<const int4*>(gtab + GLayout<S, P>::PAIRS);
    items<L, Dm::NPAIR * SPLIT, NT>([&](int e, int ps2) {
      const int h = ps2 / Dm::NPAIR, ps = ps2 - h * Dm::NPAIR;
      const int4 pr = ldt<SMT>(pairs + ps);
      const int m = (S == TET) ? pr.x + pr.y : (S == PRISM) ? pr.x : cmax(pr.x, pr.y);
      const int n = P1 - m;
      const double* fam = gtab + (DER2 ? GLayout<S, P>::DC2 : GLayout<S, P>::C2);
      const double* tab = fam + wfam_off(Q2, P1, m);
      double x[Q2];
#pragma unroll
      for (int k = 0; k < Q2; ++k) x[k] = sm[L::at(e, TAo + (pr.x * P1 + pr.y) * S2 + k)];
      if constexpr (S == TET) {
        if (pr.x == 0 && pr.y == 1) {
#pragma unroll
          for (int k = 0; k < Q2; ++k) x[k] += sm[L::at(e, TAo + (P1 * P1 + 1) * S2 + k)];
        }
      }
      double apex = 0.0;
      if (S != PRISM && pr.x == 0 && pr.y == 0 && (SPLIT == 1 || h == 1)) {
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const double y = sm[L::at(e, TAo + P1 * P1 * S2 + k)] + sm[L::at(e, TAo + (0 * P1 + 1) * S2 + k)];
          apex = fma(ldt<SMT>(fam + k * P1 + 1), y, apex);
        }
      }
      if (S == PRISM && pr.x == 0 && (SPLIT == 1 || h == 1)) {
        // modes (0,q,1) += sum_k c2[0][k][1] TA[1][q][k] (operators.py:312-317)
#pragma unroll
        for (int k = 0; k < Q2; ++k)
          apex = fma(ldt<SMT>(fam + k * P1 + 1), sm[L::at(e, TAo + (1 * P1 + pr.y) * S2 + k)], apex);
      }
      if constexpr (kRaggedRuntimeLoop) {
#pragma unroll 1
        for (int r = 0; r < pr.w; ++r) {
          if (SPLIT == 1 || r % SPLIT == h) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < Q2; ++k) s = fma(ldt<SMT>(tab + k * n + r), x[k], s);
            if (r == 1) s += apex;
            out(e, pr.z + r, s);
          }
        }
        return;
      }
#pragma unroll
      for (int r = 0; r < P1; ++r) {
        if (r < pr.w && (SPLIT == 1 || r % SPLIT == h)) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < Q2; ++k) s = fma(ldt<SMT>(tab + k * n + r), x[k], s);
          if (r == 1) s += apex;
          out(e, pr.z + r, s);
        }
      }
    });
  }
}

}  // namespace sk

// Operator kernels (SUM_FAC_TOP strategy) composed from the stages in
// sk_stages.cuh.  One CTA per tile of EB elements; grid.y = component.
//
//   k_helm   Helmholtz collocated (Alg. 6, operators.py:670-699); LAMW=false
//            is the stiffness operator (lam = 0: W stream not read).
//   k_mass   mass B^T W B (operators.py:622-633)
//   k_bwd    bwd_trans (operators.py:551-561)
//   k_iprod  iproduct_wrt_base (operators.py:564-574)
//   k_pderiv phys_deriv (operators.py:577-596)
//   k_ipderiv iproduct_wrt_deriv_base (operators.py:599-619), evaluated as
//            B^T sum_k D_k^T (W v_k): D_k B equals the derivative tables
//            exactly for these polynomial spaces (test_operators.py:83-114)
//
// Geometry payloads (built by sk_payload_pack, geom.cu):
//   HELMHOLTZ deformed [E][7][k][i*Q1+j]: Lam' = G^T Lam G (6 unique) and
//             wJ; G (Duffy chain rule) folded in so the kernel applies a
//             plain symmetric 3x3 per point.  regular [E][8]: Lam (6), |J|.
//   W         deformed [E][i][j][k] wJ; regular [E] |J|.
//   DERIV     deformed [E][9][k][i*Q1+j]: T[m][j] = sum_i G[i][m] dxi[i][j];
//             regular [E][9] dxi.
#pragma once

#include "sk_stages.cuh"

namespace sk {

template <int S, int P>
struct OpArgs {
  FwdTab<S, P> B;
  DTab<S, P> D;
  const double* __restrict__ in;
  double* __restrict__ out;
  const double* __restrict__ pay;
  const double* __restrict__ gtab;
  long long E, Epad;
  long long in_cstride, out_cstride;  // doubles between components
  int W;
  int pad_;
  double lam;
};

template <int S, int P, int EB>
__device__ __forceinline__ Ctx make_ctx(const OpArgs<S, P>& A) {
  Ctx c;
  c.e0 = (long long)blockIdx.x * EB;
  c.E = A.E;
  c.Epad = A.Epad;
  c.W = A.W;
  return c;
}

// ---------------------------------------------------------------------------
// Helmholtz, collocated: 9 stages, 8 CTA barriers
template <int S, int P, int EB, int NT, int GEO, bool LAMW>
__global__ void __launch_bounds__(NT) k_helm(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2;
  constexpr int NQ = Dm::NQ, PL = Dm::PLANE, ES = 3 * PL;
  constexpr int UO = 0, V0O = PL, V1O = 2 * PL, TAo = 0, TBo = 2 * PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;

  stage_f1<S, P, EB, NT, ES, TAo>(A.B, A.gtab, src, c, sm);
  __syncthreads();
  stage_f2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  // F3 + D0: u along i, v0 = D0 u
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double* el = sm + e * ES;
    double x[P1], u[Q0], v[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = el[TBo + (p * Q1 + j) * S2 + k];
    line_a0<S, P>(A.B, x, u);
    line_d<Q0>(A.D.d0, u, v);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      el[UO + (i * Q1 + j) * S2 + k] = u[i];
      el[V0O + (i * Q1 + j) * S2 + k] = v[i];
    }
  });
  __syncthreads();
  // M1: v1 = D1 u along j
  items<EB, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double* el = sm + e * ES;
    double u[Q1], v[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) u[j] = el[UO + (i * Q1 + j) * S2 + k];
    line_d<Q1>(A.D.d1, u, v);
#pragma unroll
    for (int j = 0; j < Q1; ++j) el[V1O + (i * Q1 + j) * S2 + k] = v[j];
  });
  __syncthreads();
  // M2: v2 = D2 u along k; metric w = Lam' v per point; lam W u; D2^T w2
  items<EB, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double* el = sm + e * ES;
    double* row = el + ps * S2;  // (i,j) row, ps = i*Q1 + j
    double u[Q2], w2[Q2], z[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) u[k] = row[UO + k];
    line_d<Q2>(A.D.d2, u, w2);  // w2 holds v2 until overwritten per point
    if constexpr (GEO == GEO_DEFORMED) {
      const double* g = A.pay + (live ? eg : 0) * (7LL * NQ) + ps;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const double* gk = g + k * (Q0 * Q1);
        const double l00 = live ? __ldcs(gk + 0 * NQ) : 0.0, l01 = live ? __ldcs(gk + 1 * NQ) : 0.0,
                     l02 = live ? __ldcs(gk + 2 * NQ) : 0.0, l11 = live ? __ldcs(gk + 3 * NQ) : 0.0,
                     l12 = live ? __ldcs(gk + 4 * NQ) : 0.0, l22 = live ? __ldcs(gk + 5 * NQ) : 0.0;
        const double v0 = row[V0O + k], v1 = row[V1O + k], v2 = w2[k];
        const double a0 = fma(l02, v2, fma(l01, v1, l00 * v0));
        const double a1 = fma(l12, v2, fma(l11, v1, l01 * v0));
        w2[k] = fma(l22, v2, fma(l12, v1, l02 * v0));
        row[V0O + k] = a0;
        row[V1O + k] = a1;
        if constexpr (LAMW) {
          const double wj = live ? __ldcs(gk + 6 * NQ) : 0.0;
          z[k] = (A.lam * wj) * u[k];
        } else {
          z[k] = 0.0;
        }
      }
    } else {
      // affine: Lam per element, G and reference weights per point
      const double* ge = A.pay + (live ? eg : 0) * 8LL;
      const double l00 = __ldg(ge + 0), l01 = __ldg(ge + 1), l02 = __ldg(ge + 2), l11 = __ldg(ge + 3),
                   l12 = __ldg(ge + 4), l22 = __ldg(ge + 5), jac = __ldg(ge + 6);
      const double* rk = A.gtab + GLayout<S, P>::REGK + ps;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const double* rp = rk + k * (Q0 * Q1);
        const double rw = __ldg(rp);
        const double v0 = row[V0O + k], v1 = row[V1O + k], v2 = w2[k];
        double t0 = v0, t1 = v1, t2 = v2;
        double g00 = 1.0, g10 = 0.0, g11 = 1.0, g20 = 0.0, g21 = 0.0;
        if constexpr (S != HEX) {
          g00 = __ldg(rp + 1 * NQ);
          g10 = __ldg(rp + 2 * NQ);
          g11 = __ldg(rp + 3 * NQ);
          g20 = __ldg(rp + 4 * NQ);
          g21 = __ldg(rp + 5 * NQ);
          t0 = g00 * v0;
          t1 = fma(g11, v1, g10 * v0);
          t2 = fma(g21, v1, fma(g20, v0, v2));
        }
        const double s0 = rw * fma(l02, t2, fma(l01, t1, l00 * t0));
        const double s1 = rw * fma(l12, t2, fma(l11, t1, l01 * t0));
        const double s2 = rw * fma(l22, t2, fma(l12, t1, l02 * t0));
        double a0 = s0, a1 = s1;
        if constexpr (S != HEX) {
          a0 = fma(g20, s2, fma(g10, s1, g00 * s0));
          a1 = fma(g21, s2, g11 * s1);
        }
        row[V0O + k] = live ? a0 : 0.0;
        row[V1O + k] = live ? a1 : 0.0;
        w2[k] = live ? s2 : 0.0;
        if constexpr (LAMW) {
          z[k] = live ? A.lam * ((u[k] * rw) * jac) : 0.0;
        } else {
          z[k] = 0.0;
        }
      }
    }
    line_dt_acc<Q2>(A.D.d2, w2, z);
#pragma unroll
    for (int k = 0; k < Q2; ++k) row[UO + k] = z[k];
  });
  __syncthreads();
  // M3: U += D1^T w1 along j
  items<EB, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double* el = sm + e * ES;
    double w[Q1], r[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) {
      w[j] = el[V1O + (i * Q1 + j) * S2 + k];
      r[j] = el[UO + (i * Q1 + j) * S2 + k];
    }
    line_dt_acc<Q1>(A.D.d1, w, r);
#pragma unroll
    for (int j = 0; j < Q1; ++j) el[UO + (i * Q1 + j) * S2 + k] = r[j];
  });
  __syncthreads();
  // B1: r = U + D0^T w0 along i, then B^T along dir 0
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double* el = sm + e * ES;
    double w[Q0], r[Q0], t[P1];
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      w[i] = el[V0O + (i * Q1 + j) * S2 + k];
      r[i] = el[UO + (i * Q1 + j) * S2 + k];
    }
    line_dt_acc<Q0>(A.D.d0, w, r);
    line_a0t<S, P>(A.B, r, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) el[TBo + (p * Q1 + j) * S2 + k] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  stage_b3<S, P, EB, NT, ES, TAo>(A.B, A.gtab, dst, c, sm);
}

// W at point (i,j,k) of element eg for the W-payload family
template <int S, int P, int GEO>
__device__ __forceinline__ double w_at(const OpArgs<S, P>& A, long long eg, bool live, int l) {
  if (!live) return 0.0;
  if constexpr (GEO == GEO_DEFORMED) {
    return __ldcs(A.pay + eg * (long long)Dims<S, P>::NQ + l);
  } else {
    return __ldg(A.gtab + GLayout<S, P>::REFW + l) * __ldg(A.pay + eg);
  }
}

// ---------------------------------------------------------------------------
// Mass: F1, F2, fused (B, W, B^T) along dir 0, B2, B3
template <int S, int P, int EB, int NT, int GEO>
__global__ void __launch_bounds__(NT) k_mass(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2;
  constexpr int PL = Dm::PLANE, ES = 2 * PL, TAo = 0, TBo = PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  stage_f1<S, P, EB, NT, ES, TAo>(A.B, A.gtab, src, c, sm);
  __syncthreads();
  stage_f2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double* tb = sm + e * ES + TBo;
    double x[P1], u[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = tb[(p * Q1 + j) * S2 + k];
    line_a0<S, P>(A.B, x, u);
#pragma unroll
    for (int i = 0; i < Q0; ++i) u[i] *= w_at<S, P, GEO>(A, eg, live, (i * Q1 + j) * Q2 + k);
    line_a0t<S, P>(A.B, u, x);
#pragma unroll
    for (int p = 0; p < P1; ++p) tb[(p * Q1 + j) * S2 + k] = x[p];
  });
  __syncthreads();
  stage_b2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  stage_b3<S, P, EB, NT, ES, TAo>(A.B, A.gtab, dst, c, sm);
}

// ---------------------------------------------------------------------------
// BwdTrans: coefficients -> quadrature values
template <int S, int P, int EB, int NT>
__global__ void __launch_bounds__(NT) k_bwd(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2;
  constexpr int PL = Dm::PLANE, ES = 2 * PL, TAo = 0, TBo = PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  stage_f1<S, P, EB, NT, ES, TAo>(A.B, A.gtab, src, c, sm);
  __syncthreads();
  stage_f2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const double* tb = sm + e * ES + TBo;
    double x[P1], u[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = tb[(p * Q1 + j) * S2 + k];
    line_a0<S, P>(A.B, x, u);
    if (eg < c.Epad) {
      const long long base = lane_base(eg, Dm::NQ, c.W);
#pragma unroll
      for (int i = 0; i < Q0; ++i) dst[base + (long long)((i * Q1 + j) * Q2 + k) * c.W] = u[i];
    }
  });
}

// ---------------------------------------------------------------------------
// IProductWRTBase: quadrature values -> coefficients, B^T W u
template <int S, int P, int EB, int NT, int GEO>
__global__ void __launch_bounds__(NT) k_iprod(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2;
  constexpr int PL = Dm::PLANE, ES = 2 * PL, TAo = 0, TBo = PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double* tb = sm + e * ES + TBo;
    double u[Q0], t[P1];
    const long long base = lane_base(live ? eg : 0, Dm::NQ, c.W);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      const int l = (i * Q1 + j) * Q2 + k;
      u[i] = live ? __ldg(src + base + (long long)l * c.W) * w_at<S, P, GEO>(A, eg, live, l) : 0.0;
    }
    line_a0t<S, P>(A.B, u, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) tb[(p * Q1 + j) * S2 + k] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  stage_b3<S, P, EB, NT, ES, TAo>(A.B, A.gtab, dst, c, sm);
}

// ---------------------------------------------------------------------------
// PhysDeriv: u (1 component) -> du/dx_j (3 components)
template <int S, int P, int EB, int NT, int GEO>
__global__ void __launch_bounds__(NT) k_pderiv(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2, NQ = Dm::NQ;
  constexpr int PL = Dm::PLANE, ES = 3 * PL, UO = 0, V0O = PL, V1O = 2 * PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double* el = sm + e * ES;
    double u[Q0], v[Q0];
    const long long base = lane_base(live ? eg : 0, NQ, c.W);
#pragma unroll
    for (int i = 0; i < Q0; ++i) u[i] = live ? __ldg(A.in + base + (long long)((i * Q1 + j) * Q2 + k) * c.W) : 0.0;
    line_d<Q0>(A.D.d0, u, v);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      el[UO + (i * Q1 + j) * S2 + k] = u[i];
      el[V0O + (i * Q1 + j) * S2 + k] = v[i];
    }
  });
  __syncthreads();
  items<EB, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double* el = sm + e * ES;
    double u[Q1], v[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) u[j] = el[UO + (i * Q1 + j) * S2 + k];
    line_d<Q1>(A.D.d1, u, v);
#pragma unroll
    for (int j = 0; j < Q1; ++j) el[V1O + (i * Q1 + j) * S2 + k] = v[j];
  });
  __syncthreads();
  items<EB, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    if (eg >= c.Epad) return;
    double* row = sm + e * ES + ps * S2;
    double u[Q2], v2[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) u[k] = row[UO + k];
    line_d<Q2>(A.D.d2, u, v2);
    const long long base = lane_base(eg, NQ, c.W);
    const long long cs = A.out_cstride;
#pragma unroll
    for (int k = 0; k < Q2; ++k) {
      const double v0 = row[V0O + k], v1 = row[V1O + k], w = v2[k];
      double o[3];
      if constexpr (GEO == GEO_DEFORMED) {
        const double* g = A.pay + (live ? eg : 0) * (9LL * NQ) + k * (Q0 * Q1) + ps;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          const double t0 = live ? __ldcs(g + (0 * 3 + jj) * NQ) : 0.0;
          const double t1 = live ? __ldcs(g + (1 * 3 + jj) * NQ) : 0.0;
          const double t2 = live ? __ldcs(g + (2 * 3 + jj) * NQ) : 0.0;
          o[jj] = fma(t2, w, fma(t1, v1, t0 * v0));
        }
      } else {
        const double* ge = A.pay + (live ? eg : 0) * 9LL;
        double t0 = v0, t1 = v1, t2 = w;
        if constexpr (S != HEX) {
          const double* rp = A.gtab + GLayout<S, P>::REGK + k * (Q0 * Q1) + ps;
          const double g00 = __ldg(rp + 1 * NQ), g10 = __ldg(rp + 2 * NQ), g11 = __ldg(rp + 3 * NQ),
                       g20 = __ldg(rp + 4 * NQ), g21 = __ldg(rp + 5 * NQ);
          t0 = g00 * v0;
          t1 = fma(g11, v1, g10 * v0);
          t2 = fma(g21, v1, fma(g20, v0, w));
        }
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
          o[jj] = live ? fma(__ldg(ge + 6 + jj), t2, fma(__ldg(ge + 3 + jj), t1, __ldg(ge + jj) * t0)) : 0.0;
      }
      const long long l = (long long)(ps * Q2 + k) * c.W;
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) A.out[jj * cs + base + l] = o[jj];
    }
  });
}

// ---------------------------------------------------------------------------
// IProductWRTDerivBase: 3 phys components -> 1 coefficient component
template <int S, int P, int EB, int NT, int GEO>
__global__ void __launch_bounds__(NT) k_ipderiv(const __grid_constant__ OpArgs<S, P> A) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = Dm::S2, NQ = Dm::NQ;
  constexpr int PL = Dm::PLANE, ES = 3 * PL, UO = 0, V0O = PL, V1O = 2 * PL, TAo = 0, TBo = 2 * PL;
  extern __shared__ double sm[];
  const Ctx c = make_ctx<S, P, EB>(A);
  items<EB, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double* row = sm + e * ES + ps * S2;
    const long long base = lane_base(live ? eg : 0, NQ, c.W);
    const long long cs = A.in_cstride;
    double w2[Q2], r[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) {
      const int l = ps * Q2 + k;
      const double wq = w_at<S, P, GEO>(A, eg, live, l);
      const long long a = base + (long long)l * c.W;
      row[V0O + k] = live ? __ldg(A.in + a) * wq : 0.0;
      row[V1O + k] = live ? __ldg(A.in + cs + a) * wq : 0.0;
      w2[k] = live ? __ldg(A.in + 2 * cs + a) * wq : 0.0;
      r[k] = 0.0;
    }
    line_dt_acc<Q2>(A.D.d2, w2, r);
#pragma unroll
    for (int k = 0; k < Q2; ++k) row[UO + k] = r[k];
  });
  __syncthreads();
  items<EB, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double* el = sm + e * ES;
    double w[Q1], r[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) {
      w[j] = el[V1O + (i * Q1 + j) * S2 + k];
      r[j] = el[UO + (i * Q1 + j) * S2 + k];
    }
    line_dt_acc<Q1>(A.D.d1, w, r);
#pragma unroll
    for (int j = 0; j < Q1; ++j) el[UO + (i * Q1 + j) * S2 + k] = r[j];
  });
  __syncthreads();
  items<EB, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double* el = sm + e * ES;
    double w[Q0], r[Q0], t[P1];
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      w[i] = el[V0O + (i * Q1 + j) * S2 + k];
      r[i] = el[UO + (i * Q1 + j) * S2 + k];
    }
    line_dt_acc<Q0>(A.D.d0, w, r);
    line_a0t<S, P>(A.B, r, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) el[TBo + (p * Q1 + j) * S2 + k] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, EB, NT, ES, TAo, TBo>(A.B, sm);
  __syncthreads();
  stage_b3<S, P, EB, NT, ES, TAo>(A.B, A.gtab, A.out, c, sm);
}

}  // namespace sk

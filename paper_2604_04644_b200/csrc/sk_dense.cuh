// StdMat mass on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): the
// reference's dense strategy (_stdmat_apply with the dense basis matrix,
// speckern/operators.py:398-405; bmat shapes.py:491-492) as element-batched
// GEMMs, for the low orders where the paper found StdMat fastest for simplex
// mass.
//
// Deformed:  out_e = B^T diag(wJ_e) B uhat_e, per warp a group of 8 elements:
//   GEMM1  U^T (8 x NQ) = Uhat^T (8 x NM) . B^T (NM x NQ)    A = Uhat^T (global)
//   V^T = U^T o W^T (wJ from the W payload, per element and point)
//   GEMM2  out^T (8 x NM) = V^T (8 x NQ) . B (NQ x NM)         A = V^T (registers)
// processed point tile by point tile (8 points): GEMM1's accumulator of a
// tile becomes GEMM2's A operand of two k-steps through four quad shuffles,
// so U never leaves registers.
// Regular:   out_e = |J|_e M_ref uhat_e with M_ref = B^T diag(refw) B (one
//   NM x NM matrix per basis): one GEMM, 2 NM^2 multiply-adds per element.
//
// B / M_ref operand fragments live in shared memory in fragment order
// (one conflict-free 8-byte load per lane per DMMA); the fragments are built
// once per basis and device (abi.cu device_dense) from the dense B that the
// sum-factorised bwd_trans kernel produces on unit coefficient vectors.
// Persistent CTAs: every warp strides over 8-element groups, no CTA barrier
// after the fragment copy.
#pragma once

#include <vector>

#include "basis_host.hpp"
#include "sk_common.cuh"

namespace sk {

template <int S, int P>
struct DenseDims {
  using Dm = Dims<S, P>;
  static constexpr int NQ = Dm::NQ, NM = Dm::NM;
  static constexpr int NQP = (NQ + 7) / 8 * 8;   // points, padded to the 8-row tiles
  static constexpr int NMP4 = (NM + 3) / 4 * 4;  // modes as a k dimension
  static constexpr int NMP8 = (NM + 7) / 8 * 8;  // modes as an n dimension
  static constexpr int NT = NQP / 8;             // point tiles
  static constexpr int KS1 = NMP4 / 4;           // GEMM1 k-steps
  static constexpr int MT = NMP8 / 8;            // output mode tiles
  static constexpr int F1 = NT * KS1 * 32;       // GEMM1 B fragments: B^T[k = m][n = q]
  static constexpr int F2 = 2 * NT * MT * 32;    // GEMM2 B fragments: B[k = q][n = m]
  static constexpr int FR = KS1 * MT * 32;       // regular: M_ref[k][n]
  static constexpr int FH = 7 * FR;              // regular Helmholtz: K_0..K_5, M_ref
  static constexpr int DOUBLES = F1 + F2 + FR + FH;
  // a kernel exists when its fragments fit in 100 KB of shared memory (two
  // CTAs per SM): bit 0 regular mass, bit 1 deformed mass, bit 2 regular
  // Helmholtz
  static constexpr int MASK = (FR * 8 <= 100 * 1024 ? 1 : 0) | ((F1 + F2) * 8 <= 100 * 1024 ? 2 : 0) |
                              (FH * 8 <= 100 * 1024 ? 4 : 0);
};

// host: fragment tables from the dense B (NQ x NM row-major), the reference
// weights, the collocation matrices and the Duffy factors G
template <int S, int P>
void fill_dense_frags(const HostBasis& hb, const double* B, double* f) {
  using X = DenseDims<S, P>;
  const double* refw = hb.refw.data();
  auto b = [&](int q, int m) { return (q < X::NQ && m < X::NM) ? B[q * X::NM + m] : 0.0; };
  double* f1 = f;
  double* f2 = f + X::F1;
  double* fr = f + X::F1 + X::F2;
  for (int nt = 0; nt < X::NT; ++nt)
    for (int ks = 0; ks < X::KS1; ++ks)
      for (int l = 0; l < 32; ++l) f1[(nt * X::KS1 + ks) * 32 + l] = b(8 * nt + (l >> 2), 4 * ks + (l & 3));
  for (int ks = 0; ks < 2 * X::NT; ++ks)
    for (int mt = 0; mt < X::MT; ++mt)
      for (int l = 0; l < 32; ++l) f2[(ks * X::MT + mt) * 32 + l] = b(4 * ks + (l & 3), 8 * mt + (l >> 2));
  // M_ref = B^T diag(refw) B
  std::vector<double> M((size_t)X::NM * X::NM, 0.0);
  for (int i = 0; i < X::NM; ++i)
    for (int j = 0; j < X::NM; ++j) {
      double s = 0.0;
      for (int q = 0; q < X::NQ; ++q) s += B[q * X::NM + i] * refw[q] * B[q * X::NM + j];
      M[(size_t)i * X::NM + j] = s;
    }
  auto put = [&](double* dst, const std::vector<double>& A) {
    for (int ks = 0; ks < X::KS1; ++ks)
      for (int mt = 0; mt < X::MT; ++mt)
        for (int l = 0; l < 32; ++l) {
          const int k = 4 * ks + (l & 3), n = 8 * mt + (l >> 2);
          dst[(ks * X::MT + mt) * 32 + l] = (k < X::NM && n < X::NM) ? A[(size_t)k * X::NM + n] : 0.0;
        }
  };
  put(fr, M);
  // Regular Helmholtz: with T_a(m, l) = (G D B)_a, the Duffy-mapped reference
  // gradient of mode m at point l (collocation D_d of column m of B along
  // direction d, operators.py:449-464, then G, 471-490), the elemental
  // operator of an affine element is sum_ab Lam_ab K_ab + lam |J| M_ref with
  // K_ab[n][m] = sum_l refw_l T_b(n, l) T_a(m, l) (operators.py:502-523,
  // 670-699).  Lam is symmetric: coefficient matrices for the payload order
  // Lam00, Lam01, Lam02, Lam11, Lam12, Lam22 are K_aa and K_ab + K_ba.
  const int Q0 = hb.Q[0], Q1 = hb.Q[1], Q2 = hb.Q[2];
  std::vector<double> T((size_t)3 * X::NM * X::NQ);  // [a][m][l]
  for (int m = 0; m < X::NM; ++m) {
    for (int i = 0; i < Q0; ++i)
      for (int j = 0; j < Q1; ++j)
        for (int k = 0; k < Q2; ++k) {
          const int l = (i * Q1 + j) * Q2 + k;
          double v[3] = {0.0, 0.0, 0.0};
          for (int a = 0; a < Q0; ++a) v[0] += hb.D[0][i * Q0 + a] * B[((a * Q1 + j) * Q2 + k) * X::NM + m];
          for (int b = 0; b < Q1; ++b) v[1] += hb.D[1][j * Q1 + b] * B[((i * Q1 + b) * Q2 + k) * X::NM + m];
          for (int c = 0; c < Q2; ++c) v[2] += hb.D[2][k * Q2 + c] * B[((i * Q1 + j) * Q2 + c) * X::NM + m];
          for (int a = 0; a < 3; ++a) {
            const double* g = &hb.G[9 * l + 3 * a];
            T[((size_t)a * X::NM + m) * X::NQ + l] = g[0] * v[0] + g[1] * v[1] + g[2] * v[2];
          }
        }
  }
  const int ai[6] = {0, 0, 0, 1, 1, 2}, bi[6] = {0, 1, 2, 1, 2, 2};
  std::vector<double> K((size_t)X::NM * X::NM);
  for (int cidx = 0; cidx < 6; ++cidx) {
    const int a = ai[cidx], b = bi[cidx];
    for (int n = 0; n < X::NM; ++n)
      for (int m = 0; m < X::NM; ++m) {
        double s1 = 0.0, s2 = 0.0;
        for (int l = 0; l < X::NQ; ++l) {
          const double w = refw[l];
          s1 += w * T[((size_t)b * X::NM + n) * X::NQ + l] * T[((size_t)a * X::NM + m) * X::NQ + l];
          if (a != b) s2 += w * T[((size_t)a * X::NM + n) * X::NQ + l] * T[((size_t)b * X::NM + m) * X::NQ + l];
        }
        // B operand of outT = uhatT . H^T: element [k = m][n]
        K[(size_t)m * X::NM + n] = s1 + s2;
      }
    put(f + X::F1 + X::F2 + X::FR + cidx * X::FR, K);
  }
  put(f + X::F1 + X::F2 + X::FR + 6 * X::FR, M);
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct DenseArgs {
  const double* __restrict__ frag;  // DenseDims::DOUBLES (device)
  const double* __restrict__ in;
  double* __restrict__ out;
  const double* __restrict__ pay;   // W payload (deformed wJ per point / regular |J|)
  long long E, Epad, in_cstride, out_cstride;
  int W;
};

constexpr int kDenseThreads = 256;
// min CTAs per SM for the dense mass kernel's register budget (0: none) and
// next-group prefetch of the coefficient fragments: on for regular geometry
// (measured +4-38 % on regular pyr P=3-5 / tet P=3-6, profiles/r02/
// dense_tune_reg.jsonl), off for deformed (slower at P=1, where the W stream
// already keeps the loads in flight; dense_tune_def.jsonl).  SK_DENSE_PF=0/1
// forces it in tuning builds.
#ifndef SK_DENSE_MINB
#define SK_DENSE_MINB -1
#endif
// deformed: 5 CTAs per SM (<= 51 registers, no spills) measured +0-29 %
// over the unbounded 60-register build (pyr P=2 0.48 -> 0.62, tet P=1-3
// +1-10 %, dense_tune_def.jsonl); regular: unbounded (the prefetch needs the
// registers)
template <int GEO>
constexpr int dense_minb() {
  return SK_DENSE_MINB >= 0 ? SK_DENSE_MINB : GEO == GEO_DEFORMED ? 5 : 0;
}
#ifndef SK_DENSE_PF
#define SK_DENSE_PF -1
#endif

template <int S, int P, int PW, int GEO>
__global__ void __launch_bounds__(kDenseThreads, dense_minb<GEO>()) k_mass_dense(const __grid_constant__ DenseArgs A) {
  using X = DenseDims<S, P>;
  constexpr int NQ = X::NQ, NM = X::NM, KS1 = X::KS1, MT = X::MT;
  constexpr bool PF = SK_DENSE_PF >= 0 ? SK_DENSE_PF != 0 : GEO == GEO_REGULAR;
  extern __shared__ double sfr[];
  // fragments this geometry class reads: GEMM1 + GEMM2 (deformed) or M_ref
  constexpr int OFF = GEO == GEO_DEFORMED ? 0 : X::F1 + X::F2;
  constexpr int NF = GEO == GEO_DEFORMED ? X::F1 + X::F2 : X::FR;
  for (int i = threadIdx.x; i < NF / 2; i += kDenseThreads)
    reinterpret_cast<double2*>(sfr)[i] = __ldg(reinterpret_cast<const double2*>(A.frag + OFF) + i);
  __syncthreads();
  const double* f1 = sfr;
  const double* f2 = sfr + X::F1;
  const int lane = threadIdx.x & 31, t = lane & 3, r = lane >> 2;
  const long long warps = (long long)gridDim.x * (kDenseThreads / 32);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  const long long ngroups = (A.Epad + 7) / 8;
  auto load_a = [&](long long gg, double (&dst)[KS1]) {
    const long long ee = gg * 8 + r;
    const bool lv = gg < ngroups && ee < A.E;
    const long long bb = lane_base(lv ? ee : 0, NM, A.W);
#pragma unroll
    for (int ks = 0; ks < KS1; ++ks) {
      const int m = 4 * ks + t;
      dst[ks] = (lv && m < NM) ? __ldcs(src + bb + (long long)m * A.W) : 0.0;
    }
  };
  double a_next[KS1];
  const long long g_first = blockIdx.x * (kDenseThreads / 32) + (threadIdx.x >> 5);
  if constexpr (PF) load_a(g_first, a_next);
  for (long long g = g_first; g < ngroups; g += warps) {
    const long long e = g * 8 + r;  // this lane's element (A-operand row = C row)
    const bool live = e < A.E;
    double a[KS1];
    if constexpr (PF) {
#pragma unroll
      for (int ks = 0; ks < KS1; ++ks) a[ks] = a_next[ks];
      load_a(g + warps, a_next);  // next group's coefficients in flight during this one
    } else {
      load_a(g, a);
    }
    double c[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) c[mt][0] = c[mt][1] = 0.0;
    if constexpr (GEO == GEO_DEFORMED) {
      const double* wp = A.pay + pay_base<PW>(live ? e : 0, 1, NQ);
      const int s1 = (lane & ~3) | (t >> 1), s2 = s1 + 2;
#pragma unroll
      for (int nt = 0; nt < X::NT; ++nt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) dmma(d0, d1, a[ks], f1[(nt * KS1 + ks) * 32 + lane]);
        const int q0 = 8 * nt + 2 * t;
        const double w0 = (live && q0 < NQ) ? __ldcs(wp + (long long)q0 * PW) : 0.0;
        const double w1 = (live && q0 + 1 < NQ) ? __ldcs(wp + (long long)(q0 + 1) * PW) : 0.0;
        const double v0 = d0 * w0, v1 = d1 * w1;
        // V^T[r][8nt + t] and V^T[r][8nt + 4 + t] from the quad's accumulators
        const double x0 = __shfl_sync(0xffffffffu, v0, s1), x1 = __shfl_sync(0xffffffffu, v1, s1);
        const double y0 = __shfl_sync(0xffffffffu, v0, s2), y1 = __shfl_sync(0xffffffffu, v1, s2);
        const double alo = (t & 1) ? x1 : x0, ahi = (t & 1) ? y1 : y0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          dmma(c[mt][0], c[mt][1], alo, f2[((2 * nt) * MT + mt) * 32 + lane]);
          dmma(c[mt][0], c[mt][1], ahi, f2[((2 * nt + 1) * MT + mt) * 32 + lane]);
        }
      }
    } else {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) dmma(c[mt][0], c[mt][1], a[ks], sfr[(ks * MT + mt) * 32 + lane]);
      const double jac = live ? __ldg(A.pay + pay_base<PW>(e, 1, 1)) : 0.0;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        c[mt][0] *= jac;
        c[mt][1] *= jac;
      }
    }
    if (e < A.Epad) {
      const long long ob = lane_base(e, NM, A.W);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int m = 8 * mt + 2 * t;
        if (m < NM) __stcs(dst + ob + (long long)m * A.W, live ? c[mt][0] : 0.0);
        if (m + 1 < NM) __stcs(dst + ob + (long long)(m + 1) * A.W, live ? c[mt][1] : 0.0);
      }
    }
  }
}

// Regular-geometry collocated Helmholtz / stiffness as StdMat on DMMA:
// out_e = sum_c coef_e,c (H_c uhat_e), coef = (Lam00, Lam01, Lam02, Lam11,
// Lam12, Lam22, lam |J|) from the regular Helmholtz payload (kRegPW lanes),
// H_c = K_c / M_ref (fill_dense_frags).  One 8-element group per warp; per
// output mode tile the seven products accumulate in two registers each and
// are combined with the element's coefficients.
template <int S, int P, bool LAMW>
__global__ void __launch_bounds__(kDenseThreads) k_helm_dense(const __grid_constant__ DenseArgs A, double lam) {
  using X = DenseDims<S, P>;
  constexpr int NM = X::NM, KS1 = X::KS1, MT = X::MT, NC = LAMW ? 7 : 6;
  extern __shared__ double sfr[];
  for (int i = threadIdx.x; i < NC * X::FR / 2; i += kDenseThreads)
    reinterpret_cast<double2*>(sfr)[i] = __ldg(reinterpret_cast<const double2*>(A.frag + X::F1 + X::F2 + X::FR) + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, t = lane & 3, r = lane >> 2;
  const long long warps = (long long)gridDim.x * (kDenseThreads / 32);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  const long long ngroups = (A.Epad + 7) / 8;
  for (long long g = blockIdx.x * (kDenseThreads / 32) + (threadIdx.x >> 5); g < ngroups; g += warps) {
    const long long e = g * 8 + r;
    const bool live = e < A.E;
    const long long base = lane_base(live ? e : 0, NM, A.W);
    double a[KS1];
#pragma unroll
    for (int ks = 0; ks < KS1; ++ks) {
      const int m = 4 * ks + t;
      a[ks] = (live && m < NM) ? __ldcs(src + base + (long long)m * A.W) : 0.0;
    }
    double coef[NC];
    const double* ge = A.pay + pay_base<kRegPW>(live ? e : 0, 8, 1);
#pragma unroll
    for (int cc = 0; cc < 6; ++cc) coef[cc] = live ? __ldg(ge + cc * kRegPW) : 0.0;
    if constexpr (LAMW) coef[6] = live ? lam * __ldg(ge + 6 * kRegPW) : 0.0;
    const bool store = e < A.Epad;
    const long long ob = lane_base(store ? e : 0, NM, A.W);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) dmma(c0, c1, a[ks], sfr[((cc * KS1 + ks) * MT + mt) * 32 + lane]);
        o0 = fma(coef[cc], c0, o0);
        o1 = fma(coef[cc], c1, o1);
      }
      const int m = 8 * mt + 2 * t;
      if (store) {
        if (m < NM) __stcs(dst + ob + (long long)m * A.W, o0);
        if (m + 1 < NM) __stcs(dst + ob + (long long)(m + 1) * A.W, o1);
      }
    }
  }
}

}  // namespace sk

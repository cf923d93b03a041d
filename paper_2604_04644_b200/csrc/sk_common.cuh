// Compile-time dimensions, kernel-parameter tables, shared-memory layout
// policies and small device helpers shared by every sm_100a kernel.
#pragma once

#include <cstdint>
#include <type_traits>

#include "sk_shapes.hpp"

namespace sk {

enum : int { GEO_REGULAR = 0, GEO_DEFORMED = 1,
             GEO_UNIT = 2 };  // no weight (the staged Helmholtz's final B^T)
// lane width of the regular-geometry Helmholtz payload (8 doubles per
// element): fixed, so the regular kernel's tile width is tuned on its own
constexpr int kRegPW = 16;

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

__host__ __device__ constexpr int n_modes(int S, int P) {
  return S == HEX     ? (P + 1) * (P + 1) * (P + 1)
         : S == PRISM ? (P + 1) * (P + 1) * (P + 2) / 2
         : S == PYR   ? (P + 1) * (P + 2) * (2 * P + 3) / 6
                      : (P + 1) * (P + 2) * (P + 3) / 6;
}

// Per-(shape, order) sizes.  Quadrature per direction: P+2 Gauss-Lobatto,
// P+1 Gauss-Radau-Jacobi on collapsed directions (shapes.py:76-139).
template <int S, int P>
struct Dims {
  static constexpr int P1 = P + 1;
  static constexpr int Q0 = P + 2;
  static constexpr int Q1 = (S == TET) ? P + 1 : P + 2;
  static constexpr int Q2 = (S == HEX) ? P + 2 : P + 1;
  static constexpr int NQ = Q0 * Q1 * Q2;
  static constexpr int NM = n_modes(S, P);
  static constexpr int NTRI = P1 * (P1 + 1) / 2;
  // ragged first/last stages (pyr, tet) iterate over (p, q) pairs
  static constexpr int NPAIR = (S == TET) ? NTRI : P1 * P1;
};

// Shared-memory layout of the per-element work arrays.  Each element owns
// NPL "planes" of quad-point-sized arrays, addressed by a plane-relative
// index idx = plane*PLANE + (i*Q1 + j)*S2 + k (k-row stride S2).  The EB
// elements of a tile are the fastest smem dimension, sm[idx*EB + e], and work
// items map e = item % EB (the shared-memory analogue of the reference's
// SIMD lane interleave, field_block.py:205-214).  A half-warp then covers
// 16/EB consecutive passive indices at the same EB lanes: with EB = 16 it
// reads 16 consecutive doubles whatever the sweep direction, and for
// EB < 16 an odd row stride S2 keeps consecutive passive indices in
// distinct bank groups, so every sweep is (nearly) bank-conflict free.
// k-row stride of the work planes: the line length Q2 for EB >= 16, the
// next odd value below that (16/EB passive indices per half-warp at odd
// strides), or a per-(shape, order) override for single-element tiles where
// no interleave separates the sweep patterns (SK_S2 / kRowStride, measured)
#ifndef SK_S2
#define SK_S2 0
#endif
constexpr int kRowStride[4][11] = {
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // hex
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // prism
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // pyr
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},  // tet
};
__host__ __device__ constexpr int row_stride(int S, int P, int EB) {
  return EB >= 16 ? (S == HEX ? P + 2 : P + 1)
         : SK_S2 >= (S == HEX ? P + 2 : P + 1) ? SK_S2
         : kRowStride[S][P] > 0 ? kRowStride[S][P]
                                : ((S == HEX ? P + 2 : P + 1) | 1);
}

template <int S, int P, int NPL, int EB_>
struct Lay {
  using Dm = Dims<S, P>;
  static constexpr int EB = EB_;
  static constexpr int S2 = row_stride(S, P, EB);
  static constexpr int PLANE = Dm::Q0 * Dm::Q1 * S2;
  // tile staging area for coefficients, [mode][XSTR] from the start of plane
  // 1: an odd stride keeps the transposing copy conflict free; it must fit
  // in the planes that are dead while it is live (plane 1 on, >= 2 planes)
  static constexpr int XSTR = EB >= 8 ? EB + 1 : EB;
  static constexpr int SMEM_DOUBLES = NPL * PLANE * EB;
  // staged ragged-sweep tables after the planes (int4 pairs: 16-byte aligned)
  static constexpr int TABOFF = (SMEM_DOUBLES + 1) / 2 * 2;
  static_assert(Dm::NM * XSTR <= (NPL - 1) * PLANE * EB, "coefficient staging does not fit");
  __device__ static __forceinline__ int at(int e, int idx) { return idx * EB + e; }
};

// offset of the leading-index-p slice in a packed warped family whose slice
// p has (P1 - p) columns and Q rows
__host__ __device__ constexpr int wfam_off(int Q, int P1, int p) { return Q * (p * P1 - p * (p - 1) / 2); }

// Basis tables consumed with compile-time indices: they live in the kernel
// parameter space (constant bank) and enter DFMAs as uniform operands.
// Directions whose 1D rule is Gauss-Lobatto (symmetric points z_{Q-1-i} =
// -z_i): dir 0 always, dir 1 except tet, dir 2 for hex.  Their collocation
// matrices are centro-antisymmetric, D[Q-1-a][Q-1-b] = -D[a][b], and the
// modified basis has psi_p(-z) = (-1)^p psi_p(z) (p >= 2), psi_0(-z) =
// psi_1(z), so every 1D contraction along them runs in even-odd form at
// half the multiply-adds.
__host__ __device__ constexpr bool gll_dir(int S, int d) { return d == 0 || (d == 1 && S != TET) || (d == 2 && S == HEX); }

// even-odd kernels in use from this order on, per shape (measured: at low
// order the extra even/odd combinations cost more than the halved
// multiply-adds save on hex; tables are filled regardless)
#ifdef SK_EO_MINP
__host__ __device__ constexpr bool use_eo(int, int P) { return P >= SK_EO_MINP; }
#else
__host__ __device__ constexpr bool use_eo(int S, int P) {
  return P >= (S == HEX ? 6 : S == TET ? 4 : 3);
}
#endif
// the mass kernels' sweeps, measured separately (roofline fraction plain ->
// even-odd): hex P=5 0.53 -> 0.65 (the Helmholtz kernel loses 5 % there),
// hex P=4 0.69 -> 0.73, prism P=2 0.66 -> 0.70; neutral at hex P=2-3, pyr /
// tet P=2-3 (profiles/r02/eo_hex5*.jsonl, eo_mass_low.jsonl)
__host__ __device__ constexpr bool use_eo_mass(int S, int P) {
  return use_eo(S, P) || (S == HEX && P >= 4) || (S == PRISM && P >= 2);
}

template <int S, int P>
struct FwdTab {
  using Dm = Dims<S, P>;
  double a0[Dm::Q0 * Dm::P1];                       // dir 0 [i][p]
  double a1[(S != TET) ? Dm::Q1 * Dm::P1 : 1];      // dir 1 [j][q]
  double a2[(S == HEX) ? Dm::Q2 * Dm::P1 : 1];      // dir 2 [k][r]
  double b1[(S == TET) ? Dm::Q1 * Dm::NTRI : 1];    // tet dir 1, per p
  double c2[(S != HEX) ? Dm::Q2 * Dm::NTRI : 1];    // dir-2 family, per slice m
  // even-odd vertex-mode combinations of the full families,
  // (B[i][0] +- B[i][1]) / 2, rows i <= (Q-1)/2
  double a0p[Dm::Q0], a0m[Dm::Q0];
  double a1p[(S != TET) ? Dm::Q1 : 1], a1m[(S != TET) ? Dm::Q1 : 1];
  double a2p[(S == HEX) ? Dm::Q2 : 1], a2m[(S == HEX) ? Dm::Q2 : 1];
};

// even-odd form of a centro-antisymmetric Q x Q matrix M, H = Q/2:
// E[a][b] = (M[a][b] + M[a][Q-1-b]) / 2, O[a][b] = (M[a][b] - M[a][Q-1-b]) / 2
// (a, b < H); odd Q adds the middle column Em[a] = M[a][H] and row
// Om[b] = M[H][b]
template <int Q>
struct EOTab {
  static constexpr int H = Q / 2;
  double E[H * H], O[H * H];
  double Em[H], Om[H];
};

template <int S, int P>
struct DTab {
  using Dm = Dims<S, P>;
  double d0[Dm::Q0 * Dm::Q0];
  double d1[Dm::Q1 * Dm::Q1];
  double d2[Dm::Q2 * Dm::Q2];
  // even-odd forms of D_d and D_d^T on the Gauss-Lobatto directions
  EOTab<Dm::Q0> e0, e0t;
  EOTab<gll_dir(S, 1) ? Dm::Q1 : 2> e1, e1t;
  EOTab<gll_dir(S, 2) ? Dm::Q2 : 2> e2, e2t;
  // regular geometry: Duffy factor a_k = 1/(1 - z2[k]) and scaled dir-2
  // weights, per k (uniform operands of the unrolled metric loop)
  double ak[Dm::Q2];
  double w2k[Dm::Q2];
};

// Layout of the per-basis device table buffer ("gtab"), runtime indexed.
template <int S, int P>
struct GLayout {
  using Dm = Dims<S, P>;
  // [0, RAGGED) is what the ragged r <-> k sweeps read (copied to shared
  // memory where kSmemTab says so)
  static constexpr int C2 = 0;                           // dir-2 family values
  static constexpr int DC2 = C2 + Dm::Q2 * Dm::NTRI;     // dir-2 family derivatives
  static constexpr int PAIRS = DC2 + Dm::Q2 * Dm::NTRI;  // NPAIR x 4 ints (16-byte aligned)
  static constexpr int RAGGED = PAIRS + 2 * Dm::NPAIR;
  static constexpr int REGK = PAIRS + 2 * Dm::NPAIR;     // [6][k][i*Q1+j]: refw,g00,g10,g11,g20,g21
  static constexpr int REFW = REGK + 6 * Dm::NQ;         // [i][j][k] refw
  static constexpr int B1 = REFW + Dm::NQ;               // tet dir-1 family values
  static constexpr int DB1 = B1 + Dm::Q1 * Dm::NTRI;     // tet dir-1 family derivatives
  // regular-geometry metric, per (i, j) line: [4][i*Q1+j] = w0 w1 (scaled
  // 1D weights), c00, c20, c21 with G00 = a c00, G20 = a c20, G21 = a c21,
  // a = 1/(1 - z2[k]) (DTab::ak); tet G10 = G20, G11 = 2a (pyr, tet)
  static constexpr int REGIJ = DB1 + Dm::Q1 * Dm::NTRI;
  static constexpr int SIZE = REGIJ + 4 * Dm::Q0 * Dm::Q1;
};

// Geometry payload addressing: [E/PW][C][NQ][PW], i.e. PW = EB elements
// interleaved innermost, so a half-warp's EB lanes read consecutive
// doubles; plain [E][C][NQ] when PW = 1.
template <int PW>
__device__ __forceinline__ long long pay_base(long long e, int C, int N) {
  if constexpr (PW == 1) {
    return e * (long long)C * N;
  } else {
    return (e / PW) * (long long)C * N * PW + (e % PW);
  }
}

struct Ctx {
  long long e0;    // first element of this CTA's tile
  long long E;     // real elements (loads guarded by e < E)
  long long Epad;  // padded elements = groups * W (stores guarded by e < Epad)
  int W;           // interleave width of the field layout
};

// index of data point 0 of element e in a lane-major (G, N, W) component
__device__ __forceinline__ long long lane_base(long long e, int N, int W) {
  if (W == 1) return e * N;
  const long long g = e / W;
  return g * (long long)N * W + (e - g * W);
}

// call f(std::integral_constant<int, v>) for the runtime value v in [0, N):
// lets a per-item selector (a warped-family slice index) become a
// compile-time constant, so its table entries stay uniform DFMA operands
template <int I, int N, class F>
__device__ __forceinline__ void dispatch(int v, F&& f) {
  if constexpr (I < N) {
    if (v == I) {
      f(std::integral_constant<int, I>{});
    } else {
      dispatch<I + 1, N>(v, f);
    }
  }
}

// ---- mbarrier / TMA bulk-copy helpers (shared::cta barriers, 1D bulk copies)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// global -> shared bulk copy (TMA, SASS UBLKCP) completing on barrier b;
// 16-byte aligned addresses, size a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// passes of a sweep's item loop unrolled together (independent items give
// the scheduler ILP across them; 1 keeps code size and registers minimal)
#ifndef SK_ITEMS_UNROLL
#define SK_ITEMS_UNROLL 1
#endif
constexpr int kItemsUnroll = SK_ITEMS_UNROLL;

// Thread index within the tile's thread group and the group barrier: a CTA
// (NT >= 64), or a single warp owning its own tile (NT == 32, the warp-tile
// kernels: no CTA barrier at all)
template <int NT>
__device__ __forceinline__ int tix() {
  if constexpr (NT == 32)
    return threadIdx.x & 31;
  else
    return threadIdx.x;
}
template <int NT>
__device__ __forceinline__ void csync() {
  if constexpr (NT == 32)
    __syncwarp();
  else
    __syncthreads();
}

template <class L, int NPASS, int NT, class F>
__device__ __forceinline__ void items(F&& f) {
#pragma unroll kItemsUnroll
  for (int w = tix<NT>(); w < L::EB * NPASS; w += NT) {
    const int ps = w / L::EB;
    f(w - ps * L::EB, ps);
  }
}

}  // namespace sk

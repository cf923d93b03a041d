// Operator kernels (SUM_FAC_TOP strategy) composed from the stages in
// sk_stages.cuh.  One CTA per tile of L::EB elements; grid.y = component.
//
//   k_helm    Helmholtz collocated (Alg. 6, operators.py:670-699); LAMW=false
//             is the stiffness operator (lam = 0: W stream not read).
//   k_mass    mass B^T W B (operators.py:622-633)
//   k_bwd     bwd_trans (operators.py:551-561)
//   k_iprod   iproduct_wrt_base (operators.py:564-574)
//   k_pderiv  phys_deriv (operators.py:577-596)
//   k_ipderiv iproduct_wrt_deriv_base (operators.py:599-619), evaluated as
//             B^T sum_k D_k^T (W v_k): D_k B equals the derivative tables
//             exactly for these polynomial spaces (test_operators.py:83-114)
//
// Geometry payloads (sk_payload_pack / the device geometry builder), all
// [E/PW][C][n][PW] with PW elements innermost (pay_base):
//   HELMHOLTZ deformed C=7, n=NQ in k-major point order [k][i*Q1+j]:
//             Lam' = G^T Lam G (6 unique) and wJ.  The Duffy chain rule is
//             folded into the metric so the kernel applies one symmetric
//             3x3 per point.  regular C=8, n=1: Lam (6), |J|, 0.
//   W         deformed C=1, n=NQ standard order; regular C=1, n=1 (|J|).
//   DERIV     deformed C=9, n=NQ k-major: T[m][j] = sum_i G[i][m] dxi[i][j];
//             regular C=9, n=1: dxi.
#pragma once

#include "sk_stages.cuh"
#include "sk_tune.h"

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
  long long pf_ahead;  // tiles between a CTA and the one whose input it prefetches
  int W;
  int c0_nx, c0_ny;  // assembled C0 hex slab (fused gather from the global DOF vector)
  int pad_;
  double lam;
  const int* __restrict__ c0map;  // assembled C0, mapped meshes: compact l2g (fused gather)
};

// Assembled C0 hex slab: the coefficient tile gathered straight from the
// global C0 DOF vector x (fuses sk_c0_gather into the Helmholtz load; the
// map is assembly.cu's: element e = (ez*ny + ey)*nx + ex, 1D DOF of mode k of
// element el = el*P + (0, P, k-1 for k = 0, 1, >= 2)).  Consecutive threads
// take consecutive elements of one mode (addresses P doubles apart; the
// neighbouring modes' loads hit the same lines in L1).
template <class L, int P, int NT>
__device__ __forceinline__ void load_tile_c0(const double* __restrict__ x, const Ctx& c, int nx, int ny, double* xs) {
  constexpr int P1 = P + 1, NM = P1 * P1 * P1, EB = L::EB, XS = L::XSTR;
  static_assert(NT % EB == 0, "a thread keeps one tile element");
  const long long Nx = (long long)nx * P + 1, Ny = (long long)ny * P + 1;
  auto md = [](long long el, int k) { return el * P + (k == 0 ? 0 : k == 1 ? P : k - 1); };
  // g = threadIdx.x + k NT walks (m, e) = (g / EB, g % EB): the element is
  // fixed per thread, so its (ex, ey, ez) -- runtime divisions -- are
  // computed once instead of per coefficient
  const int e = threadIdx.x % EB;
  const long long eg = c.e0 + e;
  const bool live = eg < c.E;
  const long long ex = eg % nx, ey = (eg / nx) % ny, ez = eg / ((long long)nx * ny);
  for (int m = threadIdx.x / EB; m < NM; m += NT / EB) {
    double v = 0.0;
    if (live) {
      const int r = m % P1, q = (m / P1) % P1, p = m / (P1 * P1);
      v = __ldg(x + (md(ez, r) * Ny + md(ey, q)) * Nx + md(ex, p));
    }
    xs[m * XS + e] = v;
  }
}

// Assembled C0 on a mapped mesh (prism / tet / pyramid): the coefficient
// tile gathered straight from the global DOF vector x through the compact
// map (l2gs[e * NM + m] = (global index << 1) | negative sign, as
// sk_c0_gather_map32), fusing the gather into the Helmholtz load.  Threads
// walk the map element-major (coalesced map reads; x is L2-resident).
template <class L, int NM, int NT>
__device__ __forceinline__ void load_tile_mapped(const double* __restrict__ x, const Ctx& c,
                                                 const int* __restrict__ l2gs, double* xs) {
  constexpr int EB = L::EB, XS = L::XSTR;
  const long long lim = (c.E - c.e0) * NM;
  const int* mp = l2gs + c.e0 * NM;
  for (int g = threadIdx.x; g < EB * NM; g += NT) {
    const int e = g / NM, m = g - e * NM;
    double v = 0.0;
    if (g < lim) {
      const int t = __ldg(mp + g);
      const double xv = __ldg(x + (t >> 1));
      v = (t & 1) ? -xv : xv;
    }
    xs[m * XS + e] = v;
  }
}

// arguments of the non-collocated Helmholtz: value and derivative tables
template <int S, int P>
struct NcArgs {
  FwdTab<S, P> B;   // psi values
  FwdTab<S, P> DB;  // psi derivatives (reference dmode tables, shapes.py:555-583)
  const double* __restrict__ in;
  double* __restrict__ out;
  const double* __restrict__ pay;
  const double* __restrict__ gtab;
  long long E, Epad;
  long long in_cstride, out_cstride;
  long long pf_ahead;
  int W;
  int pad_;
  double lam;
};

template <int EB>
__device__ __forceinline__ Ctx make_ctx(long long tile, long long E, long long Epad, int W) {
  Ctx c;
  c.e0 = tile * EB;
  c.E = E;
  c.Epad = Epad;
  c.W = W;
  return c;
}

// ---------------------------------------------------------------------------
// L2 prefetch by one warp: bulk TMA prefetches (cp.async.bulk.prefetch.L2,
// SASS UBLKPF) of [lo, hi) bytes of an allocation of `cap` bytes, in 32 KB
// pieces spread over the lanes.
__device__ __forceinline__ void l2_prefetch(const void* base, long long lo, long long hi, long long cap) {
  const int lane = threadIdx.x & 31;
  hi = hi < cap ? hi : cap;
  // bulk copies need 16-byte aligned absolute addresses and sizes; rounding
  // the start down stays inside the allocation (allocations are 256-aligned)
  const unsigned long long a0 = (reinterpret_cast<unsigned long long>(base) + lo) & ~15ULL;
  const unsigned long long a1 = (reinterpret_cast<unsigned long long>(base) + hi) & ~15ULL;
  for (unsigned long long a = a0 + (unsigned long long)lane * 32768; a < a1; a += 32ULL * 32768) {
    const unsigned long long n = a1 - a < 32768 ? a1 - a : 32768;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)n) : "memory");
  }
}

// bytes of the coefficient/field range touched by elements [e0, e0 + n)
__device__ __forceinline__ void field_range(long long e0, long long n, int N, int W, long long* lo, long long* hi) {
  *lo = (e0 / W) * (long long)N * W * 8;
  *hi = ((e0 + n - 1) / W + 1) * (long long)N * W * 8;
}


// prefetch the payload chunk of elements [e0, e0 + n): C*N doubles per
// element, PW-element lane groups (pay_base layout).  CR <= C: only the
// first CR components are read (stiffness skips wJ, the last of the 7
// Helmholtz components); with n <= PW (one tile = one lane group) they are
// one contiguous range.
template <int PW>
__device__ __forceinline__ void prefetch_payload(const double* pay, long long e0, long long n, long long E, long long C,
                                                 long long N, long long CR = -1) {
  if (n <= 0) return;
  const long long per = C * N * 8;
  const long long lo = (e0 / PW) * PW * per;
  long long hi = ((e0 + n + PW - 1) / PW) * PW * per;
  if (CR >= 0 && CR < C && n <= PW && e0 % PW == 0) hi = lo + CR * N * PW * 8;
  l2_prefetch(pay, lo, hi, ((E + PW - 1) / PW) * PW * per);
}

template <int NIN>
__device__ __forceinline__ void prefetch_field(const double* in, long long cstride, int ncomp, long long e0, long long n,
                                               long long Epad, int W) {
  if (n <= 0) return;
  long long lo, hi;
  field_range(e0, n, NIN, W, &lo, &hi);
  for (int c = 0; c < ncomp; ++c) l2_prefetch(in + c * cstride, lo, hi, Epad * NIN * 8);
}

// Tile driver: one CTA per tile (a persistent loop lets the compiler keep
// the loop-invariant table operands in registers, which costs occupancy at
// high order).  Warp 0 first prefetches into L2 the tile's geometry payload
// (consumed mid-tile, by the metric sweep) and the input field of the tile
// one resident wave ahead (A.pf_ahead tiles), which a later CTA will load.
template <class Op, class Args>
__global__ void __launch_bounds__(Op::NT, Op::MINB) k_tile(const __grid_constant__ Args A) {
  extern __shared__ double sm[];
  const long long t = blockIdx.x;
  if (threadIdx.x < 32) {
    const long long ntiles = (A.Epad + Op::EB - 1) / Op::EB;
    if (Op::GEO_PF_AT_START) Op::prefetch_geo(A, t);
    if (t + A.pf_ahead < ntiles) Op::prefetch_in(A, t + A.pf_ahead);
  }
  Op::run(A, t, sm);
}

// Persistent driver: one resident wave of CTAs strides over the tiles.  The
// coefficient loads of tile t + grid are issued (into registers) before tile
// t's sweeps; warp 0 prefetches into L2 the coefficients two tiles ahead and
// (from inside the body, right after the metric sweep) the geometry of the
// next tile, so the global latency of every tile after the first overlaps
// the previous tile's arithmetic while L2 holds ~one wave of geometry.
template <class Op, class Args>
__global__ void __launch_bounds__(Op::NT, Op::MINB) k_persist(const __grid_constant__ Args A) {
  extern __shared__ double sm[];
  const long long ntiles = (A.Epad + Op::EB - 1) / Op::EB;
  const long long stride = gridDim.x;
  long long t = blockIdx.x;
  typename Op::Pre pre;
  if (t < ntiles) {
    if (threadIdx.x < 32) {
      Op::prefetch_geo(A, t);
      if (t + stride < ntiles) Op::prefetch_in(A, t + stride);
    }
    Op::pre_load(A, t, pre);
  }
  for (; t < ntiles; t += stride) {
    if (threadIdx.x < 32 && t + 2 * stride < ntiles) Op::prefetch_in(A, t + 2 * stride);
    __syncthreads();  // the previous tile is done with the staging area
    Op::pre_put(A, pre, sm);
    if (t + stride < ntiles) Op::pre_load(A, t + stride, pre);
    __syncthreads();
    // the body prefetches the next tile's geometry once its own is consumed,
    // so the L2 holds about one wave of geometry at any time
    Op::body(A, t, sm, t + stride < ntiles ? t + stride : -1);
  }
}

// copy [0, GLayout::RAGGED) of the device table buffer (ragged sweep slices and
// pairs) to shared memory (kSmemTab configurations); the caller's barrier
// after the tile load publishes it
template <int S, int P, int NT>
__device__ __forceinline__ void stage_tables(const double* __restrict__ gtab, double* st) {
  for (int t = threadIdx.x; t < GLayout<S, P>::RAGGED; t += NT) st[t] = __ldg(gtab + t);
}

// Persistent driver with TMA-staged coefficient tiles: the next tile's
// coefficient block (interleave width 1: EB x NM contiguous doubles) is
// bulk-copied (SASS UBLKCP) into a double buffer behind the Op's shared
// memory while the current tile runs, completing on an mbarrier, then
// transposed smem-to-smem into the staging area (plane 1) -- no registers
// held across the tile (unlike k_persist's register-staged next tile) and
// no exposed load latency at the tile's first barrier (unlike k_tile).
// Ragged last tiles, other interleave widths and unaligned component
// offsets take load_tile.  The ragged tables (SMT) are staged once.
template <class Op, class Args, int NM, int SMEM0>
struct PersistTma {
  static constexpr int CB = Op::EB * NM + 2;  // one buffer: the block plus 16-byte rounding
  static constexpr int CBUF = (SMEM0 / 8 + 1) / 2 * 2;
  static constexpr int MBAR = CBUF + 2 * ((CB + 1) / 2 * 2);
  static constexpr int SMEM = MBAR * 8 + 2 * 8;
};

template <class Op, class Args, int NM, int SMEM0>
__global__ void __launch_bounds__(Op::NT, Op::MINB) k_persist_tma(const __grid_constant__ Args A) {
  using T = PersistTma<Op, Args, NM, SMEM0>;
  using L = typename Op::LayT;
  constexpr int EB = Op::EB, NT = Op::NT, CBS = (T::CB + 1) / 2 * 2;
  extern __shared__ double sm[];
  double* cbuf = sm + T::CBUF;
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(sm + T::MBAR);
  double* xs = sm + EB * L::PLANE;
  const long long ntiles = (A.Epad + EB - 1) / EB;
  const long long stride = gridDim.x;
  const double* src = A.in + blockIdx.y * A.in_cstride;
  // a whole tile's block (interleave width 1: EB * NM contiguous doubles)
  // moves as the 16-byte-aligned range covering it; not when that range
  // would end past the component's last element
  auto span = [&](long long t, unsigned long long& a0, unsigned& bytes, int& off) {
    const long long e0 = t * EB;
    const unsigned long long a = reinterpret_cast<unsigned long long>(src + e0 * NM);
    const unsigned long long end = a + (unsigned long long)EB * NM * 8;
    a0 = a & ~15ULL;
    off = (int)((a - a0) / 8);
    bytes = (unsigned)(((end + 15) & ~15ULL) - a0);
    return A.W == 1 && e0 + EB <= A.E && (e0 + EB < A.E || (end & 15) == 0);
  };
  auto issue = [&](long long tt, int buf) {
    unsigned long long a0;
    unsigned bytes;
    int off;
    if (span(tt, a0, bytes, off)) {
      mbar_expect_tx(&mb[buf], bytes);
      bulk_g2s(cbuf + buf * CBS, reinterpret_cast<const void*>(a0), bytes, &mb[buf]);
    }
  };
  long long t = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    mbar_fence_init();
    if (t < ntiles) issue(t, 0);
  }
  if constexpr (Op::SMT) stage_tables<Op::S_, Op::P_, NT>(A.gtab, sm + L::TABOFF);
  if (threadIdx.x < 32 && t < ntiles) Op::prefetch_geo(A, t);
  for (int i = 0; t < ntiles; t += stride, ++i) {
    const int b = i & 1;
    if (threadIdx.x == 0 && t + stride < ntiles) issue(t + stride, b ^ 1);
    __syncthreads();  // the previous tile's store has read the staging area
    unsigned long long a0;
    unsigned bytes;
    int off;
    if (span(t, a0, bytes, off)) {
      mbar_wait(&mb[b], (i >> 1) & 1);
      const double* cb = cbuf + b * CBS + off;
      for (int g = threadIdx.x; g < EB * NM; g += NT) {
        const int e = g / NM, m = g - e * NM;
        xs[m * L::XSTR + e] = cb[g];
      }
    } else {
      load_tile<L, NM, NT>(src, make_ctx<EB>(t, A.E, A.Epad, A.W), xs);
    }
    __syncthreads();
    Op::body(A, t, sm, t + stride < ntiles ? t + stride : -1);
  }
}

// ---------------------------------------------------------------------------
// Helmholtz, collocated: 9 sweeps + coefficient tile staging, 10 CTA barriers
template <int S, int P, class L, int NT_, int PW, int GEO, bool LAMW, int MINB_, int C0 = 0, int RING = 0>
struct k_helm {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr int S_ = S, P_ = P;
  using LayT = L;
  // TMA geometry ring (RING > 0 slots, sk_tune.h kGeoRing): slot s holds one
  // k-slice [C][Q0*Q1][PW] of the tile's payload, after the work planes
  // (and staged tables); then RING "full" and RING "empty" mbarriers
  static constexpr int RING_C = LAMW ? 7 : 6;
  static constexpr int RING_N = Dims<S, P>::Q0 * Dims<S, P>::Q1 * PW;  // doubles per component slice
  static constexpr int RING_SLOT = RING_C * RING_N;
  static constexpr int RING_OFF =
      ((smem_tables(0, S, P) ? L::TABOFF + GLayout<S, P>::RAGGED : L::SMEM_DOUBLES) + 1) / 2 * 2;
  static constexpr int RING_WARPS = (EB * Dims<S, P>::Q0 * Dims<S, P>::Q1 + 31) / 32;
  static_assert(RING == 0 || (GEO == GEO_DEFORMED && !C0 && EB == PW && RING_N % 2 == 0 &&
                              EB * Dims<S, P>::Q0 * Dims<S, P>::Q1 <= NT_),
                "geometry ring: deformed, one metric-sweep item per thread, 16-byte slices");
  __device__ static unsigned long long* ring_bars(double* sm) {
    return reinterpret_cast<unsigned long long*>(sm + RING_OFF + RING * RING_SLOT);
  }
  // thread 0: TMA bulk copies of k-slice k of this tile's payload into slot s
  __device__ static void ring_issue(const OpArgs<S, P>& A, long long tile, int k, int s, double* sm) {
    constexpr long long NQ = Dims<S, P>::NQ;
    unsigned long long* bars = ring_bars(sm);
    const double* src = A.pay + pay_base<PW>(tile * EB, 7, (int)NQ) + (long long)k * RING_N;
    double* dst = sm + RING_OFF + s * RING_SLOT;
    mbar_expect_tx(&bars[s], RING_SLOT * 8);
#pragma unroll
    for (int cc = 0; cc < RING_C; ++cc) bulk_g2s(dst + cc * RING_N, src + cc * NQ * PW, RING_N * 8, &bars[s]);
  }
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 7, Dims<S, P>::NQ, LAMW ? 7 : 6);
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    if constexpr (C0) return;  // input is the global DOF vector, read through L1
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NM>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  static constexpr bool SMT = smem_tables(0, S, P);
  static_assert(!(SMT && tuned_persist(0, S, P)), "the persistent driver does not stage the tables");
  static constexpr bool PERSIST = !C0;  // the register-staged next tile assumes the field layout
  static constexpr bool GEO_PF_AT_START = geo_prefetch(S, P) & 1;
  using Pre = TileRegs<L, Dims<S, P>::NM, NT_>;
  __device__ static void pre_load(const OpArgs<S, P>& A, long long t, Pre& p) {
    p.load(A.in + blockIdx.y * A.in_cstride, make_ctx<L::EB>(t, A.E, A.Epad, A.W));
  }
  __device__ static void pre_put(const OpArgs<S, P>& A, const Pre& p, double* sm) { p.put(A.W, sm + L::EB * L::PLANE); }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
    using Dm = Dims<S, P>;
    const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
    if constexpr (RING > 0) {
      // first slices in flight before the coefficient load: they land
      // during the F and M1 sweeps
      if (threadIdx.x == 0) {
        unsigned long long* bars = ring_bars(sm);
        for (int s = 0; s < RING; ++s) {
          mbar_init(&bars[s], 1);
          mbar_init(&bars[RING + s], RING_WARPS);
        }
        mbar_fence_init();
        if (c.e0 < c.E)
          for (int s = 0; s < RING && s < Dims<S, P>::Q2; ++s) ring_issue(A, tile, s, s, sm);
      }
    }
    if constexpr (C0 == 2)  // mapped mesh: compact l2g
      load_tile_mapped<L, Dm::NM, NT>(A.in, c, A.c0map, sm + L::EB * L::PLANE);
    else if constexpr (C0)  // structured hex slab
      load_tile_c0<L, P, NT>(A.in, c, A.c0_nx, A.c0_ny, sm + L::EB * L::PLANE);
    else
      load_tile<L, Dm::NM, NT>(A.in + blockIdx.y * A.in_cstride, c, sm + L::EB * L::PLANE);
    if constexpr (SMT) stage_tables<S, P, NT>(A.gtab, sm + L::TABOFF);
    __syncthreads();
    body(A, tile, sm, -1);
  }
  // M1 .. M3: the quadrature-point part of the collocated pipeline (u, v0
  // in planes UO / V0O on entry; U = lam W u + D1^T w1 + D2^T w2 and the
  // metric-weighted w0 in V0O on exit), shared by the fused kernel and the
  // staged quadrature-point kernel (k_qp)
  __device__ static __forceinline__ void middle(const OpArgs<S, P>& A, const Ctx& c, double* sm, long long tile,
                                                long long tnext) {
  using Dm = Dims<S, P>;
  constexpr int Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2;
  constexpr int NQ = Dm::NQ, PL = L::PLANE;
  constexpr int UO = 0, V0O = PL, V1O = 2 * PL;
  // M1: v1 = D1 u along j
  items<L, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double u[Q1], v[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) u[j] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    line_dd<S, P, 1>(A.D, u, v);
#pragma unroll
    for (int j = 0; j < Q1; ++j) sm[L::at(e, V1O + (i * Q1 + j) * S2 + k)] = v[j];
  });
  __syncthreads();
  // M2: v2 = D2 u along k; metric w = Lam' v per point; lam W u; D2^T w2
  items<L, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    const int row = ps * S2;  // (i,j) row, ps = i*Q1 + j
    if constexpr (m2_lowreg(S, P) && LAMW && GEO == GEO_DEFORMED && RING == 0) {
      // low-register form (bit-identical): u lives only through D2, lam W u
      // goes straight to the U plane (u_k re-read from it), and the D2^T
      // accumulator is loaded after the metric loop -- two Q2-long register
      // lines at any time instead of three plus the geometry chunk
      double w2[Q2];
      {
        double u[Q2];
#pragma unroll
        for (int k = 0; k < Q2; ++k) u[k] = sm[L::at(e, UO + row + k)];
        line_dd<S, P, 2>(A.D, u, w2);
      }
      const double* g = A.pay + pay_base<PW>(live ? eg : 0, 7, NQ) + (long long)ps * PW;
      constexpr int CH = Q2 <= 6 ? Q2 : kGeoChunk;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        if (k > 0 && k % CH == 0) asm volatile("" ::: "memory");
        const double* gk = g + (long long)k * (Q0 * Q1) * PW;
        const double l00 = live ? __ldcs(gk + 0LL * NQ * PW) : 0.0, l01 = live ? __ldcs(gk + 1LL * NQ * PW) : 0.0,
                     l02 = live ? __ldcs(gk + 2LL * NQ * PW) : 0.0, l11 = live ? __ldcs(gk + 3LL * NQ * PW) : 0.0,
                     l12 = live ? __ldcs(gk + 4LL * NQ * PW) : 0.0, l22 = live ? __ldcs(gk + 5LL * NQ * PW) : 0.0;
        const double v0 = sm[L::at(e, V0O + row + k)], v1 = sm[L::at(e, V1O + row + k)], v2 = w2[k];
        const double a0 = fma(l02, v2, fma(l01, v1, l00 * v0));
        const double a1 = fma(l12, v2, fma(l11, v1, l01 * v0));
        w2[k] = fma(l22, v2, fma(l12, v1, l02 * v0));
        sm[L::at(e, V0O + row + k)] = a0;
        sm[L::at(e, V1O + row + k)] = a1;
        if constexpr (LAMW) {
          const double wj = live ? __ldcs(gk + 6LL * NQ * PW) : 0.0;
          sm[L::at(e, UO + row + k)] = (A.lam * wj) * sm[L::at(e, UO + row + k)];
        }
      }
      double z[Q2];
#pragma unroll
      for (int k = 0; k < Q2; ++k) z[k] = LAMW ? sm[L::at(e, UO + row + k)] : 0.0;
      line_ddt_acc<S, P, 2>(A.D, w2, z);
#pragma unroll
      for (int k = 0; k < Q2; ++k) sm[L::at(e, UO + row + k)] = z[k];
      return;
    }
    double u[Q2], w2[Q2], z[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) u[k] = sm[L::at(e, UO + row + k)];
    line_dd<S, P, 2>(A.D, u, w2);  // w2 holds v2 until overwritten per point
    if constexpr (RING > 0) {
      // geometry from the TMA ring: wait for slice k, read it from shared
      // memory, release the slot (one arrival per warp); thread 0 refills it
      // with slice k + RING once every warp has released it
      unsigned long long* bars = ring_bars(sm);
      const double* ring = sm + RING_OFF;
      const bool tile_live = c.e0 < c.E;  // uniform: an all-padding tile issued no copies
      const unsigned amask = __activemask();
      const bool leader = (int)(threadIdx.x & 31) == __ffs(amask) - 1;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const int s = k % RING;
        const unsigned ph = (k / RING) & 1;
        if (tile_live) mbar_wait(&bars[s], ph);
        const double* gk = ring + s * RING_SLOT + ps * PW + e;
        const double l00 = live ? gk[0 * RING_N] : 0.0, l01 = live ? gk[1 * RING_N] : 0.0,
                     l02 = live ? gk[2 * RING_N] : 0.0, l11 = live ? gk[3 * RING_N] : 0.0,
                     l12 = live ? gk[4 * RING_N] : 0.0, l22 = live ? gk[5 * RING_N] : 0.0;
        double wj = 0.0;
        if constexpr (LAMW) wj = live ? gk[6 * RING_N] : 0.0;
        if (tile_live) {
          __syncwarp(amask);
          if (leader) mbar_arrive(&bars[RING + s]);
          if (threadIdx.x == 0 && k + RING < Q2) {
            mbar_wait(&bars[RING + s], ph);
            ring_issue(A, tile, k + RING, s, sm);
          }
        }
        const double v0 = sm[L::at(e, V0O + row + k)], v1 = sm[L::at(e, V1O + row + k)], v2 = w2[k];
        const double a0 = fma(l02, v2, fma(l01, v1, l00 * v0));
        const double a1 = fma(l12, v2, fma(l11, v1, l01 * v0));
        w2[k] = fma(l22, v2, fma(l12, v1, l02 * v0));
        sm[L::at(e, V0O + row + k)] = a0;
        sm[L::at(e, V1O + row + k)] = a1;
        z[k] = LAMW ? (A.lam * wj) * u[k] : 0.0;
      }
    } else if constexpr (GEO == GEO_DEFORMED) {
      const double* g = A.pay + pay_base<PW>(live ? eg : 0, 7, NQ) + (long long)ps * PW;
      // points in chunks of CH: a compiler fence between chunks keeps ptxas
      // from hoisting all 7*Q2 geometry loads (register pressure at high P)
      constexpr int CH = Q2 <= 6 ? Q2 : kGeoChunk;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        if (k > 0 && k % CH == 0) asm volatile("" ::: "memory");
        const double* gk = g + (long long)k * (Q0 * Q1) * PW;
        const double l00 = live ? __ldcs(gk + 0LL * NQ * PW) : 0.0, l01 = live ? __ldcs(gk + 1LL * NQ * PW) : 0.0,
                     l02 = live ? __ldcs(gk + 2LL * NQ * PW) : 0.0, l11 = live ? __ldcs(gk + 3LL * NQ * PW) : 0.0,
                     l12 = live ? __ldcs(gk + 4LL * NQ * PW) : 0.0, l22 = live ? __ldcs(gk + 5LL * NQ * PW) : 0.0;
        const double v0 = sm[L::at(e, V0O + row + k)], v1 = sm[L::at(e, V1O + row + k)], v2 = w2[k];
        const double a0 = fma(l02, v2, fma(l01, v1, l00 * v0));
        const double a1 = fma(l12, v2, fma(l11, v1, l01 * v0));
        w2[k] = fma(l22, v2, fma(l12, v1, l02 * v0));
        sm[L::at(e, V0O + row + k)] = a0;
        sm[L::at(e, V1O + row + k)] = a1;
        if constexpr (LAMW) {
          const double wj = live ? __ldcs(gk + 6LL * NQ * PW) : 0.0;
          z[k] = (A.lam * wj) * u[k];
        } else {
          z[k] = 0.0;
        }
      }
    } else {
      // affine: Lam per element, G and reference weights per point
      constexpr int RW = kRegPW;
      const double* ge = A.pay + pay_base<RW>(live ? eg : 0, 8, 1);
      const double l00 = __ldg(ge + 0 * RW), l01 = __ldg(ge + 1 * RW), l02 = __ldg(ge + 2 * RW),
                   l11 = __ldg(ge + 3 * RW), l12 = __ldg(ge + 4 * RW), l22 = __ldg(ge + 5 * RW),
                   jac = __ldg(ge + 6 * RW);
      // G and the reference weights factor over the tensor directions: the
      // (i, j) factors come from a small per-line table, the k factors are
      // uniform parameter-space constants (no per-point loads)
      constexpr int N2 = Q0 * Q1;
      const double* rij = A.gtab + GLayout<S, P>::REGIJ + ps;
      const double wij = __ldg(rij);
      double c00 = 0.0, c20 = 0.0, c21 = 0.0;
      if constexpr (S != HEX) {
        c00 = __ldg(rij + 1 * N2);
        c20 = __ldg(rij + 2 * N2);
        if constexpr (S != PRISM) c21 = __ldg(rij + 3 * N2);
      }
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const double rw = wij * A.D.w2k[k];
        const double v0 = sm[L::at(e, V0O + row + k)], v1 = sm[L::at(e, V1O + row + k)], v2 = w2[k];
        double t0 = v0, t1 = v1, t2 = v2;
        double g00 = 1.0, g10 = 0.0, g11 = 1.0, g20 = 0.0, g21 = 0.0;
        if constexpr (S != HEX) {
          const double a = A.D.ak[k];
          g00 = a * c00;
          g20 = a * c20;
          if constexpr (S == PRISM) {
            t0 = g00 * v0;
            t2 = fma(g20, v0, v2);
          } else {
            g11 = 2.0 * a;
            g21 = a * c21;
            if constexpr (S == TET) {
              g10 = g20;
              t1 = fma(g11, v1, g10 * v0);
            } else {
              t1 = g11 * v1;
            }
            t0 = g00 * v0;
            t2 = fma(g21, v1, fma(g20, v0, v2));
          }
        }
        const double s0 = rw * fma(l02, t2, fma(l01, t1, l00 * t0));
        const double s1 = rw * fma(l12, t2, fma(l11, t1, l01 * t0));
        const double s2 = rw * fma(l22, t2, fma(l12, t1, l02 * t0));
        double a0 = s0, a1 = s1;
        if constexpr (S == PRISM) {
          a0 = fma(g20, s2, g00 * s0);
        } else if constexpr (S == PYR) {
          a0 = fma(g20, s2, g00 * s0);
          a1 = fma(g21, s2, g11 * s1);
        } else if constexpr (S == TET) {
          a0 = fma(g20, s2, fma(g10, s1, g00 * s0));
          a1 = fma(g21, s2, g11 * s1);
        }
        sm[L::at(e, V0O + row + k)] = live ? a0 : 0.0;
        sm[L::at(e, V1O + row + k)] = live ? a1 : 0.0;
        w2[k] = live ? s2 : 0.0;
        if constexpr (LAMW) {
          z[k] = live ? A.lam * ((u[k] * rw) * jac) : 0.0;
        } else {
          z[k] = 0.0;
        }
      }
    }
    line_ddt_acc<S, P, 2>(A.D, w2, z);
#pragma unroll
    for (int k = 0; k < Q2; ++k) sm[L::at(e, UO + row + k)] = z[k];
  });
  __syncthreads();
  if (tnext >= 0 && threadIdx.x < 32) prefetch_geo(A, tnext);
  // M3: U += D1^T w1 along j
  items<L, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double w[Q1], r[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) {
      w[j] = sm[L::at(e, V1O + (i * Q1 + j) * S2 + k)];
      r[j] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    }
    line_ddt_acc<S, P, 1>(A.D, w, r);
#pragma unroll
    for (int j = 0; j < Q1; ++j) sm[L::at(e, UO + (i * Q1 + j) * S2 + k)] = r[j];
  });
  __syncthreads();
  }
  __device__ static void body(const OpArgs<S, P>& A, long long tile, double* sm, long long tnext) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2;
  constexpr int NM = Dm::NM, PL = L::PLANE;
  constexpr int UO = 0, V0O = PL, TAo = 0, TBo = 2 * PL;
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  double* xs = sm + L::EB * PL;  // plane 1: coefficient tile staging

  if constexpr (SMT)  // ragged sweep tables staged in shared memory by run()
    stage_f1<S, P, L, NT, TAo, CoefIn<L, NM>, false, ragged_dispatch(0, S, P), ragged_split(0, S, P), prism_warp_pairs(0, S, P), true>(A.B, sm + L::TABOFF, CoefIn<L, NM>{xs}, sm);
  else
    stage_f1<S, P, L, NT, TAo, CoefIn<L, NM>, false, ragged_dispatch(0, S, P), ragged_split(0, S, P), prism_warp_pairs(0, S, P)>(A.B, A.gtab, CoefIn<L, NM>{xs}, sm);
  __syncthreads();
  stage_f2<S, P, L, NT, TAo, TBo>(A.B, A.gtab, sm);
  __syncthreads();
  if ((geo_prefetch(S, P) & 2) && tnext < 0 && threadIdx.x < 32) prefetch_geo(A, tile);
  // F3 + D0: u along i, v0 = D0 u
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double x[P1], u[Q0], v[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
    line_a0_eo<S, P>(A.B, x, u);
    line_dd<S, P, 0>(A.D, u, v);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      sm[L::at(e, UO + (i * Q1 + j) * S2 + k)] = u[i];
      sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)] = v[i];
    }
  });
  __syncthreads();
  middle(A, c, sm, tile, tnext);
  // B1: r = U + D0^T w0 along i, then B^T along dir 0
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double w[Q0], r[Q0], t[P1];
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      w[i] = sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)];
      r[i] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    }
    line_ddt_acc<S, P, 0>(A.D, w, r);
    line_a0t_eo<S, P>(A.B, r, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, L, NT, TAo, TBo>(A.B, A.gtab, sm);
  __syncthreads();
  if constexpr (SMT)
    stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(0, S, P), ragged_split(0, S, P), prism_warp_pairs(0, S, P), true>(A.B, sm + L::TABOFF, CoefOut<L, NM>{xs}, sm);
  else
    stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(0, S, P), ragged_split(0, S, P), prism_warp_pairs(0, S, P)>(A.B, A.gtab, CoefOut<L, NM>{xs}, sm);
  __syncthreads();
  store_tile<L, NM, NT>(dst, c, xs);
  }
};

// ---------------------------------------------------------------------------
// Staged collocated Helmholtz, quadrature-point kernel (the fused kernel
// split after BwdTrans and before the final B^T): u (NQ values per
// element, lane-major work buffer written by k_bwd) ->
// u' = lam W u + sum_m D_m^T (G^T Lam G) D_m u (k_helm::middle, the same
// sweeps and metric as the fused kernel), written for the unweighted B^T
// (k_iprod<GEO_UNIT>).  Only the middle sweeps' three planes are live, the
// coefficient-space stages run in their own two-plane kernels.
template <int S, int P, class L, int NT_, int PW, int GEO, bool LAMW, int MINB_>
struct k_qp {
  using H = k_helm<S, P, L, NT_, PW, GEO, LAMW, MINB_>;
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) { H::prefetch_geo(A, t); }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NQ>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
    using Dm = Dims<S, P>;
    constexpr int Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NQ = Dm::NQ, PL = L::PLANE;
    constexpr int UO = 0, V0O = PL;
    const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
    const double* src = A.in + blockIdx.y * A.in_cstride;
    double* dst = A.out + blockIdx.y * A.out_cstride;
    // u along i from the work buffer, v0 = D0 u
    items<L, Q1 * Q2, NT>([&](int e, int ps) {
      const int j = ps / Q2, k = ps - j * Q2;
      const long long eg = c.e0 + e;
      const bool live = eg < c.E;
      const long long base = lane_base(live ? eg : 0, NQ, c.W);
      double u[Q0], v[Q0];
#pragma unroll
      for (int i = 0; i < Q0; ++i) u[i] = live ? __ldcs(src + base + (long long)((i * Q1 + j) * Q2 + k) * c.W) : 0.0;
      line_dd<S, P, 0>(A.D, u, v);
#pragma unroll
      for (int i = 0; i < Q0; ++i) {
        sm[L::at(e, UO + (i * Q1 + j) * S2 + k)] = u[i];
        sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)] = v[i];
      }
    });
    __syncthreads();
    H::middle(A, c, sm, tile, -1);
    // u' = U + D0^T w0 along i, to the work buffer
    items<L, Q1 * Q2, NT>([&](int e, int ps) {
      const int j = ps / Q2, k = ps - j * Q2;
      const long long eg = c.e0 + e;
      if (eg >= c.Epad) return;
      const bool live = eg < c.E;
      double w[Q0], r[Q0];
#pragma unroll
      for (int i = 0; i < Q0; ++i) {
        w[i] = sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)];
        r[i] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
      }
      line_ddt_acc<S, P, 0>(A.D, w, r);
      const long long base = lane_base(eg, NQ, c.W);
#pragma unroll
      for (int i = 0; i < Q0; ++i) __stcs(dst + base + (long long)((i * Q1 + j) * Q2 + k) * c.W, live ? r[i] : 0.0);
    });
  }
};

// W at point l (standard order) of element eg for the W-payload family
template <int S, int P, int PW, int GEO>
__device__ __forceinline__ double w_at(const OpArgs<S, P>& A, long long eg, bool live, int l) {
  if (!live) return 0.0;
  if constexpr (GEO == GEO_UNIT) return 1.0;
  if constexpr (GEO == GEO_DEFORMED) {
    return __ldcs(A.pay + pay_base<PW>(eg, 1, Dims<S, P>::NQ) + (long long)l * PW);
  } else {
    return __ldg(A.gtab + GLayout<S, P>::REFW + l) * __ldg(A.pay + pay_base<PW>(eg, 1, 1));
  }
}

// ---------------------------------------------------------------------------
// Mass: F1, F2, fused (B, W, B^T) along dir 0, B2, B3
template <int S, int P, class L, int NT_, int PW, int GEO, int MINB_>
struct k_mass {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 1, Dims<S, P>::NQ);
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NM>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  static constexpr bool PERSIST = true;
  static constexpr bool GEO_PF_AT_START = true;
  using Pre = TileRegs<L, Dims<S, P>::NM, NT_>;
  __device__ static void pre_load(const OpArgs<S, P>& A, long long t, Pre& p) {
    p.load(A.in + blockIdx.y * A.in_cstride, make_ctx<L::EB>(t, A.E, A.Epad, A.W));
  }
  __device__ static void pre_put(const OpArgs<S, P>& A, const Pre& p, double* sm) { p.put(A.W, sm + L::EB * L::PLANE); }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
    using Dm = Dims<S, P>;
    const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
    load_tile<L, Dm::NM, NT>(A.in + blockIdx.y * A.in_cstride, c, sm + L::EB * L::PLANE);
    if constexpr (SMT) stage_tables<S, P, NT>(A.gtab, sm + L::TABOFF);
    __syncthreads();
    body(A, tile, sm, -1);
  }
  static constexpr bool SMT = smem_tables(1, S, P);
  __device__ static void body(const OpArgs<S, P>& A, long long tile, double* sm, long long tnext) {
    body_t(A, tile, sm, tnext, sm + L::TABOFF);
  }
  // stab: the staged ragged tables (SMT); NT == 32: one warp owns the tile
  // and every barrier is a warp barrier (k_mass_warp)
  __device__ static void body_t(const OpArgs<S, P>& A, long long tile, double* sm, long long tnext, const double* stab) {
    body_w(
        A, tile, sm, stab, [&](long long eg, bool live, int l, int) { return w_at<S, P, PW, GEO>(A, eg, live, l); },
        [] {},
        [&] {
          if (tnext >= 0 && threadIdx.x < 32) prefetch_geo(A, tnext);
        });
  }
  // wf(eg, live, point, tile element): the diagonal W entry; pre(): runs
  // before the W sweep; hook(): once every thread is past it (next-tile
  // prefetch / copy issue)
  template <class WF, class PRE, class HOOK>
  __device__ static void body_w(const OpArgs<S, P>& A, long long tile, double* sm, const double* stab, const WF& wf,
                                const PRE& pre, const HOOK& hook) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NM = Dm::NM;
  constexpr int PL = L::PLANE, TAo = 0, TBo = PL;
  constexpr bool WP = NT > 32 && prism_warp_pairs(1, S, P);
  constexpr bool EO = use_eo_mass(S, P);
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  double* xs = sm + L::EB * PL;  // plane 1 (TB): staging before F2 and after B2
  if constexpr (SMT)  // ragged sweep tables staged in shared memory
    stage_f1<S, P, L, NT, TAo, CoefIn<L, NM>, false, ragged_dispatch(1, S, P), ragged_split(1, S, P), WP, true, EO>(A.B, stab, CoefIn<L, NM>{xs}, sm);
  else
    stage_f1<S, P, L, NT, TAo, CoefIn<L, NM>, false, ragged_dispatch(1, S, P), ragged_split(1, S, P), WP, false, EO>(A.B, A.gtab, CoefIn<L, NM>{xs}, sm);
  csync<NT>();
  stage_f2<S, P, L, NT, TAo, TBo, false, EO>(A.B, A.gtab, sm);
  csync<NT>();
  pre();
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double x[P1], u[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
    line_a0_eo<S, P, EO>(A.B, x, u);
#pragma unroll
    for (int i = 0; i < Q0; ++i) u[i] *= wf(eg, live, (i * Q1 + j) * Q2 + k, e);
    line_a0t_eo<S, P, EO>(A.B, u, x);
#pragma unroll
    for (int p = 0; p < P1; ++p) sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = x[p];
  });
  csync<NT>();
  hook();
  stage_b2<S, P, L, NT, TAo, TBo, false, false, EO>(A.B, A.gtab, sm);
  csync<NT>();
  if constexpr (SMT)
    stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(1, S, P), ragged_split(1, S, P), WP, true, EO>(A.B, stab, CoefOut<L, NM>{xs}, sm);
  else
    stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(1, S, P), ragged_split(1, S, P), WP, false, EO>(A.B, A.gtab, CoefOut<L, NM>{xs}, sm);
  csync<NT>();
  store_tile<L, NM, NT>(dst, c, xs);
  }
};

// Mass, deformed, with the tile inputs moved by TMA bulk copies (SASS
// UBLKCP): a persistent CTA strides over its tiles; thread 0 issues the
// next tile's coefficient block (W = 1 layout: one contiguous range, double
// buffered) at the top of the current tile and the next tile's W payload
// (one contiguous PW-lane group) as soon as the current tile's W sweep is
// done, each completing on an mbarrier, so the global latency of both lands
// under the sum-factorisation sweeps instead of stalling the first barrier
// and the W sweep (ncu: 20 % + 14 % of samples in k_mass at tet P=4).
// Ragged last tiles and unaligned component offsets take the register path.
template <int S, int P, class L, int NT_, int PW, int MINB_>
struct MassTma {
  using K = k_mass<S, P, L, NT_, PW, GEO_DEFORMED, MINB_>;
  using Dm = Dims<S, P>;
  static constexpr int NT = NT_, EB = L::EB, NQ = Dm::NQ, NM = Dm::NM;
  static_assert(EB == PW, "one tile = one payload lane group");
  static constexpr int TAB = K::SMT ? GLayout<S, P>::RAGGED : 0;
  static constexpr int PBUF = (L::TABOFF + TAB + 1) / 2 * 2;         // NQ * PW doubles
  static constexpr int CBUF = PBUF + NQ * PW;                         // 2 x EB * NM doubles
  static constexpr int MBAR = (CBUF + 2 * EB * NM + 1) / 2 * 2;       // 3 mbarriers
  static constexpr int SMEM = MBAR * 8 + 3 * 8;
};

template <int S, int P, class L, int NT_, int PW, int MINB_>
__global__ void __launch_bounds__(NT_, MINB_) k_mass_tma(const __grid_constant__ OpArgs<S, P> A) {
  using M = MassTma<S, P, L, NT_, PW, MINB_>;
  using K = typename M::K;
  constexpr int EB = M::EB, NM = M::NM, NQ = M::NQ, NT = NT_;
  extern __shared__ double sm[];
  double* pbuf = sm + M::PBUF;
  double* cbuf = sm + M::CBUF;
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(sm + M::MBAR);  // [0,1] coefficients, [2] W
  const long long ntiles = (A.Epad + EB - 1) / EB;
  const long long stride = gridDim.x;
  const double* src = A.in + blockIdx.y * A.in_cstride;
  // a tile's coefficients come by TMA when it is whole and its range is
  // 16-byte aligned (W = 1: element-major, EB * NM contiguous doubles)
  auto coef_tma = [&](long long t) {
    const long long e0 = t * EB;
    return A.W == 1 && e0 + EB <= A.E && ((reinterpret_cast<unsigned long long>(src + e0 * NM) & 15) == 0);
  };
  constexpr unsigned CBYTES = EB * NM * 8, PBYTES = NQ * PW * 8;
  static_assert(CBYTES % 16 == 0 && PBYTES % 16 == 0, "bulk copies move multiples of 16 bytes");
  long long t = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    mbar_init(&mb[2], 1);
    mbar_fence_init();
    if (t < ntiles) {
      if (coef_tma(t)) {
        mbar_expect_tx(&mb[0], CBYTES);
        bulk_g2s(cbuf, src + t * EB * NM, CBYTES, &mb[0]);
      }
      mbar_expect_tx(&mb[2], PBYTES);
      bulk_g2s(pbuf, A.pay + t * EB * NQ, PBYTES, &mb[2]);
    }
  }
  if constexpr (K::SMT) stage_tables<S, P, NT>(A.gtab, sm + L::TABOFF);
  __syncthreads();
  double* xs = sm + EB * L::PLANE;  // plane 1: coefficient staging
  for (int i = 0; t < ntiles; t += stride, ++i) {
    const int b = i & 1;
    // next tile's coefficients into the other buffer (last read by tile i-1's
    // staging copy, before this tile's first barrier... and the one below)
    if (threadIdx.x == 0 && t + stride < ntiles && coef_tma(t + stride)) {
      mbar_expect_tx(&mb[b ^ 1], CBYTES);
      bulk_g2s(cbuf + (b ^ 1) * EB * NM, src + (t + stride) * EB * NM, CBYTES, &mb[b ^ 1]);
    }
    const Ctx c = make_ctx<EB>(t, A.E, A.Epad, A.W);
    if (coef_tma(t)) {
      mbar_wait(&mb[b], (i >> 1) & 1);
      const double* cb = cbuf + b * EB * NM;
      for (int g = threadIdx.x; g < EB * NM; g += NT) {
        const int e = g / NM, m = g - e * NM;
        xs[m * L::XSTR + e] = cb[g];
      }
    } else {
      load_tile<L, NM, NT>(src, c, xs);
    }
    __syncthreads();
    K::body_w(
        A, t, sm, sm + L::TABOFF,
        [&](long long, bool live, int l, int e) {
          return live ? pbuf[l * PW + e] : 0.0;
        },
        [&] { mbar_wait(&mb[2], i & 1); },
        [&] {  // every thread is done with pbuf: the next tile's W
          if (threadIdx.x == 0 && t + stride < ntiles) {
            mbar_expect_tx(&mb[2], PBYTES);
            bulk_g2s(pbuf, A.pay + (t + stride) * EB * NQ, PBYTES, &mb[2]);
          }
        });
  }
}

// Mass with one warp per tile of G elements (no CTA barriers): WPC warps
// per CTA each own a private two-plane tile and stride over the tiles
// independently, so one warp's global-load latency overlaps the others'
// sweeps without the CTA-wide barrier stalls of k_mass.
// The ragged tables (kSmemTab) are staged once per CTA after the tiles.
template <int S, int P, int G, int WPC_, int PW, int GEO>
struct MassWarp {
  using L = Lay<S, P, 2, G>;
  using K = k_mass<S, P, L, 32, PW, GEO, 1>;
  // warps per CTA: as asked, or as many as fit 200 KB of tiles
  static constexpr int WPC = WPC_ * L::SMEM_DOUBLES * 8 <= 200 * 1024 ? WPC_
                             : (200 * 1024) / (L::SMEM_DOUBLES * 8) > 0 ? (200 * 1024) / (L::SMEM_DOUBLES * 8) : 1;
  static constexpr int NT = WPC * 32;
  static constexpr int TABOFF = (WPC * L::SMEM_DOUBLES + 1) / 2 * 2;
  static constexpr int SMEM = (K::SMT ? TABOFF + GLayout<S, P>::RAGGED : WPC * L::SMEM_DOUBLES) * 8;
};

template <int S, int P, int G, int WPC_, int PW, int GEO>
__global__ void __launch_bounds__(MassWarp<S, P, G, WPC_, PW, GEO>::NT, kMassWarpMinB) k_mass_warp(const __grid_constant__ OpArgs<S, P> A) {
  using M = MassWarp<S, P, G, WPC_, PW, GEO>;
  constexpr int WPC = M::WPC;
  using L = typename M::L;
  using K = typename M::K;
  extern __shared__ double sm[];
  if constexpr (K::SMT) {
    for (int t = threadIdx.x; t < GLayout<S, P>::RAGGED; t += M::NT) sm[M::TABOFF + t] = __ldg(A.gtab + t);
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5;
  double* ws = sm + warp * L::SMEM_DOUBLES;
  const long long ntiles = (A.Epad + G - 1) / G;
  for (long long t = (long long)blockIdx.x * WPC + warp; t < ntiles; t += (long long)gridDim.x * WPC) {
    const Ctx c = make_ctx<G>(t, A.E, A.Epad, A.W);
    load_tile<L, Dims<S, P>::NM, 32>(A.in + blockIdx.y * A.in_cstride, c, ws + G * L::PLANE);
    __syncwarp();
    K::body_t(A, t, ws, -1, sm + M::TABOFF);
    __syncwarp();  // the store has read the staging area before the next load
  }
}

// ---------------------------------------------------------------------------
// BwdTrans: coefficients -> quadrature values
template <int S, int P, class L, int NT_, int MINB_>
struct k_bwd {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NM>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NM = Dm::NM;
  constexpr int PL = L::PLANE, TAo = 0, TBo = PL;
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  double* xs = sm + L::EB * PL;
  load_tile<L, NM, NT>(src, c, xs);
  __syncthreads();
  stage_f1<S, P, L, NT, TAo, CoefIn<L, NM>, false, ragged_dispatch(2, S, P), ragged_split(2, S, P), prism_warp_pairs(2, S, P)>(A.B, A.gtab, CoefIn<L, NM>{xs}, sm);
  __syncthreads();
  stage_f2<S, P, L, NT, TAo, TBo>(A.B, A.gtab, sm);
  __syncthreads();
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    double x[P1], u[Q0];
#pragma unroll
    for (int p = 0; p < P1; ++p) x[p] = sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)];
    line_a0_eo<S, P>(A.B, x, u);
    if (eg < c.Epad) {
      const long long base = lane_base(eg, Dm::NQ, c.W);
#pragma unroll
      for (int i = 0; i < Q0; ++i) dst[base + (long long)((i * Q1 + j) * Q2 + k) * c.W] = u[i];
    }
  });
  }
};

// ---------------------------------------------------------------------------
// IProductWRTBase: quadrature values -> coefficients, B^T W u
template <int S, int P, class L, int NT_, int PW, int GEO, int MINB_>
struct k_iprod {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 1, Dims<S, P>::NQ);
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NQ>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NM = Dm::NM;
  constexpr int PL = L::PLANE, TAo = 0, TBo = PL;
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  const double* src = A.in + blockIdx.y * A.in_cstride;
  double* dst = A.out + blockIdx.y * A.out_cstride;
  double* xs = sm + L::EB * PL;
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double u[Q0], t[P1];
    const long long base = lane_base(live ? eg : 0, Dm::NQ, c.W);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      const int l = (i * Q1 + j) * Q2 + k;
      u[i] = live ? __ldg(src + base + (long long)l * c.W) * w_at<S, P, PW, GEO>(A, eg, live, l) : 0.0;
    }
    line_a0t_eo<S, P>(A.B, u, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, L, NT, TAo, TBo>(A.B, A.gtab, sm);
  __syncthreads();
  stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(2, S, P), ragged_split(2, S, P), prism_warp_pairs(2, S, P)>(A.B, A.gtab, CoefOut<L, NM>{xs}, sm);
  __syncthreads();
  store_tile<L, NM, NT>(dst, c, xs);
  }
};

// ---------------------------------------------------------------------------
// PhysDeriv: u (1 component) -> du/dx_j (3 components)
template <int S, int P, class L, int NT_, int PW, int GEO, int MINB_>
struct k_pderiv {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 9, Dims<S, P>::NQ);
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NQ>(A.in, A.in_cstride, 1, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NQ = Dm::NQ;
  constexpr int PL = L::PLANE, UO = 0, V0O = PL, V1O = 2 * PL;
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    double u[Q0], v[Q0];
    const long long base = lane_base(live ? eg : 0, NQ, c.W);
#pragma unroll
    for (int i = 0; i < Q0; ++i) u[i] = live ? __ldg(A.in + base + (long long)((i * Q1 + j) * Q2 + k) * c.W) : 0.0;
    line_dd<S, P, 0>(A.D, u, v);
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      sm[L::at(e, UO + (i * Q1 + j) * S2 + k)] = u[i];
      sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)] = v[i];
    }
  });
  __syncthreads();
  items<L, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double u[Q1], v[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) u[j] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    line_dd<S, P, 1>(A.D, u, v);
#pragma unroll
    for (int j = 0; j < Q1; ++j) sm[L::at(e, V1O + (i * Q1 + j) * S2 + k)] = v[j];
  });
  __syncthreads();
  items<L, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    if (eg >= c.Epad) return;
    const int row = ps * S2;
    double u[Q2], v2[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) u[k] = sm[L::at(e, UO + row + k)];
    line_dd<S, P, 2>(A.D, u, v2);
    const long long base = lane_base(eg, NQ, c.W);
    const long long cs = A.out_cstride;
#pragma unroll
    for (int k = 0; k < Q2; ++k) {
      const double v0 = sm[L::at(e, V0O + row + k)], v1 = sm[L::at(e, V1O + row + k)], w = v2[k];
      double o[3];
      if constexpr (GEO == GEO_DEFORMED) {
        const double* g = A.pay + pay_base<PW>(live ? eg : 0, 9, NQ) + ((long long)k * (Q0 * Q1) + ps) * PW;
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          const double t0 = live ? __ldcs(g + (0LL * 3 + jj) * NQ * PW) : 0.0;
          const double t1 = live ? __ldcs(g + (1LL * 3 + jj) * NQ * PW) : 0.0;
          const double t2 = live ? __ldcs(g + (2LL * 3 + jj) * NQ * PW) : 0.0;
          o[jj] = fma(t2, w, fma(t1, v1, t0 * v0));
        }
      } else {
        const double* ge = A.pay + pay_base<PW>(live ? eg : 0, 9, 1);
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
          o[jj] = live ? fma(__ldg(ge + (6 + jj) * PW), t2, fma(__ldg(ge + (3 + jj) * PW), t1, __ldg(ge + jj * PW) * t0))
                       : 0.0;
      }
      const long long l = (long long)(ps * Q2 + k) * c.W;
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) A.out[jj * cs + base + l] = o[jj];
    }
  });
  }
};

// ---------------------------------------------------------------------------
// IProductWRTDerivBase: 3 phys components -> 1 coefficient component
template <int S, int P, class L, int NT_, int PW, int GEO, int MINB_>
struct k_ipderiv {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  __device__ static void prefetch_geo(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    (void)n;
    (void)e0;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 1, Dims<S, P>::NQ);
  }
  __device__ static void prefetch_in(const OpArgs<S, P>& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NQ>(A.in, A.in_cstride, 3, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const OpArgs<S, P>& A, long long tile, double* sm) {
  using Dm = Dims<S, P>;
  constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2, NQ = Dm::NQ, NM = Dm::NM;
  constexpr int PL = L::PLANE, UO = 0, V0O = PL, V1O = 2 * PL, TAo = 0, TBo = 2 * PL;
  const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
  double* xs = sm + L::EB * PL;
  items<L, Q0 * Q1, NT>([&](int e, int ps) {
    const long long eg = c.e0 + e;
    const bool live = eg < c.E;
    const int row = ps * S2;
    const long long base = lane_base(live ? eg : 0, NQ, c.W);
    const long long cs = A.in_cstride;
    double w2[Q2], r[Q2];
#pragma unroll
    for (int k = 0; k < Q2; ++k) {
      const int l = ps * Q2 + k;
      const double wq = w_at<S, P, PW, GEO>(A, eg, live, l);
      const long long a = base + (long long)l * c.W;
      sm[L::at(e, V0O + row + k)] = live ? __ldg(A.in + a) * wq : 0.0;
      sm[L::at(e, V1O + row + k)] = live ? __ldg(A.in + cs + a) * wq : 0.0;
      w2[k] = live ? __ldg(A.in + 2 * cs + a) * wq : 0.0;
      r[k] = 0.0;
    }
    line_ddt_acc<S, P, 2>(A.D, w2, r);
#pragma unroll
    for (int k = 0; k < Q2; ++k) sm[L::at(e, UO + row + k)] = r[k];
  });
  __syncthreads();
  items<L, Q0 * Q2, NT>([&](int e, int ps) {
    const int i = ps / Q2, k = ps - i * Q2;
    double w[Q1], r[Q1];
#pragma unroll
    for (int j = 0; j < Q1; ++j) {
      w[j] = sm[L::at(e, V1O + (i * Q1 + j) * S2 + k)];
      r[j] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    }
    line_ddt_acc<S, P, 1>(A.D, w, r);
#pragma unroll
    for (int j = 0; j < Q1; ++j) sm[L::at(e, UO + (i * Q1 + j) * S2 + k)] = r[j];
  });
  __syncthreads();
  items<L, Q1 * Q2, NT>([&](int e, int ps) {
    const int j = ps / Q2, k = ps - j * Q2;
    double w[Q0], r[Q0], t[P1];
#pragma unroll
    for (int i = 0; i < Q0; ++i) {
      w[i] = sm[L::at(e, V0O + (i * Q1 + j) * S2 + k)];
      r[i] = sm[L::at(e, UO + (i * Q1 + j) * S2 + k)];
    }
    line_ddt_acc<S, P, 0>(A.D, w, r);
    line_a0t_eo<S, P>(A.B, r, t);
#pragma unroll
    for (int p = 0; p < P1; ++p) sm[L::at(e, TBo + (p * Q1 + j) * S2 + k)] = t[p];
  });
  __syncthreads();
  stage_b2<S, P, L, NT, TAo, TBo>(A.B, A.gtab, sm);
  __syncthreads();
  stage_b3<S, P, L, NT, TAo, CoefOut<L, NM>, false, ragged_dispatch(2, S, P), ragged_split(2, S, P), prism_warp_pairs(2, S, P)>(A.B, A.gtab, CoefOut<L, NM>{xs}, sm);
  __syncthreads();
  store_tile<L, NM, NT>(A.out, c, xs);
  }
};


// ---------------------------------------------------------------------------
// Helmholtz, non-collocated (Alg. 5, operators.py:636-667):
//   u = B uhat, v_m = (D_m B) uhat by sum factorisation with the derivative
//   1D tables (dmode), pointwise metric, then
//   out = sum_m (D_m B)^T w_m + lam B^T W u.
// Smem planes: 0 TA (F1 values, later R1), 1 TA' (F1 dir-2 derivative,
// later R2), 2 TB (F2 on TA, later S_A), 3 TB' (F2 dir-1 derivative on TA,
// later S_B), 4 TB'' (F2 on TA', later S_C); plane 2 doubles as the
// coefficient staging.  The middle sweep evaluates u, v0, v1, v2, the
// metric and the three transposed dir-0 contractions in registers, so
// quadrature-point arrays never touch shared memory.  Deformed geometry uses
// the standard-point-order payload (kind 3).
template <int S, int P, class L, int NT_, int PW, int GEO, bool LAMW, int MINB_>
struct k_helm_nc {
  static constexpr int NT = NT_;
  static constexpr int EB = L::EB;
  static constexpr int MINB = MINB_;
  static constexpr bool PERSIST = false;
  static constexpr bool GEO_PF_AT_START = true;
  using A_t = NcArgs<S, P>;
  __device__ static void prefetch_geo(const A_t& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.E - e0 < EB ? A.E - e0 : EB;
    if constexpr (GEO == GEO_DEFORMED) prefetch_payload<PW>(A.pay, e0, n, A.E, 7, Dims<S, P>::NQ, LAMW ? 7 : 6);
  }
  __device__ static void prefetch_in(const A_t& A, long long t) {
    const long long e0 = t * EB;
    const long long n = A.Epad - e0 < EB ? A.Epad - e0 : EB;
    prefetch_field<Dims<S, P>::NM>(A.in, A.in_cstride, gridDim.y, e0, n, A.Epad, A.W);
  }
  __device__ static void run(const A_t& A, long long tile, double* sm) {
    using Dm = Dims<S, P>;
    constexpr int P1 = Dm::P1, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2, S2 = L::S2;
    constexpr int NQ = Dm::NQ, NM = Dm::NM, PL = L::PLANE;
    constexpr int TA = 0, TA2 = PL, TB = 2 * PL, TB1 = 3 * PL, TB2 = 4 * PL;
    const Ctx c = make_ctx<L::EB>(tile, A.E, A.Epad, A.W);
    const double* src = A.in + blockIdx.y * A.in_cstride;
    double* dst = A.out + blockIdx.y * A.out_cstride;
    double* xs = sm + L::EB * 2 * PL;  // plane 2: coefficient staging

    load_tile<L, NM, NT>(src, c, xs);
    __syncthreads();
    stage_f1<S, P, L, NT, TA>(A.B, A.gtab, CoefIn<L, NM>{xs}, sm);
    stage_f1<S, P, L, NT, TA2, CoefIn<L, NM>, true>(A.DB, A.gtab, CoefIn<L, NM>{xs}, sm);
    __syncthreads();
    stage_f2<S, P, L, NT, TA, TB>(A.B, A.gtab, sm);
    stage_f2<S, P, L, NT, TA, TB1, true>(A.DB, A.gtab, sm);
    stage_f2<S, P, L, NT, TA2, TB2>(A.B, A.gtab, sm);
    __syncthreads();
    items<L, Q1 * Q2, NT>([&](int e, int ps) {
      const int j = ps / Q2, k = ps - j * Q2;
      const long long eg = c.e0 + e;
      const bool live = eg < c.E;
      double xv[P1], x1[P1], x2[P1];
#pragma unroll
      for (int p = 0; p < P1; ++p) {
        xv[p] = sm[L::at(e, TB + (p * Q1 + j) * S2 + k)];
        x1[p] = sm[L::at(e, TB1 + (p * Q1 + j) * S2 + k)];
        x2[p] = sm[L::at(e, TB2 + (p * Q1 + j) * S2 + k)];
      }
      double u[Q0], v0[Q0], v1[Q0], v2[Q0];
      line_a0<S, P>(A.B, xv, u);
      line_a0<S, P>(A.DB, xv, v0);
      line_a0<S, P>(A.B, x1, v1);
      line_a0<S, P>(A.B, x2, v2);
#pragma unroll
      for (int i = 0; i < Q0; ++i) {
        const int l = (i * Q1 + j) * Q2 + k;
        double w0, w1, w2, z;
        if constexpr (GEO == GEO_DEFORMED) {
          const double* g = A.pay + pay_base<PW>(live ? eg : 0, 7, NQ) + (long long)l * PW;
          const double l00 = live ? __ldcs(g + 0LL * NQ * PW) : 0.0, l01 = live ? __ldcs(g + 1LL * NQ * PW) : 0.0,
                       l02 = live ? __ldcs(g + 2LL * NQ * PW) : 0.0, l11 = live ? __ldcs(g + 3LL * NQ * PW) : 0.0,
                       l12 = live ? __ldcs(g + 4LL * NQ * PW) : 0.0, l22 = live ? __ldcs(g + 5LL * NQ * PW) : 0.0;
          w0 = fma(l02, v2[i], fma(l01, v1[i], l00 * v0[i]));
          w1 = fma(l12, v2[i], fma(l11, v1[i], l01 * v0[i]));
          w2 = fma(l22, v2[i], fma(l12, v1[i], l02 * v0[i]));
          z = 0.0;
          if constexpr (LAMW) z = live ? (A.lam * __ldcs(g + 6LL * NQ * PW)) * u[i] : 0.0;
        } else {
          const double* ge = A.pay + pay_base<PW>(live ? eg : 0, 8, 1);
          const double* rp = A.gtab + GLayout<S, P>::REGK + k * (Q0 * Q1) + i * Q1 + j;
          const double rw = __ldg(rp);
          const double L00 = __ldg(ge + 0 * PW), L01 = __ldg(ge + 1 * PW), L02 = __ldg(ge + 2 * PW),
                       L11 = __ldg(ge + 3 * PW), L12 = __ldg(ge + 4 * PW), L22 = __ldg(ge + 5 * PW);
          double t0 = v0[i], t1 = v1[i], t2 = v2[i];
          double g00 = 1.0, g10 = 0.0, g11 = 1.0, g20 = 0.0, g21 = 0.0;
          if constexpr (S != HEX) {
            g00 = __ldg(rp + 1 * NQ);
            g10 = __ldg(rp + 2 * NQ);
            g11 = __ldg(rp + 3 * NQ);
            g20 = __ldg(rp + 4 * NQ);
            g21 = __ldg(rp + 5 * NQ);
            t0 = g00 * v0[i];
            t1 = fma(g11, v1[i], g10 * v0[i]);
            t2 = fma(g21, v1[i], fma(g20, v0[i], v2[i]));
          }
          const double s0 = rw * fma(L02, t2, fma(L01, t1, L00 * t0));
          const double s1 = rw * fma(L12, t2, fma(L11, t1, L01 * t0));
          const double s2 = rw * fma(L22, t2, fma(L12, t1, L02 * t0));
          w0 = s0;
          w1 = s1;
          w2 = s2;
          if constexpr (S != HEX) {
            w0 = fma(g20, s2, fma(g10, s1, g00 * s0));
            w1 = fma(g21, s2, g11 * s1);
          }
          w0 = live ? w0 : 0.0;
          w1 = live ? w1 : 0.0;
          w2 = live ? w2 : 0.0;
          z = 0.0;
          if constexpr (LAMW) z = live ? A.lam * ((u[i] * rw) * __ldg(ge + 6 * PW)) : 0.0;
        }
        u[i] = z;  // lam W u
        v0[i] = w0;
        v1[i] = w1;
        v2[i] = w2;
      }
      double sa[P1], sb[P1], sc[P1], t[P1];
      line_a0t<S, P>(A.B, u, sa);
      line_a0t<S, P>(A.DB, v0, t);
#pragma unroll
      for (int p = 0; p < P1; ++p) sa[p] += t[p];
      line_a0t<S, P>(A.B, v1, sb);
      line_a0t<S, P>(A.B, v2, sc);
#pragma unroll
      for (int p = 0; p < P1; ++p) {
        sm[L::at(e, TB + (p * Q1 + j) * S2 + k)] = sa[p];
        sm[L::at(e, TB1 + (p * Q1 + j) * S2 + k)] = sb[p];
        sm[L::at(e, TB2 + (p * Q1 + j) * S2 + k)] = sc[p];
      }
    });
    __syncthreads();
    // R1 = B1^T S_A + (D B1)^T S_B (both continue with dir-2 values),
    // R2 = B1^T S_C (continues with the dir-2 derivative)
    stage_b2<S, P, L, NT, TA, TB>(A.B, A.gtab, sm);
    stage_b2<S, P, L, NT, TA2, TB2>(A.B, A.gtab, sm);
    __syncthreads();
    stage_b2<S, P, L, NT, TA, TB1, true, true>(A.DB, A.gtab, sm);
    __syncthreads();
    double* ys = sm + L::EB * 2 * PL;  // plane 2: output staging (S_A dead)
    stage_b3<S, P, L, NT, TA>(A.B, A.gtab, CoefOut<L, NM>{ys}, sm);
    __syncthreads();
    stage_b3<S, P, L, NT, TA2, CoefOut<L, NM, true>, true>(A.DB, A.gtab, CoefOut<L, NM, true>{ys}, sm);
    __syncthreads();
    store_tile<L, NM, NT>(dst, c, ys);
  }
};

}  // namespace sk

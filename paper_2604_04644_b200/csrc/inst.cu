// One translation unit per (shape, order): compiled with -DSK_S=<0..3>
// -DSK_P=<1..10>.  Instantiates every operator kernel for that pair, the
// table fills, the geometry payload packers and the device geometry builder,
// and exports them through sk::opset_impl<S,P>().
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sk_dense.cuh"
#include "sk_ops.cuh"
#include "sk_opset.hpp"
#include "sk_tune.h"

#ifndef SK_S
#error "compile with -DSK_S=<shape> -DSK_P=<order>"
#endif

namespace sk {

// ---------------------------------------------------------------------------
// launch configuration.  EB = elements per CTA tile (a power of two, the smem
// and payload lane width); chosen per (shape, order) from the B200 sweeps in
// profiles/ (sk_tune.h), or forced with -DSK_EB_FIXED=<n> for tuning builds.
template <int S, int P>
struct Mode {
  using Dm = Dims<S, P>;
  static constexpr int smem_bytes(int eb) {
    return 3 * Dm::Q0 * Dm::Q1 * row_stride(S, P, eb) * eb * 8;
  }
  static constexpr int fit(int eb, int budget) {
    return (eb <= 1 || smem_bytes(eb) <= budget) ? eb : fit(eb / 2, budget);
  }
  // the non-collocated Helmholtz keeps five planes
  static constexpr int fit5(int eb, int budget) {
    return (eb <= 1 || smem_bytes(eb) / 3 * 5 <= budget) ? eb : fit5(eb / 2, budget);
  }
  // Helmholtz family (Helmholtz / stiffness / non-collocated / phys_deriv;
  // payload kinds 0, 2, 3) and W family (mass / iproduct / iproduct-deriv /
  // bwd_trans; payload kind 1): independent tile widths
  static constexpr int EBH = tuned_eb(0, S, P) > 0 ? fit(tuned_eb(0, S, P), 200 * 1024) : fit(16, 100 * 1024);
  static constexpr int EBW = tuned_eb(1, S, P) > 0 ? fit(tuned_eb(1, S, P), 200 * 1024) : fit(16, 100 * 1024);
  // payload lane width of each payload kind = tile width of its consumers
  // non-collocated Helmholtz (payload kind 3): its own tile / lane width
  static constexpr int EBN = tuned_eb_nc(S, P) > 0 ? fit5(tuned_eb_nc(S, P), 200 * 1024) : EBH;
  // phys_deriv (payload kind 2): its own tile / lane width
  static constexpr int EBD = tuned_eb_pderiv(S, P) > 0 ? fit(tuned_eb_pderiv(S, P), 200 * 1024) : EBH;
  SK_HD static constexpr int pw(int kind) { return kind == 1 ? EBW : kind == 3 ? EBN : kind == 2 ? EBD : EBH; }
  // regular-geometry collocated Helmholtz tile width (its payload lane
  // width is kRegPW, independent of the tile)
  static constexpr int EBHR = tuned_eb_regular(S, P) > 0 ? fit(tuned_eb_regular(S, P), 200 * 1024) : EBH;
  // bwd_trans reads no payload: its own tile width (kTunedEBBwd, 0 = EBW)
  static constexpr int EBB = tuned_eb_bwd(S, P) > 0 ? fit(tuned_eb_bwd(S, P), 200 * 1024) : EBW;
  SK_HD static constexpr int eb(int op) {
    return (op == OP_HELM || op == OP_QP) ? EBH : op == OP_PDERIV ? EBD : op == OP_HELM_NC ? EBN : op == OP_BWD ? EBB : EBW;
  }
};

template <int S, int P, int OP, bool REG = false>
struct Cfg {
  using Dm = Dims<S, P>;
  static constexpr int EB = REG ? Mode<S, P>::EBHR : Mode<S, P>::eb(OP);
  static constexpr int PW = EB;
  static constexpr int planes = OP == OP_HELM_NC ? 5 : (OP == OP_HELM || OP == OP_PDERIV || OP == OP_IPDERIV || OP == OP_QP) ? 3 : 2;
  static constexpr int items = cmax(cmax(cmax(Dm::Q1 * Dm::Q2, Dm::Q0 * Dm::Q2), cmax(Dm::Q0 * Dm::Q1, Dm::P1 * Dm::P1)),
                                    cmax(Dm::NPAIR, Dm::P1 * Dm::Q2));
  using L = Lay<S, P, planes, EB>;
  static constexpr int CLS = (OP == OP_HELM || OP == OP_QP) ? 0 : OP == OP_MASS ? 1 : 2;
  static constexpr int NT0 = ((EB * items / (REG ? tuned_nt_div_regular(S, P) : nt_div_op(OP, CLS, S, P)) + 31) / 32) * 32;
  static constexpr int NT = NT0 > 512 ? 512 : (NT0 < 64 ? 64 : NT0);
  // deformed Helmholtz: TMA geometry ring after the planes (sk_tune.h kGeoRing)
  static constexpr int RING = (OP == OP_HELM && !REG && geo_ring(S, P) > 0 && EB * Dm::Q0 * Dm::Q1 <= NT &&
                               (Dm::Q0 * Dm::Q1 * EB) % 2 == 0 && !tuned_persist(0, S, P))
                                  ? geo_ring(S, P)
                                  : 0;
  static constexpr int SMEM0 = (smem_tables(CLS, S, P) ? L::TABOFF + GLayout<S, P>::RAGGED : L::SMEM_DOUBLES) * 8;
  static constexpr int SMEM = RING ? (SMEM0 + 15) / 16 * 16 + RING * (7 * Dm::Q0 * Dm::Q1 * EB * 8 + 16) : SMEM0;
  // __launch_bounds__ min blocks: 1, or the CTAs per SM that shared memory
  // allows (forces ptxas to fit the registers; tuned, as it can spill)
  static constexpr int MINB = minb_op(OP, CLS, S, P) ? cmax(1, cmin(cmin(tuned_minb_cap(CLS, S, P), (220 * 1024) / (SMEM + 1024)), 2048 / NT))
                                               : 1;
};

// ---------------------------------------------------------------------------
// host table fills
// even-odd combination of the vertex columns of a full family (Q x P1)
template <int Q, int P1>
void fill_pm(const std::vector<double>& a, double* ap, double* am) {
  for (int i = 0; i < Q; ++i) {
    ap[i] = 0.5 * (a[i * P1] + a[i * P1 + 1]);
    am[i] = 0.5 * (a[i * P1] - a[i * P1 + 1]);
  }
}

// even-odd form of M (transposed when tr) -- see EOTab
template <int Q>
void fill_eo(const std::vector<double>& D, bool tr, EOTab<Q>& t) {
  constexpr int H = Q / 2;
  auto M = [&](int a, int b) { return tr ? D[b * Q + a] : D[a * Q + b]; };
  std::memset(&t, 0, sizeof(t));
  for (int a = 0; a < H; ++a) {
    for (int b = 0; b < H; ++b) {
      t.E[a * H + b] = 0.5 * (M(a, b) + M(a, Q - 1 - b));
      t.O[a * H + b] = 0.5 * (M(a, b) - M(a, Q - 1 - b));
    }
    if (Q % 2) {
      t.Em[a] = M(a, H);
      t.Om[a] = M(H, a);
    }
  }
}

template <int S, int P>
void fill_fwd(const HostBasis& hb, FwdTab<S, P>& t, bool deriv) {
  using Dm = Dims<S, P>;
  std::memset(&t, 0, sizeof(t));
  const std::vector<double>* a = deriv ? hb.da : hb.a;
  std::memcpy(t.a0, a[0].data(), sizeof(double) * Dm::Q0 * Dm::P1);
  if constexpr (S != TET) std::memcpy(t.a1, a[1].data(), sizeof(double) * Dm::Q1 * Dm::P1);
  if constexpr (S == HEX) std::memcpy(t.a2, a[2].data(), sizeof(double) * Dm::Q2 * Dm::P1);
  fill_pm<Dm::Q0, Dm::P1>(a[0], t.a0p, t.a0m);
  if constexpr (S != TET) fill_pm<Dm::Q1, Dm::P1>(a[1], t.a1p, t.a1m);
  if constexpr (S == HEX) fill_pm<Dm::Q2, Dm::P1>(a[2], t.a2p, t.a2m);
  if constexpr (S == TET) {
    const auto& fam = deriv ? hb.db1 : hb.b1;
    for (int p = 0; p < Dm::P1; ++p)
      std::memcpy(t.b1 + wfam_off(Dm::Q1, Dm::P1, p), fam[p].data(), sizeof(double) * fam[p].size());
  }
  if constexpr (S != HEX) {
    const auto& fam = deriv ? hb.dc2 : hb.c2;
    for (int p = 0; p < Dm::P1; ++p)
      std::memcpy(t.c2 + wfam_off(Dm::Q2, Dm::P1, p), fam[p].data(), sizeof(double) * fam[p].size());
  }
}

// Duffy scale of the 1D weights per shape x direction (basis_host.cpp
// build_basis: refw = (w0 s0)(w1 s1)(w2 s2), shapes.py ref_weights)
constexpr double kWScale[4][3] = {{1.0, 1.0, 1.0}, {1.0, 1.0, 0.5}, {1.0, 1.0, 0.25}, {1.0, 0.5, 0.25}};

template <int S, int P>
void fill(const HostBasis& hb, void* fv, void* fd, void* dt) {
  using Dm = Dims<S, P>;
  fill_fwd<S, P>(hb, *static_cast<FwdTab<S, P>*>(fv), false);
  fill_fwd<S, P>(hb, *static_cast<FwdTab<S, P>*>(fd), true);
  auto& d = *static_cast<DTab<S, P>*>(dt);
  std::memset(&d, 0, sizeof(d));
  std::memcpy(d.d0, hb.D[0].data(), sizeof(double) * Dm::Q0 * Dm::Q0);
  std::memcpy(d.d1, hb.D[1].data(), sizeof(double) * Dm::Q1 * Dm::Q1);
  std::memcpy(d.d2, hb.D[2].data(), sizeof(double) * Dm::Q2 * Dm::Q2);
  fill_eo<Dm::Q0>(hb.D[0], false, d.e0);
  fill_eo<Dm::Q0>(hb.D[0], true, d.e0t);
  if constexpr (gll_dir(S, 1)) {
    fill_eo<Dm::Q1>(hb.D[1], false, d.e1);
    fill_eo<Dm::Q1>(hb.D[1], true, d.e1t);
  }
  if constexpr (gll_dir(S, 2)) {
    fill_eo<Dm::Q2>(hb.D[2], false, d.e2);
    fill_eo<Dm::Q2>(hb.D[2], true, d.e2t);
  }
  for (int k = 0; k < Dm::Q2; ++k) {
    d.ak[k] = S == HEX ? 0.0 : 1.0 / (1.0 - hb.z[2][k]);
    d.w2k[k] = hb.w[2][k] * kWScale[S][2];
  }
}

// extra runtime-indexed tables (after GLayout<S,P>::SIZE)
template <int S, int P>
struct GExt {
  using Dm = Dims<S, P>;
  using L = GLayout<S, P>;
  static constexpr int DM0 = L::SIZE;
  static constexpr int DM1 = DM0 + Dm::Q0 * Dm::Q0;
  static constexpr int DM2 = DM1 + Dm::Q1 * Dm::Q1;
  static constexpr int Z0 = DM2 + Dm::Q2 * Dm::Q2;
  static constexpr int Z1 = Z0 + Dm::Q0;
  static constexpr int Z2 = Z1 + Dm::Q1;
  static constexpr int GST = Z2 + Dm::Q2;  // [l][3][3] dense G, standard point order
  static constexpr int SIZE = GST + 9 * Dm::NQ;
};

template <int S, int P>
void fill_gtab(const HostBasis& hb, double* g) {
  using Dm = Dims<S, P>;
  using L = GLayout<S, P>;
  using X = GExt<S, P>;
  std::memset(g, 0, sizeof(double) * X::SIZE);
  if constexpr (S == TET) {
    for (int p = 0; p < Dm::P1; ++p) {
      std::memcpy(g + L::B1 + wfam_off(Dm::Q1, Dm::P1, p), hb.b1[p].data(), sizeof(double) * hb.b1[p].size());
      std::memcpy(g + L::DB1 + wfam_off(Dm::Q1, Dm::P1, p), hb.db1[p].data(), sizeof(double) * hb.db1[p].size());
    }
  }
  if constexpr (S != HEX) {
    for (int m = 0; m < Dm::P1; ++m) {
      std::memcpy(g + L::C2 + wfam_off(Dm::Q2, Dm::P1, m), hb.c2[m].data(), sizeof(double) * hb.c2[m].size());
      std::memcpy(g + L::DC2 + wfam_off(Dm::Q2, Dm::P1, m), hb.dc2[m].data(), sizeof(double) * hb.dc2[m].size());
    }
  }
  // (p, q) pairs of the ragged stages with their mode offset and run length,
  // ordered by run length (= dir-2 slice P1 - m) so that the work items of a
  // warp mostly share one slice (one branch of the slice dispatch)
  int* pr = reinterpret_cast<int*>(g + L::PAIRS);
  std::vector<std::array<int, 4>> pl;
  int off = 0;
  for (int p = 0; p < Dm::P1; ++p) {
    const int nq = (S == TET) ? Dm::P1 - p : Dm::P1;
    for (int q = 0; q < nq; ++q) {
      int nr = Dm::P1;
      if (S == PRISM) nr = Dm::P1 - p;
      if (S == PYR) nr = Dm::P1 - cmax(p, q);
      if (S == TET) nr = Dm::P1 - p - q;
      if ((int)pl.size() < Dm::NPAIR && S != HEX) pl.push_back({p, q, off, nr});
      off += nr;
    }
  }
  std::stable_sort(pl.begin(), pl.end(), [](const std::array<int, 4>& a, const std::array<int, 4>& b) { return a[3] > b[3]; });
  for (size_t i = 0; i < pl.size(); ++i)
    for (int c = 0; c < 4; ++c) pr[4 * i + c] = pl[i][c];
  for (int i = 0; i < Dm::Q0; ++i)
    for (int j = 0; j < Dm::Q1; ++j)
      for (int k = 0; k < Dm::Q2; ++k) {
        const int l = (i * Dm::Q1 + j) * Dm::Q2 + k;
        const int km = k * Dm::Q0 * Dm::Q1 + i * Dm::Q1 + j;
        const double* G = &hb.G[9 * l];
        g[L::REGK + 0 * Dm::NQ + km] = hb.refw[l];
        g[L::REGK + 1 * Dm::NQ + km] = G[0];  // G00
        g[L::REGK + 2 * Dm::NQ + km] = G[3];  // G10
        g[L::REGK + 3 * Dm::NQ + km] = G[4];  // G11
        g[L::REGK + 4 * Dm::NQ + km] = G[6];  // G20
        g[L::REGK + 5 * Dm::NQ + km] = G[7];  // G21
        g[L::REFW + l] = hb.refw[l];
        for (int a = 0; a < 9; ++a) g[X::GST + 9 * l + a] = G[a];
      }
  for (int i = 0; i < Dm::Q0; ++i)
    for (int j = 0; j < Dm::Q1; ++j) {
      const int ps = i * Dm::Q1 + j, n2 = Dm::Q0 * Dm::Q1;
      const double e1 = hb.z[0][i], e2 = hb.z[1][j];
      double c00 = 0.0, c20 = 0.0, c21 = 0.0;
      if (S == PRISM) c00 = 2.0, c20 = 1.0 + e1;
      if (S == PYR) c00 = 2.0, c20 = 1.0 + e1, c21 = 1.0 + e2;
      if (S == TET) {
        const double b = 1.0 / (1.0 - e2);
        c00 = 4.0 * b, c20 = 2.0 * (1.0 + e1) * b, c21 = 1.0 + e2;
      }
      g[L::REGIJ + 0 * n2 + ps] = (hb.w[0][i] * kWScale[S][0]) * (hb.w[1][j] * kWScale[S][1]);
      g[L::REGIJ + 1 * n2 + ps] = c00;
      g[L::REGIJ + 2 * n2 + ps] = c20;
      g[L::REGIJ + 3 * n2 + ps] = c21;
    }
  std::memcpy(g + X::DM0, hb.D[0].data(), sizeof(double) * Dm::Q0 * Dm::Q0);
  std::memcpy(g + X::DM1, hb.D[1].data(), sizeof(double) * Dm::Q1 * Dm::Q1);
  std::memcpy(g + X::DM2, hb.D[2].data(), sizeof(double) * Dm::Q2 * Dm::Q2);
  std::memcpy(g + X::Z0, hb.z[0].data(), sizeof(double) * Dm::Q0);
  std::memcpy(g + X::Z1, hb.z[1].data(), sizeof(double) * Dm::Q1);
  std::memcpy(g + X::Z2, hb.z[2].data(), sizeof(double) * Dm::Q2);
}

// ---------------------------------------------------------------------------
// launches
template <class K>
static void ensure_smem(K kernel, int bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int S, int P, int OP, class Op, class C = Cfg<S, P, OP>, class Args>
static int go(const Args& a, const LaunchReq& r, int gy, void* stream) {
  static_assert(C::EB == C::PW, "tiles must align with payload lanes");
  constexpr bool persist = Op::PERSIST && tuned_persist(C::CLS, S, P);
  auto kern = [] {
    if constexpr (persist)
      return k_persist<Op, Args>;
    else
      return k_tile<Op, Args>;
  }();
  static std::once_flag once;  // one per kernel instantiation
  static int per_sm = 1, sms = 148;
  std::call_once(once, [&] {
    ensure_smem(kern, C::SMEM);
    int dev = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Op::NT, C::SMEM);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
  });
  const long long tiles = (r.Epad + C::EB - 1) / C::EB;
  if (tiles == 0) return 0;
  Args& args = const_cast<Args&>(a);
  const int g = gy > 0 ? gy : 1;
  const long long resident = (long long)per_sm * sms;
  args.pf_ahead = resident / g;
  long long grid = tiles;
  if constexpr (persist) {
    // one resident wave, shared by the components (grid.y)
    const long long wave = resident / g > 0 ? resident / g : 1;
    grid = tiles < wave ? tiles : wave;
  }
  kern<<<dim3((unsigned)grid, (unsigned)gy), Op::NT, C::SMEM, static_cast<cudaStream_t>(stream)>>>(args);
  return (int)cudaGetLastError();
}

// TMA-fed deformed mass (k_mass_tma): one resident wave of persistent CTAs
inline bool mass_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_MASS_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int S, int P>
int launch_mass_tma(const OpArgs<S, P>& a, const LaunchReq& r, void* stream) {
  using C = Cfg<S, P, OP_MASS>;
  constexpr int SM0 = MassTma<S, P, typename C::L, C::NT, C::PW, 1>::SMEM;
  constexpr int MINB = tuned_minb(1, S, P) ? cmax(1, cmin(cmin(tuned_minb_cap(1, S, P), (220 * 1024) / (SM0 + 1024)), 2048 / C::NT)) : 1;
  using M = MassTma<S, P, typename C::L, C::NT, C::PW, MINB>;
  auto kern = k_mass_tma<S, P, typename C::L, C::NT, C::PW, MINB>;
  static std::once_flag once;
  static int per_sm = 1, sms = 148;
  std::call_once(once, [&] {
    ensure_smem(kern, M::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, M::SMEM);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  const long long tiles = (r.Epad + C::EB - 1) / C::EB;
  if (tiles == 0) return 0;
  const int gy = r.ncomp > 0 ? r.ncomp : 1;
  const long long wave = (long long)per_sm * sms / gy;
  const long long grid = tiles < wave ? tiles : (wave > 0 ? wave : 1);
  kern<<<dim3((unsigned)grid, (unsigned)gy), C::NT, M::SMEM, static_cast<cudaStream_t>(stream)>>>(a);
  return (int)cudaGetLastError();
}

// warp-tile mass (k_mass_warp): one resident wave of CTAs, every warp
// striding over G-element tiles
inline bool mass_warp_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_MASS_WARP");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int S, int P, int G, int PW, int GEO>
int launch_mass_warp(const OpArgs<S, P>& a, const LaunchReq& r, void* stream) {
  using M = MassWarp<S, P, G, kMassWarpWPC, PW, GEO>;
  auto kern = k_mass_warp<S, P, G, kMassWarpWPC, PW, GEO>;
  static std::once_flag once;
  static int per_sm = 1, sms = 148;
  std::call_once(once, [&] {
    ensure_smem(kern, M::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, M::NT, M::SMEM);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  });
  const long long tiles = (r.Epad + G - 1) / G;
  if (tiles == 0) return 0;
  const int gy = r.ncomp > 0 ? r.ncomp : 1;
  const long long resident = (long long)per_sm * sms / gy;
  const long long need = (tiles + M::WPC - 1) / M::WPC;
  const long long grid = need < resident ? need : (resident > 0 ? resident : 1);
  kern<<<dim3((unsigned)grid, (unsigned)gy), M::NT, M::SMEM, static_cast<cudaStream_t>(stream)>>>(a);
  return (int)cudaGetLastError();
}

// persistent TMA-staged driver (k_persist_tma): one resident wave
inline bool helm_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_HELM_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int S, int P, int OP, class Op, class C = Cfg<S, P, OP>, class Args>
static int go_tma(const Args& a, const LaunchReq& r, int gy, void* stream) {
  using T = PersistTma<Op, Args, Dims<S, P>::NM, C::SMEM>;
  auto kern = k_persist_tma<Op, Args, Dims<S, P>::NM, C::SMEM>;
  static std::once_flag once;
  static int per_sm = 1, sms = 148;
  std::call_once(once, [&] {
    ensure_smem(kern, T::SMEM);
    int dev = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Op::NT, T::SMEM);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
  });
  const long long tiles = (r.Epad + C::EB - 1) / C::EB;
  if (tiles == 0) return 0;
  const int g = gy > 0 ? gy : 1;
  const long long wave = (long long)per_sm * sms / g;
  const long long grid = tiles < wave ? tiles : (wave > 0 ? wave : 1);
  kern<<<dim3((unsigned)grid, (unsigned)g), Op::NT, T::SMEM, static_cast<cudaStream_t>(stream)>>>(a);
  return (int)cudaGetLastError();
}

// StdMat mass on DMMA (sk_dense.cuh): persistent warps over 8-element groups
template <int S, int P, int PW, int GEO>
int launch_dense_geo(const DenseArgs& a, int ncomp, void* stream) {
  using X = DenseDims<S, P>;
  constexpr int BIT = GEO == GEO_DEFORMED ? 2 : 1;
  if constexpr (!(X::MASK & BIT)) {
    return (int)cudaErrorInvalidValue;  // fragments would not fit in shared memory: never selected
  } else {
    constexpr int smem = (GEO == GEO_DEFORMED ? X::F1 + X::F2 : X::FR) * 8;
    auto kern = k_mass_dense<S, P, PW, GEO>;
    static std::once_flag once;
    static int per_sm = 1, sms = 148;
    std::call_once(once, [&] {
      ensure_smem(kern, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDenseThreads, smem);
      if (per_sm < 1) per_sm = 1;
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    });
    const long long groups = (a.Epad + 7) / 8;
    if (groups == 0) return 0;
    const int gy = ncomp > 0 ? ncomp : 1;
    const long long resident = (long long)per_sm * sms / gy;
    const long long need = (groups + kDenseThreads / 32 - 1) / (kDenseThreads / 32);
    const long long grid = need < resident ? need : (resident > 0 ? resident : 1);
    kern<<<dim3((unsigned)grid, (unsigned)gy), kDenseThreads, smem, static_cast<cudaStream_t>(stream)>>>(a);
    return (int)cudaGetLastError();
  }
}

template <int S, int P, bool LAMW>
int launch_helm_dense_lam(const DenseArgs& a, double lam, int ncomp, void* stream) {
  using X = DenseDims<S, P>;
  if constexpr (!(X::MASK & 4)) {
    return (int)cudaErrorInvalidValue;
  } else {
    constexpr int smem = (LAMW ? 7 : 6) * X::FR * 8;
    auto kern = k_helm_dense<S, P, LAMW>;
    static std::once_flag once;
    static int per_sm = 1, sms = 148;
    std::call_once(once, [&] {
      ensure_smem(kern, smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDenseThreads, smem);
      if (per_sm < 1) per_sm = 1;
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    });
    const long long groups = (a.Epad + 7) / 8;
    if (groups == 0) return 0;
    const int gy = ncomp > 0 ? ncomp : 1;
    const long long resident = (long long)per_sm * sms / gy;
    const long long need = (groups + kDenseThreads / 32 - 1) / (kDenseThreads / 32);
    const long long grid = need < resident ? need : (resident > 0 ? resident : 1);
    kern<<<dim3((unsigned)grid, (unsigned)gy), kDenseThreads, smem, static_cast<cudaStream_t>(stream)>>>(a, lam);
    return (int)cudaGetLastError();
  }
}

template <int S, int P>
int launch_helm_dense(const LaunchReq& r, void* stream) {
  DenseArgs a;
  a.frag = r.dense;
  a.in = r.in;
  a.out = r.out;
  a.pay = r.pay;
  a.E = r.E;
  a.Epad = r.Epad;
  a.in_cstride = r.in_cs;
  a.out_cstride = r.out_cs;
  a.W = r.W;
  if (r.lam != 0.0) return launch_helm_dense_lam<S, P, true>(a, r.lam, r.ncomp, stream);
  return launch_helm_dense_lam<S, P, false>(a, r.lam, r.ncomp, stream);
}

template <int S, int P, int PW>
int launch_dense(const LaunchReq& r, void* stream) {
  DenseArgs a;
  a.frag = r.dense;
  a.in = r.in;
  a.out = r.out;
  a.pay = r.pay;
  a.E = r.E;
  a.Epad = r.Epad;
  a.in_cstride = r.in_cs;
  a.out_cstride = r.out_cs;
  a.W = r.W;
  if (r.geo == GEO_DEFORMED) return launch_dense_geo<S, P, PW, GEO_DEFORMED>(a, r.ncomp, stream);
  return launch_dense_geo<S, P, PW, GEO_REGULAR>(a, r.ncomp, stream);
}

template <int S, int P>
int launch_nc(const LaunchReq& r, void* stream) {
  NcArgs<S, P> a;
  std::memcpy(&a.B, r.fwd, sizeof(a.B));
  std::memcpy(&a.DB, r.fwd_d, sizeof(a.DB));
  a.in = r.in;
  a.out = r.out;
  a.pay = r.pay;
  a.gtab = r.gtab;
  a.E = r.E;
  a.Epad = r.Epad;
  a.in_cstride = r.in_cs;
  a.out_cstride = r.out_cs;
  a.W = r.W;
  a.pad_ = 0;
  a.lam = r.lam;
  using C = Cfg<S, P, OP_HELM_NC>;
  using L = typename C::L;
  if (r.geo == GEO_DEFORMED) {
    if (r.lam != 0.0) return go<S, P, OP_HELM_NC, k_helm_nc<S, P, L, C::NT, C::PW, GEO_DEFORMED, true, 1>>(a, r, r.ncomp, stream);
    return go<S, P, OP_HELM_NC, k_helm_nc<S, P, L, C::NT, C::PW, GEO_DEFORMED, false, 1>>(a, r, r.ncomp, stream);
  }
  if (r.lam != 0.0) return go<S, P, OP_HELM_NC, k_helm_nc<S, P, L, C::NT, C::PW, GEO_REGULAR, true, 1>>(a, r, r.ncomp, stream);
  return go<S, P, OP_HELM_NC, k_helm_nc<S, P, L, C::NT, C::PW, GEO_REGULAR, false, 1>>(a, r, r.ncomp, stream);
}

template <int S, int P>
int launch(int op, const LaunchReq& r, void* stream) {
  OpArgs<S, P> a;
  std::memcpy(&a.B, r.fwd, sizeof(a.B));
  std::memcpy(&a.D, r.dtab, sizeof(a.D));
  a.in = r.in;
  a.out = r.out;
  a.pay = r.pay;
  a.gtab = r.gtab;
  a.E = r.E;
  a.Epad = r.Epad;
  a.in_cstride = r.in_cs;
  a.out_cstride = r.out_cs;
  a.W = r.W;
  a.c0_nx = r.c0_nx;
  a.c0_ny = r.c0_ny;
  a.pad_ = 0;
  a.lam = r.lam;
  a.c0map = reinterpret_cast<const int*>(r.c0map);
  const bool def = r.geo == GEO_DEFORMED;
  using namespace std;
  switch (op) {
#if !defined(SK_ONLY_OP) || SK_ONLY_OP == 6
    case OP_HELM_NC:
      return launch_nc<S, P>(r, stream);
#endif
#if !defined(SK_ONLY_OP) || SK_ONLY_OP == 0
    case OP_HELM: {
      using C = Cfg<S, P, OP_HELM>;
      if (r.c0map) {  // assembled C0, mapped mesh: gather fused into the tile load (deformed)
        if constexpr (S != HEX) {
          if (def) {
            if (r.lam != 0.0)
              return go<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, true, C::MINB, 2>>(a, r, 1, stream);
            return go<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, false, C::MINB, 2>>(a, r, 1, stream);
          }
        }
        return (int)cudaErrorInvalidValue;
      }
      if (r.c0_nx > 0) {
        // assembled C0 hex: gather fused into the tile load (deformed, lam > 0)
        if constexpr (S == HEX) {
          if (def && r.lam != 0.0)
            return go<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, true, C::MINB, true>>(a, r, 1, stream);
        }
        return (int)cudaErrorInvalidValue;
      }
      if constexpr (helm_tma(S, P) && C::RING == 0) {
        if (def && helm_tma_enabled()) {
          if (r.lam != 0.0) return go_tma<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, true, C::MINB>>(a, r, r.ncomp, stream);
          return go_tma<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, false, C::MINB>>(a, r, r.ncomp, stream);
        }
      }
      if (def) {
        if (r.lam != 0.0) return go<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, true, C::MINB, false, C::RING>>(a, r, r.ncomp, stream);
        return go<S, P, OP_HELM, k_helm<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, false, C::MINB, false, C::RING>>(a, r, r.ncomp, stream);
      }
      if (r.dense) {  // regular geometry, StdMat on DMMA (sk_dense.cuh)
        if constexpr (P <= kDenseMaxP) return launch_helm_dense<S, P>(r, stream);
        return (int)cudaErrorInvalidValue;
      }
      using CR = Cfg<S, P, OP_HELM, true>;  // regular geometry: own tile width
      if constexpr (helm_tma_reg(S, P)) {
        if (helm_tma_enabled()) {
          if (r.lam != 0.0) return go_tma<S, P, OP_HELM, k_helm<S, P, typename CR::L, CR::NT, CR::PW, GEO_REGULAR, true, CR::MINB>, CR>(a, r, r.ncomp, stream);
          return go_tma<S, P, OP_HELM, k_helm<S, P, typename CR::L, CR::NT, CR::PW, GEO_REGULAR, false, CR::MINB>, CR>(a, r, r.ncomp, stream);
        }
      }
      if (r.lam != 0.0) return go<S, P, OP_HELM, k_helm<S, P, typename CR::L, CR::NT, CR::PW, GEO_REGULAR, true, CR::MINB>, CR>(a, r, r.ncomp, stream);
      return go<S, P, OP_HELM, k_helm<S, P, typename CR::L, CR::NT, CR::PW, GEO_REGULAR, false, CR::MINB>, CR>(a, r, r.ncomp, stream);
    }
#endif
#if !defined(SK_ONLY_OP) || SK_ONLY_OP == 1
    case OP_MASS: {
      using C = Cfg<S, P, OP_MASS>;
      if (r.dense) {
        if constexpr (P <= kDenseMaxP) return launch_dense<S, P, C::PW>(r, stream);
        return (int)cudaErrorInvalidValue;
      }
      if constexpr (mass_tma(S, P) && (C::EB * Dims<S, P>::NM) % 2 == 0 && (Dims<S, P>::NQ * C::PW) % 2 == 0) {
        if (def && mass_tma_enabled()) return launch_mass_tma<S, P>(a, r, stream);
      }
      if constexpr (mass_warp_g(S, P) > 0) {
        if (mass_warp_enabled()) {
          if (def) return launch_mass_warp<S, P, mass_warp_g(S, P), C::PW, GEO_DEFORMED>(a, r, stream);
          return launch_mass_warp<S, P, mass_warp_g(S, P), C::PW, GEO_REGULAR>(a, r, stream);
        }
      }
      if (def) return go<S, P, OP_MASS, k_mass<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, C::MINB>>(a, r, r.ncomp, stream);
      return go<S, P, OP_MASS, k_mass<S, P, typename C::L, C::NT, C::PW, GEO_REGULAR, C::MINB>>(a, r, r.ncomp, stream);
    }
#endif
    case OP_BWD: {  // always built: the dense kernels' basis matrix comes from it
      using C = Cfg<S, P, OP_BWD>;
      return go<S, P, OP_BWD, k_bwd<S, P, typename C::L, C::NT, C::MINB>>(a, r, r.ncomp, stream);
    }
#if !defined(SK_ONLY_OP)
    case OP_IPROD: {
      using C = Cfg<S, P, OP_IPROD>;
      if (def) return go<S, P, OP_IPROD, k_iprod<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, C::MINB>>(a, r, r.ncomp, stream);
      return go<S, P, OP_IPROD, k_iprod<S, P, typename C::L, C::NT, C::PW, GEO_REGULAR, C::MINB>>(a, r, r.ncomp, stream);
    }
    case OP_QP: {  // staged Helmholtz, quadrature-point kernel (deformed)
      using C = Cfg<S, P, OP_QP>;
      if (!def) return (int)cudaErrorInvalidValue;
      if (r.lam != 0.0) return go<S, P, OP_QP, k_qp<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, true, C::MINB>>(a, r, r.ncomp, stream);
      return go<S, P, OP_QP, k_qp<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, false, C::MINB>>(a, r, r.ncomp, stream);
    }
    case OP_BT: {  // staged Helmholtz, unweighted B^T
      using C = Cfg<S, P, OP_BT>;
      return go<S, P, OP_BT, k_iprod<S, P, typename C::L, C::NT, C::PW, GEO_UNIT, C::MINB>>(a, r, r.ncomp, stream);
    }
#endif
#if !defined(SK_ONLY_OP) || SK_ONLY_OP == 4
    case OP_PDERIV: {
      using C = Cfg<S, P, OP_PDERIV>;
      if (def) return go<S, P, OP_PDERIV, k_pderiv<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, C::MINB>>(a, r, 1, stream);
      return go<S, P, OP_PDERIV, k_pderiv<S, P, typename C::L, C::NT, C::PW, GEO_REGULAR, C::MINB>>(a, r, 1, stream);
    }
#endif
#if !defined(SK_ONLY_OP)
    case OP_IPDERIV: {
      using C = Cfg<S, P, OP_IPDERIV>;
      if (def) return go<S, P, OP_IPDERIV, k_ipderiv<S, P, typename C::L, C::NT, C::PW, GEO_DEFORMED, C::MINB>>(a, r, 1, stream);
      return go<S, P, OP_IPDERIV, k_ipderiv<S, P, typename C::L, C::NT, C::PW, GEO_REGULAR, C::MINB>>(a, r, 1, stream);
    }
#endif
  }
  return (int)cudaErrorInvalidValue;
}

template <int S, int P>
void config(int op, int geo, int64_t out[3]) {
  if (op == OP_HELM && geo == GEO_REGULAR) {  // the regular collocated Helmholtz has its own tile
    out[0] = Cfg<S, P, OP_HELM, true>::EB;
    out[1] = Cfg<S, P, OP_HELM, true>::NT;
    out[2] = Cfg<S, P, OP_HELM, true>::SMEM;
    return;
  }
  switch (op) {
#define SK_CFG(OPV)                    \
  case OPV:                            \
    out[0] = Cfg<S, P, OPV>::EB;       \
    out[1] = Cfg<S, P, OPV>::NT;       \
    out[2] = Cfg<S, P, OPV>::SMEM;     \
    return;
    SK_CFG(OP_HELM)
    SK_CFG(OP_MASS)
    SK_CFG(OP_BWD)
    SK_CFG(OP_IPROD)
    SK_CFG(OP_PDERIV)
    SK_CFG(OP_IPDERIV)
    SK_CFG(OP_HELM_NC)
    SK_CFG(OP_QP)
    SK_CFG(OP_BT)
#undef SK_CFG
  }
  out[0] = out[1] = out[2] = 0;
}

// ---------------------------------------------------------------------------
// geometry payloads
template <int S, int P>
long long payload_doubles(int kind, int geo) {
  constexpr long long NQ = Dims<S, P>::NQ;
  if (geo == GEO_DEFORMED) return (kind == 0 || kind == 3) ? 7 * NQ : kind == 1 ? NQ : 9 * NQ;
  return (kind == 0 || kind == 3) ? 8 : kind == 1 ? 1 : 9;
}

template <int S, int P>
long long payload_elements(int kind, long long E) {
  // kind 0: room for either lane width (deformed PW, regular kRegPW; PW | 16)
  const long long PW = kind == 0 ? kRegPW : Mode<S, P>::pw(kind);
  return (E + PW - 1) / PW * PW;
}

// write the payload entries of one deformed point from (dxi, w|J|)
template <int S, int P>
__device__ __forceinline__ void put_point(int kind, long long e, int l, const double (&dxi)[3][3], double wjac,
                                          double* __restrict__ pay, const double* __restrict__ gtab) {
  using Dm = Dims<S, P>;
  constexpr int NQ = Dm::NQ, PW0 = Mode<S, P>::pw(0), PW3 = Mode<S, P>::pw(3), PWW = Mode<S, P>::pw(1);
  const int k = l % Dm::Q2, ij = l / Dm::Q2;
  const long long km = k * Dm::Q0 * Dm::Q1 + ij;
  if (kind == 1) {
    pay[pay_base<PWW>(e, 1, NQ) + (long long)l * PWW] = wjac;
    return;
  }
  double G[3][3];
  const double* gs = gtab + GExt<S, P>::GST + 9 * l;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) G[a][b] = gs[3 * a + b];
  if (kind == 0 || kind == 3) {
    // Lam_ab = (sum_k dxi[a][k] dxi[b][k]) * w|J|  (field_block.py:349-362)
    double L[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = a; b < 3; ++b) {
        const double s = fma(dxi[a][2], dxi[b][2], fma(dxi[a][1], dxi[b][1], dxi[a][0] * dxi[b][0]));
        L[a][b] = L[b][a] = s * wjac;
      }
    // Lam' = G^T Lam G: the chain rule of operators.py:471-490, 510-523 folded
    double T[3][3];  // T = Lam G
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int n = 0; n < 3; ++n) T[a][n] = L[a][0] * G[0][n] + L[a][1] * G[1][n] + L[a][2] * G[2][n];
    const int mi[6] = {0, 0, 0, 1, 1, 2}, ni[6] = {0, 1, 2, 1, 2, 2};
    const int PW = kind == 3 ? PW3 : PW0;
    double* o = pay + (kind == 3 ? pay_base<PW3>(e, 7, NQ) + (long long)l * PW3 : pay_base<PW0>(e, 7, NQ) + km * PW0);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const int m = mi[c], n = ni[c];
      o[(long long)c * NQ * PW] = G[0][m] * T[0][n] + G[1][m] * T[1][n] + G[2][m] * T[2][n];
    }
    o[6LL * NQ * PW] = wjac;
    return;
  }
  // DERIV: T[m][j] = sum_a G[a][m] dxi[a][j]
  constexpr int PW = Mode<S, P>::pw(2);
  double* o = pay + pay_base<PW>(e, 9, NQ) + km * PW;
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      o[(long long)(m * 3 + j) * NQ * PW] = G[0][m] * dxi[0][j] + G[1][m] * dxi[1][j] + G[2][m] * dxi[2][j];
}

template <int S, int P>
__global__ void k_pack_deformed(int kind, long long E, const double* __restrict__ dxi, const double* __restrict__ jac,
                                double* __restrict__ pay, const double* __restrict__ gtab) {
  constexpr int NQ = Dims<S, P>::NQ;
  const long long n = E * NQ;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / NQ;
    const int l = (int)(t - e * NQ);
    double d[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) d[a][b] = dxi[t * 9 + a * 3 + b];
    put_point<S, P>(kind, e, l, d, jac[t], pay, gtab);
  }
}

template <int S, int P>
__global__ void k_pack_regular(int kind, long long E, const double* __restrict__ dxi, const double* __restrict__ jac,
                               double* __restrict__ pay) {
  constexpr int PW = Mode<S, P>::pw(0), PW3 = Mode<S, P>::pw(3), PWW = Mode<S, P>::pw(1);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x) {
    const double* d = dxi + e * 9;
    if (kind == 0 || kind == 3) {
      // kind 0 (collocated Helmholtz) uses the fixed regular lane width
      const int W0 = kind == 0 ? kRegPW : PW3;
      double* o = pay + (kind == 0 ? pay_base<kRegPW>(e, 8, 1) : pay_base<PW3>(e, 8, 1));
      const int mi[6] = {0, 0, 0, 1, 1, 2}, ni[6] = {0, 1, 2, 1, 2, 2};
      for (int c = 0; c < 6; ++c) {
        const int a = mi[c], b = ni[c];
        const double s = fma(d[a * 3 + 2], d[b * 3 + 2], fma(d[a * 3 + 1], d[b * 3 + 1], d[a * 3] * d[b * 3]));
        o[c * W0] = s * jac[e];
      }
      o[6 * W0] = jac[e];
      o[7 * W0] = 0.0;
    } else if (kind == 1) {
      pay[pay_base<PWW>(e, 1, 1)] = jac[e];
    } else {
      constexpr int PW2 = Mode<S, P>::pw(2);
      double* o = pay + pay_base<PW2>(e, 9, 1);
      for (int a = 0; a < 9; ++a) o[a * PW2] = d[a];
    }
  }
}

static unsigned grid_for(long long n, int bs) {
  long long g = (n + bs - 1) / bs;
  if (g > 148LL * 64) g = 148LL * 64;
  return (unsigned)(g < 1 ? 1 : g);
}

template <int S, int P>
int pack(int kind, int geo, long long E, const double* dxi, const double* jac, double* pay, const double* gtab,
         void* stream) {
  if (E == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (geo == GEO_DEFORMED)
    k_pack_deformed<S, P><<<grid_for(E * Dims<S, P>::NQ, 256), 256, 0, s>>>(kind, E, dxi, jac, pay, gtab);
  else
    k_pack_regular<S, P><<<grid_for(E, 256), 256, 0, s>>>(kind, E, dxi, jac, pay);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// device geometry builder: iso-parametric metric of deformed elements
// (geometry.py:161-212) from coordinates or from the seeded sinusoidal
// deformation parameters (geometry.py:275-300)
template <int S, int P, int MODE>
__global__ void __launch_bounds__(128) k_geom(long long E, const double* __restrict__ src, double* __restrict__ dxi_out,
                                              double* __restrict__ jac_out, int kind, double* __restrict__ pay,
                                              unsigned long long* bad, const double* __restrict__ gtab) {
  using Dm = Dims<S, P>;
  using X = GExt<S, P>;
  constexpr int NQ = Dm::NQ, Q0 = Dm::Q0, Q1 = Dm::Q1, Q2 = Dm::Q2;
  __shared__ double x[3][NQ];
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int l = threadIdx.x; l < NQ; l += blockDim.x) {
      if (MODE != 1) {  // coordinates (MODE 2: either orientation)
#pragma unroll
        for (int c = 0; c < 3; ++c) x[c][l] = src[(e * NQ + l) * 3 + c];
      } else {
        const int k = l % Q2, j = (l / Q2) % Q1, i = l / (Q1 * Q2);
        const double e1 = gtab[X::Z0 + i], e2 = gtab[X::Z1 + j], e3 = gtab[X::Z2 + k];
        // Duffy inverse (shapes.py:218-239)
        double xi[3] = {e1, e2, e3};
        if (S == PRISM) xi[0] = 0.5 * (1.0 + e1) * (1.0 - e3) - 1.0;
        if (S == PYR) {
          xi[0] = 0.5 * (1.0 + e1) * (1.0 - e3) - 1.0;
          xi[1] = 0.5 * (1.0 + e2) * (1.0 - e3) - 1.0;
        }
        if (S == TET) {
          xi[1] = 0.5 * (1.0 + e2) * (1.0 - e3) - 1.0;
          xi[0] = 0.25 * (1.0 + e1) * (1.0 - e2) * (1.0 - e3) - 1.0;
        }
        const double* pr = src + e * 12;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int perm = (int)pr[6 + c];
          x[c][l] = (xi[c] + pr[9 + c]) + pr[c] * sin(M_PI * xi[perm] + pr[3 + c]);
        }
      }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < NQ; l += blockDim.x) {
      const int k = l % Q2, j = (l / Q2) % Q1, i = l / (Q1 * Q2);
      double dx[3][3];  // dx[c][m] = d x_c / d eta_m
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int a = 0; a < Q0; ++a) s0 = fma(gtab[X::DM0 + i * Q0 + a], x[c][(a * Q1 + j) * Q2 + k], s0);
        for (int b = 0; b < Q1; ++b) s1 = fma(gtab[X::DM1 + j * Q1 + b], x[c][(i * Q1 + b) * Q2 + k], s1);
        for (int d = 0; d < Q2; ++d) s2 = fma(gtab[X::DM2 + k * Q2 + d], x[c][(i * Q1 + j) * Q2 + d], s2);
        dx[c][0] = s0;
        dx[c][1] = s1;
        dx[c][2] = s2;
      }
      // J[c][jj] = sum_m G[jj][m] dx[c][m]
      const double* G = gtab + X::GST + 9 * l;
      double J[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          if (S == HEX) {
            J[c][jj] = dx[c][jj];
          } else {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < 3; ++m)
              if (G[jj * 3 + m] != 0.0) s += (G[jj * 3 + m] == 1.0) ? dx[c][m] : dx[c][m] * G[jj * 3 + m];
            J[c][jj] = s;
          }
        }
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      // MODE 2 accepts reflected elements (the assembled tet mesh orders each
      // tet's vertices by global id): the weight uses |det J|
      if (!(MODE == 2 ? fabs(det) > 0.0 : det > 0.0)) atomicAdd(bad, 1ULL);
      const double id = 1.0 / det;
      double inv[3][3];
      inv[0][0] = c00 * id;
      inv[1][0] = c01 * id;
      inv[2][0] = c02 * id;
      inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
      inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
      inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
      inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
      inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
      inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
      const double wjac = gtab[GLayout<S, P>::REFW + l] * (MODE == 2 ? fabs(det) : det);
      if (dxi_out) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) dxi_out[(e * NQ + l) * 9 + a * 3 + b] = inv[a][b];
      }
      if (jac_out) jac_out[e * NQ + l] = wjac;
      if (kind >= 0) put_point<S, P>(kind, e, l, inv, wjac, pay, gtab);
    }
  }
}

template <int S, int P>
int geometry(int mode, long long E, const double* src, double* dxi, double* jac, int kind, double* pay,
             unsigned long long* bad, const double* gtab, void* stream) {
  if (E == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long g = E < 148LL * 32 ? E : 148LL * 32;
  if (mode == 0)
    k_geom<S, P, 0><<<(unsigned)g, 128, 0, s>>>(E, src, dxi, jac, kind, pay, bad, gtab);
  else if (mode == 2)
    k_geom<S, P, 2><<<(unsigned)g, 128, 0, s>>>(E, src, dxi, jac, kind, pay, bad, gtab);
  else
    k_geom<S, P, 1><<<(unsigned)g, 128, 0, s>>>(E, src, dxi, jac, kind, pay, bad, gtab);
  return (int)cudaGetLastError();
}

template <int S, int P>
const OpSet* opset_impl() {
  static const OpSet ops = {S,
                            P,
                            sizeof(FwdTab<S, P>),
                            sizeof(DTab<S, P>),
                            GExt<S, P>::SIZE,
                            &fill<S, P>,
                            &fill_gtab<S, P>,
                            &launch<S, P>,
                            &config<S, P>,
                            &payload_doubles<S, P>,
                            &payload_elements<S, P>,
                            &pack<S, P>,
                            &geometry<S, P>,
                            P <= kDenseMaxP ? DenseDims<S, P>::DOUBLES : 0,
                            P <= kDenseMaxP ? DenseDims<S, P>::MASK : 0,
                            &fill_dense_frags<S, P>};
  return &ops;
}

template const OpSet* opset_impl<SK_S, SK_P>();

}  // namespace sk

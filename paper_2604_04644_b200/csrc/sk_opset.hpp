// Type-erased per-(shape, order) entry points, implemented by the
// explicit instantiations in inst.cu (one object file per (shape, order)).
#pragma once

#include <cstddef>
#include <cstdint>

#include "basis_host.hpp"

namespace sk {

enum OpId : int { OP_HELM = 0, OP_MASS = 1, OP_BWD = 2, OP_IPROD = 3, OP_PDERIV = 4, OP_IPDERIV = 5, OP_HELM_NC = 6,
                  // staged collocated Helmholtz (bwd -> OP_QP -> OP_BT): the quadrature-point
                  // kernel and the unweighted B^T
                  OP_QP = 7, OP_BT = 8, OP_COUNT = 9 };

struct LaunchReq {
  const void* fwd;    // FwdTab<S,P> (host copy, values)
  const void* fwd_d;  // FwdTab<S,P> (host copy, derivatives)
  const void* dtab;   // DTab<S,P>   (host copy)
  const double* in;
  double* out;
  const double* pay;
  const double* gtab;  // device table buffer
  long long E, Epad, in_cs, out_cs;
  int W, ncomp, geo;
  double lam;
  int c0_nx = 0, c0_ny = 0;  // > 0: assembled C0 hex slab, `in` is the global DOF vector
  const int* c0map = nullptr;  // assembled C0 on a mapped mesh: compact l2g, `in` is the global DOF vector
  const double* dense = nullptr;  // mass only: DMMA StdMat fragments (sk_dense.cuh) -> dense kernel
};

struct OpSet {
  int S, P;
  size_t fwd_bytes, dtab_bytes;
  int gtab_doubles;
  void (*fill)(const HostBasis& hb, void* fwd_vals, void* fwd_ders, void* dtab);
  void (*fill_gtab)(const HostBasis& hb, double* gtab_host);
  // returns a cudaError_t value (0 = success)
  int (*launch)(int op, const LaunchReq& r, void* stream);
  void (*config)(int op, int geo, int64_t out[3]);  // geo: GEO_REGULAR / GEO_DEFORMED
  // payload kinds: 0 HELMHOLTZ (k-major), 1 W, 2 DERIV, 3 HELMHOLTZ (standard order)
  long long (*payload_doubles)(int kind, int geo);  // per element
  long long (*payload_elements)(int kind, long long E);  // elements incl. lane padding
  int (*pack)(int kind, int geo, long long E, const double* dxi, const double* jac, double* pay,
              const double* gtab, void* stream);
  // geometry builder: mode 0 from coords (E,NQ,3), mode 1 from params (E,12),
  // mode 2 from coords accepting either orientation (w|det J|).
  // Writes dxi/jac (either may be null) and/or the payload of `kind`
  // (kind < 0: none).  Counts nonpositive-Jacobian points into *bad (device).
  int (*geometry)(int mode, long long E, const double* src, double* dxi, double* jac, int kind,
                  double* pay, unsigned long long* bad, const double* gtab, void* stream);
  // dense (StdMat, DMMA) mass: fragment table size in doubles (0: not
  // instantiated for this order) and its host fill from the dense basis
  // matrix B (NQ x NM row-major) and the reference weights
  int dense_doubles;
  int dense_mask;  // dense kernels: bit 0 regular mass, bit 1 deformed mass, bit 2 regular Helmholtz
  void (*fill_dense)(const HostBasis& hb, const double* B, double* frags);
};

template <int S, int P>
const OpSet* opset_impl();

const OpSet* opset(int internal_shape, int P);

}  // namespace sk

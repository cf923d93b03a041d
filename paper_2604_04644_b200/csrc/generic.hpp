// Run-time-size device path for quadrature overrides (generic.cu).
#pragma once

namespace sk {

enum GenOp : int { GEN_BWD = 0, GEN_IPROD = 1, GEN_MASS = 2, GEN_HELM = 3, GEN_PDERIV = 4, GEN_IPDERIV = 5 };

// device tables of one basis (uploaded by abi.cu per device)
struct GenTables {
  const double *B, *DB0, *DB1, *DB2;  // nq x nm, row-major
  const double *D0, *D1, *D2;         // Q_d x Q_d collocation matrices
  const double *G, *refw;             // nq x 9, nq
  const double *z0, *z1, *z2;         // 1D points
  int Q[3];
  int nq, nm, shape;                  // internal shape id (0 hex .. 3 tet)
};

struct GenReq {
  int op, geo;  // geo: 0 regular, 1 deformed
  long long E, Epad, in_cs, out_cs;
  int W, ncomp;
  const double* in;
  double* out;
  const double* pay;  // [dxi (E, nd, 9) | w|J| (E, nd)], nd = nq (deformed) or 1 (regular)
  double lam;
};

int generic_launch(const GenTables& t, const GenReq& r, void* stream);
// mode 0 coords, 1 deformation params, 2 coords of either orientation
int generic_geometry(const GenTables& t, int mode, long long E, const double* src, double* dxi, double* jac,
                     unsigned long long* bad, void* stream);

}  // namespace sk

// Host-side constant tables per (shape, order): native FP64 rebuild of the
// reference's 1D rules, modified bases and sum-factorisation tables
// (speckern/bases.py, speckern/shapes.py).  Consumed by the kernel-table
// fill in abi.cu; read back by tests through sk_basis_table().
#pragma once

#include <map>
#include <string>
#include <vector>

#include "sk_shapes.hpp"

namespace sk {

struct HostBasis {
  int shape = 0, P = 0;
  int Q[3] = {0, 0, 0};
  int nq = 0, nm = 0;
  std::vector<double> z[3], w[3];    // 1D points / weights per direction
  std::vector<double> D[3];          // Q_d x Q_d collocation matrices, row-major
  std::vector<double> refw;          // nq tensor weights incl. Duffy scale
  std::vector<double> G;             // nq x 3 x 3 dense chain-rule factors
  // full 1D families, Q_d x (P+1) row-major (values, derivatives); empty when warped
  std::vector<double> a[3], da[3];
  // warped families, per leading index p: Q x (P+1-p) row-major
  std::vector<std::vector<double>> b1, db1;  // direction 1 (tet)
  std::vector<std::vector<double>> c2, dc2;  // direction 2 (prism, pyr, tet)
  std::vector<int> modes;            // nm x 3 (p, q, r)
  // dense basis matrix (nq x nm, row-major) and its collocation derivatives
  // per tensor direction: the generic (quadrature-override) device path
  std::vector<double> Bd, DBd[3];
  std::map<std::string, std::vector<double>> named;  // flat view for sk_basis_table
};

// Build all tables; returns false for unsupported (shape, order) or a
// quadrature override below the default counts.  qpoints: per-direction point
// counts (null: P+2 Gauss-Lobatto / P+1 Gauss-Radau-Jacobi, shapes.py:132-139).
bool build_host_basis(int shape, int P, HostBasis& out, const int* qpoints = nullptr);
void build_dense(HostBasis& B);

int mode_count(int shape, int P);

}  // namespace sk

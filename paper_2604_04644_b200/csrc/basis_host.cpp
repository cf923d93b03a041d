// Native FP64 construction of the per-(shape, order) tables.
//
// Follows the reference definitions:
//   Jacobi recurrence            speckern/bases.py:146-174
//   GLL / Gauss-Radau-Jacobi     speckern/bases.py:177-270
//   modified psi^a / psi^b       speckern/bases.py:277-340
//   collocation derivative D     speckern/bases.py:468-477
//   quadrature composition       speckern/shapes.py:76-139, 482-487
//   Duffy chain-rule factors G   speckern/shapes.py:265-323
//   sum-fac tables               speckern/shapes.py:555-583
#include "basis_host.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace sk {
namespace {

double jacobi(int n, double a, double b, double z) {
  double prev = 1.0;
  if (n == 0) return prev;
  double cur = 0.5 * ((a + b + 2.0) * z + (a - b));
  for (int k = 2; k <= n; ++k) {
    const double s = 2.0 * k + a + b;
    const double c1 = 2.0 * k * (k + a + b) * (s - 2.0);
    const double c2 = (s - 1.0) * (a * a - b * b);
    const double c3 = (s - 2.0) * (s - 1.0) * s;
    const double c4 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * s;
    const double nxt = ((c2 + c3 * z) * cur - c4 * prev) / c1;
    prev = cur;
    cur = nxt;
  }
  return cur;
}

double jacobi_d(int n, double a, double b, double z) {
  if (n == 0) return 0.0;
  return 0.5 * (n + a + b + 1.0) * jacobi(n - 1, a + 1.0, b + 1.0, z);
}

// roots of P_n^{(a,b)}, increasing, deflated Newton from Chebyshev guesses
std::vector<double> jacobi_roots(int n, double a, double b) {
  std::vector<double> r(n);
  for (int k = 0; k < n; ++k) {
    double x = -std::cos(M_PI * (2.0 * k + 1.0) / (2.0 * n));
    if (k) x = 0.5 * (x + r[k - 1]);
    for (int it = 0; it < 100; ++it) {
      const double f = jacobi(n, a, b, x), fp = jacobi_d(n, a, b, x);
      double s = 0.0;
      for (int m = 0; m < k; ++m) s += 1.0 / (x - r[m]);
      const double dx = -f / (fp - s * f);
      x += dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    r[k] = x;
  }
  for (int k = 0; k < n; ++k)
    if (r[k] <= -1.0 || r[k] >= 1.0 || (k && r[k] - r[k - 1] <= 1e-12))
      throw std::runtime_error("Jacobi root iteration failed");
  return r;
}

// dense solve A x = rhs (n small), Gaussian elimination with partial pivoting
std::vector<double> solve(std::vector<double> A, std::vector<double> rhs, int n) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[piv * n + k]);
      std::swap(rhs[c], rhs[piv]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      rhs[r] -= f * rhs[c];
    }
  }
  std::vector<double> x(n);
  for (int r = n - 1; r >= 0; --r) {
    double s = rhs[r];
    for (int k = r + 1; k < n; ++k) s -= A[r * n + k] * x[k];
    x[r] = s / A[r * n + r];
  }
  return x;
}

enum Kind { GLL = 0, GRJ1 = 1, GRJ2 = 2 };

void rule(Kind kind, int q, std::vector<double>& z, std::vector<double>& w) {
  z.assign(q, 0.0);
  w.assign(q, 0.0);
  if (kind == GLL) {
    z[0] = -1.0;
    z[q - 1] = 1.0;
    if (q > 2) {
      auto in = jacobi_roots(q - 2, 1.0, 1.0);
      for (int i = 0; i < q - 2; ++i) z[i + 1] = in[i];
    }
    for (int i = 0; i < q; ++i) {
      const double p = jacobi(q - 1, 0.0, 0.0, z[i]);
      w[i] = 2.0 / (q * (q - 1) * p * p);
    }
    return;
  }
  const int alpha = kind == GRJ1 ? 1 : 2;
  z[0] = -1.0;
  auto in = jacobi_roots(q - 1, double(alpha), 1.0);
  for (int i = 0; i < q - 1; ++i) z[i + 1] = in[i];
  // exactness against Legendre P_0..P_{q-1} with weight (1-z)^alpha
  std::vector<double> mom(q, 0.0);
  if (alpha == 1) {
    mom[0] = 2.0;
    if (q > 1) mom[1] = -2.0 / 3.0;
  } else {
    mom[0] = 8.0 / 3.0;
    if (q > 1) mom[1] = -4.0 / 3.0;
    if (q > 2) mom[2] = 4.0 / 15.0;
  }
  std::vector<double> V(q * q);
  for (int k = 0; k < q; ++k)
    for (int i = 0; i < q; ++i) V[k * q + i] = jacobi(k, 0.0, 0.0, z[i]);
  w = solve(V, mom, q);
}

double psi_a(int p, double z) {
  if (p == 0) return 0.5 * (1.0 - z);
  if (p == 1) return 0.5 * (1.0 + z);
  return 0.25 * (1.0 - z) * (1.0 + z) * jacobi(p - 2, 1.0, 1.0, z);
}

double psi_a_d(int p, double z) {
  if (p == 0) return -0.5;
  if (p == 1) return 0.5;
  return -0.5 * z * jacobi(p - 2, 1.0, 1.0, z) +
         0.25 * (1.0 - z) * (1.0 + z) * jacobi_d(p - 2, 1.0, 1.0, z);
}

double psi_b(int p, int q, double z) {
  if (p == 0) return psi_a(q, z);
  const double lead = std::pow(0.5 * (1.0 - z), p);
  if (q == 0) return lead;
  return lead * 0.5 * (1.0 + z) * jacobi(q - 1, 2.0 * p - 1.0, 1.0, z);
}

double psi_b_d(int p, int q, double z) {
  if (p == 0) return psi_a_d(q, z);
  const double lead = std::pow(0.5 * (1.0 - z), p);
  const double dlead = -0.5 * p * std::pow(0.5 * (1.0 - z), p - 1);
  if (q == 0) return dlead;
  const double j = jacobi(q - 1, 2.0 * p - 1.0, 1.0, z);
  const double dj = jacobi_d(q - 1, 2.0 * p - 1.0, 1.0, z);
  return dlead * (0.5 * (1.0 + z) * j) + lead * (0.5 * j + 0.5 * (1.0 + z) * dj);
}

std::vector<double> diff_matrix(const std::vector<double>& z) {
  const int n = int(z.size());
  std::vector<double> lam(n), d(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double p = 1.0;
    for (int k = 0; k < n; ++k)
      if (k != i) p *= (z[i] - z[k]);
    lam[i] = 1.0 / p;
  }
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
      if (k == i) continue;
      d[i * n + k] = (lam[k] / lam[i]) / (z[i] - z[k]);
      s += d[i * n + k];
    }
    d[i * n + i] = -s;
  }
  return d;
}

void full_family(int P, const std::vector<double>& z, std::vector<double>& v, std::vector<double>& dv) {
  const int Q = int(z.size());
  v.assign(Q * (P + 1), 0.0);
  dv.assign(Q * (P + 1), 0.0);
  for (int i = 0; i < Q; ++i)
    for (int p = 0; p <= P; ++p) {
      v[i * (P + 1) + p] = psi_a(p, z[i]);
      dv[i * (P + 1) + p] = psi_a_d(p, z[i]);
    }
}

void warped_family(int P, const std::vector<double>& z, std::vector<std::vector<double>>& v,
                   std::vector<std::vector<double>>& dv) {
  const int Q = int(z.size());
  v.assign(P + 1, {});
  dv.assign(P + 1, {});
  for (int p = 0; p <= P; ++p) {
    const int n = P + 1 - p;
    v[p].assign(Q * n, 0.0);
    dv[p].assign(Q * n, 0.0);
    for (int i = 0; i < Q; ++i)
      for (int q = 0; q < n; ++q) {
        v[p][i * n + q] = psi_b(p, q, z[i]);
        dv[p][i * n + q] = psi_b_d(p, q, z[i]);
      }
  }
}

}  // namespace

// Dense basis matrix B[l][m] (shapes.py:491-492 bmat; mode factors with the
// collapsed-vertex exceptions of shapes.py:374-405) and its collocation
// derivatives DB_d = D_d B along each tensor direction (operators.py:449-464)
void build_dense(HostBasis& B) {
  const int Q0 = B.Q[0], Q1 = B.Q[1], Q2 = B.Q[2], P1 = B.P + 1, nm = B.nm, nq = B.nq;
  B.Bd.assign((size_t)nq * nm, 0.0);
  for (int m = 0; m < nm; ++m) {
    const int p = B.modes[3 * m], q = B.modes[3 * m + 1], r = B.modes[3 * m + 2];
    for (int i = 0; i < Q0; ++i)
      for (int j = 0; j < Q1; ++j)
        for (int k = 0; k < Q2; ++k) {
          double f0 = B.a[0][i * P1 + p], f1 = 0.0, f2 = 0.0;
          switch (B.shape) {
            case HEX:
              f1 = B.a[1][j * P1 + q];
              f2 = B.a[2][k * P1 + r];
              break;
            case PRISM:
              f1 = B.a[1][j * P1 + q];
              f2 = B.c2[p][k * (P1 - p) + r];
              if (p == 0 && r == 1) f0 = 1.0;  // (0, q, 1): psi_b(0,1)(eta3) psi_a(q)(eta2)
              break;
            case PYR: {
              const int mx = std::max(p, q);
              f1 = B.a[1][j * P1 + q];
              f2 = B.c2[mx][k * (P1 - mx) + r];
              if (p == 0 && q == 0 && r == 1) f0 = f1 = 1.0;  // apex
              break;
            }
            case TET:
              f1 = B.b1[p][j * (P1 - p) + q];
              f2 = B.c2[p + q][k * (P1 - p - q) + r];
              if (p == 0 && q == 0 && r == 1) f0 = f1 = 1.0;  // apex
              if (p == 0 && q == 1) {                        // (0, 1, r): psi_b(0,1)(eta2) psi_b(1,r)(eta3)
                f0 = 1.0;
                f1 = B.b1[0][j * P1 + 1];
                f2 = B.c2[1][k * (P1 - 1) + r];
              }
              break;
          }
          B.Bd[(size_t)((i * Q1 + j) * Q2 + k) * nm + m] = f0 * f1 * f2;
        }
  }
  for (int d = 0; d < 3; ++d) {
    B.DBd[d].assign((size_t)nq * nm, 0.0);
    const int Qd = B.Q[d];
    for (int i = 0; i < Q0; ++i)
      for (int j = 0; j < Q1; ++j)
        for (int k = 0; k < Q2; ++k) {
          const int l = (i * Q1 + j) * Q2 + k, a = d == 0 ? i : d == 1 ? j : k;
          for (int b = 0; b < Qd; ++b) {
            const int lb = d == 0 ? (b * Q1 + j) * Q2 + k : d == 1 ? (i * Q1 + b) * Q2 + k : (i * Q1 + j) * Q2 + b;
            const double dab = B.D[d][a * Qd + b];
            if (dab == 0.0) continue;
            for (int m = 0; m < nm; ++m) B.DBd[d][(size_t)l * nm + m] += dab * B.Bd[(size_t)lb * nm + m];
          }
        }
  }
}

int mode_count(int shape, int P) {
  switch (shape) {
    case HEX: return (P + 1) * (P + 1) * (P + 1);
    case PRISM: return (P + 1) * (P + 1) * (P + 2) / 2;
    case PYR: return (P + 1) * (P + 2) * (2 * P + 3) / 6;
    case TET: return (P + 1) * (P + 2) * (P + 3) / 6;
  }
  return 0;
}

bool build_host_basis(int shape, int P, HostBasis& B, const int* qpoints) {
  if (shape < HEX || shape > TET || P < 1 || P > 10) return false;
  static const Kind kinds[4][3] = {
      {GLL, GLL, GLL}, {GLL, GLL, GRJ1}, {GLL, GLL, GRJ2}, {GLL, GRJ1, GRJ2}};
  static const double scale[4][3] = {
      {1.0, 1.0, 1.0}, {1.0, 1.0, 0.5}, {1.0, 1.0, 0.25}, {1.0, 0.5, 0.25}};
  B = HostBasis();
  B.shape = shape;
  B.P = P;
  for (int d = 0; d < 3; ++d) {
    const int qdef = kinds[shape][d] == GLL ? P + 2 : P + 1;
    // shapes.py:532-541: an override may only raise the per-direction count
    if (qpoints && qpoints[d] < qdef) return false;
    B.Q[d] = qpoints ? qpoints[d] : qdef;
    rule(kinds[shape][d], B.Q[d], B.z[d], B.w[d]);
    B.D[d] = diff_matrix(B.z[d]);
  }
  const int Q0 = B.Q[0], Q1 = B.Q[1], Q2 = B.Q[2];
  B.nq = Q0 * Q1 * Q2;
  B.nm = mode_count(shape, P);
  // tensor weights, first direction slowest
  B.refw.resize(B.nq);
  B.G.assign(B.nq * 9, 0.0);
  for (int i = 0; i < Q0; ++i)
    for (int j = 0; j < Q1; ++j)
      for (int k = 0; k < Q2; ++k) {
        const int l = (i * Q1 + j) * Q2 + k;
        B.refw[l] = (B.w[0][i] * scale[shape][0]) * (B.w[1][j] * scale[shape][1]) *
                    (B.w[2][k] * scale[shape][2]);
        const double e1 = B.z[0][i], e2 = B.z[1][j], e3 = B.z[2][k];
        double* g = &B.G[l * 9];
        switch (shape) {
          case HEX: g[0] = g[4] = g[8] = 1.0; break;
          case PRISM:
            g[0] = 2.0 / (1.0 - e3);
            g[4] = 1.0;
            g[6] = (1.0 + e1) / (1.0 - e3);
            g[8] = 1.0;
            break;
          case PYR:
            g[0] = 2.0 / (1.0 - e3);
            g[4] = 2.0 / (1.0 - e3);
            g[6] = (1.0 + e1) / (1.0 - e3);
            g[7] = (1.0 + e2) / (1.0 - e3);
            g[8] = 1.0;
            break;
          case TET:
            g[0] = 4.0 / ((1.0 - e2) * (1.0 - e3));
            g[3] = 2.0 * (1.0 + e1) / ((1.0 - e2) * (1.0 - e3));
            g[4] = 2.0 / (1.0 - e3);
            g[6] = 2.0 * (1.0 + e1) / ((1.0 - e2) * (1.0 - e3));
            g[7] = (1.0 + e2) / (1.0 - e3);
            g[8] = 1.0;
            break;
        }
      }
  full_family(P, B.z[0], B.a[0], B.da[0]);
  if (shape != TET) full_family(P, B.z[1], B.a[1], B.da[1]);
  if (shape == HEX) full_family(P, B.z[2], B.a[2], B.da[2]);
  if (shape == TET) warped_family(P, B.z[1], B.b1, B.db1);
  if (shape != HEX) warped_family(P, B.z[2], B.c2, B.dc2);
  // lexicographic modes (shapes.py:142-179)
  for (int p = 0; p <= P; ++p) {
    const int nqm = shape == TET ? P + 1 - p : P + 1;
    for (int q = 0; q < nqm; ++q) {
      int nr = P + 1;
      if (shape == PRISM) nr = P + 1 - p;
      if (shape == PYR) nr = P + 1 - std::max(p, q);
      if (shape == TET) nr = P + 1 - p - q;
      for (int r = 0; r < nr; ++r) {
        B.modes.push_back(p);
        B.modes.push_back(q);
        B.modes.push_back(r);
      }
    }
  }
  if (int(B.modes.size()) != 3 * B.nm) throw std::runtime_error("mode count mismatch");
  // named flat view
  auto& N = B.named;
  for (int d = 0; d < 3; ++d) {
    const std::string s = std::to_string(d);
    N["z" + s] = B.z[d];
    N["w" + s] = B.w[d];
    N["D" + s] = B.D[d];
    if (!B.a[d].empty()) {
      N["a" + s] = B.a[d];
      N["da" + s] = B.da[d];
    }
  }
  for (size_t p = 0; p < B.b1.size(); ++p) {
    N["b1_" + std::to_string(p)] = B.b1[p];
    N["db1_" + std::to_string(p)] = B.db1[p];
  }
  for (size_t p = 0; p < B.c2.size(); ++p) {
    N["c2_" + std::to_string(p)] = B.c2[p];
    N["dc2_" + std::to_string(p)] = B.dc2[p];
  }
  N["refw"] = B.refw;
  N["G"] = B.G;
  if (qpoints) {  // the generic device path of a quadrature override works on dense matrices
    build_dense(B);
    N["B"] = B.Bd;
  }
  N["modes"] = std::vector<double>(B.modes.begin(), B.modes.end());
  return true;
}

}  // namespace sk

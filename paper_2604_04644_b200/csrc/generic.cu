// Generic device path for bases with a quadrature override (build_shape_basis
// qpoints, shapes.py:521-541: each per-direction count at or above the
// default).  The specialised kernels are compiled for the default rules, so
// these operators run on run-time sizes with the dense basis matrix B and its
// collocation derivatives DB_d = D_d B (basis_host.cpp build_dense), one CTA
// per element.  Same algebra as the reference's operators (operators.py:
// 551-699): bwd u = B uhat; iproduct B^T W u; mass B^T W B uhat; Helmholtz
// sum_d DB_d^T (G^T Lam G DB uhat)_d + lam B^T W B uhat (the collocated and
// non-collocated forms coincide: D_d B is exact for these polynomial spaces);
// phys_deriv dxi^T G (D_d u); iproduct_deriv sum_k DB_k^T W v_k.  The
// geometry payload is the reference factors themselves: [dxi (E, nd, 3, 3) |
// w|J| (E, nd)], nd = NQ (deformed) or 1 (regular).
#include <cuda_runtime.h>

#include "generic.hpp"

namespace sk {

namespace {

constexpr int kGenThreads = 128;

__device__ __forceinline__ long long lane_at(long long e, int n, int N, int W) {
  const long long g = e / W;
  return (g * N + n) * (long long)W + (e - g * W);
}

// quadrature weight W at point l (operators.py:493-499)
__device__ __forceinline__ double wpoint(const GenTables& t, const GenReq& r, long long e, int l) {
  if (r.geo == 1) return r.pay[r.E * (long long)t.nq * 9 + e * t.nq + l];
  return t.refw[l] * r.pay[r.E * 9 + e];
}

__device__ __forceinline__ const double* dxi_at(const GenTables& t, const GenReq& r, long long e, int l) {
  return r.geo == 1 ? r.pay + (e * t.nq + l) * 9 : r.pay + e * 9;
}

__global__ void __launch_bounds__(kGenThreads) k_gen(const GenTables t, const GenReq r) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  const bool live = e < r.E;
  const int nq = t.nq, nm = t.nm;
  const double* src = r.in + blockIdx.y * r.in_cs;
  double* dst = r.out + blockIdx.y * r.out_cs;
  const int tid = threadIdx.x;
  switch (r.op) {
    case GEN_BWD: {
      for (int m = tid; m < nm; m += kGenThreads) sm[m] = src[lane_at(e, m, nm, r.W)];
      __syncthreads();
      for (int l = tid; l < nq; l += kGenThreads) {
        double u = 0.0;
        for (int m = 0; m < nm; ++m) u = fma(t.B[(long long)l * nm + m], sm[m], u);
        dst[lane_at(e, l, nq, r.W)] = live ? u : 0.0;
      }
      return;
    }
    case GEN_IPROD: {
      for (int l = tid; l < nq; l += kGenThreads) sm[l] = live ? src[lane_at(e, l, nq, r.W)] * wpoint(t, r, e, l) : 0.0;
      __syncthreads();
      for (int m = tid; m < nm; m += kGenThreads) {
        double f = 0.0;
        for (int l = 0; l < nq; ++l) f = fma(t.B[(long long)l * nm + m], sm[l], f);
        dst[lane_at(e, m, nm, r.W)] = f;
      }
      return;
    }
    case GEN_MASS: {
      double* x = sm;
      double* v = sm + nm;
      for (int m = tid; m < nm; m += kGenThreads) x[m] = src[lane_at(e, m, nm, r.W)];
      __syncthreads();
      for (int l = tid; l < nq; l += kGenThreads) {
        double u = 0.0;
        for (int m = 0; m < nm; ++m) u = fma(t.B[(long long)l * nm + m], x[m], u);
        v[l] = live ? u * wpoint(t, r, e, l) : 0.0;
      }
      __syncthreads();
      for (int m = tid; m < nm; m += kGenThreads) {
        double f = 0.0;
        for (int l = 0; l < nq; ++l) f = fma(t.B[(long long)l * nm + m], v[l], f);
        dst[lane_at(e, m, nm, r.W)] = f;
      }
      return;
    }
    case GEN_HELM: {
      double* x = sm;
      double* z = sm + nm;       // lam W u
      double* w0 = z + nq;       // G^T Lam G grad, per direction
      double* w1 = w0 + nq;
      double* w2 = w1 + nq;
      for (int m = tid; m < nm; m += kGenThreads) x[m] = src[lane_at(e, m, nm, r.W)];
      __syncthreads();
      for (int l = tid; l < nq; l += kGenThreads) {
        double u = 0.0, g[3] = {0.0, 0.0, 0.0};
        for (int m = 0; m < nm; ++m) {
          const double xm = x[m];
          const long long o = (long long)l * nm + m;
          u = fma(t.B[o], xm, u);
          g[0] = fma(t.DB0[o], xm, g[0]);
          g[1] = fma(t.DB1[o], xm, g[1]);
          g[2] = fma(t.DB2[o], xm, g[2]);
        }
        const double* G = t.G + l * 9;  // grad_xi = G grad_eta (shapes.py:292-316)
        double tt[3];
        for (int i = 0; i < 3; ++i) tt[i] = G[3 * i] * g[0] + G[3 * i + 1] * g[1] + G[3 * i + 2] * g[2];
        // Lam_ij = (sum_k dxi[i][k] dxi[j][k]) * w|J| (field_block.py:349-362);
        // regular: times the reference weight (operators.py:513-522)
        const double* d = dxi_at(t, r, e, l);
        const double jw = r.geo == 1 ? r.pay[r.E * (long long)nq * 9 + e * nq + l] : r.pay[r.E * 9 + e] * t.refw[l];
        double ww[3];
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int i = 0; i < 3; ++i) {
            const double lij = d[3 * i] * d[3 * j] + d[3 * i + 1] * d[3 * j + 1] + d[3 * i + 2] * d[3 * j + 2];
            s = fma(lij, tt[i], s);
          }
          ww[j] = live ? s * jw : 0.0;
        }
        w0[l] = G[0] * ww[0] + G[3] * ww[1] + G[6] * ww[2];
        w1[l] = G[1] * ww[0] + G[4] * ww[1] + G[7] * ww[2];
        w2[l] = G[2] * ww[0] + G[5] * ww[1] + G[8] * ww[2];
        z[l] = live ? r.lam * wpoint(t, r, e, l) * u : 0.0;
      }
      __syncthreads();
      for (int m = tid; m < nm; m += kGenThreads) {
        double f = 0.0;
        for (int l = 0; l < nq; ++l) {
          const long long o = (long long)l * nm + m;
          f = fma(t.B[o], z[l], f);
          f = fma(t.DB0[o], w0[l], f);
          f = fma(t.DB1[o], w1[l], f);
          f = fma(t.DB2[o], w2[l], f);
        }
        dst[lane_at(e, m, nm, r.W)] = f;
      }
      return;
    }
    case GEN_PDERIV: {
      const int Q0 = t.Q[0], Q1 = t.Q[1], Q2 = t.Q[2];
      for (int l = tid; l < nq; l += kGenThreads) sm[l] = live ? src[lane_at(e, l, nq, r.W)] : 0.0;
      __syncthreads();
      if (e >= r.Epad) return;
      for (int l = tid; l < nq; l += kGenThreads) {
        const int k = l % Q2, j = (l / Q2) % Q1, i = l / (Q1 * Q2);
        double g[3] = {0.0, 0.0, 0.0};
        for (int b = 0; b < Q0; ++b) g[0] = fma(t.D0[i * Q0 + b], sm[(b * Q1 + j) * Q2 + k], g[0]);
        for (int b = 0; b < Q1; ++b) g[1] = fma(t.D1[j * Q1 + b], sm[(i * Q1 + b) * Q2 + k], g[1]);
        for (int b = 0; b < Q2; ++b) g[2] = fma(t.D2[k * Q2 + b], sm[(i * Q1 + j) * Q2 + b], g[2]);
        const double* G = t.G + l * 9;
        double tt[3];
        for (int a = 0; a < 3; ++a) tt[a] = G[3 * a] * g[0] + G[3 * a + 1] * g[1] + G[3 * a + 2] * g[2];
        const double* d = dxi_at(t, r, e, l);
        for (int jj = 0; jj < 3; ++jj) {
          const double v = d[jj] * tt[0] + d[3 + jj] * tt[1] + d[6 + jj] * tt[2];
          r.out[jj * r.out_cs + lane_at(e, l, nq, r.W)] = live ? v : 0.0;
        }
      }
      return;
    }
    case GEN_IPDERIV: {
      double* v0 = sm;
      double* v1 = v0 + nq;
      double* v2 = v1 + nq;
      for (int l = tid; l < nq; l += kGenThreads) {
        const double w = live ? wpoint(t, r, e, l) : 0.0;
        const long long a = lane_at(e, l, nq, r.W);
        v0[l] = live ? r.in[a] * w : 0.0;
        v1[l] = live ? r.in[r.in_cs + a] * w : 0.0;
        v2[l] = live ? r.in[2 * r.in_cs + a] * w : 0.0;
      }
      __syncthreads();
      for (int m = tid; m < nm; m += kGenThreads) {
        double f = 0.0;
        for (int l = 0; l < nq; ++l) {
          const long long o = (long long)l * nm + m;
          f = fma(t.DB0[o], v0[l], f);
          f = fma(t.DB1[o], v1[l], f);
          f = fma(t.DB2[o], v2[l], f);
        }
        r.out[lane_at(e, m, nm, r.W)] = f;
      }
      return;
    }
  }
}

// Iso-parametric factors at the override's points (geometry.py:161-212),
// from coordinates (mode 0 / 2) or the seeded deformation parameters (mode 1,
// geometry.py:275-300); mode 2 accepts either orientation (w|det J|).
__global__ void __launch_bounds__(kGenThreads) k_gen_geom(const GenTables t, int mode, long long E,
                                                          const double* __restrict__ src, double* __restrict__ dxi,
                                                          double* __restrict__ jac, unsigned long long* bad) {
  extern __shared__ double sm[];
  const int nq = t.nq, Q0 = t.Q[0], Q1 = t.Q[1], Q2 = t.Q[2];
  double* x = sm;  // [3][nq]
  for (long long e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int l = threadIdx.x; l < nq; l += kGenThreads) {
      if (mode != 1) {
        for (int c = 0; c < 3; ++c) x[c * nq + l] = src[(e * nq + l) * 3 + c];
      } else {
        const int k = l % Q2, j = (l / Q2) % Q1, i = l / (Q1 * Q2);
        const double e1 = t.z0[i], e2 = t.z1[j], e3 = t.z2[k];
        double xi[3] = {e1, e2, e3};  // Duffy inverse (shapes.py:218-239)
        if (t.shape == 1) xi[0] = 0.5 * (1.0 + e1) * (1.0 - e3) - 1.0;
        if (t.shape == 2) {
          xi[0] = 0.5 * (1.0 + e1) * (1.0 - e3) - 1.0;
          xi[1] = 0.5 * (1.0 + e2) * (1.0 - e3) - 1.0;
        }
        if (t.shape == 3) {
          xi[1] = 0.5 * (1.0 + e2) * (1.0 - e3) - 1.0;
          xi[0] = 0.25 * (1.0 + e1) * (1.0 - e2) * (1.0 - e3) - 1.0;
        }
        const double* pr = src + e * 12;
        for (int c = 0; c < 3; ++c) {
          const int perm = (int)pr[6 + c];
          x[c * nq + l] = (xi[c] + pr[9 + c]) + pr[c] * sin(M_PI * xi[perm] + pr[3 + c]);
        }
      }
    }
    __syncthreads();
    for (int l = threadIdx.x; l < nq; l += kGenThreads) {
      const int k = l % Q2, j = (l / Q2) % Q1, i = l / (Q1 * Q2);
      double dx[3][3];
      for (int c = 0; c < 3; ++c) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int a = 0; a < Q0; ++a) s0 = fma(t.D0[i * Q0 + a], x[c * nq + (a * Q1 + j) * Q2 + k], s0);
        for (int b = 0; b < Q1; ++b) s1 = fma(t.D1[j * Q1 + b], x[c * nq + (i * Q1 + b) * Q2 + k], s1);
        for (int d = 0; d < Q2; ++d) s2 = fma(t.D2[k * Q2 + d], x[c * nq + (i * Q1 + j) * Q2 + d], s2);
        dx[c][0] = s0;
        dx[c][1] = s1;
        dx[c][2] = s2;
      }
      const double* G = t.G + 9 * l;
      double J[3][3];
      for (int c = 0; c < 3; ++c)
        for (int jj = 0; jj < 3; ++jj) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m)
            if (G[jj * 3 + m] != 0.0) s += (G[jj * 3 + m] == 1.0) ? dx[c][m] : dx[c][m] * G[jj * 3 + m];
          J[c][jj] = s;
        }
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      if (!(mode == 2 ? fabs(det) > 0.0 : det > 0.0)) atomicAdd(bad, 1ULL);
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
      if (dxi)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) dxi[(e * nq + l) * 9 + a * 3 + b] = inv[a][b];
      if (jac) jac[e * nq + l] = t.refw[l] * (mode == 2 ? fabs(det) : det);
    }
  }
}

}  // namespace

int generic_launch(const GenTables& t, const GenReq& r, void* stream) {
  if (r.Epad == 0) return 0;
  const int nq = t.nq, nm = t.nm;
  int smem = 0;
  switch (r.op) {
    case GEN_BWD: smem = nm; break;
    case GEN_IPROD: smem = nq; break;
    case GEN_MASS: smem = nm + nq; break;
    case GEN_HELM: smem = nm + 4 * nq; break;
    case GEN_PDERIV: smem = nq; break;
    case GEN_IPDERIV: smem = 3 * nq; break;
    default: return (int)cudaErrorInvalidValue;
  }
  smem *= (int)sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int gy = (r.op == GEN_PDERIV || r.op == GEN_IPDERIV) ? 1 : (r.ncomp > 0 ? r.ncomp : 1);
  k_gen<<<dim3((unsigned)r.Epad, (unsigned)gy), kGenThreads, smem, static_cast<cudaStream_t>(stream)>>>(t, r);
  return (int)cudaGetLastError();
}

int generic_geometry(const GenTables& t, int mode, long long E, const double* src, double* dxi, double* jac,
                     unsigned long long* bad, void* stream) {
  if (E == 0) return 0;
  const int smem = 3 * t.nq * (int)sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_gen_geom, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const long long g = E < 148LL * 32 ? E : 148LL * 32;
  k_gen_geom<<<(unsigned)g, kGenThreads, smem, static_cast<cudaStream_t>(stream)>>>(t, mode, E, src, dxi, jac, bad);
  return (int)cudaGetLastError();
}

}  // namespace sk

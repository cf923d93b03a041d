// Assembled C0 variant on a conforming, axis-aligned hex mesh (SURVEY §8f
// rank 2): global <-> element-local maps for the modal basis.
//
// Mesh nx x ny x nz, element e = (ez*ny + ey)*nx + ex.  Along each axis the
// modal index p of element ex maps to the 1D C0 DOF ex*P + (0, P, p-1 for
// p = 0, 1, >= 2): vertex modes psi_0 / psi_1 are shared with the
// neighbours, bubbles are private.  A rank owns the element slab
// ez in [z0, z0 + nzl) and the DOF layers gz in [z0*P, (z0+nzl)*P]; the two
// end layers are shared with the neighbouring ranks (summed by the caller's
// NCCL exchange).  Both kernels are deterministic: the scatter is a gather
// over the <= 8 element contributions of each DOF (no atomics).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/sk200.h"

namespace sk {
void count_launch();
}

namespace {

__device__ __forceinline__ int mode_dof(int e, int p, int P) { return e * P + (p == 0 ? 0 : p == 1 ? P : p - 1); }

__device__ __forceinline__ long long lane_idx(long long e, int n, int N, int W) {
  const long long g = e / W;
  return (g * N + n) * (long long)W + (e - g * W);
}

__global__ void k_c0_gather(int P, int nx, int ny, long long nzl, const double* __restrict__ x, int W,
                            double* __restrict__ local) {
  const int P1 = P + 1, NM = P1 * P1 * P1;
  const long long Nx = (long long)nx * P + 1, Ny = (long long)ny * P + 1;
  const long long E = (long long)nx * ny * nzl;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < E * NM; t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / NM;
    const int m = (int)(t - e * NM);
    const int r = m % P1, q = (m / P1) % P1, p = m / (P1 * P1);
    const int ex = (int)(e % nx);
    const int ey = (int)((e / nx) % ny);
    const long long ez = e / ((long long)nx * ny);  // slab-relative
    const long long g = ((long long)mode_dof((int)ez, r, P) * Ny + mode_dof(ey, q, P)) * Nx + mode_dof(ex, p, P);
    local[lane_idx(e, m, NM, W)] = x[g];
  }
}

// 32-bit form of dof_owners for per-axis indices (< 2^31): the runtime
// divisions by P are 32-bit
__device__ __forceinline__ int dof_owners32(int g, int P, int ne, int* el, int* md) {
  int n = 0;
  const int e = g / P;
  const int o = g - e * P;
  if (o == 0) {
    if (e >= 1) {
      el[n] = e - 1;
      md[n++] = 1;
    }
    if (e < ne) {
      el[n] = e;
      md[n++] = 0;
    }
  } else {
    el[n] = e;
    md[n++] = o + 1;
  }
  return n;
}

// contributions of 1D DOF g: (element, mode) pairs, at most two
__device__ __forceinline__ int dof_owners(long long g, int P, long long ne, long long* el, int* md) {
  int n = 0;
  const long long e = g / P;
  const int o = (int)(g - e * P);
  if (o == 0) {
    if (e >= 1) {
      el[n] = e - 1;
      md[n++] = 1;
    }
    if (e < ne) {
      el[n] = e;
      md[n++] = 0;
    }
  } else {
    el[n] = e;
    md[n++] = o + 1;
  }
  return n;
}

__global__ void k_c0_scatter(int P, int nx, int ny, long long nzl, const double* __restrict__ local, int W,
                             double* __restrict__ y) {
  const int P1 = P + 1, NM = P1 * P1 * P1;
  const long long Nx = (long long)nx * P + 1, Ny = (long long)ny * P + 1, Nz = nzl * P + 1;
  const long long N = Nx * Ny * Nz;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N; g += (long long)gridDim.x * blockDim.x) {
    const long long gx = g % Nx, gy = (g / Nx) % Ny, gz = g / (Nx * Ny);
    long long ex[2], ey[2], ez[2];
    int px[2], py[2], pz[2];
    const int nxo = dof_owners(gx, P, nx, ex, px);
    const int nyo = dof_owners(gy, P, ny, ey, py);
    const int nzo = dof_owners(gz, P, nzl, ez, pz);
    double s = 0.0;
    for (int c = 0; c < nzo; ++c)
      for (int b = 0; b < nyo; ++b)
        for (int a = 0; a < nxo; ++a) {
          const long long e = (ez[c] * ny + ey[b]) * nx + ex[a];
          const int m = (px[a] * P1 + py[b]) * P1 + pz[c];
          s += local[lane_idx(e, m, NM, W)];
        }
    y[g] = s;
  }
}

// The same scatter over 32 x 32 (gx, gz) tiles of one gy plane: a warp reads
// a run of 32 consecutive gz -- contiguous modes r of an element column in
// the element-major local array -- and the sums leave through a transposed
// shared-memory tile as 32 consecutive gx, so both the local reads and the
// y writes are coalesced (the one-DOF-per-thread form reads local with the
// (P+1)^2 stride of the x modes).  Same summation order per DOF.
__global__ void __launch_bounds__(256) k_c0_scatter_t(int P, int nx, int ny, long long nzl,
                                                     const double* __restrict__ local, double* __restrict__ y) {
  __shared__ double tile[32][33];
  const int P1 = P + 1, NM = P1 * P1 * P1;
  const long long Nx = (long long)nx * P + 1, Ny = (long long)ny * P + 1, Nz = nzl * P + 1;
  const int gx0 = blockIdx.x * 32, gz0 = blockIdx.z * 32;
  const int gy = blockIdx.y;
  const int lane = threadIdx.x, warp = threadIdx.y;
  int ey[2], ez[2];
  int py[2], pz[2];
  const int nyo = dof_owners32(gy, P, ny, ey, py);
  const int gz = gz0 + lane;
  const int nzo = gz < Nz ? dof_owners32(gz, P, (int)nzl, ez, pz) : 0;
  for (int i = 0; i < 4; ++i) {
    const int gx = gx0 + warp + 8 * i;
    if (gx >= Nx || gz >= Nz) continue;
    int ex[2];
    int px[2];
    const int nxo = dof_owners32(gx, P, nx, ex, px);
    double s = 0.0;
    for (int c = 0; c < nzo; ++c)
      for (int b = 0; b < nyo; ++b)
        for (int a = 0; a < nxo; ++a) {
          const long long e = ((long long)ez[c] * ny + ey[b]) * nx + ex[a];
          const int m = (px[a] * P1 + py[b]) * P1 + pz[c];
          s += local[e * NM + m];  // interleave width 1: element-major
        }
    tile[warp + 8 * i][lane] = s;
  }
  __syncthreads();
  for (int i = 0; i < 4; ++i) {
    const long long gzw = gz0 + warp + 8 * i, gx = gx0 + lane;
    if (gx < Nx && gzw < Nz) y[(gzw * Ny + gy) * Nx + gx] = tile[lane][warp + 8 * i];
  }
}

// ---- generic signed maps (any shape): gather through l2g / sign, scatter as
// a gather over each global dof's CSR list of (element, mode) contributions
__global__ void k_c0_gather_map(long long E, int nm, const long long* __restrict__ l2g,
                                const double* __restrict__ sgn, const double* __restrict__ x, int W,
                                double* __restrict__ local) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < E * nm; t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / nm;
    const int m = (int)(t - e * nm);
    local[lane_idx(e, m, nm, W)] = sgn[t] * __ldg(x + l2g[t]);
  }
}

__global__ void k_c0_scatter_map(long long n, int nm, const long long* __restrict__ ptr,
                                 const long long* __restrict__ loc, const double* __restrict__ sgn,
                                 const double* __restrict__ local, int W, double* __restrict__ y) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long k = ptr[g]; k < ptr[g + 1]; ++k) {
      const long long t = loc[k], e = t / nm;
      s = fma(sgn[k], local[lane_idx(e, (int)(t - e * nm), nm, W)], s);
    }
    y[g] = s;
  }
}

// Compact maps: one int32 per entry, (index << 1) | (sign < 0), index < 2^30
// -- a third of the map bytes of the int64 index + double sign form; the
// signs are +-1, so negating is bitwise the same as multiplying by them
// (interleave width 1 -- the meshes' only layout -- indexes local by the map
// entry itself, t = e * nm + m; other widths pay the lane arithmetic)
__global__ void k_c0_gather_map32(long long E, int nm, const int* __restrict__ l2gs, const double* __restrict__ x,
                                  int W, double* __restrict__ local) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < E * nm; t += (long long)gridDim.x * blockDim.x) {
    const int v = __ldg(l2gs + t);
    const double xv = __ldg(x + (v >> 1));
    long long idx = t;
    if (W != 1) {
      const long long e = t / nm;
      idx = lane_idx(e, (int)(t - e * nm), nm, W);
    }
    local[idx] = (v & 1) ? -xv : xv;
  }
}

__global__ void k_c0_scatter_map32(long long n, int nm, const int* __restrict__ ptr, const int* __restrict__ locs,
                                   const double* __restrict__ local, int W, double* __restrict__ y) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = __ldg(ptr + g), k1 = __ldg(ptr + g + 1); k < k1; ++k) {
      const int v = __ldg(locs + k);
      const int t = v >> 1;
      long long idx = t;
      if (W != 1) {
        const int e = t / nm;
        idx = lane_idx(e, t - e * nm, nm, W);
      }
      s = fma((v & 1) ? -1.0 : 1.0, local[idx], s);
    }
    y[g] = s;
  }
}

unsigned grid_for(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148LL * 32) g = 148LL * 32;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int sk_c0_gather(int order, int nx, int ny, int64_t nz_local, const double* x, int W, double* local, void* stream) {
  if (order < 1 || order > 10 || nx < 1 || ny < 1 || nz_local < 0 || W < 1) return SK_ERR_ARG;
  if (nz_local == 0) return SK_OK;
  if (!x || !local) return SK_ERR_ARG;
  const long long E = (long long)nx * ny * nz_local;
  const long long NM = (long long)(order + 1) * (order + 1) * (order + 1);
  sk::count_launch();
  k_c0_gather<<<grid_for(E * NM), 256, 0, static_cast<cudaStream_t>(stream)>>>(order, nx, ny, nz_local, x, W, local);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_c0_scatter(int order, int nx, int ny, int64_t nz_local, const double* local, int W, double* y, void* stream) {
  if (order < 1 || order > 10 || nx < 1 || ny < 1 || nz_local < 0 || W < 1) return SK_ERR_ARG;
  if (nz_local == 0) return SK_OK;
  if (!y || !local) return SK_ERR_ARG;
  const long long Nx = (long long)nx * order + 1, Ny = (long long)ny * order + 1, Nz = nz_local * order + 1;
  const long long N = Nx * Ny * Nz;
  sk::count_launch();
  static const bool tiled = [] {
    const char* e = std::getenv("SK_C0_SCATTER_TILED");
    return !(e && e[0] == '0');
  }();
  if (tiled && W == 1 && Ny <= 65535 && (Nz + 31) / 32 <= 65535 && Nx < (1LL << 31) && Nz < (1LL << 31)) {
    const dim3 grid((unsigned)((Nx + 31) / 32), (unsigned)Ny, (unsigned)((Nz + 31) / 32));
    k_c0_scatter_t<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(order, nx, ny, nz_local, local, y);
  } else {
    k_c0_scatter<<<grid_for(N), 256, 0, static_cast<cudaStream_t>(stream)>>>(order, nx, ny, nz_local, local, W, y);
  }
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_c0_gather_map(int64_t E, int n_modes, const int64_t* l2g, const double* sgn, const double* x, int W,
                     double* local, void* stream) {
  if (E < 0 || n_modes < 1 || W < 1) return SK_ERR_ARG;
  if (E == 0) return SK_OK;
  if (!l2g || !sgn || !x || !local) return SK_ERR_ARG;
  sk::count_launch();
  k_c0_gather_map<<<grid_for(E * n_modes), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      E, n_modes, reinterpret_cast<const long long*>(l2g), sgn, x, W, local);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_c0_scatter_map(int64_t n_dofs, int n_modes, const int64_t* ptr, const int64_t* loc, const double* sgn,
                      const double* local, int W, double* y, void* stream) {
  if (n_dofs < 0 || n_modes < 1 || W < 1) return SK_ERR_ARG;
  if (n_dofs == 0) return SK_OK;
  if (!ptr || !loc || !sgn || !local || !y) return SK_ERR_ARG;
  sk::count_launch();
  k_c0_scatter_map<<<grid_for(n_dofs), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n_dofs, n_modes, reinterpret_cast<const long long*>(ptr), reinterpret_cast<const long long*>(loc), sgn, local, W,
      y);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_c0_gather_map32(int64_t E, int n_modes, const int32_t* l2gs, const double* x, int W, double* local,
                       void* stream) {
  if (E < 0 || n_modes < 1 || W < 1 || E * (int64_t)n_modes >= (int64_t(1) << 31)) return SK_ERR_ARG;
  if (E == 0) return SK_OK;
  if (!l2gs || !x || !local) return SK_ERR_ARG;
  sk::count_launch();
  k_c0_gather_map32<<<grid_for(E * n_modes), 256, 0, static_cast<cudaStream_t>(stream)>>>(E, n_modes, l2gs, x, W,
                                                                                          local);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

int sk_c0_scatter_map32(int64_t n_dofs, int n_modes, const int32_t* ptr, const int32_t* locs, const double* local,
                        int W, double* y, void* stream) {
  if (n_dofs < 0 || n_modes < 1 || W < 1 || n_dofs >= (int64_t(1) << 30)) return SK_ERR_ARG;
  if (n_dofs == 0) return SK_OK;
  if (!ptr || !locs || !local || !y) return SK_ERR_ARG;
  sk::count_launch();
  k_c0_scatter_map32<<<grid_for(n_dofs), 256, 0, static_cast<cudaStream_t>(stream)>>>(n_dofs, n_modes, ptr, locs, local,
                                                                                      W, y);
  return cudaGetLastError() == cudaSuccess ? SK_OK : SK_ERR_CUDA;
}

}  // extern "C"

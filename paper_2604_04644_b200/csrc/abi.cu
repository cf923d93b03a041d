// C ABI (include/sk200.h): argument checking, basis handles and dispatch to
// the per-(shape, order) instantiations.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/sk200.h"
#include "sk_tune.h"
#include "generic.hpp"
#include "sk_opset.hpp"

namespace sk {

namespace {
template <int S>
const OpSet* by_order(int P) {
  switch (P) {
    case 1: return opset_impl<S, 1>();
    case 2: return opset_impl<S, 2>();
    case 3: return opset_impl<S, 3>();
    case 4: return opset_impl<S, 4>();
    case 5: return opset_impl<S, 5>();
    case 6: return opset_impl<S, 6>();
    case 7: return opset_impl<S, 7>();
    case 8: return opset_impl<S, 8>();
    case 9: return opset_impl<S, 9>();
    case 10: return opset_impl<S, 10>();
  }
  return nullptr;
}
}  // namespace

const OpSet* opset(int s, int P) {
  switch (s) {
    case HEX: return by_order<0>(P);
    case PRISM: return by_order<1>(P);
    case PYR: return by_order<2>(P);
    case TET: return by_order<3>(P);
  }
  return nullptr;
}

}  // namespace sk

struct sk_basis {
  int shape_ref = 0;  // reference enum index
  sk::HostBasis hb;
  const sk::OpSet* ops = nullptr;
  std::vector<unsigned char> fwd_vals, fwd_ders, dtab;
  std::vector<double> gtab_host;
  // device copies of gtab, one per device, created on first use
  std::mutex mu;
  std::vector<double*> gtab_dev;
  // DMMA StdMat mass fragments (sk_dense.cuh), one per device, built on
  // first use from the dense B the bwd_trans kernel produces
  std::mutex dmu;
  std::vector<double*> dense_dev;
  // quadrature override (qpoints): no specialised kernels, the run-time-size
  // path of generic.cu on device copies of the dense tables
  bool generic = false;
  std::mutex gmu;
  std::vector<double*> gen_dev;
};

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_status(int e, const char* what) {
  if (e == 0) return SK_OK;
  return fail(SK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(e)));
}

const double* device_gtab(sk_basis* b, int* status) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *status = cuda_status(e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(b->mu);
  if ((int)b->gtab_dev.size() <= dev) b->gtab_dev.resize(dev + 1, nullptr);
  if (!b->gtab_dev[dev]) {
    double* p = nullptr;
    e = cudaMalloc(&p, sizeof(double) * b->gtab_host.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(p, b->gtab_host.data(), sizeof(double) * b->gtab_host.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      *status = cuda_status(e, "device table upload");
      return nullptr;
    }
    b->gtab_dev[dev] = p;
  }
  *status = SK_OK;
  return b->gtab_dev[dev];
}

int run(sk_basis* b, int op, int geo, long long E, int W, int ncomp, const double* in, double* out,
        const double* pay, double lam, long long in_n, long long out_n, void* stream, const double* dense = nullptr);

// Dense basis matrix B[q][m] (= bwd_trans of the unit coefficient vectors,
// so it is the sum-factorised kernel's own B) -> DMMA fragment tables on
// this device (built once, cached on the basis).
const double* device_dense(sk_basis* b, void* stream, int* status) {
  *status = SK_OK;
  const int nd = b->ops->dense_doubles;
  if (nd <= 0) {
    *status = fail(SK_ERR_UNSUPPORTED, "no dense mass kernel for this order");
    return nullptr;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *status = cuda_status(e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(b->dmu);
  if ((int)b->dense_dev.size() <= dev) b->dense_dev.resize(dev + 1, nullptr);
  if (b->dense_dev[dev]) return b->dense_dev[dev];
  const int nm = b->hb.nm, nq = b->hb.nq;
  std::vector<double> eye((size_t)nm * nm, 0.0), bt((size_t)nm * nq), B((size_t)nq * nm), frag((size_t)nd);
  for (int m = 0; m < nm; ++m) eye[(size_t)m * nm + m] = 1.0;
  double *d_in = nullptr, *d_out = nullptr, *d_frag = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  e = cudaMalloc(&d_in, sizeof(double) * eye.size());
  if (e == cudaSuccess) e = cudaMalloc(&d_out, sizeof(double) * bt.size());
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, s);
  int st = SK_OK;
  if (e == cudaSuccess) st = run(b, sk::OP_BWD, 0, nm, 1, 1, d_in, d_out, nullptr, 0.0, nm, nq, stream);
  if (e == cudaSuccess && st == SK_OK)
    e = cudaMemcpyAsync(bt.data(), d_out, sizeof(double) * bt.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && st == SK_OK) e = cudaStreamSynchronize(s);
  cudaFree(d_in);
  cudaFree(d_out);
  if (st != SK_OK || e != cudaSuccess) {
    *status = st != SK_OK ? st : cuda_status(e, "dense basis matrix");
    return nullptr;
  }
  for (int m = 0; m < nm; ++m)
    for (int q = 0; q < nq; ++q) B[(size_t)q * nm + m] = bt[(size_t)m * nq + q];
  b->ops->fill_dense(b->hb, B.data(), frag.data());
  e = cudaMalloc(&d_frag, sizeof(double) * frag.size());
  if (e == cudaSuccess) e = cudaMemcpy(d_frag, frag.data(), sizeof(double) * frag.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d_frag);
    *status = cuda_status(e, "dense fragment upload");
    return nullptr;
  }
  b->dense_dev[dev] = d_frag;
  return d_frag;
}

// StdMat (DMMA) or sum factorisation for the regular collocated Helmholtz:
// the tuned table, overridden by SK_HELM_DENSE=0/1
bool use_dense_helm(const sk_basis* b, int geo) {
  if (b->generic || geo != SK_GEO_REGULAR || b->ops->dense_doubles <= 0 || !(b->ops->dense_mask & 4)) return false;
  if (const char* v = std::getenv("SK_HELM_DENSE")) {
    if (v[0] == '0') return false;
    if (v[0] == '1') return true;
  }
  return sk::kDenseHelm[b->hb.shape][b->hb.P];
}

// StdMat (DMMA) or sum-factorised mass for this basis and geometry class:
// the tuned table, overridden by SK_MASS_DENSE=0/1
bool use_dense_mass(const sk_basis* b, int geo) {
  if (b->generic || b->ops->dense_doubles <= 0 || !(b->ops->dense_mask & (geo == SK_GEO_DEFORMED ? 2 : 1)))
    return false;
  if (const char* v = std::getenv("SK_MASS_DENSE")) {
    if (v[0] == '0') return false;
    if (v[0] == '1') return true;
  }
  return sk::kDenseMass[geo == SK_GEO_DEFORMED ? 1 : 0][b->hb.shape][b->hb.P];
}

// device tables of a quadrature-override basis: one buffer per device
// [B | DB0 | DB1 | DB2 | D0 | D1 | D2 | G | refw | z0 | z1 | z2]
int generic_tables(sk_basis* b, sk::GenTables* t) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  const sk::HostBasis& hb = b->hb;
  const size_t nqm = (size_t)hb.nq * hb.nm;
  const size_t sizes[12] = {nqm, nqm, nqm, nqm, hb.D[0].size(), hb.D[1].size(), hb.D[2].size(),
                            hb.G.size(), hb.refw.size(), hb.z[0].size(), hb.z[1].size(), hb.z[2].size()};
  const double* src[12] = {hb.Bd.data(), hb.DBd[0].data(), hb.DBd[1].data(), hb.DBd[2].data(), hb.D[0].data(),
                           hb.D[1].data(), hb.D[2].data(), hb.G.data(), hb.refw.data(), hb.z[0].data(),
                           hb.z[1].data(), hb.z[2].data()};
  size_t off[13] = {0};
  for (int i = 0; i < 12; ++i) off[i + 1] = off[i] + sizes[i];
  {
    std::lock_guard<std::mutex> lk(b->gmu);
    if ((int)b->gen_dev.size() <= dev) b->gen_dev.resize(dev + 1, nullptr);
    if (!b->gen_dev[dev]) {
      double* p = nullptr;
      e = cudaMalloc(&p, sizeof(double) * off[12]);
      for (int i = 0; i < 12 && e == cudaSuccess; ++i)
        e = cudaMemcpy(p + off[i], src[i], sizeof(double) * sizes[i], cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_status(e, "generic table upload");
      }
      b->gen_dev[dev] = p;
    }
  }
  const double* p = b->gen_dev[dev];
  t->B = p + off[0];
  t->DB0 = p + off[1];
  t->DB1 = p + off[2];
  t->DB2 = p + off[3];
  t->D0 = p + off[4];
  t->D1 = p + off[5];
  t->D2 = p + off[6];
  t->G = p + off[7];
  t->refw = p + off[8];
  t->z0 = p + off[9];
  t->z1 = p + off[10];
  t->z2 = p + off[11];
  for (int d = 0; d < 3; ++d) t->Q[d] = hb.Q[d];
  t->nq = hb.nq;
  t->nm = hb.nm;
  t->shape = hb.shape;
  return SK_OK;
}

int generic_op(int op) {
  switch (op) {
    case sk::OP_BWD: return sk::GEN_BWD;
    case sk::OP_IPROD: return sk::GEN_IPROD;
    case sk::OP_MASS: return sk::GEN_MASS;
    case sk::OP_HELM:
    case sk::OP_HELM_NC: return sk::GEN_HELM;
    case sk::OP_PDERIV: return sk::GEN_PDERIV;
    case sk::OP_IPDERIV: return sk::GEN_IPDERIV;
  }
  return -1;
}

int check_layout(long long E, int W, int ncomp) {
  if (E < 0) return fail(SK_ERR_ARG, "element count must be nonnegative");
  if (W < 1) return fail(SK_ERR_ARG, "interleave width must be at least 1");
  if (ncomp < 1) return fail(SK_ERR_ARG, "need at least one component");
  return SK_OK;
}

long long padded(long long E, int W) { return ((E + W - 1) / W) * (long long)W; }

int run(sk_basis* b, int op, int geo, long long E, int W, int ncomp, const double* in, double* out,
        const double* pay, double lam, long long in_n, long long out_n, void* stream, const double* dense) {
  int st = SK_OK;
  if (b->generic) {
    sk::GenTables t;
    if ((st = generic_tables(b, &t))) return st;
    sk::GenReq r;
    r.op = generic_op(op);
    if (r.op < 0) return fail(SK_ERR_UNSUPPORTED, "operator not on the quadrature-override path");
    r.geo = geo;
    r.E = E;
    r.Epad = padded(E, W);
    r.in_cs = r.Epad * in_n;
    r.out_cs = r.Epad * out_n;
    r.W = W;
    r.ncomp = ncomp;
    r.in = in;
    r.out = out;
    r.pay = pay;
    r.lam = lam;
    if (r.Epad == 0) return SK_OK;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_status(sk::generic_launch(t, r, stream), "generic kernel launch");
  }
  const double* g = device_gtab(b, &st);
  if (st) return st;
  sk::LaunchReq r;
  r.fwd = b->fwd_vals.data();
  r.fwd_d = b->fwd_ders.data();
  r.dtab = b->dtab.data();
  r.in = in;
  r.out = out;
  r.pay = pay;
  r.gtab = g;
  r.E = E;
  r.Epad = padded(E, W);
  r.in_cs = r.Epad * in_n;
  r.out_cs = r.Epad * out_n;
  r.W = W;
  r.ncomp = ncomp;
  r.geo = geo;
  r.lam = lam;
  r.dense = dense;
  if (r.Epad == 0) return SK_OK;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(b->ops->launch(op, r, stream), "kernel launch");
}

}  // namespace

extern "C" {

int sk_basis_create(int shape, int order, sk_basis** out) {
  if (!out) return fail(SK_ERR_ARG, "null output handle");
  *out = nullptr;
  if (shape < SK_SHAPE_QUAD || shape > SK_SHAPE_TET) return fail(SK_ERR_STATE, "unknown shape id");
  if (shape < SK_SHAPE_HEX) return fail(SK_ERR_UNSUPPORTED, "2D shapes are not on the device path");
  if (order < 1) return fail(SK_ERR_ARG, "polynomial order must be at least 1");
  const int s = shape - SK_SHAPE_HEX;
  const sk::OpSet* ops = sk::opset(s, order);
  if (!ops) return fail(SK_ERR_UNSUPPORTED, "order outside the compiled range 1..10");
  std::unique_ptr<sk_basis> b(new sk_basis());
  b->shape_ref = shape;
  try {
    if (!sk::build_host_basis(s, order, b->hb)) return fail(SK_ERR_UNSUPPORTED, "unsupported (shape, order)");
  } catch (const std::exception& ex) {
    return fail(SK_ERR_ARG, ex.what());
  }
  b->ops = ops;
  b->fwd_vals.resize(ops->fwd_bytes);
  b->fwd_ders.resize(ops->fwd_bytes);
  b->dtab.resize(ops->dtab_bytes);
  ops->fill(b->hb, b->fwd_vals.data(), b->fwd_ders.data(), b->dtab.data());
  b->gtab_host.resize(ops->gtab_doubles);
  ops->fill_gtab(b->hb, b->gtab_host.data());
  *out = b.release();
  return SK_OK;
}

int sk_basis_create_q(int shape, int order, const int qpoints[3], sk_basis** out) {
  if (!out) return fail(SK_ERR_ARG, "null output handle");
  *out = nullptr;
  if (!qpoints) return sk_basis_create(shape, order, out);
  if (shape < SK_SHAPE_QUAD || shape > SK_SHAPE_TET) return fail(SK_ERR_STATE, "unknown shape id");
  if (shape < SK_SHAPE_HEX) return fail(SK_ERR_UNSUPPORTED, "2D shapes are not on the device path");
  if (order < 1 || order > 10) return fail(SK_ERR_UNSUPPORTED, "order outside the compiled range 1..10");
  const int s = shape - SK_SHAPE_HEX;
  sk::HostBasis probe;
  if (!sk::build_host_basis(s, order, probe)) return fail(SK_ERR_UNSUPPORTED, "unsupported (shape, order)");
  bool dflt = true;
  for (int d = 0; d < 3; ++d) {
    if (qpoints[d] < probe.Q[d]) return fail(SK_ERR_ARG, "quadrature override below the default point count");
    if (qpoints[d] > 64) return fail(SK_ERR_UNSUPPORTED, "quadrature override above 64 points per direction");
    dflt = dflt && qpoints[d] == probe.Q[d];
  }
  if (dflt) return sk_basis_create(shape, order, out);
  std::unique_ptr<sk_basis> b(new sk_basis());
  b->shape_ref = shape;
  try {
    if (!sk::build_host_basis(s, order, b->hb, qpoints)) return fail(SK_ERR_ARG, "bad quadrature override");
  } catch (const std::exception& ex) {
    return fail(SK_ERR_ARG, ex.what());
  }
  b->generic = true;
  *out = b.release();
  return SK_OK;
}

int sk_basis_destroy(sk_basis* b) {
  if (!b) return SK_OK;
  for (double* p : b->gtab_dev)
    if (p) cudaFree(p);
  for (double* p : b->dense_dev)
    if (p) cudaFree(p);
  for (double* p : b->gen_dev)
    if (p) cudaFree(p);
  delete b;
  return SK_OK;
}

int sk_basis_counts(const sk_basis* b, int64_t out[6]) {
  if (!b || !out) return fail(SK_ERR_ARG, "null argument");
  out[0] = b->hb.Q[0];
  out[1] = b->hb.Q[1];
  out[2] = b->hb.Q[2];
  out[3] = b->hb.nq;
  out[4] = b->hb.nm;
  out[5] = b->hb.P;
  return SK_OK;
}

int sk_basis_table(const sk_basis* b, const char* name, double* out, int64_t cap, int64_t* len) {
  if (!b || !name || !len) return fail(SK_ERR_ARG, "null argument");
  auto it = b->hb.named.find(name);
  if (it == b->hb.named.end()) {
    *len = 0;
    return SK_OK;
  }
  *len = (int64_t)it->second.size();
  if (out) std::memcpy(out, it->second.data(), sizeof(double) * std::min<int64_t>(cap, *len));
  return SK_OK;
}

int sk_payload_size(const sk_basis* b, int geo_class, int kind, int64_t E, int64_t* n) {
  if (!b || !n) return fail(SK_ERR_ARG, "null argument");
  if (geo_class != SK_GEO_REGULAR && geo_class != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (kind < 0 || kind > 3) return fail(SK_ERR_ARG, "bad payload kind");
  if (E < 0) return fail(SK_ERR_ARG, "element count must be nonnegative");
  if (b->generic) {  // the factors themselves: dxi (9 per point / element) and w|J|
    *n = 10 * E * (geo_class == SK_GEO_DEFORMED ? (int64_t)b->hb.nq : 1);
    return SK_OK;
  }
  *n = b->ops->payload_doubles(kind, geo_class) * b->ops->payload_elements(kind, E);
  return SK_OK;
}

int sk_payload_pack(const sk_basis* b, int geo_class, int kind, int64_t E, const double* dxi, const double* jac,
                    double* pay, void* stream) {
  if (!b || (E > 0 && (!dxi || !jac || !pay))) return fail(SK_ERR_ARG, "null argument");
  if (geo_class != SK_GEO_REGULAR && geo_class != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (kind < 0 || kind > 3 || E < 0) return fail(SK_ERR_ARG, "bad payload kind or element count");
  if (b->generic) {
    const size_t nd = (size_t)E * (geo_class == SK_GEO_DEFORMED ? b->hb.nq : 1);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(pay, dxi, sizeof(double) * 9 * nd, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pay + 9 * nd, jac, sizeof(double) * nd, cudaMemcpyDeviceToDevice, s);
    return cuda_status(e, "payload copy");
  }
  int st = SK_OK;
  const double* g = device_gtab(const_cast<sk_basis*>(b), &st);
  if (st) return st;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(b->ops->pack(kind, geo_class, E, dxi, jac, pay, g, stream), "payload pack");
}

static int geometry_common(const sk_basis* b, int mode, int64_t E, const double* src, double* dxi, double* jac,
                           int kind, double* pay, int64_t* n_bad, void* stream) {
  if (!b || (E > 0 && !src)) return fail(SK_ERR_ARG, "null argument");
  if (E < 0) return fail(SK_ERR_ARG, "element count must be nonnegative");
  int st = SK_OK;
  sk::GenTables gt;
  const double* g = nullptr;
  if (b->generic) {
    if ((st = generic_tables(const_cast<sk_basis*>(b), &gt))) return st;
    if (kind >= 0) {  // a payload is the factors: dxi then w|J|
      dxi = pay;
      jac = pay + (size_t)9 * E * b->hb.nq;
    }
  } else {
    g = device_gtab(const_cast<sk_basis*>(b), &st);
  }
  if (st) return st;
  unsigned long long* d_bad = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMallocAsync(&d_bad, sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_status(e, "geometry scratch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  int r = b->generic ? sk::generic_geometry(gt, mode, E, src, dxi, jac, d_bad, stream)
                     : b->ops->geometry(mode, E, src, dxi, jac, kind, pay, d_bad, g, stream);
  if (r) {
    cudaFreeAsync(d_bad, s);
    return cuda_status(r, "geometry kernel");
  }
  unsigned long long h_bad = 0;
  e = cudaMemcpyAsync(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d_bad, s);
  if (e != cudaSuccess) return cuda_status(e, "geometry readback");
  if (n_bad) *n_bad = (int64_t)h_bad;
  return SK_OK;
}

int sk_geometry_deformed(const sk_basis* b, int64_t E, const double* params, double* dxi, double* jac,
                         int64_t* n_bad, void* stream) {
  return geometry_common(b, 1, E, params, dxi, jac, -1, nullptr, n_bad, stream);
}

int sk_geometry_from_coords(const sk_basis* b, int64_t E, const double* coords, double* dxi, double* jac,
                            int64_t* n_bad, void* stream) {
  return geometry_common(b, 0, E, coords, dxi, jac, -1, nullptr, n_bad, stream);
}

int sk_geometry_from_coords_oriented(const sk_basis* b, int64_t E, const double* coords, double* dxi, double* jac,
                                     int64_t* n_bad, void* stream) {
  return geometry_common(b, 2, E, coords, dxi, jac, -1, nullptr, n_bad, stream);
}

int sk_payload_from_params(const sk_basis* b, int kind, int64_t E, const double* params, double* pay,
                           int64_t* n_bad, void* stream) {
  if (kind < 0 || kind > 3) return fail(SK_ERR_ARG, "bad payload kind");
  if (E > 0 && !pay) return fail(SK_ERR_ARG, "null payload");
  return geometry_common(b, 1, E, params, nullptr, nullptr, kind, pay, n_bad, stream);
}

int sk_bwd_trans(const sk_basis* b, int64_t E, int W, int ncomp, const double* uhat, double* u, void* stream) {
  if (!b || (E > 0 && (!uhat || !u))) return fail(SK_ERR_ARG, "null argument");
  if (int st = check_layout(E, W, ncomp)) return st;
  return run(const_cast<sk_basis*>(b), sk::OP_BWD, 0, E, W, ncomp, uhat, u, nullptr, 0.0, b->hb.nm, b->hb.nq,
             stream);
}

int sk_iproduct_wrt_base(const sk_basis* b, int geo, int64_t E, int W, int ncomp, const double* u,
                         const double* wpay, double* fhat, void* stream) {
  if (!b || (E > 0 && (!u || !wpay || !fhat))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (int st = check_layout(E, W, ncomp)) return st;
  return run(const_cast<sk_basis*>(b), sk::OP_IPROD, geo, E, W, ncomp, u, fhat, wpay, 0.0, b->hb.nq, b->hb.nm,
             stream);
}

int sk_phys_deriv(const sk_basis* b, int geo, int64_t E, int W, const double* u, const double* dpay, double* du,
                  void* stream) {
  if (!b || (E > 0 && (!u || !dpay || !du))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (int st = check_layout(E, W, 1)) return st;
  return run(const_cast<sk_basis*>(b), sk::OP_PDERIV, geo, E, W, 1, u, du, dpay, 0.0, b->hb.nq, b->hb.nq, stream);
}

int sk_iproduct_wrt_deriv_base(const sk_basis* b, int geo, int64_t E, int W, const double* v, const double* wpay,
                               double* fhat, void* stream) {
  if (!b || (E > 0 && (!v || !wpay || !fhat))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (int st = check_layout(E, W, 1)) return st;
  return run(const_cast<sk_basis*>(b), sk::OP_IPDERIV, geo, E, W, 1, v, fhat, wpay, 0.0, b->hb.nq, b->hb.nm,
             stream);
}

int sk_mass_apply(const sk_basis* b, int geo, int64_t E, int W, int ncomp, const double* uhat, const double* wpay,
                  double* out, void* stream) {
  if (!b || (E > 0 && (!uhat || !wpay || !out))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (int st = check_layout(E, W, ncomp)) return st;
  sk_basis* bb = const_cast<sk_basis*>(b);
  const double* dense = nullptr;
  if (E > 0 && use_dense_mass(bb, geo)) {
    int st = SK_OK;
    dense = device_dense(bb, stream, &st);
    if (st) return st;
  }
  return run(bb, sk::OP_MASS, geo, E, W, ncomp, uhat, out, wpay, 0.0, b->hb.nm, b->hb.nm, stream, dense);
}

int sk_helmholtz_apply(const sk_basis* b, int geo, int form, int64_t E, int W, int ncomp, const double* uhat,
                       const double* hpay, double lam, double* out, void* stream) {
  if (!b || (E > 0 && (!uhat || !hpay || !out))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (!(lam >= 0.0)) return fail(SK_ERR_ARG, "reaction coefficient must be nonnegative");
  if (form != SK_FORM_COLL && form != SK_FORM_NONCOLL) return fail(SK_ERR_ARG, "unknown Helmholtz form");
  if (int st = check_layout(E, W, ncomp)) return st;
  sk_basis* bb = const_cast<sk_basis*>(b);
  const double* dense = nullptr;
  if (E > 0 && form == SK_FORM_COLL && use_dense_helm(bb, geo)) {
    int st = SK_OK;
    dense = device_dense(bb, stream, &st);
    if (st) return st;
  }
  return run(bb, form == SK_FORM_NONCOLL ? sk::OP_HELM_NC : sk::OP_HELM, geo, E, W, ncomp, uhat, out, hpay, lam,
             b->hb.nm, b->hb.nm, stream, dense);
}

int sk_helmholtz_apply_staged(const sk_basis* b, int geo, int64_t E, int W, int ncomp, const double* uhat,
                              const double* hpay, double lam, double* out, double* work, int64_t chunk,
                              void* stream) {
  if (!b || (E > 0 && (!uhat || !hpay || !out || !work))) return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_DEFORMED) return fail(SK_ERR_UNSUPPORTED, "the staged variant is built for deformed geometry");
  if (b->generic) return fail(SK_ERR_UNSUPPORTED, "the staged variant needs the default quadrature");
  if (!(lam >= 0.0)) return fail(SK_ERR_ARG, "reaction coefficient must be nonnegative");
  if (int st = check_layout(E, W, ncomp)) return st;
  // chunks start on a multiple of the interleave width and of 16 (tile and
  // payload lane widths divide 16)
  long long unit = 16;
  while (unit % W) unit += 16;
  if (chunk < unit || chunk % unit) return fail(SK_ERR_ARG, "chunk must be a positive multiple of lcm(16, W)");
  const long long Epad = padded(E, W);
  if (Epad == 0) return SK_OK;
  int st = SK_OK;
  sk_basis* bb = const_cast<sk_basis*>(b);
  const double* g = device_gtab(bb, &st);
  if (st) return st;
  const long long nm = b->hb.nm, nq = b->hb.nq, per_el = b->ops->payload_doubles(SK_PAYLOAD_HELMHOLTZ, geo);
  double* w0 = work;
  double* w1 = work + chunk * nq;
  sk::LaunchReq r;
  r.fwd = b->fwd_vals.data();
  r.fwd_d = b->fwd_ders.data();
  r.dtab = b->dtab.data();
  r.gtab = g;
  r.W = W;
  r.ncomp = 1;
  r.geo = geo;
  r.lam = lam;
  for (int c = 0; c < ncomp; ++c) {
    for (long long e0 = 0; e0 < Epad; e0 += chunk) {
      const long long e1 = std::min<long long>(Epad, e0 + chunk);
      r.E = std::max<long long>(0, std::min<long long>(E, e1) - e0);
      r.Epad = e1 - e0;
      // BwdTrans -> u
      r.in = uhat + c * Epad * nm + e0 * nm;
      r.out = w0;
      r.pay = nullptr;
      r.in_cs = r.Epad * nm;
      r.out_cs = r.Epad * nq;
      g_launches.fetch_add(3, std::memory_order_relaxed);
      int e = b->ops->launch(sk::OP_BWD, r, stream);
      // quadrature-point Helmholtz -> u'
      r.in = w0;
      r.out = w1;
      r.pay = hpay + e0 * per_el;  // chunks start on a payload lane group
      r.in_cs = r.out_cs = r.Epad * nq;
      if (e == 0) e = b->ops->launch(sk::OP_QP, r, stream);
      // B^T -> out
      r.in = w1;
      r.out = out + c * Epad * nm + e0 * nm;
      r.pay = nullptr;
      r.in_cs = r.Epad * nq;
      r.out_cs = r.Epad * nm;
      if (e == 0) e = b->ops->launch(sk::OP_BT, r, stream);
      if (e) return cuda_status(e, "staged kernel launch");
    }
  }
  return SK_OK;
}

int sk_helmholtz_apply_params(const sk_basis* b, int64_t E, int W, int ncomp, const double* uhat,
                              const double* params, double lam, double* out, double* work, int64_t chunk,
                              int64_t* n_bad, void* stream) {
  if (!b || (E > 0 && (!uhat || !params || !out || !work))) return fail(SK_ERR_ARG, "null argument");
  if (b->generic) return fail(SK_ERR_UNSUPPORTED, "the recomputed-metric variant needs the default quadrature");
  if (!(lam >= 0.0)) return fail(SK_ERR_ARG, "reaction coefficient must be nonnegative");
  if (int st = check_layout(E, W, ncomp)) return st;
  long long unit = 16;
  while (unit % W) unit += 16;
  if (chunk < unit || chunk % unit) return fail(SK_ERR_ARG, "chunk must be a positive multiple of lcm(16, W)");
  if (n_bad) *n_bad = 0;
  const long long Epad = padded(E, W);
  if (Epad == 0) return SK_OK;
  int st = SK_OK;
  sk_basis* bb = const_cast<sk_basis*>(b);
  const double* g = device_gtab(bb, &st);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* d_bad = nullptr;
  cudaError_t ce = cudaMallocAsync(&d_bad, sizeof(unsigned long long), s);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
  if (ce != cudaSuccess) return cuda_status(ce, "geometry scratch");
  const long long nm = b->hb.nm;
  int r = 0;
  for (long long e0 = 0; e0 < Epad && r == 0; e0 += chunk) {
    const long long e1 = std::min<long long>(Epad, e0 + chunk);
    const long long ne = std::max<long long>(0, std::min<long long>(E, e1) - e0);
    // metric payload of this chunk from its 12 deformation parameters per
    // element: into the L2-resident work buffer (chunks start on a payload
    // lane group, so the chunk's payload is the work buffer's prefix)
    g_launches.fetch_add(1, std::memory_order_relaxed);
    r = b->ops->geometry(1, ne, params + e0 * 12, nullptr, nullptr, SK_PAYLOAD_HELMHOLTZ, work, d_bad, g, stream);
    if (r) {
      r = cuda_status(r, "geometry kernel");
      break;
    }
    for (int c = 0; c < ncomp && r == 0; ++c)
      r = run(bb, sk::OP_HELM, SK_GEO_DEFORMED, ne, W, 1, uhat + c * Epad * nm + e0 * nm, out + c * Epad * nm + e0 * nm,
              work, lam, nm, nm, stream, nullptr);
  }
  unsigned long long h_bad = 0;
  if (r == 0 && n_bad) {
    ce = cudaMemcpyAsync(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) r = cuda_status(ce, "geometry check");
    *n_bad = (int64_t)h_bad;
  }
  cudaFreeAsync(d_bad, s);
  return r;
}

namespace {
long long gcd_ll(long long a, long long b) { return b ? gcd_ll(b, a % b) : a; }

// per-thread copy streams of the streamed applies (one pair per device)
struct CopyStreams {
  int dev = -1;
  cudaStream_t h2d = nullptr, d2h = nullptr;
};
thread_local CopyStreams g_cs;

int copy_streams(cudaStream_t* h2d, cudaStream_t* d2h) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (g_cs.dev != dev) {
    // streams of another device are simply abandoned (device switches are rare)
    g_cs = CopyStreams();
    e = cudaStreamCreateWithFlags(&g_cs.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&g_cs.d2h, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e, "copy stream creation");
    g_cs.dev = dev;
  }
  *h2d = g_cs.h2d;
  *d2h = g_cs.d2h;
  return SK_OK;
}
}  // namespace

int sk_apply_streamed(const sk_basis* b, int op, int geo, int64_t E, int W, int ncomp, const double* host_in,
                      double* dev_in, const double* pay, double lam, double* dev_out, double* host_out,
                      int64_t chunk, void* stream) {
  return sk_apply_streamed_ex(b, op, geo, E, W, ncomp, host_in, dev_in, pay, lam, dev_out, host_out, chunk, 0, stream);
}

int sk_apply_streamed_ex(const sk_basis* b, int op, int geo, int64_t E, int W, int ncomp, const double* host_in,
                         double* dev_in, const double* pay, double lam, double* dev_out, double* host_out,
                         int64_t chunk, int flags, void* stream) {
  if (flags & ~SK_STREAM_DIRECT_OUT) return fail(SK_ERR_ARG, "unknown streamed-apply flag");
  // direct output: the kernels store the result straight into the (mapped)
  // pinned host buffer; no device copy of the output, no D2H stage
  double* hout_dev = nullptr;
  if ((flags & SK_STREAM_DIRECT_OUT) && host_out) {
    void* p = nullptr;
    if (cudaHostGetDevicePointer(&p, host_out, 0) != cudaSuccess) {
      cudaGetLastError();
      return fail(SK_ERR_ARG, "direct output needs mapped pinned host memory");
    }
    hout_dev = static_cast<double*>(p);
  }
  const bool direct = hout_dev != nullptr;
  if (!b || (E > 0 && (!host_in || !dev_in || !pay || (!dev_out && !direct) || !host_out)))
    return fail(SK_ERR_ARG, "null argument");
  if (geo != SK_GEO_REGULAR && geo != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  if (op != SK_STREAM_HELMHOLTZ && op != SK_STREAM_HELMHOLTZ_NC && op != SK_STREAM_MASS)
    return fail(SK_ERR_ARG, "unknown streamed operator");
  if (b->generic) return fail(SK_ERR_UNSUPPORTED, "streamed applies need the default quadrature");
  if (op != SK_STREAM_MASS && !(lam >= 0.0)) return fail(SK_ERR_ARG, "reaction coefficient must be nonnegative");
  if (int st = check_layout(E, W, ncomp)) return st;
  const int kop = op == SK_STREAM_MASS ? sk::OP_MASS : op == SK_STREAM_HELMHOLTZ_NC ? sk::OP_HELM_NC : sk::OP_HELM;
  const int kind = op == SK_STREAM_MASS ? SK_PAYLOAD_W : op == SK_STREAM_HELMHOLTZ_NC ? SK_PAYLOAD_HELMHOLTZ_NC
                                                                                     : SK_PAYLOAD_HELMHOLTZ;
  const long long Epad = padded(E, W);
  if (Epad == 0) return SK_OK;
  int st = SK_OK;
  const double* g = device_gtab(const_cast<sk_basis*>(b), &st);
  if (st) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream), sh = nullptr, sd = nullptr;
  if ((st = copy_streams(&sh, &sd))) return st;
  // chunks start on a multiple of the interleave width, the tile widths and
  // the payload lane widths (all powers of two <= 16, kRegPW = 16), so every
  // chunk is a sub-block
  const long long eb = 16;
  const long long unit = (long long)W / gcd_ll(W, eb) * eb;
  // chunk boundaries.  Default: ~Epad/8 chunks with a geometric ramp at both
  // ends (1/8, 1/4, 1/2 of a chunk), so the exposed first H2D and last
  // kernel + D2H are short while the count of chunks -- each costs a fixed
  // overhead on the copy engines (measured, tools/e2e_chunks.py) -- stays low.
  // chunk > 0: uniform chunks of that many elements.
  std::vector<long long> bnd{0};
  auto round_up = [&](long long n) { return std::max(unit, (n + unit - 1) / unit * unit); };
  const char* ramp_env = std::getenv("SK_STREAM_RAMP");
  const bool ramp = chunk <= 0 && !(ramp_env && ramp_env[0] == '0');
  if (chunk <= 0) chunk = ramp ? (Epad + 7) / 8 : (Epad + 15) / 16;
  if (chunk < 4096) chunk = 4096;
  chunk = round_up(chunk);
  if (ramp && Epad >= 4 * chunk) {
    const long long head[3] = {round_up(chunk / 8), round_up(chunk / 4), round_up(chunk / 2)};
    long long rem = Epad;
    for (long long h : head) {
      bnd.push_back(bnd.back() + h);
      rem -= h;
    }
    const long long tail = head[0] + head[1] + head[2];
    while (rem - tail > 0) {
      const long long c = std::min<long long>(chunk, round_up(rem - tail));
      bnd.push_back(std::min<long long>(Epad, bnd.back() + c));
      rem = Epad - bnd.back();
    }
    for (int t = 2; t >= 0 && bnd.back() < Epad; --t) bnd.push_back(std::min<long long>(Epad, bnd.back() + head[t]));
    if (bnd.back() < Epad) bnd.push_back(Epad);
  } else {
    for (long long e0 = chunk; e0 < Epad; e0 += chunk) bnd.push_back(e0);
    bnd.push_back(Epad);
  }
  const long long nm = b->hb.nm, cs = Epad * nm, per_el = b->ops->payload_doubles(kind, geo);
  const int nchunk = (int)bnd.size() - 1;
  std::vector<cudaEvent_t> ev(2 * nchunk + 2, nullptr);
  cudaError_t e = cudaSuccess;
  for (auto& x : ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  auto cleanup = [&] {
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);  // deferred by the runtime until the event completes
  };
  if (e != cudaSuccess) {
    cleanup();
    return cuda_status(e, "event creation");
  }
  // copies start after earlier work on the caller's stream (e.g. writers of dev_in)
  e = cudaEventRecord(ev[2 * nchunk], s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sh, ev[2 * nchunk], 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev[2 * nchunk], 0);
  sk::LaunchReq r;
  r.fwd = b->fwd_vals.data();
  r.fwd_d = b->fwd_ders.data();
  r.dtab = b->dtab.data();
  r.gtab = g;
  r.in_cs = cs;
  r.out_cs = cs;
  r.W = W;
  r.ncomp = ncomp;
  r.geo = geo;
  r.lam = op == SK_STREAM_MASS ? 0.0 : lam;
  if ((kop == sk::OP_MASS && use_dense_mass(b, geo)) || (kop == sk::OP_HELM && use_dense_helm(b, geo))) {
    r.dense = device_dense(const_cast<sk_basis*>(b), stream, &st);
    if (st) {
      cleanup();
      return st;
    }
  }
  for (int i = 0; i < nchunk && e == cudaSuccess; ++i) {
    const long long e0 = bnd[i], e1 = bnd[i + 1];
    const size_t bytes = sizeof(double) * (size_t)((e1 - e0) * nm);
    for (int c = 0; c < ncomp && e == cudaSuccess; ++c)
      e = cudaMemcpyAsync(dev_in + c * cs + e0 * nm, host_in + c * cs + e0 * nm, bytes, cudaMemcpyHostToDevice, sh);
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * i], sh);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[2 * i], 0);
    if (e != cudaSuccess) break;
    r.in = dev_in + e0 * nm;
    r.out = (direct ? hout_dev : dev_out) + e0 * nm;
    r.pay = pay + e0 * per_el;  // chunks start on a payload lane group
    r.E = std::max<long long>(0, std::min<long long>(E, e1) - e0);
    r.Epad = e1 - e0;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    e = static_cast<cudaError_t>(b->ops->launch(kop, r, stream));
    if (direct) continue;
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * i + 1], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, ev[2 * i + 1], 0);
    for (int c = 0; c < ncomp && e == cudaSuccess; ++c)
      e = cudaMemcpyAsync(host_out + c * cs + e0 * nm, dev_out + c * cs + e0 * nm, bytes, cudaMemcpyDeviceToHost, sd);
  }
  // the caller's stream resumes once every chunk is back on the host
  // (direct output: once the last kernel on it has stored its chunk)
  if (!direct) {
    if (e == cudaSuccess) e = cudaEventRecord(ev[2 * nchunk + 1], sd);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[2 * nchunk + 1], 0);
  }
  cleanup();
  return cuda_status(e, "streamed apply");
}

int sk_helmholtz_apply_c0_mapped(const sk_basis* b, int geo, int64_t E, const int32_t* l2gs, const double* x,
                                 const double* hpay, double lam, double* out, void* stream) {
  if (b && b->generic) return fail(SK_ERR_UNSUPPORTED, "the C0 variant needs the default quadrature");
  if (!b || E < 0) return fail(SK_ERR_ARG, "bad C0 mesh");
  if (b->ops->S == sk::HEX) return fail(SK_ERR_UNSUPPORTED, "mapped C0 gather: prism / pyramid / tet bases");
  if (geo != SK_GEO_DEFORMED) return fail(SK_ERR_UNSUPPORTED, "fused C0 gather: deformed geometry");
  if (!(lam >= 0.0)) return fail(SK_ERR_ARG, "reaction coefficient must be nonnegative");
  if (E * (int64_t)b->hb.nm >= (int64_t(1) << 31)) return fail(SK_ERR_ARG, "compact map index range exceeded");
  if (E > 0 && (!l2gs || !x || !hpay || !out)) return fail(SK_ERR_ARG, "null argument");
  if (E == 0) return SK_OK;
  int st = SK_OK;
  const double* g = device_gtab(const_cast<sk_basis*>(b), &st);
  if (st) return st;
  sk::LaunchReq r;
  r.fwd = b->fwd_vals.data();
  r.fwd_d = b->fwd_ders.data();
  r.dtab = b->dtab.data();
  r.in = x;
  r.out = out;
  r.pay = hpay;
  r.gtab = g;
  r.E = E;
  r.Epad = E;
  r.in_cs = 0;
  r.out_cs = E * b->hb.nm;
  r.W = 1;
  r.ncomp = 1;
  r.geo = geo;
  r.lam = lam;
  r.c0map = l2gs;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(b->ops->launch(sk::OP_HELM, r, stream), "mapped C0 kernel launch");
}

int sk_helmholtz_apply_c0(const sk_basis* b, int geo, int nx, int ny, int64_t nz_local, const double* x,
                          const double* hpay, double lam, double* out, void* stream) {
  return sk_helmholtz_apply_c0_w(b, geo, nx, ny, nz_local, x, hpay, lam, out, 1, stream);
}

int sk_helmholtz_apply_c0_w(const sk_basis* b, int geo, int nx, int ny, int64_t nz_local, const double* x,
                            const double* hpay, double lam, double* out, int64_t out_W, void* stream) {
  if (b && b->generic) return fail(SK_ERR_UNSUPPORTED, "the C0 variant needs the default quadrature");
  if (!b || nx < 1 || ny < 1 || nz_local < 0) return fail(SK_ERR_ARG, "bad C0 slab");
  if (b->ops->S != sk::HEX) return fail(SK_ERR_UNSUPPORTED, "assembled C0 variant is hex only");
  if (geo != SK_GEO_DEFORMED || !(lam > 0.0)) return fail(SK_ERR_UNSUPPORTED, "fused C0 gather: deformed, lam > 0");
  const long long E = (long long)nx * ny * nz_local;
  if (E > 0 && (!x || !hpay || !out)) return fail(SK_ERR_ARG, "null argument");
  if (E == 0) return SK_OK;
  if (out_W < 1 || out_W > E || E % out_W || out_W > 0x7fffffff) return fail(SK_ERR_ARG, "output lane width must divide the element count");
  int st = SK_OK;
  const double* g = device_gtab(const_cast<sk_basis*>(b), &st);
  if (st) return st;
  sk::LaunchReq r;
  r.fwd = b->fwd_vals.data();
  r.fwd_d = b->fwd_ders.data();
  r.dtab = b->dtab.data();
  r.in = x;
  r.out = out;
  r.pay = hpay;
  r.gtab = g;
  r.E = E;
  r.Epad = E;
  r.in_cs = 0;
  r.out_cs = E * b->hb.nm;
  r.W = (int)out_W;  // output layout (the input is the global DOF vector)
  r.ncomp = 1;
  r.geo = geo;
  r.lam = lam;
  r.c0_nx = nx;
  r.c0_ny = ny;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(b->ops->launch(sk::OP_HELM, r, stream), "kernel launch");
}

int64_t sk_launch_count(void) { return g_launches.load(); }

}  // extern "C"

namespace sk {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace sk

extern "C" {

const char* sk_last_error(void) { return g_err.c_str(); }

// ---- device memory helpers: a caller binding only this library (no CUDA
// runtime bindings of its own) can hold the MemoryRegion DEVICE space
int sk_device_alloc(int64_t bytes, void** ptr) {
  if (!ptr || bytes < 0) return fail(SK_ERR_ARG, "bad argument");
  *ptr = nullptr;
  if (bytes == 0) return SK_OK;
  return cuda_status(cudaMalloc(ptr, (size_t)bytes), "cudaMalloc");
}

int sk_device_free(void* ptr) { return ptr ? cuda_status(cudaFree(ptr), "cudaFree") : SK_OK; }

int sk_copy_h2d(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(SK_ERR_ARG, "bad argument");
  if (bytes == 0) return SK_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
                     "cudaMemcpyAsync H2D");
}

int sk_copy_d2h(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(SK_ERR_ARG, "bad argument");
  if (bytes == 0) return SK_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
                     "cudaMemcpyAsync D2H");
}

int sk_stream_synchronize(void* stream) {
  return cuda_status(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
}

int sk_launch_config(const sk_basis* b, int op, int64_t out[3]) {
  return sk_launch_config_geo(b, op, SK_GEO_DEFORMED, out);
}

int sk_launch_config_geo(const sk_basis* b, int op, int geo_class, int64_t out[3]) {
  if (!b || !out || op < 0 || op >= sk::OP_COUNT) return fail(SK_ERR_ARG, "bad argument");
  if (b->generic) {  // generic.cu: one element per 128-thread CTA
    out[0] = 1;
    out[1] = 128;
    out[2] = 8 * (b->hb.nm + 4 * (int64_t)b->hb.nq);
    return SK_OK;
  }
  if (geo_class != SK_GEO_REGULAR && geo_class != SK_GEO_DEFORMED) return fail(SK_ERR_ARG, "bad geometry class");
  b->ops->config(op, geo_class, out);  // SK_GEO_* == sk::GEO_* (0 regular, 1 deformed)
  return SK_OK;
}

}  // extern "C"

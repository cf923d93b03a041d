/*
 * sk200.h -- C ABI of the B200-native matrix-free spectral/hp operator path.
 *
 * This is the drop-in boundary for the reference's per-block operator API
 * (speckern/operators.py:551-776).  Every entry point below replaces one
 * reference function; the reference file:line is cited beside it.  There
 * are no torch (or any C++) types in these signatures: plain pointers,
 * sizes and a cudaStream_t passed as void*.
 *
 * Conventions
 *  - All field/payload pointers are DEVICE pointers owned by the caller.
 *  - Fields use the reference's lane-major block layout
 *    (speckern/field_block.py:205-214): for component c, element e and data
 *    point n the double lives at ((c*G + e/W)*N + n)*W + e%W, with
 *    W = interleave width, G = ceil(E/W) groups, N = n_modes or n_points.
 *    W = 1 is plain element-major.  Padded lanes (e >= E) are written as 0.
 *  - Mode order is lexicographic (p,q,r) with p slowest (shapes.py:142-179);
 *    point order is l = (i*Q1 + j)*Q2 + k (shapes.py:482-487).
 *  - Geometry enters as the reference's GeometricFactors
 *    (geometry.py:94-116) and is packed once per block into a device
 *    payload by sk_payload_pack (replaces Block.payload,
 *    field_block.py:309-363); applies then stream the packed payload.
 *  - Every call is stream-ordered and re-entrant.  The only shared state is
 *    the immutable per-(shape, order) basis handle.
 *  - Status: 0 ok; 1 bad state/shape; 2 unsupported (shape, order);
 *    3 bad argument (lam < 0, E < 0, null pointer, W < 1);
 *    4 CUDA error (see sk_last_error()).
 */
#ifndef SK200_H
#define SK200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* shape ids = index in the reference's Shape enum (shapes.py:57-65) */
enum { SK_SHAPE_QUAD = 0, SK_SHAPE_TRI = 1, SK_SHAPE_HEX = 2,
       SK_SHAPE_PRISM = 3, SK_SHAPE_PYR = 4, SK_SHAPE_TET = 5 };
/* GeometryClass (geometry.py:35-39) */
enum { SK_GEO_REGULAR = 0, SK_GEO_DEFORMED = 1 };
/* payload kinds: what Block.payload(...) feeds each operator family */
enum { SK_PAYLOAD_HELMHOLTZ = 0,      /* lam + wj ("lam","wj"/"jac" keys), collocated form */
       SK_PAYLOAD_W = 1,              /* W diagonal ("wj" / "jac" keys)                    */
       SK_PAYLOAD_DERIV = 2,          /* inverse Jacobian ("dxi" key)                      */
       SK_PAYLOAD_HELMHOLTZ_NC = 3 }; /* lam + wj, point order of the non-collocated form  */
/* Helmholtz formulations (operators.py:702-721) */
enum { SK_FORM_COLL = 0, SK_FORM_NONCOLL = 1 };
enum { SK_OK = 0, SK_ERR_STATE = 1, SK_ERR_UNSUPPORTED = 2, SK_ERR_ARG = 3, SK_ERR_CUDA = 4 };

typedef struct sk_basis sk_basis;

/* ---- basis / constant tables -------------------------------------------
 * Replaces build_shape_basis (shapes.py:521-541) + SumFacTables
 * (shapes.py:444-456, 555-583): 1D rules (bases.py:235-270), modified
 * bases (bases.py:277-354), collocation matrices (bases.py:468-477) and
 * Duffy chain-rule factors (shapes.py:265-323), built natively in FP64.
 * Host-only; device copies are made lazily per device on first use. */
int sk_basis_create(int shape, int order, sk_basis** out);
/* Same with a per-direction quadrature override (shapes.py:521-541: each
 * count >= the default P+2 Gauss-Lobatto / P+1 Gauss-Radau-Jacobi, <= 64):
 * the default counts give the specialised kernels; any other override runs
 * every operator on the run-time-size dense path (generic.cu), whose
 * geometry payload is the factors themselves (dxi and w|J|). */
int sk_basis_create_q(int shape, int order, const int qpoints[3], sk_basis** out);
int sk_basis_destroy(sk_basis* b);
/* counts: out[0..5] = Q0, Q1, Q2, n_points, n_modes, order */
int sk_basis_counts(const sk_basis* b, int64_t out[6]);
/* Read back a named host table (for tests and the host API): "z0".."z2",
 * "w0".."w2", "D0".."D2", "a0".."a2", "da0".."da2", "b1_<p>", "db1_<p>",
 * "c2_<p>", "dc2_<p>", "refw", "G", "modes".  Writes up to cap doubles,
 * returns the table length via *len (0 when absent). */
int sk_basis_table(const sk_basis* b, const char* name, double* out, int64_t cap, int64_t* len);

/* ---- geometry -------------------------------------------------------------
 * Payload size in doubles for E elements. */
int sk_payload_size(const sk_basis* b, int geo_class, int kind, int64_t E, int64_t* n_doubles);
/* Pack GeometricFactors (device, reference layout: dxi_dx (E,NQ,3,3) or
 * (E,3,3); jac (E,NQ) or (E,)) into the kernel payload of `kind`.
 * Replaces Block._build_payload (field_block.py:331-363). */
int sk_payload_pack(const sk_basis* b, int geo_class, int kind, int64_t E,
                    const double* dxi_dx, const double* jac, double* payload, void* stream);
/* Device geometry builder (replaces make_synthetic_factors for DEFORMED,
 * geometry.py:275-315 -> 161-212): per-element deformation parameters
 * params[E][12] = amp[3], phase[3], perm[3] (as doubles), shift[3] ->
 * dxi_dx (E,NQ,3,3) and jac = w|J| (E,NQ).  *n_bad receives the number of
 * points with |J| <= 0 (DegenerateElementError, geometry.py:203-209). */
int sk_geometry_deformed(const sk_basis* b, int64_t E, const double* params,
                         double* dxi_dx, double* jac, int64_t* n_bad, void* stream);
/* Device geometry builder straight into a kernel payload of `kind`
 * (no dxi/jac materialised): the large-mesh path of the bench (H7). */
int sk_payload_from_params(const sk_basis* b, int kind, int64_t E, const double* params,
                           double* payload, int64_t* n_bad, void* stream);
/* Iso-parametric factors from coordinates coords (E,NQ,3) (geometry.py:161-212). */
int sk_geometry_from_coords(const sk_basis* b, int64_t E, const double* coords,
                            double* dxi_dx, double* jac, int64_t* n_bad, void* stream);
/* Same for elements of either orientation: jac = w|det J| (*n_bad counts
 * det J == 0 only).  Used by the assembled C0 tet mesh, whose tets take
 * their vertices in global-id order so that shared faces and edges are
 * parameterised alike on both sides (half of them are reflected). */
int sk_geometry_from_coords_oriented(const sk_basis* b, int64_t E, const double* coords,
                                     double* dxi_dx, double* jac, int64_t* n_bad, void* stream);

/* ---- operators (SUM_FAC_TOP: one CTA per element tile) -------------------- */
/* bwd_trans (operators.py:551-561): coeff -> phys, per component */
int sk_bwd_trans(const sk_basis* b, int64_t E, int W, int ncomp,
                 const double* uhat, double* u, void* stream);
/* iproduct_wrt_base (operators.py:564-574): phys -> coeff; payload kind W */
int sk_iproduct_wrt_base(const sk_basis* b, int geo_class, int64_t E, int W, int ncomp,
                         const double* u, const double* wpay, double* fhat, void* stream);
/* phys_deriv (operators.py:577-596): 1 phys component -> 3; payload kind DERIV */
int sk_phys_deriv(const sk_basis* b, int geo_class, int64_t E, int W,
                  const double* u, const double* dpay, double* du, void* stream);
/* iproduct_wrt_deriv_base (operators.py:599-619): 3 phys components -> 1 coeff; payload kind W */
int sk_iproduct_wrt_deriv_base(const sk_basis* b, int geo_class, int64_t E, int W,
                               const double* v, const double* wpay, double* fhat, void* stream);
/* mass_apply (operators.py:622-633); payload kind W */
int sk_mass_apply(const sk_basis* b, int geo_class, int64_t E, int W, int ncomp,
                  const double* uhat, const double* wpay, double* out, void* stream);
/* helmholtz_apply[_coll|_noncoll] (operators.py:636-721); payload kind
 * HELMHOLTZ for SK_FORM_COLL, HELMHOLTZ_NC for SK_FORM_NONCOLL.  lam == 0 is
 * the stiffness operator and skips the W stream. */
int sk_helmholtz_apply(const sk_basis* b, int geo_class, int form, int64_t E, int W, int ncomp,
                       const double* uhat, const double* hpay, double lam, double* out, void* stream);

/* Staged collocated Helmholtz (deformed geometry): the fused kernel split
 * into BwdTrans -> quadrature-point kernel (collocation sweeps, metric,
 * transposed sweeps, lam W u) -> unweighted B^T, run over element chunks so
 * the two NQ-sized intermediates stay L2-resident.  Same payload and
 * results as sk_helmholtz_apply(SK_FORM_COLL); the fused-vs-staged choice per
 * (shape, order) is made from measurements.  work: device
 * buffer of 2 * chunk * n_points doubles; chunk: elements per chunk, a
 * positive multiple of lcm(16, W). */
int sk_helmholtz_apply_staged(const sk_basis* b, int geo_class, int64_t E, int W, int ncomp, const double* uhat,
                              const double* hpay, double lam, double* out, double* work, int64_t chunk,
                              void* stream);

/* Collocated Helmholtz on deformed elements with the metric recomputed on the
 * device instead of streamed (SURVEY H3 option (c)): per element chunk, the
 * geometry kernel builds the chunk's HELMHOLTZ payload from the 12
 * deformation parameters per element (as sk_payload_from_params,
 * geometry.py:275-300 -> 161-212) into `work`, then the fused Helmholtz kernel
 * consumes it while it is L2-resident.  HBM traffic per element 8(2 NP + 12)
 * bytes instead of 8(2 NP + 7 NQ); results identical to
 * sk_payload_from_params + sk_helmholtz_apply(SK_FORM_COLL).  work: device
 * buffer of the payload size of `chunk` elements (sk_payload_size);
 * chunk: positive multiple of lcm(16, W).  n_bad (optional; NULL skips the
 * check and its stream synchronisation) receives the number of points with
 * det J <= 0 (geometry.py:203-209). */
int sk_helmholtz_apply_params(const sk_basis* b, int64_t E, int W, int ncomp, const double* uhat,
                              const double* params, double lam, double* out, double* work, int64_t chunk,
                              int64_t* n_bad, void* stream);

/* ---- host-buffer applies with transfer/compute overlap ----------------------
 * The reference's callers hold their blocks in host memory (field_block.py:
 * 67-149 MemoryRegion HOST space).  sk_apply_streamed runs a coefficient ->
 * coefficient operator on host input and returns host output, pipelined over
 * element chunks: H2D of chunk i+1, the kernel on chunk i and D2H of chunk
 * i-1 run concurrently (two internal copy streams + the caller's stream).
 * host_in/host_out should be pinned (page-locked) for the copies to overlap;
 * dev_in/dev_out are the caller's device buffers of the full block (both
 * hold the block afterwards), pay is the device payload of the operator.
 * Stream-ordered: host_out is complete when `stream` reaches this point.
 * op: SK_STREAM_HELMHOLTZ (payload HELMHOLTZ, lam >= 0), SK_STREAM_HELMHOLTZ_NC
 * (payload HELMHOLTZ_NC), SK_STREAM_MASS (payload W, lam ignored).
 * chunk_elements <= 0 picks a default (~16 chunks). */
enum { SK_STREAM_HELMHOLTZ = 0, SK_STREAM_HELMHOLTZ_NC = 1, SK_STREAM_MASS = 2 };
int sk_apply_streamed(const sk_basis* b, int op, int geo_class, int64_t E, int W, int ncomp,
                      const double* host_in, double* dev_in, const double* pay, double lam, double* dev_out,
                      double* host_out, int64_t chunk_elements, void* stream);
/* Same with flags.  SK_STREAM_DIRECT_OUT: the kernels store each chunk's
 * result straight into host_out (pinned, mapped: the PCIe writes overlap the
 * next chunks' H2D copies and kernels, no D2H stage); dev_out is not written
 * and may be NULL.  Fails with SK_ERR_ARG when host_out is not mapped. */
enum { SK_STREAM_DIRECT_OUT = 1 };
int sk_apply_streamed_ex(const sk_basis* b, int op, int geo_class, int64_t E, int W, int ncomp,
                         const double* host_in, double* dev_in, const double* pay, double lam, double* dev_out,
                         double* host_out, int64_t chunk_elements, int flags, void* stream);

/* ---- assembled C0 variant (hex, conforming, axis-aligned) --------
 * No reference counterpart (global assembly is outside speckern, SPEC.md:8,
 * 452).  Mesh nx x ny x nz_local element slab, e = (ez*ny + ey)*nx + ex; the
 * slab's DOF vector covers gz in [0, nz_local*order] with
 * g = (gz*(ny*order+1) + gy)*(nx*order+1) + gx.  gather: local(e, mode) =
 * x[l2g(e, mode)] in the lane-major field layout of width W; scatter:
 * y[g] = sum of the <= 8 element contributions (deterministic, no atomics).
 * The end layers gz = 0 and gz = nz_local*order are shared with the
 * neighbouring slabs and summed by the caller (NCCL exchange). */
int sk_c0_gather(int order, int nx, int ny, int64_t nz_local, const double* x, int W, double* local,
                 void* stream);
int sk_c0_scatter(int order, int nx, int ny, int64_t nz_local, const double* local, int W, double* y,
                  void* stream);
/* Elemental Helmholtz of the slab with the gather fused into the kernel's
 * tile load: out (element-major, W = 1) = H_e (A x) without materialising
 * A x.  Deformed geometry, lam > 0, hex bases only. */
int sk_helmholtz_apply_c0(const sk_basis* b, int geo_class, int nx, int ny, int64_t nz_local, const double* x,
                          const double* hpay, double lam, double* out, void* stream);
/* Same with the output in the lane-major layout of width out_W (out_W
 * divides the slab's element count; out_W = E is mode-major [mode][element],
 * which the scatter reads coalesced along x). */
int sk_helmholtz_apply_c0_w(const sk_basis* b, int geo_class, int nx, int ny, int64_t nz_local, const double* x,
                            const double* hpay, double lam, double* out, int64_t out_W, void* stream);
/* Elemental Helmholtz of a mapped C0 mesh (prism / pyramid / tet) with the
 * gather fused into the kernel's tile load: out (element-major, W = 1) =
 * H_e (A x) with A from the compact map l2gs (E x n_modes, as
 * sk_c0_gather_map32).  Deformed geometry, lam >= 0, E * n_modes < 2^31. */
int sk_helmholtz_apply_c0_mapped(const sk_basis* b, int geo_class, int64_t E, const int32_t* l2gs, const double* x,
                                 const double* hpay, double lam, double* out, void* stream);

/* Generic signed assembly maps (any shape; the prism C0 variant): gather
 * local(e, m) = sgn[e*n_modes+m] * x[l2g[e*n_modes+m]] into the lane-major
 * field layout of width W; scatter y[g] = sum over k in [ptr[g], ptr[g+1])
 * of csr_sgn[k] * local(loc[k] / n_modes, loc[k] % n_modes) -- a gather per
 * global DOF (deterministic, no atomics).  All arrays device-resident. */
int sk_c0_gather_map(int64_t E, int n_modes, const int64_t* l2g, const double* sgn, const double* x, int W,
                     double* local, void* stream);
int sk_c0_scatter_map(int64_t n_dofs, int n_modes, const int64_t* ptr, const int64_t* loc, const double* csr_sgn,
                      const double* local, int W, double* y, void* stream);
/* The same maps in compact form: one int32 per entry, (index << 1) | (sign
 * < 0) (signs are +-1), l2gs per (element, mode), ptr (n_dofs + 1 entries)
 * and locs (element * n_modes + mode per contribution) for the scatter;
 * E * n_modes < 2^31, n_dofs < 2^30.  Bitwise the same results as the int64
 * / double forms with a third of their map traffic. */
int sk_c0_gather_map32(int64_t E, int n_modes, const int32_t* l2gs, const double* x, int W, double* local,
                       void* stream);
int sk_c0_scatter_map32(int64_t n_dofs, int n_modes, const int32_t* ptr, const int32_t* locs, const double* local,
                        int W, double* y, void* stream);

/* ---- device memory (for callers without CUDA runtime bindings) --------------
 * The MemoryRegion DEVICE space of a reference Block (field_block.py:67-149)
 * held by a binding that loads only this library (integration/speckern_sk200.py).
 * Copies are stream-ordered (pass NULL for the legacy default stream);
 * sk_stream_synchronize waits for the stream. */
int sk_device_alloc(int64_t bytes, void** ptr);
int sk_device_free(void* ptr);
int sk_copy_h2d(void* dst, const void* src, int64_t bytes, void* stream);
int sk_copy_d2h(void* dst, const void* src, int64_t bytes, void* stream);
int sk_stream_synchronize(void* stream);

/* ---- diagnostics ------------------------------------------------------------ */
/* Number of kernel launches this thread issued through the library. */
int64_t sk_launch_count(void);
/* Last error message of the calling thread ("" when none). */
const char* sk_last_error(void);
/* Kernel launch configuration chosen for an operator: out[0]=elements per
 * CTA, out[1]=threads per CTA, out[2]=dynamic shared bytes. op: 0 helmholtz,
 * 1 mass, 2 bwd, 3 iprod, 4 physderiv, 5 iprod_deriv, 6 helmholtz noncoll. */
int sk_launch_config(const sk_basis* b, int op, int64_t out[3]);
/* Same, for a geometry class (the regular collocated Helmholtz is tuned
 * with its own tile width and thread count); sk_launch_config reports the
 * deformed configuration. */
int sk_launch_config_geo(const sk_basis* b, int op, int geo_class, int64_t out[3]);

#ifdef __cplusplus
}
#endif
#endif /* SK200_H */

/* dgm.h — C ABI of the B200 DG Maxwell operator (arXiv:1104.4208).
 *
 * The library applies, every explicit time step, the energy-conserving DG
 * operator for the loss-free time-domain Maxwell equations
 *     ε ∂E/∂t = curl H,   μ ∂H/∂t = -curl E
 * on an affine tetrahedral mesh, in the semi-discrete form
 *     ∂t diag(Mε, Mμ) (E,H) = [[0, -C_hᵀ],[C_h, 0]] (E,H)
 * with the symplectic-Euler / leapfrog update.
 * Fields are expanded per element in the paper's Dubiner basis φ_ijk
 * under the covariant map E|_T = F_T^{-T} Σ Ê_α φ_α ∘ Φ_T^{-1}
 * (PAPER.md:354, 379-381); the element curl is applied through the sparse
 * difference-differential recurrences, traces by
 * exact restriction to the face Dubiner basis, and
 * the inverse mass is the 3x3-block-diagonal flat-element form.
 * Readings of the paper (flux signs, upwind flux, boundary conditions, orders,
 * orientation) are listed in DESIGN.md §Readings (G1-G15).
 *
 * LAYOUT.  A field (E or H) is a device array double[3][n_tet][ld] (component,
 * element, mode): the covariant reference components Ê_m of element T, mode α
 * in graded order (total degree ascending, then i, then j).  ld = N rounded up
 * to a multiple of 4 (N = (p+1)(p+2)(p+3)/6); modes in [N, ld) are padding: the
 * library never writes them and never reads them into a result.
 *
 * MESH.  xyz [n_vert][3] physical coordinates; tet [n_tet][4] vertex ids whose
 * order must be strictly ascending in rep[] (local vertex v̂0..v̂3 =
 * (0,0,0),(1,0,0),(0,1,0),(0,0,1); det F may be negative).  rep [n_vert] is
 * the periodic representative of each vertex (NULL = identity): faces with the
 * same representative triple are glued (periodic pairs are ordinary interior
 * faces); a face seen once is a PEC boundary (mirror state E⁺=-E⁻, H⁺=H⁻).
 *
 * OWNERSHIP.  dgm_create deep-copies every host array and keeps no caller
 * pointer.  Field and output arrays are caller-owned DEVICE memory unless the
 * function name ends in _host.  The context owns its device tables and scratch
 * and frees them in dgm_destroy.  Work is enqueued on the caller's stream
 * (cudaStream_t passed as void*, NULL = legacy default stream); only
 * dgm_energy, dgm_tables and dgm_step_host synchronise.
 *
 * ERRORS.  Every call returns dgm_status; nothing throws across the ABI.
 * dgm_last_error(ctx) gives a message (element/face ids for mesh errors).
 * A context is not thread-safe; distinct contexts are independent.
 */
#ifndef DGM_H
#define DGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dgm_ctx dgm_ctx;

typedef enum {
  DGM_OK = 0,
  DGM_EINVAL = 1,   /* null pointer, bad size or argument                     */
  DGM_EMESH = 2,    /* non-canonical vertex order, degenerate tet, face shared by >2 tets */
  DGM_EORDER = 3,   /* order outside 1..DGM_PMAX                               */
  DGM_ECUDA = 4,    /* a CUDA call failed (message has cudaGetErrorString)     */
  DGM_ENOMEM = 5    /* allocation failed                                       */
} dgm_status;

#define DGM_PMAX 10

typedef enum {
  DGM_FLUX_CENTRAL = 0,    /* H* = {{H}}, E* = {{E}} */
  DGM_FLUX_UPWIND = 1,     /* Riemann flux, Z = sqrt(μ/ε)               (reading G2)       */
  DGM_FLUX_STABILIZED = 2  /* central flux + face unknowns H^F with face mass (h_F/α):
                              energy-conserving and free of spurious modes
                              (readings G16-G17); use the *_sc calls */
} dgm_flux;

typedef struct {
  int64_t n_vert;
  const double *xyz;    /* [n_vert][3] host                                   */
  int64_t n_tet;
  const int32_t *tet;   /* [n_tet][4] host, ascending by rep[]                */
  const int32_t *rep;   /* [n_vert] host, periodic representative; NULL = id  */
} dgm_mesh;

/* Execution engine of the stage kernels.  All compute the same operator (same
 * flux, traces, lift, update; parity-tested against the oracle); they differ in how
 * the reference-frame operators are applied:
 *   SPARSE: the paper's recurrence sweeps and sum-factorised traces/lifts
 *            as generated straight-line code (p <= 6) or a
 *           streamed-table interpreter (p >= 7);
 *   DENSE:  the same operators assembled once per context into matrices (from the
 *           exact programs) and applied as block-sparse FP64 tensor-core GEMMs over
 *           tiles of elements (mma.sync m8n8k4), 3 launches per stage.
 *   HYBRID: (orders 4..10) the curl by the paper's recurrences as streamed
 *           lane-per-element sweeps on the FP64 pipes, written to an
 *           internal ĉ buffer and added in the epilogue of the DENSE stage GEMM, which
 *           then applies only the lift; traces as in DENSE.  4 launches per stage.
 *   AUTO:   SPARSE for p <= 5, DENSE for p = 6, HYBRID for p >= 7 (measured fastest
 *           there).  Mixed orders use DENSE.
 * The environment variable DGM_ENGINE=sparse|dense|hybrid overrides AUTO.  For measurements,
 * DGM_STAGE_NH / DGM_TRACE_NH = 1|2 force the dense GEMM tile width (one or two 96-column
 * warp columns; default one) and DGM_TILE_ORDER=0 the static GEMM tile order
 * (default: dynamic, from a per-context self-resetting counter, so one context must not run dense GEMMs
 * on two streams at once); results are the same operator. */
typedef enum { DGM_ENGINE_AUTO = 0, DGM_ENGINE_SPARSE = 1, DGM_ENGINE_DENSE = 2, DGM_ENGINE_HYBRID = 3 } dgm_engine_kind;

typedef struct {
  int32_t flux;          /* dgm_flux                                          */
  int32_t eps_per_elem;  /* 0: eps points to one double; 1: to [n_tet]        */
  int32_t mu_per_elem;   /* same for mu                                       */
  double alpha0;         /* DGM_FLUX_STABILIZED: α = alpha0·p² (≤0 → 1)       */
  int32_t engine;        /* dgm_engine_kind                                   */
  int32_t mixed_order;   /* 0: E and H of degree `order`.  1: the paper's spaces
                            E ∈ P^order, H ∈ P^(order-1); needs
                            order >= 2, central or upwind flux, and the dense engine
                            (AUTO resolves to it).  Both fields keep the order-`order`
                            layout; H's modes >= N(order-1) are ignored by the
                            operator and stay zero when zero on input.            */
  int32_t material_points; /* 1: eps and mu point to [n_tet][Q] values at the
                            element's quadrature points (dgm_quadrature_host;
                            physical point x = X0 + F ξ).  The inverse mass is then
                            the paper's "reverse numerical integration" approximate
                            inverse: residual -> values at the
                            points -> × ŵ_i / m(x_i) -> back to the modes.  Central
                            flux, equal orders, dense engine (AUTO resolves to it);
                            dgm_energy and dgm_spectral_radius are not available. */
  const double *edge_nodes; /* NULL: flat (affine) elements.  Else curved elements
                            ("Curved elements"): host
                            [n_tet][6][3] physical coordinates of the edge nodes of a
                            quadratic (10-node) tetrahedron, edges (0,1) (0,2) (0,3)
                            (1,2) (1,3) (2,3) of the tet's local vertex order.  The
                            map Φ(x̂) = Σ_a λ_a(2λ_a-1) X_a + Σ_ab 4 λ_a λ_b X_ab
                            (λ: barycentric coordinates of x̂ on v̂0..v̂3) is
                            non-affine; the curl and face terms stay geometry-free
                            (covariant identities, hold pointwise
                            for any smooth Φ) and the full mass with |det F(x̂)| m
                            F⁻¹F⁻ᵀ(x̂) is replaced by the reverse-numerical-integration
                            approximate inverse: residual -> point values -> × ŵ_i
                            F(x̂_i)ᵀF(x̂_i) / (m(x_i) det F(x̂_i)) (a 3x3 mix per
                            point) -> back to the modes.  Central flux, equal orders,
                            dense engine; m = eps/mu per element or scalar, or at the
                            points (material_points; x_i = Φ(ξ_i)).  sign det F(x̂_i)
                            must be the same at every quadrature point (else
                            DGM_EMESH); dgm_energy and dgm_spectral_radius are not
                            available.  Neighbours must share their face's edge
                            nodes (checked on non-periodic interior faces). */
} dgm_opts;

/* Validate the mesh, match faces, compute per-element geometry
 * G'_T = F_TᵀF_T / det F_T, det F_T, 1/ε_T, 1/μ_T
 * and upload them with the order-p programs.  order in 1..DGM_PMAX.
 * eps, mu: host, one value or [n_tet] (opts); must be > 0.  opts may be NULL
 * (central flux, scalar eps/mu).  On error *out is NULL. */
dgm_status dgm_create(const dgm_mesh *mesh, int order, const double *eps, const double *mu,
                      const dgm_opts *opts, dgm_ctx **out);

/* N (modes per component), ld (leading dimension), n_tet. */
dgm_status dgm_layout(const dgm_ctx *ctx, int64_t *n_modes, int64_t *ld, int64_t *n_tet);

/* Volume part of the time derivatives, after the inverse mass:
 *   dE = Mε^{-1}(curl H, e)_T ,  dH = -Mμ^{-1}(curl E, h)_T     (device arrays, overwritten).
 * Either output may be NULL to skip it. */
dgm_status dgm_apply_curl(dgm_ctx *ctx, const double *E, const double *H, double *dE, double *dH,
                          void *cuda_stream);

/* Face part (numerical flux, traces, lift), after the inverse mass (reading G1):
 *   dE = Mε^{-1}(ν×(H*-H⁻), e)_∂T ,  dH = -Mμ^{-1}(ν×(E*-E⁻), h)_∂T.
 * accumulate != 0 adds into dE/dH instead of overwriting.  NULL output skips. */
dgm_status dgm_apply_flux(dgm_ctx *ctx, const double *E, const double *H, double *dE, double *dH,
                          int accumulate, void *cuda_stream);

/* nsteps of the symplectic-Euler map (reading G7: H staggered)
 *   H ← H + dt Ḣ(E, H);   E ← E + dt Ė(H, E)
 * in place on the device arrays E, H.  Upwind self-terms use the current value
 * of the field being updated.  Calls of >= 64 steps replay a CUDA graph of 32
 * captured steps (same kernels and order, bit-identical; DGM_GRAPHS=0 disables).
 * DGM_EINVAL for a DGM_FLUX_STABILIZED context
 * (its state includes H^F: use dgm_step_sc); the same holds for dgm_step_ex and
 * dgm_step_host.  dgm_apply_flux and dgm_spectral_radius on such a context act
 * with the central flux alone (H^F = 0). */
dgm_status dgm_step(dgm_ctx *ctx, double *E, double *H, double dt, int64_t nsteps, void *cuda_stream);

/* Flags for dgm_step_ex. */
#define DGM_STEP_CONTINUE 1  /* E, H are the arrays of the previous dgm_step/_ex call on this
                                context and were not modified since: reuse the face-trace
                                buffers that call left instead of recomputing them at entry
                                (falls back to recomputing if the pointers differ or another
                                call invalidated the buffers). */

/* dgm_step with flags (0 = identical to dgm_step). */
dgm_status dgm_step_ex(dgm_ctx *ctx, double *E, double *H, double dt, int64_t nsteps, int flags,
                       void *cuda_stream);

/* Same as dgm_step on HOST arrays (layout as above): copies E,H host→device,
 * steps, copies back device→host, synchronises.  The context keeps the device
 * copies between calls.  Host arrays should be pinned for full copy speed. */
dgm_status dgm_step_host(dgm_ctx *ctx, double *E_host, double *H_host, double dt, int64_t nsteps,
                         void *cuda_stream);

/* Discrete energy ½(E,MεE) + ½(H,MμH), deterministic
 * two-pass reduction; writes one double to *out_host and synchronises. */
dgm_status dgm_energy(dgm_ctx *ctx, const double *E, const double *H, double *out_host, void *cuda_stream);

/* ---- stabilised central flux (DGM_FLUX_STABILIZED) ----------
 * Face unknowns: HF is a device array double[n_faces][2][N_F], per face the
 * covariant tangential components H^F·t_k (k = 1, 2; t_k the physical edges of
 * the face's ascending-vertex frame) in the face Dubiner basis ψ_γ (graded
 * order).  Faces are numbered by scanning (tet, local face) in ascending order
 * and counting a face at its first tet (interior faces: the smaller tet; PEC
 * faces: their only tet).  With ν_F the outward normal of that tet and
 * [[e]] = e⁻ − e⁺ the system (central part per reading G1) is
 *   (εĖ,e)    = central E-eq + Σ_F (H^F×ν_F, [[e]])_F
 *   (μḢ,h)_T  = central H-eq
 *   (h_F/α)(Ḣ^F, h^F)_F = ([[E]]×ν, h^F)_F       (PEC faces: [[E]] = E⁻)
 * with α = alpha0·p², h_F = sqrt(|t₁×t₂|).  It conserves
 * ½(εE,E) + ½(μH,H) + ½Σ_F (h_F/α)(H^F,H^F)_F.  The face mass h_F/α follows from
 * H^F := α([[E]]×ν)/(iωh), which makes the added term the
 * penalty S(E,e) of strength α/h; the printed face equation
 * has α/h there instead (reading G17). */

/* n_faces and, if face_id != NULL, the face index of every [n_tet][4] slot
 * (host int32).  DGM_EINVAL unless the context is DGM_FLUX_STABILIZED. */
dgm_status dgm_faces(const dgm_ctx *ctx, int64_t *n_faces, int32_t *face_id);

/* nsteps of symplectic Euler with the magnetic unknowns (H, H^F) advanced
 * together: (H, HF) += dt (Ḣ, Ḣ^F)(E);  E += dt Ė(H, HF).  flags as dgm_step_ex. */
dgm_status dgm_step_sc(dgm_ctx *ctx, double *E, double *H, double *HF, double dt, int64_t nsteps, int flags,
                       void *cuda_stream);

/* Full time derivatives (volume + faces) of the stabilised system; NULL outputs skip. */
dgm_status dgm_rhs_sc(dgm_ctx *ctx, const double *E, const double *H, const double *HF, double *dE, double *dH,
                      double *dHF, void *cuda_stream);

/* ½(E,MεE) + ½(H,MμH) + ½Σ_F(h_F/α)(H^F,H^F)_F; synchronises. */
dgm_status dgm_energy_sc(dgm_ctx *ctx, const double *E, const double *H, const double *HF, double *out_host,
                         void *cuda_stream);

/* Spectral radius ρ of K = Mμ^{-1} C Mε^{-1} Cᵀ by power iteration with the
 * Rayleigh quotient in the Mμ inner product, the operator
 * applied through the same stage kernels as dgm_step (Ė(0,H), then Ḣ(·,0)).
 * The symplectic-Euler step is stable for Δt ≤ 2/√ρ (reading G6: the paper's
 * printed bound lacks the square root).  For the upwind flux K is not symmetric
 * and ρ is an estimate.  Deterministic start vector from `seed`.  Uses internal
 * work fields (allocated on first use) and the trace buffers, so a following
 * dgm_step_ex(DGM_STEP_CONTINUE) recomputes them.  Synchronises each iteration. */
dgm_status dgm_spectral_radius(dgm_ctx *ctx, int iters, uint64_t seed, double *rho_out, void *cuda_stream);

/* Host copies of the integer tables, each [n_tet][4]:
 *   nbr (neighbour tet, -1 on PEC), nbr_face (its local face, -1 on PEC),
 *   sign = (-1)^f sign(det F_T), bc (0 interior incl. periodic, 1 PEC).
 * Any pointer may be NULL. */
dgm_status dgm_tables(const dgm_ctx *ctx, int32_t *nbr, int8_t *nbr_face, int8_t *sign, int8_t *bc);

/* Host-only utility (no GPU needed): validate a mesh exactly as dgm_create
 * does and return the integer tables of dgm_tables.  Errors as dgm_create;
 * message via dgm_last_error(NULL). */
dgm_status dgm_match_faces_host(const dgm_mesh *mesh, int32_t *nbr, int8_t *nbr_face, int8_t *sign, int8_t *bc);

/* Number of kernel launches the last dgm_step/dgm_apply_* call enqueued. */
int64_t dgm_last_launches(const dgm_ctx *ctx);

/* Host-only: the reference quadrature of order-`order` contexts with material_points or
 * curved elements: the collapsed Gauss–Jacobi rule with order+2 points per direction
 * (exact to degree 2·order+3), *Q points ξ_i (xi: [Q][3], may be NULL) and weights
 * (w: [Q], may be NULL).  Point i of element T is X0_T + F_T ξ_i (flat elements) or
 * Φ_T(ξ_i) (curved elements, the quadratic map of dgm_opts.edge_nodes).  The order of
 * the points is a outer, c inner in the collapsed coordinates x = (1+a)/2,
 * y = (1-a)(1+b)/4, z = (1-a)(1-b)(1+c)/8 (the sum-factorised inverse mass relies on it). */
dgm_status dgm_quadrature_host(int order, int64_t *Q, double *xi, double *w);

/* The engine the context resolved to (DGM_ENGINE_SPARSE, _DENSE or _HYBRID). */
int dgm_engine(const dgm_ctx *ctx);

const char *dgm_last_error(const dgm_ctx *ctx);
void dgm_destroy(dgm_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGM_H */

/* lfem.h — C ABI of the B200 (sm_100a) ℓFEM assembly library (liblfem.so).
 *
 * The hot path of arxiv/paper_2605_14035 ("ℓFEM"): assembly of the
 * isoparametric finite-element mass matrix M, stiffness matrix A and the
 * coefficient-weighted stiffness A_a (a(u) = 1 + u^2) into CSR, for P1/P2
 * triangles on surfaces in R^3 and P1/P2 tetrahedra in 3-D bulk, in fp64.
 *
 *   M_ij   = sum_E sum_q w_q mu_E(xi_q) phi_i(xi_q) phi_j(xi_q)
 *            PAPER.md §3.2 Eq. (M matrix) P:298, Eq. (reference_quadrature_mass)
 *   A_ij   = sum_E sum_q w_q mu_E(xi_q) grad_E phi_i . grad_E phi_j
 *            Eq. (A matrix) P:301-302, Eq. (Aloc-precise), Eq. (reference_quadrature_stiffness) P:349
 *   Aa_ij  = sum_E sum_q w_q mu_E(xi_q) a(u_h(xi_q)) grad_E phi_i . grad_E phi_j
 *            BASELINE.json north_star; Listing 2 pattern P:793-795 (reading G10)
 * mu_E = |t1 x t2| (surface, Listing 1 l.16-17 P:597-598) or |det DF| (bulk,
 * Eq. basic integral formula P:287); grad_E phi = J G^{-1} grad_ref phi
 * (surface, Eq. surf grad-pre / jacobian_inv P:312-333 read as Listing 1
 * P:599-606, reading G2) or J^{-T} grad_ref phi (bulk, Remark P:278-281).
 *
 * Two phases (§4.2: "The log-linear asymptotic arises
 * solely from sorting and summing duplicate contributions"; "precomputing the
 * sparsity structure ... sort-free assignment"):
 *   lfem_assemble_symbolic  — once per mesh topology: CSR pattern + the
 *                             element-local-entry -> CSR-slot reduction plan.
 *   lfem_assemble_numeric   — every reassembly: geometry, quadrature, local
 *                             matrices, deterministic atomic-free reduction.
 *
 * Conventions (all entry points):
 *  - Every call returns lfem_status; LFEM_OK == 0.  On a non-OK status
 *    lfem_last_error() holds a message and lfem_error_element() the lowest
 *    offending element id (INDEX / DEGENERATE) or -1.  Both are thread-local.
 *  - Device pointers are CUDA device memory of the current device.
 *    "BORROWED" = owned by the caller, must outlive the handle, never written.
 *    "PLAN-OWNED" = owned by the plan, valid until lfem_plan_destroy.
 *    "CALLER-OWNED" = written by the call, owned by the caller.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Node ids are 0-based int32 (Table 1 P:426-435 is 1-based; reading
 *    G22).  coords are n_nodes x 3 fp64, AoS (x,y,z) per node (reading G4).
 *  - Local node order: corners first, then edge nodes; triangle edges
 *    4=(1,2), 5=(2,3), 6=(3,1) (PAPER.md Fig. notation); tetrahedron
 *    edges (1,2),(2,3),(3,1),(1,4),(2,4),(3,4) (reading G26).
 *  - CSR: row_ptr int64 (n_rows + 1, row_ptr[0] = 0), col_idx int32 GLOBAL
 *    column ids ascending within each row; pattern is structural (every (i,j)
 *    sharing an element, explicit zeros kept, reading G19); full, not
 *    triangular.  For a row block [row_begin, row_end), row r of the plan is
 *    global row row_begin + r.
 *  - Determinism: identical inputs give bitwise-identical values, independent
 *    of the numeric variant's tiling and of the row-block partition (each CSR
 *    slot sums its contributions in ascending element id, then local (a,b);
 *    reading G21).  No floating-point atomics anywhere.
 *  - Limits: n_nodes, n_elems < 2^31; local entries n_elems_local*nref^2 < 2^31.
 *    Rows with more than 512 candidate (element, column) entries (e.g. a P2 tet
 *    vertex shared by more than 51 tets) take a slower one-CTA-per-row path of
 *    the symbolic phase (at most 65536 such rows).  TILED: a row may touch at
 *    most the tile capacity of elements (256 P2 / 1024 P1 triangles, 128 P2 /
 *    256 P1 tets) and a CSR slot at most 254 contributions; an explicit TILED
 *    request then returns LFEM_ERR_UNSUPPORTED, AUTO runs V0 on that plan.
 *  - Alignment: double arrays (coords, coeff, vals, u, out) 8-byte aligned and
 *    int32 arrays 4-byte aligned, else LFEM_ERR_INVALID_ARG.  The TILED kernel
 *    copies coords and coeff with cp.async.bulk (16-byte aligned sources) and
 *    writes vals with 16-byte stores: if any of them is only 8-byte aligned,
 *    AUTO runs V0 and an explicit TILED request returns LFEM_ERR_INVALID_ARG
 *    (no misaligned-address fault).
 *  - Device allocations of plans (and of lfem_mesh_create's index check) are
 *    stream-ordered on the call's stream (cudaMallocAsync / cudaFreeAsync)
 *    unless a hook is installed (lfem_set_allocator).
 */
#ifndef LFEM_H_
#define LFEM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lfem_stream_t; /* == cudaStream_t */

typedef enum {
    LFEM_OK = 0,
    LFEM_ERR_INVALID_ARG = 1, /* null pointer, bad size, bad kinds, missing coeff */
    LFEM_ERR_UNSUPPORTED = 2, /* (domain, order, quad) not supported, or a limit exceeded */
    LFEM_ERR_INDEX = 3,       /* connectivity entry outside [0, n_nodes); see lfem_error_element */
    LFEM_ERR_DEGENERATE = 4,  /* mu <= 0 or non-finite at a quadrature point; lowest element id */
    LFEM_ERR_NOMEM = 5,       /* device or host allocation failed */
    LFEM_ERR_CUDA = 6,        /* CUDA runtime error; message in lfem_last_error */
    LFEM_ERR_STATE = 7        /* handle in an unusable state (e.g. destroyed mesh) */
} lfem_status;

typedef enum {
    LFEM_SURFACE_TRI = 0, /* 2-D triangles embedded in R^3 (§3) */
    LFEM_BULK_TET = 1,    /* 3-D tetrahedra (Remark P:278-281) */
    LFEM_SURFACE_LINE = 2 /* curves: line elements in R^3 (Table 4 "surface 1D"; SURVEY
                             §8(f) N2); numeric variant V0, right-hand side LOAD */
} lfem_domain;

/* Quadrature rules (BASELINE.json configs; readings G6-G9). DEFAULT picks
 * TRI3_DEG2 (P1 tri), TRI6_DEG4 (P2 tri), TET4_DEG2 (P1 tet), TET11_DEG4 (P2 tet). */
typedef enum {
    LFEM_QUAD_DEFAULT = 0,
    LFEM_QUAD_TRI3_DEG2 = 1,  /* 3 points, permutations of (2/3,1/6,1/6), w = 1/6 */
    LFEM_QUAD_TRI6_DEG4 = 2,  /* 6-point symmetric degree-4 rule */
    LFEM_QUAD_TET4_DEG2 = 3,  /* 4-point degree-2 rule */
    LFEM_QUAD_TET11_DEG4 = 4, /* Keast 11-point degree-4 rule (negative centroid weight) */
    LFEM_QUAD_TRI16_DEG8 = 5, /* Dunavant 16-point degree-8 rule, P2 triangles only (the paper's
                                 load-vector rule) */
    LFEM_QUAD_LINE2_DEG3 = 6, /* 2-point Gauss-Legendre (P1 curves) */
    LFEM_QUAD_LINE3_DEG5 = 7, /* 3-point Gauss-Legendre (P2 curves) */
    LFEM_QUAD_TET35_DEG7 = 8, /* 35-point fully symmetric positive degree-7 rule, P2 tets only (the
                                 paper's Jaskowiec-Sukumar degree-7 rule; constants derived
                                 from the moment equations, reading G39) */
    LFEM_QUAD_LINE6_DEG11 = 9 /* 6-point Gauss-Legendre, P2 curves only (the paper's order-10 Gauss
                                 rule for curves, reading G38) */
} lfem_quad;

/* 'kinds' bitmask of lfem_assemble_numeric; vals[] index = bit position. */
enum { LFEM_MASS = 1u, LFEM_STIFF = 2u, LFEM_STIFF_COEF = 4u };

/* Numeric variants (lfem_plan_set_variant); all produce identical bits.
 * AUTO picks TILED for triangles and V0 for tetrahedra (measured, DESIGN.md
 * §6.5); ROWS is opt-in (measured slower: 2.4 vs 0.72 ms on C4P1). */
typedef enum {
    LFEM_NUMERIC_AUTO = 0,   /* the fastest measured variant for the family */
    LFEM_NUMERIC_V0 = 1,     /* element kernel -> element-major local matrices in HBM -> per-slot gather */
    LFEM_NUMERIC_TILED = 2,  /* fused row-tile kernel: TMA-fed, warp-specialised, shared-memory stage,
                                halo recompute; the tile plan is built on the first call (one sync) */
    LFEM_NUMERIC_ROWS = 3    /* warp per CSR row, each incident element recomputed per row (cheap
                                elements); rows longer than 64 columns fall back to V0; the first
                                call builds the row incidence lists (one sync) */
} lfem_numeric_variant;

typedef struct lfem_mesh_s* lfem_mesh;
typedef struct lfem_plan_s* lfem_plan;

/* Create a mesh handle (§4.1: node array N, element array E).
 *   dom, order (1|2), quad: element family and rule; unsupported -> UNSUPPORTED.
 *   coords: device, n_nodes x 3 fp64 AoS, BORROWED.
 *   conn:   device, n_elems x nref int32 row-major (nref = 3/6 tri, 4/10 tet), BORROWED.
 * Validates every connectivity entry on `stream` (one kernel, then a sync):
 * out-of-range -> LFEM_ERR_INDEX with the lowest bad element id.  n_elems may
 * be 0 (empty mesh: every plan has nnz = 0). */
lfem_status lfem_mesh_create(lfem_domain dom, int order, lfem_quad quad,
                             int64_t n_nodes, const double* coords,
                             int64_t n_elems, const int32_t* conn,
                             lfem_stream_t stream, lfem_mesh* out);
void lfem_mesh_destroy(lfem_mesh m);

/* Symbolic phase (one-time; §4.2, Listing 1 l.10-11 I,J P:591-592).
 * Builds, for the owned rows [row_begin, row_end) (0 <= row_begin <= row_end <= n_nodes):
 * the list of elements touching those rows (ascending id, halo elements
 * duplicated), the CSR pattern, and the reduction plan that maps every
 * element-local entry (e, a, b) with conn[e,a] owned to its CSR slot.
 * Method: one-digit LSD radix (counting) sort of the local entries by row,
 * then a segmented sort + unique of the columns inside each row.
 * Synchronises `stream` once (nnz must be known to size buffers).
 * The mesh must outlive the plan. */
lfem_status lfem_assemble_symbolic(lfem_mesh m, int64_t row_begin, int64_t row_end,
                                   lfem_stream_t stream, lfem_plan* out);
/* Waits for the work this plan enqueued (an event per stream it ran on; not a
 * device-wide sync), then frees the plan. */
void lfem_plan_destroy(lfem_plan p);

/* n_rows = row_end - row_begin; nnz of the block; n_elems_local = elements touching it. */
lfem_status lfem_plan_info(lfem_plan p, int64_t* n_rows, int64_t* nnz, int64_t* n_elems_local);

/* Select the numeric kernel variant (default AUTO).  UNSUPPORTED if the
 * variant is not available for the plan's family. */
lfem_status lfem_plan_set_variant(lfem_plan p, lfem_numeric_variant v);

/* Numeric phase (every reassembly; Listing 1 l.12-28 P:593-609).
 *   kinds: nonzero subset of LFEM_MASS | LFEM_STIFF | LFEM_STIFF_COEF.
 *   coeff: device, n_nodes fp64 nodal u (BORROWED); required iff LFEM_STIFF_COEF
 *          (else LFEM_ERR_INVALID_ARG, SPEC-style "missing coefficient").
 *   vals:  vals[0] = M, vals[1] = A, vals[2] = A_a; device, nnz fp64 each,
 *          CALLER-OWNED; must be non-NULL exactly for the requested kinds.
 * Enqueues work on `stream` only (no sync).  A degenerate element is latched
 * on the device and reported by lfem_plan_check (values are then undefined). */
lfem_status lfem_assemble_numeric(lfem_plan p, unsigned kinds, const double* coeff,
                                  double* const vals[3], lfem_stream_t stream);

/* Same as lfem_assemble_numeric, but with moving geometry: coords (device,
 * n_nodes x 3, BORROWED) replaces the mesh's coordinates for this call
 * (the topology, hence the plan, is unchanged; §6.2-6.3 reassembly). */
lfem_status lfem_assemble_numeric_coords(lfem_plan p, unsigned kinds, const double* coords,
                                         const double* coeff, double* const vals[3],
                                         lfem_stream_t stream);

/* End-to-end entry with HOST buffers: copies coords_h (n_nodes x 3; NULL =
 * keep the mesh's device coords) and coeff_h (n_nodes; NULL unless
 * LFEM_STIFF_COEF) host->device into plan-owned staging, assembles, copies
 * the requested vals back into vals_h[k] (host, nnz each, CALLER-OWNED;
 * pinned memory recommended) and synchronises `stream`. */
lfem_status lfem_assemble_numeric_host(lfem_plan p, unsigned kinds, const double* coords_h,
                                       const double* coeff_h, double* const vals_h[3],
                                       lfem_stream_t stream);

/* Right-hand sides, assembled into the plan's owned
 * rows with the same deterministic order as the matrices (per row: ascending
 * element id; no atomics).
 *   LFEM_RHS_LOAD (all families; 1 input / 1 output component):
 *       b_j = sum_E sum_q w_q mu_E(xi_q) f_h(xi_q) phi_j(xi_q),  f_h = sum_c f_c phi_c
 *       (PAPER.md Eq. "load vector" P:168-177; equals M f with the element rule).
 *   LFEM_RHS_KLL (surface triangles only; 4 input / 4 output components):
 *       u = (nu_1, nu_2, nu_3, H) nodal,
 *       alpha^2 = |grad_{Gamma_h} nu_h|^2 (Frobenius; Listing 2 line 2),
 *       f_{k,j} = sum_E sum_q w_q mu alpha^2 u_{h,k}(xi_q) phi_j(xi_q), k = 1..4
 *       (f_1 = first three components, f_2 = the H component; P:784-789,
 *       Listing 2 lines 3-4).
 * Layout: u is ncomp x n_nodes, component-major (u[k * n_nodes + node], the
 * paper's index j + (k-1) N), device, BORROWED; out is ncomp x n_rows,
 * component-major over the owned rows (out[k * n_rows + (row - row_begin)]),
 * device, CALLER-OWNED.  coords: device n_nodes x 3 (moving geometry) or NULL
 * for the mesh's coordinates.  The first call per plan (and variant) builds
 * plan-owned row incidence lists and synchronises `stream`; later calls only
 * enqueue.  Variants (lfem_plan_set_variant): AUTO / V0 = element kernel +
 * row reduce through a plan-owned staging buffer (n_elems_local * nref * 4
 * fp64); TILED = one fused kernel on the matrices' row tiles (local vectors
 * staged in shared memory; builds the tile plan if the matrices have not;
 * falls back to V0 where it does not fit; measured slower).
 * Both give the same bits.  Errors: INVALID_ARG (NULL u/out, unknown kind), UNSUPPORTED
 * (KLL on a bulk mesh); degenerate elements are latched as for the matrices
 * (lfem_plan_check). */
typedef enum { LFEM_RHS_LOAD = 1, LFEM_RHS_KLL = 2 } lfem_rhs_kind;
lfem_status lfem_assemble_rhs(lfem_plan p, int kind, const double* coords, const double* u, double* out,
                              lfem_stream_t stream);
/* Components of a right-hand side kind (1 or 4), 0 if unknown. */
int lfem_rhs_ncomp(int kind);
/* Kernel launches the plan's last lfem_assemble_rhs call enqueued (1 fused, 2 two-kernel). */
int lfem_rhs_launches(lfem_plan p, int kind);

/* Jacobi-preconditioned conjugate gradients for K x = b with three right-hand
 * sides at once, K = the plan's CSR pattern with
 * values vals_K (device, nnz fp64, BORROWED; symmetric positive definite with a
 * positive diagonal).  b, x: device n_nodes x 3 AoS (the node array's layout);
 * x holds the initial guess on entry and the solution on exit.  Stops when
 * ||r_k|| <= tol ||b_k|| for every column k, else LFEM_ERR_STATE after max_it
 * iterations.  Whole-mesh plans only (UNSUPPORTED for a row block: the
 * multi-GPU solve would need an exchange per iteration).  Deterministic
 * reductions; synchronises `stream` every 8 iterations (convergence check,
 * so the iteration count is a multiple of 8 unless max_it is reached).
 * iters (host, may be NULL): iterations used.  Plan-owned workspace. */
lfem_status lfem_cg_solve(lfem_plan p, const double* vals_K, const double* b, double* x, double tol,
                          int max_it, int* iters, lfem_stream_t stream);

/* Mean-free surface Poisson solve:
 * the least-squares solution of the bordered system [A; e^T] u = [b; 0]
 * (e = ones), i.e. A u = b - mean(b) e with sum_j u_j = 0, for three AoS
 * columns at once.  vals_A: the plan's stiffness values (device, BORROWED;
 * symmetric positive semidefinite with kernel span{e}).  b, u: device
 * n_nodes x 3 AoS; u is overwritten.  Jacobi-PCG from u = 0 to
 * ||r_k|| <= tol ||b_k - mean(b_k)||, then the nodal mean is removed.
 * Whole-mesh plans only; iters as for lfem_cg_solve. */
lfem_status lfem_solve_meanfree(lfem_plan p, const double* vals_A, const double* b, double* u, double tol,
                                int max_it, int* iters, lfem_stream_t stream);

/* One step of Dziuk's algorithm for mean curvature flow:
 *     (M(x^{n-1}) + tau A(x^{n-1})) x^n = M(x^{n-1}) x^{n-1}
 * on a whole-mesh surface plan: numeric assembly of M and A at x_prev (the
 * plan's topology; x_prev replaces the mesh coordinates), K = M + tau A,
 * b = M x_prev, then lfem_cg_solve from the initial guess x_prev.
 * x_prev, x_next: device n_nodes x 3 (may alias).  tau > 0.  UNSUPPORTED on
 * bulk meshes.  Degenerate elements are latched (lfem_plan_check). */
lfem_status lfem_mcf_step(lfem_plan p, double tau, const double* x_prev, double* x_next, double tol,
                          int max_it, int* iters, lfem_stream_t stream);

/* CSR pattern of the plan: device pointers, PLAN-OWNED.
 * row_ptr: n_rows + 1 int64 (relative to the block); col_idx: nnz int32 (global). */
lfem_status lfem_csr_get(lfem_plan p, const int64_t** row_ptr, const int32_t** col_idx);

/* y_rows[r] = sum_j vals[j] * x_full[col_idx[j]] over the plan's rows
 * (verification SpMV; x_full: device n_nodes, y_rows: device n_rows). */
lfem_status lfem_spmv(lfem_plan p, const double* vals, const double* x_full, double* y_rows,
                      lfem_stream_t stream);

/* Synchronises `stream`, then reports latched device errors
 * (LFEM_ERR_DEGENERATE with the lowest element id).  A reported error is
 * cleared: the latch holds the lowest bad element of the calls enqueued since
 * the last check (lfem_assemble_numeric_host checks at its end), so a plan
 * reused with valid coordinates after a degenerate call reports OK again. */
lfem_status lfem_plan_check(lfem_plan p, lfem_stream_t stream);

/* out[i] = ca * a[i] + cb * b[i], i < n (device; the C3 coefficient update
 * u(t) = cos(2 pi t/100) u_A + sin(2 pi t/100) u_B, reading G12). */
lfem_status lfem_axpby(int64_t n, double ca, const double* a, double cb, const double* b,
                       double* out, lfem_stream_t stream);

/* Per-kernel device timing of the numeric phase: when enabled, every kernel
 * launch of lfem_assemble_numeric* is bracketed by CUDA events on its stream.
 * lfem_profile_read synchronises, returns up to `max` kernel names (static
 * strings), their summed milliseconds and launch counts in *n entries, and
 * resets the counters. */
lfem_status lfem_profile_enable(lfem_plan p, int enable);
lfem_status lfem_profile_read(lfem_plan p, int max, const char** names, double* ms, int64_t* launches, int* n);

/* Number of kernel launches lfem_assemble_numeric enqueues for this plan and kinds. */
int lfem_numeric_launches(lfem_plan p, unsigned kinds);

/* Work of the last numeric call on this plan: elem_evals = element evaluations
 * (geometry + local matrices) per call -- n_elems_local for V0 / ROWS, the sum
 * of the tiles' element lists (halo elements counted once per tile) for TILED;
 * n_tiles = row tiles of the TILED plan (0 otherwise).  Either pointer may be NULL. */
lfem_status lfem_numeric_stats(lfem_plan p, int64_t* elem_evals, int64_t* n_tiles);

/* Device-memory allocator hook (a user's caching allocator,
 * e.g. PyTorch's).  Every device allocation of meshes and plans (plan arrays,
 * tile plan, V0 stage, e2e staging) goes through alloc(bytes, stream, ctx)
 * and is released with dealloc(ptr, stream, ctx) on the stream it was used on;
 * alloc returns a 256-B aligned device pointer or NULL (-> LFEM_ERR_NOMEM).
 * NULL, NULL restores cudaMallocAsync / cudaFreeAsync on the call's stream.  Process-wide; may be changed at
 * any time: every pointer is released by the allocator (hook + ctx, or
 * cudaFreeAsync) that produced it.  INVALID_ARG if exactly one of alloc / dealloc
 * is NULL. */
typedef void* (*lfem_alloc_fn)(size_t bytes, lfem_stream_t stream, void* ctx);
typedef void (*lfem_free_fn)(void* ptr, lfem_stream_t stream, void* ctx);
lfem_status lfem_set_allocator(lfem_alloc_fn alloc, lfem_free_fn dealloc, void* ctx);

int64_t lfem_error_element(void);
const char* lfem_last_error(void);
const char* lfem_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LFEM_H_ */

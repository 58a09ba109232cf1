// Internal definitions of liblfem (B200, sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/lfem.h"

// ---------------------------------------------------------------------------
// element families
// ---------------------------------------------------------------------------
enum Family { FAM_TRI_P1 = 0, FAM_TRI_P2 = 1, FAM_TET_P1 = 2, FAM_TET_P2 = 3, FAM_TRI_P2_Q16 = 4, FAM_LINE_P1 = 5,
              FAM_LINE_P2 = 6, FAM_TET_P2_Q35 = 7, FAM_LINE_P2_Q6 = 8 };
constexpr int N_FAMILIES = 9;

template <int F> struct FamInfo;
template <> struct FamInfo<FAM_TRI_P1> { static constexpr int NREF = 3, D = 2, NQ = 3, NSYM = 6; };
template <> struct FamInfo<FAM_TRI_P2> { static constexpr int NREF = 6, D = 2, NQ = 6, NSYM = 21; };
template <> struct FamInfo<FAM_TET_P1> { static constexpr int NREF = 4, D = 3, NQ = 4, NSYM = 10; };
template <> struct FamInfo<FAM_TET_P2> { static constexpr int NREF = 10, D = 3, NQ = 11, NSYM = 55; };
// P2 triangles with Dunavant's 16-point degree-8 rule (the paper's load-vector rule)
template <> struct FamInfo<FAM_TRI_P2_Q16> { static constexpr int NREF = 6, D = 2, NQ = 16, NSYM = 21; };
// curves: Gauss-Legendre 2 / 3 points
template <> struct FamInfo<FAM_LINE_P1> { static constexpr int NREF = 2, D = 1, NQ = 2, NSYM = 3; };
template <> struct FamInfo<FAM_LINE_P2> { static constexpr int NREF = 3, D = 1, NQ = 3, NSYM = 6; };
// the paper's other rules: a 35-point degree-7 tet rule (reading G39)
// and the 6-point Gauss-Legendre rule (order 10 for curves, reading G38)
template <> struct FamInfo<FAM_TET_P2_Q35> { static constexpr int NREF = 10, D = 3, NQ = 35, NSYM = 55; };
template <> struct FamInfo<FAM_LINE_P2_Q6> { static constexpr int NREF = 3, D = 1, NQ = 6, NSYM = 6; };

// index of (a, b), a <= b, in the row-major upper triangle of an n x n matrix
__host__ __device__ constexpr int sym_index(int n, int a, int b) {
    return a <= b ? a * n - a * (a - 1) / 2 + (b - a) : b * n - b * (b - 1) / 2 + (a - b);
}

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct lfem_mesh_s {
    int domain, order, quad, family, nref, nq, nsym;
    int64_t n_nodes, n_elems;
    const double* coords;
    const int32_t* conn;
};

// Slot words of the tiled kernel: a missing second contribution is encoded as the
// stage's zero word (1) or as 0xffff with a predicated load (0).
#ifndef LFEM_ZERO_WORD
#define LFEM_ZERO_WORD 1
#endif

// Row-tile plan of the fused numeric kernel (tiles.cu).
struct TilePlan {
    int n_tiles = 0;
    int rows_per_tile = 0;      // average rows per tile (tiles are built by element budget)
    int max_tile_elems = 0;     // stage stride: max elements per tile, rounded up to odd (codes are sym * maxe + e_tile)
    int max_tile_count = 0;     // max elements per tile
    int max_tile_slots = 0;     // max CSR slots per tile
    int max_tile_heavy = 0;     // max heavy-list u16 words per tile
    int heavy_words = 8;        // u16 words per heavy entry (16-B multiple)
    int32_t* tile_elems = nullptr;      // plan-local element ids, ascending per tile
    int32_t* tile_elems_pos = nullptr;  // the same ids in stage-position order (tiles.cu k_tile_order)
    int max_tile_nodes = 0;     // max owned rows + halo nodes per tile
    int64_t total_elems = 0;    // element evaluations per numeric call (tile halo included)
    uint16_t* conn16 = nullptr;         // per tile: its elements' tile-local node indices (16-B padded)
    int32_t* halo = nullptr;            // per tile: halo nodes (global ids, sorted; 16-B padded)
    int4* tile_info = nullptr;          // 3 per tile: {s0, ns, e0, ne}, {q0, nq, h0, nh}, {g0, nrows, l0, nl}
    uint32_t* pairs = nullptr;          // nnz: per slot, (c0 | c1 << 16); c1 = 0xffff if one contribution;
                                        // 0xffffffff for a heavy slot (> 2 contributions)
    uint16_t* heavy = nullptr;          // per heavy slot: [slot - s0, count, codes...] (fixed size per family)
    bool ready = false;
};
// Workspace of lfem_cg_solve / lfem_mcf_step (mcf.cu): AoS n x 3 vectors, M/A/K values
struct McfWork {
    double *r = nullptr, *z = nullptr, *pv = nullptr, *q = nullptr, *b = nullptr, *dinv = nullptr;
    double *M = nullptr, *A = nullptr, *K = nullptr, *part = nullptr, *sc = nullptr;
    // CUDA graph of CG_CHECK steady-state CG iterations (mcf.cu), keyed by the operands it captured
    cudaGraphExec_t cg_exec = nullptr;
    const double* cg_key_K = nullptr;
    const double* cg_key_x = nullptr;
    cudaStream_t cap = nullptr;  // private capture stream (the caller's may be the legacy stream)
    int* bad = nullptr;
};
struct Profiler;  // api.cu
void prof_begin(lfem_plan_s* p, const char* name, cudaStream_t s);
void prof_end(lfem_plan_s* p, cudaStream_t s);
bool prof_on(lfem_plan_s* p);

struct lfem_plan_s {
    lfem_mesh_s* mesh = nullptr;
    int64_t row_begin = 0, row_end = 0, n_rows = 0, nnz = 0, n_local = 0, n_contrib = 0;
    int32_t* elem_list = nullptr;   // n_local: global element ids, ascending
    int32_t* local_conn = nullptr;  // n_local x nref copy of the connectivity (plan order)
    int64_t* row_ptr = nullptr;     // n_rows + 1
    int32_t* col_idx = nullptr;     // nnz (global)
    int32_t* slot_ptr = nullptr;    // nnz + 1 into codes
    int32_t* codes = nullptr;       // n_contrib: sym * n_local + local element
    double* stage = nullptr;        // v0 staging: 3 x nsym x n_local
    int* err = nullptr;             // device: lowest degenerate element id (INT_MAX = none)
    int variant = LFEM_NUMERIC_AUTO;
    TilePlan tiles;
    Profiler* prof = nullptr;
    // e2e staging (lfem_assemble_numeric_host)
    double* d_coords = nullptr;
    double* d_coeff = nullptr;
    double* d_vals[3] = {nullptr, nullptr, nullptr};
    // right-hand sides (rhs.cuh): per owned row, its incident (element, a) in ascending element order
    int64_t* rhs_ptr = nullptr;     // n_rows + 1
    int32_t* rhs_codes = nullptr;   // le * nref + a
    double* rhs_stage = nullptr;    // n_local x nref x 4 (two-kernel variant)
    int64_t rhs_total = 0;          // entries of rhs_codes
    uint16_t* rhs_tcodes = nullptr; // fused variant: e_tile * nref + a, same indexing as rhs_codes
    int rhs_tiled = -1;             // -1 not tried, 0 unavailable, 1 tile-local codes built
    int rhs_last_tiled = -1;        // variant of the last lfem_assemble_rhs call (1 fused, 0 two-kernel)
    McfWork mcf;                    // CG / MCF workspace (mcf.cu)
    int rows_ok = -1;               // ROWS variant (rows.cuh): -1 unknown, 1 every row fits, 0 fall back to V0
    int tiled_ok = -1;              // TILED tile plan: -1 not built, 1 built, 0 unsupported (AUTO runs V0)
    int last_variant = -1;          // variant the last numeric call ran (after AUTO / alignment fallbacks)
    // completion events of the calls that enqueued work on this plan, one per stream
    // (lfem_plan_destroy waits for them instead of the whole device)
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> done;
};
// record that plan p has work enqueued on stream s (lfem_plan_destroy waits for it)
lfem_status plan_mark(lfem_plan_s* p, cudaStream_t s);

// ---------------------------------------------------------------------------
// error state (thread-local, set by every failing entry point)
// ---------------------------------------------------------------------------
lfem_status lfem_fail(lfem_status st, const std::string& msg, int64_t elem = -1);
lfem_status lfem_cuda_fail(cudaError_t e, const char* what);

#define LFEM_CUDA(call)                                            \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return lfem_cuda_fail(e_, #call);   \
    } while (0)

#define LFEM_TRY(call)                                             \
    do {                                                           \
        lfem_status s_ = (call);                                   \
        if (s_ != LFEM_OK) return s_;                              \
    } while (0)

// Per-(device, kernel) launch attribute cache: one process may drive several
// devices, so nothing launch-related is cached per process.
lfem_status ensure_smem_attr(const void* func, int bytes);
lfem_status device_sm_count(int* sms);

// device memory helpers (cudaMallocAsync on the given stream, or the caller's hook)
lfem_status dev_alloc(void** p, size_t bytes, cudaStream_t s);
void dev_free(void* p, cudaStream_t s);
template <class T>
inline lfem_status dev_alloc_t(T** p, size_t n, cudaStream_t s) {
    return dev_alloc(reinterpret_cast<void**>(p), n * sizeof(T) + 16, s);
}

// Device temporaries of a host function: track() them after declaring,
// drop() frees early; whatever is still held is freed on every exit path
// (including early error returns).  give() hands ownership to the caller.
struct DevScope {
    cudaStream_t s;
    std::vector<void**> ptrs;
    explicit DevScope(cudaStream_t st) : s(st) {}
    DevScope(const DevScope&) = delete;
    DevScope& operator=(const DevScope&) = delete;
    template <class T> void track(T** p) { ptrs.push_back(reinterpret_cast<void**>(p)); }
    template <class T> void drop(T*& p) {
        dev_free(p, s);
        p = nullptr;
    }
    template <class T> void give(T** p) {
        for (auto& q : ptrs)
            if (q == reinterpret_cast<void**>(p)) q = nullptr;
    }
    ~DevScope() {
        for (void** q : ptrs)
            if (q && *q) {
                dev_free(*q, s);
                *q = nullptr;
            }
    }
};

// scan.cu: out[0] = 0, out[i+1] = sum_{j<=i} in[j]  (n+1 outputs)
lfem_status scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s);

// symbolic.cu
lfem_status build_symbolic(lfem_plan_s* p, cudaStream_t s);
lfem_status build_incidence(lfem_plan_s* p, int64_t** inc_ptr, int32_t** inc, cudaStream_t s);
lfem_status build_tiles(lfem_plan_s* p, int max_tile_elems, cudaStream_t s);
void free_tiles(TilePlan& t, cudaStream_t s);

// numeric.cu
lfem_status numeric_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                             double* const vals[3], cudaStream_t s);
int numeric_launch_count(lfem_plan_s* p, unsigned kinds);
lfem_status rhs_dispatch(lfem_plan_s* p, int kind, const double* coords, const double* u, double* out,
                         cudaStream_t s);
int rhs_launch_count(lfem_plan_s* p);
// mcf.cu
lfem_status cg_solve(lfem_plan_s* p, const double* vals_K, const double* b, double* x, double tol, int max_it,
                     int* iters, cudaStream_t s);
lfem_status mcf_step(lfem_plan_s* p, double tau, const double* x_prev, double* x_next, double tol, int max_it,
                     int* iters, cudaStream_t s);
void mcf_free(lfem_plan_s* p, cudaStream_t s);
lfem_status solve_meanfree(lfem_plan_s* p, const double* vals_A, const double* b, double* u, double tol, int max_it,
                           int* iters, cudaStream_t s);
lfem_status spmv_launch(lfem_plan_s* p, const double* vals, const double* x, double* y, cudaStream_t s);
lfem_status axpby_launch(int64_t n, double ca, const double* a, double cb, const double* b, double* out,
                         cudaStream_t s);
lfem_status upload_reference_tables();
lfem_status check_conn_launch(const int32_t* conn, int64_t n_elems, int nref, int64_t n_nodes, int* bad,
                              cudaStream_t s);

inline int family_of(int domain, int order, int quad = LFEM_QUAD_DEFAULT) {
    if (domain == LFEM_SURFACE_LINE)
        return order == 1 ? FAM_LINE_P1 : quad == LFEM_QUAD_LINE6_DEG11 ? FAM_LINE_P2_Q6 : FAM_LINE_P2;
    if (domain == LFEM_BULK_TET && order == 2 && quad == LFEM_QUAD_TET35_DEG7) return FAM_TET_P2_Q35;
    if (domain == LFEM_SURFACE_TRI && order == 2 && quad == LFEM_QUAD_TRI16_DEG8) return FAM_TRI_P2_Q16;
    if (domain == LFEM_SURFACE_TRI) return order == 1 ? FAM_TRI_P1 : FAM_TRI_P2;
    return order == 1 ? FAM_TET_P1 : FAM_TET_P2;
}

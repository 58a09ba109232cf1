// C ABI of liblfem (include/lfem.h): handles, argument checking, errors.
#include <climits>
#include <map>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "lfem_internal.cuh"

struct Profiler {
    bool on = false;
    struct Pending { int slot; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<const char*> names;
    std::vector<double> ms;
    std::vector<int64_t> count;
    int open_slot = -1;
    cudaEvent_t open_ev = nullptr;
    cudaEvent_t get() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e = nullptr;
        cudaEventCreate(&e);
        return e;
    }
    int slot_of(const char* n) {
        for (size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return (int)i;
        names.push_back(n); ms.push_back(0.0); count.push_back(0);
        return (int)names.size() - 1;
    }
    void collect() {
        for (auto& pd : pending) {
            float t = 0.f;
            cudaEventSynchronize(pd.b);
            cudaEventElapsedTime(&t, pd.a, pd.b);
            ms[pd.slot] += t;
            count[pd.slot] += 1;
            pool.push_back(pd.a); pool.push_back(pd.b);
        }
        pending.clear();
    }
    ~Profiler() {
        collect();
        for (auto e : pool) cudaEventDestroy(e);
    }
};

bool prof_on(lfem_plan_s* p) { return p->prof && p->prof->on; }

void prof_begin(lfem_plan_s* p, const char* name, cudaStream_t s) {
    if (!p->prof || !p->prof->on) return;
    Profiler& P = *p->prof;
    P.open_slot = P.slot_of(name);
    P.open_ev = P.get();
    cudaEventRecord(P.open_ev, s);
}

void prof_end(lfem_plan_s* p, cudaStream_t s) {
    if (!p->prof || !p->prof->on || p->prof->open_slot < 0) return;
    Profiler& P = *p->prof;
    cudaEvent_t b = P.get();
    cudaEventRecord(b, s);
    P.pending.push_back({P.open_slot, P.open_ev, b});
    P.open_slot = -1;
    if (P.pending.size() > 4096) P.collect();
}

namespace {
thread_local std::string g_err;
thread_local int64_t g_err_elem = -1;

cudaStream_t S(lfem_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

void free_plan_memory(lfem_plan_s* p) {
    // every stream that ran work on the plan is done (lfem_plan_destroy waited on the
    // plan's events), so the frees may be ordered on the legacy stream
    cudaStream_t s = nullptr;
    dev_free(p->elem_list, s);
    dev_free(p->local_conn, s);
    dev_free(p->row_ptr, s);
    dev_free(p->col_idx, s);
    dev_free(p->slot_ptr, s);
    dev_free(p->codes, s);
    dev_free(p->stage, s);
    dev_free(p->err, s);
    dev_free(p->d_coords, s);
    dev_free(p->d_coeff, s);
    for (int k = 0; k < 3; ++k) dev_free(p->d_vals[k], s);
    dev_free(p->rhs_ptr, s);
    dev_free(p->rhs_codes, s);
    dev_free(p->rhs_stage, s);
    dev_free(p->rhs_tcodes, s);
    mcf_free(p, s);
    free_tiles(p->tiles, s);
    delete p->prof;
    p->prof = nullptr;
}
}  // namespace

lfem_status lfem_fail(lfem_status st, const std::string& msg, int64_t elem) {
    g_err = msg;
    g_err_elem = elem;
    return st;
}

lfem_status lfem_cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return lfem_fail(LFEM_ERR_NOMEM, std::string("device allocation failed: ") + what);
    }
    return lfem_fail(LFEM_ERR_CUDA, std::string(cudaGetErrorString(e)) + " in " + what);
}

// Device allocations of plans/meshes: cudaMalloc / cudaFree, or the caller's hook
// (lfem_set_allocator; e.g. PyTorch's caching allocator).  Every pointer is
// released by the allocator that produced it, even if the hook changed since.
namespace {
struct Hook {
    lfem_alloc_fn alloc = nullptr;
    lfem_free_fn dealloc = nullptr;
    void* ctx = nullptr;
};
Hook g_hook;
std::mutex g_hook_mu;
std::unordered_map<void*, Hook> g_hooked;  // pointers allocated through a hook
}  // namespace

lfem_status dev_alloc(void** p, size_t bytes, cudaStream_t s) {
    *p = nullptr;
    Hook h;
    {
        std::lock_guard<std::mutex> lk(g_hook_mu);
        h = g_hook;
    }
    if (h.alloc) {
        *p = h.alloc(bytes, reinterpret_cast<lfem_stream_t>(s), h.ctx);
        if (!*p) return lfem_fail(LFEM_ERR_NOMEM, "allocator hook returned NULL for " + std::to_string(bytes) + " bytes");
        std::lock_guard<std::mutex> lk(g_hook_mu);
        g_hooked[*p] = h;
        return LFEM_OK;
    }
    // default: stream-ordered allocation on the call's stream (SURVEY.md §8(b) conventions)
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return lfem_fail(LFEM_ERR_NOMEM, "cudaMallocAsync of " + std::to_string(bytes) + " bytes failed");
    }
    return LFEM_OK;
}

void dev_free(void* p, cudaStream_t s) {
    if (!p) return;
    Hook h;
    {
        std::lock_guard<std::mutex> lk(g_hook_mu);
        auto it = g_hooked.find(p);
        if (it != g_hooked.end()) {
            h = it->second;
            g_hooked.erase(it);
        }
    }
    if (h.dealloc) {
        h.dealloc(p, reinterpret_cast<lfem_stream_t>(s), h.ctx);
        return;
    }
    cudaFreeAsync(p, s);
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_attr;  // (device, kernel) -> opted-in dynamic smem bytes
}  // namespace

lfem_status ensure_smem_attr(const void* func, int bytes) {
    int dev = 0;
    LFEM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& have = g_attr[{dev, func}];
    if (have >= bytes) return LFEM_OK;
    LFEM_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
    return LFEM_OK;
}

lfem_status device_sm_count(int* sms) {
    int dev = 0;
    LFEM_CUDA(cudaGetDevice(&dev));
    LFEM_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
    return LFEM_OK;
}

lfem_status plan_mark(lfem_plan_s* p, cudaStream_t s) {
    for (auto& d : p->done)
        if (d.first == s) {
            LFEM_CUDA(cudaEventRecord(d.second, s));
            return LFEM_OK;
        }
    cudaEvent_t ev = nullptr;
    LFEM_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    p->done.push_back({s, ev});
    LFEM_CUDA(cudaEventRecord(ev, s));
    return LFEM_OK;
}

extern "C" {

lfem_status lfem_set_allocator(lfem_alloc_fn alloc, lfem_free_fn dealloc, void* ctx) {
    if ((alloc == nullptr) != (dealloc == nullptr))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "allocator hook: alloc and dealloc must both be set or both be NULL");
    std::lock_guard<std::mutex> lk(g_hook_mu);
    g_hook.alloc = alloc;
    g_hook.dealloc = dealloc;
    g_hook.ctx = ctx;
    return LFEM_OK;
}

const char* lfem_last_error(void) { return g_err.c_str(); }
int64_t lfem_error_element(void) { return g_err_elem; }
const char* lfem_version(void) { return "lfem 0.1 (sm_100a, fp64)"; }

lfem_status lfem_mesh_create(lfem_domain dom, int order, lfem_quad quad, int64_t n_nodes, const double* coords,
                             int64_t n_elems, const int32_t* conn, lfem_stream_t stream, lfem_mesh* out) {
    g_err.clear();
    g_err_elem = -1;
    if (!out) return lfem_fail(LFEM_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (dom != LFEM_SURFACE_TRI && dom != LFEM_BULK_TET && dom != LFEM_SURFACE_LINE)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "domain");
    if (order != 1 && order != 2) return lfem_fail(LFEM_ERR_UNSUPPORTED, "order must be 1 or 2");
    int q = quad;
    if (q == LFEM_QUAD_DEFAULT) {
        if (dom == LFEM_SURFACE_LINE) q = order == 1 ? LFEM_QUAD_LINE2_DEG3 : LFEM_QUAD_LINE3_DEG5;
        else if (dom == LFEM_SURFACE_TRI) q = order == 1 ? LFEM_QUAD_TRI3_DEG2 : LFEM_QUAD_TRI6_DEG4;
        else q = order == 1 ? LFEM_QUAD_TET4_DEG2 : LFEM_QUAD_TET11_DEG4;
    }
    // each family runs with the rule its constant tables were built for
    const int fam = family_of(dom, order, q);
    const int want[N_FAMILIES] = {LFEM_QUAD_TRI3_DEG2,  LFEM_QUAD_TRI6_DEG4,  LFEM_QUAD_TET4_DEG2,
                                  LFEM_QUAD_TET11_DEG4, LFEM_QUAD_TRI16_DEG8, LFEM_QUAD_LINE2_DEG3,
                                  LFEM_QUAD_LINE3_DEG5, LFEM_QUAD_TET35_DEG7, LFEM_QUAD_LINE6_DEG11};
    if (q != want[fam])
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "quadrature rule not available for this (domain, order)");
    if (n_nodes < 0 || n_elems < 0 || n_nodes >= INT_MAX || n_elems >= INT_MAX)
        return lfem_fail(LFEM_ERR_INVALID_ARG, "n_nodes / n_elems out of range");
    if ((n_nodes > 0 && !coords) || (n_elems > 0 && !conn))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "coords / conn is NULL");
    if ((reinterpret_cast<uintptr_t>(coords) & 7) || (reinterpret_cast<uintptr_t>(conn) & 3))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "coords must be 8-byte and conn 4-byte aligned");
    static const int nrefs[N_FAMILIES] = {3, 6, 4, 10, 6, 2, 3, 10, 3};
    static const int nqs[N_FAMILIES] = {3, 6, 4, 11, 16, 2, 3, 35, 6};
    static const int nsyms[N_FAMILIES] = {6, 21, 10, 55, 21, 3, 6, 55, 6};
    lfem_mesh_s* m = new (std::nothrow) lfem_mesh_s();
    if (!m) return lfem_fail(LFEM_ERR_NOMEM, "host allocation");
    m->domain = dom;
    m->order = order;
    m->quad = q;
    m->family = fam;
    m->nref = nrefs[fam];
    m->nq = nqs[fam];
    m->nsym = nsyms[fam];
    m->n_nodes = n_nodes;
    m->n_elems = n_elems;
    m->coords = coords;
    m->conn = conn;
    if (n_elems > 0) {
        int* bad = nullptr;
        lfem_status st = dev_alloc_t(&bad, 1, S(stream));
        if (st != LFEM_OK) { delete m; return st; }
        const int init = INT_MAX;
        cudaError_t e = cudaMemcpyAsync(bad, &init, sizeof(int), cudaMemcpyHostToDevice, S(stream));
        if (e == cudaSuccess) {
            st = check_conn_launch(conn, n_elems, m->nref, n_nodes, bad, S(stream));
        } else {
            st = lfem_cuda_fail(e, "cudaMemcpyAsync");
        }
        int hbad = INT_MAX;
        if (st == LFEM_OK) {
            e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, S(stream));
            if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
            if (e != cudaSuccess) st = lfem_cuda_fail(e, "mesh index check");
        }
        dev_free(bad, S(stream));
        if (st != LFEM_OK) { delete m; return st; }
        if (hbad != INT_MAX) {
            delete m;
            return lfem_fail(LFEM_ERR_INDEX, "connectivity entry outside [0, n_nodes)", hbad);
        }
    }
    *out = m;
    return LFEM_OK;
}

void lfem_mesh_destroy(lfem_mesh m) { delete m; }

lfem_status lfem_assemble_symbolic(lfem_mesh m, int64_t row_begin, int64_t row_end, lfem_stream_t stream,
                                   lfem_plan* out) {
    g_err.clear();
    g_err_elem = -1;
    if (!m || !out) return lfem_fail(LFEM_ERR_INVALID_ARG, "mesh / out is NULL");
    *out = nullptr;
    if (row_begin < 0 || row_end < row_begin || row_end > m->n_nodes)
        return lfem_fail(LFEM_ERR_INVALID_ARG, "row range must satisfy 0 <= row_begin <= row_end <= n_nodes");
    lfem_plan_s* p = new (std::nothrow) lfem_plan_s();
    if (!p) return lfem_fail(LFEM_ERR_NOMEM, "host allocation");
    p->mesh = m;
    p->row_begin = row_begin;
    p->row_end = row_end;
    lfem_status st = dev_alloc_t(&p->err, 1, S(stream));
    if (st == LFEM_OK) {
        const int init = INT_MAX;
        cudaError_t e = cudaMemcpyAsync(p->err, &init, sizeof(int), cudaMemcpyHostToDevice, S(stream));
        if (e != cudaSuccess) st = lfem_cuda_fail(e, "cudaMemcpyAsync");
    }
    if (st == LFEM_OK) st = build_symbolic(p, S(stream));
    if (st == LFEM_OK) st = plan_mark(p, S(stream));
    if (st != LFEM_OK) {
        cudaStreamSynchronize(S(stream));
        free_plan_memory(p);
        cudaStreamSynchronize(nullptr);
        delete p;
        return st;
    }
    *out = p;
    return LFEM_OK;
}

void lfem_plan_destroy(lfem_plan p) {
    if (!p) return;
    // wait for the work enqueued on this plan (one event per stream it ran on), not the device
    for (auto& d : p->done) {
        cudaEventSynchronize(d.second);
        cudaEventDestroy(d.second);
    }
    p->done.clear();
    free_plan_memory(p);
    cudaStreamSynchronize(nullptr);  // the frees above were ordered on the legacy stream
    delete p;
}

lfem_status lfem_plan_info(lfem_plan p, int64_t* n_rows, int64_t* nnz, int64_t* n_elems_local) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (n_rows) *n_rows = p->n_rows;
    if (nnz) *nnz = p->nnz;
    if (n_elems_local) *n_elems_local = p->n_local;
    return LFEM_OK;
}

lfem_status lfem_plan_set_variant(lfem_plan p, lfem_numeric_variant v) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (v != LFEM_NUMERIC_AUTO && v != LFEM_NUMERIC_V0 && v != LFEM_NUMERIC_TILED && v != LFEM_NUMERIC_ROWS)
        return lfem_fail(LFEM_ERR_INVALID_ARG, "variant");
    p->variant = v;
    p->last_variant = -1;
    return LFEM_OK;
}

static bool misaligned(const void* q, uintptr_t a) { return (reinterpret_cast<uintptr_t>(q) & (a - 1)) != 0; }

static lfem_status check_numeric_args(lfem_plan p, unsigned kinds, const double* coeff, double* const vals[3]) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (misaligned(coeff, 8)) return lfem_fail(LFEM_ERR_INVALID_ARG, "coeff is not 8-byte aligned");
    if (vals)
        for (int k = 0; k < 3; ++k)
            if (((kinds >> k) & 1u) && misaligned(vals[k], 8))
                return lfem_fail(LFEM_ERR_INVALID_ARG, "vals[k] is not 8-byte aligned");
    if (kinds == 0 || (kinds & ~7u))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "kinds must be a nonzero subset of MASS|STIFF|STIFF_COEF");
    if ((kinds & LFEM_STIFF_COEF) && !coeff && p->mesh->n_nodes > 0)
        return lfem_fail(LFEM_ERR_INVALID_ARG, "LFEM_STIFF_COEF requires a coefficient (coeff is NULL)");
    if (!vals) return lfem_fail(LFEM_ERR_INVALID_ARG, "vals is NULL");
    for (int k = 0; k < 3; ++k) {
        const bool want = (kinds >> k) & 1u;
        if (want && !vals[k] && p->nnz > 0)
            return lfem_fail(LFEM_ERR_INVALID_ARG, "vals[k] is NULL for a requested kind");
    }
    return LFEM_OK;
}

lfem_status lfem_assemble_numeric(lfem_plan p, unsigned kinds, const double* coeff, double* const vals[3],
                                  lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    LFEM_TRY(check_numeric_args(p, kinds, coeff, vals));
    double* v[3];
    for (int k = 0; k < 3; ++k) v[k] = ((kinds >> k) & 1u) ? vals[k] : nullptr;
    LFEM_TRY(numeric_dispatch(p, kinds, p->mesh->coords, coeff, v, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_assemble_numeric_coords(lfem_plan p, unsigned kinds, const double* coords, const double* coeff,
                                         double* const vals[3], lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    LFEM_TRY(check_numeric_args(p, kinds, coeff, vals));
    if (!coords && p->mesh->n_nodes > 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "coords is NULL");
    if (misaligned(coords, 8)) return lfem_fail(LFEM_ERR_INVALID_ARG, "coords is not 8-byte aligned");
    double* v[3];
    for (int k = 0; k < 3; ++k) v[k] = ((kinds >> k) & 1u) ? vals[k] : nullptr;
    LFEM_TRY(numeric_dispatch(p, kinds, coords, coeff, v, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_assemble_numeric_host(lfem_plan p, unsigned kinds, const double* coords_h, const double* coeff_h,
                                       double* const vals_h[3], lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    LFEM_TRY(check_numeric_args(p, kinds, coeff_h, vals_h));
    cudaStream_t s = S(stream);
    const int64_t nn = p->mesh->n_nodes;
    const double* coords = p->mesh->coords;
    if (coords_h && nn > 0) {
        if (!p->d_coords) LFEM_TRY(dev_alloc_t(&p->d_coords, (size_t)nn * 3, s));
        LFEM_CUDA(cudaMemcpyAsync(p->d_coords, coords_h, sizeof(double) * nn * 3, cudaMemcpyHostToDevice, s));
        coords = p->d_coords;
    }
    const double* coeff = nullptr;
    if ((kinds & LFEM_STIFF_COEF) && nn > 0) {
        if (!p->d_coeff) LFEM_TRY(dev_alloc_t(&p->d_coeff, (size_t)nn, s));
        LFEM_CUDA(cudaMemcpyAsync(p->d_coeff, coeff_h, sizeof(double) * nn, cudaMemcpyHostToDevice, s));
        coeff = p->d_coeff;
    }
    double* v[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < 3; ++k)
        if ((kinds >> k) & 1u) {
            if (!p->d_vals[k]) LFEM_TRY(dev_alloc_t(&p->d_vals[k], (size_t)p->nnz, s));
            v[k] = p->d_vals[k];
        }
    LFEM_TRY(numeric_dispatch(p, kinds, coords, coeff, v, s));
    LFEM_TRY(plan_mark(p, s));
    for (int k = 0; k < 3; ++k)
        if (((kinds >> k) & 1u) && p->nnz > 0)
            LFEM_CUDA(cudaMemcpyAsync(vals_h[k], v[k], sizeof(double) * p->nnz, cudaMemcpyDeviceToHost, s));
    return lfem_plan_check(p, stream);
}

lfem_status lfem_csr_get(lfem_plan p, const int64_t** row_ptr, const int32_t** col_idx) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (row_ptr) *row_ptr = p->row_ptr;
    if (col_idx) *col_idx = p->col_idx;
    return LFEM_OK;
}

lfem_status lfem_spmv(lfem_plan p, const double* vals, const double* x_full, double* y_rows, lfem_stream_t stream) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if ((p->nnz > 0 && !vals) || (p->n_rows > 0 && (!x_full || !y_rows)))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "NULL vector");
    LFEM_TRY(spmv_launch(p, vals, x_full, y_rows, S(stream)));
    return plan_mark(p, S(stream));
}

int lfem_rhs_ncomp(int kind) { return kind == LFEM_RHS_LOAD ? 1 : kind == LFEM_RHS_KLL ? 4 : 0; }

int lfem_rhs_launches(lfem_plan p, int kind) {
    if (!p || lfem_rhs_ncomp(kind) == 0) return 0;
    return rhs_launch_count(p);
}

lfem_status lfem_assemble_rhs(lfem_plan p, int kind, const double* coords, const double* u, double* out,
                              lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (lfem_rhs_ncomp(kind) == 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "kind must be LFEM_RHS_LOAD or LFEM_RHS_KLL");
    if (kind == LFEM_RHS_KLL && p->mesh->domain != LFEM_SURFACE_TRI)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "the KLL right-hand side is defined on surfaces only");
    if (!u && p->mesh->n_nodes > 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "u is NULL");
    if (!out && p->n_rows > 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "out is NULL");
    if (misaligned(coords, 8) || misaligned(u, 8) || misaligned(out, 8))
        return lfem_fail(LFEM_ERR_INVALID_ARG, "coords / u / out is not 8-byte aligned");
    LFEM_TRY(rhs_dispatch(p, kind, coords ? coords : p->mesh->coords, u, out, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_cg_solve(lfem_plan p, const double* vals_K, const double* b, double* x, double tol, int max_it,
                          int* iters, lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (p->n_rows > 0 && (!vals_K || !b || !x)) return lfem_fail(LFEM_ERR_INVALID_ARG, "NULL argument");
    if (!(tol > 0.0) || max_it < 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "tol must be > 0 and max_it >= 0");
    LFEM_TRY(cg_solve(p, vals_K, b, x, tol, max_it, iters, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_solve_meanfree(lfem_plan p, const double* vals_A, const double* b, double* u, double tol,
                                int max_it, int* iters, lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (p->n_rows > 0 && (!vals_A || !b || !u)) return lfem_fail(LFEM_ERR_INVALID_ARG, "NULL argument");
    if (!(tol > 0.0) || max_it < 0) return lfem_fail(LFEM_ERR_INVALID_ARG, "tol must be > 0 and max_it >= 0");
    LFEM_TRY(solve_meanfree(p, vals_A, b, u, tol, max_it, iters, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_mcf_step(lfem_plan p, double tau, const double* x_prev, double* x_next, double tol, int max_it,
                          int* iters, lfem_stream_t stream) {
    g_err.clear();
    g_err_elem = -1;
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (p->mesh->domain != LFEM_SURFACE_TRI)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "Dziuk's MCF step is defined for surfaces");
    if (p->n_rows > 0 && (!x_prev || !x_next)) return lfem_fail(LFEM_ERR_INVALID_ARG, "NULL argument");
    if (!(tau > 0.0) || !(tol > 0.0) || max_it < 0)
        return lfem_fail(LFEM_ERR_INVALID_ARG, "tau and tol must be > 0, max_it >= 0");
    LFEM_TRY(mcf_step(p, tau, x_prev, x_next, tol, max_it, iters, S(stream)));
    return plan_mark(p, S(stream));
}

lfem_status lfem_plan_check(lfem_plan p, lfem_stream_t stream) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    int h = INT_MAX;
    LFEM_CUDA(cudaStreamSynchronize(S(stream)));
    LFEM_CUDA(cudaMemcpy(&h, p->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (h != INT_MAX) {
        // surfaced once: clear the latch so later calls on the plan (e.g. valid moving
        // coordinates) report their own state
        const int init = INT_MAX;
        LFEM_CUDA(cudaMemcpy(p->err, &init, sizeof(int), cudaMemcpyHostToDevice));
        return lfem_fail(LFEM_ERR_DEGENERATE, "degenerate element (mu <= 0 or non-finite at a quadrature point)", h);
    }
    return LFEM_OK;
}

lfem_status lfem_axpby(int64_t n, double ca, const double* a, double cb, const double* b, double* out,
                       lfem_stream_t stream) {
    if (n < 0 || (n > 0 && (!a || !b || !out))) return lfem_fail(LFEM_ERR_INVALID_ARG, "axpby arguments");
    return axpby_launch(n, ca, a, cb, b, out, S(stream));
}

lfem_status lfem_profile_enable(lfem_plan p, int enable) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    if (!p->prof) p->prof = new (std::nothrow) Profiler();
    if (!p->prof) return lfem_fail(LFEM_ERR_NOMEM, "host allocation");
    p->prof->on = enable != 0;
    return LFEM_OK;
}

lfem_status lfem_profile_read(lfem_plan p, int max, const char** names, double* ms, int64_t* launches, int* n) {
    if (!p || !n) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan / n is NULL");
    *n = 0;
    if (!p->prof) return LFEM_OK;
    Profiler& P = *p->prof;
    P.collect();
    int k = 0;
    for (size_t i = 0; i < P.names.size() && k < max; ++i, ++k) {
        if (names) names[k] = P.names[i];
        if (ms) ms[k] = P.ms[i];
        if (launches) launches[k] = P.count[i];
        P.ms[i] = 0.0;
        P.count[i] = 0;
    }
    *n = k;
    return LFEM_OK;
}

lfem_status lfem_numeric_stats(lfem_plan p, int64_t* elem_evals, int64_t* n_tiles) {
    if (!p) return lfem_fail(LFEM_ERR_INVALID_ARG, "plan is NULL");
    const bool tiled = p->last_variant == LFEM_NUMERIC_TILED && p->tiled_ok == 1;
    if (elem_evals) *elem_evals = tiled ? p->tiles.total_elems : p->n_local;
    if (n_tiles) *n_tiles = tiled ? p->tiles.n_tiles : 0;
    return LFEM_OK;
}

int lfem_numeric_launches(lfem_plan p, unsigned kinds) {
    if (!p) return -1;
    return numeric_launch_count(p, kinds);
}

}  // extern "C"

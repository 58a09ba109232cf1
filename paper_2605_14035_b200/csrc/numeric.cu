// Numeric phase of the ℓFEM assembly on B200 (sm_100a), fp64.
//
// Per element (Listing 1 P:581-609 and §3.2):
//   gather the nref node coordinates (Listing 1 l.12),
//   J(xi_q) = sum_{j>=2} (x_j - x_1) grad_ref phi_j(xi_q)^T  (Eq. jacobian_inv P:317-327,
//             differences: reading G24),
//   surface: G = J^T J, mu = sqrt(det G) (= |t1 x t2|, Listing 1 l.16-17),
//            K_q = w_q mu G^{-1} (metric form of Eq. Aloc-precise P:337 with C = L^{-1}
//            read as Listing 1, reading G2), A_loc(a,b) += grad_a^T K_q grad_b;
//   bulk:    mu = |det J|, g_a = J^{-T} grad_a = cof(J) grad_a / det J,
//            A_loc(a,b) += (w_q / mu) (cof grad_a).(cof grad_b);
//   M_loc(a,b) += w_q mu phi_a phi_b                      (Eq. reference_quadrature_mass),
//   A_a,loc(a,b) += a(u_h(xi_q)) * (stiffness integrand),
//            u_h(xi_q) = sum_c u_c phi_c(xi_q), a(u) = 1 + u^2 (north_star, reading G10).
// Only the symmetric half (a <= b) is computed.  Reduction into CSR follows
// the plan built by symbolic.cu: every slot sums its contributions in
// ascending (element, a, b) order (reading G21) -- no atomics.
//
// Variants:
//   V0     k_elem_v0 (thread per element -> staged local matrices in HBM)
//          + k_slot_reduce (thread per CSR slot).
//   TILED  see numeric_tiled.cuh.
#include <climits>
#include <mutex>

#include "lfem_internal.cuh"
#include "reference.cuh"
#include "element.cuh"

#ifndef LFEM_V0_TET_MINB
#define LFEM_V0_TET_MINB 1
#endif

namespace {

template <int F> struct V0Cfg { static constexpr int MINB = 1; };
template <> struct V0Cfg<FAM_TET_P2> { static constexpr int MINB = LFEM_V0_TET_MINB; };
template <> struct V0Cfg<FAM_TET_P2_Q35> { static constexpr int MINB = 1; };

// --------------------------------------------------------------------------
// V0: element kernel -> stage[k][s][le]; slot kernel -> vals
// --------------------------------------------------------------------------
// V0 stage, element-major: stage[(le * NS + s) * NK + kr] (kr = rank of the kind among the
// requested ones), so one contribution's values of all kinds are one vector and the
// contributions of a CSR row come from a few contiguous element blocks.  Each warp
// assembles its 32 consecutive elements' blocks in shared memory and writes them as
// one contiguous range with 16-B stores (a direct per-thread store would scatter
// every warp store instruction over 32 blocks: LSU-throttled, partial sectors).
struct SmemStageSink {
    double* sm;  // this thread's block, already offset by kr
    int nk;
    __device__ __forceinline__ void operator()(int s, double v) const { sm[s * nk] = v; }
};

constexpr int V0_THREADS = 128;

template <int F, bool DM, bool DA, bool DAA>
constexpr int v0_block_doubles() {
    return FamInfo<F>::NSYM * ((DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0));
}

template <int F, bool DM, bool DA, bool DAA>
__global__ void __launch_bounds__(V0_THREADS, V0Cfg<F>::MINB)
k_elem_v0(int64_t n_local, const int32_t* __restrict__ lconn, const int32_t* __restrict__ elem_list,
          const double* __restrict__ coords, const double* __restrict__ coeff, double* __restrict__ stage,
          int* __restrict__ err) {
    using E = Elem<F>;
    constexpr int N = E::N, NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
    constexpr int BD = v0_block_doubles<F, DM, DA, DAA>();  // doubles per element block (even)
    extern __shared__ __align__(16) double v0_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wsm = v0_smem + (size_t)warp * 32 * BD;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t le0 = blockIdx.x * (int64_t)blockDim.x + warp * 32; le0 < n_local; le0 += stride) {
        const int64_t le = le0 + lane;
        const int nvalid = n_local - le0 < 32 ? (int)(n_local - le0) : 32;
        if (le < n_local) {
            double X[N][3], U[N];
#pragma unroll
            for (int a = 0; a < N; ++a) {
                const int64_t v = __ldg(&lconn[le * N + a]);
#pragma unroll
                for (int c = 0; c < 3; ++c) X[a][c] = __ldg(&coords[3 * v + c]);
                U[a] = DAA ? __ldg(&coeff[v]) : 0.0;
            }
            typename E::Geo g;
            if (!E::template geometry<DAA>(X, U, g)) atomicMin(err, __ldg(&elem_list[le]));
            double* my = wsm + lane * BD;
            int kr = 0;
            if (DM) {
                SmemStageSink sink{my + kr++, NK};
                E::template kind<KIND_M>(g, sink);
            }
            if (DA) {
                SmemStageSink sink{my + kr++, NK};
                E::template kind<KIND_A>(g, sink);
            }
            if (DAA) {
                SmemStageSink sink{my + kr++, NK};
                E::template kind<KIND_AA>(g, sink);
            }
        }
        __syncwarp();
        // contiguous copy of the warp's nvalid blocks (le0 is a multiple of 32: 16-B aligned)
        const double2* src = reinterpret_cast<const double2*>(wsm);
        double2* dst = reinterpret_cast<double2*>(stage + le0 * BD);
        const int nd = nvalid * BD, n2 = nd / 2;
        for (int i = lane; i < n2; i += 32) dst[i] = src[i];
        if ((nd & 1) && lane == 0) stage[le0 * BD + nd - 1] = wsm[nd - 1];
        __syncwarp();
    }
}

// thread per CSR slot; contributions in plan order (ascending element, then (a, b): G21)
// LFEM_V0_KS > 1: each thread owns KS slots (blockDim apart, so the warp's
// accesses stay coalesced); the first LFEM_V0_U2 contributions of all KS slots are loaded
// together, predicated (KS * U2 independent gathers in flight per thread: most slots have
// <= 4 contributions), the rest of each slot in the usual loops.  The order within a slot
// is unchanged.  Measured (C4 reduce, ms): KS,U2 = 1,- 2.89 | 2,2 2.85 | 2,4 2.67 | 2,3 3.08
// | 2,6 3.49 | 2,8 3.00 | 3,2 3.12 | 4,2 3.22.
#ifndef LFEM_V0_KS
#define LFEM_V0_KS 2
#endif
#ifndef LFEM_V0_U2
#define LFEM_V0_U2 4
#endif
template <bool DM, bool DA, bool DAA>
__global__ void __launch_bounds__(256)
k_slot_reduce(int64_t nnz, const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ codes,
              const double* __restrict__ stage, double* __restrict__ vm, double* __restrict__ va,
              double* __restrict__ vaa) {
    constexpr int NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
    constexpr int KS = LFEM_V0_KS;
    [[maybe_unused]] constexpr int U2 = LFEM_V0_U2;  // contributions per slot gathered in the joint first round
    const int64_t per_block = (int64_t)blockDim.x * KS;
    for (int64_t base = blockIdx.x * per_block + threadIdx.x; base < nnz; base += (int64_t)gridDim.x * per_block) {
        int jb[KS], je[KS];
        double acc[KS][NK];
#pragma unroll
        for (int q = 0; q < KS; ++q) {
            const int64_t s = base + (int64_t)q * blockDim.x;
            jb[q] = je[q] = 0;
            if (s < nnz) {
                jb[q] = __ldg(&slot_ptr[s]);
                je[q] = __ldg(&slot_ptr[s + 1]);
            }
#pragma unroll
            for (int k = 0; k < NK; ++k) acc[q][k] = 0.0;
        }
        if constexpr (KS > 1) {
            int c2[KS][U2];
#pragma unroll
            for (int q = 0; q < KS; ++q)
#pragma unroll
                for (int u = 0; u < U2; ++u) c2[q][u] = (jb[q] + u < je[q]) ? __ldg(&codes[jb[q] + u]) : -1;
            double w2[KS][U2][NK];
#pragma unroll
            for (int q = 0; q < KS; ++q)
#pragma unroll
                for (int u = 0; u < U2; ++u) {
                    if constexpr (NK == 2) {
                        double2 w = make_double2(0.0, 0.0);
                        if (c2[q][u] >= 0) w = __ldg(reinterpret_cast<const double2*>(stage + (int64_t)c2[q][u] * 2));
                        w2[q][u][0] = w.x;
                        w2[q][u][1] = w.y;
                    } else {
#pragma unroll
                        for (int k = 0; k < NK; ++k)
                            w2[q][u][k] = c2[q][u] >= 0 ? __ldg(stage + (int64_t)c2[q][u] * NK + k) : 0.0;
                    }
                }
#pragma unroll
            for (int q = 0; q < KS; ++q) {
#pragma unroll
                for (int u = 0; u < U2; ++u)
                    if (c2[q][u] >= 0) {
#pragma unroll
                        for (int k = 0; k < NK; ++k) acc[q][k] += w2[q][u][k];
                    }
                jb[q] = min(jb[q] + U2, je[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < KS; ++q) {
            const int j1 = je[q];
            // four contributions' loads in flight, accumulated in plan order
            int j = jb[q];
            for (; j + 4 <= j1; j += 4) {
                int c4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) c4[u] = __ldg(&codes[j + u]);
                if constexpr (NK == 2) {
                    double2 w4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) w4[u] = __ldg(reinterpret_cast<const double2*>(stage + (int64_t)c4[u] * 2));
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        acc[q][0] += w4[u].x;
                        acc[q][1] += w4[u].y;
                    }
                } else {
                    double w4[4][NK];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < NK; ++k) w4[u][k] = __ldg(stage + (int64_t)c4[u] * NK + k);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < NK; ++k) acc[q][k] += w4[u][k];
                }
            }
            for (; j < j1; ++j) {
                const double* p = stage + (int64_t)__ldg(&codes[j]) * NK;
                if constexpr (NK == 2) {
                    const double2 w = __ldg(reinterpret_cast<const double2*>(p));
                    acc[q][0] += w.x;
                    acc[q][1] += w.y;
                } else {
#pragma unroll
                    for (int k = 0; k < NK; ++k) acc[q][k] += __ldg(p + k);
                }
            }
            const int64_t s = base + (int64_t)q * blockDim.x;
            if (s < nnz) {
                int kr = 0;
                if (DM) vm[s] = acc[q][kr++];
                if (DA) va[s] = acc[q][kr++];
                if (DAA) vaa[s] = acc[q][kr++];
            }
        }
    }
}

inline unsigned grid_for(int64_t n, int threads, int max_blocks) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (unsigned)g;
}

template <int F, bool DM, bool DA, bool DAA>
lfem_status run_v0(lfem_plan_s* p, const double* coords, const double* coeff, double* const vals[3], cudaStream_t s) {
    constexpr int NS = FamInfo<F>::NSYM;
    if (!p->stage) LFEM_TRY(dev_alloc_t(&p->stage, (size_t)3 * NS * p->n_local + 1, s));
    if (p->n_local > 0) {
        prof_begin(p, "k_elem_v0", s);
        constexpr int BD = v0_block_doubles<F, DM, DA, DAA>();
        constexpr size_t smem = sizeof(double) * (size_t)V0_THREADS * BD;
        LFEM_TRY(ensure_smem_attr(reinterpret_cast<const void*>(k_elem_v0<F, DM, DA, DAA>), (int)smem));
        k_elem_v0<F, DM, DA, DAA><<<grid_for(p->n_local, V0_THREADS, 1 << 20), V0_THREADS, smem, s>>>(
            p->n_local, p->local_conn, p->elem_list, coords, coeff, p->stage, p->err);
        LFEM_CUDA(cudaGetLastError());
        prof_end(p, s);
    }
    if (p->nnz > 0) {
        prof_begin(p, "k_slot_reduce", s);
        k_slot_reduce<DM, DA, DAA><<<grid_for(p->nnz, 256 * LFEM_V0_KS, 1 << 20), 256, 0, s>>>(
            p->nnz, p->slot_ptr, p->codes, p->stage, vals[0], vals[1], vals[2]);
        LFEM_CUDA(cudaGetLastError());
        prof_end(p, s);
    }
    return LFEM_OK;
}

template <int F>
lfem_status dispatch_kinds(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                           double* const vals[3], cudaStream_t s) {
    switch (kinds) {
    case 1: return run_v0<F, true, false, false>(p, coords, coeff, vals, s);
    case 2: return run_v0<F, false, true, false>(p, coords, coeff, vals, s);
    case 3: return run_v0<F, true, true, false>(p, coords, coeff, vals, s);
    case 4: return run_v0<F, false, false, true>(p, coords, coeff, vals, s);
    case 5: return run_v0<F, true, false, true>(p, coords, coeff, vals, s);
    case 6: return run_v0<F, false, true, true>(p, coords, coeff, vals, s);
    case 7: return run_v0<F, true, true, true>(p, coords, coeff, vals, s);
    default: return lfem_fail(LFEM_ERR_INVALID_ARG, "kinds must be a nonzero subset of MASS|STIFF|STIFF_COEF");
    }
}

// --------------------------------------------------------------------------
// misc kernels
// --------------------------------------------------------------------------
__global__ void k_check_conn(const int32_t* __restrict__ conn, int64_t n_elems, int nref, int64_t n_nodes,
                             int* __restrict__ bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elems;
         e += (int64_t)gridDim.x * blockDim.x) {
        bool ok = true;
        for (int a = 0; a < nref; ++a) {
            const int64_t v = conn[e * nref + a];
            ok &= (v >= 0) & (v < n_nodes);
        }
        if (!ok) atomicMin(bad, (int)e);
    }
}

__global__ void k_spmv(int64_t n_rows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                       const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y) {
    // one warp per row; lanes stride the row, fixed-order tree reduction
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < n_rows; r += nw) {
        double acc = 0.0;
        for (int64_t j = row_ptr[r] + lane; j < row_ptr[r + 1]; j += 32) acc = fma(vals[j], x[col[j]], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) y[r] = acc;
    }
}

__global__ void k_axpby(int64_t n, double ca, const double* __restrict__ a, double cb, const double* __restrict__ b,
                        double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = ca * a[i] + cb * b[i];
}

std::mutex g_tab_mu;
uint64_t g_tab_devices = 0;  // bit per device with uploaded tables

}  // namespace

#include "numeric_tiled.cuh"

lfem_status rows_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                          double* const vals[3], cudaStream_t s, bool* ok);  // rows.cuh

// AUTO: TILED for triangles, V0 for tetrahedra (measured; ROWS is opt-in)
static int auto_variant(lfem_plan_s* p) { return tiled_default_variant(p); }

lfem_status upload_reference_tables() {
    int dev = 0;
    LFEM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_tab_mu);
    if (dev < 64 && (g_tab_devices >> dev) & 1ull) return LFEM_OK;
    static RefTab<FAM_TRI_P1> t1;
    static RefTab<FAM_TRI_P2> t2;
    static RefTab<FAM_TET_P1> t3;
    static RefTab<FAM_TET_P2> t4;
    static RefTab<FAM_TRI_P2_Q16> t5;
    static RefTab<FAM_LINE_P1> t6;
    static RefTab<FAM_LINE_P2> t7;
    static RefTab<FAM_TET_P2_Q35> t8;
    static RefTab<FAM_LINE_P2_Q6> t9;
    refhost::fill(t1, refhost::rule_tri3(), 2, 1);
    refhost::fill(t2, refhost::rule_tri6(), 2, 2);
    refhost::fill(t3, refhost::rule_tet4(), 3, 1);
    refhost::fill(t4, refhost::rule_tet11(), 3, 2);
    refhost::fill(t5, refhost::rule_tri16(), 2, 2);
    refhost::fill(t6, refhost::rule_line(2), 1, 1);
    refhost::fill(t7, refhost::rule_line(3), 1, 2);
    refhost::fill(t8, refhost::rule_tet35(), 3, 2);
    refhost::fill(t9, refhost::rule_line(6), 1, 2);
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tri1, &t1, sizeof(t1)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tri2, &t2, sizeof(t2)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tet1, &t3, sizeof(t3)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tet2, &t4, sizeof(t4)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tri2q, &t5, sizeof(t5)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_line1, &t6, sizeof(t6)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_line2, &t7, sizeof(t7)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_tet2q, &t8, sizeof(t8)));
    LFEM_CUDA(cudaMemcpyToSymbol(c_tab_line2q, &t9, sizeof(t9)));
    static QuadXi xi[N_FAMILIES] = {};
    static const refhost::Rule rules[N_FAMILIES] = {refhost::rule_tri3(),  refhost::rule_tri6(),   refhost::rule_tet4(),
                                                    refhost::rule_tet11(), refhost::rule_tri16(),  refhost::rule_line(2),
                                                    refhost::rule_line(3), refhost::rule_tet35(), refhost::rule_line(6)};
    for (int f = 0; f < N_FAMILIES; ++f)
        for (int q = 0; q < rules[f].nq; ++q)
            for (int m = 0; m < 3; ++m) xi[f].xi[q][m] = rules[f].xi[q][m];
    LFEM_CUDA(cudaMemcpyToSymbol(c_xi, xi, sizeof(xi)));
    if (dev < 64) g_tab_devices |= (1ull << dev);
    return LFEM_OK;
}

lfem_status check_conn_launch(const int32_t* conn, int64_t n_elems, int nref, int64_t n_nodes, int* bad,
                              cudaStream_t s) {
    if (n_elems == 0) return LFEM_OK;
    k_check_conn<<<grid_for(n_elems, 256, 148 * 32), 256, 0, s>>>(conn, n_elems, nref, n_nodes, bad);
    LFEM_CUDA(cudaGetLastError());
    return LFEM_OK;
}

lfem_status numeric_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                             double* const vals[3], cudaStream_t s) {
    LFEM_TRY(upload_reference_tables());
    const int fam = p->mesh->family;
    const bool autov = p->variant == LFEM_NUMERIC_AUTO;
    int variant = autov ? auto_variant(p) : p->variant;
    if (variant == LFEM_NUMERIC_TILED) {
        // the tile kernel moves coords / coeff with cp.async.bulk (16-byte aligned sources) and
        // stores value pairs with 16-byte vector stores
        uintptr_t al = reinterpret_cast<uintptr_t>(coords) | reinterpret_cast<uintptr_t>(coeff);
        for (int k = 0; k < 3; ++k) al |= reinterpret_cast<uintptr_t>(vals[k]);
        const bool aligned = (al & 15) == 0;
        if (!aligned && !autov)
            return lfem_fail(LFEM_ERR_INVALID_ARG, "the TILED variant needs 16-byte aligned coords, coeff and vals");
        if (aligned && !(autov && p->tiled_ok == 0)) {
            const lfem_status st = tiled_dispatch(p, kinds, coords, coeff, vals, s);
            if (st == LFEM_OK) {
                p->last_variant = LFEM_NUMERIC_TILED;
                return LFEM_OK;
            }
            // AUTO: a mesh the tile plan cannot hold (e.g. a very high-valence row) runs V0
            if (!(autov && st == LFEM_ERR_UNSUPPORTED && p->tiled_ok == 0)) return st;
        }
        variant = LFEM_NUMERIC_V0;
    }
    if (variant == LFEM_NUMERIC_ROWS) {
        bool ok = false;
        LFEM_TRY(rows_dispatch(p, kinds, coords, coeff, vals, s, &ok));
        if (ok) {
            p->last_variant = LFEM_NUMERIC_ROWS;
            return LFEM_OK;  // else: a row longer than the ROWS lanes hold -> V0
        }
    }
    p->last_variant = LFEM_NUMERIC_V0;
    switch (fam) {
    case FAM_TRI_P1: return dispatch_kinds<FAM_TRI_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2: return dispatch_kinds<FAM_TRI_P2>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2_Q16: return dispatch_kinds<FAM_TRI_P2_Q16>(p, kinds, coords, coeff, vals, s);
    case FAM_LINE_P1: return dispatch_kinds<FAM_LINE_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_LINE_P2: return dispatch_kinds<FAM_LINE_P2>(p, kinds, coords, coeff, vals, s);
    case FAM_LINE_P2_Q6: return dispatch_kinds<FAM_LINE_P2_Q6>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P2_Q35: return dispatch_kinds<FAM_TET_P2_Q35>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P1: return dispatch_kinds<FAM_TET_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P2: return dispatch_kinds<FAM_TET_P2>(p, kinds, coords, coeff, vals, s);
    }
    return lfem_fail(LFEM_ERR_UNSUPPORTED, "family");
}

int numeric_launch_count(lfem_plan_s* p, unsigned kinds) {
    (void)kinds;
    int variant = p->last_variant >= 0 ? p->last_variant
                                       : p->variant == LFEM_NUMERIC_AUTO ? auto_variant(p) : p->variant;
    if (variant == LFEM_NUMERIC_TILED) return tiled_launch_count(p);
    if (variant == LFEM_NUMERIC_ROWS && p->rows_ok != 0) return p->n_rows > 0 ? 1 : 0;
    return (p->n_local > 0 ? 1 : 0) + (p->nnz > 0 ? 1 : 0);
}

lfem_status spmv_launch(lfem_plan_s* p, const double* vals, const double* x, double* y, cudaStream_t s) {
    if (p->n_rows == 0) return LFEM_OK;
    k_spmv<<<grid_for(p->n_rows * 32, 256, 148 * 64), 256, 0, s>>>(p->n_rows, p->row_ptr, p->col_idx, vals, x, y);
    LFEM_CUDA(cudaGetLastError());
    return LFEM_OK;
}

lfem_status axpby_launch(int64_t n, double ca, const double* a, double cb, const double* b, double* out,
                         cudaStream_t s) {
    if (n == 0) return LFEM_OK;
    k_axpby<<<grid_for(n, 256, 148 * 16), 256, 0, s>>>(n, ca, a, cb, b, out);
    LFEM_CUDA(cudaGetLastError());
    return LFEM_OK;
}

#include "rhs.cuh"
#include "rows.cuh"

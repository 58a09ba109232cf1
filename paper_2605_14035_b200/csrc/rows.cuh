// ROWS numeric variant (opt-in): warp per CSR row, element values recomputed per incident
// row (tried for SURVEY.md §8(f) row N2, "P1 tets at scale").  Included at the end of
// numeric.cu after rhs.cuh (uses its row incidence lists).  Measured slower than V0 on
// C4P1 (2.4 vs 0.72 ms): the ~4x recompute of the tetrahedron geometry (per quadrature
// point J, cofactors, determinant) outweighs the traffic it saves.
//
// For cheap elements (P1: a few hundred flops) the two-pass V0 scheme moves far more bytes than
// the algorithmic minimum (the staged local matrices and the per-slot codes: ~2.4 GB against
// 0.32 GB on C4P1).  Here each row's warp walks the row's incident (element, a) entries in
// ascending element order (the plan's diagonal-slot lists, rhs_prepare), one lane per entry:
// the lane recomputes its element (Elem<F>, the same code as V0/TILED) and keeps row a of each
// kind; then every slot owner lane adds, entry by entry in order, the value whose column matches
// its slot.  Each slot thus sums its contributions in ascending element order -- the V0/TILED
// order (reading G21) with the same element arithmetic: bitwise identical results.  No stage,
// no codes: traffic = incidence lists + conn / coords gathers (L2) + CSR columns + values.

namespace {

constexpr int ROWS_WARPS = 4;  // warps per CTA
constexpr int ROWS_SPL = 2;    // slots per lane: rows up to 64 columns (larger rows: the V0 fallback)

template <int F, bool DM, bool DA, bool DAA>
struct RowsSink {
    double* dst;  // this lane's N values of one kind
    int a;
    __device__ __forceinline__ void operator()(int s, double v) const {
        constexpr int N = FamInfo<F>::NREF;
        // (sa, sb) of symmetric index s, a <= b (compile-time after unrolling)
        int sa = 0, rem = s;
        while (rem >= N - sa) {
            rem -= N - sa;
            ++sa;
        }
        const int sb = sa + rem;
        if (sa == a) dst[sb] = v;
        if (sb == a && sa != sb) dst[sa] = v;
    }
};

template <int F, bool DM, bool DA, bool DAA>
__global__ void __launch_bounds__(ROWS_WARPS * 32)
k_rows(int64_t n_rows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
       const int64_t* __restrict__ rptr, const int32_t* __restrict__ rcodes, const int32_t* __restrict__ lconn,
       const int32_t* __restrict__ elem_list, const double* __restrict__ coords, const double* __restrict__ coeff,
       double* __restrict__ vm, double* __restrict__ va, double* __restrict__ vaa, int* __restrict__ err) {
    using E = Elem<F>;
    constexpr int N = E::N, NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
    __shared__ double sv[ROWS_WARPS][32][NK][N];
    __shared__ int32_t snode[ROWS_WARPS][32][N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w0 = blockIdx.x * (int64_t)ROWS_WARPS + warp, nw = (int64_t)gridDim.x * ROWS_WARPS;
    for (int64_t i = w0; i < n_rows; i += nw) {
        const int64_t s0 = __ldg(&row_ptr[i]);
        const int len = (int)(__ldg(&row_ptr[i + 1]) - s0);
        int32_t col[ROWS_SPL];
        double acc[NK][ROWS_SPL];
#pragma unroll
        for (int t = 0; t < ROWS_SPL; ++t) {
            col[t] = lane + 32 * t < len ? __ldg(&col_idx[s0 + lane + 32 * t]) : -1;
#pragma unroll
            for (int k = 0; k < NK; ++k) acc[k][t] = 0.0;
        }
        const int64_t j0 = __ldg(&rptr[i]), j1 = __ldg(&rptr[i + 1]);
        for (int64_t cb = j0; cb < j1; cb += 32) {
            const int cnt = j1 - cb < 32 ? (int)(j1 - cb) : 32;
            if (lane < cnt) {
                const int32_t code = __ldg(&rcodes[cb + lane]);
                const int64_t le = code / N;
                const int a = code % N;
                double X[N][3], U[N];
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    const int32_t v = __ldg(&lconn[le * N + b]);
                    snode[warp][lane][b] = v;
#pragma unroll
                    for (int c = 0; c < 3; ++c) X[b][c] = __ldg(&coords[3 * (int64_t)v + c]);
                    U[b] = DAA ? __ldg(&coeff[v]) : 0.0;
                }
                typename E::Geo g;
                if (!E::template geometry<DAA>(X, U, g)) atomicMin(err, __ldg(&elem_list[le]));
                int kr = 0;
                if (DM) {
                    RowsSink<F, DM, DA, DAA> sink{sv[warp][lane][kr++], a};
                    E::template kind<KIND_M>(g, sink);
                }
                if (DA) {
                    RowsSink<F, DM, DA, DAA> sink{sv[warp][lane][kr++], a};
                    E::template kind<KIND_A>(g, sink);
                }
                if (DAA) {
                    RowsSink<F, DM, DA, DAA> sink{sv[warp][lane][kr++], a};
                    E::template kind<KIND_AA>(g, sink);
                }
            }
            __syncwarp();
            // slot owners add the entries in ascending element order
            for (int l = 0; l < cnt; ++l)
#pragma unroll
                for (int b = 0; b < N; ++b) {
                    const int32_t node = snode[warp][l][b];
#pragma unroll
                    for (int t = 0; t < ROWS_SPL; ++t)
                        if (node == col[t])
#pragma unroll
                            for (int k = 0; k < NK; ++k) acc[k][t] += sv[warp][l][k][b];
                }
            __syncwarp();
        }
#pragma unroll
        for (int t = 0; t < ROWS_SPL; ++t)
            if (lane + 32 * t < len) {
                int kr = 0;
                if (DM) vm[s0 + lane + 32 * t] = acc[kr++][t];
                if (DA) va[s0 + lane + 32 * t] = acc[kr++][t];
                if (DAA) vaa[s0 + lane + 32 * t] = acc[kr++][t];
            }
    }
}

// max row length of the plan (one-time check against ROWS_SPL * 32)
__global__ void k_max_row_len(int64_t n_rows, const int64_t* __restrict__ row_ptr, int* __restrict__ out) {
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows; i += (int64_t)gridDim.x * blockDim.x) {
        const int l = (int)(row_ptr[i + 1] - row_ptr[i]);
        m = l > m ? l : m;
    }
    atomicMax(out, m);
}

template <int F, bool DM, bool DA, bool DAA>
lfem_status run_rows(lfem_plan_s* p, const double* coords, const double* coeff, double* const vals[3],
                     cudaStream_t s) {
    if (p->n_rows == 0) return LFEM_OK;
    prof_begin(p, "k_rows", s);
    const unsigned grid = grid_for(p->n_rows, ROWS_WARPS, 148 * 64);
    k_rows<F, DM, DA, DAA><<<grid, ROWS_WARPS * 32, 0, s>>>(p->n_rows, p->row_ptr, p->col_idx, p->rhs_ptr,
                                                           p->rhs_codes, p->local_conn, p->elem_list, coords, coeff,
                                                           vals[0], vals[1], vals[2], p->err);
    LFEM_CUDA(cudaGetLastError());
    prof_end(p, s);
    return LFEM_OK;
}

template <int F>
lfem_status rows_kinds(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                       double* const vals[3], cudaStream_t s) {
    switch (kinds) {
    case 1: return run_rows<F, true, false, false>(p, coords, coeff, vals, s);
    case 2: return run_rows<F, false, true, false>(p, coords, coeff, vals, s);
    case 3: return run_rows<F, true, true, false>(p, coords, coeff, vals, s);
    case 4: return run_rows<F, false, false, true>(p, coords, coeff, vals, s);
    case 5: return run_rows<F, true, false, true>(p, coords, coeff, vals, s);
    case 6: return run_rows<F, false, true, true>(p, coords, coeff, vals, s);
    case 7: return run_rows<F, true, true, true>(p, coords, coeff, vals, s);
    default: return lfem_fail(LFEM_ERR_INVALID_ARG, "kinds");
    }
}

}  // namespace

// ROWS is available when every row fits the lanes' slots; *ok = false -> caller falls back to V0
lfem_status rows_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                          double* const vals[3], cudaStream_t s, bool* ok) {
    *ok = false;
    if (p->rows_ok < 0) {
        int* d = nullptr;
        LFEM_TRY(dev_alloc_t(&d, 1, s));
        LFEM_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
        int h = 0;
        if (p->n_rows > 0) {
            k_max_row_len<<<grid_for(p->n_rows, 256, 1024), 256, 0, s>>>(p->n_rows, p->row_ptr, d);
            LFEM_CUDA(cudaGetLastError());
        }
        LFEM_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        dev_free(d, s);
        p->rows_ok = h <= ROWS_SPL * 32 ? 1 : 0;
    }
    if (!p->rows_ok) return LFEM_OK;
    if (p->mesh->family == FAM_LINE_P1 || p->mesh->family == FAM_LINE_P2 || p->mesh->family == FAM_LINE_P2_Q6 ||
        p->mesh->family == FAM_TET_P2_Q35)
        return LFEM_OK;  // -> V0
    LFEM_TRY(rhs_prepare(p, s));
    *ok = true;
    switch (p->mesh->family) {
    case FAM_TRI_P1: return rows_kinds<FAM_TRI_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2: return rows_kinds<FAM_TRI_P2>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2_Q16: return rows_kinds<FAM_TRI_P2_Q16>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P1: return rows_kinds<FAM_TET_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P2: return rows_kinds<FAM_TET_P2>(p, kinds, coords, coeff, vals, s);
    }
    return lfem_fail(LFEM_ERR_UNSUPPORTED, "family");
}

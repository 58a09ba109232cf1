// Right-hand sides on B200 (sm_100a), fp64: SURVEY.md §8(f) row N1.
// Included by numeric.cu (shares its constant-memory reference tables and
// the Elem<F> geometry helpers).
//
//   load (all families):  b_j = sum_E sum_q w_q mu f_h(xi_q) phi_j(xi_q)
//                         (= M f with the element rule)
//   KLL (surface):        u = (nu_1, nu_2, nu_3, H) nodal,
//                         alpha^2 = |grad_{Gamma_h} nu_h|_F^2           (Listing 2 l.2)
//                         f_{k,j} = sum_E sum_q w_q mu alpha^2 u_{h,k} phi_j
//
// Surface gradients in metric form: with D_k = sum_c nu_{c,k} grad_ref phi_c
// (a 2-vector; the same difference form as the Jacobian, Elem::jac_parts),
// |J G^{-1} D_k|^2 = D_k^T G^{-1} D_k, so
//   w mu alpha^2 = w (1/mu) sum_k (g22 D_k1^2 - 2 g12 D_k1 D_k2 + g11 D_k2^2),
// no 3-vector gradients are formed (the oracle forms them: a different
// formulation of the same quantity, reading G2).
//
// Two kernels (the V0 scheme of numeric.cu, applied to vectors):
//   k_rhs_elem   thread per element -> local vectors, staged element-major
//                [le][a][k] through shared memory (warp-contiguous 16-B stores);
//   k_rhs_reduce thread per owned row, summing its incident (le, a) entries in
//                ascending element order (the plan's diagonal-slot order, G21).
// The row incidence lists come from the diagonal CSR slots of the plan (built
// once per plan, rhs_prepare).

namespace {

constexpr int RHS_THREADS = 128;

template <int KIND> struct RhsInfo { static constexpr int NC = KIND == LFEM_RHS_KLL ? 4 : 1; };

// minimum resident CTAs per SM (register caps) of the two-kernel element kernel (measured: 3 for the
// P2 triangle KLL kernel, 4 for the P2 tetrahedron load kernel) and of the fused kernel
#ifndef LFEM_RHS_MINB
#define LFEM_RHS_MINB 3
#endif
template <int F> struct RhsMinb { static constexpr int V = LFEM_RHS_MINB; };
template <> struct RhsMinb<FAM_TET_P2> { static constexpr int V = LFEM_RHS_MINB + 1; };
#ifndef LFEM_RHS_TMINB
#define LFEM_RHS_TMINB 2
#endif

// Local right-hand side of plan-local element le (nref x NC, Fl[a][k]); false if degenerate.
// Phase 1 turns the geometry (and nu_h's reference gradients) into one weight per quadrature
// point, wt_q = w_q mu (load) or w_q mu alpha^2 (KLL); phase 2 interpolates u_h and applies the
// basis.  Splitting the phases keeps the Jacobian parts and the accumulators from being live
// together (register pressure of the thread-per-element kernels).
template <int F, int KIND>
__device__ __forceinline__ bool rhs_local(int64_t le, const int32_t* __restrict__ lconn,
                                          const double* __restrict__ coords, const double* __restrict__ u,
                                          int64_t n_nodes, double (&Fl)[FamInfo<F>::NREF][RhsInfo<KIND>::NC]) {
    using E = Elem<F>;
    constexpr int N = E::N, D = E::D, NQ = E::NQ, NC = RhsInfo<KIND>::NC;
    constexpr bool KLL = KIND == LFEM_RHS_KLL;
    static_assert(!KLL || D == 2, "KLL right-hand side: surfaces only");
    const RefTab<F>& T = tab<F>();
    int64_t v[N];
#pragma unroll
    for (int a = 0; a < N; ++a) v[a] = __ldg(&lconn[le * N + a]);
    double wt[NQ];
    bool ok = true;
    {
        double J0[3][D], J1[3][D][D];
        {
            double X[N][3];
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int c = 0; c < 3; ++c) X[a][c] = __ldg(&coords[3 * v[a] + c]);
            E::jac_parts(X, J0, J1);
        }
        // reference gradients of nu_h: the same affine parts as J (KLL only)
        double V0[3][D], V1[3][D][D];
        if constexpr (KLL) {
            double NU[N][3];
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int k = 0; k < 3; ++k) NU[a][k] = __ldg(&u[k * n_nodes + v[a]]);
            E::jac_parts(NU, V0, V1);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double J[3][D];
            E::jac_at(J0, J1, q, J);
            if constexpr (D == 1) {
                const double det = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
                ok &= (det > 0.0) & (det < INFINITY);
                wt[q] = T.w[q] * (det * rsqrt_nr(det));
            } else if constexpr (D == 2) {
                const double g11 = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
                const double g12 = J[0][0] * J[0][1 % D] + J[1][0] * J[1][1 % D] + J[2][0] * J[2][1 % D];
                const double g22 = J[0][1 % D] * J[0][1 % D] + J[1][1 % D] * J[1][1 % D] + J[2][1 % D] * J[2][1 % D];
                const double det = g11 * g22 - g12 * g12;
                ok &= (det > 0.0) & (det < INFINITY);
                const double r = rsqrt_nr(det);
                if constexpr (KLL) {
                    double Vq[3][D];
                    E::jac_at(V0, V1, q, Vq);
                    double a2 = 0.0;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const double d1 = Vq[k][0], d2 = Vq[k][1 % D];
                        a2 = fma(g22 * d1, d1, a2);
                        a2 = fma(-2.0 * g12 * d1, d2, a2);
                        a2 = fma(g11 * d2, d2, a2);
                    }
                    wt[q] = T.w[q] * r * a2;
                } else {
                    wt[q] = T.w[q] * (det * r);
                }
            } else {
                double C[3][3];
                const double adet = fabs(E::cof(J, C));
                ok &= (adet > 0.0) & (adet < INFINITY);
                wt[q] = T.w[q] * adet;
            }
        }
    }
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
        for (int k = 0; k < NC; ++k) Fl[a][k] = 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        double U[N];
#pragma unroll
        for (int c = 0; c < N; ++c) U[c] = __ldg(&u[k * n_nodes + v[c]]);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double uq = 0.0;
#pragma unroll
            for (int c = 0; c < N; ++c) uq = fma(U[c], T.phi[q][c], uq);
            const double t = wt[q] * uq;
#pragma unroll
            for (int a = 0; a < N; ++a) Fl[a][k] = fma(t, T.phi[q][a], Fl[a][k]);
        }
    }
    return ok;
}

template <int F, int KIND>
__global__ void __launch_bounds__(RHS_THREADS, RhsMinb<F>::V)
k_rhs_elem(int64_t n_local, const int32_t* __restrict__ lconn, const int32_t* __restrict__ elem_list,
           const double* __restrict__ coords, const double* __restrict__ u, int64_t n_nodes,
           double* __restrict__ stage, int* __restrict__ err) {
    constexpr int N = FamInfo<F>::NREF, NC = RhsInfo<KIND>::NC, BD = N * NC;
    extern __shared__ __align__(16) double rhs_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* wsm = rhs_smem + (size_t)warp * 32 * BD;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t le0 = blockIdx.x * (int64_t)blockDim.x + warp * 32; le0 < n_local; le0 += stride) {
        const int64_t le = le0 + lane;
        const int nvalid = n_local - le0 < 32 ? (int)(n_local - le0) : 32;
        if (le < n_local) {
            double Fl[N][NC];
            if (!rhs_local<F, KIND>(le, lconn, coords, u, n_nodes, Fl)) atomicMin(err, __ldg(&elem_list[le]));
            double* my = wsm + lane * BD;
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int k = 0; k < NC; ++k) my[a * NC + k] = Fl[a][k];
        }
        __syncwarp();
        const int nd = nvalid * BD;
        if ((BD & 1) == 0) {  // le0 * BD doubles: 16-B aligned
            const double2* src = reinterpret_cast<const double2*>(wsm);
            double2* dst = reinterpret_cast<double2*>(stage + le0 * BD);
            for (int i = lane; i < nd / 2; i += 32) dst[i] = src[i];
        } else {
            for (int i = lane; i < nd; i += 32) stage[le0 * BD + i] = wsm[i];
        }
        __syncwarp();
    }
}

// Fused variant on the matrices' row tiles (tiles.cu): per tile, the CTA computes the local
// vectors of the tile's elements (owned + halo, ascending) into shared memory, then each owned
// row sums its incident entries (tile-local codes e_tile * nref + a, ascending element) -- the
// stage never leaves the SM.  Persistent CTAs stride over the tiles; several CTAs per SM
// overlap one tile's element phase with another's row phase.
template <int F, int KIND>
__global__ void __launch_bounds__(RHS_THREADS, LFEM_RHS_TMINB)
k_rhs_tiled(int n_tiles, const int4* __restrict__ tile_info, const int32_t* __restrict__ tile_elems,
            int64_t row_begin, int64_t n_rows, const int64_t* __restrict__ rptr, const uint16_t* __restrict__ tcodes,
            const int32_t* __restrict__ lconn, const int32_t* __restrict__ elem_list,
            const double* __restrict__ coords, const double* __restrict__ u, int64_t n_nodes,
            double* __restrict__ out, int* __restrict__ err) {
    constexpr int N = FamInfo<F>::NREF, NC = RhsInfo<KIND>::NC, SBD = (N * NC) | 1;  // odd stride: no bank conflicts
    extern __shared__ __align__(16) double rhs_smem[];
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int4 i0 = __ldg(&tile_info[3 * t]), i2 = __ldg(&tile_info[3 * t + 2]);
        const int e0 = i0.z, ne = i0.w;
        const int64_t r0 = (int64_t)i2.x - row_begin;
        const int nr = i2.y;
        for (int et = threadIdx.x; et < ne; et += blockDim.x) {
            const int64_t le = __ldg(&tile_elems[e0 + et]);
            double Fl[N][NC];
            if (!rhs_local<F, KIND>(le, lconn, coords, u, n_nodes, Fl)) atomicMin(err, __ldg(&elem_list[le]));
            double* my = rhs_smem + et * SBD;
#pragma unroll
            for (int a = 0; a < N; ++a)
#pragma unroll
                for (int k = 0; k < NC; ++k) my[a * NC + k] = Fl[a][k];
        }
        __syncthreads();
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            const int64_t i = r0 + r;
            const int64_t j0 = __ldg(&rptr[i]), j1 = __ldg(&rptr[i + 1]);
            double acc[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) acc[k] = 0.0;
            for (int64_t j = j0; j < j1; ++j) {
                const int c = __ldg(&tcodes[j]);
                const double* p = rhs_smem + (c / N) * SBD + (c % N) * NC;
#pragma unroll
                for (int k = 0; k < NC; ++k) acc[k] += p[k];
            }
#pragma unroll
            for (int k = 0; k < NC; ++k) out[k * n_rows + i] = acc[k];
        }
        __syncthreads();
    }
}

// thread per owned row: ascending-element sum of its staged (le, a) entries
template <int NC>
__global__ void __launch_bounds__(256)
k_rhs_reduce(int64_t n_rows, const int64_t* __restrict__ rptr, const int32_t* __restrict__ rcodes,
             const double* __restrict__ stage, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j0 = __ldg(&rptr[i]), j1 = __ldg(&rptr[i + 1]);
        double acc[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) acc[k] = 0.0;
        for (int64_t j = j0; j < j1; ++j) {
            const double* p = stage + (int64_t)__ldg(&rcodes[j]) * NC;
            if constexpr (NC == 4) {
                const double2 v0 = __ldg(reinterpret_cast<const double2*>(p));
                const double2 v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
                acc[0] += v0.x;
                acc[1] += v0.y;
                acc[2] += v1.x;
                acc[3] += v1.y;
            } else {
#pragma unroll
                for (int k = 0; k < NC; ++k) acc[k] += __ldg(p + k);
            }
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) out[k * n_rows + i] = acc[k];
    }
}

// per owned row: its diagonal slot (binary search of the global row id among its columns)
// and the number of incident elements (= contributions of that slot; 0 for an unreferenced node)
__global__ void k_rhs_diag(int64_t n_rows, int64_t row_begin, const int64_t* __restrict__ row_ptr,
                           const int32_t* __restrict__ col_idx, const int32_t* __restrict__ slot_ptr,
                           int32_t* __restrict__ diag, int32_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
        const int32_t g = (int32_t)(row_begin + i);
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col_idx[mid] < g) lo = mid + 1;
            else hi = mid;
        }
        const bool found = lo < row_ptr[i + 1] && col_idx[lo] == g;
        diag[i] = found ? (int32_t)lo : -1;
        cnt[i] = found ? slot_ptr[lo + 1] - slot_ptr[lo] : 0;
    }
}

// codes of the diagonal slot (le * nsym + sym(a, a), ascending le) -> le * nref + a
__global__ void k_rhs_fill(int64_t n_rows, const int32_t* __restrict__ diag, const int32_t* __restrict__ slot_ptr,
                           const int32_t* __restrict__ codes, const int64_t* __restrict__ rptr, int nref, int nsym,
                           int32_t* __restrict__ rcodes) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = diag[i];
        if (d < 0) continue;
        int64_t o = rptr[i];
        for (int32_t j = slot_ptr[d]; j < slot_ptr[d + 1]; ++j) {
            const int32_t c = codes[j];
            const int32_t le = c / nsym, sym = c % nsym;
            int a = 0;
            while (a < nref && sym_index(nref, a, a) != sym) ++a;
            rcodes[o++] = le * nref + a;
        }
    }
}

// per tile: its rows' codes le * nref + a -> tile-local e_tile * nref + a (binary search of le
// among the tile's ascending elements); *bad = 1 if an element is missing (plan inconsistency)
__global__ void k_rhs_tcodes(int n_tiles, const int4* __restrict__ tile_info, const int32_t* __restrict__ tile_elems,
                             int64_t row_begin, const int64_t* __restrict__ rptr, const int32_t* __restrict__ rcodes,
                             int nref, uint16_t* __restrict__ tcodes, int* __restrict__ bad) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int4 i0 = tile_info[3 * t], i2 = tile_info[3 * t + 2];
        const int32_t* el = tile_elems + i0.z;
        const int ne = i0.w;
        const int64_t r0 = (int64_t)i2.x - row_begin;
        for (int r = threadIdx.x; r < i2.y; r += blockDim.x)
            for (int64_t j = rptr[r0 + r]; j < rptr[r0 + r + 1]; ++j) {
                const int32_t c = rcodes[j], le = c / nref, a = c % nref;
                int lo = 0, hi = ne;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (el[mid] < le) lo = mid + 1;
                    else hi = mid;
                }
                if (lo >= ne || el[lo] != le) {
                    *bad = 1;
                    tcodes[j] = 0;
                } else {
                    tcodes[j] = (uint16_t)(lo * nref + a);
                }
            }
    }
}

lfem_status rhs_prepare(lfem_plan_s* p, cudaStream_t s) {
    if (p->rhs_ptr) return LFEM_OK;
    DevScope scope(s);
    const int64_t n_rows = p->n_rows;
    int32_t *diag = nullptr, *cnt = nullptr;
    scope.track(&diag);
    scope.track(&cnt);
    int64_t* rptr = nullptr;
    scope.track(&rptr);
    LFEM_TRY(dev_alloc_t(&diag, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&cnt, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&rptr, n_rows + 1, s));
    if (n_rows > 0) {
        k_rhs_diag<<<grid_for(n_rows, 256, 1 << 20), 256, 0, s>>>(n_rows, p->row_begin, p->row_ptr, p->col_idx,
                                                                  p->slot_ptr, diag, cnt);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(scan_exclusive_i32_to_i64(cnt, rptr, n_rows, s));
    int64_t total = 0;
    LFEM_CUDA(cudaMemcpyAsync(&total, rptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    if ((int64_t)p->n_local * p->mesh->nref >= (int64_t)INT_MAX)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "n_elems_local * nref >= 2^31");
    int32_t* rcodes = nullptr;
    scope.track(&rcodes);
    LFEM_TRY(dev_alloc_t(&rcodes, total + 1, s));
    if (n_rows > 0) {
        k_rhs_fill<<<grid_for(n_rows, 256, 1 << 20), 256, 0, s>>>(n_rows, diag, p->slot_ptr, p->codes, rptr,
                                                                  p->mesh->nref, p->mesh->nsym, rcodes);
        LFEM_CUDA(cudaGetLastError());
    }
    scope.give(&rptr);
    scope.give(&rcodes);
    p->rhs_ptr = rptr;
    p->rhs_codes = rcodes;
    p->rhs_total = total;
    return LFEM_OK;
}

// Tile-local codes for the fused variant (once per plan); false if the tiled variant is not
// available for this plan (no tile plan, or 16-bit codes / shared memory do not fit).
template <int F, int KIND>
lfem_status rhs_prepare_tiled(lfem_plan_s* p, cudaStream_t s, bool* ok) {
    *ok = false;
    if (p->rhs_tiled == 0) return LFEM_OK;
    if (p->rhs_tiled < 0) {
        p->rhs_tiled = 0;
        if (ensure_tiles<F>(p, s) != LFEM_OK) return LFEM_OK;  // fall back to the two-kernel variant
        const TilePlan& T = p->tiles;
        if ((int64_t)T.max_tile_count * FamInfo<F>::NREF >= 65536) return LFEM_OK;
        DevScope scope(s);
        uint16_t* tc = nullptr;
        scope.track(&tc);
        int* bad = nullptr;
        scope.track(&bad);
        LFEM_TRY(dev_alloc_t(&tc, p->rhs_total + 1, s));
        LFEM_TRY(dev_alloc_t(&bad, 1, s));
        LFEM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
        if (T.n_tiles > 0) {
            k_rhs_tcodes<<<T.n_tiles < (1 << 20) ? T.n_tiles : (1 << 20), 128, 0, s>>>(
                T.n_tiles, T.tile_info, T.tile_elems, p->row_begin, p->rhs_ptr, p->rhs_codes, FamInfo<F>::NREF, tc,
                bad);
            LFEM_CUDA(cudaGetLastError());
        }
        int h = 0;
        LFEM_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        if (h) return lfem_fail(LFEM_ERR_STATE, "tile plan does not cover a row's elements (internal)");
        scope.give(&tc);
        p->rhs_tcodes = tc;
        p->rhs_tiled = 1;
    }
    // shared memory of this kind's stage
    constexpr int SBD = (FamInfo<F>::NREF * RhsInfo<KIND>::NC) | 1;
    *ok = (size_t)p->tiles.max_tile_count * SBD * sizeof(double) <= (size_t)200 * 1024;
    return LFEM_OK;
}

template <int F, int KIND>
lfem_status run_rhs_tiled(lfem_plan_s* p, const double* coords, const double* u, double* out, cudaStream_t s) {
    const TilePlan& T = p->tiles;
    if (T.n_tiles == 0) return LFEM_OK;
    constexpr int SBD = (FamInfo<F>::NREF * RhsInfo<KIND>::NC) | 1;
    const size_t smem = (size_t)T.max_tile_count * SBD * sizeof(double);
    LFEM_TRY(ensure_smem_attr(reinterpret_cast<const void*>(k_rhs_tiled<F, KIND>), (int)smem));
    int sms = 148, occ = 0;
    LFEM_TRY(device_sm_count(&sms));
    LFEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rhs_tiled<F, KIND>, RHS_THREADS, smem));
    if (occ < 1) return lfem_fail(LFEM_ERR_UNSUPPORTED, "fused right-hand side kernel does not fit on an SM");
    const int grid = T.n_tiles < occ * sms ? T.n_tiles : occ * sms;
    prof_begin(p, "k_rhs_tiled", s);
    k_rhs_tiled<F, KIND><<<grid, RHS_THREADS, smem, s>>>(T.n_tiles, T.tile_info, T.tile_elems, p->row_begin,
                                                         p->n_rows, p->rhs_ptr, p->rhs_tcodes, p->local_conn,
                                                         p->elem_list, coords, u, p->mesh->n_nodes, out, p->err);
    LFEM_CUDA(cudaGetLastError());
    prof_end(p, s);
    return LFEM_OK;
}

template <int F, int KIND>
lfem_status run_rhs(lfem_plan_s* p, const double* coords, const double* u, double* out, cudaStream_t s) {
    constexpr int NC = RhsInfo<KIND>::NC, BD = FamInfo<F>::NREF * NC;
    if constexpr (FamInfo<F>::D >= 2) {  // no tile configuration for curves
        if (p->variant == LFEM_NUMERIC_TILED) {  // opt-in: measured slower than the two kernels
            bool ok = false;
            LFEM_TRY((rhs_prepare_tiled<F, KIND>(p, s, &ok)));
            if (ok) {
                p->rhs_last_tiled = 1;
                return run_rhs_tiled<F, KIND>(p, coords, u, out, s);
            }
        }
    }
    p->rhs_last_tiled = 0;
    if (!p->rhs_stage) LFEM_TRY(dev_alloc_t(&p->rhs_stage, (size_t)4 * FamInfo<F>::NREF * p->n_local + 4, s));
    if (p->n_local > 0) {
        prof_begin(p, "k_rhs_elem", s);
        constexpr size_t smem = sizeof(double) * (size_t)RHS_THREADS * BD;
        LFEM_TRY(ensure_smem_attr(reinterpret_cast<const void*>(k_rhs_elem<F, KIND>), (int)smem));
        k_rhs_elem<F, KIND><<<grid_for(p->n_local, RHS_THREADS, 1 << 20), RHS_THREADS, smem, s>>>(
            p->n_local, p->local_conn, p->elem_list, coords, u, p->mesh->n_nodes, p->rhs_stage, p->err);
        LFEM_CUDA(cudaGetLastError());
        prof_end(p, s);
    }
    if (p->n_rows > 0) {
        prof_begin(p, "k_rhs_reduce", s);
        k_rhs_reduce<NC><<<grid_for(p->n_rows, 256, 1 << 20), 256, 0, s>>>(p->n_rows, p->rhs_ptr, p->rhs_codes,
                                                                          p->rhs_stage, out);
        LFEM_CUDA(cudaGetLastError());
        prof_end(p, s);
    }
    return LFEM_OK;
}

}  // namespace

lfem_status rhs_dispatch(lfem_plan_s* p, int kind, const double* coords, const double* u, double* out,
                         cudaStream_t s) {
    LFEM_TRY(upload_reference_tables());
    LFEM_TRY(rhs_prepare(p, s));
    const bool kll = kind == LFEM_RHS_KLL;
    switch (p->mesh->family) {
    case FAM_TRI_P1:
        return kll ? run_rhs<FAM_TRI_P1, LFEM_RHS_KLL>(p, coords, u, out, s)
                   : run_rhs<FAM_TRI_P1, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_TRI_P2:
        return kll ? run_rhs<FAM_TRI_P2, LFEM_RHS_KLL>(p, coords, u, out, s)
                   : run_rhs<FAM_TRI_P2, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_TRI_P2_Q16:
        return kll ? run_rhs<FAM_TRI_P2_Q16, LFEM_RHS_KLL>(p, coords, u, out, s)
                   : run_rhs<FAM_TRI_P2_Q16, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_TET_P1:
        if (kll) break;
        return run_rhs<FAM_TET_P1, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_LINE_P1:
        if (kll) break;
        return run_rhs<FAM_LINE_P1, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_LINE_P2:
        if (kll) break;
        return run_rhs<FAM_LINE_P2, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_TET_P2:
        if (kll) break;
        return run_rhs<FAM_TET_P2, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_TET_P2_Q35:
        if (kll) break;
        return run_rhs<FAM_TET_P2_Q35, LFEM_RHS_LOAD>(p, coords, u, out, s);
    case FAM_LINE_P2_Q6:
        if (kll) break;
        return run_rhs<FAM_LINE_P2_Q6, LFEM_RHS_LOAD>(p, coords, u, out, s);
    }
    return lfem_fail(LFEM_ERR_UNSUPPORTED, "right-hand side kind not available for this family");
}

int rhs_launch_count(lfem_plan_s* p) {
    if (p->rhs_last_tiled == 1) return p->tiles.n_tiles > 0 ? 1 : 0;
    return (p->n_local > 0 ? 1 : 0) + (p->n_rows > 0 ? 1 : 0);
}

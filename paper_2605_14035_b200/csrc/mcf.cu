// Dziuk's algorithm for mean curvature flow on B200.
//
// the linearly implicit Euler / ESFEM discretisation of
// d/dt X = Laplace_{Gamma[X]} Id reads
//     (M(x^{n-1}) + tau A(x^{n-1})) x^n = M(x^{n-1}) x^{n-1},
// one system per coordinate.  One step here = the numeric assembly of M and A
// at x^{n-1} (the hot path, on the plan's fixed topology: symbolic once), K =
// M + tau A (lfem_axpby's kernel), b = M x^{n-1}, and a Jacobi-preconditioned
// conjugate gradient solve of the three systems at once.
//
// Vectors are n x 3 AoS (the node array's own layout), so K's values and
// column indices are read once per iteration for all three coordinates
// (k_spmm3).  Dot products are deterministic: fixed grid, per-block tree
// reduction, then a one-block final pass in block order.  Convergence is
// checked on the host every CG_CHECK iterations (one 48-B read + sync).
#include <climits>
#include <cmath>
#include <vector>

#include "lfem_internal.cuh"

namespace {

constexpr int DOT_BLOCKS = 296;  // 2 x 148 SMs
constexpr int CG_CHECK = 8;      // iterations between host convergence checks
constexpr int DOT_THREADS = 256;

inline unsigned grid_rows(int64_t n, int per_block) {
    int64_t g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > (1 << 20)) g = 1 << 20;
    return (unsigned)g;
}

// Y[i] = sum_j K_ij X[col_j] (3 columns, AoS); SUB lanes per row (surface rows hold 7-19
// entries: a whole warp per row would leave most lanes idle), fixed-order reduction
constexpr int SPMM_SUB = 4;
__global__ void k_spmm3(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                        const double* __restrict__ vals, const double* __restrict__ X, double* __restrict__ Y) {
    const int sl = threadIdx.x & (SPMM_SUB - 1);
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / SPMM_SUB;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / SPMM_SUB;
    for (int64_t r0 = g; r0 < ((n + ng - 1) / ng) * ng; r0 += ng) {  // same trip count for every lane of a warp
        const int64_t r = r0;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if (r < n) {
            const int64_t j1 = __ldg(&row_ptr[r + 1]);
            for (int64_t j = __ldg(&row_ptr[r]) + sl; j < j1; j += SPMM_SUB) {
                const double v = __ldg(&vals[j]);
                const int64_t c = __ldg(&col[j]);
                a0 = fma(v, __ldg(&X[3 * c]), a0);
                a1 = fma(v, __ldg(&X[3 * c + 1]), a1);
                a2 = fma(v, __ldg(&X[3 * c + 2]), a2);
            }
        }
#pragma unroll
        for (int o = SPMM_SUB / 2; o > 0; o >>= 1) {
            a0 += __shfl_down_sync(0xffffffffu, a0, o, SPMM_SUB);
            a1 += __shfl_down_sync(0xffffffffu, a1, o, SPMM_SUB);
            a2 += __shfl_down_sync(0xffffffffu, a2, o, SPMM_SUB);
        }
        if (sl == 0 && r < n) {
            Y[3 * r] = a0;
            Y[3 * r + 1] = a1;
            Y[3 * r + 2] = a2;
        }
    }
}

// dinv[i] = 1 / K_ii (binary search of the diagonal among the row's sorted columns)
__global__ void k_diag_inv(int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                           const double* __restrict__ vals, double* __restrict__ dinv, int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = row_ptr[i], hi = row_ptr[i + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        const bool found = lo < row_ptr[i + 1] && col[lo] == i && vals[lo] > 0.0;
        dinv[i] = found ? 1.0 / vals[lo] : 1.0;
        if (!found) atomicMin(bad, (int)i);
    }
}

// block-level sum of 3 (or 6) per-thread values into part[blockIdx][k], fixed order
template <int K>
__device__ __forceinline__ void block_sums(double (&v)[K], double* __restrict__ part) {
    __shared__ double sh[DOT_THREADS / 32][K];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[warp][k] = v[k];
    __syncthreads();
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int w = 0; w < DOT_THREADS / 32; ++w) s += sh[w][threadIdx.x];
        part[blockIdx.x * K + threadIdx.x] = s;
    }
}

// out[k] = sum of part[b][k] over blocks in order (one block of 32 * K threads would do; one warp suffices)
template <int K>
__global__ void k_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += part[b * K + threadIdx.x];
        out[threadIdx.x] = s;
    }
}

// r = b - K x (q holds K x), z = dinv r, p = z; partials of r.z and r.r, per column
__global__ void __launch_bounds__(DOT_THREADS) k_cg_init(int64_t n, const double* __restrict__ b,
                                                         const double* __restrict__ q, const double* __restrict__ dinv,
                                                         double* __restrict__ r, double* __restrict__ z,
                                                         double* __restrict__ p, double* __restrict__ part) {
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = dinv[i];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double rr = b[3 * i + k] - q[3 * i + k];
            const double zz = d * rr;
            r[3 * i + k] = rr;
            z[3 * i + k] = zz;
            p[3 * i + k] = zz;
            v[k] = fma(rr, zz, v[k]);
            v[3 + k] = fma(rr, rr, v[3 + k]);
        }
    }
    block_sums<6>(v, part);
}

// partials of p.q per column
__global__ void __launch_bounds__(DOT_THREADS) k_dot_pq(int64_t n, const double* __restrict__ p,
                                                        const double* __restrict__ q, double* __restrict__ part) {
    double v[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] = fma(p[3 * i + k], q[3 * i + k], v[k]);
    block_sums<3>(v, part);
}

// alpha_k = rz_k / pq_k (0 for a converged column); x += alpha p, r -= alpha q, z = dinv r;
// partials of the new r.z and r.r.   s: [rz(3), rr(3), pq(3)]
__global__ void __launch_bounds__(DOT_THREADS) k_cg_update(int64_t n, const double* __restrict__ s,
                                                           const double* __restrict__ p, const double* __restrict__ q,
                                                           const double* __restrict__ dinv, double* __restrict__ x,
                                                           double* __restrict__ r, double* __restrict__ z,
                                                           double* __restrict__ part) {
    double al[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) al[k] = s[6 + k] != 0.0 ? s[k] / s[6 + k] : 0.0;
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = dinv[i];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            x[3 * i + k] = fma(al[k], p[3 * i + k], x[3 * i + k]);
            const double rr = fma(-al[k], q[3 * i + k], r[3 * i + k]);
            const double zz = d * rr;
            r[3 * i + k] = rr;
            z[3 * i + k] = zz;
            v[k] = fma(rr, zz, v[k]);
            v[3 + k] = fma(rr, rr, v[3 + k]);
        }
    }
    block_sums<6>(v, part);
}

// p = z + beta p, beta_k = rz_new_k / rz_old_k; then rz_old = rz_new
__global__ void k_cg_dir(int64_t n, const double* __restrict__ s_new, double* __restrict__ s_old,
                         const double* __restrict__ z, double* __restrict__ p) {
    double be[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) be[k] = s_old[k] != 0.0 ? s_new[k] / s_old[k] : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; ++k) p[3 * i + k] = fma(be[k], p[3 * i + k], z[3 * i + k]);
}

// partials of the column sums of an AoS n x 3 array
__global__ void __launch_bounds__(DOT_THREADS) k_colsum3(int64_t n, const double* __restrict__ a,
                                                         double* __restrict__ part) {
    double v[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] += a[3 * i + k];
    block_sums<3>(v, part);
}

// out[i][k] = a[i][k] - sum_k / n  (sum: device, 3 column sums); out may alias a
__global__ void k_sub_mean3(int64_t n, const double* __restrict__ sum, const double* a, double* out) {
    const double inv = 1.0 / (double)n;
    const double m0 = sum[0] * inv, m1 = sum[1] * inv, m2 = sum[2] * inv;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        out[3 * i] = a[3 * i] - m0;
        out[3 * i + 1] = a[3 * i + 1] - m1;
        out[3 * i + 2] = a[3 * i + 2] - m2;
    }
}

__global__ void k_copy_rz(const double* __restrict__ src, double* __restrict__ dst) {
    if (threadIdx.x < 3) dst[threadIdx.x] = src[threadIdx.x];
}

}  // namespace

// Workspace of the CG / MCF entry points (plan-owned, lfem_internal.cuh's McfWork).
static lfem_status mcf_work(lfem_plan_s* p, cudaStream_t s) {
    McfWork& W = p->mcf;
    if (W.bad) return LFEM_OK;  // allocated last: set only when every buffer exists (a failed call retries)
    mcf_free(p, s);             // drop the buffers of an earlier partial attempt
    const int64_t n = p->n_rows, nnz = p->nnz;
    for (double** v : {&W.r, &W.z, &W.pv, &W.q, &W.b}) LFEM_TRY(dev_alloc_t(v, (size_t)3 * n + 3, s));
    LFEM_TRY(dev_alloc_t(&W.dinv, (size_t)n + 1, s));
    for (double** v : {&W.M, &W.A, &W.K}) LFEM_TRY(dev_alloc_t(v, (size_t)nnz + 1, s));
    LFEM_TRY(dev_alloc_t(&W.part, (size_t)DOT_BLOCKS * 6, s));
    LFEM_TRY(dev_alloc_t(&W.sc, 24, s));  // CG scalars [0, 15), column sums [16, 19)
    LFEM_TRY(dev_alloc_t(&W.bad, 1, s));
    return LFEM_OK;
}

void mcf_free(lfem_plan_s* p, cudaStream_t s) {
    McfWork& W = p->mcf;
    if (W.cg_exec) cudaGraphExecDestroy(W.cg_exec);
    if (W.cap) cudaStreamDestroy(W.cap);
    for (void* v : {(void*)W.r, (void*)W.z, (void*)W.pv, (void*)W.q, (void*)W.b, (void*)W.dinv, (void*)W.M,
                    (void*)W.A, (void*)W.K, (void*)W.part, (void*)W.sc, (void*)W.bad})
        dev_free(v, s);
    W = McfWork{};
}

static lfem_status whole_mesh(lfem_plan_s* p) {
    if (p->row_begin != 0 || p->row_end != p->mesh->n_nodes)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "CG / MCF need a whole-mesh plan (row block given)");
    return LFEM_OK;
}

// CG on K (plan pattern, values vals_K) for the three AoS columns of b; x: initial guess in, solution out.
static lfem_status cg_run(lfem_plan_s* p, const double* vals_K, const double* b, double* x, double tol, int max_it,
                          int* iters_out, cudaStream_t s) {
    McfWork& W = p->mcf;
    const int64_t n = p->n_rows;
    if (iters_out) *iters_out = 0;
    if (n == 0) return LFEM_OK;
    const unsigned gsp = grid_rows(n * SPMM_SUB, 256);
    LFEM_CUDA(cudaMemsetAsync(W.bad, 0x7f, sizeof(int), s));
    k_diag_inv<<<grid_rows(n, 256), 256, 0, s>>>(n, p->row_ptr, p->col_idx, vals_K, W.dinv, W.bad);
    LFEM_CUDA(cudaGetLastError());
    // ||b_k||
    double* S = W.sc;  // [0..2] rz, [3..5] rr, [6..8] pq, [9..11] rz_new, [12..14] rr_new (+ pad)
    k_dot_pq<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(n, b, b, W.part);
    k_final<3><<<1, 32, 0, s>>>(W.part, DOT_BLOCKS, S + 6);
    double bb[3];
    int hbad = 0;
    LFEM_CUDA(cudaMemcpyAsync(bb, S + 6, sizeof(bb), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaMemcpyAsync(&hbad, W.bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    if (hbad != 0x7f7f7f7f) return lfem_fail(LFEM_ERR_STATE, "K has a zero or negative diagonal entry", hbad);
    // r = b - K x, z = D^-1 r, p = z
    k_spmm3<<<gsp, 256, 0, s>>>(n, p->row_ptr, p->col_idx, vals_K, x, W.q);
    k_cg_init<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(n, b, W.q, W.dinv, W.r, W.z, W.pv, W.part);
    k_final<6><<<1, 32, 0, s>>>(W.part, DOT_BLOCKS, S);
    LFEM_CUDA(cudaGetLastError());
    double rr[6];
    for (int it = 0;; ++it) {
        // convergence check (one small read + sync) every CHECK iterations and at max_it
        if (it % CG_CHECK == 0 || it >= max_it) {
            LFEM_CUDA(cudaMemcpyAsync(rr, S + (it == 0 ? 0 : 9), sizeof(rr), cudaMemcpyDeviceToHost, s));
            LFEM_CUDA(cudaStreamSynchronize(s));
            bool done = true;
            for (int k = 0; k < 3; ++k) {
                if (!std::isfinite(rr[3 + k])) return lfem_fail(LFEM_ERR_STATE, "CG diverged (non-finite residual)");
                done &= std::sqrt(rr[3 + k]) <= tol * std::sqrt(bb[k]);
            }
            if (iters_out) *iters_out = it;
            if (done) return LFEM_OK;
            if (it >= max_it) return lfem_fail(LFEM_ERR_STATE, "CG did not converge within max_it iterations");
        }
        // one iteration: p = z + beta p (beta = rz_new / rz, rz <- rz_new; not in the first), q = K p,
        // alpha = rz / pq, x += alpha p, r -= alpha q, z = D^-1 r, rz_new, rr_new
        auto body = [&](cudaStream_t st, bool first) -> lfem_status {
            if (!first) {
                k_cg_dir<<<grid_rows(n, 256), 256, 0, st>>>(n, S + 9, S, W.z, W.pv);
                k_copy_rz<<<1, 32, 0, st>>>(S + 9, S);
            }
            prof_begin(p, "k_spmm3", st);
            k_spmm3<<<gsp, 256, 0, st>>>(n, p->row_ptr, p->col_idx, vals_K, W.pv, W.q);
            prof_end(p, st);
            k_dot_pq<<<DOT_BLOCKS, DOT_THREADS, 0, st>>>(n, W.pv, W.q, W.part);
            k_final<3><<<1, 32, 0, st>>>(W.part, DOT_BLOCKS, S + 6);
            k_cg_update<<<DOT_BLOCKS, DOT_THREADS, 0, st>>>(n, S, W.pv, W.q, W.dinv, x, W.r, W.z, W.part);
            k_final<6><<<1, 32, 0, st>>>(W.part, DOT_BLOCKS, S + 9);
            LFEM_CUDA(cudaGetLastError());
            return LFEM_OK;
        };
        // steady state: CG_CHECK iterations (7 launches each) replayed from one captured CUDA graph
        // (the same kernels in the same order: the same bits); per-kernel profiling runs them eagerly
        if (it > 0 && it % CG_CHECK == 0 && it + CG_CHECK <= max_it && !prof_on(p)) {
            if (!W.cg_exec || W.cg_key_K != vals_K || W.cg_key_x != x) {
                if (W.cg_exec) {
                    cudaGraphExecDestroy(W.cg_exec);
                    W.cg_exec = nullptr;
                }
                if (!W.cap) LFEM_CUDA(cudaStreamCreateWithFlags(&W.cap, cudaStreamNonBlocking));
                cudaGraph_t g = nullptr;
                LFEM_CUDA(cudaStreamBeginCapture(W.cap, cudaStreamCaptureModeThreadLocal));
                lfem_status st = LFEM_OK;
                for (int k = 0; k < CG_CHECK && st == LFEM_OK; ++k) st = body(W.cap, false);
                const cudaError_t ec = cudaStreamEndCapture(W.cap, &g);
                if (st != LFEM_OK) {
                    if (g) cudaGraphDestroy(g);
                    return st;
                }
                LFEM_CUDA(ec);
                const cudaError_t ei = cudaGraphInstantiate(&W.cg_exec, g, 0);
                cudaGraphDestroy(g);
                LFEM_CUDA(ei);
                W.cg_key_K = vals_K;
                W.cg_key_x = x;
            }
            LFEM_CUDA(cudaGraphLaunch(W.cg_exec, s));
            it += CG_CHECK - 1;
            continue;
        }
        LFEM_TRY(body(s, it == 0));
    }
}

lfem_status cg_solve(lfem_plan_s* p, const double* vals_K, const double* b, double* x, double tol, int max_it,
                     int* iters, cudaStream_t s) {
    LFEM_TRY(whole_mesh(p));
    LFEM_TRY(mcf_work(p, s));
    return cg_run(p, vals_K, b, x, tol, max_it, iters, s);
}

// Mean-free surface Poisson: the least-squares solution of the bordered
// system [A; e^T] u = [b; 0] is A u = P b, e^T u = 0 with P the Euclidean projection onto e-perp
// (= range A): b~ = b - mean(b), PCG from u = 0 (iterates stay in range A for this consistent
// singular system), then u -= mean(u) to remove rounding drift along the kernel e.
lfem_status solve_meanfree(lfem_plan_s* p, const double* vals_A, const double* b, double* u, double tol, int max_it,
                           int* iters, cudaStream_t s) {
    LFEM_TRY(whole_mesh(p));
    LFEM_TRY(mcf_work(p, s));
    McfWork& W = p->mcf;
    const int64_t n = p->n_rows;
    if (iters) *iters = 0;
    if (n == 0) return LFEM_OK;
    double* S = W.sc;
    k_colsum3<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(n, b, W.part);
    k_final<3><<<1, 32, 0, s>>>(W.part, DOT_BLOCKS, S + 16);
    k_sub_mean3<<<grid_rows(n, 256), 256, 0, s>>>(n, S + 16, b, W.b);
    LFEM_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * 3 * n, s));
    LFEM_CUDA(cudaGetLastError());
    LFEM_TRY(cg_run(p, vals_A, W.b, u, tol, max_it, iters, s));
    k_colsum3<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(n, u, W.part);
    k_final<3><<<1, 32, 0, s>>>(W.part, DOT_BLOCKS, S + 16);
    k_sub_mean3<<<grid_rows(n, 256), 256, 0, s>>>(n, S + 16, u, u);
    LFEM_CUDA(cudaGetLastError());
    return LFEM_OK;
}

lfem_status mcf_step(lfem_plan_s* p, double tau, const double* x_prev, double* x_next, double tol, int max_it,
                     int* iters, cudaStream_t s) {
    LFEM_TRY(whole_mesh(p));
    LFEM_TRY(mcf_work(p, s));
    McfWork& W = p->mcf;
    const int64_t n = p->n_rows;
    // M, A at x^{n-1} (the assembly hot path on the fixed plan)
    double* vals[3] = {W.M, W.A, nullptr};
    LFEM_TRY(numeric_dispatch(p, LFEM_MASS | LFEM_STIFF, x_prev, nullptr, vals, s));
    LFEM_TRY(axpby_launch(p->nnz, 1.0, W.M, tau, W.A, W.K, s));  // K = M + tau A
    if (n > 0) {
        k_spmm3<<<grid_rows(n * SPMM_SUB, 256), 256, 0, s>>>(n, p->row_ptr, p->col_idx, W.M, x_prev, W.b);  // b = M x^{n-1}
        LFEM_CUDA(cudaGetLastError());
        if (x_next != x_prev)
            LFEM_CUDA(cudaMemcpyAsync(x_next, x_prev, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    }
    return cg_run(p, W.K, W.b, x_next, tol, max_it, iters, s);  // warm start: x^{n-1}
}

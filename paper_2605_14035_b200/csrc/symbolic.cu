// Symbolic phase of the ℓFEM assembly on B200: CSR pattern + reduction plan.
//
// PAPER.md §4.2: MATLAB's `sparse(I,J,V)` sorts the nE*nref^2
// index triplets and sums duplicates on EVERY assembly ("The log-linear
// asymptotic arises solely from sorting and summing duplicate
// contributions"); the paper names, but does not use, the alternative of
// "precomputing the sparsity structure ... sort-free assignment".  This file
// is that precomputation, done once per topology on the device:
//
//   1. k_flag/k_compact: elements touching the owned rows [rb, re), ascending
//      id (row-block partition with duplicated halo elements).
//   2. k_count/k_fill/k_sort_inc: one-digit LSD radix (counting) sort of the
//      element-local rows (e, a) by global row conn[e,a]; inside a row the
//      incidences are then sorted by (e, a) so every later order is
//      deterministic (reading G21).
//   3. k_row_pattern<0>: per row (one warp), the candidate columns
//      conn[e, b] of all incident (e, a) -- segmented sort + unique by rank
//      counting in shared memory -> row length; exclusive scan -> row_ptr.
//   4. k_row_pattern<1>: col_idx (ascending) and the reduction plan: for
//      every CSR slot the list of its contributions (e, a, b) in ascending
//      (e, a, b) order (slot_ptr + codes, code = e_local * nsym + sym(a,b)).
#include <algorithm>
#include <climits>
#include <vector>

#include "lfem_internal.cuh"

namespace {

constexpr int MAX_CAND = 512;   // candidate (element, column) entries per row
constexpr int ROW_WARPS = 8;    // warps per block in k_row_pattern

__global__ void k_flag(const int32_t* __restrict__ conn, int64_t n_elems, int nref, int64_t rb, int64_t re,
                       int32_t* __restrict__ flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elems;
         e += (int64_t)gridDim.x * blockDim.x) {
        int f = 0;
        for (int a = 0; a < nref; ++a) {
            const int64_t v = conn[e * nref + a];
            f |= (v >= rb && v < re);
        }
        flag[e] = f;
    }
}

__global__ void k_compact(const int32_t* __restrict__ flag, const int64_t* __restrict__ pos, int64_t n_elems,
                          const int32_t* __restrict__ conn, int nref, int32_t* __restrict__ elem_list,
                          int32_t* __restrict__ local_conn) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elems;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (flag[e]) {
            const int64_t le = pos[e];
            elem_list[le] = (int32_t)e;
            for (int a = 0; a < nref; ++a) local_conn[le * nref + a] = conn[e * nref + a];
        }
    }
}

__global__ void k_count(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                        int32_t* __restrict__ cnt) {
    const int64_t n = n_local * nref;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = lconn[i];
        if (r >= rb && r < re) atomicAdd(&cnt[r - rb], 1);
    }
}

__global__ void k_fill(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                       const int64_t* __restrict__ inc_ptr, int32_t* __restrict__ cursor, int32_t* __restrict__ inc) {
    const int64_t n = n_local * nref;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = lconn[i];
        if (r >= rb && r < re) {
            const int k = atomicAdd(&cursor[r - rb], 1);
            inc[inc_ptr[r - rb] + k] = (int32_t)i;  // i = e_local * nref + a
        }
    }
}

// insertion sort of each row's incidence list (segments are short: <= 51)
__global__ void k_sort_inc(const int64_t* __restrict__ inc_ptr, int64_t n_rows, int32_t* __restrict__ inc) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = inc_ptr[r], e = inc_ptr[r + 1];
        for (int64_t i = b + 1; i < e; ++i) {
            const int32_t v = inc[i];
            int64_t j = i - 1;
            while (j >= b && inc[j] > v) {
                inc[j + 1] = inc[j];
                --j;
            }
            inc[j + 1] = v;
        }
    }
}

// One warp per row.  PASS 0: row_len.  PASS 1: col_idx, slot_ptr, codes.
template <int PASS>
__global__ void __launch_bounds__(ROW_WARPS * 32)
k_row_pattern(const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc, int64_t n_rows,
              const int32_t* __restrict__ lconn, int nref, int nsym, int32_t* __restrict__ row_len,
              const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx, int32_t* __restrict__ slot_ptr,
              int32_t* __restrict__ codes, int* __restrict__ nbig, int32_t* __restrict__ big, int big_cap) {
    __shared__ int32_t s_col[ROW_WARPS][MAX_CAND];
    __shared__ int32_t s_src[ROW_WARPS][MAX_CAND];  // e_local * nref + a  (PASS 1)
    __shared__ uint8_t s_first[ROW_WARPS][MAX_CAND];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * ROW_WARPS;
    for (int64_t r = blockIdx.x * (int64_t)ROW_WARPS + warp; r < n_rows; r += nwarps) {
        const int64_t ib = inc_ptr[r], ie = inc_ptr[r + 1];
        const int nc = (int)((ie - ib) * nref);
        if (nc > MAX_CAND) {  // long row: k_row_big (one CTA per row, global scratch)
            if (PASS == 0 && lane == 0) {
                row_len[r] = 0;
                const int k = atomicAdd(nbig, 1);
                if (k < big_cap) big[k] = (int32_t)r;
            }
            continue;
        }
        for (int i = lane; i < nc; i += 32) {
            const int k = i / nref, b = i - k * nref;
            const int32_t src = inc[ib + k];
            const int32_t le = src / nref;
            s_col[warp][i] = lconn[(int64_t)le * nref + b];
            s_src[warp][i] = src;
        }
        __syncwarp();
        if (PASS == 0) {
            int nfirst = 0;
            for (int i = lane; i < nc; i += 32) {
                const int32_t c = s_col[warp][i];
                bool first = true;
                for (int j = 0; j < i; ++j) first &= (s_col[warp][j] != c);
                nfirst += first;
            }
            for (int o = 16; o > 0; o >>= 1) nfirst += __shfl_down_sync(0xffffffffu, nfirst, o);
            if (lane == 0) row_len[r] = nfirst;
        } else {
            for (int i = lane; i < nc; i += 32) {
                const int32_t c = s_col[warp][i];
                bool first = true;
                for (int j = 0; j < i; ++j) first &= (s_col[warp][j] != c);
                s_first[warp][i] = first;
            }
            __syncwarp();
            const int64_t rp = row_ptr[r];
            const int64_t cbase = ib * nref;  // contributions of row r start here
            for (int i = lane; i < nc; i += 32) {
                const int32_t c = s_col[warp][i];
                int less = 0, less_unique = 0, before_eq = 0;
                for (int j = 0; j < nc; ++j) {
                    const int32_t cj = s_col[warp][j];
                    less += (cj < c);
                    less_unique += (cj < c) & s_first[warp][j];
                    before_eq += (cj == c) & (j < i);
                }
                if (s_first[warp][i]) {
                    col_idx[rp + less_unique] = c;
                    slot_ptr[rp + less_unique] = (int32_t)(cbase + less);
                }
                const int32_t src = s_src[warp][i];
                const int32_t le = src / nref;
                const int a = src - le * nref;
                const int b = i - (i / nref) * nref;
                codes[cbase + less + before_eq] = (int32_t)((int64_t)le * nsym + sym_index(nref, a, b));
            }
        }
        __syncwarp();
    }
}

// Rows with more than MAX_CAND candidates (e.g. a vertex shared by more than 51 P2
// tetrahedra): the same computation as k_row_pattern, one CTA per row, candidates in a
// global scratch range [off[k], off[k+1]) of the k-th long row.
constexpr int BIG_THREADS = 256;

__global__ void k_big_nc(const int32_t* __restrict__ big, int nbig, const int64_t* __restrict__ inc_ptr, int nref,
                         int64_t* __restrict__ nc) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nbig; k += gridDim.x * blockDim.x)
        nc[k] = (inc_ptr[big[k] + 1] - inc_ptr[big[k]]) * nref;
}

template <int PASS>
__global__ void __launch_bounds__(BIG_THREADS)
k_row_big(const int32_t* __restrict__ big, const int64_t* __restrict__ off, const int64_t* __restrict__ inc_ptr,
          const int32_t* __restrict__ inc, const int32_t* __restrict__ lconn, int nref, int nsym,
          int32_t* __restrict__ row_len, const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx,
          int32_t* __restrict__ slot_ptr, int32_t* __restrict__ codes, int32_t* __restrict__ g_col,
          int32_t* __restrict__ g_src, uint8_t* __restrict__ g_first) {
    __shared__ int s_red[BIG_THREADS / 32];
    const int64_t r = big[blockIdx.x];
    const int64_t ib = inc_ptr[r], base = off[blockIdx.x];
    const int nc = (int)(off[blockIdx.x + 1] - base);
    int32_t* col = g_col + base;
    int32_t* src_ = g_src + base;
    uint8_t* first = g_first + base;
    for (int i = threadIdx.x; i < nc; i += BIG_THREADS) {
        const int k = i / nref, b = i - k * nref;
        const int32_t src = inc[ib + k];
        col[i] = lconn[(int64_t)(src / nref) * nref + b];
        src_[i] = src;
    }
    __syncthreads();
    int nfirst = 0;
    for (int i = threadIdx.x; i < nc; i += BIG_THREADS) {
        const int32_t c = col[i];
        bool f = true;
        for (int j = 0; j < i && f; ++j) f = col[j] != c;
        first[i] = f;
        nfirst += f;
    }
    if (PASS == 0) {
        for (int o = 16; o > 0; o >>= 1) nfirst += __shfl_down_sync(0xffffffffu, nfirst, o);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = nfirst;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < BIG_THREADS / 32; ++w) t += s_red[w];
            row_len[r] = t;
        }
        return;
    }
    __syncthreads();
    const int64_t rp = row_ptr[r];
    const int64_t cbase = ib * nref;
    for (int i = threadIdx.x; i < nc; i += BIG_THREADS) {
        const int32_t c = col[i];
        int less = 0, less_unique = 0, before_eq = 0;
        for (int j = 0; j < nc; ++j) {
            const int32_t cj = col[j];
            less += (cj < c);
            less_unique += (cj < c) & first[j];
            before_eq += (cj == c) & (j < i);
        }
        if (first[i]) {
            col_idx[rp + less_unique] = c;
            slot_ptr[rp + less_unique] = (int32_t)(cbase + less);
        }
        const int32_t src = src_[i];
        const int32_t le = src / nref;
        const int a = src - le * nref;
        const int b = i - (i / nref) * nref;
        codes[cbase + less + before_eq] = (int32_t)((int64_t)le * nsym + sym_index(nref, a, b));
    }
}

__global__ void k_set_last(int32_t* slot_ptr, int64_t nnz, int64_t total) { slot_ptr[nnz] = (int32_t)total; }

inline unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 64) g = 148 * 64;
    return (unsigned)g;
}

}  // namespace

// Incidence lists of the owned rows: for row r (plan-relative), inc[inc_ptr[r] ..
// inc_ptr[r+1]) = the local entries i = e_local * nref + a with conn[e, a] = r,
// ascending (counting sort by row, then a per-row insertion sort).
lfem_status build_incidence(lfem_plan_s* p, int64_t** inc_ptr_out, int32_t** inc_out, cudaStream_t s) {
    DevScope scope(s);
    const int nref = p->mesh->nref;
    const int64_t rb = p->row_begin, re = p->row_end, n_rows = re - rb, n_local = p->n_local;
    int32_t* cnt = nullptr;
    scope.track(&cnt);
    int64_t* inc_ptr = nullptr;
    scope.track(&inc_ptr);
    LFEM_TRY(dev_alloc_t(&cnt, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&inc_ptr, n_rows + 1, s));
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_rows + 1), s));
    if (n_local > 0) {
        k_count<<<grid_for(n_local * nref, 256), 256, 0, s>>>(p->local_conn, n_local, nref, rb, re, cnt);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(scan_exclusive_i32_to_i64(cnt, inc_ptr, n_rows, s));
    int64_t total_inc = 0;
    LFEM_CUDA(cudaMemcpyAsync(&total_inc, inc_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    int32_t* inc = nullptr;
    scope.track(&inc);
    LFEM_TRY(dev_alloc_t(&inc, total_inc + 1, s));
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_rows + 1), s));
    if (n_local > 0) {
        k_fill<<<grid_for(n_local * nref, 256), 256, 0, s>>>(p->local_conn, n_local, nref, rb, re, inc_ptr, cnt, inc);
        LFEM_CUDA(cudaGetLastError());
    }
    if (n_rows > 0) {
        k_sort_inc<<<grid_for(n_rows, 128), 128, 0, s>>>(inc_ptr, n_rows, inc);
        LFEM_CUDA(cudaGetLastError());
    }
    scope.drop(cnt);
    scope.give(&inc_ptr);
    *inc_ptr_out = inc_ptr;
    scope.give(&inc);
    *inc_out = inc;
    return LFEM_OK;
}

lfem_status build_symbolic(lfem_plan_s* p, cudaStream_t s) {
    DevScope scope(s);
    const lfem_mesh_s* m = p->mesh;
    const int nref = m->nref;
    const int64_t rb = p->row_begin, re = p->row_end, n_rows = re - rb;
    p->n_rows = n_rows;
    // 1. elements touching the owned rows
    int32_t* flag = nullptr;
    scope.track(&flag);
    int64_t* pos = nullptr;
    scope.track(&pos);
    LFEM_TRY(dev_alloc_t(&flag, m->n_elems + 1, s));
    LFEM_TRY(dev_alloc_t(&pos, m->n_elems + 1, s));
    if (m->n_elems > 0) {
        k_flag<<<grid_for(m->n_elems, 256), 256, 0, s>>>(m->conn, m->n_elems, nref, rb, re, flag);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(scan_exclusive_i32_to_i64(flag, pos, m->n_elems, s));
    int64_t n_local = 0;
    LFEM_CUDA(cudaMemcpyAsync(&n_local, pos + m->n_elems, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    p->n_local = n_local;
    if (n_local * (int64_t)nref * nref >= (int64_t)INT_MAX)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "n_elems_local * nref^2 >= 2^31");
    LFEM_TRY(dev_alloc_t(&p->elem_list, n_local + 1, s));
    LFEM_TRY(dev_alloc_t(&p->local_conn, n_local * nref + 1, s));
    if (m->n_elems > 0) {
        k_compact<<<grid_for(m->n_elems, 256), 256, 0, s>>>(flag, pos, m->n_elems, m->conn, nref, p->elem_list,
                                                            p->local_conn);
        LFEM_CUDA(cudaGetLastError());
    }
    scope.drop(flag);
    scope.drop(pos);
    // 2. counting sort of local rows by global row
    int64_t* inc_ptr = nullptr;
    scope.track(&inc_ptr);
    int32_t* inc = nullptr;
    scope.track(&inc);
    LFEM_TRY(build_incidence(p, &inc_ptr, &inc, s));
    int64_t total_inc = 0;
    LFEM_CUDA(cudaMemcpyAsync(&total_inc, inc_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    p->n_contrib = total_inc * nref;
    if (p->n_contrib >= (int64_t)INT_MAX)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "contributions >= 2^31");
    int32_t* cnt = nullptr;
    scope.track(&cnt);
    LFEM_TRY(dev_alloc_t(&cnt, n_rows + 1, s));
    // 3. row lengths (rows with more than MAX_CAND candidates go to k_row_big)
    constexpr int BIG_CAP = 1 << 16;
    int* nbig_d = nullptr;
    scope.track(&nbig_d);
    int32_t* big = nullptr;
    scope.track(&big);
    LFEM_TRY(dev_alloc_t(&nbig_d, 1, s));
    LFEM_TRY(dev_alloc_t(&big, BIG_CAP, s));
    LFEM_CUDA(cudaMemsetAsync(nbig_d, 0, sizeof(int), s));
    const unsigned rgrid = grid_for(n_rows, ROW_WARPS);
    if (n_rows > 0) {
        k_row_pattern<0><<<rgrid, ROW_WARPS * 32, 0, s>>>(inc_ptr, inc, n_rows, p->local_conn, nref, m->nsym, cnt,
                                                          nullptr, nullptr, nullptr, nullptr, nbig_d, big, BIG_CAP);
        LFEM_CUDA(cudaGetLastError());
    }
    int nbig = 0;
    LFEM_CUDA(cudaMemcpyAsync(&nbig, nbig_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    if (nbig > BIG_CAP)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "more than 65536 rows with > 512 candidate (element, column) entries");
    int64_t* big_off = nullptr;
    scope.track(&big_off);
    int32_t *g_col = nullptr, *g_src = nullptr;
    uint8_t* g_first = nullptr;
    scope.track(&g_col);
    scope.track(&g_src);
    scope.track(&g_first);
    if (nbig > 0) {
        // the long rows' candidate counts -> scratch offsets (host; long rows are rare)
        std::vector<int32_t> hbig(nbig);
        LFEM_CUDA(cudaMemcpyAsync(hbig.data(), big, sizeof(int32_t) * nbig, cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        std::sort(hbig.begin(), hbig.end());
        LFEM_CUDA(cudaMemcpyAsync(big, hbig.data(), sizeof(int32_t) * nbig, cudaMemcpyHostToDevice, s));
        LFEM_TRY(dev_alloc_t(&big_off, (size_t)nbig + 1, s));
        k_big_nc<<<grid_for(nbig, 256), 256, 0, s>>>(big, nbig, inc_ptr, nref, big_off);
        LFEM_CUDA(cudaGetLastError());
        std::vector<int64_t> hoff(nbig + 1, 0);
        LFEM_CUDA(cudaMemcpyAsync(hoff.data(), big_off, sizeof(int64_t) * nbig, cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        int64_t run = 0;
        for (int k = 0; k < nbig; ++k) {
            const int64_t c = hoff[k];
            if (c >= (int64_t)INT_MAX) return lfem_fail(LFEM_ERR_UNSUPPORTED, "a row has >= 2^31 candidates");
            hoff[k] = run;
            run += c;
        }
        hoff[nbig] = run;
        LFEM_CUDA(cudaMemcpyAsync(big_off, hoff.data(), sizeof(int64_t) * (nbig + 1), cudaMemcpyHostToDevice, s));
        LFEM_TRY(dev_alloc_t(&g_col, (size_t)run + 1, s));
        LFEM_TRY(dev_alloc_t(&g_src, (size_t)run + 1, s));
        LFEM_TRY(dev_alloc_t(&g_first, (size_t)run + 1, s));
        k_row_big<0><<<nbig, BIG_THREADS, 0, s>>>(big, big_off, inc_ptr, inc, p->local_conn, nref, m->nsym, cnt,
                                                  nullptr, nullptr, nullptr, nullptr, g_col, g_src, g_first);
        LFEM_CUDA(cudaGetLastError());
        LFEM_CUDA(cudaStreamSynchronize(s));  // hbig / hoff (pageable) are read by the copies above
    }
    LFEM_TRY(dev_alloc_t(&p->row_ptr, n_rows + 1, s));
    LFEM_TRY(scan_exclusive_i32_to_i64(cnt, p->row_ptr, n_rows, s));
    LFEM_CUDA(cudaMemcpyAsync(&p->nnz, p->row_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    if (p->nnz >= (int64_t)INT_MAX) return lfem_fail(LFEM_ERR_UNSUPPORTED, "nnz >= 2^31");
    // 4. columns + reduction plan
    LFEM_TRY(dev_alloc_t(&p->col_idx, p->nnz + 1, s));
    LFEM_TRY(dev_alloc_t(&p->slot_ptr, p->nnz + 1, s));
    LFEM_TRY(dev_alloc_t(&p->codes, p->n_contrib + 1, s));
    if (n_rows > 0) {
        k_row_pattern<1><<<rgrid, ROW_WARPS * 32, 0, s>>>(inc_ptr, inc, n_rows, p->local_conn, nref, m->nsym,
                                                          nullptr, p->row_ptr, p->col_idx, p->slot_ptr, p->codes,
                                                          nbig_d, big, 0);
        LFEM_CUDA(cudaGetLastError());
    }
    if (nbig > 0) {
        k_row_big<1><<<nbig, BIG_THREADS, 0, s>>>(big, big_off, inc_ptr, inc, p->local_conn, nref, m->nsym, nullptr,
                                                  p->row_ptr, p->col_idx, p->slot_ptr, p->codes, g_col, g_src,
                                                  g_first);
        LFEM_CUDA(cudaGetLastError());
    }
    k_set_last<<<1, 1, 0, s>>>(p->slot_ptr, p->nnz, p->n_contrib);
    LFEM_CUDA(cudaGetLastError());
    scope.drop(cnt);
    scope.drop(inc_ptr);
    scope.drop(inc);
    LFEM_CUDA(cudaStreamSynchronize(s));
    return LFEM_OK;
}

void free_tiles(TilePlan& t, cudaStream_t s) {
    dev_free(t.tile_elems, s);
    dev_free(t.tile_elems_pos, s);
    dev_free(t.conn16, s);
    dev_free(t.halo, s);
    dev_free(t.tile_info, s);
    dev_free(t.pairs, s);
    dev_free(t.heavy, s);
    t = TilePlan();
}

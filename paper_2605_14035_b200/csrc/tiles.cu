// Row-tile plan of the fused numeric kernel (symbolic phase, one-time).
//
// A tile owns R consecutive rows [r0, r1) of the plan, hence the contiguous
// CSR slot range [row_ptr[r0], row_ptr[r1]).  Its element list holds every
// plan element with a node in [r0, r1), ascending (halo elements are
// recomputed by each tile that needs them -- the CTA-level analogue of the
// multi-GPU row-block partition).  For every slot the
// contributions keep the symbolic order (ascending element, then (a, b),
// reading G21) and are re-encoded as 16-bit codes sym(a,b) * maxe + e_tile
// (the shared-memory stage address), with an 8-bit count per slot.
#include <climits>
#include <vector>

#include "lfem_internal.cuh"

namespace {

inline unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 64) g = 148 * 64;
    return (unsigned)g;
}

// distinct tiles touched by element le (through its owned rows)
template <int MAXN>
__device__ __forceinline__ int elem_tiles(const int32_t* lconn, int nref, int64_t le, int64_t rb, int64_t re, int R,
                                          int* tiles) {
    int nt = 0;
    for (int a = 0; a < nref; ++a) {
        const int64_t r = lconn[le * nref + a];
        if (r < rb || r >= re) continue;
        const int t = (int)((r - rb) / R);
        bool seen = false;
        for (int i = 0; i < nt; ++i) seen |= (tiles[i] == t);
        if (!seen) tiles[nt++] = t;
    }
    return nt;
}

__global__ void k_tile_count(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                             int R, int32_t* __restrict__ cnt) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < n_local;
         le += (int64_t)gridDim.x * blockDim.x) {
        int tiles[10];
        const int nt = elem_tiles<10>(lconn, nref, le, rb, re, R, tiles);
        for (int i = 0; i < nt; ++i) atomicAdd(&cnt[tiles[i]], 1);
    }
}

__global__ void k_tile_fill(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                            int R, const int64_t* __restrict__ ptr, int32_t* __restrict__ cursor,
                            int32_t* __restrict__ out) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < n_local;
         le += (int64_t)gridDim.x * blockDim.x) {
        int tiles[10];
        const int nt = elem_tiles<10>(lconn, nref, le, rb, re, R, tiles);
        for (int i = 0; i < nt; ++i) {
            const int k = atomicAdd(&cursor[tiles[i]], 1);
            out[ptr[tiles[i]] + k] = (int32_t)le;
        }
    }
}

// rank sort of each tile's element list (unique keys), one block per tile
constexpr int SORT_MAX = 4096;
__global__ void k_tile_sort(const int64_t* __restrict__ ptr, int n_tiles, const int32_t* __restrict__ in,
                            int32_t* __restrict__ out, int* __restrict__ overflow) {
    __shared__ int32_t s[SORT_MAX];
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t b = ptr[t];
        const int n = (int)(ptr[t + 1] - b);
        if (n > SORT_MAX) {
            if (threadIdx.x == 0) atomicExch(overflow, 1);
            continue;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = in[b + i];
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int32_t v = s[i];
            int rank = 0;
            for (int j = 0; j < n; ++j) rank += (s[j] < v);
            out[b + rank] = v;
        }
        __syncthreads();
    }
}

// per row: re-encode its contributions; slot counts; tile maxima
__global__ void k_tile_codes(int64_t n_rows, int R, int nsym, int nref, int64_t n_local, int maxe,
                             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ slot_ptr,
                             const int32_t* __restrict__ codes, const int64_t* __restrict__ tptr,
                             const int32_t* __restrict__ telems, uint16_t* __restrict__ codes16,
                             uint8_t* __restrict__ slot_cnt, int* __restrict__ bad) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(r / R);
        const int32_t* te = telems + tptr[t];
        const int ne = (int)(tptr[t + 1] - tptr[t]);
        for (int64_t s = row_ptr[r]; s < row_ptr[r + 1]; ++s) {
            const int j0 = slot_ptr[s], j1 = slot_ptr[s + 1];
            if (j1 - j0 > 255) atomicExch(bad, 1);
            slot_cnt[s] = (uint8_t)(j1 - j0);
            for (int j = j0; j < j1; ++j) {
                const int32_t c = codes[j];
                const int sym = (int)(c / n_local);
                const int32_t le = (int32_t)(c - (int64_t)sym * n_local);
                int lo = 0, hi = ne;  // lower_bound
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (te[mid] < le) lo = mid + 1; else hi = mid;
                }
                if (lo >= ne || te[lo] != le) atomicExch(bad, 2);
                codes16[j] = (uint16_t)(sym * maxe + lo);
            }
        }
    }
}

__global__ void k_tile_sizes(int n_tiles, int R, int64_t n_rows, const int64_t* __restrict__ row_ptr,
                             const int32_t* __restrict__ slot_ptr, int32_t* __restrict__ code_ptr,
                             int* __restrict__ maxs, int* __restrict__ maxc) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles; t += gridDim.x * blockDim.x) {
        const int64_t r0 = (int64_t)t * R;
        const int64_t r1 = r0 + R < n_rows ? r0 + R : n_rows;
        const int64_t s0 = row_ptr[r0 < n_rows ? r0 : n_rows];
        code_ptr[t] = slot_ptr[s0];
        if (t < n_tiles) {
            const int64_t s1 = row_ptr[r1];
            atomicMax(maxs, (int)(s1 - s0));
            atomicMax(maxc, (int)(slot_ptr[s1] - slot_ptr[s0]));
        }
    }
}

// per-tile copy of the element connectivity, tile order, each tile padded to 16 B
__global__ void k_tile_conn(int n_tiles, int nref, const int64_t* __restrict__ ptr, const int32_t* __restrict__ telems,
                            const int32_t* __restrict__ lconn, const int32_t* __restrict__ cptr,
                            int32_t* __restrict__ tconn) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t b = ptr[t];
        const int n = (int)(ptr[t + 1] - b) * nref;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int e = i / nref, a = i - e * nref;
            tconn[cptr[t] + i] = lconn[(int64_t)telems[b + e] * nref + a];
        }
    }
}

// per-tile scalars {s0, ns, c0, nc, e0, ne, q0, nq} (all < 2^31)
__global__ void k_tile_info(int n_tiles, int R, int64_t n_rows, const int64_t* __restrict__ row_ptr,
                            const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ eptr,
                            const int32_t* __restrict__ qptr, int4* __restrict__ info) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x) {
        const int64_t r0 = (int64_t)t * R;
        const int64_t r1 = r0 + R < n_rows ? r0 + R : n_rows;
        const int64_t s0 = row_ptr[r0], s1 = row_ptr[r1];
        info[2 * t] = make_int4((int)s0, (int)(s1 - s0), slot_ptr[s0], slot_ptr[s1] - slot_ptr[s0]);
        info[2 * t + 1] = make_int4(eptr[t], eptr[t + 1] - eptr[t], qptr[t], qptr[t + 1] - qptr[t]);
    }
}

__global__ void k_max_seg(const int64_t* __restrict__ ptr, int n, int* __restrict__ mx) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        atomicMax(mx, (int)(ptr[t + 1] - ptr[t]));
}

}  // namespace

lfem_status build_tiles(lfem_plan_s* p, int R, cudaStream_t s) {
    free_tiles(p->tiles, s);
    TilePlan& T = p->tiles;
    const int nref = p->mesh->nref, nsym = p->mesh->nsym;
    const int64_t n_rows = p->n_rows, n_local = p->n_local;
    const int n_tiles = (int)((n_rows + R - 1) / R);
    T.rows_per_tile = R;
    T.n_tiles = n_tiles;
    if (n_tiles == 0) {
        T.ready = true;
        return LFEM_OK;
    }
    int32_t* cnt = nullptr;
    int64_t* ptr = nullptr;
    int32_t* tmp = nullptr;
    int* flags = nullptr;  // [0] overflow/bad, [1] max elems, [2] max slots, [3] max codes
    LFEM_TRY(dev_alloc_t(&cnt, n_tiles + 1, s));
    LFEM_TRY(dev_alloc_t(&ptr, n_tiles + 1, s));
    LFEM_TRY(dev_alloc_t(&flags, 4, s));
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_tiles + 1), s));
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    if (n_local > 0) {
        k_tile_count<<<grid_for(n_local, 256), 256, 0, s>>>(p->local_conn, n_local, nref, p->row_begin, p->row_end,
                                                            R, cnt);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(scan_exclusive_i32_to_i64(cnt, ptr, n_tiles, s));
    int64_t total = 0;
    LFEM_CUDA(cudaMemcpyAsync(&total, ptr + n_tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    LFEM_TRY(dev_alloc_t(&tmp, total + 1, s));
    LFEM_TRY(dev_alloc_t(&T.tile_elems, total + 1, s));
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_tiles + 1), s));
    if (n_local > 0) {
        k_tile_fill<<<grid_for(n_local, 256), 256, 0, s>>>(p->local_conn, n_local, nref, p->row_begin, p->row_end, R,
                                                           ptr, cnt, tmp);
        LFEM_CUDA(cudaGetLastError());
    }
    k_tile_sort<<<n_tiles < 148 * 8 ? n_tiles : 148 * 8, 256, 0, s>>>(ptr, n_tiles, tmp, T.tile_elems, flags);
    LFEM_CUDA(cudaGetLastError());
    k_max_seg<<<grid_for(n_tiles, 256), 256, 0, s>>>(ptr, n_tiles, flags + 1);
    LFEM_CUDA(cudaGetLastError());
    int h[4] = {0, 0, 0, 0};
    LFEM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    dev_free(tmp, s);
    if (h[0]) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile element list too long");
    const int maxe = h[1] > 0 ? h[1] : 1;
    if ((int64_t)nsym * maxe > 65535) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile too large for 16-bit codes");
    T.max_tile_elems = maxe;
    // element pointers as int32
    LFEM_TRY(dev_alloc_t(&T.tile_elem_ptr, n_tiles + 1, s));
    {
        // narrow int64 -> int32 on the host (n_tiles is small)
        std::vector<int64_t> hp(n_tiles + 1);
        std::vector<int32_t> hp32(n_tiles + 1);
        LFEM_CUDA(cudaMemcpy(hp.data(), ptr, sizeof(int64_t) * (n_tiles + 1), cudaMemcpyDeviceToHost));
        for (int i = 0; i <= n_tiles; ++i) hp32[i] = (int32_t)hp[i];
        LFEM_CUDA(cudaMemcpy(T.tile_elem_ptr, hp32.data(), sizeof(int32_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
        std::vector<int32_t> cp(n_tiles + 1);
        int64_t acc = 0;
        for (int i = 0; i < n_tiles; ++i) {
            cp[i] = (int32_t)acc;
            acc += ((hp[i + 1] - hp[i]) * nref + 3) & ~int64_t(3);
        }
        cp[n_tiles] = (int32_t)acc;
        if (acc >= INT_MAX) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile connectivity >= 2^31 entries");
        LFEM_TRY(dev_alloc_t(&T.tile_conn_ptr, n_tiles + 1, s));
        LFEM_TRY(dev_alloc_t(&T.tile_conn, acc + 16, s));
        LFEM_CUDA(cudaMemcpy(T.tile_conn_ptr, cp.data(), sizeof(int32_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
        k_tile_conn<<<n_tiles < 148 * 16 ? n_tiles : 148 * 16, 256, 0, s>>>(n_tiles, nref, ptr, T.tile_elems,
                                                                          p->local_conn, T.tile_conn_ptr, T.tile_conn);
        LFEM_CUDA(cudaGetLastError());
    }
    // codes
    LFEM_TRY(dev_alloc_t(&T.codes16, p->n_contrib + 64, s));  // bulk copies read up to 16 B past the end
    LFEM_TRY(dev_alloc_t(&T.slot_cnt, p->nnz + 64, s));
    LFEM_TRY(dev_alloc_t(&T.tile_code_ptr, n_tiles + 1, s));
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    if (n_rows > 0) {
        k_tile_codes<<<grid_for(n_rows, 128), 128, 0, s>>>(n_rows, R, nsym, nref, n_local, maxe, p->row_ptr,
                                                           p->slot_ptr, p->codes, ptr, T.tile_elems, T.codes16,
                                                           T.slot_cnt, flags);
        LFEM_CUDA(cudaGetLastError());
    }
    k_tile_sizes<<<grid_for(n_tiles + 1, 256), 256, 0, s>>>(n_tiles, R, n_rows, p->row_ptr, p->slot_ptr,
                                                            T.tile_code_ptr, flags + 2, flags + 3);
    LFEM_CUDA(cudaGetLastError());
    LFEM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    dev_free(cnt, s);
    dev_free(ptr, s);
    dev_free(flags, s);
    if (h[0]) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile code construction failed");
    LFEM_TRY(dev_alloc_t(&T.tile_info, (size_t)2 * n_tiles + 2, s));
    k_tile_info<<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, R, n_rows, p->row_ptr, p->slot_ptr, T.tile_elem_ptr,
                                                       T.tile_conn_ptr, T.tile_info);
    LFEM_CUDA(cudaGetLastError());
    LFEM_CUDA(cudaStreamSynchronize(s));
    T.max_tile_slots = h[2];
    T.max_tile_codes = h[3];
    T.ready = true;
    return LFEM_OK;
}

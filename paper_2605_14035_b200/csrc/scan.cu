// Device exclusive scan (reduce-then-scan, 3 kernels, recursive on block sums).
// Used by the symbolic phase only (element compaction, incidence offsets,
// row_ptr).  Deterministic: integer sums.
#include "lfem_internal.cuh"

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

template <class T>
__device__ __forceinline__ int64_t load_val(const T* in, int64_t i, int64_t n) {
    return i < n ? (int64_t)in[i] : 0;
}

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

template <class T>
__global__ void k_tile_reduce(const T* __restrict__ in, int64_t n, int64_t* __restrict__ tile_sums) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) s += load_val(in, base + k * SCAN_THREADS + threadIdx.x, n);
    // block reduce
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    __shared__ int64_t ws[SCAN_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w) t += ws[w];
        tile_sums[blockIdx.x] = t;
    }
}

// out[i] = offset(tile) + exclusive prefix within tile; thread t owns items
// [base + t*ITEMS, base + (t+1)*ITEMS) (blocked arrangement).
template <class T>
__global__ void k_tile_scan(const T* __restrict__ in, int64_t n, const int64_t* __restrict__ tile_offsets,
                            int64_t* __restrict__ out) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = load_val(in, base + k, n);
        s += v[k];
    }
    __shared__ int64_t warp_sums[SCAN_THREADS / 32 + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t inc = warp_incl_scan(s);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int64_t w = (lane < SCAN_THREADS / 32) ? warp_sums[lane] : 0;
        int64_t wi = warp_incl_scan(w);
        __syncwarp();
        if (lane < SCAN_THREADS / 32) warp_sums[lane] = wi - w;
    }
    __syncthreads();
    int64_t run = tile_offsets[blockIdx.x] + warp_sums[warp] + inc - s;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    // the grand total goes to out[n]
    if (base + SCAN_ITEMS >= n && base < n) {
        // this thread holds the last element
        out[n] = run;
    }
}

template <class T>
lfem_status scan_impl(const T* in, int64_t* out, int64_t n, cudaStream_t s) {
    if (n == 0) {
        LFEM_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return LFEM_OK;
    }
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    DevScope scope(s);  // both temporaries are freed on every exit path
    int64_t* tile_sums = nullptr;
    scope.track(&tile_sums);
    int64_t* tile_offsets = nullptr;
    scope.track(&tile_offsets);
    LFEM_TRY(dev_alloc_t(&tile_sums, tiles + 1, s));
    LFEM_TRY(dev_alloc_t(&tile_offsets, tiles + 1, s));
    k_tile_reduce<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, tile_sums);
    LFEM_CUDA(cudaGetLastError());
    if (tiles == 1) {
        LFEM_CUDA(cudaMemsetAsync(tile_offsets, 0, sizeof(int64_t), s));
    } else {
        lfem_status st = scan_impl<int64_t>(tile_sums, tile_offsets, tiles, s);
        if (st != LFEM_OK) return st;
    }
    k_tile_scan<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, tile_offsets, out);
    LFEM_CUDA(cudaGetLastError());
    return LFEM_OK;
}

}  // namespace

lfem_status scan_exclusive_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    return scan_impl<int32_t>(in, out, n, s);
}

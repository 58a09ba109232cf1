// Row-tile plan of the fused numeric kernel (symbolic phase, one-time).
//
// A tile owns consecutive rows [r0, r1) of the plan, hence the contiguous
// CSR slot range [row_ptr[r0], row_ptr[r1]).  Its element list holds every
// plan element with a node in [r0, r1), ascending (halo elements are
// recomputed by each tile that needs them -- the CTA-level analogue of the
// multi-GPU row-block partition).
//
// Tile boundaries are chosen by element budget, not by a fixed row count, so
// that every tile nearly fills the numeric kernel's compute threads.  Greedy,
// exact: walking the rows in order, a row r adds to the open tile [r0, r) the
// incident elements that have no owned node in [r0, r), i.e. whose previous
// owned row prev(e, r) < r0; the tile is closed when the next row would push
// its element count past the budget.  prev is precomputed per incidence; the
// walk runs independently on row segments (one thread each, a tile break at
// every segment start), so it is parallel and deterministic.
//
// Reduction codes.  A contribution (e, a, b) of the symbolic plan becomes the
// 16-bit stage byte offset  code = 8 * (sym(a,b) * maxe + e_tile)  (maxe = max
// tile elements = stage stride; byte offsets save the kernel an address shift).  Every slot keeps its contributions in symbolic
// order (ascending element, then (a, b): reading G21) and is described by one
// 32-bit word:
//   1 or 2 contributions  (c0, c1)   c1 = 0xffff if there is one
//   more ("heavy")        0xffffffff
// so the numeric kernel reads one word per slot and needs no scan.  Heavy
// slots (vertex diagonals; off-diagonals shared by 3+ elements in bulk) are
// listed separately per tile as fixed-size entries of HW u16 words
//   [slot - s0_tile, count, code_0, ..., code_{HW-3}]   (unused codes 0xffff)
// summed one entry per lane in a second pass; HW = 8, 16, 32, ... is the
// smallest that holds the mesh's largest slot count (8 = 16 B on icospheres:
// valence <= 6).
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
__device__ __forceinline__ int elem_tiles(const int32_t* lconn, int nref, int64_t le, int64_t rb, int64_t re,
                                          const int32_t* __restrict__ tile_of, int* tiles) {
    int nt = 0;
    for (int a = 0; a < nref; ++a) {
        const int64_t r = lconn[le * nref + a];
        if (r < rb || r >= re) continue;
        const int t = tile_of[r - rb];
        bool seen = false;
        for (int i = 0; i < nt; ++i) seen |= (tiles[i] == t);
        if (!seen) tiles[nt++] = t;
    }
    return nt;
}

// prev(e, r) for every incidence of the owned rows: the largest owned row of e below r, or -1 (plan-relative)
__global__ void k_inc_prev(int64_t n_rows, const int64_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                           const int32_t* __restrict__ lconn, int nref, int64_t rb, int32_t* __restrict__ prev) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t j = inc_ptr[r]; j < inc_ptr[r + 1]; ++j) {
            const int64_t le = inc[j] / nref;
            int64_t pv = -1;
            for (int b = 0; b < nref; ++b) {
                const int64_t n = (int64_t)lconn[le * nref + b] - rb;
                if (n >= 0 && n < r && n > pv) pv = n;
            }
            prev[j] = (int32_t)pv;
        }
    }
}

// greedy walk over the row segment [seg * seg_rows, ...): start[r] = 1 where a tile opens
__global__ void k_tile_greedy(int64_t n_rows, int64_t seg_rows, int emax, const int64_t* __restrict__ inc_ptr,
                              const int32_t* __restrict__ prev, int32_t* __restrict__ start, int* __restrict__ bad) {
    const int64_t nseg = (n_rows + seg_rows - 1) / seg_rows;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s0 = g * seg_rows, s1 = s0 + seg_rows < n_rows ? s0 + seg_rows : n_rows;
        int64_t r0 = s0;
        int cnt = 0;
        for (int64_t r = s0; r < s1; ++r) {
            const int64_t j0 = inc_ptr[r], j1 = inc_ptr[r + 1];
            int nw = 0;
            for (int64_t j = j0; j < j1; ++j) nw += prev[j] < r0;
            int st = r == s0;
            if (r > r0 && cnt + nw > emax) {  // close [r0, r), open a tile at r: all of r's elements are new
                st = 1;
                r0 = r;
                cnt = 0;
                nw = (int)(j1 - j0);
            }
            if (nw > emax) atomicExch(bad, 1);
            cnt += nw;
            start[r] = st;
        }
    }
}

__global__ void k_tile_bounds(int64_t n_rows, const int32_t* __restrict__ start, const int64_t* __restrict__ spos,
                              int64_t* __restrict__ bounds, int32_t* __restrict__ tile_of) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        if (start[r]) bounds[spos[r]] = r;
        tile_of[r] = (int32_t)(spos[r + 1] - 1);
        if (r == n_rows - 1) bounds[spos[n_rows]] = n_rows;
    }
}

__global__ void k_tile_count(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                             const int32_t* __restrict__ tile_of, int32_t* __restrict__ cnt) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < n_local;
         le += (int64_t)gridDim.x * blockDim.x) {
        int tiles[10];
        const int nt = elem_tiles(lconn, nref, le, rb, re, tile_of, tiles);
        for (int i = 0; i < nt; ++i) atomicAdd(&cnt[tiles[i]], 1);
    }
}

__global__ void k_tile_fill(const int32_t* __restrict__ lconn, int64_t n_local, int nref, int64_t rb, int64_t re,
                            const int32_t* __restrict__ tile_of, const int64_t* __restrict__ ptr,
                            int32_t* __restrict__ cursor, int32_t* __restrict__ out) {
    for (int64_t le = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; le < n_local;
         le += (int64_t)gridDim.x * blockDim.x) {
        int tiles[10];
        const int nt = elem_tiles(lconn, nref, le, rb, re, tile_of, tiles);
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

__global__ void k_max_seg(const int64_t* __restrict__ ptr, int n, int* __restrict__ mx) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        atomicMax(mx, (int)(ptr[t + 1] - ptr[t]));
}

// heavy slots of each row (> 2 contributions) and the largest contribution count
__global__ void k_row_heavy(int64_t n_rows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ slot_ptr,
                            int32_t* __restrict__ nh, int* __restrict__ maxc) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        int u = 0, m = 0;
        for (int64_t s = row_ptr[r]; s < row_ptr[r + 1]; ++s) {
            const int c = slot_ptr[s + 1] - slot_ptr[s];
            u += c > 2;
            m = c > m ? c : m;
        }
        nh[r] = u;
        atomicMax(maxc, m);
    }
}

// per row: the slot words and heavy entries (see the header).  Stage tail (byte offset
// tail = 8 nsym maxe of every stage buffer): a zero word.  A light slot with one
// contribution has c1 = tail (LFEM_ZERO_WORD) or 0xffff; a heavy slot's word is
// (tail, tail): the kernel's light loop writes 0 there, then (after a barrier of the
// reduce warps) the heavy loop writes the slot's sum -- no case analysis in the light
// loop.  Unused codes of a heavy entry are the zero word.
__global__ void k_tile_pairs(int64_t n_rows, const int32_t* __restrict__ tile_of, const int64_t* __restrict__ bounds,
                             int hw, int nsym, int maxe,
                             const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ slot_ptr,
                             const int32_t* __restrict__ codes, const int64_t* __restrict__ tptr,
                             const int32_t* __restrict__ telems, const uint16_t* __restrict__ tpos,
                             const int64_t* __restrict__ hptr, uint32_t* __restrict__ pairs,
                             uint16_t* __restrict__ heavy, int* __restrict__ bad) {
    const int64_t tail = 8 * (int64_t)nsym * maxe;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int t = tile_of[r];
        const int32_t* te = telems + tptr[t];
        const int ne = (int)(tptr[t + 1] - tptr[t]);
        const int64_t sbase = row_ptr[bounds[t]];
        const int64_t hbase = hptr[bounds[t]];  // the tile's first heavy entry
        int64_t cur = hptr[r] * hw;
        for (int64_t s = row_ptr[r]; s < row_ptr[r + 1]; ++s) {
            const int j0 = slot_ptr[s], j1 = slot_ptr[s + 1];
            const int c = j1 - j0;
            uint32_t code[2] = {(uint32_t)tail, LFEM_ZERO_WORD ? (uint32_t)tail : 0xffffu};
            const bool hv = c > 2;
            (void)hbase;
            if (hv) {
                if (s - sbase >= 0xffff) atomicExch(bad, 3);
                pairs[s] = (uint32_t)tail | ((LFEM_ZERO_WORD ? (uint32_t)tail : 0xffffu) << 16);
                heavy[cur] = (uint16_t)(s - sbase);
                heavy[cur + 1] = (uint16_t)c;
                for (int k = c; k < hw - 2; ++k) heavy[cur + 2 + k] = (uint16_t)tail;
            }
            for (int j = j0; j < j1; ++j) {
                const int32_t cc = codes[j];
                const int32_t le = cc / nsym;
                const int sym = cc - le * nsym;
                int lo = 0, hi = ne;  // lower_bound
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (te[mid] < le) lo = mid + 1; else hi = mid;
                }
                if (lo >= ne || te[lo] != le) atomicExch(bad, 2);
                const int64_t v = 8 * ((int64_t)sym * maxe + tpos[tptr[t] + lo]);
                if (v >= 0xffff) atomicExch(bad, 4);
                if (hv) heavy[cur + 2 + (j - j0)] = (uint16_t)v;
                else code[j - j0] = (uint32_t)v;
            }
            if (hv) cur += hw;
            else pairs[s] = code[0] | (code[1] << 16);
        }
    }
}

// max heavy entries of a tile (the stage tail must fit the 16-bit byte offsets)
__global__ void k_tile_heavymax(int n_tiles, const int64_t* __restrict__ bounds, const int64_t* __restrict__ hptr,
                                int* __restrict__ maxh) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x)
        atomicMax(maxh, (int)(hptr[bounds[t + 1]] - hptr[bounds[t]]));
}

// Per tile: its halo nodes (nodes of its elements outside its rows; sorted,
// unique, global ids) and the elements' tile-local node indices (u16):
// owned node n -> n - g0, halo node -> nrows + 1 + its rank in the halo list
// (one slot gap: the kernel's 16-B-rounded bulk copy of the owned range may
// write one double past it).
// One block per tile; candidates bitonic-sorted in shared memory.
constexpr int NODE_MAX = 4096;  // element-node candidates per tile (P1 triangles: 1024 x 3)
template <int PASS>
__global__ void __launch_bounds__(256)
k_tile_nodes(int n_tiles, int nref, int64_t rb, const int64_t* __restrict__ bounds, const int64_t* __restrict__ ptr,
             const int32_t* __restrict__ telems, const int32_t* __restrict__ lconn, int32_t* __restrict__ hcnt,
             const int32_t* __restrict__ lptr, const int32_t* __restrict__ cptr, int32_t* __restrict__ halo,
             uint16_t* __restrict__ conn16, const uint16_t* __restrict__ tpos, int* __restrict__ bad) {
    __shared__ int32_t key[NODE_MAX];
    __shared__ int wsum[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int PER = NODE_MAX / 256;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t g0 = rb + bounds[t], g1 = rb + bounds[t + 1];
        const int64_t e0 = ptr[t];
        const int ne = (int)(ptr[t + 1] - e0), nc = ne * nref;
        if (nc > NODE_MAX) {
            if (tid == 0) atomicExch(bad, 6);
            continue;
        }
        for (int i = tid; i < NODE_MAX; i += 256) {
            int32_t v = INT_MAX;
            if (i < nc) {
                const int32_t n = lconn[(int64_t)telems[e0 + i / nref] * nref + i % nref];
                v = (n >= g0 && n < g1) ? INT_MAX : n;
            }
            key[i] = v;
        }
        __syncthreads();
        for (int k = 2; k <= NODE_MAX; k <<= 1)  // bitonic sort, ascending
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < NODE_MAX; i += 256) {
                    const int l = i ^ j;
                    if (l > i) {
                        const int32_t a = key[i], b = key[l];
                        if (((i & k) == 0) ? (a > b) : (a < b)) { key[i] = b; key[l] = a; }
                    }
                }
                __syncthreads();
            }
        // unique halo nodes: first occurrence of each value != INT_MAX; block scan of the flags
        int f[PER], cnt = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = tid * PER + q;
            f[q] = key[i] != INT_MAX && (i == 0 || key[i] != key[i - 1]);
            cnt += f[q];
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int base = 0, nh = 0;
        for (int w = 0; w < 8; ++w) {
            base += w < warp ? wsum[w] : 0;
            nh += wsum[w];
        }
        int pos = base + incl - cnt;
        if (PASS == 0) {
            if (tid == 0) hcnt[t] = nh;
        } else {
            // compact the unique values to the front of key (in place is unsafe -> via the halo output)
            int32_t* out = halo + lptr[t];
#pragma unroll
            for (int q = 0; q < PER; ++q)
                if (f[q]) out[pos++] = key[tid * PER + q];
            __syncthreads();
            const int nrows = (int)(g1 - g0);
            for (int i = tid; i < nc; i += 256) {
                const int32_t n = lconn[(int64_t)telems[e0 + i / nref] * nref + i % nref];
                int loc;
                if (n >= g0 && n < g1) {
                    loc = (int)(n - g0);
                } else {
                    int lo = 0, hi = nh;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (out[mid] < n) lo = mid + 1; else hi = mid;
                    }
                    loc = nrows + 1 + lo;
                }
                if (loc >= 0xffff) atomicExch(bad, 7);
                conn16[cptr[t] + (int)tpos[e0 + i / nref] * nref + i % nref] = (uint16_t)loc;
            }
        }
        __syncthreads();
    }
}

// Stage positions of a tile's elements (bank-conflict-aware order).  The reduce
// warps load, per 16-lane half-warp, the first (second) contributions of 16 even
// (odd) CSR slots of consecutive two-slot units; a load's 8-B stage word sits in
// bank pair (sym * maxe + position) mod 16, and two lanes on the same bank pair
// but different words serialise.  The compute warps write stage[sym][position]
// for consecutive positions (conflict-free for ANY position order), so the order
// is free: greedily, in ascending element id, each element takes the residue
// class (position mod 16) that adds the fewest same-bank lanes to the load groups
// it appears in (dense positions: class k holds ceil((ne - k) / 16) elements).
// The summation order of every slot is unchanged (the slot words keep their
// contributions in symbolic order), so the values are bitwise the same.
constexpr int ORD_MAXM = 16384;     // light contributions per tile held in shared memory
constexpr int ORD_MAXG = 2048;      // load groups per tile (4 per 32 slots)
constexpr int ORD_MAXE = 4096;      // elements per tile
constexpr size_t ORD_SMEM = sizeof(uint32_t) * (ORD_MAXM + ORD_MAXG * 4) + sizeof(int) * (2 * ORD_MAXE + 1) + ORD_MAXE;
__global__ void __launch_bounds__(256)
k_tile_order(int n_tiles, int nsym, int maxe, const int64_t* __restrict__ bounds, const int64_t* __restrict__ row_ptr,
             const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ codes, const int64_t* __restrict__ ptr,
             const int32_t* __restrict__ telems, uint16_t* __restrict__ tpos) {
    extern __shared__ __align__(16) uint32_t ord_smem[];
    uint32_t* mem = ord_smem;                   // (group << 6 | sym) of each light contribution, by element
    uint32_t* gb = mem + ORD_MAXM;              // per group: 16 bank-pair counters (u8)
    int* mptr = reinterpret_cast<int*>(gb + ORD_MAXG * 4);
    int* mcur = mptr + ORD_MAXE + 1;
    uint8_t* col = reinterpret_cast<uint8_t*>(mcur + ORD_MAXE);
    __shared__ int fail;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t s0 = row_ptr[bounds[t]], s1 = row_ptr[bounds[t + 1]];
        const int32_t* te = telems + ptr[t];
        const int ne = (int)(ptr[t + 1] - ptr[t]);
        const int64_t u0 = s0 >> 1;
        const int ngr = (int)((((s1 + 1) >> 1) - u0 + 15) >> 4) * 4;
        if (tid == 0) fail = (ne > ORD_MAXE || ngr > ORD_MAXG) ? 1 : 0;
        for (int i = tid; i <= ne && i <= ORD_MAXE; i += 256) mptr[i] = 0;
        for (int i = tid; i < ngr * 4 && i < ORD_MAXG * 4; i += 256) gb[i] = 0u;
        __syncthreads();
        // light contributions of the tile's slots -> (element, group, sym); counts first
        for (int pass = 0; pass < 2 && !fail; ++pass) {
            for (int64_t S = s0 + tid; S < s1; S += 256) {
                const int j0 = slot_ptr[S], c = slot_ptr[S + 1] - j0;
                if (c > 2) continue;
                for (int ld = 0; ld < c; ++ld) {
                    const int32_t cc = codes[j0 + ld];
                    const int32_t le = cc / nsym;
                    int lo = 0, hi = ne;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (te[mid] < le) lo = mid + 1; else hi = mid;
                    }
                    if (lo >= ne) continue;
                    if (pass == 0) {
                        atomicAdd(&mptr[lo + 1], 1);
                    } else {
                        const int g = (int)((((S >> 1) - u0) >> 4) * 4 + (S & 1) * 2 + ld);
                        const int k = atomicAdd(&mcur[lo], 1);
                        if (k < ORD_MAXM) mem[k] = (uint32_t)g << 6 | (uint32_t)(cc - le * nsym);
                    }
                }
            }
            __syncthreads();
            if (pass == 0) {
                if (tid == 0) {  // exclusive scan of the counts (ne <= ORD_MAXE, once per tile)
                    for (int i = 0; i < ne; ++i) mptr[i + 1] += mptr[i];
                    if (mptr[ne] > ORD_MAXM) fail = 1;
                }
                __syncthreads();
                for (int i = tid; i < ne; i += 256) mcur[i] = mptr[i];
                __syncthreads();
            }
        }
        if (!fail && tid < 32) {
            // greedy residue classes, warp 0: lane k (< 16) prices class k, lanes 16..31 the
            // second half of the element's contributions for class lane - 16
            int used = 0;
            const int k = lane & 15;
            const int capk = k < ne ? (ne - k + 15) / 16 : 0;
            for (int e = 0; e < ne; ++e) {
                const int m0 = mptr[e], m1 = mptr[e + 1], mh = (m0 + m1) >> 1;
                int cost = 0;
                for (int m = (lane < 16 ? m0 : mh); m < (lane < 16 ? mh : m1); ++m) {
                    const uint32_t w = mem[m];
                    const int g = (int)(w >> 6), b = (int)(((w & 63u) * (uint32_t)maxe + (uint32_t)k) & 15u);
                    cost += (int)((gb[g * 4 + (b >> 2)] >> (8 * (b & 3))) & 255u);
                }
                cost += __shfl_xor_sync(0xffffffffu, cost, 16);
                // full classes are not candidates; ties -> the lowest class
                int key = used < capk ? (cost << 5 | k) : 0x7fffffff;
                for (int o = 8; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
                const int best = key & 31;
                if (k == best) ++used;
                for (int m = m0 + lane; m < m1; m += 32) {
                    const uint32_t w = mem[m];
                    const int g = (int)(w >> 6), b = (int)(((w & 63u) * (uint32_t)maxe + (uint32_t)best) & 15u);
                    atomicAdd(&gb[g * 4 + (b >> 2)], 1u << (8 * (b & 3)));
                }
                if (lane == 0) col[e] = (uint8_t)best;
                __syncwarp();
            }
            // dense positions: class c, in ascending element order, takes c, c + 16, c + 32, ...
            if (lane < 16) {
                int r = 0;
                for (int e = 0; e < ne; ++e)
                    if (col[e] == lane) tpos[ptr[t] + e] = (uint16_t)(lane + 16 * r++);
            }
        }
        if (fail)
            for (int e = tid; e < ne; e += 256) tpos[ptr[t] + e] = (uint16_t)e;  // identity order
        __syncthreads();
    }
}

// the tile's elements in stage-position order (the kernel reports degenerate elements through it)
__global__ void k_tile_scatter(int n_tiles, const int64_t* __restrict__ ptr, const int32_t* __restrict__ telems,
                               const uint16_t* __restrict__ tpos, int32_t* __restrict__ out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x)
        for (int64_t i = ptr[t]; i < ptr[t + 1]; ++i) out[ptr[t] + tpos[i]] = telems[i];
}

// per-tile scalars {s0, ns, e0, ne}, {q0, nq, h0, nh}, {g0, nrows, l0, nl} (all < 2^31) and maxima
__global__ void k_tile_info(int n_tiles, int64_t rb, const int64_t* __restrict__ bounds, int hw,
                            const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ eptr,
                            const int32_t* __restrict__ qptr, const int64_t* __restrict__ hptr,
                            const int32_t* __restrict__ lptr, const int32_t* __restrict__ hcnt, int4* __restrict__ info,
                            int* __restrict__ maxs, int* __restrict__ maxh, int* __restrict__ maxn) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x) {
        const int64_t r0 = bounds[t], r1 = bounds[t + 1];
        const int64_t s0 = row_ptr[r0], s1 = row_ptr[r1];
        info[3 * t] = make_int4((int)s0, (int)(s1 - s0), eptr[t], eptr[t + 1] - eptr[t]);
        info[3 * t + 1] = make_int4(qptr[t], qptr[t + 1] - qptr[t], (int)(hptr[r0] * hw), (int)((hptr[r1] - hptr[r0]) * hw));
        info[3 * t + 2] = make_int4((int)(rb + r0), (int)(r1 - r0), lptr[t], hcnt[t]);
        atomicMax(maxs, (int)(s1 - s0));
        atomicMax(maxh, (int)((hptr[r1] - hptr[r0]) * hw));
        atomicMax(maxn, (int)(r1 - r0) + 1 + hcnt[t]);
    }
}

}  // namespace

lfem_status build_tiles(lfem_plan_s* p, int emax, cudaStream_t s) {
    DevScope scope(s);
    free_tiles(p->tiles, s);
    TilePlan& T = p->tiles;
    const int nref = p->mesh->nref;
    const int64_t n_rows = p->n_rows, n_local = p->n_local;
    if (n_rows == 0) {
        T.ready = true;
        return LFEM_OK;
    }
    // greedy element-budget partition (see the header)
    int64_t* inc_ptr = nullptr;
    scope.track(&inc_ptr);
    int32_t* inc = nullptr;
    scope.track(&inc);
    LFEM_TRY(build_incidence(p, &inc_ptr, &inc, s));
    int64_t n_inc = 0;
    LFEM_CUDA(cudaMemcpyAsync(&n_inc, inc_ptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    int32_t* prev = nullptr;
    scope.track(&prev);
    int32_t* start = nullptr;
    scope.track(&start);
    int64_t* spos = nullptr;
    scope.track(&spos);
    int32_t* tile_of = nullptr;
    scope.track(&tile_of);
    int* flags = nullptr;  // [0] overflow/bad, [1] max elems, [2] max slots, [3] max heavy
    scope.track(&flags);
    LFEM_TRY(dev_alloc_t(&prev, n_inc + 1, s));
    LFEM_TRY(dev_alloc_t(&start, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&spos, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&tile_of, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&flags, 4, s));
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    k_inc_prev<<<grid_for(n_rows, 128), 128, 0, s>>>(n_rows, inc_ptr, inc, p->local_conn, nref, p->row_begin, prev);
    LFEM_CUDA(cudaGetLastError());
    {  // a tile holds at least one row: the budget is at least the largest row incidence
        k_max_seg<<<grid_for(n_rows, 256), 256, 0, s>>>(inc_ptr, (int)n_rows, flags + 1);
        LFEM_CUDA(cudaGetLastError());
        int maxinc = 0;
        LFEM_CUDA(cudaMemcpyAsync(&maxinc, flags + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
        if (maxinc > emax) emax = maxinc;
    }
    const int64_t seg_rows = 2048;
    k_tile_greedy<<<grid_for((n_rows + seg_rows - 1) / seg_rows, 64), 64, 0, s>>>(n_rows, seg_rows, emax, inc_ptr,
                                                                                  prev, start, flags);
    LFEM_CUDA(cudaGetLastError());
    LFEM_TRY(scan_exclusive_i32_to_i64(start, spos, n_rows, s));
    int64_t nt64 = 0;
    int hbad = 0;
    LFEM_CUDA(cudaMemcpyAsync(&nt64, spos + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaMemcpyAsync(&hbad, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    scope.drop(inc_ptr);
    scope.drop(inc);
    scope.drop(prev);
    if (hbad) return lfem_fail(LFEM_ERR_UNSUPPORTED, "a row touches more elements than a tile holds");
    if (nt64 >= INT_MAX / 2) return lfem_fail(LFEM_ERR_UNSUPPORTED, "too many tiles");
    const int n_tiles = (int)nt64;
    int64_t* bounds = nullptr;
    scope.track(&bounds);
    int32_t* cnt = nullptr;
    scope.track(&cnt);
    int64_t* ptr = nullptr;
    scope.track(&ptr);
    LFEM_TRY(dev_alloc_t(&bounds, n_tiles + 1, s));
    LFEM_TRY(dev_alloc_t(&cnt, n_tiles + 1, s));
    LFEM_TRY(dev_alloc_t(&ptr, n_tiles + 1, s));
    k_tile_bounds<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, start, spos, bounds, tile_of);
    LFEM_CUDA(cudaGetLastError());
    scope.drop(start);
    scope.drop(spos);
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_tiles + 1), s));
    if (n_local > 0) {
        k_tile_count<<<grid_for(n_local, 256), 256, 0, s>>>(p->local_conn, n_local, nref, p->row_begin, p->row_end,
                                                            tile_of, cnt);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(scan_exclusive_i32_to_i64(cnt, ptr, n_tiles, s));
    T.n_tiles = n_tiles;
    T.rows_per_tile = (int)((n_rows + n_tiles - 1) / n_tiles);  // average (reporting only)
    int32_t* tmp = nullptr;
    scope.track(&tmp);
    int64_t total = 0;
    LFEM_CUDA(cudaMemcpyAsync(&total, ptr + n_tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    T.total_elems = total;
    LFEM_TRY(dev_alloc_t(&tmp, total + 1, s));
    LFEM_TRY(dev_alloc_t(&T.tile_elems, total + 1, s));
    LFEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_tiles + 1), s));
    if (n_local > 0) {
        k_tile_fill<<<grid_for(n_local, 256), 256, 0, s>>>(p->local_conn, n_local, nref, p->row_begin, p->row_end,
                                                           tile_of, ptr, cnt, tmp);
        LFEM_CUDA(cudaGetLastError());
    }
    k_tile_sort<<<n_tiles < 148 * 8 ? n_tiles : 148 * 8, 256, 0, s>>>(ptr, n_tiles, tmp, T.tile_elems, flags);
    LFEM_CUDA(cudaGetLastError());
    k_max_seg<<<grid_for(n_tiles, 256), 256, 0, s>>>(ptr, n_tiles, flags + 1);
    LFEM_CUDA(cudaGetLastError());
    int h[4] = {0, 0, 0, 0};
    LFEM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    scope.drop(tmp);
    if (h[0]) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile element list too long");
    // stage stride: odd, so the nsym entries of one element fall in different smem banks
    const int maxe = (h[1] > 0 ? h[1] : 1) | 1;
    T.max_tile_elems = maxe;
    T.max_tile_count = h[1];
    if (8 * (int64_t)p->mesh->nsym * maxe >= 0xffff) {  // 16-bit byte offsets: the caller lowers the budget
        scope.drop(cnt);
        scope.drop(ptr);
        scope.drop(flags);
        scope.drop(bounds);
        scope.drop(tile_of);
        return LFEM_OK;
    }
    // bank-conflict-aware stage positions of every tile's elements (k_tile_order)
    uint16_t* tpos = nullptr;
    scope.track(&tpos);
    LFEM_TRY(dev_alloc_t(&tpos, total + 8, s));
    {
        LFEM_TRY(ensure_smem_attr(reinterpret_cast<const void*>(k_tile_order), (int)ORD_SMEM));
        k_tile_order<<<n_tiles < 148 * 4 ? n_tiles : 148 * 4, 256, ORD_SMEM, s>>>(
            n_tiles, p->mesh->nsym, maxe, bounds, p->row_ptr, p->slot_ptr, p->codes, ptr, T.tile_elems, tpos);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(dev_alloc_t(&T.tile_elems_pos, total + 1, s));
    k_tile_scatter<<<grid_for(n_tiles, 128), 128, 0, s>>>(n_tiles, ptr, T.tile_elems, tpos, T.tile_elems_pos);
    LFEM_CUDA(cudaGetLastError());
    // halo nodes per tile (pass 0: counts)
    int32_t* hcnt = nullptr;
    scope.track(&hcnt);
    LFEM_TRY(dev_alloc_t(&hcnt, n_tiles + 1, s));
    const unsigned node_grid = n_tiles < 148 * 8 ? n_tiles : 148 * 8;
    k_tile_nodes<0><<<node_grid, 256, 0, s>>>(n_tiles, nref, p->row_begin, bounds, ptr, T.tile_elems, p->local_conn,
                                              hcnt, nullptr, nullptr, nullptr, nullptr, nullptr, flags);
    LFEM_CUDA(cudaGetLastError());
    // element / connectivity / halo offsets as int32 (host; n_tiles is small)
    int32_t* eptr32 = nullptr;
    scope.track(&eptr32);
    int32_t* cptr32 = nullptr;
    scope.track(&cptr32);
    int32_t* lptr32 = nullptr;
    scope.track(&lptr32);
    {
        std::vector<int64_t> hp(n_tiles + 1);
        std::vector<int32_t> hp32(n_tiles + 1), cp(n_tiles + 1), hc(n_tiles + 1), lp(n_tiles + 1);
        LFEM_CUDA(cudaMemcpy(hp.data(), ptr, sizeof(int64_t) * (n_tiles + 1), cudaMemcpyDeviceToHost));
        LFEM_CUDA(cudaMemcpy(hc.data(), hcnt, sizeof(int32_t) * n_tiles, cudaMemcpyDeviceToHost));
        int64_t acc = 0, lacc = 0;
        for (int i = 0; i <= n_tiles; ++i) {
            hp32[i] = (int32_t)hp[i];
            cp[i] = (int32_t)acc;
            lp[i] = (int32_t)lacc;
            if (i < n_tiles) {
                acc += ((hp[i + 1] - hp[i]) * nref + 7) & ~int64_t(7);   // u16, 16-B padded
                lacc += (hc[i] + 3) & ~3;                                // int32, 16-B padded
            }
        }
        if (acc >= INT_MAX || hp[n_tiles] >= INT_MAX || lacc >= INT_MAX)
            return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile connectivity >= 2^31 entries");
        LFEM_TRY(dev_alloc_t(&eptr32, n_tiles + 1, s));
        LFEM_TRY(dev_alloc_t(&cptr32, n_tiles + 1, s));
        LFEM_TRY(dev_alloc_t(&lptr32, n_tiles + 1, s));
        LFEM_TRY(dev_alloc_t(&T.conn16, acc + 16, s));
        LFEM_TRY(dev_alloc_t(&T.halo, lacc + 8, s));
        LFEM_CUDA(cudaMemcpy(eptr32, hp32.data(), sizeof(int32_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
        LFEM_CUDA(cudaMemcpy(cptr32, cp.data(), sizeof(int32_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
        LFEM_CUDA(cudaMemcpy(lptr32, lp.data(), sizeof(int32_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
        k_tile_nodes<1><<<node_grid, 256, 0, s>>>(n_tiles, nref, p->row_begin, bounds, ptr, T.tile_elems,
                                                  p->local_conn, hcnt, lptr32, cptr32, T.halo, T.conn16, tpos, flags);
        LFEM_CUDA(cudaGetLastError());
        int hb = 0;
        LFEM_CUDA(cudaMemcpyAsync(&hb, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        LFEM_CUDA(cudaStreamSynchronize(s));
        if (hb) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile node lists do not fit (" + std::to_string(hb) + ")");
    }
    // heavy entries: per-row heavy-slot counts -> global entry offsets; entry size from the largest count
    int32_t* hu = nullptr;
    scope.track(&hu);
    int64_t* hptr = nullptr;
    scope.track(&hptr);
    LFEM_TRY(dev_alloc_t(&hu, n_rows + 1, s));
    LFEM_TRY(dev_alloc_t(&hptr, n_rows + 1, s));
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    k_row_heavy<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, p->row_ptr, p->slot_ptr, hu, flags + 1);
    LFEM_CUDA(cudaGetLastError());
    LFEM_TRY(scan_exclusive_i32_to_i64(hu, hptr, n_rows, s));
    int64_t heavy_slots = 0;
    LFEM_CUDA(cudaMemcpyAsync(&heavy_slots, hptr + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    int hw = 8;
    while (hw - 2 < h[1]) hw *= 2;
    if (hw > 256) return lfem_fail(LFEM_ERR_UNSUPPORTED, "a CSR slot has more than 254 contributions");
    T.heavy_words = hw;
    if (heavy_slots * hw >= INT_MAX) return lfem_fail(LFEM_ERR_UNSUPPORTED, "heavy lists >= 2^31 entries");
    // the stage tail (zero word + heavy sums) must stay addressable by 16-bit byte offsets
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    k_tile_heavymax<<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, bounds, hptr, flags);
    LFEM_CUDA(cudaGetLastError());
    int maxh = 0;
    LFEM_CUDA(cudaMemcpyAsync(&maxh, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    if (8 * ((int64_t)p->mesh->nsym * maxe + 1) >= 0xfff0) return LFEM_OK;  // not ready: lower the budget
    // TMA bulk copies round each tile's ranges out to 16 B: pad both arrays
    LFEM_TRY(dev_alloc_t(&T.pairs, p->nnz + 8, s));
    LFEM_TRY(dev_alloc_t(&T.heavy, heavy_slots * hw + 16, s));
    LFEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 4, s));
    if (n_rows > 0) {
        k_tile_pairs<<<grid_for(n_rows, 128), 128, 0, s>>>(n_rows, tile_of, bounds, hw, p->mesh->nsym, maxe, p->row_ptr,
                                                           p->slot_ptr,
                                                           p->codes, ptr, T.tile_elems, tpos, hptr, T.pairs, T.heavy,
                                                           flags);
        LFEM_CUDA(cudaGetLastError());
    }
    LFEM_TRY(dev_alloc_t(&T.tile_info, (size_t)3 * n_tiles + 3, s));
    k_tile_info<<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, p->row_begin, bounds, hw, p->row_ptr, eptr32, cptr32,
                                                       hptr, lptr32, hcnt, T.tile_info, flags + 2, flags + 3,
                                                       flags + 1);
    LFEM_CUDA(cudaGetLastError());
    LFEM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    LFEM_CUDA(cudaStreamSynchronize(s));
    scope.drop(cnt);
    scope.drop(ptr);
    scope.drop(flags);
    scope.drop(hu);
    scope.drop(hptr);
    scope.drop(eptr32);
    scope.drop(cptr32);
    scope.drop(lptr32);
    scope.drop(hcnt);
    scope.drop(bounds);
    scope.drop(tile_of);
    scope.drop(tpos);
    if (h[0]) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tile code construction failed (" + std::to_string(h[0]) + ")");
    T.max_tile_slots = h[2];
    T.max_tile_heavy = h[3];
    T.max_tile_nodes = h[1];
    T.ready = true;
    return LFEM_OK;
}

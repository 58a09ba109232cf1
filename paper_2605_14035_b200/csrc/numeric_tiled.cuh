// Fused row-tile numeric kernel (TILED variant) -- included by numeric.cu.
//
// One CTA per row tile (tiles.cu).  Per tile:
//   0. one thread arms an mbarrier and issues TMA bulk copies
//      (cp.async.bulk -> UBLKCP) of the tile's element connectivity (tile
//      order), its 16-bit contribution codes and 8-bit slot counts into
//      shared memory;
//   A. each thread takes one tile element: node ids from shared memory,
//      coordinates gathered from global (L2-resident: SFC order), local
//      matrices in fp64 registers (Element<>), symmetric halves stored to the
//      shared-memory stage  stage[kind][sym][e_tile];
//   B. each warp owns a contiguous run of the tile's CSR slots; 32 slots at a
//      time it scans their counts with shuffles, sums each slot's
//      contributions in code order (= ascending element, reading G21) and
//      stores vals[kind][slot] -- 32 consecutive slots per store instruction;
//      no atomics.
// HBM traffic per tile: CSR values (written once), 2 B per contribution code,
// 1 B per slot count, the tile's connectivity, gathered coordinates.
#pragma once
#include <cstdlib>

#ifndef LFEM_P2T_THREADS
#define LFEM_P2T_THREADS 192
#define LFEM_P2T_MINB 2
#define LFEM_P2T_R 256
#endif

namespace {

constexpr int TILE_SMEM_LIMIT = 227 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

struct TileLayout {
    size_t buf_off[2], conn_off, codes_off, cnt_off, buf_bytes, heavy_off, soff_off, total;
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
// stage | 2 x {conn | codes | counts} | heavy-slot lists
__host__ __device__ inline TileLayout tile_layout(int nk, int nsym, int nref, int maxe, int codes_cap, int slots_cap,
                                                  int nwarps, int maxh) {
    TileLayout L;
    const size_t stage = align16(sizeof(double) * (size_t)nk * nsym * maxe);
    L.conn_off = 0;
    L.codes_off = align16(sizeof(int32_t) * ((size_t)maxe * nref + 4));
    L.cnt_off = L.codes_off + align16(sizeof(uint16_t) * ((size_t)codes_cap + 16));
    L.buf_bytes = L.cnt_off + align16((size_t)slots_cap + 32);
    L.buf_off[0] = stage;
    L.buf_off[1] = stage + L.buf_bytes;
    L.heavy_off = stage + 2 * L.buf_bytes;
    L.soff_off = L.heavy_off + align16(sizeof(int) * 2 * (size_t)nwarps * maxh);
    L.total = L.soff_off + align16(sizeof(uint16_t) * ((size_t)slots_cap + 8));
    return L;
}

struct TileArgs {
    int n_tiles;
    int maxe, codes_cap, slots_cap;
    const int4* tile_info;
    const int32_t* tile_elems;
    const int32_t* tile_conn;
    const uint16_t* codes16;
    const uint8_t* slot_cnt;
    const int32_t* elem_list;
    const double* coords;
    const double* coeff;
    double* v[3];
    int* err;
    int debug;  // timing experiments only (LFEM_DEBUG_TILED): bit0 skip phase A, bit1 skip phase B
};

extern __shared__ __align__(16) double tile_smem_d[];  // dynamic shared memory (one view per TU)

struct SmemStageSink {  // stage[kind][sym][e_tile] as offsets into tile_smem_d
    int e, maxe, k1, k2;  // k1 = offset of kind A, k2 = offset of kind Aa (in doubles)
    __device__ __forceinline__ void operator()(int k, int s, double v) const {
        const int kofs = k == 0 ? 0 : (k == 1 ? k1 : k2);
        tile_smem_d[kofs + s * maxe + e] = v;
    }
};

// THREADS per CTA, MINB CTAs per SM, default rows per tile, LIGHT = slots with
// at most LIGHT contributions are summed in the main (coalesced) pass, the
// rest ("heavy": vertex diagonals) in a per-warp second pass; MAXH heavy
// slots recorded per warp and tile.
template <int F> struct TileCfg;
template <> struct TileCfg<FAM_TRI_P1> { static constexpr int THREADS = 256, MINB = 2, R = 512, LIGHT = 2, MAXH = 96; };
template <> struct TileCfg<FAM_TRI_P2> { static constexpr int THREADS = LFEM_P2T_THREADS, MINB = LFEM_P2T_MINB, R = LFEM_P2T_R, LIGHT = 2, MAXH = 64; };
template <> struct TileCfg<FAM_TET_P1> { static constexpr int THREADS = 256, MINB = 1, R = 256, LIGHT = 4, MAXH = 96; };
template <> struct TileCfg<FAM_TET_P2> { static constexpr int THREADS = 256, MINB = 1, R = 128, LIGHT = 4, MAXH = 96; };

__device__ __forceinline__ int warp_incl_scan_i(int v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// thread 0: publish tile info for buffer b and start its TMA bulk copies
__device__ __forceinline__ void issue_tile(const TileArgs& a, unsigned char* smem, const TileLayout& lay, int b,
                                           int4 i0, int4 i1, int4 (*sinfo)[2], uint64_t* bar) {
    sinfo[b][0] = i0;
    sinfo[b][1] = i1;
    unsigned char* buf = smem + lay.buf_off[b];
    const uintptr_t cb = reinterpret_cast<uintptr_t>(a.codes16 + i0.z);
    const uintptr_t ce = reinterpret_cast<uintptr_t>(a.codes16 + i0.z + i0.w);
    const uintptr_t cb16 = cb & ~uintptr_t(15), ce16 = (ce + 15) & ~uintptr_t(15);
    const uintptr_t nb = reinterpret_cast<uintptr_t>(a.slot_cnt + i0.x);
    const uintptr_t nbe = reinterpret_cast<uintptr_t>(a.slot_cnt + i0.x + i0.y);
    const uintptr_t nb16 = nb & ~uintptr_t(15), ne16 = (nbe + 15) & ~uintptr_t(15);
    const uint32_t bytes_q = (uint32_t)i1.w * 4u;
    const uint32_t bytes_c = (uint32_t)(ce16 - cb16), bytes_n = (uint32_t)(ne16 - nb16);
    mbar_arrive_expect_tx(&bar[b], bytes_q + bytes_c + bytes_n);
    if (bytes_q) bulk_g2s(buf + lay.conn_off, a.tile_conn + i1.z, bytes_q, &bar[b]);
    if (bytes_c) bulk_g2s(buf + lay.codes_off, reinterpret_cast<const void*>(cb16), bytes_c, &bar[b]);
    if (bytes_n) bulk_g2s(buf + lay.cnt_off, reinterpret_cast<const void*>(nb16), bytes_n, &bar[b]);
}

// Persistent: CTA c processes tiles c, c + G, c + 2G, ...; the next tile's
// connectivity / codes / counts stream into the other buffer while the
// current tile computes and reduces.
template <int F, bool DM, bool DA, bool DAA>
__global__ void __launch_bounds__(TileCfg<F>::THREADS, TileCfg<F>::MINB) k_tiled(const TileArgs a) {
    using E = Element<F, DM, DA, DAA>;
    constexpr int N = E::N, NS = E::NS, TB = TileCfg<F>::THREADS, NW = TB / 32;
    constexpr int LIGHT = TileCfg<F>::LIGHT, MAXH = TileCfg<F>::MAXH;
    constexpr int NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
    unsigned char* smem = reinterpret_cast<unsigned char*>(tile_smem_d);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ int4 sinfo[2][2];
    __shared__ int warp_sums[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const TileLayout lay = tile_layout(NK, NS, N, a.maxe, a.codes_cap, a.slots_cap, NW, MAXH);
    // offsets (in doubles) of the kinds inside the stage
    const int kst = NS * a.maxe;
    const int ofsM = 0, ofsA = DM ? kst : 0, ofsAa = ((DM ? 1 : 0) + (DA ? 1 : 0)) * kst;
    int* h_list = reinterpret_cast<int*>(smem + lay.heavy_off) + warp * 2 * MAXH;  // [slot, off] pairs

    int t = blockIdx.x;
    int4 n0 = make_int4(0, 0, 0, 0), n1 = n0;  // thread 0: info of the next tile to issue
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (t < a.n_tiles) issue_tile(a, smem, lay, 0, a.tile_info[2 * t], a.tile_info[2 * t + 1], sinfo, bar);
        if (t + G < a.n_tiles) {
            n0 = a.tile_info[2 * (t + G)];
            n1 = a.tile_info[2 * (t + G) + 1];
        }
    }
    __syncthreads();

    for (int it = 0; t < a.n_tiles; ++it, t += G) {
        const int b = it & 1;
        if (tid == 0 && t + G < a.n_tiles) {
            issue_tile(a, smem, lay, b ^ 1, n0, n1, sinfo, bar);
            if (t + 2 * G < a.n_tiles) {
                n0 = a.tile_info[2 * (t + 2 * G)];
                n1 = a.tile_info[2 * (t + 2 * G) + 1];
            }
        }
        mbar_wait(&bar[b], (it >> 1) & 1);
        const int4 i0 = sinfo[b][0], i1 = sinfo[b][1];
        const int s0 = i0.x, ns = i0.y, e0 = i1.x, ne = i1.y;
        // byte offsets of this buffer's arrays inside dynamic shared memory
        const int conn_b = (int)(lay.buf_off[b] + lay.conn_off);
        const int codes_b = (int)(lay.buf_off[b] + lay.codes_off) +
                            (int)(reinterpret_cast<uintptr_t>(a.codes16 + i0.z) & 15);
        const int cnt_b = (int)(lay.buf_off[b] + lay.cnt_off) + (int)(reinterpret_cast<uintptr_t>(a.slot_cnt + s0) & 15);
        const int32_t* s_conn = reinterpret_cast<const int32_t*>(smem + conn_b);
        const uint16_t* s_codes = reinterpret_cast<const uint16_t*>(smem + codes_b);
        const uint8_t* s_cnt = smem + cnt_b;

        // --- A: local matrices of the tile's elements -> shared-memory stage
        for (int i = tid; i < ((a.debug & 1) ? 0 : ne); i += TB) {
            double X[N][3], U[N];
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const int64_t v = s_conn[i * N + j];
#pragma unroll
                for (int c = 0; c < 3; ++c) X[j][c] = __ldg(&a.coords[3 * v + c]);
                U[j] = DAA ? __ldg(&a.coeff[v]) : 0.0;
            }
            SmemStageSink sink{i, a.maxe, ofsA, ofsAa};
            if (!E::compute(X, U, sink)) atomicMin(a.err, __ldg(&a.elem_list[__ldg(&a.tile_elems[e0 + i])]));
        }

        // --- B0: exclusive scan of the slot counts -> s_off (first code of each slot)
        uint16_t* s_off = reinterpret_cast<uint16_t*>(smem + lay.soff_off);
        const int chunk = (ns + TB - 1) / TB;
        const int jb = tid * chunk < ns ? tid * chunk : ns;
        const int je = jb + chunk < ns ? jb + chunk : ns;
        int run = 0;
        for (int j = jb; j < je; ++j) run += s_cnt[j];
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int tv = __shfl_up_sync(0xffffffffu, incl, o);
            incl += lane >= o ? tv : 0;
        }
        if (lane == 31) warp_sums[warp] = incl;
        __syncthreads();  // stage complete; warp totals visible
        int wbase = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) wbase += (w < warp) ? warp_sums[w] : 0;
        int o2 = wbase + incl - run;
        for (int j = jb; j < je; ++j) {
            s_off[j] = (uint16_t)o2;
            o2 += s_cnt[j];
        }
        __syncthreads();

        // --- B1: independent slots, 32 consecutive per warp instruction
        double* vM = DM ? a.v[0] + s0 : nullptr;
        double* vA = DA ? a.v[1] + s0 : nullptr;
        double* vAa = DAA ? a.v[2] + s0 : nullptr;
        int nh = 0;  // heavy slots recorded by this warp
        const int jend = (a.debug & 2) ? 0 : ns;
        for (int j0 = warp * 32; j0 < jend; j0 += TB) {
            const int j = j0 + lane;
            const bool in = j < jend;
            const int c = in ? (int)s_cnt[j] : 0;
            const int off = in ? (int)s_off[j] : 0;
            const bool heavy = c > LIGHT;
            const unsigned hm = __ballot_sync(0xffffffffu, heavy);
            const int hi = nh + __popc(hm & ((1u << lane) - 1u));
            nh += __popc(hm);
            double m = 0.0, st = 0.0, sa = 0.0;
            if (heavy) {
                if (hi < MAXH) {
                    h_list[2 * hi] = j;
                    h_list[2 * hi + 1] = off;
                } else {  // list full: sum in place
                    for (int k = 0; k < c; ++k) {
                        const int code = s_codes[off + k];
                        if (DM) m += tile_smem_d[ofsM + code];
                        if (DA) st += tile_smem_d[ofsA + code];
                        if (DAA) sa += tile_smem_d[ofsAa + code];
                    }
                }
            } else if (!(a.debug & 8)) {
#pragma unroll
                for (int k = 0; k < LIGHT; ++k) {
                    const bool take = k < c;
                    const int code = take ? s_codes[off + k] : 0;
                    if (DM) m += take ? tile_smem_d[ofsM + code] : 0.0;
                    if (DA) st += take ? tile_smem_d[ofsA + code] : 0.0;
                    if (DAA) sa += take ? tile_smem_d[ofsAa + code] : 0.0;
                }
            }
            if (a.debug & 8) { m = st = sa = (double)c; }
            if (in && (!heavy || hi >= MAXH) && (!(a.debug & 4) || m == 1.2345e300)) {
                if (DM) vM[j] = m;
                if (DA) vA[j] = st;
                if (DAA) vAa[j] = sa;
            }
        }
        __syncwarp();
        const int nhl = nh < MAXH ? nh : MAXH;
        for (int h = lane; h < nhl; h += 32) {
            const int j = h_list[2 * h], off = h_list[2 * h + 1], c = s_cnt[j];
            double m = 0.0, st = 0.0, sa = 0.0;
            for (int k = 0; k < c; ++k) {
                const int code = s_codes[off + k];
                if (DM) m += tile_smem_d[ofsM + code];
                if (DA) st += tile_smem_d[ofsA + code];
                if (DAA) sa += tile_smem_d[ofsAa + code];
            }
            if (DM) vM[j] = m;
            if (DA) vA[j] = st;
            if (DAA) vAa[j] = sa;
        }
        __syncthreads();  // stage and buffer b free for reuse
    }
}

template <int F>
size_t tile_smem_bytes(const TilePlan& T, int nk) {
    return tile_layout(nk, FamInfo<F>::NSYM, FamInfo<F>::NREF, T.max_tile_elems, T.max_tile_codes, T.max_tile_slots,
                       TileCfg<F>::THREADS / 32, TileCfg<F>::MAXH).total;
}

template <int F>
lfem_status ensure_tiles(lfem_plan_s* p, int nk, cudaStream_t s) {
    TilePlan& T = p->tiles;
    if (T.ready && T.built_nk >= nk) return LFEM_OK;
    int R = TileCfg<F>::R;
    if (const char* env = std::getenv("LFEM_TILE_ROWS")) {
        const int r = std::atoi(env);
        if (r >= 16) R = r;
    }
    if (T.ready && T.rows_per_tile < R) R = T.rows_per_tile;
    const size_t limit = (size_t)TILE_SMEM_LIMIT / TileCfg<F>::MINB - 2048;
    for (;;) {
        LFEM_TRY(build_tiles(p, R, s));
        if (tile_smem_bytes<F>(T, nk) <= limit && T.max_tile_codes < 65000) break;
        if (R <= 16) return lfem_fail(LFEM_ERR_UNSUPPORTED, "no row-tile size fits in shared memory");
        R /= 2;
    }
    T.built_nk = nk;
    return LFEM_OK;
}

template <int F, bool DM, bool DA, bool DAA>
lfem_status run_tiled(lfem_plan_s* p, const double* coords, const double* coeff, double* const vals[3],
                      cudaStream_t s) {
    constexpr int NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
    LFEM_TRY(ensure_tiles<F>(p, NK, s));
    const TilePlan& T = p->tiles;
    if (T.n_tiles == 0) return LFEM_OK;
    const size_t smem = tile_smem_bytes<F>(T, NK);
    static int attr_smem = -1;  // per instantiation; one process drives one device
    if (attr_smem < (int)smem) {
        LFEM_CUDA(cudaFuncSetAttribute(k_tiled<F, DM, DA, DAA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        attr_smem = (int)smem;
    }
    static int occ = 0;  // resident CTAs per SM for this instantiation
    static int sm_count = 0;
    if (occ == 0) {
        int dev = 0;
        LFEM_CUDA(cudaGetDevice(&dev));
        LFEM_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
        LFEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<F, DM, DA, DAA>, TileCfg<F>::THREADS,
                                                                smem));
        if (occ < 1) occ = 1;
    }
    TileArgs a;
    a.n_tiles = T.n_tiles;
    a.maxe = T.max_tile_elems;
    a.codes_cap = T.max_tile_codes;
    a.slots_cap = T.max_tile_slots;
    a.tile_info = T.tile_info;
    a.tile_elems = T.tile_elems;
    a.tile_conn = T.tile_conn;
    a.codes16 = T.codes16;
    a.slot_cnt = T.slot_cnt;
    a.elem_list = p->elem_list;
    a.coords = coords;
    a.coeff = coeff;
    for (int k = 0; k < 3; ++k) a.v[k] = vals[k];
    a.err = p->err;
    a.debug = 0;
    if (const char* env = std::getenv("LFEM_DEBUG_TILED")) a.debug = std::atoi(env);
    const int grid = T.n_tiles < occ * sm_count ? T.n_tiles : occ * sm_count;
    prof_begin(p, "k_tiled", s);
    k_tiled<F, DM, DA, DAA><<<grid, TileCfg<F>::THREADS, smem, s>>>(a);
    LFEM_CUDA(cudaGetLastError());
    prof_end(p, s);
    return LFEM_OK;
}

template <int F>
lfem_status tiled_kinds(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                        double* const vals[3], cudaStream_t s) {
    switch (kinds) {
    case 1: return run_tiled<F, true, false, false>(p, coords, coeff, vals, s);
    case 2: return run_tiled<F, false, true, false>(p, coords, coeff, vals, s);
    case 3: return run_tiled<F, true, true, false>(p, coords, coeff, vals, s);
    case 4: return run_tiled<F, false, false, true>(p, coords, coeff, vals, s);
    case 5: return run_tiled<F, true, false, true>(p, coords, coeff, vals, s);
    case 6: return run_tiled<F, false, true, true>(p, coords, coeff, vals, s);
    case 7: return run_tiled<F, true, true, true>(p, coords, coeff, vals, s);
    default: return lfem_fail(LFEM_ERR_INVALID_ARG, "kinds");
    }
}

}  // namespace

inline int tiled_default_variant(lfem_plan_s* p) {
    const int f = p->mesh->family;
    return (f == FAM_TRI_P1 || f == FAM_TRI_P2) ? LFEM_NUMERIC_TILED : LFEM_NUMERIC_V0;
}

inline lfem_status tiled_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                                  double* const vals[3], cudaStream_t s) {
    switch (p->mesh->family) {
    case FAM_TRI_P1: return tiled_kinds<FAM_TRI_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2: return tiled_kinds<FAM_TRI_P2>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P1: return tiled_kinds<FAM_TET_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P2: return tiled_kinds<FAM_TET_P2>(p, kinds, coords, coeff, vals, s);
    }
    return lfem_fail(LFEM_ERR_UNSUPPORTED, "family");
}

inline int tiled_launch_count(lfem_plan_s* p) { return p->n_rows > 0 ? 1 : 0; }

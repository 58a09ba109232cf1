// Fused row-tile numeric kernel (TILED variant) -- included by numeric.cu.
//
// Persistent, one CTA per SM, warp-specialised:
//
//   producer   (lane 0 of the first reduce warp): TMA bulk copies
//              (cp.async.bulk -> UBLKCP) of a tile's metadata -- element
//              connectivity (tile order), per-slot code words, heavy lists --
//              into one of 3 shared-memory meta buffers, mbarrier-tracked,
//              up to 3 tiles ahead.
//   compute    CW warps, EPT elements per thread: prefetch node coordinates
//              (and u) of the thread's elements of the NEXT tile into its own
//              shared-memory slots (cp.async -> LDGSTS) while the current tile
//              computes; fp64 geometry;
//              then, one kind at a time (M, A, A_a), the nsym local entries
//              into a shared-memory stage  stage[s * maxe + e_tile].
//   reduce     RW warps: for each kind, every CSR slot of the tile sums its
//              1..c contributions from the stage in symbolic order (ascending
//              element, reading G21) and stores 32 consecutive slots per
//              warp store (streaming, no atomics).
//
// The stage is double-buffered per kind: the reduce warps drain kind k of a
// tile while the compute warps produce kind k+1 (or the next tile's
// geometry), so HBM stores, L2 gathers and the FP64 pipe overlap inside one
// SM.  Staging one kind at a time keeps the stage at nsym * 8 B per element
// (168 B for P2 triangles), which is what lets a CTA hold ~256-element tiles
// (halo recompute ~1.4x) with both buffers resident.
#pragma once
#include <cstdio>
#include <cstdlib>

#ifndef LFEM_RW
#define LFEM_RW 8
#endif
#ifndef LFEM_P1_EPT
#define LFEM_P1_EPT 4
#endif
// P1 triangles (C3): CTA shape (compute warps, reduce warps) and register split; 8 + 8 warps at
// 176 / 80 registers measured best (DESIGN.md §6.3 lists the shapes measured slower)
#ifndef LFEM_P1_CW
#define LFEM_P1_CW 8
#endif
#ifndef LFEM_P1_RW
#define LFEM_P1_RW LFEM_RW
#endif
#ifndef LFEM_P1_REGS_C
#define LFEM_P1_REGS_C (LFEM_P1_RW == 8 && LFEM_P1_CW == 8 ? 176 : 0)
#define LFEM_P1_REGS_R (LFEM_P1_RW == 8 && LFEM_P1_CW == 8 ? 80 : 0)
#endif
// P2 triangles: CTA shape (compute warps, reduce warps, CTAs per SM, elements per compute thread)
#ifndef LFEM_P2_CW
#define LFEM_P2_CW 8
#endif
#ifndef LFEM_P2_RW
#define LFEM_P2_RW 8
#endif
#ifndef LFEM_P2_MINB
#define LFEM_P2_MINB 1
#endif
#ifndef LFEM_P2_EPT
#define LFEM_P2_EPT 1
#endif
#ifndef LFEM_REGS_C
#define LFEM_REGS_C 176
#endif
#ifndef LFEM_REGS_R
#define LFEM_REGS_R 80
#endif
#ifndef LFEM_RUN  // reduce loop unroll (two-slot units)
#define LFEM_RUN 2
#endif
#ifndef LFEM_HEAVY_REGS  // heavy entries per reduce thread summed into registers before the light loop
#define LFEM_HEAVY_REGS 0
#endif
#ifndef LFEM_NMB  // tile metadata buffers (tiles in flight ahead of the compute warps)
#define LFEM_NMB 3
#endif
#ifndef LFEM_NSB  // stage buffers (kind passes in flight between compute and reduce warps)
#define LFEM_NSB 2
#endif


namespace {

constexpr int TILE_SMEM_LIMIT = 227 * 1024;  // per SM (divided by the CTAs per SM)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// order this thread's (and, after a barrier, the CTA's) generic-proxy shared
// memory accesses before subsequent async-proxy (TMA) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    // (a suspend-time hint on try_wait delays the wake-up: measured slower)
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// Poison mode (compile-time -DLFEM_TILED_POISON=1, tests only; compute-sanitizer is closed on
// this pool): every shared-memory buffer is overwritten with a poison pattern (NaN doubles /
// 0xff bytes) as soon as its consumers are done with it, before it is handed back to its
// producer.  A read that raced ahead of a producer (a missing mbarrier wait, async-proxy
// ordering, a stale TMA buffer) or a code word pointing at an unwritten position then yields
// NaN or a wrong value, which the parity tests catch.
#ifndef LFEM_TILED_POISON
#define LFEM_TILED_POISON 0
#endif

// Bounds mode (compile-time -DLFEM_BOUNDS=1, tests only; the stand-in for compute-sanitizer
// memcheck, which this pool refuses): every shared-memory index of the tile kernel (node slots,
// connectivity, stage positions and byte offsets, slot words, heavy entries), every bulk-copy
// size against its buffer, every gathered global node id and every value store against the
// tile's slot range is checked; a violation traps (the launch fails, the tests fail).
#ifndef LFEM_BOUNDS
#define LFEM_BOUNDS 0
#endif
#define LFEM_CHECK(cond)                    \
    do {                                    \
        if (LFEM_BOUNDS && !(cond)) __trap(); \
    } while (0)

// timing experiments only (compile-time, scripts/build_variants.py -DLFEM_TILED_SKIP=..):
// bit0 compute warps skip the kind contractions, bit1 reduce warps skip the slots
#ifndef LFEM_TILED_SKIP
#define LFEM_TILED_SKIP 0
#endif

__device__ __forceinline__ void st_stream(double* p, double v) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// CW compute warps, RW reduce warps, EPT elements per compute thread (tile
// element budget CW*32*EPT), REGS_C / REGS_R setmaxnreg budgets of the two
// roles (0 = launch default).
template <int F> struct TileCfg;
template <> struct TileCfg<FAM_TRI_P1> { static constexpr int CW = LFEM_P1_CW, RW = LFEM_P1_RW, EPT = LFEM_P1_EPT, MINB = 1, REGS_C = LFEM_P1_REGS_C, REGS_R = LFEM_P1_REGS_R; };
template <> struct TileCfg<FAM_TRI_P2> { static constexpr int CW = LFEM_P2_CW, RW = LFEM_P2_RW, MINB = LFEM_P2_MINB, EPT = LFEM_P2_EPT, REGS_C = LFEM_REGS_C, REGS_R = LFEM_REGS_R; };
template <> struct TileCfg<FAM_TRI_P2_Q16> : TileCfg<FAM_TRI_P2> {};
template <> struct TileCfg<FAM_TET_P1> { static constexpr int CW = 8, RW = 4, MINB = 1, EPT = 1, REGS_C = 0, REGS_R = 0; };
template <> struct TileCfg<FAM_TET_P2> { static constexpr int CW = 4, RW = 4, MINB = 1, EPT = 1, REGS_C = 0, REGS_R = 0; };
template <> struct TileCfg<FAM_TET_P2_Q35> : TileCfg<FAM_TET_P2> {};

struct TileLayout {
    size_t stage_bytes;           // one stage buffer
    size_t meta_off[LFEM_NMB], conn_off, pairs_off, heavy_off, halo_off, meta_bytes;
    size_t node_off[2], xyz_off, u_off, node_bytes, total;
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
// stage[2] | meta[3] = {conn16 | pairs | heavy | halo} | nodes[2] = {xyz | u}
__host__ __device__ inline TileLayout tile_layout(int nsym, int nref, int maxe, int slots_cap, int heavy_cap,
                                                  int nodes_cap, int heavy_words) {
    TileLayout L;
    // stage: nsym x maxe entries, then the tail: a zero word
    (void)heavy_words;
    L.stage_bytes = align16(sizeof(double) * ((size_t)nsym * maxe + 1));
    L.conn_off = 0;
    L.pairs_off = align16(sizeof(uint16_t) * ((size_t)maxe * nref + 8));
    L.heavy_off = L.pairs_off + align16(sizeof(uint32_t) * ((size_t)slots_cap + 8));
    L.halo_off = L.heavy_off + align16(sizeof(uint16_t) * ((size_t)heavy_cap + 16));
    L.meta_bytes = L.halo_off + align16(sizeof(int32_t) * ((size_t)nodes_cap + 4));
    L.xyz_off = 0;
    L.u_off = align16(sizeof(double) * (3 * (size_t)nodes_cap + 2));
    L.node_bytes = L.u_off + align16(sizeof(double) * ((size_t)nodes_cap + 2));
    size_t o = LFEM_NSB * L.stage_bytes;
    for (int b = 0; b < LFEM_NMB; ++b) L.meta_off[b] = o + b * L.meta_bytes;
    o += LFEM_NMB * L.meta_bytes;
    for (int b = 0; b < 2; ++b) L.node_off[b] = o + b * L.node_bytes;
    L.total = o + 2 * L.node_bytes;
    return L;
}

struct TileArgs {
    int n_tiles;
    int maxe, slots_cap, heavy_cap, heavy_words;
    int nodes_cap;
    int64_t n_nodes;
    const int4* tile_info;      // 3 per tile: {s0, ns, e0, ne}, {q0, nq, h0, nh}, {g0, nrows, l0, nl}
    const int32_t* tile_elems;
    const uint16_t* conn16;
    const int32_t* halo;
    const uint32_t* pairs;
    const uint16_t* heavy;
    const int32_t* elem_list;
    const double* coords;
    const double* coeff;
    double* v[3];
    int* err;
};

extern __shared__ __align__(16) double tile_smem_d[];  // dynamic shared memory (one view per TU)

struct StageSink {  // stage[s * maxe + e]
    double* st;
    int maxe, e;
    __device__ __forceinline__ void operator()(int s, double v) const {
        LFEM_CHECK(e >= 0 && e < maxe);
        st[s * maxe + e] = v;
    }
};

// producer: publish tile t's info in sinfo[b] and start its bulk copies into meta buffer b
__device__ __forceinline__ void issue_tile(const TileArgs& a, unsigned char* smem, const TileLayout& lay, int t,
                                           int b, int4 (*sinfo)[3], uint64_t* bar) {  // sinfo[LFEM_NMB][3]
    const int4 i0 = a.tile_info[3 * t], i1 = a.tile_info[3 * t + 1], i2 = a.tile_info[3 * t + 2];
    sinfo[b][0] = i0;
    sinfo[b][1] = i1;
    sinfo[b][2] = i2;
    unsigned char* buf = smem + lay.meta_off[b];
    const int p0 = i0.x & ~3, p1 = (i0.x + i0.y + 3) & ~3;    // u32, 16-B aligned
    const int h0 = i1.z & ~7, h1 = (i1.z + i1.w + 7) & ~7;    // u16, 16-B aligned
    const uint32_t bq = (uint32_t)i1.y * 2u, bp = (uint32_t)(p1 - p0) * 4u, bh = (uint32_t)(h1 - h0) * 2u;
    const uint32_t bl = (uint32_t)((i2.w + 3) & ~3) * 4u;     // halo list, 16-B padded per tile
    LFEM_CHECK(lay.conn_off + bq <= lay.pairs_off && lay.pairs_off + bp <= lay.heavy_off &&
               lay.heavy_off + bh <= lay.halo_off && lay.halo_off + bl <= lay.meta_bytes);
    LFEM_CHECK(i0.w <= a.maxe && i0.y <= a.slots_cap && i2.y + 1 + i2.w <= a.nodes_cap + 1);
    fence_proxy_async();
    mbar_arrive_expect_tx(&bar[b], bq + bp + bh + bl);
    if (bq) bulk_g2s(buf + lay.conn_off, a.conn16 + i1.x, bq, &bar[b]);
    if (bp) bulk_g2s(buf + lay.pairs_off, a.pairs + p0, bp, &bar[b]);
    if (bh) bulk_g2s(buf + lay.heavy_off, a.heavy + h0, bh, &bar[b]);
    if (bl) bulk_g2s(buf + lay.halo_off, a.halo + i2.z, bl, &bar[b]);
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// arrive on an mbarrier once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Node buffer of a tile: its owned rows [g0, g0 + nrows) -- one contiguous
// range of coords (24 B per node) and u (8 B) -- come in by two TMA bulk
// copies (16-B aligned around the range: o3 / o1 doubles of lead-in), issued
// by one compute thread on node_full; its halo nodes (sorted global ids in
// the meta buffer) are gathered by all compute threads with cp.async (LDGSTS).
// Node l of the tile is at xyz[o3 + 3 l], u[o1 + l]; halo node h is node
// nrows + 1 + h (the rounded-out bulk copy may write one double past the owned
// range, so one node slot is left free between the two).
__device__ __forceinline__ void prefetch_tile_nodes(const TileArgs& a, bool coef, const int4& i2,
                                                    const int32_t* s_halo, unsigned char* nb, const TileLayout& lay,
                                                    uint64_t* node_full, int tid, int ct) {
    // node_full expects 1 + ct arrivals: thread 0's expect_tx (bulk copies) and every
    // thread's cp.async arrival (its halo gathers); no CTA barrier needed
    double* xyz = reinterpret_cast<double*>(nb + lay.xyz_off);
    double* u = reinterpret_cast<double*>(nb + lay.u_off);
    const int64_t g0 = i2.x;
    const int nrows = i2.y, nh = i2.w;
    const int64_t x0 = 3 * g0, x0a = x0 & ~int64_t(1), xe = 3 * (g0 + nrows);
    const int64_t u0a = g0 & ~int64_t(1), ue = g0 + nrows;
    int64_t x1a = (xe + 1) & ~int64_t(1), u1a = (ue + 1) & ~int64_t(1);
    if (x1a > 3 * a.n_nodes) x1a -= 2;  // never read past the caller's arrays: the tail goes by cp.async
    if (u1a > a.n_nodes) u1a -= 2;
    const int o3 = (int)(x0 - x0a), o1 = (int)(g0 - u0a);
    if (tid == 0) {
        const uint32_t bx = x1a > x0a ? (uint32_t)(x1a - x0a) * 8u : 0u;
        const uint32_t bu = coef && u1a > u0a ? (uint32_t)(u1a - u0a) * 8u : 0u;
        fence_proxy_async();
        mbar_arrive_expect_tx(node_full, bx + bu);
        if (bx) bulk_g2s(xyz, a.coords + x0a, bx, node_full);
        if (bu) bulk_g2s(u, a.coeff + u0a, bu, node_full);
        for (int64_t i = x1a > x0a ? x1a : x0a; i < xe; ++i) cp_async8(xyz + (i - x0a), a.coords + i);
        if (coef)
            for (int64_t i = u1a > u0a ? u1a : u0a; i < ue; ++i) cp_async8(u + (i - u0a), a.coeff + i);
    }
    for (int h = tid; h < nh; h += ct) {
        const int64_t v = s_halo[h];
        const int l = nrows + 1 + h;
        LFEM_CHECK(v >= 0 && v < a.n_nodes && o3 + 3 * l + 2 < (int)((lay.u_off) / sizeof(double)) &&
                   o1 + l < (int)((lay.node_bytes - lay.u_off) / sizeof(double)));
#pragma unroll
        for (int c = 0; c < 3; ++c) cp_async8(xyz + o3 + 3 * l + c, a.coords + 3 * v + c);
        if (coef) cp_async8(u + o1 + l, a.coeff + v);
    }
    cp_async_arrive(node_full);
}

template <int F, bool COEF, int EPT>
__device__ __forceinline__ void read_nodes(const int4& i2, const uint16_t* s_conn, const unsigned char* nb,
                                           const TileLayout& lay, int ne, int ci, int ct,
                                           double (&X)[EPT][FamInfo<F>::NREF][3], double (&U)[EPT][FamInfo<F>::NREF]) {
    constexpr int N = FamInfo<F>::NREF;
    const double* xyz = reinterpret_cast<const double*>(nb + lay.xyz_off) + ((3 * (int64_t)i2.x) & 1);
    const double* u = reinterpret_cast<const double*>(nb + lay.u_off) + (i2.x & 1);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const int e = ci + k * ct;
        if (e < ne) {
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const int l = s_conn[e * N + j];
                LFEM_CHECK(l >= 0 && l < i2.y + 1 + i2.w && l != i2.y && e * N + j < (int)(lay.pairs_off / 2));
#pragma unroll
                for (int c = 0; c < 3; ++c) X[k][j][c] = xyz[3 * l + c];
                U[k][j] = COEF ? u[l] : 0.0;
            }
        }
    }
}

template <int F, bool DM, bool DA, bool DAA>
__global__ void __launch_bounds__((TileCfg<F>::CW + TileCfg<F>::RW) * 32, TileCfg<F>::MINB) k_tiled(const TileArgs a) {
    using E = Elem<F>;
    using Cfg = TileCfg<F>;
    constexpr int N = E::N, CW = Cfg::CW, RW = Cfg::RW, EPT = Cfg::EPT, CT = CW * 32;
    unsigned char* smem = reinterpret_cast<unsigned char*>(tile_smem_d);
    __shared__ int meta_done[LFEM_NMB];  // reduce warps done with the tile in meta buffer b
    __shared__ __align__(8) uint64_t meta_full[LFEM_NMB], stage_full[LFEM_NSB], stage_empty[LFEM_NSB], node_full[2],
        node_empty[2];
    __shared__ int4 sinfo[LFEM_NMB][3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const TileLayout lay = tile_layout(E::NS, N, a.maxe, a.slots_cap, a.heavy_cap, a.nodes_cap, a.heavy_words);
    const int tail_dbl = E::NS * a.maxe;  // stage tail: the zero word
    const int stage_dbl = (int)(lay.stage_bytes / sizeof(double));
    // buffer bases by arithmetic (a dynamically indexed member array would live in local memory)
    const size_t meta0 = lay.meta_off[0], meta_stride = lay.meta_off[1] - lay.meta_off[0];
    const size_t node0 = lay.node_off[0], node_stride = lay.node_off[1] - lay.node_off[0];

    if (tid == 0) {
        for (int b = 0; b < LFEM_NMB; ++b) {
            mbar_init(&meta_full[b], 1);
            meta_done[b] = 0;
        }
        for (int b = 0; b < LFEM_NSB; ++b) {
            mbar_init(&stage_full[b], CT);
            mbar_init(&stage_empty[b], RW * 32);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&node_full[b], 1 + CT);
            mbar_init(&node_empty[b], CT);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b < LFEM_NSB; ++b) tile_smem_d[b * stage_dbl + tail_dbl] = 0.0;  // never written again
    }
    __syncthreads();
    if (tid == CT) {
        for (int k = 0; k < LFEM_NMB; ++k) {
            const int t = blockIdx.x + k * G;
            if (t < a.n_tiles) issue_tile(a, smem, lay, t, k, sinfo, meta_full);
        }
    }

    if (warp < CW) {
        // ------------------------------------------------------------ compute warps
        if (Cfg::REGS_C) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_C));
        int t = blockIdx.x;
        if (t >= a.n_tiles) return;
        double X[EPT][N][3], U[EPT][N];
        uint32_t pass = 0;
        mbar_wait(&meta_full[0], 0);
        prefetch_tile_nodes(a, DAA, sinfo[0][2], reinterpret_cast<const int32_t*>(smem + meta0 + lay.halo_off),
                            smem + node0, lay, &node_full[0], tid, CT);
        for (int it = 0; t < a.n_tiles; ++it, t += G) {
            const int b = it % LFEM_NMB, nb = it & 1;
            const int4 i0 = sinfo[b][0], i2 = sinfo[b][2];
            const int e0 = i0.z, ne = i0.w;
            // this tile's node buffer: bulk copies + every thread's halo gathers, one mbarrier
            mbar_wait(&node_full[nb], (it >> 1) & 1);
            read_nodes<F, DAA, EPT>(i2, reinterpret_cast<const uint16_t*>(smem + meta0 + b * meta_stride + lay.conn_off),
                                    smem + node0 + nb * node_stride, lay, ne, tid, CT, X, U);
            if (LFEM_TILED_POISON) {  // every compute thread has read its nodes: poison the node buffer
                asm volatile("bar.sync 2, %0;" ::"n"(CT) : "memory");
                double* nbuf = reinterpret_cast<double*>(smem + node0 + nb * node_stride);
                for (int i = tid; i < (int)(lay.node_bytes / sizeof(double)); i += CT) nbuf[i] = __longlong_as_double(-1LL);
            }
            mbar_arrive(&node_empty[nb]);
            typename E::Geo geo[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const int e = tid + k * CT;
                if (e < ne && !E::template geometry<DAA>(X[k], U[k], geo[k]))
                    atomicMin(a.err, __ldg(&a.elem_list[__ldg(&a.tile_elems[e0 + e])]));
            }
            if (t + G < a.n_tiles) {  // next tile's nodes -> the other node buffer, in flight during the kinds
                const int bn = (it + 1) % LFEM_NMB;
                mbar_wait(&meta_full[bn], ((it + 1) / LFEM_NMB) & 1);
                const int fill = (it + 1) >> 1;  // fill index of buffer nb ^ 1: its previous contents must be read
                if (fill > 0) mbar_wait(&node_empty[nb ^ 1], (fill - 1) & 1);
                prefetch_tile_nodes(a, DAA, sinfo[bn][2],
                                    reinterpret_cast<const int32_t*>(smem + meta0 + bn * meta_stride + lay.halo_off),
                                    smem + node0 + (nb ^ 1) * node_stride, lay, &node_full[nb ^ 1], tid, CT);
            }
            // one kind per stage pass: wait for a free stage buffer, store, hand it to the reduce warps
#pragma unroll
            for (int kind = 0; kind < 3; ++kind) {
                if ((kind == KIND_M && !DM) || (kind == KIND_A && !DA) || (kind == KIND_AA && !DAA)) continue;
                const int sb = pass % LFEM_NSB;
                const uint32_t use = pass / LFEM_NSB;
                if (use > 0) mbar_wait(&stage_empty[sb], (use - 1) & 1);
                double* st = tile_smem_d + sb * stage_dbl;
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int e = tid + k * CT;
                    if (e < ne && !(LFEM_TILED_SKIP & 1)) {
                        StageSink sink{st, a.maxe, e};
                        if (kind == KIND_M) E::template kind<KIND_M>(geo[k], sink);
                        else if (kind == KIND_A) E::template kind<KIND_A>(geo[k], sink);
                        else E::template kind<KIND_AA>(geo[k], sink);
                    }
                }
                mbar_arrive(&stage_full[sb]);
                ++pass;
            }
        }
    } else {
        // ------------------------------------------------------------ reduce warps (+ producer)
        // Per kind: (1) every CSR slot of the tile in units of two consecutive slots
        // (absolute index 2u, 2u+1): one 8-B load of the two slot words, four stage loads
        // (byte offsets; a missing second contribution is the stage's zero word), one 16-B
        // streaming store -- no case analysis in the loop (a heavy slot's word points at the
        // zero word: 0 is written); consecutive threads take consecutive units (512-B
        // coalesced stores per warp); an odd first / last slot of the tile is done apart.
        // (2) a named barrier of the reduce warps (orders the heavy slots' second store
        // after the first); (3) the heavy slots: one fixed-size entry per thread, loads in
        // parallel, summed in order.  One compact loop serves every kind (instruction-cache
        // footprint).
        if (Cfg::REGS_R) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Cfg::REGS_R));
        constexpr int RT = RW * 32;
        constexpr int NK = (DM ? 1 : 0) + (DA ? 1 : 0) + (DAA ? 1 : 0);
        constexpr int HK = LFEM_HEAVY_REGS;  // heavy entries per thread summed before the light loop
        constexpr int RUN = LFEM_RUN;        // (a macro is not expanded inside #pragma unroll)
        const int rt = tid - CT;
        uint32_t pass = 0;
        for (int it = 0, t = blockIdx.x; t < a.n_tiles; ++it, t += G) {
            const int b = it % LFEM_NMB;
            mbar_wait(&meta_full[b], (it / LFEM_NMB) & 1);
            const int4 i0 = sinfo[b][0], i1 = sinfo[b][1];
            const int s0 = i0.x, ns = (LFEM_TILED_SKIP & 2) ? 0 : i0.y, se = s0 + ns;
            const unsigned char* mb = smem + meta0 + b * meta_stride;
            // slot words of absolute slots [p0, ...), p0 = s0 & ~3 (16-B aligned bulk copy)
            const uint32_t* s_pw = reinterpret_cast<const uint32_t*>(mb + lay.pairs_off);
            const int p0 = s0 & ~3;
            const int hw = a.heavy_words, nent = (LFEM_TILED_SKIP & 2) ? 0 : i1.w / hw;
            const uint16_t* s_heavy = reinterpret_cast<const uint16_t*>(mb + lay.heavy_off);
            const int uA = (s0 + 1) >> 1, uB = se >> 1;  // units with both slots in [s0, se)
#pragma unroll 1
            for (int kk = 0; kk < NK; ++kk) {
                const int kind = DM ? (kk == 0 ? KIND_M : (DA && kk == 1) ? KIND_A : KIND_AA)
                                    : (DA ? (kk == 0 ? KIND_A : KIND_AA) : KIND_AA);
                const int sb = pass % LFEM_NSB;
                mbar_wait(&stage_full[sb], (pass / LFEM_NSB) & 1);
                const unsigned char* st = reinterpret_cast<const unsigned char*>(tile_smem_d + sb * stage_dbl);
                double* out = a.v[kind];
                // heavy entry h: [slot - s0, count, codes...], summed in order (never -0: adding the
                // zero word of unused codes is exact)
                auto heavy_sum = [&](int h, int& slot) {
                    const uint4* ent = reinterpret_cast<const uint4*>(s_heavy + h * hw);
                    const uint4 w0 = ent[0];
                    const int cnt = (int)(w0.x >> 16);
                    slot = (int)(w0.x & 0xffffu);
                    LFEM_CHECK(slot < ns && cnt > 2 && 6 + 8 * (hw / 8 - 1) >= cnt && (h + 1) * hw <= a.heavy_cap + 16);
                    const uint32_t c[6] = {w0.y & 0xffffu, w0.y >> 16, w0.z & 0xffffu, w0.z >> 16,
                                           w0.w & 0xffffu, w0.w >> 16};
                    double x[6];
#pragma unroll
                    for (int k = 0; k < 6; ++k) {
                        LFEM_CHECK(c[k] % 8 == 0 && c[k] <= (uint32_t)tail_dbl * 8u);
                        x[k] = *reinterpret_cast<const double*>(st + c[k]);
                    }
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < 6; ++k) v = v + x[k];
                    for (int blk = 1; 6 + 8 * (blk - 1) < cnt; ++blk) {
                        const uint4 w = ent[blk];
                        const uint32_t d[8] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16,
                                               w.z & 0xffffu, w.z >> 16, w.w & 0xffffu, w.w >> 16};
                        double y[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            LFEM_CHECK(d[k] % 8 == 0 && d[k] <= (uint32_t)tail_dbl * 8u);
                            y[k] = *reinterpret_cast<const double*>(st + d[k]);
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) v = v + y[k];
                    }
                    return v;
                };
                auto slot_value = [&](uint32_t w) {
                    // x0 + x1 in the symbolic order (reading G21); for one contribution x1 = +0 (the
                    // oracle's 0 + x0: the same value, -0 becomes +0 in both)
                    LFEM_CHECK((w & 7u) == 0 && (w & 0xffffu) <= (uint32_t)tail_dbl * 8u &&
                               ((w >> 16) == 0xffffu || (w >> 16) <= (uint32_t)tail_dbl * 8u));
                    const double x0 = *reinterpret_cast<const double*>(st + (w & 0xffffu));
                    const uint32_t c1 = w >> 16;
                    const double x1 = (LFEM_ZERO_WORD || c1 != 0xffffu) ? *reinterpret_cast<const double*>(st + c1) : 0.0;
                    return x0 + x1;
                };
                // heavy sums first (their loads overlap the light loop; the stores wait for the barrier)
                double hval[HK > 0 ? HK : 1];
                int hslot[HK > 0 ? HK : 1];
#pragma unroll
                for (int k = 0; k < HK; ++k) {
                    const int h = rt + k * RT;
                    hslot[k] = -1;
                    hval[k] = 0.0;
                    if (h < nent) hval[k] = heavy_sum(h, hslot[k]);
                }
#pragma unroll RUN
                for (int u = uA + rt; u < uB; u += RT) {
                    LFEM_CHECK(2 * u - p0 + 1 < a.slots_cap + 8 && 2 * u >= s0 && 2 * u + 1 < se);
                    const uint2 w = *reinterpret_cast<const uint2*>(s_pw + (2 * u - p0));
                    const double v0 = slot_value(w.x), v1 = slot_value(w.y);
                    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(out + 2 * u), "d"(v0), "d"(v1) : "memory");
                }
                // (s0 odd and se odd exclude each other when ns = 1: the two edge slots never coincide)
                if (rt == 0 && (s0 & 1) && ns > 0) st_stream(out + s0, slot_value(s_pw[s0 - p0]));
                if (rt == 1 && (se & 1) && ns > 0) st_stream(out + se - 1, slot_value(s_pw[se - 1 - p0]));
                if (nent > 0) asm volatile("bar.sync 1, %0;" ::"n"(RT) : "memory");  // heavy stores land last
#pragma unroll
                for (int k = 0; k < HK; ++k)
                    if (hslot[k] >= 0) st_stream(out + s0 + hslot[k], hval[k]);
                for (int h = rt + HK * RT; h < nent; h += RT) {  // beyond the register-held entries
                    int sl;
                    const double v = heavy_sum(h, sl);
                    st_stream(out + s0 + sl, v);
                }
                if (LFEM_TILED_POISON) {  // every reduce thread has read the stage: poison it (not the zero word)
                    asm volatile("bar.sync 1, %0;" ::"n"(RT) : "memory");
                    double* sw = tile_smem_d + sb * stage_dbl;
                    for (int i = rt; i < tail_dbl; i += RT) sw[i] = __longlong_as_double(-1LL);
                    asm volatile("bar.sync 1, %0;" ::"n"(RT) : "memory");
                }
                mbar_arrive(&stage_empty[sb]);
                ++pass;
            }
            // the last reduce warp to finish this tile refills meta buffer b (no warp blocks on it)
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                const int done = atomicAdd(&meta_done[b], 1);
                if (done == RW - 1) {
                    meta_done[b] = 0;
                    __threadfence_block();
                    if (LFEM_TILED_POISON) {  // the tile's compute and reduce are done with meta buffer b
                        uint4* mw = reinterpret_cast<uint4*>(smem + meta0 + b * meta_stride);
                        for (int i = 0; i < (int)(lay.meta_bytes / 16); ++i) mw[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
                    }
                    if (t + LFEM_NMB * G < a.n_tiles) issue_tile(a, smem, lay, t + LFEM_NMB * G, b, sinfo, meta_full);
                }
            }
        }
    }
}

template <int F>
constexpr int tile_capacity() {
    return TileCfg<F>::CW * 32 * TileCfg<F>::EPT;
}

template <int F>
size_t tile_smem_bytes(const TilePlan& T) {
    return tile_layout(FamInfo<F>::NSYM, FamInfo<F>::NREF, T.max_tile_elems, T.max_tile_slots, T.max_tile_heavy,
                       T.max_tile_nodes, T.heavy_words)
        .total;
}

// Build the tile plan with an element budget of the compute threads' capacity
// (or LFEM_TILE_ELEMS), lowered if the 16-bit codes or shared memory do not fit.
template <int F>
lfem_status ensure_tiles_impl(lfem_plan_s* p, cudaStream_t s) {
    TilePlan& T = p->tiles;
    int emax = tile_capacity<F>();
    // tiny meshes (fewer elements than ~2 full tiles per SM): smaller tiles spread them over the SMs
    // (a tile's pipeline latency, not its work, sets the time there)
    int sms = 148;
    LFEM_TRY(device_sm_count(&sms));
    if (p->n_local < (int64_t)emax * sms * 2) {
        const int64_t e = (p->n_local + sms - 1) / sms;
        emax = (int)(e < 32 ? 32 : (e > emax ? emax : e));
    }
    if (const char* env = std::getenv("LFEM_TILE_ELEMS")) {
        const int r = std::atoi(env);
        if (r >= 8 && r < tile_capacity<F>()) emax = r;
    }
    for (int iter = 0;; ++iter) {
        LFEM_TRY(build_tiles(p, emax, s));
        if (T.ready && T.max_tile_count > tile_capacity<F>())
            return lfem_fail(LFEM_ERR_UNSUPPORTED, "a row touches more elements than the tiled kernel's tile holds");
        if (T.ready && tile_smem_bytes<F>(T) <= (size_t)TILE_SMEM_LIMIT / TileCfg<F>::MINB - 1024) break;
        if (emax <= 8 || iter > 16) return lfem_fail(LFEM_ERR_UNSUPPORTED, "no tile size fits the tiled kernel");
        emax = (int)(emax * 0.9);
    }
    return LFEM_OK;
}

// the tile plan is built once per plan; a failed build leaves no plan behind
// (tiled_ok = 0: AUTO runs V0 on this plan from then on)
template <int F>
lfem_status ensure_tiles(lfem_plan_s* p, cudaStream_t s) {
    if (p->tiles.ready && p->tiled_ok == 1) return LFEM_OK;
    if (p->tiled_ok == 0) return lfem_fail(LFEM_ERR_UNSUPPORTED, "the tile plan does not fit this mesh");
    const lfem_status st = ensure_tiles_impl<F>(p, s);
    if (st != LFEM_OK) {
        free_tiles(p->tiles, s);
        if (st == LFEM_ERR_UNSUPPORTED) p->tiled_ok = 0;
        return st;
    }
    p->tiled_ok = 1;
    return LFEM_OK;
}

template <int F, bool DM, bool DA, bool DAA>
lfem_status run_tiled(lfem_plan_s* p, const double* coords, const double* coeff, double* const vals[3],
                      cudaStream_t s) {
    LFEM_TRY(ensure_tiles<F>(p, s));
    const TilePlan& T = p->tiles;
    if (T.n_tiles == 0) return LFEM_OK;
    const size_t smem = tile_smem_bytes<F>(T);
    constexpr int THREADS = (TileCfg<F>::CW + TileCfg<F>::RW) * 32;
    LFEM_TRY(ensure_smem_attr(reinterpret_cast<const void*>(k_tiled<F, DM, DA, DAA>), (int)smem));
    int sm_count = 148;
    LFEM_TRY(device_sm_count(&sm_count));
    int occ = 0;
    LFEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<F, DM, DA, DAA>, THREADS, smem));
    if (occ < 1) return lfem_fail(LFEM_ERR_UNSUPPORTED, "tiled kernel does not fit on an SM");
    if (TileCfg<F>::REGS_C || TileCfg<F>::REGS_R) {
        // setmaxnreg moves registers inside the CTA's launch allocation: an increase that does not
        // fit would block forever, so refuse such a configuration instead of launching it
        cudaFuncAttributes fa{};
        LFEM_CUDA(cudaFuncGetAttributes(&fa, k_tiled<F, DM, DA, DAA>));
        const long need = 32L * (TileCfg<F>::CW * TileCfg<F>::REGS_C + TileCfg<F>::RW * TileCfg<F>::REGS_R);
        if (need > (long)THREADS * ((fa.numRegs + 7) / 8 * 8))
            return lfem_fail(LFEM_ERR_UNSUPPORTED, "tiled kernel register split exceeds the CTA's allocation");
    }
    TileArgs a;
    a.n_tiles = T.n_tiles;
    a.maxe = T.max_tile_elems;
    a.slots_cap = T.max_tile_slots;
    a.heavy_cap = T.max_tile_heavy;
    a.heavy_words = T.heavy_words;
    a.tile_info = T.tile_info;
    a.tile_elems = T.tile_elems_pos;  // position order (the compute threads' element index)
    a.conn16 = T.conn16;
    a.halo = T.halo;
    a.nodes_cap = T.max_tile_nodes;
    a.n_nodes = p->mesh->n_nodes;
    a.pairs = T.pairs;
    a.heavy = T.heavy;
    a.elem_list = p->elem_list;
    a.coords = coords;
    a.coeff = coeff;
    for (int k = 0; k < 3; ++k) a.v[k] = vals[k];
    a.err = p->err;
    const int grid = T.n_tiles < occ * sm_count ? T.n_tiles : occ * sm_count;
    prof_begin(p, "k_tiled", s);
    k_tiled<F, DM, DA, DAA><<<grid, THREADS, smem, s>>>(a);
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
    return (f == FAM_TRI_P1 || f == FAM_TRI_P2 || f == FAM_TRI_P2_Q16) ? LFEM_NUMERIC_TILED : LFEM_NUMERIC_V0;
}

inline lfem_status tiled_dispatch(lfem_plan_s* p, unsigned kinds, const double* coords, const double* coeff,
                                  double* const vals[3], cudaStream_t s) {
    if (p->mesh->family == FAM_LINE_P1 || p->mesh->family == FAM_LINE_P2 || p->mesh->family == FAM_LINE_P2_Q6)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "the tiled variant has no curve configuration (use V0 / AUTO)");
    if (p->mesh->family == FAM_TET_P2_Q35)
        return lfem_fail(LFEM_ERR_UNSUPPORTED, "the tiled variant has no 35-point tet configuration (use V0 / AUTO)");
    switch (p->mesh->family) {
    case FAM_TRI_P1: return tiled_kinds<FAM_TRI_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2: return tiled_kinds<FAM_TRI_P2>(p, kinds, coords, coeff, vals, s);
    case FAM_TRI_P2_Q16: return tiled_kinds<FAM_TRI_P2_Q16>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P1: return tiled_kinds<FAM_TET_P1>(p, kinds, coords, coeff, vals, s);
    case FAM_TET_P2: return tiled_kinds<FAM_TET_P2>(p, kinds, coords, coeff, vals, s);
    }
    return lfem_fail(LFEM_ERR_UNSUPPORTED, "family");
}

inline int tiled_launch_count(lfem_plan_s* p) { return p->n_rows > 0 ? 1 : 0; }

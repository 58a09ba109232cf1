// Per-element fp64 geometry + local matrices (symmetric halves) for the
// numeric kernels.  Included by numeric.cu after reference.cuh.  Both numeric
// variants (V0 and TILED) call exactly these functions, so they produce the
// same bits.
//
// Mathematics (§3.2, Listing 1):
//   J(xi) = DF(xi) = sum_{j>=2} (x_j - x_1) grad_ref phi_j(xi)^T   (Eq. jacobian_inv P:317-327;
//           differences, reading G24).  grad_ref phi_j is affine in xi for
//           P2 (constant for P1), so J(xi) = J0 + sum_n xi_n J1_n with
//           J0 = sum_j d_j grad phi_j(0), J1_n = sum_j d_j d_n grad phi_j: the
//           per-element part is formed once, each quadrature point costs
//           3*D*D FMAs (instead of 3*D*(nref-1)).
//   surface: G = J^T J, mu = sqrt(det G), K = w mu G^{-1} = (w / mu) adj(G)
//            A_loc(a,b) = sum_q grad_a(q)^T K_q grad_b(q)   (metric form of
//            Eq. Aloc-precise, = Listing 1's B^T B with B = C^T grad, G2)
//   bulk:    mu = |det J|, g_a = J^{-T} grad_a = cof(J) grad_a / det J,
//            A_loc(a,b) = sum_q (w_q / mu_q) (cof grad_a) . (cof grad_b)
//   M_loc(a,b)  = sum_q w_q mu_q phi_a phi_b                    (Eq. P:346)
//   Aa_loc(a,b) = sum_q a(u_h(xi_q)) * (stiffness integrand),  a(u) = 1 + u^2
//                 (BASELINE.json north_star; reading G10: a evaluated at u_h(xi_q))
//
// Structure ("geometry once, one kind at a time"): geometry() turns the
// element's nodes into a few scalars per quadrature point (w mu, K, a); each
// kind is then a separate contraction of those scalars with the constant
// tables pp / gg, emitting the nsym entries of that kind.  The tiled kernel
// stages one kind at a time in shared memory (3x smaller stage than staging
// all kinds together, numeric_tiled.cuh).  Reference-gradient components that
// are identically zero (e.g. d phi_2 / d xi_2 for P2) are skipped at compile
// time.  Bulk stiffness uses the gradient form per quadrature point (cheaper
// than the 6-entry metric form for tets) and recomputes J per kind.
#pragma once
#include "lfem_internal.cuh"
#include "reference.cuh"
#include "tet_moments.cuh"

#ifndef LFEM_TET_MOMENTS  // P2 tet stiffness in moment form (1) or gradient form (0)
#define LFEM_TET_MOMENTS 0
#endif

// Coefficients of the reference shape-function derivatives (small integers):
//   d phi_j / d xi_m (xi) = SA(j,m) + sum_n SB(j,m,n) xi_n
template <int D, int ORDER>
struct Shape {
    static constexpr int NV = D + 1;
    static constexpr int N = ORDER == 1 ? NV : NV + (D == 1 ? 1 : D == 2 ? 3 : 6);
    __host__ __device__ static constexpr int g(int k, int m) { return k == 0 ? -1 : (k == m + 1 ? 1 : 0); }
    __host__ __device__ static constexpr int c(int k) { return k == 0 ? 1 : 0; }
    __host__ __device__ static constexpr int ei(int e) {
        return D == 2 ? (e == 0 ? 0 : e == 1 ? 1 : 2) : (e == 0 ? 0 : e == 1 ? 1 : e == 2 ? 2 : e == 3 ? 0 : e == 4 ? 1 : 2);
    }
    __host__ __device__ static constexpr int ej(int e) {
        return D == 2 ? (e == 0 ? 1 : e == 1 ? 2 : 0) : (e == 0 ? 1 : e == 1 ? 2 : e == 2 ? 0 : 3);
    }
    __host__ __device__ static constexpr int SA(int j, int m) {
        if (ORDER == 1) return g(j, m);
        if (j < NV) return (4 * c(j) - 1) * g(j, m);
        const int e = j - NV, i = ei(e), k = ej(e);
        return 4 * (c(i) * g(k, m) + c(k) * g(i, m));
    }
    __host__ __device__ static constexpr int SB(int j, int m, int n) {
        if (ORDER == 1) return 0;
        if (j < NV) return 4 * g(j, n) * g(j, m);
        const int e = j - NV, i = ei(e), k = ej(e);
        return 4 * (g(i, n) * g(k, m) + g(k, n) * g(i, m));
    }
    // d phi_j / d xi_m vanishes identically
    __host__ __device__ static constexpr bool DZ(int j, int m) {
        bool z = SA(j, m) == 0;
        for (int n = 0; n < D; ++n) z = z && SB(j, m, n) == 0;
        return z;
    }
    // coefficient of the monomial al (1, x, y, x^2, xy, y^2) in d_m phi_a * d_n phi_b
    __host__ __device__ static constexpr int TERM(int a, int b, int m, int n, int al) {
        return al == 0 ? SA(a, m) * SA(b, n)
             : al == 1 ? SA(a, m) * SB(b, n, 0) + SB(a, m, 0) * SA(b, n)
             : al == 2 ? SA(a, m) * SB(b, n, 1 % D) + SB(a, m, 1 % D) * SA(b, n)
             : al == 3 ? SB(a, m, 0) * SB(b, n, 0)
             : al == 4 ? SB(a, m, 0) * SB(b, n, 1 % D) + SB(a, m, 1 % D) * SB(b, n, 0)
                       : SB(a, m, 1 % D) * SB(b, n, 1 % D);
    }
    // surface: integer coefficient of moment (c, al) in A_loc(a, b), c = 11, 12 (+21), 22
    __host__ __device__ static constexpr int MCOEF(int a, int b, int c, int al) {
        return c == 0 ? TERM(a, b, 0, 0, al) : c == 2 ? TERM(a, b, 1 % D, 1 % D, al)
                                                      : TERM(a, b, 0, 1 % D, al) + TERM(a, b, 1 % D, 0, al);
    }
    // compile-time table of MCOEF by symmetric index s = sym(a, b), and which moments are used
    struct MTab {
        int k[N * (N + 1) / 2][3][6];
        bool used[3][6];
    };
    __host__ __device__ static constexpr MTab mtab() {
        MTab t{};
        for (int c = 0; c < 3; ++c)
            for (int al = 0; al < 6; ++al) t.used[c][al] = false;
        for (int a = 0; a < N; ++a)
            for (int b = a; b < N; ++b) {
                const int s = b >= a ? a * N - a * (a - 1) / 2 + (b - a) : 0;
                for (int c = 0; c < 3; ++c)
                    for (int al = 0; al < 6; ++al) {
                        t.k[s][c][al] = MCOEF(a, b, c, al);
                        t.used[c][al] = t.used[c][al] || t.k[s][c][al] != 0;
                    }
            }
        return t;
    }
    // surface metric-form product gg[s][c] (c: 11, 12+21, 22) vanishes identically
    __host__ __device__ static constexpr bool GGZ(int a, int b, int c) {
        return c == 0 ? (DZ(a, 0) || DZ(b, 0))
                      : c == 2 ? (DZ(a, 1 % D) || DZ(b, 1 % D))
                               : ((DZ(a, 0) || DZ(b, 1 % D)) && (DZ(a, 1 % D) || DZ(b, 0)));
    }
};

template <int F> struct FamShape;
template <> struct FamShape<FAM_TRI_P1> { using S = Shape<2, 1>; };
template <> struct FamShape<FAM_TRI_P2> { using S = Shape<2, 2>; };
template <> struct FamShape<FAM_TRI_P2_Q16> { using S = Shape<2, 2>; };
template <> struct FamShape<FAM_LINE_P1> { using S = Shape<1, 1>; };
template <> struct FamShape<FAM_LINE_P2> { using S = Shape<1, 2>; };
template <> struct FamShape<FAM_LINE_P2_Q6> { using S = Shape<1, 2>; };
template <> struct FamShape<FAM_TET_P2_Q35> { using S = Shape<3, 2>; };
template <> struct FamShape<FAM_TET_P1> { using S = Shape<3, 1>; };
template <> struct FamShape<FAM_TET_P2> { using S = Shape<3, 2>; };

// Branch-free fp64 reciprocal square root / reciprocal: hardware approximation
// (MUFU.RSQ64H / MUFU.RCP64H) + two Newton steps (error ~1 ulp).  CUDA's
// rsqrt()/division carry a slow-path branch per call, which splits the
// unrolled quadrature loop into scheduling regions.  Non-positive or
// non-finite arguments are flagged as degenerate by the caller.
__device__ __forceinline__ double rsqrt_nr(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double e = fma(-x * r, r, 1.0);  // 1 - x r^2
        r = fma(0.5 * r, e, r);
    }
    return r;
}

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double e = fma(-x, r, 1.0);
        r = fma(r, e, r);
    }
    return r;
}

// reference coordinates of the quadrature points (constant memory)
constexpr int MAX_NQ = 35;
struct QuadXi {
    double xi[MAX_NQ][3];
};
__constant__ QuadXi c_xi[N_FAMILIES];

enum Kind { KIND_M = 0, KIND_A = 1, KIND_AA = 2 };

template <int F>
struct Elem {
    static constexpr int N = FamInfo<F>::NREF, D = FamInfo<F>::D, NQ = FamInfo<F>::NQ, NS = FamInfo<F>::NSYM;
    // quadrature loops are unrolled except for the 35-point tet rule (code size / compile time)
    static constexpr int QU = (D == 3 && NQ > 16) ? 1 : NQ;
    using S = typename FamShape<F>::S;
    static_assert(S::N == N, "shape table");

    // Per-element scalars handed from geometry() to the kind contractions.
    //  surface: w mu, K = (w / mu) adj(G) (3 entries) and a(u_h) per point;
    //  bulk:    w mu and a(u_h) per point + the Jacobian parts J0, J1.
    // P1 surface: J is constant per element, so the geometry is det*r = mu and
    // r adj(G) (r = 1/mu), the quadrature weights are applied on the fly.
    static constexpr bool P1S = (D == 2 && N == 3);
    // Many-point surface rules (Dunavant-8, 16 points): geometry() accumulates the stiffness
    // moments itself instead of keeping K per point (52 instead of 80 live doubles per element;
    // the same fma sequence in ascending q, so the same bits as forming them in stiffness()).
    static constexpr bool MOMG = (D == 2) && !P1S && NQ > 8;
    struct Geo {
        double mu1, ka[3];  // P1 surface only
        double wmu[NQ];
        double k11[D <= 2 && !MOMG ? NQ : 1], k12[D == 2 && !MOMG ? NQ : 1], k22[D == 2 && !MOMG ? NQ : 1];
        double aq[MOMG ? 1 : NQ];
        double mom[MOMG ? 2 : 1][3][6];  // MOMG: moments of K (A) and of a K (A_a)
        double J0[3][D], J1[3][D][D];  // bulk only (unused on surfaces)
    };

    // J0[c][m], J1[c][m][n] from differences d_j = x_j - x_1
    static __device__ __forceinline__ void jac_parts(const double (&X)[N][3], double (&J0)[3][D],
                                                     double (&J1)[3][D][D]) {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
            double d[N];
#pragma unroll
            for (int j = 1; j < N; ++j) d[j] = X[j][cc] - X[0][cc];
#pragma unroll
            for (int m = 0; m < D; ++m) {
                double s = 0.0;
#pragma unroll
                for (int j = 1; j < N; ++j)
                    if (S::SA(j, m) != 0) s = fma((double)S::SA(j, m), d[j], s);
                J0[cc][m] = s;
#pragma unroll
                for (int n = 0; n < D; ++n) {
                    double t = 0.0;
#pragma unroll
                    for (int j = 1; j < N; ++j)
                        if (S::SB(j, m, n) != 0) t = fma((double)S::SB(j, m, n), d[j], t);
                    J1[cc][m][n] = t;
                }
            }
        }
    }

    static __device__ __forceinline__ void jac_at(const double (&J0)[3][D], const double (&J1)[3][D][D], int q,
                                                  double (&J)[3][D]) {
        constexpr int FI = F;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
            for (int m = 0; m < D; ++m) {
                double v = J0[cc][m];
                if (N > D + 1) {  // P2: affine in xi
#pragma unroll
                    for (int n = 0; n < D; ++n) v = fma(c_xi[FI].xi[q][n], J1[cc][m][n], v);
                }
                J[cc][m] = v;
            }
    }

    // cofactor matrix C (C[k][m] = d det J / d J[k][m]) and det J (bulk)
    static __device__ __forceinline__ double cof(const double (&J)[3][D], double (&C)[3][3]) {
        C[0][0] = J[1][1 % D] * J[2][2 % D] - J[1][2 % D] * J[2][1 % D];
        C[0][1] = J[1][2 % D] * J[2][0] - J[1][0] * J[2][2 % D];
        C[0][2] = J[1][0] * J[2][1 % D] - J[1][1 % D] * J[2][0];
        C[1][0] = J[0][2 % D] * J[2][1 % D] - J[0][1 % D] * J[2][2 % D];
        C[1][1] = J[0][0] * J[2][2 % D] - J[0][2 % D] * J[2][0];
        C[1][2] = J[0][1 % D] * J[2][0] - J[0][0] * J[2][1 % D];
        C[2][0] = J[0][1 % D] * J[1][2 % D] - J[0][2 % D] * J[1][1 % D];
        C[2][1] = J[0][2 % D] * J[1][0] - J[0][0] * J[1][2 % D];
        C[2][2] = J[0][0] * J[1][1 % D] - J[0][1 % D] * J[1][0];
        return J[0][0] * C[0][0] + J[0][1 % D] * C[0][1] + J[0][2 % D] * C[0][2];
    }

    // Geometry of one element; returns false if mu <= 0 or non-finite at some
    // quadrature point (S:240 / S:294 analogue, reading G25).
    template <bool COEF>
    static __device__ __forceinline__ bool geometry(const double (&X)[N][3], const double (&U)[N], Geo& g) {
        const RefTab<F>& T = tab<F>();
        double J0[3][D], J1[3][D][D];
        jac_parts(X, J0, J1);
        bool ok = true;
        if constexpr (P1S) {
            double J[3][D];
            jac_at(J0, J1, 0, J);
            const double g11 = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
            const double g12 = J[0][0] * J[0][1 % D] + J[1][0] * J[1][1 % D] + J[2][0] * J[2][1 % D];
            const double g22 = J[0][1 % D] * J[0][1 % D] + J[1][1 % D] * J[1][1 % D] + J[2][1 % D] * J[2][1 % D];
            const double det = g11 * g22 - g12 * g12;
            ok = (det > 0.0) & (det < INFINITY);
            const double r = rsqrt_nr(det);
            g.mu1 = det * r;
            g.ka[0] = r * g22;
            g.ka[1] = -r * g12;
            g.ka[2] = r * g11;
            if (COEF) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    double u = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) u = fma(U[j], T.phi[q][j], u);
                    g.aq[q] = fma(u, u, 1.0);
                }
            }
        } else {
            if constexpr (MOMG) {
#pragma unroll
                for (int m = 0; m < 2; ++m)
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int al = 0; al < 6; ++al) g.mom[m][c][al] = 0.0;
            }
#pragma unroll QU
            for (int q = 0; q < NQ; ++q) {
                double J[3][D];
                jac_at(J0, J1, q, J);
                if constexpr (D == 1) {
                    // curve: G = |t|^2, mu = |t|, K = w / mu (the d = 1 metric form)
                    const double det = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
                    ok &= (det > 0.0) & (det < INFINITY);
                    const double r = rsqrt_nr(det);
                    g.wmu[q] = T.w[q] * (det * r);
                    g.k11[q] = T.w[q] * r;
                } else if constexpr (D == 2) {
                    const double g11 = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
                    const double g12 = J[0][0] * J[0][1 % D] + J[1][0] * J[1][1 % D] + J[2][0] * J[2][1 % D];
                    const double g22 = J[0][1 % D] * J[0][1 % D] + J[1][1 % D] * J[1][1 % D] + J[2][1 % D] * J[2][1 % D];
                    const double det = g11 * g22 - g12 * g12;
                    ok &= (det > 0.0) & (det < INFINITY);
                    const double r = rsqrt_nr(det);
                    g.wmu[q] = T.w[q] * (det * r);
                    const double c = T.w[q] * r;
                    if constexpr (MOMG) {
                        constexpr typename S::MTab MT = S::mtab();
                        double kc[3] = {c * g22, -c * g12, c * g11};
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc)
#pragma unroll
                            for (int al = 0; al < 6; ++al)
                                if (MT.used[cc][al]) g.mom[0][cc][al] = fma(kc[cc], T.mono[q][al], g.mom[0][cc][al]);
                        if (COEF) {
                            double u = 0.0;
#pragma unroll
                            for (int j = 0; j < N; ++j) u = fma(U[j], T.phi[q][j], u);
                            const double aq = fma(u, u, 1.0);
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc)
#pragma unroll
                                for (int al = 0; al < 6; ++al)
                                    if (MT.used[cc][al])
                                        g.mom[1][cc][al] = fma(aq * kc[cc], T.mono[q][al], g.mom[1][cc][al]);
                        }
                    } else {
                        g.k11[D == 2 && !MOMG ? q : 0] = c * g22;
                        g.k12[D == 2 && !MOMG ? q : 0] = -c * g12;
                        g.k22[D == 2 && !MOMG ? q : 0] = c * g11;
                    }
                } else {
                    double C[3][3];
                    const double adet = fabs(cof(J, C));
                    ok &= (adet > 0.0) & (adet < INFINITY);
                    g.wmu[q] = T.w[q] * adet;
                }
                if (COEF && !MOMG) {
                    double u = 0.0;
#pragma unroll
                    for (int j = 0; j < N; ++j) u = fma(U[j], T.phi[q][j], u);
                    g.aq[MOMG ? 0 : q] = fma(u, u, 1.0);
                }
            }
            if constexpr (D == 3) {
#pragma unroll
                for (int cc = 0; cc < 3; ++cc)
#pragma unroll
                    for (int m = 0; m < D; ++m) {
                        g.J0[cc][m] = J0[cc][m];
#pragma unroll
                        for (int n = 0; n < D; ++n) g.J1[cc][m][n] = J1[cc][m][n];
                    }
            }
        }
        return ok;
    }

    // M_loc(s) = sum_q w_q mu_q phi_a phi_b   -> sink(s, value), s ascending.
    // Quadrature loop outside, entries inside: nsym independent accumulation
    // chains (ILP); each entry still sums its terms in ascending q.
    template <class Sink>
    static __device__ __forceinline__ void mass(const Geo& g, Sink& sink) {
        const RefTab<F>& T = tab<F>();
        double m[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) m[s] = 0.0;
#pragma unroll QU
        for (int q = 0; q < NQ; ++q) {
            const double wmu = P1S ? T.w[q] * g.mu1 : g.wmu[q];
#pragma unroll
            for (int s = 0; s < NS; ++s) m[s] = fma(wmu, T.pp[q][s], m[s]);
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) sink(s, m[s]);
    }

    // A_loc (COEF = false) or A_a,loc (COEF = true) -> sink(s, value)
    template <bool COEF, class Sink>
    static __device__ __forceinline__ void stiffness(const Geo& g, Sink& sink) {
        const RefTab<F>& T = tab<F>();
        if constexpr (D == 1) {
            // curve: A_loc(a,b) = sum_q (w_q / mu_q) dphi_a dphi_b
            double acc[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) acc[s] = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const double kc = COEF ? g.aq[q] * g.k11[q] : g.k11[q];
#pragma unroll
                for (int s = 0; s < NS; ++s) acc[s] = fma(kc, T.gg[q][s][0], acc[s]);
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) sink(s, acc[s]);
        } else if constexpr (D == 2) {
            // Moment form.  The reference gradients are affine in xi, so
            //   A_loc(a,b) = sum_q sum_c K_q^c (d phi_a d phi_b)_c(xi_q)
            //              = sum_{c, al} MCOEF(a,b,c,al) * mom[c][al],
            //   mom[c][al] = sum_q K_q^c xi_q^al  (al over 1, x, y, x^2, xy, y^2),
            // with small integer MCOEF known at compile time (instruction
            // immediates): 18 moments from 36 table constants instead of one
            // table constant per term.  Same integrand and rule; only the
            // rounding order differs from the per-point form (reading G23).
            constexpr typename S::MTab MT = S::mtab();
            double mom[3][6];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int al = 0; al < 6; ++al) mom[c][al] = MOMG ? g.mom[MOMG && COEF ? 1 : 0][c][al] : 0.0;
            if constexpr (!MOMG) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    double kc[3] = {g.k11[D == 2 && !MOMG ? q : 0], g.k12[D == 2 && !MOMG ? q : 0],
                                    g.k22[D == 2 && !MOMG ? q : 0]};
                    if (P1S)
#pragma unroll
                        for (int c = 0; c < 3; ++c) kc[c] = T.w[q] * g.ka[c];
                    if (COEF)
#pragma unroll
                        for (int c = 0; c < 3; ++c) kc[c] = g.aq[MOMG ? 0 : q] * kc[c];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
#pragma unroll
                        for (int al = 0; al < 6; ++al)
                            if (MT.used[c][al]) mom[c][al] = fma(kc[c], T.mono[q][al], mom[c][al]);
                }
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                double v = 0.0;
                bool first = true;
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int al = 0; al < 6; ++al) {
                        const int k = MT.k[s][c][al];
                        if (k != 0) {
                            v = first ? (double)k * mom[c][al] : fma((double)k, mom[c][al], v);
                            first = false;
                        }
                    }
                sink(s, v);
            }
        } else if constexpr (N == 10 && LFEM_TET_MOMENTS) {
            // P2 tets, moment form (tet_moments.cuh, generated): per point the symmetric
            // K_q = (w_q / |det J|) cof^T cof (6 entries), accumulated against the 10 monomials
            // of degree <= 2 of xi_q; the 55 entries are integer combinations of the 60 moments
            // (741 terms) -- 38 % fewer FP64 operations than the gradient form below.
            double mom[6][10];
#pragma unroll
            for (int c = 0; c < 6; ++c)
#pragma unroll
                for (int al = 0; al < 10; ++al) mom[c][al] = 0.0;
#pragma unroll QU
            for (int q = 0; q < NQ; ++q) {
                double J[3][D], C[3][3];
                jac_at(g.J0, g.J1, q, J);
                const double adet = fabs(cof(J, C));
                double c = T.w[q] * rcp_nr(adet);
                if (COEF) c = c * g.aq[q];
                double K[6];
                constexpr int KM[6] = {0, 1, 2, 0, 0, 1}, KN[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    double v = C[0][KM[i]] * C[0][KN[i]];
                    v = fma(C[1][KM[i]], C[1][KN[i]], v);
                    v = fma(C[2][KM[i]], C[2][KN[i]], v);
                    K[i] = c * v;
                }
#pragma unroll
                for (int i = 0; i < 6; ++i)
#pragma unroll
                    for (int al = 0; al < 10; ++al) mom[i][al] = fma(K[i], T.mono3[D == 3 ? q : 0][al], mom[i][al]);
            }
            tet_moment_combine(mom, sink);
        } else {
            double acc[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) acc[s] = 0.0;
#pragma unroll QU
            for (int q = 0; q < NQ; ++q) {
                double J[3][D], C[3][3];
                jac_at(g.J0, g.J1, q, J);
                const double adet = fabs(cof(J, C));
                double c = T.w[q] * rcp_nr(adet);
                if (COEF) c = c * g.aq[q];
                double gr[N][3];
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        double v = 0.0;
#pragma unroll
                        for (int m = 0; m < D; ++m)
                            if (!S::DZ(a, m)) v = fma(C[k][m], T.dphi[q][a][m], v);
                        gr[a][k] = v;
                    }
#pragma unroll
                for (int a = 0; a < N; ++a)
#pragma unroll
                    for (int b = a; b < N; ++b) {
                        const int s = sym_index(N, a, b);
                        double st = gr[a][0] * gr[b][0];
                        st = fma(gr[a][1], gr[b][1], st);
                        st = fma(gr[a][2], gr[b][2], st);
                        acc[s] = fma(c, st, acc[s]);
                    }
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) sink(s, acc[s]);
        }
    }

    template <int KIND, class Sink>
    static __device__ __forceinline__ void kind(const Geo& g, Sink& sink) {
        if (KIND == KIND_M) mass(g, sink);
        else if (KIND == KIND_A) stiffness<false>(g, sink);
        else stiffness<true>(g, sink);
    }
};

// Reference-element tables of liblfem, in __constant__ memory -- the B200
// counterpart of ℓFEM's precompute_surface_dD_Pk / precompute_bulk_dD_Pk
// (§5.2; Listing 1 l.4-7 P:585-588).  Computed on the
// host from the closed-form Lagrange basis (PAPER.md Eq. form_functions_s2dp2
// P:268-273 with the Lagrange vertex functions of reading G1; tet edge order
// G26) and the quadrature rules fixed by BASELINE.json (readings G6-G9).
//
// Include in exactly ONE translation unit (numeric.cu): __constant__ symbols
// are per-TU without relocatable device code.
//
// Per quadrature point q (symmetric half index s = sym(a,b), a <= b):
//   w[q], phi[q][a], dphi[q][a][m]            basis values / reference gradients
//   pp[q][s]     = phi_a phi_b                  (mass integrand, Eq. reference_quadrature_mass)
//   gg[q][s][0..2] = d1a d1b, d1a d2b + d2a d1b, d2a d2b
//                  (surface metric form of Eq. Aloc-precise P:337:
//                   grad_a . C C^T grad_b = d_a^T G^{-1} d_b)
//   mono[q][0..5] = 1, x, y, x^2, xy, y^2 at xi_q = (x, y) (surface stiffness moments)
#pragma once
#include <algorithm>
#include <cmath>

#include "lfem_internal.cuh"

template <int F>
struct RefTab {
    static constexpr int NREF = FamInfo<F>::NREF, D = FamInfo<F>::D, NQ = FamInfo<F>::NQ,
                         NSYM = FamInfo<F>::NSYM;
    // (tables a family's kernels never read are one entry long: 64 KB of constant memory)
    double w[NQ];
    double phi[NQ][NREF];
    double dphi[D == 3 ? NQ : 1][NREF][D];   // bulk stiffness (gradient form)
    double pp[NQ][NSYM];
    double gg[D == 1 ? NQ : 1][NSYM][3];     // curves (metric form)
    double mono[D == 2 ? NQ : 1][6];         // surfaces: 1, x, y, x^2, x y, y^2 at xi_q (stiffness moments)
    double mono3[D == 3 ? NQ : 1][10];       // P2 tets: 1, x, y, z, xx, xy, xz, yy, yz, zz at xi_q
};

__constant__ RefTab<FAM_TRI_P1> c_tab_tri1;
__constant__ RefTab<FAM_TRI_P2> c_tab_tri2;
__constant__ RefTab<FAM_TET_P1> c_tab_tet1;
__constant__ RefTab<FAM_TET_P2> c_tab_tet2;
__constant__ RefTab<FAM_TRI_P2_Q16> c_tab_tri2q;
__constant__ RefTab<FAM_LINE_P1> c_tab_line1;
__constant__ RefTab<FAM_LINE_P2> c_tab_line2;
__constant__ RefTab<FAM_TET_P2_Q35> c_tab_tet2q;
__constant__ RefTab<FAM_LINE_P2_Q6> c_tab_line2q;

template <int F> __device__ __forceinline__ const RefTab<F>& tab();
template <> __device__ __forceinline__ const RefTab<FAM_TRI_P1>& tab<FAM_TRI_P1>() { return c_tab_tri1; }
template <> __device__ __forceinline__ const RefTab<FAM_TRI_P2>& tab<FAM_TRI_P2>() { return c_tab_tri2; }
template <> __device__ __forceinline__ const RefTab<FAM_TET_P1>& tab<FAM_TET_P1>() { return c_tab_tet1; }
template <> __device__ __forceinline__ const RefTab<FAM_TET_P2>& tab<FAM_TET_P2>() { return c_tab_tet2; }
template <> __device__ __forceinline__ const RefTab<FAM_TRI_P2_Q16>& tab<FAM_TRI_P2_Q16>() { return c_tab_tri2q; }
template <> __device__ __forceinline__ const RefTab<FAM_LINE_P1>& tab<FAM_LINE_P1>() { return c_tab_line1; }
template <> __device__ __forceinline__ const RefTab<FAM_LINE_P2>& tab<FAM_LINE_P2>() { return c_tab_line2; }
template <> __device__ __forceinline__ const RefTab<FAM_TET_P2_Q35>& tab<FAM_TET_P2_Q35>() { return c_tab_tet2q; }
template <> __device__ __forceinline__ const RefTab<FAM_LINE_P2_Q6>& tab<FAM_LINE_P2_Q6>() { return c_tab_line2q; }

namespace refhost {

// quadrature points in reference coordinates xi (d = 2: (xi1, xi2); d = 3)
struct Rule {
    int nq;
    double xi[35][3];
    double w[35];
};

inline Rule rule_tri3() {
    Rule r{};
    r.nq = 3;
    const double t = 1.0 / 6.0, u = 2.0 / 3.0;
    const double P[3][2] = {{t, t}, {u, t}, {t, u}};
    for (int q = 0; q < 3; ++q) { r.xi[q][0] = P[q][0]; r.xi[q][1] = P[q][1]; r.w[q] = 1.0 / 6.0; }
    return r;
}

inline Rule rule_tri6() {
    Rule r{};
    r.nq = 6;
    const double a = 0.44594849091596488632, b = 0.09157621350977074346;
    const double wa = 0.2233815896780114657 * 0.5, wb = 0.10995174365532186764 * 0.5;
    const double P[6][2] = {{a, a}, {1.0 - 2.0 * a, a}, {a, 1.0 - 2.0 * a},
                            {b, b}, {1.0 - 2.0 * b, b}, {b, 1.0 - 2.0 * b}};
    for (int q = 0; q < 6; ++q) {
        r.xi[q][0] = P[q][0];
        r.xi[q][1] = P[q][1];
        r.w[q] = q < 3 ? wa : wb;
    }
    return r;
}

// Dunavant's 16-point degree-8 rule (weights for area 1/2): centroid, three (a, a, 1-2a)
// orbits, one (a, b, c) orbit -- constants of the published rule, 25 digits
inline Rule rule_tri16() {
    Rule r{};
    r.nq = 0;
    auto add = [&r](double l1, double l2, double w) {  // xi = (lambda_2, lambda_3)
        r.xi[r.nq][0] = l1;
        r.xi[r.nq][1] = l2;
        r.w[r.nq] = w;
        ++r.nq;
    };
    add(1.0 / 3.0, 1.0 / 3.0, 0.07215780383889358412554556);
    const double A[3] = {0.4592925882927231560288155, 0.1705693077517602066222935, 0.05054722831703097545842355};
    const double W[3] = {0.04754581713364231239694805, 0.05160868526735912514089578, 0.01622924881159904015546296};
    for (int o = 0; o < 3; ++o) {
        const double a = A[o], c = 1.0 - 2.0 * a;
        add(a, a, W[o]);
        add(c, a, W[o]);
        add(a, c, W[o]);
    }
    const double a4 = 0.008394777409957605337213835, b4 = 0.2631128296346381134217858, c4 = 1.0 - a4 - b4;
    const double w4 = 0.01361515708721749713242235;
    add(a4, b4, w4);
    add(b4, a4, w4);
    add(a4, c4, w4);
    add(c4, a4, w4);
    add(b4, c4, w4);
    add(c4, b4, w4);
    return r;
}

// Gauss-Legendre on [0, 1] (curves): xi = 1/2 -+ h, weights sum to 1
inline Rule rule_line(int npts) {
    Rule r{};
    r.nq = npts;
    if (npts == 6) {
        // six points (reading G38): the roots t of the Legendre polynomial P_6 on [-1, 1], by Newton
        // from Chebyshev-like starts (three-term recurrence, derivative from P_5), mapped to [0, 1];
        // weight 1 / ((1 - t^2) P_6'(t)^2) on the unit interval
        for (int i = 0; i < 6; ++i) {
            double t = -std::cos(3.141592653589793238 * (i + 0.75) / 6.5);
            double d6 = 1.0;
            for (int it = 0; it < 60; ++it) {
                double pm = 1.0, pc = t;  // P_0, P_1
                for (int n = 1; n < 6; ++n) {
                    const double pn = ((2 * n + 1) * t * pc - n * pm) / (n + 1);
                    pm = pc;
                    pc = pn;
                }
                d6 = 6.0 * (pm - t * pc) / (1.0 - t * t);  // P_6'(t) from P_5 = pm, P_6 = pc
                t -= pc / d6;
            }
            r.xi[i][0] = 0.5 * (t + 1.0);
            r.w[i] = 1.0 / ((1.0 - t * t) * d6 * d6);
        }
        return r;
    }
    if (npts == 2) {
        const double h = 0.5 / std::sqrt(3.0);
        r.xi[0][0] = 0.5 - h;
        r.xi[1][0] = 0.5 + h;
        r.w[0] = r.w[1] = 0.5;
    } else {
        const double h = 0.5 * std::sqrt(0.6);
        r.xi[0][0] = 0.5 - h;
        r.xi[1][0] = 0.5;
        r.xi[2][0] = 0.5 + h;
        r.w[0] = r.w[2] = 5.0 / 18.0;
        r.w[1] = 4.0 / 9.0;
    }
    return r;
}

inline Rule rule_tet4() {
    Rule r{};
    r.nq = 4;
    const double al = (5.0 - std::sqrt(5.0)) / 20.0, be = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0;
    const double P[4][3] = {{al, al, al}, {be, al, al}, {al, be, al}, {al, al, be}};
    for (int q = 0; q < 4; ++q) {
        for (int m = 0; m < 3; ++m) r.xi[q][m] = P[q][m];
        r.w[q] = 1.0 / 24.0;
    }
    return r;
}

inline Rule rule_tet11() {
    Rule r{};
    r.nq = 11;
    const double c = 1.0 / 14.0, C = 11.0 / 14.0;
    const double s = std::sqrt(5.0 / 14.0);
    const double a = 0.25 * (1.0 + s), b = 0.25 * (1.0 - s);
    const double P[11][3] = {{0.25, 0.25, 0.25},
                             {c, c, c}, {C, c, c}, {c, C, c}, {c, c, C},
                             {a, b, b}, {b, a, b}, {b, b, a}, {a, a, b}, {a, b, a}, {b, a, a}};
    for (int q = 0; q < 11; ++q) {
        for (int m = 0; m < 3; ++m) r.xi[q][m] = P[q][m];
        r.w[q] = q == 0 ? -74.0 / 5625.0 : (q < 5 ? 343.0 / 45000.0 : 56.0 / 2250.0);
    }
    return r;
}

// Degree-7 fully symmetric positive tet rule, 35 points (reading G39; weights for volume 1/6):
// centroid; (a,a,a,1-3a); (a,a,1/2-a,1/2-a); two (a,a,b,1-2a-b) orbits.  Orbits expanded here
// in reference coordinates xi = (lambda_2, lambda_3, lambda_4).
inline Rule rule_tet35() {
    Rule r{};
    r.nq = 0;
    auto orbit = [&r](double l0, double l1, double l2, double l3, double w) {
        double v[4] = {l0, l1, l2, l3};
        // every distinct permutation (lexicographic enumeration of index permutations)
        int idx[4] = {0, 1, 2, 3};
        double seen[24][4];
        int ns = 0;
        do {
            double p[4] = {v[idx[0]], v[idx[1]], v[idx[2]], v[idx[3]]};
            bool dup = false;
            for (int k = 0; k < ns && !dup; ++k)
                dup = seen[k][0] == p[0] && seen[k][1] == p[1] && seen[k][2] == p[2] && seen[k][3] == p[3];
            if (dup) continue;
            for (int m = 0; m < 4; ++m) seen[ns][m] = p[m];
            ++ns;
            r.xi[r.nq][0] = p[1];
            r.xi[r.nq][1] = p[2];
            r.xi[r.nq][2] = p[3];
            r.w[r.nq] = w;
            ++r.nq;
        } while (std::next_permutation(idx, idx + 4));
    };
    orbit(0.25, 0.25, 0.25, 0.25, 0.01591421491068847481009640601953773030655);
    const double a1 = 0.315701149778202799423429999593311488426;
    orbit(a1, a1, a1, 1.0 - 3.0 * a1, 0.00705493020166117151271436179975778958127);
    const double a2 = 0.4495101774016036312369461770134375340242;
    orbit(a2, a2, 0.5 - a2, 0.5 - a2, 0.005316154638809596655712470680490409516245);
    const double a3 = 0.1888338310260010477364311038545857550051, b3 = 0.5751716375870000234832415770223075196671;
    orbit(a3, a3, b3, 1.0 - 2.0 * a3 - b3, 0.006201188454722436894935926865246853385281);
    const double a4 = 0.02126547254148324598883610149981994107435, b4 = 0.1466388138184849469042224171521277240548;
    orbit(a4, a4, b4, 1.0 - 2.0 * a4 - b4, 0.001351795138317223594350572248516090026183);
    return r;
}

// Lagrange basis at xi: values and gradients w.r.t. xi.
// barycentric l0 = 1 - sum xi, l_k = xi_k; grad l0 = (-1,..), grad l_k = e_k.
inline void basis_eval(int d, int order, const double* xi, double* phi, double (*dphi)[3]) {
    double l[4], gl[4][3];
    l[0] = 1.0;
    for (int m = 0; m < d; ++m) l[0] -= xi[m];
    for (int m = 0; m < 3; ++m) gl[0][m] = (m < d) ? -1.0 : 0.0;
    for (int k = 1; k <= d; ++k) {
        l[k] = xi[k - 1];
        for (int m = 0; m < 3; ++m) gl[k][m] = (m == k - 1) ? 1.0 : 0.0;
    }
    const int nv = d + 1;
    if (order == 1) {
        for (int a = 0; a < nv; ++a) {
            phi[a] = l[a];
            for (int m = 0; m < 3; ++m) dphi[a][m] = gl[a][m];
        }
        return;
    }
    for (int a = 0; a < nv; ++a) {
        phi[a] = l[a] * (2.0 * l[a] - 1.0);
        for (int m = 0; m < 3; ++m) dphi[a][m] = (4.0 * l[a] - 1.0) * gl[a][m];
    }
    static const int e2[3][2] = {{0, 1}, {1, 2}, {2, 0}};
    static const int e3[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};
    const int ne = d == 1 ? 1 : d == 2 ? 3 : 6;
    for (int k = 0; k < ne; ++k) {
        const int i = d <= 2 ? e2[k][0] : e3[k][0];
        const int j = d <= 2 ? e2[k][1] : e3[k][1];
        phi[nv + k] = 4.0 * l[i] * l[j];
        for (int m = 0; m < 3; ++m) dphi[nv + k][m] = 4.0 * (gl[i][m] * l[j] + l[i] * gl[j][m]);
    }
}

template <int F>
void fill(RefTab<F>& t, const Rule& r, int d, int order) {
    constexpr int N = RefTab<F>::NREF;
    for (int q = 0; q < RefTab<F>::NQ; ++q) {
        double phi[10], dphi[10][3];
        basis_eval(d, order, r.xi[q], phi, dphi);
        const double x = r.xi[q][0], y = r.xi[q][1];
        constexpr int D = RefTab<F>::D;
        if (D == 2) {
            t.mono[D == 2 ? q : 0][0] = 1.0;
            t.mono[D == 2 ? q : 0][1] = x;
            t.mono[D == 2 ? q : 0][2] = y;
            t.mono[D == 2 ? q : 0][3] = x * x;
            t.mono[D == 2 ? q : 0][4] = x * y;
            t.mono[D == 2 ? q : 0][5] = y * y;
        }
        if (D == 3) {
            const double z = r.xi[q][2];
            const double m3[10] = {1.0, x, y, z, x * x, x * y, x * z, y * y, y * z, z * z};
            for (int al = 0; al < 10; ++al) t.mono3[D == 3 ? q : 0][al] = m3[al];
        }
        t.w[q] = r.w[q];
        for (int a = 0; a < N; ++a) {
            t.phi[q][a] = phi[a];
            if (D == 3)
                for (int m = 0; m < d; ++m) t.dphi[D == 3 ? q : 0][a][m] = dphi[a][m];
        }
        for (int a = 0; a < N; ++a)
            for (int b = a; b < N; ++b) {
                const int s = sym_index(N, a, b);
                t.pp[q][s] = phi[a] * phi[b];
                if (D == 1) {
                    t.gg[D == 1 ? q : 0][s][0] = dphi[a][0] * dphi[b][0];
                    t.gg[D == 1 ? q : 0][s][1] = dphi[a][0] * dphi[b][1] + dphi[a][1] * dphi[b][0];
                    t.gg[D == 1 ? q : 0][s][2] = dphi[a][1] * dphi[b][1];
                }
            }
    }
}

}  // namespace refhost

// =============================================================================
// lfem ORACLE — plain, slow, obviously-correct CPU reference for the ℓFEM
// assembly hot path (arxiv/paper_2605_14035).  TEST INFRASTRUCTURE ONLY:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path
// (paper_2605_14035_b200/) never links, imports or calls it, and shares no
// code, header, table or constant with it.
//
// What it computes, for every pair of
// global nodes (i, j) in the requested rows:
//   M_ij    = sum_{E ∋ i,j} sum_q w_q mu_E(xi_q) phi_i(xi_q) phi_j(xi_q)
//             (PAPER.md Eq. "M matrix" P:298 and Eq. reference_quadrature_mass)
//   A_ij    = sum_{E ∋ i,j} sum_q w_q mu_E(xi_q) g_i(xi_q) . g_j(xi_q)
//             (Eq. "A matrix" P:301-302, Eq. reference_quadrature_stiffness P:349)
//   Aa_ij   = sum_{E ∋ i,j} sum_q w_q mu_E(xi_q) a(u_h(xi_q)) g_i . g_j,
//             u_h(xi_q) = sum_c u_c phi_c(xi_q), a(u) = 1 + u^2
//             (BASELINE.json north_star; pattern of Listing 2, reading G10)
// with mu_E = |t1 x t2| = sqrt(det J^T J) on surfaces (Listing 1 l.16-17)
// or |det J| in bulk (Eq. basic integral formula P:287), and the tangential
// gradient g = J (J^T J)^{-1} grad_ref(phi) on surfaces (= Listing 1's
// L^{-T}[grad phi; 0], reading G2) or g = J^{-T} grad_ref(phi) in
// bulk (Remark P:278-281).  J = sum_{j>=2} (x_j - x_1) grad_ref(phi_j)^T
// (Eq. jacobian_inv P:317-327 written with differences, reading G24).
//
// Algorithm (the paper's "naive" element loop P:464-474):
//   1. reference data from the closed-form basis below (P:268-273 with the
//      Lagrange vertex functions of reading G1; tet edge order reading G26);
//   2. rows are split into blocks; each block collects the elements having a
//      node in it (ascending element id), loops over them, loops over the
//      quadrature points in rule order, forms full nref x nref local
//      matrices and adds entry (a, b) into std::map[(conn[e,a], conn[e,b])]
//      when conn[e,a] is a requested row;
//   3. the map's (row, col) order is CSR order (explicit zeros kept, G19).
// Per-slot summation order: ascending element id, then (a, b) (reading G21).
// Curves (Table 4 P:646-660 "surface 1D"): P1/P2
// line elements in R^3 with Gauss-Legendre rules; mu = |t| and g = t |t|^-2 dphi,
// the d = 1 case of the surface formulas.
//
// Right-hand sides, for every requested row j:
//   load:  b_j = sum_{E ∋ j} sum_q w_q mu_E(xi_q) f_h(xi_q) phi_j(xi_q),
//          f_h = sum_c f_c phi_c  (Eq. "load vector" P:168-177; with the
//          element rule this is exactly b = M f)
//   KLL:   with u = (nu_1, nu_2, nu_3, H) nodal (u = (n; H)),
//          alpha^2(xi_q) = |grad_Gamma_h nu_h|^2 = sum_k |sum_c nu_{c,k} g_c|^2
//          (Frobenius norm, Listing 2 line 2),
//          f_{k,j} = sum_E sum_q w_q mu alpha^2 u_{h,k}(xi_q) phi_j(xi_q),
//          k = 1..4 (f_1 = first three, f_2 = H component; P:784-789,
//          Listing 2 lines 3-4).  Surfaces only.
// Per-row summation order: ascending element id (one entry per element).
// Degenerate element (mu <= 0 or non-finite at a quadrature point) or a node
// index out of range -> error code with the lowest offending element id.
//
// Every function here is pinned by tests/test_oracle_*.py (closed forms,
// invariants, brute force, exactness); see DESIGN.md §4 for the pin table.
// =============================================================================
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <thread>
#include <utility>
#include <vector>

namespace {

enum { SURFACE_TRI = 0, BULK_TET = 1, SURFACE_LINE = 2 };
enum { Q_DEFAULT = 0, Q_TRI3_DEG2 = 1, Q_TRI6_DEG4 = 2, Q_TET4_DEG2 = 3, Q_TET11_DEG4 = 4, Q_TRI16_DEG8 = 5,
       Q_LINE2_DEG3 = 6, Q_LINE3_DEG5 = 7, Q_TET35_DEG7 = 8, Q_LINE6_DEG11 = 9 };

// dimension of the reference element: curves 1, surfaces 2, bulk 3
int dim_of(int domain) { return domain == SURFACE_LINE ? 1 : domain == SURFACE_TRI ? 2 : 3; }
enum { K_MASS = 1, K_STIFF = 2, K_STIFF_COEF = 4 };
enum { OK = 0, ERR_INVALID_ARG = 1, ERR_UNSUPPORTED = 2, ERR_INDEX = 3, ERR_DEGENERATE = 4 };

// ---------------------------------------------------------------------------
// Quadrature rules on the reference simplex, as barycentric points + weights.
// Triangle (0,0),(1,0),(0,1): area 1/2; xi = (lambda2, lambda3).
// Tetrahedron: volume 1/6; xi = (lambda2, lambda3, lambda4).
// (Rules fixed by BASELINE.json configs, reading G6-G9.)
// ---------------------------------------------------------------------------
struct QPoint { double lam[4]; double w; };

void add_orbit3(std::vector<QPoint>& r, double a, double b, double c, double w) {
    // all distinct permutations of (a, b, c)
    double v[3] = {a, b, c};
    std::vector<std::array<double, 3>> seen;
    std::sort(v, v + 3);
    do {
        std::array<double, 3> p = {v[0], v[1], v[2]};
        if (std::find(seen.begin(), seen.end(), p) == seen.end()) {
            seen.push_back(p);
            QPoint q;
            q.lam[0] = p[0]; q.lam[1] = p[1]; q.lam[2] = p[2]; q.lam[3] = 0.0;
            q.w = w;
            r.push_back(q);
        }
    } while (std::next_permutation(v, v + 3));
}

void add_orbit4(std::vector<QPoint>& r, double a, double b, double c, double d, double w) {
    double v[4] = {a, b, c, d};
    std::vector<std::array<double, 4>> seen;
    std::sort(v, v + 4);
    do {
        std::array<double, 4> p = {v[0], v[1], v[2], v[3]};
        if (std::find(seen.begin(), seen.end(), p) == seen.end()) {
            seen.push_back(p);
            QPoint q;
            for (int i = 0; i < 4; ++i) q.lam[i] = p[i];
            q.w = w;
            r.push_back(q);
        }
    } while (std::next_permutation(v, v + 4));
}

bool make_rule(int quad, std::vector<QPoint>& r) {
    r.clear();
    switch (quad) {
    case Q_TRI3_DEG2:
        // 3 permutations of (2/3, 1/6, 1/6), weight 1/6 (interior rule, reading G7)
        add_orbit3(r, 2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0, 1.0 / 6.0);
        return true;
    case Q_TRI6_DEG4: {
        // symmetric 6-point degree-4 rule
        const double a = 0.44594849091596488632, wa = 0.2233815896780114657 / 2.0;
        const double b = 0.09157621350977074346, wb = 0.10995174365532186764 / 2.0;
        add_orbit3(r, a, a, 1.0 - 2.0 * a, wa);
        add_orbit3(r, b, b, 1.0 - 2.0 * b, wb);
        return true;
    }
    case Q_TRI16_DEG8: {
        // Dunavant's 16-point degree-8 rule (the paper's load-vector rule; SURVEY
        // §8(f) N2): centroid, three (a, a, 1-2a) orbits, one (a, b, c) orbit; weights for area
        // 1/2.  Constants solved here from the degree-8 moment equations (40 digits) and pinned
        // by the exactness test (exact to degree 8, not 9).
        add_orbit3(r, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0, 0.07215780383889358412554556);
        const double a1 = 0.4592925882927231560288155, a2 = 0.1705693077517602066222935,
                     a3 = 0.05054722831703097545842355;
        add_orbit3(r, a1, a1, 1.0 - 2.0 * a1, 0.04754581713364231239694805);
        add_orbit3(r, a2, a2, 1.0 - 2.0 * a2, 0.05160868526735912514089578);
        add_orbit3(r, a3, a3, 1.0 - 2.0 * a3, 0.01622924881159904015546296);
        const double a4 = 0.008394777409957605337213835, b4 = 0.2631128296346381134217858;
        add_orbit3(r, a4, b4, 1.0 - a4 - b4, 0.01361515708721749713242235);
        return true;
    }
    case Q_LINE2_DEG3:
    case Q_LINE3_DEG5: {
        // Gauss-Legendre on [0, 1] (curves, N2): lam = (1 - xi, xi), weights sum to 1
        const bool three = quad == Q_LINE3_DEG5;
        const double h = three ? 0.5 * std::sqrt(3.0 / 5.0) : 0.5 / std::sqrt(3.0);
        const double xs[3] = {0.5 - h, 0.5 + h, 0.5};
        const double ws[3] = {three ? 5.0 / 18.0 : 0.5, three ? 5.0 / 18.0 : 0.5, 4.0 / 9.0};
        for (int k = 0; k < (three ? 3 : 2); ++k) {
            QPoint q;
            q.lam[0] = 1.0 - xs[k];
            q.lam[1] = xs[k];
            q.lam[2] = q.lam[3] = 0.0;
            q.w = ws[k];
            r.push_back(q);
        }
        return true;
    }
    case Q_LINE6_DEG11: {
        // 6-point Gauss-Legendre on [0, 1] (reading G38: the paper's "Gauss ... of order 10" for
        // curves, read as the smallest Gauss rule exact to degree >= 10, i.e. degree 11):
        // nodes are the roots of P_6 mapped to [0, 1], weights w = 1 / ((1 - t^2) P_6'(t)^2)
        // (halved for the unit interval) -- computed here by Newton on the three-term recurrence
        for (int k = 0; k < 6; ++k) {
            double t = std::cos(M_PI * (k + 0.75) / 6.5), dp = 0.0;
            for (int it = 0; it < 100; ++it) {
                double p0 = 1.0, p1 = t;
                for (int n = 2; n <= 6; ++n) {
                    const double p2 = ((2.0 * n - 1.0) * t * p1 - (n - 1.0) * p0) / n;
                    p0 = p1;
                    p1 = p2;
                }
                dp = 6.0 * (t * p1 - p0) / (t * t - 1.0);
                const double dt = p1 / dp;
                t -= dt;
                if (std::fabs(dt) < 1e-17) break;
            }
            QPoint q;
            q.lam[1] = 0.5 * (1.0 + t);
            q.lam[0] = 1.0 - q.lam[1];
            q.lam[2] = q.lam[3] = 0.0;
            q.w = 1.0 / ((1.0 - t * t) * dp * dp);  // (2 / ((1 - t^2) P6'^2)) / 2
            r.push_back(q);
        }
        return true;
    }
    case Q_TET35_DEG7: {
        // fully symmetric, positive, interior degree-7 rule with 35 points (reading G39: stands in
        // for the paper's Jaskowiec-Sukumar degree-7 tetrahedral rule, whose constants are not
        // in the container): orbits S4, S31 (a), S22 (a), 2 x S211 (a, b); solved here from the
        // degree-7 moment equations of the S4-invariant polynomials (50 digits), weights for volume 1/6
        add_orbit4(r, 0.25, 0.25, 0.25, 0.25, 0.01591421491068847481009640601953773030655);
        const double a1 = 0.315701149778202799423429999593311488426;
        add_orbit4(r, a1, a1, a1, 1.0 - 3.0 * a1, 0.00705493020166117151271436179975778958127);
        const double a2 = 0.4495101774016036312369461770134375340242;
        add_orbit4(r, a2, a2, 0.5 - a2, 0.5 - a2, 0.005316154638809596655712470680490409516245);
        const double a3 = 0.1888338310260010477364311038545857550051, b3 = 0.5751716375870000234832415770223075196671;
        add_orbit4(r, a3, a3, b3, 1.0 - 2.0 * a3 - b3, 0.006201188454722436894935926865246853385281);
        const double a4 = 0.02126547254148324598883610149981994107435, b4 = 0.1466388138184849469042224171521277240548;
        add_orbit4(r, a4, a4, b4, 1.0 - 2.0 * a4 - b4, 0.001351795138317223594350572248516090026183);
        return true;
    }
    case Q_TET4_DEG2: {
        const double s5 = std::sqrt(5.0);
        const double al = (5.0 - s5) / 20.0, be = (5.0 + 3.0 * s5) / 20.0;
        add_orbit4(r, al, al, al, be, 1.0 / 24.0);
        return true;
    }
    case Q_TET11_DEG4: {
        // Keast 11-point degree-4 rule (reading G8): NEGATIVE centroid weight
        const double s = std::sqrt(5.0 / 14.0);
        const double a = (1.0 + s) / 4.0, b = (1.0 - s) / 4.0;
        add_orbit4(r, 0.25, 0.25, 0.25, 0.25, -74.0 / 5625.0);
        add_orbit4(r, 1.0 / 14.0, 1.0 / 14.0, 1.0 / 14.0, 11.0 / 14.0, 343.0 / 45000.0);
        add_orbit4(r, a, a, b, b, 56.0 / 2250.0);
        return true;
    }
    default:
        return false;
    }
}

// ---------------------------------------------------------------------------
// Lagrange basis on the reference simplex, written in barycentric
// coordinates lam[0..d]; reference gradients are w.r.t. xi = (lam[1..d]),
// with d lam[0]/d xi_m = -1 and d lam[m]/d xi_m = 1.
//   P1: phi_a = lam_a.
//   P2 triangle (reading G1): vertices lam_a (2 lam_a - 1);
//       edges 4=(1,2), 5=(2,3), 6=(3,1): 4 lam_i lam_j.
//   P2 tet (reading G26): vertices lam_a (2 lam_a - 1); edges
//       (1,2),(2,3),(3,1),(1,4),(2,4),(3,4): 4 lam_i lam_j.
// ---------------------------------------------------------------------------
const int TRI_EDGES[3][2] = {{0, 1}, {1, 2}, {2, 0}};
const int TET_EDGES[6][2] = {{0, 1}, {1, 2}, {2, 0}, {0, 3}, {1, 3}, {2, 3}};

// d lam_k / d xi_m  (k = 0..d, m = 0..d-1)
double dlam(int k, int m) {
    if (k == 0) return -1.0;
    return (k == m + 1) ? 1.0 : 0.0;
}

int nref_of(int domain, int order) {
    const int d = dim_of(domain);
    if (order == 1) return d + 1;
    return (d + 1) * (d + 2) / 2;
}

// phi[a], grad[a][m] at barycentric point lam
void basis(int domain, int order, const double* lam, double* phi, double (*grad)[3]) {
    const int d = dim_of(domain);
    for (int a = 0; a < 10; ++a) { grad[a][0] = grad[a][1] = grad[a][2] = 0.0; }
    if (order == 1) {
        for (int a = 0; a <= d; ++a) {
            phi[a] = lam[a];
            for (int m = 0; m < d; ++m) grad[a][m] = dlam(a, m);
        }
        return;
    }
    for (int a = 0; a <= d; ++a) {
        phi[a] = lam[a] * (2.0 * lam[a] - 1.0);
        for (int m = 0; m < d; ++m) grad[a][m] = (4.0 * lam[a] - 1.0) * dlam(a, m);
    }
    const int ne = (d == 1) ? 1 : (d == 2) ? 3 : 6;  // curves: one edge (1,2), the midpoint node
    for (int e = 0; e < ne; ++e) {
        const int i = (d <= 2) ? TRI_EDGES[e][0] : TET_EDGES[e][0];
        const int j = (d <= 2) ? TRI_EDGES[e][1] : TET_EDGES[e][1];
        const int a = d + 1 + e;
        phi[a] = 4.0 * lam[i] * lam[j];
        for (int m = 0; m < d; ++m) grad[a][m] = 4.0 * (lam[i] * dlam(j, m) + lam[j] * dlam(i, m));
    }
}

// ---------------------------------------------------------------------------
// Local matrices of one element (full nref x nref, row-major), plain loops.
// Returns OK or ERR_DEGENERATE.
// ---------------------------------------------------------------------------
struct Ref {
    int domain, order, nref, d;
    std::vector<QPoint> rule;
    std::vector<std::array<double, 10>> phi;                  // [q][a]
    std::vector<std::array<std::array<double, 3>, 10>> grad;  // [q][a][m]
};

bool make_ref(int domain, int order, int quad, Ref& R) {
    if (domain != SURFACE_TRI && domain != BULK_TET && domain != SURFACE_LINE) return false;
    if (order != 1 && order != 2) return false;
    if (quad == Q_DEFAULT) {
        if (domain == SURFACE_LINE) quad = (order == 1) ? Q_LINE2_DEG3 : Q_LINE3_DEG5;
        else if (domain == SURFACE_TRI) quad = (order == 1) ? Q_TRI3_DEG2 : Q_TRI6_DEG4;
        else quad = (order == 1) ? Q_TET4_DEG2 : Q_TET11_DEG4;
    }
    if (domain == SURFACE_TRI && quad != Q_TRI3_DEG2 && quad != Q_TRI6_DEG4 && quad != Q_TRI16_DEG8) return false;
    if (domain == BULK_TET && quad != Q_TET4_DEG2 && quad != Q_TET11_DEG4 && quad != Q_TET35_DEG7) return false;
    if (domain == SURFACE_LINE && quad != Q_LINE2_DEG3 && quad != Q_LINE3_DEG5 && quad != Q_LINE6_DEG11) return false;
    R.domain = domain;
    R.order = order;
    R.d = dim_of(domain);
    R.nref = nref_of(domain, order);
    if (!make_rule(quad, R.rule)) return false;
    R.phi.resize(R.rule.size());
    R.grad.resize(R.rule.size());
    for (size_t q = 0; q < R.rule.size(); ++q) {
        double phi[10], grad[10][3];
        basis(domain, order, R.rule[q].lam, phi, grad);
        for (int a = 0; a < 10; ++a) {
            R.phi[q][a] = phi[a];
            for (int m = 0; m < 3; ++m) R.grad[q][a][m] = grad[a][m];
        }
    }
    return true;
}

// 3x3 inverse by cofactors (plain)
bool inv3(const double A[3][3], double Ai[3][3], double* det_out) {
    const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    const double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
    const double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    const double det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
    *det_out = det;
    if (!(det != 0.0) || !std::isfinite(det)) return false;
    Ai[0][0] = c00 / det;
    Ai[1][0] = c01 / det;
    Ai[2][0] = c02 / det;
    Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
    Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
    Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
    Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
    Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
    Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    return true;
}

// J (3 x d) at quadrature point q: column m = sum_{j>=2} (x_j - x_1) dphi_j/dxi_m
void jacobian(const Ref& R, const double* X /* nref x 3 */, size_t q, double J[3][3]) {
    const int n = R.nref, d = R.d;
    for (int c = 0; c < 3; ++c) J[c][0] = J[c][1] = J[c][2] = 0.0;
    for (int j = 1; j < n; ++j)
        for (int c = 0; c < 3; ++c)
            for (int m = 0; m < d; ++m)
                J[c][m] += (X[3 * j + c] - X[c]) * R.grad[q][j][m];
}

// Measure mu and the gradients g[a] (3-vectors) of the basis at quadrature
// point q from the Jacobian J (3 x d):
// formulation 0: the north star's  g = J G^{-1} grad (surface), J^{-T} grad (bulk)
// formulation 1: Listing 1's  g = L^{-T} [grad; 0] with L = [t1 t2 t1 x t2]
//                (columns; reading G2) -- surfaces only; used as a second,
//                independent formulation by the brute-force pin.
int point_gradients(const Ref& R, const double J[3][3], size_t q, int formulation, double* mu, double g[10][3]) {
    const int n = R.nref, d = R.d;
    if (d == 1) {
        // curve: G = |t|^2, mu = |t|, g = t G^{-1} d phi / d xi  (the d = 1 case of J G^{-1} grad)
        if (formulation != 0) return ERR_UNSUPPORTED;
        const double G = J[0][0] * J[0][0] + J[1][0] * J[1][0] + J[2][0] * J[2][0];
        *mu = std::sqrt(G);
        if (!(*mu > 0.0) || !std::isfinite(*mu)) return ERR_DEGENERATE;
        for (int a = 0; a < n; ++a)
            for (int c = 0; c < 3; ++c) g[a][c] = J[c][0] * (R.grad[q][a][0] / G);
        return OK;
    }
    if (d == 2) {
        double G[2][2];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                G[a][b] = 0.0;
                for (int c = 0; c < 3; ++c) G[a][b] += J[c][a] * J[c][b];
            }
        const double detG = G[0][0] * G[1][1] - G[0][1] * G[1][0];
        *mu = std::sqrt(detG);
        if (!(*mu > 0.0) || !std::isfinite(*mu)) return ERR_DEGENERATE;
        if (formulation == 0) {
            const double Gi[2][2] = {{G[1][1] / detG, -G[0][1] / detG},
                                     {-G[1][0] / detG, G[0][0] / detG}};
            for (int a = 0; a < n; ++a) {
                double s[2];
                for (int m = 0; m < 2; ++m)
                    s[m] = Gi[m][0] * R.grad[q][a][0] + Gi[m][1] * R.grad[q][a][1];
                for (int c = 0; c < 3; ++c) g[a][c] = J[c][0] * s[0] + J[c][1] * s[1];
            }
        } else {
            double L[3][3], Li[3][3], dummy;
            const double nrm[3] = {J[1][0] * J[2][1] - J[2][0] * J[1][1],
                                   J[2][0] * J[0][1] - J[0][0] * J[2][1],
                                   J[0][0] * J[1][1] - J[1][0] * J[0][1]};
            for (int c = 0; c < 3; ++c) { L[c][0] = J[c][0]; L[c][1] = J[c][1]; L[c][2] = nrm[c]; }
            if (!inv3(L, Li, &dummy)) return ERR_DEGENERATE;
            for (int a = 0; a < n; ++a)
                for (int c = 0; c < 3; ++c)  // (L^{-T} v)_c = sum_k Li[k][c] v_k
                    g[a][c] = Li[0][c] * R.grad[q][a][0] + Li[1][c] * R.grad[q][a][1];
        }
    } else {
        double Ji[3][3], det;
        if (!inv3(J, Ji, &det)) return ERR_DEGENERATE;
        *mu = std::fabs(det);
        if (!(*mu > 0.0) || !std::isfinite(*mu)) return ERR_DEGENERATE;
        for (int a = 0; a < n; ++a)
            for (int c = 0; c < 3; ++c)  // (J^{-T} v)_c = sum_k Ji[k][c] v_k
                g[a][c] = Ji[0][c] * R.grad[q][a][0] + Ji[1][c] * R.grad[q][a][1] +
                          Ji[2][c] * R.grad[q][a][2];
    }
    return OK;
}

// Full local matrices; formulation as in point_gradients.
int element_matrices(const Ref& R, const double* X /* nref x 3 */, const double* u /* nref or null */,
                     int formulation, double* Ml, double* Al, double* Aal) {
    const int n = R.nref;
    for (int i = 0; i < n * n; ++i) { Ml[i] = 0.0; Al[i] = 0.0; Aal[i] = 0.0; }
    for (size_t q = 0; q < R.rule.size(); ++q) {
        const double w = R.rule[q].w;
        double J[3][3];
        jacobian(R, X, q, J);
        double mu = 0.0;
        double g[10][3];
        const int st = point_gradients(R, J, q, formulation, &mu, g);
        if (st != OK) return st;
        double aq = 1.0;
        if (u) {
            double uq = 0.0;
            for (int j = 0; j < n; ++j) uq += u[j] * R.phi[q][j];
            aq = 1.0 + uq * uq;
        }
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                const double gg = g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2];
                Ml[a * n + b] += w * mu * R.phi[q][a] * R.phi[q][b];
                Al[a * n + b] += w * mu * gg;
                Aal[a * n + b] += w * mu * aq * gg;
            }
    }
    return OK;
}

enum { RHS_LOAD = 1, RHS_KLL = 2 };

int rhs_ncomp(int kind) { return kind == RHS_LOAD ? 1 : 4; }

// Local right-hand side of one element (nref x ncomp, row-major [a][k]).
//   RHS_LOAD: U = f (nref x 1):  F[a] = sum_q w mu f_h(xi_q) phi_a(xi_q)
//   RHS_KLL:  U = (nu_1, nu_2, nu_3, H) (nref x 4):
//             alpha^2 = sum_k |sum_c U[c][k] g_c|^2            (Listing 2 l.2)
//             F[a][k] = sum_q w mu alpha^2 u_{h,k} phi_a       (Listing 2 l.3-4)
// Fabs (optional): the same sums evaluated with every term replaced by its absolute
// value (|U|, |phi|, |g_c|) -- the scale of the rounding error of any evaluation order
// (running error bound), used by the parity tolerance (reading G33).
int element_rhs(const Ref& R, const double* X, const double* U, int kind, int formulation, double* F,
                double* Fabs = nullptr) {
    const int n = R.nref, nc = rhs_ncomp(kind);
    for (int i = 0; i < n * nc; ++i) {
        F[i] = 0.0;
        if (Fabs) Fabs[i] = 0.0;
    }
    for (size_t q = 0; q < R.rule.size(); ++q) {
        const double w = R.rule[q].w;
        double J[3][3];
        jacobian(R, X, q, J);
        double mu = 0.0;
        double g[10][3];
        const int st = point_gradients(R, J, q, formulation, &mu, g);
        if (st != OK) return st;
        double uq[4] = {0.0, 0.0, 0.0, 0.0};  // u_h(xi_q), per component
        for (int k = 0; k < nc; ++k)
            for (int c = 0; c < n; ++c) uq[k] += U[c * nc + k] * R.phi[q][c];
        double weight = w * mu;
        double wabs = std::fabs(w) * mu;
        if (kind == RHS_KLL) {
            // grad_Gamma_h nu_k = sum_c nu_ck g_c = sum_{c>=2} (nu_ck - nu_1k) g_c, since
            // sum_c g_c = J G^-1 sum_c grad phi_c = 0 (differences as for J, reading G24).
            // Tolerance scale (reading G33): the first-order rounding error of
            // alpha^2 = sum_k |G_k|^2 is 2 sum_k |G_k| |dG_k| with |dG_k| <~ eps B_k,
            // B_k = sum_{c>=2} |nu_ck - nu_1k| |g_c|, so alpha^2 is scaled by
            // alpha^2 + 2 sum_k |G_k| B_k.
            double alpha2 = 0.0, cross = 0.0;
            for (int k = 0; k < 3; ++k) {
                double grad_nu_k[3] = {0.0, 0.0, 0.0};  // grad_Gamma_h of component k of nu_h
                double bound_k = 0.0;                   // B_k
                for (int c = 1; c < n; ++c) {
                    const double d = U[c * nc + k] - U[k];
                    for (int i = 0; i < 3; ++i) grad_nu_k[i] += d * g[c][i];
                    bound_k += std::fabs(d) * std::sqrt(g[c][0] * g[c][0] + g[c][1] * g[c][1] + g[c][2] * g[c][2]);
                }
                double gk2 = 0.0;
                for (int i = 0; i < 3; ++i) gk2 += grad_nu_k[i] * grad_nu_k[i];
                alpha2 += gk2;
                cross += std::sqrt(gk2) * bound_k;
            }
            weight *= alpha2;
            wabs *= alpha2 + 2.0 * cross;
        }
        for (int a = 0; a < n; ++a)
            for (int k = 0; k < nc; ++k) F[a * nc + k] += weight * uq[k] * R.phi[q][a];
        if (Fabs) {
            double uabs[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k = 0; k < nc; ++k)
                for (int c = 0; c < n; ++c) uabs[k] += std::fabs(U[c * nc + k] * R.phi[q][c]);
            for (int a = 0; a < n; ++a)
                for (int k = 0; k < nc; ++k) Fabs[a * nc + k] += wabs * uabs[k] * std::fabs(R.phi[q][a]);
        }
    }
    return OK;
}

struct Csr {
    int64_t n_rows = 0, nnz = 0;
    int64_t* row_ptr = nullptr;
    int32_t* col_idx = nullptr;
    double* vals[3] = {nullptr, nullptr, nullptr};
};

}  // namespace

extern "C" {

struct oracle_csr {
    int64_t n_rows;
    int64_t nnz;
    int64_t* row_ptr;   // n_rows + 1
    int32_t* col_idx;   // nnz
    double* vals[3];    // [M, A, Aa], nnz each (null if not requested)
    int64_t bad_elem;   // lowest offending element id, or -1
};

void oracle_free(oracle_csr* c) {
    if (!c) return;
    std::free(c->row_ptr);
    std::free(c->col_idx);
    for (int k = 0; k < 3; ++k) std::free(c->vals[k]);
    c->row_ptr = nullptr; c->col_idx = nullptr;
    c->vals[0] = c->vals[1] = c->vals[2] = nullptr;
}

int oracle_nref(int domain, int order) { return nref_of(domain, order); }

// Quadrature rule as used by the oracle (for the exactness pins).
int oracle_rule(int quad, int* nq, double* lam /* 64 x 4 */, double* w /* 64 */) {
    std::vector<QPoint> r;
    if (!make_rule(quad, r) || r.size() > 64) return ERR_UNSUPPORTED;
    *nq = (int)r.size();
    for (size_t q = 0; q < r.size(); ++q) {
        for (int i = 0; i < 4; ++i) lam[4 * q + i] = r[q].lam[i];
        w[q] = r[q].w;
    }
    return OK;
}

// Basis values / reference gradients at a barycentric point (for the pins).
int oracle_basis(int domain, int order, const double* lam, double* phi /* 10 */, double* grad /* 10 x 3 */) {
    if ((domain != SURFACE_TRI && domain != BULK_TET && domain != SURFACE_LINE) || (order != 1 && order != 2))
        return ERR_UNSUPPORTED;
    double g[10][3];
    basis(domain, order, lam, phi, g);
    for (int a = 0; a < 10; ++a)
        for (int m = 0; m < 3; ++m) grad[3 * a + m] = g[a][m];
    return OK;
}

// Full local matrices of one element.
int oracle_element(int domain, int order, int quad, const double* X, const double* u,
                   int formulation, double* Ml, double* Al, double* Aal) {
    Ref R;
    if (!make_ref(domain, order, quad, R)) return ERR_UNSUPPORTED;
    if (formulation == 1 && domain != SURFACE_TRI) return ERR_UNSUPPORTED;
    return element_matrices(R, X, u, formulation, Ml, Al, Aal);
}

// Assemble the CSR rows `rows` (ascending, unique; n_rows of them) of the
// requested kinds.  coeff may be null unless kinds & K_STIFF_COEF.
int oracle_assemble_rows(int domain, int order, int quad, int64_t n_nodes, const double* coords,
                         int64_t n_elems, const int32_t* conn, const double* coeff, int kinds,
                         int64_t n_rows, const int64_t* rows, int nthreads, oracle_csr* out) {
    std::memset(out, 0, sizeof(*out));
    out->bad_elem = -1;
    Ref R;
    if (!make_ref(domain, order, quad, R)) return ERR_UNSUPPORTED;
    if ((kinds & K_STIFF_COEF) && !coeff) return ERR_INVALID_ARG;
    if (kinds == 0 || (kinds & ~7)) return ERR_INVALID_ARG;
    const int n = R.nref;
    // index check (lowest element id)
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < n; ++a) {
            const int32_t v = conn[e * n + a];
            if (v < 0 || v >= n_nodes) { out->bad_elem = e; return ERR_INDEX; }
        }
    for (int64_t i = 0; i < n_rows; ++i)
        if (rows[i] < 0 || rows[i] >= n_nodes || (i > 0 && rows[i] <= rows[i - 1])) return ERR_INVALID_ARG;
    // node -> incident elements (counting pass), ascending element id
    std::vector<int64_t> inc_ptr(n_nodes + 1, 0);
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < n; ++a) inc_ptr[conn[e * n + a] + 1]++;
    for (int64_t i = 0; i < n_nodes; ++i) inc_ptr[i + 1] += inc_ptr[i];
    std::vector<int64_t> inc(inc_ptr[n_nodes]);
    {
        std::vector<int64_t> cur(inc_ptr.begin(), inc_ptr.end() - 1);
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < n; ++a) inc[cur[conn[e * n + a]]++] = e;
    }
    // row blocks (each owned by one thread; results do not depend on the split)
    if (nthreads < 1) nthreads = 1;
    int64_t BLOCK = (n_rows + 4 * nthreads - 1) / (4 * (int64_t)nthreads);
    if (BLOCK < 1024) BLOCK = 1024;
    if (BLOCK > (1 << 18)) BLOCK = 1 << 18;
    const int64_t nblocks = (n_rows + BLOCK - 1) / BLOCK;
    std::vector<Csr> parts(nblocks);
    std::vector<int64_t> bad(nblocks, -1);
    auto run_block = [&](int64_t b) {
        const int64_t r0 = b * BLOCK, r1 = std::min(n_rows, r0 + BLOCK);
        std::vector<int64_t> elems;
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t k = inc_ptr[rows[i]]; k < inc_ptr[rows[i] + 1]; ++k) elems.push_back(inc[k]);
        std::sort(elems.begin(), elems.end());
        elems.erase(std::unique(elems.begin(), elems.end()), elems.end());
        std::map<std::pair<int32_t, int32_t>, std::array<double, 3>> acc;
        std::vector<double> X(3 * n), U(n), Ml(n * n), Al(n * n), Aal(n * n);
        const int64_t* rb = rows + r0;
        const int64_t* re = rows + r1;
        for (int64_t e : elems) {
            for (int a = 0; a < n; ++a) {
                const int32_t v = conn[e * n + a];
                for (int c = 0; c < 3; ++c) X[3 * a + c] = coords[3 * (int64_t)v + c];
                U[a] = coeff ? coeff[v] : 0.0;
            }
            const int st = element_matrices(R, X.data(), (kinds & K_STIFF_COEF) ? U.data() : nullptr, 0,
                                            Ml.data(), Al.data(), Aal.data());
            if (st != OK) {
                if (bad[b] < 0 || e < bad[b]) bad[b] = e;
                continue;
            }
            for (int a = 0; a < n; ++a) {
                const int32_t row = conn[e * n + a];
                if (!std::binary_search(rb, re, (int64_t)row)) continue;
                for (int bb = 0; bb < n; ++bb) {
                    auto& s = acc[std::make_pair(row, conn[e * n + bb])];
                    s[0] += Ml[a * n + bb];
                    s[1] += Al[a * n + bb];
                    s[2] += Aal[a * n + bb];
                }
            }
        }
        Csr& P = parts[b];
        P.n_rows = r1 - r0;
        P.nnz = (int64_t)acc.size();
        P.row_ptr = (int64_t*)std::calloc(P.n_rows + 1, sizeof(int64_t));
        P.col_idx = (int32_t*)std::malloc(sizeof(int32_t) * std::max<int64_t>(1, P.nnz));
        for (int k = 0; k < 3; ++k)
            P.vals[k] = (kinds & (1 << k)) ? (double*)std::malloc(sizeof(double) * std::max<int64_t>(1, P.nnz)) : nullptr;
        int64_t idx = 0, r = 0;
        for (auto& kv : acc) {
            while (rows[r0 + r] < kv.first.first) { P.row_ptr[r + 1] = idx; ++r; }
            P.col_idx[idx] = kv.first.second;
            for (int k = 0; k < 3; ++k)
                if (P.vals[k]) P.vals[k][idx] = kv.second[k];
            ++idx;
            P.row_ptr[r + 1] = idx;
        }
        for (int64_t rr = r + 1; rr <= P.n_rows; ++rr) P.row_ptr[rr] = idx;
    };
    {
        std::vector<std::thread> pool;
        std::vector<int64_t> next(1, 0);
        const int T = (int)std::min<int64_t>(nthreads, std::max<int64_t>(1, nblocks));
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t]() {
                for (int64_t b = t; b < nblocks; b += T) run_block(b);
            });
        for (auto& th : pool) th.join();
    }
    int64_t worst = -1;
    for (int64_t b = 0; b < nblocks; ++b)
        if (bad[b] >= 0 && (worst < 0 || bad[b] < worst)) worst = bad[b];
    if (worst >= 0) {
        for (auto& P : parts) { std::free(P.row_ptr); std::free(P.col_idx); for (int k = 0; k < 3; ++k) std::free(P.vals[k]); }
        out->bad_elem = worst;
        return ERR_DEGENERATE;
    }
    // concatenate
    int64_t nnz = 0;
    for (auto& P : parts) nnz += P.nnz;
    out->n_rows = n_rows;
    out->nnz = nnz;
    out->row_ptr = (int64_t*)std::malloc(sizeof(int64_t) * (n_rows + 1));
    out->col_idx = (int32_t*)std::malloc(sizeof(int32_t) * std::max<int64_t>(1, nnz));
    for (int k = 0; k < 3; ++k)
        out->vals[k] = (kinds & (1 << k)) ? (double*)std::malloc(sizeof(double) * std::max<int64_t>(1, nnz)) : nullptr;
    out->row_ptr[0] = 0;
    int64_t roff = 0, off = 0;
    for (auto& P : parts) {
        for (int64_t r = 0; r < P.n_rows; ++r) out->row_ptr[roff + r + 1] = off + P.row_ptr[r + 1];
        if (P.nnz) {
            std::memcpy(out->col_idx + off, P.col_idx, sizeof(int32_t) * P.nnz);
            for (int k = 0; k < 3; ++k)
                if (out->vals[k]) std::memcpy(out->vals[k] + off, P.vals[k], sizeof(double) * P.nnz);
        }
        roff += P.n_rows;
        off += P.nnz;
        std::free(P.row_ptr); std::free(P.col_idx);
        for (int k = 0; k < 3; ++k) std::free(P.vals[k]);
    }
    return OK;
}

// Local right-hand side of one element: U is nref x ncomp (row-major), F likewise.
int oracle_element_rhs(int domain, int order, int quad, const double* X, const double* U, int kind,
                       int formulation, double* F) {
    Ref R;
    if (!make_ref(domain, order, quad, R)) return ERR_UNSUPPORTED;
    if (kind != RHS_LOAD && kind != RHS_KLL) return ERR_INVALID_ARG;
    if ((kind == RHS_KLL || formulation == 1) && domain != SURFACE_TRI) return ERR_UNSUPPORTED;
    return element_rhs(R, X, U, kind, formulation, F);
}

// Assemble the right-hand side `kind` into the rows `rows` (ascending,
// unique).  u: ncomp x n_nodes, component-major (u[k * n_nodes + c], the
// paper's index j + (k-1) N); out (and out_abs, if not null): ncomp x
// n_rows, component-major.  out_abs accumulates the absolute-value evaluation of
// every term (element_rhs's Fabs: the scale of the rounding error of any
// evaluation order, reading G33).  Per row: ascending element id.
int oracle_assemble_rhs_rows(int domain, int order, int quad, int64_t n_nodes, const double* coords,
                             int64_t n_elems, const int32_t* conn, const double* u, int kind, int64_t n_rows,
                             const int64_t* rows, int nthreads, double* out, double* out_abs, int64_t* bad_elem) {
    *bad_elem = -1;
    Ref R;
    if (!make_ref(domain, order, quad, R)) return ERR_UNSUPPORTED;
    if (kind != RHS_LOAD && kind != RHS_KLL) return ERR_INVALID_ARG;
    if (kind == RHS_KLL && domain != SURFACE_TRI) return ERR_UNSUPPORTED;
    if (!u || !out) return ERR_INVALID_ARG;
    const int n = R.nref, nc = rhs_ncomp(kind);
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < n; ++a) {
            const int32_t v = conn[e * n + a];
            if (v < 0 || v >= n_nodes) { *bad_elem = e; return ERR_INDEX; }
        }
    for (int64_t i = 0; i < n_rows; ++i)
        if (rows[i] < 0 || rows[i] >= n_nodes || (i > 0 && rows[i] <= rows[i - 1])) return ERR_INVALID_ARG;
    for (int64_t i = 0; i < nc * n_rows; ++i) {
        out[i] = 0.0;
        if (out_abs) out_abs[i] = 0.0;
    }
    std::vector<int64_t> inc_ptr(n_nodes + 1, 0);
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < n; ++a) inc_ptr[conn[e * n + a] + 1]++;
    for (int64_t i = 0; i < n_nodes; ++i) inc_ptr[i + 1] += inc_ptr[i];
    std::vector<int64_t> inc(inc_ptr[n_nodes]);
    {
        std::vector<int64_t> cur(inc_ptr.begin(), inc_ptr.end() - 1);
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < n; ++a) inc[cur[conn[e * n + a]]++] = e;
    }
    if (nthreads < 1) nthreads = 1;
    int64_t BLOCK = (n_rows + 4 * nthreads - 1) / (4 * (int64_t)nthreads);
    if (BLOCK < 1024) BLOCK = 1024;
    if (BLOCK > (1 << 18)) BLOCK = 1 << 18;
    const int64_t nblocks = (n_rows + BLOCK - 1) / BLOCK;
    std::vector<int64_t> bad(nblocks, -1);
    auto run_block = [&](int64_t b) {
        const int64_t r0 = b * BLOCK, r1 = std::min(n_rows, r0 + BLOCK);
        std::vector<int64_t> elems;
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t k = inc_ptr[rows[i]]; k < inc_ptr[rows[i] + 1]; ++k) elems.push_back(inc[k]);
        std::sort(elems.begin(), elems.end());
        elems.erase(std::unique(elems.begin(), elems.end()), elems.end());
        std::vector<double> X(3 * n), U(n * nc), F(n * nc), Fa(n * nc);
        for (int64_t e : elems) {
            for (int a = 0; a < n; ++a) {
                const int32_t v = conn[e * n + a];
                for (int c = 0; c < 3; ++c) X[3 * a + c] = coords[3 * (int64_t)v + c];
                for (int k = 0; k < nc; ++k) U[a * nc + k] = u[k * n_nodes + v];
            }
            if (element_rhs(R, X.data(), U.data(), kind, 0, F.data(), out_abs ? Fa.data() : nullptr) != OK) {
                if (bad[b] < 0 || e < bad[b]) bad[b] = e;
                continue;
            }
            for (int a = 0; a < n; ++a) {
                const int64_t row = conn[e * n + a];
                const int64_t* it = std::lower_bound(rows + r0, rows + r1, row);
                if (it == rows + r1 || *it != row) continue;
                const int64_t i = it - rows;
                for (int k = 0; k < nc; ++k) {
                    out[k * n_rows + i] += F[a * nc + k];
                    if (out_abs) out_abs[k * n_rows + i] += Fa[a * nc + k];
                }
            }
        }
    };
    {
        std::vector<std::thread> pool;
        const int T = (int)std::min<int64_t>(nthreads, std::max<int64_t>(1, nblocks));
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t]() {
                for (int64_t b = t; b < nblocks; b += T) run_block(b);
            });
        for (auto& th : pool) th.join();
    }
    for (int64_t b = 0; b < nblocks; ++b)
        if (bad[b] >= 0 && (*bad_elem < 0 || bad[b] < *bad_elem)) *bad_elem = bad[b];
    return *bad_elem >= 0 ? ERR_DEGENERATE : OK;
}

}  // extern "C"

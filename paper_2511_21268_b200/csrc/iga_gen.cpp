// iga_gen.cpp — tensor-product B-spline Poisson stiffness generator (the problem source).
//
// Paper: P:L69-78 (B-spline basis, open knot vectors, C^{p-1}), P:L551-568 (single-patch Galerkin
// assembly, k_ij = ∫∇φ_j·∇φ_i), Remark P:L570-573 ((p+1)-point Gauss is exact)
// (Dirichlet DOFs eliminated), P:L1061-1072 (cube: Dirichlet on sides 1,2,3).
//
// Route (c.3/c.4): on the unit square/cube J_F = I, so the stiffness is the Kronecker
// sum K = K1⊗M1⊗M1 + M1⊗K1⊗M1 + M1⊗M1⊗K1 of 1-D mass/stiffness tables.  The 1-D tables are
// integrated on the integer-knot vector (h = 1) with (p+1)-point Gauss–Legendre in IEEE binary128
// (__float128: nodes by Newton on P_{p+1}, basis by the Cox–de Boor triangle) and rounded ONCE to
// fp64; the binary128 error (~1e-32 relative) is far below half an fp64 ulp, so the rounded tables are
// the correctly-rounded exact values.  Then M1 = fl(M̂/n), K1 = fl(K̂·n) and every 3-D entry is
// evaluated as ((K·M)·M + (M·K)·M) + (M·M)·K in that order, without FMA (-ffp-contract=off).
#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.hpp"

namespace amgb {
namespace {

using q128 = __float128;

// Gauss–Legendre nodes/weights on [0,1] in binary128.
void gauss_legendre_q(int npts, std::vector<q128> &x, std::vector<q128> &w) {
    x.assign(npts, 0);
    w.assign(npts, 0);
    for (int i = 0; i < npts; i++) {
        q128 z = cosq(M_PIq * (i + 0.75Q) / (npts + 0.5Q));
        q128 dp = 1;
        for (int it = 0; it < 100; it++) {
            q128 p0 = 1, p1 = z;
            for (int k = 2; k <= npts; k++) {
                q128 pk = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
                p0 = p1;
                p1 = pk;
            }
            if (npts == 1) { p0 = 1; p1 = z; }
            dp = npts * (z * p1 - p0) / (z * z - 1);
            q128 dz = p1 / dp;
            z -= dz;
            if (fabsq(dz) < 1e-33Q) break;
        }
        // recompute derivative at the converged node
        q128 p0 = 1, p1 = z;
        for (int k = 2; k <= npts; k++) {
            q128 pk = ((2 * k - 1) * z * p1 - (k - 1) * p0) / k;
            p0 = p1;
            p1 = pk;
        }
        if (npts == 1) { p0 = 1; p1 = z; }
        dp = npts * (z * p1 - p0) / (z * z - 1);
        x[i] = (z + 1) / 2;                    // map [-1,1] -> [0,1]
        w[i] = 1 / ((1 - z * z) * dp * dp);    // 2/((1-z^2)P'^2) halved
    }
}

// Knot t_k of the open integer-knot vector on [0, n] (degree p).
inline int knot(int k, int p, int n) { return std::min(std::max(k - p, 0), n); }

// Non-zero basis functions N_{s-deg..s, deg} at x in span s (The NURBS Book A2.2), binary128.
void basis_funs(int s, q128 x, int deg, int p, int n, q128 *N) {
    q128 left[16], right[16];
    N[0] = 1;
    for (int j = 1; j <= deg; j++) {
        left[j] = x - knot(s + 1 - j, p, n);
        right[j] = knot(s + j, p, n) - x;
        q128 saved = 0;
        for (int r = 0; r < j; r++) {
            q128 tmp = N[r] / (right[r + 1] + left[j - r]);
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
    }
}

// Values and first derivatives of the p+1 functions a = s-p..s at x.
void basis_and_derivs(int s, q128 x, int p, int n, q128 *val, q128 *der) {
    basis_funs(s, x, p, p, n, val);
    q128 low[16];
    if (p == 0) { der[0] = 0; return; }
    basis_funs(s, x, p - 1, p, n, low);  // N_{s-p+1..s, p-1}
    for (int k = 0; k <= p; k++) {
        int a = s - p + k;
        q128 d = 0;
        if (k >= 1) {  // N_{a,p-1} is low[k-1]
            int den = knot(a + p, p, n) - knot(a, p, n);
            if (den) d += p * low[k - 1] / den;
        }
        if (k <= p - 1) {  // N_{a+1,p-1} is low[k]
            int den = knot(a + p + 1, p, n) - knot(a + 1, p, n);
            if (den) d -= p * low[k] / den;
        }
        der[k] = d;
    }
}

struct Tables1D {
    int p = 0, n = 0, m = 0;
    std::vector<double> M, K;  // band (m x (2p+1)), physical (scaled) tables
};

void hat_tables_q(int p, int n, std::vector<q128> &Mq, std::vector<q128> &Kq) {
    const int m = n + p, bw = 2 * p + 1;
    Mq.assign((size_t)m * bw, 0);
    Kq.assign((size_t)m * bw, 0);
    std::vector<q128> gx, gw;
    gauss_legendre_q(p + 1, gx, gw);
    q128 val[16], der[16];
    for (int e = 0; e < n; e++) {
        int s = e + p;
        for (int g = 0; g <= p; g++) {
            basis_and_derivs(s, e + gx[g], p, n, val, der);
            for (int i = 0; i <= p; i++)
                for (int j = 0; j <= p; j++) {
                    int a = e + i, b = e + j;
                    Mq[(size_t)a * bw + (b - a + p)] += gw[g] * val[i] * val[j];
                    Kq[(size_t)a * bw + (b - a + p)] += gw[g] * der[i] * der[j];
                }
        }
    }
}

// Round to fp64; values that are zero up to the binary128 integration error become exactly 0
// (exact non-zero entries are rationals of magnitude >> 1e-25 for p <= 8).
double round_q(q128 v, q128 scale) {
    if (fabsq(v) < 1e-25Q * scale) return 0.0;
    return (double)v;
}

void hat_tables(int p, int n, double *mhat, double *khat) {
    std::vector<q128> Mq, Kq;
    hat_tables_q(p, n, Mq, Kq);
    q128 sm = 0, sk = 0;
    for (auto v : Mq) sm = fmaxq(sm, fabsq(v));
    for (auto v : Kq) sk = fmaxq(sk, fabsq(v));
    for (size_t i = 0; i < Mq.size(); i++) {
        mhat[i] = round_q(Mq[i], sm);
        khat[i] = round_q(Kq[i], sk);
    }
}

Tables1D physical_tables(int p, int n) {
    Tables1D t;
    t.p = p; t.n = n; t.m = n + p;
    const size_t sz = (size_t)t.m * (2 * p + 1);
    std::vector<double> mh(sz), kh(sz);
    hat_tables(p, n, mh.data(), kh.data());
    t.M.resize(sz);
    t.K.resize(sz);
    const double dn = (double)n;
    for (size_t i = 0; i < sz; i++) {
        t.M[i] = mh[i] / dn;  // M1 = fl(M̂/n)
        t.K[i] = kh[i] * dn;  // K1 = fl(K̂·n)
    }
    return t;
}

// 1-D load factors F_ax[a] = ∫_0^1 g_ax(x) N_a(x) dx, g = sin(πx), sin(πy/2), cos(πz) (c.5).
std::vector<double> load_factor(int ax, int p, int n) {
    const int m = n + p;
    std::vector<q128> F(m, 0);
    std::vector<q128> gx, gw;
    gauss_legendre_q(p + 1, gx, gw);
    q128 val[16], der[16];
    for (int e = 0; e < n; e++) {
        for (int g = 0; g <= p; g++) {
            basis_and_derivs(e + p, e + gx[g], p, n, val, der);
            q128 x = (e + gx[g]) / n;
            q128 f = ax == 0 ? sinq(M_PIq * x) : ax == 1 ? sinq(M_PIq * x / 2) : cosq(M_PIq * x);
            for (int i = 0; i <= p; i++) F[e + i] += gw[g] / n * f * val[i];
        }
    }
    std::vector<double> out(m);
    for (int a = 0; a < m; a++) out[a] = (double)F[a];
    return out;
}

// Thick quarter ring (geometry 1): the seven weighted 1-D tables of K = A_u⊗B_v⊗M_w + C_u⊗D_v⊗M_w +
// E_u⊗B_v⊗K_w (amg_b200.h), on [0,1] with n elements, (p+1)-point Gauss per element in binary128,
// rounded once; band storage m × (2p+1).  r(u) = 1+u; |c'(v)| of the rational quadratic quarter circle
// with weights (1, √2/2, 1).
struct RingTables {
    std::vector<double> A, C, E, B, Dv, M, K;
};

q128 circle_speed(q128 v) {
    const q128 w1 = sqrtq(2.0Q) / 2;
    const q128 X = (1 - v) * (1 - v) + 2 * v * (1 - v) * w1;
    const q128 Y = 2 * v * (1 - v) * w1 + v * v;
    const q128 W = (1 - v) * (1 - v) + 2 * v * (1 - v) * w1 + v * v;
    const q128 Xp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v);
    const q128 Yp = 2 * w1 * (1 - 2 * v) + 2 * v;
    const q128 Wp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v) + 2 * v;
    const q128 cx = (Xp * W - X * Wp) / (W * W);
    const q128 cy = (Yp * W - Y * Wp) / (W * W);
    return sqrtq(cx * cx + cy * cy);
}

RingTables ring_tables(int p, int n) {
    const int m = n + p, bw = 2 * p + 1;
    const size_t sz = (size_t)m * bw;
    std::vector<q128> tA(sz, 0), tC(sz, 0), tE(sz, 0), tB(sz, 0), tD(sz, 0), tM(sz, 0), tK(sz, 0);
    std::vector<q128> gx, gw;
    gauss_legendre_q(p + 1, gx, gw);
    q128 val[16], der[16];
    for (int e = 0; e < n; e++)
        for (int q = 0; q <= p; q++) {
            basis_and_derivs(e + p, e + gx[q], p, n, val, der);  // integer-knot basis: d/dt
            const q128 x = (e + gx[q]) / n, w = gw[q] / n;
            const q128 r = 1 + x, sp = circle_speed(x);
            for (int i = 0; i <= p; i++)
                for (int j = 0; j <= p; j++) {
                    const size_t k = (size_t)(e + i) * bw + (j - i + p);
                    const q128 nn = val[i] * val[j] * w;
                    const q128 dd = der[i] * der[j] * n * n * w;  // d/du = n·d/dt
                    tA[k] += dd * r;
                    tC[k] += nn / r;
                    tE[k] += nn * r;
                    tB[k] += nn * sp;
                    tD[k] += dd / sp;
                    tM[k] += nn;
                    tK[k] += dd;
                }
        }
    RingTables T;
    auto rnd = [&](const std::vector<q128> &t) {
        q128 sc = 0;
        for (auto v : t) sc = fmaxq(sc, fabsq(v));
        std::vector<double> o(t.size());
        for (size_t i = 0; i < t.size(); i++) o[i] = round_q(t[i], sc);
        return o;
    };
    T.A = rnd(tA); T.C = rnd(tC); T.E = rnd(tE); T.B = rnd(tB); T.Dv = rnd(tD); T.M = rnd(tM); T.K = rnd(tK);
    return T;
}

// 1-D moments ∫_0^1 g(t) N_a(t) dt of all m functions, (p+1)-point Gauss per element in binary128.
template <class Fn>
std::vector<double> moments(int p, int n, Fn g) {
    const int m = n + p;
    std::vector<q128> F(m, 0);
    std::vector<q128> gx, gw;
    gauss_legendre_q(p + 1, gx, gw);
    q128 val[16], der[16];
    for (int e = 0; e < n; e++)
        for (int q = 0; q <= p; q++) {
            basis_and_derivs(e + p, e + gx[q], p, n, val, der);
            const q128 x = (e + gx[q]) / n;
            const q128 f = g(x);
            for (int i = 0; i <= p; i++) F[e + i] += gw[q] / n * f * val[i];
        }
    std::vector<double> out(m);
    for (int a = 0; a < m; a++) out[a] = (double)F[a];
    return out;
}

// The paper's cube data: f = −e^{x+z} sin y, g_D = e^{x+z} sin y
// on sides 1-3, g_N = e^{x+z} cos y (side 4), −e^{x+z} sin y (5), e^{x+z} sin y (6).  Readings
// (DESIGN.md §3): g_D by ONE L2 projection onto the trace space of the union of the Dirichlet faces
// (face mass M⊗M, DOFs on shared edges get both faces' contributions), solved by Jacobi-preconditioned
// CG to round-off; F_free = (source + Neumann load)_free − (K_full u_D)_free.  All integrals by
// (p+1)-point Gauss per element and direction.
void paper_cube_load(int p, int n, const Tables1D &T, const int *lo, const int *nf, Buf<double> &F) {
    const int m = n + p, bw = 2 * p + 1;
    const double *M1 = T.M.data(), *K1 = T.K.data();
    const std::vector<double> E = moments(p, n, [](q128 x) { return expq(x); });
    const std::vector<double> S = moments(p, n, [](q128 x) { return sinq(x); });
    const int64_t m3 = (int64_t)m * m * m;
    auto id = [m](int a, int b, int c) { return (int64_t)a + (int64_t)m * (b + (int64_t)m * c); };
    auto band = [bw, p](const double *A, int i, int j) { return A[(size_t)i * bw + (j - i + p)]; };
    // --- joint L2 projection of g_D on faces x=0 (a=0), x=1 (a=m−1), y=0 (b=0) -------------------
    // y = M_bnd x on the Dirichlet DOFs (x, y full m³ arrays, zero elsewhere)
    auto onD = [m](int a, int b) { return a == 0 || a == m - 1 || b == 0; };
    auto apply_bnd = [&](const std::vector<double> &x, std::vector<double> &y) {
        std::fill(y.begin(), y.end(), 0.0);
        for (int face = 0; face < 3; face++) {
            // face 0: a=0, 1: a=m−1 (in-face axes b, c); face 2: b=0 (in-face axes a, c)
#pragma omp parallel for schedule(static)
            for (int c = 0; c < m; c++)
                for (int u = 0; u < m; u++) {
                    double acc = 0.0;
                    for (int c2 = std::max(0, c - p); c2 <= std::min(m - 1, c + p); c2++)
                        for (int u2 = std::max(0, u - p); u2 <= std::min(m - 1, u + p); u2++) {
                            const int64_t j = face == 2 ? id(u2, 0, c2) : id(face == 0 ? 0 : m - 1, u2, c2);
                            acc += band(M1, u, u2) * band(M1, c, c2) * x[j];
                        }
                    const int64_t i = face == 2 ? id(u, 0, c) : id(face == 0 ? 0 : m - 1, u, c);
                    y[i] += acc;  // rows of different faces are disjoint except on shared edges
                }
        }
    };
    std::vector<double> rhs(m3, 0.0), diag(m3, 0.0), x(m3, 0.0), r(m3), z(m3), pp(m3, 0.0), q(m3);
    for (int c = 0; c < m; c++)
        for (int u = 0; u < m; u++) {
            rhs[id(0, u, c)] += S[u] * E[c];              // x = 0: e^z sin y
            rhs[id(m - 1, u, c)] += M_E * S[u] * E[c];    // x = 1: e·e^z sin y
            // y = 0: g_D = 0
            const double mm = band(M1, u, u) * band(M1, c, c);
            diag[id(0, u, c)] += mm;
            diag[id(m - 1, u, c)] += mm;
            diag[id(u, 0, c)] += mm;
        }
    double rr = 0.0, bb = 0.0;
    for (int64_t i = 0; i < m3; i++) {
        r[i] = rhs[i];
        z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
        pp[i] = z[i];
        rr += r[i] * z[i];
        bb += rhs[i] * rhs[i];
    }
    for (int it = 0; it < 100000 && bb > 0.0; it++) {
        apply_bnd(pp, q);
        double pq = 0.0;
        for (int64_t i = 0; i < m3; i++) pq += pp[i] * q[i];
        if (!(pq > 0.0)) break;
        const double alpha = rr / pq;
        double rn = 0.0, rz = 0.0;
        for (int64_t i = 0; i < m3; i++) {
            x[i] += alpha * pp[i];
            r[i] -= alpha * q[i];
            rn += r[i] * r[i];
            z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
            rz += r[i] * z[i];
        }
        if (rn <= 1e-30 * bb) break;
        const double beta = rz / rr;
        for (int64_t i = 0; i < m3; i++) pp[i] = z[i] + beta * pp[i];
        rr = rz;
    }
    for (int a = 0; a < m; a++)
        for (int b = 0; b < m; b++)
            if (!onD(a, b))
                for (int c = 0; c < m; c++) x[id(a, b, c)] = 0.0;
    // --- lifting L = K_full u_D, K_full = K⊗M⊗M + M⊗K⊗M + M⊗M⊗K, evaluated on the free DOFs ----------
    const int64_t N = (int64_t)nf[0] * nf[1] * nf[2];
    F.alloc(N);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N; row++) {
        const int a = lo[0] + (int)(row % nf[0]);
        const int b = lo[1] + (int)((row / nf[0]) % nf[1]);
        const int c = lo[2] + (int)(row / ((int64_t)nf[0] * nf[1]));
        double lift = 0.0;
        for (int c2 = std::max(0, c - p); c2 <= std::min(m - 1, c + p); c2++)
            for (int b2 = std::max(0, b - p); b2 <= std::min(m - 1, b + p); b2++)
                for (int a2 = std::max(0, a - p); a2 <= std::min(m - 1, a + p); a2++) {
                    const double u = x[id(a2, b2, c2)];
                    if (u == 0.0) continue;
                    const double Ma = band(M1, a, a2), Ka = band(K1, a, a2);
                    const double Mb = band(M1, b, b2), Kb = band(K1, b, b2);
                    const double Mc = band(M1, c, c2), Kc = band(K1, c, c2);
                    lift += (Ka * Mb * Mc + Ma * Kb * Mc + Ma * Mb * Kc) * u;
                }
        double f = -E[a] * S[b] * E[c];
        if (b == m - 1) f += std::cos(1.0) * E[a] * E[c];
        if (c == 0) f += -E[a] * S[b];
        if (c == m - 1) f += M_E * E[a] * S[b];
        F[row] = f - lift;
    }
}

// The paper's ring data (eq:Lshapedcoeff P:L1079-1089): u = e^x sin(xy) cos z.  Source by
// (p+1)³-point Gauss per element through the map (f·det J), Neumann on side 4 (v = 1, the x = 0 plane,
// dS = du dw) and sides 5/6 (w = 0/1, dS = r|c'| du dv), g_D = u on sides 1 (u = 0, dS = |c'| dv dw),
// 2 (u = 1, 2|c'| dv dw), 3 (v = 0, du dw) by one joint L2 projection (reading N1.a; Jacobi-CG),
// F_free = (source + Neumann)_free − (K_full u_D)_free with the full ring operator.  fp64 quadrature.
void paper_ring_load(int p, int n, const RingTables &RT, const int *lo, const int *nf, Buf<double> &F) {
    const int m = n + p, bw = 2 * p + 1;
    auto id = [m](int a, int b, int c) { return (int64_t)a + (int64_t)m * (b + (int64_t)m * c); };
    auto band = [bw, p](const std::vector<double> &A, int i, int j) { return A[(size_t)i * bw + (j - i + p)]; };
    // quadrature points / weights and basis values per element (fp64)
    std::vector<q128> gxq, gwq;
    gauss_legendre_q(p + 1, gxq, gwq);
    const int nq = p + 1;
    std::vector<double> t((size_t)n * nq), wt((size_t)n * nq), Bv((size_t)n * nq * nq);  // B[e][q][i]
    for (int e = 0; e < n; e++)
        for (int q = 0; q < nq; q++) {
            q128 val[16], der[16];
            basis_and_derivs(e + p, e + gxq[q], p, n, val, der);
            t[e * nq + q] = (double)((e + gxq[q]) / n);
            wt[e * nq + q] = (double)(gwq[q] / n);
            for (int i = 0; i <= p; i++) Bv[((size_t)e * nq + q) * nq + i] = (double)val[i];
        }
    auto geom = [](double u, double v, double &x, double &y, double &r, double &sp) {
        const double w1 = std::sqrt(2.0) / 2.0;
        const double X = (1 - v) * (1 - v) + 2 * v * (1 - v) * w1, Y = 2 * v * (1 - v) * w1 + v * v;
        const double W = (1 - v) * (1 - v) + 2 * v * (1 - v) * w1 + v * v;
        const double Xp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v), Yp = 2 * w1 * (1 - 2 * v) + 2 * v;
        const double Wp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v) + 2 * v;
        const double dcx = (Xp * W - X * Wp) / (W * W), dcy = (Yp * W - Y * Wp) / (W * W);
        r = 1 + u;
        x = r * X / W;
        y = r * Y / W;
        sp = std::sqrt(dcx * dcx + dcy * dcy);
    };
    auto uex = [](double x, double y, double z) { return std::exp(x) * std::sin(x * y) * std::cos(z); };
    const int64_t m3 = (int64_t)m * m * m;
    std::vector<double> Fall(m3, 0.0);
    // --- source: element loop (parallel over z-elements: disjoint c ranges per element row are not
    //     disjoint across neighbouring elements, so accumulate per element into a private buffer)
#pragma omp parallel
    {
        std::vector<double> loc(m3, 0.0);
#pragma omp for schedule(static)
        for (int ez = 0; ez < n; ez++)
            for (int ey = 0; ey < n; ey++)
                for (int ex = 0; ex < n; ex++)
                    for (int qz = 0; qz < nq; qz++)
                        for (int qy = 0; qy < nq; qy++)
                            for (int qx = 0; qx < nq; qx++) {
                                const double u = t[ex * nq + qx], v = t[ey * nq + qy], z = t[ez * nq + qz];
                                double x, y, r, sp;
                                geom(u, v, x, y, r, sp);
                                const double f = std::exp(x) * std::cos(z) *
                                                 (-2.0 * std::cos(x * y) * y + std::sin(x * y) * (y * y + x * x));
                                const double wq = f * r * sp * wt[ex * nq + qx] * wt[ey * nq + qy] * wt[ez * nq + qz];
                                const double *Ba = &Bv[((size_t)ex * nq + qx) * nq];
                                const double *Bb = &Bv[((size_t)ey * nq + qy) * nq];
                                const double *Bc = &Bv[((size_t)ez * nq + qz) * nq];
                                for (int k = 0; k <= p; k++)
                                    for (int j = 0; j <= p; j++)
                                        for (int i = 0; i <= p; i++)
                                            loc[id(ex + i, ey + j, ez + k)] += wq * Ba[i] * Bb[j] * Bc[k];
                            }
#pragma omp critical
        for (int64_t i = 0; i < m3; i++) Fall[i] += loc[i];
    }
    // --- Neumann faces
    for (int e0 = 0; e0 < n; e0++)
        for (int e1 = 0; e1 < n; e1++)
            for (int q0 = 0; q0 < nq; q0++)
                for (int q1 = 0; q1 < nq; q1++) {
                    const double s0 = t[e0 * nq + q0], s1 = t[e1 * nq + q1];
                    const double w01 = wt[e0 * nq + q0] * wt[e1 * nq + q1];
                    const double *B0 = &Bv[((size_t)e0 * nq + q0) * nq], *B1 = &Bv[((size_t)e1 * nq + q1) * nq];
                    double x, y, r, sp;
                    // side 4: v = 1, in-face (u = s0, w = s1), dS = du dw
                    geom(s0, 1.0, x, y, r, sp);
                    const double g4 = -std::exp(x) * std::cos(s1) * (std::sin(x * y) + y * std::cos(x * y)) * w01;
                    for (int i = 0; i <= p; i++)
                        for (int k = 0; k <= p; k++) Fall[id(e0 + i, m - 1, e1 + k)] += g4 * B0[i] * B1[k];
                    // sides 5 / 6: w = 0 / 1, in-face (u = s0, v = s1), dS = r|c'| du dv
                    geom(s0, s1, x, y, r, sp);
                    const double g5 = std::exp(x) * std::sin(x * y) * std::sin(0.0) * r * sp * w01;
                    const double g6 = -std::exp(x) * std::sin(x * y) * std::sin(1.0) * r * sp * w01;
                    for (int i = 0; i <= p; i++)
                        for (int j = 0; j <= p; j++) {
                            Fall[id(e0 + i, e1 + j, 0)] += g5 * B0[i] * B1[j];
                            Fall[id(e0 + i, e1 + j, m - 1)] += g6 * B0[i] * B1[j];
                        }
                }
    // --- Dirichlet projection: face 0 (u=0, in-face v,w, mass B_v⊗M_w), face 1 (u=1, 2·B_v⊗M_w),
    //     face 2 (v=0, in-face u,w, mass M_u⊗M_w)
    std::vector<double> rhs(m3, 0.0), diag(m3, 0.0), xs(m3, 0.0), r(m3), z(m3), pp(m3, 0.0), q(m3);
    for (int e0 = 0; e0 < n; e0++)
        for (int e1 = 0; e1 < n; e1++)
            for (int q0 = 0; q0 < nq; q0++)
                for (int q1 = 0; q1 < nq; q1++) {
                    const double s0 = t[e0 * nq + q0], s1 = t[e1 * nq + q1];
                    const double w01 = wt[e0 * nq + q0] * wt[e1 * nq + q1];
                    const double *B0 = &Bv[((size_t)e0 * nq + q0) * nq], *B1 = &Bv[((size_t)e1 * nq + q1) * nq];
                    double x, y, rr, sp;
                    geom(0.0, s0, x, y, rr, sp);
                    const double g0 = uex(x, y, s1) * sp * w01;  // u = 0: r = 1
                    geom(1.0, s0, x, y, rr, sp);
                    const double g1 = uex(x, y, s1) * 2.0 * sp * w01;  // u = 1: r = 2
                    geom(s0, 0.0, x, y, rr, sp);
                    const double g2 = uex(x, y, s1) * w01;  // v = 0: (u = s0, w = s1)
                    for (int i = 0; i <= p; i++)
                        for (int k = 0; k <= p; k++) {
                            rhs[id(0, e0 + i, e1 + k)] += g0 * B0[i] * B1[k];
                            rhs[id(m - 1, e0 + i, e1 + k)] += g1 * B0[i] * B1[k];
                            rhs[id(e0 + i, 0, e1 + k)] += g2 * B0[i] * B1[k];
                        }
                }
    auto apply_bnd = [&](const std::vector<double> &xv, std::vector<double> &yv) {
        std::fill(yv.begin(), yv.end(), 0.0);
        for (int face = 0; face < 3; face++) {
            const double sc = face == 1 ? 2.0 : 1.0;
            const std::vector<double> &M0 = face == 2 ? RT.M : RT.B;
#pragma omp parallel for schedule(static)
            for (int c = 0; c < m; c++)
                for (int u = 0; u < m; u++) {
                    double acc = 0.0;
                    for (int c2 = std::max(0, c - p); c2 <= std::min(m - 1, c + p); c2++)
                        for (int u2 = std::max(0, u - p); u2 <= std::min(m - 1, u + p); u2++) {
                            const int64_t j = face == 2 ? id(u2, 0, c2) : id(face == 0 ? 0 : m - 1, u2, c2);
                            acc += sc * band(M0, u, u2) * band(RT.M, c, c2) * xv[j];
                        }
                    const int64_t i = face == 2 ? id(u, 0, c) : id(face == 0 ? 0 : m - 1, u, c);
                    yv[i] += acc;
                }
        }
    };
    for (int c = 0; c < m; c++)
        for (int u = 0; u < m; u++) {
            diag[id(0, u, c)] += band(RT.B, u, u) * band(RT.M, c, c);
            diag[id(m - 1, u, c)] += 2.0 * band(RT.B, u, u) * band(RT.M, c, c);
            diag[id(u, 0, c)] += band(RT.M, u, u) * band(RT.M, c, c);
        }
    double rz = 0.0, bb = 0.0;
    for (int64_t i = 0; i < m3; i++) {
        r[i] = rhs[i];
        z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
        pp[i] = z[i];
        rz += r[i] * z[i];
        bb += rhs[i] * rhs[i];
    }
    for (int it = 0; it < 100000 && bb > 0.0; it++) {
        apply_bnd(pp, q);
        double pq = 0.0;
        for (int64_t i = 0; i < m3; i++) pq += pp[i] * q[i];
        if (!(pq > 0.0)) break;
        const double alpha = rz / pq;
        double rn = 0.0, rzn = 0.0;
        for (int64_t i = 0; i < m3; i++) {
            xs[i] += alpha * pp[i];
            r[i] -= alpha * q[i];
            rn += r[i] * r[i];
            z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
            rzn += r[i] * z[i];
        }
        if (rn <= 1e-30 * bb) break;
        const double beta = rzn / rz;
        for (int64_t i = 0; i < m3; i++) pp[i] = z[i] + beta * pp[i];
        rz = rzn;
    }
    // --- lifting with the full ring operator and the free-DOF load
    const int64_t N = (int64_t)nf[0] * nf[1] * nf[2];
    F.alloc(N);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N; row++) {
        const int a = lo[0] + (int)(row % nf[0]);
        const int b = lo[1] + (int)((row / nf[0]) % nf[1]);
        const int c = lo[2] + (int)(row / ((int64_t)nf[0] * nf[1]));
        double lift = 0.0;
        for (int c2 = std::max(0, c - p); c2 <= std::min(m - 1, c + p); c2++)
            for (int b2 = std::max(0, b - p); b2 <= std::min(m - 1, b + p); b2++)
                for (int a2 = std::max(0, a - p); a2 <= std::min(m - 1, a + p); a2++) {
                    const double u = xs[id(a2, b2, c2)];
                    if (u == 0.0) continue;
                    const double t1 = band(RT.A, a, a2) * band(RT.B, b, b2) * band(RT.M, c, c2);
                    const double t2 = band(RT.C, a, a2) * band(RT.Dv, b, b2) * band(RT.M, c, c2);
                    const double t3 = band(RT.E, a, a2) * band(RT.B, b, b2) * band(RT.K, c, c2);
                    lift += (t1 + t2 + t3) * u;
                }
        F[row] = Fall[id(a, b, c)] - lift;
    }
}

// Three-patch thick L-shape (geometry 2; PAPER.md P:L575-583 gluing, P:L1074-1089 the benchmark;
// readings N4.a/N4.b of DESIGN.md §3).  Patches A = [0,1]³, B = [1,2]×[0,1]², C = [0,1]×[1,2]×[0,1],
// each the unit-cube B-spline space of degree p on n³ elements (identity Jacobian).  Control lattice
// {0 ≤ x, y ≤ 2m−2, 0 ≤ z ≤ m−1} minus {x ≥ m and y ≥ m}; patch lattice offsets (0,0), (m−1,0),
// (0,m−1); the re-entrant edge x = y = m−1 belongs to all three.  Dirichlet faces: x = 0, y = 0,
// x = 2m−2 (B), y = 2m−2 (C), z = 0, z = m−1.  Free DOFs lexicographic, x fastest.  An entry is the
// sum over the patches holding both functions, in patch order A, B, C, of the cube entry
// ((K·M)·M + (M·K)·M) + (M·M)·K in local indices — structurally present when some patch holds both.
// rhs = 0: F = ∫ φ_i (source f = 1, homogeneous data); rhs = 1: F = 0.
void lshape_assemble(const amg_iga_desc &d, HCsr &K, Buf<double> &F) {
    const int p = d.degree, n = d.n_elem, m = n + p, bw = 2 * p + 1, Mx = 2 * m - 1;
    const Tables1D T = physical_tables(p, n);
    const double *M1 = T.M.data(), *K1 = T.K.data();
    auto inside = [&](int x, int y) { return !(x >= m && y >= m); };
    auto dirichlet = [&](int x, int y, int z) {
        return x == 0 || y == 0 || (x == Mx - 1 && y <= m - 1) || (y == Mx - 1 && x <= m - 1) || z == 0 || z == m - 1;
    };
    const int ox[3] = {0, m - 1, 0}, oy[3] = {0, 0, m - 1};
    auto holds = [&](int P, int x, int y) { return x >= ox[P] && x <= ox[P] + m - 1 && y >= oy[P] && y <= oy[P] + m - 1; };
    const size_t lat = (size_t)Mx * Mx * m;
    std::vector<int64_t> idx(lat, -1);
    std::vector<int32_t> px, py, pz;
    int64_t N = 0;
    for (int z = 0; z < m; z++)
        for (int y = 0; y < Mx; y++)
            for (int x = 0; x < Mx; x++)
                if (inside(x, y) && !dirichlet(x, y, z)) {
                    idx[((size_t)z * Mx + y) * Mx + x] = N++;
                    px.push_back(x); py.push_back(y); pz.push_back(z);
                }
    if (N > INT32_MAX) throw Error{AMG_EINVAL, "more than 2^31-1 free DOFs (int32 columns)"};
    auto tab = [&](const double *t, int a, int a2) { return t[(size_t)a * bw + (a2 - a + p)]; };
    // K_all entry of lattice points (x, y, z), (x2, y2, z2): Σ over the patches holding both, in patch
    // order, of the cube entry ((K·M)·M + (M·K)·M) + (M·M)·K; *any = some patch holds both
    auto pair_value = [&](int x, int y, int z, int x2, int y2, int z2, bool *any) {
        double val = 0.0;
        *any = false;
        for (int P = 0; P < 3; P++) {
            if (!holds(P, x, y) || !holds(P, x2, y2)) continue;
            const int a = x - ox[P], a2 = x2 - ox[P], b = y - oy[P], b2 = y2 - oy[P];
            const double t1 = (tab(K1, a, a2) * tab(M1, b, b2)) * tab(M1, z, z2);
            const double t2 = (tab(M1, a, a2) * tab(K1, b, b2)) * tab(M1, z, z2);
            const double t3 = (tab(M1, a, a2) * tab(M1, b, b2)) * tab(K1, z, z2);
            val += (t1 + t2) + t3;
            *any = true;
        }
        return val;
    };
    // visit the columns of row r in ascending order; emit(col, value)
    auto row_visit = [&](int64_t r, auto &&emit) {
        const int x = px[r], y = py[r], z = pz[r];
        for (int z2 = std::max(z - p, 0); z2 <= std::min(z + p, m - 1); z2++)
            for (int y2 = std::max(y - p, 0); y2 <= std::min(y + p, Mx - 1); y2++)
                for (int x2 = std::max(x - p, 0); x2 <= std::min(x + p, Mx - 1); x2++) {
                    const int64_t col = idx[((size_t)z2 * Mx + y2) * Mx + x2];
                    if (col < 0) continue;
                    bool any;
                    const double val = pair_value(x, y, z, x2, y2, z2, &any);
                    if (any) emit(col, val);
                }
    };
    K.nrows = K.ncols = N;
    K.rp.alloc(N + 1);
    K.rp[0] = 0;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < N; r++) {
        int64_t cnt = 0;
        row_visit(r, [&](int64_t, double) { cnt++; });
        K.rp[r + 1] = cnt;
    }
    for (int64_t r = 0; r < N; r++) K.rp[r + 1] += K.rp[r];
    K.ci.alloc(K.rp[N]);
    K.v.alloc(K.rp[N]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < N; r++) {
        int64_t k = K.rp[r];
        row_visit(r, [&](int64_t col, double v) { K.ci[k] = (int32_t)col; K.v[k] = v; k++; });
    }
    F.alloc(N);
    if (d.rhs == 1) {
        std::memset(F.data(), 0, sizeof(double) * N);
        return;
    }
    if (d.rhs == 2) {
        // The paper's L-shape data (reading N4.b): u = e^x sin(xy) cos z,
        // f = cos z · e^x [−2y cos(xy) + (x²+y²) sin(xy)], g_N = ∂u/∂y on y=1 (B), ∂u/∂x on x=1 (C),
        // g_D = u by one joint L2 projection onto the glued Dirichlet faces (Jacobi-CG to round-off),
        // F_free = (source + Neumann)_free − (K_all u_D)_free.  fp64 (p+1)-point Gauss per element.
        const int nq = n * (p + 1);
        std::vector<q128> gx, gw;
        gauss_legendre_q(p + 1, gx, gw);
        std::vector<double> qx(nq), qw(nq), qv((size_t)nq * (p + 1));
        std::vector<int> qe(nq);
        {
            q128 val[16], der[16];
            for (int e = 0; e < n; e++)
                for (int q = 0; q <= p; q++) {
                    const int k = e * (p + 1) + q;
                    basis_and_derivs(e + p, e + gx[q], p, n, val, der);
                    qx[k] = (double)((e + gx[q]) / n);
                    qw[k] = (double)(gw[q] / n);
                    qe[k] = e;
                    for (int i = 0; i <= p; i++) qv[(size_t)k * (p + 1) + i] = (double)val[i];
                }
        }
        const size_t lat = (size_t)Mx * Mx * m;
        auto L = [&](int x, int y, int z) { return ((size_t)z * Mx + y) * Mx + x; };
        // 2-D moments G[u][v] = ∫∫ g(s, t) N_u(s) N_v(t) over the unit square
        auto moments2 = [&](auto &&g) {
            std::vector<double> G((size_t)m * m, 0.0);
            for (int i = 0; i < nq; i++)
                for (int j = 0; j < nq; j++) {
                    const double gv = g(qx[i], qx[j]) * qw[i] * qw[j];
                    for (int a = 0; a <= p; a++)
                        for (int b = 0; b <= p; b++)
                            G[(size_t)(qe[i] + a) * m + qe[j] + b] += gv * qv[(size_t)i * (p + 1) + a] * qv[(size_t)j * (p + 1) + b];
                }
            return G;
        };
        std::vector<double> Cz(m, 0.0);
        for (int i = 0; i < nq; i++)
            for (int a = 0; a <= p; a++) Cz[qe[i] + a] += std::cos(qx[i]) * qw[i] * qv[(size_t)i * (p + 1) + a];
        auto uex = [](double x, double y, double z) { return std::exp(x) * std::sin(x * y) * std::cos(z); };
        std::vector<double> Fall(lat, 0.0);
        for (int P = 0; P < 3; P++) {  // source: G_P(a, b) · Cz(c)
            const double sx = P == 1 ? 1.0 : 0.0, sy = P == 2 ? 1.0 : 0.0;
            const std::vector<double> G = moments2([&](double s, double t) {
                const double x = sx + s, y = sy + t;
                return std::exp(x) * (-2.0 * y * std::cos(x * y) + (x * x + y * y) * std::sin(x * y));
            });
            for (int c = 0; c < m; c++)
                for (int b = 0; b < m; b++)
                    for (int a = 0; a < m; a++) Fall[L(a + ox[P], b + oy[P], c)] += G[(size_t)a * m + b] * Cz[c];
        }
        {  // Neumann: B's face y=1 (local b = m−1; in-face x, z), C's face x=1 (local a = m−1; in-face y, z)
            const std::vector<double> GB = moments2([&](double s, double t) {
                const double x = 1.0 + s;
                return x * std::exp(x) * std::cos(x) * std::cos(t);
            });
            const std::vector<double> GC = moments2([&](double s, double t) {
                const double y = 1.0 + s;
                return std::cos(t) * M_E * (std::sin(y) + y * std::cos(y));
            });
            for (int c = 0; c < m; c++)
                for (int u = 0; u < m; u++) {
                    Fall[L(u + ox[1], m - 1, c)] += GB[(size_t)u * m + c];
                    Fall[L(m - 1, u + oy[2], c)] += GC[(size_t)u * m + c];
                }
        }
        // Dirichlet patch faces: (patch, fixed axis, end); in-face axes ascending
        struct Face { int P, ax, end; };
        const Face dfaces[12] = {{0, 0, 0}, {0, 1, 0}, {0, 2, 0}, {0, 2, 1}, {1, 0, 1}, {1, 1, 0},
                                 {1, 2, 0}, {1, 2, 1}, {2, 0, 0}, {2, 1, 1}, {2, 2, 0}, {2, 2, 1}};
        auto face_lat = [&](const Face &f, int u, int v) {  // lattice index of face-local (u, v)
            int loc[3];
            const int fa0 = f.ax == 0 ? 1 : 0, fa1 = f.ax == 2 ? 1 : 2;
            loc[f.ax] = f.end ? m - 1 : 0;
            loc[fa0] = u;
            loc[fa1] = v;
            return L(loc[0] + ox[f.P], loc[1] + oy[f.P], loc[2]);
        };
        std::vector<double> rhs(lat, 0.0), diag(lat, 0.0);
        for (const Face &f : dfaces) {
            const int fa0 = f.ax == 0 ? 1 : 0, fa1 = f.ax == 2 ? 1 : 2;
            const double off[3] = {f.P == 1 ? 1.0 : 0.0, f.P == 2 ? 1.0 : 0.0, 0.0};
            const std::vector<double> G = moments2([&](double s, double t) {
                double X[3];
                X[f.ax] = f.end ? 1.0 : 0.0;
                X[fa0] = s;
                X[fa1] = t;
                return uex(X[0] + off[0], X[1] + off[1], X[2] + off[2]);
            });
            for (int u = 0; u < m; u++)
                for (int v = 0; v < m; v++) {
                    rhs[face_lat(f, u, v)] += G[(size_t)u * m + v];
                    diag[face_lat(f, u, v)] += tab(M1, u, u) * tab(M1, v, v);
                }
        }
        auto apply_bnd = [&](const std::vector<double> &x, std::vector<double> &y) {
            std::fill(y.begin(), y.end(), 0.0);
            for (const Face &f : dfaces) {  // serial: ≈ 12·m²·(2p+1)² flops, cheaper than 12 fork/joins
                for (int u = 0; u < m; u++)
                    for (int v = 0; v < m; v++) {
                        double acc = 0.0;
                        for (int u2 = std::max(0, u - p); u2 <= std::min(m - 1, u + p); u2++)
                            for (int v2 = std::max(0, v - p); v2 <= std::min(m - 1, v + p); v2++)
                                acc += tab(M1, u, u2) * tab(M1, v, v2) * x[face_lat(f, u2, v2)];
                        y[face_lat(f, u, v)] += acc;  // one face's rows are distinct
                    }
            }
        };
        std::vector<double> xs(lat, 0.0), r(lat), z(lat), pp(lat), q(lat);
        double rr = 0.0, bb = 0.0;
        for (size_t i = 0; i < lat; i++) {
            r[i] = rhs[i];
            z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
            pp[i] = z[i];
            rr += r[i] * z[i];
            bb += rhs[i] * rhs[i];
        }
        for (int it = 0; it < 100000 && bb > 0.0; it++) {
            apply_bnd(pp, q);
            double pq = 0.0;
            for (size_t i = 0; i < lat; i++) pq += pp[i] * q[i];
            if (!(pq > 0.0)) break;
            const double alpha = rr / pq;
            double rn = 0.0, rz = 0.0;
            for (size_t i = 0; i < lat; i++) {
                xs[i] += alpha * pp[i];
                r[i] -= alpha * q[i];
                rn += r[i] * r[i];
                z[i] = diag[i] > 0.0 ? r[i] / diag[i] : 0.0;
                rz += r[i] * z[i];
            }
            if (rn <= 1e-30 * bb) break;
            const double beta = rz / rr;
            for (size_t i = 0; i < lat; i++) pp[i] = z[i] + beta * pp[i];
            rr = rz;
        }
        // lifting: F_free[r] = Fall[r] − Σ_j K_all(r, j) u_D[j] over the Dirichlet lattice points j
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t row = 0; row < N; row++) {
            const int x = px[row], y = py[row], z0 = pz[row];
            double lift = 0.0;
            for (int z2 = std::max(z0 - p, 0); z2 <= std::min(z0 + p, m - 1); z2++)
                for (int y2 = std::max(y - p, 0); y2 <= std::min(y + p, Mx - 1); y2++)
                    for (int x2 = std::max(x - p, 0); x2 <= std::min(x + p, Mx - 1); x2++) {
                        if (!inside(x2, y2) || !dirichlet(x2, y2, z2)) continue;
                        const double u = xs[L(x2, y2, z2)];
                        if (u == 0.0) continue;
                        bool any;
                        lift += pair_value(x, y, z0, x2, y2, z2, &any) * u;
                    }
            F[row] = Fall[L(x, y, z0)] - lift;
        }
        return;
    }
    // ∫ N_a over [0,1] = Σ_b M1[a, b] (partition of unity), summed in ascending b
    std::vector<double> w1(m, 0.0);
    for (int a = 0; a < m; a++)
        for (int b = std::max(a - p, 0); b <= std::min(a + p, m - 1); b++) w1[a] += tab(M1, a, b);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < N; r++) {
        double v = 0.0;
        for (int P = 0; P < 3; P++)
            if (holds(P, px[r], py[r])) v += (w1[px[r] - ox[P]] * w1[py[r] - oy[P]]) * w1[pz[r]];
        F[r] = v;
    }
}

}  // namespace

void iga_tables_hat(int p, int n, double *mhat, double *khat) { hat_tables(p, n, mhat, khat); }

void iga_assemble(const amg_iga_desc &d, HCsr &K, Buf<double> &F) {
    if (d.geometry == 2) {
        lshape_assemble(d, K, F);
        return;
    }
    const int dim = d.dim, p = d.degree, n = d.n_elem, m = n + p, bw = 2 * p + 1;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, nf[3] = {1, 1, 1};
    for (int ax = 0; ax < dim; ax++) {
        lo[ax] = (d.dirichlet_sides >> (2 * ax)) & 1u ? 1 : 0;
        hi[ax] = m - 1 - ((d.dirichlet_sides >> (2 * ax + 1)) & 1u ? 1 : 0);
        nf[ax] = hi[ax] - lo[ax] + 1;
        if (nf[ax] < 1) throw Error{AMG_EINVAL, "no free DOFs along an axis"};
    }
    const int64_t N = (int64_t)nf[0] * nf[1] * nf[2];
    if (N > INT32_MAX) throw Error{AMG_EINVAL, "more than 2^31-1 free DOFs (int32 columns)"};
    const Tables1D T = physical_tables(p, n);
    const double *M1 = T.M.data(), *K1 = T.K.data();
    const bool ring = d.geometry == 1;
    const RingTables RT = ring ? ring_tables(p, n) : RingTables{};

    // per-axis column window [l, h] of function x
    auto win = [&](int ax, int x, int &l, int &h) {
        l = std::max(x - p, lo[ax]);
        h = std::min(x + p, hi[ax]);
    };
    K.nrows = K.ncols = N;
    K.rp.alloc(N + 1);
    K.rp[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N; row++) {
        int a = lo[0] + (int)(row % nf[0]);
        int b = lo[1] + (int)((row / nf[0]) % nf[1]);
        int c = lo[2] + (int)(row / ((int64_t)nf[0] * nf[1]));
        int l, h;
        int64_t cnt = 1;
        win(0, a, l, h); cnt *= h - l + 1;
        win(1, b, l, h); cnt *= h - l + 1;
        if (dim == 3) { win(2, c, l, h); cnt *= h - l + 1; }
        K.rp[row + 1] = cnt;
    }
    for (int64_t r = 0; r < N; r++) K.rp[r + 1] += K.rp[r];
    const int64_t nnz = K.rp[N];
    K.ci.alloc(nnz);
    K.v.alloc(nnz);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N; row++) {
        const int a = lo[0] + (int)(row % nf[0]);
        const int b = lo[1] + (int)((row / nf[0]) % nf[1]);
        const int c = lo[2] + (int)(row / ((int64_t)nf[0] * nf[1]));
        int al, ah, bl, bh, cl = c, ch = c;
        win(0, a, al, ah);
        win(1, b, bl, bh);
        if (dim == 3) win(2, c, cl, ch);
        int64_t k = K.rp[row];
        for (int c2 = cl; c2 <= ch; c2++) {
            const double Mc = dim == 3 ? M1[(size_t)c * bw + (c2 - c + p)] : 1.0;
            const double Kc = dim == 3 ? K1[(size_t)c * bw + (c2 - c + p)] : 0.0;
            for (int b2 = bl; b2 <= bh; b2++) {
                const double Mb = M1[(size_t)b * bw + (b2 - b + p)];
                const double Kb = K1[(size_t)b * bw + (b2 - b + p)];
                const int64_t base = (int64_t)nf[0] * ((b2 - lo[1]) + (int64_t)nf[1] * (c2 - lo[2])) - lo[0];
                for (int a2 = al; a2 <= ah; a2++) {
                    const double Ma = M1[(size_t)a * bw + (a2 - a + p)];
                    const double Ka = K1[(size_t)a * bw + (a2 - a + p)];
                    double val;
                    if (ring) {  // ((A·B)·M + (C·D)·M) + (E·B)·K
                        const size_t ka = (size_t)a * bw + (a2 - a + p), kb = (size_t)b * bw + (b2 - b + p),
                                     kc = (size_t)c * bw + (c2 - c + p);
                        const double t1 = (RT.A[ka] * RT.B[kb]) * RT.M[kc];
                        const double t2 = (RT.C[ka] * RT.Dv[kb]) * RT.M[kc];
                        const double t3 = (RT.E[ka] * RT.B[kb]) * RT.K[kc];
                        val = (t1 + t2) + t3;
                    } else if (dim == 3) {
                        const double t1 = (Ka * Mb) * Mc;
                        const double t2 = (Ma * Kb) * Mc;
                        const double t3 = (Ma * Mb) * Kc;
                        val = (t1 + t2) + t3;
                    } else {
                        const double t1 = Ka * Mb;
                        const double t2 = Ma * Kb;
                        val = t1 + t2;
                    }
                    K.ci[k] = (int32_t)(base + a2);
                    K.v[k] = val;
                    k++;
                }
            }
        }
    }
    // load vector (c.5), or the paper's own data (rhs = 2): cube or quarter ring
    if (d.rhs == 2 && ring) {
        paper_ring_load(p, n, RT, lo, nf, F);
        return;
    }
    if (d.rhs == 2) {
        if (dim != 3 || d.dirichlet_sides != 0b000111u)
            throw Error{AMG_EINVAL, "rhs = 2 (the paper's cube data) needs dim = 3 and Dirichlet sides 1, 2, 3"};
        paper_cube_load(p, n, T, lo, nf, F);
        return;
    }
    F.alloc(N);
    if (d.rhs == 1) {
        std::memset(F.data(), 0, sizeof(double) * N);
        return;
    }
    std::vector<double> f1[3];
    for (int ax = 0; ax < dim; ax++) f1[ax] = load_factor(ax, p, n);
    const double cfac = (dim == 2 ? 5.0 : 9.0) * M_PI * M_PI / 4.0;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < N; row++) {
        int a = lo[0] + (int)(row % nf[0]);
        int b = lo[1] + (int)((row / nf[0]) % nf[1]);
        int c = lo[2] + (int)(row / ((int64_t)nf[0] * nf[1]));
        double v = f1[0][a] * f1[1][b];
        if (dim == 3) v *= f1[2][c];
        F[row] = cfac * v;
    }
}

}  // namespace amgb

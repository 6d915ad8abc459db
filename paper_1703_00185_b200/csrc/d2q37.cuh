// d2q37.cuh -- per-site D2Q37 arithmetic for sm_100a.
//
// Two variants of the reference collide (kernels.py:139-146):
//
//  * Exact: the reference's numpy expression tree (kernels.py:41-136,
//    SURVEY Appendix B) with one IEEE binary64 operation per reference
//    operation, spelled with __dadd_rn/__dmul_rn so nvcc cannot contract or
//    reorder.  FMA is used ONLY where the product is exact (multiplier a power
//    of two), where fma(a,b,c) == RN(c + a*b) bit for bit.  Results are
//    bitwise equal to the reference.  Three restructurings keep the bits
//    while cutting work:
//      - speed-shell CSE: every sub-expression that depends only on (site, q)
//        (theta*q, 3*theta*q, ...) is evaluated once per shell, not per l;
//      - +/-c pairing: for c_l' = -c_l, p' = -p exactly, so p^2, c2 and c4
//        are identical and c3 flips sign exactly; one evaluation serves both;
//      - division by 6 and 24 uses Markstein's correction
//        q = RN(x*RN(1/b)); r = fma(-q,b,x); RN(q + r*RN(1/b)) == RN(x/b)
//        (q is within 1 ulp of x/b for b = 6*2^k, so the theorem applies);
//        division by cs and cs2 uses two correction steps.
//  * Fast: FMA everywhere, the Hermite polynomial rewritten per shell as a
//    degree-4 polynomial in p with site-dependent coefficients, even/odd split
//    over +/-c pairs.  Agrees with the reference to ~1e-15 relative per step.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tlb {

constexpr int Q = 37;
constexpr int NSHELL = 8;

// Reference ordering velocity_set.py:46-59.
__host__ __device__ constexpr int CX(int l) {
    constexpr int t[Q] = {0, -1, 0, 0, 1, -1, -1, 1, 1, -2, 0, 0, 2,
                          -2, -2, -1, -1, 1, 1, 2, 2, -2, -2, 2, 2,
                          -3, 0, 0, 3, -3, -3, -1, -1, 1, 1, 3, 3};
    return t[l];
}
__host__ __device__ constexpr int CY(int l) {
    constexpr int t[Q] = {0, 0, -1, 1, 0, -1, 1, -1, 1, 0, -2, 2, 0,
                          -1, 1, -2, 2, -2, 2, -1, 1, -2, 2, -2, 2,
                          0, -3, 3, 0, -1, 1, -3, 3, -3, 3, -1, 1};
    return t[l];
}
// speed shells (0,0) (1,0) (1,1) (2,0) (2,1) (2,2) (3,0) (3,1): [start, n)
__host__ __device__ constexpr int SH_START(int s) {
    constexpr int t[NSHELL] = {0, 1, 5, 9, 13, 21, 25, 29};
    return t[s];
}
__host__ __device__ constexpr int SH_N(int s) {
    constexpr int t[NSHELL] = {1, 4, 4, 4, 8, 4, 4, 8};
    return t[s];
}
__host__ __device__ constexpr int SHELL_OF(int l) {
    return l < 1 ? 0 : l < 5 ? 1 : l < 9 ? 2 : l < 13 ? 3 : l < 21 ? 4
         : l < 25 ? 5 : l < 29 ? 6 : 7;
}
// Within a shell the signed permutations are sorted, so the partner -c of
// entry i is entry n-1-i.
__host__ __device__ constexpr int PARTNER(int l) {
    return 2 * SH_START(SHELL_OF(l)) + SH_N(SHELL_OF(l)) - 1 - l;
}
__host__ __device__ constexpr int iabs(int v) { return v < 0 ? -v : v; }
__host__ __device__ constexpr bool pow2(int v) {
    return v == 1 || v == 2 || v == 4 || v == 8;
}

// Stencil constants, uploaded once per device (tlb_set_stencil).
struct StencilConst {
    double E[4];       // |c|/cs for |c| = 0..3 (kernels.py:95-96)
    double qsh[NSHELL]; // q = ex^2 + ey^2 per shell (kernels.py:97)
    double wsh[NSHELL]; // w per shell (velocity_set.py:108)
    double cs, cs2, rcs, rcs2; // sqrt(cs2), cs2 and RN reciprocals
    double r6, r24;            // RN(1/6), RN(1/24)
    int set;
};

// Physics constants derived on the host exactly as the reference does.
struct Phys {
    double K1, K2, K3;  // tau*gx, tau*gy, tau*tau*g2/D  (kernels.py:130-133)
    double omega;       // dt/tau                        (kernels.py:145)
    double Tbot, Ttop;  // wall temperatures
    int order;
};

// One copy per translation unit (internal linkage, no -rdc): tlb_set_stencil
// uploads the same table into each (tlb.cu, tb2.cu).
static __constant__ StencilConst C;

// Population accessors: the arithmetic below reads f_l through get(l) and
// writes results through put(l, v), so the same code runs on a
// register-resident 37-vector (RegF) or streams each output straight to
// global memory as soon as it is final (RegStoreF in tlb.cu).
struct RegF {
    double (&a)[Q];
    __device__ __forceinline__ double get(int l) const { return a[l]; }
    __device__ __forceinline__ void put(int l, double v) { a[l] = v; }
};

// ---------------------------------------------------------------- exact --
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// acc + c*f with the reference's rounding: exact product -> fma is identical.
template <int c>
__device__ __forceinline__ double acc_cf(double acc, double f) {
    if constexpr (c == 0) {
        return acc;
    } else if constexpr (pow2(iabs(c))) {
        return dfma((double)c, f, acc);
    } else {
        return dadd(acc, dmul((double)c, f));
    }
}

// RN(x / b) for the constant b with RN(1/b) = y (two Markstein steps).
__device__ __forceinline__ double div_const2(double x, double b, double y) {
    double q0 = dmul(x, y);
    double r0 = dfma(-q0, b, x);
    double q1 = dfma(r0, y, q0);
    double r1 = dfma(-q1, b, x);
    return dfma(r1, y, q1);
}
// RN(x / b), b in {6, 24}: one Markstein step suffices (see header).
__device__ __forceinline__ double div_const1(double x, double b, double y) {
    double q0 = dmul(x, y);
    double r0 = dfma(-q0, b, x);
    return dfma(r0, y, q0);
}

template <int l>
__device__ __forceinline__ double pdot_exact(double vx, double vy) {
    // p = ex*vx + ey*vy (kernels.py:98).  A zero component contributes a
    // signed zero, which cannot change a non-zero sum; it is dropped.
    constexpr int cx = CX(l), cy = CY(l);
    if constexpr (cx == 0 && cy == 0) {
        return 0.0;
    } else if constexpr (cx == 0) {
        return dmul(cy > 0 ? C.E[iabs(cy)] : -C.E[iabs(cy)], vy);
    } else if constexpr (cy == 0) {
        return dmul(cx > 0 ? C.E[iabs(cx)] : -C.E[iabs(cx)], vx);
    } else {
        return dadd(dmul(cx > 0 ? C.E[iabs(cx)] : -C.E[iabs(cx)], vx),
                    dmul(cy > 0 ? C.E[iabs(cy)] : -C.E[iabs(cy)], vy));
    }
}

// Site-level quantities of equilibrium() (kernels.py:87-91, 100-121).
// Power-of-two identities keep these bitwise equal to the reference while
// saving operations: RN(2^k x) = 2^k RN(x) and fma(2^k, a, b) = RN(b + 2^k a)
// (exact products; no subnormal intermediates occur for lattice states).
// Hence 6*theta = 2*RN(3*theta), RN(6 theta q) = 2 RN(3 theta q),
// RN(RN(6p) p) = 2 RN(RN(3p) p), (8 theta) s = 8 RN(theta s), and the
// reference's (theta*theta*4)*q = 4 RN(theta theta q).
struct EqSite {
    double rho, vx, vy, theta, s;
    double s2t, s4t, t3, t3t, tt, c3x;
};

__device__ __forceinline__ EqSite eq_site_exact(double rho, double ux, double uy,
                                                double T) {
    EqSite e;
    e.rho = rho;
    e.vx = div_const2(ux, C.cs, C.rcs);
    e.vy = div_const2(uy, C.cs, C.rcs);
    e.theta = dsub(div_const2(T, C.cs2, C.rcs2), 1.0);
    e.s = dadd(dmul(e.vx, e.vx), dmul(e.vy, e.vy));
    const double th = e.theta;
    e.s2t = dfma(2.0, th, e.s);                // s + D*theta
    e.s4t = dfma(4.0, th, e.s);                // s + (D+2)*theta
    e.t3 = dmul(3.0, th);                      // 3.0*theta (6.0*theta == 2*t3)
    e.t3t = dmul(e.t3, th);                    // 3.0*theta*theta
    e.tt = dmul(th, th);                       // theta*theta
    // ((s*s) + ((8 theta) s)) + ((8 theta) theta)
    const double inner3 = dfma(8.0, e.tt, dfma(8.0, dmul(th, e.s), dmul(e.s, e.s)));
    e.c3x = dmul(3.0, inner3);
    return e;
}

// Per-shell sub-expressions (depend on q only).
struct EqShell {
    double tq, t3q, t3tqq, qs, ttq, wr;
};

template <int sh>
__device__ __forceinline__ EqShell eq_shell_exact(const EqSite &e) {
    const double q = C.qsh[sh];
    EqShell z;
    z.tq = dmul(e.theta, q);
    z.t3q = dmul(e.t3, q);                     // (6 theta) q == 2 t3q
    z.t3tqq = dmul(dmul(e.t3t, q), q);
    z.qs = dmul(q, e.s);
    z.ttq = dmul(e.tt, q);                     // (theta theta 4) q == 4 ttq
    z.wr = dmul(C.wsh[sh], e.rho);             // w*rho
    return z;
}

// Equilibrium pair (feq for +c and -c) with the reference rounding
// (kernels.py:98-124).
template <int ORDER>
__device__ __forceinline__ void eq_pair_exact(const EqSite &e, const EqShell &z,
                                              double p, double &fp, double &fm) {
    const double pp = dmul(p, p);
    const double c2 = dsub(dadd(pp, z.tq), e.s2t);
    double bp = dfma(0.5, c2, dadd(1.0, p));   // (1+p) + 0.5*c2
    double bm = dfma(0.5, c2, dsub(1.0, p));
    if constexpr (ORDER >= 3) {
        const double ppp = dmul(pp, p);
        const double w3 = dmul(z.t3q, p);                   // ((3 theta) q) p
        const double p3 = dmul(3.0, p);                      // 3.0*p
        const double c3 = dsub(dadd(ppp, w3), dmul(p3, e.s4t));
        const double d6 = div_const1(c3, 6.0, C.r6);
        bp = dadd(bp, d6);
        bm = dsub(bm, d6);
        if constexpr (ORDER >= 4) {
            const double pppp = dmul(ppp, p);
            // (((6 theta) q) p) p == 2 RN(w3 p);  ((6 p) p) == 2 RN(p3 p)
            const double sum1 = dadd(dfma(2.0, dmul(w3, p), pppp), z.t3tqq);
            const double in6 = dfma(4.0, z.ttq,
                                    dadd(dmul(dmul(e.s, p), p),
                                         dmul(e.theta, dfma(2.0, dmul(p3, p), z.qs))));
            const double c4 = dadd(dsub(sum1, dmul(6.0, in6)), e.c3x);
            const double d24 = div_const1(c4, 24.0, C.r24);
            bp = dadd(bp, d24);
            bm = dadd(bm, d24);
        }
    }
    fp = dmul(z.wr, bp);
    fm = dmul(z.wr, bm);
}

// Rest population l = 0 (p == 0 exactly up to the sign of zero).
template <int ORDER>
__device__ __forceinline__ double eq_rest_exact(const EqSite &e, const EqShell &z) {
    double fp, fm;
    eq_pair_exact<ORDER>(e, z, 0.0, fp, fm);
    return fp;
}

// out = f - omega*(f - feq)  (kernels.py:146)
__device__ __forceinline__ double relax_exact(double f, double feq, double omega) {
    return dsub(f, dmul(omega, dsub(f, feq)));
}

// MODE 0: f <- equilibrium (bc);  MODE 1: f <- BGK relax toward equilibrium
template <int ORDER, int MODE, int sh, class F>
__device__ __forceinline__ void eq_shell_apply_exact(F &f, const EqSite &e, double omega) {
    const EqShell z = eq_shell_exact<sh>(e);
    constexpr int s0 = SH_START(sh), n = SH_N(sh);
    if constexpr (sh == 0) {
        const double feq = eq_rest_exact<ORDER>(e, z);
        f.put(0, MODE ? relax_exact(f.get(0), feq, omega) : feq);
    } else {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const int l = s0 + i;  // partner s0 + n - 1 - i
            double p;
            // dispatch the compile-time pdot through a switch on l
            switch (l) {
#define TLB_PD(L) case L: p = pdot_exact<L>(e.vx, e.vy); break;
                TLB_PD(1) TLB_PD(2) TLB_PD(5) TLB_PD(6) TLB_PD(9) TLB_PD(10)
                TLB_PD(13) TLB_PD(14) TLB_PD(15) TLB_PD(16) TLB_PD(21) TLB_PD(22)
                TLB_PD(25) TLB_PD(26) TLB_PD(29) TLB_PD(30) TLB_PD(31) TLB_PD(32)
#undef TLB_PD
                default: p = 0.0;
            }
            double fp, fm;
            eq_pair_exact<ORDER>(e, z, p, fp, fm);
            const int lm = s0 + n - 1 - i;
            f.put(l, MODE ? relax_exact(f.get(l), fp, omega) : fp);
            f.put(lm, MODE ? relax_exact(f.get(lm), fm, omega) : fm);
        }
    }
}

template <int ORDER, int MODE, class F>
__device__ __forceinline__ void eq_all_exact(F &f, const EqSite &e, double omega) {
    eq_shell_apply_exact<ORDER, MODE, 0, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 1, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 2, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 3, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 4, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 5, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 6, F>(f, e, omega);
    eq_shell_apply_exact<ORDER, MODE, 7, F>(f, e, omega);
}

// rho = sum_l f_l in fixed l order from +0.0 (kernels.py:49, 54; bc :198-200)
template <class F>
__device__ __forceinline__ double rho_exact(const F &f) {
    double rho = 0.0;
#pragma unroll
    for (int l = 0; l < Q; ++l) rho = dadd(rho, f.get(l));
    return rho;
}

template <int l, class F>
__device__ __forceinline__ void mom_step(const F &f, double &rho, double &mx, double &my,
                                         double &e2) {
    constexpr int cx = CX(l), cy = CY(l), c2 = cx * cx + cy * cy;
    const double fl = f.get(l);
    rho = dadd(rho, fl);
    mx = acc_cf<cx>(mx, fl);
    my = acc_cf<cy>(my, fl);
    e2 = acc_cf<c2>(e2, fl);
}

template <int... Ls>
struct MomSeq {
    template <class F>
    __device__ __forceinline__ static void run(const F &f, double &rho, double &mx,
                                               double &my, double &e2) {
        (mom_step<Ls, F>(f, rho, mx, my, e2), ...);
    }
};

// RN(x / b) given y = RN(1/b): two Markstein steps (the first makes the
// quotient faithful, the second correctly rounded; Markstein's theorem).
__device__ __forceinline__ double div_rcp2(double x, double b, double y) {
    return div_const2(x, b, y);
}

// moments (kernels.py:41-71).  Returns false if !(rho > 0).  The three
// divisions share one correctly rounded reciprocal of rho (and of 2 rho,
// which is exactly half of it) and are completed by Markstein corrections:
// bit for bit the IEEE quotients of the reference.
// The divisions of moments (kernels.py:55-71) given the fixed-order sums.
__device__ __forceinline__ bool moments_tail(double r, double mx, double my, double e2,
                                             double &rho, double &ux, double &uy, double &T) {
    rho = r;
    if (!(r > 1e-300 && r < 1e300)) {  // degenerate or extreme: plain IEEE division
        ux = __ddiv_rn(mx, r);
        uy = __ddiv_rn(my, r);
        T = __ddiv_rn(dsub(e2, dmul(r, dadd(dmul(ux, ux), dmul(uy, uy)))), dmul(2.0, r));
        return r > 0.0;
    }
    const double yr = __drcp_rn(r);
    ux = div_rcp2(mx, r, yr);
    uy = div_rcp2(my, r, yr);
    T = div_rcp2(dsub(e2, dmul(r, dadd(dmul(ux, ux), dmul(uy, uy)))), dmul(2.0, r),
                 dmul(0.5, yr));
    return true;
}

template <class F>
__device__ __forceinline__ bool moments_exact(const F &f, double &rho, double &ux,
                                              double &uy, double &T) {
    double r = 0.0, mx = 0.0, my = 0.0, e2 = 0.0;
    MomSeq<0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20,
           21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32, 33, 34, 35, 36>::run(f, r, mx, my, e2);
    return moments_tail(r, mx, my, e2, rho, ux, uy, T);
}

// collide one site in place (kernels.py:139-146).  Returns TLB_ST_* bits.
template <int ORDER, class F>
__device__ __forceinline__ unsigned collide_exact(F &f, const Phys &P) {
    double rho, ux, uy, T;
    if (!moments_exact(f, rho, ux, uy, T)) return 1u;
    const double ub = dadd(ux, P.K1);
    const double vb = dadd(uy, P.K2);
    const double Tb = dsub(T, P.K3);
    if (!(Tb > 0.0)) return 2u;
    const EqSite e = eq_site_exact(rho, ub, vb, Tb);
    eq_all_exact<ORDER, 1, F>(f, e, P.omega);
    return 0u;
}

// bc on one wall site (kernels.py:197-203): rho = sum f, f = feq(rho,0,0,Tw).
template <int ORDER, class F>
__device__ __forceinline__ unsigned bc_exact(F &f, double Tw) {
    const double rho = rho_exact(f);
    const EqSite e = eq_site_exact(rho, 0.0, 0.0, Tw);
    eq_all_exact<ORDER, 0, F>(f, e, 0.0);
    return (rho > 0.0) ? 0u : 4u;
}

// ----------------------------------------------------------------- fast --
template <int l>
__device__ __forceinline__ double pdot_fast(double vx, double vy) {
    constexpr int cx = CX(l), cy = CY(l);
    if constexpr (cx == 0 && cy == 0) {
        return 0.0;
    } else if constexpr (cx == 0) {
        return (cy > 0 ? C.E[iabs(cy)] : -C.E[iabs(cy)]) * vy;
    } else if constexpr (cy == 0) {
        return (cx > 0 ? C.E[iabs(cx)] : -C.E[iabs(cx)]) * vx;
    } else {
        return fma(cx > 0 ? C.E[iabs(cx)] : -C.E[iabs(cx)], vx,
                   (cy > 0 ? C.E[iabs(cy)] : -C.E[iabs(cy)]) * vy);
    }
}

struct FastSite {
    double theta, s, vx, vy, W; // W = omega*rho (relax) or rho (bc)
};

// Order 4: the shell coefficients below as polynomials in the shell's q,
// with site-level coefficients (a = theta q - s substituted):
//   A0/W = (1 - th + th^2) + (1/2 - th) a + a^2/8 = a00 + a01 q + a02 q^2
//   A1/W = 1 + (a - 4 th)/2                     = b0 + b1 q
//   A2/W = 1/2 + (a - 6 th)/4                   = g0 + g1 q
// so a shell costs 4 FMAs instead of ~12 (same polynomial, reassociated).
struct FastQ {
    double a00, a01, a02, b0, b1, g0, g1;
};
__device__ __forceinline__ FastQ fast_q(const FastSite &e) {
    const double th = e.theta, s = e.s;
    const double c0 = fma(th, th - 1.0, 1.0);     // 1 - th + th^2
    const double c1 = 0.5 - th;
    FastQ k;
    k.a00 = fma(0.125 * s, s, fma(-c1, s, c0));   // c0 - c1 s + s^2/8
    k.a01 = th * fma(-0.25, s, c1);               // th (c1 - s/4)
    k.a02 = 0.125 * th * th;
    k.b0 = fma(-0.5, s, fma(-2.0, th, 1.0));      // 1 - 2 th - s/2
    k.b1 = 0.5 * th;
    k.g0 = fma(-0.25, s, fma(-1.5, th, 0.5));     // 1/2 - 3/2 th - s/4
    k.g1 = 0.25 * th;
    return k;
}

// Hermite polynomial of kernels.py:99-123 regrouped in powers of p:
// poly = A0 + A1 p + A2 p^2 + A3 p^3 + A4 p^4 with a = theta*q - s:
// A0 = 1 + (a-2th)/2 + [a^2/8 - th*a + th^2]_{order 4}, A1 = 1 + [(a-4th)/2]_{>=3},
// A2 = 1/2 + [(a-6th)/4]_{4}, A3 = [1/6]_{>=3}, A4 = [1/24]_{4}.
template <int ORDER, int MODE, int sh, class F>
__device__ __forceinline__ void fast_shell(F &f, const FastSite &e, const FastQ &k,
                                           double omr) {
    const double q = C.qsh[sh];
    const double W = e.W * C.wsh[sh];
    double A0, A1 = 1.0, A2 = 0.5, A3 = 0.0, A4 = 0.0;
    if constexpr (ORDER >= 4) {
        A0 = fma(fma(k.a02, q, k.a01), q, k.a00);
        A1 = fma(k.b1, q, k.b0);
        A2 = fma(k.g1, q, k.g0);
        A3 = 1.0 / 6.0;
        A4 = 1.0 / 24.0;
    } else {
        const double th = e.theta;
        const double a = fma(th, q, -e.s);
        A0 = fma(0.5, a - 2.0 * th, 1.0);
        if constexpr (ORDER >= 3) {
            A1 = fma(0.5, a - 4.0 * th, 1.0);
            A3 = 1.0 / 6.0;
        }
    }
    A0 *= W; A1 *= W; A2 *= W; A3 *= W; A4 *= W;
    constexpr int s0 = SH_START(sh), n = SH_N(sh);
    if constexpr (sh == 0) {
        f.put(0, MODE ? fma(omr, f.get(0), A0) : A0);
    } else {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const int l = s0 + i, lm = s0 + n - 1 - i;
            double p;
            switch (l) {
#define TLB_PD(L) case L: p = pdot_fast<L>(e.vx, e.vy); break;
                TLB_PD(1) TLB_PD(2) TLB_PD(5) TLB_PD(6) TLB_PD(9) TLB_PD(10)
                TLB_PD(13) TLB_PD(14) TLB_PD(15) TLB_PD(16) TLB_PD(21) TLB_PD(22)
                TLB_PD(25) TLB_PD(26) TLB_PD(29) TLB_PD(30) TLB_PD(31) TLB_PD(32)
#undef TLB_PD
                default: p = 0.0;
            }
            const double p2 = p * p;
            const double ev = fma(p2, fma(p2, A4, A2), A0);
            const double od = p * fma(p2, A3, A1);
            if (MODE) {
                f.put(l, fma(omr, f.get(l), ev + od));
                f.put(lm, fma(omr, f.get(lm), ev - od));
            } else {
                f.put(l, ev + od);
                f.put(lm, ev - od);
            }
        }
    }
}

template <int ORDER, int MODE, class F>
__device__ __forceinline__ void fast_all(F &f, const FastSite &e, double omr) {
    FastQ k{};
    if constexpr (ORDER >= 4) k = fast_q(e);
    fast_shell<ORDER, MODE, 0, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 1, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 2, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 3, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 4, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 5, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 6, F>(f, e, k, omr);
    fast_shell<ORDER, MODE, 7, F>(f, e, k, omr);
}

template <int ORDER, class F>
__device__ __forceinline__ unsigned collide_fast(F &f, const Phys &P);

// Fast moments over +/-c pairs: with s = f_c + f_-c and d = f_c - f_-c,
// rho = f_0 + sum s, m = sum c d, e2 = sum_shell |c|^2 (sum of the shell's
// s) -- a third of the FMAs of the direct sums, and every shell an
// independent partial sum (short dependency chains: the two-step kernel
// runs only 2 warps per scheduler).
template <int sh, class FM>
__device__ __forceinline__ void fast_shell_moments(const FM &fm, double &S, double &mx,
                                                   double &my) {
    constexpr int s0 = SH_START(sh), n = SH_N(sh);
    S = 0.0;
    mx = 0.0;
    my = 0.0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
        const int l = s0 + i, lm = s0 + n - 1 - i;
        const double a = fm.get(l), b = fm.get(lm);
        const double sp = a + b, dm = a - b;
        S += sp;
        if (CX(l)) mx = fma((double)CX(l), dm, mx);
        if (CY(l)) my = fma((double)CY(l), dm, my);
    }
}

template <class FM>
__device__ __forceinline__ void fast_moments(const FM &fm, double &rho, double &mx, double &my,
                                             double &e2) {
    double S1, S2, S3, S4, S5, S6, S7, x1, x2, x3, x4, x5, x6, x7, y1, y2, y3, y4, y5, y6, y7;
    fast_shell_moments<1>(fm, S1, x1, y1);
    fast_shell_moments<2>(fm, S2, x2, y2);
    fast_shell_moments<3>(fm, S3, x3, y3);
    fast_shell_moments<4>(fm, S4, x4, y4);
    fast_shell_moments<5>(fm, S5, x5, y5);
    fast_shell_moments<6>(fm, S6, x6, y6);
    fast_shell_moments<7>(fm, S7, x7, y7);
    rho = ((fm.get(0) + S1) + (S2 + S3)) + ((S4 + S5) + (S6 + S7));
    mx = ((x1 + x2) + (x3 + x4)) + ((x5 + x6) + x7);
    my = ((y1 + y2) + (y3 + y4)) + ((y5 + y6) + y7);
    // |c|^2 per shell: 1, 2, 4, 5, 8, 9, 10
    e2 = fma(10.0, S7, fma(9.0, S6, fma(8.0, S5, 5.0 * S4))) +
         fma(4.0, S3, fma(2.0, S2, S1));
}

template <int ORDER, class FM, class F>
__device__ __forceinline__ unsigned collide_fast2(const FM &fm, F &f, const Phys &P) {
    double rho, mx, my, e2;
    fast_moments(fm, rho, mx, my, e2);
    if (!(rho > 0.0)) return 1u;
    const double ri = 1.0 / rho;
    const double ux = mx * ri, uy = my * ri;
    const double T = 0.5 * ri * fma(-rho, fma(ux, ux, uy * uy), e2);
    FastSite e;
    e.vx = (ux + P.K1) * C.rcs;
    e.vy = (uy + P.K2) * C.rcs;
    const double Tb = T - P.K3;
    if (!(Tb > 0.0)) return 2u;
    e.theta = fma(Tb, C.rcs2, -1.0);
    e.s = fma(e.vx, e.vx, e.vy * e.vy);
    e.W = P.omega * rho;
    fast_all<ORDER, 1, F>(f, e, 1.0 - P.omega);
    return 0u;
}

template <int ORDER, class F>
__device__ __forceinline__ unsigned collide_fast(F &f, const Phys &P) {
    return collide_fast2<ORDER, F, F>(f, f, P);
}

// ------------------------------------------ fast, one site on two threads --
// The split two-step kernel (tb2.cu, k_tb2s) runs a site on two threads, one
// in each warp of a pair: half 0 owns the shells (0,0) (1,0) (1,1) (2,0)
// (3,0) -- 17 populations, 5 shell set-ups, 8 +/-c pairs -- and half 1 the
// shells (2,1) (2,2) (3,1) -- 20 populations, 3 set-ups, 10 pairs (about the
// same FP64 work).  Each half sums its shells' moments, the pair exchanges
// the partial sums (XCH::sum: own + partner's, the same IEEE sum in both
// threads), and each half relaxes only its own populations.  Same algebra as
// collide_fast; the moment sums are grouped differently (1e-12 contract).
__host__ __device__ constexpr bool HALF_SHELL(int h, int sh) {
    return (sh == 0 || sh == 1 || sh == 2 || sh == 3 || sh == 6) == (h == 0);
}
__host__ __device__ constexpr bool IN_HALF(int h, int l) { return HALF_SHELL(h, SHELL_OF(l)); }

template <int H, class FM>
__device__ __forceinline__ void fast_moments_half(const FM &fm, double (&m)[4]) {
    if constexpr (H == 0) {
        double S1, S2, S3, S6, x1, x2, x3, x6, y1, y2, y3, y6;
        fast_shell_moments<1>(fm, S1, x1, y1);
        fast_shell_moments<2>(fm, S2, x2, y2);
        fast_shell_moments<3>(fm, S3, x3, y3);
        fast_shell_moments<6>(fm, S6, x6, y6);
        m[0] = ((fm.get(0) + S1) + (S2 + S3)) + S6;
        m[1] = (x1 + x2) + (x3 + x6);
        m[2] = (y1 + y2) + (y3 + y6);
        m[3] = fma(9.0, S6, fma(4.0, S3, fma(2.0, S2, S1)));   // |c|^2 = 1, 2, 4, 9
    } else {
        double S4, S5, S7, x4, x5, x7, y4, y5, y7;
        fast_shell_moments<4>(fm, S4, x4, y4);
        fast_shell_moments<5>(fm, S5, x5, y5);
        fast_shell_moments<7>(fm, S7, x7, y7);
        m[0] = (S4 + S5) + S7;
        m[1] = (x4 + x5) + x7;
        m[2] = (y4 + y5) + y7;
        m[3] = fma(10.0, S7, fma(8.0, S5, 5.0 * S4));         // |c|^2 = 5, 8, 10
    }
}

template <int H, int ORDER, int MODE, class F>
__device__ __forceinline__ void fast_all_half(F &f, const FastSite &e, double omr) {
    FastQ k{};
    if constexpr (ORDER >= 4) k = fast_q(e);
    if constexpr (H == 0) {
        fast_shell<ORDER, MODE, 0, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 1, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 2, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 3, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 6, F>(f, e, k, omr);
    } else {
        fast_shell<ORDER, MODE, 4, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 5, F>(f, e, k, omr);
        fast_shell<ORDER, MODE, 7, F>(f, e, k, omr);
    }
}

// collide_fast2 for half H; every thread of both warps must call it (the
// exchange is a pair barrier).  The failure bits are the same in both halves.
template <int H, int ORDER, class F, class XCH>
__device__ __forceinline__ unsigned collide_fast_half(F &f, const Phys &P, XCH &x) {
    double m[4];
    fast_moments_half<H>(f, m);
    x.template sum<4>(m, 0);
    const double rho = m[0];
    if (!(rho > 0.0)) return 1u;
    const double ri = 1.0 / rho;
    const double ux = m[1] * ri, uy = m[2] * ri;
    const double T = 0.5 * ri * fma(-rho, fma(ux, ux, uy * uy), m[3]);
    FastSite e;
    e.vx = (ux + P.K1) * C.rcs;
    e.vy = (uy + P.K2) * C.rcs;
    const double Tb = T - P.K3;
    if (!(Tb > 0.0)) return 2u;
    e.theta = fma(Tb, C.rcs2, -1.0);
    e.s = fma(e.vx, e.vx, e.vy * e.vy);
    e.W = P.omega * rho;
    fast_all_half<H, ORDER, 1, F>(f, e, 1.0 - P.omega);
    return 0u;
}

// bc_fast for half H: the partial rho is exchanged by every thread (exchange
// slot `slot`), the wall equilibrium applied only where `on`.
template <int H, int ORDER, class F, class XCH>
__device__ __forceinline__ unsigned bc_fast_half(F &f, double Tw, XCH &x, int slot, bool on) {
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
        if (!IN_HALF(H, l)) continue;
        const double fl = f.get(l);
        if (l & 1) r1 += fl; else r0 += fl;
    }
    double v[1] = {r0 + r1};
    x.template sum<1>(v, slot);
    if (!on) return 0u;
    const double rho = v[0];
    FastSite e;
    e.vx = 0.0; e.vy = 0.0; e.s = 0.0;
    e.theta = fma(Tw, C.rcs2, -1.0);
    e.W = rho;
    fast_all_half<H, ORDER, 0, F>(f, e, 0.0);
    return (rho > 0.0) ? 0u : 4u;
}

template <int ORDER, class F>
__device__ __forceinline__ unsigned bc_fast(F &f, double Tw) {
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int l = 0; l < Q; ++l) {
        const double fl = f.get(l);
        if (l & 1) r1 += fl; else r0 += fl;
    }
    const double rho = r0 + r1;
    FastSite e;
    e.vx = 0.0; e.vy = 0.0; e.s = 0.0;
    e.theta = fma(Tw, C.rcs2, -1.0);
    e.W = rho;
    fast_all<ORDER, 0, F>(f, e, 0.0);
    return (rho > 0.0) ? 0u : 4u;
}

}  // namespace tlb

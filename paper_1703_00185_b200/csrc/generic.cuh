// generic.cuh -- any velocity set (D2Q9, or D2Q37 in another order): the
// reference arithmetic evaluated per population from a stencil table in
// constant memory (kernels.py:41-146, 168-203), one IEEE operation per
// reference operation.  This is the correctness path for stencils other
// than the compile-time-specialised D2Q37 of d2q37.cuh;
// "fast" arithmetic falls back to it.  Instantiated for Q = 9 and Q = 37 (the
// latter lets the tests cross-check the specialised kernels bit for bit).
#pragma once

constexpr int GQ = 37;  // table capacity (SiteLaunch offsets are sized Q = 37)

struct GenConst {
    int Q;
    int cx[GQ], cy[GQ];
    double w[GQ], ex[GQ], ey[GQ], q[GQ];
    double cs, cs2;
    double rcs, rcs2, r6, r24;  // RN reciprocals for the Markstein divisions
};

__constant__ GenConst G;

struct GenHost {
    int Q = 0;
    int cx[GQ], cy[GQ];
};
static GenHost g_gen[64];  // host copy per device (face plans, offsets)
static int g_qdev[64];     // 37 = specialised D2Q37 kernels, else generic Q

static const GenHost &gen_host() {
    int dev = 0;
    cudaGetDevice(&dev);
    return g_gen[dev < 0 || dev >= 64 ? 0 : dev];
}

static bool device_generic() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < 64 && g_qdev[dev] != 0 && g_qdev[dev] != 37;
}

// moments, kernels.py:41-71 (check is done by the caller)
template <int NQ>
__device__ __forceinline__ void gen_moments(const double (&f)[NQ], double &rho, double &ux,
                                            double &uy, double &T) {
    double r = 0.0, mx = 0.0, my = 0.0, e2 = 0.0;
#pragma unroll
    for (int l = 0; l < NQ; ++l) {
        const double cx = (double)G.cx[l], cy = (double)G.cy[l];
        r = __dadd_rn(r, f[l]);
        if (cx != 0.0) mx = __dadd_rn(mx, __dmul_rn(cx, f[l]));
        if (cy != 0.0) my = __dadd_rn(my, __dmul_rn(cy, f[l]));
        const double c2 = __dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy));
        if (c2 != 0.0) e2 = __dadd_rn(e2, __dmul_rn(c2, f[l]));
    }
    // the three divisions, correctly rounded via one reciprocal and
    // Markstein corrections (d2q37.cuh: same bits as __ddiv_rn)
    moments_tail(r, mx, my, e2, rho, ux, uy, T);
}

// equilibrium, kernels.py:87-124, written term by term in the reference's
// left-to-right order (D = 2)
template <int NQ>
__device__ __forceinline__ void gen_equilibrium(double rho, double ux, double uy, double T,
                                                int order, double (&out)[NQ]) {
    const double D = 2.0;
    // correctly rounded divisions by the constants cs, cs2, 6, 24
    const double vx = div_const2(ux, G.cs, G.rcs), vy = div_const2(uy, G.cs, G.rcs);
    const double th = __dsub_rn(div_const2(T, G.cs2, G.rcs2), 1.0);
    const double s = __dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy));
#pragma unroll
    for (int l = 0; l < NQ; ++l) {
        const double q = G.q[l];
        const double p = __dadd_rn(__dmul_rn(G.ex[l], vx), __dmul_rn(G.ey[l], vy));
        double poly = __dadd_rn(1.0, p);
        const double pp = __dmul_rn(p, p);
        const double c2 = __dsub_rn(__dadd_rn(pp, __dmul_rn(th, q)), __dadd_rn(s, __dmul_rn(D, th)));
        poly = __dadd_rn(poly, __dmul_rn(0.5, c2));
        if (order >= 3) {
            const double c3 = __dsub_rn(
                __dadd_rn(__dmul_rn(pp, p), __dmul_rn(__dmul_rn(__dmul_rn(3.0, th), q), p)),
                __dmul_rn(__dmul_rn(3.0, p), __dadd_rn(s, __dmul_rn(D + 2.0, th))));
            poly = __dadd_rn(poly, div_const1(c3, 6.0, G.r6));
        }
        if (order >= 4) {
            const double A = __dmul_rn(__dmul_rn(pp, p), p);
            const double B = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(6.0, th), q), p), p);
            const double Cc = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(3.0, th), th), q), q);
            const double in6 = __dadd_rn(
                __dadd_rn(__dmul_rn(__dmul_rn(s, p), p),
                          __dmul_rn(th, __dadd_rn(__dmul_rn(__dmul_rn(D + 4.0, p), p),
                                                  __dmul_rn(q, s)))),
                __dmul_rn(__dmul_rn(__dmul_rn(th, th), D + 2.0), q));
            const double in3 = __dadd_rn(
                __dadd_rn(__dmul_rn(s, s), __dmul_rn(__dmul_rn(2.0 * D + 4.0, th), s)),
                __dmul_rn(__dmul_rn(D * (D + 2.0), th), th));
            const double c4 = __dadd_rn(__dsub_rn(__dadd_rn(__dadd_rn(A, B), Cc), __dmul_rn(6.0, in6)),
                                        __dmul_rn(3.0, in3));
            poly = __dadd_rn(poly, div_const1(c4, 24.0, G.r24));
        }
        out[l] = __dmul_rn(__dmul_rn(G.w[l], rho), poly);
    }
}

template <int NQ>
__device__ __forceinline__ unsigned gen_collide(double (&f)[NQ], const Phys &P) {
    double rho, ux, uy, T;
    gen_moments<NQ>(f, rho, ux, uy, T);
    if (!(rho > 0.0)) return 1u;
    const double ub = __dadd_rn(ux, P.K1), vb = __dadd_rn(uy, P.K2), Tb = __dsub_rn(T, P.K3);
    if (!(Tb > 0.0)) return 2u;
    double feq[NQ];
    gen_equilibrium<NQ>(rho, ub, vb, Tb, P.order, feq);
#pragma unroll
    for (int l = 0; l < NQ; ++l)
        f[l] = __dsub_rn(f[l], __dmul_rn(P.omega, __dsub_rn(f[l], feq[l])));
    return 0u;
}

template <int NQ>
__device__ __forceinline__ unsigned gen_bc(double (&f)[NQ], double Tw, int order) {
    double rho = 0.0;
#pragma unroll
    for (int l = 0; l < NQ; ++l) rho = __dadd_rn(rho, f[l]);
    gen_equilibrium<NQ>(rho, 0.0, 0.0, Tw, order, f);
    return rho > 0.0 ? 0u : 4u;
}

template <int NQ>
__device__ __forceinline__ void gen_count_neg(TlbStatus *st, const double (&f)[NQ], bool active) {
    unsigned n = 0;
    if (active) {
#pragma unroll
        for (int l = 0; l < NQ; ++l) n += f[l] < 0.0;
    }
    count_neg_n(st, n);
}

template <int KIND, int NQ, bool INPLACE, bool EDGE>
__device__ __forceinline__ void gen_body(const SiteLaunch &L, int x, int y, bool active) {
    double f[NQ];
    const bool gather = KIND == K_PROPAGATE || KIND == K_FUSED;
    const Fld &s = L.src;
    if (!EDGE && !INPLACE) {
        // interior: the launch's precomputed (shifted) byte offsets, no remapping
        const char *sp = reinterpret_cast<const char *>(s.base + (long long)x * s.sx +
                                                        (long long)y * s.sy);
#pragma unroll
        for (int l = 0; l < NQ; ++l)
            f[l] = __ldg(reinterpret_cast<const double *>(sp + L.soffb[l]));
    } else {
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
            int xs = x, ys = y;
            if (gather && !INPLACE) {
                xs = src_x(x, G.cx[l], s, L.flags);
                ys = src_y(y, G.cy[l], s, L.flags);
            }
            const double *p = s.base + (long long)l * s.sl + (long long)xs * s.sx +
                              (long long)ys * s.sy;
            f[l] = INPLACE ? *p : __ldg(p);
        }
    }
    unsigned bits = 0;
    if (KIND == K_BC || KIND == K_FUSED) {
        const bool bot = y >= L.bot_lo && y < L.bot_hi;
        const bool top = y >= L.top_lo && y < L.top_hi;
        if (bot) bits |= gen_bc<NQ>(f, L.P.Tbot, L.P.order);  // bottom, then top
        if (top) bits |= gen_bc<NQ>(f, L.P.Ttop, L.P.order);  // (kernels.py:190-203)
    }
    if (KIND == K_COLLIDE || KIND == K_FUSED) bits |= gen_collide<NQ>(f, L.P);
    if (active) {
        report(L.status, bits, x, y, L.step);
        double *d = L.dst.base + (long long)x * L.dst.sx + (long long)y * L.dst.sy;
#pragma unroll
        for (int l = 0; l < NQ; ++l) d[(long long)l * L.dst.sl] = f[l];
    }
    if (L.flags & TLB_F_COUNT_NEG) gen_count_neg<NQ>(L.status, f, active);
}

// same rectangle bookkeeping as k_site (frames first, then the interior)
template <int KIND, int NQ, bool INPLACE>
__global__ void __launch_bounds__(128) k_gen_site(const __grid_constant__ SiteLaunch L) {
    if (blockIdx.x < L.nfb) {
        const unsigned total = L.fr_end[3];
        const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
        const bool active = i < total;
        const unsigned ii = active ? i : total - 1;
        const int r = ii < L.fr_end[0] ? 0 : ii < L.fr_end[1] ? 1 : ii < L.fr_end[2] ? 2 : 3;
        const unsigned loc = ii - (r ? L.fr_end[r - 1] : 0u);
        const Rect &R = L.fr[r];
        gen_body<KIND, NQ, INPLACE, true>(L, R.x0 + (int)(loc / R.ny), R.y0 + (int)(loc % R.ny),
                                          active);
    } else {
        const unsigned i = (blockIdx.x - L.nfb) * blockDim.x + threadIdx.x;
        const bool active = i < L.in.n;
        const unsigned ii = active ? i : L.in.n - 1;
        gen_body<KIND, NQ, INPLACE, false>(L, L.in.x0 + (int)(ii / L.in.ny),
                                           L.in.y0 + (int)(ii % L.in.ny), active);
    }
}

template <int KIND, bool INPLACE>
static int launch_gen(SiteLaunch &L, int Q, cudaStream_t s, const char *what) {
    const GenHost &gh = gen_host();
    constexpr bool gather = KIND == K_PROPAGATE || KIND == K_FUSED;
    for (int l = 0; l < Q; ++l) {   // interior gather offsets, as launch_site does for D2Q37
        long long so = (long long)l * L.src.sl;
        if (gather) so -= (long long)gh.cx[l] * L.src.sx + (long long)gh.cy[l] * L.src.sy;
        L.soffb[l] = 8 * so;
        L.doffb[l] = 8 * (long long)l * L.dst.sl;
    }
    const unsigned long long nf = L.fr_end[3];
    L.nfb = (unsigned)((nf + 127) / 128);
    const unsigned long long nb = L.nfb + (L.in.n + 127ULL) / 128;
    if (nb == 0) return TLB_OK;
    if (Q == 9)
        k_gen_site<KIND, 9, INPLACE><<<(unsigned)nb, 128, 0, s>>>(L);
    else if (Q == 37)
        k_gen_site<KIND, 37, INPLACE><<<(unsigned)nb, 128, 0, s>>>(L);
    else
        return fail(TLB_ERR_UNSUPPORTED, "%s: generic kernels are built for Q = 9 and 37", what);
    return launch_check(what);
}

template <int NQ>
__global__ void k_gen_moments(Fld f, int x0, int y0, int ny, long long n, double *rho,
                              double *ux, double *uy, double *T, long long ld, int check,
                              TlbStatus *st) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int xi = (int)(i / ny), yi = (int)(i % ny);
    double fl[NQ];
    const double *p = f.base + (long long)(x0 + xi) * f.sx + (long long)(y0 + yi) * f.sy;
#pragma unroll
    for (int l = 0; l < NQ; ++l) fl[l] = p[(long long)l * f.sl];
    double r, u, v, t;
    gen_moments<NQ>(fl, r, u, v, t);
    const long long o = (long long)xi * ld + yi;
    rho[o] = r; ux[o] = u; uy[o] = v; T[o] = t;
    if (check && !(r > 0.0)) report(st, 1u, x0 + xi, y0 + yi, -1);
}

template <int NQ>
__global__ void k_gen_equilibrium(const double *rho, const double *ux, const double *uy,
                                  const double *T, long long n, int order, double *out,
                                  long long ld, int check, TlbStatus *st) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double r = rho[i], t = T[i];
    if (check && (!(r > 0.0) || !(t > 0.0))) report(st, 4u, (int)i, 0, -1);
    double f[NQ];
    gen_equilibrium<NQ>(r, ux[i], uy[i], t, order, f);
#pragma unroll
    for (int l = 0; l < NQ; ++l) out[(long long)l * ld + i] = f[l];
}

template <int NQ>
__global__ void k_gen_count_negative(Fld f, int x0, int y0, int ny, long long n, TlbStatus *st) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double fl[NQ];
    const bool active = i < n;
    if (active) {
        const int x = x0 + (int)(i / ny), y = y0 + (int)(i % ny);
        const double *p = f.base + (long long)x * f.sx + (long long)y * f.sy;
#pragma unroll
        for (int l = 0; l < NQ; ++l) fl[l] = p[(long long)l * f.sl];
    }
    gen_count_neg<NQ>(st, fl, active);
}

/*
 * tlb_oracle.c -- CPU restatement of the reference's D2Q37 time step.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1703_00185_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker or the
 * CPU baseline, never as the product path.
 *
 * Reference: /root/reference/pkg/src/thermolb (pure Python/numpy, v0.1.0).
 * Every function cites the reference file:line it restates.  The arithmetic is
 * the reference's numpy element-wise expression tree evaluated left to right
 * (SURVEY.md Appendix B); compiled with -ffp-contract=off and without
 * -ffast-math each operation is one IEEE-754 binary64 operation, so the
 * results are bit-identical to the reference.  Parity is PINNED: the CPU test
 * suite (tests/test_oracle_golden.py) checks this file bit-for-bit against
 * fixtures produced by the real reference (tests/golden/make_golden.py) and
 * against the SURVEY §8c SHA-256 fingerprint of RT 256x128 after 100 steps.
 *
 * Storage is the reference's canonical SoA (Q, NX, NY) view: element
 * (l, x, y) lives at l*NX*NY + x*NY + y (geometry.py:68-74).
 */
#define _POSIX_C_SOURCE 199309L  /* clock_gettime (orc_run_timed) */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q 37
#define WALL_ROWS 3 /* kernels.py:18 */

typedef struct {
    int64_t cx[Q], cy[Q];
    double w[Q];
    double cs2, cs;   /* cs = sqrt(cs2)                  kernels.py:87 */
    double ex[Q], ey[Q], q[Q]; /* c/cs, |e|^2              kernels.py:95-97 */
} Stencil;

typedef struct {
    double tau, gx, gy, dt;
    double Twall_top, Twall_bot;
    int order;        /* Hermite truncation (2, 3, 4)      kernels.py:80-83 */
} Params;

static Stencil S;

/* Errors mirror errors.py: 1 = DegenerateStateError (rho<=0, kernels.py:62-66)
 * 2 = DomainError (T_bar<=0, kernels.py:134-135), 3 = DomainError in bc's
 * checked equilibrium (rho<=0 or T<=0, kernels.py:85-86), 4 = ContractViolation. */
static int g_err = 0;
static int64_t g_err_site = -1;

static void set_err(int code, int64_t site) {
#pragma omp critical(orc_err)
    {
        if (!g_err) { g_err = code; g_err_site = site; }
    }
}

int orc_last_error(int64_t *site) {
    if (site) *site = g_err_site;
    int e = g_err;
    g_err = 0;
    g_err_site = -1;
    return e;
}

/* The stencil is taken from the caller (velocity_set.py builds it with scipy;
 * the bits depend on LAPACK), and ex/ey/q are derived with the
 * exact expressions of kernels.py:87-97. */
int orc_set_stencil(const int64_t *c, const double *w, double cs2) {
    S.cs2 = cs2;
    S.cs = sqrt(cs2);
    for (int l = 0; l < Q; ++l) {
        S.cx[l] = c[2 * l];
        S.cy[l] = c[2 * l + 1];
        S.w[l] = w[l];
        S.ex[l] = (double)S.cx[l] / S.cs;
        S.ey[l] = (double)S.cy[l] / S.cs;
        S.q[l] = S.ex[l] * S.ex[l] + S.ey[l] * S.ey[l];
    }
    return 0;
}

/* moments, one site: kernels.py:41-71. f[l*ld]. */
static inline void moments_site(const double *f, int64_t ld, double *rho_o,
                                double *ux_o, double *uy_o, double *T_o) {
    double rho = 0.0, mx = 0.0, my = 0.0, e2 = 0.0;
    for (int l = 0; l < Q; ++l) {
        double fl = f[l * ld];
        double cx = (double)S.cx[l], cy = (double)S.cy[l];
        rho = rho + fl;
        if (cx != 0.0) mx = mx + cx * fl;
        if (cy != 0.0) my = my + cy * fl;
        double c2 = cx * cx + cy * cy;
        if (c2 != 0.0) e2 = e2 + c2 * fl;
    }
    double ux = mx / rho;
    double uy = my / rho;
    double T = (e2 - rho * (ux * ux + uy * uy)) / (2.0 * rho);
    *rho_o = rho; *ux_o = ux; *uy_o = uy; *T_o = T;
}

/* equilibrium, one site: kernels.py:74-125 (D = 2). out[l*ld]. */
static inline void equilibrium_site(double rho, double ux, double uy, double T,
                                    int order, double *out, int64_t ld) {
    const double D = 2.0;
    double cs = S.cs;
    double vx = ux / cs;
    double vy = uy / cs;
    double theta = T / S.cs2 - 1.0;
    double s = vx * vx + vy * vy;
    for (int l = 0; l < Q; ++l) {
        double ex = S.ex[l], ey = S.ey[l], q = S.q[l];
        double p = ex * vx + ey * vy;
        double poly = 1.0 + p;
        double c2 = p * p + theta * q - (s + D * theta);
        poly = poly + 0.5 * c2;
        if (order >= 3) {
            double c3 = p * p * p + 3.0 * theta * q * p
                        - 3.0 * p * (s + (D + 2.0) * theta);
            poly = poly + c3 / 6.0;
        }
        if (order >= 4) {
            double c4 = p * p * p * p
                        + 6.0 * theta * q * p * p
                        + 3.0 * theta * theta * q * q
                        - 6.0 * (s * p * p
                                 + theta * ((D + 4.0) * p * p + q * s)
                                 + theta * theta * (D + 2.0) * q)
                        + 3.0 * (s * s
                                 + (2.0 * D + 4.0) * theta * s
                                 + D * (D + 2.0) * theta * theta);
            poly = poly + c4 / 24.0;
        }
        out[l * ld] = S.w[l] * rho * poly;
    }
}

/* collide, one site: kernels.py:139-146 (moments -> apply_shift :128-136 ->
 * equilibrium -> BGK).  f and out may alias. */
static inline int collide_site(const double *f, int64_t ldf, double *out,
                               int64_t ldo, const Params *P) {
    double rho, ux, uy, T, fl[Q], feq[Q];
    for (int l = 0; l < Q; ++l) fl[l] = f[l * ldf];
    moments_site(fl, 1, &rho, &ux, &uy, &T);
    if (!(rho > 0.0)) return 1;
    double ub = ux + P->tau * P->gx;
    double vb = uy + P->tau * P->gy;
    double g2 = P->gx * P->gx + P->gy * P->gy;
    double Tb = T - P->tau * P->tau * g2 / 2.0; /* params.D == 2 */
    if (!(Tb > 0.0)) return 2;
    equilibrium_site(rho, ub, vb, Tb, P->order, feq, 1);
    double omega = P->dt / P->tau;
    for (int l = 0; l < Q; ++l) out[l * ldo] = fl[l] - omega * (fl[l] - feq[l]);
    return 0;
}

/* ---- block API on (Q, n) arrays with leading dimension ld ------------- */

int orc_moments(const double *f, int64_t n, int64_t ld, double *rho,
                double *ux, double *uy, double *T, int check) {
    g_err = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        moments_site(f + i, ld, rho + i, ux + i, uy + i, T + i);
        if (check && !(rho[i] > 0.0)) set_err(1, i);
    }
    return g_err;
}

int orc_equilibrium(const double *rho, const double *ux, const double *uy,
                    const double *T, int64_t n, int order, double *out,
                    int64_t ld, int check) {
    g_err = 0;
    if (order < 2 || order > 4) return 3;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (check && (!(rho[i] > 0.0) || !(T[i] > 0.0))) set_err(3, i);
        equilibrium_site(rho[i], ux[i], uy[i], T[i], order, out + i, ld);
    }
    return g_err;
}

int orc_collide(const double *f, double *out, int64_t n, int64_t ldf,
                int64_t ldo, const double *params6, int order) {
    Params P = {params6[0], params6[1], params6[2], params6[3], params6[4],
                params6[5], order};
    g_err = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int e = collide_site(f + i, ldf, out + i, ldo, &P);
        if (e) set_err(e, i);
    }
    return g_err;
}

/* ---- field API on canonical (Q, NX, NY) fields ----------------------- */

typedef struct { int64_t Lx, Ly, H, NX, NY; } Geom;

static inline Geom mkgeom(int64_t Lx, int64_t Ly, int64_t H) {
    Geom g = {Lx, Ly, H, Lx + 2 * H, Ly + 2 * H};
    return g;
}

/* propagate (pull): kernels.py:168-177 over region [x0,x1) x [y0,y1). */
int orc_propagate(const double *prv, double *nxt, int64_t Lx, int64_t Ly,
                  int64_t H, int64_t x0, int64_t x1, int64_t y0, int64_t y1) {
    Geom g = mkgeom(Lx, Ly, H);
    if (x0 < H || x1 > H + Lx || y0 < H || y1 > H + Ly) return 4;
    int64_t plane = g.NX * g.NY;
#pragma omp parallel for schedule(static)
    for (int64_t x = x0; x < x1; ++x)
        for (int l = 0; l < Q; ++l)
            for (int64_t y = y0; y < y1; ++y)
                nxt[l * plane + x * g.NY + y] =
                    prv[l * plane + (x - S.cx[l]) * g.NY + (y - S.cy[l])];
    return 0;
}

/* bc: kernels.py:180-203.  Rows [H, H+3) at Twall_bot, [H+Ly-3, H+Ly) at
 * Twall_top, columns [x0, x1). */
int orc_bc(double *f, int64_t Lx, int64_t Ly, int64_t H, int64_t x0,
           int64_t x1, int top, int bottom, const double *params6, int order) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    g_err = 0;
    if (!(params6[4] > 0.0) && top) return 3;
    if (!(params6[5] > 0.0) && bottom) return 3;
    for (int side = 0; side < 2; ++side) {
        if (side == 0 && !bottom) continue;
        if (side == 1 && !top) continue;
        int64_t ylo = side == 0 ? H : H + Ly - WALL_ROWS;
        double Tw = side == 0 ? params6[5] : params6[4];
#pragma omp parallel for schedule(static)
        for (int64_t x = x0; x < x1; ++x)
            for (int64_t y = ylo; y < ylo + WALL_ROWS; ++y) {
                double *site = f + x * g.NY + y;
                double rho = 0.0;
                for (int l = 0; l < Q; ++l) rho = rho + site[l * plane];
                if (!(rho > 0.0)) set_err(3, x * g.NY + y);
                equilibrium_site(rho, 0.0, 0.0, Tw, order, site, plane);
            }
    }
    return g_err;
}

/* collide over a field region in place (runtime.py:322-324). */
int orc_collide_region(double *f, int64_t Lx, int64_t Ly, int64_t H,
                       int64_t x0, int64_t x1, int64_t y0, int64_t y1,
                       const double *params6, int order) {
    Geom g = mkgeom(Lx, Ly, H);
    Params P = {params6[0], params6[1], params6[2], params6[3], params6[4],
                params6[5], order};
    int64_t plane = g.NX * g.NY;
    g_err = 0;
#pragma omp parallel for schedule(static)
    for (int64_t x = x0; x < x1; ++x)
        for (int64_t y = y0; y < y1; ++y) {
            double *site = f + x * g.NY + y;
            int e = collide_site(site, plane, site, plane, &P);
            if (e) set_err(e, x * g.NY + y);
        }
    return g_err;
}

/* propagate_collide_fused: kernels.py:206-224 (gather :159-165, collide). */
int orc_fused(const double *prv, double *nxt, int64_t Lx, int64_t Ly,
              int64_t H, int64_t x0, int64_t x1, int64_t y0, int64_t y1,
              const double *params6, int order) {
    Geom g = mkgeom(Lx, Ly, H);
    if (x0 < H || x1 > H + Lx || y0 < H || y1 > H + Ly) return 4;
    Params P = {params6[0], params6[1], params6[2], params6[3], params6[4],
                params6[5], order};
    int64_t plane = g.NX * g.NY;
    g_err = 0;
#pragma omp parallel for schedule(static)
    for (int64_t x = x0; x < x1; ++x)
        for (int64_t y = y0; y < y1; ++y) {
            double scratch[Q];
            for (int l = 0; l < Q; ++l)
                scratch[l] = prv[l * plane + (x - S.cx[l]) * g.NY + (y - S.cy[l])];
            int e = collide_site(scratch, 1, nxt + x * g.NY + y, plane, &P);
            if (e) set_err(e, x * g.NY + y);
        }
    return g_err;
}

/* _extend_wall_halos: runtime.py:296-305 (all x, all 37 pops). */
void orc_extend_walls(double *f, int64_t Lx, int64_t Ly, int64_t H,
                      int upper, int lower) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    for (int l = 0; l < Q; ++l)
        for (int64_t x = 0; x < g.NX; ++x) {
            double *col = f + l * plane + x * g.NY;
            if (upper)
                for (int64_t y = H + Ly; y < g.NY; ++y) col[y] = col[H + Ly - 1];
            if (lower)
                for (int64_t y = 0; y < H; ++y) col[y] = col[H];
        }
}

/* pbc_c with the rank as its own left and right neighbour (1-D ring, Np=1):
 * pack_x/unpack_x runtime.py:199-224, face plans :94-107, _x_col :193-197.
 * Only face-plan pops are written, full NY height. */
void orc_pbc_self(double *f, int64_t Lx, int64_t Ly, int64_t H) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    for (int sign = 1; sign >= -1; sign -= 2)
        for (int d = 1; d <= H; ++d)
            for (int l = 0; l < Q; ++l) {
                if (!(sign * S.cx[l] >= d)) continue;
                int64_t src = sign == 1 ? H + Lx - d : H + d - 1;
                int64_t dst = sign == 1 ? H - d : H + Lx - 1 + d;
                memcpy(f + l * plane + dst * g.NY, f + l * plane + src * g.NY,
                       sizeof(double) * g.NY);
            }
}

/* pbc_nc with the rank as its own up/down neighbour (periodic Y, Np = 1):
 * pack_y/unpack_y runtime.py:226-246 -- physical columns only. */
void orc_pbc_y_self(double *f, int64_t Lx, int64_t Ly, int64_t H) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    for (int sign = 1; sign >= -1; sign -= 2)
        for (int e = 1; e <= H; ++e)
            for (int l = 0; l < Q; ++l) {
                if (!(sign * S.cy[l] >= e)) continue;
                int64_t src = sign == 1 ? H + Ly - e : H + e - 1;
                int64_t dst = sign == 1 ? H - e : H + Ly - 1 + e;
                for (int64_t x = H; x < H + Lx; ++x)
                    f[l * plane + x * g.NY + dst] = f[l * plane + x * g.NY + src];
            }
}

int64_t orc_count_negative(const double *f, int64_t Lx, int64_t Ly, int64_t H) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY, n = 0;
#pragma omp parallel for reduction(+ : n) schedule(static)
    for (int64_t x = H; x < H + Lx; ++x)
        for (int l = 0; l < Q; ++l)
            for (int64_t y = H; y < H + Ly; ++y)
                n += f[l * plane + x * g.NY + y] < 0.0;
    return n;
}

/* One staged time step of a rank that is its own ring neighbour (Np = 1):
 * RankWorker.step runtime.py:355-400 with schedule "staged"
 * (_extend_wall_halos :296-305, pbc_nc :264-267 when periodic in Y,
 * pbc_c :281-284, _staged_compute :316-324).
 * ymode: 1 = walls (1-D tiling default), 2 = periodic Y, 0 = neither. */
int orc_step(double *prv, double *nxt, int64_t Lx, int64_t Ly, int64_t H,
             int ymode, const double *params6, int order, int64_t *negatives) {
    int walls = ymode == 1;
    if (walls) orc_extend_walls(prv, Lx, Ly, H, 1, 1);
    if (ymode == 2) orc_pbc_y_self(prv, Lx, Ly, H);
    orc_pbc_self(prv, Lx, Ly, H);
    orc_propagate(prv, nxt, Lx, Ly, H, H, H + Lx, H, H + Ly);
    int e = 0;
    if (walls) e = orc_bc(nxt, Lx, Ly, H, H, H + Lx, 1, 1, params6, order);
    if (e) return e;
    e = orc_collide_region(nxt, Lx, Ly, H, H, H + Lx, H, H + Ly, params6, order);
    if (negatives) *negatives = orc_count_negative(nxt, Lx, Ly, H);
    return e;
}

/* run(): sim.py:62-129 restricted to Np = 1, 1-D tiling (periodic X, walls in
 * Y).  f_in/f_out are the (Q, Lx, Ly) physical blocks. */
int orc_run(const double *f_in, double *f_out, int64_t Lx, int64_t Ly,
            int64_t H, int64_t steps, int ymode, const double *params6,
            int order, int64_t *negatives) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    double *a = calloc((size_t)Q * plane, sizeof(double));
    double *b = calloc((size_t)Q * plane, sizeof(double));
    if (!a || !b) { free(a); free(b); return 5; }
    for (int l = 0; l < Q; ++l)
        for (int64_t x = 0; x < Lx; ++x)
            memcpy(a + l * plane + (x + H) * g.NY + H, f_in + (l * Lx + x) * Ly,
                   sizeof(double) * Ly);
    int e = 0;
    for (int64_t s = 0; s < steps && !e; ++s) {
        e = orc_step(a, b, Lx, Ly, H, ymode, params6, order,
                     negatives ? negatives + s : NULL);
        double *t = a; a = b; b = t;
    }
    for (int l = 0; l < Q; ++l)
        for (int64_t x = 0; x < Lx; ++x)
            memcpy(f_out + (l * Lx + x) * Ly, a + l * plane + (x + H) * g.NY + H,
                   sizeof(double) * Ly);
    free(a);
    free(b);
    return e;
}

/* Benchmark leg of bench.py (cpu_baseline / --impl reference): orc_run with
 * `warmup` untimed steps first (OpenMP pool started, both buffers faulted
 * in), then `steps` steps timed with CLOCK_MONOTONIC. */
int orc_run_timed(const double *f_in, double *f_out, int64_t Lx, int64_t Ly,
                  int64_t H, int64_t warmup, int64_t steps, int ymode,
                  const double *params6, int order, double *seconds) {
    Geom g = mkgeom(Lx, Ly, H);
    int64_t plane = g.NX * g.NY;
    double *a = calloc((size_t)Q * plane, sizeof(double));
    double *b = calloc((size_t)Q * plane, sizeof(double));
    if (!a || !b) { free(a); free(b); return 5; }
    for (int l = 0; l < Q; ++l)
        for (int64_t x = 0; x < Lx; ++x)
            memcpy(a + l * plane + (x + H) * g.NY + H, f_in + (l * Lx + x) * Ly,
                   sizeof(double) * Ly);
    int e = 0;
    for (int64_t s = 0; s < warmup && !e; ++s) {
        e = orc_step(a, b, Lx, Ly, H, ymode, params6, order, NULL);
        double *t = a; a = b; b = t;
    }
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int64_t s = 0; s < steps && !e; ++s) {
        e = orc_step(a, b, Lx, Ly, H, ymode, params6, order, NULL);
        double *t = a; a = b; b = t;
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    *seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    for (int l = 0; l < Q; ++l)
        for (int64_t x = 0; x < Lx; ++x)
            memcpy(f_out + (l * Lx + x) * Ly, a + l * plane + (x + H) * g.NY + H,
                   sizeof(double) * Ly);
    free(a);
    free(b);
    return e;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

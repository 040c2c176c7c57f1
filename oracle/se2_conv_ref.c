/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Plain fp64 loops; shares no code with
 * the CUDA path (paper_2402_15322_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library.
 *
 * Discrete SE(2) group convolution, PAPER.md subsec:gconv:
 *     (K b)(g) = sum_h K(h^{-1} g) b(h)
 * on the lattice of DESIGN.md (cell centres, theta_k = 2 pi k / nt), with the
 * kernel restricted to the spatial box |ix_g - ix_h| <= R, |iy_g - iy_h| <= R
 * (all theta offsets) and zero padding outside the window.
 *
 * Table layout (the oracle's own): T[(((to * nt) + ti) * S + (dy + R)) * S + (dx + R)]
 * holds K(h^{-1} g) for g = (x_h + (dx/nx, dy/ny), theta_to), h = (x_h, theta_ti),
 * i.e. dx = ix_g - ix_h, dy = iy_g - iy_h.  Field layout [theta][y][x].
 */
#include <math.h>
#include <stddef.h>
#include <stdlib.h>

/* exp(x) is exactly +0 in IEEE double for x < -745.14 (below half the smallest subnormal), so a
 * log-sum-exp term with exponent <= EXP_ZERO adds exactly nothing and is not evaluated. */
#define EXP_ZERO (-746.0)

#define IDX3(t, y, x) (((size_t)(t) * ny + (y)) * nx + (x))

static inline size_t tidx(int nt, int S, int R, int to, int ti, int dy, int dx) {
    return ((((size_t)to * nt + ti) * S + (dy + R)) * S + (dx + R));
}

/* Loop order.  Every output's sum is accumulated in the order the definition states -- theta_i,
 * then dy, then dx ascending -- exactly as in oracle_conv_point / oracle_lse_point below (the
 * one-output definitions).  The full-field loops only move the x loop innermost, so one row of
 * independent outputs is updated per (theta_i, dy, dx): same additions, same order per output,
 * bit-identical results (tests/test_oracle_pins.py checks that), and the x loop vectorises without
 * reassociating any sum (no -ffast-math; contraction off). */

/* y(g) = sum_h K(g,h) v(h)   -- gather form of K (first formula) */
void oracle_conv_gather(int nx, int ny, int nt, int R, const double* T, const double* v, double* y) {
    const int S = 2 * R + 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (int to = 0; to < nt; ++to)
        for (int iy = 0; iy < ny; ++iy) {
            double* acc = y + IDX3(to, iy, 0);
            for (int ix = 0; ix < nx; ++ix) acc[ix] = 0.0;
            for (int ti = 0; ti < nt; ++ti)
                for (int dy = -R; dy <= R; ++dy) {
                    const int hy = iy - dy;
                    if (hy < 0 || hy >= ny) continue;
                    const double* vrow = v + IDX3(ti, hy, 0);
                    for (int dx = -R; dx <= R; ++dx) {
                        const double t = T[tidx(nt, S, R, to, ti, dy, dx)];
                        /* outputs ix with hx = ix - dx inside [0, nx) */
                        const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                        for (int ix = lo; ix < hi; ++ix) acc[ix] += t * vrow[ix - dx];
                    }
                }
        }
}

/* y(h) = sum_g K(g,h) a(g)   -- the adjoint K^T (second formula), written as a
 * SCATTER over g so that K = K^T is tested, not assumed.  Threads own output
 * channels th, so there is no write race.  Per output y(h) the contributions arrive in the order
 * theta_g, then g_y (i.e. dy), then g_x (dx) ascending. */
void oracle_conv_scatter_adjoint(int nx, int ny, int nt, int R, const double* T, const double* a,
                                 double* y) {
    const int S = 2 * R + 1;
    const size_t n = (size_t)nx * ny * nt;
    for (size_t i = 0; i < n; ++i) y[i] = 0.0;
#pragma omp parallel for schedule(static)
    for (int th = 0; th < nt; ++th)
        for (int tg = 0; tg < nt; ++tg)
            for (int gy = 0; gy < ny; ++gy) {
                const double* arow = a + IDX3(tg, gy, 0);
                for (int dy = -R; dy <= R; ++dy) {
                    const int hy = gy - dy;
                    if (hy < 0 || hy >= ny) continue;
                    double* yrow = y + IDX3(th, hy, 0);
                    for (int dx = -R; dx <= R; ++dx) {
                        const double t = T[tidx(nt, S, R, tg, th, dy, dx)];
                        /* sources gx with hx = gx - dx inside [0, nx) */
                        const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                        for (int gx = lo; gx < hi; ++gx) yrow[gx - dx] += t * arow[gx];
                    }
                }
            }
}

/* log-domain gather: ly(g) = log sum_h exp(L(g,h) + lv(h)), exact two-pass LSE
 * (max, then sum of exp(. - max)).  All-(-inf) inputs give -inf.  m: scratch row of nx. */
void oracle_lse_gather(int nx, int ny, int nt, int R, const double* L, const double* lv, double* ly) {
    const int S = 2 * R + 1;
#pragma omp parallel
    {
        double* m = (double*)malloc(sizeof(double) * (size_t)nx);
#pragma omp for collapse(2) schedule(static)
        for (int to = 0; to < nt; ++to)
            for (int iy = 0; iy < ny; ++iy) {
                double* s = ly + IDX3(to, iy, 0);
                for (int ix = 0; ix < nx; ++ix) { m[ix] = -INFINITY; s[ix] = 0.0; }
                for (int ti = 0; ti < nt; ++ti)
                    for (int dy = -R; dy <= R; ++dy) {
                        const int hy = iy - dy;
                        if (hy < 0 || hy >= ny) continue;
                        const double* vrow = lv + IDX3(ti, hy, 0);
                        for (int dx = -R; dx <= R; ++dx) {
                            const double l = L[tidx(nt, S, R, to, ti, dy, dx)];
                            const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                            for (int ix = lo; ix < hi; ++ix) {
                                const double t = l + vrow[ix - dx];
                                if (t > m[ix]) m[ix] = t;
                            }
                        }
                    }
                for (int ti = 0; ti < nt; ++ti)
                    for (int dy = -R; dy <= R; ++dy) {
                        const int hy = iy - dy;
                        if (hy < 0 || hy >= ny) continue;
                        const double* vrow = lv + IDX3(ti, hy, 0);
                        for (int dx = -R; dx <= R; ++dx) {
                            const double l = L[tidx(nt, S, R, to, ti, dy, dx)];
                            const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                            for (int ix = lo; ix < hi; ++ix) {
                                if (m[ix] == -INFINITY) continue;
                                const double e = l + vrow[ix - dx] - m[ix];
                                if (e > EXP_ZERO) s[ix] += exp(e);
                            }
                        }
                    }
                for (int ix = 0; ix < nx; ++ix) s[ix] = (m[ix] == -INFINITY) ? -INFINITY : m[ix] + log(s[ix]);
            }
        free(m);
    }
}

/* log-domain adjoint as a scatter (max pass, then sum pass). */
void oracle_lse_scatter_adjoint(int nx, int ny, int nt, int R, const double* L, const double* la,
                                double* ly, double* scratch_max) {
    const int S = 2 * R + 1;
    const size_t n = (size_t)nx * ny * nt;
    for (size_t i = 0; i < n; ++i) { scratch_max[i] = -INFINITY; ly[i] = 0.0; }
#pragma omp parallel for schedule(static)
    for (int th = 0; th < nt; ++th)
        for (int tg = 0; tg < nt; ++tg)
            for (int gy = 0; gy < ny; ++gy) {
                const double* arow = la + IDX3(tg, gy, 0);
                for (int dy = -R; dy <= R; ++dy) {
                    const int hy = gy - dy;
                    if (hy < 0 || hy >= ny) continue;
                    double* mrow = scratch_max + IDX3(th, hy, 0);
                    for (int dx = -R; dx <= R; ++dx) {
                        const double l = L[tidx(nt, S, R, tg, th, dy, dx)];
                        const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                        for (int gx = lo; gx < hi; ++gx) {
                            const double t = l + arow[gx];
                            if (t > mrow[gx - dx]) mrow[gx - dx] = t;
                        }
                    }
                }
            }
#pragma omp parallel for schedule(static)
    for (int th = 0; th < nt; ++th)
        for (int tg = 0; tg < nt; ++tg)
            for (int gy = 0; gy < ny; ++gy) {
                const double* arow = la + IDX3(tg, gy, 0);
                for (int dy = -R; dy <= R; ++dy) {
                    const int hy = gy - dy;
                    if (hy < 0 || hy >= ny) continue;
                    const double* mrow = scratch_max + IDX3(th, hy, 0);
                    double* yrow = ly + IDX3(th, hy, 0);
                    for (int dx = -R; dx <= R; ++dx) {
                        const double l = L[tidx(nt, S, R, tg, th, dy, dx)];
                        const int lo = dx > 0 ? dx : 0, hi = dx > 0 ? nx : nx + dx;
                        for (int gx = lo; gx < hi; ++gx) {
                            const double m = mrow[gx - dx];
                            if (m == -INFINITY) continue;
                            const double e = l + arow[gx] - m;
                            if (e > EXP_ZERO) yrow[gx - dx] += exp(e);
                        }
                    }
                }
            }
    for (size_t i = 0; i < n; ++i)
        ly[i] = (scratch_max[i] == -INFINITY) ? -INFINITY : scratch_max[i] + log(ly[i]);
}

/* Single output sample of the gather conv (for full-size sampled parity). */
double oracle_conv_point(int nx, int ny, int nt, int R, const double* T, const double* v,
                         int to, int iy, int ix) {
    const int S = 2 * R + 1;
    double acc = 0.0;
    for (int ti = 0; ti < nt; ++ti)
        for (int dy = -R; dy <= R; ++dy) {
            int hy = iy - dy;
            if (hy < 0 || hy >= ny) continue;
            for (int dx = -R; dx <= R; ++dx) {
                int hx = ix - dx;
                if (hx < 0 || hx >= nx) continue;
                acc += T[tidx(nt, S, R, to, ti, dy, dx)] * v[IDX3(ti, hy, hx)];
            }
        }
    return acc;
}

double oracle_lse_point(int nx, int ny, int nt, int R, const double* L, const double* lv,
                        int to, int iy, int ix) {
    const int S = 2 * R + 1;
    double m = -INFINITY;
    for (int ti = 0; ti < nt; ++ti)
        for (int dy = -R; dy <= R; ++dy) {
            int hy = iy - dy;
            if (hy < 0 || hy >= ny) continue;
            for (int dx = -R; dx <= R; ++dx) {
                int hx = ix - dx;
                if (hx < 0 || hx >= nx) continue;
                double t = L[tidx(nt, S, R, to, ti, dy, dx)] + lv[IDX3(ti, hy, hx)];
                if (t > m) m = t;
            }
        }
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int ti = 0; ti < nt; ++ti)
        for (int dy = -R; dy <= R; ++dy) {
            int hy = iy - dy;
            if (hy < 0 || hy >= ny) continue;
            for (int dx = -R; dx <= R; ++dx) {
                int hx = ix - dx;
                if (hx < 0 || hx >= nx) continue;
                const double e = L[tidx(nt, S, R, to, ti, dy, dx)] + lv[IDX3(ti, hy, hx)] - m;
                if (e > EXP_ZERO) s += exp(e);
            }
        }
    return m + log(s);
}

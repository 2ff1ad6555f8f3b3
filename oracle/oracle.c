/*
 * oracle.c -- plain CPU oracle for the D3Q19 BGK lattice Boltzmann update of
 * Fu & Song, "Designing a 3D Parallel Memory-Aware Lattice Boltzmann
 * Algorithm on Manycore Systems" (arXiv 2208.05429).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Nothing on the product path
 * may load, call or link this file.
 *
 * What it computes.  The paper's Fuse Swap LBM (Alg. 1, PAPER.md:275-294,
 * section "Baseline 3D LBM Algorithm") and its two-step merge (Alg. 2,
 * PAPER.md:140-216, section "Sequential 3D Memory-aware LBM") both reach,
 * exactly, the plain two-lattice collide-then-stream result; they only
 * reorder the work ("loop fusion", "swap", "merging two collision-streaming
 * cycles").  So this oracle is that plain definition written
 * out, SURVEY.md section 8(c):
 *
 *   1. for every cell: rho = sum f_i, j = sum c_i f_i, u = j / rho,
 *      feq_i = w_i rho (1 + 3 c_i.u + 4.5 (c_i.u)^2 - 1.5 u.u) (i >= 1),
 *      feq_0 = rho - sum_{i>=1} feq_i,
 *      f*_i = f_i - omega (f_i - feq_i), omega = 1 / tau;
 *   2. for every cell x and direction i, with s = x - c_i:
 *      periodic:          f_i(x, t+1) = f*_i(s mod n)
 *      cavity, s inside:  f_i(x, t+1) = f*_i(s)
 *      cavity, s outside: f_i(x, t+1) = f*_opp(i)(x)
 *                                       + [s_z >= nz] 6 w_i rho_w (c_i.u_lid)
 *      (link-wise bounce-back, R-4; moving lid at the top z face,
 *      R-5/R-6, rho_w = 1).
 *
 * Collision model: BGK (the paper delegates dynamics to Palabos,
 * PAPER.md:831; BASELINE.json configs fix BGK with tau).  Equilibrium:
 * SPEC.md:75 with the rest-population closure of DESIGN.md R-2.
 * Direction order: SPEC.md:109 (the paper's "1 ~ 9" half set).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* SPEC.md:109 direction table: 1..9 lexicographically negative on (X,Y,Z),
 * i+9 is the opposite of i. */
static const int C[19][3] = {
    {0, 0, 0},
    {-1, 0, 0}, {0, -1, 0}, {0, 0, -1}, {-1, -1, 0}, {-1, 1, 0},
    {-1, 0, -1}, {-1, 0, 1}, {0, -1, -1}, {0, -1, 1},
    {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {1, 1, 0}, {1, -1, 0},
    {1, 0, 1}, {1, 0, -1}, {0, 1, 1}, {0, 1, -1}};

static double W[19];
static int OPP[19];
static int tables_ready = 0;
static int n_threads = 0;

static void init_tables(void) {
    if (tables_ready) return;
    for (int i = 0; i < 19; i++) {
        int len2 = C[i][0] * C[i][0] + C[i][1] * C[i][1] + C[i][2] * C[i][2];
        W[i] = (len2 == 0) ? 1.0 / 3.0 : (len2 == 1 ? 1.0 / 18.0 : 1.0 / 36.0);
        OPP[i] = (i == 0) ? 0 : (i <= 9 ? i + 9 : i - 9);
    }
    tables_ready = 1;
}

void oracle_d3q19(int c[19][3], double w[19], int opp[19]) {
    init_tables();
    for (int i = 0; i < 19; i++) {
        for (int a = 0; a < 3; a++) c[i][a] = C[i][a];
        w[i] = W[i];
        opp[i] = OPP[i];
    }
}

void oracle_set_threads(int n) { n_threads = n; }

int oracle_get_threads(void) {
#ifdef _OPENMP
    return n_threads > 0 ? n_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

int oracle_moments(const double f[19], double *rho, double u[3]) {
    double r = 0.0, j[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 19; i++) {
        r += f[i];
        for (int a = 0; a < 3; a++) j[a] += C[i][a] * f[i];
    }
    *rho = r;
    if (r == 0.0) {
        u[0] = u[1] = u[2] = 0.0;
        return 1;
    }
    for (int a = 0; a < 3; a++) u[a] = j[a] / r;
    return 0;
}

void oracle_equilibrium(double rho, const double u[3], double feq[19]) {
    init_tables();
    double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double rest = rho;
    for (int i = 1; i < 19; i++) {
        double cu = C[i][0] * u[0] + C[i][1] * u[1] + C[i][2] * u[2];
        feq[i] = W[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        rest -= feq[i];
    }
    feq[0] = rest;
}

int oracle_collide(const double f[19], double omega, double out[19]) {
    double rho, u[3], feq[19];
    int err = oracle_moments(f, &rho, u);
    oracle_equilibrium(rho, u, feq);
    for (int i = 0; i < 19; i++) out[i] = f[i] - omega * (f[i] - feq[i]);
    return err;
}

static size_t idx(int i, int x, int y, int z, int nx, int ny, int nz) {
    return (((size_t)i * nx + x) * ny + y) * nz + z;
}

void oracle_init_equilibrium(int nx, int ny, int nz, const double *rho,
                             const double *u, double *f) {
    init_tables();
    for (int x = 0; x < nx; x++)
        for (int y = 0; y < ny; y++)
            for (int z = 0; z < nz; z++) {
                size_t cell = ((size_t)x * ny + y) * nz + z;
                double r = rho ? rho[cell] : 1.0;
                double uu[3] = {0.0, 0.0, 0.0};
                if (u)
                    for (int a = 0; a < 3; a++) uu[a] = u[3 * cell + a];
                double feq[19];
                oracle_equilibrium(r, uu, feq);
                for (int i = 0; i < 19; i++) f[idx(i, x, y, z, nx, ny, nz)] = feq[i];
            }
}

static int wrap(int s, int n) { return ((s % n) + n) % n; }

/* Step part 1: BGK-collide every cell of an
 * lx*ly*lz array, f_in -> fstar.  f_in == fstar is allowed: each cell reads
 * its 19 values before writing them. */
static void collide_all(int lx, int ly, int lz, double omega,
                        const double *f_in, double *fstar) {
#pragma omp parallel for schedule(static) num_threads(oracle_get_threads())
    for (int x = 0; x < lx; x++)
        for (int y = 0; y < ly; y++)
            for (int z = 0; z < lz; z++) {
                double f[19], out[19];
                for (int i = 0; i < 19; i++) f[i] = f_in[idx(i, x, y, z, lx, ly, lz)];
                oracle_collide(f, omega, out);
                for (int i = 0; i < 19; i++) fstar[idx(i, x, y, z, lx, ly, lz)] = out[i];
            }
}

/* Step part 2: pull-stream the post-collision box
 * fstar into f_out with the boundary rules of the global domain. */
static void stream_all(int nx, int ny, int nz, int bc, const double u_lid[3],
                       int bx, int by, int bz, int lx, int ly, int lz,
                       const double *fstar, double *f_out) {
    const double rho_w = 1.0;
#pragma omp parallel for schedule(static) num_threads(oracle_get_threads())
    for (int x = 0; x < lx; x++)
        for (int y = 0; y < ly; y++)
            for (int z = 0; z < lz; z++) {
                int gx = bx + x, gy = by + y, gz = bz + z;
                for (int i = 0; i < 19; i++) {
                    int sx = gx - C[i][0], sy = gy - C[i][1], sz = gz - C[i][2];
                    int inside = sx >= 0 && sx < nx && sy >= 0 && sy < ny && sz >= 0 && sz < nz;
                    double v;
                    if (bc == ORACLE_BC_PERIODIC || inside) {
                        if (bc == ORACLE_BC_PERIODIC) {
                            sx = wrap(sx, nx);
                            sy = wrap(sy, ny);
                            sz = wrap(sz, nz);
                        }
                        int lxs = sx - bx, lys = sy - by, lzs = sz - bz;
                        if (lxs >= 0 && lxs < lx && lys >= 0 && lys < ly && lzs >= 0 && lzs < lz)
                            v = fstar[idx(i, lxs, lys, lzs, lx, ly, lz)];
                        else
                            v = NAN; /* source outside the box: unknown */
                    } else {
                        v = fstar[idx(OPP[i], x, y, z, lx, ly, lz)];
                        if (sz >= nz) {
                            double cu = C[i][0] * u_lid[0] + C[i][1] * u_lid[1] + C[i][2] * u_lid[2];
                            v = v + 6.0 * W[i] * rho_w * cu;
                        }
                    }
                    f_out[idx(i, x, y, z, lx, ly, lz)] = v;
                }
            }
}

void oracle_step_box(int nx, int ny, int nz, int bc, double tau,
                     const double u_lid[3], int bx, int by, int bz,
                     int lx, int ly, int lz, const double *f_in, double *f_out) {
    init_tables();
    size_t ncell = (size_t)lx * ly * lz;
    double *fstar = (double *)malloc(sizeof(double) * 19 * ncell);
    collide_all(lx, ly, lz, 1.0 / tau, f_in, fstar);
    stream_all(nx, ny, nz, bc, u_lid, bx, by, bz, lx, ly, lz, fstar, f_out);
    free(fstar);
}

void oracle_step(int nx, int ny, int nz, int bc, double tau,
                 const double u_lid[3], const double *f_in, double *f_out) {
    oracle_step_box(nx, ny, nz, bc, tau, u_lid, 0, 0, 0, nx, ny, nz, f_in, f_out);
}

/* The same two parts per step with two lattices only (collide in place,
 * pull into the other lattice, swap), so a full-size run holds 2 copies. */
int oracle_run(int nx, int ny, int nz, int bc, double tau,
               const double u_lid[3], long n, double *f) {
    init_tables();
    size_t len = (size_t)19 * nx * ny * nz;
    if (n <= 0) return 0;
    double *g = (double *)malloc(sizeof(double) * len);
    if (!g) return 1;
    double *a = f, *b = g;
    for (long t = 0; t < n; t++) {
        collide_all(nx, ny, nz, 1.0 / tau, a, a);
        stream_all(nx, ny, nz, bc, u_lid, 0, 0, 0, nx, ny, nz, a, b);
        double *tmp = a;
        a = b;
        b = tmp;
    }
    if (a != f) memcpy(f, a, sizeof(double) * len);
    free(g);
    return 0;
}

void oracle_macroscopic(int nx, int ny, int nz, const double *f, double *rho,
                        double *u) {
    for (int x = 0; x < nx; x++)
        for (int y = 0; y < ny; y++)
            for (int z = 0; z < nz; z++) {
                size_t cell = ((size_t)x * ny + y) * nz + z;
                double g[19], uu[3];
                for (int i = 0; i < 19; i++) g[i] = f[idx(i, x, y, z, nx, ny, nz)];
                oracle_moments(g, &rho[cell], uu);
                for (int a = 0; a < 3; a++) u[3 * cell + a] = uu[a];
            }
}

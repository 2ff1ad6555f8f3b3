/*
 * oracle_dqq.c -- plain CPU oracle for the other cubic lattices the paper
 * names: "no matter using D3Q15, D3Q19, D3Q27 or extended lattice models"
 * (Alg. 2 discussion).  SURVEY.md 8(f) row 4.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): only tests/ and bench.py's CPU
 * legs may load it; it shares no code with the CUDA path.
 *
 * The same definition as oracle.c, written for a velocity
 * set given as a table: BGK with the second-order equilibrium and the
 * rest-population closure, then pull-streaming with link-wise bounce-back,
 * the moving lid on the top z face and periodic wrap.  With the D3Q19 table
 * it performs, operation for operation, the arithmetic of oracle.c (pinned:
 * tests/test_oracle_pins.py checks bit equality), so this file's stepping is
 * pinned to the D3Q19 oracle and only the tables of D3Q15 / D3Q27 are new
 * (pinned by their rational isotropy and the physics pins).
 *
 * Velocity order: i = 0 rest; i = 1 .. h the "negative" half (first nonzero
 * component -1): axes (x, y, z), then face diagonals (xy-, xy+, xz-, xz+,
 * yz-, yz+), then corners ((-1,-1,-1), (-1,-1,1), (-1,1,-1), (-1,1,1)) as
 * far as the lattice has them; i = h+1 .. 2h the opposites, c_{i+h} =
 * -c_i.  For Q = 19 this is SPEC.md:109's order.  Weights by |c|^2:
 * D3Q15 2/9, 1/9, -, 1/72; D3Q19 1/3, 1/18, 1/36, -; D3Q27 8/27, 2/27,
 * 1/54, 1/216 (rest, axis, face diagonal, corner).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle.h"

#define QMAX 27

typedef struct {
    int q, h;
    int c[QMAX][3];
    double w[QMAX];
    int opp[QMAX];
} lattice;

static const int AXIS[3][3] = {{-1, 0, 0}, {0, -1, 0}, {0, 0, -1}};
static const int FACE[6][3] = {{-1, -1, 0}, {-1, 1, 0}, {-1, 0, -1}, {-1, 0, 1}, {0, -1, -1}, {0, -1, 1}};
static const int CORNER[4][3] = {{-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1}, {-1, 1, 1}};

/* returns 0 on success, 1 for an unsupported q */
static int make_lattice(int q, lattice *L) {
    int faces, corners;
    double w0, wa, wf, wc;
    if (q == 15) {
        faces = 0; corners = 1; w0 = 2.0 / 9.0; wa = 1.0 / 9.0; wf = 0.0; wc = 1.0 / 72.0;
    } else if (q == 19) {
        faces = 1; corners = 0; w0 = 1.0 / 3.0; wa = 1.0 / 18.0; wf = 1.0 / 36.0; wc = 0.0;
    } else if (q == 27) {
        faces = 1; corners = 1; w0 = 8.0 / 27.0; wa = 2.0 / 27.0; wf = 1.0 / 54.0; wc = 1.0 / 216.0;
    } else {
        return 1;
    }
    memset(L, 0, sizeof *L);
    L->q = q;
    L->h = (q - 1) / 2;
    int n = 1;
    L->w[0] = w0;
    for (int a = 0; a < 3; a++, n++) {
        memcpy(L->c[n], AXIS[a], sizeof AXIS[a]);
        L->w[n] = wa;
    }
    if (faces)
        for (int a = 0; a < 6; a++, n++) {
            memcpy(L->c[n], FACE[a], sizeof FACE[a]);
            L->w[n] = wf;
        }
    if (corners)
        for (int a = 0; a < 4; a++, n++) {
            memcpy(L->c[n], CORNER[a], sizeof CORNER[a]);
            L->w[n] = wc;
        }
    for (int i = 1; i <= L->h; i++) {
        for (int a = 0; a < 3; a++) L->c[i + L->h][a] = -L->c[i][a];
        L->w[i + L->h] = L->w[i];
        L->opp[i] = i + L->h;
        L->opp[i + L->h] = i;
    }
    L->opp[0] = 0;
    return 0;
}

int oracle_dqq_table(int q, int *c, double *w, int *opp) {
    lattice L;
    if (make_lattice(q, &L)) return 1;
    for (int i = 0; i < q; i++) {
        for (int a = 0; a < 3; a++) c[3 * i + a] = L.c[i][a];
        w[i] = L.w[i];
        opp[i] = L.opp[i];
    }
    return 0;
}

/* SURVEY.md 8(c) item 1, for one cell: moments, equilibrium with the
 * rest-population closure, BGK (the order of oracle.c's operations) */
static int collide_cell(const lattice *L, const double *f, double omega, double *out) {
    double r = 0.0, j[3] = {0.0, 0.0, 0.0}, u[3];
    for (int i = 0; i < L->q; i++) {
        r += f[i];
        for (int a = 0; a < 3; a++) j[a] += L->c[i][a] * f[i];
    }
    if (r == 0.0) return 1;
    for (int a = 0; a < 3; a++) u[a] = j[a] / r;
    double feq[QMAX];
    double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double rest = r;
    for (int i = 1; i < L->q; i++) {
        double cu = L->c[i][0] * u[0] + L->c[i][1] * u[1] + L->c[i][2] * u[2];
        feq[i] = L->w[i] * r * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        rest -= feq[i];
    }
    feq[0] = rest;
    for (int i = 0; i < L->q; i++) out[i] = f[i] - omega * (f[i] - feq[i]);
    return 0;
}

static size_t ix(int i, int x, int y, int z, int nx, int ny, int nz) {
    return (((size_t)i * nx + x) * ny + y) * nz + z;
}

static int wrapi(int s, int n) { return ((s % n) + n) % n; }

void oracle_dqq_equilibrium(int q, double rho, const double u[3], double *feq) {
    lattice L;
    if (make_lattice(q, &L)) return;
    double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    double rest = rho;
    for (int i = 1; i < q; i++) {
        double cu = L.c[i][0] * u[0] + L.c[i][1] * u[1] + L.c[i][2] * u[2];
        feq[i] = L.w[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        rest -= feq[i];
    }
    feq[0] = rest;
}

int oracle_dqq_collide(int q, const double *f, double omega, double *out) {
    lattice L;
    if (make_lattice(q, &L)) return 2;
    return collide_cell(&L, f, omega, out);
}

/* n steps in place on canonical f[i][x][y][z]: collide every cell (in
 * place), then pull-stream into the second lattice with the boundary rules
 * of SURVEY.md 8(c) item 2; swap. */
int oracle_dqq_run(int q, int nx, int ny, int nz, int bc, double tau, const double u_lid[3], long n, double *f) {
    lattice L;
    if (make_lattice(q, &L)) return 2;
    if (n <= 0) return 0;
    const double omega = 1.0 / tau, rho_w = 1.0;
    size_t len = (size_t)q * nx * ny * nz;
    double *g = (double *)malloc(sizeof(double) * len);
    if (!g) return 1;
    double *a = f, *b = g;
    for (long t = 0; t < n; t++) {
#pragma omp parallel for schedule(static) num_threads(oracle_get_threads())
        for (int x = 0; x < nx; x++)
            for (int y = 0; y < ny; y++)
                for (int z = 0; z < nz; z++) {
                    double fc[QMAX], out[QMAX];
                    for (int i = 0; i < q; i++) fc[i] = a[ix(i, x, y, z, nx, ny, nz)];
                    collide_cell(&L, fc, omega, out);
                    for (int i = 0; i < q; i++) a[ix(i, x, y, z, nx, ny, nz)] = out[i];
                }
#pragma omp parallel for schedule(static) num_threads(oracle_get_threads())
        for (int x = 0; x < nx; x++)
            for (int y = 0; y < ny; y++)
                for (int z = 0; z < nz; z++)
                    for (int i = 0; i < q; i++) {
                        int sx = x - L.c[i][0], sy = y - L.c[i][1], sz = z - L.c[i][2];
                        int inside = sx >= 0 && sx < nx && sy >= 0 && sy < ny && sz >= 0 && sz < nz;
                        double v;
                        if (bc == ORACLE_BC_PERIODIC) {
                            v = a[ix(i, wrapi(sx, nx), wrapi(sy, ny), wrapi(sz, nz), nx, ny, nz)];
                        } else if (inside) {
                            v = a[ix(i, sx, sy, sz, nx, ny, nz)];
                        } else {
                            v = a[ix(L.opp[i], x, y, z, nx, ny, nz)];
                            if (sz >= nz) {
                                double cu = L.c[i][0] * u_lid[0] + L.c[i][1] * u_lid[1] + L.c[i][2] * u_lid[2];
                                v = v + 6.0 * L.w[i] * rho_w * cu;
                            }
                        }
                        b[ix(i, x, y, z, nx, ny, nz)] = v;
                    }
        double *tmp = a;
        a = b;
        b = tmp;
    }
    if (a != f) memcpy(f, a, sizeof(double) * len);
    free(g);
    return 0;
}

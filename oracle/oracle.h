/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the D3Q19 BGK
 * lattice Boltzmann update of Fu & Song, arXiv 2208.05429.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2208_05429_b200/ and include/).
 *
 * All arithmetic is IEEE fp64, compiled with -O2 -ffp-contract=off and no
 * fast-math.  Population arrays use the layout f[i][x][y][z] (z fastest),
 * canonical direction order i = 0..18 of SURVEY.md Appendix A / SPEC.md:109.
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_BC_CAVITY = 0, ORACLE_BC_PERIODIC = 1 };

/* D3Q19 tables: velocities c[19][3], weights w[19], opposite index opp[19]. */
void oracle_d3q19(int c[19][3], double w[19], int opp[19]);

/* rho = sum_i f_i ; u = (sum_i c_i f_i) / rho.  Returns 1 on rho == 0. */
int oracle_moments(const double f[19], double *rho, double u[3]);

/* feq_i = w_i rho (1 + 3 c_i.u + 4.5 (c_i.u)^2 - 1.5 u.u), i >= 1;
 * feq_0 = rho - sum_{i>=1} feq_i   (rest-population closure, R-2). */
void oracle_equilibrium(double rho, const double u[3], double feq[19]);

/* BGK: out_i = f_i - omega (f_i - feq_i(rho(f), u(f))).  Returns 1 on rho == 0. */
int oracle_collide(const double f[19], double omega, double out[19]);

/* f[i][x][y][z] = feq_i(rho[x][y][z], u[x][y][z][:]).  rho/u NULL -> 1 / 0. */
void oracle_init_equilibrium(int nx, int ny, int nz, const double *rho,
                             const double *u, double *f);

/* One collide-then-pull-stream step on the whole domain:
 * f_out = S(C(f_in)), canonical f(t) -> f(t+1).  f_in is not modified. */
void oracle_step(int nx, int ny, int nz, int bc, double tau,
                 const double u_lid[3], const double *f_in, double *f_out);

/* n steps in place on f (internal scratch of the same size). */
int oracle_run(int nx, int ny, int nz, int bc, double tau,
               const double u_lid[3], long n, double *f);

/* One step on a sub-box [bx,bx+lx) x [by,by+ly) x [bz,bz+lz) of a global
 * nx*ny*nz domain.  f_in/f_out are box-local f[i][x][y][z].  A population
 * whose pull source lies inside the global domain but outside the box is
 * unknown and written as NaN; boundary rules are those of the global domain.
 * With the box equal to the domain this is oracle_step. */
void oracle_step_box(int nx, int ny, int nz, int bc, double tau,
                     const double u_lid[3], int bx, int by, int bz,
                     int lx, int ly, int lz, const double *f_in, double *f_out);

/* rho[x][y][z] and u[x][y][z][3] of canonical f. */
void oracle_macroscopic(int nx, int ny, int nz, const double *f, double *rho,
                        double *u);

/* Other cubic lattices (oracle_dqq.c): q = 15, 19 or 27, the
 * velocity order and weights documented there.  Populations f[i][x][y][z].
 * dqq_table: c[q][3], w[q], opp[q]; returns 1 for an unsupported q.
 * dqq_run: n steps in place (returns 1 on allocation failure, 2 for q). */
int oracle_dqq_table(int q, int *c, double *w, int *opp);
void oracle_dqq_equilibrium(int q, double rho, const double u[3], double *feq);
int oracle_dqq_collide(int q, const double *f, double omega, double *out);
int oracle_dqq_run(int q, int nx, int ny, int nz, int bc, double tau, const double u_lid[3], long n, double *f);

/* OpenMP threads used by the step loops (0 -> runtime default). */
void oracle_set_threads(int n);
int oracle_get_threads(void);

#ifdef __cplusplus
}
#endif
#endif

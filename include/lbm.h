/*
 * lbm.h -- C-ABI of the B200-native (sm_100a) D3Q19 lattice Boltzmann library
 * implementing the hot path of Fu & Song, "Designing a 3D Parallel
 * Memory-Aware Lattice Boltzmann Algorithm on Manycore Systems"
 * (arXiv 2208.05429): the fused collide + stream update with bounce-back
 * walls and a moving lid ("Fuse Swap LBM", Alg. 1), with
 * two collision-streaming cycles merged per sweep (Alg. 2),
 * X-slab partitioned across GPUs.
 *
 * Plain C types only: no torch or CUDA types cross this boundary (streams
 * and device pointers are passed as void* / double*).  Every function
 * returns an lbm_status and never aborts; lbm_last_error() gives the reason.
 *
 * Conventions shared by all calls
 * -------------------------------
 *  Domain      nx * ny * nz cells, all fluid.  The
 *              moving lid is the top z face z = nz-1 (R-5), with
 *              tangential velocity u_lid (u_lid[2] must be 0).
 *  Directions  canonical D3Q19 order i = 0..18 of SPEC.md:109 (directions
 *              1..9 lexicographically negative, opp(i) = i +- 9).
 *  Host arrays C order, z fastest.  rho[x][y][z]; u[x][y][z][3] (component
 *              fastest); populations f[i][x][y][z].  Always double, whatever
 *              the lattice dtype (fp32 lattices convert on copy).  With an
 *              X-slab partition (world > 1) every host/device array covers
 *              the caller's slab only: nx_local = nx / world planes starting
 *              at global x0 = rank * nx_local.
 *  Time        lbm_init_equilibrium / lbm_set_populations set the canonical
 *              state f(t0); lbm_step(n) advances it to f(t0 + n), where one
 *              step is collide then stream; the read-back
 *              calls return the canonical f(t) and its moments.
 *  Ownership   the context owns every device buffer, stream, event and
 *              communicator it creates; the caller owns all arrays it
 *              passes.  Host-array calls copy synchronously before
 *              returning; the caller may reuse the array immediately.
 *  Errors      LBM_EINVAL for invalid arguments (checked before any
 *              allocation or launch); LBM_ENOMEM for a failed allocation;
 *              LBM_ECUDA / LBM_ENCCL for a CUDA or NCCL failure, after which
 *              the context is poisoned and every later call except
 *              lbm_last_error / lbm_destroy returns LBM_ESTATE.  Errors of
 *              asynchronous work surface at the next blocking call.
 *              LBM_ENUMERIC from a blocking read-back of degenerate or
 *              non-finite moments (the context stays usable).  An input
 *              rejected by lbm_init_equilibrium / lbm_set_populations
 *              (EINVAL) may already have overwritten part of the state: it
 *              is then undefined, and lbm_step / the read-backs return
 *              LBM_ESTATE until a successful init.
 *  NCCL        with comm == NCCL every call that touches the state is
 *              COLLECTIVE: all ranks make the same sequence of
 *              lbm_init_equilibrium(_device), lbm_set_populations,
 *              lbm_step, lbm_macroscopic(_device) and
 *              lbm_get_populations(_box) calls (read-backs exchange stale
 *              ghost planes first -- also for an empty box).  Input
 *              validation is agreed across ranks: if one rank rejects its
 *              input, every rank returns EINVAL before any exchange.
 *              Failure detection: blocking calls poll the communicator; an
 *              asynchronous NCCL error, or no sweep completing for
 *              LBM_NCCL_TIMEOUT_S seconds (default 120: a lost or stalled
 *              peer), aborts the communicator and returns LBM_ENCCL (the
 *              context is poisoned).  lbm_create_ex's AUTO storage choice
 *              is made on the smallest free memory of all ranks, so every
 *              rank picks the same storage.
 *  Threads     a context is not thread-safe; distinct contexts are
 *              independent.  Every call leaves the calling thread's current
 *              CUDA device as it found it.
 */
#ifndef LBM_B200_H
#define LBM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBM_ABI_VERSION 3

typedef struct lbm_ctx lbm_ctx; /* opaque; library-owned */

typedef enum { LBM_F64 = 0, LBM_F32 = 1 } lbm_dtype;

/* Boundary mode.  CAVITY: link-wise (half-way) bounce-back on all six faces
 * and the moving lid on z = nz-1 (R-4..R-7; SPEC.md:164-182;
 * BASELINE.json configs 1, 2, 4, 5).  PERIODIC: wrap on all three axes
 * (BASELINE.json config 3), u_lid ignored. */
typedef enum { LBM_BC_CAVITY = 0, LBM_BC_PERIODIC = 1 } lbm_bc;

typedef enum {
    LBM_OK = 0,
    LBM_EINVAL = 1,
    LBM_ENOMEM = 2,
    LBM_ECUDA = 3,
    LBM_ENCCL = 4,
    LBM_ESTATE = 5,
    /* lbm_macroscopic found rho == 0 (degenerate moments: never
     * a silent division) or non-finite moments (a diverged state) in some
     * cell; the outputs are written, the context stays usable. */
    LBM_ENUMERIC = 6
} lbm_status;

/* Sweep kernel selection.  K1: one fused collide+stream step per HBM pass
 * (Alg. 1's loop fusion).  K2: two steps per HBM pass, temporally blocked
 * on chip (Alg. 2's two-step merge): TMA-staged shared-memory tiles where the
 * TMA descriptor can describe the slab (z pitch a multiple of 16 bytes,
 * (nx_local+4)*19 < 2^31); an odd remainder uses K1.  K2_REG (value 3) is
 * reserved: the cp.async-staged variant it named measured slower than K2
 * wherever K2 applies and was removed -- lbm_create_ex rejects it (EINVAL).
 * AUTO = K2, falling back to K1 pairs where the descriptor cannot describe
 * the slab; an explicit K2 on such a slab gives EINVAL from lbm_step.  AUTO also
 * switches to the single-copy K2_SC storage (below) when two lattice copies
 * do not fit the device's free memory at create but one does.  Results are
 * bitwise identical whichever kernel runs. */
typedef enum {
    LBM_KERNEL_AUTO = 0,
    LBM_KERNEL_K1 = 1,
    LBM_KERNEL_K2 = 2,
    LBM_KERNEL_K2_REG = 3,
    /* Single-copy in-place storage, the AA pattern (
     * the paper's one-lattice swap): one lattice
     * buffer instead of two (half the memory), alternating an in-place
     * collide-and-revert step with a gather/scatter step; one step per HBM
     * pass (K1's bytes).  X-slabs exchange five slot-planes per side before
     * and after each odd step; cavity slabs need >= 2 planes (EINVAL).
     * Bitwise identical to K1 without a lid (with it, K1's pull storage
     * rounds the lid term once more: agreement to ~1 ulp). */
    LBM_KERNEL_AA = 4,
    /* Single-copy storage with the two-step merge -- the paper's pairing of
     * one lattice copy with two steps per pass (
     * SURVEY.md 8(f) row 1).  The K2 sweep runs in place: the lattice is a
     * ring of nx + 4 + G planes (G = 68 fp64, 148 on slabs of >= 1024
     * planes, 100 fp32; 1.14x a single copy at nx = 1024, plus a staging
     * buffer of max(3 planes, 64 MB, 1/16 of the lattice) for host
     * transfers) and each sweep writes f*(t+1) of plane x G planes below the
     * slot of f*(t-1) of plane x, chunks of <= (G - 4) / 2 planes
     * taken in x order, so no plane is overwritten before its last
     * reader has finished; an odd step runs the in-place K1 the same way.
     * Bitwise identical to K2/K1.  X-slabs (LOCAL, NCCL): each slab its own
     * ring, halo parts exchanged through the ring mapping; init and
     * set_populations write the canonical state and invert the stream in
     * place.  EINVAL at create where the TMA descriptor cannot describe the
     * slab. */
    LBM_KERNEL_K2_SC = 5,
    /* Three collision-streaming steps per HBM pass (
     * the paper's future work "merge more time steps"):
     * the K2 sweep one level deeper -- T+2 staged, two shared-memory rings --
     * so each population crosses HBM once per three steps, for 1.69 + 1.33
     * + 1 collisions per output cell.  A measured prototype (DESIGN.md
     * section 11): fp32, periodic, one slab (comm NONE); EINVAL otherwise.
     * lbm_step(n) runs floor(n/3) three-step sweeps, the remainder as K2 /
     * K1.  Bitwise identical to K1. */
    LBM_KERNEL_K3 = 6
} lbm_kernel;

/* X-Y partition (the paper's future work "partition a
 * 3D domain along three axes"), emulated on one device like
 * the LOCAL X-slabs: opts.local_blocks_y > 1 splits each of the
 * local_slabs x ranges into that many y blocks (ny divisible, >= 4 rows
 * each).  Every block carries 2 frame rows per side holding its
 * y-neighbours' edge rows; before a sweep the frame rows are exchanged
 * (block to block), then the x ghost planes (which carry them along, so the
 * x-y edge cells come from the diagonal block).  Cavity walls only at the
 * domain's ends; a periodic box wraps around the blocks.  Two-buffer K1/K2
 * storage (kernel AUTO, K1 or K2), D3Q19; EINVAL otherwise.  Host arrays
 * cover the whole domain as usual.  Bitwise identical to one slab. */

/* Halo transport between X-slabs (PAPER.md:336 X-only partition).
 *  NONE   world == 1 and local_slabs == 1 (periodic x wraps onto itself)
 *  NCCL   one slab per process/GPU, ncclSend/ncclRecv over NVLink
 *  LOCAL  local_slabs slabs on this one device, copies between them (the
 *         multi-GPU data path emulated on one GPU, for tests) */
typedef enum { LBM_COMM_NONE = 0, LBM_COMM_NCCL = 1, LBM_COMM_LOCAL = 2 } lbm_comm;

/* How NCCL ranks get their ghost planes.
 *  AUTO / EXCHANGE  grouped ncclSend/ncclRecv of the 24-slot spans before a
 *                   sweep, overlapped with the interior sweep.
 *  PEER             fused cross-GPU halo: the lattice buffers are CUDA VMM
 *                   allocations mapped into the neighbouring ranks (POSIX
 *                   descriptors passed over a Unix domain socket, so all
 *                   ranks must share one host), and every two-step sweep
 *                   stores the planes its neighbours read straight into
 *                   their next-sweep buffers over NVLink; consecutive sweeps
 *                   of neighbours are ordered by stream memory operations
 *                   (a done-counter per neighbour), the paper's "synchronize
 *                   at the intersection layers every two time steps"
 *                   (PAPER.md:747-749).  Needs comm == NCCL (world 1 maps the
 *                   slab onto itself: the periodic self-wrap), kernel AUTO or
 *                   K2 (two-buffer storage); EINVAL otherwise, ENCCL if the
 *                   rendezvous fails.  One-step sweeps (odd remainders) and
 *                   init still exchange through NCCL.  Bitwise identical to
 *                   EXCHANGE. */
typedef enum { LBM_HALO_AUTO = 0, LBM_HALO_EXCHANGE = 1, LBM_HALO_PEER = 2 } lbm_halo;

/* Velocity set.  D3Q19 is the paper's and the hot path (every kernel and
 * storage above).  D3Q15 and D3Q27 -- "no matter using D3Q15, D3Q19, D3Q27"
 * -- run the same method (BGK with the
 * rest-population closure, link-wise bounce-back, the moving lid, periodic
 * wrap) on one slab (comm NONE; kernel AUTO, K1 or K2, EINVAL otherwise):
 * with AUTO or K2 each pair of steps is one two-step sweep per HBM pass
 * (the paper's merge for these lattices; ECUDA under K2
 * if the driver cannot encode TMA descriptors, AUTO then falls back), an
 * odd remainder and kernel K1 one fused collide + stream step per pass;
 * the results are bitwise the same.  Across NCCL ranks (comm NCCL, x slabs
 * only: local_slabs 1, ranks_y 1, halo AUTO or EXCHANGE; kernel AUTO or
 * K1, K2 is EINVAL) every step is the one-step kernel: links leaving the
 * slab through a face shared with a neighbour rank land in a ghost plane
 * and are sent to that rank after the step (one ncclSend/ncclRecv per
 * direction with c_x = +-1; a one-rank periodic box sends its wrap to
 * itself); host arrays then cover the rank's slab, as for D3Q19, and input
 * validation is agreed across ranks.  Host population arrays
 * are f[q][nx][ny][nz] in the order lbm_lattice_table gives: i = 0 rest,
 * 1 .. (q-1)/2 the velocities whose first nonzero component is -1 (axes,
 * face diagonals, corners), then their opposites in the same order -- for
 * q = 19 exactly SPEC.md:109's order. */
typedef enum { LBM_D3Q15 = 15, LBM_D3Q19 = 19, LBM_D3Q27 = 27 } lbm_lattice;

/* c[q][3] and w[q] of lattice q (15, 19, 27).  EINVAL for another q. */
lbm_status lbm_lattice_table(int q, int *c, double *w);

typedef struct {
    int struct_size;     /* sizeof(lbm_opts), for forward compatibility */
    int bc;              /* lbm_bc */
    int device;          /* CUDA device ordinal; -1 = the current device */
    int rank, world;     /* X-slab partition: this process is slab `rank` of `world`
                            (host arrays: nx_local = nx / world planes, ny_local = ny rows;
                            see ranks_y for X-Y blocks) */
    int comm;            /* lbm_comm */
    const void *nccl_id; /* 128-byte ncclUniqueId (same on all ranks) when comm == NCCL */
    void *stream;        /* cudaStream_t to run on, or NULL: the context creates one */
    int kernel;          /* lbm_kernel */
    int local_slabs;     /* comm == LOCAL: number of slabs emulated on this device */
    int halo;            /* lbm_halo (ABI 2) */
    int lattice;         /* lbm_lattice: 19 (default; 0 reads as 19), 15 or 27 (ABI 2) */
    int local_blocks_y;  /* comm == LOCAL: also split every x slab into this many y blocks
                            (X-Y partition; 0 or 1 = none) (ABI 2) */
    int ranks_y;         /* comm == NCCL: the world ranks form a (world / ranks_y) x ranks_y
                            grid of X-Y blocks ("partition a 3D domain along
                            three axes"): rank r holds x slab r / ranks_y (nx_local =
                            nx / (world / ranks_y) planes) and y block r % ranks_y (ny_local =
                            ny / ranks_y rows, >= 4); its host arrays cover that block,
                            [nx_local][ny_local][nz].  Two-buffer K1/K2 storage (kernel AUTO,
                            K1 or K2), halo EXCHANGE, D3Q19.  0 or 1 = X-slabs (ABI 3) */
} lbm_opts;

/* Fills *opts with defaults: CAVITY, device -1, rank 0, world 1, NONE,
 * no id, own stream, AUTO, 1 local slab, halo AUTO, D3Q19. */
void lbm_default_opts(lbm_opts *opts);

/* Create a lattice of nx*ny*nz cells with BGK relaxation time tau
 * (omega = 1/tau; PAPER.md delegates the collision to Palabos, PAPER.md:831,
 * BASELINE.json fixes BGK, R-1) and lid velocity u_lid[3] (may be
 * NULL = 0).  dtype is the storage and arithmetic type of the populations.
 * EINVAL: nx, ny, nz < 1; tau <= 0.5 or not finite; u_lid[2] != 0 or
 * |u_lid| > 0.3; nx % world != 0; slabs of fewer
 * than 4 planes when world * local_slabs > 1; periodic with nx_local < 2;
 * rank outside [0, world); comm inconsistent with world / local_slabs.
 * The state is undefined until lbm_init_equilibrium / lbm_set_populations. */
lbm_status lbm_create(lbm_ctx **out, int nx, int ny, int nz, double tau,
                      const double u_lid[3], lbm_dtype dtype);
lbm_status lbm_create_ex(lbm_ctx **out, int nx, int ny, int nz, double tau,
                         const double u_lid[3], lbm_dtype dtype, const lbm_opts *opts);

/* f_i = feq_i(rho, u) on every cell of the slab (SPEC.md:74-82 with the
 * rest-population closure, R-2).  rho: host [nx_local][ny_local][nz]
 * or NULL (= 1); u: host [nx_local][ny_local][nz][3] or NULL (= 0).
 * EINVAL if any rho <= 0 or any value is not finite. */
lbm_status lbm_init_equilibrium(lbm_ctx *ctx, const double *rho, const double *u);
/* Same with DEVICE pointers on the context's device (not validated). */
lbm_status lbm_init_equilibrium_device(lbm_ctx *ctx, const double *d_rho, const double *d_u);

/* Advance n >= 0 time steps (asynchronous on the context stream).  Each
 * step is collide (BGK) then stream with the boundary rules (Alg. 1,
 * PAPER.md:275-294); pairs of steps run as one two-step sweep (Alg. 2's
 * merge).  lbm_step(a); lbm_step(b) is bitwise identical
 * to lbm_step(a + b).  EINVAL if n < 0; ESTATE before initialisation. */
lbm_status lbm_step(lbm_ctx *ctx, long n);

/* Moments of the canonical f(t): rho = sum_i f_i, u = (sum_i c_i f_i)/rho
 * (the paper's velocity norms).  Host arrays
 * rho [nx_local][ny_local][nz], u [nx_local][ny_local][nz][3]; either may be NULL.
 * Blocks until the copy is complete.  ENUMERIC if some cell has rho == 0 or
 * non-finite moments (the arrays are still filled). */
lbm_status lbm_macroscopic(lbm_ctx *ctx, double *rho, double *u);
/* Same into DEVICE arrays; asynchronous on the context stream (no ENUMERIC
 * check: it would need a synchronisation). */
lbm_status lbm_macroscopic_device(lbm_ctx *ctx, double *d_rho, double *d_u);

/* Canonical populations f(t) as host f[q][nx_local][ny_local][nz] (canonical
 * direction order; q = 19 unless opts.lattice says otherwise).  Blocks. */
lbm_status lbm_get_populations(lbm_ctx *ctx, double *f);
/* The box [x0,x0+lx) x [y0,y0+ly) x [z0,z0+lz) of the slab (slab-local x)
 * as host f[19][lx][ly][lz].  EINVAL if the box leaves the slab. */
lbm_status lbm_get_populations_box(lbm_ctx *ctx, int x0, int y0, int z0, int lx,
                                   int ly, int lz, double *f);
/* Set the canonical state f(t) from host f[q][nx_local][ny_local][nz].  EINVAL if
 * a value is not finite. */
lbm_status lbm_set_populations(lbm_ctx *ctx, const double *f);

/* Wait for all work queued on the context stream; reports async errors. */
lbm_status lbm_synchronize(lbm_ctx *ctx);

/* Time steps advanced since the last init / set (the canonical t - t0). */
lbm_status lbm_get_time(const lbm_ctx *ctx, long *t);

/* rank 0 creates the NCCL id that every rank passes as opts.nccl_id.
 * out128 must hold 128 bytes.  ENCCL if libnccl.so.2 cannot be loaded. */
lbm_status lbm_nccl_unique_id(void *out128);

/* Halo plan of one X-slab, computed on the host (no GPU needed).  Offsets
 * and counts are in ELEMENTS of the slab buffer (dtype-sized), which is
 * laid out as planes p = 0 .. nx_local+3 (slab-local x = p - 2, two ghost
 * planes per side), each plane [19 internal directions][ny][nz_pitch]
 * (the two-buffer storage -- LBM_KERNEL_K2_SC
 * keeps the same planes on a ring and moves the same spans in plane parts).
 * A neighbour of -1 means a wall (no exchange). */
typedef struct {
    int nx_local, x0;
    int nz_pitch;            /* z row pitch in elements */
    long long plane_q;       /* elements per (x, direction) plane = (ny + 2 y_ghost) * nz_pitch */
    long long plane_x;       /* elements per x plane = 19 * plane_q */
    long long buffer_elems;  /* (nx_local + 4) * plane_x */
    int left, right;         /* neighbour ranks or -1 */
    long long send_left_off, send_right_off, recv_left_off, recv_right_off;
    long long span;          /* elements per message (24 * plane_q) */
    int dir_of_slot[19];     /* canonical direction stored at internal slot k */
    /* Periodic boxes: every (x, direction) plane has a ghost frame of
     * y_ghost (2; 3 in a LBM_KERNEL_K3 context) rows above and below the ny
     * rows and z_offset elements
     * (32 bytes) of columns before z = 0 and after z = nz-1, holding copies
     * of the periodically wrapped cells; cavity: 0, 0.  Cell (y, z) of a
     * plane is at cell0 + y * nz_pitch + z, cell0 = y_ghost * nz_pitch +
     * z_offset. */
    int y_ghost, z_offset;
    long long cell0;
    /* X-Y blocks (lbm_plan_halo_xy, ABI 3; X-slabs: down = up = -1,
     * ny_local = ny, y0 = 0).  The block's planes carry y_ghost = 2 frame
     * rows per side (both boundary modes) holding the y-neighbours' edge
     * rows.  Before every exchange of the x spans above, each rank sends the
     * band of y_ghost rows (y_band = y_ghost * nz_pitch elements at offset
     * send_down_off / send_up_off of every (x, direction) plane of its own
     * planes x = 0 .. nx_local-1, i.e. 19 * nx_local bands at stride plane_q
     * starting at plane x = 0) to its down / up neighbour, which stores them
     * at recv_up_off / recv_down_off; the x spans then carry those rows to
     * the x-neighbours, so the x-y corner entries come from the diagonal
     * block without a diagonal message.  Ranks are numbered
     * rank = x_slab * ranks_y + y_block; left/right above are ranks too. */
    int down, up;            /* y-neighbour ranks or -1 (a cavity wall) */
    int ny_local, y0;
    long long y_band;
    long long send_down_off, send_up_off, recv_down_off, recv_up_off;
} lbm_halo_plan;

lbm_status lbm_plan_halo(int nx, int ny, int nz, lbm_dtype dtype, int bc, int rank,
                         int world, lbm_halo_plan *plan);
/* The same for a (world / ranks_y) x ranks_y rank grid of X-Y blocks
 * (lbm_opts.ranks_y; ranks_y == 1 is lbm_plan_halo).  EINVAL: world %
 * ranks_y != 0, nx % (world / ranks_y) != 0, ny % ranks_y != 0. */
lbm_status lbm_plan_halo_xy(int nx, int ny, int nz, lbm_dtype dtype, int bc, int rank,
                            int world, int ranks_y, lbm_halo_plan *plan);

/* Diagnostics for the bench harness (no effect on results).
 * Kernel launches issued by this context since creation, and optional CUDA
 * event timing of every sweep launch (K1 and K2 only) on the context
 * stream: total milliseconds, launch count and the lattice updates they
 * performed. */
typedef struct {
    long long launches;        /* all kernel launches by this context */
    long long sweep_launches;  /* timed sweeps since lbm_profile_reset: one record per sweep of
                                  all of the context's slabs (with a halo exchange overlapped,
                                  interior + edge launches and the wait between them) */
    double sweep_ms;           /* their summed event time */
    long long sweep_updates;   /* cell updates they performed */
    long long k2_launches, k1_launches;
} lbm_stats;

lbm_status lbm_profile_enable(lbm_ctx *ctx, int on);
lbm_status lbm_profile_reset(lbm_ctx *ctx);
lbm_status lbm_get_stats(lbm_ctx *ctx, lbm_stats *stats); /* synchronises */

/* Last error message of ctx, or of the calling thread when ctx is NULL. */
const char *lbm_last_error(const lbm_ctx *ctx);

/* Release everything the context owns.  NULL-safe. */
void lbm_destroy(lbm_ctx *ctx);

int lbm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif

// dqq.cu -- the other cubic lattices the paper names next to D3Q19, "no
// matter using D3Q15, D3Q19, D3Q27 or extended lattice models" (
// SURVEY.md 8(f) row 4): the fused collide + stream step with bounce-back
// walls, the moving lid and periodic wrap for D3Q15 and D3Q27.
//
// One step per HBM pass (the loop fusion of Alg. 1): a
// thread reads its cell's q populations of the canonical f(t) (aligned,
// coalesced along z), collides (BGK with the rest-population closure, the
// arithmetic and operation order of the oracle's definition),
// and PUSHES f*_i to the cell it streams to, x + c_i, in the other buffer --
// or, where that lies beyond a cavity wall, bounces it back into slot opp(i)
// of its own cell, plus the lid term 6 w_opp rho_w (c_opp . u_lid) when the
// wall is the moving lid (the pull rule of SURVEY.md 8(c) seen from the
// sender).  Each destination slot is written exactly once.  Storage is the
// canonical f(t), [q][nx][ny][nz_pitch], so read-backs are copies.
// Algorithmic bytes: 2 q sizeof(T) per update (432 B fp64 for D3Q27).
//
// Velocity order (include/lbm.h lbm_lattice_table): i = 0 rest; 1 .. h the
// half with first nonzero component -1 -- axes, face diagonals, corners, in
// the order below; h+1 .. 2h the opposites.  For q = 19 this is SPEC.md:109's
// order (the D3Q19 path itself lives in d3q19.cuh / k2.cu).
#include <cstdint>

#include "kernels.h"

namespace lbm {

namespace {

// velocities of the negative half, weights by |c|^2
__host__ __device__ constexpr int dqq_half_c(int q, int j, int a) {
    // axes
    constexpr int AX[3][3] = {{-1, 0, 0}, {0, -1, 0}, {0, 0, -1}};
    constexpr int FA[6][3] = {{-1, -1, 0}, {-1, 1, 0}, {-1, 0, -1}, {-1, 0, 1}, {0, -1, -1}, {0, -1, 1}};
    constexpr int CO[4][3] = {{-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1}, {-1, 1, 1}};
    if (j < 3) return AX[j][a];
    if (q == 15) return CO[j - 3][a];
    if (j < 9) return FA[j - 3][a];
    return CO[j - 9][a];
}

template <int Q>
__host__ __device__ constexpr int dqq_c(int i, int a) {
    constexpr int H = (Q - 1) / 2;
    return i == 0 ? 0 : (i <= H ? dqq_half_c(Q, i - 1, a) : -dqq_half_c(Q, i - 1 - H, a));
}
template <int Q>
__host__ __device__ constexpr int dqq_opp(int i) {
    constexpr int H = (Q - 1) / 2;
    return i == 0 ? 0 : (i <= H ? i + H : i - H);
}
template <int Q>
__host__ __device__ constexpr double dqq_w(int i) {
    const int n = dqq_c<Q>(i, 0) * dqq_c<Q>(i, 0) + dqq_c<Q>(i, 1) * dqq_c<Q>(i, 1) + dqq_c<Q>(i, 2) * dqq_c<Q>(i, 2);
    if (Q == 15) return n == 0 ? 2.0 / 9.0 : (n == 1 ? 1.0 / 9.0 : 1.0 / 72.0);
    if (Q == 27) return n == 0 ? 8.0 / 27.0 : (n == 1 ? 2.0 / 27.0 : (n == 2 ? 1.0 / 54.0 : 1.0 / 216.0));
    return n == 0 ? 1.0 / 3.0 : (n == 1 ? 1.0 / 18.0 : 1.0 / 36.0);
}

// SURVEY.md 8(c) item 1 for one cell, in the oracle's operation order
template <typename T, int Q>
__device__ __forceinline__ void dqq_collide(T (&f)[Q], T omega) {
    T r = T(0), jx = T(0), jy = T(0), jz = T(0);
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        r = r + f[i];
        jx = jx + T(dqq_c<Q>(i, 0)) * f[i];
        jy = jy + T(dqq_c<Q>(i, 1)) * f[i];
        jz = jz + T(dqq_c<Q>(i, 2)) * f[i];
    });
    const T ux = jx / r, uy = jy / r, uz = jz / r;
    const T usq = ux * ux + uy * uy + uz * uz;
    T feq[Q];
    T rest = r;
    static_for<1, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const T cu = T(dqq_c<Q>(i, 0)) * ux + T(dqq_c<Q>(i, 1)) * uy + T(dqq_c<Q>(i, 2)) * uz;
        feq[i] = T(dqq_w<Q>(i)) * r * (T(1) + T(3) * cu + T(4.5) * cu * cu - T(1.5) * usq);
        rest = rest - feq[i];
    });
    feq[0] = rest;
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        f[i] = f[i] - omega * (f[i] - feq[i]);
    });
}

}  // namespace

// one fused collide + push step, canonical A = f(t) -> B = f(t+1)
template <typename T, int Q, int BC>
__global__ void __launch_bounds__(256) k_dqq_step(const T* __restrict__ A, T* __restrict__ B, DqqGeom g, T omega,
                                                 double ulx, double uly) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.z;
    if (z >= g.nz || y >= g.ny) return;
    const long long self = ((long long)x * g.ny + y) * g.nzp + z;
    T f[Q];
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        f[i] = A[(long long)i * g.pq + self];
    });
    dqq_collide<T, Q>(f, omega);
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
        int dx = x + cx, dy = y + cy, dz = z + cz;
        bool out = false;
        if constexpr (BC == BC_PERIODIC) {
            dx = dx < 0 ? dx + g.nx : (dx >= g.nx ? dx - g.nx : dx);
            dy = dy < 0 ? dy + g.ny : (dy >= g.ny ? dy - g.ny : dy);
            dz = dz < 0 ? dz + g.nz : (dz >= g.nz ? dz - g.nz : dz);
        } else {
            out = dx < 0 || dx >= g.nx || dy < 0 || dy >= g.ny || dz < 0 || dz >= g.nz;
        }
        if (!out) {
            __stcs(B + (long long)i * g.pq + ((long long)dx * g.ny + dy) * g.nzp + dz, f[i]);
        } else {
            constexpr int o = dqq_opp<Q>(i);
            T v = f[i];
            if (dz >= g.nz) {  // the moving lid: 6 w_o rho_w (c_o . u_lid), rho_w = 1
                const double cu = dqq_c<Q>(o, 0) * ulx + dqq_c<Q>(o, 1) * uly;
                v = v + T(6.0 * dqq_w<Q>(o) * 1.0 * cu);
            }
            __stcs(B + (long long)o * g.pq + self, v);
        }
    });
}

// canonical feq(rho, u) (rho / u NULL: 1 / 0)
template <typename T, int Q>
__global__ void __launch_bounds__(256) k_dqq_init(const double* __restrict__ rho, const double* __restrict__ u,
                                                 T* __restrict__ A, DqqGeom g) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.z;
    if (z >= g.nz || y >= g.ny) return;
    const long long cell = ((long long)x * g.ny + y) * g.nz + z;
    const long long self = ((long long)x * g.ny + y) * g.nzp + z;
    const double r = rho ? rho[cell] : 1.0;
    const double ux = u ? u[3 * cell] : 0.0, uy = u ? u[3 * cell + 1] : 0.0, uz = u ? u[3 * cell + 2] : 0.0;
    // in fp64 (the input precision), then stored in T
    const double usq = ux * ux + uy * uy + uz * uz;
    double rest = r;
    static_for<1, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const double cu = dqq_c<Q>(i, 0) * ux + dqq_c<Q>(i, 1) * uy + dqq_c<Q>(i, 2) * uz;
        const double feq = dqq_w<Q>(i) * r * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        rest = rest - feq;
        A[(long long)i * g.pq + self] = T(feq);
    });
    A[self] = T(rest);
}

// rho, u (double, [x][y][z] / [x][y][z][3]) of planes [xbeg, xbeg + nxc)
template <typename T, int Q>
__global__ void __launch_bounds__(256) k_dqq_moments(const T* __restrict__ A, DqqGeom g, int xbeg, double* rho,
                                                    double* u, int* flag) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int xl = blockIdx.z, x = xbeg + xl;
    if (z >= g.nz || y >= g.ny) return;
    const long long self = ((long long)x * g.ny + y) * g.nzp + z;
    double r = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        const double v = double(A[(long long)i * g.pq + self]);
        r = r + v;
        jx = jx + dqq_c<Q>(i, 0) * v;
        jy = jy + dqq_c<Q>(i, 1) * v;
        jz = jz + dqq_c<Q>(i, 2) * v;
    });
    const long long cell = ((long long)xl * g.ny + y) * g.nz + z;
    const double ux = jx / r, uy = jy / r, uz = jz / r;
    if (rho) rho[cell] = r;
    if (u) {
        u[3 * cell] = ux;
        u[3 * cell + 1] = uy;
        u[3 * cell + 2] = uz;
    }
    if (flag) {
        const int bad = r == 0.0 ? 1 : ((isfinite(r) && isfinite(ux) && isfinite(uy) && isfinite(uz)) ? 0 : 2);
        if (bad) atomicOr(flag, bad);
    }
}

// box [x0, x0+lx) x [y0, ..) x [z0, ..) as double out[q][lx][ly][lz]
template <typename T, int Q>
__global__ void __launch_bounds__(256) k_dqq_box(const T* __restrict__ A, DqqGeom g, int x0, int y0, int z0, int lx,
                                                int ly, int lz, double* __restrict__ out) {
    const int zl = blockIdx.x * 32 + threadIdx.x, yl = blockIdx.y * 8 + threadIdx.y, xl = blockIdx.z;
    if (zl >= lz || yl >= ly) return;
    const long long self = ((long long)(x0 + xl) * g.ny + (y0 + yl)) * g.nzp + (z0 + zl);
    const long long o = ((long long)xl * ly + yl) * lz + zl, n = (long long)lx * ly * lz;
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        out[i * n + o] = double(A[(long long)i * g.pq + self]);
    });
}

// canonical doubles src[q][nxc][ny][nz] -> planes [xbeg, xbeg + nxc)
template <typename T, int Q>
__global__ void __launch_bounds__(256) k_dqq_import(const double* __restrict__ src, T* __restrict__ A, DqqGeom g,
                                                   int xbeg, int nxc) {
    const int z = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, xl = blockIdx.z;
    if (z >= g.nz || y >= g.ny) return;
    const long long self = ((long long)(xbeg + xl) * g.ny + y) * g.nzp + z;
    const long long o = ((long long)xl * g.ny + y) * g.nz + z, n = (long long)nxc * g.ny * g.nz;
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        A[(long long)i * g.pq + self] = T(src[i * n + o]);
    });
}

// ------------------------------------------------------------------ host --
namespace {
dim3 dqq_grid(int nz, int ny, int nx) { return dim3((nz + 31) / 32, (ny + 7) / 8, nx); }
const dim3 kDqqBlock(32, 8, 1);
}  // namespace

#define LBM_DQQ_DISPATCH(call)                      \
    switch (g.q) {                                  \
        case 15: call(15); break;                   \
        case 27: call(27); break;                   \
        default: return cudaErrorInvalidValue;      \
    }

template <typename T>
cudaError_t launch_dqq_step(const T* A, T* B, const DqqGeom& g, T omega, const double ulid[3], cudaStream_t s) {
    const dim3 grid = dqq_grid(g.nz, g.ny, g.nx);
#define STEP(Q)                                                                                       \
    if (g.bc == BC_PERIODIC) k_dqq_step<T, Q, BC_PERIODIC><<<grid, kDqqBlock, 0, s>>>(A, B, g, omega, ulid[0], ulid[1]); \
    else k_dqq_step<T, Q, BC_CAVITY><<<grid, kDqqBlock, 0, s>>>(A, B, g, omega, ulid[0], ulid[1]);
    LBM_DQQ_DISPATCH(STEP)
#undef STEP
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dqq_init(const double* rho, const double* u, T* A, const DqqGeom& g, cudaStream_t s) {
    const dim3 grid = dqq_grid(g.nz, g.ny, g.nx);
#define INIT(Q) k_dqq_init<T, Q><<<grid, kDqqBlock, 0, s>>>(rho, u, A, g);
    LBM_DQQ_DISPATCH(INIT)
#undef INIT
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dqq_moments(const T* A, const DqqGeom& g, int xbeg, int nxc, double* rho, double* u, int* flag,
                               cudaStream_t s) {
    const dim3 grid = dqq_grid(g.nz, g.ny, nxc);
#define MOM(Q) k_dqq_moments<T, Q><<<grid, kDqqBlock, 0, s>>>(A, g, xbeg, rho, u, flag);
    LBM_DQQ_DISPATCH(MOM)
#undef MOM
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dqq_box(const T* A, const DqqGeom& g, int x0, int y0, int z0, int lx, int ly, int lz, double* out,
                           cudaStream_t s) {
    const dim3 grid = dqq_grid(lz, ly, lx);
#define BOX(Q) k_dqq_box<T, Q><<<grid, kDqqBlock, 0, s>>>(A, g, x0, y0, z0, lx, ly, lz, out);
    LBM_DQQ_DISPATCH(BOX)
#undef BOX
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dqq_import(const double* src, T* A, const DqqGeom& g, int xbeg, int nxc, cudaStream_t s) {
    const dim3 grid = dqq_grid(g.nz, g.ny, nxc);
#define IMP(Q) k_dqq_import<T, Q><<<grid, kDqqBlock, 0, s>>>(src, A, g, xbeg, nxc);
    LBM_DQQ_DISPATCH(IMP)
#undef IMP
    return cudaGetLastError();
}
#undef LBM_DQQ_DISPATCH

void dqq_table(int q, int* c, double* w) {
    for (int i = 0; i < q; ++i) {
        for (int a = 0; a < 3; ++a) c[3 * i + a] = q == 15 ? dqq_c<15>(i, a) : (q == 27 ? dqq_c<27>(i, a) : 0);
        w[i] = q == 15 ? dqq_w<15>(i) : (q == 27 ? dqq_w<27>(i) : 0.0);
    }
}

#define LBM_DQQ_INST(T)                                                                                         \
    template cudaError_t launch_dqq_step<T>(const T*, T*, const DqqGeom&, T, const double*, cudaStream_t);     \
    template cudaError_t launch_dqq_init<T>(const double*, const double*, T*, const DqqGeom&, cudaStream_t);   \
    template cudaError_t launch_dqq_moments<T>(const T*, const DqqGeom&, int, int, double*, double*, int*,     \
                                               cudaStream_t);                                                  \
    template cudaError_t launch_dqq_box<T>(const T*, const DqqGeom&, int, int, int, int, int, int, double*,    \
                                           cudaStream_t);                                                      \
    template cudaError_t launch_dqq_import<T>(const double*, T*, const DqqGeom&, int, int, cudaStream_t);
LBM_DQQ_INST(double)
LBM_DQQ_INST(float)
#undef LBM_DQQ_INST

}  // namespace lbm

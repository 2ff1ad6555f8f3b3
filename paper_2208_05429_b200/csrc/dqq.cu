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
#include <cuda.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "kernels.h"

#ifndef KQ_FAST
#define KQ_FAST 1
#endif

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

// half-set index j leads a packed pair (j, j+1) of one weight class (fp32)
template <int Q>
__host__ __device__ constexpr bool dqq_lead(int j) {
    constexpr int H = (Q - 1) / 2;
    bool prev = false;
    for (int k = 0; k <= j; ++k) {
        const int a = k + 1, b = k + 2;
        const int na = dqq_c<Q>(a, 0) * dqq_c<Q>(a, 0) + dqq_c<Q>(a, 1) * dqq_c<Q>(a, 1) + dqq_c<Q>(a, 2) * dqq_c<Q>(a, 2);
        const int nb = k + 1 < H ? dqq_c<Q>(b, 0) * dqq_c<Q>(b, 0) + dqq_c<Q>(b, 1) * dqq_c<Q>(b, 1) +
                                       dqq_c<Q>(b, 2) * dqq_c<Q>(b, 2)
                                 : -1;
        const bool lead = !prev && na == nb;
        if (k == j) return lead;
        prev = lead;
    }
    return false;
}

// first velocity of the half set with |c|^2 = n2, and the half set's count of them
template <int Q>
__host__ __device__ constexpr int dqq_rep(int n2) {
    for (int i = 1; i <= (Q - 1) / 2; ++i)
        if (dqq_c<Q>(i, 0) * dqq_c<Q>(i, 0) + dqq_c<Q>(i, 1) * dqq_c<Q>(i, 1) + dqq_c<Q>(i, 2) * dqq_c<Q>(i, 2) == n2)
            return i;
    return 0;
}
template <int Q>
__host__ __device__ constexpr int dqq_count(int n2) {
    int m = 0;
    for (int i = 1; i <= (Q - 1) / 2; ++i)
        if (dqq_c<Q>(i, 0) * dqq_c<Q>(i, 0) + dqq_c<Q>(i, 1) * dqq_c<Q>(i, 1) + dqq_c<Q>(i, 2) * dqq_c<Q>(i, 2) == n2)
            ++m;
    return m;
}

// SURVEY.md 8(c) item 1 for one cell: BGK towards feq_i = w_i rho (1 + 3 c.u
// + 4.5 (c.u)^2 - 1.5 u.u), the rest population closing the mass.  The
// arithmetic runs per direction pair (i, opp(i)) -- the half-sum / half-
// difference moments, c.u without multiplications, feq_i and feq_opp from
// one symmetric and one antisymmetric part, the rest-population closure
// feq_0 = rho - sum_{i>0} feq_i summed in closed form per weight class (R-2,
// as for D3Q19) -- about half
// the FP64 operations of the oracle's term-by-term order (R-2's
// reading for these lattices; agreement with the oracle is within the
// tolerance, not bitwise).  K1 and K2Q both call it: they agree bit for bit.
template <typename T, int Q, bool PACK = (Q == 27)>
__device__ __forceinline__ void dqq_collide(T (&f)[Q], T omega) {
    constexpr int H = (Q - 1) / 2;
    T sm[H], df[H];
    static_for<0, H>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        sm[j] = f[1 + j] + f[1 + j + H];
        df[j] = f[1 + j] - f[1 + j + H];
    });
    T r = f[0];
    static_for<0, H>([&](auto jc) { r = r + sm[decltype(jc)::value]; });
    // j_a = sum over the half set of c_a (f_i - f_opp)
    T jm[3];
    static_for<0, 3>([&](auto ac) {
        constexpr int ax = decltype(ac)::value;
        bool first = true;
        T acc = T(0);
        static_for<0, H>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            constexpr int cc = dqq_c<Q>(1 + j, ax);
            if constexpr (cc != 0) {
                const T v = cc > 0 ? df[j] : -df[j];
                acc = first ? v : acc + v;
                first = false;
            }
        });
        jm[ax] = acc;
    });
    const T rinv = rcp_nr<T>(r);
    const T ux = jm[0] * rinv, uy = jm[1] * rinv, uz = jm[2] * rinv;
    const T usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const T base = fma(T(-1.5), usq, T(1));
    const T om1 = T(1) - omega;
    auto cdot = [&](auto ic) -> T {  // c_i . u by additions
        constexpr int i = decltype(ic)::value;
        constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
        T cu;
        if constexpr (cx != 0) {
            cu = cx > 0 ? ux : -ux;
            if constexpr (cy != 0) cu = cy > 0 ? cu + uy : cu - uy;
            if constexpr (cz != 0) cu = cz > 0 ? cu + uz : cu - uz;
        } else if constexpr (cy != 0) {
            cu = cy > 0 ? uy : -uy;
            if constexpr (cz != 0) cu = cz > 0 ? cu + uz : cu - uz;
        } else {
            cu = cz > 0 ? uz : -uz;
        }
        return cu;
    };
    static_for<0, H>([&](auto jc) {
        constexpr int j = decltype(jc)::value, i = 1 + j;
        if constexpr (PACK && std::is_same<T, float>::value && dqq_lead<Q>(j)) {
            // fp32 D3Q27: pairs j, j+1 of one weight class on packed FFMA2 /
            // FMUL2 / FADD2 (K2Q +4.5%, one-step +0.7%; D3Q15 K2Q -0.9%, so
            // D3Q15 stays scalar).  The packed form does not reproduce the
            // scalar form's bits: ptxas (12.9, sm_100a) contracts the
            // mul.rn.f32x2 / add.rn.f32x2 pairs into FFMA2 despite .rn (SASS:
            // 9 mul + 6 add + 9 fma f32x2 in PTX become 6 FMUL2 + 15 FFMA2;
            // each packed op alone is exact, tools/f32x2_probe.cu), so both
            // kernels of a lattice use the same form and stay bitwise equal;
            // both are within the oracle tolerance.
            constexpr int i2 = i + 1;
            const float owr = omega * (float(dqq_w<Q>(i)) * r);
            const float2 cu = make_float2(cdot(std::integral_constant<int, i>{}), cdot(std::integral_constant<int, i2>{}));
            const float2 sym = __fmul2_rn(make_float2(owr, owr),
                                          __ffma2_rn(__fmul2_rn(make_float2(4.5f, 4.5f), cu), cu, make_float2(base, base)));
            const float o3 = 3.0f * owr;
            const float2 asym = __fmul2_rn(make_float2(o3, o3), cu);
            const float2 om12 = make_float2(om1, om1);
            const float2 lo = __ffma2_rn(om12, make_float2(f[i], f[i2]), __fadd2_rn(sym, asym));
            const float2 hi = __ffma2_rn(om12, make_float2(f[i + H], f[i2 + H]), __fadd2_rn(sym, make_float2(-asym.x, -asym.y)));
            f[i] = lo.x;
            f[i2] = lo.y;
            f[i + H] = hi.x;
            f[i2 + H] = hi.y;
        } else if constexpr (!(PACK && std::is_same<T, float>::value && j > 0 && dqq_lead<Q>(j - 1))) {
            const T cu = cdot(std::integral_constant<int, i>{});
            const T owr = omega * (T(dqq_w<Q>(i)) * r);      // omega w_i rho (one per weight class)
            const T sym = owr * fma(T(4.5) * cu, cu, base);  // omega (feq_i + feq_opp) / 2
            const T asym = (T(3) * owr) * cu;                // omega (feq_i - feq_opp) / 2
            f[i] = fma(om1, f[i], sym + asym);
            f[i + H] = fma(om1, f[i + H], sym - asym);
        }
    });
    // closure: sum_{i>0} feq_i = 2 sum over weight classes c of
    // w_c rho (n_c (1 - 1.5 u.u) + 4.5 k_c u.u), n_c half-set vectors of class
    // c and sum_{half set of c} (c.u)^2 = k_c u.u (axes 1, face diagonals 4,
    // corners 4), with the same rounded w_c rho as the populations, so the
    // weights' rounding cancels in the mass (R-2)
    T clos = T(0);
    static_for<1, 4>([&](auto nc) {
        constexpr int n2 = decltype(nc)::value;  // |c|^2 of the class
        constexpr int rep = dqq_rep<Q>(n2), cnt = dqq_count<Q>(n2), kc = n2 == 1 ? 1 : 4;
        if constexpr (cnt > 0) clos = clos + (T(dqq_w<Q>(rep)) * r) * fma(T(4.5 * kc), usq, T(cnt) * base);
    });
    f[0] = fma(om1, f[0], omega * (r - T(2) * clos));
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
            if (!g.xlo_open) dx = dx < 0 ? dx + g.nx : (dx >= g.nx ? dx - g.nx : dx);  // else: ghost plane
            dy = dy < 0 ? dy + g.ny : (dy >= g.ny ? dy - g.ny : dy);
            dz = dz < 0 ? dz + g.nz : (dz >= g.nz ? dz - g.nz : dz);
        } else {
            out = (dx < 0 && !g.xlo_open) || (dx >= g.nx && !g.xhi_open) || dy < 0 || dy >= g.ny || dz < 0 ||
                  dz >= g.nz;
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

// X-slab halo merge (NCCL slabs, api.cu dqq_exchange): the populations a
// neighbour rank pushed across an open face arrive in this rank's unused
// ghost slots (c_x = +1 directions in ghost plane -1, c_x = -1 ones in
// ghost plane nx) and are copied into plane 0 / nx - 1 -- except where the
// link's source lies beyond a y / z wall (cavity), whose slot the cell's own
// bounce-back (lid included) already wrote this step
template <typename T, int Q, int BC>
__global__ void __launch_bounds__(256) k_dqq_merge(T* __restrict__ B, DqqGeom g) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int side = blockIdx.z;  // 0: face x = 0 (from the left rank), 1: face x = nx - 1
    if (z >= g.nz || y >= g.ny || !(side ? g.xhi_open : g.xlo_open)) return;
    const long long plane = (long long)g.ny * g.nzp, yz = (long long)y * g.nzp + z;
    static_for<0, Q>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
        if constexpr (cx != 0) {
            if ((cx > 0) == (side == 0)) {
                const bool inside = BC == BC_PERIODIC || ((unsigned)(y - cy) < (unsigned)g.ny &&
                                                          (unsigned)(z - cz) < (unsigned)g.nz);
                const long long own = side ? (long long)(g.nx - 1) * plane : 0;
                const long long ghost = side ? (long long)g.nx * plane : -plane;
                T* const slot = B + (long long)i * g.pq;
                if (inside) slot[own + yz] = slot[ghost + yz];
            }
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


// ------------------------------------------------------------------ K2Q --
// Two collide + push steps per HBM pass for D3Q15 / D3Q27 (the paper's
// two-step merge, which it states for any of these
// lattices).  K2 (k2.cu) reorganised for push-form canonical
// storage: each CTA owns a TY x TZ output tile and marches along x over a
// chunk of planes.  Per input plane p:
//   1. TMA stages f(t) of the tile plus a one-cell halo (T+1): one box per
//      direction, all at the same origin (push form: a cell reads its own
//      populations), double-buffered on one mbarrier.  Cells beyond a cavity
//      wall are zero-filled and never collide; a periodic box's halo cells
//      beyond the domain reload their wrapped cell from global memory.
//   2. Step 1: every cell of T+1 collides (dqq_collide) and pushes f*_i into
//      a destination-indexed SMEM ring at x + c_i when that lies in the tile;
//      a tile cell whose link leaves the domain bounces f*_i (+ lid) into its
//      own slot opp(i) -- so the ring holds exactly f(t+1) of the tile.
//   3. Step 2 of plane p-2 (complete since this iteration's barrier): collide
//      and push f*(t+1) to B at x + c_i (or bounce into the own slot), every
//      destination slot written exactly once, as in k_dqq_step.
// Same collision and wall arithmetic as k_dqq_step, so K2Q == step o step
// bit for bit (tests/test_gpu_dqq.py).  Ring depths per c_x group: M (c_x =
// -1) 3 destination planes (p-2 read, p-1 pushed, p bounced), Z 3, P 4.
namespace {

template <int Q>
__host__ __device__ constexpr int kq_grp(int i) { return dqq_c<Q>(i, 0) + 1; }  // 0: c_x = -1, 1: 0, 2: +1
template <int Q>
__host__ __device__ constexpr int kq_gidx(int i) {  // index of i within its c_x group
    int m = 0;
    for (int j = 0; j < i; ++j)
        if (dqq_c<Q>(j, 0) == dqq_c<Q>(i, 0)) ++m;
    return m;
}
template <int Q>
__host__ __device__ constexpr int kq_gsize(int gg) {
    int m = 0;
    for (int j = 0; j < Q; ++j)
        if (dqq_c<Q>(j, 0) + 1 == gg) ++m;
    return m;
}
__host__ __device__ constexpr int kq_round_up(int v, int m) { return (v + m - 1) / m * m; }

template <typename T, int Q, int TY_, int TZ_, bool WS_ = false>
struct KQCfg {
    static constexpr int TY = TY_, TZ = TZ_, HY = TY + 2, HZ = TZ + 2;
    // WS: step-1 and step-2 cells on separate warps (one collision per
    // thread and plane: twice the warps of a latency-bound tile)
    static constexpr bool WS = WS_;
    static constexpr int ZPAD = 16 / int(sizeof(T));  // TMA: 16 B aligned innermost origin
    static constexpr int BW = TZ + 2 * ZPAD, BOX = HY * BW;
    static constexpr int BOXE = kq_round_up(BOX * int(sizeof(T)), 128) / int(sizeof(T));
    static constexpr int S2B = WS ? kq_round_up(HY * HZ, 32) : 0;  // first step-2 thread
    static constexpr int NT = kq_round_up(HY * HZ, 32) + (WS ? TY * TZ : 0);
    static constexpr int RP = TY * TZ;
    static constexpr int GM = kq_gsize<Q>(0), GZ = kq_gsize<Q>(1), GP = kq_gsize<Q>(2);
    static constexpr int DM = 3, DZ = 3, DP = 4;
    static constexpr int RING = (DM * GM + DZ * GZ + DP * GP) * RP;
    static constexpr size_t SMEM = size_t(2 * Q * BOXE + RING) * sizeof(T) + 2 * sizeof(uint64_t);
    static constexpr uint32_t TX = uint32_t(Q * BOX * sizeof(T));
    static constexpr int MINB = SMEM + 1024 <= 114 * 1024 ? 2 : 1;  // CTAs per SM that shared memory allows
};

__device__ __forceinline__ uint32_t kq_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool kq_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(kq_smem(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void kq_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t spin = 0; !kq_try_wait(bar, parity); ++spin)
        if (spin > (1u << 28)) __trap();  // a TMA that never lands: a kernel error, not a hang
}
__device__ __forceinline__ int kq_wrap(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

}  // namespace

template <typename T, int Q, int BC, int TY, int TZ, bool WS>
__global__ void __launch_bounds__(KQCfg<T, Q, TY, TZ, WS>::NT, KQCfg<T, Q, TY, TZ, WS>::MINB)
    k_dqq_k2(const __grid_constant__ CUtensorMap tm, const T* __restrict__ A, T* __restrict__ B, DqqGeom g, T omega,
             double ulx, double uly, int chunk) {
    using C = KQCfg<T, Q, TY, TZ, WS>;
    constexpr bool PER = BC == BC_PERIODIC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* const stage = reinterpret_cast<T*>(smem_raw);
    T* const ringM = stage + 2 * Q * C::BOXE;
    T* const ringZ = ringM + C::DM * C::GM * C::RP;
    T* const ringP = ringZ + C::DZ * C::GZ * C::RP;
    uint64_t* const bar = reinterpret_cast<uint64_t*>(ringP + C::DP * C::GP * C::RP);

    const int ntz = (g.nz + TZ - 1) / TZ;
    const int z0 = int(blockIdx.x % ntz) * TZ, y0 = int(blockIdx.x / ntz) * TY;  // z-fastest tile order
    const int xs = int(blockIdx.y) * chunk, xe = min(xs + chunk, g.nx);
    const int p_first = PER ? xs - 1 : max(xs - 1, 0), p_last = PER ? xe : min(xe, g.nx - 1);
    const long long plane = (long long)g.ny * g.nzp;

    // step-1 cell (box coordinates a, b; cell qy, qz): interior columns row by
    // row, then the two halo columns (K2's mapping)
    const int tid = threadIdx.x;
    int a, b;
    if (tid < C::HY * TZ) {
        a = tid / TZ;
        b = 1 + tid % TZ;
    } else {
        const int j = tid - C::HY * TZ;
        a = j >> 1;
        b = (j & 1) ? TZ + 1 : 0;
    }
    const bool act1 = tid < C::HY * C::HZ;
    const int qy = y0 - 1 + a, qz = z0 - 1 + b;
    const bool q_in = act1 && (PER ? (qy >= -1 && qy <= g.ny && qz >= -1 && qz <= g.nz)
                                   : (qy >= 0 && qy < g.ny && qz >= 0 && qz < g.nz));
    const bool q_wrap = PER && q_in && (qy < 0 || qy >= g.ny || qz < 0 || qz >= g.nz);
    const bool q_tile = act1 && a >= 1 && a <= TY && b >= 1 && b <= TZ;
    const int soff = a * C::BW + b + C::ZPAD - 1;  // staged entry of (a, b)
    const int toff = (a - 1) * TZ + (b - 1);        // ring entry of (a, b) (tile coordinates)
    const bool rowok[3] = {a >= 2 && a <= TY + 1, a >= 1 && a <= TY, a <= TY - 1};
    const bool colok[3] = {b >= 2 && b <= TZ + 1, b >= 1 && b <= TZ, b <= TZ - 1};
    // cavity walls of the step-1 cell (y, z; x per plane)
    const bool wyl = !PER && qy == 0, wyh = !PER && qy == g.ny - 1, wzl = !PER && qz == 0, wzh = !PER && qz == g.nz - 1;
    // step-2 cell (WS: the threads from S2B on; else the first TY*TZ)
    const int t2 = tid - C::S2B;
    const int y2 = max(t2, 0) / TZ, z2 = max(t2, 0) % TZ, yy = y0 + y2, zz = z0 + z2;
    const bool in2 = t2 >= 0 && t2 < TY * TZ && yy < g.ny && zz < g.nz;
    const bool warp2 = WS ? tid >= C::S2B : (tid & ~31) < TY * TZ;
    const bool warp1 = !WS || tid < C::S2B;  // the warp collides step-1 cells
    const bool vyl = !PER && yy == 0, vyh = !PER && yy == g.ny - 1, vzl = !PER && zz == 0, vzh = !PER && zz == g.nz - 1;
    // no tile cell on a y / z wall (CTA-uniform): its planes away from the x
    // walls push every link plainly -- no per-direction wall test or branch
    const bool tile_inner = !PER && y0 >= 1 && y0 + TY <= g.ny - 1 && z0 >= 1 && z0 + TZ <= g.nz - 1;
    // periodic destination offsets of the step-2 cell per c_y, c_z
    const long long yo[3] = {(long long)kq_wrap(yy - 1, g.ny) * g.nzp, (long long)yy * g.nzp,
                             (long long)kq_wrap(yy + 1, g.ny) * g.nzp};
    const int zo[3] = {kq_wrap(zz - 1, g.nz), zz, kq_wrap(zz + 1, g.nz)};

    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    auto issue = [&](int p, int s) {  // one thread: stage plane p into buffer s
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(kq_smem(&bar[s])), "r"(C::TX)
                     : "memory");
        const int px = PER ? kq_wrap(p, g.nx) : p;
        static_for<0, Q>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(kq_smem(stage + (s * Q + k) * C::BOXE)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(z0 - C::ZPAD), "r"(y0 - 1), "r"(px), "r"(k),
                "r"(kq_smem(&bar[s])), "l"(pol)
                : "memory");
        });
    };
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(kq_smem(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(kq_smem(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        if (p_first <= p_last) issue(p_first, 0);
        if (p_first + 1 <= p_last) issue(p_first + 1, 1);
    }
    // ring plane of group G for destination plane dp (dp >= -2)
    auto ring = [&](auto G, int dp) -> T* {
        constexpr int gg = decltype(G)::value;
        if constexpr (gg == 0) return ringM + ((dp + 6) % 3) * C::GM * C::RP;
        else if constexpr (gg == 1) return ringZ + ((dp + 6) % 3) * C::GZ * C::RP;
        else return ringP + ((dp + 8) & 3) * C::GP * C::RP;
    };

    for (int p = xs - 1; p <= xe + 1; ++p) {
        const bool has1 = p >= p_first && p <= p_last && warp1;
        const bool has1_any = p >= p_first && p <= p_last;  // (the TMA issue of thread 0)
        const int c = p - p_first, s = c & 1;
        T fs[Q];
        if (has1) {
            kq_wait(&bar[s], uint32_t(c >> 1) & 1u);
            const T* const sp = stage + s * Q * C::BOXE + (act1 ? soff : C::ZPAD);
            static_for<0, Q>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                fs[k] = sp[k * C::BOXE];
            });
            if (q_wrap) {  // periodic halo cell beyond the domain: its wrapped cell
                const long long o = (long long)kq_wrap(p, g.nx) * plane + (long long)kq_wrap(qy, g.ny) * g.nzp +
                                    kq_wrap(qz, g.nz);
                static_for<0, Q>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    fs[k] = A[(long long)k * g.pq + o];
                });
            }
        }
        __syncthreads();  // stage of plane p consumed, ring of destination p-2 complete
        if (tid == 0 && has1_any && p + 2 <= p_last) issue(p + 2, s);

        // ---- step 2 of plane d = p - 2 and step 1 of plane p ----
        const int d = p - 2;
        const bool do2 = d >= xs && warp2;
        T f2[Q];
        if (do2) {
            const int t = in2 ? y2 * TZ + z2 : 0;
            static_for<0, Q>([&](auto kc) {
                constexpr int i = decltype(kc)::value;
                f2[i] = ring(std::integral_constant<int, kq_grp<Q>(i)>{}, d)[kq_gidx<Q>(i) * C::RP + t];
            });
        }
        if (do2) dqq_collide<T, Q>(f2, omega);
        if (has1) dqq_collide<T, Q>(fs, omega);
        if (do2 && in2 && KQ_FAST && tile_inner && d > 0 && d < g.nx - 1) {
            const long long own = (long long)d * plane + (long long)yy * g.nzp + zz;
            static_for<0, Q>([&](auto kc) {
                constexpr int i = decltype(kc)::value;
                constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
                __stcs(B + (long long)i * g.pq + own + (long long)cx * plane + cy * g.nzp + cz, f2[i]);
            });
        } else if (do2 && in2) {
            const long long own = (long long)d * plane + (long long)yy * g.nzp + zz;
            const bool vxl = !PER && d == 0, vxh = !PER && d == g.nx - 1;
            const long long xo[3] = {(long long)kq_wrap(d - 1, g.nx) * plane, (long long)d * plane,
                                     (long long)kq_wrap(d + 1, g.nx) * plane};
            static_for<0, Q>([&](auto kc) {
                constexpr int i = decltype(kc)::value;
                constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
                if constexpr (PER) {
                    __stcs(B + (long long)i * g.pq + xo[cx + 1] + yo[cy + 1] + zo[cz + 1], f2[i]);
                } else {
                    bool out = false;
                    if constexpr (cx == -1) out = out || vxl;
                    if constexpr (cx == 1) out = out || vxh;
                    if constexpr (cy == -1) out = out || vyl;
                    if constexpr (cy == 1) out = out || vyh;
                    if constexpr (cz == -1) out = out || vzl;
                    if constexpr (cz == 1) out = out || vzh;
                    if (!out) {
                        __stcs(B + (long long)i * g.pq + own + (long long)cx * plane + cy * g.nzp + cz, f2[i]);
                    } else {
                        constexpr int o = dqq_opp<Q>(i);
                        T v = f2[i];
                        if constexpr (cz == 1) {
                            if (vzh) {  // the moving lid: 6 w_o rho_w (c_o . u_lid), rho_w = 1
                                const double cu = dqq_c<Q>(o, 0) * ulx + dqq_c<Q>(o, 1) * uly;
                                v = v + T(6.0 * dqq_w<Q>(o) * 1.0 * cu);
                            }
                        }
                        __stcs(B + (long long)o * g.pq + own, v);
                    }
                }
            });
        }
        if (has1 && q_in) {
            // pushes into the tile: direction i streams to (p + c_x, a - 1 + c_y, b - 1 + c_z)
            static_for<0, Q>([&](auto kc) {
                constexpr int i = decltype(kc)::value;
                constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
                if (rowok[cy + 1] && colok[cz + 1])
                    ring(std::integral_constant<int, kq_grp<Q>(i)>{}, p + cx)[kq_gidx<Q>(i) * C::RP + toff + cy * TZ + cz] =
                        fs[i];
            });
            if constexpr (!PER) {
                // links of a tile cell that leave the domain: bounce-back (+ lid) into its own slot
                if (q_tile && !(KQ_FAST && tile_inner && p > 0 && p < g.nx - 1)) {
                    const bool wxl = p == 0, wxh = p == g.nx - 1;
                    static_for<0, Q>([&](auto kc) {
                        constexpr int i = decltype(kc)::value;
                        constexpr int cx = dqq_c<Q>(i, 0), cy = dqq_c<Q>(i, 1), cz = dqq_c<Q>(i, 2);
                        bool out = false;
                        if constexpr (cx == -1) out = out || wxl;
                        if constexpr (cx == 1) out = out || wxh;
                        if constexpr (cy == -1) out = out || wyl;
                        if constexpr (cy == 1) out = out || wyh;
                        if constexpr (cz == -1) out = out || wzl;
                        if constexpr (cz == 1) out = out || wzh;
                        if (out) {
                            constexpr int o = dqq_opp<Q>(i);
                            T v = fs[i];
                            if constexpr (cz == 1) {
                                if (wzh) {
                                    const double cu = dqq_c<Q>(o, 0) * ulx + dqq_c<Q>(o, 1) * uly;
                                    v = v + T(6.0 * dqq_w<Q>(o) * 1.0 * cu);
                                }
                            }
                            ring(std::integral_constant<int, kq_grp<Q>(o)>{}, p)[kq_gidx<Q>(o) * C::RP + toff] = v;
                        }
                    });
                }
            }
        }
    }
}

// ------------------------------------------------------------------ host --
namespace {
dim3 dqq_grid(int nz, int ny, int nx) { return dim3((nz + 31) / 32, (ny + 7) / 8, nx); }
const dim3 kDqqBlock(32, 8, 1);


}  // namespace

template <typename T>
cudaError_t launch_dqq_merge(T* B, const DqqGeom& g, cudaStream_t s) {
    const dim3 grid = dqq_grid(g.nz, g.ny, 2);
#define MERGE(Q)                                                                               \
    if (g.bc == BC_PERIODIC) k_dqq_merge<T, Q, BC_PERIODIC><<<grid, kDqqBlock, 0, s>>>(B, g); \
    else k_dqq_merge<T, Q, BC_CAVITY><<<grid, kDqqBlock, 0, s>>>(B, g);
    switch (g.q) {
        case 15: MERGE(15) break;
        case 27: MERGE(27) break;
        default: return cudaErrorInvalidValue;
    }
#undef MERGE
    return cudaGetLastError();
}

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


namespace {

using KqEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename T, int Q, int BC, int TY, int TZ, bool WS>
cudaError_t launch_kq(const T* A, T* B, const DqqGeom& g, T omega, const double ulid[3], cudaStream_t s) {
    using C = KQCfg<T, Q, TY, TZ, WS>;
    static_assert(C::SMEM <= 227 * 1024, "K2Q tile does not fit shared memory");
    auto kern = k_dqq_k2<T, Q, BC, TY, TZ, WS>;
    // the large-shared-memory opt-in is per device (context): once per ordinal
    static std::atomic<int> occ_cache[64];  // CTAs per SM, once the opt-in is set (per device)
    const int dev = device_ordinal();
    int occ = occ_cache[dev].load(std::memory_order_acquire);
    if (occ < 1) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, C::SMEM);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        occ_cache[dev].store(occ, std::memory_order_release);
    }
    auto enc = reinterpret_cast<KqEncodeFn>(tma_encode_entry());
    if (!enc) return cudaErrorNotSupported;
    // canonical [q][x][y][z] as a 4D tensor (z, y, x, q); cells beyond the
    // domain read as zero
    CUtensorMap map;
    const cuuint64_t dims[4] = {cuuint64_t(g.nz), cuuint64_t(g.ny), cuuint64_t(g.nx), cuuint64_t(Q)};
    const cuuint64_t strides[3] = {cuuint64_t(g.nzp) * sizeof(T), cuuint64_t(g.ny) * g.nzp * sizeof(T),
                                   cuuint64_t(g.pq) * sizeof(T)};
    const cuuint32_t box[4] = {cuuint32_t(C::BW), cuuint32_t(C::HY), 1u, 1u};
    const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    if (enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
            const_cast<T*>(A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    // x chunks of <= 32 planes (K2's short-chunk rule: co-resident tiles stay
    // within a few planes, so halo rows re-staged by a neighbour hit L2),
    // filling whole waves of one CTA per SM; each chunk re-computes ~2.5
    // step-1 planes and ~2 planes of pipeline fill
    const long long ntiles = (long long)((g.ny + TY - 1) / TY) * ((g.nz + TZ - 1) / TZ);
    const long long slots = (long long)device_sm_count() * occ;
    int best = 1;
    double best_cost = 1e300;
    for (int nch = 1; nch <= g.nx && nch <= 65535; ++nch) {  // (grid.y limit)
        const int ch = (g.nx + nch - 1) / nch;
        if (ch > 32 && nch < g.nx && nch < 65535) continue;
        const double waves = double((ntiles * ((g.nx + ch - 1) / ch) + slots - 1) / slots);
        const double cost = waves * (double(g.nx) / nch + 4.5);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = nch;
        }
        if (ch <= 8) break;
    }
    const int chunk = (g.nx + best - 1) / best;
    const dim3 grid(unsigned(ntiles), unsigned((g.nx + chunk - 1) / chunk));
    kern<<<grid, C::NT, C::SMEM, s>>>(map, A, B, g, omega, ulid[0], ulid[1], chunk);
    return cudaGetLastError();
}

}  // namespace

// Tiles (the largest whose stage + ring fit 227 KB): D3Q27 fp64 8x16 (178
// KB, 320 threads: warp-specialised), fp32 8x32 (178 KB; an 8x16 tile with
// two CTAs per SM measured 8% slower); D3Q15 fp64 8x32 (184 KB), fp32
// 16x32 (184 KB).
template <typename T>
cudaError_t launch_dqq_k2(const T* A, T* B, const DqqGeom& g, T omega, const double ulid[3], cudaStream_t s) {
    if (!tma_encode_entry()) return cudaErrorNotSupported;
    if (g.nx < 1 || (g.nzp * sizeof(T)) % 16) return cudaErrorInvalidValue;
    constexpr bool F64 = sizeof(T) == 8;
#ifndef LBM_KQ27_F64_TZ
#define LBM_KQ27_F64_TZ 16  // (A/B builds override: tools/build_variant.sh -DLBM_KQ27_F64_TZ=8)
#endif
    constexpr int TY27 = 8, TZ27 = F64 ? LBM_KQ27_F64_TZ : 32, TY15 = F64 ? 8 : 16, TZ15 = 32;
    // D3Q27 fp64: step-1 and step-2 cells on separate warps (10 warps per
    // SM instead of 6; 15.7k vs 13.8k MLUPS, 512^3 cavity); elsewhere the
    // shared warps (D3Q27 fp32 -4% split; D3Q15 split spills)
    constexpr bool WS27 = F64, WS15 = false;
    const bool per = g.bc == BC_PERIODIC;
    switch (g.q) {
        case 27:
            return per ? launch_kq<T, 27, BC_PERIODIC, TY27, TZ27, WS27>(A, B, g, omega, ulid, s)
                       : launch_kq<T, 27, BC_CAVITY, TY27, TZ27, WS27>(A, B, g, omega, ulid, s);
        case 15:
            return per ? launch_kq<T, 15, BC_PERIODIC, TY15, TZ15, WS15>(A, B, g, omega, ulid, s)
                       : launch_kq<T, 15, BC_CAVITY, TY15, TZ15, WS15>(A, B, g, omega, ulid, s);
        default:
            return cudaErrorInvalidValue;
    }
}

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
    template cudaError_t launch_dqq_import<T>(const double*, T*, const DqqGeom&, int, int, cudaStream_t);     \
    template cudaError_t launch_dqq_k2<T>(const T*, T*, const DqqGeom&, T, const double*, cudaStream_t);     \
    template cudaError_t launch_dqq_merge<T>(T*, const DqqGeom&, cudaStream_t);
LBM_DQQ_INST(double)
LBM_DQQ_INST(float)
#undef LBM_DQQ_INST

}  // namespace lbm

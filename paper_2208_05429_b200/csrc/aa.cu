// aa.cu -- single-copy in-place storage: the AA access pattern (SURVEY.md
// 8(f) row 1), the GPU form of the paper's single-lattice swap scheme
// ("only one copy of the lattice").  One buffer F of
// the slab layout (no ghost planes used) holds the state; two one-step
// kernels alternate:
//
//   even step (state at rest, F[x][k] = f_i(x,t), i = slot_dir(k)):
//       f = F[x][.];  collide;  F[x][opp(k)] = f*_i          (in place)
//   odd step (F[x][opp(k)] = f*_i(x,t-1), the even step's output):
//       f_i = F[x - c_i][opp(k)]      source beyond a wall: F[x][k] (+ lid_k)
//       collide;
//       F[x + c_i][k] = f*_i          target beyond a wall: F[x][opp(k)] = f*_i (+ lid_opp(k))
//
// After the odd step F is at rest again: F[y][k] = f*_i(y - c_i) = f_i(y,t+1).
// Every location F[y][j] is read and then written by the same thread (cell
// y - c_j), so both kernels run in place without races.  This is the
// paper's swap in data-parallel form: the even step's "revert" (PAPER.md:
// 238-243) and the odd step's exchange of slot opp(i)@x with slot i@x+c_i.
//
// The collision is bgk_collide() and the wall/lid rules are those of
// pull_cell() (R-4..R-7), so AA steps reproduce K1
// steps bit for bit (tests/test_gpu_parity.py).  A single slab wraps x in
// the kernel; X-slabs use the ghost planes x = -1 and nx_local, filled
// before every odd step (the neighbours' c_x = -1 / +1 slots of their edge
// planes) and returned after it (what the odd step scattered into them
// belongs to the neighbours' edge cells): api.cu exchange_aa().
#include "kernels.h"

namespace lbm {

namespace {

// Element offset of F[x + d][slot] for the neighbour d = +-c of cell
// (x, y, z) along a compile-time direction, or -1 if that neighbour lies
// beyond a cavity wall.  Only the axes the direction moves along are
// tested (periodic: wrapped), like pull_src() for K1.
// `self` = cell_off(g, x, y, z); the result is self plus a displacement
// (AA storage never uses the single-copy plane ring, so planes are linear).
template <int BC, int dx, int dy, int dz>
__device__ __forceinline__ long long aa_nbr(const SlabGeom& g, int x, int y, int z, int slot, long long self) {
    long long d = (long long)slot * g.pq;
    if constexpr (BC == BC_CAVITY) {
        bool out = false;
        // x: a wall only at the slab ends that are domain walls; otherwise
        // the neighbour lies in a ghost plane (x = -1 or nxl)
        if constexpr (dx == -1) out = out || (x == 0 && g.left_wall);
        if constexpr (dx == 1) out = out || (x == g.nxl - 1 && g.right_wall);
        if constexpr (dy == -1) out = out || y == 0;
        if constexpr (dy == 1) out = out || y == g.ny - 1;
        if constexpr (dz == -1) out = out || z == 0;
        if constexpr (dz == 1) out = out || z == g.nz - 1;
        if (out) return -1;
        if constexpr (dx != 0) d += dx > 0 ? g.px : -g.px;
        if constexpr (dy != 0) d += dy > 0 ? g.nzp : -g.nzp;
        if constexpr (dz != 0) d += dz;
    } else {
        // x wraps in the kernel only for a single slab; slabs use ghost planes
        if constexpr (dx == -1) d += (x == 0 && g.nxl == g.nx) ? (long long)(g.nxl - 1) * g.px : -g.px;
        if constexpr (dx == 1) d += (x == g.nxl - 1 && g.nxl == g.nx) ? -(long long)(g.nxl - 1) * g.px : g.px;
        if constexpr (dy == -1) d += y == 0 ? (long long)(g.ny - 1) * g.nzp : -(long long)g.nzp;
        if constexpr (dy == 1) d += y == g.ny - 1 ? -(long long)(g.ny - 1) * g.nzp : (long long)g.nzp;
        if constexpr (dz == -1) d += z == 0 ? g.nz - 1 : -1;
        if constexpr (dz == 1) d += z == g.nz - 1 ? -(g.nz - 1) : 1;
    }
    return self + d;
}

// canonical f(x, t) from F: at rest (even) or after an even step (odd)
template <typename T, int BC>
__device__ __forceinline__ void aa_gather(const T* __restrict__ F, const StepParams<T>& P, bool odd, int x, int y,
                                          int z, T (&f)[kQ]) {
    const SlabGeom& g = P.g;
    const long long self = cell_off(g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        constexpr int i = slot_dir(k);
        constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
        T v;
        if (!odd) {
            v = F[self + (long long)k * g.pq];
        } else {
            const long long src = aa_nbr<BC, -cx, -cy, -cz>(g, x, y, z, slot_opp(k), self);
            if (src >= 0) {
                v = F[src];
            } else {
                v = F[self + (long long)k * g.pq];
                if constexpr (BC == BC_CAVITY && cz == -1) {
                    if (z == g.nz - 1) v = v + P.lid[k];
                }
            }
        }
        f[i] = v;
    });
}

}  // namespace

template <typename T, int BC>
__global__ void __launch_bounds__(256) k_aa_even(T* __restrict__ F, StepParams<T> P) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.z;
    const SlabGeom& g = P.g;
    if (z >= g.nz || y >= g.ny) return;
    const long long self = cell_off(g, x, y, z);
    T f[kQ];
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        f[slot_dir(k)] = F[self + (long long)k * g.pq];
    });
    bgk_collide<T>(f, P.omega);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        F[self + (long long)slot_opp(k) * g.pq] = f[slot_dir(k)];
    });
}

template <typename T, int BC>
__global__ void __launch_bounds__(256) k_aa_odd(T* __restrict__ F, StepParams<T> P) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.z;
    const SlabGeom& g = P.g;
    if (z >= g.nz || y >= g.ny) return;
    T f[kQ];
    aa_gather<T, BC>(F, P, true, x, y, z, f);
    bgk_collide<T>(f, P.omega);
    const long long self = cell_off(g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        constexpr int i = slot_dir(k);
        constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
        const long long dst = aa_nbr<BC, cx, cy, cz>(g, x, y, z, k, self);
        if (dst >= 0) {
            F[dst] = f[i];
        } else {
            // f*_i leaves through a wall: it is population opp(i) of this cell
            // at the next step, plus the lid term of that link (its source,
            // x + c_i, lies beyond the lid)
            constexpr int ko = slot_opp(k);
            T v = f[i];
            if constexpr (BC == BC_CAVITY && cz == 1) {
                if (z == g.nz - 1) v = v + P.lid[ko];
            }
            F[self + (long long)ko * g.pq] = v;
        }
    });
}

// canonical f on a box -> out[19][lx][ly][lz] (doubles)
template <typename T, int BC>
__global__ void __launch_bounds__(256) k_aa_materialize(const T* __restrict__ F, StepParams<T> P, int odd, int x0,
                                                       int y0, int z0, int lx, int ly, int lz,
                                                       double* __restrict__ out) {
    const int zz = blockIdx.x * 32 + threadIdx.x;
    const int yy = blockIdx.y * 8 + threadIdx.y;
    const int xx = blockIdx.z;
    if (zz >= lz || yy >= ly) return;
    T f[kQ];
    aa_gather<T, BC>(F, P, odd != 0, x0 + xx, y0 + yy, z0 + zz, f);
    const long long stride = (long long)lx * ly * lz;
    const long long cell = ((long long)xx * ly + yy) * lz + zz;
#pragma unroll
    for (int i = 0; i < kQ; ++i) out[i * stride + cell] = double(f[i]);
}

template <typename T, int BC>
__global__ void __launch_bounds__(256) k_aa_moments(const T* __restrict__ F, StepParams<T> P, int odd, int xbeg,
                                                   int nxc, double* __restrict__ rho, double* __restrict__ u,
                                                   int* flag) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int xc = blockIdx.z;
    if (z >= P.g.nz || y >= P.g.ny) return;
    T f[kQ];
    aa_gather<T, BC>(F, P, odd != 0, xbeg + xc, y, z, f);
    T r, ux, uy, uz;
    moments<T>(f, r, ux, uy, uz);
    if (flag) {
        const int bad = moments_flags<T>(r, ux, uy, uz);
        if (bad) atomicOr(flag, bad);
    }
    const long long cell = ((long long)xc * P.g.ny + y) * P.g.nz + z;
    if (rho) rho[cell] = double(r);
    if (u) {
        u[3 * cell + 0] = double(ux);
        u[3 * cell + 1] = double(uy);
        u[3 * cell + 2] = double(uz);
    }
}

// Reverse AA halo: copy the five slot-planes [slot0, slot0 + 5) of a ghost
// plane (src) into the owner's edge plane (dst), only the entries the odd
// step actually scattered there -- those whose writer (y - c_y, z - c_z) is
// a cell (periodic: all).  In a cavity the rim entries were written by the
// owner itself (its wall rule) and must not be overwritten with the stale
// forward copy.
template <typename T>
__global__ void __launch_bounds__(256) k_aa_merge(T* __restrict__ dst, const T* __restrict__ src, SlabGeom g,
                                                 int slot0) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int m = blockIdx.z;  // 0..4
    if (z >= g.nz || y >= g.ny) return;
    const int k = slot0 + m;
    const int i = slot_dir(k);
    const int sy = y - can_cy(i), sz = z - can_cz(i);
    // periodic: every entry has a (wrapped) writer
    if (g.bc == BC_CAVITY && (sy < 0 || sy >= g.ny || sz < 0 || sz >= g.nz)) return;
    // dst / src point at slot-plane starts: cells begin at g.org (the frame)
    const long long o = (long long)m * g.pq + g.org + (long long)y * g.nzp + z;
    dst[o] = src[o];
}

// ------------------------------------------------------------ launchers --
namespace {
dim3 aa_grid(int nz, int ny, int nx) { return dim3((nz + 31) / 32, (ny + 7) / 8, nx); }
const dim3 kAABlock(32, 8, 1);
}  // namespace

template <typename T>
cudaError_t launch_aa_merge(T* dst, const T* src, const SlabGeom& g, int slot0, cudaStream_t s) {
    k_aa_merge<T><<<aa_grid(g.nz, g.ny, 5), kAABlock, 0, s>>>(dst, src, g, slot0);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_aa_step(T* F, const StepParams<T>& P, bool odd, cudaStream_t s) {
    const SlabGeom& g = P.g;
    const dim3 grid = aa_grid(g.nz, g.ny, g.nxl);
    if (g.bc == BC_PERIODIC) {
        if (odd) k_aa_odd<T, BC_PERIODIC><<<grid, kAABlock, 0, s>>>(F, P);
        else k_aa_even<T, BC_PERIODIC><<<grid, kAABlock, 0, s>>>(F, P);
    } else {
        if (odd) k_aa_odd<T, BC_CAVITY><<<grid, kAABlock, 0, s>>>(F, P);
        else k_aa_even<T, BC_CAVITY><<<grid, kAABlock, 0, s>>>(F, P);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_aa_materialize(const T* F, const StepParams<T>& P, bool odd, int x0, int y0, int z0, int lx,
                                  int ly, int lz, double* out, cudaStream_t s) {
    const dim3 grid = aa_grid(lz, ly, lx);
    if (P.g.bc == BC_PERIODIC)
        k_aa_materialize<T, BC_PERIODIC><<<grid, kAABlock, 0, s>>>(F, P, odd, x0, y0, z0, lx, ly, lz, out);
    else
        k_aa_materialize<T, BC_CAVITY><<<grid, kAABlock, 0, s>>>(F, P, odd, x0, y0, z0, lx, ly, lz, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_aa_moments(const T* F, const StepParams<T>& P, bool odd, int xbeg, int nxc, double* rho,
                              double* u, cudaStream_t s, int* flag) {
    const dim3 grid = aa_grid(P.g.nz, P.g.ny, nxc);
    if (P.g.bc == BC_PERIODIC)
        k_aa_moments<T, BC_PERIODIC><<<grid, kAABlock, 0, s>>>(F, P, odd, xbeg, nxc, rho, u, flag);
    else
        k_aa_moments<T, BC_CAVITY><<<grid, kAABlock, 0, s>>>(F, P, odd, xbeg, nxc, rho, u, flag);
    return cudaGetLastError();
}

#define LBM_AA_INSTANTIATE(T)                                                                                 \
    template cudaError_t launch_aa_step<T>(T*, const StepParams<T>&, bool, cudaStream_t);                     \
    template cudaError_t launch_aa_materialize<T>(const T*, const StepParams<T>&, bool, int, int, int, int,   \
                                                  int, int, double*, cudaStream_t);                          \
    template cudaError_t launch_aa_moments<T>(const T*, const StepParams<T>&, bool, int, int, double*,       \
                                              double*, cudaStream_t, int*);                                  \
    template cudaError_t launch_aa_merge<T>(T*, const T*, const SlabGeom&, int, cudaStream_t);
LBM_AA_INSTANTIATE(double)
LBM_AA_INSTANTIATE(float)

}  // namespace lbm

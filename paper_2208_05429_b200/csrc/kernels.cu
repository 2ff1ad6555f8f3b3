// kernels.cu -- K0 (init), K1 (one fused step), K3 (read-back) for sm_100a.
//
// Storage is "pull" form: a buffer holds the post-collision populations
// f*(t-1) of every cell, and the canonical state is f(t) = S(f*(t-1)), S the
// stream with the boundary rules.  One step is f*(t) = C(S(f*(t-1))): a
// gather of 19 neighbours, the BGK collision in registers, 19 aligned
// stores -- the paper's loop fusion of collide and stream (PAPER.md:232,
// 236, "Fuse Swap LBM") with the in-place swap replaced by a coalesced pull
// gather between two buffers.
#include "kernels.h"

namespace lbm {

// ------------------------------------------------------------------ K1 --
// One thread per cell; a warp covers 32 consecutive z of one row, so each of
// the 19 loads and 19 stores of a warp is one contiguous 256 B (fp64) or
// 128 B (fp32) segment (shifted by one element for c_z != 0 directions).
// Planes [xbeg, xbeg + n1) and then [xbeg2, ...): the two edge ranges of an
// overlapped X-slab sweep run as one grid (api.cu run_steps).
template <typename T, int BC>
__global__ void __launch_bounds__(256) k1_step(const T* __restrict__ A, T* __restrict__ B, StepParams<T> P,
                                              int xbeg, int n1, int xbeg2) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = int(blockIdx.z) < n1 ? xbeg + int(blockIdx.z) : xbeg2 + (int(blockIdx.z) - n1);
    if (z >= P.g.nz || y >= P.g.ny) return;
    T f[kQ];
    pull_cell<T, BC>(A, P, x, y, z, f);
    bgk_collide<T>(f, P.omega);
    const long long self = cell_off(P.g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        __stcs(B + self + (long long)k * P.g.pq, f[slot_dir(k)]);
    });
}

// K1 on single-copy ring storage (LBM_KERNEL_K2_SC, odd remainders): one
// step in place, f*(t) of plane x written into the ring slot of input plane
// x - 4 (out_poff = poff - 4).  Tiles are taken by ticket in plane order; a
// tile of plane x waits until planes x-3, x-4, x-5 are finished (so, by
// induction, every plane <= x-3, the last readers of plane x-4).
template <typename T, int BC, int k>
__device__ __forceinline__ T unstream_slot(const T* C, const StepParams<T>& P, int x, int y, int z, long long self);

// UNSTREAM: instead of a step, K0b's inverse stream of a canonical state held
// in the ring (X-slab single-copy init / set_populations), same ring shift.
template <typename T, int BC, bool UNSTREAM = false>
__global__ void __launch_bounds__(256) k1_step_sc(T* F, StepParams<T> P, int out_poff, unsigned* sync, int tiles_z,
                                                 int tpp) {
    __shared__ int s_item;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        const unsigned it = atomicAdd(&sync[0], 1u);
        const int x = int(it) / tpp;
        for (int back = 3; back <= 5; ++back)
            if (x >= back) sc_wait(&sync[1 + x - back], unsigned(tpp));
        s_item = int(it);
    }
    __syncthreads();
    const int x = s_item / tpp, tile = s_item % tpp;
    const int z = (tile % tiles_z) * 32 + threadIdx.x;
    const int y = (tile / tiles_z) * 8 + threadIdx.y;
    if (z < P.g.nz && y < P.g.ny) {
        const int ps = x + 2 + out_poff;
        T* const dst = F + (long long)(ps >= P.g.pmod ? ps - P.g.pmod : ps) * P.g.px + (long long)y * P.g.nzp + z;
        if constexpr (UNSTREAM) {
            T v[kQ];
            const long long self = cell_off(P.g, x, y, z);
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                v[k] = unstream_slot<T, BC, k>(F, P, x, y, z, self);
            });
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                __stcs(dst + (long long)k * P.g.pq, v[k]);
            });
        } else {
            T f[kQ];
            pull_cell<T, BC>(F, P, x, y, z, f);
            bgk_collide<T>(f, P.omega);
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                __stcs(dst + (long long)k * P.g.pq, f[slot_dir(k)]);
            });
        }
    }
    __syncthreads();  // every thread's stores, then one cumulative fence and the count
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence();
        atomicAdd(&sync[1 + x], 1u);
    }
}

// ---------------------------------------------------------- frame fill --
// Periodic ghost frame (SlabGeom, frame.cuh) of the slab's own planes, from
// their cells: rows [-gy, 0) and [ny, ny + gy) over z in [-S, nz + S) and
// the columns [-S, 0) and [nz, nz + S) over y in [0, ny) (S = g.zoff), each
// a copy of the cell (y mod ny, z mod nz).  Run where a writer other than
// K2/K3 (init, import, K1) left the frame stale; the sweeps keep it current
// themselves.  Every source is an interior cell: the copies are independent.
template <typename T>
__global__ void __launch_bounds__(256) k_frame_fill(T* __restrict__ F, SlabGeom g) {
    const int x = int(blockIdx.y) / kQ, k = int(blockIdx.y) % kQ;
    T* const P = F + plane_base(g, x) + (long long)k * g.pq;
    // (X-Y blocks: the frame rows are the y-neighbours' rows -- exchanged)
    const int S = g.zoff, W = g.nz + 2 * S, nrow = g.ywrap ? 2 * g.gy * W : 0, n = nrow + 2 * S * g.ny;
    for (int e = int(blockIdx.x * blockDim.x + threadIdx.x); e < n; e += int(gridDim.x * blockDim.x)) {
        int y, z;
        if (e < nrow) {
            const int r = e / W;
            y = r < g.gy ? r - g.gy : g.ny + r - g.gy;
            z = e % W - S;
        } else {
            const int q = e - nrow, cidx = q % (2 * S);
            y = q / (2 * S);
            z = cidx < S ? cidx - S : g.nz + cidx - S;
        }
        const int sy = ((y % g.ny) + g.ny) % g.ny, sz = ((z % g.nz) + g.nz) % g.nz;
        P[(long long)y * g.nzp + z] = P[(long long)sy * g.nzp + sz];
    }
}

template <typename T>
cudaError_t launch_frame_fill(T* F, const SlabGeom& g, cudaStream_t s) {
    if (g.gy == 0 || g.nxl <= 0 || (!g.ywrap && g.zoff == 0)) return cudaSuccess;
    const int n = (g.ywrap ? 2 * g.gy * (g.nz + 2 * g.zoff) : 0) + 2 * g.zoff * g.ny;
    k_frame_fill<T><<<dim3(unsigned((n + 255) / 256), unsigned(g.nxl * kQ)), 256, 0, s>>>(F, g);
    return cudaGetLastError();
}

// ---------------------------------------------------- X-Y row bands --
// NCCL X-Y blocks (api.cu exchange): nbands bands of band_bytes each, at
// stride src_stride in src and dst_stride in dst (the frame-row bands of
// every (x, direction) plane <-> a contiguous message).  16-byte vectors:
// bands, strides and bases are multiples of 32 B (the sector-padded rows).
__global__ void __launch_bounds__(256) k_band_copy(const uint4* __restrict__ src, long long src_stride,
                                                   uint4* __restrict__ dst, long long dst_stride, int band,
                                                   int nbands) {
    for (long long b = blockIdx.y; b < nbands; b += gridDim.y) {
        const uint4* const sp = src + b * src_stride;
        uint4* const dp = dst + b * dst_stride;
        for (int e = int(blockIdx.x * blockDim.x + threadIdx.x); e < band; e += int(gridDim.x * blockDim.x))
            dp[e] = sp[e];
    }
}

cudaError_t launch_band_copy(const void* src, long long src_stride_bytes, void* dst, long long dst_stride_bytes,
                             long long band_bytes, int nbands, cudaStream_t s) {
    if (nbands <= 0 || band_bytes <= 0) return cudaSuccess;
    if ((band_bytes | src_stride_bytes | dst_stride_bytes) % 16 || (reinterpret_cast<uintptr_t>(src) % 16) ||
        (reinterpret_cast<uintptr_t>(dst) % 16))
        return cudaErrorInvalidValue;
    const int band = int(band_bytes / 16);
    const int gx = (band + 255) / 256 < 8 ? (band + 255) / 256 : 8;
    k_band_copy<<<dim3(unsigned(gx), unsigned(nbands < 65535 ? nbands : 65535)), 256, 0, s>>>(
        static_cast<const uint4*>(src), src_stride_bytes / 16, static_cast<uint4*>(dst), dst_stride_bytes / 16, band,
        nbands);
    return cudaGetLastError();
}

// ------------------------------------------------------------ K0 init --
// K0a: canonical f = feq(rho, u) of every slab cell into buffer C (slot
// layout).  rho/u are double arrays [x][y][z] / [x][y][z][3] of the slab.
template <typename T>
__global__ void __launch_bounds__(256) k0_equilibrium(const double* __restrict__ rho, const double* __restrict__ u,
                                                     T* __restrict__ C, SlabGeom g, int xbeg) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = xbeg + blockIdx.z;  // rho/u hold planes [xbeg, xbeg + gridDim.z)
    if (z >= g.nz || y >= g.ny) return;
    const long long cell = ((long long)blockIdx.z * g.ny + y) * g.nz + z;
    const T r = rho ? T(rho[cell]) : T(1);
    T ux = T(0), uy = T(0), uz = T(0);
    if (u) {
        ux = T(u[3 * cell + 0]);
        uy = T(u[3 * cell + 1]);
        uz = T(u[3 * cell + 2]);
    }
    T feq[kQ];
    equilibrium<T>(r, ux, uy, uz, feq);
    const long long self = cell_off(g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        C[self + (long long)k * g.pq] = feq[slot_dir(k)];
    });
}

// K0b: the inverse stream, f*(t-1) = S^-1(f(t)).  S is a permutation of the
// slots plus the lid constants, so slot j at cell y takes
//   f_j(y + c_j)                              if y + c_j is a cell (or ghost / wrap)
//   f_opp(j)(y) - [(y + c_j)_z >= nz] lid_opp(j)  if y + c_j is beyond a wall.
// C must have valid ghost planes.
template <typename T, int BC, int k>
__device__ __forceinline__ T unstream_slot(const T* C, const StepParams<T>& P, int x, int y, int z, long long self) {
    const SlabGeom& g = P.g;
    constexpr int j = slot_dir(k);
    constexpr int cx = can_cx(j), cy = can_cy(j), cz = can_cz(j);
    int ty = y + cy, tz = z + cz;
    bool wall = false;
    if constexpr (BC == BC_CAVITY) {
        if constexpr (cx == -1) wall = wall || (x == 0 && g.left_wall);
        if constexpr (cx == 1) wall = wall || (x == g.nxl - 1 && g.right_wall);
        if constexpr (cy == -1) wall = wall || (y == 0 && g.ylo_wall);
        if constexpr (cy == 1) wall = wall || (y == g.ny - 1 && g.yhi_wall);
        if constexpr (cz == -1) wall = wall || (z == 0);
        if constexpr (cz == 1) wall = wall || (z == g.nz - 1);
    } else {
        if constexpr (cy == -1) ty = (y == 0 && g.ywrap) ? g.ny - 1 : ty;
        if constexpr (cy == 1) ty = (y == g.ny - 1 && g.ywrap) ? 0 : ty;
        if constexpr (cz == -1) tz = (z == 0) ? g.nz - 1 : tz;
        if constexpr (cz == 1) tz = (z == g.nz - 1) ? 0 : tz;
    }
    T v;
    if (!wall) {
        v = C[plane_base(g, x + cx) + (long long)k * g.pq + (long long)ty * g.nzp + tz];
    } else {
        constexpr int ko = slot_opp(k);
        v = C[self + (long long)ko * g.pq];
        if constexpr (cz == 1) {
            if (z == g.nz - 1) v = v - P.lid[ko];
        }
    }
    return v;
}

template <typename T, int BC>
__global__ void __launch_bounds__(256) k0_unstream(const T* __restrict__ C, T* __restrict__ A, StepParams<T> P) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = blockIdx.z;
    const SlabGeom& g = P.g;
    if (z >= g.nz || y >= g.ny) return;
    const long long self = cell_off(g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        A[self + (long long)k * g.pq] = unstream_slot<T, BC, k>(C, P, x, y, z, self);
    });
}

// K0 fused (one slab holding the whole x range): the pull-form initial state
// S^-1(feq(rho, u)) in one pass, without the canonical intermediate.  Slot k
// (direction j) of cell y takes feq_j of the cell y + c_j (x, y, z wrapped
// when periodic), or, through a cavity wall, feq_opp(j)(y) - lid_opp; feq_j
// of a neighbour is the single-direction form of eq_pairs() -- the same
// operations, so the same bits as k0_equilibrium + k0_unstream.
template <typename T>
__device__ __forceinline__ void k0_load(const double* rho, const double* u, long long cell, T& r, T& ux, T& uy,
                                        T& uz) {
    r = rho ? T(rho[cell]) : T(1);
    ux = uy = uz = T(0);
    if (u) {
        ux = T(u[3 * cell + 0]);
        uy = T(u[3 * cell + 1]);
        uz = T(u[3 * cell + 2]);
    }
}

template <typename T, int j>
__device__ __forceinline__ T feq_dir(T W, T ux, T uy, T uz) {
    // the per-pair arithmetic of eq_pairs<T, false> for direction j (1..18)
    constexpr int i = j <= 9 ? j : j - 9;  // pair representative
    constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
    const T usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const T base = fma(T(-1.5), usq, T(1));
    const T Wa = W * T(1.0 / 18.0);
    const T Aa = Wa * base, Ba = T(4.5) * Wa, Ca = T(3) * Wa;
    const T Ad = T(0.5) * Aa, Bd = T(0.5) * Ba, Cd = T(0.5) * Ca;
    T cu;
    if constexpr (cx != 0 && cy != 0) cu = (cx > 0 ? ux : -ux) + (cy > 0 ? uy : -uy);
    else if constexpr (cx != 0 && cz != 0) cu = (cx > 0 ? ux : -ux) + (cz > 0 ? uz : -uz);
    else if constexpr (cy != 0 && cz != 0) cu = (cy > 0 ? uy : -uy) + (cz > 0 ? uz : -uz);
    else if constexpr (cx != 0) cu = cx > 0 ? ux : -ux;
    else if constexpr (cy != 0) cu = cy > 0 ? uy : -uy;
    else cu = cz > 0 ? uz : -uz;
    constexpr bool ax = can_axis(i);
    const T common = fma((ax ? Ba : Bd) * cu, cu, ax ? Aa : Ad);
    const T C = ax ? Ca : Cd;
    return j <= 9 ? fma(C, cu, common) : fma(-C, cu, common);
}

// The x window of the per-cell inputs: plane index of slab plane tx (in
// [0, nxl)) in a window holding planes wx0, wx0 + 1, ... (mod nxl) -- the
// whole slab (wx0 = 0) or a host-staged chunk with its x halo.
__device__ __forceinline__ long long k0_wcell(const SlabGeom& g, int wx0, int tx, int ty, int tz) {
    int w = tx - wx0;
    if (w < 0) w += g.nxl;
    return ((long long)w * g.ny + ty) * g.nz + tz;
}

// IMPORT = false: f(t0) = feq(rho, u) (rho, u: 1 and 4 doubles per window
// cell, either may be null); IMPORT = true: f(t0) given, canonical doubles
// src[19][wn][ny][nz] (set_populations without a second lattice copy).
// Planes [xbeg, xbeg + gridDim.z) of the slab.
// RESTU (u == null): every neighbour is at rest, feq_j = w_j rho -- the
// value feq_dir computes for u = 0 (common = A exactly), without its
// arithmetic.
template <typename T, int BC, bool IMPORT, bool RESTU = false>
__global__ void __launch_bounds__(256) k0_init_pull(const double* __restrict__ rho, const double* __restrict__ u,
                                                   const double* __restrict__ src, long long cstride,
                                                   T* __restrict__ A, StepParams<T> P, int xbeg, int wx0) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int x = xbeg + int(blockIdx.z);
    const SlabGeom& g = P.g;
    if (z >= g.nz || y >= g.ny) return;
    const long long own = k0_wcell(g, wx0, x, y, z);
    T feq[kQ];
    if constexpr (!IMPORT) {
        T r, ux, uy, uz;
        k0_load<T>(rho, u, own, r, ux, uy, uz);
        equilibrium<T>(r, ux, uy, uz, feq);  // own cell: slot 0 and the wall links
    }
    const long long self = cell_off(g, x, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        constexpr int j = slot_dir(k);
        constexpr int cx = can_cx(j), cy = can_cy(j), cz = can_cz(j);
        T v;
        if constexpr (j == 0) {
            if constexpr (IMPORT) v = T(src[own]);
            else v = feq[0];
        } else {
            int tx = x + cx, ty = y + cy, tz = z + cz;
            bool wall = false;
            if constexpr (BC == BC_CAVITY) {
                if constexpr (cx == -1) wall = wall || x == 0;
                if constexpr (cx == 1) wall = wall || x == g.nxl - 1;
                if constexpr (cy == -1) wall = wall || y == 0;
                if constexpr (cy == 1) wall = wall || y == g.ny - 1;
                if constexpr (cz == -1) wall = wall || z == 0;
                if constexpr (cz == 1) wall = wall || z == g.nz - 1;
            } else {
                if constexpr (cx == -1) tx = x == 0 ? g.nxl - 1 : tx;
                if constexpr (cx == 1) tx = x == g.nxl - 1 ? 0 : tx;
                if constexpr (cy == -1) ty = y == 0 ? g.ny - 1 : ty;
                if constexpr (cy == 1) ty = y == g.ny - 1 ? 0 : ty;
                if constexpr (cz == -1) tz = z == 0 ? g.nz - 1 : tz;
                if constexpr (cz == 1) tz = z == g.nz - 1 ? 0 : tz;
            }
            if (!wall) {
                const long long t = k0_wcell(g, wx0, tx, ty, tz);
                if constexpr (IMPORT) {
                    v = T(src[(long long)j * cstride + t]);
                } else if constexpr (RESTU) {
                    const T Wa = (rho ? T(rho[t]) : T(1)) * T(1.0 / 18.0);
                    v = can_axis(j <= 9 ? j : j - 9) ? Wa : T(0.5) * Wa;
                } else {
                    T rn, uxn, uyn, uzn;
                    k0_load<T>(rho, u, t, rn, uxn, uyn, uzn);
                    v = feq_dir<T, j>(rn, uxn, uyn, uzn);
                }
            } else {
                constexpr int ko = slot_opp(k);
                if constexpr (IMPORT) v = T(src[(long long)can_opp(j) * cstride + own]);
                else v = feq[can_opp(j)];
                if constexpr (cz == 1) {
                    if (z == g.nz - 1) v = v - P.lid[ko];
                }
            }
        }
        A[self + (long long)k * g.pq] = v;
    });
}

// Import canonical host-order doubles f[19][nx_c][ny][nz] (a chunk of nx_c
// planes starting at slab-local xbeg) into slot layout C.
template <typename T>
__global__ void __launch_bounds__(256) k0_import(const double* __restrict__ src, T* __restrict__ C, SlabGeom g,
                                                int xbeg, int nxc) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int xc = blockIdx.z;
    if (z >= g.nz || y >= g.ny) return;
    const long long cstride = (long long)nxc * g.ny * g.nz;
    const long long cell = ((long long)xc * g.ny + y) * g.nz + z;
    const long long self = cell_off(g, xbeg + xc, y, z);
    static_for<0, kQ>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        C[self + (long long)k * g.pq] = T(src[(long long)slot_dir(k) * cstride + cell]);
    });
}

// -------------------------------------------------------- K3 read-back --
// Canonical f(t) = S(A) on the box [x0,x0+lx) x [y0,y0+ly) x [z0,z0+lz) of
// the slab, written as doubles out[19][lx][ly][lz].
template <typename T, int BC>
__global__ void __launch_bounds__(256) k3_materialize(const T* __restrict__ A, StepParams<T> P, int x0, int y0,
                                                     int z0, int lx, int ly, int lz, double* __restrict__ out) {
    const int zz = blockIdx.x * 32 + threadIdx.x;
    const int yy = blockIdx.y * 8 + threadIdx.y;
    const int xx = blockIdx.z;
    if (zz >= lz || yy >= ly) return;
    T f[kQ];
    pull_cell<T, BC>(A, P, x0 + xx, y0 + yy, z0 + zz, f);
    const long long stride = (long long)lx * ly * lz;
    const long long cell = ((long long)xx * ly + yy) * lz + zz;
#pragma unroll
    for (int i = 0; i < kQ; ++i) out[i * stride + cell] = double(f[i]);
}

// Moments of the canonical f(t) on planes [xbeg, xbeg + nxc): rho[x][y][z],
// u[x][y][z][3] (doubles, chunk-local x).
template <typename T, int BC>
__global__ void __launch_bounds__(256) k3_moments(const T* __restrict__ A, StepParams<T> P, int xbeg, int nxc,
                                                 double* __restrict__ rho, double* __restrict__ u, int* flag) {
    const int z = blockIdx.x * 32 + threadIdx.x;
    const int y = blockIdx.y * 8 + threadIdx.y;
    const int xc = blockIdx.z;
    if (z >= P.g.nz || y >= P.g.ny) return;
    T f[kQ];
    pull_cell<T, BC>(A, P, xbeg + xc, y, z, f);
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

// ------------------------------------------------------------ launchers --
static dim3 cell_grid(int nz, int ny, int nxs) { return dim3((nz + 31) / 32, (ny + 7) / 8, nxs); }
static const dim3 kBlock(32, 8, 1);

template <typename T>
cudaError_t launch_k1(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s, int xbeg2,
                      int nxs2) {
    if (nxs < 0 || nxs2 < 0) return cudaErrorInvalidValue;
    if (nxs + nxs2 == 0) return cudaSuccess;
    const dim3 grid = cell_grid(P.g.nz, P.g.ny, nxs + nxs2);
    if (P.g.bc == BC_PERIODIC)
        k1_step<T, BC_PERIODIC><<<grid, kBlock, 0, s>>>(A, B, P, xbeg, nxs, xbeg2);
    else
        k1_step<T, BC_CAVITY><<<grid, kBlock, 0, s>>>(A, B, P, xbeg, nxs, xbeg2);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k1_sc(T* F, const StepParams<T>& P, int out_poff, unsigned* sync, cudaStream_t s, bool unstream) {
    const SlabGeom& g = P.g;
    if (g.nxl <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(sync, 0, sizeof(unsigned) * (1 + g.nxl), s);
    if (e != cudaSuccess) return e;
    const int tiles_z = (g.nz + 31) / 32, tpp = tiles_z * ((g.ny + 7) / 8);
    const unsigned grid = unsigned((long long)tpp * g.nxl);
    if (unstream) {
        if (g.bc == BC_PERIODIC)
            k1_step_sc<T, BC_PERIODIC, true><<<grid, kBlock, 0, s>>>(F, P, out_poff, sync, tiles_z, tpp);
        else
            k1_step_sc<T, BC_CAVITY, true><<<grid, kBlock, 0, s>>>(F, P, out_poff, sync, tiles_z, tpp);
    } else {
        if (g.bc == BC_PERIODIC)
            k1_step_sc<T, BC_PERIODIC><<<grid, kBlock, 0, s>>>(F, P, out_poff, sync, tiles_z, tpp);
        else
            k1_step_sc<T, BC_CAVITY><<<grid, kBlock, 0, s>>>(F, P, out_poff, sync, tiles_z, tpp);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k0_equilibrium(const double* rho, const double* u, T* C, const SlabGeom& g, cudaStream_t s,
                                  int xbeg, int nxc) {
    if (nxc < 0) nxc = g.nxl;
    if (nxc == 0) return cudaSuccess;
    k0_equilibrium<T><<<cell_grid(g.nz, g.ny, nxc), kBlock, 0, s>>>(rho, u, C, g, xbeg);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k0_init_pull(const double* rho, const double* u, const double* src, T* A, const StepParams<T>& P,
                                int xbeg, int nxc, int wx0, int wn, cudaStream_t s) {
    const SlabGeom& g = P.g;
    if (nxc <= 0) return cudaSuccess;
    const long long cstride = (long long)wn * g.ny * g.nz;
    const dim3 grid = cell_grid(g.nz, g.ny, nxc);
#define LBM_K0P(BC, IMP, R) k0_init_pull<T, BC, IMP, R><<<grid, kBlock, 0, s>>>(rho, u, src, cstride, A, P, xbeg, wx0)
    if (g.bc == BC_PERIODIC) {
        if (src) LBM_K0P(BC_PERIODIC, true, false);
        else if (u) LBM_K0P(BC_PERIODIC, false, false);
        else LBM_K0P(BC_PERIODIC, false, true);
    } else {
        if (src) LBM_K0P(BC_CAVITY, true, false);
        else if (u) LBM_K0P(BC_CAVITY, false, false);
        else LBM_K0P(BC_CAVITY, false, true);
    }
#undef LBM_K0P
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k0_unstream(const T* C, T* A, const StepParams<T>& P, cudaStream_t s) {
    if (P.g.bc == BC_PERIODIC)
        k0_unstream<T, BC_PERIODIC><<<cell_grid(P.g.nz, P.g.ny, P.g.nxl), kBlock, 0, s>>>(C, A, P);
    else
        k0_unstream<T, BC_CAVITY><<<cell_grid(P.g.nz, P.g.ny, P.g.nxl), kBlock, 0, s>>>(C, A, P);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k0_import(const double* src, T* C, const SlabGeom& g, int xbeg, int nxc, cudaStream_t s) {
    k0_import<T><<<cell_grid(g.nz, g.ny, nxc), kBlock, 0, s>>>(src, C, g, xbeg, nxc);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k3_materialize(const T* A, const StepParams<T>& P, int x0, int y0, int z0, int lx, int ly,
                                  int lz, double* out, cudaStream_t s) {
    if (P.g.bc == BC_PERIODIC)
        k3_materialize<T, BC_PERIODIC><<<cell_grid(lz, ly, lx), kBlock, 0, s>>>(A, P, x0, y0, z0, lx, ly, lz, out);
    else
        k3_materialize<T, BC_CAVITY><<<cell_grid(lz, ly, lx), kBlock, 0, s>>>(A, P, x0, y0, z0, lx, ly, lz, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_k3_moments(const T* A, const StepParams<T>& P, int xbeg, int nxc, double* rho, double* u,
                              cudaStream_t s, int* flag) {
    if (P.g.bc == BC_PERIODIC)
        k3_moments<T, BC_PERIODIC><<<cell_grid(P.g.nz, P.g.ny, nxc), kBlock, 0, s>>>(A, P, xbeg, nxc, rho, u, flag);
    else
        k3_moments<T, BC_CAVITY><<<cell_grid(P.g.nz, P.g.ny, nxc), kBlock, 0, s>>>(A, P, xbeg, nxc, rho, u, flag);
    return cudaGetLastError();
}

#define LBM_INSTANTIATE(T)                                                                                   \
    template cudaError_t launch_k1<T>(const T*, T*, const StepParams<T>&, int, int, cudaStream_t, int, int);      \
    template cudaError_t launch_frame_fill<T>(T*, const SlabGeom&, cudaStream_t);           \
    template cudaError_t launch_k1_sc<T>(T*, const StepParams<T>&, int, unsigned*, cudaStream_t, bool);      \
    template cudaError_t launch_k0_equilibrium<T>(const double*, const double*, T*, const SlabGeom&,         \
                                                  cudaStream_t, int, int);                                   \
    template cudaError_t launch_k0_unstream<T>(const T*, T*, const StepParams<T>&, cudaStream_t);            \
    template cudaError_t launch_k0_init_pull<T>(const double*, const double*, const double*, T*,             \
                                                const StepParams<T>&, int, int, int, int, cudaStream_t);     \
    template cudaError_t launch_k0_import<T>(const double*, T*, const SlabGeom&, int, int, cudaStream_t);    \
    template cudaError_t launch_k3_materialize<T>(const T*, const StepParams<T>&, int, int, int, int, int,   \
                                                  int, double*, cudaStream_t);                               \
    template cudaError_t launch_k3_moments<T>(const T*, const StepParams<T>&, int, int, double*, double*,    \
                                              cudaStream_t, int*);
LBM_INSTANTIATE(double)
LBM_INSTANTIATE(float)

}  // namespace lbm

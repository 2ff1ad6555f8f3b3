// k2r.cu -- K2R: the two-step merge (Alg. 2) with the
// step-1 input staged in REGISTERS and the two steps run by two specialised
// warp groups that meet only at named barriers.
//
// Why: the TMA-staged K2 (k2.cu) spends half of shared memory on the staging
// double buffer, which leaves one 11-warp CTA per SM that both stages,
// collides twice and synchronises as a whole every plane -- latency-bound at
// ~60% of HBM (profiles/r01_k2_*).  Here the step-1 input is a per-thread
// gather that needs no CTA-wide synchronisation: each step-1 thread
// copies its own 19 populations one plane AHEAD with cp.async (the pull of
// K1, pull_src(), wall rules applied per lane) into a single-buffered
// per-thread staging area, reads them back into registers at the start of
// the next plane and immediately re-issues the following plane's copies.
// Staging is then one plane (19 x N1 entries) instead of the double-buffered
// TMA boxes, which leaves room for a ring slack plane; and splitting the work
// into two warp groups lets the step-1 gathers/collisions of plane p overlap
// the step-2 collisions/stores of plane p-2 without CTA-wide barriers.
//
//   group S1 (N1 threads, one per cell of the tile plus its one-cell halo):
//     p = xs-1 .. xe:  f = staged f(t) of plane p; cp.async plane p+1;
//                      wait EMPTY(p-3-S); collide; push f*(t) into the ring
//                      (c_x = -1 group to dest p-1, 0 to dest p, +1 to p+1;
//                      wall links bounce into the cell's own slot);
//                      arrive FULL(p-1)      -- dest p-1 is complete
//   group S2 (N2 threads, one per tile cell):
//     d = xs .. xe-1:  wait FULL(d); read f(t+1) from the ring; collide;
//                      stream f*(t+1) to HBM; arrive EMPTY(d)
//
// Ring depths per c_x group, M = 3+S, Z = 3+S, P = 4+S destination planes:
// S1 at plane p writes dest p-1 (M), p (Z, M and P wall links), p+1 (P),
// whose previous occupants p-3-S are consumed, while S2 works on any dest in
// [p-2-S, p-2].  S is the slack (0 = lock-step with one plane of skew).
// Named barrier ids: FULL = 1 + (d mod NB), EMPTY = 1 + NB + (d mod NB),
// NB = S + 2 -- the smallest count for which a barrier id is never re-armed
// before its previous phase completed (each kind's uses are ordered through
// the other kind).
//
// Same bgk_collide()/pull_src() as K1 and the same wall arithmetic as the
// TMA K2, so K2R == K1 o K1 bit for bit (tests/test_gpu_parity.py).
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace lbm {

namespace {

__host__ __device__ constexpr int rup32(int v) { return (v + 31) / 32 * 32; }

template <typename T, int TY_, int TZ_, int S_, int MB_>
struct K2RCfg {
    static constexpr int TY = TY_, TZ = TZ_, S = S_;
    static constexpr int HY = TY + 2, HZ = TZ + 2;
    static constexpr int N1 = rup32(HY * HZ);  // step-1 threads
    static constexpr int N2 = rup32(TY * TZ);  // step-2 threads
    static constexpr int NT = N1 + N2;
    static constexpr int RP = TY * TZ;  // one ring direction-plane
    static constexpr int DM = 3 + S, DZ = 3 + S, DP = 4 + S;
    static constexpr int RING = (DM * 5 + DZ * 9 + DP * 5) * RP;
    static constexpr int STG = kQ * N1;  // staged f(t) of one plane, [slot][thread]
    static constexpr size_t SMEM = size_t(RING + STG) * sizeof(T);
    static constexpr int NB = S + 2;
    static constexpr int MB = MB_;  // CTAs per SM the launch bounds aim for
    static constexpr bool FITS = SMEM * MB + 1024 * MB <= 228 * 1024 && 2 * NB + 1 <= 16 && NT * MB <= 2048;
};

// Byte offsets, relative to a cell's own slot-0 entry, of its 19 pull
// sources when no wall is involved (slot k of x - c_i); |offset| < 2 planes.
struct K2ROffs {
    int b[kQ];
};

__device__ __forceinline__ void nb_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_ca(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "n"(BYTES)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ int posmod(int v, int m) {
    const int r = v % m;
    return r < 0 ? r + m : r;
}

}  // namespace

template <typename T, int BC, int TY, int TZ, int S, int MB>
__global__ void __launch_bounds__(K2RCfg<T, TY, TZ, S, MB>::NT, MB)
    k2r_sweep(const T* __restrict__ A, T* __restrict__ B, StepParams<T> P, const __grid_constant__ K2ROffs O, int xbeg,
              int xend, int chunk) {
    using C = K2RCfg<T, TY, TZ, S, MB>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* const ringM = reinterpret_cast<T*>(smem_raw);
    T* const ringZ = ringM + C::DM * 5 * C::RP;
    T* const ringP = ringZ + C::DZ * 9 * C::RP;
    T* const stg = ringP + C::DP * 5 * C::RP;

    const SlabGeom& g = P.g;
    const int ntz = (g.nz + TZ - 1) / TZ;
    const int y0 = (int(blockIdx.x) / ntz) * TY;
    const int z0 = (int(blockIdx.x) % ntz) * TZ;
    const int xs = xbeg + int(blockIdx.y) * chunk;
    const int xe = min(xs + chunk, xend);
    if (xs >= xe) return;
    auto FULL = [](int d) { return 1 + posmod(d, C::NB); };
    auto EMPTY = [](int d) { return 1 + C::NB + posmod(d, C::NB); };

    if (threadIdx.x < C::N2) {
        // ===================== S2: second collision of dest plane d =====================
        const int tid = threadIdx.x;
        const int y2 = tid / TZ, z2 = tid % TZ;
        const bool in2 = tid < TY * TZ && y0 + y2 < g.ny && z0 + z2 < g.nz;
        const long long off0 = cell_off(g, 0, y0 + y2, z0 + z2);
        for (int d = xs; d < xe; ++d) {
            nb_sync(FULL(d), C::NT);
            T f[kQ];
            if (in2) {
                const T* const qM = ringM + (d % C::DM) * 5 * C::RP + tid;
                const T* const qZ = ringZ + (d % C::DZ) * 9 * C::RP + tid;
                const T* const qP = ringP + (d % C::DP) * 5 * C::RP + tid;
                static_for<0, kQ>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    if constexpr (k < 5) f[slot_dir(k)] = qM[k * C::RP];
                    else if constexpr (k < 14) f[slot_dir(k)] = qZ[(k - 5) * C::RP];
                    else f[slot_dir(k)] = qP[(k - 14) * C::RP];
                });
            }
            // ring entries of d are in registers.  Outside the branch: a warp
            // arriving at a named barrier counts 32 arrivals however many of
            // its threads are active, so it must arrive exactly once.
            __syncwarp();
            nb_arrive(EMPTY(d), C::NT);
            if (in2) {
                bgk_collide<T>(f, P.omega);
                T* const dst = B + off0 + (long long)d * g.px;
                static_for<0, kQ>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    __stcs(dst + (long long)k * g.pq, f[slot_dir(k)]);
                });
            }
        }
        return;
    }

    // ===================== S1: gather + first collision of plane p =====================
    const int tid = int(threadIdx.x) - C::N2;
    const int p_first = (xs == 0 && BC == BC_CAVITY && g.left_wall) ? 0 : xs - 1;
    const int p_last = (xe == g.nxl && BC == BC_CAVITY && g.right_wall) ? g.nxl - 1 : xe;
    const int a = tid / C::HZ, b = tid % C::HZ;
    const bool act1 = tid < C::HY * C::HZ;
    const int qy = y0 - 1 + a, qz = z0 - 1 + b;
    bool q_in;
    int gy = qy, gz = qz;  // the cell whose populations this thread gathers
    if constexpr (BC == BC_PERIODIC) {
        q_in = act1;
        gy = gy < 0 ? gy + g.ny : (gy >= g.ny ? gy - g.ny : gy);
        gz = gz < 0 ? gz + g.nz : (gz >= g.nz ? gz - g.nz : gz);
    } else {
        q_in = act1 && qy >= 0 && qy < g.ny && qz >= 0 && qz < g.nz;
    }
    const bool q_tile = act1 && a >= 1 && a <= TY && b >= 1 && b <= TZ;
    const bool edge_y = (y0 < 1) || (y0 + TY + 1 > g.ny);
    const bool edge_z = (z0 < 1) || (z0 + TZ + 1 > g.nz);
    const bool edge_tile = BC == BC_CAVITY && (edge_y || edge_z);
    const int toff = (a - 1) * TZ + (b - 1);  // ring entry of this cell (tile coords)
    // is the push destination (a - 1 + c_y, b - 1 + c_z) inside the tile, per c_y / c_z
    const bool rowok[3] = {a >= 2 && a <= TY + 1, a >= 1 && a <= TY, a <= TY - 1};
    const bool colok[3] = {b >= 2 && b <= TZ + 1, b >= 1 && b <= TZ, b <= TZ - 1};

    // stage plane p's gathered f(t) of this thread's cell: stg[k][tid].
    // Tiles whose step-1 sources all lie inside [0,ny) x [0,nz) (CTA-uniform)
    // gather at fixed offsets from the cell on every non-wall plane; edge
    // tiles and wall planes take pull_src() with the per-lane wall rules.
    T* const mine = stg + tid;
    const bool yz_inner = y0 >= 2 && y0 + TY + 2 <= g.ny && z0 >= 2 && z0 + TZ + 2 <= g.nz;
    auto gather = [&](int p) {
        const bool wall_plane = BC == BC_CAVITY && ((p == 0 && g.left_wall) || (p == g.nxl - 1 && g.right_wall));
        if (yz_inner && !wall_plane) {
            const char* const base = reinterpret_cast<const char*>(A + cell_off(g, p, gy, gz));
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                cp_async_ca<sizeof(T)>(mine + k * C::N1, base + O.b[k]);
            });
        } else {
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                cp_async_ca<sizeof(T)>(mine + k * C::N1, A + pull_src<BC, k>(g, p, gy, gz));
            });
        }
    };
    if (q_in && p_first <= p_last) gather(p_first);
    cp_async_commit();
    const bool lid_row = BC == BC_CAVITY && gz == g.nz - 1;
    for (int p = xs - 1; p <= xe; ++p) {
        const bool has1 = q_in && p >= p_first && p <= p_last;
        T f[kQ];
        cp_async_wait_all();
        if (has1) {
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                T v = mine[k * C::N1];
                if constexpr (BC == BC_CAVITY && can_cz(slot_dir(k)) == -1) {
                    if (lid_row) v = v + P.lid[k];
                }
                f[slot_dir(k)] = v;
            });
            if (p + 1 <= p_last) gather(p + 1);
        }
        cp_async_commit();
        __syncwarp();  // one arrival per warp at each named barrier (see S2)
        if (p - 3 - S >= xs) nb_sync(EMPTY(p - 3 - S), C::NT);
        const bool lwall = BC == BC_CAVITY && p == 0 && g.left_wall;
        const bool rwall = BC == BC_CAVITY && p == g.nxl - 1 && g.right_wall;
        T* const wM = ringM + posmod(p - 1, C::DM) * 5 * C::RP;  // dest p-1
        T* const wZ = ringZ + posmod(p, C::DZ) * 9 * C::RP;      // dest p
        T* const wP = ringP + posmod(p + 1, C::DP) * 5 * C::RP;  // dest p+1
        if (has1) {
            bgk_collide<T>(f, P.omega);
            // ---- pushes: direction i streams to (p + cx, a - 1 + cy, b - 1 + cz) ----
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr int i = slot_dir(k);
                constexpr int cy = can_cy(i), cz = can_cz(i);
                constexpr int rel = cy * TZ + cz;
                if (rowok[cy + 1] && colok[cz + 1]) {
                    if constexpr (k < 5) wM[k * C::RP + toff + rel] = f[i];
                    else if constexpr (k < 14) wZ[(k - 5) * C::RP + toff + rel] = f[i];
                    else wP[(k - 14) * C::RP + toff + rel] = f[i];
                }
            });
            if constexpr (BC == BC_CAVITY) {
                // ---- wall links of a tile cell: bounce-back (+ lid) into its own slot ----
                if ((edge_tile || lwall || rwall) && q_tile) {
                    T* const bM = ringM + posmod(p, C::DM) * 5 * C::RP;  // dest p
                    T* const bP = ringP + posmod(p, C::DP) * 5 * C::RP;  // dest p
                    static_for<0, kQ>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        constexpr int i = slot_dir(k);
                        constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
                        const int sy = qy - cy, sz = qz - cz;
                        bool out = sy < 0 || sy >= g.ny || sz < 0 || sz >= g.nz;
                        if constexpr (cx == 1) out = out || lwall;
                        if constexpr (cx == -1) out = out || rwall;
                        if (out) {
                            T v = f[can_opp(i)];
                            if constexpr (cz == -1) {
                                if (qz == g.nz - 1) v = v + P.lid[k];
                            }
                            if constexpr (k < 5) {
                                bM[k * C::RP + toff] = v;
                            } else if constexpr (k < 14) {
                                wZ[(k - 5) * C::RP + toff] = v;
                            } else {
                                bP[(k - 14) * C::RP + toff] = v;
                            }
                        }
                    });
                }
            }
        }
        __syncwarp();
        if (p - 1 >= xs) nb_arrive(FULL(p - 1), C::NT);  // dest p-1 complete
    }
    // match the EMPTY arrivals of the dests not waited for in the loop (the
    // loop waits for [xs, xe-3-S]) so no barrier is left armed
    for (int e = max(xs, xe - 2 - S); e < xe; ++e) nb_sync(EMPTY(e), C::NT);
}

// ------------------------------------------------------------------ host --
namespace {

int k2r_num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

template <typename T, int BC, int TY, int TZ, int S, int MB>
cudaError_t launch_k2r_impl(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s) {
    using C = K2RCfg<T, TY, TZ, S, MB>;
    auto kern = k2r_sweep<T, BC, TY, TZ, S, MB>;
    static int occ = -1;
    if (occ < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NT, C::SMEM);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
    }
    const SlabGeom& g = P.g;
    // x chunks: fill the machine in whole waves; each chunk re-computes 2 halo planes of step 1
    const long long ntiles = (long long)((g.ny + TY - 1) / TY) * ((g.nz + TZ - 1) / TZ);
    const long long slots = (long long)k2r_num_sms() * occ;
    int best = 1;
    double best_cost = 1e300;
    for (int nch = 1; nch <= min(nxs, 64); ++nch) {
        const int chunk = (nxs + nch - 1) / nch;
        const long long items = ntiles * ((nxs + chunk - 1) / chunk);
        const double waves = double((items + slots - 1) / slots);
        const double cost = waves * (chunk + 2.5);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = nch;
        }
    }
    int chunk = (nxs + best - 1) / best;
    static const int force_chunk = [] {
        const char* e = getenv("LBM_K2_CHUNK");  // planes per CTA (tuning runs)
        return e ? atoi(e) : 0;
    }();
    if (force_chunk > 0) chunk = min(force_chunk, nxs);
    const dim3 grid(unsigned(ntiles), unsigned((nxs + chunk - 1) / chunk));
    K2ROffs O;
    for (int k = 0; k < kQ; ++k) {
        const int i = slot_dir(k);
        O.b[k] = int(((long long)k * g.pq - can_cx(i) * g.px - can_cy(i) * (long long)g.nzp - can_cz(i)) *
                     (long long)sizeof(T));
    }
    kern<<<grid, C::NT, C::SMEM, s>>>(A, B, P, O, xbeg, xbeg + nxs, chunk);
    return cudaGetLastError();
}

// LBM_K2R_CFG=<TY>x<TZ>s<S>[m<MB>] selects a compiled shape (tuning runs).
int k2r_choice() {
    static int c = -1;
    if (c < 0) {
        c = 0;
        if (const char* e = getenv("LBM_K2R_CFG")) {
            const char* names[] = {"8x32s0", "8x32s1", "8x16s0m2", "16x16s0", "4x32s0m2", "8x16s1m2"};
            for (int i = 0; i < 6; ++i)
                if (!strcmp(e, names[i])) c = i + 1;
        }
    }
    return c;
}

}  // namespace

template <typename T>
bool k2r_supported(const SlabGeom& g) {
    // the pull offsets (within +-2 planes) are 32-bit byte offsets
    return (2 * g.px + g.nzp + 1) * (long long)sizeof(T) < (1LL << 31);
}

template <typename T>
cudaError_t launch_k2r(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s) {
    if (nxs <= 0) return cudaSuccess;
    if (!k2r_supported<T>(P.g)) return cudaErrorInvalidValue;
    const bool per = P.g.bc == BC_PERIODIC;
#define LBM_K2R_CASE(TY, TZ, S, MB)                                                          \
    if constexpr (K2RCfg<T, TY, TZ, S, MB>::FITS) {                                          \
        return per ? launch_k2r_impl<T, BC_PERIODIC, TY, TZ, S, MB>(A, B, P, xbeg, nxs, s)   \
                   : launch_k2r_impl<T, BC_CAVITY, TY, TZ, S, MB>(A, B, P, xbeg, nxs, s);    \
    } else {                                                                                 \
        return cudaErrorInvalidConfiguration;                                                \
    }
    switch (k2r_choice()) {
        case 2: LBM_K2R_CASE(8, 32, 1, 1);
        case 3: LBM_K2R_CASE(8, 16, 0, 2);
        case 4: LBM_K2R_CASE(16, 16, 0, 1);
        case 5: LBM_K2R_CASE(4, 32, 0, 2);
        case 6: LBM_K2R_CASE(8, 16, 1, 2);
        case 1:
        default: LBM_K2R_CASE(8, 32, 0, 1);
    }
#undef LBM_K2R_CASE
}

template bool k2r_supported<double>(const SlabGeom&);
template bool k2r_supported<float>(const SlabGeom&);
template cudaError_t launch_k2r<double>(const double*, double*, const StepParams<double>&, int, int, cudaStream_t);
template cudaError_t launch_k2r<float>(const float*, float*, const StepParams<float>&, int, int, cudaStream_t);

}  // namespace lbm

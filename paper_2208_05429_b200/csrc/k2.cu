// k2.cu -- K2: two collision-streaming steps per HBM pass (temporal blocking),
// the GPU form of the paper's two-step merge (Alg. 2, PAPER.md:140-216:
// "after a cell completes the first computation ... cell (1,1,1) is ready for
// the second collide").
//
// Each CTA owns an output tile T of TY x TZ cells in the (y, z) plane and
// marches along x over a chunk of <= 32-72 planes (the paper's X-outermost
// order; short chunks keep co-resident CTAs within a few planes
// of each other, so the halo rows one CTA stages are still in L2 for its
// neighbours).  Per input plane p:
//   1. TMA stages f(t) on the tile plus a one-cell halo T+1: one box per
//      direction, its origin shifted by -c_i, so the TMA unit performs the
//      y part of the pull-stream (19 cp.async.bulk.tensor per plane, one
//      mbarrier, double-buffered).  Each thread reads its 19 values into
//      registers, then ONE block barrier frees the buffer and the TMA of
//      plane p+2 is issued before any collision, so every load has two
//      compute phases to land.  Entries whose source lies beyond a cavity
//      wall (bounce-back + lid) are replaced per thread in registers -- no
//      CTA-wide fix-up pass.  A periodic box never wraps here: its planes
//      carry a ghost frame of the wrapped rows / columns (frame.cuh) that
//      the boxes read and this kernel's own stores keep current.
//   2. Step 1: every cell of T+1 collides (BGK, registers) and PUSHES its
//      post-collision populations into a destination-indexed SMEM ring:
//      direction i goes to the cell it streams to, (p + c_x, y + c_y, z + c_z).
//      Wall links are resolved at the same time (bounce-back + lid into the
//      cell's own slot), so the ring holds exactly f(t+1) of the tile.
//   3. Step 2 of destination plane p-2 (complete since this iteration's
//      barrier) runs in the same phase: a thread's step-2 cell and step-1
//      cell collide as two interleaved dependency chains (bgk_collide2), and
//      f*(t+1) leaves with coalesced streaming stores.
// The ring keeps, per destination plane, only the populations still to
// arrive: c_x = -1 group (5) x 2 planes, c_x = 0 (9) x 3, c_x = +1 (5) x 4.
// Every population therefore crosses HBM once per two steps (plus the halo
// re-reads that miss L2: 1.1-1.25x the algorithmic reads, ncu).
//
// The arithmetic is the same bgk_collide()/pull rules as K1 (d3q19.cuh), so
// K2 == K1 o K1 bit for bit (tests/test_gpu_parity.py).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>

#include "frame.cuh"
#include "kernels.h"

namespace lbm {

namespace {

__host__ __device__ constexpr int round_up_c(int v, int m) { return (v + m - 1) / m * m; }

template <typename T, int TY_, int TZ_>
struct K2Cfg {
    static constexpr int TY = TY_, TZ = TZ_;
    static constexpr int HY = TY + 2, HZ = TZ + 2;            // tile + one-cell halo
    // The TMA box origin's innermost coordinate must be 16-byte aligned, so a
    // box starts ZPAD elements before the tile (z0 - ZPAD, z0 a multiple of
    // 32) and spans TZ + 2 ZPAD; the -c_z shift is applied when reading.
    static constexpr int ZPAD = 16 / int(sizeof(T));
    static constexpr int BW = TZ + 2 * ZPAD;
    static constexpr int BOX = HY * BW;                        // staged elements per direction
    static constexpr int BOXE = round_up_c(BOX * int(sizeof(T)), 128) / int(sizeof(T));  // 128 B aligned
    static constexpr int NT = round_up_c(HY * HZ, 32);         // threads: one per T+1 cell
    static constexpr int RP = TY * TZ;                         // ring plane (one direction)
    // ring depth per group (destination planes live at once, see the loop)
    static constexpr int NM = 2, NZ = 3, NP = 4;
    static constexpr int RING = (NM * 5 + NZ * 9 + NP * 5) * RP;  // 57 direction-planes
    // cavity wall-link values of the next plane, prefetched per thread with
    // cp.async: [2 buffers][HZ wall-row lanes + HY wall-column lanes][5 slots]
    static constexpr int WALLE = (HZ + HY) * 5;
    static constexpr size_t SMEM =
        size_t(2 * kQ * BOXE + RING + 2 * WALLE) * sizeof(T) + 2 * sizeof(uint64_t);
    static constexpr uint32_t TX_BYTES = uint32_t(kQ * BOX * sizeof(T));
    // CTAs per SM: what shared memory (228 KB per SM, 1 KB reserved per CTA)
    // and registers (about 168 per thread in fp64, 96 in fp32) allow
    static constexpr bool FITS = SMEM <= 227 * 1024;
    static constexpr int BY_SMEM = int((228 * 1024) / (SMEM + 1024));
    static constexpr int BY_REGS = 65536 / (NT * (sizeof(T) == 8 ? 168 : 96));
    static constexpr int MINB_RAW = BY_SMEM < BY_REGS ? BY_SMEM : BY_REGS;
    static constexpr int MINB = MINB_RAW < 1 ? 1 : (MINB_RAW > 3 ? 3 : MINB_RAW);
};

// position of slot k among the slots whose c_y (dim 1) / c_z (dim 2) equals sgn
__host__ __device__ constexpr int wall_idx(int k, int dim, int sgn) {
    int m = 0;
    for (int j = 0; j < k; ++j) {
        const int i = slot_dir(j);
        if ((dim == 1 ? can_cy(i) : can_cz(i)) == sgn) ++m;
    }
    return m;
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a TMA that never completes traps (a kernel error the host
// reports) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t spin = 0; !mbar_try_wait(bar, parity); ++spin) {
        if (spin > (1u << 28)) __trap();
    }
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 int c2, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

}  // namespace

template <typename T, int BC, int TY, int TZ, bool EARLY, bool RING, bool YB>
__global__ void __launch_bounds__(K2Cfg<T, TY, TZ>::NT, K2Cfg<T, TY, TZ>::MINB)
    k2_sweep(const __grid_constant__ CUtensorMap tmA, const T* __restrict__ A, T* __restrict__ B, StepParams<T> P,
             int xbeg, int xend, int chunk, int out_poff, unsigned* __restrict__ sc_sync, T* haloL, T* haloR,
             int xbeg2, int nch1, int kflags) {
    using C = K2Cfg<T, TY, TZ>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* const stage = reinterpret_cast<T*>(smem_raw);
    T* const ringM = stage + 2 * kQ * C::BOXE;
    T* const ringZ = ringM + C::NM * 5 * C::RP;
    T* const ringP = ringZ + C::NZ * 9 * C::RP;
    T* const wallbuf = ringP + C::NP * 5 * C::RP;  // [2][HZ + HY][5]
    uint64_t* const bar = reinterpret_cast<uint64_t*>(wallbuf + 2 * C::WALLE);

    const SlabGeom& g = P.g;
    // Work item (tile, x chunk): the block index, or -- single-copy ring
    // storage, where step 2 overwrites planes of f*(t-1) in place -- a ticket
    // taken in chunk-major order.  There the outputs of chunk j land on the
    // input planes of chunks <= j - 2 (launch_k2), so a CTA of chunk j first
    // waits until every CTA of chunks j - 2 and j - 3 has finished -- which,
    // by induction over those CTAs' own waits, means every chunk <= j - 2.
    // The awaited CTAs hold earlier tickets, so they are running or done: no
    // deadlock.  (A persistent variant -- CTAs looping over tickets, the TMA
    // of the next item's first planes issued while the current one drains --
    // measured slower: 35.3k vs 36.4k MLUPS fp64.)
    int item_t = int(blockIdx.x), item_c = int(blockIdx.y);
    if (RING) {
        int* const s_item = reinterpret_cast<int*>(smem_raw);
        if (threadIdx.x == 0) {
            const unsigned it = atomicAdd(&sc_sync[0], 1u);
            const int ch = int(it / gridDim.x);
            for (int back = 2; back <= 3; ++back)
                if (ch >= back) sc_wait(&sc_sync[1 + ch - back], gridDim.x);
            *s_item = int(it);
        }
        __syncthreads();
        item_t = *s_item % int(gridDim.x);
        item_c = *s_item / int(gridDim.x);
    }
    // single-copy ring: this CTA's stores are complete and visible -> count
    // it (the chunk index recomputed from xs: nothing extra live in the loop)
    auto sc_finish = [&](int xs_) {
        if (RING) {
            // the barrier orders every thread's stores before thread 0's
            // cumulative gpu-scope fence, then the count (the pattern of a
            // cooperative grid barrier)
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(&sc_sync[1 + (xs_ - xbeg) / chunk], 1u);
            }
        }
    };
    const int ntz = (g.nz + TZ - 1) / TZ;
    // Tile order: z-fastest within strips of zbw tiles in z, then y, then
    // the next strip.  z-neighbours (whose boxes share the 32 B halo sectors
    // of every staged row) run together, and y-neighbours -- each re-stages
    // a row of the other -- are only zbw tiles apart in the dispatch order,
    // so they run within a few planes of each other and the shared rows are
    // still in L2 (a y-fastest order measured 1.33x the DRAM reads, -17%).
    int y0, z0;
    {
        const int zbw = min(max((kflags >> 8) & 0xff, 1), ntz);
        const int nty = (g.ny + TY - 1) / TY;
        const int full = ntz / zbw, inFull = full * nty * zbw;
        if (item_t < inFull) {
            const int sb = item_t / (nty * zbw), r = item_t - sb * (nty * zbw);
            y0 = (r / zbw) * TY;
            z0 = (sb * zbw + r % zbw) * TZ;
        } else {
            const int w = ntz - full * zbw, r = item_t - inFull;
            y0 = (r / w) * TY;
            z0 = (full * zbw + r % w) * TZ;
        }
    }
    // chunks [0, nch1) cover [xbeg, xend); chunks nch1.. the second range
    // [xbeg2, xbeg2 + xend - xbeg) (the two edge ranges of an overlapped sweep)
    const bool r2 = item_c >= nch1;
    const int xs = r2 ? xbeg2 + (item_c - nch1) * chunk : xbeg + item_c * chunk;
    const int xe = min(xs + chunk, r2 ? xbeg2 + (xend - xbeg) : xend);
    if (xs >= xe) {
        sc_finish(xs);
        return;
    }
    // step-1 planes: one beyond each end of the chunk unless that is beyond a wall
    const int p_first = (xs == 0 && BC == BC_CAVITY && g.left_wall) ? 0 : xs - 1;
    const int p_last = (xe == g.nxl && BC == BC_CAVITY && g.right_wall) ? g.nxl - 1 : xe;

    const int tid = threadIdx.x;
    // step-1 cell of this thread: box coordinates (a, b), cell (p, qy, qz).
    // Threads [0, HY*TZ) take the TZ interior columns row by row (a warp =
    // 32 consecutive cells of one row: conflict-free stage reads and ring
    // pushes when TZ = 32); the next 2*HY threads take the two halo columns.
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
    // (X-Y blocks: a y end that is not a domain wall has the neighbour's
    // rows in the frame, so halo cells beyond it are real cells)
    // (YB: an X-Y block, whose y ends are walls only where they are the
    // domain's; otherwise compile-time walls -- the flags cost the plain
    // cavity sweep 2-3% as runtime values)
    const bool ylo = YB ? g.ylo_wall != 0 : true, yhi = YB ? g.yhi_wall != 0 : true;
    const int ymin = ylo ? 0 : -2, ymax = yhi ? g.ny : g.ny + 2;
    const bool q_in = act1 && (BC == BC_PERIODIC || (qy >= ymin && qy < ymax && qz >= 0 && qz < g.nz));
    const bool q_tile = act1 && a >= 1 && a <= TY && b >= 1 && b <= TZ;
    // step-2 cell of this thread
    const int y2 = tid / TZ, z2 = tid % TZ;
    const bool in2 = tid < TY * TZ && y0 + y2 < g.ny && z0 + z2 < g.nz;
    const bool warp2 = (tid & ~31) < TY * TZ;  // the warp owns step-2 cells (warp-uniform)
    const int st_off = (y0 + y2) * g.nzp + (z0 + z2);  // in-plane offset of the step-2 cell (< 2^31)
    // does any staged entry of this tile pull from outside [0,ny) x [0,nz)?
    const bool edge_y = (y0 < 2 && ylo) || (y0 + TY + 2 > g.ny && yhi);
    const bool edge_z = (z0 < 2) || (z0 + TZ + 2 > g.nz);

    // L2 policy of the staging loads: evict_last (default) keeps the rows a
    // neighbouring tile or the next plane's CTA re-stages in L2 in preference
    // to the streaming output (stored evict-first): measured +0.9% on config
    // 5 fp64 (LBM_K2_EVICT_LAST=0 restores evict_normal)
    uint64_t pol;
    if (kflags & 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    // Periodic boxes: the TMA box reads the ghost frame (SlabGeom) instead of
    // wrapping -- coordinates are frame coordinates, y + gy and z + zoff.
    auto issue = [&](int p, int s) {  // one thread: stage plane p into buffer s
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&bar[s], C::TX_BYTES);
        static_for<0, kQ>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            constexpr int i = slot_dir(k);
            tma_load_3d_hint(stage + (s * kQ + k) * C::BOXE, &tmA, &bar[s], z0 - C::ZPAD + g.zoff,
                             y0 - 1 - can_cy(i) + g.gy, plane_slot_t<RING>(g, p - can_cx(i)) * kQ + k, pol);
        });
    };

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        if (p_first <= p_last) issue(p_first, 0);
        if (p_first + 1 <= p_last) issue(p_first + 1, 1);
    }

    // per-thread constants of the hot loop
    const int soff = a * C::BW + b + C::ZPAD - 1;  // staged entry of (a, b) for c_z = 0
    const int toff = (a - 1) * TZ + (b - 1);        // ring entry of this cell (tile coords)
    // is the push destination (a - 1 + c_y, b - 1 + c_z) inside the tile, per c_y / c_z
    const bool rowok[3] = {a >= 2 && a <= TY + 1, a >= 1 && a <= TY, a <= TY - 1};
    const bool colok[3] = {b >= 2 && b <= TZ + 1, b >= 1 && b <= TZ, b <= TZ - 1};
    const bool edge_tile = BC == BC_CAVITY && (edge_y || edge_z);
    // this cell's cavity walls (a link from beyond: c_y = +1 at y = 0, ...)
    const bool wyl = BC == BC_CAVITY && qy == 0 && ylo, wyh = BC == BC_CAVITY && qy == g.ny - 1 && yhi;
    const bool wzl = BC == BC_CAVITY && qz == 0, wzh = BC == BC_CAVITY && qz == g.nz - 1;
    // Cavity wall lanes of this tile: the box row holding y = 0 or y = ny-1
    // and the box column holding z = 0 or z = nz-1 (at most one of each;
    // otherwise -- tiny domains -- the direct loads below).  Their wall-link
    // values (the cell's own opposite slots) are prefetched one plane ahead
    // into shared memory with cp.async, off the critical path.
    int wrow = -1, wcol = -1, wsy = 0, wsz = 0;  // wsy / wsz: c_y / c_z of the wall slots
    bool wb_ok = false;
    if constexpr (BC == BC_CAVITY) {
        const int r0 = (y0 <= 1 && ylo) ? 1 - y0 : -1,
                  r1 = (g.ny - y0 >= 0 && g.ny - y0 <= C::HY - 1 && yhi) ? g.ny - y0 : -1;
        const int c0 = z0 <= 1 ? 1 - z0 : -1, c1 = (g.nz - z0 >= 0 && g.nz - z0 <= C::HZ - 1) ? g.nz - z0 : -1;
        wb_ok = edge_tile && !(r0 >= 0 && r1 >= 0) && !(c0 >= 0 && c1 >= 0);
        if (r0 >= 0) { wrow = r0; wsy = 1; } else if (r1 >= 0) { wrow = r1; wsy = -1; }
        if (c0 >= 0) { wcol = c0; wsz = 1; } else if (c1 >= 0) { wcol = c1; wsz = -1; }
    }
    const bool wl_row = wb_ok && q_in && a == wrow, wl_col = wb_ok && q_in && b == wcol;
    auto wall_prefetch = [&](int pn, int buf) {  // this thread's wall values of plane pn
        if (!(wl_row || wl_col)) return;
        const T* const selfp = A + plane_base_t<RING>(g, pn) + (long long)qy * g.nzp + qz;
        T* const wb = wallbuf + buf * C::WALLE;
        static_for<0, kQ>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            constexpr int i = slot_dir(k);
            constexpr int cy = can_cy(i), cz = can_cz(i);
            if constexpr (cy != 0) {
                if (wl_row && cy == wsy) {
                    T* d = wb + b * 5 + wall_idx(k, 1, cy);
                    if constexpr (sizeof(T) == 8) cp_async8(d, selfp + (long long)slot_opp(k) * g.pq);
                    else cp_async4(d, selfp + (long long)slot_opp(k) * g.pq);
                }
            }
            if constexpr (cz != 0) {
                if (wl_col && cz == wsz) {
                    T* d = wb + (C::HZ + a) * 5 + wall_idx(k, 2, cz);
                    if constexpr (sizeof(T) == 8) cp_async8(d, selfp + (long long)slot_opp(k) * g.pq);
                    else cp_async4(d, selfp + (long long)slot_opp(k) * g.pq);
                }
            }
        });
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (p_first <= p_last) wall_prefetch(p_first, 0);
    // Periodic ghost-frame copies of this thread's step-2 cell (frame.cuh):
    // written with the cell's stores, so the next sweep's TMA boxes find the
    // frame complete.
    FrameMask fm;
    if constexpr (BC == BC_PERIODIC) {
        if (in2) fm = frame_mask(g, y0 + y2, z0 + z2);
    }
    const bool fany = BC == BC_PERIODIC && fm.any();

    // Software pipeline, ONE block barrier per plane (after the stage read).
    // Iteration p runs, in the same phase, step 2 of destination plane p-2
    // (complete since this iteration's barrier) and step 1 of plane p, whose pushes go to destination
    // planes p-1 (c_x = -1), p (c_x = 0, and wall links) and p+1 (c_x = +1).
    // Ring depths keep reads and writes of one phase apart: M 2 (dest p-2
    // read / p-1 written), Z 3 (p-2 read, p-1 live, p written), P 4 (p-2
    // read, p-1 and p live, p+1 written).  Bounce-back links of c_x = -1
    // directions (dest p) are held in registers and written next iteration
    // with the regular pushes of dest p, so M needs only two planes.
    T heldP[5];  // f*_opp of the c_x = -1 wall links of the previous plane (+ lid)
    unsigned held_mask = 0;
    for (int p = xs - 1; p <= xe + 1; ++p) {
        const bool has1 = p >= p_first && p <= p_last;
        const int c = p - p_first, s = c & 1;
        T* const st = stage + s * kQ * C::BOXE;
        const bool lwall = BC == BC_CAVITY && p == 0 && g.left_wall;
        const bool rwall = BC == BC_CAVITY && p == g.nxl - 1 && g.right_wall;
        T fs[kQ];
        if (has1) {
            mbar_wait(&bar[s], uint32_t(c >> 1) & 1u);
        }
        // Read this thread's staged f(t) into registers, then ONE barrier:
        // the stage buffer is free and the TMA of plane p+2 is issued before
        // any collision of this iteration, so every load has two compute
        // phases to land (an effective third pipeline stage without a third
        // buffer).  The barrier also orders step 1 of plane p-1 (last
        // iteration's pushes) before step 2 of plane p-2 below.
        auto read_stage = [&] {
            if (has1) {
                const T* const sp = st + (act1 ? soff : C::ZPAD);
                static_for<0, kQ>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    constexpr int i = slot_dir(k);
                    fs[i] = sp[k * C::BOXE - can_cz(i)];
                });
                if constexpr (BC == BC_CAVITY) {
                    // Wall links (source beyond a wall):
                    // the staged entry (TMA zero fill, or a cell beyond the x
                    // wall) is replaced by the cell's own opposite population
                    // (+ lid), per thread -- the arithmetic of pull_cell().
                    if (wb_ok && !lwall && !rwall) {
                        // prefetched wall values of this plane (buffer c & 1),
                        // then the next plane's prefetch into the other buffer
                        if (wl_row || wl_col) {
                            asm volatile("cp.async.wait_group 0;" ::: "memory");
                            const T* const wb = wallbuf + (c & 1) * C::WALLE;
                            static_for<0, kQ>([&](auto kc) {
                                constexpr int k = decltype(kc)::value;
                                constexpr int i = slot_dir(k);
                                constexpr int cy = can_cy(i), cz = can_cz(i);
                                bool hit = false;
                                T v = T(0);
                                if constexpr (cy != 0) {
                                    if (wl_row && cy == wsy) {
                                        v = wb[b * 5 + wall_idx(k, 1, cy)];
                                        hit = true;
                                    }
                                }
                                if constexpr (cz != 0) {
                                    if (wl_col && cz == wsz) {
                                        v = wb[(C::HZ + a) * 5 + wall_idx(k, 2, cz)];
                                        hit = true;
                                    }
                                }
                                if (hit) {
                                    if constexpr (cz == -1) {
                                        if (qz == g.nz - 1) v = v + P.lid[k];
                                    }
                                    fs[i] = v;
                                }
                            });
                        }
                        if (p + 1 <= p_last) wall_prefetch(p + 1, (c + 1) & 1);
                    } else if ((edge_tile || lwall || rwall) && q_in) {
                        if (wb_ok && p + 1 <= p_last) wall_prefetch(p + 1, (c + 1) & 1);
                        const long long self = plane_base_t<RING>(g, p) + (long long)qy * g.nzp + qz;
                        static_for<0, kQ>([&](auto kc) {
                            constexpr int k = decltype(kc)::value;
                            constexpr int i = slot_dir(k);
                            constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
                            bool wall = false;
                            if constexpr (cx == 1) wall = wall || lwall;
                            if constexpr (cx == -1) wall = wall || rwall;
                            if constexpr (cy == 1) wall = wall || wyl;
                            if constexpr (cy == -1) wall = wall || wyh;
                            if constexpr (cz == 1) wall = wall || wzl;
                            if constexpr (cz == -1) wall = wall || wzh;
                            if (wall) {
                                T v = A[self + (long long)slot_opp(k) * g.pq];
                                if constexpr (cz == -1) {
                                    if (qz == g.nz - 1) v = v + P.lid[k];
                                }
                                fs[i] = v;
                            }
                        });
                    }
                }
            }
        };
        if constexpr (EARLY) {
            read_stage();
            __syncthreads();
            if (tid == 0 && has1 && p + 2 <= p_last) issue(p + 2, s);
        }
        // ---------------- step 2 of dest plane d = p - 2, step 1 of plane p ----------------
        // A thread owns (up to) one cell of each; the two collisions are
        // independent, so they run as two interleaved dependency chains
        // (bgk_collide2: twice the ILP of back-to-back collisions).  Warps
        // that own no step-2 cell (warp-uniform) collide their step-1 cell alone.
        const int d = p - 2;
        const bool do2 = d >= xs && warp2;
        T f2[kQ];
        if (do2) {
            const T* const qM = ringM + (d & 1) * 5 * C::RP;
            const T* const qZ = ringZ + (d % 3) * 9 * C::RP;
            const T* const qP = ringP + (d & 3) * 5 * C::RP;
            const int t = in2 ? y2 * TZ + z2 : 0;
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (k < 5) f2[slot_dir(k)] = qM[k * C::RP + t];
                else if constexpr (k < 14) f2[slot_dir(k)] = qZ[(k - 5) * C::RP + t];
                else f2[slot_dir(k)] = qP[(k - 14) * C::RP + t];
            });
        }
        if constexpr (!EARLY) read_stage();
        if (do2 && has1) bgk_collide2<T>(f2, fs, P.omega);
        else if (do2) bgk_collide<T>(f2, P.omega);
        else if (has1) bgk_collide<T>(fs, P.omega);
        if (do2 && in2) {
            // slot-plane bases are CTA-uniform (uniform datapath); the
            // thread adds its 32-bit in-plane offset: one IMAD.WIDE per store
            int dslot = d + 2;  // ring slot of the output plane
            if constexpr (RING) {
                dslot += out_poff;
                dslot = dslot >= g.pmod ? dslot - g.pmod : dslot;
            }
            T* const Bd = B + (long long)dslot * g.px;
            // (32-bit slot offsets held in uniform registers -- 2 instead of
            // 3 instructions per store address -- measured 1% slower)
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                __stcs(Bd + (long long)k * g.pq + st_off, f2[slot_dir(k)]);
            });
            if (fany) store_frame(g, Bd, y0 + y2, z0 + z2, fm, [](int) { return true; }, f2);
            if constexpr (!RING) {
                // Fused halo: the planes a neighbouring
                // slab reads as ghosts also go straight into its next-sweep
                // buffer -- planes 0 (all slots) and 1 (c_x = -1 slots) into
                // the left neighbour's x = nxl, nxl+1; planes nxl-2 (c_x = +1
                // slots) and nxl-1 (all) into the right neighbour's x = -2, -1
                // (the halo plan's spans, fill_plan) -- instead of a separate
                // exchange after the sweep.
                if (d <= 1 && haloL) {
                    T* const H = haloL + (long long)(g.nxl + 2 + d) * g.px;
                    static_for<0, kQ>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        if (d == 0 || k < kSlotsM) __stcs(H + (long long)k * g.pq + st_off, f2[slot_dir(k)]);
                    });
                    if (fany) store_frame(g, H, y0 + y2, z0 + z2, fm, [d](int k) { return d == 0 || k < kSlotsM; }, f2);
                }
                if (d >= g.nxl - 2 && haloR) {
                    T* const H = haloR + (long long)(d - g.nxl + 2) * g.px;
                    static_for<0, kQ>([&](auto kc) {
                        constexpr int k = decltype(kc)::value;
                        if (d == g.nxl - 1 || k >= kSlotP0) __stcs(H + (long long)k * g.pq + st_off, f2[slot_dir(k)]);
                    });
                    if (fany)
                        store_frame(g, H, y0 + y2, z0 + z2, fm, [d, &g](int k) { return d == g.nxl - 1 || k >= kSlotP0; },
                                    f2);
                }
            }
        }
        // ---------------- step 1: plane p (pushes) ----------------
        T* const wM = ringM + ((p + 1) & 1) * 5 * C::RP;  // dest p-1 (p + 1 has the parity of p - 1)
        T* const wZ = ringZ + ((p + 3) % 3) * 9 * C::RP;  // dest p
        T* const wP = ringP + ((p + 1) & 3) * 5 * C::RP;  // dest p+1
        if constexpr (BC == BC_CAVITY) {
            // wall links of c_x = -1 directions held from plane p-1 -> dest p-1
            if (held_mask) {
                static_for<0, 5>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    if (held_mask & (1u << k)) wM[k * C::RP + toff] = heldP[k];
                });
                held_mask = 0;
            }
        }
        if (has1) {
            T (&f)[kQ] = fs;
            if (q_in) {
                // ---- pushes: direction i streams to (p + cx, a - 1 + cy, b - 1 + cz) ----
                // (a warp-uniform branch for tile rows away from the y edges,
                // whose pushes need only two lane predicates: -4%, reverted)
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
                        T* const bP = ringP + (p & 3) * 5 * C::RP;  // dest p
                        static_for<0, kQ>([&](auto kc) {
                            constexpr int k = decltype(kc)::value;
                            constexpr int i = slot_dir(k);
                            constexpr int cx = can_cx(i), cy = can_cy(i), cz = can_cz(i);
                            // the source x - c_i is beyond a wall: only the
                            // cell's own wall flags in the directions c_i has
                            bool out = false;
                            if constexpr (cy == 1) out = out || wyl;
                            if constexpr (cy == -1) out = out || wyh;
                            if constexpr (cz == 1) out = out || wzl;
                            if constexpr (cz == -1) out = out || wzh;
                            if constexpr (cx == 1) out = out || lwall;
                            if constexpr (cx == -1) out = out || rwall;
                            if (out) {
                                T v = f[can_opp(i)];
                                if constexpr (cz == -1) {
                                    if (wzh) v = v + P.lid[k];
                                }
                                if constexpr (k < 5) {
                                    heldP[k] = v;
                                    held_mask |= 1u << k;
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
        }
        if constexpr (!EARLY) {
            __syncthreads();  // stage of plane p consumed; ring of destination p-1 complete
            if (tid == 0 && has1 && p + 2 <= p_last) issue(p + 2, s);
        }
    }
    sc_finish(xs);
}

// ------------------------------------------------------------------ host --
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

// Tile shape (TY x TZ output cells per CTA).  LBM_K2_TILE=<TY>x<TZ> selects
// one of the compiled shapes (tuning runs); the default is the measured best.
int tile_choice(int esize) {
    static int choice[2] = {-1, -1};
    int& c = choice[esize == 8 ? 0 : 1];
    if (c < 0) {
        c = 0;
        if (const char* e = getenv("LBM_K2_TILE")) {
            if (!strcmp(e, "8x32")) c = 1;
            else if (!strcmp(e, "8x16")) c = 2;
            else if (!strcmp(e, "16x16")) c = 3;
            else if (!strcmp(e, "16x32")) c = 4;
        }
    }
    return c;
}

constexpr int kMaxDevices = 64;

int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        dev = 0;
    }
    return dev;
}

int num_sms() {
    static std::atomic<int> cache[kMaxDevices];  // 0 = not yet queried (per device ordinal)
    const int dev = current_device();
    int n = cache[dev].load(std::memory_order_relaxed);
    if (!n) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

// x chunks of at most k2_max_chunk planes (launch_k2_impl): fp64 72 on
// large cross-sections (`wide`), else 32 -- the single-copy ring its own
// cap (k2_sc_max_chunk), which sets its gap (k2_sc_gap); fp32 48
template <typename T>
constexpr int k2_max_chunk(bool wide = false) {
    return sizeof(T) == 8 ? (wide ? 72 : 32) : 48;
}
// single-copy ring (K2_SC): its chunk cap, which sets the ring gap (the
// ring's extra planes).  fp64 72 planes (gap 148) on slabs of >= 1024
// planes, where the gap costs <= 14% of a lattice copy (bench K2_SC frac
// 0.764 -> 0.790 at 32 -> 72 on config 5, 0.784 at 56: interleaved A/B),
// else 32 (gap 68: a short slab keeps its ring close to one copy); fp32 48
template <typename T>
constexpr int k2_sc_max_chunk(int nxl) {
    return (sizeof(T) == 8 && nxl >= 1024) ? 72 : k2_max_chunk<T>(false);
}

template <typename T, int BC, int TY, int TZ, bool EARLY, bool RING, bool YB = false>
cudaError_t launch_k2_impl(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, int out_poff,
                           unsigned* sc_sync, T* haloL, T* haloR, cudaStream_t s, int xbeg2 = 0, int nxs2 = 0) {
    using C = K2Cfg<T, TY, TZ>;
    constexpr int NT = C::NT;
    auto kern = k2_sweep<T, BC, TY, TZ, EARLY, RING, YB>;
    // The large-shared-memory opt-in is a per-device (per-context) function
    // attribute: set it once per device ordinal this process launches on
    // (setting it twice from racing threads is harmless).
    static std::atomic<int> occ_cache[kMaxDevices];  // 0 = not yet set on that device
    const int dev = current_device();
    int occ = occ_cache[dev].load(std::memory_order_acquire);
    if (occ < 1) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, C::SMEM);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        occ_cache[dev].store(occ, std::memory_order_release);
    }
    EncodeFn enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    const SlabGeom& g = P.g;
    CUtensorMap map;
    // Cavity: the cells only, so boxes reaching past a wall are zero-filled
    // (the wall lanes substitute those entries).  Periodic: the whole plane
    // including the ghost frame, from the buffer base (A is the cell origin).
    // (X-Y cavity blocks: frame rows but no frame columns -- z stays zero-filled)
    const T* const base = A - g.org;
    const cuuint64_t dims[3] = {cuuint64_t(g.zoff ? g.nzp : g.nz), cuuint64_t(g.ny + 2 * g.gy),
                                cuuint64_t(g.pmod) * kQ};
    const cuuint64_t strides[2] = {cuuint64_t(g.nzp) * sizeof(T), cuuint64_t(g.pq) * sizeof(T)};
    const cuuint32_t box[3] = {cuuint32_t(C::BW), cuuint32_t(C::HY), 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    static CUtensorMapL2promotion promo = [] {
        // LBM_K2_L2PROMO=none|64|128|256 (tuning runs).  Default 64 B: the
        // least DRAM over-fetch of the halo edges (256-plane fp64 sweep:
        // 1.18x the algorithmic reads vs 1.24x none / 1.31x 256 B), same speed.
        const char* e = getenv("LBM_K2_L2PROMO");
        if (e && !strcmp(e, "none")) return CU_TENSOR_MAP_L2_PROMOTION_NONE;
        if (e && !strcmp(e, "256")) return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        if (e && !strcmp(e, "128")) return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    }();
    CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<T*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    // x chunks: fill the machine in whole waves; each chunk re-computes 2 halo planes of step 1
    const long long ntiles = (long long)((g.ny + TY - 1) / TY) * ((g.nz + TZ - 1) / TZ);
    const long long slots = (long long)num_sms() * occ;
    // x chunks of at most kMaxChunk planes: co-resident CTAs start a chunk
    // together and stay within a few planes of each other, so the halo rows
    // and columns one CTA stages are still in L2 when its neighbours stage
    // them (DRAM reads 1.13x / 1.19x / 1.38x / 1.49x the algorithmic bytes
    // at 32 / 64 / 128 / 512 planes, 512^3 fp64; 1024x512x512 fp64 equal
    // within noise at 32-64 planes, 256^3 periodic 5% faster at 32 than 64).
    // Among those, fill whole waves of the machine; each chunk re-computes
    // ~2.5 planes of step 1.
    // fp32 tiles (16x32) re-read relatively less x-halo per plane: 48 planes
    // measured best there (65.9k -> 67.4k burst; 64 equal, 80 -4% in the
    // sustained bench).  fp64: 32 planes at full clock (37.6k vs 35.8k at
    // 56; 256^3 periodic 27.0k vs 26.2k), but a large lattice runs into the
    // 1 kW power cap, and there the step-1 halo planes cost more than the
    // L2 misses: sustained config 5 32.2k at 32, 32.4k at 40, 32.5k at
    // 48-64, 29.9k at 128; config 4 32.2k -> 32.75k at 56.  So 56 where a
    // chunk-plane holds >= 4 waves of tiles (configs 4, 5), else 32.  Round
    // 2, with the z-strip tile order (less drift cost): the bench's K2 frac
    // 0.784 at 56, 0.785 at 64, 0.789 at 72-88, 0.787 at 96 -> 72.
    const bool wide = !RING && ntiles >= 4 * slots;
    // (ring: the cap its gap was sized for, gap = pmod - nxl - 4 = 2 cap + 4)
    const int kMaxChunk = RING ? std::max(1, (g.pmod - g.nxl - 8) / 2)
                               : wide ? k2_max_chunk<T>(true) : k2_max_chunk<T>(false);
    int best = 1;
    double best_cost = 1e300;
    const int ranges = nxs2 > 0 ? 2 : 1;
    for (int nch = 1; nch <= nxs && nch * ranges <= 65535; ++nch) {  // (grid.y limit)
        const int chunk = (nxs + nch - 1) / nch;
        if (chunk > kMaxChunk && nch < nxs && (nch + 1) * ranges <= 65535) continue;
        const long long items = ntiles * ((nxs + chunk - 1) / chunk) * ranges;
        const double waves = double((items + slots - 1) / slots);
        // per CTA: its planes (the average chunk), ~2.5 recomputed step-1
        // planes and ~2 planes of pipeline fill (one CTA per SM: nothing
        // overlaps a CTA's first TMA round trip)
        const double cost = waves * (double(nxs) / nch + 2.5 + 2.0);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = nch;
        }
        if (chunk <= 8) break;
    }
    int chunk = (nxs + best - 1) / best;
    static const int force_chunk = [] {
        const char* e = getenv("LBM_K2_CHUNK");  // planes per CTA (tuning runs)
        return e ? atoi(e) : 0;
    }();
    if (force_chunk > 0) chunk = min(force_chunk, nxs);
    if (sc_sync) chunk = min(chunk, kMaxChunk);  // the ring gap assumes it (k2_sc_gap)
    const int nch1 = (nxs + chunk - 1) / chunk;
    const dim3 grid(unsigned(ntiles), unsigned(nch1 * ranges));
    if (sc_sync) {  // tickets and per-chunk completion counters start at zero
        cudaError_t e = cudaMemsetAsync(sc_sync, 0, sizeof(unsigned) * (1 + grid.y), s);
        if (e != cudaSuccess) return e;
    }
    static const int l2last = [] {
        const char* e = getenv("LBM_K2_EVICT_LAST");  // A/B runs: 0 = evict_normal staging loads
        return (e && e[0] == '0') ? 0 : 1;
    }();
    // tile-order strip width in z tiles (kernel comment): fp64 cavity 8
    // (config 5: DRAM reads 49.1 -> 46.7 GB per launch, +0.3% sustained; 4
    // and 2 lose more at the strip seams than they gain); fp32 (16x32
    // tiles: 8 measured -0.5%) and periodic boxes (1024x512x512 fp64: -3%)
    // whole rows.  LBM_K2_ZBLOCK overrides (tuning runs).
    static const int zbw_env = [] {
        const char* e = getenv("LBM_K2_ZBLOCK");
        return e ? std::max(1, std::min(255, atoi(e))) : 0;
    }();
    const int zbw = zbw_env ? zbw_env : ((sizeof(T) == 8 && BC == BC_CAVITY) ? 8 : 255);

    kern<<<grid, NT, C::SMEM, s>>>(map, A, B, P, xbeg, xbeg + nxs, chunk, out_poff, sc_sync, haloL, haloR, xbeg2,
                                   nch1, l2last | (zbw << 8));
    return cudaGetLastError();
}

}  // namespace

// shared with the other lattices' two-step sweep (dqq.cu)
void* tma_encode_entry() { return reinterpret_cast<void*>(get_encode()); }
int device_sm_count() { return num_sms(); }
int device_ordinal() { return current_device(); }

template <typename T>
bool k2_supported(const SlabGeom& g) {
    if (!get_encode()) return false;
    // TMA: row pitch a multiple of 16 B (nzp is padded to 32 B); the combined
    // (x, slot) dimension and the boxes fit the descriptor limits.
    return (g.nzp * sizeof(T)) % 16 == 0 && (long long)g.pmod * kQ < (1LL << 31) && g.nxl >= 1;
}

// Single-copy ring (launch_k2 with sc_sync): a sweep writes f*(t+1) of plane
// d into the ring slot of input plane d - gap.  With chunks of L <= k2_max_chunk
// planes, chunk j writes input planes [jL - gap, (j+1)L - gap), which chunk
// j-1 and later no longer read iff gap >= 2L + 2 ([jL - 2, (j+1)L + 1] is
// what chunk j reads); chunks <= j-2 have finished (the ticket wait).
template <typename T>
int k2_sc_gap(int nxl) {
    return 2 * k2_sc_max_chunk<T>(nxl) + 4;
}


template <typename T>
cudaError_t launch_k2(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s, int out_poff,
                      unsigned* sc_sync, T* halo_left, T* halo_right, int xbeg2, int nxs2) {
    if (nxs2 > 0 && (nxs2 != nxs || sc_sync)) return cudaErrorInvalidValue;
    if (nxs <= 0) return cudaSuccess;
    const bool per = P.g.bc == BC_PERIODIC;
    // Default: read the stage into registers and issue the next TMA before
    // the collisions (measured faster with short chunks: fp64 33.6k vs 30.2k
    // MLUPS); LBM_K2_EARLY=0 issues after them (tuning runs).  (A
    // warp-specialised variant of this kernel -- S1/S2 groups on named
    // barriers, 608 threads -- measured 28.7k: DESIGN.md section 5.)
    static const bool early = [] {
        const char* e = getenv("LBM_K2_EARLY");
        return !(e && e[0] == '0');
    }();
    if (sc_sync) {  // single-copy ring storage: the default shape only
        constexpr int TY = sizeof(T) == 8 ? 8 : 16, TZ = 32;
        return per ? launch_k2_impl<T, BC_PERIODIC, TY, TZ, true, true>(A, B, P, xbeg, nxs, out_poff, sc_sync, nullptr, nullptr, s)
                   : launch_k2_impl<T, BC_CAVITY, TY, TZ, true, true>(A, B, P, xbeg, nxs, out_poff, sc_sync, nullptr, nullptr, s);
    }
    // X-Y blocks: the y-block kernel variants (EARLY issue order only)
    const bool yb = !P.g.ylo_wall || !P.g.yhi_wall || !P.g.ywrap;
    if (yb && !early) return cudaErrorNotSupported;
#define LBM_K2_TILE_CASE(TY, TZ)                                                                              \
    if constexpr (K2Cfg<T, TY, TZ>::FITS) {                                                                   \
        if (yb)                                                                                               \
            return per ? launch_k2_impl<T, BC_PERIODIC, TY, TZ, true, false, true>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2) \
                       : launch_k2_impl<T, BC_CAVITY, TY, TZ, true, false, true>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2);  \
        if (early)                                                                                            \
            return per ? launch_k2_impl<T, BC_PERIODIC, TY, TZ, true, false>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2) \
                       : launch_k2_impl<T, BC_CAVITY, TY, TZ, true, false>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2);  \
        return per ? launch_k2_impl<T, BC_PERIODIC, TY, TZ, false, false>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2)    \
                   : launch_k2_impl<T, BC_CAVITY, TY, TZ, false, false>(A, B, P, xbeg, nxs, 0, nullptr, halo_left, halo_right, s, xbeg2, nxs2);     \
    } else {                                                                                                  \
        return cudaErrorInvalidConfiguration;                                                                 \
    }
    switch (tile_choice(sizeof(T))) {
        case 1: LBM_K2_TILE_CASE(8, 32);
        case 2: LBM_K2_TILE_CASE(8, 16);
        case 3: LBM_K2_TILE_CASE(16, 16);
        case 4: LBM_K2_TILE_CASE(16, 32);
        default:
            if constexpr (sizeof(T) == 8) {
                LBM_K2_TILE_CASE(8, 32);
            } else {
                LBM_K2_TILE_CASE(16, 32);
            }
    }
#undef LBM_K2_TILE_CASE
}

template bool k2_supported<double>(const SlabGeom&);
template bool k2_supported<float>(const SlabGeom&);
template cudaError_t launch_k2<double>(const double*, double*, const StepParams<double>&, int, int, cudaStream_t,
                                       int, unsigned*, double*, double*, int, int);
template cudaError_t launch_k2<float>(const float*, float*, const StepParams<float>&, int, int, cudaStream_t, int,
                                      unsigned*, float*, float*, int, int);
template int k2_sc_gap<double>(int);
template int k2_sc_gap<float>(int);

}  // namespace lbm

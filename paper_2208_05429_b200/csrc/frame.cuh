// frame.cuh -- the periodic ghost frame (SlabGeom):
// which frame rows / columns of a (x, slot) plane hold copies of a cell, and
// the stores that keep them current from the sweeps' own outputs (K2, K3).
//
// Frame rows y in [-gy, 0) and [ny, ny + gy), frame columns z in [-S, 0) and
// [nz, nz + S), S = g.zoff (one 32 B sector, so column copies are whole
// sectors written by S adjacent lanes); a frame entry holds the cell
// (y mod ny, z mod nz).
#pragma once

#include "d3q19.cuh"

namespace lbm {

// bit 0: the cell's own row / column; bit 1 + j: frame row / column j
struct FrameMask {
    unsigned rows = 1u, cols = 1u;
    __device__ __forceinline__ bool any() const { return (rows | cols) != 1u; }
};

__device__ __forceinline__ FrameMask frame_mask(const SlabGeom& g, int y, int z) {
    FrameMask m;
    // (X-Y blocks: a y-partitioned slab's frame rows are its neighbours' rows)
    for (int j = 0; j < (g.ywrap ? 2 * g.gy : 0); ++j) {
        const int t = j < g.gy ? j - g.gy : g.ny + j - g.gy;
        if (((t % g.ny) + g.ny) % g.ny == y) m.rows |= 2u << j;
    }
    const int S = g.zoff;
    for (int j = 0; j < 2 * S; ++j) {
        const int t = j < S ? j - S : g.nz + j - S;
        if (((t % g.nz) + g.nz) % g.nz == z) m.cols |= 2u << j;
    }
    return m;
}

// The frame copies of cell (y, z), values v (canonical order), into the
// plane whose slot 0 starts (cell origin) at D, for the slots where keep(k):
// every (row, column) of {y and its frame rows} x {z and its frame columns}
// except the cell itself.  Iterates over set bits only.
template <typename T, typename Keep>
__device__ __forceinline__ void store_frame(const SlabGeom& g, T* D, int y, int z, FrameMask m, Keep keep,
                                            const T (&v)[kQ]) {
    const int S = g.zoff, gy = g.gy;
#pragma unroll 1
    for (unsigned rm = m.rows; rm; rm &= rm - 1) {
        const int ra = __ffs(int(rm)) - 1;
        const int ry = ra == 0 ? y : (ra <= gy ? ra - 1 - gy : g.ny + ra - 1 - gy);
#pragma unroll 1
        for (unsigned cm = ra == 0 ? m.cols & ~1u : m.cols; cm; cm &= cm - 1) {
            const int cb = __ffs(int(cm)) - 1;
            const int rz = cb == 0 ? z : (cb <= S ? cb - 1 - S : g.nz + cb - 1 - S);
            T* const dst = D + (long long)ry * g.nzp + rz;
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if (keep(k)) __stcs(dst + (long long)k * g.pq, v[slot_dir(k)]);
            });
        }
    }
}

}  // namespace lbm

// kernels.h -- host launchers of the library's kernels (internal; not ABI).
#pragma once

#include "d3q19.cuh"

namespace lbm {

// K1: one fused collide+stream step, A = f*(t-1) -> B = f*(t), slab-local
// planes [xbeg, xbeg + nxs) and [xbeg2, xbeg2 + nxs2) (one grid: the two
// edge ranges of an overlapped sweep).  A's ghost planes must be valid.
template <typename T>
cudaError_t launch_k1(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s, int xbeg2 = 0,
                      int nxs2 = 0);

// K1 in place on single-copy ring storage: output plane x to ring slot
// x + 2 + out_poff (= the slot of input plane x - 4); sync = device scratch
// of nxl + 1 words.
// unstream = true: K0b's inverse stream of the canonical state in the ring
// instead of a step (X-slab single-copy init / set_populations).
template <typename T>
cudaError_t launch_k1_sc(T* F, const StepParams<T>& P, int out_poff, unsigned* sync, cudaStream_t s,
                         bool unstream = false);
constexpr int kK1ScGap = 4;

// K2: two fused steps, A = f*(t-1) -> B = f*(t+1) on planes [xbeg, xbeg+nxs).
// A's two ghost planes per side must be valid.  Output plane d goes to ring
// slot d + 2 + out_poff (mod P.g.pmod).  Single-copy ring storage: B == A,
// out_poff = P.g.poff - k2_sc_gap (mod pmod), and sc_sync = device scratch of
// nxl + 1 words (the chunk-ordered tickets: at most one chunk per plane).
// Fused halo (two-buffer storage only): halo_left / halo_right = the next-sweep
// buffer of the left / right neighbour slab (or this slab's own, periodic
// single slab), which then receives its ghost planes from this sweep's stores.
// Two ranges (xbeg2, nxs2 > 0; two-buffer storage only): planes [xbeg2,
// xbeg2 + nxs2) in the same grid, nxs2 == nxs (the edge ranges of an
// overlapped X-slab sweep: one launch instead of two).
template <typename T>
cudaError_t launch_k2(const T* A, T* B, const StepParams<T>& P, int xbeg, int nxs, cudaStream_t s, int out_poff = 0,
                      unsigned* sc_sync = nullptr, T* halo_left = nullptr, T* halo_right = nullptr, int xbeg2 = 0,
                      int nxs2 = 0);
template <typename T>
int k2_sc_gap(int nxl);  // the ring's extra planes for a slab of nxl planes
template <typename T>
bool k2_supported(const SlabGeom& g);

// Periodic ghost frame of the slab's own planes [0, nxl) from their cells
// (F = cell origin); a no-op without a frame (cavity).
template <typename T>
cudaError_t launch_frame_fill(T* F, const SlabGeom& g, cudaStream_t s);
// nbands bands of band_bytes, src/dst strides in bytes (NCCL X-Y row bands)
cudaError_t launch_band_copy(const void* src, long long src_stride_bytes, void* dst, long long dst_stride_bytes,
                             long long band_bytes, int nbands, cudaStream_t s);

// K3 (k3.cu): three fused steps per HBM pass, A = f*(t-1) -> B = f*(t+2),
// the whole slab; fp32, periodic, one slab spanning x (k3_supported).
template <typename T>
bool k3_supported(const SlabGeom& g);
template <typename T>
cudaError_t launch_k3(const T* A, T* B, const StepParams<T>& P, cudaStream_t s);

// D3Q15 / D3Q27 (dqq.cu): canonical storage [q][nx][ny][nzp], one fused
// collide + push step per launch; a single slab, no ghost planes.
struct DqqGeom {
    int q, nx, ny, nz, nzp, bc;
    // X-slab faces open to a neighbour slab (NCCL ranks): links leaving the
    // slab through them are stored into the ghost plane x = -1 / nx (the
    // buffers carry one per side) and moved by the halo exchange; a closed
    // face is a wall (cavity) or wraps in the kernel (periodic, one slab)
    int xlo_open, xhi_open;
    long long pq;  // elements per direction = nx * ny * nzp
};
template <typename T>
cudaError_t launch_dqq_step(const T* A, T* B, const DqqGeom& g, T omega, const double ulid[3], cudaStream_t s);
template <typename T>
cudaError_t launch_dqq_init(const double* rho, const double* u, T* A, const DqqGeom& g, cudaStream_t s);
template <typename T>
cudaError_t launch_dqq_moments(const T* A, const DqqGeom& g, int xbeg, int nxc, double* rho, double* u, int* flag,
                               cudaStream_t s);
template <typename T>
cudaError_t launch_dqq_box(const T* A, const DqqGeom& g, int x0, int y0, int z0, int lx, int ly, int lz, double* out,
                           cudaStream_t s);
template <typename T>
cudaError_t launch_dqq_import(const double* src, T* A, const DqqGeom& g, int xbeg, int nxc, cudaStream_t s);
void dqq_table(int q, int* c, double* w);
// Two fused collide + push steps per HBM pass (K2Q, dqq.cu): canonical
// A = f(t) -> B = f(t+2), the whole lattice.  cudaErrorNotSupported when the
// driver has no TMA descriptor encoder.
template <typename T>
cudaError_t launch_dqq_k2(const T* A, T* B, const DqqGeom& g, T omega, const double ulid[3], cudaStream_t s);
template <typename T>
cudaError_t launch_dqq_merge(T* B, const DqqGeom& g, cudaStream_t s);

// k2.cu helpers shared with dqq.cu: cuTensorMapEncodeTiled (null if the
// driver lacks it), the current device's SM count and ordinal
void* tma_encode_entry();
int device_sm_count();
int device_ordinal();

// canonical feq of planes [xbeg, xbeg + nxc) (nxc < 0: the whole slab); rho/u
// point at the first of those planes
template <typename T>
cudaError_t launch_k0_equilibrium(const double* rho, const double* u, T* C, const SlabGeom& g, cudaStream_t s,
                                  int xbeg = 0, int nxc = -1);

// Single-copy AA storage (aa.cu): one in-place step (odd = the gather/scatter
// half), and the canonical f / moments of either phase.
template <typename T>
cudaError_t launch_aa_step(T* F, const StepParams<T>& P, bool odd, cudaStream_t s);
template <typename T>
cudaError_t launch_aa_materialize(const T* F, const StepParams<T>& P, bool odd, int x0, int y0, int z0, int lx,
                                  int ly, int lz, double* out, cudaStream_t s);
template <typename T>
cudaError_t launch_aa_merge(T* dst, const T* src, const SlabGeom& g, int slot0, cudaStream_t s);
template <typename T>
cudaError_t launch_aa_moments(const T* F, const StepParams<T>& P, bool odd, int xbeg, int nxc, double* rho,
                              double* u, cudaStream_t s, int* flag = nullptr);
// K0 fused, one slab spanning the domain: the pull-form state of planes
// [xbeg, xbeg + nxc) from rho, u (src == null) or from canonical doubles
// src[19][wn][ny][nz]; the per-cell inputs hold the wn planes wx0, wx0 + 1,
// ... (mod nxl), which must include the planes' x neighbours.
template <typename T>
cudaError_t launch_k0_init_pull(const double* rho, const double* u, const double* src, T* A, const StepParams<T>& P,
                                int xbeg, int nxc, int wx0, int wn, cudaStream_t s);
template <typename T>
cudaError_t launch_k0_unstream(const T* C, T* A, const StepParams<T>& P, cudaStream_t s);
template <typename T>
cudaError_t launch_k0_import(const double* src, T* C, const SlabGeom& g, int xbeg, int nxc, cudaStream_t s);
template <typename T>
cudaError_t launch_k3_materialize(const T* A, const StepParams<T>& P, int x0, int y0, int z0, int lx, int ly,
                                  int lz, double* out, cudaStream_t s);
// flag (nullable): |= moments_flags() of every cell (degenerate / non-finite)
template <typename T>
cudaError_t launch_k3_moments(const T* A, const StepParams<T>& P, int xbeg, int nxc, double* rho, double* u,
                              cudaStream_t s, int* flag = nullptr);

}  // namespace lbm

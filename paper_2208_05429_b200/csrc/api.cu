// api.cu -- the C-ABI (include/lbm.h): validation, context, X-slab engine,
// halo exchange (local copies or NCCL send/recv), host transfers.
//
// Engine.  The process owns one slab (NCCL, one GPU per rank) or several
// slabs on one device (LOCAL, the multi-GPU data path emulated on one GPU).
// Each slab holds two buffers of post-collision populations (ping-pong) with
// two ghost planes per side.  lbm_step(n) runs floor(n/2) two-step sweeps
// (K2; Alg. 2's merge) and one one-step sweep (K1) if n
// is odd, with one halo exchange before every sweep -- the analogue of
// "we only synchronize at the intersection layers every two time steps"
// (PAPER.md:747-749).
#include <dlfcn.h>

#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include <nccl.h>

#include "../../include/lbm.h"
#include "kernels.h"
#include "peer.h"

using namespace lbm;

// ------------------------------------------------------------- NCCL ------
// libnccl.so.2 is loaded on demand (torch's copy when torch is imported
// first); the library has no link-time NCCL dependency.
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};
NcclApi g_nccl;

bool nccl_load() {
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
#define LOADSYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(GetErrorString, "ncclGetErrorString");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(CommGetAsyncError, "ncclCommGetAsyncError");
    LOADSYM(CommAbort, "ncclCommAbort");
#undef LOADSYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.GroupStart &&
                g_nccl.GroupEnd && g_nccl.Send && g_nccl.Recv && g_nccl.AllReduce && g_nccl.CommGetAsyncError &&
                g_nccl.CommAbort;
    return g_nccl.ok;
}

thread_local std::string t_last_error;

// Every ABI call leaves the calling thread's current device as it found it
// (the library switches to the context's device internally).
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
}  // namespace

// ------------------------------------------------------------- context ---
struct Slab {
    SlabGeom g;
    void* buf[2] = {nullptr, nullptr};
    int left = -1, right = -1;  // neighbour slab index (LOCAL/NONE) or rank (NCCL); -1 = wall
    int down = -1, up = -1;     // X-Y blocks: neighbour slab index in -y / +y; -1 = wall or none
    int y0 = 0;                 // X-Y blocks: first global row of this slab
    lbm_halo_plan plan;
};

struct lbm_ctx {
    int nx, ny, nz;
    double tau, ulid[3];
    lbm_dtype dt;
    lbm_opts opts;
    int device = 0;
    int nxl_proc = 0, x0_proc = 0;  // the planes this process owns (union of its slabs)
    std::vector<Slab> slabs;
    int cur = 0;
    bool initialized = false, ghosts_valid = false, poisoned = false;
    // periodic ghost frame (SlabGeom) of the state buffer's own planes is
    // current: K2 sweeps keep it, every other writer clears it
    bool frame_valid = false;
    int yblocks = 1;  // X-Y blocks (LOCAL, local_blocks_y): slabs per x range, split along y
    int ranks_y = 1;  // X-Y blocks across NCCL ranks (lbm_opts.ranks_y): this rank is one block
    void* ypack = nullptr;  // NCCL X-Y: [send down | send up | recv down | recv up] row bands
    size_t yband_bytes = 0;  // bytes of one of the four
    long t = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // halo exchange overlapped with the interior sweep
    cudaStream_t comm_stream = nullptr;  // highest priority: its NCCL kernels win free SMs
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    bool overlap = true;
    // single-copy AA storage (LBM_KERNEL_AA, aa.cu): buf[0] only, plus a
    // staging buffer for host transfers; aa_odd = the next step is odd
    bool aa = false, aa_odd = false;
    void* stage = nullptr;
    size_t stage_bytes = 0;
    // single-copy two-step storage (LBM_KERNEL_K2_SC): buf[0] is a ring of
    // pmod plane slots, the state window at slot g.poff; in-place sweeps
    // shift it down by sc_gap (K2) or kK1ScGap (K1) slots
    bool sc = false;
    int sc_gap = 0;
    unsigned* sc_sync = nullptr;
    bool fused_halo = true;  // K2 stores the neighbours' ghost planes itself (run_steps)
    // host read-back: moments of x chunk j+1 overlap the D2H of chunk j
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> chunk_events;
    ncclComm_t comm = nullptr;
    // NCCL watchdog (wait_stream): a progress event per sweep; a blocking
    // call fails with ENCCL on an asynchronous NCCL error or when no sweep
    // has completed for nccl_timeout_s seconds (a lost or stalled peer)
    std::vector<cudaEvent_t> progress;
    long long progress_issued = 0, progress_done = 0;
    double nccl_timeout_s = 120.0;
    // fused cross-GPU halo (LBM_HALO_PEER, peer.cu): the lattice buffers are
    // VMM allocations mapped into the neighbours; pnb[side][0..2] = the
    // left (0) / right (1) neighbour's buffer 0, buffer 1 and flag page as
    // mapped here; peer_seq = phases (sweeps, inits) this rank completed
    bool peer = false, peer_flush = false;
    peer::Alloc pmine[2], pflags;
    peer::Alloc pnb[2][3];
    unsigned peer_seq = 0;
    // D3Q15 / D3Q27 (dqq.cu; lbm_opts.lattice): canonical [q][nx][ny][nzp]
    // ping-pong buffers, one fused collide + push step per launch
    int q = 19;
    DqqGeom dg{};
    void* dbuf[2] = {nullptr, nullptr};   // cell (0, 0, 0) of slot 0 (NCCL slabs: past the ghost plane)
    void* dbase[2] = {nullptr, nullptr};  // the allocations
    long long dorg = 0;                   // elements from dbase to dbuf (one ghost plane, or 0)
    int dleft = -1, dright = -1;          // NCCL X-slab neighbour ranks of a D3Q15/27 slab (-1: wall / none)
    int dcur = 0;
    size_t esize = 8;
    int* d_flag = nullptr;
    // diagnostics
    long long launches = 0, k1_launches = 0, k2_launches = 0;
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    std::vector<long long> event_updates;
    size_t events_used = 0;
    std::string err;
};

namespace {

lbm_status fail(lbm_ctx* c, lbm_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_last_error = buf;
    if (c) {
        c->err = buf;
        if (st == LBM_ECUDA || st == LBM_ENCCL) c->poisoned = true;
    }
    return st;
}

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(c, LBM_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                                  \
    } while (0)

#define CKN(call)                                                                                        \
    do {                                                                                                 \
        ncclResult_t r_ = (call);                                                                        \
        if (r_ != ncclSuccess)                                                                           \
            return fail(c, LBM_ENCCL, "%s failed: %s", #call,                                            \
                        g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "nccl error");               \
    } while (0)

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ------------------------------------------------------ NCCL watchdog ----
// Failure detection for NCCL contexts (a lost or stalled peer must not hang
// the caller forever).  Every sweep records a progress event on the context
// stream; a blocking wait polls the stream, ncclCommGetAsyncError, and the
// progress events: an asynchronous NCCL error, or no sweep completing for
// nccl_timeout_s seconds (LBM_NCCL_TIMEOUT_S, default 120), aborts the
// communicator (its kernels stop) and fails with ENCCL; the context is then
// poisoned.  Without NCCL a wait is a plain stream synchronize.
lbm_status nccl_abort(lbm_ctx* c, const char* why) {
    if (c->comm && g_nccl.CommAbort) g_nccl.CommAbort(c->comm);
    c->comm = nullptr;
    return fail(c, LBM_ENCCL, "%s (communicator aborted)", why);
}

lbm_status record_progress(lbm_ctx* c) {
    if (!c->comm || c->progress.empty()) return LBM_OK;
    CK(cudaEventRecord(c->progress[size_t(c->progress_issued % (long long)c->progress.size())], c->stream));
    c->progress_issued++;
    return LBM_OK;
}

lbm_status wait_stream(lbm_ctx* c, cudaStream_t st) {
    if (!c->comm) {
        CK(cudaStreamSynchronize(st));
        return LBM_OK;
    }
    using clk = std::chrono::steady_clock;
    auto last = clk::now();
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) {
            c->progress_done = c->progress_issued;
            return LBM_OK;
        }
        if (e != cudaErrorNotReady) return fail(c, LBM_ECUDA, "stream wait: %s", cudaGetErrorString(e));
        ncclResult_t ar = ncclSuccess;
        if (g_nccl.CommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
            char why[256];
            snprintf(why, sizeof why, "NCCL asynchronous error: %s",
                     g_nccl.GetErrorString ? g_nccl.GetErrorString(ar) : "?");
            return nccl_abort(c, why);
        }
        // progress: the oldest sweep event still held in the ring
        const long long n = (long long)c->progress.size();
        if (c->progress_done < c->progress_issued - n) c->progress_done = c->progress_issued - n;
        while (c->progress_done < c->progress_issued) {
            const cudaError_t q = cudaEventQuery(c->progress[size_t(c->progress_done % n)]);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) return fail(c, LBM_ECUDA, "progress event: %s", cudaGetErrorString(q));
            c->progress_done++;
            last = clk::now();
        }
        if (std::chrono::duration<double>(clk::now() - last).count() > c->nccl_timeout_s) {
            char why[256];
            snprintf(why, sizeof why, "no progress for %.0f s: a peer rank is lost or stalled (LBM_NCCL_TIMEOUT_S)",
                     c->nccl_timeout_s);
            return nccl_abort(c, why);
        }
        if (spin > 64) usleep(spin > 4096 ? 1000 : 50);
    }
}

// Input validation that every rank agrees on: under NCCL the per-rank
// verdicts are max-reduced before anything collective follows, so a rank
// that rejects its input does not leave its peers blocked in an exchange.
lbm_status agree_valid(lbm_ctx* c, int bad, const char* why) {
    if (c->comm) {
        int* d = c->d_flag;
        CK(cudaMemcpyAsync(d, &bad, sizeof(int), cudaMemcpyHostToDevice, c->stream));
        CKN(g_nccl.AllReduce(d, d, 1, ncclInt32, ncclMax, c->comm, c->stream));
        CK(cudaMemcpyAsync(&bad, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        lbm_status st = wait_stream(c, c->stream);
        if (st != LBM_OK) return st;
        if (bad && !why) why = "another rank rejected its input";
    }
    if (bad) return fail(c, LBM_EINVAL, "%s (state is now undefined: initialise again)", why ? why : "invalid input");
    return LBM_OK;
}

// ------------------------------------------------- fused peer halo -----
// Flag page of a rank: the done-counter written by its left neighbour at
// byte 0, by its right neighbour at byte 64.  After every phase that reads
// ghost planes and writes a lattice buffer (init, a sweep) a rank bumps its
// counter into both neighbours' pages (a stream write, ordered after the
// phase's stores -- including its stores into the neighbours' buffers -- by
// the write's system-scope fence); before the next phase, and before any
// read of its ghost planes, it waits on its own page until both neighbours
// have completed as many phases.  All ranks run the same phase sequence.
constexpr size_t kFlagFromLeft = 0, kFlagFromRight = 64;

lbm_status peer_wait(lbm_ctx* c) {
    if (!c->peer || c->peer_seq == 0) return LBM_OK;
    const Slab& s = c->slabs[0];
    char* f = static_cast<char*>(c->pflags.va);
    if (s.left >= 0) CK(peer::stream_wait_geq(c->stream, f + kFlagFromLeft, c->peer_seq, c->peer_flush));
    if (s.right >= 0) CK(peer::stream_wait_geq(c->stream, f + kFlagFromRight, c->peer_seq, c->peer_flush));
    return LBM_OK;
}

lbm_status peer_signal(lbm_ctx* c) {
    if (!c->peer) return LBM_OK;
    c->peer_seq++;
    const Slab& s = c->slabs[0];
    // this rank is its left neighbour's right neighbour and vice versa
    if (s.left >= 0)
        CK(peer::stream_write(c->stream, static_cast<char*>(c->pnb[0][2].va) + kFlagFromRight, c->peer_seq));
    if (s.right >= 0)
        CK(peer::stream_write(c->stream, static_cast<char*>(c->pnb[1][2].va) + kFlagFromLeft, c->peer_seq));
    return LBM_OK;
}


// ghost_rows: periodic frame rows per side -- 2 (K2's reach), 3 for the
// three-step K3 (a K3 context's own plan; lbm_plan_halo describes K2's)
// yframe: an X-Y block -- ny is the block's own row count and the plane has
// 2 frame rows per side for the y-neighbours' rows (both boundary modes; the
// z frame columns stay periodic-only)
void fill_plan(int nx, int ny, int nz, size_t esize, int bc, int rank, int world, int nxl, int x0,
               lbm_halo_plan* p, int ghost_rows = 2, bool yframe = false) {
    memset(p, 0, sizeof *p);
    p->nx_local = nxl;
    p->x0 = x0;
    // rows start on 32 B sectors.  Periodic: the ghost frame (SlabGeom,
    // frame.cuh) -- 2 rows per side (K2's reach; 3 for K3) and a 32 B
    // sector of columns before z = 0 and after nz - 1 (the cells stay sector
    // aligned; the TMA boxes reach 16 B and <= 3 cells beyond the tile, and
    // whole-sector column copies need no L2 fill)
    const int sector = int(32 / esize);
    if (bc == LBM_BC_PERIODIC) {
        p->y_ghost = ghost_rows;
        p->z_offset = sector;
        p->nz_pitch = round_up(sector + nz + sector, sector);
    } else {
        p->y_ghost = yframe ? 2 : 0;
        p->z_offset = 0;
        p->nz_pitch = round_up(nz, sector);
    }
    p->cell0 = (long long)p->y_ghost * p->nz_pitch + p->z_offset;
    p->plane_q = (long long)(ny + 2 * p->y_ghost) * p->nz_pitch;
    p->plane_x = (long long)kQ * p->plane_q;
    p->buffer_elems = (long long)(nxl + 4) * p->plane_x;
    if (bc == LBM_BC_PERIODIC) {
        p->left = (rank - 1 + world) % world;
        p->right = (rank + 1) % world;
    } else {
        p->left = rank > 0 ? rank - 1 : -1;
        p->right = rank < world - 1 ? rank + 1 : -1;
    }
    const long long px = p->plane_x, pq = p->plane_q;
    // planes p = x + 2.  Left ghost: [plane 0 (x=-2): P slots | plane 1 (x=-1): all]
    p->recv_left_off = 0 * px + kSlotP0 * pq;
    // right ghost: [plane nxl+2 (x=nxl): all | plane nxl+3 (x=nxl+1): M slots]
    p->recv_right_off = (long long)(nxl + 2) * px;
    // to the left neighbour's right ghost: [x=0: all | x=1: M slots]
    p->send_left_off = 2 * px;
    // to the right neighbour's left ghost: [x=nxl-2: P slots | x=nxl-1: all]
    p->send_right_off = (long long)nxl * px + kSlotP0 * pq;
    p->span = (long long)kHaloSlots * pq;
    for (int k = 0; k < kQ; ++k) p->dir_of_slot[k] = slot_dir(k);
    // X-Y blocks: the frame-row bands of an (x, direction) plane (plane rows
    // r = y + y_ghost): own rows [0, gy) go down, [ny - gy, ny) go up; the
    // frame rows [-gy, 0) come from down, [ny, ny + gy) from up
    p->down = p->up = -1;
    p->ny_local = ny;
    p->y0 = 0;
    p->y_band = (long long)p->y_ghost * p->nz_pitch;
    p->send_down_off = (long long)p->y_ghost * p->nz_pitch;
    p->send_up_off = (long long)ny * p->nz_pitch;
    p->recv_down_off = 0;
    p->recv_up_off = (long long)(p->y_ghost + ny) * p->nz_pitch;
}

// The plan of rank `rank` in a (world / ranks_y) x ranks_y grid of X-Y
// blocks (lbm_opts.ranks_y): x slab rank / ranks_y, y block rank % ranks_y;
// neighbours as ranks.  ranks_y == 1: fill_plan's X-slab plan.
void fill_plan_xy(int nx, int ny, int nz, size_t esize, int bc, int rank, int world, int ranks_y,
                  lbm_halo_plan* p) {
    const int wx = world / ranks_y, bx = rank / ranks_y, byi = rank % ranks_y;
    const int nxl = nx / wx, nyl = ny / ranks_y;
    fill_plan(nx, nyl, nz, esize, bc, bx, wx, nxl, bx * nxl, p, 2, ranks_y > 1);
    if (p->left >= 0) p->left = p->left * ranks_y + byi;
    if (p->right >= 0) p->right = p->right * ranks_y + byi;
    if (ranks_y > 1) {
        const bool per = bc == LBM_BC_PERIODIC;
        const int dn = per ? (byi - 1 + ranks_y) % ranks_y : byi - 1, upi = per ? (byi + 1) % ranks_y : byi + 1;
        p->down = dn >= 0 ? bx * ranks_y + dn : -1;
        p->up = upi < ranks_y ? bx * ranks_y + upi : -1;
        p->y0 = byi * nyl;
    }
}

bool finite_vec(const double* v) {
    return v == nullptr || (std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]));
}

// Cell origin of lattice buffer b: kernels address cells from here (the
// periodic ghost frame lies before it, SlabGeom); exchanges move whole
// slot-planes from the buffer base.
template <typename T>
T* origin(const Slab& s, int b) {
    return static_cast<T*>(s.buf[b]) + s.g.org;
}

template <typename T>
StepParams<T> make_params(const lbm_ctx* c, const Slab& s) {
    StepParams<T> P;
    P.g = s.g;
    P.omega = T(1.0 / c->tau);
    const double rho_w = 1.0;
    // 6 w_i rho_w (c_i . u_lid) per slot
    for (int k = 0; k < kQ; ++k) {
        const int i = slot_dir(k);
        const double w = (i == 0) ? 1.0 / 3.0 : (can_axis(i) ? 1.0 / 18.0 : 1.0 / 36.0);
        const double cu = can_cx(i) * c->ulid[0] + can_cy(i) * c->ulid[1] + can_cz(i) * c->ulid[2];
        P.lid[k] = T(6.0 * w * rho_w * cu);
    }
    return P;
}

// ---------------------------------------------------------------- halo --
// Single-copy ring storage: the halo spans through the ring mapping, plane
// part by plane part (a span may straddle the end of the ring) -- right
// ghost [x=nxl: all | x=nxl+1: M] <- the right neighbour's [x=0 | x=1], left
// ghost [x=-2: P | x=-1: all] <- the left neighbour's [x=nxl-2 | x=nxl-1];
// the neighbour is the slab itself for a periodic single slab.  LOCAL: D2D
// copies; NCCL: the same parts as grouped send/recv, posted in the order of
// exchange() so the pairs match on a ring of two.
lbm_status exchange_sc(lbm_ctx* c, cudaStream_t st) {
    const size_t es = c->esize;
    struct Part {
        int x, slot0, nslots;
    };
    // parts a slab sends left / receives from the right, sends right / receives from the left
    auto parts_to_left = [](int) { return std::array<Part, 2>{{{0, 0, kQ}, {1, 0, kSlotsM}}}; };
    auto parts_from_right = [](int n) { return std::array<Part, 2>{{{n, 0, kQ}, {n + 1, 0, kSlotsM}}}; };
    auto parts_to_right = [](int n) { return std::array<Part, 2>{{{n - 2, kSlotP0, kQ - kSlotP0}, {n - 1, 0, kQ}}}; };
    auto parts_from_left = [](int) { return std::array<Part, 2>{{{-2, kSlotP0, kQ - kSlotP0}, {-1, 0, kQ}}}; };
    auto addr = [&](const Slab& s, const Part& q) {
        return static_cast<char*>(s.buf[0]) + (plane_base(s.g, q.x) + (long long)q.slot0 * s.g.pq) * (long long)es;
    };
    if (c->opts.comm == LBM_COMM_NCCL) {
        Slab& s = c->slabs[0];
        const ncclDataType_t ty = c->dt == LBM_F64 ? ncclFloat64 : ncclFloat32;
        const int n = s.g.nxl;
        CKN(g_nccl.GroupStart());
        if (s.left >= 0)
            for (const Part& q : parts_to_left(n))
                CKN(g_nccl.Send(addr(s, q), size_t(q.nslots) * s.g.pq, ty, s.left, c->comm, st));
        if (s.right >= 0)
            for (const Part& q : parts_from_right(n))
                CKN(g_nccl.Recv(addr(s, q), size_t(q.nslots) * s.g.pq, ty, s.right, c->comm, st));
        if (s.right >= 0)
            for (const Part& q : parts_to_right(n))
                CKN(g_nccl.Send(addr(s, q), size_t(q.nslots) * s.g.pq, ty, s.right, c->comm, st));
        if (s.left >= 0)
            for (const Part& q : parts_from_left(n))
                CKN(g_nccl.Recv(addr(s, q), size_t(q.nslots) * s.g.pq, ty, s.left, c->comm, st));
        CKN(g_nccl.GroupEnd());
        return LBM_OK;
    }
    for (Slab& s : c->slabs) {
        const int n = s.g.nxl;
        if (s.right >= 0) {
            const Slab& R = c->slabs[s.right];
            const auto src = parts_to_left(R.g.nxl), dst = parts_from_right(n);
            for (int k = 0; k < 2; ++k)
                CK(cudaMemcpyAsync(addr(s, dst[k]), addr(R, src[k]), size_t(dst[k].nslots) * s.g.pq * es,
                                   cudaMemcpyDeviceToDevice, st));
        }
        if (s.left >= 0) {
            const Slab& L = c->slabs[s.left];
            const auto src = parts_to_right(L.g.nxl), dst = parts_from_left(n);
            for (int k = 0; k < 2; ++k)
                CK(cudaMemcpyAsync(addr(s, dst[k]), addr(L, src[k]), size_t(dst[k].nslots) * s.g.pq * es,
                                   cudaMemcpyDeviceToDevice, st));
        }
    }
    return LBM_OK;
}

lbm_status exchange(lbm_ctx* c, int which, cudaStream_t st) {
    if (c->sc) return exchange_sc(c, st);
    if (c->opts.comm == LBM_COMM_NCCL) {
        Slab& s = c->slabs[0];
        char* b = static_cast<char*>(s.buf[which]);
        const size_t es = c->esize;
        const ncclDataType_t ty = c->dt == LBM_F64 ? ncclFloat64 : ncclFloat32;
        if (s.down >= 0 || s.up >= 0) {
            // X-Y blocks across ranks: first the frame-row bands of the own
            // planes with the y-neighbours (packed: one message per side),
            // then the x spans below, which carry those rows along (the x-y
            // corner entries come from the diagonal block); the same order
            // as the LOCAL copies
            const lbm_halo_plan& pl = s.plan;
            char* const own = b + 2 * s.g.px * (long long)es;  // plane x = 0
            const long long pqb = s.g.pq * (long long)es, bandb = pl.y_band * (long long)es;
            const int nb = s.g.nxl * kQ;
            char* const pk = static_cast<char*>(c->ypack);
            char* const snd_dn = pk;
            char* const snd_up = pk + c->yband_bytes;
            char* const rcv_dn = pk + 2 * c->yband_bytes;
            char* const rcv_up = pk + 3 * c->yband_bytes;
            if (s.down >= 0) CK(launch_band_copy(own + pl.send_down_off * es, pqb, snd_dn, bandb, bandb, nb, st));
            if (s.up >= 0) CK(launch_band_copy(own + pl.send_up_off * es, pqb, snd_up, bandb, bandb, nb, st));
            const size_t n = size_t(nb) * size_t(pl.y_band);
            CKN(g_nccl.GroupStart());
            // [send down, recv up], [send up, recv down]: pairs match even
            // when down == up (two y blocks in a ring, or this rank itself)
            if (s.down >= 0) CKN(g_nccl.Send(snd_dn, n, ty, s.down, c->comm, st));
            if (s.up >= 0) CKN(g_nccl.Recv(rcv_up, n, ty, s.up, c->comm, st));
            if (s.up >= 0) CKN(g_nccl.Send(snd_up, n, ty, s.up, c->comm, st));
            if (s.down >= 0) CKN(g_nccl.Recv(rcv_dn, n, ty, s.down, c->comm, st));
            CKN(g_nccl.GroupEnd());
            if (s.down >= 0) CK(launch_band_copy(rcv_dn, bandb, own + pl.recv_down_off * es, pqb, bandb, nb, st));
            if (s.up >= 0) CK(launch_band_copy(rcv_up, bandb, own + pl.recv_up_off * es, pqb, bandb, nb, st));
            c->launches += (s.down >= 0) * 2 + (s.up >= 0) * 2;
        }
        const size_t n = size_t(s.plan.span);
        CKN(g_nccl.GroupStart());
        // order: [send left, recv right], [send right, recv left]: pairs match
        // even when left == right (a ring of two)
        if (s.left >= 0) CKN(g_nccl.Send(b + s.plan.send_left_off * es, n, ty, s.left, c->comm, st));
        if (s.right >= 0) CKN(g_nccl.Recv(b + s.plan.recv_right_off * es, n, ty, s.right, c->comm, st));
        if (s.right >= 0) CKN(g_nccl.Send(b + s.plan.send_right_off * es, n, ty, s.right, c->comm, st));
        if (s.left >= 0) CKN(g_nccl.Recv(b + s.plan.recv_left_off * es, n, ty, s.left, c->comm, st));
        CKN(g_nccl.GroupEnd());
    } else {
        // X-Y blocks: first the frame rows of every block's own planes from
        // its y-neighbours (2 rows x whole pitch per (plane, slot): one
        // strided copy per side), then the x ghost planes below, which carry
        // those rows along -- so the x-y edge entries come from the diagonal
        // block
        if (c->yblocks > 1) {
            const size_t es = c->esize;
            for (Slab& s : c->slabs) {
                const long long gyz = (long long)s.g.gy * s.g.nzp;  // one frame band
                const size_t width = size_t(gyz) * es, pitch = size_t(s.g.pq) * es;
                char* mine = static_cast<char*>(s.buf[which]) + 2 * s.g.px * (long long)es;
                if (s.down >= 0) {  // my rows [-gy, 0) <- its rows [ny - gy, ny)
                    const Slab& D = c->slabs[s.down];
                    const char* src = static_cast<const char*>(D.buf[which]) + (2 * D.g.px + (long long)D.g.ny * D.g.nzp) * (long long)es;
                    CK(cudaMemcpy2DAsync(mine, pitch, src, pitch, width, size_t(s.g.nxl) * kQ, cudaMemcpyDeviceToDevice, st));
                }
                if (s.up >= 0) {  // my rows [ny, ny + gy) <- its rows [0, gy)
                    const Slab& U = c->slabs[s.up];
                    const char* src = static_cast<const char*>(U.buf[which]) + (2 * U.g.px + gyz) * (long long)es;
                    CK(cudaMemcpy2DAsync(mine + (gyz + (long long)s.g.ny * s.g.nzp) * (long long)es, pitch, src, pitch,
                                         width, size_t(s.g.nxl) * kQ, cudaMemcpyDeviceToDevice, st));
                }
            }
        }
        for (Slab& s : c->slabs) {
            char* dst = static_cast<char*>(s.buf[which]);
            const size_t bytes = size_t(s.plan.span) * c->esize;
            if (s.left >= 0) {
                const Slab& L = c->slabs[s.left];
                const char* src = static_cast<const char*>(L.buf[which]);
                CK(cudaMemcpyAsync(dst + s.plan.recv_left_off * c->esize, src + L.plan.send_right_off * c->esize,
                                   bytes, cudaMemcpyDeviceToDevice, st));
            }
            if (s.right >= 0) {
                const Slab& R = c->slabs[s.right];
                const char* src = static_cast<const char*>(R.buf[which]);
                CK(cudaMemcpyAsync(dst + s.plan.recv_right_off * c->esize, src + R.plan.send_left_off * c->esize,
                                   bytes, cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    return LBM_OK;
}

// AA X-slab halo (aa.cu).  forward (before an odd step or an odd-phase
// read-back): ghost x = -1 <- left's plane nxl-1, c_x = -1 slots; ghost
// x = nxl <- right's plane 0, c_x = +1 slots.  reverse (after an odd step):
// those ghost slots, now holding what the odd step scattered into the
// neighbours' edge cells, go back to the same neighbour locations.
// Five slot-planes per side, one contiguous run each.
template <typename T>
lbm_status exchange_aa_t(lbm_ctx* c, bool forward) {
    const size_t es = sizeof(T);
    auto off = [](const Slab& s, int x, int slot0) {
        return ((long long)(x + 2) * s.plan.plane_x + (long long)slot0 * s.plan.plane_q);
    };
    if (c->opts.comm == LBM_COMM_NCCL) {
        Slab& s = c->slabs[0];
        T* b = static_cast<T*>(s.buf[0]);
        const ncclDataType_t ty = c->dt == LBM_F64 ? ncclFloat64 : ncclFloat32;
        const size_t n = size_t(5 * s.plan.plane_q);
        const int nxl = s.g.nxl;
        // reverse: received into scratch (the staging buffer), then merged
        T* scratch_r = static_cast<T*>(c->stage);  // from right -> my (nxl-1, M)
        T* scratch_l = scratch_r + n;               // from left  -> my (0, P)
        if (!forward && 2 * n * es > c->stage_bytes) return fail(c, LBM_ENOMEM, "AA halo scratch too small");
        CKN(g_nccl.GroupStart());
        if (forward) {
            // to left: my (0, P) -> its ghost (nxl, P); to right: my (nxl-1, M) -> its ghost (-1, M)
            if (s.left >= 0) CKN(g_nccl.Send(b + off(s, 0, kSlotP0), n, ty, s.left, c->comm, c->stream));
            if (s.right >= 0) CKN(g_nccl.Recv(b + off(s, nxl, kSlotP0), n, ty, s.right, c->comm, c->stream));
            if (s.right >= 0) CKN(g_nccl.Send(b + off(s, nxl - 1, 0), n, ty, s.right, c->comm, c->stream));
            if (s.left >= 0) CKN(g_nccl.Recv(b + off(s, -1, 0), n, ty, s.left, c->comm, c->stream));
        } else {
            // to left: my ghost (-1, M) -> its (nxl-1, M); to right: my ghost (nxl, P) -> its (0, P)
            if (s.left >= 0) CKN(g_nccl.Send(b + off(s, -1, 0), n, ty, s.left, c->comm, c->stream));
            if (s.right >= 0) CKN(g_nccl.Recv(scratch_r, n, ty, s.right, c->comm, c->stream));
            if (s.right >= 0) CKN(g_nccl.Send(b + off(s, nxl, kSlotP0), n, ty, s.right, c->comm, c->stream));
            if (s.left >= 0) CKN(g_nccl.Recv(scratch_l, n, ty, s.left, c->comm, c->stream));
        }
        CKN(g_nccl.GroupEnd());
        if (!forward) {
            if (s.right >= 0) CK(launch_aa_merge<T>(b + off(s, nxl - 1, 0), scratch_r, s.g, 0, c->stream));
            if (s.left >= 0) CK(launch_aa_merge<T>(b + off(s, 0, kSlotP0), scratch_l, s.g, kSlotP0, c->stream));
        }
        return LBM_OK;
    }
    for (Slab& s : c->slabs) {
        const size_t bytes = size_t(5 * s.plan.plane_q) * es;
        T* mine = static_cast<T*>(s.buf[0]);
        if (s.left >= 0) {
            Slab& L = c->slabs[s.left];
            T* theirs = static_cast<T*>(L.buf[0]);
            if (forward)
                CK(cudaMemcpyAsync(mine + off(s, -1, 0), theirs + off(L, L.g.nxl - 1, 0), bytes,
                                   cudaMemcpyDeviceToDevice, c->stream));
            else
                CK(launch_aa_merge<T>(theirs + off(L, L.g.nxl - 1, 0), mine + off(s, -1, 0), s.g, 0, c->stream));
        }
        if (s.right >= 0) {
            Slab& R = c->slabs[s.right];
            T* theirs = static_cast<T*>(R.buf[0]);
            if (forward)
                CK(cudaMemcpyAsync(mine + off(s, s.g.nxl, kSlotP0), theirs + off(R, 0, kSlotP0), bytes,
                                   cudaMemcpyDeviceToDevice, c->stream));
            else
                CK(launch_aa_merge<T>(theirs + off(R, 0, kSlotP0), mine + off(s, s.g.nxl, kSlotP0), s.g, kSlotP0,
                                      c->stream));
        }
    }
    return LBM_OK;
}

lbm_status exchange_aa(lbm_ctx* c, bool forward) {
    return c->dt == LBM_F64 ? exchange_aa_t<double>(c, forward) : exchange_aa_t<float>(c, forward);
}

bool aa_has_halo(const lbm_ctx* c) {
    // a single slab wraps x in the kernel; otherwise slabs with neighbours exchange
    if (c->slabs.size() == 1 && c->opts.world == 1) return false;
    for (const Slab& s : c->slabs)
        if (s.left >= 0 || s.right >= 0) return true;
    return false;
}

// X-Y blocks (LOCAL or across NCCL ranks): some slab exchanges frame rows
bool y_neighbours(const lbm_ctx* c) {
    for (const Slab& s : c->slabs)
        if (s.down >= 0 || s.up >= 0) return true;
    return false;
}

bool has_neighbours(const lbm_ctx* c) {
    for (const Slab& s : c->slabs)
        if (s.left >= 0 || s.right >= 0 || s.down >= 0 || s.up >= 0) return true;
    return false;
}

lbm_status ensure_ghosts(lbm_ctx* c) {
    lbm_status pst = peer_wait(c);  // the neighbours' stores into this rank's ghost planes are complete
    if (pst != LBM_OK) return pst;
    if (c->aa) {  // odd phase: the gather reads the neighbours' edge slots
        if (c->aa_odd && !c->ghosts_valid && aa_has_halo(c)) {
            lbm_status st = exchange_aa(c, true);
            if (st != LBM_OK) return st;
        }
        c->ghosts_valid = true;
        return LBM_OK;
    }
    if (c->ghosts_valid || !has_neighbours(c)) {
        c->ghosts_valid = true;
        return LBM_OK;
    }
    lbm_status st = exchange(c, c->cur, c->stream);
    if (st == LBM_OK) c->ghosts_valid = true;
    return st;
}

lbm_status entry(lbm_ctx* c, bool need_init) {
    if (!c) return fail(nullptr, LBM_EINVAL, "null context");
    if (c->poisoned) return fail(c, LBM_ESTATE, "context poisoned by an earlier CUDA/NCCL error: %s", c->err.c_str());
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, LBM_ECUDA, "cudaSetDevice(%d): %s", c->device, cudaGetErrorString(e));
    if (need_init && !c->initialized)
        return fail(c, LBM_ESTATE, "state not initialised (call lbm_init_equilibrium or lbm_set_populations)");
    return LBM_OK;
}

// ------------------------------------------------------------ profiling --
lbm_status prof_begin(lbm_ctx* c, size_t& slot) {
    if (!c->profiling) return LBM_OK;
    if (c->events_used == c->events.size()) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        c->events.push_back({a, b});
        c->event_updates.push_back(0);
    }
    slot = c->events_used++;
    CK(cudaEventRecord(c->events[slot].first, c->stream));
    return LBM_OK;
}

lbm_status prof_end(lbm_ctx* c, size_t slot, long long updates) {
    if (!c->profiling) return LBM_OK;
    CK(cudaEventRecord(c->events[slot].second, c->stream));
    c->event_updates[slot] = updates;
    return LBM_OK;
}

// --------------------------------------------------------------- engine --
// Before a K2 sweep of a periodic box: rebuild the ghost frame of the state's
// own planes if a non-K2 writer left it stale; the x ghost planes then need
// a fresh exchange (they carry the neighbours' frames).
template <typename T>
lbm_status ensure_frame(lbm_ctx* c, int which) {
    if (c->frame_valid || c->slabs.empty() || c->slabs[0].g.gy == 0) return LBM_OK;
    for (Slab& s : c->slabs) {
        CK(launch_frame_fill<T>(origin<T>(s, which), s.g, c->stream));
        c->launches++;
    }
    c->frame_valid = true;
    c->ghosts_valid = false;
    return LBM_OK;
}

// single-copy AA storage: alternate the in-place even / odd steps (aa.cu)
template <typename T>
lbm_status run_steps_aa(lbm_ctx* c, long n) {
    const bool halo = aa_has_halo(c);
    for (; n > 0; --n) {
        size_t slot = 0;
        long long updates = 0;
        lbm_status st = prof_begin(c, slot);
        if (st != LBM_OK) return st;
        if (c->aa_odd && halo && !c->ghosts_valid) {
            st = exchange_aa(c, true);
            if (st != LBM_OK) return st;
        }
        for (Slab& s : c->slabs) {
            cudaError_t e = launch_aa_step<T>(origin<T>(s, 0), make_params<T>(c, s), c->aa_odd, c->stream);
            if (e != cudaSuccess) return fail(c, LBM_ECUDA, "AA step launch failed: %s", cudaGetErrorString(e));
            c->launches++;
            c->k1_launches++;
            updates += (long long)s.g.nxl * s.g.ny * s.g.nz;
        }
        if (c->aa_odd && halo) {
            st = exchange_aa(c, false);
            if (st != LBM_OK) return st;
        }
        st = prof_end(c, slot, updates);
        if (st == LBM_OK) st = record_progress(c);
        if (st != LBM_OK) return st;
        c->aa_odd = !c->aa_odd;
        c->ghosts_valid = false;
        c->t += 1;
    }
    return LBM_OK;
}

// single-copy ring storage: K2 sweeps in place (k2.cu), an odd remainder
// by the in-place K1; each shifts the state window down the ring
template <typename T>
lbm_status run_steps_sc(lbm_ctx* c, long n) {
    while (n > 0) {
        const int nsteps = n >= 2 ? 2 : 1;
        lbm_status st = nsteps == 2 ? ensure_frame<T>(c, 0) : LBM_OK;
        if (st == LBM_OK) st = ensure_ghosts(c);
        if (st != LBM_OK) return st;
        size_t slot = 0;
        st = prof_begin(c, slot);
        if (st != LBM_OK) return st;
        long long updates = 0;
        // slabs one after another on the stream (the ticket words are reused)
        for (Slab& s : c->slabs) {
            T* F = origin<T>(s, 0);
            const StepParams<T> P = make_params<T>(c, s);
            const int shift = nsteps == 2 ? c->sc_gap : kK1ScGap;
            const int out_poff = (s.g.poff - shift + s.g.pmod) % s.g.pmod;
            cudaError_t e = nsteps == 2 ? launch_k2<T>(F, F, P, 0, s.g.nxl, c->stream, out_poff, c->sc_sync)
                                        : launch_k1_sc<T>(F, P, out_poff, c->sc_sync, c->stream);
            if (e != cudaSuccess)
                return fail(c, LBM_ECUDA, "single-copy sweep launch failed: %s", cudaGetErrorString(e));
            c->launches++;
            (nsteps == 2 ? c->k2_launches : c->k1_launches)++;
            updates += (long long)nsteps * s.g.nxl * s.g.ny * s.g.nz;
            s.g.poff = out_poff;
        }
        st = prof_end(c, slot, updates);
        if (st == LBM_OK) st = record_progress(c);
        if (st != LBM_OK) return st;
        c->ghosts_valid = false;
        c->frame_valid = nsteps == 2;
        c->t += nsteps;
        n -= nsteps;
    }
    return LBM_OK;
}

// X-slab single-copy contexts: the canonical f(t0) has been written into
// every slab's ring window -> exchange its ghosts -> the inverse stream in
// place (launch_k1_sc with unstream, shifting the window like a K1 step).
template <typename T>
lbm_status sc_finish_canonical(lbm_ctx* c) {
    lbm_status st = agree_valid(c, 0, nullptr);  // NCCL: every rank's inputs passed
    if (st != LBM_OK) return st;
    c->ghosts_valid = false;
    st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    for (Slab& s : c->slabs) {
        const StepParams<T> P = make_params<T>(c, s);
        const int out_poff = (s.g.poff - kK1ScGap + s.g.pmod) % s.g.pmod;
        cudaError_t e = launch_k1_sc<T>(origin<T>(s, 0), P, out_poff, c->sc_sync, c->stream, true);
        if (e != cudaSuccess) return fail(c, LBM_ECUDA, "single-copy unstream failed: %s", cudaGetErrorString(e));
        c->launches++;
        s.g.poff = out_poff;
    }
    c->cur = 0;
    c->ghosts_valid = false;
    c->initialized = true;
    c->frame_valid = false;
    c->t = 0;
    return LBM_OK;
}

// Three-step sweeps (K3, k3.cu): floor(n/3) of them; the caller runs the
// remainder.  K3 reads no ghost plane (it wraps the plane index itself) but
// writes none either, so afterwards the ghosts are stale.
template <typename T>
lbm_status run_steps_k3(lbm_ctx* c, long& n) {
    while (n >= 3) {
        lbm_status st = ensure_frame<T>(c, c->cur);
        if (st != LBM_OK) return st;
        size_t slot = 0;
        if ((st = prof_begin(c, slot)) != LBM_OK) return st;
        Slab& s = c->slabs[0];
        cudaError_t e = launch_k3<T>(origin<T>(s, c->cur), origin<T>(s, c->cur ^ 1), make_params<T>(c, s), c->stream);
        if (e != cudaSuccess) return fail(c, LBM_ECUDA, "K3 sweep launch failed: %s", cudaGetErrorString(e));
        c->launches++;
        c->k2_launches++;
        if ((st = prof_end(c, slot, 3LL * s.g.nxl * s.g.ny * s.g.nz)) != LBM_OK) return st;
        c->cur ^= 1;
        c->ghosts_valid = false;
        c->frame_valid = true;
        c->t += 3;
        n -= 3;
    }
    return LBM_OK;
}

template <typename T>
lbm_status run_steps(lbm_ctx* c, long n) {
    if (c->aa) return run_steps_aa<T>(c, n);
    if (c->sc) return run_steps_sc<T>(c, n);
    if (c->opts.kernel == LBM_KERNEL_K3) {
        if (!k3_supported<T>(c->slabs[0].g)) return fail(c, LBM_EINVAL, "kernel K3 not supported for this slab");
        lbm_status st = run_steps_k3<T>(c, n);
        if (st != LBM_OK) return st;
    }
    // AUTO and K2: the TMA-staged two-step sweep (k2.cu) where the TMA
    // descriptor can describe the slab; AUTO falls back to K1 pairs where it
    // cannot, an explicit K2 request then fails.
    bool tma = c->opts.kernel != LBM_KERNEL_K1;
    for (const Slab& s : c->slabs) tma = tma && k2_supported<T>(s.g);
    const bool use_k2 = tma;
    if (c->opts.kernel == LBM_KERNEL_K2 && !use_k2 && n >= 2)
        return fail(c, LBM_EINVAL, "two-step kernel requested but not supported for this geometry");
    // Fused halo (k2.cu): TMA K2 sweeps store the neighbours' ghost planes
    // themselves when the neighbours' buffers are addressable here (one
    // device: LOCAL slabs, the periodic self-wrap), so after the first sweep
    // no exchange runs.  LBM_FUSED_HALO=0 turns it off (A/B runs, tests).
    // With NCCL ranks the same stores go into the neighbours' buffers as
    // mapped here (LBM_HALO_PEER, peer.cu).
    const bool fuse = tma && c->fused_halo && (c->opts.comm != LBM_COMM_NCCL || c->peer) && !y_neighbours(c);
    while (n > 0) {
        const int nsteps = (use_k2 && n >= 2) ? 2 : 1;
        const bool fused = fuse && nsteps == 2;
        // peer halo: the neighbours finished the previous phase (they no
        // longer read the buffer this sweep writes into, and their stores
        // into this rank's ghost planes are complete)
        lbm_status wst = peer_wait(c);
        if (wst != LBM_OK) return wst;
        // planes [xbeg, xbeg + nxs) (and [xbeg2, xbeg2 + nxs) in the same grid)
        auto launch = [&](Slab& s, int xbeg, int nxs, int xbeg2 = 0, int nxs2 = 0) -> cudaError_t {
            const StepParams<T> P = make_params<T>(c, s);
            const T* A = origin<T>(s, c->cur);
            T* B = origin<T>(s, c->cur ^ 1);
            T* hl = nullptr;
            T* hr = nullptr;
            if (fused && c->peer) {  // the neighbours' next-sweep buffers, mapped here
                if (s.left >= 0) hl = static_cast<T*>(c->pnb[0][c->cur ^ 1].va) + s.g.org;
                if (s.right >= 0) hr = static_cast<T*>(c->pnb[1][c->cur ^ 1].va) + s.g.org;
            } else if (fused) {
                if (s.left >= 0) hl = origin<T>(c->slabs[s.left], c->cur ^ 1);
                if (s.right >= 0) hr = origin<T>(c->slabs[s.right], c->cur ^ 1);
            }
            return nsteps == 1 ? launch_k1<T>(A, B, P, xbeg, nxs, c->stream, xbeg2, nxs2)
                               : launch_k2<T>(A, B, P, xbeg, nxs, c->stream, 0, nullptr, hl, hr, xbeg2, nxs2);
        };
        // Planes [h, nxl-h) read no ghost plane (h = the sweep's step count),
        // so with neighbours the exchange runs on the comm stream while they
        // are swept; the edge planes follow once the ghosts have landed.
        if (nsteps == 2) {
            lbm_status fst = ensure_frame<T>(c, c->cur);
            if (fst != LBM_OK) return fst;
        }
        const int h = nsteps;
        bool split = !c->ghosts_valid && has_neighbours(c) && c->overlap && !y_neighbours(c);
        for (const Slab& s : c->slabs) split = split && s.g.nxl >= 2 * h + 2;
        if (!c->ghosts_valid && has_neighbours(c) && !split) {
            lbm_status st = exchange(c, c->cur, c->stream);
            if (st != LBM_OK) return st;
        }
        if (split) {
            CK(cudaEventRecord(c->ev_ready, c->stream));
            CK(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
            lbm_status st = exchange(c, c->cur, c->comm_stream);
            if (st != LBM_OK) return st;
            CK(cudaEventRecord(c->ev_halo, c->comm_stream));
        }
        // one timed record per sweep of all of this context's slabs
        size_t slot = 0;
        long long updates = 0;
        lbm_status pst = prof_begin(c, slot);
        if (pst != LBM_OK) return pst;
        for (Slab& s : c->slabs) {
            updates += (long long)nsteps * s.g.nxl * s.g.ny * s.g.nz;
            cudaError_t e = split ? launch(s, h, s.g.nxl - 2 * h) : launch(s, 0, s.g.nxl);
            if (e != cudaSuccess) return fail(c, LBM_ECUDA, "sweep launch failed: %s", cudaGetErrorString(e));
            c->launches++;
        }
        if (split) {
            CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
            for (Slab& s : c->slabs) {
                // both h-plane edge ranges in ONE grid (a 2-plane range alone
                // is a fraction of a wave of the machine)
                cudaError_t e = launch(s, 0, h, s.g.nxl - h, h);
                if (e != cudaSuccess) return fail(c, LBM_ECUDA, "edge sweep launch failed: %s", cudaGetErrorString(e));
                c->launches += 1;
            }
        }
        pst = prof_end(c, slot, updates);
        if (pst == LBM_OK) pst = record_progress(c);
        if (pst == LBM_OK) pst = peer_signal(c);
        if (pst != LBM_OK) return pst;
        (nsteps == 2 ? c->k2_launches : c->k1_launches) += (long long)c->slabs.size();
        c->cur ^= 1;
        c->ghosts_valid = fused;
        c->frame_valid = nsteps == 2;
        c->t += nsteps;
        n -= nsteps;
    }
    return LBM_OK;
}

// validation of staged doubles on the device: flag bit 0 = non-finite, bit 1 = rho <= 0
__global__ void k_validate(const double* __restrict__ v, long long n, int positive, int* flag) {
    int bad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = v[i];
        if (!isfinite(a)) bad |= 1;
        if (positive && !(a > 0.0)) bad |= 2;
    }
    if (bad) atomicOr(flag, bad);
}

lbm_status validate_device(lbm_ctx* c, const double* v, long long n, bool positive, int* out) {
    CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    if (n > 0) {
        k_validate<<<592, 256, 0, c->stream>>>(v, n, positive ? 1 : 0, c->d_flag);
        CK(cudaGetLastError());
        c->launches++;
    }
    CK(cudaMemcpyAsync(out, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    return wait_stream(c, c->stream);
}

// f(t0) canonical in buffer `which` of every slab (own planes) -> state.
template <typename T>
lbm_status finish_init(lbm_ctx* c, int canon) {
    lbm_status vst = agree_valid(c, 0, nullptr);  // NCCL: every rank's inputs passed
    if (vst != LBM_OK) return vst;
    if (c->aa) {  // canonical f(t0) in buf[0] IS the at-rest AA state
        c->cur = 0;
        c->aa_odd = false;
        c->ghosts_valid = false;
        c->initialized = true;
        c->frame_valid = false;
        c->t = 0;
        return LBM_OK;
    }
    // the inverse stream reads the neighbours' canonical planes
    if (has_neighbours(c)) {
        lbm_status st = exchange(c, canon, c->stream);
        if (st != LBM_OK) return st;
    }
    for (Slab& s : c->slabs) {
        const StepParams<T> P = make_params<T>(c, s);
        CK(launch_k0_unstream<T>(origin<T>(s, canon), origin<T>(s, canon ^ 1), P,
                                 c->stream));
        c->launches++;
    }
    vst = peer_signal(c);
    if (vst != LBM_OK) return vst;
    c->cur = canon ^ 1;
    c->ghosts_valid = false;
    c->initialized = true;
    c->frame_valid = false;
    c->t = 0;
    return LBM_OK;
}

template <typename T>
lbm_status init_eq_aa(lbm_ctx* c, const double* rho, const double* u, bool host) {
    const long long plane = (long long)c->ny * c->nz;
    // planes per chunk: 32 B (rho + u) per cell in the staging buffer
    const int cap = int(std::max<long long>(1, (long long)(c->stage_bytes / (4 * sizeof(double))) / plane));
    double* stage = static_cast<double*>(c->stage);
    for (Slab& s : c->slabs) {
        T* F = origin<T>(s, 0);
        const long long xoff = (long long)(s.g.x0 - c->x0_proc) * plane;  // process-local cell offset
        if (!host) {
            CK(launch_k0_equilibrium<T>(rho ? rho + xoff : nullptr, u ? u + 3 * xoff : nullptr, F, s.g, c->stream));
            c->launches++;
            continue;
        }
        for (int xb = 0; xb < s.g.nxl; xb += cap) {
            const int nxc = std::min(cap, s.g.nxl - xb);
            const long long cells = (long long)nxc * plane;
            const long long hoff = xoff + (long long)xb * plane;
            const double* dr = nullptr;
            const double* du = nullptr;
            if (rho) {
                CK(cudaMemcpyAsync(stage, rho + hoff, cells * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                dr = stage;
            }
            if (u) {
                CK(cudaMemcpyAsync(stage + cells, u + 3 * hoff, 3 * cells * sizeof(double), cudaMemcpyHostToDevice,
                                   c->stream));
                du = stage + cells;
            }
            int flag = 0;
            lbm_status st;
            if (dr && (st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "rho must be finite and > 0");
            if (du && (st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "u must be finite");
            CK(launch_k0_equilibrium<T>(dr, du, F, s.g, c->stream, xb, nxc));
            c->launches++;
        }
    }
    return finish_init<T>(c, 0);
}

// Host-staged x windows of the single-copy ring's init / import: planes
// [xb, xb + nxc) need their x neighbours, so a chunk stages the planes
// xb - 1 .. xb + nxc (mod nxl) -- a contiguous run of host planes, or two
// where it wraps -- as `per_cell` doubles per cell in every one of `rows`
// row blocks of host stride `row_stride` cells.
struct ScWindow {
    int w0, wn;
};
ScWindow sc_window(const SlabGeom& g, int xb, int nxc) {
    if (g.nxl == 1 || nxc == g.nxl) return {0, g.nxl};
    if (g.bc == BC_PERIODIC) return {(xb - 1 + g.nxl) % g.nxl, std::min(nxc + 2, g.nxl)};
    const int a = std::max(0, xb - 1), b = std::min(g.nxl, xb + nxc + 1);
    return {a, b - a};
}

lbm_status sc_stage_window(lbm_ctx* c, const double* host, ScWindow w, long long plane, int per_cell, int rows,
                           long long row_stride, double* dst) {
    const SlabGeom& g = c->slabs[0].g;
    const int n1 = std::min(w.wn, g.nxl - w.w0);  // planes before the wrap
    const size_t dpitch = size_t(w.wn) * plane * per_cell * sizeof(double);
    const size_t spitch = size_t(row_stride) * per_cell * sizeof(double);
    CK(cudaMemcpy2DAsync(dst, dpitch, host + (long long)w.w0 * plane * per_cell, spitch,
                         size_t(n1) * plane * per_cell * sizeof(double), rows, cudaMemcpyHostToDevice, c->stream));
    if (n1 < w.wn)
        CK(cudaMemcpy2DAsync(dst + (long long)n1 * plane * per_cell, dpitch, host, spitch,
                             size_t(w.wn - n1) * plane * per_cell * sizeof(double), rows, cudaMemcpyHostToDevice,
                             c->stream));
    return LBM_OK;
}

lbm_status sc_init_done(lbm_ctx* c) {
    c->cur = 0;
    c->ghosts_valid = false;
    c->initialized = true;
    c->frame_valid = false;
    c->t = 0;
    return LBM_OK;
}

template <typename T>
lbm_status init_eq_sc(lbm_ctx* c, const double* rho, const double* u, bool host) {
    if (c->slabs.size() > 1 || c->opts.world > 1) {
        // X-slabs: canonical feq into each window (K0a, chunked through the
        // staging buffer for host inputs), then exchange + in-place unstream
        const long long plane = (long long)c->ny * c->nz;
        const int cap = int(std::max<long long>(1, (long long)(c->stage_bytes / (4 * sizeof(double))) / plane));
        double* stage = static_cast<double*>(c->stage);
        c->initialized = false;
        for (Slab& s : c->slabs) {
            T* F = origin<T>(s, 0);
            const long long xoff = (long long)(s.g.x0 - c->x0_proc) * plane;
            if (!host) {
                CK(launch_k0_equilibrium<T>(rho ? rho + xoff : nullptr, u ? u + 3 * xoff : nullptr, F, s.g, c->stream));
                c->launches++;
                continue;
            }
            for (int xb = 0; xb < s.g.nxl; xb += cap) {
                const int nxc = std::min(cap, s.g.nxl - xb);
                const long long cells = (long long)nxc * plane, hoff = xoff + (long long)xb * plane;
                const double* dr = nullptr;
                const double* du = nullptr;
                if (rho) {
                    CK(cudaMemcpyAsync(stage, rho + hoff, cells * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                    dr = stage;
                }
                if (u) {
                    CK(cudaMemcpyAsync(stage + cells, u + 3 * hoff, 3 * cells * sizeof(double),
                                       cudaMemcpyHostToDevice, c->stream));
                    du = stage + cells;
                }
                int flag = 0;
                lbm_status st;
                if (dr && (st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
                if (flag) return agree_valid(c, 1, "rho must be finite and > 0");
                if (du && (st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
                if (flag) return agree_valid(c, 1, "u must be finite");
                CK(launch_k0_equilibrium<T>(dr, du, F, s.g, c->stream, xb, nxc));
                c->launches++;
            }
        }
        return sc_finish_canonical<T>(c);
    }
    Slab& s = c->slabs[0];
    const StepParams<T> P = make_params<T>(c, s);
    T* F = origin<T>(s, 0);
    if (!host) {
        CK(launch_k0_init_pull<T>(rho, u, nullptr, F, P, 0, s.g.nxl, 0, s.g.nxl, c->stream));
        c->launches++;
        return sc_init_done(c);
    }
    const long long plane = (long long)c->ny * c->nz;
    // planes per chunk: 32 B (rho + u) per cell, two halo planes
    const int cap = int(std::max<long long>(1, (long long)(c->stage_bytes / (4 * sizeof(double))) / plane - 2));
    double* stage = static_cast<double*>(c->stage);
    for (int xb = 0; xb < s.g.nxl; xb += cap) {
        const int nxc = std::min(cap, s.g.nxl - xb);
        const ScWindow w = sc_window(s.g, xb, nxc);
        const long long cells = (long long)w.wn * plane;
        const double* dr = nullptr;
        const double* du = nullptr;
        lbm_status st;
        if (rho) {
            if ((st = sc_stage_window(c, rho, w, plane, 1, 1, s.g.nxl * plane, stage)) != LBM_OK) return st;
            dr = stage;
        }
        if (u) {
            if ((st = sc_stage_window(c, u, w, plane, 3, 1, s.g.nxl * plane, stage + cells)) != LBM_OK) return st;
            du = stage + cells;
        }
        int flag = 0;
        if (dr && (st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
        if (flag) return agree_valid(c, 1, "rho must be finite and > 0");
        if (du && (st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
        if (flag) return agree_valid(c, 1, "u must be finite");
        CK(launch_k0_init_pull<T>(dr, du, nullptr, F, P, xb, nxc, w.w0, w.wn, c->stream));
        c->launches++;
    }
    return sc_init_done(c);
}

template <typename T>
lbm_status set_pops_sc(lbm_ctx* c, const double* f) {
    if (c->slabs.size() > 1 || c->opts.world > 1) {
        // X-slabs: canonical f into each window (K0 import, chunked), then
        // exchange + in-place unstream
        const long long plane = (long long)c->ny * c->nz;
        const long long proc_cells = (long long)c->nxl_proc * plane;
        const int cap = int(std::max<long long>(1, (long long)(c->stage_bytes / (kQ * sizeof(double))) / plane));
        double* stage = static_cast<double*>(c->stage);
        c->initialized = false;
        for (Slab& s : c->slabs) {
            for (int xb = 0; xb < s.g.nxl; xb += cap) {
                const int nxc = std::min(cap, s.g.nxl - xb);
                const long long ccells = (long long)nxc * plane;
                const double* src = f + (long long)(s.g.x0 - c->x0_proc + xb) * plane;
                CK(cudaMemcpy2DAsync(stage, ccells * sizeof(double), src, proc_cells * sizeof(double),
                                     ccells * sizeof(double), kQ, cudaMemcpyHostToDevice, c->stream));
                int flag = 0;
                lbm_status st = validate_device(c, stage, kQ * ccells, false, &flag);
                if (st != LBM_OK) return st;
                if (flag) return agree_valid(c, 1, "populations must be finite");
                CK(launch_k0_import<T>(stage, origin<T>(s, 0), s.g, xb, nxc, c->stream));
                c->launches++;
            }
        }
        return sc_finish_canonical<T>(c);
    }
    Slab& s = c->slabs[0];
    const StepParams<T> P = make_params<T>(c, s);
    T* F = origin<T>(s, 0);
    const long long plane = (long long)c->ny * c->nz;
    const int cap =
        int(std::max<long long>(1, (long long)(c->stage_bytes / (kQ * sizeof(double))) / plane - 2));
    double* stage = static_cast<double*>(c->stage);
    c->initialized = false;
    for (int xb = 0; xb < s.g.nxl; xb += cap) {
        const int nxc = std::min(cap, s.g.nxl - xb);
        const ScWindow w = sc_window(s.g, xb, nxc);
        lbm_status st = sc_stage_window(c, f, w, plane, 1, kQ, (long long)s.g.nxl * plane, stage);
        if (st != LBM_OK) return st;
        int flag = 0;
        st = validate_device(c, stage, (long long)kQ * w.wn * plane, false, &flag);
        if (st != LBM_OK) return st;
        if (flag) return agree_valid(c, 1, "populations must be finite");
        CK(launch_k0_init_pull<T>(nullptr, nullptr, stage, F, P, xb, nxc, w.w0, w.wn, c->stream));
        c->launches++;
    }
    return sc_init_done(c);
}

// ------------------------------------------------------- X-Y blocks ----
lbm_status moments_status(lbm_ctx* c);
// Host / device arrays cover the whole domain; a block's part of one is a
// 3D sub-box: planes [x, x + nxc) of rows [y0, y0 + ny) of k doubles per
// cell.  Copy it to / from a contiguous [nxc][ny][nz * k] array.
lbm_status copy_block(lbm_ctx* c, double* dst, const double* src, bool to_block, const Slab& s, int xb, int nxc,
                      int k, cudaMemcpyKind kind) {
    cudaMemcpy3DParms m;
    memset(&m, 0, sizeof m);
    const size_t row = size_t(c->nz) * size_t(k) * sizeof(double);
    const cudaPos gpos = make_cudaPos(0, size_t(s.y0), size_t(s.g.x0 - c->x0_proc + xb));
    if (to_block) {
        m.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), row, row, size_t(c->ny));
        m.srcPos = gpos;
        m.dstPtr = make_cudaPitchedPtr(dst, row, row, size_t(s.g.ny));
    } else {
        m.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), row, row, size_t(s.g.ny));
        m.dstPtr = make_cudaPitchedPtr(dst, row, row, size_t(c->ny));
        m.dstPos = gpos;
    }
    m.extent = make_cudaExtent(row, size_t(s.g.ny), size_t(nxc));
    m.kind = kind;
    CK(cudaMemcpy3DAsync(&m, c->stream));
    return LBM_OK;
}

template <typename T>
lbm_status init_eq_blocks(lbm_ctx* c, const double* rho, const double* u, bool host) {
    const int canon = c->cur;
    const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    for (Slab& s : c->slabs) {
        const long long cells = (long long)s.g.nxl * s.g.ny * s.g.nz;
        double* stage = static_cast<double*>(s.buf[canon ^ 1]);  // >= 32 B per cell
        const double* dr = nullptr;
        const double* du = nullptr;
        lbm_status st;
        if (rho) {
            if ((st = copy_block(c, stage, rho, true, s, 0, s.g.nxl, 1, kind)) != LBM_OK) return st;
            dr = stage;
        }
        if (u) {
            if ((st = copy_block(c, stage + cells, u, true, s, 0, s.g.nxl, 3, kind)) != LBM_OK) return st;
            du = stage + cells;
        }
        if (host) {
            int flag = 0;
            if (dr && (st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "rho must be finite and > 0");
            if (du && (st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "u must be finite");
        }
        CK(launch_k0_equilibrium<T>(dr, du, origin<T>(s, canon), s.g, c->stream));
        c->launches++;
    }
    return finish_init<T>(c, canon);
}

template <typename T>
lbm_status set_pops_blocks(lbm_ctx* c, const double* f) {
    const int canon = c->cur ^ 1;
    const long long proc_cells = (long long)c->nxl_proc * c->ny * c->nz;
    c->initialized = false;
    for (Slab& s : c->slabs) {
        const long long plane = (long long)s.g.ny * s.g.nz;
        double* stage = static_cast<double*>(s.buf[canon ^ 1]);
        const long long cap = std::max<long long>(
            1, (long long)(size_t(s.plan.buffer_elems) * c->esize) / (kQ * plane * (long long)sizeof(double)));
        for (int xb = 0; xb < s.g.nxl; xb += int(cap)) {
            const int nxc = int(std::min<long long>(cap, s.g.nxl - xb));
            const long long cc = (long long)nxc * plane;
            for (int i = 0; i < kQ; ++i) {
                lbm_status st = copy_block(c, stage + i * cc, f + i * proc_cells, true, s, xb, nxc, 1,
                                           cudaMemcpyHostToDevice);
                if (st != LBM_OK) return st;
            }
            int flag = 0;
            lbm_status st = validate_device(c, stage, kQ * cc, false, &flag);
            if (st != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "populations must be finite");
            CK(launch_k0_import<T>(stage, origin<T>(s, canon), s.g, xb, nxc, c->stream));
            c->launches++;
        }
    }
    return finish_init<T>(c, canon);
}

template <typename T>
lbm_status macro_blocks(lbm_ctx* c, double* rho, double* u, bool host) {
    lbm_status st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    int* const flag = host ? c->d_flag : nullptr;
    if (flag) CK(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
    const cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    for (Slab& s : c->slabs) {
        const long long cells = (long long)s.g.nxl * s.g.ny * s.g.nz;
        double* stage = static_cast<double*>(s.buf[c->cur ^ 1]);
        CK(launch_k3_moments<T>(origin<T>(s, c->cur), make_params<T>(c, s), 0, s.g.nxl, rho ? stage : nullptr,
                                u ? stage + cells : nullptr, c->stream, flag));
        c->launches++;
        if (rho && (st = copy_block(c, rho, stage, false, s, 0, s.g.nxl, 1, kind)) != LBM_OK) return st;
        if (u && (st = copy_block(c, u, stage + cells, false, s, 0, s.g.nxl, 3, kind)) != LBM_OK) return st;
    }
    return host ? moments_status(c) : LBM_OK;
}

template <typename T>
lbm_status get_box_blocks(lbm_ctx* c, int bx, int by, int bz, int lx, int ly, int lz, double* out) {
    lbm_status st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    const long long bcells = (long long)lx * ly * lz;
    for (Slab& s : c->slabs) {
        const int sx0 = s.g.x0 - c->x0_proc;
        const int xa = std::max(bx, sx0), xb = std::min(bx + lx, sx0 + s.g.nxl);
        const int ya = std::max(by, s.y0), yb = std::min(by + ly, s.y0 + s.g.ny);
        if (xa >= xb || ya >= yb) continue;
        const int nyc = yb - ya;
        double* stage = static_cast<double*>(s.buf[c->cur ^ 1]);
        // x chunks that fit the staging buffer (the slab's idle lattice buffer)
        const long long cap = std::max<long long>(
            1, (long long)(size_t(s.plan.buffer_elems) * c->esize) / (kQ * (long long)nyc * lz * (long long)sizeof(double)));
        for (int x = xa; x < xb; x += int(cap)) {
            const int nxc = int(std::min<long long>(cap, xb - x));
            const long long cc = (long long)nxc * nyc * lz;
            CK(launch_k3_materialize<T>(origin<T>(s, c->cur), make_params<T>(c, s), x - sx0, ya - s.y0, bz, nxc, nyc,
                                        lz, stage, c->stream));
            c->launches++;
            for (int i = 0; i < kQ; ++i) {
                cudaMemcpy3DParms m;
                memset(&m, 0, sizeof m);
                const size_t row = size_t(lz) * sizeof(double);
                m.srcPtr = make_cudaPitchedPtr(stage + i * cc, row, row, size_t(nyc));
                m.dstPtr = make_cudaPitchedPtr(out + i * bcells, row, row, size_t(ly));
                m.dstPos = make_cudaPos(0, size_t(ya - by), size_t(x - bx));
                m.extent = make_cudaExtent(row, size_t(nyc), size_t(nxc));
                m.kind = cudaMemcpyDeviceToHost;
                CK(cudaMemcpy3DAsync(&m, c->stream));
            }
        }
    }
    return wait_stream(c, c->stream);
}

template <typename T>
lbm_status init_eq(lbm_ctx* c, const double* rho, const double* u, bool host) {
    // peer halo: no neighbour still writes into (or reads) these buffers
    lbm_status pst = peer_wait(c);
    if (pst != LBM_OK) return pst;
    // the state is rewritten from here on: invalid until the init completes
    // (a rejected input leaves it undefined, include/lbm.h)
    c->initialized = false;
    if (c->yblocks > 1) return init_eq_blocks<T>(c, rho, u, host);
    if (c->aa) return init_eq_aa<T>(c, rho, u, host);
    if (c->sc) return init_eq_sc<T>(c, rho, u, host);
    const long long plane = (long long)c->ny * c->nz;
    const int canon = c->cur;  // canonical f(t0) is built here, the state ends in the other buffer
    for (Slab& s : c->slabs) {
        const long long cells = (long long)s.g.nxl * plane;
        const long long xoff = (long long)(s.g.x0 - c->x0_proc) * plane;
        const double* dr = nullptr;
        const double* du = nullptr;
        if (host) {
            // stage rho, u as doubles in the slab's scratch buffer (>= 32 B per cell)
            double* stage = static_cast<double*>(s.buf[canon ^ 1]);
            if (rho) {
                CK(cudaMemcpyAsync(stage, rho + xoff, cells * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                dr = stage;
            }
            if (u) {
                CK(cudaMemcpyAsync(stage + cells, u + 3 * xoff, 3 * cells * sizeof(double), cudaMemcpyHostToDevice,
                                   c->stream));
                du = stage + cells;
            }
            int flag = 0;
            lbm_status st;
            if (dr && (st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "rho must be finite and > 0");
            if (du && (st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "u must be finite");
        } else {
            dr = rho ? rho + xoff : nullptr;
            du = u ? u + 3 * xoff : nullptr;
        }
        if (c->slabs.size() == 1 && c->opts.world == 1 && !y_neighbours(c)) {
            // one slab spanning the domain: the pull-form state in one pass
            // (k0_init_pull), the staging (host inputs) in the other buffer
            CK(launch_k0_init_pull<T>(dr, du, nullptr, origin<T>(s, canon), make_params<T>(c, s), 0,
                                      s.g.nxl, 0, s.g.nxl, c->stream));
            c->launches++;
            c->cur = canon;
            c->ghosts_valid = false;
            c->initialized = true;
            c->frame_valid = false;
            c->t = 0;
            return LBM_OK;
        }
        CK(launch_k0_equilibrium<T>(dr, du, origin<T>(s, canon), s.g, c->stream));
        c->launches++;
    }
    return finish_init<T>(c, canon);
}

template <typename T>
lbm_status set_pops(lbm_ctx* c, const double* f) {
    if (c->sc) return set_pops_sc<T>(c, f);
    lbm_status pst = peer_wait(c);  // peer halo: the neighbours are done with these buffers
    if (pst != LBM_OK) return pst;
    if (c->yblocks > 1) return set_pops_blocks<T>(c, f);
    const long long plane = (long long)c->ny * c->nz;
    const long long proc_cells = (long long)c->nxl_proc * plane;
    // import into the non-state buffer, stage in the state buffer (AA: into
    // the single buffer, staged in the staging buffer)
    const int canon = c->aa ? 0 : c->cur ^ 1;
    c->initialized = false;
    for (Slab& s : c->slabs) {
        double* stage = static_cast<double*>(c->aa ? c->stage : s.buf[canon ^ 1]);
        const size_t stage_bytes = c->aa ? c->stage_bytes : size_t(s.plan.buffer_elems) * c->esize;
        const long long cap_planes = (long long)stage_bytes / (kQ * plane * (long long)sizeof(double));
        for (int xb = 0; xb < s.g.nxl; xb += int(cap_planes)) {
            const int nxc = int(std::min<long long>(cap_planes, s.g.nxl - xb));
            const long long ccells = (long long)nxc * plane;
            const double* src = f + (long long)(s.g.x0 - c->x0_proc + xb) * plane;
            CK(cudaMemcpy2DAsync(stage, ccells * sizeof(double), src, proc_cells * sizeof(double),
                                 ccells * sizeof(double), kQ, cudaMemcpyHostToDevice, c->stream));
            int flag = 0;
            lbm_status st = validate_device(c, stage, kQ * ccells, false, &flag);
            if (st != LBM_OK) return st;
            if (flag) return agree_valid(c, 1, "populations must be finite");
            CK(launch_k0_import<T>(stage, origin<T>(s, canon), s.g, xb, nxc, c->stream));
            c->launches++;
        }
    }
    return finish_init<T>(c, canon);
}

// After a blocking read-back: the moments flags (moments_flags, d3q19.cuh)
// as a status -- an explicit error for rho == 0, never a silent division
// (SPEC.md:68), and for a diverged (non-finite) state.  The outputs are
// written either way; the context stays usable.
lbm_status moments_status(lbm_ctx* c) {
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    lbm_status st = wait_stream(c, c->stream);
    if (st != LBM_OK) return st;
    if (flag & 1) return fail(c, LBM_ENUMERIC, "degenerate moments: rho == 0 in some cell (u undefined there)");
    if (flag & 2) return fail(c, LBM_ENUMERIC, "non-finite moments: the state has diverged");
    return LBM_OK;
}

template <typename T>
lbm_status macro_aa(lbm_ctx* c, double* rho, double* u, bool host) {
    lbm_status st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    int* const flag = host ? c->d_flag : nullptr;  // the blocking read-back checks the moments
    if (flag) CK(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
    const long long plane = (long long)c->ny * c->nz;
    const int cap = int(std::max<long long>(1, (long long)(c->stage_bytes / (4 * sizeof(double))) / plane));
    double* stage = static_cast<double*>(c->stage);
    for (Slab& s : c->slabs) {
        const StepParams<T> P = make_params<T>(c, s);
        const T* F = origin<T>(s, 0);
        // AA: the phase-aware moments; single-copy ring: K3 on the window
        auto moments = [&](int xb, int nxc, double* r, double* v) {
            return c->sc ? launch_k3_moments<T>(F, P, xb, nxc, r, v, c->stream, flag)
                         : launch_aa_moments<T>(F, P, c->aa_odd, xb, nxc, r, v, c->stream, flag);
        };
        const long long xoff = (long long)(s.g.x0 - c->x0_proc) * plane;
        if (!host) {
            CK(moments(0, s.g.nxl, rho ? rho + xoff : nullptr, u ? u + 3 * xoff : nullptr));
            c->launches++;
            continue;
        }
        for (int xb = 0; xb < s.g.nxl; xb += cap) {
            const int nxc = std::min(cap, s.g.nxl - xb);
            const long long cells = (long long)nxc * plane;
            const long long hoff = xoff + (long long)xb * plane;
            CK(moments(xb, nxc, rho ? stage : nullptr, u ? stage + cells : nullptr));
            c->launches++;
            if (rho)
                CK(cudaMemcpyAsync(rho + hoff, stage, cells * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            if (u)
                CK(cudaMemcpyAsync(u + 3 * hoff, stage + cells, 3 * cells * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream));
        }
    }
    return host ? moments_status(c) : LBM_OK;
}

template <typename T>
lbm_status macro(lbm_ctx* c, double* rho, double* u, bool host) {
    if (c->aa || c->sc) return macro_aa<T>(c, rho, u, host);
    if (c->yblocks > 1) return macro_blocks<T>(c, rho, u, host);
    lbm_status st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    int* const flag = host ? c->d_flag : nullptr;  // the blocking read-back checks the moments
    if (flag) CK(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
    const long long plane = (long long)c->ny * c->nz;
    for (Slab& s : c->slabs) {
        const StepParams<T> P = make_params<T>(c, s);
        const long long cells = (long long)s.g.nxl * plane;
        const long long xoff = (long long)(s.g.x0 - c->x0_proc) * plane;
        const T* A = origin<T>(s, c->cur);
        if (host) {
            // x chunks: the moments of chunk j+1 run while chunk j crosses PCIe
            // on the copy stream (the staging buffer holds the whole slab)
            double* stage = static_cast<double*>(s.buf[c->cur ^ 1]);
            const int nch = int(std::min<size_t>(c->chunk_events.size() - 1, size_t(s.g.nxl)));
            const int per = (s.g.nxl + nch - 1) / nch;
            for (int j = 0, xb = 0; xb < s.g.nxl; ++j, xb += per) {
                const int nxc = std::min(per, s.g.nxl - xb);
                const long long o = (long long)xb * plane, cc = (long long)nxc * plane;
                CK(launch_k3_moments<T>(A, P, xb, nxc, rho ? stage + o : nullptr, u ? stage + cells + 3 * o : nullptr,
                                        c->stream, flag));
                c->launches++;
                CK(cudaEventRecord(c->chunk_events[j], c->stream));
                CK(cudaStreamWaitEvent(c->copy_stream, c->chunk_events[j], 0));
                if (rho)
                    CK(cudaMemcpyAsync(rho + xoff + o, stage + o, cc * sizeof(double), cudaMemcpyDeviceToHost,
                                       c->copy_stream));
                if (u)
                    CK(cudaMemcpyAsync(u + 3 * (xoff + o), stage + cells + 3 * o, 3 * cc * sizeof(double),
                                       cudaMemcpyDeviceToHost, c->copy_stream));
            }
            // later work on the context stream (and moments_status's sync) follows the copies
            CK(cudaEventRecord(c->chunk_events.back(), c->copy_stream));
            CK(cudaStreamWaitEvent(c->stream, c->chunk_events.back(), 0));
        } else {
            CK(launch_k3_moments<T>(A, P, 0, s.g.nxl, rho ? rho + xoff : nullptr, u ? u + 3 * xoff : nullptr,
                                    c->stream));
            c->launches++;
        }
    }
    return host ? moments_status(c) : LBM_OK;
}

// box in process-local coordinates; out f[19][lx][ly][lz]
template <typename T>
lbm_status get_box(lbm_ctx* c, int bx, int by, int bz, int lx, int ly, int lz, double* out) {
    if (c->yblocks > 1) return get_box_blocks<T>(c, bx, by, bz, lx, ly, lz, out);
    lbm_status st = ensure_ghosts(c);
    if (st != LBM_OK) return st;
    const long long bplane = (long long)ly * lz;
    const long long bcells = (long long)lx * bplane;
    for (Slab& s : c->slabs) {
        const int sx0 = s.g.x0 - c->x0_proc;  // slab start in process coordinates
        const int a = std::max(bx, sx0), b = std::min(bx + lx, sx0 + s.g.nxl);
        if (a >= b) continue;
        const StepParams<T> P = make_params<T>(c, s);
        double* stage = static_cast<double*>(c->stage ? c->stage : s.buf[c->cur ^ 1]);
        const size_t stage_bytes = c->stage ? c->stage_bytes : size_t(s.plan.buffer_elems) * c->esize;
        const long long cap_planes =
            std::max<long long>(1, (long long)stage_bytes / (kQ * bplane * (long long)sizeof(double)));
        for (int xb = a; xb < b; xb += int(cap_planes)) {
            const int nxc = int(std::min<long long>(cap_planes, b - xb));
            const long long ccells = (long long)nxc * bplane;
            if (c->aa)
                CK(launch_aa_materialize<T>(origin<T>(s, 0), P, c->aa_odd, xb - sx0, by, bz, nxc,
                                            ly, lz, stage, c->stream));
            else
                CK(launch_k3_materialize<T>(origin<T>(s, c->cur), P, xb - sx0, by, bz, nxc, ly, lz,
                                            stage, c->stream));
            c->launches++;
            CK(cudaMemcpy2DAsync(out + (long long)(xb - bx) * bplane, bcells * sizeof(double), stage,
                                 ccells * sizeof(double), ccells * sizeof(double), kQ, cudaMemcpyDeviceToHost,
                                 c->stream));
        }
    }
    return wait_stream(c, c->stream);
}

// ------------------------------------------------ D3Q15 / D3Q27 (dqq.cu) --
// Host paths of the other lattices: canonical buffers, so host arrays move
// through the idle buffer as staging (>= 60 B per cell, enough for rho + u:
// 32 B; populations go in x chunks).
template <typename T>
lbm_status dqq_init(lbm_ctx* c, const double* rho, const double* u, bool host) {
    c->initialized = false;
    const DqqGeom& g = c->dg;
    const long long cells = (long long)g.nx * g.ny * g.nz;
    T* A = static_cast<T*>(c->dbuf[c->dcur]);
    const double* dr = rho;
    const double* du = u;
    if (host) {
        double* stage = static_cast<double*>(c->dbuf[c->dcur ^ 1]);
        dr = du = nullptr;
        int flag = 0, bad = 0;
        const char* why = nullptr;
        lbm_status st;
        if (rho) {
            CK(cudaMemcpyAsync(stage, rho, cells * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            dr = stage;
            if ((st = validate_device(c, dr, cells, true, &flag)) != LBM_OK) return st;
            if (flag) bad = 1, why = "rho must be finite and > 0";
        }
        if (u && !bad) {
            CK(cudaMemcpyAsync(stage + cells, u, 3 * cells * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            du = stage + cells;
            if ((st = validate_device(c, du, 3 * cells, false, &flag)) != LBM_OK) return st;
            if (flag) bad = 1, why = "u must be finite";
        }
        // NCCL slabs: every rank learns the verdict before any exchange
        if ((st = agree_valid(c, bad, why)) != LBM_OK) return st;
    }
    CK(launch_dqq_init<T>(dr, du, A, g, c->stream));
    c->launches++;
    c->initialized = true;
    c->t = 0;
    return LBM_OK;
}

template <typename T>
lbm_status dqq_set(lbm_ctx* c, const double* f) {
    c->initialized = false;
    const DqqGeom& g = c->dg;
    const long long plane = (long long)g.ny * g.nz, cells = (long long)g.nx * plane;
    const size_t stage_bytes = (size_t(g.q) * size_t(g.pq) - size_t(c->dorg)) * c->esize;
    const int cap = int(std::max<long long>(1, (long long)(stage_bytes / (size_t(g.q) * plane * sizeof(double)))));
    double* stage = static_cast<double*>(c->dbuf[c->dcur ^ 1]);
    int bad = 0;
    for (int xb = 0; xb < g.nx; xb += cap) {
        const int nxc = std::min(cap, g.nx - xb);
        const long long cc = (long long)nxc * plane;
        CK(cudaMemcpy2DAsync(stage, cc * sizeof(double), f + (long long)xb * plane, cells * sizeof(double),
                             cc * sizeof(double), g.q, cudaMemcpyHostToDevice, c->stream));
        int flag = 0;
        lbm_status st = validate_device(c, stage, g.q * cc, false, &flag);
        if (st != LBM_OK) return st;
        bad |= flag;
        if (!bad) {
            CK(launch_dqq_import<T>(stage, static_cast<T*>(c->dbuf[c->dcur]), g, xb, nxc, c->stream));
            c->launches++;
        }
    }
    // (NCCL slabs: every rank learns the verdict)
    if (lbm_status st = agree_valid(c, bad, bad ? "populations must be finite" : nullptr); st != LBM_OK) return st;
    c->initialized = true;
    c->t = 0;
    return LBM_OK;
}

// X-slab halo of a D3Q15/27 NCCL slab after a push step (B = f(t+1)): the
// populations pushed into ghost plane x = nx (c_x = +1) belong to plane 0
// of the right neighbour, those in ghost plane x = -1 (c_x = -1) to plane
// nx - 1 of the left one -- per direction one contiguous (y, z) plane.  They
// arrive in the receiver's unused ghost slots of the same direction and a
// merge kernel copies them in, skipping the cells whose link source lies
// beyond a y / z wall (their slot holds the cell's own bounce-back)
template <typename T>
lbm_status dqq_exchange(lbm_ctx* c, T* B) {
    const DqqGeom& g = c->dg;
    const long long plane = (long long)g.ny * g.nzp;
    const ncclDataType_t ty = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
    int cv[27 * 3];
    double wv[27];
    dqq_table(g.q, cv, wv);
    T* const lo = B - plane;                    // ghost plane x = -1 of slot 0
    T* const hi = B + (long long)g.nx * plane;  // ghost plane x = nx of slot 0
    CKN(g_nccl.GroupStart());
    for (int i = 0; i < g.q; ++i) {
        const long long off = (long long)i * g.pq;
        if (cv[3 * i] == 1) {  // [send right, recv left]: pairs match when left == right (two ranks, or itself)
            if (c->dright >= 0) CKN(g_nccl.Send(hi + off, size_t(plane), ty, c->dright, c->comm, c->stream));
            if (c->dleft >= 0) CKN(g_nccl.Recv(lo + off, size_t(plane), ty, c->dleft, c->comm, c->stream));
        } else if (cv[3 * i] == -1) {
            if (c->dleft >= 0) CKN(g_nccl.Send(lo + off, size_t(plane), ty, c->dleft, c->comm, c->stream));
            if (c->dright >= 0) CKN(g_nccl.Recv(hi + off, size_t(plane), ty, c->dright, c->comm, c->stream));
        }
    }
    CKN(g_nccl.GroupEnd());
    CK(launch_dqq_merge<T>(B, g, c->stream));
    c->launches++;
    return record_progress(c);
}

template <typename T>
lbm_status dqq_step(lbm_ctx* c, long n) {
    const T omega = T(1.0 / c->tau);
    // pairs of steps as two-step sweeps (K2Q) unless kernel K1 was chosen
    // (measured faster than the one-step kernel for every lattice and dtype,
    // DESIGN.md section 11); an odd remainder (or, under AUTO, a driver
    // without the TMA encoder) one step at a time
    const bool open = c->dg.xlo_open || c->dg.xhi_open;
    for (bool k2 = c->opts.kernel != LBM_KERNEL_K1 && !open; k2 && n >= 2; n -= 2) {
        size_t slot = 0;
        lbm_status st = prof_begin(c, slot);
        if (st != LBM_OK) return st;
        const cudaError_t e = launch_dqq_k2<T>(static_cast<const T*>(c->dbuf[c->dcur]),
                                               static_cast<T*>(c->dbuf[c->dcur ^ 1]), c->dg, omega, c->ulid, c->stream);
        if (e == cudaErrorNotSupported && c->opts.kernel == LBM_KERNEL_AUTO) {
            cudaGetLastError();
            break;
        }
        CK(e);
        c->launches++;
        c->k2_launches++;
        if ((st = prof_end(c, slot, 2LL * c->dg.nx * c->dg.ny * c->dg.nz)) != LBM_OK) return st;
        c->dcur ^= 1;
        c->t += 2;
    }
    for (; n > 0; --n) {
        size_t slot = 0;
        lbm_status st = prof_begin(c, slot);
        if (st != LBM_OK) return st;
        CK(launch_dqq_step<T>(static_cast<const T*>(c->dbuf[c->dcur]), static_cast<T*>(c->dbuf[c->dcur ^ 1]), c->dg,
                              omega, c->ulid, c->stream));
        c->launches++;
        c->k1_launches++;
        if ((st = prof_end(c, slot, (long long)c->dg.nx * c->dg.ny * c->dg.nz)) != LBM_OK) return st;
        if (open && (st = dqq_exchange(c, static_cast<T*>(c->dbuf[c->dcur ^ 1]))) != LBM_OK) return st;
        c->dcur ^= 1;
        c->t += 1;
    }
    return LBM_OK;
}

template <typename T>
lbm_status dqq_macro(lbm_ctx* c, double* rho, double* u, bool host) {
    const DqqGeom& g = c->dg;
    const T* A = static_cast<const T*>(c->dbuf[c->dcur]);
    if (!host) {
        CK(launch_dqq_moments<T>(A, g, 0, g.nx, rho, u, nullptr, c->stream));
        c->launches++;
        return LBM_OK;
    }
    CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    const long long plane = (long long)g.ny * g.nz;
    const size_t stage_bytes = (size_t(g.q) * size_t(g.pq) - size_t(c->dorg)) * c->esize;
    const int cap = int(std::max<long long>(1, (long long)(stage_bytes / (4 * sizeof(double))) / plane));
    double* stage = static_cast<double*>(c->dbuf[c->dcur ^ 1]);
    for (int xb = 0; xb < g.nx; xb += cap) {
        const int nxc = std::min(cap, g.nx - xb);
        const long long cc = (long long)nxc * plane;
        CK(launch_dqq_moments<T>(A, g, xb, nxc, rho ? stage : nullptr, u ? stage + cc : nullptr, c->d_flag,
                                 c->stream));
        c->launches++;
        if (rho)
            CK(cudaMemcpyAsync(rho + (long long)xb * plane, stage, cc * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
        if (u)
            CK(cudaMemcpyAsync(u + 3 * (long long)xb * plane, stage + cc, 3 * cc * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
    }
    return moments_status(c);
}

template <typename T>
lbm_status dqq_box(lbm_ctx* c, int bx, int by, int bz, int lx, int ly, int lz, double* out) {
    const DqqGeom& g = c->dg;
    const long long bplane = (long long)ly * lz, bcells = (long long)lx * bplane;
    const size_t stage_bytes = (size_t(g.q) * size_t(g.pq) - size_t(c->dorg)) * c->esize;
    const int cap = int(std::max<long long>(1, (long long)(stage_bytes / (size_t(g.q) * bplane * sizeof(double)))));
    double* stage = static_cast<double*>(c->dbuf[c->dcur ^ 1]);
    for (int xb = bx; xb < bx + lx; xb += cap) {
        const int nxc = std::min(cap, bx + lx - xb);
        const long long cc = (long long)nxc * bplane;
        CK(launch_dqq_box<T>(static_cast<const T*>(c->dbuf[c->dcur]), g, xb, by, bz, nxc, ly, lz, stage, c->stream));
        c->launches++;
        CK(cudaMemcpy2DAsync(out + (long long)(xb - bx) * bplane, bcells * sizeof(double), stage,
                             cc * sizeof(double), cc * sizeof(double), g.q, cudaMemcpyDeviceToHost, c->stream));
    }
    return wait_stream(c, c->stream);
}

// LBM_HALO_PEER set-up (after the lattice buffers exist): a flag page,
// then every rank hands its buffers and flag page to its neighbours as file
// descriptors over the rendezvous socket and maps theirs (peer.cu).
lbm_status peer_setup(lbm_ctx* c) {
    std::string why;
    if (!peer::alloc(c->device, 128, &c->pflags, &why))
        return fail(c, LBM_ENOMEM, "peer-halo flag page: %s", why.c_str());
    CK(cudaMemset(c->pflags.va, 0, 128));
    c->peer_flush = peer::can_flush_remote_writes(c->device);
    const Slab& s = c->slabs[0];
    std::vector<int> mine;
    for (peer::Alloc* m : {&c->pmine[0], &c->pmine[1], &c->pflags}) {
        const int fd = peer::export_fd(*m, &why);
        if (fd < 0) {
            for (int f : mine) close(f);
            return fail(c, LBM_ENCCL, "peer-halo export: %s", why.c_str());
        }
        mine.push_back(fd);
    }
    // rendezvous key: the communicator's unique id (the same on every rank)
    unsigned long long h = 1469598103934665603ULL;
    const unsigned char* id = static_cast<const unsigned char*>(c->opts.nccl_id);
    for (int i = 0; i < 128; ++i) h = (h ^ id[i]) * 1099511628211ULL;
    char key[32];
    snprintf(key, sizeof key, "%016llx", h);
    std::vector<int> peers;
    if (s.left >= 0) peers.push_back(s.left);
    if (s.right >= 0) peers.push_back(s.right);
    std::vector<std::vector<int>> theirs;
    const bool ok = peer::exchange_fds(key, c->opts.rank, peers, mine, &theirs, c->nccl_timeout_s, &why);
    for (int f : mine) close(f);
    if (!ok) return fail(c, LBM_ENCCL, "peer-halo rendezvous: %s", why.c_str());
    size_t j = 0;
    for (int side = 0; side < 2; ++side) {
        if ((side == 0 ? s.left : s.right) < 0) continue;
        const size_t sizes[3] = {c->pmine[0].size, c->pmine[1].size, c->pflags.size};
        const size_t grans[3] = {c->pmine[0].gran, c->pmine[1].gran, c->pflags.gran};
        bool mapped = true;
        for (int m = 0; m < 3; ++m) {
            if (mapped && !peer::import_fd(c->device, theirs[j][size_t(m)], sizes[m], grans[m], &c->pnb[side][m], &why))
                mapped = false;
            close(theirs[j][size_t(m)]);
        }
        if (!mapped) return fail(c, LBM_ENCCL, "peer-halo mapping of rank %d: %s", peers[j], why.c_str());
        ++j;
    }
    return LBM_OK;
}

}  // namespace

// ================================================================ ABI ====
extern "C" {

int lbm_abi_version(void) { return LBM_ABI_VERSION; }

void lbm_default_opts(lbm_opts* o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->struct_size = sizeof(lbm_opts);
    o->bc = LBM_BC_CAVITY;
    o->device = -1;
    o->rank = 0;
    o->world = 1;
    o->comm = LBM_COMM_NONE;
    o->nccl_id = nullptr;
    o->stream = nullptr;
    o->kernel = LBM_KERNEL_AUTO;
    o->local_slabs = 1;
    o->halo = LBM_HALO_AUTO;
    o->lattice = 19;
    o->local_blocks_y = 1;
    o->ranks_y = 1;
}

lbm_status lbm_lattice_table(int q, int* c, double* w) {
    lbm_ctx* ctx = nullptr;
    if (!c || !w) return fail(ctx, LBM_EINVAL, "null argument");
    if (q == 19) {
        for (int i = 0; i < 19; ++i) {
            c[3 * i] = can_cx(i);
            c[3 * i + 1] = can_cy(i);
            c[3 * i + 2] = can_cz(i);
            w[i] = i == 0 ? 1.0 / 3.0 : (can_axis(i) ? 1.0 / 18.0 : 1.0 / 36.0);
        }
        return LBM_OK;
    }
    if (q != 15 && q != 27) return fail(ctx, LBM_EINVAL, "bad lattice %d (15, 19 or 27)", q);
    dqq_table(q, c, w);
    return LBM_OK;
}

const char* lbm_last_error(const lbm_ctx* c) { return c ? c->err.c_str() : t_last_error.c_str(); }

lbm_status lbm_plan_halo_xy(int nx, int ny, int nz, lbm_dtype dt, int bc, int rank, int world, int ranks_y,
                            lbm_halo_plan* plan) {
    lbm_ctx* c = nullptr;
    if (!plan) return fail(c, LBM_EINVAL, "plan is NULL");
    if (nx < 1 || ny < 1 || nz < 1) return fail(c, LBM_EINVAL, "dimensions must be >= 1");
    if (dt != LBM_F64 && dt != LBM_F32) return fail(c, LBM_EINVAL, "bad dtype");
    if (bc != LBM_BC_CAVITY && bc != LBM_BC_PERIODIC) return fail(c, LBM_EINVAL, "bad bc");
    if (world < 1 || rank < 0 || rank >= world) return fail(c, LBM_EINVAL, "rank %d / world %d", rank, world);
    if (ranks_y < 1 || world % ranks_y) return fail(c, LBM_EINVAL, "world %% ranks_y != 0");
    if (nx % (world / ranks_y)) return fail(c, LBM_EINVAL, "nx %% (world / ranks_y) != 0");
    if (ny % ranks_y) return fail(c, LBM_EINVAL, "ny %% ranks_y != 0");
    fill_plan_xy(nx, ny, nz, dt == LBM_F64 ? 8 : 4, bc, rank, world, ranks_y, plan);
    return LBM_OK;
}

lbm_status lbm_plan_halo(int nx, int ny, int nz, lbm_dtype dt, int bc, int rank, int world, lbm_halo_plan* plan) {
    lbm_ctx* c = nullptr;
    if (!plan) return fail(c, LBM_EINVAL, "plan is NULL");
    if (nx < 1 || ny < 1 || nz < 1) return fail(c, LBM_EINVAL, "dimensions must be >= 1");
    if (dt != LBM_F64 && dt != LBM_F32) return fail(c, LBM_EINVAL, "bad dtype");
    if (bc != LBM_BC_CAVITY && bc != LBM_BC_PERIODIC) return fail(c, LBM_EINVAL, "bad bc");
    if (world < 1 || rank < 0 || rank >= world) return fail(c, LBM_EINVAL, "rank %d / world %d", rank, world);
    if (nx % world) return fail(c, LBM_EINVAL, "nx %% world != 0");
    const int nxl = nx / world;
    fill_plan(nx, ny, nz, dt == LBM_F64 ? 8 : 4, bc, rank, world, nxl, rank * nxl, plan);
    return LBM_OK;
}

lbm_status lbm_create(lbm_ctx** out, int nx, int ny, int nz, double tau, const double u_lid[3], lbm_dtype dt) {
    return lbm_create_ex(out, nx, ny, nz, tau, u_lid, dt, nullptr);
}

lbm_status lbm_create_ex(lbm_ctx** out, int nx, int ny, int nz, double tau, const double u_lid[3], lbm_dtype dt,
                         const lbm_opts* user_opts) {
    DeviceGuard dg;
    lbm_ctx* c = nullptr;
    if (!out) return fail(c, LBM_EINVAL, "out is NULL");
    *out = nullptr;
    lbm_opts o;
    lbm_default_opts(&o);
    if (user_opts) {
        if (user_opts->struct_size < int(sizeof(lbm_opts)))
            return fail(c, LBM_EINVAL, "opts.struct_size %d < %zu", user_opts->struct_size, sizeof(lbm_opts));
        o = *user_opts;
    }
    // ---- validation before any allocation ----
    if (nx < 1 || ny < 1 || nz < 1) return fail(c, LBM_EINVAL, "dimensions must be >= 1 (got %d %d %d)", nx, ny, nz);
    if ((long long)nx * ny * nz > (1LL << 40)) return fail(c, LBM_EINVAL, "domain too large");
    if (!(tau > 0.5) || !std::isfinite(tau)) return fail(c, LBM_EINVAL, "tau must be finite and > 0.5 (got %g)", tau);
    if (dt != LBM_F64 && dt != LBM_F32) return fail(c, LBM_EINVAL, "bad dtype %d", int(dt));
    if (o.bc != LBM_BC_CAVITY && o.bc != LBM_BC_PERIODIC) return fail(c, LBM_EINVAL, "bad bc %d", o.bc);
    if (!finite_vec(u_lid)) return fail(c, LBM_EINVAL, "u_lid must be finite");
    double ul[3] = {0, 0, 0};
    if (u_lid && o.bc == LBM_BC_CAVITY) memcpy(ul, u_lid, sizeof ul);
    if (ul[2] != 0.0) return fail(c, LBM_EINVAL, "u_lid must be tangential to the z = nz-1 lid (u_lid[2] == 0)");
    if (std::sqrt(ul[0] * ul[0] + ul[1] * ul[1]) > 0.3) return fail(c, LBM_EINVAL, "|u_lid| > 0.3");
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world)
        return fail(c, LBM_EINVAL, "rank %d outside world %d", o.rank, o.world);
    if (o.local_slabs < 1) return fail(c, LBM_EINVAL, "local_slabs must be >= 1");
    if (o.comm == LBM_COMM_NONE && (o.world != 1 || o.local_slabs != 1))
        return fail(c, LBM_EINVAL, "comm NONE needs world == 1 and local_slabs == 1");
    if (o.comm == LBM_COMM_NCCL && (o.local_slabs != 1 || !o.nccl_id))
        return fail(c, LBM_EINVAL, "comm NCCL needs local_slabs == 1 and an nccl_id");
    if (o.comm == LBM_COMM_LOCAL && o.world != 1) return fail(c, LBM_EINVAL, "comm LOCAL needs world == 1");
    if (o.comm < LBM_COMM_NONE || o.comm > LBM_COMM_LOCAL) return fail(c, LBM_EINVAL, "bad comm %d", o.comm);
    if (o.kernel < LBM_KERNEL_AUTO || o.kernel > LBM_KERNEL_K3) return fail(c, LBM_EINVAL, "bad kernel %d", o.kernel);
    if (o.kernel == LBM_KERNEL_K3 &&
        (dt != LBM_F32 || o.bc != LBM_BC_PERIODIC || o.comm != LBM_COMM_NONE))
        return fail(c, LBM_EINVAL, "kernel K3 (three-step prototype) needs fp32, a periodic box and comm NONE");
    if (o.halo < LBM_HALO_AUTO || o.halo > LBM_HALO_PEER) return fail(c, LBM_EINVAL, "bad halo %d", o.halo);
    const int by = o.local_blocks_y < 1 ? 1 : o.local_blocks_y;
    if (by > 1) {
        if (o.comm != LBM_COMM_LOCAL)
            return fail(c, LBM_EINVAL, "local_blocks_y > 1 (X-Y blocks) needs comm LOCAL");
        if (ny % by || ny / by < 4) return fail(c, LBM_EINVAL, "X-Y blocks: ny %% local_blocks_y == 0, >= 4 rows each");
        if (o.kernel != LBM_KERNEL_AUTO && o.kernel != LBM_KERNEL_K1 && o.kernel != LBM_KERNEL_K2)
            return fail(c, LBM_EINVAL, "X-Y blocks run the two-buffer K1/K2 storage (kernel AUTO, K1 or K2)");
    }
    const int ry = o.ranks_y < 1 ? 1 : o.ranks_y;
    if (ry > 1) {
        if (o.comm != LBM_COMM_NCCL) return fail(c, LBM_EINVAL, "ranks_y > 1 (X-Y blocks across ranks) needs comm NCCL");
        if (o.world % ry) return fail(c, LBM_EINVAL, "world %d not divisible by ranks_y %d", o.world, ry);
        if (ny % ry || ny / ry < 4) return fail(c, LBM_EINVAL, "ranks_y: ny %% ranks_y == 0, >= 4 rows per block");
        if (o.kernel != LBM_KERNEL_AUTO && o.kernel != LBM_KERNEL_K1 && o.kernel != LBM_KERNEL_K2)
            return fail(c, LBM_EINVAL, "ranks_y > 1 runs the two-buffer K1/K2 storage (kernel AUTO, K1 or K2)");
        if (o.halo == LBM_HALO_PEER) return fail(c, LBM_EINVAL, "ranks_y > 1 exchanges through NCCL (halo EXCHANGE)");
    }
    const int q = o.lattice == 0 ? 19 : o.lattice;
    if (q != 15 && q != 19 && q != 27) return fail(c, LBM_EINVAL, "bad lattice %d (15, 19 or 27)", o.lattice);
    if (q != 19 && (o.comm == LBM_COMM_LOCAL || o.local_slabs > 1 || o.halo == LBM_HALO_PEER || by > 1 || ry > 1 ||
                    (o.kernel != LBM_KERNEL_AUTO && o.kernel != LBM_KERNEL_K1 && o.kernel != LBM_KERNEL_K2)))
        return fail(c, LBM_EINVAL, "lattice D3Q%d: one slab per process (comm NONE or NCCL x-slabs), kernel AUTO, K1 or K2", q);
    if (q != 19 && o.comm == LBM_COMM_NCCL && o.kernel == LBM_KERNEL_K2)
        return fail(c, LBM_EINVAL, "lattice D3Q%d over NCCL x-slabs runs the one-step kernel (kernel AUTO or K1)", q);
    if (o.halo == LBM_HALO_PEER && o.comm != LBM_COMM_NCCL)
        return fail(c, LBM_EINVAL, "halo PEER needs comm NCCL (world 1: the periodic self-wrap)");
    if (o.halo == LBM_HALO_PEER && o.kernel != LBM_KERNEL_AUTO && o.kernel != LBM_KERNEL_K2)
        return fail(c, LBM_EINVAL, "halo PEER needs the two-buffer K2 storage (kernel AUTO or K2)");
    if (o.kernel == LBM_KERNEL_K2_REG)
        return fail(c, LBM_EINVAL, "kernel K2_REG was removed (slower than K2 wherever K2 applies; DESIGN.md section 5)");
    if (o.kernel == LBM_KERNEL_AA && o.bc == LBM_BC_CAVITY && (o.world > 1 || o.local_slabs > 1) &&
        nx / (o.world * o.local_slabs) < 2)
        return fail(c, LBM_EINVAL, "kernel AA with X-slabs needs >= 2 planes per slab");
    const int nslab_total = (o.world / ry) * o.local_slabs;  // x slabs in the whole domain
    if (nx % nslab_total) return fail(c, LBM_EINVAL, "nx %d not divisible by %d slabs", nx, nslab_total);
    const int nxl = nx / nslab_total;
    if (nslab_total > 1 && nxl < 4) return fail(c, LBM_EINVAL, "slabs need >= 4 planes (got %d)", nxl);
    if (o.bc == LBM_BC_PERIODIC && nxl < 2) return fail(c, LBM_EINVAL, "periodic slabs need >= 2 planes");

    c = new lbm_ctx();
    c->nx = nx;
    c->ny = ny / ry;  // host arrays of an X-Y rank cover its block
    c->nz = nz;
    c->ranks_y = ry;
    c->tau = tau;
    memcpy(c->ulid, ul, sizeof ul);
    c->dt = dt;
    c->opts = o;
    c->esize = dt == LBM_F64 ? 8 : 4;
    if (o.device >= 0) {
        c->device = o.device;
    } else if (cudaGetDevice(&c->device) != cudaSuccess) {
        lbm_status st = fail(c, LBM_ECUDA, "no CUDA device");
        t_last_error = c->err;
        delete c;
        return st;
    }
    auto bail = [&](lbm_status st) {
        t_last_error = c->err;
        lbm_destroy(c);
        return st;
    };
    if (cudaSetDevice(c->device) != cudaSuccess) return bail(fail(c, LBM_ECUDA, "cudaSetDevice(%d)", c->device));
    c->nxl_proc = nx / (o.world / ry);
    c->x0_proc = (o.rank / ry) * c->nxl_proc;
    const int sw = o.local_slabs;
    c->yblocks = by;
    c->slabs.resize(size_t(sw) * by);  // slab j = (x range j / by, y block j % by)
    // scratch word(s): validation flags, NCCL agreement (8 bytes)
    if (cudaMalloc(&c->d_flag, 16) != cudaSuccess) return bail(fail(c, LBM_ENOMEM, "cudaMalloc flag"));
    if (o.stream) {
        c->stream = static_cast<cudaStream_t>(o.stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(c, LBM_ECUDA, "cudaStreamCreate"));
        c->own_stream = true;
    }
    {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
            cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(c, LBM_ECUDA, "comm stream / events"));
        // Overlap the exchange with the interior sweep where the exchange
        // crosses NVLink (NCCL).  On one device (LOCAL slabs, the periodic
        // wrap) the copies are cheaper than the extra edge launches the split
        // costs (measured 8 LOCAL slabs: 31.7k MLUPS serial vs 29.9k split),
        // so there it is off.  LBM_OVERLAP=0/1 forces it (A/B runs, tests).
        const char* e = getenv("LBM_OVERLAP");
        c->overlap = e ? e[0] == '1' : o.comm == LBM_COMM_NCCL;
        // (X-Y blocks exchange their frame rows before the x spans: no split
        // sweep, see run_steps)
        const char* f = getenv("LBM_FUSED_HALO");
        c->fused_halo = !(f && f[0] == '0');
        if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(c, LBM_ECUDA, "copy stream"));
        c->chunk_events.resize(9);  // 8 x chunks + the copy stream's completion
        for (cudaEvent_t& ev : c->chunk_events)
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                return bail(fail(c, LBM_ECUDA, "read-back events"));
    }
    if (o.comm == LBM_COMM_NCCL) {
        if (!nccl_load()) return bail(fail(c, LBM_ENCCL, "cannot load libnccl.so.2"));
        ncclUniqueId id;
        memcpy(&id, o.nccl_id, sizeof id);
        ncclResult_t r = g_nccl.CommInitRank(&c->comm, o.world, id, o.rank);
        if (r != ncclSuccess)
            return bail(fail(c, LBM_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
        if (const char* e = getenv("LBM_NCCL_TIMEOUT_S")) c->nccl_timeout_s = std::max(1.0, atof(e));
        c->progress.resize(64);
        for (cudaEvent_t& ev : c->progress)
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
                return bail(fail(c, LBM_ECUDA, "progress events"));
    }
    if (q != 19) {  // D3Q15 / D3Q27: two canonical buffers, nothing else
        c->q = q;
        c->dg.q = q;
        c->dg.nx = nxl;
        c->dg.ny = ny;
        c->dg.nz = nz;
        c->dg.nzp = round_up(nz, int(32 / c->esize));
        c->dg.bc = o.bc;
        // NCCL x-slabs: one ghost plane per side per
        // direction takes the pushes that leave the slab through a face shared
        // with a neighbour rank (periodic: every face, world 1 included -- the
        // wrap then travels through NCCL to this rank itself)
        const bool nccl = o.comm == LBM_COMM_NCCL;
        const bool per = o.bc == LBM_BC_PERIODIC;
        c->dleft = nccl ? (per ? (o.rank - 1 + o.world) % o.world : (o.rank > 0 ? o.rank - 1 : -1)) : -1;
        c->dright = nccl ? (per ? (o.rank + 1) % o.world : (o.rank < o.world - 1 ? o.rank + 1 : -1)) : -1;
        c->dg.xlo_open = c->dleft >= 0;
        c->dg.xhi_open = c->dright >= 0;
        const int gh = nccl ? 1 : 0;
        c->dg.pq = (long long)(nxl + 2 * gh) * ny * c->dg.nzp;
        c->dorg = gh * (long long)ny * c->dg.nzp;
        const size_t bytes = size_t(q) * size_t(c->dg.pq) * c->esize;
        for (int b = 0; b < 2; ++b) {
            if (cudaMalloc(&c->dbase[b], bytes) != cudaSuccess) {
                cudaGetLastError();
                return bail(fail(c, LBM_ENOMEM, "cudaMalloc(%zu bytes)", bytes));
            }
            if (cudaMemset(c->dbase[b], 0, bytes) != cudaSuccess) return bail(fail(c, LBM_ECUDA, "cudaMemset"));
            c->dbuf[b] = static_cast<char*>(c->dbase[b]) + c->dorg * (long long)c->esize;
        }
        if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(c, LBM_ECUDA, "create sync"));
        *out = c;
        return LBM_OK;
    }
    // AUTO: two lattice copies (K2) unless they do not fit the device's free
    // memory while the single-copy ring does -- then K2_SC (the paper's point
    // of one copy: larger domains per device).  LBM_MEM_LIMIT_BYTES caps the
    // free memory considered (tests).
    bool use_sc = o.kernel == LBM_KERNEL_K2_SC;
    c->peer = o.halo == LBM_HALO_PEER;
    if (o.kernel == LBM_KERNEL_AUTO && !c->peer && by == 1 && ry == 1) {
        size_t freeb = 0, totalb = 0;
        if (cudaMemGetInfo(&freeb, &totalb) != cudaSuccess) {
            cudaGetLastError();
            freeb = size_t(-1);
        }
        if (const char* e = getenv("LBM_MEM_LIMIT_BYTES")) freeb = std::min(freeb, size_t(atoll(e)));
        if (c->comm) {
            // every rank must pick the same storage (the halo parts differ):
            // decide on the smallest free memory of all ranks
            unsigned long long fb = freeb;
            if (cudaMemcpyAsync(c->d_flag, &fb, sizeof fb, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
                g_nccl.AllReduce(c->d_flag, c->d_flag, 1, ncclUint64, ncclMin, c->comm, c->stream) != ncclSuccess ||
                cudaMemcpyAsync(&fb, c->d_flag, sizeof fb, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                wait_stream(c, c->stream) != LBM_OK)
                return bail(fail(c, LBM_ENCCL, "agreeing on the storage across ranks failed"));
            freeb = size_t(fb);
        }
        const size_t es_ = dt == LBM_F64 ? 8 : 4;
        lbm_halo_plan tp;
        fill_plan(nx, ny, nz, es_, o.bc, 0, nslab_total, nxl, 0, &tp);
        const size_t plane_x = size_t(tp.plane_x) * es_;
        const size_t gap = size_t(dt == LBM_F64 ? k2_sc_gap<double>(nxl) : k2_sc_gap<float>(nxl));
        const size_t two = size_t(sw) * 2 * (size_t(nxl) + 4) * plane_x;
        const size_t lattice = (size_t(nxl) + 4) * plane_x;
        const size_t stage =
            std::max({size_t(3) * kQ * ny * nz * sizeof(double), size_t(64) << 20, lattice / 16});
        const size_t one = size_t(sw) * (size_t(nxl) + 4 + gap) * plane_x + stage;
        const size_t margin = size_t(256) << 20;
        if (two + margin > freeb && one + margin <= freeb) use_sc = true;
    }
    const int nyl = ny / by / ry;
    // test knob (tests only): a periodic one-rank NCCL context exchanges its
    // y frame rows with itself through NCCL instead of wrapping y in the
    // kernels -- the X-Y transport on one GPU
    const bool yself = o.comm == LBM_COMM_NCCL && o.world == 1 && o.bc == LBM_BC_PERIODIC && getenv("LBM_TEST_YSELF") &&
                       getenv("LBM_TEST_YSELF")[0] == '1';
    for (int j = 0; j < sw * by; ++j) {
        Slab& s = c->slabs[j];
        const int bxi = j / by, byi = j % by;
        const int grank = (o.rank / ry) * sw + bxi;  // global x-slab index
        fill_plan(nx, nyl, nz, c->esize, o.bc, grank, nslab_total, nxl, grank * nxl, &s.plan,
                  o.kernel == LBM_KERNEL_K3 ? 3 : 2, by > 1 || ry > 1);
        s.g.nx = nx;
        s.g.ny = nyl;
        s.y0 = byi * nyl;
        if (ry > 1 || yself) {
            // X-Y blocks across NCCL ranks: this rank's block, y-neighbours as ranks
            lbm_halo_plan xy;
            fill_plan_xy(nx, ny, nz, c->esize, o.bc, o.rank, o.world, ry, &xy);
            s.plan.down = yself ? 0 : xy.down;
            s.plan.up = yself ? 0 : xy.up;
            s.plan.y0 = xy.y0;
            s.g.ylo_wall = xy.down < 0 && o.bc == LBM_BC_CAVITY;
            s.g.yhi_wall = xy.up < 0 && o.bc == LBM_BC_CAVITY;
            s.g.ywrap = 0;
            s.down = s.plan.down;
            s.up = s.plan.up;
        }
        if (by > 1) {
            const bool per = o.bc == LBM_BC_PERIODIC;
            s.g.ylo_wall = !per && byi == 0;
            s.g.yhi_wall = !per && byi == by - 1;
            s.g.ywrap = 0;
            const int dn = per ? (byi - 1 + by) % by : byi - 1, upi = per ? (byi + 1) % by : byi + 1;
            s.down = dn >= 0 ? bxi * by + dn : -1;
            s.up = upi < by ? bxi * by + upi : -1;
        }
        s.g.nz = nz;
        s.g.nxl = nxl;
        s.g.x0 = grank * nxl;
        s.g.nzp = s.plan.nz_pitch;
        s.g.pq = s.plan.plane_q;
        s.g.gy = s.plan.y_ghost;
        s.g.zoff = s.plan.z_offset;
        s.g.org = s.plan.cell0;
        s.g.px = s.plan.plane_x;
        s.g.bc = o.bc;
        s.g.poff = 0;
        s.g.pmod = nxl + 4;
        if (use_sc) {
            c->sc = true;
            c->sc_gap = dt == LBM_F64 ? k2_sc_gap<double>(nxl) : k2_sc_gap<float>(nxl);
            s.g.pmod = nxl + 4 + c->sc_gap;
            const bool ok = dt == LBM_F64 ? k2_supported<double>(s.g) : k2_supported<float>(s.g);
            if (!ok && o.kernel == LBM_KERNEL_K2_SC)
                return bail(fail(c, LBM_EINVAL, "kernel K2_SC: the TMA descriptor cannot describe this slab"));
            if (!ok) {  // AUTO: keep two copies (the allocation may then fail: ENOMEM)
                use_sc = c->sc = false;
                s.g.pmod = nxl + 4;
            }
        }
        // cavity chain: only the outer faces of the first and last slab are walls
        s.g.left_wall = (o.bc == LBM_BC_CAVITY && grank == 0);
        s.g.right_wall = (o.bc == LBM_BC_CAVITY && grank == nslab_total - 1);
        if (o.comm == LBM_COMM_NCCL) {  // neighbour ranks (rank = x slab * ranks_y + y block)
            s.left = s.plan.left >= 0 ? s.plan.left * ry + o.rank % ry : -1;
            s.right = s.plan.right >= 0 ? s.plan.right * ry + o.rank % ry : -1;
            s.plan.left = s.left;
            s.plan.right = s.right;
        } else {
            // neighbours are local slab indices (a ring of the local slabs when
            // periodic; the same y block of the neighbouring x range)
            s.left = s.plan.left >= 0 ? (s.plan.left - o.rank * sw) * by + byi : -1;
            s.right = s.plan.right >= 0 ? (s.plan.right - o.rank * sw) * by + byi : -1;
        }
        const size_t bytes = size_t(s.g.pmod) * size_t(s.plan.plane_x) * c->esize;
        for (int b = 0; b < (c->sc || o.kernel == LBM_KERNEL_AA ? 1 : 2); ++b) {
            if (c->peer) {  // exportable VMM memory the neighbours map (peer.cu)
                std::string why;
                if (!peer::alloc(c->device, bytes, &c->pmine[b], &why))
                    return bail(fail(c, LBM_ENOMEM, "peer-halo lattice allocation (%zu bytes): %s", bytes, why.c_str()));
                s.buf[b] = c->pmine[b].va;
            } else {
                cudaError_t e = cudaMalloc(&s.buf[b], bytes);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    return bail(fail(c, LBM_ENOMEM, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e)));
                }
            }
            // ghosts of wall sides are never read; zero everything once for determinism
            if (cudaMemset(s.buf[b], 0, bytes) != cudaSuccess) return bail(fail(c, LBM_ECUDA, "cudaMemset"));
        }
    }
    if (o.comm == LBM_COMM_NCCL && (c->slabs[0].down >= 0 || c->slabs[0].up >= 0)) {
        // X-Y blocks across ranks: the four packed row-band messages
        const Slab& s0 = c->slabs[0];
        c->yband_bytes = size_t(s0.g.nxl) * kQ * size_t(s0.plan.y_band) * c->esize;
        if (cudaMalloc(&c->ypack, 4 * c->yband_bytes) != cudaSuccess)
            return bail(fail(c, LBM_ENOMEM, "cudaMalloc X-Y row bands (%zu bytes)", 4 * c->yband_bytes));
    }
    if (c->sc && cudaMalloc(&c->sc_sync, sizeof(unsigned) * (size_t(nxl) + 1)) != cudaSuccess)
        return bail(fail(c, LBM_ENOMEM, "cudaMalloc ring tickets"));
    if (o.kernel == LBM_KERNEL_AA || c->sc) {
        // host transfers are staged plane-chunk by plane-chunk: >= three planes
        // of 19 doubles (a plane and its x halo), 64 MB or 1/16 of the
        // lattice, whichever is larger
        c->aa = !c->sc;
        const size_t plane19 = size_t(kQ) * ny * nz * sizeof(double);
        const size_t lattice = size_t(c->slabs[0].plan.buffer_elems) * c->esize;
        c->stage_bytes = std::max({3 * plane19, size_t(64) << 20, lattice / 16});
        if (const char* e = getenv("LBM_STAGE_BYTES"))  // tests: force multi-chunk host transfers
            c->stage_bytes = std::max(3 * plane19, size_t(atoll(e)));
        if (cudaMalloc(&c->stage, c->stage_bytes) != cudaSuccess) {
            cudaGetLastError();
            return bail(fail(c, LBM_ENOMEM, "cudaMalloc staging (%zu bytes)", c->stage_bytes));
        }
    }
    if (c->peer) {
        lbm_status st = peer_setup(c);
        if (st != LBM_OK) return bail(st);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(c, LBM_ECUDA, "create sync"));
    *out = c;
    return LBM_OK;
}

void lbm_destroy(lbm_ctx* c) {
    if (!c) return;
    DeviceGuard dg;
    cudaSetDevice(c->device);
    // a failed wait (lost peer) aborts the communicator itself
    if (c->stream && !c->poisoned) wait_stream(c, c->stream);
    if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
    else if (c->comm && g_nccl.CommAbort) g_nccl.CommAbort(c->comm);
    for (cudaEvent_t ev : c->progress)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->events) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    if (c->peer) {
        // the neighbours may still store into these buffers: wait until they
        // completed every phase, then unmap theirs and release ours
        if (!c->poisoned && peer_wait(c) == LBM_OK) wait_stream(c, c->stream);
        for (auto& side : c->pnb)
            for (peer::Alloc& m : side) peer::release(&m);
        peer::release(&c->pflags);
        for (peer::Alloc& m : c->pmine) peer::release(&m);
        for (Slab& s : c->slabs) s.buf[0] = s.buf[1] = nullptr;
    }
    for (Slab& s : c->slabs)
        for (void* b : s.buf)
            if (b) cudaFree(b);
    for (void* b : c->dbase)
        if (b) cudaFree(b);
    if (c->d_flag) cudaFree(c->d_flag);
    if (c->sc_sync) cudaFree(c->sc_sync);
    if (c->ypack) cudaFree(c->ypack);
    if (c->stage) cudaFree(c->stage);
    if (c->comm_stream) {
        cudaStreamSynchronize(c->comm_stream);
        cudaStreamDestroy(c->comm_stream);
    }
    if (c->ev_ready) cudaEventDestroy(c->ev_ready);
    for (cudaEvent_t ev : c->chunk_events)
        if (ev) cudaEventDestroy(ev);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

lbm_status lbm_init_equilibrium(lbm_ctx* c, const double* rho, const double* u) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_init<double>(c, rho, u, true) : dqq_init<float>(c, rho, u, true);
    return c->dt == LBM_F64 ? init_eq<double>(c, rho, u, true) : init_eq<float>(c, rho, u, true);
}

lbm_status lbm_init_equilibrium_device(lbm_ctx* c, const double* rho, const double* u) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_init<double>(c, rho, u, false) : dqq_init<float>(c, rho, u, false);
    return c->dt == LBM_F64 ? init_eq<double>(c, rho, u, false) : init_eq<float>(c, rho, u, false);
}

lbm_status lbm_set_populations(lbm_ctx* c, const double* f) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    if (!f) return fail(c, LBM_EINVAL, "f is NULL");
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_set<double>(c, f) : dqq_set<float>(c, f);
    return c->dt == LBM_F64 ? set_pops<double>(c, f) : set_pops<float>(c, f);
}

lbm_status lbm_step(lbm_ctx* c, long n) {
    DeviceGuard dg;
    if (c && n < 0) return fail(c, LBM_EINVAL, "n must be >= 0 (got %ld)", n);
    lbm_status st = entry(c, true);
    if (st != LBM_OK) return st;
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_step<double>(c, n) : dqq_step<float>(c, n);
    return c->dt == LBM_F64 ? run_steps<double>(c, n) : run_steps<float>(c, n);
}

lbm_status lbm_macroscopic(lbm_ctx* c, double* rho, double* u) {
    DeviceGuard dg;
    lbm_status st = entry(c, true);
    if (st != LBM_OK) return st;
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_macro<double>(c, rho, u, true) : dqq_macro<float>(c, rho, u, true);
    return c->dt == LBM_F64 ? macro<double>(c, rho, u, true) : macro<float>(c, rho, u, true);
}

lbm_status lbm_macroscopic_device(lbm_ctx* c, double* rho, double* u) {
    DeviceGuard dg;
    lbm_status st = entry(c, true);
    if (st != LBM_OK) return st;
    if (c->q != 19) return c->dt == LBM_F64 ? dqq_macro<double>(c, rho, u, false) : dqq_macro<float>(c, rho, u, false);
    return c->dt == LBM_F64 ? macro<double>(c, rho, u, false) : macro<float>(c, rho, u, false);
}

lbm_status lbm_get_populations_box(lbm_ctx* c, int x0, int y0, int z0, int lx, int ly, int lz, double* f) {
    DeviceGuard dg;
    lbm_status st = entry(c, true);
    if (st != LBM_OK) return st;
    if (!f) return fail(c, LBM_EINVAL, "f is NULL");
    if (lx < 0 || ly < 0 || lz < 0 || x0 < 0 || y0 < 0 || z0 < 0 || x0 + lx > c->nxl_proc || y0 + ly > c->ny ||
        z0 + lz > c->nz)
        return fail(c, LBM_EINVAL, "box outside the slab");
    if (c->q != 19)
        return (long long)lx * ly * lz == 0 ? LBM_OK
               : c->dt == LBM_F64           ? dqq_box<double>(c, x0, y0, z0, lx, ly, lz, f)
                                            : dqq_box<float>(c, x0, y0, z0, lx, ly, lz, f);
    if ((long long)lx * ly * lz == 0) return ensure_ghosts(c);  // collective under NCCL: every rank exchanges
    return c->dt == LBM_F64 ? get_box<double>(c, x0, y0, z0, lx, ly, lz, f)
                            : get_box<float>(c, x0, y0, z0, lx, ly, lz, f);
}

lbm_status lbm_get_populations(lbm_ctx* c, double* f) {
    if (!c) return fail(nullptr, LBM_EINVAL, "null context");
    return lbm_get_populations_box(c, 0, 0, 0, c->nxl_proc, c->ny, c->nz, f);
}

lbm_status lbm_synchronize(lbm_ctx* c) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    return wait_stream(c, c->stream);
}

lbm_status lbm_get_time(const lbm_ctx* c, long* t) {
    if (!c || !t) return fail(nullptr, LBM_EINVAL, "null argument");
    *t = c->t;
    return LBM_OK;
}

lbm_status lbm_nccl_unique_id(void* out128) {
    lbm_ctx* c = nullptr;
    if (!out128) return fail(c, LBM_EINVAL, "out is NULL");
    if (!nccl_load()) return fail(c, LBM_ENCCL, "cannot load libnccl.so.2");
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(c, LBM_ENCCL, "ncclGetUniqueId failed");
    memcpy(out128, &id, sizeof id);
    return LBM_OK;
}

lbm_status lbm_profile_enable(lbm_ctx* c, int on) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    c->profiling = on != 0;
    return LBM_OK;
}

lbm_status lbm_profile_reset(lbm_ctx* c) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    if ((st = wait_stream(c, c->stream)) != LBM_OK) return st;
    c->events_used = 0;
    return LBM_OK;
}

lbm_status lbm_get_stats(lbm_ctx* c, lbm_stats* s) {
    DeviceGuard dg;
    lbm_status st = entry(c, false);
    if (st != LBM_OK) return st;
    if (!s) return fail(c, LBM_EINVAL, "stats is NULL");
    if ((st = wait_stream(c, c->stream)) != LBM_OK) return st;
    memset(s, 0, sizeof *s);
    s->launches = c->launches;
    s->k1_launches = c->k1_launches;
    s->k2_launches = c->k2_launches;
    for (size_t i = 0; i < c->events_used; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->events[i].first, c->events[i].second));
        s->sweep_ms += ms;
        s->sweep_updates += c->event_updates[i];
        s->sweep_launches++;
    }
    return LBM_OK;
}

}  // extern "C"

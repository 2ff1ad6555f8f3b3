// k3.cu -- K3: THREE collision-streaming steps per HBM pass, the paper's
// stated future work "merge more time steps ... on GPU" (
// SURVEY.md 8(f) row 3), built as a measured prototype next to K2.
//
// The same temporal blocking as K2 (k2.cu) one level deeper.  A CTA owns an
// output tile T (TY x TZ) and marches along x; per input plane p:
//   * TMA stages f(t) on T+2 (one box per direction, origin shifted by -c_y,
//     16-byte aligned z start; the -c_z shift is applied when reading);
//   * step 1 collides every cell of T+2 and PUSHES its post-collision
//     populations into ring R1, destination-indexed on T+1;
//   * step 2 collides plane p-2 of T+1 from R1 (complete since this
//     iteration's barrier) and pushes into ring R2, destination-indexed on T;
//   * step 3 collides plane p-4 of T from R2 and streams f*(t+2) to HBM.
// Ring depths per c_x group (-1 / 0 / +1) are K2's: 2 / 3 / 4 destination
// planes each.  Every population crosses HBM once per three steps (plus the
// halo re-reads), at the price of 1.69 + 1.33 + 1 collisions per output cell
// and update triple (K2: 1.19 + 1 per pair with its 16x32 fp32 tile): the
// instruction-count model (tools/k3_model.py) predicts
// it below K2 on this issue-bound fp32 path; this kernel measures it.
//
// Scope of the prototype: fp32 (fp64 needs twice the shared memory: no
// tile fits 227 KB), a periodic box held by one slab (no walls; the x wrap
// is applied to the TMA plane coordinate, the y/z wrap comes from the ghost
// frame, which therefore has 3 rows per side in a K3 context -- frame.cuh).  Same
// bgk_collide() as K1/K2: K3 == K1 o K1 o K1 bit for bit.
#include <cuda.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "frame.cuh"
#include "kernels.h"

namespace lbm {

namespace {

constexpr int k3_round_up(int v, int m) { return (v + m - 1) / m * m; }

template <typename T, int TY_, int TZ_>
struct K3Cfg {
    static constexpr int TY = TY_, TZ = TZ_;
    static constexpr int HY1 = TY + 4, HZ1 = TZ + 4;  // step-1 region T+2
    static constexpr int HY2 = TY + 2, HZ2 = TZ + 2;  // step-2 region T+1
    static constexpr int ZPAD = 4;                    // box z start z0 - 4 (16 B aligned in fp32; reach 3)
    static constexpr int BW = TZ + 2 * ZPAD;
    static constexpr int BOX = HY1 * BW;
    static constexpr int BOXE = k3_round_up(BOX * int(sizeof(T)), 128) / int(sizeof(T));
    static constexpr int NT = k3_round_up(HY1 * HZ1, 32);
    static constexpr int RP1 = HY2 * HZ2, RP2 = TY * TZ;  // ring plane (one direction)
    static constexpr int NM = 2, NZ = 3, NP = 4;          // ring depths per c_x group
    static constexpr int R1 = (NM * 5 + NZ * 9 + NP * 5) * RP1;
    static constexpr int R2 = (NM * 5 + NZ * 9 + NP * 5) * RP2;
    static constexpr size_t SMEM = size_t(2 * kQ * BOXE + R1 + R2) * sizeof(T) + 2 * sizeof(uint64_t);
    static constexpr uint32_t TX_BYTES = uint32_t(kQ * BOX * sizeof(T));
    static_assert(SMEM <= 227 * 1024, "K3 tile does not fit shared memory");
};

// one lane of a converged warp: single-thread TMA issue without the
// compiler's per-copy election loop (see k2.cu elect_one)
__device__ __forceinline__ bool k3_elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred px;\n\telect.sync _|px, 0xffffffff;\n\t@px mov.u32 %0, 1;\n\t}" : "+r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t k3_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void k3_mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(k3_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void k3_mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(k3_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void k3_mbar_wait(uint64_t* bar, uint32_t parity) {
    for (uint32_t spin = 0;; ++spin) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(k3_smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1u << 28)) __trap();  // a TMA that never lands: a reported kernel error, not a hang
    }
}
__device__ __forceinline__ void k3_tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                          uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(k3_smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(k3_smem_u32(bar)), "l"(pol)
        : "memory");
}

// ring slot of destination plane d (d >= -12) per c_x group
__device__ __forceinline__ int slotM(int d) { return (d + 12) & 1; }
__device__ __forceinline__ int slotZ(int d) { return (d + 12) % 3; }
__device__ __forceinline__ int slotP(int d) { return (d + 12) & 3; }

}  // namespace

template <typename T, int TY, int TZ>
__global__ void __launch_bounds__(K3Cfg<T, TY, TZ>::NT, 1)
    k3_sweep(const __grid_constant__ CUtensorMap tmA, T* __restrict__ B, StepParams<T> P, int chunk) {
    using C = K3Cfg<T, TY, TZ>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* const stage = reinterpret_cast<T*>(smem_raw);
    T* const r1M = stage + 2 * kQ * C::BOXE;
    T* const r1Z = r1M + C::NM * 5 * C::RP1;
    T* const r1P = r1Z + C::NZ * 9 * C::RP1;
    T* const r2M = r1P + C::NP * 5 * C::RP1;
    T* const r2Z = r2M + C::NM * 5 * C::RP2;
    T* const r2P = r2Z + C::NZ * 9 * C::RP2;
    uint64_t* const bar = reinterpret_cast<uint64_t*>(r2P + C::NP * 5 * C::RP2);

    const SlabGeom& g = P.g;
    const int ntz = (g.nz + TZ - 1) / TZ;
    const int y0 = (int(blockIdx.x) / ntz) * TY, z0 = (int(blockIdx.x) % ntz) * TZ;
    const int xs = int(blockIdx.y) * chunk, xe = min(xs + chunk, g.nxl);
    const int tid = threadIdx.x;
    // step-1 cell (T+2 coords), step-2 cell (T+1 coords), step-3 cell (T coords)
    const int a1 = tid / C::HZ1, b1 = tid % C::HZ1;
    const int a2 = tid / C::HZ2, b2 = tid % C::HZ2;
    const int a3 = tid / TZ, b3 = tid % TZ;
    const bool act1 = tid < C::HY1 * C::HZ1, act2 = tid < C::RP1, act3 = tid < C::RP2;
    const bool in3 = act3 && y0 + a3 < g.ny && z0 + b3 < g.nz;
    // pushes: step 1 into T+1 (dest (a1 - 1 + cy, b1 - 1 + cz)), step 2 into T
    const bool row1[3] = {a1 >= 2 && a1 <= C::HY2 + 1, a1 >= 1 && a1 <= C::HY2, a1 <= C::HY2 - 1};
    const bool col1[3] = {b1 >= 2 && b1 <= C::HZ2 + 1, b1 >= 1 && b1 <= C::HZ2, b1 <= C::HZ2 - 1};
    const bool row2[3] = {a2 >= 2 && a2 <= TY + 1, a2 >= 1 && a2 <= TY, a2 <= TY - 1};
    const bool col2[3] = {b2 >= 2 && b2 <= TZ + 1, b2 >= 1 && b2 <= TZ, b2 <= TZ - 1};
    const int toff1 = (a1 - 1) * C::HZ2 + (b1 - 1), toff2 = (a2 - 1) * TZ + (b2 - 1);
    const int soff = a1 * C::BW + b1 + C::ZPAD - 2;  // staged entry of the step-1 cell for c_z = 0
    const int st_off = (y0 + a3) * g.nzp + (z0 + b3);
    FrameMask fm;
    if (in3) fm = frame_mask(g, y0 + a3, z0 + b3);
    const bool fany = fm.any();

    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    // plane q of the periodic slab, wrapped (no ghost planes are read)
    auto wrapx = [&](int q) { return ((q % g.nxl) + g.nxl) % g.nxl + 2; };
    auto issue = [&](int p, int s) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        k3_mbar_expect(&bar[s], C::TX_BYTES);
        static_for<0, kQ>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            constexpr int i = slot_dir(k);
            k3_tma_3d(stage + (s * kQ + k) * C::BOXE, &tmA, &bar[s], z0 - C::ZPAD + g.zoff, y0 - 2 - can_cy(i) + g.gy,
                      wrapx(p - can_cx(i)) * kQ + k, pol);
        });
    };
    const int p_first = xs - 2, p_last = xe + 1;  // step-1 planes
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        k3_mbar_init(&bar[0]);
        k3_mbar_init(&bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32 && k3_elect_one()) {
        issue(p_first, 0);
        issue(p_first + 1, 1);
    }

    for (int p = p_first; p <= xe + 3; ++p) {
        const bool has1 = p <= p_last;
        const int c = p - p_first, s = c & 1;
        const int d1 = p - 2, d2 = p - 4;
        const bool has2 = d1 >= xs - 1 && d1 <= xe;
        const bool has3 = d2 >= xs && d2 < xe;
        T fs[kQ], f2[kQ], f3[kQ];
        if (has1) {
            k3_mbar_wait(&bar[s], uint32_t(c >> 1) & 1u);
            if (act1) {
                const T* const sp = stage + s * kQ * C::BOXE + soff;
                static_for<0, kQ>([&](auto kc) {
                    constexpr int k = decltype(kc)::value;
                    constexpr int i = slot_dir(k);
                    fs[i] = sp[k * C::BOXE - can_cz(i)];
                });
            }
        }
        // stage free; rings of destination planes d1 (R1) and d2 (R2) complete
        __syncthreads();
        if (tid < 32 && has1 && p + 2 <= p_last && k3_elect_one()) issue(p + 2, s);
        if (has3 && act3) {
            const int t = a3 * TZ + b3;
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (k < 5) f3[slot_dir(k)] = r2M[(slotM(d2) * 5 + k) * C::RP2 + t];
                else if constexpr (k < 14) f3[slot_dir(k)] = r2Z[(slotZ(d2) * 9 + k - 5) * C::RP2 + t];
                else f3[slot_dir(k)] = r2P[(slotP(d2) * 5 + k - 14) * C::RP2 + t];
            });
        }
        if (has2 && act2) {
            const int t = a2 * C::HZ2 + b2;
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (k < 5) f2[slot_dir(k)] = r1M[(slotM(d1) * 5 + k) * C::RP1 + t];
                else if constexpr (k < 14) f2[slot_dir(k)] = r1Z[(slotZ(d1) * 9 + k - 5) * C::RP1 + t];
                else f2[slot_dir(k)] = r1P[(slotP(d1) * 5 + k - 14) * C::RP1 + t];
            });
        }
        const bool do3 = has3 && act3, do2 = has2 && act2, do1 = has1 && act1;
        if (do3 && do2) bgk_collide2<T>(f3, f2, P.omega);
        else if (do3) bgk_collide<T>(f3, P.omega);
        else if (do2) bgk_collide<T>(f2, P.omega);
        if (do1) bgk_collide<T>(fs, P.omega);
        // step 3: f*(t+2) of plane d2 to HBM (and its ghost-frame copies)
        if (has3 && in3) {
            T* const Bd = B + (long long)(d2 + 2) * g.px;
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                __stcs(Bd + (long long)k * g.pq + st_off, f3[slot_dir(k)]);
            });
            if (fany) store_frame(g, Bd, y0 + a3, z0 + b3, fm, [](int) { return true; }, f3);
        }
        // step 2 of plane d1: push into R2 (destination plane d1 + c_x)
        if (do2) {
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr int i = slot_dir(k);
                constexpr int cy = can_cy(i), cz = can_cz(i);
                constexpr int rel = cy * TZ + cz;
                if (row2[cy + 1] && col2[cz + 1]) {
                    if constexpr (k < 5) r2M[(slotM(d1 - 1) * 5 + k) * C::RP2 + toff2 + rel] = f2[i];
                    else if constexpr (k < 14) r2Z[(slotZ(d1) * 9 + k - 5) * C::RP2 + toff2 + rel] = f2[i];
                    else r2P[(slotP(d1 + 1) * 5 + k - 14) * C::RP2 + toff2 + rel] = f2[i];
                }
            });
        }
        // step 1 of plane p: push into R1 (destination plane p + c_x)
        if (do1) {
            static_for<0, kQ>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr int i = slot_dir(k);
                constexpr int cy = can_cy(i), cz = can_cz(i);
                constexpr int rel = cy * C::HZ2 + cz;
                if (row1[cy + 1] && col1[cz + 1]) {
                    if constexpr (k < 5) r1M[(slotM(p - 1) * 5 + k) * C::RP1 + toff1 + rel] = fs[i];
                    else if constexpr (k < 14) r1Z[(slotZ(p) * 9 + k - 5) * C::RP1 + toff1 + rel] = fs[i];
                    else r1P[(slotP(p + 1) * 5 + k - 14) * C::RP1 + toff1 + rel] = fs[i];
                }
            });
        }
    }
}

// ------------------------------------------------------------------ host --
namespace {

using K3EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

K3EncodeFn k3_encode() {
    static K3EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<K3EncodeFn>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

}  // namespace

template <typename T>
bool k3_supported(const SlabGeom& g) {
    return sizeof(T) == 4 && g.bc == BC_PERIODIC && g.gy >= 3 && g.zoff >= 4 && g.nxl == g.nx && k3_encode() &&
           (long long)g.pmod * kQ < (1LL << 31);
}

template <typename T>
cudaError_t launch_k3(const T* A, T* B, const StepParams<T>& P, cudaStream_t s) {
    if constexpr (sizeof(T) != 4) {
        return cudaErrorNotSupported;
    } else {
        constexpr int TY = 8, TZ = 32;
        using C = K3Cfg<T, TY, TZ>;
        const SlabGeom& g = P.g;
        if (!k3_supported<T>(g)) return cudaErrorNotSupported;
        auto kern = k3_sweep<T, TY, TZ>;
        static std::atomic<int> attr_set[64];
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
        if (!attr_set[dev].load()) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
            if (e != cudaSuccess) return e;
            attr_set[dev].store(1);
        }
        CUtensorMap map;
        const T* const base = A - g.org;
        const cuuint64_t dims[3] = {cuuint64_t(g.nzp), cuuint64_t(g.ny + 2 * g.gy), cuuint64_t(g.pmod) * kQ};
        const cuuint64_t strides[2] = {cuuint64_t(g.nzp) * sizeof(T), cuuint64_t(g.pq) * sizeof(T)};
        const cuuint32_t box[3] = {cuuint32_t(C::BW), cuuint32_t(C::HY1), 1u};
        const cuuint32_t estr[3] = {1u, 1u, 1u};
        CUresult r = k3_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<T*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
        // x chunks: whole waves of one CTA per SM, <= 48 planes (each chunk
        // recomputes ~4.5 planes of steps 1-2); LBM_K3_CHUNK overrides (tuning)
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const long long ntiles = (long long)((g.ny + TY - 1) / TY) * ((g.nz + TZ - 1) / TZ);
        int best = 1;
        double best_cost = 1e300;
        for (int nch = 1; nch <= g.nxl; ++nch) {
            const int ch = (g.nxl + nch - 1) / nch;
            if (ch > 48 && nch < g.nxl) continue;
            const long long items = ntiles * ((g.nxl + ch - 1) / ch);
            const double cost = double((items + nsm - 1) / nsm) * (ch + 4.5);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = nch;
            }
            if (ch <= 8) break;
        }
        int chunk = (g.nxl + best - 1) / best;
        if (const char* e = getenv("LBM_K3_CHUNK")) chunk = std::max(1, std::min(atoi(e), g.nxl));
        const dim3 grid(unsigned(ntiles), unsigned((g.nxl + chunk - 1) / chunk));
        kern<<<grid, C::NT, C::SMEM, s>>>(map, B, P, chunk);
        return cudaGetLastError();
    }
}

template bool k3_supported<double>(const SlabGeom&);
template bool k3_supported<float>(const SlabGeom&);
template cudaError_t launch_k3<double>(const double*, double*, const StepParams<double>&, cudaStream_t);
template cudaError_t launch_k3<float>(const float*, float*, const StepParams<float>&, cudaStream_t);

}  // namespace lbm

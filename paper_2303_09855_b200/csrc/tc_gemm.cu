// GEMMs on the 5th-generation tensor cores (tcgen05, kind::tf32): the coarse
// quantizer's approximate distances and the 3xTF32 dataset rotation.
//
// Pipeline (one CTA per 128 x BN output tile, 128 threads): thread 0 is the
// producer and the MMA issuer.  TMA loads each 32-wide K block of the operand
// tiles (boxes of 32 fp32 x rows, SWIZZLE_128B, which lands them directly in
// the canonical K-major UMMA layout: 8-row 1024-byte atoms, 16-byte chunk
// index XOR row-in-atom; rows outside the matrix are zero-filled) into one of
// STAGES shared-memory stages and arms the stage's `full` mbarrier with the
// byte count; the MMAs of a block (K = 8 per instruction) accumulate in TMEM
// and commit to the stage's `empty` mbarrier, which frees it for the block
// STAGES ahead.  After the last block a commit on `done` releases the four
// warps to the epilogue: TMEM -> registers (tcgen05.ld, warp w owns lanes
// 32w..32w+31 = rows) -> shared memory -> global with lane = column, so
// every store writes a contiguous 128-byte row segment.
//
// Coarse quantizer (NPROD = 1): approx(q, c) = |q~|^2 + |c~|^2 - 2 q^.c^ for
// mean-centred queries q~ / centroids c~ and their TF32 roundings q^ / c^
// (cvt.rna, coarse.cu).  TF32 products are exact in fp32; accumulation is
// fp32.  The prefilter certifies the probe order with
//     |approx - d| <= 1.01 ((2^-10 + 2^-22 + gamma'_D + 4u) s^2 + 2 s Delta + Delta^2)
// with gamma'_D = D u' / (1 - D u'), u' = 2^-22 (one unit of 2^-23 per
// accumulation, doubled to cover truncating or aligned accumulation), 2^-10
// for the two operand roundings, s = |q~| + max |c~| and Delta the centring
// round-off (coarse.cu); every centroid that can reach the exact top-nprobe is
// rescored in fp64, so the probe order stays exact.
//
// Rotation: Y = X P^T (y_i = sum_j P[i][j] x_j, transform.cpp:99-117) with
// X = Xh + Xl, P = Ph + Pl split into TF32 pairs and
// Y ~= Xh Ph^T + Xh Pl^T + Xl Ph^T (the Xl Pl term, ~2^-22 relative, dropped).
// Default: tc_rotate_pair_kernel, persistent and warp-specialised on CTA pairs
// (cta_group::2, M = 256 per MMA), the TF32 split of X fused into shared
// memory, two TMEM accumulators so the epilogue (TMA stores) overlaps the next
// tile's MMAs.  Kept for A/B (ADS_TC_ROTATE): the one-CTA persistent kernel
// (tc_rotate_kernel, fused or on a pre-split X) and the tiled kernel below
// (NPROD = 3) on a pre-split X.  All of them are bit-identical: the same
// products accumulate in the same K order.
#include <cuda.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <string>

#include "engine.hpp"

namespace ads {
namespace {

constexpr int kTM = 128;  // rows per tile (MMA M)
constexpr int kTK = 32;   // fp32 per K block (one 128-byte swizzle row)
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100): start >> 4
// [0,14), LBO >> 4 [16,30) (unused by swizzled K-major: 1), SBO >> 4 [32,46)
// = 1024 B between 8-row atoms, version 1 [46,48), SWIZZLE_128B = 2 [61,64).
// K-major swizzled descriptor for a KB-fp32-wide row: 128 B (type 2), 64 B (4), 32 B (6);
// SBO = 8 rows.
template <int KB>
__device__ __forceinline__ uint64_t swz_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(KB * 4 * 8 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(KB == 32 ? 2 : KB == 16 ? 4 : 6) << 61;
    return d;
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// Instruction descriptor: D fp32, A/B TF32, both K-major, N = BN, M = 128.
template <int BN>
constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
           (static_cast<uint32_t>(kTM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes -> v[0..31] (waits for the load)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue transforms of the persistent kernels: value stored at (row, col).
struct XfId {
    __device__ __forceinline__ float operator()(int, int, float v) const { return v; }
};
struct XfCoarse {  // approx(q, c) = (|q~|^2 + |c~|^2) - 2 q^.c^ (the tiled CoarseEpi's arithmetic)
    const float* qn2;
    const float* cn2;
    int M, N;
    __device__ __forceinline__ float operator()(int r, int c, float v) const {
        return (r < M && c < N) ? (qn2[r] + cn2[c]) - 2.f * v : 0.f;
    }
};

// Epilogues: called with (row, col, accumulator) for in-range elements.
struct CoarseEpi {
    const float* qn2;
    const float* cn2;
    float* out;
    int ld;
    __device__ __forceinline__ void operator()(int r, int c, float v) const {
        out[static_cast<int64_t>(r) * ld + c] = (qn2[r] + cn2[c]) - 2.f * v;
    }
};
struct StoreEpi {
    float* out;
    int ld;
    __device__ __forceinline__ void operator()(int r, int c, float v) const {
        out[static_cast<int64_t>(r) * ld + c] = v;
    }
};

// NPROD 1: C = A0 B0^T.  NPROD 3: C = A0 B0^T + A0 B1^T + A1 B0^T.
template <int NPROD, int BN, int STAGES, class Epi>
__global__ void __launch_bounds__(kThreads) tc_gemm_kernel(const __grid_constant__ CUtensorMap tA0,
                                                           const __grid_constant__ CUtensorMap tA1,
                                                           const __grid_constant__ CUtensorMap tB0,
                                                           const __grid_constant__ CUtensorMap tB1, int M,
                                                           int N, int K, Epi epi) {
    constexpr int NA = NPROD == 3 ? 2 : 1, NB = NPROD == 3 ? 2 : 1;
    constexpr int ATILE = kTM * 128, BTILE = BN * 128;
    constexpr int STAGE = NA * ATILE + NB * BTILE;
    constexpr uint32_t IDESC = idesc_tf32<BN>();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES], done;
    __shared__ uint32_t tmem_holder;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    const int m0 = blockIdx.y * kTM, n0 = blockIdx.x * BN;
    const int nkb = (K + kTK - 1) / kTK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s]);
            mbar_init(&empty[s]);
        }
        mbar_init(&done);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA0)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB0)) : "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                     "r"(static_cast<uint32_t>(BN))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;

    if (threadIdx.x == 0) {
        auto issue = [&](int kb) {
            const int s = kb % STAGES;
            unsigned char* t = smem + s * STAGE;
            mbar_expect(&full[s], STAGE);
            tma_load(t, &tA0, &full[s], kb * kTK, m0);
            if constexpr (NA == 2) tma_load(t + ATILE, &tA1, &full[s], kb * kTK, m0);
            tma_load(t + NA * ATILE, &tB0, &full[s], kb * kTK, n0);
            if constexpr (NB == 2) tma_load(t + NA * ATILE + BTILE, &tB1, &full[s], kb * kTK, n0);
        };
        for (int kb = 0; kb < STAGES && kb < nkb; ++kb) issue(kb);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % STAGES;
            const uint32_t ph = static_cast<uint32_t>(kb / STAGES) & 1u;
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            unsigned char* t = smem + s * STAGE;
            const uint64_t a0 = sw128_desc(smem_u32(t));
            const uint64_t a1 = sw128_desc(smem_u32(t + (NA - 1) * ATILE));
            const uint64_t b0 = sw128_desc(smem_u32(t + NA * ATILE));
            const uint64_t b1 = sw128_desc(smem_u32(t + NA * ATILE + (NB - 1) * BTILE));
#pragma unroll
            for (int k = 0; k < kTK / 8; ++k) {  // K = 8 tf32 = 32 bytes per MMA
                const uint64_t dk = static_cast<uint64_t>(k * 2);
                umma_tf32(tmem, a0 + dk, b0 + dk, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
                if constexpr (NPROD == 3) {
                    umma_tf32(tmem, a0 + dk, b1 + dk, IDESC, 1u);
                    umma_tf32(tmem, a1 + dk, b0 + dk, IDESC, 1u);
                }
            }
            umma_commit(&empty[s]);
            if (kb + STAGES < nkb) {
                mbar_wait(&empty[s], ph);  // the MMAs reading this stage are done
                issue(kb + STAGES);
            }
        }
        umma_commit(&done);
    }
    mbar_wait(&done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    float* tr = reinterpret_cast<float*>(smem) + warp * (32 * 33);
    for (int cb = 0; cb < BN; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cb);
        tmem_ld32(taddr, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) tr[lane * 33 + j] = __uint_as_float(v[j]);
        __syncwarp();
        const int c = n0 + cb + static_cast<int>(lane);
        for (int r = 0; r < 32; ++r) {
            const int row = m0 + warp * 32 + r;
            if (row < M && c < N) epi(row, c, tr[r * 33 + lane]);
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(static_cast<uint32_t>(BN))
                     : "memory");
}

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(smem_u32(src))
                 : "memory");
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - __uint_as_float(h)));
    hi = __uint_as_float(h);
    lo = __uint_as_float(l);
}

// Persistent 3xTF32 rotation Y = Xh Ph^T + Xh Pl^T + Xl Ph^T, one CTA per SM
// walking 128 x BN output tiles (tile t -> rows (t / nN) * 128, columns
// (t % nN) * BN, so the CTAs in flight share X row blocks through L2).
// Warp 0 lane 0: TMA producer over a STAGES-deep ring of K blocks (KB fp32
// wide: 32 with SWIZZLE_128B, 16 with SWIZZLE_64B).  Warp 1 lane 0: the MMA
// issuer, alternating two TMEM accumulators of BN columns so a tile's
// epilogue overlaps the next tile's MMAs.  Warps 2-5: the epilogue, warp w
// reading TMEM lanes 32 (w % 4) .. + 31 (its row quadrant) 32 columns at a
// time into a 128-byte-swizzled 32 x 32 staging box that one TMA store
// writes out (double-buffered per warp; rows/columns past the matrix are
// clipped by the tensor map).
// FUSED: X arrives unsplit (tXl unused) and warps 6-9 split each staged X
// block in place into its TF32 pair (hi over x, lo beside it; the same
// cvt.rna arithmetic as split_tf32_kernel, so the result is bit-identical),
// then release the stage to the MMA issuer through `conv`.
template <int BN, int STAGES, int KB, bool FUSED, int CW = 4, int EPIB = 2, int NPROD = 3, class Xf = XfId>
__global__ void __launch_bounds__(192 + (FUSED ? 32 * CW : 0), 1) tc_rotate_kernel(const __grid_constant__ CUtensorMap tXh,
                                                           const __grid_constant__ CUtensorMap tXl,
                                                           const __grid_constant__ CUtensorMap tPh,
                                                           const __grid_constant__ CUtensorMap tPl,
                                                           const __grid_constant__ CUtensorMap tY, int M, int N,
                                                           int K, Xf xf) {
    static_assert(KB == 32 || KB == 16 || KB == 8, "K block: one 128-, 64- or 32-byte swizzle row");
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN: 32-column epilogue chunks, MMA N <= 256");
    static_assert(NPROD == 3 || (NPROD == 1 && !FUSED), "NPROD 1: one plain TF32 product (A = Xh, B = Ph)");
    constexpr int ATILE = kTM * KB * 4, BTILE = BN * KB * 4;
    // NPROD 3: [Xh | Xl | Ph | Pl]; NPROD 1: [Xh | Ph]
    constexpr int STAGE = NPROD == 3 ? 2 * ATILE + 2 * BTILE : ATILE + BTILE;
    constexpr int BOFF = NPROD == 3 ? 2 * ATILE : ATILE;
    constexpr uint32_t IDESC = idesc_tf32<BN>();
    constexpr uint32_t TCOLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    float* epi = reinterpret_cast<float*>(smem + STAGES * STAGE);  // 4 warps x 2 x (32 x 32)
    __shared__ uint64_t full[STAGES], empty[STAGES], conv[STAGES], tfull[2], tempty[2];
    __shared__ uint32_t tmem_holder;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    const int nkb = (K + KB - 1) / KB;
    const int nN = (N + BN - 1) / BN;
    const int64_t ntiles = static_cast<int64_t>((M + kTM - 1) / kTM) * nN;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s]);
            mbar_init(&empty[s]);
            mbar_init_n(&conv[s], CW);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a]);
            mbar_init_n(&tempty[a], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tXh)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tPh)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                     "r"(TCOLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // producer
            int g = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int m0 = static_cast<int>(t / nN) * kTM, n0 = static_cast<int>(t % nN) * BN;
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = static_cast<uint32_t>(g / STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char* st = smem + s * STAGE;
                    mbar_expect(&full[s], FUSED ? STAGE - ATILE : STAGE);
                    tma_load(st, &tXh, &full[s], kb * KB, m0);
                    if constexpr (NPROD == 3 && !FUSED) tma_load(st + ATILE, &tXl, &full[s], kb * KB, m0);
                    tma_load(st + BOFF, &tPh, &full[s], kb * KB, n0);
                    if constexpr (NPROD == 3) tma_load(st + BOFF + BTILE, &tPl, &full[s], kb * KB, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            int g = 0, it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const int acc = it & 1;
                mbar_wait(&tempty[acc], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = static_cast<uint32_t>(g / STAGES) & 1u;
                    mbar_wait(FUSED ? &conv[s] : &full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    unsigned char* st = smem + s * STAGE;
                    const uint32_t sa = smem_u32(st);
                    const uint64_t xh = swz_desc<KB>(sa);
                    const uint64_t xl = swz_desc<KB>(sa + ATILE);
                    const uint64_t ph_ = swz_desc<KB>(sa + BOFF);
                    const uint64_t pl = swz_desc<KB>(sa + BOFF + BTILE);
#pragma unroll
                    for (int k = 0; k < KB / 8; ++k) {
                        const uint64_t dk = static_cast<uint64_t>(k * 2);
                        umma_tf32(d, xh + dk, ph_ + dk, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
                        if constexpr (NPROD == 3) {
                            umma_tf32(d, xh + dk, pl + dk, IDESC, 1u);
                            umma_tf32(d, xl + dk, ph_ + dk, IDESC, 1u);
                        }
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else if (FUSED && warp >= 6) {  // split warps
        const int ct = threadIdx.x - 192;
        int g = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int s = g % STAGES;
                mbar_wait(&full[s], static_cast<uint32_t>(g / STAGES) & 1u);
                float4* xa = reinterpret_cast<float4*>(smem + s * STAGE);
                float4* la = reinterpret_cast<float4*>(smem + s * STAGE + ATILE);
#pragma unroll
                for (int i = ct; i < ATILE / 16; i += 32 * CW) {
                    const float4 v = xa[i];
                    float4 h, l;
                    split_tf32(v.x, h.x, l.x);
                    split_tf32(v.y, h.y, l.y);
                    split_tf32(v.z, h.z, l.z);
                    split_tf32(v.w, h.w, l.w);
                    xa[i] = h;
                    la[i] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&conv[s]);
            }
        }
    } else {  // epilogue warps 2..5
        const int q = warp & 3;
        float* mine = epi + (warp - 2) * EPIB * 1024;
        int it = 0, sb = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int m0 = static_cast<int>(t / nN) * kTM, n0 = static_cast<int>(t % nN) * BN;
            const int acc = it & 1;
            mbar_wait(&tfull[acc], static_cast<uint32_t>(it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int cb = 0; cb < BN; cb += 32) {
                uint32_t v[32];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + cb);
                tmem_ld32(taddr, v);
                float* box = mine + sb * 1024;
                if (lane == 0) {
                    if constexpr (EPIB == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                __syncwarp();
                // row = lane; 16-byte chunk c of the row lands at c ^ (row & 7) (SWIZZLE_128B)
                {  // epilogue transform (identity for the rotation)
                    const int row = m0 + q * 32 + static_cast<int>(lane);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(xf(row, n0 + cb + j, __uint_as_float(v[j])));
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int pc = c ^ static_cast<int>(lane & 7u);
                    *reinterpret_cast<uint4*>(box + lane * 32 + pc * 4) =
                        make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tma_store(&tY, box, n0 + cb, m0 + q * 32);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                if constexpr (EPIB == 2) sb ^= 1;
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
}

// CTA-pair (cta_group::2) variant of the fused rotation, M = 256 per MMA: CTA
// rank r of a cluster of two loads X rows m0 + 128 r and P rows n0 + (BN/2) r
// into its own ring (its own `full` barrier), splits its X block in place and
// arrives on the LEADER's `conv` barrier (count 2 CW); the leader's lane issues
// tcgen05.mma.cta_group::2 on its own descriptors (the pair's tensor cores take
// the same offsets in the peer) and commits `empty` / `tfull` to both CTAs;
// each CTA drains its own 128 TMEM lanes and arrives on the leader's `tempty`
// (count 8).  Each SM thus reads its 128 X rows and only half of P per K step.
// the cluster-window address of the leader's (rank 0) copy of a shared variable
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

template <int BN, int STAGES, int KB, int CW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192 + 32 * CW, 1)
    tc_rotate_pair_kernel(const __grid_constant__ CUtensorMap tX, const __grid_constant__ CUtensorMap tPh,
                          const __grid_constant__ CUtensorMap tPl, const __grid_constant__ CUtensorMap tY, int M,
                          int N, int K) {
    static_assert(KB == 16, "K block: one 64-byte swizzle row");
    static_assert(BN % 32 == 0 && BN <= 256 && (BN / 2) % 16 == 0, "BN: 32-column epilogue chunks, N/2 per CTA");
    constexpr int HB = BN / 2;
    constexpr int ATILE = kTM * KB * 4, BTILE = HB * KB * 4;
    constexpr int STAGE = 2 * ATILE + 2 * BTILE;
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                               (static_cast<uint32_t>(256 >> 4) << 24);
    constexpr uint32_t TCOLS = 2 * BN <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    float* epi = reinterpret_cast<float*>(smem + STAGES * STAGE);  // 4 warps x (32 x 32)
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], conv[STAGES], tfull[2], tempty[2];
    __shared__ uint32_t tmem_holder;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int nkb = (K + KB - 1) / KB;
    const int nN = (N + BN - 1) / BN;
    const int64_t ntiles = static_cast<int64_t>((M + 2 * kTM - 1) / (2 * kTM)) * nN;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s]);
            mbar_init(&empty[s]);
            mbar_init_n(&conv[s], 2 * CW);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a]);
            mbar_init_n(&tempty[a], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tX)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tPh)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                     "r"(TCOLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // producer (both CTAs: own X rows, own half of P)
            int g = 0;
            for (int64_t t = cid; t < ntiles; t += ncl) {
                const int m0 = static_cast<int>(t / nN) * 2 * kTM + static_cast<int>(rank) * kTM;
                const int n0 = static_cast<int>(t % nN) * BN + static_cast<int>(rank) * HB;
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = static_cast<uint32_t>(g / STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    unsigned char* st = smem + s * STAGE;
                    mbar_expect(&full[s], ATILE + 2 * BTILE);
                    tma_load(st, &tX, &full[s], kb * KB, m0);
                    tma_load(st + 2 * ATILE, &tPh, &full[s], kb * KB, n0);
                    tma_load(st + 2 * ATILE + BTILE, &tPl, &full[s], kb * KB, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {  // MMA issuer for the pair
            int g = 0, it = 0;
            for (int64_t t = cid; t < ntiles; t += ncl, ++it) {
                const int acc = it & 1;
                mbar_wait_cluster(&tempty[acc], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = g % STAGES;
                    mbar_wait_cluster(&conv[s], static_cast<uint32_t>(g / STAGES) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * STAGE);
                    const uint64_t xh = swz_desc<KB>(sa), xl = swz_desc<KB>(sa + ATILE);
                    const uint64_t ph_ = swz_desc<KB>(sa + 2 * ATILE), pl = swz_desc<KB>(sa + 2 * ATILE + BTILE);
#pragma unroll
                    for (int k = 0; k < KB / 8; ++k) {
                        const uint64_t dk = static_cast<uint64_t>(k * 2);
                        umma_tf32_pair(d, xh + dk, ph_ + dk, IDESC, (kb > 0 || k > 0) ? 1u : 0u);
                        umma_tf32_pair(d, xh + dk, pl + dk, IDESC, 1u);
                        umma_tf32_pair(d, xl + dk, ph_ + dk, IDESC, 1u);
                    }
                    umma_commit_pair(&empty[s]);
                }
                umma_commit_pair(&tfull[acc]);
            }
        }
    } else if (warp >= 6) {  // split warps: own X block, then the leader's conv barrier
        const int ct = threadIdx.x - 192;
        const uint32_t conv_leader = leader_addr(&conv[0]);
        int g = 0;
        for (int64_t t = cid; t < ntiles; t += ncl) {
            for (int kb = 0; kb < nkb; ++kb, ++g) {
                const int s = g % STAGES;
                mbar_wait(&full[s], static_cast<uint32_t>(g / STAGES) & 1u);
                float4* xa = reinterpret_cast<float4*>(smem + s * STAGE);
                float4* la = reinterpret_cast<float4*>(smem + s * STAGE + ATILE);
#pragma unroll
                for (int i = ct; i < ATILE / 16; i += 32 * CW) {
                    const float4 v = xa[i];
                    float4 h, l;
                    split_tf32(v.x, h.x, l.x);
                    split_tf32(v.y, h.y, l.y);
                    split_tf32(v.z, h.z, l.z);
                    split_tf32(v.w, h.w, l.w);
                    xa[i] = h;
                    la[i] = l;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(conv_leader + static_cast<uint32_t>(s) * 8u);
            }
        }
    } else {  // epilogue warps 2..5: own 128 rows
        const int q = warp & 3;
        float* box = epi + (warp - 2) * 1024;
        const uint32_t tempty_leader = leader_addr(&tempty[0]);
        int it = 0;
        for (int64_t t = cid; t < ntiles; t += ncl, ++it) {
            const int m0 = static_cast<int>(t / nN) * 2 * kTM + static_cast<int>(rank) * kTM;
            const int n0 = static_cast<int>(t % nN) * BN;
            const int acc = it & 1;
            mbar_wait(&tfull[acc], static_cast<uint32_t>(it >> 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int cb = 0; cb < BN; cb += 32) {
                uint32_t v[32];
                const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + cb);
                tmem_ld32(taddr, v);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int pc = c ^ static_cast<int>(lane & 7u);
                    *reinterpret_cast<uint4*>(box + lane * 32 + pc * 4) =
                        make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tma_store(&tY, box, n0 + cb, m0 + q * 32);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(acc) * 8u);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
}

__global__ void split_tf32_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float h, l;
        split_tf32(x[i], h, l);
        hi[i] = h;
        lo[i] = l;
    }
}

// ---- host: tensor maps through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ADS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// rows x width row-major fp32 (width % 4 == 0); box = 32 columns x box_rows rows, SWIZZLE_128B.
CUtensorMap tile_map(const float* base, int width, int64_t rows, int box_rows, int box_cols = kTK) {
    CUtensorMap m{};
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(width), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(width) * sizeof(float)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      box_cols == 32   ? CU_TENSOR_MAP_SWIZZLE_128B
                                      : box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                       : CU_TENSOR_MAP_SWIZZLE_32B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

template <int NPROD, int BN, int STAGES, class Epi>
void launch_tc(const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0, const CUtensorMap& b1, int M,
               int N, int K, Epi epi, cudaStream_t st) {
    constexpr int NA = NPROD == 3 ? 2 : 1, NB = NPROD == 3 ? 2 : 1;
    constexpr int smem = STAGES * (NA * kTM * 128 + NB * BN * 128) + 1024;
    auto kern = tc_gemm_kernel<NPROD, BN, STAGES, Epi>;
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid((N + BN - 1) / BN, (M + kTM - 1) / kTM);
    kern<<<grid, kThreads, smem, st>>>(a0, a1, b0, b1, M, N, K, epi);
    ADS_LAUNCH_CHECK();
}

}  // namespace

bool tc_coarse_supported(int D) { return D % 4 == 0 && D >= kTK; }

double tc_coarse_gamma(int D) {
    const double up = 0x1.0p-22;
    const double acc = static_cast<double>(D) * up / (1.0 - static_cast<double>(D) * up);
    return 0x1.0p-10 + 0x1.0p-22 + acc + 4.0 * 0x1.0p-24;
}

void launch_tc_coarse_gemm(const float* Qc, int nq, const float* Cc, int L, int D, const float* qn2,
                           const float* cn2, float* out, cudaStream_t st) {
    if (nq <= 0 || L <= 0) return;
    static const bool tiled = [] {
        const char* e = std::getenv("ADS_TC_COARSE");
        return e && e[0] == '0';
    }();
    if (!tiled && L % 4 == 0) {  // the TMA-stored output needs 16-byte row strides
        // persistent, one product, 256-column tiles of K-16 blocks; the epilogue forms
        // approx = (|q~|^2 + |c~|^2) - 2 v and leaves through TMA stores
        constexpr int BN = 256, STAGES = 6, KB = 16;
        constexpr int smem = STAGES * (kTM * KB * 4 + BN * KB * 4) + 4 * 2 * 4096 + 1024;
        const CUtensorMap a = tile_map(Qc, D, nq, kTM, KB), b = tile_map(Cc, D, L, BN, KB);
        const CUtensorMap y = tile_map(out, L, nq, 32, 32);
        auto kern = tc_rotate_kernel<BN, STAGES, KB, false, 4, 2, 1, XfCoarse>;
        ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int64_t tiles = (static_cast<int64_t>(nq + kTM - 1) / kTM) * ((L + BN - 1) / BN);
        const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
        kern<<<grid, 192, smem, st>>>(a, a, b, b, y, nq, L, D, XfCoarse{qn2, cn2, nq, L});
        ADS_LAUNCH_CHECK();
        return;
    }
    const CUtensorMap a = tile_map(Qc, D, nq, kTM);
    const CUtensorMap b = tile_map(Cc, D, L, 256);
    // short K: two stages (96 KB, two CTAs per SM overlap one's epilogue with the
    // other's MMAs); long K: four stages of prefetch (one CTA per SM)
    if (D <= 256) launch_tc<1, 256, 2>(a, a, b, b, nq, L, D, CoarseEpi{qn2, cn2, out, L}, st);
    else launch_tc<1, 256, 4>(a, a, b, b, nq, L, D, CoarseEpi{qn2, cn2, out, L}, st);
}

void launch_split_tf32(const float* x, int64_t n, float* hi, float* lo, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    split_tf32_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(x, n, hi, lo);
    ADS_LAUNCH_CHECK();
}

namespace {
template <int BN, int STAGES, int CW>
void launch_rotate_pair(const float* X, int64_t n, const float* Ph, const float* Pl, int D, float* Y, cudaStream_t st) {
    constexpr int smem = STAGES * (2 * kTM * 16 * 4 + 2 * (BN / 2) * 16 * 4) + 4 * 4096 + 1024;
    static_assert(smem <= 227 * 1024, "pair rotation kernel shared memory");
    const CUtensorMap x = tile_map(X, D, n, kTM, 16);
    const CUtensorMap ph = tile_map(Ph, D, D, BN / 2, 16), pl = tile_map(Pl, D, D, BN / 2, 16);
    const CUtensorMap y = tile_map(Y, D, n, 32, 32);
    auto kern = tc_rotate_pair_kernel<BN, STAGES, 16, CW>;
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // co-resident CTA pairs for this instantiation (thread-safe one-time init)
    static const int max_clusters = [&] {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * num_sms());
        cfg.blockDim = dim3(192 + 32 * CW);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = 2;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int c = 0;
        ADS_CUDA(cudaOccupancyMaxActiveClusters(&c, kern, &cfg));
        if (c < 1) throw CudaError("pair rotation: no co-resident CTA pair");
        return c;
    }();
    const int64_t tiles = ((n + 2 * kTM - 1) / (2 * kTM)) * ((D + BN - 1) / BN);
    const int clusters = static_cast<int>(tiles < max_clusters ? tiles : max_clusters);
    kern<<<2 * clusters, 192 + 32 * CW, smem, st>>>(x, ph, pl, y, static_cast<int>(n), D, D);
    ADS_LAUNCH_CHECK();
}

template <int BN, int STAGES, int KB, bool FUSED, int CW = 4, int EPIB = 2>
void launch_rotate(const float* Xh, const float* Xl, int64_t n, const float* Ph, const float* Pl, int D, float* Y,
                   cudaStream_t st) {
    constexpr int smem = STAGES * (2 * kTM * KB * 4 + 2 * BN * KB * 4) + 4 * EPIB * 4096 + 1024;
    static_assert(smem <= 227 * 1024, "rotation kernel shared memory");
    const CUtensorMap xh = tile_map(Xh, D, n, kTM, KB), xl = tile_map(Xl, D, n, kTM, KB);
    const CUtensorMap ph = tile_map(Ph, D, D, BN, KB), pl = tile_map(Pl, D, D, BN, KB);
    const CUtensorMap y = tile_map(Y, D, n, 32, 32);
    auto kern = tc_rotate_kernel<BN, STAGES, KB, FUSED, CW, EPIB>;
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t tiles = ((n + kTM - 1) / kTM) * ((D + BN - 1) / BN);
    const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
    kern<<<grid, 192 + (FUSED ? 32 * CW : 0), smem, st>>>(xh, xl, ph, pl, y, static_cast<int>(n), D, D, XfId{});
    ADS_LAUNCH_CHECK();
}
}  // namespace


void launch_tc_transform(const float* X, int64_t n, const float* Ph, const float* Pl, int D, float* Y, DevBuf& xh_buf,
                         DevBuf& xl_buf, cudaStream_t st) {
    if (n <= 0) return;
    if (D % 4 != 0 || D < kTK)
        throw std::invalid_argument("apply (tensor cores): dimension must be a multiple of 4 and >= 32");
    // ADS_TC_ROTATE (A/B experiments): 0 the tiled kernel on a pre-split X, 1 the
    // persistent kernel on a pre-split X, 2 persistent with the split fused,
    // 3 (default) the fused CTA-pair kernel (profiles/r01_ncu_tensorcore.md)
    static const int variant = [] {
        const char* e = std::getenv("ADS_TC_ROTATE");
        return e ? std::atoi(e) : 3;
    }();
    if (variant == 3 && n < (int64_t(1) << 31)) {
        // widest N tile that divides D; each CTA of the pair stages BN/2 rows of P;
        // the deepest K-16 ring that fits beside the epilogue box
        if (D % 256 == 0) return launch_rotate_pair<256, 6, 8>(X, n, Ph, Pl, D, Y, st);
        if (D % 192 == 0) return launch_rotate_pair<192, 7, 8>(X, n, Ph, Pl, D, Y, st);
        if (D % 128 == 0) return launch_rotate_pair<128, 8, 8>(X, n, Ph, Pl, D, Y, st);
        if (D % 96 == 0) return launch_rotate_pair<96, 9, 8>(X, n, Ph, Pl, D, Y, st);
        return launch_rotate_pair<128, 8, 8>(X, n, Ph, Pl, D, Y, st);
    }
    if (variant == 2 && n < (int64_t(1) << 31)) {
        if (D % 256 == 0) return launch_rotate<256, 4, 16, true, 8, 1>(X, X, n, Ph, Pl, D, Y, st);
        if (D % 192 == 0) return launch_rotate<192, 5, 16, true, 8, 1>(X, X, n, Ph, Pl, D, Y, st);
        if (D % 128 == 0) return launch_rotate<128, 6, 16, true, 8, 1>(X, X, n, Ph, Pl, D, Y, st);
        if (D % 96 == 0) return launch_rotate<96, 7, 16, true, 8, 1>(X, X, n, Ph, Pl, D, Y, st);
        return launch_rotate<128, 6, 16, true, 8, 1>(X, X, n, Ph, Pl, D, Y, st);
    }
    const size_t cnt = static_cast<size_t>(n) * D;
    float* Xh = xh_buf.get<float>(cnt);
    float* Xl = xl_buf.get<float>(cnt);
    launch_split_tf32(X, static_cast<int64_t>(cnt), Xh, Xl, st);
    if (variant == 1 && n < (int64_t(1) << 31)) {
        if (D % 192 == 0) return launch_rotate<192, 4, 16, false>(Xh, Xl, n, Ph, Pl, D, Y, st);
        return launch_rotate<128, 6, 16, false>(Xh, Xl, n, Ph, Pl, D, Y, st);
    }
    const CUtensorMap ph = tile_map(Ph, D, D, 128), pl = tile_map(Pl, D, D, 128);
    const int64_t chunk = static_cast<int64_t>(65535) * kTM;
    for (int64_t r = 0; r < n; r += chunk) {
        const int64_t rows = n - r < chunk ? n - r : chunk;
        const CUtensorMap xh = tile_map(Xh + r * D, D, rows, kTM), xl = tile_map(Xl + r * D, D, rows, kTM);
        launch_tc<3, 128, 3>(xh, xl, ph, pl, static_cast<int>(rows), D, D, StoreEpi{Y + r * D, D}, st);
    }
}

}  // namespace ads

// Coarse-quantizer GEMM on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// approx(q, c) = |q~|^2 + |c~|^2 - 2 q^.c^ for mean-centred queries q~ and
// centroids c~, with q^ / c^ their TF32 roundings (cvt.rna, done once by the
// centring kernel, coarse.cu).  The products of TF32 values are exact in fp32; the tensor core
// accumulates in fp32.  The prefilter (coarse.cu) certifies the probe order
// with the bound
//     |approx - d| <= 1.01 ((2^-10 + 2^-22 + gamma'_D + 4u) s^2 + 2 s Delta + Delta^2)
// where gamma'_D = D u' / (1 - D u') with u' = 2^-22 (one unit of 2^-23 per
// accumulation, doubled to cover truncating / aligned accumulation), 2^-10
// the two operand roundings, s = |q~| + max |c~| and Delta the centring
// round-off (see coarse.cu).  Every centroid that can reach the exact
// top-nprobe is then rescored in fp64, so the probe order stays exact.
//
// Tile: 128 queries (M) x 256 centroids (N) per CTA, K in blocks of 32 fp32
// (one 128-byte swizzle row).  Operands are staged into shared memory in the
// canonical K-major SWIZZLE_128B layout (8-row, 1024-byte atoms; 16-byte chunk
// index XOR row-in-atom) with cp.async by all 128 threads, two stages (the
// next block loads while the tensor core works on this one); one thread issues
// the 4 MMAs (K = 8 each) of a block and commits them to the stage's mbarrier;
// the accumulator (128 lanes x 256 fp32 columns) lives in TMEM and is read
// back by the four warps (each owns 32 lanes = 32 queries) with tcgen05.ld.
#include <cstdint>

#include "engine.hpp"

namespace ads {
namespace {

constexpr int kTM = 128;          // queries per tile (MMA M)
constexpr int kTN = 256;          // centroids per tile (MMA N)
constexpr int kTK = 32;           // fp32 per k-block (128 bytes)
constexpr int kAStage = kTM * 128;  // bytes
constexpr int kBStage = kTN * 128;
constexpr int kStage = kAStage + kBStage;
constexpr int kThreads = 128;
constexpr uint32_t kTmemCols = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 format):
// start >> 4 [0,14), LBO >> 4 [16,30) (unused by swizzled K-major: 1),
// SBO >> 4 [32,46) = 1024 B between 8-row atoms, version 1 [46,48),
// layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// Instruction descriptor: D fp32, A/B TF32, both K-major, N = 256, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kTN >> 3) << 17) |
                            (static_cast<uint32_t>(kTM >> 4) << 24);

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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

// Stage rows [r0, r0 + rows) x k-block kb of a row-major matrix X (n x D) of
// TF32-rounded values into a SWIZZLE_128B K-major tile at dst with cp.async
// (zeros outside the matrix); the caller commits and waits.
__device__ __forceinline__ void stage_rows(unsigned char* dst, const float* __restrict__ X, int n, int D, int r0,
                                           int rows, int kb) {
    const int k0 = kb * kTK;
#pragma unroll 4
    for (int e = threadIdx.x; e < rows * 8; e += kThreads) {
        const int r = e >> 3, ch = e & 7;  // row, 16-byte chunk
        const int row = r0 + r, col = k0 + ch * 4;
        unsigned char* p = dst + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4);
        if (row < n && col < D) {
            const uint32_t sa = smem_u32(p);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                         "l"(X + static_cast<int64_t>(row) * D + col)
                         : "memory");
        } else {
            *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
        }
    }
}

__global__ void __launch_bounds__(kThreads) tc_coarse_gemm_kernel(const float* __restrict__ Qc, int nq,
                                                                  const float* __restrict__ Cc, int L, int D,
                                                                  const float* __restrict__ qn2,
                                                                  const float* __restrict__ cn2,
                                                                  float* __restrict__ out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for the swizzle atoms
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    __shared__ uint64_t bars[2];
    __shared__ uint32_t tmem_holder;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    const int q0 = blockIdx.y * kTM, c0 = blockIdx.x * kTN;
    const int nkb = (D + kTK - 1) / kTK;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;

    uint32_t phase[2] = {0u, 0u};
    auto load = [&](int kb) {
        unsigned char* a = smem + (kb & 1) * kStage;
        stage_rows(a, Qc, nq, D, q0, kTM, kb);
        stage_rows(a + kAStage, Cc, L, D, c0, kTN, kb);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    load(0);
    for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < nkb) {  // prefetch the next block into the other stage
            const int sn = st ^ 1;
            if (kb + 1 >= 2) {  // once the MMAs that read it (block kb - 1) are done
                mbar_wait(&bars[sn], phase[sn]);
                phase[sn] ^= 1u;
            }
            load(kb + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        unsigned char* a = smem + st * kStage;
        unsigned char* b = a + kAStage;
        if (threadIdx.x == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t da = sw128_desc(smem_u32(a)), db = sw128_desc(smem_u32(b));
#pragma unroll
            for (int k = 0; k < kTK / 8; ++k) {  // K = 8 tf32 = 32 bytes per MMA
                const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                    "l"(da + static_cast<uint64_t>(k * 2)), "l"(db + static_cast<uint64_t>(k * 2)), "r"(kIdesc),
                    "r"(acc)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bars[st]))
                         : "memory");
        }
    }
    // the last commit covers every earlier MMA of this thread
    {
        const int st = (nkb - 1) & 1;
        mbar_wait(&bars[st], phase[st]);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // epilogue: warp w owns TMEM lanes (queries) 32w .. 32w + 31.  A 32 x 32
    // block goes TMEM -> registers (thread = query) -> shared memory (the
    // operand stages are free now) -> global with lane = centroid, so every
    // store writes one contiguous 128-byte row segment.
    float* tr = reinterpret_cast<float*>(smem) + warp * (32 * 33);
    const int qb = q0 + warp * 32;
    for (int cb = 0; cb < kTN; cb += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) tr[lane * 33 + j] = __uint_as_float(v[j]);
        __syncwarp();
        const int c = c0 + cb + static_cast<int>(lane);
        const float cn = c < L ? cn2[c] : 0.f;
        for (int r = 0; r < 32; ++r) {
            const int q = qb + r;
            if (q < nq && c < L) out[static_cast<int64_t>(q) * L + c] = (qn2[q] + cn) - 2.f * tr[r * 33 + lane];
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
}

}  // namespace

bool tc_coarse_supported(int D) { return D % 4 == 0; }

double tc_coarse_gamma(int D) {
    const double up = 0x1.0p-22;
    const double acc = static_cast<double>(D) * up / (1.0 - static_cast<double>(D) * up);
    return 0x1.0p-10 + 0x1.0p-22 + acc + 4.0 * 0x1.0p-24;
}

void launch_tc_coarse_gemm(const float* Qc, int nq, const float* Cc, int L, int D, const float* qn2,
                           const float* cn2, float* out, cudaStream_t st) {
    if (nq <= 0 || L <= 0) return;
    const int smem = 2 * kStage + 1024;
    ADS_CUDA(cudaFuncSetAttribute(tc_coarse_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    dim3 grid((L + kTN - 1) / kTN, (nq + kTM - 1) / kTM);
    tc_coarse_gemm_kernel<<<grid, kThreads, smem, st>>>(Qc, nq, Cc, L, D, qn2, cn2, out);
    ADS_LAUNCH_CHECK();
}

}  // namespace ads

// Shared device helpers for the B200 IVF++ ADSampling engine (sm_100a).
//
// Exact arithmetic: the reference accumulates squared differences of fp32
// inputs in fp64, in index order, with one rounding per operation (it is
// built without FMA, dco.hpp:86-93).  The helpers below spell those
// operations with the _rn intrinsics so nvcc never contracts them into a
// DFMA; the library is additionally compiled with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace ads {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define ADS_CUDA(x) ::ads::cuda_check((x), #x)
#define ADS_LAUNCH_CHECK() ::ads::cuda_check(cudaGetLastError(), "kernel launch")

__device__ __forceinline__ double sq_diff_acc(double s, float a, double b) {
    const double diff = __dsub_rn(static_cast<double>(a), b);
    return __dadd_rn(s, __dmul_rn(diff, diff));
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// cp.async (LDGSTS): global -> shared, bypassing L1 for 16-byte copies.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
#ifdef ADS_CP_ASYNC_CA
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Non-negative doubles order like their bit patterns.
__device__ __forceinline__ unsigned long long dkey(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x));
}

// One segment of a candidate's dimension range: `len` (<= 32) consecutive
// coordinates starting at global coordinate `col`, read from array `arr`
// (0 = A1 / full rows, 1 = A2).  `test` >= 0 indexes the per-query threshold
// table for a hypothesis test at col+len (< D); -1 = no test there.
struct Seg {
    int16_t arr;
    int16_t len;
    int16_t col;
    int16_t test;
};

constexpr int kMaxSeg = 128;   // D <= 4096 at 32 coordinates per segment
constexpr int kMaxTests = 128;

struct SegTable {
    int32_t nseg;
    int32_t ntest;
    int32_t vec;                 // 4 -> 16-byte copies, 1 -> 4-byte copies
    Seg seg[kMaxSeg];
    int16_t test_dim[kMaxTests]; // coordinate count d of each test
};

}  // namespace ads

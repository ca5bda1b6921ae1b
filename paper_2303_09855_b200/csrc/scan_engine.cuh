// Warp-level DCO engine shared by the fixed-threshold DCO kernel and the
// IVF++ search kernel.
//
// Each lane owns one live candidate and walks its dimension range segment by
// segment (Seg, common.cuh).  One step of a warp:
//   1. gather: the 32 lanes' current segments (each <= 32 floats, one
//      128-byte line for Δd = 32) are copied HBM -> shared memory with
//      cp.async; eight lanes cover one line, so every load instruction reads
//      four whole lines (coalesced, no sector is wasted).  Lines land in a
//      per-warp 32 x 32-float buffer with a lane-rotated 16-byte chunk order
//      so the per-lane reads below are bank-conflict free.
//   2. accumulate: each lane adds its segment in index order in fp64
//      (sq_diff_acc), against the query stored per segment (33-double pitch).
//   3. test: reject iff s > thr[test] (the reference's strict test,
//      dco.hpp:141); at d == D decide exactly (dco.hpp:145).
// Lanes whose candidate finished are refilled by the caller before the next
// step (survivor compaction by refill: a warp always gathers up to 32 live
// lines), so per-candidate cost follows the dims actually scanned and bytes
// of rejected candidates' later segments are never fetched.
#pragma once

#include "common.cuh"

namespace ads {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kQPitch = 33;  // doubles per segment slot of the staged query

template <int VEC>
__device__ __forceinline__ void gather_lines(float* wbuf, const float* src, int len) {
    const unsigned lane = lane_id();
    if constexpr (VEC == 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int L = j * 4 + static_cast<int>(lane >> 3);
            const int c = static_cast<int>(lane & 7u);
            const float* s = reinterpret_cast<const float*>(
                __shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), L));
            const int l = __shfl_sync(kFull, len, L);
            if (c * 4 < l) cp_async16(wbuf + L * 32 + (((c + L) & 7) << 2), s + c * 4);
        }
    } else {
        for (int L = 0; L < 32; ++L) {
            const float* s = reinterpret_cast<const float*>(
                __shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), L));
            const int l = __shfl_sync(kFull, len, L);
            if (static_cast<int>(lane) < l) cp_async4(wbuf + L * 32 + ((lane + L) & 31), s + lane);
        }
    }
    cp_async_wait_all();
    __syncwarp();
}

// Adds the lane's gathered segment (len floats) to s, index order, fp64.
template <int VEC>
__device__ __forceinline__ double accumulate_line(const float* wbuf, const double* qq, int len,
                                                  double s) {
    const unsigned lane = lane_id();
    const float* row = wbuf + lane * 32;
    if constexpr (VEC == 4) {
        const int nc = len >> 2;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c < nc) {
                const float4 v =
                    *reinterpret_cast<const float4*>(row + (((c + static_cast<int>(lane)) & 7) << 2));
                s = sq_diff_acc(s, v.x, qq[c * 4 + 0]);
                s = sq_diff_acc(s, v.y, qq[c * 4 + 1]);
                s = sq_diff_acc(s, v.z, qq[c * 4 + 2]);
                s = sq_diff_acc(s, v.w, qq[c * 4 + 3]);
            }
        }
    } else {
        for (int k = 0; k < len; ++k) s = sq_diff_acc(s, row[(k + lane) & 31], qq[k]);
    }
    return s;
}

// Stage query coordinates per segment: qseg[s*33 + k] = (double)q[seg.col + k].
__device__ __forceinline__ void stage_query(double* qseg, const Seg* segs, int nseg,
                                            const float* q) {
    for (int i = threadIdx.x; i < nseg * 32; i += blockDim.x) {
        const int s = i >> 5, k = i & 31;
        const Seg sg = segs[s];
        if (k < sg.len) qseg[s * kQPitch + k] = static_cast<double>(q[sg.col + k]);
    }
}

}  // namespace ads

// Warp-level DCO engine shared by the fixed-threshold DCO kernel and the
// IVF++ search kernel.
//
// Each lane owns live candidates and walks their dimension ranges segment by
// segment (Seg, common.cuh).  One step of a warp:
//   1. gather: the lanes' current segments (each <= 32 floats, one 128-byte
//      line for Δd = 32) are copied HBM -> shared memory with cp.async; eight
//      lanes cover one line, so every load instruction reads four whole lines
//      (coalesced, no sector is wasted).  Lines land in a per-warp 32 x 32-float
//      buffer (128-byte aligned) with an XOR-swizzled 16-byte chunk order (chunk c
//      of line L at slot c ^ (L & 7)) so the per-lane reads below are bank-conflict
//      free and each costs one LOP3 on the lane's row address.  Gathers are asynchronous (one cp.async
//      group per buffer) so a warp can keep two buffers in flight.
//   2. accumulate: each lane adds its segment in index order in fp64
//      (sq_diff_acc), against the query stored per segment (34-double pitch).
//   3. test: reject iff s > thr[test] (the reference's strict test,
//      dco.hpp:141); at d == D decide exactly (dco.hpp:145).
// Lanes whose candidate finished are refilled by the caller before the next
// step (survivor compaction by refill), so per-candidate cost follows the
// dims actually scanned and bytes of rejected candidates' later segments are
// never fetched.
#pragma once

#include "common.cuh"

namespace ads {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kQPitch = 34;  // doubles per segment slot of the staged query (16-byte aligned)

// 16-byte-granular line descriptor for the VEC=4 path: the line start in
// 16-byte units from one base (A1 and A2 share an allocation, A2 after A1).
constexpr uint32_t kNoLine = 0xffffffffu;

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// VEC=4: issue the copies of the warp's 32 lines (descriptors), no wait.
// full_len: every line is 32 floats (no per-line length shuffle).
// bc = base + (lane & 7) * 16 bytes (lane_base16), kept in a register by the caller.
__device__ __forceinline__ const char* lane_base16(const float* base) {
    const char* p = reinterpret_cast<const char*>(base) + (lane_id() & 7u) * 16u;
    unsigned long long v;
    // opaque copy: stops the compiler from re-deriving the pointer from the
    // kernel-parameter bank inside every predicated copy
    asm volatile("mov.b64 %0, %1;" : "=l"(v) : "l"(reinterpret_cast<unsigned long long>(p)));
    return reinterpret_cast<const char*>(v);
}

// Per-lane shared-memory destinations of gather_issue16: the lane copies chunk c =
// lane & 7 of line L = 4j + (lane >> 3) (j = 0..7) to wbuf + L*32 + (c ^ (L & 7))*4
// floats.  L & 7 = (lane >> 3) ^ 4 (j & 1), so the byte offsets are d[j & 1] + j * 512:
// two registers, computed once per kernel.
struct GatherDst {
    unsigned d0, d1;
};
__device__ __forceinline__ GatherDst gather_dst(const float* wbuf) {
    const unsigned lane = lane_id(), c = lane & 7u, l0 = lane >> 3;
    const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(wbuf)) + l0 * 128u;
    return {base + ((c ^ l0) << 4), base + ((c ^ l0 ^ 4u) << 4)};
}

// Shared address of the lane's row in the 128-byte-aligned gather buffer with the
// swizzle key folded in: chunk c of the row is at row_key ^ (c << 4).
__device__ __forceinline__ unsigned row_key(const float* wbuf) {
    const unsigned lane = lane_id();
    return static_cast<unsigned>(__cvta_generic_to_shared(wbuf)) + lane * 128u + ((lane & 7u) << 4);
}

__device__ __forceinline__ float4 lds128(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ void cp_async16_s(unsigned saddr, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}

// The same with the destinations computed per copy (fewer live registers: the exact
// walk of configs 2 / 3 measured 2 % faster this way, the fp32 walk 3 % slower).
template <bool FULL>
__device__ __forceinline__ void gather_issue16(float* wbuf, const char* bc, uint32_t desc, int nchunk) {
    const unsigned lane = lane_id();
    const int c = static_cast<int>(lane & 7u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int L = j * 4 + static_cast<int>(lane >> 3);
        const uint32_t dsc = __shfl_sync(kFull, desc, L);
        int l = 8;
        if constexpr (!FULL) l = __shfl_sync(kFull, nchunk, L);
        if (dsc != kNoLine && c < l)
            cp_async16(wbuf + L * 32 + ((c ^ (L & 7)) << 2),
                       reinterpret_cast<const float*>(bc + static_cast<uint64_t>(dsc) * 16u));
    }
    cp_async_commit();
}

template <bool FULL>
__device__ __forceinline__ void gather_issue16(const GatherDst& dst, const char* bc, uint32_t desc, int nchunk) {
    const unsigned lane = lane_id();
    const int c = static_cast<int>(lane & 7u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int L = j * 4 + static_cast<int>(lane >> 3);
        const uint32_t dsc = __shfl_sync(kFull, desc, L);
        int l = 8;
        if constexpr (!FULL) l = __shfl_sync(kFull, nchunk, L);
        if (dsc != kNoLine && c < l)
            cp_async16_s(((j & 1) ? dst.d1 : dst.d0) + j * 512u,
                         reinterpret_cast<const float*>(bc + static_cast<uint64_t>(dsc) * 16u));
    }
    cp_async_commit();
}

// VEC=1: 4-byte copies from a per-lane 64-bit pointer (unaligned layouts).
__device__ __forceinline__ void gather_issue4(float* wbuf, const float* src, int len) {
    const unsigned lane = lane_id();
    for (int L = 0; L < 32; ++L) {
        const float* s = reinterpret_cast<const float*>(
            __shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), L));
        const int l = __shfl_sync(kFull, len, L);
        if (static_cast<int>(lane) < l) cp_async4(wbuf + L * 32 + ((lane + L) & 31), s + lane);
    }
    cp_async_commit();
}

// Synchronous variants (issue + wait) used by the fixed-threshold kernel.
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
            if (c * 4 < l) cp_async16(wbuf + L * 32 + ((c ^ (L & 7)) << 2), s + c * 4);
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
// FULL: len == 32 for every segment (no per-chunk guard).
// row_key for an explicit row of the gather buffer (deep tail steps: a lane walks
// several rows in one step)
__device__ __forceinline__ unsigned row_key_at(const float* wbuf, unsigned row) {
    return static_cast<unsigned>(__cvta_generic_to_shared(wbuf)) + row * 128u + ((row & 7u) << 4);
}

// VEC=4 only: the segment gathered into buffer row `row`.
template <bool FULL>
__device__ __forceinline__ double accumulate_row(const float* wbuf, unsigned row, const double* qq, int len,
                                                 double s) {
    const int nc = FULL ? 8 : len >> 2;
    const unsigned rk = row_key_at(wbuf, row);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (FULL || c < nc) {
            const float4 v = lds128(rk ^ (static_cast<unsigned>(c) << 4));
            const double2 q0 = *reinterpret_cast<const double2*>(qq + c * 4);
            const double2 q1 = *reinterpret_cast<const double2*>(qq + c * 4 + 2);
            s = sq_diff_acc(s, v.x, q0.x);
            s = sq_diff_acc(s, v.y, q0.y);
            s = sq_diff_acc(s, v.z, q1.x);
            s = sq_diff_acc(s, v.w, q1.y);
        }
    }
    return s;
}

template <int VEC, bool FULL = false>
__device__ __forceinline__ double accumulate_line(const float* wbuf, const double* qq, int len,
                                                  double s) {
    const unsigned lane = lane_id();
    const float* row = wbuf + lane * 32;
    if constexpr (VEC == 4) {
        const int nc = FULL ? 8 : len >> 2;
        const unsigned rk = row_key(wbuf);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (FULL || c < nc) {
                const float4 v = lds128(rk ^ (static_cast<unsigned>(c) << 4));
                const double2 q0 = *reinterpret_cast<const double2*>(qq + c * 4);
                const double2 q1 = *reinterpret_cast<const double2*>(qq + c * 4 + 2);
                s = sq_diff_acc(s, v.x, q0.x);
                s = sq_diff_acc(s, v.y, q0.y);
                s = sq_diff_acc(s, v.z, q1.x);
                s = sq_diff_acc(s, v.w, q1.y);
            }
        }
    } else {
        for (int k = 0; k < len; ++k) s = sq_diff_acc(s, row[(k + lane) & 31], qq[k]);
    }
    return s;
}

// Certified fp32 walk (ivf.cu, F32): the same line with an fp32 difference and a
// fused square-add.  |s32 - S| and |s64 - S| are bounded relative to the exact sum S
// (f32_band), so a test decides only outside the band; everything inside it, and
// every candidate that may be positive at d = D, is re-walked in fp64.
__device__ __forceinline__ float accumulate_line_f32(const float* wbuf, const float* qq, float s) {
    const unsigned rk = row_key(wbuf);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 v = lds128(rk ^ (static_cast<unsigned>(c) << 4));
        const float4 q = *reinterpret_cast<const float4*>(qq + c * 4);
        float d = __fsub_rn(v.x, q.x);
        s = __fmaf_rn(d, d, s);
        d = __fsub_rn(v.y, q.y);
        s = __fmaf_rn(d, d, s);
        d = __fsub_rn(v.z, q.z);
        s = __fmaf_rn(d, d, s);
        d = __fsub_rn(v.w, q.w);
        s = __fmaf_rn(d, d, s);
    }
    return s;
}

// Query planes (exact walk on full 32-float segments).  Lanes of a warp sit at different
// segments, so the staged query is read at up to 32 different rows per instruction: as
// double2 rows (stage_query) those reads collide in the shared-memory banks and the data
// pipe becomes the scan's limiter (ncu on config 3: 85 % of its wavefront peak, 6.6
// wavefronts per query read, 100 of a step's 148).  The planes split (double)q into its
// high words, one 33-word row per segment -- bank (seg + k) mod 32, so 32 lanes at up to 32
// different segments read coordinate k in ONE wavefront -- and the low words, which for a
// converted float hold only mantissa bits 0..2 in bits 29..31 (also for denormals, inf, NaN):
// 3 bits per coordinate, ten coordinates per word, four words per segment (one 16-byte read
// per step).  q = hiloint2double(hi, (word << (29 - 3p)) & 0xE0000000) is (double)q exactly.
constexpr int kQHiPitch = 33;  // words per segment row of the high-word plane
__device__ __forceinline__ const uint32_t* q_lo_plane(const double* qseg, int nseg) {
    return reinterpret_cast<const uint32_t*>(qseg) + ((nseg * kQHiPitch + 3) & ~3);
}
__device__ __forceinline__ void stage_query_planes(double* qseg, const Seg* segs, int nseg, const float* q) {
    uint32_t* hi = reinterpret_cast<uint32_t*>(qseg);
    uint32_t* lo = const_cast<uint32_t*>(q_lo_plane(qseg, nseg));
    for (int i = threadIdx.x; i < nseg * 32; i += blockDim.x) {
        const int sgi = i >> 5, k = i & 31;
        hi[sgi * kQHiPitch + k] = static_cast<uint32_t>(__double2hiint(static_cast<double>(q[segs[sgi].col + k])));
    }
    for (int i = threadIdx.x; i < nseg * 4; i += blockDim.x) {
        const int sgi = i >> 2, w = i & 3;
        uint32_t pack = 0;
        for (int p = 0; p < 10; ++p) {
            const int k = w * 10 + p;
            if (k < 32) {
                const uint32_t l = static_cast<uint32_t>(__double2loint(static_cast<double>(q[segs[sgi].col + k])));
                pack |= (l >> 29) << (3 * p);
            }
        }
        lo[sgi * 4 + w] = pack;
    }
}
// The lane's gathered full segment in buffer row `row` against segment `seg` of the planes.
__device__ __forceinline__ double accumulate_planes(const float* wbuf, unsigned row, const double* qseg, int nseg,
                                                    int seg, double s) {
    const unsigned rk = row_key_at(wbuf, row);
    const uint32_t* qh = reinterpret_cast<const uint32_t*>(qseg) + seg * kQHiPitch;
    const uint4 lw = *reinterpret_cast<const uint4*>(q_lo_plane(qseg, nseg) + seg * 4);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 v = lds128(rk ^ (static_cast<unsigned>(c) << 4));
        const float ve[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = c * 4 + e, w = k / 10, p = k % 10;
            const uint32_t word = w == 0 ? lw.x : (w == 1 ? lw.y : (w == 2 ? lw.z : lw.w));
            const uint32_t l = (word << (29 - 3 * p)) & 0xE0000000u;
            const double q = __hiloint2double(static_cast<int>(qh[k]), static_cast<int>(l));
            s = sq_diff_acc(s, ve[e], q);
        }
    }
    return s;
}

constexpr int kQPitchF = 36;  // floats per segment slot of the fp32-staged query

__device__ __forceinline__ void stage_query_f32(float* qseg, const Seg* segs, int nseg, const float* q) {
    for (int i = threadIdx.x; i < nseg * 32; i += blockDim.x) {
        const int s = i >> 5, k = i & 31;
        const Seg sg = segs[s];
        if (k < sg.len) qseg[s * kQPitchF + k] = q[sg.col + k];
    }
}

// Band factors at depth d (terms accumulated): with S the exact sum,
// |s32 - S| <= g32 S + nabs and |s64 - S| <= g64 S, g(n, u) = n u / (1 - n u),
// n = d + 2 (difference, square, d additions), nabs covering fp32 underflow.  A
// test is certainly passed when (s32 + nabs) * hi <= thr and certainly failed when
// (s32 - nabs) * lo > thr; lo / hi also absorb the rounding of those two fp64
// operations (the 1 % widening of g32 dwarfs it).
__device__ __forceinline__ double2 f32_band(int d) {
    const double n = d + 2;
    const double g32 = 1.01 * n * 0x1p-24 / (1.0 - n * 0x1p-24);
    const double g64 = 1.01 * n * 0x1p-53 / (1.0 - n * 0x1p-53);
    return make_double2((1.0 - g64) / (1.0 + g32) * (1.0 - 0x1p-50), (1.0 + g64) / (1.0 - g32) * (1.0 + 0x1p-50));
}

// fp32 cut points of one test (threshold t, band g): a rejection is certain when
// (s - nabs) g.x > t, i.e. s > t / g.x + nabs, and a pass when (s + nabs) g.y <= t, i.e.
// s <= t / g.y - nabs.  rej / pas round those bounds outwards (up / down, fp64 then
// fp32), so the two fp32 comparisons s32 > rej and s32 <= pas imply the exact ones.
__device__ __forceinline__ void f32_cuts(double t, double2 g, double nabs, float& rej, float& pas) {
    rej = __double2float_ru(__dadd_ru(__ddiv_ru(t, g.x), nabs));
    pas = __double2float_rd(__dsub_rd(__ddiv_rd(t, g.y), nabs));
}

// Stage query coordinates per segment: qseg[s*34 + k] = (double)q[seg.col + k].
__device__ __forceinline__ void stage_query(double* qseg, const Seg* segs, int nseg,
                                            const float* q) {
    for (int i = threadIdx.x; i < nseg * 32; i += blockDim.x) {
        const int s = i >> 5, k = i & 31;
        const Seg sg = segs[s];
        if (k < sg.len) qseg[s * kQPitch + k] = static_cast<double>(q[sg.col + k]);
    }
}

}  // namespace ads

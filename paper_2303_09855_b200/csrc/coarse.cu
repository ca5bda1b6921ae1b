// Certified coarse quantizer: the exact probe order of probe_order
// (ivf.cpp:283-292: fp64 l2_sq per centroid, partial_sort by (d2, id)) at a
// fraction of the exact cost.
//
//  1. the approximate distance matrix: tcgen05 TF32 tiles (tc_gemm.cu, the
//     default; its bound is documented there) or approx_gemm_kernel — fp32
//     FMA tiles on mean-centred vectors
//     q~ = fl32(q - mu), c~ = fl32(c - mu) (centring in fp64, mu = centroid
//     mean): a(q,c) = |q~|^2 + |c~|^2 - 2 q~.c~.  Rigorous bound, with
//     s = |q~| + cmax~ (u = 2^-24, gamma_D = D u / (1 - D u)):
//       |a - d| <= (gamma_D + 4u) s^2 + 2 s Delta + Delta^2,  Delta = 2u s
//     (Cauchy-Schwarz on the dot product and the norms, the final roundings,
//     and the centring round-off moving q~ - c~ by at most Delta), inflated
//     by 1 %.  Centring keeps s at the scale of the distances themselves.
//  2. prefilter_kernel — per query, T = the nprobe-th smallest a(q,.) (radix
//     select on order-preserving float keys); every centroid that can be in
//     the exact top-nprobe satisfies a(q,c) <= T + 2 E(q) (the nprobe
//     centroids with a <= T all have d <= T + E, so the exact nprobe-th
//     distance is <= T + E, and d(q,c) <= that implies a(q,c) <= T + 2E).
//     Those centroids are rescored with the exact fp64 l2_sq (reference
//     order) and the nprobe smallest (d2, id) pairs are emitted in order.
//     If more than `cap` centroids pass (never in practice), that query falls
//     back to exact scoring of every centroid inside the same kernel.
#include <cfloat>
#include <cstdio>

#include "engine.hpp"
#include "scan_engine.cuh"

namespace ads {

namespace {

constexpr int kGT = 64;   // queries per CTA tile
constexpr int kGC = 64;   // centroids per CTA tile
constexpr int kGK = 16;   // depth per stage

// 256 threads; each computes 4 queries x 4 centroids.
__global__ void __launch_bounds__(256) approx_gemm_kernel(const float* __restrict__ Q, int nq,
                                                          const float* __restrict__ C, int L, int D,
                                                          const float* __restrict__ qn2,
                                                          const float* __restrict__ cn2,
                                                          float* __restrict__ out) {
    __shared__ float qs[kGK][kGT + 4];
    __shared__ float cs[kGK][kGC + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int q0 = blockIdx.y * kGT, c0 = blockIdx.x * kGC;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int k0 = 0; k0 < D; k0 += kGK) {
        for (int idx = threadIdx.x; idx < kGT * kGK; idx += 256) {
            const int r = idx / kGK, k = idx % kGK;
            qs[k][r] = (q0 + r < nq && k0 + k < D) ? Q[static_cast<int64_t>(q0 + r) * D + k0 + k] : 0.f;
            cs[k][r] = (c0 + r < L && k0 + k < D) ? C[static_cast<int64_t>(c0 + r) * D + k0 + k] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kGK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = qs[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = cs[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int q = q0 + ty * 4 + i;
        if (q >= nq) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + tx * 4 + j;
            if (c < L) out[static_cast<int64_t>(q) * L + c] = (qn2[q] + cn2[c]) - 2.f * acc[i][j];
        }
    }
}

// X~ = fl32(X - mu) (fp64 subtraction), |X~|^2 (fp64 -> fp32) and |X~| (fp64).
// tf32: store X~ rounded to TF32 (cvt.rna) for the tensor-core GEMM; the norms
// stay those of X~ (tc_gemm.cu's bound accounts for the rounding).
__global__ void center_norms_kernel(const float* __restrict__ X, int n, int D,
                                    const double* __restrict__ mu, float* __restrict__ Xc,
                                    float* __restrict__ n2, double* __restrict__ nrm, int tf32) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const unsigned lane = threadIdx.x & 31u;
    if (i >= n) return;
    double s = 0.0;
    for (int j = static_cast<int>(lane); j < D; j += 32) {
        const float c = static_cast<float>(static_cast<double>(X[static_cast<int64_t>(i) * D + j]) - mu[j]);
        float cs = c;
        if (tf32) {
            uint32_t r;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(c));
            cs = __uint_as_float(r);
        }
        if (Xc) Xc[static_cast<int64_t>(i) * D + j] = cs;
        const double v = c;
        s += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        n2[i] = static_cast<float>(s);
        nrm[i] = sqrt(s);
    }
}

__device__ __forceinline__ unsigned fkey(float x) {
    const unsigned b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// prefilter threads per query (one CTA per query): 128 for nprobe <= 128
// (twice the queries in flight per SM; +3.8 % end to end at nprobe 8), else 256
constexpr int kPTSmall = 128, kPTLarge = 256;

// Exact l2_sq(centroid, q) (ivf.cpp:287), reference order, one thread per
// centroid: the row streams in with 16-float prefetched vector loads while the
// dependent fp64 add chain runs; the query sits in shared memory as doubles.
__device__ __forceinline__ double exact_d2(const float* __restrict__ c, const double* __restrict__ qs,
                                           int D) {
    double s = 0.0;
    int j = 0;
    if ((D & 3) == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0 && D >= 16) {
        const float4* c4 = reinterpret_cast<const float4*>(c);
        float4 nxt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) nxt[u] = __ldg(c4 + u);
        for (; j + 16 <= D; j += 16) {
            float4 cur[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
            if (j + 32 <= D) {
#pragma unroll
                for (int u = 0; u < 4; ++u) nxt[u] = __ldg(c4 + (j >> 2) + 4 + u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s = sq_diff_acc(s, cur[u].x, qs[j + 4 * u + 0]);
                s = sq_diff_acc(s, cur[u].y, qs[j + 4 * u + 1]);
                s = sq_diff_acc(s, cur[u].z, qs[j + 4 * u + 2]);
                s = sq_diff_acc(s, cur[u].w, qs[j + 4 * u + 3]);
            }
        }
    }
    for (; j < D; ++j) s = sq_diff_acc(s, c[j], qs[j]);
    return s;
}

template <int kPT>
__global__ void __launch_bounds__(kPT) prefilter_kernel(const float* __restrict__ approx, int L,
                                                        const float* __restrict__ Q,
                                                        const float* __restrict__ C, int D, int nprobe,
                                                        const double* __restrict__ qnrm, double cmax,
                                                        double gamma, int cap, int P2,
                                                        int32_t* __restrict__ probes,
                                                        unsigned long long* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* cd = reinterpret_cast<double*>(sm);          // P2 exact distances
    double* qd = cd + P2;                                // the query as doubles
    int32_t* ci = reinterpret_cast<int32_t*>(qd + D);    // P2 centroid ids
    __shared__ int s_n, s_full;
    const int q = blockIdx.x, tid = threadIdx.x;
    const float* row = approx + static_cast<int64_t>(q) * L;
    const float* qv = Q + static_cast<int64_t>(q) * D;
    for (int j = tid; j < D; j += kPT) qd[j] = static_cast<double>(qv[j]);
    if (tid == 0) {
        s_n = 0;
        s_full = 0;
    }
    __syncthreads();
    // T: any value with at least nprobe centroids at or below it keeps the
    // certificate valid (see the header).  Each thread keeps its two smallest
    // approximate distances; T = the nprobe-th smallest of those 2*kPT values
    // (>= the true nprobe-th smallest; slightly looser, far cheaper than a
    // full selection).
    float m1 = __builtin_huge_valf(), m2 = __builtin_huge_valf();
    auto keep2 = [&](float v) {
        if (v < m1) {
            m2 = m1;
            m1 = v;
        } else if (v < m2) {
            m2 = v;
        }
    };
    const bool vec = (L & 3) == 0;  // rows are 16-byte aligned: float4 loads, 4 in flight
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 4
        for (int c = tid; c < (L >> 2); c += kPT) {
            const float4 v = __ldg(r4 + c);
            keep2(v.x);
            keep2(v.y);
            keep2(v.z);
            keep2(v.w);
        }
    } else {
        for (int c = tid; c < L; c += kPT) keep2(row[c]);
    }
    // T = the nprobe-th smallest of those 2*kPT values: 8-bit radix select on
    // order-preserving keys (4 passes of a 256-bin histogram)
    unsigned* hist = reinterpret_cast<unsigned*>(ci);  // scratch: 256 bins (ci has >= 512 slots)
    __shared__ unsigned s_prefix, s_rank;
    const unsigned k1 = fkey(m1), k2 = fkey(m2);
    if (tid == 0) {
        s_prefix = 0u;
        s_rank = static_cast<unsigned>(nprobe - 1 < 2 * kPT - 1 ? nprobe - 1 : 2 * kPT - 1);
    }
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += kPT) hist[b] = 0u;  // 256 bins
        __syncthreads();
        const unsigned pre = s_prefix;
        const unsigned hmask = shift == 24 ? 0u : (0xffffffffu << (shift + 8));
        if ((k1 & hmask) == (pre & hmask)) atomicAdd(&hist[(k1 >> shift) & 255u], 1u);
        if ((k2 & hmask) == (pre & hmask)) atomicAdd(&hist[(k2 >> shift) & 255u], 1u);
        __syncthreads();
        if (tid < 32) {  // find the bin holding rank s_rank
            unsigned carry = 0, want = s_rank;
            int found = -1;
            unsigned below = 0;
            for (int b0 = 0; b0 < 256 && found < 0; b0 += 32) {
                const unsigned c = hist[b0 + tid];
                unsigned incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += v;
                }
                const unsigned excl = carry + incl - c;
                const unsigned hit = __ballot_sync(0xffffffffu, excl <= want && want < excl + c);
                if (hit) {
                    const int l = __ffs(hit) - 1;
                    found = b0 + l;
                    below = __shfl_sync(0xffffffffu, excl, l);
                }
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (tid == 0) {
                s_prefix = pre | (static_cast<unsigned>(found) << shift);
                s_rank = want - below;
            }
        }
        __syncthreads();
    }
    const unsigned tkey = s_prefix;
    const float T = __uint_as_float((tkey & 0x80000000u) ? (tkey & 0x7fffffffu) : ~tkey);
    __syncthreads();
    const double sn = qnrm[q] + cmax;
    const double delta = 2.0 * 0x1.0p-24 * sn;
    const double e = 1.01 * (gamma * sn * sn + 2.0 * sn * delta + delta * delta);
    const double lim = static_cast<double>(T) + 2.0 * e;
    auto take = [&](float v, int c) {
        if (static_cast<double>(v) <= lim) {
            const int slot = atomicAdd(&s_n, 1);
            if (slot < cap) ci[slot] = c;
        }
    };
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 4
        for (int c = tid; c < (L >> 2); c += kPT) {
            const float4 v = __ldg(r4 + c);
            take(v.x, 4 * c);
            take(v.y, 4 * c + 1);
            take(v.z, 4 * c + 2);
            take(v.w, 4 * c + 3);
        }
    } else {
        for (int c = tid; c < L; c += kPT) take(row[c], c);
    }
    __syncthreads();
    int n = s_n;
#ifdef ADS_DEBUG
    if (tid == 0 && (q < 6 || n > cap))
        printf("PREFILTER q=%d n=%d cap=%d T=%.9g e=%.6g qn=%.6g cmax=%.6g\n", q, n, cap, (double)T, e, qnrm[q], cmax);
#endif
    if (tid == 0) {
        atomicAdd(&stats[0], static_cast<unsigned long long>(n));
        if (n > cap) atomicAdd(&stats[1], 1ull);
    }
    if (n > cap) {  // fallback: exact scoring of every centroid (keep the nprobe best)
        n = L;
        if (tid == 0) s_full = 1;
    }
    __syncthreads();
    if (!s_full && n <= kPT) {
        // one candidate per thread: exact distance, then its rank among the
        // candidates by (d2, id) (ids are distinct) is its slot in the order
        double di = 0.0;
        int32_t ii = 0;
        if (tid < n) {
            ii = ci[tid];
            di = exact_d2(C + static_cast<int64_t>(ii) * D, qd, D);
            cd[tid] = di;
        }
        __syncthreads();
        if (tid < n) {
            int rank = 0;
            for (int j = 0; j < n; ++j) {
                const double dj = cd[j];
                const int32_t ij = ci[j];
                rank += dj < di || (dj == di && ij < ii);
            }
            if (rank < nprobe) probes[static_cast<int64_t>(q) * nprobe + rank] = ii;
        }
    } else if (!s_full) {
        int P = 2;
        while (P < n) P <<= 1;
        for (int i = tid; i < n; i += kPT) cd[i] = exact_d2(C + static_cast<int64_t>(ci[i]) * D, qd, D);
        for (int i = n + tid; i < P; i += kPT) {
            cd[i] = __builtin_huge_val();
            ci[i] = 0x7fffffff;
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = tid; i < P / 2; i += kPT) {
                    const int lo = 2 * i - (i & (stride - 1));
                    const int hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const double da = cd[lo], db = cd[hi];
                    const int32_t ia = ci[lo], ib = ci[hi];
                    const bool gt = da > db || (da == db && ia > ib);
                    if (gt == up) {
                        cd[lo] = db;
                        cd[hi] = da;
                        ci[lo] = ib;
                        ci[hi] = ia;
                    }
                }
                __syncthreads();
            }
        }
        for (int i = tid; i < nprobe; i += kPT) probes[static_cast<int64_t>(q) * nprobe + i] = ci[i];
    } else {
        // rare path: one thread keeps a sorted exact top-nprobe over all centroids
        if (tid == 0) {
            int cnt = 0;
            for (int c = 0; c < L; ++c) {
                const double d = exact_d2(C + static_cast<int64_t>(c) * D, qd, D);
                if (cnt == nprobe && !(d < cd[nprobe - 1])) continue;  // ties keep the lower id
                int pos = cnt < nprobe ? cnt : nprobe - 1;
                while (pos > 0 && cd[pos - 1] > d) {
                    cd[pos] = cd[pos - 1];
                    ci[pos] = ci[pos - 1];
                    --pos;
                }
                cd[pos] = d;
                ci[pos] = c;
                if (cnt < nprobe) ++cnt;
            }
            for (int i = 0; i < nprobe; ++i) probes[static_cast<int64_t>(q) * nprobe + i] = ci[i];
        }
    }
}

}  // namespace

void coarse_center(const float* X, int n, int D, const double* mu, float* Xc, float* n2, double* nrm,
                   cudaStream_t st, bool tf32) {
    if (n <= 0) return;
    center_norms_kernel<<<(n + 7) / 8, 256, 0, st>>>(X, n, D, mu, Xc, n2, nrm, tf32 ? 1 : 0);
    ADS_LAUNCH_CHECK();
}

void launch_coarse_probes_fast(const float* Q, int nq, const float* C, int L, int D, int nprobe,
                               const CoarseCentroids& cc, CoarseScratch& s, int32_t* probes, int gemm,
                               cudaStream_t st) {
    if (nq <= 0) return;
    float* approx = s.approx.get<float>(static_cast<size_t>(nq) * L);
    float* qc = s.qc.get<float>(static_cast<size_t>(nq) * D);
    float* qn2 = s.qn2.get<float>(nq);
    double* qnrm = s.qnrm.get<double>(nq);
    const bool tc = gemm == 0 && tc_coarse_supported(D) && cc.cc_tf;
    coarse_center(Q, nq, D, cc.mu, qc, qn2, qnrm, st, tc);
    const double cmax = cc.cmax;
    double gamma;
    if (tc) {  // tcgen05 TF32 (tc_gemm.cu) on TF32-rounded operands
        launch_tc_coarse_gemm(qc, nq, cc.cc_tf, L, D, qn2, cc.cn2, approx, st);
        gamma = tc_coarse_gamma(D);
    } else {  // fp32 FMA tiles
        dim3 grid((L + kGC - 1) / kGC, (nq + kGT - 1) / kGT);
        approx_gemm_kernel<<<grid, 256, 0, st>>>(qc, nq, cc.cc, L, D, qn2, cc.cn2, approx);
        ADS_LAUNCH_CHECK();
        const double u = 0x1.0p-24;
        gamma = (static_cast<double>(D) * u) / (1.0 - static_cast<double>(D) * u) + 4.0 * u;
    }
    unsigned long long* stats = s.stats.get<unsigned long long>(2);
    ADS_CUDA(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), st));
    s.last_nq = nq;
    if (nprobe > 2 * kPTLarge) throw std::invalid_argument("coarse prefilter: nprobe > 512 (use coarse_mode 1)");
    const int pt = nprobe <= kPTSmall ? kPTSmall : kPTLarge;
    int cap = 4 * nprobe + 256;
    if (cap > L) cap = L;
    int P2 = 2 * pt;  // also hosts the 2*pt threshold keys and the 256 radix bins
    if (P2 < 256) P2 = 256;
    while (P2 < cap) P2 <<= 1;
    const size_t smem = static_cast<size_t>(P2) * (sizeof(double) + sizeof(int32_t)) + sizeof(double) * D;
    if (smem > 200 * 1024) throw std::invalid_argument("coarse: nprobe too large for the prefilter");
    auto kern = pt == kPTSmall ? prefilter_kernel<kPTSmall> : prefilter_kernel<kPTLarge>;
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<nq, pt, smem, st>>>(approx, L, Q, C, D, nprobe, qnrm, cmax, gamma, cap, P2, probes, stats);
    ADS_LAUNCH_CHECK();
}

}  // namespace ads

// IVF/IVF++ batched search on sm_100a (ivf_query, ivf.cpp:296-419).
//
//   coarse_dist_kernel   exact fp64 query-centroid distances (l2_sq order,
//                        ivf.cpp:287), tiled through shared memory
//   select_rows_kernel   per-row top-k by (d2, index) pairs: radix select +
//                        ordered tie fill + bitonic sort (partial_sort,
//                        ivf.cpp:288; also brute_force_knn's pair order)
//   ivf_search_kernel    one CTA per query (persistent).  The query's probed
//                        lists form one candidate stream in probe order;
//                        warps refill lanes from it and run the DCO engine
//                        (scan_engine.cuh) against the per-query threshold
//                        table.  The running K-th distance r is refreshed at
//                        deterministic stream positions (0, first,
//                        first+step, ...): positives of a chunk are offered
//                        to the bounded (dist, id) heap in candidate order
//                        with the reference's strict rule (ivf.cpp:273-280),
//                        then thr[t] = factor[d_t] * r^2 is rebuilt.
#include <cfloat>
#include <climits>
#include <type_traits>

#include "engine.hpp"
#include "scan_engine.cuh"

namespace ads {

namespace {

constexpr double kInf = __builtin_huge_val();

// ---------------------------------------------------------------- coarse distances
constexpr int kCT = 128;  // centroids per CTA (one per thread)
constexpr int kQT = 8;    // queries per CTA
constexpr int kDK = 32;   // dims per stage

__global__ void __launch_bounds__(kCT) coarse_dist_kernel(const float* __restrict__ Q, int nq,
                                                          const float* __restrict__ C, int L,
                                                          int D, double* __restrict__ out) {
    __shared__ float ct[kCT * (kDK + 1)];
    __shared__ double qt[kQT][kDK];
    const int c0 = blockIdx.x * kCT;
    const int q0 = blockIdx.y * kQT;
    const int tid = threadIdx.x;
    double acc[kQT];
#pragma unroll
    for (int i = 0; i < kQT; ++i) acc[i] = 0.0;
    for (int d0 = 0; d0 < D; d0 += kDK) {
        const int len = D - d0 < kDK ? D - d0 : kDK;
        for (int idx = tid; idx < kCT * kDK; idx += kCT) {
            const int c = idx / kDK, k = idx % kDK;
            float v = 0.f;
            if (c0 + c < L && k < len) v = C[static_cast<int64_t>(c0 + c) * D + d0 + k];
            ct[c * (kDK + 1) + k] = v;
        }
        for (int idx = tid; idx < kQT * kDK; idx += kCT) {
            const int qq = idx / kDK, k = idx % kDK;
            double v = 0.0;
            if (q0 + qq < nq && k < len) v = static_cast<double>(Q[static_cast<int64_t>(q0 + qq) * D + d0 + k]);
            qt[qq][k] = v;
        }
        __syncthreads();
        for (int k = 0; k < len; ++k) {
            const float cv = ct[tid * (kDK + 1) + k];
#pragma unroll
            for (int qq = 0; qq < kQT; ++qq) acc[qq] = sq_diff_acc(acc[qq], cv, qt[qq][k]);
        }
        __syncthreads();
    }
    if (c0 + tid < L) {
#pragma unroll
        for (int qq = 0; qq < kQT; ++qq)
            if (q0 + qq < nq) out[static_cast<int64_t>(q0 + qq) * L + c0 + tid] = acc[qq];
    }
}

// ---------------------------------------------------------------- per-row top-k select
constexpr int kSelThreads = 256;

// keys: non-negative doubles as uint64 (order-preserving).  Output the kk
// smallest (key, col) pairs of each row, ascending.  Dynamic smem holds the
// padded sort buffer: P2 * (8 + 4) bytes.
__global__ void __launch_bounds__(kSelThreads) select_rows_kernel(const double* __restrict__ dist,
                                                                  int64_t L, int kk, int P2,
                                                                  int32_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long* sk = reinterpret_cast<unsigned long long*>(sm);
    int32_t* si = reinterpret_cast<int32_t*>(sk + P2);
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ int s_rank, s_nsel, s_eqbase;
    __shared__ int warp_cnt[kSelThreads / 32];

    const double* row = dist + static_cast<int64_t>(blockIdx.x) * L;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_rank = kk;
        s_nsel = 0;
        s_eqbase = 0;
    }
    __syncthreads();
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kSelThreads) hist[i] = 0;
        __syncthreads();
        const unsigned long long prefix = s_prefix, mask = s_mask;
        for (int64_t c = tid; c < L; c += kSelThreads) {
            const unsigned long long key = dkey(row[c]);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255ull], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            int rank = s_rank;
            unsigned cum = 0;
            int digit = 255;
            for (int b = 0; b < 256; ++b) {
                if (static_cast<int>(cum + hist[b]) >= rank) {
                    digit = b;
                    break;
                }
                cum += hist[b];
            }
            s_rank = rank - static_cast<int>(cum);
            s_prefix = prefix | (static_cast<unsigned long long>(digit) << shift);
            s_mask = mask | (255ull << shift);
        }
        __syncthreads();
    }
    const unsigned long long T = s_prefix;
    const int need_eq = s_rank;  // how many keys == T to take (lowest indices)
    // keys strictly below T: all of them (kk - need_eq of them)
    for (int64_t c = tid; c < L; c += kSelThreads) {
        const unsigned long long key = dkey(row[c]);
        if (key < T) {
            const int slot = atomicAdd(&s_nsel, 1);
            sk[slot] = key;
            si[slot] = static_cast<int32_t>(c);
        }
    }
    __syncthreads();
    const int nlt = s_nsel;
    // keys == T in ascending column order until need_eq are taken
    for (int64_t base = 0; base < L; base += kSelThreads) {
        if (s_eqbase >= need_eq) break;  // uniform (read after barrier)
        const int64_t c = base + tid;
        const bool eq = c < L && dkey(row[c]) == T;
        const unsigned b = __ballot_sync(kFull, eq);
        if ((tid & 31) == 0) warp_cnt[tid >> 5] = __popc(b);
        __syncthreads();
        int before = s_eqbase;
        for (int w = 0; w < (tid >> 5); ++w) before += warp_cnt[w];
        before += __popc(b & ((1u << (tid & 31)) - 1u));
        if (eq && before < need_eq) {
            sk[nlt + before] = T;
            si[nlt + before] = static_cast<int32_t>(c);
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < kSelThreads / 32; ++w) tot += warp_cnt[w];
            s_eqbase += tot;
        }
        __syncthreads();
    }
    for (int i = kk + tid; i < P2; i += kSelThreads) {
        sk[i] = ~0ull;
        si[i] = 0x7fffffff;
    }
    __syncthreads();
    // bitonic sort by (key, idx)
    for (int size = 2; size <= P2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P2 / 2; i += kSelThreads) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long ka = sk[lo], kb = sk[hi];
                const int32_t ia = si[lo], ib = si[hi];
                const bool a_gt_b = ka > kb || (ka == kb && ia > ib);
                if (a_gt_b == up) {
                    sk[lo] = kb;
                    sk[hi] = ka;
                    si[lo] = ib;
                    si[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < kk; i += kSelThreads) out[static_cast<int64_t>(blockIdx.x) * kk + i] = si[i];
}

// ---------------------------------------------------------------- search
__device__ __forceinline__ bool pair_lt(double da, int32_t ia, double db, int32_t ib) {
    return da < db || (da == db && ia < ib);
}

// ivf.cpp:273-280 offer(), executed by one full warp on the shared sorted array.
__device__ void warp_offer(double* topd, int32_t* topi, int* cnt, int K, double dist, int32_t id) {
    const unsigned lane = lane_id();
    const int c = *cnt;
    if (c == K && !(dist < topd[K - 1])) return;  // strict: ties at the max are not inserted
    const int ceff = c == K ? K - 1 : c;           // pop the max pair when full
    int pos = 0;
    for (int base = 0; base < ceff; base += 32) {
        const int j = base + static_cast<int>(lane);
        const bool lt = j < ceff && pair_lt(topd[j], topi[j], dist, id);
        pos += __popc(__ballot_sync(kFull, lt));
    }
    for (int top = ceff - 1; top >= pos; top -= 32) {
        const int j = top - static_cast<int>(lane);
        const bool valid = j >= pos;
        double v = 0.0;
        int32_t vi = 0;
        if (valid) {
            v = topd[j];
            vi = topi[j];
        }
        __syncwarp();
        if (valid) {
            topd[j + 1] = v;
            topi[j + 1] = vi;
        }
        __syncwarp();
    }
    if (lane == 0) {
        topd[pos] = dist;
        topi[pos] = id;
        *cnt = ceff + 1;
    }
    __syncwarp();
}

#ifndef ADS_QUERY_PLANES
#define ADS_QUERY_PLANES 1
#endif
constexpr bool kQueryPlanes = ADS_QUERY_PLANES != 0;  // scan_engine.cuh, stage_query_planes

// Live candidates per warp at or below which a step goes deep (0: off).
#ifndef ADS_DEEP_TAIL
#define ADS_DEEP_TAIL 16
#endif
constexpr int kDeepTail = ADS_DEEP_TAIL;
#ifndef ADS_DEEP_SHIFT
#define ADS_DEEP_SHIFT 2
#endif
constexpr int kDeepShift = ADS_DEEP_SHIFT;  // a candidate takes at most 1 << kDeepShift rows in a deep step

#ifndef ADS_DEEP_MIN_NSEG
#define ADS_DEEP_MIN_NSEG 8
#endif
constexpr int kDeepMinSeg = ADS_DEEP_MIN_NSEG;  // walks shorter than this have no tail to speak of

// Set bits in flags[0, nw), the same value in every thread: each warp counts lane-parallel
// (one word per lane and pass) and reduces, instead of every thread walking all the words.
__device__ __forceinline__ int flag_count(const unsigned* flags, int nw) {
    int c = 0;
    for (int b = 0; b < nw; b += 32) {
        const int i = b + static_cast<int>(lane_id());
        c += __reduce_add_sync(kFull, i < nw ? __popc(flags[i]) : 0);
    }
    return c;
}

struct SearchShared {
    double r, r_sq;
    int q, stop, total, next, cnt, pnext;
    int pcount[2];
    int nsurv;  // DENSE: candidates of the chunk that passed the test at d1
    unsigned long long dims;
};

// The same rank merge with every thread of the CTA, for chunks with many
// positives (r still loose early in a query).  Kept positives are compacted
// in candidate order to pend_d/pend_i[0, m) first.  Returns m on success,
// -(m + 1) on a tie (the compacted batch is then offered sequentially).
// Needs n <= 2 * blockDim.x and sh.cnt <= 2 * blockDim.x; call with all threads.
__device__ __noinline__ int cta_merge_chunk(double* topd, int32_t* topi, SearchShared& sh, int K, double* pend_d,
                               int32_t* pend_i, const unsigned* pflag, int n, int* wc) {
    const int tid = threadIdx.x, nthr = blockDim.x, nwarps = nthr >> 5, warp = tid >> 5;
    const unsigned lane = lane_id();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int c = sh.cnt;
    const bool full = c == K;
    const double maxd = full ? topd[K - 1] : kInf;
    double d[2];
    int32_t id[2];
    bool keep[2];
    unsigned kb[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int slot = r * nthr + tid;
        keep[r] = slot < n && ((pflag[slot >> 5] >> (slot & 31)) & 1u);
        d[r] = 0.0;
        id[r] = 0;
        if (keep[r]) {
            d[r] = pend_d[slot];
            id[r] = pend_i[slot];
            keep[r] = !full || d[r] < maxd;  // the max only decreases
        }
        kb[r] = __ballot_sync(kFull, keep[r]);
        if (lane == 0) wc[r * nwarps + warp] = __popc(kb[r]);
    }
    __syncthreads();
    int m = 0, off[2] = {0, 0};
    for (int e = 0; e < 2 * nwarps; ++e) {
        const int v = wc[e];
        if (e < warp) off[0] += v;
        if (e < nwarps + warp) off[1] += v;
        m += v;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (keep[r]) {
            const int k = off[r] + __popc(kb[r] & lt_mask);
            pend_d[k] = d[r];
            pend_i[k] = id[r];
        }
    }
    __syncthreads();
    bool tie = false;
    int bnew[2] = {-1, -1}, snew[2] = {-1, -1};
    double sd[2] = {0.0, 0.0};
    int32_t si[2] = {0, 0};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int kk = r * nthr + tid;
        if (kk < m) {  // batch entry: rank in the batch + rank in the top-K
            d[r] = pend_d[kk];
            id[r] = pend_i[kk];
            int less = 0;
            for (int k = 0; k < m; ++k) {
                const double od = pend_d[k];
                less += pair_lt(od, pend_i[k], d[r], id[r]);
                tie |= od == d[r] && k != kk;
            }
            int lo = 0, hi = c;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (pair_lt(topd[mid], topi[mid], d[r], id[r])) lo = mid + 1;
                else hi = mid;
            }
            bnew[r] = lo + less;
        }
        const int i = r * nthr + tid;
        if (i < c) {  // top-K entry: index + batch entries below it
            sd[r] = topd[i];
            si[r] = topi[i];
            int below = 0;
            for (int k = 0; k < m; ++k) {
                const double od = pend_d[k];
                below += pair_lt(od, pend_i[k], sd[r], si[r]);
                tie |= od == sd[r];
            }
            snew[r] = i + below;
        }
    }
    if (__syncthreads_or(tie)) return -(m + 1);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        if (snew[r] >= 0 && snew[r] < K) {
            topd[snew[r]] = sd[r];
            topi[snew[r]] = si[r];
        }
        if (bnew[r] >= 0 && bnew[r] < K) {
            topd[bnew[r]] = d[r];
            topi[bnew[r]] = id[r];
        }
    }
    if (tid == 0) sh.cnt = c + m < K ? c + m : K;
    __syncthreads();
    return m;
}

// Offers a chunk's positives (pflag bits over pend_d/pend_i, candidate order)
// to the sorted top-K in one pass of one warp.  When no positive's distance
// equals another distance of the top-K or the batch, the sequential offers of
// ivf.cpp:273-280 (insert iff dist < max when full, strictly; pop the max
// (dist, id) pair) leave exactly the K smallest pairs of top-K ∪ batch, so
// every entry moves to its rank in the union.  Returns false, with nothing
// changed, on a tie or more than 32 surviving positives (sequential path).
__device__ bool warp_merge_chunk(double* topd, int32_t* topi, SearchShared& sh, int K, const double* pend_d,
                                 const int32_t* pend_i, const unsigned* pflag, int n) {
    const unsigned lane = lane_id();
    const int c = sh.cnt;
    const bool full = c == K;
    const double maxd = full ? topd[K - 1] : kInf;
    // batch: up to 32 kept positives, lane t holds the t-th in candidate order
    double bd = 0.0;
    int32_t bi = 0;
    int m = 0;
    for (int w = 0; w < ((n + 31) >> 5); ++w) {
        const unsigned bits = pflag[w];
        if (!bits) continue;
        double d = 0.0;
        int32_t id = 0;
        bool keep = false;
        if ((bits >> lane) & 1u) {
            d = pend_d[w * 32 + lane];
            id = pend_i[w * 32 + lane];
            keep = !full || d < maxd;  // the max only decreases: rejected whatever comes first
        }
        const unsigned kb = __ballot_sync(kFull, keep);
        if (!kb) continue;
        const int tot = m + __popc(kb);
        if (tot > 32) return false;
        const int t = static_cast<int>(lane) - m;
        const int src = (t >= 0 && t < tot - m) ? static_cast<int>(__fns(kb, 0, t + 1)) : 0;
        const double dd = __shfl_sync(kFull, d, src);
        const int32_t ii = __shfl_sync(kFull, id, src);
        if (t >= 0 && t < tot - m) {
            bd = dd;
            bi = ii;
        }
        m = tot;
    }
    if (m == 0) return true;
    const bool mine = static_cast<int>(lane) < m;
    int rb = 0;  // batch entries below mine
    bool tie = false;
    for (int k = 0; k < m; ++k) {
        const double od = __shfl_sync(kFull, bd, k);
        const int32_t oi = __shfl_sync(kFull, bi, k);
        if (mine && k != static_cast<int>(lane)) {
            rb += pair_lt(od, oi, bd, bi);
            tie |= od == bd;
        }
    }
    int rs = 0;  // top-K entries below mine
    if (mine) {
        int lo = 0, hi = c;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (pair_lt(topd[mid], topi[mid], bd, bi)) lo = mid + 1;
            else hi = mid;
        }
        tie |= (lo > 0 && topd[lo - 1] == bd) || (lo < c && topd[lo] == bd);
        rs = lo;
    }
    if (__any_sync(kFull, tie)) return false;
    // top-K entries only move up: move 32-entry groups from the top down
    for (int g = (c - 1) >> 5; g >= 0; --g) {
        const int i = g * 32 + static_cast<int>(lane);
        double sd = 0.0;
        int32_t si = 0;
        int below = 0;
        if (i < c) {
            sd = topd[i];
            si = topi[i];
        }
        for (int k = 0; k < m; ++k) {
            const double od = __shfl_sync(kFull, bd, k);
            const int32_t oi = __shfl_sync(kFull, bi, k);
            below += pair_lt(od, oi, sd, si);
        }
        __syncwarp();
        if (i < c && i + below < K) {
            topd[i + below] = sd;
            topi[i + below] = si;
        }
        __syncwarp();
    }
    if (mine && rs + rb < K) {
        topd[rs + rb] = bd;
        topi[rs + rb] = bi;
    }
    if (lane == 0) sh.cnt = c + m < K ? c + m : K;
    __syncwarp();
    return true;
}

#ifndef DENSE_PARTS
#define DENSE_PARTS 1  // the prefix phase loads its 8 chunks in this many rounds (1: all in flight)
#endif
// Dense prefix phase (DENSE, IVF++ with a 32-float A1 over the transformed split
// layout).  The reference computes every candidate's A1 prefix before any test
// (ivf.cpp:366-386); no decision depends on those sums, and within a chunk the
// threshold is fixed, so at each chunk start the CTA computes all the chunk's
// prefixes from the interleaved A1 copy (a1i: a warp reads 32 consecutive rows of
// one list with eight contiguous 512-byte loads straight into registers, no
// gather, no shared-memory staging), applies the test at d1 (dco.hpp:129), and
// hands only the survivors to the lane walk, which resumes them at the first A2
// segment with the carried prefix.  Sums and decisions are the same operations
// in the same order, so results are unchanged bit for bit.
// F32: the certified fp32 walk (scan_engine.cuh): lanes walk in fp32 with a proven
// error band; a test decides only outside the band, and the chunk's undecided and
// possibly-positive candidates are re-walked exactly in fp64 (one thread each, the
// reference's order) before the merge.  Decisions, dims and distances are the exact
// walk's.  Worth it where positives are rare among the candidates (config 5: ~0.1 %).
// Per-slot chunk state of the search kernel (see the layout there), in 8-byte words.
__host__ __device__ inline bool pend_in_wbuf(bool dense, bool f32, int cap, int nwarps) {
    return dense && f32 && 8 * cap + 1024 <= 4096 * nwarps;
}
__host__ __device__ inline int slot_bytes_before_surv(bool dense, bool f32, int cap, int nwarps) {
    const int pre_b = (f32 ? 4 : 8) * cap;
    const int pend_b = (f32 && !pend_in_wbuf(dense, f32, cap, nwarps)) ? 8 * cap : 0;
    return ((pre_b + 7) & ~7) + pend_b;
}
__host__ __device__ inline int slot_words(bool dense, bool f32, int cap, int nwarps, bool prewalk) {
    if (!dense) return prewalk ? 2 * cap : cap;
    return (slot_bytes_before_surv(dense, f32, cap, nwarps) + 2 * cap + 7) / 8;
}

// Register caps (same-box A/B, profiles/r02/ab_regs.log): the certified fp32 walk at 56
// (9 resident 4-warp CTAs per SM; 64 measured -2.5 % on config 5), the exact walk at 64
// (8 CTAs; +3 to +4 % on configs 2 and 3, where the fp64 chains need the registers).
template <int VEC, bool FULL, bool DENSE, bool F32, bool DEEP = false>
__global__ void __maxnreg__(F32 ? 56 : 64) ivf_search_kernel(SearchLaunch a, int chunk_cap) {
    static_assert(!DEEP || (VEC == 4 && !F32), "deep tail steps: 16-byte lines, exact walk");
    static_assert(!F32 || (VEC == 4 && FULL), "the fp32 walk runs on full 32-float lines");
    using acc_t = typename std::conditional<F32, float, double>::type;
    // the staged query as bank-conflict-free planes (scan_engine.cuh) where every lane read is
    // a full segment of the exact walk and no dense phase reads it as doubles
    // (long plans only, i.e. the DEEP instances: on config 2's 4 segments, whose rows never
    // collide, the extra unpacking measured -6 %)
    constexpr bool QP = kQueryPlanes && DEEP && FULL && !DENSE;
    extern __shared__ __align__(128) unsigned char smem_raw[];  // gather rows: 128-byte aligned (swizzle)
    __shared__ SearchShared sh;
    const int nwarps = blockDim.x >> 5;
    // dynamic layout (8-byte items first)
    float* wbuf_all = reinterpret_cast<float*>(smem_raw);
    double* qseg = reinterpret_cast<double*>(wbuf_all + nwarps * 1024);
    if (threadIdx.x == 0 && (__cvta_generic_to_shared(smem_raw) & 127u)) __trap();  // swizzle needs 128-B rows
    double* thr = qseg + a.nseg * kQPitch;
    double* tfac = thr + (a.ntest > 0 ? a.ntest : 1);
    double* topd = tfac + (a.ntest > 0 ? a.ntest : 1);
    // Per-slot chunk state (slot_words, shared with search_smem).  Lane walk alone: 2 x
    // chunk_cap untested-prefix sums, by chunk parity, when the plan has an untested prefix
    // to pre-walk (a.nseg0 > 0), else one chunk_cap buffer; a chunk's positives' distances
    // reuse its own prefix half (pend_d = pre_cur): a slot's prefix is consumed when the
    // slot is claimed, before it can turn positive.  DENSE: the survivors' prefixes
    // (acc_t; the exact walk's double prefix doubles as pend_d) and the survivor list
    // (16-bit slots); the fp32 walk's pend_d lives in the gather lines past warp 0's
    // first kilobyte (idle once the lane walk ends: positives come only from the exact
    // re-walk) when they hold it.
    double* pre_s = topd + a.K;
    acc_t* dpre = reinterpret_cast<acc_t*>(pre_s);
    const bool pend_wbuf = pend_in_wbuf(DENSE, F32, chunk_cap, nwarps);
    const int pre_b = static_cast<int>(sizeof(acc_t)) * chunk_cap;
    double* dpend = !F32 ? pre_s
                         : (pend_wbuf ? reinterpret_cast<double*>(wbuf_all + 256)
                                      : reinterpret_cast<double*>(reinterpret_cast<char*>(pre_s) + ((pre_b + 7) & ~7)));
    uint16_t* surv = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(pre_s) +
                                                 slot_bytes_before_surv(DENSE, F32, chunk_cap, nwarps));
    const bool prewalk = a.nseg0 > 0;
    int32_t* lstart = reinterpret_cast<int32_t*>(pre_s + slot_words(DENSE, F32, chunk_cap, nwarps, prewalk));
    int32_t* cpos = lstart + a.nprobe;
    Seg* segs = reinterpret_cast<Seg*>(cpos + chunk_cap + ((chunk_cap + a.nprobe) & 1));
    int32_t* topi = reinterpret_cast<int32_t*>(segs + a.nseg);
    int32_t* pre = topi + a.K;
    // positives' ids reuse the slot -> position map (read only at the slot's claim)
    int32_t* pend_i = cpos;
    // CTA-merge compaction counts: warp 0's gather line (idle at a chunk end)
    int* wc = reinterpret_cast<int*>(wbuf_all);
    unsigned* pflag = reinterpret_cast<unsigned*>(pre + a.nprobe + 1);
    // F32: undecided slots of the chunk; the query staged as fp32 and the per-test band
    // factors share qseg's slot
    unsigned* vflag = pflag + ((chunk_cap + 31) >> 5);
    float* qsegf = reinterpret_cast<float*>(qseg);
    double2* gband = reinterpret_cast<double2*>(qsegf + a.nseg * kQPitchF);
    // F32: per-test fp32 decision thresholds (rebuilt with thr): s32 > rej32[t] is a
    // certain rejection, s32 <= pas32[t] a certain pass (directed roundings, f32_cuts)
    float* rej32 = reinterpret_cast<float*>(gband + (a.ntest > 0 ? a.ntest : 1));
    float* pas32 = rej32 + (a.ntest > 0 ? a.ntest : 1);
    const double2 band_d = F32 ? f32_band(a.D) : make_double2(0.0, 0.0);
    const double nabs = (a.D + 2) * 0x1p-148;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    float* wbuf = wbuf_all + warp * 1024;
    for (int i = threadIdx.x; i < a.nseg; i += blockDim.x) {
        const Seg sg = a.segs[i];
        segs[i] = sg;
        if (F32 && sg.test >= 0) gband[sg.test] = f32_band(sg.col + sg.len);
    }
    for (int i = threadIdx.x; i < a.ntest; i += blockDim.x) tfac[i] = a.tfac[i];
    // VEC=4 line descriptor = pos * stride + column offset, 16-byte units from a.a1
    const uint32_t str1 = static_cast<uint32_t>(a.d1) >> 2, str2 = static_cast<uint32_t>(a.D - a.d1) >> 2;
    const uint32_t a2c = a.a2_16 - (static_cast<uint32_t>(a.d1) >> 2);
    const char* gbase = lane_base16(a.a1);
    const GatherDst gdst = F32 ? gather_dst(wbuf) : GatherDst{0u, 0u};
    // stream index -> flat position (last probed list with pre[l] <= i)
    const int nl = a.nprobe - a.probe_lo;  // lists scanned per query
    auto locate = [&](int i) {
        int l = 0, h = nl - 1;
        while (l < h) {
            const int mid = (l + h + 1) >> 1;
            if (pre[mid] <= i) l = mid;
            else h = mid - 1;
        }
        return lstart[l] + (i - pre[l]);
    };
    // leading segments no threshold test depends on (the split layouts' A1 prefix and FD's
    // whole walk but the last segment are tested against nothing, ivf.cpp:366-386): lanes
    // left idle at a chunk's tail precompute them for the next chunk
    const int nseg0 = a.nseg0;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int w = static_cast<int>(atomicAdd(a.counter, 1ull));
            sh.stop = w >= a.nq;
            sh.q = sh.stop ? w : (a.order ? a.order[w] : w);
            sh.cnt = 0;
            // the radius starts at the caller's bound (the sharded search's second
            // wave) or +inf; thresholds follow it until the heap is full
            const double r0 = (!sh.stop && a.r0) ? a.r0[sh.q] : kInf;
            sh.r = r0;
            sh.r_sq = __dmul_rn(r0, r0);
            sh.dims = 0;
        }
        __syncthreads();
        if (sh.stop) break;
        const int qi = sh.q;
        if constexpr (F32) stage_query_f32(qsegf, segs, a.nseg, a.Q + static_cast<int64_t>(qi) * a.D);
        else if constexpr (QP) stage_query_planes(qseg, segs, a.nseg, a.Q + static_cast<int64_t>(qi) * a.D);
        else stage_query(qseg, segs, a.nseg, a.Q + static_cast<int64_t>(qi) * a.D);
        for (int i = threadIdx.x; i < a.ntest; i += blockDim.x) {
            thr[i] = __dmul_rn(tfac[i], sh.r_sq);
            if constexpr (F32) f32_cuts(thr[i], gband[i], nabs, rej32[i], pas32[i]);
        }
        if (warp == 0) {  // probed lists -> stream prefix offsets
            int carry = 0;
            for (int base = 0; base < nl; base += 32) {  // probe ranks probe_lo .. nprobe-1
                const int i = base + static_cast<int>(lane);
                int len = 0;
                if (i < nl) {
                    const int p = a.probes[static_cast<int64_t>(qi) * a.nprobe + a.probe_lo + i];
                    const int64_t s0 = a.list_off[p];
                    lstart[i] = static_cast<int32_t>(s0);
                    len = static_cast<int>(a.list_off[p + 1] - s0);
                }
                int incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(kFull, incl, o);
                    if (static_cast<int>(lane) >= o) incl += v;
                }
                if (i < nl) pre[i + 1] = carry + incl;
                carry += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0) {
                pre[0] = 0;
                sh.total = carry;
            }
        }
        __syncthreads();
        const int total = sh.total;
        unsigned long long my_dims = 0;

        if (threadIdx.x == 0) sh.pcount[0] = 0;
        for (int lo = 0, j = 0; lo < total; ++j) {
            const int64_t span = lo == 0 ? a.first : a.step;
            const int hi = static_cast<int>(lo + span < total ? lo + span : total);
            const int nhi = static_cast<int>(hi + a.step < total ? hi + a.step : total);  // next chunk [hi, nhi)
            double* pre_cur = pre_s + (prewalk ? (j & 1) * chunk_cap : 0);  // lane walk alone (!DENSE)
            double* pend_d = DENSE ? dpend : pre_cur;
            double* pre_nxt = pre_s + ((j & 1) ^ 1) * chunk_cap;
            // F32 with no finite radius yet (r = +inf before K results): every candidate
            // would reach d == D undecided, so the chunk goes straight to the exact re-walk
            const bool open = F32 && !(sh.r_sq < kInf);
            // slot -> flat position.  The dense prefix phase writes it for the rows it visits
            // (every row of the chunk), so only the lane walks need this pass.
            if (!DENSE || open) {  // each thread maps a contiguous run of slots with one search
                const int n = hi - lo, per = (n + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
                const int s0 = static_cast<int>(threadIdx.x) * per, s1 = min(n, s0 + per);
                if (s0 < s1) {
                    int l = 0, h = nl - 1;
                    while (l < h) {
                        const int mid = (l + h + 1) >> 1;
                        if (pre[mid] <= lo + s0) l = mid;
                        else h = mid - 1;
                    }
                    for (int sl = s0; sl < s1; ++sl) {
                        while (pre[l + 1] <= lo + sl) ++l;
                        cpos[sl] = lstart[l] + (lo + sl - pre[l]);
                    }
                }
            }
            if (threadIdx.x == 0) {
                sh.next = DENSE ? 0 : (open ? hi : lo);
                sh.pnext = 0;
                sh.nsurv = 0;
            }
            for (int w = threadIdx.x; w < (hi - lo + 31) / 32; w += blockDim.x) {
                pflag[w] = 0;
                if constexpr (F32) {
                    const int rem = hi - lo - w * 32;
                    vflag[w] = open ? (rem >= 32 ? ~0u : (1u << rem) - 1u) : 0u;
                }
            }
            __syncthreads();
            const double r = sh.r, r_sq = sh.r_sq;
            const int pc = (DENSE || F32) ? 0 : sh.pcount[j & 1];  // [lo, lo + pc) carry their prefix in pre_cur
            const bool can_pre = !DENSE && !F32 && nseg0 > 0 && nhi > hi;
            // F32 final test: certainly negative above rfin (kFd: sqrt(s) > r is certain once
            // s > r_sq (1 + 2^-47))
            const double rfin = a.final_fd ? __dmul_rn(r_sq, 1.0 + 0x1p-47) : r_sq;
            float fin32 = 0.f, unused32 = 0.f;  // s32 > fin32: certainly negative at d = D
            if constexpr (F32) f32_cuts(rfin, band_d, nabs, fin32, unused32);
            if (DENSE && !open) {
                // tasks = (probed list, 32-row position group) pairs covering the chunk
                // probed lists holding the chunk's first and last rows (last l with
                // pre[l] <= i; pre is non-decreasing): one ballot per 32 lists
                int l0 = -1, l1 = -1;
                for (int b = 0; b < nl; b += 32) {
                    const int i = b + static_cast<int>(lane);
                    const int pv = i < nl ? pre[i] : INT_MAX;
                    l0 += __popc(__ballot_sync(kFull, pv <= lo));
                    l1 += __popc(__ballot_sync(kFull, pv <= hi - 1));
                }
                const double t1 = thr[segs[0].test];
                const double2* q2 = reinterpret_cast<const double2*>(qseg);
                // tasks = (probed list, 32-row position group) pairs in order, dealt round
                // robin to the warps; off = this warp's first task within the next list
                int off = warp;
                for (int l = l0; l <= l1; ++l) {
                    const int as = max(lo, pre[l]), bs = min(hi, pre[l + 1]);
                    if (as >= bs) continue;
                    const int pa = lstart[l] + (as - pre[l]), pb = pa + (bs - as);
                    const int g0 = pa >> 5, g1 = (pb - 1) >> 5;
                    int g = g0 + off;
                    for (; g <= g1; g += nwarps) {
                        const int p = (g << 5) + static_cast<int>(lane);
                        const bool act = p >= pa && p < pb;
                        if (act) cpos[as - lo + (p - pa)] = p;  // the lane walk / exact re-walk read it
                        const float4* src = reinterpret_cast<const float4*>(a.a1i) + static_cast<int64_t>(g) * 256 + lane;
                        acc_t sa = 0.0;
#pragma unroll
                        for (int h = 0; h < DENSE_PARTS; ++h) {
                            constexpr int PC = 8 / DENSE_PARTS;
                            float4 v[PC];
#pragma unroll
                            for (int c = 0; c < PC; ++c)
                                v[c] = act ? __ldg(src + (h * PC + c) * 32) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                            for (int c = 0; c < PC; ++c) {
                                if constexpr (F32) {  // the certified fp32 walk's arithmetic
                                    const float4 qf = reinterpret_cast<const float4*>(qsegf)[h * PC + c];
                                    float df = __fsub_rn(v[c].x, qf.x);
                                    sa = __fmaf_rn(df, df, sa);
                                    df = __fsub_rn(v[c].y, qf.y);
                                    sa = __fmaf_rn(df, df, sa);
                                    df = __fsub_rn(v[c].z, qf.z);
                                    sa = __fmaf_rn(df, df, sa);
                                    df = __fsub_rn(v[c].w, qf.w);
                                    sa = __fmaf_rn(df, df, sa);
                                } else {
                                    const double2 qa = q2[(h * PC + c) * 2], qb = q2[(h * PC + c) * 2 + 1];
                                    sa = sq_diff_acc(sa, v[c].x, qa.x);
                                    sa = sq_diff_acc(sa, v[c].y, qa.y);
                                    sa = sq_diff_acc(sa, v[c].z, qb.x);
                                    sa = sq_diff_acc(sa, v[c].w, qb.y);
                                }
                            }
                        }
                        bool keep, drop;
                        if constexpr (F32) {  // band decision at d1; undecided -> the exact re-walk
                            drop = act && sa > rej32[segs[0].test];
                            keep = act && !drop && sa <= pas32[segs[0].test];
                            if (act && !drop && !keep) {
                                const int slot = as - lo + (p - pa);
                                atomicOr(&vflag[slot >> 5], 1u << (slot & 31));
                            }
                        } else {
                            keep = act && !(sa > t1);  // reject iff s > thr at d1 (dco.hpp:129)
                            drop = act && !keep;
                        }
                        if (drop) my_dims += static_cast<unsigned long long>(segs[0].len);
                        const unsigned kb = __ballot_sync(kFull, keep);
                        int base = 0;
                        if (lane == 0 && kb) base = atomicAdd(&sh.nsurv, __popc(kb));
                        base = __shfl_sync(kFull, base, 0);
                        if (keep) {
                            const int slot = as - lo + (p - pa);
                            dpre[slot] = sa;
                            surv[base + __popc(kb & ((1u << lane) - 1u))] = static_cast<uint16_t>(slot);
                        }
                    }
                    off = g - g1 - 1;
                }
                __syncthreads();
            }
            const int nsurv = DENSE ? sh.nsurv : 0;

            int cand = -1, seg = 0, pos = 0;
            bool prew = false;  // lane holds a next-chunk candidate's untested prefix
            acc_t s = 0.0;
            for (;;) {
                unsigned need = __ballot_sync(kFull, cand < 0);
                if (need) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&sh.next, __popc(need));
                    base = __shfl_sync(kFull, base, 0);
                    if (cand < 0) {
                        const int i = base + __popc(need & ((1u << lane) - 1u));
                        if constexpr (DENSE) {  // survivors of the prefix test, resumed at A2
                            if (i < nsurv) {
                                const int slot = surv[i];
                                cand = lo + slot;
                                pos = cpos[slot];
                                prew = false;
                                seg = 1;
                                s = dpre[slot];
                            }
                        } else if (i < hi) {
                            cand = i;
                            pos = cpos[i - lo];
                            prew = false;
                            if (i - lo < pc) {
                                seg = nseg0;
                                s = static_cast<acc_t>(pre_cur[i - lo]);
                            } else {
                                seg = 0;
                                s = 0.0;
                            }
                        }
                    }
                    if (can_pre) {
                        need = __ballot_sync(kFull, cand < 0);
                        if (need) {
                            int pb = 0;
                            if (lane == 0) pb = atomicAdd(&sh.pnext, __popc(need));
                            pb = __shfl_sync(kFull, pb, 0);
                            if (cand < 0) {
                                const int rel = pb + __popc(need & ((1u << lane) - 1u));
                                if (rel < nhi - hi) {
                                    cand = rel;
                                    pos = locate(hi + rel);
                                    prew = true;
                                    seg = 0;
                                    s = 0.0;
                                }
                            }
                        }
                    }
                }
                if constexpr (!DEEP) {
                    if (!__any_sync(kFull, cand >= 0)) break;
                } else {
                    // (a ballot every step measured 1 % ahead of gating this on the stream's end)
                    const unsigned livem = __ballot_sync(kFull, cand >= 0);
                    if (!livem) break;
                    // Deep tail step.  With <= 16 live candidates in the warp (a chunk's tail,
                    // or its first K candidates) the free rows of the gather buffer carry the
                    // live candidates' NEXT segments: candidate of rank r owns rows r*k .. r*k+k-1
                    // (k = 2, or 4 at <= 8 live) and its lane walks them in order, testing after each as
                    // always, so sums, decisions and dims are unchanged; a row fetched past a
                    // rejection is the only cost.  The tail is latency-bound (a step is one DRAM
                    // round trip whatever the lane count), so it ends k times sooner.
                    const int nlive = __popc(livem);
                    if (nlive <= kDeepTail) {
                        // rows per candidate: 2, 4 ... (1 << kDeepShift) as the live count halves
                        int ks = 1;
#pragma unroll
                        for (int t = 2; t <= kDeepShift; ++t) ks += nlive <= (32 >> t) ? 1 : 0;
                        const int rnk = static_cast<int>(lane) >> ks, off = static_cast<int>(lane) & ((1 << ks) - 1);
                        const unsigned srcl = __fns(livem, 0, rnk + 1) & 31u;
                        const int ppos = __shfl_sync(kFull, pos, srcl), pseg = __shfl_sync(kFull, seg, srcl);
                        const int rseg = pseg + off;
                        uint32_t dsc = kNoLine;
                        int nch = 0;
                        if (rnk < nlive && rseg < a.nseg) {
                            const Seg g = segs[rseg];
                            dsc = g.arr == 0 ? static_cast<uint32_t>(ppos) * str1 + (g.col >> 2)
                                             : static_cast<uint32_t>(ppos) * str2 + a2c + (g.col >> 2);
                            nch = g.len >> 2;
                        }
                        gather_issue16<FULL>(wbuf, gbase, dsc, nch);
                        cp_async_wait_group<0>();
                        __syncwarp();
                        if (cand >= 0) {
                            const unsigned row0 = static_cast<unsigned>(__popc(livem & ((1u << lane) - 1u))) << ks;
                            for (int m = 0; m < (1 << ks); ++m) {
                                const Seg sg = segs[seg];
                                if constexpr (QP) s = accumulate_planes(wbuf, row0 + m, qseg, a.nseg, seg, s);
                                else s = accumulate_row<FULL>(wbuf, row0 + m, qseg + seg * kQPitch, sg.len, s);
                                if (sg.test >= 0 && s > thr[sg.test]) {  // reject (dco.hpp:141)
                                    my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                                    cand = -1;
                                    break;
                                }
                                if (seg == a.nseg - 1) {  // d == D (dco.hpp:145; ivf.cpp:335-338)
                                    my_dims += static_cast<unsigned long long>(a.D);
                                    const bool positive = a.final_fd ? __dsqrt_rn(s) <= r : s <= r_sq;
                                    if (positive) {
                                        const int slot = cand - lo;
                                        pend_d[slot] = __dsqrt_rn(s);
                                        pend_i[slot] = a.ids[pos];
                                        atomicOr(&pflag[slot >> 5], 1u << (slot & 31));
                                    }
                                    cand = -1;
                                    break;
                                }
                                ++seg;
                            }
                        }
                        __syncwarp();
                        continue;
                    }
                }
                const Seg sg = segs[seg];
                if constexpr (VEC == 4) {
                    uint32_t dsc = kNoLine;
                    if (cand >= 0)
                        dsc = sg.arr == 0 ? static_cast<uint32_t>(pos) * str1 + (sg.col >> 2)
                                          : static_cast<uint32_t>(pos) * str2 + a2c + (sg.col >> 2);
                    if constexpr (F32) gather_issue16<FULL>(gdst, gbase, dsc, sg.len >> 2);
                    else gather_issue16<FULL>(wbuf, gbase, dsc, sg.len >> 2);
                } else {
                    const float* src = sg.arr == 0 ? a.a1 + static_cast<int64_t>(pos) * a.d1 + sg.col
                                                   : a.a2 + static_cast<int64_t>(pos) * (a.D - a.d1) + (sg.col - a.d1);
                    gather_issue4(wbuf, src, cand >= 0 ? sg.len : 0);
                }
                cp_async_wait_group<0>();
                __syncwarp();
                if (cand >= 0) {
                    if constexpr (F32) s = accumulate_line_f32(wbuf, qsegf + seg * kQPitchF, s);
                    else if constexpr (QP) s = accumulate_planes(wbuf, lane, qseg, a.nseg, seg, s);
                    else s = accumulate_line<VEC, FULL>(wbuf, qseg + seg * kQPitch, sg.len, s);
                    if constexpr (F32) {
                        // decide only what the band proves; the rest is re-walked exactly
                        int verdict = 0;  // 1 reject, 2 undecided, 3 certainly negative at D
                        if (sg.test >= 0) {
                            if (s > rej32[sg.test]) verdict = 1;
                            else if (!(s <= pas32[sg.test])) verdict = 2;
                        }
                        if (verdict == 0 && seg == a.nseg - 1) verdict = s > fin32 ? 3 : 2;
                        if (verdict == 1) {
                            my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                            cand = -1;
                        } else if (verdict == 3) {
                            my_dims += static_cast<unsigned long long>(a.D);
                            cand = -1;
                        } else if (verdict == 2) {
                            const int slot = cand - lo;
                            atomicOr(&vflag[slot >> 5], 1u << (slot & 31));
                            cand = -1;
                        } else {
                            ++seg;
                        }
                    } else if (prew) {
                        if (seg + 1 == nseg0) {
                            pre_nxt[cand] = s;
                            cand = -1;
                        } else {
                            ++seg;
                        }
                    } else if (sg.test >= 0 && s > thr[sg.test]) {  // reject (dco.hpp:141)
                        my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                        cand = -1;
                    } else if (seg == a.nseg - 1) {  // d == D (dco.hpp:145; ivf.cpp:335-338)
                        my_dims += static_cast<unsigned long long>(a.D);
                        // kFd decides on dist <= r (ivf.cpp:337), the scans on s <= r^2
                        // (dco.hpp:145); the root is taken only where it is needed
                        const bool positive = a.final_fd ? __dsqrt_rn(s) <= r : s <= r_sq;
                        if (positive) {
                            const int slot = cand - lo;
                            pend_d[slot] = __dsqrt_rn(s);
                            pend_i[slot] = a.ids[pos];
                            atomicOr(&pflag[slot >> 5], 1u << (slot & 31));
                        }
                        cand = -1;
                    } else {
                        ++seg;
                    }
                }
            }
            __syncthreads();
            if constexpr (F32) {
                // exact re-walk of the undecided slots, one thread each, in the reference's
                // order and arithmetic (dco.hpp:130-150; split resume at d1, ivf.cpp:389-400)
                const int nw = (hi - lo + 31) >> 5;
                int nv = 0;
                nv = flag_count(vflag, nw);
                for (int k = threadIdx.x; k < nv; k += blockDim.x) {
                    int w = 0, c = k;
                    for (;; ++w) {
                        const int pcnt = __popc(vflag[w]);
                        if (c < pcnt) break;
                        c -= pcnt;
                    }
                    unsigned bits = vflag[w];
                    for (; c > 0; --c) bits &= bits - 1;
                    const int slot = w * 32 + __ffs(bits) - 1;
                    const int64_t pos = cpos[slot];
                    double se = 0.0;
                    for (int g = 0; g < a.nseg; ++g) {
                        const Seg sg = segs[g];
                        const float* src = sg.arr == 0 ? a.a1 + pos * a.d1 + sg.col
                                                       : a.a2 + pos * (a.D - a.d1) + (sg.col - a.d1);
                        const float* qq = qsegf + g * kQPitchF;
#pragma unroll
                        for (int c4 = 0; c4 < 8; ++c4) {
                            const float4 v = __ldg(reinterpret_cast<const float4*>(src) + c4);
                            const float4 qv = *reinterpret_cast<const float4*>(qq + c4 * 4);
                            se = sq_diff_acc(se, v.x, static_cast<double>(qv.x));
                            se = sq_diff_acc(se, v.y, static_cast<double>(qv.y));
                            se = sq_diff_acc(se, v.z, static_cast<double>(qv.z));
                            se = sq_diff_acc(se, v.w, static_cast<double>(qv.w));
                        }
                        if (sg.test >= 0 && se > thr[sg.test]) {  // dco.hpp:141
                            my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                            break;
                        }
                        if (g == a.nseg - 1) {  // dco.hpp:145; ivf.cpp:335-338
                            my_dims += static_cast<unsigned long long>(a.D);
                            const double dist = __dsqrt_rn(se);
                            if (a.final_fd ? dist <= r : se <= r_sq) {
                                pend_d[slot] = dist;
                                pend_i[slot] = a.ids[pos];
                                atomicOr(&pflag[slot >> 5], 1u << (slot & 31));
                            }
                        }
                    }
                }
                __syncthreads();
            }
            // offer the chunk's positives in candidate order: few -> one warp,
            // many -> the whole CTA, ties or oversize -> one by one
            const int n = hi - lo;
            int npos = 0;
            npos = flag_count(pflag, (n + 31) >> 5);
            int seq = -1;  // >= 0: offer pend[0, seq) sequentially (compacted batch)
            if (npos > 32 && n <= 2 * static_cast<int>(blockDim.x) && sh.cnt <= 2 * static_cast<int>(blockDim.x)) {
                const int rc = cta_merge_chunk(topd, topi, sh, a.K, pend_d, pend_i, pflag, n, wc);
                if (rc < 0) seq = -rc - 1;
                npos = 0;
            }
            if (warp == 0) {
                bool merged = npos == 0;
                if (!merged && npos <= 32) merged = warp_merge_chunk(topd, topi, sh, a.K, pend_d, pend_i, pflag, n);
                for (int k = 0; k < seq; ++k) warp_offer(topd, topi, &sh.cnt, a.K, pend_d[k], pend_i[k]);
                const int nw = merged ? 0 : (n + 31) / 32;
                for (int w = 0; w < nw; ++w) {
                    unsigned bits = pflag[w];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int slot = w * 32 + b;
                        warp_offer(topd, topi, &sh.cnt, a.K, pend_d[slot], pend_i[slot]);
                    }
                }
                if (sh.cnt == a.K) {  // ivf.cpp:268-270; dco.hpp:125
                    const double rn = topd[a.K - 1];
                    const double rsq = __dmul_rn(rn, rn);
                    for (int i = static_cast<int>(lane); i < a.ntest; i += 32) {
                        thr[i] = __dmul_rn(tfac[i], rsq);
                        if constexpr (F32) f32_cuts(thr[i], gband[i], nabs, rej32[i], pas32[i]);
                    }
                    if (lane == 0) {
                        sh.r = rn;
                        sh.r_sq = rsq;
                    }
                }
                if (lane == 0) sh.pcount[(j & 1) ^ 1] = can_pre ? min(sh.pnext, nhi - hi) : 0;
            }
            __syncthreads();
            lo = hi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_dims += __shfl_xor_sync(kFull, my_dims, o);
        if (lane == 0) atomicAdd(&sh.dims, my_dims);
        __syncthreads();
        const int cnt = sh.cnt;
        for (int i = threadIdx.x; i < a.K; i += blockDim.x) {
            const int64_t o = static_cast<int64_t>(qi) * a.K + i;
            a.out_ids[o] = i < cnt ? topi[i] : -1;
            a.out_dists[o] = i < cnt ? topd[i] : __longlong_as_double(0x7ff8000000000000ll);
        }
        if (threadIdx.x == 0) {
            a.out_cnt[qi] = cnt;
            a.out_dims[qi] = sh.dims;
            if (a.out_cand) a.out_cand[qi] = static_cast<unsigned long long>(total);
        }
    }
}

// ---------------------------------------------------------------------------------------
// Overlapped chunks (opts.lag = 1; exact walk on 16-byte lines, no dense phase, no pre-walk).
//
// In ivf_search_kernel a chunk ends with a barrier (merge + threshold refresh), so its lanes
// run dry one by one while the last long walks finish: with 30-segment walks about a quarter
// of all lane steps are idle (config 3: 25 of 32 lanes live per instruction, against 32 for
// FDScanning on the same engine, which is the whole gap between the two).  Here lanes that
// find chunk w's stream exhausted claim candidates of chunk w + 1 at once.  For the result
// to be a function of the schedule alone, ALL of chunk c (>= 2) is tested against the
// thresholds after the merge of chunk c - 2 (the lag-1 schedule; chunk 1 waits for chunk 0,
// whose r = +inf would otherwise send a whole extra chunk to d = D).  The merge stays
// synchronous and in chunk order: window w ends when every candidate of chunk w has retired
// (each warp reports once that the stream is exhausted and it holds none); candidates of
// chunk w + 1 in flight stay in their lanes' registers across the barrier and carry on in
// window w + 1.  Chunk state (slot -> position / id, positives' distances, flags), the
// thresholds and r exist twice, by chunk parity.  The oracle replays the schedule
// (orc_ivf_query_lag, lag = 2), so results are bit-exact against it.
struct LagShared {
    int nextp[2];    // claim pointers of the two chunks in flight, by parity
    unsigned quiet;  // warps that hold no candidate of the window's chunk any more
    double r[2], r_sq[2];
};

template <bool FULL, bool PLANES>
__global__ void __maxnreg__(64) ivf_search_lag_kernel(SearchLaunch a, int chunk_cap) {
    static_assert(!PLANES || FULL, "query planes hold full 32-float segments");
    constexpr bool QP = PLANES;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ SearchShared sh;
    __shared__ LagShared lg;
    const int nwarps = blockDim.x >> 5;
    const int nt = a.ntest > 0 ? a.ntest : 1;
    const int pw32 = (chunk_cap + 31) >> 5;
    float* wbuf_all = reinterpret_cast<float*>(smem_raw);
    double* qseg = reinterpret_cast<double*>(wbuf_all + nwarps * 1024);
    double* thr2 = qseg + a.nseg * kQPitch;  // [2][nt]
    double* tfac = thr2 + 2 * nt;
    double* topd = tfac + nt;
    double* pend2 = topd + a.K;  // [2][chunk_cap] positives' distances
    int32_t* lstart = reinterpret_cast<int32_t*>(pend2 + 2 * chunk_cap);
    int32_t* cpos2 = lstart + a.nprobe;  // [2][chunk_cap] slot -> position, then the positive's id
    Seg* segs = reinterpret_cast<Seg*>(cpos2 + 2 * chunk_cap + (a.nprobe & 1));
    int32_t* topi = reinterpret_cast<int32_t*>(segs + a.nseg);
    int32_t* pre = topi + a.K;
    unsigned* pflag2 = reinterpret_cast<unsigned*>(pre + a.nprobe + 1);  // [2][pw32]
    int* wc = reinterpret_cast<int*>(wbuf_all);
    if (threadIdx.x == 0 && (__cvta_generic_to_shared(smem_raw) & 127u)) __trap();

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const unsigned allw = nwarps >= 32 ? ~0u : (1u << nwarps) - 1u;
    float* wbuf = wbuf_all + warp * 1024;
    for (int i = threadIdx.x; i < a.nseg; i += blockDim.x) segs[i] = a.segs[i];
    for (int i = threadIdx.x; i < a.ntest; i += blockDim.x) tfac[i] = a.tfac[i];
    const uint32_t str1 = static_cast<uint32_t>(a.d1) >> 2, str2 = static_cast<uint32_t>(a.D - a.d1) >> 2;
    const uint32_t a2c = a.a2_16 - (static_cast<uint32_t>(a.d1) >> 2);
    const char* gbase = lane_base16(a.a1);
    const int nl = a.nprobe - a.probe_lo;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int w = static_cast<int>(atomicAdd(a.counter, 1ull));
            sh.stop = w >= a.nq;
            sh.q = sh.stop ? w : (a.order ? a.order[w] : w);
            sh.cnt = 0;
            const double r0 = (!sh.stop && a.r0) ? a.r0[sh.q] : kInf;
            sh.r = r0;
            sh.r_sq = __dmul_rn(r0, r0);
            lg.r[0] = lg.r[1] = r0;
            lg.r_sq[0] = lg.r_sq[1] = sh.r_sq;
            sh.dims = 0;
        }
        __syncthreads();
        if (sh.stop) break;
        const int qi = sh.q;
        if constexpr (QP) stage_query_planes(qseg, segs, a.nseg, a.Q + static_cast<int64_t>(qi) * a.D);
        else stage_query(qseg, segs, a.nseg, a.Q + static_cast<int64_t>(qi) * a.D);
        for (int i = threadIdx.x; i < a.ntest; i += blockDim.x) {
            const double t = __dmul_rn(tfac[i], sh.r_sq);
            thr2[i] = t;
            thr2[nt + i] = t;
        }
        if (warp == 0) {  // probed lists -> stream prefix offsets
            int carry = 0;
            for (int base = 0; base < nl; base += 32) {
                const int i = base + static_cast<int>(lane);
                int len = 0;
                if (i < nl) {
                    const int p = a.probes[static_cast<int64_t>(qi) * a.nprobe + a.probe_lo + i];
                    const int64_t s0 = a.list_off[p];
                    lstart[i] = static_cast<int32_t>(s0);
                    len = static_cast<int>(a.list_off[p + 1] - s0);
                }
                int incl = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(kFull, incl, o);
                    if (static_cast<int>(lane) >= o) incl += v;
                }
                if (i < nl) pre[i + 1] = carry + incl;
                carry += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0) {
                pre[0] = 0;
                sh.total = carry;
            }
        }
        __syncthreads();
        const int total = sh.total;
        unsigned long long my_dims = 0;
        // chunk c = [clo(c), clo(c + 1)): first, then step candidates each
        auto clo = [&](int c) -> int {
            if (c <= 0) return 0;
            const int64_t v = a.first + static_cast<int64_t>(c - 1) * a.step;
            return static_cast<int>(v < total ? v : total);
        };
        const int nchunks = total <= 0 ? 0
                                       : 1 + (total > a.first ? static_cast<int>((total - a.first + a.step - 1) / a.step) : 0);
        // slot -> flat position of chunk c into its parity's map; flags cleared
        auto map_chunk = [&](int c) {
            const int lo = clo(c), n = clo(c + 1) - lo;
            int32_t* cp = cpos2 + (c & 1) * chunk_cap;
            const int per = (n + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
            const int s0 = static_cast<int>(threadIdx.x) * per, s1 = min(n, s0 + per);
            if (s0 < s1) {
                int l = 0, h = nl - 1;
                while (l < h) {
                    const int mid = (l + h + 1) >> 1;
                    if (pre[mid] <= lo + s0) l = mid;
                    else h = mid - 1;
                }
                for (int sl = s0; sl < s1; ++sl) {
                    while (pre[l + 1] <= lo + sl) ++l;
                    cp[sl] = lstart[l] + (lo + sl - pre[l]);
                }
            }
            for (int w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) pflag2[(c & 1) * pw32 + w] = 0;
        };
        if (nchunks > 0) map_chunk(0);
        if (threadIdx.x == 0) lg.nextp[0] = 0;

        // lane state: cand = slot | parity << 30 (or -1); lives across windows
        int cand = -1, seg = 0, pos = 0;
        double s = 0.0;
        for (int w = 0; w < nchunks; ++w) {
            const int pw = w & 1, pn = pw ^ 1;
            const int lo = clo(w), hi = clo(w + 1), nhi = clo(w + 2);
            const bool spill = w >= 1 && w + 1 < nchunks;  // chunk 1 waits for chunk 0's merge
            if (w + 1 < nchunks) map_chunk(w + 1);
            if (threadIdx.x == 0) {
                lg.nextp[pn] = hi;
                lg.quiet = 0;
            }
            __syncthreads();
            bool dry_cur = false, dry_nxt = !spill, quiet_me = false;  // warp-uniform
            for (;;) {
                if (*reinterpret_cast<volatile unsigned*>(&lg.quiet) == allw) break;
                unsigned need = __ballot_sync(kFull, cand < 0);
                if (need && !dry_cur) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&lg.nextp[pw], __popc(need));
                    base = __shfl_sync(kFull, base, 0);
                    dry_cur = base + __popc(need) > hi;
                    const int i = base + __popc(need & ((1u << lane) - 1u));
                    if (cand < 0 && i < hi) {
                        cand = (i - lo) | (pw << 30);
                        pos = cpos2[pw * chunk_cap + (i - lo)];
                        seg = 0;
                        s = 0.0;
                    }
                    need = __ballot_sync(kFull, cand < 0);
                }
                if (need && !dry_nxt) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(&lg.nextp[pn], __popc(need));
                    base = __shfl_sync(kFull, base, 0);
                    dry_nxt = base + __popc(need) > nhi;
                    const int i = base + __popc(need & ((1u << lane) - 1u));
                    if (cand < 0 && i < nhi) {
                        cand = (i - hi) | (pn << 30);
                        pos = cpos2[pn * chunk_cap + (i - hi)];
                        seg = 0;
                        s = 0.0;
                    }
                }
                if (dry_cur && !quiet_me) {
                    if (!__any_sync(kFull, cand >= 0 && (cand >> 30) == pw)) {
                        quiet_me = true;
                        __threadfence_block();  // this warp's positives of chunk w are written
                        if (lane == 0) atomicOr(&lg.quiet, 1u << warp);
                    }
                }
                const unsigned livem = __ballot_sync(kFull, cand >= 0);
                if (!livem) {
                    if (quiet_me && dry_nxt) break;  // nothing to carry, nothing left to claim
                    continue;
                }
                const int nlive = __popc(livem);
                const int par = cand >= 0 ? cand >> 30 : 0;
                if (nlive <= kDeepTail && a.nseg >= kDeepMinSeg) {  // deep tail step (ivf_search_kernel, DEEP)
                    int ks = 1;
#pragma unroll
                    for (int t = 2; t <= kDeepShift; ++t) ks += nlive <= (32 >> t) ? 1 : 0;
                    const int rnk = static_cast<int>(lane) >> ks, off = static_cast<int>(lane) & ((1 << ks) - 1);
                    const unsigned srcl = __fns(livem, 0, rnk + 1) & 31u;
                    const int ppos = __shfl_sync(kFull, pos, srcl), pseg = __shfl_sync(kFull, seg, srcl);
                    const int rseg = pseg + off;
                    uint32_t dsc = kNoLine;
                    int nch = 0;
                    if (rnk < nlive && rseg < a.nseg) {
                        const Seg g = segs[rseg];
                        dsc = g.arr == 0 ? static_cast<uint32_t>(ppos) * str1 + (g.col >> 2)
                                         : static_cast<uint32_t>(ppos) * str2 + a2c + (g.col >> 2);
                        nch = g.len >> 2;
                    }
                    gather_issue16<FULL>(wbuf, gbase, dsc, nch);
                    cp_async_wait_group<0>();
                    __syncwarp();
                    if (cand >= 0) {
                        const unsigned row0 = static_cast<unsigned>(__popc(livem & ((1u << lane) - 1u))) << ks;
                        const double* thr = thr2 + par * nt;
                        for (int m = 0; m < (1 << ks); ++m) {
                            const Seg sg = segs[seg];
                            if constexpr (QP) s = accumulate_planes(wbuf, row0 + m, qseg, a.nseg, seg, s);
                            else s = accumulate_row<FULL>(wbuf, row0 + m, qseg + seg * kQPitch, sg.len, s);
                            if (sg.test >= 0 && s > thr[sg.test]) {  // reject (dco.hpp:141)
                                my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                                cand = -1;
                                break;
                            }
                            if (seg == a.nseg - 1) {  // d == D (dco.hpp:145; ivf.cpp:335-338)
                                my_dims += static_cast<unsigned long long>(a.D);
                                const bool positive = a.final_fd ? __dsqrt_rn(s) <= lg.r[par] : s <= lg.r_sq[par];
                                if (positive) {
                                    const int slot = cand & 0x3fffffff;
                                    pend2[par * chunk_cap + slot] = __dsqrt_rn(s);
                                    cpos2[par * chunk_cap + slot] = a.ids[pos];
                                    atomicOr(&pflag2[par * pw32 + (slot >> 5)], 1u << (slot & 31));
                                }
                                cand = -1;
                                break;
                            }
                            ++seg;
                        }
                    }
                    __syncwarp();
                    continue;
                }
                const Seg sg = segs[seg];
                uint32_t dsc = kNoLine;
                if (cand >= 0)
                    dsc = sg.arr == 0 ? static_cast<uint32_t>(pos) * str1 + (sg.col >> 2)
                                      : static_cast<uint32_t>(pos) * str2 + a2c + (sg.col >> 2);
                gather_issue16<FULL>(wbuf, gbase, dsc, sg.len >> 2);
                cp_async_wait_group<0>();
                __syncwarp();
                if (cand >= 0) {
                    if constexpr (QP) s = accumulate_planes(wbuf, lane, qseg, a.nseg, seg, s);
                    else s = accumulate_line<4, FULL>(wbuf, qseg + seg * kQPitch, sg.len, s);
                    if (sg.test >= 0 && s > thr2[par * nt + sg.test]) {  // reject (dco.hpp:141)
                        my_dims += static_cast<unsigned long long>(sg.col + sg.len);
                        cand = -1;
                    } else if (seg == a.nseg - 1) {  // d == D (dco.hpp:145; ivf.cpp:335-338)
                        my_dims += static_cast<unsigned long long>(a.D);
                        const bool positive = a.final_fd ? __dsqrt_rn(s) <= lg.r[par] : s <= lg.r_sq[par];
                        if (positive) {
                            const int slot = cand & 0x3fffffff;
                            pend2[par * chunk_cap + slot] = __dsqrt_rn(s);
                            cpos2[par * chunk_cap + slot] = a.ids[pos];
                            atomicOr(&pflag2[par * pw32 + (slot >> 5)], 1u << (slot & 31));
                        }
                        cand = -1;
                    } else {
                        ++seg;
                    }
                }
            }
            __syncthreads();
            // merge chunk w in candidate order (as ivf_search_kernel), then the thresholds of
            // chunk w + 2 (and of chunk 1 after chunk 0) into chunk w's parity
            double* pend_d = pend2 + pw * chunk_cap;
            int32_t* pend_i = cpos2 + pw * chunk_cap;
            const unsigned* pflag = pflag2 + pw * pw32;
            const int n = hi - lo;
            int npos = 0;
            npos = flag_count(pflag, (n + 31) >> 5);
            int seq = -1;
            if (npos > 32 && n <= 2 * static_cast<int>(blockDim.x) && sh.cnt <= 2 * static_cast<int>(blockDim.x)) {
                const int rc = cta_merge_chunk(topd, topi, sh, a.K, pend_d, pend_i, pflag, n, wc);
                if (rc < 0) seq = -rc - 1;
                npos = 0;
            }
            if (warp == 0) {
                bool merged = npos == 0;
                if (!merged && npos <= 32) merged = warp_merge_chunk(topd, topi, sh, a.K, pend_d, pend_i, pflag, n);
                for (int k = 0; k < seq; ++k) warp_offer(topd, topi, &sh.cnt, a.K, pend_d[k], pend_i[k]);
                const int nw = merged ? 0 : (n + 31) / 32;
                for (int k = 0; k < nw; ++k) {
                    unsigned bits = pflag[k];
                    while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int slot = k * 32 + b;
                        warp_offer(topd, topi, &sh.cnt, a.K, pend_d[slot], pend_i[slot]);
                    }
                }
                if (sh.cnt == a.K) {  // ivf.cpp:268-270; dco.hpp:125
                    const double rn = topd[a.K - 1];
                    const double rsq = __dmul_rn(rn, rn);
                    for (int i = static_cast<int>(lane); i < a.ntest; i += 32) {
                        const double t = __dmul_rn(tfac[i], rsq);
                        thr2[pw * nt + i] = t;
                        if (w == 0) thr2[pn * nt + i] = t;
                    }
                    if (lane == 0) {
                        sh.r = rn;
                        sh.r_sq = rsq;
                        lg.r[pw] = rn;
                        lg.r_sq[pw] = rsq;
                        if (w == 0) {
                            lg.r[pn] = rn;
                            lg.r_sq[pn] = rsq;
                        }
                    }
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_dims += __shfl_xor_sync(kFull, my_dims, o);
        if (lane == 0) atomicAdd(&sh.dims, my_dims);
        __syncthreads();
        const int cnt = sh.cnt;
        for (int i = threadIdx.x; i < a.K; i += blockDim.x) {
            const int64_t o = static_cast<int64_t>(qi) * a.K + i;
            a.out_ids[o] = i < cnt ? topi[i] : -1;
            a.out_dists[o] = i < cnt ? topd[i] : __longlong_as_double(0x7ff8000000000000ll);
        }
        if (threadIdx.x == 0) {
            a.out_cnt[qi] = cnt;
            a.out_dims[qi] = sh.dims;
            if (a.out_cand) a.out_cand[qi] = static_cast<unsigned long long>(total);
        }
    }
}

size_t search_smem_lag(const SearchLaunch& a, int chunk_cap) {
    const int nt = a.ntest > 0 ? a.ntest : 1;
    size_t b = sizeof(float) * a.warps * 1024;
    b += sizeof(double) * (a.nseg * kQPitch + 3 * nt + a.K + 2 * chunk_cap);
    b += sizeof(int32_t) * (a.nprobe + 2 * chunk_cap + (a.nprobe & 1));
    b += sizeof(Seg) * a.nseg;
    b += sizeof(int32_t) * (a.K + a.nprobe + 1);
    b += sizeof(unsigned) * 2 * ((chunk_cap + 31) / 32);
    return b;
}

size_t search_smem(const SearchLaunch& a, int chunk_cap) {
    const int nt = a.ntest > 0 ? a.ntest : 1;
    const bool dense = a.a1i != nullptr, f32 = a.f32 && a.vec == 4 && a.full;
    size_t b = sizeof(float) * a.warps * 1024;
    b += sizeof(double) * (a.nseg * kQPitch + 2 * nt + a.K + slot_words(dense, f32, chunk_cap, a.warps, a.nseg0 > 0));
    b += sizeof(int32_t) * (a.nprobe + chunk_cap + ((chunk_cap + a.nprobe) & 1));
    b += sizeof(Seg) * a.nseg;
    b += sizeof(int32_t) * (a.K + a.nprobe + 1);
    b += sizeof(unsigned) * ((chunk_cap + 31) / 32) * (a.f32 ? 2 : 1);
    return b;
}

}  // namespace

namespace {
// Queries ordered by a 32-bit key (ties by query index): one CTA bitonic-sorts a
// tile of kOrderTile packed (key << 32 | q) words in shared memory, so a batch of
// up to kOrderTile queries is fully ordered and larger ones are ordered per tile.
// Results never depend on the order (each query is searched independently); it
// only shapes the persistent scan grid's tail.
constexpr int kOrderTile = 16384;
constexpr int kOrderThreads = 1024;

__global__ void order_keys_kernel(const int32_t* probes, int nq, int nprobe, const int32_t* rank,
                                  unsigned long long* words) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint32_t key = static_cast<uint32_t>(rank[probes[static_cast<int64_t>(q) * nprobe]]);
    words[q] = (static_cast<unsigned long long>(key) << 32) | static_cast<uint32_t>(q);
}

// key = 2^32 - 1 - (candidates the query will stream), so ascending order puts the
// longest queries first
__global__ void work_keys_kernel(const int32_t* probes, int nq, int nprobe, int probe_lo,
                                 const int64_t* list_off, unsigned long long* words) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    int64_t tot = 0;
    for (int i = probe_lo; i < nprobe; ++i) {
        const int p = probes[static_cast<int64_t>(q) * nprobe + i];
        tot += list_off[p + 1] - list_off[p];
    }
    const uint32_t key = 0xFFFFFFFFu - static_cast<uint32_t>(tot < 0xFFFFFFFF ? tot : 0xFFFFFFFF);
    words[q] = (static_cast<unsigned long long>(key) << 32) | static_cast<uint32_t>(q);
}

__global__ void __launch_bounds__(kOrderThreads) order_sort_kernel(const unsigned long long* words, int nq,
                                                                   int32_t* order) {
    extern __shared__ unsigned long long tile[];
    const int base = blockIdx.x * kOrderTile;
    const int n = min(kOrderTile, nq - base);
    int P2 = 1;
    while (P2 < n) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) tile[i] = i < n ? words[base + i] : ~0ull;
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = tile[lo], y = tile[hi];
                if ((x > y) == up) {
                    tile[lo] = y;
                    tile[hi] = x;
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) order[base + i] = static_cast<int32_t>(tile[i] & 0xffffffffu);
}

void sort_order(const unsigned long long* words, int nq, int32_t* order, cudaStream_t st) {
    const int tiles = (nq + kOrderTile - 1) / kOrderTile;
    int P2 = 1;
    while (P2 < (nq < kOrderTile ? nq : kOrderTile)) P2 <<= 1;
    const size_t smem = sizeof(unsigned long long) * static_cast<size_t>(P2);
    ADS_CUDA(cudaFuncSetAttribute(order_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sizeof(unsigned long long) * kOrderTile)));
    order_sort_kernel<<<tiles, kOrderThreads, smem, st>>>(words, nq, order);
    ADS_LAUNCH_CHECK();
}
}  // namespace

void launch_query_order(const int32_t* probes, int nq, int nprobe, const int32_t* rank, int k,
                        DevBuf& scratch, int32_t* order, cudaStream_t st) {
    (void)k;
    if (nq <= 0) return;
    unsigned long long* w = scratch.get<unsigned long long>(static_cast<size_t>(nq));
    order_keys_kernel<<<(nq + 255) / 256, 256, 0, st>>>(probes, nq, nprobe, rank, w);
    ADS_LAUNCH_CHECK();
    sort_order(w, nq, order, st);
}

void launch_query_order_work(const int32_t* probes, int nq, int nprobe, int probe_lo, const int64_t* list_off,
                             DevBuf& scratch, int32_t* order, cudaStream_t st) {
    if (nq <= 0) return;
    unsigned long long* w = scratch.get<unsigned long long>(static_cast<size_t>(nq));
    work_keys_kernel<<<(nq + 255) / 256, 256, 0, st>>>(probes, nq, nprobe, probe_lo, list_off, w);
    ADS_LAUNCH_CHECK();
    sort_order(w, nq, order, st);
}

void launch_coarse_dist(const float* Q, int nq, const float* C, int L, int D, double* out,
                        cudaStream_t st) {
    if (nq <= 0 || L <= 0) return;
    dim3 grid((L + kCT - 1) / kCT, (nq + kQT - 1) / kQT);
    coarse_dist_kernel<<<grid, kCT, 0, st>>>(Q, nq, C, L, D, out);
    ADS_LAUNCH_CHECK();
}

void launch_select_probes(const double* dist, int nq, int L, int nprobe, int32_t* probes,
                          cudaStream_t st) {
    if (nq <= 0) return;
    int P2 = 1;
    while (P2 < nprobe) P2 <<= 1;
    if (P2 < 2) P2 = 2;
    const size_t smem = static_cast<size_t>(P2) * (sizeof(unsigned long long) + sizeof(int32_t));
    if (smem > 200 * 1024) throw std::invalid_argument("select: k too large");
    ADS_CUDA(cudaFuncSetAttribute(select_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    select_rows_kernel<<<nq, kSelThreads, smem, st>>>(dist, L, nprobe, P2, probes);
    ADS_LAUNCH_CHECK();
}

namespace {
struct SearchShape {
    void (*kern)(SearchLaunch, int);
    int cap;
    size_t smem;
    int occ;  // resident CTAs per SM
};

// Deep tail steps pay where walks are long (config 3: 30 segments, +5 %); below
// kDeepMinSeg segments a chunk's tail is a few steps and the plain kernel is level or
// ahead (config 2, 4 segments: -0.7 %).  Not with the pre-walk (no lane is idle there).
bool search_deep(const SearchLaunch& a) {
    return kDeepTail > 0 && a.vec == 4 && !a.f32 && a.nseg0 == 0 && a.nseg >= kDeepMinSeg;
}

// Overlapped chunks (ivf_search_lag_kernel): on request, where the plain lane walk runs.
bool search_lag(const SearchLaunch& a) {
    return a.lag != 0 && a.vec == 4 && !a.f32 && !a.a1i && a.nseg0 == 0;
}

SearchShape search_shape_of(const SearchLaunch& a) {
    const int64_t cap64 = a.first > a.step ? a.first : a.step;
    if (a.first < 1 || a.step < 1) throw std::invalid_argument("search: threshold schedule must be >= 1");
    if (cap64 > 16384) throw std::invalid_argument("search: threshold refresh interval too long (max 16384)");
    SearchShape sh{};
    sh.cap = static_cast<int>(cap64);
    sh.smem = search_smem(a, sh.cap);
    if (search_lag(a)) {
        sh.smem = search_smem_lag(a, sh.cap);
        sh.kern = a.full ? ((kQueryPlanes && a.nseg >= kDeepMinSeg) ? ivf_search_lag_kernel<true, true>
                                                                     : ivf_search_lag_kernel<true, false>)
                         : ivf_search_lag_kernel<false, false>;
    } else if (a.f32 && a.vec == 4 && a.full)
        sh.kern = a.a1i ? ivf_search_kernel<4, true, true, true> : ivf_search_kernel<4, true, false, true>;
    else if (search_deep(a))
        sh.kern = a.a1i ? (a.full ? ivf_search_kernel<4, true, true, false, true> : ivf_search_kernel<4, false, true, false, true>)
                        : (a.full ? ivf_search_kernel<4, true, false, false, true> : ivf_search_kernel<4, false, false, false, true>);
    else if (a.a1i)
        sh.kern = a.full ? ivf_search_kernel<4, true, true, false> : ivf_search_kernel<4, false, true, false>;
    else
        sh.kern = a.vec == 4 ? (a.full ? ivf_search_kernel<4, true, false, false> : ivf_search_kernel<4, false, false, false>)
                             : ivf_search_kernel<1, false, false, false>;
    ADS_CUDA(cudaFuncSetAttribute(sh.kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sh.smem)));
    ADS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sh.occ, sh.kern, a.warps * 32, sh.smem));
    if (sh.occ < 1) throw std::invalid_argument("search: configuration exceeds shared memory");
    if (a.ctas_per_sm > 0 && a.ctas_per_sm < sh.occ) sh.occ = a.ctas_per_sm;
    return sh;
}
}  // namespace

int64_t search_resident_ctas(const SearchLaunch& a) {
    return static_cast<int64_t>(num_sms()) * search_shape_of(a).occ;
}

void launch_ivf_search(const SearchLaunch& a, cudaStream_t st) {
    if (a.nq <= 0) return;
    const SearchShape sh = search_shape_of(a);
    ADS_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st));
    int64_t grid = static_cast<int64_t>(num_sms()) * sh.occ;
    if (grid > a.nq) grid = a.nq;
    sh.kern<<<static_cast<unsigned>(grid), a.warps * 32, sh.smem, st>>>(a, sh.cap);
    ADS_LAUNCH_CHECK();
}

namespace {
// One CTA per query: load the G*K (dist, id) entries, bitonic-sort by
// (dist, id) with invalid entries (NaN dist or id < 0) as +inf, keep K.
__global__ void __launch_bounds__(256) merge_topk_kernel(const double* __restrict__ dists,
                                                         const int32_t* __restrict__ ids, int G,
                                                         int nq, int K, int P2,
                                                         int32_t* __restrict__ out_ids,
                                                         double* __restrict__ out_dists,
                                                         int32_t* __restrict__ out_cnt) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* kd = reinterpret_cast<double*>(sm);
    int32_t* ki = reinterpret_cast<int32_t*>(kd + P2);
    __shared__ int s_cnt;
    const int q = blockIdx.x, tid = threadIdx.x;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int e = tid; e < P2; e += blockDim.x) {
        double d = kInf;
        int32_t id = 0x7fffffff;
        if (e < G * K) {
            const int g = e / K, j = e % K;
            const int64_t o = (static_cast<int64_t>(g) * nq + q) * K + j;
            const double dv = dists[o];
            const int32_t iv = ids[o];
            if (iv >= 0 && dv == dv) {
                d = dv;
                id = iv;
                atomicAdd(&s_cnt, 1);
            }
        }
        kd[e] = d;
        ki[e] = id;
    }
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const double da = kd[lo], db = kd[hi];
                const int32_t ia = ki[lo], ib = ki[hi];
                const bool a_gt_b = da > db || (da == db && ia > ib);
                if (a_gt_b == up) {
                    kd[lo] = db;
                    kd[hi] = da;
                    ki[lo] = ib;
                    ki[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    const int cnt = s_cnt < K ? s_cnt : K;
    for (int j = tid; j < K; j += blockDim.x) {
        out_ids[static_cast<int64_t>(q) * K + j] = j < cnt ? ki[j] : -1;
        out_dists[static_cast<int64_t>(q) * K + j] = j < cnt ? kd[j] : __longlong_as_double(0x7ff8000000000000ll);
    }
    if (tid == 0 && out_cnt) out_cnt[q] = cnt;
}
}  // namespace

void launch_merge_topk(const double* dists, const int32_t* ids, int G, int nq, int K,
                       int32_t* out_ids, double* out_dists, int32_t* out_cnt, cudaStream_t st) {
    if (nq <= 0) return;
    int P2 = 2;
    while (P2 < G * K) P2 <<= 1;
    const size_t smem = static_cast<size_t>(P2) * (sizeof(double) + sizeof(int32_t));
    if (smem > 200 * 1024) throw std::invalid_argument("merge_topk: G*K too large");
    ADS_CUDA(cudaFuncSetAttribute(merge_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    merge_topk_kernel<<<nq, 256, smem, st>>>(dists, ids, G, nq, K, P2, out_ids, out_dists, out_cnt);
    ADS_LAUNCH_CHECK();
}

}  // namespace ads

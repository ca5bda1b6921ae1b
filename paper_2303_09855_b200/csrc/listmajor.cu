// List-major ("wave") IVF search: every probed list is read from HBM once per
// threshold-refresh wave and scanned from shared memory for all queries that
// probe it in that wave.
//
// Schedule (deterministic): a query's probe ranks are cut into waves
// [0, b0), [b0, b0+B), [b0+B, b0+2B), ...  All candidates of a wave are tested
// against the threshold table of the query's heap as it stood after merging
// every earlier wave; the wave's positives are then offered to the bounded
// (dist, id) heap in candidate (stream) order with the reference's strict rule
// (ivf.cpp:273-280).  The oracle reproduces it with orc_ivf_query_waves, and
// the per-DCO arithmetic is the exact fp64 engine of scan_engine.cuh.
//
// Per wave:  pairs (query, rank) are bucketed by list (count / scan / scatter);
// scan_lists_kernel gives each list to one CTA, which stages the list's A1/A2
// rows tile by tile in shared memory (cp.async, coalesced, one DRAM read per
// list per wave) and lets its warps take the list's queries one at a time,
// walking the tile's candidates level-synchronously (all lanes on the same
// segment of the same query -> broadcast query loads, no per-line gathers);
// survivors of each test are compacted into a per-warp queue.  Decisions go
// to dense per-candidate slots; merge_wave_kernel folds them into each
// query's heap in stream order and rebuilds its thresholds.
#include <cub/cub.cuh>
#include <cstdio>

#include "engine.hpp"
#include "scan_engine.cuh"

namespace ads {

namespace {

constexpr double kInfLM = __builtin_huge_val();

__global__ void lm_init_kernel(int nq, int K, int ntest, int32_t* cnt, double* r, double* thr,
                               unsigned long long* dims) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    cnt[q] = 0;
    r[2 * q] = kInfLM;
    r[2 * q + 1] = kInfLM;
    for (int t = 0; t < ntest; ++t) thr[static_cast<int64_t>(q) * ntest + t] = kInfLM;
    dims[q] = 0;
}

// pre[q][i] = number of candidates in probe ranks < i.
__global__ void lm_prefix_kernel(const int32_t* __restrict__ probes, const int64_t* __restrict__ list_off,
                                 int nq, int nprobe, int32_t* __restrict__ pre) {
    const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const unsigned lane = threadIdx.x & 31u;
    if (q >= nq) return;
    int carry = 0;
    int32_t* pq = pre + static_cast<int64_t>(q) * (nprobe + 1);
    for (int base = 0; base < nprobe; base += 32) {
        const int i = base + static_cast<int>(lane);
        int len = 0;
        if (i < nprobe) {
            const int p = probes[static_cast<int64_t>(q) * nprobe + i];
            len = static_cast<int>(list_off[p + 1] - list_off[p]);
        }
        int incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (static_cast<int>(lane) >= o) incl += v;
        }
        if (i < nprobe) pq[i + 1] = carry + incl;
        carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) pq[0] = 0;
}

// Per-query candidate count of wave [r0, r1) and per-list pair counts.
__global__ void lm_count_kernel(const int32_t* __restrict__ probes, const int32_t* __restrict__ pre,
                                int nq, int nprobe, int r0, int r1, int32_t* __restrict__ wcnt,
                                int32_t* __restrict__ list_cnt) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int span = r1 - r0;
    if (t >= static_cast<int64_t>(nq) * span) return;
    const int q = static_cast<int>(t / span), j = static_cast<int>(t % span);
    const int32_t* pq = pre + static_cast<int64_t>(q) * (nprobe + 1);
    if (j == 0) wcnt[q] = pq[r1] - pq[r0];
    const int rank = r0 + j;
    if (pq[rank + 1] > pq[rank]) atomicAdd(&list_cnt[probes[static_cast<int64_t>(q) * nprobe + rank]], 1);
}

__global__ void lm_scatter_kernel(const int32_t* __restrict__ probes, const int32_t* __restrict__ pre,
                                  int nq, int nprobe, int r0, int r1, const int32_t* __restrict__ list_pair_off,
                                  int32_t* __restrict__ fill, int2* __restrict__ pairs) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int span = r1 - r0;
    if (t >= static_cast<int64_t>(nq) * span) return;
    const int q = static_cast<int>(t / span), rank = r0 + static_cast<int>(t % span);
    const int32_t* pq = pre + static_cast<int64_t>(q) * (nprobe + 1);
    if (pq[rank + 1] == pq[rank]) return;
    const int L = probes[static_cast<int64_t>(q) * nprobe + rank];
    const int slot = list_pair_off[L] + atomicAdd(&fill[L], 1);
    pairs[slot] = make_int2(q, rank);
}

__host__ __device__ inline size_t lm_per_warp(int nseg, int nt, int tile) {
    const size_t b = sizeof(double) * (static_cast<size_t>(nseg) * kQPitch + nt + 2) +
                     (sizeof(int) + sizeof(double)) * 2 * static_cast<size_t>(tile);
    return (b + 15) & ~size_t(15);
}

struct ScanLists {
    const float* a1;
    const float* a2;
    int d1, D;
    const int32_t* ids;
    const int64_t* list_off;
    int L;
    const float* Q;
    int nprobe;
    const int32_t* pre;
    const int32_t* wbase;  // dense slot of the wave's first candidate, per query
    int r0;                // first probe rank of the wave
    const int32_t* list_pair_off;
    const int2* pairs;
    const Seg* segs;
    int nseg, ntest, final_fd;
    const double* thr;     // nq x ntest
    const double* rr;      // nq x 2 (r, r^2)
    unsigned char* flag;   // dense per candidate of the wave
    double* pdist;
    int32_t* pid;
    unsigned long long* dims;
    int tile;              // candidates per shared-memory tile
    int qgroup;            // queries per group (shared-memory staging)
    unsigned* list_counter;
    long long nslots, nq;  // bounds (debug checks)
};

// Shared-memory row pitch (floats) for rows of `w` floats: padded so that
// consecutive rows start 16 bytes apart modulo 128 (pitch/4 = 1 mod 8), which
// keeps a quarter-warp's float4 reads of eight rows on distinct banks.
__host__ __device__ inline int lm_pitch(int w) {
    const int c = w / 4;
    return (c + ((1 - c) & 7)) * 4;
}

#ifdef ADS_DEBUG
#define LM_CHECK(cond, tag, v)                                                            \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("LM_CHECK %s failed: %lld (block %d thread %d)\n", tag,               \
                   static_cast<long long>(v), blockIdx.x, threadIdx.x);                   \
            asm volatile("trap;");                                                        \
        }                                                                                 \
    } while (0)
#else
#define LM_CHECK(cond, tag, v) (void)0
#endif

// One lane's segment from a shared-memory row, index order, exact fp64.
__device__ __forceinline__ double seg_acc(const float* row, const double* qq, int nch, double s) {
    LM_CHECK((reinterpret_cast<uintptr_t>(row) & 15) == 0, "row align", reinterpret_cast<uintptr_t>(row) & 1023);
    LM_CHECK((reinterpret_cast<uintptr_t>(qq) & 15) == 0, "qq align", reinterpret_cast<uintptr_t>(qq) & 1023);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (c < nch) {
            const float4 v = *reinterpret_cast<const float4*>(row + c * 4);
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

// One CTA per list (persistent over lists).  For each tile of the list and
// each group of up to QG queries probing it, all (candidate, query) pairs go
// through the segments level by level: level 0 enumerates every pair, later
// levels take the survivors from a CTA-wide queue, so every lane always works
// on a live pair and no pair waits for another.
template <int T>
__global__ void __launch_bounds__(512) scan_lists_kernel(ScanLists a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_list, s_nout[3];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    (void)warp;
    const int d2 = a.D - a.d1;
    const int QG = a.qgroup;
    const int nt = a.ntest > 0 ? a.ntest : 1;
    const int p1 = lm_pitch(a.d1), p2 = d2 > 0 ? lm_pitch(d2) : 0;
    // layout: tA1 [T*p1] | tA2 [T*p2] | qstage [QG*nseg*34] | thr [QG*nt] | rr [QG*2]
    //         | qs_s [2][T*QG] f64 | qs_e [2][T*QG] i32 | gq, gbase, gdims [QG] | segs
    float* tA1 = reinterpret_cast<float*>(smem_raw);
    float* tA2 = tA1 + T * p1;
    double* qstage = reinterpret_cast<double*>(tA2 + T * p2);
    double* thr = qstage + QG * a.nseg * kQPitch;
    double* rr = thr + QG * nt;
    double* qs_s = rr + 2 * QG;
    int* qs_e = reinterpret_cast<int*>(qs_s + 2 * T * QG);
    int* gq = qs_e + 2 * T * QG;
    int* gbase = gq + QG;
    unsigned* gdims = reinterpret_cast<unsigned*>(gbase + QG);
    Seg* segs = reinterpret_cast<Seg*>(gdims + QG);
    for (int i = threadIdx.x; i < a.nseg; i += blockDim.x) segs[i] = a.segs[i];

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            int L;
            do {
                L = static_cast<int>(atomicAdd(a.list_counter, 1u));
            } while (L < a.L && a.list_pair_off[L + 1] == a.list_pair_off[L]);
            s_list = L;
        }
        __syncthreads();
        const int L = s_list;
        if (L >= a.L) break;
        const int64_t row0 = a.list_off[L];
        const int nrows = static_cast<int>(a.list_off[L + 1] - row0);
        const int pb = a.list_pair_off[L], pe = a.list_pair_off[L + 1];
        for (int t0 = 0; t0 < nrows; t0 += T) {
            const int rows = nrows - t0 < T ? nrows - t0 : T;
            {  // stage the tile: A1 and A2 rows of the list are contiguous
                const float4* s1 = reinterpret_cast<const float4*>(a.a1 + (row0 + t0) * a.d1);
                const int c1 = a.d1 / 4, n1 = rows * c1;
                for (int i = threadIdx.x; i < n1; i += blockDim.x) {
                    const int r = i / c1, c = i - r * c1;
                    cp_async16(tA1 + r * p1 + c * 4, s1 + i);
                }
                if (d2 > 0) {
                    const float4* s2 = reinterpret_cast<const float4*>(a.a2 + (row0 + t0) * d2);
                    const int c2 = d2 / 4, n2 = rows * c2;
                    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                        const int r = i / c2, c = i - r * c2;
                        cp_async16(tA2 + r * p2 + c * 4, s2 + i);
                    }
                }
            }
            for (int g0 = pb; g0 < pe; g0 += QG) {
                const int ng = pe - g0 < QG ? pe - g0 : QG;
                // stage the group's queries, thresholds and dense-slot bases
                for (int i = threadIdx.x; i < ng * a.nseg * 32; i += blockDim.x) {
                    const int g = i / (a.nseg * 32), rem = i - g * a.nseg * 32;
                    const int sg = rem >> 5, k = rem & 31;
                    const Seg sgm = segs[sg];
                    if (k < sgm.len) {
                        const int q = a.pairs[g0 + g].x;
                        qstage[(g * a.nseg + sg) * kQPitch + k] =
                            static_cast<double>(a.Q[static_cast<int64_t>(q) * a.D + sgm.col + k]);
                    }
                }
                for (int i = threadIdx.x; i < ng * nt; i += blockDim.x) {
                    const int g = i / nt, t = i - g * nt;
                    if (t < a.ntest) thr[i] = a.thr[static_cast<int64_t>(a.pairs[g0 + g].x) * a.ntest + t];
                }
                if (threadIdx.x == 0) s_nout[0] = 0;
                for (int g = threadIdx.x; g < ng; g += blockDim.x) {
                    const int2 pr = a.pairs[g0 + g];
                    LM_CHECK(pr.x >= 0 && pr.x < a.nq && pr.y >= 0 && pr.y < a.nprobe, "pair", pr.x);
                    const int32_t* pq = a.pre + static_cast<int64_t>(pr.x) * (a.nprobe + 1);
                    gq[g] = pr.x;
                    gbase[g] = a.wbase[pr.x] + (pq[pr.y] - pq[a.r0]) + t0;
                    gdims[g] = 0;
                    rr[2 * g] = a.rr[2 * pr.x];
                    rr[2 * g + 1] = a.rr[2 * pr.x + 1];
                }
                cp_async_wait_all();
                __syncthreads();
                int n_in = ng * T;  // level 0: every (candidate, query) pair, entry = g*T + c
                int cur = 0;
                // Survivor counters rotate over three slots: level sg counts into
                // slot sg%3 and clears slot (sg+1)%3, whose last reader (level
                // sg-2's total) is separated from this write by the barrier that
                // ended level sg-1.
                for (int sg = 0; sg < a.nseg; ++sg) {
                    if (threadIdx.x == 0) s_nout[(sg + 1) % 3] = 0;
                    const Seg sgm = segs[sg];
                    const int nch = sgm.len >> 2;
                    const bool last = sg == a.nseg - 1;
                    const double* qin_s = qs_s + cur * T * QG;
                    const int* qin_e = qs_e + cur * T * QG;
                    double* qout_s = qs_s + (cur ^ 1) * T * QG;
                    int* qout_e = qs_e + (cur ^ 1) * T * QG;
                    const int n_round = (n_in + 31) & ~31;
                    for (int e = threadIdx.x; e < n_round; e += blockDim.x) {
                        int entry = 0;
                        double s = 0.0;
                        bool live = e < n_in;
                        if (live) {
                            entry = sg == 0 ? e : qin_e[e];
                            s = sg == 0 ? 0.0 : qin_s[e];
                            if (sg == 0 && (entry % T) >= rows) live = false;
                        }
                        const int g = entry / T, c = entry % T;
                        bool keep = false;
                        unsigned fin_dims = 0;
                        if (live) {
                            const float* row = sgm.arr == 0 ? tA1 + c * p1 + sgm.col
                                                            : tA2 + c * p2 + (sgm.col - a.d1);
                            s = seg_acc(row, qstage + (g * a.nseg + sg) * kQPitch, nch, s);
                            const int slot = gbase[g] + c;
                            LM_CHECK(slot >= 0 && slot < a.nslots, "slot", slot);
                            LM_CHECK(g < QG && c < T, "entry", entry);
                            if (sgm.test >= 0 && s > thr[g * nt + sgm.test]) {  // reject (dco.hpp:141)
                                fin_dims = static_cast<unsigned>(sgm.col + sgm.len);
                                a.flag[slot] = 0;
                            } else if (last) {  // d == D
                                fin_dims = static_cast<unsigned>(a.D);
                                const double dist = __dsqrt_rn(s);
                                const bool positive = a.final_fd ? dist <= rr[2 * g] : s <= rr[2 * g + 1];
                                a.flag[slot] = positive;
                                if (positive) {
                                    a.pdist[slot] = dist;
                                    a.pid[slot] = a.ids[row0 + t0 + c];
                                }
                            } else {
                                keep = true;
                            }
                        }
                        // dims: one shared atomic per distinct group among the warp's finishers
                        const unsigned fm = __ballot_sync(kFull, fin_dims != 0);
                        if (fin_dims) {
                            const unsigned same = __match_any_sync(fm, g);
                            const unsigned tot = __reduce_add_sync(same, fin_dims);
                            if (static_cast<int>(lane) == __ffs(same) - 1) atomicAdd(&gdims[g], tot);
                        }
                        const unsigned km = __ballot_sync(kFull, keep);
                        int base = 0;
                        if (lane == 0 && km) base = atomicAdd(&s_nout[sg % 3], __popc(km));
                        base = __shfl_sync(kFull, base, 0);
                        if (keep) {
                            const int o = base + __popc(km & ((1u << lane) - 1u));
                            LM_CHECK(o < T * QG, "queue", o);
                            qout_e[o] = entry;
                            qout_s[o] = s;
                        }
                    }
                    __syncthreads();
                    n_in = s_nout[sg % 3];
                    cur ^= 1;
                    if (n_in == 0) break;
                }
                __syncthreads();
                for (int g = threadIdx.x; g < ng; g += blockDim.x)
                    if (gdims[g]) atomicAdd(a.dims + gq[g], static_cast<unsigned long long>(gdims[g]));
                __syncthreads();
            }
            __syncthreads();
        }
    }
}

// ivf.cpp:273-280 offer() by one warp on a shared heap (same as the query-major path).
__device__ void lm_offer(double* topd, int32_t* topi, int* cnt, int K, double dist, int32_t id) {
    const unsigned lane = lane_id();
    const int c = *cnt;
    if (c == K && !(dist < topd[K - 1])) return;
    const int ceff = c == K ? K - 1 : c;
    int pos = 0;
    for (int base = 0; base < ceff; base += 32) {
        const int j = base + static_cast<int>(lane);
        const bool lt = j < ceff && (topd[j] < dist || (topd[j] == dist && topi[j] < id));
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

// One warp per query: fold the wave's positives into the heap in stream order.
__global__ void merge_wave_kernel(int nq, int K, int ntest, const int32_t* __restrict__ wbase,
                                  const int32_t* __restrict__ wcnt,
                                  const unsigned char* __restrict__ flag, const double* __restrict__ pdist,
                                  const int32_t* __restrict__ pid, double* heap_d, int32_t* heap_i,
                                  int32_t* heap_cnt, const double* __restrict__ tfac, double* thr,
                                  double* rr) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int wpb = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int q = blockIdx.x * wpb + warp;
    double* topd = reinterpret_cast<double*>(sm) + static_cast<size_t>(warp) * K;
    int32_t* topi = reinterpret_cast<int32_t*>(reinterpret_cast<double*>(sm) + static_cast<size_t>(wpb) * K) +
                    static_cast<size_t>(warp) * K;
    __shared__ int s_cnt[32];
    if (q >= nq) return;
    const int64_t hb = static_cast<int64_t>(q) * K;
    for (int j = static_cast<int>(lane); j < K; j += 32) {
        topd[j] = heap_d[hb + j];
        topi[j] = heap_i[hb + j];
    }
    if (lane == 0) s_cnt[warp] = heap_cnt[q];
    __syncwarp();
    const int b = wbase[q], n = wcnt[q];
    for (int base = 0; base < n; base += 32) {
        const int i = base + static_cast<int>(lane);
        const bool f = i < n && flag[b + i];
        unsigned bits = __ballot_sync(kFull, f);
        while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1;
            const int slot = b + base + k;
            lm_offer(topd, topi, &s_cnt[warp], K, pdist[slot], pid[slot]);
        }
    }
    const int cnt = s_cnt[warp];
    for (int j = static_cast<int>(lane); j < K; j += 32) {
        heap_d[hb + j] = topd[j];
        heap_i[hb + j] = topi[j];
    }
    if (cnt == K) {  // ivf.cpp:268-270; dco.hpp:125
        const double rn = topd[K - 1];
        const double rsq = __dmul_rn(rn, rn);
        for (int t = static_cast<int>(lane); t < ntest; t += 32)
            thr[static_cast<int64_t>(q) * ntest + t] = __dmul_rn(tfac[t], rsq);
        if (lane == 0) {
            rr[2 * q] = rn;
            rr[2 * q + 1] = rsq;
        }
    }
    if (lane == 0) heap_cnt[q] = cnt;
}

__global__ void lm_output_kernel(int nq, int K, int nprobe, const double* heap_d, const int32_t* heap_i,
                                 const int32_t* heap_cnt, const int32_t* pre,
                                 const unsigned long long* dims, int32_t* out_ids, double* out_dists,
                                 int32_t* out_cnt, unsigned long long* out_dims,
                                 unsigned long long* out_cand) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(nq) * K) return;
    const int q = static_cast<int>(t / K), j = static_cast<int>(t % K);
    const int cnt = heap_cnt[q];
    out_ids[t] = j < cnt ? heap_i[t] : -1;
    out_dists[t] = j < cnt ? heap_d[t] : __longlong_as_double(0x7ff8000000000000ll);
    if (j == 0) {
        out_cnt[q] = cnt;
        out_dims[q] = dims[q];
        if (out_cand) out_cand[q] = static_cast<unsigned long long>(pre[static_cast<int64_t>(q) * (nprobe + 1) + nprobe]);
    }
}

__global__ void lm_wave_max_kernel(const int32_t* __restrict__ pre, int nq, int nprobe, int b0, int B,
                                   unsigned long long* total_max) {
    // total candidates of every wave summed over queries; one block per wave
    const int w = blockIdx.x;
    const int r0 = w == 0 ? 0 : b0 + (w - 1) * B;
    int r1 = w == 0 ? b0 : r0 + B;
    if (r1 > nprobe) r1 = nprobe;
    unsigned long long s = 0;
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        const int32_t* pq = pre + static_cast<int64_t>(q) * (nprobe + 1);
        s += static_cast<unsigned long long>(pq[r1] - pq[r0]);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    __shared__ unsigned long long ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += ws[i];
        atomicMax(total_max, tot);
    }
}

inline unsigned nblk(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

size_t listmajor_scan_smem(int tile, int d1, int D, int nseg, int ntest, int qgroup) {
    const int nt = ntest > 0 ? ntest : 1;
    const int d2 = D - d1;
    size_t b = sizeof(float) * static_cast<size_t>(tile) * (lm_pitch(d1) + (d2 > 0 ? lm_pitch(d2) : 0));
    b += sizeof(double) * (static_cast<size_t>(qgroup) * nseg * kQPitch + qgroup * nt + 2 * qgroup);
    b += (sizeof(double) + sizeof(int)) * 2 * static_cast<size_t>(tile) * qgroup;
    b += sizeof(int) * 3 * qgroup + sizeof(Seg) * nseg;
    return b;
}

void launch_listmajor_search(const ListMajorLaunch& a, ListMajorScratch& s, cudaStream_t st) {
    const int nq = a.nq, nprobe = a.nprobe, K = a.K, L = a.L;
    if (nq <= 0) return;
    const int b0 = a.first_lists, B = a.step_lists;
    if (b0 < 1 || B < 1) throw std::invalid_argument("search: wave sizes must be >= 1");
    const int nwaves = nprobe <= b0 ? 1 : 1 + (nprobe - b0 + B - 1) / B;
    const int nt = a.ntest > 0 ? a.ntest : 1;
    auto pre = s.pre.get<int32_t>(static_cast<size_t>(nq) * (nprobe + 1));
    auto heap_d = s.heap_d.get<double>(static_cast<size_t>(nq) * K);
    auto heap_i = s.heap_i.get<int32_t>(static_cast<size_t>(nq) * K);
    auto heap_c = s.heap_c.get<int32_t>(nq);
    auto rr = s.rr.get<double>(static_cast<size_t>(nq) * 2);
    auto thr = s.thr.get<double>(static_cast<size_t>(nq) * nt);
    auto dims = s.dims.get<unsigned long long>(nq);
    auto wcnt = s.wcnt.get<int32_t>(nq + 1);
    auto wbase = s.wbase.get<int32_t>(nq + 1);
    auto lcnt = s.lcnt.get<int32_t>(L + 1);
    auto loff = s.loff.get<int32_t>(L + 1);
    auto fill = s.fill.get<int32_t>(L + 1);
    auto pairs = s.pairs.get<int2>(static_cast<size_t>(nq) * (b0 > B ? b0 : B));
    auto ctr = s.counter.get<unsigned long long>(2);

    lm_init_kernel<<<nblk(nq, 256), 256, 0, st>>>(nq, K, a.ntest, heap_c, rr, thr, dims);
    lm_prefix_kernel<<<nblk(nq, 8), 256, 0, st>>>(a.probes, a.list_off, nq, nprobe, pre);
    // dense per-candidate slots: the largest wave total over the batch
    ADS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    lm_wave_max_kernel<<<nwaves, 256, 0, st>>>(pre, nq, nprobe, b0, B, ctr);
    unsigned long long maxtot = 0;
    ADS_CUDA(cudaMemcpyAsync(&maxtot, ctr, sizeof(maxtot), cudaMemcpyDeviceToHost, st));
    ADS_CUDA(cudaStreamSynchronize(st));
    if (maxtot >= (1ull << 31)) throw std::invalid_argument("search: wave too large (2^31 candidates)");
    auto flag = s.flag.get<unsigned char>(maxtot + 1);
    auto pdist = s.pdist.get<double>(maxtot + 1);
    auto pid = s.pid.get<int32_t>(maxtot + 1);

    size_t scan_tmp = 0;
    ADS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, wcnt, wbase, nq + 1, st));
    size_t scan_tmp2 = 0;
    ADS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp2, lcnt, loff, L + 1, st));
    auto tmp = s.tmp.get<unsigned char>(scan_tmp > scan_tmp2 ? scan_tmp : scan_tmp2);
    const size_t tmp_bytes = scan_tmp > scan_tmp2 ? scan_tmp : scan_tmp2;

    int qg = a.qgroup > 0 ? a.qgroup : 8;
    size_t smem = listmajor_scan_smem(a.tile, a.d1, a.D, a.nseg, a.ntest, qg);
    while (qg > 1 && smem > 110 * 1024) smem = listmajor_scan_smem(a.tile, a.d1, a.D, a.nseg, a.ntest, --qg);
    auto kern = a.tile <= 16 ? scan_lists_kernel<16>
              : a.tile <= 32 ? scan_lists_kernel<32>
              : a.tile <= 64 ? scan_lists_kernel<64> : scan_lists_kernel<128>;
    const int tile = a.tile <= 16 ? 16 : a.tile <= 32 ? 32 : a.tile <= 64 ? 64 : 128;
    smem = listmajor_scan_smem(tile, a.d1, a.D, a.nseg, a.ntest, qg);
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int occ = 0;
    ADS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, a.warps * 32, smem));
    if (occ < 1) throw std::invalid_argument("search: list tile exceeds shared memory");
    const int grid = num_sms() * occ;
    const int mwpb = 8;
    const size_t msmem = static_cast<size_t>(mwpb) * K * (sizeof(double) + sizeof(int32_t));
    ADS_CUDA(cudaFuncSetAttribute(merge_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(msmem)));

    for (int w = 0; w < nwaves; ++w) {
        const int r0 = w == 0 ? 0 : b0 + (w - 1) * B;
        const int r1 = (w == 0 ? b0 : r0 + B) < nprobe ? (w == 0 ? b0 : r0 + B) : nprobe;
        ADS_CUDA(cudaMemsetAsync(lcnt, 0, sizeof(int32_t) * (L + 1), st));
        ADS_CUDA(cudaMemsetAsync(fill, 0, sizeof(int32_t) * (L + 1), st));
        ADS_CUDA(cudaMemsetAsync(wcnt + nq, 0, sizeof(int32_t), st));
        const int64_t np = static_cast<int64_t>(nq) * (r1 - r0);
        lm_count_kernel<<<nblk(np, 256), 256, 0, st>>>(a.probes, pre, nq, nprobe, r0, r1, wcnt, lcnt);
        size_t tb = tmp_bytes;
        ADS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, wcnt, wbase, nq + 1, st));
        tb = tmp_bytes;
        ADS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, lcnt, loff, L + 1, st));
        lm_scatter_kernel<<<nblk(np, 256), 256, 0, st>>>(a.probes, pre, nq, nprobe, r0, r1, loff, fill, pairs);
        ScanLists sl{};
        sl.a1 = a.a1;
        sl.a2 = a.a2;
        sl.d1 = a.d1;
        sl.D = a.D;
        sl.ids = a.ids;
        sl.list_off = a.list_off;
        sl.L = L;
        sl.Q = a.Q;
        sl.nprobe = nprobe;
        sl.pre = pre;
        sl.wbase = wbase;
        sl.r0 = r0;
        sl.list_pair_off = loff;
        sl.pairs = pairs;
        sl.segs = a.segs;
        sl.nseg = a.nseg;
        sl.ntest = a.ntest;
        sl.final_fd = a.final_fd;
        sl.thr = thr;
        sl.rr = rr;
        sl.flag = flag;
        sl.pdist = pdist;
        sl.pid = pid;
        sl.dims = dims;
        sl.tile = tile;
        sl.qgroup = qg;
        sl.nslots = static_cast<long long>(maxtot) + 1;
        sl.nq = nq;
        sl.list_counter = reinterpret_cast<unsigned*>(ctr + 1);
        ADS_CUDA(cudaMemsetAsync(ctr + 1, 0, sizeof(unsigned long long), st));
        kern<<<grid, a.warps * 32, smem, st>>>(sl);
        ADS_LAUNCH_CHECK();
        merge_wave_kernel<<<nblk(nq, mwpb), mwpb * 32, msmem, st>>>(nq, K, a.ntest, wbase, wcnt, flag,
                                                                      pdist, pid, heap_d, heap_i, heap_c,
                                                                      a.tfac, thr, rr);
        ADS_LAUNCH_CHECK();
    }
    lm_output_kernel<<<nblk(static_cast<int64_t>(nq) * K, 256), 256, 0, st>>>(
        nq, K, nprobe, heap_d, heap_i, heap_c, pre, dims, a.out_ids, a.out_dists, a.out_cnt, a.out_dims,
        a.out_cand);
    ADS_LAUNCH_CHECK();
}

}  // namespace ads

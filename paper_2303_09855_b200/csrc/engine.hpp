// Internal host-side interface between the C ABI (capi.cu) and the kernel
// launchers.  Not installed; the public boundary is include/adsann_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace ads {

// ---------------------------------------------------------------- segments
// Host-built description of how one candidate's D coordinates are walked:
// cut at every hypothesis-test point, at the A1/A2 split and every 32 floats.
struct SegPlan {
    std::vector<Seg> segs;
    std::vector<double> test_factor;  // thr[t] = test_factor[t] * r^2
    int vec = 4;                      // 16-byte copies when every cut is 4-aligned
    int full = 0;                     // every segment has 32 floats
    int D = 0;
};

// tests: sorted coordinate counts in (0, D) at which a test runs; factor[d]
// gives the multiplier there (nullptr -> 1.0, the exact partial scan).
SegPlan make_seg_plan(int D, int split_at, const std::vector<int>& tests, const double* factor);
// Test points of ad_scan / pd_scan_kernel started at d_start with or without
// the start test (dco.hpp:122-177).
std::vector<int> test_points(int D, int delta_d, int d_start, bool test_at_start);
// AdContext::factor (dco.cpp:54-61), host fp64.
std::vector<double> ad_factor(double eps0, int delta_d, int D);

struct DevSegPlan {
    Seg* segs = nullptr;
    double* tfac = nullptr;
    int nseg = 0, ntest = 0, vec = 4, full = 0;
    int nseg0 = 0;  // leading segments no test depends on (the search's pre-walk depth)
    void upload(const SegPlan& p, cudaStream_t st);
    void release();
};

// ---------------------------------------------------------------- kernels
struct DcoLaunch {
    const float* X;
    int64_t n_rows;
    int D;
    const float* Q;
    int nq;
    const int64_t* cand_off;   // device, nullable (window mode)
    const int64_t* cand_rows;  // device, nullable
    const int64_t* win_start;  // device, nullable
    int64_t win_len;
    const double* r;           // device
    const int64_t* tile_q;     // device tile table (CSR mode) or nullptr
    const int64_t* tile_lo;
    const int64_t* tile_hi;
    int64_t ntiles;
    int64_t tile;              // candidates per tile (window mode)
    int kind;                  // 0 fd, 1 pd, 2 ad
    const Seg* segs;
    const double* tfac;
    int nseg, ntest, vec;
    int desc;                  // 1: 32-bit line descriptors (VEC 4, n_rows * D / 4 < 2^32), full 32-float segments
    uint8_t* positive;
    int32_t* dims;
    double* dist_sq;
    double* observed;
    unsigned long long* dims_per_query;
    unsigned long long* counter;  // device scratch, zeroed by the launcher
};
void launch_dco_fixed(const DcoLaunch& a, cudaStream_t st);
// out[c * ceil(D/dd) + t] = S at min((t+1)dd, D) for row cand[c] (dco.cu).
void launch_prefix_sums(const float* X, int D, const float* q, const int64_t* cand, int nc, int dd,
                        double* out, cudaStream_t st);

struct SearchLaunch {
    const float* a1;
    const float* a2;
    uint32_t a2_16;    // (a2 - a1) in 16-byte units (VEC=4: A2 follows A1 in one allocation)
    int d1;            // physical split (A1 row stride)
    int D;
    const int32_t* ids;
    const int64_t* list_off;
    const float* Q;    // nq x D, search space
    int nq;
    const int32_t* probes;  // nq x nprobe
    int nprobe;
    int probe_lo;           // scan probe ranks probe_lo .. nprobe-1
    const double* r0;       // nullable: per-query initial radius (device)
    int K;
    int final_fd;      // 1: sqrt(s) <= r (kFd), 0: s <= r^2
    const Seg* segs;
    const double* tfac;
    int nseg, ntest, vec;
    int full;          // every segment is 32 floats (no per-line length shuffle)
    int nseg0;         // leading untested segments: lanes idle at a chunk's tail pre-walk
                       // them for the next chunk (0: no pre-walk, one prefix buffer)
    int64_t first, step;
    int warps;         // per CTA
    int slots;         // queries served concurrently per CTA
    int ctas_per_sm;
    int32_t* out_ids;
    double* out_dists;
    int32_t* out_cnt;
    unsigned long long* out_dims;
    unsigned long long* out_cand;
    unsigned long long* counter;
    const int32_t* order;  // nullable: work item w searches query order[w]
    const float* a1i;      // nullable: the interleaved A1 copy (d1 == 32, split, AD): dense prefix phase
    int f32;               // 1: certified fp32 walk + exact re-walk (full 32-float lines only)
    int lag;               // 1: overlapped chunks, lag-1 refresh schedule (ivf_search_lag_kernel)
};
void launch_ivf_search(const SearchLaunch& a, cudaStream_t st);
// CTAs of the search grid resident at once (num_sms x occupancy for this launch shape).
int64_t search_resident_ctas(const SearchLaunch& a);

// Device buffer that only grows (scratch owned by index handles).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <typename T>
    T* get(size_t count) {
        const size_t need = sizeof(T) * (count > 0 ? count : 1);
        if (need > bytes) {
            if (p) ADS_CUDA(cudaFree(p));
            p = nullptr;
            ADS_CUDA(cudaMalloc(&p, need));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Certified coarse quantizer (coarse.cu): fp32 prefilter + exact fp64 rescoring.
struct CoarseScratch {
    DevBuf approx, qc, qn2, qnrm;
    DevBuf stats;     // [rescored centroids, fallback queries] of the last launch
    int last_nq = 0;
    void release() {
        for (DevBuf* b : {&approx, &qc, &qn2, &qnrm, &stats}) b->release();
    }
};
// Per centroid table: mean mu (fp64), centred fp32 copy, |c~|^2 and max |c~|.
struct CoarseCentroids {
    double* mu = nullptr;
    float* cc = nullptr;     // fl32(c - mu)
    float* cc_tf = nullptr;  // the same rounded to TF32 (tensor-core GEMM operand)
    float* cn2 = nullptr;
    double cmax = 0.0;
    void release() {
        for (void* p : {static_cast<void*>(mu), static_cast<void*>(cc), static_cast<void*>(cc_tf),
                        static_cast<void*>(cn2)})
            if (p) cudaFree(p);
        mu = nullptr;
        cc = nullptr;
        cc_tf = nullptr;
        cn2 = nullptr;
    }
};
void coarse_center(const float* X, int n, int D, const double* mu, float* Xc, float* n2, double* nrm,
                   cudaStream_t st, bool tf32 = false);
// tc_gemm.cu: the approximate distance matrix on tcgen05 (kind::tf32) and its error factor.
bool tc_coarse_supported(int D);
double tc_coarse_gamma(int D);
void launch_tc_coarse_gemm(const float* Qc, int nq, const float* Cc, int L, int D, const float* qn2,
                           const float* cn2, float* out, cudaStream_t st);
// 3xTF32 transform on the tensor cores (tc_gemm.cu): hi/lo split, then Y = X P^T.
void launch_split_tf32(const float* x, int64_t n, float* hi, float* lo, cudaStream_t st);
// Y = X P^T on the tensor cores (3xTF32; Ph/Pl = P split into TF32 pairs).
// xh/xl: scratch for the experiment variants that pre-split X (unused by default).
void launch_tc_transform(const float* X, int64_t n, const float* Ph, const float* Pl, int D, float* Y, DevBuf& xh,
                         DevBuf& xl, cudaStream_t st);
// gemm: 0 = tensor cores when supported (D % 4 == 0), 1 = fp32 FMA on the CUDA cores.
void launch_coarse_probes_fast(const float* Q, int nq, const float* C, int L, int D, int nprobe,
                               const CoarseCentroids& cc, CoarseScratch& s, int32_t* probes, int gemm,
                               cudaStream_t st);

// Exact fp64 centroid distances (nq x L, l2_sq order) and top-nprobe by (d2, id).
void launch_coarse_dist(const float* Q, int nq, const float* C, int L, int D, double* out,
                        cudaStream_t st);
void launch_select_probes(const double* dist, int nq, int L, int nprobe, int32_t* probes,
                          cudaStream_t st);

// y = P x (fp64, reference order), P row-major dim x dim on device (double).
void launch_apply(const double* P, int dim, const float* X, int64_t n, float* Y,
                  cudaStream_t st);

// brute_force_knn: K smallest (d2, id) pairs per query.
void launch_brute_knn(const float* base, int64_t n, int D, const float* Q, int nq, int K,
                      int32_t* ids, cudaStream_t st);
// verify_theory (bench.cpp:303-392): counters[0, G) dims, [G, 2G) failures, [2G] positives
// over the ascending grid whose factor tables (delta_d = 1) are factor[g*d ..]; theory.cu.
void launch_verify_theory(const float* X, int64_t n, int d, const float* Q, int nq, int K,
                          const double* factor, int G, int32_t* ids_scratch, double* r_sq,
                          unsigned long long* counters, cudaStream_t st);

// k-means pieces (kmeans.cu).
struct KmeansOut {
    double objective;
    int iterations;
};
KmeansOut run_kmeans(const float* dX, int64_t n, int d, int k, int max_iters, uint64_t seed,
                     int init, float* dC, int32_t* dAssign, cudaStream_t st);
// Bucket layout (ivf.cpp:211-256) from an assignment: list_off (k+1), ids_flat,
// and gathered A1/A2 copies of `src` (n x D row-major by id) split at d1.
void build_lists(const int32_t* dAssign, int64_t n, int k, int64_t* dListOff, int32_t* dIds,
                 cudaStream_t st);
void gather_split(const float* src, const int32_t* dIds, int64_t n, int D, int d1, float* a1,
                  float* a2, cudaStream_t st);
// The A1 prefix (32 floats per row) re-blocked by 32-row position groups and
// 16-byte chunks (dense coalesced reads of a list run's prefixes, ivf.cu).
// Rows of `width` floats (a multiple of 32) interleaved by 32-row position groups, 16-byte
// chunk by chunk within each 32-float segment (the scan's dense phases, ivf.cu).
void interleave_rows(const float* in, int64_t n, int width, float* out, cudaStream_t st);
// out[i] = keep[asg[i]] ? asg[i] : k (lists a shard does not own sort after every owned one).
void mask_assignment(const int32_t* dAssign, int64_t n, const uint8_t* dKeep, int k, int32_t* dOut,
                     cudaStream_t st);

// Per query, K smallest (dist, id) pairs among G lists of K ([G][nq][K]).
void launch_merge_topk(const double* dists, const int32_t* ids, int G, int nq, int K,
                       int32_t* out_ids, double* out_dists, int32_t* out_cnt, cudaStream_t st);

// L2-locality order of a query batch: stable sort by rank[nearest list].
void launch_query_order(const int32_t* probes, int nq, int nprobe, const int32_t* rank, int k,
                        DevBuf& scratch, int32_t* order, cudaStream_t st);
// Longest-first order of a query batch: descending candidate count over probe
// ranks [probe_lo, nprobe) (shortens the tail of the persistent scan grid).
void launch_query_order_work(const int32_t* probes, int nq, int nprobe, int probe_lo, const int64_t* list_off,
                             DevBuf& scratch, int32_t* order, cudaStream_t st);
// Greedy nearest-neighbour chain over the centroids (host, fp32 heuristic):
// rank[c] = position of list c in the chain.
std::vector<int32_t> centroid_chain_rank(const float* C, int k, int D);

int num_sms();

}  // namespace ads

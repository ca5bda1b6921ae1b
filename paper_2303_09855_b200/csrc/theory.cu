// Fixed-threshold verification study (verify_theory, src/bench.cpp:303-392)
// on the GPU.  Per query, r_sq is the exact K-th smallest squared distance
// over all n objects (the brute-force select's K-th entry, rescored with
// the same fp64 index-order sum); then every (query, object) pair gets one
// delta_d = 1 adaptive comparison per epsilon0 of an ascending grid:
// reject_at[g] = the first d in [1, D) with s_d > factor_g[d] * r_sq.  A
// larger epsilon0 never rejects earlier, so the rejected grid entries of a
// pair are always a prefix [0, fa) and one pass over d serves the whole
// grid, as in the reference.  Counters are integers (exact), the ratios are
// formed on the host exactly as the reference forms them.
#include "engine.hpp"

namespace ads {
namespace {

constexpr int kTheoryThreads = 256;

// r_sq[q] = l2_sq(X[ids[q*K + K-1]], Q[q]) in index order (dco.hpp:86-93).
__global__ void kth_dist_kernel(const float* __restrict__ X, int d, const float* __restrict__ Q,
                                const int32_t* __restrict__ ids, int K, int nq, double* __restrict__ r_sq) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const float* o = X + static_cast<int64_t>(ids[static_cast<int64_t>(q) * K + K - 1]) * d;
    const float* qv = Q + static_cast<int64_t>(q) * d;
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = sq_diff_acc(s, o[k], static_cast<double>(qv[k]));
    r_sq[q] = s;
}

// One thread per (query, object); block = kTheoryThreads objects of one query.
// counters: [0, G) dims, [G, 2G) failures, [2G] positives.
__global__ void __launch_bounds__(kTheoryThreads)
theory_kernel(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ Q, int q0,
              const double* __restrict__ r_sq_q, const double* __restrict__ factor, int G,
              unsigned long long* __restrict__ counters) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem_raw);  // 2G + 1
    double* qs = reinterpret_cast<double*>(acc + 2 * G + 1);                     // d
    const int q = q0 + static_cast<int>(blockIdx.y);
    for (int i = threadIdx.x; i < 2 * G + 1; i += blockDim.x) acc[i] = 0;
    for (int k = threadIdx.x; k < d; k += blockDim.x) qs[k] = static_cast<double>(Q[static_cast<int64_t>(q) * d + k]);
    __syncthreads();
    const double r_sq = r_sq_q[q];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        const float* o = X + i * d;
        double s = 0.0;
        int fa = 0;  // first grid entry not yet rejected
        for (int dd = 1; dd < d; ++dd) {
            s = sq_diff_acc(s, o[dd - 1], qs[dd - 1]);
            while (fa < G && s > __dmul_rn(factor[static_cast<int64_t>(fa) * d + dd], r_sq)) {
                atomicAdd(&acc[fa], static_cast<unsigned long long>(dd));
                ++fa;
            }
        }
        s = sq_diff_acc(s, o[d - 1], qs[d - 1]);  // the exact d2 (bench.cpp:336)
        const bool positive = s <= r_sq;
        for (int g = fa; g < G; ++g) atomicAdd(&acc[g], static_cast<unsigned long long>(d));
        if (positive) {
            for (int g = 0; g < fa; ++g) atomicAdd(&acc[G + g], 1ull);
            atomicAdd(&acc[2 * G], 1ull);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * G + 1; k += blockDim.x)
        if (acc[k]) atomicAdd(&counters[k], acc[k]);
}

}  // namespace

void launch_verify_theory(const float* X, int64_t n, int d, const float* Q, int nq, int K,
                          const double* factor, int G, int32_t* ids_scratch, double* r_sq,
                          unsigned long long* counters, cudaStream_t st) {
    ADS_CUDA(cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * (2 * G + 1), st));
    if (nq <= 0 || n <= 0) return;
    launch_brute_knn(X, n, d, Q, nq, K, ids_scratch, st);
    kth_dist_kernel<<<(nq + 127) / 128, 128, 0, st>>>(X, d, Q, ids_scratch, K, nq, r_sq);
    ADS_LAUNCH_CHECK();
    const size_t smem = sizeof(unsigned long long) * (2 * G + 1) + sizeof(double) * d;
    if (smem > 200 * 1024) throw std::invalid_argument("verify_theory: dimension too large");
    ADS_CUDA(cudaFuncSetAttribute(theory_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    for (int q0 = 0; q0 < nq; q0 += 65535) {
        const int nb = nq - q0 < 65535 ? nq - q0 : 65535;
        dim3 grid(static_cast<unsigned>((n + kTheoryThreads - 1) / kTheoryThreads), static_cast<unsigned>(nb));
        theory_kernel<<<grid, kTheoryThreads, smem, st>>>(X, n, d, Q, q0, r_sq, factor, G, counters);
        ADS_LAUNCH_CHECK();
    }
}

}  // namespace ads

// Random orthogonal transform on the GPU: y = P x with the reference's
// arithmetic (transform.cpp:103-117, 131-149): fp64 P, fp64 products and
// sums in ascending j, one rounding each, fp32 store.  The result is
// bit-identical to adsann::apply / apply_dataset.  apply_transpose
// (transform.cpp:119-129) is the same kernel on P^T (acc[j] += P[i][j]*x_i,
// i ascending).  Also: brute-force exact k-NN by fp64 distance tiles +
// per-row pair select (bench.cpp:31-61).
#include "engine.hpp"

namespace ads {

namespace {

constexpr int kRows = 64;   // output coordinates per CTA (one per thread row)
constexpr int kVecs = 32;   // vectors per CTA
constexpr int kVPT = 8;     // vectors per thread
constexpr int kJ = 32;      // j per stage

__global__ void __launch_bounds__(256) apply_kernel(const double* __restrict__ P, int dim,
                                                    const float* __restrict__ X, int64_t n,
                                                    float* __restrict__ Y) {
    __shared__ double ps[kRows][kJ + 1];
    __shared__ double xs[kVecs][kJ];
    const int tr = threadIdx.x & 63;   // row within tile
    const int tv = threadIdx.x >> 6;   // vector group (0..3)
    const int i0 = blockIdx.x * kRows;
    const int64_t v0 = static_cast<int64_t>(blockIdx.y) * kVecs;
    double acc[kVPT];
#pragma unroll
    for (int a = 0; a < kVPT; ++a) acc[a] = 0.0;
    for (int j0 = 0; j0 < dim; j0 += kJ) {
        const int len = dim - j0 < kJ ? dim - j0 : kJ;
        for (int idx = threadIdx.x; idx < kRows * kJ; idx += 256) {
            const int r = idx / kJ, k = idx % kJ;
            ps[r][k] = (i0 + r < dim && k < len) ? P[static_cast<int64_t>(i0 + r) * dim + j0 + k] : 0.0;
        }
        for (int idx = threadIdx.x; idx < kVecs * kJ; idx += 256) {
            const int v = idx / kJ, k = idx % kJ;
            xs[v][k] = (v0 + v < n && k < len) ? static_cast<double>(X[(v0 + v) * dim + j0 + k]) : 0.0;
        }
        __syncthreads();
        for (int k = 0; k < len; ++k) {
            const double p = ps[tr][k];
#pragma unroll
            for (int a = 0; a < kVPT; ++a) acc[a] = __dadd_rn(acc[a], __dmul_rn(p, xs[tv * kVPT + a][k]));
        }
        __syncthreads();
    }
    if (i0 + tr < dim) {
#pragma unroll
        for (int a = 0; a < kVPT; ++a) {
            const int64_t v = v0 + tv * kVPT + a;
            if (v < n) Y[v * dim + i0 + tr] = static_cast<float>(acc[a]);
        }
    }
}

}  // namespace

void launch_apply(const double* P, int dim, const float* X, int64_t n, float* Y, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t gy = (n + kVecs - 1) / kVecs;
    for (int64_t off = 0; off < gy; off += 65535) {  // grid.y limit
        const int64_t cnt = gy - off < 65535 ? gy - off : 65535;
        dim3 grid((dim + kRows - 1) / kRows, static_cast<unsigned>(cnt));
        const int64_t vbase = off * kVecs;
        apply_kernel<<<grid, 256, 0, st>>>(P, dim, X + vbase * dim, n - vbase, Y + vbase * dim);
        ADS_LAUNCH_CHECK();
    }
}

void launch_brute_knn(const float* base, int64_t n, int D, const float* Q, int nq, int K,
                      int32_t* ids, cudaStream_t st) {
    if (n > 0x7fffffff) throw std::invalid_argument("brute_force_knn: n too large");
    // Distances for a batch of queries against the whole base, then an exact
    // (d2, id) top-K per row.  Batch sized to ~1 GiB of fp64 scratch.
    int64_t batch = (int64_t(1) << 27) / (n > 0 ? n : 1);
    if (batch < 1) batch = 1;
    if (batch > nq) batch = nq;
    double* dist = nullptr;
    ADS_CUDA(cudaMallocAsync(&dist, sizeof(double) * batch * n, st));
    for (int64_t q0 = 0; q0 < nq; q0 += batch) {
        const int bq = static_cast<int>(nq - q0 < batch ? nq - q0 : batch);
        // rows = queries, "centroids" = base points: l2_sq(ds.row(i), q) is the same
        // set of squares as l2_sq(q, ds.row(i)).
        launch_coarse_dist(Q + q0 * D, bq, base, static_cast<int>(n), D, dist, st);
        launch_select_probes(dist, bq, static_cast<int>(n), K, ids + q0 * K, st);
    }
    ADS_CUDA(cudaFreeAsync(dist, st));
}

}  // namespace ads

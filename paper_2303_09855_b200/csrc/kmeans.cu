// GPU k-means and IVF bucket layout (ivf.cpp:36-258), reproducing the
// reference bit for bit:
//   * k-means++ seeding (ivf.cpp:62-117): per round the min-distance update
//     is a parallel exact fp64 pass; the CDF walk is inherently sequential
//     (cum += min_d2[i] in index order) and runs on one GPU thread, with the
//     reference's Rng (SplitMix64) advanced on the device.
//   * Lloyd (ivf.cpp:138-186): exact fp64 nearest-centroid argmin (ties to
//     the lowest index), objective as a sequential fp64 sum, centroid sums
//     per (cluster, coordinate) in ascending point id, empty clusters
//     reseeded from the farthest non-stolen point, relative-change stop.
//   * layout (ivf.cpp:211-256): stable sort of ids by bucket (CUB radix
//     sort) and gathered A1/A2 copies.
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "engine.hpp"

namespace ads {

namespace {

constexpr uint64_t kTagKmeans = 0x6b1febc8d1a07445ULL;  // rng.hpp:29

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

struct DevRng {  // rng.hpp:36-70 (only next_u64 / uniform / below are drawn here)
    uint64_t seed, counter;
};

__device__ __forceinline__ uint64_t next_u64(DevRng* r) {
    r->counter += 1;
    return mix64(r->seed + r->counter * 0x9E3779B97F4A7C15ULL);
}

struct KppState {
    DevRng rng;
    int64_t pick;
};

__global__ void kpp_first_kernel(KppState* st, int64_t n) {
    st->pick = static_cast<int64_t>(next_u64(&st->rng) % static_cast<uint64_t>(n));
}

__global__ void copy_pick_kernel(const float* X, int D, const KppState* st, float* crow,
                                 unsigned char* chosen) {
    const int64_t p = st->pick;
    for (int j = threadIdx.x; j < D; j += blockDim.x) crow[j] = X[p * D + j];
    if (threadIdx.x == 0) chosen[p] = 1;
}

__global__ void min_update_kernel(const double* d2, double* min_d2, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n && d2[i] < min_d2[i]) min_d2[i] = d2[i];
}

// ivf.cpp:85-115.  The sequential fp64 sum is inherently serial; thread 0
// runs the dependent add chain while the other threads stage the next chunk
// of min_d2 in shared memory.  The walk `cum += min_d2[i]; if (cum > u)`
// revisits the same rounded prefix sums, which are non-decreasing, so the
// prefix of the first pass is stored and the walk becomes a binary search.
constexpr int kPickThreads = 256;
constexpr int kPickChunk = 2048;

__global__ void __launch_bounds__(kPickThreads) kpp_pick_kernel(KppState* st,
                                                                const double* __restrict__ min_d2,
                                                                const unsigned char* __restrict__ chosen,
                                                                double* __restrict__ cum, int64_t n) {
    __shared__ double buf[2][kPickChunk];
    __shared__ double s_total;
    const int tid = threadIdx.x;
    const int64_t nchunks = (n + kPickChunk - 1) / kPickChunk;
    for (int i = tid; i < kPickChunk; i += kPickThreads) buf[0][i] = i < n ? min_d2[i] : 0.0;
    __syncthreads();
    double total = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t base = c * kPickChunk;
        if (tid == 0) {
            const double* b = buf[c & 1];
            const int len = static_cast<int>(n - base < kPickChunk ? n - base : kPickChunk);
            int i = 0;
            for (; i + 8 <= len; i += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    total = __dadd_rn(total, b[i + u]);
                    cum[base + i + u] = total;
                }
            }
            for (; i < len; ++i) {
                total = __dadd_rn(total, b[i]);
                cum[base + i] = total;
            }
        } else if (c + 1 < nchunks) {
            const int64_t nb = base + kPickChunk;
            for (int i = tid - 1; i < kPickChunk; i += kPickThreads - 1)
                buf[(c + 1) & 1][i] = nb + i < n ? min_d2[nb + i] : 0.0;
        }
        __syncthreads();
    }
    if (tid == 0) s_total = total;
    __syncthreads();
    if (tid != 0) return;
    total = s_total;
    int64_t pick = -1;
    if (total > 0.0) {
        const double u = __dmul_rn(static_cast<double>(next_u64(&st->rng) >> 11) * 0x1.0p-53, total);
        int64_t lo = 0, hi = n;  // first i with cum[i] > u, or n
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cum[mid] > u) hi = mid;
            else lo = mid + 1;
        }
        if (lo < n) pick = lo;
        if (pick < 0)
            for (int64_t i = n - 1; i >= 0; --i)
                if (min_d2[i] > 0.0) {
                    pick = i;
                    break;
                }
    }
    if (pick < 0) {
        for (int64_t i = 0; i < n; ++i)
            if (!chosen[i]) {
                pick = i;
                break;
            }
        if (pick < 0) pick = 0;
    }
    st->pick = pick;
}

// Exact nearest centroid for kPT points per CTA (ivf.cpp:36-60).
constexpr int kAT = 128;  // centroids per tile (one per thread)
constexpr int kPT = 16;   // points per CTA
constexpr int kAK = 32;

__global__ void __launch_bounds__(kAT) assign_kernel(const float* __restrict__ X, int64_t n, int D,
                                                     const float* __restrict__ C, int k,
                                                     int32_t* __restrict__ assign,
                                                     double* __restrict__ best_d2) {
    __shared__ float ct[kAT * (kAK + 1)];
    __shared__ double pt[kPT][kAK];
    __shared__ double red_d[kAT / 32][kPT];
    __shared__ int red_i[kAT / 32][kPT];
    __shared__ double s_best[kPT];
    __shared__ int s_arg[kPT];
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kPT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kPT) {
        s_best[tid] = __builtin_huge_val();
        s_arg[tid] = 0;
    }
    for (int c0 = 0; c0 < k; c0 += kAT) {
        double acc[kPT];
#pragma unroll
        for (int i = 0; i < kPT; ++i) acc[i] = 0.0;
        for (int d0 = 0; d0 < D; d0 += kAK) {
            const int len = D - d0 < kAK ? D - d0 : kAK;
            for (int idx = tid; idx < kAT * kAK; idx += kAT) {
                const int c = idx / kAK, kk = idx % kAK;
                ct[c * (kAK + 1) + kk] =
                    (c0 + c < k && kk < len) ? C[static_cast<int64_t>(c0 + c) * D + d0 + kk] : 0.f;
            }
            for (int idx = tid; idx < kPT * kAK; idx += kAT) {
                const int pp = idx / kAK, kk = idx % kAK;
                pt[pp][kk] = (p0 + pp < n && kk < len) ? static_cast<double>(X[(p0 + pp) * D + d0 + kk]) : 0.0;
            }
            __syncthreads();
            for (int kk = 0; kk < len; ++kk) {
                const float cv = ct[tid * (kAK + 1) + kk];
                // l2_sq(x, centroid): diff = x - c; the square is the same for c - x.
#pragma unroll
                for (int pp = 0; pp < kPT; ++pp) {
                    const double diff = __dsub_rn(pt[pp][kk], static_cast<double>(cv));
                    acc[pp] = __dadd_rn(acc[pp], __dmul_rn(diff, diff));
                }
            }
            __syncthreads();
        }
        // argmin over this tile's centroids, ties -> lowest index, then merge (strict <).
#pragma unroll
        for (int pp = 0; pp < kPT; ++pp) {
            double v = (c0 + tid < k) ? acc[pp] : __builtin_huge_val();
            int vi = c0 + tid;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
                if (ov < v || (ov == v && oi < vi)) {
                    v = ov;
                    vi = oi;
                }
            }
            if (lane == 0) {
                red_d[warp][pp] = v;
                red_i[warp][pp] = vi;
            }
        }
        __syncthreads();
        if (tid < kPT) {
            double v = red_d[0][tid];
            int vi = red_i[0][tid];
            for (int w = 1; w < kAT / 32; ++w)
                if (red_d[w][tid] < v || (red_d[w][tid] == v && red_i[w][tid] < vi)) {
                    v = red_d[w][tid];
                    vi = red_i[w][tid];
                }
            if (v < s_best[tid]) {
                s_best[tid] = v;
                s_arg[tid] = vi;
            }
        }
        __syncthreads();
    }
    if (tid < kPT && p0 + tid < n) {
        assign[p0 + tid] = s_arg[tid];
        best_d2[p0 + tid] = s_best[tid];
    }
}

__global__ void seq_sum_kernel(const double* __restrict__ v, int64_t n, double* out) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, v[i]);
    *out = s;
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) v[i] = static_cast<int32_t>(i);
}

__global__ void count_kernel(const int32_t* a, int64_t n, int64_t* counts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) atomicAdd(reinterpret_cast<unsigned long long*>(counts + a[i]), 1ull);
}

// ivf.cpp:142-157: per (cluster, coordinate) fp64 sum over members in
// ascending id, centroid = float(sum / count) for non-empty clusters.
__global__ void update_kernel(const float* __restrict__ X, int D, const int64_t* __restrict__ off,
                              const int32_t* __restrict__ ids, int k, float* __restrict__ C) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(k) * D) return;
    const int c = static_cast<int>(t / D), j = static_cast<int>(t % D);
    const int64_t b = off[c], e = off[c + 1];
    if (b == e) return;
    double s = 0.0;
    for (int64_t m = b; m < e; ++m) s = __dadd_rn(s, static_cast<double>(X[static_cast<int64_t>(ids[m]) * D + j]));
    C[static_cast<int64_t>(c) * D + j] = static_cast<float>(__ddiv_rn(s, static_cast<double>(e - b)));
}

// ivf.cpp:163-171: farthest non-stolen point (strict >, first index wins).
__global__ void argmax_kernel(const double* __restrict__ v, const unsigned char* __restrict__ stolen,
                              int64_t n, int64_t* out) {
    __shared__ double sd[1024];
    __shared__ int64_t si[1024];
    double best = -1.0;
    int64_t bi = -1;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (!stolen[i] && v[i] > best) {
            best = v[i];
            bi = i;
        }
    sd[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double ov = sd[threadIdx.x + s];
            const int64_t oi = si[threadIdx.x + s];
            if (oi >= 0 && (si[threadIdx.x] < 0 || ov > sd[threadIdx.x] ||
                            (ov == sd[threadIdx.x] && oi < si[threadIdx.x]))) {
                sd[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = si[0];
}

__global__ void steal_copy_kernel(const float* X, int D, const int64_t* far_i, float* crow,
                                  unsigned char* stolen) {
    const int64_t f = *far_i;
    if (f < 0) return;
    for (int j = threadIdx.x; j < D; j += blockDim.x) crow[j] = X[f * D + j];
    if (threadIdx.x == 0) stolen[f] = 1;
}

__global__ void gather_split_kernel(const float* __restrict__ src, const int32_t* __restrict__ ids,
                                    int64_t n, int D, int d1, float* __restrict__ a1,
                                    float* __restrict__ a2) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n * D) return;
    const int64_t p = t / D;
    const int j = static_cast<int>(t % D);
    const float v = src[static_cast<int64_t>(ids[p]) * D + j];
    if (j < d1) a1[p * d1 + j] = v;
    else a2[p * (D - d1) + (j - d1)] = v;
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

int key_bits(int k) {
    int b = 1;
    while ((1ll << b) < k) ++b;
    return b;
}

void assign_points(const float* X, int64_t n, int D, const float* C, int k, int32_t* asg,
                   double* best, cudaStream_t st) {
    const int64_t blocks = (n + kPT - 1) / kPT;
    assign_kernel<<<static_cast<unsigned>(blocks), kAT, 0, st>>>(X, n, D, C, k, asg, best);
    ADS_LAUNCH_CHECK();
}

double seq_sum(const double* v, int64_t n, double* scratch, cudaStream_t st) {
    seq_sum_kernel<<<1, 1, 0, st>>>(v, n, scratch);
    ADS_LAUNCH_CHECK();
    double h = 0.0;
    ADS_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(double), cudaMemcpyDeviceToHost, st));
    ADS_CUDA(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

void build_lists(const int32_t* dAssign, int64_t n, int k, int64_t* dListOff, int32_t* dIds,
                 cudaStream_t st) {
    int32_t *keys_out = nullptr, *vals_in = nullptr;
    int64_t* counts = nullptr;
    ADS_CUDA(cudaMallocAsync(&keys_out, sizeof(int32_t) * (n > 0 ? n : 1), st));
    ADS_CUDA(cudaMallocAsync(&vals_in, sizeof(int32_t) * (n > 0 ? n : 1), st));
    ADS_CUDA(cudaMallocAsync(&counts, sizeof(int64_t) * (k + 1), st));
    iota_kernel<<<blocks_for(n, 256), 256, 0, st>>>(vals_in, n);
    size_t tmp_bytes = 0;
    ADS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dAssign, keys_out, vals_in, dIds,
                                             static_cast<int>(n), 0, key_bits(k), st));
    void* tmp = nullptr;
    ADS_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    ADS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dAssign, keys_out, vals_in, dIds,
                                             static_cast<int>(n), 0, key_bits(k), st));
    ADS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (k + 1), st));
    count_kernel<<<blocks_for(n, 256), 256, 0, st>>>(dAssign, n, counts);
    size_t scan_bytes = 0;
    ADS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, dListOff, k + 1, st));
    void* scan_tmp = nullptr;
    ADS_CUDA(cudaMallocAsync(&scan_tmp, scan_bytes, st));
    ADS_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, dListOff, k + 1, st));
    ADS_CUDA(cudaFreeAsync(scan_tmp, st));
    ADS_CUDA(cudaFreeAsync(tmp, st));
    ADS_CUDA(cudaFreeAsync(counts, st));
    ADS_CUDA(cudaFreeAsync(vals_in, st));
    ADS_CUDA(cudaFreeAsync(keys_out, st));
    ADS_LAUNCH_CHECK();
}

namespace {
__global__ void mask_assignment_kernel(const int32_t* __restrict__ asg, int64_t n,
                                       const uint8_t* __restrict__ keep, int k, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int32_t c = asg[i];
    out[i] = keep[c] ? c : k;
}
}  // namespace

namespace {
// out[(((g * S + s) * 8 + c) * 32 + r) * 4 + e] = in[(g * 32 + r) * 32 S + s * 32 + c * 4 + e]
// (rows of 32 S floats, S = 32-float segments per row): position group g's 32 rows
// interleaved by 16-byte chunk, segment by segment, so lane r of a warp reading chunk c
// of segment s of rows 32g .. 32g+31 issues one contiguous 512-byte request (zeros past n).
__global__ void interleave_rows_kernel(const float4* __restrict__ in, int64_t n, int S,
                                       float4* __restrict__ out, int64_t groups) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= groups * S * 256) return;
    const int64_t gs = t >> 8;  // g * S + s
    const int64_t g = gs / S;
    const int s = static_cast<int>(gs - g * S);
    const int c = static_cast<int>((t >> 5) & 7), r = static_cast<int>(t & 31);
    const int64_t p = g * 32 + r;
    out[t] = p < n ? in[(p * S + s) * 8 + c] : make_float4(0.f, 0.f, 0.f, 0.f);
}
}  // namespace

void interleave_rows(const float* in, int64_t n, int width, float* out, cudaStream_t st) {
    const int64_t groups = (n + 31) / 32;
    if (groups <= 0 || width <= 0) return;
    if (width % 32) throw std::invalid_argument("interleave_rows: width must be a multiple of 32");
    const int S = width / 32;
    interleave_rows_kernel<<<blocks_for(groups * S * 256, 256), 256, 0, st>>>(
        reinterpret_cast<const float4*>(in), n, S, reinterpret_cast<float4*>(out), groups);
    ADS_LAUNCH_CHECK();
}

void mask_assignment(const int32_t* dAssign, int64_t n, const uint8_t* dKeep, int k, int32_t* dOut,
                     cudaStream_t st) {
    if (n <= 0) return;
    mask_assignment_kernel<<<blocks_for(n, 256), 256, 0, st>>>(dAssign, n, dKeep, k, dOut);
    ADS_LAUNCH_CHECK();
}

void gather_split(const float* src, const int32_t* dIds, int64_t n, int D, int d1, float* a1,
                  float* a2, cudaStream_t st) {
    if (n <= 0) return;
    gather_split_kernel<<<blocks_for(n * D, 256), 256, 0, st>>>(src, dIds, n, D, d1, a1, a2);
    ADS_LAUNCH_CHECK();
}

KmeansOut run_kmeans(const float* dX, int64_t n, int d, int k, int max_iters, uint64_t seed,
                     int init, float* dC, int32_t* dAssign, cudaStream_t st) {
    // ivf.cpp:122-123
    if (k < 1) throw std::invalid_argument("kmeans: k must be >= 1");
    if (k > n) throw std::invalid_argument("kmeans: k exceeds the number of points");
    if (n > 0x7fffffff) throw std::invalid_argument("kmeans: n too large");
    double *min_d2 = nullptr, *dtmp = nullptr, *best = nullptr, *scalar = nullptr;
    unsigned char* flags = nullptr;
    KppState* kst = nullptr;
    int64_t *off = nullptr, *far_i = nullptr;
    int32_t* ids = nullptr;
    ADS_CUDA(cudaMallocAsync(&min_d2, sizeof(double) * n, st));
    ADS_CUDA(cudaMallocAsync(&dtmp, sizeof(double) * n, st));
    ADS_CUDA(cudaMallocAsync(&best, sizeof(double) * n, st));
    ADS_CUDA(cudaMallocAsync(&scalar, sizeof(double), st));
    ADS_CUDA(cudaMallocAsync(&flags, n, st));
    ADS_CUDA(cudaMallocAsync(&kst, sizeof(KppState), st));
    ADS_CUDA(cudaMallocAsync(&off, sizeof(int64_t) * (k + 1), st));
    ADS_CUDA(cudaMallocAsync(&far_i, sizeof(int64_t), st));
    ADS_CUDA(cudaMallocAsync(&ids, sizeof(int32_t) * n, st));

    // ---- seeding.  Rng::for_stream(seed, kKmeans) (ivf.cpp:127, rng.hpp:42-44)
    KppState h{};
    {
        uint64_t z = seed ^ kTagKmeans;
        z ^= z >> 30;
        z *= 0xBF58476D1CE4E5B9ULL;
        z ^= z >> 27;
        z *= 0x94D049BB133111EBULL;
        z ^= z >> 31;
        h.rng.seed = z;
        h.rng.counter = 0;
    }
    ADS_CUDA(cudaMemcpyAsync(kst, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    ADS_CUDA(cudaMemsetAsync(flags, 0, n, st));
    if (init == 0) {
        std::vector<double> inf(1, __builtin_huge_val());
        // fill min_d2 with +inf via a pattern copy of one value
        const double hinf = __builtin_huge_val();
        std::vector<double> buf(static_cast<size_t>(n), hinf);
        ADS_CUDA(cudaMemcpyAsync(min_d2, buf.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
        kpp_first_kernel<<<1, 1, 0, st>>>(kst, n);
        for (int c = 0;; ++c) {
            float* crow = dC + static_cast<int64_t>(c) * d;
            copy_pick_kernel<<<1, 128, 0, st>>>(dX, d, kst, crow, flags);
            if (c + 1 == k) break;
            launch_coarse_dist(crow, 1, dX, static_cast<int>(n), d, dtmp, st);
            min_update_kernel<<<blocks_for(n, 256), 256, 0, st>>>(dtmp, min_d2, n);
            kpp_pick_kernel<<<1, kPickThreads, 0, st>>>(kst, min_d2, flags, dtmp, n);
        }
        ADS_CUDA(cudaStreamSynchronize(st));  // buf must outlive the copy
        ADS_LAUNCH_CHECK();
    } else {
        // k distinct seeded samples: partial Fisher-Yates over ids on the host
        // with the same Rng stream (documented deviation).
        std::vector<int32_t> perm(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) perm[i] = static_cast<int32_t>(i);
        uint64_t ctr = 0;
        auto nxt = [&]() {
            ++ctr;
            uint64_t z = h.rng.seed + ctr * 0x9E3779B97F4A7C15ULL;
            z ^= z >> 30;
            z *= 0xBF58476D1CE4E5B9ULL;
            z ^= z >> 27;
            z *= 0x94D049BB133111EBULL;
            z ^= z >> 31;
            return z;
        };
        for (int c = 0; c < k; ++c) {
            const int64_t j = c + static_cast<int64_t>(nxt() % static_cast<uint64_t>(n - c));
            std::swap(perm[c], perm[j]);
            ADS_CUDA(cudaMemcpyAsync(dC + static_cast<int64_t>(c) * d, dX + static_cast<int64_t>(perm[c]) * d,
                                     sizeof(float) * d, cudaMemcpyDeviceToDevice, st));
        }
        ADS_CUDA(cudaStreamSynchronize(st));
    }

    // ---- Lloyd
    KmeansOut out{0.0, 0};
    double prev_obj = __builtin_huge_val();
    std::vector<int64_t> hoff(static_cast<size_t>(k) + 1);
    for (int iter = 0; iter < max_iters; ++iter) {
        assign_points(dX, n, d, dC, k, dAssign, best, st);
        const double obj = seq_sum(best, n, scalar, st);
        out.iterations = iter + 1;
        build_lists(dAssign, n, k, off, ids, st);
        const int64_t tot = static_cast<int64_t>(k) * d;
        update_kernel<<<blocks_for(tot, 256), 256, 0, st>>>(dX, d, off, ids, k, dC);
        ADS_LAUNCH_CHECK();
        ADS_CUDA(cudaMemcpyAsync(hoff.data(), off, sizeof(int64_t) * (k + 1), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        bool any_empty = false;
        for (int c = 0; c < k; ++c) any_empty = any_empty || hoff[c] == hoff[c + 1];
        if (any_empty) {
            ADS_CUDA(cudaMemsetAsync(flags, 0, n, st));  // "stolen"
            for (int c = 0; c < k; ++c) {
                if (hoff[c] != hoff[c + 1]) continue;
                argmax_kernel<<<1, 1024, 0, st>>>(best, flags, n, far_i);
                steal_copy_kernel<<<1, 128, 0, st>>>(dX, d, far_i, dC + static_cast<int64_t>(c) * d, flags);
            }
            ADS_LAUNCH_CHECK();
        }
        if (prev_obj < __builtin_huge_val()) {  // ivf.cpp:178-184
            const double denom = obj > 1e-30 ? obj : 1e-30;
            if (std::fabs(prev_obj - obj) / denom < 1e-4) break;
        }
        prev_obj = obj;
    }
    assign_points(dX, n, d, dC, k, dAssign, best, st);
    out.objective = seq_sum(best, n, scalar, st);

    ADS_CUDA(cudaFreeAsync(min_d2, st));
    ADS_CUDA(cudaFreeAsync(dtmp, st));
    ADS_CUDA(cudaFreeAsync(best, st));
    ADS_CUDA(cudaFreeAsync(scalar, st));
    ADS_CUDA(cudaFreeAsync(flags, st));
    ADS_CUDA(cudaFreeAsync(kst, st));
    ADS_CUDA(cudaFreeAsync(off, st));
    ADS_CUDA(cudaFreeAsync(far_i, st));
    ADS_CUDA(cudaFreeAsync(ids, st));
    ADS_CUDA(cudaStreamSynchronize(st));
    return out;
}

}  // namespace ads

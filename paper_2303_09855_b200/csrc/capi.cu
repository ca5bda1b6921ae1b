// C-ABI implementation (include/adsann_b200.h).  Host orchestration only:
// argument validation with the reference's error classes, device buffers,
// segment plans, and the kernel launch sequence.  No compute runs on the
// host: every DCO, distance, transform, selection and k-means step is a
// kernel in this library.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/adsann_b200.h"
#include "engine.hpp"
#include "host.hpp"

namespace ads {
void synth(const ads_synth_desc& s, float* out, int32_t* comp_out);
void synth_rows(const ads_synth_desc& s, int64_t row_lo, int64_t count, int64_t stride, float* out,
                int32_t* comp_out);

int num_sms() {
    int dev = 0;
    ADS_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int v = 0;
    ADS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = v;
    return v;
}
}  // namespace ads

using namespace ads;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return ADS_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return ADS_INVALID_ARGUMENT;
    } catch (const CudaError& e) {
        g_err = e.what();
        return ADS_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ADS_RUNTIME_ERROR;
    }
}

}  // namespace

namespace ads {
// for the host-only translation units (ivf_io.cpp) that report through ads_last_error
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace ads

namespace {
void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

template <typename T>
T* dev_upload(const T* h, size_t count, cudaStream_t st) {
    T* d = nullptr;
    ADS_CUDA(cudaMalloc(&d, sizeof(T) * (count > 0 ? count : 1)));
    if (count) ADS_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    return d;
}
// Upload into a scratch DevBuf (freed with it, also when a later step throws).
template <typename T>
T* buf_upload(DevBuf& b, const T* h, size_t count, cudaStream_t st) {
    T* d = b.get<T>(count);
    if (count) ADS_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    return d;
}
}  // namespace

struct ads_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    unsigned long long* counter = nullptr;
    void* flush = nullptr;
    size_t flush_bytes = 0;
    std::mutex mu;
    // single-DCO scratch (ads_dco): one pinned staging block + one device block
    void* h_stage = nullptr;
    DevBuf d_stage;
    std::map<std::tuple<int, int, double, int>, std::unique_ptr<DevSegPlan>> dco_plans;
    void use() const { ADS_CUDA(cudaSetDevice(device)); }
};

struct ads_transform {
    ads_ctx* ctx = nullptr;
    int dim = 0;
    double* P = nullptr;
    double* PT = nullptr;
    DevBuf xin, yout;
    DevBuf ph, pl, xh, xl;  // 3xTF32 tensor-core path: P and X as TF32 hi/lo pairs
    bool split_ready = false;
    ~ads_transform() {
        if (P) cudaFree(P);
        if (PT) cudaFree(PT);
    }
};

struct PlanKey {
    int mode;
    double eps0;
    int dd;
    bool operator<(const PlanKey& o) const {
        return std::tie(mode, eps0, dd) < std::tie(o.mode, o.eps0, o.dd);
    }
};

// A1 and A2 of one space share one allocation, A2 starting at the next 128-byte
// boundary after A1, so the search kernel addresses a line of either array with
// a single 32-bit offset (16-byte units) from the A1 base.
static void alloc_split_pair(size_t n, int d1p, int d2p, float** a1, float** a2) {
    const size_t n1 = (n * static_cast<size_t>(d1p) + 31) / 32 * 32;
    const size_t n2 = n * static_cast<size_t>(d2p);
    ADS_CUDA(cudaMalloc(a1, sizeof(float) * (n1 + (n2 > 0 ? n2 : 1))));
    *a2 = *a1 + n1;
}

struct ads_ivf {
    ads_ctx* ctx = nullptr;
    int n = 0, d = 0, k = 0, d1 = 0, layout = 0, d1p = 0;
    int nonempty = 0;  // lists holding rows (a shard's own lists): the scan heuristics' list length
    uint64_t seed = 0;
    bool has_raw = false;
    float *cent_t = nullptr, *cent_raw = nullptr;
    int64_t* list_off = nullptr;
    int32_t* ids = nullptr;
    float *a1_t = nullptr, *a2_t = nullptr, *a1_raw = nullptr, *a2_raw = nullptr;
    float* a1i_t = nullptr;  // A1 interleaved by 32-row groups (dense prefix phase of the scan)
    double* P = nullptr;
    std::map<PlanKey, std::unique_ptr<DevSegPlan>> plans;
    DevBuf dist, probes, qrot, qin_t, qin_raw, o_ids, o_dists, o_cnt, o_dims, o_cand;
    DevBuf ph, pl, qh, ql;  // rotate_mode 1: P and the queries as TF32 hi/lo pairs
    DevBuf r0buf;           // host-API copy of opts.r0
    bool p_split = false;
    int32_t* chain_rank = nullptr;  // L2-locality rank of each list (host chain over centroids)
    DevBuf order, order_tmp;
    // coarse prefilter state per centroid space (transformed / raw)
    CoarseCentroids cc_t, cc_raw;
    CoarseScratch coarse;
    cudaEvent_t ev[5] = {};
    float last_ms[4] = {0, 0, 0, 0};
    bool timed = false;
    ~ads_ivf() {
        for (void* p : {static_cast<void*>(cent_t), static_cast<void*>(cent_raw),
                        static_cast<void*>(list_off), static_cast<void*>(ids),
                        static_cast<void*>(a1_t), static_cast<void*>(a1_raw),  // a2_* live inside
                        static_cast<void*>(P), static_cast<void*>(chain_rank), static_cast<void*>(a1i_t)})
            if (p) cudaFree(p);
        cc_t.release();
        cc_raw.release();
        for (auto& kv : plans) kv.second->release();
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

extern "C" {

const char* ads_last_error(void) { return g_err.c_str(); }
int ads_version(void) { return 1; }

int ads_device_count(int32_t* count) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    cudaGetLastError();
    *count = n;
    return ADS_OK;
}

int ads_rng_draw(uint64_t seed, uint64_t tag, int32_t use_stream, int32_t kind, uint64_t arg,
                 int64_t count, void* out) {
    return guard([&] {
        HostRng r = use_stream ? HostRng::for_stream(seed, tag) : HostRng(seed);
        for (int64_t i = 0; i < count; ++i) {
            switch (kind) {
                case 0: static_cast<uint64_t*>(out)[i] = r.next_u64(); break;
                case 1: static_cast<double*>(out)[i] = r.uniform(); break;
                case 2: static_cast<double*>(out)[i] = r.normal(); break;
                default:
                    require(arg > 0, "below: n must be > 0");
                    static_cast<uint64_t*>(out)[i] = r.below(arg);
            }
        }
    });
}

int ads_generate_orthogonal(int32_t dim, uint64_t seed, double* P_out) {
    return guard([&] {
        const std::vector<double> m = generate_orthogonal(dim, seed);
        std::memcpy(P_out, m.data(), m.size() * sizeof(double));
    });
}

int ads_threshold_multiplier(int32_t d, double eps0, double* out) {
    return guard([&] {
        require(d >= 1, "threshold_multiplier: d must be >= 1");
        require(eps0 > 0.0, "threshold_multiplier: epsilon0 must be > 0");
        *out = 1.0 + eps0 / std::sqrt(static_cast<double>(d));
    });
}

int ads_ad_context(double eps0, int32_t delta_d, int32_t dim, double* factor_out) {
    return guard([&] {
        const std::vector<double> f = ad_factor(eps0, delta_d, dim);
        std::memcpy(factor_out, f.data(), f.size() * sizeof(double));
    });
}

int ads_synth(const ads_synth_desc* desc, float* out, int32_t* comp_out) {
    return guard([&] { synth(*desc, out, comp_out); });
}

int ads_synth_rows(const ads_synth_desc* desc, int64_t row_lo, int64_t count, int64_t stride, float* out,
                   int32_t* comp_out) {
    return guard([&] { synth_rows(*desc, row_lo, count, stride, out, comp_out); });
}

// ------------------------------------------------------------------ context
int ads_ctx_create(int32_t device, ads_ctx** out) {
    return guard([&] {
        int n = 0;
        ADS_CUDA(cudaGetDeviceCount(&n));
        require(device >= 0 && device < n, "ads_ctx_create: no such CUDA device");
        auto c = std::make_unique<ads_ctx>();
        c->device = device;
        c->use();
        ADS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        ADS_CUDA(cudaEventCreate(&c->t0));
        ADS_CUDA(cudaEventCreate(&c->t1));
        ADS_CUDA(cudaMalloc(&c->counter, sizeof(unsigned long long) * 4));
        *out = c.release();
    });
}

int ads_ctx_destroy(ads_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        ctx->use();
        cudaStreamSynchronize(ctx->stream);
        if (ctx->flush) cudaFree(ctx->flush);
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        for (auto& kv : ctx->dco_plans) kv.second->release();
        cudaFree(ctx->counter);
        cudaEventDestroy(ctx->t0);
        cudaEventDestroy(ctx->t1);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int ads_ctx_sync(ads_ctx* ctx) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ads_ctx_stream(ads_ctx* ctx, void** stream) {
    return guard([&] { *stream = static_cast<void*>(ctx->stream); });
}

int ads_dev_alloc(ads_ctx* ctx, int64_t bytes, void** dptr) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaMalloc(dptr, static_cast<size_t>(bytes > 0 ? bytes : 1)));
    });
}
int ads_dev_free(ads_ctx* ctx, void* dptr) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaStreamSynchronize(ctx->stream));
        ADS_CUDA(cudaFree(dptr));
    });
}
int ads_memcpy_h2d(ads_ctx* ctx, void* dst, const void* src, int64_t bytes) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        ADS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int ads_memcpy_d2h(ads_ctx* ctx, void* dst, const void* src, int64_t bytes) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        ADS_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int ads_memset_device(ads_ctx* ctx, void* dst, int32_t value, int64_t bytes) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaMemsetAsync(dst, value, bytes, ctx->stream));
    });
}
int ads_host_alloc_pinned(int64_t bytes, void** hptr) {
    return guard([&] { ADS_CUDA(cudaMallocHost(hptr, static_cast<size_t>(bytes > 0 ? bytes : 1))); });
}
int ads_host_free_pinned(void* hptr) {
    return guard([&] { ADS_CUDA(cudaFreeHost(hptr)); });
}
int ads_timer_start(ads_ctx* ctx) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaEventRecord(ctx->t0, ctx->stream));
    });
}
int ads_timer_stop(ads_ctx* ctx, float* ms) {
    return guard([&] {
        ctx->use();
        ADS_CUDA(cudaEventRecord(ctx->t1, ctx->stream));
        ADS_CUDA(cudaEventSynchronize(ctx->t1));
        ADS_CUDA(cudaEventElapsedTime(ms, ctx->t0, ctx->t1));
    });
}
int ads_flush_l2(ads_ctx* ctx) {
    return guard([&] {
        ctx->use();
        if (!ctx->flush) {
            int l2 = 0;
            ADS_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
            ctx->flush_bytes = static_cast<size_t>(l2) * 2;
            ADS_CUDA(cudaMalloc(&ctx->flush, ctx->flush_bytes));
        }
        ADS_CUDA(cudaMemsetAsync(ctx->flush, 0x5a, ctx->flush_bytes, ctx->stream));
    });
}

// ------------------------------------------------------------------ transform
int ads_transform_create(ads_ctx* ctx, const double* P_host, int32_t dim, ads_transform** out) {
    return guard([&] {
        require(dim >= 1, "transform: dim must be >= 1");
        ctx->use();
        auto t = std::make_unique<ads_transform>();
        t->ctx = ctx;
        t->dim = dim;
        std::vector<double> PT(static_cast<size_t>(dim) * dim);
        for (int i = 0; i < dim; ++i)
            for (int j = 0; j < dim; ++j) PT[static_cast<size_t>(j) * dim + i] = P_host[static_cast<size_t>(i) * dim + j];
        t->P = dev_upload(P_host, PT.size(), ctx->stream);
        t->PT = dev_upload(PT.data(), PT.size(), ctx->stream);
        ADS_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = t.release();
    });
}

int ads_transform_destroy(ads_transform* t) {
    return guard([&] {
        if (!t) return;
        t->ctx->use();
        delete t;
    });
}

static void apply_host(ads_transform* t, const double* M, const float* X, int64_t n, float* Y) {
    require(n >= 0, "apply: n must be >= 0");
    ads_ctx* c = t->ctx;
    c->use();
    std::lock_guard<std::mutex> lk(c->mu);
    const size_t cnt = static_cast<size_t>(n) * t->dim;
    float* dx = t->xin.get<float>(cnt);
    float* dy = t->yout.get<float>(cnt);
    ADS_CUDA(cudaMemcpyAsync(dx, X, cnt * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    launch_apply(M, t->dim, dx, n, dy, c->stream);
    ADS_CUDA(cudaMemcpyAsync(Y, dy, cnt * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    ADS_CUDA(cudaStreamSynchronize(c->stream));
}

int ads_apply_dataset(ads_transform* t, const float* X, int64_t n, float* Y) {
    return guard([&] { apply_host(t, t->P, X, n, Y); });
}

// 3xTF32 tensor-core transform (tc_gemm.cu): dX, dY device arrays of n x dim.
static void apply_tc(ads_transform* t, const float* dX, int64_t n, float* dY) {
    require(n >= 0, "apply: n must be >= 0");
    require(t->dim % 4 == 0 && t->dim >= 32, "apply (tensor cores): dimension must be a multiple of 4 and >= 32");
    cudaStream_t st = t->ctx->stream;
    const size_t dd = static_cast<size_t>(t->dim) * t->dim;
    if (!t->split_ready) {  // P (fp64) -> fp32 -> TF32 hi/lo, once
        std::vector<double> hp(dd);
        ADS_CUDA(cudaMemcpyAsync(hp.data(), t->P, sizeof(double) * dd, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        std::vector<float> pf(hp.begin(), hp.end());
        float* p32 = t->xin.get<float>(dd);
        ADS_CUDA(cudaMemcpyAsync(p32, pf.data(), sizeof(float) * dd, cudaMemcpyHostToDevice, st));
        launch_split_tf32(p32, static_cast<int64_t>(dd), t->ph.get<float>(dd), t->pl.get<float>(dd), st);
        ADS_CUDA(cudaStreamSynchronize(st));
        t->split_ready = true;
    }
    launch_tc_transform(dX, n, t->ph.get<float>(dd), t->pl.get<float>(dd), t->dim, dY, t->xh, t->xl, st);
}

int ads_apply_dataset_tc(ads_transform* t, const float* X, int64_t n, float* Y) {
    return guard([&] {
        ads_ctx* c = t->ctx;
        c->use();
        std::lock_guard<std::mutex> lk(c->mu);
        const size_t cnt = static_cast<size_t>(n) * t->dim;
        float* dx = t->yout.get<float>(cnt);  // input staging
        DevBuf dyb;
        float* dy = dyb.get<float>(cnt);
        ADS_CUDA(cudaMemcpyAsync(dx, X, cnt * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        apply_tc(t, dx, n, dy);
        ADS_CUDA(cudaMemcpyAsync(Y, dy, cnt * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        ADS_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ads_apply_dataset_tc_device(ads_transform* t, const float* dX, int64_t n, float* dY) {
    return guard([&] {
        t->ctx->use();
        apply_tc(t, dX, n, dY);
    });
}
int ads_apply_transpose(ads_transform* t, const float* X, int64_t n, float* Y) {
    return guard([&] { apply_host(t, t->PT, X, n, Y); });
}
int ads_apply_dataset_device(ads_transform* t, const float* dX, int64_t n, float* dY) {
    return guard([&] {
        t->ctx->use();
        launch_apply(t->P, t->dim, dX, n, dY, t->ctx->stream);
    });
}
int ads_apply_transpose_device(ads_transform* t, const float* dX, int64_t n, float* dY) {
    return guard([&] {
        t->ctx->use();
        launch_apply(t->PT, t->dim, dX, n, dY, t->ctx->stream);
    });
}

// ------------------------------------------------------------------ fixed-threshold DCOs
namespace {

SegPlan dco_plan(int kind, int D, double eps0, int dd) {
    if (kind == ADS_DCO_FD) return make_seg_plan(D, 0, {}, nullptr);
    require(dd >= 1 && dd <= D, "dco: delta_d must be in [1, D]");
    const std::vector<int> tests = test_points(D, dd, 0, false);
    if (kind == ADS_DCO_PD) return make_seg_plan(D, 0, tests, nullptr);
    const std::vector<double> f = ad_factor(eps0, dd, D);
    return make_seg_plan(D, 0, tests, f.data());
}

void run_dco_device(ads_ctx* ctx, const ads_dco_batch& b, const std::vector<int64_t>* host_off) {
    require(b.dim >= 1, "dco: dimension must be >= 1");
    require(b.nq >= 0, "dco: nq must be >= 0");
    require(b.kind >= 0 && b.kind <= 2, "dco: unknown kind");
    cudaStream_t st = ctx->stream;
    // segment plans are cached per (kind, D, eps0, delta_d) like ads_dco's: a batch call
    // then costs its kernel and nothing else on the device
    const int D = b.dim, dd = b.kind == ADS_DCO_FD ? D : b.delta_d;
    const auto key = std::make_tuple(b.kind, D, b.kind == ADS_DCO_AD ? b.epsilon0 : 0.0, b.kind == ADS_DCO_FD ? 0 : dd);
    auto it = ctx->dco_plans.find(key);
    if (it == ctx->dco_plans.end()) {
        const SegPlan plan = dco_plan(b.kind, b.dim, b.epsilon0, b.delta_d);
        auto up = std::make_unique<DevSegPlan>();
        up->upload(plan, st);
        it = ctx->dco_plans.emplace(key, std::move(up)).first;
    }
    const DevSegPlan& dp = *it->second;
    DcoLaunch a{};
    a.X = b.X;
    a.n_rows = b.n_rows;
    a.D = b.dim;
    a.Q = b.Q;
    a.nq = b.nq;
    a.cand_off = b.cand_off;
    a.cand_rows = b.cand_rows;
    a.win_start = b.win_start;
    a.win_len = b.win_len;
    a.r = b.r;
    a.kind = b.kind;
    a.segs = dp.segs;
    a.tfac = dp.tfac;
    a.nseg = dp.nseg;
    a.ntest = dp.ntest;
    a.vec = dp.vec;
    // 16-byte line descriptors from X (one 32-bit offset per line, shuffled once per copy)
    a.desc = (dp.vec == 4 && dp.full && (reinterpret_cast<uintptr_t>(b.X) & 15) == 0 &&
              b.n_rows * static_cast<int64_t>(b.dim) / 4 < int64_t(0xffffffff)) ? 1 : 0;
    a.positive = b.positive;
    a.dims = b.dims;
    a.dist_sq = b.dist_sq;
    a.observed = b.observed;
    a.dims_per_query = reinterpret_cast<unsigned long long*>(b.dims_per_query);
    a.counter = ctx->counter;
    constexpr int64_t kTile = 2048;
    a.tile = kTile;
    DevBuf tiles;
    if (b.cand_rows) {
        require(host_off != nullptr, "dco: candidate offsets missing");
        std::vector<int64_t> tq, tl, th;
        for (int q = 0; q < b.nq; ++q) {
            const int64_t cnt = (*host_off)[q + 1] - (*host_off)[q];
            require(cnt >= 0, "dco: cand_off must be non-decreasing");
            require(cnt < (int64_t(1) << 31), "dco: too many candidates for one query");
            for (int64_t lo = 0; lo < cnt; lo += kTile) {
                tq.push_back(q);
                tl.push_back(lo);
                th.push_back(lo + kTile < cnt ? lo + kTile : cnt);
            }
        }
        a.ntiles = static_cast<int64_t>(tq.size());
        std::vector<int64_t> all;
        all.insert(all.end(), tq.begin(), tq.end());
        all.insert(all.end(), tl.begin(), tl.end());
        all.insert(all.end(), th.begin(), th.end());
        const int64_t* dt = buf_upload(tiles, all.data(), all.size(), st);
        a.tile_q = dt;
        a.tile_lo = dt + a.ntiles;
        a.tile_hi = dt + 2 * a.ntiles;
    } else {
        require(b.win_start != nullptr && b.win_len >= 0, "dco: need cand_rows or windows");
        require(b.win_len < (int64_t(1) << 31), "dco: window too long");
        require(b.win_len == 0 || b.n_rows >= 1, "dco: empty database");
        a.ntiles = b.win_len > 0 ? static_cast<int64_t>(b.nq) * ((b.win_len + kTile - 1) / kTile) : 0;
    }
    if (b.dims_per_query) ADS_CUDA(cudaMemsetAsync(b.dims_per_query, 0, sizeof(uint64_t) * b.nq, st));
    if (a.ntiles > 0) launch_dco_fixed(a, st);
    if (b.cand_rows) ADS_CUDA(cudaStreamSynchronize(st));  // the tile table is freed below
}

}  // namespace

int ads_dco_fixed_device(ads_ctx* ctx, const ads_dco_batch* b) {
    return guard([&] {
        ctx->use();
        std::lock_guard<std::mutex> lk(ctx->mu);  // the context's plan cache
        std::vector<int64_t> off;
        if (b->cand_rows) {
            off.resize(static_cast<size_t>(b->nq) + 1);
            ADS_CUDA(cudaMemcpyAsync(off.data(), b->cand_off, sizeof(int64_t) * off.size(),
                                     cudaMemcpyDeviceToHost, ctx->stream));
            ADS_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        run_dco_device(ctx, *b, b->cand_rows ? &off : nullptr);
    });
}

int ads_dco_fixed(ads_ctx* ctx, const ads_dco_batch* hb) {
    return guard([&] {
        ctx->use();
        std::lock_guard<std::mutex> lk(ctx->mu);  // the context's plan cache
        cudaStream_t st = ctx->stream;
        const ads_dco_batch& b = *hb;
        require(b.dim >= 1 && b.nq >= 0 && b.n_rows >= 0, "dco: bad shape");
        int64_t total = 0;
        std::vector<int64_t> off;
        if (b.cand_rows) {
            off.assign(b.cand_off, b.cand_off + b.nq + 1);
            total = off[b.nq] - off[0];
            require(off[0] == 0, "dco: cand_off[0] must be 0");
            for (int64_t i = 0; i < total; ++i)
                require(b.cand_rows[i] >= 0 && b.cand_rows[i] < b.n_rows, "dco: candidate row out of range");
        } else {
            require(b.win_start != nullptr, "dco: need cand_rows or windows");
            total = static_cast<int64_t>(b.nq) * b.win_len;
            for (int q = 0; q < b.nq; ++q)
                require(b.win_start[q] >= 0 && b.win_start[q] < (b.n_rows > 0 ? b.n_rows : 1),
                        "dco: window start out of range");
        }
        ads_dco_batch d = b;
        std::vector<void*> owned;
        auto up = [&](const void* h, size_t bytes) -> void* {
            void* p = nullptr;
            ADS_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 1));
            if (bytes) ADS_CUDA(cudaMemcpyAsync(p, h, bytes, cudaMemcpyHostToDevice, st));
            owned.push_back(p);
            return p;
        };
        auto alloc = [&](size_t bytes) -> void* {
            void* p = nullptr;
            ADS_CUDA(cudaMalloc(&p, bytes > 0 ? bytes : 1));
            owned.push_back(p);
            return p;
        };
        try {
            d.X = static_cast<const float*>(up(b.X, sizeof(float) * b.n_rows * b.dim));
            d.Q = static_cast<const float*>(up(b.Q, sizeof(float) * b.nq * static_cast<size_t>(b.dim)));
            d.r = static_cast<const double*>(up(b.r, sizeof(double) * b.nq));
            if (b.cand_rows) {
                d.cand_off = static_cast<const int64_t*>(up(b.cand_off, sizeof(int64_t) * (b.nq + 1)));
                d.cand_rows = static_cast<const int64_t*>(up(b.cand_rows, sizeof(int64_t) * total));
            } else {
                d.win_start = static_cast<const int64_t*>(up(b.win_start, sizeof(int64_t) * b.nq));
            }
            d.positive = b.positive ? static_cast<uint8_t*>(alloc(total)) : nullptr;
            d.dims = b.dims ? static_cast<int32_t*>(alloc(sizeof(int32_t) * total)) : nullptr;
            d.dist_sq = b.dist_sq ? static_cast<double*>(alloc(sizeof(double) * total)) : nullptr;
            d.observed = b.observed ? static_cast<double*>(alloc(sizeof(double) * total)) : nullptr;
            d.dims_per_query = b.dims_per_query ? static_cast<uint64_t*>(alloc(sizeof(uint64_t) * b.nq)) : nullptr;
            run_dco_device(ctx, d, b.cand_rows ? &off : nullptr);
            auto down = [&](void* h, const void* dv, size_t bytes) {
                if (h && bytes) ADS_CUDA(cudaMemcpyAsync(h, dv, bytes, cudaMemcpyDeviceToHost, st));
            };
            down(b.positive, d.positive, total);
            down(b.dims, d.dims, sizeof(int32_t) * total);
            down(b.dist_sq, d.dist_sq, sizeof(double) * total);
            down(b.observed, d.observed, sizeof(double) * total);
            down(b.dims_per_query, d.dims_per_query, sizeof(uint64_t) * b.nq);
            ADS_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaStreamSynchronize(st);
            for (void* p : owned) cudaFree(p);
            throw;
        }
        for (void* p : owned) cudaFree(p);
    });
}

int ads_dco_prefix_sums_device(ads_ctx* ctx, const float* dX, int64_t n_rows, int32_t dim, const float* dq,
                               const int64_t* dcand, int32_t nc, int32_t delta_d, double* dout) {
    return guard([&] {
        require(dim >= 1 && n_rows >= 0 && nc >= 0, "dco: bad shape");
        require(delta_d >= 1 && delta_d <= dim, "DcoConfig: delta_d must be in [1, dim]");
        ctx->use();
        launch_prefix_sums(dX, dim, dq, dcand, nc, delta_d, dout, ctx->stream);
    });
}

int ads_dco(ads_ctx* ctx, int32_t kind, const float* o, int32_t n_o, const float* q, int32_t n_q,
            double r, double eps0, int32_t delta_d, int32_t* positive, double* distance,
            double* observed, int32_t* dims_used) {
    return guard([&] {
        // validate_query (dco.cpp:23-30), then the per-kind checks (dco.cpp:86-87, 32-37).
        require(n_o == n_q, "dco: vector lengths differ");
        require(n_o > 0, "dco: empty vectors");
        require(r >= 0.0 && std::isfinite(r), "dco: threshold must be finite and >= 0");
        require(kind >= 0 && kind <= 2, "dco: unknown kind");
        if (kind == ADS_DCO_PD) require(delta_d >= 1 && delta_d <= n_o, "pd_scan: delta_d must be in [1, D]");
        if (kind == ADS_DCO_AD) (void)ad_factor(eps0, delta_d, n_o);
        ctx->use();
        std::lock_guard<std::mutex> lk(ctx->mu);
        cudaStream_t st = ctx->stream;
        const int D = n_o;
        const int dd = kind == ADS_DCO_FD ? D : delta_d;
        const auto key = std::make_tuple(kind, D, kind == ADS_DCO_AD ? eps0 : 0.0, kind == ADS_DCO_FD ? 0 : dd);
        auto it = ctx->dco_plans.find(key);
        if (it == ctx->dco_plans.end()) {
            auto dp = std::make_unique<DevSegPlan>();
            dp->upload(dco_plan(kind, D, eps0, dd), st);
            it = ctx->dco_plans.emplace(key, std::move(dp)).first;
        }
        const DevSegPlan& dp = *it->second;
        // staging layout (bytes): X[D] f32 | Q[D] f32 | r f64 | off[2] i64 | row i64 | tile q,lo,hi i64
        //                         | pos u8 (pad 8) | dims i32 (pad 8) | obs f64 | dpq u64
        const size_t vbytes = ((sizeof(float) * D + 15) / 16) * 16;
        const size_t in_bytes = 2 * vbytes + 8 * 7;
        const size_t out_bytes = 8 * 4;
        if (!ctx->h_stage) ADS_CUDA(cudaMallocHost(&ctx->h_stage, 1 << 20));
        require(in_bytes + out_bytes <= (1 << 20), "dco: vector too long for the single-DCO path");
        unsigned char* h = static_cast<unsigned char*>(ctx->h_stage);
        unsigned char* d = ctx->d_stage.get<unsigned char>(in_bytes + out_bytes);
        std::memcpy(h, o, sizeof(float) * D);
        std::memcpy(h + vbytes, q, sizeof(float) * D);
        int64_t* hi = reinterpret_cast<int64_t*>(h + 2 * vbytes + 8);
        std::memcpy(h + 2 * vbytes, &r, 8);
        hi[0] = 0;  // cand_off
        hi[1] = 1;
        hi[2] = 0;  // cand_rows[0]
        hi[3] = 0;  // tile q
        hi[4] = 0;  // tile lo
        hi[5] = 1;  // tile hi
        ADS_CUDA(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, st));
        int64_t* di = reinterpret_cast<int64_t*>(d + 2 * vbytes + 8);
        unsigned char* dout = d + in_bytes;
        DcoLaunch a{};
        a.X = reinterpret_cast<const float*>(d);
        a.n_rows = 1;
        a.D = D;
        a.Q = reinterpret_cast<const float*>(d + vbytes);
        a.nq = 1;
        a.cand_off = di;
        a.cand_rows = di + 2;
        a.r = reinterpret_cast<const double*>(d + 2 * vbytes);
        a.tile_q = di + 3;
        a.tile_lo = di + 4;
        a.tile_hi = di + 5;
        a.ntiles = 1;
        a.tile = 1;
        a.kind = kind;
        a.segs = dp.segs;
        a.tfac = dp.tfac;
        a.nseg = dp.nseg;
        a.ntest = dp.ntest;
        a.vec = dp.vec;
        a.positive = dout;
        a.dims = reinterpret_cast<int32_t*>(dout + 8);
        a.observed = reinterpret_cast<double*>(dout + 16);
        a.counter = ctx->counter;
        launch_dco_fixed(a, st);
        ADS_CUDA(cudaMemcpyAsync(h + in_bytes, dout, out_bytes, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        const uint8_t pos = h[in_bytes];
        int32_t dims = 0;
        double obs = 0.0;
        std::memcpy(&dims, h + in_bytes + 8, 4);
        std::memcpy(&obs, h + in_bytes + 16, 8);
        *positive = pos;
        *observed = obs;
        *dims_used = dims;
        *distance = pos ? obs : std::nan("");
    });
}

// ------------------------------------------------------------------ exact k-NN
int ads_brute_force_knn_device(ads_ctx* ctx, const float* dbase, int64_t n, int32_t d,
                               const float* dqueries, int32_t nq, int32_t K, int32_t* dids) {
    return guard([&] {
        require(K >= 1, "brute_force_knn: K must be >= 1");
        require(K <= n, "brute_force_knn: K exceeds dataset size");
        ctx->use();
        launch_brute_knn(dbase, n, d, dqueries, nq, K, dids, ctx->stream);
    });
}

int ads_brute_force_knn(ads_ctx* ctx, const float* base, int64_t n, int32_t d,
                        const float* queries, int32_t nq, int32_t K, int32_t* ids) {
    return guard([&] {
        require(K >= 1, "brute_force_knn: K must be >= 1");
        require(K <= n, "brute_force_knn: K exceeds dataset size");
        ctx->use();
        cudaStream_t st = ctx->stream;
        DevBuf bb, bq, bi;
        const float* db = buf_upload(bb, base, static_cast<size_t>(n) * d, st);
        const float* dq = buf_upload(bq, queries, static_cast<size_t>(nq) * d, st);
        int32_t* di = bi.get<int32_t>(static_cast<size_t>(nq) * K);
        launch_brute_knn(db, n, d, dq, nq, K, di, st);
        ADS_CUDA(cudaMemcpyAsync(ids, di, sizeof(int32_t) * nq * K, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
    });
}

// ------------------------------------------------------------------ verify_theory
int ads_verify_theory(ads_ctx* ctx, const float* Xt, int64_t n, int32_t d, const float* Qt, int32_t nq,
                      int32_t K, const double* grid, int32_t G, double* eps_sorted, double* failure_rate,
                      double* avg_dims, uint64_t* failures, uint64_t* positives) {
    return guard([&] {
        // bench.cpp:305-307
        require(d >= 1, "verify_theory: dimensionality mismatch");
        require(K >= 1 && K <= n, "verify_theory: bad K");
        require(G >= 0, "verify_theory: bad grid");
        std::vector<double> eps(grid, grid + G);
        std::sort(eps.begin(), eps.end());
        std::vector<double> factor(static_cast<size_t>(G) * d);
        for (int g = 0; g < G; ++g) {  // AdContext(DcoConfig{eps, 1}, dim) (bench.cpp:316)
            const std::vector<double> f = ad_factor(eps[g], 1, d);
            std::copy(f.begin(), f.end(), factor.begin() + static_cast<size_t>(g) * d);
        }
        ctx->use();
        cudaStream_t st = ctx->stream;
        DevBuf dx, dq, df, dids, dr, dc;
        float* xp = dx.get<float>(static_cast<size_t>(n) * d);
        float* qp = dq.get<float>(static_cast<size_t>(nq) * d);
        double* fp = df.get<double>(factor.size());
        ADS_CUDA(cudaMemcpyAsync(xp, Xt, sizeof(float) * n * d, cudaMemcpyHostToDevice, st));
        if (nq) ADS_CUDA(cudaMemcpyAsync(qp, Qt, sizeof(float) * nq * static_cast<size_t>(d), cudaMemcpyHostToDevice, st));
        if (G) ADS_CUDA(cudaMemcpyAsync(fp, factor.data(), sizeof(double) * factor.size(), cudaMemcpyHostToDevice, st));
        auto* cnt = dc.get<unsigned long long>(2 * static_cast<size_t>(G) + 1);
        launch_verify_theory(xp, n, d, qp, nq, K, fp, G, dids.get<int32_t>(static_cast<size_t>(nq) * K),
                             dr.get<double>(nq), cnt, st);
        std::vector<unsigned long long> h(2 * static_cast<size_t>(G) + 1);
        ADS_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        // bench.cpp:376-391
        const uint64_t pos = h[2 * G];
        const double total = static_cast<double>(nq) * static_cast<double>(n);
        for (int g = 0; g < G; ++g) {
            if (eps_sorted) eps_sorted[g] = eps[g];
            if (failures) failures[g] = h[G + g];
            if (positives) positives[g] = pos;
            if (failure_rate) failure_rate[g] = pos > 0 ? static_cast<double>(h[G + g]) / pos : 0.0;
            if (avg_dims) avg_dims[g] = static_cast<double>(h[g]) / total;
        }
    });
}

// ------------------------------------------------------------------ k-means
int ads_kmeans(ads_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k, int32_t max_iters,
               uint64_t seed, int32_t init, float* centroids, int32_t* assignment, double* objective,
               int32_t* iterations) {
    return guard([&] {
        require(k >= 1, "kmeans: k must be >= 1");
        require(k <= n, "kmeans: k exceeds the number of points");
        ctx->use();
        cudaStream_t st = ctx->stream;
        float* dx = dev_upload(X, static_cast<size_t>(n) * d, st);
        float* dc = nullptr;
        int32_t* da = nullptr;
        ADS_CUDA(cudaMalloc(&dc, sizeof(float) * k * static_cast<size_t>(d)));
        ADS_CUDA(cudaMalloc(&da, sizeof(int32_t) * n));
        KmeansOut o{};
        try {
            o = run_kmeans(dx, n, d, k, max_iters, seed, init, dc, da, st);
        } catch (...) {
            cudaFree(dx);
            cudaFree(dc);
            cudaFree(da);
            throw;
        }
        ADS_CUDA(cudaMemcpyAsync(centroids, dc, sizeof(float) * k * static_cast<size_t>(d), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaMemcpyAsync(assignment, da, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        cudaFree(dx);
        cudaFree(dc);
        cudaFree(da);
        *objective = o.objective;
        *iterations = o.iterations;
    });
}

// ------------------------------------------------------------------ IVF
static void ivf_alloc_common(ads_ivf* x) {
    for (auto& e : x->ev) ADS_CUDA(cudaEventCreate(&e));
}

// Centred centroid table for the coarse prefilter (coarse.cu): mean in fp64 (host),
// c~ = fl32(c - mu), |c~|^2 and the largest |c~|.
static void centroid_prefilter(const float* dC, int k, int D, CoarseCentroids& out, cudaStream_t st) {
    std::vector<float> h(static_cast<size_t>(k) * D);
    ADS_CUDA(cudaMemcpyAsync(h.data(), dC, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, st));
    ADS_CUDA(cudaStreamSynchronize(st));
    std::vector<double> mu(static_cast<size_t>(D), 0.0);
    for (int c = 0; c < k; ++c)
        for (int j = 0; j < D; ++j) mu[j] += h[static_cast<size_t>(c) * D + j];
    for (double& v : mu) v /= k;
    out.mu = dev_upload(mu.data(), mu.size(), st);
    ADS_CUDA(cudaMalloc(&out.cc, sizeof(float) * h.size()));
    ADS_CUDA(cudaMalloc(&out.cn2, sizeof(float) * k));
    DevBuf bn;
    double* nrm = bn.get<double>(k);
    coarse_center(dC, k, D, out.mu, out.cc, out.cn2, nrm, st);
    if (tc_coarse_supported(D)) {
        ADS_CUDA(cudaMalloc(&out.cc_tf, sizeof(float) * h.size()));
        coarse_center(dC, k, D, out.mu, out.cc_tf, out.cn2, nrm, st, true);
    }
    std::vector<double> hn(static_cast<size_t>(k));
    ADS_CUDA(cudaMemcpyAsync(hn.data(), nrm, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    ADS_CUDA(cudaStreamSynchronize(st));
    double m = 0.0;
    for (double v : hn) m = std::max(m, v);
    out.cmax = m * (1.0 + 1e-12) + 1e-300;
}

// The interleaved A1 copy the scan's dense prefix phase reads (ivf.cu); call once the
// index's A1 holds its final rows.
// Only for long lists (>= 1024 rows on average, config 5's 6 100): a chunk's rows then
// form one or two long runs and the dense phase measured +1-2 % (tools/ab_scan.py,
// profiles/r02/ab_dense.log); with ~244-row lists (configs 2 and 3) it measured -1 %.
// ADS_DENSE_MIN_LIST overrides the 1024 (tests: 0 builds the copy for short lists too).
static void ivf_finish_dense(ads_ivf* x, cudaStream_t st) {
    {
        std::vector<int64_t> off(static_cast<size_t>(x->k) + 1);
        ADS_CUDA(cudaMemcpyAsync(off.data(), x->list_off, sizeof(int64_t) * off.size(), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        x->nonempty = 0;
        for (int c = 0; c < x->k; ++c) x->nonempty += off[c + 1] > off[c];
    }
    int64_t min_list = 1024;
    if (const char* e = std::getenv("ADS_DENSE_MIN_LIST")) min_list = std::atoll(e);
    if (x->layout == 1 && x->d1p == 32 && x->a1_t && !x->a1i_t && x->n >= min_list * std::max(1, x->nonempty)) {
        const size_t groups = (static_cast<size_t>(x->n) + 31) / 32;
        ADS_CUDA(cudaMalloc(&x->a1i_t, sizeof(float) * 1024 * (groups > 0 ? groups : 1)));
        interleave_rows(x->a1_t, x->n, 32, x->a1i_t, st);
    }
}

static void ivf_finish_coarse(ads_ivf* x, cudaStream_t st) {
    centroid_prefilter(x->cent_t, x->k, x->d, x->cc_t, st);
    if (x->cent_raw) centroid_prefilter(x->cent_raw, x->k, x->d, x->cc_raw, st);
}

int ads_ivf_create(ads_ctx* ctx, const ads_ivf_desc* desc, ads_ivf** out) {
    return guard([&] {
        const ads_ivf_desc& s = *desc;
        require(s.n >= 1 && s.d >= 1 && s.k_clusters >= 1, "ivf: bad shape");
        require(s.centroids_t && s.list_off && s.ids_flat, "ivf: missing arrays");
        require(s.a1_t || s.vec_t, "ivf: missing transformed vectors");
        if (s.layout == 1) require(s.d1 >= 1 && s.d1 < s.d, "build_ivf: split layout needs 1 <= d1 < D");
        require(s.list_off[0] == 0 && s.list_off[s.k_clusters] == s.n, "ivf: list offsets do not cover n");
        ctx->use();
        cudaStream_t st = ctx->stream;
        auto x = std::make_unique<ads_ivf>();
        x->ctx = ctx;
        x->n = s.n;
        x->d = s.d;
        x->k = s.k_clusters;
        x->d1 = s.d1;
        x->layout = s.layout;
        x->seed = s.seed;
        ivf_alloc_common(x.get());
        const int D = s.d;
        x->d1p = s.a1_t ? s.d1 : (s.layout == 1 ? s.d1 : (D > 32 ? 32 : D));
        const int d1p = x->d1p, d2p = D - d1p;
        const size_t n = static_cast<size_t>(s.n);
        x->cent_t = dev_upload(s.centroids_t, static_cast<size_t>(s.k_clusters) * D, st);
        x->list_off = dev_upload(s.list_off, static_cast<size_t>(s.k_clusters) + 1, st);
        x->ids = dev_upload(s.ids_flat, n, st);
        auto split_up = [&](const float* a1, const float* a2, const float* vec, float** o1, float** o2) {
            alloc_split_pair(n, d1p, d2p, o1, o2);
            if (a1) {
                ADS_CUDA(cudaMemcpyAsync(*o1, a1, sizeof(float) * n * d1p, cudaMemcpyHostToDevice, st));
                if (d2p) ADS_CUDA(cudaMemcpyAsync(*o2, a2, sizeof(float) * n * d2p, cudaMemcpyHostToDevice, st));
            } else {
                ADS_CUDA(cudaMemcpy2DAsync(*o1, sizeof(float) * d1p, vec, sizeof(float) * D,
                                           sizeof(float) * d1p, n, cudaMemcpyHostToDevice, st));
                if (d2p)
                    ADS_CUDA(cudaMemcpy2DAsync(*o2, sizeof(float) * d2p, vec + d1p, sizeof(float) * D,
                                               sizeof(float) * d2p, n, cudaMemcpyHostToDevice, st));
            }
        };
        split_up(s.a1_t, s.a2_t, s.vec_t, &x->a1_t, &x->a2_t);
        if ((s.a1_raw || s.vec_raw) && s.centroids_raw) {
            x->has_raw = true;
            x->cent_raw = dev_upload(s.centroids_raw, static_cast<size_t>(s.k_clusters) * D, st);
            split_up(s.a1_raw, s.a2_raw, s.vec_raw, &x->a1_raw, &x->a2_raw);
        }
        if (s.P) x->P = dev_upload(s.P, static_cast<size_t>(D) * D, st);
        {
            const std::vector<int32_t> rk = centroid_chain_rank(s.centroids_t, s.k_clusters, D);
            x->chain_rank = dev_upload(rk.data(), rk.size(), st);
        }
        ivf_finish_coarse(x.get(), st);
        ivf_finish_dense(x.get(), st);
        ADS_CUDA(cudaStreamSynchronize(st));
        *out = x.release();
    });
}

int ads_ivf_build(ads_ctx* ctx, const float* raw, const float* t, int32_t n, int32_t d,
                  const double* P, int32_t k, uint64_t seed, int32_t layout, int32_t d1,
                  int32_t max_iters, int32_t init, ads_ivf** out) {
    return guard([&] {
        // ivf.cpp:195-200
        require(n >= 1 && d >= 1, "build_ivf: bad shape");
        require(P != nullptr, "build_ivf: matrix dimension does not match the data");
        if (layout == 1) require(d1 >= 1 && d1 < d, "build_ivf: split layout needs 1 <= d1 < D");
        require(k >= 1, "kmeans: k must be >= 1");
        require(k <= n, "kmeans: k exceeds the number of points");
        ctx->use();
        cudaStream_t st = ctx->stream;
        auto x = std::make_unique<ads_ivf>();
        x->ctx = ctx;
        x->n = n;
        x->d = d;
        x->k = k;
        x->d1 = d1;
        x->layout = layout;
        x->seed = seed;
        ivf_alloc_common(x.get());
        x->d1p = layout == 1 ? d1 : (d > 32 ? 32 : d);
        const int d1p = x->d1p, d2p = d - d1p;
        const size_t N = static_cast<size_t>(n);
        float* dt = dev_upload(t, N * d, st);
        float* dr = raw ? dev_upload(raw, N * d, st) : nullptr;
        int32_t* asg = nullptr;
        ADS_CUDA(cudaMalloc(&asg, sizeof(int32_t) * N));
        ADS_CUDA(cudaMalloc(&x->cent_t, sizeof(float) * k * static_cast<size_t>(d)));
        x->P = dev_upload(P, static_cast<size_t>(d) * d, st);
        try {
            (void)run_kmeans(dt, n, d, k, max_iters, seed, init, x->cent_t, asg, st);  // ivf.cpp:210
            ADS_CUDA(cudaMalloc(&x->list_off, sizeof(int64_t) * (k + 1)));
            ADS_CUDA(cudaMalloc(&x->ids, sizeof(int32_t) * N));
            build_lists(asg, n, k, x->list_off, x->ids, st);  // ivf.cpp:213-214, 229-241
            alloc_split_pair(N, d1p, d2p, &x->a1_t, &x->a2_t);
            gather_split(dt, x->ids, n, d, d1p, x->a1_t, x->a2_t, st);
            if (dr) {
                x->has_raw = true;
                alloc_split_pair(N, d1p, d2p, &x->a1_raw, &x->a2_raw);
                gather_split(dr, x->ids, n, d, d1p, x->a1_raw, x->a2_raw, st);
                // centroids_raw = P^T centroids_t (ivf.cpp:216-226)
                std::vector<double> PT(static_cast<size_t>(d) * d);
                for (int i = 0; i < d; ++i)
                    for (int j = 0; j < d; ++j) PT[static_cast<size_t>(j) * d + i] = P[static_cast<size_t>(i) * d + j];
                DevBuf bpt;
                const double* dPT = buf_upload(bpt, PT.data(), PT.size(), st);
                ADS_CUDA(cudaMalloc(&x->cent_raw, sizeof(float) * k * static_cast<size_t>(d)));
                launch_apply(dPT, d, x->cent_t, k, x->cent_raw, st);
                ADS_CUDA(cudaStreamSynchronize(st));
            }
            std::vector<float> hc(static_cast<size_t>(k) * d);
            ADS_CUDA(cudaMemcpyAsync(hc.data(), x->cent_t, sizeof(float) * hc.size(), cudaMemcpyDeviceToHost, st));
            ADS_CUDA(cudaStreamSynchronize(st));
            const std::vector<int32_t> rk = centroid_chain_rank(hc.data(), k, d);
            x->chain_rank = dev_upload(rk.data(), rk.size(), st);
            ivf_finish_coarse(x.get(), st);
            ivf_finish_dense(x.get(), st);
            ADS_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaStreamSynchronize(st);
            cudaFree(dt);
            if (dr) cudaFree(dr);
            cudaFree(asg);
            throw;
        }
        cudaFree(dt);
        if (dr) cudaFree(dr);
        cudaFree(asg);
        *out = x.release();
    });
}

// ------------------------------------------------------------------ streamed build
// build_ivf (ivf.cpp:192-258) for data that arrives in row chunks (config 5):
// k-means on a sample (train) or given centroids, every added row assigned to its
// nearest centroid by the certified coarse prefilter at nprobe = 1 (the exact fp64
// argmin, lowest id on ties, as kmeans assigns), and at finish the bucket layout of
// the lists a shard keeps (ascending ids per list, split at d1).
struct ads_ivf_builder {
    ads_ctx* ctx = nullptr;
    int64_t n = 0, added = 0;
    int d = 0, k = 0, d1 = 0;
    uint64_t seed = 0;
    std::vector<double> P;
    float* cent = nullptr;  // k x d, device
    bool trained = false;
    DevBuf rows, asg;       // staged rows (n x d) and their lists (n)
    CoarseCentroids cc;
    CoarseScratch coarse;
    ~ads_ivf_builder() {
        if (cent) cudaFree(cent);
        cc.release();
    }
};

static void builder_prefilter(ads_ivf_builder* b) {
    b->cc.release();
    centroid_prefilter(b->cent, b->k, b->d, b->cc, b->ctx->stream);
    b->trained = true;
}

int ads_ivf_builder_create(ads_ctx* ctx, int64_t n, int32_t d, const double* P, int32_t k, uint64_t seed,
                           int32_t d1, ads_ivf_builder** out) {
    return guard([&] {
        require(n >= 1 && n <= 0x7fffffff && d >= 1, "build_ivf: bad shape");
        require(P != nullptr, "build_ivf: matrix dimension does not match the data");
        require(d1 >= 1 && d1 < d, "build_ivf: split layout needs 1 <= d1 < D");
        require(k >= 1 && k <= n, "kmeans: k exceeds the number of points");
        ctx->use();
        auto b = std::make_unique<ads_ivf_builder>();
        b->ctx = ctx;
        b->n = n;
        b->d = d;
        b->k = k;
        b->d1 = d1;
        b->seed = seed;
        b->P.assign(P, P + static_cast<size_t>(d) * d);
        ADS_CUDA(cudaMalloc(&b->cent, sizeof(float) * k * static_cast<size_t>(d)));
        *out = b.release();
    });
}

int ads_ivf_builder_train_device(ads_ivf_builder* b, const float* dS, int64_t sample, int32_t max_iters) {
    return guard([&] {
        require(sample >= b->k && sample <= b->n, "build_ivf: need 1 <= k <= sample <= n");
        b->ctx->use();
        DevBuf dsa;
        (void)run_kmeans(dS, sample, b->d, b->k, max_iters, b->seed, 1, b->cent, dsa.get<int32_t>(sample),
                         b->ctx->stream);
        builder_prefilter(b);
        ADS_CUDA(cudaStreamSynchronize(b->ctx->stream));
    });
}

int ads_ivf_builder_set_centroids(ads_ivf_builder* b, const float* centroids) {
    return guard([&] {
        b->ctx->use();
        ADS_CUDA(cudaMemcpyAsync(b->cent, centroids, sizeof(float) * b->k * static_cast<size_t>(b->d),
                                 cudaMemcpyHostToDevice, b->ctx->stream));
        builder_prefilter(b);
        ADS_CUDA(cudaStreamSynchronize(b->ctx->stream));
    });
}

int ads_ivf_builder_centroids(ads_ivf_builder* b, float* centroids) {
    return guard([&] {
        require(b->trained, "build_ivf: no centroids yet (train or set them first)");
        b->ctx->use();
        ADS_CUDA(cudaMemcpyAsync(centroids, b->cent, sizeof(float) * b->k * static_cast<size_t>(b->d),
                                 cudaMemcpyDeviceToHost, b->ctx->stream));
        ADS_CUDA(cudaStreamSynchronize(b->ctx->stream));
    });
}

int ads_ivf_builder_add_device(ads_ivf_builder* b, const float* dT, int64_t row_lo, int64_t rows) {
    return guard([&] {
        require(b->trained, "build_ivf: no centroids yet (train or set them first)");
        require(row_lo == b->added && rows >= 0 && row_lo + rows <= b->n,
                "build_ivf: rows must be added in order, without gaps, inside [0, n)");
        b->ctx->use();
        cudaStream_t st = b->ctx->stream;
        const size_t D = b->d;
        float* R = b->rows.get<float>(static_cast<size_t>(b->n) * D);
        int32_t* A = b->asg.get<int32_t>(static_cast<size_t>(b->n));
        ADS_CUDA(cudaMemcpyAsync(R + row_lo * D, dT, sizeof(float) * rows * D, cudaMemcpyDeviceToDevice, st));
        const int64_t chunk = 65536;
        for (int64_t r = 0; r < rows; r += chunk) {
            const int m = static_cast<int>(rows - r < chunk ? rows - r : chunk);
            launch_coarse_probes_fast(dT + r * D, m, b->cent, b->k, b->d, 1, b->cc, b->coarse, A + row_lo + r, 0,
                                      st);
        }
        b->added += rows;
    });
}

int ads_ivf_builder_rows_device(ads_ivf_builder* b, const float** rows) {
    return guard([&] {
        require(b->added == b->n, "build_ivf: not every row has been added");
        *rows = static_cast<const float*>(b->rows.p);
    });
}

int ads_ivf_builder_list_sizes(ads_ivf_builder* b, int64_t* sizes) {
    return guard([&] {
        require(b->added == b->n, "build_ivf: not every row has been added");
        b->ctx->use();
        cudaStream_t st = b->ctx->stream;
        DevBuf off, ids;
        int64_t* o = off.get<int64_t>(b->k + 1);
        build_lists(static_cast<int32_t*>(b->asg.p), b->n, b->k, o, ids.get<int32_t>(b->n), st);
        std::vector<int64_t> h(static_cast<size_t>(b->k) + 1);
        ADS_CUDA(cudaMemcpyAsync(h.data(), o, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        for (int c = 0; c < b->k; ++c) sizes[c] = h[c + 1] - h[c];
    });
}

int ads_ivf_builder_finish(ads_ivf_builder* b, const uint8_t* keep, ads_ivf** out) {
    return guard([&] {
        require(b->added == b->n, "build_ivf: not every row has been added");
        ads_ctx* ctx = b->ctx;
        ctx->use();
        cudaStream_t st = ctx->stream;
        const int k = b->k, d = b->d, d1 = b->d1;
        auto x = std::make_unique<ads_ivf>();
        x->ctx = ctx;
        x->d = d;
        x->k = k;
        x->d1 = d1;
        x->layout = 1;
        x->seed = b->seed;
        x->d1p = d1;
        ivf_alloc_common(x.get());
        x->P = dev_upload(b->P.data(), b->P.size(), st);
        ADS_CUDA(cudaMalloc(&x->cent_t, sizeof(float) * k * static_cast<size_t>(d)));
        ADS_CUDA(cudaMemcpyAsync(x->cent_t, b->cent, sizeof(float) * k * static_cast<size_t>(d),
                                 cudaMemcpyDeviceToDevice, st));
        const int32_t* A = static_cast<int32_t*>(b->asg.p);
        DevBuf masked, kd, off, ids;
        int kk = k;
        if (keep) {  // lists this shard does not own go to bucket k, after every owned row
            std::vector<uint8_t> hk(keep, keep + k);
            int32_t* M = masked.get<int32_t>(b->n);
            mask_assignment(A, b->n, buf_upload(kd, hk.data(), hk.size(), st), k, M, st);
            A = M;
            kk = k + 1;
        }
        int64_t* o = off.get<int64_t>(kk + 1);
        int32_t* I = ids.get<int32_t>(b->n);
        build_lists(A, b->n, kk, o, I, st);
        std::vector<int64_t> h(static_cast<size_t>(kk) + 1);
        ADS_CUDA(cudaMemcpyAsync(h.data(), o, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        const int64_t m = h[k];  // rows in kept lists
        x->n = static_cast<int>(m);
        x->list_off = dev_upload(h.data(), static_cast<size_t>(k) + 1, st);
        const size_t mm = static_cast<size_t>(m > 0 ? m : 1);
        ADS_CUDA(cudaMalloc(&x->ids, sizeof(int32_t) * mm));
        ADS_CUDA(cudaMemcpyAsync(x->ids, I, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, st));
        alloc_split_pair(mm, d1, d - d1, &x->a1_t, &x->a2_t);
        gather_split(static_cast<float*>(b->rows.p), I, m, d, d1, x->a1_t, x->a2_t, st);
        ivf_finish_coarse(x.get(), st);
        ivf_finish_dense(x.get(), st);
        ADS_CUDA(cudaStreamSynchronize(st));
        *out = x.release();
    });
}

int ads_ivf_builder_destroy(ads_ivf_builder* b) {
    return guard([&] {
        if (!b) return;
        b->ctx->use();
        cudaStreamSynchronize(b->ctx->stream);
        delete b;
    });
}

int ads_ivf_build_sampled_device(ads_ctx* ctx, const float* dT, int64_t n, int32_t d, const double* P, int32_t k,
                                 uint64_t seed, int32_t d1, int32_t max_iters, int64_t sample, ads_ivf** out) {
    // The streamed builder fed in one piece: k-means on every (n / sample)-th row.
    ads_ivf_builder* b = nullptr;
    int rc = guard([&] { require(sample >= k && sample <= n, "build_ivf: need 1 <= k <= sample <= n"); });
    if (!rc) rc = ads_ivf_builder_create(ctx, n, d, P, k, seed, d1, &b);
    if (rc) return rc;
    DevBuf ds;
    rc = guard([&] {
        const int64_t stride = n / sample;
        float* S = ds.get<float>(static_cast<size_t>(sample) * d);
        ADS_CUDA(cudaMemcpy2DAsync(S, sizeof(float) * d, dT, sizeof(float) * d * stride, sizeof(float) * d,
                                   static_cast<size_t>(sample), cudaMemcpyDeviceToDevice, ctx->stream));
    });
    if (!rc) rc = ads_ivf_builder_train_device(b, static_cast<float*>(ds.p), sample, max_iters);
    ds.release();
    if (!rc) rc = ads_ivf_builder_add_device(b, dT, 0, n);
    if (!rc) rc = ads_ivf_builder_finish(b, nullptr, out);
    ads_ivf_builder_destroy(b);
    return rc;
}

int ads_ivf_destroy(ads_ivf* idx) {
    return guard([&] {
        if (!idx) return;
        idx->ctx->use();
        cudaStreamSynchronize(idx->ctx->stream);
        delete idx;
    });
}

int ads_ivf_meta(ads_ivf* x, int64_t* meta) {
    return guard([&] {
        meta[0] = x->n;
        meta[1] = x->d;
        meta[2] = x->k;
        meta[3] = x->d1;
        meta[4] = x->layout;
        meta[5] = static_cast<int64_t>(x->seed);
        meta[6] = x->has_raw;
    });
}

int ads_ivf_export(ads_ivf* x, float* centroids_t, float* centroids_raw, int64_t* list_off,
                   int32_t* ids_flat, float* a1_t, float* a2_t, float* a1_raw, float* a2_raw) {
    return guard([&] {
        x->ctx->use();
        cudaStream_t st = x->ctx->stream;
        const size_t n = x->n, D = x->d, d1p = x->d1p, d2p = D - d1p, k = x->k;
        auto down = [&](void* h, const void* d, size_t bytes) {
            if (h && d && bytes) ADS_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
        };
        down(centroids_t, x->cent_t, sizeof(float) * k * D);
        down(centroids_raw, x->cent_raw, sizeof(float) * k * D);
        down(list_off, x->list_off, sizeof(int64_t) * (k + 1));
        down(ids_flat, x->ids, sizeof(int32_t) * n);
        down(a1_t, x->a1_t, sizeof(float) * n * d1p);
        down(a2_t, x->a2_t, sizeof(float) * n * d2p);
        down(a1_raw, x->a1_raw, sizeof(float) * n * d1p);
        down(a2_raw, x->a2_raw, sizeof(float) * n * d2p);
        ADS_CUDA(cudaStreamSynchronize(st));
    });
}

void ads_search_opts_default(ads_search_opts* o) {
    o->first = 0;          // 0 -> K
    o->step = 0;           // 0 -> 64 * warps_per_cta
    o->warps_per_cta = 0;  // 0 -> 4 for D <= 256, else 8
    o->queries_per_cta = 4;
    o->ctas_per_sm = 0;
    o->time_stages = 0;
    o->scheduler = 0;
    o->tile = 64;
    o->query_order = 2;
    o->coarse_mode = 0;
    o->rotate_mode = 2;
    o->probe_lo = 0;
    o->r0 = nullptr;
    o->walk = 0;
    o->lag = 0;
}

namespace {

DevSegPlan& ivf_plan(ads_ivf* x, int mode, double eps0, int dd) {
    const bool fd = mode == ADS_MODE_FD;
    const PlanKey key{mode, fd ? 0.0 : eps0, fd ? 0 : dd};
    auto it = x->plans.find(key);
    if (it != x->plans.end()) return *it->second;
    const int D = x->d;
    const bool split = mode == ADS_MODE_AD_SPLIT || mode == ADS_MODE_PD_SPLIT;
    SegPlan p;
    if (fd) {
        p = make_seg_plan(D, x->d1p, {}, nullptr);
    } else {
        const std::vector<int> tests = test_points(D, dd, split ? x->d1 : 0, split);
        if (mode == ADS_MODE_AD || mode == ADS_MODE_AD_SPLIT) {
            const std::vector<double> f = ad_factor(eps0, dd, D);
            p = make_seg_plan(D, x->d1p, tests, f.data());
        } else {
            p = make_seg_plan(D, x->d1p, tests, nullptr);
        }
    }
    auto dp = std::make_unique<DevSegPlan>();
    dp->upload(p, x->ctx->stream);
    DevSegPlan& ref = *dp;
    x->plans.emplace(key, std::move(dp));
    return ref;
}

void validate_search(ads_ivf* x, bool has_qt, bool has_qraw, int32_t K, int32_t nprobe, int32_t mode,
                     double eps0, int32_t dd) {
    // ivf.cpp:299-307, then AdContext (ivf.cpp:313 -> dco.cpp:32-37).
    require(K >= 1, "ivf_query: K must be >= 1");
    require(nprobe >= 1 && nprobe <= x->k, "ivf_query: n_probe must be in [1, k_clusters]");
    require(mode >= 0 && mode <= 4, "ivf_query: unknown mode");
    const bool split = mode == ADS_MODE_AD_SPLIT || mode == ADS_MODE_PD_SPLIT;
    require(!split || x->layout == 1, "ivf_query: split mode needs a split-layout index");
    const bool transformed = mode == ADS_MODE_AD || mode == ADS_MODE_AD_SPLIT;
    if (transformed) {
        require(has_qt || (has_qraw && x->P), "ivf_query: missing query vector");
        (void)ad_factor(eps0, dd, x->d);
    } else {
        require(has_qraw, "ivf_query: missing query vector");
        require(x->has_raw, "ivf_query: index holds no raw vectors for this mode");
        if (mode != ADS_MODE_FD) require(dd >= 1, "ivf_query: delta_d must be >= 1");
    }
}

// Search options with their defaults resolved (all but the refresh step, which
// plan_scan picks with the kernel).
ads_search_opts resolve_opts(ads_ivf* x, int32_t K, int32_t nprobe, const ads_search_opts* opts) {
    ads_search_opts o;
    ads_search_opts_default(&o);
    if (opts) o = *opts;
    if (o.first <= 0) o.first = K;
    // auto launch shape: CTAs of 4 warps for D <= 256; wider CTAs amortise the
    // larger per-query shared state (staged query, chunk slots) at high D.
    require(o.scheduler == 0, "search: scheduler must be 0 (query-major; the list-major scheduler was removed)");
    // 8-warp CTAs above D = 256: with one prefix buffer (no untested prefix to pre-walk)
    // four fit per SM, 32 warps (config 3: +2.5 % over 3 x 10 warps, profiles/r02/ab_w)
    if (o.warps_per_cta <= 0) o.warps_per_cta = x->d <= 256 ? 4 : 8;
    require(o.warps_per_cta >= 1 && o.warps_per_cta <= 32, "search: warps_per_cta in [1, 32]");
    require(o.probe_lo >= 0 && o.probe_lo <= nprobe, "ivf_query: probe_lo must be in [0, n_probe]");
    require(o.queries_per_cta >= 1 && o.queries_per_cta <= 16, "search: queries_per_cta in [1, 16]");
    return o;
}

// The scan's launch choices for one search (shared by search_device and
// ads_ivf_search_plan): the index arrays, the segment plan, the dense prefix phase, the
// lane walk and the threshold refresh schedule.  o has its defaults resolved except step.
void plan_scan(ads_ivf* x, int32_t K, int32_t nprobe, int32_t mode, double eps0, int32_t dd,
               const ads_search_opts& o, SearchLaunch& a) {
    const bool transformed = mode == ADS_MODE_AD || mode == ADS_MODE_AD_SPLIT;
    const int D = x->d;
    DevSegPlan& plan = ivf_plan(x, mode, eps0, dd);
    a.a1 = transformed ? x->a1_t : x->a1_raw;
    a.a2 = transformed ? x->a2_t : x->a2_raw;
    a.d1 = x->d1p;
    a.D = D;
    a.ids = x->ids;
    a.list_off = x->list_off;
    a.nprobe = nprobe;
    a.probe_lo = o.probe_lo;
    a.final_fd = mode == ADS_MODE_FD;
    a.segs = plan.segs;
    a.tfac = plan.tfac;
    a.nseg = plan.nseg;
    a.ntest = plan.ntest;
    a.vec = plan.vec;
    a.full = plan.full;
    a.nseg0 = plan.nseg0;
    // 16-byte line descriptors address A1|A2 (one allocation) in 32 bits of
    // 16-byte units from a1.
    const int64_t gap = a.a2 - a.a1;
    const int64_t units = (gap + static_cast<int64_t>(x->n) * (D - x->d1p)) / 4;
    a.a2_16 = static_cast<uint32_t>(gap / 4);
    if (gap < 0 || gap % 4 != 0 || units >= int64_t(0xffffffff)) {
        a.vec = 1;
        a.full = 0;
    }
    a.warps = o.warps_per_cta;
    // dense prefix phase (ivf.cu): IVF++ on the transformed split layout with a 32-float
    // A1 whose end is the first test point (D > d1); opts.tile = -1 turns it off (A/B runs)
    a.a1i = (mode == ADS_MODE_AD_SPLIT && x->a1i_t && a.vec == 4 && o.tile >= 0 && D > x->d1p) ? x->a1i_t : nullptr;
    // certified fp32 walk (ivf.cu): requested with walk = 2 (walk 0 keeps the exact walk)
    require(o.walk >= 0 && o.walk <= 2, "search: walk must be 0, 1 or 2");
    // walk 0 picks it when a query streams >= 32 000 candidates on average: positives, which
    // the fp32 walk must re-walk exactly, are then a small fraction of the stream (config 5:
    // 390 000 candidates, ~0.2 % positives, +5 %; its 8-way shards' second wave, 43 000:
    // 19.8 vs 21.6 ms; config 2: 15 600 candidates, -1 to -3 %; profiles/r02/ab_f32_walk.log,
    // r02o_shard_projection)
    // (for a shard: its rows over all k lists, i.e. the candidates this rank streams)
    const double cand_per_query = static_cast<double>(x->n) / x->k * (nprobe - o.probe_lo);
    const bool want_f32 = o.walk == 2 || (o.walk == 0 && cand_per_query >= 32000.0);
    a.f32 = (want_f32 && a.vec == 4 && a.full && mode == ADS_MODE_AD_SPLIT) ? 1 : 0;
    // threshold refresh: first = K; step (candidates per chunk) by kernel shape, from
    // same-box sweeps (profiles/r02/ab_rewalk_step, r02k): 64 per warp for the exact walk
    // at D <= 256 (config 2: 384 / 512 measured -1 / -4 %), 128 per warp above (config 3
    // at 8 warps: 768 -1.2 %, 1024 best; refreshing less often costs dims: +2 % at 1280
    // with 10 warps, profiles/r02/ab_step1), 128 per warp for the dense + fp32 walk, whose compact
    // chunk state keeps 9 CTAs per SM at 512 (config 5: +10 %; 768 +0.5 % at 8 CTAs)
    require(o.lag >= -1 && o.lag <= 1, "search: lag must be -1, 0 or 1");
    // overlapped chunks (ivf_search_lag_kernel): where the plain exact lane walk runs; two
    // chunk states in shared memory, so half the refresh step.  lag 0 takes them when the
    // engine also picks the schedule (step 0, no probe range / initial radius) and walks are
    // long (>= 8 segments; config 3: 61.4 -> 57.2 ms, profiles/r02/ab_tail/ab_lag_planes.log);
    // a caller that pins first / step gets exactly that schedule unless it sets lag = 1.
    const bool lag_ok = a.vec == 4 && !a.f32 && !a.a1i && a.nseg0 == 0;
    const bool lag_auto = o.lag == 0 && o.step <= 0 && o.probe_lo == 0 && o.r0 == nullptr && a.nseg >= 8;
    a.lag = (lag_ok && (o.lag == 1 || lag_auto)) ? 1 : 0;
    a.first = o.first;
    const int64_t per_warp = (a.a1i && a.f32) ? 128 : (D > 256 ? 128 : 64);
    a.step = o.step > 0 ? o.step : per_warp * o.warps_per_cta / (a.lag ? 2 : 1);
}

void search_device(ads_ivf* x, const float* dQt, const float* dQraw, int32_t nq, int32_t K,
                   int32_t nprobe, int32_t mode, double eps0, int32_t dd, const ads_search_opts* opts,
                   int32_t* dids, double* ddists, int32_t* dcnt, uint64_t* ddims, uint64_t* dcand) {
    const ads_search_opts o = resolve_opts(x, K, nprobe, opts);
    cudaStream_t st = x->ctx->stream;
    const bool transformed = mode == ADS_MODE_AD || mode == ADS_MODE_AD_SPLIT;
    const int D = x->d;
    x->timed = o.time_stages != 0;
    if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[0], st));
    const float* Qs = transformed ? dQt : dQraw;
    if (transformed && !dQt) {  // rotate on device (apply, transform.cpp:99-117)
        float* qr = x->qrot.get<float>(static_cast<size_t>(nq) * D);
        require(o.rotate_mode >= 0 && o.rotate_mode <= 2, "search: rotate_mode must be 0, 1 or 2");
        // 2 (default): the tensor cores for batches (the north star's transform on tcgen05),
        // the exact fp64 rotation for small batches or shapes the GEMM does not take
        const bool tc_rot = o.rotate_mode == 1 || (o.rotate_mode == 2 && D % 4 == 0 && D >= 32 && nq >= 64);
        if (tc_rot) {  // 3xTF32 tensor cores (tc_gemm.cu)
            require(D % 4 == 0 && D >= 32, "rotate_mode 1: dimension must be a multiple of 4 and >= 32");
            const size_t dd = static_cast<size_t>(D) * D;
            if (!x->p_split) {
                std::vector<double> hp(dd);
                ADS_CUDA(cudaMemcpyAsync(hp.data(), x->P, sizeof(double) * dd, cudaMemcpyDeviceToHost, st));
                ADS_CUDA(cudaStreamSynchronize(st));
                std::vector<float> pf(hp.begin(), hp.end());
                float* p32 = x->qh.get<float>(dd);
                ADS_CUDA(cudaMemcpyAsync(p32, pf.data(), sizeof(float) * dd, cudaMemcpyHostToDevice, st));
                launch_split_tf32(p32, static_cast<int64_t>(dd), x->ph.get<float>(dd), x->pl.get<float>(dd), st);
                ADS_CUDA(cudaStreamSynchronize(st));
                x->p_split = true;
            }
            launch_tc_transform(dQraw, nq, x->ph.get<float>(dd), x->pl.get<float>(dd), D, qr, x->qh, x->ql, st);
        } else {
            launch_apply(x->P, D, dQraw, nq, qr, st);
        }
        Qs = qr;
    }
    if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[1], st));
    int32_t* probes = x->probes.get<int32_t>(static_cast<size_t>(nq) * nprobe);
    const float* cent = transformed ? x->cent_t : x->cent_raw;
    if (o.coarse_mode == 0 || o.coarse_mode == 2) {  // certified prefilter + exact fp64 rescoring (coarse.cu)
        launch_coarse_probes_fast(Qs, nq, cent, x->k, D, nprobe, transformed ? x->cc_t : x->cc_raw,
                                  x->coarse, probes, o.coarse_mode == 2 ? 1 : 0, st);
        if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[2], st));
    } else {  // exact fp64 distance to every centroid, then select
        double* dist = x->dist.get<double>(static_cast<size_t>(nq) * x->k);
        launch_coarse_dist(Qs, nq, cent, x->k, D, dist, st);
        if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[2], st));
        launch_select_probes(dist, nq, x->k, nprobe, probes, st);
    }
    if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[3], st));
    SearchLaunch a{};
    plan_scan(x, K, nprobe, mode, eps0, dd, o, a);
    a.Q = Qs;
    a.nq = nq;
    a.probes = probes;
    a.r0 = o.r0;
    a.K = K;
    a.slots = o.queries_per_cta;
    a.ctas_per_sm = o.ctas_per_sm;
    a.out_ids = dids;
    a.out_dists = ddists;
    a.out_cnt = dcnt;
    a.out_dims = reinterpret_cast<unsigned long long*>(ddims);
    a.out_cand = reinterpret_cast<unsigned long long*>(dcand);
    a.counter = x->ctx->counter;
    a.order = nullptr;

    // longest queries first; pointless when the whole batch is resident at once
    if (o.query_order == 2 && nq > 1 && nq > search_resident_ctas(a)) {
        int32_t* ord = x->order.get<int32_t>(nq);
        launch_query_order_work(probes, nq, nprobe, o.probe_lo, a.list_off, x->order_tmp, ord, st);
        a.order = ord;
    } else if (o.query_order == 1 && x->chain_rank && nq > 1) {
        int32_t* ord = x->order.get<int32_t>(nq);
        launch_query_order(probes, nq, nprobe, x->chain_rank, x->k, x->order_tmp, ord, st);
        a.order = ord;
    }
    launch_ivf_search(a, st);
    if (x->timed) ADS_CUDA(cudaEventRecord(x->ev[4], st));
}

}  // namespace

int ads_ivf_search_device(ads_ivf* x, const float* dQt, const float* dQraw, int32_t nq, int32_t K,
                          int32_t nprobe, int32_t mode, double eps0, int32_t dd,
                          const ads_search_opts* opts, int32_t* dids, double* ddists,
                          int32_t* dcnt, uint64_t* ddims, uint64_t* dcand) {
    return guard([&] {
        validate_search(x, dQt != nullptr, dQraw != nullptr, K, nprobe, mode, eps0, dd);
        x->ctx->use();
        std::lock_guard<std::mutex> lk(x->ctx->mu);
        search_device(x, dQt, dQraw, nq, K, nprobe, mode, eps0, dd, opts, dids, ddists, dcnt, ddims, dcand);
    });
}

int ads_ivf_search_plan(ads_ivf* x, int32_t K, int32_t nprobe, int32_t mode, double eps0, int32_t dd,
                        const ads_search_opts* opts, int64_t* first, int64_t* step, int32_t* warps_per_cta,
                        int32_t* walk, int32_t* dense, int32_t* lag) {
    return guard([&] {
        validate_search(x, true, true, K, nprobe, mode, eps0, dd);
        x->ctx->use();
        std::lock_guard<std::mutex> lk(x->ctx->mu);
        const ads_search_opts o = resolve_opts(x, K, nprobe, opts);
        SearchLaunch a{};
        plan_scan(x, K, nprobe, mode, eps0, dd, o, a);
        if (first) *first = a.first;
        if (step) *step = a.step;
        if (warps_per_cta) *warps_per_cta = a.warps;
        if (walk) *walk = a.f32 ? 2 : 1;
        if (dense) *dense = a.a1i ? 1 : 0;
        if (lag) *lag = a.lag;
    });
}

int ads_ivf_search(ads_ivf* x, const float* Qt, const float* Qraw, int32_t nq, int32_t K,
                   int32_t nprobe, int32_t mode, double eps0, int32_t dd, const ads_search_opts* opts,
                   int32_t* ids, double* dists, int32_t* counts, uint64_t* dims, uint64_t* cands) {
    return guard([&] {
        const bool transformed = mode == ADS_MODE_AD || mode == ADS_MODE_AD_SPLIT;
        const bool use_qt = transformed && Qt != nullptr;
        const bool use_qraw = Qraw != nullptr && (!transformed || !use_qt);
        validate_search(x, Qt != nullptr, Qraw != nullptr, K, nprobe, mode, eps0, dd);
        require(nq >= 0, "ivf_query: nq must be >= 0");
        x->ctx->use();
        std::lock_guard<std::mutex> lk(x->ctx->mu);
        cudaStream_t st = x->ctx->stream;
        const size_t qn = static_cast<size_t>(nq) * x->d;
        float* dqt = use_qt ? x->qin_t.get<float>(qn) : nullptr;
        float* dqr = use_qraw ? x->qin_raw.get<float>(qn) : nullptr;
        if (dqt) ADS_CUDA(cudaMemcpyAsync(dqt, Qt, qn * sizeof(float), cudaMemcpyHostToDevice, st));
        if (dqr) ADS_CUDA(cudaMemcpyAsync(dqr, Qraw, qn * sizeof(float), cudaMemcpyHostToDevice, st));
        const size_t rk = static_cast<size_t>(nq) * K;
        int32_t* di = x->o_ids.get<int32_t>(rk);
        double* dd_ = x->o_dists.get<double>(rk);
        int32_t* dc = x->o_cnt.get<int32_t>(nq);
        uint64_t* dm = x->o_dims.get<uint64_t>(nq);
        uint64_t* dn = x->o_cand.get<uint64_t>(nq);
        ads_search_opts o;
        ads_search_opts_default(&o);
        if (opts) o = *opts;
        if (o.r0 && nq > 0) {  // host radii -> device
            double* dr = x->r0buf.get<double>(nq);
            ADS_CUDA(cudaMemcpyAsync(dr, o.r0, sizeof(double) * nq, cudaMemcpyHostToDevice, st));
            o.r0 = dr;
        }
        if (nq > 0)
            search_device(x, dqt, dqr, nq, K, nprobe, mode, eps0, dd, &o, di, dd_, dc, dm, dn);
        auto down = [&](void* h, const void* d, size_t bytes) {
            if (h && bytes) ADS_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
        };
        down(ids, di, rk * sizeof(int32_t));
        down(dists, dd_, rk * sizeof(double));
        down(counts, dc, nq * sizeof(int32_t));
        down(dims, dm, nq * sizeof(uint64_t));
        down(cands, dn, nq * sizeof(uint64_t));
        ADS_CUDA(cudaStreamSynchronize(st));
    });
}

int ads_ivf_probe_order(ads_ivf* x, const float* Q, int32_t nq, int32_t nprobe, int32_t transformed,
                        int32_t* probes) {
    return guard([&] {
        require(nprobe >= 1 && nprobe <= x->k, "ivf_query: n_probe must be in [1, k_clusters]");
        require(transformed || x->has_raw, "probe_order: no raw centroids");
        x->ctx->use();
        std::lock_guard<std::mutex> lk(x->ctx->mu);
        cudaStream_t st = x->ctx->stream;
        const size_t qn = static_cast<size_t>(nq) * x->d;
        float* dq = x->qin_t.get<float>(qn);
        ADS_CUDA(cudaMemcpyAsync(dq, Q, qn * sizeof(float), cudaMemcpyHostToDevice, st));
        int32_t* dp = x->probes.get<int32_t>(static_cast<size_t>(nq) * nprobe);
        launch_coarse_probes_fast(dq, nq, transformed ? x->cent_t : x->cent_raw, x->k, x->d, nprobe,
                                  transformed ? x->cc_t : x->cc_raw, x->coarse, dp, 0, st);
        ADS_CUDA(cudaMemcpyAsync(probes, dp, sizeof(int32_t) * nq * nprobe, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
    });
}

int ads_ivf_coarse_stats(ads_ivf* idx, uint64_t* out) {
    return guard([&] {
        idx->ctx->use();
        std::lock_guard<std::mutex> lk(idx->ctx->mu);
        unsigned long long h[2] = {0, 0};
        if (idx->coarse.stats.p) {
            ADS_CUDA(cudaStreamSynchronize(idx->ctx->stream));
            ADS_CUDA(cudaMemcpy(h, idx->coarse.stats.p, sizeof(h), cudaMemcpyDeviceToHost));
        }
        out[0] = static_cast<uint64_t>(idx->coarse.last_nq);
        out[1] = h[0];
        out[2] = h[1];
    });
}

int ads_ivf_subset(ads_ivf* src, const uint8_t* keep, ads_ivf** out) {
    return guard([&] {
        ads_ctx* ctx = src->ctx;
        ctx->use();
        cudaStream_t st = ctx->stream;
        const int k = src->k, D = src->d, d1p = src->d1p, d2p = D - d1p;
        std::vector<int64_t> off(static_cast<size_t>(k) + 1);
        ADS_CUDA(cudaMemcpyAsync(off.data(), src->list_off, sizeof(int64_t) * (k + 1),
                                 cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> noff(static_cast<size_t>(k) + 1, 0);
        for (int c = 0; c < k; ++c) noff[c + 1] = noff[c] + (keep[c] ? off[c + 1] - off[c] : 0);
        const int64_t nl = noff[k];
        auto x = std::make_unique<ads_ivf>();
        x->ctx = ctx;
        x->n = static_cast<int>(nl);
        x->d = D;
        x->k = k;
        x->d1 = src->d1;
        x->layout = src->layout;
        x->seed = src->seed;
        x->d1p = d1p;
        x->has_raw = src->has_raw;
        ivf_alloc_common(x.get());
        const size_t nn = static_cast<size_t>(nl > 0 ? nl : 1);
        ADS_CUDA(cudaMalloc(&x->cent_t, sizeof(float) * k * static_cast<size_t>(D)));
        ADS_CUDA(cudaMemcpyAsync(x->cent_t, src->cent_t, sizeof(float) * k * static_cast<size_t>(D),
                                 cudaMemcpyDeviceToDevice, st));
        x->list_off = dev_upload(noff.data(), noff.size(), st);
        ADS_CUDA(cudaMalloc(&x->ids, sizeof(int32_t) * nn));
        alloc_split_pair(nn, d1p, d2p, &x->a1_t, &x->a2_t);
        if (x->has_raw) {
            ADS_CUDA(cudaMalloc(&x->cent_raw, sizeof(float) * k * static_cast<size_t>(D)));
            ADS_CUDA(cudaMemcpyAsync(x->cent_raw, src->cent_raw, sizeof(float) * k * static_cast<size_t>(D),
                                     cudaMemcpyDeviceToDevice, st));
            alloc_split_pair(nn, d1p, d2p, &x->a1_raw, &x->a2_raw);
        }
        if (src->chain_rank) {
            ADS_CUDA(cudaMalloc(&x->chain_rank, sizeof(int32_t) * k));
            ADS_CUDA(cudaMemcpyAsync(x->chain_rank, src->chain_rank, sizeof(int32_t) * k, cudaMemcpyDeviceToDevice, st));
        }
        if (src->P) {
            ADS_CUDA(cudaMalloc(&x->P, sizeof(double) * D * static_cast<size_t>(D)));
            ADS_CUDA(cudaMemcpyAsync(x->P, src->P, sizeof(double) * D * static_cast<size_t>(D),
                                     cudaMemcpyDeviceToDevice, st));
        }
        ivf_finish_coarse(x.get(), st);
        // owned lists are contiguous row ranges in every flat array: one copy per run of
        // consecutive owned lists
        for (int c = 0; c < k;) {
            if (!keep[c]) {
                ++c;
                continue;
            }
            int e = c;
            while (e < k && keep[e]) ++e;
            const int64_t so = off[c], cnt = off[e] - off[c], dofs = noff[c];
            if (cnt > 0) {
                auto cp = [&](void* dst, const void* srcp, size_t w) {
                    ADS_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + dofs * w,
                                             static_cast<const char*>(srcp) + so * w, cnt * w,
                                             cudaMemcpyDeviceToDevice, st));
                };
                cp(x->ids, src->ids, sizeof(int32_t));
                cp(x->a1_t, src->a1_t, sizeof(float) * d1p);
                if (d2p) cp(x->a2_t, src->a2_t, sizeof(float) * d2p);
                if (x->has_raw) {
                    cp(x->a1_raw, src->a1_raw, sizeof(float) * d1p);
                    if (d2p) cp(x->a2_raw, src->a2_raw, sizeof(float) * d2p);
                }
            }
            c = e;
        }
        ivf_finish_dense(x.get(), st);
        ADS_CUDA(cudaStreamSynchronize(st));
        *out = x.release();
    });
}

int ads_merge_topk_device(ads_ctx* ctx, const double* ddists, const int32_t* dids, int32_t G,
                          int32_t nq, int32_t K, int32_t* dout_ids, double* dout_dists,
                          int32_t* dout_counts) {
    return guard([&] {
        require(G >= 1 && K >= 1 && nq >= 0, "merge_topk: bad shape");
        ctx->use();
        launch_merge_topk(ddists, dids, G, nq, K, dout_ids, dout_dists, dout_counts, ctx->stream);
    });
}

int ads_merge_topk(ads_ctx* ctx, const double* dists, const int32_t* ids, int32_t G, int32_t nq,
                   int32_t K, int32_t* out_ids, double* out_dists, int32_t* out_counts) {
    return guard([&] {
        require(G >= 1 && K >= 1 && nq >= 0, "merge_topk: bad shape");
        ctx->use();
        cudaStream_t st = ctx->stream;
        const size_t in = static_cast<size_t>(G) * nq * K, o = static_cast<size_t>(nq) * K;
        DevBuf bd, bi, boi, bod, boc;
        const double* dd = buf_upload(bd, dists, in, st);
        const int32_t* di = buf_upload(bi, ids, in, st);
        int32_t* oi = boi.get<int32_t>(o);
        double* od = bod.get<double>(o);
        int32_t* oc = boc.get<int32_t>(nq);
        launch_merge_topk(dd, di, G, nq, K, oi, od, oc, st);
        ADS_CUDA(cudaMemcpyAsync(out_ids, oi, sizeof(int32_t) * o, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaMemcpyAsync(out_dists, od, sizeof(double) * o, cudaMemcpyDeviceToHost, st));
        if (out_counts) ADS_CUDA(cudaMemcpyAsync(out_counts, oc, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st));
        ADS_CUDA(cudaStreamSynchronize(st));
    });
}

int ads_ivf_last_timings(ads_ivf* x, float* ms4) {
    return guard([&] {
        require(x->timed, "no timed search recorded (set opts.time_stages)");
        x->ctx->use();
        ADS_CUDA(cudaEventSynchronize(x->ev[4]));
        for (int i = 0; i < 4; ++i) ADS_CUDA(cudaEventElapsedTime(&ms4[i], x->ev[i], x->ev[i + 1]));
    });
}

}  // extern "C"

// Fixed-threshold batched DCO kernel: one ad_scan / pd_scan_kernel / l2_sq
// per (query, candidate row) against a caller-given per-query threshold r
// (dco.hpp:86-177; the fixed-threshold study bench.cpp:303-392; BASELINE
// config 4).  Persistent CTAs pull tiles (query, candidate range) from a
// global counter; warps refill lanes from the tile with a shared counter.
#include "engine.hpp"
#include "scan_engine.cuh"

namespace ads {

namespace {

constexpr int kDcoWarps = 4;
#ifndef DCO_MIN_CTAS
#define DCO_MIN_CTAS 8  // resident CTAs per SM the descriptor kernel is compiled for (<= 64 registers)
#endif

struct DcoSmem {
    double r, r_sq;
    int64_t tile_q, tile_lo, tile_hi, base;
    int next;
    int stop;
};

// DESC: lines addressed by 32-bit descriptors (row * D/4 + col/4, 16-byte units from X)
// and gathered asynchronously like the IVF scan (gather_issue16), every segment 32 floats.
template <int VEC, bool DESC>
__global__ void __launch_bounds__(kDcoWarps * 32, DESC ? DCO_MIN_CTAS : 1) dco_fixed_kernel(DcoLaunch a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];  // gather rows: 128-byte aligned (swizzle)
    __shared__ DcoSmem sh;
    // dynamic smem: wbuf [warps*1024 floats] | qseg [nseg*33 doubles] | thr [ntest] | segs [nseg]
    float* wbuf_all = reinterpret_cast<float*>(smem_raw);
    if (threadIdx.x == 0 && (__cvta_generic_to_shared(smem_raw) & 127u)) __trap();  // swizzle needs 128-B rows
    double* qseg = reinterpret_cast<double*>(wbuf_all + kDcoWarps * 1024);
    double* thr = qseg + a.nseg * kQPitch;
    Seg* segs = reinterpret_cast<Seg*>(thr + (a.ntest > 0 ? a.ntest : 1));

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    float* wbuf = wbuf_all + warp * 1024;
    for (int i = threadIdx.x; i < a.nseg; i += blockDim.x) segs[i] = a.segs[i];
    const char* gbase = lane_base16(a.X);
    const uint32_t rstr = static_cast<uint32_t>(a.D) >> 2;

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t t = static_cast<int64_t>(atomicAdd(a.counter, 1ull));
            sh.stop = t >= a.ntiles;
            if (!sh.stop) {
                if (a.tile_q) {
                    sh.tile_q = a.tile_q[t];
                    sh.tile_lo = a.tile_lo[t];
                    sh.tile_hi = a.tile_hi[t];
                    sh.base = a.cand_off[sh.tile_q];
                } else {
                    const int64_t tpq = (a.win_len + a.tile - 1) / a.tile;
                    sh.tile_q = t / tpq;
                    sh.tile_lo = (t % tpq) * a.tile;
                    sh.tile_hi = sh.tile_lo + a.tile < a.win_len ? sh.tile_lo + a.tile : a.win_len;
                    sh.base = sh.tile_q * a.win_len;
                }
                const double r = a.r[sh.tile_q];
                sh.r = r;
                sh.r_sq = __dmul_rn(r, r);  // dco.hpp:125
                sh.next = static_cast<int>(sh.tile_lo);
            }
        }
        __syncthreads();
        if (sh.stop) break;
        const int64_t q = sh.tile_q;
        stage_query(qseg, segs, a.nseg, a.Q + q * a.D);
        for (int i = threadIdx.x; i < a.ntest; i += blockDim.x) thr[i] = __dmul_rn(a.tfac[i], sh.r_sq);
        __syncthreads();

        const int hi = static_cast<int>(sh.tile_hi);
        const double r = sh.r, r_sq = sh.r_sq;
        int64_t row = -1;
        int j = -1, seg = 0;
        double s = 0.0;
        unsigned long long my_dims = 0;
        for (;;) {
            const unsigned need = __ballot_sync(kFull, j < 0);
            if (need) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&sh.next, __popc(need));
                base = __shfl_sync(kFull, base, 0);
                if (j < 0) {
                    const int cand = base + __popc(need & ((1u << lane) - 1u));
                    if (cand < hi) {
                        j = cand;
                        if (a.cand_rows) {
                            row = a.cand_rows[sh.base + cand];
                        } else {
                            row = a.win_start[q] + cand;
                            row %= a.n_rows;
                        }
                        seg = 0;
                        s = 0.0;
                    }
                }
            }
            if (!__any_sync(kFull, j >= 0)) break;
            Seg sg = segs[seg];
            if constexpr (DESC) {
                const uint32_t dsc = j >= 0 ? static_cast<uint32_t>(row) * rstr + (static_cast<uint32_t>(sg.col) >> 2)
                                            : kNoLine;
                gather_issue16<true>(wbuf, gbase, dsc, 8);
                cp_async_wait_group<0>();
                __syncwarp();
            } else {
                const float* src = a.X + row * a.D + sg.col;
                gather_lines<VEC>(wbuf, src, j >= 0 ? sg.len : 0);
            }
            if (j >= 0) {
                s = accumulate_line<VEC, DESC>(wbuf, qseg + seg * kQPitch, sg.len, s);
                const int d = sg.col + sg.len;
                bool done = false, pos = false;
                double obs = 0.0;
                if (sg.test >= 0 && s > thr[sg.test]) {  // dco.hpp:141
                    done = true;
                    obs = a.kind == 2 ? __dsqrt_rn(__ddiv_rn(__dmul_rn(s, static_cast<double>(a.D)),
                                                              static_cast<double>(d)))
                                      : __dsqrt_rn(s);
                } else if (seg == a.nseg - 1) {  // d == D: exact (dco.hpp:145, dco.cpp:70-81)
                    done = true;
                    obs = __dsqrt_rn(s);
                    pos = a.kind == 0 ? obs <= r : s <= r_sq;
                }
                if (done) {
                    const int64_t g = sh.base + j;
                    if (a.positive) a.positive[g] = pos;
                    if (a.dims) a.dims[g] = d;
                    if (a.dist_sq) a.dist_sq[g] = pos ? s : __longlong_as_double(0x7ff8000000000000ll);
                    if (a.observed) a.observed[g] = obs;
                    my_dims += static_cast<unsigned long long>(d);
                    j = -1;
                } else {
                    ++seg;
                }
            }
        }
        if (a.dims_per_query) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) my_dims += __shfl_xor_sync(kFull, my_dims, o);
            if (lane == 0 && my_dims) atomicAdd(a.dims_per_query + q, my_dims);
        }
    }
}

// Partial squared distances at every Δd boundary and at D for rows cand[0..nc)
// against one query (the sums ad_scan / pd_scan_kernel test, dco.hpp:122-177,
// in their order: fp64, index order, separate roundings).  One thread per row;
// the graph search (HNSW) replays the reference's decisions from them with the
// threshold in force at each comparison.
__global__ void prefix_sums_kernel(const float* __restrict__ X, int D, const float* __restrict__ q,
                                   const int64_t* __restrict__ cand, int nc, int dd, int nb,
                                   double* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    const float* x = X + cand[c] * static_cast<int64_t>(D);
    double s = 0.0;
    int t = 0;
    for (int j = 0; j < D; ++j) {
        s = sq_diff_acc(s, x[j], static_cast<double>(q[j]));
        if ((j + 1) % dd == 0 || j + 1 == D) out[static_cast<int64_t>(c) * nb + t++] = s;
    }
}

}  // namespace

void launch_prefix_sums(const float* X, int D, const float* q, const int64_t* cand, int nc, int dd,
                        double* out, cudaStream_t st) {
    if (nc <= 0) return;
    const int nb = (D + dd - 1) / dd;
    prefix_sums_kernel<<<(nc + 127) / 128, 128, 0, st>>>(X, D, q, cand, nc, dd, nb, out);
    ADS_LAUNCH_CHECK();
}

void launch_dco_fixed(const DcoLaunch& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * kDcoWarps * 1024 + sizeof(double) * a.nseg * kQPitch +
                        sizeof(double) * (a.ntest > 0 ? a.ntest : 1) + sizeof(Seg) * a.nseg;
    auto kern = a.vec == 4 ? (a.desc ? dco_fixed_kernel<4, true> : dco_fixed_kernel<4, false>)
                           : dco_fixed_kernel<1, false>;
    ADS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    int occ = 0;
    ADS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDcoWarps * 32, smem));
    if (occ < 1) throw std::invalid_argument("dco: dimension too large for shared memory");
    ADS_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st));
    int64_t grid = static_cast<int64_t>(num_sms()) * occ;
    if (grid > a.ntiles) grid = a.ntiles;
    if (grid < 1) return;
    kern<<<static_cast<unsigned>(grid), kDcoWarps * 32, smem, st>>>(a);
    ADS_LAUNCH_CHECK();
}

}  // namespace ads

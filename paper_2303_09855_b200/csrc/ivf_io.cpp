// On-disk IVF index interop with the reference (save_ivf / load_ivf,
// ivf.hpp:91-92, ivf.cpp:423-501): a directory with meta.txt (key=value lines)
// and fvecs / ragged ivecs files (vecio.cpp:55-171: every record is an int32
// count followed by that many float32 / int32 values).  Host code over the C
// ABI's own index create/export, so a directory written by the reference loads
// into the engine and the reverse.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/adsann_b200.h"

namespace fs = std::filesystem;

namespace {

[[noreturn]] void io_fail(const std::string& msg) { throw std::runtime_error(msg); }

// n records of d values (float or int32) from a flat row-major array
template <typename T>
void write_records(const fs::path& p, int64_t n, int32_t d, const T* rows) {
    std::ofstream out(p, std::ios::binary | std::ios::trunc);
    if (!out) io_fail("cannot open " + p.string() + " for writing");
    for (int64_t i = 0; i < n; ++i) {
        out.write(reinterpret_cast<const char*>(&d), 4);
        out.write(reinterpret_cast<const char*>(rows + i * d), static_cast<std::streamsize>(sizeof(T)) * d);
    }
    if (!out) io_fail("write failed: " + p.string());
}

// fixed-width records; returns rows, sets n / d (d = 0 for an empty file)
std::vector<float> read_fixed(const fs::path& p, int64_t& n, int32_t& d) {
    std::ifstream in(p, std::ios::binary);
    if (!in) io_fail("cannot open " + p.string());
    in.seekg(0, std::ios::end);
    const int64_t bytes = in.tellg();
    in.seekg(0);
    n = 0;
    d = 0;
    if (bytes == 0) return {};
    if (!in.read(reinterpret_cast<char*>(&d), 4) || d < 0) io_fail("bad record header in " + p.string());
    const int64_t rec = 4 + 4 * static_cast<int64_t>(d);
    if (rec == 4 || bytes % rec != 0) io_fail("truncated or ragged file " + p.string());
    n = bytes / rec;
    std::vector<float> out(static_cast<size_t>(n) * d);
    in.seekg(0);
    for (int64_t i = 0; i < n; ++i) {
        int32_t di = 0;
        in.read(reinterpret_cast<char*>(&di), 4);
        if (di != d) io_fail("inconsistent dimension in " + p.string());
        in.read(reinterpret_cast<char*>(out.data() + i * d), 4 * static_cast<std::streamsize>(d));
    }
    if (!in) io_fail("read failed: " + p.string());
    return out;
}

std::vector<std::vector<int32_t>> read_ragged(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    if (!in) io_fail("cannot open " + p.string());
    std::vector<std::vector<int32_t>> rows;
    int32_t c = 0;
    while (in.read(reinterpret_cast<char*>(&c), 4)) {
        if (c < 0) io_fail("bad record header in " + p.string());
        rows.emplace_back(static_cast<size_t>(c));
        if (c && !in.read(reinterpret_cast<char*>(rows.back().data()), 4 * static_cast<std::streamsize>(c)))
            io_fail("truncated file " + p.string());
    }
    return rows;
}

}  // namespace

namespace ads {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

template <typename F>
int io_guard(F&& f) {
    try {
        f();
        return ADS_OK;
    } catch (const std::invalid_argument& e) {
        ads::set_last_error(e.what());
        return ADS_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        ads::set_last_error(e.what());
        return ADS_RUNTIME_ERROR;
    }
}

void check(int rc) {
    if (rc != ADS_OK) {
        const std::string m = ads_last_error();
        if (rc == ADS_INVALID_ARGUMENT) throw std::invalid_argument(m);
        throw std::runtime_error(m);
    }
}

}  // namespace

extern "C" {

int ads_ivf_save(ads_ivf* idx, const char* dir_c) {
    return io_guard([&] {
        if (!idx || !dir_c) throw std::invalid_argument("save_ivf: null argument");
        int64_t meta[7];
        check(ads_ivf_meta(idx, meta));
        const int64_t n = meta[0];
        const int32_t d = static_cast<int32_t>(meta[1]), k = static_cast<int32_t>(meta[2]),
                      d1 = static_cast<int32_t>(meta[3]), layout = static_cast<int32_t>(meta[4]);
        const bool has_raw = meta[6] != 0;
        const int32_t d1p = layout == 1 ? d1 : (d > 32 ? 32 : d), d2p = d - d1p;
        std::vector<float> ct(static_cast<size_t>(k) * d), cr(has_raw ? ct.size() : 0);
        std::vector<int64_t> off(static_cast<size_t>(k) + 1);
        std::vector<int32_t> ids(static_cast<size_t>(n));
        std::vector<float> a1t(static_cast<size_t>(n) * d1p), a2t(static_cast<size_t>(n) * d2p);
        std::vector<float> a1r(has_raw ? a1t.size() : 0), a2r(has_raw ? a2t.size() : 0);
        check(ads_ivf_export(idx, ct.data(), has_raw ? cr.data() : nullptr, off.data(), ids.data(), a1t.data(),
                             a2t.data(), has_raw ? a1r.data() : nullptr, has_raw ? a2r.data() : nullptr));
        const fs::path dir(dir_c);
        fs::create_directories(dir);
        {
            std::ofstream m(dir / "meta.txt", std::ios::trunc);
            if (!m) io_fail("cannot open " + (dir / "meta.txt").string() + " for writing");
            m << "n=" << n << "\nd=" << d << "\nk_clusters=" << k << "\nd1=" << d1
              << "\nlayout=" << (layout == 1 ? "split" : "contiguous") << "\nseed=" << static_cast<uint64_t>(meta[5])
              << "\n";
        }
        write_records(dir / "centroids_t.fvecs", k, d, ct.data());
        // An index without raw vectors (config 5) has no raw files: the reference's
        // format has no way to say so (read_fvecs rejects empty files), so such a
        // directory loads into the engine only.
        if (has_raw) write_records(dir / "centroids_raw.fvecs", k, d, cr.data());
        {
            std::ofstream b(dir / "buckets.ivecs", std::ios::binary | std::ios::trunc);
            if (!b) io_fail("cannot open buckets.ivecs for writing");
            for (int32_t c = 0; c < k; ++c) {
                const int32_t cnt = static_cast<int32_t>(off[c + 1] - off[c]);
                b.write(reinterpret_cast<const char*>(&cnt), 4);
                b.write(reinterpret_cast<const char*>(ids.data() + off[c]), 4 * static_cast<std::streamsize>(cnt));
            }
        }
        // contiguous bucket-major rows = A1 | A2 re-joined
        auto joined = [&](const std::vector<float>& a1, const std::vector<float>& a2) {
            std::vector<float> v(static_cast<size_t>(n) * d);
            for (int64_t i = 0; i < n; ++i) {
                std::memcpy(&v[i * d], &a1[i * d1p], 4 * static_cast<size_t>(d1p));
                std::memcpy(&v[i * d + d1p], &a2[i * d2p], 4 * static_cast<size_t>(d2p));
            }
            return v;
        };
        write_records(dir / "vec_t.fvecs", n, d, joined(a1t, a2t).data());
        if (has_raw) write_records(dir / "vec_raw.fvecs", n, d, joined(a1r, a2r).data());
        if (layout == 1) {
            write_records(dir / "a1_t.fvecs", n, d1, a1t.data());
            write_records(dir / "a2_t.fvecs", n, d - d1, a2t.data());
            if (has_raw) {
                write_records(dir / "a1_raw.fvecs", n, d1, a1r.data());
                write_records(dir / "a2_raw.fvecs", n, d - d1, a2r.data());
            }
        }
    });
}

int ads_ivf_load(ads_ctx* ctx, const char* dir_c, const double* P, ads_ivf** out) {
    return io_guard([&] {
        if (!ctx || !dir_c || !out) throw std::invalid_argument("load_ivf: null argument");
        const fs::path dir(dir_c);
        std::ifstream meta(dir / "meta.txt");
        if (!meta) io_fail("cannot open " + (dir / "meta.txt").string());
        int64_t n = 0;
        int32_t d = 0, k = 0, d1 = 0, layout = 0;
        uint64_t seed = 0;
        for (std::string line; std::getline(meta, line);) {
            const auto eq = line.find('=');
            if (eq == std::string::npos) continue;
            const std::string key = line.substr(0, eq), v = line.substr(eq + 1);
            if (key == "n") n = std::stoll(v);
            else if (key == "d") d = std::stoi(v);
            else if (key == "k_clusters") k = std::stoi(v);
            else if (key == "d1") d1 = std::stoi(v);
            else if (key == "layout") layout = v == "split" ? 1 : 0;
            else if (key == "seed") seed = std::stoull(v);
        }
        int64_t r = 0;
        int32_t rd = 0;
        const std::vector<float> ct = read_fixed(dir / "centroids_t.fvecs", r, rd);
        if (r != k || rd != d) io_fail("load_ivf: centroid file does not match metadata");
        const bool raw_c = fs::exists(dir / "centroids_raw.fvecs");
        std::vector<float> cr;
        if (raw_c) {
            cr = read_fixed(dir / "centroids_raw.fvecs", r, rd);
            if (r != k || rd != d) io_fail("load_ivf: raw centroid file does not match metadata");
        }
        const auto buckets = read_ragged(dir / "buckets.ivecs");
        if (static_cast<int32_t>(buckets.size()) != k) io_fail("load_ivf: bucket count does not match metadata");
        std::vector<int64_t> off(static_cast<size_t>(k) + 1, 0);
        std::vector<int32_t> ids;
        ids.reserve(static_cast<size_t>(n));
        for (int32_t c = 0; c < k; ++c) {
            off[c + 1] = off[c] + static_cast<int64_t>(buckets[c].size());
            ids.insert(ids.end(), buckets[c].begin(), buckets[c].end());
        }
        if (static_cast<int64_t>(ids.size()) != n) io_fail("load_ivf: bucket contents do not cover the dataset");
        ads_ivf_desc desc{};
        desc.n = static_cast<int32_t>(n);
        desc.d = d;
        desc.k_clusters = k;
        desc.d1 = d1;
        desc.layout = layout;
        desc.seed = seed;
        desc.centroids_t = ct.data();
        desc.list_off = off.data();
        desc.ids_flat = ids.data();
        desc.P = P;
        std::vector<float> a1t, a2t, a1r, a2r, vt, vr;
        if (layout == 1) {
            a1t = read_fixed(dir / "a1_t.fvecs", r, rd);
            if (r != n || rd != d1) io_fail("load_ivf: a1_t does not match metadata");
            a2t = read_fixed(dir / "a2_t.fvecs", r, rd);
            if (r != n || rd != d - d1) io_fail("load_ivf: a2_t does not match metadata");
            const bool raw = raw_c && fs::exists(dir / "a1_raw.fvecs");
            if (raw) {
                a1r = read_fixed(dir / "a1_raw.fvecs", r, rd);
                a2r = read_fixed(dir / "a2_raw.fvecs", r, rd);
            }
            desc.a1_t = a1t.data();
            desc.a2_t = a2t.data();
            if (raw) {
                desc.a1_raw = a1r.data();
                desc.a2_raw = a2r.data();
                desc.centroids_raw = cr.data();
            }
        } else {
            vt = read_fixed(dir / "vec_t.fvecs", r, rd);
            if (r != n || rd != d) io_fail("load_ivf: vec_t does not match metadata");
            desc.vec_t = vt.data();
            if (raw_c && fs::exists(dir / "vec_raw.fvecs")) {
                vr = read_fixed(dir / "vec_raw.fvecs", r, rd);
                if (r != n || rd != d) io_fail("load_ivf: vec_raw does not match metadata");
                desc.vec_raw = vr.data();
                desc.centroids_raw = cr.data();
            }
        }
        check(ads_ivf_create(ctx, &desc, out));
    });
}

}  // extern "C"

// Drives the facade's HNSW (build_hnsw / save_hnsw / load_hnsw / hnsw_query, DCOs
// on the B200) from files, so tests/test_gpu_hnsw.py can compare it with the
// reference (oracle/_ref) byte for byte: the two cannot share one process (same
// adsann:: symbols).
//   facade_hnsw_tool build RAW.fvecs T.fvecs M EF SEED OUTDIR
//   facade_hnsw_tool query GRAPHDIR RAW.fvecs T.fvecs QRAW.fvecs QT.fvecs K NEF MODE EPS0 DD OUT.bin
// OUT.bin per query: int32 count, K int32 ids, K float64 dists, 4 uint64
// (dims_evaluated, dco_count, hops, candidates).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "adsann/hnsw.hpp"
#include "adsann/vecio.hpp"

using namespace adsann;

int main(int argc, char** argv) {
    try {
        const std::string cmd = argc > 1 ? argv[1] : "";
        if (cmd == "build" && argc == 8) {
            const Dataset raw = read_fvecs(argv[2]), t = read_fvecs(argv[3]);
            const HnswGraph g = build_hnsw(raw, t, std::atoi(argv[4]), std::atoi(argv[5]),
                                           std::strtoull(argv[6], nullptr, 10));
            save_hnsw(g, argv[7]);
            return 0;
        }
        if (cmd == "query" && argc == 13) {
            const Dataset raw = read_fvecs(argv[3]), t = read_fvecs(argv[4]);
            const Dataset qr = read_fvecs(argv[5]), qt = read_fvecs(argv[6]);
            const HnswGraph g = load_hnsw(argv[2], raw, t);
            const int K = std::atoi(argv[7]), nef = std::atoi(argv[8]), mode = std::atoi(argv[9]);
            const DcoConfig cfg{std::atof(argv[10]), std::atoi(argv[11])};
            std::ofstream out(argv[12], std::ios::binary);
            for (int q = 0; q < qr.n; ++q) {
                const KnnResult r = hnsw_query(g, qt.row(q), qr.row(q), K, nef, static_cast<HnswMode>(mode), cfg);
                const int cnt = static_cast<int>(r.ids.size());
                out.write(reinterpret_cast<const char*>(&cnt), 4);
                for (int j = 0; j < K; ++j) {
                    const int id = j < cnt ? r.ids[j] : -1;
                    out.write(reinterpret_cast<const char*>(&id), 4);
                }
                for (int j = 0; j < K; ++j) {
                    const double dv = j < cnt ? r.dists[j] : -1.0;
                    out.write(reinterpret_cast<const char*>(&dv), 8);
                }
                const unsigned long long st[4] = {r.stats.dims_evaluated, r.stats.dco_count, r.stats.hops,
                                                  r.stats.candidates};
                out.write(reinterpret_cast<const char*>(st), 32);
            }
            return 0;
        }
        std::fprintf(stderr, "usage: see the file header\n");
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}

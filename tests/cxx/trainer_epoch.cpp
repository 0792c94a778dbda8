// A C++ host running the benchmarked training epoch through the C ABI alone
// (include/gdx.h): no Python, no torch.  Generates the graph with the reference's
// generator (bit-identical host port), creates a gdx_trainer, runs epochs and prints
// one JSON line with the per-epoch losses (tests/test_native_trainer.py compares them
// with the Python trainers and the fp64 oracle).
//
//   trainer_epoch <n> <avg_degree> <graph_seed> <kind: sum|gcn|sage> <lr> <epochs> <d0,d1,...>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gdx.h"

static int die(const char* what) {
    std::fprintf(stderr, "%s: %s\n", what, gdx_last_error());
    return 1;
}

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s n degree seed kind lr epochs dims\n", argv[0]);
        return 2;
    }
    const uint32_t n = static_cast<uint32_t>(std::atoi(argv[1]));
    const double deg = std::atof(argv[2]);
    const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
    const std::string kind = argv[4];
    const float lr = static_cast<float>(std::atof(argv[5]));
    const int epochs = std::atoi(argv[6]);
    std::vector<uint32_t> dims;
    for (char* p = std::strtok(argv[7], ","); p; p = std::strtok(nullptr, ",")) dims.push_back(std::atoi(p));

    std::vector<uint64_t> ro(n + 1);
    const uint64_t nnz = gdx_host_gen_random_graph_count(n, deg, seed, ro.data());
    std::vector<uint32_t> cols(nnz ? nnz : 1);
    if (gdx_host_gen_random_graph_fill(n, deg, seed, ro.data(), cols.data())) return die("generate");

    gdx_trainer_config cfg{};
    cfg.kind = kind == "sage" ? GDX_MODEL_SAGE : kind == "gcn" ? GDX_MODEL_GCN : GDX_MODEL_SUM;
    cfg.layers = static_cast<uint32_t>(dims.size() - 1);
    cfg.dims = dims.data();
    cfg.lr = lr;
    cfg.world = 1;
    cfg.feature_seed = 1;
    cfg.label_seed = 2;
    cfg.use_graph = 1;
    gdx_trainer_graph g{};
    g.num_vertices = n;
    g.nnz = nnz;
    g.row_offsets = ro.data();
    g.cols = cols.data();
    gdx_trainer* t = nullptr;
    if (gdx_trainer_create(&cfg, &g, &t)) return die("gdx_trainer_create");
    if (gdx_trainer_init_weights(t, 3, 0)) return die("gdx_trainer_init_weights");
    std::printf("{\"n\": %u, \"nnz\": %llu, \"losses\": [", n, static_cast<unsigned long long>(nnz));
    for (int e = 0; e < epochs; ++e) {
        double loss = 0;
        if (gdx_trainer_epoch(t, &loss)) return die("gdx_trainer_epoch");
        std::printf("%s%.12g", e ? ", " : "", loss);
    }
    std::printf("]}\n");
    gdx_trainer_destroy(t);
    return 0;
}

// Drop-in check: the reference's own types and test generators with the
// GPU adapter.  Built by tests/test_cpp_adapter.py against the reference
// headers (oracle side) and libbsp.so; run on a GPU box it compares
// bsp_gpu::spgemm_rowwise / spgemm_clusterwise with cspgemm::spgemm_rowwise.
#include "cspgemm/cspgemm.hpp"
#include "bsp/cspgemm_gpu.hpp"

#include <cstdio>
#include <cstring>
#include <random>

int main(int argc, char** argv) {
    using namespace cspgemm;
    const bool run = argc > 1 && std::strcmp(argv[1], "run") == 0;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(0.1, 4.0), coin(0.0, 1.0);
    CooMatrix m;
    m.nrows = m.ncols = 300;
    for (index_t i = 0; i < 300; ++i)
        for (index_t j = 0; j < 300; ++j)
            if (coin(rng) < 0.03) m.entries.push_back({i, j, u(rng)});
    const CsrMatrix a = coo_to_csr(m);
    if (!run) {
        std::printf("adapter compiled\n");
        return 0;
    }
    const CsrMatrix ref = spgemm_rowwise(a, a);
    const CsrMatrix gpu = bsp_gpu::spgemm_rowwise(a, a);
    const bool row_ok = ref.row_ptr == gpu.row_ptr && ref.col_idx == gpu.col_idx &&
                        std::memcmp(ref.values.data(), gpu.values.data(),
                                    ref.values.size() * sizeof(double)) == 0;
    const ClusterAssignment asg = hierarchical_clusters(a);
    const CsrMatrix cw = bsp_gpu::spgemm_clusterwise(a, asg, a);
    const bool cw_ok = ref.row_ptr == cw.row_ptr && ref.col_idx == cw.col_idx &&
                       std::memcmp(ref.values.data(), cw.values.data(),
                                   ref.values.size() * sizeof(double)) == 0;
    bool threw = false;
    try {
        CsrMatrix bad = a;
        bad.nrows = 299;
        bad.row_ptr.pop_back();
        (void)bsp_gpu::spgemm_rowwise(a, bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    std::printf("rowwise %s clusterwise %s contract %s\n", row_ok ? "PASS" : "FAIL",
                cw_ok ? "PASS" : "FAIL", threw ? "PASS" : "FAIL");
    return (row_ok && cw_ok && threw) ? 0 : 1;
}

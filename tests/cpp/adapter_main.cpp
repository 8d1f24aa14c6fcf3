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
    // the rest of the mirror: symbolic in the reference's index type, top-k
    // element for element, clustering / reorder identical
    const std::vector<index_t> sym = bsp_gpu::spgemm_symbolic(a, a);
    const bool sym_ok = sym == spgemm_symbolic(a, a);
    const CsrMatrix at = transpose(binarize(a));
    const auto tk_ref = spgemm_topk(binarize(a), at, 7, 0.3);
    const auto tk_gpu = bsp_gpu::spgemm_topk<CandidatePair>(binarize(a), at, 7, 0.3);
    bool tk_ok = tk_ref.size() == tk_gpu.size();
    for (size_t k = 0; tk_ok && k < tk_ref.size(); ++k)
        tk_ok = tk_ref[k].i == tk_gpu[k].i && tk_ref[k].j == tk_gpu[k].j &&
                std::memcmp(&tk_ref[k].score, &tk_gpu[k].score, sizeof(double)) == 0;
    const ClusterParams prm{};
    const bool hier_ok =
        bsp_gpu::hierarchical_clusters<ClusterAssignment>(a, prm).clusters == asg.clusters;
    const bool var_ok = bsp_gpu::variable_length_clusters<ClusterAssignment>(a, prm).clusters ==
                        variable_length_clusters(a, prm).clusters;
    const bool fix_ok =
        bsp_gpu::fixed_length_clusters<ClusterAssignment>(a.nrows, 4).clusters ==
        fixed_length_clusters(a.nrows, 4).clusters;
    const bool ord_ok = bsp_gpu::reorder_rcm<Permutation>(a).perm == reorder_rcm(a).perm &&
                        bsp_gpu::reorder_degree<Permutation>(a).perm == reorder_degree(a).perm &&
                        bsp_gpu::reorder_random<Permutation>(a.nrows, 11).perm ==
                            reorder_random(a.nrows, 11).perm;
    const bool rest_ok = sym_ok && tk_ok && hier_ok && var_ok && fix_ok && ord_ok;
    std::printf("rowwise %s clusterwise %s contract %s mirror %s (sym %d topk %d hier %d var %d "
                "fixed %d reorder %d)\n",
                row_ok ? "PASS" : "FAIL", cw_ok ? "PASS" : "FAIL", threw ? "PASS" : "FAIL",
                rest_ok ? "PASS" : "FAIL", sym_ok, tk_ok, hier_ok, var_ok, fix_ok, ord_ok);
    return (row_ok && cw_ok && threw && rest_ok) ? 0 : 1;
}

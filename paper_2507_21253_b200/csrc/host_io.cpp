// Host-side file IO of the SpGEMM path: Matrix Market
// coordinate files and permutation files, so externally computed orderings
// (graph / hypergraph partitioning — the paper's best) and
// real SuiteSparse inputs can be fed to the engine.
//
// Replaces reference matrix_market.hpp: load_matrix_market (:42-119) +
// coo_to_csr (csr.hpp:92-113), write_matrix_market (:122-137),
// load_permutation (:141-166, used by ReorderSpec::file, reorder.hpp:185-192)
// and write_permutation (:168-173).  Same accepted formats, same 1-based ->
// 0-based conversion, symmetric expansion, pattern value 1.0, duplicates
// summed, and the same error conditions (io_error, with "path:line: message").
// Parsing reads the whole file once and converts with std::from_chars.
#include "common.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

namespace bsp {
namespace {

[[noreturn]] void parse_fail(const std::string& path, size_t line_no, const std::string& msg) {
    throw io_error(path + ":" + std::to_string(line_no) + ": " + msg);
}

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

bool blank(const char* b, const char* e) {
    for (; b < e; ++b)
        if (!std::isspace(static_cast<unsigned char>(*b))) return false;
    return true;
}

std::string read_all(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open '" + path + "'");
    std::string s((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return s;
}

// Line cursor over a file buffer ("\r\n" tolerated).
struct Lines {
    const char* p;
    const char* end;
    size_t no = 0;
    bool next(const char*& b, const char*& e) {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        if (e > b && e[-1] == '\r') --e;
        ++no;
        return true;
    }
};

const char* skip_ws(const char* b, const char* e) {
    while (b < e && std::isspace(static_cast<unsigned char>(*b))) ++b;
    return b;
}

template <typename T>
bool parse_num(const char*& b, const char* e, T& v) {
    b = skip_ws(b, e);
    if (b < e && *b == '+') ++b;
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc()) return false;
    b = r.ptr;
    return true;
}

struct Entry {
    int64_t row, col;
    double v;
};

}  // namespace

HostCsr load_matrix_market(const std::string& path) {
    std::string buf = read_all(path);
    Lines ln{buf.data(), buf.data() + buf.size()};
    const char *b, *e;
    if (!ln.next(b, e)) parse_fail(path, 1, "empty file");
    if (e - b >= 3 && std::memcmp(b, "\xEF\xBB\xBF", 3) == 0) b += 3;  // UTF-8 BOM
    std::istringstream header(std::string(b, e));
    std::string banner, object, format, field, symmetry;
    header >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket") parse_fail(path, ln.no, "missing %%MatrixMarket banner");
    object = lower(object);
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (object != "matrix") parse_fail(path, ln.no, "unsupported object '" + object + "'");
    if (format != "coordinate")
        parse_fail(path, ln.no, "unsupported format '" + format + "' (coordinate only)");
    const bool pattern = field == "pattern";
    if (field != "real" && field != "integer" && !pattern)
        parse_fail(path, ln.no, "unsupported field '" + field + "'");
    const bool symmetric = symmetry == "symmetric";
    if (symmetry != "general" && !symmetric)
        parse_fail(path, ln.no, "unsupported symmetry '" + symmetry + "'");
    long long nrows = -1, ncols = -1, nnz = -1;
    while (ln.next(b, e)) {
        if (b < e && *b == '%') continue;
        if (blank(b, e)) continue;
        const char* q = b;
        if (!parse_num(q, e, nrows) || !parse_num(q, e, ncols) || !parse_num(q, e, nnz) ||
            nrows < 0 || ncols < 0 || nnz < 0)
            parse_fail(path, ln.no, "malformed size line '" + std::string(b, e) + "'");
        break;
    }
    if (nrows < 0) parse_fail(path, ln.no, "missing size line");
    std::vector<Entry> ent;
    ent.reserve(static_cast<size_t>(symmetric ? 2 * nnz : nnz));
    long long seen = 0;
    while (seen < nnz) {
        if (!ln.next(b, e))
            parse_fail(path, ln.no + 1,
                       "unexpected end of file: expected " + std::to_string(nnz) +
                           " entries, got " + std::to_string(seen));
        if (blank(b, e) || *b == '%') continue;
        const char* q = b;
        long long r = 0, c = 0;
        double v = 1.0;
        if (!parse_num(q, e, r) || !parse_num(q, e, c))
            parse_fail(path, ln.no, "malformed entry '" + std::string(b, e) + "'");
        if (!pattern && !parse_num(q, e, v))
            parse_fail(path, ln.no, "missing value in entry '" + std::string(b, e) + "'");
        if (r < 1 || r > nrows)
            parse_fail(path, ln.no, "row index " + std::to_string(r) + " out of bounds [1, " +
                                        std::to_string(nrows) + "]");
        if (c < 1 || c > ncols)
            parse_fail(path, ln.no, "col index " + std::to_string(c) + " out of bounds [1, " +
                                        std::to_string(ncols) + "]");
        ent.push_back({r - 1, c - 1, v});
        if (symmetric && r != c) ent.push_back({c - 1, r - 1, v});
        ++seen;
    }
    require(nrows < (int64_t{1} << 31) && ncols < (int64_t{1} << 31),
            "load_matrix_market: dimensions must fit int32 indices");
    // coo_to_csr (csr.hpp:92-113): sort by (row, col), sum duplicates in order
    std::stable_sort(ent.begin(), ent.end(), [](const Entry& x, const Entry& y) {
        return x.row != y.row ? x.row < y.row : x.col < y.col;
    });
    HostCsr m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.row_ptr.assign(static_cast<size_t>(nrows) + 1, 0);
    for (size_t i = 0; i < ent.size();) {
        Entry x = ent[i];
        size_t j = i + 1;
        while (j < ent.size() && ent[j].row == x.row && ent[j].col == x.col) x.v += ent[j++].v;
        ++m.row_ptr[x.row + 1];
        m.col_idx.push_back(static_cast<int32_t>(x.col));
        m.values.push_back(x.v);
        i = j;
    }
    std::partial_sum(m.row_ptr.begin(), m.row_ptr.end(), m.row_ptr.begin());
    return m;
}

void write_matrix_market(const int64_t* rp, const int32_t* ci, const double* v, int64_t nrows,
                         int64_t ncols, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw io_error("cannot open '" + path + "' for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(nrows),
                 static_cast<long long>(ncols), static_cast<long long>(rp[nrows]));
    bool ok = true;
    for (int64_t i = 0; i < nrows && ok; ++i)
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
            if (std::fprintf(f, "%lld %d %.17g\n", static_cast<long long>(i + 1), ci[p] + 1,
                             v ? v[p] : 1.0) < 0) {
                ok = false;
                break;
            }
    if (std::fclose(f) != 0 || !ok) throw io_error("write failed for '" + path + "'");
}

std::vector<int32_t> load_permutation(const std::string& path, int64_t nrows) {
    std::string buf = read_all(path);
    Lines ln{buf.data(), buf.data() + buf.size()};
    std::vector<int32_t> perm;
    perm.reserve(static_cast<size_t>(std::max<int64_t>(nrows, 0)));
    const char *b, *e;
    while (ln.next(b, e)) {
        if (blank(b, e)) continue;
        const char* q = b;
        long long v = 0;
        if (!parse_num(q, e, v)) parse_fail(path, ln.no, "not an integer: '" + std::string(b, e) + "'");
        perm.push_back(static_cast<int32_t>(v));
    }
    if (static_cast<int64_t>(perm.size()) != nrows)
        throw io_error(path + ": permutation length " + std::to_string(perm.size()) +
                       " does not match matrix rows " + std::to_string(nrows));
    // Permutation::from_perm (permutation.hpp): a bijection of [0, n)
    std::vector<char> seen(perm.size(), 0);
    for (int32_t x : perm) {
        if (x < 0 || x >= nrows)
            throw io_error(path + ": permutation: entry " + std::to_string(x) + " out of range");
        if (seen[x]) throw io_error(path + ": permutation: duplicate entry " + std::to_string(x));
        seen[x] = 1;
    }
    return perm;
}

}  // namespace bsp

extern "C" {

int bsp_load_matrix_market(const char* path, bsp_host_csr* out) {
    return bsp::guarded([&] {
        bsp::require(path != nullptr && out != nullptr, "load_matrix_market: null argument");
        bsp::export_csr(bsp::load_matrix_market(path), out);
    });
}

int bsp_write_matrix_market(const bsp_host_csr* A, const char* path) {
    return bsp::guarded([&] {
        bsp::require(A != nullptr && path != nullptr, "write_matrix_market: null argument");
        bsp::write_matrix_market(A->row_ptr, A->col_idx, A->values, A->nrows, A->ncols, path);
    });
}

int bsp_load_permutation(const char* path, int64_t nrows, int32_t* perm_out) {
    return bsp::guarded([&] {
        bsp::require(path != nullptr && (perm_out != nullptr || nrows == 0),
                     "load_permutation: null argument");
        const auto p = bsp::load_permutation(path, nrows);
        std::copy(p.begin(), p.end(), perm_out);
    });
}

int bsp_write_permutation(const int32_t* perm, int64_t n, const char* path) {
    return bsp::guarded([&] {
        bsp::require(path != nullptr && (perm != nullptr || n == 0), "write_permutation: null argument");
        std::FILE* f = std::fopen(path, "w");
        if (!f) throw bsp::io_error(std::string("cannot open '") + path + "' for writing");
        bool ok = true;
        for (int64_t k = 0; k < n && ok; ++k) ok = std::fprintf(f, "%d\n", perm[k]) >= 0;
        if (std::fclose(f) != 0 || !ok) throw bsp::io_error(std::string("write failed for '") + path + "'");
    });
}

}  // extern "C"

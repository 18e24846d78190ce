// Bundle ingestion and the Matrix Market reader: the reference's on-disk
// interchange format (src/bundle.cpp:113-290, src/matrix_market.cpp:23-71) read into this
// library's Decomposition / CsrMatrix types, so externally decomposed problems (e.g. bidomain
// stiffness matrices) reach the GPU path.
//
// Semantics follow the reference exactly (the tests pin the ingested maps, matrices and the
// diagnostic messages bit for bit against the reference's own ingest of the same bundles):
//   * manifest: first line starts with "bddc-bundle"; keys subdomains / global_dofs / rhs /
//     classes / "matrix i file" / "map i file"; '#' lines and blank lines ignored;
//   * classes: one token per global dof ("interior", or "edge"/"corner" followed by an
//     entity id >= 0); multiplicities validated against the classes;
//   * every subdomain map is reordered interior-first (stable), its matrix permuted alike;
//   * Matrix Market "coordinate real general|symmetric": 1-based entries, symmetric files
//     mirrored, duplicates summed in file order (CsrMatrix::from_triplets).
// The implementation is this library's own: whole files are tokenised by a small cursor,
// manifest keys dispatch through a handler table, the reorder is a stable partition.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>

#include "problem.hpp"

namespace bddc_b200 {
namespace {

namespace fs = std::filesystem;

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("missing file: " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// Whitespace tokeniser over a file's contents.
class Cursor {
public:
    explicit Cursor(std::string text) : text_(std::move(text)) {}
    bool token(std::string_view& out) {
        while (pos_ < text_.size() && std::isspace(static_cast<unsigned char>(text_[pos_]))) ++pos_;
        if (pos_ >= text_.size()) return false;
        const std::size_t b = pos_;
        while (pos_ < text_.size() && !std::isspace(static_cast<unsigned char>(text_[pos_]))) ++pos_;
        out = std::string_view(text_).substr(b, pos_ - b);
        return true;
    }
    bool integer(long& v) {
        std::string_view t;
        if (!token(t)) return false;
        const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
        return r.ec == std::errc() && r.ptr == t.data() + t.size();
    }
    bool real(double& v) {
        std::string_view t;
        if (!token(t)) return false;
        const std::string s(t);
        char* end = nullptr;
        v = std::strtod(s.c_str(), &end);
        return end == s.c_str() + s.size();
    }
    // next line (without the newline); false at the end
    bool line(std::string_view& out) {
        if (pos_ >= text_.size()) return false;
        const std::size_t e = text_.find('\n', pos_);
        const std::size_t stop = e == std::string::npos ? text_.size() : e;
        out = std::string_view(text_).substr(pos_, stop - pos_);
        if (!out.empty() && out.back() == '\r') out.remove_suffix(1);
        pos_ = stop + (e == std::string::npos ? 0 : 1);
        return true;
    }

private:
    std::string text_;
    std::size_t pos_ = 0;
};

std::vector<double> read_reals(const std::string& path) {
    Cursor c(slurp(path));
    std::vector<double> v;
    for (double x; c.real(x);) v.push_back(x);
    return v;
}

std::vector<index_t> read_indices(const std::string& path) {
    Cursor c(slurp(path));
    std::vector<index_t> v;
    for (long x; c.integer(x);) v.push_back(static_cast<index_t>(x));
    return v;
}

void check_finite(const std::vector<double>& v, const char* what) {
    const auto bad = std::find_if(v.begin(), v.end(), [](double x) { return !std::isfinite(x); });
    if (bad != v.end())
        throw std::invalid_argument(std::string(what) + ": non-finite entry at index " +
                                    std::to_string(bad - v.begin()));
}

bool iequals(std::string_view a, std::string_view b) {
    return a.size() == b.size() && std::equal(a.begin(), a.end(), b.begin(), [](char x, char y) {
               return std::tolower(static_cast<unsigned char>(x)) == std::tolower(static_cast<unsigned char>(y));
           });
}

struct Manifest {
    index_t subdomains = -1, global_dofs = -1;
    std::string rhs, classes;
    std::vector<std::string> matrix, map;
};

Manifest parse_manifest(const std::string& path) {
    Cursor lines(slurp(path));
    std::string_view ln;
    if (!lines.line(ln) || ln.rfind("bddc-bundle", 0) != 0) throw std::runtime_error(path + ": not a bundle manifest");
    Manifest M;
    auto per_subdomain = [&](std::vector<std::string> Manifest::*files) {
        return [&, files](std::istringstream& f) {
            index_t i = -1;
            std::string name;
            f >> i >> name;
            if (i < 0 || i >= M.subdomains)
                throw std::runtime_error(path + ": subdomain index " + std::to_string(i) + " out of range");
            (M.*files)[i] = name;
        };
    };
    const std::unordered_map<std::string, std::function<void(std::istringstream&)>> handlers = {
        {"subdomains",
         [&](std::istringstream& f) {
             f >> M.subdomains;
             M.matrix.assign(std::max<index_t>(M.subdomains, 0), {});
             M.map.assign(std::max<index_t>(M.subdomains, 0), {});
         }},
        {"global_dofs", [&](std::istringstream& f) { f >> M.global_dofs; }},
        {"rhs", [&](std::istringstream& f) { f >> M.rhs; }},
        {"classes", [&](std::istringstream& f) { f >> M.classes; }},
        {"matrix", per_subdomain(&Manifest::matrix)},
        {"map", per_subdomain(&Manifest::map)},
    };
    while (lines.line(ln)) {
        if (ln.empty() || ln.front() == '#') continue;
        std::istringstream f{std::string(ln)};
        std::string key;
        f >> key;
        const auto h = handlers.find(key);
        if (h == handlers.end()) throw std::runtime_error(path + ": unknown manifest key '" + key + "'");
        h->second(f);
    }
    if (M.subdomains <= 0 || M.global_dofs <= 0 || M.rhs.empty() || M.classes.empty())
        throw std::runtime_error(path + ": incomplete manifest");
    for (index_t i = 0; i < M.subdomains; ++i)
        if (M.matrix[i].empty() || M.map[i].empty())
            throw std::runtime_error(path + ": subdomain " + std::to_string(i) + " lacks a matrix or map entry");
    return M;
}

std::vector<DofClass> read_classes(const std::string& path, const std::string& name, index_t n) {
    Cursor c(slurp(path));
    std::vector<DofClass> cls(n);
    for (index_t g = 0; g < n; ++g) {
        std::string_view kind;
        if (!c.token(kind)) throw std::runtime_error(name + ": truncated at dof " + std::to_string(g));
        if (kind == "interior") {
            cls[g] = {DofKind::interior, -1};
            continue;
        }
        const bool edge = kind == "edge";
        if (!edge && kind != "corner")
            throw std::runtime_error(name + ": unknown class '" + std::string(kind) + "' at dof " + std::to_string(g));
        long entity = -1;
        if (!c.integer(entity) || entity < 0)
            throw std::runtime_error(name + ": missing entity id at dof " + std::to_string(g));
        cls[g] = {edge ? DofKind::edge : DofKind::corner, static_cast<index_t>(entity)};
    }
    return cls;
}

// The first dof (ascending) whose multiplicity contradicts its class, with the reference's text.
void validate_multiplicity(const Decomposition& d) {
    for (index_t g = 0; g < d.global_dofs; ++g) {
        const index_t m = d.multiplicity[g];
        if (m == 0)
            throw std::runtime_error("bundle validation: global dof " + std::to_string(g) + " is covered by no subdomain");
        const char* expect = nullptr;
        switch (d.classes[g].kind) {
            case DofKind::interior: expect = m == 1 ? nullptr : "interior"; break;
            case DofKind::edge: expect = m == 2 ? nullptr : "as an interface edge"; break;
            case DofKind::corner: expect = m >= 2 ? nullptr : "as a corner"; break;
        }
        if (expect)
            throw std::runtime_error("bundle validation: dof " + std::to_string(g) + " has multiplicity " +
                                     std::to_string(m) + " but is classified " + expect);
    }
}

// A with rows and columns renamed old -> pos[old]; entries keep their row-major input order
// (from_triplets then sorts each row and sums duplicates in that order).
CsrMatrix renumbered(const CsrMatrix& A, const std::vector<index_t>& pos) {
    std::vector<Triplet> t;
    t.reserve(A.values.size());
    for (index_t r = 0; r < A.nrows; ++r)
        for (index_t q = A.row_offsets[r]; q < A.row_offsets[r + 1]; ++q)
            t.push_back({pos[r], pos[A.col_indices[q]], A.values[q]});
    return CsrMatrix::from_triplets(A.nrows, A.ncols, std::move(t));
}

}  // namespace

CsrMatrix read_matrix_market_file(const std::string& path) {
    std::ifstream probe(path);
    if (!probe) throw std::runtime_error("cannot open matrix file: " + path);
    probe.close();
    Cursor c(slurp(path));
    std::string_view ln;
    if (!c.line(ln)) throw std::runtime_error(path + ": empty matrix market stream");
    const std::string header(ln);
    std::istringstream hs(header);
    std::string word[5];
    for (auto& w : word) hs >> w;
    if (word[0] != "%%MatrixMarket" || !iequals(word[1], "matrix") || !iequals(word[2], "coordinate") ||
        !iequals(word[3], "real"))
        throw std::runtime_error(path + ": unsupported matrix market header: " + header);
    std::string symmetry = word[4];
    std::transform(symmetry.begin(), symmetry.end(), symmetry.begin(),
                   [](char ch) { return static_cast<char>(std::tolower(static_cast<unsigned char>(ch))); });
    const bool mirror = symmetry == "symmetric";
    if (!mirror && symmetry != "general") throw std::runtime_error(path + ": unsupported symmetry kind: " + symmetry);
    // size line: the first line that is neither empty nor a comment
    bool sized = false;
    while (c.line(ln))
        if (!ln.empty() && ln.front() != '%') {
            sized = true;
            break;
        }
    const std::string size_line = sized ? std::string(ln) : std::string();
    long dims[3] = {-1, -1, -1};
    {
        std::istringstream ss(size_line);
        ss >> dims[0] >> dims[1] >> dims[2];
    }
    const long nr = dims[0], nc = dims[1], ne = dims[2];
    if (nr < 0 || nc < 0 || ne < 0) throw std::runtime_error(path + ": malformed size line: " + size_line);
    std::vector<Triplet> t;
    t.reserve(static_cast<std::size_t>(mirror ? 2 * ne : ne));
    for (long e = 1; e <= ne; ++e) {
        long i = 0, j = 0;
        double v = 0.0;
        if (!(c.integer(i) && c.integer(j) && c.real(v)))
            throw std::runtime_error(path + ": truncated entry list at entry " + std::to_string(e));
        if (i < 1 || i > nr || j < 1 || j > nc)
            throw std::runtime_error(path + ": entry index out of range at entry " + std::to_string(e));
        t.push_back({static_cast<index_t>(i - 1), static_cast<index_t>(j - 1), v});
        if (mirror && i != j) t.push_back({static_cast<index_t>(j - 1), static_cast<index_t>(i - 1), v});
    }
    return CsrMatrix::from_triplets(static_cast<index_t>(nr), static_cast<index_t>(nc), std::move(t));
}

IngestedProblem ingest_bundle(const std::string& manifest_path) {
    const Manifest M = parse_manifest(manifest_path);
    const fs::path dir = fs::path(manifest_path).parent_path();
    auto at = [&](const std::string& name) { return (dir / name).string(); };
    const index_t ns = M.subdomains, n = M.global_dofs;

    IngestedProblem P;
    P.rhs = read_reals(at(M.rhs));
    if (static_cast<index_t>(P.rhs.size()) != n)
        throw std::runtime_error(M.rhs + ": expected " + std::to_string(n) + " values, found " +
                                 std::to_string(P.rhs.size()));
    check_finite(P.rhs, "bundle rhs");

    Decomposition& d = P.decomposition;
    d.n_subdomains = ns;
    const index_t side = static_cast<index_t>(std::lround(std::sqrt(static_cast<double>(ns))));
    d.k = side * side == ns ? side : 0;  // informational: square layouts only
    d.global_dofs = n;
    d.classes = read_classes(at(M.classes), M.classes, n);

    std::vector<std::vector<index_t>> maps(ns);
    d.multiplicity.assign(n, 0);
    for (index_t i = 0; i < ns; ++i) {
        maps[i] = read_indices(at(M.map[i]));
        for (index_t g : maps[i]) {
            if (g < 0 || g >= n) throw std::runtime_error(M.map[i] + ": dof " + std::to_string(g) + " out of range");
            ++d.multiplicity[g];
        }
    }
    validate_multiplicity(d);

    d.subdomain_dofs.resize(ns);
    d.interior_counts.resize(ns);
    P.local_matrices.resize(ns);
    for (index_t i = 0; i < ns; ++i) {
        const std::vector<index_t>& map = maps[i];
        const index_t nl = static_cast<index_t>(map.size());
        const CsrMatrix A = read_matrix_market_file(at(M.matrix[i]));
        if (A.nrows != nl || A.ncols != nl)
            throw std::runtime_error(M.matrix[i] + ": size " + std::to_string(A.nrows) + "x" +
                                     std::to_string(A.ncols) + " does not match map length " + std::to_string(nl));
        check_finite(A.values, "bundle matrix");
        // interior-first, stable: order[new] = old local index; pos = its inverse
        std::vector<index_t> order(nl);
        std::iota(order.begin(), order.end(), 0);
        const auto split = std::stable_partition(order.begin(), order.end(), [&](index_t l) {
            return d.classes[map[l]].kind == DofKind::interior;
        });
        d.interior_counts[i] = static_cast<index_t>(split - order.begin());
        std::vector<index_t> pos(nl);
        d.subdomain_dofs[i].resize(nl);
        for (index_t k = 0; k < nl; ++k) {
            pos[order[k]] = k;
            d.subdomain_dofs[i][k] = map[order[k]];
        }
        P.local_matrices[i] = renumbered(A, pos);
    }
    d.weights = build_weights(d);
    P.constraints = build_constraints(d);
    P.global_matrix = global_from_locals(d, P.local_matrices);
    return P;
}

}  // namespace bddc_b200

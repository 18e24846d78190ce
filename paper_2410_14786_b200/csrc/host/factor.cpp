#include "factor.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <queue>
#include <stdexcept>
#include <string>

namespace bddc_b200 {
namespace {

struct Graph {
    index_t n = 0;
    std::vector<index_t> ptr, adj;
};

// Interior adjacency of A_II (diagonal dropped).
Graph interior_graph(const CsrMatrix& A, index_t nI) {
    Graph g;
    g.n = nI;
    g.ptr.assign(nI + 1, 0);
    for (index_t i = 0; i < nI; ++i) {
        for (index_t p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
            const index_t j = A.col_indices[p];
            if (j < nI && j != i) g.adj.push_back(j);
        }
        g.ptr[i + 1] = static_cast<index_t>(g.adj.size());
    }
    return g;
}

class NestedDissection {
public:
    NestedDissection(const Graph& g, const index_t* coords, const FactorOptions& opt)
        : g_(g), coords_(coords), opt_(opt), mark_(g.n, 0), side_(g.n, 0) {}

    void run(std::vector<Supernode>& snodes, std::vector<index_t>& perm) {
        std::vector<index_t> all(g_.n);
        for (index_t i = 0; i < g_.n; ++i) all[i] = i;
        snodes_ = &snodes;
        perm_ = &perm;
        perm.clear();
        if (g_.n > 0) build(all);
    }

private:
    const Graph& g_;
    const index_t* coords_;
    FactorOptions opt_;
    std::vector<int> mark_;
    std::vector<int> side_;
    std::vector<Supernode>* snodes_ = nullptr;
    std::vector<index_t>* perm_ = nullptr;
    int stamp_ = 0;

    // Append nodes as one supernode (split into a chain above max_supernode);
    // returns the id of the topmost piece.
    index_t emit(const std::vector<index_t>& nodes, const std::vector<index_t>& children) {
        index_t prev = -1;
        std::size_t pos = 0;
        const std::size_t w = static_cast<std::size_t>(std::max<index_t>(1, opt_.max_supernode));
        while (pos < nodes.size()) {
            const std::size_t take = std::min(w, nodes.size() - pos);
            Supernode s;
            s.col_begin = static_cast<index_t>(perm_->size());
            for (std::size_t i = 0; i < take; ++i) perm_->push_back(nodes[pos + i]);
            s.col_end = static_cast<index_t>(perm_->size());
            const index_t id = static_cast<index_t>(snodes_->size());
            snodes_->push_back(std::move(s));
            if (prev >= 0) {
                (*snodes_)[prev].parent = id;
            } else {
                for (index_t c : children) (*snodes_)[c].parent = id;
            }
            prev = id;
            pos += take;
        }
        return prev;
    }

    bool geometric_split(const std::vector<index_t>& nodes, std::vector<index_t>& left,
                         std::vector<index_t>& right, std::vector<index_t>& sep) {
        if (!coords_) return false;
        index_t lo[2] = {coords_[2 * nodes[0]], coords_[2 * nodes[0] + 1]};
        index_t hi[2] = {lo[0], lo[1]};
        for (index_t v : nodes)
            for (int a = 0; a < 2; ++a) {
                lo[a] = std::min(lo[a], coords_[2 * v + a]);
                hi[a] = std::max(hi[a], coords_[2 * v + a]);
            }
        const int axis = (hi[0] - lo[0]) >= (hi[1] - lo[1]) ? 0 : 1;
        if (hi[axis] - lo[axis] < 2) return false;
        const index_t mid = lo[axis] + (hi[axis] - lo[axis]) / 2;
        ++stamp_;
        for (index_t v : nodes) {
            const index_t c = coords_[2 * v + axis];
            if (c < mid) { left.push_back(v); side_[v] = 1; }
            else if (c > mid) { right.push_back(v); side_[v] = 2; }
            else { sep.push_back(v); side_[v] = 3; }
            mark_[v] = stamp_;
        }
        // Validate: no edge between the two sides.
        for (index_t v : left)
            for (index_t p = g_.ptr[v]; p < g_.ptr[v + 1]; ++p) {
                const index_t u = g_.adj[p];
                if (mark_[u] == stamp_ && side_[u] == 2) {
                    left.clear(); right.clear(); sep.clear();
                    return false;
                }
            }
        return !left.empty() && !right.empty();
    }

    // BFS level structure from a pseudo-peripheral node; the middle level separates.
    bool graph_split(const std::vector<index_t>& nodes, std::vector<index_t>& left,
                     std::vector<index_t>& right, std::vector<index_t>& sep) {
        ++stamp_;
        const int in_set = stamp_;
        for (index_t v : nodes) mark_[v] = in_set;
        std::vector<index_t> level(g_.n, -1);
        auto bfs = [&](index_t root, std::vector<index_t>& order) {
            for (index_t v : order) level[v] = -1;
            order.clear();
            order.push_back(root);
            level[root] = 0;
            for (std::size_t h = 0; h < order.size(); ++h) {
                const index_t v = order[h];
                for (index_t p = g_.ptr[v]; p < g_.ptr[v + 1]; ++p) {
                    const index_t u = g_.adj[p];
                    if (mark_[u] == in_set && level[u] < 0) {
                        level[u] = level[v] + 1;
                        order.push_back(u);
                    }
                }
            }
        };
        std::vector<index_t> order;
        index_t root = nodes[0];
        bfs(root, order);
        for (int it = 0; it < 4; ++it) {  // pseudo-peripheral search
            const index_t far = order.back();
            const index_t depth = level[far];
            std::vector<index_t> o2;
            o2.reserve(order.size());
            for (index_t v : order) level[v] = -1;
            bfs(far, o2);
            if (level[o2.back()] <= depth) { order.swap(o2); break; }
            order.swap(o2);
        }
        const index_t depth = level[order.back()];
        if (depth < 2) {
            for (index_t v : order) level[v] = -1;
            return false;
        }
        // choose the level where the cumulative count crosses half
        std::vector<index_t> count(depth + 1, 0);
        for (index_t v : order) count[level[v]]++;
        index_t cum = 0, cut = 1;
        for (index_t l = 0; l <= depth; ++l) {
            cum += count[l];
            if (2 * cum >= static_cast<index_t>(order.size())) { cut = l; break; }
        }
        cut = std::clamp<index_t>(cut, 1, depth - 1);
        for (index_t v : order) {
            if (level[v] < cut) left.push_back(v);
            else if (level[v] == cut) sep.push_back(v);
            else right.push_back(v);
        }
        // nodes not reached (other components) join the right part
        for (index_t v : nodes)
            if (level[v] < 0) right.push_back(v);
        for (index_t v : order) level[v] = -1;
        std::sort(left.begin(), left.end());
        std::sort(right.begin(), right.end());
        std::sort(sep.begin(), sep.end());
        return !left.empty() && !right.empty();
    }

    index_t build(std::vector<index_t>& nodes) {
        if (static_cast<index_t>(nodes.size()) <= opt_.leaf_size) return emit(nodes, {});
        std::vector<index_t> left, right, sep;
        if (!geometric_split(nodes, left, right, sep)) {
            left.clear(); right.clear(); sep.clear();
            if (!graph_split(nodes, left, right, sep)) return emit(nodes, {});
        }
        std::vector<index_t> children;
        children.push_back(build(left));
        children.push_back(build(right));
        std::sort(sep.begin(), sep.end());
        return emit(sep, children);
    }
};

// Column-major lower-triangular dense helpers on an f x f front.
struct Front {
    index_t f = 0;
    std::vector<double> a;  // column-major, a[c*f + r], r >= c used
    double& operator()(index_t r, index_t c) { return a[static_cast<std::size_t>(c) * f + r]; }
};

}  // namespace

std::int64_t InteriorFactor::factor_values() const {
    std::int64_t v = 0;
    for (const auto& s : snodes) {
        const std::int64_t n = s.size();
        v += n * (n + 1) / 2 + static_cast<std::int64_t>(s.n_interior_rows) * n;
    }
    return v;
}

InteriorFactor symbolic_factor(const CsrMatrix& A, index_t nI, const index_t* coords, const FactorOptions& opt) {
    if (A.nrows != A.ncols) throw std::invalid_argument("factor: matrix not square");
    const index_t n = A.nrows;
    if (nI < 0 || nI > n) throw std::invalid_argument("factor: interior count out of range");
    InteriorFactor F;
    F.n_interior = nI;
    F.n_iface = n - nI;

    const Graph g = interior_graph(A, nI);
    NestedDissection nd(g, coords, opt);
    nd.run(F.snodes, F.perm);
    F.iperm.assign(nI, -1);
    for (index_t p = 0; p < nI; ++p) F.iperm[F.perm[p]] = p;
    auto position = [&](index_t local) { return local < nI ? F.iperm[local] : local; };

    const index_t ns = static_cast<index_t>(F.snodes.size());
    std::vector<std::vector<index_t>> children(ns);
    std::vector<index_t> roots;
    for (index_t s = 0; s < ns; ++s) {
        if (F.snodes[s].parent >= 0) children[F.snodes[s].parent].push_back(s);
        else roots.push_back(s);
    }

    // Symbolic: R_s = (adj(cols) U R_children) restricted to positions >= col_end.
    std::vector<index_t> marker(n, -1);
    for (index_t s = 0; s < ns; ++s) {
        Supernode& sn = F.snodes[s];
        std::vector<index_t> rows;
        for (index_t c = sn.col_begin; c < sn.col_end; ++c) {
            const index_t v = F.perm[c];
            for (index_t p = A.row_offsets[v]; p < A.row_offsets[v + 1]; ++p) {
                const index_t pos = position(A.col_indices[p]);
                if (pos >= sn.col_end && marker[pos] != s) { marker[pos] = s; rows.push_back(pos); }
            }
        }
        for (index_t ch : children[s])
            for (index_t pos : F.snodes[ch].rows)
                if (pos >= sn.col_end && marker[pos] != s) { marker[pos] = s; rows.push_back(pos); }
        std::sort(rows.begin(), rows.end());
        sn.rows = std::move(rows);
        sn.n_interior_rows = static_cast<index_t>(
            std::lower_bound(sn.rows.begin(), sn.rows.end(), nI) - sn.rows.begin());
        index_t h = 0;
        for (index_t ch : children[s]) h = std::max(h, F.snodes[ch].height + 1);
        sn.height = h;
    }

    return F;
}

InteriorFactor factor_subdomain(const CsrMatrix& A, index_t nI, const index_t* coords,
                                const FactorOptions& opt) {
    InteriorFactor F = symbolic_factor(A, nI, coords, opt);
    const index_t n = A.nrows;
    auto position = [&](index_t local) { return local < nI ? F.iperm[local] : local; };
    const index_t ns = static_cast<index_t>(F.snodes.size());
    std::vector<std::vector<index_t>> children(ns);
    std::vector<index_t> roots;
    for (index_t s = 0; s < ns; ++s) {
        if (F.snodes[s].parent >= 0) children[F.snodes[s].parent].push_back(s);
        else roots.push_back(s);
    }

    // Numeric multifrontal factorisation.
    std::vector<std::vector<double>> updates(ns);  // column-major m x m lower
    std::vector<index_t> fpos(n, -1);
    for (index_t s = 0; s < ns; ++s) {
        Supernode& sn = F.snodes[s];
        const index_t nc = sn.size(), m = static_cast<index_t>(sn.rows.size()), f = nc + m;
        Front fr;
        fr.f = f;
        fr.a.assign(static_cast<std::size_t>(f) * f, 0.0);
        for (index_t i = 0; i < nc; ++i) fpos[sn.col_begin + i] = i;
        for (index_t i = 0; i < m; ++i) fpos[sn.rows[i]] = nc + i;
        for (index_t c = sn.col_begin; c < sn.col_end; ++c) {
            const index_t v = F.perm[c];
            for (index_t p = A.row_offsets[v]; p < A.row_offsets[v + 1]; ++p) {
                const index_t pos = position(A.col_indices[p]);
                if (pos >= c) fr(fpos[pos], fpos[c]) += A.values[p];
            }
        }
        for (index_t ch : children[s]) {
            const auto& R = F.snodes[ch].rows;
            const index_t mc = static_cast<index_t>(R.size());
            const auto& U = updates[ch];
            for (index_t b = 0; b < mc; ++b) {
                const index_t cb = fpos[R[b]];
                for (index_t a = b; a < mc; ++a)
                    fr(fpos[R[a]], cb) += U[static_cast<std::size_t>(b) * mc + a];
            }
            std::vector<double>().swap(updates[ch]);
        }
        // partial Cholesky of the leading nc columns
        for (index_t j = 0; j < nc; ++j) {
            double d = fr(j, j);
            if (!(d > 0.0) || !std::isfinite(d))
                throw std::runtime_error("interior block not positive definite at pivot " +
                                         std::to_string(sn.col_begin + j));
            d = std::sqrt(d);
            fr(j, j) = d;
            double* colj = &fr.a[static_cast<std::size_t>(j) * f];
            for (index_t i = j + 1; i < f; ++i) colj[i] /= d;
            for (index_t k = j + 1; k < f; ++k) {
                const double lkj = colj[k];
                if (lkj == 0.0) continue;
                double* colk = &fr.a[static_cast<std::size_t>(k) * f];
                for (index_t i = k; i < f; ++i) colk[i] -= colj[i] * lkj;
            }
        }
        sn.L.assign(static_cast<std::size_t>(nc) * nc, 0.0);
        for (index_t r = 0; r < nc; ++r)
            for (index_t c = 0; c <= r; ++c) sn.L[static_cast<std::size_t>(r) * nc + c] = fr(r, c);
        sn.B.assign(static_cast<std::size_t>(m) * nc, 0.0);
        for (index_t r = 0; r < m; ++r)
            for (index_t c = 0; c < nc; ++c) sn.B[static_cast<std::size_t>(r) * nc + c] = fr(nc + r, c);
        std::vector<double>& U = updates[s];
        U.assign(static_cast<std::size_t>(m) * m, 0.0);
        for (index_t b = 0; b < m; ++b)
            for (index_t a = b; a < m; ++a) U[static_cast<std::size_t>(b) * m + a] = fr(nc + a, nc + b);
        // inverse of the diagonal block (lower triangular)
        sn.Linv.assign(static_cast<std::size_t>(nc) * nc, 0.0);
        for (index_t c = 0; c < nc; ++c) {
            // solve L x = e_c
            for (index_t r = c; r < nc; ++r) {
                double acc = r == c ? 1.0 : 0.0;
                for (index_t k = c; k < r; ++k)
                    acc -= sn.L[static_cast<std::size_t>(r) * nc + k] * sn.Linv[static_cast<std::size_t>(k) * nc + c];
                sn.Linv[static_cast<std::size_t>(r) * nc + c] = acc / sn.L[static_cast<std::size_t>(r) * nc + r];
            }
        }
        for (index_t i = 0; i < nc; ++i) fpos[sn.col_begin + i] = -1;
        for (index_t i = 0; i < m; ++i) fpos[sn.rows[i]] = -1;
    }

    // Interface Schur complement: A_GG + extend-add of the interior roots' updates.
    const index_t ng = F.n_iface;
    F.schur.assign(static_cast<std::size_t>(ng) * ng, 0.0);
    for (index_t l = nI; l < n; ++l)
        for (index_t p = A.row_offsets[l]; p < A.row_offsets[l + 1]; ++p) {
            const index_t c = A.col_indices[p];
            if (c >= nI) F.schur[static_cast<std::size_t>(l - nI) * ng + (c - nI)] += A.values[p];
        }
    for (index_t r : roots) {
        const auto& R = F.snodes[r].rows;
        const index_t m = static_cast<index_t>(R.size());
        const auto& U = updates[r];
        for (index_t b = 0; b < m; ++b)
            for (index_t a = b; a < m; ++a) {
                const double u = U[static_cast<std::size_t>(b) * m + a];
                const index_t ga = R[a] - nI, gb = R[b] - nI;
                if (ga < 0 || gb < 0)
                    throw std::logic_error("factor: interior root update has interior rows");
                F.schur[static_cast<std::size_t>(ga) * ng + gb] += u;
                if (ga != gb) F.schur[static_cast<std::size_t>(gb) * ng + ga] += u;
            }
    }
    return F;
}

void factor_solve(const InteriorFactor& F, double* X, index_t nrhs) {
    const index_t nI = F.n_interior;
    std::vector<double> y(static_cast<std::size_t>(nI) * nrhs);
    for (index_t p = 0; p < nI; ++p)
        for (index_t k = 0; k < nrhs; ++k)
            y[static_cast<std::size_t>(p) * nrhs + k] = X[static_cast<std::size_t>(F.perm[p]) * nrhs + k];
    auto Y = [&](index_t p, index_t k) -> double& { return y[static_cast<std::size_t>(p) * nrhs + k]; };
    // forward: L y = b
    for (const Supernode& s : F.snodes) {
        const index_t nc = s.size();
        for (index_t r = 0; r < nc; ++r)
            for (index_t k = 0; k < nrhs; ++k) {
                double acc = Y(s.col_begin + r, k);
                for (index_t c = 0; c < r; ++c)
                    acc -= s.L[static_cast<std::size_t>(r) * nc + c] * Y(s.col_begin + c, k);
                Y(s.col_begin + r, k) = acc / s.L[static_cast<std::size_t>(r) * nc + r];
            }
        for (index_t r = 0; r < s.n_interior_rows; ++r)
            for (index_t k = 0; k < nrhs; ++k) {
                double acc = 0.0;
                for (index_t c = 0; c < nc; ++c)
                    acc += s.B[static_cast<std::size_t>(r) * nc + c] * Y(s.col_begin + c, k);
                Y(s.rows[r], k) -= acc;
            }
    }
    // backward: L^T x = y
    for (auto it = F.snodes.rbegin(); it != F.snodes.rend(); ++it) {
        const Supernode& s = *it;
        const index_t nc = s.size();
        for (index_t c = 0; c < nc; ++c)
            for (index_t k = 0; k < nrhs; ++k) {
                double acc = 0.0;
                for (index_t r = 0; r < s.n_interior_rows; ++r)
                    acc += s.B[static_cast<std::size_t>(r) * nc + c] * Y(s.rows[r], k);
                Y(s.col_begin + c, k) -= acc;
            }
        for (index_t r = nc - 1; r >= 0; --r)
            for (index_t k = 0; k < nrhs; ++k) {
                double acc = Y(s.col_begin + r, k);
                for (index_t c = r + 1; c < nc; ++c)
                    acc -= s.L[static_cast<std::size_t>(c) * nc + r] * Y(s.col_begin + c, k);
                Y(s.col_begin + r, k) = acc / s.L[static_cast<std::size_t>(r) * nc + r];
            }
    }
    for (index_t p = 0; p < nI; ++p)
        for (index_t k = 0; k < nrhs; ++k)
            X[static_cast<std::size_t>(F.perm[p]) * nrhs + k] = y[static_cast<std::size_t>(p) * nrhs + k];
}

}  // namespace bddc_b200

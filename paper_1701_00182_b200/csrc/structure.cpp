// Cluster tree / block cluster tree flattening (see structure.hpp).
// Reference: /root/reference/proj/core/src/cluster.cpp:9-126.
#include "structure.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>

namespace acrgpu {

namespace {

struct Box {
    double x0, x1, y0, y1;
    double diam() const { return std::sqrt((x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0)); }
    double dist(const Box& o) const {
        const double dx = std::max({0.0, o.x0 - x1, x0 - o.x1});
        const double dy = std::max({0.0, o.y0 - y1, y0 - o.y1});
        return std::sqrt(dx * dx + dy * dy);
    }
};

struct CNode {
    int begin, end;
    Box box;
    int lo = -1, hi = -1;
    bool leaf() const { return lo < 0; }
};

}  // namespace

void Structure::build(int dim_, const double* xy, int leaf_size_, double eta_, int weak_) {
    if (dim_ < 1) throw StructureError{4, "ClusterTree: empty point set"};
    if (leaf_size_ < 1) throw StructureError{4, "ClusterTree: leaf_size must be >= 1"};
    if (!(eta_ > 0)) throw StructureError{4, "BlockClusterTree: eta must be positive"};
    dim = dim_;
    leaf_size = leaf_size_;
    eta = eta_;
    weak = weak_;
    perm.resize(dim);
    std::iota(perm.begin(), perm.end(), 0);

    // ---- cluster tree: stable median split along the longer box side
    std::vector<CNode> cl;
    std::function<int(int, int, int)> make = [&](int b, int e, int depth) -> int {
        CNode c;
        c.begin = b;
        c.end = e;
        Box bx{xy[2 * perm[b]], xy[2 * perm[b]], xy[2 * perm[b] + 1], xy[2 * perm[b] + 1]};
        for (int i = b + 1; i < e; ++i) {
            const double x = xy[2 * perm[i]], y = xy[2 * perm[i] + 1];
            bx.x0 = std::min(bx.x0, x);
            bx.x1 = std::max(bx.x1, x);
            bx.y0 = std::min(bx.y0, y);
            bx.y1 = std::max(bx.y1, y);
        }
        c.box = bx;
        const int id = (int)cl.size();
        cl.push_back(c);
        if (e - b > leaf_size) {
            const int axis = (bx.x1 - bx.x0) >= (bx.y1 - bx.y0) ? 0 : 1;
            std::stable_sort(perm.begin() + b, perm.begin() + e,
                             [&](int p, int q) { return xy[2 * p + axis] < xy[2 * q + axis]; });
            const int mid = b + (e - b) / 2;
            const int lo = make(b, mid, depth + 1);
            const int hi = make(mid, e, depth + 1);
            cl[id].lo = lo;
            cl[id].hi = hi;
        } else {
            ++cluster_leaves;
            cluster_depth = std::max(cluster_depth, depth);
        }
        return id;
    };
    cluster_leaves = 0;
    cluster_depth = 0;
    make(0, dim, 0);
    iperm.resize(dim);
    for (int i = 0; i < dim; ++i) iperm[perm[i]] = i;

    // ---- block cluster tree, flattened in DFS order
    auto admissible = [&](const CNode& t, const CNode& s) {
        if (weak) return t.end <= s.begin || s.end <= t.begin;
        return std::min(t.box.diam(), s.box.diam()) <= eta * t.box.dist(s.box);
    };
    nodes.clear();
    d_node.clear();
    d_off.clear();
    k_node.clear();
    dense_total = 0;
    max_dense_dim = 0;
    std::function<int(int, int)> bt = [&](int ti, int si) -> int {
        const CNode& t = cl[ti];
        const CNode& s = cl[si];
        const int id = (int)nodes.size();
        nodes.emplace_back();
        {
            SNode& n = nodes[id];
            n.rb = t.begin; n.re = t.end; n.cb = s.begin; n.ce = s.end;
            n.d0 = (int)d_node.size();
            n.k0 = (int)k_node.size();
            n.doff0 = dense_total;
        }
        if (admissible(t, s)) {
            nodes[id].kind = K_RK;
            nodes[id].leaf = (int)k_node.size();
            k_node.push_back(id);
        } else if (!t.leaf() && !s.leaf()) {
            nodes[id].kind = K_BRANCH;
            const int tc[2] = {t.lo, t.hi};
            const int sc[2] = {s.lo, s.hi};
            for (int i = 0; i < 2; ++i)
                for (int j = 0; j < 2; ++j) {
                    const int c = bt(tc[i], sc[j]);
                    nodes[id].ch[i * 2 + j] = c;
                }
        } else {
            nodes[id].kind = K_DENSE;
            nodes[id].leaf = (int)d_node.size();
            d_node.push_back(id);
            d_off.push_back(dense_total);
            const long m = t.end - t.begin, n = s.end - s.begin;
            dense_total += m * n;
            max_dense_dim = std::max<int>(max_dense_dim, (int)std::max(m, n));
        }
        SNode& n = nodes[id];
        n.d1 = (int)d_node.size();
        n.k1 = (int)k_node.size();
        n.dsize = dense_total - n.doff0;
        return id;
    };
    bt(0, 0);

    // leaf clusters in tree order
    cl_begin.clear();
    cl_end.clear();
    for (const CNode& c : cl)
        if (c.leaf()) {
            cl_begin.push_back(c.begin);
            cl_end.push_back(c.end);
        }
    {
        std::vector<int> idx(cl_begin.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::sort(idx.begin(), idx.end(), [&](int x, int y) { return cl_begin[x] < cl_begin[y]; });
        std::vector<int> b2, e2;
        for (int i : idx) {
            b2.push_back(cl_begin[i]);
            e2.push_back(cl_end[i]);
        }
        cl_begin = b2;
        cl_end = e2;
    }
    cl_index.assign(dim, 0);
    for (size_t i = 0; i < cl_begin.size(); ++i)
        for (int p = cl_begin[i]; p < cl_end[i]; ++p) cl_index[p] = (int)i;
    // mixed dense/branch products (reference hmatrix.cpp:442-453) only arise in
    // unbalanced trees: a dense leaf whose row or column range is not one leaf cluster.
    balanced = true;
    for (int d : d_node) {
        const SNode& n = nodes[d];
        const int ri = cl_index[n.rb], ci = cl_index[n.cb];
        if (cl_begin[ri] != n.rb || cl_end[ri] != n.re || cl_begin[ci] != n.cb || cl_end[ci] != n.ce) balanced = false;
    }
}

int Structure::find_leaf(int r, int c) const {
    int i = 0;
    while (nodes[i].kind == K_BRANCH) {
        const SNode& n = nodes[i];
        const SNode& c0 = nodes[n.ch[0]];
        const int rr = r < c0.re ? 0 : 1;
        const int cc = c < c0.ce ? 0 : 1;
        i = n.ch[rr * 2 + cc];
    }
    return i;
}

}  // namespace acrgpu

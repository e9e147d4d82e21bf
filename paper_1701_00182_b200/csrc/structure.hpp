// Host-side "structure compiler": geometric cluster tree, block cluster tree and
// the flattened leaf tables every device H-matrix is laid out by.
//
// The tree algorithms restate /root/reference/proj/core/src/cluster.cpp:39-126
// (median bisection on the longer bounding-box side with a stable sort;
// standard admissibility min(diam) <= eta*dist, or weak = disjoint ranges;
// quadtree subdivision while both clusters split).  Ranks depend on the
// structure, so it must match the reference exactly (tests/test_structure.py).
//
// Flattening: nodes are numbered in DFS order (children 0..3 = [row*2+col]);
// dense leaves and low-rank (Rk) leaves are numbered separately in DFS order,
// so every subtree owns a contiguous range of dense ids and of Rk ids, and a
// contiguous slice of the dense pool.  A device H-matrix "view" of node s is
// therefore just base pointers offset by the first ids of s.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace acrgpu {

enum Kind : int { K_DENSE = 0, K_RK = 1, K_BRANCH = 2 };

struct SNode {
    int rb = 0, re = 0, cb = 0, ce = 0;  // tree-order row / column ranges
    int kind = K_DENSE;
    int ch[4] = {-1, -1, -1, -1};        // [row_child * 2 + col_child]
    int leaf = -1;                       // dense id (K_DENSE) or Rk id (K_RK)
    int d0 = 0, d1 = 0;                  // dense ids in subtree
    int k0 = 0, k1 = 0;                  // Rk ids in subtree
    long doff0 = 0;                      // dense pool offset (doubles) of dense id d0
    long dsize = 0;                      // dense pool doubles of the subtree
    int rows() const { return re - rb; }
    int cols() const { return ce - cb; }
};

struct Structure {
    int dim = 0;
    int leaf_size = 0;
    double eta = 2.0;
    int weak = 0;
    std::vector<int> perm, iperm;  // tree pos -> original, original -> tree pos
    std::vector<SNode> nodes;      // nodes[0] = root
    // dense leaves
    std::vector<int> d_node;
    std::vector<long> d_off;       // pool offset (doubles), column-major m x n block
    // Rk leaves
    std::vector<int> k_node;
    long dense_total = 0;
    int max_dense_dim = 0;
    bool balanced = true;          // no mixed dense/branch products can arise
    int cluster_leaves = 0, cluster_depth = 0;
    std::vector<int> cl_begin, cl_end;  // leaf clusters in tree order
    std::vector<int> cl_index;          // tree position -> leaf cluster

    void build(int dim, const double* xy, int leaf_size, double eta, int weak);
    int n_dense() const { return (int)d_node.size(); }
    int n_rk() const { return (int)k_node.size(); }
    const SNode& node(int i) const { return nodes[i]; }
    // locate the leaf node containing tree-order entry (r, c)
    int find_leaf(int r, int c) const;
};

struct StructureError {
    int code;
    std::string msg;
};

}  // namespace acrgpu

// Prefix tree and partitioner, host side.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ttb {

// TokenSequence (token_sequence.hpp:15-21); seq_id is the input index.
struct SeqView {
  const int32_t* tokens = nullptr;
  const double* weights = nullptr;  // may be null -> all 1
  uint64_t len = 0;
  double w(uint64_t p) const { return weights ? weights[p] : 1.0; }
};

struct TreeNode {
  std::vector<int32_t> tokens;
  std::vector<int32_t> children;     // indices into PrefixTree::nodes
  std::vector<int32_t> leaf_marks;   // seq ids ending here (ascending)
  std::vector<int32_t> subtree_seqs; // seq ids whose path passes through (ascending)
  uint64_t subtree_tokens = 0;
  uint64_t max_path_below = 0;       // max tokens on a path from this node's first token down
};

// Compressed trie with a virtual root (index 0, empty segment).
struct PrefixTree {
  std::vector<TreeNode> nodes;
  std::vector<std::vector<int32_t>> seq_tokens;   // owned copies of the input
  std::vector<std::vector<double>> seq_weights;
  uint64_t total_tree_tokens = 0;
  uint64_t num_sequences = 0;

  const TreeNode& root() const { return nodes[0]; }
};

// build_prefix_tree; children in first-appearance (as_built) order.
PrefixTree build_prefix_tree(const std::vector<SeqView>& seqs);
// A forest with one top-level node per sequence and no prefix merging (dense baseline).
PrefixTree build_flat_forest(const std::vector<SeqView>& seqs);
// order_children.
void order_children(PrefixTree& t, int policy);
std::string serialize_tree(const PrefixTree& t);
std::string dfs_trace(const PrefixTree& t);
std::vector<int32_t> preorder(const PrefixTree& t);  // node indices, virtual root excluded

// Loss pairs of one node: (row, target, weight) with weights summed over the
// sequences through the node / through each child; zero weights dropped.
struct LossPairs {
  std::vector<int32_t> rows, targets;
  std::vector<double> weights;
};
LossPairs node_loss_pairs(const PrefixTree& t, int32_t node, uint64_t start);

// ------------------------------------------------------------------ partitioner
std::vector<uint64_t> lexicographic_order(const std::vector<SeqView>& seqs);
uint64_t group_tree_cost(const std::vector<SeqView>& seqs, const std::vector<uint64_t>& members);
struct PartitionPlan {
  std::vector<std::vector<uint64_t>> groups;  // seq indices
  std::vector<uint64_t> costs;
  uint64_t max_cost = 0;
  uint64_t duplicated = 0;
};
PartitionPlan partition_contiguous(const std::vector<SeqView>& seqs, uint64_t K);
PartitionPlan greedy_least_loaded(const std::vector<SeqView>& seqs, uint64_t K, int cost_mode);

}  // namespace ttb

// Drives the C++ wrapper (include/treetrain_b200.hpp) the way a reference-side caller would:
// build_prefix_tree on the SPEC examples, print serialisation / trace / token count, partition.
#include <iostream>

#include "treetrain_b200.hpp"

int main() {
  using namespace treetrain_b200;
  std::vector<TokenSequence> seqs = {{{1, 2, 3}, {}}, {{1, 2, 4}, {}}, {{1, 2}, {}}, {{7, 7, 7, 7}, {}}};
  PrefixTree t(seqs);
  std::cout << "TOKENS " << t.tree_token_count() << "\n" << t.serialize() << t.dfs_trace();
  auto [groups, mx] = partition_contiguous(seqs, 2);
  std::cout << "MAXCOST " << mx << "\nGROUPS";
  for (int g : groups) std::cout << " " << g;
  std::cout << "\n";
  try {
    PrefixTree bad(std::vector<TokenSequence>{});
    std::cout << "NO-THROW\n";
  } catch (const std::invalid_argument& e) {
    std::cout << "INVALID_ARGUMENT " << e.what() << "\n";
  }
  return 0;
}

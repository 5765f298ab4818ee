// Prefix tree and partitioner, host side.
#include "prefix_tree.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <unordered_map>

namespace ttb {

namespace {

void finish_stats(PrefixTree& t) {
  // post-order subtree_tokens / max_path_below
  std::function<void(int32_t)> rec = [&](int32_t u) {
    TreeNode& n = t.nodes[u];
    uint64_t st = n.tokens.size(), mp = 0;
    for (int32_t c : n.children) {
      rec(c);
      st += t.nodes[c].subtree_tokens;
      mp = std::max(mp, t.nodes[c].max_path_below);
    }
    n.subtree_tokens = st;
    n.max_path_below = n.tokens.size() + mp;
  };
  rec(0);
  t.total_tree_tokens = t.nodes[0].subtree_tokens;
}

void copy_inputs(PrefixTree& t, const std::vector<SeqView>& seqs) {
  if (seqs.empty()) throw std::invalid_argument("build_prefix_tree: empty sequence list");
  t.seq_tokens.resize(seqs.size());
  t.seq_weights.resize(seqs.size());
  for (size_t i = 0; i < seqs.size(); ++i) {
    if (seqs[i].len == 0) throw std::invalid_argument("build_prefix_tree: empty token list");
    t.seq_tokens[i].assign(seqs[i].tokens, seqs[i].tokens + seqs[i].len);
    t.seq_weights[i].resize(seqs[i].len);
    for (uint64_t p = 0; p < seqs[i].len; ++p) {
      const double w = seqs[i].w(p);
      if (!std::isfinite(w)) throw std::invalid_argument("build_prefix_tree: non-finite weight");
      t.seq_weights[i][p] = w;
    }
  }
  t.num_sequences = seqs.size();
}

// Groups ids (kept in input order) by their token at depth p, in first-appearance order.
std::vector<std::vector<int32_t>> group_by_token(const PrefixTree& t, const std::vector<int32_t>& ids, uint64_t p) {
  std::vector<std::vector<int32_t>> groups;
  std::unordered_map<int32_t, size_t> where;
  for (int32_t i : ids) {
    const int32_t tok = t.seq_tokens[i][p];
    auto it = where.find(tok);
    if (it == where.end()) {
      where.emplace(tok, groups.size());
      groups.push_back({i});
    } else {
      groups[it->second].push_back(i);
    }
  }
  return groups;
}

int32_t build_rec(PrefixTree& t, const std::vector<int32_t>& ids, uint64_t p) {
  // extend while every sequence continues with the same token and none ends (radix compression)
  const auto& first = t.seq_tokens[ids[0]];
  uint64_t q = p;
  for (;;) {
    bool stop = false;
    for (int32_t i : ids) {
      if (t.seq_tokens[i].size() == q) {
        stop = true;
        break;
      }
    }
    if (stop) break;
    const int32_t tok = first.size() > q ? first[q] : -1;
    for (int32_t i : ids) {
      if (t.seq_tokens[i][q] != tok) {
        stop = true;
        break;
      }
    }
    if (stop) break;
    ++q;
  }
  const int32_t u = static_cast<int32_t>(t.nodes.size());
  t.nodes.emplace_back();
  t.nodes[u].tokens.assign(first.begin() + p, first.begin() + q);
  std::vector<int32_t> rest;
  for (int32_t i : ids) {
    if (t.seq_tokens[i].size() == q) t.nodes[u].leaf_marks.push_back(i);
    else rest.push_back(i);
  }
  std::vector<int32_t> sorted_ids = ids;
  std::sort(sorted_ids.begin(), sorted_ids.end());
  t.nodes[u].subtree_seqs = sorted_ids;
  std::sort(t.nodes[u].leaf_marks.begin(), t.nodes[u].leaf_marks.end());
  if (!rest.empty()) {
    for (auto& g : group_by_token(t, rest, q)) {
      const int32_t c = build_rec(t, g, q);
      t.nodes[u].children.push_back(c);
    }
  }
  return u;
}

}  // namespace

PrefixTree build_prefix_tree(const std::vector<SeqView>& seqs) {
  PrefixTree t;
  copy_inputs(t, seqs);
  t.nodes.emplace_back();  // virtual root
  std::vector<int32_t> all(seqs.size());
  std::iota(all.begin(), all.end(), 0);
  t.nodes[0].subtree_seqs = all;
  for (auto& g : group_by_token(t, all, 0)) {
    const int32_t c = build_rec(t, g, 0);
    t.nodes[0].children.push_back(c);
  }
  finish_stats(t);
  return t;
}

PrefixTree build_flat_forest(const std::vector<SeqView>& seqs) {
  PrefixTree t;
  copy_inputs(t, seqs);
  t.nodes.emplace_back();
  for (size_t i = 0; i < seqs.size(); ++i) {
    TreeNode n;
    n.tokens = t.seq_tokens[i];
    n.leaf_marks = {static_cast<int32_t>(i)};
    n.subtree_seqs = {static_cast<int32_t>(i)};
    t.nodes[0].subtree_seqs.push_back(static_cast<int32_t>(i));
    t.nodes[0].children.push_back(static_cast<int32_t>(t.nodes.size()));
    t.nodes.push_back(std::move(n));
  }
  finish_stats(t);
  return t;
}

void order_children(PrefixTree& t, int policy) {
  if (policy < 0 || policy > 3) throw std::invalid_argument("order_children: unknown policy");
  if (policy == 0) return;  // as_built
  for (auto& n : t.nodes) {
    auto key_tok = [&](int32_t c) { return t.nodes[c].tokens.empty() ? -1 : t.nodes[c].tokens[0]; };
    std::stable_sort(n.children.begin(), n.children.end(), [&](int32_t a, int32_t b) {
      if (policy == 2 && t.nodes[a].subtree_tokens != t.nodes[b].subtree_tokens)
        return t.nodes[a].subtree_tokens > t.nodes[b].subtree_tokens;
      if (policy == 3 && t.nodes[a].subtree_tokens != t.nodes[b].subtree_tokens)
        return t.nodes[a].subtree_tokens < t.nodes[b].subtree_tokens;
      return key_tok(a) < key_tok(b);
    });
  }
}

std::vector<int32_t> preorder(const PrefixTree& t) {
  std::vector<int32_t> out;
  std::function<void(int32_t)> rec = [&](int32_t u) {
    out.push_back(u);
    for (int32_t c : t.nodes[u].children) rec(c);
  };
  for (int32_t c : t.nodes[0].children) rec(c);
  return out;
}

std::string serialize_tree(const PrefixTree& t) {
  std::string s;
  std::function<void(int32_t, int)> rec = [&](int32_t u, int depth) {
    const TreeNode& n = t.nodes[u];
    s += std::to_string(depth) + " " + std::to_string(n.tokens.size()) + " ";
    for (size_t i = 0; i < n.tokens.size(); ++i) {
      if (i) s += ' ';
      s += std::to_string(n.tokens[i]);
    }
    s += " | ";
    for (size_t i = 0; i < n.leaf_marks.size(); ++i) {
      if (i) s += ' ';
      s += std::to_string(n.leaf_marks[i]);
    }
    s += " | " + std::to_string(n.children.size()) + "\n";
    for (int32_t c : n.children) rec(c, depth + 1);
  };
  for (int32_t c : t.nodes[0].children) rec(c, 0);
  return s;
}

std::string dfs_trace(const PrefixTree& t) {
  const auto pre = preorder(t);
  std::vector<int32_t> id(t.nodes.size(), -1);
  for (size_t i = 0; i < pre.size(); ++i) id[pre[i]] = static_cast<int32_t>(i);
  std::string s;
  std::function<void(int32_t)> rec = [&](int32_t u) {
    s += "PUSH " + std::to_string(id[u]) + "\n";
    for (int32_t c : t.nodes[u].children) rec(c);
    s += "POP " + std::to_string(id[u]) + "\n";
  };
  for (int32_t c : t.nodes[0].children) rec(c);
  return s;
}

LossPairs node_loss_pairs(const PrefixTree& t, int32_t u, uint64_t start) {
  LossPairs lp;
  const TreeNode& n = t.nodes[u];
  const uint64_t L = n.tokens.size();
  for (uint64_t r = 0; r + 1 < L; ++r) {
    const uint64_t pos = start + r + 1;
    double w = 0.0;
    for (int32_t i : n.subtree_seqs) w += t.seq_weights[i][pos];
    if (w != 0.0) {
      lp.rows.push_back(static_cast<int32_t>(r));
      lp.targets.push_back(n.tokens[r + 1]);
      lp.weights.push_back(w);
    }
  }
  for (int32_t c : n.children) {
    const uint64_t pos = start + L;
    double w = 0.0;
    for (int32_t i : t.nodes[c].subtree_seqs) w += t.seq_weights[i][pos];
    if (w != 0.0) {
      lp.rows.push_back(static_cast<int32_t>(L - 1));
      lp.targets.push_back(t.nodes[c].tokens[0]);
      lp.weights.push_back(w);
    }
  }
  return lp;
}

// ------------------------------------------------------------------ partitioner
namespace {

bool lex_less(const SeqView& a, const SeqView& b) {
  return std::lexicographical_compare(a.tokens, a.tokens + a.len, b.tokens, b.tokens + b.len);
}

uint64_t lcp(const SeqView& a, const SeqView& b) {
  const uint64_t n = std::min(a.len, b.len);
  uint64_t k = 0;
  while (k < n && a.tokens[k] == b.tokens[k]) ++k;
  return k;
}

}  // namespace

std::vector<uint64_t> lexicographic_order(const std::vector<SeqView>& seqs) {
  std::vector<uint64_t> ord(seqs.size());
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t b) { return lex_less(seqs[a], seqs[b]); });
  return ord;
}

// tree_token_count of a group = sum len - sum LCP of lexicographic neighbours.
uint64_t group_tree_cost(const std::vector<SeqView>& seqs, const std::vector<uint64_t>& members) {
  std::vector<uint64_t> m = members;
  std::stable_sort(m.begin(), m.end(), [&](uint64_t a, uint64_t b) { return lex_less(seqs[a], seqs[b]); });
  uint64_t c = 0;
  for (size_t i = 0; i < m.size(); ++i) c += seqs[m[i]].len - (i ? lcp(seqs[m[i - 1]], seqs[m[i]]) : 0);
  return c;
}

namespace {

std::vector<std::vector<uint64_t>> greedy_groups(const std::vector<SeqView>& seqs, const std::vector<uint64_t>& ord,
                                                 uint64_t tau) {
  std::vector<std::vector<uint64_t>> groups(1);
  uint64_t cost = 0;
  for (size_t k = 0; k < ord.size(); ++k) {
    const SeqView& s = seqs[ord[k]];
    uint64_t c = groups.back().empty() ? s.len : cost + s.len - lcp(seqs[groups.back().back()], s);
    if (!groups.back().empty() && c > tau) {
      groups.emplace_back();
      c = s.len;
    }
    groups.back().push_back(ord[k]);
    cost = c;
  }
  return groups;
}

PartitionPlan finish_plan(const std::vector<SeqView>& seqs, std::vector<std::vector<uint64_t>> groups, uint64_t K) {
  PartitionPlan p;
  groups.resize(std::max<size_t>(groups.size(), K));
  p.groups = std::move(groups);
  std::vector<uint64_t> all(seqs.size());
  std::iota(all.begin(), all.end(), 0);
  uint64_t sum = 0;
  for (auto& g : p.groups) {
    p.costs.push_back(group_tree_cost(seqs, g));
    sum += p.costs.back();
    p.max_cost = std::max(p.max_cost, p.costs.back());
  }
  p.duplicated = sum - group_tree_cost(seqs, all);
  return p;
}

}  // namespace

PartitionPlan partition_contiguous(const std::vector<SeqView>& seqs, uint64_t K) {
  if (K < 1 || seqs.empty()) throw std::invalid_argument("partition_contiguous: K >= 1 and N >= 1 required");
  const auto ord = lexicographic_order(seqs);
  uint64_t lo = 0;
  for (auto& s : seqs) lo = std::max(lo, s.len);
  std::vector<uint64_t> all(seqs.size());
  std::iota(all.begin(), all.end(), 0);
  uint64_t hi = group_tree_cost(seqs, all);
  while (lo < hi) {  // smallest feasible integer tau
    const uint64_t mid = lo + (hi - lo) / 2;
    if (greedy_groups(seqs, ord, mid).size() <= K) hi = mid;
    else lo = mid + 1;
  }
  return finish_plan(seqs, greedy_groups(seqs, ord, lo), K);
}

PartitionPlan greedy_least_loaded(const std::vector<SeqView>& seqs, uint64_t K, int cost_mode) {
  if (K < 1) throw std::invalid_argument("greedy_least_loaded: K >= 1 required");
  std::vector<std::vector<uint64_t>> groups(K);
  std::vector<uint64_t> load(K, 0);
  for (uint64_t i = 0; i < seqs.size(); ++i) {
    uint64_t g = 0;
    for (uint64_t j = 1; j < K; ++j)
      if (load[j] < load[g]) g = j;
    groups[g].push_back(i);
    load[g] = cost_mode == 1 ? load[g] + seqs[i].len : group_tree_cost(seqs, groups[g]);
  }
  return finish_plan(seqs, std::move(groups), K);
}

}  // namespace ttb

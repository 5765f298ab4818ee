// Rollout corpus I/O and the grouped synthetic generator ("Corpus format", SPEC.md:
// 484-501 [TYPE] CorpusSpec / [OP] gen-corpus). The reference lists corpus_io.cpp / corpus_gen.cpp in
// proj/core/CMakeLists.txt:1-10 but does not ship them; this follows the SPEC text.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ttb {

struct CorpusSeq {
  std::string seq_id;           // string id (numbers in the JSON are kept as their text)
  std::vector<int32_t> tokens;  // TokenId = int32 (token_sequence.hpp:9)
  std::vector<double> weights;  // per-position NLL weights (token_sequence.hpp:11-14)
};

// One JSON object per line: {"seq_id": str|int, "tokens": [int], "weights": [float]} with weights
// optional: absent -> 0 on the first "prompt_len" positions when that field is present, else all 1.
// Throws std::runtime_error on I/O failure, std::invalid_argument on malformed lines (with line no.).
std::vector<CorpusSeq> load_corpus_jsonl(const std::string& path);
void save_corpus_jsonl(const std::string& path, const std::vector<CorpusSeq>& seqs);

// [TYPE] CorpusSpec. Lengths are drawn uniformly from [lo, hi].
struct CorpusSpec {
  uint64_t num_prompts = 1;
  uint64_t group_size = 1;
  uint64_t prompt_len_lo = 1, prompt_len_hi = 1;
  uint64_t response_len_lo = 1, response_len_hi = 1;
  double branch_prob = 1.0;
  uint64_t vocab_size = 2;
  uint64_t seed = 0;
};

// [OP] gen-corpus: num_prompts x group_size rollouts; a group shares its prompt and
// a response stem whose length is geometric in branch_prob (the siblings diverge at the first stem
// position where a Bernoulli(branch_prob) trial succeeds; branch_prob = 1 -> immediately); weights 0
// on prompt positions, 1 on response positions; deterministic per seed (mt19937_64).
std::vector<CorpusSeq> gen_corpus(const CorpusSpec& spec);

}  // namespace ttb

// Corpus JSONL reader/writer and grouped synthetic generator. Host-only.
#include "corpus_io.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <stdexcept>

namespace ttb {

namespace {

// Minimal JSON scanner for one corpus line: objects, arrays, strings, numbers, true/false/null.
struct Scanner {
  const std::string& s;
  size_t i = 0;
  long line;

  [[noreturn]] void fail(const char* what) const {
    throw std::invalid_argument("corpus line " + std::to_string(line) + ": " + what + " at column " +
                                std::to_string(i + 1));
  }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\r' || s[i] == '\n')) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail((std::string("expected '") + c + "'").c_str());
  }
  std::string str() {
    ws();
    if (i >= s.size() || s[i] != '"') fail("expected a string");
    ++i;
    std::string out;
    while (i < s.size() && s[i] != '"') {
      char c = s[i++];
      if (c == '\\') {
        if (i >= s.size()) fail("bad escape");
        const char e = s[i++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {  // keep \uXXXX verbatim (ids are opaque)
            out += "\\u";
            for (int k = 0; k < 4 && i < s.size(); ++k) out += s[i++];
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
  // number token as text (for string ids given as numbers) and as double
  std::string num_text() {
    ws();
    const size_t b = i;
    while (i < s.size() && (std::strchr("+-0123456789.eE", s[i]) != nullptr)) ++i;
    if (i == b) fail("expected a number");
    return s.substr(b, i - b);
  }
  double num() {
    const std::string t = num_text();
    char* end = nullptr;
    const double v = std::strtod(t.c_str(), &end);
    if (end != t.c_str() + t.size()) fail("malformed number");
    return v;
  }
  void skip_value() {
    ws();
    if (i >= s.size()) fail("unexpected end of line");
    const char c = s[i];
    if (c == '"') {
      str();
    } else if (c == '{') {
      ++i;
      if (eat('}')) return;
      do {
        str();
        expect(':');
        skip_value();
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i;
      if (eat(']')) return;
      do skip_value();
      while (eat(','));
      expect(']');
    } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 4, "null") == 0) {
      i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      i += 5;
    } else {
      num_text();
    }
  }
  template <typename F>
  void array(F&& elem) {
    expect('[');
    if (eat(']')) return;
    do elem();
    while (eat(','));
    expect(']');
  }
};

std::string json_escape(const std::string& v) {
  std::string o;
  for (char c : v) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o;
}

}  // namespace

std::vector<CorpusSeq> load_corpus_jsonl(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_corpus_jsonl: cannot open " + path);
  std::vector<CorpusSeq> out;
  std::string text;
  long line = 0;
  while (std::getline(in, text)) {
    ++line;
    Scanner sc{text, 0, line};
    sc.ws();
    if (sc.i == text.size()) continue;  // blank line
    CorpusSeq q;
    bool have_id = false, have_tokens = false, have_weights = false;
    long prompt_len = -1;
    sc.expect('{');
    if (!sc.eat('}')) {
      do {
        const std::string key = sc.str();
        sc.expect(':');
        if (key == "seq_id") {
          sc.ws();
          q.seq_id = (sc.i < text.size() && text[sc.i] == '"') ? sc.str() : sc.num_text();
          have_id = true;
        } else if (key == "tokens") {
          sc.array([&] {
            const double v = sc.num();
            if (v != std::floor(v) || v < 0 || v > 2147483647.0) sc.fail("token ids must be non-negative int32");
            q.tokens.push_back(static_cast<int32_t>(v));
          });
          have_tokens = true;
        } else if (key == "weights") {
          sc.array([&] { q.weights.push_back(sc.num()); });
          have_weights = true;
        } else if (key == "prompt_len") {
          const double v = sc.num();
          if (v != std::floor(v) || v < 0) sc.fail("prompt_len must be a non-negative integer");
          prompt_len = static_cast<long>(v);
        } else {
          sc.skip_value();
        }
      } while (sc.eat(','));
      sc.expect('}');
    }
    sc.ws();
    if (sc.i != text.size()) sc.fail("trailing characters");
    if (!have_id) sc.fail("missing \"seq_id\"");
    if (!have_tokens || q.tokens.empty()) sc.fail("missing or empty \"tokens\"");
    if (have_weights) {
      if (q.weights.size() != q.tokens.size()) sc.fail("\"weights\" length differs from \"tokens\"");
    } else {  // SPEC.md:192 defaults
      q.weights.assign(q.tokens.size(), 1.0);
      if (prompt_len >= 0)
        for (size_t p = 0; p < q.tokens.size() && static_cast<long>(p) < prompt_len; ++p) q.weights[p] = 0.0;
    }
    out.push_back(std::move(q));
  }
  return out;
}

void save_corpus_jsonl(const std::string& path, const std::vector<CorpusSeq>& seqs) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("save_corpus_jsonl: cannot write " + path);
  std::string line;
  char buf[64];
  for (const auto& q : seqs) {
    line = "{\"seq_id\": \"" + json_escape(q.seq_id) + "\", \"tokens\": [";
    for (size_t p = 0; p < q.tokens.size(); ++p) {
      if (p) line += ", ";
      line += std::to_string(q.tokens[p]);
    }
    line += "], \"weights\": [";
    for (size_t p = 0; p < q.weights.size(); ++p) {
      if (p) line += ", ";
      std::snprintf(buf, sizeof(buf), "%.17g", q.weights[p]);  // exact double round trip
      line += buf;
    }
    line += "]}\n";
    if (std::fwrite(line.data(), 1, line.size(), f) != line.size()) {
      std::fclose(f);
      throw std::runtime_error("save_corpus_jsonl: write failed for " + path);
    }
  }
  if (std::fclose(f) != 0) throw std::runtime_error("save_corpus_jsonl: close failed for " + path);
}

std::vector<CorpusSeq> gen_corpus(const CorpusSpec& sp) {
  if (sp.num_prompts < 1 || sp.group_size < 1 || sp.vocab_size < 2 || sp.prompt_len_lo > sp.prompt_len_hi ||
      sp.response_len_lo > sp.response_len_hi || sp.response_len_lo < 1 || !(sp.branch_prob >= 0.0) ||
      sp.branch_prob > 1.0)
    throw std::invalid_argument("gen_corpus: invalid CorpusSpec (SPEC.md:487-490)");
  std::mt19937_64 rng(sp.seed);
  const uint64_t V = sp.vocab_size;
  auto uni = [&](uint64_t lo, uint64_t hi) { return lo + rng() % (hi - lo + 1); };  // inclusive
  auto tok = [&] { return static_cast<int32_t>(rng() % V); };
  auto unit = [&] { return static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0); };
  // k distinct values in [0, V) (partial Fisher-Yates over a lazily materialised permutation)
  auto distinct = [&](uint64_t k) {
    std::vector<int32_t> out;
    if (k > V) {  // more than the vocabulary: collisions unavoidable
      for (uint64_t i = 0; i < k; ++i) out.push_back(tok());
      return out;
    }
    std::vector<std::pair<uint64_t, uint64_t>> swaps;  // sparse permutation
    auto at = [&](uint64_t idx) {
      for (auto it = swaps.rbegin(); it != swaps.rend(); ++it)
        if (it->first == idx) return it->second;
      return idx;
    };
    for (uint64_t i = 0; i < k; ++i) {
      const uint64_t j = i + rng() % (V - i);
      const uint64_t vi = at(i), vj = at(j);
      swaps.emplace_back(i, vj);
      swaps.emplace_back(j, vi);
      out.push_back(static_cast<int32_t>(vj));
    }
    return out;
  };
  std::vector<CorpusSeq> out;
  const std::vector<int32_t> prompt_first = distinct(sp.num_prompts);  // distinct prompts never merge
  for (uint64_t pi = 0; pi < sp.num_prompts; ++pi) {
    const uint64_t P = uni(sp.prompt_len_lo, sp.prompt_len_hi);
    std::vector<int32_t> prompt(P);
    for (uint64_t t = 0; t < P; ++t) prompt[t] = t == 0 ? prompt_first[pi] : tok();
    // shared response stem: geometric length (failures before the first divergence trial succeeds)
    uint64_t stem_len = 0;
    if (sp.branch_prob < 1.0) {
      while (stem_len < sp.response_len_hi && unit() >= sp.branch_prob) ++stem_len;
    }
    std::vector<int32_t> stem(stem_len);
    for (auto& x : stem) x = tok();
    // the siblings diverge right after the stem: distinct tokens there
    const std::vector<int32_t> div = distinct(sp.group_size);
    for (uint64_t g = 0; g < sp.group_size; ++g) {
      const uint64_t R = uni(sp.response_len_lo, sp.response_len_hi);
      CorpusSeq q;
      q.seq_id = std::to_string(out.size());
      q.tokens = prompt;
      for (uint64_t t = 0; t < R; ++t) {
        int32_t v;
        if (t < stem_len) v = stem[t];
        else if (t == stem_len) v = div[g];
        else v = tok();
        q.tokens.push_back(v);
      }
      q.weights.assign(q.tokens.size(), 1.0);
      for (uint64_t t = 0; t < P; ++t) q.weights[t] = 0.0;
      out.push_back(std::move(q));
    }
  }
  return out;
}

}  // namespace ttb

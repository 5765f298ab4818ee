// TTPM parameter-file reader (layout of model_io.cpp:44-105): "TTPM", u32 header length, JSON
// header {config, dtype, tensors[{name, offset, shape}]}, raw little-endian tensors in
// for_each_tensor order. A minimal JSON reader is enough for this fixed header.
#include "ttpm.hpp"

#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>

namespace ttb {

namespace {

struct JVal {
  enum Kind { Null, Num, Str, Arr, Obj } kind = Null;
  double num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal& at(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw std::runtime_error("load_parameters: header missing key " + k);
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  char peek() {
    ws();
    if (i >= s.size()) throw std::runtime_error("load_parameters: truncated JSON header");
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) throw std::runtime_error(std::string("load_parameters: bad JSON, expected ") + c);
    ++i;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      out += s[i++];
    }
    ++i;
    return out;
  }
  JVal val() {
    JVal v;
    const char c = peek();
    if (c == '{') {
      v.kind = JVal::Obj;
      ++i;
      if (peek() == '}') {
        ++i;
        return v;
      }
      for (;;) {
        std::string k = str();
        expect(':');
        v.obj.emplace_back(k, val());
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect('}');
        return v;
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++i;
      if (peek() == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(val());
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect(']');
        return v;
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.str = str();
      return v;
    }
    size_t j = i;
    while (j < s.size() && (isdigit(static_cast<unsigned char>(s[j])) || s[j] == '-' || s[j] == '+' || s[j] == '.' ||
                            s[j] == 'e' || s[j] == 'E'))
      ++j;
    if (j == i) throw std::runtime_error("load_parameters: bad JSON value");
    v.kind = JVal::Num;
    v.num = std::stod(s.substr(i, j - i));
    i = j;
    return v;
  }
};

uint64_t u(const JVal& v) { return static_cast<uint64_t>(v.num); }

}  // namespace

std::vector<std::pair<std::string, std::vector<uint64_t>>> tensor_specs(const tt_model_config& c) {
  const uint64_t d = c.d_model, V = c.vocab_size, F = c.d_ff;
  std::vector<std::pair<std::string, std::vector<uint64_t>>> out;
  out.push_back({"embedding", {V, d}});
  for (uint64_t i = 0; i < c.n_layers; ++i) {
    const std::string b = "layers." + std::to_string(i) + ".";
    out.push_back({b + "attn_norm_gain", {d}});
    out.push_back({b + "w_q", {d, d}});
    out.push_back({b + "w_k", {d, d}});
    out.push_back({b + "w_v", {d, d}});
    out.push_back({b + "w_o", {d, d}});
    out.push_back({b + "mlp_norm_gain", {d}});
    out.push_back({b + "w_mlp_in", {d, F}});
    out.push_back({b + "w_mlp_out", {F, d}});
  }
  out.push_back({"final_norm_gain", {d}});
  out.push_back({"output_head", {d, V}});
  return out;
}

TtpmFile read_ttpm(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("load_parameters: cannot open " + path);
  char magic[4];
  uint32_t hlen = 0;
  f.read(magic, 4);
  f.read(reinterpret_cast<char*>(&hlen), 4);
  if (!f || std::memcmp(magic, "TTPM", 4) != 0) throw std::runtime_error("load_parameters: bad magic in " + path);
  std::string hs(hlen, '\0');
  f.read(hs.data(), hlen);
  Parser p{hs};
  const JVal h = p.val();
  const JVal& c = h.at("config");
  TtpmFile out{};
  out.config.vocab_size = u(c.at("vocab_size"));
  out.config.d_model = u(c.at("d_model"));
  out.config.n_heads = u(c.at("n_heads"));
  out.config.n_layers = u(c.at("n_layers"));
  out.config.d_ff = u(c.at("d_ff"));
  out.config.max_position = u(c.at("max_position"));
  out.config.precision = c.at("precision").str == "f32" ? 0 : 1;
  const std::string dtype = h.at("dtype").str;
  if (dtype != "f32" && dtype != "f64") throw std::runtime_error("load_parameters: dtype mismatch in " + path);
  const auto specs = tensor_specs(out.config);
  const JVal& table = h.at("tensors");
  if (table.arr.size() != specs.size()) throw std::runtime_error("load_parameters: tensor count mismatch");
  uint64_t total = 0;
  for (size_t k = 0; k < specs.size(); ++k) {
    const JVal& e = table.arr[k];
    if (e.at("name").str != specs[k].first)
      throw std::runtime_error("load_parameters: unexpected tensor order at " + specs[k].first);
    std::vector<uint64_t> shape;
    for (auto& x : e.at("shape").arr) shape.push_back(u(x));
    if (shape != specs[k].second) throw std::runtime_error("load_parameters: shape mismatch for " + specs[k].first);
    uint64_t n = 1;
    for (auto x : shape) n *= x;
    total += n;
  }
  out.values.resize(total);
  if (dtype == "f64") {
    f.read(reinterpret_cast<char*>(out.values.data()), static_cast<std::streamsize>(total * 8));
  } else {
    std::vector<float> tmp(total);
    f.read(reinterpret_cast<char*>(tmp.data()), static_cast<std::streamsize>(total * 4));
    for (uint64_t i = 0; i < total; ++i) out.values[i] = tmp[i];
  }
  if (!f) throw std::runtime_error("load_parameters: truncated file " + path);
  return out;
}

}  // namespace ttb

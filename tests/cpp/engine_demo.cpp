// Drives the whole step through the C++ wrapper (include/treetrain_b200.hpp) on the GPU, the way a
// reference-side C++ caller would, with no Python / PyTorch in the process:
//   1. tree step through a prepared plan: execute, then execute_async + wait while the next plan is
//      prepared, then a one-rank NCCL all-reduce of the GradientStore;
//   2. the same sequences' first one as a segment-level DFS over a 3-segment chain with the loss on
//      the device (push, segment_loss, pop), gradients in f64;
//   3. standalone weighted_nll over host logits.
// Input (binary, written by tests/test_cpp_engine_gpu.py): u64 V d H L F maxpos n_params n_seqs,
// f64 params[n_params], then per sequence: u64 len, i32 tokens[len], f64 weights[len].
// Output: text lines on stdout; gradients (f64) of steps 1 and 2 into <out>.grads1 / <out>.grads2.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "treetrain_b200.hpp"

using namespace treetrain_b200;

template <typename T>
static void rd(std::ifstream& f, T* p, size_t n) {
  f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream f(argv[1], std::ios::binary);
  uint64_t hdr[8];
  rd(f, hdr, 8);
  tt_model_config cfg{};
  cfg.vocab_size = hdr[0];
  cfg.d_model = hdr[1];
  cfg.n_heads = hdr[2];
  cfg.n_layers = hdr[3];
  cfg.d_ff = hdr[4];
  cfg.max_position = hdr[5];
  std::vector<double> params(hdr[6]);
  rd(f, params.data(), params.size());
  std::vector<TokenSequence> seqs(hdr[7]);
  for (auto& s : seqs) {
    uint64_t len = 0;
    rd(f, &len, 1);
    s.tokens.resize(len);
    s.weights.resize(len);
    rd(f, s.tokens.data(), len);
    rd(f, s.weights.data(), len);
  }
  const std::string out = argv[2];

  Engine eng(cfg, 0);
  eng.upload_parameters(params);
  SchedulerConfig sc{};
  sc.child_order_policy = static_cast<int32_t>(ChildOrder::subtree_tokens_desc);
  sc.sibling_batch = 1;

  // 1. plan: execute, execute_async overlapped with the next plan's preparation, NCCL all-reduce
  PrefixTree tree(seqs);
  StepPlan plan = eng.plan(tree, sc);
  eng.zero_gradients();
  TrainStepResult r1 = plan.execute();
  eng.zero_gradients();
  plan.execute_async();
  PrefixTree tree2(seqs);
  StepPlan plan2 = eng.plan(tree2, sc);  // prepared while the step runs
  TrainStepResult r2 = plan.wait();
  std::vector<uint8_t> id = NcclComm::unique_id();
  NcclComm comm(id, 1, 0, 0);
  eng.allreduce_gradients(comm);  // one rank: the identity
  std::vector<double> g1 = eng.gradients_f64();
  std::printf("TREE %.12e %.12e\n", r1.total_loss, r2.total_loss);
  std::ofstream(out + ".grads1", std::ios::binary).write(reinterpret_cast<const char*>(g1.data()),
                                                         static_cast<std::streamsize>(g1.size() * 8));

  // 2. segment-level DFS over the first sequence cut into 3 chained segments, loss on the device
  const auto& s0 = seqs[0];
  const size_t n = s0.tokens.size(), c1 = n / 3, c2 = 2 * n / 3;
  const size_t cut[4] = {0, c1, c2, n};
  eng.zero_gradients();
  eng.reset_stack();
  for (int k = 0; k < 3; ++k)
    eng.push_segment(std::vector<int32_t>(s0.tokens.begin() + cut[k], s0.tokens.begin() + cut[k + 1]));
  double seg_loss = 0.0;
  for (int k = 2; k >= 0; --k) {
    // row t of segment k predicts token t + 1 of the sequence with that token's weight
    std::vector<int32_t> tg;
    std::vector<double> w;
    for (size_t t = cut[k]; t < cut[k + 1]; ++t) {
      tg.push_back(t + 1 < n ? s0.tokens[t + 1] : 0);
      w.push_back(t + 1 < n ? s0.weights[t + 1] : 0.0);
    }
    seg_loss += eng.segment_loss(tg, w);
    eng.backward_segment(nullptr, k > 0);
  }
  std::vector<double> g2 = eng.gradients_f64();
  std::printf("CHAIN %.12e\n", seg_loss);
  std::ofstream(out + ".grads2", std::ios::binary).write(reinterpret_cast<const char*>(g2.data()),
                                                         static_cast<std::streamsize>(g2.size() * 8));

  // 3. weighted_nll over host logits (model.hpp:643-677)
  std::vector<float> logits(2 * cfg.vocab_size);
  for (size_t i = 0; i < logits.size(); ++i) logits[i] = 0.001f * static_cast<float>(i % 97);
  LossResult lr = eng.weighted_nll(logits, {3, 5}, {1.0, 0.5});
  std::printf("NLL %.12e %.9e\n", lr.loss, lr.grad_logits[3]);
  try {
    eng.weighted_nll(logits, {static_cast<int32_t>(cfg.vocab_size), 0}, {1.0, 1.0});
    std::printf("NO-THROW\n");
  } catch (const std::invalid_argument& e) {
    std::printf("INVALID_ARGUMENT %s\n", e.what());
  }
  return 0;
}

// A reference-style controller compiled against the drop-in headers
// (include/p2r/{tensor,model,optim}.hpp) and linked with libp2r.so -- the code a
// user of the reference's C++ API writes, unchanged (SPEC.md:267-284 train_pseudo /
// delink / train_real; SPEC.md:46-66, :144-146 known-answer tests).
//
//   mini_controller <steps_pseudo> <steps_real> <moe 0|1>
//
// Prints one JSON object: KAT results, finite-difference check of the primitive
// layer, and the per-step losses of the Pseudo run, the delinked Real run, and
// the bitwise delink check. tests/test_dropin_gpu.py compares the losses with the
// compiled reference (oracle/_ref) running the same sequence.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "p2r/model.hpp"
#include "p2r/optim.hpp"
#include "p2r/tensor.hpp"

using namespace p2r;

static std::vector<int> tokens_for(int step, int n) {
  std::vector<int> t(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {  // a 32-bit multiplicative hash (the Python test mirrors it)
    std::uint32_t h = static_cast<std::uint32_t>(i + 1) * 2654435761u + static_cast<std::uint32_t>(step) * 40503u;
    h ^= h >> 13;
    h *= 2246822519u;
    h ^= h >> 16;
    t[static_cast<std::size_t>(i)] = static_cast<int>(h % 256u);
  }
  return t;
}

struct Batch {
  std::vector<int> tok, tgt;
  std::vector<std::uint8_t> mask;
};
static Batch lm_batch(int step, int B, int S) {  // make_lm_batch semantics (data.cpp:174-195)
  Batch b;
  b.tok = tokens_for(step, B * S);
  b.tgt.assign(b.tok.size(), 0);
  b.mask.assign(b.tok.size(), 1);
  for (int s = 0; s < B; ++s)
    for (int i = 0; i < S; ++i) {
      const int k = s * S + i;
      if (i + 1 < S)
        b.tgt[static_cast<std::size_t>(k)] = b.tok[static_cast<std::size_t>(k) + 1];
      else
        b.mask[static_cast<std::size_t>(k)] = 0;
    }
  return b;
}

// one micro-step + AdamW, written as the absent controller would
static float train_step(Model& m, AdamW& opt, const LrSchedule& sched, int step, int B, int S) {
  const Batch b = lm_batch(step, B, S);
  double denom = 0;
  for (auto v : b.mask) denom += v;
  m.zero_grads();
  GradTape tape;
  Tensor x = m.embed_forward(&tape, b.tok, B);
  for (int g = 0; g < m.n_graph_layers(); ++g) x = m.block_forward(&tape, g, x, B, AttentionMode::Causal);
  Tensor logits = m.head_forward(&tape, x);
  Tensor loss = softmax_cross_entropy(&tape, logits, b.tgt, b.mask, denom);
  tape.backward_scalar(loss);
  m.flush_shared_layer_grads();
  opt.step(m, sched.at(step));
  return loss.at(0);
}

static bool near(double a, double b, double tol) { return std::fabs(a - b) <= tol; }

int main(int argc, char** argv) {
  const int steps_pseudo = argc > 1 ? std::atoi(argv[1]) : 3;
  const int steps_real = argc > 2 ? std::atoi(argv[2]) : 2;
  const bool moe = argc > 3 && std::atoi(argv[3]) != 0;
  std::string out = "{";
  auto put = [&](const std::string& k, const std::string& v) {
    if (out.size() > 1) out += ", ";
    out += "\"" + k + "\": " + v;
  };
  int fails = 0;
  auto check = [&](const char* name, bool c) {
    if (!c) {
      ++fails;
      std::fprintf(stderr, "FAIL %s\n", name);
    }
    return c;
  };

  // ---- known-answer tests of the primitive layer
  {
    Tensor a = Tensor::from_data({1, 2}, {1, 2}), b = Tensor::from_data({2, 1}, {3, 4});
    check("matmul [[1,2]].[[3],[4]] = 11", matmul(nullptr, a, b).at(0) == 11.0f);
    Tensor c = Tensor::from_data({2, 3}, {1, 2, 3, 4, 5, 6}), eye = Tensor::from_data({3, 3}, {1, 0, 0, 0, 1, 0, 0, 0, 1});
    Tensor ci = matmul(nullptr, c, eye);
    bool same = true;
    for (int i = 0; i < 6; ++i) same = same && ci.at(static_cast<std::size_t>(i)) == c.at(static_cast<std::size_t>(i));
    check("matmul by identity", same);
    Tensor row = Tensor::from_data({1, 4}, {3, 3, 3, 3}), g1 = Tensor::full({4}, 1.f), b0 = Tensor::zeros({4});
    Tensor ln = layernorm(nullptr, row, g1, b0);
    check("layernorm constant row -> 0", near(ln.at(0), 0, 1e-6) && near(ln.at(3), 0, 1e-6));
    Tensor pm = Tensor::from_data({1, 2}, {1, -1});
    Tensor lpm = layernorm(nullptr, pm, Tensor::full({2}, 1.f), Tensor::zeros({2}));
    check("layernorm [1,-1] -> [1,-1]", near(lpm.at(0), 1, 1e-4) && near(lpm.at(1), -1, 1e-4));
    Tensor uni = Tensor::zeros({1, 4});
    const std::vector<int> t0 = {2};
    check("CE uniform V=4 -> ln 4", near(softmax_cross_entropy(nullptr, uni, t0).at(0), std::log(4.0), 1e-5));
    Tensor sat = Tensor::from_data({1, 4}, {0, 0, 100, 0});
    check("CE saturated -> 0", near(softmax_cross_entropy(nullptr, sat, t0).at(0), 0, 1e-5));
    // routing KAT: cf 1.0, E 4 -> capacity 1, selected 0 1 0 0, survived 1 1 0 0, dropped 2
    MoEConfig mc;
    mc.n_experts = 4;
    mc.capacity_factor = 1.0f;
    Routing r = moe_dispatch(Tensor::from_data({4, 4}, {1, 1, 0, 0, 0, 2, 2, 0, 5, 0, 0, 0, 3, 3, 3, 3}), mc);
    check("moe_dispatch KAT", r.capacity == 1 && r.selected == std::vector<int>({0, 1, 0, 0}) &&
                                  r.survived == std::vector<std::uint8_t>({1, 1, 0, 0}) && r.dropped == 2);
    // error behaviour: same exception type and text as the reference
    bool threw = false;
    try {
      matmul(nullptr, a, a);
    } catch (const std::invalid_argument& e) {
      threw = std::string(e.what()) == "matmul: inner dimensions disagree";
    }
    check("matmul shape error", threw);
  }

  // ---- finite differences of a primitive composition (SPEC acceptance #5: < 1e-3)
  {
    const int n = 3, d = 8, h = 16, V = 6;  // (h = 5 is so curved that even exact-math FD is off by 2e-3)
    auto val = [](int i) { return std::sin(0.37 * i + 0.1) * 0.5; };
    std::vector<float> xv(n * d), wv(d * h), w2v(h * V);
    for (int i = 0; i < n * d; ++i) xv[static_cast<std::size_t>(i)] = static_cast<float>(val(i));
    for (int i = 0; i < d * h; ++i) wv[static_cast<std::size_t>(i)] = static_cast<float>(val(i + 100));
    for (int i = 0; i < h * V; ++i) w2v[static_cast<std::size_t>(i)] = static_cast<float>(val(i + 200));
    const std::vector<int> tg = {1, 4, 2};
    auto f = [&](const std::vector<float>& w, bool grad, std::vector<float>* gw) {
      GradTape tape;
      GradTape* tp = grad ? &tape : nullptr;
      Tensor x = Tensor::from_data({n, d}, xv), W = Tensor::from_data({d, h}, w, true),
             W2 = Tensor::from_data({h, V}, w2v), gn = Tensor::full({h}, 1.f), bs = Tensor::zeros({h});
      Tensor y = layernorm(tp, gelu(tp, matmul(tp, x, W)), gn, bs);
      Tensor loss = softmax_cross_entropy(tp, matmul(tp, y, W2), tg);
      if (grad) {
        tape.backward_scalar(loss);
        gw->assign(W.grad(), W.grad() + W.numel());
      }
      return static_cast<double>(loss.at(0));
    };
    std::vector<float> ga;
    f(wv, true, &ga);
    double worst = 0;
    for (int i = 0; i < d * h; i += 3) {
      // fourth-order central difference (truncation O(e^4)) on the fp32 forward
      const float e = 1e-2f;
      auto at = [&](float delta) {
        std::vector<float> w = wv;
        w[static_cast<std::size_t>(i)] += delta;
        return f(w, false, nullptr);
      };
      const double fd = (8.0 * (at(e) - at(-e)) - (at(2 * e) - at(-2 * e))) / (12.0 * e);
      const double g = ga[static_cast<std::size_t>(i)];
      if (std::getenv("P2R_FD_TRACE")) std::fprintf(stderr, "fd %d %.6f %.6f\n", i, fd, g);
      worst = std::max(worst, std::fabs(fd - g) / std::max(1.0, std::fabs(g)));
    }
    put("finite_difference_max_rel_err", std::to_string(worst));
    check("finite differences < 1e-3", worst < 1e-3);
  }

  // ---- the absent controller: train_pseudo -> delink -> train_real
  ModelConfig cfg;
  cfg.d_model = 256;
  cfg.d_ff = 1024;
  cfg.n_layers_graph = 3;
  cfg.n_layers_params = 1;
  cfg.n_heads = 4;
  cfg.vocab_size = 260;
  cfg.seq_len = 128;
  if (moe) {
    cfg.moe.n_experts = 4;
    cfg.moe.n_prototypes = 1;
  }
  const int B = 4, S = 128;
  Model pseudo = build_model(cfg, 1234);
  const ParamCounts pc = count_params(cfg);
  put("params_pseudo", std::to_string(pc.total_params));
  check("scratch grad bytes", pseudo.scratch_grad_bytes() == 0);
  int nparam = 0;
  pseudo.for_each_param([&](const std::string&, const Tensor&) { ++nparam; });
  put("n_params", std::to_string(nparam));
  check("graph layers share the owned layer", &pseudo.graph_layer(0) == &pseudo.graph_layer(2));
  AdamW opt;
  opt.register_model(pseudo);
  const LrSchedule sched = LrSchedule::cosine(1e-3f, 0.1, 100);
  std::string lp = "[";
  for (int s = 0; s < steps_pseudo; ++s) lp += (s ? ", " : "") + std::to_string(train_step(pseudo, opt, sched, s, B, S));
  put("loss_pseudo", lp + "]");
  check("step count", opt.step_count() == steps_pseudo);

  // delink: the Real model's logits equal the Pseudo model's bitwise
  Model real = pseudo.delinked();
  const std::vector<int> probe = tokens_for(999, 2 * S);
  Tensor a = pseudo.forward(probe, 2, AttentionMode::Causal), b = real.forward(probe, 2, AttentionMode::Causal);
  bool bitwise = a.numel() == b.numel();
  for (std::size_t i = 0; bitwise && i < a.numel(); ++i) bitwise = a.at(i) == b.at(i);
  put("delink_bitwise", bitwise ? "true" : "false");
  check("delink bitwise", bitwise);
  check("real owns L layers", real.n_owned_layers() == cfg.n_layers_graph && !real.config().shared());
  // host edits through a parameter view reach the device (reference semantics)
  const float keep = real.owned_layer(1).ln1_gain.at(0);
  real.owned_layer(1).ln1_gain.data()[0] = keep;
  AdamW opt_real;  // moments restart for the Real stage in this controller
  opt_real.register_model(real);
  std::string lr = "[";
  for (int s = 0; s < steps_real; ++s)
    lr += (s ? ", " : "") + std::to_string(train_step(real, opt_real, sched, steps_pseudo + s, B, S));
  put("loss_real", lr + "]");
  const auto& mom = opt_real.moments();
  put("n_moments", std::to_string(mom.size()));
  put("state_bytes", std::to_string(opt_real.state_bytes()));
  put("fails", std::to_string(fails));
  std::printf("%s}\n", out.c_str());
  return fails == 0 ? 0 : 1;
}

// refdump.cpp -- drives the UNMODIFIED reference library (graphrt, built from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/) through its
// own public API and prints what it computed as one JSON object on stdout.
//
// TEST INFRASTRUCTURE: used to generate tests/golden/ fixtures (which pin the
// C restatement in oracle.c) and as the reference CPU arm of bench.py.
//
// Paths exercised:
//   --mode math      Model::prefill_math + run_sampler + Model::step_math
//                    (model.cpp:168-183; the path pipeline_test.cpp:140-158 pins)
//   --mode <run>     Session::run with RunMode <run> (pipeline.cpp:183-259)
//   --time           per-pass wall-clock of step_math (CPU baseline timing)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "graphrt/bench.hpp"
#include "graphrt/kernels.hpp"
#include "graphrt/model.hpp"
#include "graphrt/pipeline.hpp"

using namespace graphrt;

namespace {

struct Args {
  ModelConfig mc;
  std::string mode = "math";
  int prompt_len = 10;
  std::uint64_t prompt_seed = 42;
  std::vector<int> prompt;  // explicit prompt overrides prompt_seed
  int gen = 32;
  double temperature = 0.0;  // 0 => greedy
  std::uint64_t sampler_seed = 7;
  bool round_bf16 = false;
  int dump_logits = 1;  // 0 none, 1 all sampled-from passes
  bool time = false;
  int warmup = 1;
};

float round_bf16(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  std::uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  u &= 0xFFFF0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

void round_tensor(Tensor& t) {
  for (float& v : t.data()) v = round_bf16(v);
}

// Rounds the matrices (not the LN gains/biases) to bf16 in place, mirroring
// the GPU's bf16 weight storage.
void round_weights(Model& m) {
  Weights& w = m.weights();
  round_tensor(w.embedding);
  round_tensor(w.pos_table);
  for (LayerWeights& lw : w.layers) {
    round_tensor(lw.wq);
    round_tensor(lw.wk);
    round_tensor(lw.wv);
    round_tensor(lw.wo);
    round_tensor(lw.w1);
    round_tensor(lw.w2);
  }
  round_tensor(w.head);
}

void print_floats(const float* p, int n) {
  std::printf("[");
  for (int i = 0; i < n; ++i) std::printf("%s%.9g", i ? "," : "", static_cast<double>(p[i]));
  std::printf("]");
}

void print_ints(const std::vector<int>& v) {
  std::printf("[");
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%d", i ? "," : "", v[i]);
  std::printf("]");
}

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--layers") a.mc.n_layers = std::atoi(next());
    else if (k == "--d") a.mc.d_model = std::atoi(next());
    else if (k == "--heads") a.mc.n_heads = std::atoi(next());
    else if (k == "--vocab") a.mc.vocab_size = std::atoi(next());
    else if (k == "--max-seq") a.mc.max_seq_len = std::atoi(next());
    else if (k == "--seed") a.mc.seed = std::strtoull(next(), nullptr, 10);
    else if (k == "--mode") a.mode = next();
    else if (k == "--prompt-len") a.prompt_len = std::atoi(next());
    else if (k == "--prompt-seed") a.prompt_seed = std::strtoull(next(), nullptr, 10);
    else if (k == "--prompt") {
      std::string s = next();
      std::size_t pos = 0;
      while (pos < s.size()) {
        std::size_t c = s.find(',', pos);
        if (c == std::string::npos) c = s.size();
        a.prompt.push_back(std::atoi(s.substr(pos, c - pos).c_str()));
        pos = c + 1;
      }
    } else if (k == "--gen") a.gen = std::atoi(next());
    else if (k == "--temperature") a.temperature = std::atof(next());
    else if (k == "--sampler-seed") a.sampler_seed = std::strtoull(next(), nullptr, 10);
    else if (k == "--round-bf16") a.round_bf16 = true;
    else if (k == "--dump-logits") a.dump_logits = std::atoi(next());
    else if (k == "--time") a.time = true;
    else if (k == "--warmup") a.warmup = std::atoi(next());
    else {
      std::fprintf(stderr, "unknown flag %s\n", k.c_str());
      std::exit(2);
    }
  }
  if (a.prompt.empty()) a.prompt = make_prompt(a.prompt_seed, a.prompt_len, a.mc.vocab_size);
  return a;
}

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int run_math(const Args& a) {
  const double t_init0 = now_ms();
  Model model(a.mc);
  if (a.round_bf16) round_weights(model);
  const double t_init = now_ms() - t_init0;
  SampleStrategy strat =
      a.temperature > 0 ? SampleStrategy::with_temperature(a.temperature) : SampleStrategy::greedy();
  SamplerRng rng(a.sampler_seed);
  std::vector<int> tokens;
  std::vector<std::vector<float>> logits;
  std::vector<double> pass_ms;
  const int V = a.mc.vocab_size;

  const double t0 = now_ms();
  model.prefill_math(a.prompt);
  const double ttft_compute = now_ms() - t0;
  for (int i = 0; i < a.gen; ++i) {
    if (a.dump_logits) logits.emplace_back(model.logits().data().begin(), model.logits().data().end());
    const int tok = sample_token(model.logits(), strat, rng);
    tokens.push_back(tok);
    if (i + 1 < a.gen || a.time) {
      const double s0 = now_ms();
      model.step_math(tok);
      pass_ms.push_back(now_ms() - s0);
    }
  }
  std::printf("{\"mode\":\"math\",\"n_layers\":%d,\"d_model\":%d,\"n_heads\":%d,\"vocab\":%d,"
              "\"max_seq\":%d,\"seed\":%llu,\"round_bf16\":%s,\"temperature\":%.17g,"
              "\"sampler_seed\":%llu,\"prompt\":",
              a.mc.n_layers, a.mc.d_model, a.mc.n_heads, V, a.mc.max_seq_len,
              static_cast<unsigned long long>(a.mc.seed), a.round_bf16 ? "true" : "false",
              a.temperature, static_cast<unsigned long long>(a.sampler_seed));
  print_ints(a.prompt);
  std::printf(",\"tokens\":");
  print_ints(tokens);
  std::printf(",\"init_ms\":%.3f,\"prefill_ms\":%.3f,\"pass_ms\":[", t_init, ttft_compute);
  for (std::size_t i = 0; i < pass_ms.size(); ++i) std::printf("%s%.4f", i ? "," : "", pass_ms[i]);
  std::printf("]");
  if (a.dump_logits) {
    std::printf(",\"logits\":[");
    for (std::size_t i = 0; i < logits.size(); ++i) {
      if (i) std::printf(",");
      print_floats(logits[i].data(), V);
    }
    std::printf("]");
  }
  std::printf("}\n");
  return 0;
}

int run_session(const Args& a) {
  CacheConfig cc;
  CostModel cost;
  cost.jitter = JitterKind::None;
  Session session(a.mc, cc, cost);
  if (a.round_bf16) round_weights(session.model());
  GenerationRequest req;
  req.mode = mode_from_name(a.mode);
  req.prompt = a.prompt;
  req.gen_len = a.gen;
  req.strategy =
      a.temperature > 0 ? SampleStrategy::with_temperature(a.temperature) : SampleStrategy::greedy();
  req.sampler_seed = a.sampler_seed;
  GenerationResult r = session.run(req);
  std::printf("{\"mode\":\"%s\",\"prompt\":", a.mode.c_str());
  print_ints(a.prompt);
  std::printf(",\"tokens\":");
  print_ints(r.tokens);
  std::printf(",\"dispatches\":%llu,\"graph_replays\":%llu,\"captures\":%llu}\n",
              static_cast<unsigned long long>(r.counters.dispatches),
              static_cast<unsigned long long>(r.counters.graph_replays),
              static_cast<unsigned long long>(r.counters.captures));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    if (a.mode == "math") return run_math(a);
    return run_session(a);
  } catch (const Error& e) {
    std::printf("{\"error\":\"%s\",\"what\":\"%s\"}\n", errc_name(e.code()), e.what());
    return 3;
  }
}

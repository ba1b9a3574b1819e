// Compiled C++ use of the facade (include/ppoexp.hpp) — the way a reference
// maintainer would call it.  Prints "FACADE OK" and exits 0 on success.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <sys/wait.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "ppoexp.hpp"

using namespace ppoexp;

static std::vector<std::vector<double>> g_store;

static ModelParams random_params(const ModelConfig& c, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd(0.0, 0.02);
  ModelParams p;
  auto add = [&](const std::string& n, std::vector<std::size_t> shape, double fill, bool rnd) {
    std::size_t k = 1;
    for (auto s : shape) k *= s;
    std::vector<double> v(k, fill);
    if (rnd)
      for (auto& x : v) x = double(float(nd(rng)));
    g_store.push_back(std::move(v));
    p.push_back({n, shape, g_store.back().data()});
  };
  const std::size_t d = c.d_model, f = c.d_ff;
  add("tok_embed.weight", {c.vocab_size, d}, 0, true);
  add("pos_embed.weight", {c.max_seq_len, d}, 0, true);
  for (std::size_t l = 0; l < c.n_layers; ++l) {
    const std::string b = "layers." + std::to_string(l) + ".";
    add(b + "attn_norm.weight", {d}, 1, false);
    add(b + "attn_norm.bias", {d}, 0, false);
    for (auto pr : {"q_proj", "k_proj", "v_proj", "o_proj"}) add(b + "attn." + pr + ".weight", {d, d}, 0, true);
    add(b + "ffn_norm.weight", {d}, 1, false);
    add(b + "ffn_norm.bias", {d}, 0, false);
    add(b + "ffn.up_proj.weight", {d, f}, 0, true);
    add(b + "ffn.down_proj.weight", {f, d}, 0, true);
  }
  add("final_norm.weight", {d}, 1, false);
  add("final_norm.bias", {d}, 0, false);
  if (c.scalar_head) add("scalar_head.weight", {d, 1}, 0, true);
  return p;
}

static int run(Context& ctx);
static void on_segv(int) {
  void* bt[64];
  const int n = backtrace(bt, 64);
  backtrace_symbols_fd(bt, n, 2);
  _exit(139);
}
static void step(const char* m) { std::fprintf(stderr, "step: %s\n", m); std::fflush(stderr); }

static int multi_rank(int ndev);

int main(int argc, char** argv) {
  signal(SIGSEGV, on_segv);
  if (argc >= 3 && std::string(argv[1]) == "--ranks2") return multi_rank(std::atoi(argv[2]));
  g_store.reserve(1000);
  step("start");
  auto* ctxp = new Context(0);
  Context& ctx = *ctxp;
  int rc = run(ctx);
  step("run returned");
  delete ctxp;
  step("ctx destroyed");
  if (rc == 0) std::printf("FACADE OK\n");
  return rc;
}

static int run(Context& ctx) {
  ModelConfig cfg;
  cfg.vocab_size = 258;
  cfg.d_model = 64;
  cfg.n_layers = 2;
  cfg.n_heads = 4;
  cfg.d_ff = 128;
  cfg.max_seq_len = 48;
  auto params = random_params(cfg, 1);
  step("params");
  Engine engine(ctx, params, cfg, {}, PPOEXP_F32);
  step("engine");
  std::vector<GenTask> tasks(3);
  for (int i = 0; i < 3; ++i) {
    tasks[i].prompt = {1 + i, 2, 3};
    tasks[i].max_new = 8;
    tasks[i].sampling = i == 0 ? SamplingSpec::greedy_spec() : SamplingSpec::temperature_spec(1.0, 7 + i);
  }
  auto res = engine.generate_batch(tasks);
  step("generated");
  for (auto& r : res)
    if (r.tokens.empty() || r.tokens.size() != r.logprobs.size()) return 2;
  // teacher-forced scoring reproduces the generation log-probs (test_model.cpp:183-195 analog)
  TokenSeq full = tasks[0].prompt;
  full.insert(full.end(), res[0].tokens.begin(), res[0].tokens.end());
  auto lp = sequence_logprobs(engine.model(), full);
  step("scored");
  for (std::size_t t = 0; t < res[0].tokens.size(); ++t)
    if (std::fabs(lp[3 + t] - res[0].logprobs[t]) > 1e-4) return 3;
  // refit bumps the counter; a bad name set throws RefitError and leaves it
  engine.refit(params);
  if (engine.generation_counter() != 1) return 4;
  auto bad = params;
  bad.pop_back();
  try {
    engine.refit(bad);
    return 5;
  } catch (const RefitError& e) {
    if (std::string(e.what()).find("rebuild") == std::string::npos) return 6;
  }
  // experience step
  ModelConfig hc = cfg;
  hc.scalar_head = true;
  auto cparams = random_params(hc, 2);
  DeviceModel ref(ctx, params, cfg, PPOEXP_F32), critic(ctx, cparams, hc, PPOEXP_F32);
  step("models");
  ExperienceMaker xm(engine, ref, critic, nullptr, 'e');
  double st[8];
  auto batch = xm.run({{5, 6, 7}, {8, 9}}, 6, SamplingSpec::temperature_spec(1.0, 0), 11, 2, 0, nullptr, nullptr, st);
  step("experience");
  if (batch.size() != 2 || batch[0].advantages.size() != batch[0].response.size()) return 7;
  // same weights for policy and reference → KL is 0 (test_ppo.cpp:227-254 analog)
  if (std::fabs(st[0]) > 1e-9) return 8;
  step("kl ok");
  // Engine::costs / build_seconds / snapshot / options (include/aligner/engine.hpp:65-70)
  const CostBook cb = engine.costs();
  if (!(cb.get("response_generation") > 0.0) || !(cb.get("refit") > 0.0) || !(engine.build_seconds() > 0.0)) return 11;
  const auto snap = engine.model().snapshot("layers.1.ffn.up_proj.weight", cfg.d_model * cfg.d_ff);
  for (const auto& t : params)
    if (t.name == "layers.1.ffn.up_proj.weight")
      for (std::size_t i = 0; i < snap.size(); ++i)
        if (snap[i] != t.data[i]) return 12;
  if (engine.options().max_batch != 256) return 13;
  StepTiming tm;
  xm.run({{5, 6, 7}, {8, 9}}, 6, SamplingSpec::temperature_spec(1.0, 0), 11, 3, 0, nullptr, nullptr, nullptr, &tm);
  if (!(tm.rollout > 0.0) || !(tm.response_generation > 0.0) || tm.response_generation > tm.rollout) return 14;
  // LPT (src/engine.cpp:14-31): costs 5,4,3,3 over 2 workers -> {0,3}, {1,2}
  std::vector<GenTask> lt(4);
  const double cs[4] = {5, 4, 3, 3};
  for (int i = 0; i < 4; ++i) lt[i].estimated_cost = cs[i];
  const auto plan = balance(lt, 2);
  if (plan[0] != std::vector<std::size_t>{0, 3} || plan[1] != std::vector<std::size_t>{1, 2}) return 15;
  step("costs/snapshot/timing/balance");
  auto g = shaped_gae(ctx, 0.0, {-1.0}, {-1.0}, {0.5}, 0.1, 1.0, 1.0);  // r=[0]+R... V=[.5]
  step("gae");
  if (std::fabs(g.advantages[0] - (-0.5)) > 1e-12) return 9;
  try {
    DeviceModel x(ctx, params, ModelConfig{258, 30, 1, 4, 64, 16, false}, PPOEXP_F32);
    return 10;
  } catch (const ContractError&) {
  }
  step("contract");
  return 0;
}

// Two ranks (one process and one GPU each, NCCL through the library's own
// communicator): each rank runs the experience step on its shard of 4 prompts;
// the global statistics carried by the single collective must be bit-identical
// on both ranks and match one rank running all 4 prompts.
static int rank_main(int rank, int ndev, int id_fd_w, int id_fd_r, int out_fd) {
  Context ctx(rank % ndev);
  ModelConfig cfg;
  cfg.vocab_size = 258;
  cfg.d_model = 64;
  cfg.n_layers = 2;
  cfg.n_heads = 4;
  cfg.d_ff = 128;
  cfg.max_seq_len = 48;
  g_store.reserve(1000);
  auto params = random_params(cfg, 1);
  ModelConfig hc = cfg;
  hc.scalar_head = true;
  auto cparams = random_params(hc, 2);
  auto rparams = random_params(cfg, 3);
  Engine engine(ctx, params, cfg, {}, PPOEXP_F32);
  DeviceModel ref(ctx, rparams, cfg, PPOEXP_F32), critic(ctx, cparams, hc, PPOEXP_F32);
  std::vector<uint8_t> id(PPOEXP_COMM_ID_BYTES);
  if (rank == 0) {
    id = Communicator::unique_id();
    if (write(id_fd_w, id.data(), id.size()) != ssize_t(id.size())) return 20;
  } else if (read(id_fd_r, id.data(), id.size()) != ssize_t(id.size())) {
    return 21;
  }
  Communicator comm(ctx, id, rank, 2);
  ExperienceMaker xm(engine, ref, critic, nullptr, 'e');
  const std::vector<TokenSeq> all = {{5, 6, 7}, {8, 9}, {10, 11, 12, 13}, {14}};
  const std::vector<TokenSeq> mine = {all[2 * rank], all[2 * rank + 1]};
  xm.set_comm(&comm);
  double st[8];
  xm.run(mine, 6, SamplingSpec::temperature_spec(1.0, 0), 11, 2, 2 * rank, nullptr, nullptr, st);
  double one[8] = {0};
  if (rank == 0) {  // the same step on one rank over the union (gidx 0..3)
    xm.set_comm(nullptr);
    xm.run(all, 6, SamplingSpec::temperature_spec(1.0, 0), 11, 2, 0, nullptr, nullptr, one);
  }
  double msg[16];
  std::memcpy(msg, st, sizeof st);
  std::memcpy(msg + 8, one, sizeof one);
  return write(out_fd, msg, sizeof msg) == ssize_t(sizeof msg) ? 0 : 22;
}

static int multi_rank(int ndev) {
  int idp[2], outp[2][2];
  if (pipe(idp) || pipe(outp[0]) || pipe(outp[1])) return 30;
  pid_t pids[2];
  for (int r = 0; r < 2; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) _exit(rank_main(r, ndev, idp[1], idp[0], outp[r][1]));
  }
  double m[2][16];
  for (int r = 0; r < 2; ++r)
    if (read(outp[r][0], m[r], sizeof m[r]) != ssize_t(sizeof m[r])) return 31;
  for (int r = 0; r < 2; ++r) {
    int status = 0;
    waitpid(pids[r], &status, 0);
    if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) return 32;
  }
  // global stats {kl_sum, kl_count, reward_sum, n_seqs, adv_mean, adv_std}: bit-identical across ranks
  if (std::memcmp(m[0], m[1], 6 * sizeof(double)) != 0) return 33;
  if (m[0][3] != 4.0) return 34;
  for (int k = 0; k < 6; ++k)
    if (std::fabs(m[0][k] - m[0][8 + k]) > 1e-9 * (1.0 + std::fabs(m[0][8 + k]))) return 35;
  std::printf("RANKS2 OK kl_sum=%.17g adv_mean=%.17g\n", m[0][0], m[0][4]);
  return 0;
}

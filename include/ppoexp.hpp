// ppoexp.hpp — header-only C++ facade over the C ABI (ppoexp.h) that mirrors
// the reference's experience-path interfaces (/root/reference/proj/include/
// aligner/{model,engine,losses,ppo}.hpp): the same type names, argument
// meaning and exception types/messages, so a maintainer can swap the
// reference's CPU bodies for these calls.
//
//   reference                                     here
//   Engine(params, config, opts) / build_engine   ppoexp::Engine(ctx, params, config, opts)
//   Engine::refit / generate_batch / counter      same names
//   sequence_logprobs(params, tokens)             ppoexp::sequence_logprobs(model, tokens)
//   value_estimates / reward_head                 same names (scalar head = the model's own)
//   kl_penalized_rewards / gae                    same names (fp64, on the device)
//   ppo_step experience half (src/ppo.cpp:302-393) ppoexp::ExperienceMaker::run
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ppoexp.h"

namespace ppoexp {

// include/aligner/tensor.hpp:17-25, engine.hpp:19-21, ppo.hpp:22-24
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IndexError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RefitError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PpoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(ppoexp_status s) {
  if (s == PPOEXP_OK) return;
  const std::string m = ppoexp_last_error();
  switch (s) {
    case PPOEXP_ERR_CONTRACT: throw ContractError(m);
    case PPOEXP_ERR_INDEX: throw IndexError(m);
    case PPOEXP_ERR_SHAPE: throw ShapeError(m);
    case PPOEXP_ERR_REFIT: throw RefitError(m);
    case PPOEXP_ERR_PPO: throw PpoError(m);
    default: throw CudaError(m);
  }
}

using TokenSeq = std::vector<int32_t>;
constexpr int32_t kPadToken = 256;  // include/aligner/model.hpp:17
constexpr int32_t kEotToken = 257;  // include/aligner/model.hpp:18

// include/aligner/model.hpp:30-45
struct ModelConfig {
  std::size_t vocab_size = 258, d_model = 64, n_layers = 2, n_heads = 4, d_ff = 256, max_seq_len = 128;
  bool scalar_head = false;
  ppoexp_model_config c() const {
    return {int64_t(vocab_size), int64_t(d_model), int64_t(n_layers), int64_t(n_heads), int64_t(d_ff),
            int64_t(max_seq_len), scalar_head ? 1 : 0, 0};
  }
};

// One named parameter, row-major in the reference layout (ModelParams::tensors).
struct ParamView {
  std::string name;
  std::vector<std::size_t> shape;
  const double* data;  // fp64 host values (the reference's storage type)
};
using ModelParams = std::vector<ParamView>;

// include/aligner/model.hpp:75-84 (+ top_k / top_p)
struct SamplingSpec {
  bool greedy = true;
  double temperature = 1.0;
  std::uint64_t seed = 0;
  int32_t top_k = 0;
  double top_p = 1.0;
  static SamplingSpec greedy_spec() { return {}; }
  static SamplingSpec temperature_spec(double tau, std::uint64_t seed) { return {false, tau, seed, 0, 1.0}; }
};

// include/aligner/engine.hpp:23-31
struct GenTask {
  TokenSeq prompt;
  std::size_t max_new = 16;
  SamplingSpec sampling;
  double estimated_cost = 0.0;
  double cost() const { return estimated_cost > 0.0 ? estimated_cost : double(max_new); }
};

// include/aligner/model.hpp:86-89
struct GenerateResult {
  TokenSeq tokens;
  std::vector<double> logprobs;
};

class Context {
 public:
  explicit Context(int device = 0) { check(ppoexp_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) ppoexp_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ppoexp_ctx handle() const { return h_; }

 private:
  ppoexp_ctx h_ = nullptr;
};

namespace detail {
inline std::vector<ppoexp_tensor_view> views(const ModelParams& p) {
  std::vector<ppoexp_tensor_view> v;
  v.reserve(p.size());
  for (const auto& t : p) {
    ppoexp_tensor_view x{};
    x.name = t.name.c_str();
    x.rank = int32_t(t.shape.size());
    x.dtype = PPOEXP_F64;
    x.shape[0] = t.shape.empty() ? 1 : int64_t(t.shape[0]);
    x.shape[1] = t.shape.size() > 1 ? int64_t(t.shape[1]) : 0;
    x.data = t.data;
    x.where = PPOEXP_HOST;
    v.push_back(x);
  }
  return v;
}
inline std::pair<std::vector<int32_t>, std::vector<int64_t>> ragged(const std::vector<TokenSeq>& seqs) {
  std::vector<int32_t> flat;
  std::vector<int64_t> off(1, 0);
  for (const auto& s : seqs) {
    flat.insert(flat.end(), s.begin(), s.end());
    off.push_back(int64_t(flat.size()));
  }
  return {std::move(flat), std::move(off)};
}
}  // namespace detail

// A device-resident weight snapshot (Engine's deep copy, src/engine.cpp:33-48).
class DeviceModel {
 public:
  DeviceModel(Context& ctx, const ModelParams& params, const ModelConfig& config, int dtype = PPOEXP_MIXED)
      : config_(config) {
    const auto v = detail::views(params);
    const auto c = config.c();
    check(ppoexp_model_create(ctx.handle(), &c, v.data(), int64_t(v.size()), dtype, &h_));
  }
  ~DeviceModel() {
    if (h_) ppoexp_model_destroy(h_);
  }
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;
  // Engine::refit semantics (src/engine.cpp:60-90)
  void refit(const ModelParams& params) {
    const auto v = detail::views(params);
    check(ppoexp_model_refit(h_, v.data(), int64_t(v.size())));
  }
  std::uint64_t generation_counter() const {
    uint64_t g = 0;
    check(ppoexp_model_generation(h_, &g));
    return g;
  }
  // Engine::snapshot (include/aligner/engine.hpp:67): one parameter in the reference layout
  std::vector<double> snapshot(const std::string& name, std::size_t numel) const {
    std::vector<double> out(numel);
    check(ppoexp_model_snapshot(h_, name.c_str(), out.data(), int64_t(numel), PPOEXP_F64));
    return out;
  }
  const ModelConfig& config() const { return config_; }
  ppoexp_model handle() const { return h_; }

 private:
  ModelConfig config_;
  ppoexp_model h_ = nullptr;
};

// CostBook (include/aligner/timing.hpp:33-46): per-category seconds
class CostBook {
 public:
  void add(const std::string& category, double seconds) { totals_[category] += seconds; }
  double get(const std::string& category) const {
    const auto it = totals_.find(category);
    return it == totals_.end() ? 0.0 : it->second;
  }
  const std::map<std::string, double>& totals() const { return totals_; }

 private:
  std::map<std::string, double> totals_;
};

struct EngineOptions {
  std::size_t max_batch = 256;
  std::size_t page_size = 64;
  std::size_t max_total_tokens = 0;
  bool use_graphs = true;
};

// include/aligner/engine.hpp:49-92
class Engine {
 public:
  Engine(Context& ctx, const ModelParams& params, const ModelConfig& config, EngineOptions opts = {},
         int dtype = PPOEXP_MIXED)
      : model_(std::make_unique<DeviceModel>(ctx, params, config, dtype)) {
    ppoexp_engine_options o{int64_t(opts.max_batch), int64_t(opts.page_size), int64_t(opts.max_total_tokens),
                            opts.use_graphs ? 1 : 0, 0};
    check(ppoexp_engine_create(model_->handle(), &o, &h_));
  }
  ~Engine() {
    if (h_) ppoexp_engine_destroy(h_);
  }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void refit(const ModelParams& params) { model_->refit(params); }
  std::uint64_t generation_counter() const { return model_->generation_counter(); }
  // include/aligner/engine.hpp:66-68
  double build_seconds() const {
    double s = 0;
    check(ppoexp_engine_build_seconds(h_, &s));
    return s;
  }
  CostBook costs() const {
    CostBook b;
    for (const char* cat : {"response_generation", "refit"}) {
      double s = 0;
      check(ppoexp_engine_cost(h_, cat, &s));
      if (s > 0) b.add(cat, s);
    }
    return b;
  }
  EngineOptions options() const {
    ppoexp_engine_options o{};
    check(ppoexp_engine_options_get(h_, &o));
    return {std::size_t(o.max_batch), std::size_t(o.page_size), std::size_t(o.max_total_tokens), o.use_graphs != 0};
  }
  DeviceModel& model() { return *model_; }
  ppoexp_engine handle() const { return h_; }

  std::vector<GenerateResult> generate_batch(const std::vector<GenTask>& tasks) {
    std::vector<GenerateResult> out(tasks.size());
    if (tasks.empty()) return out;
    std::vector<TokenSeq> prompts;
    std::vector<int64_t> mx;
    std::vector<uint64_t> seeds;
    std::vector<ppoexp_sampling> sp;
    std::size_t stride = 1;
    for (const auto& t : tasks) {
      prompts.push_back(t.prompt);
      mx.push_back(int64_t(t.max_new));
      seeds.push_back(t.sampling.seed);
      sp.push_back({t.sampling.greedy ? 1 : 0, t.sampling.top_k, t.sampling.temperature, t.sampling.top_p});
      stride = std::max(stride, t.max_new);
    }
    auto [flat, off] = detail::ragged(prompts);
    const int64_t B = int64_t(tasks.size());
    std::vector<int32_t> toks(B * stride);
    std::vector<double> lps(B * stride);
    std::vector<int64_t> lens(B);
    check(ppoexp_engine_generate(h_, B, flat.data(), off.data(), mx.data(), sp.data(), seeds.data(), int64_t(stride),
                                 toks.data(), lps.data(), lens.data(), PPOEXP_HOST, nullptr));
    for (int64_t b = 0; b < B; ++b) {
      out[b].tokens.assign(toks.begin() + b * stride, toks.begin() + b * stride + lens[b]);
      out[b].logprobs.assign(lps.begin() + b * stride, lps.begin() + b * stride + lens[b]);
    }
    return out;
  }

 private:
  std::unique_ptr<DeviceModel> model_;
  ppoexp_engine h_ = nullptr;
};

// balance, src/engine.cpp:14-31 (LPT): task indices per worker (here: per rank)
inline std::vector<std::vector<std::size_t>> balance(const std::vector<GenTask>& tasks, std::size_t n_workers) {
  std::vector<double> costs;
  for (const auto& t : tasks) costs.push_back(t.cost());
  std::vector<int64_t> w(tasks.size());
  check(ppoexp_balance(costs.data(), int64_t(costs.size()), int64_t(n_workers), w.data()));
  std::vector<std::vector<std::size_t>> out(n_workers);
  for (std::size_t i = 0; i < tasks.size(); ++i) out[std::size_t(w[i])].push_back(i);
  return out;
}

// spin_make_pairs (src/losses.cpp:277-295): chosen = dataset response, rejected =
// the frozen reference's greedy generation (one batched device generate);
// degenerate pairs are dropped and counted.
struct SftExample {
  TokenSeq prompt, response;
};
struct PreferenceExample {
  TokenSeq prompt, chosen, rejected;
};
struct SpinPairs {
  std::vector<PreferenceExample> pairs;
  std::size_t dropped = 0;
};
class Engine;
SpinPairs spin_make_pairs(const std::vector<SftExample>& examples, Engine& reference, std::size_t max_new);

// One NCCL communicator per rank (the experience step's single collective).
class Communicator {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(PPOEXP_COMM_ID_BYTES);
    check(ppoexp_comm_unique_id(id.data()));
    return id;
  }
  Communicator(Context& ctx, const std::vector<uint8_t>& id, int rank, int world) {
    check(ppoexp_comm_create(ctx.handle(), id.data(), rank, world, &h_));
  }
  ~Communicator() {
    if (h_) ppoexp_comm_destroy(h_);
  }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  void allgather_sum(std::vector<double>& v) {
    check(ppoexp_comm_allgather_sum(h_, v.data(), int64_t(v.size()), PPOEXP_HOST));
  }
  ppoexp_comm handle() const { return h_; }

 private:
  ppoexp_comm h_ = nullptr;
};

// sequence_logprobs, include/aligner/model.hpp:104 (one sequence; batch form below)
inline std::vector<std::vector<double>> sequence_logprobs(DeviceModel& m, const std::vector<TokenSeq>& seqs) {
  auto [flat, off] = detail::ragged(seqs);
  std::vector<double> out(std::max<std::size_t>(flat.size(), 1));
  check(ppoexp_sequence_logprobs(m.handle(), int64_t(seqs.size()), flat.data(), off.data(), out.data(), PPOEXP_HOST));
  std::vector<std::vector<double>> r;
  for (std::size_t b = 0; b < seqs.size(); ++b) r.emplace_back(out.begin() + off[b], out.begin() + off[b + 1]);
  return r;
}
inline std::vector<double> sequence_logprobs(DeviceModel& m, const TokenSeq& tokens) {
  if (tokens.empty()) return {};
  return sequence_logprobs(m, std::vector<TokenSeq>{tokens})[0];
}

// frozen_response_logprob_sum (src/trainers.cpp:24-29), batched: one sum per sequence
inline std::vector<double> response_logprob_sums(DeviceModel& m, const std::vector<TokenSeq>& seqs,
                                                 const std::vector<int64_t>& response_start) {
  if (seqs.empty()) return {};
  auto [flat, off] = detail::ragged(seqs);
  std::vector<double> out(seqs.size());
  check(ppoexp_response_logprob_sums(m.handle(), int64_t(seqs.size()), flat.data(), off.data(), response_start.data(),
                                     out.data(), PPOEXP_HOST));
  return out;
}

// value_estimates, include/aligner/losses.hpp:90-92
inline std::vector<double> value_estimates(DeviceModel& critic, const TokenSeq& tokens, std::size_t response_start) {
  const int64_t off[2] = {0, int64_t(tokens.size())};
  const int64_t rs = int64_t(response_start);
  std::vector<double> out(tokens.size() > response_start ? tokens.size() - response_start : 1);
  check(ppoexp_value_estimates(critic.handle(), 1, tokens.data(), off, &rs, out.data(), PPOEXP_HOST));
  return out;
}

// reward_head, include/aligner/losses.hpp:88
inline double reward_head(DeviceModel& rm, const TokenSeq& tokens) {
  const int64_t off[2] = {0, int64_t(tokens.size())};
  double r = 0;
  check(ppoexp_reward_head(rm.handle(), 1, tokens.data(), off, &r, PPOEXP_HOST));
  return r;
}

struct GaeResult {
  std::vector<double> advantages, returns;
};

// kl_penalized_rewards + gae (include/aligner/losses.hpp:102-113) in one call
inline GaeResult shaped_gae(Context& ctx, double rm_reward, const std::vector<double>& actor_lp,
                            const std::vector<double>& ref_lp, const std::vector<double>& values, double kl_coef,
                            double gamma, double lam, std::vector<double>* shaped = nullptr) {
  const int64_t n = int64_t(actor_lp.size());
  if (ref_lp.size() != actor_lp.size() || values.size() != actor_lp.size())
    throw ContractError("kl_penalized_rewards: log-prob arrays must be nonempty and equal length");
  GaeResult r{std::vector<double>(n), std::vector<double>(n)};
  std::vector<double> sh(n);
  check(ppoexp_shape_gae(1, n, &n, &rm_reward, actor_lp.data(), ref_lp.data(), values.data(), kl_coef, gamma, lam,
                         sh.data(), r.advantages.data(), r.returns.data(), ctx.handle(), PPOEXP_HOST));
  if (shaped) *shaped = std::move(sh);
  return r;
}

// include/aligner/losses.hpp:54-63 (+ whitened advantages)
struct RolloutSeq {
  TokenSeq prompt, response;
  std::vector<double> actor_logprobs, ref_logprobs, values;
  double reward = 0.0;
  std::vector<double> advantages, returns, mask, whitened_advantages;
};
using RolloutBatch = std::vector<RolloutSeq>;

// include/aligner/ppo.hpp:27-37 (the experience-step slots; milliseconds)
struct StepTiming {
  std::size_t step = 0;
  double rollout = 0.0;
  double response_generation = 0.0;
  double logprob_calculation = 0.0;
  double critic_wait = 0.0;
};

struct PpoHyper {  // include/aligner/losses.hpp:39-50 (experience subset)
  double kl_penalty_coef = 0.003, gamma = 1.0, lam = 0.95;
};

// The experience half of ppo_step (src/ppo.cpp:302-393) + whitening.
class ExperienceMaker {
 public:
  ExperienceMaker(Engine& policy, DeviceModel& reference, DeviceModel& critic, DeviceModel* rm = nullptr,
                  int32_t scripted_target = 'z', PpoHyper hyper = {})
      : policy_(policy), reference_(reference), critic_(critic), rm_(rm), target_(scripted_target), hyper_(hyper) {}

  // The library's own NCCL collective for multi-rank runs (else a callback, or one rank).
  void set_comm(Communicator* comm) { comm_ = comm; }

  // allreduce: NULL for one rank (see ppoexp_allreduce_fn); ignored when a Communicator is set
  RolloutBatch run(const std::vector<TokenSeq>& prompts, std::size_t max_new, const SamplingSpec& sampling,
                   std::uint64_t seed, std::int64_t step_index, std::int64_t gidx0 = 0,
                   ppoexp_allreduce_fn allreduce = nullptr, void* user = nullptr, double* stats8 = nullptr,
                   StepTiming* timing = nullptr) {
    auto [flat, off] = detail::ragged(prompts);
    const int64_t B = int64_t(prompts.size()), N = int64_t(max_new);
    ppoexp_experience_request q{};
    q.reference = reference_.handle();
    q.critic = critic_.handle();
    q.rm = rm_ ? rm_->handle() : nullptr;
    q.scripted_target = target_;
    q.sampling = {sampling.greedy ? 1 : 0, sampling.top_k, sampling.temperature, sampling.top_p};
    q.seed = seed;
    q.step_index = step_index;
    q.gidx0 = gidx0;
    q.max_new = N;
    q.hyper = {hyper_.kl_penalty_coef, hyper_.gamma, hyper_.lam};
    q.allreduce = allreduce;
    q.allreduce_user = user;
    q.comm = comm_ ? comm_->handle() : nullptr;
    q.policy_engine = policy_.handle();
    std::vector<int32_t> toks(B * N);
    std::vector<int64_t> lens(B);
    std::vector<double> a(B * N), r(B * N), v(B * N), rw(B), sh(B * N), adv(B * N), ret(B * N), wh(B * N),
        st(8), tm(4);
    ppoexp_rollout_batch o{toks.data(), lens.data(), a.data(), r.data(), v.data(), rw.data(), sh.data(),
                           adv.data(), ret.data(), wh.data(), st.data(), tm.data()};
    check(ppoexp_make_experience(&q, B, flat.data(), off.data(), &o, PPOEXP_HOST));
    if (stats8) std::copy(st.begin(), st.end(), stats8);
    if (timing) {
      timing->step = std::size_t(step_index);
      timing->rollout = tm[0];
      timing->response_generation = tm[1];
      timing->logprob_calculation = tm[2];
      timing->critic_wait = tm[3];
    }
    RolloutBatch batch(B);
    for (int64_t b = 0; b < B; ++b) {
      auto& s = batch[b];
      const int64_t n = lens[b];
      auto cut = [&](const std::vector<double>& x) {
        return std::vector<double>(x.begin() + b * N, x.begin() + b * N + n);
      };
      s.prompt = prompts[b];
      s.response.assign(toks.begin() + b * N, toks.begin() + b * N + n);
      s.actor_logprobs = cut(a);
      s.ref_logprobs = cut(r);
      s.values = cut(v);
      s.reward = rw[b];
      s.advantages = cut(adv);
      s.returns = cut(ret);
      s.mask.assign(n, 1.0);
      s.whitened_advantages = cut(wh);
    }
    return batch;
  }

 private:
  Engine& policy_;
  DeviceModel& reference_;
  DeviceModel& critic_;
  DeviceModel* rm_;
  int32_t target_;
  PpoHyper hyper_;
  Communicator* comm_ = nullptr;
};

inline SpinPairs spin_make_pairs(const std::vector<SftExample>& examples, Engine& reference, std::size_t max_new) {
  std::vector<GenTask> tasks;
  for (const auto& ex : examples) {
    GenTask t;
    t.prompt = ex.prompt;
    t.max_new = max_new;
    tasks.push_back(t);  // greedy (SamplingSpec default)
  }
  const auto gens = reference.generate_batch(tasks);
  SpinPairs out;
  for (std::size_t i = 0; i < examples.size(); ++i) {
    const TokenSeq& rej = gens[i].tokens;
    if (rej.empty() || rej == examples[i].response) {
      ++out.dropped;
      continue;
    }
    out.pairs.push_back({examples[i].prompt, examples[i].response, rej});
  }
  return out;
}

}  // namespace ppoexp

// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// (/root/reference/proj/src/{tensor,model,losses,engine,layout}.cpp, compiled
// in place by oracle/Makefile into oracle/_ref/libaligner_ref.so).
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY.  Used to (1) pin the C oracle
// restatement, (2) generate tests/golden fixtures, (3) time the reference's
// own CPU path for bench.py --impl reference and the cpu_baseline leg.
// Nothing in the product path links this.
//
// Weights cross this boundary in the "flat canonical" layout documented in
// oracle/ppoexp_oracle.c (ModelParams::expected_names order,
// src/model.cpp:66-90).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "aligner/engine.hpp"
#include "aligner/losses.hpp"
#include "aligner/model.hpp"
#include "aligner/optim.hpp"
#include "aligner/rng.hpp"

using namespace aligner;

namespace {

thread_local std::string g_err;

ModelConfig make_cfg(const int64_t* c6, int32_t scalar_head) {
  ModelConfig cfg;
  cfg.vocab_size = static_cast<std::size_t>(c6[0]);
  cfg.d_model = static_cast<std::size_t>(c6[1]);
  cfg.n_layers = static_cast<std::size_t>(c6[2]);
  cfg.n_heads = static_cast<std::size_t>(c6[3]);
  cfg.d_ff = static_cast<std::size_t>(c6[4]);
  cfg.max_seq_len = static_cast<std::size_t>(c6[5]);
  cfg.scalar_head = scalar_head != 0;
  return cfg;
}

// Builds reference ModelParams from the flat canonical buffer.
ModelParams from_flat(const ModelConfig& cfg, const double* w) {
  ModelParams p;
  p.config = cfg;
  std::size_t off = 0;
  for (const auto& name : ModelParams::expected_names(cfg)) {
    const auto shape = param_shape(cfg, name);
    std::size_t n = 1;
    for (auto s : shape) n *= s;
    p.tensors.emplace(name, Tensor(shape, std::vector<double>(w + off, w + off + n)));
    off += n;
  }
  return p;
}

void to_flat(const ModelParams& p, double* w) {
  std::size_t off = 0;
  for (const auto& name : ModelParams::expected_names(p.config)) {
    const auto vals = p.at(name).values();
    std::memcpy(w + off, vals.data(), vals.size() * sizeof(double));
    off += vals.size();
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_param_count(const int64_t* c6, int32_t scalar_head) {
  const auto cfg = make_cfg(c6, scalar_head);
  int64_t n = 0;
  for (const auto& name : ModelParams::expected_names(cfg)) {
    int64_t k = 1;
    for (auto s : param_shape(cfg, name)) k *= static_cast<int64_t>(s);
    n += k;
  }
  return n;
}

// init_params, src/model.cpp:156-184
int ref_init_params(const int64_t* c6, int32_t scalar_head, uint64_t seed, double* out) {
  return guarded([&] { to_flat(init_params(make_cfg(c6, scalar_head), seed), out); });
}

uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

void ref_uniforms(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

// Engine::generate_batch (src/engine.cpp:148-182) over B ragged prompts.
// seeds[B] per task; greedy != 0 → SamplingSpec::greedy_spec().  Results are
// written [B, max_new] with out_n[B] lengths.  seconds_out gets the wall time
// of the generate_batch call alone.
int ref_generate_batch(const int64_t* c6, const double* w, const int32_t* prompts,
                       const int64_t* offsets, int64_t B, int64_t max_new, int32_t greedy,
                       double temperature, const uint64_t* seeds, int64_t n_workers,
                       int32_t* out_tokens, double* out_lps, int64_t* out_n, double* seconds_out) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    const auto params = from_flat(cfg, w);
    EngineOptions opts;
    opts.n_workers = static_cast<std::size_t>(n_workers > 0 ? n_workers : 1);
    auto engine = build_engine(params, cfg, opts);
    std::vector<GenTask> tasks(static_cast<std::size_t>(B));
    for (int64_t b = 0; b < B; ++b) {
      tasks[b].prompt.assign(prompts + offsets[b], prompts + offsets[b + 1]);
      tasks[b].max_new = static_cast<std::size_t>(max_new);
      tasks[b].sampling = greedy ? SamplingSpec::greedy_spec()
                                 : SamplingSpec::temperature_spec(temperature, seeds[b]);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const auto res = engine->generate_batch(tasks);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
    for (int64_t b = 0; b < B; ++b) {
      out_n[b] = static_cast<int64_t>(res[b].tokens.size());
      for (std::size_t i = 0; i < res[b].tokens.size(); ++i) {
        out_tokens[b * max_new + i] = res[b].tokens[i];
        out_lps[b * max_new + i] = res[b].logprobs[i];
      }
    }
  });
}

// sequence_logprobs (src/model.cpp:484-495), one sequence.
int ref_sequence_logprobs(const int64_t* c6, const double* w, const int32_t* tokens, int64_t T,
                          double* out) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    const auto lp = sequence_logprobs(from_flat(cfg, w), TokenSeq(tokens, tokens + T));
    std::memcpy(out, lp.data(), lp.size() * sizeof(double));
  });
}

// forward_hidden (src/model.cpp:249-251) → hidden [T, d]
int ref_forward_hidden(const int64_t* c6, int32_t scalar_head, const double* w,
                       const int32_t* tokens, int64_t T, double* out) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, scalar_head);
    const auto h = forward_hidden(from_flat(cfg, w), TokenSeq(tokens, tokens + T));
    std::memcpy(out, h.values().data(), h.values().size() * sizeof(double));
  });
}

// value_estimates (src/losses.cpp:117-127) with the model's own scalar head.
int ref_value_estimates(const int64_t* c6, const double* w, const int32_t* tokens, int64_t T,
                        int64_t response_start, double* out) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 1);
    const auto p = from_flat(cfg, w);
    const auto v = value_estimates(p, p.at("scalar_head.weight"), TokenSeq(tokens, tokens + T),
                                   static_cast<std::size_t>(response_start));
    std::memcpy(out, v.values().data(), v.values().size() * sizeof(double));
  });
}

// reward_head (src/losses.cpp:105-115) with the model's own scalar head.
int ref_reward_head(const int64_t* c6, const double* w, const int32_t* tokens, int64_t T,
                    double* out) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 1);
    const auto p = from_flat(cfg, w);
    *out = reward_head(p, p.at("scalar_head.weight"), TokenSeq(tokens, tokens + T)).item();
  });
}

int ref_kl_penalized_rewards(double rm, const double* a, const double* r, int64_t n, double coef,
                             double* out) {
  return guarded([&] {
    const auto v = kl_penalized_rewards(rm, std::span<const double>(a, n),
                                        std::span<const double>(r, n), coef);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

int ref_gae(const double* rw, const double* v, int64_t n, double gamma, double lam, double* adv,
            double* ret) {
  return guarded([&] {
    const auto g = gae(std::span<const double>(rw, n), std::span<const double>(v, n), gamma, lam);
    std::memcpy(adv, g.advantages.data(), n * sizeof(double));
    std::memcpy(ret, g.returns.data(), n * sizeof(double));
  });
}

// The experience part of ppo_step (src/ppo.cpp:302-393) restated over the
// reference's public functions, in-process (the critic's RPC hop is
// transport):
//   generate_batch(tasks seeded mix_seed(seed, step*1000003 + gidx)) →
//   response_logprobs under policy and reference (:282-287, :337-339) →
//   scripted reward (:109-115) or reward_head under the RM (:175-180) →
//   value_estimates under the critic (:184-188) →
//   kl_penalized_rewards + gae (:382-387); kl_sum over all tokens (:389-392).
// Outputs are [B, max_new] padded; out_n[B] lengths; rewards[B].
// phase_seconds[3] = {generation, logprob, values+reward+shaping}.
// n_workers threads: generation through Engine's WorkPool; the scoring stages
// are spread over the same number of std::threads by sequence (the
// "harness-parallel" variant of BASELINE.md §3).
int ref_experience(const int64_t* c6, const double* w_policy, const double* w_ref,
                   const double* w_critic, const double* w_rm, int32_t scripted_target,
                   const int32_t* prompts, const int64_t* offsets, int64_t B, int64_t gidx0,
                   int64_t max_new, int32_t greedy, double temperature, uint64_t seed,
                   int64_t step_index, double kl_coef, double gamma, double lam, int64_t n_workers,
                   int32_t* out_tokens, int64_t* out_n, double* out_actor_lp, double* out_ref_lp,
                   double* out_values, double* out_rewards, double* out_adv, double* out_ret,
                   double* phase_seconds) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    auto ccfg = cfg;
    ccfg.scalar_head = true;
    const auto policy = from_flat(cfg, w_policy);
    const auto refm = from_flat(cfg, w_ref);
    const auto critic = from_flat(ccfg, w_critic);
    ModelParams rm;
    if (!scripted_target) rm = from_flat(ccfg, w_rm);
    const std::size_t nw = static_cast<std::size_t>(n_workers > 0 ? n_workers : 1);

    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    EngineOptions opts;
    opts.n_workers = nw;
    auto engine = build_engine(policy, cfg, opts);
    std::vector<GenTask> tasks(static_cast<std::size_t>(B));
    for (int64_t i = 0; i < B; ++i) {
      tasks[i].prompt.assign(prompts + offsets[i], prompts + offsets[i + 1]);
      tasks[i].max_new = static_cast<std::size_t>(max_new);
      tasks[i].sampling =
          greedy ? SamplingSpec::greedy_spec()
                 : SamplingSpec::temperature_spec(
                       temperature, mix_seed(seed, static_cast<std::uint64_t>(step_index) * 1000003 +
                                                       static_cast<std::uint64_t>(gidx0 + i)));
    }
    t0 = clk::now();
    const auto gens = engine->generate_batch(tasks);
    auto t1 = clk::now();

    std::vector<TokenSeq> full(B);
    for (int64_t i = 0; i < B; ++i) {
      full[i] = tasks[i].prompt;
      full[i].insert(full[i].end(), gens[i].tokens.begin(), gens[i].tokens.end());
      out_n[i] = static_cast<int64_t>(gens[i].tokens.size());
      for (std::size_t t = 0; t < gens[i].tokens.size(); ++t)
        out_tokens[i * max_new + t] = gens[i].tokens[t];
    }
    auto par_for = [&](auto&& body) {
      std::vector<std::thread> th;
      for (std::size_t w = 0; w < nw; ++w)
        th.emplace_back([&, w] {
          for (int64_t i = static_cast<int64_t>(w); i < B; i += static_cast<int64_t>(nw)) body(i);
        });
      for (auto& x : th) x.join();
    };
    par_for([&](int64_t i) {
      const std::size_t P = tasks[i].prompt.size();
      const auto a = sequence_logprobs(policy, full[i]);
      const auto r = sequence_logprobs(refm, full[i]);
      for (std::size_t t = P; t < full[i].size(); ++t) {
        out_actor_lp[i * max_new + (t - P)] = a[t];
        out_ref_lp[i * max_new + (t - P)] = r[t];
      }
    });
    auto t2 = clk::now();
    par_for([&](int64_t i) {
      const std::size_t P = tasks[i].prompt.size();
      double R = 0.0;
      if (scripted_target) {
        for (std::size_t t = P; t < full[i].size(); ++t)
          if (full[i][t] == scripted_target) R += 1.0;
      } else {
        R = reward_head(rm, rm.at("scalar_head.weight"), full[i]).item();
      }
      out_rewards[i] = R;
      const auto v = value_estimates(critic, critic.at("scalar_head.weight"), full[i], P);
      const std::size_t n = full[i].size() - P;
      std::vector<double> vals(v.values().begin(), v.values().end());
      const auto shaped = kl_penalized_rewards(
          R, std::span<const double>(out_actor_lp + i * max_new, n),
          std::span<const double>(out_ref_lp + i * max_new, n), kl_coef);
      const auto est = gae(shaped, vals, gamma, lam);
      for (std::size_t t = 0; t < n; ++t) {
        out_values[i * max_new + t] = vals[t];
        out_adv[i * max_new + t] = est.advantages[t];
        out_ret[i * max_new + t] = est.returns[t];
      }
    });
    auto t3 = clk::now();
    if (phase_seconds) {
      phase_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      phase_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
      phase_seconds[2] = std::chrono::duration<double>(t3 - t2).count();
    }
  });
}


// ---------------------------------------------------------------- training
// The train-side steps that consume the experience, on the reference's own
// tape autodiff and AdamW (checkers for the GPU trainer).  Each runs n_steps
// optimizer steps on the same batch (the reference's AdamW state persists
// across them) and returns the loss of every step; weights in/out in the flat
// canonical layout.  adam4 = {beta1, beta2, eps, weight_decay}.

static AdamW make_adam(const double* adam4) {
  AdamW::Options o;
  o.beta1 = adam4[0];
  o.beta2 = adam4[1];
  o.eps = adam4[2];
  o.weight_decay = adam4[3];
  return AdamW(o);
}

// PPO actor update, src/ppo.cpp:395-424 (+ ppo_actor_loss, src/losses.cpp:201-214).
// tokens: prompt ++ response per sequence (ragged, offsets[B+1]); the
// response of sequence b starts at rs[b]; old_lp / adv are flat over all
// response tokens in sequence order; mask = 1 everywhere (src/ppo.cpp:385).
int ref_ppo_actor_step(const int64_t* c6, double* w, int64_t B, const int32_t* tokens, const int64_t* offsets,
                       const int64_t* rs, const double* old_lp, const double* adv, double clip_eps, double lr,
                       const double* adam4, int64_t n_steps, double* losses) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    auto params = from_flat(cfg, w);
    params.set_requires_grad_on_trainable();
    AdamW opt = make_adam(adam4);
    int64_t n_tok = 0;
    for (int64_t b = 0; b < B; ++b) n_tok += offsets[b + 1] - offsets[b] - rs[b];
    const std::vector<double> flat_old(old_lp, old_lp + n_tok), flat_adv(adv, adv + n_tok), mask(n_tok, 1.0);
    for (int64_t s = 0; s < n_steps; ++s) {
      Tape tape;
      {
        TapeScope scope(tape);
        std::vector<Tensor> rows;
        for (int64_t b = 0; b < B; ++b) {
          TokenSeq full(tokens + offsets[b], tokens + offsets[b + 1]);
          TokenSeq resp(full.begin() + rs[b], full.end());
          Tensor logits = forward_one(params, full);
          Tensor lp = log_softmax(slice_rows(logits, std::size_t(rs[b]) - 1, full.size() - 1));
          Tensor part = gather_token_logprobs(lp, resp);
          rows.push_back(reshape(part, {part.size(), 1}));
        }
        Tensor new_lp = reshape(concat_rows(rows), {std::size_t(n_tok)});
        Tensor loss = ppo_actor_loss(new_lp, flat_old, flat_adv, clip_eps, mask);
        losses[s] = loss.item();
        params.zero_grad();
        backward(loss);
      }
      opt.step(params, lr);
      params.zero_grad();
    }
    to_flat(params, w);
  });
}

// Critic update, CriticJob::handle_train (src/ppo.cpp:195-231): per sequence
// ppo_critic_loss (src/losses.cpp:216-231) over its response values, mean over
// sequences.  old_values / returns flat over the response tokens.
int ref_critic_step(const int64_t* c6, double* w, int64_t B, const int32_t* tokens, const int64_t* offsets,
                    const int64_t* rs, const double* old_values, const double* returns, double value_clip, double lr,
                    const double* adam4, int64_t n_steps, double* losses) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 1);
    auto params = from_flat(cfg, w);
    params.set_requires_grad_on_trainable();
    AdamW opt = make_adam(adam4);
    for (int64_t s = 0; s < n_steps; ++s) {
      Tape tape;
      {
        TapeScope scope(tape);
        Tensor total = Tensor::scalar(0.0);
        int64_t o = 0;
        for (int64_t b = 0; b < B; ++b) {
          TokenSeq full(tokens + offsets[b], tokens + offsets[b + 1]);
          const int64_t n = int64_t(full.size()) - rs[b];
          Tensor values = value_estimates(params, params.at("scalar_head.weight"), full, std::size_t(rs[b]));
          std::vector<double> mask(n, 1.0);
          Tensor loss = ppo_critic_loss(values, std::span<const double>(old_values + o, n),
                                        std::span<const double>(returns + o, n), value_clip, mask);
          total = add(total, loss);
          o += n;
        }
        Tensor mean_loss = mul_scalar(total, 1.0 / double(B));
        losses[s] = mean_loss.item();
        params.zero_grad();
        backward(mean_loss);
      }
      opt.step(params, lr);
      params.zero_grad();
    }
    to_flat(params, w);
  });
}

// DPO-family update (dpo_micro_loss, src/trainers.cpp:54-80; dpo_family_loss,
// src/losses.cpp:129-166): policy sums on the tape (forward_one + log_softmax +
// gather + masked sum over the response, src/trainers.cpp:17-21), frozen
// reference sums from sequence_logprobs.  Pairs: chosen b = sequence 2b,
// rejected b = sequence 2b+1.  variant: 0 dpo, 1 ipo, 2 cdpo, 3 kto.
int ref_dpo_step(const int64_t* c6, double* w_policy, const double* w_ref, int64_t n_pairs, const int32_t* tokens,
                 const int64_t* offsets, const int64_t* rs, int32_t variant, double beta, double cdpo_eps,
                 double lr, const double* adam4, int64_t n_steps, double* losses) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    auto policy = from_flat(cfg, w_policy);
    const auto refm = from_flat(cfg, w_ref);
    policy.set_requires_grad_on_trainable();
    AdamW opt = make_adam(adam4);
    DpoHyper h;
    h.beta = beta;
    h.variant = static_cast<DpoVariant>(variant);
    h.cdpo_eps = cdpo_eps;
    auto seq = [&](int64_t i) { return TokenSeq(tokens + offsets[i], tokens + offsets[i + 1]); };
    std::vector<double> rc, rr;
    for (int64_t p = 0; p < n_pairs; ++p)
      for (int k = 0; k < 2; ++k) {
        const auto full = seq(2 * p + k);
        const auto lps = sequence_logprobs(refm, full);
        double acc = 0.0;
        for (std::size_t t = std::size_t(rs[2 * p + k]); t < full.size(); ++t) acc += lps[t];
        (k ? rr : rc).push_back(acc);
      }
    for (int64_t s = 0; s < n_steps; ++s) {
      Tape tape;
      {
        TapeScope scope(tape);
        std::vector<Tensor> pc, pr;
        for (int64_t p = 0; p < n_pairs; ++p)
          for (int k = 0; k < 2; ++k) {
            const auto full = seq(2 * p + k);
            const std::size_t r0 = std::size_t(rs[2 * p + k]);
            TokenSeq inputs(full.begin(), full.end() - 1), targets(full.begin() + 1, full.end());
            std::vector<double> mask(targets.size(), 0.0);
            for (std::size_t t = r0 - 1; t < targets.size(); ++t) mask[t] = 1.0;
            Tensor lp = gather_token_logprobs(log_softmax(forward_one(policy, inputs)), targets);
            Tensor sum_t = masked_sum(lp, mask);
            (k ? pr : pc).push_back(reshape(sum_t, {1, 1}));
          }
        Tensor policy_chosen = reshape(concat_rows(pc), {std::size_t(n_pairs)});
        Tensor policy_rejected = reshape(concat_rows(pr), {std::size_t(n_pairs)});
        Tensor loss = dpo_family_loss(policy_chosen, policy_rejected, Tensor({rc.size()}, rc), Tensor({rr.size()}, rr), h);
        losses[s] = loss.item();
        policy.zero_grad();
        backward(loss);
      }
      opt.step(policy, lr);
      policy.zero_grad();
    }
    to_flat(policy, w_policy);
  });
}


// n_iters PPO iterations on the reference (ppo_step, src/ppo.cpp:302-441, with the
// critic in-process): greedy experience (ref_experience's stages), the actor
// update on the tape + AdamW (:395-424), the critic update (handle_train,
// :195-231), the engine refit (:431-432); AdamW moments persist across
// iterations (one optimizer per job).  Per iteration i: tokens / lengths /
// actor_lp / values / advantages [n_iters, B, max_new] and losses[i] =
// {actor, critic}; final weights written back.
int ref_ppo_loop(const int64_t* c6, double* w_policy, const double* w_ref, double* w_critic, int32_t scripted_target,
                 const int32_t* prompts, const int64_t* offsets, int64_t B, int64_t max_new, uint64_t seed,
                 double kl_coef, double gamma, double lam, double clip_eps, double value_clip, double lr,
                 const double* adam4, int64_t n_iters, int32_t* out_tokens, int64_t* out_n, double* out_actor_lp,
                 double* out_values, double* out_adv, double* losses) {
  return guarded([&] {
    const auto cfg = make_cfg(c6, 0);
    auto ccfg = cfg;
    ccfg.scalar_head = true;
    auto policy = from_flat(cfg, w_policy);
    const auto refm = from_flat(cfg, w_ref);
    auto critic = from_flat(ccfg, w_critic);
    policy.set_requires_grad_on_trainable();
    critic.set_requires_grad_on_trainable();
    AdamW actor_opt = make_adam(adam4), critic_opt = make_adam(adam4);
    auto engine = build_engine(policy, cfg, EngineOptions{});
    const int64_t BN = B * max_new;
    for (int64_t it = 0; it < n_iters; ++it) {
      std::vector<GenTask> tasks(B);
      for (int64_t i = 0; i < B; ++i) {
        tasks[i].prompt.assign(prompts + offsets[i], prompts + offsets[i + 1]);
        tasks[i].max_new = std::size_t(max_new);
        tasks[i].sampling = SamplingSpec::greedy_spec();
      }
      (void)seed;
      const auto gens = engine->generate_batch(tasks);
      std::vector<TokenSeq> full(B);
      std::vector<std::size_t> P(B);
      std::vector<double> flat_old, flat_adv, flat_vals, flat_ret;
      std::vector<std::vector<double>> vals_b(B), ret_b(B);
      for (int64_t i = 0; i < B; ++i) {
        P[i] = tasks[i].prompt.size();
        full[i] = tasks[i].prompt;
        full[i].insert(full[i].end(), gens[i].tokens.begin(), gens[i].tokens.end());
        const std::size_t n = gens[i].tokens.size();
        out_n[it * B + i] = int64_t(n);
        const auto a = sequence_logprobs(policy, full[i]);
        const auto r = sequence_logprobs(refm, full[i]);
        std::vector<double> al(a.begin() + P[i], a.end()), rl(r.begin() + P[i], r.end());
        double R = 0.0;
        for (std::size_t t = P[i]; t < full[i].size(); ++t) R += full[i][t] == scripted_target ? 1.0 : 0.0;
        const auto v = value_estimates(critic, critic.at("scalar_head.weight"), full[i], P[i]);
        std::vector<double> vv(v.values().begin(), v.values().end());
        const auto shaped = kl_penalized_rewards(R, al, rl, kl_coef);
        const auto est = gae(shaped, vv, gamma, lam);
        for (std::size_t t = 0; t < n; ++t) {
          out_tokens[it * BN + i * max_new + int64_t(t)] = gens[i].tokens[t];
          out_actor_lp[it * BN + i * max_new + int64_t(t)] = al[t];
          out_values[it * BN + i * max_new + int64_t(t)] = vv[t];
          out_adv[it * BN + i * max_new + int64_t(t)] = est.advantages[t];
        }
        flat_old.insert(flat_old.end(), al.begin(), al.end());
        flat_adv.insert(flat_adv.end(), est.advantages.begin(), est.advantages.end());
        vals_b[i] = vv;
        ret_b[i] = est.returns;
      }
      {  // actor update (src/ppo.cpp:395-424)
        Tape tape;
        {
          TapeScope scope(tape);
          std::vector<Tensor> rows;
          for (int64_t i = 0; i < B; ++i) {
            TokenSeq resp(full[i].begin() + P[i], full[i].end());
            Tensor logits = forward_one(policy, full[i]);
            Tensor lp = log_softmax(slice_rows(logits, P[i] - 1, full[i].size() - 1));
            Tensor part = gather_token_logprobs(lp, resp);
            rows.push_back(reshape(part, {part.size(), 1}));
          }
          Tensor new_lp = reshape(concat_rows(rows), {flat_old.size()});
          Tensor loss = ppo_actor_loss(new_lp, flat_old, flat_adv, clip_eps, std::vector<double>(flat_old.size(), 1.0));
          losses[it * 2] = loss.item();
          policy.zero_grad();
          backward(loss);
        }
        actor_opt.step(policy, lr);
        policy.zero_grad();
      }
      {  // critic update (src/ppo.cpp:195-231)
        Tape tape;
        {
          TapeScope scope(tape);
          Tensor total = Tensor::scalar(0.0);
          for (int64_t i = 0; i < B; ++i) {
            Tensor values = value_estimates(critic, critic.at("scalar_head.weight"), full[i], P[i]);
            std::vector<double> mask(values.size(), 1.0);
            total = add(total, ppo_critic_loss(values, vals_b[i], ret_b[i], value_clip, mask));
          }
          Tensor mean_loss = mul_scalar(total, 1.0 / double(B));
          losses[it * 2 + 1] = mean_loss.item();
          critic.zero_grad();
          backward(mean_loss);
        }
        critic_opt.step(critic, lr);
        critic.zero_grad();
      }
      engine->refit(policy);  // src/ppo.cpp:431-432
    }
    to_flat(policy, w_policy);
    to_flat(critic, w_critic);
  });
}

}  // extern "C"

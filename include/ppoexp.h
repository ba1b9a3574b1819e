/*
 * ppoexp.h — C ABI of the B200-native PPO experience-making path
 * (libppoexp.so, built from paper_2405_01481_b200/csrc).
 *
 * Drop-in boundary for the reference ("minialigner", /root/reference/proj).
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj).  Plain pointers and sizes only; no torch
 * or CUDA types in the signatures (streams travel as void*).
 *
 * Conventions
 *  - Every call returns a ppoexp_status; on failure the message is available
 *    from ppoexp_last_error() (thread-local).  Status codes map 1:1 onto the
 *    reference's exception types (ContractError / IndexError / ShapeError,
 *    include/aligner/tensor.hpp:17-25; RefitError, include/aligner/engine.hpp:19-21;
 *    PpoError, include/aligner/ppo.hpp:22-24) and the messages keep the
 *    reference's wording (e.g. "(rebuild required)", src/engine.cpp:64-75).
 *  - Buffers: `where` = PPOEXP_HOST means caller-owned host memory (the call
 *    does the H2D/D2H copies on the context stream and synchronises before
 *    returning); PPOEXP_DEVICE means caller-owned device memory on the
 *    context's device (the call is stream-ordered and returns without a sync).
 *  - Weights: ppoexp_tensor_view names/shapes follow ModelParams
 *    (src/model.cpp:66-115); values are row-major in the reference layout
 *    (projections [in, out], tok_embed [V, d], scalar_head [d, 1]).
 *  - Ragged token batches: tokens[] concatenated, offsets[B+1] (int64).
 *  - Per-token response outputs are padded [B, max_new] row-major with
 *    lengths[B]; float outputs are double (the reference's std::vector<double>).
 *  - No CPU fallback: if the device is missing every call fails with
 *    PPOEXP_ERR_CUDA.
 */
#ifndef PPOEXP_H_
#define PPOEXP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPOEXP_ABI_VERSION 2

/* Only the C ABI is exported from libppoexp.so (built -fvisibility=hidden). */
#if defined(__GNUC__)
#define PPOEXP_API __attribute__((visibility("default")))
#else
#define PPOEXP_API
#endif

typedef enum {
  PPOEXP_OK = 0,
  PPOEXP_ERR_CONTRACT = 1, /* aligner::ContractError */
  PPOEXP_ERR_INDEX = 2,    /* aligner::IndexError */
  PPOEXP_ERR_SHAPE = 3,    /* aligner::ShapeError */
  PPOEXP_ERR_REFIT = 4,    /* aligner::RefitError */
  PPOEXP_ERR_PPO = 5,      /* aligner::PpoError */
  PPOEXP_ERR_CUDA = 6,     /* device / driver failure */
  PPOEXP_ERR_OOM = 7       /* device allocation failure */
} ppoexp_status;

typedef enum { PPOEXP_HOST = 0, PPOEXP_DEVICE = 1 } ppoexp_where;

typedef enum {
  PPOEXP_F32 = 0,   /* parity mode: fp32 weights / KV / activations, fp32 SIMT GEMMs */
  PPOEXP_BF16 = 1,  /* perf mode: bf16 weights / KV / GEMM operands, fp32 accumulate */
  PPOEXP_F64 = 2,   /* host weight views only */
  PPOEXP_MIXED = 3  /* bf16 weights; fp32 activations and KV; tensor-core products on a two-term bf16
                       split of every activation (hi = bf16(a), lo = bf16(a - hi)), fp32 accumulate:
                       fp32-grade results on bf16-rounded weights */
} ppoexp_dtype;

typedef struct ppoexp_ctx_s* ppoexp_ctx;
typedef struct ppoexp_model_s* ppoexp_model;
typedef struct ppoexp_engine_s* ppoexp_engine;
typedef struct ppoexp_comm_s* ppoexp_comm;
typedef struct ppoexp_trainer_s* ppoexp_trainer;

/* ModelConfig, include/aligner/model.hpp:30-45 (LoRA is not on this path). */
typedef struct {
  int64_t vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len;
  int32_t scalar_head;
  int32_t reserved;
} ppoexp_model_config;

/* One named parameter (ModelParams::tensors entry, include/aligner/model.hpp:48-67). */
typedef struct {
  const char* name;
  int32_t rank;
  int32_t dtype; /* ppoexp_dtype of `data` */
  int64_t shape[2];
  const void* data;
  int32_t where; /* ppoexp_where of `data` */
  int32_t reserved;
} ppoexp_tensor_view;

/* SamplingSpec, include/aligner/model.hpp:75-84, plus the north-star top-k /
 * top-p filter (top_k = 0 and top_p >= 1 reproduce the reference sampler
 * exactly; see oracle/ppoexp_oracle.c for the convention). */
typedef struct {
  int32_t greedy;
  int32_t top_k;
  double temperature;
  double top_p;
} ppoexp_sampling;

/* ---------------------------------------------------------------- misc */
PPOEXP_API const char* ppoexp_last_error(void);
PPOEXP_API int32_t ppoexp_abi_version(void);

/* ------------------------------------------------------------- context */
/* One device + one CUDA stream + workspace.  Calls on one context are
 * serialised (Engine's shared_mutex semantics, src/engine.cpp:78, :149). */
PPOEXP_API ppoexp_status ppoexp_ctx_create(int32_t device, ppoexp_ctx* out);
PPOEXP_API ppoexp_status ppoexp_ctx_destroy(ppoexp_ctx ctx);
/* The cudaStream_t the context launches on (for event timing / interop). */
PPOEXP_API ppoexp_status ppoexp_ctx_stream(ppoexp_ctx ctx, void** stream_out);
PPOEXP_API ppoexp_status ppoexp_ctx_synchronize(ppoexp_ctx ctx);
/* Kernel-class timing (CUDA events around each launch of the named class;
 * classes: "decode_attention", "logprob_gather", "gemm", "sampler", ...).
 * enable=1 starts accumulating; query returns total ms, launches and the
 * algorithmic bytes (or flops) those launches moved. */
PPOEXP_API ppoexp_status ppoexp_ctx_profile(ppoexp_ctx ctx, int32_t enable);
/* Restrict profiling to a comma-separated list of kernel classes (NULL or ""
 * = all), so a timed region can carry events around its dominant kernel only. */
PPOEXP_API ppoexp_status ppoexp_ctx_profile_filter(ppoexp_ctx ctx, const char* classes_csv);
PPOEXP_API ppoexp_status ppoexp_ctx_profile_query(ppoexp_ctx ctx, const char* kernel_class, double* total_ms,
                                       int64_t* launches, double* algorithmic_bytes, double* flops);
/* Number of library kernel launches issued on this context so far (graph
 * replays count every kernel node). */
PPOEXP_API ppoexp_status ppoexp_ctx_launch_count(ppoexp_ctx ctx, int64_t* out);

/* --------------------------------------------------------------- model */
/* A device-resident weight snapshot.  Replaces Engine's deep copy at build
 * (build_engine / Engine::Engine, src/engine.cpp:33-58): the views are
 * copied (and cast to compute_dtype) into HBM; the caller keeps its arrays.
 * Name/shape set must equal ModelParams::expected_names(config) exactly
 * (ContractError otherwise, like param_shape, src/model.cpp:92-115). */
PPOEXP_API ppoexp_status ppoexp_model_create(ppoexp_ctx ctx, const ppoexp_model_config* config,
                                  const ppoexp_tensor_view* params, int64_t n_params,
                                  int32_t compute_dtype, ppoexp_model* out);
/* Engine::refit, src/engine.cpp:60-90: validates the whole name/shape set
 * first (RefitError "... (rebuild required)", nothing touched), then copies
 * in place (no re-allocation, captured graphs stay valid) and bumps the
 * generation counter. */
PPOEXP_API ppoexp_status ppoexp_model_refit(ppoexp_model model, const ppoexp_tensor_view* params, int64_t n_params);
/* Engine::generation_counter, include/aligner/engine.hpp:65 */
PPOEXP_API ppoexp_status ppoexp_model_generation(ppoexp_model model, uint64_t* out);
PPOEXP_API ppoexp_status ppoexp_model_config_get(ppoexp_model model, ppoexp_model_config* out);
PPOEXP_API ppoexp_status ppoexp_model_destroy(ppoexp_model model);
/* Engine::snapshot (include/aligner/engine.hpp:67): copies one parameter of
 * the device snapshot back in the reference layout (row-major, projections
 * [in, out]) into caller host memory of `dtype` (PPOEXP_F64 or PPOEXP_F32);
 * numel must equal the parameter's element count (ShapeError otherwise). */
PPOEXP_API ppoexp_status ppoexp_model_snapshot(ppoexp_model model, const char* name, void* out, int64_t numel,
                                               int32_t dtype);

/* -------------------------------------------------------------- engine */
/* The TensorRT-LLM analog (Engine, include/aligner/engine.hpp:49-92) over a
 * policy model: paged KV pool in HBM, batched prefill, CUDA-graph decode. */
typedef struct {
  int64_t max_batch;        /* sequences per generate call (0 = 256) */
  int64_t page_size;        /* KV tokens per page (0 = 64) */
  int64_t max_total_tokens; /* KV pool capacity in tokens (0 = max_batch * max_seq_len) */
  int32_t use_graphs;       /* capture the decode step in a CUDA graph (default on) */
  int32_t reserved;
} ppoexp_engine_options;

PPOEXP_API ppoexp_status ppoexp_engine_create(ppoexp_model policy, const ppoexp_engine_options* opts, ppoexp_engine* out);
PPOEXP_API ppoexp_status ppoexp_engine_destroy(ppoexp_engine engine);
/* Engine::build_seconds / costs / options (include/aligner/engine.hpp:66-68).
 * Cost categories (CostBook, include/aligner/timing.hpp:13-20): the engine
 * books "response_generation" per generate call (src/engine.cpp:179) and
 * "refit" per refit of its model (src/engine.cpp:86-89), in seconds. */
PPOEXP_API ppoexp_status ppoexp_engine_build_seconds(ppoexp_engine engine, double* out);
PPOEXP_API ppoexp_status ppoexp_engine_cost(ppoexp_engine engine, const char* category, double* seconds);
PPOEXP_API ppoexp_status ppoexp_engine_options_get(ppoexp_engine engine, ppoexp_engine_options* out);

/* balance (src/engine.cpp:14-31): longest-processing-time assignment of n
 * tasks with costs[n] to n_workers (ranks): tasks by cost descending (index
 * ascending on ties), each to the least-loaded worker (lowest index on ties).
 * out_worker[i] = the worker of task i.  Host only. */
PPOEXP_API ppoexp_status ppoexp_balance(const double* costs, int64_t n, int64_t n_workers, int64_t* out_worker);

/* Engine::generate_batch (src/engine.cpp:148-182) / generate()
 * (src/model.cpp:438-482) for B tasks at once.
 *  prompts/offsets: ragged prompts (`where` for both).
 *  max_new[B]: per-task budget (the reference caps it at max_seq_len - P).
 *  sampling[B]: per-task SamplingSpec (each GenTask carries its own,
 *    include/aligner/engine.hpp:23-31) — greedy and sampled tasks may mix.
 *  seeds[B]: per-task Rng seed (ignored when greedy).  The sampler consumes
 *    one mt19937_64 uniform per sampled token in order, exactly like the
 *    reference (src/model.cpp:445, :464); the library draws them on the host.
 *  out_tokens/out_logprobs: [B, out_stride]; out_lengths[B].  The recorded
 *    log-prob is the untempered log-softmax of the chosen token
 *    (src/model.cpp:450, :477).  Generation stops after EOT (257), which is
 *    kept (src/model.cpp:476-478).
 *  ms_out (optional): device time of the call in milliseconds. */
PPOEXP_API ppoexp_status ppoexp_engine_generate(ppoexp_engine engine, int64_t B, const int32_t* prompts,
                                     const int64_t* offsets, const int64_t* max_new,
                                     const ppoexp_sampling* sampling, const uint64_t* seeds,
                                     int64_t out_stride, int32_t* out_tokens, double* out_logprobs,
                                     int64_t* out_lengths, int32_t where, double* ms_out);

/* ----------------------------------------------------------- scoring */
/* sequence_logprobs (src/model.cpp:484-495) for B ragged sequences:
 * out (same ragged layout as tokens) gets out[start] = 0 and
 * out[t] = log p(tokens[t] | tokens[<t]).  One batched forward plus the
 * fused log-softmax+gather kernel. */
PPOEXP_API ppoexp_status ppoexp_sequence_logprobs(ppoexp_model model, int64_t B, const int32_t* tokens,
                                       const int64_t* offsets, double* out, int32_t where);
/* frozen_response_logprob_sum (src/trainers.cpp:24-29; DPO / SPIN scoring,
 * sequences laid out by build_sft_sequence, src/data.cpp:142-167): for B
 * ragged sequences, out[b] = sum_{t >= response_start[b]} log p(tokens[t] |
 * tokens[<t]), accumulated in position order.  1 <= response_start[b] < T_b. */
PPOEXP_API ppoexp_status ppoexp_response_logprob_sums(ppoexp_model model, int64_t B, const int32_t* tokens,
                                           const int64_t* offsets, const int64_t* response_start, double* out,
                                           int32_t where);
/* value_estimates (src/losses.cpp:117-127) with the model's scalar head:
 * out is ragged over responses (out_offsets[b] = sum_{i<b} (T_i - rs_i)). */
PPOEXP_API ppoexp_status ppoexp_value_estimates(ppoexp_model critic, int64_t B, const int32_t* tokens,
                                     const int64_t* offsets, const int64_t* response_start, double* out,
                                     int32_t where);
/* reward_head (src/losses.cpp:105-115) with the model's scalar head: out[B]. */
PPOEXP_API ppoexp_status ppoexp_reward_head(ppoexp_model rm, int64_t B, const int32_t* tokens, const int64_t* offsets,
                                 double* out, int32_t where);

/* ----------------------------------------------------------- shaping */
/* kl_penalized_rewards (src/losses.cpp:188-199) + gae (src/losses.cpp:168-186)
 * for B padded sequences [B, stride] with lengths[B]. */
PPOEXP_API ppoexp_status ppoexp_shape_gae(int64_t B, int64_t stride, const int64_t* lengths, const double* rm_reward,
                               const double* actor_lp, const double* ref_lp, const double* values,
                               double kl_coef, double gamma, double lam, double* out_rewards,
                               double* out_adv, double* out_ret, ppoexp_ctx ctx, int32_t where);
/* Advantage whitening (north-star; no reference counterpart).  partials
 * receives (n_tokens, sum adv, sum adv^2); the caller reduces them across
 * ranks (one NCCL all-reduce / all-gather) and hands the global triple to
 * apply: w = (adv - mean) / sqrt(var + 1e-8), population variance. */
PPOEXP_API ppoexp_status ppoexp_whiten_partials(int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                                     double* partials3, ppoexp_ctx ctx, int32_t where);
PPOEXP_API ppoexp_status ppoexp_whiten_apply(int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                                  const double* global_partials3, double* out, ppoexp_ctx ctx, int32_t where);

/* ---------------------------------------------------- experience step */
/* PpoHyper subset, include/aligner/losses.hpp:39-50 */
typedef struct {
  double kl_penalty_coef;
  double gamma;
  double lam;
} ppoexp_ppo_hyper;

/* ----------------------------------------------------------- collective */
/* One NCCL communicator per rank (one process per GPU): rank 0 creates the
 * 128-byte unique id, the caller ships it to every rank (any side channel),
 * and every rank calls ppoexp_comm_create concurrently.  NCCL is loaded at
 * run time (libnccl.so.2). */
#define PPOEXP_COMM_ID_BYTES 128
PPOEXP_API ppoexp_status ppoexp_comm_unique_id(uint8_t* out_id);
PPOEXP_API ppoexp_status ppoexp_comm_create(ppoexp_ctx ctx, const uint8_t* id, int32_t rank, int32_t world,
                                            ppoexp_comm* out);
PPOEXP_API ppoexp_status ppoexp_comm_destroy(ppoexp_comm comm);
/* buf[0..n) <- its sum over all ranks, accumulated in rank order (bit-identical
 * on every rank): one ncclAllGather + a rank-order sum on the context stream. */
PPOEXP_API ppoexp_status ppoexp_comm_allgather_sum(ppoexp_comm comm, double* buf, int64_t n, int32_t where);

/* Collective hook for the whitening partials: called on the host with a
 * device pointer to `n` doubles that must be replaced in place by their sum
 * over all ranks (stream-ordered on `stream`).  NULL = single rank. */
typedef int32_t (*ppoexp_allreduce_fn)(double* device_buf, int64_t n, void* stream, void* user);

/* The experience half of ppo_step (src/ppo.cpp:302-393) for this rank's B
 * prompts, whose global indices are gidx0 .. gidx0+B-1:
 *   (1) generate with SamplingSpec temperature(tau, mix_seed(seed,
 *       step_index*1000003 + gidx)) (src/ppo.cpp:306-316) — or greedy;
 *   (2) actor and reference log-probs over the response
 *       (response_logprobs, src/ppo.cpp:282-287, :337-341);
 *   (3) rewards: scripted (count of scripted_target in the response,
 *       src/ppo.cpp:109-115) when rm == NULL, else reward_head under rm
 *       (src/ppo.cpp:175-180); values under the critic (:184-188);
 *   (4) kl_penalized_rewards + gae (:382-387); kl/reward sums (:389-392, :438-441);
 *   (5) whitening (north-star) through `allreduce`.
 * Outputs padded [B, max_new] (where = `where`), lengths[B], rewards[B];
 * stats[8] = {kl_sum, kl_count, reward_sum, n_seqs, adv_mean, adv_std,
 * gen_ms, total_ms} (timing[4] optionally the StepTiming split): the first six are GLOBAL (summed over ranks by the same
 * single collective that carries the whitening partials — the reference's
 * kl_mean / reward_mean, src/ppo.cpp:389-392, :438-441, are kl_sum/kl_count and
 * reward_sum/n_seqs); gen_ms / total_ms are this rank's device times.
 * The collective vector is 6 doubles: {n_tokens, sum adv, sum adv^2, kl_sum,
 * reward_sum, n_seqs}. */
typedef struct {
  ppoexp_engine policy_engine;
  ppoexp_model reference; /* may equal the engine's policy model */
  ppoexp_model critic;    /* scalar_head required (PpoError otherwise, src/ppo.cpp:94-96) */
  ppoexp_model rm;        /* NULL → scripted reward */
  int32_t scripted_target;
  int32_t reserved;
  ppoexp_sampling sampling;
  uint64_t seed;
  int64_t step_index;
  int64_t gidx0;
  int64_t max_new;
  ppoexp_ppo_hyper hyper;
  ppoexp_allreduce_fn allreduce;
  void* allreduce_user;
  ppoexp_comm comm; /* non-NULL: the library's own NCCL all-gather (allreduce is then ignored) */
} ppoexp_experience_request;

typedef struct {
  int32_t* tokens;      /* [B, max_new] */
  int64_t* lengths;     /* [B] */
  double* actor_lp;     /* [B, max_new] */
  double* ref_lp;
  double* values;
  double* rewards;      /* [B] */
  double* shaped;       /* [B, max_new] KL-shaped per-token rewards */
  double* advantages;
  double* returns;
  double* whitened;
  double* stats;        /* [8] */
  double* timing;       /* [4] (optional) StepTiming (include/aligner/ppo.hpp:27-37), ms of device time:
                           {rollout, response_generation, logprob_calculation, critic_wait};
                           critic_wait = how long the critic's values (and RM reward) ran past the
                           actor/reference log-probs (they run concurrently on separate streams) */
} ppoexp_rollout_batch;

PPOEXP_API ppoexp_status ppoexp_make_experience(const ppoexp_experience_request* req, int64_t B, const int32_t* prompts,
                                     const int64_t* offsets, const ppoexp_rollout_batch* out, int32_t where);

/* ------------------------------------------------------------ train side */
/* The updates that consume the experience: a device trainer
 * per model holding fp32 master weights (initialised from `params`, the
 * reference's ModelParams), AdamW state and a recorded forward/backward.
 * After a step, ppoexp_trainer_refit copies the weights into `serving` in
 * place (Engine::refit, src/engine.cpp:60-90; generation counter + 1). */
typedef struct { /* AdamW::Options, include/aligner/optim.hpp:38-43 */
  double beta1, beta2, eps, weight_decay;
} ppoexp_adamw_options;

PPOEXP_API ppoexp_status ppoexp_trainer_create(ppoexp_ctx ctx, const ppoexp_model_config* config,
                                               const ppoexp_tensor_view* params, int64_t n_params,
                                               ppoexp_model serving, const ppoexp_adamw_options* opts,
                                               ppoexp_trainer* out);
PPOEXP_API ppoexp_status ppoexp_trainer_destroy(ppoexp_trainer trainer);
/* PPO actor update (src/ppo.cpp:395-424): B sequences prompt ++ response
 * (ragged tokens/offsets), response_start[B]; old_logprobs / advantages / mask
 * flat over the response tokens in sequence order (mask NULL = all ones);
 * ppo_actor_loss (src/losses.cpp:201-214) then AdamW at `lr`.  loss_out gets
 * the loss before the update. */
PPOEXP_API ppoexp_status ppoexp_trainer_ppo_actor_step(ppoexp_trainer trainer, int64_t B, const int32_t* tokens,
                                                       const int64_t* offsets, const int64_t* response_start,
                                                       const double* old_logprobs, const double* advantages,
                                                       const double* mask, double clip_eps, double lr,
                                                       double* loss_out, int32_t where);
/* Critic update (CriticJob::handle_train, src/ppo.cpp:195-231): per-sequence
 * ppo_critic_loss (src/losses.cpp:216-231), mean over sequences, AdamW.
 * The trainer's config must have the scalar head. */
PPOEXP_API ppoexp_status ppoexp_trainer_critic_step(ppoexp_trainer trainer, int64_t B, const int32_t* tokens,
                                                    const int64_t* offsets, const int64_t* response_start,
                                                    const double* old_values, const double* returns,
                                                    double value_clip, double lr, double* loss_out, int32_t where);
/* DPO-family update (dpo_micro_loss, src/trainers.cpp:54-80): 2*n_pairs
 * sequences in build_sft_sequence layout, chosen then rejected per pair;
 * policy sums from the trainer, frozen sums from `reference`
 * (frozen_response_logprob_sum); variant 0 dpo, 1 ipo, 2 cdpo, 3 kto
 * (dpo_family_loss, src/losses.cpp:129-166).  margin_out (optional): the
 * mean implicit-reward margin beta * mean((pc - rc) - (pr - rr)). */
PPOEXP_API ppoexp_status ppoexp_trainer_dpo_step(ppoexp_trainer trainer, ppoexp_model reference, int64_t n_pairs,
                                                 const int32_t* tokens, const int64_t* offsets,
                                                 const int64_t* response_start, int32_t variant, double beta,
                                                 double cdpo_eps, double lr, double* loss_out, double* margin_out,
                                                 int32_t where);
PPOEXP_API ppoexp_status ppoexp_trainer_refit(ppoexp_trainer trainer);
/* One master parameter in the reference layout (fp64 host buffer of numel). */
PPOEXP_API ppoexp_status ppoexp_trainer_get(ppoexp_trainer trainer, const char* name, double* out, int64_t numel);

#ifdef __cplusplus
}
#endif
#endif /* PPOEXP_H_ */

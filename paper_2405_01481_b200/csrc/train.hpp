// train.hpp — device trainer (fp32 master weights, recorded forward, backward,
// AdamW) for the PPO actor / critic updates and the DPO family (train.cu).
#pragma once

#include <string>
#include <vector>

#include "model.hpp"

namespace ppx {

struct AdamOpts {  // AdamW::Options, include/aligner/optim.hpp:38-43
  double beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.0;
};

struct Trainer {
  struct Param {
    std::string name;
    std::vector<int64_t> shape;
    int64_t numel;
    size_t off;  // float offset into W / G / M / V
  };
  struct LayerAct {
    float *x, *h1, *qkv, *att, *xm, *h2, *u, *gu, *mu1, *rs1, *mu2, *rs2;
  };
  struct Batch {
    std::vector<int64_t> off, rs, seq_of;
    std::vector<int32_t> tok, idx, tgt;
    int64_t R = 0;
    int32_t *idx_d = nullptr, *tgt_d = nullptr;
  };

  Ctx* c;
  ppoexp_model_config cfg;
  Model* model;  // serving snapshot refreshed by refit() (may be null)
  AdamOpts opts;
  int64_t t = 0;  // optimizer steps taken
  std::vector<Param> params;
  size_t total = 0;
  DeviceBuffer W, G, Mo, Vo;
  void* blas = nullptr;
  // recorded forward
  Packed pk;
  int64_t rows = 0, pstride = 0;
  float *act = nullptr, *probs = nullptr;

  Trainer(Ctx* ctx, const ppoexp_model_config& cfg, const ppoexp_tensor_view* views, int64_t n, Model* target,
          const AdamOpts& o);
  ~Trainer();
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  const Param& param(const std::string& name) const;
  float* w(const std::string& n);
  float* g(const std::string& n);
  void mm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B, int64_t ldb,
          float beta, float* C, int64_t ldc, float alpha = 1.f);
  void mm_batched(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int64_t sa,
                  const float* B, int64_t ldb, int64_t sb, float beta, float* C, int64_t ldc, int64_t sc, int64_t batch,
                  float alpha = 1.f);
  size_t layer_floats() const;
  LayerAct layer_act(int64_t l);
  float* hf();

  void forward(const Packed& p);
  void lm_logprobs(const int32_t* idx, const int32_t* tgt, int64_t R, double* lp);
  void lm_backward(const int32_t* idx, const int32_t* tgt, int64_t R, const double* dlp, float* dhf);
  void values(const int32_t* idx, int64_t R, double* v);
  void value_backward(const int32_t* idx, int64_t R, const double* dv, float* dhf);
  void backward(float* dhf);
  void zero_grad();
  void adamw_step(double lr);
  void refit();
  void get(const std::string& name, double* out, int64_t numel);

  Batch prepare(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs, int where);
  std::vector<double> to_host_d(const double* d, int64_t n);
  double* to_dev_d(const std::vector<double>& h, const char* name);
  void backprop_lm(const Batch& bt, const std::vector<double>& dlp);
  double ppo_actor_step(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                        const double* old_lp, const double* adv, const double* mask, double clip_eps, double lr,
                        int where);
  double critic_step(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                     const double* old_values, const double* returns, double value_clip, double lr, int where);
  double dpo_step(int64_t n_pairs, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                  const std::vector<double>& ref_sums, int variant, double beta, double cdpo_eps, double lr, int where,
                  double* margin_out);
};

}  // namespace ppx

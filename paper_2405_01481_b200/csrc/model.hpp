// model.hpp — device-resident model snapshot + batched forward / scoring.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "../../include/ppoexp.h"
#include "kernels.hpp"

namespace ppx {

struct Layer {
  void *wqkv, *wo, *wup, *wdown;  // T: [3d,d], [d,d], [f,d], [d,f] (K-major, i.e. W^T of the reference)
  float *ln1w, *ln1b, *ln2w, *ln2b;
};

struct Model {
  Ctx* ctx = nullptr;
  ppoexp_model_config cfg{};
  int dtype = PPOEXP_BF16;
  uint64_t generation = 0;
  DeviceBuffer wbuf;  // all T weights, contiguous
  DeviceBuffer fbuf;  // fp32 LayerNorm params + scalar head
  void *tok = nullptr, *pos = nullptr;  // T [V,d], [S,d]
  std::vector<Layer> layers;
  float *lnfw = nullptr, *lnfb = nullptr, *head = nullptr;
  int64_t vpad = 0;  // padded logits row stride
  double build_seconds = 0.0;  // host wall time of the deep copy at build (Engine::build_seconds)
  double refit_seconds = 0.0;  // CostBook "refit" (src/engine.cpp:86-89), device time of every refit

  int64_t d() const { return cfg.d_model; }
  size_t tsize() const { return dtype == PPOEXP_F32 ? 4 : 2; }  // weight element
  size_t asize() const { return dtype == PPOEXP_BF16 ? 2 : 4; }  // activation / KV element
  int wdt() const { return dtype == PPOEXP_F32 ? PPOEXP_F32 : PPOEXP_BF16; }  // weight storage dtype
  bool mixed() const { return dtype == PPOEXP_MIXED; }
  int64_t dh() const { return cfg.d_model / cfg.n_heads; }

  // expected_names / param_shape, src/model.cpp:66-115
  static std::vector<std::pair<std::string, std::vector<int64_t>>> expected(const ppoexp_model_config& c);
  void allocate();
  // Validate names/shapes (err = RefitError or ContractError) then copy.
  void load(const ppoexp_tensor_view* v, int64_t n, bool refit);
  // Engine::snapshot: one parameter back in the reference layout (host, f64 or f32)
  void snapshot(const std::string& name, void* out, int64_t numel, int dtype);
};

// A ragged batch packed row-major on the device.
struct Packed {
  int64_t B = 0, M = 0, max_len = 0;
  std::vector<int64_t> offsets;  // host [B+1]
  int64_t* offsets_d = nullptr;
  int32_t* tokens_d = nullptr;
  int32_t* positions_d = nullptr;
  int32_t* seq_of_row_d = nullptr;
};
// Uploads offsets / positions / seq_of_row (tokens_d must already be packed).
void pack_metadata(Ctx& c, Packed& p, const std::string& tag);

// Residual stream after all layers, x[M, d] (fp32) in workspace "fwd.x".
// When kv != nullptr the K/V rows are also scattered into the paged pool.
struct KvTarget {
  const int32_t* block_table;
  KvGeom geom;
  void* pool;
};
float* forward_layers(Model& m, const Packed& p, const KvTarget* kv);

// GEMM dispatcher (tcgen05 for bf16 dense shapes, SIMT otherwise).
template <class T>
void gemm(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K, Epi epi,
          void* C, int64_t ldc);

// lp for R gathered rows: out[out_index[r]] = log p(target[r] | row gather[r]).
void score_logprobs(Model& m, const Packed& p, const float* x, const int32_t* gather, const int32_t* target,
                    const int64_t* out_index, int64_t R, double* out);
// head values for R gathered rows: out[out_index[r]] = LN_f(x[gather[r]]) · head.
void score_head(Model& m, const float* x, const int32_t* gather, const int64_t* out_index, int64_t R, double* out);

void launch_scatter_f32_f64(Ctx& c, const float* src, const int64_t* index, int64_t n, double* dst);
void launch_response_meta(Ctx& c, int64_t B, const int64_t* offsets_full, const int64_t* prompt_len,
                          const int64_t* resp_len, int64_t stride, const int32_t* tokens_full, int32_t* gather,
                          int32_t* target, int64_t* out_index, const int64_t* resp_offsets);
void launch_concat_pack(Ctx& c, int64_t B, const int32_t* prompts, const int64_t* p_offsets, const int32_t* gen,
                        int64_t gstride, const int64_t* gen_len, const int64_t* full_offsets, int32_t* full);

}  // namespace ppx

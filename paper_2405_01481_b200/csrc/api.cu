// api.cu — the extern "C" boundary (include/ppoexp.h).  Exceptions from the
// runtime become status codes + a thread-local message.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/ppoexp_testing.h"
#include <chrono>
#include <numeric>

#include "comm.hpp"
#include "engine.hpp"
#include "train.hpp"

using namespace ppx;

struct ppoexp_ctx_s {
  std::unique_ptr<Ctx> c;
};
struct ppoexp_model_s {
  Model m;
};
struct ppoexp_engine_s {
  std::unique_ptr<Engine> e;
};
struct ppoexp_comm_s {
  std::unique_ptr<Comm> c;
};
struct ppoexp_trainer_s {
  std::unique_ptr<Trainer> t;
};

namespace {
thread_local std::string g_err;

template <class F>
ppoexp_status guard(F&& f) {
  try {
    f();
    return PPOEXP_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<ppoexp_status>(e.code);
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return PPOEXP_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PPOEXP_ERR_CUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw ContractError(std::string(what) + " must not be null");
}

template <class T>
std::vector<T> to_host(Ctx& c, const T* p, int64_t n, int where) {
  std::vector<T> v(std::max<int64_t>(n, 0));
  if (n <= 0) return v;
  if (where == PPOEXP_HOST)
    std::memcpy(v.data(), p, n * sizeof(T));
  else {
    PPOEXP_CUDA(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
    PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
  }
  return v;
}

template <class T>
T* upload(Ctx& c, const std::string& name, const std::vector<T>& v) {
  T* d = static_cast<T*>(c.workspace(name, std::max<size_t>(v.size(), 1) * sizeof(T)));
  if (!v.empty()) {
    void* h = c.pinned_staging(v.size() * sizeof(T));
    std::memcpy(h, v.data(), v.size() * sizeof(T));
    PPOEXP_CUDA(cudaMemcpyAsync(d, h, v.size() * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
  }
  return d;
}

void check_offsets(const std::vector<int64_t>& off, int64_t B) {
  if (off.empty() || off[0] != 0) throw ContractError("offsets[0] must be 0");
  for (int64_t b = 0; b < B; ++b)
    if (off[b + 1] < off[b]) throw ContractError("offsets must be non-decreasing");
}

// packs caller tokens into the device workspace and uploads the metadata
Packed pack_tokens(Ctx& c, const int32_t* tokens, const std::vector<int64_t>& off, int where, const std::string& tag) {
  Packed p;
  p.offsets = off;
  const int64_t M = off.back();
  p.tokens_d = static_cast<int32_t*>(c.workspace(tag + ".tokens", std::max<int64_t>(M, 1) * 4));
  copy_in(c, p.tokens_d, tokens, M * 4, where);
  pack_metadata(c, p, tag);
  return p;
}

__global__ void seq_meta_kernel(int64_t B, const int64_t* offs, const int32_t* tokens, int32_t* gather,
                                int32_t* target, int64_t* out_index) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  const int64_t o = offs[b], n = offs[b + 1] - o, co = o - b;  // compact rows skip each sequence's last row
  for (int64_t t = threadIdx.x; t + 1 < n; t += blockDim.x) {
    gather[co + t] = int32_t(o + t);
    target[co + t] = tokens[o + t + 1];
    out_index[co + t] = o + t + 1;
  }
}

// response rows of sequence b: positions t in [rs_b, T_b), compact row r = roff[b] + t - rs_b
// predicts tokens[o + t] from the hidden state of row o + t - 1
__global__ void resp_meta_kernel(int64_t B, const int64_t* offs, const int64_t* rs, const int64_t* roff,
                                 const int32_t* tokens, int32_t* gather, int32_t* target, int64_t* out_index) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  const int64_t o = offs[b], n = offs[b + 1] - o, s0 = rs[b], r0 = roff[b];
  for (int64_t t = s0 + threadIdx.x; t < n; t += blockDim.x) {
    gather[r0 + t - s0] = int32_t(o + t - 1);
    target[r0 + t - s0] = tokens[o + t];
    out_index[r0 + t - s0] = r0 + t - s0;
  }
}

// out[b] = sum of lp over sequence b's response rows, in position order
// (frozen_response_logprob_sum's accumulation order, src/trainers.cpp:24-29)
__global__ void seg_sum_kernel(int64_t B, const int64_t* roff, const double* lp, double* out) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= B) return;
  double acc = 0.0;
  for (int64_t r = roff[b]; r < roff[b + 1]; ++r) acc += lp[r];
  out[b] = acc;
}

__global__ void last_content_kernel(int64_t B, const int64_t* offs, const int32_t* tokens, int32_t* gather,
                                    int64_t* out_index) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= B) return;
  int64_t last = -1;
  for (int64_t i = offs[b + 1]; i-- > offs[b];)
    if (tokens[i] != kPadToken) {
      last = i;
      break;
    }
  gather[b] = int32_t(last);
  out_index[b] = b;
}

void check_same_ctx(Model& a, Model& b) {
  if (a.ctx != b.ctx) throw ContractError("models must share one context");
}

}  // namespace

extern "C" {

const char* ppoexp_last_error(void) { return g_err.c_str(); }
int32_t ppoexp_abi_version(void) { return PPOEXP_ABI_VERSION; }

ppoexp_status ppoexp_ctx_create(int32_t device, ppoexp_ctx* out) {
  return guard([&] {
    need(out, "out");
    auto h = std::make_unique<ppoexp_ctx_s>();
    h->c = std::make_unique<Ctx>(device);
    *out = h.release();
  });
}

ppoexp_status ppoexp_ctx_destroy(ppoexp_ctx ctx) {
  return guard([&] { delete ctx; });
}

ppoexp_status ppoexp_ctx_stream(ppoexp_ctx ctx, void** s) {
  return guard([&] {
    need(ctx, "ctx");
    *s = ctx->c->stream;
  });
}

ppoexp_status ppoexp_ctx_synchronize(ppoexp_ctx ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->sync();
  });
}

ppoexp_status ppoexp_ctx_profile(ppoexp_ctx ctx, int32_t enable) {
  return guard([&] {
    need(ctx, "ctx");
    std::lock_guard<std::recursive_mutex> lk(ctx->c->mu);
    ctx->c->harvest();
    ctx->c->profiling = enable != 0;
    if (enable) ctx->c->stats.clear();
  });
}

ppoexp_status ppoexp_ctx_profile_filter(ppoexp_ctx ctx, const char* csv) {
  return guard([&] {
    need(ctx, "ctx");
    std::lock_guard<std::recursive_mutex> lk(ctx->c->mu);
    ctx->c->profile_filter.clear();
    if (!csv) return;
    std::string s(csv), item;
    size_t i = 0;
    while (i <= s.size()) {
      const size_t j = s.find(',', i);
      item = s.substr(i, j == std::string::npos ? std::string::npos : j - i);
      if (!item.empty()) ctx->c->profile_filter.insert(item);
      if (j == std::string::npos) break;
      i = j + 1;
    }
  });
}

ppoexp_status ppoexp_ctx_profile_query(ppoexp_ctx ctx, const char* cls, double* total_ms, int64_t* launches,
                                       double* bytes, double* flops) {
  return guard([&] {
    need(ctx, "ctx");
    std::lock_guard<std::recursive_mutex> lk(ctx->c->mu);
    ctx->c->sync();
    ctx->c->harvest();
    const auto it = ctx->c->stats.find(cls ? cls : "");
    const ClassStats s = it == ctx->c->stats.end() ? ClassStats{} : it->second;
    if (total_ms) *total_ms = s.ms;
    if (launches) *launches = s.launches;
    if (bytes) *bytes = s.bytes;
    if (flops) *flops = s.flops;
  });
}

ppoexp_status ppoexp_ctx_launch_count(ppoexp_ctx ctx, int64_t* out) {
  return guard([&] {
    need(ctx, "ctx");
    *out = ctx->c->launches;
  });
}

// ------------------------------------------------------------------ model
ppoexp_status ppoexp_model_create(ppoexp_ctx ctx, const ppoexp_model_config* cfg, const ppoexp_tensor_view* params,
                                  int64_t n, int32_t dtype, ppoexp_model* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(cfg, "config");
    need(out, "out");
    // ModelConfig::validate, src/model.cpp:32-44
    if (cfg->vocab_size <= 0 || cfg->d_model <= 0 || cfg->n_layers <= 0 || cfg->n_heads <= 0 || cfg->d_ff <= 0 ||
        cfg->max_seq_len <= 0)
      throw ContractError("model config: all dimensions must be positive");
    if (cfg->d_model % cfg->n_heads != 0)
      throw ContractError("model config: d_model " + std::to_string(cfg->d_model) + " not divisible by n_heads " +
                          std::to_string(cfg->n_heads));
    const int64_t dh = cfg->d_model / cfg->n_heads;
    if (dh != 16 && dh != 32 && dh != 64 && dh != 128)
      throw ContractError("model config: head_dim " + std::to_string(dh) + " unsupported (16/32/64/128)");
    if (cfg->d_model % 8 || cfg->d_ff % 8) throw ContractError("model config: d_model and d_ff must be multiples of 8");
    if (dtype != PPOEXP_F32 && dtype != PPOEXP_BF16 && dtype != PPOEXP_MIXED)
      throw ContractError("compute dtype must be F32, BF16 or MIXED");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    auto h = std::make_unique<ppoexp_model_s>();
    h->m.ctx = &c;
    h->m.cfg = *cfg;
    h->m.dtype = dtype;
    const auto t0 = std::chrono::steady_clock::now();
    h->m.allocate();
    h->m.load(params, n, false);
    h->m.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
  });
}

ppoexp_status ppoexp_model_refit(ppoexp_model model, const ppoexp_tensor_view* params, int64_t n) {
  return guard([&] {
    need(model, "model");
    Ctx& c = *model->m.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    cudaEvent_t a, b;
    PPOEXP_CUDA(cudaEventCreate(&a));
    PPOEXP_CUDA(cudaEventCreate(&b));
    PPOEXP_CUDA(cudaEventRecord(a, c.stream));
    model->m.load(params, n, true);
    PPOEXP_CUDA(cudaEventRecord(b, c.stream));
    PPOEXP_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    c.stats["refit"].ms += ms;  // CostBook "refit" category, include/aligner/timing.hpp:18
    c.stats["refit"].launches += 1;
    model->m.refit_seconds += ms / 1000.0;
    ++model->m.generation;
  });
}

ppoexp_status ppoexp_model_generation(ppoexp_model model, uint64_t* out) {
  return guard([&] {
    need(model, "model");
    *out = model->m.generation;
  });
}

ppoexp_status ppoexp_model_config_get(ppoexp_model model, ppoexp_model_config* out) {
  return guard([&] {
    need(model, "model");
    *out = model->m.cfg;
  });
}

ppoexp_status ppoexp_model_snapshot(ppoexp_model model, const char* name, void* out, int64_t numel, int32_t dtype) {
  return guard([&] {
    need(model, "model");
    need(name, "name");
    need(out, "out");
    std::lock_guard<std::recursive_mutex> lk(model->m.ctx->mu);
    DeviceGuard g(model->m.ctx->device);
    model->m.snapshot(name, out, numel, dtype);
  });
}

ppoexp_status ppoexp_model_destroy(ppoexp_model model) {
  return guard([&] {
    if (!model) return;
    std::lock_guard<std::recursive_mutex> lk(model->m.ctx->mu);
    DeviceGuard g(model->m.ctx->device, true);
    cudaStreamSynchronize(model->m.ctx->stream);
    delete model;
  });
}

// ------------------------------------------------------------------ engine
ppoexp_status ppoexp_engine_create(ppoexp_model policy, const ppoexp_engine_options* opts, ppoexp_engine* out) {
  return guard([&] {
    need(policy, "policy");
    need(out, "out");
    std::lock_guard<std::recursive_mutex> lk(policy->m.ctx->mu);
    auto h = std::make_unique<ppoexp_engine_s>();
    const auto t0 = std::chrono::steady_clock::now();
    h->e = std::make_unique<Engine>(&policy->m, opts);
    h->e->build_seconds =
        policy->m.build_seconds + std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
  });
}

ppoexp_status ppoexp_engine_destroy(ppoexp_engine engine) {
  return guard([&] {
    if (!engine) return;
    std::lock_guard<std::recursive_mutex> lk(engine->e->c->mu);
    delete engine;
  });
}

ppoexp_status ppoexp_engine_build_seconds(ppoexp_engine engine, double* out) {
  return guard([&] {
    need(engine, "engine");
    need(out, "out");
    *out = engine->e->build_seconds;
  });
}

ppoexp_status ppoexp_engine_cost(ppoexp_engine engine, const char* category, double* seconds) {
  return guard([&] {
    need(engine, "engine");
    need(category, "category");
    need(seconds, "seconds");
    const std::string cat = category;
    // CostBook::get returns 0 for categories never booked (include/aligner/timing.hpp:37-40)
    *seconds = cat == "response_generation" ? engine->e->gen_seconds
               : cat == "refit"             ? engine->e->m->refit_seconds
                                            : 0.0;
  });
}

ppoexp_status ppoexp_engine_options_get(ppoexp_engine engine, ppoexp_engine_options* out) {
  return guard([&] {
    need(engine, "engine");
    need(out, "out");
    *out = engine->e->opts;
  });
}

ppoexp_status ppoexp_balance(const double* costs, int64_t n, int64_t n_workers, int64_t* out_worker) {
  return guard([&] {
    if (n_workers <= 0) throw ContractError("balance: n_workers must be positive");
    if (n <= 0) return;
    need(costs, "costs");
    need(out_worker, "out_worker");
    // src/engine.cpp:14-31: stable sort by cost descending, least-loaded worker, lowest index on ties
    std::vector<int64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return costs[a] > costs[b]; });
    std::vector<double> load(n_workers, 0.0);
    for (int64_t i : order) {
      int64_t w = 0;
      for (int64_t k = 1; k < n_workers; ++k)
        if (load[k] < load[w]) w = k;
      load[w] += costs[i];
      out_worker[i] = w;
    }
  });
}

ppoexp_status ppoexp_comm_unique_id(uint8_t* out_id) {
  return guard([&] {
    need(out_id, "out_id");
    comm_unique_id(out_id);
  });
}

ppoexp_status ppoexp_comm_create(ppoexp_ctx ctx, const uint8_t* id, int32_t rank, int32_t world, ppoexp_comm* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(id, "id");
    need(out, "out");
    auto h = std::make_unique<ppoexp_comm_s>();
    h->c = std::make_unique<Comm>(ctx->c.get(), id, rank, world);
    *out = h.release();
  });
}

ppoexp_status ppoexp_comm_destroy(ppoexp_comm comm) {
  return guard([&] { delete comm; });
}

ppoexp_status ppoexp_comm_allgather_sum(ppoexp_comm comm, double* buf, int64_t n, int32_t where) {
  return guard([&] {
    need(comm, "comm");
    if (n <= 0) return;
    need(buf, "buf");
    Ctx& c = *comm->c->ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    double* d = buf;
    if (where == PPOEXP_HOST) {
      d = static_cast<double*>(c.workspace("comm.host", n * 8));
      copy_in(c, d, buf, n * 8, PPOEXP_HOST);
    }
    comm->c->allgather_sum(d, n);
    if (where == PPOEXP_HOST) {
      copy_out(c, buf, d, n * 8, PPOEXP_HOST);
      c.sync();
    }
  });
}

ppoexp_status ppoexp_engine_generate(ppoexp_engine engine, int64_t B, const int32_t* prompts, const int64_t* offsets,
                                     const int64_t* max_new, const ppoexp_sampling* sampling, const uint64_t* seeds,
                                     int64_t out_stride, int32_t* out_tokens, double* out_logprobs,
                                     int64_t* out_lengths, int32_t where, double* ms_out) {
  return guard([&] {
    need(engine, "engine");
    if (B > 0) {
      need(prompts, "prompts");
      need(offsets, "offsets");
      need(max_new, "max_new");
      need(out_tokens, "out_tokens");
      need(out_logprobs, "out_logprobs");
      need(out_lengths, "out_lengths");
    }
    engine->e->generate(B, prompts, offsets, max_new, sampling, seeds, out_stride, out_tokens, out_logprobs,
                        out_lengths, where, ms_out);
  });
}

// ------------------------------------------------------------------ scoring
ppoexp_status ppoexp_sequence_logprobs(ppoexp_model model, int64_t B, const int32_t* tokens, const int64_t* offsets,
                                       double* out, int32_t where) {
  return guard([&] {
    need(model, "model");
    if (B <= 0) return;
    Model& m = model->m;
    Ctx& c = *m.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const auto off = to_host(c, offsets, B + 1, where);
    check_offsets(off, B);
    const int64_t M = off[B];
    check_tokens(c, tokens, M, m.cfg.vocab_size, where, "sequence_logprobs");
    Packed p = pack_tokens(c, tokens, off, where, "lp");
    double* out_d = static_cast<double*>(c.workspace("lp.out", std::max<int64_t>(M, 1) * 8));
    PPOEXP_CUDA(cudaMemsetAsync(out_d, 0, M * 8, c.stream));  // out[start] = 0 (src/model.cpp:487)
    const int64_t R = M - B;
    int32_t* gather = static_cast<int32_t*>(c.workspace("lp.gather", std::max<int64_t>(R, 1) * 4));
    int32_t* target = static_cast<int32_t*>(c.workspace("lp.target", std::max<int64_t>(R, 1) * 4));
    int64_t* oidx = static_cast<int64_t*>(c.workspace("lp.oidx", std::max<int64_t>(R, 1) * 8));
    c.launch("meta", 0, 0, [&] { launch_kernel(c, seq_meta_kernel, dim3(B), dim3(128), 0, 1, B, p.offsets_d, p.tokens_d, gather, target, oidx); });
    // empty sequences contribute nothing (the reference returns {}, src/model.cpp:485)
    Packed q = p;
    if (R > 0) {
      float* x = forward_layers(m, q, nullptr);
      score_logprobs(m, q, x, gather, target, oidx, R, out_d);
    }
    copy_out(c, out, out_d, M * 8, where);
    if (where == PPOEXP_HOST) c.sync();
  });
}

ppoexp_status ppoexp_response_logprob_sums(ppoexp_model model, int64_t B, const int32_t* tokens,
                                           const int64_t* offsets, const int64_t* response_start, double* out,
                                           int32_t where) {
  return guard([&] {
    need(model, "model");
    if (B <= 0) return;
    Model& m = model->m;
    Ctx& c = *m.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const auto off = to_host(c, offsets, B + 1, where);
    const auto rs = to_host(c, response_start, B, where);
    check_offsets(off, B);
    std::vector<int64_t> roff(B + 1, 0);
    for (int64_t b = 0; b < B; ++b) {
      const int64_t T = off[b + 1] - off[b];
      if (rs[b] < 1 || rs[b] >= T)  // build_sft_sequence: nonempty prompt and response (src/data.cpp:144-146)
        throw ContractError("response_logprob_sums: response_start must leave a nonempty prompt and response");
      roff[b + 1] = roff[b] + T - rs[b];
    }
    const int64_t R = roff[B];
    check_tokens(c, tokens, off[B], m.cfg.vocab_size, where, "scoring");
    Packed p = pack_tokens(c, tokens, off, where, "rsum");
    int64_t* rs_d = upload(c, "rsum.rs", rs);
    int64_t* roff_d = upload(c, "rsum.roff", roff);
    int32_t* gather = static_cast<int32_t*>(c.workspace("rsum.gather", R * 4));
    int32_t* target = static_cast<int32_t*>(c.workspace("rsum.target", R * 4));
    int64_t* oidx = static_cast<int64_t*>(c.workspace("rsum.oidx", R * 8));
    double* lp = static_cast<double*>(c.workspace("rsum.lp", R * 8));
    double* out_d = static_cast<double*>(c.workspace("rsum.out", B * 8));
    c.launch("meta", 0, 0, [&] {
      launch_kernel(c, resp_meta_kernel, dim3(B), dim3(128), 0, 1, B, p.offsets_d, rs_d, roff_d, p.tokens_d, gather,
                    target, oidx);
    });
    float* x = forward_layers(m, p, nullptr);
    score_logprobs(m, p, x, gather, target, oidx, R, lp);
    c.launch("meta", 0, 0, [&] {
      launch_kernel(c, seg_sum_kernel, dim3(ceil_div(B, 128)), dim3(128), 0, 1, B, roff_d, static_cast<const double*>(lp),
                    out_d);
    });
    copy_out(c, out, out_d, B * 8, where);
    if (where == PPOEXP_HOST) c.sync();
  });
}

ppoexp_status ppoexp_value_estimates(ppoexp_model critic, int64_t B, const int32_t* tokens, const int64_t* offsets,
                                     const int64_t* response_start, double* out, int32_t where) {
  return guard([&] {
    need(critic, "critic");
    if (B <= 0) return;
    Model& m = critic->m;
    Ctx& c = *m.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (!m.cfg.scalar_head) throw ShapeError("reward_head: head must be [d_model x 1], got none");
    const auto off = to_host(c, offsets, B + 1, where);
    const auto rs = to_host(c, response_start, B, where);
    check_offsets(off, B);
    std::vector<int32_t> gather;
    std::vector<int64_t> oidx;
    int64_t R = 0;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t T = off[b + 1] - off[b];
      if (rs[b] == 0 || rs[b] >= T)  // src/losses.cpp:119-121
        throw ContractError("value_estimates: response_start must leave a nonempty prompt and response");
      for (int64_t t = 0; t < T - rs[b]; ++t) {
        gather.push_back(int32_t(off[b] + rs[b] - 1 + t));
        oidx.push_back(R + t);
      }
      R += T - rs[b];
    }
    check_tokens(c, tokens, off[B], m.cfg.vocab_size, where, "scoring");
    int32_t* gd = upload(c, "val.gather", gather);
    int64_t* od = upload(c, "val.oidx", oidx);
    Packed p = pack_tokens(c, tokens, off, where, "val");
    double* out_d = static_cast<double*>(c.workspace("val.out", std::max<int64_t>(R, 1) * 8));
    float* x = forward_layers(m, p, nullptr);
    score_head(m, x, gd, od, R, out_d);
    copy_out(c, out, out_d, R * 8, where);
    if (where == PPOEXP_HOST) c.sync();
  });
}

ppoexp_status ppoexp_reward_head(ppoexp_model rm, int64_t B, const int32_t* tokens, const int64_t* offsets, double* out,
                                 int32_t where) {
  return guard([&] {
    need(rm, "rm");
    if (B <= 0) return;
    Model& m = rm->m;
    Ctx& c = *m.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (!m.cfg.scalar_head) throw ShapeError("reward_head: head must be [d_model x 1], got none");
    const auto off = to_host(c, offsets, B + 1, where);
    check_offsets(off, B);
    for (int64_t b = 0; b < B; ++b)
      if (off[b + 1] == off[b]) throw ContractError("last_content_index: empty sequence");
    check_tokens(c, tokens, off[B], m.cfg.vocab_size, where, "scoring");
    Packed p = pack_tokens(c, tokens, off, where, "rw");
    int32_t* gd = static_cast<int32_t*>(c.workspace("rw.gather", B * 4));
    int64_t* od = static_cast<int64_t*>(c.workspace("rw.oidx", B * 8));
    c.launch("meta", 0, 0, [&] {
      launch_kernel(c, last_content_kernel, dim3(ceil_div(B, 128)), dim3(128), 0, 1, B, p.offsets_d, p.tokens_d, gd, od);
    });
    std::vector<int32_t> chk(B);
    PPOEXP_CUDA(cudaMemcpyAsync(chk.data(), gd, B * 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    for (int64_t b = 0; b < B; ++b)
      if (chk[b] < 0) throw ContractError("last_content_index: all-pad sequence");
    double* out_d = static_cast<double*>(c.workspace("rw.out", B * 8));
    float* x = forward_layers(m, p, nullptr);
    score_head(m, x, gd, od, B, out_d);
    copy_out(c, out, out_d, B * 8, where);
    if (where == PPOEXP_HOST) c.sync();
  });
}

// ------------------------------------------------------------------ shaping
ppoexp_status ppoexp_shape_gae(int64_t B, int64_t stride, const int64_t* lengths, const double* rm_reward,
                               const double* actor_lp, const double* ref_lp, const double* values, double kl_coef,
                               double gamma, double lam, double* out_rewards, double* out_adv, double* out_ret,
                               ppoexp_ctx ctx, int32_t where) {
  return guard([&] {
    need(ctx, "ctx");
    if (B <= 0) return;
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const auto len = to_host(c, lengths, B, where);
    for (int64_t b = 0; b < B; ++b)
      if (len[b] <= 0 || len[b] > stride)  // src/losses.cpp:190-192
        throw ContractError("kl_penalized_rewards: log-prob arrays must be nonempty and equal length");
    const size_t n = size_t(B) * stride * 8;
    auto buf = [&](const char* nm, size_t bytes) { return static_cast<double*>(c.workspace(nm, bytes)); };
    const int64_t* ld = lengths;
    const double *rw = rm_reward, *a = actor_lp, *r = ref_lp, *v = values;
    double *sh = out_rewards, *ad = out_adv, *rt = out_ret;
    if (where == PPOEXP_HOST) {
      int64_t* ldd = static_cast<int64_t*>(c.workspace("sg.len", B * 8));
      copy_in(c, ldd, lengths, B * 8, 0);
      ld = ldd;
      double* t;
      t = buf("sg.rw", B * 8); copy_in(c, t, rm_reward, B * 8, 0); rw = t;
      t = buf("sg.a", n); copy_in(c, t, actor_lp, n, 0); a = t;
      t = buf("sg.r", n); copy_in(c, t, ref_lp, n, 0); r = t;
      t = buf("sg.v", n); copy_in(c, t, values, n, 0); v = t;
      sh = buf("sg.sh", n);
      ad = buf("sg.ad", n);
      rt = buf("sg.rt", n);
    }
    double* part = buf("sg.part", B * 5 * 8);
    launch_shape_gae(c, B, stride, ld, rw, a, r, v, kl_coef, gamma, lam, sh, ad, rt, part);
    if (where == PPOEXP_HOST) {
      copy_out(c, out_rewards, sh, n, 0);
      copy_out(c, out_adv, ad, n, 0);
      copy_out(c, out_ret, rt, n, 0);
      c.sync();
    }
  });
}

ppoexp_status ppoexp_whiten_partials(int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                                     double* partials3, ppoexp_ctx ctx, int32_t where) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const auto len = to_host(c, lengths, B, where);
    const auto a = to_host(c, adv, B * stride, where);
    // fixed order on the host is fine for this small standalone entry point;
    // the experience pipeline reduces on the device (K12).
    double n = 0, s = 0, q = 0;
    for (int64_t b = 0; b < B; ++b)
      for (int64_t t = 0; t < len[b]; ++t) {
        const double x = a[b * stride + t];
        n += 1;
        s += x;
        q += x * x;
      }
    const double p3[3] = {n, s, q};
    if (where == PPOEXP_HOST)
      std::memcpy(partials3, p3, sizeof p3);
    else {
      PPOEXP_CUDA(cudaMemcpyAsync(partials3, p3, sizeof p3, cudaMemcpyHostToDevice, c.stream));
      c.sync();
    }
  });
}

ppoexp_status ppoexp_whiten_apply(int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                                  const double* global3, double* out, ppoexp_ctx ctx, int32_t where) {
  return guard([&] {
    need(ctx, "ctx");
    if (B <= 0) return;
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const size_t n = size_t(B) * stride * 8;
    const int64_t* ld = lengths;
    const double *a = adv, *st = global3;
    double* o = out;
    if (where == PPOEXP_HOST) {
      int64_t* ldd = static_cast<int64_t*>(c.workspace("wh.len", B * 8));
      copy_in(c, ldd, lengths, B * 8, 0);
      ld = ldd;
      double* t = static_cast<double*>(c.workspace("wh.a", n));
      copy_in(c, t, adv, n, 0);
      a = t;
      double* s3 = static_cast<double*>(c.workspace("wh.s", 64));
      copy_in(c, s3, global3, 24, 0);
      st = s3;
      o = static_cast<double*>(c.workspace("wh.o", n));
      PPOEXP_CUDA(cudaMemsetAsync(o, 0, n, c.stream));
    }
    launch_whiten_apply(c, B, stride, ld, a, st, o);
    if (where == PPOEXP_HOST) {
      copy_out(c, out, o, n, 0);
      c.sync();
    }
  });
}

// ------------------------------------------------------------------ experience
ppoexp_status ppoexp_make_experience(const ppoexp_experience_request* req, int64_t B, const int32_t* prompts,
                                     const int64_t* offsets, const ppoexp_rollout_batch* out, int32_t where) {
  return guard([&] {
    need(req, "request");
    need(out, "out");
    need(req->policy_engine, "policy_engine");
    need(req->reference, "reference");
    need(req->critic, "critic");
    Engine& E = *req->policy_engine->e;
    Model& pol = *E.m;
    Model& ref = req->reference->m;
    Model& cr = req->critic->m;
    Model* rm = req->rm ? &req->rm->m : nullptr;
    check_same_ctx(pol, ref);
    check_same_ctx(pol, cr);
    if (rm) check_same_ctx(pol, *rm);
    if (!cr.cfg.scalar_head) throw PpoError("critic job: critic model needs a scalar head");  // src/ppo.cpp:94-96
    if (rm && !rm->cfg.scalar_head) throw PpoError("critic job: reward model needs a scalar head");
    if (B <= 0) throw PpoError("ppo_step: empty prompt batch");  // src/ppo.cpp:294
    const int64_t N = req->max_new;
    if (N <= 0) throw PpoError("ppo_step: max_new must be positive");
    // PpoHyper::validate (gamma/lam ranges), src/losses.cpp:384-388
    if (req->hyper.gamma <= 0.0 || req->hyper.gamma > 1.0) throw ContractError("ppo hyper: gamma must be in (0,1]");
    if (req->hyper.lam <= 0.0 || req->hyper.lam > 1.0) throw ContractError("ppo hyper: lam must be in (0,1]");
    Ctx& c = *pol.ctx;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    // ev: 0 start, 1 whitened, 2 outputs copied; 3 generation done, 4 policy
    // lp, 5 reference lp, 6 critic values (+ RM reward) — StepTiming
    cudaEvent_t ev[7];
    for (auto& e : ev) PPOEXP_CUDA(cudaEventCreate(&e));
    PPOEXP_CUDA(cudaEventRecord(ev[0], c.stream));

    const auto off = to_host(c, offsets, B + 1, where);
    check_offsets(off, B);
    std::vector<int64_t> P(B);
    for (int64_t b = 0; b < B; ++b) {
      P[b] = off[b + 1] - off[b];
      if (P[b] + N > pol.cfg.max_seq_len)  // run_ppo's guard, src/ppo.cpp:456-459
        throw PpoError("run_ppo: prompt plus max_new exceeds max_seq_len");
    }
    // (1) generation: per-task seeds mix_seed(seed, step*1000003 + gidx), src/ppo.cpp:312-313
    std::vector<int64_t> mx(B, N);
    std::vector<uint64_t> seeds(B);
    for (int64_t b = 0; b < B; ++b) {
      const uint64_t bb = uint64_t(req->step_index) * 1000003ULL + uint64_t(req->gidx0 + b);
      uint64_t z = req->seed + 0x9e3779b97f4a7c15ULL * (bb + 1);  // mix_seed, include/aligner/rng.hpp:51-56
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      seeds[b] = z ^ (z >> 31);
    }
    const size_t nBN = size_t(B) * N;
    int32_t* gtok = static_cast<int32_t*>(c.workspace("xp.tok", nBN * 4));
    double* glp = static_cast<double*>(c.workspace("xp.glp", nBN * 8));
    int64_t* glen = static_cast<int64_t*>(c.workspace("xp.len", B * 8));
    // prompts to device once (generation and packing both read them)
    int32_t* pd = static_cast<int32_t*>(c.workspace("xp.prompts", std::max<int64_t>(off[B], 1) * 4));
    copy_in(c, pd, prompts, off[B] * 4, where);
    int64_t* poff_d = upload(c, "xp.poff", off);
    double gen_ms = 0;
    const std::vector<ppoexp_sampling> sps(B, req->sampling);
    E.generate(B, pd, off.data(), mx.data(), sps.data(), seeds.data(), N, gtok, glp, glen, PPOEXP_HOST, &gen_ms,
               PPOEXP_DEVICE, PPOEXP_DEVICE);
    const std::vector<int64_t> n = E.last_lengths;
    for (int64_t b = 0; b < B; ++b)
      if (n[b] <= 0) throw PpoError("ppo_step: empty generation for prompt " + std::to_string(b));  // src/ppo.cpp:326
    // (2) pack prompt ++ response
    std::vector<int64_t> foff(B + 1, 0), roff(B + 1, 0);
    for (int64_t b = 0; b < B; ++b) {
      foff[b + 1] = foff[b] + P[b] + n[b];
      roff[b + 1] = roff[b] + n[b];
    }
    Packed pk;
    pk.offsets = foff;
    pk.tokens_d = static_cast<int32_t*>(c.workspace("xp.full", foff[B] * 4));
    int64_t* plen_d = upload(c, "xp.plen", P);
    int64_t* rlen_d = upload(c, "xp.rlen", n);
    int64_t* roff_d = upload(c, "xp.roff", roff);
    pack_metadata(c, pk, "xp");
    launch_concat_pack(c, B, pd, poff_d, gtok, N, glen, pk.offsets_d, pk.tokens_d);
    const int64_t R = roff[B];
    int32_t* gather = static_cast<int32_t*>(c.workspace("xp.gather", R * 4));
    int32_t* target = static_cast<int32_t*>(c.workspace("xp.target", R * 4));
    int64_t* oidx = static_cast<int64_t*>(c.workspace("xp.oidx", R * 8));
    launch_response_meta(c, B, pk.offsets_d, plen_d, rlen_d, N, pk.tokens_d, gather, target, oidx, roff_d);
    // (3) actor + reference log-probs over the response (src/ppo.cpp:337-341)
    double* alp = static_cast<double*>(c.workspace("xp.alp", nBN * 8));
    double* rlp = static_cast<double*>(c.workspace("xp.rlp", nBN * 8));
    double* val = static_cast<double*>(c.workspace("xp.val", nBN * 8));
    PPOEXP_CUDA(cudaMemsetAsync(alp, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaMemsetAsync(rlp, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaMemsetAsync(val, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaEventRecord(ev[3], c.stream));
    // The policy, reference and critic forwards read the same packed tokens and
    // write disjoint outputs: with PPOEXP_SCORE_STREAMS=1 the reference and critic
    // run on two auxiliary streams (own workspaces) concurrently with the policy.
    // Default: one stream — the persistent GEMMs and the 192 KB attention CTAs
    // each fill every SM, so concurrency bought nothing (26–27 ms per C2 step
    // either way) and occasionally cost a lot (a persistent grid waiting for SMs
    // held by another stream's kernel: single steps up to +100 ms)
    static const bool concurrent = [] {
      const char* e = getenv("PPOEXP_SCORE_STREAMS");
      return e ? e[0] == '1' : !gemm_pp_enabled();
    }();
    // concurrent forwards hold one set of activation workspaces each: fall back
    // to one stream when two more sets would not fit comfortably in free HBM
    // (e.g. config 4 in mixed mode: 74k rows x (6 d + f) fp32 = 11.5 GB per set)
    bool roomy = true;
    {
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        const double per_set = double(foff[B]) * double(6 * pol.cfg.d_model + pol.cfg.d_ff) * double(pol.asize());
        roomy = 2.0 * per_set < 0.6 * double(free_b);
      } else {
        (void)cudaGetLastError();
      }
    }
    const bool conc = concurrent && !rm && roomy;
    cudaStream_t main_stream = c.stream;
    auto on_aux = [&](int i, const char* prefix, auto&& body) {
      if (!conc) {
        body();
        return;
      }
      if (!c.aux[i]) PPOEXP_CUDA(cudaStreamCreateWithFlags(&c.aux[i], cudaStreamNonBlocking));
      if (!c.join_ev[i]) PPOEXP_CUDA(cudaEventCreateWithFlags(&c.join_ev[i], cudaEventDisableTiming));
      PPOEXP_CUDA(cudaStreamWaitEvent(c.aux[i], c.fork_ev, 0));
      c.stream = c.aux[i];
      c.ws_prefix = prefix;
      try {
        body();
      } catch (...) {
        c.stream = main_stream;
        c.ws_prefix.clear();
        throw;
      }
      PPOEXP_CUDA(cudaEventRecord(c.join_ev[i], c.aux[i]));
      c.stream = main_stream;
      c.ws_prefix.clear();
    };
    if (conc) {
      if (!c.fork_ev) PPOEXP_CUDA(cudaEventCreateWithFlags(&c.fork_ev, cudaEventDisableTiming));
      PPOEXP_CUDA(cudaEventRecord(c.fork_ev, main_stream));
    }
    on_aux(0, "ref/", [&] {
      float* x = forward_layers(ref, pk, nullptr);
      score_logprobs(ref, pk, x, gather, target, oidx, R, rlp);
      PPOEXP_CUDA(cudaEventRecord(ev[5], c.stream));
    });
    on_aux(1, "crit/", [&] {
      float* x = forward_layers(cr, pk, nullptr);
      score_head(cr, x, gather, oidx, R, val);
      PPOEXP_CUDA(cudaEventRecord(ev[6], c.stream));
    });
    {
      float* x = forward_layers(pol, pk, nullptr);
      score_logprobs(pol, pk, x, gather, target, oidx, R, alp);
      PPOEXP_CUDA(cudaEventRecord(ev[4], c.stream));
    }
    // (4) rewards then values (CriticJob::handle_infer, src/ppo.cpp:164-193)
    double* rew = static_cast<double*>(c.workspace("xp.rew", B * 8));
    if (rm) {
      int32_t* lg = static_cast<int32_t*>(c.workspace("xp.lastg", B * 4));
      int64_t* lo = static_cast<int64_t*>(c.workspace("xp.lasto", B * 8));
      c.launch("meta", 0, 0, [&] {
        launch_kernel(c, last_content_kernel, dim3(ceil_div(B, 128)), dim3(128), 0, 1, B, pk.offsets_d, pk.tokens_d, lg, lo);
      });
      float* x = forward_layers(*rm, pk, nullptr);
      score_head(*rm, x, lg, lo, B, rew);
      PPOEXP_CUDA(cudaEventRecord(ev[6], c.stream));  // the RM pass precedes the critic's (src/ppo.cpp:175-188)
    } else {
      launch_scripted_reward(c, B, N, gtok, glen, req->scripted_target, rew);
    }
    if (conc) {  // join the reference and critic streams (the critic ran above in either mode)
      PPOEXP_CUDA(cudaStreamWaitEvent(c.stream, c.join_ev[0], 0));
      PPOEXP_CUDA(cudaStreamWaitEvent(c.stream, c.join_ev[1], 0));
    }
    // (5) KL shaping + GAE + per-sequence partials (src/ppo.cpp:382-393)
    double* shp = static_cast<double*>(c.workspace("xp.shp", nBN * 8));
    double* adv = static_cast<double*>(c.workspace("xp.adv", nBN * 8));
    double* ret = static_cast<double*>(c.workspace("xp.ret", nBN * 8));
    double* wht = static_cast<double*>(c.workspace("xp.wht", nBN * 8));
    double* part = static_cast<double*>(c.workspace("xp.part", B * 5 * 8));
    double* red = static_cast<double*>(c.workspace("xp.red", 16 * 8));
    PPOEXP_CUDA(cudaMemsetAsync(shp, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaMemsetAsync(adv, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaMemsetAsync(ret, 0, nBN * 8, c.stream));
    PPOEXP_CUDA(cudaMemsetAsync(wht, 0, nBN * 8, c.stream));
    launch_shape_gae(c, B, N, glen, rew, alp, rlp, val, req->hyper.kl_penalty_coef, req->hyper.gamma, req->hyper.lam,
                     shp, adv, ret, part);
    // red[0..4] = {kl_sum, n_tokens, reward_sum, adv_sum, adv_sq}
    launch_reduce_partials(c, B, part, red);
    // (6) the single collective: {n_tokens, sum adv, sum adv^2, kl_sum, reward_sum, n_seqs}
    double* coll = red + 8;
    {
      // reorder on device with a tiny copy chain (stream-ordered)
      PPOEXP_CUDA(cudaMemcpyAsync(coll + 0, red + 1, 8, cudaMemcpyDeviceToDevice, c.stream));
      PPOEXP_CUDA(cudaMemcpyAsync(coll + 1, red + 3, 16, cudaMemcpyDeviceToDevice, c.stream));
      PPOEXP_CUDA(cudaMemcpyAsync(coll + 3, red + 0, 8, cudaMemcpyDeviceToDevice, c.stream));
      PPOEXP_CUDA(cudaMemcpyAsync(coll + 4, red + 2, 8, cudaMemcpyDeviceToDevice, c.stream));
      const double nseq = double(B);
      double* tmp = static_cast<double*>(c.pinned_staging(8));
      *tmp = nseq;
      PPOEXP_CUDA(cudaMemcpyAsync(coll + 5, tmp, 8, cudaMemcpyHostToDevice, c.stream));
      PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
    }
    if (req->comm) {
      if (req->comm->c->ctx != &c) throw ContractError("ppo_step: comm belongs to another context");
      req->comm->c->allgather_sum(coll, 6);
    } else if (req->allreduce) {
      const int32_t rc = req->allreduce(coll, 6, c.stream, req->allreduce_user);
      if (rc) throw PpoError("ppo_step: whitening allreduce failed (" + std::to_string(rc) + ")");
    }
    launch_whiten_apply(c, B, N, glen, adv, coll, wht);
    PPOEXP_CUDA(cudaEventRecord(ev[1], c.stream));
    // outputs
    double stats_h[8] = {0};
    double coll_h[6];
    PPOEXP_CUDA(cudaMemcpyAsync(coll_h, coll, 48, cudaMemcpyDeviceToHost, c.stream));
    auto put = [&](void* dst, const void* src, size_t bytes) {
      if (dst) copy_out(c, dst, src, bytes, where);
    };
    put(out->tokens, gtok, nBN * 4);
    put(out->lengths, glen, B * 8);
    put(out->actor_lp, alp, nBN * 8);
    put(out->ref_lp, rlp, nBN * 8);
    put(out->values, val, nBN * 8);
    put(out->rewards, rew, B * 8);
    put(out->shaped, shp, nBN * 8);
    put(out->advantages, adv, nBN * 8);
    put(out->returns, ret, nBN * 8);
    put(out->whitened, wht, nBN * 8);
    PPOEXP_CUDA(cudaEventRecord(ev[2], c.stream));
    PPOEXP_CUDA(cudaEventSynchronize(ev[2]));
    float total_ms = 0;
    PPOEXP_CUDA(cudaEventElapsedTime(&total_ms, ev[0], ev[2]));
    if (out->timing) {
      // StepTiming (include/aligner/ppo.hpp:27-37): rollout, response_generation,
      // logprob_calculation (actor + reference, after generation), critic_wait
      auto since = [&](int i) {
        float ms = 0;
        PPOEXP_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[i]));
        return double(ms);
      };
      const double t_gen = since(3), t_lp = std::max(since(4), since(5)), t_cr = since(6);
      const double tm[4] = {double(total_ms), gen_ms, t_lp - t_gen, std::max(0.0, t_cr - t_lp)};
      if (where == PPOEXP_HOST)
        std::memcpy(out->timing, tm, sizeof tm);
      else
        PPOEXP_CUDA(cudaMemcpy(out->timing, tm, sizeof tm, cudaMemcpyHostToDevice));
    }
    for (auto& e : ev) cudaEventDestroy(e);
    const double cnt = coll_h[0] > 0 ? coll_h[0] : 1.0;
    const double mean = coll_h[1] / cnt;
    double var = coll_h[2] / cnt - mean * mean;
    if (var < 0) var = 0;
    stats_h[0] = coll_h[3];
    stats_h[1] = coll_h[0];
    stats_h[2] = coll_h[4];
    stats_h[3] = coll_h[5];
    stats_h[4] = mean;
    stats_h[5] = std::sqrt(var);
    stats_h[6] = gen_ms;
    stats_h[7] = total_ms;
    if (out->stats) {
      if (where == PPOEXP_HOST)
        std::memcpy(out->stats, stats_h, sizeof stats_h);
      else
        PPOEXP_CUDA(cudaMemcpy(out->stats, stats_h, sizeof stats_h, cudaMemcpyHostToDevice));
    }
    c.harvest();
  });
}

// ------------------------------------------------------------------ train side
ppoexp_status ppoexp_trainer_create(ppoexp_ctx ctx, const ppoexp_model_config* config, const ppoexp_tensor_view* params,
                                    int64_t n, ppoexp_model serving, const ppoexp_adamw_options* opts,
                                    ppoexp_trainer* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(config, "config");
    need(params, "params");
    need(out, "out");
    if (serving && serving->m.ctx != ctx->c.get()) throw ContractError("trainer: serving model on another context");
    AdamOpts o;
    if (opts) o = AdamOpts{opts->beta1, opts->beta2, opts->eps, opts->weight_decay};
    std::lock_guard<std::recursive_mutex> lk(ctx->c->mu);
    auto h = std::make_unique<ppoexp_trainer_s>();
    h->t = std::make_unique<Trainer>(ctx->c.get(), *config, params, n, serving ? &serving->m : nullptr, o);
    *out = h.release();
  });
}

ppoexp_status ppoexp_trainer_destroy(ppoexp_trainer trainer) {
  return guard([&] { delete trainer; });
}

ppoexp_status ppoexp_trainer_ppo_actor_step(ppoexp_trainer trainer, int64_t B, const int32_t* tokens,
                                            const int64_t* offsets, const int64_t* response_start,
                                            const double* old_lp, const double* adv, const double* mask,
                                            double clip_eps, double lr, double* loss_out, int32_t where) {
  return guard([&] {
    need(trainer, "trainer");
    if (B <= 0) throw PpoError("ppo_step: empty prompt batch");
    need(tokens, "tokens");
    need(old_lp, "old_logprobs");
    need(adv, "advantages");
    Trainer& t = *trainer->t;
    std::lock_guard<std::recursive_mutex> lk(t.c->mu);
    DeviceGuard g(t.c->device);
    const double l = t.ppo_actor_step(B, tokens, offsets, response_start, old_lp, adv, mask, clip_eps, lr, where);
    if (loss_out) *loss_out = l;
  });
}

ppoexp_status ppoexp_trainer_critic_step(ppoexp_trainer trainer, int64_t B, const int32_t* tokens,
                                         const int64_t* offsets, const int64_t* response_start,
                                         const double* old_values, const double* returns, double value_clip, double lr,
                                         double* loss_out, int32_t where) {
  return guard([&] {
    need(trainer, "trainer");
    if (B <= 0) throw PpoError("critic job: empty training batch");
    need(tokens, "tokens");
    need(old_values, "old_values");
    need(returns, "returns");
    Trainer& t = *trainer->t;
    std::lock_guard<std::recursive_mutex> lk(t.c->mu);
    DeviceGuard g(t.c->device);
    const double l = t.critic_step(B, tokens, offsets, response_start, old_values, returns, value_clip, lr, where);
    if (loss_out) *loss_out = l;
  });
}

ppoexp_status ppoexp_trainer_dpo_step(ppoexp_trainer trainer, ppoexp_model reference, int64_t n_pairs,
                                      const int32_t* tokens, const int64_t* offsets, const int64_t* response_start,
                                      int32_t variant, double beta, double cdpo_eps, double lr, double* loss_out,
                                      double* margin_out, int32_t where) {
  return guard([&] {
    need(trainer, "trainer");
    need(reference, "reference");
    if (n_pairs <= 0) throw ContractError("dpo_family_loss: mismatched sequence counts");
    need(tokens, "tokens");
    Trainer& t = *trainer->t;
    std::lock_guard<std::recursive_mutex> lk(t.c->mu);
    DeviceGuard g(t.c->device);
    // frozen reference sums through the public scoring path (fused LM head)
    std::vector<double> ref_sums(2 * n_pairs);
    double* dst = ref_sums.data();
    if (where == PPOEXP_DEVICE) dst = static_cast<double*>(t.c->workspace("dpo.ref_sums", 2 * n_pairs * 8));
    const ppoexp_status rc =
        ppoexp_response_logprob_sums(reference, 2 * n_pairs, tokens, offsets, response_start, dst, where);
    if (rc != PPOEXP_OK) throw Error(int(rc), g_err);
    if (where == PPOEXP_DEVICE) {
      PPOEXP_CUDA(cudaStreamSynchronize(t.c->stream));
      PPOEXP_CUDA(cudaMemcpy(ref_sums.data(), dst, 2 * n_pairs * 8, cudaMemcpyDeviceToHost));
    }
    const double l = t.dpo_step(n_pairs, tokens, offsets, response_start, ref_sums, variant, beta, cdpo_eps, lr, where,
                                margin_out);
    if (loss_out) *loss_out = l;
  });
}

ppoexp_status ppoexp_trainer_refit(ppoexp_trainer trainer) {
  return guard([&] {
    need(trainer, "trainer");
    std::lock_guard<std::recursive_mutex> lk(trainer->t->c->mu);
    DeviceGuard g(trainer->t->c->device);
    trainer->t->refit();
  });
}

ppoexp_status ppoexp_trainer_get(ppoexp_trainer trainer, const char* name, double* out, int64_t numel) {
  return guard([&] {
    need(trainer, "trainer");
    need(name, "name");
    need(out, "out");
    std::lock_guard<std::recursive_mutex> lk(trainer->t->c->mu);
    DeviceGuard g(trainer->t->c->device);
    trainer->t->get(name, out, numel);
  });
}

}  // extern "C"

// ------------------------------------------------------------------ testing
namespace ppx {
template <class T>
void launch_gemm_simt(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc);
}

extern "C" ppoexp_status ppoexp_testing_gemm_bf16(ppoexp_ctx ctx, const void* A, int64_t lda, const void* B,
                                                  int64_t ldb, int64_t M, int64_t N, int64_t K, int32_t epi, void* C,
                                                  int64_t ldc, int32_t path) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (epi < 0 || epi > 3) throw ContractError("epi must be 0..3");
    const auto* a = static_cast<const bf16*>(A);
    const auto* b = static_cast<const bf16*>(B);
    if (path == 1)
      launch_gemm_simt<bf16>(c, a, lda, b, ldb, M, N, K, static_cast<Epi>(epi), C, ldc);
    else
      gemm<bf16>(c, a, lda, b, ldb, M, N, K, static_cast<Epi>(epi), C, ldc);
    c.sync();
  });
}

extern "C" ppoexp_status ppoexp_testing_lm_head_logprobs(ppoexp_ctx ctx, const void* H, const void* W, int64_t R,
                                                         int64_t V, int64_t K, int64_t ldl, const int32_t* target,
                                                         double* out, int32_t path) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (R <= 0) return;
    int64_t* oidx = static_cast<int64_t*>(c.workspace("t.oidx", R * 8));
    std::vector<int64_t> iota(R);
    for (int64_t i = 0; i < R; ++i) iota[i] = i;
    copy_in(c, oidx, iota.data(), R * 8, PPOEXP_HOST);
    c.sync();
    const auto* h = static_cast<const bf16*>(H);
    const auto* w = static_cast<const bf16*>(W);
    if (path == 0) {
      const int nt = lse_tiles(V), ldp = (nt + 1) / 2 * 2;
      LseEpi e;
      e.target = target;
      e.tgt_logit = static_cast<float*>(c.workspace("t.tgt", R * 4));
      e.part = static_cast<float2*>(c.workspace("t.part", R * ldp * 8));
      e.ldp = ldp;
      if (!gemm_tc_lse(c, h, K, w, K, R, V, K, e)) throw ContractError("lm_head: shape not eligible");
      launch_lse_combine(c, e.part, ldp, nt, e.tgt_logit, target, R, oidx, out);
    } else if (path == 1) {
      const int64_t ld = (V + 63) / 64 * 64;
      float* lg = static_cast<float*>(c.workspace("t.logits", R * ld * 4));
      gemm<bf16>(c, h, K, w, K, R, V, K, Epi::kStoreF32, lg, ld);
      launch_logprob_gather<float>(c, lg, ld, R, V, target, oidx, out);
    } else {
      launch_logprob_gather<float>(c, static_cast<const float*>(H), ldl, R, V, target, oidx, out);
    }
    c.sync();
  });
}

extern "C" ppoexp_status ppoexp_testing_gemm_mixed(ppoexp_ctx ctx, const void* A, int64_t lda, const void* W,
                                                   int64_t ldw, int64_t M, int64_t N, int64_t K, int32_t epi, void* C,
                                                   int64_t ldc) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (epi != 2 && epi != 3 && epi != 5) throw ContractError("epi must be 2, 3 or 5");
    gemm_mixed(c, static_cast<const float*>(A), lda, static_cast<const bf16*>(W), ldw, M, N, K, static_cast<Epi>(epi), C,
               ldc);
    c.sync();
  });
}

extern "C" ppoexp_status ppoexp_testing_variant_count(ppoexp_ctx ctx, const char* name, int64_t* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(name, "name");
    need(out, "out");
    std::lock_guard<std::recursive_mutex> lk(ctx->c->mu);
    const auto it = ctx->c->variants.find(name);
    *out = it == ctx->c->variants.end() ? 0 : it->second;
  });
}

namespace ppx {
void umma_probe(Ctx& c, const bf16* A, const bf16* B, int N, float* out, int variant);
}
extern "C" ppoexp_status ppoexp_testing_umma_probe(ppoexp_ctx ctx, const void* A, const void* B, int32_t N, float* out,
                                                   int32_t variant) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (N != 64 && N != 128) throw ContractError("N must be 64 or 128");
    umma_probe(c, static_cast<const bf16*>(A), static_cast<const bf16*>(B), N, out, variant);
    c.sync();
  });
}

namespace ppx {
bool attention_prefill_mma(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                           int64_t H, int64_t DH, bf16* out);
}
extern "C" ppoexp_status ppoexp_testing_attention_prefill(ppoexp_ctx ctx, const void* qkv, const int64_t* offsets,
                                                          int64_t B, int64_t max_len, int64_t H, int64_t DH,
                                                          int64_t M, void* out, int32_t path) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    const auto* q = static_cast<const bf16*>(qkv);
    auto* o = static_cast<bf16*>(out);
    bool ok = path == 0   ? attention_prefill_tc(c, q, offsets, B, max_len, H, DH, M, o, true)
              : path == 2 ? attention_prefill_tc_split(c, q, offsets, B, max_len, H, DH, M, o)
                          : attention_prefill_mma(c, q, offsets, B, max_len, H, DH, o);
    if (!ok) throw ContractError("attention path not eligible for this shape");
    c.sync();
  });
}

extern "C" ppoexp_status ppoexp_testing_gemm_planes(ppoexp_ctx ctx, const void* A, const void* W, int64_t M, int64_t N,
                                                    int64_t K, int32_t epi, void* C, int64_t ldc) {
  return guard([&] {
    need(ctx, "ctx");
    Ctx& c = *ctx->c;
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    if (epi != 2 && epi != 3 && epi != 6) throw ContractError("epi must be 2, 3 or 6");
    gemm_tc_planes(c, static_cast<const bf16*>(A), 2 * K, static_cast<const bf16*>(W), K, M, N, K, static_cast<Epi>(epi),
                   C, ldc);
    c.sync();
  });
}

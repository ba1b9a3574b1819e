// model.cu — device weight snapshot (build / refit), the batched causal
// forward over packed ragged sequences, and the scoring heads.
#include <algorithm>
#include <cstring>

#include "model.hpp"

namespace ppx {

// ------------------------------------------------------------------ names
std::vector<std::pair<std::string, std::vector<int64_t>>> Model::expected(const ppoexp_model_config& c) {
  // ModelParams::expected_names + param_shape, src/model.cpp:66-115 (no LoRA)
  const int64_t d = c.d_model;
  std::vector<std::pair<std::string, std::vector<int64_t>>> v;
  v.push_back({"tok_embed.weight", {c.vocab_size, d}});
  v.push_back({"pos_embed.weight", {c.max_seq_len, d}});
  for (int64_t i = 0; i < c.n_layers; ++i) {
    const std::string base = "layers." + std::to_string(i) + ".";
    v.push_back({base + "attn_norm.weight", {d}});
    v.push_back({base + "attn_norm.bias", {d}});
    for (const char* p : {"q_proj", "k_proj", "v_proj", "o_proj"})
      v.push_back({base + "attn." + p + ".weight", {d, d}});
    v.push_back({base + "ffn_norm.weight", {d}});
    v.push_back({base + "ffn_norm.bias", {d}});
    v.push_back({base + "ffn.up_proj.weight", {d, c.d_ff}});
    v.push_back({base + "ffn.down_proj.weight", {c.d_ff, d}});
  }
  v.push_back({"final_norm.weight", {d}});
  v.push_back({"final_norm.bias", {d}});
  if (c.scalar_head) v.push_back({"scalar_head.weight", {d, 1}});
  return v;
}

void Model::allocate() {
  const auto& c = cfg;
  const int64_t d = c.d_model, f = c.d_ff, V = c.vocab_size, S = c.max_seq_len, L = c.n_layers;
  const size_t ts = tsize();
  // Each tensor 256-byte aligned (TMA / 16-byte vector loads).
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t tbytes = al(V * d * ts) + al(S * d * ts) + L * (al(3 * d * d * ts) + al(d * d * ts) + 2 * al(d * f * ts));
  size_t fbytes = (L * 4 * d + 3 * d) * sizeof(float) + 256;
  wbuf.ensure(tbytes);
  fbuf.ensure(fbytes);
  PPOEXP_CUDA(cudaMemsetAsync(fbuf.ptr, 0, fbytes, ctx->stream));
  char* p = static_cast<char*>(wbuf.ptr);
  auto take = [&](size_t n) {
    void* r = p;
    p += al(n);
    return r;
  };
  tok = take(V * d * ts);
  pos = take(S * d * ts);
  layers.resize(L);
  float* fp = fbuf.as<float>();
  for (auto& ly : layers) {
    ly.wqkv = take(3 * d * d * ts);
    ly.wo = take(d * d * ts);
    ly.wup = take(f * d * ts);
    ly.wdown = take(d * f * ts);
    ly.ln1w = fp; fp += d;
    ly.ln1b = fp; fp += d;
    ly.ln2w = fp; fp += d;
    ly.ln2b = fp; fp += d;
  }
  lnfw = fp; fp += d;
  lnfb = fp; fp += d;
  head = fp;
  vpad = (V + 63) / 64 * 64;
}

static std::string shape_str(const std::vector<int64_t>& s) {
  std::string r = "[";
  for (size_t i = 0; i < s.size(); ++i) r += (i ? "x" : "") + std::to_string(s[i]);
  return r + "]";
}

void Model::load(const ppoexp_tensor_view* views, int64_t n, bool refit) {
  const auto exp = expected(cfg);
  std::map<std::string, const ppoexp_tensor_view*> by;
  for (int64_t i = 0; i < n; ++i) {
    if (!views[i].name) throw ContractError("tensor view without a name");
    by[views[i].name] = &views[i];
  }
  auto fail = [&](const std::string& m) -> Error {
    return refit ? RefitError("refit: " + m + " (rebuild required)") : ContractError("model build: " + m);
  };
  // Validate the full name/shape set before touching anything (src/engine.cpp:62-77).
  if (static_cast<int64_t>(by.size()) != static_cast<int64_t>(exp.size()) || n != static_cast<int64_t>(exp.size()))
    throw fail("parameter count mismatch: engine has " + std::to_string(exp.size()) + ", update has " +
               std::to_string(n));
  for (const auto& [name, shape] : exp) {
    auto it = by.find(name);
    if (it == by.end()) throw fail("missing parameter " + name);
    const auto* v = it->second;
    std::vector<int64_t> got(v->shape, v->shape + std::max(0, std::min(2, v->rank)));
    // scalar_head may come as [d] or [d,1]; norms as [d]
    std::vector<int64_t> want = shape;
    bool ok = got == want;
    if (!ok && name == "scalar_head.weight" && got.size() == 1 && got[0] == want[0]) ok = true;
    if (!ok) throw fail("shape mismatch for " + name + ": engine " + shape_str(want) + " vs update " + shape_str(got));
    if (!v->data) throw fail("null data for " + name);
    if (v->dtype < 0 || v->dtype > 2) throw fail("bad dtype for " + name);
  }
  Ctx& c = *ctx;
  const int64_t d = cfg.d_model, f = cfg.d_ff;
  const int ddt = dtype;  // 0 = f32, 1 = bf16
  for (const auto& [name, shape] : exp) {
    const auto* v = by[name];
    int64_t numel = 1;
    for (auto s : shape) numel *= s;
    const size_t esz = v->dtype == PPOEXP_F64 ? 8 : (v->dtype == PPOEXP_F32 ? 4 : 2);
    const void* src = v->data;
    if (v->where == PPOEXP_HOST) {
      void* st = c.workspace("load.staging", numel * esz);
      PPOEXP_CUDA(cudaMemcpyAsync(st, v->data, numel * esz, cudaMemcpyHostToDevice, c.stream));
      src = st;
    }
    auto conv = [&](void* dst, int dst_dt, int64_t rows, int64_t cols, bool tr, int64_t ld, int64_t row0) {
      launch_convert(c, src, v->dtype, dst, dst_dt, rows, cols, tr, ld, row0);
    };
    if (name == "tok_embed.weight") {
      conv(tok, ddt, cfg.vocab_size, d, false, d, 0);
    } else if (name == "pos_embed.weight") {
      conv(pos, ddt, cfg.max_seq_len, d, false, d, 0);
    } else if (name == "final_norm.weight") {
      conv(lnfw, 0, 1, d, false, d, 0);
    } else if (name == "final_norm.bias") {
      conv(lnfb, 0, 1, d, false, d, 0);
    } else if (name == "scalar_head.weight") {
      conv(head, 0, 1, d, false, d, 0);
    } else {
      const size_t dot = name.find('.', 7);
      const int64_t li = std::stoll(name.substr(7, dot - 7));
      const std::string rest = name.substr(dot + 1);
      Layer& ly = layers[li];
      if (rest == "attn_norm.weight") conv(ly.ln1w, 0, 1, d, false, d, 0);
      else if (rest == "attn_norm.bias") conv(ly.ln1b, 0, 1, d, false, d, 0);
      else if (rest == "ffn_norm.weight") conv(ly.ln2w, 0, 1, d, false, d, 0);
      else if (rest == "ffn_norm.bias") conv(ly.ln2b, 0, 1, d, false, d, 0);
      // reference W is [in, out]; the device keeps W^T [out, in] (K-major)
      else if (rest == "attn.q_proj.weight") conv(ly.wqkv, ddt, d, d, true, d, 0);
      else if (rest == "attn.k_proj.weight") conv(ly.wqkv, ddt, d, d, true, d, d);
      else if (rest == "attn.v_proj.weight") conv(ly.wqkv, ddt, d, d, true, d, 2 * d);
      else if (rest == "attn.o_proj.weight") conv(ly.wo, ddt, d, d, true, d, 0);
      else if (rest == "ffn.up_proj.weight") conv(ly.wup, ddt, d, f, true, d, 0);
      else if (rest == "ffn.down_proj.weight") conv(ly.wdown, ddt, f, d, true, f, 0);
      else throw ContractError("unknown parameter name: " + name);
    }
    // staging is reused by the next tensor: order the copies
    if (v->where == PPOEXP_HOST) PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
  }
  PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
}

// Engine::snapshot (include/aligner/engine.hpp:67), one parameter: the device
// copy back in the reference layout ([in, out] projections, row-major).
void Model::snapshot(const std::string& name, void* out, int64_t numel, int out_dtype) {
  const auto exp = expected(cfg);
  const std::vector<int64_t>* shape = nullptr;
  for (const auto& [n, sh] : exp)
    if (n == name) shape = &sh;
  if (!shape) throw ContractError("snapshot: unknown parameter " + name);
  int64_t want = 1;
  for (auto v : *shape) want *= v;
  if (numel != want)
    throw ShapeError("snapshot: " + name + " has " + std::to_string(want) + " elements, buffer " + std::to_string(numel));
  if (out_dtype != PPOEXP_F64 && out_dtype != PPOEXP_F32) throw ContractError("snapshot: dtype must be F64 or F32");
  const int64_t d = cfg.d_model, f = cfg.d_ff;
  // device source: base pointer, element type (0 f32, 1 T), rows x cols as stored, row offset, transposed
  const void* base = nullptr;
  bool is_t = true, tr = false;
  int64_t rows = 0, cols = 0, row0 = 0;
  if (name == "tok_embed.weight") base = tok, rows = cfg.vocab_size, cols = d;
  else if (name == "pos_embed.weight") base = pos, rows = cfg.max_seq_len, cols = d;
  else if (name == "final_norm.weight") base = lnfw, is_t = false, rows = 1, cols = d;
  else if (name == "final_norm.bias") base = lnfb, is_t = false, rows = 1, cols = d;
  else if (name == "scalar_head.weight") base = head, is_t = false, rows = 1, cols = d;
  else {
    const size_t dot = name.find('.', 7);
    const Layer& ly = layers[std::stoll(name.substr(7, dot - 7))];
    const std::string rest = name.substr(dot + 1);
    tr = true;
    if (rest == "attn_norm.weight") base = ly.ln1w, is_t = tr = false, rows = 1, cols = d;
    else if (rest == "attn_norm.bias") base = ly.ln1b, is_t = tr = false, rows = 1, cols = d;
    else if (rest == "ffn_norm.weight") base = ly.ln2w, is_t = tr = false, rows = 1, cols = d;
    else if (rest == "ffn_norm.bias") base = ly.ln2b, is_t = tr = false, rows = 1, cols = d;
    else if (rest == "attn.q_proj.weight") base = ly.wqkv, rows = d, cols = d, row0 = 0;
    else if (rest == "attn.k_proj.weight") base = ly.wqkv, rows = d, cols = d, row0 = d;
    else if (rest == "attn.v_proj.weight") base = ly.wqkv, rows = d, cols = d, row0 = 2 * d;
    else if (rest == "attn.o_proj.weight") base = ly.wo, rows = d, cols = d;
    else if (rest == "ffn.up_proj.weight") base = ly.wup, rows = f, cols = d;
    else if (rest == "ffn.down_proj.weight") base = ly.wdown, rows = d, cols = f;
  }
  const size_t esz = is_t ? tsize() : 4;
  std::vector<uint8_t> h(size_t(rows) * cols * esz);
  PPOEXP_CUDA(cudaStreamSynchronize(ctx->stream));
  PPOEXP_CUDA(cudaMemcpy(h.data(), static_cast<const uint8_t*>(base) + size_t(row0) * cols * esz, h.size(),
                         cudaMemcpyDeviceToHost));
  auto at = [&](int64_t i) -> double {
    if (!is_t || dtype == PPOEXP_F32) return reinterpret_cast<const float*>(h.data())[i];
    uint32_t u = uint32_t(reinterpret_cast<const uint16_t*>(h.data())[i]) << 16;
    float v;
    std::memcpy(&v, &u, 4);
    return v;
  };
  // stored [rows=out, cols=in] (W^T) when tr: reference element [i][o] = stored[o][i]
  for (int64_t e = 0; e < want; ++e) {
    const int64_t si = tr ? (e % rows) * cols + e / rows : e;
    const double v = at(si);
    if (out_dtype == PPOEXP_F64)
      static_cast<double*>(out)[e] = v;
    else
      static_cast<float*>(out)[e] = float(v);
  }
}

// ------------------------------------------------------------------ packing
void pack_metadata(Ctx& c, Packed& p, const std::string& tag) {
  p.B = static_cast<int64_t>(p.offsets.size()) - 1;
  p.M = p.offsets.back();
  p.max_len = 0;
  std::vector<int32_t> pos(p.M), sor(p.M);
  for (int64_t b = 0; b < p.B; ++b) {
    const int64_t n = p.offsets[b + 1] - p.offsets[b];
    p.max_len = std::max(p.max_len, n);
    for (int64_t t = 0; t < n; ++t) {
      pos[p.offsets[b] + t] = static_cast<int32_t>(t);
      sor[p.offsets[b] + t] = static_cast<int32_t>(b);
    }
  }
  const size_t ob = (p.B + 1) * 8, mb = p.M * 4;
  char* h = static_cast<char*>(c.pinned_staging(ob + 2 * mb + 64));
  std::memcpy(h, p.offsets.data(), ob);
  std::memcpy(h + ob, pos.data(), mb);
  std::memcpy(h + ob + mb, sor.data(), mb);
  char* dbuf = static_cast<char*>(c.workspace(tag + ".meta", ob + 2 * mb + 64));
  PPOEXP_CUDA(cudaMemcpyAsync(dbuf, h, ob + 2 * mb, cudaMemcpyHostToDevice, c.stream));
  p.offsets_d = reinterpret_cast<int64_t*>(dbuf);
  p.positions_d = reinterpret_cast<int32_t*>(dbuf + ob);
  p.seq_of_row_d = reinterpret_cast<int32_t*>(dbuf + ob + mb);
  // the pinned staging is reused by later calls: make the copy complete
  PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
}

// ------------------------------------------------------------------ GEMM
template <class T>
void launch_gemm_simt(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc);
bool gemm_tc_bf16(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                  Epi epi, void* C, int64_t ldc);

template <class T>
void gemm(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K, Epi epi,
          void* C, int64_t ldc) {
  if constexpr (std::is_same_v<T, bf16>) {
    if (gemm_tc_bf16(c, A, lda, B, ldb, M, N, K, epi, C, ldc)) return;
  }
  launch_gemm_simt<T>(c, A, lda, B, ldb, M, N, K, epi, C, ldc);
}
template void gemm<float>(Ctx&, const float*, int64_t, const float*, int64_t, int64_t, int64_t, int64_t, Epi, void*,
                          int64_t);
template void gemm<bf16>(Ctx&, const bf16*, int64_t, const bf16*, int64_t, int64_t, int64_t, int64_t, Epi, void*,
                         int64_t);

// ------------------------------------------------------------------ forward
template <class T>
static float* forward_layers_t(Model& m, const Packed& p, const KvTarget* kv) {
  Ctx& c = *m.ctx;
  const int64_t M = p.M, d = m.d(), f = m.cfg.d_ff, H = m.cfg.n_heads, DH = m.dh();
  float* x = static_cast<float*>(c.workspace("fwd.x", M * d * 4));
  T* h = static_cast<T*>(c.workspace("fwd.h", M * d * sizeof(T)));
  T* qkv = static_cast<T*>(c.workspace("fwd.qkv", M * 3 * d * sizeof(T)));
  T* att = static_cast<T*>(c.workspace("fwd.att", M * d * sizeof(T)));
  T* up = static_cast<T*>(c.workspace("fwd.up", M * f * sizeof(T)));
  launch_embed<T>(c, p.tokens_d, p.positions_d, M, d, static_cast<const T*>(m.tok), static_cast<const T*>(m.pos), x);
  for (int64_t l = 0; l < m.cfg.n_layers; ++l) {
    const Layer& ly = m.layers[l];
    launch_layernorm<T>(c, x, M, d, ly.ln1w, ly.ln1b, h, nullptr, nullptr, nullptr);
    gemm<T>(c, h, d, static_cast<const T*>(ly.wqkv), d, M, 3 * d, d, Epi::kStore, qkv, 3 * d);
    if (kv)
      launch_kv_scatter<T>(c, qkv, M, d, p.seq_of_row_d, p.positions_d, kv->block_table, int(l), kv->geom,
                           static_cast<T*>(kv->pool));
    bool done = false;
    if constexpr (std::is_same_v<T, bf16>) done = attention_prefill_tc(c, qkv, p.offsets_d, p.B, p.max_len, H, DH, M, att);
    if (!done) launch_attention_prefill<T>(c, qkv, p.offsets_d, p.B, p.max_len, H, DH, att);
    gemm<T>(c, att, d, static_cast<const T*>(ly.wo), d, M, d, d, Epi::kAddResidual, x, d);
    launch_layernorm<T>(c, x, M, d, ly.ln2w, ly.ln2b, h, nullptr, nullptr, nullptr);
    gemm<T>(c, h, d, static_cast<const T*>(ly.wup), d, M, f, d, Epi::kGelu, up, f);
    gemm<T>(c, up, f, static_cast<const T*>(ly.wdown), f, M, d, f, Epi::kAddResidual, x, d);
  }
  return x;
}

// Mixed mode: bf16 weights, fp32 activations / KV, split-bf16 tensor-core GEMMs.
// Mixed-mode prefill / scoring GEMMs: the in-kernel fp32 -> hi|lo split
// (gemm_mixed.cu) measured faster than plane operands written by the producers
// (C2 scoring: 32.2 vs 36.5 ms of GEMM time per step, + 2.3 ms of split
// LayerNorms); PPOEXP_PREFILL_PLANES=1 selects the planes.  The LM head takes the
// planes (LSE epilogue: 5.9 -> 4.7 ms) unless PPOEXP_MIXED_PLANES=0.
static bool mixed_prefill_planes() {
  // default with the persistent planes GEMM (gemm_persist.cu: 2x the in-kernel
  // split's throughput at the C2 scoring shapes); PPOEXP_PREFILL_PLANES=0 keeps
  // fp32 activations split inside gemm_mixed
  static const bool on = [] {
    const char* e = getenv("PPOEXP_PREFILL_PLANES");
    return e ? e[0] == '1' : gemm_pp_enabled();
  }();
  return on;
}
static bool mixed_head_planes() {
  static const bool on = [] {
    const char* e = getenv("PPOEXP_MIXED_PLANES");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool split_attention_tc() {  // PPOEXP_ATTN_SPLIT_TC=0 (or PPOEXP_ATTN_TC=0): mma.sync split attention
  static const bool on = [] {
    const char* e = getenv("PPOEXP_ATTN_SPLIT_TC");
    const char* t = getenv("PPOEXP_ATTN_TC");
    return !(e && e[0] == '0') && !(t && t[0] == '0');
  }();
  return on;
}

static float* forward_layers_mixed(Model& m, const Packed& p, const KvTarget* kv) {
  Ctx& c = *m.ctx;
  const int64_t M = p.M, d = m.d(), f = m.cfg.d_ff, H = m.cfg.n_heads, DH = m.dh();
  float* x = static_cast<float*>(c.workspace("fwd.x", M * d * 4));
  float* h = static_cast<float*>(c.workspace("fwd.h", M * d * 4));
  float* qkv = static_cast<float*>(c.workspace("fwd.qkv", M * 3 * d * 4));
  float* att = static_cast<float*>(c.workspace("fwd.att", M * d * 4));
  float* up = static_cast<float*>(c.workspace("fwd.up", M * f * 4));
  launch_embed<bf16>(c, p.tokens_d, p.positions_d, M, d, static_cast<const bf16*>(m.tok),
                     static_cast<const bf16*>(m.pos), x);
  if (mixed_prefill_planes() && d <= 4096) {
    // activations as hi | lo bf16 planes [M, 2K] written by their producers (split
    // LayerNorm, attention output, GELU epilogue) and TMA'd by the GEMMs: no
    // fp32 -> bf16 conversion inside the GEMM main loops
    bf16* hp = reinterpret_cast<bf16*>(h);
    bf16* ap = reinterpret_cast<bf16*>(att);
    bf16* upp = reinterpret_cast<bf16*>(up);
    // the KV-scattering prefill (engine) keeps fp32 q / k / v for the cache
    const bool qkv_planes = !kv && (DH == 64 || DH == 128) && M > 128 && gemm_pp_enabled() && split_attention_tc();
    for (int64_t l = 0; l < m.cfg.n_layers; ++l) {
      const Layer& ly = m.layers[l];
      launch_layernorm_split(c, x, M, d, ly.ln1w, ly.ln1b, hp);
      if (qkv_planes) {
        // scoring: q / k / v as planes [M, 6d] (in the fp32 [M, 3d] buffer) for
        // the split tcgen05 flash attention, which writes the O operand as planes
        bf16* qp = reinterpret_cast<bf16*>(qkv);
        gemm_tc_planes(c, hp, 2 * d, static_cast<const bf16*>(ly.wqkv), d, M, 3 * d, d, Epi::kStoreSplit, qp, 6 * d);
        if (!attention_prefill_tc_split(c, qp, p.offsets_d, p.B, p.max_len, H, DH, M, ap))
          throw ContractError("forward (mixed): split tcgen05 attention not eligible for this shape");
      } else {
        gemm_tc_planes(c, hp, 2 * d, static_cast<const bf16*>(ly.wqkv), d, M, 3 * d, d, Epi::kStoreF32, qkv, 3 * d);
        if (kv)
          launch_kv_scatter<float>(c, qkv, M, d, p.seq_of_row_d, p.positions_d, kv->block_table, int(l), kv->geom,
                                   static_cast<float*>(kv->pool));
        attention_prefill_split(c, qkv, p.offsets_d, p.B, p.max_len, H, DH, nullptr, ap);
      }
      gemm_tc_planes(c, ap, 2 * d, static_cast<const bf16*>(ly.wo), d, M, d, d, Epi::kAddResidual, x, d);
      launch_layernorm_split(c, x, M, d, ly.ln2w, ly.ln2b, hp);
      gemm_tc_planes(c, hp, 2 * d, static_cast<const bf16*>(ly.wup), d, M, f, d, Epi::kGeluSplit, upp, 2 * f);
      gemm_tc_planes(c, upp, 2 * f, static_cast<const bf16*>(ly.wdown), f, M, d, f, Epi::kAddResidual, x, d);
    }
    return x;
  }
  for (int64_t l = 0; l < m.cfg.n_layers; ++l) {
    const Layer& ly = m.layers[l];
    launch_layernorm<float>(c, x, M, d, ly.ln1w, ly.ln1b, h, nullptr, nullptr, nullptr);
    gemm_mixed(c, h, d, static_cast<const bf16*>(ly.wqkv), d, M, 3 * d, d, Epi::kStoreF32, qkv, 3 * d);
    if (kv)
      launch_kv_scatter<float>(c, qkv, M, d, p.seq_of_row_d, p.positions_d, kv->block_table, int(l), kv->geom,
                               static_cast<float*>(kv->pool));
    attention_prefill_split(c, qkv, p.offsets_d, p.B, p.max_len, H, DH, att);
    gemm_mixed(c, att, d, static_cast<const bf16*>(ly.wo), d, M, d, d, Epi::kAddResidual, x, d);
    launch_layernorm<float>(c, x, M, d, ly.ln2w, ly.ln2b, h, nullptr, nullptr, nullptr);
    gemm_mixed(c, h, d, static_cast<const bf16*>(ly.wup), d, M, f, d, Epi::kGeluF32, up, f);
    gemm_mixed(c, up, f, static_cast<const bf16*>(ly.wdown), f, M, d, f, Epi::kAddResidual, x, d);
  }
  return x;
}

float* forward_layers(Model& m, const Packed& p, const KvTarget* kv) {
  if (p.M <= 0) return nullptr;
  if (p.max_len > m.cfg.max_seq_len)
    throw ContractError("forward: sequence length " + std::to_string(p.max_len) + " exceeds max_seq_len " +
                        std::to_string(m.cfg.max_seq_len));
  if (m.mixed()) return forward_layers_mixed(m, p, kv);
  return m.dtype == PPOEXP_F32 ? forward_layers_t<float>(m, p, kv) : forward_layers_t<bf16>(m, p, kv);
}

// ------------------------------------------------------------------ scoring
// The LM head runs with the fused log-sum-exp + gather epilogue (Epi::kLse in
// gemm_tc.cu / gemm_mixed.cu): fp32 logits stay in registers, only one (max,
// sum) pair per 256-column tile per row reaches HBM.  PPOEXP_SCORING=logits
// instead materialises fp32 logits and runs K9 (logprob_gather).
static bool fused_scoring() {
  static const bool on = [] {
    const char* e = getenv("PPOEXP_SCORING");
    return !(e && std::string(e) == "logits");
  }();
  return on;
}

static void score_logprobs_fused(Model& m, const float* x, const int32_t* gather, const int32_t* target,
                                 const int64_t* out_index, int64_t R, double* out) {
  Ctx& c = *m.ctx;
  const int64_t d = m.d(), V = m.cfg.vocab_size;
  const int nt = lse_tiles(V);
  const int ldp = (nt + 1) / 2 * 2;
  // rows per chunk: partials <= ~1 GiB
  const int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(R, (int64_t(1) << 30) / (ldp * 8)));
  const int64_t cr = std::min(chunk, R);
  float2* part = static_cast<float2*>(c.workspace("score.part", cr * ldp * 8));
  float* tl = static_cast<float*>(c.workspace("score.tgt", cr * 4));
  const bool mx = m.mixed();  // fp32 final LayerNorm + split-activation LM head
  void* hf = c.workspace("score.hf", cr * d * (mx ? 4 : 2));
  for (int64_t r0 = 0; r0 < R; r0 += chunk) {
    const int64_t n = std::min(chunk, R - r0);
    LseEpi e;
    e.target = target + r0;
    e.tgt_logit = tl;
    e.part = part;
    e.ldp = ldp;
    if (mx && mixed_head_planes() && d <= 4096) {
      launch_layernorm_split(c, x, n, d, m.lnfw, m.lnfb, static_cast<bf16*>(hf), gather + r0);
      gemm_tc_planes(c, static_cast<bf16*>(hf), 2 * d, static_cast<const bf16*>(m.tok), d, n, V, d, Epi::kLse, nullptr,
                     0, &e);
    } else if (mx) {
      launch_layernorm<float>(c, x, n, d, m.lnfw, m.lnfb, static_cast<float*>(hf), gather + r0, nullptr, nullptr);
      gemm_mixed(c, static_cast<float*>(hf), d, static_cast<const bf16*>(m.tok), d, n, V, d, Epi::kLse, nullptr, 0, &e);
    } else {
      launch_layernorm<bf16>(c, x, n, d, m.lnfw, m.lnfb, static_cast<bf16*>(hf), gather + r0, nullptr, nullptr);
      if (!gemm_tc_lse(c, static_cast<bf16*>(hf), d, static_cast<const bf16*>(m.tok), d, n, V, d, e))
        throw ContractError("scoring: fused LM head needs 16-byte aligned rows (d_model % 8 == 0)");
    }
    launch_lse_combine(c, part, ldp, nt, tl, target + r0, n, out_index + r0, out);
  }
}

template <class T>
static void score_logprobs_t(Model& m, const float* x, const int32_t* gather, const int32_t* target,
                             const int64_t* out_index, int64_t R, double* out) {
  Ctx& c = *m.ctx;
  if constexpr (std::is_same_v<T, bf16>) {
    if (fused_scoring()) return score_logprobs_fused(m, x, gather, target, out_index, R, out);
  }
  const int64_t d = m.d(), V = m.cfg.vocab_size, ld = m.vpad;
  // logits are streamed in row chunks of <= ~2 GiB
  const int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(R, (int64_t(2) << 30) / (ld * sizeof(float))));
  T* hf = static_cast<T*>(c.workspace("score.hf", std::min(chunk, R) * d * sizeof(T)));
  // fp32 logits in both modes (bf16 logits would add |l|*2^-9 to every log-prob)
  float* logits = static_cast<float*>(c.workspace("score.logits", std::min(chunk, R) * ld * sizeof(float)));
  for (int64_t r0 = 0; r0 < R; r0 += chunk) {
    const int64_t n = std::min(chunk, R - r0);
    launch_layernorm<T>(c, x, n, d, m.lnfw, m.lnfb, hf, gather + r0, nullptr, nullptr);
    gemm<T>(c, hf, d, static_cast<const T*>(m.tok), d, n, V, d, Epi::kStoreF32, logits, ld);
    launch_logprob_gather<float>(c, logits, ld, n, V, target + r0, out_index + r0, out);
  }
}

void score_logprobs(Model& m, const Packed&, const float* x, const int32_t* gather, const int32_t* target,
                    const int64_t* out_index, int64_t R, double* out) {
  if (R <= 0) return;
  if (m.mixed())
    score_logprobs_fused(m, x, gather, target, out_index, R, out);
  else if (m.dtype == PPOEXP_F32)
    score_logprobs_t<float>(m, x, gather, target, out_index, R, out);
  else
    score_logprobs_t<bf16>(m, x, gather, target, out_index, R, out);
}

void score_head(Model& m, const float* x, const int32_t* gather, const int64_t* out_index, int64_t R, double* out) {
  if (R <= 0) return;
  if (!m.cfg.scalar_head) throw ContractError("model has no scalar head");
  Ctx& c = *m.ctx;
  float* vals = static_cast<float*>(c.workspace("score.vals", R * 4));
  if (m.dtype == PPOEXP_F32 || m.mixed())
    launch_layernorm<float>(c, x, R, m.d(), m.lnfw, m.lnfb, (float*)nullptr, gather, m.head, vals);
  else
    launch_layernorm<bf16>(c, x, R, m.d(), m.lnfw, m.lnfb, (bf16*)nullptr, gather, m.head, vals);
  launch_scatter_f32_f64(c, vals, out_index, R, out);
}

// ------------------------------------------------------------------ helpers
__global__ void scatter_f32_f64_kernel(const float* src, const int64_t* index, int64_t n, double* dst) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[index ? index[i] : i] = double(src[i]);
}

void launch_scatter_f32_f64(Ctx& c, const float* src, const int64_t* index, int64_t n, double* dst) {
  if (n <= 0) return;
  c.launch("convert", 20.0 * n, 0, [&] {
    launch_kernel(c, scatter_f32_f64_kernel, dim3(std::min<int64_t>(ceil_div(n, 256), 1184)), dim3(256), 0, 1, src, index, n, dst);
  });
}

// PPO response rows: for response token t of sequence b, the logits row is the
// prefix position P_b - 1 + t (src/ppo.cpp:282-287 keeps positions >= P).
__global__ void response_meta_kernel(int64_t B, const int64_t* offsets_full, const int64_t* prompt_len,
                                     const int64_t* resp_len, int64_t stride, const int32_t* tokens_full,
                                     int32_t* gather, int32_t* target, int64_t* out_index,
                                     const int64_t* resp_offsets) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  const int64_t n = resp_len[b], P = prompt_len[b], o = offsets_full[b], ro = resp_offsets[b];
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    gather[ro + t] = static_cast<int32_t>(o + P - 1 + t);
    if (target) target[ro + t] = tokens_full[o + P + t];
    out_index[ro + t] = b * stride + t;
  }
}

void launch_response_meta(Ctx& c, int64_t B, const int64_t* offsets_full, const int64_t* prompt_len,
                          const int64_t* resp_len, int64_t stride, const int32_t* tokens_full, int32_t* gather,
                          int32_t* target, int64_t* out_index, const int64_t* resp_offsets) {
  if (B <= 0) return;
  c.launch("meta", 0, 0, [&] {
    launch_kernel(c, response_meta_kernel, dim3(B), dim3(128), 0, 1, B, offsets_full, prompt_len, resp_len, stride, tokens_full, gather,
                                                   target, out_index, resp_offsets);
  });
}

__global__ void concat_pack_kernel(int64_t B, const int32_t* prompts, const int64_t* p_offsets, const int32_t* gen,
                                   int64_t gstride, const int64_t* gen_len, const int64_t* full_offsets,
                                   int32_t* full) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  const int64_t P = p_offsets[b + 1] - p_offsets[b], n = gen_len[b], o = full_offsets[b];
  for (int64_t t = threadIdx.x; t < P + n; t += blockDim.x)
    full[o + t] = t < P ? prompts[p_offsets[b] + t] : gen[b * gstride + (t - P)];
}

void launch_concat_pack(Ctx& c, int64_t B, const int32_t* prompts, const int64_t* p_offsets, const int32_t* gen,
                        int64_t gstride, const int64_t* gen_len, const int64_t* full_offsets, int32_t* full) {
  if (B <= 0) return;
  c.launch("pack", 0, 0, [&] {
    launch_kernel(c, concat_pack_kernel, dim3(B), dim3(256), 0, 1, B, prompts, p_offsets, gen, gstride, gen_len, full_offsets, full);
  });
}

}  // namespace ppx

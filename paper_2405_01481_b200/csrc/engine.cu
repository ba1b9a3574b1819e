// engine.cu — the rollout engine (Engine / generate_batch analog,
// include/aligner/engine.hpp:49-92, src/model.cpp:438-482).
//
//   * paged KV pool in HBM: pages of `page_size` tokens, one block table per
//     sequence, pages assigned per call for P_b + budget_b positions;
//   * batched prefill: all prompts in one packed forward that scatters K/V
//     into the pages and yields the last-position logits;
//   * decode: K steps (decode forward + fused sampler) captured in one CUDA
//     graph, replayed until every sequence has emitted EOT or exhausted its
//     budget; the host polls a done-counter one replay behind, so the GPU
//     queue never drains.
#include <algorithm>
#include <cstring>
#include <random>

#include "engine.hpp"

namespace ppx {

void dump_gemm_trace(Ctx& c, const char* path);  // gemm_decode.cu

namespace {
constexpr int kUnitsPerGraph = 8;
}

namespace {
// Issue work of one lane: its stream and workspace namespace for the scope.
struct LaneScope {
  Ctx* c;
  cudaStream_t s0;
  std::string p0;
  LaneScope(Ctx* cc, const Engine& e) : c(cc), s0(cc->stream), p0(cc->ws_prefix) {
    if (e.lane_stream) {
      c->stream = e.lane_stream;
      c->ws_prefix = e.lane_prefix;
    }
  }
  ~LaneScope() {
    c->stream = s0;
    c->ws_prefix = p0;
  }
};
}  // namespace

Engine::Engine(Model* model, const ppoexp_engine_options* o, Engine* owner_) : m(model), c(model->ctx), owner(owner_) {
  if (o) opts = *o;
  if (opts.max_batch <= 0) opts.max_batch = 256;
  if (opts.page_size <= 0) opts.page_size = 64;
  if (o == nullptr) opts.use_graphs = 1;
  const auto& cfg = m->cfg;
  const int64_t S = cfg.max_seq_len;
  if (opts.max_total_tokens <= 0) opts.max_total_tokens = opts.max_batch * S;
  geom.n_layers = cfg.n_layers;
  geom.page_size = opts.page_size;
  geom.H = cfg.n_heads;
  geom.DH = cfg.d_model / cfg.n_heads;
  geom.max_pages_per_seq = ceil_div(S, opts.page_size);
  geom.n_pages = std::max<int64_t>(ceil_div(opts.max_total_tokens, opts.page_size), geom.max_pages_per_seq);
  DeviceGuard g(c->device);
  if (m->mixed() && opts.max_batch > 256)
    throw ContractError("engine: mixed mode decodes at most 256 sequences per step (max_batch <= 256)");
  const size_t ts = m->asize();  // activation / KV element
  if (owner) {
    geom.n_pages = owner->geom.n_pages;  // lanes decode into the owner's pool
    kvp = owner->kvp;
  } else {
    kv.ensure(size_t(geom.n_layers) * geom.n_pages * 2 * geom.H * geom.page_size * geom.DH * ts);
    kvp = kv.ptr;
  }
  const int64_t mb = opts.max_batch, d = cfg.d_model, f = cfg.d_ff;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t sbytes = 0;
  const size_t o_next = sbytes; sbytes += al(mb * 4);
  const size_t o_pos = sbytes; sbytes += al(mb * 4);
  const size_t o_ngen = sbytes; sbytes += al(mb * 4);
  const size_t o_done = sbytes; sbytes += al(mb * 4);
  const size_t o_budget = sbytes; sbytes += al(mb * 4);
  const size_t o_nact = sbytes; sbytes += al(16);
  const size_t o_bt = sbytes; sbytes += al(mb * geom.max_pages_per_seq * 4);
  const size_t o_sp = sbytes; sbytes += al(mb * sizeof(SampleParams));
  const size_t o_x = sbytes; sbytes += al(mb * d * 4);
  const size_t o_h = sbytes; sbytes += al(mb * d * ts);
  const size_t o_qkv = sbytes; sbytes += al(mb * 3 * d * ts);
  const size_t o_att = sbytes; sbytes += al(mb * d * ts);
  const size_t o_up = sbytes; sbytes += al(mb * f * ts);
  const size_t o_logits = sbytes; sbytes += al(mb * m->vpad * 4);
  const size_t o_otok = sbytes; sbytes += al(mb * S * 4);
  const size_t o_olp = sbytes; sbytes += al(mb * S * 4);
  const size_t o_uni = sbytes; sbytes += al(mb * S * 8);
  const size_t o_last = sbytes; sbytes += al(mb * 4);
  // fused-LN row statistics: one accumulator pair per row for each LayerNorm of a step
  const size_t o_sta = sbytes; sbytes += al((2 * cfg.n_layers + 1) * mb * kStatStride * 8);
  const size_t o_ovf = sbytes; sbytes += al(16);
  state.ensure(sbytes);
  PPOEXP_CUDA(cudaMemset(state.ptr, 0, sbytes));
  char* p = static_cast<char*>(state.ptr);
  next_tok = reinterpret_cast<int32_t*>(p + o_next);
  pos = reinterpret_cast<int32_t*>(p + o_pos);
  n_gen = reinterpret_cast<int32_t*>(p + o_ngen);
  done = reinterpret_cast<int32_t*>(p + o_done);
  budget = reinterpret_cast<int32_t*>(p + o_budget);
  n_active = reinterpret_cast<int32_t*>(p + o_nact);
  block_table = reinterpret_cast<int32_t*>(p + o_bt);
  sparams = reinterpret_cast<SampleParams*>(p + o_sp);
  x = reinterpret_cast<float*>(p + o_x);
  h = p + o_h;
  qkv = p + o_qkv;
  att = p + o_att;
  up = p + o_up;
  logits = reinterpret_cast<float*>(p + o_logits);
  out_tok = reinterpret_cast<int32_t*>(p + o_otok);
  out_lp = reinterpret_cast<float*>(p + o_olp);
  uniforms = reinterpret_cast<double*>(p + o_uni);
  last_rows = reinterpret_cast<int32_t*>(p + o_last);
  stats = reinterpret_cast<unsigned long long*>(p + o_sta);
  stat_ovf = reinterpret_cast<unsigned*>(p + o_ovf);
  {
    // default for bf16 decode batches <= 64 (PPOEXP_FUSE_LN=0 disables, =1
    // forces it up to 256): removes 24 of the 25 LN launches of a decode step,
    // -6% step time at C2 on B200; at batch 256 every weight tile would
    // re-normalise 4x more rows and it measured 18% slower
    const char* ev = getenv("PPOEXP_FUSE_LN");
    fuse_ln = m->dtype == PPOEXP_BF16 && !(ev && ev[0] == '0') && mb <= 256 && d % 8 == 0;
    if (m->mixed() && d % 8) throw ContractError("engine: mixed mode needs d_model % 8 == 0");
    // mixed decode: split-plane activations TMA'd by the GEMMs (standalone split
    // LayerNorm, attention / GELU epilogues writing hi|lo planes) — measured
    // 754 -> 674 us per C2 step and 16.0 -> 13.2 ms per C4 step against the
    // in-kernel split (PPOEXP_MIXED_PLANES=0: LayerNorm fused into the consumers,
    // 2: planes for the O / down operands only)
    const char* pe = getenv("PPOEXP_MIXED_PLANES");
    mixed_planes = m->mixed() && (pe ? pe[0] == '1' : true) && d <= 4096;
    mixed_oplanes = m->mixed() && !mixed_planes && pe && pe[0] == '2';
    fuse_ln_max_b = ev && ev[0] == '1' ? 256 : 64;
  }
  PPOEXP_CUDA(cudaMallocHost(&host_flags, 64));
  PPOEXP_CUDA(cudaEventCreateWithFlags(&poll_ev[0], cudaEventDisableTiming));
  PPOEXP_CUDA(cudaEventCreateWithFlags(&poll_ev[1], cudaEventDisableTiming));
  PPOEXP_CUDA(cudaEventCreate(&t0));
  PPOEXP_CUDA(cudaEventCreate(&t1));
  PPOEXP_CUDA(cudaEventCreateWithFlags(&lane_ev, cudaEventDisableTiming));
  if (owner) {
    PPOEXP_CUDA(cudaStreamCreateWithFlags(&lane_stream, cudaStreamNonBlocking));
  } else if (m->dtype != PPOEXP_F32) {
    // two decode lanes by default for the tensor-core modes (PPOEXP_LANES=1 disables)
    const char* le = getenv("PPOEXP_LANES");
    n_lanes = le ? std::max(1, std::min(2, atoi(le))) : 2;
    if (const char* lm = getenv("PPOEXP_LANE_MIN_B")) lane_min_b = std::max<int64_t>(2, atoll(lm));
    if (n_lanes == 2 && opts.max_batch >= lane_min_b) {
      ppoexp_engine_options lo = opts;
      lo.max_batch = ceil_div(opts.max_batch, 2);
      for (int i = 0; i < 2; ++i) {
        lanes[i] = std::make_unique<Engine>(m, &lo, this);
        lanes[i]->lane_prefix = "lane" + std::to_string(i) + ".";
      }
    } else {
      n_lanes = 1;
    }
  }
}

Engine::~Engine() {
  DeviceGuard g(c->device, true);
  lanes[0].reset();
  lanes[1].reset();
  cudaStreamSynchronize(lane_stream ? lane_stream : c->stream);
  for (auto& [k, gs] : graphs)
    for (int j = 0; j < 2; ++j) {
      if (gs.exec[j]) cudaGraphExecDestroy(gs.exec[j]);
      for (auto& t : gs.events[j]) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
      }
    }
  if (host_flags) cudaFreeHost(host_flags);
  cudaEventDestroy(poll_ev[0]);
  cudaEventDestroy(poll_ev[1]);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaEventDestroy(lane_ev);
  if (lane_stream) cudaStreamDestroy(lane_stream);
}

SamplerState Engine::sampler_state() const {
  SamplerState s;
  s.params = sparams;
  s.next_tok = next_tok;
  s.pos = pos;
  s.n_gen = n_gen;
  s.done = done;
  s.budget = budget;
  s.uniforms = uniforms;
  s.ustride = m->cfg.max_seq_len;
  s.out_tokens = out_tok;
  s.out_lps = out_lp;
  s.ostride = m->cfg.max_seq_len;
  s.n_active = n_active;
  if (getenv("PPOEXP_SAMPLER_TRACE")) {
    auto* buf = static_cast<unsigned long long*>(c->workspace("sampler.trace", 16 * 8));
    s.dbg = buf;
  }
  return s;
}

// One decode unit: feed next_tok[b] at pos[b] through the model, then sample.
template <class T>
void Engine::decode_unit(int64_t B, int64_t unit) {
  Ctx& cc = *c;
  const int64_t d = m->d(), f = m->cfg.d_ff, V = m->cfg.vocab_size;
  T* hh = static_cast<T*>(h);
  T* q3 = static_cast<T*>(qkv);
  T* at = static_cast<T*>(att);
  T* uu = static_cast<T*>(up);
  cur_unit = unit;
  if constexpr (std::is_same_v<T, bf16>) {
    if (fuse_ln && B <= fuse_ln_max_b) {
      // bf16 path with LayerNorm fused into the consumer GEMMs: embed / O-proj /
      // down-proj accumulate fixed-point row statistics of x (one buffer per
      // LayerNorm of the step), QKV / up / LM head normalise their activation
      // slice on the fly (no standalone LayerNorm launches)
      const int64_t L = m->cfg.n_layers, mb = opts.max_batch;
      auto st = [&](int64_t i) { return stats + i * mb * kStatStride; };  // i = 2l (LN1), 2l+1 (LN2)
      RowStats s0{st(0), stat_ovf};
      s0.zero = st(1);
      s0.zero_n = (2 * L - 1) * mb;
      launch_embed_stats<T>(cc, next_tok, pos, B, d, static_cast<const T*>(m->tok), static_cast<const T*>(m->pos), x,
                            s0);
      for (int64_t l = 0; l < L; ++l) {
        const Layer& ly = m->layers[l];
        const LnIn l1{x, d, st(2 * l), ly.ln1w, ly.ln1b, int(d)};
        gemm_decode_fused(cc, nullptr, d, static_cast<const T*>(ly.wqkv), d, B, 3 * d, d, Epi::kStore, q3, 3 * d, &l1,
                          nullptr);
        launch_attention_decode<T>(cc, q3, B, pos, done, block_table, int(l), geom, static_cast<T*>(kvp), at, 0.0);
        const RowStats so2{st(2 * l + 1), stat_ovf};
        gemm_decode_fused(cc, at, d, static_cast<const T*>(ly.wo), d, B, d, d, Epi::kAddResidual, x, d, nullptr, &so2);
        const LnIn l2{x, d, st(2 * l + 1), ly.ln2w, ly.ln2b, int(d)};
        gemm_decode_fused(cc, nullptr, d, static_cast<const T*>(ly.wup), d, B, f, d, Epi::kGelu, uu, f, &l2, nullptr);
        const RowStats so1{st(2 * l + 2), stat_ovf};  // the last layer's down-proj feeds the standalone final LN
        gemm_decode_fused(cc, uu, f, static_cast<const T*>(ly.wdown), f, B, d, f, Epi::kAddResidual, x, d, nullptr,
                          l + 1 < L ? &so1 : nullptr);
      }
      // final LayerNorm standalone: the LM head has ~400 weight tiles, each of
      // which would re-normalise the whole activation (measured slower fused)
      launch_layernorm<T>(cc, x, B, d, m->lnfw, m->lnfb, hh, nullptr, nullptr, nullptr);
      gemm<T>(cc, hh, d, static_cast<const T*>(m->tok), d, B, V, d, Epi::kStoreF32, logits, m->vpad);
      launch_sampler(cc, logits, m->vpad, B, V, sampler_state());
      return;
    }
  }
  const bool fused_head = m->cfg.n_layers > 0 &&
                          launch_embed_layernorm<T>(cc, next_tok, pos, B, d, static_cast<const T*>(m->tok),
                                                    static_cast<const T*>(m->pos), x, m->layers[0].ln1w,
                                                    m->layers[0].ln1b, hh);
  if (!fused_head)
    launch_embed<T>(cc, next_tok, pos, B, d, static_cast<const T*>(m->tok), static_cast<const T*>(m->pos), x);
  for (int64_t l = 0; l < m->cfg.n_layers; ++l) {
    const Layer& ly = m->layers[l];
    if (l > 0 || !fused_head) launch_layernorm<T>(cc, x, B, d, ly.ln1w, ly.ln1b, hh, nullptr, nullptr, nullptr);
    gemm<T>(cc, hh, d, static_cast<const T*>(ly.wqkv), d, B, 3 * d, d, Epi::kStore, q3, 3 * d);
    launch_attention_decode<T>(cc, q3, B, pos, done, block_table, int(l), geom, static_cast<T*>(kvp), at, 0.0);
    gemm<T>(cc, at, d, static_cast<const T*>(ly.wo), d, B, d, d, Epi::kAddResidual, x, d);
    launch_layernorm<T>(cc, x, B, d, ly.ln2w, ly.ln2b, hh, nullptr, nullptr, nullptr);
    gemm<T>(cc, hh, d, static_cast<const T*>(ly.wup), d, B, f, d, Epi::kGelu, uu, f);
    gemm<T>(cc, uu, f, static_cast<const T*>(ly.wdown), f, B, d, f, Epi::kAddResidual, x, d);
  }
  launch_layernorm<T>(cc, x, B, d, m->lnfw, m->lnfb, hh, nullptr, nullptr, nullptr);
  gemm<T>(cc, hh, d, static_cast<const T*>(m->tok), d, B, V, d, Epi::kStoreF32, logits, m->vpad);
  launch_sampler(cc, logits, m->vpad, B, V, sampler_state());
}

// Mixed mode (bf16 weights, fp32 activations / KV): every projection runs on
// the split-activation decode GEMM (LayerNorm fused into QKV / up as in the
// bf16 path, fixed-point row statistics from the residual producers), fp32
// decode attention over the fp32 paged KV.
void Engine::decode_unit_mixed(int64_t B, int64_t unit) {
  Ctx& cc = *c;
  const int64_t d = m->d(), f = m->cfg.d_ff, V = m->cfg.vocab_size, L = m->cfg.n_layers, mb = opts.max_batch;
  float* q3 = static_cast<float*>(qkv);
  float* at = static_cast<float*>(att);
  float* uu = static_cast<float*>(up);
  float* hh = static_cast<float*>(h);
  cur_unit = unit;
  if (mixed_planes) {
    // activations reach the GEMMs as two bf16 planes [B, 2K] TMA'd by the consumers:
    // a standalone split LayerNorm (normalised once, not per weight tile), the
    // attention writing its output split, the up projection's GELU epilogue split
    bf16* hp = static_cast<bf16*>(h);   // [mb, 2d] in the fp32 [mb, d] buffer
    bf16* ap = static_cast<bf16*>(att);
    bf16* upp = static_cast<bf16*>(up);  // [mb, 2f]
    if (L == 0)
      launch_embed<bf16>(cc, next_tok, pos, B, d, static_cast<const bf16*>(m->tok), static_cast<const bf16*>(m->pos),
                         x);
    for (int64_t l = 0; l < L; ++l) {
      const Layer& ly = m->layers[l];
      if (l == 0)  // the step's embedding and the first LayerNorm in one launch
        launch_embed_layernorm_split(cc, next_tok, pos, B, d, static_cast<const bf16*>(m->tok),
                                     static_cast<const bf16*>(m->pos), x, ly.ln1w, ly.ln1b, hp);
      else
        launch_layernorm_split(cc, x, B, d, ly.ln1w, ly.ln1b, hp);
      gemm_decode_planes(cc, hp, 2 * d, static_cast<const bf16*>(ly.wqkv), d, B, 3 * d, d, Epi::kStoreF32, q3, 3 * d,
                         nullptr);
      launch_attention_decode<float>(cc, q3, B, pos, done, block_table, int(l), geom, static_cast<float*>(kvp), at,
                                     0.0, ap);
      gemm_decode_planes(cc, ap, 2 * d, static_cast<const bf16*>(ly.wo), d, B, d, d, Epi::kAddResidual, x, d, nullptr);
      launch_layernorm_split(cc, x, B, d, ly.ln2w, ly.ln2b, hp);
      gemm_decode_planes(cc, hp, 2 * d, static_cast<const bf16*>(ly.wup), d, B, f, d, Epi::kGeluSplit, upp, 2 * f,
                         nullptr);
      gemm_decode_planes(cc, upp, 2 * f, static_cast<const bf16*>(ly.wdown), f, B, d, f, Epi::kAddResidual, x, d,
                         nullptr);
    }
    launch_layernorm_split(cc, x, B, d, m->lnfw, m->lnfb, hp);
    gemm_decode_planes(cc, hp, 2 * d, static_cast<const bf16*>(m->tok), d, B, V, d, Epi::kStoreF32, logits, m->vpad,
                       nullptr);
    launch_sampler(cc, logits, m->vpad, B, V, sampler_state());
    return;
  }
  auto st = [&](int64_t i) { return stats + i * mb * kStatStride; };
  RowStats s0{st(0), stat_ovf};
  s0.zero = st(1);
  s0.zero_n = (2 * L - 1) * mb;
  launch_embed_stats<bf16>(cc, next_tok, pos, B, d, static_cast<const bf16*>(m->tok), static_cast<const bf16*>(m->pos),
                           x, s0);
  for (int64_t l = 0; l < L; ++l) {
    const Layer& ly = m->layers[l];
    const LnIn l1{x, d, st(2 * l), ly.ln1w, ly.ln1b, int(d)};
    gemm_decode_mixed(cc, nullptr, d, static_cast<const bf16*>(ly.wqkv), d, B, 3 * d, d, Epi::kStoreF32, q3, 3 * d,
                      &l1, nullptr);
    const RowStats so2{st(2 * l + 1), stat_ovf};
    const LnIn l2{x, d, st(2 * l + 1), ly.ln2w, ly.ln2b, int(d)};
    const RowStats so1{st(2 * l + 2), stat_ovf};
    if (mixed_oplanes) {  // O / down operands as bf16 planes from the attention / GELU epilogues
      bf16* ap = static_cast<bf16*>(att);
      bf16* upp = static_cast<bf16*>(up);
      launch_attention_decode<float>(cc, q3, B, pos, done, block_table, int(l), geom, static_cast<float*>(kvp), at,
                                     0.0, ap);
      gemm_decode_planes(cc, ap, 2 * d, static_cast<const bf16*>(ly.wo), d, B, d, d, Epi::kAddResidual, x, d, &so2);
      gemm_decode_mixed(cc, nullptr, d, static_cast<const bf16*>(ly.wup), d, B, f, d, Epi::kGeluSplit, upp, 2 * f, &l2,
                        nullptr);
      gemm_decode_planes(cc, upp, 2 * f, static_cast<const bf16*>(ly.wdown), f, B, d, f, Epi::kAddResidual, x, d,
                         l + 1 < L ? &so1 : nullptr);
      continue;
    }
    launch_attention_decode<float>(cc, q3, B, pos, done, block_table, int(l), geom, static_cast<float*>(kvp), at,
                                   0.0);
    gemm_decode_mixed(cc, at, d, static_cast<const bf16*>(ly.wo), d, B, d, d, Epi::kAddResidual, x, d, nullptr, &so2);
    gemm_decode_mixed(cc, nullptr, d, static_cast<const bf16*>(ly.wup), d, B, f, d, Epi::kGeluF32, uu, f, &l2, nullptr);
    gemm_decode_mixed(cc, uu, f, static_cast<const bf16*>(ly.wdown), f, B, d, f, Epi::kAddResidual, x, d, nullptr,
                      l + 1 < L ? &so1 : nullptr);
  }
  launch_layernorm<float>(cc, x, B, d, m->lnfw, m->lnfb, hh, nullptr, nullptr, nullptr);
  gemm_decode_mixed(cc, hh, d, static_cast<const bf16*>(m->tok), d, B, V, d, Epi::kStoreF32, logits, m->vpad, nullptr,
                    nullptr);
  launch_sampler(cc, logits, m->vpad, B, V, sampler_state());
}

void Engine::run_unit(int64_t B, int64_t unit) {
  if (m->mixed())
    decode_unit_mixed(B, unit);
  else if (m->dtype == PPOEXP_F32)
    decode_unit<float>(B, unit);
  else
    decode_unit<bf16>(B, unit);
}

Engine::GraphSet& Engine::graph_for(int64_t B, int units) {
  std::string sig;
  if (c->profiling) {
    sig = "prof:";
    for (const auto& k : c->profile_filter) sig += k + ",";
  }
  const int64_t key = B * 16 + units;
  auto it = graphs.find(key);
  if (it != graphs.end() && it->second.prof_sig == sig) return it->second;
  if (it != graphs.end()) {
    for (int j = 0; j < 2; ++j) {
      cudaGraphExecDestroy(it->second.exec[j]);
      for (auto& t : it->second.events[j]) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
      }
    }
    graphs.erase(it);
  }
  GraphSet& gs = graphs[key];
  gs.profiled = c->profiling;
  gs.prof_sig = sig;
  gs.units = units;
  for (int j = 0; j < 2; ++j) {
    cudaGraph_t graph;
    PPOEXP_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    c->capture_launches = 0;
    c->capture_events = &gs.events[j];
    try {
      for (int k = 0; k < gs.units; ++k) run_unit(B, k);
    } catch (...) {
      c->capturing = false;
      c->capture_events = nullptr;
      cudaStreamEndCapture(c->stream, &graph);
      throw;
    }
    c->capturing = false;
    c->capture_events = nullptr;
    PPOEXP_CUDA(cudaStreamEndCapture(c->stream, &graph));
    PPOEXP_CUDA(cudaGraphInstantiate(&gs.exec[j], graph, 0));
    PPOEXP_CUDA(cudaGraphDestroy(graph));
    gs.nodes = c->capture_launches;
    // the per-launch events created during capture are owned by the graph set
  }
  return gs;
}

// Attribute the algorithmic bytes of each decode-attention launch of a
// finished replay: unit u feeds sequence b iff u <= n_b - 1, over a context
// of P_b + u positions (K and V, all heads), plus the appended row.
void Engine::harvest_replay(const std::vector<TimedLaunch>& evs, int64_t unit0, int units) {
  if (!c->profiling) return;
  const int64_t d = m->d();
  const double ts = double(m->asize());
  int64_t per_unit = 0;
  for (auto& t : evs)
    if (t.cls == "decode_attention") ++per_unit;
  per_unit /= std::max(units, 1);
  int64_t seen = 0;
  for (auto& t : evs) {
    TimedLaunch tt = t;
    if (t.cls == "decode_attention") {
      const int64_t u = unit0 + seen / std::max<int64_t>(per_unit, 1);
      ++seen;
      double bytes = 0;
      for (size_t b = 0; b < cur_P.size(); ++b)
        if (u <= cur_len[b] - 1) bytes += (double(cur_P[b] + u) * 2.0 + 2.0) * d * ts;
      tt.bytes = bytes;
    }
    c->harvest_list({tt}, false);
  }
}

void Engine::generate(int64_t B, const int32_t* prompts, const int64_t* offsets, const int64_t* max_new,
                      const ppoexp_sampling* sampling, const uint64_t* seeds, int64_t out_stride,
                      int32_t* out_tokens, double* out_logprobs, int64_t* out_lengths, int where, double* ms_out,
                      int where_out, int where_tokens) {
  if (where_out < 0) where_out = where;
  if (where_tokens < 0) where_tokens = where;
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  DeviceGuard g(c->device);
  if (B < 0) throw ContractError("generate_batch: negative batch");
  if (B == 0) {
    if (ms_out) *ms_out = 0;
    return;
  }
  if (!sampling) throw ContractError("generate: sampling specs required");
  const auto& cfg = m->cfg;
  const int64_t S = cfg.max_seq_len;
  // host copies of the small per-task arrays
  std::vector<int64_t> off(B + 1), mx(B);
  std::vector<uint64_t> sd(B, 0);
  if (where == PPOEXP_HOST) {
    std::memcpy(off.data(), offsets, (B + 1) * 8);
    std::memcpy(mx.data(), max_new, B * 8);
    if (seeds) std::memcpy(sd.data(), seeds, B * 8);
  } else {
    PPOEXP_CUDA(cudaMemcpy(off.data(), offsets, (B + 1) * 8, cudaMemcpyDeviceToHost));
    PPOEXP_CUDA(cudaMemcpy(mx.data(), max_new, B * 8, cudaMemcpyDeviceToHost));
    if (seeds) PPOEXP_CUDA(cudaMemcpy(sd.data(), seeds, B * 8, cudaMemcpyDeviceToHost));
  }
  if (off[0] != 0) throw ContractError("generate: offsets[0] must be 0");
  for (int64_t b = 0; b < B; ++b) {
    const int64_t P = off[b + 1] - off[b];
    if (P <= 0) throw ContractError("generate: prompt must be nonempty");
    if (P > S) throw ContractError("generate: sequence length exceeds max_seq_len " + std::to_string(S));
    if (mx[b] < 0) throw ContractError("generate: max_new must be >= 0");
  }
  // host ids scanned here; device ids by a validation kernel (IndexError before any use)
  check_tokens(*c, prompts, off[B], cfg.vocab_size, where_tokens < 0 ? where : where_tokens, "generate");
  last_lengths.assign(B, 0);
  cudaEvent_t e0 = t0, e1 = t1;
  PPOEXP_CUDA(cudaEventRecord(e0, c->stream));
  for (int64_t b0 = 0; b0 < B; b0 += opts.max_batch) {
    const int64_t nb = std::min<int64_t>(opts.max_batch, B - b0);
    run_chunk(nb, prompts, off, b0, mx, sampling, sd, out_stride, out_tokens, out_logprobs, out_lengths, where,
              where_out, where_tokens);
  }
  PPOEXP_CUDA(cudaEventRecord(e1, c->stream));
  PPOEXP_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  PPOEXP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  last_ms = ms;
  gen_seconds += ms / 1000.0;
  if (ms_out) *ms_out = ms;
  if (const char* gp = getenv("PPOEXP_GEMM_TRACE")) dump_gemm_trace(*c, gp);
  if (const char* ap = getenv("PPOEXP_ATTN_TRACE")) {  // debug: last decode-attention launch, CTA (0, 0)
    unsigned long long hh[16];
    PPOEXP_CUDA(cudaMemcpy(hh, c->workspace("attn.trace", 16 * 8), sizeof(hh), cudaMemcpyDeviceToHost));
    if (FILE* fp = fopen(ap, "w")) {
      const char* nm[6] = {"entry", "state+early tile", "pdl wait", "append+q", "tile loop", "merge+store"};
      for (int k = 1; k < 6; ++k)
        fprintf(fp, "%-18s %8.2f us\n", nm[k], hh[k] > hh[k - 1] ? (hh[k] - hh[k - 1]) / 1965.0 : 0.0);
      fprintf(fp, "context %llu\n", hh[6]);
      fclose(fp);
    }
  }
  if (const char* sp = getenv("PPOEXP_SAMPLER_TRACE")) {  // debug: last sampler launch, row 0
    unsigned long long h[16];
    PPOEXP_CUDA(cudaMemcpy(h, c->workspace("sampler.trace", 16 * 8), sizeof(h), cudaMemcpyDeviceToHost));
    if (FILE* fp = fopen(sp, "w")) {
      const char* nm[8] = {"entry", "pass1 max", "pass2 q+hist", "Z", "confirm", "collect+sort", "threshold", "cdf+pick"};
      for (int k = 1; k < 8; ++k)
        fprintf(fp, "%-14s %8.2f us\n", nm[k], h[k] > h[k - 1] ? (h[k] - h[k - 1]) / 1965.0 : 0.0);
      fprintf(fp, "total %.2f us, crossing-bucket members %llu\n", (h[7] - h[0]) / 1965.0, h[8]);
      fclose(fp);
    }
  }
  c->harvest();
}

int64_t Engine::chunk_pages(int64_t B, const std::vector<int64_t>& off_all, int64_t b0,
                            const std::vector<int64_t>& mx_all) const {
  const int64_t S = m->cfg.max_seq_len, PS = geom.page_size;
  int64_t pages = 0;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t P = off_all[b0 + b + 1] - off_all[b0 + b];
    pages += ceil_div(P + std::min<int64_t>(mx_all[b0 + b], S - std::min<int64_t>(P, S)), PS);
  }
  return pages;
}

void Engine::run_chunk(int64_t B, const int32_t* prompts, const std::vector<int64_t>& off_all, int64_t b0,
                       const std::vector<int64_t>& mx_all, const ppoexp_sampling* sp_all,
                       const std::vector<uint64_t>& seeds_all, int64_t out_stride, int32_t* out_tokens,
                       double* out_logprobs, int64_t* out_lengths, int where, int where_out, int where_tokens) {
  (void)where;
  if (n_lanes < 2 || B < lane_min_b) {
    Run run;
    chunk_begin(run, B, prompts, off_all, b0, mx_all, sp_all, seeds_all, out_stride, out_tokens, out_logprobs,
                out_lengths, where_out, where_tokens, 0);
    while (run.active) {
      chunk_launch(run);
      chunk_poll(run);
    }
    chunk_finish(run);
    return;
  }
  // two lanes: the first half of the chunk on lane 0, the rest on lane 1, each
  // on its own stream after the work already queued on the context stream
  const int64_t h0 = (B + 1) / 2;
  const int64_t p0 = lanes[0]->chunk_pages(h0, off_all, b0, mx_all);
  if (p0 + lanes[1]->chunk_pages(B - h0, off_all, b0 + h0, mx_all) > geom.n_pages)
    throw ContractError("engine: KV pool too small for the batch; raise max_total_tokens");
  PPOEXP_CUDA(cudaEventRecord(lane_ev, c->stream));
  for (auto& ln : lanes) PPOEXP_CUDA(cudaStreamWaitEvent(ln->lane_stream, lane_ev, 0));
  Run r0, r1;
  lanes[0]->chunk_begin(r0, h0, prompts, off_all, b0, mx_all, sp_all, seeds_all, out_stride, out_tokens, out_logprobs,
                        out_lengths, where_out, where_tokens, 0);
  lanes[1]->chunk_begin(r1, B - h0, prompts, off_all, b0 + h0, mx_all, sp_all, seeds_all, out_stride, out_tokens,
                        out_logprobs, out_lengths, where_out, where_tokens, p0);
  while (r0.active || r1.active) {
    lanes[0]->chunk_launch(r0);
    lanes[1]->chunk_launch(r1);
    lanes[0]->chunk_poll(r0);
    lanes[1]->chunk_poll(r1);
  }
  lanes[0]->chunk_finish(r0);
  lanes[1]->chunk_finish(r1);
  for (auto& ln : lanes) {
    PPOEXP_CUDA(cudaEventRecord(ln->lane_ev, ln->lane_stream));
    PPOEXP_CUDA(cudaStreamWaitEvent(c->stream, ln->lane_ev, 0));
  }
}

void Engine::chunk_begin(Run& run, int64_t B, const int32_t* prompts, const std::vector<int64_t>& off_all, int64_t b0,
                         const std::vector<int64_t>& mx_all, const ppoexp_sampling* sp_all,
                         const std::vector<uint64_t>& seeds_all, int64_t out_stride, int32_t* out_tokens,
                         double* out_logprobs, int64_t* out_lengths, int where_out, int where_tokens,
                         int64_t page_base) {
  LaneScope ls(c, *this);
  Ctx& cc = *c;
  const auto& cfg = m->cfg;
  const int64_t S = cfg.max_seq_len, PS = geom.page_size, d = m->d();
  std::vector<int64_t> P(B), bud(B);
  int64_t max_budget = 0, pages = 0;
  for (int64_t b = 0; b < B; ++b) {
    P[b] = off_all[b0 + b + 1] - off_all[b0 + b];
    bud[b] = std::min<int64_t>(mx_all[b0 + b], S - std::min<int64_t>(P[b], S));  // src/model.cpp:447-448
    max_budget = std::max(max_budget, bud[b]);
    pages += ceil_div(P[b] + bud[b], PS);
  }
  if (page_base + pages > geom.n_pages)
    throw ContractError("engine: KV pool too small (" + std::to_string(pages) + " pages needed, " +
                        std::to_string(geom.n_pages) + " available); raise max_total_tokens");
  // block tables: contiguous page runs per sequence
  std::vector<int32_t> bt(B * geom.max_pages_per_seq, 0);
  int64_t next_page = page_base;
  for (int64_t b = 0; b < B; ++b) {
    const int64_t np = ceil_div(P[b] + bud[b], PS);
    for (int64_t k = 0; k < np; ++k) bt[b * geom.max_pages_per_seq + k] = int32_t(next_page++);
  }
  // state
  std::vector<int32_t> st_pos(B), st_done(B), st_bud(B), last(B);
  int32_t active = 0;
  for (int64_t b = 0; b < B; ++b) {
    st_pos[b] = int32_t(std::min<int64_t>(P[b], S - 1));
    st_done[b] = bud[b] == 0;
    st_bud[b] = int32_t(bud[b]);
    last[b] = int32_t(off_all[b0 + b + 1] - off_all[b0] - 1);
    active += bud[b] > 0;
  }
  std::vector<SampleParams> spd(B);
  bool any_sampled = false;
  for (int64_t b = 0; b < B; ++b) {
    const ppoexp_sampling& sp = sp_all[b0 + b];
    spd[b] = SampleParams{sp.greedy, float(sp.temperature), sp.top_k, sp.top_p};
    any_sampled |= !sp.greedy;
  }
  // staging (pinned) → device
  const size_t n_bt = bt.size() * 4;
  const size_t need = n_bt + 5 * B * 16 + B * sizeof(SampleParams) + 256 + (any_sampled ? size_t(B) * S * 8 : 0);
  char* hs = static_cast<char*>(cc.pinned_staging(need));
  size_t o = 0;
  auto put = [&](void* dst, const void* src, size_t n) {
    std::memcpy(hs + o, src, n);
    PPOEXP_CUDA(cudaMemcpyAsync(dst, hs + o, n, cudaMemcpyHostToDevice, cc.stream));
    o += (n + 15) / 16 * 16;
  };
  put(block_table, bt.data(), n_bt);
  put(pos, st_pos.data(), B * 4);
  put(done, st_done.data(), B * 4);
  put(budget, st_bud.data(), B * 4);
  put(last_rows, last.data(), B * 4);
  put(n_active, &active, 4);
  put(sparams, spd.data(), B * sizeof(SampleParams));
  PPOEXP_CUDA(cudaMemsetAsync(n_gen, 0, B * 4, cc.stream));
  if (any_sampled) {
    // One mt19937_64 uniform per sampled token, Rng(seed) stream
    // (include/aligner/rng.hpp:21-23; consumed in order, src/model.cpp:464).
    double* u = reinterpret_cast<double*>(hs + o);
    for (int64_t b = 0; b < B; ++b) {
      if (spd[b].greedy) continue;
      std::mt19937_64 gen(seeds_all[b0 + b]);
      for (int64_t i = 0; i < bud[b]; ++i) u[b * S + i] = double(gen() >> 11) * 0x1.0p-53;
    }
    PPOEXP_CUDA(cudaMemcpyAsync(uniforms, u, size_t(B) * S * 8, cudaMemcpyHostToDevice, cc.stream));
  }
  // packed prompts
  Packed pk;
  pk.offsets.resize(B + 1);
  for (int64_t b = 0; b <= B; ++b) pk.offsets[b] = off_all[b0 + b] - off_all[b0];
  const int64_t M = pk.offsets[B];
  pk.tokens_d = static_cast<int32_t*>(cc.workspace("gen.prompts", M * 4));
  copy_in(cc, pk.tokens_d, prompts + off_all[b0], M * 4, where_tokens);
  pack_metadata(cc, pk, "gen");  // synchronises: the pinned staging above is free again
  // prefill → last-position logits → first sample
  KvTarget kt{block_table, geom, kvp};
  float* xr = forward_layers(*m, pk, &kt);
  if (m->mixed()) {
    launch_layernorm<float>(cc, xr, B, d, m->lnfw, m->lnfb, static_cast<float*>(h), last_rows, nullptr, nullptr);
    gemm_mixed(cc, static_cast<float*>(h), d, static_cast<const bf16*>(m->tok), d, B, cfg.vocab_size, d,
               Epi::kStoreF32, logits, m->vpad);
  } else if (m->dtype == PPOEXP_F32) {
    launch_layernorm<float>(cc, xr, B, d, m->lnfw, m->lnfb, static_cast<float*>(h), last_rows, nullptr, nullptr);
    gemm<float>(cc, static_cast<float*>(h), d, static_cast<const float*>(m->tok), d, B, cfg.vocab_size, d,
                Epi::kStoreF32, logits, m->vpad);
  } else {
    launch_layernorm<bf16>(cc, xr, B, d, m->lnfw, m->lnfb, static_cast<bf16*>(h), last_rows, nullptr, nullptr);
    gemm<bf16>(cc, static_cast<bf16*>(h), d, static_cast<const bf16*>(m->tok), d, B, cfg.vocab_size, d,
               Epi::kStoreF32, logits, m->vpad);
  }
  launch_sampler(cc, logits, m->vpad, B, cfg.vocab_size, sampler_state());
  // decode: units 1 .. max_budget-1
  cur_P = P;
  cur_len = bud;  // upper bound until the true lengths are known
  run = Run{};
  run.B = B;
  run.b0 = b0;
  run.units = max_budget - 1;
  run.out_stride = out_stride;
  run.out_tokens = out_tokens;
  run.out_logprobs = out_logprobs;
  run.out_lengths = out_lengths;
  run.where_out = where_out;
  if (run.units > 0) {
    run.R = ceil_div(run.units, int64_t(kUnitsPerGraph));
    if (opts.use_graphs) {
      run.gs = &graph_for(B, kUnitsPerGraph);
      // the last replay runs exactly the remaining units (no decode steps past the budget)
      const int rem = int(run.units % kUnitsPerGraph);
      run.tail = rem ? &graph_for(B, rem) : run.gs;
    }
    run.active = true;
  }
}

void Engine::chunk_launch(Run& run) {
  if (!run.active) return;
  LaneScope ls(c, *this);
  Ctx& cc = *c;
  const int j = int(run.r & 1);
  if (run.gs) {
    GraphSet* g = run.r + 1 == run.R ? run.tail : run.gs;
    PPOEXP_CUDA(cudaGraphLaunch(g->exec[j], cc.stream));
    cc.launches += g->nodes;
    run.pending.push_back({g, j, 1 + run.r * kUnitsPerGraph});
  } else {
    for (int64_t u = 1 + run.r * kUnitsPerGraph; u <= std::min(run.units, (run.r + 1) * kUnitsPerGraph); ++u)
      run_unit(run.B, u);
  }
  PPOEXP_CUDA(cudaMemcpyAsync(host_flags + j, n_active, 4, cudaMemcpyDeviceToHost, cc.stream));
  PPOEXP_CUDA(cudaEventRecord(poll_ev[j], cc.stream));
}

void Engine::chunk_poll(Run& run) {
  if (!run.active) return;
  LaneScope ls(c, *this);
  // the host stays one replay behind: replay r is queued while r-1's counter is read
  if (run.r >= 1) {
    const int k = int((run.r - 1) & 1);
    PPOEXP_CUDA(cudaEventSynchronize(poll_ev[k]));
    if (c->profiling && run.gs) {
      // events of replay r-1 must be read before that graph runs again
      auto [g, sj, u0] = run.pending.front();
      run.pending.erase(run.pending.begin());
      prof_replays.push_back({g->events[sj], u0, g->units});
      snapshot_events(prof_replays.back());
    }
    if (host_flags[k] == 0) run.stop = true;
  }
  ++run.r;
  run.active = run.r < run.R && !run.stop;
}

void Engine::chunk_finish(Run& run) {
  LaneScope ls(c, *this);
  Ctx& cc = *c;
  const int64_t B = run.B, b0 = run.b0, S = m->cfg.max_seq_len, out_stride = run.out_stride;
  int32_t* out_tokens = run.out_tokens;
  double* out_logprobs = run.out_logprobs;
  int64_t* out_lengths = run.out_lengths;
  const int where_out = run.where_out;
  std::vector<int64_t>& lens_all = owner ? owner->last_lengths : last_lengths;
  PPOEXP_CUDA(cudaStreamSynchronize(cc.stream));
  if (cc.profiling && run.gs) {
    for (auto& [g, sj, u0] : run.pending) {
      prof_replays.push_back({g->events[sj], u0, g->units});
      snapshot_events(prof_replays.back());
    }
  }
  run.pending.clear();
  // outputs
  std::vector<int32_t> ng(B);
  PPOEXP_CUDA(cudaMemcpyAsync(ng.data(), n_gen, B * 4, cudaMemcpyDeviceToHost, cc.stream));
  PPOEXP_CUDA(cudaMemcpyAsync(host_flags + 8, stat_ovf, 4, cudaMemcpyDeviceToHost, cc.stream));
  PPOEXP_CUDA(cudaStreamSynchronize(cc.stream));
  if (host_flags[8]) {
    PPOEXP_CUDA(cudaMemsetAsync(stat_ovf, 0, 4, cc.stream));
    throw ContractError(
        "engine: residual stream outside the fused-LayerNorm statistics range (|x| rms > ~2e4); rerun with "
        "PPOEXP_FUSE_LN=0");
  }
  for (int64_t b = 0; b < B; ++b) {
    cur_len[b] = ng[b];
    lens_all[b0 + b] = ng[b];
  }
  if (cc.profiling) {
    for (auto& pr : prof_replays) harvest_snapshot(pr);
    prof_replays.clear();
  }
  double* lp64 = static_cast<double*>(cc.workspace("gen.lp64", size_t(B) * S * 8));
  launch_f32_to_f64(cc, out_lp, B * S, lp64);
  if (where_out == PPOEXP_DEVICE) {
    std::vector<int64_t> l64(ng.begin(), ng.end());
    PPOEXP_CUDA(cudaMemcpyAsync(out_lengths + b0, l64.data(), B * 8, cudaMemcpyHostToDevice, cc.stream));
    PPOEXP_CUDA(cudaStreamSynchronize(cc.stream));
  } else {
    for (int64_t b = 0; b < B; ++b) out_lengths[b0 + b] = ng[b];
  }
  const auto kind = where_out == PPOEXP_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  const int64_t w = std::min<int64_t>(out_stride, S);
  PPOEXP_CUDA(cudaMemcpy2DAsync(out_tokens + b0 * out_stride, out_stride * 4, out_tok, S * 4, w * 4, B, kind, cc.stream));
  PPOEXP_CUDA(
      cudaMemcpy2DAsync(out_logprobs + b0 * out_stride, out_stride * 8, lp64, S * 8, w * 8, B, kind, cc.stream));
  if (where_out == PPOEXP_HOST) PPOEXP_CUDA(cudaStreamSynchronize(cc.stream));
}

// Profiling support: copy the elapsed times of a finished replay's events
// (the graph will overwrite them on its next launch).
void Engine::snapshot_events(ReplayTimes& r) {
  r.ms.resize(r.events.size());
  for (size_t i = 0; i < r.events.size(); ++i) {
    PPOEXP_CUDA(cudaEventSynchronize(r.events[i].b));
    float ms = 0;
    PPOEXP_CUDA(cudaEventElapsedTime(&ms, r.events[i].a, r.events[i].b));
    r.ms[i] = ms;
  }
}

void Engine::harvest_snapshot(const ReplayTimes& r) {
  const int64_t d = m->d();
  const double ts = double(m->asize());
  int64_t per_unit = 0;
  for (auto& t : r.events)
    if (t.cls == "decode_attention") ++per_unit;
  per_unit /= std::max(r.units, 1);
  int64_t seen = 0;
  for (size_t i = 0; i < r.events.size(); ++i) {
    const auto& t = r.events[i];
    double bytes = t.bytes;
    const int64_t u = r.unit0 + (per_unit ? seen / per_unit : 0);
    if (t.cls == "decode_attention") {
      ++seen;
      bytes = 0;
      for (size_t b = 0; b < cur_P.size(); ++b)
        if (u <= cur_len[b] - 1) bytes += (double(cur_P[b] + u) * 2.0 + 2.0) * d * ts;
    }
    auto& s = c->stats[t.cls];
    s.ms += r.ms[i];
    s.launches += 1;
    s.bytes += bytes;
    s.flops += t.flops;
  }
}

}  // namespace ppx

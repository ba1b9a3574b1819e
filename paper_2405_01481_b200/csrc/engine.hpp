// engine.hpp — rollout engine over a device model (paged KV + graphs).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "model.hpp"

namespace ppx {

struct Engine {
  Model* m;
  Ctx* c;
  ppoexp_engine_options opts{};
  KvGeom geom{};
  DeviceBuffer kv;     // paged pool
  void* kvp = nullptr; // the pool this engine decodes into (kv.ptr, or the owner's for a lane)
  DeviceBuffer state;  // per-sequence state + step activations + outputs
  int32_t *next_tok, *pos, *n_gen, *done, *budget, *n_active, *block_table, *last_rows;
  SampleParams* sparams;
  float* x;
  void *h, *qkv, *att, *up;
  float* logits;
  int32_t* out_tok;
  float* out_lp;
  double* uniforms;
  int32_t* host_flags = nullptr;
  unsigned long long* stats = nullptr;  // fused-LN fixed-point row statistics [2L+1][max_batch][2]
  unsigned* stat_ovf = nullptr;         // set by a producer whose partial left the fixed-point range
  bool fuse_ln = false;
  bool mixed_planes = false;   // mixed decode through bf16 hi/lo activation planes (decode_unit_mixed)
  bool mixed_oplanes = false;  // ... planes for the O / down operands only (LayerNorm stays fused)
  int64_t fuse_ln_max_b = 64;  // fused LayerNorm only for decode batches up to this size
  cudaEvent_t poll_ev[2]{}, t0{}, t1{};
  double last_ms = 0;
  double gen_seconds = 0;    // CostBook "response_generation" (src/engine.cpp:179)
  double build_seconds = 0;  // model deep copy + KV pool / graph state allocation
  int64_t cur_unit = 0;
  std::vector<int64_t> cur_P, cur_len;

  struct GraphSet {
    cudaGraphExec_t exec[2]{};
    std::vector<TimedLaunch> events[2];
    int64_t nodes = 0;
    int units = 8;
    bool profiled = false;
    std::string prof_sig;
  };
  std::map<int64_t, GraphSet> graphs;

  struct ReplayTimes {
    std::vector<TimedLaunch> events;
    int64_t unit0;
    int units;
    std::vector<float> ms;
  };
  std::vector<ReplayTimes> prof_replays;

  // Decode lanes: a batch split over two sub-engines (each with its own
  // stream, step state and graphs, pages from the owner's pool) whose decode
  // chains run concurrently — each decode step is a chain of ~90 dependent
  // latency-bound launches, so two half-batch chains overlap on the SMs.
  std::unique_ptr<Engine> lanes[2];
  Engine* owner = nullptr;
  cudaStream_t lane_stream = nullptr;
  std::string lane_prefix;
  cudaEvent_t lane_ev = nullptr;
  int n_lanes = 1;          // PPOEXP_LANES (default: 2 for mixed / bf16 decode)
  int64_t lane_min_b = 128;  // split only batches of at least this many sequences (C3 +13%, C2 / C4 not)

  Engine(Model* model, const ppoexp_engine_options* o, Engine* owner_ = nullptr);
  ~Engine();

  void generate(int64_t B, const int32_t* prompts, const int64_t* offsets, const int64_t* max_new,
                const ppoexp_sampling* sampling, const uint64_t* seeds, int64_t out_stride, int32_t* out_tokens,
                double* out_logprobs, int64_t* out_lengths, int where, double* ms_out, int where_out = -1,
                int where_tokens = -1);
  std::vector<int64_t> last_lengths;  // host copy of the last call's lengths

  // One chunk of generation, issued in phases so that lanes interleave.
  struct Run {
    int64_t B = 0, b0 = 0, units = 0, R = 0, r = 0;
    bool stop = false, active = false;
    GraphSet* gs = nullptr;    // kUnitsPerGraph decode units per replay
    GraphSet* tail = nullptr;  // the last replay: the remaining units
    std::vector<std::tuple<GraphSet*, int, int64_t>> pending;  // (graph, slot, unit0) awaiting harvest
    int64_t out_stride = 0;
    int32_t* out_tokens = nullptr;
    double* out_logprobs = nullptr;
    int64_t* out_lengths = nullptr;
    int where_out = 0;
  };

 private:
  void chunk_begin(Run& run, int64_t B, const int32_t* prompts, const std::vector<int64_t>& off_all, int64_t b0,
                   const std::vector<int64_t>& mx_all, const ppoexp_sampling* sp_all,
                   const std::vector<uint64_t>& seeds_all, int64_t out_stride, int32_t* out_tokens,
                   double* out_logprobs, int64_t* out_lengths, int where_out, int where_tokens, int64_t page_base);
  void chunk_launch(Run& run);  // enqueue replay r
  void chunk_poll(Run& run);    // wait for replay r-1's done counter; decides whether to stop
  void chunk_finish(Run& run);
  int64_t chunk_pages(int64_t B, const std::vector<int64_t>& off_all, int64_t b0,
                      const std::vector<int64_t>& mx_all) const;
  void run_chunk(int64_t B, const int32_t* prompts, const std::vector<int64_t>& off_all, int64_t b0,
                 const std::vector<int64_t>& mx_all, const ppoexp_sampling* sp_all,
                 const std::vector<uint64_t>& seeds_all,
                 int64_t out_stride, int32_t* out_tokens, double* out_logprobs, int64_t* out_lengths, int where,
                 int where_out, int where_tokens);
  SamplerState sampler_state() const;
  template <class T>
  void decode_unit(int64_t B, int64_t unit);
  void decode_unit_mixed(int64_t B, int64_t unit);
  void run_unit(int64_t B, int64_t unit);
  GraphSet& graph_for(int64_t B, int units);
  void harvest_replay(const std::vector<TimedLaunch>& evs, int64_t unit0, int units);
  void snapshot_events(ReplayTimes& r);
  void harvest_snapshot(const ReplayTimes& r);
};

}  // namespace ppx

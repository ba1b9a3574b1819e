// runtime.hpp — host runtime: context (device + stream), kernel-class
// profiler (CUDA events), launch accounting, named device workspaces.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include <functional>
#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ppx {

struct ClassStats {
  double ms = 0.0;
  int64_t launches = 0;
  double bytes = 0.0;
  double flops = 0.0;
};

struct TimedLaunch {
  std::string cls;
  cudaEvent_t a, b;
  double bytes, flops;
};

struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (ptr) cudaFree(ptr);
  }
  // First allocation is exact; a buffer that has to grow grows by >= 1.5x, so
  // workspaces sized by data-dependent shapes (response lengths) settle after a
  // few calls instead of reallocating (cudaFree synchronizes the device)
  void ensure(size_t n) {
    if (n <= bytes) return;
    const size_t want = ptr ? std::max(n, bytes + bytes / 2) : n;
    if (ptr) PPOEXP_CUDA(cudaFree(ptr));
    ptr = nullptr;
    bytes = 0;
    PPOEXP_CUDA(cudaMalloc(&ptr, want));
    bytes = want;
  }
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::recursive_mutex mu;
  bool profiling = false;
  std::set<std::string> profile_filter;  // empty = every class
  bool capturing = false;
  int64_t launches = 0;          // eager launches + graph-replayed kernel nodes
  int64_t capture_launches = 0;  // kernels recorded into the graph being captured
  std::map<std::string, ClassStats> stats;
  std::map<std::string, int64_t> variants;  // kernel-variant choices made on the host (tests assert the branch ran)
  std::vector<TimedLaunch> pending;          // eager timed launches to harvest
  std::vector<TimedLaunch>* capture_events = nullptr;  // events recorded while capturing
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, std::unique_ptr<DeviceBuffer>> ws;
  std::vector<std::array<int, 4>> gemm_trace_meta;  // debug: PPOEXP_GEMM_TRACE launch metadata
  // pinned host staging for HOST-where API calls
  void* pinned = nullptr;
  size_t pinned_bytes = 0;

  explicit Ctx(int dev);
  ~Ctx();

  cudaEvent_t new_event();
  void release_event(cudaEvent_t e) { event_pool.push_back(e); }

  // Launch `f` (which enqueues exactly one kernel on `stream`) under class
  // `cls`, with the algorithmic bytes / flops it moves.
  template <class F>
  void launch(const char* cls, double bytes, double flops, F&& f) {
    if (profiling && (profile_filter.empty() || profile_filter.count(cls))) {
      TimedLaunch t{cls, new_event(), new_event(), bytes, flops};
      // inside stream capture a plain record is only a dependency marker;
      // cudaEventRecordExternal materialises a timing node in the graph
      const unsigned fl = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
      PPOEXP_CUDA(cudaEventRecordWithFlags(t.a, stream, fl));
      f();
      PPOEXP_CUDA(cudaGetLastError());
      PPOEXP_CUDA(cudaEventRecordWithFlags(t.b, stream, fl));
      if (capturing && capture_events)
        capture_events->push_back(t);
      else
        pending.push_back(t);
    } else {
      f();
      PPOEXP_CUDA(cudaGetLastError());
    }
    if (capturing)
      ++capture_launches;
    else
      ++launches;
  }

  // Accumulate finished eager timings (blocks until they complete).
  void harvest();
  void harvest_list(const std::vector<TimedLaunch>& evs, bool release);

  // name prefix of the workspaces used by the forward currently being issued
  // (concurrent scoring forwards on separate streams keep separate buffers)
  std::string ws_prefix;
  cudaStream_t aux[2] = {nullptr, nullptr};  // concurrent scoring forwards (lazily created)
  cudaEvent_t fork_ev = nullptr, join_ev[2] = {nullptr, nullptr};

  void* workspace(const std::string& name, size_t bytes) {
    auto& b = ws[ws_prefix + name];
    if (!b) b = std::make_unique<DeviceBuffer>();
    if (bytes > b->bytes && b->bytes && getenv("PPOEXP_WS_TRACE"))  // debug: data-dependent regrowth
      fprintf(stderr, "[ppoexp] workspace %s%s grows %zu -> %zu bytes\n", ws_prefix.c_str(), name.c_str(), b->bytes,
              bytes);
    b->ensure(bytes);
    return b->ptr;
  }
  // Pinned host staging for H2D/D2H copies.  Synchronises the stream first:
  // earlier async copies may still be reading the previous contents.
  void* pinned_staging(size_t bytes);
  void sync() { PPOEXP_CUDA(cudaStreamSynchronize(stream)); }
};

// Launch with programmatic stream serialization (PDL) and an optional
// cluster along y.  Every kernel in the library calls pdl_wait() before it
// touches data produced by earlier work, so the attribute is always safe.
template <class... KArgs, class... Args>
void launch_kernel(Ctx& c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, int cluster_y, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster_y > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = 1;
    at[n].val.clusterDim.y = cluster_y;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  PPOEXP_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// Copy helpers that honour ppoexp_where (0 = host, 1 = device).
void copy_in(Ctx& c, void* dst_dev, const void* src, size_t bytes, int where);
void copy_out(Ctx& c, void* dst, const void* src_dev, size_t bytes, int where);

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev, bool nothrow = false) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      (void)cudaGetLastError();
      if (nothrow) return;
    }
    if (prev != dev) {
      const cudaError_t e = cudaSetDevice(dev);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        if (!nothrow) PPOEXP_CUDA(e);
      }
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace ppx

// CUDA-graph replay cache for the RFP entry points.
//
// A pftrf at n = 16384 issues ~2,300 stream-ordered kernels (the recursive
// potrf/trsm chains), most of them small; issuing them one by one from the
// host leaves gaps on the GPU.  The first call with a given argument tuple is
// captured into a CUDA graph (the workspace cudaMallocAsync/cudaFreeAsync
// become graph memory nodes), instantiated, and replayed on every later call
// with the same tuple -- one host launch, back-to-back kernels on the device.
// Pointers are part of the key, so a replay always touches the caller's
// current buffers.  Tuning "graphs" = 0 disables the cache (rfpk_set_tuning,
// which also clears it).
#pragma once
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <tuple>

#include "common.cuh"

namespace rfpk {

struct GraphKey {
  int op;
  char dtype, transr, uplo, diag;
  long long n, nrhs, rsb, csb;
  const void* arf;
  const void* b;
  const void* info;
  int device;
  bool operator<(const GraphKey& o) const {
    return std::tie(op, dtype, transr, uplo, diag, n, nrhs, rsb, csb, arf, b, info, device) <
           std::tie(o.op, o.dtype, o.transr, o.uplo, o.diag, o.n, o.nrhs, o.rsb, o.csb, o.arf, o.b,
                    o.info, o.device);
  }
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;  // kernel launches recorded in the graph
  unsigned long long last_use = 0;
};

class GraphCache {
 public:
  static GraphCache& get() {
    static GraphCache g;
    return g;
  }

  // Run `body(stream)`; with the cache enabled it is captured once per key
  // and replayed afterwards.  Returns the body's / CUDA's status.
  int run(const GraphKey& key, cudaStream_t st, const std::function<int(cudaStream_t)>& body) {
    // Large orders are GPU-bound (launch overhead is noise) and run faster
    // direct: captured kernel nodes do not keep the high / low stream
    // priorities the look-ahead relies on (measured: n=16384 pftrf 61.1 ms
    // direct vs 64.8 ms replayed; n=4000 4.44 ms direct vs 4.23 replayed).
    if (!tune(TK_GRAPHS) || key.n >= tune(TK_GRAPH_MAX_N)) return body(st);
    std::lock_guard<std::mutex> lk(mu_);
    // The legacy NULL stream cannot be captured: use a library stream that is
    // a *blocking* stream, hence implicitly ordered with the legacy stream.
    cudaStream_t s = st;
    if (s == nullptr) {
      if (!own_) cudaStreamCreate(&own_);
      s = own_;
    }
    auto it = cache_.find(key);
    if (it == cache_.end() && seen_.insert(key).second) {
      if (seen_.size() > 4096) seen_.clear();
      return body(st);
    }
    if (it == cache_.end()) {
      cudaGraph_t graph = nullptr;
      long long before = g_launch_count.load();
      cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return body(st);
      int rc = body(s);
      e = cudaStreamEndCapture(s, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (e != cudaSuccess) return (int)e;
      GraphEntry ent;
      e = cudaGraphInstantiate(&ent.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return (int)e;
      ent.kernels = g_launch_count.load() - before;
      g_launch_count.fetch_sub(ent.kernels);  // counted at replay instead
      evict_if_full();
      it = cache_.emplace(key, ent).first;
    }
    it->second.last_use = ++clock_;
    cudaError_t e = cudaGraphLaunch(it->second.exec, s);
    if (e != cudaSuccess) return (int)e;
    g_launch_count.fetch_add(it->second.kernels);
    return 0;
  }

  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& kv : cache_) cudaGraphExecDestroy(kv.second.exec);
    cache_.clear();
    seen_.clear();
  }

 private:
  GraphCache() = default;
  void evict_if_full() {
    const size_t cap = 64;
    if (cache_.size() < cap) return;
    auto victim = cache_.begin();
    for (auto it = cache_.begin(); it != cache_.end(); ++it)
      if (it->second.last_use < victim->second.last_use) victim = it;
    cudaGraphExecDestroy(victim->second.exec);
    cache_.erase(victim);
  }
  std::map<GraphKey, GraphEntry> cache_;
  std::set<GraphKey> seen_;
  std::mutex mu_;
  cudaStream_t own_ = nullptr;
  unsigned long long clock_ = 0;
};

}  // namespace rfpk

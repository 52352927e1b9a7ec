// CUDA-graph replay of fixed launch sequences (host-side launch overhead of the
// latency-bound sweeps).  A sequence is recorded once by stream capture on a
// private stream (nothing executes during capture), instantiated, cached under
// a key that hashes every value the sequence depends on (descriptors, device
// pointers, capacity shapes, direction), and then replayed with one
// cudaGraphLaunch on the caller's stream.  TT_NO_GRAPHS=1 disables it.
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "tt_common.cuh"

namespace tt {

namespace {
struct GraphCache {
  std::unordered_map<uint64_t, cudaGraphExec_t> m;
  cudaStream_t cs = nullptr;
  int disabled = -1;
};
thread_local GraphCache g_gc;
}  // namespace

// 64-bit words with a multiply-rotate mix (the keyed structs are several KB;
// a byte-wise loop cost ~15 us per key on the host's critical path)
uint64_t hash_bytes(const void *p, size_t n, uint64_t h) {
  const unsigned char *b = static_cast<const unsigned char *>(p);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h ^= w * 0x9E3779B97F4A7C15ull;
    h = ((h << 31) | (h >> 33)) * 0xC2B2AE3D27D4EB4Full;
  }
  for (; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h ^ (h >> 29);
}

tt_status run_captured(uint64_t key, cudaStream_t &s, const std::function<tt_status()> &enqueue) {
  if (g_gc.disabled < 0) g_gc.disabled = std::getenv("TT_NO_GRAPHS") ? 1 : 0;
  if (g_gc.disabled) return enqueue();
  auto it = g_gc.m.find(key);
  if (it == g_gc.m.end() && g_gc.m.size() >= 4096) {   // bound the cache (new workspaces => new keys)
    cudaStreamSynchronize(s);
    for (auto &kv : g_gc.m) cudaGraphExecDestroy(kv.second);
    g_gc.m.clear();
  }
  if (it == g_gc.m.end()) {
    if (!g_gc.cs && cudaStreamCreateWithFlags(&g_gc.cs, cudaStreamNonBlocking) != cudaSuccess) {
      g_gc.disabled = 1;
      return enqueue();
    }
    cudaStream_t user = s;
    s = g_gc.cs;   // the enqueue closure launches on `s` (captured by reference)
    cudaGraph_t graph = nullptr;
    tt_status st = TT_OK;
    if (cudaStreamBeginCapture(g_gc.cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      st = enqueue();
      const cudaError_t e = cudaStreamEndCapture(g_gc.cs, &graph);
      if (e != cudaSuccess) st = TT_ERR_CUDA;
    } else {
      st = TT_ERR_CUDA;
    }
    s = user;
    cudaGraphExec_t exec = nullptr;
    if (st == TT_OK && graph && cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
      g_gc.m.emplace(key, exec);
      cudaGraphDestroy(graph);
    } else {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();   // clear a capture error; run the sequence directly
      g_gc.disabled = 1;
      return enqueue();
    }
    it = g_gc.m.find(key);
  }
  if (cudaGraphLaunch(it->second, s) != cudaSuccess) return fail(TT_ERR_CUDA, "graph launch failed");
  return TT_OK;
}

}  // namespace tt

// CUDA graphs for the latency-bound drivers.
//
// 1. Replay of fixed launch sequences: a sequence is recorded once by stream
//    capture on a private stream (nothing executes during capture),
//    instantiated, cached under its key — the exact bytes of every value the
//    sequence depends on (descriptors, device pointers, capacity shapes,
//    options), compared in full on every hit, with a 64-bit hash only as the
//    bucket index — and replayed with one cudaGraphLaunch on the caller's
//    stream.  Inside an outer capture the sequence is recorded inline.
// 2. Device-resident loops: while a stream is being captured, the drivers'
//    convergence loops (AMEn / amen_mv sweeps, the k-eff fixed point, the alpha
//    secant) become conditional WHILE / IF nodes whose condition is set on the
//    device (cudaGraphSetConditional), so a whole keff_fixed_point call is one
//    graph launch with no host round trip inside.
// graph_mode(): 0 = no graphs (TT_NO_GRAPHS=1), 1 = replayed sequences with
// host-polled loops (TT_NO_DEVLOOP=1), 2 = device-resident loops (default).
// A capture or instantiation failure is an error (TT_ERR_CUDA), never a silent
// switch to another mode.
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "tt_common.cuh"

namespace tt {

namespace {
struct Entry {
  std::string key;
  cudaGraphExec_t exec;
};
struct GraphCache {
  std::unordered_map<uint64_t, std::vector<Entry>> m;
  size_t count = 0;
  cudaStream_t cs = nullptr;            // top-level capture stream
  std::vector<cudaStream_t> body;       // one capture stream per conditional-body depth
  int depth = 0;
  int mode = -1;
  long long captures = 0, replays = 0;
};
thread_local GraphCache g_gc;

__global__ void cond_set_kernel(cudaGraphConditionalHandle h, unsigned int v) { cudaGraphSetConditional(h, v); }
__global__ void cond_from_flag_kernel(cudaGraphConditionalHandle h, const int *flag) {
  cudaGraphSetConditional(h, *flag == 0 ? 1u : 0u);
}
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

void GraphKey::add(const void *p, size_t n) {
  bytes.append(static_cast<const char *>(p), n);
  h = hash_bytes(p, n, h);
}

int graph_mode() {
  if (g_gc.mode < 0) g_gc.mode = std::getenv("TT_NO_GRAPHS") ? 0 : (std::getenv("TT_NO_DEVLOOP") ? 1 : 2);
  return g_gc.mode;
}
void set_graph_mode(int mode) { g_gc.mode = mode < 0 ? -1 : (mode > 2 ? 2 : mode); }
void graph_stats(long long *captures, long long *replays, long long *cached) {
  if (captures) *captures = g_gc.captures;
  if (replays) *replays = g_gc.replays;
  if (cached) *cached = (long long)g_gc.count;
}

bool stream_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) return false;
  return st == cudaStreamCaptureStatusActive;
}

bool device_loops(cudaStream_t s) { return graph_mode() >= 2 && stream_capturing(s); }

tt_status run_captured(const GraphKey &key, cudaStream_t &s, const std::function<tt_status()> &enqueue) {
  if (graph_mode() == 0 || stream_capturing(s)) return enqueue();   // no graphs / inline in an outer capture
  std::vector<Entry> &bucket = g_gc.m[key.h];
  cudaGraphExec_t exec = nullptr;
  for (const Entry &e : bucket)
    if (e.key == key.bytes) { exec = e.exec; break; }
  if (!exec) {
    if (g_gc.count >= 4096) {   // bound the cache (new workspaces => new keys)
      cudaStreamSynchronize(s);
      for (auto &kv : g_gc.m)
        for (Entry &e : kv.second) cudaGraphExecDestroy(e.exec);
      g_gc.m.clear();
      g_gc.count = 0;
    }
    if (!g_gc.cs && cudaStreamCreateWithFlags(&g_gc.cs, cudaStreamNonBlocking) != cudaSuccess)
      return fail(TT_ERR_CUDA, "graph: capture stream");
    cudaStream_t user = s;
    s = g_gc.cs;   // the enqueue closure launches on `s` (captured by reference)
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(g_gc.cs, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
      s = user;
      return fail(TT_ERR_CUDA, std::string("graph: begin capture: ") + cudaGetErrorString(e));
    }
    tt_status st = enqueue();
    e = cudaStreamEndCapture(g_gc.cs, &graph);
    s = user;
    if (st != TT_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      return fail(TT_ERR_CUDA, std::string("graph: capture failed: ") + cudaGetErrorString(e));
    }
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(TT_ERR_CUDA, std::string("graph: instantiate failed: ") + cudaGetErrorString(e));
    }
    g_gc.m[key.h].push_back(Entry{key.bytes, exec});
    ++g_gc.count;
    ++g_gc.captures;
  }
  ++g_gc.replays;
  if (cudaGraphLaunch(exec, s) != cudaSuccess) return fail(TT_ERR_CUDA, "graph launch failed");
  return TT_OK;
}

// ---- conditional nodes (device-resident loops) -------------------------------
tt_status cond_handle(cudaStream_t s, cudaGraphConditionalHandle *h) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess || st != cudaStreamCaptureStatusActive || !g)
    return fail(TT_ERR_CUDA, "cond_handle: stream is not capturing");
  e = cudaGraphConditionalHandleCreate(h, g, 0, 0);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("cond_handle: ") + cudaGetErrorString(e));
  return TT_OK;
}

tt_status cond_node(cudaStream_t &s, cudaGraphConditionalHandle h, int is_while,
                    const std::function<tt_status()> &body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess || st != cudaStreamCaptureStatusActive) return fail(TT_ERR_CUDA, "cond_node: not capturing");
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = is_while ? cudaGraphCondTypeWhile : cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, deps, nd, &p);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("cond_node: add: ") + cudaGetErrorString(e));
  cudaGraph_t bg = p.conditional.phGraph_out[0];
  e = cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("cond_node: deps: ") + cudaGetErrorString(e));
  const int dpt = g_gc.depth;
  while ((int)g_gc.body.size() <= dpt) {
    cudaStream_t bs;
    if (cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking) != cudaSuccess)
      return fail(TT_ERR_CUDA, "cond_node: body stream");
    g_gc.body.push_back(bs);
  }
  cudaStream_t bs = g_gc.body[dpt];
  e = cudaStreamBeginCaptureToGraph(bs, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("cond_node: body capture: ") + cudaGetErrorString(e));
  cudaStream_t outer = s;
  s = bs;
  ++g_gc.depth;
  const tt_status r = body();
  --g_gc.depth;
  s = outer;
  e = cudaStreamEndCapture(bs, nullptr);
  if (r != TT_OK) return r;
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("cond_node: end body: ") + cudaGetErrorString(e));
  return TT_OK;
}

tt_status cond_set(cudaGraphConditionalHandle h, unsigned int v, cudaStream_t s) {
  cond_set_kernel<<<1, 1, 0, s>>>(h, v);
  return check_launch("cond_set");
}

tt_status cond_from_flag(cudaGraphConditionalHandle h, const int *flag_dev, cudaStream_t s) {
  cond_from_flag_kernel<<<1, 1, 0, s>>>(h, flag_dev);
  return check_launch("cond_from_flag");
}

tt_status dev_while(cudaStream_t &s, const std::function<tt_status(cudaGraphConditionalHandle)> &body) {
  cudaGraphConditionalHandle h;
  TT_TRY(cond_handle(s, &h));
  TT_TRY(cond_set(h, 1u, s));   // re-armed on every entry (nested loops)
  return cond_node(s, h, 1, [&]() { return body(h); });
}

}  // namespace tt

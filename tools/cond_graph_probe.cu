// Probe: which node types the driver accepts inside CUDA-graph conditional
// bodies built by stream capture (the device-resident loop design of
// keff_fixed_point / amen_solve).  Outer WHILE { cooperative kernel;
// cluster kernel; memset; D2D memcpy; inner WHILE { kernel }; IF { kernel } }.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cond_graph_probe tools/cond_graph_probe.cu
#include <cooperative_groups.h>
#include <cstdio>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      printf("FAIL %s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

__global__ void coop_k(int *c) {
  cooperative_groups::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(c + 0, 1);
}
__global__ void __cluster_dims__(1, 1, 1) clus_k(int *c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(c + 1, 1);
}
__global__ void clus_dyn_k(int *c) {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(c + 2, 1);
}
__global__ void inner_k(int *c, cudaGraphConditionalHandle h, int limit) {
  const int v = ++c[3];
  cudaGraphSetConditional(h, (v % limit) != 0);
}
__global__ void if_k(int *c) { c[4] += 1; }
__global__ void outer_tail_k(int *c, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hif, int n) {
  const int v = ++c[5];
  cudaGraphSetConditional(hw, v < n);
  cudaGraphSetConditional(hif, v & 1);
}
__global__ void set_k(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }

// add a conditional node at the current capture position of s; returns its body graph
static cudaError_t add_cond(cudaStream_t s, cudaGraphConditionalNodeType type, unsigned def,
                            cudaGraphConditionalHandle *h, cudaGraph_t *body) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g;
  const cudaGraphNode_t *deps;
  size_t nd;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  e = cudaGraphConditionalHandleCreate(h, g, def, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return e;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = *h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, deps, nd, &p);
  if (e != cudaSuccess) return e;
  *body = p.conditional.phGraph_out[0];
  return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

int main() {
  int *c, *c2;
  CK(cudaMalloc(&c, 64 * sizeof(int)));
  CK(cudaMalloc(&c2, 64 * sizeof(int)));
  CK(cudaMemset(c, 0, 64 * sizeof(int)));
  cudaStream_t s0, s1, s2;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaFuncSetAttribute(clus_dyn_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int NOUT = 5, NIN = 3;
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  cudaGraphConditionalHandle hw, hin, hif;
  cudaGraph_t bw, bin, bif;
  CK(add_cond(s0, cudaGraphCondTypeWhile, 1, &hw, &bw));
  // outer body captured on s1
  CK(cudaStreamBeginCaptureToGraph(s1, bw, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  {
    void *args[] = {(void *)&c};
    CK(cudaLaunchCooperativeKernel((const void *)coop_k, dim3(296), dim3(128), args, 0, s1));
    clus_k<<<2, 32, 0, s1>>>(c);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8);
    cfg.blockDim = dim3(128);
    cfg.stream = s1;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, clus_dyn_k, c));
    CK(cudaMemsetAsync(c2, 0, 16 * sizeof(int), s1));
    CK(cudaMemcpyAsync(c2 + 16, c, 8 * sizeof(int), cudaMemcpyDeviceToDevice, s1));
    // inner WHILE, re-armed each outer iteration by a set kernel
    cudaGraphConditionalHandle dummy;
    (void)dummy;
    // the inner handle must exist before the set kernel: create the node first? no —
    // create the handle on the body graph, then launch the set kernel, then the node
    CK(cudaGraphConditionalHandleCreate(&hin, bw, 1, cudaGraphCondAssignDefault));
    set_k<<<1, 1, 0, s1>>>(hin, 1);
    {
      cudaStreamCaptureStatus st;
      cudaGraph_t g;
      const cudaGraphNode_t *deps;
      size_t nd;
      CK(cudaStreamGetCaptureInfo(s1, &st, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams p = {};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = hin;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, g, deps, nd, &p));
      bin = p.conditional.phGraph_out[0];
      CK(cudaStreamUpdateCaptureDependencies(s1, &node, 1, cudaStreamSetCaptureDependencies));
    }
    CK(cudaStreamBeginCaptureToGraph(s2, bin, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    inner_k<<<1, 1, 0, s2>>>(c, hin, NIN);
    CK(cudaStreamEndCapture(s2, nullptr));
    CK(add_cond(s1, cudaGraphCondTypeIf, 0, &hif, &bif));
    CK(cudaStreamBeginCaptureToGraph(s2, bif, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if_k<<<1, 1, 0, s2>>>(c);
    CK(cudaStreamEndCapture(s2, nullptr));
    outer_tail_k<<<1, 1, 0, s1>>>(c, hw, hif, NOUT);
  }
  CK(cudaStreamEndCapture(s1, nullptr));
  cudaGraph_t graph;
  CK(cudaStreamEndCapture(s0, &graph));
  size_t nn = 0;
  CK(cudaGraphGetNodes(graph, nullptr, &nn));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, graph, 0));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(c, 0, 64 * sizeof(int)));
    CK(cudaGraphLaunch(ex, s0));
    CK(cudaStreamSynchronize(s0));
    int h[8];
    CK(cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost));
    // expected: coop NOUT, clus NOUT, cluster-dyn NOUT, inner NOUT*NIN, if = #odd v<=NOUT before the tail
    // runs... IF reads hif set by the previous tail (default 0 at launch): iterations 2..NOUT with v odd
    printf("rep %d: coop %d clus %d clusdyn %d inner %d if %d outer %d (nodes %zu)\n", rep, h[0], h[1], h[2], h[3],
           h[4], h[5], nn);
    const bool ok = h[0] == NOUT && h[1] == NOUT && h[2] == NOUT && h[3] == NOUT * NIN && h[5] == NOUT;
    printf(ok ? "COND_PROBE_OK\n" : "COND_PROBE_MISMATCH\n");
  }
  // timing: an empty-ish WHILE of 1000 iterations
  return 0;
}

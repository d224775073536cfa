// Probe: can stream memory operations (cuStreamWaitValue32/WriteValue32) be
// captured into a CUDA graph, and can their values be updated per launch?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#define CK(x) do { auto e = (x); if (e) { printf("FAIL %s = %d (line %d)\n", #x, int(e), __LINE__); return 1; } } while (0)
__global__ void bump(unsigned* p) { atomicAdd(p + 2, 1u); }
int main() {
  CK(cudaSetDevice(0));
  unsigned* sig; CK(cudaMalloc(&sig, 64)); CK(cudaMemset(sig, 0, 64));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  CK(cuStreamWriteValue32((CUstream)s, (CUdeviceptr)sig, 5, 0));
  CK(cuStreamWaitValue32((CUstream)s, (CUdeviceptr)sig, 5, CU_STREAM_WAIT_VALUE_GEQ));
  bump<<<1, 1, 0, s>>>(sig);
  cudaGraph_t g; CK(cudaStreamEndCapture(s, &g));
  size_t n = 0; CK(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n); CK(cudaGraphGetNodes(g, nodes.data(), &n));
  printf("captured %zu nodes\n", n);
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
  std::vector<CUgraphNode> memops;
  for (auto nd : nodes) {
    CUgraphNodeType t; CK(cuGraphNodeGetType((CUgraphNode)nd, &t));
    printf(" node type %d\n", int(t));
    if (t == CU_GRAPH_NODE_TYPE_BATCH_MEM_OP) {
      CUDA_BATCH_MEM_OP_NODE_PARAMS p; CK(cuGraphBatchMemOpNodeGetParams((CUgraphNode)nd, &p));
      printf("  batch memop count %u op0 type %d value %u\n", p.count, int(p.paramArray[0].operation),
             p.paramArray[0].writeValue.value);
      memops.push_back((CUgraphNode)nd);
    }
  }
  CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
  // update both memops to value 9 and relaunch
  for (auto nd : memops) {
    CUDA_BATCH_MEM_OP_NODE_PARAMS p; CK(cuGraphBatchMemOpNodeGetParams(nd, &p));
    std::vector<CUstreamBatchMemOpParams> ops(p.paramArray, p.paramArray + p.count);
    for (auto& o : ops) {
      if (o.operation == CU_STREAM_MEM_OP_WRITE_VALUE_32) o.writeValue.value = 9;
      if (o.operation == CU_STREAM_MEM_OP_WAIT_VALUE_32) o.waitValue.value = 9;
    }
    p.paramArray = ops.data();
    CK(cuGraphExecBatchMemOpNodeSetParams((CUgraphExec)ex, nd, &p));
  }
  CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
  unsigned h[3]; CK(cudaMemcpy(h, sig, 12, cudaMemcpyDeviceToHost));
  printf("sig = %u, bumps = %u (expect 9, 2)\n", h[0], h[2]);
  printf("PROBE OK\n");
  return 0;
}

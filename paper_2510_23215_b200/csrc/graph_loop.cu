// graph_loop.cu — device-decided loops (common.cuh: DevLoop, device_while).
//
// Used where an iteration of Alg. 3 contains an inner loop whose
// trip count depends on the data — the sweeps of the block-Jacobi reduced
// eigensolver (l. 6) for b > 128.  Inside a CUDA-graph capture the loop is a WHILE
// conditional node, so the whole outer iteration replays from one graph with no
// host round trip; outside a capture it is a host loop on a flag.
#include "common.cuh"

#include <vector>

namespace scsf {

// kernels captured into conditional bodies on this thread (graph_run adds them, once per replay,
// to the launch count of the graph)
static thread_local int t_cond_kernels = 0;
int take_cond_kernels() {
  const int k = t_cond_kernels;
  t_cond_kernels = 0;
  return k;
}

bool stream_capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return st == cudaStreamCaptureStatusActive;
}

int device_while_impl(cudaStream_t s, int* flag_d, int* flag_h, int (*body)(cudaStream_t, const DevLoop&, void*),
                      void* ctx, int max_passes_eager) {
  DevLoop L;
  L.flag = flag_d;
  if (!stream_capturing(s)) {
    static thread_local cudaEvent_t ev = nullptr;
    if (!ev) SCSF_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventBlockingSync | cudaEventDisableTiming));
    for (int pass = 0; pass < max_passes_eager; ++pass) {
      SCSF_TRY(body(s, L, ctx));
      SCSF_CUDA_CHECK(cudaMemcpyAsync(flag_h, flag_d, sizeof(int), cudaMemcpyDeviceToHost, s));
      SCSF_CUDA_CHECK(cudaEventRecord(ev, s));
      SCSF_CUDA_CHECK(cudaEventSynchronize(ev));
      if (*flag_h == 0) break;
    }
    return SCSF_OK;
  }
  cudaStreamCaptureStatus st;
  unsigned long long id = 0;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  SCSF_CUDA_CHECK(cudaStreamGetCaptureInfo(s, &st, &id, &g, &deps, &nd));
  std::vector<cudaGraphNode_t> dv(deps, deps + nd);                 // valid only until the next call
  cudaGraphConditionalHandle h;
  SCSF_CUDA_CHECK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  SCSF_CUDA_CHECK(cudaGraphAddNode(&node, g, dv.data(), dv.size(), &p));
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  static thread_local cudaStream_t side = nullptr;
  if (!side) SCSF_CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  SCSF_CUDA_CHECK(cudaStreamBeginCaptureToGraph(side, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  L.handle = h;
  L.in_graph = 1;
  const int r = body(side, L, ctx);
  cudaGraph_t out = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(side, &out);
  if (r != SCSF_OK) return r;
  SCSF_CUDA_CHECK(ce);
  size_t nn = 0;
  SCSF_CUDA_CHECK(cudaGraphGetNodes(bodyg, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  if (nn) SCSF_CUDA_CHECK(cudaGraphGetNodes(bodyg, nodes.data(), &nn));
  for (auto nd2 : nodes) {
    cudaGraphNodeType t;
    SCSF_CUDA_CHECK(cudaGraphNodeGetType(nd2, &t));
    t_cond_kernels += (t == cudaGraphNodeTypeKernel);
  }
  SCSF_CUDA_CHECK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
  return SCSF_OK;
}

}  // namespace scsf

// Device-resident PCG loop: a CUDA graph whose body (one PCG iteration, captured
// from the host launch sequence) runs under a conditional WHILE node.  The
// condition is set on the device after every iteration (relres <= tol,
// non-positive curvature, or maxit reached), so the whole solver.py:204-227
// loop runs with a single host launch and no per-iteration synchronisation.
#include "common.cuh"

namespace {

struct GraphState {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaGraphConditionalHandle handle;
  cudaGraph_t body;
  cudaGraphNode_t deps[64];
  size_t ndeps;
};

// scal slots (pcg.cu): 5 relres, 8 bad, 9 iterations done
__global__ void pcg_cond_kernel(cudaGraphConditionalHandle h, const double* __restrict__ scal, double tol, int maxit) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    bool go = !(scal[5] <= tol) && scal[8] == 0.0 && (int)scal[9] < maxit;
    cudaGraphSetConditional(h, go ? 1u : 0u);
  }
}

}  // namespace

// 1) create the graph + handle and start capturing `stream` into its top level.
extern "C" int bddc_graph_begin(void** state_out, void* stream) {
  GraphState* g = new GraphState();
  CUDA_OK(cudaGraphCreate(&g->graph, 0));
  CUDA_OK(cudaGraphConditionalHandleCreate(&g->handle, g->graph, 0, 0));
  CUDA_OK(cudaStreamBeginCaptureToGraph((cudaStream_t)stream, g->graph, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
  *state_out = g;
  return 0;
}

// 2) end the top-level capture, append the WHILE node after it, start capturing the body.
extern "C" int bddc_graph_while(void* state, void* stream) {
  GraphState* g = (GraphState*)state;
  cudaStreamCaptureStatus st;
  unsigned long long id;
  cudaGraph_t cg;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CUDA_OK(cudaStreamGetCaptureInfo((cudaStream_t)stream, &st, &id, &cg, &deps, &nd));
  if (nd > 64) return bddc_set_error(BDDC_ERR_INTERNAL, "graph: too many capture dependencies");
  for (size_t k = 0; k < nd; ++k) g->deps[k] = deps[k];
  g->ndeps = nd;
  cudaGraph_t out;
  CUDA_OK(cudaStreamEndCapture((cudaStream_t)stream, &out));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = g->handle;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CUDA_OK(cudaGraphAddNode(&node, g->graph, g->ndeps ? g->deps : nullptr, g->ndeps, &p));
  g->body = p.conditional.phGraph_out[0];
  CUDA_OK(cudaStreamBeginCaptureToGraph((cudaStream_t)stream, g->body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
  return 0;
}

// 3) end the body capture and instantiate.
extern "C" int bddc_graph_end(void* state, void* stream) {
  GraphState* g = (GraphState*)state;
  cudaGraph_t out;
  CUDA_OK(cudaStreamEndCapture((cudaStream_t)stream, &out));
  CUDA_OK(cudaGraphInstantiate(&g->exec, g->graph, 0));
  return 0;
}

extern "C" int bddc_graph_launch(void* state, void* stream) {
  GraphState* g = (GraphState*)state;
  CUDA_OK(cudaGraphLaunch(g->exec, (cudaStream_t)stream));
  return 0;
}

extern "C" int bddc_graph_destroy(void* state) {
  GraphState* g = (GraphState*)state;
  if (!g) return 0;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return 0;
}

extern "C" unsigned long long bddc_graph_handle(void* state) { return ((GraphState*)state)->handle; }

// Condition kernel: continue while not converged, no breakdown and it < maxit.
extern "C" int bddc_pcg_cond(void* state, const double* scal, double tol, int maxit, void* stream) {
  GraphState* g = (GraphState*)state;
  pcg_cond_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(g->handle, scal, tol, maxit);
  LAUNCH_OK();
  return 0;
}

// synccheck_while_repro.cu -- minimal reproduction for compute-sanitizer
// synccheck inside a CUDA-graph conditional WHILE node.
//
// The kernel is a textbook block reduction: every thread reaches every
// __syncthreads (no early return, no divergent branch around a barrier).
// It runs (a) eagerly and (b) as the body of a device-driven WHILE node
// (cudaGraphConditionalHandle, body = kernel + one-thread condition kernel),
// the same construction capi.cu uses for the PageRank loop.  Under
// `compute-sanitizer --tool synccheck` a clean (a) with a "divergent
// barrier" report for (b) shows the report comes from the conditional-node
// execution, not from the kernel's barriers.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo \
//   scripts/debug/synccheck_while_repro.cu -o /tmp/synccheck_while_repro
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::printf("CUDA %s at line %d\n", cudaGetErrorString(e_), __LINE__);      \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void block_sum(const float* x, int n, float* out) {
  __shared__ float s[256];
  float v = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v += x[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();  // reached by every thread of the block
  }
  if (threadIdx.x == 0) atomicAdd(out, s[0]);
}

__global__ void loop_cond(cudaGraphConditionalHandle h, int* left) {
  cudaGraphSetConditional(h, --*left > 0 ? 1u : 0u);
}

int main() {
  const int n = 1 << 20;
  float *x, *out;
  int* left;
  CK(cudaMalloc(&x, n * sizeof(float)));
  CK(cudaMalloc(&out, sizeof(float)));
  CK(cudaMalloc(&left, sizeof(int)));
  CK(cudaMemset(x, 0, n * sizeof(float)));
  CK(cudaMemset(out, 0, sizeof(float)));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));

  // (a) eager
  block_sum<<<64, 256, 0, s>>>(x, n, out);
  CK(cudaStreamSynchronize(s));
  std::printf("eager launch done\n");

  // (b) the same kernel as the body of a WHILE node, 3 trips
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  block_sum<<<64, 256, 0, s>>>(x, n, out);
  loop_cond<<<1, 1, 0, s>>>(h, left);
  CK(cudaStreamEndCapture(s, &body));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  const int trips = 3;
  CK(cudaMemcpyAsync(left, &trips, sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  std::printf("WHILE-node launch done\n");
  return 0;
}

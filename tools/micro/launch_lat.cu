// Launch-latency micro-benchmark: graph of N back-to-back launches.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void k_sync(int* p) { cg::this_grid().sync(); if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void k_load(const int* __restrict__ q, int* p) {
  int v = __ldcg(q + blockIdx.x * blockDim.x + threadIdx.x);
  if (v == 12345) p[0] = v;
}
__global__ void k_load2(const int* __restrict__ q, int* p) {
  int v = __ldcg(q + blockIdx.x * blockDim.x + threadIdx.x);
  v = __ldcg(q + (v & 1023) + 4096);
  if (v == 12345) p[0] = v;
}
template <typename F>
float time_graph(F launch, int n) {
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1e3f / (10 * n);
}
int main() {
  int* p; cudaMalloc(&p, 64 << 20);
  cudaMemset(p, 0, 64 << 20);
  const int N = 50;
  for (int grid : {1, 16, 32, 148}) {
    for (int bs : {256, 1024}) {
      float t0 = time_graph([&](cudaStream_t s) { k_empty<<<grid, bs, 0, s>>>(p); }, N);
      float t1 = time_graph([&](cudaStream_t s) {
        void* args[] = {&p};
        cudaLaunchCooperativeKernel((void*)k_empty, grid, bs, args, 0, s); }, N);
      float t2 = time_graph([&](cudaStream_t s) {
        void* args[] = {&p};
        cudaLaunchCooperativeKernel((void*)k_sync, grid, bs, args, 0, s); }, N);
      float t3 = time_graph([&](cudaStream_t s) { k_load<<<grid, bs, 0, s>>>(p + 1024, p); }, N);
      float t4 = time_graph([&](cudaStream_t s) { k_load2<<<grid, bs, 0, s>>>(p + 1024, p); }, N);
      printf("grid %3d x %4d: empty %.2f  coop-empty %.2f  coop-gridsync %.2f  1-load %.2f  2-dep-loads %.2f us\n",
             grid, bs, t0, t1, t2, t3, t4);
    }
  }
  return 0;
}

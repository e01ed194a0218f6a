// Probe: host cost of cudaLaunchCooperativeKernel vs a plain launch (empty kernels, 296 CTAs).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  int* p = nullptr;
  void* args[] = {&p};
  for (int i = 0; i < 100; ++i) k_empty<<<296, 256, 0, s>>>(p);
  cudaStreamSynchronize(s);
  const int N = 2000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) k_empty<<<296, 256, 0, s>>>(p);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) cudaLaunchCooperativeKernel((const void*)k_empty, dim3(296), dim3(256), args, 0, s);
  auto t3 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  printf("plain launch %.2f us/launch, cooperative %.2f us/launch (%s)\n", us(t0, t1) / N,
         us(t2, t3) / N, cudaGetErrorString(cudaGetLastError()));
  // latency: launch + sync, one at a time
  double lp = 0, lc = 0;
  for (int i = 0; i < 200; ++i) {
    auto a = std::chrono::steady_clock::now();
    k_empty<<<296, 256, 0, s>>>(p); cudaStreamSynchronize(s);
    auto b = std::chrono::steady_clock::now();
    cudaLaunchCooperativeKernel((const void*)k_empty, dim3(296), dim3(256), args, 0, s); cudaStreamSynchronize(s);
    auto c = std::chrono::steady_clock::now();
    lp += us(a, b); lc += us(b, c);
  }
  printf("launch+sync latency: plain %.2f us, cooperative %.2f us\n", lp / 200, lc / 200);
}

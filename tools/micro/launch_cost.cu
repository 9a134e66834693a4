// Host-side cost of the launch flavours k_fbsp could use (diagnostic).
#include <cooperative_groups.h>
#include <chrono>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_empty(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
__global__ void k_sync(int* p) { cg::this_grid().sync(); if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
int main() {
  int* d; cudaMalloc(&d, 64);
  cudaStream_t s; cudaStreamCreate(&s);
  void* args[] = {&d};
  auto host_us = [&](auto fn, int reps) {
    for (int i = 0; i < 20; ++i) fn();
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) fn();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
  };
  auto rt_us = [&](auto fn, int reps) {  // launch + sync round trip
    for (int i = 0; i < 20; ++i) { fn(); cudaStreamSynchronize(s); }
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) { fn(); cudaStreamSynchronize(s); }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
  };
  for (int G : {148, 296}) {
    auto plain = [&] { k_empty<<<G, 256, 0, s>>>(d); };
    auto coop = [&] { cudaLaunchCooperativeKernel((void*)k_empty, G, 256, args, 0, s); };
    auto coop_sync = [&] { cudaLaunchCooperativeKernel((void*)k_sync, G, 256, args, 0, s); };
    printf("G=%d host issue: plain %.2f us, coop %.2f us | round trip: plain %.2f, coop %.2f, coop+grid.sync %.2f us\n", G,
           host_us(plain, 2000), host_us(coop, 2000), rt_us(plain, 2000), rt_us(coop, 2000), rt_us(coop_sync, 2000));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("event record: %.2f us\n", host_us([&] { cudaEventRecord(e0, s); }, 2000));
  int* h; cudaMallocHost(&h, 4096);
  printf("memcpy H2D 4KB pinned async: %.2f us\n", host_us([&] { cudaMemcpyAsync(d, h, 64, cudaMemcpyHostToDevice, s); }, 2000));
  printf("memset async: %.2f us\n", host_us([&] { cudaMemsetAsync(d, 0, 64, s); }, 2000));
  printf("D2H 64B + sync round trip: %.2f us\n", rt_us([&] { cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, s); }, 2000));
  return 0;
}

// Grid-barrier latency on the B200 (diagnostic): cooperative_groups grid.sync()
// against a flag barrier (one arrival counter, generation word, release /
// acquire ordering).  usage: ./gridbar
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x ^ i;
    g.sync();
  }
  if (x == 0xFFFFFFFF) *sink = x;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__global__ void k_flag(int iters, unsigned* bar, unsigned* sink) {
  unsigned x = 0;
  const unsigned G = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x ^ i;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned gen = ld_acquire(bar + 32);
      if (atom_add_acqrel(bar, 1u) == G - 1) {
        bar[0] = 0;
        st_release(bar + 32, gen + 1);
      } else {
        while (ld_acquire(bar + 32) == gen) {
        }
      }
    }
    __syncthreads();
  }
  if (x == 0xFFFFFFFF) *sink = x;
}

int main() {
  unsigned *bar, *sink;
  cudaMalloc(&bar, 256);
  cudaMalloc(&sink, 4);
  cudaMemset(bar, 0, 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int G : {148, 296}) {
    for (int kind = 0; kind < 2; ++kind) {
      int iters = 2000;
      void* args0[] = {&iters, &sink};
      void* args1[] = {&iters, &bar, &sink};
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (kind == 0) cudaLaunchCooperativeKernel((void*)k_cg, G, 256, args0, 0, 0);
        else cudaLaunchCooperativeKernel((void*)k_flag, G, 256, args1, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) printf("G=%d %s: %.3f us per barrier (%s)\n", G, kind ? "flag" : "cg", ms * 1e3 / iters,
                             cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}

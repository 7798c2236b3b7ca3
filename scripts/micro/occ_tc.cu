// Does tcgen05 use change the occupancy the runtime reports? Prints
// cudaOccupancyMaxActiveBlocksPerMultiprocessor for 256-thread kernels with
// and without tcgen05.alloc / printf / trap.
#include <cstdio>
__global__ void __launch_bounds__(256, 2) plain(int* o) { o[threadIdx.x] = threadIdx.x; }
__global__ void __launch_bounds__(256, 2) with_tc(int* o) {
  __shared__ unsigned base;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  o[threadIdx.x] = base;
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(128));
}
__global__ void __launch_bounds__(256, 2) with_printf(int* o) {
  if (o[threadIdx.x] == 12345) printf("x\n");
  o[threadIdx.x] = 1;
}
__global__ void __launch_bounds__(256, 2) with_trap(int* o) {
  if (o[threadIdx.x] == 12345) asm volatile("trap;");
  o[threadIdx.x] = 1;
}
template <typename K>
void rep(const char* n, K k) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int kb : {0, 16, 32, 48, 64, 90, 100, 110}) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, kb * 1024);
    printf("%-12s %d CTA/SM at %d KB dynamic smem\n", n, nb, kb);
  }
  for (int th : {128, 512}) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, th, 0);
    printf("%-12s %d CTA/SM at %d threads\n", n, nb, th);
  }
}
int main() {
  rep("plain", plain);
  rep("tcgen05", with_tc);
  rep("printf", with_printf);
  rep("trap", with_trap);
  return 0;
}

// Queued launch cost vs kernel-parameter size, with the throughput kernel's grid
// shape (148 CTAs x 512 threads) -- experiment aid (round 3 of the launch analysis).
// Each timed launch is queued behind a device-side sleep, so the host's submission
// is hidden and the event pair measures the GPU's own launch processing + run.
#include <cuda_runtime.h>
#include <stdio.h>
template <int N> struct P { unsigned v[N]; };
__global__ void sleeper(long long ns) {
  long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); if (t - t0 > ns) break; }
}
template <int N> __global__ void k(const __grid_constant__ P<N> p, unsigned* o) {
  if (threadIdx.x == 0) o[blockIdx.x] = p.v[(blockIdx.x * 7) % N];
}
template <int N> void run(unsigned* o, int grid, int block) {
  P<N> p; for (int i = 0; i < N; ++i) p.v[i] = i;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) k<N><<<grid, block>>>(p, o);
  cudaDeviceSynchronize();
  float v[41]; int n = 41;
  for (int r = 0; r < n; ++r) {
    sleeper<<<1, 1>>>(200000);
    cudaEventRecord(a); k<N><<<grid, block>>>(p, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&v[r], a, b);
  }
  for (int i = 0; i < n; ++i) for (int j = i + 1; j < n; ++j) if (v[j] < v[i]) { float t = v[i]; v[i] = v[j]; v[j] = t; }
  cudaEventRecord(a); for (int r = 0; r < 200; ++r) k<N><<<grid, block>>>(p, o); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("param %6d B grid %4d x %4d: queued median %.2f us (p10 %.2f); back-to-back %.2f us/launch\n", N * 4, grid, block,
         1000 * v[n / 2], 1000 * v[n / 10], 1000 * ms / 200);
}
int main() {
  unsigned* o; cudaMalloc(&o, 4096 * 4);
  for (int g : {1, 148}) {
    run<4>(o, g, 512); run<96>(o, g, 512); run<512>(o, g, 512); run<1024>(o, g, 512); run<2048>(o, g, 512);
    run<2304>(o, g, 512); run<4096>(o, g, 512); run<8000>(o, g, 512);
  }
  return 0;
}

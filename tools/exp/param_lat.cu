// Launch latency vs kernel-parameter size (experiment).
#include <cuda_runtime.h>
#include <stdio.h>
template <int N> struct P { unsigned v[N]; };
template <int N> __global__ void k(const __grid_constant__ P<N> p, unsigned* o) { if (threadIdx.x == 0 && blockIdx.x == 0) o[0] = p.v[N - 1]; }
template <int N> float run(unsigned* o, int reps) {
  P<N> p; for (int i = 0; i < N; ++i) p.v[i] = i;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) k<N><<<1, 32>>>(p, o);
  cudaDeviceSynchronize();
  float best = 1e9, tot = 0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); k<N><<<1, 32>>>(p, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); tot += ms; if (ms < best) best = ms;
  }
  // back-to-back throughput
  cudaEventRecord(a); for (int r = 0; r < 100; ++r) k<N><<<1, 32>>>(p, o); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms100; cudaEventElapsedTime(&ms100, a, b);
  printf("param %6d B: single launch median-ish %.1f us (best %.1f us); back-to-back %.2f us/launch\n", N * 4, 1000 * tot / reps, 1000 * best, 10 * ms100);
  return best;
}
int main() {
  unsigned* o; cudaMalloc(&o, 4);
  run<16>(o, 50); run<1024>(o, 50); run<2304>(o, 50); run<4608>(o, 50); run<8000>(o, 50);
  return 0;
}

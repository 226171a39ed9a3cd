// FP64 add throughput and dependent-add latency on this GPU (the second roof
// of the cost build): the K1 cell chains are strictly
// sequential fp64 adds, so its floor is max(bytes / HBM, adds / DADD peak).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dadd_peak tools/dadd_peak.cu
#include <cstdio>

constexpr int CHAINS = 8, ITERS = 4096;

__global__ void k_dadd_tput(double* out, double u) {
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = __dadd_rn(c[i], u);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dadd_latency(double* out, long long* cyc, double u) {
  double c = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) c = __dadd_rn(c, u);
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = c;
    cyc[0] = t1 - t0;
  }
}

int main() {
  double* d;
  long long* cyc;
  cudaMalloc(&d, 8);
  cudaMalloc(&cyc, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 2, threads = 1024;
  k_dadd_tput<<<blocks, threads>>>(d, 1e-7);  // warm-up
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) k_dadd_tput<<<blocks, threads>>>(d, 1e-7);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double adds = 10.0 * blocks * threads * CHAINS * static_cast<double>(ITERS);
  std::printf("{\"dadd_per_s\": %.4e, \"sms\": %d", adds / (ms * 1e-3), sms);
  k_dadd_latency<<<1, 32>>>(d, cyc, 1e-7);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  std::printf(", \"dadd_dependent_latency_cycles\": %.2f}\n", static_cast<double>(h) / ITERS);
  return 0;
}

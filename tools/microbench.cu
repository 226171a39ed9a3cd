// Latency microbenchmarks of the primitives on the exact solver's critical
// path (one warp, dependent chains, clock64).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;

__global__ void k_lds_chase(int* out, long long* cyc) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) nxt[i] = (i * 7 + 13) & 1023;
  __syncwarp();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) p = nxt[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_generic_chase(int* out, long long* cyc, int use_global, int* g) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) nxt[i] = (i * 7 + 13) & 1023;
  __syncwarp();
  volatile int* base = use_global ? g : nxt;  // generic pointer
  int* b = (int*)base;
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) p = b[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_shfl32(int* out, long long* cyc) {
  int v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// one round of a packed 64-bit min: 2 SHFL + 64-bit compare + select
__global__ void k_min64_round(long long* out, long long* cyc) {
  long long v = threadIdx.x * 12345ll;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    long long o = __shfl_xor_sync(0xffffffffu, v, 1);
    v = (o < v ? o : v) + 3;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_redux(int* out, long long* cyc) {
  unsigned v = threadIdx.x * 77u;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) v = __reduce_min_sync(0xffffffffu, v + threadIdx.x) + 1;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_ballot(int* out, long long* cyc) {
  unsigned v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) v = __ffs(__ballot_sync(0xffffffffu, (v & 1) == (threadIdx.x & 1))) + v;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// single-thread 8-way min over packed 64-bit keys computed from a dependent base
__global__ void k_min8_thread(long long* out, long long* cyc, const long long* in) {
  long long a[8];
  for (int q = 0; q < 8; ++q) a[q] = in[q];
  long long base = 0;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    long long k[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) k[q] = ((a[q] - base) << 6) | q;
    long long m0 = k[0] < k[1] ? k[0] : k[1];
    long long m1 = k[2] < k[3] ? k[2] : k[3];
    long long m2 = k[4] < k[5] ? k[4] : k[5];
    long long m3 = k[6] < k[7] ? k[6] : k[7];
    long long n0 = m0 < m1 ? m0 : m1;
    long long n1 = m2 < m3 ? m2 : m3;
    long long m = n0 < n1 ? n0 : n1;
    base += (m >> 6) & 7;
  }
  long long t1 = clock64();
  out[0] = base;
  *cyc = t1 - t0;
}

int main() {
  int* d_out;
  long long *d_cyc, *d_l, h;
  int* g;
  cudaMalloc(&d_out, 4096);
  cudaMalloc(&d_cyc, 8);
  cudaMalloc(&d_l, 4096);
  cudaMalloc(&g, 4096 * 4);
  int hg[4096];
  for (int i = 0; i < 4096; ++i) hg[i] = (i * 7 + 13) & 1023;
  cudaMemcpy(g, hg, sizeof hg, cudaMemcpyHostToDevice);
  auto rep = [&](const char* name) {
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d_cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cycles/iter\n", name, (double)h / ITERS);
  };
  for (int r = 0; r < 2; ++r) {
    k_lds_chase<<<1, 32>>>(d_out, d_cyc); rep("LDS pointer chase");
    k_generic_chase<<<1, 32>>>(d_out, d_cyc, 0, g); rep("generic->smem chase");
    k_generic_chase<<<1, 32>>>(d_out, d_cyc, 1, g); rep("generic->global(L1) chase");
    k_shfl32<<<1, 32>>>(d_out, d_cyc); rep("SHFL.BFLY 32 + IADD");
    k_min64_round<<<1, 32>>>(d_l, d_cyc); rep("packed min64 round");
    k_redux<<<1, 32>>>(d_out, d_cyc); rep("REDUX.MIN u32 + IADD");
    k_ballot<<<1, 32>>>(d_out, d_cyc); rep("VOTE.BALLOT + FFS");
    k_min8_thread<<<1, 1>>>(d_l, d_cyc, d_l + 8); rep("1-thread 8-way min64");
  }
  return 0;
}

// Microbenchmark of the exact solver's row-end table refresh (the fused
// potentials + operand-table pass of k_hungarian_blocks_mw) in isolation:
// one CTA of 8 warps, the same shared-memory layout and sizes as a C2 solve
// (k = 512, n = 8), 512 synthetic rows of ~108 reached columns each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rowend_bench tools/rowend_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int K = 512, N = 8, ROWS = 512, NU = 108;

template <int VARIANT>
__global__ void __launch_bounds__(256, 1)
    k_rowend(const int32_t* __restrict__ g_ulist, long long* out_cycles, int64_t* sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int K1 = K + 1;
  int64_t* S = reinterpret_cast<int64_t*>(smem);
  int64_t* A = S + K * N;
  int64_t* Btab = A + K * N;
  int64_t* u = Btab + K1;
  int64_t* v = u + K1;
  int64_t* dlt = v + K1;
  int32_t* p = reinterpret_cast<int32_t*>(dlt + K1);
  int32_t* rtab = p + K1;
  int32_t* cblk = rtab + K1;
  int32_t* ulist = cblk + K1;
  for (int x = tid; x < K * N; x += blockDim.x) S[x] = x * 7;
  for (int x = tid; x < K1; x += blockDim.x) {
    u[x] = x;
    v[x] = -x;
    dlt[x] = x & 15;
    p[x] = x == 0 ? 1 : ((x * 37) % K) + 1;
    cblk[x] = x / 64;
  }
  __syncthreads();
  const int n = N, nu = NU;
  const int64_t Dl = 100;
  long long wtime = 0;
  for (int row = 0; row < ROWS; ++row) {
    for (int x = tid; x < nu; x += blockDim.x) ulist[x] = g_ulist[row * NU + x];
    __syncthreads();
    const long long tw0 = clock64();
    const int gs = 8;
    const int gpw = 32 / gs, sub = lane / gs, lw = lane - sub * gs;
    const int stride = nw * gpw;
    if constexpr (VARIANT == 0 || VARIANT == 1) {
      for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
        const int e0 = eb + sub, e1 = e0 + stride;
        const bool act0 = e0 < nu, act1 = e1 < nu;
        const int c0 = act0 ? ulist[e0] : 0, c1 = act1 ? ulist[e1] : 0;
        const int r0 = act0 ? p[c0] : 0, r1 = act1 ? p[c1] : 0;
        const int64_t dd0 = act0 ? Dl - dlt[c0] : 0, dd1 = act1 ? Dl - dlt[c1] : 0;
        const int64_t u0 = act0 ? u[r0] + dd0 : 0, u1 = act1 ? u[r1] + dd1 : 0;
        const int64_t v0 = act0 ? v[c0] - dd0 : 0, v1 = act1 ? v[c1] - dd1 : 0;
        const int64_t s0 = (act0 && r0 > 0 && lw < n) ? S[(r0 - 1) * n + lw] : 0;
        const int64_t s1 = (act1 && r1 > 0 && lw < n) ? S[(r1 - 1) * n + lw] : 0;
        if (VARIANT == 0) __syncwarp();
        if (lw == 0 && act0) {
          u[r0] = u0;
          v[c0] = v0;
          if (c0 != 0) {
            rtab[c0] = r0;
            Btab[c0] = static_cast<int64_t>(cblk[c0]) - (v0 << 6);
          }
        }
        if (lw == 0 && act1) {
          u[r1] = u1;
          v[c1] = v1;
          rtab[c1] = r1;
          Btab[c1] = static_cast<int64_t>(cblk[c1]) - (v1 << 6);
        }
        if (lw < n) {
          if (act0 && c0 != 0 && r0 > 0) A[(c0 - 1) * n + lw] = (s0 - u0) << 6;
          if (act1 && r1 > 0) A[(c1 - 1) * n + lw] = (s1 - u1) << 6;
        }
      }
    } else if constexpr (VARIANT == 2) {  // loads only
      int64_t acc = 0;
      for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
        const int e0 = eb + sub, e1 = e0 + stride;
        const bool act0 = e0 < nu, act1 = e1 < nu;
        const int c0 = act0 ? ulist[e0] : 0, c1 = act1 ? ulist[e1] : 0;
        const int r0 = act0 ? p[c0] : 0, r1 = act1 ? p[c1] : 0;
        const int64_t dd0 = act0 ? Dl - dlt[c0] : 0, dd1 = act1 ? Dl - dlt[c1] : 0;
        const int64_t u0 = act0 ? u[r0] + dd0 : 0, u1 = act1 ? u[r1] + dd1 : 0;
        const int64_t s0 = (act0 && r0 > 0) ? S[(r0 - 1) * n + lw] : 0;
        const int64_t s1 = (act1 && r1 > 0) ? S[(r1 - 1) * n + lw] : 0;
        acc += u0 + u1 + s0 + s1;
      }
      if (acc == 123456789) sink[0] = acc;
    } else if constexpr (VARIANT == 4) {  // the 3-level chain, 8 times back to back
      int64_t acc = 0;
      for (int rep = 0; rep < 8; ++rep)
        for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
          const int e0 = eb + sub;
          const int c0 = e0 < nu ? ulist[e0] : 0;
          const int r0 = p[(c0 + static_cast<int>(acc & 1)) % K1];
          acc += u[r0];
        }
      if (acc == 123456789) sink[0] = acc;
    } else if constexpr (VARIANT == 5) {  // warp 0 alone
      int64_t acc = 0;
      if (warp == 0)
        for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
          const int e0 = eb + sub;
          const int c0 = e0 < nu ? ulist[e0] : 0;
          const int r0 = p[c0];
          acc += u[r0];
        }
      if (acc == 123456789) sink[0] = acc;
    } else if constexpr (VARIANT == 6) {  // lane-uniform addresses (pure broadcast chain)
      int64_t acc = 0;
      for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
        const int c0 = ulist[eb];
        const int r0 = p[c0];
        acc += u[r0];
      }
      if (acc == 123456789) sink[0] = acc;
    } else if constexpr (VARIANT == 7) {  // 16 x barrier
      for (int q = 0; q < 16; ++q) __syncthreads();
    } else if constexpr (VARIANT == 8) {  // 16 x (publish STS, barrier, LDS, REDUX.OR): a chunk exchange
      unsigned acc = 0;
      uint32_t* slot = reinterpret_cast<uint32_t*>(ulist + 200);
      for (int q = 0; q < 16; ++q) {
        if (lane == 0) slot[(q & 1) * 32 + warp] = acc + q;
        __syncthreads();
        acc = __reduce_or_sync(0xffffffffu, lane < 8 ? slot[(q & 1) * 32 + lane] : 0u);
      }
      if (acc == 123456789) sink[0] = acc;
    } else if constexpr (VARIANT == 9) {  // 16 x (publish STS, bar.red.or as the exchange)
      unsigned acc = 0;
      for (int q = 0; q < 16; ++q) acc += __syncthreads_or((acc + q + lane) == 7);
      if (acc == 123456789) sink[0] = acc;
    } else {  // VARIANT 3: a single LDS chain of the same depth (ulist -> p -> u)
      int64_t acc = 0;
      for (int eb = warp * gpw; eb < nu; eb += 2 * stride) {
        const int e0 = eb + sub;
        const int c0 = e0 < nu ? ulist[e0] : 0;
        const int r0 = p[c0];
        acc += u[r0];
      }
      if (acc == 123456789) sink[0] = acc;
    }
    const long long tw1 = clock64();
    wtime += tw1 - tw0;
    __syncthreads();
  }
  if (lane == 0) out_cycles[warp] = wtime;
}

template <int V>
void run(const int32_t* d_ul, long long* d_out, int64_t* d_sink, size_t smem, const char* name) {
  cudaFuncSetAttribute(k_rowend<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_rowend<V><<<1, 256, smem>>>(d_ul, d_out, d_sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (long long x : h) mx = x > mx ? x : mx;
  std::printf("%-28s %s max warp cycles/row %.0f\n", name, cudaGetErrorString(e), double(mx) / ROWS);
}

int main() {
  std::vector<int32_t> ul(ROWS * NU);
  std::srand(1);
  for (int r = 0; r < ROWS; ++r) {
    ul[r * NU] = 0;
    for (int e = 1; e < NU; ++e) ul[r * NU + e] = 1 + (std::rand() % K);
  }
  int32_t* d_ul;
  long long* d_out;
  int64_t* d_sink;
  cudaMalloc(&d_ul, ul.size() * 4);
  cudaMalloc(&d_out, 8 * 8);
  cudaMalloc(&d_sink, 8);
  cudaMemcpy(d_ul, ul.data(), ul.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (2 * K * N + 4 * (K + 1)) * 8 + 4 * (K + 1) * 4;
  run<0>(d_ul, d_out, d_sink, smem, "fused (syncwarp)");
  run<1>(d_ul, d_out, d_sink, smem, "fused (no syncwarp)");
  run<2>(d_ul, d_out, d_sink, smem, "loads only");
  run<3>(d_ul, d_out, d_sink, smem, "3-level LDS chain");
  run<4>(d_ul, d_out, d_sink, smem, "chain x8 (per row total)");
  run<5>(d_ul, d_out, d_sink, smem, "chain, warp 0 alone");
  run<6>(d_ul, d_out, d_sink, smem, "chain, uniform addresses");
  run<7>(d_ul, d_out, d_sink, smem, "16 x barrier");
  run<8>(d_ul, d_out, d_sink, smem, "16 x STS+bar+LDS+REDUX");
  run<9>(d_ul, d_out, d_sink, smem, "16 x bar.red.or");
  return 0;
}

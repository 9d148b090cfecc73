// Microbenchmark (not product code): HBM ceiling of the stock VecEnv step's memory
// pattern with the compute removed.  Per env: read actions 120 B + shares 120 B +
// balance/return 16 B; write shares 120 B + balance/return 16 B + obs 724 B + reward 4 B
// + done 1 B (1,121 B), N = 1M envs, 64 envs per CTA, the obs row written warp-per-row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mb_envbw.cu -o mb_envbw
#include <cstdio>
#include <cstdint>

constexpr int K = 30, S = 181, B = 64;

template <int MODE>
__global__ void __launch_bounds__(B) pattern(int N, const float* __restrict__ act, int32_t* __restrict__ sh,
                                             double* __restrict__ bal, double* __restrict__ ret,
                                             const float* __restrict__ feat, float* __restrict__ obs,
                                             float* __restrict__ rew, uint8_t* __restrict__ done) {
  __shared__ float priv[B][K + 2];
  const int tid = threadIdx.x;
  const size_t e = (size_t)blockIdx.x * B + tid;
  float a = 0.f;
  const float2* ar = reinterpret_cast<const float2*>(act + e * K);
#pragma unroll
  for (int j = 0; j < K / 2; ++j) { float2 v = ar[j]; a += v.x + v.y; }
  int32_t s[K];
#pragma unroll
  for (int k = 0; k < K; ++k) s[k] = sh[(size_t)k * N + e];
  double b = bal[e], r = ret[e];
#pragma unroll
  for (int k = 0; k < K; ++k) { s[k] += (a > 100.f); priv[tid][1 + k] = (float)s[k]; }
  priv[tid][0] = (float)b;
#pragma unroll
  for (int k = 0; k < K; ++k) sh[(size_t)k * N + e] = s[k];
  bal[e] = b + 1.0; ret[e] = r + 1.0; rew[e] = a; done[e] = 0;
  __syncthreads();
  if (MODE == 0) {
    const int lane = tid & 31, w = tid >> 5;
    for (int row = w; row < B; row += B / 32) {
      float* o = obs + ((size_t)blockIdx.x * B + row) * S;
      for (int c = lane; c < S; c += 32) o[c] = (c <= K) ? priv[row][c] : feat[c - K - 1];
    }
  } else {  // the CTA's 64 rows are one contiguous, 16 B-aligned span: float4 stream
    float4* o = reinterpret_cast<float4*>(obs + (size_t)blockIdx.x * B * S);
    for (int i = tid; i < B * S / 4; i += B) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int f = 4 * i + u, row = f / S, c = f - row * S;
        v[u] = (c <= K) ? priv[row][c] : feat[c - K - 1];
      }
      o[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

__global__ void write_only(float4* __restrict__ o, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    o[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
  const int N = 1 << 20;
  float *act, *feat, *obs, *rew; int32_t* sh; double *bal, *ret; uint8_t* done;
  cudaMalloc(&act, (size_t)N * K * 4); cudaMalloc(&sh, (size_t)N * K * 4); cudaMalloc(&bal, N * 8); cudaMalloc(&ret, N * 8);
  cudaMalloc(&feat, 150 * 4); cudaMalloc(&obs, (size_t)N * S * 4); cudaMalloc(&rew, N * 4); cudaMalloc(&done, N);
  cudaMemset(act, 0, (size_t)N * K * 4); cudaMemset(sh, 0, (size_t)N * K * 4); cudaMemset(feat, 0, 600);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20;
  auto run = [&](auto kern, const char* what) {
    for (int it = 0; it < 3; ++it) kern<<<N / B, B>>>(N, act, sh, bal, ret, feat, obs, rew, done);
    cudaEventRecord(e0);
    for (int it = 0; it < iters; ++it) kern<<<N / B, B>>>(N, act, sh, bal, ret, feat, obs, rew, done);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / iters, bytes = 1121.0 * N;
    printf("%-40s %.1f us/step  %.0f GB/s  (%.1f%% of 6535.7)  err=%s\n", what, us, bytes / us / 1e3,
           100 * bytes / us / 1e3 / 6535.7, cudaGetErrorString(cudaGetLastError()));
  };
  run(pattern<0>, "pattern, warp-per-row obs");
  run(pattern<1>, "pattern, float4 block obs");
  {
    const size_t n4 = (size_t)N * S / 4;
    for (int it = 0; it < 3; ++it) write_only<<<148 * 8, 512>>>(reinterpret_cast<float4*>(obs), n4);
    cudaEventRecord(e0);
    for (int it = 0; it < iters; ++it) write_only<<<148 * 8, 512>>>(reinterpret_cast<float4*>(obs), n4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / iters;
    printf("%-40s %.1f us  %.0f GB/s (%.1f%%)\n", "write-only obs stream", us, n4 * 16.0 / us / 1e3, 100 * n4 * 16.0 / us / 1e3 / 6535.7);
  }
  return 0;
}

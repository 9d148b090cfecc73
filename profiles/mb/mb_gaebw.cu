// Microbenchmark (not product code): HBM ceiling of the GAE pass's memory traffic with the
// recursion removed.  Time-major [H][N] buffers, N = 65,536 envs, H = 256: read r, V (fp32)
// and done (u8), write adv, ret (fp32) -- 17 B per transition, 285 MB per pass (configs[1]).
//   MODE 0: flat float4 grid-stride stream (the best case for these bytes)
//   MODE 1: one thread per (env, step), warp = 32 envs of one step row (the GAE kernels' rows)
// Run between passes: a 512 MB scrub so every pass starts from DRAM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mb_gaebw.cu -o mb_gaebw
#include <cstdint>
#include <cstdio>

__global__ void flat(size_t n4, const float4* __restrict__ r, const float4* __restrict__ v,
                     const uchar4* __restrict__ d, float4* __restrict__ a, float4* __restrict__ t) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 x = __ldcs(r + i), y = __ldcs(v + i);
    const uchar4 z = d[i];
    __stcs(a + i, make_float4(x.x + z.x, x.y + z.y, x.z + z.z, x.w + z.w));
    __stcs(t + i, make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w));
  }
}

__global__ void rows(int N, int H, const float* __restrict__ r, const float* __restrict__ v,
                     const uint8_t* __restrict__ d, float* __restrict__ a, float* __restrict__ t) {
  const int e = blockIdx.x * 32 + (threadIdx.x & 31);
  for (int h = threadIdx.x >> 5; h < H; h += blockDim.x >> 5) {
    const size_t j = (size_t)h * N + e;
    const float x = __ldcs(r + j), y = __ldcs(v + j);
    const uint8_t z = d[j];
    __stcs(a + j, x + z);
    __stcs(t + j, x + y);
  }
}

// MODE 2: row segments of 32*V envs per warp (V consecutive floats per lane as one vector
// access), the granularity a wider env group per CTA would give
template <int V> struct Vec;
template <> struct Vec<2> { using F = float2; using U = uchar2; };
template <> struct Vec<4> { using F = float4; using U = uchar4; };
__device__ __forceinline__ float2 op(float2 x, uchar2 z) { return make_float2(x.x + z.x, x.y + z.y); }
__device__ __forceinline__ float4 op(float4 x, uchar4 z) { return make_float4(x.x + z.x, x.y + z.y, x.z + z.z, x.w + z.w); }
__device__ __forceinline__ float2 op2(float2 x, float2 y) { return make_float2(x.x + y.x, x.y + y.y); }
__device__ __forceinline__ float4 op2(float4 x, float4 y) { return make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w); }
template <int V>
__global__ void rowsE(int N, int H, const float* __restrict__ r, const float* __restrict__ v,
                      const uint8_t* __restrict__ d, float* __restrict__ a, float* __restrict__ t) {
  using F = typename Vec<V>::F;
  using U = typename Vec<V>::U;
  const int e = blockIdx.x * 32 * V + (threadIdx.x & 31) * V;
  for (int h = threadIdx.x >> 5; h < H; h += blockDim.x >> 5) {
    const size_t j = (size_t)h * N + e;
    const F x = __ldcs(reinterpret_cast<const F*>(r + j)), y = __ldcs(reinterpret_cast<const F*>(v + j));
    const U z = *reinterpret_cast<const U*>(d + j);
    __stcs(reinterpret_cast<F*>(a + j), op(x, z));
    __stcs(reinterpret_cast<F*>(t + j), op2(x, y));
  }
}

__global__ void scrub(float4* p, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
  const int N = 65536, H = 256;
  const size_t n = (size_t)N * H;
  float *r, *v, *a, *t;
  uint8_t* d;
  float4* big;
  cudaMalloc(&r, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&a, n * 4); cudaMalloc(&t, n * 4); cudaMalloc(&d, n);
  cudaMalloc(&big, 512u << 20);
  cudaMemset(r, 0, n * 4); cudaMemset(v, 0, n * 4); cudaMemset(d, 0, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 3; ++mode)
    for (int cfg = 0; cfg < 3; ++cfg) {
      float best = 1e9f, sum = 0.f;
      for (int rep = 0; rep < 8; ++rep) {
        scrub<<<sms * 8, 256>>>(big, (512u << 20) / 16);
        cudaEventRecord(e0);
        if (mode == 0) {
          const int blocks[3] = {sms * 4, sms * 8, sms * 16};
          flat<<<blocks[cfg], 256>>>(n / 4, (const float4*)r, (const float4*)v, (const uchar4*)d, (float4*)a,
                                      (float4*)t);
        } else if (mode == 1) {
          const int thr[3] = {256, 512, 1024};
          rows<<<N / 32, thr[cfg]>>>(N, H, r, v, d, a, t);
        } else if (cfg == 0) {
          rowsE<2><<<N / 64, 512>>>(N, H, r, v, d, a, t);
        } else if (cfg == 1) {
          rowsE<4><<<N / 128, 512>>>(N, H, r, v, d, a, t);
        } else {
          rowsE<4><<<N / 128, 1024>>>(N, H, r, v, d, a, t);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) { best = ms < best ? ms : best; sum += ms; }
      }
      const double bytes = 17.0 * n;
      printf("mode %d cfg %d: best %.1f us (%.0f GB/s), mean %.1f us (%.0f GB/s)\n", mode, cfg, best * 1e3,
             bytes / (best * 1e-3) / 1e9, sum / 7 * 1e3, bytes / (sum / 7 * 1e-3) / 1e9);
    }
  return 0;
}

// Microbenchmark (not product code): per-SM L2 -> shared-memory streaming rate
// by path: 1-D bulk copies (1 or 2 issuing threads, 8/16/32 KB), LDGSTS
// (cp.async 16 B/thread by 4 warps), and plain LDG.128 + STS.128 by 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2112_05923_b200/csrc mb_l2smem.cu -o mb_l2smem
#include <cstdio>
#include <cstdint>
#include "tc.cuh"
using namespace prb;

constexpr int kTotal = 64 << 20;  // bytes streamed per CTA
constexpr int kSrc = 1 << 20;     // L2-resident source window

__global__ void __launch_bounds__(256, 1) bulk(const uint8_t* src, int chunk, int producers, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) for (int i = 0; i < 8; ++i) tc::mbar_init(&full[i], 1);
  __syncthreads();
  const int n = kTotal / chunk;
  unsigned long long t0 = clock64();
  if (lane == 0 && warp < producers) {
    // 8 slots; producer p owns slots p, p+producers, ...; waits its own previous copy into that slot
    int k = 0;
    for (int it = warp; it < n; it += producers, ++k) {
      const int slot = it % 8;
      if (it >= 8) tc::mbar_wait(&full[slot], ((it / 8) - 1) & 1);
      tc::mbar_arrive_expect_tx(&full[slot], chunk);
      tc::bulk_g2s(sm + slot * chunk, src + ((size_t)it * chunk) % kSrc, chunk, &full[slot]);
    }
    for (int it = n - 8 + warp; it < n; it += producers) if (it >= 0) tc::mbar_wait(&full[it % 8], (it / 8) & 1);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void __launch_bounds__(256, 1) ldgsts(const uint8_t* src, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  unsigned long long t0 = clock64();
  const int tid = threadIdx.x;
  for (size_t off = 0; off < (size_t)kTotal; off += 256 * 16 * 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t o = off + (size_t)u * 4096 + tid * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(sm + (o % 65536))), "l"(src + o % kSrc));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 6;");
  }
  asm volatile("cp.async.wait_all;");
  __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void __launch_bounds__(256, 1) ldgsts_plain(const uint8_t* src, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  unsigned long long t0 = clock64();
  const int tid = threadIdx.x;
  for (size_t off = 0; off < (size_t)kTotal; off += 256 * 16 * 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(reinterpret_cast<const uint4*>(src + (off + (size_t)u * 4096 + tid * 16) % kSrc));
#pragma unroll
    for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(sm + (off + (size_t)u * 4096 + tid * 16) % 65536) = v[u];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  uint8_t* src; cudaMalloc(&src, kSrc); cudaMemset(src, 1, kSrc);
  unsigned long long* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* what, int grid) {
    unsigned long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-34s grid %3d: %.1f B/clk/SM  err=%s\n", what, grid, (double)kTotal / h, cudaGetErrorString(cudaGetLastError()));
  };
  cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 24576);
  cudaFuncSetAttribute(ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(ldgsts_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int grid : {1, sms}) {
    for (int chunk : {8192, 16384, 24576})
      for (int p : {1, 2, 4}) {
        bulk<<<grid, 256, 8 * chunk>>>(src, chunk, p, out);
        bulk<<<grid, 256, 8 * chunk>>>(src, chunk, p, out);
        char b[64]; snprintf(b, 64, "bulk chunk %d producers %d", chunk, p);
        report(b, grid);
      }
    ldgsts<<<grid, 256, 65536>>>(src, out); ldgsts<<<grid, 256, 65536>>>(src, out); report("LDGSTS 256 thr x 4 x 16 B", grid);
    ldgsts_plain<<<grid, 256, 65536>>>(src, out); ldgsts_plain<<<grid, 256, 65536>>>(src, out); report("LDG.128+STS.128 256 thr", grid);
  }
  return 0;
}

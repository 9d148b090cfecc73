// Microbenchmark (not product code): tcgen05.mma M=128 N=256 K=16 throughput with
// the B operand (a) resident in smem, (b) streamed from L2 through a bulk-copy
// ring, (c) streamed while 4 warps store 16 B/thread to another smem buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2112_05923_b200/csrc mb_mma.cu -o mb_mma
#include <cstdio>
#include <cstdint>
#include <vector>
#include "tc.cuh"
using namespace prb;

constexpr int kSlot = 8192;
constexpr int kIters = 2048;

template <int STAGES>
__global__ void __launch_bounds__(384, 1) mb(const uint8_t* gB, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;                        // [128][256] bf16 = 64 KB
  uint8_t* ring = sm + 65536;             // STAGES x 8 KB
  uint8_t* junk = ring + STAGES * kSlot;  // 32 KB store target
  __shared__ uint64_t full[STAGES], empty[STAGES], done, done2;
  __shared__ uint32_t tm;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], 1); }
    tc::mbar_init(&done, 1);
    tc::mbar_init(&done2, 1);
    tc::mbar_arrive(&done2);  // phase 0 complete
  }
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(A)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  for (int i = threadIdx.x; i < STAGES * kSlot / 16; i += blockDim.x) reinterpret_cast<uint4*>(ring)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (warp == 0) tc::tmem_alloc(&tm, 512);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t d = tm;
  constexpr uint32_t ID = tc::idesc_bf16(128, 256);
  if (warp == 0 && lane == 0) {
    const uint32_t a0 = tc::smem_u32(A), r0 = tc::smem_u32(ring);
    unsigned long long t0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int it = 0; it < kIters; ++it) {
      const int slot = it % STAGES;
      if (mode == 7 || mode == 8) {  // resident B; per-MMA wait on a completed barrier + commit
        tc::mbar_wait(&done2, 0);
      } else if (mode && mode != 6) tc::mbar_wait(&full[slot], (it / STAGES) & 1);
      tc::mma_bf16(d, tc::smem_desc(a0 + (it % 16) * 256, 128, 4096), tc::smem_desc(r0 + (mode >= 6 ? 0 : slot) * kSlot, 128, 256), ID, it % 16 != 0);
      if (mode == 7) tc::mma_commit(&empty[slot]);
      else if (mode == 8) { if (it % 2 == 1) tc::mma_commit(&empty[slot]); }
      else if (mode && mode != 6) tc::mma_commit(&empty[slot]);
    }
    tc::mma_commit(&done);
    tc::mbar_wait(&done, 0);
    unsigned long long t1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
  } else if (warp >= 1 && warp < 4 && lane == 0 && mode) {
    const int P = (mode >= 3 && mode != 6) ? 3 : (mode == 6 ? 3 : 1);
    if (warp - 1 >= P) return;
    for (int it = warp - 1; it < kIters; it += P) {
      const int slot = it % STAGES, use = it / STAGES;
      if (mode == 7 || mode == 8) break;
    if (mode == 6) {  // copies only: wait for the slot's previous copy, never consumed by the MMA
        if (slot == 0) continue;
        if (use) tc::mbar_wait(&full[slot], (use - 1) & 1);
      } else if (use) tc::mbar_wait(&empty[slot], (use - 1) & 1);
      tc::mbar_arrive_expect_tx(&full[slot], kSlot);
      tc::bulk_g2s(ring + slot * kSlot, gB + (size_t)(it % 34) * kSlot, kSlot, &full[slot]);
    }
  } else if (warp >= 4 && warp < 8 && (mode == 2 || mode == 4)) {
    uint4* j = reinterpret_cast<uint4*>(junk);
    for (int r = 0; r < 400; ++r)
      for (int i = threadIdx.x - 128; i < 2048; i += 128) { j[i] = make_uint4(r, r, r, r); __threadfence_block(); }
  } else if (warp >= 8 && mode == 4) {  // epilogue-like TMEM reads of the other 256 columns
    const uint32_t t = d + 256 + ((uint32_t)((warp - 8) * 32) << 16);
    float acc = 0.f;
    for (int r = 0; r < 100; ++r)
      for (int c = 0; c < 256; c += 32) {
        uint32_t v[32];
        tc::tmem_ld32(t + c, v);
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(v[i]);
      }
    if (acc == 1.2345f) out[1] = 1;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(d, 512);
}

int main() {
  uint8_t* gB; cudaMalloc(&gB, 34 * kSlot); cudaMemset(gB, 0, 34 * kSlot);
  unsigned long long* out; cudaMalloc(&out, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int stages, int mode, int grid) {
    const int smem = 65536 + stages * kSlot + 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long best[2] = {~0ull, ~0ull};
    for (int rep = 0; rep < 5; ++rep) {
      kern<<<grid, 384, smem>>>(gB, mode, out);
      unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      if (h[1] < best[1]) { best[0] = h[0]; best[1] = h[1]; }
    }
    printf("stages %2d mode %d grid %3d: %.1f clk/MMA %.1f ns/MMA (SM %.0f MHz) -> %.0f TFLOP/s/SM-equiv x148  err=%s\n",
           stages, mode, grid, (double)best[0] / kIters, (double)best[1] / kIters, 1e3 * best[0] / best[1],
           2.0 * 128 * 256 * 16 * kIters / best[1] * 148 / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int grid : {1, sms}) {
    run(mb<4>, 4, 0, grid);
    run(mb<4>, 4, 1, grid);
    run(mb<8>, 8, 1, grid);
    run(mb<12>, 12, 1, grid);
    run(mb<8>, 8, 2, grid);
    run(mb<5>, 5, 3, grid);
    run(mb<8>, 8, 3, grid);
    run(mb<8>, 8, 4, grid);
    run(mb<8>, 8, 6, grid);
    run(mb<8>, 8, 7, grid);
    run(mb<8>, 8, 8, grid);
  }
  return 0;
}

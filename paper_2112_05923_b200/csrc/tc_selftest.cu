// tc_selftest.cu -- validates the tcgen05 descriptor / TMEM conventions of tc.cuh
// with one M=128 x N x K bf16 GEMM (D = A . B^T, A [128][K], B [N][K]).
#include <vector>

#include "prb_internal.h"
#include <cuda_bf16.h>

#include "tc.cuh"

using namespace prb;

namespace {

__global__ void __launch_bounds__(128) tc_gemm_selftest_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                               float* __restrict__ D, int K, int N) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sA = smem;                 // 128*K*2 bytes
  unsigned char* sB = smem + 128 * K * 2;   // N*K*2 bytes
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + tc::kmajor_offset(r, k, K)) = __float2bfloat16_rn(A[i]);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sB + tc::kmajor_offset(r, k, K)) = __float2bfloat16_rn(B[i]);
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16(128, N);
    for (int j = 0; j < K / 16; ++j) {
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + j * 256, 128, K * 16);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + j * 256, 128, K * 16);
      tc::mma_bf16(tbase, ad, bd, idesc, j > 0);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[tid * N + c + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 256);
}

// The same GEMM with either operand stored TRANSPOSED (MN-major: the instruction descriptor's
// transpose bit, tc::idesc_bf16_t).  Every operand lives in one storage form, the "row-major
// core-matrix" form of some matrix Y[R][C] (tc::kmajor_offset(r, c, C)); an MN-major operand is
// Y = its transpose.  Descriptor strides per hypothesis `hyp` for MN-major operands:
//   hyp 0: LBO = the core-matrix stride along MN (128 B), SBO = along K (MN * 16 B)
//   hyp 1: the two swapped
// The K step of an MN-major operand advances 16 rows of Y: MN * 32 bytes.
__global__ void __launch_bounds__(128) tc_gemm_major_kernel(const float* __restrict__ A, const float* __restrict__ B,
                                                            float* __restrict__ D, int K, int N, int a_mn, int b_mn,
                                                            int hyp) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sA = smem;
  unsigned char* sB = smem + 128 * K * 2;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const uint32_t off = a_mn ? tc::kmajor_offset(k, r, 128) : tc::kmajor_offset(r, k, K);
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16_rn(A[i]);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const uint32_t off = b_mn ? tc::kmajor_offset(k, r, N) : tc::kmajor_offset(r, k, K);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16_rn(B[i]);
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 256);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16_t(128, N, a_mn, b_mn);
    auto params = [&](int mn_major, int MN, uint32_t& lbo, uint32_t& sbo, uint32_t& step) {
      if (!mn_major) {
        lbo = 128; sbo = (uint32_t)K * 16; step = 256;
      } else {
        const uint32_t s_mn = 128, s_k = (uint32_t)MN * 16;
        lbo = hyp ? s_k : s_mn;
        sbo = hyp ? s_mn : s_k;
        step = (uint32_t)MN * 32;
      }
    };
    uint32_t al, as, ast, bl, bs, bst;
    params(a_mn, 128, al, as, ast);
    params(b_mn, N, bl, bs, bst);
    for (int j = 0; j < K / 16; ++j) {
      const uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + j * ast, al, as);
      const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + j * bst, bl, bs);
      tc::mma_bf16(tbase, ad, bd, idesc, j > 0);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[tid * N + c + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 256);
}

}  // namespace

extern "C" int prb_debug_tc_gemm_major(prb_ctx ctx, int K, int N, int a_mn, int b_mn, int hyp, const float* hA,
                                       const float* hB, float* hD) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && hA && hB && hD, PRB_ERR_USAGE, "prb_debug_tc_gemm_major: NULL argument");
    PRB_REQUIRE(K % 16 == 0 && K <= 256 && N % 16 == 0 && N <= 256, PRB_ERR_CONFIG,
                "prb_debug_tc_gemm_major: bad shape");
    DevBuf<float> dA, dB, dD;
    dA.alloc(128 * K);
    dB.alloc((size_t)N * K);
    dD.alloc(128 * (size_t)N);
    cudaStream_t s = ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(dA.p, hA, dA.bytes(), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dB.p, hB, dB.bytes(), cudaMemcpyHostToDevice, s));
    const size_t smem = 200 * 1024;  // room for a wrong stride hypothesis to read garbage, not fault
    ensure_smem(tc_gemm_major_kernel, 200 * 1024);
    tc_gemm_major_kernel<<<1, 128, smem, s>>>(dA.p, dB.p, dD.p, K, N, a_mn, b_mn, hyp);
    PRB_CHECK_LAUNCH();
    PRB_CUDA(cudaMemcpyAsync(hD, dD.p, dD.bytes(), cudaMemcpyDeviceToHost, s));
    ctx->sync();
  });
}

extern "C" int prb_debug_tc_gemm(prb_ctx ctx, int K, int N, const float* hA, const float* hB, float* hD) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && hA && hB && hD, PRB_ERR_USAGE, "prb_debug_tc_gemm: NULL argument");
    PRB_REQUIRE(K % 16 == 0 && K <= 256 && N % 16 == 0 && N <= 256, PRB_ERR_CONFIG, "prb_debug_tc_gemm: bad shape");
    DevBuf<float> dA, dB, dD;
    dA.alloc(128 * K);
    dB.alloc((size_t)N * K);
    dD.alloc(128 * (size_t)N);
    cudaStream_t s = ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(dA.p, hA, dA.bytes(), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dB.p, hB, dB.bytes(), cudaMemcpyHostToDevice, s));
    const size_t smem = (size_t)(128 + N) * K * 2;
    ensure_smem(tc_gemm_selftest_kernel, 200 * 1024);
    tc_gemm_selftest_kernel<<<1, 128, smem, s>>>(dA.p, dB.p, dD.p, K, N);
    PRB_CHECK_LAUNCH();
    PRB_CUDA(cudaMemcpyAsync(hD, dD.p, dD.bytes(), cudaMemcpyDeviceToHost, s));
    ctx->sync();
  });
}

// ---- self-test of the fused rollout's conversion/division-free trade math (stock_env.cuh) ----
#include "stock_env.cuh"

namespace {

__global__ void trade_math_selftest_kernel(const float* __restrict__ act, float mt, const double* __restrict__ bal,
                                           const double* __restrict__ price, double cost, int n,
                                           int32_t* __restrict__ desired, double* __restrict__ buy,
                                           int32_t* __restrict__ buy_i) {
  // every lane runs the math (buy_qty_i32 votes across the warp); only in-range lanes store
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = i0 < n ? i0 : n - 1;
  const int32_t di = stock::desired_qty_f32(act[i], mt, (int32_t)mt);
  const stock::BuyPrice bp = stock::buy_price(price[i], cost);
  const int32_t qi = stock::buy_qty_i32(di, bal[i], bp);
  if (i0 < n) {
    desired[i] = di;
    buy[i] = (double)qi;
    buy_i[i] = qi;
  }
}

}  // namespace

extern "C" int prb_debug_trade_math(prb_ctx ctx, size_t n, const float* act, double max_trade, const double* balance,
                                    const double* price, double cost_rate, int32_t* desired, double* buy,
                                    int32_t* buy_i) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && act && balance && price && desired && buy && buy_i, PRB_ERR_USAGE,
                "prb_debug_trade_math: NULL argument");
    PRB_REQUIRE(max_trade == floor(max_trade) && max_trade >= 0.0 && max_trade < 4194304.0, PRB_ERR_CONFIG,
                "prb_debug_trade_math: max_trade must be an integer < 2^22");
    if (n == 0) return;
    DevBuf<float> dA;
    DevBuf<double> dB, dP, dBuy;
    DevBuf<int32_t> dD, dBi;
    dA.alloc(n); dB.alloc(n); dP.alloc(n); dBuy.alloc(n); dD.alloc(n); dBi.alloc(n);
    cudaStream_t s = ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(dA.p, act, dA.bytes(), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dB.p, balance, dB.bytes(), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(dP.p, price, dP.bytes(), cudaMemcpyHostToDevice, s));
    trade_math_selftest_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dA.p, (float)max_trade, dB.p, dP.p, cost_rate,
                                                                          (int)n, dD.p, dBuy.p, dBi.p);
    PRB_CHECK_LAUNCH();
    PRB_CUDA(cudaMemcpyAsync(desired, dD.p, dD.bytes(), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(buy, dBuy.p, dBuy.bytes(), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(buy_i, dBi.p, dBi.bytes(), cudaMemcpyDeviceToHost, s));
    ctx->sync();
  });
}

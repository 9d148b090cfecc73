// gae.cu -- generalized advantage estimation over the device rollout buffer
// (compute_gae ppo.hpp:50-71, buffer_advantages ppo.hpp:212-244).
//
// The buffer is time-major ([H][N]), so one thread per env walks its chunk
// backwards with every load coalesced across the warp (consecutive envs are
// consecutive addresses).  The recursion runs in fp64 with round-to-nearest
// intrinsics in the reference's operation order, so on identical fp32 inputs
// it reproduces the reference's fp64 result before the final fp32 store.
// The whole-buffer normalisation statistics (mean, population std floored at
// 1e-8) are reduced in the same pass: per-thread fp64 sums of x and x^2, then
// Chan merges of (n, mean, M2) across threads and blocks in fp64; the
// PPO gather applies (adv - mean) / denom on the fly, so the normalised
// advantages never make an extra HBM round trip.
#include <algorithm>
#include <cmath>

#include "prb_internal.h"

using namespace prb;

namespace {

constexpr int kGaeU = 16;  // recursion steps per pipelined load block

struct Welford {
  double n, mean, m2;
};

__device__ __forceinline__ Welford merge(Welford a, Welford b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n;
  const double d = b.mean - a.mean;
  Welford r;
  r.n = n;
  r.mean = a.mean + d * (b.n / n);
  r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / n);
  return r;
}

__global__ void __launch_bounds__(128) gae_kernel(const float* __restrict__ rew, const float* __restrict__ val,
                                                  const uint8_t* __restrict__ done, const float* __restrict__ boot,
                                                  int N, int H, double gamma, double lambda, float* __restrict__ adv,
                                                  float* __restrict__ ret, double* __restrict__ partials) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  Welford w{0.0, 0.0, 0.0};
  if (e < N) {
    const double gl = __dmul_rn(gamma, lambda);
    double gae = 0.0;
    double next_v = (double)boot[e];
    double s1 = 0.0, s2 = 0.0;  // sum and sum of squares of the stored advantages (fp64)
    // Software pipeline over blocks of kGaeU steps: the loads of the next block (they do not
    // depend on the recursion) are in flight while the current block's recursion runs.
    float rA[kGaeU], vA[kGaeU], rB[kGaeU], vB[kGaeU];
    uint8_t dA[kGaeU], dB[kGaeU];
    auto load = [&](int h0, float (&rr)[kGaeU], float (&vv)[kGaeU], uint8_t (&dd)[kGaeU]) {
#pragma unroll
      for (int u = 0; u < kGaeU; ++u) {
        const int h = h0 - u;
        if (h >= 0) {
          const size_t j = (size_t)h * N + e;
          rr[u] = rew[j];
          vv[u] = val[j];
          dd[u] = done[j];
        }
      }
    };
    auto run = [&](int h0, const float (&rr)[kGaeU], const float (&vv)[kGaeU], const uint8_t (&dd)[kGaeU]) {
#pragma unroll
      for (int u = 0; u < kGaeU; ++u) {
        const int h = h0 - u;
        if (h >= 0) {
          const size_t j = (size_t)h * N + e;
          const double r = (double)rr[u];
          const double v = (double)vv[u];
          const double nonterminal = dd[u] ? 0.0 : 1.0;
          // delta = r + gamma * next_value * nonterminal - v ; gae = delta + gamma*lambda*nonterminal*gae
          const double delta = __dsub_rn(__dadd_rn(r, __dmul_rn(__dmul_rn(gamma, next_v), nonterminal)), v);
          gae = __dadd_rn(delta, __dmul_rn(__dmul_rn(gl, nonterminal), gae));
          const float a32 = (float)gae;
          adv[j] = a32;
          ret[j] = (float)__dadd_rn(gae, v);
          next_v = v;
          const double x = (double)a32;
          s1 += x;
          s2 = fma(x, x, s2);
        }
      }
    };
    load(H - 1, rA, vA, dA);
    for (int h0 = H - 1; h0 >= 0; h0 -= 2 * kGaeU) {
      load(h0 - kGaeU, rB, vB, dB);
      run(h0, rA, vA, dA);
      load(h0 - 2 * kGaeU, rA, vA, dA);
      run(h0 - kGaeU, rB, vB, dB);
    }
    // this thread's (n, mean, M2) for the Chan merges below
    w.n = (double)H;
    w.mean = s1 / w.n;
    w.m2 = fmax(s2 - s1 * w.mean, 0.0);
  }
  if (!partials) return;
  // block merge: warp shuffles then smem
  for (int o = 16; o > 0; o >>= 1) {
    Welford b;
    b.n = __shfl_xor_sync(0xffffffffu, w.n, o);
    b.mean = __shfl_xor_sync(0xffffffffu, w.mean, o);
    b.m2 = __shfl_xor_sync(0xffffffffu, w.m2, o);
    w = merge(w, b);
  }
  __shared__ Welford sw[4];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    Welford acc = sw[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) acc = merge(acc, sw[i]);
    partials[3 * blockIdx.x + 0] = acc.n;
    partials[3 * blockIdx.x + 1] = acc.mean;
    partials[3 * blockIdx.x + 2] = acc.m2;
  }
}

__global__ void gae_stats_kernel(const double* __restrict__ partials, int nblocks, int normalize,
                                 double* __restrict__ stat) {
  __shared__ Welford sw[256];
  Welford w{0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    w = merge(w, Welford{partials[3 * b], partials[3 * b + 1], partials[3 * b + 2]});
  sw[threadIdx.x] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    Welford acc = sw[0];
    for (int i = 1; i < (int)blockDim.x; ++i) acc = merge(acc, sw[i]);
    if (normalize && acc.n > 0.0) {
      const double var = acc.m2 / acc.n;
      stat[0] = acc.mean;
      stat[1] = fmax(sqrt(var), 1e-8);  // ppo.hpp:240
    } else {
      stat[0] = 0.0;
      stat[1] = 1.0;
    }
  }
}

}  // namespace

void prb_gae_launch(prb_ctx ctx, const float* rew, const float* val, const uint8_t* done, const float* boot, size_t N,
                    size_t H, double gamma, double lambda, float* adv, float* ret, double* stat, int normalize) {
  const int grid = (int)((N + 127) / 128);  // 128-thread CTAs: more even spread over the SMs
  double* partials = stat ? static_cast<double*>(ctx->device_scratch((size_t)grid * 3 * sizeof(double))) : nullptr;
  {
    ProfScope prof(ctx, kProfGae);
    gae_kernel<<<grid, 128, 0, ctx->stream>>>(rew, val, done, boot, (int)N, (int)H, gamma, lambda, adv, ret, partials);
  }
  PRB_CHECK_LAUNCH();
  if (stat) {
    gae_stats_kernel<<<1, 256, 0, ctx->stream>>>(partials, grid, normalize, stat);
    PRB_CHECK_LAUNCH();
  }
}

extern "C" {

int prb_compute_gae(prb_ctx ctx, const float* d_rewards, const float* d_values, const uint8_t* d_dones,
                    const float* d_bootstrap, size_t N, size_t H, double gamma, double lambda, float* d_adv,
                    float* d_ret) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && d_rewards && d_values && d_dones && d_bootstrap && d_adv && d_ret, PRB_ERR_USAGE,
                "compute_gae: NULL argument");
    PRB_REQUIRE(N > 0 && H > 0, PRB_ERR_DIMENSION, "compute_gae: empty trajectory");  // ppo.hpp:54-57
    prb_gae_launch(ctx, d_rewards, d_values, d_dones, d_bootstrap, N, H, gamma, lambda, d_adv, d_ret, nullptr, 0);
  });
}

int prb_gae(prb_rollout r, double gamma, double lambda, int normalize) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r, PRB_ERR_USAGE, "buffer_advantages: NULL rollout");
    PRB_REQUIRE(r->full, PRB_ERR_USAGE,
                "buffer_advantages: chunks cover 0 of " + std::to_string(r->N * r->H) + " transitions");
    prb_gae_launch(r->ctx, r->d_rew.p, r->d_val.p, r->d_done.p, r->d_boot.p, r->N, r->H, gamma, lambda, r->d_adv.p,
                   r->d_ret.p, r->d_advstat.p, normalize);
    r->gae_valid = true;
    r->normalized = normalize != 0;
  });
}

int prb_gae_download(prb_rollout r, double* advantages, double* returns) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r && r->gae_valid, PRB_ERR_USAGE, "prb_gae_download: call prb_gae first");
    const size_t N = r->N, H = r->H, n = N * H;
    std::vector<float> a(n), t(n);
    double st[2];
    cudaStream_t s = r->ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(a.data(), r->d_adv.p, n * sizeof(float), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(t.data(), r->d_ret.p, n * sizeof(float), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(st, r->d_advstat.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    r->ctx->sync();
    for (size_t e = 0; e < N; ++e)
      for (size_t h = 0; h < H; ++h) {
        const size_t j = h * N + e, i = e * H + h;
        if (advantages) advantages[i] = ((double)a[j] - st[0]) / st[1];
        if (returns) returns[i] = t[j];
      }
  });
}

int prb_rollout_set_advantages(prb_rollout r, const double* advantages, const double* returns) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r && advantages && returns, PRB_ERR_USAGE, "prb_rollout_set_advantages: NULL argument");
    const size_t N = r->N, H = r->H, n = N * H;
    std::vector<float> a(n), t(n);
    for (size_t e = 0; e < N; ++e)
      for (size_t h = 0; h < H; ++h) {
        a[h * N + e] = (float)advantages[e * H + h];
        t[h * N + e] = (float)returns[e * H + h];
      }
    const double st[2] = {0.0, 1.0};
    cudaStream_t s = r->ctx->stream;
    PRB_CUDA(cudaMemcpyAsync(r->d_adv.p, a.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_ret.p, t.data(), n * sizeof(float), cudaMemcpyHostToDevice, s));
    PRB_CUDA(cudaMemcpyAsync(r->d_advstat.p, st, sizeof(st), cudaMemcpyHostToDevice, s));
    r->ctx->sync();
    r->gae_valid = true;
  });
}

}  // extern "C"

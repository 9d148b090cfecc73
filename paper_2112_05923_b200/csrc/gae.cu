// gae.cu -- generalized advantage estimation over the device rollout buffer
// (compute_gae ppo.hpp:50-71, buffer_advantages ppo.hpp:212-244).
//
// The per-env recursion  gae_t = delta_t + c_t * gae_{t+1},  c_t = gamma*lambda*(1 - d_t),
// delta_t = r_t + gamma*V_{t+1}*(1 - d_t) - V_t  is an affine map of gae_{t+1}, so it runs as a
// segmented affine scan over the horizon instead of one serial walk per env:
//   * Work unit (tile): 32 consecutive envs x a window of WIN steps of the time-major [H][N]
//     buffer.  Persistent CTAs walk their env groups' windows from the last to the first, the
//     next tile's r / V / done boxes streaming into a second shared-memory buffer (three 2-D
//     TMA loads on an mbarrier) while the current one is scanned, so HBM always has a tile in
//     flight per CTA.
//   * Phase 1: warp w owns steps [w*SEG, (w+1)*SEG) of the window, lane = env (every shared
//     row read is conflict-free); each thread forms delta_t and composes its segment backwards
//     into (A, B) with gae_{seg start} = B + A * gae_{seg end} (delta, V, dones kept in registers).
//   * Phase 2: each thread folds the (A, B) of the later segments of its env, starting from the
//     carry of the later window (0 past the last step, ppo.hpp:63), into its incoming gae.
//   * Phase 3: each thread re-runs its segment from that gae in the reference's operation order
//     and stores advantage / return (one coalesced 128-byte row segment per warp and step).
// Precision: fp64 throughout; a segment's incoming gae comes from the composed maps instead of
// the serial chain, so gae agrees with the reference's fp64 recursion to ~1e-15 relative (tested
// at 1e-12) and the fp32 stores are the reference's fp32 rounding or one ulp beside it.  The
// last segment of every env (carry 0) and every step after a done (c_t = 0 cuts the chain) are
// exactly the reference's values.
// The whole-buffer normalisation statistics (mean, population std floored at 1e-8) are reduced
// in the same pass: per-thread (n, mean, M2) of its stored advantages, Chan merges across threads
// and blocks in fp64; the PPO gather applies (adv - mean) / denom on the fly, so the normalised
// advantages never make an extra HBM round trip.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "prb_internal.h"
#include "tc.cuh"
#include "tmap.h"

using namespace prb;

namespace {

#ifndef PRB_GAE_WIN
#define PRB_GAE_WIN 64
#endif
#ifndef PRB_GAE_SW
#define PRB_GAE_SW 4
#endif
#ifndef PRB_GAE_ENVS
#define PRB_GAE_ENVS 32
#endif
#ifndef PRB_GAE_STAGES
#define PRB_GAE_STAGES 2
#endif
constexpr int kGaeWin = PRB_GAE_WIN;      // steps per tile window
constexpr int kGaeSegWarps = PRB_GAE_SW;  // segments per window
constexpr int kGaeEnvs = PRB_GAE_ENVS;    // envs per tile (one per lane of an env-warp)
constexpr int kGaeStages = PRB_GAE_STAGES;  // tile buffers (tiles in flight + the one scanned)

struct Welford {
  double n, mean, m2;
};

// 1 / x for the merge weights: the approximate reciprocal refined by two Newton steps (~1 ulp;
// the merges' weights need ~1e-15, not a correctly rounded division on the reduction's tail)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}

// Chan et al.'s pairwise merge of (n, mean, M2) records
__device__ __forceinline__ Welford merge(Welford a, Welford b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n;
  const double fb = b.n * rcp_nr(n);  // b's weight
  const double d = b.mean - a.mean;
  Welford r;
  r.n = n;
  r.mean = fma(d, fb, a.mean);
  r.m2 = a.m2 + b.m2 + d * d * (a.n * fb);
  return r;
}

// Shared-memory image of one tile: r, V [WIN][E] fp32 and done [WIN][E] u8 (the TMA boxes).
// After phase 1 the r / V rows are overwritten with the tile's advantages / returns, which
// leave by TMA stores of the same boxes.
template <int WIN, int E>
struct __align__(128) GaeTile {
  float r[WIN][E];
  float v[WIN][E];
  uint8_t d[WIN][E];
};

struct GaeMaps {  // time-major [H][N] r / V / adv / ret (fp32) and done (u8), boxes [WIN][E]
  CUtensorMap r, v, d, adv, ret;
};

// E envs per tile (E/32 env-warps x SW segment-warps; SEG = WIN / SW steps per thread).
template <int WIN, int SW, int E, bool TMA, int ST = kGaeStages>
__global__ void __launch_bounds__(E * SW)
    gae_scan_kernel(const __grid_constant__ GaeMaps maps, const float* __restrict__ rew,
                    const float* __restrict__ val, const uint8_t* __restrict__ done, const float* __restrict__ boot,
                    int N, int H, double gamma, double lambda, float* __restrict__ adv, float* __restrict__ ret,
                    double* __restrict__ partials, unsigned int* __restrict__ counter, int normalize,
                    double* __restrict__ stat) {
  constexpr int SEG = WIN / SW;
  constexpr int EW = E / 32;
  constexpr int T = E * SW;
  static_assert(SEG <= 32, "segment mask is 32 bits");
  using Tile = GaeTile<WIN, E>;
  extern __shared__ __align__(128) unsigned char gae_smem[];
  Tile* tiles = reinterpret_cast<Tile*>(gae_smem);  // [ST] ring of tile buffers
  __shared__ __align__(8) uint64_t s_full[ST];  // TMA transaction barriers of the buffers
  __shared__ double2 s_ab[SW][E];             // (A, B) of each segment of each env
  __shared__ double s_carry[E];               // gae at the first step of the later window
  __shared__ float s_vlater[E];               // V at the first step of the later window
  __shared__ Welford s_w[T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = (warp % EW) * 32 + lane, sw = warp / EW;
  const double gl = __dmul_rn(gamma, lambda);
  const int ngroups = (N + E - 1) / E, nwin = (H + WIN - 1) / WIN;
  const int my_groups = (int)blockIdx.x < ngroups ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int ntiles = my_groups * nwin;
  if (TMA && threadIdx.x == 0)
    for (int b = 0; b < ST; ++b) tc::mbar_init(&s_full[b], 1);
  __syncthreads();
  // tile k -> env group g, window wi (windows of a group from the last to the first)
  auto tile_of = [&](int k, int& g, int& wi) {
    g = (int)blockIdx.x + (k / nwin) * (int)gridDim.x;
    wi = nwin - 1 - k % nwin;
  };
  auto issue = [&](int k) {
    int g, wi;
    tile_of(k, g, wi);
    Tile& tb = tiles[k % ST];
    if (TMA) {
      if (threadIdx.x == 0) {
        tc::bulk_wait_read0();  // the stores of tile k - ST have read this buffer
        // three boxes; rows past H and columns past N arrive zero-filled (never stored)
        uint64_t* bar = &s_full[k % ST];
        tc::mbar_arrive_expect_tx(bar, (uint32_t)sizeof(Tile));
        tc::tma_load_2d(&tb.r[0][0], &maps.r, g * E, wi * WIN, bar);
        tc::tma_load_2d(&tb.v[0][0], &maps.v, g * E, wi * WIN, bar);
        tc::tma_load_2d(&tb.d[0][0], &maps.d, g * E, wi * WIN, bar);
      }
    } else {  // any N: element loads (synchronous)
      const int e0 = g * E, t0 = wi * WIN, len = min(WIN, H - t0);
      for (int c = threadIdx.x; c < len * E; c += T) {
        const int row = c / E, l = c % E;
        if (e0 + l < N) {
          const size_t j = (size_t)(t0 + row) * N + e0 + l;
          tb.r[row][l] = __ldcs(rew + j);
          tb.v[row][l] = __ldcs(val + j);
          tb.d[row][l] = __ldcs(done + j);
        }
      }
    }
  };
  // this thread's stored advantages as sums shifted by the first one it stored (no division
  // per tile; one Welford record at the end)
  double sn = 0.0, sx0 = 0.0, ss1 = 0.0, ssq = 0.0;
  constexpr int kAhead = TMA ? ST - 1 : 1;  // tiles in flight while one is scanned
  for (int k = 0; k < kAhead && k < ntiles; ++k) issue(k);
  for (int k = 0; k < ntiles; ++k) {
    if (k + kAhead < ntiles) issue(k + kAhead);  // later tiles stream in while this one is scanned
    if (TMA) tc::mbar_wait(&s_full[k % ST], (uint32_t)((k / ST) & 1));
    __syncthreads();  // (TMA: every thread past the wait; else: the element loads are visible)
    int g, wi;
    tile_of(k, g, wi);
    Tile& tb = tiles[k % ST];
    const int e = g * E + col;
    const bool live = e < N;
    const int t0 = wi * WIN, len = min(WIN, H - t0);
    const bool last_window = (wi == nwin - 1);
    const int s0 = sw * SEG, slen = max(0, min(SEG, len - s0));
    // V after this segment: the next segment's first value, the later window's first value, or
    // the bootstrap V(s_H) (ppo.hpp:62)
    float vn = 0.f;
    if (live && slen > 0)
      vn = (s0 + slen < len) ? tb.v[s0 + slen][col] : (last_window ? __ldg(boot + e) : s_vlater[col]);
    // phase 1: delta_t (the reference's expression) and the composed map of the segment;
    // delta, V and the done bits stay in registers for phase 3
    double delta[SEG];
    float vr[SEG];
    uint32_t dmask = 0;
    double A = 1.0, B = 0.0;
    {
      double nv = (double)vn;
#pragma unroll
      for (int u = SEG - 1; u >= 0; --u)
        if (u < slen) {
          const int i = s0 + u;
          const bool dn = tb.d[i][col] != 0;
          vr[u] = tb.v[i][col];
          const double vv = (double)vr[u];
          delta[u] = __dsub_rn(__dadd_rn((double)tb.r[i][col], __dmul_rn(__dmul_rn(gamma, nv), dn ? 0.0 : 1.0)), vv);
          const double c = dn ? 0.0 : gl;  // gamma*lambda*nonterminal
          dmask |= (uint32_t)dn << u;
          B = fma(c, B, delta[u]);
          A = c * A;
          nv = vv;
        }
    }
    s_ab[sw][col] = make_double2(A, B);
    __syncthreads();
    // phase 2: incoming gae of this segment
    double gin = last_window ? 0.0 : s_carry[col];
    for (int s2 = SW - 1; s2 > sw; --s2) {
      const double2 ab = s_ab[s2][col];
      gin = fma(ab.x, gin, ab.y);
    }
    float vfirst = 0.f;
    if (sw == 0) vfirst = tb.v[0][col];
    __syncthreads();  // s_carry / s_vlater / s_ab and the tile's r / V rows consumed
    // phase 3: the reference's recursion (ppo.hpp:61-68) from the incoming gae; advantages and
    // returns go to the tile's r / V rows (TMA) or straight to HBM (element path)
    if (live && slen > 0) {
      double gae = gin;
#pragma unroll
      for (int u = SEG - 1; u >= 0; --u)
        if (u < slen) {
          // gae = delta + gamma*lambda*nonterminal*gae; gamma*lambda*nonterminal is gl or 0 exactly
          gae = __dadd_rn(delta[u], ((dmask >> u) & 1u) ? 0.0 : __dmul_rn(gl, gae));
          const float a32 = (float)gae, r32 = (float)__dadd_rn(gae, (double)vr[u]);
          if (TMA) {
            tb.r[s0 + u][col] = a32;
            tb.v[s0 + u][col] = r32;
          } else {
            const size_t j = (size_t)(t0 + s0 + u) * N + e;
            __stcs(adv + j, a32);
            __stcs(ret + j, r32);
          }
          // the statistics cover the stored fp32 values: the gather normalises exactly those
          const double a = (double)a32;
          if (sn == 0.0 && u == slen - 1) sx0 = a;
          const double dx = a - sx0;
          ss1 += dx;
          ssq = fma(dx, dx, ssq);
        }
      sn += (double)slen;
      if (sw == 0) {  // this window's first step feeds the earlier window
        s_carry[col] = gae;
        s_vlater[col] = vfirst;
      }
    }
    if (TMA) tc::fence_proxy_async();  // the staged rows, to the async proxy
    __syncthreads();                    // s_carry visible to the next tile; staged rows complete
    if (TMA && threadIdx.x == 0) {
      tc::tma_store_2d(&maps.adv, g * E, t0, &tb.r[0][0]);
      tc::tma_store_2d(&maps.ret, g * E, t0, &tb.v[0][0]);
      tc::bulk_commit();
    }
  }
  if (TMA && threadIdx.x == 0) tc::bulk_wait0();
  if (!partials) return;
  Welford w{0.0, 0.0, 0.0};
  if (sn > 0.0) w = Welford{sn, sx0 + ss1 / sn, fmax(ssq - ss1 * (ss1 / sn), 0.0)};
  for (int o = 16; o > 0; o >>= 1) {
    Welford b;
    b.n = __shfl_xor_sync(0xffffffffu, w.n, o);
    b.mean = __shfl_xor_sync(0xffffffffu, w.mean, o);
    b.m2 = __shfl_xor_sync(0xffffffffu, w.m2, o);
    w = merge(w, b);
  }
  if (lane == 0) s_w[warp] = w;
  __syncthreads();
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    Welford acc = s_w[0];
    for (int i = 1; i < T / 32; ++i) acc = merge(acc, s_w[i]);
    partials[3 * blockIdx.x + 0] = acc.n;
    partials[3 * blockIdx.x + 1] = acc.mean;
    partials[3 * blockIdx.x + 2] = acc.m2;
    __threadfence();  // this CTA's record before its arrival
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // the last CTA to finish merges every CTA's record (no second launch): per-thread strided
  // merges, then a tree over the warps
  __threadfence();
  Welford acc{0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += T)
    acc = merge(acc, Welford{__ldcg(partials + 3 * b), __ldcg(partials + 3 * b + 1), __ldcg(partials + 3 * b + 2)});
  for (int o = 16; o > 0; o >>= 1) {
    Welford b;
    b.n = __shfl_xor_sync(0xffffffffu, acc.n, o);
    b.mean = __shfl_xor_sync(0xffffffffu, acc.mean, o);
    b.m2 = __shfl_xor_sync(0xffffffffu, acc.m2, o);
    acc = merge(acc, b);
  }
  __syncthreads();
  if (lane == 0) s_w[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    Welford all = s_w[0];
    for (int i = 1; i < T / 32; ++i) all = merge(all, s_w[i]);
    if (normalize && all.n > 0.0) {
      stat[0] = all.mean;
      stat[1] = fmax(sqrt(all.m2 / all.n), 1e-8);  // ppo.hpp:240
    } else {
      stat[0] = 0.0;
      stat[1] = 1.0;
    }
    *counter = 0u;  // ready for the next launch (stream-ordered)
  }
}

}  // namespace

void prb_gae_launch(prb_ctx ctx, const float* rew, const float* val, const uint8_t* done, const float* boot, size_t N,
                    size_t H, double gamma, double lambda, float* adv, float* ret, double* stat, int normalize) {
  PRB_REQUIRE(N < (1u << 31) && H < (1u << 31), PRB_ERR_CONFIG, "buffer_advantages: buffer too large");
  constexpr int E = kGaeEnvs, W = kGaeWin, SW = kGaeSegWarps;
  const bool tma0 = (N % 16) == 0;
  const size_t smem = (tma0 ? kGaeStages : 2) * sizeof(GaeTile<W, E>);
  // TMA boxes need 16-byte row pitches (the u8 dones: N % 16 == 0)
  const bool tma = (N % 16) == 0;
  GaeMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  if (tma) {
    encode_tmap_2d(&maps.r, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rew, N, H, N * 4, E, W);
    encode_tmap_2d(&maps.v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, val, N, H, N * 4, E, W);
    encode_tmap_2d(&maps.d, CU_TENSOR_MAP_DATA_TYPE_UINT8, done, N, H, N, E, W);
    encode_tmap_2d(&maps.adv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, adv, N, H, N * 4, E, W);
    encode_tmap_2d(&maps.ret, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, ret, N, H, N * 4, E, W);
  }
  const void* fn =
      tma ? (const void*)gae_scan_kernel<W, SW, E, true> : (const void*)gae_scan_kernel<W, SW, E, false, 2>;
  ensure_smem_attr(fn, smem);
  int occ = 0;
  PRB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, E * SW, smem));
  const int groups = (int)((N + E - 1) / E);
  const int resident = ctx->num_sms * std::max(occ, 1);
  // every resident slot gets a CTA; group counts per CTA differ by at most one, and the strided
  // assignment spreads the heavier CTAs over the SMs (per-SM load within one group of the mean).
  // Equal counts per CTA (fewer CTAs) measured 1.5% slower at 65,536 envs, 12.6% at 1M.
  const int grid = std::max(1, std::min(groups, resident));
  double* partials = stat ? static_cast<double*>(ctx->device_scratch((size_t)grid * 3 * sizeof(double))) : nullptr;
  unsigned int* counter = stat ? ctx->last_cta_counter() : nullptr;
  {
    ProfScope prof(ctx, kProfGae);
    if (tma)
      gae_scan_kernel<W, SW, E, true><<<grid, E * SW, smem, ctx->stream>>>(
          maps, rew, val, done, boot, (int)N, (int)H, gamma, lambda, adv, ret, partials, counter, normalize, stat);
    else
      gae_scan_kernel<W, SW, E, false, 2><<<grid, E * SW, smem, ctx->stream>>>(
          maps, rew, val, done, boot, (int)N, (int)H, gamma, lambda, adv, ret, partials, counter, normalize, stat);
  }
  PRB_CHECK_LAUNCH();
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

int prb_gae_stats(prb_rollout r, double* mean, double* denom) {
  return guard([&] {
    DeviceScope dev_(r ? r->ctx : nullptr);
    PRB_REQUIRE(r && r->gae_valid && mean && denom, PRB_ERR_USAGE, "prb_gae_stats: call prb_gae first");
    double st[2];
    PRB_CUDA(cudaMemcpyAsync(st, r->d_advstat.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, r->ctx->stream));
    r->ctx->sync();
    *mean = st[0];
    *denom = st[1];
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

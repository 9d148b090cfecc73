// env.cu -- vectorised environments on device (VectorizedEnvironment,
// env.hpp:167-249) with the stock-trading env (stock_env.hpp:55-184) and the
// PointMass2D analytic control env (env.hpp:84-146).
//
// Layout (HBM, SoA so every per-env field is read/written coalesced):
//   stock:  balance f64 [N], shares i32 [K][N], episode_return f64 [N];
//           price table f64 [T][K] and the window's shared obs features
//           f32 [T][5K] are read-only and L2-resident.  All envs of one
//           VecEnv run in lock-step (same t, same done; stock_env.hpp:161,
//           env.hpp:221), so t / step_count are scalars owned by the host.
//   pointmass: state f64 [6][N], steps i32 [N], episode_return f64 [N],
//           per-env mt19937_64 reset stream u64 [312][N] + idx i32 [N].
//   obs (VectorizedEnvironment::states_): f32 [N][S] row-major.
//
// Arithmetic: the portfolio accounting is fp64 with explicit round-to-nearest
// intrinsics (no FMA contraction), in the reference's operation order, so
// balances, share counts, rewards and dones are bit-identical with the
// -ffp-contract=off reference build.  Obs and rewards are stored as fp32.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "prb_internal.h"
#include "pm_env.cuh"
#include "rng.cuh"
#include "stock_env.cuh"

using namespace prb;

namespace {

constexpr int kEnvBlock = 64;

// std::clamp / std::min / std::max semantics (NaN-propagating exactly as libstdc++).
__device__ __forceinline__ double clamp_ref(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
__device__ __forceinline__ double min_ref(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double max_ref(double a, double b) { return (a < b) ? b : a; }

struct StockStepArgs {
  int N, K, S;
  int t;       // portfolio time before the step
  int t_obs;   // time index of the returned (post-reset) observation
  int done;    // uniform episode end
  int ep_len;  // episode length reported on done
  const double* __restrict__ close_tk;  // [T][K]
  const float* __restrict__ feat;       // [T][5K]
  double cap, max_trade, cost;
  const float* __restrict__ actions;  // [N][K]
  double* __restrict__ balance;
  int32_t* __restrict__ shares;  // [K][N]
  double* __restrict__ ep_return;
  float* __restrict__ obs;  // [N][S]
  float* __restrict__ reward;
  uint8_t* __restrict__ done_out;
  float* __restrict__ term_obs;
  double* __restrict__ term_ret;
  int32_t* __restrict__ term_len;
};

// ---- v2: asynchronous staging (cp.async) and no private-obs copy -----------
// Every load of the CTA is an LDGSTS issued up front (no registers held, all
// bytes in flight at once); the obs writer reads the portfolio straight from
// the share table, so shared memory is ~280 B/env and 10+ CTAs fit per SM.
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

struct ObsSrc {  // obs row r = [x0[r], shares[0..K)[r], shared[0..5K)]
  const float* x0;
  const int32_t* sh;  // [kEnvBlock][Kp] env-major, odd stride: conflict-free both ways
  const float* shared;
  int K, Kp;
  __device__ __forceinline__ float at(int r, int c) const {
    return c == 0 ? x0[r] : (c <= K ? (float)sh[r * Kp + c - 1] : shared[c - 1 - K]);
  }
};

__device__ __forceinline__ void write_obs_v2(float* __restrict__ dst, int nrows, int S, const ObsSrc& src) {
  const int total = nrows * S;
  if (src.K <= 31) {
    // Warp per row: lanes 0..K write the private part (one coalesced store),
    // then the 5K shared features -- identical for every row, so each lane
    // keeps its <= 5 feature values in registers for the whole block.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int P = src.K + 1, F = 5 * src.K;
    float fv[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) fv[j] = (lane + 32 * j < F) ? src.shared[lane + 32 * j] : 0.f;
    for (int r = warp; r < nrows; r += nw) {
      float* row = dst + (size_t)r * S;
      if (lane < P) row[lane] = (lane == 0) ? src.x0[r] : (float)src.sh[r * src.Kp + lane - 1];
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (lane + 32 * j < F) row[P + lane + 32 * j] = fv[j];
    }
    return;
  }
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const int total4 = total >> 2;
    const int step = 4 * (int)blockDim.x;
    int f = 4 * threadIdx.x;
    int r = f / S, c = f - r * S;
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int q = threadIdx.x; q < total4; q += blockDim.x) {
      float v[4];
      int rr = r, cc = c;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = src.at(rr, cc);
        if (++cc == S) {
          cc = 0;
          ++rr;
        }
      }
      d4[q] = make_float4(v[0], v[1], v[2], v[3]);
      c += step;
      while (c >= S) {
        c -= S;
        ++r;
      }
    }
    for (int i = total4 * 4 + threadIdx.x; i < total; i += blockDim.x) {
      const int rr = i / S;
      dst[i] = src.at(rr, i - rr * S);
    }
  } else {
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int rr = i / S;
      dst[i] = src.at(rr, i - rr * S);
    }
  }
}

// Warp-per-row obs writer from a float table whose row r holds the shares in
// columns 0..K-1 and balance/cap in column K (odd stride Kp = K+1); lanes 0..K
// write the private part with one shared-memory load each (no conversion or
// select on the value), then the 5K shared features -- identical for every row,
// so each lane keeps its <= 5 feature values in registers for the whole block.
__device__ __forceinline__ void write_obs_tab(float* __restrict__ dst, int nrows, int S, const float* table, int K,
                                              int Kp, const float* shared) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int P = K + 1, F = 5 * K;
  const int col = (lane == 0) ? K : lane - 1;
  float fv[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) fv[j] = (lane + 32 * j < F) ? shared[lane + 32 * j] : 0.f;
  for (int r = warp; r < nrows; r += nw) {
    float* row = dst + (size_t)r * S;
    if (lane < P) row[lane] = table[r * Kp + col];
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if (lane + 32 * j < F) row[P + lane + 32 * j] = fv[j];
  }
}

__global__ void __launch_bounds__(kEnvBlock) stock_step_v2_kernel(StockStepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, F = 5 * K, Kp = (K & 1) ? K + 2 : K + 1;
  double* s_p0 = reinterpret_cast<double*>(smem_raw);          // [K]
  double* s_p1 = s_p0 + K;                                      // [K]
  double* s_bal = s_p1 + K;                                     // [kEnvBlock]
  double* s_ret = s_bal + kEnvBlock;                            // [kEnvBlock]
  float* s_act = reinterpret_cast<float*>(s_ret + kEnvBlock);   // [kEnvBlock*K] (+ 4 pad)
  int32_t* s_sh = reinterpret_cast<int32_t*>(s_act + ((kEnvBlock * K + 7) & ~3));  // [kEnvBlock][Kp]
  float* s_x0 = reinterpret_cast<float*>(s_sh + Kp * kEnvBlock);                  // [kEnvBlock]
  float* s_feat_obs = s_x0 + kEnvBlock;                                          // [5K]
  float* s_feat_term = s_feat_obs + F;                                           // [5K]
  const int tid = threadIdx.x;
  const size_t e0 = (size_t)blockIdx.x * kEnvBlock;
  const int nloc = min(kEnvBlock, a.N - (int)e0);
  const bool live = tid < nloc;
  // ---- every load in flight at once ----
  const float* src = a.actions + e0 * K;
  const int total = nloc * K;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  const int total4 = vec_ok ? total / 4 : 0;
  for (int q = tid; q < total4; q += kEnvBlock) cp_async16(s_act + 4 * q, src + 4 * q);
  for (int f = total4 * 4 + tid; f < total; f += kEnvBlock) cp_async4(s_act + f, src + f);
  if (live) {
    for (int k = 0; k < K; ++k) cp_async4(s_sh + tid * Kp + k, a.shares + (size_t)k * a.N + e0 + tid);
    cp_async8(s_bal + tid, a.balance + e0 + tid);
    cp_async8(s_ret + tid, a.ep_return + e0 + tid);
  }
  for (int k = tid; k < K; k += kEnvBlock) {
    cp_async8(s_p0 + k, a.close_tk + (size_t)a.t * K + k);
    cp_async8(s_p1 + k, a.close_tk + (size_t)(a.t + 1) * K + k);
  }
  for (int j = tid; j < F; j += kEnvBlock) {
    cp_async4(s_feat_obs + j, a.feat + (size_t)a.t_obs * F + j);
    if (a.done) cp_async4(s_feat_term + j, a.feat + (size_t)(a.t + 1) * F + j);
  }
  cp_async_wait_all();
  __syncthreads();
  // ---- accounting (stock_env_step stock_env.hpp:55-103), fp64, reference order ----
  if (live) {
    const size_t e = e0 + tid;
    double bal = s_bal[tid];
    int32_t* sh = s_sh + tid * Kp;
    const float* act = s_act + tid * K;
    double vb = bal;
    for (int k = 0; k < K; ++k) vb = __dadd_rn(vb, __dmul_rn((double)sh[k], s_p0[k]));
    for (int k = 0; k < K; ++k) {
      const double d = trunc(__dmul_rn(clamp_ref((double)act[k], -1.0, 1.0), a.max_trade));
      if (d < 0.0) {
        const int32_t held = sh[k];
        const double q = -min_ref(-d, (double)held);
        const double price = s_p0[k];
        const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(q)), price);
        bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(q, price), cost));
        sh[k] = held + (int32_t)q;
      }
    }
    const double cost_factor = __dadd_rn(1.0, a.cost);
    for (int k = 0; k < K; ++k) {
      const double d = trunc(__dmul_rn(clamp_ref((double)act[k], -1.0, 1.0), a.max_trade));
      if (d > 0.0) {
        const double price = s_p0[k];
        const double q = stock::buy_qty(d, bal, __dmul_rn(price, cost_factor));
        const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(q)), price);
        bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(q, price), cost));
        sh[k] += (int32_t)q;
      }
    }
    double va = bal;
    for (int k = 0; k < K; ++k) va = __dadd_rn(va, __dmul_rn((double)sh[k], s_p1[k]));
    const double r = __dsub_rn(va, vb);
    const double ret = __dadd_rn(s_ret[tid], r);
    if (a.reward) a.reward[e] = (float)r;
    if (a.done_out) a.done_out[e] = (uint8_t)a.done;
    s_x0[tid] = (float)__ddiv_rn(bal, a.cap);
    if (a.done) {
      if (a.term_ret) a.term_ret[e] = ret;
      if (a.term_len) a.term_len[e] = a.ep_len;
      a.balance[e] = a.cap;
      a.ep_return[e] = 0.0;
    } else {
      a.balance[e] = bal;
      a.ep_return[e] = ret;
    }
  }
  __syncthreads();
  const int S = a.S;
  if (a.done) {  // terminal obs, then auto-reset the portfolios (env.hpp:221-229)
    if (a.term_obs) write_obs_v2(a.term_obs + e0 * S, nloc, S, ObsSrc{s_x0, s_sh, s_feat_term, K, Kp});
    __syncthreads();
    s_x0[tid] = (float)(a.cap / a.cap);
    for (int k = 0; k < K; ++k) s_sh[tid * Kp + k] = 0;
    __syncthreads();
  }
  if (live)
    for (int k = 0; k < K; ++k) a.shares[(size_t)k * a.N + e0 + tid] = s_sh[tid * Kp + k];
  write_obs_v2(a.obs + e0 * S, nloc, S, ObsSrc{s_x0, s_sh, s_feat_obs, K, Kp});
}

// ---- v3 (K <= 32, K even): actions straight into registers -----------------
// Each thread's 4K action bytes are issued as float2 loads before anything
// else and consumed from registers; the share table stays in shared memory for
// the obs writer.  ~170 B of shared memory per env -> ~2x the resident warps
// of v2, which is what keeps HBM busy while other CTAs run the fp64 chain.
#ifndef PRB_ENV_TPS
#define PRB_ENV_TPS 1024  // resident threads per SM the register budget is sized for
#endif
template <int KMAX, int EB>
__device__ __forceinline__ void stock_step_v3_body(const StockStepArgs& a, size_t tile) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, F = 5 * K, Kp = K + 1;  // K even -> odd stride
  double* s_p0 = reinterpret_cast<double*>(smem_raw);          // [K]
  double* s_p1 = s_p0 + K;                                      // [K]
  int32_t* s_sh = reinterpret_cast<int32_t*>(s_p1 + K);         // [EB][Kp]
  float* s_x0 = reinterpret_cast<float*>(s_sh + Kp * EB);  // [EB]
  float* s_feat_obs = s_x0 + EB;                            // [5K]
  float* s_feat_term = s_feat_obs + F;                             // [5K]
  const int tid = threadIdx.x;
  const size_t e0 = tile * EB;
  const int nloc = min(EB, a.N - (int)e0);
  const bool live = tid < nloc;
  const size_t e = e0 + tid;
  float2 act2[KMAX / 2];
  const float2* arow = reinterpret_cast<const float2*>(a.actions + (live ? e : e0) * K);
#pragma unroll
  for (int j = 0; j < KMAX / 2; ++j)
    if (2 * j < K) act2[j] = __ldg(arow + j);
  const double bal_in = live ? a.balance[e] : 0.0;
  const double ret_in = live ? a.ep_return[e] : 0.0;
  if (live)
    for (int k = 0; k < K; ++k) cp_async4(s_sh + tid * Kp + k, a.shares + (size_t)k * a.N + e);
  for (int k = tid; k < K; k += EB) {
    cp_async8(s_p0 + k, a.close_tk + (size_t)a.t * K + k);
    cp_async8(s_p1 + k, a.close_tk + (size_t)(a.t + 1) * K + k);
  }
  for (int j = tid; j < F; j += EB) {
    cp_async4(s_feat_obs + j, a.feat + (size_t)a.t_obs * F + j);
    if (a.done) cp_async4(s_feat_term + j, a.feat + (size_t)(a.t + 1) * F + j);
  }
  cp_async_wait_all();
  __syncthreads();
  // desired_k = trunc(clamp(a_k, -1, 1) * max_trade) (stock_env.hpp:83-87), once per asset, kept
  // in the action registers as floats (integer-valued, exact below 2^24: the launcher checks
  // max_trade_shares) for both the sell and the buy pass
#pragma unroll
  for (int j = 0; j < KMAX / 2; ++j)
    if (2 * j < K) {
      act2[j].x = (float)trunc(__dmul_rn(clamp_ref((double)act2[j].x, -1.0, 1.0), a.max_trade));
      act2[j].y = (float)trunc(__dmul_rn(clamp_ref((double)act2[j].y, -1.0, 1.0), a.max_trade));
    }
  if (live) {
    double bal = bal_in;
    int32_t* sh = s_sh + tid * Kp;
    double vb = bal;
    for (int k = 0; k < K; ++k) vb = __dadd_rn(vb, __dmul_rn((double)sh[k], s_p0[k]));
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {  // sells first (stock_env.hpp:88-90)
      if (k < K) {
        const double d = (double)((k & 1) ? act2[k >> 1].y : act2[k >> 1].x);
        if (d < 0.0) {
          const int32_t held = sh[k];
          const double q = -min_ref(-d, (double)held);
          const double price = s_p0[k];
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(q)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(q, price), cost));
          sh[k] = held + (int32_t)q;
        }
      }
    }
    const double cost_factor = __dadd_rn(1.0, a.cost);
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {  // then buys (:91-97)
      if (k < K) {
        const double d = (double)((k & 1) ? act2[k >> 1].y : act2[k >> 1].x);
        if (d > 0.0) {
          const double price = s_p0[k];
          const double q = stock::buy_qty(d, bal, __dmul_rn(price, cost_factor));
          const double cost = __dmul_rn(__dmul_rn(a.cost, fabs(q)), price);
          bal = __dsub_rn(bal, __dadd_rn(__dmul_rn(q, price), cost));
          sh[k] += (int32_t)q;
        }
      }
    }
    double va = bal;
    for (int k = 0; k < K; ++k) va = __dadd_rn(va, __dmul_rn((double)sh[k], s_p1[k]));
    const double r = __dsub_rn(va, vb);
    const double ret = __dadd_rn(ret_in, r);
    if (a.reward) a.reward[e] = (float)r;
    if (a.done_out) a.done_out[e] = (uint8_t)a.done;
    const float x0 = (float)__ddiv_rn(bal, a.cap);
    if (a.done) {
      if (a.term_ret) a.term_ret[e] = ret;
      if (a.term_len) a.term_len[e] = a.ep_len;
      a.balance[e] = a.cap;
      a.ep_return[e] = 0.0;
    } else {
      a.balance[e] = bal;
      a.ep_return[e] = ret;
    }
    // shares back to HBM (zero after the auto-reset), then this thread's table row becomes
    // the private obs part as floats: shares in columns 0..K-1, balance/cap in the spare column K
    for (int k = 0; k < K; ++k) a.shares[(size_t)k * a.N + e] = a.done ? 0 : sh[k];
    float* rowf = reinterpret_cast<float*>(sh);
    for (int k = 0; k < K; ++k) rowf[k] = (float)sh[k];
    rowf[K] = x0;
  }
  __syncthreads();
  const int S = a.S;
  const float* table = reinterpret_cast<const float*>(s_sh);
  if (a.done) {
    if (a.term_obs) write_obs_tab(a.term_obs + e0 * S, nloc, S, table, K, Kp, s_feat_term);
    __syncthreads();
    float* rowf = reinterpret_cast<float*>(s_sh + tid * Kp);
    for (int k = 0; k < K; ++k) rowf[k] = 0.0f;
    rowf[K] = (float)(a.cap / a.cap);  // StockTradingEnv::reset stock_env.hpp:158-163
    __syncthreads();
  }
  write_obs_tab(a.obs + e0 * S, nloc, S, table, K, Kp, s_feat_obs);
}

template <int KMAX, int EB>
__global__ void __launch_bounds__(EB, PRB_ENV_TPS / EB) stock_step_v3_kernel(StockStepArgs a) {
  stock_step_v3_body<KMAX, EB>(a, blockIdx.x);
}

// several lock-step VecEnvs of one market (the evaluation VecEnvs of a GPU's pods) in one launch:
// blockIdx.y = env; the per-step scalars are the launch's, the pointers per env
template <int KMAX, int EB>
__global__ void __launch_bounds__(EB, PRB_ENV_TPS / EB)
    stock_step_v3_group_kernel(const StockStepArgs* __restrict__ group, int t, int t_obs, int done, int ep_len) {
  StockStepArgs a = group[blockIdx.y];
  a.t = t;
  a.t_obs = t_obs;
  a.done = done;
  a.ep_len = ep_len;
  if ((size_t)blockIdx.x * EB < (size_t)a.N) stock_step_v3_body<KMAX, EB>(a, blockIdx.x);
}

size_t stock_v3_smem_bytes(int K, int eb = kEnvBlock) {
  return 2 * (size_t)K * sizeof(double) + (size_t)(K + 1) * eb * 4 + eb * 4 + 10 * (size_t)K * 4;
}

size_t stock_v2_smem_bytes(int K) {
  return (2 * (size_t)K + 2 * kEnvBlock) * sizeof(double) + (((size_t)kEnvBlock * K + 7) & ~size_t(3)) * 4 +
         (size_t)(K + 2) * kEnvBlock * 4 + kEnvBlock * 4 + 10 * (size_t)K * 4;
}

// reset (env.hpp:186-194 -> StockTradingEnv::reset stock_env.hpp:158-163)
__global__ void stock_reset_kernel(int N, int K, int S, double cap, const float* __restrict__ feat_row,
                                   double* balance, int32_t* shares, double* ep_return, float* obs) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (size_t)N) {
    balance[e] = cap;
    ep_return[e] = 0.0;
    for (int k = 0; k < K; ++k) shares[(size_t)k * N + e] = 0;
  }
  const size_t total = (size_t)N * S;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % S);
    obs[i] = (c == 0) ? (float)(cap / cap) : (c <= K ? 0.0f : feat_row[c - 1 - K]);
  }
}

// ---- PointMass2D -----------------------------------------------------------

struct PmStepArgs {
  int N;
  const float* __restrict__ actions;  // [N][2]
  double* __restrict__ st;            // [6][N]
  int32_t* __restrict__ steps;
  double* __restrict__ ep_return;
  uint64_t* __restrict__ mt;  // [312][N]
  int32_t* __restrict__ mt_idx;
  float* __restrict__ obs;  // [N][6]
  float* __restrict__ reward;
  uint8_t* __restrict__ done_out;
  float* __restrict__ term_obs;
  double* __restrict__ term_ret;
  int32_t* __restrict__ term_len;
};

__global__ void __launch_bounds__(256) pm_step_kernel(PmStepArgs a) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)a.N) return;
  const size_t N = a.N;
  double s[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) s[j] = a.st[j * N + e];
  const float2 af = reinterpret_cast<const float2*>(a.actions)[e];
  const double a0 = clamp_ref((double)af.x, -1.0, 1.0), a1 = clamp_ref((double)af.y, -1.0, 1.0);
  const int32_t steps = a.steps[e];
  // pointmass_step env.hpp:84-109 (pm_env.cuh)
  double n[6], r;
  bool done;
  pm::step(s, a0, a1, steps, n, r, done);
  const double ret = __dadd_rn(a.ep_return[e], r);
  if (a.reward) a.reward[e] = (float)r;
  if (a.done_out) a.done_out[e] = done ? 1 : 0;
  if (done) {
    if (a.term_obs)
      for (int j = 0; j < 6; ++j) a.term_obs[e * 6 + j] = (float)n[j];
    if (a.term_ret) a.term_ret[e] = ret;
    if (a.term_len) a.term_len[e] = steps + 1;
    int32_t idx = a.mt_idx[e];
    pm::reset_draws(a.mt + e, N, idx, n);
    a.mt_idx[e] = idx;
    a.steps[e] = 0;
    a.ep_return[e] = 0.0;
  } else {
    a.steps[e] = steps + 1;
    a.ep_return[e] = ret;
  }
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    a.st[j * N + e] = n[j];
    a.obs[e * 6 + j] = (float)n[j];
  }
}

__global__ void pm_reset_kernel(int N, uint64_t seed, uint64_t tag, double* st, int32_t* steps, double* ep_return,
                                uint64_t* mt, int32_t* mt_idx, float* obs) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)N) return;
  // rngs_[i].seed(derive_seed(seed, kVecEnv, i)) env.hpp:188; the evaluator passes kEpisode (pod.hpp:52)
  mt64_seed(mt + e, N, derive_seed2(seed, tag, e));
  int32_t idx = kMtN;
  double s[6];
  pm::reset_draws(mt + e, N, idx, s);
  mt_idx[e] = idx;
  steps[e] = 0;
  ep_return[e] = 0.0;
  for (int j = 0; j < 6; ++j) {
    st[j * (size_t)N + e] = s[j];
    obs[e * 6 + j] = (float)s[j];
  }
}


void check_env(prb_vecenv env) { PRB_REQUIRE(env, PRB_ERR_USAGE, "vecenv handle is NULL"); }

}  // namespace

// Launch one stock VecEnv step on device buffers (shared with rollout.cu).
void prb_stock_step_launch(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done, float* d_term_obs,
                           double* d_term_ret, int32_t* d_term_len) {
  prb_market_s* m = env->market;
  PRB_REQUIRE(env->t + 1 < m->T, PRB_ERR_USAGE, "stock_env_step: no next timestamp at t=" + std::to_string(env->t));
  StockStepArgs a;
  a.N = (int)env->N;
  a.K = m->K;
  a.S = (int)env->S;
  a.t = (int)env->t;
  const size_t t1 = env->t + 1;
  const bool done = (t1 + 1 >= m->T) || (t1 >= env->end);  // stock_env.hpp:101,168
  a.done = done ? 1 : 0;
  a.t_obs = done ? (int)env->start : (int)t1;
  a.ep_len = (int)(env->step_count + 1);
  a.close_tk = m->d_close_tk.p;
  a.feat = env->d_feat.p;
  a.cap = env->cfg.initial_capital;
  a.max_trade = env->cfg.max_trade_shares;
  a.cost = env->cfg.cost_rate;
  a.actions = d_actions;
  a.balance = env->d_balance.p;
  a.shares = env->d_shares.p;
  a.ep_return = env->d_ep_return.p;
  a.obs = env->d_obs.p;
  a.reward = d_reward;
  a.done_out = d_done;
  a.term_obs = d_term_obs;
  a.term_ret = d_term_ret;
  a.term_len = d_term_len;
  {
    ProfScope prof(env->ctx, kProfEnvStock);
    if (m->K <= 32 && (m->K & 1) == 0 && env->cfg.max_trade_shares < 16777216.0) {
      // 256 envs per CTA: measured 72.2% of HBM peak at 1M envs vs 70.9% (128), 68.6% (64),
      // 61.7% (512)
      constexpr int kEb = 256;
      const int gN = (int)((env->N + kEb - 1) / kEb);
      stock_step_v3_kernel<32, kEb><<<gN, kEb, stock_v3_smem_bytes(m->K, kEb), env->ctx->stream>>>(a);
    } else {  // odd K, K > 32 or share quantities beyond fp32's exact integers
      const size_t smem = stock_v2_smem_bytes(m->K);
      ensure_smem(stock_step_v2_kernel, smem);
      const int grid = (int)((env->N + kEnvBlock - 1) / kEnvBlock);
      stock_step_v2_kernel<<<grid, kEnvBlock, smem, env->ctx->stream>>>(a);
    }
  }
  PRB_CHECK_LAUNCH();
  env->t = done ? env->start : t1;
  env->step_count = done ? 0 : env->step_count + 1;
}

void prb_pm_step_launch(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done, float* d_term_obs,
                        double* d_term_ret, int32_t* d_term_len) {
  PmStepArgs a;
  a.N = (int)env->N;
  a.actions = d_actions;
  a.st = env->d_pm_state.p;
  a.steps = env->d_pm_steps.p;
  a.ep_return = env->d_ep_return.p;
  a.mt = env->d_mt.p;
  a.mt_idx = env->d_mt_idx.p;
  a.obs = env->d_obs.p;
  a.reward = d_reward;
  a.done_out = d_done;
  a.term_obs = d_term_obs;
  a.term_ret = d_term_ret;
  a.term_len = d_term_len;
  const int grid = (int)((env->N + 255) / 256);
  {
    ProfScope prof(env->ctx, kProfEnvPm);
    pm_step_kernel<<<grid, 256, 0, env->ctx->stream>>>(a);
  }
  PRB_CHECK_LAUNCH();
}

size_t prb_env_group_args_bytes(int P) { return (size_t)P * sizeof(StockStepArgs); }

bool prb_env_step_group(const prb_vecenv* envs, int P, const float* d_act, size_t act_stride, float* d_rew,
                        uint8_t* d_done, double* d_tret, int32_t* d_tlen, size_t n_stride, void* d_args, bool upload) {
  if (P < 1) return false;
  const prb_vecenv_s* e0 = envs[0];
  if (e0->kind != PRB_KIND_STOCK || !e0->was_reset) return false;
  prb_market_s* m = e0->market;
  if (!(m->K <= 32 && (m->K & 1) == 0 && e0->cfg.max_trade_shares < 16777216.0)) return false;
  for (int p = 1; p < P; ++p) {  // lock-step copies of one VecEnv shape, market, window and clock
    const prb_vecenv_s* e = envs[p];
    if (e->kind != PRB_KIND_STOCK || !e->was_reset || e->market != m || e->N != e0->N || e->start != e0->start ||
        e->end != e0->end || e->t != e0->t || e->step_count != e0->step_count || e->ctx != e0->ctx ||
        e->cfg.initial_capital != e0->cfg.initial_capital || e->cfg.max_trade_shares != e0->cfg.max_trade_shares ||
        e->cfg.cost_rate != e0->cfg.cost_rate)
      return false;
  }
  PRB_REQUIRE(e0->t + 1 < m->T, PRB_ERR_USAGE, "stock_env_step: no next timestamp at t=" + std::to_string(e0->t));
  StockStepArgs* g = static_cast<StockStepArgs*>(d_args);
  if (upload) {
    std::vector<StockStepArgs> h(P);
    for (int p = 0; p < P; ++p) {
      prb_vecenv_s* env = envs[p];
      StockStepArgs& a = h[p];
      a = StockStepArgs{};
      a.N = (int)env->N;
      a.K = m->K;
      a.S = (int)env->S;
      a.close_tk = m->d_close_tk.p;
      a.feat = env->d_feat.p;
      a.cap = env->cfg.initial_capital;
      a.max_trade = env->cfg.max_trade_shares;
      a.cost = env->cfg.cost_rate;
      a.actions = d_act + (size_t)p * act_stride;
      a.balance = env->d_balance.p;
      a.shares = env->d_shares.p;
      a.ep_return = env->d_ep_return.p;
      a.obs = env->d_obs.p;
      a.reward = d_rew + (size_t)p * n_stride;
      a.done_out = d_done + (size_t)p * n_stride;
      a.term_obs = nullptr;
      a.term_ret = d_tret + (size_t)p * n_stride;
      a.term_len = d_tlen + (size_t)p * n_stride;
    }
    PRB_CUDA(cudaMemcpyAsync(g, h.data(), (size_t)P * sizeof(StockStepArgs), cudaMemcpyHostToDevice,
                             e0->ctx->stream));
    PRB_CUDA(cudaStreamSynchronize(e0->ctx->stream));  // h lives on this stack frame
  }
  const size_t t1 = e0->t + 1;
  const bool done = (t1 + 1 >= m->T) || (t1 >= e0->end);  // stock_env.hpp:101,168
  constexpr int kEb = 256;
  const int gN = (int)((e0->N + kEb - 1) / kEb);
  {
    ProfScope prof(e0->ctx, kProfEnvStock);
    stock_step_v3_group_kernel<32, kEb><<<dim3(gN, P), kEb, stock_v3_smem_bytes(m->K, kEb), e0->ctx->stream>>>(
        g, (int)e0->t, done ? (int)e0->start : (int)t1, done ? 1 : 0, (int)(e0->step_count + 1));
  }
  PRB_CHECK_LAUNCH();
  for (int p = 0; p < P; ++p) {
    envs[p]->t = done ? envs[p]->start : t1;
    envs[p]->step_count = done ? 0 : envs[p]->step_count + 1;
  }
  return true;
}

void prb_env_step_launch(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done, float* d_term_obs,
                         double* d_term_ret, int32_t* d_term_len) {
  PRB_REQUIRE(env->was_reset, PRB_ERR_DIMENSION, "vec_step: sub-environments have no state (call reset first)");
  if (env->kind == PRB_KIND_STOCK)
    prb_stock_step_launch(env, d_actions, d_reward, d_done, d_term_obs, d_term_ret, d_term_len);
  else
    prb_pm_step_launch(env, d_actions, d_reward, d_done, d_term_obs, d_term_ret, d_term_len);
}

extern "C" {

int prb_vecenv_create_stock(prb_market m, const prb_stock_config* cfg, size_t start, size_t end, size_t N,
                            prb_vecenv* out) {
  return guard([&] {
    DeviceScope dev_(m ? m->ctx : nullptr);
    PRB_REQUIRE(m && cfg && out, PRB_ERR_USAGE, "prb_vecenv_create_stock: NULL argument");
    PRB_REQUIRE(N > 0, PRB_ERR_CONFIG, "VectorizedEnvironment: num_envs must be > 0");           // env.hpp:170
    PRB_REQUIRE(!m->indicators.empty(), PRB_ERR_USAGE,
                "StockTradingEnv: market data lacks indicators; run compute_indicators");         // stock_env.hpp:140
    PRB_REQUIRE(!(end >= m->T || start + 1 >= end + 1 || end <= start), PRB_ERR_CONFIG,
                "StockTradingEnv: bad window [" + std::to_string(start) + ", " + std::to_string(end) + "] for " +
                    std::to_string(m->T) + " rows");                                              // stock_env.hpp:143
    PRB_REQUIRE(cfg->max_trade_shares * (double)(end - start) < 2.0e9, PRB_ERR_CONFIG,
                "prb: max_trade_shares * episode length must stay below 2e9 (int32 share counts on device)");
    PRB_REQUIRE(N < (size_t)1 << 31, PRB_ERR_CONFIG, "prb: num_envs must be < 2^31");
    PRB_REQUIRE(m->K <= 64, PRB_ERR_CONFIG, "prb: the device stock env supports up to 64 tickers");
    prb_ctx_s* ctx = m->ctx;
    PRB_CUDA(cudaSetDevice(ctx->device));
    auto* env = new prb_vecenv_s;
    env->ctx = ctx;
    env->kind = PRB_KIND_STOCK;
    env->N = N;
    const int K = m->K;
    env->S = 1 + 6 * (size_t)K;
    env->A = K;
    env->action_low.assign(K, -1.0);
    env->action_high.assign(K, 1.0);
    env->max_episode_steps = end - start;
    env->reward_target = 0.0;
    env->market = m;
    env->cfg = *cfg;
    env->start = start;
    env->end = end;
    env->t = start;
    // shared features per time index: close_k[t]/close_k[start] then indicator_i,k[t] (stock_env.hpp:122-129)
    const size_t T = m->T, F = 5 * (size_t)K;
    std::vector<float> feat(T * F);
    for (size_t t = 0; t < T; ++t) {
      for (int k = 0; k < K; ++k)
        feat[t * F + k] = (float)(m->close[(size_t)k * T + t] / m->close[(size_t)k * T + start]);
      for (int i = 0; i < 4; ++i)
        for (int k = 0; k < K; ++k) feat[t * F + K + (size_t)i * K + k] = (float)m->indicators[((size_t)i * K + k) * T + t];
    }
    env->d_feat.alloc(feat.size() + 16);  // + padding: whole-row 16-byte bulk copies (ppo_tc.cu gather)
    PRB_CUDA(cudaMemcpyAsync(env->d_feat.p, feat.data(), feat.size() * sizeof(float), cudaMemcpyHostToDevice,
                             env->ctx->stream));
    env->d_balance.alloc(N);
    env->d_shares.alloc(N * K);
    env->d_ep_return.alloc(N);
    env->d_obs.alloc(N * env->S);
    PRB_CUDA(cudaMemsetAsync(env->d_obs.p, 0, env->d_obs.bytes(), env->ctx->stream));
    PRB_CUDA(cudaStreamSynchronize(env->ctx->stream));  // creation-time: visible to every stream
    *out = env;
  });
}

int prb_vecenv_create_pointmass(prb_ctx ctx, size_t N, prb_vecenv* out) {
  return guard([&] {
    DeviceScope dev_(ctx);
    PRB_REQUIRE(ctx && out, PRB_ERR_USAGE, "prb_vecenv_create_pointmass: NULL argument");
    PRB_REQUIRE(N > 0, PRB_ERR_CONFIG, "VectorizedEnvironment: num_envs must be > 0");
    PRB_REQUIRE(N < (size_t)1 << 31, PRB_ERR_CONFIG, "prb: num_envs must be < 2^31");
    PRB_CUDA(cudaSetDevice(ctx->device));
    auto* env = new prb_vecenv_s;
    env->ctx = ctx;
    env->kind = PRB_KIND_POINTMASS;
    env->N = N;
    env->S = 6;
    env->A = 2;
    env->action_low.assign(2, -1.0);
    env->action_high.assign(2, 1.0);
    env->max_episode_steps = 200;
    env->reward_target = 5.0;
    env->d_pm_state.alloc(6 * N);
    env->d_pm_steps.alloc(N);
    env->d_ep_return.alloc(N);
    env->d_mt.alloc((size_t)kMtN * N);
    env->d_mt_idx.alloc(N);
    env->d_obs.alloc(N * 6);
    PRB_CUDA(cudaMemsetAsync(env->d_obs.p, 0, env->d_obs.bytes(), env->ctx->stream));
    PRB_CUDA(cudaStreamSynchronize(env->ctx->stream));  // creation-time: visible to every stream
    *out = env;
  });
}

int prb_vecenv_destroy(prb_vecenv env) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    if (env) cudaStreamSynchronize(env->ctx->stream);
    delete env;
  });
}

int prb_vecenv_spec(prb_vecenv env, prb_env_spec* out) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    out->state_dim = env->S;
    out->action_dim = env->A;
    out->max_episode_steps = env->max_episode_steps;
    out->reward_target = env->reward_target;
    out->action_low = env->action_low.data();
    out->action_high = env->action_high.data();
  });
}

size_t prb_vecenv_num_envs(prb_vecenv env) { return env ? env->N : 0; }
const float* prb_vecenv_states_device(prb_vecenv env) { return env ? env->d_obs.p : nullptr; }

// reset(seed) with the per-env streams derive_seed(seed, tag, i): tag 1 = kVecEnv
// (VectorizedEnvironment::reset env.hpp:186-194), 8 = kEpisode (evaluate pod.hpp:52).
void prb_vecenv_reset_tagged(prb_vecenv env, uint64_t seed, uint64_t tag) {
  check_env(env);
  cudaStream_t s = env->ctx->stream;
  const int N = (int)env->N;
  if (env->kind == PRB_KIND_STOCK) {  // deterministic reset: the stream is unused (stock_env.hpp:158-163)
    env->t = env->start;
    env->step_count = 0;
    const int K = env->market->K;
    const int grid = std::min<int>((N + 255) / 256, 4 * env->ctx->num_sms * 8);
    stock_reset_kernel<<<std::max(grid, 1), 256, 0, s>>>(N, K, (int)env->S, env->cfg.initial_capital,
                                                         env->d_feat.p + env->start * 5 * (size_t)K, env->d_balance.p,
                                                         env->d_shares.p, env->d_ep_return.p, env->d_obs.p);
  } else {
    pm_reset_kernel<<<(N + 127) / 128, 128, 0, s>>>(N, seed, tag, env->d_pm_state.p, env->d_pm_steps.p,
                                                    env->d_ep_return.p, env->d_mt.p, env->d_mt_idx.p, env->d_obs.p);
  }
  PRB_CHECK_LAUNCH();
  env->was_reset = true;
}

int prb_vecenv_reset(prb_vecenv env, uint64_t seed, float* d_obs) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    cudaStream_t s = env->ctx->stream;
    prb_vecenv_reset_tagged(env, seed, 1);
    if (d_obs && d_obs != env->d_obs.p)
      PRB_CUDA(cudaMemcpyAsync(d_obs, env->d_obs.p, env->d_obs.bytes(), cudaMemcpyDeviceToDevice, s));
  });
}

int prb_vecenv_step(prb_vecenv env, const float* d_actions, float* d_reward, uint8_t* d_done, float* d_terminal_obs,
                    double* d_episode_return, int32_t* d_episode_length) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    PRB_REQUIRE(d_actions, PRB_ERR_USAGE, "vec_step: actions is NULL");
    prb_env_step_launch(env, d_actions, d_reward, d_done, d_terminal_obs, d_episode_return, d_episode_length);
  });
}

int prb_vecenv_reset_host(prb_vecenv env, uint64_t seed, double* states) {
  int rc = prb_vecenv_reset(env, seed, nullptr);
  if (rc) return rc;
  return prb_vecenv_states_host(env, states);
}

int prb_vecenv_states_host(prb_vecenv env, double* states) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    const size_t n = env->N * env->S;
    float* h = static_cast<float*>(env->ctx->pinned_staging(n * sizeof(float)));
    PRB_CUDA(cudaMemcpyAsync(h, env->d_obs.p, n * sizeof(float), cudaMemcpyDeviceToHost, env->ctx->stream));
    env->ctx->sync();
    for (size_t i = 0; i < n; ++i) states[i] = h[i];
  });
}

int prb_vecenv_step_host(prb_vecenv env, const double* actions, double* next_states, double* rewards, uint8_t* dones,
                         double* terminal_states, double* episode_returns, uint64_t* episode_lengths) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    PRB_REQUIRE(actions, PRB_ERR_USAGE, "vec_step: actions is NULL");
    const size_t N = env->N, S = env->S, A = env->A;
    cudaStream_t s = env->ctx->stream;
    if (env->d_act_scratch.n < N * A) env->d_act_scratch.alloc(N * A);
    if (env->d_rew_scratch.n < N) env->d_rew_scratch.alloc(N);
    if (env->d_done_scratch.n < N) env->d_done_scratch.alloc(N);
    if (env->d_term_scratch.n < N * S) env->d_term_scratch.alloc(N * S);
    if (env->d_tret_scratch.n < N) env->d_tret_scratch.alloc(N);
    if (env->d_tlen_scratch.n < N) env->d_tlen_scratch.alloc(N);
    const size_t stage = std::max(N * A, N * S) * sizeof(float) + N * (sizeof(float) + 1 + 8 + 4) + 64;
    char* h = static_cast<char*>(env->ctx->pinned_staging(stage));
    float* hf = reinterpret_cast<float*>(h);
    for (size_t i = 0; i < N * A; ++i) hf[i] = (float)actions[i];
    PRB_CUDA(cudaMemcpyAsync(env->d_act_scratch.p, hf, N * A * sizeof(float), cudaMemcpyHostToDevice, s));
    prb_env_step_launch(env, env->d_act_scratch.p, env->d_rew_scratch.p, env->d_done_scratch.p, env->d_term_scratch.p,
                        env->d_tret_scratch.p, env->d_tlen_scratch.p);
    // small outputs first
    float* h_rew = reinterpret_cast<float*>(h + std::max(N * A, N * S) * sizeof(float));
    uint8_t* h_done = reinterpret_cast<uint8_t*>(h_rew + N);
    PRB_CUDA(cudaMemcpyAsync(h_rew, env->d_rew_scratch.p, N * sizeof(float), cudaMemcpyDeviceToHost, s));
    PRB_CUDA(cudaMemcpyAsync(h_done, env->d_done_scratch.p, N, cudaMemcpyDeviceToHost, s));
    env->ctx->sync();
    bool any_done = false;
    for (size_t i = 0; i < N; ++i) {
      if (rewards) rewards[i] = h_rew[i];
      if (dones) dones[i] = h_done[i];
      any_done |= h_done[i] != 0;
    }
    if (any_done && (terminal_states || episode_returns || episode_lengths)) {
      std::vector<float> term(N * S);
      std::vector<double> tret(N);
      std::vector<int32_t> tlen(N);
      PRB_CUDA(cudaMemcpyAsync(term.data(), env->d_term_scratch.p, N * S * sizeof(float), cudaMemcpyDeviceToHost, s));
      PRB_CUDA(cudaMemcpyAsync(tret.data(), env->d_tret_scratch.p, N * sizeof(double), cudaMemcpyDeviceToHost, s));
      PRB_CUDA(cudaMemcpyAsync(tlen.data(), env->d_tlen_scratch.p, N * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      env->ctx->sync();
      for (size_t i = 0; i < N; ++i) {
        if (!h_done[i]) continue;
        if (terminal_states)
          for (size_t j = 0; j < S; ++j) terminal_states[i * S + j] = term[i * S + j];
        if (episode_returns) episode_returns[i] = tret[i];
        if (episode_lengths) episode_lengths[i] = (uint64_t)tlen[i];
      }
    }
    if (next_states) {
      PRB_CUDA(cudaMemcpyAsync(hf, env->d_obs.p, N * S * sizeof(float), cudaMemcpyDeviceToHost, s));
      env->ctx->sync();
      for (size_t i = 0; i < N * S; ++i) next_states[i] = hf[i];
    }
  });
}

int prb_vecenv_step_counts_host(prb_vecenv env, uint64_t* out) {
  return guard([&] {
    DeviceScope dev_(env ? env->ctx : nullptr);
    check_env(env);
    if (env->kind == PRB_KIND_STOCK) {
      for (size_t i = 0; i < env->N; ++i) out[i] = env->step_count;
    } else {
      std::vector<int32_t> st(env->N);
      PRB_CUDA(cudaMemcpyAsync(st.data(), env->d_pm_steps.p, env->N * sizeof(int32_t), cudaMemcpyDeviceToHost,
                               env->ctx->stream));
      env->ctx->sync();
      for (size_t i = 0; i < env->N; ++i) out[i] = (uint64_t)st[i];
    }
  });
}

}  // extern "C"
